"""A few Krylov iterations of one config (for ncu captures of the SpMV / vector kernels).
    python tools/spmv_profile.py [kind] [N] [backend] [fparam] [p2]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_13994_b200 import sparsla as S  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "poisson3d"
p1 = int(sys.argv[2]) if len(sys.argv) > 2 else 464
backend = sys.argv[3] if len(sys.argv) > 3 else "cg"
fp = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
p2 = int(sys.argv[5]) if len(sys.argv) > 5 else (2601 if kind == "fem2d" else 0)
nr, n, rp, ci, v = S.generate_i32(kind, p1, p2, fp)
D = S.DeviceCsr(None, 0, i32=(n, n, rp, ci, v))
sv = S.Solver(D, np.ones(n), backend, S.SolveOptions(atol=0.0, rtol=1e-30, max_iter=10**6))
sv.iterate(3)
print(sv.kernel_times(2), D.format())
