"""A few CG iterations of config B (for ncu captures of the SpMV / vector kernels)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_13994_b200 import sparsla as S  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "poisson3d"
p1 = int(sys.argv[2]) if len(sys.argv) > 2 else 464
nr, n, rp, ci, v = S.generate_i32(kind, p1, 0)
D = S.DeviceCsr(None, 0, i32=(n, n, rp, ci, v))
sv = S.Solver(D, np.ones(n), "cg", S.SolveOptions(atol=0.0, rtol=1e-30, max_iter=10**6))
sv.iterate(3)
print(sv.kernel_times(2), D.format())
