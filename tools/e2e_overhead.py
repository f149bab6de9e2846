"""Fixed costs of one sparsla_cg_solve call at config B (host buffers): max_iter = 1 and a
full solve, wall-clock, pinned b / x."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_13994_b200 import sparsla as S  # noqa: E402

nr, n, rp, ci, v = S.generate_i32("poisson3d", 464, 0)
D = S.DeviceCsr(None, 0, i32=(n, n, rp, ci, v))
b = torch.ones(n, dtype=torch.float64).pin_memory()
x = torch.empty(n, dtype=torch.float64).pin_memory()
lib = S.lib()
for mi in (1, 1, 10, 100000):
    o = S.SolveOptions(atol=0.0, rtol=1e-8, max_iter=mi).c()
    rep = S._Report()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S._check(lib.sparsla_cg_solve(D.h, C.cast(b.data_ptr(), S._f64p), C.cast(x.data_ptr(), S._f64p), C.byref(o),
                                  C.byref(rep), C.c_int32(0)))
    print(mi, rep.iterations, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
