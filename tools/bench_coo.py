"""SparseCoo canonicalization (§8 row a1) at scale: shuffled triplets of 3-D Poisson N^3,
host path (sparsla_coo_canonicalize, all host threads) vs the GPU path
(sparsla_coo_canonicalize_device, host buffers: the copies are inside the timing).
The survey's probe timed the reference's own single-threaded SparseCoo at 12.2 s for
N = 256 (117M entries).  Usage: python tools/bench_coo.py [N ...]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_13994_b200 import sparsla as S  # noqa: E402


def main():
    for N in [int(a) for a in sys.argv[1:]] or [256]:
        A = S.generate("poisson3d", N)
        n, nnz = A.nrows, A.nnz
        perm = np.random.default_rng(2601).permutation(nnz)
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(A.row_ptr))[perm]
        cols = A.col_idx[perm].copy()
        vals = A.vals[perm].copy()
        S.SparseCoo(rows[:1000], cols[:1000], vals[:1000], (n, n), device=0)  # warm-up
        t0 = time.perf_counter()
        g = S.SparseCoo(rows, cols, vals, (n, n), device=0)
        tg = time.perf_counter() - t0
        t0 = time.perf_counter()
        h = S.SparseCoo(rows, cols, vals, (n, n))
        th = time.perf_counter() - t0
        ok = (np.array_equal(g.rows, h.rows) and np.array_equal(g.cols, h.cols)
              and np.array_equal(g.vals.view(np.int64), h.vals.view(np.int64)))
        print(json.dumps({"case": f"poisson3d N={N} shuffled", "nnz": nnz, "gpu_s": tg, "host_s": th,
                          "host_threads": os.cpu_count(), "bitwise_equal": bool(ok),
                          "gpu_entries_per_s": nnz / tg}), flush=True)


if __name__ == "__main__":
    main()
