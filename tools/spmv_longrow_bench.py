"""Long-row (power-law hub) SpMV on one B200: warp-per-row split vs the staged kernel's hub
bypass.  1M-row matrix, Pareto row degrees + hub rows of 1e4..1e5 entries (symmetric,
diagonally dominant).  The SpMV is timed inside the CG loop (kernel_times: the SpMV point =
long-row kernel + staged kernel on the short-row view, CUDA events on the solver stream);
bytes = 12 nnz + 4 (n+1) + 24 n (gathered x once, q written, p read for p.q).

    python tools/spmv_longrow_bench.py [n] [threshold ...]   (thresholds: auto | <entries> | 0 = off;
                                                             default: auto 0)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import pyoracle as O  # noqa: E402
from paper_2601_13994_b200 import sparsla as S  # noqa: E402
from test_gpu_parity import power_law_csr  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    O.set_threads(os.cpu_count() or 1)
    t0 = time.time()
    hubs = [100_000, 50_000] + [20_000] * 3 + [10_000] * 10
    A = power_law_csr(O, n, 2601, hubs)
    tgen = time.time() - t0
    lens = np.diff(A.row_ptr)
    x = np.random.default_rng(1).standard_normal(n)
    yref = O.spmv(A, x)
    b = np.ones(n)
    thrs = [None if t == "auto" else t for t in sys.argv[2:]] or [None, "0"]
    for thr in thrs:
        if thr is None:
            os.environ.pop("SPARSLA_LONG_ROW", None)
        else:
            os.environ["SPARSLA_LONG_ROW"] = thr
        D = S.CsrMatrix(A.nrows, A.ncols, A.row_ptr, A.col_idx, A.vals).device(0)
        ok = np.array_equal(S.spmv(D, x).view(np.int64), yref.view(np.int64))
        sv = S.Solver(D, b, "cg", S.SolveOptions(atol=0.0, rtol=1e-30, max_iter=100000))
        sv.reset()
        sv.iterate(3)
        kms = sv.kernel_times(50)
        sv.close()
        byt = 12 * A.nnz + 4 * (n + 1) + 24 * n
        lr = D.long_rows()
        print(json.dumps({"n": n, "nnz": int(A.nnz), "threshold_env": thr or "auto", "max_row": int(lens.max()), "p99_row": float(np.percentile(lens, 99)),
                          "long_rows": lr, "mode": "warp-per-row split" if lr["rows"] else "staged + hub bypass",
                          "spmv_ms": kms[0], "spmv_gbs": byt / (kms[0] * 1e-3) / 1e9,
                          "frac": byt / (kms[0] * 1e-3) / 1e9 / PEAK, "bitwise_vs_oracle": bool(ok),
                          "cg_update_ms": kms[1:], "generate_s": tgen}), flush=True)
        D.close()


if __name__ == "__main__":
    main()
