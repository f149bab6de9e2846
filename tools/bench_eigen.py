"""LOBPCG measurement (SPEC.md:289 eig_smallest; Table 4 'Eigenvalue (k=6)'):
k smallest eigenpairs of large Poisson matrices on one B200, checked against the closed-form
spectrum.  Prints one JSON object per case.

  python tools/bench_eigen.py [2d:1000 3d:128 ...] [--k 6] [--tol 1e-8]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_13994_b200 import sparsla as S  # noqa: E402


def spectrum(dims, N, k):
    t = 2.0 - 2.0 * np.cos(np.pi * np.arange(1, min(N, 8) + 1) / (N + 1))
    s = np.add.outer(t, t) if dims == 2 else np.add.outer(np.add.outer(t, t), t)
    return np.sort(s.ravel())[:k]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    k = int(sys.argv[sys.argv.index("--k") + 1]) if "--k" in sys.argv else 6
    tol = float(sys.argv[sys.argv.index("--tol") + 1]) if "--tol" in sys.argv else 1e-8
    for case in args or ["2d:1000", "3d:128"]:
        dims, N = case.split(":")
        dims, N = int(dims[0]), int(N)
        A = S.generate("poisson2d" if dims == 2 else "poisson3d", N)
        D = A.device(0)
        S.eig_smallest(D, k, tol=1e-2, max_iter=3)  # warm-up (allocations, module load)
        t0 = time.perf_counter()
        r = S.eig_smallest(D, k, tol=tol, max_iter=100000)
        dt = time.perf_counter() - t0
        err = float(np.max(np.abs(r.lambdas - spectrum(dims, N, k))))
        print(json.dumps({"case": f"poisson{dims}d N={N}", "n": A.nrows, "nnz": A.nnz, "k": k, "tol": tol,
                          "iterations": r.report.iterations, "converged": r.report.converged,
                          "time_s": dt, "ms_per_iteration": 1e3 * dt / max(1, r.report.iterations),
                          "spmm_count": r.report.spmm_count, "max_lambda_err_vs_closed_form": err,
                          "max_residual": float(np.max(r.report.residual_norms)),
                          "orthogonality_err": float(np.max(np.abs(r.vectors.T @ r.vectors - np.eye(k))))}),
              flush=True)


if __name__ == "__main__":
    main()
