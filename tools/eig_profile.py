"""Short LOBPCG run for profiling (ncu launch lists): 2-D Poisson N=1000, k=6, 30 iterations."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_13994_b200 import sparsla as S  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
it = int(sys.argv[2]) if len(sys.argv) > 2 else 30
A = S.generate("poisson2d", N)
r = S.eig_smallest(A, 6, tol=1e-8, max_iter=it)
print(r.report.iterations, r.report.diagnostic)
