"""Sweep the value-dictionary SpMV variants (SPARSLA_VD_VARIANT) on one matrix: CG-mode SpMV
time, its stored-format GB/s and the CSR-equivalent GB/s.  Usage: python tools/vd_sweep.py [kind] [p1]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2601_13994_b200 import sparsla as S
kind, p1, p2 = %r, %d, %d
nr, n, rp, ci, v = S.generate_i32(kind, p1, p2)
D = S.DeviceCsr(None, 0, i32=(n, n, rp, ci, v))
nnz = int(rp[-1])
sv = S.Solver(D, np.ones(n), "cg", S.SolveOptions(atol=0.0, rtol=1e-30, max_iter=10**6))
sv.iterate(3)
ms = sv.kernel_times(20)
fmt = D.format()
b = ((1 if fmt["value_dict"] else 8) + (1 if fmt.get("col_dict") else 4)) * nnz + 20 * n + 4
print(json.dumps({"spmv_ms": ms[0], "stored_gbs": b / ms[0] / 1e6, "csr_equiv_gbs": (12 * nnz + 20 * n + 4) / ms[0] / 1e6,
                  "u1_ms": ms[1], "u2_ms": ms[2], "fmt": fmt}))
'''


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "poisson3d"
    p1 = int(sys.argv[2]) if len(sys.argv) > 2 else 464
    p2 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    for v in range(int(os.environ.get("NVAR", "7"))):
        env = dict(os.environ, SPARSLA_VD_VARIANT=str(v))
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, kind, p1, p2)], env=env, capture_output=True,
                             text=True, timeout=600)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
        print(f"vd variant {v}: {line}", flush=True)


if __name__ == "__main__":
    main()
