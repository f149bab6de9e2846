"""A/B of the x-window staged SpMV (csrc/spmv_xw.cuh) against the gather kernels, per config
and kernel variant, on one B200.  Times come from Solver.kernel_times (CUDA events on the
solver stream, inside the Krylov loop); the SpMV bytes are the stored-format bytes of
bench.py (dictionary: 5 B/entry + 2 KB; plain: 12 B/entry) + row_ptr + x + y (+ the fused
dot's operand).  Prints one JSON line per (config, setting).

    python tools/xw_sweep.py [B E D C] [--variants 0,1,2,...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_13994_b200 import sparsla as S  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
XW_STREAM = [1, 1, 1, 0, 0, 0, 2, 2, 2, 1, 2, 0, 2]  # value stream of kXwVariants (device.cu)
CFG = {"B": ("poisson3d", 464, 0, 0.0, "cg"), "E": ("poisson3d", 368, 0, 0.0, "cg"),
       "D": ("convdiff3d", 368, 0, 0.1, "bicgstab"), "C": ("fem2d", 4474, 2601, 0.0, "cg")}


def run(name, arrays, setting, env):
    kind, p1, p2, fp, backend = CFG[name]
    nr, n, rp, ci, v = arrays
    for k in ("SPARSLA_XWIN", "SPARSLA_XW_VARIANT", "SPARSLA_VALUE_DICT", "SPARSLA_XW_PAIR", "SPARSLA_DIA"):
        os.environ.pop(k, None)
    os.environ.update(env)
    D = S.DeviceCsr(None, 0, i32=(n, n, rp, ci, v))
    sv = S.Solver(D, np.ones(n), backend, S.SolveOptions(atol=0.0, rtol=1e-30, max_iter=10**6))
    sv.reset()
    sv.iterate(3)
    ms = sv.kernel_times(30)
    fmt, xw = D.format(), D.xwin()
    nnz = int(rp[-1])
    per_e = 5 if fmt["value_dict"] else 12
    base = per_e * nnz + (2048 if fmt["value_dict"] else 0) + 4 * (n + 1) + 16 * n
    if backend == "cg":
        names, byts = ["spmv_cg", "u1", "u2"], [base + 8 * n, None, None]
    else:
        names = ["u1", "spmv_v", "u2", "spmv_t", "u3"]
        byts = [None, base + 8 * n, None, base + 8 * n, None]
    out = {"config": name, "setting": setting, "format": fmt, "xwin": xw, "dia": D.dia(),
           "ms": dict(zip(names, ms)), "iteration_ms": float(sum(ms))}
    for nm, b, t in zip(names, byts, ms):
        if b:
            out[f"{nm}_frac"] = b / (t * 1e-3) / 1e9 / PEAK
    print(json.dumps(out), flush=True)
    sv.close()
    D.close()


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    variants = None
    for a in sys.argv[1:]:
        if a.startswith("--variants="):
            variants = [int(x) for x in a.split("=")[1].split(",")]
    for name in args or ["B", "E", "D", "C"]:
        kind, p1, p2, fp, backend = CFG[name]
        arrays = S.generate_i32(kind, p1, p2, fp)
        run(name, arrays, "gather", {"SPARSLA_XWIN": "0", "SPARSLA_DIA": "0"})
        run(name, arrays, "xwin-1", {"SPARSLA_XWIN": "1", "SPARSLA_DIA": "0"})
        run(name, arrays, "dia", {"SPARSLA_DIA": "1"})
        for var in variants or []:
            env = {"SPARSLA_XWIN": "2", "SPARSLA_XW_VARIANT": str(var)}
            vs = XW_STREAM[var]
            if vs == 0:
                env["SPARSLA_VALUE_DICT"] = "0"
            env["SPARSLA_XW_PAIR"] = "1" if vs == 2 else "0"
            env["SPARSLA_DIA"] = "0"
            run(name, arrays, f"xwin-v{var}", env)
        if name != "C":  # plain CSR beside the dictionary
            run(name, arrays, "gather-plain", {"SPARSLA_XWIN": "0", "SPARSLA_VALUE_DICT": "0", "SPARSLA_DIA": "0"})
            run(name, arrays, "xwin-plain", {"SPARSLA_XWIN": "1", "SPARSLA_VALUE_DICT": "0", "SPARSLA_DIA": "0"})


if __name__ == "__main__":
    main()
