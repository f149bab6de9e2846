"""Secondary measurement: every BASELINE.json config on one B200 (device-resident data).

For each config: generate on the host, upload, solve to tolerance through the persistent
solver (CUDA-graph loop), report iterations, time to tolerance, it/s, per-kernel times and
GB/s against the canonical bytes/iteration; config C adds the adjoint backward (one
transposed solve + gradient gather).  Prints one JSON object per config.

  python tools/bench_configs.py [A C D E] [--fem-m 4474]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_13994_b200 import sparsla as S  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def solve_cfg(name, kind, p1, p2, fp, backend, rtol, extra=None):
    t0 = time.time()
    nr, n, rp, ci, v = S.generate_i32(kind, p1, p2, fp)
    tgen = time.time() - t0
    nnz = int(rp[-1])
    D = S.DeviceCsr(None, 0, i32=(n, n, rp, ci, v))
    b = np.ones(n)
    opts = S.SolveOptions(atol=0.0, rtol=rtol, max_iter=200000)
    sv = S.Solver(D, b, backend, opts)
    import torch
    stream = torch.cuda.ExternalStream(sv.stream())
    sv.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sv.run()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    rep = sv.report()
    sv.reset()
    sv.iterate(3)
    kms = sv.kernel_times(10)
    fmt = D.format()
    mat = 5 * nnz + 2048 if fmt["value_dict"] else 12 * nnz  # stored matrix stream per SpMV
    dn = 0 if fmt["uniform_diag"] else 8 * n                  # one streamed-diagonal read
    if backend == "cg":
        it_bytes = 12 * nnz + 108 * n + 4                     # SURVEY canonical (CSR, 3 passes)
        stored_bytes = mat + 4 * (n + 1) + 16 * n + 32 * n - (8 * n - dn) + 48 * n - (8 * n - dn)
        names = ["spmv_cg", "cg_update1", "cg_update2"]
    else:
        it_bytes = 24 * nnz + 208 * n + 8
        stored_bytes = 2 * mat + 8 * (n + 1) + 208 * n - 2 * (8 * n - dn)
        names = ["bicg_update1", "spmv_v", "bicg_update2", "spmv_t", "bicg_update3"]
    per_it = sum(kms)
    out = {"config": name, "kind": kind, "n": n, "nnz": nnz, "backend": backend, "rtol": rtol,
           "iterations": rep.iterations, "converged": rep.converged, "spmv_count": rep.spmv_count,
           "diagnostic": rep.diagnostic, "residual_norm": rep.residual_norm,
           "time_to_tolerance_s": ms / 1e3, "it_per_s": rep.iterations / (ms / 1e3),
           "kernel_ms": dict(zip(names, kms)), "bytes_per_iteration": it_bytes,
           "iteration_gbs_from_kernels": it_bytes / (per_it * 1e-3) / 1e9,
           "iteration_frac_of_measured_peak": it_bytes / (per_it * 1e-3) / 1e9 / PEAK,
           "iteration_gbs_wall": it_bytes * rep.iterations / (ms * 1e-3) / 1e9,
           "format": fmt, "stored_bytes_per_iteration": stored_bytes,
           "stored_iteration_frac_of_measured_peak": stored_bytes / (per_it * 1e-3) / 1e9 / PEAK,
           "generate_s": tgen, "device_info": D.info()}
    if extra:
        out.update(extra(D, sv, n, nnz, opts))
    sv.close()
    D.close()
    return out


def adjoint_extra(D, sv, n, nnz, opts):
    """config C: forward x, then one adjoint solve with g = ones (L = sum x) + gather."""
    import ctypes as C
    import torch
    sv.reset()
    sv.run()
    x = sv.x()
    g = np.ones(n)
    gb = np.empty(n)
    gv = np.empty(nnz)
    rep = S._Report()
    o = opts.c()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S._check(S.lib().sparsla_adjoint_backward(D.h, S._p(x, S._f64p), S._p(g, S._f64p), C.c_int32(0),
                                              C.byref(o), S._p(gb, S._f64p), S._p(gv, S._f64p),
                                              C.byref(rep), C.c_int32(S.MEM_HOST)))
    dt = time.perf_counter() - t0
    r = S.SolveReport._from(rep)
    return {"adjoint": {"iterations": r.iterations, "converged": r.converged, "wall_s_host_io": dt,
                        "grad_b_norm": float(np.linalg.norm(gb)), "grad_vals_absmax": float(np.abs(gv).max())}}


def main():
    want = [a for a in sys.argv[1:] if not a.startswith("--") and not a.isdigit()] or ["A", "C", "D", "D01", "E"]
    m = 4474
    if "--fem-m" in sys.argv:
        m = int(sys.argv[sys.argv.index("--fem-m") + 1])
    cfgs = {
        "A": ("A: 2-D Poisson 1000^2 (1M DOF)", "poisson2d", 1000, 0, 0.0, "cg", 1e-8, None),
        "C": (f"C: P1 FEM m={m} (~20M DOF) + adjoint", "fem2d", m, 2601, 0.0, "cg", 1e-8, adjoint_extra),
        "D": ("D: 3-D convection-diffusion 368^3 (50M DOF), c=1.0, BiCGStab, 1 GPU", "convdiff3d", 368, 0, 1.0,
              "bicgstab", 1e-8, None),
        "D01": ("D': 3-D convection-diffusion 368^3 (50M DOF), c=0.1, BiCGStab, 1 GPU", "convdiff3d", 368, 0, 0.1,
                "bicgstab", 1e-8, None),
        "E": ("E: 3-D Poisson 368^3 per-GPU slab (50M DOF), P=1", "poisson3d", 368, 0, 0.0, "cg", 1e-8, None),
    }
    for k in want:
        name, kind, p1, p2, fp, be, rtol, ex = cfgs[k]
        print(json.dumps(solve_cfg(name, kind, p1, p2, fp, be, rtol, ex)), flush=True)


if __name__ == "__main__":
    main()
