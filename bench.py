#!/usr/bin/env python
"""bench.py — CG iterations/s and SpMV HBM GB/s on 3-D Poisson (BASELINE.json metric).

Workload (N=1): BASELINE configs[1] = config B, 3-D 7-point Poisson 464^3
(n = 99,897,344, nnz = 697,989,632), fp64, Jacobi-PCG to rel-res 1e-8.  A "step" is one
CG iteration of the hot loop (SpMV + fused p.q, fused x/r update + r.z/r.r, p update;
device-side scalars) with every input resident in HBM; the matrix (8.4 GB) and vectors
exceed the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `e2e` is the same metric through the public C ABI call
sparsla_cg_solve with pinned HOST b and x (H2D/D2H inside the timed region), solved to
tolerance; `roofline` is the dominant kernel (the SpMV) against MEASURED_PEAKS.json;
`cpu_baseline` is the oracle port timed on this host (rank 0, N=1).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CG iters/s & SpMV HBM GB/s, 3D Poisson 100M DOF fp64, 1/2/4/8 B200"
SPEC_PEAK_GBS = 8000.0


def load_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        time.sleep(0.3)
        if self.p:
            self.p.terminate()
            out, _ = self.p.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]
        else:
            self.lines = []

    def summary(self):
        sm, mx, reasons, pw = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


def gen_config(args):
    from paper_2601_13994_b200 import sparsla as S
    t0 = time.time()
    nr, n, rp, ci, v = S.generate_i32("poisson3d", args.size)
    return n, rp, ci, v, time.time() - t0


def iteration_bytes(n, nnz, value_dict=False, uniform_diag=False):
    """Algorithmic bytes of THIS implementation's CG iteration in the storage format the
    library chose (x += a p moved into update 2 so p is streamed once).  Plain CSR:
    12 nnz + 100 n + 4; with the value dictionary the matrix stream is 5 nnz (+ a 2 KB
    table); with a constant Jacobi diagonal the two vector passes skip d (-16 n).
    SURVEY.md's canonical 3-pass CSR accounting, 12 nnz + 108 n + 4, is reported beside it."""
    mat = (5 * nnz + 2048) if value_dict else 12 * nnz
    spmv = mat + 4 * (n + 1) + 8 * n + 8 * n        # matrix, row_ptr, p (once), q write
    u1 = (24 if uniform_diag else 32) * n           # read r q (d), write r
    u2 = (40 if uniform_diag else 48) * n           # read x p r (d), write x p
    return spmv, u1, u2


def cpu_baseline(rp, ci, v, n, nnz, threads, budget_s=20.0):
    """Oracle port (test infrastructure) on this host: per-iteration time of the same CG."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    O.set_threads(threads)
    A = O.Csr(n, n, rp.astype(np.int64), ci.astype(np.int64), v)
    b = np.ones(n)
    t0 = time.perf_counter()
    O.cg_fixed(A, b, 1)
    t1 = time.perf_counter()
    per_guess = max(1e-3, (t1 - t0) / 2.0)
    m = int(max(2, min(20, budget_s / per_guess)))
    t2 = time.perf_counter()
    O.cg_fixed(A, b, 1 + m)
    t3 = time.perf_counter()
    per_it = ((t3 - t2) - (t1 - t0)) / m
    return {"value": 1.0 / per_it, "unit": "it/s", "cores": threads, "kind": "port",
            "sample": f"{m} CG iterations of config B (full 99.9M-DOF matrix) with {threads} host "
                      f"threads, oracle/liboracle.so (SpMV bit-identical to reference sparse.cpp)",
            "s_per_iteration": per_it}


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port of SPEC cg_solve over the
    reference spmv semantics; the reference tree has no solver sources) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n, rp, ci, v, tgen = gen_config(args)
    nnz = int(rp[-1])
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    O.set_threads(threads)
    A = O.Csr(n, n, rp.astype(np.int64), ci.astype(np.int64), v)
    del rp, ci
    b = np.ones(n)
    t0 = time.perf_counter()
    O.cg_fixed(A, b, args.warmup)        # init + W iterations
    t1 = time.perf_counter()
    O.cg_fixed(A, b, args.warmup + args.steps)
    t2 = time.perf_counter()
    per = ((t2 - t1) - (t1 - t0)) / args.steps
    val = 1.0 / per
    line = {"metric": METRIC, "value": val, "unit": "it/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"B: 3-D 7-pt Poisson {args.size}^3 ({n} DOF, nnz {nnz}), "
                                   "Jacobi-PCG rtol 1e-8", "n": n, "nnz": nnz},
            "cpu_baseline": {"value": val, "unit": "it/s", "cores": threads, "kind": "port",
                             "sample": f"{args.steps} timed CG iterations after {args.warmup} warm-up "
                                       "iterations (difference of two oracle runs)"},
            "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    from paper_2601_13994_b200 import sparsla as S
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 or args.gpus > 1 or args.dist:
        from paper_2601_13994_b200 import dist_bench
        return dist_bench.run(args, METRIC)
    dev = 0
    torch.cuda.set_device(dev)
    peak, peak_src = load_peak()
    n, rp, ci, v, tgen = gen_config(args)
    nnz = int(rp[-1])
    t0 = time.time()
    D = S.DeviceCsr(None, dev, i32=(n, n, rp, ci, v))
    tup = time.time() - t0
    info = D.info()
    fmt = D.format()
    b_host = torch.ones(n, dtype=torch.float64).pin_memory()
    x_host = torch.empty(n, dtype=torch.float64).pin_memory()
    opts = S.SolveOptions(atol=0.0, rtol=args.rtol, max_iter=args.max_iter)
    lib = S.lib()
    import ctypes as C

    # ---------------- e2e: public C ABI call, host buffers, solve to tolerance ----------
    # one untimed warm-up call (W iterations): the matrix handle's parked solver workspace
    # and graphs are built there, as in any application that solves more than once
    wo = S.SolveOptions(atol=0.0, rtol=args.rtol, max_iter=max(1, args.warmup)).c()
    S._check(lib.sparsla_cg_solve(D.h, C.cast(b_host.data_ptr(), S._f64p), C.cast(x_host.data_ptr(), S._f64p),
                                  C.byref(wo), C.byref(S._Report()), C.c_int32(S.MEM_HOST)))
    e2e_its, e2e_t, reps = 0, 0.0, []
    for _ in range(max(1, args.e2e_steps)):
        rep = S._Report()
        o = opts.c()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S._check(lib.sparsla_cg_solve(D.h, C.cast(b_host.data_ptr(), S._f64p),
                                      C.cast(x_host.data_ptr(), S._f64p), C.byref(o), C.byref(rep),
                                      C.c_int32(S.MEM_HOST)))
        dt = time.perf_counter() - t0
        reps.append(S.SolveReport._from(rep))
        e2e_its += rep.iterations
        e2e_t += dt
    r0 = reps[0]
    k_tol = r0.iterations
    # correctness gate before reporting: true residual of the GPU solution
    x = x_host.numpy().copy()
    ax = S.spmv(D, x)
    true_rel = float(np.linalg.norm(1.0 - ax) / np.sqrt(n))
    gate_ok = bool(r0.converged and true_rel <= 10 * args.rtol)

    # ---------------- device-resident timed loop -----------------------------------------
    sv = S.Solver(D, b_host.numpy(), "cg", opts)
    stream = torch.cuda.ExternalStream(sv.stream())
    launches = sv.launches_per_iteration()
    budget = max(1, k_tol - 1)  # iterations available before the solve terminates
    done = 0
    resets = 0

    def advance(k):
        nonlocal done, resets
        while k > 0:
            if done >= budget:
                sv.reset()
                resets += 1
                done = 0
            m = min(k, budget - done)
            sv.iterate(m)
            done += m
            k -= m

    sv.reset()
    with ClockSampler(dev) as clk:
        advance(args.warmup)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        resets_before = resets
        e0.record(stream)
        advance(args.steps)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    timed_resets = resets - resets_before
    rep_loop = sv.report()
    value = args.steps / (ms / 1e3)
    # per-kernel durations (CUDA events around each kernel, individual launches)
    sv.reset()
    sv.iterate(5)
    kms = sv.kernel_times(args.kernel_iters)
    spmv_b, u1_b, u2_b = iteration_bytes(n, nnz, fmt["value_dict"], fmt["uniform_diag"])
    it_bytes = spmv_b + u1_b + u2_b
    spmv_gbs = spmv_b / (kms[0] * 1e-3) / 1e9
    sv.close()
    # plain-CSR reference point of the same loop (value dictionary and scalar diagonal off)
    plain = None
    if args.plain_steps > 0:
        os.environ["SPARSLA_VALUE_DICT"] = "0"
        os.environ["SPARSLA_UNIFORM_DIAG"] = "0"
        try:
            Dp = S.DeviceCsr(None, dev, i32=(n, n, rp, ci, v))
            svp = S.Solver(Dp, b_host.numpy(), "cg", opts)
            sp = torch.cuda.ExternalStream(svp.stream())
            svp.reset()
            svp.iterate(5)
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(sp)
            svp.iterate(args.plain_steps)
            q1.record(sp)
            q1.synchronize()
            pms = q0.elapsed_time(q1) / args.plain_steps
            pk = svp.kernel_times(10)
            ps_b, pu1, pu2 = iteration_bytes(n, nnz)
            plain = {"value": 1e3 / pms, "unit": "it/s", "steps": args.plain_steps, "ms_per_step": pms,
                     "kernel_ms": {"spmv_cg": pk[0], "cg_update1": pk[1], "cg_update2": pk[2]},
                     "spmv_gbs": ps_b / (pk[0] * 1e-3) / 1e9,
                     "iteration_gbs": (ps_b + pu1 + pu2) / (pms * 1e-3) / 1e9,
                     "format": "plain CSR (int32 col, fp64 val), streamed Jacobi diagonal"}
            svp.close()
            del Dp
        finally:
            del os.environ["SPARSLA_VALUE_DICT"], os.environ["SPARSLA_UNIFORM_DIAG"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "spmv_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("size") == args.size:
            traffic = tj["value_dict" if fmt["value_dict"] else "plain"]["dram_bytes_per_launch"]
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated 3-D Poisson, b = ones)",
        "config": {"workload": f"B: 3-D 7-pt Poisson {args.size}^3 ({n} DOF, nnz {nnz}), Jacobi-PCG "
                               f"rtol {args.rtol}, x0 = 0", "n": n, "nnz": nnz, "partition": "single GPU",
                   "l2": "no flush: matrix + vectors (>12 GB) exceed the 126 MB L2",
                   "spmv_variant": "tma-bulk-staged" if info["variant"] == 0 else "direct",
                   "storage": ("value dictionary (1-byte index into %d distinct fp64 values) + int32 col"
                               % fmt["distinct_values"]) if fmt["value_dict"] else "CSR int32 col + fp64 val",
                   "jacobi_diag": "constant (scalar)" if fmt["uniform_diag"] else "streamed"},
        "spmv_gbs": spmv_gbs,
        "iteration_gbs": it_bytes / (ms / args.steps * 1e-3) / 1e9,
        "bytes_per_iteration": it_bytes,
        "canonical_bytes_per_iteration": 12 * nnz + 108 * n + 4,
        "canonical_iteration_gbs": (12 * nnz + 108 * n + 4) / (ms / args.steps * 1e-3) / 1e9,
        "kernel_ms": {"spmv_cg": kms[0], "cg_update1": kms[1], "cg_update2": kms[2]},
        "csr_equivalent_spmv_gbs": (12 * nnz + 20 * n + 4) / (kms[0] * 1e-3) / 1e9,
        "plain_csr": plain,
        "roofline": {"bound": "hbm", "kernel": "spmv_ws_kernel<SPMV_CG,staged%s>" % (",value-dict" if fmt["value_dict"] else ""), "achieved": spmv_gbs,
                     "peak": peak, "unit": "GB/s", "frac": spmv_gbs / peak, "traffic": traffic,
                     "peak_source": peak_src, "frac_of_spec_8tbs": spmv_gbs / SPEC_PEAK_GBS,
                     "algorithmic_bytes_per_launch": spmv_b,
                     "bytes_basis": "bytes of the stored format (value dictionary: 5 B/entry)" if fmt["value_dict"]
                                    else "CSR 12 B/entry",
                     "iteration_frac": (it_bytes / (ms / args.steps * 1e-3) / 1e9) / peak},
        "time_to_tolerance_s": e2e_t / len(reps), "iterations_to_tolerance": k_tol,
        "e2e": {"value": e2e_its / e2e_t, "unit": "it/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n + 184, "step": "one sparsla_cg_solve call to rtol "
                f"{args.rtol} with pinned host b/x", "steps": len(reps)},
        "gpu_launches": args.steps * launches + 2 * timed_resets,
        "clocks": clk.summary(),
        "parity_gate": {"converged": r0.converged, "residual_norm": r0.residual_norm,
                        "true_rel_residual": true_rel, "ok": gate_ok},
        "setup_s": {"generate": tgen, "upload": tup},
    }
    if not args.no_cpu_baseline and rank == 0:
        del D, sv
        line["cpu_baseline"] = cpu_baseline(rp, ci, v, n, nnz, os.cpu_count() or 1)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=464)
    ap.add_argument("--config", default="B", choices=["B", "E"],
                    help="B: 464^3 strong-scaled over N GPUs; E: 368^2 x (368 N) weak scaling (368^3 per GPU)")
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--max-iter", type=int, default=100000)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--kernel-iters", type=int, default=20)
    ap.add_argument("--plain-steps", type=int, default=100, help="plain-CSR comparison run (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true", help="force the NCCL distributed path (also at N=1)")
    ap.add_argument("--fused", action="store_true",
                    help="N>1: fused peer-memory collectives inside the kernels instead of NCCL calls")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
