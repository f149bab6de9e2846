"""bench.py's N>1 arm: config B strong-scaled over N GPUs (one process per GPU, torchrun).

Each rank generates only its z-slab of the 464^3 Poisson matrix (partition_contiguous),
builds its owned/halo maps on the host, and joins the NCCL-backed plan.  One step = one
distributed Jacobi-PCG iteration (halo exchange overlapped with the interior SpMV, two
all-gather reduction points, device-side scalars), captured in a CUDA graph.  Time is
taken with CUDA events on every rank's solver stream between barriers; the reported
ms/step is the max over ranks.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np


def run(args, metric):
    import torch
    import torch.distributed as dist
    from . import bootstrap
    from . import sparsla as S

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")  # --dist at N=1 outside torchrun
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    t0 = time.time()
    if getattr(args, "config", "B") == "E":  # weak scaling: 368 x 368 x (368 P) z-slab grid
        plan, owned, n = bootstrap.nccl_plan_box(368, 368, 368 * world, rank, world, local)
    else:
        plan, owned, n = bootstrap.nccl_plan("poisson3d", args.size, 0, 0.0, rank, world, local)
    if getattr(args, "fused", False):
        plan.set_fused(True)  # reductions and halos inside the kernels, over peer memory
    tsetup = time.time() - t0
    info = plan.info()
    fmt = plan.format()
    opts = S.SolveOptions(atol=0.0, rtol=args.rtol, max_iter=args.max_iter)
    b = torch.ones(len(owned), dtype=torch.float64).pin_memory().numpy()  # pinned host buffers
    x_host = torch.empty(len(owned), dtype=torch.float64).pin_memory().numpy()

    # e2e: the public distributed solve with host buffers, to tolerance (after one untimed
    # warm-up call of W iterations that builds the plan's parked solver, as bench.py does)
    plan.cg(b, S.SolveOptions(atol=0.0, rtol=args.rtol, max_iter=max(1, args.warmup)))
    dist.barrier()
    t0 = time.perf_counter()
    x, rep = plan.cg(b, opts, out=x_host)
    t_e2e = time.perf_counter() - t0
    tt = torch.tensor([t_e2e], dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_e2e = float(tt[0])
    k_tol = rep.iterations

    sv = plan.solver(b, "cg", opts)
    stream = torch.cuda.ExternalStream(sv.stream())
    budget = max(1, k_tol - 1)
    state = {"done": 0, "resets": 0}

    def advance(k):
        while k > 0:
            if state["done"] >= budget:
                sv.reset()
                state["resets"] += 1
                state["done"] = 0
            m = min(k, budget - state["done"])
            sv.iterate(m)
            state["done"] += m
            k -= m

    sv.reset()
    advance(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    r0 = state["resets"]
    e0.record(stream)
    advance(args.steps)
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms[0])
    kms = sv.kernel_times(args.kernel_iters)
    nnz_local = plan.nnz_local
    no, nh = info["n_owned"], info["n_halo"]
    # bytes of the stored format in use (value dictionary 5 B/entry, scalar diagonal: no d
    # stream); the canonical CSR accounting is reported beside it
    mat = 5 * nnz_local + 2048 if fmt["value_dict"] else 12 * nnz_local
    dn = 0 if fmt["uniform_diag"] else 16 * no
    it_bytes = mat + 4 * (no + 1) + 8 * (no + nh) + 8 * no + 24 * no + 40 * no + dn
    spmv_bytes = mat + 4 * (no + 1) + 8 * (no + nh) + 8 * no
    canon_bytes = 12 * nnz_local + 108 * no + 8 * nh + 4
    if rank == 0:
        try:
            peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)),
                                                     "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            peak = 6650.0
        it_gbs = it_bytes / (ms / args.steps * 1e-3) / 1e9
        line = {
            "metric": metric, "value": args.steps / (ms / 1e3), "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if getattr(args, "config", "B") == "E" else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated 3-D Poisson, b = ones)",
            "config": {"workload": (f"E: 3-D 7-pt Poisson 368x368x{368 * world} ({n} DOF, 368^3 per GPU)"
                                    if getattr(args, "config", "B") == "E" else
                                    f"B: 3-D 7-pt Poisson {args.size}^3 ({n} DOF)") + f", Jacobi-PCG rtol {args.rtol}",
                       "n": n, "partition": f"contiguous z-slabs x{world}", "parallelism": f"dp{world} (row partition)",
                       "n_owned_rank0": no, "halo_rank0": nh, "interior_chunks": info["interior_chunks"],
                       "boundary_chunks": info["boundary_chunks"],
                       "l2": "no flush: per-GPU matrix + vectors exceed the 126 MB L2"},
            "iteration_gbs_per_gpu": it_gbs,
            "canonical_bytes_per_iteration_per_gpu": canon_bytes,
            "format": fmt, "collectives": "fused peer-memory (in-kernel)" if getattr(args, "fused", False)
            else "NCCL (grouped send/recv halo overlapped with the interior SpMV, all-gathered totals)",
            "roofline": {"bound": "hbm", "kernel": "iteration (spmv + halo + 2 fused updates)",
                         "achieved": it_gbs, "peak": peak, "unit": "GB/s", "frac": it_gbs / peak,
                         "traffic": None, "algorithmic_bytes_per_iteration_per_gpu": it_bytes},
            "kernel_ms_rank0": {"spmv_point(incl. halo+allgather)": kms[0], "cg_update1(+allgather)": kms[1],
                                "cg_update2": kms[2]},
            "spmv_gbs_rank0": spmv_bytes / (kms[0] * 1e-3) / 1e9,
            "time_to_tolerance_s": t_e2e, "iterations_to_tolerance": k_tol,
            "e2e": {"value": k_tol / t_e2e, "unit": "it/s", "h2d_bytes_per_step": 8 * no,
                    "d2h_bytes_per_step": 8 * no + 184, "step": "one sparsla_dist_cg_solve per rank to tolerance"},
            "gpu_launches": args.steps * sv.launches_per_iteration() + 2 * (state["resets"] - r0),
            "setup_s": tsetup,
            "parity_gate": {"converged": rep.converged, "residual_norm": rep.residual_norm},
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    sv.close()
    plan.close()
