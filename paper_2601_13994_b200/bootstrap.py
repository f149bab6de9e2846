"""Multi-process bootstrap of the NCCL-backed distributed plan (one process per GPU).

torch.distributed is only plumbing here: it carries the 128-byte NCCL unique id from rank
0 to the other ranks (broadcast_object_list over whatever backend the job initialised,
gloo on CPU or nccl on GPUs) and provides barriers / max-over-ranks timing in bench.py.
The solver's own communication goes through libsparsla_b200's NCCL communicator.
"""
from __future__ import annotations

import numpy as np

from . import sparsla as S


def share_unique_id(rank: int) -> bytes:
    import torch.distributed as dist
    obj = [S.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def contiguous_range(n: int, P: int, rank: int):
    blk = (n + P - 1) // P
    return min(n, rank * blk), min(n, (rank + 1) * blk)


def local_rows(kind: str, p1: int, p2: int, fparam: float, P: int, rank: int):
    """This rank's rows of a generated problem under partition_contiguous (no global
    matrix is ever built): (rows CsrMatrix with global columns, owned ids, n_global)."""
    n, _, _ = S.gen_size(kind, p1, p2, fparam)
    r0, r1 = contiguous_range(n, P, rank)
    rows = S.generate(kind, p1, p2, fparam, r0, r1)
    return rows, np.arange(r0, r1, dtype=np.int64), n


def nccl_plan(kind: str, p1: int, p2: int, fparam: float, rank: int, world: int, device: int):
    """Build this rank's NCCL plan for a contiguous row partition (collective)."""
    rows, owned, n = local_rows(kind, p1, p2, fparam, world, rank)
    uid = share_unique_id(rank)
    return S.DistPlan.create_nccl(device, world, rank, uid, rows, owned, None, n), owned, n


def nccl_plan_box(nx: int, ny: int, nz: int, rank: int, world: int, device: int):
    """Config E: N x N x Nz 7-point Poisson box (nx == ny) in z-slabs, one per rank."""
    assert nx == ny
    return nccl_plan("poisson3d_box", nx, nz, 0.0, rank, world, device)
