"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path.

Each process plays one rank exactly as bench.py --gpus N does: it generates only its own
rows (contiguous partition), builds its owned/halo maps with the product's build_local
(part_of = NULL fast path), bootstraps the NCCL id through torch.distributed, and then
drives a distributed Jacobi-PCG whose halo exchange and rank-ordered reductions go over
gloo.  The local SpMV / canonical dots are the oracle's (test infrastructure): the point is
the maps and the protocol, which must reproduce the oracle's in-process distributed CG bit
for bit with exactly 1 halo exchange + 2 all-reduce points per iteration.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, p1, outq):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        import pyoracle as O
        from paper_2601_13994_b200 import bootstrap, sparsla as S
        dist.init_process_group("gloo", rank=rank, world_size=world)
        # NCCL id bootstrap (the same helper the GPU bench uses)
        uid = bootstrap.share_unique_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(i == ids[0] for i in ids)
        rows, owned, n = bootstrap.local_rows(kind, p1, 0, 1.0, world, rank)
        L = S.build_local(rows, owned, None, world, rank)
        # count handshake over gloo
        for q in L.neighbors:
            q = int(q)
            mine = torch.tensor([len(L.send_to(q)), len(L.recv_from(q))], dtype=torch.int64)
            theirs = torch.empty(2, dtype=torch.int64)
            reqs = [dist.isend(mine, q), dist.irecv(theirs, q)]
            for r in reqs:
                r.wait()
            assert theirs[0] == mine[1] and theirs[1] == mine[0]
        no, nh = len(L.owned), len(L.halo)
        counters = {"exchanges": 0, "allreduces": 0}

        def exchange(xl):
            reqs, bufs = [], []
            for q in L.neighbors:
                q = int(q)
                s = torch.from_numpy(np.ascontiguousarray(xl[L.send_to(q)]))
                r = torch.empty(len(L.recv_from(q)), dtype=torch.float64)
                reqs += [dist.isend(s, q), dist.irecv(r, q)]
                bufs.append((q, r))
            for rq in reqs:
                rq.wait()
            for q, r in bufs:
                xl[L.recv_from(q)] = r.numpy()
            counters["exchanges"] += 1

        # halo exchange delivers exactly the neighbours' owned values (canonical order)
        g = np.random.default_rng(0).standard_normal(n)
        xl = np.zeros(no + nh)
        xl[:no] = g[L.owned]
        exchange(xl)
        assert np.array_equal(xl[no:], g[L.halo])
        Lc = O.Csr(no, no + nh, L.row_ptr, L.col_idx, L.vals)

        def spmv(v):
            xl = np.zeros(no + nh)
            xl[:no] = v
            exchange(xl)
            return O.spmv(Lc, xl)

        def allreduce(vals):  # rank-ordered sequential sum
            t = torch.tensor(vals, dtype=torch.float64)
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            counters["allreduces"] += 1
            s = out[0].clone().numpy()
            for q in range(1, world):
                s = s + out[q].numpy()
            return s

        # distributed Jacobi-PCG, same recurrence as cg_core (x0 = 0, rtol 1e-8)
        d = np.empty(no)
        for i in range(no):
            a = [L.vals[k] for k in range(L.row_ptr[i], L.row_ptr[i + 1]) if L.col_idx[k] == i]
            d[i] = 1.0 / a[0] if a and a[0] != 0.0 and np.isfinite(1.0 / a[0]) else 1.0
        b = np.ones(no)
        x = np.zeros(no)
        q_ = spmv(x)
        r = b - q_
        z = d * r
        p = z.copy()
        rz, rr, bb = allreduce([O.cdot(r, z), O.cdot(r, r), O.cdot(b, b)])
        tol = max(0.0, 1e-8 * np.sqrt(bb))
        k = 0
        rnorm = np.sqrt(rr)
        while rnorm > tol and k < 5000:
            q_ = spmv(p)
            pq = allreduce([O.cdot(p, q_)])[0]
            alpha = rz / pq
            x = x + alpha * p
            r = r - alpha * q_
            z = d * r
            rz_new, rr = allreduce([O.cdot(r, z), O.cdot(r, r)])
            k += 1
            rnorm = np.sqrt(rr)
            if rnorm <= tol:
                break
            beta = rz_new / rz
            rz = rz_new
            p = z + beta * p
        outq.put((rank, owned, x, k, dict(counters)))
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        import traceback
        outq.put((rank, "error", traceback.format_exc(), None, None))


@pytest.mark.parametrize("kind,p1", [("poisson3d", 10), ("poisson2d", 24)])
def test_gloo_two_ranks_reproduce_oracle_dist_cg(O, kind, p1):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, p1, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert not isinstance(r[1], str), r[2]
    A = O.generate(kind, p1)
    b = np.ones(A.nrows)
    xo, ro, co = O.dist_solve(A, b, O.partition_contiguous(A.nrows, world), world, atol=0.0, rtol=1e-8)
    x = np.empty(A.nrows)
    for rank, owned, xr, k, cnt in res:
        x[owned] = xr
        assert k == ro["iterations"]
        assert cnt["exchanges"] == 2 + k  # map check + initial residual + one per iteration
        assert cnt["allreduces"] == 1 + 2 * k
    assert np.array_equal(x.view(np.int64), xo.view(np.int64))
