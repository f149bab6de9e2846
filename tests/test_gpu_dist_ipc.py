"""Multi-PROCESS distributed CG on ONE B200: 2 ranks as 2 processes sharing cuda:0, setup
traffic over torch.distributed (gloo host callbacks), iterations through fused peer
collectives on cudaIpc-mapped memory (cross-process peer stores + system-scope epoch
flags) — the code path real multi-GPU runs use for peers in other processes.  The result
must equal the oracle's distributed CG bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, kind, p1, fused, outq, backend="cg", c=0.0):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        from paper_2601_13994_b200 import bootstrap, sparsla as S
        dist.init_process_group("gloo", rank=rank, world_size=world)
        rows, owned, n = bootstrap.local_rows(kind, p1, 0, c, world, rank)
        T = S.torch_host_transport(world)
        plan = S.DistPlan.create_host(0, world, rank, T, rows, owned, None, n)
        plan.set_fused(fused)
        solve = plan.cg if backend == "cg" else plan.bicgstab
        x, rep = solve(np.ones(len(owned)), S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=5000))
        x2, rep2 = solve(np.ones(len(owned)), S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=5000))
        c = plan.counters()
        outq.put((rank, owned, x, rep.iterations, rep.residual_norm, np.array_equal(x, x2), c))
        dist.barrier()
        plan.close()
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        outq.put((rank, "error", traceback.format_exc(), None, None, None, None))


@pytest.mark.parametrize("fused", [True, False])
def test_two_processes_one_gpu(O, gpu, fused):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, "poisson3d", 24, fused, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert not isinstance(r[1], str), r[2]
    A = O.generate("poisson3d", 24)
    b = np.ones(A.nrows)
    xo, ro, _ = O.dist_solve(A, b, O.partition_contiguous(A.nrows, 2), 2, atol=0.0, rtol=1e-10, max_iter=5000)
    x = np.empty(A.nrows)
    for rank, owned, xr, k, rn, same, c in res:
        x[owned] = xr
        assert k == ro["iterations"] and same
        if fused:
            # two solves: transport traffic is each solve's init only (~70 iterations each run
            # through peer memory; the unfused path makes one exchange per iteration)
            assert c["raw_exchanges"] <= 4 and c["raw_allgathers"] <= 4, c
        else:
            assert c["raw_exchanges"] >= 2 * ro["iterations"], c
    assert np.array_equal(x.view(np.int64), xo.view(np.int64))


def test_two_processes_one_gpu_bicgstab_fused(O, gpu):
    """BiCGStab through cross-process fused peer collectives (p-hat / s-hat halo pushes and
    three reduction points per iteration over cudaIpc memory)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, "convdiff3d", 20, True, q, "bicgstab", 0.3))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert not isinstance(r[1], str), r[2]
    A = O.generate("convdiff3d", 20, 0, 0.3)
    b = np.ones(A.nrows)
    xo, ro, _ = O.dist_solve(A, b, O.partition_contiguous(A.nrows, 2), 2, kind="bicgstab", atol=0.0,
                             rtol=1e-10, max_iter=5000)
    x = np.empty(A.nrows)
    for rank, owned, xr, k, rn, same, c in res:
        x[owned] = xr
        assert k == ro["iterations"] and same
        assert c["raw_exchanges"] <= 4 and c["raw_allgathers"] <= 4, c
    assert np.array_equal(x.view(np.int64), xo.view(np.int64))


def _rank_timeout(rank, world, port, outq):
    """rank 1 stops contributing after 3 iterations (its own max_iter); rank 0's fused
    peer-collective waits must give up after SPARSLA_TRANSPORT_TIMEOUT and raise
    TransportError instead of spinning forever."""
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPARSLA_TRANSPORT_TIMEOUT="2")
        import time
        import torch.distributed as dist
        from paper_2601_13994_b200 import bootstrap, sparsla as S
        dist.init_process_group("gloo", rank=rank, world_size=world)
        rows, owned, n = bootstrap.local_rows("poisson3d", 24, 0, 0.0, world, rank)
        plan = S.DistPlan.create_host(0, world, rank, S.torch_host_transport(world), rows, owned, None, n)
        plan.set_fused(True)
        t0 = time.time()
        try:
            _, rep = plan.cg(np.ones(len(owned)), S.SolveOptions(atol=0.0, rtol=1e-10,
                                                                 max_iter=3 if rank == 1 else 5000))
            out = ("ok", rep.iterations, rep.diagnostic)
        except S.TransportError as e:
            out = ("transport_error", str(e), None)
        outq.put((rank, out, time.time() - t0))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        outq.put((rank, ("error", traceback.format_exc(), None), 0.0))


def test_fused_peer_wait_times_out_with_transport_error(gpu):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_timeout, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (o, t)) for r, o, t in [q.get(timeout=240) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
    assert res[1][0][0] == "ok" and res[1][0][1] == 3, res[1]
    assert res[0][0][0] == "transport_error", res[0]
    assert "timed out" in res[0][0][1]
    assert res[0][1] < 30.0, res[0]  # bounded by the 2 s timeout, not a hang
