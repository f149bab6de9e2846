"""DSparseMatrix.from_global(...).solve on the GPU: one partition per
process, distributed CG/BiCGStab forward, one distributed adjoint solve backward.  Results
equal the oracle's distributed solve / adjoint bit for bit (P=1 in-process; P=2 as two
processes sharing cuda:0 over gloo host callbacks + fused peer collectives)."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _triplets(O, kind, p1, c):
    A = (O.generate(kind, p1, 0, c) if kind == "convdiff3d" else
         O.generate(kind, p1, 2601) if kind == "fem2d" else O.generate(kind, p1))
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    return A, rows


def test_single_partition_matches_oracle(O, gpu):
    import torch
    from paper_2601_13994_b200.torch_sla import DSparseMatrix
    A, rows = _triplets(O, "poisson2d", 20, 0.0)
    vals = torch.tensor(A.vals, device="cuda:0", requires_grad=True)
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda:0", requires_grad=True)
    D = DSparseMatrix.from_global(vals, rows, A.col_idx, (A.nrows, A.nrows), num_partitions=1, my_partition=0)
    assert D.symmetric
    x = D.solve(b, atol=1e-12)
    g = torch.linspace(-1.0, 2.0, A.nrows, dtype=torch.float64, device="cuda:0")
    (x * g).sum().backward()
    po = O.partition_contiguous(A.nrows, 1)
    xo, ro, _ = O.dist_solve(A, np.ones(A.nrows), po, 1, atol=1e-12)
    assert np.array_equal(bits(x.detach().cpu().numpy()), bits(xo))
    gbo, gvo, _ = O.dist_adjoint(A, xo, g.cpu().numpy(), po, 1, atol=1e-12)
    assert np.array_equal(bits(b.grad.cpu().numpy()), bits(gbo))
    assert np.array_equal(bits(vals.grad.cpu().numpy()), bits(gvo))
    assert np.array_equal(D.gather(x), x.detach().cpu().numpy())
    D.close()


def _rank(rank, world, port, kind, p1, c, outq, rcb=False):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle as O
        from paper_2601_13994_b200.torch_sla import DSparseMatrix
        dist.init_process_group("gloo", rank=rank, world_size=world)
        A, rows = _triplets(O, kind, p1, c)
        # shuffled triplets with every diagonal split in two duplicates
        diag = rows == A.col_idx
        r = np.concatenate([rows, rows[diag]])
        cc = np.concatenate([A.col_idx, A.col_idx[diag]])
        v = np.concatenate([np.where(diag, 0.5 * A.vals, A.vals), 0.5 * A.vals[diag]])  # exact halves
        perm = np.random.default_rng(5).permutation(len(r))
        vals = torch.tensor(v[perm], device="cuda:0", requires_grad=True)
        coords = O.gen_coords(kind, p1, 2601) if rcb else None
        D = DSparseMatrix.from_global(vals, r[perm], cc[perm], (A.nrows, A.nrows), num_partitions=world,
                                      my_partition=rank, coords=coords)
        b = torch.ones(D.n_owned, dtype=torch.float64, device="cuda:0", requires_grad=True)
        x = D.solve(b, atol=0.0, rtol=1e-11)
        g = torch.as_tensor(np.cos(np.arange(A.nrows))[D.owned], device="cuda:0")
        (x * g).sum().backward()
        xg = D.gather(x)
        out = (rank, D.owned, x.detach().cpu().numpy(), b.grad.cpu().numpy(), vals.grad.cpu().numpy(), perm,
               D.symmetric, xg)
        outq.put(out)
        dist.barrier()
        D.close()
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        outq.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("kind,p1,c,rcb", [("poisson3d", 16, 0.0, False), ("convdiff3d", 14, 0.4, False),
                                           ("fem2d", 40, 0.0, True)])
def test_two_processes_solve_and_backward(O, gpu, kind, p1, c, rcb):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, kind, p1, c, q, rcb)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for t in res:
        assert not isinstance(t[1], str), t[2]
    A, rows = _triplets(O, kind, p1, c)
    n = A.nrows
    po = O.partition_rcb(*O.gen_coords(kind, p1, 2601), 2) if rcb else O.partition_contiguous(n, 2)
    nonsym = kind == "convdiff3d"
    xo, _, _ = O.dist_solve(A, np.ones(n), po, 2, kind="bicgstab" if nonsym else "cg", atol=0.0, rtol=1e-11)
    g = np.cos(np.arange(n))
    x = np.empty(n)
    gb = np.empty(n)
    gv_canon = np.zeros(A.nnz)
    for rank, owned, xr, gbr, gvr, perm, sym, xg in res:
        assert sym == (not nonsym)
        x[owned] = xr
        gb[owned] = gbr
        if rank == 0:
            assert np.array_equal(bits(xg), bits(xo))
        else:
            assert xg is None
    assert np.array_equal(bits(x), bits(xo))
    # per-input-entry gradients, summed over ranks; map back to canonical entries: every
    # duplicate of a canonical entry carries the canonical entry's gradient
    gin = res[0][4] + res[1][4]
    perm = res[0][5]
    diag = rows == A.col_idx
    canon_of = np.concatenate([np.arange(A.nnz), np.nonzero(diag)[0]])[perm]
    gv_canon[canon_of] = gin
    assert np.array_equal(gin, gv_canon[canon_of])
    if not nonsym:
        gbo, gvo, _ = O.dist_adjoint(A, xo, g, po, 2, atol=0.0, rtol=1e-11)
        assert np.array_equal(bits(gb), bits(gbo)) and np.array_equal(bits(gv_canon), bits(gvo))
    else:
        T = O.transpose(A)
        lt, _, _ = O.dist_solve(T, g, po, 2, kind="bicgstab", atol=0.0, rtol=1e-11)
        assert np.array_equal(bits(gb), bits(lt))
        assert np.array_equal(bits(gv_canon), bits(-(lt[rows] * xo[A.col_idx])))


def test_values_changed_between_solves_are_used(O, gpu):
    """The plan copies the values at build time; a later in-place change of the values
    tensor (an optimizer step) must reach the next solve and its backward."""
    import torch
    from paper_2601_13994_b200.torch_sla import DSparseMatrix
    A, rows = _triplets(O, "convdiff3d", 8, 0.3)
    vals = torch.tensor(A.vals, device="cuda:0", requires_grad=True)
    D = DSparseMatrix.from_global(vals, rows, A.col_idx, (A.nrows, A.nrows), num_partitions=1, my_partition=0)
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda:0")
    x1 = D.solve(b, atol=0.0, rtol=1e-12)
    with torch.no_grad():
        vals.mul_(2.0)                        # A -> 2A: x -> x/2, still nonsymmetric
    x2 = D.solve(b, atol=0.0, rtol=1e-12)
    A2 = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, 2.0 * A.vals)
    po = O.partition_contiguous(A.nrows, 1)
    xo, _, _ = O.dist_solve(A2, np.ones(A.nrows), po, 1, kind="bicgstab", atol=0.0, rtol=1e-12)
    assert np.array_equal(bits(x2.detach().cpu().numpy()), bits(xo))
    assert not np.array_equal(bits(x1.detach().cpu().numpy()), bits(xo))
    x2.sum().backward()
    lam = np.linalg.solve(A2.dense().T, np.ones(A.nrows))       # dense adjoint of the NEW matrix
    gv_ref = -(lam[rows] * xo[A.col_idx])
    err = np.abs(vals.grad.cpu().numpy() - gv_ref).max() / np.abs(gv_ref).max()
    assert err <= 1e-7, err
    # symmetrising the values flips the default backend to CG on the next solve
    with torch.no_grad():
        vals.copy_(torch.as_tensor(O.generate("poisson3d", 8).vals))
    D.solve(b, atol=1e-12)
    assert D.symmetric
    D.close()


def test_structurally_nonsymmetric_pattern_rejected(O, gpu):
    import torch
    from paper_2601_13994_b200 import sparsla as S
    from paper_2601_13994_b200.torch_sla import DSparseMatrix
    rows = np.array([0, 0, 1, 1, 2])
    cols = np.array([0, 1, 1, 2, 2])       # (0,1) and (1,2) have no mirror
    vals = torch.tensor([4.0, -1.0, 4.0, -1.0, 4.0], dtype=torch.float64, device="cuda:0")
    with pytest.raises(S.UnsupportedInputError):
        DSparseMatrix.from_global(vals, rows, cols, (3, 3), num_partitions=1, my_partition=0)
