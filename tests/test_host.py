"""CPU tests of the product's host side (no GPU): the C ABI loads and exports every symbol
include/sparsla_c.h declares; canonical assembly, generators, partitioners and build_local
are bit-exact with the oracle / the reference's golden fixtures; errors map to the
reference's exception classes; device entry points fail loudly without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sparsla_c.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sparsla_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol(S):
    L = S.lib()
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    out = os.popen(f"nm -D --defined-only {S.LIB_PATH}").read()
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a(S):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {S.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {S.LIB_PATH} 2>&1 | grep -c UBLKCP").read()
    assert int(sass.strip() or 0) > 0  # TMA bulk copies in the staged SpMV


def test_canonicalize_matches_reference_golden(S):
    G = np.load(os.path.join(ROOT, "tests", "golden", "sparse_core.npz"))
    for i in range(int(G["ncases"])):
        nr, nc = (int(t) for t in G[f"c{i}_shape"])
        rin = G[f"c{i}_in"]
        a = S.SparseCoo(rin[0].astype(np.int64), rin[1].astype(np.int64), G[f"c{i}_vin"], (nr, nc))
        assert np.array_equal(a.rows, G[f"c{i}_rows"]) and np.array_equal(a.cols, G[f"c{i}_cols"])
        assert np.array_equal(bits(a.vals), bits(G[f"c{i}_vals"])), i
        A = S.CsrMatrix.from_coo(a)
        assert np.array_equal(A.row_ptr, G[f"c{i}_rp"])
        assert A.bytes() == int(G[f"c{i}_bytes"])
        back = A.to_coo()
        assert np.array_equal(back.rows, a.rows) and np.array_equal(bits(back.vals), bits(a.vals))
        t = S.transpose(a)
        assert np.array_equal(t.rows, G[f"c{i}_trows"]) and np.array_equal(t.cols, G[f"c{i}_tcols"])
        assert np.array_equal(bits(t.vals), bits(G[f"c{i}_tvals"]))
        if nr == nc:
            s1, s2 = (bool(v) for v in G[f"c{i}_sym"])
            assert S.is_structurally_symmetric(a) == s1 and S.is_symmetric(a) == s2, i


def test_spec_sparse_core_examples(S):
    a = S.SparseCoo([0, 0], [0, 0], [1.0, 2.0], (1, 1))
    assert list(a.vals) == [3.0] and a.nnz == 1
    b = S.SparseCoo([1, 0], [0, 0], [5, 7], (2, 1))
    assert list(zip(b.rows, b.cols, b.vals)) == [(0, 0, 7.0), (1, 0, 5.0)]
    with pytest.raises(S.BoundsError):
        S.SparseCoo([0], [3], [1.0], (2, 2))
    with pytest.raises(S.DimensionError):
        S.SparseCoo([0, 1], [0], [1.0], (2, 2))
    e = S.CsrMatrix.from_coo(S.SparseCoo([], [], [], (3, 3)))
    assert list(e.row_ptr) == [0, 0, 0, 0]
    I = S.CsrMatrix.from_coo(S.SparseCoo([0, 1], [0, 1], [1.0, 1.0], (2, 2)))
    assert list(I.row_ptr) == [0, 1, 2] and list(I.col_idx) == [0, 1]
    z = S.SparseCoo([0, 1], [1, 0], [0.0, 0.0], (2, 2))  # explicit zeros kept
    assert z.nnz == 2 and z.find(1, 0) == 1 and z.find(0, 0) == -1
    w = z.with_values([3.0, 4.0])
    assert list(w.vals) == [3.0, 4.0] and list(w.rows) == [0, 1]
    with pytest.raises(S.DimensionError):
        z.with_values([1.0])
    with pytest.raises(S.BoundsError):
        S.SparseCoo([], [], [], (5000, 5000)).to_dense()
    P, _ = S.poisson2d(2)
    assert P.nrows == 4 and np.all(np.diff(P.row_ptr) == 3)
    D = S.SparseCoo(*coo_of(P), (4, 4)).to_dense()
    assert np.all(np.diag(D) == 4)


def coo_of(A):
    return np.repeat(np.arange(A.nrows), np.diff(A.row_ptr)), A.col_idx, A.vals


@pytest.mark.parametrize("kind,p1,p2,fp", [("poisson2d", 33, 0, 0.0), ("poisson3d", 11, 0, 0.0),
                                           ("convdiff3d", 9, 0, 1.0), ("convdiff3d", 7, 0, 0.37),
                                           ("fem2d", 3, 2601, 0.0), ("fem2d", 57, 2601, 0.0),
                                           ("fem2d", 40, 7, 0.0), ("poisson3d_box", 6, 17, 0.0)])
def test_generators_bitwise_vs_oracle(S, O, kind, p1, p2, fp):
    A = S.generate(kind, p1, p2, fp)
    B = O.generate(kind, p1, p2, fp)
    assert np.array_equal(A.row_ptr, B.row_ptr) and np.array_equal(A.col_idx, B.col_idx)
    assert np.array_equal(bits(A.vals), bits(B.vals))
    # per-rank generation == the slice of global generation (row ranges)
    n = A.nrows
    for r0, r1 in [(0, n // 3), (n // 3, n), (n // 2, n // 2 + 1)]:
        R = S.generate(kind, p1, p2, fp, r0, r1)
        k0, k1 = A.row_ptr[r0], A.row_ptr[r1]
        assert np.array_equal(R.row_ptr, A.row_ptr[r0:r1 + 1] - k0)
        assert np.array_equal(R.col_idx, A.col_idx[k0:k1])
        assert np.array_equal(bits(R.vals), bits(A.vals[k0:k1]))
    nr, nn, rp, ci, v = S.generate_i32(kind, p1, p2, fp)
    assert np.array_equal(rp, A.row_ptr) and np.array_equal(ci, A.col_idx)


def test_generator_sizes(S):
    for N in (2, 5, 464):
        n, nnz, _ = S.gen_size("poisson3d", N)
        assert n == N ** 3 and nnz == 7 * N ** 3 - 6 * N ** 2
    n, nnz, _ = S.gen_size("poisson2d", 1000)
    assert n == 10 ** 6 and nnz == 4_996_000
    with pytest.raises(S.InvalidArgumentError):
        S.gen_size("poisson2d", 1)


def test_fem_mesh_properties(S):
    A = S.generate("fem2d", 120, 2601)
    lens = np.diff(A.row_ptr)
    assert lens.min() >= 3 and lens.max() <= 9 and 6.5 < lens.mean() < 7.1
    coo = S.SparseCoo(*coo_of(A), A.shape, _canonical=True)
    assert S.is_symmetric(coo, 1e-14)  # P1 stiffness is symmetric
    # row sums: interior rows of a Laplacian stiffness sum to ~0, boundary rows > 0
    rs = np.add.reduceat(A.vals, A.row_ptr[:-1])
    assert rs.min() > -1e-9


def test_partitioners_match_oracle(S, O):
    for n, P in [(6, 2), (5, 2), (9, 4), (1000, 7), (10, 10)]:
        assert np.array_equal(S.partition_contiguous(n, P), O.partition_contiguous(n, P))
    with pytest.raises(S.InvalidArgumentError):
        S.partition_contiguous(3, 4)
    xs, ys = np.array([0.0, 1.0, 0.0, 1.0]), np.array([0.0, 0.0, 1.0, 1.0])
    assert list(S.partition_rcb(xs, ys, 2)) == [0, 1, 0, 1]
    for kind, p1 in [("poisson2d", 16), ("poisson2d", 37), ("fem2d", 50)]:
        xs, ys = S.gen_coords(kind, p1, 2601)
        for P in (1, 2, 4, 8):
            assert np.array_equal(S.partition_rcb(xs, ys, P), O.partition_rcb(xs, ys, P))
    with pytest.raises(S.InvalidArgumentError):
        S.partition_rcb(xs, ys, 3)  # non-power-of-two


@pytest.mark.parametrize("kind,p1,P,part", [("poisson2d", 8, 2, "contig"), ("poisson2d", 20, 3, "contig"),
                                            ("poisson3d", 9, 4, "contig"), ("fem2d", 30, 4, "rcb"),
                                            ("poisson2d", 24, 8, "rcb"), ("convdiff3d", 8, 2, "contig")])
def test_build_local_bitwise_vs_oracle(S, O, kind, p1, P, part):
    A = S.generate(kind, p1, 2601 if kind == "fem2d" else 0, 1.0)
    Ao = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, A.vals)
    if part == "contig":
        po = S.partition_contiguous(A.nrows, P)
    else:
        po = S.partition_rcb(*S.gen_coords(kind, p1, 2601), P)
    sends = {}
    for rank in range(P):
        owned = np.nonzero(po == rank)[0]
        rp = np.concatenate([[0], np.cumsum(np.diff(A.row_ptr)[owned])])
        sel = np.concatenate([np.arange(A.row_ptr[i], A.row_ptr[i + 1]) for i in owned]) \
            if len(owned) else np.zeros(0, np.int64)
        rows = S.CsrMatrix(len(owned), A.ncols, rp, A.col_idx[sel], A.vals[sel])
        L = S.build_local(rows, owned, po, P, rank)
        R = O.build_local(Ao, po, P, rank)
        for k in ("owned", "halo", "neighbors", "send_ptr", "send_idx", "recv_ptr", "recv_idx",
                  "row_ptr", "col_idx"):
            assert np.array_equal(getattr(L, k), R[k]), (k, rank)
        assert np.array_equal(bits(L.vals), bits(R["vals"]))
        for q in L.neighbors:
            sends[(rank, int(q))] = L.owned[L.send_to(q)]
    # |send p->q| == |recv q<-p| and the payload order is canonical (ascending global)
    for (p, q), g in sends.items():
        assert np.all(np.diff(g) > 0)
        assert np.array_equal(g, np.sort(g))
        assert (q, p) in sends


def test_build_local_contiguous_halo_size(S):
    """Contiguous N x N: each neighbour sends exactly N values (one grid row)."""
    N = 32
    A = S.generate("poisson2d", N)
    po = S.partition_contiguous(A.nrows, 4)
    for rank in range(4):
        owned = np.nonzero(po == rank)[0]
        r0, r1 = owned[0], owned[-1] + 1
        L = S.build_local(S.generate("poisson2d", N, 0, 0, r0, r1), owned, po, 4, rank)
        for q in L.neighbors:
            assert len(L.recv_from(q)) == N and len(L.send_to(q)) == N
        assert len(L.halo) == N * len(L.neighbors)


def test_device_calls_fail_loudly_without_gpu(S):
    if S.device_count() > 0:
        pytest.skip("GPU present")
    A, b = S.poisson2d(4)
    with pytest.raises(S.Error, match="no CUDA device"):
        S.cg_solve(A, b)
    with pytest.raises(S.Error, match="no CUDA device"):
        S.spmv(A, b)
    with pytest.raises(S.Error, match="no CUDA device"):
        S.eig_smallest(A, 2)
    with pytest.raises(S.InvalidArgumentError):
        S.eig_smallest(A, 0)  # argument checks come first


def test_eig_backward_argument_checks(S):
    """eig_backward validates shapes and convergence flags before any device work."""
    A, _ = S.poisson2d(4)
    n = A.nrows
    rep = S.EigenReport(iterations=1, residual_norms=np.zeros(2), pair_converged=np.array([True, False]))
    res = S.EigenResult(np.array([1.0, 2.0]), np.zeros((n, 2)), rep)
    with pytest.raises(S.DimensionError):
        S.eig_backward(res, A, [1.0])
    with pytest.raises(S.InvalidArgumentError):
        S.eig_backward(res, A, [1.0, 1.0])
    bad = S.EigenResult(np.array([1.0, 2.0]), np.zeros((n + 1, 2)), rep)
    with pytest.raises(S.DimensionError):
        S.eig_backward(bad, A, [1.0, 1.0])


def test_options_validation(S):
    with pytest.raises(S.InvalidArgumentError):
        S.SolveOptions(preconditioner="ilu").c()


def test_dsparse_argument_errors(S):
    """DSparseMatrix.from_global checks its partition arguments before touching a device."""
    import torch
    from paper_2601_13994_b200.torch_sla import DSparseMatrix
    v = torch.ones(3, dtype=torch.float64)
    with pytest.raises(S.InvalidArgumentError):
        DSparseMatrix.from_global(v, [0, 1, 2], [0, 1, 2], (3, 3), num_partitions=2, my_partition=0)
    with pytest.raises(S.InvalidArgumentError):
        DSparseMatrix.from_global(v, [0, 1, 2], [0, 1, 2], (3, 3), num_partitions=1, my_partition=1)
    with pytest.raises(TypeError):
        DSparseMatrix()
