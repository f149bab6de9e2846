"""The oracle is pinned before it is trusted (CPU only).

1. Against the committed golden fixtures produced by the reference's own compiled
   sparse.cpp (tests/golden/make_golden.py): canonicalization, CSR, spmv, spmv_transpose,
   transpose — bit for bit.
2. Against the live reference build (oracle/_ref) when it is present (this container).
3. Against every SPEC.md known-answer example for the solver / adjoint / distributed
   contracts, and the survey's probe iteration counts of the reference spmv + SPEC-rule PCG.
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "sparse_core.npz")


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


@pytest.fixture(scope="module")
def G():
    return np.load(GOLD)


def golden_cases(G):
    for i in range(int(G["ncases"])):
        nr, nc = (int(t) for t in G[f"c{i}_shape"])
        rin = G[f"c{i}_in"]
        yield i, nr, nc, rin[0].astype(np.int64), rin[1].astype(np.int64), G[f"c{i}_vin"]


def test_oracle_canonicalize_matches_reference_golden(O, G):
    for i, nr, nc, r, c, v in golden_cases(G):
        cr, cc, cv = O.canonicalize(nr, nc, r, c, v)
        assert np.array_equal(cr, G[f"c{i}_rows"]) and np.array_equal(cc, G[f"c{i}_cols"]), i
        assert np.array_equal(bits(cv), bits(G[f"c{i}_vals"])), i
        A = O.csr_from_coo(nr, nc, cr, cc, cv)
        assert np.array_equal(A.row_ptr, G[f"c{i}_rp"]), i


def test_oracle_spmv_matches_reference_golden(O, G):
    for i, nr, nc, r, c, v in golden_cases(G):
        A = O.csr_from_coo(nr, nc, G[f"c{i}_rows"], G[f"c{i}_cols"], G[f"c{i}_vals"])
        assert np.array_equal(bits(O.spmv(A, G[f"c{i}_x"])), bits(G[f"c{i}_y"])), i
        # reference spmv_transpose == row-ordered spmv on the canonical transpose
        yt = O.spmv(O.transpose(A), G[f"c{i}_xt"])
        assert np.array_equal(bits(yt), bits(G[f"c{i}_yt"])), i
        T = O.transpose(A)
        trows = np.repeat(np.arange(T.nrows), np.diff(T.row_ptr))
        assert np.array_equal(trows, G[f"c{i}_trows"]) and np.array_equal(T.col_idx, G[f"c{i}_tcols"])


def test_oracle_generators_match_reference_canonicalization(O, G):
    for kind, p1, p2, fp in [("poisson2d", 12, 0, 0.0), ("poisson3d", 6, 0, 0.0),
                             ("convdiff3d", 5, 0, 1.0), ("fem2d", 14, 2601, 0.0)]:
        A = O.generate(kind, p1, p2, fp)
        key = f"gen_{kind}"
        assert np.array_equal(A.row_ptr, G[key + "_rp"]) and np.array_equal(A.col_idx, G[key + "_ci"])
        assert np.array_equal(bits(A.vals), bits(G[key + "_v"])), kind


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle",
                                                    "_ref", "libsparsla_ref.so")),
                    reason="reference build absent")
def test_oracle_vs_live_reference_random(O):
    rng = np.random.default_rng(11)
    for t in range(20):
        nr, nc = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        nnz = int(rng.integers(0, 3000))
        r, c = rng.integers(0, nr, nnz), rng.integers(0, nc, nnz)
        v = rng.standard_normal(nnz)
        ro, co, vo = O.ref_canonicalize(nr, nc, r, c, v)
        cr, cc, cv = O.canonicalize(nr, nc, r, c, v)
        assert np.array_equal(ro, cr) and np.array_equal(co, cc) and np.array_equal(bits(vo), bits(cv))
        A = O.csr_from_coo(nr, nc, cr, cc, cv)
        x = rng.standard_normal(nc)
        assert np.array_equal(bits(O.spmv(A, x)), bits(O.ref_spmv(A, x)))
    # a mid-size stencil through the reference canonicalization
    A = O.generate("poisson3d", 40)
    n, r, c, v = O.gen_triplets("poisson3d", 40)
    Ar, _ = O.ref_csr_from_coo(n, n, r, c, v)
    assert np.array_equal(A.row_ptr, Ar.row_ptr) and np.array_equal(A.col_idx, Ar.col_idx)
    x = np.random.default_rng(3).standard_normal(n)
    assert np.array_equal(bits(O.spmv(A, x)), bits(O.ref_spmv(Ar, x)))
    with pytest.raises(O.RefError) as e:
        O.ref_canonicalize(2, 2, [0], [3], [1.0])
    assert e.value.code == 2  # BoundsError


# ----------------------------------------------------------- SPEC known answers -------
def test_spec_jacobi(O):
    A = O.csr_from_triplets(2, 2, [0, 1], [0, 1], [2.0, 4.0])
    assert list(O.jacobi(A)) == [0.5, 0.25]
    B = O.csr_from_triplets(2, 2, [0, 1, 1], [0, 0, 1], [0.0, 1.0, 4.0])
    assert list(O.jacobi(B)) == [1.0, 0.25]
    assert np.all(O.jacobi(O.generate("poisson2d", 6)) == 0.25)


def test_spec_cg(O):
    A = O.csr_from_triplets(4, 4, range(4), range(4), [2.0] * 4)
    x, r = O.cg(A, [2, 4, 6, 8])
    assert list(x) == [1, 2, 3, 4] and r["iterations"] == 1 and r["spmv_count"] == 2
    P = O.generate("poisson2d", 32)
    b = np.ones(P.nrows)
    x, r = O.cg(P, b, atol=1e-10)
    assert r["converged"] and r["residual_norm"] <= 1e-10
    assert np.max(np.abs(x - np.linalg.solve(P.dense(), b))) <= 1e-8
    x1, r1 = O.cg(P, b, atol=1e-10, max_iter=1)
    assert not r1["converged"] and r1["residual_norm"] > 1e-10
    its = [O.cg(O.generate("poisson2d", N), np.ones(N * N), atol=1e-10)[1]["iterations"]
           for N in (16, 32, 64, 128)]
    assert all(1.5 <= its[i + 1] / its[i] <= 3.0 for i in range(3)), its


def test_survey_probe_iteration_counts(O):
    """reference spmv + SPEC-rule PCG (rtol 1e-8, b = ones)."""
    for kind, N, want in [("poisson2d", 100, 187), ("poisson2d", 200, 369),
                          ("poisson3d", 32, 79), ("poisson3d", 64, 159)]:
        A = O.generate(kind, N)
        _, r = O.cg(A, np.ones(A.nrows), atol=0.0, rtol=1e-8, max_iter=10000)
        assert r["iterations"] == want, (kind, N, r)


def test_spec_bicgstab(O):
    A = O.csr_from_triplets(2, 2, [0, 0, 1], [0, 1, 1], [4.0, 1.0, 3.0])
    x, r = O.bicgstab(A, [5, 3])
    assert r["converged"] and np.allclose(x, [1, 1], atol=1e-12)
    P = O.generate("poisson2d", 16)
    b = np.ones(P.nrows)
    assert np.max(np.abs(O.bicgstab(P, b, atol=1e-12)[0] - O.cg(P, b, atol=1e-12)[0])) <= 1e-8
    Z = O.csr_from_triplets(2, 2, [], [], [])
    _, rz = O.bicgstab(Z, [1, 1])
    assert not rz["converged"] and rz["diagnostic"].startswith("breakdown")


def test_spec_adjoint(O):
    A = O.csr_from_triplets(3, 3, range(3), range(3), [2.0] * 3)
    x, _ = O.cg(A, [2, 4, 6])
    gb, gv, r = O.adjoint_backward(A, x, np.ones(3))
    assert list(gb) == [0.5, 0.5, 0.5] and list(gv) == [-0.5, -1.0, -1.5]
    # central finite differences on Poisson n = 1024 (Table 4 magnitude)
    P = O.generate("poisson2d", 32)
    b = np.random.default_rng(0).uniform(0.5, 1.5, P.nrows)
    x, _ = O.cg(P, b, atol=1e-13)
    gb, gv, _ = O.adjoint_backward(P, x, np.ones(P.nrows), atol=1e-13)
    eps = 1e-5
    for k in (0, 17, 500, 3000):
        vp, vm = P.vals.copy(), P.vals.copy()
        vp[k] += eps
        vm[k] -= eps
        Lp = O.cg(O.Csr(P.nrows, P.ncols, P.row_ptr, P.col_idx, vp), b, atol=1e-13)[0].sum()
        Lm = O.cg(O.Csr(P.nrows, P.ncols, P.row_ptr, P.col_idx, vm), b, atol=1e-13)[0].sum()
        fd = (Lp - Lm) / (2 * eps)
        assert abs(fd - gv[k]) / max(abs(fd), abs(gv[k]), 1e-12) < 1e-5
    for i in (0, 100, 1000):
        bp, bm = b.copy(), b.copy()
        bp[i] += eps
        bm[i] -= eps
        fd = (O.cg(P, bp, atol=1e-13)[0].sum() - O.cg(P, bm, atol=1e-13)[0].sum()) / (2 * eps)
        assert abs(fd - gb[i]) / max(abs(fd), abs(gb[i]), 1e-12) < 1e-5


def test_spec_partition_and_local(O):
    assert list(O.partition_contiguous(6, 2)) == [0, 0, 0, 1, 1, 1]
    assert list(O.partition_contiguous(5, 2)) == [0, 0, 0, 1, 1]
    assert list(O.partition_contiguous(9, 4)) == [0, 0, 0, 1, 1, 1, 2, 2, 2]
    xs, ys = np.array([0.0, 1.0, 0.0, 1.0]), np.array([0.0, 0.0, 1.0, 1.0])
    assert list(O.partition_rcb(xs, ys, 2)) == [0, 1, 0, 1]
    gx, gy = np.meshgrid(np.arange(16.0), np.arange(16.0))
    p = O.partition_rcb(gx.ravel(), gy.ravel(), 4).reshape(16, 16)
    for q in range(4):
        blk = np.argwhere(p == q)
        assert len(blk) == 64 and np.ptp(blk[:, 0]) == 7 and np.ptp(blk[:, 1]) == 7
    # Figure 1 chain: tridiagonal 6x6, P=2, rank 0 -> owned {0,1,2}, halo {3}, send {2}, recv {3}
    n = 6
    r = [i for i in range(n) for j in (i - 1, i, i + 1) if 0 <= j < n]
    c = [j for i in range(n) for j in (i - 1, i, i + 1) if 0 <= j < n]
    A = O.csr_from_triplets(n, n, r, c, [2.0 if a == b else -1.0 for a, b in zip(r, c)])
    L = O.build_local(A, O.partition_contiguous(6, 2), 2, 0)
    assert list(L["owned"]) == [0, 1, 2] and list(L["halo"]) == [3]
    assert list(L["send_idx"]) == [2] and list(L["recv_idx"]) == [3]  # local positions
    D = O.csr_from_triplets(5, 5, range(5), range(5), np.ones(5))
    L = O.build_local(D, O.partition_contiguous(5, 2), 2, 1)
    assert len(L["halo"]) == 0 and len(L["neighbors"]) == 0
    P8 = O.generate("poisson2d", 8)
    for rank in (0, 1):
        assert len(O.build_local(P8, O.partition_contiguous(64, 2), 2, rank)["halo"]) == 8


def test_spec_distributed(O):
    P = O.generate("poisson2d", 16)
    b = np.ones(P.nrows)
    xs, rs = O.cg(P, b, atol=1e-10)
    x1, r1, c1 = O.dist_solve(P, b, O.partition_contiguous(P.nrows, 1), 1, atol=1e-10)
    assert np.array_equal(bits(x1), bits(xs)) and r1["iterations"] == rs["iterations"]
    assert c1["messages"] == 0
    for N, Pn, part in [(32, 2, "contig"), (32, 3, "contig"), (32, 4, "contig"),
                        (64, 4, "rcb"), (32, 2, "rcb")]:
        A = O.generate("poisson2d", N)
        b = np.ones(A.nrows)
        po = (O.partition_contiguous(A.nrows, Pn) if part == "contig"
              else O.partition_rcb(*O.gen_coords("poisson2d", N), Pn))
        xs, rs = O.cg(A, b, atol=1e-10)
        xd, rd, cnt = O.dist_solve(A, b, po, Pn, atol=1e-10)
        assert rd["iterations"] == rs["iterations"], (N, Pn, part)
        assert np.max(np.abs(xd - xs)) <= 1e-10
        # 1 halo exchange per spmv (1 + k) and 2 all_reduce per iteration (+1 init point)
        assert cnt["halo_exchanges"] == 1 + rd["iterations"]
        assert cnt["all_reduces"] == 1 + 2 * rd["iterations"]
        y = O.dist_spmv(A, xs, po, Pn)
        assert np.array_equal(bits(y), bits(O.spmv(A, xs)))  # 0 ulps per row
    # contiguous N x N: interior-rank halo == 2N (two grid rows), edge ranks N
    A = O.generate("poisson2d", 32)
    po = O.partition_contiguous(A.nrows, 4)
    assert [len(O.build_local(A, po, 4, r)["halo"]) for r in range(4)] == [32, 64, 64, 32]
    # distributed adjoint == serial adjoint
    A = O.generate("poisson2d", 32)
    b = np.ones(A.nrows)
    x, _ = O.cg(A, b, atol=1e-12)
    gb, gv, _ = O.adjoint_backward(A, x, np.ones(A.nrows), atol=1e-12)
    gbd, gvd, _ = O.dist_adjoint(A, x, np.ones(A.nrows), O.partition_contiguous(A.nrows, 2), 2,
                                 atol=1e-12)
    assert np.max(np.abs(gbd - gb)) <= 1e-9 * np.max(np.abs(gb))
    assert np.max(np.abs(gvd - gv)) <= 1e-9 * np.max(np.abs(gv))


def test_oracle_thread_count_invariance(O):
    A = O.generate("poisson3d", 48)
    b = np.ones(A.nrows)
    O.set_threads(1)
    x1, _ = O.cg_fixed(A, b, 10)
    O.set_threads(os.cpu_count() or 1)
    x2, _ = O.cg_fixed(A, b, 10)
    assert np.array_equal(bits(x1), bits(x2))
