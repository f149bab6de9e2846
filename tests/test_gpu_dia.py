"""Diagonal-warp SpMV (csrc/spmv_dia.cuh): 32-row warps whose rows all sit on the same <= 7
diagonals with the same dictionary values (up to two missing entries: the x-boundary rows of
a stencil line) are described by one 48-byte table entry instead of their CSR, and x is read
with coalesced loads along each diagonal; other warps run the CSR loop.  The arithmetic is
the reference's row-ordered sum (sparse.cpp:144-152) in stored column order, so every SpMV
and every Krylov trajectory must stay bit-identical to the oracle."""
import numpy as np
import pytest

from test_gpu_parity import _banded, assert_bitwise, random_csr, rep_eq, to_S

pytestmark = pytest.mark.gpu


def _gen(O, case):
    if case == "poisson3d":      # 40-row lines: exceptions + unstructured plane-boundary warps
        return O.generate("poisson3d", 40)
    if case == "poisson3d_odd":  # 37-row lines, 50653 rows: a partial last warp and chunk
        return O.generate("poisson3d", 37)
    if case == "poisson2d":      # 300-row lines, 5 diagonals, 90000 rows (partial warp)
        return O.generate("poisson2d", 300)
    if case == "convdiff3d":     # non-symmetric values per direction
        return O.generate("convdiff3d", 40, 0, 0.3)
    if case == "banded_far":     # 7 diagonals far apart
        return _banded(O, 70000, (1, 300, 2000), 20.0, -1.0)
    if case == "perturbed":      # one row with a different off-diagonal value: its warp is unstructured
        A = O.generate("poisson3d", 40)
        v = A.vals.copy()
        k = int(A.row_ptr[20001]) + 1
        v[k] = -1.25
        return O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v)
    raise ValueError(case)


CASES = ["poisson3d", "poisson3d_odd", "poisson2d", "convdiff3d", "banded_far", "perturbed"]


@pytest.fixture(autouse=True)
def _dia_on(monkeypatch):
    """The diagonal-warp kernel (the default for stencils; SPARSLA_DIA=1 set explicitly)."""
    monkeypatch.setenv("SPARSLA_DIA", "1")


@pytest.mark.parametrize("variant", list(range(18)))
def test_dia_variants_bitwise(S, O, gpu, monkeypatch, variant):
    """Every kDiaVariants entry (1 or 2 rounds per step, occupancy), odd round counts."""
    monkeypatch.setenv("SPARSLA_DIA_VARIANT", str(variant))
    for case in CASES:
        A = _gen(O, case)
        D = to_S(S, A).device(0)
        assert D.dia()["on"]
        x = np.random.default_rng(variant).standard_normal(A.ncols)
        assert_bitwise(S.spmv(D, x), O.spmv(A, x), f"{case} variant {variant}")


def test_dia_selection(S, O, gpu, monkeypatch):
    """On (every SpMV mode) for stencils (>= 90% structured warps), off for scattered
    columns and for matrices without a value dictionary, and with SPARSLA_DIA=0."""
    D = to_S(S, O.generate("poisson3d", 40)).device(0)
    d = D.dia()
    assert d["on"] and 0.9 <= d["structured"] < 1.0 and d["bytes"] > 0, d
    # 48 B per 32 rows plus the unstructured warps' CSR: far below the 12 B/entry CSR
    assert d["bytes"] < 0.2 * 12 * O.generate("poisson3d", 40).nnz, d
    assert not to_S(S, random_csr(O, 20000, 20000, 9, 1)).device(0).dia()["on"]
    assert not to_S(S, O.generate("fem2d", 200, 2601, 0.0)).device(0).dia()["on"]  # no dictionary
    monkeypatch.delenv("SPARSLA_DIA")
    d = to_S(S, O.generate("poisson3d", 40)).device(0).dia()
    assert d["on"] and d["modes"] == [0, 1, 2, 3], d
    # default kernel: the pattern table (a 3-D stencil has a handful of diagonal/value
    # patterns: interior, boundary planes and lines), 4 bytes per warp
    assert 1 <= d["patterns"] <= 64, d
    monkeypatch.setenv("SPARSLA_DIA", "0")
    d = to_S(S, O.generate("poisson3d", 40)).device(0).dia()
    assert d["modes"] == [] and d["structured"] == 0, d


@pytest.mark.parametrize("case", CASES)
def test_dia_spmv_bitwise(S, O, gpu, case):
    A = _gen(O, case)
    D = to_S(S, A).device(0)
    d = D.dia()
    assert d["on"], d
    if case == "perturbed":
        assert d["structured"] < 1.0
    x = np.random.default_rng(5).standard_normal(A.ncols)
    assert_bitwise(S.spmv(D, x), O.spmv(A, x), case)
    x[::7] = 0.0
    x[3::11] = -0.0
    assert_bitwise(S.spmv(D, x), O.spmv(A, x), case + " (signed zeros)")


@pytest.mark.parametrize("case", ["poisson3d", "poisson3d_odd", "poisson2d", "banded_far"])
@pytest.mark.parametrize("fused", ["0", "1"])
def test_dia_cg_trajectory_bitwise(S, O, gpu, monkeypatch, case, fused):
    """CG p.q fused into the diagonal-warp SpMV; fused=1 lets small problems take the fused
    CG kernel (which has its own SpMV), fused=0 forces the per-kernel path."""
    monkeypatch.setenv("SPARSLA_FUSED", fused)
    A = _gen(O, case)
    D = to_S(S, A).device(0)
    assert D.dia()["on"]
    b = np.linspace(0.5, 1.5, A.nrows)
    xo, ro = O.cg(A, b, atol=0.0, rtol=1e-10, max_iter=20000)
    x, r = S.cg_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=20000))
    assert ro["converged"]
    rep_eq(r, ro)
    assert_bitwise(x, xo, case)


@pytest.mark.parametrize("case", ["convdiff3d", "poisson3d_odd"])
def test_dia_bicgstab_trajectory_bitwise(S, O, gpu, case):
    """BiCGStab r-hat.v and t.t / t.s fused into the diagonal-warp SpMV."""
    A = _gen(O, case)
    D = to_S(S, A).device(0)
    assert D.dia()["on"]
    b = np.ones(A.nrows)
    xo, ro = O.bicgstab(A, b, atol=0.0, rtol=1e-9, max_iter=5000)
    x, r = S.bicgstab_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-9, max_iter=5000))
    assert ro["converged"]
    rep_eq(r, ro)
    assert_bitwise(x, xo, case)


def test_dia_set_values(S, O, gpu):
    """The table follows the values: > 256 distinct values drop the dictionary (and the
    table), restoring them rebuilds it, new stencil values rebuild it — bitwise throughout."""
    A = O.generate("poisson3d", 40)
    D = to_S(S, A).device(0)
    x = np.random.default_rng(9).standard_normal(A.ncols)
    v2 = A.vals * (1.0 + 1e-3 * np.arange(A.nnz) / A.nnz)
    D.set_values(v2)
    assert not D.dia()["on"]
    assert_bitwise(S.spmv(D, x), O.spmv(O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v2), x))
    D.set_values(A.vals)
    assert D.dia()["on"]
    assert_bitwise(S.spmv(D, x), O.spmv(A, x))
    v3 = np.where(A.vals < 0, -1.5, A.vals)
    D.set_values(v3)
    assert D.dia()["on"]
    assert_bitwise(S.spmv(D, x), O.spmv(O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v3), x))


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("kind,p1,P,solver", [("poisson3d", 40, 2, "cg"), ("convdiff3d", 40, 2, "bicgstab")])
def test_dia_distributed_bitwise(S, O, gpu, kind, p1, P, solver, fused):
    """Rank-local matrices ([owned | halo] columns: the halo diagonals are contiguous in the
    halo block) through the diagonal-warp kernel, interior chunks while the halo moves
    (transport) or boundary chunks after the peers' pushes (fused peer memory)."""
    from test_gpu_dist import Ocsr, bits, make_plans, partition
    A = S.generate(kind, p1, 0, 0.3 if kind == "convdiff3d" else 1.0)
    po = partition(S, kind, p1, A, P, "contig")
    hub, plans, owned = make_plans(S, A, po, P)
    for p in plans:
        assert p.dia()["structured"] > 0.5, p.dia()
        p.set_fused(fused)
    b = np.ones(A.nrows)
    opts = S.SolveOptions(atol=0.0, rtol=1e-9, max_iter=5000)
    res = S.run_ranks(P, lambda r: (plans[r].cg if solver == "cg" else plans[r].bicgstab)(b[owned[r]], opts))
    xd = np.empty(A.nrows)
    for r in range(P):
        xd[owned[r]] = res[r][0]
    xo, ro, co = O.dist_solve(Ocsr(O, A), b, po, P, kind=solver, atol=0.0, rtol=1e-9, max_iter=5000)
    rep = res[0][1]
    assert rep.converged and rep.iterations == ro["iterations"], (rep, ro)
    assert np.array_equal(bits(xd), bits(xo))


def _many_patterns(O, n, npat):
    """Tridiagonal, every 32-row warp with its own off-diagonal value (npat distinct, cycling;
    nonsymmetric, diagonally dominant): warps share diagonals but not values -> npat distinct
    structured patterns."""
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
                vals.append(4.0 if i == j else -(1.0 + ((i // 32) % npat) / 128.0))
    return O.csr_from_triplets(n, n, rows, cols, vals)


@pytest.mark.parametrize("npat", [40, 100])
def test_dia_pattern_table_limit(S, O, gpu, monkeypatch, npat):
    """<= 64 distinct patterns: the pattern-table kernel; more: the 48-byte-entry kernel
    (patterns == 0).  Both bit-identical to the oracle (SpMV and a BiCGStab trajectory)."""
    monkeypatch.delenv("SPARSLA_DIA_VARIANT", raising=False)
    A = _many_patterns(O, 32 * 300 + 17, npat)
    D = to_S(S, A).device(0)
    d = D.dia()
    assert d["on"], d
    if npat <= 64:
        assert 1 <= d["patterns"] <= 64, d
    else:
        assert d["patterns"] == 0, d
    x = np.random.default_rng(npat).standard_normal(A.ncols)
    assert_bitwise(S.spmv(D, x), O.spmv(A, x), f"{npat} patterns")
    b = np.linspace(0.5, 1.5, A.nrows)
    xo, ro = O.bicgstab(A, b, atol=0.0, rtol=1e-10, max_iter=5000)
    xg, rg = S.bicgstab_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=5000))
    assert ro["converged"]
    rep_eq(rg, ro)
    assert_bitwise(xg, xo, f"{npat} patterns BiCGStab")
