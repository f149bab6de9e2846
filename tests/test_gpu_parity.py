"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar (north star / SURVEY.md §8): integer and structural data bit-exact; SpMV bit-exact with
the reference's row-ordered accumulation (sparse.cpp:144-152); Krylov trajectories bit-exact
with the oracle (canonical dots, same operation order), hence identical iteration counts and
||x - x_ref|| / ||x_ref|| = 0 <= 1e-8; adjoint gradients bit-exact (<= 1e-7 relative).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def assert_bitwise(a, b, what=""):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert a.shape == b.shape, what
    diff = np.nonzero(bits(a) != bits(b))[0]
    assert len(diff) == 0, f"{what}: {len(diff)} entries differ, first at {diff[:5]}: " \
                           f"{a[diff[:5]]} vs {b[diff[:5]]}"


def to_S(S, A):
    return S.CsrMatrix(A.nrows, A.ncols, A.row_ptr, A.col_idx, A.vals)


def random_csr(O, n, m, density_rows, seed, long_rows=()):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        k = int(rng.integers(0, density_rows + 1))
        if i in long_rows:
            k = long_rows[i] if isinstance(long_rows, dict) else 3000
        c = rng.choice(m, size=min(k, m), replace=False)
        rows += [i] * len(c)
        cols += list(c)
    vals = rng.standard_normal(len(rows))
    return O.csr_from_triplets(n, m, rows, cols, vals)


GENS = [("poisson2d", 37, 0, 0.0), ("poisson3d", 17, 0, 0.0), ("convdiff3d", 13, 0, 1.0),
        ("fem2d", 60, 2601, 0.0)]


@pytest.mark.parametrize("kind,p1,p2,fp", GENS)
def test_spmv_bitwise_generators(S, O, gpu, kind, p1, p2, fp):
    A = O.generate(kind, p1, p2, fp)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(A.ncols)
    assert_bitwise(S.spmv(to_S(S, A), x), O.spmv(A, x), kind)


def test_spmv_spec_examples(S, O, gpu):
    # I x = x; Poisson 3x3 grid * ones = {corner 2, edge 1, centre 0}; [[2,0],[1,3]][1,1]=[2,4]
    I = S.CsrMatrix.from_coo(S.SparseCoo(range(5), range(5), np.ones(5), (5, 5)))
    x = np.array([1.5, -2.0, 3.25, 0.0, 7.0])
    assert_bitwise(S.spmv(I, x), x)
    A, _ = S.poisson2d(3)
    assert list(S.spmv(A, np.ones(9))) == [2, 1, 2, 1, 0, 1, 2, 1, 2]
    B = S.CsrMatrix.from_coo(S.SparseCoo([0, 1, 1], [0, 0, 1], [2.0, 1.0, 3.0], (2, 2)))
    assert list(S.spmv(B, [1, 1])) == [2.0, 4.0]
    T = S.CsrMatrix.from_coo(S.SparseCoo([0], [1], [1.0], (2, 2)))
    assert list(S.spmv_transpose(T, [1, 0])) == [0.0, 1.0]
    with pytest.raises(S.DimensionError):
        S.spmv(B, [1, 1, 1])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_spmv_random_rectangular_and_ragged(S, O, gpu, seed):
    A = random_csr(O, 3001 + seed, 2500, 12, seed)  # empty rows, ragged rows, n % 2048 != 0
    x = np.random.default_rng(seed).standard_normal(A.ncols)
    D = to_S(S, A).device(0)
    assert D.info()["variant"] == 0
    assert_bitwise(S.spmv(D, x), O.spmv(A, x))
    # spmv_transpose == row-ordered spmv on canonical A^T (== reference scatter order)
    y = np.random.default_rng(seed + 7).standard_normal(A.nrows)
    assert_bitwise(S.spmv_transpose(D, y), O.spmv(O.transpose(A), y))


def test_spmv_long_rows_hub_bypass(S, O, gpu, monkeypatch):
    """Rounds larger than a ring stage (hub rows) bypass the smem ring inside the staged
    kernel; everything stays bit-exact, incl. the fused dot and CG.  (Long-row split off, so
    the staged kernel itself meets the hubs.)"""
    monkeypatch.setenv("SPARSLA_LONG_ROW", "0")
    A = random_csr(O, 5000, 5000, 5, 3, long_rows={3: 4000, 500: 4500, 4999: 3000})
    D = to_S(S, A).device(0)
    assert D.info()["variant"] == 0
    x = np.random.default_rng(3).standard_normal(A.ncols)
    assert_bitwise(S.spmv(D, x), O.spmv(A, x))


def test_spmv_direct_kernel(S, O, gpu, monkeypatch):
    monkeypatch.setenv("SPARSLA_SPMV_DIRECT", "1")
    A = random_csr(O, 3100, 3000, 9, 4, long_rows={7: 2500})
    D = to_S(S, A).device(0)
    assert D.info()["variant"] == 1
    x = np.random.default_rng(4).standard_normal(A.ncols)
    assert_bitwise(S.spmv(D, x), O.spmv(A, x))
    P = O.generate("poisson2d", 50)
    DP = to_S(S, P).device(0)
    b = np.ones(P.nrows)
    xo, ro = O.cg(P, b, atol=0.0, rtol=1e-9)
    xg, rg = S.cg_solve(DP, b, S.SolveOptions(atol=0.0, rtol=1e-9))
    rep_eq(rg, ro)
    assert_bitwise(xg, xo)


@pytest.mark.parametrize("n", [1, 2, 3, 2047, 2048, 2049, 4097, 300001, 2_100_000])
def test_canonical_dot(S, O, gpu, n):
    rng = np.random.default_rng(n)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    assert bits([S.dot(a, b)])[0] == bits([O.cdot(a, b)])[0]


def test_jacobi(S, O, gpu):
    A = O.csr_from_triplets(4, 4, [0, 1, 2, 3, 0], [0, 1, 3, 3, 1], [2.0, 0.0, 1.0, 4.0, 5.0])
    d = S.jacobi_build(to_S(S, A)).inv_diag
    assert list(d) == [0.5, 1.0, 1.0, 0.25]  # A_11 = 0 -> 1.0, A_22 missing -> 1.0
    P = O.generate("poisson2d", 8)
    assert np.all(S.jacobi_build(to_S(S, P)).inv_diag == 0.25)
    F = O.generate("fem2d", 50, 2601)
    assert_bitwise(S.jacobi_build(to_S(S, F)).inv_diag, O.jacobi(F))


def rep_eq(r, ro):
    assert r.iterations == ro["iterations"], (r, ro)
    assert r.spmv_count == ro["spmv_count"], (r, ro)
    assert r.converged == ro["converged"], (r, ro)
    assert bits([r.residual_norm])[0] == bits([ro["residual_norm"]])[0], (r, ro)
    assert r.diagnostic == ro["diagnostic"], (r, ro)


CG_CASES = [("poisson2d", 64, 0, 0.0, 1e-8), ("poisson3d", 24, 0, 0.0, 1e-8),
            ("fem2d", 90, 2601, 0.0, 1e-8), ("poisson2d", 150, 0, 0.0, 1e-10)]


@pytest.mark.parametrize("kind,p1,p2,fp,rtol", CG_CASES)
def test_cg_bitwise_trajectory(S, O, gpu, kind, p1, p2, fp, rtol):
    A = O.generate(kind, p1, p2, fp)
    b = np.ones(A.nrows)
    xo, ro = O.cg(A, b, atol=0.0, rtol=rtol, max_iter=20000)
    x, r = S.cg_solve(to_S(S, A), b, S.SolveOptions(atol=0.0, rtol=rtol, max_iter=20000))
    assert ro["converged"]
    rep_eq(r, ro)
    assert_bitwise(x, xo, kind)


def test_cg_spec_examples(S, O, gpu):
    A = S.CsrMatrix.from_coo(S.SparseCoo(range(4), range(4), [2.0] * 4, (4, 4)))
    x, r = S.cg_solve(A, [2, 4, 6, 8])
    assert list(x) == [1, 2, 3, 4] and r.iterations == 1 and r.converged and r.spmv_count == 2
    P, b = S.poisson2d(32)
    x, r = S.cg_solve(P, b, S.SolveOptions(atol=1e-10))
    assert r.converged and r.residual_norm <= 1e-10 and r.spmv_count == 1 + r.iterations
    xd = np.linalg.solve(S.SparseCoo(*_coo(P), (1024, 1024)).to_dense(), b)
    assert np.max(np.abs(x - xd)) <= 1e-8
    x1, r1 = S.cg_solve(P, b, S.SolveOptions(atol=1e-10, max_iter=1))
    assert not r1.converged and r1.residual_norm > 1e-10 and r1.diagnostic == "max_iter reached"
    # indefinite: p^T A p <= 0 breakdown is reported, not raised
    N = S.CsrMatrix.from_coo(S.SparseCoo(range(3), range(3), [-1.0, -2.0, -3.0], (3, 3)))
    xn, rn = S.cg_solve(N, [1, 1, 1])
    assert not rn.converged and rn.diagnostic.startswith("breakdown: p^T A p <= 0")
    with pytest.raises(S.InvalidArgumentError):
        S.cg_solve(P, b, S.SolveOptions(atol=0.0, rtol=0.0))


def _coo(A):
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    return rows, A.col_idx, A.vals


def test_cg_iteration_scaling(S, gpu):
    its = []
    for N in (16, 32, 64, 128):
        P, b = S.poisson2d(N)
        its.append(S.cg_solve(P, b, S.SolveOptions(atol=1e-10))[1].iterations)
    ratios = [its[i + 1] / its[i] for i in range(3)]
    assert all(1.5 <= q <= 3.0 for q in ratios), its


BI_CASES = [("convdiff3d", 16, 0, 1.0), ("convdiff3d", 24, 0, 0.3), ("poisson2d", 40, 0, 0.0),
            ("fem2d", 50, 2601, 0.0)]


@pytest.mark.parametrize("kind,p1,p2,fp", BI_CASES)
def test_bicgstab_bitwise_trajectory(S, O, gpu, kind, p1, p2, fp):
    A = O.generate(kind, p1, p2, fp)
    b = np.ones(A.nrows)
    xo, ro = O.bicgstab(A, b, atol=0.0, rtol=1e-8, max_iter=5000)
    x, r = S.bicgstab_solve(to_S(S, A), b, S.SolveOptions(atol=0.0, rtol=1e-8, max_iter=5000))
    assert ro["converged"]
    rep_eq(r, ro)
    assert_bitwise(x, xo, kind)


def test_bicgstab_spec_examples(S, O, gpu):
    A = S.CsrMatrix.from_coo(S.SparseCoo([0, 0, 1], [0, 1, 1], [4.0, 1.0, 3.0], (2, 2)))
    x, r = S.bicgstab_solve(A, [5, 3])
    assert r.converged and np.allclose(x, [1, 1], atol=1e-12)
    xo, ro = O.bicgstab(O.csr_from_triplets(2, 2, [0, 0, 1], [0, 1, 1], [4.0, 1.0, 3.0]), [5, 3])
    rep_eq(r, ro)
    assert_bitwise(x, xo)
    P, b = S.poisson2d(16)
    xb, rb = S.bicgstab_solve(P, b, S.SolveOptions(atol=1e-12))
    xc, rc = S.cg_solve(P, b, S.SolveOptions(atol=1e-12))
    assert np.max(np.abs(xb - xc)) <= 1e-8
    Z = S.CsrMatrix(2, 2, [0, 0, 0], [], [])
    xz, rz = S.bicgstab_solve(Z, [1, 1])
    assert not rz.converged and rz.diagnostic.startswith("breakdown")


def test_adjoint_spec_examples(S, O, gpu):
    A = S.SparseCoo(range(3), range(3), [2.0, 2.0, 2.0], (3, 3))
    x, ctx, rep = S.solve_forward(A, [2, 4, 6])
    assert list(x) == [1, 2, 3]
    g = S.solve_backward(ctx, np.ones(3))
    assert list(g.grad_b) == [0.5, 0.5, 0.5]
    assert list(g.grad_vals) == [-0.5, -1.0, -1.5]
    I = S.SparseCoo(range(4), range(4), np.ones(4), (4, 4))
    gx = np.array([1.0, -2.0, 3.0, 0.5])
    xi, ci, _ = S.solve_forward(I, [4.0, 3.0, 2.0, 1.0])
    gi = S.solve_backward(ci, gx)
    assert_bitwise(gi.grad_b, gx)
    assert_bitwise(gi.grad_vals, -(gx * xi))
    z = S.solve_backward(ci, np.zeros(4))  # short-circuit: zero gradients, zero iterations
    assert np.all(z.grad_b == 0) and np.all(z.grad_vals == 0) and z.report.iterations == 0


@pytest.mark.parametrize("kind,p1,fp,backend", [("poisson2d", 40, 0.0, 0), ("fem2d", 45, 0.0, 0),
                                                 ("convdiff3d", 12, 1.0, 1)])
def test_adjoint_bitwise(S, O, gpu, kind, p1, fp, backend):
    A = O.generate(kind, p1, 2601 if kind == "fem2d" else 0, fp)
    b = np.ones(A.nrows)
    solve = O.bicgstab if backend else O.cg
    xo, _ = solve(A, b, atol=1e-12)
    g = np.random.default_rng(5).standard_normal(A.nrows)
    gbo, gvo, ro = O.adjoint_backward(A, xo, g, backend=backend, atol=1e-12)
    coo = S.SparseCoo(*_coo(A), (A.nrows, A.ncols))
    x, ctx, _ = S.solve_forward(coo, b, S.SolveOptions(atol=1e-12),
                                backend="bicgstab" if backend else "cg")
    assert_bitwise(x, xo)
    gr = S.solve_backward(ctx, g, S.SolveOptions(atol=1e-12), backend="bicgstab" if backend else "cg")
    rep_eq(gr.report, ro)
    assert_bitwise(gr.grad_b, gbo)
    assert_bitwise(gr.grad_vals, gvo)
    # linearity in grad_x
    g2 = np.random.default_rng(6).standard_normal(A.nrows)
    ga = S.solve_backward(ctx, g, S.SolveOptions(atol=1e-13))
    gb = S.solve_backward(ctx, g2, S.SolveOptions(atol=1e-13))
    gc = S.solve_backward(ctx, 2.0 * g - 3.0 * g2, S.SolveOptions(atol=1e-13))
    ref = 2.0 * ga.grad_b - 3.0 * gb.grad_b
    assert np.max(np.abs(gc.grad_b - ref)) <= 1e-7 * np.max(np.abs(ref))


def test_config_A_full(S, O, gpu):
    """BASELINE configs[0]: 2-D Poisson 1000x1000, Jacobi-PCG to rel-res 1e-8."""
    A = O.generate("poisson2d", 1000)
    b = np.ones(A.nrows)
    xo, ro = O.cg(A, b, atol=0.0, rtol=1e-8, max_iter=100000)
    x, r = S.cg_solve(to_S(S, A), b, S.SolveOptions(atol=0.0, rtol=1e-8, max_iter=100000))
    assert ro["iterations"] == 1853
    rep_eq(r, ro)
    assert_bitwise(x, xo)


@pytest.mark.parametrize("fused", ["1", "0"])
def test_persistent_solver_fixed_iterations(S, O, gpu, monkeypatch, fused):
    """Solver.iterate(k) after reset == oracle CG truncated at k iterations, bitwise.  With
    the multi-kernel loop (SPARSLA_FUSED=0) x is updated every other iteration from two
    direction buffers: odd k leave a lagging step that reading x must flush, and the solve
    must continue bit-exactly after such a mid-solve read."""
    monkeypatch.setenv("SPARSLA_FUSED", fused)
    A = O.generate("poisson3d", 64)
    b = np.ones(A.nrows)
    sv = S.Solver(to_S(S, A), b, "cg", S.SolveOptions(atol=0.0, rtol=1e-30, max_iter=10**6))
    for k in (1, 2, 7, 40):
        sv.reset()
        sv.iterate(k)
        xo, _ = O.cg_fixed(A, b, k)
        assert sv.report().iterations == k
        assert_bitwise(sv.x(), xo, f"k={k}")
    sv.reset()
    for k0, k in ((3, 3), (4, 7), (17, 24), (1, 25)):  # reads after odd and even counts
        sv.iterate(k0)
        xo, _ = O.cg_fixed(A, b, k)
        assert_bitwise(sv.x(), xo, f"resumed k={k}")
    rep = sv.report()
    assert rep.iterations == 25


@pytest.mark.parametrize("kind,p1,p2,fp,backend", [("poisson3d", 40, 0, 0.0, "cg"), ("poisson2d", 200, 0, 0.0, "cg"),
                                                   ("convdiff3d", 24, 0, 0.1, "bicgstab"),
                                                   # row counts that leave idle lanes in the last round
                                                   ("poisson3d", 13, 0, 0.0, "cg"), ("poisson2d", 37, 0, 0.0, "cg"),
                                                   ("convdiff3d", 11, 0, 0.3, "bicgstab")])
def test_value_dictionary_and_scalar_diagonal_bitwise(S, O, gpu, monkeypatch, kind, p1, p2, fp, backend):
    """Stored-format choices are invisible in the results: the 1-byte value dictionary
    (<= 256 distinct values) and the scalar constant Jacobi diagonal give the same bits as
    plain CSR with a streamed diagonal, and as the oracle."""
    A = O.generate(kind, p1, p2, fp)
    b = np.random.default_rng(5).standard_normal(A.nrows)
    opts = S.SolveOptions(atol=0.0, rtol=1e-9, max_iter=20000)
    fn = S.cg_solve if backend == "cg" else S.bicgstab_solve
    D1 = to_S(S, A).device(0)
    f1 = D1.format()
    assert f1["value_dict"] and f1["distinct_values"] <= 4 and f1["uniform_diag"], f1
    x1, r1 = fn(D1, b, opts)
    y1 = S.spmv(D1, b)
    monkeypatch.setenv("SPARSLA_VALUE_DICT", "0")
    monkeypatch.setenv("SPARSLA_UNIFORM_DIAG", "0")
    D2 = to_S(S, A).device(0)
    assert not D2.format()["value_dict"]
    x2, r2 = fn(D2, b, opts)
    assert r1.iterations == r2.iterations and r1.converged
    assert_bitwise(x1, x2, "dictionary/scalar-diagonal vs plain solve")
    assert_bitwise(y1, S.spmv(D2, b), "dictionary vs plain spmv")
    assert_bitwise(y1, O.spmv(A, b), "dictionary spmv vs oracle")
    xo, ro = (O.cg if backend == "cg" else O.bicgstab)(A, b, atol=0.0, rtol=1e-9, max_iter=20000)
    assert ro["iterations"] == r1.iterations
    assert_bitwise(x1, xo, "vs oracle")


def test_value_dictionary_rebuilt_by_set_values(S, O, gpu):
    """set_values (= SparseCoo::with_values) rebuilds the dictionary; more than 256 distinct
    values fall back to the plain value stream, still bit-exact."""
    A = O.generate("poisson3d", 20)
    D = to_S(S, A).device(0)
    assert D.format()["value_dict"]
    rng = np.random.default_rng(9)
    v2 = A.vals * (1.0 + 0.01 * rng.random(len(A.vals)))  # all distinct
    S.lib().sparsla_dcsr_set_values(D.h, v2.ctypes.data_as(S._f64p), 0)
    assert not D.format()["value_dict"]
    x = rng.standard_normal(A.ncols)
    A2 = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v2)
    assert_bitwise(S.spmv(D, x), O.spmv(A2, x))
    v3 = np.where(A.vals > 0, 7.5, -1.25)
    S.lib().sparsla_dcsr_set_values(D.h, v3.ctypes.data_as(S._f64p), 0)
    assert D.format()["value_dict"] and D.format()["distinct_values"] == 2
    A3 = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v3)
    assert_bitwise(S.spmv(D, x), O.spmv(A3, x))


@pytest.mark.parametrize("nvals", [1, 255, 256, 257])
def test_value_dictionary_limits_and_signed_zero(S, O, gpu, nvals):
    """Dictionary selection is by bit pattern: 256 distinct values use it, 257 fall back;
    -0.0 and +0.0 are distinct entries, and either way the SpMV is bitwise the oracle's."""
    A = O.generate("poisson3d", 14)
    nnz = len(A.vals)
    pool = np.linspace(-3.0, 3.0, nvals)
    if nvals >= 2:
        pool[0], pool[1] = 0.0, -0.0
    vals = pool[np.arange(nnz) % nvals]
    B = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, vals)
    D = to_S(S, B).device(0)
    f = D.format()
    distinct = len(np.unique(pool.view(np.int64)))
    assert f["value_dict"] == (distinct <= 256), f
    if f["value_dict"]:
        assert f["distinct_values"] == distinct
    x = np.random.default_rng(nvals).standard_normal(A.ncols)
    x[::7] = -x[::7]
    assert_bitwise(S.spmv(D, x), O.spmv(B, x), f"{nvals} values")


def test_parked_solver_reuse_bitwise(S, O, gpu, monkeypatch):
    """Host-buffer solves on one matrix handle reuse its parked solver (workspace + graphs):
    different tolerances, right-hand sides and backends, then new values — every result is
    bit-identical to a fresh solver (SPARSLA_SOLVER_CACHE=0) and to the oracle."""
    A = O.generate("convdiff3d", 18, 0, 0.2)
    D = to_S(S, A).device(0)
    rng = np.random.default_rng(3)
    runs = [("bicgstab", 1e-6), ("bicgstab", 1e-10), ("cg", 1e-8), ("bicgstab", 1e-8)]
    out = []
    for be, rtol in runs:
        b = rng.standard_normal(A.nrows)
        fn = S.cg_solve if be == "cg" else S.bicgstab_solve
        x, r = fn(D, b, S.SolveOptions(atol=0.0, rtol=rtol, max_iter=3000))
        out.append((be, rtol, b, x, r))
    v2 = np.where(A.vals > 0, A.vals * 1.5, A.vals)
    S.lib().sparsla_dcsr_set_values(D.h, v2.ctypes.data_as(S._f64p), 0)
    b = rng.standard_normal(A.nrows)
    x2, r2 = S.bicgstab_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-9, max_iter=3000))
    out.append(("bicgstab", 1e-9, b, x2, r2, v2))
    monkeypatch.setenv("SPARSLA_SOLVER_CACHE", "0")
    for item in out:
        be, rtol, b, x, r = item[:5]
        vals = item[5] if len(item) > 5 else A.vals
        Ao = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, vals)
        xo, ro = (O.cg if be == "cg" else O.bicgstab)(Ao, b, atol=0.0, rtol=rtol, max_iter=3000)
        assert r.iterations == ro["iterations"], (be, rtol)
        assert_bitwise(x, xo, f"{be} rtol={rtol}")


def test_value_dictionary_empty_rows_and_partial_rounds(S, O, gpu):
    """Dictionary SpMV on a stencil with emptied rows and a row count that ends mid-round:
    empty rows give exactly 0.0, every other row the oracle's bits."""
    A = O.generate("poisson3d", 19)  # 6859 rows: the last 256-row round is partial
    n = A.nrows
    keep = np.ones(A.nnz, bool)
    rows = np.repeat(np.arange(n), np.diff(A.row_ptr))
    keep[(rows % 7) == 3] = False
    B = O.csr_from_triplets(n, n, rows[keep], A.col_idx[keep], A.vals[keep])
    assert (np.diff(B.row_ptr) == 0).sum() > 0
    D = to_S(S, B).device(0)
    assert D.format()["value_dict"]
    x = np.random.default_rng(4).standard_normal(n)
    y = S.spmv(D, x)
    assert_bitwise(y, O.spmv(B, x))
    assert np.all(y[np.diff(B.row_ptr) == 0] == 0.0)


def _banded(O, n, offsets, diag, off, extra_vals=None):
    """Symmetric diagonally dominant band matrix (CG-safe): diag on the diagonal, `off` on
    +-offsets; extra_vals (optional) varies the off-diagonal values (more distinct values)."""
    rows, cols, vals = [], [], []
    for i in range(n):
        for o in sorted([-d for d in offsets] + [0] + list(offsets)):
            j = i + o
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
                v = diag if o == 0 else off
                if extra_vals is not None and o != 0:
                    v = off * (1.0 + extra_vals * ((min(i, j) * 7919) % 1000) / 1000.0)
                vals.append(v)
    return O.csr_from_triplets(n, n, rows, cols, vals)


@pytest.mark.parametrize("case", ["resident", "far_columns", "dense_chunks", "no_dictionary"])
def test_fused_cg_resident_images_and_fallbacks(S, O, gpu, case):
    """The fused small-problem CG keeps chunk images resident in shared memory when every
    entry is within 2^15 of the diagonal, a chunk holds <= 65535 entries and the values form
    a dictionary; otherwise it runs the non-resident kernel.  Every case's trajectory equals
    the oracle's bit for bit."""
    if case == "resident":
        A = _banded(O, 30000, (1, 150), 5.0, -1.0)
    elif case == "far_columns":      # +-40000 > int16: no resident image
        A = _banded(O, 90000, (1, 40000), 5.0, -1.0)
    elif case == "dense_chunks":     # 2048 rows x 41 entries > 65535 per chunk
        A = _banded(O, 6000, tuple(range(1, 21)), 45.0, -1.0)
    else:                            # many distinct values: no dictionary, no image
        A = _banded(O, 30000, (1, 150), 5.0, -1.0, extra_vals=0.2)
    b = np.linspace(0.5, 1.5, A.nrows)
    xo, ro = O.cg(A, b, atol=0.0, rtol=1e-10, max_iter=20000)
    x, r = S.cg_solve(to_S(S, A), b, S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=20000))
    assert ro["converged"]
    rep_eq(r, ro)
    assert_bitwise(x, xo, case)


def test_config_D_c1_breakdown_matches_oracle(S, O, gpu):
    """SURVEY config D as defined (cell Peclet c = 1.0) is not solvable by plain right-Jacobi
    BiCGStab: from N = 128 the residual diverges and the SPEC rho-breakdown fires.  The GPU
    must break down exactly where the oracle does, with the same bits — which is why the
    bench measures D at c = 0.1 and says so (bench.py D_DEVIATION)."""
    A = O.generate_csr("convdiff3d", 128, 0, 1.0)
    b = np.ones(A.nrows)
    xo, ro = O.bicgstab(A, b, atol=0.0, rtol=1e-8, max_iter=3000)
    assert not ro["converged"] and ro["iterations"] < 3000  # breakdown, not max_iter
    x, r = S.bicgstab_solve(to_S(S, A), b, S.SolveOptions(atol=0.0, rtol=1e-8, max_iter=3000))
    rep_eq(r, ro)
    assert_bitwise(x, xo, "convdiff c=1 N=128")


def power_law_csr(O, n, seed, hubs, symmetric=True):
    """Irregular matrix: Pareto row degrees plus a few hub rows of `hubs` entries each;
    symmetric + diagonally dominant (SPD) unless symmetric=False."""
    rng = np.random.default_rng(seed)
    deg = np.minimum((rng.pareto(1.6, n) * 2).astype(np.int64) + 1, n // 4)
    deg[rng.choice(n, len(hubs), replace=False)] = hubs
    r = np.repeat(np.arange(n), deg)
    c = rng.integers(0, n, len(r))
    v = -rng.random(len(r))
    if symmetric:
        r, c, v = np.concatenate([r, c]), np.concatenate([c, r]), np.concatenate([v, v])
    off = np.zeros(n)
    np.add.at(off, r, np.abs(v))
    r = np.concatenate([r, np.arange(n)])
    c = np.concatenate([c, np.arange(n)])
    v = np.concatenate([v, off + 1.0])
    return O.csr_from_triplets(n, n, r, c, v)


@pytest.mark.parametrize("threshold", [None, "32", "0"])
def test_long_rows_warp_per_row_bitwise(S, O, gpu, monkeypatch, threshold):
    """Power-law hubs (2e4-6e4 entries) summed warp-per-row with the reference's left-to-right
    order: SpMV, CG (fused p.q over the short-row view) and set_values all bitwise."""
    if threshold is not None:
        monkeypatch.setenv("SPARSLA_LONG_ROW", threshold)
    A = power_law_csr(O, 120_000, 7, [60_000, 41_000, 20_000, 20_000, 3000])
    D = to_S(S, A).device(0)
    lr = D.long_rows()
    if threshold == "0":
        assert lr["rows"] == 0
    else:
        assert lr["rows"] >= 5 and lr["entries"] >= 140_000, lr
    x = np.random.default_rng(11).standard_normal(A.ncols)
    assert_bitwise(S.spmv(D, x), O.spmv(A, x), "spmv")
    b = np.ones(A.nrows)
    xo, ro = O.cg(A, b, atol=0.0, rtol=1e-10, max_iter=3000)
    xg, rg = S.cg_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=3000))
    rep_eq(rg, ro)
    assert_bitwise(xg, xo, "cg")
    v2 = A.vals * 1.5
    D.set_values(v2)
    A2 = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v2)
    assert_bitwise(S.spmv(D, x), O.spmv(A2, x), "spmv after set_values")


def test_long_rows_bicgstab_bitwise(S, O, gpu):
    A = power_law_csr(O, 60_000, 5, [30_000, 8000], symmetric=False)
    D = to_S(S, A).device(0)
    assert D.long_rows()["rows"] >= 2
    b = np.ones(A.nrows)
    xo, ro = O.bicgstab(A, b, atol=0.0, rtol=1e-10, max_iter=2000)
    xg, rg = S.bicgstab_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=2000))
    rep_eq(rg, ro)
    assert_bitwise(xg, xo, "bicgstab")
