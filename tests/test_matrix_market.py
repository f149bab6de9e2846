"""Matrix Market ingestion (matrix_market.hpp:10-20) and the GPU path
on irregular matrices read from .mtx files."""
import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def test_spec_examples(S):
    a = S.read_matrix_market("%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 2.5\n")
    assert a.shape == S.Shape(1, 1) and list(a.vals) == [2.5] and list(a.rows) == [0]
    s = S.read_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n% c\n2 2 1\n2 1 3.0\n")
    assert list(zip(s.rows, s.cols, s.vals)) == [(0, 1, 3.0), (1, 0, 3.0)]
    with pytest.raises(S.FormatError, match="non-coordinate"):
        S.read_matrix_market("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n")
    with pytest.raises(S.FormatError, match=r"line 3"):
        S.read_matrix_market("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 x 1.0\n2 2 1.0\n")
    with pytest.raises(S.FormatError, match=r"line 3"):
        S.read_matrix_market("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(S.FormatError, match="expected 2 entries"):
        S.read_matrix_market("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n")
    with pytest.raises(S.FormatError, match="complex"):
        S.read_matrix_market("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n")
    with pytest.raises(S.FormatError):
        S.read_matrix_market("/nonexistent/file.mtx")
    d = S.read_matrix_market("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 1 2.0\n2 1 5\n")
    assert list(d.vals) == [3.0, 5.0]  # duplicates summed (SparseCoo semantics)


def test_roundtrip_bit_exact(S, tmp_path):
    rng = np.random.default_rng(7)
    r, c = rng.integers(0, 300, 4000), rng.integers(0, 250, 4000)
    v = rng.standard_normal(4000) * 10.0 ** rng.integers(-300, 300, 4000).astype(float)
    a = S.SparseCoo(r, c, v, (300, 250))
    p = tmp_path / "a.mtx"
    S.write_matrix_market(a, p)
    b = S.read_matrix_market(str(p))
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.cols, b.cols)
    assert np.array_equal(bits(a.vals), bits(b.vals))


def _power_law_mtx(path, n, seed):
    """Irregular structurally symmetric SPD-ish matrix with a few very long rows."""
    rng = np.random.default_rng(seed)
    deg = np.minimum((rng.pareto(1.2, n) * 3).astype(int), n // 2)
    deg[rng.integers(0, n, 3)] = n // 3  # some hubs far above one stage's capacity
    lines = []
    for i in range(n):
        for j in rng.choice(n, size=deg[i], replace=False):
            if j < i:
                lines.append((i + 1, j + 1, -rng.random()))
    diag = np.zeros(n)
    for i, j, x in lines:
        diag[i - 1] += -x
        diag[j - 1] += -x
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        f.write(f"{n} {n} {len(lines) + n}\n")
        for i in range(n):
            f.write(f"{i + 1} {i + 1} {diag[i] + 1.0:.17g}\n")
        for i, j, x in lines:
            f.write(f"{i} {j} {x:.17g}\n")


@pytest.mark.gpu
def test_irregular_mtx_on_gpu_bitwise(S, O, gpu, tmp_path):
    p = tmp_path / "pl.mtx"
    _power_law_mtx(p, 6000, 3)
    a = S.read_matrix_market(str(p))
    A = S.CsrMatrix.from_coo(a)
    lens = np.diff(A.row_ptr)
    assert lens.max() > 1500 and np.median(lens) < 20
    Ao = O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, A.vals)
    x = np.random.default_rng(1).standard_normal(A.ncols)
    assert np.array_equal(bits(S.spmv(A, x)), bits(O.spmv(Ao, x)))
    b = np.ones(A.nrows)
    xs, rs = S.cg_solve(A, b, S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=5000))
    xo, ro = O.cg(Ao, b, atol=0.0, rtol=1e-10, max_iter=5000)
    assert rs.iterations == ro["iterations"] and rs.converged
    assert np.array_equal(bits(xs), bits(xo))
