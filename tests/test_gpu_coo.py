"""SparseCoo canonicalization on the GPU (sparse.cpp:9-53): bit-identical
to the reference's golden fixtures and to the host path — order, duplicate sums in input
order, explicit and signed zeros, empty input, bounds errors with the same message."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def same(a, b):
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.cols, b.cols)
    assert np.array_equal(bits(a.vals), bits(b.vals))


def test_golden_fixtures_on_device(S, gpu):
    G = np.load(os.path.join(ROOT, "tests", "golden", "sparse_core.npz"))
    for i in range(int(G["ncases"])):
        nr, nc = (int(t) for t in G[f"c{i}_shape"])
        rin = G[f"c{i}_in"]
        a = S.SparseCoo(rin[0].astype(np.int64), rin[1].astype(np.int64), G[f"c{i}_vin"], (nr, nc), device=0)
        assert np.array_equal(a.rows, G[f"c{i}_rows"]) and np.array_equal(a.cols, G[f"c{i}_cols"])
        assert np.array_equal(bits(a.vals), bits(G[f"c{i}_vals"])), i


@pytest.mark.parametrize("n,m,nnz,seed", [(1, 1, 5, 0), (40, 30, 2000, 1), (1000, 1000, 200000, 2),
                                          (300000, 300000, 3000000, 3)])
def test_random_duplicates_bitwise_vs_host(S, gpu, n, m, nnz, seed):
    rng = np.random.default_rng(seed)
    # heavy duplication: indices drawn from a small pool so segments have many entries
    pool = max(1, nnz // 7)
    pr, pc = rng.integers(0, n, pool), rng.integers(0, m, pool)
    pick = rng.integers(0, pool, nnz)
    rows, cols = pr[pick], pc[pick]
    vals = rng.standard_normal(nnz) * 10.0 ** rng.integers(-8, 8, nnz)
    vals[::11] = 0.0
    vals[::13] = -0.0
    same(S.SparseCoo(rows, cols, vals, (n, m), device=0), S.SparseCoo(rows, cols, vals, (n, m)))


def test_empty_and_bounds(S, gpu):
    e = S.SparseCoo([], [], [], (3, 4), device=0)
    assert e.nnz == 0 and e.nrows == 3
    with pytest.raises(S.BoundsError) as gpu_err:
        S.SparseCoo([0, 1, 2, 5, 9], [0, 1, 7, 0, 0], [1.0] * 5, (4, 4), device=0)
    with pytest.raises(S.BoundsError) as host_err:
        S.SparseCoo([0, 1, 2, 5, 9], [0, 1, 7, 0, 0], [1.0] * 5, (4, 4))
    assert str(gpu_err.value) == str(host_err.value)
    with pytest.raises(S.BoundsError):
        S.SparseCoo([-1], [0], [1.0], (2, 2), device=0)
    with pytest.raises(S.DimensionError):
        S.SparseCoo([0, 1], [0], [1.0], (2, 2), device=0)


def test_generator_triplets_at_scale(S, O, gpu):
    """The FEM generator's element-order triplets (duplicates summed in element order)
    canonicalized on the GPU equal the generator's canonical CSR."""
    n, r, c, v = O.gen_triplets("fem2d", 300, 2601)
    a = S.SparseCoo(r, c, v, (n, n), device=0)
    A = S.generate("fem2d", 300, 2601)
    assert np.array_equal(a.cols, A.col_idx) and np.array_equal(bits(a.vals), bits(A.vals))
    assert np.array_equal(np.repeat(np.arange(n), np.diff(A.row_ptr)), a.rows)


def test_sort_permutation_matches_host_order(S, gpu):
    """sparsla_coo_sort_device: the stable (row, col, input) order and the canonical entry of
    every sorted position, as numpy's lexsort gives them."""
    import ctypes as C
    rng = np.random.default_rng(11)
    n, nnz = 5000, 400000
    rows, cols = rng.integers(0, n, nnz), rng.integers(0, n // 50, nnz)
    order = np.empty(nnz, np.int64)
    group = np.empty(nnz, np.int64)
    m = C.c_int64()
    S._check(S.lib().sparsla_coo_sort_device(C.c_int(0), C.c_int64(n), C.c_int64(n), C.c_int64(nnz),
                                             S._p(rows, S._i64p), S._p(cols, S._i64p), C.c_int32(0), C.byref(m),
                                             S._p(order, S._i64p), S._p(group, S._i64p)))
    ref = np.lexsort((np.arange(nnz), cols, rows))
    assert np.array_equal(order, ref)
    r_s, c_s = rows[ref], cols[ref]
    new = np.ones(nnz, bool)
    new[1:] = (r_s[1:] != r_s[:-1]) | (c_s[1:] != c_s[:-1])
    assert np.array_equal(group, np.cumsum(new) - 1) and m.value == int(new.sum())


def test_torch_sparse_tensor_large_unsorted_input(S, O, gpu):
    """SparseTensor from 300K shuffled triplets with duplicates (GPU sort path): the solve
    and its gradients equal those of the canonical matrix."""
    import torch
    from paper_2601_13994_b200.torch_sla import SparseTensor
    A = O.generate("poisson2d", 120)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    # duplicates: every entry split into halves, then shuffled
    r = np.concatenate([rows, rows])
    c = np.concatenate([A.col_idx, A.col_idx])
    v = np.concatenate([A.vals * 0.5, A.vals * 0.5])
    perm = np.random.default_rng(5).permutation(len(r))
    vals = torch.tensor(v[perm], dtype=torch.float64, device="cuda:0", requires_grad=True)
    T = SparseTensor(vals, r[perm], c[perm], (A.nrows, A.ncols))
    assert len(r) >= (1 << 17) and T.nnz == A.nnz
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda:0")
    x = T.solve(b, atol=1e-12)
    xo, _ = O.cg(A, np.ones(A.nrows), atol=1e-12)
    assert np.max(np.abs(x.detach().cpu().numpy() - xo)) <= 1e-12 * np.max(np.abs(xo))
    x.sum().backward()
    g = vals.grad.cpu().numpy()
    # both halves of an entry get the gradient of their canonical entry
    inv = np.empty_like(perm); inv[perm] = np.arange(len(perm))
    assert np.array_equal(g[inv[:len(rows)]], g[inv[len(rows):]])
