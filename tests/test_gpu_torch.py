"""torch-sla autograd binding on the GPU path: forward = the sm_100a solve, backward = one
adjoint solve; gradients equal the oracle's adjoint bit for bit and agree with central
finite differences (Table 4 / SPEC.md:242)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def test_autograd_matches_oracle_adjoint(S, O, gpu):
    import torch
    from paper_2601_13994_b200.torch_sla import SparseTensor
    A = O.generate("poisson2d", 24)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    vals = torch.tensor(A.vals, dtype=torch.float64, device="cuda:0", requires_grad=True)
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda:0", requires_grad=True)
    T = SparseTensor(vals, rows, A.col_idx, (A.nrows, A.ncols))
    x = T.solve(b, atol=1e-12)
    loss = (x * x).sum()
    loss.backward()
    xo, _ = O.cg(A, np.ones(A.nrows), atol=1e-12)
    assert np.array_equal(bits(x.detach().cpu().numpy()), bits(xo))
    gbo, gvo, _ = O.adjoint_backward(A, xo, 2.0 * xo, atol=1e-12)
    assert np.array_equal(bits(b.grad.cpu().numpy()), bits(gbo))
    assert np.array_equal(bits(vals.grad.cpu().numpy()), bits(gvo))


def test_autograd_finite_differences_and_duplicates(S, gpu):
    import torch
    from paper_2601_13994_b200.torch_sla import SparseTensor
    P = S.generate("poisson2d", 10)
    rows = np.repeat(np.arange(P.nrows), np.diff(P.row_ptr))
    # split every diagonal entry into two duplicates (summed like SparseCoo) and shuffle
    diag = rows == P.col_idx
    r = np.concatenate([rows, rows[diag]])
    c = np.concatenate([P.col_idx, P.col_idx[diag]])
    v = np.concatenate([np.where(diag, 3.0, P.vals), np.full(diag.sum(), 1.0)])
    perm = np.random.default_rng(0).permutation(len(r))
    r, c, v = r[perm], c[perm], v[perm]
    vals = torch.tensor(v, dtype=torch.float64, device="cuda:0", requires_grad=True)
    b = torch.linspace(0.5, 1.5, P.nrows, dtype=torch.float64, device="cuda:0")
    T = SparseTensor(vals, r, c, (P.nrows, P.nrows))
    x = T.solve(b, atol=1e-13)
    x.sum().backward()
    g = vals.grad.cpu().numpy()
    eps = 1e-5
    for k in [0, 7, len(v) - 1, int(np.nonzero(r == c)[0][0])]:
        vp, vm = v.copy(), v.copy()
        vp[k] += eps
        vm[k] -= eps
        Lp = SparseTensor(torch.tensor(vp, device="cuda:0"), r, c, T.shape).solve(b, atol=1e-13).sum().item()
        Lm = SparseTensor(torch.tensor(vm, device="cuda:0"), r, c, T.shape).solve(b, atol=1e-13).sum().item()
        fd = (Lp - Lm) / (2 * eps)
        assert abs(fd - g[k]) / max(abs(fd), abs(g[k]), 1e-12) < 1e-5, (k, fd, g[k])


def test_autograd_nonsymmetric_bicgstab(S, O, gpu):
    import torch
    from paper_2601_13994_b200.torch_sla import SparseTensor
    A = O.generate("convdiff3d", 8, 0, 0.5)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    vals = torch.tensor(A.vals, dtype=torch.float64, device="cuda:0", requires_grad=True)
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda:0", requires_grad=True)
    x = SparseTensor(vals, rows, A.col_idx, (A.nrows, A.nrows)).solve(b, atol=1e-12, backend="bicgstab")
    x.sum().backward()
    xo, _ = O.bicgstab(A, np.ones(A.nrows), atol=1e-12)
    gbo, gvo, _ = O.adjoint_backward(A, xo, np.ones(A.nrows), backend=1, atol=1e-12)
    assert np.array_equal(bits(b.grad.cpu().numpy()), bits(gbo))
    assert np.array_equal(bits(vals.grad.cpu().numpy()), bits(gvo))


def test_eigsh_autograd_eq4(S, O, gpu):
    """SparseTensor.eigsh: LOBPCG forward, Eq. 4 backward (no solves) equals the oracle's
    gather sum_m g_m v_m[i] v_m[j] on the returned vectors; FD on a few stored entries."""
    import torch
    from paper_2601_13994_b200.torch_sla import SparseTensor
    P = O.generate("poisson2d", 20)
    rows = np.repeat(np.arange(P.nrows), np.diff(P.row_ptr))
    v0 = P.vals.copy()
    v0[rows == P.col_idx] += 0.3 * np.arange(P.nrows) / P.nrows  # simple spectrum
    vals = torch.tensor(v0, dtype=torch.float64, device="cuda:0", requires_grad=True)
    T = SparseTensor(vals, rows, P.col_idx, (P.nrows, P.ncols))
    lam, V = T.eigsh(k=4, tol=1e-11)
    g = torch.tensor([1.0, -0.5, 0.25, 2.0], dtype=torch.float64, device="cuda:0")
    (lam * g).sum().backward()
    A = O.Csr(P.nrows, P.ncols, P.row_ptr, P.col_idx, v0)
    w, _ = O.eig_dense(A, 4)
    assert np.max(np.abs(lam.detach().cpu().numpy() - w)) <= 1e-8
    ref = O.eig_backward(A, V.cpu().numpy(), g.cpu().numpy())
    assert np.max(np.abs(vals.grad.cpu().numpy() - ref)) <= 1e-14
    ent = [0, 7, 100, len(v0) - 1]
    fd = O.eig_fd(A, 4, g.cpu().numpy(), entries=ent)
    assert np.max(np.abs(fd - ref[ent])) / np.max(np.abs(ref[ent])) < 1e-5


@pytest.mark.parametrize("nnz", [5000, 300_000])  # host lexsort / GPU radix-sort patterns
def test_duplicate_values_sum_in_input_order(S, gpu, nnz):
    """Canonical values of triplets with duplicates come from the GPU group sum and equal the
    host SparseCoo canonicalization (sparse.cpp:45-47 order) bit for bit; the gradient of
    every duplicate is its canonical entry's gradient."""
    import torch
    from paper_2601_13994_b200.torch_sla import SparseTensor
    rng = np.random.default_rng(7)
    n = 64 if nnz < 10_000 else 400
    r = rng.integers(0, n, nnz)
    c = rng.integers(0, n, nnz)
    v = rng.standard_normal(nnz) * 10.0 ** rng.integers(-8, 8, nnz)
    ref = S.SparseCoo(r, c, v, (n, n))
    vals = torch.tensor(v, device="cuda:0", requires_grad=True)
    T = SparseTensor(vals, r, c, (n, n))
    cv = T.canonical_values()
    assert np.array_equal(bits(cv.detach().cpu().numpy()), bits(ref.vals))
    w = torch.linspace(-1.0, 1.0, T.nnz, dtype=torch.float64, device="cuda:0")
    (cv * w).sum().backward()
    assert np.array_equal(vals.grad.cpu().numpy(), w.cpu().numpy()[T._group_of_input])
