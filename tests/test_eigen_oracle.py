"""CPU tests of the eigen-solver ORACLE (dense eigensolver + Eq. 4 + finite differences),
pinned on the SPEC's own examples before it is used to check
the GPU LOBPCG (tests/test_gpu_eigen.py)."""
import numpy as np
import pytest


def csr(O, D):
    D = np.asarray(D, dtype=np.float64)
    n = D.shape[0]
    rows, cols = np.nonzero(D)
    return O.csr_from_triplets(n, n, rows.astype(np.int64), cols.astype(np.int64), D[rows, cols])


def test_spec_eig_examples(O):
    A = csr(O, np.diag([1.0, 2.0, 3.0, 4.0]))
    w, V = O.eig_dense(A, 2)
    assert np.allclose(w, [1, 2], atol=1e-14)
    assert np.allclose(V, np.eye(4)[:, :2], atol=1e-14)
    B = csr(O, [[2.0, 1.0], [1.0, 2.0]])
    w, V = O.eig_dense(B, 1)
    assert abs(w[0] - 1.0) < 1e-14
    # |v0| == |v1|: the first index carries the sign convention
    assert np.allclose(V[:, 0], np.array([1.0, -1.0]) / np.sqrt(2), atol=1e-14)


def test_spec_eig_backward_example(O):
    B = csr(O, [[2.0, 1.0], [1.0, 2.0]])
    w, V = O.eig_dense(B, 1)
    g = O.eig_backward(B, V, [1.0])
    assert np.allclose(g, [0.5, -0.5, -0.5, 0.5], atol=1e-14)
    fd = O.eig_fd(B, 1, [1.0])
    assert np.allclose(fd, g, rtol=1e-5, atol=1e-9)
    assert np.all(O.eig_backward(B, V, [0.0]) == 0.0)


def test_eig_backward_fd_random_symmetric(O):
    rng = np.random.default_rng(2601)
    n, k = 40, 4
    M = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.15)
    M = M + M.T + np.diag(np.arange(n, dtype=np.float64))
    A = csr(O, M)
    w, V = O.eig_dense(A, k)
    assert np.all(np.diff(w) > 1e-8)
    g = rng.standard_normal(k)
    an = O.eig_backward(A, V, g)
    ent = list(range(0, A.nnz, max(1, A.nnz // 25)))
    fd = O.eig_fd(A, k, g, entries=ent)
    assert np.max(np.abs(fd - an[ent])) / np.max(np.abs(an[ent])) < 1e-5


def test_trace_consistency(O):
    A = O.generate("poisson2d", 5)
    w, _ = O.eig_dense(A, A.nrows)
    assert abs(w.sum() - np.trace(A.dense())) < 1e-9
