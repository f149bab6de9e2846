"""Newton on the GPU Krylov loop + newton_backward (examples)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def poisson_coo(S, N):
    A = S.generate("poisson2d", N)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    return A, rows


def test_linear_residual_one_newton_step(S, gpu):
    from paper_2601_13994_b200.nonlinear import ResidualSystem, newton_solve
    A, rows = poisson_coo(S, 16)
    coo = S.SparseCoo(rows, A.col_idx, A.vals, A.shape, _canonical=True)
    b = np.ones(A.nrows)
    sys_ = ResidualSystem(F=lambda u, th: S.spmv(A, u) - th, J=lambda u, th: coo)
    u, ctx, rep = newton_solve(sys_, np.zeros(A.nrows), b, tol=1e-10)
    assert rep.converged and rep.newton_iterations == 1 and rep.line_search_steps_total == 0


def test_scalar_cube_root_and_backward(S, gpu):
    from paper_2601_13994_b200.nonlinear import ResidualSystem, newton_backward, newton_solve
    sys_ = ResidualSystem(
        F=lambda u, th: u ** 3 - th,
        J=lambda u, th: S.SparseCoo([0], [0], [3.0 * u[0] ** 2], (1, 1)),
        vjp_theta=lambda u, th, lam: -lam)  # dF/dtheta = -1
    u, ctx, rep = newton_solve(sys_, np.array([3.0]), np.array([8.0]), tol=1e-12)
    assert rep.converged and abs(u[0] - 2.0) <= 1e-12
    g = newton_backward(ctx, sys_, np.array([1.0]))
    # Alg. 2 stores the LAST iteration's J (evaluated at u_{k-1}), so the
    # gradient is 1/(3 u_{k-1}^2) = 1/12 up to the last Newton step (~1e-6 here)
    assert abs(g[0] - 1.0 / 12.0) <= 1e-6 and rep.linear_solves_backward == 1


def test_diffusion_newton_vs_dense_and_fd(S, gpu):
    """F(u, theta) = A u + u^3 - theta on Poisson 16x16; grad of L = sum(u) w.r.t. theta."""
    from paper_2601_13994_b200.nonlinear import ResidualSystem, newton_backward, newton_solve
    A, rows = poisson_coo(S, 16)
    n = A.nrows
    Ad = np.zeros((n, n))
    Ad[rows, A.col_idx] = A.vals
    diag_pos = np.nonzero(rows == A.col_idx)[0]

    def J(u, th):
        v = A.vals.copy()
        v[diag_pos] += 3.0 * u ** 2
        return S.SparseCoo(rows, A.col_idx, v, A.shape, _canonical=True)

    sys_ = ResidualSystem(F=lambda u, th: S.spmv(A, u) + u ** 3 - th, J=J,
                          vjp_theta=lambda u, th, lam: -lam)
    theta = np.ones(n)
    u, ctx, rep = newton_solve(sys_, np.zeros(n), theta, tol=1e-10)
    assert rep.converged and rep.final_residual_norm <= 1e-10 and 2 <= rep.newton_iterations <= 10
    # dense reference solution (numpy Newton with exact linear solves)
    ud = np.zeros(n)
    for _ in range(50):
        Fd = Ad @ ud + ud ** 3 - theta
        ud -= np.linalg.solve(Ad + np.diag(3 * ud ** 2), Fd)
    assert np.max(np.abs(u - ud)) <= 1e-8
    g = newton_backward(ctx, sys_, np.ones(n))
    assert rep.linear_solves_backward == 1
    eps = 1e-5
    for i in (0, 37, 255):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += eps
        tm[i] -= eps
        up, _, _ = newton_solve(sys_, u, tp, tol=1e-12)
        um, _, _ = newton_solve(sys_, u, tm, tol=1e-12)
        fd = (up.sum() - um.sum()) / (2 * eps)
        assert abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1e-12) < 1e-5
