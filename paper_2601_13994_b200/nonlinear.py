"""Newton-Raphson on the GPU Krylov loop + its adjoint.

Restates the nonlinear-solvers contract (Alg. 2, Eq. 5) over
this repo's solver: every Newton step solves J du = -F with the sm_100a CG (structurally
symmetric J) or BiCGStab (otherwise), Jacobi-preconditioned, to the inexact-Newton
tolerance min(0.1 ||F||, tol); the Jacobian's pattern is uploaded once and
only its values are refreshed per step (SparseCoo::with_values semantics).  Backtracking:
alpha = 1, halved until ||F(u + alpha du)|| <= (1 - 1e-4 alpha) ||F(u)||, alpha_min = 2^-20
(SPEC.md:402).  newton_backward performs exactly one transposed solve J^T lambda = grad_u
and returns -vjp_theta(u*, theta, lambda) (Eq. 5); the saved context is (u*, J, theta)
only (Theorem-1 style).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import sparsla as S


@dataclass
class ResidualSystem:
    F: Callable[[np.ndarray, np.ndarray], np.ndarray]            # F(u, theta) -> (n,)
    J: Callable[[np.ndarray, np.ndarray], S.SparseCoo]           # dF/du (fixed pattern)
    vjp_theta: Callable[[np.ndarray, np.ndarray, np.ndarray], np.ndarray] | None = None


@dataclass
class NonlinearReport:
    newton_iterations: int = 0
    linear_solves_forward: int = 0
    linear_solves_backward: int = 0
    final_residual_norm: float = 0.0
    line_search_steps_total: int = 0
    converged: bool = False


@dataclass
class NewtonContext:
    u: np.ndarray
    J: S.SparseCoo
    theta: np.ndarray
    _csr: S.CsrMatrix | None = field(default=None, repr=False)
    _backend: str = "cg"


class _Jacobian:
    """Device copy of J's fixed pattern; values refreshed in place each Newton step."""

    def __init__(self, J: S.SparseCoo):
        self.rows, self.cols = J.rows.copy(), J.cols.copy()
        self.csr = S.CsrMatrix.from_coo(J)
        self.D = self.csr.device(0)
        self.backend = "cg" if S.is_structurally_symmetric(J) else "bicgstab"

    def set(self, J: S.SparseCoo):
        if not (np.array_equal(J.rows, self.rows) and np.array_equal(J.cols, self.cols)):
            raise S.InvalidArgumentError("Jacobian pattern changed between Newton steps (SPEC.md:337)")
        v = np.ascontiguousarray(J.vals, np.float64)
        S._check(S.lib().sparsla_dcsr_set_values(self.D.h, S._p(v, S._f64p), C.c_int32(S.MEM_HOST)))
        self.csr._v = v

    def solve(self, rhs, atol, max_iter):
        opts = S.SolveOptions(atol=max(atol, 1e-300), rtol=0.0, max_iter=max_iter)
        fn = S.cg_solve if self.backend == "cg" else S.bicgstab_solve
        return fn(self.D, rhs, opts)


def newton_solve(sys: ResidualSystem, u0, theta, tol: float = 1e-10, max_iter: int = 50,
                 inner_max_iter: int = 20000):
    """-> (u*, NewtonContext, NonlinearReport); non-convergence is reported, line-search
    failure raises Error."""
    u = np.array(u0, dtype=np.float64, copy=True)
    theta = np.asarray(theta, dtype=np.float64)
    rep = NonlinearReport()
    Fu = np.asarray(sys.F(u, theta), dtype=np.float64)
    fn = float(np.linalg.norm(Fu))
    jac = None
    Jm = None
    while fn > tol and rep.newton_iterations < max_iter:
        Jm = sys.J(u, theta)
        if jac is None:
            jac = _Jacobian(Jm)
        jac.set(Jm)
        du, lrep = jac.solve(-Fu, min(0.1 * fn, tol), inner_max_iter)
        rep.linear_solves_forward += 1
        alpha = 1.0
        while True:
            un = u + alpha * du
            Fn = np.asarray(sys.F(un, theta), dtype=np.float64)
            fnn = float(np.linalg.norm(Fn))
            if fnn <= (1.0 - 1e-4 * alpha) * fn:
                break
            alpha *= 0.5
            rep.line_search_steps_total += 1
            if alpha < 2.0 ** -20:
                raise S.Error(f"line search failed at Newton iteration {rep.newton_iterations}")
        u, Fu, fn = un, Fn, fnn
        rep.newton_iterations += 1
    rep.final_residual_norm = fn
    rep.converged = fn <= tol
    if Jm is None:  # converged at u0: the context still needs J(u*)
        Jm = sys.J(u, theta)
    ctx = NewtonContext(u.copy(), Jm, theta.copy(), _csr=None,
                        _backend=jac.backend if jac else ("cg" if S.is_structurally_symmetric(Jm) else "bicgstab"))
    ctx._report = rep
    return u, ctx, rep


def newton_backward(ctx: NewtonContext, sys: ResidualSystem, grad_u, tol: float = 1e-12,
                    max_iter: int = 20000) -> np.ndarray:
    """Eq. 5: one solve J^T lambda = grad_u, grad_theta = -vjp_theta(u*, theta, lambda)."""
    if sys.vjp_theta is None:
        raise S.InvalidArgumentError("ResidualSystem.vjp_theta is required for the backward pass")
    g = np.ascontiguousarray(grad_u, np.float64)
    csr = S.CsrMatrix.from_coo(ctx.J)
    D = csr.device(0)
    lam = np.empty(csr.nrows)
    gv = np.empty(csr.nnz)
    zeros = np.zeros(csr.nrows)
    rep = S._Report()
    o = S.SolveOptions(atol=tol, rtol=0.0, max_iter=max_iter).c()
    be = S.BACKEND_CG if ctx._backend == "cg" else S.BACKEND_BICGSTAB
    # sparsla_adjoint_backward solves J^T lambda = g (exactly one Krylov solve); its
    # grad_vals output (x = 0 here) is not needed
    S._check(S.lib().sparsla_adjoint_backward(D.h, S._p(zeros, S._f64p), S._p(g, S._f64p), C.c_int32(be),
                                              C.byref(o), S._p(lam, S._f64p), S._p(gv, S._f64p), C.byref(rep),
                                              C.c_int32(S.MEM_HOST)))
    r = S.SolveReport._from(rep)
    if not r.converged:
        raise S.Error(f"newton_backward: adjoint solve did not converge: {r.diagnostic}")
    if hasattr(ctx, "_report"):
        ctx._report.linear_solves_backward += 1
    return -np.asarray(sys.vjp_theta(ctx.u, ctx.theta, lam), dtype=np.float64)
