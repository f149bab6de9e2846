// sparsla/adjoint.hpp — adjoint engine contracts of SPEC.md:208-272 (Eq. 3, Alg. 1).
#pragma once

#include "sparsla/solve.hpp"

namespace sparsla {

struct AdjointContext {  // exactly (A, x): no per-iteration state (Theorem 1)
    SparseCoo matrix;
    std::vector<double> x;
    Backend backend = Backend::cg;
    CsrMatrix csr;
};

struct GradientBundle {
    std::vector<double> grad_b;
    std::vector<double> grad_vals;  // aligned with matrix's stored entries
};

/// Forward solve; CG on a structurally symmetric pattern, else BiCGStab.
inline std::pair<std::vector<double>, AdjointContext> solve_forward(const SparseCoo& a, std::span<const double> b,
                                                                   const SolveOptions& opts = {}) {
    AdjointContext ctx;
    ctx.matrix = a;
    ctx.csr = CsrMatrix::from_coo(a);
    ctx.backend = is_structurally_symmetric(a) ? Backend::cg : Backend::bicgstab;
    auto [x, rep] = ctx.backend == Backend::cg ? cg_solve(ctx.csr, b, opts) : bicgstab_solve(ctx.csr, b, opts);
    if (!rep.converged) throw Error("solve_forward: solver did not converge: " + rep.diagnostic);
    ctx.x = x;
    return {std::move(x), std::move(ctx)};
}

/// One solve A^T lambda = grad_x; grad_b = lambda; grad_vals[k] = -lambda[i_k] x[j_k].
inline GradientBundle solve_backward(const AdjointContext& ctx, std::span<const double> grad_x,
                                     const SolveOptions& opts = {}) {
    if (static_cast<index_t>(grad_x.size()) != ctx.csr.nrows()) throw DimensionError("solve_backward: grad_x length");
    GradientBundle g;
    g.grad_b.resize(grad_x.size());
    g.grad_vals.resize(static_cast<std::size_t>(ctx.csr.nnz()));
    sparsla_solve_report r{};
    const auto o = detail::c_opts(opts);
    detail::check(sparsla_adjoint_backward(ctx.csr.device_handle(), ctx.x.data(), grad_x.data(),
                                           ctx.backend == Backend::cg ? SPARSLA_BACKEND_CG : SPARSLA_BACKEND_BICGSTAB,
                                           &o, g.grad_b.data(), g.grad_vals.data(), &r, SPARSLA_MEM_HOST));
    if (!r.converged) throw Error("solve_backward: adjoint solve did not converge");
    return g;
}

}  // namespace sparsla
