// sparsla/solve.hpp — linear-solver contracts of SPEC.md:122-206 (the reference's
// src/solve.cpp is missing from its tree) on the GPU Krylov loop.
#pragma once

#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "sparsla/sparse.hpp"

namespace sparsla {

enum class Preconditioner { none, jacobi };
enum class Backend { cg, bicgstab, dense_lu };

struct SolveOptions {  // SPEC.md:127-130 (atol default 1e-10, Listing 2)
    double atol = 1e-10;
    double rtol = 0.0;
    index_t max_iter = 10000;
    Preconditioner preconditioner = Preconditioner::jacobi;
};

struct SolveReport {
    index_t iterations = 0;
    double residual_norm = 0.0;
    bool converged = false;
    index_t spmv_count = 0;
    Backend backend = Backend::cg;
    std::string diagnostic;
};

struct JacobiPreconditioner {
    std::vector<double> inverse_diagonal;
};

namespace detail {
inline sparsla_solve_options c_opts(const SolveOptions& o) {
    sparsla_solve_options c{};
    c.atol = o.atol;
    c.rtol = o.rtol;
    c.max_iter = o.max_iter;
    c.preconditioner = o.preconditioner == Preconditioner::jacobi ? SPARSLA_PRECOND_JACOBI : SPARSLA_PRECOND_NONE;
    return c;
}
inline SolveReport from_c(const sparsla_solve_report& r) {
    SolveReport s;
    s.iterations = r.iterations;
    s.residual_norm = r.residual_norm;
    s.converged = r.converged != 0;
    s.spmv_count = r.spmv_count;
    s.backend = r.backend == SPARSLA_BACKEND_BICGSTAB ? Backend::bicgstab : Backend::cg;
    s.diagnostic = std::string(r.diagnostic, strnlen(r.diagnostic, sizeof(r.diagnostic)));
    return s;
}
}  // namespace detail

inline JacobiPreconditioner jacobi_build(const CsrMatrix& a) {
    if (a.nrows() != a.ncols()) throw DimensionError("jacobi_build requires a square matrix");
    JacobiPreconditioner p;
    p.inverse_diagonal.resize(static_cast<std::size_t>(a.nrows()));
    detail::check(sparsla_jacobi(a.device_handle(), p.inverse_diagonal.data(), SPARSLA_MEM_HOST));
    return p;
}

/// Jacobi-PCG from x0 = 0; breakdown / non-convergence reported, not thrown.
inline std::pair<std::vector<double>, SolveReport> cg_solve(const CsrMatrix& a, std::span<const double> b,
                                                           const SolveOptions& opts = {}) {
    if (a.nrows() != a.ncols()) throw DimensionError("cg_solve requires a square matrix");
    if (static_cast<index_t>(b.size()) != a.nrows()) throw DimensionError("cg_solve: rhs length mismatch");
    std::vector<double> x(b.size());
    sparsla_solve_report r{};
    const auto o = detail::c_opts(opts);
    detail::check(sparsla_cg_solve(a.device_handle(), b.data(), x.data(), &o, &r, SPARSLA_MEM_HOST));
    return {std::move(x), detail::from_c(r)};
}

/// Right-Jacobi BiCGStab from x0 = 0.
inline std::pair<std::vector<double>, SolveReport> bicgstab_solve(const CsrMatrix& a, std::span<const double> b,
                                                                 const SolveOptions& opts = {}) {
    if (a.nrows() != a.ncols()) throw DimensionError("bicgstab_solve requires a square matrix");
    if (static_cast<index_t>(b.size()) != a.nrows()) throw DimensionError("bicgstab_solve: rhs length mismatch");
    std::vector<double> x(b.size());
    sparsla_solve_report r{};
    const auto o = detail::c_opts(opts);
    detail::check(sparsla_bicgstab_solve(a.device_handle(), b.data(), x.data(), &o, &r, SPARSLA_MEM_HOST));
    return {std::move(x), detail::from_c(r)};
}

}  // namespace sparsla
