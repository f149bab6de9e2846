// sparsla/eigen.hpp — eigen-solver contracts of SPEC.md:274-327 (the reference's eigen
// sources are missing from its tree) on the GPU LOBPCG of libsparsla_b200.
#pragma once

#include <cstring>
#include <string>
#include <vector>

#include "sparsla/sparse.hpp"

namespace sparsla {

struct EigenReport {  // iterations, residual norms per pair (+ per-pair flags)
    index_t iterations = 0;
    std::vector<double> residual_norms;
    std::vector<bool> pair_converged;
    bool converged = false;
    index_t spmm_count = 0;
    std::string diagnostic;
};

struct EigenResult {
    std::vector<double> lambdas;  // k, ascending
    std::vector<double> vectors;  // n x k row-major: v_m[i] = vectors[i * k + m]
    index_t k = 0;
    EigenReport report;
};

/// k smallest eigenpairs of a symmetric matrix: Jacobi-preconditioned
/// LOBPCG; UnsupportedInputError for nonsymmetric input; non-convergence -> partial result.
inline EigenResult eig_smallest(const SparseCoo& a, index_t k, double tol = 1e-8, index_t max_iter = 10000,
                                std::uint64_t seed = 2601) {
    const CsrMatrix csr = CsrMatrix::from_coo(a);
    const auto n = static_cast<std::size_t>(csr.nrows());
    if (k < 1 || k > csr.nrows()) throw InvalidArgumentError("eig_smallest: need 1 <= k <= n");
    EigenResult r;
    r.k = k;
    r.lambdas.resize(static_cast<std::size_t>(k));
    r.vectors.resize(n * static_cast<std::size_t>(k));
    r.report.residual_norms.resize(static_cast<std::size_t>(k));
    std::vector<int32_t> conv(static_cast<std::size_t>(k));
    sparsla_eig_options o{};
    o.tol = tol;
    o.max_iter = max_iter;
    o.seed = seed;
    o.preconditioner = SPARSLA_PRECOND_JACOBI;
    sparsla_eig_report rep{};
    detail::check(sparsla_eig_smallest(csr.device_handle(), k, &o, r.lambdas.data(), r.vectors.data(),
                                       r.report.residual_norms.data(), conv.data(), &rep, SPARSLA_MEM_HOST));
    r.report.iterations = rep.iterations;
    r.report.converged = rep.converged != 0;
    r.report.spmm_count = rep.spmm_count;
    r.report.pair_converged.assign(conv.begin(), conv.end());
    r.report.diagnostic = std::string(rep.diagnostic, strnlen(rep.diagnostic, sizeof(rep.diagnostic)));
    return r;
}

/// Eq. 4: grad_vals[e] = sum_m grad_lambdas[m] v_m[i_e] v_m[j_e] over the
/// stored entries of a_pattern; no linear solves.  Degenerate eigenvalues ->
/// UnsupportedInputError; unconverged pairs -> InvalidArgumentError.
inline std::vector<double> eig_backward(const EigenResult& result, const SparseCoo& a_pattern,
                                        std::span<const double> grad_lambdas) {
    if (static_cast<index_t>(grad_lambdas.size()) != result.k) throw DimensionError("eig_backward: grad_lambdas length");
    for (bool c : result.report.pair_converged)
        if (!c) throw InvalidArgumentError("eig_backward: not all eigenpairs converged");
    const CsrMatrix csr = CsrMatrix::from_coo(a_pattern);
    if (result.vectors.size() != static_cast<std::size_t>(csr.nrows() * result.k))
        throw DimensionError("eig_backward: vectors do not match the pattern");
    std::vector<double> gv(static_cast<std::size_t>(csr.nnz()));
    detail::check(sparsla_eig_backward(csr.device_handle(), result.k, result.lambdas.data(), result.vectors.data(),
                                       grad_lambdas.data(), gv.data(), SPARSLA_MEM_HOST));
    return gv;
}

}  // namespace sparsla
