// sparsla/distributed.hpp — domain-decomposition contracts of SPEC.md:417-544 on 1..8 GPUs.
#pragma once

#include <memory>

#include "sparsla/solve.hpp"

namespace sparsla {

inline std::vector<int> partition_contiguous(index_t n, int nparts) {
    std::vector<int> part(static_cast<std::size_t>(n));
    detail::check(sparsla_partition_contiguous(n, nparts, part.data()));
    return part;
}

inline std::vector<int> partition_rcb(std::span<const double> xs, std::span<const double> ys, int nparts) {
    if (xs.size() != ys.size()) throw DimensionError("partition_rcb: coordinate arrays differ in length");
    std::vector<int> part(xs.size());
    detail::check(sparsla_partition_rcb(static_cast<index_t>(xs.size()), xs.data(), ys.data(), nparts, part.data()));
    return part;
}

/// LocalPartition built from this rank's owned rows (global columns).
class LocalPartition {
public:
    LocalPartition(index_t n_global, const std::vector<int>* part_of, int nparts, int rank,
                   std::span<const index_t> owned, const CsrMatrix& owned_rows) {
        sparsla_local* h = nullptr;
        detail::check(sparsla_local_build(n_global, part_of ? part_of->data() : nullptr, nparts, rank,
                                          static_cast<index_t>(owned.size()), owned.data(), owned_rows.row_ptr().data(),
                                          owned_rows.col_idx().data(), owned_rows.vals().data(), &h));
        h_.reset(h, [](sparsla_local* p) { sparsla_local_destroy(p); });
        std::int64_t s[6];
        detail::check(sparsla_local_sizes(h, s));
        owned_.resize(s[0]); halo_.resize(s[1]); neighbors_.resize(s[2]);
        send_ptr_.resize(s[2] + 1); recv_ptr_.resize(s[2] + 1); send_idx_.resize(s[4]); recv_idx_.resize(s[5]);
        detail::check(sparsla_local_get(h, owned_.data(), halo_.data(), neighbors_.data(), send_ptr_.data(),
                                        send_idx_.data(), recv_ptr_.data(), recv_idx_.data(), nullptr, nullptr, nullptr));
        rank_ = rank;
    }
    int rank() const { return rank_; }
    std::span<const index_t> owned() const { return owned_; }
    std::span<const index_t> halo() const { return halo_; }
    std::span<const int> neighbors() const { return neighbors_; }
    std::span<const index_t> send_ptr() const { return send_ptr_; }
    std::span<const index_t> send_idx() const { return send_idx_; }
    std::span<const index_t> recv_ptr() const { return recv_ptr_; }
    std::span<const index_t> recv_idx() const { return recv_idx_; }
    const sparsla_local* handle() const { return h_.get(); }
private:
    std::shared_ptr<sparsla_local> h_;
    int rank_ = 0;
    std::vector<index_t> owned_, halo_, send_ptr_, send_idx_, recv_ptr_, recv_idx_;
    std::vector<int> neighbors_;
};

/// One rank of the distributed solver; every member call is collective.
class DistSolver {
public:
    /// NCCL-backed (one rank per GPU); id from sparsla_nccl_unique_id on rank 0.
    DistSolver(int device, int nranks, int rank, const unsigned char* nccl_id, const LocalPartition& L) {
        sparsla_dist* d = nullptr;
        detail::check(sparsla_dist_create_nccl(device, nranks, rank, nccl_id, L.handle(), &d));
        d_.reset(d, [](sparsla_dist* p) { sparsla_dist_destroy(p); });
        n_owned_ = static_cast<index_t>(L.owned().size());
    }
    std::vector<double> spmv(std::span<const double> x_owned) {
        std::vector<double> y(static_cast<std::size_t>(n_owned_));
        detail::check(sparsla_dist_spmv(d_.get(), x_owned.data(), y.data(), SPARSLA_MEM_HOST));
        return y;
    }
    std::pair<std::vector<double>, SolveReport> cg(std::span<const double> b_owned, const SolveOptions& opts = {}) {
        std::vector<double> x(static_cast<std::size_t>(n_owned_));
        sparsla_solve_report r{};
        const auto o = detail::c_opts(opts);
        detail::check(sparsla_dist_cg_solve(d_.get(), b_owned.data(), x.data(), &o, &r, SPARSLA_MEM_HOST));
        return {std::move(x), detail::from_c(r)};
    }
    std::pair<std::vector<double>, SolveReport> bicgstab(std::span<const double> b_owned, const SolveOptions& opts = {}) {
        std::vector<double> x(static_cast<std::size_t>(n_owned_));
        sparsla_solve_report r{};
        const auto o = detail::c_opts(opts);
        detail::check(sparsla_dist_bicgstab_solve(d_.get(), b_owned.data(), x.data(), &o, &r, SPARSLA_MEM_HOST));
        return {std::move(x), detail::from_c(r)};
    }
    sparsla_dist* handle() const { return d_.get(); }
private:
    std::shared_ptr<sparsla_dist> d_;
    index_t n_owned_ = 0;
};

}  // namespace sparsla
