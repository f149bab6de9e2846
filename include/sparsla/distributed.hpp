// sparsla/distributed.hpp — domain-decomposition contracts of SPEC.md:417-544 on 1..8 GPUs.
#pragma once

#include <map>
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

class Transport;

/// LocalPartition built from this rank's owned rows (global columns).
class LocalPartition {
public:
    LocalPartition(index_t n_global, const std::vector<int>* part_of, int nparts, int rank,
                   std::span<const index_t> owned, const CsrMatrix& owned_rows)
        : LocalPartition(n_global, part_of, nparts, rank, owned, owned_rows.row_ptr(), owned_rows.col_idx(),
                         owned_rows.vals()) {}
    /// owned rows as raw CSR arrays (row_ptr over the owned rows, global column ids)
    LocalPartition(index_t n_global, const std::vector<int>* part_of, int nparts, int rank,
                   std::span<const index_t> owned, std::span<const index_t> row_ptr, std::span<const index_t> col_idx,
                   std::span<const double> vals) {
        if (row_ptr.size() != owned.size() + 1) throw DimensionError("build_local: row_ptr length != owned + 1");
        sparsla_local* h = nullptr;
        detail::check(sparsla_local_build(n_global, part_of ? part_of->data() : nullptr, nparts, rank,
                                          static_cast<index_t>(owned.size()), owned.data(), row_ptr.data(),
                                          col_idx.data(), vals.data(), &h));
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
    /// this partition's device plan on transport T (built on first use; collective)
    sparsla_dist* plan(Transport& T) const;
private:
    std::shared_ptr<sparsla_local> h_;
    std::shared_ptr<std::map<const void*, std::shared_ptr<sparsla_dist>>> plans_ =
        std::make_shared<std::map<const void*, std::shared_ptr<sparsla_dist>>>();
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


/// In-process rank group (threads, possibly sharing one GPU) for Transport::in_process.
class LocalHub {
public:
    explicit LocalHub(int nranks) {
        sparsla_local_hub* h = nullptr;
        detail::check(sparsla_local_hub_create(nranks, &h));
        h_.reset(h, [](sparsla_local_hub* p) { sparsla_local_hub_destroy(p); });
    }
    sparsla_local_hub* handle() const { return h_.get(); }
private:
    std::shared_ptr<sparsla_local_hub> h_;
};

/// Transport: point-to-point halo traffic and rank-ordered reductions.
/// One object per rank; every operation is collective over the ranks.
class Transport {
public:
    /// one rank per GPU over NCCL (id from nccl_unique_id() on rank 0, shared out of band)
    static Transport nccl(int device, int nranks, int rank, const unsigned char* id) {
        sparsla_transport* t = nullptr;
        detail::check(sparsla_transport_create_nccl(device, nranks, rank, id, &t));
        return Transport(t);
    }
    /// in-process workers (desk-scale backing); each rank's thread calls this
    static Transport in_process(const LocalHub& hub, int rank, int device = 0) {
        sparsla_transport* t = nullptr;
        detail::check(sparsla_transport_create_local(device, hub.handle(), rank, &t));
        return Transport(t);
    }
    /// caller-provided collectives (e.g. an MPI or torch.distributed backing)
    static Transport host(int device, int nranks, int rank, const sparsla_host_transport& cb) {
        sparsla_transport* t = nullptr;
        detail::check(sparsla_transport_create_host(device, nranks, rank, &cb, &t));
        return Transport(t);
    }
    static std::vector<unsigned char> nccl_unique_id() {
        std::vector<unsigned char> id(128);
        detail::check(sparsla_nccl_unique_id(id.data()));
        return id;
    }
    int nranks() const { return static_cast<int>(info(0)); }
    int rank() const { return static_cast<int>(info(1)); }
    std::int64_t exchanges() const { return info(2); }
    std::int64_t all_reduces() const { return info(3); }
    std::int64_t messages() const { return info(4); }
    sparsla_transport* handle() const { return h_.get(); }
private:
    explicit Transport(sparsla_transport* t) : h_(t, [](sparsla_transport* p) { sparsla_transport_destroy(p); }) {}
    std::int64_t info(int k) const {
        std::int64_t o[5];
        detail::check(sparsla_transport_info(h_.get(), o));
        return o[k];
    }
    std::shared_ptr<sparsla_transport> h_;
};

inline sparsla_dist* LocalPartition::plan(Transport& T) const {
    auto& p = (*plans_)[T.handle()];
    if (!p) {
        sparsla_dist* d = nullptr;
        detail::check(sparsla_dist_create(T.handle(), h_.get(), &d));
        p.reset(d, [](sparsla_dist* q) { sparsla_dist_destroy(q); });
    }
    return p.get();
}

/// build_local(A, part_of, rank): this rank's owned rows of the global
/// matrix, halo = referenced non-owned columns, HaloMap in canonical global order.
inline LocalPartition build_local(const SparseCoo& a, const std::vector<int>& part_of, int rank) {
    if (static_cast<index_t>(part_of.size()) != a.nrows()) throw DimensionError("build_local: part_of length != n");
    const CsrMatrix g = CsrMatrix::from_coo(a);
    int nparts = 0;
    for (int p : part_of) nparts = std::max(nparts, p + 1);
    std::vector<index_t> owned, rp{0}, ci;
    std::vector<double> v;
    const auto grp = g.row_ptr();
    for (index_t i = 0; i < a.nrows(); ++i) {
        if (part_of[static_cast<std::size_t>(i)] != rank) continue;
        owned.push_back(i);
        for (index_t k = grp[i]; k < grp[i + 1]; ++k) {
            ci.push_back(g.col_idx()[k]);
            v.push_back(g.vals()[k]);
        }
        rp.push_back(static_cast<index_t>(ci.size()));
    }
    return LocalPartition(a.nrows(), &part_of, std::max(nparts, rank + 1), rank, owned, rp, ci, v);
}

/// halo_exchange: the halo slice (neighbours' owned values, ascending
/// global index) for the owned slice x_owned.
inline std::vector<double> halo_exchange(const LocalPartition& local, Transport& t, std::span<const double> x_owned) {
    if (x_owned.size() != local.owned().size()) throw DimensionError("halo_exchange: x_owned length != owned count");
    std::vector<double> halo(local.halo().size());
    detail::check(sparsla_dist_halo_exchange(local.plan(t), x_owned.data(), halo.data(), SPARSLA_MEM_HOST));
    return halo;
}

/// dist_spmv: owned rows of A x, bit-identical to the serial rows.
inline std::vector<double> dist_spmv(const LocalPartition& local, Transport& t, std::span<const double> x_owned) {
    if (x_owned.size() != local.owned().size()) throw DimensionError("dist_spmv: x_owned length != owned count");
    std::vector<double> y(x_owned.size());
    detail::check(sparsla_dist_spmv(local.plan(t), x_owned.data(), y.data(), SPARSLA_MEM_HOST));
    return y;
}

/// all_reduce_sum: Σ_p local_p in ascending rank order, on every rank.
inline double all_reduce_sum(Transport& t, double local) {
    double g = 0.0;
    detail::check(sparsla_transport_all_reduce_sum(t.handle(), local, &g));
    return g;
}

/// dist_cg (Algorithm 4) with SolveOptions as cg_solve (Jacobi default).
inline std::pair<std::vector<double>, SolveReport> dist_cg(const LocalPartition& local, Transport& t,
                                                          std::span<const double> b_owned, const SolveOptions& opts) {
    if (b_owned.size() != local.owned().size()) throw DimensionError("dist_cg: b_owned length != owned count");
    std::vector<double> x(b_owned.size());
    sparsla_solve_report r{};
    const auto o = detail::c_opts(opts);
    detail::check(sparsla_dist_cg_solve(local.plan(t), b_owned.data(), x.data(), &o, &r, SPARSLA_MEM_HOST));
    return {std::move(x), detail::from_c(r)};
}
/// the SPEC signature: dist_cg(local, transport, b_owned, atol, max_iter)
inline std::pair<std::vector<double>, SolveReport> dist_cg(const LocalPartition& local, Transport& t,
                                                          std::span<const double> b_owned, double atol,
                                                          index_t max_iter) {
    SolveOptions o;
    o.atol = atol;
    o.max_iter = max_iter;
    return dist_cg(local, t, b_owned, o);
}
/// distributed right-Jacobi BiCGStab (config D's nonsymmetric systems)
inline std::pair<std::vector<double>, SolveReport> dist_bicgstab(const LocalPartition& local, Transport& t,
                                                                std::span<const double> b_owned,
                                                                const SolveOptions& opts = {}) {
    if (b_owned.size() != local.owned().size()) throw DimensionError("dist_bicgstab: b_owned length != owned count");
    std::vector<double> x(b_owned.size());
    sparsla_solve_report r{};
    const auto o = detail::c_opts(opts);
    detail::check(sparsla_dist_bicgstab_solve(local.plan(t), b_owned.data(), x.data(), &o, &r, SPARSLA_MEM_HOST));
    return {std::move(x), detail::from_c(r)};
}

struct DistGradient {  // dist_adjoint_solve result
    std::vector<double> grad_b_owned;     // λ over the owned rows
    std::vector<double> grad_vals_local;  // per local entry (owned rows, global column order)
    SolveReport report;
};

/// dist_adjoint_solve: one distributed solve of Aᵀλ = grad_x on the forward
/// halo maps (structural symmetry required) + the local gather grad_vals = −λ_i x_j.  The
/// forward solution x_owned is passed explicitly (the reference keeps it in its context);
/// vals_t = Aᵀ's values in the local entry order, empty when A is symmetric.
inline DistGradient dist_adjoint_solve(const LocalPartition& local, Transport& t, std::span<const double> x_owned,
                                       std::span<const double> grad_x_owned, const SolveOptions& opts = {},
                                       std::span<const double> vals_t = {}, Backend backend = Backend::cg) {
    if (x_owned.size() != local.owned().size() || grad_x_owned.size() != local.owned().size())
        throw DimensionError("dist_adjoint_solve: owned-slice length mismatch");
    sparsla_dist* d = local.plan(t);
    std::int64_t info[9];
    detail::check(sparsla_dist_info(d, info));
    DistGradient g;
    g.grad_b_owned.resize(x_owned.size());
    std::int64_t nnz_local = 0;
    {
        std::int64_t s[6];
        detail::check(sparsla_local_sizes(local.handle(), s));
        nnz_local = s[3];
    }
    g.grad_vals_local.resize(static_cast<std::size_t>(nnz_local));
    sparsla_solve_report r{};
    const auto o = detail::c_opts(opts);
    detail::check(sparsla_dist_adjoint_backward(d, x_owned.data(), grad_x_owned.data(),
                                                vals_t.empty() ? nullptr : vals_t.data(),
                                                backend == Backend::bicgstab ? SPARSLA_BACKEND_BICGSTAB : SPARSLA_BACKEND_CG,
                                                &o, g.grad_b_owned.data(), g.grad_vals_local.data(), &r,
                                                SPARSLA_MEM_HOST));
    g.report = detail::from_c(r);
    return g;
}

/// gather_solution: the global x assembled by global index on rank 0;
/// other ranks receive an empty vector.
inline std::vector<double> gather_solution(const LocalPartition& local, Transport& t, std::span<const double> x_owned) {
    sparsla_dist* d = local.plan(t);
    std::int64_t info[9];
    detail::check(sparsla_dist_info(d, info));
    std::vector<double> x(static_cast<std::size_t>(info[6] == 0 ? info[8] : 0));
    detail::check(sparsla_dist_gather(d, x_owned.data(), info[6] == 0 ? x.data() : nullptr, SPARSLA_MEM_HOST));
    return x;
}

}  // namespace sparsla
