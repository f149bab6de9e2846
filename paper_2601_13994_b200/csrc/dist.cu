// dist.cu — row-partitioned (domain-decomposition) Krylov loop on 1..8 GPUs.
//
// Restates the reference's distributed module (Alg. 3/4) on the
// device:
//   dist_spmv       halo exchange of the SpMV input (zero-copy for contiguous ranges,
//                   halo_pack/halo_unpack kernels otherwise) on a comm stream, overlapped
//                   with the interior-chunk SpMV; boundary chunks run once the halo landed.
//                   Rows keep their global column order, so every owned row sum equals the
//                   serial one bit for bit.
//   all_reduce_sum  each reduction point all-gathers the per-rank canonical-dot totals and
//                   sums them in ascending rank order on the device:
//                   deterministic, identical on every rank.
//   dist_cg / dist_bicgstab / dist_adjoint_solve / gather_solution.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "device.hpp"
#include "kernels.cuh"
#include "transport.hpp"

namespace sparsla_b200 {

#define CKD(x) cuda_check((x), #x)

template <class T>
static T* dmalloc(size_t n) {
    void* p = nullptr;
    CKD(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
}
template <class T>
static T* dalloc_zero(size_t n) {
    T* p = dmalloc<T>(n);
    CKD(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    return p;
}

DistCtx::~DistCtx() {
    cudaFree(d_all_chunks);
    cudaFree(d_send_idx); cudaFree(d_recv_idx); cudaFree(sendbuf); cudaFree(recvbuf);
    cudaFree(d_interior); cudaFree(d_boundary); cudaFree(red_send); cudaFree(red_all);
    if (ev_x) cudaEventDestroy(ev_x);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (comm) cudaStreamDestroy(comm);
}

void DistCtx::exchange(cudaStream_t s, double* x) {
    CKD(cudaEventRecord(ev_x, s));
    CKD(cudaStreamWaitEvent(comm, ev_x, 0));
    std::vector<HaloPeer> peers(nbr.size());
    for (size_t a = 0; a < nbr.size(); ++a) {
        HaloPeer& p = peers[a];
        p.rank = nbr[a];
        p.scount = s_cnt[a];
        p.rcount = r_cnt[a];
        if (s_base[a] >= 0) {
            p.send = x + s_base[a];  // contiguous: zero-copy send
        } else {
            p.send = sendbuf + s_off[a];
            if (p.scount)
                halo_pack_kernel<<<(unsigned)((p.scount + 255) / 256), 256, 0, comm>>>(x, d_send_idx + s_off[a],
                                                                                     p.scount, sendbuf + s_off[a]);
        }
        p.recv = r_base[a] >= 0 ? x + r_base[a] : recvbuf + r_off[a];
    }
    CKD(cudaGetLastError());
    tr->exchange(comm, peers);
    for (size_t a = 0; a < nbr.size(); ++a)
        if (r_base[a] < 0 && r_cnt[a])
            halo_unpack_kernel<<<(unsigned)((r_cnt[a] + 255) / 256), 256, 0, comm>>>(x, d_recv_idx + r_off[a], r_cnt[a],
                                                                                   recvbuf + r_off[a]);
    CKD(cudaGetLastError());
    CKD(cudaEventRecord(ev_halo, comm));
}

// ---------------------------------------------- fused peer-memory collectives setup ----
// Collective over the plan's transport.  Every rank publishes (pid, raw pointers, cudaIpc
// handles) of its mailbox, flags and SpMV-input vector; peers in the same process use the
// raw pointers (peer access enabled across devices), peers in other processes open the IPC
// handles.  Then each rank learns where its send values land in every neighbour's vector
// and builds per-chunk push tables for the in-kernel halo push.
void Solver::p2p_setup() {
    DistCtx* C = dist;
    Transport* tr = C->tr;
    const int P = tr->P, me = tr->rank;
    cudaStream_t s0 = stream;
    double* mail = dalloc_zero<double>((size_t)8 * P * 8);
    auto* mflag = dalloc_zero<unsigned long long>((size_t)8 * P);
    auto* hflag = dalloc_zero<unsigned long long>((size_t)4 * P);
    p2p_allocs = {mail, mflag, hflag};
    // the SpMV inputs whose halos the kernels push: CG p; BiCGStab p-hat and s-hat
    const bool bicg = backend == SPARSLA_BACKEND_BICGSTAB;
    constexpr int NB = 5;
    void* mine[NB] = {mail, mflag, hflag, bicg ? (void*)ph : (void*)p, bicg ? (void*)sh : (void*)p};
    constexpr int W = 2 + NB + 8 * NB;  // doubles per rank: pid, device, pointers, 64-byte handles
    std::vector<double> blob(W, 0.0);
    blob[0] = (double)getpid();
    blob[1] = (double)A->device;
    for (int i = 0; i < NB; ++i) std::memcpy(&blob[2 + i], &mine[i], 8);
    std::string ipc_err;
    for (int i = 0; i < NB; ++i) {
        cudaIpcMemHandle_t hd;
        const cudaError_t e = cudaIpcGetMemHandle(&hd, mine[i]);
        if (e == cudaSuccess) std::memcpy(&blob[2 + NB + 8 * i], &hd, 64);
        else { ipc_err = cudaGetErrorString(e); cudaGetLastError(); }  // in-process peers do not need it
    }
    double* dblob = dalloc_zero<double>((size_t)W * (P + 1));
    CKD(memcpy_sync(dblob, blob.data(), W * 8, cudaMemcpyHostToDevice));
    tr->allgather(s0, dblob, dblob + W, W);
    std::vector<double> all((size_t)W * P);
    CKD(cudaMemcpyAsync(all.data(), dblob + W, all.size() * 8, cudaMemcpyDeviceToHost, s0));
    CKD(cudaStreamSynchronize(s0));
    cudaFree(dblob);
    tr->allgathers -= 1;
    std::vector<void*> peer[NB];
    C->p2p_shared_device = false;
    for (int q = 0; q < P; ++q) {
        const double* bq = &all[(size_t)q * W];
        // same ordinal = same GPU for in-process peers; processes with different
        // CUDA_VISIBLE_DEVICES mappings are treated conservatively the same way
        if (q != me && (int)bq[1] == A->device) C->p2p_shared_device = true;
        for (int i = 0; i < NB; ++i) {
            void* ptr = nullptr;
            if (q == me) {
                ptr = mine[i];
            } else if ((long long)bq[0] == (long long)getpid()) {
                std::memcpy(&ptr, &bq[2 + i], 8);
                const int pdev = (int)bq[1];
                if (pdev != A->device) {
                    int can = 0;
                    CKD(cudaDeviceCanAccessPeer(&can, A->device, pdev));
                    if (!can) fail(SPARSLA_ERR_UNSUPPORTED, "fused collectives need peer access between GPUs");
                    cudaError_t e = cudaDeviceEnablePeerAccess(pdev, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else CKD(e);
                }
            } else {
                cudaIpcMemHandle_t hd;
                std::memcpy(&hd, &bq[2 + NB + 8 * i], 64);
                const cudaError_t e = cudaIpcOpenMemHandle(&ptr, hd, cudaIpcMemLazyEnablePeerAccess);
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    unsigned sum = 0;
                    for (int b = 0; b < 64; ++b) sum += (unsigned char)hd.reserved[b];
                    fail(SPARSLA_ERR_CUDA, std::string("cudaIpcOpenMemHandle(rank ") + std::to_string(q) + ", buffer " +
                                               std::to_string(i) + "): " + cudaGetErrorString(e) +
                                               " (handle byte sum " + std::to_string(sum) + "; local GetMemHandle: " +
                                               (ipc_err.empty() ? "ok" : ipc_err) + ")");
                }
                p2p_ipc_opened.push_back(ptr);
            }
            peer[i].push_back(ptr);
        }
    }
    // where my send values land: each neighbour tells me its recv positions for me
    const size_t nn = C->nbr.size();
    std::vector<long long> rpos_cnt(nn);
    long long tot_recv = 0, tot_send = 0;
    for (size_t a = 0; a < nn; ++a) { tot_recv += C->r_cnt[a]; tot_send += C->s_cnt[a]; }
    std::vector<int32_t> my_recv(tot_recv);
    if (tot_recv) CKD(memcpy_sync(my_recv.data(), C->d_recv_idx, tot_recv * 4, cudaMemcpyDeviceToHost));
    std::vector<double> recv_d(my_recv.begin(), my_recv.end());
    double* dbuf = dalloc_zero<double>((size_t)tot_recv + tot_send + 2);
    if (tot_recv) CKD(memcpy_sync(dbuf, recv_d.data(), tot_recv * 8, cudaMemcpyHostToDevice));
    std::vector<HaloPeer> hp(nn);
    for (size_t a = 0; a < nn; ++a)
        hp[a] = HaloPeer{C->nbr[a], dbuf + C->r_off[a], C->r_cnt[a], dbuf + tot_recv + C->s_off[a], C->s_cnt[a]};
    tr->exchange(s0, hp);
    tr->exchanges -= 1;
    tr->messages -= (long long)nn;
    std::vector<double> remote(tot_send);
    if (tot_send) CKD(cudaMemcpyAsync(remote.data(), dbuf + tot_recv, tot_send * 8, cudaMemcpyDeviceToHost, s0));
    CKD(cudaStreamSynchronize(s0));
    cudaFree(dbuf);
    std::vector<int32_t> my_send(tot_send);
    if (tot_send) CKD(memcpy_sync(my_send.data(), C->d_send_idx, tot_send * 4, cudaMemcpyDeviceToHost));
    // non-contiguous send lists live in d_send_idx; contiguous ones were not uploaded there
    // as positions, so rebuild the send rows from the plan: row = s_base + j when contiguous
    struct E { int32_t row, nbr; long long pos; };
    std::vector<E> ent;
    ent.reserve(tot_send);
    for (size_t a = 0; a < nn; ++a)
        for (long long j = 0; j < C->s_cnt[a]; ++j) {
            const int32_t row = C->s_base[a] >= 0 ? (int32_t)(C->s_base[a] + j) : my_send[C->s_off[a] + j];
            ent.push_back(E{row, (int32_t)a, (long long)remote[C->s_off[a] + j]});
        }
    const long long nch = (n + kChunk - 1) / kChunk;
    std::stable_sort(ent.begin(), ent.end(), [](const E& u, const E& v) { return u.row / kChunk < v.row / kChunk; });
    std::vector<int32_t> pptr(nch + 1, 0), prow(ent.size()), pnbr(ent.size());
    std::vector<long long> ppos(ent.size());
    for (size_t e = 0; e < ent.size(); ++e) {
        ++pptr[ent[e].row / kChunk + 1];
        prow[e] = ent[e].row; pnbr[e] = ent[e].nbr; ppos[e] = ent[e].pos;
    }
    for (long long c = 0; c < nch; ++c) pptr[c + 1] += pptr[c];
    auto upload = [&](const void* src, size_t bytes) {
        void* dst = nullptr;
        CKD(cudaMalloc(&dst, std::max<size_t>(bytes, 8)));
        if (bytes) CKD(memcpy_sync(dst, src, bytes, cudaMemcpyHostToDevice));
        p2p_allocs.push_back(dst);
        return dst;
    };
    std::vector<double*> pv(nn), pv2(nn);
    std::vector<int32_t> nr(nn);
    for (size_t a = 0; a < nn; ++a) {
        pv[a] = static_cast<double*>(peer[3][C->nbr[a]]);
        pv2[a] = static_cast<double*>(peer[4][C->nbr[a]]);
        nr[a] = C->nbr[a];
    }
    P2PCtx X{};
    X.P = P; X.me = me; X.nnbr = (int)nn;
    X.peer_mail = (double**)upload(peer[0].data(), P * sizeof(void*));
    X.peer_mflag = (unsigned long long**)upload(peer[1].data(), P * sizeof(void*));
    X.peer_hflag = (unsigned long long**)upload(peer[2].data(), P * sizeof(void*));
    X.my_mail = mail; X.my_mflag = mflag; X.my_hflag = hflag;
    X.nbr_rank = (const int32_t*)upload(nr.data(), nn * 4);
    X.push_ptr = (const int32_t*)upload(pptr.data(), pptr.size() * 4);
    X.push_row = (const int32_t*)upload(prow.data(), prow.size() * 4);
    X.push_nbr = (const int32_t*)upload(pnbr.data(), pnbr.size() * 4);
    X.push_pos = (const long long*)upload(ppos.data(), ppos.size() * 8);
    X.peer_vec = (double**)upload(pv.data(), nn * sizeof(void*));
    X.peer_vec2 = (double**)upload(pv2.data(), nn * sizeof(void*));
    const int zero = 0;
    X.err = (int*)upload(&zero, sizeof(int));
    p2p_err = X.err;
    X.timeout_ns = (unsigned long long)(transport_timeout_s() * 1e9);
    d_p2p = (P2PCtx*)upload(&X, sizeof(X));
}

void Solver::p2p_release() noexcept {
    for (void* p2 : p2p_ipc_opened) cudaIpcCloseMemHandle(p2);
    for (void* p2 : p2p_allocs) cudaFree(p2);
    p2p_ipc_opened.clear();
    p2p_allocs.clear();
    d_p2p = nullptr;
    p2p_err = nullptr;
    cudaGetLastError();
}

}  // namespace sparsla_b200

using namespace sparsla_b200;

struct sparsla_local_hub { std::shared_ptr<LocalHub> hub; };

// A Transport handle shared by every plan built on it.
struct sparsla_transport {
    std::shared_ptr<Transport> tr;
    int device = 0;
    cudaStream_t stream = nullptr;
    double* buf = nullptr;  // [1 + P] all_reduce staging
    ~sparsla_transport() {
        DeviceGuard g(device, true);
        cudaFree(buf);
        if (stream) cudaStreamDestroy(stream);
    }
};

struct sparsla_dist {
    std::shared_ptr<Transport> tr;
    std::unique_ptr<DistCtx> ctx;
    DevCsr* A = nullptr;
    DevCsr* AT = nullptr;            // transposed values in A's local pattern (adjoint)
    std::vector<int64_t> owned;      // this rank's global ids
    std::vector<int64_t> all_owned;  // rank 0: concatenation over ranks (gather_solution)
    std::vector<int64_t> all_count;  // rank 0: owned count per rank
    long long n_global = 0;
    long long alg_exchanges = 0, alg_allreduces = 0, alg_messages = 0;  // live algorithm work
    // parked host-buffer solvers per backend (workspace, graphs, fused-collective mappings),
    // reused by the next collective solve with the same preconditioner and fused setting
    Solver* parked[2] = {nullptr, nullptr};
    bool parked_fused[2] = {false, false};
    ~sparsla_dist() {
        if (A) {
            DeviceGuard g(A->device, true);
            for (auto*& p : parked) { delete p; p = nullptr; }
            ctx.reset(); delete AT; delete A;
        }
    }
};

namespace {
bool solver_cache_enabled() {
    static const bool on = [] { const char* e = getenv("SPARSLA_SOLVER_CACHE"); return !e || atoi(e) != 0; }();
    return on;
}

bool contiguous_range(const std::vector<int64_t>& v, size_t b, size_t e, long long& base) {
    if (b == e) { base = 0; return true; }
    for (size_t k = b + 1; k < e; ++k)
        if (v[k] != v[k - 1] + 1) { base = -1; return false; }
    base = v[b];
    return true;
}

// Builds the device plan for one rank.  Collective over the transport (count handshake).
sparsla_dist* build_plan(int device, std::shared_ptr<Transport> tr, const sparsla_local* L) {
    DeviceGuard g(device);
    auto D = std::make_unique<sparsla_dist>();
    const long long no = (long long)L->owned.size(), nh = (long long)L->halo.size();
    // device layout of SpMV inputs: [owned | gap | halo], the halo starting on its own
    // 128-byte lines (>= 16 doubles after the last owned value): halo values may be written
    // by peers while this rank's SpMV already streams owned lines through the read-only
    // cache, so no line may mix owned and halo data.  SPEC-layout maps stay n_owned-based.
    const long long hb = ((no + 16 + 15) / 16) * 16;
    std::vector<int32_t> rp(L->rp.begin(), L->rp.end()), ci(L->ci.size());
    for (size_t k = 0; k < ci.size(); ++k) ci[k] = (int32_t)(L->ci[k] < no ? L->ci[k] : L->ci[k] - no + hb);
    D->A = DevCsr::create<int32_t>(device, no, hb + nh, rp.data(), ci.data(), L->v.data(), true);
    auto C = std::make_unique<DistCtx>();
    C->tr = tr.get();
    C->device = device;
    C->n_owned = no;
    C->n_halo = nh;
    C->halo_base = hb;
    C->vec_len = hb + nh;
    const size_t nn = L->neighbors.size();
    for (size_t a = 0; a < nn; ++a) {
        C->nbr.push_back(L->neighbors[a]);
        C->s_off.push_back(L->send_ptr[a]);
        C->s_cnt.push_back(L->send_ptr[a + 1] - L->send_ptr[a]);
        C->r_off.push_back(L->recv_ptr[a]);
        C->r_cnt.push_back(L->recv_ptr[a + 1] - L->recv_ptr[a]);
        long long sb, rb;
        contiguous_range(L->send_idx, L->send_ptr[a], L->send_ptr[a + 1], sb);
        contiguous_range(L->recv_idx, L->recv_ptr[a], L->recv_ptr[a + 1], rb);
        if (rb >= 0 && L->recv_ptr[a + 1] > L->recv_ptr[a]) rb = rb - no + hb;
        C->s_base.push_back(sb);
        C->r_base.push_back(rb);
    }
    std::vector<int32_t> si(L->send_idx.begin(), L->send_idx.end()), ri(L->recv_idx.size());
    for (size_t k = 0; k < ri.size(); ++k) ri[k] = (int32_t)(L->recv_idx[k] - no + hb);
    C->d_send_idx = dmalloc<int32_t>(si.size());
    C->d_recv_idx = dmalloc<int32_t>(ri.size());
    if (!si.empty()) CKD(memcpy_sync(C->d_send_idx, si.data(), si.size() * 4, cudaMemcpyHostToDevice));
    if (!ri.empty()) CKD(memcpy_sync(C->d_recv_idx, ri.data(), ri.size() * 4, cudaMemcpyHostToDevice));
    C->sendbuf = dmalloc<double>(si.size());
    C->recvbuf = dmalloc<double>(ri.size());
    // interior chunks reference no halo column; boundary chunks wait for the exchange
    const long long nch = (no + kChunk - 1) / kChunk;
    std::vector<int32_t> inter, bound;
    for (long long c = 0; c < nch; ++c) {
        bool b = false;
        const long long r1 = std::min(no, (c + 1) * kChunk);
        for (long long k = L->rp[c * kChunk]; k < L->rp[r1] && !b; ++k) b = L->ci[k] >= no;  // SPEC-layout ids
        (b ? bound : inter).push_back((int32_t)c);
    }
    C->n_interior = (long long)inter.size();
    C->n_boundary = (long long)bound.size();
    {
        std::vector<int32_t> all(inter);
        all.insert(all.end(), bound.begin(), bound.end());
        C->d_all_chunks = dmalloc<int32_t>(all.size());
        if (!all.empty()) CKD(memcpy_sync(C->d_all_chunks, all.data(), all.size() * 4, cudaMemcpyHostToDevice));
    }
    if (const char* e = getenv("SPARSLA_P2P")) C->p2p_enabled = atoi(e) != 0;
    C->d_interior = dmalloc<int32_t>(inter.size());
    C->d_boundary = dmalloc<int32_t>(bound.size());
    if (!inter.empty()) CKD(memcpy_sync(C->d_interior, inter.data(), inter.size() * 4, cudaMemcpyHostToDevice));
    if (!bound.empty()) CKD(memcpy_sync(C->d_boundary, bound.data(), bound.size() * 4, cudaMemcpyHostToDevice));
    C->red_send = dmalloc<double>(8 * 8);
    C->red_all = dmalloc<double>((size_t)8 * tr->P * 8);
    CKD(cudaMemset(C->red_send, 0, 64 * sizeof(double)));
    CKD(cudaStreamCreateWithFlags(&C->comm, cudaStreamNonBlocking));
    CKD(cudaEventCreateWithFlags(&C->ev_x, cudaEventDisableTiming));
    CKD(cudaEventCreateWithFlags(&C->ev_halo, cudaEventDisableTiming));
    D->owned = L->owned;

    // handshake without point-to-point traffic: all-gather every rank's send / recv count
    // rows so that all ranks reach the same verdict before any send/recv is posted
    // (|send p->q| must equal |recv q<-p|: structural symmetry)
    cudaStream_t s = D->A->stream;
    const int P = tr->P;
    std::vector<double> row(2 * (size_t)P + 1, 0.0);
    for (size_t a = 0; a < nn; ++a) {
        row[C->nbr[a]] = (double)C->s_cnt[a];
        row[P + C->nbr[a]] = (double)C->r_cnt[a];
    }
    row[2 * P] = (double)no;
    const int W = 2 * P + 1;
    double* hs = dmalloc<double>((size_t)W * (P + 1));
    CKD(memcpy_sync(hs, row.data(), W * 8, cudaMemcpyHostToDevice));
    tr->allgather(s, hs, hs + W, W);
    std::vector<double> all((size_t)W * P);
    CKD(cudaMemcpyAsync(all.data(), hs + W, all.size() * 8, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    cudaFree(hs);
    bool any_bad = false;
    D->n_global = 0;
    for (int p = 0; p < P; ++p) {
        for (int q = 0; q < P; ++q)
            any_bad |= all[(size_t)p * W + q] != all[(size_t)q * W + P + p];  // send p->q vs recv q<-p
        D->all_count.push_back((int64_t)all[(size_t)p * W + 2 * P]);
        D->n_global += (int64_t)all[(size_t)p * W + 2 * P];
    }
    if (D->all_count[tr->rank] != no) {
        std::string got;
        for (int p = 0; p < P; ++p) got += " " + std::to_string(D->all_count[p]);
        fail(SPARSLA_ERR_TRANSPORT, "handshake all-gather returned inconsistent owned counts (own " +
                                        std::to_string(no) + ", gathered" + got + ")");
    }
    if (any_bad)
        fail(SPARSLA_ERR_UNSUPPORTED,
             "halo maps disagree between ranks: the distributed path requires a structurally "
             "symmetric pattern (SPEC.md:510)");
    // gather_solution needs every rank's owned ids on rank 0 (ids travel bit-cast as doubles)
    {
        std::vector<HaloPeer> gp;
        double* ids = dmalloc<double>(no + 1);
        std::vector<double> idd(no);
        std::memcpy(idd.data(), L->owned.data(), no * 8);
        if (no) CKD(memcpy_sync(ids, idd.data(), no * 8, cudaMemcpyHostToDevice));
        double* rbuf = nullptr;
        if (tr->rank == 0) {
            rbuf = dmalloc<double>(D->n_global + 1);
            long long off = 0;
            for (int q = 0; q < tr->P; ++q) {
                if (q == 0) { if (no) CKD(memcpy_sync(rbuf, ids, no * 8, cudaMemcpyDeviceToDevice)); }
                else gp.push_back(HaloPeer{q, nullptr, 0, rbuf + off, D->all_count[q]});
                off += D->all_count[q];
            }
        } else {
            gp.push_back(HaloPeer{0, ids, no, nullptr, 0});
        }
        tr->exchange(s, gp);
        if (tr->rank == 0) {
            std::vector<double> h(D->n_global);
            if (D->n_global) CKD(cudaMemcpyAsync(h.data(), rbuf, D->n_global * 8, cudaMemcpyDeviceToHost, s));
            CKD(cudaStreamSynchronize(s));
            D->all_owned.resize(D->n_global);
            std::memcpy(D->all_owned.data(), h.data(), D->n_global * 8);
            cudaFree(rbuf);
        }
        CKD(cudaStreamSynchronize(s));
        cudaFree(ids);
        tr->exchanges -= 1;  // setup traffic is not part of the solver counters
        tr->messages -= (long long)gp.size();
    }
    tr->allgathers -= 1;
    D->ctx = std::move(C);
    D->tr = std::move(tr);
    return D.release();
}

struct DVec {  // staging of an owned-length vector argument (+ optional halo slots)
    double* d = nullptr;
    bool own = false;
    DVec(const double* src, long long n, long long extra, int mem, cudaStream_t s, bool copy = true) {
        if (mem == SPARSLA_MEM_DEVICE && extra == 0) { d = const_cast<double*>(src); return; }
        d = dmalloc<double>(n + extra + 2);
        own = true;
        if (copy && n)
            CKD(cudaMemcpyAsync(d, src, n * 8, mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    }
    void out(double* dst, long long n, int mem, cudaStream_t s) {
        if (own && n) CKD(cudaMemcpyAsync(dst, d, n * 8, mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    }
    ~DVec() { if (own) cudaFree(d); }
};

void dist_krylov(sparsla_dist* D, int backend, const double* b, double* x, const sparsla_solve_options* o,
                 sparsla_solve_report* rep, int mem, DevCsr* M = nullptr) {
    DevCsr* A = M ? M : D->A;
    DeviceGuard g(A->device);
    // every rank makes the same parking decisions (same call sequence), so collective setup
    // inside a new Solver happens on all ranks or on none
    const int slot = backend == SPARSLA_BACKEND_CG ? 0 : 1;
    const bool cache = !M && mem != SPARSLA_MEM_DEVICE && solver_cache_enabled();
    std::unique_ptr<Solver> Sp;
    if (cache && D->parked[slot] && D->parked[slot]->opts.preconditioner == o->preconditioner &&
        D->parked_fused[slot] == D->ctx->p2p_enabled) {
        Solver::validate(*o, true);
        Sp.reset(D->parked[slot]);
        D->parked[slot] = nullptr;
        Sp->opts = *o;
    } else {
        if (cache && D->parked[slot]) { delete D->parked[slot]; D->parked[slot] = nullptr; }
        Sp = std::make_unique<Solver>(A, backend, *o, D->ctx.get());
    }
    Solver& S = *Sp;
    S.set_b(b, mem);
    if (mem == SPARSLA_MEM_DEVICE) S.x = x;
    S.reset();
    S.run();
    S.report(rep);
    int perr = 0;
    if (S.p2p_err) CKD(memcpy_sync(&perr, S.p2p_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (S.h_st->status == ST_TRANSPORT || perr)
        fail(SPARSLA_ERR_TRANSPORT, "fused peer collective timed out after " + std::to_string(transport_timeout_s()) +
                                        " s: a peer rank stopped contributing (SPEC.md:534)");
    D->alg_exchanges += S.h_st->spmv_count;  // one halo exchange per SpMV (incl. the initial one)
    D->alg_allreduces += S.h_st->reductions;
    D->alg_messages += S.h_st->spmv_count * (long long)D->ctx->nbr.size();
    if (mem != SPARSLA_MEM_DEVICE && A->nrows)
        CKD(cudaMemcpyAsync(x, S.x, A->nrows * 8, cudaMemcpyDeviceToHost, A->stream));
    CKD(cudaStreamSynchronize(A->stream));
    if (cache) {
        D->parked_fused[slot] = D->ctx->p2p_enabled;
        D->parked[slot] = Sp.release();
    }
}

}  // namespace

extern "C" {

int sparsla_nccl_unique_id(unsigned char* out) {
    return guarded([&] { nccl_unique_id(out); });
}

int sparsla_dist_create_nccl(int device, int nranks, int rank, const unsigned char* id, const sparsla_local* L,
                             sparsla_dist** out) {
    return guarded([&] {
        if (!L || !out || !id) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(device);
        std::shared_ptr<Transport> tr(new NcclTransport(nranks, rank, id));
        *out = build_plan(device, std::move(tr), L);
    });
}

int sparsla_dist_create_host(int device, int nranks, int rank, const sparsla_host_transport* T,
                             const sparsla_local* L, sparsla_dist** out) {
    return guarded([&] {
        if (!L || !out || !T || !T->allgather || !T->exchange) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(device);
        HostCallbacks cb{T->user, T->allgather, T->exchange};
        std::shared_ptr<Transport> tr(new HostTransport(nranks, rank, cb));
        *out = build_plan(device, std::move(tr), L);
    });
}

int sparsla_local_hub_create(int nranks, sparsla_local_hub** out) {
    return guarded([&] {
        if (nranks < 1) fail(SPARSLA_ERR_INVALID_ARGUMENT, "nranks >= 1");
        *out = new sparsla_local_hub{std::make_shared<LocalHub>(nranks)};
    });
}

int sparsla_local_hub_destroy(sparsla_local_hub* h) {
    delete h;
    return SPARSLA_OK;
}

int sparsla_dist_create_local(int device, sparsla_local_hub* hub, int rank, const sparsla_local* L,
                              sparsla_dist** out) {
    return guarded([&] {
        if (!L || !out || !hub) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(device);
        std::shared_ptr<Transport> tr(new LocalTransport(hub->hub, rank));
        *out = build_plan(device, std::move(tr), L);
    });
}

// ---- first-class transports: one per rank, shared by its plans ----
static sparsla_transport* wrap_transport(int device, std::shared_ptr<Transport> tr) {
    auto T = std::make_unique<sparsla_transport>();
    T->device = device;
    T->tr = std::move(tr);
    CKD(cudaStreamCreateWithFlags(&T->stream, cudaStreamNonBlocking));
    T->buf = dmalloc<double>(1 + (size_t)T->tr->P + 1);
    return T.release();
}

int sparsla_transport_create_nccl(int device, int nranks, int rank, const unsigned char* id, sparsla_transport** out) {
    return guarded([&] {
        if (!out || !id) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(device);
        *out = wrap_transport(device, std::make_shared<NcclTransport>(nranks, rank, id));
    });
}

int sparsla_transport_create_local(int device, sparsla_local_hub* hub, int rank, sparsla_transport** out) {
    return guarded([&] {
        if (!out || !hub) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(device);
        *out = wrap_transport(device, std::make_shared<LocalTransport>(hub->hub, rank));
    });
}

int sparsla_transport_create_host(int device, int nranks, int rank, const sparsla_host_transport* T,
                                  sparsla_transport** out) {
    return guarded([&] {
        if (!out || !T || !T->allgather || !T->exchange) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(device);
        HostCallbacks cb{T->user, T->allgather, T->exchange};
        *out = wrap_transport(device, std::make_shared<HostTransport>(nranks, rank, cb));
    });
}

int sparsla_transport_destroy(sparsla_transport* T) {
    return guarded([&] { delete T; });
}

// all_reduce_sum: every rank's scalar, summed in ascending rank order.
int sparsla_transport_all_reduce_sum(sparsla_transport* T, double local, double* global) {
    return guarded([&] {
        if (!T || !global) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(T->device);
        const int P = T->tr->P;
        CKD(cudaMemcpyAsync(T->buf, &local, 8, cudaMemcpyHostToDevice, T->stream));
        T->tr->allgather(T->stream, T->buf, T->buf + 1, 1);
        std::vector<double> all((size_t)P);
        CKD(cudaMemcpyAsync(all.data(), T->buf + 1, (size_t)P * 8, cudaMemcpyDeviceToHost, T->stream));
        CKD(cudaStreamSynchronize(T->stream));
        double acc = all[0];
        for (int q = 1; q < P; ++q) acc = acc + all[(size_t)q];
        *global = acc;
        T->tr->check();
    });
}

int sparsla_transport_info(const sparsla_transport* T, int64_t* out) {
    return guarded([&] {
        if (!T || !out) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        out[0] = T->tr->P; out[1] = T->tr->rank; out[2] = T->tr->exchanges; out[3] = T->tr->allgathers;
        out[4] = T->tr->messages;
    });
}

int sparsla_dist_create(sparsla_transport* T, const sparsla_local* L, sparsla_dist** out) {
    return guarded([&] {
        if (!T || !L || !out) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(T->device);
        *out = build_plan(T->device, T->tr, L);
    });
}

// halo_exchange: the neighbours' current owned values of this rank's halo
// (ascending global index, the HaloMap's canonical order), from the owned slice.
int sparsla_dist_halo_exchange(sparsla_dist* D, const double* x_owned, double* halo, int32_t mem) {
    return guarded([&] {
        DevCsr* A = D->A;
        DistCtx* C = D->ctx.get();
        DeviceGuard g(A->device);
        cudaStream_t s = A->stream;
        DVec X(x_owned, C->n_owned, C->vec_len - C->n_owned, mem, s);
        C->exchange(s, X.d);
        CKD(cudaStreamWaitEvent(s, C->ev_halo, 0));
        if (C->n_halo)
            CKD(cudaMemcpyAsync(halo, X.d + C->halo_base, C->n_halo * 8,
                                mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        CKD(cudaStreamSynchronize(s));
        D->alg_exchanges += 1;
        D->alg_messages += (long long)C->nbr.size();
        D->tr->check();
    });
}

int sparsla_dist_destroy(sparsla_dist* D) {
    return guarded([&] { delete D; });
}

int sparsla_dist_info(const sparsla_dist* D, int64_t* info) {
    return guarded([&] {
        const DistCtx& C = *D->ctx;
        info[0] = C.n_owned; info[1] = C.n_halo; info[2] = (int64_t)C.nbr.size();
        info[3] = C.n_interior; info[4] = C.n_boundary; info[5] = D->tr->P; info[6] = D->tr->rank;
        long long zc = 0;
        for (size_t a = 0; a < C.nbr.size(); ++a) zc += (C.s_base[a] >= 0) + (C.r_base[a] >= 0);
        info[7] = zc;  // zero-copy (contiguous) halo segments
        info[8] = D->n_global;
    });
}

int sparsla_dist_format(sparsla_dist* D, int64_t* fmt) {
    return guarded([&] {
        DevCsr* A = D->A;
        DeviceGuard g(A->device);
        fmt[0] = A->vd ? 1 : 0;
        fmt[1] = A->vd ? A->nvals : 0;
        double v = 0.0;
        fmt[2] = A->jacobi_uniform(&v) ? 1 : 0;
    });
}

int sparsla_dist_xwin(const sparsla_dist* D, int64_t* out) {
    return guarded([&] {
        if (!D || !out) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        devcsr_xwin_info(D->A, out);
    });
}

int sparsla_dist_dia(const sparsla_dist* D, int64_t* out) {
    return guarded([&] {
        if (!D || !out) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        devcsr_dia_info(D->A, out);
    });
}

int sparsla_dist_set_fused(sparsla_dist* D, int32_t on) {
    return guarded([&] { D->ctx->p2p_enabled = on != 0; });
}

int sparsla_dist_counters(const sparsla_dist* D, int64_t* out) {
    return guarded([&] {
        out[0] = D->alg_exchanges;
        out[1] = D->alg_allreduces;
        out[2] = D->alg_messages;
        out[3] = D->tr->exchanges;  // raw transport calls (include the no-op tail of the
        out[4] = D->tr->allgathers; // last graph replay after convergence)
        out[5] = D->tr->messages;
    });
}

int sparsla_dist_reset_counters(sparsla_dist* D) {
    return guarded([&] {
        D->tr->exchanges = D->tr->allgathers = D->tr->messages = 0;
        D->alg_exchanges = D->alg_allreduces = D->alg_messages = 0;
    });
}

// dist_spmv: y_owned = owned rows of A x, bit-identical to serial rows.
int sparsla_dist_set_values(sparsla_dist* D, const double* vals_local, int32_t mem) {
    return guarded([&] {
        if (!D) fail(SPARSLA_ERR_INVALID_ARGUMENT, "plan is null");
        DevCsr* A = D->A;
        DeviceGuard g(A->device);
        cudaStream_t s = A->stream;
        // barrier: every rank has left its previous solve before peer mappings go away
        double* f = dmalloc<double>(1 + (size_t)D->tr->P);
        CKD(cudaMemsetAsync(f, 0, 8, s));
        D->tr->allgather(s, f, f + 1, 1);
        CKD(cudaStreamSynchronize(s));
        cudaFree(f);
        D->tr->allgathers -= 1;
        for (auto*& p : D->parked) { delete p; p = nullptr; }
        devcsr_set_values(A, vals_local, mem);
        delete D->AT;
        D->AT = nullptr;
        D->tr->check();
    });
}

int sparsla_dist_spmv(sparsla_dist* D, const double* x_owned, double* y_owned, int32_t mem) {
    return guarded([&] {
        DevCsr* A = D->A;
        DistCtx* C = D->ctx.get();
        DeviceGuard g(A->device);
        cudaStream_t s = A->stream;
        DVec X(x_owned, C->n_owned, C->vec_len - C->n_owned, mem, s);
        DVec Y(y_owned, C->n_owned, 0, mem, s, false);
        C->exchange(s, X.d);
        RedParams none{};
        const unsigned gi = spmv_grid(A, C->n_interior), gb = spmv_grid(A, C->n_boundary);
        launch_spmv_part(A, s, SPMV_PLAIN, X.d, Y.d, nullptr, none, 0, C->d_interior, C->n_interior, gi + gb);
        CKD(cudaStreamWaitEvent(s, C->ev_halo, 0));
        launch_spmv_part(A, s, SPMV_PLAIN, X.d, Y.d, nullptr, none, 0, C->d_boundary, C->n_boundary, gi + gb);
        Y.out(y_owned, C->n_owned, mem, s);
        CKD(cudaStreamSynchronize(s));
        D->alg_exchanges += 1;
        D->alg_messages += (long long)C->nbr.size();
        D->tr->check();
    });
}

// dist_cg (Alg. 4) with SolveOptions (Jacobi, rtol) like cg_solve.
int sparsla_dist_cg_solve(sparsla_dist* D, const double* b, double* x, const sparsla_solve_options* o,
                          sparsla_solve_report* rep, int32_t mem) {
    return guarded([&] { dist_krylov(D, SPARSLA_BACKEND_CG, b, x, o, rep, mem); D->tr->check(); });
}

int sparsla_dist_bicgstab_solve(sparsla_dist* D, const double* b, double* x, const sparsla_solve_options* o,
                                sparsla_solve_report* rep, int32_t mem) {
    return guarded([&] { dist_krylov(D, SPARSLA_BACKEND_BICGSTAB, b, x, o, rep, mem); D->tr->check(); });
}

// dist_adjoint_solve: one distributed solve with A^T on the forward halo
// maps (structural symmetry), grad_b = lambda (owned), grad_vals over the local entries
// with x taken from [owned | halo] after one exchange of x.  vals_t: A^T's values in A's
// local entry order (nullptr when A is symmetric).
int sparsla_dist_adjoint_backward(sparsla_dist* D, const double* x_owned, const double* g_owned,
                                  const double* vals_t, int32_t backend, const sparsla_solve_options* o,
                                  double* grad_b, double* grad_vals, sparsla_solve_report* rep, int32_t mem) {
    return guarded([&] {
        DevCsr* A = D->A;
        DistCtx* C = D->ctx.get();
        DeviceGuard g(A->device);
        cudaStream_t s = A->stream;
        const long long no = C->n_owned;
        // global "grad_x == 0" short-circuit decided identically on every rank
        std::vector<double> hg(no);
        if (no) CKD(memcpy_sync(hg.data(), g_owned, no * 8, mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
        double nz = 0.0;
        for (double v : hg) if (v != 0.0) { nz = 1.0; break; }
        double* f = dmalloc<double>(2 + (size_t)D->tr->P);
        CKD(memcpy_sync(f, &nz, 8, cudaMemcpyHostToDevice));
        D->tr->allgather(s, f, f + 1, 1);
        std::vector<double> fl(D->tr->P);
        CKD(cudaMemcpyAsync(fl.data(), f + 1, fl.size() * 8, cudaMemcpyDeviceToHost, s));
        CKD(cudaStreamSynchronize(s));
        cudaFree(f);
        D->tr->allgathers -= 1;
        bool any = false;
        for (double v : fl) any |= v != 0.0;
        DVec GB(grad_b, no, 0, mem, s, false);
        std::memset(rep, 0, sizeof(*rep));
        rep->backend = backend;
        if (!any) {
            if (no) CKD(cudaMemsetAsync(GB.d, 0, no * 8, s));
            rep->converged = 1;
            std::snprintf(rep->diagnostic, 128, "grad_x == 0: short-circuit");
        } else {
            DevCsr* M = A;
            if (vals_t) {
                if (!D->AT) {
                    std::vector<int32_t> hrp(A->nrows + 1), hci(A->nnz);
                    CKD(memcpy_sync(hrp.data(), A->rp, (A->nrows + 1) * 4, cudaMemcpyDeviceToHost));
                    CKD(memcpy_sync(hci.data(), A->ci, A->nnz * 4, cudaMemcpyDeviceToHost));
                    std::vector<double> hv(A->nnz);
                    CKD(memcpy_sync(hv.data(), vals_t, A->nnz * 8, mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
                    D->AT = DevCsr::create<int32_t>(A->device, A->nrows, A->ncols, hrp.data(), hci.data(), hv.data(), true);
                } else {
                    CKD(memcpy_sync(D->AT->val, vals_t, A->nnz * 8, mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
                    cudaFree(D->AT->dinv);
                    D->AT->dinv = nullptr;
                    D->AT->dinv_uniform = -1;
                }
                M = D->AT;
            }
            DVec G(g_owned, no, 0, mem, s);
            CKD(cudaStreamSynchronize(s));
            dist_krylov(D, backend, G.d, GB.d, o, rep, SPARSLA_MEM_DEVICE, M);
        }
        // grad_vals: x over [owned | halo] (one exchange), lambda owned
        DVec XL(x_owned, no, C->vec_len - no, mem, s);
        C->exchange(s, XL.d);
        CKD(cudaStreamWaitEvent(s, C->ev_halo, 0));
        DVec GV(grad_vals, A->nnz, 0, mem, s, false);
        if (no) adjoint_gather_kernel<<<(unsigned)((no + 255) / 256), 256, 0, s>>>(A->rp, A->ci, no, GB.d, XL.d, GV.d);
        CKD(cudaGetLastError());
        GB.out(grad_b, no, mem, s);
        GV.out(grad_vals, A->nnz, mem, s);
        CKD(cudaStreamSynchronize(s));
        D->tr->check();
    });
}

// gather_solution: rank 0 receives every rank's owned values and places
// them by global index.  x_global is only written on rank 0 (host memory).
int sparsla_dist_gather(sparsla_dist* D, const double* x_owned, double* x_global, int32_t mem) {
    return guarded([&] {
        DevCsr* A = D->A;
        DeviceGuard g(A->device);
        cudaStream_t s = A->stream;
        const long long no = D->ctx->n_owned;
        DVec X(x_owned, no, 0, mem, s);
        std::vector<HaloPeer> gp;
        double* rbuf = nullptr;
        if (D->tr->rank == 0) {
            rbuf = dmalloc<double>(D->n_global + 1);
            long long off = 0;
            for (int q = 0; q < D->tr->P; ++q) {
                if (q == 0) { if (no) CKD(cudaMemcpyAsync(rbuf, X.d, no * 8, cudaMemcpyDeviceToDevice, s)); }
                else gp.push_back(HaloPeer{q, nullptr, 0, rbuf + off, D->all_count[q]});
                off += D->all_count[q];
            }
        } else {
            gp.push_back(HaloPeer{0, X.d, no, nullptr, 0});
        }
        D->tr->exchange(s, gp);
        D->tr->exchanges -= 1;
        D->tr->messages -= (long long)gp.size();
        if (D->tr->rank == 0) {
            std::vector<double> h(D->n_global);
            if (D->n_global) CKD(cudaMemcpyAsync(h.data(), rbuf, D->n_global * 8, cudaMemcpyDeviceToHost, s));
            CKD(cudaStreamSynchronize(s));
            for (long long k = 0; k < D->n_global; ++k) x_global[D->all_owned[k]] = h[k];
            cudaFree(rbuf);
        }
        CKD(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

// persistent distributed solver for the benchmark (same sparsla_solver handle as 1 GPU)

extern "C" int sparsla_dist_solver_create(sparsla_dist* D, int32_t backend, const double* b, int32_t mem,
                                          const sparsla_solve_options* o, sparsla_solver** out) {
    return guarded([&] {
        DeviceGuard g(D->A->device);
        auto S = std::make_unique<Solver>(D->A, backend, *o, D->ctx.get());
        S->set_b(b, mem);
        CKD(cudaStreamSynchronize(S->stream));
        S->reset();
        *out = new sparsla_solver{S.release(), nullptr, 0};
    });
}
