// transport.cu — NCCL (dlopen'ed) and in-process transports; see transport.hpp.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "common.hpp"
#include "device.hpp"
#include "transport.hpp"

namespace sparsla_b200 {

#define CKT(x) cuda_check((x), #x)

struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        // Reuse the libnccl.so.2 already mapped by the host framework (torch) if any.
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { err = std::string("cannot load libnccl.so.2: ") + dlerror(); return; }
#define LD(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name)); \
        if (!api.name) { err = "libnccl missing symbol nccl" #name; return; }
        LD(GetUniqueId) LD(CommInitRank) LD(CommDestroy) LD(CommAbort) LD(CommGetAsyncError)
        LD(GetErrorString) LD(GroupStart) LD(GroupEnd) LD(Send) LD(Recv) LD(AllGather)
#undef LD
    });
    if (!err.empty()) fail(SPARSLA_ERR_NCCL, err);
    return api;
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress)
        fail(SPARSLA_ERR_NCCL, std::string(what) + ": " + nccl_api().GetErrorString(r));
}

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

NcclTransport::NcclTransport(int nranks, int r, const unsigned char idb[128]) {
    P = nranks;
    rank = r;
    ncclUniqueId id;
    std::memcpy(&id, idb, sizeof(id));
    ncclComm_t c;
    nccl_check(nccl_api().CommInitRank(&c, nranks, id, r), "ncclCommInitRank");
    comm = c;
}

NcclTransport::~NcclTransport() {
    if (comm) nccl_api().CommDestroy(static_cast<ncclComm_t>(comm));
}

void NcclTransport::abort() {
    if (comm) nccl_api().CommAbort(static_cast<ncclComm_t>(comm));
    comm = nullptr;
}

double transport_timeout_s() {
    static const double t = [] {
        const char* e = getenv("SPARSLA_TRANSPORT_TIMEOUT");
        const double v = e ? atof(e) : 30.0;
        return v > 0.0 ? v : 30.0;
    }();
    return t;
}

void NcclTransport::check() {
    if (!comm) fail(SPARSLA_ERR_TRANSPORT, "NCCL communicator was aborted after a transport timeout");
    ncclResult_t a = ncclSuccess;
    nccl_check(nccl_api().CommGetAsyncError(static_cast<ncclComm_t>(comm), &a), "ncclCommGetAsyncError");
    if (a != ncclSuccess && a != ncclInProgress) {
        nccl_api().CommAbort(static_cast<ncclComm_t>(comm));
        comm = nullptr;
        fail(SPARSLA_ERR_NCCL, std::string("NCCL asynchronous error: ") + nccl_api().GetErrorString(a));
    }
}

void NcclTransport::exchange(cudaStream_t s, const std::vector<HaloPeer>& peers) {
    if (peers.empty()) { ++exchanges; return; }
    const NcclApi& A = nccl_api();
    auto c = static_cast<ncclComm_t>(comm);
    nccl_check(A.GroupStart(), "ncclGroupStart");
    for (const HaloPeer& p : peers) {
        if (p.scount) nccl_check(A.Send(p.send, (size_t)p.scount, ncclDouble, p.rank, c, s), "ncclSend");
        if (p.rcount) nccl_check(A.Recv(p.recv, (size_t)p.rcount, ncclDouble, p.rank, c, s), "ncclRecv");
    }
    nccl_check(A.GroupEnd(), "ncclGroupEnd");
    ++exchanges;
    messages += (long long)peers.size();
}

void NcclTransport::allgather(cudaStream_t s, const double* send, double* recv, int count) {
    nccl_check(nccl_api().AllGather(send, recv, (size_t)count, ncclDouble, static_cast<ncclComm_t>(comm), s),
               "ncclAllGather");
    ++allgathers;
}

// ----------------------------------------------------------------------- host ----
void HostTransport::exchange(cudaStream_t s, const std::vector<HaloPeer>& peers) {
    CKT(cudaStreamSynchronize(s));
    std::vector<std::vector<double>> sb(peers.size()), rb(peers.size());
    std::vector<const double*> sp(peers.size());
    std::vector<double*> rp(peers.size());
    std::vector<int32_t> rk(peers.size());
    std::vector<int64_t> sc(peers.size()), rc(peers.size());
    for (size_t a = 0; a < peers.size(); ++a) {
        sb[a].resize((size_t)peers[a].scount);
        rb[a].resize((size_t)peers[a].rcount);
        if (peers[a].scount)
            CKT(memcpy_sync(sb[a].data(), peers[a].send, peers[a].scount * 8, cudaMemcpyDeviceToHost));
        sp[a] = sb[a].data(); rp[a] = rb[a].data(); rk[a] = peers[a].rank;
        sc[a] = peers[a].scount; rc[a] = peers[a].rcount;
    }
    if (cb.exchange(cb.user, (int32_t)peers.size(), rk.data(), sp.data(), sc.data(), rp.data(), rc.data()) != 0)
        fail(SPARSLA_ERR_TRANSPORT, "host transport exchange callback failed");
    for (size_t a = 0; a < peers.size(); ++a)
        if (peers[a].rcount)
            CKT(memcpy_sync(peers[a].recv, rb[a].data(), peers[a].rcount * 8, cudaMemcpyHostToDevice));
    ++exchanges;
    messages += (long long)peers.size();
}

void HostTransport::allgather(cudaStream_t s, const double* send, double* recv, int count) {
    CKT(cudaStreamSynchronize(s));
    std::vector<double> h(count), all((size_t)count * P);
    CKT(memcpy_sync(h.data(), send, count * 8, cudaMemcpyDeviceToHost));
    if (cb.allgather(cb.user, h.data(), all.data(), count) != 0)
        fail(SPARSLA_ERR_TRANSPORT, "host transport allgather callback failed");
    CKT(memcpy_sync(recv, all.data(), all.size() * 8, cudaMemcpyHostToDevice));
    ++allgathers;
}

// ---------------------------------------------------------------------- local ----
void TimedBarrier::arrive_and_wait() {
    const double timeout_s = transport_timeout_s();
    std::unique_lock<std::mutex> lk(mu);
    if (broken) fail(SPARSLA_ERR_TRANSPORT, "collective aborted: a peer rank timed out earlier");
    const long long gen = generation;
    if (++waiting == n) {
        waiting = 0;
        ++generation;
        cv.notify_all();
        return;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                [&] { return generation != gen || broken; });
    if (!ok || broken) {
        broken = true;
        cv.notify_all();
        fail(SPARSLA_ERR_TRANSPORT, "collective timed out after " + std::to_string(timeout_s) +
                                        " s: a rank did not join (SPEC.md:534)");
    }
}

LocalHub::LocalHub(int p)
    : P(p), bar(p), ev_sent(p, nullptr), ev_done(p, nullptr),
      sendp(p, std::vector<const double*>(p, nullptr)), scount(p, std::vector<long long>(p, 0)) {}

LocalHub::~LocalHub() {
    for (auto e : ev_sent) if (e) cudaEventDestroy(e);
    for (auto e : ev_done) if (e) cudaEventDestroy(e);
}

LocalTransport::LocalTransport(std::shared_ptr<LocalHub> h, int r) : hub(std::move(h)) {
    P = hub->P;
    rank = r;
    // events live on this rank's device (the calling thread's current device)
    CKT(cudaEventCreateWithFlags(&hub->ev_sent[r], cudaEventDisableTiming));
    CKT(cudaEventCreateWithFlags(&hub->ev_done[r], cudaEventDisableTiming));
    hub->bar.arrive_and_wait();
}

void LocalTransport::exchange(cudaStream_t s, const std::vector<HaloPeer>& peers) {
    LocalHub& H = *hub;
    const int me = rank;
    for (const HaloPeer& p : peers) {
        H.sendp[me][p.rank] = p.send;
        H.scount[me][p.rank] = p.scount;
    }
    CKT(cudaEventRecord(H.ev_sent[me], s));
    H.bar.arrive_and_wait();
    bool ok = true;
    for (const HaloPeer& p : peers) {
        const int q = p.rank;
        if (H.scount[q][me] != p.rcount) { ok = false; continue; }
        CKT(cudaStreamWaitEvent(s, H.ev_sent[q], 0));
        if (p.rcount)
            CKT(cudaMemcpyAsync(p.recv, H.sendp[q][me], p.rcount * sizeof(double), cudaMemcpyDefault, s));
    }
    CKT(cudaEventRecord(H.ev_done[me], s));
    H.bar.arrive_and_wait();
    for (const HaloPeer& p : peers) CKT(cudaStreamWaitEvent(s, H.ev_done[p.rank], 0));
    ++exchanges;
    messages += (long long)peers.size();
    if (!ok) fail(SPARSLA_ERR_TRANSPORT, "halo payload size mismatch between ranks");
}

void LocalTransport::allgather(cudaStream_t s, const double* send, double* recv, int count) {
    LocalHub& H = *hub;
    const int me = rank;
    H.sendp[me][me] = send;
    CKT(cudaEventRecord(H.ev_sent[me], s));
    H.bar.arrive_and_wait();
    for (int q = 0; q < P; ++q) {
        CKT(cudaStreamWaitEvent(s, H.ev_sent[q], 0));
        CKT(cudaMemcpyAsync(recv + (size_t)q * count, H.sendp[q][q], count * sizeof(double), cudaMemcpyDefault, s));
    }
    CKT(cudaEventRecord(H.ev_done[me], s));
    H.bar.arrive_and_wait();
    for (int q = 0; q < P; ++q)
        if (q != me) CKT(cudaStreamWaitEvent(s, H.ev_done[q], 0));
    ++allgathers;
}

}  // namespace sparsla_b200
