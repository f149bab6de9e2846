// transport.hpp — rank-to-rank communication of the distributed Krylov loop.
//
// Restates the reference Transport contract (FIFO per pair,
// exactly-once delivery, collectives on all ranks) over two backings:
//   NcclTransport  — one rank per GPU (one process per GPU or one thread per GPU),
//                    ncclSend/ncclRecv per neighbour inside ncclGroupStart/End for the halo,
//                    ncclAllGather of the per-rank dot totals (summed in rank order on the
//                    device afterwards).  Stream-ordered and CUDA-graph
//                    capturable; NCCL is dlopen'ed so single-GPU users need no NCCL.
//   LocalTransport — P ranks as threads of one process that may share ONE device
//                    (the in-process-worker model of SPEC.md:529).  Device-to-device
//                    copies ordered by cross-stream events and host barriers.  Used to
//                    validate the distributed kernels on a single B200.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <memory>
#include <vector>

namespace sparsla_b200 {

struct HaloPeer {
    int rank;
    const double* send;  // device, `scount` values in canonical order
    long long scount;
    double* recv;        // device, `rcount` values in canonical order
    long long rcount;
};

struct Transport {
    int P = 1, rank = 0;
    long long exchanges = 0, allgathers = 0, messages = 0;
    virtual ~Transport() = default;
    virtual void exchange(cudaStream_t s, const std::vector<HaloPeer>& peers) = 0;
    // recv[q * count + j] = rank q's send[j]
    virtual void allgather(cudaStream_t s, const double* send, double* recv, int count) = 0;
    virtual bool capturable() const = 0;
    virtual void check() {}
    virtual void abort() {}  // tear the communicator down so device-side waits on it end
};

// SPEC.md:534 collective timeout in seconds (SPARSLA_TRANSPORT_TIMEOUT, default 30)
double transport_timeout_s();

// ---- NCCL ----
struct NcclApi;
const NcclApi& nccl_api();  // loads libnccl.so.2 on first use (TransportError if absent)
void nccl_unique_id(unsigned char out[128]);

struct NcclTransport : Transport {
    void* comm = nullptr;  // ncclComm_t
    NcclTransport(int nranks, int rank, const unsigned char id[128]);
    ~NcclTransport() override;
    void exchange(cudaStream_t s, const std::vector<HaloPeer>& peers) override;
    void allgather(cudaStream_t s, const double* send, double* recv, int count) override;
    bool capturable() const override { return true; }
    void check() override;
    void abort() override;
};

// ---- host callbacks (caller-provided collectives, e.g. torch.distributed gloo) ----
// Setup / init traffic only: device buffers are staged through host memory and the
// callbacks run synchronously on the calling thread.  With fused peer collectives the
// iteration itself never calls the transport, so this backing also lets several processes
// share ONE GPU (cudaIpc peers) — which NCCL refuses.
struct HostCallbacks {
    void* user;
    int (*allgather)(void* user, const double* send, double* recv, int64_t count);
    int (*exchange)(void* user, int32_t npeers, const int32_t* ranks, const double* const* sbuf,
                    const int64_t* scount, double* const* rbuf, const int64_t* rcount);
};

struct HostTransport : Transport {
    HostCallbacks cb;
    HostTransport(int nranks, int r, const HostCallbacks& c) : cb(c) { P = nranks; rank = r; }
    void exchange(cudaStream_t s, const std::vector<HaloPeer>& peers) override;
    void allgather(cudaStream_t s, const double* send, double* recv, int count) override;
    bool capturable() const override { return false; }
};

// ---- in-process (threads) ----
// Barrier with the reference's collective timeout (default 30 s,
// SPARSLA_TRANSPORT_TIMEOUT seconds): a rank missing from a collective surfaces as
// TransportError instead of a deadlock.
struct TimedBarrier {
    int n;
    int waiting = 0;
    long long generation = 0;
    bool broken = false;
    std::mutex mu;
    std::condition_variable cv;
    explicit TimedBarrier(int n_) : n(n_) {}
    void arrive_and_wait();
};

struct LocalHub {
    int P;
    TimedBarrier bar;
    std::vector<cudaEvent_t> ev_sent, ev_done;
    std::vector<std::vector<const double*>> sendp;  // [src][dst]
    std::vector<std::vector<long long>> scount;     // [src][dst]
    explicit LocalHub(int p);
    ~LocalHub();
};

struct LocalTransport : Transport {
    std::shared_ptr<LocalHub> hub;
    LocalTransport(std::shared_ptr<LocalHub> h, int rank);
    void exchange(cudaStream_t s, const std::vector<HaloPeer>& peers) override;
    void allgather(cudaStream_t s, const double* send, double* recv, int count) override;
    bool capturable() const override { return false; }
};

}  // namespace sparsla_b200
