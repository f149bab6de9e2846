// kernels.cuh — sm_100a kernels of the sparse Krylov hot path.
//
//   spmv_kernel<MODE,STAGED>   y = A x, rows accumulated left to right from 0.0 with
//                              separate multiply/add (__dmul_rn/__dadd_rn): bitwise equal to
//                              the reference spmv (sparse.cpp:144-152).  STAGED: the CTA's
//                              256-row round segments of row_ptr/col_idx/vals are streamed
//                              into shared memory by the TMA bulk-copy engine
//                              (cp.async.bulk + mbarrier, L2 evict_first), 4-stage ring;
//                              x is gathered through the read-only path.  The epilogue fuses
//                              the dot products the solver needs next (p.q for CG; rhat.v,
//                              and t.t, t.s, s.s for BiCGStab).
//   cg_* / bi_*                fused Jacobi-PCG / BiCGStab vector updates: every axpy of an
//                              iteration step plus its dot products in one HBM pass.
//   canonical reductions       every dot uses the fixed shape of DESIGN.md §3.2 (chunks of
//                              2048 = 256 slots x 8 rounds, slot-pair binary tree, then a
//                              1024-slot final stage done by the last CTA to finish), so
//                              results are bitwise identical to the oracle and independent of
//                              launch geometry.  Scalars (alpha, beta, omega, convergence)
//                              are computed on the device by that last CTA: no host sync
//                              inside the loop.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sparsla_b200 {

constexpr int kChunkSlots = 256;
constexpr int kChunkRounds = 8;
constexpr int64_t kChunk = kChunkSlots * kChunkRounds;  // 2048 rows / elements per chunk
constexpr int kFinalSlots = 1024;
constexpr int kSpmvThreads = 256;
constexpr int kVecThreads = 128;
constexpr int kStages = 4;
constexpr int kRpCopy = 260;  // row_ptr entries staged per round (257 needed, 16B multiple)

// ---------------------------------------------------------------- solver state -------
enum Status : int {
    ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_BD_PQ = 3, ST_BD_RHO = 4,
    ST_BD_RV = 5, ST_BD_TT = 6, ST_BD_OMEGA = 7,
    ST_TRANSPORT = 8  // fused peer collectives: a peer flag did not arrive within the timeout
};

struct KState {
    double atol, rtol;
    long long max_iter;
    double tol, bnorm, rnorm, rz, alpha, beta, omega, rho, rho_prev, rho_thr, ss;
    long long k, spmv_count, breakdown_iter;
    long long reductions;  // reduction points applied while the solve was live
    int pending_x;         // CG: alpha of this iteration computed, x += alpha p still to apply
    int x_lag;             // CG, deferred x update: x still lacks alpha_prev * p_prev (U2E -> U2O)
    double alpha_prev;
    unsigned long long ep[8];       // fused peer collectives: epochs pushed per reduction point
    unsigned long long ep_halo[4];  // ... and per halo-pushed vector
    int done, converged, status, halfstep;
    double scratch[8];  // plain dot outputs
};

enum Scalar : int {
    SC_NONE = 0, SC_STORE = 1, SC_CG_INIT = 2, SC_CG_PQ = 3, SC_CG_RR = 4,
    SC_BI_INIT = 5, SC_BI_RV = 6, SC_BI_T = 7, SC_BI_U3 = 8
};

__device__ __forceinline__ double dmax_ref(double a, double b) { return a < b ? b : a; }

// Scalar bookkeeping after a reduction point (the same decisions, in the same order, as
// the oracle's cg_core / bicgstab_core loops).
__device__ inline void apply_scalar(int which, KState* st, const double* t) {
    if (which != SC_STORE && which != SC_NONE) st->reductions += 1;
    switch (which) {
        case SC_STORE:
            for (int j = 0; j < 3; ++j) st->scratch[j] = t[j];
            break;
        case SC_CG_INIT: {
            st->rz = t[0];
            const double rr = t[1];
            st->bnorm = sqrt(t[2]);
            st->tol = dmax_ref(st->atol, __dmul_rn(st->rtol, st->bnorm));
            st->rnorm = sqrt(rr);
            st->k = 0;
            if (st->rnorm <= st->tol) { st->converged = 1; st->status = ST_CONVERGED; st->done = 1; }
            break;
        }
        case SC_CG_PQ: {
            st->spmv_count += 1;
            const double pq = t[0];
            if (!(pq > 0.0)) { st->status = ST_BD_PQ; st->breakdown_iter = st->k; st->done = 1; }
            else { st->alpha = st->rz / pq; st->pending_x = 1; }
            break;
        }
        case SC_CG_RR: {
            const double rz_new = t[0], rr = t[1];
            st->k += 1;
            st->rnorm = sqrt(rr);
            if (st->rnorm <= st->tol) { st->converged = 1; st->status = ST_CONVERGED; st->done = 1; }
            else if (st->k >= st->max_iter) { st->status = ST_MAXITER; st->done = 1; }
            else { st->beta = rz_new / st->rz; st->rz = rz_new; }
            break;
        }
        case SC_BI_INIT: {
            st->rho = t[0];
            const double rr = t[1];
            st->bnorm = sqrt(t[2]);
            st->tol = dmax_ref(st->atol, __dmul_rn(st->rtol, st->bnorm));
            st->rho_thr = __dmul_rn(1e-30, __dmul_rn(st->bnorm, st->bnorm));
            st->rnorm = sqrt(rr);
            st->k = 0;
            st->rho_prev = 1.0; st->alpha = 1.0; st->omega = 1.0;
            if (st->rnorm <= st->tol) { st->converged = 1; st->status = ST_CONVERGED; st->done = 1; }
            else if (!(fabs(st->rho) >= st->rho_thr) || !isfinite(st->rho)) {
                st->status = ST_BD_RHO; st->breakdown_iter = 0; st->done = 1;
            }
            break;
        }
        case SC_BI_RV: {
            st->spmv_count += 1;
            const double rv = t[0];
            if (!(rv != 0.0) || !isfinite(rv)) { st->status = ST_BD_RV; st->breakdown_iter = st->k; st->done = 1; }
            else st->alpha = st->rho / rv;
            break;
        }
        case SC_BI_T: {
            st->spmv_count += 1;
            const double tt = t[0], ts = t[1], ss = t[2];
            st->ss = ss;
            if (sqrt(ss) <= st->tol) st->halfstep = 1;
            else if (!(tt > 0.0)) { st->status = ST_BD_TT; st->breakdown_iter = st->k; st->done = 1; }
            else st->omega = ts / tt;
            break;
        }
        case SC_BI_U3: {
            if (st->halfstep) {
                st->k += 1;
                st->rnorm = sqrt(st->ss);
                st->converged = 1; st->status = ST_CONVERGED; st->done = 1;
                break;
            }
            st->rho_prev = st->rho;
            st->rho = t[0];
            const double rr = t[1];
            st->k += 1;
            st->rnorm = sqrt(rr);
            if (st->rnorm <= st->tol) { st->converged = 1; st->status = ST_CONVERGED; st->done = 1; }
            else if (st->omega == 0.0) { st->status = ST_BD_OMEGA; st->breakdown_iter = st->k; st->done = 1; }
            else if (st->k >= st->max_iter) { st->status = ST_MAXITER; st->done = 1; }
            else if (!(fabs(st->rho) >= st->rho_thr) || !isfinite(st->rho)) {
                st->status = ST_BD_RHO; st->breakdown_iter = st->k; st->done = 1;
            } else {
                st->beta = __dmul_rn(st->rho / st->rho_prev, st->alpha / st->omega);
            }
            break;
        }
        default: break;
    }
}

// ------------------------------------------------------ canonical reduction helpers --
// Binary tree over NW values in smem, left + right (matches the oracle's tree_reduce).
template <int NW>
__device__ __forceinline__ double tree_smem(volatile double* a) {
#pragma unroll
    for (int w = 1; w < NW; w *= 2)
#pragma unroll
        for (int i = 0; i + w < NW; i += 2 * w) a[i] = __dadd_rn(a[i], a[i + w]);
    return a[0];
}

// Slot-group value per thread (thread t holds the group sum of slots [t*G, (t+1)*G)) ->
// chunk partial on thread 0.  xor-butterfly levels 1..16 realise the pairwise tree over
// consecutive groups (IEEE addition is commutative, so both lanes get the same bits).
// CTA (BAR == 0) or named-barrier (BAR > 0, the first NT threads) synchronisation.
template <int BAR, int NT>
__device__ __forceinline__ void group_sync() {
    if constexpr (BAR == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}

template <int NT, int NDOT, int BAR = 0>
__device__ __forceinline__ void block_tree(double (&v)[NDOT], double* sred) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < NDOT; ++d) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) v[d] = __dadd_rn(v[d], __shfl_xor_sync(0xffffffffu, v[d], off));
        if (lane == 0) sred[d * NW + w] = v[d];
    }
    group_sync<BAR, NT>();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d) v[d] = tree_smem<NW>(sred + d * NW);
    }
    group_sync<BAR, NT>();  // sred reusable afterwards
}

// Level-2 reduction over m chunk partials per dot (layout [NDOT][m]); called by every
// thread of the last CTA; result valid on thread 0.  Slot s sums partials s, s + 1024, ...
// from 0.0 in that order; the loop walks the 1024-wide rows of partials so that every slot
// of every dot of this thread has its next load in flight at once (one L2 round trip per
// row instead of one per four partials of one slot — this tail runs on a single CTA after
// the whole grid, so its latency is on the iteration's critical path).
template <int NT, int NDOT, int BAR = 0>
__device__ void final_reduce(const double* partials, long long m, double (&out)[NDOT], double* sred) {
    constexpr int SPT = kFinalSlots / NT;  // consecutive slots per thread
    const int t = threadIdx.x;
    double s[NDOT][SPT];
#pragma unroll
    for (int d = 0; d < NDOT; ++d)
#pragma unroll
        for (int j = 0; j < SPT; ++j) s[d][j] = 0.0;
    const long long rows = m / kFinalSlots;  // complete rows of 1024 partials
    const double* P0 = partials + (long long)t * SPT;
    // two rows per step when the loads fit the register budget (same per-slot order)
    constexpr int RR = NDOT * SPT <= 8 ? 2 : 1;
    long long c = 0;
    for (; c + RR <= rows; c += RR) {
        double a[RR][NDOT][SPT];
#pragma unroll
        for (int q = 0; q < RR; ++q)
#pragma unroll
            for (int d = 0; d < NDOT; ++d)
#pragma unroll
                for (int j = 0; j < SPT; ++j) a[q][d][j] = __ldcg(P0 + d * m + (c + q) * kFinalSlots + j);
#pragma unroll
        for (int q = 0; q < RR; ++q)
#pragma unroll
            for (int d = 0; d < NDOT; ++d)
#pragma unroll
                for (int j = 0; j < SPT; ++j) s[d][j] = __dadd_rn(s[d][j], a[q][d][j]);
    }
    for (; c < rows; ++c) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d)
#pragma unroll
            for (int j = 0; j < SPT; ++j) s[d][j] = __dadd_rn(s[d][j], __ldcg(P0 + d * m + c * kFinalSlots + j));
    }
    const long long tail = m - rows * kFinalSlots;  // last, partial row
#pragma unroll
    for (int d = 0; d < NDOT; ++d)
#pragma unroll
        for (int j = 0; j < SPT; ++j)
            if ((long long)t * SPT + j < tail) s[d][j] = __dadd_rn(s[d][j], __ldcg(P0 + d * m + rows * kFinalSlots + j));
#pragma unroll
    for (int d = 0; d < NDOT; ++d) {
#pragma unroll
        for (int w = 1; w < SPT; w *= 2)
#pragma unroll
            for (int i = 0; i + w < SPT; i += 2 * w) s[d][i] = __dadd_rn(s[d][i], s[d][i + w]);
        out[d] = s[d][0];
    }
    block_tree<NT, NDOT, BAR>(out, sred);
}

// ------------------------------------------ fused peer-memory collectives (N>1) ----
// Distributed CG without per-iteration NCCL calls: the last CTA of a reduction kernel
// stores the rank's totals straight into every rank's mailbox (NVLink peer stores, or
// same-device stores for in-process ranks), fences at system scope and release-stores an
// epoch flag; the consuming kernel's CTAs acquire-wait on all P flags, sum the totals in
// ascending rank order and run the scalar step themselves.  The producer of the next SpMV
// input pushes its boundary values into the neighbours' halo slots inside the same kernel
// and raises a halo flag; the SpMV waits for it only before its first boundary chunk.
// Mailboxes are single-buffered: a rank can only overwrite a slot after the reader has
// pushed its own next contribution, which it does after consuming the slot.
struct P2PCtx {
    int P, me, nnbr;
    double** peer_mail;                // [P] -> rank q's mailbox [8 points][P][8]
    unsigned long long** peer_mflag;   // [P] -> rank q's flags [8 points][P]
    unsigned long long** peer_hflag;   // [P] -> rank q's halo flags [4][P]
    double* my_mail;
    unsigned long long* my_mflag;
    unsigned long long* my_hflag;
    const int32_t* nbr_rank;           // [nnbr]
    const int32_t* push_ptr;           // [nchunks+1]: halo-push entries of each chunk
    const int32_t* push_row;           // local owned row
    const int32_t* push_nbr;           // neighbour index (0..nnbr-1)
    const long long* push_pos;         // element offset in that neighbour's vector
    double** peer_vec;                 // [nnbr] -> neighbour's SpMV-input vector (p / BiCGStab p-hat)
    double** peer_vec2;                // [nnbr] -> neighbour's second SpMV input (BiCGStab s-hat)
    int* err;                          // this rank's transport-error flag (host maps it to TransportError)
    unsigned long long timeout_ns;     // SPEC.md:534 collective timeout (SPARSLA_TRANSPORT_TIMEOUT, 30 s)
};


__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// last CTA of a producer kernel (single thread)
__device__ inline void p2p_push_totals(const P2PCtx* X, KState* st, int point, const double* tot, int k) {
    const unsigned long long e = ++st->ep[point];
    for (int q = 0; q < X->P; ++q) {
        double* dst = X->peer_mail[q] + ((size_t)point * X->P + X->me) * 8;
        for (int j = 0; j < k; ++j) dst[j] = tot[j];
    }
    __threadfence_system();
    for (int q = 0; q < X->P; ++q) st_release_sys(X->peer_mflag[q] + point * X->P + X->me, e);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Bounded spin on a peer flag (collectives time out -> TransportError).  Gives
// up when the flag has not reached `e` within the timeout, or at once when another CTA of
// this rank already gave up; the first to give up raises the rank's error flag.
__device__ inline bool p2p_wait_flag(const P2PCtx* X, const unsigned long long* flag, unsigned long long e) {
    if (ld_acquire_sys(flag) >= e) return true;
    const unsigned long long t0 = globaltimer_ns();
    unsigned spins = 0;
    while (ld_acquire_sys(flag) < e) {
        __nanosleep(32);
        if ((++spins & 255) == 0) {
            if (*(volatile int*)X->err) return false;
            if (globaltimer_ns() - t0 > X->timeout_ns) {
                atomicExch(X->err, 1);
                __threadfence_system();
                return false;
            }
        }
    }
    return true;
}

// one thread per CTA of a consumer kernel: wait for every rank's totals of `point`, sum
// them in ascending rank order and apply the scalar step to S.  A timed-out
// wait ends the solve with ST_TRANSPORT instead (every kernel then exits at entry).
__device__ inline void p2p_consume(const P2PCtx* X, KState* S, int point, int k, int which) {
    const unsigned long long e = S->ep[point];
    for (int q = 0; q < X->P; ++q)
        if (!p2p_wait_flag(X, X->my_mflag + point * X->P + q, e)) {
            S->status = ST_TRANSPORT;
            S->done = 1;
            return;
        }
    double t[4] = {0, 0, 0, 0};
    for (int j = 0; j < k; ++j) {
        double s = ld_relaxed_sys(X->my_mail + ((size_t)point * X->P) * 8 + j);
        for (int q = 1; q < X->P; ++q) s = __dadd_rn(s, ld_relaxed_sys(X->my_mail + ((size_t)point * X->P + q) * 8 + j));
        t[j] = s;
    }
    apply_scalar(which, S, t);
}

// this CTA's chunk of boundary values of v straight into the neighbours' halo slots
__device__ __forceinline__ void p2p_push_halo_chunk(const P2PCtx* X, long long chunk, const double* v,
                                                    double* const* peers) {
    for (int e = X->push_ptr[chunk] + threadIdx.x; e < X->push_ptr[chunk + 1]; e += blockDim.x)
        peers[X->push_nbr[e]][X->push_pos[e]] = v[X->push_row[e]];
}
// last CTA of the producer: raise halo flag v on every neighbour (after a system fence)
__device__ inline void p2p_raise_halo(const P2PCtx* X, KState* st, int v) {
    const unsigned long long e = ++st->ep_halo[v];
    for (int a = 0; a < X->nnbr; ++a) st_release_sys(X->peer_hflag[X->nbr_rank[a]] + v * X->P + X->me, e);
}

// wait until every neighbour has pushed this epoch's halo of vector v (bounded: on a
// timeout the SpMV proceeds on stale halo values and the next consume ends the solve)
__device__ inline void p2p_wait_halo(const P2PCtx* X, int v, unsigned long long e) {
    for (int a = 0; a < X->nnbr; ++a) {
        const int q = X->nbr_rank[a];
        if (!p2p_wait_flag(X, X->my_hflag + v * X->P + q, e)) return;
    }
}

// Publish this CTA's chunk partials; the last CTA (ticket) finishes the reduction and runs
// the scalar step (or, distributed, writes the rank's totals for the all-gather).
struct RedParams {
    double* partials;     // [NDOT][nchunks]
    long long nchunks;
    unsigned* ticket;     // reset to 0 by the last CTA
    unsigned expected;    // number of CTAs contributing (all launches of this point)
    KState* st;
    double* red_out;      // distributed: rank totals -> all-gather; else nullptr
    int scalar;           // Scalar op applied by the last CTA (single rank)
    const P2PCtx* p2p;    // fused peer collectives: push the totals of `point` instead
    int point;
    const KState* s_loc;  // consumer kernels: CTA-local scalar state to write back first
    double* slotsum;      // [4][kFinalSlots] scratch: the last kFinishers CTAs split the
    unsigned* ticket2;    //   level-2 slot sums (multi_finish); nullptr = one finishing CTA
};

// Parallel level-2 reduction.  The CTAs that draw the last kFinishers tickets of a
// reduction point each wait until every CTA has published its partials, then sum 1/K of
// the kFinalSlots slots (slot s: 0.0 + partials s, s + 1024, ... in that order, 8 loads in
// flight) into `slotsum`; the last of them combines the slot sums exactly as final_reduce
// does (4 consecutive slots per thread, pairwise, then block_tree) — the same additions in
// the same order, bit-identical, but the ~48 sequential L2 round trips of one CTA become ~6
// per finisher.  Returns true on the CTA whose thread 0 then holds the totals in `out`.
constexpr int kFinishers = 8;
// Only for a reduction point that is ONE launch (the finishers wait on CTAs of their own
// grid, which free SM slots always let run: an interior/boundary split whose second launch
// waits for the first would deadlock) and without fused peer collectives (a same-GPU peer's
// kernel spinning on this rank's totals could hold the slots the remaining CTAs need).
__device__ __forceinline__ bool multi_ok(const RedParams& R) {
    return R.slotsum != nullptr && R.p2p == nullptr && R.expected >= (unsigned)kFinishers &&
           R.expected == gridDim.x;
}
template <int NT, int NFIN, int BAR = 0>
__device__ bool multi_finish(const RedParams& R, int fin, double (&out)[NFIN], double* sred, int* s_flag) {
    constexpr int SPF = kFinalSlots / kFinishers;  // slots per finisher
    const int t = threadIdx.x;
    const long long m = R.nchunks;
    if (t == 0) {
        while (*reinterpret_cast<volatile unsigned*>(R.ticket) < R.expected) __nanosleep(64);
    }
    group_sync<BAR, NT>();
    __threadfence();
    for (int it = t; it < NFIN * SPF; it += NT) {
        const int d = it / SPF, sl = fin * SPF + it % SPF;
        const double* pp = R.partials + d * m;
        double acc = 0.0;
        long long c = sl;
        for (; c + 7 * kFinalSlots < m; c += 8 * kFinalSlots) {
            double a[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] = __ldcg(pp + c + q * kFinalSlots);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, a[q]);
        }
        for (; c < m; c += kFinalSlots) acc = __dadd_rn(acc, __ldcg(pp + c));
        R.slotsum[d * kFinalSlots + sl] = acc;
    }
    __threadfence();
    group_sync<BAR, NT>();
    if (t == 0) *s_flag = atomicAdd(R.ticket2, 1u) == kFinishers - 1;
    group_sync<BAR, NT>();
    if (!*s_flag) return false;
    __threadfence();
    constexpr int SPT = kFinalSlots / NT;
#pragma unroll
    for (int d = 0; d < NFIN; ++d) {
        double v[SPT];
#pragma unroll
        for (int j = 0; j < SPT; ++j) v[j] = __ldcg(R.slotsum + d * kFinalSlots + t * SPT + j);
#pragma unroll
        for (int w = 1; w < SPT; w *= 2)
#pragma unroll
            for (int i = 0; i + w < SPT; i += 2 * w) v[i] = __dadd_rn(v[i], v[i + w]);
        out[d] = v[0];
    }
    block_tree<NT, NFIN, BAR>(out, sred);
    if (t == 0) *R.ticket2 = 0u;
    return true;
}

// NFIN >= NDOT: the last CTA reduces NFIN partial rows; rows NDOT.. were published per
// chunk by an earlier kernel of the same reduction point (BiCGStab: s.s by update 2).
template <int NT, int NDOT, int NFIN = NDOT>
__device__ void publish_and_finish(double (&part)[NDOT], long long chunk, const RedParams& R,
                                   double* sred) {
    __shared__ int s_last;
    __shared__ int s_fin;
    const bool multi = multi_ok(R);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d) R.partials[d * R.nchunks + chunk] = part[d];
        __threadfence();
        const unsigned prev = atomicAdd(R.ticket, 1u);
        s_last = (prev == R.expected - 1);
        s_fin = multi && prev >= R.expected - kFinishers ? (int)(prev - (R.expected - kFinishers)) : -1;
    }
    __syncthreads();
    double tot[NFIN];
    if (multi) {
        if (s_fin < 0) return;
        if (!multi_finish<NT, NFIN>(R, s_fin, tot, sred, &s_last)) return;
    } else {
        if (!s_last) return;
        __threadfence();
        final_reduce<NT, NFIN>(R.partials, R.nchunks, tot, sred);
    }
    if (threadIdx.x == 0) {
        if (R.p2p) {
            if (R.s_loc) *R.st = *R.s_loc;
            if (!R.st->done) {
                double t3[4] = {0, 0, 0, 0};
#pragma unroll
                for (int d = 0; d < NFIN; ++d) t3[d] = tot[d];
                p2p_push_totals(R.p2p, R.st, R.point, t3, NFIN);
            }
        } else if (R.red_out) {
#pragma unroll
            for (int d = 0; d < NFIN; ++d) R.red_out[d] = tot[d];
        } else {
            double t3[4] = {0, 0, 0, 0};
#pragma unroll
            for (int d = 0; d < NFIN; ++d) t3[d] = tot[d];
            apply_scalar(R.scalar, R.st, t3);
        }
        *R.ticket = 0u;
        __threadfence();
    }
}

// Persistent kernels: each CTA publishes several chunk partials, then takes ONE ticket;
// the last CTA to finish reduces all chunks (same canonical result as publish_and_finish).
template <int NT, int NDOT, int BAR, int NFIN = NDOT>
__device__ void ticket_and_finish(const RedParams& R, double* sred, int* s_flag) {
    const bool multi = multi_ok(R);
    __shared__ int s_fin;
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(R.ticket, 1u);
        *s_flag = (prev == R.expected - 1);
        s_fin = multi && prev >= R.expected - kFinishers ? (int)(prev - (R.expected - kFinishers)) : -1;
    }
    group_sync<BAR, NT>();
    double tot[NFIN];
    if (multi) {
        if (s_fin < 0) return;
        if (!multi_finish<NT, NFIN, BAR>(R, s_fin, tot, sred, s_flag)) return;
    } else {
        if (!*s_flag) return;
        __threadfence();
        final_reduce<NT, NFIN, BAR>(R.partials, R.nchunks, tot, sred);
    }
    if (threadIdx.x == 0) {
        if (R.p2p) {
            if (R.s_loc) *R.st = *R.s_loc;
            if (!R.st->done) {
                double t3[4] = {0, 0, 0, 0};
#pragma unroll
                for (int d = 0; d < NFIN; ++d) t3[d] = tot[d];
                p2p_push_totals(R.p2p, R.st, R.point, t3, NFIN);
            }
        } else if (R.red_out) {
#pragma unroll
            for (int d = 0; d < NFIN; ++d) R.red_out[d] = tot[d];
        } else {
            double t3[4] = {0, 0, 0, 0};
#pragma unroll
            for (int d = 0; d < NFIN; ++d) t3[d] = tot[d];
            apply_scalar(R.scalar, R.st, t3);
        }
        *R.ticket = 0u;
        __threadfence();
    }
}

// ------------------------------------------------------------------ PTX helpers ------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// TMA bulk copy global -> shared (non-tensor), completion on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

// ------------------------------------------------------------------------ SpMV -------
enum SpmvMode : int { SPMV_PLAIN = 0, SPMV_CG = 1, SPMV_BICG_V = 2, SPMV_BICG_T = 3 };
template <int MODE> struct SpmvDots { static constexpr int n = 0; };
template <> struct SpmvDots<SPMV_CG> { static constexpr int n = 1; };
template <> struct SpmvDots<SPMV_BICG_V> { static constexpr int n = 1; };
template <> struct SpmvDots<SPMV_BICG_T> { static constexpr int n = 2; };  // t.t, t.s (s.s: update 2)
// partial rows reduced at the SpMV's reduction point (BiCGStab t: t.t, t.s and s.s, whose
// per-chunk partials bicg_update2 published when it produced s — same canonical shape)
template <int MODE> struct SpmvFin { static constexpr int n = SpmvDots<MODE>::n; };
template <> struct SpmvFin<SPMV_BICG_T> { static constexpr int n = 3; };

struct SpmvParams {
    const int32_t* rp;
    const int32_t* ci;
    const double* val;
    const double* x;    // gathered input ([owned | halo] when distributed)
    double* y;
    long long n;        // rows
    long long chunk0;   // first chunk index handled by this launch (interior/boundary split)
    long long nch;      // number of chunks handled by this launch
    const int32_t* chunk_list;  // optional: chunk ids of this launch (interior / boundary rows)
    const P2PCtx* p2p;          // fused peer collectives: list = [interior | boundary] in ONE launch,
    long long n_interior;       //   consumers wait for the halo before list index n_interior
    int halo_v;
    const double* aux;  // BICG_V: rhat, BICG_T: s
    const uint8_t* vidx;  // value-dictionary kernels: 1-byte value index per entry ...
    const double* vtab;   // ... into this table of the matrix's <= 256 distinct values
    int cap_v, cap_c;   // staged capacities (elements) per round
    int l2_keep;        // 1: matrix stream evict_last (working set fits L2), 0: evict_first
    int check_done;
    const uint32_t* long_bits;  // rows summed by spmv_longrow_kernel (empty in this view): bit set
    const int32_t* xw;    // x-window kernels (spmv_xw.cuh): per-round window descriptors
    const uint16_t* xwo;  //   per-entry offsets into the round's staged windows
    int cap_x;            //   staged x elements per round
    const int32_t* dia;   // diagonal-warp table (spmv_dia.cuh): [chunks * 8 rounds * 8 warps][12]
    int dia_ahead;        //   chunks ahead whose leading x lines a CTA prefetches (one wave)
    const uint32_t* diaw; //   pattern-table kernel: one 32-bit word per 32-row warp
    long long ncols;      //   x length (prefetch bound)
    RedParams red;
};

// A row that spmv_longrow_kernel sums (concurrently, on a forked stream) is empty in the
// short-row view, so its staged sum is +0.0: the short-row kernel must not store it (the
// bit is only read for rows whose sum is exactly zero, and only when the matrix has long
// rows at all).  Long-row SpMVs run the short-row kernel in SPMV_PLAIN mode; their fused
// dots come from spmv_dots_kernel after the join.
__device__ __forceinline__ bool long_row_skip(const SpmvParams& P, long long row, double y) {
    return P.long_bits != nullptr && y == 0.0 && ((__ldg(P.long_bits + (row >> 5)) >> (row & 31)) & 1u);
}

template <int MODE>
__device__ __forceinline__ void spmv_epilogue(const SpmvParams& P, long long row, double y,
                                              double (&acc)[SpmvDots<MODE>::n > 0 ? SpmvDots<MODE>::n : 1]) {
    if constexpr (MODE == SPMV_CG) {
        acc[0] = __dadd_rn(acc[0], __dmul_rn(__ldg(P.x + row), y));
    } else if constexpr (MODE == SPMV_BICG_V) {
        acc[0] = __dadd_rn(acc[0], __dmul_rn(__ldg(P.aux + row), y));
    } else if constexpr (MODE == SPMV_BICG_T) {
        acc[0] = __dadd_rn(acc[0], __dmul_rn(y, y));
        acc[1] = __dadd_rn(acc[1], __dmul_rn(y, __ldg(P.aux + row)));
    }
}

// Row-sequential accumulation over entries [kb, ke) read through accessor `ld(k, c, v)`.
template <class LD>
__device__ __forceinline__ double row_sum(int kb, int ke, const double* __restrict__ x, LD ld) {
    double sum = 0.0;
    for (int k = kb; k < ke; k += 8) {
        double pr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (k + u < ke) {
                int c;
                double v;
                ld(k + u, c, v);
                pr[u] = __dmul_rn(v, __ldg(x + c));
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k + u < ke) sum = __dadd_rn(sum, pr[u]);
    }
    return sum;
}

// Direct variant (rows too long for shared-memory staging): one CTA = one chunk of 2048
// rows = 8 rounds of 256 rows; thread t owns row (round*256 + t); vals/cols via the
// read-only path.
template <int MODE>
__global__ void __launch_bounds__(kSpmvThreads, 2) spmv_direct_kernel(SpmvParams P) {
    constexpr int ND = SpmvDots<MODE>::n;
    constexpr int NA = ND > 0 ? ND : 1;
    if (P.check_done && P.red.st->done) return;
    const int t = threadIdx.x;
    if (P.p2p && (long long)blockIdx.x >= P.n_interior) {
        if (t == 0) p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
        __syncthreads();
    }
    const long long chunk = P.chunk_list ? (long long)P.chunk_list[blockIdx.x] : P.chunk0 + blockIdx.x;
    const long long base = chunk * kChunk;
    const long long rem_rounds = (P.n - base + kChunkSlots - 1) / kChunkSlots;
    const int nrounds = rem_rounds < kChunkRounds ? (int)rem_rounds : kChunkRounds;
    double acc[NA];
#pragma unroll
    for (int d = 0; d < NA; ++d) acc[d] = 0.0;
    for (int r = 0; r < nrounds; ++r) {
        const long long row = base + (long long)r * kChunkSlots + t;
        if (row < P.n) {
            double y = row_sum(__ldg(P.rp + row), __ldg(P.rp + row + 1), P.x,
                                     [&](int k, int& c, double& v) {
                                         c = __ldg(P.ci + k);
                                         v = __ldg(P.val + k);
                                     });
            if (!long_row_skip(P, row, y)) P.y[row] = y;
            spmv_epilogue<MODE>(P, row, y, acc);
        }
    }
    if constexpr (ND > 0) {
        __shared__ double sred[SpmvFin<MODE>::n * (kSpmvThreads / 32)];
        block_tree<kSpmvThreads, ND>(acc, sred);
        publish_and_finish<kSpmvThreads, ND, SpmvFin<MODE>::n>(acc, chunk, P.red, sred);
    }
}

// Staged variant: persistent, warp-specialised.  Warp 8 (one elected lane) is the
// producer: it walks this CTA's (chunk, round) sequence and streams each round's
// row_ptr / col_idx / vals segment into a kStages-deep shared-memory ring with TMA bulk
// copies (cp.async.bulk, L2 evict_first), signalling full[s] through the mbarrier
// transaction count.  Warps 0-7 consume two rounds at a time (two rows per thread, all
// x gathers of both rows in flight together), release the stages through empty[s]
// (one arrive per warp), and never wait on a CTA-wide barrier inside the loop.
constexpr int kConsumerWarps = 8;
constexpr int kWsThreads = (kConsumerWarps + 1) * 32;

struct StageLayout {
    size_t vbytes, cbytes, rbytes, stage;
    // vd: value-dictionary stream (1 byte per entry + 16-byte copy granule slack)
    __host__ __device__ StageLayout(int cap_v, int cap_c, bool vd = false) {
        vbytes = ((size_t)cap_v * (vd ? 1 : 8) + (vd ? 32 : 0) + 127) & ~size_t(127);
        cbytes = ((size_t)cap_c * 4 + 127) & ~size_t(127);
        rbytes = (kRpCopy * 4 + 127) & ~size_t(127);
        stage = vbytes + cbytes + rbytes;
    }
};

// RPT: rounds (= rows per consumer thread) in flight together; STG: ring depth;
// MINB: resident CTAs per SM requested from ptxas (register budget).
// VD (value dictionary): the value stream is one byte per entry indexing a table of the
// matrix's distinct values (<= 256, e.g. {6, -1} for the 7-point Laplacian) held in shared
// memory, so the matrix costs 5 instead of 12 bytes per entry; the products use the same
// fp64 values in the same order, so results are bit-identical to the plain kernel.
template <int MODE, int RPT, int STG, int MINB, bool EARLY, int W = 8, bool HUB = false, bool VD = false>
__global__ void __launch_bounds__(kWsThreads, MINB) spmv_ws_kernel(SpmvParams P) {
    constexpr int ND = SpmvDots<MODE>::n;
    constexpr int NA = ND > 0 ? ND : 1;
    constexpr int VALIGN = VD ? 16 : 2;  // value-stream copy granule (16 bytes)
    if (P.check_done && P.red.st->done) return;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double s_vtab[VD ? 256 : 1];
    if constexpr (VD) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_vtab[i] = P.vtab[i];
    }
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + STG;
    const StageLayout L(P.cap_v, P.cap_c, VD);
    unsigned char* stage0 = smem + 256;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int s = 0; s < STG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {  // ------------------------------- producer warp ----
        if (lane == 0) {
            const uint64_t pol = P.l2_keep ? policy_evict_last() : policy_evict_first();
            long long g = 0;
            for (long long c = blockIdx.x; c < P.nch; c += gridDim.x) {
                const long long base = (P.chunk_list ? (long long)P.chunk_list[c] : P.chunk0 + c) * kChunk;
                const long long rem = (P.n - base + kChunkSlots - 1) / kChunkSlots;
                const int nr = rem < kChunkRounds ? (int)rem : kChunkRounds;
                for (int r = 0; r < nr; ++r, ++g) {
                    const int s = (int)(g % STG);
                    mbar_wait(&empty[s], (uint32_t)(((g / STG) & 1) ^ 1));
                    const long long rs = base + (long long)r * kChunkSlots;
                    const long long re = min(rs + kChunkSlots, P.n);
                    const int nz0 = __ldg(P.rp + rs), nz1 = __ldg(P.rp + re);
                    const int a0 = nz0 & ~(VALIGN - 1), a1 = (nz1 + VALIGN - 1) & ~(VALIGN - 1);
                    const int c0 = nz0 & ~3, c1 = (nz1 + 3) & ~3;
                    // rounds larger than the ring's stage (hub rows of irregular matrices)
                    // bypass it: only row_ptr is staged, col/val are read from global
                    const bool big = HUB && (a1 - a0 > P.cap_v || c1 - c0 > P.cap_c);
                    const uint32_t vb = big ? 0u : (uint32_t)(a1 - a0) * (VD ? 1u : 8u);
                    const uint32_t cb = big ? 0u : (uint32_t)(c1 - c0) * 4u;
                    unsigned char* st = stage0 + s * L.stage;
                    reinterpret_cast<int32_t*>(st + L.vbytes + L.cbytes)[kRpCopy] = big ? 1 : 0;
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(kRpCopy * 4) + vb + cb);
                    bulk_g2s(st + L.vbytes + L.cbytes, P.rp + rs, kRpCopy * 4, &full[s], pol);
                    if constexpr (VD) {
                        if (vb) bulk_g2s(st, P.vidx + a0, vb, &full[s], pol);
                    } else {
                        if (vb) bulk_g2s(st, P.val + a0, vb, &full[s], pol);
                    }
                    if (cb) bulk_g2s(st + L.vbytes, P.ci + c0, cb, &full[s], pol);
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------------ consumers ----
    __shared__ double sred[(SpmvFin<MODE>::n > 0 ? SpmvFin<MODE>::n : 1) * kConsumerWarps];
    __shared__ int s_flag;
    static_assert(!VD || (RPT == 1 && !HUB), "value-dictionary kernels use the lean consumer");
    if constexpr (VD) {
        // Lean consumer of the value-dictionary stream: one row per thread per round, the
        // ring position kept incrementally, row segments addressed once per round, entries
        // read with immediate offsets.  Rows of <= W entries issue their x gathers straight
        // from the staged columns, keep the 1-byte value indices, and release the stage
        // while the gathers are in flight; a round with a longer row finishes from the held
        // stage (same left-to-right order).
        int s = 0;
        uint32_t ph = 0;
        bool halo_ok = P.p2p == nullptr;
        for (long long c = blockIdx.x; c < P.nch; c += gridDim.x) {
            if (!halo_ok && c >= P.n_interior) {
                if (lane == 0) p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
                __syncwarp();
                halo_ok = true;
            }
            const long long chunk = P.chunk_list ? (long long)P.chunk_list[c] : P.chunk0 + c;
            const long long base = chunk * kChunk;
            const long long rem = (P.n - base + kChunkSlots - 1) / kChunkSlots;
            const int nr = rem < kChunkRounds ? (int)rem : kChunkRounds;
            double acc[NA];
#pragma unroll
            for (int d = 0; d < NA; ++d) acc[d] = 0.0;
            for (int r = 0; r < nr; ++r) {
                mbar_wait(&full[s], ph);
                const unsigned char* A = stage0 + s * L.stage;
                const int32_t* rps = reinterpret_cast<const int32_t*>(A + L.vbytes + L.cbytes);
                const long long row = base + (long long)r * kChunkSlots + t;
                const bool live = row < P.n;
                const int o0 = rps[0];
                const int kb = live ? rps[t] : o0, ke = live ? rps[t + 1] : o0;
                const int len = ke - kb;
                const int32_t* cp = reinterpret_cast<const int32_t*>(A + L.vbytes) + (kb - (o0 & ~3));
                const uint8_t* vp = A + (kb - (o0 & ~(VALIGN - 1)));
                double y = 0.0;
                double eop = 0.0;  // the fused dot's operand (p[row] / r-hat[row] / s[row])
                if (__all_sync(0xffffffffu, len <= W)) {
                    // issue every gather straight from the staged columns; the stage is
                    // released once the gathers are in flight (their addresses consumed)
                    double xv[W];
                    uint32_t vi[(W + 3) / 4];  // value indices, 4 per register
#pragma unroll
                    for (int q = 0; q < (W + 3) / 4; ++q) vi[q] = 0u;
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (u < len) { xv[u] = __ldg(P.x + cp[u]); vi[u / 4] |= (uint32_t)vp[u] << (8 * (u % 4)); }
                    // BiCGStab epilogues stream a second vector (r-hat / s): its load joins the
                    // gathers instead of adding a dependent DRAM round trip at the end
                    if constexpr (MODE == SPMV_BICG_V || MODE == SPMV_BICG_T) eop = live ? __ldg(P.aux + row) : 0.0;
                    if constexpr (MODE == SPMV_CG) eop = live ? __ldg(P.x + row) : 0.0;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (u < len) y = __dadd_rn(y, __dmul_rn(s_vtab[(vi[u / 4] >> (8 * (u % 4))) & 0xffu], xv[u]));
                } else {
                    if constexpr (MODE == SPMV_BICG_V || MODE == SPMV_BICG_T) eop = live ? __ldg(P.aux + row) : 0.0;
                    if constexpr (MODE == SPMV_CG) eop = live ? __ldg(P.x + row) : 0.0;
                    for (int k0 = 0; k0 < len; k0 += W) {
                        double pr[W];
#pragma unroll
                        for (int u = 0; u < W; ++u)
                            if (k0 + u < len) pr[u] = __dmul_rn(s_vtab[vp[k0 + u]], __ldg(P.x + cp[k0 + u]));
#pragma unroll
                        for (int u = 0; u < W; ++u)
                            if (k0 + u < len) y = __dadd_rn(y, pr[u]);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                }
                if (live) {
                    P.y[row] = y;
                    if constexpr (MODE == SPMV_CG) {
                        acc[0] = __dadd_rn(acc[0], __dmul_rn(eop, y));
                    } else if constexpr (MODE == SPMV_BICG_V) {
                        acc[0] = __dadd_rn(acc[0], __dmul_rn(eop, y));
                    } else if constexpr (MODE == SPMV_BICG_T) {
                        acc[0] = __dadd_rn(acc[0], __dmul_rn(y, y));
                        acc[1] = __dadd_rn(acc[1], __dmul_rn(y, eop));
                    } else {
                        spmv_epilogue<MODE>(P, row, y, acc);
                    }
                }
                if (++s == STG) { s = 0; ph ^= 1u; }
            }
            if constexpr (ND > 0) {
                block_tree<kConsumerWarps * 32, ND, 1>(acc, sred);
                if (t == 0) {
#pragma unroll
                    for (int d = 0; d < ND; ++d) P.red.partials[d * P.red.nchunks + chunk] = acc[d];
                }
            }
        }
        if constexpr (ND > 0) ticket_and_finish<kConsumerWarps * 32, ND, 1, SpmvFin<MODE>::n>(P.red, sred, &s_flag);
        return;
    }
    long long g = 0;
    bool halo_ready = P.p2p == nullptr;
    for (long long c = blockIdx.x; c < P.nch; c += gridDim.x) {
        if (!halo_ready && c >= P.n_interior) {  // first boundary chunk: neighbours' pushes landed
            if (lane == 0) p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
            __syncwarp();
            halo_ready = true;
        }
        const long long chunk = P.chunk_list ? (long long)P.chunk_list[c] : P.chunk0 + c;
        const long long base = chunk * kChunk;
        const long long rem = (P.n - base + kChunkSlots - 1) / kChunkSlots;
        const int nr = rem < kChunkRounds ? (int)rem : kChunkRounds;
        double acc[NA];
#pragma unroll
        for (int d = 0; d < NA; ++d) acc[d] = 0.0;
        for (int r = 0; r < nr; r += RPT) {
            const int cnt = nr - r < RPT ? nr - r : RPT;
            int k[RPT], ke[RPT], ov[RPT], oc[RPT];
            bool big[RPT];
            const double* vs[RPT];
            const int32_t* cs[RPT];
            double y[RPT];
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                k[j] = 0; ke[j] = 0; ov[j] = 0; oc[j] = 0; y[j] = 0.0; big[j] = false;
                const int s = (int)((g + j) % STG);
                const unsigned char* A = stage0 + s * L.stage;
                vs[j] = reinterpret_cast<const double*>(A);
                cs[j] = reinterpret_cast<const int32_t*>(A + L.vbytes);
                if (j < cnt) {
                    mbar_wait(&full[s], (uint32_t)(((g + j) / STG) & 1));
                    const long long row = base + (long long)(r + j) * kChunkSlots + t;
                    const int32_t* rps = reinterpret_cast<const int32_t*>(A + L.vbytes + L.cbytes);
                    if constexpr (HUB) big[j] = rps[kRpCopy] != 0;  // oversized round: col/val from global
                    if (row < P.n) {
                        k[j] = rps[t]; ke[j] = rps[t + 1];
                        ov[j] = rps[0] & ~(VALIGN - 1); oc[j] = rps[0] & ~3;
                    }
                }
            }
            if constexpr (EARLY) {
                // Copy the first 8 entries of every row to registers and release the stages
                // before the x gathers: the ring is held only for one shared-memory read.
                int cc[RPT][W];
                double vv[RPT][W];
                bool fits = true;
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    if (!HUB || !big[j]) {
#pragma unroll
                        for (int u = 0; u < W; ++u)
                            if (k[j] + u < ke[j]) { cc[j][u] = cs[j][k[j] + u - oc[j]]; vv[j][u] = vs[j][k[j] + u - ov[j]]; }
                    } else {
#pragma unroll
                        for (int u = 0; u < W; ++u)
                            if (k[j] + u < ke[j]) { cc[j][u] = __ldg(P.ci + k[j] + u); vv[j][u] = __ldg(P.val + k[j] + u); }
                    }
                    fits &= ke[j] - k[j] <= W;
                }
                fits = __all_sync(0xffffffffu, fits);
                if (fits) {
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int j = 0; j < RPT; ++j)
                            if (j < cnt) mbar_arrive(&empty[(g + j) % STG]);
                    }
                }
                double pr[RPT][W];
#pragma unroll
                for (int j = 0; j < RPT; ++j)
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (k[j] + u < ke[j]) pr[j][u] = __dmul_rn(vv[j][u], __ldg(P.x + cc[j][u]));
#pragma unroll
                for (int j = 0; j < RPT; ++j)
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (k[j] + u < ke[j]) y[j] = __dadd_rn(y[j], pr[j][u]);
                if (!fits) {  // long rows: finish from the (still held) stages, then release
                    bool more = false;
#pragma unroll
                    for (int j = 0; j < RPT; ++j) { k[j] += W; more |= k[j] < ke[j]; }
                    while (more) {
#pragma unroll
                        for (int j = 0; j < RPT; ++j)
#pragma unroll
                            for (int u = 0; u < W; ++u)
                                if (k[j] + u < ke[j]) {
                                    const int kk = k[j] + u;
                                    const double vvv = (HUB && big[j]) ? __ldg(P.val + kk) : vs[j][kk - ov[j]];
                                    const int ccc = (HUB && big[j]) ? __ldg(P.ci + kk) : cs[j][kk - oc[j]];
                                    pr[j][u] = __dmul_rn(vvv, __ldg(P.x + ccc));
                                }
#pragma unroll
                        for (int j = 0; j < RPT; ++j)
#pragma unroll
                            for (int u = 0; u < W; ++u)
                                if (k[j] + u < ke[j]) y[j] = __dadd_rn(y[j], pr[j][u]);
                        more = false;
#pragma unroll
                        for (int j = 0; j < RPT; ++j) { k[j] += W; more |= k[j] < ke[j]; }
                    }
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int j = 0; j < RPT; ++j)
                            if (j < cnt) mbar_arrive(&empty[(g + j) % STG]);
                    }
                }
            } else {
            bool more = true;
            while (more) {
                double pr[RPT][8];
#pragma unroll
                for (int j = 0; j < RPT; ++j)
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (k[j] + u < ke[j]) {
                            const int kk = k[j] + u;
                            const double vvv = (HUB && big[j]) ? __ldg(P.val + kk) : vs[j][kk - ov[j]];
                            const int ccc = (HUB && big[j]) ? __ldg(P.ci + kk) : cs[j][kk - oc[j]];
                            pr[j][u] = __dmul_rn(vvv, __ldg(P.x + ccc));
                        }
#pragma unroll
                for (int j = 0; j < RPT; ++j)
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (k[j] + u < ke[j]) y[j] = __dadd_rn(y[j], pr[j][u]);
                more = false;
#pragma unroll
                for (int j = 0; j < RPT; ++j) { k[j] += 8; more |= k[j] < ke[j]; }
            }
            __syncwarp();
            if (lane == 0) {  // stage contents fully read by this warp
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    if (j < cnt) mbar_arrive(&empty[(g + j) % STG]);
            }
            }
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const long long row = base + (long long)(r + j) * kChunkSlots + t;
                if (j < cnt && row < P.n) {
                    if (!long_row_skip(P, row, y[j])) P.y[row] = y[j];
                    spmv_epilogue<MODE>(P, row, y[j], acc);
                }
            }
            g += cnt;
        }
        if constexpr (ND > 0) {
            block_tree<kConsumerWarps * 32, ND, 1>(acc, sred);
            if (t == 0) {
#pragma unroll
                for (int d = 0; d < ND; ++d) P.red.partials[d * P.red.nchunks + chunk] = acc[d];
            }
        }
    }
    if constexpr (ND > 0) ticket_and_finish<kConsumerWarps * 32, ND, 1, SpmvFin<MODE>::n>(P.red, sred, &s_flag);
}

// Warp-pipelined staged variant (persistent, no producer/consumer hand-off).  Each warp
// owns slots [32w, 32w+32) of every round, so it streams its own 32-row segments
// (row_ptr, col_idx, vals) through a private D-deep shared-memory ring with TMA bulk
// copies; lane 0 re-arms a stage right after the warp has read it.  Only 3 KB of shared
// memory is held per segment being consumed, so almost all of it is in flight.  Segment
// boundaries (row_ptr at the segment ends) are prefetched one issue ahead so the
// issuing lane never stalls on a dependent global load.
struct WarpStage {
    int vbytes, cbytes, stage;
    __host__ __device__ WarpStage(int cap_v, int cap_c) {
        vbytes = (cap_v * 8 + 127) & ~127;
        cbytes = (cap_c * 4 + 127) & ~127;
        stage = vbytes + cbytes + 256;  // + row_ptr[36]
    }
};
constexpr int kWarpRp = 36;

template <int MODE, int D, int MINB>
__global__ void __launch_bounds__(kSpmvThreads, MINB) spmv_wp_kernel(SpmvParams P) {
    constexpr int ND = SpmvDots<MODE>::n;
    constexpr int NA = ND > 0 ? ND : 1;
    constexpr int NW = kSpmvThreads / 32;
    if (P.check_done && P.red.st->done) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const WarpStage L(P.cap_v, P.cap_c);
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + w * D;
    unsigned char* ring = smem + 1024 + (size_t)w * D * L.stage;
    __shared__ double sred[(SpmvFin<MODE>::n > 0 ? SpmvFin<MODE>::n : 1) * NW];
    __shared__ int s_flag;
    if (lane == 0) {
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // issue iterator over this CTA's (chunk, round) sequence
    long long ic = blockIdx.x;
    int ir = 0;
    auto chunk_of = [&](long long c) { return P.chunk_list ? (long long)P.chunk_list[c] : P.chunk0 + c; };
    auto nrounds = [&](long long c) {
        const long long base = chunk_of(c) * kChunk;
        const long long rem = (P.n - base + kChunkSlots - 1) / kChunkSlots;
        return rem < kChunkRounds ? (int)rem : kChunkRounds;
    };
    // segment row range for (c, r) of this warp
    auto seg = [&](long long c, int r, long long& rs, long long& re) {
        rs = chunk_of(c) * kChunk + (long long)r * kChunkSlots + 32 * w;
        re = min(rs + 32, P.n);
    };
    uint64_t pol = 0;
    int nz0n = 0, nz1n = 0;  // prefetched boundaries of the next segment to issue
    bool have_next = ic < P.nch;
    if (lane == 0) {
        pol = policy_evict_first();
        if (have_next) {
            long long rs, re;
            seg(ic, ir, rs, re);
            if (rs < re) { nz0n = __ldg(P.rp + rs); nz1n = __ldg(P.rp + re); }
        }
    }
    long long issued = 0;
    auto issue_next = [&]() {  // lane 0 only
        if (!have_next) return;
        const int s = (int)(issued % D);
        long long rs, re;
        seg(ic, ir, rs, re);
        unsigned char* st = ring + s * L.stage;
        if (rs < re) {
            const int nz0 = nz0n, nz1 = nz1n;
            const int a0 = nz0 & ~1, a1 = (nz1 + 1) & ~1;
            const int c0 = nz0 & ~3, c1 = (nz1 + 3) & ~3;
            const uint32_t vb = (uint32_t)(a1 - a0) * 8u, cb = (uint32_t)(c1 - c0) * 4u;
            mbar_arrive_expect_tx(&bars[s], (uint32_t)(kWarpRp * 4) + vb + cb);
            bulk_g2s(st + L.vbytes + L.cbytes, P.rp + rs, kWarpRp * 4, &bars[s], pol);
            if (vb) bulk_g2s(st, P.val + a0, vb, &bars[s], pol);
            if (cb) bulk_g2s(st + L.vbytes, P.ci + c0, cb, &bars[s], pol);
        } else {
            mbar_arrive_expect_tx(&bars[s], 0);  // empty segment (tail): complete the phase
        }
        ++issued;
        if (++ir >= nrounds(ic)) { ir = 0; ic += gridDim.x; }
        have_next = ic < P.nch;
        if (have_next) {  // prefetch the following segment's boundaries
            seg(ic, ir, rs, re);
            if (rs < re) { nz0n = __ldg(P.rp + rs); nz1n = __ldg(P.rp + re); }
        }
    };
    if (lane == 0)
        for (int s = 0; s < D; ++s) issue_next();

    long long g = 0;
    for (long long c = blockIdx.x; c < P.nch; c += gridDim.x) {
        const long long chunk = chunk_of(c);
        const long long base = chunk * kChunk;
        const int nr = nrounds(c);
        double acc[NA];
#pragma unroll
        for (int d = 0; d < NA; ++d) acc[d] = 0.0;
        for (int r = 0; r < nr; ++r, ++g) {
            const int s = (int)(g % D);
            mbar_wait(&bars[s], (uint32_t)((g / D) & 1));
            const unsigned char* st = ring + s * L.stage;
            const int32_t* rps = reinterpret_cast<const int32_t*>(st + L.vbytes + L.cbytes);
            const double* vs = reinterpret_cast<const double*>(st);
            const int32_t* cs = reinterpret_cast<const int32_t*>(st + L.vbytes);
            const long long row = base + (long long)r * kChunkSlots + t;
            double y = 0.0;
            if (row < P.n) {
                const int ov = rps[0] & ~1, oc = rps[0] & ~3;
                y = row_sum(rps[lane], rps[lane + 1], P.x, [&](int k, int& cc, double& v) {
                    cc = cs[k - oc];
                    v = vs[k - ov];
                });
            }
            __syncwarp();
            if (lane == 0) {
                fence_proxy_async_smem();
                issue_next();
            }
            if (row < P.n) {
                if (!long_row_skip(P, row, y)) P.y[row] = y;
                spmv_epilogue<MODE>(P, row, y, acc);
            }
        }
        if constexpr (ND > 0) {
            block_tree<kSpmvThreads, ND, 1>(acc, sred);
            if (t == 0) {
#pragma unroll
                for (int d = 0; d < ND; ++d) P.red.partials[d * P.red.nchunks + chunk] = acc[d];
            }
        }
    }
    if constexpr (ND > 0) ticket_and_finish<kSpmvThreads, ND, 1, SpmvFin<MODE>::n>(P.red, sred, &s_flag);
}

// -------------------------------------------------------------- vector kernels -------
// Thread t of a 128-thread CTA owns slots 2t and 2t+1 of each 256-element round (one
// double2), rounds 0..7 of the CTA's 2048-element chunk.  Inputs of 4 rounds are loaded
// before any arithmetic (ILP); all operations are separate IEEE mul/add/sub in the
// oracle's order (no FMA).
struct VecParams {
    long long n;
    const double* d;  // Jacobi inverse diagonal; nullptr: uniform diagonal d_uni (not streamed)
    double d_uni;
    double *x, *r, *p, *q;
    double* p2;  // CG deferred x update: the other direction buffer (previous / next p)
    double *rh, *ph, *v, *s, *sh, *tt;
    const double* b;
    int check_done;
    RedParams red;
    // fused peer collectives (distributed CG): consume reduction point `consume_point`
    // (scalar op consume_scalar over consume_k totals) at entry; CG_U2 also pushes the halo
    const P2PCtx* p2p;
    int consume_point, consume_scalar, consume_k;
    int resident;  // host: launch a resident (persistent) grid
};

__device__ __forceinline__ double2 ld2(const double* p, long long i, long long n) {
    if (i + 1 < n) return *reinterpret_cast<const double2*>(p + i);
    double2 z;
    z.x = i < n ? p[i] : 0.0;
    z.y = 0.0;
    return z;
}
__device__ __forceinline__ void st2(double* p, long long i, long long n, double2 v) {
    if (i + 1 < n) *reinterpret_cast<double2*>(p + i) = v;
    else if (i < n) p[i] = v.x;
}
// Jacobi inverse diagonal pair: streamed, or the uniform value of a constant diagonal
// (Poisson / constant-coefficient stencils, and the identity when unpreconditioned).
__device__ __forceinline__ double2 ldd(const double* d, double d_uni, long long i, long long n) {
    return d ? ld2(d, i, n) : make_double2(d_uni, d_uni);
}
__device__ __forceinline__ double lane(const double2& v, int e) { return e ? v.y : v.x; }
__device__ __forceinline__ void set_lane(double2& v, int e, double x) { if (e) v.y = x; else v.x = x; }

// ------------------------------------------------------------------ long rows ------
// Rows longer than the thread-per-row kernels handle well (power-law hubs; threshold from
// the row-length histogram, DevCsr::create) get one warp each.  Lanes load col/val
// coalesced, gather x and form the products in parallel (__dmul_rn); lane 0 then adds them
// strictly left to right from 0.0 — the reference's per-row order (sparse.cpp:144-152),
// bit-identical.  That dependent add chain is the floor of a bit-exact row sum, so the
// loads are software-pipelined around it: while lane 0 runs the chain of batch b, the x
// gathers of batch b+1 and the col/val loads of batch b+2 are in flight.  The list is
// sorted longest first and walked grid-stride, so the longest chains start at once.
// The staged SpMV runs concurrently (forked stream) on the short-row view, where the long
// rows are empty and not stored (long_row_skip); after the join spmv_dots_kernel forms the
// fused dots in canonical order.  So the SpMV costs max(longest chain, short rows) + one
// 16-24 B/row dot pass instead of their sum.
// one warp per CTA: the long-row kernel runs beside the persistent short-row kernel, so its
// CTAs must fit in the register / shared-memory slack that kernel leaves on each SM (an
// 8-warp CTA holding a hub row kept a short-row CTA off its SM for the whole hub chain)
constexpr int kLongWarps = 1;
constexpr int kLongU = 4;                    // entries per lane per batch
constexpr int kLongBatch = 32 * kLongU;      // 128 entries per batch

struct LongRowParams {
    const int32_t* rp;
    const int32_t* ci;
    const double* val;
    const double* x;
    double* y;
    const int32_t* rows;  // long rows, longest first
    long long nlong;
    const KState* st;
    int check_done;
};

static __global__ void __launch_bounds__(kLongWarps * 32) spmv_longrow_kernel(LongRowParams P) {
    if (P.check_done && P.st->done) return;
    __shared__ __align__(16) double prod[kLongWarps][kLongBatch];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (long long li = (long long)blockIdx.x * kLongWarps + w; li < P.nlong; li += (long long)gridDim.x * kLongWarps) {
        const int row = __ldg(P.rows + li);
        const int kb = __ldg(P.rp + row), ke = __ldg(P.rp + row + 1);
        int cn[kLongU];
        double vn[kLongU], vc[kLongU], xc[kLongU];
        auto load_cv = [&](int k0) {
#pragma unroll
            for (int u = 0; u < kLongU; ++u) {
                const int k = k0 + u * 32 + lane;
                cn[u] = k < ke ? __ldcs(P.ci + k) : -1;
                vn[u] = k < ke ? __ldcs(P.val + k) : 0.0;
            }
        };
        auto gather = [&]() {
#pragma unroll
            for (int u = 0; u < kLongU; ++u) { xc[u] = cn[u] >= 0 ? __ldg(P.x + cn[u]) : 0.0; vc[u] = vn[u]; }
        };
        load_cv(kb);
        gather();
        load_cv(kb + kLongBatch);
        double sum = 0.0;
        for (int k0 = kb; k0 < ke; k0 += kLongBatch) {
#pragma unroll
            for (int u = 0; u < kLongU; ++u) prod[w][u * 32 + lane] = __dmul_rn(vc[u], xc[u]);
            gather();                         // batch b+1: its columns arrived meanwhile
            load_cv(k0 + 2 * kLongBatch);     // batch b+2
            __syncwarp();
            if (lane == 0) {
                const int cnt = min(kLongBatch, ke - k0);
                const double2* p2 = reinterpret_cast<const double2*>(prod[w]);
                if (cnt == kLongBatch) {
#pragma unroll 8
                    for (int j = 0; j < kLongBatch / 2; ++j) {
                        const double2 q = p2[j];
                        sum = __dadd_rn(sum, q.x);
                        sum = __dadd_rn(sum, q.y);
                    }
                } else {
                    for (int j = 0; j < cnt; ++j) sum = __dadd_rn(sum, prod[w][j]);
                }
            }
            __syncwarp();
        }
        if (lane == 0) P.y[row] = sum;
    }
}

// Fused dots of an SpMV whose rows were summed by two concurrent kernels (long rows warp-
// per-row, the rest staged): one CTA per 2048-row chunk re-reads y (and the dot operand)
// and reduces them in the canonical chunk shape (slot t, rounds 0..7, then the block tree)
// — the same bits as the staged kernels' fused epilogue; the last CTA runs the scalar step.
template <int MODE>
static __global__ void __launch_bounds__(kSpmvThreads) spmv_dots_kernel(SpmvParams P) {
    constexpr int ND = SpmvDots<MODE>::n;
    if (P.check_done && P.red.st->done) return;
    const int t = threadIdx.x;
    const long long chunk = blockIdx.x;
    const long long base = chunk * kChunk;
    double acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = 0.0;
#pragma unroll
    for (int r = 0; r < kChunkRounds; ++r) {
        const long long row = base + (long long)r * kChunkSlots + t;
        if (row < P.n) spmv_epilogue<MODE>(P, row, __ldg(P.y + row), acc);
    }
    __shared__ double sred[SpmvFin<MODE>::n * (kSpmvThreads / 32)];
    block_tree<kSpmvThreads, ND>(acc, sred);
    publish_and_finish<kSpmvThreads, ND, SpmvFin<MODE>::n>(acc, chunk, P.red, sred);
}

// short-row view values after set_values: copy every row that is not long
static __global__ void short_view_values_kernel(const int32_t* rp, const double* val, const int32_t* s_rp,
                                         double* s_val, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = s_rp[i], e = s_rp[i + 1], o = rp[i];
    for (int k = b; k < e; ++k) s_val[k] = val[o + (k - b)];
}

enum VecOp : int { V_CG_INIT, V_CG_U1, V_CG_U2, V_BI_INIT, V_BI_U1, V_BI_U2, V_BI_U3, V_CG_U2E, V_CG_U2O };
// Deferred x update (single GPU CG): two p buffers alternate.  Even iterations (U2E) only
// form the next direction p' = z + beta p into the other buffer — x keeps lagging alpha p;
// odd iterations (U2O) apply both steps, x = (x + alpha_prev p_prev) + alpha p, then form p'.
// The same two roundings in the same order as updating x every iteration (bit-identical),
// with x streamed every other iteration: 36 instead of 40 bytes per row per iteration.
// CG iteration split used by the solver: U1 = r -= a q, z = d r, {r.z, r.r} (reads r q d);
// U2 = x += a p, then p = z + b p unless the solve just terminated (reads x p r d).  p is
// streamed once per iteration instead of twice (100 n instead of 108 n bytes); the x update
// is the oracle's x + a p, only applied one kernel later.
template <int OP> struct VecTraits;
template <> struct VecTraits<V_CG_INIT> { static constexpr int nin = 3, ndot = 3; };  // b q d
template <> struct VecTraits<V_CG_U1>   { static constexpr int nin = 3, ndot = 2; };  // r q d
template <> struct VecTraits<V_CG_U2>   { static constexpr int nin = 4, ndot = 0; };  // x p r d
template <> struct VecTraits<V_CG_U2E>  { static constexpr int nin = 4, ndot = 0; };  // p r d (x only at the end)
template <> struct VecTraits<V_CG_U2O>  { static constexpr int nin = 5, ndot = 0; };  // x p_prev p r d
template <> struct VecTraits<V_BI_INIT> { static constexpr int nin = 2, ndot = 3; };  // b v
template <> struct VecTraits<V_BI_U1>   { static constexpr int nin = 4, ndot = 0; };  // r p v d
template <> struct VecTraits<V_BI_U2>   { static constexpr int nin = 3, ndot = 1; };  // r v d; s.s
// kernels whose chunk partials are reduced by a LATER kernel (no ticket, no finish): U2's
// s.s partials land in row 2 of the t-SpMV's reduction point
template <int OP> struct VecPublishOnly { static constexpr int row = -1; };
template <> struct VecPublishOnly<V_BI_U2> { static constexpr int row = 2; };
template <> struct VecTraits<V_BI_U3>   { static constexpr int nin = 6, ndot = 2; };  // x ph s sh t rh

struct VecScalars {
    double alpha, beta, omega, alpha_prev;
    int first, half, live, lag, pend;
};

template <int OP>
__device__ __forceinline__ void vec_load(const VecParams& P, const VecScalars& S, long long i,
                                         double2 (&in)[VecTraits<OP>::nin]) {
    const long long n = P.n;
    if constexpr (OP == V_CG_U2E) {  // x only when the solve ends here (apply alpha p at once)
        in[0] = ld2(P.p, i, n); in[1] = ld2(P.r, i, n); in[2] = ldd(P.d, P.d_uni, i, n);
        in[3] = S.live ? make_double2(0.0, 0.0) : ld2(P.x, i, n);
    }
    if constexpr (OP == V_CG_U2O) {
        in[0] = ld2(P.x, i, n); in[1] = ld2(P.p2, i, n); in[2] = ld2(P.p, i, n); in[3] = ld2(P.r, i, n);
        in[4] = ldd(P.d, P.d_uni, i, n);
    }
    if constexpr (OP == V_CG_INIT) { in[0] = ld2(P.b, i, n); in[1] = ld2(P.q, i, n); in[2] = ldd(P.d, P.d_uni, i, n); }
    if constexpr (OP == V_CG_U1) { in[0] = ld2(P.r, i, n); in[1] = ld2(P.q, i, n); in[2] = ldd(P.d, P.d_uni, i, n); }
    if constexpr (OP == V_CG_U2) {
        in[0] = ld2(P.x, i, n); in[1] = ld2(P.p, i, n); in[2] = ld2(P.r, i, n); in[3] = ldd(P.d, P.d_uni, i, n);
    }
    if constexpr (OP == V_BI_INIT) { in[0] = ld2(P.b, i, n); in[1] = ld2(P.v, i, n); }
    if constexpr (OP == V_BI_U1) {
        in[0] = ld2(P.r, i, n); in[1] = ld2(P.p, i, n); in[2] = ld2(P.v, i, n); in[3] = ldd(P.d, P.d_uni, i, n);
    }
    if constexpr (OP == V_BI_U2) { in[0] = ld2(P.r, i, n); in[1] = ld2(P.v, i, n); in[2] = ldd(P.d, P.d_uni, i, n); }
    if constexpr (OP == V_BI_U3) {
        in[0] = ld2(P.x, i, n); in[1] = ld2(P.ph, i, n); in[2] = ld2(P.s, i, n);
        in[3] = ld2(P.sh, i, n); in[4] = ld2(P.tt, i, n); in[5] = ld2(P.rh, i, n);
    }
}

// Computes both lanes of the pair at i, stores outputs, returns per-lane dot products.
template <int OP>
__device__ __forceinline__ void vec_compute(const VecParams& P, const VecScalars& S, long long i,
                                            const double2 (&in)[VecTraits<OP>::nin],
                                            double (&pr)[VecTraits<OP>::ndot > 0 ? VecTraits<OP>::ndot : 1][2]) {
    const long long n = P.n;
    double2 o0 = make_double2(0.0, 0.0), o1 = make_double2(0.0, 0.0);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        if constexpr (OP == V_CG_INIT) {  // r = b - q; z = d r; p = z; {r.z, r.r, b.b}
            const double b = lane(in[0], e);
            const double r = __dsub_rn(b, lane(in[1], e));
            const double z = __dmul_rn(lane(in[2], e), r);
            set_lane(o0, e, r); set_lane(o1, e, z);
            pr[0][e] = __dmul_rn(r, z); pr[1][e] = __dmul_rn(r, r); pr[2][e] = __dmul_rn(b, b);
        }
        if constexpr (OP == V_CG_U1) {  // r -= a q; z = d r; {r.z, r.r}
            const double rn = __dsub_rn(lane(in[0], e), __dmul_rn(S.alpha, lane(in[1], e)));
            const double z = __dmul_rn(lane(in[2], e), rn);
            set_lane(o1, e, rn);
            pr[0][e] = __dmul_rn(rn, z); pr[1][e] = __dmul_rn(rn, rn);
        }
        if constexpr (OP == V_CG_U2) {  // x += a p (old p); then p = z + beta p, z = d r
            set_lane(o0, e, __dadd_rn(lane(in[0], e), __dmul_rn(S.alpha, lane(in[1], e))));
            const double z = __dmul_rn(lane(in[3], e), lane(in[2], e));
            set_lane(o1, e, __dadd_rn(z, __dmul_rn(S.beta, lane(in[1], e))));
        }
        if constexpr (OP == V_CG_U2E) {  // p' = z + beta p (x lags alpha p), or x += alpha p at the end
            if (S.live) {
                const double z = __dmul_rn(lane(in[2], e), lane(in[1], e));
                set_lane(o1, e, __dadd_rn(z, __dmul_rn(S.beta, lane(in[0], e))));
            } else {
                set_lane(o0, e, __dadd_rn(lane(in[3], e), __dmul_rn(S.alpha, lane(in[0], e))));
            }
        }
        if constexpr (OP == V_CG_U2O) {  // x = (x + a_prev p_prev) + a p; p' = z + beta p
            double xn = lane(in[0], e);
            if (S.lag) xn = __dadd_rn(xn, __dmul_rn(S.alpha_prev, lane(in[1], e)));
            if (S.pend) xn = __dadd_rn(xn, __dmul_rn(S.alpha, lane(in[2], e)));
            set_lane(o0, e, xn);
            const double z = __dmul_rn(lane(in[4], e), lane(in[3], e));
            set_lane(o1, e, __dadd_rn(z, __dmul_rn(S.beta, lane(in[2], e))));
        }
        if constexpr (OP == V_BI_INIT) {  // r = b - v; rhat = r; {rh.r, r.r, b.b}
            const double b = lane(in[0], e);
            const double r = __dsub_rn(b, lane(in[1], e));
            set_lane(o0, e, r);
            pr[0][e] = __dmul_rn(r, r); pr[1][e] = __dmul_rn(r, r); pr[2][e] = __dmul_rn(b, b);
        }
        if constexpr (OP == V_BI_U1) {  // p = r + beta (p - omega v)  (p = r at k = 0); ph = d p
            const double r = lane(in[0], e);
            const double p = S.first ? r
                : __dadd_rn(r, __dmul_rn(S.beta, __dsub_rn(lane(in[1], e), __dmul_rn(S.omega, lane(in[2], e)))));
            set_lane(o0, e, p); set_lane(o1, e, __dmul_rn(lane(in[3], e), p));
        }
        if constexpr (OP == V_BI_U2) {  // s = r - alpha v; sh = d s
            const double s = __dsub_rn(lane(in[0], e), __dmul_rn(S.alpha, lane(in[1], e)));
            set_lane(o0, e, s); set_lane(o1, e, __dmul_rn(lane(in[2], e), s));
            pr[0][e] = __dmul_rn(s, s);
        }
        if constexpr (OP == V_BI_U3) {
            if (S.half) {  // x += alpha ph; r = s
                set_lane(o0, e, __dadd_rn(lane(in[0], e), __dmul_rn(S.alpha, lane(in[1], e))));
                set_lane(o1, e, lane(in[2], e));
                pr[0][e] = 0.0; pr[1][e] = 0.0;
            } else {       // x = (x + alpha ph) + omega sh; r = s - omega t; {rh.r, r.r}
                const double xn = __dadd_rn(__dadd_rn(lane(in[0], e), __dmul_rn(S.alpha, lane(in[1], e))),
                                            __dmul_rn(S.omega, lane(in[3], e)));
                const double rn = __dsub_rn(lane(in[2], e), __dmul_rn(S.omega, lane(in[4], e)));
                set_lane(o0, e, xn); set_lane(o1, e, rn);
                pr[0][e] = __dmul_rn(lane(in[5], e), rn); pr[1][e] = __dmul_rn(rn, rn);
            }
        }
    }
    if constexpr (OP == V_CG_INIT) { st2(P.r, i, n, o0); st2(P.p, i, n, o1); }
    if constexpr (OP == V_CG_U1) { st2(P.r, i, n, o1); }
    if constexpr (OP == V_CG_U2) {
        st2(P.x, i, n, o0);
        if (S.live) st2(P.p, i, n, o1);  // the solve continues: new direction
    }
    if constexpr (OP == V_CG_U2E) {
        if (S.live) st2(P.p2, i, n, o1);
        else st2(P.x, i, n, o0);
    }
    if constexpr (OP == V_CG_U2O) {
        st2(P.x, i, n, o0);
        if (S.live) st2(P.p2, i, n, o1);  // overwrites p_prev, read above by this thread
    }
    if constexpr (OP == V_BI_INIT) { st2(P.r, i, n, o0); st2(P.rh, i, n, o0); }
    if constexpr (OP == V_BI_U1) { st2(P.p, i, n, o0); st2(P.ph, i, n, o1); }
    if constexpr (OP == V_BI_U2) { st2(P.s, i, n, o0); st2(P.sh, i, n, o1); }
    if constexpr (OP == V_BI_U3) { st2(P.x, i, n, o0); st2(P.r, i, n, o1); }
}

template <int OP, int G = 4, bool PERSIST = false>
__global__ void __launch_bounds__(kVecThreads) vec_kernel(VecParams P) {
    constexpr int NIN = VecTraits<OP>::nin;
    constexpr int ND = VecTraits<OP>::ndot;
    constexpr int NA = ND > 0 ? ND : 1;
    KState* st = P.red.st;
    if constexpr (OP == V_CG_U2E) {
        if (!st->pending_x) return;
    } else if constexpr (OP == V_CG_U2O) {
        if (!st->pending_x && !st->x_lag) return;  // also after a breakdown: the lagging step
    } else if constexpr (OP == V_CG_U2) {
        if (!st->pending_x) return;  // runs once more after termination to apply x += a p
    } else {
        if (P.check_done && st->done) return;
    }
    __shared__ KState s_loc;  // fused peer collectives: this CTA's copy of the scalar state
    const KState* sc = st;
    bool skip = false;
    constexpr bool CONSUMES = OP == V_CG_U1 || OP == V_CG_U2 || OP == V_BI_U1 || OP == V_BI_U2 || OP == V_BI_U3;
    if constexpr (CONSUMES) {
        if (P.p2p) {
            if (threadIdx.x == 0) {
                s_loc = *st;
                // BiCGStab U1 consumes the previous iteration's U3 totals (flagged in
                // pending_x by that U3; there are none before the first iteration)
                if (OP != V_BI_U1 || s_loc.pending_x) {
                    p2p_consume(P.p2p, &s_loc, P.consume_point, P.consume_k, P.consume_scalar);
                    if constexpr (OP == V_BI_U1) s_loc.pending_x = 0;
                }
                if constexpr (OP == V_BI_U3) s_loc.pending_x = !s_loc.done;  // its totals follow
            }
            __syncthreads();
            sc = &s_loc;
            if constexpr (OP != V_CG_U2) skip = s_loc.done != 0;  // breakdown / convergence decided here
        }
    }
    VecScalars S;
    if constexpr (OP == V_CG_U1 || OP == V_BI_U2) S.alpha = sc->alpha;
    if constexpr (OP == V_CG_U2) { S.alpha = sc->alpha; S.beta = sc->beta; S.live = !sc->done; }
    if constexpr (OP == V_CG_U2E) { S.alpha = sc->alpha; S.beta = sc->beta; S.live = !sc->done; }
    if constexpr (OP == V_CG_U2O) {
        S.alpha = sc->alpha; S.beta = sc->beta; S.alpha_prev = sc->alpha_prev; S.live = !sc->done;
        S.lag = sc->x_lag; S.pend = sc->pending_x;
    }
    if constexpr (OP == V_BI_U1) { S.beta = sc->beta; S.omega = sc->omega; S.first = sc->k == 0; }
    if constexpr (OP == V_BI_U3) { S.alpha = sc->alpha; S.omega = sc->omega; S.half = sc->halfstep; }
    const int t = threadIdx.x;
    __shared__ double sred[NA * (kVecThreads / 32)];
    __shared__ int s_flag;
    const long long nchunks = P.red.nchunks;
    // PERSIST: a resident grid loops over chunks (one ticket per CTA); else one chunk per CTA
    for (long long chunk = blockIdx.x; chunk < nchunks; chunk += PERSIST ? gridDim.x : nchunks) {
    const long long base = chunk * kChunk;
    double acc[NA][2];
#pragma unroll
    for (int d = 0; d < NA; ++d) acc[d][0] = acc[d][1] = 0.0;
#pragma unroll
    for (int g = 0; g < kChunkRounds; g += G) {
        double2 in[G][NIN];
#pragma unroll
        for (int u = 0; u < G; ++u) vec_load<OP>(P, S, base + (long long)(g + u) * kChunkSlots + 2 * t, in[u]);
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const long long i = base + (long long)(g + u) * kChunkSlots + 2 * t;
            if (i >= P.n || skip) continue;
            double pr[NA][2];
            vec_compute<OP>(P, S, i, in[u], pr);
            if constexpr (ND > 0) {
#pragma unroll
                for (int d = 0; d < ND; ++d) {
                    acc[d][0] = __dadd_rn(acc[d][0], pr[d][0]);
                    if (i + 1 < P.n) acc[d][1] = __dadd_rn(acc[d][1], pr[d][1]);
                }
            }
        }
    }
    if constexpr (OP == V_CG_U2 || OP == V_BI_U1 || OP == V_BI_U2) {
        // fused halo push: this chunk's boundary values of the next SpMV input (p; p-hat;
        // s-hat) go straight into the neighbours' halo slots (written above by this CTA,
        // visible after the barrier)
        bool push = P.p2p != nullptr;
        if constexpr (OP == V_CG_U2) push = push && S.live;
        else push = push && !skip;
        if (push) {
            __syncthreads();
            if constexpr (OP == V_CG_U2) p2p_push_halo_chunk(P.p2p, chunk, P.p, P.p2p->peer_vec);
            if constexpr (OP == V_BI_U1) p2p_push_halo_chunk(P.p2p, chunk, P.ph, P.p2p->peer_vec);
            if constexpr (OP == V_BI_U2) p2p_push_halo_chunk(P.p2p, chunk, P.sh, P.p2p->peer_vec2);
        }
    }
    if constexpr (ND > 0) {
        double v[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) v[d] = __dadd_rn(acc[d][0], acc[d][1]);  // slot pair
        block_tree<kVecThreads, ND>(v, sred);
        if constexpr (VecPublishOnly<OP>::row >= 0) {
            if (t == 0) P.red.partials[VecPublishOnly<OP>::row * P.red.nchunks + chunk] = v[0];
        } else if constexpr (PERSIST) {
            if (t == 0) {
#pragma unroll
                for (int d = 0; d < ND; ++d) P.red.partials[d * P.red.nchunks + chunk] = v[d];
            }
        } else {
            RedParams R = P.red;
            if (P.p2p) { R.p2p = P.p2p; R.s_loc = &s_loc; }
            publish_and_finish<kVecThreads, ND>(v, chunk, R, sred);
        }
    }
    }  // chunk loop
    if constexpr (ND > 0 && PERSIST && VecPublishOnly<OP>::row < 0) {
        RedParams R = P.red;
        if (P.p2p) { R.p2p = P.p2p; R.s_loc = &s_loc; }
        ticket_and_finish<kVecThreads, ND, 0>(R, sred, &s_flag);
    } else if constexpr (OP == V_BI_U1 || OP == V_BI_U2) {
        // fused peer collectives: the last CTA publishes the consumed scalar state and
        // raises this vector's halo flag once every CTA's peer stores are ordered before it
        if (P.p2p) {
            __syncthreads();
            if (t == 0) {
                __threadfence_system();
                if (atomicAdd(P.red.ticket, 1u) == P.red.expected - 1) {
                    __threadfence_system();
                    *st = s_loc;
                    if (!s_loc.done) p2p_raise_halo(P.p2p, st, OP == V_BI_U1 ? 0 : 1);
                    *P.red.ticket = 0u;
                    __threadfence();
                }
            }
        }
    } else if constexpr (OP == V_CG_U2) {
        // the last CTA clears pending_x once every CTA has read it; with fused peer
        // collectives it also publishes this rank's scalar step and raises the halo flags
        __syncthreads();
        if (t == 0) {
            if (P.p2p) __threadfence_system();  // order this CTA's peer halo stores first
            else __threadfence();
            if (atomicAdd(P.red.ticket, 1u) == P.red.expected - 1) {
                if (P.p2p) {
                    __threadfence_system();
                    *st = s_loc;
                    st->pending_x = 0;
                    if (S.live) p2p_raise_halo(P.p2p, st, 0);
                } else {
                    st->pending_x = 0;
                }
                *P.red.ticket = 0u;
                __threadfence();
            }
        }
    } else if constexpr (OP == V_CG_U2E || OP == V_CG_U2O) {
        // the last CTA (every CTA has read the scalars) updates the deferral state: after an
        // even step that continues, x lags alpha p; after an odd step x is complete
        __syncthreads();
        if (t == 0) {
            __threadfence();
            if (atomicAdd(P.red.ticket, 1u) == P.red.expected - 1) {
                if constexpr (OP == V_CG_U2E) {
                    if (S.live) { st->alpha_prev = S.alpha; st->x_lag = 1; }
                } else {
                    st->x_lag = 0;
                }
                st->pending_x = 0;
                *P.red.ticket = 0u;
                __threadfence();
            }
        }
    }
}

// ------------------------------------------------ fused small-problem CG kernel -------
// Whole Jacobi-PCG iterations in ONE cooperative persistent kernel (problems whose chunks
// fit the co-resident grid, e.g. config A): per iteration
//   SpMV + p.q chunk partials | grid barrier | every CTA finishes the canonical reduction
//   and the scalar step itself (identical inputs -> identical decisions) | update 1 +
//   {r.z, r.r} partials | grid barrier | reduction + scalar step | update 2 | grid barrier.
// Same canonical slot / round / tree order as the multi-kernel path, so the trajectory is
// bit-identical.  Vectors written inside the kernel are read with ld.global.cg (L2) so no
// SM sees a stale L1 line of another CTA's rows.
struct FusedParams {
    const int32_t* rp;
    const int32_t* ci;
    const double* val;
    const uint8_t* vidx;  // value dictionary (or nullptr: val)
    const double* vtab;
    const double* d;      // nullptr: constant diagonal d_uni
    double d_uni;
    double *x, *r, *p, *q;
    long long n, nch;
    double* partials;  // [3][nch]
    unsigned* bar;     // grid barrier counter, zeroed before every launch
    KState* st;
    int iters;         // iterations this launch (stops earlier when the solve terminates)
    int res_cap;       // RES: entry capacity of the chunk image in shared memory
};

// Resident chunk image (RES): the matrix does not change across iterations, so each CTA
// keeps its chunk's structure in shared memory for the whole launch — uint16 local row
// offsets, int16 column deltas (col - row) and the 1-byte dictionary indices — and the
// SpMV's only global accesses are the p gathers (one L2 round trip per row instead of
// three: row_ptr -> col/val -> p).
__host__ __device__ constexpr size_t fused_res_bytes(int cap) {
    return (((size_t)kChunk + 1) * 2 + 15) / 16 * 16 + ((size_t)cap * 2 + 15) / 16 * 16 + ((size_t)cap + 15) / 16 * 16;
}

// Host-side eligibility of the resident image: res[0] = max entries of a chunk, res[1] = 1
// if some |col - row| exceeds the int16 range.
static __global__ void __launch_bounds__(kSpmvThreads) fused_res_check_kernel(const int32_t* rp, const int32_t* ci,
                                                                              long long n, int* res) {
    const long long c = blockIdx.x, base = c * kChunk;
    const long long end = base + kChunk < n ? base + kChunk : n;
    if (threadIdx.x == 0) atomicMax(res, rp[end] - rp[base]);
    bool far = false;
    for (long long i = base + threadIdx.x; i < end; i += blockDim.x)
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const long long d = (long long)ci[k] - i;
            far |= d < -32768 || d > 32767;
        }
    if (far) atomicMax(res + 1, 1);
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned target = (epoch + 1) * gridDim.x;
        atomicAdd(bar, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v < target) __nanosleep(20);
        } while (v < target);
    }
    ++epoch;
    __syncthreads();
}

template <int ND>
__device__ __forceinline__ void fused_total(const double* partials, long long m, double* out, double* sred,
                                            volatile double* sbc) {
    double tot[ND];
    final_reduce<kSpmvThreads, ND>(partials, m, tot, sred);
    if (threadIdx.x == 0)
        for (int d = 0; d < ND; ++d) sbc[d] = tot[d];
    __syncthreads();
    for (int d = 0; d < ND; ++d) out[d] = sbc[d];
    __syncthreads();
}

constexpr int kPairW = 6;  // RES: rows of <= kPairW entries are processed two at a time

template <bool RES>
static __global__ void __launch_bounds__(kSpmvThreads, 4) cg_fused_kernel(FusedParams P) {
    __shared__ KState S;
    __shared__ double sred[3 * (kSpmvThreads / 32)];
    __shared__ double sbc[4];
    __shared__ double s_vtab[256];
    extern __shared__ __align__(16) unsigned char fres[];
    const int t = threadIdx.x;
    if (t == 0) S = *P.st;
    if (P.vidx) s_vtab[t] = P.vtab[t];  // kSpmvThreads == 256
    [[maybe_unused]] uint16_t* s_rp = reinterpret_cast<uint16_t*>(fres);
    [[maybe_unused]] int16_t* s_cd = reinterpret_cast<int16_t*>(fres + (((size_t)kChunk + 1) * 2 + 15) / 16 * 16);
    [[maybe_unused]] uint8_t* s_vi =
        fres + (((size_t)kChunk + 1) * 2 + 15) / 16 * 16 + ((size_t)P.res_cap * 2 + 15) / 16 * 16;
    if constexpr (RES) {  // one chunk per CTA (gridDim.x == nch): load its image once
        const long long base = (long long)blockIdx.x * kChunk;
        const int e0 = __ldg(P.rp + base);
        for (int li = t; li <= kChunk; li += kSpmvThreads) {
            const long long row = base + li < P.n ? base + li : P.n;
            s_rp[li] = (uint16_t)(__ldg(P.rp + row) - e0);
        }
        for (int li = t; li < kChunk && base + li < P.n; li += kSpmvThreads) {
            const long long row = base + li;
            for (int k = __ldg(P.rp + row); k < __ldg(P.rp + row + 1); ++k) {
                s_cd[k - e0] = (int16_t)(__ldg(P.ci + k) - row);
                s_vi[k - e0] = __ldg(P.vidx + k);  // RES implies the value dictionary
            }
        }
    }
    __syncthreads();
    if (S.done) return;
    const uint8_t* __restrict__ vidx = P.vidx;
    unsigned epoch = 0;
    const long long m = P.nch;
    for (int it = 0; it < P.iters; ++it) {
        // ---- SpMV q = A p (thread per row, L2-coherent gathers) + p.q chunk partials
        if constexpr (RES) {
            const long long base = (long long)blockIdx.x * kChunk;
            double acc[1] = {0.0};
#pragma unroll 1
            for (int r = 0; r < kChunkRounds; r += 2) {
                // two rows per step: both rows' gathers are in flight together
                const int la = r * kChunkSlots + t, lb = la + kChunkSlots;
                const long long ra = base + la, rb = base + lb;
                const int ka = s_rp[la], kea = s_rp[la + 1], kb = s_rp[lb], keb = s_rp[lb + 1];
                if (rb < P.n && kea - ka <= kPairW && keb - kb <= kPairW) {
                    double xa[kPairW], xb[kPairW];
#pragma unroll
                    for (int u = 0; u < kPairW; ++u) {
                        if (ka + u < kea) xa[u] = __ldcg(P.p + ra + s_cd[ka + u]);
                        if (kb + u < keb) xb[u] = __ldcg(P.p + rb + s_cd[kb + u]);
                    }
                    double ya = 0.0, yb = 0.0;
#pragma unroll
                    for (int u = 0; u < kPairW; ++u) {
                        if (ka + u < kea)
                            ya = __dadd_rn(ya, __dmul_rn(s_vtab[s_vi[ka + u]], xa[u]));
                    }
#pragma unroll
                    for (int u = 0; u < kPairW; ++u) {
                        if (kb + u < keb)
                            yb = __dadd_rn(yb, __dmul_rn(s_vtab[s_vi[kb + u]], xb[u]));
                    }
                    P.q[ra] = ya;
                    P.q[rb] = yb;
                    acc[0] = __dadd_rn(acc[0], __dmul_rn(__ldcg(P.p + ra), ya));
                    acc[0] = __dadd_rn(acc[0], __dmul_rn(__ldcg(P.p + rb), yb));
                    continue;
                }
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                const int li = h ? lb : la;
                const long long row = base + li;
                if (row < P.n) {
                    const int kk = s_rp[li], ke = s_rp[li + 1];
                    double y = 0.0;
                    for (int k0 = kk; k0 < ke; k0 += 8) {
                        double pr[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (k0 + u < ke)
                                pr[u] = __dmul_rn(s_vtab[s_vi[k0 + u]], __ldcg(P.p + row + s_cd[k0 + u]));
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (k0 + u < ke) y = __dadd_rn(y, pr[u]);
                    }
                    P.q[row] = y;
                    acc[0] = __dadd_rn(acc[0], __dmul_rn(__ldcg(P.p + row), y));
                }
                }
            }
            block_tree<kSpmvThreads, 1>(acc, sred);
            if (t == 0) P.partials[blockIdx.x] = acc[0];
        }
        for (long long c = blockIdx.x; !RES && c < m; c += gridDim.x) {
            const long long base = c * kChunk;
            double acc[1] = {0.0};
            int kk = 0, ke = 0;
            long long row = base + t;
            if (row < P.n) { kk = __ldg(P.rp + row); ke = __ldg(P.rp + row + 1); }
#pragma unroll 1
            for (int r = 0; r < kChunkRounds; ++r) {
                // prefetch the next round's row bounds while this row's gathers are in flight
                const long long nrow = row + kChunkSlots;
                int nk = 0, nke = 0;
                if (r + 1 < kChunkRounds && nrow < P.n) { nk = __ldg(P.rp + nrow); nke = __ldg(P.rp + nrow + 1); }
                if (row < P.n) {
                    double y = 0.0;
                    for (int k0 = kk; k0 < ke; k0 += 8) {
                        double pr[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (k0 + u < ke)
                                pr[u] = __dmul_rn(vidx ? s_vtab[__ldg(vidx + k0 + u)] : __ldg(P.val + k0 + u),
                                                  __ldcg(P.p + __ldg(P.ci + k0 + u)));
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (k0 + u < ke) y = __dadd_rn(y, pr[u]);
                    }
                    P.q[row] = y;
                    acc[0] = __dadd_rn(acc[0], __dmul_rn(__ldcg(P.p + row), y));
                }
                row = nrow; kk = nk; ke = nke;
            }
            block_tree<kSpmvThreads, 1>(acc, sred);
            if (t == 0) P.partials[c] = acc[0];
        }
        grid_barrier(P.bar, epoch);
        double pq[1];
        fused_total<1>(P.partials, m, pq, sred, sbc);
        if (t == 0) apply_scalar(SC_CG_PQ, &S, pq);
        __syncthreads();
        if (S.done) break;  // p^T A p <= 0: breakdown (uniform decision)
        const double alpha = S.alpha;
        // ---- update 1: r -= alpha q; z = d r; {r.z, r.r}
        for (long long c = blockIdx.x; c < m; c += gridDim.x) {
            const long long base = c * kChunk;
            double acc[2] = {0.0, 0.0};
#pragma unroll
            for (int r = 0; r < kChunkRounds; ++r) {
                const long long i = base + (long long)r * kChunkSlots + t;
                if (i < P.n) {
                    const double rn = __dsub_rn(__ldcg(P.r + i), __dmul_rn(alpha, __ldcg(P.q + i)));
                    const double z = __dmul_rn(P.d ? __ldg(P.d + i) : P.d_uni, rn);
                    P.r[i] = rn;
                    acc[0] = __dadd_rn(acc[0], __dmul_rn(rn, z));
                    acc[1] = __dadd_rn(acc[1], __dmul_rn(rn, rn));
                }
            }
            block_tree<kSpmvThreads, 2>(acc, sred);
            if (t == 0) { P.partials[m + c] = acc[0]; P.partials[2 * m + c] = acc[1]; }
        }
        grid_barrier(P.bar, epoch);
        double rr2[2];
        fused_total<2>(P.partials + m, m, rr2, sred, sbc);  // per-dot trees: same bits as two calls
        if (t == 0) apply_scalar(SC_CG_RR, &S, rr2);
        __syncthreads();
        const bool live = !S.done;
        const double beta = S.beta;
        // ---- update 2: x += alpha p; p = z + beta p (own rows only)
        for (long long c = blockIdx.x; c < m; c += gridDim.x) {
            const long long base = c * kChunk;
#pragma unroll
            for (int r = 0; r < kChunkRounds; ++r) {
                const long long i = base + (long long)r * kChunkSlots + t;
                if (i < P.n) {
                    const double pv = __ldcg(P.p + i);
                    P.x[i] = __dadd_rn(__ldcg(P.x + i), __dmul_rn(alpha, pv));
                    if (live) P.p[i] = __dadd_rn(__dmul_rn(P.d ? __ldg(P.d + i) : P.d_uni, __ldcg(P.r + i)), __dmul_rn(beta, pv));
                }
            }
        }
        if (!live) break;
        grid_barrier(P.bar, epoch);
    }
    if (blockIdx.x == 0 && t == 0) {
        S.pending_x = 0;
        *P.st = S;
        __threadfence();
    }
}

// Generic canonical dot a.b (level 1 + last-CTA level 2), same chunk shape.
struct DotParams {
    long long n;
    const double* a;
    const double* b;
    RedParams red;
};
static __global__ void __launch_bounds__(kVecThreads) dot_kernel(DotParams P) {
    const int t = threadIdx.x;
    const long long chunk = blockIdx.x;
    const long long base = chunk * kChunk;
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int rd = 0; rd < kChunkRounds; ++rd) {
        const long long i = base + (long long)rd * kChunkSlots + 2 * t;
        const double2 A = ld2(P.a, i, P.n), B = ld2(P.b, i, P.n);
        if (i < P.n) acc[0] = __dadd_rn(acc[0], __dmul_rn(A.x, B.x));
        if (i + 1 < P.n) acc[1] = __dadd_rn(acc[1], __dmul_rn(A.y, B.y));
    }
    __shared__ double sred[kVecThreads / 32];
    double v[1] = {__dadd_rn(acc[0], acc[1])};
    block_tree<kVecThreads, 1>(v, sred);
    publish_and_finish<kVecThreads, 1>(v, chunk, P.red, sred);
}

// Distributed reduction points: rank totals were all-gathered into g[P][k]; sum in
// ascending rank order starting from rank 0 and run the scalar step.
static __global__ void scalar_kernel(const double* g, int nranks, int k, int which, KState* st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (st->done) return;  // (the half step runs with done == 0; SC_BI_U3 sets it)
    double t[4] = {0, 0, 0, 0};
    for (int j = 0; j < k; ++j) {
        double s = g[j];
        for (int q = 1; q < nranks; ++q) s = __dadd_rn(s, g[q * 8 + j]);
        t[j] = s;
    }
    apply_scalar(which, st, t);
}

// Jacobi inverse diagonal: 1/A_ii, or 1.0 when missing / zero / non-finite.
static __global__ void jacobi_kernel(const int32_t* rp, const int32_t* ci, const double* val, long long n,
                              long long col_offset, double* dinv) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long g = i + col_offset;  // local column id of the diagonal
    int lo = rp[i], hi = rp[i + 1];
    double r = 1.0;
    for (int k = lo; k < hi; ++k) {
        if (ci[k] == g) {
            const double a = val[k];
            if (a != 0.0) {
                const double inv = 1.0 / a;
                if (isfinite(inv)) r = inv;
            }
            break;
        }
    }
    dinv[i] = r;
}

// Exact value symmetry (A^T == A bitwise) for adjoint operator reuse.
static __global__ void symmetry_kernel(const int32_t* rp, const int32_t* ci, const double* val, long long n,
                                int* flags) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        int lo = rp[j], hi = rp[j + 1];
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ci[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo == rp[j + 1] || ci[lo] != i) { flags[0] = 0; flags[1] = 0; return; }
        if (val[lo] != val[k]) flags[1] = 0;
    }
}

// Adjoint gradient gather (Eq. 3): grad_vals[k] = -(lam[row_k] * x[col_k]),
// in CSR (= canonical COO) order; one thread per row.
static __global__ void adjoint_gather_kernel(const int32_t* rp, const int32_t* ci, long long n,
                                      const double* lam, const double* x, double* gv) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double l = lam[i];
    const int k1 = rp[i + 1];
    for (int k = rp[i]; k < k1; ++k) gv[k] = -__dmul_rn(l, __ldg(x + ci[k]));
}

static __global__ void fill_kernel(double* p, long long n, double v) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

static __global__ void i64_to_i32_kernel(const long long* in, int32_t* out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)in[i];
}

// Halo pack: sendbuf[j] = x[idx[j]] (canonical global order).
static __global__ void halo_pack_kernel(const double* x, const int32_t* idx, long long m, double* out) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < m) out[j] = x[idx[j]];
}
// Halo unpack: x[idx[j]] = recvbuf[j].
static __global__ void halo_unpack_kernel(double* x, const int32_t* idx, long long m, const double* in) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < m) x[idx[j]] = in[j];
}

}  // namespace sparsla_b200
