// spmv_dia.cuh — "diagonal warp" SpMV for stencil-like CSR matrices.
//
// Same arithmetic as every other SpMV kernel of the library (row-ordered __dmul_rn /
// __dadd_rn sums in stored column order, the fused dots in the canonical chunk shape):
// bit-identical.  At matrix creation (and after set_values) one warp per 32 consecutive
// rows classifies its rows: when every row's entries lie on the same <= 7 "diagonals"
// (entry k of row i in column i + delta_k, with dictionary value v_k), in stored order,
// except at most two entries missing from some rows (the x-boundary rows of a stencil
// line), the warp is "structured" and its 48-byte table entry replaces the rows' row
// pointers, columns and value indices: the SpMV then reads 1.5 B of matrix per 32 rows
// plus x and y.  x is read with coalesced loads straight from global memory (each diagonal
// of a warp is 256 contiguous bytes; neighbouring diagonals share L1 lines), so there is
// no staging pipeline at all.  Other warps ("unstructured") run the CSR loop on the fp64
// values.  The table is kept only when at least 90% of the warps are structured.
//
// Table entry (12 ints per warp): [0..6] delta_k (0 past the last diagonal), [7] v0..v3,
// [8] v4..v6 | m << 24 (m diagonals; 0xFF = unstructured), [9] exception bytes
// (lane << 3 | k, 0x07 = none), [10] link flag (dia_link_kernel), [11] 0.
#pragma once

#include "kernels.cuh"

namespace sparsla_b200 {

constexpr int kDiaInts = 12;            // per warp
constexpr uint32_t kDiaUnstructured = 0xFFu;
constexpr uint32_t kDiaNoEx = 0x07u;

// one warp per 32 rows: classify and write the table entry; cnt[0] += structured warps,
// cnt[1] += CSR bytes the unstructured warps read (row pointers, columns, values)
static __global__ void dia_build_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                        const uint8_t* __restrict__ vidx, long long n, long long nwarps,
                                        int32_t* __restrict__ tab, unsigned long long* cnt) {
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nwarps) return;  // warp-uniform
    const long long row = w * 32 + lane;
    const bool live = row < n;
    int32_t e[kDiaInts] = {0, 0, 0, 0, 0, 0, 0, 0, (int32_t)(kDiaUnstructured << 24), 0, 0, 0};
    const int kb = live ? rp[row] : 0;
    const int len = live ? rp[row + 1] - kb : 0;
    int m = len;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    bool ok;
    if (!__any_sync(0xffffffffu, live)) {  // past the last row: structured, no diagonals
        ok = false;
        e[8] = 0;
        e[9] = (int32_t)(kDiaNoEx | (kDiaNoEx << 8));
    } else if (__all_sync(0xffffffffu, live) && m >= 1 && m <= 7) {
        const int tl = __ffs(__ballot_sync(0xffffffffu, len == m)) - 1;
        long long dk[7];
        uint32_t vk[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const bool mine = lane == tl && k < len;
            dk[k] = __shfl_sync(0xffffffffu, mine ? (long long)ci[kb + k] - row : 0ll, tl);
            vk[k] = __shfl_sync(0xffffffffu, mine ? (uint32_t)vidx[kb + k] : 0u, tl);
        }
        bool tok = true;
#pragma unroll
        for (int k = 0; k < 7; ++k)
            if (k < m) tok = tok && dk[k] >= INT32_MIN && dk[k] <= INT32_MAX;
        int j = 0, miss = 0;
        uint32_t exb[2] = {kDiaNoEx, kDiaNoEx};
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            if (k < m) {
                const bool hit = j < len && (long long)ci[kb + j] - row == dk[k] && (uint32_t)vidx[kb + j] == vk[k];
                if (hit) {
                    ++j;
                } else {
                    if (miss < 2) exb[miss] = ((uint32_t)lane << 3) | (uint32_t)k;
                    ++miss;
                }
            }
        }
        ok = __all_sync(0xffffffffu, tok && j == len);
        int tot = miss;
#pragma unroll
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        ok = ok && tot <= 2;
        if (ok) {
            uint32_t ex[2] = {kDiaNoEx, kDiaNoEx};
            int ne = 0;
            uint32_t b = __ballot_sync(0xffffffffu, miss > 0);
            while (b && ne < 2) {
                const int l = __ffs(b) - 1;
                b &= b - 1;
                const uint32_t e0 = __shfl_sync(0xffffffffu, exb[0], l), e1 = __shfl_sync(0xffffffffu, exb[1], l);
                ex[ne++] = e0;
                if (e1 != kDiaNoEx && ne < 2) ex[ne++] = e1;
            }
#pragma unroll
            for (int k = 0; k < 7; ++k) e[k] = k < m ? (int32_t)dk[k] : 0;
            e[7] = (int32_t)(vk[0] | (vk[1] << 8) | (vk[2] << 16) | (vk[3] << 24));
            e[8] = (int32_t)(vk[4] | (vk[5] << 8) | (vk[6] << 16) | ((uint32_t)m << 24));
            e[9] = (int32_t)(ex[0] | (ex[1] << 8));
        }
    } else {
        ok = false;
    }
    if (lane == 0) {
        int4* t4 = reinterpret_cast<int4*>(tab + w * kDiaInts);
        t4[0] = make_int4(e[0], e[1], e[2], e[3]);
        t4[1] = make_int4(e[4], e[5], e[6], e[7]);
        t4[2] = make_int4(e[8], e[9], e[10], e[11]);
        if (ok) {
            atomicAdd(cnt, 1ull);
        } else if (((uint32_t)e[8] >> 24) == kDiaUnstructured) {
            const long long re = min(w * 32 + 32, n);
            atomicAdd(cnt + 1, (unsigned long long)(4 * (re - w * 32 + 1) + 12 * (long long)(rp[re] - rp[w * 32])));
        }
    }
}

// Per round and warp: the skip mask of this lane (slots past the warp's last diagonal, the
// lane's missing entries, dead rows) and the 7 x loads (skipped slots read x[row]).
__device__ __forceinline__ uint32_t dia_loads(const int32_t* e, const double* __restrict__ x, int row, bool live,
                                              int lane, double (&xv)[7]) {
    const uint32_t m = (uint32_t)e[8] >> 24, ex = (uint32_t)e[9];
    uint32_t skip = (0x7Fu << m) & 0x7Fu;
    if (((ex >> 3) & 31u) == (uint32_t)lane) skip |= 1u << (ex & 7u);
    if (((ex >> 11) & 31u) == (uint32_t)lane) skip |= 1u << ((ex >> 8) & 7u);
    if (!live) skip = 0x7Fu;
    const int rb = live ? row : 0;  // 32-bit column arithmetic: one IMAD.WIDE per address
#pragma unroll
    for (int u = 0; u < 7; ++u) xv[u] = __ldg(x + (((skip >> u) & 1u) ? rb : rb + e[u]));
    return skip;
}
// stencil-interior warp (7 diagonals, no missing entry, every row live): no masks at all
__device__ __forceinline__ double dia_full(const int4& q0, const int4& q1, const int4& q2, const double* __restrict__ x,
                                           const double* s_vtab, int row) {
    const int dl[7] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z};
    double xv[7];
#pragma unroll
    for (int u = 0; u < 7; ++u) xv[u] = __ldg(x + (row + dl[u]));
    const uint32_t vw0 = (uint32_t)q1.w, vw1 = (uint32_t)q2.x;
    double y = 0.0;
#pragma unroll
    for (int u = 0; u < 7; ++u)
        y = __dadd_rn(y, __dmul_rn(s_vtab[((u < 4 ? vw0 : vw1) >> (8 * (u & 3))) & 0xFFu], xv[u]));
    return y;
}
__device__ __forceinline__ bool dia_is_full(const int4& q2) {
    return ((uint32_t)q2.x >> 24) == 7u && (uint32_t)q2.y == (kDiaNoEx | (kDiaNoEx << 8));
}

// the row sum over the present slots in stored order (guard-free when no lane skips)
__device__ __forceinline__ double dia_sum(const int32_t* e, const double* s_vtab, uint32_t skip, const double (&xv)[7]) {
    const uint32_t vw0 = (uint32_t)e[7], vw1 = (uint32_t)e[8];
    double y = 0.0;
    if (__all_sync(0xffffffffu, skip == 0)) {
#pragma unroll
        for (int u = 0; u < 7; ++u)
            y = __dadd_rn(y, __dmul_rn(s_vtab[((u < 4 ? vw0 : vw1) >> (8 * (u & 3))) & 0xFFu], xv[u]));
    } else {
#pragma unroll
        for (int u = 0; u < 7; ++u) {
            const double s = __dadd_rn(y, __dmul_rn(s_vtab[((u < 4 ? vw0 : vw1) >> (8 * (u & 3))) & 0xFFu], xv[u]));
            y = ((skip >> u) & 1u) ? y : s;
        }
    }
    return y;
}
__device__ __forceinline__ double dia_csr_row(const SpmvParams& P, int row) {
    const int kb = __ldg(P.rp + row), ke = __ldg(P.rp + row + 1);
    double y = 0.0;
#pragma unroll 1
    for (int k = kb; k < ke; ++k) y = __dadd_rn(y, __dmul_rn(__ldg(P.val + k), __ldg(P.x + __ldg(P.ci + k))));
    return y;
}

// One CTA = one chunk (8 rounds of 256 rows, thread t owns row round * 256 + t), like
// spmv_direct_kernel.  The chunk's 64 table entries (3 KB) are staged in shared memory at
// the start; rounds are taken two at a time so each warp has 14 independent x loads in
// flight (the kernel is bound by load latency, not bandwidth).  Warps whose rows all have
// every diagonal (the stencil interior) sum guard-free; the others select per slot;
// unstructured warps run the CSR loop.  Sums and dot accumulation in round order.
template <int MODE, int R, int MINB>
__global__ void __launch_bounds__(kSpmvThreads, MINB) spmv_dia_kernel(SpmvParams P) {
    constexpr int ND = SpmvDots<MODE>::n;
    constexpr int NA = ND > 0 ? ND : 1;
    constexpr int kW = kSpmvThreads / 32;
    if (P.check_done && P.red.st->done) return;
    __shared__ double s_vtab[256];
    __shared__ __align__(16) int32_t s_tab[kChunkRounds * kW * kDiaInts];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long chunk = P.chunk_list ? (long long)P.chunk_list[blockIdx.x] : P.chunk0 + blockIdx.x;
    s_vtab[t] = P.vtab[t];  // kSpmvThreads == 256
    const int4* tc = reinterpret_cast<const int4*>(P.dia) + chunk * kChunkRounds * kW * 3;
    if (t < kChunkRounds * kW * 3) reinterpret_cast<int4*>(s_tab)[t] = __ldg(tc + t);
    if (P.dia_ahead > 0 && !P.chunk_list && t >= 192) {
        // one wave ahead: the chunk a successor CTA on this SM will take reads its leading
        // diagonal (the z+1 plane of a 3-D stencil) from DRAM for the first time — pull
        // those 2048 x values and its table into L2 now, so its rounds wait on L2 hits
        const long long ca = chunk + P.dia_ahead;
        if (ca < P.nch) {
            const int4 e0 = __ldg(tc), e1 = __ldg(tc + 1);
            const int dmax = max(max(max(e0.x, e0.y), max(e0.z, e0.w)), max(max(e1.x, e1.y), e1.z));
            const int q = t - 192;  // 64 threads: 2 lines of x each, 24 of them a table line
            const long long j = ca * kChunk + dmax + 32 * q;
            if (j >= 0 && j < P.ncols) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.x + j));
            if (j + 16 >= 0 && j + 16 < P.ncols) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.x + j + 16));
            if (q < 24)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const int4*>(P.dia) + ca * kChunkRounds * kW * 3 + 8 * q));
        }
    }
    if (P.p2p && (long long)blockIdx.x >= P.n_interior) {
        if (t == 0) p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
    }
    __syncthreads();
    const long long base = chunk * kChunk;
    const long long rem_rounds = (P.n - base + kChunkSlots - 1) / kChunkSlots;
    const int nrounds = rem_rounds < kChunkRounds ? (int)rem_rounds : kChunkRounds;
    const int n = (int)P.n;  // int32 CSR: rows < 2^31
    double acc[NA];
#pragma unroll
    for (int d = 0; d < NA; ++d) acc[d] = 0.0;
    auto finish = [&](int row, double y) {
        if (row < n) {
            P.y[row] = y;
            spmv_epilogue<MODE>(P, row, y, acc);
        }
    };
    int r = 0;
    for (; R == 2 && r + 1 < nrounds; r += 2) {
        const int32_t* e0 = s_tab + (r * kW + warp) * kDiaInts;
        const int32_t* e1 = e0 + kW * kDiaInts;
        const int row0 = (int)base + r * kChunkSlots + t, row1 = row0 + kChunkSlots;
        const bool u0 = ((uint32_t)e0[8] >> 24) == kDiaUnstructured, u1 = ((uint32_t)e1[8] >> 24) == kDiaUnstructured;
        if (!u0 && !u1) {  // warp-uniform
            double x0[7], x1[7];
            const uint32_t s0 = dia_loads(e0, P.x, row0, row0 < n, lane, x0);
            const uint32_t s1 = dia_loads(e1, P.x, row1, row1 < n, lane, x1);
            finish(row0, dia_sum(e0, s_vtab, s0, x0));
            finish(row1, dia_sum(e1, s_vtab, s1, x1));
        } else {
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int32_t* e = h ? e1 : e0;
                const int row = h ? row1 : row0;
                double y = 0.0;
                if (((uint32_t)e[8] >> 24) != kDiaUnstructured) {
                    double xv[7];
                    const uint32_t sk = dia_loads(e, P.x, row, row < n, lane, xv);
                    y = dia_sum(e, s_vtab, sk, xv);
                } else if (row < n) {
                    y = dia_csr_row(P, row);
                }
                finish(row, y);
            }
        }
    }
#pragma unroll 1
    for (; r < nrounds; ++r) {  // one round at a time (R = 1; the odd last round for R = 2)
        const int32_t* e = s_tab + (r * kW + warp) * kDiaInts;
        const int row = (int)base + r * kChunkSlots + t;
        const int4* q = reinterpret_cast<const int4*>(e);
        const int4 q2 = q[2];
        double y = 0.0;
        if (dia_is_full(q2)) {  // warp-uniform
            y = dia_full(q[0], q[1], q2, P.x, s_vtab, row);
        } else if (((uint32_t)e[8] >> 24) != kDiaUnstructured) {
            double xv[7];
            const uint32_t sk = dia_loads(e, P.x, row, row < n, lane, xv);
            y = dia_sum(e, s_vtab, sk, xv);
        } else if (row < n) {
            y = dia_csr_row(P, row);
        }
        finish(row, y);
    }
    if constexpr (ND > 0) {
        __shared__ double sred[SpmvFin<MODE>::n * kW];
        block_tree<kSpmvThreads, ND>(acc, sred);
        publish_and_finish<kSpmvThreads, ND, SpmvFin<MODE>::n>(acc, chunk, P.red, sred);
    }
}

// Second build pass: e[10] = kDiaSame when the entry's diagonals and values (words 0..8)
// equal those of the same warp slot one round earlier in the same chunk and both are
// structured — spmv_diar_kernel then keeps that round's registers instead of re-decoding.
constexpr int32_t kDiaSame = 1;
static __global__ void dia_link_kernel(int32_t* __restrict__ tab, long long nwarps) {
    const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwarps) return;
    constexpr int kW = kSpmvThreads / 32;
    const int r = (int)((w / kW) % kChunkRounds);
    int32_t* e = tab + w * kDiaInts;
    int same = 0;
    if (r > 0) {
        const int32_t* p = e - kW * kDiaInts;
        same = ((uint32_t)e[8] >> 24) != kDiaUnstructured && ((uint32_t)p[8] >> 24) != kDiaUnstructured;
        for (int k = 0; k < 9 && same; ++k) same = e[k] == p[k];
    }
    e[10] = same ? kDiaSame : 0;
}

// v = x[a] when p (one predicated ld.global.nc: the compiler would branch around a guarded
// __ldg per slot)
__device__ __forceinline__ void ldg_pred(double& v, const double* a, bool p) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.f64 %0, [%1];\n\t}"
                 : "+d"(v) : "l"(a), "r"((unsigned)p));
}

// The 7 x operands of a row.  C > 0: slots C-1, C, C+1 are the diagonals -1, 0, +1 (a
// canonical stencil row), taken from x[row] and its neighbouring lanes (one predicated
// load at each warp edge); C == 0: any pattern.  Other slots load x[row + delta], skipped
// slots (missing entry, past the last diagonal, dead row) load nothing.
template <int C>
__device__ __forceinline__ void dia_gather(const int (&dl)[7], uint32_t skip, const double* __restrict__ x, int rb,
                                           int lane, double xc, double (&xv)[7]) {
    if constexpr (C > 0) {
        // every load is issued before the shuffles, which wait on x[row]
        double em = 0.0, ep = 0.0;  // (no copy of xc: a predicated load would wait on it)
        ldg_pred(em, x + (rb - 1), lane == 0 && !((skip >> (C - 1)) & 1u));
        ldg_pred(ep, x + (rb + 1), lane == 31 && !((skip >> (C + 1)) & 1u));
#pragma unroll
        for (int u = 0; u < 7; ++u) {
            if (u < C - 1 || u > C + 1) {
                xv[u] = 0.0;  // skipped slots are masked out of the sum
                ldg_pred(xv[u], x + (rb + dl[u]), !((skip >> u) & 1u));
            }
        }
        const double sm = __shfl_up_sync(0xffffffffu, xc, 1), sp = __shfl_down_sync(0xffffffffu, xc, 1);
        xv[C - 1] = lane == 0 ? em : sm;
        xv[C] = xc;
        xv[C + 1] = lane == 31 ? ep : sp;
    } else {
#pragma unroll
        for (int u = 0; u < 7; ++u) {
            xv[u] = 0.0;
            ldg_pred(xv[u], x + (rb + dl[u]), !((skip >> u) & 1u));
        }
    }
}

// Register-pattern variant.  The l1tex data pipe was the limiter of spmv_dia_kernel (76%
// of its wavefronts: ~16 per warp-row were uniform shared-memory reads of the table entry
// and the 7 dictionary values).  Here a warp decodes its entry into registers (7 deltas, 7
// fp64 values) only when it differs from the previous round's (e[10]), reads one 8-byte
// word per round otherwise, takes x[row] once (reused by the diagonal-0 slot and the CG
// epilogue) and forms the +-1 diagonals by warp shuffles of it (one single-lane load at the
// warp edge).  Same products and sums in the same order: bit-identical.
template <int MODE, int MINB>
__global__ void __launch_bounds__(kSpmvThreads, MINB) spmv_diar_kernel(SpmvParams P) {
    constexpr int ND = SpmvDots<MODE>::n;
    constexpr int NA = ND > 0 ? ND : 1;
    constexpr int kW = kSpmvThreads / 32;
    if (P.check_done && P.red.st->done) return;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long chunk = P.chunk_list ? (long long)P.chunk_list[blockIdx.x] : P.chunk0 + blockIdx.x;
    const int4* tc = reinterpret_cast<const int4*>(P.dia) + chunk * kChunkRounds * kW * 3;
    if (P.dia_ahead > 0 && !P.chunk_list && t >= 192) {  // as spmv_dia_kernel
        const long long ca = chunk + P.dia_ahead;
        if (ca < P.nch) {
            const int4 e0 = __ldg(tc), e1 = __ldg(tc + 1);
            const int dmax = max(max(max(e0.x, e0.y), max(e0.z, e0.w)), max(max(e1.x, e1.y), e1.z));
            const int q = t - 192;
            const long long j = ca * kChunk + dmax + 32 * q;
            if (j >= 0 && j < P.ncols) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.x + j));
            if (j + 16 >= 0 && j + 16 < P.ncols) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.x + j + 16));
            if (q < 24)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const int4*>(P.dia) + ca * kChunkRounds * kW * 3 + 8 * q));
        }
    }
    if (P.p2p && (long long)blockIdx.x >= P.n_interior) {  // CTA-uniform
        if (t == 0) p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
        __syncthreads();
    }
    // no shared-memory staging: this warp's entries are read straight from the table (L1),
    // word 2 (diagonal count, exceptions, link flag) one round ahead
    const int4* tw = tc + warp * 3;
    const long long base = chunk * kChunk;
    const long long rem_rounds = (P.n - base + kChunkSlots - 1) / kChunkSlots;
    const int nrounds = rem_rounds < kChunkRounds ? (int)rem_rounds : kChunkRounds;
    const int n = (int)P.n;  // int32 CSR: rows < 2^31
    const double* __restrict__ x = P.x;
    double acc[NA];
#pragma unroll
    for (int d = 0; d < NA; ++d) acc[d] = 0.0;
    int dl[7];
    double vv[7];
    uint32_t full = 0;  // 0x7F >> (7 - m): slots present in a row with no missing entry
    int cls = 0;        // dia_gather shape of the decoded pattern
#pragma unroll
    for (int u = 0; u < 7; ++u) { dl[u] = 0; vv[u] = 0.0; }
    int4 q2n = __ldg(tw + 2);
#pragma unroll 1
    for (int r = 0; r < nrounds; ++r) {
        const int4* te = tw + r * kW * 3;
        const int4 q2 = q2n;
        if (r + 1 < nrounds) q2n = __ldg(te + kW * 3 + 2);
        const int row = (int)base + r * kChunkSlots + t;
        const bool live = row < n;
        const uint32_t w8 = (uint32_t)q2.x;
        double y = 0.0, xc = 0.0;
        if ((w8 >> 24) == kDiaUnstructured) {  // warp-uniform: CSR loop on the fp64 values
            if (live) {
                y = dia_csr_row(P, row);
                if constexpr (MODE == SPMV_CG) xc = __ldg(x + row);
            }
        } else {
            if (!(q2.z & kDiaSame)) {  // decode: deltas and values into registers
                const int4 q0 = __ldg(te), q1 = __ldg(te + 1);
                dl[0] = q0.x; dl[1] = q0.y; dl[2] = q0.z; dl[3] = q0.w; dl[4] = q1.x; dl[5] = q1.y; dl[6] = q1.z;
                const uint32_t vw0 = (uint32_t)q1.w;
#pragma unroll
                for (int u = 0; u < 7; ++u) vv[u] = __ldg(P.vtab + (((u < 4 ? vw0 : w8) >> (8 * (u & 3))) & 0xFFu));
                const int m = (int)(w8 >> 24);
                full = 0x7Fu >> (7 - m);
                cls = 0;
#pragma unroll
                for (int c = 1; c <= 3; ++c)
                    if (c + 1 < m && dl[c - 1] == -1 && dl[c] == 0 && dl[c + 1] == 1) cls = c;
            }
            const uint32_t ex = (uint32_t)q2.y;
            uint32_t skip = ~full & 0x7Fu;
            if (ex != (kDiaNoEx | (kDiaNoEx << 8))) {  // warp-uniform: a row misses entries
                if (((ex >> 3) & 31u) == (uint32_t)lane) skip |= 1u << (ex & 7u);
                if (((ex >> 11) & 31u) == (uint32_t)lane) skip |= 1u << ((ex >> 8) & 7u);
                skip &= 0x7Fu;  // (a lone exception's "none" byte names slot 7)
            }
            if (!live) skip = 0x7Fu;
            const int rb = live ? row : 0;
            xc = __ldg(x + rb);
            double xv[7];
            if (cls == 3) dia_gather<3>(dl, skip, x, rb, lane, xc, xv);  // warp-uniform
            else if (cls == 2) dia_gather<2>(dl, skip, x, rb, lane, xc, xv);
            else if (cls == 1) dia_gather<1>(dl, skip, x, rb, lane, xc, xv);
            else dia_gather<0>(dl, skip, x, rb, lane, xc, xv);
            if (__all_sync(0xffffffffu, skip == 0)) {  // 7 diagonals, nothing missing
#pragma unroll
                for (int u = 0; u < 7; ++u) y = __dadd_rn(y, __dmul_rn(vv[u], xv[u]));
            } else {
#pragma unroll
                for (int u = 0; u < 7; ++u) {
                    const double s = __dadd_rn(y, __dmul_rn(vv[u], xv[u]));
                    y = ((skip >> u) & 1u) ? y : s;
                }
            }
        }
        if (live) {
            P.y[row] = y;
            if constexpr (MODE == SPMV_CG) acc[0] = __dadd_rn(acc[0], __dmul_rn(xc, y));
            else spmv_epilogue<MODE>(P, row, y, acc);
        }
    }
    if constexpr (ND > 0) {
        __shared__ double sred[SpmvFin<MODE>::n * kW];
        block_tree<kSpmvThreads, ND>(acc, sred);
        publish_and_finish<kSpmvThreads, ND, SpmvFin<MODE>::n>(acc, chunk, P.red, sred);
    }
}

}  // namespace sparsla_b200

namespace sparsla_b200 {

// ---------------------------------------------------------------------------------------
// Pattern-table variant (spmv_diac_kernel).  The distinct structured table entries of a
// matrix ("patterns": diagonals + values; a 3-D stencil has ~10: interior, boundary planes
// and lines) are deduplicated at build time and passed by value as a __grid_constant__
// kernel parameter, so a warp's per-round description shrinks to one 32-bit word (pattern
// id + exceptions: 4 B per 32 rows instead of 48) and the deltas and fp64 values are read
// through the constant cache (LDC) instead of the l1tex pipe that bounds spmv_dia_kernel.
constexpr int kDiaPatterns = 64;
constexpr uint32_t kDiaPidUnstructured = 0xFFu;
struct DiaPattern {
    int d[8];      // deltas of the m diagonals (0 past the last), d[7] = m
    double v[8];   // their fp64 values (v[7] unused)
};
struct DiaConst {
    DiaPattern pat[kDiaPatterns];
};
constexpr int kDiaHashSlots = 512;

// build pass 1: hash each structured entry's words 0..8 into an open-addressed table of
// kDiaHashSlots 64-bit keys; the lowest warp index of a slot is its representative
static __global__ void dia_hash_kernel(const int32_t* __restrict__ tab, long long nwarps,
                                       unsigned long long* keys, unsigned long long* rep, int16_t* slot,
                                       int* overflow, unsigned* count) {
    const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwarps) return;
    const int32_t* e = tab + w * kDiaInts;
    if (((uint32_t)e[8] >> 24) == kDiaUnstructured) { slot[w] = -1; return; }
    unsigned long long h = 1469598103934665603ull;
#pragma unroll
    for (int k = 0; k < 9; ++k) h = (h ^ (uint32_t)e[k]) * 1099511628211ull;
    h |= 1ull;  // 0 marks an empty slot
    int i = (int)(h % kDiaHashSlots);
    for (int probe = 0; probe < kDiaHashSlots; ++probe) {
        const unsigned long long prev = atomicCAS(keys + i, 0ull, h);
        if (prev == 0ull || prev == h) {
            atomicMin(rep + i, (unsigned long long)w);
            atomicAdd(count + i, 1u);
            slot[w] = (int16_t)i;
            return;
        }
        i = (i + 1) % kDiaHashSlots;
    }
    slot[w] = -2;
    atomicExch(overflow, 1);
}

// build pass 2: per warp the 32-bit word [pid | ex0 << 8 | ex1 << 16]; an entry that differs
// from its slot's representative (a hash collision) raises *bad (the host then keeps the
// 48-byte table kernel)
static __global__ void dia_compact_kernel(const int32_t* __restrict__ tab, long long nwarps,
                                          const int16_t* __restrict__ slot, const unsigned long long* __restrict__ rep,
                                          const int* __restrict__ pid_of, uint32_t* __restrict__ words, int* bad) {
    const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwarps) return;
    const int32_t* e = tab + w * kDiaInts;
    const int s = slot[w];
    uint32_t pid = kDiaPidUnstructured;
    if (s >= 0) {
        const int32_t* r = tab + (long long)rep[s] * kDiaInts;
        for (int k = 0; k < 9; ++k)
            if (e[k] != r[k]) atomicExch(bad, 1);
        pid = (uint32_t)pid_of[s];
    } else if (s == -2) {
        atomicExch(bad, 1);
    }
    words[w] = pid | (((uint32_t)e[9] & 0xFFFFu) << 8);
}

// PERS: a resident grid loops over the launch's chunks (list index i = blockIdx.x, + gridDim.x,
// ...), stores one partial per chunk and takes ONE reduction ticket at the end (no per-chunk
// atomic round trip holding the CTA slot); otherwise one chunk per CTA.
// x operand of one diagonal: NA: diagonals farther than kDiaFar rows (the +-plane ones of a
// 3-D stencil, never re-read from L1) bypass L1 allocation so the near diagonals' lines
// (+-1, +-line, re-read by the rows a line later) stay resident
constexpr int kDiaFar = 4096;
template <bool NA>
__device__ __forceinline__ double dia_x(const double* __restrict__ a, int d) {
    if constexpr (NA) {
        if (d >= kDiaFar || d <= -kDiaFar) {  // warp-uniform
            double v;
            asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(a));
            return v;
        }
    }
    return __ldg(a);
}

// SPEC: round 0's x operands are loaded with pattern 0 (the most frequent: patterns are
// numbered by count) at CTA start, in parallel with the load of the warp's pattern words —
// used when round 0 turns out to be a pattern-0 interior warp, otherwise reloaded.
template <int MODE, int MINB, int UNR = 1, bool PERS = false, bool L1NA = false, bool SPEC = false>
__global__ void __launch_bounds__(kSpmvThreads, MINB) spmv_diac_kernel(SpmvParams P, const __grid_constant__ DiaConst C) {
    constexpr int ND = SpmvDots<MODE>::n;
    constexpr int NA = ND > 0 ? ND : 1;
    constexpr int kW = kSpmvThreads / 32;
    if (P.check_done && P.red.st->done) return;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    __shared__ double sred[(SpmvFin<MODE>::n > 0 ? SpmvFin<MODE>::n : 1) * kW];
    __shared__ int s_flag;
    bool halo_ok = false;
    for (long long li = blockIdx.x; li < (PERS ? P.nch : (long long)blockIdx.x + 1); li += gridDim.x) {
    const long long chunk = P.chunk_list ? (long long)P.chunk_list[li] : P.chunk0 + li;
    const uint32_t* wc = P.diaw + chunk * kChunkRounds * kW;
    const long long base = chunk * kChunk;
    const long long rem_rounds = (P.n - base + kChunkSlots - 1) / kChunkSlots;
    const int nrounds = rem_rounds < kChunkRounds ? (int)rem_rounds : kChunkRounds;
    // lane r holds this warp's word of round r
    const uint32_t wpre = lane < nrounds ? __ldg(wc + lane * kW + warp) : kDiaPidUnstructured;
    if (P.dia_ahead > 0 && !P.chunk_list && t >= 192) {
        // one wave ahead: the leading diagonal of the chunk a successor CTA will take (the
        // largest delta of this chunk's first pattern), pulled into L2
        const long long ca = chunk + P.dia_ahead;
        if (ca < P.nch) {
            const uint32_t p0 = __ldg(wc) & 0xFFu;
            int dmax = 0;
            if (p0 != kDiaPidUnstructured) {
#pragma unroll
                for (int u = 0; u < 7; ++u) dmax = max(dmax, C.pat[p0].d[u]);
            }
            const int q = t - 192;
            const long long j = ca * kChunk + dmax + 32 * q;
            if (j >= 0 && j < P.ncols) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.x + j));
            if (j + 16 >= 0 && j + 16 < P.ncols) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.x + j + 16));
            if (q < 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.diaw + ca * kChunkRounds * kW + 32 * q));
        }
    }
    if (P.p2p && li >= P.n_interior && !halo_ok) {  // CTA-uniform
        if (t == 0) p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
        __syncthreads();
        halo_ok = true;
    }
    const int n = (int)P.n;  // int32 CSR: rows < 2^31
    const double* __restrict__ x = P.x;
    double xs[7];
    if constexpr (SPEC) {  // after the halo wait: the operands may be halo values
        const int rs = (int)base + t;
#pragma unroll
        for (int u = 0; u < 7; ++u) {
            const int c = rs + C.pat[0].d[u];
            xs[u] = 0.0;
            ldg_pred(xs[u], x + c, rs < n && c >= 0 && (long long)c < P.ncols);
        }
    }
    double acc[NA];
#pragma unroll
    for (int d = 0; d < NA; ++d) acc[d] = 0.0;
#pragma unroll UNR
    for (int r = 0; r < nrounds; ++r) {
        const uint32_t wd = __shfl_sync(0xffffffffu, wpre, r);
        const uint32_t pid = wd & 0xFFu;
        const int row = (int)base + r * kChunkSlots + t;
        const bool live = row < n;
        double y = 0.0;
        // the epilogue operand, loaded with the row's x operands (not after the sum)
        double ea = 0.0;
        if constexpr (MODE == SPMV_CG) ea = live ? __ldg(x + row) : 0.0;
        if constexpr (MODE == SPMV_BICG_V || MODE == SPMV_BICG_T) ea = live ? __ldg(P.aux + row) : 0.0;
        if (pid == kDiaPidUnstructured) {  // warp-uniform: CSR loop on the fp64 values
            if (live) y = dia_csr_row(P, row);
        } else {
            const DiaPattern& pt = C.pat[pid];
            const int m = pt.d[7];
            const uint32_t ex = wd >> 8;
            const int rb = live ? row : 0;
            double xv[7];
            if (m == 7 && ex == (kDiaNoEx | (kDiaNoEx << 8)) && __all_sync(0xffffffffu, live)) {
                if (SPEC && r == 0 && pid == 0) {
#pragma unroll
                    for (int u = 0; u < 7; ++u) xv[u] = xs[u];
                } else {
#pragma unroll
                    for (int u = 0; u < 7; ++u) xv[u] = dia_x<L1NA>(x + (rb + pt.d[u]), pt.d[u]);
                }
#pragma unroll
                for (int u = 0; u < 7; ++u) y = __dadd_rn(y, __dmul_rn(pt.v[u], xv[u]));
            } else {
                uint32_t skip = (0x7Fu << m) & 0x7Fu;
                if (((ex >> 3) & 31u) == (uint32_t)lane) skip |= 1u << (ex & 7u);
                if (((ex >> 11) & 31u) == (uint32_t)lane) skip |= 1u << ((ex >> 8) & 7u);
                skip &= 0x7Fu;
                if (!live) skip = 0x7Fu;
#pragma unroll
                for (int u = 0; u < 7; ++u) xv[u] = dia_x<L1NA>(x + (((skip >> u) & 1u) ? rb : rb + pt.d[u]), pt.d[u]);
#pragma unroll
                for (int u = 0; u < 7; ++u) {
                    const double s = __dadd_rn(y, __dmul_rn(pt.v[u], xv[u]));
                    y = ((skip >> u) & 1u) ? y : s;
                }
            }
        }
        if (live) {
            P.y[row] = y;
            if constexpr (MODE == SPMV_CG || MODE == SPMV_BICG_V) {  // as spmv_epilogue
                acc[0] = __dadd_rn(acc[0], __dmul_rn(ea, y));
            } else if constexpr (MODE == SPMV_BICG_T) {
                acc[0] = __dadd_rn(acc[0], __dmul_rn(y, y));
                acc[1] = __dadd_rn(acc[1], __dmul_rn(y, ea));
            }
        }
    }
    if constexpr (ND > 0) {
        block_tree<kSpmvThreads, ND>(acc, sred);
        if constexpr (PERS) {
            if (t == 0) {
#pragma unroll
                for (int d = 0; d < ND; ++d) P.red.partials[d * P.red.nchunks + chunk] = acc[d];
            }
        } else {
            publish_and_finish<kSpmvThreads, ND, SpmvFin<MODE>::n>(acc, chunk, P.red, sred);
        }
    }
    }  // chunk loop
    if constexpr (PERS && ND > 0) ticket_and_finish<kSpmvThreads, ND, 0, SpmvFin<MODE>::n>(P.red, sred, &s_flag);
}

}  // namespace sparsla_b200
