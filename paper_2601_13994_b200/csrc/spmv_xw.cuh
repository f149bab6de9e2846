// spmv_xw.cuh — x-window staged SpMV (banded / structured-mesh matrices).
//
// Same arithmetic as spmv_ws_kernel (row-ordered __dmul_rn/__dadd_rn sums in stored column
// order, the same fused dots in the same canonical chunk shape) — bit-identical — but the x
// operand is not gathered by the consumer threads.  For each 256-row round a setup pass
// (DevCsr::create, build_xwin) records up to kXwMax contiguous windows of x covering the
// round's columns (7-point stencil: the z-1 plane, y-1 line, centre, y+1 line and z+1 plane
// segments, ~260 elements each), and re-expresses every entry's column as a 16-bit offset
// into the round's staged windows (0xFFFF: outside every window).  The producer warp
// streams, per round, the row_ptr segment, the value stream (fp64 values or 1-byte
// dictionary indices), the 16-bit window offsets (instead of the 4-byte columns) and the x
// windows themselves (plus, for BiCGStab, the epilogue vector's segment) into the stage with
// TMA bulk copies, so the leading-plane DRAM latency is covered by the ring instead of by
// consumer registers, and a consumer entry costs two shared-memory reads.  Entries outside
// the windows read their column and x from global memory, so any window set is correct;
// the windows only decide how fast.  The per-round descriptors are themselves prefetched a
// whole chunk ahead into shared memory by TMA.
#pragma once

#include "kernels.cuh"

namespace sparsla_b200 {

constexpr int kXwMax = 8;       // windows per round
constexpr int kXwDescInts = 16; // per-round descriptor (64 B):
//   [0..7]  window start (x element index)     [8..11] window lengths, 2 x uint16 per int
//   [12]    row_ptr[rs]  [13] row_ptr[re]       [14] staged offset of x[rs] when rows
//   [rs, re) lie inside one window (CG's p.q operand), else -1      [15] 1: every entry of
//   the round is staged (the consumer skips the per-entry fallback test)
constexpr uint16_t kXwNone = 0xFFFFu;
// pair stream: (window offset << 3) | dictionary index (<= 8 values); offset 0x1FFF = not
// staged.  With the index in the low bits, e & ~7 is the byte offset of x in the staged
// windows and (e & 7) * 8 the byte offset of the value in the table: one mask per address.
constexpr int kXwPairValBits = 3;
constexpr uint32_t kXwPairValMask = (1u << kXwPairValBits) - 1u;
constexpr uint32_t kXwPairNone = 0xFFFFu >> kXwPairValBits;  // offset field of an unstaged entry

// pair stream from the dictionary indices and the window offsets (device, after every
// dictionary (re)build)
static __global__ void xw_pair_kernel(const uint8_t* vidx, const uint16_t* xwo, uint16_t* xvo, long long m) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t o = xwo[k];
    xvo[k] = (uint16_t)(((o == kXwNone ? kXwPairNone : o) << kXwPairValBits) | vidx[k]);
}
constexpr int kXwPad = 32;  // offsets past the last entry (bulk-copy granule slack)


__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// TMA bulk copy global -> shared without an L2 policy (x windows are re-read by later rounds)
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

struct XwLayout {
    size_t vbytes, obytes, rbytes, xbytes, abytes, stage;
    size_t ooff, roff, xoff, aoff;
    // vs: value stream 0 = fp64 values, 1 = 1-byte dictionary indices, 2 = none (the value
    // index travels in the top 5 bits of the 16-bit offset: "pair" stream)
    __host__ __device__ constexpr XwLayout(int cap_v, int cap_c, int cap_x, int vs, bool aux)
        : vbytes(0), obytes(0), rbytes(0), xbytes(0), abytes(0), stage(0), ooff(0), roff(0), xoff(0), aoff(0) {
        vbytes = vs == 2 ? 0 : ((size_t)cap_v * (vs ? 1 : 8) + (vs ? 32 : 0) + 127) & ~size_t(127);
        obytes = ((size_t)cap_c * 2 + 64 + 127) & ~size_t(127);  // 16-bit window offsets (+ spares)
        rbytes = (kRpCopy * 4 + 127) & ~size_t(127);
        xbytes = ((size_t)cap_x * 8 + 127) & ~size_t(127);
        abytes = aux ? (size_t)kChunkSlots * 8 : 0;
        ooff = vbytes;
        roff = ooff + obytes;
        xoff = roff + rbytes;
        aoff = xoff + xbytes;
        stage = aoff + abytes;
    }
};
// shared memory in front of the stages: full/empty barriers, descriptor barriers, and the
// double-buffered per-chunk descriptor block [2][kChunkRounds][kXwDescInts]
constexpr size_t kXwHead = 1024 + 2 * kChunkRounds * kXwDescInts * 4;

template <int MODE> struct XwAux { static constexpr bool on = (MODE == SPMV_BICG_V || MODE == SPMV_BICG_T); };

// FIX: compile-time stage layout for matrices whose rounds fit kXwFixCapC offsets and
// kXwFixCapX staged x elements (stencils): the per-round stage addressing folds into
// immediates instead of being rematerialised from the parameters at 56 registers
constexpr int kXwFixCapC = 2016;  // (2016 * 2 + 64) bytes = 4 KB of offsets
__host__ __device__ constexpr int xw_fix_cap_x(int fix) { return fix == 1 ? 1536 : 1408; }
template <int MODE, int STG, int MINB, int W, int VS, int FIX = 0>
__global__ void __launch_bounds__(kWsThreads, MINB) spmv_xw_kernel(SpmvParams P) {
    constexpr bool VD = VS != 0;     // values from the dictionary table
    constexpr bool PAIR = VS == 2;   // ... indexed by the top bits of the offset stream
    constexpr int ND = SpmvDots<MODE>::n;
    constexpr int NA = ND > 0 ? ND : 1;
    constexpr bool AUX = XwAux<MODE>::on;
    constexpr int VALIGN = VD ? 16 : 2;
    if (P.check_done && P.red.st->done) return;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double s_vtab[VD ? 256 : 1];
    if constexpr (VD) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_vtab[i] = P.vtab[i];
    }
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + STG;
    uint64_t* dbar = empty + STG;  // [2]
    int32_t* dbuf = reinterpret_cast<int32_t*>(smem + 1024);
    const XwLayout L = FIX ? XwLayout(0, kXwFixCapC, xw_fix_cap_x(FIX), VS, AUX) : XwLayout(P.cap_v, P.cap_c, P.cap_x, VS, AUX);
    unsigned char* stage0 = smem + kXwHead;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int s = 0; s < STG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        mbar_init(&dbar[0], 1);
        mbar_init(&dbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {  // ------------------------------- producer warp ----
        // Lane-parallel issue: per round, lanes 0-7 copy the x windows (one each), lane 8 the
        // row_ptr segment, lane 9 the value stream, lane 10 the offset stream, lane 11 the
        // epilogue vector segment — one SIMT bulk-copy instruction instead of ~8 serial ones
        // (the producer sits on the critical path: a few extra scalar instructions per
        // window measurably slowed the kernel).
        const uint64_t pol = P.l2_keep ? policy_evict_last() : policy_evict_first();
        constexpr uint32_t kDescBytes = kChunkRounds * kXwDescInts * 4;
        auto chunk_of = [&](long long c) { return P.chunk_list ? (long long)P.chunk_list[c] : P.chunk0 + c; };
        auto fetch_desc = [&](long long c, int b) {
            mbar_arrive_expect_tx(&dbar[b], kDescBytes);
            bulk_g2s(dbuf + b * kChunkRounds * kXwDescInts, P.xw + chunk_of(c) * kChunkRounds * kXwDescInts,
                     kDescBytes, &dbar[b], pol);
        };
        if (lane == 0 && (long long)blockIdx.x < P.nch) fetch_desc(blockIdx.x, 0);
        bool halo_ok = P.p2p == nullptr;
        long long g = 0;
        int ci = 0;
        for (long long c = blockIdx.x; c < P.nch; c += gridDim.x, ++ci) {
            const int b = ci & 1;
            if (lane == 0 && c + gridDim.x < P.nch) {  // one chunk ahead (buffer b^1 was read last chunk)
                fence_proxy_async_smem();
                fetch_desc(c + gridDim.x, b ^ 1);
            }
            if (!halo_ok && c >= P.n_interior) {
                // the boundary rounds' x windows include halo values pushed by the peers:
                // wait for them, then order the async-proxy reads after the acquire
                if (lane == 0) {
                    p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
                    fence_proxy_async_global();
                }
                __syncwarp();
                halo_ok = true;
            }
            mbar_wait(&dbar[b], (uint32_t)((ci >> 1) & 1));
            const long long base = chunk_of(c) * kChunk;
            const long long rem = (P.n - base + kChunkSlots - 1) / kChunkSlots;
            const int nr = rem < kChunkRounds ? (int)rem : kChunkRounds;
            for (int r = 0; r < nr; ++r, ++g) {
                const int s = (int)(g % STG);
                const int32_t* d = dbuf + (b * kChunkRounds + r) * kXwDescInts;
                const long long rs = base + (long long)r * kChunkSlots;
                // this lane's window (lanes 0-7) and its offset in the staged x: shuffle scan
                const uint32_t wlen = lane < kXwMax ? ((uint32_t)d[8 + lane / 2] >> (16 * (lane & 1))) & 0xffffu : 0u;
                uint32_t incl = wlen;
#pragma unroll
                for (int o = 1; o < kXwMax; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const uint32_t xb = __shfl_sync(0xffffffffu, incl, kXwMax - 1) * 8u;
                const int nz0 = d[12], nz1 = d[13];
                const int a0 = nz0 & ~(VALIGN - 1), a1 = (nz1 + VALIGN - 1) & ~(VALIGN - 1);
                const int o0 = nz0 & ~7, o1 = (nz1 + 7) & ~7;
                const uint32_t vb = PAIR ? 0u : (uint32_t)(a1 - a0) * (VD ? 1u : 8u);
                const uint32_t ob = (uint32_t)(o1 - o0) * 2u;
                const uint32_t ab = AUX ? (uint32_t)((min(rs + kChunkSlots, P.n) - rs) & ~1LL) * 8u : 0u;
                mbar_wait(&empty[s], (uint32_t)(((g / STG) & 1) ^ 1));
                unsigned char* st = stage0 + s * L.stage;
                if (lane == 0) {
                    reinterpret_cast<int32_t*>(st + L.roff)[kRpCopy] = d[14];      // staged x[rs] offset
                    reinterpret_cast<int32_t*>(st + L.roff)[kRpCopy + 1] = d[15];  // every entry staged
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(kRpCopy * 4) + vb + ob + xb + ab);
                }
                __syncwarp();
                if (lane < kXwMax) {
                    if (wlen) bulk_g2s_plain(st + L.xoff + (incl - wlen) * 8u, P.x + d[lane], wlen * 8u, &full[s]);
                } else if (lane == kXwMax) {
                    bulk_g2s(st + L.roff, P.rp + rs, kRpCopy * 4, &full[s], pol);
                } else if (lane == kXwMax + 1) {
                    if constexpr (VD) {
                        if (vb) bulk_g2s(st, P.vidx + a0, vb, &full[s], pol);
                    } else {
                        if (vb) bulk_g2s(st, P.val + a0, vb, &full[s], pol);
                    }
                } else if (lane == kXwMax + 2) {
                    if (ob) bulk_g2s(st + L.ooff, P.xwo + o0, ob, &full[s], pol);
                } else if (lane == kXwMax + 3) {
                    if constexpr (AUX)
                        if (ab) bulk_g2s(st + L.aoff, P.aux + rs, ab, &full[s], pol);
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------------ consumers ----
    __shared__ double sred[(SpmvFin<MODE>::n > 0 ? SpmvFin<MODE>::n : 1) * kConsumerWarps];
    __shared__ int s_flag;
    int s = 0;
    uint32_t ph = 0;
    bool halo_ok = P.p2p == nullptr;
    for (long long c = blockIdx.x; c < P.nch; c += gridDim.x) {
        if (!halo_ok && c >= P.n_interior) {  // global fallback reads of halo columns
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
            const int32_t* rps = reinterpret_cast<const int32_t*>(A + L.roff);
            const double* sx = reinterpret_cast<const double*>(A + L.xoff);
            const long long rs = base + (long long)r * kChunkSlots;
            const long long row = rs + t;
            const bool live = row < P.n;
            const int o0 = rps[0];
            const int kb = live ? rps[t] : o0, ke = live ? rps[t + 1] : o0;
            const int len = ke - kb;
            const uint16_t* xo = reinterpret_cast<const uint16_t*>(A + L.ooff) + (kb - (o0 & ~7));
            const uint8_t* vp = A + (kb - (o0 & ~(VALIGN - 1)));
            const double* vs = reinterpret_cast<const double*>(A) + (kb - (o0 & ~(VALIGN - 1)));
            auto value = [&](int u) -> double {
                if constexpr (PAIR) return s_vtab[xo[u] & kXwPairValMask];
                else if constexpr (VD) return s_vtab[vp[u]];
                else return vs[u];
            };
            auto xval = [&](int u) -> double {
                if constexpr (PAIR) {
                    const uint32_t o = (uint32_t)xo[u] >> kXwPairValBits;
                    return o != kXwPairNone ? sx[o] : __ldg(P.x + __ldg(P.ci + kb + u));
                } else {
                    const uint32_t o = xo[u];
                    return o != kXwNone ? sx[o] : __ldg(P.x + __ldg(P.ci + kb + u));
                }
            };
            double y = 0.0;
            const bool all_staged = rps[kRpCopy + 1] != 0;  // round-uniform
            auto product = [&](int u) -> double {
                if constexpr (PAIR) {
                    const uint32_t e = xo[u];
                    return __dmul_rn(s_vtab[e & kXwPairValMask], sx[e >> kXwPairValBits]);
                } else {
                    return __dmul_rn(value(u), sx[xo[u]]);
                }
            };
            const bool exact = __all_sync(0xffffffffu, len == W || !live);  // warp-uniform
            if (all_staged && exact) {
                // every live row of the warp has exactly W entries (stencil interiors with
                // the W = 7 variants): straight-line code, no per-entry guards (idle lanes
                // read the round's first row, always staged, and discard the sum)
                double pr[W];
#pragma unroll
                for (int u = 0; u < W; ++u) pr[u] = product(u);
#pragma unroll
                for (int u = 0; u < W; ++u) y = __dadd_rn(y, pr[u]);
                if (!live) y = 0.0;
            } else if (all_staged && __all_sync(0xffffffffu, len <= W)) {
                // common case: every x operand of the round is in the staged windows (the
                // per-entry guards stay branches: reading all W slots unconditionally was
                // measured slower — shared-memory bandwidth, profiles/r02_xwin.md)
                double pr[W];
#pragma unroll
                for (int u = 0; u < W; ++u)
                    if (u < len) {
                        if constexpr (PAIR) {
                            const uint32_t e = xo[u];
                            pr[u] = __dmul_rn(s_vtab[e & kXwPairValMask], sx[e >> kXwPairValBits]);
                        } else {
                            pr[u] = __dmul_rn(value(u), sx[xo[u]]);
                        }
                    }
#pragma unroll
                for (int u = 0; u < W; ++u)
                    if (u < len) y = __dadd_rn(y, pr[u]);
            } else {
                // rounds with unstaged entries or long rows: one entry at a time, same order
#pragma unroll 1
                for (int k = 0; k < len; ++k) y = __dadd_rn(y, __dmul_rn(value(k), xval(k)));
            }
            // the fused dot's operand: p[row] (CG: staged when the round's rows lie inside
            // one window) or the staged r-hat / s segment (BiCGStab)
            double eop = 0.0;
            if (live) {
                if constexpr (MODE == SPMV_CG) {
                    const int xr = rps[kRpCopy];
                    eop = xr >= 0 ? sx[xr + t] : __ldg(P.x + row);
                } else if constexpr (AUX) {
                    const double* sa = reinterpret_cast<const double*>(A + L.aoff);
                    eop = t < (int)((min(rs + kChunkSlots, P.n) - rs) & ~1LL) ? sa[t] : __ldg(P.aux + row);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (live) {
                P.y[row] = y;
                if constexpr (MODE == SPMV_CG || MODE == SPMV_BICG_V) {
                    acc[0] = __dadd_rn(acc[0], __dmul_rn(eop, y));
                } else if constexpr (MODE == SPMV_BICG_T) {
                    acc[0] = __dadd_rn(acc[0], __dmul_rn(y, y));
                    acc[1] = __dadd_rn(acc[1], __dmul_rn(y, eop));
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
}

}  // namespace sparsla_b200
