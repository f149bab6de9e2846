// spmv_xw.cuh — x-window staged SpMV (banded / structured-mesh matrices).
//
// Same arithmetic as spmv_ws_kernel (row-ordered __dmul_rn/__dadd_rn sums in stored column
// order, the same fused dots in the same canonical chunk shape) — bit-identical — but the x
// operand is no longer gathered by the consumer threads.  For each 256-row round a setup
// pass (DevCsr::create, build_xwin) records up to kXwMax contiguous windows of x that cover
// the round's columns (for a 7-point stencil: the z-1 plane, y-1 line, centre, y+1 line and
// z+1 plane segments, ~260 elements each).  The producer warp streams those windows into the
// stage with TMA bulk copies next to the round's row_ptr / col_idx / value stream (and, for
// BiCGStab, the epilogue vector's segment), so the leading-plane DRAM latency is hidden by
// the ring instead of by consumer registers, and consumers only read shared memory.  A
// column outside every window (boundary rows, truncated windows) is read from global
// memory, so any window set is correct; the windows only decide how fast.
#pragma once

#include "kernels.cuh"

namespace sparsla_b200 {

constexpr int kXwMax = 8;  // windows per round; descriptor = int32 start[8], len[8] (elements)

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
    size_t vbytes, cbytes, rbytes, dbytes, xbytes, abytes, stage;
    size_t coff, roff, doff, xoff, aoff;
    __host__ __device__ XwLayout(int cap_v, int cap_c, int cap_x, bool vd, bool aux) {
        vbytes = ((size_t)cap_v * (vd ? 1 : 8) + (vd ? 32 : 0) + 127) & ~size_t(127);
        cbytes = ((size_t)cap_c * 4 + 127) & ~size_t(127);
        rbytes = (kRpCopy * 4 + 127) & ~size_t(127);
        dbytes = 128;  // consumer view of the windows: start[8], end[8], base[8]
        xbytes = ((size_t)cap_x * 8 + 127) & ~size_t(127);
        abytes = aux ? (size_t)kChunkSlots * 8 : 0;
        coff = vbytes;
        roff = coff + cbytes;
        doff = roff + rbytes;
        xoff = doff + dbytes;
        aoff = xoff + xbytes;
        stage = aoff + abytes;
    }
};

template <int MODE> struct XwAux { static constexpr bool on = (MODE == SPMV_BICG_V || MODE == SPMV_BICG_T); };

// Window lookup for column c, walking from window w (monotone within a row; restarts when a
// column precedes the current window, e.g. the relabelled halo columns of a local matrix).
__device__ __forceinline__ double xw_load(const int32_t* D, const double* sx, const double* __restrict__ x,
                                          int c, int& w) {
    if (c < D[w]) w = 0;
    while (w < kXwMax - 1 && c >= D[kXwMax + w]) ++w;
    if (c >= D[w] && c < D[kXwMax + w]) return sx[c + D[2 * kXwMax + w]];
    return __ldg(x + c);
}

template <int MODE, int STG, int MINB, int W, bool VD>
__global__ void __launch_bounds__(kWsThreads, MINB) spmv_xw_kernel(SpmvParams P) {
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
    const XwLayout L(P.cap_v, P.cap_c, P.cap_x, VD, AUX);
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
            bool halo_ok = P.p2p == nullptr;
            long long g = 0;
            for (long long c = blockIdx.x; c < P.nch; c += gridDim.x) {
                if (!halo_ok && c >= P.n_interior) {
                    // the boundary rounds' x windows include halo values pushed by the peers:
                    // wait for them, then order the async-proxy reads after the acquire
                    p2p_wait_halo(P.p2p, P.halo_v, P.red.st->ep_halo[P.halo_v]);
                    fence_proxy_async_global();
                    halo_ok = true;
                }
                const long long chunk = P.chunk_list ? (long long)P.chunk_list[c] : P.chunk0 + c;
                const long long base = chunk * kChunk;
                const long long rem = (P.n - base + kChunkSlots - 1) / kChunkSlots;
                const int nr = rem < kChunkRounds ? (int)rem : kChunkRounds;
                for (int r = 0; r < nr; ++r, ++g) {
                    const int s = (int)(g % STG);
                    const long long rs = base + (long long)r * kChunkSlots;
                    const long long re = min(rs + kChunkSlots, P.n);
                    // this round's loads go out before the wait for a free stage
                    const int nz0 = __ldg(P.rp + rs), nz1 = __ldg(P.rp + re);
                    const int4* dsc = reinterpret_cast<const int4*>(P.xw + (chunk * kChunkRounds + r) * (2 * kXwMax));
                    const int4 st0 = __ldg(dsc), st1 = __ldg(dsc + 1), ln0 = __ldg(dsc + 2), ln1 = __ldg(dsc + 3);
                    mbar_wait(&empty[s], (uint32_t)(((g / STG) & 1) ^ 1));
                    const int a0 = nz0 & ~(VALIGN - 1), a1 = (nz1 + VALIGN - 1) & ~(VALIGN - 1);
                    const int c0 = nz0 & ~3, c1 = (nz1 + 3) & ~3;
                    const uint32_t vb = (uint32_t)(a1 - a0) * (VD ? 1u : 8u);
                    const uint32_t cb = (uint32_t)(c1 - c0) * 4u;
                    unsigned char* st = stage0 + s * L.stage;
                    const int ws[kXwMax] = {st0.x, st0.y, st0.z, st0.w, st1.x, st1.y, st1.z, st1.w};
                    const int wl[kXwMax] = {ln0.x, ln0.y, ln0.z, ln0.w, ln1.x, ln1.y, ln1.z, ln1.w};
                    int32_t* D = reinterpret_cast<int32_t*>(st + L.doff);
                    uint32_t xb = 0;
#pragma unroll
                    for (int w = 0; w < kXwMax; ++w) {
                        const int xo = (int)(xb >> 3);
                        D[w] = wl[w] ? ws[w] : 0x7fffffff;
                        D[kXwMax + w] = wl[w] ? ws[w] + wl[w] : 0x7fffffff;
                        D[2 * kXwMax + w] = xo - ws[w];
                        xb += (uint32_t)wl[w] * 8u;
                    }
                    const uint32_t ab = AUX ? (uint32_t)((re - rs) & ~1LL) * 8u : 0u;
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(kRpCopy * 4) + vb + cb + xb + ab);
                    bulk_g2s(st + L.roff, P.rp + rs, kRpCopy * 4, &full[s], pol);
                    if constexpr (VD) {
                        if (vb) bulk_g2s(st, P.vidx + a0, vb, &full[s], pol);
                    } else {
                        if (vb) bulk_g2s(st, P.val + a0, vb, &full[s], pol);
                    }
                    if (cb) bulk_g2s(st + L.coff, P.ci + c0, cb, &full[s], pol);
                    uint32_t xo = 0;
#pragma unroll
                    for (int w = 0; w < kXwMax; ++w)
                        if (wl[w]) {
                            bulk_g2s_plain(st + L.xoff + xo, P.x + ws[w], (uint32_t)wl[w] * 8u, &full[s]);
                            xo += (uint32_t)wl[w] * 8u;
                        }
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
            const int32_t* D = reinterpret_cast<const int32_t*>(A + L.doff);
            const double* sx = reinterpret_cast<const double*>(A + L.xoff);
            const long long rs = base + (long long)r * kChunkSlots;
            const long long row = rs + t;
            const bool live = row < P.n;
            const int o0 = rps[0];
            const int kb = live ? rps[t] : o0, ke = live ? rps[t + 1] : o0;
            const int len = ke - kb;
            const int32_t* cp = reinterpret_cast<const int32_t*>(A + L.coff) + (kb - (o0 & ~3));
            const uint8_t* vp = A + (kb - (o0 & ~(VALIGN - 1)));
            const double* vs = reinterpret_cast<const double*>(A) + (kb - (o0 & ~(VALIGN - 1)));
            auto value = [&](int u) -> double {
                if constexpr (VD) return s_vtab[vp[u]];
                else return vs[u];
            };
            double y = 0.0;
            int w = 0;
            if (__all_sync(0xffffffffu, len <= W)) {
                double xv[W];
#pragma unroll
                for (int u = 0; u < W; ++u)
                    if (u < len) xv[u] = xw_load(D, sx, P.x, cp[u], w);
#pragma unroll
                for (int u = 0; u < W; ++u)
                    if (u < len) y = __dadd_rn(y, __dmul_rn(value(u), xv[u]));
            } else {
                for (int k0 = 0; k0 < len; k0 += W) {
                    double pr[W];
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (k0 + u < len) pr[u] = __dmul_rn(value(k0 + u), xw_load(D, sx, P.x, cp[k0 + u], w));
#pragma unroll
                    for (int u = 0; u < W; ++u)
                        if (k0 + u < len) y = __dadd_rn(y, pr[u]);
                }
            }
            // the fused dot's operand: p[row] (CG, usually inside the centre window) or the
            // staged r-hat / s segment (BiCGStab)
            double eop = 0.0;
            if (live) {
                if constexpr (MODE == SPMV_CG) {
                    int w2 = 0;
                    eop = xw_load(D, sx, P.x, (int)row, w2);
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
