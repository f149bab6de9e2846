// eigen.cu — smallest-k eigenpairs by LOBPCG and the eigenvalue adjoint on sm_100a
// (eigen-solver module; Eq. 4).
//
// Everything that touches an n-length vector runs on the GPU; the host only solves the
// tiny dense problems (Rayleigh-Ritz and the SVQB Gram eigenproblems, q <= 48).
//
// Data layout: one row-major basis buffer S (n x LD, LD = 3m) holds the blocks
// [X | W | P] in fixed column slots [0,m) [m,2m) [2m,3m); AS holds A S in the same slots.
// Every block kernel takes column LISTS, so the active subsets of W and P (soft locking:
// converged pairs contribute no W / P directions) need no compaction copies.  One basis
// row (144 B at m = 6) is contiguous, so the SpMM gathers S[col] as whole 16-byte lines.
//
// Per LOBPCG iteration (m = k block vectors):
//   (R = AX - X diag(lambda), ||R_j||, W = |D|^-1 R come out of the previous RR update)
//   W: twice { Y = X^T W (gram), W -= X Y (combine), SVQB(W) }           orthonormal W
//   P: twice { Y = [X W]^T P, P -= [X W] Y, SVQB(P) }                    orthonormal P
//   spmm_kernel    AS[:, W P] = A S[:, W P]                               1 SpMM of <= 2m columns
//   gram           G = S_B^T AS_B, B = X u W u P (q <= 3m)               host: eig(G)
//   rr_apply       X' = S_B C, AX' = AS_B C, P' = S_{W,P} C_{W,P}        (Hetmaniuk-Lehoucq P)
//                  + R' = AX' - X' Lambda', ||R'_j||, W' = |D|^-1 R'      1 fused pass
// Reductions use a fixed grid (kRedCTAs) and fixed in-CTA orders, so a run is
// deterministic.  Parity is tolerance-based (eigenvalues to 1e-8 against
// a dense symmetric eigensolver) — there is no bitwise reference for this module.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "common.hpp"
#include "device.hpp"

namespace sparsla_b200 {
namespace {

#define CK(x) cuda_check((x), #x)

constexpr int kMaxK = 16;             // block size limit of the GPU LOBPCG
constexpr int kMaxQ = 3 * kMaxK;      // basis columns [X | W | P]
constexpr int kRedCTAs = 296;         // fixed reduction grid (device-independent result)
constexpr int kPartRows = 4 * 148;     // >= kRedCTAs and the rr_apply grid (pinned readback rows)
constexpr int kT = 256;

template <class T>
T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

struct Cols {  // column list of a row-major block buffer (kernel parameter)
    int n = 0;
    unsigned char c[kMaxQ] = {};
};

struct Mat {  // small dense coefficient matrix a x c (row-major, c <= 2 kMaxK), kernel parameter
    double v[kMaxQ * 2 * kMaxK];
};

// Copy a column list into shared memory with constant indices (a dynamically indexed
// kernel-parameter array would be copied to local memory first).
__device__ __forceinline__ void stage_cols(const Cols& c, int* dst) {
#pragma unroll
    for (int j = 0; j < kMaxQ; ++j)
        if ((int)threadIdx.x == j && j < c.n) dst[j] = c.c[j];
}

struct Vec16 {
    double v[kMaxK];
};

// Coefficient matrices of the block transforms live in constant memory (warp-uniform
// broadcast reads, usable as direct FMA operands): the host path copies them in before each
// launch, the device-resident iteration copies them from the small-problem kernels' output
// with device-to-device memcpy nodes of the captured graph.  One LOBPCG runs at a time per
// process (eig_mutex).
__constant__ double c_coef[kMaxQ * 2 * kMaxK];  // apply_kernel: a x C (row-major)
__constant__ double c_rrC[kMaxQ * kMaxK];       // rr_apply_kernel: q x m
__constant__ double c_rrlam[kMaxK];             // rr_apply_kernel: the m Ritz values

// device-resident iteration: kernels of a captured iteration exit at entry once the solve
// has stopped (or this step is skipped)
__device__ __forceinline__ bool halted(const int* stop) { return stop && *(volatile const int*)stop; }

__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// contiguous row range of CTA `b` of the fixed reduction grid
__device__ __forceinline__ void cta_rows(long long n, long long& r0, long long& r1) {
    const long long per = (n + gridDim.x - 1) / gridDim.x;
    r0 = (long long)blockIdx.x * per;
    r1 = min(n, r0 + per);
}

// ------------------------------------------------------------------------ kernels ----
// Initial block: uniform(-1, 1) from a counter-based hash of (seed, row, column), so the
// start vectors do not depend on the launch geometry.
__global__ void eig_init_kernel(double* S, long long n, int ld, int m, uint64_t seed) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int j = 0; j < m; ++j) {
        const uint64_t h = splitmix64(seed ^ splitmix64((uint64_t)i * (uint64_t)m + (uint64_t)j));
        S[i * ld + j] = (double)(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
}

__global__ void eye_kernel(double* S, long long n, int ld) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int j = 0; j < ld; ++j) S[i * ld + j] = (j == i) ? 1.0 : 0.0;
}

// Block SpMV: Y[i, out_j] = sum_k A_ik S[c_k, in_j] for NW listed columns (one thread per
// row, all NW accumulators in registers).  VEC: the columns are one contiguous, even-aligned
// range (the usual case), so every gathered row segment and every output row segment moves
// as 16-byte double2 accesses.
template <int NW, bool VEC>
__global__ void __launch_bounds__(kT) spmm_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                  const double* __restrict__ val, long long n,
                                                  const double* __restrict__ S, int lds, Cols in, double* Y,
                                                  int ldy, Cols out, const int* stop) {
    if (halted(stop)) return;
    __shared__ int s_in[kMaxQ], s_out[kMaxQ];
    stage_cols(in, s_in);
    stage_cols(out, s_out);
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int col[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) col[j] = s_in[j];
    const int kb = __ldg(rp + i), ke = __ldg(rp + i + 1);
    double acc[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) acc[j] = 0.0;
    for (int k = kb; k < ke; ++k) {
        const double v = __ldg(val + k);
        const double* srow = S + (size_t)__ldg(ci + k) * lds;
        if constexpr (VEC) {
            const double2* s2 = reinterpret_cast<const double2*>(srow + col[0]);
#pragma unroll
            for (int j = 0; j < NW / 2; ++j) {
                const double2 x = __ldg(s2 + j);
                acc[2 * j] = fma(v, x.x, acc[2 * j]);
                acc[2 * j + 1] = fma(v, x.y, acc[2 * j + 1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < NW; ++j) acc[j] = fma(v, __ldg(srow + col[j]), acc[j]);
        }
    }
    double* yrow = Y + i * ldy;
    if constexpr (VEC) {
        double2* y2 = reinterpret_cast<double2*>(yrow + s_out[0]);
#pragma unroll
        for (int j = 0; j < NW / 2; ++j) y2[j] = make_double2(acc[2 * j], acc[2 * j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < NW; ++j) yrow[s_out[j]] = acc[j];
    }
}

// Coalesced block SpMV for a contiguous, even-aligned column range of NW columns: L = NW/2
// lanes share a row (each owns one double2 column pair), 32/L rows per warp.  Every gathered
// row segment S[c, in:in+NW] is one contiguous NW*8-byte access by the row's lanes (one or two
// L1 wavefronts instead of NW/2 scattered 16-byte requests), the row's (col, val) pairs are
// broadcast loads, and the outputs are contiguous double2 stores.
template <int NW>
__global__ void __launch_bounds__(kT) spmm_lanes_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                        const double* __restrict__ val, long long n,
                                                        const double* __restrict__ S, int lds, int c_in,
                                                        double* Y, int ldy, int c_out, const int* stop) {
    if (halted(stop)) return;
    constexpr int L = NW / 2, RPW = 32 / L;
    const int lane = threadIdx.x & 31, sub = lane / L, part = lane - sub * L;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long i = warp * RPW + sub;
    if (sub >= RPW || i >= n) return;
    const int kb = __ldg(rp + i), ke = __ldg(rp + i + 1);
    double2 acc = make_double2(0.0, 0.0);
    const double* base = S + c_in + 2 * part;
    for (int k = kb; k < ke; ++k) {
        const double v = __ldg(val + k);
        const double2 x = __ldg(reinterpret_cast<const double2*>(base + (size_t)__ldg(ci + k) * lds));
        acc.x = fma(v, x.x, acc.x);
        acc.y = fma(v, x.y, acc.y);
    }
    *reinterpret_cast<double2*>(Y + i * ldy + c_out + 2 * part) = acc;
}

#define SPARSLA_FOR_1_32(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
    X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32)

// ------------------------------------------------- row-tile staging (TMA bulk) ----
// The block kernels below stream whole basis rows: a tile of kTR consecutive rows of a
// row-major buffer is one contiguous range (kTR * ld doubles, ld even -> 16-byte multiple),
// copied into shared memory by one cp.async.bulk per buffer with mbarrier completion.  Each
// CTA walks the tiles t = blockIdx.x + j * gridDim.x through a kEStages-deep ring; thread 0
// re-arms a stage right after the CTA barrier that ends its use.  Outputs are assembled in
// shared memory and written back by bulk stores (cp.async.bulk.global.shared::cta).
constexpr int kTR = 64;    // Gram tiles
constexpr int kTRa = 128;  // apply tiles (one thread per row)
constexpr int kEStages = 3;
constexpr int kTileR = 6;  // 6x6 register tile of the Gram matrix per thread

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(smem_addr(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int TR>
struct TileWalk {
    long long n, ntiles, mine;
    int ld;
    __device__ TileWalk(long long n_, int ld_) : n(n_), ld(ld_) {
        ntiles = (n + TR - 1) / TR;
        mine = (long long)blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    }
    __device__ long long row0(long long j) const { return ((long long)blockIdx.x + j * gridDim.x) * TR; }
    __device__ int rows(long long j) const { return (int)min((long long)TR, n - row0(j)); }
    // thread 0: load tile j of up to two buffers into stage s
    __device__ void issue(long long j, int s, uint64_t* bar, double* stage, const double* A, const double* B) const {
        const long long r0 = row0(j);
        const uint32_t bytes = (uint32_t)rows(j) * (uint32_t)ld * 8u;
        const size_t te = (size_t)TR * ld;
        mbar_arrive_expect_tx(&bar[s], B ? 2 * bytes : bytes);
        bulk_load(stage, A + r0 * ld, bytes, &bar[s]);
        if (B) bulk_load(stage + te, B + r0 * ld, bytes, &bar[s]);
    }
};

// Gram block G = U_uc^T V_vc (a x b <= 48 x 48).  Each thread owns a 6x6 register tile of G
// and a residue class of every tile's rows; row groups are combined in ascending order, CTA
// partials land in `partial`, and the last CTA (ticket) sums them in CTA order into `out`.
// The grid is fixed (kRedCTAs), so the result is deterministic and device-independent.
__global__ void __launch_bounds__(kT) gram_kernel(const double* __restrict__ U, const double* __restrict__ V, int ld,
                                                  Cols uc, Cols vc, long long n, double* partial,
                                                  unsigned* ticket, double* out, int nst, const int* stop) {
    if (halted(stop)) return;
    constexpr int R = kTileR;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // [nst <= 8]
    int* s_uc = reinterpret_cast<int*>(smem + 64);
    int* s_vc = s_uc + kMaxQ;
    double* red = reinterpret_cast<double*>(smem + 512);
    double* ring = red + kMaxQ * kMaxQ;
    const bool two = U != V;
    const size_t te = (size_t)kTR * ld, st_el = two ? 2 * te : te;
    const int a = uc.n, b = vc.n, ab = a * b;
    const int TI = (a + R - 1) / R, TJ = (b + R - 1) / R, tiles = TI * TJ;
    const int ngroups = min(kTR, max(1, kT / tiles));
    const int tid = threadIdx.x, grp = tid / tiles, tt = tid - grp * tiles;
    const bool act = grp < ngroups;
    const int ti = tt / TJ, tj = tt - ti * TJ;
    stage_cols(uc, s_uc);
    stage_cols(vc, s_vc);
    const TileWalk<kTR> W(n, ld);
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (long long j = 0; j < min((long long)nst, W.mine); ++j)
            W.issue(j, (int)j, bar, ring + j * st_el, U, two ? V : nullptr);
    }
    __syncthreads();
    int cu[R], cv[R];
#pragma unroll
    for (int x = 0; x < R; ++x) {
        cu[x] = ti * R + x < a ? s_uc[ti * R + x] : 0;
        cv[x] = tj * R + x < b ? s_vc[tj * R + x] : 0;
    }
    double acc[R][R];
#pragma unroll
    for (int x = 0; x < R; ++x)
#pragma unroll
        for (int y = 0; y < R; ++y) acc[x][y] = 0.0;
    for (long long j = 0; j < W.mine; ++j) {
        const int s = (int)(j % nst);
        mbar_wait(&bar[s], (uint32_t)((j / nst) & 1));
        const double* Ut = ring + s * st_el;
        const double* Vt = two ? Ut + te : Ut;
        const int nr = W.rows(j);
        if (act) {
            for (int r = grp; r < nr; r += ngroups) {
                double u[R], v[R];
#pragma unroll
                for (int x = 0; x < R; ++x) u[x] = Ut[r * ld + cu[x]];
#pragma unroll
                for (int y = 0; y < R; ++y) v[y] = Vt[r * ld + cv[y]];
#pragma unroll
                for (int x = 0; x < R; ++x)
#pragma unroll
                    for (int y = 0; y < R; ++y) acc[x][y] = fma(u[x], v[y], acc[x][y]);
            }
        }
        __syncthreads();
        if (tid == 0 && j + nst < W.mine) {
            fence_proxy_async_smem();
            W.issue(j + nst, s, bar, ring + s * st_el, U, two ? V : nullptr);
        }
    }
    // row groups in ascending order: every group's tile into the drained ring
    // (ngroups * ab <= 36 * 256 doubles), then one ordered sum per entry
    double* gbuf = ring;
    if (act) {
#pragma unroll
        for (int x = 0; x < R; ++x)
#pragma unroll
            for (int y = 0; y < R; ++y) {
                const int i = ti * R + x, k = tj * R + y;
                if (i < a && k < b) gbuf[(size_t)grp * ab + i * b + k] = acc[x][y];
            }
    }
    __syncthreads();
    for (int e = tid; e < ab; e += kT) {
        double sum = 0.0;
        for (int g = 0; g < ngroups; ++g) sum += gbuf[(size_t)g * ab + e];
        red[e] = sum;
    }
    __syncthreads();
    for (int e = tid; e < ab; e += kT) partial[(size_t)blockIdx.x * ab + e] = red[e];
    (void)ticket; (void)out;  // the CTA partials are summed by gram_finish_kernel
}

// Warp-specialised Gram block (same result, same fixed grid and combination order as
// gram_kernel): warp kGwConsumers is the producer — lane 0 streams the CTA's 64-row tiles
// of U (and V) into a kGwStages-deep ring by TMA, re-arming a stage once every consumer warp
// has released it (empty mbarrier) — and the consumer warps never meet at a CTA barrier
// inside the tile loop.  gram_kernel's per-tile __syncthreads was its largest stall
// (profiles/r02_lobpcg.md).
constexpr int kGwConsumers = 7;  // + 1 producer warp = 256 threads: 2 CTAs/SM at <= 128 registers
constexpr int kGwMaxStages = 8;
__global__ void __launch_bounds__((kGwConsumers + 1) * 32, 2) gram_ws_kernel(const double* __restrict__ U,
                                                                          const double* __restrict__ V, int ld,
                                                                          Cols uc, Cols vc, long long n,
                                                                          double* partial, unsigned* ticket,
                                                                          double* out, int nst, const int* stop) {
    if (halted(stop)) return;
    constexpr int R = kTileR;
    constexpr int NT = kGwConsumers * 32;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [nst <= kGwMaxStages]
    uint64_t* empty = full + kGwMaxStages;                // [nst]
    int* s_uc = reinterpret_cast<int*>(smem + 256);
    int* s_vc = s_uc + kMaxQ;
    double* red = reinterpret_cast<double*>(smem + 512);
    double* ring = red + kMaxQ * kMaxQ;
    const bool two = U != V;
    const size_t te = (size_t)kTR * ld, st_el = two ? 2 * te : te;
    const int a = uc.n, b = vc.n, ab = a * b;
    const int TI = (a + R - 1) / R, TJ = (b + R - 1) / R, tiles = TI * TJ;
    const int ngroups = min(kTR, max(1, NT / tiles));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp = tid / tiles, tt = tid - grp * tiles;
    const bool act = warp < kGwConsumers && grp < ngroups;
    const int ti = tt / TJ, tj = tt - ti * TJ;
    stage_cols(uc, s_uc);
    stage_cols(vc, s_vc);
    const TileWalk<kTR> W(n, ld);
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kGwConsumers);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kGwConsumers) {  // producer
        if (lane == 0) {
            for (long long j = 0; j < W.mine; ++j) {
                const int s = (int)(j % nst);
                mbar_wait(&empty[s], (uint32_t)(((j / nst) & 1) ^ 1));
                W.issue(j, s, full, ring + s * st_el, U, two ? V : nullptr);
            }
        }
    } else {
        int cu[R], cv[R];
#pragma unroll
        for (int x = 0; x < R; ++x) {
            cu[x] = ti * R + x < a ? s_uc[ti * R + x] : 0;
            cv[x] = tj * R + x < b ? s_vc[tj * R + x] : 0;
        }
        double acc[R][R];
#pragma unroll
        for (int x = 0; x < R; ++x)
#pragma unroll
            for (int y = 0; y < R; ++y) acc[x][y] = 0.0;
        for (long long j = 0; j < W.mine; ++j) {
            const int s = (int)(j % nst);
            mbar_wait(&full[s], (uint32_t)((j / nst) & 1));
            const double* Ut = ring + s * st_el;
            const double* Vt = two ? Ut + te : Ut;
            const int nr = W.rows(j);
            if (act) {
                for (int r = grp; r < nr; r += ngroups) {
                    double u[R], v[R];
#pragma unroll
                    for (int x = 0; x < R; ++x) u[x] = Ut[r * ld + cu[x]];
#pragma unroll
                    for (int y = 0; y < R; ++y) v[y] = Vt[r * ld + cv[y]];
#pragma unroll
                    for (int x = 0; x < R; ++x)
#pragma unroll
                        for (int y = 0; y < R; ++y) acc[x][y] = fma(u[x], v[y], acc[x][y]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        // consumers finished reading the ring: reuse it for the row-group combination
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
        double* gbuf = ring;
        if (act) {
#pragma unroll
            for (int x = 0; x < R; ++x)
#pragma unroll
                for (int y = 0; y < R; ++y) {
                    const int i = ti * R + x, k = tj * R + y;
                    if (i < a && k < b) gbuf[(size_t)grp * ab + i * b + k] = acc[x][y];
                }
        }
    }
    __syncthreads();
    for (int e = tid; e < ab; e += blockDim.x) {
        double sum = 0.0;
        for (int g = 0; g < ngroups; ++g) sum += ring[(size_t)g * ab + e];
        red[e] = sum;
    }
    __syncthreads();
    for (int e = tid; e < ab; e += blockDim.x) partial[(size_t)blockIdx.x * ab + e] = red[e];
    (void)ticket; (void)out;  // the CTA partials are summed by gram_finish_kernel
}

// Sum of the Gram kernels' CTA partials (partial[p * ab + e], p < P) into out[e].  One
// last CTA summing P x ab partials with 8 loads in flight per thread was a ~30 us serial
// tail; here 32 entries per block, 8 warps each summing a residue class of p (coalesced
// rows), combined in warp order: deterministic, independent of the device.
__global__ void __launch_bounds__(256) gram_finish_kernel(const double* __restrict__ partial, int P, int ab,
                                                          double* out, const int* stop) {
    if (halted(stop)) return;
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int e = blockIdx.x * 32 + lane;
    double sum = 0.0;
    if (e < ab) {
        int p = w;
        for (; p + 24 < P; p += 32) {
            const double a0 = __ldcg(partial + (size_t)p * ab + e), a1 = __ldcg(partial + (size_t)(p + 8) * ab + e);
            const double a2 = __ldcg(partial + (size_t)(p + 16) * ab + e), a3 = __ldcg(partial + (size_t)(p + 24) * ab + e);
            sum += a0; sum += a1; sum += a2; sum += a3;
        }
        for (; p < P; p += 8) sum += __ldcg(partial + (size_t)p * ab + e);
    }
    red[w][lane] = sum;
    __syncthreads();
    if (w == 0 && e < ab) {
        double t = red[0][lane];
        for (int q = 1; q < 8; ++q) t += red[q][lane];
        out[e] = t;
    }
}

// In-place block transform of whole rows: S[:, out_j] = sum_l S[:, in_l] M[l, j]
// (a = in.n <= 48 inputs, c = out.n <= 32 outputs).  One thread per row (kTRa rows per
// tile): the coefficients are warp-uniform constant-bank reads; the row's inputs are read
// from the staged tile before its outputs are written back into it, then the whole rows
// are bulk-stored.
// DEV: coefficients from the c_coef symbol (device-resident iteration) instead of the
// kernel parameter M (host driver)
template <int C, bool DEV>
__global__ void __launch_bounds__(kTRa) apply_kernel(double* S, int ld, Cols in, Cols out, long long n,
                                                     const Mat M, const int* stop) {
    if (halted(stop)) return;
    const double* Mc = DEV ? c_coef : M.v;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    int* s_in = reinterpret_cast<int*>(smem + 64);
    int* s_out = s_in + kMaxQ;
    double* ring = reinterpret_cast<double*>(smem + 512);
    const size_t te = (size_t)kTRa * ld;
    const int a = in.n;
    stage_cols(in, s_in);
    stage_cols(out, s_out);
    const TileWalk<kTRa> W(n, ld);
    const int row = threadIdx.x;
    if (row == 0) {
        for (int s = 0; s < kEStages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (long long j = 0; j < min((long long)kEStages, W.mine); ++j)
            W.issue(j, (int)j, bar, ring + j * te, S, nullptr);
    }
    __syncthreads();
    for (long long j = 0; j < W.mine; ++j) {
        const int s = (int)(j % kEStages);
        mbar_wait(&bar[s], (uint32_t)((j / kEStages) & 1));
        double* T = ring + s * te;
        const int nr = W.rows(j);
        if (row < nr) {
            double* t = T + row * ld;
            double acc[C];
#pragma unroll
            for (int q = 0; q < C; ++q) acc[q] = 0.0;
            for (int l = 0; l < a; ++l) {  // warp-uniform coefficient row l
                const double u = t[s_in[l]];
                const double* Ml = Mc + l * C;
#pragma unroll
                for (int q = 0; q < C; ++q) acc[q] = fma(u, Ml[q], acc[q]);
            }
#pragma unroll
            for (int q = 0; q < C; ++q) t[s_out[q]] = acc[q];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (row == 0) {
            bulk_store(S + W.row0(j) * ld, T, (uint32_t)nr * ld * 8u);
            bulk_commit();
            if (j + kEStages < W.mine) {
                bulk_wait_read();  // the store has read the stage
                W.issue(j + kEStages, s, bar, T, S, nullptr);
            }
        }
    }
    if (row == 0) bulk_wait_all();
}

// Rayleigh-Ritz update of whole rows from the basis B = [X | Z] (q = B.n) with C (q x m):
//   P' = S_Z C_Z,   X' = P' + S_X C_X,   AX' = AS_B C     into Sn (X, P slots) and ASn (X slot).
// Two threads per row, each owning the output columns k = half, half + 2, ... (the row's
// inputs are broadcast reads of the staged tiles); S and AS tiles are staged together
// (kRRStages deep); the two output tiles are single-buffered in shared memory and
// bulk-stored (the W slot of Sn and the W, P slots of ASn carry don't-care values, rewritten
// before they are read).
constexpr int kRRStages = 2;
constexpr int kHalfK = kMaxK / 2;
template <int TR, bool DEV>
__global__ void __launch_bounds__(2 * TR) rr_apply_kernel(const double* S, const double* AS, double* Sn, double* ASn,
                                                          int ld, Cols B, int m, long long n, const Mat C,
                                                          const Vec16 lam, const int* stop,
                                                          const double* __restrict__ dinv, double* rpart) {
    if (halted(stop)) return;
    const double* Cc = DEV ? c_rrC : C.v;
    const double* lamc = DEV ? c_rrlam : lam.v;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    int* s_b = reinterpret_cast<int*>(smem + 64);
    double* outS = reinterpret_cast<double*>(smem + 512);
    const size_t te = (size_t)TR * ld;
    double* outA = outS + te;
    double* ring = outA + te;
    const int q = B.n;
    stage_cols(B, s_b);
    const TileWalk<TR> W(n, ld);
    const int row = threadIdx.x >> 1, half = threadIdx.x & 1;
    double lk[kHalfK];  // lambda of this thread's columns (constant-index parameter reads)
#pragma unroll
    for (int i = 0; i < kHalfK; ++i) lk[i] = half ? lamc[2 * i + 1] : lamc[2 * i];
    double racc[kHalfK];  // ||R_k||^2 of this thread's columns over its rows
#pragma unroll
    for (int i = 0; i < kHalfK; ++i) racc[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRRStages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (long long j = 0; j < min((long long)kRRStages, W.mine); ++j)
            W.issue(j, (int)j, bar, ring + j * 2 * te, S, AS);
    }
    __syncthreads();
    for (long long j = 0; j < W.mine; ++j) {
        const int s = (int)(j % kRRStages);
        mbar_wait(&bar[s], (uint32_t)((j / kRRStages) & 1));
        const double* Ts = ring + s * 2 * te;
        const double* Ta = Ts + te;
        const int nr = W.rows(j);
        double xs[kHalfK], xa[kHalfK];
#pragma unroll
        for (int i = 0; i < kHalfK; ++i) { xs[i] = 0.0; xa[i] = 0.0; }
        if (row < nr) {
            const double* ts = Ts + row * ld;
            const double* ta = Ta + row * ld;
            for (int l = m; l < q; ++l) {  // Z part first: P'
                const double u = ts[s_b[l]], v = ta[s_b[l]];
#pragma unroll
                for (int i = 0; i < kHalfK; ++i) {
                    const int k = half + 2 * i;
                    if (k < m) {
                        xs[i] = fma(u, Cc[l * m + k], xs[i]);
                        xa[i] = fma(v, Cc[l * m + k], xa[i]);
                    }
                }
            }
        }
        if (threadIdx.x == 0) bulk_wait_read();  // the previous tile's stores have read the out tiles
        __syncthreads();
        if (row < nr) {
            const double* ts = Ts + row * ld;
            const double* ta = Ta + row * ld;
#pragma unroll
            for (int i = 0; i < kHalfK; ++i) {
                const int k = half + 2 * i;
                if (k < m) outS[row * ld + 2 * m + k] = xs[i];
            }
            for (int l = 0; l < m; ++l) {
                const double u = ts[s_b[l]], v = ta[s_b[l]];
#pragma unroll
                for (int i = 0; i < kHalfK; ++i) {
                    const int k = half + 2 * i;
                    if (k < m) {
                        xs[i] = fma(u, Cc[l * m + k], xs[i]);
                        xa[i] = fma(v, Cc[l * m + k], xa[i]);
                    }
                }
            }
            // fused residual of the new Ritz pairs: R = AX' - X' diag(lambda), its norms, and
            // the Jacobi-preconditioned W = |D|^-1 R for the next iteration (W slot)
            const double d = dinv ? fabs(__ldg(dinv + W.row0(j) + row)) : 1.0;
#pragma unroll
            for (int i = 0; i < kHalfK; ++i) {
                const int k = half + 2 * i;
                if (k < m) {
                    outS[row * ld + k] = xs[i];
                    outA[row * ld + k] = xa[i];
                    const double r = fma(-lk[i], xs[i], xa[i]);
                    racc[i] = fma(r, r, racc[i]);
                    outS[row * ld + m + k] = d * r;
                }
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t bytes = (uint32_t)nr * ld * 8u;
            bulk_store(Sn + W.row0(j) * ld, outS, bytes);
            bulk_store(ASn + W.row0(j) * ld, outA, bytes);
            bulk_commit();
            if (j + kRRStages < W.mine) W.issue(j + kRRStages, s, bar, ring + s * 2 * te, S, AS);
        }
    }
    // per-CTA residual partials: same-parity lanes folded by shuffles (even offsets), lane 0
    // / 1 hold the warp's even / odd columns, then warps in order
    __shared__ double rred[2 * TR / 32][kMaxK];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < kHalfK; ++i) {
        double v = racc[i];
#pragma unroll
        for (int off = 16; off > 1; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        const int k = lane + 2 * i;
        if (lane < 2 && k < m) rred[wp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < m) {
        double v = 0.0;
        for (int q2 = 0; q2 < 2 * TR / 32; ++q2) v += rred[q2][threadIdx.x];
        rpart[(size_t)blockIdx.x * m + threadIdx.x] = v;
    }
    if (threadIdx.x == 0) bulk_wait_all();
}

// The ring doubles as the row-group reduction buffer after the tile loop.
int gram_stages(int, bool) { return kEStages; }  // deeper rings measured slower (profiles/)
bool gram_ws_on() {
    static const bool on = [] { const char* e = std::getenv("SPARSLA_GRAM_WS"); return !e || std::atoi(e) != 0; }();
    return on;
}
// warp-specialised Gram: as many stages (<= 8) as fit two CTAs per SM (the fixed 296-CTA
// grid is then one wave)
int gram_ws_stages(int ld, bool two) {
    const size_t per = (size_t)kTR * ld * 8 * (two ? 2 : 1);
    const size_t room = 92 * 1024;
    return (int)std::max<size_t>(2, std::min<size_t>(kGwMaxStages, room / per));
}
size_t gram_ws_smem(int ld, bool two, int a, int b) {
    const int tiles = ((a + kTileR - 1) / kTileR) * ((b + kTileR - 1) / kTileR);
    const int ngroups = std::min(kTR, std::max(1, kGwConsumers * 32 / std::max(1, tiles)));
    const size_t ring = (size_t)gram_ws_stages(ld, two) * kTR * ld * 8 * (two ? 2 : 1);
    return 512 + kMaxQ * kMaxQ * 8 + std::max(ring, (size_t)ngroups * a * b * 8);
}
size_t gram_smem(int ld, bool two, int a, int b) {
    const int tiles = ((a + kTileR - 1) / kTileR) * ((b + kTileR - 1) / kTileR);
    const int ngroups = std::min(kTR, std::max(1, kT / std::max(1, tiles)));
    const size_t ring = (size_t)gram_stages(ld, two) * kTR * ld * 8 * (two ? 2 : 1);
    return 512 + kMaxQ * kMaxQ * 8 + std::max(ring, (size_t)ngroups * a * b * 8);
}
size_t apply_smem(int ld) { return 512 + (size_t)kEStages * kTRa * ld * 8; }
// 128-row tiles up to ld = 24 (k <= 8), 64-row tiles above (shared-memory limit)
int rr_rows(int ld) { return ld <= 24 ? 128 : 64; }
size_t rr_apply_smem(int ld) { return 512 + (size_t)(2 + 2 * kRRStages) * rr_rows(ld) * ld * 8; }

// O[i, oc_j] = (add ? O[i, oc_j] : 0) + sum_l U[i, uc_l] M[l, j]  (c = oc.n <= kMaxK).
// The coefficient matrix lives in the kernel's constant bank (uniform broadcast reads);
// every input of a row is read before its outputs are written, so O may alias U.
__global__ void __launch_bounds__(kT) combine_kernel(double* O, int ldo, Cols oc, int add, const double* U, int ldu,
                                                     Cols uc, long long n, const Mat M) {
    __shared__ int s_uc[kMaxQ], s_oc[kMaxQ];
    stage_cols(uc, s_uc);
    stage_cols(oc, s_oc);
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = uc.n, c = oc.n;
    double acc[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) acc[j] = (j < c && add) ? O[i * ldo + s_oc[j]] : 0.0;
    const double* u = U + i * ldu;
    for (int l = 0; l < a; ++l) {
        const double ul = u[s_uc[l]];
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j < c) acc[j] = fma(ul, M.v[l * c + j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < kMaxK; ++j)
        if (j < c) O[i * ldo + s_oc[j]] = acc[j];
}

// R_j = AX_j - lambda_j X_j for j < m: per-CTA partials of ||R_j||^2, and the
// preconditioned residual W_j = R_j / |A_jj| (Jacobi) into columns w0 + j.
__global__ void __launch_bounds__(kT) resid_kernel(double* S, const double* AS, int ld, int m, const Vec16 lam,
                                                   const double* __restrict__ dinv, int w0, long long n,
                                                   double* partial) {
    __shared__ double red[kT / 32][kMaxK];
    double acc[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) acc[j] = 0.0;
    long long r0, r1;
    cta_rows(n, r0, r1);
    for (long long i = r0 + threadIdx.x; i < r1; i += kT) {
        const double d = dinv ? fabs(__ldg(dinv + i)) : 1.0;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j < m) {
                const double r = fma(-lam.v[j], S[i * ld + j], AS[i * ld + j]);
                acc[j] = fma(r, r, acc[j]);
                S[i * ld + w0 + j] = d * r;
            }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
        if (j >= m) break;
        double v = acc[j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if (lane == 0) red[w][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < m) {
        double s = 0.0;
        for (int q = 0; q < kT / 32; ++q) s += red[q][threadIdx.x];
        partial[(size_t)blockIdx.x * m + threadIdx.x] = s;
    }
}

// Per column: largest |v| and its first row index (sign convention).
__global__ void __launch_bounds__(kT) argmax_kernel(const double* S, int ld, int m, long long n, double* pv,
                                                    long long* pi) {
    __shared__ double sv[kT];
    __shared__ long long si[kT];
    long long r0, r1;
    cta_rows(n, r0, r1);
    for (int j = 0; j < m; ++j) {
        double best = -1.0;
        long long bi = -1;
        for (long long i = r0 + threadIdx.x; i < r1; i += kT) {
            const double v = fabs(S[i * ld + j]);
            if (v > best) { best = v; bi = i; }
        }
        sv[threadIdx.x] = best;
        si[threadIdx.x] = bi;
        __syncthreads();
        for (int s = kT / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                const double ov = sv[threadIdx.x + s];
                const long long oi = si[threadIdx.x + s];
                if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi >= 0 && (si[threadIdx.x] < 0 || oi < si[threadIdx.x]))) {
                    sv[threadIdx.x] = ov;
                    si[threadIdx.x] = oi;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            pv[(size_t)blockIdx.x * m + j] = sv[0];
            pi[(size_t)blockIdx.x * m + j] = si[0];
        }
        __syncthreads();
    }
}

// Eq. 4: grad_vals[e] = sum_m g_m v_m[row_e] v_m[col_e], m ascending, in CSR (= canonical
// COO) order; one thread per row, the row's v values held in registers.
__global__ void __launch_bounds__(kT) eig_grad_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                      long long n, const double* __restrict__ V, int k,
                                                      const Vec16 g, double* gv) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double gi[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) gi[j] = j < k ? g.v[j] * __ldg(V + i * k + j) : 0.0;
    const int ke = __ldg(rp + i + 1);
    for (int e = __ldg(rp + i); e < ke; ++e) {
        const double* vc = V + (size_t)__ldg(ci + e) * k;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j < k) s = fma(gi[j], __ldg(vc + j), s);
        gv[e] = s;
    }
}

// max |a_ij - a_ji| over stored entries (pattern symmetry checked too); flags[0] = pattern ok
__global__ void sym_tol_kernel(const int32_t* rp, const int32_t* ci, const double* val, long long n, int* flags,
                               unsigned long long* maxdiff_bits) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double md = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        int lo = rp[j], hi = rp[j + 1];
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ci[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo == rp[j + 1] || ci[lo] != i) { flags[0] = 0; return; }
        const double d = fabs(val[lo] - val[k]);
        md = d > md || d != d ? d : md;
    }
    if (md != md) { flags[0] = 0; return; }
    // non-negative doubles order like their bit patterns
    if (md > 0.0) atomicMax(maxdiff_bits, (unsigned long long)__double_as_longlong(md));
}

// Y[:, out] = A X[:, in] in groups of <= 16 columns (templated register blocks).
bool lanes_off() {
    static const bool off = [] { const char* e = std::getenv("SPARSLA_SPMM_LANES"); return e && std::atoi(e) == 0; }();
    return off;
}

void launch_spmm(const DevCsr* A, const double* X, int ldx, const Cols& in, double* Y, int ldy, const Cols& out,
                 cudaStream_t st, const int* stop = nullptr) {
    const long long n = A->nrows;
    const unsigned g = (unsigned)((n + kT - 1) / kT);
    for (int b = 0; b < in.n; b += 16) {
        Cols ci, co;
        ci.n = co.n = std::min(16, in.n - b);
        bool contig = ci.n % 2 == 0 && in.c[b] % 2 == 0 && out.c[b] % 2 == 0 && ldx % 2 == 0 && ldy % 2 == 0;
        for (int j = 0; j < ci.n; ++j) {
            ci.c[j] = in.c[b + j];
            co.c[j] = out.c[b + j];
            if (j && (ci.c[j] != ci.c[j - 1] + 1 || co.c[j] != co.c[j - 1] + 1)) contig = false;
        }
        if (contig && ci.n >= 4 && !lanes_off()) {  // coalesced lanes-per-row kernel
            const long long rpw = 32 / (ci.n / 2);
            const unsigned gl = (unsigned)((n + rpw * (kT / 32) - 1) / (rpw * (kT / 32)));
            switch (ci.n) {
#define SPARSLA_SPMML(W) \
    case W: spmm_lanes_kernel<W><<<gl, kT, 0, st>>>(A->rp, A->ci, A->val, n, X, ldx, ci.c[0], Y, ldy, co.c[0], stop); break;
                SPARSLA_SPMML(4) SPARSLA_SPMML(6) SPARSLA_SPMML(8) SPARSLA_SPMML(10) SPARSLA_SPMML(12)
                SPARSLA_SPMML(14) SPARSLA_SPMML(16)
#undef SPARSLA_SPMML
                default: fail(SPARSLA_ERR_INTERNAL, "spmm: bad column count");
            }
            CK(cudaGetLastError());
            continue;
        }
        switch (ci.n * 2 + (contig ? 1 : 0)) {
#define SPARSLA_SPMM(W) \
    case 2 * W: spmm_kernel<W, false><<<g, kT, 0, st>>>(A->rp, A->ci, A->val, n, X, ldx, ci, Y, ldy, co, stop); break;
#define SPARSLA_SPMM2(W) \
    SPARSLA_SPMM(W) case 2 * W + 1: spmm_kernel<W, true><<<g, kT, 0, st>>>(A->rp, A->ci, A->val, n, X, ldx, ci, Y, ldy, co, stop); break;
            SPARSLA_SPMM(1) SPARSLA_SPMM2(2) SPARSLA_SPMM(3) SPARSLA_SPMM2(4) SPARSLA_SPMM(5) SPARSLA_SPMM2(6)
            SPARSLA_SPMM(7) SPARSLA_SPMM2(8) SPARSLA_SPMM(9) SPARSLA_SPMM2(10) SPARSLA_SPMM(11) SPARSLA_SPMM2(12)
            SPARSLA_SPMM(13) SPARSLA_SPMM2(14) SPARSLA_SPMM(15) SPARSLA_SPMM2(16)
#undef SPARSLA_SPMM2
#undef SPARSLA_SPMM
            default: fail(SPARSLA_ERR_INTERNAL, "spmm: bad column count");
        }
        CK(cudaGetLastError());
    }
}

// ------------------------------------------------------------ host dense algebra ----
// Cyclic Jacobi eigendecomposition of a symmetric q x q matrix (row-major).  Returns
// eigenvalues ascending in w and the matching orthonormal eigenvectors as the COLUMNS of
// V (row-major q x q).  Quadratically convergent, accurate to working precision for the
// small Rayleigh-Ritz and Gram problems of LOBPCG.
// SPARSLA_EIG_TIMING=1: host-time breakdown of the LOBPCG driver (printed to stderr)
struct EigTiming {
    bool on = false;
    double eig_s = 0, sync_s = 0;
    long long eigs = 0, syncs = 0;
    EigTiming() { const char* e = std::getenv("SPARSLA_EIG_TIMING"); on = e && std::atoi(e) != 0; }
};
EigTiming& eig_timing() { static EigTiming t; return t; }
double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

void sym_eig_impl(int q, std::vector<double> A, std::vector<double>& w, std::vector<double>& V);
void sym_eig(int q, std::vector<double> A, std::vector<double>& w, std::vector<double>& V) {
    EigTiming& T = eig_timing();
    const double t0 = T.on ? now_s() : 0.0;
    sym_eig_impl(q, std::move(A), w, V);
    if (T.on) { T.eig_s += now_s() - t0; ++T.eigs; }
}
void stream_sync_timed(cudaStream_t s) {
    EigTiming& T = eig_timing();
    const double t0 = T.on ? now_s() : 0.0;
    CK(cudaStreamSynchronize(s));
    if (T.on) { T.sync_s += now_s() - t0; ++T.syncs; }
}

void sym_eig_impl(int q, std::vector<double> A, std::vector<double>& w, std::vector<double>& V) {
    V.assign((size_t)q * q, 0.0);
    for (int i = 0; i < q; ++i) V[(size_t)i * q + i] = 1.0;
    auto a = [&](int i, int j) -> double& { return A[(size_t)i * q + j]; };
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int i = 0; i < q; ++i) {
            dia += a(i, i) * a(i, i);
            for (int j = i + 1; j < q; ++j) off += a(i, j) * a(i, j);
        }
        if (off == 0.0 || off <= 1e-32 * dia) break;
        for (int p = 0; p < q - 1; ++p)
            for (int r = p + 1; r < q; ++r) {
                const double apr = a(p, r);
                if (apr == 0.0) continue;
                // after the first sweeps, an element too small to change either diagonal
                // entry in floating point is zeroed without a rotation (the classic cyclic
                // Jacobi threshold rule): the converged sweeps cost O(q^2) instead of O(q^3)
                if (sweep >= 3) {
                    const double g = 100.0 * std::fabs(apr);
                    if (std::fabs(a(p, p)) + g == std::fabs(a(p, p)) && std::fabs(a(r, r)) + g == std::fabs(a(r, r))) {
                        a(p, r) = 0.0;
                        a(r, p) = 0.0;
                        continue;
                    }
                }
                const double theta = (a(r, r) - a(p, p)) / (2.0 * apr);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < q; ++k) {  // columns p, r
                    const double akp = a(k, p), akr = a(k, r);
                    a(k, p) = c * akp - s * akr;
                    a(k, r) = s * akp + c * akr;
                }
                for (int k = 0; k < q; ++k) {  // rows p, r
                    const double apk = a(p, k), ark = a(r, k);
                    a(p, k) = c * apk - s * ark;
                    a(r, k) = s * apk + c * ark;
                }
                a(p, r) = 0.0;
                a(r, p) = 0.0;
                for (int k = 0; k < q; ++k) {
                    const double vkp = V[(size_t)k * q + p], vkr = V[(size_t)k * q + r];
                    V[(size_t)k * q + p] = c * vkp - s * vkr;
                    V[(size_t)k * q + r] = s * vkp + c * vkr;
                }
            }
    }
    std::vector<int> ord(q);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return a(x, x) < a(y, y); });
    w.resize(q);
    std::vector<double> Vs((size_t)q * q);
    for (int j = 0; j < q; ++j) {
        w[j] = a(ord[j], ord[j]);
        for (int i = 0; i < q; ++i) Vs[(size_t)i * q + j] = V[(size_t)i * q + ord[j]];
    }
    V.swap(Vs);
}

Cols cols_range(int b, int e) {
    Cols c;
    c.n = e - b;
    for (int j = 0; j < c.n; ++j) c.c[j] = (unsigned char)(b + j);
    return c;
}
Cols cols_cat(const Cols& x, const Cols& y) {
    Cols c = x;
    for (int j = 0; j < y.n; ++j) c.c[c.n + j] = y.c[j];
    c.n += y.n;
    return c;
}

// --------------------------------------------------------------- LOBPCG driver ------
bool cgs2_always() {
    static const bool on = [] { const char* e = std::getenv("SPARSLA_EIG_CGS2"); return e && std::atoi(e) != 0; }();
    return on;
}

struct Lobpcg {
    DevCsr* A;
    cudaStream_t s;
    long long n;
    int m, ld;
    double *S = nullptr, *AS = nullptr, *Sn = nullptr, *ASn = nullptr;
    double* partial = nullptr;  // [kRedCTAs][kMaxQ*kMaxQ]
    double* gout = nullptr;     // [kMaxQ*kMaxQ]
    unsigned* ticket = nullptr;
    double* h_pin = nullptr;    // pinned [kMaxQ*kMaxQ]
    double* h_part = nullptr;   // pinned per-CTA partials read back for the residual norms
    long long* ipart = nullptr;
    long long spmm_count = 0;

    Lobpcg(DevCsr* A_, int m_) : A(A_), s(A_->stream), n(A_->nrows), m(m_), ld((3 * m_ + 1) & ~1) {
        const size_t el = (size_t)n * ld + 2;
        S = dalloc<double>(el); AS = dalloc<double>(el);
        Sn = dalloc<double>(el); ASn = dalloc<double>(el);
        CK(cudaMemsetAsync(S, 0, el * 8, s)); CK(cudaMemsetAsync(AS, 0, el * 8, s));
        CK(cudaMemsetAsync(Sn, 0, el * 8, s)); CK(cudaMemsetAsync(ASn, 0, el * 8, s));
        partial = dalloc<double>((size_t)kRedCTAs * kMaxQ * kMaxQ);
        gout = dalloc<double>((size_t)kMaxQ * kMaxQ);
        ticket = dalloc<unsigned>(1);
        CK(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
        ipart = dalloc<long long>((size_t)kRedCTAs * kMaxK);
        CK(cudaMallocHost(&h_pin, sizeof(double) * kMaxQ * kMaxQ));
        CK(cudaMallocHost(&h_part, sizeof(double) * kPartRows * kMaxQ));

        // dynamic shared memory up to the opt-in limit minus each kernel's static part
        auto allow = [&](const void* f, const char* what) {
            int optin = 0;
            cuda_check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, A->device), what);
            cudaFuncAttributes fa{};
            cuda_check(cudaFuncGetAttributes(&fa, f), what);
            cuda_check(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            optin - (int)fa.sharedSizeBytes), what);
        };
        allow((const void*)gram_kernel, "gram smem");
        allow((const void*)gram_ws_kernel, "gram smem");
#define SPARSLA_ALLOW(C) allow((const void*)apply_kernel<C, false>, "apply smem"); \
    allow((const void*)apply_kernel<C, true>, "apply smem");
        SPARSLA_FOR_1_32(SPARSLA_ALLOW)
#undef SPARSLA_ALLOW
        allow((const void*)rr_apply_kernel<128, false>, "rr smem");
        allow((const void*)rr_apply_kernel<64, false>, "rr smem");
        allow((const void*)rr_apply_kernel<128, true>, "rr smem");
        allow((const void*)rr_apply_kernel<64, true>, "rr smem");
    }
    ~Lobpcg() {
        DeviceGuard g(A->device, true);
        cudaFree(S); cudaFree(AS); cudaFree(Sn); cudaFree(ASn);
        cudaFree(partial); cudaFree(gout); cudaFree(ticket); cudaFree(ipart);
        if (h_pin) cudaFreeHost(h_pin);
        if (h_part) cudaFreeHost(h_part);

    }
    unsigned grid() const { return (unsigned)((n + kT - 1) / kT); }
    unsigned tile_grid() const {  // persistent over row tiles, 4 CTAs per SM
        const long long nt = (n + kTRa - 1) / kTRa;
        return (unsigned)std::max<long long>(1, std::min<long long>(nt, 4LL * 148));
    }

    // G = U_uc^T V_vc (host, row-major a x b); U, V are S / AS buffers (row stride ld)
    // G = U_uc^T V_vc into gout (device); stop: device-resident iteration's halt flag
    void gram_launch(const double* U, const Cols& uc, const double* V, const Cols& vc, double* out,
                     const int* stop = nullptr) {
        if (gram_ws_on())
            gram_ws_kernel<<<kRedCTAs, (kGwConsumers + 1) * 32, gram_ws_smem(ld, U != V, uc.n, vc.n), s>>>(
                U, V, ld, uc, vc, n, partial, ticket, out, gram_ws_stages(ld, U != V), stop);
        else
            gram_kernel<<<kRedCTAs, kT, gram_smem(ld, U != V, uc.n, vc.n), s>>>(U, V, ld, uc, vc, n, partial, ticket,
                                                                          out, gram_stages(ld, U != V), stop);
        const int ab = uc.n * vc.n;
        gram_finish_kernel<<<(unsigned)((ab + 31) / 32), 256, 0, s>>>(partial, kRedCTAs, ab, out, stop);
        CK(cudaGetLastError());
    }
    std::vector<double> gram(const double* U, const Cols& uc, const double* V, const Cols& vc) {
        const int ab = uc.n * vc.n;
        std::vector<double> G(ab, 0.0);
        if (ab == 0 || n == 0) return G;
        gram_launch(U, uc, V, vc, gout);
        CK(cudaMemcpyAsync(h_pin, gout, ab * sizeof(double), cudaMemcpyDeviceToHost, s));
        stream_sync_timed(s);
        std::memcpy(G.data(), h_pin, ab * sizeof(double));
        return G;
    }
    // in place: S[:, out] = S[:, in] M
    void apply(const Cols& in, const Cols& out, const std::vector<double>& M) {
        if (out.n == 0 || n == 0) return;
        Mat Mt;
        std::memset(&Mt, 0, sizeof(Mt));
        std::copy(M.begin(), M.end(), Mt.v);
        apply_launch<false>(in, out, Mt);
    }
    // DEV: coefficients already in c_coef (device-resident iteration)
    template <bool DEV>
    void apply_launch(const Cols& in, const Cols& out, const Mat& Mt, const int* stop = nullptr) {
        const unsigned g = tile_grid();
        const size_t sm = apply_smem(ld);
        switch (out.n) {
#define SPARSLA_APPLY(C) case C: apply_kernel<C, DEV><<<g, kTRa, sm, s>>>(S, ld, in, out, n, Mt, stop); break;
            SPARSLA_FOR_1_32(SPARSLA_APPLY)
#undef SPARSLA_APPLY
            default: fail(SPARSLA_ERR_INTERNAL, "apply: more than 32 output columns");
        }
        CK(cudaGetLastError());
    }
    void spmm(const double* X, const Cols& in, double* Y) {
        if (in.n == 0 || n == 0) return;
        launch_spmm(A, X, ld, in, Y, ld, in, s);
        ++spmm_count;
    }
    std::vector<double> resid(const std::vector<double>& lam, const double* dinv) {
        Vec16 L{};
        for (int j = 0; j < m; ++j) L.v[j] = lam[j];
        resid_kernel<<<kRedCTAs, kT, 0, s>>>(S, AS, ld, m, L, dinv, m, n, partial);
        CK(cudaGetLastError());
        const double* h = h_part;  // pinned: no pageable staging copy on this per-iteration readback
        CK(cudaMemcpyAsync(h_part, partial, (size_t)kRedCTAs * m * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<double> r(m, 0.0);
        for (int p = 0; p < kRedCTAs; ++p)
            for (int j = 0; j < m; ++j) r[j] += h[(size_t)p * m + j];
        for (auto& v : r) v = std::sqrt(v);
        return r;
    }

    // Orthonormalise the columns Z of S against the orthonormal columns B and among
    // themselves.  One pass = ONE Gram launch ([B Z]^T Z) + ONE in-place apply launch:
    // the block Gram-Schmidt step Z - B Y (Y = B^T Z) and the SVQB step (Stathopoulos & Wu)
    // are composed in the small space, Gram(Z - B Y) = Z^T Z - Y^T Y, T = D U sigma^-1/2, and
    // applied at once as Z' = [B Z] [[-Y T]; [T]].  Two passes (CGS2 + SVQB2): the second
    // pass sees an almost orthonormal block, so its Gram has no cancellation.  Directions
    // whose norm after orthogonalisation falls below the drop rule are removed;
    // the survivors are a prefix of Z's column slots.
    Cols ortho(const Cols& B, const Cols& Z) {
        Cols z = Z;
        for (int pass = 0; pass < 2 && z.n > 0; ++pass) {
            const int b = B.n, w = z.n;
            const Cols BZ = cols_cat(B, z);
            const std::vector<double> G = gram(S, BZ, S, z);  // (b + w) x w
            std::vector<double> H((size_t)w * w);
            for (int i = 0; i < w; ++i)
                for (int j = 0; j < w; ++j) {
                    double h = G[(size_t)(b + i) * w + j];
                    for (int l = 0; l < b; ++l) h -= G[(size_t)l * w + i] * G[(size_t)l * w + j];
                    H[(size_t)i * w + j] = h;
                }
            // pass 0 subtracts B's component in the small space (cancellation ~ eps / rho^2
            // for a relative remaining norm rho): drop rho < 1e-7 there; pass 1 applies the
            // SPEC rule (norm after orthogonalisation < 1e-12 relative)
            const double rel = pass == 0 ? 1e-14 : 1e-24;
            std::vector<double> D(w, 0.0);
            for (int i = 0; i < w; ++i) {
                const double h0 = G[(size_t)(b + i) * w + i], h = H[(size_t)i * w + i];
                if (std::isfinite(h) && h > 1e-300 && h > rel * h0) D[i] = 1.0 / std::sqrt(h);
            }
            std::vector<double> K((size_t)w * w);
            for (int i = 0; i < w; ++i)
                for (int j = 0; j < w; ++j)
                    K[(size_t)i * w + j] = D[i] * 0.5 * (H[(size_t)i * w + j] + H[(size_t)j * w + i]) * D[j];
            std::vector<double> sig, U;
            sym_eig(w, K, sig, U);
            const double smax = std::max(sig.empty() ? 0.0 : sig.back(), 0.0);
            std::vector<int> keep;
            for (int j = w - 1; j >= 0; --j)
                if (sig[j] > rel * smax && sig[j] > 0.0) keep.push_back(j);
            const int w2 = (int)keep.size();
            std::vector<double> T((size_t)w * w2);
            for (int i = 0; i < w; ++i)
                for (int c = 0; c < w2; ++c) T[(size_t)i * w2 + c] = D[i] * U[(size_t)i * w + keep[c]] / std::sqrt(sig[keep[c]]);
            std::vector<double> M((size_t)(b + w) * w2, 0.0);
            for (int l = 0; l < b; ++l)  // -Y T
                for (int c = 0; c < w2; ++c) {
                    double v = 0.0;
                    for (int i = 0; i < w; ++i) v += G[(size_t)l * w + i] * T[(size_t)i * w2 + c];
                    M[(size_t)l * w2 + c] = -v;
                }
            for (int i = 0; i < w; ++i)
                for (int c = 0; c < w2; ++c) M[(size_t)(b + i) * w2 + c] = T[(size_t)i * w2 + c];
            Cols out = z;
            out.n = w2;
            apply(BZ, out, M);
            z = out;
            // "Twice is enough" (Kahan / Parlett): when no column lost more than half of its
            // norm to B and the normalised Gram is well conditioned, the first pass is already
            // orthonormal to working precision and the second is skipped (SPARSLA_EIG_CGS2=1
            // forces it).
            if (pass == 0 && !cgs2_always()) {
                double worst = 1.0;
                for (int i = 0; i < w; ++i) {
                    const double h0 = G[(size_t)(b + i) * w + i], h = H[(size_t)i * w + i];
                    worst = std::min(worst, h0 > 0 ? h / h0 : 0.0);
                }
                const double smin = sig.empty() ? 0.0 : sig.front();
                if (w2 == w && worst > 0.25 && smin > 1e-6 * smax) break;
            }
        }
        return z;
    }

    // Rayleigh-Ritz on the orthonormal basis S_B, B = [X | Z] (AS_B = A S_B): one Gram launch
    // and one fused update launch writing X', AX', P' into Sn / ASn — plus the new pairs'
    // residual norms and W = |D|^-1 (AX' - X' Lambda) for the next iteration — then swap.
    // rr_apply over basis columns B (DEV: coefficients in c_rrC / c_rrlam); returns its grid
    template <bool DEV>
    unsigned rr_launch(const Cols& B, const Mat& C, const Vec16& L, const double* dinv, const int* stop = nullptr) {
        const int tr = rr_rows(ld);
        const unsigned g = (unsigned)std::max<long long>(1, std::min<long long>((n + tr - 1) / tr, 4LL * 148));
        if (tr == 128)
            rr_apply_kernel<128, DEV><<<g, 256, rr_apply_smem(ld), s>>>(S, AS, Sn, ASn, ld, B, m, n, C, L, stop, dinv,
                                                                         partial);
        else
            rr_apply_kernel<64, DEV><<<g, 128, rr_apply_smem(ld), s>>>(S, AS, Sn, ASn, ld, B, m, n, C, L, stop, dinv,
                                                                        partial);
        CK(cudaGetLastError());
        return g;
    }
    void rayleigh_ritz(const Cols& B, std::vector<double>& lam, const double* dinv, std::vector<double>& res) {
        const int q = B.n;
        std::vector<double> G = gram(S, B, AS, B);
        for (int i = 0; i < q; ++i)
            for (int j = i + 1; j < q; ++j) {
                const double h = 0.5 * (G[(size_t)i * q + j] + G[(size_t)j * q + i]);
                G[(size_t)i * q + j] = G[(size_t)j * q + i] = h;
            }
        std::vector<double> th, U;
        sym_eig(q, G, th, U);
        Mat C;
        std::memset(&C, 0, sizeof(C));
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < m; ++j) C.v[i * m + j] = U[(size_t)i * q + j];
        Vec16 L{};
        for (int j = 0; j < m; ++j) L.v[j] = th[j];
        res.assign(m, 0.0);
        if (n > 0) {
            const unsigned g = rr_launch<false>(B, C, L, dinv);
            const double* h = h_part;
            CK(cudaMemcpyAsync(h_part, partial, (size_t)g * m * sizeof(double), cudaMemcpyDeviceToHost, s));
            stream_sync_timed(s);
            for (unsigned p = 0; p < g; ++p)
                for (int j = 0; j < m; ++j) res[j] += h[(size_t)p * m + j];
            for (auto& v : res) v = std::sqrt(v);
        }
        std::swap(S, Sn);
        std::swap(AS, ASn);
        lam.assign(th.begin(), th.begin() + m);
    }
};

// ------------------------------------------------ device-resident LOBPCG iteration ----
// The host driver above synchronises three times per iteration (two Gram read-backs and the
// residual norms) and solves the small dense problems on the host.  Here every decision of
// an iteration — soft locking, the CGS2 + SVQB orthogonalisation with its drop rule and
// "twice is enough" test, the Rayleigh-Ritz eigenproblem, termination — runs in one-CTA
// kernels on the device, the block kernels take fixed column lists (X | W | P) with the
// inactive directions expressed as zero / identity coefficients, and two iterations are one
// CUDA graph (S <-> Sn ping-pong).  The host only polls the stop flag, one graph behind.
// Same algorithm as the host driver; the small eigenproblems use a parallel (round-robin)
// cyclic Jacobi instead of the serial one, so results agree to rounding (tolerance parity,
// like the rest of this module).
struct EigDevState {
    int done;    // solve stopped: every later kernel exits at entry
    int halt1;   // done, or the second orthogonalisation pass is not needed
    int it, have_p, cur;  // completed iterations, P block present, buffer pair holding S (0/1)
    int nza;     // active Z directions (indices into the 2m W|P slots); after ortho: survivors
    int za[2 * kMaxK];
    int m, k, cgs2;
    int nspmm;   // SpMMs executed (one per iteration that ran)
    int jac_sweeps_max;  // largest Jacobi sweep count of the small solves (diagnostics)
    long long max_iter;
    double tol;
    double res[kMaxK], lam[kMaxK];
};

constexpr int kEigThreads = 256;
constexpr int kQ = kMaxQ;  // leading dimension of the small matrices in shared memory

// Parallel cyclic Jacobi on the q x q symmetric matrix A (shared, ld kQ) by one CTA: q/2
// disjoint rotations per step in round-robin order, each element updated from its 2 x 2
// block of the previous step.  On return w[0..q) ascending and the matching eigenvectors
// in the columns of U (ld kQ).  Work buffers A2, V, V2 (q x q, ld kQ), small arrays in sm.
struct JacobiSmem {
    double alpha[kQ], beta[kQ], red[kEigThreads / 32][2];
    int part[kQ], zero[kQ];
    int sweeps;
};
constexpr int kJacobiSweeps = 30;
__device__ void block_sym_eig(int q, double* A, double* A2, double* V, double* V2, double* w, double* U,
                              JacobiSmem& J) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < q * q; e += nt) V[(e / q) * kQ + e % q] = (e / q == e % q) ? 1.0 : 0.0;
    if (tid == 0) J.sweeps = 0;
    const int qq = q + (q & 1);
    __syncthreads();
    for (int sweep = 0; sweep < kJacobiSweeps && q > 1; ++sweep) {
        // convergence: off-diagonal vs diagonal mass (same rule as the host solver)
        double off = 0.0, dia = 0.0;
        for (int e = tid; e < q * q; e += nt) {
            const int i = e / q, j = e % q;
            const double a = A[i * kQ + j];
            if (i == j) dia += a * a;
            else if (i < j) off += a * a;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            dia += __shfl_xor_sync(0xffffffffu, dia, o);
        }
        if ((tid & 31) == 0) { J.red[tid >> 5][0] = off; J.red[tid >> 5][1] = dia; }
        __syncthreads();
        off = 0.0; dia = 0.0;
        for (int wv = 0; wv < nt / 32; ++wv) { off += J.red[wv][0]; dia += J.red[wv][1]; }
        __syncthreads();
        if (off == 0.0 || off <= 1e-30 * dia) break;  // off-diagonal below 1e-15 of the diagonal (norm)
        if (tid == 0) J.sweeps = sweep + 1;
        for (int step = 0; step < qq - 1; ++step) {
            if (tid < qq / 2) {
                auto player = [&](int sl) { return sl == 0 ? 0 : 1 + (sl - 1 + step) % (qq - 1); };
                const int i0 = player(tid), j0 = player(qq - 1 - tid);
                const int lo = min(i0, j0), hi = max(i0, j0);
                if (hi < q) {
                    const double apr = A[lo * kQ + hi];
                    bool rot = apr != 0.0, zero = false;
                    if (rot && sweep >= 3) {  // threshold rule: too small to change the diagonal
                        const double g = 100.0 * fabs(apr);
                        if (fabs(A[lo * kQ + lo]) + g == fabs(A[lo * kQ + lo]) &&
                            fabs(A[hi * kQ + hi]) + g == fabs(A[hi * kQ + hi])) { rot = false; zero = true; }
                    }
                    if (rot) {
                        const double theta = (A[hi * kQ + hi] - A[lo * kQ + lo]) / (2.0 * apr);
                        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                        J.alpha[lo] = c; J.beta[lo] = -s; J.part[lo] = hi;
                        J.alpha[hi] = c; J.beta[hi] = s; J.part[hi] = lo;
                    } else {
                        J.alpha[lo] = 1.0; J.beta[lo] = 0.0; J.part[lo] = lo;
                        J.alpha[hi] = 1.0; J.beta[hi] = 0.0; J.part[hi] = hi;
                    }
                    J.zero[lo] = (rot || zero) ? hi : -1;
                    J.zero[hi] = (rot || zero) ? lo : -1;
                } else if (lo < q) {  // paired with the padding index
                    J.alpha[lo] = 1.0; J.beta[lo] = 0.0; J.part[lo] = lo; J.zero[lo] = -1;
                }
            }
            __syncthreads();
            for (int e = tid; e < q * q; e += nt) {
                const int i = e / q, j = e % q;
                const double ai = J.alpha[i], bi = J.beta[i], aj = J.alpha[j], bj = J.beta[j];
                const int pi = J.part[i], pj = J.part[j];
                double v = ai * (aj * A[i * kQ + j] + bj * A[i * kQ + pj]) +
                           bi * (aj * A[pi * kQ + j] + bj * A[pi * kQ + pj]);
                if (J.zero[i] == j) v = 0.0;  // the annihilated (or negligible) pair element
                A2[i * kQ + j] = v;
                V2[i * kQ + j] = aj * V[i * kQ + j] + bj * V[i * kQ + pj];
            }
            __syncthreads();
            double* t = A; A = A2; A2 = t;
            t = V; V = V2; V2 = t;
        }
    }
    // ascending order, ties by index (as std::stable_sort on the diagonal)
    for (int i = tid; i < q; i += nt) {
        const double wi = A[i * kQ + i];
        int r = 0;
        for (int j = 0; j < q; ++j) {
            const double wj = A[j * kQ + j];
            r += (wj < wi || (wj == wi && j < i)) ? 1 : 0;
        }
        w[r] = wi;
        for (int row = 0; row < q; ++row) U[row * kQ + r] = V[row * kQ + i];
    }
    __syncthreads();
}

struct EigSmem {  // dynamic shared memory of the small-problem kernels
    double A[kQ * kQ], A2[kQ * kQ], V[kQ * kQ], V2[kQ * kQ], U[kQ * kQ];
    double H[kQ * kQ];
    double w[kQ], D[kQ], h0[kQ];
    int keep[kQ];
    JacobiSmem J;
    int w2, skip;
};

// soft locking and termination for the coming iteration (host driver: top of its loop)
__global__ void eig_decide_kernel(EigDevState* st) {
    if (threadIdx.x != 0 || st->done) return;
    const int m = st->m;
    int n = 0;
    bool wanted_done = true;
    for (int j = 0; j < m; ++j) {
        const bool conv = st->res[j] <= st->tol;
        if (!conv) st->za[n++] = j;  // W_j
        if (j < st->k && !conv) wanted_done = false;
    }
    if (wanted_done || n == 0 || st->it >= st->max_iter) {
        st->done = 1;
        st->halt1 = 1;
        return;
    }
    if (st->have_p) {
        const int nw = n;
        for (int t = 0; t < nw; ++t) st->za[n++] = m + st->za[t];  // P slot of each active W
    }
    st->nza = n;
    st->halt1 = 0;
}

// One CGS + SVQB orthogonalisation pass of the active Z directions against X (host driver:
// Lobpcg::ortho).  G = [X | W | P]^T [W | P] (3m x 2m).  Writes the coefficients of the in-place
// transform S[:, W|P] = S[:, X|W|P] M (3m x 2m, row-major) to Mout; survivors stay a prefix of
// the active list, dropped and inactive slots get identity columns.
__global__ void __launch_bounds__(kEigThreads) eig_ortho_kernel(EigDevState* st, const double* G, double* Mout,
                                                                int pass) {
    if (pass == 0 ? st->done : st->halt1) return;
    extern __shared__ __align__(16) unsigned char esm[];
    EigSmem& E = *reinterpret_cast<EigSmem*>(esm);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int m = st->m, b = m, w = st->nza, zc = 2 * m;
    const int* za = st->za;
    const double rel = pass == 0 ? 1e-14 : 1e-24;
    // H = G_ZZ - G_XZ^T G_XZ (host order: subtract l = 0, 1, ...)
    for (int e = tid; e < w * w; e += nt) {
        const int i = e / w, j = e % w;
        double h = G[(b + za[i]) * zc + za[j]];
        for (int l = 0; l < b; ++l) h -= G[l * zc + za[i]] * G[l * zc + za[j]];
        E.H[i * kQ + j] = h;
    }
    __syncthreads();
    for (int i = tid; i < w; i += nt) {
        const double h0 = G[(b + za[i]) * zc + za[i]], h = E.H[i * kQ + i];
        E.h0[i] = h0;
        E.D[i] = (isfinite(h) && h > 1e-300 && h > rel * h0) ? 1.0 / sqrt(h) : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < w * w; e += nt) {
        const int i = e / w, j = e % w;
        E.A[i * kQ + j] = E.D[i] * 0.5 * (E.H[i * kQ + j] + E.H[j * kQ + i]) * E.D[j];
    }
    __syncthreads();
    block_sym_eig(w, E.A, E.A2, E.V, E.V2, E.w, E.U, E.J);
    if (tid == 0) {
        const double smax = fmax(w > 0 ? E.w[w - 1] : 0.0, 0.0);
        int w2 = 0;
        for (int j = w - 1; j >= 0; --j)
            if (E.w[j] > rel * smax && E.w[j] > 0.0) E.keep[w2++] = j;
        E.w2 = w2;
        int skip = 0;
        if (pass == 0 && !st->cgs2) {
            double worst = 1.0;
            for (int i = 0; i < w; ++i) worst = fmin(worst, E.h0[i] > 0 ? E.H[i * kQ + i] / E.h0[i] : 0.0);
            const double smin = w > 0 ? E.w[0] : 0.0;
            skip = (w2 == w && worst > 0.25 && smin > 1e-6 * smax) ? 1 : 0;
        }
        E.skip = skip;
    }
    __syncthreads();
    const int w2 = E.w2;
    // T (w x w2) = D U_keep sigma^-1/2, into A2
    for (int e = tid; e < w * w2; e += nt) {
        const int i = e / w2, c = e % w2;
        E.A2[i * kQ + c] = E.D[i] * E.U[i * kQ + E.keep[c]] / sqrt(E.w[E.keep[c]]);
    }
    for (int e = tid; e < 3 * m * zc; e += nt) Mout[e] = 0.0;
    __syncthreads();
    for (int e = tid; e < (b + w) * w2; e += nt) {
        const int r = e / w2, c = e % w2, o = za[c];  // output slot of survivor c
        double v;
        if (r < b) {  // -Y T
            v = 0.0;
            for (int i = 0; i < w; ++i) v += G[r * zc + za[i]] * E.A2[i * kQ + c];
            v = -v;
            Mout[r * zc + o] = v;
        } else {
            Mout[(b + za[r - b]) * zc + o] = E.A2[(r - b) * kQ + c];
        }
    }
    __syncthreads();
    for (int o = tid; o < zc; o += nt) {  // slots that are not survivors keep their column
        bool surv = false;
        for (int c = 0; c < w2; ++c) surv |= za[c] == o;
        if (!surv) Mout[(b + o) * zc + o] = 1.0;
    }
    __syncthreads();
    if (tid == 0) {
        st->nza = w2;
        if (pass == 0) st->halt1 = (E.skip || w2 == 0) ? 1 : 0;
    }
}

// Rayleigh-Ritz on the orthonormal basis X | surviving Z: G = [X|W|P]^T A [X|W|P] (3m x 3m)
// restricted to the active slots; writes C (3m x m, zero rows for inactive slots) and the
// m smallest Ritz values.
__global__ void __launch_bounds__(kEigThreads) eig_rr_kernel(EigDevState* st, const double* G, double* Cout,
                                                             double* lamout) {
    if (st->done) return;
    extern __shared__ __align__(16) unsigned char esm[];
    EigSmem& E = *reinterpret_cast<EigSmem*>(esm);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int m = st->m, q = m + st->nza, ac = 3 * m;
    __shared__ int slot[kQ];
    for (int i = tid; i < q; i += nt) slot[i] = i < m ? i : m + st->za[i - m];
    __syncthreads();
    for (int e = tid; e < q * q; e += nt) {
        const int i = e / q, j = e % q;
        const double gij = G[slot[i] * ac + slot[j]], gji = G[slot[j] * ac + slot[i]];
        E.A[i * kQ + j] = i == j ? gij : 0.5 * (i < j ? gij + gji : gji + gij);
    }
    __syncthreads();
    block_sym_eig(q, E.A, E.A2, E.V, E.V2, E.w, E.U, E.J);
    if (tid == 0) st->jac_sweeps_max = max(st->jac_sweeps_max, E.J.sweeps);
    for (int e = tid; e < ac * m; e += nt) Cout[e] = 0.0;
    __syncthreads();
    for (int e = tid; e < q * m; e += nt) {
        const int i = e / m, j = e % m;
        Cout[slot[i] * m + j] = E.U[i * kQ + j];
    }
    for (int j = tid; j < m; j += nt) {
        lamout[j] = E.w[j];
        st->lam[j] = E.w[j];
    }
}

// residual norms of the new pairs (rr_apply's per-CTA partials, summed in CTA order) and
// the end-of-iteration bookkeeping
__global__ void __launch_bounds__(kEigThreads) eig_post_kernel(EigDevState* st, const double* partial, int g) {
    if (st->done) return;
    const int m = st->m;
    __shared__ double part[kEigThreads][kMaxK];
    // fixed two-level order: thread t sums CTAs t, t + 256, ...; then threads in order
    for (int j = 0; j < m; ++j) {
        double r = 0.0;
        for (int p = threadIdx.x; p < g; p += blockDim.x) r += partial[(size_t)p * m + j];
        part[threadIdx.x][j] = r;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        double r = 0.0;
        for (int t = 0; t < (int)blockDim.x; ++t) r += part[t][j];
        st->res[j] = sqrt(r);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        st->cur ^= 1;
        st->nspmm += 1;
        st->have_p = st->nza > 0;
        if (st->nza == 0) { st->done = 1; st->halt1 = 1; }
        else st->it += 1;
    }
}

size_t eig_smem_bytes() { return sizeof(EigSmem); }


// opt-in (SPARSLA_EIG_DEVICE=1): measured slower than the host driver — the one-CTA
// Jacobi of the 18 x 18 Rayleigh-Ritz problem takes ~125 us on the GPU against ~19 us on
// the host (profiles/r02_lobpcg.md)
bool eig_device_on() {
    const char* e = std::getenv("SPARSLA_EIG_DEVICE");
    return e && std::atoi(e) != 0;
}

// Device-resident LOBPCG loop (see above).  Entry: X (and AX, W, res) from the initial
// Rayleigh-Ritz in L.S / L.AS, lam / res on the host.  Exit: L.S / L.AS hold the final basis,
// lam / res / it updated.
const Mat kNoMat{};  // parameter of the DEV launches (coefficients come from the symbols)

void lobpcg_device_loop(Lobpcg& L, int k, double tol, long long max_iter, const double* dinv,
                        std::vector<double>& lam, std::vector<double>& res, long long& it) {
    const int m = L.m;
    cudaStream_t s = L.s;
    static std::once_flag attr_once;
    std::call_once(attr_once, [] {
        CK(cudaFuncSetAttribute(eig_ortho_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)eig_smem_bytes()));
        CK(cudaFuncSetAttribute(eig_rr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)eig_smem_bytes()));
    });
    EigDevState h{};
    h.m = m; h.k = k; h.tol = tol; h.max_iter = max_iter; h.cgs2 = cgs2_always() ? 1 : 0;
    for (int j = 0; j < m; ++j) { h.res[j] = res[j]; h.lam[j] = lam[j]; }
    EigDevState* st = dalloc<EigDevState>(1);
    double* Mbuf = dalloc<double>((size_t)kMaxQ * 2 * kMaxK);
    double* Cbuf = dalloc<double>((size_t)kMaxQ * kMaxK);
    double* lbuf = dalloc<double>(kMaxK);
    EigDevState* hs = nullptr;  // pinned: [2] polled states
    CK(cudaMallocHost(&hs, 2 * sizeof(EigDevState)));
    CK(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, s));
    const Cols All = cols_range(0, 3 * m), Zf = cols_range(m, 3 * m);
    double* b0S = L.S; double* b0A = L.AS; double* b1S = L.Sn; double* b1A = L.ASn;
    const size_t esm = eig_smem_bytes();
    auto iteration = [&](double* S, double* AS, double* Sn, double* ASn) {
        L.S = S; L.AS = AS; L.Sn = Sn; L.ASn = ASn;
        eig_decide_kernel<<<1, 32, 0, s>>>(st);
        for (int pass = 0; pass < 2; ++pass) {
            const int* stop = pass == 0 ? &st->done : &st->halt1;
            L.gram_launch(S, All, S, Zf, L.gout, stop);
            eig_ortho_kernel<<<1, kEigThreads, esm, s>>>(st, L.gout, Mbuf, pass);
            CK(cudaMemcpyToSymbolAsync(c_coef, Mbuf, (size_t)3 * m * 2 * m * sizeof(double), 0,
                                       cudaMemcpyDeviceToDevice, s));
            L.apply_launch<true>(All, Zf, kNoMat, stop);
        }
        launch_spmm(L.A, S, L.ld, Zf, AS, L.ld, Zf, s, &st->done);
        L.gram_launch(S, All, AS, All, L.gout, &st->done);
        eig_rr_kernel<<<1, kEigThreads, esm, s>>>(st, L.gout, Cbuf, lbuf);
        CK(cudaMemcpyToSymbolAsync(c_rrC, Cbuf, (size_t)3 * m * m * sizeof(double), 0, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyToSymbolAsync(c_rrlam, lbuf, m * sizeof(double), 0, cudaMemcpyDeviceToDevice, s));
        const unsigned g = L.rr_launch<true>(All, kNoMat, Vec16{}, dinv, &st->done);
        eig_post_kernel<<<1, kEigThreads, 0, s>>>(st, L.partial, (int)g);
        CK(cudaGetLastError());
    };
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    iteration(b0S, b0A, b1S, b1A);
    iteration(b1S, b1A, b0S, b0A);
    CK(cudaStreamEndCapture(s, &graph));
    cudaGraphExec_t exec;
    CK(cudaGraphInstantiate(&exec, graph, 0));
    CK(cudaGraphDestroy(graph));
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    // launch graphs, poll the stop flag one launch behind
    for (long long i = 0;; ++i) {
        CK(cudaGraphLaunch(exec, s));
        CK(cudaMemcpyAsync(&hs[i & 1], st, sizeof(EigDevState), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ev[i & 1], s));
        if (i >= 1) {
            CK(cudaEventSynchronize(ev[(i - 1) & 1]));
            if (hs[(i - 1) & 1].done) break;
        }
        if (i > 2 * max_iter + 8) break;  // cannot happen: decide stops at max_iter
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(&h, st, sizeof h, cudaMemcpyDeviceToHost));
    cudaEventDestroy(ev[0]); cudaEventDestroy(ev[1]);
    cudaGraphExecDestroy(exec);
    cudaFreeHost(hs);
    cudaFree(st); cudaFree(Mbuf); cudaFree(Cbuf); cudaFree(lbuf);
    // h.cur: the pair that holds the current basis
    L.S = h.cur ? b1S : b0S; L.AS = h.cur ? b1A : b0A;
    L.Sn = h.cur ? b0S : b1S; L.ASn = h.cur ? b0A : b1A;
    lam.assign(h.lam, h.lam + m);
    res.assign(h.res, h.res + m);
    it = h.it;
    L.spmm_count += h.nspmm;
    if (eig_timing().on) std::fprintf(stderr, "[eig device] max Jacobi sweeps of the Rayleigh-Ritz solves: %d\n", h.jac_sweeps_max);
}

struct EigOut {
    std::vector<double> lam, res;
    std::vector<int> conv;
    long long iters = 0, spmm = 0;
    int method = 0;
    int all_conv = 0;
    std::string diag;
};

// Final stage shared by both methods: exact residuals (fresh SpMM), sign convention,
// copy of the first k columns into V (row-major n x k).
void finish(Lobpcg& L, int k, double tol, const double* dinv, EigOut& o, double* V) {
    const Cols Xc = cols_range(0, L.m);
    L.spmm(L.S, Xc, L.AS);
    o.res = L.resid(o.lam, dinv);
    o.res.resize(k);
    o.conv.assign(k, 0);
    int nc = 0;
    for (int j = 0; j < k; ++j) nc += (o.conv[j] = o.res[j] <= tol ? 1 : 0);
    o.all_conv = nc == k;
    // sign: largest-magnitude component positive (first index on ties)
    argmax_kernel<<<kRedCTAs, kT, 0, L.s>>>(L.S, L.ld, L.m, L.n, L.partial, L.ipart);
    CK(cudaGetLastError());
    std::vector<double> pv((size_t)kRedCTAs * L.m);
    std::vector<long long> pi((size_t)kRedCTAs * L.m);
    CK(cudaMemcpyAsync(pv.data(), L.partial, pv.size() * 8, cudaMemcpyDeviceToHost, L.s));
    CK(cudaMemcpyAsync(pi.data(), L.ipart, pi.size() * 8, cudaMemcpyDeviceToHost, L.s));
    CK(cudaStreamSynchronize(L.s));
    std::vector<double> sign(k, 1.0);
    for (int j = 0; j < k; ++j) {
        double bv = -1.0;
        long long bi = -1;
        for (int p = 0; p < kRedCTAs; ++p) {
            const double v = pv[(size_t)p * L.m + j];
            const long long i = pi[(size_t)p * L.m + j];
            if (i >= 0 && (v > bv)) { bv = v; bi = i; }  // CTAs ascend in rows: first max wins
        }
        if (bi >= 0) {
            double val = 0.0;
            CK(cudaMemcpyAsync(&val, L.S + bi * L.ld + j, 8, cudaMemcpyDeviceToHost, L.s));
            CK(cudaStreamSynchronize(L.s));
            sign[j] = val < 0 ? -1.0 : 1.0;
        }
    }
    // V = X_{:, :k} diag(sign), row-major n x k
    std::vector<double> M((size_t)L.m * k, 0.0);
    for (int j = 0; j < k; ++j) M[(size_t)j * k + j] = sign[j];
    if (L.n > 0) {
        Mat Mt;
        std::memset(&Mt, 0, sizeof(Mt));
        std::copy(M.begin(), M.end(), Mt.v);
        combine_kernel<<<L.grid(), kT, 0, L.s>>>(V, k, cols_range(0, k), 0, L.S, L.ld, Xc, L.n, Mt);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(L.s));
    o.spmm = L.spmm_count;
}


int eig_guard(int k) {
    if (const char* e = std::getenv("SPARSLA_EIG_GUARD")) return std::max(0, std::atoi(e));
    (void)k;
    return 0;
}

int dense_threshold() {
    const char* e = std::getenv("SPARSLA_EIG_DENSE_THRESHOLD");
    return e ? std::max(0, std::atoi(e)) : 64;
}

std::mutex& eig_mutex() {  // one LOBPCG at a time per process: coefficient symbols are global
    static std::mutex mu;
    return mu;
}

void eig_smallest(DevCsr* A, int k, double tol, long long max_iter, uint64_t seed, int precond, double* V,
                  EigOut& o) {
    std::lock_guard<std::mutex> lk(eig_mutex());
    const long long n = A->nrows;
    const double* dinv = precond == SPARSLA_PRECOND_JACOBI ? A->jacobi_dinv() : nullptr;
    int m = k;
    if (n <= dense_threshold()) {
        // Rayleigh-Ritz on the whole space (S = I): A is formed column block by column
        // block with the same SpMM kernel, then the n x n symmetric problem is solved.
        o.method = 1;
        const int nn = (int)n;
        std::vector<double> Ad((size_t)nn * nn);
        double *E = dalloc<double>((size_t)nn * nn), *AE = dalloc<double>((size_t)nn * nn);
        eye_kernel<<<(nn + 127) / 128, 128, 0, A->stream>>>(E, nn, nn);
        for (int b = 0; b < nn; b += kMaxQ) {
            const Cols c = cols_range(b, std::min(nn, b + kMaxQ));
            launch_spmm(A, E, nn, c, AE, nn, c, A->stream);
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(Ad.data(), AE, Ad.size() * 8, cudaMemcpyDeviceToHost, A->stream));
        CK(cudaStreamSynchronize(A->stream));
        cudaFree(E); cudaFree(AE);
        std::vector<double> w, U;
        sym_eig(nn, Ad, w, U);
        Lobpcg L(A, m);
        std::vector<double> X((size_t)nn * L.ld, 0.0);
        for (int i = 0; i < nn; ++i)
            for (int j = 0; j < m; ++j) X[(size_t)i * L.ld + j] = U[(size_t)i * nn + j];
        CK(cudaMemcpyAsync(L.S, X.data(), X.size() * 8, cudaMemcpyHostToDevice, A->stream));
        CK(cudaStreamSynchronize(A->stream));
        o.lam.assign(w.begin(), w.begin() + m);
        L.spmm_count = (nn + kMaxQ - 1) / kMaxQ;
        finish(L, k, tol, dinv, o, V);
        o.diag = "dense Rayleigh-Ritz on the full space (n <= dense threshold)";
        return;
    }
    // guard vectors: the block carries g extra Ritz pairs so the k wanted ones converge at the
    // rate of the gap to lambda_{k+g+1} (SPARSLA_EIG_GUARD overrides the default)
    {
        int g = eig_guard(k);
        g = (int)std::min<long long>(g, std::min<long long>(kMaxK - k, n / 4 - k));
        m = k + std::max(0, g);
    }
    Lobpcg L(A, m);
    const Cols Xc = cols_range(0, m);
    eig_init_kernel<<<L.grid(), kT, 0, L.s>>>(L.S, n, L.ld, m, seed);
    CK(cudaGetLastError());
    if (L.ortho(Cols{}, Xc).n < m) fail(SPARSLA_ERR_INTERNAL, "eig_smallest: initial block is rank deficient");
    L.spmm(L.S, Xc, L.AS);
    std::vector<double> lam, res;
    L.rayleigh_ritz(Xc, lam, dinv, res);  // also ||R_j|| and W = |D|^-1 R into the W slot
    bool have_p = false;
    long long it = 0;
    if (eig_device_on()) {  // device-resident iterations (CUDA graph, no host round trips)
        lobpcg_device_loop(L, k, tol, max_iter, dinv, lam, res, it);
    }
    for (; !eig_device_on(); ++it) {
        Cols Z;
        bool wanted_done = true;  // the first k (wanted) pairs decide termination
        for (int j = 0; j < m; ++j) {  // soft locking: only unconverged pairs add directions
            if (!(res[j] <= tol)) Z.c[Z.n++] = (unsigned char)(m + j);
            if (j < k && !(res[j] <= tol)) wanted_done = false;
        }
        if (wanted_done || Z.n == 0 || it >= max_iter) break;
        if (have_p) {
            const int nw = Z.n;
            for (int t = 0; t < nw; ++t) Z.c[Z.n++] = (unsigned char)(m + Z.c[t]);  // P slot = W slot + m
        }
        Z = L.ortho(Xc, Z);
        L.spmm(L.S, Z, L.AS);
        L.rayleigh_ritz(cols_cat(Xc, Z), lam, dinv, res);
        have_p = Z.n > 0;
        if (Z.n == 0) break;  // no new directions: the block cannot improve
    }
    o.iters = it;
    o.lam = lam;
    finish(L, k, tol, dinv, o, V);
    if (eig_timing().on) {
        EigTiming& T = eig_timing();
        std::fprintf(stderr, "[eig timing] host sym_eig %.3f ms (%lld calls), stream syncs %.3f ms (%lld), iterations %lld\n",
                     T.eig_s * 1e3, T.eigs, T.sync_s * 1e3, T.syncs, it);
    }
    char buf[128];
    std::snprintf(buf, sizeof buf, "lobpcg: %lld iterations, block %d (k %d), %s", it, m, k,
                  o.all_conv ? "all pairs converged" : "not all pairs converged");
    o.diag = buf;
}

}  // namespace
}  // namespace sparsla_b200

// =============================================================== C ABI ==============
using namespace sparsla_b200;

struct sparsla_dcsr { DevCsr* A; };

extern "C" {

int sparsla_eig_smallest(sparsla_dcsr* H, int64_t k, const sparsla_eig_options* o, double* lambdas, double* vectors,
                         double* residual_norms, int32_t* pair_converged, sparsla_eig_report* rep, int32_t mem) {
    return guarded([&] {
        if (!H || !o || !rep || !lambdas || !vectors) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DevCsr* A = H->A;
        const long long n = A->nrows;
        if (A->nrows != A->ncols) fail(SPARSLA_ERR_DIMENSION, "eig_smallest: matrix must be square");
        if (k < 1 || k > n) fail(SPARSLA_ERR_INVALID_ARGUMENT, "eig_smallest: need 1 <= k <= n");
        if (k > kMaxK) fail(SPARSLA_ERR_UNSUPPORTED, "eig_smallest: the GPU LOBPCG supports k <= 16");
        if (n > dense_threshold() && 4 * k > n) fail(SPARSLA_ERR_INVALID_ARGUMENT, "eig_smallest: need k <= n/4");
        if (!(o->tol > 0.0)) fail(SPARSLA_ERR_INVALID_ARGUMENT, "eig_smallest: tol must be > 0");
        if (o->max_iter < 1) fail(SPARSLA_ERR_INVALID_ARGUMENT, "eig_smallest: max_iter must be >= 1");
        if (mem != SPARSLA_MEM_HOST && mem != SPARSLA_MEM_DEVICE) fail(SPARSLA_ERR_INVALID_ARGUMENT, "bad mem");
        DeviceGuard g(A->device);
        // symmetric in pattern and values, checked to 1e-12
        {
            int* flags = dalloc<int>(1);
            unsigned long long* md = dalloc<unsigned long long>(1);
            const int one = 1;
            CK(cudaMemcpyAsync(flags, &one, sizeof one, cudaMemcpyHostToDevice, A->stream));
            CK(cudaMemsetAsync(md, 0, 8, A->stream));
            if (n) sym_tol_kernel<<<(unsigned)((n + 255) / 256), 256, 0, A->stream>>>(A->rp, A->ci, A->val, n, flags, md);
            CK(cudaGetLastError());
            int hf = 0;
            unsigned long long hm = 0;
            CK(cudaMemcpyAsync(&hf, flags, sizeof hf, cudaMemcpyDeviceToHost, A->stream));
            CK(cudaMemcpyAsync(&hm, md, sizeof hm, cudaMemcpyDeviceToHost, A->stream));
            CK(cudaStreamSynchronize(A->stream));
            cudaFree(flags); cudaFree(md);
            double dm;
            std::memcpy(&dm, &hm, 8);
            if (!hf || dm > 1e-12)
                fail(SPARSLA_ERR_UNSUPPORTED, "eig_smallest: matrix is not symmetric (pattern and values to 1e-12)");
        }
        double* dV = vectors;
        if (mem == SPARSLA_MEM_HOST) dV = dalloc<double>((size_t)n * k);
        EigOut out;
        try {
            eig_smallest(A, (int)k, o->tol, o->max_iter, o->seed, o->preconditioner, dV, out);
        } catch (...) {
            if (mem == SPARSLA_MEM_HOST) cudaFree(dV);
            throw;
        }
        if (mem == SPARSLA_MEM_HOST) {
            CK(cudaMemcpyAsync(vectors, dV, (size_t)n * k * 8, cudaMemcpyDeviceToHost, A->stream));
            CK(cudaStreamSynchronize(A->stream));
            cudaFree(dV);
        }
        for (int j = 0; j < k; ++j) {
            lambdas[j] = out.lam[j];
            if (residual_norms) residual_norms[j] = out.res[j];
            if (pair_converged) pair_converged[j] = out.conv[j];
        }
        std::memset(rep, 0, sizeof *rep);
        rep->iterations = out.iters;
        rep->spmm_count = out.spmm;
        long long nc = 0;
        for (int c : out.conv) nc += c;
        rep->converged_pairs = nc;
        rep->converged = out.all_conv;
        rep->method = out.method;
        std::snprintf(rep->diagnostic, sizeof rep->diagnostic, "%s", out.diag.c_str());
    });
}

int sparsla_eig_backward(sparsla_dcsr* H, int64_t k, const double* lambdas, const double* vectors,
                         const double* grad_lambdas, double* grad_vals, int32_t mem) {
    return guarded([&] {
        if (!H || !lambdas || !vectors || !grad_lambdas || !grad_vals)
            fail(SPARSLA_ERR_INVALID_ARGUMENT, "null argument");
        DevCsr* A = H->A;
        const long long n = A->nrows;
        if (A->nrows != A->ncols) fail(SPARSLA_ERR_DIMENSION, "eig_backward: matrix must be square");
        if (k < 1 || k > n) fail(SPARSLA_ERR_INVALID_ARGUMENT, "eig_backward: need 1 <= k <= n");
        if (k > kMaxK) fail(SPARSLA_ERR_UNSUPPORTED, "eig_backward: k <= 16");
        if (mem != SPARSLA_MEM_HOST && mem != SPARSLA_MEM_DEVICE) fail(SPARSLA_ERR_INVALID_ARGUMENT, "bad mem");
        // simple eigenvalues (gap > 1e-8 between consecutive lambdas)
        for (int j = 0; j + 1 < k; ++j)
            if (!(lambdas[j + 1] - lambdas[j] > 1e-8))
                fail(SPARSLA_ERR_UNSUPPORTED,
                     "eig_backward: degenerate eigenvalues (gap <= 1e-8): Eq. 4 does not apply");
        Vec16 g{};
        for (int j = 0; j < k; ++j) g.v[j] = grad_lambdas[j];
        DeviceGuard gd(A->device);
        const double* dV = vectors;
        double* ownV = nullptr;
        double* dG = grad_vals;
        if (mem == SPARSLA_MEM_HOST) {
            ownV = dalloc<double>((size_t)n * k);
            CK(cudaMemcpyAsync(ownV, vectors, (size_t)n * k * 8, cudaMemcpyHostToDevice, A->stream));
            dV = ownV;
            dG = dalloc<double>(A->nnz + 1);
        }
        if (n) eig_grad_kernel<<<(unsigned)((n + kT - 1) / kT), kT, 0, A->stream>>>(A->rp, A->ci, n, dV, (int)k, g, dG);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess && mem == SPARSLA_MEM_HOST && A->nnz)
            e = cudaMemcpyAsync(grad_vals, dG, A->nnz * 8, cudaMemcpyDeviceToHost, A->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(A->stream);
        if (mem == SPARSLA_MEM_HOST) { cudaFree(ownV); cudaFree(dG); }
        CK(e);
    });
}

}  // extern "C"
