// device.cu — device CSR handle, Krylov solver driver, adjoint backward and their C ABI.
//
// Single-GPU solve loop (per iteration, all on one stream, captured once into a CUDA graph):
//   CG:        spmv<CG> (q = A p, p.q, alpha)   vec<CG_U1> (x, r, r.z, r.r, beta/conv)
//              vec<CG_U2> (p = z + beta p)                               = 3 launches
//   BiCGStab:  vec<BI_U1> spmv<BICG_V> vec<BI_U2> spmv<BICG_T> vec<BI_U3> = 5 launches
// Every scalar decision is made on the device (kernels.cuh apply_scalar); once the solve
// terminates every kernel exits at entry, so extra graph replays are no-ops and the host
// only polls a pinned flag once per graph (G iterations) — never per iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"
#include "device.hpp"
#include "spmv_xw.cuh"
#include "spmv_dia.cuh"
#include "kernels.cuh"
#include "transport.hpp"

namespace sparsla_b200 {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SPARSLA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

DeviceGuard::DeviceGuard(int dev, bool nothrow) {
    if (nothrow) {  // destructors: never throw (the runtime may already be shut down)
        if (cudaGetDevice(&prev_) != cudaSuccess) { cudaGetLastError(); prev_ = dev; return; }
        if (prev_ != dev && cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
        return;
    }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(SPARSLA_ERR_NO_DEVICE, "no CUDA device visible (the sparsla B200 path has no CPU fallback)");
    }
    if (dev < 0 || dev >= n) fail(SPARSLA_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    CK(cudaGetDevice(&prev_));
    if (prev_ != dev) CK(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() { cudaSetDevice(prev_); }

template <class T>
T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

static inline unsigned grid_for(long long n, int per) { return (unsigned)((n + per - 1) / per); }
static inline long long nchunks_of(long long n) { return (n + kChunk - 1) / kChunk; }

// Staged SpMV variants (RPT rows in flight per thread, STG-deep ring, MINB CTAs/SM).
// Variant 0 is the default; SPARSLA_WS_VARIANT selects another for sweeps.
struct WsVariant {
    int rpt, stg, minb;
    const void* fn[4];      // per SpmvMode
    const void* fn_hub[4];  // same, with the oversized-round bypass compiled in
};
#define WSVW(R, S, M, E, W)                                                                        \
    {R, S, M, {(const void*)spmv_ws_kernel<SPMV_PLAIN, R, S, M, E, W>, (const void*)spmv_ws_kernel<SPMV_CG, R, S, M, E, W>, \
               (const void*)spmv_ws_kernel<SPMV_BICG_V, R, S, M, E, W>, (const void*)spmv_ws_kernel<SPMV_BICG_T, R, S, M, E, W>}, \
              {(const void*)spmv_ws_kernel<SPMV_PLAIN, R, S, M, E, W, true>, (const void*)spmv_ws_kernel<SPMV_CG, R, S, M, E, W, true>, \
               (const void*)spmv_ws_kernel<SPMV_BICG_V, R, S, M, E, W, true>, (const void*)spmv_ws_kernel<SPMV_BICG_T, R, S, M, E, W, true>}}
#define WSV(R, S, M, E) WSVW(R, S, M, E, 8)
#define WPV(D, M)                                                                                 \
    {0, D, M, {(const void*)spmv_wp_kernel<SPMV_PLAIN, D, M>, (const void*)spmv_wp_kernel<SPMV_CG, D, M>,  \
               (const void*)spmv_wp_kernel<SPMV_BICG_V, D, M>, (const void*)spmv_wp_kernel<SPMV_BICG_T, D, M>}, \
              {(const void*)spmv_wp_kernel<SPMV_PLAIN, D, M>, (const void*)spmv_wp_kernel<SPMV_CG, D, M>,  \
               (const void*)spmv_wp_kernel<SPMV_BICG_V, D, M>, (const void*)spmv_wp_kernel<SPMV_BICG_T, D, M>}}
// rpt == 0 marks the warp-pipelined kernel (stg = per-warp ring depth)
// Measured on B200 (tools/spmv_sweep.py, profiles/r01_spmv_sweep.md): variant 0 is the
// fastest on both the 7-point stencil (6.2 TB/s) and the P1 FEM matrix (5.4 TB/s).
// Value-dictionary kernels (for matrices that use staged variant 0: rows of <= 8 entries),
// indexed [hub][mode].  The matrix stream is 5 instead of 12 bytes per entry, so more rows
// must be in flight per SM to keep HBM busy: the variants trade ring depth and CTAs per
// SM (2 rows per thread spilled and ran 2x slower).  SPARSLA_VD_VARIANT selects one (sweeps).
struct VdVariant {
    int rpt, stg, minb;
    const void* fn[4];  // per SpmvMode
};
#define VDV(R, S, M)                                                                                 \
    {R, S, M, {(const void*)spmv_ws_kernel<SPMV_PLAIN, R, S, M, true, 8, false, true>,                \
               (const void*)spmv_ws_kernel<SPMV_CG, R, S, M, true, 8, false, true>,                   \
               (const void*)spmv_ws_kernel<SPMV_BICG_V, R, S, M, true, 8, false, true>,               \
               (const void*)spmv_ws_kernel<SPMV_BICG_T, R, S, M, true, 8, false, true>}}
// Measured on config B (tools/vd_sweep.py, profiles/r01_value_dict.md): 3 CTAs/SM at 72
// registers (no spills) is the best 8-wide point; 4 CTAs/SM (56 registers) spills.  For rows
// of <= 7 entries the 7-wide kernel at 4 CTAs/SM (variant 3, 32 bytes of spills in CG mode)
// is faster still: occupancy beats spill-free code for this gather-latency-bound loop.
#define VDVW(R, S, M, W)                                                                             \
    {R, S, M, {(const void*)spmv_ws_kernel<SPMV_PLAIN, R, S, M, true, W, false, true>,                \
               (const void*)spmv_ws_kernel<SPMV_CG, R, S, M, true, W, false, true>,                   \
               (const void*)spmv_ws_kernel<SPMV_BICG_V, R, S, M, true, W, false, true>,               \
               (const void*)spmv_ws_kernel<SPMV_BICG_T, R, S, M, true, W, false, true>}}
static const VdVariant kVdVariants[] = {VDV(1, 3, 3), VDV(1, 4, 3), VDV(1, 3, 4), VDVW(1, 3, 4, 7), VDVW(1, 3, 3, 7)};
#undef VDVW
#undef VDV
constexpr int kNumVdVariants = sizeof(kVdVariants) / sizeof(kVdVariants[0]);
static int vd_variant() {
    if (const char* e = getenv("SPARSLA_VD_VARIANT")) {
        const int x = atoi(e);
        if (x >= 0 && x < kNumVdVariants) return x;
    }
    return 0;
}

static const WsVariant kWsVariants[] = {WSV(1, 3, 3, true), WSV(1, 4, 2, true), WSV(1, 4, 2, false),
                                        WSV(2, 4, 2, false), WPV(2, 3), WSVW(1, 3, 3, true, 12),
                                        WSVW(1, 4, 2, true, 12)};
#undef WSV
#undef WSVW
#undef WPV
constexpr int kNumWsVariants = sizeof(kWsVariants) / sizeof(kWsVariants[0]);

// Per-matrix choice (measured, profiles/r01_spmv_sweep.md): rows of <= 8 entries -> the
// 8-wide register variant at 3 CTAs/SM; <= 12 -> the 12-wide variant at 2 CTAs/SM (FEM);
// longer -> 8-wide with the held-stage tail path.  SPARSLA_WS_VARIANT overrides (sweeps).
// Long-row split threshold (entries): rows longer than this are summed warp-per-row by
// spmv_longrow_kernel.  Chosen from the row-length histogram: only when the longest row
// exceeds kLongMin AND is far above the typical row (max > 16 x the 99th percentile), so
// stencil / FEM matrices (max/mean ~ 1.3) never take it.  SPARSLA_LONG_ROW=<n> forces a
// threshold, 0 disables.
static constexpr long long kLongMin = 64;
template <class I>
static long long long_row_threshold(long long nrows, const I* h_rp, long long max_row) {
    if (const char* e = getenv("SPARSLA_LONG_ROW")) return std::max(0LL, atoll(e));
    if (max_row <= kLongMin || nrows == 0) return 0;
    // 99th percentile of the row lengths (histogram up to kLongMin, the rest counted above)
    std::vector<long long> hist(kLongMin + 2, 0);
    for (long long i = 0; i < nrows; ++i)
        ++hist[std::min<long long>((long long)h_rp[i + 1] - (long long)h_rp[i], kLongMin + 1)];
    long long acc = 0, p99 = kLongMin + 1;
    for (long long l = 0; l < kLongMin + 2; ++l) {
        acc += hist[l];
        if (acc * 100 >= nrows * 99) { p99 = l; break; }
    }
    if (max_row < 16 * std::max(1LL, p99)) return 0;
    return std::max(kLongMin, 4 * std::max(1LL, p99));
}

static int choose_ws_variant(long long max_row) {
    if (const char* e = getenv("SPARSLA_WS_VARIANT")) {
        const int x = atoi(e);
        if (x >= 0 && x < kNumWsVariants) return x;
    }
    if (max_row <= 8) return 0;
    if (max_row <= 12) return 6;
    return 1;
}

// x-window kernels (spmv_xw.cuh), indexed by variant; `vd` selects the value stream.
// SPARSLA_XW_VARIANT overrides the choice (sweeps).
struct XwVariant {
    int vs;  // value stream: 0 fp64 values, 1 dictionary indices, 2 pair (index in the offset)
    int w, stg, minb;
    const void* fn[4];  // per SpmvMode
    int fix;            // compile-time stage layout (kXwFixCapC / xw_fix_cap_x(fix)), 0 = runtime
};
#define XWV(VS, W, S, M)                                                                            \
    {VS, W, S, M, {(const void*)spmv_xw_kernel<SPMV_PLAIN, S, M, W, VS>, (const void*)spmv_xw_kernel<SPMV_CG, S, M, W, VS>, \
                   (const void*)spmv_xw_kernel<SPMV_BICG_V, S, M, W, VS>, (const void*)spmv_xw_kernel<SPMV_BICG_T, S, M, W, VS>}, 0}
#define XWVF(VS, W, S, M, F)                                                                        \
    {VS, W, S, M, {(const void*)spmv_xw_kernel<SPMV_PLAIN, S, M, W, VS, F>, (const void*)spmv_xw_kernel<SPMV_CG, S, M, W, VS, F>, \
                   (const void*)spmv_xw_kernel<SPMV_BICG_V, S, M, W, VS, F>, (const void*)spmv_xw_kernel<SPMV_BICG_T, S, M, W, VS, F>}, F}
static const XwVariant kXwVariants[] = {XWV(1, 8, 3, 3), XWV(1, 8, 2, 4), XWV(1, 8, 3, 4),
                                        XWV(0, 8, 3, 2), XWV(0, 12, 3, 2), XWV(0, 12, 2, 3),
                                        XWV(2, 8, 3, 3), XWV(2, 8, 2, 4), XWV(2, 8, 3, 4),
                                        XWV(1, 7, 3, 4), XWV(2, 7, 3, 4), XWV(0, 7, 2, 3),
                                        XWVF(2, 7, 3, 4, 1)};
// (measured and dropped: pair 7-wide at 4 stages / 3 CTAs per SM 0.840 ms and at 2 stages /
// 5 CTAs per SM, 40 registers with spills, 0.999 ms — vs 0.792 ms for 3 stages / 4 CTAs;
// a 1408-element fixed x area: same 4 CTAs per SM, same time as 1536)
#undef XWV
#undef XWVF
constexpr int kNumXwVariants = sizeof(kXwVariants) / sizeof(kXwVariants[0]);

static size_t xw_smem_bytes(const DevCsr* A, int var, bool aux) {
    const XwVariant& V = kXwVariants[var];
    const XwLayout L = V.fix ? XwLayout(0, kXwFixCapC, xw_fix_cap_x(V.fix), V.vs, aux) : XwLayout(A->cap_v, A->cap_c, A->cap_x, V.vs, aux);
    return kXwHead + (size_t)V.stg * L.stage;
}

// Variant per value stream and row lengths; -1 = none.
static void choose_xw_variants(DevCsr* A) {
    for (int d = 0; d < 3; ++d) A->xw_var[d] = -1;
    if (!A->xw) return;
    // measured on B200 (tools/xw_sweep.py, profiles/r02_xwin.md): rows of <= 7 entries take the
    // 7-wide kernels, whose warps of exactly-7-entry rows run the guard-free path; longer rows:
    // plain 12-wide 2-stage 3 CTAs/SM, dictionary 8-wide 3 stages 3 CTAs/SM
    const bool w7 = A->max_row <= 7;
    A->xw_var[0] = w7 ? 11 : 5;
    A->xw_var[1] = w7 ? 9 : 0;
    A->xw_var[2] = w7 ? 10 : 8;
    // compile-time layout when the rounds fit it (7-point stencils up to 464^3 and beyond)
    const bool fix = w7 && A->cap_c <= kXwFixCapC && A->cap_x <= xw_fix_cap_x(1);
    if (fix && !getenv("SPARSLA_XW_NOFIX")) A->xw_var[2] = 12;
    if (const char* e = getenv("SPARSLA_XW_VARIANT")) {
        const int x = atoi(e);
        if (x >= 0 && x < kNumXwVariants) {
            const XwVariant& V = kXwVariants[x];
            const bool fits = !V.fix || (A->cap_c <= kXwFixCapC && A->cap_x <= xw_fix_cap_x(V.fix));
            if (fits) A->xw_var[V.vs] = x;
        }
    }
    int dev = A->device, sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    A->sms = sms;
    for (int d = 0; d < 3; ++d) {
        if (A->xw_var[d] < 0) continue;
        for (int aux = 0; aux < 2; ++aux) {
            const int v = A->xw_var[d];
            int per_sm = 0;
            const size_t sm = xw_smem_bytes(A, v, aux);
            if (sm <= 200 * 1024)
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kXwVariants[v].fn[aux ? SPMV_BICG_T : SPMV_CG],
                                                                 kWsThreads, sm));
            A->xw_ctas[d][aux] = sms * per_sm;
        }
        // every mode must fit at least one CTA per SM
        if (A->xw_ctas[d][0] == 0 || A->xw_ctas[d][1] == 0) A->xw_var[d] = -1;
    }
}

size_t ws_smem_bytes(const DevCsr* A, int variant, bool vd = false) {
    if (vd) return 256 + (size_t)kVdVariants[A->vd_var].stg * StageLayout(A->cap_v, A->cap_c, true).stage;
    const WsVariant& V = kWsVariants[variant];
    if (V.rpt == 0) return 1024 + (size_t)(kSpmvThreads / 32) * V.stg * WarpStage(A->cap_v32, A->cap_c32).stage;
    return 256 + (size_t)V.stg * StageLayout(A->cap_v, A->cap_c).stage;
}

static void configure_ws_variants(int device) {
    for (int v = 0; v < kNumWsVariants; ++v)
        for (int m = 0; m < 4; ++m) {
            CK(cudaFuncSetAttribute(kWsVariants[v].fn[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            CK(cudaFuncSetAttribute(kWsVariants[v].fn_hub[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        }
    for (int v = 0; v < kNumVdVariants; ++v)
        for (int m = 0; m < 4; ++m)
            CK(cudaFuncSetAttribute(kVdVariants[v].fn[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int v = 0; v < kNumXwVariants; ++v)
        for (int m = 0; m < 4; ++m)
            CK(cudaFuncSetAttribute(kXwVariants[v].fn[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    (void)device;
}


// ------------------------------------------------------------------ DevCsr ---------
void DevCsr::drop_parked() noexcept {
    std::lock_guard<std::mutex> lk(solver_mu);
    for (auto*& p : parked) { delete p; p = nullptr; }
    ++values_version;  // solvers still running on the old values must not park afterwards
}

DevCsr::~DevCsr() {
    drop_parked();
    DeviceGuard g(device, true);
    cudaFree(rp); cudaFree(ci); cudaFree(val); cudaFree(dinv); cudaFree(ones);
    cudaFree(vidx); cudaFree(vtab);
    cudaFree(long_rows); cudaFree(long_bits); cudaFree(s_rp); cudaFree(s_ci); cudaFree(s_val);
    cudaFree(xw); cudaFree(xwo); cudaFree(xvo); cudaFree(dia); cudaFree(diaw);
    delete[] diac;
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
    delete transpose;
}

static void configure_kernels_once(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    configure_ws_variants(device);
    done.push_back(device);
}

// Value dictionary: when the matrix has at most 256 distinct values (bit patterns), the
// staged SpMV streams a 1-byte index per entry instead of the 8-byte value (constant-
// coefficient stencils: {6, -1}).  The table holds the exact fp64 values, so every product
// and sum is bit-identical.  SPARSLA_VALUE_DICT=0 disables.
static void drop_value_dictionary(DevCsr* A) {
    cudaFree(A->vidx); cudaFree(A->vtab); cudaFree(A->dia); cudaFree(A->diaw);
    delete[] A->diac;
    A->vidx = nullptr; A->vtab = nullptr; A->vd = false;
    A->dia = nullptr; A->diaw = nullptr; A->diac = nullptr; A->dia_npat = 0;
}

// diagonal-warp kernel variants: rounds per step, min CTAs per SM (SPARSLA_DIA_VARIANT)
struct DiaVariant {
    const void* fn[4];
    bool pattern = false;  // spmv_diac_kernel: second argument = the DiaConst patterns
    bool pers = false;     // resident grid looping over chunks (one ticket per CTA)
};
#define DIAV(R, M)                                                                                   \
    {{(const void*)spmv_dia_kernel<SPMV_PLAIN, R, M>, (const void*)spmv_dia_kernel<SPMV_CG, R, M>,      \
      (const void*)spmv_dia_kernel<SPMV_BICG_V, R, M>, (const void*)spmv_dia_kernel<SPMV_BICG_T, R, M>}}
// measured on B200, config B CG SpMV (tools/r02_call34.sh): 1 round / 5 CTAs per SM
// 0.776 ms, 1 / 4: 0.813, 2 / 4: 0.820, 1 / 6: 0.799, 2 / 3: 0.912 (x-window pair: 0.771)
#define DIARV(M)                                                                                     \
    {{(const void*)spmv_diar_kernel<SPMV_PLAIN, M>, (const void*)spmv_diar_kernel<SPMV_CG, M>,          \
      (const void*)spmv_diar_kernel<SPMV_BICG_V, M>, (const void*)spmv_diar_kernel<SPMV_BICG_T, M>}}
#define DIACV(M, U)                                                                                  \
    {{(const void*)spmv_diac_kernel<SPMV_PLAIN, M, U>, (const void*)spmv_diac_kernel<SPMV_CG, M, U>,    \
      (const void*)spmv_diac_kernel<SPMV_BICG_V, M, U>, (const void*)spmv_diac_kernel<SPMV_BICG_T, M, U>}, true}
#define DIACN(M)                                                                                     \
    {{(const void*)spmv_diac_kernel<SPMV_PLAIN, M, 1, false, true>,                                   \
      (const void*)spmv_diac_kernel<SPMV_CG, M, 1, false, true>,                                      \
      (const void*)spmv_diac_kernel<SPMV_BICG_V, M, 1, false, true>,                                  \
      (const void*)spmv_diac_kernel<SPMV_BICG_T, M, 1, false, true>}, true}
#define DIACS(M)                                                                                     \
    {{(const void*)spmv_diac_kernel<SPMV_PLAIN, M, 1, false, false, true>,                            \
      (const void*)spmv_diac_kernel<SPMV_CG, M, 1, false, false, true>,                               \
      (const void*)spmv_diac_kernel<SPMV_BICG_V, M, 1, false, false, true>,                           \
      (const void*)spmv_diac_kernel<SPMV_BICG_T, M, 1, false, false, true>}, true}
#define DIACP(M)                                                                                     \
    {{(const void*)spmv_diac_kernel<SPMV_PLAIN, M, 1, true>, (const void*)spmv_diac_kernel<SPMV_CG, M, 1, true>, \
      (const void*)spmv_diac_kernel<SPMV_BICG_V, M, 1, true>,                                         \
      (const void*)spmv_diac_kernel<SPMV_BICG_T, M, 1, true>}, true, true}
// 3..5: register-pattern kernel (spmv_diar_kernel) at 4 / 5 / 3 CTAs per SM; 6..8: pattern-
// table kernel (spmv_diac_kernel) at 5 / 6 / 4 / 8 CTAs per SM; 10, 11: rounds unrolled by 2
// at 6 / 5 CTAs per SM; 12, 13: persistent at 6 / 8 CTAs per SM; 14, 15: far diagonals
// without L1 allocation at 6 / 8 CTAs per SM; 16, 17: round 0 loaded speculatively with the
// most frequent pattern at 6 / 5 CTAs per SM
static const DiaVariant kDiaVariants[] = {DIAV(1, 5), DIAV(1, 4), DIAV(2, 4), DIARV(4), DIARV(5), DIARV(3),
                                          DIACV(5, 1), DIACV(6, 1), DIACV(4, 1), DIACV(8, 1), DIACV(6, 2), DIACV(5, 2),
                                          DIACP(6), DIACP(8), DIACN(6), DIACN(8), DIACS(6), DIACS(5)};
#undef DIAV
#undef DIARV
#undef DIACV
#undef DIACP
#undef DIACN
#undef DIACS
constexpr int kNumDiaVariants = sizeof(kDiaVariants) / sizeof(kDiaVariants[0]);

// diagonal-warp table (spmv_dia.cuh) from the device CSR and dictionary indices; kept when
// at least 90% of the 32-row warps are structured, and then every SpMV mode takes it.
// Measured on B200 (profiles/r02_dia.md): half the DRAM bytes of the x-window pair kernel,
// config B CG SpMV 0.773 -> 0.68 ms, config D 0.49/0.51 -> 0.43/0.46 ms.  SPARSLA_DIA=0: off.
// Pattern table (spmv_diac_kernel): deduplicate the structured entries by a 64-bit hash of
// their diagonals and values, verify every entry against its slot's representative, and keep
// a 32-bit word per warp plus <= kDiaPatterns patterns (deltas, fp64 values) for the kernel
// parameter.  Any overflow or collision leaves the pattern table off.
static void build_dia_patterns(DevCsr* A, const int32_t* tab, long long nwarps) {
    cudaFree(A->diaw);
    delete[] A->diac;
    A->diaw = nullptr;
    A->diac = nullptr;
    A->dia_npat = 0;
    cudaStream_t s = A->stream;
    unsigned long long* keys = dalloc<unsigned long long>(2 * kDiaHashSlots);
    unsigned long long* rep = keys + kDiaHashSlots;
    int* flags = dalloc<int>(2 + kDiaHashSlots);  // overflow, collision, pid per slot
    int16_t* slot = dalloc<int16_t>(nwarps);
    CK(cudaMemsetAsync(keys, 0, kDiaHashSlots * 8, s));
    CK(cudaMemsetAsync(rep, 0xFF, kDiaHashSlots * 8, s));
    CK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
    unsigned* count = dalloc<unsigned>(kDiaHashSlots);
    CK(cudaMemsetAsync(count, 0, kDiaHashSlots * sizeof(unsigned), s));
    dia_hash_kernel<<<grid_for(nwarps, 256), 256, 0, s>>>(tab, nwarps, keys, rep, slot, flags, count);
    CK(cudaGetLastError());
    std::vector<unsigned long long> hk(2 * kDiaHashSlots);
    std::vector<unsigned> hc(kDiaHashSlots);
    int hf[2] = {0, 0};
    CK(cudaMemcpyAsync(hc.data(), count, kDiaHashSlots * sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hk.data(), keys, hk.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // (representative warp, slot), most frequent pattern first (ties: lowest warp) — the
    // speculative variant loads round 0 with pattern 0
    std::vector<std::pair<unsigned long long, int>> used;
    for (int i = 0; i < kDiaHashSlots; ++i)
        if (hk[i] != 0ull) used.push_back({hk[kDiaHashSlots + i], i});
    std::sort(used.begin(), used.end(), [&](const std::pair<unsigned long long, int>& a,
                                            const std::pair<unsigned long long, int>& b) {
        return hc[a.second] != hc[b.second] ? hc[a.second] > hc[b.second] : a.first < b.first;
    });
    bool ok = !hf[0] && !used.empty() && (int)used.size() <= kDiaPatterns;
    if (ok) {
        std::vector<int> pid_of(kDiaHashSlots, (int)kDiaPidUnstructured);
        std::vector<double> vt(256);
        CK(cudaMemcpyAsync(vt.data(), A->vtab, 256 * 8, cudaMemcpyDeviceToHost, s));
        auto* C = new DiaConst();
        std::memset(C, 0, sizeof(DiaConst));
        for (size_t p = 0; p < used.size(); ++p) {
            int32_t e[kDiaInts];
            CK(cudaMemcpyAsync(e, tab + (long long)used[p].first * kDiaInts, sizeof(e), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const int m = (int)((uint32_t)e[8] >> 24);
            for (int u = 0; u < 7; ++u) {
                C->pat[p].d[u] = e[u];
                const uint32_t w = u < 4 ? (uint32_t)e[7] : (uint32_t)e[8];
                C->pat[p].v[u] = vt[(w >> (8 * (u & 3))) & 0xFFu];
            }
            C->pat[p].d[7] = m;
            pid_of[used[p].second] = (int)p;
        }
        CK(cudaMemcpyAsync(flags + 2, pid_of.data(), kDiaHashSlots * sizeof(int), cudaMemcpyHostToDevice, s));
        uint32_t* words = dalloc<uint32_t>(nwarps);
        dia_compact_kernel<<<grid_for(nwarps, 256), 256, 0, s>>>(tab, nwarps, slot, rep, flags + 2, words, flags + 1);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hf[1] == 0) {
            A->diaw = words;
            A->diac = reinterpret_cast<unsigned char*>(C);
            A->dia_npat = (int)used.size();
        } else {
            cudaFree(words);
            delete C;
        }
    }
    cudaFree(keys);
    cudaFree(flags);
    cudaFree(slot);
    cudaFree(count);
}

static void build_dia(DevCsr* A) {
    cudaFree(A->dia);
    cudaFree(A->diaw);
    delete[] A->diac;
    A->dia = nullptr;
    A->diaw = nullptr;
    A->diac = nullptr;
    A->dia_npat = 0;
    A->dia_frac = 0.0;
    A->dia_bytes = 0;
    const char* e = getenv("SPARSLA_DIA");
    const int dm = e ? atoi(e) : -1;
    A->dia_modes = 0xF;
    if (dm == 0 || !A->vd || A->nrows == 0) return;
    const long long nwarps = nchunks_of(A->nrows) * kChunkRounds * (kSpmvThreads / 32);
    unsigned long long* cnt = dalloc<unsigned long long>(2);
    CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), A->stream));
    int32_t* tab = dalloc<int32_t>(nwarps * kDiaInts);
    dia_build_kernel<<<grid_for(nwarps * 32, 256), 256, 0, A->stream>>>(A->rp, A->ci, A->vidx, A->nrows, nwarps,
                                                                          tab, cnt);
    CK(cudaGetLastError());
    dia_link_kernel<<<grid_for(nwarps, 256), 256, 0, A->stream>>>(tab, nwarps);
    CK(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, A->stream));
    CK(cudaStreamSynchronize(A->stream));
    cudaFree(cnt);
    const long long live = (A->nrows + 31) / 32;
    A->dia_frac = (double)h[0] / (double)live;
    // per SpMV: the live warps' table entries + the unstructured warps' CSR reads
    A->dia_bytes = live * kDiaInts * 4 + (long long)h[1];
    if (A->dia_frac >= 0.9) A->dia = tab;
    else cudaFree(tab);
    if (A->dia) build_dia_patterns(A, A->dia, nwarps);
    // default: the pattern-table kernel at 6 CTAs/SM when the patterns fit (measured on B200,
    // profiles/r02_dia.md: config B CG SpMV 0.573 -> 0.487 ms, D' 0.40/0.43 -> 0.30/0.33 ms)
    A->dia_var = A->diac ? 7 : 0;
    if (const char* v = getenv("SPARSLA_DIA_VARIANT")) {
        const int x = atoi(v);
        if (x >= 0 && x < kNumDiaVariants) A->dia_var = x;
    }
    if (kDiaVariants[A->dia_var].pattern && !A->diac) A->dia_var = 0;  // no pattern table
    int sms = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, A->device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kDiaVariants[A->dia_var].fn[SPMV_CG], kSpmvThreads, 0));
    // prefetch distance in waves of resident CTAs (SPARSLA_DIA_PREFETCH, default 1; 0 = off)
    const char* pe = getenv("SPARSLA_DIA_PREFETCH");
    A->dia_ahead = (pe ? atoi(pe) : 1) * sms * per_sm;
    A->dia_ctas = sms * per_sm;
}

static void build_value_dictionary(DevCsr* A, const double* h_val) {
    drop_value_dictionary(A);
    if (const char* e = getenv("SPARSLA_VALUE_DICT")) if (atoi(e) == 0) return;
    const long long nnz = A->nnz;
    if (nnz == 0) return;
    // distinct bit patterns, per thread, abandoned past 256
    const int nt = std::max(1, host_threads());
    std::vector<std::vector<uint64_t>> seen(nt);
    std::atomic<bool> too_many{false};
    {
        std::vector<std::thread> th;
        const long long per = (nnz + nt - 1) / nt;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                const long long b = t * per, e = std::min(nnz, b + per);
                auto& S = seen[t];
                uint64_t last = 0;
                bool have_last = false;
                for (long long k = b; k < e && !too_many.load(std::memory_order_relaxed); ++k) {
                    uint64_t u;
                    std::memcpy(&u, h_val + k, 8);
                    if (have_last && u == last) continue;
                    if (std::find(S.begin(), S.end(), u) == S.end()) {
                        if (S.size() >= 256) { too_many = true; break; }
                        S.push_back(u);
                    }
                    last = u;
                    have_last = true;
                }
            });
        for (auto& x : th) x.join();
    }
    if (too_many) return;
    std::vector<uint64_t> tab;
    for (auto& S : seen) tab.insert(tab.end(), S.begin(), S.end());
    std::sort(tab.begin(), tab.end());
    tab.erase(std::unique(tab.begin(), tab.end()), tab.end());
    if (tab.size() > 256) return;
    std::vector<uint8_t> idx((size_t)nnz);
    parallel_for(nnz, [&](int64_t b, int64_t e) {
        uint64_t last = ~0ULL;
        uint8_t li = 0;
        for (int64_t k = b; k < e; ++k) {
            uint64_t u;
            std::memcpy(&u, h_val + k, 8);
            if (u != last) {
                li = (uint8_t)(std::lower_bound(tab.begin(), tab.end(), u) - tab.begin());
                last = u;
            }
            idx[(size_t)k] = li;
        }
    });
    std::vector<double> vt(256, 0.0);
    for (size_t i = 0; i < tab.size(); ++i) std::memcpy(&vt[i], &tab[i], 8);
    A->vidx = dalloc<uint8_t>(nnz + 32);
    A->vtab = dalloc<double>(256);
    CK(cudaMemset(A->vidx + nnz, 0, 32));
    CK(memcpy_sync(A->vidx, idx.data(), nnz, cudaMemcpyHostToDevice));
    CK(memcpy_sync(A->vtab, vt.data(), 256 * 8, cudaMemcpyHostToDevice));
    A->vd = true;
    A->nvals = (int)tab.size();
    build_dia(A);
}

// x windows (spmv_xw.cuh): for every 256-row round, up to kXwMax contiguous segments of x
// covering the round's columns.  Columns closer than kXwGap elements join one window; more
// than kXwMax windows are merged across their smallest gaps; a round whose windows exceed
// kXwCapMax elements keeps its most-referenced windows (the other entries read x from
// global memory).  Windows are 16-byte granules inside x.  SPARSLA_XWIN: 0 = off, 1 = on
// when it pays (default: >= 90% of the entries staged, staged elements <= entries; see
// xw_pick for the per-stream choice), 2 = forced (every mode, every stream).
static constexpr long long kXwGap = 32;
static constexpr long long kXwCapMax = 2048;
static int xwin_mode() {
    const char* e = getenv("SPARSLA_XWIN");
    return e ? atoi(e) : 1;
}

static void build_xw_pair(DevCsr* A);

static void drop_xwin(DevCsr* A) {
    cudaFree(A->xw);
    cudaFree(A->xwo);
    cudaFree(A->xvo);
    A->xw = nullptr;
    A->xwo = nullptr;
    A->xvo = nullptr;
    A->cap_x = 0;
    A->xw_var[0] = A->xw_var[1] = A->xw_var[2] = -1;
    A->xw_cover = 0.0;
}

template <class I>
static void build_xwin(DevCsr* A, const I* h_rp, const I* h_ci) {
    drop_xwin(A);
    const int mode = xwin_mode();
    if (mode == 0 || A->nrows == 0 || A->nnz == 0 || A->has_hub || A->nlong > 0 || !A->staged) return;
    const long long nr = (A->nrows + kChunkSlots - 1) / kChunkSlots;
    const long long ncx = A->ncols & ~1LL;
    std::vector<int32_t> desc((size_t)nchunks_of(A->nrows) * kChunkRounds * kXwDescInts, 0);
    std::vector<uint16_t> xoff((size_t)A->nnz + kXwPad, kXwNone);
    std::fill(xoff.end() - kXwPad, xoff.end(), (uint16_t)0);  // read as spares, never used
    std::atomic<long long> covered{0}, staged{0};
    std::atomic<int> capx{0};
    parallel_for(nr, [&](int64_t a, int64_t b) {
        std::vector<std::pair<long long, long long>> iv;
        std::vector<long long> cnt, off;
        long long cov = 0, stg = 0;
        int cx = 0;
        for (int64_t q = a; q < b; ++q) {
            const long long rs = q * kChunkSlots, re = std::min<long long>(rs + kChunkSlots, A->nrows);
            const long long k0 = (long long)h_rp[rs], k1 = (long long)h_rp[re];
            int32_t* d = desc.data() + (size_t)q * kXwDescInts;
            d[12] = (int32_t)k0;
            d[13] = (int32_t)k1;
            d[14] = -1;
            iv.clear();
            bool bad = false;
            for (long long k = k0; k < k1 && !bad; ++k) {
                const long long c = (long long)h_ci[k];
                size_t j = 0;
                while (j < iv.size() && iv[j].second + kXwGap < c) ++j;
                if (j < iv.size() && iv[j].first - kXwGap <= c) {
                    iv[j].first = std::min(iv[j].first, c);
                    iv[j].second = std::max(iv[j].second, c + 1);
                    if (j > 0 && iv[j - 1].second + kXwGap >= iv[j].first) {
                        iv[j - 1].second = std::max(iv[j - 1].second, iv[j].second);
                        iv.erase(iv.begin() + (long)j);
                        --j;
                    }
                    while (j + 1 < iv.size() && iv[j + 1].first - kXwGap <= iv[j].second) {
                        iv[j].second = std::max(iv[j].second, iv[j + 1].second);
                        iv.erase(iv.begin() + (long)j + 1);
                    }
                } else {
                    iv.insert(iv.begin() + (long)j, {c, c + 1});
                    bad = iv.size() > 64;
                }
            }
            if (bad) continue;  // scattered columns: this round gathers from global memory
            while (iv.size() > (size_t)kXwMax) {  // merge across the smallest gap
                size_t jm = 0;
                for (size_t j = 1; j + 1 < iv.size(); ++j)
                    if (iv[j + 1].first - iv[j].second < iv[jm + 1].first - iv[jm].second) jm = j;
                iv[jm].second = iv[jm + 1].second;
                iv.erase(iv.begin() + (long)jm + 1);
            }
            for (auto& w : iv) {  // 16-byte granules inside x
                w.first &= ~1LL;
                w.second = std::min((w.second + 1) & ~1LL, ncx);
            }
            iv.erase(std::remove_if(iv.begin(), iv.end(), [](auto& w) { return w.second <= w.first; }), iv.end());
            auto find = [&](long long c) -> int {
                for (size_t j = 0; j < iv.size(); ++j)
                    if (c >= iv[j].first && c < iv[j].second) return (int)j;
                return -1;
            };
            cnt.assign(iv.size(), 0);
            for (long long k = k0; k < k1; ++k) {
                const int j = find((long long)h_ci[k]);
                if (j >= 0) ++cnt[(size_t)j];
            }
            long long tot = 0;
            for (auto& w : iv) tot += w.second - w.first;
            while (tot > kXwCapMax && !iv.empty()) {  // keep the most-referenced windows
                size_t jm = 0;
                for (size_t j = 1; j < iv.size(); ++j)
                    if (cnt[j] * (iv[jm].second - iv[jm].first) < cnt[jm] * (iv[j].second - iv[j].first)) jm = j;
                tot -= iv[jm].second - iv[jm].first;
                iv.erase(iv.begin() + (long)jm);
                cnt.erase(cnt.begin() + (long)jm);
            }
            off.assign(iv.size(), 0);
            for (size_t j = 0; j < iv.size(); ++j) {
                off[j] = j ? off[j - 1] + (iv[j - 1].second - iv[j - 1].first) : 0;
                d[j] = (int32_t)iv[j].first;
                d[8 + j / 2] |= (int32_t)((uint32_t)(iv[j].second - iv[j].first) << (16 * (j & 1)));
                cov += cnt[j];
                if (iv[j].first <= rs && re <= iv[j].second) d[14] = (int32_t)(off[j] + rs - iv[j].first);
            }
            bool all = true;
            for (long long k = k0; k < k1; ++k) {
                const long long c = (long long)h_ci[k];
                const int j = find(c);
                if (j >= 0) xoff[(size_t)k] = (uint16_t)(off[(size_t)j] + c - iv[(size_t)j].first);
                else all = false;
            }
            d[15] = all ? 1 : 0;
            stg += tot;
            cx = std::max(cx, (int)tot);
        }
        covered += cov;
        staged += stg;
        int prev = capx.load();
        while (cx > prev && !capx.compare_exchange_weak(prev, cx)) {}
    });
    const double cover = (double)covered.load() / (double)A->nnz;
    if (mode == 1 && (cover < 0.9 || staged.load() > A->nnz)) return;
    A->xw_mode = mode;
    A->cap_x = std::max(16, (capx.load() + 15) & ~15);
    A->xw_cover = cover;
    A->xw = dalloc<int32_t>(desc.size());
    A->xwo = dalloc<uint16_t>(xoff.size());
    CK(memcpy_sync(A->xw, desc.data(), desc.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(memcpy_sync(A->xwo, xoff.data(), xoff.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    choose_xw_variants(A);
    if (A->xw_var[0] < 0 && A->xw_var[1] < 0 && A->xw_var[2] < 0) drop_xwin(A);
    build_xw_pair(A);
}

template <class I>
DevCsr* DevCsr::create(int device, long long nrows, long long ncols, const I* h_rp, const I* h_ci,
                       const double* h_val, bool local_layout) {
    if (nrows < 0 || ncols < 0) fail(SPARSLA_ERR_DIMENSION, "negative matrix shape");
    // rank-local matrices keep the global column order of every row, so their relabelled
    // [owned|halo] column ids need not increase within a row
    if (!local_layout) validate_csr<I>(nrows, ncols, h_rp, h_ci);
    const long long nnz = static_cast<long long>(h_rp[nrows]);
    if (nrows >= (1LL << 31) || ncols >= (1LL << 31) || nnz >= (1LL << 31))
        fail(SPARSLA_ERR_UNSUPPORTED,
             "this build stores int32 row_ptr/col_idx per device: rows, cols and nnz must be < 2^31 "
             "(shard larger matrices across GPUs)");
    DeviceGuard g(device);
    configure_kernels_once(device);
    auto A = std::make_unique<DevCsr>();
    A->device = device;
    A->local_layout = local_layout;
    A->nrows = nrows; A->ncols = ncols; A->nnz = nnz;
    CK(cudaStreamCreateWithFlags(&A->stream, cudaStreamNonBlocking));
    // int32 device layout (+ padding for the bulk-copy over-read)
    A->rp = dalloc<int32_t>(nrows + 1 + kRpCopy + 8);
    A->ci = dalloc<int32_t>(nnz + 8);
    A->val = dalloc<double>(nnz + 4);
    CK(cudaMemset(A->rp, 0, (nrows + 1 + kRpCopy + 8) * sizeof(int32_t)));
    CK(cudaMemset(A->ci + nnz, 0, 8 * sizeof(int32_t)));
    CK(cudaMemset(A->val + nnz, 0, 4 * sizeof(double)));
    if constexpr (sizeof(I) == 4) {
        CK(memcpy_sync(A->rp, h_rp, (nrows + 1) * sizeof(int32_t), cudaMemcpyHostToDevice));
        CK(memcpy_sync(A->ci, h_ci, nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
    } else {
        std::vector<int32_t> tmp(static_cast<size_t>(std::max(nrows + 1, nnz)));
        parallel_for(nrows + 1, [&](int64_t a, int64_t b) { for (int64_t i = a; i < b; ++i) tmp[i] = (int32_t)h_rp[i]; });
        CK(memcpy_sync(A->rp, tmp.data(), (nrows + 1) * sizeof(int32_t), cudaMemcpyHostToDevice));
        parallel_for(nnz, [&](int64_t a, int64_t b) { for (int64_t i = a; i < b; ++i) tmp[i] = (int32_t)h_ci[i]; });
        CK(memcpy_sync(A->ci, tmp.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    CK(memcpy_sync(A->val, h_val, nnz * sizeof(double), cudaMemcpyHostToDevice));
    A->vd_var = vd_variant();
    build_value_dictionary(A.get(), h_val);
    long long mr_all = 0;
    for (long long i = 0; i < nrows; ++i) mr_all = std::max<long long>(mr_all, (long long)h_rp[i + 1] - (long long)h_rp[i]);
    // long rows -> warp-per-row kernel + short-row view for the staged kernels
    std::vector<long long> srp;  // short-view row_ptr (host), when long rows exist
    if (!local_layout) {
        const long long LT = long_row_threshold<I>(nrows, h_rp, mr_all);
        std::vector<int32_t> lr;
        if (LT > 0)
            for (long long i = 0; i < nrows; ++i)
                if ((long long)h_rp[i + 1] - (long long)h_rp[i] > LT) lr.push_back((int32_t)i);
        if (!lr.empty()) {
            std::stable_sort(lr.begin(), lr.end(), [&](int32_t a, int32_t b) {
                return h_rp[a + 1] - h_rp[a] > h_rp[b + 1] - h_rp[b];
            });
            std::vector<uint32_t> bits((size_t)(nrows + 31) / 32, 0u);
            for (int32_t r : lr) bits[(size_t)r >> 5] |= 1u << (r & 31);
            srp.assign((size_t)nrows + 1, 0);
            for (long long i = 0; i < nrows; ++i) {
                const bool lg = (bits[(size_t)i >> 5] >> (i & 31)) & 1u;
                srp[i + 1] = srp[i] + (lg ? 0 : (long long)h_rp[i + 1] - (long long)h_rp[i]);
            }
            const long long snz = srp[nrows];
            std::vector<int32_t> hsrp((size_t)nrows + 1), hsci((size_t)snz);
            std::vector<double> hsv((size_t)snz);
            for (long long i = 0; i <= nrows; ++i) hsrp[i] = (int32_t)srp[i];
            parallel_for(nrows, [&](int64_t a, int64_t b) {
                for (int64_t i = a; i < b; ++i) {
                    const long long o = (long long)h_rp[i], d = srp[i];
                    for (long long k = 0; k < srp[i + 1] - d; ++k) {
                        hsci[d + k] = (int32_t)h_ci[o + k];
                        hsv[d + k] = h_val[o + k];
                    }
                }
            });
            A->nlong = (long long)lr.size();
            A->long_nnz = nnz - snz;
            A->long_threshold = LT;
            A->long_rows = dalloc<int32_t>(lr.size());
            A->long_bits = dalloc<uint32_t>(bits.size());
            A->s_rp = dalloc<int32_t>(nrows + 1 + kRpCopy + 8);
            A->s_ci = dalloc<int32_t>(snz + 8);
            A->s_val = dalloc<double>(snz + 4);
            CK(cudaMemset(A->s_rp, 0, (nrows + 1 + kRpCopy + 8) * sizeof(int32_t)));
            CK(cudaMemset(A->s_ci + snz, 0, 8 * sizeof(int32_t)));
            CK(cudaMemset(A->s_val + snz, 0, 4 * sizeof(double)));
            CK(memcpy_sync(A->long_rows, lr.data(), lr.size() * 4, cudaMemcpyHostToDevice));
            CK(memcpy_sync(A->long_bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice));
            CK(memcpy_sync(A->s_rp, hsrp.data(), hsrp.size() * 4, cudaMemcpyHostToDevice));
            if (snz) {
                CK(memcpy_sync(A->s_ci, hsci.data(), snz * 4, cudaMemcpyHostToDevice));
                CK(memcpy_sync(A->s_val, hsv.data(), snz * 8, cudaMemcpyHostToDevice));
            }
            drop_value_dictionary(A.get());  // the dictionary indexes the full entry order
        }
    }
    // row-length statistics (of the view the staged kernels stream) -> SpMV variant and
    // staging capacity
    auto rpv = [&](long long i) { return srp.empty() ? (long long)h_rp[i] : srp[i]; };
    long long mb = 0, mr = 0;
    for (long long b = 0; b < nrows; b += kChunkSlots) {
        const long long e = std::min(b + kChunkSlots, nrows);
        mb = std::max<long long>(mb, rpv(e) - rpv(b));
    }
    for (long long i = 0; i < nrows; ++i) mr = std::max<long long>(mr, rpv(i + 1) - rpv(i));
    // rows of <= 7 entries (7-point stencils): the 7-wide dictionary kernel at 4 CTAs/SM
    // (56 registers) — more gathers in flight per SM than 8-wide at 3 CTAs/SM (config B
    // SpMV 1.050 -> 0.967 ms, profiles/r01b_notes.md)
    if (!getenv("SPARSLA_VD_VARIANT") && mr <= 7) A->vd_var = 3;
    long long mb32 = 0;
    for (long long b = 0; b < nrows; b += 32) {
        const long long e = std::min(b + 32, nrows);
        mb32 = std::max<long long>(mb32, rpv(e) - rpv(b));
    }
    A->cap_v32 = (int)(((mb32 + 2) + 1) & ~1LL);
    A->cap_c32 = (int)(((mb32 + 6) + 3) & ~3LL);
    A->max_block_nnz = mb;
    A->max_row = mr_all;
    A->cap_v = (int)(((mb + 2) + 1) & ~1LL);
    A->cap_c = (int)(((mb + 6) + 3) & ~3LL);
    A->ws_var = choose_ws_variant(mr);
    {
        // Size the ring for the chosen variant's occupancy; rounds above the resulting
        // capacity (hub rows) bypass the ring inside the kernel instead of demoting the
        // whole matrix to the direct kernel.
        const WsVariant& V = kWsVariants[A->ws_var];
        if (V.rpt != 0) {
            const long long per_cta = 227LL * 1024 / V.minb - 1024 - 256 - 256;
            const long long stage_budget = per_cta / V.stg;
            const long long cap = (stage_budget - 2 * 128 - ((kRpCopy + 1) * 4 + 127)) / 12;
            if (cap < A->cap_v) {
                A->cap_v = (int)(cap & ~1LL);
                A->cap_c = (int)(cap & ~3LL);
                A->has_hub = true;  // some rounds exceed the stage: use the bypass kernels
            }
        }
    }
    {
        // Keep the matrix stream in L2 (evict_last) when matrix + Krylov vectors fit in it;
        // stream it evict_first otherwise so x's reuse lines survive.  SPARSLA_L2_KEEP=0/1
        // overrides (sweeps).
        int l2 = 0;
        CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
        const double ws = 12.0 * nnz + 4.0 * nrows + 48.0 * nrows;
        A->l2_keep = ws <= 0.9 * l2 ? 1 : 0;
        if (const char* e = getenv("SPARSLA_L2_KEEP")) A->l2_keep = atoi(e) ? 1 : 0;
    }
    // dictionary kernels: variant 0 (rows of <= 8 entries) without oversized rounds only
    if (A->ws_var != 0 || A->has_hub) drop_value_dictionary(A.get());
    A->smem_bytes = ws_smem_bytes(A.get(), A->ws_var, A->vd);
    A->staged = A->cap_v >= 512 && A->smem_bytes <= 200 * 1024;  // else: direct kernel
    if (const char* e = getenv("SPARSLA_SPMV_DIRECT")) if (atoi(e)) A->staged = false;
    build_xwin<I>(A.get(), h_rp, h_ci);
    {
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        for (int v = 0; v < kNumWsVariants; ++v) {
            int per_sm = 0;
            const bool vd = A->vd && v == 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, vd ? kVdVariants[A->vd_var].fn[SPMV_CG] : kWsVariants[v].fn[SPMV_CG],
                kWsVariants[v].rpt == 0 ? kSpmvThreads : kWsThreads, ws_smem_bytes(A.get(), v, vd)));
            A->ws_ctas[v] = sms * std::max(1, per_sm);
        }
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kVdVariants[0].fn[SPMV_BICG_T], kWsThreads,
                                                         ws_smem_bytes(A.get(), 0, true)));
        A->vdt_ctas = sms * std::max(1, per_sm);
    }
    CK(cudaDeviceSynchronize());
    return A.release();
}
template DevCsr* DevCsr::create<int64_t>(int, long long, long long, const int64_t*, const int64_t*, const double*, bool);
template DevCsr* DevCsr::create<int32_t>(int, long long, long long, const int32_t*, const int32_t*, const double*, bool);

const double* DevCsr::jacobi_dinv() {
    std::lock_guard<std::mutex> lk(lazy_mu);
    if (!dinv) {
        DeviceGuard g(device);
        if (nrows != ncols && !local_layout) fail(SPARSLA_ERR_DIMENSION, "jacobi_build requires a square matrix");
        dinv = dalloc<double>(nrows + 2);
        if (nrows > 0)
            jacobi_kernel<<<grid_for(nrows, 256), 256, 0, stream>>>(rp, ci, val, nrows, 0, dinv);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(stream));
    }
    return dinv;
}

// every d[i] bit-identical to d[0]?  (flag cleared by any mismatch)
static __global__ void uniform_kernel(const double* d, long long n, int* flag) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && __double_as_longlong(d[i]) != __double_as_longlong(d[0])) *flag = 0;
}

bool DevCsr::jacobi_uniform(double* value) {
    const double* d = jacobi_dinv();
    std::lock_guard<std::mutex> lk(lazy_mu);
    if (dinv_uniform < 0) {
        DeviceGuard g(device);
        dinv_uniform = 0;
        if (nrows > 0) {
            int* flag = dalloc<int>(1);
            const int one = 1;
            CK(cudaMemcpyAsync(flag, &one, sizeof one, cudaMemcpyHostToDevice, stream));
            uniform_kernel<<<grid_for(nrows, 256), 256, 0, stream>>>(d, nrows, flag);
            CK(cudaGetLastError());
            int h = 0;
            CK(cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, stream));
            CK(cudaMemcpyAsync(&dinv_value, d, sizeof(double), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            cudaFree(flag);
            dinv_uniform = h;
        }
    }
    *value = dinv_value;
    return dinv_uniform == 1;
}

const double* DevCsr::ones_vec() {
    std::lock_guard<std::mutex> lk(lazy_mu);
    if (!ones) {
        DeviceGuard g(device);
        ones = dalloc<double>(nrows + 2);
        if (nrows > 0) fill_kernel<<<grid_for(nrows, 256), 256, 0, stream>>>(ones, nrows, 1.0);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(stream));
    }
    return ones;
}

bool DevCsr::exactly_symmetric() {
    std::lock_guard<std::mutex> lk(lazy_mu);
    if (sym_checked < 0) {
        DeviceGuard g(device);
        if (nrows != ncols) { sym_checked = 0; return false; }
        int* flags = dalloc<int>(2);
        const int one[2] = {1, 1};
        CK(memcpy_sync(flags, one, sizeof(one), cudaMemcpyHostToDevice));
        if (nrows > 0) symmetry_kernel<<<grid_for(nrows, 256), 256, 0, stream>>>(rp, ci, val, nrows, flags);
        CK(cudaGetLastError());
        int h[2];
        CK(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        cudaFree(flags);
        sym_checked = h[1] ? 1 : 0;
    }
    return sym_checked == 1;
}

// canonical A^T (setup, nonsymmetric adjoint / spmv_transpose)
DevCsr* DevCsr::get_transpose() {
    std::lock_guard<std::mutex> lk(lazy_mu);
    if (!transpose) {
        DeviceGuard g(device);
        CK(cudaStreamSynchronize(stream));  // the values may have just been (re)written
        std::vector<int32_t> trp(ncols + 1, 0), tci(std::max<long long>(nnz, 1));
        std::vector<double> tv(std::max<long long>(nnz, 1));
        csr_transpose_device(device, nrows, ncols, nnz, rp, ci, val, trp.data(), tci.data(), tv.data());
        transpose = DevCsr::create<int32_t>(device, ncols, nrows, trp.data(), tci.data(), tv.data());
    }
    return transpose;
}

// ------------------------------------------------------------------ launches -------
// Dictionary variant per SpMV mode: the 7-wide 4-CTA kernel (variant 3) serves every mode
// but BiCGStab's t = A s-hat, whose three fused dots spill it; that one keeps the 8-wide
// 3-CTA kernel (config D: 0.69 vs 0.73 ms).
static int vd_var_of(const DevCsr* A, int mode) {
    static const bool t7 = [] { const char* e = getenv("SPARSLA_BICGT_VD7"); return e && atoi(e) != 0; }();
    return (mode == SPMV_BICG_T && A->vd_var == 3 && !t7) ? 0 : A->vd_var;
}

// pair stream: the dictionary index in the low 3 bits of the 16-bit window offset (one
// 2-byte stream per entry instead of 1 + 2 bytes); needs <= 8 distinct values and
// <= 8176 staged elements per round.  Rebuilt on the device whenever the dictionary is.
// Same products in the same order: bit-identical to the other streams.
static void build_xw_pair(DevCsr* A) {
    cudaFree(A->xvo);
    A->xvo = nullptr;
    // default for rows of <= 7 entries (the 7-wide guard-free kernel: config B SpMV 0.962 ->
    // 0.840 ms); with longer rows the 8-wide pair kernel is slower than the gather dictionary
    // kernel (profiles/r02_xwin.md).  SPARSLA_XW_PAIR=0 disables, =1 forces it.
    const char* pe = getenv("SPARSLA_XW_PAIR");
    const int pm = pe ? atoi(pe) : -1;
    if (pm == 0 || (pm < 0 && A->max_row > 7)) return;
    if (!A->xw || !A->vd || A->nvals > (1 << kXwPairValBits) || A->cap_x > (int)kXwPairNone - 15) return;
    if (A->xw_var[2] < 0) return;
    const long long m = A->nnz + kXwPad;
    A->xvo = dalloc<uint16_t>(m);
    xw_pair_kernel<<<grid_for(m, 256), 256, 0, A->stream>>>(A->vidx, A->xwo, A->xvo, m);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(A->stream));
}

// value stream of the x-window path: 0 fp64 values, 1 dictionary indices, 2 pair
static int xw_stream(const DevCsr* A) {
    if (!(A->vd && A->ws_var == 0)) return 0;
    return A->xvo ? 2 : 1;
}

// x-window kernel variant for the matrix's current value stream and this SpMV mode, or -1.
// Measured on B200 (tools/xw_sweep.py, profiles/r02_xwin.md): with the plain fp64 value
// stream the x-window kernel wins everywhere (FEM config C 0.407 -> 0.31 ms; plain 7-point
// stencil 1.78 -> 1.35 ms at 464^3); with the 1-byte value dictionary the gather kernel is
// as fast or faster except for BiCGStab's t = A s-hat (0.615 -> 0.589 ms at 368^3).
static int xw_pick(const DevCsr* A, int mode) {
    if (!A->staged || !A->xw) return -1;
    const int vs = xw_stream(A);
    if (vs == 1 && mode != SPMV_BICG_T && A->xw_mode < 2) return -1;
    return A->xw_var[vs];
}
static bool xw_aligned(const double* x, const double* aux) {  // TMA sources: 16-byte aligned
    return ((uintptr_t)x & 15) == 0 && ((uintptr_t)aux & 15) == 0;
}
static bool mode_has_aux(int mode) { return mode == SPMV_BICG_V || mode == SPMV_BICG_T; }

void devcsr_xwin_info(const DevCsr* A, int64_t* out) {
    out[0] = A->xw ? A->xw_var[xw_stream(A)] : -1;
    out[1] = A->cap_x;
    out[2] = (int64_t)(A->xw_cover * 1e6 + 0.5);
    out[3] = 0;
    for (int m = 0; m < 4; ++m) out[3] |= (xw_pick(A, m) >= 0 ? 1 : 0) << m;
    out[4] = xw_stream(A);
    const int v = out[0];
    out[5] = v >= 0 ? A->xw_ctas[xw_stream(A)][0] / std::max(1, A->sms) : 0;
    out[6] = 0;
    out[7] = 0;
}

// the diagonal-warp kernel (one CTA per chunk) takes every SpMV mode when its table exists
static bool dia_pick(const DevCsr* A, int mode) {
    return A->dia && A->nlong == 0 && !A->has_hub && ((A->dia_modes >> mode) & 1);
}

void devcsr_dia_info(const DevCsr* A, int64_t* out) {
    out[0] = 0;
    for (int m = 0; m < 4; ++m) out[0] |= (dia_pick(A, m) ? 1 : 0) << m;
    out[1] = (int64_t)(A->dia_frac * 1e6 + 0.5);
    out[2] = A->dia ? A->dia_bytes : 0;
    out[3] = 0;
    if (A->dia && kDiaVariants[A->dia_var].pattern) {  // 4-byte words instead of 48-byte entries
        out[2] -= ((A->nrows + 31) / 32) * (kDiaInts * 4 - 4);
        out[3] = A->dia_npat;
    }
}

unsigned spmv_grid(const DevCsr* A, long long nch, int mode, bool xw_ok) {
    if (nch <= 0) return 0;
    if (dia_pick(A, mode))
        return kDiaVariants[A->dia_var].pers ? (unsigned)std::min<long long>(nch, (long long)A->dia_ctas) : (unsigned)nch;
    if (xw_ok && xw_pick(A, mode) >= 0)
        return (unsigned)std::min<long long>(nch, (long long)A->xw_ctas[xw_stream(A)][mode_has_aux(mode)]);
    if (A->staged) {
        const bool vdt = A->vd && A->ws_var == 0 && vd_var_of(A, mode) != A->vd_var;
        return (unsigned)std::min<long long>(nch, (long long)(vdt ? A->vdt_ctas : A->ws_ctas[A->ws_var]));
    }
    return (unsigned)nch;
}

// One SpMV launch over `nch` chunks (all chunks when list == nullptr).  `expected` is the
// number of CTAs of every launch of this reduction point (interior + boundary).
void launch_spmv_part(DevCsr* A, cudaStream_t s, int mode, const double* x, double* y, const double* aux,
                      const RedParams& red, int check_done, const int32_t* list, long long nch,
                      unsigned expected, const P2PCtx* p2p, long long n_interior, int halo_v,
                      unsigned grid_cap) {
    const bool xw_ok = xw_aligned(x, aux);
    unsigned grid = spmv_grid(A, nch, mode, xw_ok);
    const bool dia = dia_pick(A, mode);
    if (grid_cap && A->staged && !dia && grid > grid_cap) grid = grid_cap;  // persistent kernels only
    if (grid == 0) return;
    SpmvParams P{};
    P.rp = A->rp; P.ci = A->ci; P.val = A->val;
    if (A->nlong > 0) {  // short-row view (long rows empty, summed by launch_spmv's fork)
        P.rp = A->s_rp; P.ci = A->s_ci; P.val = A->s_val;
        P.long_bits = A->long_bits;
    }
    P.vidx = A->vidx; P.vtab = A->vtab;
    P.x = x; P.y = y; P.n = A->nrows; P.chunk0 = 0; P.aux = aux;
    P.nch = nch;
    P.chunk_list = list;
    P.p2p = p2p;
    P.n_interior = n_interior;
    P.halo_v = halo_v;
    P.cap_v = A->cap_v; P.cap_c = A->cap_c;
    P.l2_keep = A->l2_keep;
    P.check_done = check_done;
    P.red = red;
    P.red.nchunks = nchunks_of(A->nrows);
    P.red.expected = expected;
    const int xv = xw_ok ? xw_pick(A, mode) : -1;
    if (dia) {
        P.dia = A->dia;
        P.dia_ahead = A->dia_ahead;
        P.ncols = A->ncols;
        void* args[] = {&P};
        if (kDiaVariants[A->dia_var].pattern) {
            P.diaw = A->diaw;
            void* args2[] = {&P, A->diac};
            CK(cudaLaunchKernel(kDiaVariants[A->dia_var].fn[mode], dim3(grid), dim3(kSpmvThreads), args2, 0, s));
        } else {
            CK(cudaLaunchKernel(kDiaVariants[A->dia_var].fn[mode], dim3(grid), dim3(kSpmvThreads), args, 0, s));
        }
    } else if (xv >= 0) {
        P.xw = A->xw;
        P.xwo = xw_stream(A) == 2 ? A->xvo : A->xwo;
        P.cap_x = A->cap_x;
        void* args[] = {&P};
        CK(cudaLaunchKernel(kXwVariants[xv].fn[mode], dim3(grid), dim3(kWsThreads), args,
                            xw_smem_bytes(A, xv, mode_has_aux(mode)), s));
    } else if (A->staged) {
        const int v = A->ws_var;
        const bool wp = kWsVariants[v].rpt == 0;
        if (wp) { P.cap_v = A->cap_v32; P.cap_c = A->cap_c32; }
        void* args[] = {&P};
        const bool vd = A->vd && v == 0;
        const void* fn = vd ? kVdVariants[vd_var_of(A, mode)].fn[mode]
                            : (A->has_hub ? kWsVariants[v].fn_hub[mode] : kWsVariants[v].fn[mode]);
        CK(cudaLaunchKernel(fn, dim3(grid), dim3(wp ? kSpmvThreads : kWsThreads), args, ws_smem_bytes(A, v, vd), s));
    } else {
#define DIRECT_CASE(M) spmv_direct_kernel<M><<<grid, kSpmvThreads, 0, s>>>(P);
        switch (mode) {
            case SPMV_PLAIN: DIRECT_CASE(SPMV_PLAIN) break;
            case SPMV_CG: DIRECT_CASE(SPMV_CG) break;
            case SPMV_BICG_V: DIRECT_CASE(SPMV_BICG_V) break;
            case SPMV_BICG_T: DIRECT_CASE(SPMV_BICG_T) break;
        }
#undef DIRECT_CASE
    }
    CK(cudaGetLastError());
}

// Long rows (single GPU): fork a side stream for the warp-per-row kernel, run the staged
// kernel over the short-row view in SPMV_PLAIN mode meanwhile, join, then form the fused
// dots with spmv_dots_kernel (same canonical reduction, same bits).  Stream-ordered and
// capturable (the fork/join becomes graph edges).
static void launch_spmv_longsplit(DevCsr* A, cudaStream_t s, int mode, const double* x, double* y,
                                  const double* aux, const RedParams& red, int check_done) {
    {
        std::lock_guard<std::mutex> lk(A->lazy_mu);
        if (!A->side) {
            CK(cudaStreamCreateWithFlags(&A->side, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&A->ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&A->ev_join, cudaEventDisableTiming));
        }
    }
    std::lock_guard<std::mutex> lk(A->split_mu);  // one fork in flight per matrix on the host
    CK(cudaEventRecord(A->ev_fork, s));
    CK(cudaStreamWaitEvent(A->side, A->ev_fork, 0));
    LongRowParams L{A->rp, A->ci, A->val, x, y, A->long_rows, A->nlong, red.st, check_done && red.st};
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, A->device));
    const long long want = (A->nlong + kLongWarps - 1) / kLongWarps;
    spmv_longrow_kernel<<<(unsigned)std::min<long long>(want, (long long)sms * 16), kLongWarps * 32, 0, A->side>>>(L);
    CK(cudaGetLastError());
    CK(cudaEventRecord(A->ev_join, A->side));
    const long long nch = nchunks_of(A->nrows);
    RedParams none{};
    none.st = red.st;
    launch_spmv_part(A, s, SPMV_PLAIN, x, y, aux, none, check_done && red.st, nullptr, nch,
                     spmv_grid(A, nch, SPMV_PLAIN, xw_aligned(x, aux)));
    CK(cudaStreamWaitEvent(s, A->ev_join, 0));
    if (mode == SPMV_PLAIN) return;
    SpmvParams P{};
    P.x = x; P.y = y; P.aux = aux; P.n = A->nrows; P.check_done = check_done;
    P.red = red;
    P.red.nchunks = nch;
    P.red.expected = (unsigned)nch;
    switch (mode) {
        case SPMV_CG: spmv_dots_kernel<SPMV_CG><<<(unsigned)nch, kSpmvThreads, 0, s>>>(P); break;
        case SPMV_BICG_V: spmv_dots_kernel<SPMV_BICG_V><<<(unsigned)nch, kSpmvThreads, 0, s>>>(P); break;
        case SPMV_BICG_T: spmv_dots_kernel<SPMV_BICG_T><<<(unsigned)nch, kSpmvThreads, 0, s>>>(P); break;
    }
    CK(cudaGetLastError());
}

void launch_spmv(DevCsr* A, cudaStream_t s, int mode, const double* x, double* y, const double* aux,
                 const RedParams& red, int check_done) {
    if (A->nrows == 0) return;
    if (A->nlong > 0) {
        launch_spmv_longsplit(A, s, mode, x, y, aux, red, check_done);
        return;
    }
    const long long nch = nchunks_of(A->nrows);
    launch_spmv_part(A, s, mode, x, y, aux, red, check_done, nullptr, nch, spmv_grid(A, nch, mode, xw_aligned(x, aux)));
}

static int u1_group() {
    static int g = [] {
        const char* e = getenv("SPARSLA_U1_GROUP");
        return e ? atoi(e) : 4;
    }();
    return g;
}

static bool vec_persist() {
    static bool p = [] {
        const char* e = getenv("SPARSLA_VEC_PERSIST");
        return e ? atoi(e) != 0 : false;
    }();
    return p;
}

template <int OP>
void launch_vec(cudaStream_t s, const VecParams& P0, RedParams red) {
    if (P0.n == 0) return;
    VecParams P = P0;
    P.red = red;
    P.red.nchunks = nchunks_of(P.n);
    P.red.expected = (unsigned)P.red.nchunks;
    const unsigned grid = (unsigned)nchunks_of(P.n);
    // fused peer collectives with every peer on another GPU: a resident grid, so the per-CTA
    // consume of the reduction point and the system-scope fences run once per CTA slot, not
    // once per 2048-row chunk.  (With a peer rank on the same GPU a resident grid spinning on
    // its flags could keep that peer's producer kernel off the SMs.)
    if (vec_persist() || P.resident) {
        int dev = 0, per_sm = 0, sms = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vec_kernel<OP, 4, true>, kVecThreads, 0));
        const unsigned pg = (unsigned)std::min<long long>(grid, (long long)sms * std::max(1, per_sm));
        P.red.expected = pg;
        vec_kernel<OP, 4, true><<<pg, kVecThreads, 0, s>>>(P);
    } else if (OP == V_CG_U1 && u1_group() == 2) vec_kernel<OP, 2><<<grid, kVecThreads, 0, s>>>(P);
    else if (OP == V_CG_U1 && u1_group() == 8) vec_kernel<OP, 8><<<grid, kVecThreads, 0, s>>>(P);
    else vec_kernel<OP><<<grid, kVecThreads, 0, s>>>(P);
    CK(cudaGetLastError());
}

// ------------------------------------------------------------------ Solver ---------
void Solver::validate(const sparsla_solve_options& o, bool square) {
    if (!(o.atol >= 0.0) || !(o.rtol >= 0.0) || (o.atol == 0.0 && o.rtol == 0.0))
        fail(SPARSLA_ERR_INVALID_ARGUMENT, "SolveOptions: atol >= 0, rtol >= 0, not both zero (SPEC.md:129)");
    if (o.max_iter < 1) fail(SPARSLA_ERR_INVALID_ARGUMENT, "SolveOptions: max_iter >= 1");
    if (o.preconditioner != SPARSLA_PRECOND_NONE && o.preconditioner != SPARSLA_PRECOND_JACOBI)
        fail(SPARSLA_ERR_INVALID_ARGUMENT, "SolveOptions: unknown preconditioner");
    if (!square) fail(SPARSLA_ERR_DIMENSION, "Krylov solve requires a square matrix");
}

Solver::Solver(DevCsr* A_, int backend_, const sparsla_solve_options& o, DistCtx* dist_)
    : A(A_), backend(backend_), opts(o), dist(dist_) {
    validate(o, dist || A->nrows == A->ncols);
    DeviceGuard g(A->device);
    n = A->nrows;
    stream = A->stream;
    dinv = o.preconditioner == SPARSLA_PRECOND_JACOBI ? A->jacobi_dinv() : A->ones_vec();
    // A constant Jacobi diagonal (constant-coefficient stencils; the identity when
    // unpreconditioned) is passed as a scalar instead of being streamed: 16 bytes per row
    // less per CG iteration, same operands, same bits.  SPARSLA_UNIFORM_DIAG=0 disables.
    {
        const char* e = getenv("SPARSLA_UNIFORM_DIAG");
        if (!e || atoi(e) != 0) {
            if (o.preconditioner == SPARSLA_PRECOND_JACOBI) d_is_uniform = A->jacobi_uniform(&d_uniform);
            else { d_is_uniform = true; d_uniform = 1.0; }
        }
    }
    const long long m = std::max<long long>(1, nchunks_of(n));
    const long long nv = n + 2;
    const long long nh = (dist ? dist->vec_len : n) + 2;  // SpMV inputs: [owned | gap | halo]
    try {
    x_own = dalloc<double>(nv); b_own = dalloc<double>(nv);
    r = dalloc<double>(nv); p = dalloc<double>(nh); q = dalloc<double>(nv);
    if (backend == SPARSLA_BACKEND_BICGSTAB) {
        rh = dalloc<double>(nv); ph = dalloc<double>(nh); s = dalloc<double>(nv);
        sh = dalloc<double>(nh); t = dalloc<double>(nv);
    }
    partials = dalloc<double>(3 * m);
    // single-GPU CG: x updated every other iteration from two alternating direction
    // buffers (bit-identical; SPARSLA_CG_DEFER_X=0 disables).  Not with the fused kernel.
    {
        const char* e = getenv("SPARSLA_CG_DEFER_X");
        defer_x = !dist && backend == SPARSLA_BACKEND_CG && n > 0 && !(e && atoi(e) == 0);
    }
    // small single-GPU CG problems: whole iterations in one cooperative kernel
    if (!dist && backend == SPARSLA_BACKEND_CG && n > 0) {
        int coop = 0, sms = 0, per_sm = 0;
        CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, A->device));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, A->device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_fused_kernel<false>, kSpmvThreads, 0));
        const long long cap = (long long)sms * per_sm;
        fused_grid = (int)std::min<long long>(m, cap);
        // one chunk per CTA (measured: 2 per CTA ~ break-even); thread-per-row, so never for
        // matrices with long (hub) rows — those take the warp-per-row split of the SpMV
        fused = coop && cap > 0 && m <= cap && A->nlong == 0 && A->max_row <= kLongMin;
        if (const char* e = getenv("SPARSLA_FUSED")) fused = coop && cap > 0 && atoi(e) != 0;
        if (fused) { fused_bar = dalloc<unsigned>(1); defer_x = false; }
        // resident chunk images when every chunk fits uint16 offsets / int16 column deltas and
        // the whole grid stays co-resident with the larger shared-memory footprint
        const char* re = getenv("SPARSLA_FUSED_RESIDENT");
        if (fused && m <= cap && !(re && atoi(re) == 0)) {
            int* chk = dalloc<int>(2);
            int h[2] = {0, 0};
            CK(cudaMemsetAsync(chk, 0, 8, stream));
            fused_res_check_kernel<<<(unsigned)m, kSpmvThreads, 0, stream>>>(A->rp, A->ci, n, chk);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(h, chk, 8, cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            cudaFree(chk);
            if (h[0] <= 65535 && h[1] == 0) {
                const int cap_e = (h[0] + 7) / 8 * 8;
                const size_t bytes = fused_res_bytes(cap_e);
                int rs = 0;
                // the attribute is process-wide: raise it once per device to the opt-in
                // maximum (never lowered per solver, so a parked solver with a larger image
                // keeps launching); occupancy below uses this solver's own footprint
                {
                    static std::mutex mu;
                    static bool raised[64] = {false};
                    std::lock_guard<std::mutex> lk(mu);
                    if (A->device < 64 && !raised[A->device]) {
                        int optin = 0;
                        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, A->device));
                        cudaFuncAttributes fa{};
                        CK(cudaFuncGetAttributes(&fa, cg_fused_kernel<true>));  // minus its static smem
                        CK(cudaFuncSetAttribute(cg_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                optin - (int)fa.sharedSizeBytes));
                        raised[A->device] = true;
                    }
                }
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rs, cg_fused_kernel<true>, kSpmvThreads, bytes));
                if ((long long)sms * rs >= m) { fused_res = cap_e; fused_grid = (int)m; }
            }
        }
    }
    if (defer_x) p2 = dalloc<double>(nh);
    tickets = dalloc<unsigned>(16);  // [0, 8): per reduction point; [8, 16): multi_finish
    CK(cudaMemset(tickets, 0, 16 * sizeof(unsigned)));
    if (!getenv("SPARSLA_MULTI_FINISH") || atoi(getenv("SPARSLA_MULTI_FINISH")) != 0)
        slotsum = dalloc<double>(4 * kFinalSlots);
    st = dalloc<KState>(1);
    CK(cudaMallocHost(&h_st, sizeof(KState)));
    CK(cudaMallocHost(&h_flag, 2 * sizeof(int)));
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    if (dist && dist->p2p_enabled) p2p_setup();
    } catch (...) {
        release();  // a constructor that throws runs no destructor: free what was allocated
        throw;
    }
    x = x_own; b = b_own;
}

void Solver::release() noexcept {
    DeviceGuard g(A->device, true);
    p2p_release();
    if (g_many) cudaGraphExecDestroy(g_many);
    if (g_one) cudaGraphExecDestroy(g_one);
    if (g_one_odd) cudaGraphExecDestroy(g_one_odd);
    for (double* v : {x_own, b_own, r, p, p2, q, rh, ph, s, sh, t}) cudaFree(v);
    cudaFree(partials); cudaFree(tickets); cudaFree(st); cudaFree(fused_bar); cudaFree(slotsum);
    if (h_st) cudaFreeHost(h_st);
    if (h_flag) cudaFreeHost(h_flag);
    if (ev[0]) cudaEventDestroy(ev[0]);
    if (ev[1]) cudaEventDestroy(ev[1]);
    g_many = g_one = g_one_odd = nullptr;
    x_own = b_own = r = p = p2 = q = rh = ph = s = sh = t = nullptr;
    partials = nullptr; tickets = nullptr; st = nullptr; fused_bar = nullptr; slotsum = nullptr;
    h_st = nullptr; h_flag = nullptr; ev[0] = ev[1] = nullptr;
    cudaGetLastError();
}

Solver::~Solver() { release(); }

RedParams Solver::red(int which, int slot) const {
    RedParams R{};
    R.partials = partials; R.ticket = tickets + slot; R.st = st; R.red_out = nullptr; R.scalar = which;
    R.slotsum = slotsum; R.ticket2 = tickets + 8 + slot;
    return R;
}

VecParams Solver::vparams() const {
    VecParams P{};
    P.n = n; P.d = d_is_uniform ? nullptr : dinv; P.d_uni = d_uniform; P.x = x; P.r = r; P.q = q;
    P.p = swap_p ? p2 : p;   // deferred x update, odd iterations: the current direction is in p2
    P.p2 = swap_p ? p : p2;
    P.rh = rh; P.ph = ph; P.v = q; P.s = s; P.sh = sh; P.tt = t; P.b = b;
    P.check_done = 1;
    return P;
}

// One SpMV reduction point: (distributed: halo exchange on the comm stream overlapped
// with the interior-row SpMV, then the boundary rows, then the all-gather of the rank
// totals and the rank-ordered scalar step) or a single launch.
void Solver::spmv_point(int mode, double* xin, double* y, const double* aux, int scalar, int slot, int check_done) {
    RedParams R = scalar == SC_NONE ? RedParams{} : red(scalar, slot);
    const int nd = mode == SPMV_BICG_T ? 3 : (mode == SPMV_PLAIN ? 0 : 1);
    if (!dist) {
        launch_spmv(A, stream, mode, xin, y, aux, R, check_done);
        return;
    }
    if (d_p2p && check_done) {  // fused peer collectives: one launch, halo pushed by the producer
        R.p2p = d_p2p;
        R.point = slot;
        const unsigned gall = spmv_grid(A, dist->n_interior + dist->n_boundary, mode);
        launch_spmv_part(A, stream, mode, xin, y, aux, R, check_done, dist->d_all_chunks,
                         dist->n_interior + dist->n_boundary, gall, d_p2p, dist->n_interior,
                         mode == SPMV_BICG_T ? 1 : 0);  // halo flag: p / p-hat = 0, s-hat = 1
        return;
    }
    if (nd > 0) R.red_out = dist->red_send + slot * 8;
    dist->exchange(stream, xin);
    // The interior launch runs while the halo moves: with peers, cap its persistent grid two
    // SMs short of the device so the transport's kernels (NCCL send/recv) are not queued
    // behind a GPU-filling grid.  (The persistent kernels loop over their chunks, so any grid
    // works; the ticket count `expected` uses the same capped grid.)
    unsigned cap = 0;
    if (dist->tr && dist->tr->P > 1 && A->staged && !dia_pick(A, mode)) {
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, A->device));
        const unsigned full = spmv_grid(A, 1LL << 40, mode);
        const unsigned per_sm = std::max(1u, full / (unsigned)std::max(1, sms));
        if (full > 4 * per_sm) cap = full - 2 * per_sm;
    }
    unsigned gi = spmv_grid(A, dist->n_interior, mode);
    if (cap && gi > cap) gi = cap;
    const unsigned gb = spmv_grid(A, dist->n_boundary, mode);
    launch_spmv_part(A, stream, mode, xin, y, aux, R, check_done, dist->d_interior, dist->n_interior, gi + gb,
                     nullptr, 0, 0, cap);
    CK(cudaStreamWaitEvent(stream, dist->ev_halo, 0));
    launch_spmv_part(A, stream, mode, xin, y, aux, R, check_done, dist->d_boundary, dist->n_boundary, gi + gb);
    if (nd > 0) reduce_point(scalar, slot, nd);
}

void Solver::reduce_point(int scalar, int slot, int nd) {
    dist->tr->allgather(stream, dist->red_send + slot * 8, dist->red_all + (size_t)slot * dist->tr->P * 8, 8);
    scalar_kernel<<<1, 32, 0, stream>>>(dist->red_all + (size_t)slot * dist->tr->P * 8, dist->tr->P, nd, scalar, st);
    CK(cudaGetLastError());
}

template <int OP>
void Solver::vec_point(int scalar, int slot, int check_done) {
    VecParams P = vparams();
    P.check_done = check_done;
    RedParams R = red(scalar, slot);  // (CG_U2 uses the slot's ticket to clear pending_x)
    constexpr int nd = VecTraits<OP>::ndot;
    if (d_p2p && (OP == V_CG_U1 || OP == V_CG_U2 || OP == V_BI_U1 || OP == V_BI_U2 || OP == V_BI_U3)) {
        // consume the previous reduction point in-kernel (CG: U1 <- p.q, U2 <- r.z/r.r;
        // BiCGStab: U1 <- previous U3's rho/r.r, U2 <- rhat.v, U3 <- t.t/t.s/s.s); kernels
        // with dot products push their own totals as point `slot`
        P.p2p = d_p2p;
        P.resident = dist->p2p_shared_device ? 0 : 1;
        switch (OP) {
            case V_CG_U1: P.consume_point = 1; P.consume_scalar = SC_CG_PQ; P.consume_k = 1; break;
            case V_CG_U2: P.consume_point = 2; P.consume_scalar = SC_CG_RR; P.consume_k = 2; break;
            case V_BI_U1: P.consume_point = 5; P.consume_scalar = SC_BI_U3; P.consume_k = 2; break;
            case V_BI_U2: P.consume_point = 2; P.consume_scalar = SC_BI_RV; P.consume_k = 1; break;
            default: P.consume_point = 4; P.consume_scalar = SC_BI_T; P.consume_k = 3; break;
        }
        R.point = slot;
        launch_vec<OP>(stream, P, R);
        return;
    }
    constexpr bool reduces = nd > 0 && VecPublishOnly<OP>::row < 0;  // U2's s.s is reduced by the t-SpMV
    if (dist && reduces) R.red_out = dist->red_send + slot * 8;
    launch_vec<OP>(stream, P, R);
    if (dist && reduces) reduce_point(scalar, slot, nd);
}

void Solver::enqueue_init() {
    KState h{};
    h.atol = opts.atol; h.rtol = opts.rtol; h.max_iter = opts.max_iter;
    h.spmv_count = 1;
    *h_st = h;
    CK(cudaMemcpyAsync(st, h_st, sizeof(KState), cudaMemcpyHostToDevice, stream));
    CK(cudaMemsetAsync(tickets, 0, 16 * sizeof(unsigned), stream));
    CK(cudaMemsetAsync(x, 0, n * sizeof(double), stream));
    // initial residual r0 = b - A x0 (one SpMV, spmv_count = 1); x0 = 0 lives in p's storage
    // for the distributed case so the halo exchange has its slots
    double* x0 = dist ? p : x;
    if (dist) CK(cudaMemsetAsync(p, 0, dist->vec_len * sizeof(double), stream));
    if (d_p2p) {  // fused-collective epochs restart at 0 on every rank (ordered by the init all-gather)
        CK(cudaMemsetAsync(p2p_allocs[1], 0, 8 * dist->tr->P * sizeof(unsigned long long), stream));
        CK(cudaMemsetAsync(p2p_allocs[2], 0, 4 * dist->tr->P * sizeof(unsigned long long), stream));
    }
    spmv_point(SPMV_PLAIN, x0, q, nullptr, SC_NONE, 0, 0);
    if (backend == SPARSLA_BACKEND_CG) vec_point<V_CG_INIT>(SC_CG_INIT, 0, 0);
    else vec_point<V_BI_INIT>(SC_BI_INIT, 0, 0);
    if (d_p2p && backend == SPARSLA_BACKEND_CG) {  // halo of p0 through the transport once;
        dist->exchange(stream, p);                    // later iterations push it in-kernel
        CK(cudaStreamWaitEvent(stream, dist->ev_halo, 0));
    }
    if (n == 0 && !dist) {  // empty system: converged with zero residual
        KState z = h;
        z.converged = 1; z.status = ST_CONVERGED; z.done = 1;
        *h_st = z;
        CK(cudaMemcpyAsync(st, h_st, sizeof(KState), cudaMemcpyHostToDevice, stream));
    }
}

void Solver::enqueue_iteration(cudaEvent_t* evs, int par) {
    // evs (optional): launches_per_iteration()+1 events recorded around every kernel;
    // par: iteration parity (deferred x update: which direction buffer is current)
    auto mark = [&](int i) { if (evs) CK(cudaEventRecord(evs[i], stream)); };
    mark(0);
    if (backend == SPARSLA_BACKEND_CG && defer_x) {
        swap_p = par != 0;
        spmv_point(SPMV_CG, swap_p ? p2 : p, q, nullptr, SC_CG_PQ, 1, 1); mark(1);
        vec_point<V_CG_U1>(SC_CG_RR, 2, 1); mark(2);
        if (par == 0) vec_point<V_CG_U2E>(SC_NONE, 3, 1);
        else vec_point<V_CG_U2O>(SC_NONE, 3, 1);
        mark(3);
        swap_p = false;
    } else if (backend == SPARSLA_BACKEND_CG) {
        spmv_point(SPMV_CG, p, q, nullptr, SC_CG_PQ, 1, 1); mark(1);
        vec_point<V_CG_U1>(SC_CG_RR, 2, 1); mark(2);
        vec_point<V_CG_U2>(SC_NONE, 3, 1); mark(3);
    } else {
        vec_point<V_BI_U1>(SC_NONE, 1, 1); mark(1);
        spmv_point(SPMV_BICG_V, ph, q, rh, SC_BI_RV, 2, 1); mark(2);
        vec_point<V_BI_U2>(SC_NONE, 3, 1); mark(3);
        spmv_point(SPMV_BICG_T, sh, t, s, SC_BI_T, 4, 1); mark(4);
        vec_point<V_BI_U3>(SC_BI_U3, 5, 1); mark(5);
    }
}

void Solver::kernel_times(long long iters, double* ms) {
    DeviceGuard g(A->device);
    const int L = (int)launches_per_iteration();
    if (fused) {  // one kernel runs whole iterations: report the per-iteration time in ms[0]
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, stream));
        enqueue_fused(iters);
        CK(cudaEventRecord(e1, stream));
        CK(cudaEventSynchronize(e1));
        float t = 0;
        CK(cudaEventElapsedTime(&t, e0, e1));
        for (int k = 0; k < L; ++k) ms[k] = 0.0;
        ms[0] = t / (double)iters;
        cudaEventDestroy(e0); cudaEventDestroy(e1);
        return;
    }
    std::vector<cudaEvent_t> evs((size_t)iters * (L + 1));
    for (auto& e : evs) CK(cudaEventCreate(&e));
    for (long long it = 0; it < iters; ++it) {
        enqueue_iteration(evs.data() + it * (L + 1), parity);
        if (defer_x) parity ^= 1;
    }
    CK(cudaStreamSynchronize(stream));
    for (int k = 0; k < L; ++k) ms[k] = 0.0;
    for (long long it = 0; it < iters; ++it)
        for (int k = 0; k < L; ++k) {
            float t = 0;
            CK(cudaEventElapsedTime(&t, evs[it * (L + 1) + k], evs[it * (L + 1) + k + 1]));
            ms[k] += t / (double)iters;
        }
    for (auto& e : evs) cudaEventDestroy(e);
}

long long Solver::launches_per_iteration() const { return backend == SPARSLA_BACKEND_CG ? 3 : 5; }

void Solver::build_graphs() {
    if (g_many || !capturable()) return;
    auto capture = [&](int iters, int par0) {  // deferred x: parities alternate from par0
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < iters; ++i) enqueue_iteration(nullptr, defer_x ? (par0 + i) & 1 : 0);
        CK(cudaStreamEndCapture(stream, &graph));
        cudaGraphExec_t exec;
        CK(cudaGraphInstantiate(&exec, graph, 0));
        CK(cudaGraphDestroy(graph));
        return exec;
    };
    g_many = capture(kGraphIters, 0);  // even length: starts and ends on an even iteration
    g_one = capture(1, 0);
    if (defer_x) g_one_odd = capture(1, 1);
}

void Solver::set_b(const double* src, int mem) {
    DeviceGuard g(A->device);
    if (mem == SPARSLA_MEM_DEVICE) b = src;
    else { b = b_own; CK(cudaMemcpyAsync(b_own, src, n * sizeof(double), cudaMemcpyHostToDevice, stream)); }
}

// Deferred x update: after an even number of iterations x lacks alpha_prev * p_prev (p_prev
// is in p: even iterations leave the next direction in p2).  Apply it before x is read
// mid-solve; the flag is cleared so the next odd iteration does not apply it again.
static __global__ void cg_flush_x_kernel(double* x, const double* pprev, long long n, double a) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = __dadd_rn(x[i], __dmul_rn(a, pprev[i]));
}
void Solver::flush_x() {
    if (!defer_x) return;
    CK(cudaMemcpyAsync(h_st, st, sizeof(KState), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (!h_st->x_lag) return;
    cg_flush_x_kernel<<<grid_for(n, 256), 256, 0, stream>>>(x, p, n, h_st->alpha_prev);
    CK(cudaGetLastError());
    const int zero = 0;
    CK(cudaMemcpyAsync(&st->x_lag, &zero, sizeof(int), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));
}

void Solver::reset() {
    DeviceGuard g(A->device);
    build_graphs();
    enqueue_init();
    parity = 0;
}

bool Solver::capturable() const { return !fused && (!dist || dist->tr->capturable()); }

void Solver::enqueue_fused(long long iters) {
    FusedParams F{};
    F.rp = A->rp; F.ci = A->ci; F.val = A->val; F.d = d_is_uniform ? nullptr : dinv; F.d_uni = d_uniform;
    F.vidx = A->vd ? A->vidx : nullptr; F.vtab = A->vtab;
    F.x = x; F.r = r; F.p = p; F.q = q;
    F.n = n; F.nch = nchunks_of(n);
    F.partials = partials; F.bar = fused_bar; F.st = st;
    while (iters > 0) {
        F.iters = (int)std::min<long long>(iters, 1 << 20);
        CK(cudaMemsetAsync(fused_bar, 0, sizeof(unsigned), stream));
        void* args[] = {&F};
        if (fused_res > 0 && F.vidx) {
            F.res_cap = fused_res;
            CK(cudaLaunchCooperativeKernel((const void*)cg_fused_kernel<true>, dim3(fused_grid), dim3(kSpmvThreads),
                                           args, fused_res_bytes(fused_res), stream));
        } else {
            CK(cudaLaunchCooperativeKernel((const void*)cg_fused_kernel<false>, dim3(fused_grid), dim3(kSpmvThreads),
                                           args, 0, stream));
        }
        iters -= F.iters;
    }
}

void Solver::iterate(long long iters) {
    DeviceGuard g(A->device);
    build_graphs();
    if (fused) {
        enqueue_fused(iters);
        return;
    }
    if (!capturable()) {
        while (iters-- > 0) {
            enqueue_iteration(nullptr, parity);
            if (defer_x) parity ^= 1;
        }
        return;
    }
    if (parity && iters > 0) { CK(cudaGraphLaunch(g_one_odd, stream)); --iters; parity = 0; }
    while (iters >= kGraphIters) { CK(cudaGraphLaunch(g_many, stream)); iters -= kGraphIters; }
    while (iters-- > 0) {
        CK(cudaGraphLaunch(parity ? g_one_odd : g_one, stream));
        if (defer_x) parity ^= 1;
    }
}

void Solver::run() {
    DeviceGuard g(A->device);
    build_graphs();
    // Poll the device 'done' flag once per graph, one graph behind (no per-iteration sync).
    const long long max_graphs = opts.max_iter / kGraphIters + 3;  // (fused: 4x more per launch)
    h_flag[0] = h_flag[1] = 0;
    // All ranks of a distributed solve see identical device flags (same all-gathered
    // totals, same scalar step), so they stop after the same number of graph launches.
    long long last = -1;
    for (long long i = 0; i < max_graphs; ++i) {
        last = i;
        if (fused) enqueue_fused(4 * kGraphIters);
        else if (capturable()) {
            if (parity) { CK(cudaGraphLaunch(g_one_odd, stream)); parity = 0; }  // back to even
            CK(cudaGraphLaunch(g_many, stream));
        } else {
            for (int k = 0; k < kGraphIters; ++k) {
                enqueue_iteration(nullptr, parity);
                if (defer_x) parity ^= 1;
            }
        }
        CK(cudaMemcpyAsync(h_flag + (i & 1), &st->done, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaEventRecord(ev[i & 1], stream));
        if (i > 0) {
            wait_event(ev[(i - 1) & 1]);
            if (h_flag[(i - 1) & 1]) break;
        }
    }
    if (last >= 0) wait_event(ev[last & 1]);
    CK(cudaStreamSynchronize(stream));
}

// Single GPU: a blocking event wait.  Distributed: poll the event and the transport
// (NCCL asynchronous errors) meanwhile; a graph that makes no progress within the
// collective timeout (+5 s, so the fused mode's device-side timeout reports first) aborts
// the communicator and raises TransportError instead of hanging.
void Solver::wait_event(cudaEvent_t e) {
    if (!dist || !dist->tr) { CK(cudaEventSynchronize(e)); return; }
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = transport_timeout_s() + 5.0;
    for (unsigned k = 0;; ++k) {
        const cudaError_t q = cudaEventQuery(e);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) CK(q);
        if ((k & 63) == 0) {
            dist->tr->check();
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
                dist->tr->abort();
                fail(SPARSLA_ERR_TRANSPORT, "distributed iteration made no progress within " +
                                                std::to_string(limit) + " s: collective timeout (SPEC.md:534)");
            }
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

void Solver::report(sparsla_solve_report* rep) {
    DeviceGuard g(A->device);
    CK(cudaMemcpyAsync(h_st, st, sizeof(KState), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    const KState& S = *h_st;
    std::memset(rep, 0, sizeof(*rep));
    rep->iterations = S.k;
    rep->spmv_count = S.spmv_count;
    rep->residual_norm = S.rnorm;
    rep->converged = S.converged;
    rep->backend = backend;
    const long long k = S.breakdown_iter;
    switch (S.status) {
        case ST_CONVERGED: case ST_RUNNING: break;
        case ST_MAXITER: std::snprintf(rep->diagnostic, 128, "max_iter reached"); break;
        case ST_BD_PQ: std::snprintf(rep->diagnostic, 128, "breakdown: p^T A p <= 0 at iteration %lld", k); break;
        case ST_BD_RHO: std::snprintf(rep->diagnostic, 128, "breakdown: |rho| < 1e-30*||b||^2 at iteration %lld", k); break;
        case ST_BD_RV: std::snprintf(rep->diagnostic, 128, "breakdown: rhat^T v = 0 at iteration %lld", k); break;
        case ST_BD_TT: std::snprintf(rep->diagnostic, 128, "breakdown: t^T t = 0 at iteration %lld", k); break;
        case ST_BD_OMEGA: std::snprintf(rep->diagnostic, 128, "breakdown: omega = 0 at iteration %lld", k); break;
        case ST_TRANSPORT: std::snprintf(rep->diagnostic, 128, "transport timeout at iteration %lld", S.k); break;
    }
    if (S.status == ST_RUNNING && !S.converged) std::snprintf(rep->diagnostic, 128, "running");
}

// canonical dot of device vectors (result on host); scratch is per thread and device
struct DotScratch {
    int device = -1;
    long long cap = -1;
    double* partials = nullptr;
    unsigned* ticket = nullptr;
    KState* st = nullptr;
    cudaStream_t stream = nullptr;
    ~DotScratch() {
        if (device < 0) return;
        cudaSetDevice(device);
        cudaFree(partials); cudaFree(ticket); cudaFree(st);
        cudaStreamDestroy(stream);
    }
};

double device_dot(int device, long long n, const double* a, const double* b, cudaStream_t s) {
    if (n == 0) return 0.0;
    static thread_local DotScratch S;
    const long long m = nchunks_of(n);
    if (S.device != device || S.cap < m) {
        S.~DotScratch();
        new (&S) DotScratch();
        S.device = device;
        S.cap = m;
        S.partials = dalloc<double>(m);
        S.ticket = dalloc<unsigned>(1);
        CK(cudaMemset(S.ticket, 0, sizeof(unsigned)));
        S.st = dalloc<KState>(1);
        CK(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
    }
    (void)s;
    DotParams P{};
    P.n = n; P.a = a; P.b = b;
    P.red.partials = S.partials;
    P.red.nchunks = m;
    P.red.expected = (unsigned)m;
    P.red.ticket = S.ticket;
    P.red.st = S.st;
    P.red.scalar = SC_STORE;
    CK(cudaDeviceSynchronize());
    dot_kernel<<<(unsigned)m, kVecThreads, 0, S.stream>>>(P);
    CK(cudaGetLastError());
    double out;
    CK(cudaMemcpyAsync(&out, &S.st->scratch[0], sizeof(double), cudaMemcpyDeviceToHost, S.stream));
    CK(cudaStreamSynchronize(S.stream));
    return out;
}

// SparseCoo::with_values (sparse.hpp:58-61) on a device matrix: same pattern, new values.
// Every value-dependent cache is dropped (parked solvers hold the old diagonal; the value
// dictionary, the Jacobi diagonal, the symmetry verdict and A^T are rebuilt lazily).
void devcsr_set_values(DevCsr* A, const double* vals, int32_t mem) {
    DeviceGuard g(A->device);
    CK(cudaMemcpyAsync(A->val, vals, A->nnz * sizeof(double),
                       mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, A->stream));
    CK(cudaStreamSynchronize(A->stream));
    A->drop_parked();
    if (A->nlong > 0 && A->nrows > 0) {
        short_view_values_kernel<<<grid_for(A->nrows, 256), 256, 0, A->stream>>>(A->rp, A->val, A->s_rp, A->s_val,
                                                                                A->nrows);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(A->stream));
    }
    // value dictionary: rebuilt from host values (the scan stops at the 257th distinct
    // value); device values are only downloaded when the matrix had a dictionary
    if (A->ws_var == 0 && !A->has_hub && A->nlong == 0 && (mem != SPARSLA_MEM_DEVICE || A->vd)) {
        if (mem != SPARSLA_MEM_DEVICE) {
            build_value_dictionary(A, vals);
        } else {
            std::vector<double> hv((size_t)A->nnz);
            CK(memcpy_sync(hv.data(), A->val, A->nnz * sizeof(double), cudaMemcpyDeviceToHost));
            build_value_dictionary(A, hv.data());
        }
    } else {
        drop_value_dictionary(A);
    }
    A->smem_bytes = ws_smem_bytes(A, A->ws_var, A->vd);
    build_xw_pair(A);  // the pair stream carries dictionary indices
    if (A->dinv) { cudaFree(A->dinv); A->dinv = nullptr; }
    A->dinv_uniform = -1;
    A->sym_checked = -1;
    delete A->transpose;
    A->transpose = nullptr;
}

}  // namespace sparsla_b200

// =============================================================== C ABI (device) ======
using namespace sparsla_b200;

struct sparsla_dcsr { DevCsr* A; };

namespace {
// host/device staging of a vector argument
struct VecArg {
    const double* dptr = nullptr;
    double* owned = nullptr;
    VecArg(const double* src, long long n, int mem, cudaStream_t s) {
        if (mem == SPARSLA_MEM_DEVICE) { dptr = src; return; }
        if (mem != SPARSLA_MEM_HOST) fail(SPARSLA_ERR_INVALID_ARGUMENT, "mem must be SPARSLA_MEM_HOST or _DEVICE");
        owned = dalloc<double>(n + 2);
        if (n) CK(cudaMemcpyAsync(owned, src, n * sizeof(double), cudaMemcpyHostToDevice, s));
        dptr = owned;
    }
    ~VecArg() { if (owned) cudaFree(owned); }
};
struct OutArg {
    double* dptr = nullptr;
    double* user;
    long long n;
    int mem;
    cudaStream_t s;
    OutArg(double* dst, long long n_, int mem_, cudaStream_t s_) : user(dst), n(n_), mem(mem_), s(s_) {
        if (mem == SPARSLA_MEM_DEVICE) dptr = dst;
        else dptr = dalloc<double>(n + 2);
    }
    void finish() {
        if (mem != SPARSLA_MEM_DEVICE && n) CK(cudaMemcpyAsync(user, dptr, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    ~OutArg() { if (mem != SPARSLA_MEM_DEVICE) cudaFree(dptr); }
};
void need(const void* p, const char* what) {
    if (!p) fail(SPARSLA_ERR_INVALID_ARGUMENT, std::string(what) + " is null");
}

bool solver_cache_on() {
    static const bool on = [] { const char* e = getenv("SPARSLA_SOLVER_CACHE"); return !e || atoi(e) != 0; }();
    return on;
}

int krylov(sparsla_dcsr* H, int backend, const double* b, double* x, const sparsla_solve_options* o,
           sparsla_solve_report* rep, int32_t mem) {
    return guarded([&] {
        need(H, "matrix"); need(o, "options"); need(rep, "report");
        DevCsr* A = H->A;
        DeviceGuard g(A->device);
        // Host-buffer calls reuse the matrix's parked solver of this backend (workspace and
        // captured graphs address only solver-owned vectors); device-buffer calls bind the
        // caller's x into the graphs and get their own.
        std::unique_ptr<Solver> S;
        const bool cache = mem != SPARSLA_MEM_DEVICE && solver_cache_on();
        if (cache) {
            Solver::validate(*o, A->nrows == A->ncols);
            std::lock_guard<std::mutex> lk(A->solver_mu);
            Solver*& slot = A->parked[backend == SPARSLA_BACKEND_CG ? 0 : 1];
            if (slot && slot->opts.preconditioner == o->preconditioner) {
                S.reset(slot);
                slot = nullptr;
                S->opts = *o;  // tolerances / max_iter enter through reset() (KState)
            }
        }
        if (!S) {
            long long ver;
            {
                std::lock_guard<std::mutex> lk(A->solver_mu);
                ver = A->values_version;
            }
            S = std::make_unique<Solver>(A, backend, *o);
            S->values_version = ver;
        }
        S->set_b(b, mem);
        if (mem == SPARSLA_MEM_DEVICE) S->x = x;
        S->reset();
        S->run();
        S->report(rep);
        if (mem != SPARSLA_MEM_DEVICE && A->nrows)
            CK(cudaMemcpyAsync(x, S->x, A->nrows * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
        CK(cudaStreamSynchronize(A->stream));
        if (cache) {
            std::lock_guard<std::mutex> lk(A->solver_mu);
            Solver*& slot = A->parked[backend == SPARSLA_BACKEND_CG ? 0 : 1];
            if (!slot && S->values_version == A->values_version) slot = S.release();
        }
    });
}
}  // namespace

extern "C" {

int sparsla_device_count(int* count) {
    return guarded([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); n = 0; }
        *count = n;
    });
}

int sparsla_dcsr_create(int device, int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                        const double* v, sparsla_dcsr** out) {
    return guarded([&] {
        need(rp, "row_ptr"); need(out, "out");
        *out = new sparsla_dcsr{DevCsr::create<int64_t>(device, nrows, ncols, rp, ci, v)};
    });
}

int sparsla_dcsr_create_i32(int device, int64_t nrows, int64_t ncols, const int32_t* rp, const int32_t* ci,
                            const double* v, sparsla_dcsr** out) {
    return guarded([&] {
        need(rp, "row_ptr"); need(out, "out");
        *out = new sparsla_dcsr{DevCsr::create<int32_t>(device, nrows, ncols, rp, ci, v)};
    });
}

int sparsla_dcsr_set_values(sparsla_dcsr* H, const double* vals, int32_t mem) {
    return guarded([&] {
        need(H, "matrix");
        devcsr_set_values(H->A, vals, mem);
    });
}

int sparsla_dcsr_destroy(sparsla_dcsr* H) {
    return guarded([&] {
        if (!H) return;
        delete H->A;
        delete H;
    });
}

int sparsla_dcsr_long_rows(const sparsla_dcsr* H, int64_t* out) {
    return guarded([&] {
        need(H, "matrix"); need(out, "out");
        out[0] = H->A->nlong; out[1] = H->A->long_nnz; out[2] = H->A->long_threshold;
    });
}

int sparsla_dcsr_info(const sparsla_dcsr* H, int64_t* info) {
    return guarded([&] {
        need(H, "matrix");
        const DevCsr* A = H->A;
        info[0] = A->nrows; info[1] = A->ncols; info[2] = A->nnz;
        info[3] = (A->nrows + 1) * 4 + A->nnz * 12;
        info[4] = A->max_block_nnz; info[5] = A->max_row; info[6] = A->staged ? 0 : 1;
        info[7] = A->ws_var;
    });
}

int sparsla_dcsr_xwin(const sparsla_dcsr* H, int64_t* out) {
    return guarded([&] {
        need(H, "matrix"); need(out, "out");
        devcsr_xwin_info(H->A, out);
    });
}

int sparsla_dcsr_dia(const sparsla_dcsr* H, int64_t* out) {
    return guarded([&] {
        need(H, "matrix"); need(out, "out");
        devcsr_dia_info(H->A, out);
    });
}

int sparsla_dcsr_format(sparsla_dcsr* H, int64_t* fmt) {
    return guarded([&] {
        need(H, "matrix");
        DevCsr* A = H->A;
        DeviceGuard g(A->device);
        fmt[0] = A->vd ? 1 : 0;
        fmt[1] = A->vd ? A->nvals : 0;
        double v = 0.0;
        fmt[2] = (A->nrows == A->ncols || A->local_layout) && A->jacobi_uniform(&v) ? 1 : 0;
    });
}

int sparsla_spmv(sparsla_dcsr* H, const double* x, double* y, int32_t mem) {
    return guarded([&] {
        need(H, "matrix");
        DevCsr* A = H->A;
        DeviceGuard g(A->device);
        VecArg X(x, A->ncols, mem, A->stream);
        OutArg Y(y, A->nrows, mem, A->stream);
        RedParams none{};
        launch_spmv(A, A->stream, SPMV_PLAIN, X.dptr, Y.dptr, nullptr, none, 0);
        Y.finish();
    });
}

int sparsla_spmv_transpose(sparsla_dcsr* H, const double* x, double* y, int32_t mem) {
    return guarded([&] {
        need(H, "matrix");
        DevCsr* A = H->A;
        DeviceGuard g(A->device);
        DevCsr* T = A->get_transpose();
        VecArg X(x, A->nrows, mem, T->stream);
        OutArg Y(y, A->ncols, mem, T->stream);
        RedParams none{};
        launch_spmv(T, T->stream, SPMV_PLAIN, X.dptr, Y.dptr, nullptr, none, 0);
        Y.finish();
    });
}

int sparsla_dot(int device, int64_t n, const double* a, const double* b, int32_t mem, double* out) {
    return guarded([&] {
        DeviceGuard g(device);
        if (n < 0) fail(SPARSLA_ERR_DIMENSION, "negative length");
        VecArg A(a, n, mem, nullptr), B(b, n, mem, nullptr);
        CK(cudaDeviceSynchronize());
        *out = device_dot(device, n, A.dptr, B.dptr, nullptr);
    });
}

int sparsla_jacobi(sparsla_dcsr* H, double* dinv, int32_t mem) {
    return guarded([&] {
        need(H, "matrix");
        DevCsr* A = H->A;
        DeviceGuard g(A->device);
        const double* d = A->jacobi_dinv();
        CK(cudaMemcpyAsync(dinv, d, A->nrows * sizeof(double),
                           mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, A->stream));
        CK(cudaStreamSynchronize(A->stream));
    });
}

int sparsla_cg_solve(sparsla_dcsr* A, const double* b, double* x, const sparsla_solve_options* o,
                     sparsla_solve_report* rep, int32_t mem) {
    return krylov(A, SPARSLA_BACKEND_CG, b, x, o, rep, mem);
}

int sparsla_bicgstab_solve(sparsla_dcsr* A, const double* b, double* x, const sparsla_solve_options* o,
                           sparsla_solve_report* rep, int32_t mem) {
    return krylov(A, SPARSLA_BACKEND_BICGSTAB, b, x, o, rep, mem);
}

int sparsla_adjoint_backward(sparsla_dcsr* H, const double* x, const double* grad_x, int32_t backend,
                             const sparsla_solve_options* o, double* grad_b, double* grad_vals,
                             sparsla_solve_report* rep, int32_t mem) {
    return guarded([&] {
        need(H, "matrix"); need(o, "options"); need(rep, "report");
        DevCsr* A = H->A;
        if (A->nrows != A->ncols) fail(SPARSLA_ERR_DIMENSION, "adjoint requires a square matrix");
        if (backend != SPARSLA_BACKEND_CG && backend != SPARSLA_BACKEND_BICGSTAB)
            fail(SPARSLA_ERR_INVALID_ARGUMENT, "unknown backend");
        DeviceGuard g(A->device);
        const long long n = A->nrows;
        VecArg X(x, n, mem, A->stream), G(grad_x, n, mem, A->stream);
        OutArg GB(grad_b, n, mem, A->stream), GV(grad_vals, A->nnz, mem, A->stream);
        // grad_x == 0 exactly -> lambda = 0 short-circuit
        bool all_zero = true;
        {
            std::vector<double> hg(n);
            if (n) CK(cudaMemcpyAsync(hg.data(), G.dptr, n * sizeof(double), cudaMemcpyDeviceToHost, A->stream));
            CK(cudaStreamSynchronize(A->stream));
            for (double v : hg) if (v != 0.0) { all_zero = false; break; }
        }
        std::memset(rep, 0, sizeof(*rep));
        rep->backend = backend;
        if (all_zero) {
            if (n) CK(cudaMemsetAsync(GB.dptr, 0, n * sizeof(double), A->stream));
            rep->converged = 1;
            std::snprintf(rep->diagnostic, 128, "grad_x == 0: short-circuit");
        } else {
            // exactly one solve with A^T (A itself when it is exactly symmetric: same bits)
            DevCsr* AT = A->exactly_symmetric() ? A : A->get_transpose();
            Solver S(AT, backend, *o);
            S.set_b(G.dptr, SPARSLA_MEM_DEVICE);
            S.x = GB.dptr;
            S.reset();
            S.run();
            S.report(rep);
            CK(cudaStreamSynchronize(AT->stream));
        }
        if (n) adjoint_gather_kernel<<<grid_for(n, 256), 256, 0, A->stream>>>(A->rp, A->ci, n, GB.dptr, X.dptr, GV.dptr);
        CK(cudaGetLastError());
        GB.finish();
        GV.finish();
    });
}

int sparsla_solver_create(sparsla_dcsr* H, int32_t backend, const double* b, int32_t mem,
                          const sparsla_solve_options* o, sparsla_solver** out) {
    return guarded([&] {
        need(H, "matrix"); need(o, "options"); need(out, "out");
        if (backend != SPARSLA_BACKEND_CG && backend != SPARSLA_BACKEND_BICGSTAB)
            fail(SPARSLA_ERR_INVALID_ARGUMENT, "unknown backend");
        auto S = std::make_unique<Solver>(H->A, backend, *o);
        S->set_b(b, mem);
        if (mem == SPARSLA_MEM_HOST) {  // keep a resident copy: b may be freed by the caller
            DeviceGuard g(H->A->device);
            CK(cudaStreamSynchronize(S->stream));
        }
        S->reset();
        *out = new sparsla_solver{S.release(), nullptr, 0};
    });
}

int sparsla_solver_reset(sparsla_solver* S) { return guarded([&] { S->S->reset(); }); }
int sparsla_solver_iterate(sparsla_solver* S, int64_t iters) { return guarded([&] { S->S->iterate(iters); }); }
int sparsla_solver_run(sparsla_solver* S) { return guarded([&] { S->S->run(); }); }
int sparsla_solver_report(sparsla_solver* S, sparsla_solve_report* rep) {
    return guarded([&] { S->S->report(rep); });
}
int sparsla_solver_get_x(sparsla_solver* S, double* x, int32_t mem) {
    return guarded([&] {
        Solver* s = S->S;
        DeviceGuard g(s->A->device);
        s->flush_x();
        CK(cudaMemcpyAsync(x, s->x, s->n * sizeof(double),
                           mem == SPARSLA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
    });
}
int sparsla_solver_stream(sparsla_solver* S, void** stream) {
    return guarded([&] { *stream = reinterpret_cast<void*>(S->S->stream); });
}
int sparsla_solver_launches_per_iteration(sparsla_solver* S, int64_t* l) {
    return guarded([&] { *l = S->S->launches_per_iteration(); });
}
int sparsla_solver_kernel_times(sparsla_solver* S, int64_t iters, double* ms) {
    return guarded([&] {
        if (iters < 1) fail(SPARSLA_ERR_INVALID_ARGUMENT, "iters >= 1");
        S->S->kernel_times(iters, ms);
    });
}
int sparsla_solver_destroy(sparsla_solver* S) {
    return guarded([&] {
        if (!S) return;
        delete S->S;
        delete S;
    });
}

int sparsla_spmv_bench(sparsla_dcsr* H, int32_t reps, double* ms) {
    return guarded([&] {
        DevCsr* A = H->A;
        DeviceGuard g(A->device);
        double* xin = dalloc<double>(A->ncols + 2);
        double* y = dalloc<double>(A->nrows + 2);
        if (A->ncols) fill_kernel<<<grid_for(A->ncols, 256), 256, 0, A->stream>>>(xin, A->ncols, 1.0);
        RedParams none{};
        launch_spmv(A, A->stream, SPMV_PLAIN, xin, y, nullptr, none, 0);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, A->stream));
        for (int i = 0; i < reps; ++i) launch_spmv(A, A->stream, SPMV_PLAIN, xin, y, nullptr, none, 0);
        CK(cudaEventRecord(e1, A->stream));
        CK(cudaEventSynchronize(e1));
        float t = 0;
        CK(cudaEventElapsedTime(&t, e0, e1));
        *ms = t / std::max(1, reps);
        cudaEventDestroy(e0); cudaEventDestroy(e1);
        cudaFree(xin); cudaFree(y);
    });
}

}  // extern "C"
