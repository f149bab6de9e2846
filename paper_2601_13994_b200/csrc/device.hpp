// device.hpp — device-side objects of libsparsla_b200 (host declarations).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

#include "copy_sync.hpp"
#include "kernels.cuh"
#include "sparsla_c.h"

namespace sparsla_b200 {

void cuda_check(cudaError_t e, const char* what);

struct DeviceGuard {
    explicit DeviceGuard(int dev, bool nothrow = false);
    ~DeviceGuard();
    int prev_ = 0;
};

// Device CSR: int32 row_ptr / col_idx (padded for the bulk-copy over-read), fp64 values.
struct DevCsr {
    int device = 0;
    long long nrows = 0, ncols = 0, nnz = 0;
    int32_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* val = nullptr;
    long long max_block_nnz = 0, max_row = 0;
    int cap_v = 0, cap_c = 0;      // per 256-row round (+alignment slack)
    int cap_v32 = 0, cap_c32 = 0;  // per 32-row warp segment
    size_t smem_bytes = 0;
    bool staged = true;
    int l2_keep = 0;  // matrix stream L2 policy (see DevCsr::create)
    int ws_var = 0;   // staged-SpMV variant (choose_ws_variant)
    bool has_hub = false;  // rounds above the stage capacity exist (bypass kernels)
    bool local_layout = false;  // rank-local [owned | halo] columns (diagonal of row i is column i)
    int ws_ctas[8] = {0};  // persistent grid per staged-SpMV variant (SMs x resident CTAs)
    int vdt_ctas = 0;      // persistent grid of the BiCGStab t-SpMV dictionary kernel (8-wide)
    double* dinv = nullptr;
    double* ones = nullptr;
    uint8_t* vidx = nullptr;  // value dictionary (<= 256 distinct values): 1-byte index per entry
    double* vtab = nullptr;   // [256] distinct values
    bool vd = false;          // staged SpMV streams vidx instead of val
    int nvals = 0;            // distinct values in vtab
    int vd_var = 0;           // value-dictionary kernel variant
    int dinv_uniform = -1;    // 1: every dinv entry has the same bits (dinv_value); -1: unknown
    double dinv_value = 0.0;
    int sym_checked = -1;
    // long rows (single GPU): one warp per row in spmv_longrow_kernel; the staged SpMV runs
    // on a short-row view of the matrix in which those rows are empty
    long long nlong = 0, long_nnz = 0, long_threshold = 0;
    int32_t* long_rows = nullptr;    // [nlong], longest first
    uint32_t* long_bits = nullptr;   // [ceil(n/32)]
    cudaStream_t side = nullptr;     // forked stream of the long-row kernel (launch_spmv)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::mutex split_mu;
    int32_t* s_rp = nullptr;         // short-row view (same padding as rp/ci/val)
    int32_t* s_ci = nullptr;
    double* s_val = nullptr;
    // x windows (spmv_xw.cuh): per-round descriptors of the x segments the staged SpMV
    // streams into shared memory next to the matrix (banded / mesh-ordered matrices)
    int32_t* xw = nullptr;     // [chunks * 8 rounds][kXwDescInts] window descriptors
    uint16_t* xwo = nullptr;   // [nnz + kXwPad] entry -> offset in its round's staged windows
    int cap_x = 0;             // max staged x elements per round
    int xw_mode = 0;           // SPARSLA_XWIN at creation (2: every mode and stream)
    uint16_t* xvo = nullptr;   // [nnz + kXwPad] pair stream: dictionary index << 11 | offset
    int xw_var[3] = {-1, -1, -1};  // x-window kernel variant per value stream [plain, dictionary, pair]
    int xw_ctas[3][2] = {{0, 0}, {0, 0}, {0, 0}};  // persistent grid [stream][aux vector staged]
    // diagonal-warp table (spmv_dia.cuh): [chunks * 64 warps][12], kept when >= 90% of the
    // warps are structured; the SpMV then takes spmv_dia_kernel in every mode
    int32_t* dia = nullptr;
    double dia_frac = 0.0;       // structured warps / warps (last build)
    long long dia_bytes = 0;     // matrix bytes one diagonal-warp SpMV reads
    int dia_ahead = 0;           // chunks ahead a diagonal-warp CTA prefetches (whole waves)
    int dia_var = 0;             // kDiaVariants index
    int dia_modes = 0;           // SpMV modes (bit per SpmvMode) that take it
    uint32_t* diaw = nullptr;    // pattern-table kernel: [chunks * 64 warps] pattern id + exceptions
    unsigned char* diac = nullptr;  // host DiaConst (the deduplicated patterns), kernel parameter
    int dia_npat = 0;            // distinct patterns (0: no pattern table)
    int dia_ctas = 0;            // resident CTAs of the diagonal-warp variant (persistent grid)
    double xw_cover = 0.0;     // fraction of entries whose x operand is staged
    int sms = 0;               // multiprocessors of the device (set with the variants)
    DevCsr* transpose = nullptr;
    cudaStream_t stream = nullptr;
    std::mutex lazy_mu;  // guards the lazily built caches (dinv, ones, symmetry, transpose)
    // one parked host-buffer Krylov solver per backend (workspace + captured graphs), reused
    // by the next cg_solve / bicgstab_solve call with host buffers (SPARSLA_SOLVER_CACHE=0: off)
    std::mutex solver_mu;
    struct Solver* parked[2] = {nullptr, nullptr};
    long long values_version = 0;  // bumped by set_values: a solver built before never parks
    void drop_parked() noexcept;

    template <class I>
    static DevCsr* create(int device, long long nrows, long long ncols, const I* rp, const I* ci,
                          const double* val, bool local_layout = false);
    ~DevCsr();
    const double* jacobi_dinv();
    bool jacobi_uniform(double* value);  // constant Jacobi diagonal? (checked once per values)
    const double* ones_vec();
    bool exactly_symmetric();
    DevCsr* get_transpose();
};

// x-window staging summary (sparsla_dcsr_xwin layout)
void devcsr_xwin_info(const DevCsr* A, int64_t* out);
// diagonal-warp summary (sparsla_dcsr_dia layout)
void devcsr_dia_info(const DevCsr* A, int64_t* out);

// new values in A's entry order (host or device pointer); drops every value-dependent cache
void devcsr_set_values(DevCsr* A, const double* vals, int32_t mem);

// canonical A^T of a device CSR into host arrays (coo_device.cu)
void csr_transpose_device(int device, long long nrows, long long ncols, long long nnz, const int32_t* rp,
                          const int32_t* ci, const double* val, int32_t* trp, int32_t* tci, double* tv);

void launch_spmv(DevCsr* A, cudaStream_t s, int mode, const double* x, double* y, const double* aux,
                 const RedParams& red, int check_done);
unsigned spmv_grid(const DevCsr* A, long long nch, int mode = 0, bool xw_ok = true);
void launch_spmv_part(DevCsr* A, cudaStream_t s, int mode, const double* x, double* y, const double* aux,
                      const RedParams& red, int check_done, const int32_t* list, long long nch,
                      unsigned expected, const P2PCtx* p2p = nullptr, long long n_interior = 0,
                      int halo_v = 0, unsigned grid_cap = 0);

struct Transport;

// One rank's distributed plan on its device (dist.cu): halo maps, interior/boundary chunk
// lists, comm stream and the per-reduction-point all-gather buffers.
struct DistCtx {
    Transport* tr = nullptr;
    int device = 0;
    long long n_owned = 0, n_halo = 0;
    long long halo_base = 0, vec_len = 0;  // device layout [owned | gap | halo]
    std::vector<int> nbr;
    std::vector<long long> s_off, s_cnt, r_off, r_cnt;  // per neighbour into send/recv maps
    std::vector<long long> s_base, r_base;              // contiguous range start, or -1
    int32_t* d_send_idx = nullptr;
    int32_t* d_recv_idx = nullptr;
    double* sendbuf = nullptr;
    double* recvbuf = nullptr;
    int32_t* d_interior = nullptr;
    int32_t* d_boundary = nullptr;
    long long n_interior = 0, n_boundary = 0;
    double* red_send = nullptr;  // [8 points][8]
    double* red_all = nullptr;   // [8 points][P][8]
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_x = nullptr, ev_halo = nullptr;
    bool p2p_enabled = false;     // fused peer-memory collectives (sparsla_dist_set_fused)
    bool p2p_shared_device = false;  // a peer rank runs on this GPU: its kernels compete for the SMs
    int32_t* d_all_chunks = nullptr;  // [interior | boundary] for the single fused-mode launch
    void exchange(cudaStream_t s, double* x);  // halo of x ([owned|halo]) -> ev_halo
    ~DistCtx();
};

// Jacobi-PCG / BiCGStab solver with device-resident state and graph-captured iterations.
struct Solver {
    static constexpr int kGraphIters = 16;
    static void validate(const sparsla_solve_options& o, bool square);
    DevCsr* A;
    int backend;
    sparsla_solve_options opts;
    long long n = 0;
    cudaStream_t stream = nullptr;
    const double* dinv = nullptr;
    bool d_is_uniform = false;   // constant diagonal: the vector kernels take d_uniform, not dinv
    double d_uniform = 0.0;
    const double* b = nullptr;
    double* x = nullptr;
    double *x_own = nullptr, *b_own = nullptr;
    double *r = nullptr, *p = nullptr, *q = nullptr;
    // deferred x update (single-GPU CG, kernels.cuh V_CG_U2E / V_CG_U2O): second direction
    // buffer, host-side iteration parity, and which buffer holds the current direction
    double* p2 = nullptr;
    bool defer_x = false;
    int parity = 0;
    bool swap_p = false;
    double *rh = nullptr, *ph = nullptr, *s = nullptr, *sh = nullptr, *t = nullptr;
    double* partials = nullptr;
    unsigned* tickets = nullptr;
    double* slotsum = nullptr;   // multi_finish scratch [4][kFinalSlots] (SPARSLA_MULTI_FINISH=0: off)
    KState* st = nullptr;
    KState* h_st = nullptr;
    int* h_flag = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaGraphExec_t g_many = nullptr, g_one = nullptr, g_one_odd = nullptr;
    bool fused = false;          // small CG: cg_fused_kernel runs whole iterations
    long long values_version = 0;  // A->values_version when this solver was built
    // fused peer-memory collectives (distributed CG)
    P2PCtx* d_p2p = nullptr;
    int* p2p_err = nullptr;      // device flag raised by a timed-out peer wait (P2PCtx::err)
    std::vector<void*> p2p_allocs, p2p_ipc_opened;
    int fused_grid = 0;
    unsigned* fused_bar = nullptr;
    int fused_res = 0;               // > 0: resident chunk images of this many entries (cg_fused_kernel<true>)

    DistCtx* dist = nullptr;
    Solver(DevCsr* A, int backend, const sparsla_solve_options& o, DistCtx* dist = nullptr);
    ~Solver();
    void release() noexcept;
    void set_b(const double* src, int mem);
    void reset();
    void iterate(long long iters);
    void run();
    void wait_event(cudaEvent_t e);  // distributed: polls the transport, times out
    void report(sparsla_solve_report* rep);
    void flush_x();  // deferred x update: complete x before it is read mid-solve
    long long launches_per_iteration() const;
    void kernel_times(long long iters, double* ms);

    bool capturable() const;

   private:
    void spmv_point(int mode, double* xin, double* y, const double* aux, int scalar, int slot, int check_done);
    template <int OP>
    void vec_point(int scalar, int slot, int check_done);
    void reduce_point(int scalar, int slot, int nd);
    RedParams red(int which, int slot) const;
    VecParams vparams() const;
    void enqueue_init();
    void p2p_setup();     // collective (dist.cu)
    void p2p_release() noexcept;
    void enqueue_fused(long long iters);
    void enqueue_iteration(cudaEvent_t* evs = nullptr, int par = 0);
    void build_graphs();
};

}  // namespace sparsla_b200

struct sparsla_solver {
    sparsla_b200::Solver* S;
    double* x_user;
    int x_mem;
};
