/*
 * sparsla_c.h — C ABI of the B200-native sparse Krylov solve loop (libsparsla_b200.so).
 *
 * Drop-in boundary for the reference's sparse-tensor / solve API in proj/core
 * (namespace sparsla, /root/reference/proj/core/include/sparsla/sparse.hpp:18-149 and
 * the SPEC.md:122-544 contracts whose sources are missing from the reference tree).
 * The C++ headers in include/sparsla/ are header-only wrappers over this ABI that keep
 * the reference's signatures and exception classes (errors.hpp:9-62).
 *
 * Conventions
 *   - Every function returns a sparsla_status (0 = OK).  The message of the last error on
 *     the calling thread is sparsla_last_error_message().
 *   - Index arrays use the reference layout (int64, sparse.hpp:20) unless the name ends in
 *     _i32.  On the device the library stores int32 local indices and fp64 values.
 *   - `mem` selects whether vector pointers are host (SPARSLA_MEM_HOST: copied in/out inside
 *     the call) or device (SPARSLA_MEM_DEVICE: resident, zero-copy) memory.
 *   - Each device handle binds one CUDA device and owns one non-default stream; calls on
 *     distinct handles are reentrant.
 *   - There is no CPU fallback: device entry points fail with SPARSLA_ERR_NO_DEVICE when no
 *     CUDA device is visible.
 */
#ifndef SPARSLA_C_H
#define SPARSLA_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One code per exception class of errors.hpp:9-62, plus device/transport failures. */
typedef enum {
    SPARSLA_OK = 0,
    SPARSLA_ERR_DIMENSION = 1,        /* DimensionError        errors.hpp:15-18 */
    SPARSLA_ERR_BOUNDS = 2,           /* BoundsError           errors.hpp:21-24 */
    SPARSLA_ERR_FORMAT = 3,           /* FormatError           errors.hpp:27-38 */
    SPARSLA_ERR_SINGULAR = 4,         /* SingularMatrixError   errors.hpp:41-44 */
    SPARSLA_ERR_UNSUPPORTED = 5,      /* UnsupportedInputError errors.hpp:48-51 */
    SPARSLA_ERR_INVALID_ARGUMENT = 6, /* InvalidArgumentError  errors.hpp:53-56 */
    SPARSLA_ERR_TRANSPORT = 7,        /* TransportError        errors.hpp:59-62 */
    SPARSLA_ERR_CUDA = 8,             /* -> Error */
    SPARSLA_ERR_NCCL = 9,             /* -> TransportError */
    SPARSLA_ERR_NO_DEVICE = 10,       /* -> Error */
    SPARSLA_ERR_INTERNAL = 11         /* -> Error */
} sparsla_status;

typedef enum { SPARSLA_MEM_HOST = 0, SPARSLA_MEM_DEVICE = 1 } sparsla_mem;
typedef enum { SPARSLA_PRECOND_NONE = 0, SPARSLA_PRECOND_JACOBI = 1 } sparsla_precond;
typedef enum { SPARSLA_BACKEND_CG = 0, SPARSLA_BACKEND_BICGSTAB = 1 } sparsla_backend;

/* SolveOptions: atol >= 0, rtol >= 0, not both zero, max_iter >= 1. */
typedef struct {
    double atol;
    double rtol;
    int64_t max_iter;
    int32_t preconditioner; /* sparsla_precond */
    int32_t _pad;
} sparsla_solve_options;

/* SolveReport.  Non-convergence and breakdown are reported here, not
 * returned as errors. */
typedef struct {
    int64_t iterations;
    int64_t spmv_count;
    double residual_norm;
    int32_t converged;
    int32_t backend; /* sparsla_backend */
    char diagnostic[128];
} sparsla_solve_report;

const char* sparsla_last_error_message(void);
int sparsla_version(void); /* major*10000 + minor*100 + patch */

/* ======================= host-side sparse core (no GPU needed) ======================= */

/* SparseCoo canonicalizing constructor (sparse.hpp:43-47, sparse.cpp:9-53): stable order
 * by (row, col), duplicates summed in input order, explicit zeros kept.  Outputs have room
 * for nnz entries; *out_nnz receives the canonical count. */
int sparsla_coo_canonicalize(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                             const int64_t* cols, const double* vals, int64_t* out_nnz,
                             int64_t* rows_out, int64_t* cols_out, double* vals_out);
/* The same canonicalization on a GPU (radix sort of (row*ncols + col, input position), duplicate
 * sums in input order): bit-identical outputs and errors; nnz < 2^31; `mem` selects host or
 * device pointers for inputs and outputs alike. */
int sparsla_coo_canonicalize_device(int device, int64_t nrows, int64_t ncols, int64_t nnz,
                                    const int64_t* rows, const int64_t* cols, const double* vals,
                                    int32_t mem, int64_t* out_nnz, int64_t* rows_out,
                                    int64_t* cols_out, double* vals_out);
/* The canonicalization's permutation on a GPU: order[j] = input entry at sorted position j
 * (stable by (row, col)), group[j] = the canonical entry it is summed into (ascending from 0);
 * *out_nnz = number of canonical entries.  Bounds errors as above. */
int sparsla_coo_sort_device(int device, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                            const int64_t* cols, int32_t mem, int64_t* out_nnz, int64_t* order,
                            int64_t* group);
/* SparseCoo::with_values for triplets that carried duplicates (sparse.hpp:58-61 over the
 * pattern sparse.cpp:9-53 built): DEVICE arrays order/group from sparsla_coo_sort_device and
 * input-order vals[nnz] -> canonical vals_out[nout], each sum left to right in input order. */
int sparsla_coo_group_sum_device(int device, int64_t nnz, int64_t nout, const int64_t* order,
                                 const int64_t* group, const double* vals, double* vals_out);
/* CsrMatrix::from_coo (sparse.hpp:84, sparse.cpp:94-116), input must be canonical. */
int sparsla_csr_from_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                         const int64_t* cols, const double* vals, int64_t* row_ptr,
                         int64_t* col_idx, double* vals_out);
/* CsrMatrix::to_coo (sparse.hpp:86-87, sparse.cpp:118-127): expands row ids. */
int sparsla_csr_to_coo_rows(int64_t nrows, const int64_t* row_ptr, int64_t* rows_out);
/* canonical A^T as CSR (transpose, sparse.hpp:141, sparse.cpp:176-182). */
int sparsla_csr_transpose(int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                          const int64_t* col_idx, const double* vals, int64_t* t_row_ptr,
                          int64_t* t_col_idx, double* t_vals);
/* is_structurally_symmetric / is_symmetric (sparse.hpp:144-147, sparse.cpp:184-205) on a
 * canonical CSR.  out = 0/1. */
int sparsla_csr_symmetry(int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                         const int64_t* col_idx, const double* vals, double tol,
                         int32_t* structurally_symmetric, int32_t* symmetric);

/* Problem generators (SPEC.md:551-569 + SURVEY.md §8d), emitting canonical CSR rows
 * [row_begin, row_end) directly (equal, bit for bit, to SparseCoo canonicalization of the
 * element-order triplets).  kind: 0 poisson2d(N=p1), 1 poisson3d(N=p1),
 * 2 convdiff3d(N=p1, c=fparam), 3 fem2d(m=p1, seed=p2), 4 poisson3d box N x N x Nz
 * (N=p1, Nz=p2; the weak-scaling slabs of config E).
 * sparsla_gen_size: global n and the nnz of the row range.
 * sparsla_gen_csr: row_ptr[row_end-row_begin+1] (starts at 0), col_idx/vals[nnz]. */
int sparsla_gen_size(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t row_begin,
                     int64_t row_end, int64_t* n_global, int64_t* nnz_range);
int sparsla_gen_csr(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t row_begin,
                    int64_t row_end, int64_t* row_ptr, int64_t* col_idx, double* vals);
int sparsla_gen_csr_i32(int32_t kind, int64_t p1, int64_t p2, double fparam,
                        int64_t row_begin, int64_t row_end, int32_t* row_ptr,
                        int32_t* col_idx, double* vals);
/* 2-D node coordinates (kind 0 grid, kind 3 FEM interior nodes) for partition_rcb. */
int sparsla_gen_coords(int32_t kind, int64_t p1, int64_t p2, double* xs, double* ys);

/* Partitioners. */
int sparsla_partition_contiguous(int64_t n, int32_t nparts, int32_t* part_of);
int sparsla_partition_rcb(int64_t n, const double* xs, const double* ys, int32_t nparts,
                          int32_t* part_of);

/* build_local for a structurally symmetric pattern, from this rank's
 * owned rows only.  Inputs: part_of[n_global] (NULL = contiguous partition
 * partition_contiguous(n_global, nparts)), the owned rows (ascending global ids) as a
 * CSR with GLOBAL column ids.  The result handle exposes the SPEC-layout maps:
 *   owned (ascending global), halo (ascending global), neighbors (ascending rank),
 *   send_ptr/send_idx, recv_ptr/recv_idx (local positions in [owned | halo], canonical
 *   global order), and the local matrix with columns relabelled to [owned | halo] while
 *   every row keeps its global column order (so local SpMV reproduces serial row sums).
 * sizes[0]=n_owned [1]=n_halo [2]=n_neighbors [3]=nnz_local [4]=total_send [5]=total_recv */
typedef struct sparsla_local sparsla_local;
int sparsla_local_build(int64_t n_global, const int32_t* part_of, int32_t nparts, int32_t rank,
                        int64_t n_owned, const int64_t* owned, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* vals, sparsla_local** out);
int sparsla_local_sizes(const sparsla_local* L, int64_t* sizes);
int sparsla_local_get(const sparsla_local* L, int64_t* owned, int64_t* halo, int32_t* neighbors,
                      int64_t* send_ptr, int64_t* send_idx, int64_t* recv_ptr,
                      int64_t* recv_idx, int64_t* l_row_ptr, int64_t* l_col_idx,
                      double* l_vals);
int sparsla_local_destroy(sparsla_local* L);

/* Matrix Market coordinate I/O (matrix_market.hpp:10-20): real
 * general|symmetric, '%' comments, 1-based -> 0-based, symmetric expanded, result
 * canonical (SparseCoo).  SPARSLA_ERR_FORMAT with "(line N)" on malformed input.  The writer
 * emits coordinate/real/general with 17 significant digits (bit-exact round trip). */
typedef struct sparsla_coo sparsla_coo;
int sparsla_mtx_read(const char* path, sparsla_coo** out);
int sparsla_mtx_read_buffer(const char* data, int64_t len, sparsla_coo** out);
int sparsla_coo_sizes(const sparsla_coo* coo, int64_t* nrows, int64_t* ncols, int64_t* nnz);
int sparsla_coo_get(const sparsla_coo* coo, int64_t* rows, int64_t* cols, double* vals);
int sparsla_coo_destroy(sparsla_coo* coo);
int sparsla_mtx_write(const char* path, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                      const int64_t* cols, const double* vals);

/* ============================ device CSR (one GPU) =================================== */
typedef struct sparsla_dcsr sparsla_dcsr;

int sparsla_device_count(int* count);
/* Upload a canonical CSR (reference int64 layout) to `device`.  Rows must have strictly
 * increasing columns (CsrMatrix invariant, sparse.hpp:76-78). */
int sparsla_dcsr_create(int device, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* vals, sparsla_dcsr** out);
/* Same with int32 host arrays (no index conversion on the host). */
int sparsla_dcsr_create_i32(int device, int64_t nrows, int64_t ncols, const int32_t* row_ptr,
                            const int32_t* col_idx, const double* vals, sparsla_dcsr** out);
/* SparseCoo::with_values (sparse.hpp:58-61): same pattern, new values. */
int sparsla_dcsr_set_values(sparsla_dcsr* A, const double* vals, int32_t mem);
int sparsla_dcsr_destroy(sparsla_dcsr* A);
/* info[0]=nrows [1]=ncols [2]=nnz [3]=device bytes of the matrix [4]=max nnz per 256-row
 * block [5]=max row length [6]=kernel variant used by spmv (0 staged, 1 long-row)
 * [7]=staged-SpMV variant index (8 entries) */
int sparsla_dcsr_info(const sparsla_dcsr* A, int64_t* info);
/* Long-row split chosen from the row-length histogram (single GPU): out[0]=rows summed
 * warp-per-row, out[1]=their entries, out[2]=the length threshold (0: no split).
 * SPARSLA_LONG_ROW=<n> forces the threshold at matrix creation, 0 disables. */
int sparsla_dcsr_long_rows(const sparsla_dcsr* A, int64_t* out);
/* Storage format chosen for the SpMV stream: fmt[0]=1 when the value dictionary is in use
 * (<= 256 distinct values: 1-byte index per entry instead of the 8-byte value), fmt[1]=number
 * of distinct values in it (0 otherwise), fmt[2]=1 when the Jacobi inverse diagonal is
 * constant (the CG/BiCGStab vector kernels then take it as a scalar). */
int sparsla_dcsr_format(sparsla_dcsr* A, int64_t* fmt);
/* x-window staging of the SpMV (banded / mesh-ordered matrices): out[0]=x-window kernel
 * variant for the current value stream (-1: none built), out[1]=staged x elements per
 * 256-row round, out[2]=parts per million of the entries whose x operand is staged,
 * out[3]=bit m set when SpMV mode m (0 plain, 1 CG p.q, 2 BiCGStab r-hat.v, 3 BiCGStab
 * t.t/t.s) runs the x-window kernel, out[4]=its value stream (0 fp64 values, 1 1-byte
 * dictionary indices, 2 "pair": the dictionary index inside the 16-bit offset), out[5]=its
 * resident CTAs per SM, out[6..7] reserved (0).  out has 8 entries.  SPARSLA_XWIN at
 * matrix creation: 0 disables, 1 (the default) stages when it pays, 2 forces every mode.
 * (When the diagonal-warp kernel is on, sparsla_dcsr_dia, it takes every SpMV instead.) */
int sparsla_dcsr_xwin(const sparsla_dcsr* A, int64_t* out);
/* diagonal-warp SpMV (stencil-like matrices: >= 90% of the 32-row warps have all rows on
 * the same <= 7 diagonals with the same dictionary values, up to two missing entries):
 * out[0]=bit m set when SpMV mode m (as in sparsla_dcsr_xwin) runs the diagonal-warp
 * kernel, out[1]=parts per million of structured warps (last build, also when below the
 * threshold), out[2]=matrix bytes one such SpMV reads (48-byte warp entries + the other
 * warps' CSR), out[3]=distinct patterns when the pattern-table kernel runs (a 4-byte word
 * per 32-row warp; the <= 64 patterns travel as a kernel parameter), else 0.  4 entries.
 * SPARSLA_DIA=0 at creation / set_values disables. */
int sparsla_dcsr_dia(const sparsla_dcsr* A, int64_t* out);

/* y = A x (sparse.cpp:135-154): rows accumulated left to right from 0.0, separate
 * multiply and add — bitwise equal to the reference.  mem: see above. */
int sparsla_spmv(sparsla_dcsr* A, const double* x, double* y, int32_t mem);
/* y = A^T x (spmv_transpose, sparse.cpp:156-174), via an explicit canonical A^T kept on
 * the device, bitwise equal to the reference scatter order. */
int sparsla_spmv_transpose(sparsla_dcsr* A, const double* x, double* y, int32_t mem);
/* canonical dot of two device/host vectors. */
int sparsla_dot(int device, int64_t n, const double* a, const double* b, int32_t mem,
                double* out);
/* Jacobi inverse diagonal (jacobi_build). */
int sparsla_jacobi(sparsla_dcsr* A, double* dinv, int32_t mem);

/* cg_solve / bicgstab_solve, x0 = 0. */
int sparsla_cg_solve(sparsla_dcsr* A, const double* b, double* x,
                     const sparsla_solve_options* opts, sparsla_solve_report* report,
                     int32_t mem);
int sparsla_bicgstab_solve(sparsla_dcsr* A, const double* b, double* x,
                           const sparsla_solve_options* opts, sparsla_solve_report* report,
                           int32_t mem);

/* solve_backward (Alg. 1): exactly one solve A^T lam = grad_x
 * with `backend`; grad_b = lam; grad_vals[k] = -(lam[row_k] * x[col_k]) in CSR (= canonical
 * COO) order.  A exactly-symmetric A is reused as its own transpose. */
int sparsla_adjoint_backward(sparsla_dcsr* A, const double* x, const double* grad_x,
                             int32_t backend, const sparsla_solve_options* opts,
                             double* grad_b, double* grad_vals, sparsla_solve_report* report,
                             int32_t mem);

/* ===================== eigen-solver (Eq. 4) ================== */
/* eig_smallest options: a pair converges when ||A v - lambda v||_2 <= tol. */
typedef struct {
    double tol;
    int64_t max_iter;
    uint64_t seed;          /* initial block, counter-based hash; e.g. 2601 */
    int32_t preconditioner; /* sparsla_precond: JACOBI or NONE */
    int32_t _pad;
} sparsla_eig_options;

/* EigenResult.report.  Non-convergence is reported with per-pair flags,
 * not returned as an error. */
typedef struct {
    int64_t iterations;
    int64_t spmm_count;      /* block SpMV launches */
    int64_t converged_pairs;
    int32_t converged;       /* all k pairs converged */
    int32_t method;          /* 0 = LOBPCG, 1 = dense Rayleigh-Ritz on the full space */
    char diagnostic[128];
} sparsla_eig_report;

/* eig_smallest: the k smallest eigenpairs of a symmetric A (pattern and
 * values checked to 1e-12, else SPARSLA_ERR_UNSUPPORTED), 1 <= k <= 16 and k <= n/4 above
 * the dense threshold (64 rows; env SPARSLA_EIG_DENSE_THRESHOLD).  Jacobi-preconditioned
 * LOBPCG on the GPU.  lambdas[k] ascending; vectors row-major n x k (column m = v_m,
 * ||v_m|| = 1, largest-magnitude component positive); residual_norms[k] and
 * pair_converged[k] may be NULL. */
int sparsla_eig_smallest(sparsla_dcsr* A, int64_t k, const sparsla_eig_options* opts,
                         double* lambdas, double* vectors, double* residual_norms,
                         int32_t* pair_converged, sparsla_eig_report* report, int32_t mem);
/* eig_backward (Eq. 4): grad_vals[e] = sum_m grad_lambdas[m] v_m[i_e] v_m[j_e]
 * in CSR (= canonical COO) order, no linear solves.  Degenerate eigenvalues (consecutive gap
 * <= 1e-8) -> SPARSLA_ERR_UNSUPPORTED.  lambdas and grad_lambdas are host arrays; vectors
 * (n x k) and grad_vals (nnz) follow `mem`. */
int sparsla_eig_backward(sparsla_dcsr* A, int64_t k, const double* lambdas, const double* vectors,
                         const double* grad_lambdas, double* grad_vals, int32_t mem);

/* ============ bench / instrumentation hooks (persistent device-resident solver) ========= */
/* A prepared solver keeps b, x and all work vectors resident and captures the iteration
 * in a CUDA graph; `iterate` runs up to `iters` more iterations (stops early when the
 * solve terminates).  Used by bench.py to time iterations with inputs resident in HBM. */
typedef struct sparsla_solver sparsla_solver;
int sparsla_solver_create(sparsla_dcsr* A, int32_t backend, const double* b, int32_t mem,
                          const sparsla_solve_options* opts, sparsla_solver** out);
int sparsla_solver_reset(sparsla_solver* S); /* x = 0, initial residual, state reset */
int sparsla_solver_iterate(sparsla_solver* S, int64_t iters);
int sparsla_solver_run(sparsla_solver* S); /* to termination */
int sparsla_solver_report(sparsla_solver* S, sparsla_solve_report* report);
int sparsla_solver_get_x(sparsla_solver* S, double* x, int32_t mem);
/* device pointer of the handle's CUDA stream (cudaStream_t), for event timing */
int sparsla_solver_stream(sparsla_solver* S, void** stream);
/* number of kernel launches one iteration issues */
int sparsla_solver_launches_per_iteration(sparsla_solver* S, int64_t* launches);
/* run `iters` iterations launched individually with CUDA events around every kernel; ms[k]
 * = average duration of the k-th kernel of an iteration (launches_per_iteration entries) */
int sparsla_solver_kernel_times(sparsla_solver* S, int64_t iters, double* ms);
int sparsla_solver_destroy(sparsla_solver* S);
/* time `reps` SpMV launches on the handle stream, returns avg ms per launch */
int sparsla_spmv_bench(sparsla_dcsr* A, int32_t reps, double* ms_per_launch);

/* ===================== distributed (row partition, 1..8 GPUs) ======================= */
/* One handle per rank.  All calls below are collective over the ranks of the handle.
 * NCCL backing: one rank per GPU (one process per GPU, e.g. torchrun); the 128-byte id
 * comes from sparsla_nccl_unique_id on rank 0 and is broadcast by the caller.
 * Local backing: P ranks as threads of one process sharing a sparsla_local_hub (they may
 * share one device) — the in-process-worker model of SPEC.md:529. */
typedef struct sparsla_dist sparsla_dist;
typedef struct sparsla_local_hub sparsla_local_hub;
int sparsla_nccl_unique_id(unsigned char* id128);
int sparsla_dist_create_nccl(int device, int nranks, int rank, const unsigned char* id128,
                             const sparsla_local* L, sparsla_dist** out);
/* Host-callback backing (setup / init traffic through caller-provided collectives, e.g.
 * torch.distributed gloo; host buffers, synchronous).  Combined with sparsla_dist_set_fused
 * the iterations use cudaIpc peer memory only, so several processes may share one GPU. */
typedef struct {
    void* user;
    int (*allgather)(void* user, const double* send, double* recv, int64_t count);
    int (*exchange)(void* user, int32_t npeers, const int32_t* ranks, const double* const* sbuf,
                    const int64_t* scount, double* const* rbuf, const int64_t* rcount);
} sparsla_host_transport;
int sparsla_dist_create_host(int device, int nranks, int rank, const sparsla_host_transport* T,
                             const sparsla_local* L, sparsla_dist** out);
int sparsla_local_hub_create(int nranks, sparsla_local_hub** out);
int sparsla_local_hub_destroy(sparsla_local_hub* hub);
int sparsla_dist_create_local(int device, sparsla_local_hub* hub, int rank, const sparsla_local* L,
                              sparsla_dist** out);
int sparsla_dist_destroy(sparsla_dist* D);
/* ---- Transport as a first-class object ----
 * One per rank; plans built on it share it (and its counters).  Backings: NCCL (one rank per
 * GPU), in-process ranks (threads on a sparsla_local_hub) and host callbacks (e.g.
 * torch.distributed gloo). */
typedef struct sparsla_transport sparsla_transport;
int sparsla_transport_create_nccl(int device, int nranks, int rank, const unsigned char* nccl_id,
                                  sparsla_transport** out);
int sparsla_transport_create_local(int device, sparsla_local_hub* hub, int rank, sparsla_transport** out);
int sparsla_transport_create_host(int device, int nranks, int rank, const sparsla_host_transport* T,
                                  sparsla_transport** out);
int sparsla_transport_destroy(sparsla_transport* T);
/* all_reduce_sum: sum of every rank's scalar in ascending rank order. */
int sparsla_transport_all_reduce_sum(sparsla_transport* T, double local, double* global);
/* out[0]=nranks [1]=rank [2]=exchanges [3]=all-gathers [4]=messages (raw transport calls) */
int sparsla_transport_info(const sparsla_transport* T, int64_t* out);
/* build this rank's device plan for L on T's device (collective over T) */
int sparsla_dist_create(sparsla_transport* T, const sparsla_local* L, sparsla_dist** out);
/* halo_exchange: halo[n_halo] = the neighbours' owned values of this
 * rank's halo nodes (ascending global index), from x_owned.  Collective. */
int sparsla_dist_halo_exchange(sparsla_dist* D, const double* x_owned, double* halo, int32_t mem);
/* info[0]=n_owned [1]=n_halo [2]=neighbors [3]=interior chunks [4]=boundary chunks [5]=P
 * [6]=rank [7]=zero-copy halo segments [8]=n_global */
int sparsla_dist_info(const sparsla_dist* D, int64_t* info);
/* this rank's local-matrix storage format (same fields as sparsla_dcsr_format) */
int sparsla_dist_format(sparsla_dist* D, int64_t* fmt);
/* this rank's local-matrix x-window staging (same fields as sparsla_dcsr_xwin) */
int sparsla_dist_xwin(const sparsla_dist* D, int64_t* out);
/* this rank's local-matrix diagonal-warp kernel (same fields as sparsla_dcsr_dia) */
int sparsla_dist_dia(const sparsla_dist* D, int64_t* out);
/* counters[0]=halo exchanges [1]=all_reduce points [2]=p2p messages performed by the live
 * algorithm (SPEC.md:524 accounting); [3..5] = raw transport calls of the same kinds (they
 * also include the no-op tail replayed after convergence).  6 entries. */
int sparsla_dist_counters(const sparsla_dist* D, int64_t* counters);
int sparsla_dist_reset_counters(sparsla_dist* D);
/* Fused peer-memory collectives for distributed CG (default off; SPARSLA_P2P=1 also
 * enables): per iteration no NCCL call — reduction totals and halo values are stored by
 * the kernels straight into the peers' memory (NVLink / cudaIpc, or same-device for
 * in-process ranks) with release/acquire epoch flags.  Must be set identically on all
 * ranks before a solve. */
int sparsla_dist_set_fused(sparsla_dist* D, int32_t on);
/* SparseCoo::with_values (sparse.hpp:58-61) on this rank's local matrix: new values in the
 * local entry order of the sparsla_local it was built from (owned rows ascending, entries in
 * global column order).  Collective (a barrier over the transport: no peer may still use a
 * parked solver's peer mappings); drops the plan's parked solvers and the A^T values. */
int sparsla_dist_set_values(sparsla_dist* D, const double* vals_local, int32_t mem);
/* dist_spmv */
int sparsla_dist_spmv(sparsla_dist* D, const double* x_owned, double* y_owned, int32_t mem);
/* dist_cg (Alg. 4) / distributed BiCGStab, SolveOptions as cg_solve */
int sparsla_dist_cg_solve(sparsla_dist* D, const double* b_owned, double* x_owned,
                          const sparsla_solve_options* opts, sparsla_solve_report* report,
                          int32_t mem);
int sparsla_dist_bicgstab_solve(sparsla_dist* D, const double* b_owned, double* x_owned,
                                const sparsla_solve_options* opts, sparsla_solve_report* report,
                                int32_t mem);
/* dist_adjoint_solve; vals_t = A^T values in A's local entry order, or
 * NULL when A is symmetric; grad_vals in the local entry order */
int sparsla_dist_adjoint_backward(sparsla_dist* D, const double* x_owned, const double* grad_x_owned,
                                  const double* vals_t, int32_t backend,
                                  const sparsla_solve_options* opts, double* grad_b_owned,
                                  double* grad_vals_local, sparsla_solve_report* report,
                                  int32_t mem);
/* gather_solution: x_global (host, n_global) written on rank 0 only */
int sparsla_dist_gather(sparsla_dist* D, const double* x_owned, double* x_global, int32_t mem);
/* persistent distributed solver (bench): use the sparsla_solver_* calls on the result */
int sparsla_dist_solver_create(sparsla_dist* D, int32_t backend, const double* b_owned, int32_t mem,
                               const sparsla_solve_options* opts, sparsla_solver** out);

#ifdef __cplusplus
}
#endif
#endif /* SPARSLA_C_H */
