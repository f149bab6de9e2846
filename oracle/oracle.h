/*
 * oracle.h — C ABI of the CPU ORACLE for the sparsla Krylov hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product library (paper_2601_13994_b200/) never links or calls it.
 *
 * The oracle is a plain C++ restatement of the reference's algorithms:
 *   - sparse core            /root/reference/proj/core/src/sparse.cpp:9-205
 *   - linear solvers          SPEC.md:122-206  (cg_solve, bicgstab_solve, jacobi_build)
 *   - adjoint engine          SPEC.md:208-272  (solve_backward), PAPER.md:109-131 (Alg. 1)
 *   - distributed             SPEC.md:417-544  (partition_*, build_local, halo_exchange,
 *                                               dist_spmv, all_reduce_sum, dist_cg,
 *                                               dist_adjoint_solve, gather_solution),
 *                             PAPER.md:247-311 (Alg. 3, Alg. 4)
 *   - generators              SPEC.md:551-569 (poisson2d) + the 3-D / convection-diffusion /
 *                             FEM generators defined in SURVEY.md §8(d)
 * Its SpMV and canonicalization are pinned bit-for-bit against the reference's own
 * compiled sparse.cpp (oracle/_ref, see oracle/Makefile) by tests/test_oracle.py.
 *
 * Choices SPEC leaves open are fixed here and documented in DESIGN.md §3
 * ("canonical dot", Jacobi threshold, BiCGStab side, RCB tie-breaks).
 */
#ifndef SPARSLA_ORACLE_H
#define SPARSLA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double atol;
    double rtol;
    int64_t max_iter;
    int32_t preconditioner; /* 0 none, 1 jacobi */
    int32_t _pad;
} orc_opts;

typedef struct {
    int64_t iterations;
    int64_t spmv_count;
    double residual_norm;
    int32_t converged;
    int32_t backend; /* 0 cg, 1 bicgstab */
    char diagnostic[128];
} orc_report;

void orc_set_threads(int nthreads);
int orc_get_threads(void);

/* ---- canonical dot ---- */
double orc_cdot(int64_t n, const double* a, const double* b);
/* chunk partials only (level 1), m = ceil(n/2048) outputs */
void orc_cdot_partials(int64_t n, const double* a, const double* b, double* partials);

/* ---- sparse core (int64 indices, reference layout sparse.hpp:20) ---- */
/* canonicalize COO: returns nnz_out; outputs sized nnz_in. -1 on bad input. */
int64_t orc_coo_canonicalize(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                             const int64_t* cols, const double* vals, int64_t* rows_out,
                             int64_t* cols_out, double* vals_out);
void orc_csr_from_coo(int64_t nrows, int64_t nnz, const int64_t* rows, const int64_t* cols,
                      const double* vals, int64_t* row_ptr, int64_t* col_idx, double* out_vals);
void orc_spmv(int64_t nrows, const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
              const double* x, double* y);
void orc_csr_transpose(int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                       const int64_t* col_idx, const double* vals, int64_t* t_row_ptr,
                       int64_t* t_col_idx, double* t_vals);
void orc_jacobi(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                double* dinv);

/* ---- solvers ---- returns 0, or 6 (invalid argument) */
int orc_cg(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
           const double* b, double* x, const orc_opts* opts, orc_report* rep);
int orc_bicgstab(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                 const double* b, double* x, const orc_opts* opts, orc_report* rep);
/* run exactly `iters` iterations of the CG loop (ignores tolerance); x and r out */
int orc_cg_fixed(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                 const double* b, int64_t iters, int32_t precond, double* x, double* r);
/* adjoint backward: one solve A^T lam = g; grad_b = lam,
 * grad_vals[k] = -(lam[row_k] * x[col_k]); backend 0 cg, 1 bicgstab */
int orc_adjoint_backward(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                         const double* vals, const double* x, const double* g, int32_t backend,
                         const orc_opts* opts, double* grad_b, double* grad_vals,
                         orc_report* rep);

/* ---- generators: COO triplets in emission order (NOT canonical) ----
 * kind 0 poisson2d(N=p1), 1 poisson3d(N=p1), 2 convdiff3d(N=p1, c=fparam),
 *      3 fem2d(m=p1, seed=p2)
 * With rows==NULL: only *n and *ntrip are written. */
int orc_gen_triplets(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t* n,
                     int64_t* ntrip, int64_t* rows, int64_t* cols, double* vals);
/* ---- generators straight to canonical CSR (int64 row_ptr/col_idx, fp64 vals) ----
 * Same matrices as orc_gen_triplets followed by the SparseCoo canonicalization
 * (sparse.cpp:9-53: stable sort by (row, col), duplicates summed in input order), without
 * the O(nnz log nnz) permutation sort: stencil kinds already emit canonical rows; fem2d is
 * bucketed by row in emission order (stable), then each short row is stably ordered by
 * column and its duplicates summed in emission order.  Used for full-size (>= 20M DOF)
 * configs.  With row_ptr==NULL only *n and *ntrip (an upper bound on nnz) are written;
 * otherwise col_idx/vals must hold *ntrip entries and *nnz receives the canonical count. */
int orc_gen_csr(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t* n, int64_t* ntrip,
                int64_t* row_ptr, int64_t* col_idx, double* vals, int64_t* nnz);
/* node coordinates (x,y) for 2-D kinds (0: grid, 3: fem interior nodes) */
int orc_gen_coords(int32_t kind, int64_t p1, int64_t p2, double* xs, double* ys);

/* ---- partitioning ---- returns 0 or 6 */
int orc_partition_contiguous(int64_t n, int32_t nparts, int32_t* part_of);
int orc_partition_rcb(int64_t n, const double* xs, const double* ys, int32_t nparts,
                      int32_t* part_of);

/* ---- build_local ---- */
typedef struct orc_local orc_local;
orc_local* orc_local_build(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           const double* vals, const int32_t* part_of, int32_t nparts,
                           int32_t rank);
/* sizes[0]=n_owned [1]=n_halo [2]=n_neighbors [3]=nnz_local [4]=total_send [5]=total_recv */
void orc_local_sizes(const orc_local* L, int64_t* sizes);
void orc_local_get(const orc_local* L, int64_t* owned, int64_t* halo, int32_t* neighbors,
                   int64_t* send_ptr, int64_t* send_idx, int64_t* recv_ptr, int64_t* recv_idx,
                   int64_t* l_row_ptr, int64_t* l_col_idx, double* l_vals);
void orc_local_free(orc_local* L);

/* ---- distributed solve with in-process workers ----
 * kind 0 cg, 1 bicgstab. x_global gathered on "rank 0" (gather_solution).
 * counters[0] = halo exchanges (per rank), counters[1] = all_reduce calls (per rank),
 * counters[2] = point-to-point messages (total)  */
int orc_dist_solve(int32_t kind, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                   const double* vals, const double* b, const int32_t* part_of, int32_t nparts,
                   const orc_opts* opts, double* x_global, orc_report* rep, int64_t* counters);
/* distributed spmv (halo exchange + local spmv), gathered */
int orc_dist_spmv(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                  const double* x, const int32_t* part_of, int32_t nparts, double* y);
/* dist_adjoint_solve: structurally symmetric A only (returns 5 otherwise) */
int orc_dist_adjoint(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                     const double* vals, const double* x, const double* g,
                     const int32_t* part_of, int32_t nparts, const orc_opts* opts,
                     double* grad_b, double* grad_vals, orc_report* rep);

#ifdef __cplusplus
}
#endif
#endif
