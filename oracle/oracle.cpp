// oracle.cpp — CPU ORACLE (test infrastructure, NOT the product).
//
// A plain C++ restatement of the reference's sparse Krylov path, used only as the
// parity checker for the CUDA implementation in paper_2601_13994_b200/.
// See oracle.h for the file:line map.  Build: oracle/Makefile (g++ -O3, no -march,
// -ffp-contract=off: the reference's Release flags proj/CMakeLists.txt:8-10 give
// separate mulsd/addsd, so no fused multiply-add may appear here either).
//
// Parity pin: orc_spmv / orc_coo_canonicalize / orc_csr_transpose are checked bit-for-bit
// against the reference's own compiled sparse.cpp (oracle/_ref) and against the committed
// fixtures in tests/golden/ (tests/test_oracle.py).  The solver/distributed/adjoint parts
// have no executable reference; they are pinned by the SPEC.md examples.
#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numeric>
#include <thread>
#include <vector>

namespace {

int g_threads = 1;

// Row/chunk-parallel loop.  Every parallel region below partitions work so that each
// output element is produced by exactly one thread with a fixed operation order, so
// results are bitwise independent of the thread count.
template <class F>
void parallel_for(int64_t n, F&& f, int64_t min_per_thread = 1 << 15) {
    int nt = g_threads;
    if (nt <= 1 || n < 2 * min_per_thread) {
        f(int64_t{0}, n);
        return;
    }
    int64_t want = (n + min_per_thread - 1) / min_per_thread;
    if (want < nt) nt = static_cast<int>(want);
    std::vector<std::thread> th;
    th.reserve(nt);
    int64_t per = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        int64_t b = t * per, e = std::min(n, b + per);
        if (b >= e) break;
        th.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& t : th) t.join();
}

// ---------------------------------------------------------------------------------
// Canonical dot.  The reference leaves the dot summation order open
// (SPEC.md:488-496 only fixes the cross-rank order).  Both the oracle and the CUDA path
// use this fixed shape so that Krylov trajectories are bitwise identical:
//   level 1: chunks of 2048 consecutive products; product j of chunk c goes to slot
//            s = j % 256, round r = j / 256; slot sum = ((0 + p_r0) + p_r1) + ... (r asc);
//            chunk partial = pairwise binary tree over the 256 slots.
//   level 2: m chunk partials; slot s (of 1024) sums partials s, s+1024, ... from 0.0 in
//            ascending order; result = pairwise binary tree over the 1024 slots.
// Products are a_j * b_j rounded to double (no FMA).
// ---------------------------------------------------------------------------------
constexpr int kChunkSlots = 256;
constexpr int kChunkRounds = 8;
constexpr int64_t kChunk = kChunkSlots * kChunkRounds;  // 2048
constexpr int kFinalSlots = 1024;

double tree_reduce(double* s, int len) {
    for (int w = 1; w < len; w *= 2)
        for (int i = 0; i + w < len; i += 2 * w) s[i] = s[i] + s[i + w];
    return s[0];
}

double chunk_partial(const double* a, const double* b, int64_t len) {
    double slot[kChunkSlots];
    for (int s = 0; s < kChunkSlots; ++s) {
        double acc = 0.0;
        for (int r = 0; r < kChunkRounds; ++r) {
            int64_t j = int64_t{r} * kChunkSlots + s;
            if (j < len) acc = acc + a[j] * b[j];
        }
        slot[s] = acc;
    }
    return tree_reduce(slot, kChunkSlots);
}

double final_reduce(const double* part, int64_t m) {
    double slot[kFinalSlots];
    for (int s = 0; s < kFinalSlots; ++s) {
        double acc = 0.0;
        for (int64_t c = s; c < m; c += kFinalSlots) acc = acc + part[c];
        slot[s] = acc;
    }
    return tree_reduce(slot, kFinalSlots);
}

void cdot_partials(int64_t n, const double* a, const double* b, double* part) {
    int64_t m = (n + kChunk - 1) / kChunk;
    parallel_for(m, [&](int64_t c0, int64_t c1) {
        for (int64_t c = c0; c < c1; ++c) {
            int64_t base = c * kChunk;
            part[c] = chunk_partial(a + base, b + base, std::min(kChunk, n - base));
        }
    }, 16);
}

double cdot(int64_t n, const double* a, const double* b) {
    if (n <= 0) return 0.0;
    int64_t m = (n + kChunk - 1) / kChunk;
    std::vector<double> part(static_cast<size_t>(m));
    cdot_partials(n, a, b, part.data());
    return final_reduce(part.data(), m);
}

// y = A x, row-ordered, sum from 0.0 left to right: restates sparse.cpp:135-154.
template <class IdxT>
void spmv_rows(int64_t r0, int64_t r1, const int64_t* rp, const IdxT* ci, const double* v,
               const double* x, double* y) {
    for (int64_t i = r0; i < r1; ++i) {
        double sum = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) sum += v[k] * x[ci[k]];
        y[i] = sum;
    }
}

void spmv(int64_t nrows, const int64_t* rp, const int64_t* ci, const double* v, const double* x,
          double* y) {
    parallel_for(nrows, [&](int64_t a, int64_t b) { spmv_rows(a, b, rp, ci, v, x, y); });
}

// Jacobi inverse diagonal.  Degenerate threshold (SPEC leaves
// it open): an entry falls back to 1.0 when A_ii is missing, exactly zero, or its
// reciprocal is not finite.
void jacobi(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, double* d) {
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            double aii = 0.0;
            bool found = false;
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
                if (ci[k] == i) { aii = v[k]; found = true; break; }
            double r = 1.0;
            if (found && aii != 0.0) {
                double t = 1.0 / aii;
                if (std::isfinite(t)) r = t;
            }
            d[i] = r;
        }
    });
}

void set_diag(orc_report* rep, const char* msg) {
    std::snprintf(rep->diagnostic, sizeof(rep->diagnostic), "%s", msg);
}

// ---------------------------------------------------------------------------------
// Krylov cores, written once over an abstract "space": serial (local == global) or one
// rank of the in-process distributed run.  Space must provide:
//   int64_t n;  void spmv(const double* x_owned, double* y_owned);
//   double dot(a, b) (global);  void dot2/dot3 (fused reduction points, one all_reduce)
// ---------------------------------------------------------------------------------
struct SerialSpace {
    int64_t n;
    const int64_t* rp;
    const int64_t* ci;
    const double* v;
    void spmv(const double* x, double* y) { ::spmv(n, rp, ci, v, x, y); }
    double dot(const double* a, const double* b) { return cdot(n, a, b); }
    void dots(int k, const double* const* a, const double* const* b, double* out) {
        for (int i = 0; i < k; ++i) out[i] = cdot(n, a[i], b[i]);
    }
};

bool validate_opts(const orc_opts* o) {
    if (!(o->atol >= 0.0) || !(o->rtol >= 0.0)) return false;
    if (o->atol == 0.0 && o->rtol == 0.0) return false;
    if (o->max_iter < 1) return false;
    return true;
}

// Jacobi-PCG, x0 = 0 (PAPER.md:295-308 with local reductions).
template <class Space>
void cg_core(Space& S, const double* b, double* x, const double* dinv, const orc_opts* o,
             orc_report* rep, int64_t fixed_iters = -1, double* r_out = nullptr) {
    const int64_t n = S.n;
    std::vector<double> r(n), z(n), p(n), q(n);
    std::memset(rep, 0, sizeof(*rep));
    rep->backend = 0;
    parallel_for(n, [&](int64_t a, int64_t e) { for (int64_t i = a; i < e; ++i) x[i] = 0.0; });
    S.spmv(x, q.data());
    int64_t spmv_count = 1;
    parallel_for(n, [&](int64_t a, int64_t e) {
        for (int64_t i = a; i < e; ++i) {
            r[i] = b[i] - q[i];
            z[i] = dinv[i] * r[i];
            p[i] = z[i];
        }
    });
    double rz, rr, bb;
    {
        const double* A[3] = {r.data(), r.data(), b};
        const double* B[3] = {z.data(), r.data(), b};
        double out[3];
        S.dots(3, A, B, out);  // init reduction point: {rz, rr, bb}
        rz = out[0]; rr = out[1]; bb = out[2];
    }
    const double bnorm = std::sqrt(bb);
    const double tol = std::max(o->atol, o->rtol * bnorm);
    double rnorm = std::sqrt(rr);
    bool converged = fixed_iters < 0 && rnorm <= tol;
    int64_t k = 0;
    const int64_t kmax = fixed_iters >= 0 ? fixed_iters : o->max_iter;
    set_diag(rep, "");
    while (!converged && k < kmax) {
        S.spmv(p.data(), q.data());
        ++spmv_count;
        const double pq = S.dot(p.data(), q.data());
        if (!(pq > 0.0)) {  // p^T A p <= 0 (or NaN): breakdown, reported not thrown
            char buf[128];
            std::snprintf(buf, sizeof(buf), "breakdown: p^T A p <= 0 at iteration %lld",
                          (long long)k);
            set_diag(rep, buf);
            break;
        }
        const double alpha = rz / pq;
        parallel_for(n, [&](int64_t a, int64_t e) {
            for (int64_t i = a; i < e; ++i) {
                x[i] = x[i] + alpha * p[i];
                r[i] = r[i] - alpha * q[i];
                z[i] = dinv[i] * r[i];
            }
        });
        double rz_new;
        {
            const double* A[2] = {r.data(), r.data()};
            const double* B[2] = {z.data(), r.data()};
            double out[2];
            S.dots(2, A, B, out);
            rz_new = out[0]; rr = out[1];
        }
        ++k;
        rnorm = std::sqrt(rr);
        if (fixed_iters < 0 && rnorm <= tol) { converged = true; break; }
        if (k >= kmax) break;
        const double beta = rz_new / rz;
        rz = rz_new;
        parallel_for(n, [&](int64_t a, int64_t e) {
            for (int64_t i = a; i < e; ++i) p[i] = z[i] + beta * p[i];
        });
    }
    if (!converged && rep->diagnostic[0] == 0 && fixed_iters < 0)
        set_diag(rep, "max_iter reached");
    rep->iterations = k;
    rep->spmv_count = spmv_count;
    rep->residual_norm = rnorm;
    rep->converged = converged ? 1 : 0;
    if (r_out) std::memcpy(r_out, r.data(), sizeof(double) * n);
}

// BiCGStab with right Jacobi preconditioning, x0 = 0.  The half-step
// test on ||s|| uses s.s computed at the same reduction point as t.t and t.s.
template <class Space>
void bicgstab_core(Space& S, const double* b, double* x, const double* dinv,
                   const orc_opts* o, orc_report* rep) {
    const int64_t n = S.n;
    std::vector<double> r(n), rh(n), p(n), ph(n), v(n), s(n), sh(n), t(n);
    std::memset(rep, 0, sizeof(*rep));
    rep->backend = 1;
    parallel_for(n, [&](int64_t a, int64_t e) { for (int64_t i = a; i < e; ++i) x[i] = 0.0; });
    S.spmv(x, v.data());
    int64_t spmv_count = 1;
    parallel_for(n, [&](int64_t a, int64_t e) {
        for (int64_t i = a; i < e; ++i) {
            r[i] = b[i] - v[i];
            rh[i] = r[i];
        }
    });
    double rho, rr, bb;
    {
        const double* A[3] = {rh.data(), r.data(), b};
        const double* B[3] = {r.data(), r.data(), b};
        double out[3];
        S.dots(3, A, B, out);
        rho = out[0]; rr = out[1]; bb = out[2];
    }
    const double bnorm = std::sqrt(bb);
    const double tol = std::max(o->atol, o->rtol * bnorm);
    const double rho_thr = 1e-30 * (bnorm * bnorm);
    double rnorm = std::sqrt(rr);
    bool converged = rnorm <= tol;
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    int64_t k = 0;
    set_diag(rep, "");
    char buf[128];
    while (!converged && k < o->max_iter) {
        if (!(std::fabs(rho) >= rho_thr) || !std::isfinite(rho)) {
            std::snprintf(buf, sizeof(buf), "breakdown: |rho| < 1e-30*||b||^2 at iteration %lld",
                          (long long)k);
            set_diag(rep, buf);
            break;
        }
        if (k == 0) {
            parallel_for(n, [&](int64_t a, int64_t e) {
                for (int64_t i = a; i < e; ++i) { p[i] = r[i]; ph[i] = dinv[i] * p[i]; }
            });
        } else {
            const double beta = (rho / rho_prev) * (alpha / omega);
            parallel_for(n, [&](int64_t a, int64_t e) {
                for (int64_t i = a; i < e; ++i) {
                    p[i] = r[i] + beta * (p[i] - omega * v[i]);
                    ph[i] = dinv[i] * p[i];
                }
            });
        }
        S.spmv(ph.data(), v.data());
        ++spmv_count;
        const double rv = S.dot(rh.data(), v.data());
        if (!(rv != 0.0) || !std::isfinite(rv)) {
            std::snprintf(buf, sizeof(buf), "breakdown: rhat^T v = 0 at iteration %lld",
                          (long long)k);
            set_diag(rep, buf);
            break;
        }
        alpha = rho / rv;
        parallel_for(n, [&](int64_t a, int64_t e) {
            for (int64_t i = a; i < e; ++i) {
                s[i] = r[i] - alpha * v[i];
                sh[i] = dinv[i] * s[i];
            }
        });
        S.spmv(sh.data(), t.data());
        ++spmv_count;
        double tt, ts, ss;
        {
            const double* A[3] = {t.data(), t.data(), s.data()};
            const double* B[3] = {t.data(), s.data(), s.data()};
            double out[3];
            S.dots(3, A, B, out);
            tt = out[0]; ts = out[1]; ss = out[2];
        }
        if (std::sqrt(ss) <= tol) {  // half-step convergence: x += alpha*phat, r = s
            parallel_for(n, [&](int64_t a, int64_t e) {
                for (int64_t i = a; i < e; ++i) { x[i] = x[i] + alpha * ph[i]; r[i] = s[i]; }
            });
            rnorm = std::sqrt(ss);
            ++k;
            converged = true;
            break;
        }
        if (!(tt > 0.0)) {
            std::snprintf(buf, sizeof(buf), "breakdown: t^T t = 0 at iteration %lld", (long long)k);
            set_diag(rep, buf);
            break;
        }
        omega = ts / tt;
        parallel_for(n, [&](int64_t a, int64_t e) {
            for (int64_t i = a; i < e; ++i) {
                x[i] = (x[i] + alpha * ph[i]) + omega * sh[i];
                r[i] = s[i] - omega * t[i];
            }
        });
        rho_prev = rho;
        {
            const double* A[2] = {rh.data(), r.data()};
            const double* B[2] = {r.data(), r.data()};
            double out[2];
            S.dots(2, A, B, out);
            rho = out[0]; rr = out[1];
        }
        ++k;
        rnorm = std::sqrt(rr);
        if (rnorm <= tol) { converged = true; break; }
        if (omega == 0.0) {
            std::snprintf(buf, sizeof(buf), "breakdown: omega = 0 at iteration %lld", (long long)k);
            set_diag(rep, buf);
            break;
        }
    }
    if (!converged && rep->diagnostic[0] == 0) set_diag(rep, "max_iter reached");
    rep->iterations = k;
    rep->spmv_count = spmv_count;
    rep->residual_norm = rnorm;
    rep->converged = converged ? 1 : 0;
}

// ---------------------------------------------------------------------------------
// Generators (3-D / CD / FEM per SURVEY.md §8(d)).  Emission order is
// the natural stencil / element order; canonicalization happens in orc_coo_canonicalize.
// ---------------------------------------------------------------------------------
uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
double uniform01(uint64_t seed, uint64_t id, uint64_t comp) {
    uint64_t u = splitmix64(splitmix64(seed) ^ (2 * id + comp));
    return static_cast<double>(u >> 11) * 0x1.0p-53;
}

struct FemMesh {
    int64_t m;
    uint64_t seed;
    double h;
    FemMesh(int64_t m_, uint64_t s) : m(m_), seed(s), h(1.0 / static_cast<double>(m_ - 1)) {}
    bool interior(int64_t i, int64_t j) const { return i >= 1 && i <= m - 2 && j >= 1 && j <= m - 2; }
    int64_t dof(int64_t i, int64_t j) const { return (j - 1) * (m - 2) + (i - 1); }
    void coord(int64_t i, int64_t j, double& x, double& y) const {
        x = static_cast<double>(i) * h;
        y = static_cast<double>(j) * h;
        if (interior(i, j)) {
            uint64_t id = static_cast<uint64_t>(j * m + i);
            x = x + ((uniform01(seed, id, 0) - 0.5) * 0.5) * h;
            y = y + ((uniform01(seed, id, 1) - 0.5) * 0.5) * h;
        }
    }
    // Cell (ci,cj): corners a=(ci,cj) b=(ci+1,cj) c=(ci+1,cj+1) d=(ci,cj+1), ccw.
    // Delaunay choice by the in-circle determinant; returns the two ccw triangles.
    void cell_tris(int64_t ci, int64_t cj, int64_t tri[2][3][2]) const {
        double ax, ay, bx, by, cx, cy, dx, dy;
        coord(ci, cj, ax, ay);
        coord(ci + 1, cj, bx, by);
        coord(ci + 1, cj + 1, cx, cy);
        coord(ci, cj + 1, dx, dy);
        double adx = ax - dx, ady = ay - dy, bdx = bx - dx, bdy = by - dy, cdx = cx - dx, cdy = cy - dy;
        double alift = adx * adx + ady * ady;
        double blift = bdx * bdx + bdy * bdy;
        double clift = cdx * cdx + cdy * cdy;
        double t1 = alift * (bdx * cdy - cdx * bdy);
        double t2 = blift * (cdx * ady - adx * cdy);
        double t3 = clift * (adx * bdy - bdx * ady);
        double det = (t1 + t2) + t3;
        int64_t A[2] = {ci, cj}, B[2] = {ci + 1, cj}, C[2] = {ci + 1, cj + 1}, D[2] = {ci, cj + 1};
        const int64_t* T[2][3];
        if (det > 0.0) {  // d inside circumcircle(a,b,c): use diagonal b-d
            T[0][0] = A; T[0][1] = B; T[0][2] = D;
            T[1][0] = B; T[1][1] = C; T[1][2] = D;
        } else {          // diagonal a-c
            T[0][0] = A; T[0][1] = B; T[0][2] = C;
            T[1][0] = A; T[1][1] = C; T[1][2] = D;
        }
        for (int t = 0; t < 2; ++t)
            for (int v = 0; v < 3; ++v) { tri[t][v][0] = T[t][v][0]; tri[t][v][1] = T[t][v][1]; }
    }
    // P1 stiffness K[k][l] = (b_k b_l + c_k c_l) / (2 * area2)
    void stiffness(const int64_t tri[3][2], double K[3][3]) const {
        double x[3], y[3];
        for (int v = 0; v < 3; ++v) coord(tri[v][0], tri[v][1], x[v], y[v]);
        double bb[3] = {y[1] - y[2], y[2] - y[0], y[0] - y[1]};
        double cc[3] = {x[2] - x[1], x[0] - x[2], x[1] - x[0]};
        double area2 = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
        double den = 2.0 * area2;
        for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l) K[k][l] = (bb[k] * bb[l] + cc[k] * cc[l]) / den;
    }
};

// ---------------------------------------------------------------------------------
// build_local + in-process transport
// ---------------------------------------------------------------------------------
struct Local {
    int32_t rank = 0;
    std::vector<int64_t> owned, halo;
    std::vector<int32_t> neighbors;
    std::vector<int64_t> send_ptr, send_idx, recv_ptr, recv_idx;  // local positions
    std::vector<int64_t> rp, ci;  // local CSR, entries in global column order
    std::vector<double> v;
};

Local build_local(int64_t n, const int64_t* rp, const int64_t* ci, const double* vals,
                  const int32_t* part_of, int32_t nparts, int32_t rank) {
    Local L;
    L.rank = rank;
    for (int64_t i = 0; i < n; ++i)
        if (part_of[i] == rank) L.owned.push_back(i);
    std::vector<char> is_halo(n, 0);
    // halo: h not owned with an edge (i,h) or (h,i), i owned
    for (int64_t i : L.owned)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (part_of[ci[k]] != rank) is_halo[ci[k]] = 1;
    for (int64_t h = 0; h < n; ++h) {
        if (part_of[h] == rank) continue;
        for (int64_t k = rp[h]; k < rp[h + 1]; ++k)
            if (part_of[ci[k]] == rank) { is_halo[h] = 1; break; }
    }
    for (int64_t h = 0; h < n; ++h)
        if (is_halo[h]) L.halo.push_back(h);
    const int64_t no = static_cast<int64_t>(L.owned.size());
    std::vector<int64_t> g2l(n, -1);
    for (int64_t a = 0; a < no; ++a) g2l[L.owned[a]] = a;
    for (size_t a = 0; a < L.halo.size(); ++a) g2l[L.halo[a]] = no + static_cast<int64_t>(a);
    // neighbors = owners of halo nodes (symmetric by construction of the halo rule)
    std::vector<char> nb(nparts, 0);
    for (int64_t h : L.halo) nb[part_of[h]] = 1;
    for (int32_t q = 0; q < nparts; ++q)
        if (nb[q]) L.neighbors.push_back(q);
    // recv from q: my halo slots owned by q, ascending global
    L.recv_ptr.push_back(0);
    for (int32_t q : L.neighbors) {
        for (int64_t h : L.halo)
            if (part_of[h] == q) L.recv_idx.push_back(g2l[h]);
        L.recv_ptr.push_back(static_cast<int64_t>(L.recv_idx.size()));
    }
    // send to q: my owned nodes in q's halo, ascending global.  i is in H_q iff an edge
    // (j,i) or (i,j) exists with j owned by q.
    L.send_ptr.push_back(0);
    std::vector<char> need(static_cast<size_t>(no), 0);
    for (int32_t q : L.neighbors) {
        std::fill(need.begin(), need.end(), 0);
        for (int64_t a = 0; a < no; ++a) {  // edges (i,j), j owned by q
            const int64_t i = L.owned[a];
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
                if (part_of[ci[k]] == q) { need[a] = 1; break; }
        }
        for (int64_t h : L.halo) {  // edges (j,i), j owned by q (j is necessarily my halo)
            if (part_of[h] != q) continue;
            for (int64_t k = rp[h]; k < rp[h + 1]; ++k)
                if (part_of[ci[k]] == rank) need[g2l[ci[k]]] = 1;
        }
        for (int64_t a = 0; a < no; ++a)
            if (need[a]) L.send_idx.push_back(a);
        L.send_ptr.push_back(static_cast<int64_t>(L.send_idx.size()));
    }
    L.rp.push_back(0);
    for (int64_t i : L.owned) {
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            L.ci.push_back(g2l[ci[k]]);
            L.v.push_back(vals[k]);
        }
        L.rp.push_back(static_cast<int64_t>(L.ci.size()));
    }
    return L;
}

// In-process transport: per-(src,dst) mailboxes + barrier collectives.  all_reduce sums in
// ascending rank order starting from rank 0's value.
struct Transport {
    int32_t P;
    std::barrier<> bar;
    std::vector<std::vector<double>> mailbox;  // [src*P + dst]
    std::vector<double> red;                   // [rank*8 + j]
    std::atomic<int64_t> messages{0};
    explicit Transport(int32_t p) : P(p), bar(p), mailbox(size_t(p) * p), red(size_t(p) * 8) {}
};

struct DistSpace {
    Local* L;
    Transport* T;
    int64_t n;  // owned
    std::vector<double> xl;  // [owned | halo]
    int64_t halo_exchanges = 0, allreduces = 0;
    void exchange() {
        const int32_t me = L->rank;
        for (size_t a = 0; a < L->neighbors.size(); ++a) {
            int32_t q = L->neighbors[a];
            auto& box = T->mailbox[size_t(me) * T->P + q];
            box.clear();
            for (int64_t k = L->send_ptr[a]; k < L->send_ptr[a + 1]; ++k)
                box.push_back(xl[L->send_idx[k]]);
            T->messages.fetch_add(1);
        }
        T->bar.arrive_and_wait();
        for (size_t a = 0; a < L->neighbors.size(); ++a) {
            int32_t q = L->neighbors[a];
            auto& box = T->mailbox[size_t(q) * T->P + me];
            int64_t cnt = L->recv_ptr[a + 1] - L->recv_ptr[a];
            if (static_cast<int64_t>(box.size()) != cnt) std::abort();  // payload mismatch
            for (int64_t k = 0; k < cnt; ++k) xl[L->recv_idx[L->recv_ptr[a] + k]] = box[k];
        }
        T->bar.arrive_and_wait();
        ++halo_exchanges;
    }
    void spmv(const double* x, double* y) {
        std::memcpy(xl.data(), x, sizeof(double) * n);
        exchange();
        for (int64_t i = 0; i < n; ++i) {
            double sum = 0.0;
            for (int64_t k = L->rp[i]; k < L->rp[i + 1]; ++k) sum += L->v[k] * xl[L->ci[k]];
            y[i] = sum;
        }
    }
    void allreduce(int k, const double* loc, double* out) {
        const int32_t me = L->rank;
        for (int j = 0; j < k; ++j) T->red[size_t(me) * 8 + j] = loc[j];
        T->bar.arrive_and_wait();
        for (int j = 0; j < k; ++j) {
            double s = T->red[j];
            for (int32_t q = 1; q < T->P; ++q) s = s + T->red[size_t(q) * 8 + j];
            out[j] = s;
        }
        T->bar.arrive_and_wait();
        ++allreduces;
    }
    double dot(const double* a, const double* b) {
        double l = cdot(n, a, b), g;
        allreduce(1, &l, &g);
        return g;
    }
    void dots(int k, const double* const* a, const double* const* b, double* out) {
        double l[8];
        for (int i = 0; i < k; ++i) l[i] = cdot(n, a[i], b[i]);
        allreduce(k, l, out);
    }
};

}  // namespace

// =================================================================================
extern "C" {

void orc_set_threads(int nthreads) { g_threads = nthreads < 1 ? 1 : nthreads; }
int orc_get_threads(void) { return g_threads; }

double orc_cdot(int64_t n, const double* a, const double* b) { return cdot(n, a, b); }
void orc_cdot_partials(int64_t n, const double* a, const double* b, double* partials) {
    cdot_partials(n, a, b, partials);
}

// Restates SparseCoo::SparseCoo (sparse.cpp:9-53): bounds check, stable sort by (row,col),
// duplicates summed in input order, explicit zeros kept.
int64_t orc_coo_canonicalize(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                             const int64_t* cols, const double* vals, int64_t* ro, int64_t* co,
                             double* vo) {
    if (nrows < 0 || ncols < 0) return -1;
    for (int64_t k = 0; k < nnz; ++k)
        if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols) return -2;
    std::vector<int64_t> perm(nnz);
    std::iota(perm.begin(), perm.end(), int64_t{0});
    std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) {
        if (rows[a] != rows[b]) return rows[a] < rows[b];
        return cols[a] < cols[b];
    });
    int64_t out = 0;
    for (int64_t k = 0; k < nnz; ++k) {
        int64_t p = perm[k];
        if (out > 0 && ro[out - 1] == rows[p] && co[out - 1] == cols[p]) {
            vo[out - 1] += vals[p];
        } else {
            ro[out] = rows[p]; co[out] = cols[p]; vo[out] = vals[p];
            ++out;
        }
    }
    return out;
}

// Restates CsrMatrix::from_coo (sparse.cpp:94-116).
void orc_csr_from_coo(int64_t nrows, int64_t nnz, const int64_t* rows, const int64_t* cols,
                      const double* vals, int64_t* rp, int64_t* ci, double* v) {
    for (int64_t i = 0; i <= nrows; ++i) rp[i] = 0;
    for (int64_t k = 0; k < nnz; ++k) ++rp[rows[k] + 1];
    for (int64_t i = 0; i < nrows; ++i) rp[i + 1] += rp[i];
    for (int64_t k = 0; k < nnz; ++k) { ci[k] = cols[k]; v[k] = vals[k]; }
}

void orc_spmv(int64_t nrows, const int64_t* rp, const int64_t* ci, const double* v,
              const double* x, double* y) {
    spmv(nrows, rp, ci, v, x, y);
}

// Canonical CSR of A^T (= CsrMatrix::from_coo(transpose(coo)), sparse.cpp:176-182):
// row j of A^T lists i ascending, which is the scatter order of spmv_transpose
// (sparse.cpp:165-172), so row-ordered spmv on A^T equals spmv_transpose bitwise.
void orc_csr_transpose(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                       const double* v, int64_t* trp, int64_t* tci, double* tv) {
    for (int64_t j = 0; j <= ncols; ++j) trp[j] = 0;
    const int64_t nnz = rp[nrows];
    for (int64_t k = 0; k < nnz; ++k) ++trp[ci[k] + 1];
    for (int64_t j = 0; j < ncols; ++j) trp[j + 1] += trp[j];
    std::vector<int64_t> fill(trp, trp + ncols);
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            int64_t pos = fill[ci[k]]++;
            tci[pos] = i;
            tv[pos] = v[k];
        }
}

void orc_jacobi(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, double* d) {
    jacobi(n, rp, ci, v, d);
}

static void precond_vec(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        int32_t pc, std::vector<double>& d) {
    d.assign(static_cast<size_t>(n), 1.0);
    if (pc == 1) jacobi(n, rp, ci, v, d.data());
}

int orc_cg(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b,
           double* x, const orc_opts* o, orc_report* rep) {
    if (!validate_opts(o)) return 6;
    std::vector<double> d;
    precond_vec(n, rp, ci, v, o->preconditioner, d);
    SerialSpace S{n, rp, ci, v};
    cg_core(S, b, x, d.data(), o, rep);
    return 0;
}

int orc_cg_fixed(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                 const double* b, int64_t iters, int32_t pc, double* x, double* r) {
    std::vector<double> d;
    precond_vec(n, rp, ci, v, pc, d);
    SerialSpace S{n, rp, ci, v};
    orc_opts o{1e-300, 0.0, iters < 1 ? 1 : iters, pc, 0};
    orc_report rep;
    cg_core(S, b, x, d.data(), &o, &rep, iters, r);
    return 0;
}

int orc_bicgstab(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                 const double* b, double* x, const orc_opts* o, orc_report* rep) {
    if (!validate_opts(o)) return 6;
    std::vector<double> d;
    precond_vec(n, rp, ci, v, o->preconditioner, d);
    SerialSpace S{n, rp, ci, v};
    bicgstab_core(S, b, x, d.data(), o, rep);
    return 0;
}

// solve_backward (Eq. 3).
int orc_adjoint_backward(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                         const double* x, const double* g, int32_t backend, const orc_opts* o,
                         double* grad_b, double* grad_vals, orc_report* rep) {
    if (!validate_opts(o)) return 6;
    const int64_t nnz = rp[n];
    std::vector<double> lam(static_cast<size_t>(n), 0.0);
    bool all_zero = true;
    for (int64_t i = 0; i < n; ++i)
        if (g[i] != 0.0) { all_zero = false; break; }
    std::memset(rep, 0, sizeof(*rep));
    rep->backend = backend;
    if (all_zero) {  // lambda = 0 short-circuit
        rep->converged = 1;
        set_diag(rep, "grad_x == 0: short-circuit");
    } else {
        std::vector<int64_t> trp(n + 1), tci(nnz);
        std::vector<double> tv(nnz);
        orc_csr_transpose(n, n, rp, ci, v, trp.data(), tci.data(), tv.data());
        int rc = backend == 1 ? orc_bicgstab(n, trp.data(), tci.data(), tv.data(), g, lam.data(), o, rep)
                              : orc_cg(n, trp.data(), tci.data(), tv.data(), g, lam.data(), o, rep);
        if (rc) return rc;
    }
    for (int64_t i = 0; i < n; ++i) grad_b[i] = lam[i];
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) grad_vals[k] = -(lam[i] * x[ci[k]]);
    return 0;
}

int orc_gen_triplets(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t* n_out,
                     int64_t* ntrip, int64_t* rows, int64_t* cols, double* vals) {
    int64_t cnt = 0;
    auto emit = [&](int64_t r, int64_t c, double val) {
        if (rows) { rows[cnt] = r; cols[cnt] = c; vals[cnt] = val; }
        ++cnt;
    };
    if (kind == 0) {  // poisson2d(N): k = i*N + j, diag 4, -1
        const int64_t N = p1;
        if (N < 2) return 6;
        *n_out = N * N;
        for (int64_t i = 0; i < N; ++i)
            for (int64_t j = 0; j < N; ++j) {
                int64_t k = i * N + j;
                if (i > 0) emit(k, k - N, -1.0);
                if (j > 0) emit(k, k - 1, -1.0);
                emit(k, k, 4.0);
                if (j < N - 1) emit(k, k + 1, -1.0);
                if (i < N - 1) emit(k, k + N, -1.0);
            }
    } else if (kind == 1 || kind == 2) {  // 3-D 7-pt, k = (z*N + y)*N + x
        const int64_t N = p1;
        if (N < 2) return 6;
        const double c = kind == 2 ? fparam : 0.0;
        const double diag = kind == 2 ? 6.0 + 3.0 * c : 6.0;
        const double lo = kind == 2 ? -1.0 - c : -1.0;
        *n_out = N * N * N;
        for (int64_t z = 0; z < N; ++z)
            for (int64_t y = 0; y < N; ++y)
                for (int64_t x = 0; x < N; ++x) {
                    int64_t k = (z * N + y) * N + x;
                    if (z > 0) emit(k, k - N * N, lo);
                    if (y > 0) emit(k, k - N, lo);
                    if (x > 0) emit(k, k - 1, lo);
                    emit(k, k, diag);
                    if (x < N - 1) emit(k, k + 1, -1.0);
                    if (y < N - 1) emit(k, k + N, -1.0);
                    if (z < N - 1) emit(k, k + N * N, -1.0);
                }
    } else if (kind == 4) {  // 3-D 7-pt Poisson box N x N x Nz (config E weak-scaling slabs)
        const int64_t N = p1, Nz = p2;
        if (N < 2 || Nz < 2) return 6;
        *n_out = N * N * Nz;
        for (int64_t z = 0; z < Nz; ++z)
            for (int64_t y = 0; y < N; ++y)
                for (int64_t x = 0; x < N; ++x) {
                    int64_t k = (z * N + y) * N + x;
                    if (z > 0) emit(k, k - N * N, -1.0);
                    if (y > 0) emit(k, k - N, -1.0);
                    if (x > 0) emit(k, k - 1, -1.0);
                    emit(k, k, 6.0);
                    if (x < N - 1) emit(k, k + 1, -1.0);
                    if (y < N - 1) emit(k, k + N, -1.0);
                    if (z < Nz - 1) emit(k, k + N * N, -1.0);
                }
    } else if (kind == 3) {  // P1 FEM on jittered lattice, element order
        const int64_t m = p1;
        if (m < 3) return 6;
        FemMesh M(m, static_cast<uint64_t>(p2));
        *n_out = (m - 2) * (m - 2);
        for (int64_t cj = 0; cj < m - 1; ++cj)
            for (int64_t cix = 0; cix < m - 1; ++cix) {
                int64_t tri[2][3][2];
                M.cell_tris(cix, cj, tri);
                for (int t = 0; t < 2; ++t) {
                    double K[3][3];
                    bool any = false;
                    for (int a = 0; a < 3; ++a) any |= M.interior(tri[t][a][0], tri[t][a][1]);
                    if (!any) continue;
                    M.stiffness(tri[t], K);
                    for (int a = 0; a < 3; ++a) {
                        if (!M.interior(tri[t][a][0], tri[t][a][1])) continue;
                        for (int b = 0; b < 3; ++b) {
                            if (!M.interior(tri[t][b][0], tri[t][b][1])) continue;
                            emit(M.dof(tri[t][a][0], tri[t][a][1]), M.dof(tri[t][b][0], tri[t][b][1]),
                                 K[a][b]);
                        }
                    }
                }
            }
    } else {
        return 6;
    }
    *ntrip = cnt;
    return 0;
}

int orc_gen_csr(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t* n_out,
                int64_t* ntrip, int64_t* row_ptr, int64_t* col_idx, double* vals, int64_t* nnz) {
    int rc = orc_gen_triplets(kind, p1, p2, fparam, n_out, ntrip, nullptr, nullptr, nullptr);
    if (rc || !row_ptr) return rc;
    const int64_t n = *n_out, nt = *ntrip;
    if (kind != 3) {
        // stencil emission is already canonical: rows ascending, columns ascending within a
        // row, no duplicates (checked below) -- fill CSR in emission order
        std::fill(row_ptr, row_ptr + n + 1, int64_t{0});
        int64_t cnt = 0, last_r = -1, last_c = -1;
        bool ok = true;
        auto emit = [&](int64_t r, int64_t c, double v) {
            if (r < last_r || (r == last_r && c <= last_c)) ok = false;
            last_r = r; last_c = c;
            ++row_ptr[r + 1];
            col_idx[cnt] = c;
            vals[cnt] = v;
            ++cnt;
        };
        // the stencil loops of orc_gen_triplets, emitting into CSR (order asserted above)
        if (kind == 0) {
            const int64_t N = p1;
            for (int64_t i = 0; i < N; ++i)
                for (int64_t j = 0; j < N; ++j) {
                    int64_t k = i * N + j;
                    if (i > 0) emit(k, k - N, -1.0);
                    if (j > 0) emit(k, k - 1, -1.0);
                    emit(k, k, 4.0);
                    if (j < N - 1) emit(k, k + 1, -1.0);
                    if (i < N - 1) emit(k, k + N, -1.0);
                }
        } else {
            const int64_t N = p1, Nz = kind == 4 ? p2 : p1;
            const double c = kind == 2 ? fparam : 0.0;
            const double diag = kind == 2 ? 6.0 + 3.0 * c : 6.0;
            const double lo = kind == 2 ? -1.0 - c : -1.0;
            for (int64_t z = 0; z < Nz; ++z)
                for (int64_t y = 0; y < N; ++y)
                    for (int64_t x = 0; x < N; ++x) {
                        int64_t k = (z * N + y) * N + x;
                        if (z > 0) emit(k, k - N * N, lo);
                        if (y > 0) emit(k, k - N, lo);
                        if (x > 0) emit(k, k - 1, lo);
                        emit(k, k, diag);
                        if (x < N - 1) emit(k, k + 1, -1.0);
                        if (y < N - 1) emit(k, k + N, -1.0);
                        if (z < Nz - 1) emit(k, k + N * N, -1.0);
                    }
        }
        if (!ok || cnt != nt) return 7;
        for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
        *nnz = cnt;
        return 0;
    }
    // fem2d: stable bucket by row (emission order kept inside a row), then per row a stable
    // insertion sort by column and an in-order duplicate sum (== SparseCoo semantics)
    std::vector<int64_t> tr(static_cast<size_t>(nt)), tc(static_cast<size_t>(nt));
    std::vector<double> tv(static_cast<size_t>(nt));
    int64_t dummy_n, dummy_t;
    orc_gen_triplets(kind, p1, p2, fparam, &dummy_n, &dummy_t, tr.data(), tc.data(), tv.data());
    std::vector<int64_t> start(static_cast<size_t>(n) + 1, 0);
    for (int64_t k = 0; k < nt; ++k) ++start[tr[k] + 1];
    for (int64_t i = 0; i < n; ++i) start[i + 1] += start[i];
    {
        std::vector<int64_t> pos(start.begin(), start.end() - 1);
        for (int64_t k = 0; k < nt; ++k) {
            int64_t p = pos[tr[k]]++;
            col_idx[p] = tc[k];
            vals[p] = tv[k];
        }
    }
    std::vector<int64_t>().swap(tr);
    std::vector<int64_t>().swap(tc);
    std::vector<double>().swap(tv);
    int64_t out = 0;
    row_ptr[0] = 0;
    std::vector<std::pair<int64_t, double>> row;
    for (int64_t i = 0; i < n; ++i) {
        row.clear();
        for (int64_t p = start[i]; p < start[i + 1]; ++p) row.emplace_back(col_idx[p], vals[p]);
        std::stable_sort(row.begin(), row.end(),
                         [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t q = 0; q < row.size(); ++q) {
            if (out > row_ptr[i] && col_idx[out - 1] == row[q].first) {
                vals[out - 1] += row[q].second;
            } else {
                col_idx[out] = row[q].first;
                vals[out] = row[q].second;
                ++out;
            }
        }
        row_ptr[i + 1] = out;
    }
    *nnz = out;
    return 0;
}

int orc_gen_coords(int32_t kind, int64_t p1, int64_t p2, double* xs, double* ys) {
    if (kind == 0) {
        const int64_t N = p1;
        for (int64_t i = 0; i < N; ++i)
            for (int64_t j = 0; j < N; ++j) {
                xs[i * N + j] = static_cast<double>(j);
                ys[i * N + j] = static_cast<double>(i);
            }
        return 0;
    }
    if (kind == 3) {
        FemMesh M(p1, static_cast<uint64_t>(p2));
        for (int64_t j = 1; j <= p1 - 2; ++j)
            for (int64_t i = 1; i <= p1 - 2; ++i) M.coord(i, j, xs[M.dof(i, j)], ys[M.dof(i, j)]);
        return 0;
    }
    return 6;
}

// partition_contiguous: rank p owns [p*ceil(n/P), min((p+1)*ceil(n/P), n)).
int orc_partition_contiguous(int64_t n, int32_t P, int32_t* part_of) {
    if (P < 1 || P > n) return 6;
    const int64_t blk = (n + P - 1) / P;
    for (int64_t i = 0; i < n; ++i) part_of[i] = static_cast<int32_t>(i / blk);
    return 0;
}

// partition_rcb: recursive median split on the longer bounding-box axis
// (ties -> x), nodes ordered by (coordinate, global index), left half gets ceil(len/2).
static void rcb_rec(std::vector<int64_t>& idx, int64_t b, int64_t e, const double* xs,
                    const double* ys, int32_t P, int32_t off, int32_t* part_of) {
    if (P == 1) {
        for (int64_t k = b; k < e; ++k) part_of[idx[k]] = off;
        return;
    }
    double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    for (int64_t k = b; k < e; ++k) {
        xmin = std::min(xmin, xs[idx[k]]); xmax = std::max(xmax, xs[idx[k]]);
        ymin = std::min(ymin, ys[idx[k]]); ymax = std::max(ymax, ys[idx[k]]);
    }
    const double* c = (xmax - xmin >= ymax - ymin) ? xs : ys;
    std::sort(idx.begin() + b, idx.begin() + e, [c](int64_t a, int64_t q) {
        if (c[a] != c[q]) return c[a] < c[q];
        return a < q;
    });
    const int64_t mid = b + (e - b + 1) / 2;
    rcb_rec(idx, b, mid, xs, ys, P / 2, off, part_of);
    rcb_rec(idx, mid, e, xs, ys, P / 2, off + P / 2, part_of);
}

int orc_partition_rcb(int64_t n, const double* xs, const double* ys, int32_t P, int32_t* part_of) {
    if (P < 1 || (P & (P - 1)) != 0 || P > n) return 6;
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), int64_t{0});
    rcb_rec(idx, 0, n, xs, ys, P, 0, part_of);
    return 0;
}

struct orc_local { Local L; };

orc_local* orc_local_build(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                           const int32_t* part_of, int32_t P, int32_t rank) {
    auto* h = new orc_local;
    h->L = build_local(n, rp, ci, v, part_of, P, rank);
    return h;
}
void orc_local_sizes(const orc_local* h, int64_t* s) {
    const Local& L = h->L;
    s[0] = static_cast<int64_t>(L.owned.size());
    s[1] = static_cast<int64_t>(L.halo.size());
    s[2] = static_cast<int64_t>(L.neighbors.size());
    s[3] = static_cast<int64_t>(L.ci.size());
    s[4] = static_cast<int64_t>(L.send_idx.size());
    s[5] = static_cast<int64_t>(L.recv_idx.size());
}
void orc_local_get(const orc_local* h, int64_t* owned, int64_t* halo, int32_t* nb, int64_t* sp,
                   int64_t* si, int64_t* rcp, int64_t* rci, int64_t* lrp, int64_t* lci,
                   double* lv) {
    const Local& L = h->L;
    auto cp = [](auto* dst, const auto& src) {
        if (dst) std::copy(src.begin(), src.end(), dst);
    };
    cp(owned, L.owned); cp(halo, L.halo); cp(nb, L.neighbors);
    cp(sp, L.send_ptr); cp(si, L.send_idx); cp(rcp, L.recv_ptr); cp(rci, L.recv_idx);
    cp(lrp, L.rp); cp(lci, L.ci); cp(lv, L.v);
}
void orc_local_free(orc_local* h) { delete h; }

int orc_dist_solve(int32_t kind, int64_t n, const int64_t* rp, const int64_t* ci,
                   const double* v, const double* b, const int32_t* part_of, int32_t P,
                   const orc_opts* o, double* x_global, orc_report* rep, int64_t* counters) {
    if (!validate_opts(o)) return 6;
    std::vector<Local> locs(P);
    for (int32_t r = 0; r < P; ++r) locs[r] = build_local(n, rp, ci, v, part_of, P, r);
    std::vector<double> d;
    precond_vec(n, rp, ci, v, o->preconditioner, d);
    Transport T(P);
    std::vector<orc_report> reps(P);
    std::vector<int64_t> hx(P), ar(P);
    const int saved = g_threads;
    g_threads = 1;  // one worker per rank, single-threaded within a rank
    std::vector<std::thread> th;
    for (int32_t r = 0; r < P; ++r) {
        th.emplace_back([&, r] {
            Local& L = locs[r];
            DistSpace S{&L, &T, static_cast<int64_t>(L.owned.size()), {}};
            S.xl.assign(L.owned.size() + L.halo.size(), 0.0);
            std::vector<double> bl(S.n), xl(S.n), dl(S.n);
            for (int64_t a = 0; a < S.n; ++a) { bl[a] = b[L.owned[a]]; dl[a] = d[L.owned[a]]; }
            if (kind == 1) bicgstab_core(S, bl.data(), xl.data(), dl.data(), o, &reps[r]);
            else cg_core(S, bl.data(), xl.data(), dl.data(), o, &reps[r]);
            for (int64_t a = 0; a < S.n; ++a) x_global[L.owned[a]] = xl[a];  // gather_solution
            hx[r] = S.halo_exchanges;
            ar[r] = S.allreduces;
        });
    }
    for (auto& t : th) t.join();
    g_threads = saved;
    *rep = reps[0];
    if (counters) {
        counters[0] = hx[0];
        counters[1] = ar[0];
        counters[2] = T.messages.load();
    }
    return 0;
}

int orc_dist_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  const double* x, const int32_t* part_of, int32_t P, double* y) {
    std::vector<Local> locs(P);
    for (int32_t r = 0; r < P; ++r) locs[r] = build_local(n, rp, ci, v, part_of, P, r);
    Transport T(P);
    std::vector<std::thread> th;
    for (int32_t r = 0; r < P; ++r) {
        th.emplace_back([&, r] {
            Local& L = locs[r];
            DistSpace S{&L, &T, static_cast<int64_t>(L.owned.size()), {}};
            S.xl.assign(L.owned.size() + L.halo.size(), 0.0);
            std::vector<double> xo(S.n), yo(S.n);
            for (int64_t a = 0; a < S.n; ++a) xo[a] = x[L.owned[a]];
            S.spmv(xo.data(), yo.data());
            for (int64_t a = 0; a < S.n; ++a) y[L.owned[a]] = yo[a];
        });
    }
    for (auto& t : th) t.join();
    return 0;
}

// dist_adjoint_solve: distributed solve on A^T reusing the forward halo
// maps (valid under structural symmetry), then grad_vals from owned lambda and x over
// [owned|halo] (one extra exchange of x).
int orc_dist_adjoint(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     const double* x, const double* g, const int32_t* part_of, int32_t P,
                     const orc_opts* o, double* grad_b, double* grad_vals, orc_report* rep) {
    if (!validate_opts(o)) return 6;
    // structural symmetry check (build-time)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            int64_t j = ci[k];
            if (!std::binary_search(ci + rp[j], ci + rp[j + 1], i)) return 5;
        }
    const int64_t nnz = rp[n];
    std::vector<int64_t> trp(n + 1), tci(nnz);
    std::vector<double> tv(nnz);
    orc_csr_transpose(n, n, rp, ci, v, trp.data(), tci.data(), tv.data());
    std::vector<double> lam(n, 0.0);
    bool all_zero = true;
    for (int64_t i = 0; i < n; ++i)
        if (g[i] != 0.0) { all_zero = false; break; }
    if (all_zero) {
        std::memset(rep, 0, sizeof(*rep));
        rep->converged = 1;
        set_diag(rep, "grad_x == 0: short-circuit");
    } else {
        int64_t counters[3];
        int rc = orc_dist_solve(0, n, trp.data(), tci.data(), tv.data(), g, part_of, P, o,
                                lam.data(), rep, counters);
        if (rc) return rc;
    }
    for (int64_t i = 0; i < n; ++i) grad_b[i] = lam[i];
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) grad_vals[k] = -(lam[i] * x[ci[k]]);
    return 0;
}

}  // extern "C"
