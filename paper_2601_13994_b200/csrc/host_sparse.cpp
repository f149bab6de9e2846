// host_sparse.cpp — host side of the drop-in: canonical COO/CSR assembly, transpose,
// symmetry checks, the deterministic problem generators, the METIS-free partitioners and
// the owned/halo index maps (build_local).  Per the north star these stay on the host;
// they are multi-threaded C++ and never touch the GPU.
//
// Reference behaviour restated (not copied):
//   SparseCoo ctor       sparse.cpp:9-53    -> canonicalize_coo (counting sort by row +
//                                              per-row stable sort by col: same order as
//                                              the reference's stable (row,col) sort)
//   CsrMatrix::from_coo  sparse.cpp:94-116  -> sparsla_csr_from_coo
//   CsrMatrix::to_coo    sparse.cpp:118-127 -> sparsla_csr_to_coo_rows
//   transpose            sparse.cpp:176-182 -> csr_transpose_host
//   is_*symmetric        sparse.cpp:184-205 -> sparsla_csr_symmetry
//   poisson2d            SPEC.md:561-569    -> generator kind 0
//   partition_*          SPEC.md:443-460    -> sparsla_partition_contiguous / _rcb
//   build_local          SPEC.md:461-469    -> sparsla_local_build
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "common.hpp"

namespace sparsla_b200 {

namespace {
thread_local std::string t_last_error;
}

void set_last_error(const std::string& msg) { t_last_error = msg; }

int host_threads() {
    static int n = [] {
        unsigned h = std::thread::hardware_concurrency();
        return h == 0 ? 1 : static_cast<int>(h);
    }();
    return n;
}

template <class I>
void validate_csr(int64_t nrows, int64_t ncols, const I* rp, const I* ci) {
    if (nrows < 0 || ncols < 0) fail(SPARSLA_ERR_DIMENSION, "negative matrix shape");
    if (rp[0] != 0) fail(SPARSLA_ERR_INVALID_ARGUMENT, "row_ptr[0] must be 0");
    std::atomic<int> bad{0};
    parallel_for(nrows, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            if (rp[i + 1] < rp[i]) { bad = 1; return; }
            for (int64_t k = rp[i]; k < static_cast<int64_t>(rp[i + 1]); ++k) {
                if (ci[k] < 0 || ci[k] >= ncols) { bad = 2; return; }
                if (k > rp[i] && ci[k] <= ci[k - 1]) { bad = 3; return; }
            }
        }
    });
    if (bad == 1) fail(SPARSLA_ERR_INVALID_ARGUMENT, "row_ptr must be non-decreasing");
    if (bad == 2) fail(SPARSLA_ERR_BOUNDS, "column index outside matrix shape");
    if (bad == 3) fail(SPARSLA_ERR_INVALID_ARGUMENT,
                       "columns must be strictly increasing within each row (canonical CSR)");
}
template void validate_csr<int64_t>(int64_t, int64_t, const int64_t*, const int64_t*);
template void validate_csr<int32_t>(int64_t, int64_t, const int32_t*, const int32_t*);

int64_t canonicalize_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                         const int64_t* cols, const double* vals, int64_t* ro, int64_t* co,
                         double* vo) {
    if (nrows < 0 || ncols < 0) fail(SPARSLA_ERR_DIMENSION, "negative matrix shape");
    for (int64_t k = 0; k < nnz; ++k)
        if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols)
            fail(SPARSLA_ERR_BOUNDS, "coo index (" + std::to_string(rows[k]) + ", " +
                                         std::to_string(cols[k]) + ") outside shape (" +
                                         std::to_string(nrows) + ", " + std::to_string(ncols) +
                                         ") at entry " + std::to_string(k));
    // Stable counting sort by row: entries of a row keep their input order.
    std::vector<int64_t> start(static_cast<size_t>(nrows) + 1, 0);
    for (int64_t k = 0; k < nnz; ++k) ++start[static_cast<size_t>(rows[k]) + 1];
    for (int64_t i = 0; i < nrows; ++i) start[i + 1] += start[i];
    std::vector<int64_t> perm(static_cast<size_t>(nnz));
    {
        std::vector<int64_t> fill(start.begin(), start.end() - 1);
        for (int64_t k = 0; k < nnz; ++k) perm[fill[rows[k]]++] = k;
    }
    // Per row: stable sort by column (ties keep input order), then sum duplicates in
    // input order.  Row i's output lands at [out_start[i], ...).
    std::vector<int64_t> ucount(static_cast<size_t>(nrows), 0);
    parallel_for(nrows, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            int64_t* p = perm.data() + start[i];
            const int64_t len = start[i + 1] - start[i];
            std::stable_sort(p, p + len, [cols](int64_t x, int64_t y) { return cols[x] < cols[y]; });
            int64_t u = 0;
            for (int64_t k = 0; k < len; ++k)
                if (k == 0 || cols[p[k]] != cols[p[k - 1]]) ++u;
            ucount[i] = u;
        }
    });
    std::vector<int64_t> out_start(static_cast<size_t>(nrows) + 1, 0);
    for (int64_t i = 0; i < nrows; ++i) out_start[i + 1] = out_start[i] + ucount[i];
    parallel_for(nrows, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            const int64_t* p = perm.data() + start[i];
            const int64_t len = start[i + 1] - start[i];
            int64_t o = out_start[i] - 1;
            for (int64_t k = 0; k < len; ++k) {
                const int64_t e = p[k];
                if (k > 0 && cols[e] == co[o]) {
                    vo[o] += vals[e];
                } else {
                    ++o;
                    ro[o] = i;
                    co[o] = cols[e];
                    vo[o] = vals[e];
                }
            }
        }
    });
    return out_start[nrows];
}

void csr_transpose_host(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                        const double* v, int64_t* trp, int64_t* tci, double* tv) {
    std::fill(trp, trp + ncols + 1, int64_t{0});
    const int64_t nnz = rp[nrows];
    for (int64_t k = 0; k < nnz; ++k) ++trp[ci[k] + 1];
    for (int64_t j = 0; j < ncols; ++j) trp[j + 1] += trp[j];
    std::vector<int64_t> next(trp, trp + ncols);
    // rows ascending -> each A^T row lists source rows ascending (canonical order)
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t pos = next[ci[k]]++;
            tci[pos] = i;
            tv[pos] = v[k];
        }
}

// ------------------------------------------------------------------------------------
// Generators.  Matrices are defined by their element-order triplets (SparseCoo semantic:
// duplicates summed in emission order); here each row is produced directly in canonical
// column order with the same per-entry floating-point operations, so the result equals
// canonicalizing the triplets bit for bit (checked against the oracle in tests).
// ------------------------------------------------------------------------------------
namespace gen {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Jittered P1 mesh: lattice (i,j) in [0,m)^2, h = 1/(m-1),
// interior points moved by ((u - 0.5) * 0.5) * h, u ~ U[0,1) from a counter-based hash
// (seed, node id, component); each cell split along the Delaunay (in-circle) diagonal.
struct Fem {
    int64_t m;
    uint64_t hseed;
    double h;
    Fem(int64_t m_, uint64_t seed) : m(m_), hseed(splitmix64(seed)), h(1.0 / double(m_ - 1)) {}
    bool interior(int64_t i, int64_t j) const { return i >= 1 && i <= m - 2 && j >= 1 && j <= m - 2; }
    int64_t dof(int64_t i, int64_t j) const { return (j - 1) * (m - 2) + (i - 1); }
    double u01(uint64_t id, uint64_t comp) const {
        return double(splitmix64(hseed ^ (2 * id + comp)) >> 11) * 0x1.0p-53;
    }
    void coord(int64_t i, int64_t j, double& x, double& y) const {
        x = double(i) * h;
        y = double(j) * h;
        if (interior(i, j)) {
            const uint64_t id = uint64_t(j * m + i);
            x = x + ((u01(id, 0) - 0.5) * 0.5) * h;
            y = y + ((u01(id, 1) - 0.5) * 0.5) * h;
        }
    }
    // two ccw triangles of cell (ci, cj) as vertex lattice coords
    void tris(int64_t ci, int64_t cj, int64_t T[2][3][2]) const {
        double ax, ay, bx, by, cx, cy, dx, dy;
        coord(ci, cj, ax, ay);
        coord(ci + 1, cj, bx, by);
        coord(ci + 1, cj + 1, cx, cy);
        coord(ci, cj + 1, dx, dy);
        const double adx = ax - dx, ady = ay - dy, bdx = bx - dx, bdy = by - dy;
        const double cdx = cx - dx, cdy = cy - dy;
        const double al = adx * adx + ady * ady;
        const double bl = bdx * bdx + bdy * bdy;
        const double cl = cdx * cdx + cdy * cdy;
        const double t1 = al * (bdx * cdy - cdx * bdy);
        const double t2 = bl * (cdx * ady - adx * cdy);
        const double t3 = cl * (adx * bdy - bdx * ady);
        const double det = (t1 + t2) + t3;
        const int64_t a[2] = {ci, cj}, b[2] = {ci + 1, cj}, c[2] = {ci + 1, cj + 1}, d[2] = {ci, cj + 1};
        const int64_t* V[2][3];
        if (det > 0.0) { V[0][0] = a; V[0][1] = b; V[0][2] = d; V[1][0] = b; V[1][1] = c; V[1][2] = d; }
        else           { V[0][0] = a; V[0][1] = b; V[0][2] = c; V[1][0] = a; V[1][1] = c; V[1][2] = d; }
        for (int t = 0; t < 2; ++t)
            for (int k = 0; k < 3; ++k) { T[t][k][0] = V[t][k][0]; T[t][k][1] = V[t][k][1]; }
    }
    // row `a` of the P1 stiffness of triangle T: (b_a b_l + c_a c_l) / (2 * area2)
    void stiff_row(const int64_t T[3][2], int a, double out[3]) const {
        double x[3], y[3];
        for (int k = 0; k < 3; ++k) coord(T[k][0], T[k][1], x[k], y[k]);
        const double bb[3] = {y[1] - y[2], y[2] - y[0], y[0] - y[1]};
        const double cc[3] = {x[2] - x[1], x[0] - x[2], x[1] - x[0]};
        const double area2 = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
        const double den = 2.0 * area2;
        for (int l = 0; l < 3; ++l) out[l] = (bb[a] * bb[l] + cc[a] * cc[l]) / den;
    }
    // entries of row (i,j): (col, value) sorted by col; value summed in element order
    int row(int64_t i, int64_t j, int64_t* cols, double* vals) const {
        int cnt = 0;
        const int64_t cells[4][2] = {{i - 1, j - 1}, {i, j - 1}, {i - 1, j}, {i, j}};
        for (auto& cell : cells) {
            int64_t T[2][3][2];
            tris(cell[0], cell[1], T);
            for (int t = 0; t < 2; ++t) {
                int a = -1;
                for (int k = 0; k < 3; ++k)
                    if (T[t][k][0] == i && T[t][k][1] == j) a = k;
                if (a < 0) continue;
                double K[3];
                stiff_row(T[t], a, K);
                for (int l = 0; l < 3; ++l) {
                    if (!interior(T[t][l][0], T[t][l][1])) continue;
                    const int64_t c = dof(T[t][l][0], T[t][l][1]);
                    int s = 0;
                    while (s < cnt && cols[s] != c) ++s;
                    if (s == cnt) { cols[cnt] = c; vals[cnt] = K[l]; ++cnt; }
                    else vals[s] += K[l];
                }
            }
        }
        // insertion sort by column (values travel with their column)
        for (int a = 1; a < cnt; ++a)
            for (int b = a; b > 0 && cols[b - 1] > cols[b]; --b) {
                std::swap(cols[b - 1], cols[b]);
                std::swap(vals[b - 1], vals[b]);
            }
        return cnt;
    }
};

struct Spec {
    int32_t kind;
    int64_t p1, p2;
    double fparam;
    int64_t n() const {
        switch (kind) {
            case 0: return p1 * p1;
            case 1: case 2: return p1 * p1 * p1;
            case 3: return (p1 - 2) * (p1 - 2);
            case 4: return p1 * p1 * p2;
        }
        return -1;
    }
    void check() const {
        if (kind < 0 || kind > 4) fail(SPARSLA_ERR_INVALID_ARGUMENT, "unknown generator kind");
        if (kind == 4 && p2 < 2) fail(SPARSLA_ERR_INVALID_ARGUMENT, "generator size too small (Nz >= 2)");
        if ((kind <= 2 && p1 < 2) || (kind == 3 && p1 < 3) || (kind == 4 && p1 < 2))
            fail(SPARSLA_ERR_INVALID_ARGUMENT, "generator size too small (N >= 2, m >= 3)");
    }
    // entries of global row k, canonical order; returns count (<= 9)
    int row(int64_t k, int64_t* cols, double* vals, const Fem* fem) const {
        int cnt = 0;
        auto put = [&](int64_t c, double v) { cols[cnt] = c; vals[cnt] = v; ++cnt; };
        if (kind == 0) {
            const int64_t N = p1, i = k / N, j = k % N;
            if (i > 0) put(k - N, -1.0);
            if (j > 0) put(k - 1, -1.0);
            put(k, 4.0);
            if (j < N - 1) put(k + 1, -1.0);
            if (i < N - 1) put(k + N, -1.0);
        } else if (kind == 4) {  // N x N x Nz box (weak-scaling slabs, config E)
            const int64_t N = p1, NN = N * N, Nz = p2, z = k / NN, y = (k / N) % N, x = k % N;
            if (z > 0) put(k - NN, -1.0);
            if (y > 0) put(k - N, -1.0);
            if (x > 0) put(k - 1, -1.0);
            put(k, 6.0);
            if (x < N - 1) put(k + 1, -1.0);
            if (y < N - 1) put(k + N, -1.0);
            if (z < Nz - 1) put(k + NN, -1.0);
        } else if (kind == 1 || kind == 2) {
            const int64_t N = p1, NN = N * N, z = k / NN, y = (k / N) % N, x = k % N;
            const double c = fparam;
            const double diag = kind == 2 ? 6.0 + 3.0 * c : 6.0;
            const double lo = kind == 2 ? -1.0 - c : -1.0;
            if (z > 0) put(k - NN, lo);
            if (y > 0) put(k - N, lo);
            if (x > 0) put(k - 1, lo);
            put(k, diag);
            if (x < N - 1) put(k + 1, -1.0);
            if (y < N - 1) put(k + N, -1.0);
            if (z < N - 1) put(k + NN, -1.0);
        } else {
            const int64_t w = p1 - 2;
            cnt = fem->row(k % w + 1, k / w + 1, cols, vals);
        }
        return cnt;
    }
};

template <class RP, class CI>
void fill(const Spec& s, int64_t r0, int64_t r1, RP* rp, CI* ci, double* v) {
    const int64_t nr = r1 - r0;
    Fem fem(s.kind == 3 ? s.p1 : 3, static_cast<uint64_t>(s.p2));
    std::vector<int64_t> cnt(static_cast<size_t>(nr));
    parallel_for(nr, [&](int64_t a, int64_t b) {
        int64_t c[16];
        double x[16];
        for (int64_t i = a; i < b; ++i) cnt[i] = s.row(r0 + i, c, x, &fem);
    }, 1 << 12);
    rp[0] = 0;
    for (int64_t i = 0; i < nr; ++i) rp[i + 1] = static_cast<RP>(rp[i] + cnt[i]);
    parallel_for(nr, [&](int64_t a, int64_t b) {
        int64_t c[16];
        double x[16];
        for (int64_t i = a; i < b; ++i) {
            const int m = s.row(r0 + i, c, x, &fem);
            const int64_t o = static_cast<int64_t>(rp[i]);
            for (int q = 0; q < m; ++q) { ci[o + q] = static_cast<CI>(c[q]); v[o + q] = x[q]; }
        }
    }, 1 << 12);
}

int64_t count(const Spec& s, int64_t r0, int64_t r1) {
    if (s.kind == 0) {  // closed forms for the stencils
        const int64_t N = s.p1;
        int64_t t = 0;
        for (int64_t k = r0; k < r1; ++k) {
            const int64_t i = k / N, j = k % N;
            t += 1 + (i > 0) + (j > 0) + (j < N - 1) + (i < N - 1);
        }
        return t;
    }
    if (s.kind == 4) {
        const int64_t N = s.p1, Nz = s.p2;
        std::atomic<int64_t> tot{0};
        parallel_for(r1 - r0, [&](int64_t a, int64_t b) {
            int64_t t = 0;
            for (int64_t k = r0 + a; k < r0 + b; ++k) {
                const int64_t z = k / (N * N), y = (k / N) % N, x = k % N;
                t += 1 + (z > 0) + (y > 0) + (x > 0) + (x < N - 1) + (y < N - 1) + (z < Nz - 1);
            }
            tot += t;
        });
        return tot.load();
    }
    if (s.kind == 1 || s.kind == 2) {
        const int64_t N = s.p1;
        std::atomic<int64_t> tot{0};
        parallel_for(r1 - r0, [&](int64_t a, int64_t b) {
            int64_t t = 0;
            for (int64_t k = r0 + a; k < r0 + b; ++k) {
                const int64_t z = k / (N * N), y = (k / N) % N, x = k % N;
                t += 1 + (z > 0) + (y > 0) + (x > 0) + (x < N - 1) + (y < N - 1) + (z < N - 1);
            }
            tot += t;
        });
        return tot.load();
    }
    Fem fem(s.p1, static_cast<uint64_t>(s.p2));
    std::atomic<int64_t> tot{0};
    parallel_for(r1 - r0, [&](int64_t a, int64_t b) {
        int64_t c[16];
        double x[16];
        int64_t t = 0;
        for (int64_t k = r0 + a; k < r0 + b; ++k) t += s.row(k, c, x, &fem);
        tot += t;
    }, 1 << 12);
    return tot.load();
}

}  // namespace gen

// ------------------------------------------------------------------------------------
// RCB: split the longer bounding-box axis (ties -> x) at the median of
// the strict order (coordinate, global index); left half takes ceil(len/2).
// ------------------------------------------------------------------------------------
void rcb(std::vector<int64_t>& idx, int64_t b, int64_t e, const double* xs, const double* ys,
         int32_t P, int32_t off, int32_t* part) {
    if (P == 1) {
        for (int64_t k = b; k < e; ++k) part[idx[k]] = off;
        return;
    }
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (int64_t k = b; k < e; ++k) {
        const double x = xs[idx[k]], y = ys[idx[k]];
        x0 = std::min(x0, x); x1 = std::max(x1, x);
        y0 = std::min(y0, y); y1 = std::max(y1, y);
    }
    const double* c = (x1 - x0 >= y1 - y0) ? xs : ys;
    const int64_t mid = b + (e - b + 1) / 2;
    auto less = [c](int64_t p, int64_t q) { return c[p] != c[q] ? c[p] < c[q] : p < q; };
    std::nth_element(idx.begin() + b, idx.begin() + mid, idx.begin() + e, less);
    rcb(idx, b, mid, xs, ys, P / 2, off, part);
    rcb(idx, mid, e, xs, ys, P / 2, off + P / 2, part);
}

}  // namespace sparsla_b200

using namespace sparsla_b200;

// ------------------------------------------------------------------------------------
// build_local result
// ------------------------------------------------------------------------------------

extern "C" {

const char* sparsla_last_error_message(void) { return t_last_error.c_str(); }
int sparsla_version(void) { return 100; }

int sparsla_coo_canonicalize(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                             const int64_t* cols, const double* vals, int64_t* out_nnz,
                             int64_t* ro, int64_t* co, double* vo) {
    return guarded([&] {
        if (nnz < 0) fail(SPARSLA_ERR_DIMENSION, "negative nnz");
        *out_nnz = canonicalize_coo(nrows, ncols, nnz, rows, cols, vals, ro, co, vo);
    });
}

int sparsla_csr_from_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                         const int64_t* cols, const double* vals, int64_t* rp, int64_t* ci,
                         double* vo) {
    return guarded([&] {
        if (nrows < 0 || ncols < 0) fail(SPARSLA_ERR_DIMENSION, "negative matrix shape");
        std::fill(rp, rp + nrows + 1, int64_t{0});
        for (int64_t k = 0; k < nnz; ++k) {
            if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols)
                fail(SPARSLA_ERR_BOUNDS, "coo index outside shape");
            if (k > 0 && (rows[k] < rows[k - 1] || (rows[k] == rows[k - 1] && cols[k] <= cols[k - 1])))
                fail(SPARSLA_ERR_INVALID_ARGUMENT, "coo input is not canonical");
            ++rp[rows[k] + 1];
        }
        for (int64_t i = 0; i < nrows; ++i) rp[i + 1] += rp[i];
        std::memcpy(ci, cols, sizeof(int64_t) * static_cast<size_t>(nnz));
        std::memcpy(vo, vals, sizeof(double) * static_cast<size_t>(nnz));
    });
}

int sparsla_csr_to_coo_rows(int64_t nrows, const int64_t* rp, int64_t* rows_out) {
    return guarded([&] {
        parallel_for(nrows, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i)
                for (int64_t k = rp[i]; k < rp[i + 1]; ++k) rows_out[k] = i;
        });
    });
}

int sparsla_csr_transpose(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                          const double* v, int64_t* trp, int64_t* tci, double* tv) {
    return guarded([&] { csr_transpose_host(nrows, ncols, rp, ci, v, trp, tci, tv); });
}

int sparsla_csr_symmetry(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                         const double* v, double tol, int32_t* ssym, int32_t* sym) {
    return guarded([&] {
        if (nrows != ncols) { *ssym = 0; *sym = 0; return; }
        std::atomic<int> s1{1}, s2{1};
        parallel_for(nrows, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i)
                for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                    const int64_t j = ci[k];
                    const int64_t* lo = ci + rp[j];
                    const int64_t* hi = ci + rp[j + 1];
                    const int64_t* f = std::lower_bound(lo, hi, i);
                    if (f == hi || *f != i) { s1 = 0; s2 = 0; return; }
                    if (std::abs(v[k] - v[f - ci]) > tol) s2 = 0;
                }
        });
        *ssym = s1.load();
        *sym = s1.load() && s2.load();
    });
}

int sparsla_gen_size(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t r0, int64_t r1,
                     int64_t* n_global, int64_t* nnz) {
    return guarded([&] {
        gen::Spec s{kind, p1, p2, fparam};
        s.check();
        const int64_t n = s.n();
        if (r0 < 0 || r1 < r0 || r1 > n) fail(SPARSLA_ERR_BOUNDS, "row range outside matrix");
        *n_global = n;
        *nnz = gen::count(s, r0, r1);
    });
}

int sparsla_gen_csr(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t r0, int64_t r1,
                    int64_t* rp, int64_t* ci, double* v) {
    return guarded([&] {
        gen::Spec s{kind, p1, p2, fparam};
        s.check();
        if (r0 < 0 || r1 < r0 || r1 > s.n()) fail(SPARSLA_ERR_BOUNDS, "row range outside matrix");
        gen::fill(s, r0, r1, rp, ci, v);
    });
}

int sparsla_gen_csr_i32(int32_t kind, int64_t p1, int64_t p2, double fparam, int64_t r0,
                        int64_t r1, int32_t* rp, int32_t* ci, double* v) {
    return guarded([&] {
        gen::Spec s{kind, p1, p2, fparam};
        s.check();
        if (r0 < 0 || r1 < r0 || r1 > s.n()) fail(SPARSLA_ERR_BOUNDS, "row range outside matrix");
        if (s.n() >= (int64_t{1} << 31)) fail(SPARSLA_ERR_UNSUPPORTED, "n exceeds int32 columns");
        if (gen::count(s, r0, r1) >= (int64_t{1} << 31))
            fail(SPARSLA_ERR_UNSUPPORTED, "nnz of the row range exceeds int32 row_ptr");
        gen::fill(s, r0, r1, rp, ci, v);
    });
}

int sparsla_gen_coords(int32_t kind, int64_t p1, int64_t p2, double* xs, double* ys) {
    return guarded([&] {
        if (kind == 0) {
            const int64_t N = p1;
            for (int64_t i = 0; i < N; ++i)
                for (int64_t j = 0; j < N; ++j) { xs[i * N + j] = double(j); ys[i * N + j] = double(i); }
        } else if (kind == 3) {
            gen::Fem f(p1, static_cast<uint64_t>(p2));
            for (int64_t j = 1; j <= p1 - 2; ++j)
                for (int64_t i = 1; i <= p1 - 2; ++i) f.coord(i, j, xs[f.dof(i, j)], ys[f.dof(i, j)]);
        } else {
            fail(SPARSLA_ERR_INVALID_ARGUMENT, "coordinates exist for 2-D kinds (0, 3) only");
        }
    });
}

int sparsla_partition_contiguous(int64_t n, int32_t P, int32_t* part_of) {
    return guarded([&] {
        if (P < 1 || P > n) fail(SPARSLA_ERR_INVALID_ARGUMENT, "partition_contiguous requires 1 <= P <= n");
        const int64_t blk = (n + P - 1) / P;
        parallel_for(n, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i) part_of[i] = static_cast<int32_t>(i / blk);
        });
    });
}

int sparsla_partition_rcb(int64_t n, const double* xs, const double* ys, int32_t P, int32_t* part_of) {
    return guarded([&] {
        if (P < 1 || (P & (P - 1)) != 0)
            fail(SPARSLA_ERR_INVALID_ARGUMENT, "partition_rcb requires P to be a power of two");
        if (P > n) fail(SPARSLA_ERR_INVALID_ARGUMENT, "partition_rcb requires P <= n");
        std::vector<int64_t> idx(static_cast<size_t>(n));
        std::iota(idx.begin(), idx.end(), int64_t{0});
        rcb(idx, 0, n, xs, ys, P, 0, part_of);
    });
}

// build_local from owned rows only (structurally symmetric pattern):
// halo = referenced non-owned columns (equals SPEC.md:426's union rule under symmetry);
// send to q = owned rows referencing a column owned by q; recv from q = halo owned by q.
int sparsla_local_build(int64_t n_global, const int32_t* part_of, int32_t P, int32_t rank,
                        int64_t no, const int64_t* owned, const int64_t* rp, const int64_t* ci,
                        const double* v, sparsla_local** out) {
    return guarded([&] {
        if (rank < 0 || rank >= P) fail(SPARSLA_ERR_INVALID_ARGUMENT, "rank outside [0, P)");
        // part_of == nullptr: contiguous partition computed on the fly, so
        // a rank of a 400M-row problem never materialises the global map
        const int64_t blk = (n_global + P - 1) / std::max<int32_t>(P, 1);
        auto part = [&](int64_t g) -> int32_t { return part_of ? part_of[g] : (int32_t)(g / blk); };
        for (int64_t a = 0; a < no; ++a) {
            if (owned[a] < 0 || owned[a] >= n_global || part(owned[a]) != rank)
                fail(SPARSLA_ERR_INVALID_ARGUMENT, "owned list disagrees with part_of");
            if (a > 0 && owned[a] <= owned[a - 1])
                fail(SPARSLA_ERR_INVALID_ARGUMENT, "owned list must be strictly ascending");
        }
        auto* L = new sparsla_local;
        std::unique_ptr<sparsla_local> guard_L(L);
        L->owned.assign(owned, owned + no);
        const int64_t nnz = rp[no];
        std::vector<int64_t> cand;
        for (int64_t k = 0; k < nnz; ++k) {
            const int64_t c = ci[k];
            if (c < 0 || c >= n_global) fail(SPARSLA_ERR_BOUNDS, "column outside matrix");
            if (part(c) != rank) cand.push_back(c);
        }
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        L->halo = std::move(cand);
        const int64_t nh = static_cast<int64_t>(L->halo.size());
        std::vector<char> nb(static_cast<size_t>(P), 0);
        for (int64_t h : L->halo) nb[part(h)] = 1;
        for (int32_t q = 0; q < P; ++q)
            if (nb[q]) L->neighbors.push_back(q);
        const bool contiguous = no == 0 || owned[no - 1] - owned[0] == no - 1;
        auto g2l = [&](int64_t g) -> int64_t {
            if (part(g) == rank) {
                if (contiguous) return g - owned[0];
                return std::lower_bound(L->owned.begin(), L->owned.end(), g) - L->owned.begin();
            }
            return no + (std::lower_bound(L->halo.begin(), L->halo.end(), g) - L->halo.begin());
        };
        L->recv_ptr.push_back(0);
        for (int32_t q : L->neighbors) {
            for (int64_t a = 0; a < nh; ++a)
                if (part(L->halo[a]) == q) L->recv_idx.push_back(no + a);
            L->recv_ptr.push_back(static_cast<int64_t>(L->recv_idx.size()));
        }
        L->send_ptr.push_back(0);
        for (int32_t q : L->neighbors) {
            for (int64_t a = 0; a < no; ++a) {
                bool need = false;
                for (int64_t k = rp[a]; k < rp[a + 1] && !need; ++k) need = part(ci[k]) == q;
                if (need) L->send_idx.push_back(a);
            }
            L->send_ptr.push_back(static_cast<int64_t>(L->send_idx.size()));
        }
        L->rp.assign(rp, rp + no + 1);
        L->ci.resize(static_cast<size_t>(nnz));
        L->v.assign(v, v + nnz);
        parallel_for(nnz, [&](int64_t a, int64_t b) {
            for (int64_t k = a; k < b; ++k) L->ci[k] = g2l(ci[k]);
        });
        *out = guard_L.release();
    });
}

int sparsla_local_sizes(const sparsla_local* L, int64_t* s) {
    return guarded([&] {
        s[0] = static_cast<int64_t>(L->owned.size());
        s[1] = static_cast<int64_t>(L->halo.size());
        s[2] = static_cast<int64_t>(L->neighbors.size());
        s[3] = static_cast<int64_t>(L->ci.size());
        s[4] = static_cast<int64_t>(L->send_idx.size());
        s[5] = static_cast<int64_t>(L->recv_idx.size());
    });
}

int sparsla_local_get(const sparsla_local* L, int64_t* owned, int64_t* halo, int32_t* nb,
                      int64_t* sp, int64_t* si, int64_t* rcp, int64_t* rci, int64_t* lrp,
                      int64_t* lci, double* lv) {
    return guarded([&] {
        auto cp = [](auto* dst, const auto& src) {
            if (dst) std::copy(src.begin(), src.end(), dst);
        };
        cp(owned, L->owned); cp(halo, L->halo); cp(nb, L->neighbors);
        cp(sp, L->send_ptr); cp(si, L->send_idx); cp(rcp, L->recv_ptr); cp(rci, L->recv_idx);
        cp(lrp, L->rp); cp(lci, L->ci); cp(lv, L->v);
    });
}

int sparsla_local_destroy(sparsla_local* L) {
    delete L;
    return SPARSLA_OK;
}

}  // extern "C"
