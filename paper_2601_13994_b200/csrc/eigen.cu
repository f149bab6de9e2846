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
//   resid_kernel   R = AX - X diag(lambda), ||R_j||, W = |D|^-1 R         1 pass
//   W: twice { Y = X^T W (gram), W -= X Y (combine), SVQB(W) }           orthonormal W
//   P: twice { Y = [X W]^T P, P -= [X W] Y, SVQB(P) }                    orthonormal P
//   spmm_kernel    AS[:, W P] = A S[:, W P]                               1 SpMM of <= 2m columns
//   gram           G = S_B^T AS_B, B = X u W u P (q <= 3m)               host: eig(G)
//   combine        X' = S_B C, AX' = AS_B C, P' = S_{W,P} C_{W,P}        (Hetmaniuk-Lehoucq P)
// Reductions use a fixed grid (kRedCTAs) and fixed in-CTA orders, so a run is
// deterministic.  Parity is tolerance-based (eigenvalues to 1e-8 against
// a dense symmetric eigensolver) — there is no bitwise reference for this module.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
constexpr int kT = 256;
constexpr int kGramTile = 32;         // rows per shared-memory tile in gram_kernel
constexpr int kGramR = 3;             // 3x3 register tile of the Gram matrix per thread

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

struct Mat {  // small dense coefficient matrix a x c (row-major), kernel parameter
    double v[kMaxQ * kMaxK];
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

// Block SpMV: Y[i, out_j] = sum_k A_ik S[c_k, in_j] for the listed columns, 8 columns per
// pass over the row (the matrix row is re-read from L1 for wider blocks).
__global__ void __launch_bounds__(kT) spmm_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                  const double* __restrict__ val, long long n,
                                                  const double* __restrict__ S, int lds, Cols in, double* Y,
                                                  int ldy, Cols out) {
    __shared__ int s_in[kMaxQ], s_out[kMaxQ];
    stage_cols(in, s_in);
    stage_cols(out, s_out);
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int kb = __ldg(rp + i), ke = __ldg(rp + i + 1);
    for (int g = 0; g < in.n; g += 8) {
        const int w = min(8, in.n - g);
        int col[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) col[j] = j < w ? s_in[g + j] : 0;
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0;
        for (int k = kb; k < ke; ++k) {
            const double v = __ldg(val + k);
            const double* s = S + (size_t)__ldg(ci + k) * lds;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < w) acc[j] = fma(v, __ldg(s + col[j]), acc[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < w) Y[i * ldy + s_out[g + j]] = acc[j];
    }
}

// Gram block G = U_uc^T V_vc (a x b) over the CTA's row range: rows are staged through
// shared memory 32 at a time; each thread owns a 3x3 register tile of G and a residue
// class of the tile's rows; groups are combined in a fixed order.  One partial per CTA.
__global__ void __launch_bounds__(kT) gram_kernel(const double* __restrict__ U, int ldu, Cols uc,
                                                  const double* __restrict__ V, int ldv, Cols vc, long long n,
                                                  double* partial) {
    constexpr int TR = kGramTile, R = kGramR, LDS = kMaxQ + 1;
    __shared__ double sh[2 * TR * LDS];
    __shared__ int s_uc[kMaxQ], s_vc[kMaxQ];
    stage_cols(uc, s_uc);
    stage_cols(vc, s_vc);
    double* Us = sh;
    double* Vs = sh + TR * LDS;
    const int a = uc.n, b = vc.n;
    const int TI = (a + R - 1) / R, TJ = (b + R - 1) / R, tiles = TI * TJ;
    const int ngroups = max(1, kT / tiles);
    const int tid = threadIdx.x, grp = tid / tiles, tt = tid % tiles;
    const bool act = grp < ngroups;
    const int ti = tt / TJ, tj = tt % TJ;
    double acc[R][R];
#pragma unroll
    for (int x = 0; x < R; ++x)
#pragma unroll
        for (int y = 0; y < R; ++y) acc[x][y] = 0.0;
    long long r0, r1;
    cta_rows(n, r0, r1);
    __syncthreads();
    for (long long base = r0; base < r1; base += TR) {
        const int nr = (int)min((long long)TR, r1 - base);
        for (int e = tid; e < nr * a; e += kT) {
            const int r = e / a, l = e - r * a;
            Us[r * LDS + l] = __ldg(U + (base + r) * ldu + s_uc[l]);
        }
        for (int e = tid; e < nr * b; e += kT) {
            const int r = e / b, l = e - r * b;
            Vs[r * LDS + l] = __ldg(V + (base + r) * ldv + s_vc[l]);
        }
        __syncthreads();
        if (act) {
            for (int r = grp; r < nr; r += ngroups) {
                double u[R], v[R];
#pragma unroll
                for (int x = 0; x < R; ++x) u[x] = ti * R + x < a ? Us[r * LDS + ti * R + x] : 0.0;
#pragma unroll
                for (int y = 0; y < R; ++y) v[y] = tj * R + y < b ? Vs[r * LDS + tj * R + y] : 0.0;
#pragma unroll
                for (int x = 0; x < R; ++x)
#pragma unroll
                    for (int y = 0; y < R; ++y) acc[x][y] = fma(u[x], v[y], acc[x][y]);
            }
        }
        __syncthreads();
    }
    // combine the row groups in ascending group order (ngroups * a * b <= 9 * 256 doubles)
    const int ab = a * b;
    if (act) {
#pragma unroll
        for (int x = 0; x < R; ++x)
#pragma unroll
            for (int y = 0; y < R; ++y) {
                const int i = ti * R + x, j = tj * R + y;
                if (i < a && j < b) sh[grp * ab + i * b + j] = acc[x][y];
            }
    }
    __syncthreads();
    for (int e = tid; e < ab; e += kT) {
        double s = 0.0;
        for (int g = 0; g < ngroups; ++g) s += sh[g * ab + e];
        partial[(size_t)blockIdx.x * ab + e] = s;
    }
}

// Sum of the per-CTA partials in CTA order (one thread per entry).
__global__ void partial_sum_kernel(const double* partial, int nparts, int ab, double* out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ab) return;
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += partial[(size_t)p * ab + e];
    out[e] = s;
}

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

// ------------------------------------------------------------ host dense algebra ----
// Cyclic Jacobi eigendecomposition of a symmetric q x q matrix (row-major).  Returns
// eigenvalues ascending in w and the matching orthonormal eigenvectors as the COLUMNS of
// V (row-major q x q).  Quadratically convergent, accurate to working precision for the
// small Rayleigh-Ritz and Gram problems of LOBPCG.
void sym_eig(int q, std::vector<double> A, std::vector<double>& w, std::vector<double>& V) {
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
struct Lobpcg {
    DevCsr* A;
    cudaStream_t s;
    long long n;
    int m, ld;
    double *S = nullptr, *AS = nullptr, *Sn = nullptr, *ASn = nullptr;
    double* partial = nullptr;  // [kRedCTAs][kMaxQ*kMaxQ]
    double* gout = nullptr;     // [kMaxQ*kMaxQ]
    double* h_pin = nullptr;    // pinned [kMaxQ*kMaxQ]
    long long* ipart = nullptr;
    long long spmm_count = 0;

    Lobpcg(DevCsr* A_, int m_) : A(A_), s(A_->stream), n(A_->nrows), m(m_), ld(3 * m_) {
        const size_t bytes = (size_t)n * ld;
        S = dalloc<double>(bytes); AS = dalloc<double>(bytes);
        Sn = dalloc<double>(bytes); ASn = dalloc<double>(bytes);
        CK(cudaMemsetAsync(S, 0, bytes * 8, s)); CK(cudaMemsetAsync(AS, 0, bytes * 8, s));
        CK(cudaMemsetAsync(Sn, 0, bytes * 8, s)); CK(cudaMemsetAsync(ASn, 0, bytes * 8, s));
        partial = dalloc<double>((size_t)kRedCTAs * kMaxQ * kMaxQ);
        gout = dalloc<double>((size_t)kMaxQ * kMaxQ);
        ipart = dalloc<long long>((size_t)kRedCTAs * kMaxK);
        CK(cudaMallocHost(&h_pin, sizeof(double) * kMaxQ * kMaxQ));
    }
    ~Lobpcg() {
        DeviceGuard g(A->device, true);
        cudaFree(S); cudaFree(AS); cudaFree(Sn); cudaFree(ASn);
        cudaFree(partial); cudaFree(gout); cudaFree(ipart);
        if (h_pin) cudaFreeHost(h_pin);
    }
    unsigned grid() const { return (unsigned)((n + kT - 1) / kT); }

    // G = U_uc^T V_vc (host, row-major a x b)
    std::vector<double> gram(const double* U, const Cols& uc, const double* V, const Cols& vc) {
        const int ab = uc.n * vc.n;
        std::vector<double> G(ab, 0.0);
        if (ab == 0) return G;
        gram_kernel<<<kRedCTAs, kT, 0, s>>>(U, ld, uc, V, ld, vc, n, partial);
        partial_sum_kernel<<<(ab + 127) / 128, 128, 0, s>>>(partial, kRedCTAs, ab, gout);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h_pin, gout, ab * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::memcpy(G.data(), h_pin, ab * sizeof(double));
        return G;
    }
    void combine(double* O, const Cols& oc, bool add, const double* U, const Cols& uc, const std::vector<double>& M) {
        if (oc.n == 0 || n == 0) return;
        Mat Mt;
        std::memset(&Mt, 0, sizeof(Mt));
        std::copy(M.begin(), M.end(), Mt.v);
        combine_kernel<<<grid(), kT, 0, s>>>(O, ld, oc, add ? 1 : 0, U, ld, uc, n, Mt);
        CK(cudaGetLastError());
    }
    void spmm(const double* X, const Cols& in, double* Y) {
        if (in.n == 0 || n == 0) return;
        spmm_kernel<<<grid(), kT, 0, s>>>(A->rp, A->ci, A->val, n, X, ld, in, Y, ld, in);
        CK(cudaGetLastError());
        ++spmm_count;
    }
    std::vector<double> resid(const std::vector<double>& lam, const double* dinv) {
        Vec16 L{};
        for (int j = 0; j < m; ++j) L.v[j] = lam[j];
        resid_kernel<<<kRedCTAs, kT, 0, s>>>(S, AS, ld, m, L, dinv, m, n, partial);
        CK(cudaGetLastError());
        std::vector<double> h((size_t)kRedCTAs * m);
        CK(cudaMemcpyAsync(h.data(), partial, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<double> r(m, 0.0);
        for (int p = 0; p < kRedCTAs; ++p)
            for (int j = 0; j < m; ++j) r[j] += h[(size_t)p * m + j];
        for (auto& v : r) v = std::sqrt(v);
        return r;
    }

    // Z -= B (B^T Z): classical Gram-Schmidt of block Z against the orthonormal block B
    void orth_against(const Cols& B, const Cols& Z) {
        if (B.n == 0 || Z.n == 0) return;
        std::vector<double> Y = gram(S, B, S, Z);  // B.n x Z.n
        for (auto& v : Y) v = -v;
        combine(S, Z, true, S, B, Y);
    }
    // SVQB (Stathopoulos & Wu): Z <- Z D U diag(sigma)^-1/2 on the columns whose normalised
    // Gram eigenvalue survives the drop rule (norm after orthogonalisation
    // below 1e-12 relative -> dropped).  Returns the surviving columns (a prefix of Z).
    Cols svqb(const Cols& Z) {
        const int w = Z.n;
        if (w == 0) return Z;
        std::vector<double> G = gram(S, Z, S, Z);
        double dmax = 0.0;
        for (int i = 0; i < w; ++i) dmax = std::max(dmax, G[(size_t)i * w + i]);
        std::vector<double> D(w, 0.0);
        for (int i = 0; i < w; ++i) {
            const double d = G[(size_t)i * w + i];
            if (d > 1e-300 && d > 1e-28 * dmax && std::isfinite(d)) D[i] = 1.0 / std::sqrt(d);
        }
        std::vector<double> H((size_t)w * w);
        for (int i = 0; i < w; ++i)
            for (int j = 0; j < w; ++j) H[(size_t)i * w + j] = D[i] * G[(size_t)i * w + j] * D[j];
        for (int i = 0; i < w; ++i)
            for (int j = i + 1; j < w; ++j) {
                const double h = 0.5 * (H[(size_t)i * w + j] + H[(size_t)j * w + i]);
                H[(size_t)i * w + j] = H[(size_t)j * w + i] = h;
            }
        std::vector<double> sig, U;
        sym_eig(w, H, sig, U);
        const double smax = std::max(sig.empty() ? 0.0 : sig.back(), 0.0);
        std::vector<int> keep;
        for (int j = w - 1; j >= 0; --j)  // largest first: best-conditioned directions
            if (sig[j] > 1e-24 * smax && sig[j] > 0.0) keep.push_back(j);
        const int w2 = (int)keep.size();
        std::vector<double> T((size_t)w * w2, 0.0);
        for (int i = 0; i < w; ++i)
            for (int c = 0; c < w2; ++c)
                T[(size_t)i * w2 + c] = D[i] * U[(size_t)i * w + keep[c]] / std::sqrt(sig[keep[c]]);
        Cols out = Z;
        out.n = w2;
        combine(S, out, false, S, Z, T);
        return out;
    }
    Cols orthonormalize(const Cols& B, const Cols& Z) {
        Cols z = Z;
        for (int pass = 0; pass < 2; ++pass) {
            orth_against(B, z);
            z = svqb(z);
        }
        return z;
    }

    // Rayleigh-Ritz on the orthonormal basis S_B (AS_B = A S_B): X, AX, P into Sn / ASn.
    void rayleigh_ritz(const Cols& B, const Cols& WP, std::vector<double>& lam) {
        const int q = B.n;
        std::vector<double> G = gram(S, B, AS, B);
        for (int i = 0; i < q; ++i)
            for (int j = i + 1; j < q; ++j) {
                const double h = 0.5 * (G[(size_t)i * q + j] + G[(size_t)j * q + i]);
                G[(size_t)i * q + j] = G[(size_t)j * q + i] = h;
            }
        std::vector<double> th, U;
        sym_eig(q, G, th, U);
        std::vector<double> C((size_t)q * m);
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < m; ++j) C[(size_t)i * m + j] = U[(size_t)i * q + j];
        const Cols Xc = cols_range(0, m);
        combine(Sn, Xc, false, S, B, C);
        combine(ASn, Xc, false, AS, B, C);
        if (WP.n > 0) {  // P' = S_{W,P} C_{W,P}: rows m.. of C
            std::vector<double> Cp(C.begin() + (size_t)m * m, C.end());
            combine(Sn, cols_range(2 * m, 3 * m), false, S, WP, Cp);
        }
        std::swap(S, Sn);
        std::swap(AS, ASn);
        lam.assign(th.begin(), th.begin() + m);
    }
};

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

int dense_threshold() {
    const char* e = std::getenv("SPARSLA_EIG_DENSE_THRESHOLD");
    return e ? std::max(0, std::atoi(e)) : 64;
}

void eig_smallest(DevCsr* A, int k, double tol, long long max_iter, uint64_t seed, int precond, double* V,
                  EigOut& o) {
    const long long n = A->nrows;
    const double* dinv = precond == SPARSLA_PRECOND_JACOBI ? A->jacobi_dinv() : nullptr;
    const int m = k;
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
            spmm_kernel<<<(nn + kT - 1) / kT, kT, 0, A->stream>>>(A->rp, A->ci, A->val, nn, E, nn, c, AE, nn, c);
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
    Lobpcg L(A, m);
    const Cols Xc = cols_range(0, m);
    eig_init_kernel<<<L.grid(), kT, 0, L.s>>>(L.S, n, L.ld, m, seed);
    CK(cudaGetLastError());
    Cols x0 = L.orthonormalize(Cols{}, Xc);
    if (x0.n < m) fail(SPARSLA_ERR_INTERNAL, "eig_smallest: initial block is rank deficient");
    L.spmm(L.S, Xc, L.AS);
    std::vector<double> lam;
    L.rayleigh_ritz(Xc, Cols{}, lam);
    bool have_p = false;
    long long it = 0;
    std::vector<double> res;
    for (;; ++it) {
        res = L.resid(lam, dinv);
        Cols act;
        for (int j = 0; j < m; ++j)
            if (!(res[j] <= tol)) act.c[act.n++] = (unsigned char)j;
        if (act.n == 0 || it >= max_iter) break;
        Cols Wc, Pc;
        for (int t = 0; t < act.n; ++t) {
            Wc.c[Wc.n++] = (unsigned char)(m + act.c[t]);
            if (have_p) Pc.c[Pc.n++] = (unsigned char)(2 * m + act.c[t]);
        }
        Wc = L.orthonormalize(Xc, Wc);
        const Cols XW = cols_cat(Xc, Wc);
        Pc = L.orthonormalize(XW, Pc);
        const Cols WP = cols_cat(Wc, Pc);
        L.spmm(L.S, WP, L.AS);
        L.rayleigh_ritz(cols_cat(Xc, WP), WP, lam);
        have_p = WP.n > 0;
        if (WP.n == 0) break;  // no new directions: the block cannot improve
    }
    o.iters = it;
    o.lam = lam;
    finish(L, k, tol, dinv, o, V);
    char buf[128];
    std::snprintf(buf, sizeof buf, "lobpcg: %lld iterations, block %d, %s", it, m,
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
