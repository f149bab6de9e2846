// coo_device.cu — SparseCoo canonicalization on the GPU (
// reference sparse.cpp:9-53): bounds check, stable order by (row, col), duplicates summed in
// input order, explicit zeros kept.  The reference sorts a permutation with a two-key
// comparator on one core (12.2 s at 117M entries, SURVEY probe P1); here the keys
// row * ncols + col are radix-sorted with their input positions (LSD radix sort is stable,
// so equal keys keep their input order), segment heads are flagged and scanned, and one
// thread per output entry sums its duplicates left to right — the reference's
// vals_.back() += vals[p] order, so the result is bit-identical to the host path.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "common.hpp"
#include "device.hpp"

namespace sparsla_b200 {
namespace {

#define CK(x) cuda_check((x), #x)

template <class T>
struct DBuf {  // device buffer owned for the duration of a call
    T* p = nullptr;
    explicit DBuf(size_t n) { CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~DBuf() { cudaFree(p); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
};

// first entry (in input order) outside the shape -> bad[0] (atomicMin)
__global__ void coo_bounds_kernel(const int64_t* rows, const int64_t* cols, long long nnz, int64_t nrows,
                                  int64_t ncols, unsigned long long* bad) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const int64_t r = rows[k], c = cols[k];
    if (r < 0 || r >= nrows || c < 0 || c >= ncols) atomicMin(bad, (unsigned long long)k);
}

__global__ void coo_keys_kernel(const int64_t* rows, const int64_t* cols, long long nnz, int64_t ncols,
                                unsigned long long* keys, int32_t* idx) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    keys[k] = (unsigned long long)rows[k] * (unsigned long long)ncols + (unsigned long long)cols[k];
    idx[k] = (int32_t)k;
}

__global__ void coo_heads_kernel(const unsigned long long* keys, long long nnz, int32_t* head) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    head[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

// one thread per segment head: output entry seg[k] - 1 = (row, col, sum of its duplicates
// in sorted = input order)
__global__ void coo_emit_kernel(const unsigned long long* keys, const int32_t* idx, const int32_t* seg,
                                const double* vals, long long nnz, int64_t ncols, int64_t* ro, int64_t* co,
                                double* vo) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const unsigned long long key = keys[k];
    if (k > 0 && keys[k - 1] == key) return;
    double s = vals[idx[k]];
    for (long long j = k + 1; j < nnz && keys[j] == key; ++j) s = __dadd_rn(s, vals[idx[j]]);
    const long long o = (long long)seg[k] - 1;
    ro[o] = (int64_t)(key / (unsigned long long)ncols);
    co[o] = (int64_t)(key % (unsigned long long)ncols);
    vo[o] = s;
}

// sorted position j: order[j] = input entry, group[j] = its canonical entry
__global__ void coo_perm_kernel(const int32_t* idx, const int32_t* seg, long long nnz, int64_t* order, int64_t* group) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnz) return;
    order[j] = idx[j];
    group[j] = (int64_t)seg[j] - 1;
}

// one thread per group head in sorted order: out[group[j]] = vals[order[j]] + ... left to right
// over the group's sorted positions (the reference's vals_.back() += vals[p], sparse.cpp:45-47)
__global__ void group_sum_kernel(const int64_t* order, const int64_t* group, const double* vals, long long nnz,
                                 double* out) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnz) return;
    const int64_t g = group[j];
    if (j > 0 && group[j - 1] == g) return;
    double s = vals[order[j]];
    for (long long i = j + 1; i < nnz && group[i] == g; ++i) s = __dadd_rn(s, vals[order[i]]);
    out[g] = s;
}

__global__ void csr_rows_kernel(const int32_t* rp, long long n, int32_t* rows) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) rows[k] = (int32_t)i;
}

__global__ void iota_hist_kernel(const int32_t* ci, long long nnz, int32_t* idx, int32_t* count) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    idx[k] = (int32_t)k;
    atomicAdd(count + ci[k], 1);
}

__global__ void transpose_emit_kernel(const int32_t* idx, const int32_t* rows, const double* val, long long nnz,
                                      int32_t* tci, double* tv) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnz) return;
    const int32_t k = idx[j];
    tci[j] = rows[k];
    tv[j] = val[k];
}

int key_bits(unsigned long long maxkey) {
    int b = 1;
    while (b < 64 && (maxkey >> b) != 0) ++b;
    return b;
}

}  // namespace

// Canonical A^T of a device CSR (sparse.cpp:176-182 / the reference's spmv_transpose scatter
// order): entries stably radix-sorted by column keep their row-major order, so every row of
// A^T lists its columns (A's rows) ascending.  Results land in host arrays trp[ncols+1],
// tci[nnz], tv[nnz] (the device handle of A^T is built from them).
void csr_transpose_device(int device, long long nrows, long long ncols, long long nnz, const int32_t* rp,
                          const int32_t* ci, const double* val, int32_t* trp, int32_t* tci, double* tv) {
    DeviceGuard g(device);
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{s};
    const size_t n = (size_t)std::max<long long>(nnz, 1);
    DBuf<int32_t> rows(n), cnt((size_t)ncols + 1), k0(n), k1(n), i0(n), i1(n), otc(n), orp((size_t)ncols + 1);
    DBuf<double> otv(n);
    CK(cudaMemsetAsync(cnt.p, 0, ((size_t)ncols + 1) * 4, s));
    if (nrows > 0) csr_rows_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(rp, nrows, rows.p);
    if (nnz > 0) {
        iota_hist_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(ci, nnz, i0.p, cnt.p);
        CK(cudaMemcpyAsync(k0.p, ci, (size_t)nnz * 4, cudaMemcpyDeviceToDevice, s));
        const int bits = key_bits((unsigned long long)std::max<long long>(ncols, 1));
        cub::DoubleBuffer<int32_t> kb(k0.p, k1.p), ib(i0.p, i1.p);
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, ib, (int)nnz, 0, bits, s));
        DBuf<unsigned char> tmp(tb);
        CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kb, ib, (int)nnz, 0, bits, s));
        transpose_emit_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(ib.Current(), rows.p, val, nnz, otc.p,
                                                                           otv.p);
    }
    CK(cudaGetLastError());
    size_t sb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, cnt.p, orp.p, (int)(ncols + 1), s));
    DBuf<unsigned char> stmp(sb);
    CK(cub::DeviceScan::ExclusiveSum(stmp.p, sb, cnt.p, orp.p, (int)(ncols + 1), s));
    CK(cudaMemcpyAsync(trp, orp.p, ((size_t)ncols + 1) * 4, cudaMemcpyDeviceToHost, s));
    if (nnz > 0) {
        CK(cudaMemcpyAsync(tci, otc.p, (size_t)nnz * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(tv, otv.p, (size_t)nnz * 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
}

}  // namespace sparsla_b200

using namespace sparsla_b200;

namespace {
// Shared by both entry points: vals == nullptr -> permutation outputs (order, group) instead
// of the canonical COO.
int coo_device_impl(int device, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows, const int64_t* cols,
                    const double* vals, int32_t mem, int64_t* out_nnz, int64_t* rows_out, int64_t* cols_out,
                    double* vals_out, int64_t* order, int64_t* group) {
    return guarded([&] {
        if (nrows < 0 || ncols < 0) fail(SPARSLA_ERR_DIMENSION, "negative matrix shape");
        if (nnz < 0) fail(SPARSLA_ERR_DIMENSION, "negative nnz");
        if (nnz >= (1LL << 31)) fail(SPARSLA_ERR_UNSUPPORTED, "device canonicalization: nnz must be < 2^31");
        if (mem != SPARSLA_MEM_HOST && mem != SPARSLA_MEM_DEVICE) fail(SPARSLA_ERR_INVALID_ARGUMENT, "bad mem");
        if (!out_nnz) fail(SPARSLA_ERR_INVALID_ARGUMENT, "out_nnz is null");
        if (nrows > 0 && ncols > 0 && (unsigned long long)nrows > ~0ULL / (unsigned long long)ncols)
            fail(SPARSLA_ERR_UNSUPPORTED, "device canonicalization: nrows * ncols must fit 64 bits");
        DeviceGuard g(device);
        *out_nnz = 0;
        if (nnz == 0) return;
        cudaStream_t s = nullptr;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{s};
        const size_t n = (size_t)nnz;
        const unsigned grid = (unsigned)((nnz + 255) / 256);
        // inputs on the device
        const int64_t *dr = rows, *dc = cols;
        const double* dv = vals;
        DBuf<int64_t> hr(mem == SPARSLA_MEM_HOST ? n : 0), hc(mem == SPARSLA_MEM_HOST ? n : 0);
        DBuf<double> hv(mem == SPARSLA_MEM_HOST && vals ? n : 0);
        if (mem == SPARSLA_MEM_HOST) {
            CK(cudaMemcpyAsync(hr.p, rows, n * 8, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(hc.p, cols, n * 8, cudaMemcpyHostToDevice, s));
            if (vals) CK(cudaMemcpyAsync(hv.p, vals, n * 8, cudaMemcpyHostToDevice, s));
            dr = hr.p; dc = hc.p; dv = vals ? hv.p : nullptr;
        }
        // bounds (the first offending entry in input order, as the host path reports it)
        DBuf<unsigned long long> bad(1);
        const unsigned long long none = ~0ULL;
        CK(cudaMemcpyAsync(bad.p, &none, 8, cudaMemcpyHostToDevice, s));
        coo_bounds_kernel<<<grid, 256, 0, s>>>(dr, dc, nnz, nrows, ncols, bad.p);
        CK(cudaGetLastError());
        unsigned long long hb = 0;
        CK(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hb != none) {
            int64_t r = 0, c = 0;
            CK(cudaMemcpy(&r, dr + hb, 8, mem == SPARSLA_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDefault));
            CK(cudaMemcpy(&c, dc + hb, 8, mem == SPARSLA_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDefault));
            fail(SPARSLA_ERR_BOUNDS, "coo index (" + std::to_string(r) + ", " + std::to_string(c) + ") outside shape (" +
                                         std::to_string(nrows) + ", " + std::to_string(ncols) + ") at entry " +
                                         std::to_string(hb));
        }
        // stable radix sort of (key, input position)
        DBuf<unsigned long long> k0(n), k1(n);
        DBuf<int32_t> i0(n), i1(n);
        coo_keys_kernel<<<grid, 256, 0, s>>>(dr, dc, nnz, ncols, k0.p, i0.p);
        CK(cudaGetLastError());
        const int bits = key_bits((unsigned long long)(nrows > 0 ? nrows : 1) * (unsigned long long)(ncols > 0 ? ncols : 1));
        cub::DoubleBuffer<unsigned long long> kb(k0.p, k1.p);
        cub::DoubleBuffer<int32_t> ib(i0.p, i1.p);
        size_t tmp_bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, ib, (int)nnz, 0, bits, s));
        DBuf<unsigned char> tmp(tmp_bytes);
        CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kb, ib, (int)nnz, 0, bits, s));
        // segment heads -> output positions
        DBuf<int32_t> head(n), seg(n);
        coo_heads_kernel<<<grid, 256, 0, s>>>(kb.Current(), nnz, head.p);
        CK(cudaGetLastError());
        size_t scan_bytes = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, head.p, seg.p, (int)nnz, s));
        DBuf<unsigned char> stmp(scan_bytes);
        CK(cub::DeviceScan::InclusiveSum(stmp.p, scan_bytes, head.p, seg.p, (int)nnz, s));
        int32_t nout = 0;
        CK(cudaMemcpyAsync(&nout, seg.p + (n - 1), 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (!vals) {  // permutation outputs
            int64_t *oo = order, *og = group;
            DBuf<int64_t> to(mem == SPARSLA_MEM_HOST ? n : 0), tg(mem == SPARSLA_MEM_HOST ? n : 0);
            if (mem == SPARSLA_MEM_HOST) { oo = to.p; og = tg.p; }
            coo_perm_kernel<<<grid, 256, 0, s>>>(ib.Current(), seg.p, nnz, oo, og);
            CK(cudaGetLastError());
            if (mem == SPARSLA_MEM_HOST) {
                CK(cudaMemcpyAsync(order, to.p, n * 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemcpyAsync(group, tg.p, n * 8, cudaMemcpyDeviceToHost, s));
            }
            CK(cudaStreamSynchronize(s));
            *out_nnz = nout;
            return;
        }
        // outputs
        int64_t *orr = rows_out, *occ = cols_out;
        double* ovv = vals_out;
        DBuf<int64_t> tr(mem == SPARSLA_MEM_HOST ? (size_t)nout : 0), tc(mem == SPARSLA_MEM_HOST ? (size_t)nout : 0);
        DBuf<double> tv(mem == SPARSLA_MEM_HOST ? (size_t)nout : 0);
        if (mem == SPARSLA_MEM_HOST) { orr = tr.p; occ = tc.p; ovv = tv.p; }
        coo_emit_kernel<<<grid, 256, 0, s>>>(kb.Current(), ib.Current(), seg.p, dv, nnz, ncols, orr, occ, ovv);
        CK(cudaGetLastError());
        if (mem == SPARSLA_MEM_HOST) {
            CK(cudaMemcpyAsync(rows_out, tr.p, (size_t)nout * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(cols_out, tc.p, (size_t)nout * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(vals_out, tv.p, (size_t)nout * 8, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        *out_nnz = nout;
    });
}
}  // namespace

extern "C" int sparsla_coo_canonicalize_device(int device, int64_t nrows, int64_t ncols, int64_t nnz,
                                               const int64_t* rows, const int64_t* cols, const double* vals,
                                               int32_t mem, int64_t* out_nnz, int64_t* rows_out,
                                               int64_t* cols_out, double* vals_out) {
    if (!vals && nnz > 0) {
        set_last_error("vals is null");
        return SPARSLA_ERR_INVALID_ARGUMENT;
    }
    static const double dummy = 0.0;
    return coo_device_impl(device, nrows, ncols, nnz, rows, cols, nnz > 0 ? vals : &dummy, mem, out_nnz, rows_out,
                           cols_out, vals_out, nullptr, nullptr);
}

extern "C" int sparsla_coo_sort_device(int device, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                                       const int64_t* cols, int32_t mem, int64_t* out_nnz, int64_t* order,
                                       int64_t* group) {
    if (nnz > 0 && (!order || !group)) {
        set_last_error("order / group is null");
        return SPARSLA_ERR_INVALID_ARGUMENT;
    }
    return coo_device_impl(device, nrows, ncols, nnz, rows, cols, nullptr, mem, out_nnz, nullptr, nullptr, nullptr,
                           order, group);
}

// Values of a canonicalised pattern from new input-order values (the with_values step of a
// differentiable SparseCoo whose triplets carry duplicates): device arrays order[nnz],
// group[nnz] from sparsla_coo_sort_device, vals[nnz] in input order -> vals_out[nout].
extern "C" int sparsla_coo_group_sum_device(int device, int64_t nnz, int64_t nout, const int64_t* order,
                                            const int64_t* group, const double* vals, double* vals_out) {
    return guarded([&] {
        if (nnz < 0 || nout < 0 || nout > nnz) fail(SPARSLA_ERR_DIMENSION, "bad nnz / nout");
        if (nnz >= (1LL << 31)) fail(SPARSLA_ERR_UNSUPPORTED, "group sum: nnz must be < 2^31");
        if (nnz > 0 && (!order || !group || !vals || !vals_out)) fail(SPARSLA_ERR_INVALID_ARGUMENT, "null pointer");
        if (nnz == 0) return;
        DeviceGuard g(device);
        cudaStream_t s = nullptr;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{s};
        group_sum_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(order, group, vals, nnz, vals_out);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
    });
}
