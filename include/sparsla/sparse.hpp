// sparsla/sparse.hpp — drop-in for the reference's sparse core
// (proj/core/include/sparsla/sparse.hpp:18-149): same types, members and free functions;
// canonicalization / CSR assembly run on the host (libsparsla_b200 C ABI), spmv and
// spmv_transpose run on the GPU (bit-identical to the reference's row-ordered sums).
// Header-only over include/sparsla_c.h; link with -lsparsla_b200.
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <memory>
#include <mutex>
#include <span>
#include <vector>

#include "sparsla/errors.hpp"

namespace sparsla {

using index_t = std::int64_t;

struct Shape {
    index_t rows = 0;
    index_t cols = 0;
    bool operator==(const Shape&) const = default;
};

class DenseMatrix;
inline constexpr index_t kDenseElementCap = index_t{1} << 24;

class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(index_t rows, index_t cols) : data_(static_cast<std::size_t>(rows * cols), 0.0), shape_{rows, cols} {}
    Shape shape() const { return shape_; }
    index_t nrows() const { return shape_.rows; }
    index_t ncols() const { return shape_.cols; }
    double operator()(index_t i, index_t j) const { return data_[static_cast<std::size_t>(i * shape_.cols + j)]; }
    double& operator()(index_t i, index_t j) { return data_[static_cast<std::size_t>(i * shape_.cols + j)]; }
    std::span<const double> data() const { return data_; }
private:
    std::vector<double> data_;
    Shape shape_;
};

class SparseCoo {
public:
    SparseCoo() = default;
    /// Canonicalizing constructor (sort by (row, col), duplicates summed in input order).
    SparseCoo(std::vector<index_t> rows, std::vector<index_t> cols, std::vector<double> vals, Shape shape)
        : shape_(shape) {
        if (rows.size() != cols.size() || rows.size() != vals.size())
            throw DimensionError("coo arrays must have equal length: rows=" + std::to_string(rows.size()) +
                                 " cols=" + std::to_string(cols.size()) + " vals=" + std::to_string(vals.size()));
        if (shape.rows < 0 || shape.cols < 0) throw DimensionError("negative matrix shape");
        const auto n = rows.size();
        rows_.resize(n); cols_.resize(n); vals_.resize(n);
        std::int64_t m = 0;
        detail::check(sparsla_coo_canonicalize(shape.rows, shape.cols, static_cast<std::int64_t>(n), rows.data(),
                                               cols.data(), vals.data(), &m, rows_.data(), cols_.data(), vals_.data()));
        rows_.resize(static_cast<std::size_t>(m)); cols_.resize(static_cast<std::size_t>(m)); vals_.resize(static_cast<std::size_t>(m));
    }
    Shape shape() const { return shape_; }
    index_t nrows() const { return shape_.rows; }
    index_t ncols() const { return shape_.cols; }
    index_t nnz() const { return static_cast<index_t>(vals_.size()); }
    std::span<const index_t> rows() const { return rows_; }
    std::span<const index_t> cols() const { return cols_; }
    std::span<const double> vals() const { return vals_; }
    SparseCoo with_values(std::span<const double> vals) const {
        if (static_cast<index_t>(vals.size()) != nnz())
            throw DimensionError("with_values: expected " + std::to_string(nnz()) + " values, got " + std::to_string(vals.size()));
        SparseCoo out;
        out.rows_ = rows_; out.cols_ = cols_; out.vals_.assign(vals.begin(), vals.end()); out.shape_ = shape_;
        return out;
    }
    index_t find(index_t i, index_t j) const {
        auto lo = std::lower_bound(rows_.begin(), rows_.end(), i);
        auto hi = std::upper_bound(lo, rows_.end(), i);
        auto c = std::lower_bound(cols_.begin() + (lo - rows_.begin()), cols_.begin() + (hi - rows_.begin()), j);
        if (c != cols_.begin() + (hi - rows_.begin()) && *c == j) return static_cast<index_t>(c - cols_.begin());
        return -1;
    }
    DenseMatrix to_dense(index_t cap = kDenseElementCap) const {
        if (shape_.rows * shape_.cols > cap)
            throw BoundsError("to_dense: " + std::to_string(shape_.rows) + "x" + std::to_string(shape_.cols) +
                              " exceeds dense element cap " + std::to_string(cap));
        DenseMatrix d(shape_.rows, shape_.cols);
        for (index_t k = 0; k < nnz(); ++k) d(rows_[k], cols_[k]) = vals_[k];
        return d;
    }
    // already-canonical arrays (internal)
    static SparseCoo adopt(std::vector<index_t> r, std::vector<index_t> c, std::vector<double> v, Shape s) {
        SparseCoo out;
        out.rows_ = std::move(r); out.cols_ = std::move(c); out.vals_ = std::move(v); out.shape_ = s;
        return out;
    }
private:
    std::vector<index_t> rows_, cols_;
    std::vector<double> vals_;
    Shape shape_;
};

/// CSR; the device copy (int32 indices, fp64 values) is created on first GPU use.
class CsrMatrix {
public:
    CsrMatrix() = default;
    static CsrMatrix from_coo(const SparseCoo& coo) {
        CsrMatrix m;
        m.shape_ = coo.shape();
        m.row_ptr_.resize(static_cast<std::size_t>(coo.nrows() + 1));
        m.col_idx_.resize(static_cast<std::size_t>(coo.nnz()));
        m.vals_.resize(static_cast<std::size_t>(coo.nnz()));
        detail::check(sparsla_csr_from_coo(coo.nrows(), coo.ncols(), coo.nnz(), coo.rows().data(), coo.cols().data(),
                                           coo.vals().data(), m.row_ptr_.data(), m.col_idx_.data(), m.vals_.data()));
        return m;
    }
    SparseCoo to_coo() const {
        std::vector<index_t> rows(static_cast<std::size_t>(nnz()));
        detail::check(sparsla_csr_to_coo_rows(nrows(), row_ptr_.data(), rows.data()));
        return SparseCoo::adopt(std::move(rows), col_idx_, vals_, shape_);
    }
    Shape shape() const { return shape_; }
    index_t nrows() const { return shape_.rows; }
    index_t ncols() const { return shape_.cols; }
    index_t nnz() const { return static_cast<index_t>(vals_.size()); }
    std::span<const index_t> row_ptr() const { return row_ptr_; }
    std::span<const index_t> col_idx() const { return col_idx_; }
    std::span<const double> vals() const { return vals_; }
    std::int64_t bytes() const {
        return static_cast<std::int64_t>(row_ptr_.size() * sizeof(index_t) + col_idx_.size() * sizeof(index_t) +
                                         vals_.size() * sizeof(double));
    }
    /// Device handle on GPU `device` (lazily uploaded once; thread-safe).
    sparsla_dcsr* device_handle(int device = 0) const {
        std::call_once(dev_->once, [&] {
            sparsla_dcsr* h = nullptr;
            detail::check(sparsla_dcsr_create(device, nrows(), ncols(), row_ptr_.data(), col_idx_.data(), vals_.data(), &h));
            dev_->h.reset(h, [](sparsla_dcsr* p) { sparsla_dcsr_destroy(p); });
        });
        return dev_->h.get();
    }
private:
    struct Dev { std::once_flag once; std::shared_ptr<sparsla_dcsr> h; };
    std::vector<index_t> row_ptr_{0}, col_idx_;
    std::vector<double> vals_;
    Shape shape_;
    std::shared_ptr<Dev> dev_ = std::make_shared<Dev>();
};

inline std::vector<double> spmv(const CsrMatrix& a, std::span<const double> x) {
    if (static_cast<index_t>(x.size()) != a.ncols())
        throw DimensionError("spmv: x has length " + std::to_string(x.size()) + ", expected " + std::to_string(a.ncols()));
    std::vector<double> y(static_cast<std::size_t>(a.nrows()));
    detail::check(sparsla_spmv(a.device_handle(), x.data(), y.data(), SPARSLA_MEM_HOST));
    return y;
}

inline std::vector<double> spmv_transpose(const CsrMatrix& a, std::span<const double> x) {
    if (static_cast<index_t>(x.size()) != a.nrows())
        throw DimensionError("spmv_transpose: x has length " + std::to_string(x.size()) + ", expected " +
                             std::to_string(a.nrows()));
    std::vector<double> y(static_cast<std::size_t>(a.ncols()));
    detail::check(sparsla_spmv_transpose(a.device_handle(), x.data(), y.data(), SPARSLA_MEM_HOST));
    return y;
}

inline SparseCoo transpose(const SparseCoo& a) {
    std::vector<index_t> r(a.cols().begin(), a.cols().end()), c(a.rows().begin(), a.rows().end());
    std::vector<double> v(a.vals().begin(), a.vals().end());
    return SparseCoo(std::move(r), std::move(c), std::move(v), Shape{a.ncols(), a.nrows()});
}

inline bool is_structurally_symmetric(const SparseCoo& a) {
    CsrMatrix m = CsrMatrix::from_coo(a);
    std::int32_t s1 = 0, s2 = 0;
    detail::check(sparsla_csr_symmetry(m.nrows(), m.ncols(), m.row_ptr().data(), m.col_idx().data(), m.vals().data(),
                                       0.0, &s1, &s2));
    return s1 != 0;
}

inline bool is_symmetric(const SparseCoo& a, double tol = 1e-12) {
    CsrMatrix m = CsrMatrix::from_coo(a);
    std::int32_t s1 = 0, s2 = 0;
    detail::check(sparsla_csr_symmetry(m.nrows(), m.ncols(), m.row_ptr().data(), m.col_idx().data(), m.vals().data(),
                                       tol, &s1, &s2));
    return s2 != 0;
}

}  // namespace sparsla
