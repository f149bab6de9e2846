// sparsla/matrix_market.hpp — drop-in for the reference's declared Matrix Market interface
// (proj/core/include/sparsla/matrix_market.hpp:10-20).
#pragma once

#include <iomanip>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <string>

#include "sparsla/sparse.hpp"

namespace sparsla {

namespace detail {
inline SparseCoo adopt_coo(sparsla_coo* h) {
    std::int64_t nr = 0, nc = 0, nz = 0;
    detail::check(sparsla_coo_sizes(h, &nr, &nc, &nz));
    std::vector<index_t> r(static_cast<std::size_t>(nz)), c(static_cast<std::size_t>(nz));
    std::vector<double> v(static_cast<std::size_t>(nz));
    const int rc = sparsla_coo_get(h, r.data(), c.data(), v.data());
    sparsla_coo_destroy(h);
    detail::check(rc);
    return SparseCoo::adopt(std::move(r), std::move(c), std::move(v), Shape{nr, nc});
}
}  // namespace detail

inline SparseCoo read_matrix_market(const std::string& path) {
    sparsla_coo* h = nullptr;
    detail::check(sparsla_mtx_read(path.c_str(), &h));
    return detail::adopt_coo(h);
}

inline SparseCoo read_matrix_market(std::istream& in) {
    std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    sparsla_coo* h = nullptr;
    detail::check(sparsla_mtx_read_buffer(data.data(), static_cast<std::int64_t>(data.size()), &h));
    return detail::adopt_coo(h);
}

inline void write_matrix_market(const SparseCoo& a, const std::string& path) {
    detail::check(sparsla_mtx_write(path.c_str(), a.nrows(), a.ncols(), a.nnz(), a.rows().data(), a.cols().data(),
                                    a.vals().data()));
}

inline void write_matrix_market(const SparseCoo& a, std::ostream& out) {
    out << "%%MatrixMarket matrix coordinate real general\n" << a.nrows() << ' ' << a.ncols() << ' ' << a.nnz() << '\n';
    out << std::setprecision(17);
    for (index_t k = 0; k < a.nnz(); ++k) out << a.rows()[k] + 1 << ' ' << a.cols()[k] + 1 << ' ' << a.vals()[k] << '\n';
}

}  // namespace sparsla
