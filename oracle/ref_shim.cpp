// ref_shim.cpp — C ABI over the REFERENCE's own sparse core, for parity pinning.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with
// /root/reference/proj/core/src/sparse.cpp (read in place, never copied) under
// -Dsparsla=sparsla_ref into oracle/_ref/libsparsla_ref.so.  Each function below calls
// exactly one reference entry point:
//   ref_coo_canonicalize -> SparseCoo::SparseCoo           sparse.cpp:9-53
//   ref_csr_from_coo     -> CsrMatrix::from_coo            sparse.cpp:94-116
//   ref_spmv             -> spmv                           sparse.cpp:135-154
//   ref_spmv_transpose   -> spmv_transpose                 sparse.cpp:156-174
//   ref_transpose        -> transpose                      sparse.cpp:176-182
//   ref_is_struct_sym    -> is_structurally_symmetric      sparse.cpp:184-192
//   ref_is_symmetric     -> is_symmetric                   sparse.cpp:194-205
//   ref_find             -> SparseCoo::find                sparse.cpp:68-79
//   ref_bytes            -> CsrMatrix::bytes               sparse.cpp:129-133
// Errors are mapped to the status codes of include/sparsla_c.h.
#include "sparsla/errors.hpp"
#include "sparsla/sparse.hpp"

#include <cstdint>
#include <cstring>
#include <vector>

using namespace sparsla;  // renamed to sparsla_ref by the Makefile

namespace {
thread_local std::string g_msg;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const DimensionError& e) { g_msg = e.what(); return 1; }
    catch (const BoundsError& e) { g_msg = e.what(); return 2; }
    catch (const FormatError& e) { g_msg = e.what(); return 3; }
    catch (const SingularMatrixError& e) { g_msg = e.what(); return 4; }
    catch (const UnsupportedInputError& e) { g_msg = e.what(); return 5; }
    catch (const InvalidArgumentError& e) { g_msg = e.what(); return 6; }
    catch (const TransportError& e) { g_msg = e.what(); return 7; }
    catch (const std::exception& e) { g_msg = e.what(); return 11; }
}

SparseCoo make_coo(int64_t nr, int64_t nc, int64_t nnz, const int64_t* r, const int64_t* c,
                   const double* v) {
    return SparseCoo(std::vector<index_t>(r, r + nnz), std::vector<index_t>(c, c + nnz),
                     std::vector<double>(v, v + nnz), Shape{nr, nc});
}

CsrMatrix make_csr(int64_t nr, int64_t nc, const int64_t* rp, const int64_t* ci, const double* v) {
    const int64_t nnz = rp[nr];
    std::vector<index_t> rows(static_cast<size_t>(nnz));
    for (int64_t i = 0; i < nr; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) rows[static_cast<size_t>(k)] = i;
    SparseCoo coo(std::move(rows), std::vector<index_t>(ci, ci + nnz),
                  std::vector<double>(v, v + nnz), Shape{nr, nc});
    return CsrMatrix::from_coo(coo);
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

int ref_coo_canonicalize(int64_t nr, int64_t nc, int64_t nnz, const int64_t* r, const int64_t* c,
                         const double* v, int64_t* out_nnz, int64_t* ro, int64_t* co, double* vo) {
    return guard([&] {
        SparseCoo a = make_coo(nr, nc, nnz, r, c, v);
        *out_nnz = a.nnz();
        std::memcpy(ro, a.rows().data(), sizeof(int64_t) * a.nnz());
        std::memcpy(co, a.cols().data(), sizeof(int64_t) * a.nnz());
        std::memcpy(vo, a.vals().data(), sizeof(double) * a.nnz());
    });
}

int ref_csr_from_coo(int64_t nr, int64_t nc, int64_t nnz, const int64_t* r, const int64_t* c,
                     const double* v, int64_t* rp, int64_t* ci, double* vo, int64_t* bytes) {
    return guard([&] {
        CsrMatrix m = CsrMatrix::from_coo(make_coo(nr, nc, nnz, r, c, v));
        std::memcpy(rp, m.row_ptr().data(), sizeof(int64_t) * (nr + 1));
        std::memcpy(ci, m.col_idx().data(), sizeof(int64_t) * m.nnz());
        std::memcpy(vo, m.vals().data(), sizeof(double) * m.nnz());
        *bytes = m.bytes();
    });
}

int ref_spmv(int64_t nr, int64_t nc, const int64_t* rp, const int64_t* ci, const double* v,
             int64_t nx, const double* x, double* y) {
    return guard([&] {
        CsrMatrix m = make_csr(nr, nc, rp, ci, v);
        std::vector<double> out = spmv(m, std::span<const double>(x, static_cast<size_t>(nx)));
        std::memcpy(y, out.data(), sizeof(double) * out.size());
    });
}

int ref_spmv_transpose(int64_t nr, int64_t nc, const int64_t* rp, const int64_t* ci,
                       const double* v, int64_t nx, const double* x, double* y) {
    return guard([&] {
        CsrMatrix m = make_csr(nr, nc, rp, ci, v);
        std::vector<double> out =
            spmv_transpose(m, std::span<const double>(x, static_cast<size_t>(nx)));
        std::memcpy(y, out.data(), sizeof(double) * out.size());
    });
}

int ref_transpose(int64_t nr, int64_t nc, int64_t nnz, const int64_t* r, const int64_t* c,
                  const double* v, int64_t* ro, int64_t* co, double* vo) {
    return guard([&] {
        SparseCoo t = transpose(make_coo(nr, nc, nnz, r, c, v));
        std::memcpy(ro, t.rows().data(), sizeof(int64_t) * t.nnz());
        std::memcpy(co, t.cols().data(), sizeof(int64_t) * t.nnz());
        std::memcpy(vo, t.vals().data(), sizeof(double) * t.nnz());
    });
}

int ref_is_struct_sym(int64_t nr, int64_t nc, int64_t nnz, const int64_t* r, const int64_t* c,
                      const double* v, int32_t* out) {
    return guard([&] { *out = is_structurally_symmetric(make_coo(nr, nc, nnz, r, c, v)) ? 1 : 0; });
}

int ref_is_symmetric(int64_t nr, int64_t nc, int64_t nnz, const int64_t* r, const int64_t* c,
                     const double* v, double tol, int32_t* out) {
    return guard([&] { *out = is_symmetric(make_coo(nr, nc, nnz, r, c, v), tol) ? 1 : 0; });
}

int ref_find(int64_t nr, int64_t nc, int64_t nnz, const int64_t* r, const int64_t* c,
             const double* v, int64_t i, int64_t j, int64_t* out) {
    return guard([&] { *out = make_coo(nr, nc, nnz, r, c, v).find(i, j); });
}

}  // extern "C"
