// matrix_market.cpp — Matrix Market coordinate I/O (host), the ingestion side of the path.
//
// Restates the reference's declared interface (proj/core/include/sparsla/matrix_market.hpp:
// 10-20; contract SPEC.md:92-100, 106, 115): "%%MatrixMarket matrix coordinate real
// general|symmetric", '%' comment lines, 1-based indices converted to 0-based, symmetric
// files expanded to full storage, result canonicalised like SparseCoo (duplicates summed in
// file order); malformed input raises FormatError carrying the 1-based line number.  The
// writer emits coordinate/real/general with 17 significant digits, so read(write(A)) == A
// bit for bit.
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "common.hpp"

using namespace sparsla_b200;

struct sparsla_coo {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> rows, cols;
    std::vector<double> vals;
};

namespace {

[[noreturn]] void format_error(const std::string& msg, long line) {
    fail(SPARSLA_ERR_FORMAT, line > 0 ? msg + " (line " + std::to_string(line) + ")" : msg);
}

std::string lower(std::string s) {
    for (char& c : s) c = (char)std::tolower((unsigned char)c);
    return s;
}

sparsla_coo* parse(std::istream& in) {
    std::string line;
    long ln = 0;
    if (!std::getline(in, line)) format_error("empty Matrix Market input", 1);
    ++ln;
    std::istringstream hs(line);
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket") format_error("missing %%MatrixMarket header", ln);
    object = lower(object); format = lower(format); field = lower(field); symmetry = lower(symmetry);
    if (object != "matrix") format_error("unsupported Matrix Market object '" + object + "'", ln);
    if (format != "coordinate") format_error("non-coordinate Matrix Market format '" + format + "'", ln);
    if (field != "real" && field != "integer" && field != "double")
        format_error("unsupported Matrix Market field '" + field + "' (real only)", ln);
    const bool sym = symmetry == "symmetric";
    if (!sym && symmetry != "general")
        format_error("unsupported Matrix Market symmetry '" + symmetry + "'", ln);
    // size line (after comments / blank lines)
    int64_t M = -1, N = -1, L = -1;
    while (std::getline(in, line)) {
        ++ln;
        size_t p = line.find_first_not_of(" \t\r");
        if (p == std::string::npos || line[p] == '%') continue;
        std::istringstream ss(line);
        if (!(ss >> M >> N >> L) || M < 0 || N < 0 || L < 0) format_error("malformed size line", ln);
        break;
    }
    if (L < 0) format_error("missing size line", ln);
    auto* out = new sparsla_coo;
    std::unique_ptr<sparsla_coo> guard(out);
    std::vector<int64_t> r, c;
    std::vector<double> v;
    r.reserve((size_t)(sym ? 2 * L : L));
    c.reserve(r.capacity());
    v.reserve(r.capacity());
    int64_t got = 0;
    while (got < L && std::getline(in, line)) {
        ++ln;
        const char* s = line.c_str();
        while (*s == ' ' || *s == '\t') ++s;
        if (*s == '\0' || *s == '\r' || *s == '%') continue;
        char* e = nullptr;
        errno = 0;
        const long long i = std::strtoll(s, &e, 10);
        if (e == s) format_error("malformed entry (row index)", ln);
        s = e;
        const long long j = std::strtoll(s, &e, 10);
        if (e == s) format_error("malformed entry (column index)", ln);
        s = e;
        const double x = std::strtod(s, &e);
        if (e == s || errno == ERANGE) format_error("malformed entry (value)", ln);
        while (*e == ' ' || *e == '\t' || *e == '\r') ++e;
        if (*e != '\0') format_error("trailing characters after entry", ln);
        if (i < 1 || i > M || j < 1 || j > N) format_error("entry index outside the declared size", ln);
        r.push_back(i - 1); c.push_back(j - 1); v.push_back(x);
        if (sym && i != j) { r.push_back(j - 1); c.push_back(i - 1); v.push_back(x); }
        ++got;
    }
    if (got < L) format_error("expected " + std::to_string(L) + " entries, found " + std::to_string(got), ln);
    out->nrows = M;
    out->ncols = N;
    out->rows.resize(r.size()); out->cols.resize(r.size()); out->vals.resize(r.size());
    const int64_t m = canonicalize_coo(M, N, (int64_t)r.size(), r.data(), c.data(), v.data(), out->rows.data(),
                                       out->cols.data(), out->vals.data());
    out->rows.resize(m); out->cols.resize(m); out->vals.resize(m);
    return guard.release();
}

}  // namespace

extern "C" {

int sparsla_mtx_read(const char* path, sparsla_coo** out) {
    return guarded([&] {
        std::ifstream f(path);
        if (!f) fail(SPARSLA_ERR_FORMAT, std::string("cannot open Matrix Market file ") + path);
        *out = parse(f);
    });
}

int sparsla_mtx_read_buffer(const char* data, int64_t len, sparsla_coo** out) {
    return guarded([&] {
        std::istringstream s(std::string(data, (size_t)len));
        *out = parse(s);
    });
}

int sparsla_coo_sizes(const sparsla_coo* h, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
    return guarded([&] {
        *nrows = h->nrows;
        *ncols = h->ncols;
        *nnz = (int64_t)h->vals.size();
    });
}

int sparsla_coo_get(const sparsla_coo* h, int64_t* rows, int64_t* cols, double* vals) {
    return guarded([&] {
        std::memcpy(rows, h->rows.data(), h->rows.size() * 8);
        std::memcpy(cols, h->cols.data(), h->cols.size() * 8);
        std::memcpy(vals, h->vals.data(), h->vals.size() * 8);
    });
}

int sparsla_coo_destroy(sparsla_coo* h) {
    delete h;
    return SPARSLA_OK;
}

int sparsla_mtx_write(const char* path, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                      const int64_t* cols, const double* vals) {
    return guarded([&] {
        FILE* f = std::fopen(path, "w");
        if (!f) fail(SPARSLA_ERR_FORMAT, std::string("cannot write Matrix Market file ") + path);
        std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
        std::fprintf(f, "%lld %lld %lld\n", (long long)nrows, (long long)ncols, (long long)nnz);
        for (int64_t k = 0; k < nnz; ++k)
            std::fprintf(f, "%lld %lld %.17g\n", (long long)rows[k] + 1, (long long)cols[k] + 1, vals[k]);
        if (std::fclose(f) != 0) fail(SPARSLA_ERR_FORMAT, std::string("write failed: ") + path);
    });
}

}  // extern "C"
