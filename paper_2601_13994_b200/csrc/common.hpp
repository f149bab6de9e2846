// common.hpp — error model and host threading helpers of libsparsla_b200.
//
// Errors: every C ABI entry point runs inside guarded(); internal code throws
// sparsla_b200::Error carrying a sparsla_status code (one per exception class of the
// reference's errors.hpp:9-62) and the message is kept per thread for
// sparsla_last_error_message().
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sparsla_c.h"

namespace sparsla_b200 {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(const std::string& msg);

template <class F>
int guarded(F&& f) noexcept {
    try {
        f();
        return SPARSLA_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return SPARSLA_ERR_INTERNAL;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SPARSLA_ERR_INTERNAL;
    }
}

int host_threads();

// Static block partition over [0, n) on host threads.  Each index is handled by exactly
// one thread, so any per-index computation is independent of the thread count.
template <class F>
void parallel_for(int64_t n, F&& f, int64_t grain = 1 << 14) {
    int nt = host_threads();
    if (nt <= 1 || n < 2 * grain) {
        if (n > 0) f(int64_t{0}, n);
        return;
    }
    int64_t want = (n + grain - 1) / grain;
    if (want < nt) nt = static_cast<int>(want);
    const int64_t per = (n + nt - 1) / nt;
    std::vector<std::thread> th;
    th.reserve(static_cast<size_t>(nt));
    for (int t = 0; t < nt; ++t) {
        const int64_t b = t * per, e = b + per < n ? b + per : n;
        if (b >= e) break;
        th.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& t : th) t.join();
}

// ---- host sparse core (host_sparse.cpp) ----
int64_t canonicalize_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                         const int64_t* cols, const double* vals, int64_t* ro, int64_t* co,
                         double* vo);
void csr_transpose_host(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                        const double* v, int64_t* trp, int64_t* tci, double* tv);
template <class I>
void validate_csr(int64_t nrows, int64_t ncols, const I* rp, const I* ci);

}  // namespace sparsla_b200

// build_local result (host, SPEC.md:433-436 layout)
struct sparsla_local {
    std::vector<int64_t> owned, halo;
    std::vector<int32_t> neighbors;
    std::vector<int64_t> send_ptr, send_idx, recv_ptr, recv_idx, rp, ci;
    std::vector<double> v;
};
