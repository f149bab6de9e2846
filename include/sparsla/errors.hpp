// sparsla/errors.hpp — exception hierarchy of the drop-in API.
// Same classes and bases as the reference (proj/core/include/sparsla/errors.hpp:9-62); the
// C ABI status codes (sparsla_c.h) map 1:1 onto them in sparsla::detail::check().
#pragma once

#include <stdexcept>
#include <string>

#include "sparsla_c.h"

namespace sparsla {

class Error : public std::runtime_error {
public:
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class DimensionError : public Error { public: using Error::Error; };
class BoundsError : public Error { public: using Error::Error; };
class FormatError : public Error {
public:
    FormatError(const std::string& msg, long line = 0)
        : Error(line > 0 ? msg + " (line " + std::to_string(line) + ")" : msg), line_(line) {}
    long line() const { return line_; }
private:
    long line_ = 0;
};
class SingularMatrixError : public Error { public: using Error::Error; };
class UnsupportedInputError : public Error { public: using Error::Error; };
class InvalidArgumentError : public Error { public: using Error::Error; };
class TransportError : public Error { public: using Error::Error; };

namespace detail {
inline void check(int rc) {
    if (rc == SPARSLA_OK) return;
    const std::string m = sparsla_last_error_message();
    switch (rc) {
        case SPARSLA_ERR_DIMENSION: throw DimensionError(m);
        case SPARSLA_ERR_BOUNDS: throw BoundsError(m);
        case SPARSLA_ERR_FORMAT: throw FormatError(m);
        case SPARSLA_ERR_SINGULAR: throw SingularMatrixError(m);
        case SPARSLA_ERR_UNSUPPORTED: throw UnsupportedInputError(m);
        case SPARSLA_ERR_INVALID_ARGUMENT: throw InvalidArgumentError(m);
        case SPARSLA_ERR_TRANSPORT:
        case SPARSLA_ERR_NCCL: throw TransportError(m);
        default: throw Error(m);
    }
}
}  // namespace detail

}  // namespace sparsla
