// portten-b200 — error classes of the reference operator API
// (mirrors proj/include/portten/errors.hpp:24-52: ValidationError -> exit 2,
// BackendError -> exit 3, PORTTEN_CHECK always on).
#pragma once

#include <stdexcept>
#include <string>

namespace portten {

class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

/// Bad arguments, malformed inputs, shape mismatches (CLI exit code 2).
class ValidationError : public Error {
public:
    explicit ValidationError(const std::string& what) : Error(what) {}
};

/// Device/runtime trouble: no device, CUDA failures, kernel launch errors (exit code 3).
class BackendError : public Error {
public:
    explicit BackendError(const std::string& what) : Error(what) {}
};

#define PORTTEN_CHECK(cond, msg)                              \
    do {                                                      \
        if (!(cond)) throw ::portten::ValidationError(msg);   \
    } while (false)

/// Rethrow a libpt_b200 status code (include/pt_b200.h) as the reference's exception.
void throw_if_error(int status);

}  // namespace portten
