// fusim/errors.hpp — B200 façade: the exception taxonomy of the reference API.
//
// Drop-in for /root/reference/proj/include/fusim/errors.hpp (class names and
// hierarchy are the API; every class derives from fusim::Error, itself a
// std::runtime_error).  The C ABI below the façade returns mlora_status codes;
// throw_status() turns them back into these types at the C++ boundary.
#pragma once

#include <stdexcept>
#include <string>

namespace fusim {

/// Root of every error raised by the library.
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
    explicit Error(const char* what) : std::runtime_error(what) {}
};

/// Invalid experiment configuration or input file.
class ConfigError : public Error { public: using Error::Error; };
/// A precondition of the call was violated by the caller.
class UsageError : public Error { public: using Error::Error; };
/// The object is not in a state that permits the operation.
class StateError : public Error { public: using Error::Error; };
/// Operand dimensions do not agree.
class ShapeError : public Error { public: using Error::Error; };
/// A value that must be finite is NaN or infinite.
class NumericError : public Error { public: using Error::Error; };
/// A fused sequence is routed to a job that has no adapter.
class RoutingError : public Error { public: using Error::Error; };
/// A least-squares fit cannot be carried out.
class FitError : public Error { public: using Error::Error; };

/// Device/runtime failure below the façade (no reference counterpart).
class DeviceError : public Error { public: using Error::Error; };

}  // namespace fusim
