#pragma once
// Exception taxonomy of the reference API (reference include/ttstream/errors.hpp:9-55),
// kept class-for-class so callers of the drop-in catch the same types.  The
// C ABI (ttg.h) returns status codes; detail::throw_status maps them back.

#include <stdexcept>
#include <string>

namespace ttstream {

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class DimensionError : public Error { public: using Error::Error; };
class NumericError : public Error { public: using Error::Error; };
class StateError : public Error { public: using Error::Error; };
class FormatError : public Error { public: using Error::Error; };
class IndexError : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class ResourceError : public Error { public: using Error::Error; };
/// CUDA / NCCL failures of the device path (no reference analogue).
class DeviceError : public Error { public: using Error::Error; };

namespace detail {
[[noreturn]] void throw_status(int status, const std::string& msg);
}  // namespace detail

}  // namespace ttstream
