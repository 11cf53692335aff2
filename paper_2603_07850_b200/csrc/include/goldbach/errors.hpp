// errors.hpp -- exception taxonomy of the drop-in C++ API.
// Same classes as the reference (proj/include/goldbach/errors.hpp:9-22);
// DeviceError is the B200 addition for CUDA failures.  Status codes of the
// C-ABI (include/goldbach_b200.h) are mapped back here by raise_status().
#pragma once

#include <stdexcept>
#include <string>

namespace goldbach {

struct ParamError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

struct ResourceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct InternalError : std::logic_error {
    using std::logic_error::logic_error;
};

// A CUDA runtime failure on the device path.
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Throws the exception matching a non-zero gb_* status code.
[[noreturn]] void raise_status(int status, const std::string& message);

} // namespace goldbach
