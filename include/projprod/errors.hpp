#pragma once
// Exception taxonomy of the projprod API (proj/include/projprod/errors.hpp:9-37);
// the C-ABI status codes of include/ppc.h map one-to-one onto these.
#include <stdexcept>
#include <string>

namespace projprod {

struct shape_error : std::invalid_argument {            // PPC_SHAPE
    using std::invalid_argument::invalid_argument;
};
struct bounds_error : std::out_of_range {               // PPC_BOUNDS
    using std::out_of_range::out_of_range;
};
struct argument_error : std::invalid_argument {         // PPC_ARGUMENT
    using std::invalid_argument::invalid_argument;
};
struct degenerate_input_error : std::invalid_argument { // PPC_DEGENERATE
    using std::invalid_argument::invalid_argument;
};
struct numeric_error : std::runtime_error {             // PPC_NUMERIC
    using std::runtime_error::runtime_error;
};
struct format_error : std::runtime_error {              // PPC_FORMAT
    using std::runtime_error::runtime_error;
};
// CUDA runtime failure or no usable B200 (no reference analogue; the engine
// has no CPU path).
struct device_error : std::runtime_error {              // PPC_CUDA, PPC_NO_DEVICE
    using std::runtime_error::runtime_error;
};

// Throws the exception matching a ppc status code (no-op for PPC_OK).
void throw_status(int code, const char* message);

}  // namespace projprod
