// mh/abi.hpp -- glue between the C ABI (mhg.h) and the C++ mirror of the
// reference's header API (namespace mh).  Status codes become the exception
// classes the reference throws.
#pragma once

#include <stdexcept>
#include <string>

#include "mhg.h"

namespace mh::gpu {

[[noreturn]] inline void raise(mhg_status st) {
    const std::string msg = mhg_last_error();
    switch (st) {
        case MHG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case MHG_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case MHG_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error("mhg: " + msg);
    }
}

inline void check(mhg_status st) {
    if (st != MHG_OK) raise(st);
}

}  // namespace mh::gpu
