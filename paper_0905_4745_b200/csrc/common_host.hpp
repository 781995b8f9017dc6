// Host-only shared definitions (no CUDA headers).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/minnorm_b200.h"

namespace mnb {

// Error carrying a C-ABI status code (include/minnorm_b200.h) -- mirrors the
// reference's exception taxonomy (include/minnorm/errors.hpp:10-49).
struct Error : std::runtime_error {
    int code;
    int64_t deficient;
    Error(int c, const std::string& what, int64_t d = 0) : std::runtime_error(what), code(c), deficient(d) {}
};

inline void require(bool ok, int code, const std::string& what) {
    if (!ok) throw Error(code, what);
}

// generate_instance of the reference front end (instance.cpp; src/bench.cpp:46-74)
void generate_instance(int64_t m, int64_t n, double kappa, uint64_t stream_seed, double* A_out, double* b_out,
                       double* p_out);

}  // namespace mnb
