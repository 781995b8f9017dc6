// Shared definitions for the B200-native min-norm hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "common_host.hpp"

namespace mnb {

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        const int code = (e == cudaErrorMemoryAllocation) ? MNB_ERR_OUT_OF_MEMORY : MNB_ERR_CUDA;
        throw Error(code, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                              std::to_string(line) + ")");
    }
}
#define MNB_CUDA(x) ::mnb::cuda_check((x), #x, __FILE__, __LINE__)
#define MNB_LAUNCH_CHECK() ::mnb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// ----------------------------------------------------------- complex ------
// Exact-rounding complex helpers.  `_rn` forms forbid FMA contraction so the
// H stage reproduces the reference scalar backend bit for bit
// (src/kernels_scalar.cpp:7-33: gcc's complex product is
//  re = ac - bd, im = ad + bc, each term rounded; no FMA on baseline x86-64).
__device__ __forceinline__ double2 c_mul_rn(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 c_conj(double2 a) { return make_double2(a.x, -a.y); }

// Free (FMA-allowed) arithmetic for the FFT / GEMV paths.
__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 c_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

inline unsigned ceil_div(int64_t a, int64_t b) { return unsigned((a + b - 1) / b); }

}  // namespace mnb
