// ct_common.cuh -- shared helpers for libct (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/ct.h"

typedef int64_t i64;
typedef uint64_t u64;

#define CT_NUM_SMS 148

namespace ct {

void set_error(const char *fmt, ...);

// Return CT_ERR_CUDA (with message) if the last launch failed.
int check_launch(const char *what);

__host__ __device__ inline i64 clampi(i64 v, i64 lo, i64 hi) { return v < lo ? lo : (v > hi ? hi : v); }

inline int grid_for(i64 n, int block, int max_blocks = CT_NUM_SMS * 16) {
    i64 g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

template <typename T> struct dtype_of;
template <> struct dtype_of<uint8_t> { static constexpr int value = CT_U8; };
template <> struct dtype_of<uint16_t> { static constexpr int value = CT_U16; };
template <> struct dtype_of<double> { static constexpr int value = CT_F64; };

__device__ __forceinline__ double to_f64(uint8_t v) { return (double)v; }
__device__ __forceinline__ double to_f64(uint16_t v) { return (double)v; }
__device__ __forceinline__ double to_f64(double v) { return v; }

// numpy rint + clip(0, 65535) (segment.py:160-161) for the histogram bin
__device__ __forceinline__ int hist_bin(uint8_t v) { return v; }
__device__ __forceinline__ int hist_bin(uint16_t v) { return v; }
__device__ __forceinline__ int hist_bin(double v) {
    double q = rint(v);
    if (!(q > 0.0)) return 0;  // also NaN -> 0 (numpy would misbehave; not reachable on real data)
    if (q >= 65535.0) return 65535;
    return (int)q;
}

// "rint(v) > t" of binarize (segment.py:204)
__device__ __forceinline__ bool above(uint8_t v, i64 t) { return (i64)v > t; }
__device__ __forceinline__ bool above(uint16_t v, i64 t) { return (i64)v > t; }
__device__ __forceinline__ bool above(double v, i64 t) { return rint(v) > (double)t; }

}  // namespace ct

// Dispatch a lambda-like body over a volume dtype.
#define CT_DISPATCH(dtype, T, ...)                                   \
    switch (dtype) {                                                 \
        case CT_U8: { typedef uint8_t T; __VA_ARGS__; break; }       \
        case CT_U16: { typedef uint16_t T; __VA_ARGS__; break; }     \
        case CT_F64: { typedef double T; __VA_ARGS__; break; }       \
        default:                                                     \
            ct::set_error("unsupported dtype code %d", (int)(dtype)); \
            return CT_ERR_UNSUPPORTED;                               \
    }
