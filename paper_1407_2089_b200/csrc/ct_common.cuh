// ct_common.cuh -- shared helpers for libct (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/ct.h"

typedef int64_t i64;
typedef uint64_t u64;

#define CT_NUM_SMS 148

// Device-side bounds checks of the debug build (make debug -> libct_debug.so,
// -DCT_DEBUG; loaded when CT_LIB=debug): a failed check prints the site and
// traps, so the launch fails with an error instead of corrupting memory.  The
// stand-in for compute-sanitizer, which is closed on the GPU pool.  No-ops in
// the product build.
#ifdef CT_DEBUG
#define CT_DCHECK(cond)                                                                  \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("CT_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                            \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define CT_DCHECK(cond) ((void)0)
#endif

namespace ct {

void set_error(const char *fmt, ...);

// Return CT_ERR_CUDA (with message) if the last launch failed.
int check_launch(const char *what);

// n / d for a divisor fixed per kernel or per work item (round-up
// multiply-shift, exact for every 32-bit n): runtime 32-bit divides were ~20%
// of the instructions of the K1 tile loops and of the K6 bounding-box walk.
// Construct it on the host (kernel argument) where every thread would build
// it: the constructor's loop and 64-bit divide were ~8% of close1_bits.
struct FastDiv {
    uint32_t d, m, s;
    __host__ __device__ explicit FastDiv(uint32_t d_) : d(d_) {
        s = 0;
        while ((1ull << s) < d) ++s;
        m = (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return (uint32_t)(((unsigned long long)__umulhi(n, m) + n) >> s);
    }
};

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
// exact double of an integer 0 <= v < 2^31 on the FP64 pipe (one DADD:
// 2^52 + v built from its bits, minus 2^52) instead of an I2F.F64 on the
// quarter-rate XU pipe
__device__ __forceinline__ double u2d(uint32_t v) {
    return __dadd_rn(__hiloint2double(0x43300000, (int)v), -4503599627370496.0);
}
// x[a] + x[b] of two raw (integer) values in double: exact, so the integer sum
// converted once equals scipy's float64 sum of the two converted values
__device__ __forceinline__ double pair_f64(uint8_t a, uint8_t b) { return u2d((uint32_t)a + b); }
__device__ __forceinline__ double pair_f64(uint16_t a, uint16_t b) { return u2d((uint32_t)a + b); }
__device__ __forceinline__ double pair_f64(double a, double b) { return __dadd_rn(a, b); }

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

namespace ct {

__device__ __forceinline__ unsigned laneid() {
    unsigned l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

// Conflict-free 256-bin histogram for 256-thread CTAs: every thread owns a
// private 8-bit counter per bin (no atomics).  Counter (bin, thread) lives in
// byte (warp % 4) of word [(warp / 4) * 256 + bin] * 32 + lane, so a warp's
// 32 increments always hit 32 distinct banks whatever the values.  Each
// thread may add at most 255 values between flush() calls; flush() folds the
// bytes into per-CTA 32-bit totals with one DP4A per word.
// SMEM: 64 KB of counters + 1 KB totals.
struct ByteHist256 {
    uint32_t *words;  // [2][256][32]
    uint32_t *tot;    // [256]
    static constexpr size_t kBytes = 2 * 256 * 32 * 4 + 256 * 4;

    __device__ void init(void *smem) {
        words = (uint32_t *)smem;
        tot = words + 2 * 256 * 32;
        for (int i = threadIdx.x; i < 2 * 256 * 32; i += blockDim.x) words[i] = 0;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) tot[i] = 0;
    }
    __device__ __forceinline__ void add(int v) {
        const unsigned w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        uint8_t *p = (uint8_t *)(words + ((w >> 2) * 256 + v) * 32 + lane) + (w & 3);
        *p = (uint8_t)(*p + 1);
    }
    // all threads; blockDim.x == 256
    __device__ void flush() {
        __syncthreads();
        const int b = threadIdx.x;
        unsigned s = tot[b];
        for (int g = 0; g < 2; ++g) {
            uint32_t *row = words + (g * 256 + b) * 32;
#pragma unroll 8
            for (int l = 0; l < 32; ++l) {
                const int c = (l + b) & 31;  // rotate: lanes hit distinct banks
                s = __dp4a(row[c], 0x01010101u, s);
                row[c] = 0;
            }
        }
        tot[b] = s;
        __syncthreads();
    }
    __device__ void to_global(unsigned long long *g) {
        const int b = threadIdx.x;
        if (tot[b]) atomicAdd(g + b, (unsigned long long)tot[b]);
    }
};

// z-row words: u64 for nz <= 64, unsigned __int128 for nz <= 128 (bit k = voxel k)
using u128 = unsigned __int128;
__device__ __forceinline__ int rffs(unsigned long long x) { return __ffsll((long long)x); }
__device__ __forceinline__ int rffs(u128 x) {
    const unsigned long long lo = (unsigned long long)x, hi = (unsigned long long)(x >> 64);
    return lo ? __ffsll((long long)lo) : (hi ? 64 + __ffsll((long long)hi) : 0);
}
__device__ __forceinline__ int rclz(unsigned long long x) { return __clzll((long long)x); }  // 64 bits
__device__ __forceinline__ int rclz(u128 x) {  // 128 bits
    const unsigned long long lo = (unsigned long long)x, hi = (unsigned long long)(x >> 64);
    return hi ? __clzll((long long)hi) : 64 + __clzll((long long)lo);
}
__device__ __forceinline__ int rpopc(unsigned long long x) { return __popcll(x); }
__device__ __forceinline__ int rpopc(u128 x) {
    return __popcll((unsigned long long)x) + __popcll((unsigned long long)(x >> 64));
}
template <typename R> __host__ __device__ constexpr int rbits() { return (int)(8 * sizeof(R)); }
template <typename R> __device__ __forceinline__ R rmask(int n) { return n >= rbits<R>() ? ~(R)0 : (((R)1 << n) - 1); }

}  // namespace ct
