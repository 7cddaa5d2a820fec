// k_ingest.cu -- device half of the ingest step: the
// (z, y, x) page order of a TIFF stack to the (x, y, z) grid order of the
// path, after the raw pages were copied H2D (ref imaging.py:219-220 does
// this transpose on the host: np.ascontiguousarray(pages.transpose(2, 1, 0))).
//
// dst[c][b][a] = src[a][b][c]: per b, a TILE x TILE tile is read along c
// (coalesced), staged in SMEM, and written along a (coalesced).  HBM-bound:
// 2 * elem bytes per element.  Optional per-element byte swap for
// big-endian files, folded into the store.
#include "ct_common.cuh"

namespace {

template <typename T>
__device__ __forceinline__ T bswap(T v);
template <>
__device__ __forceinline__ uint8_t bswap(uint8_t v) { return v; }
template <>
__device__ __forceinline__ uint16_t bswap(uint16_t v) { return (uint16_t)__byte_perm(v, 0, 0x3201) ; }
template <>
__device__ __forceinline__ uint32_t bswap(uint32_t v) { return __byte_perm(v, 0, 0x0123); }
template <>
__device__ __forceinline__ uint64_t bswap(uint64_t v) {
    return ((uint64_t)__byte_perm((uint32_t)v, 0, 0x0123) << 32) | __byte_perm((uint32_t)(v >> 32), 0, 0x0123);
}

template <typename T, int TILE>
__global__ void __launch_bounds__(256) transpose_xz(const T *__restrict__ src, T *__restrict__ dst, i64 na, i64 nb,
                                                    i64 nc, int swap) {
    constexpr int RY = 256 / TILE;
    __shared__ T tile[TILE][TILE + 1];
    const int tx = threadIdx.x % TILE, ty = threadIdx.x / TILE;
    const i64 c0 = (i64)blockIdx.x * TILE, a0 = (i64)blockIdx.y * TILE;
    for (i64 b = blockIdx.z; b < nb; b += gridDim.z) {
#pragma unroll
        for (int r = ty; r < TILE; r += RY) {
            const i64 a = a0 + r, c = c0 + tx;
            if (a < na && c < nc) tile[r][tx] = src[(a * nb + b) * nc + c];
        }
        __syncthreads();
#pragma unroll
        for (int r = ty; r < TILE; r += RY) {
            const i64 c = c0 + r, a = a0 + tx;
            if (a < na && c < nc) {
                T v = tile[tx][r];
                if (swap) v = bswap(v);
                dst[(c * nb + b) * na + a] = v;
            }
        }
        __syncthreads();
    }
}

template <typename T, int TILE>
void launch(const void *src, void *dst, i64 na, i64 nb, i64 nc, int swap, cudaStream_t s) {
    const dim3 grid((unsigned)((nc + TILE - 1) / TILE), (unsigned)((na + TILE - 1) / TILE), (unsigned)min(nb, (i64)65535));
    transpose_xz<T, TILE><<<grid, 256, 0, s>>>((const T *)src, (T *)dst, na, nb, nc, swap);
}

}  // namespace

extern "C" int ct_transpose_xz(const void *src, void *dst, int64_t na, int64_t nb, int64_t nc, int32_t elem_bytes,
                               int32_t byteswap, void *stream) {
    if (na <= 0 || nb <= 0 || nc <= 0 || (nc + 63) / 64 > 2147483647 || (na + 63) / 64 > 65535) {
        ct::set_error("ct_transpose_xz: bad sizes (%lld, %lld, %lld)", (long long)na, (long long)nb, (long long)nc);
        return CT_ERR_PARAM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    switch (elem_bytes) {
        case 1: launch<uint8_t, 64>(src, dst, na, nb, nc, byteswap, s); break;
        case 2: launch<uint16_t, 64>(src, dst, na, nb, nc, byteswap, s); break;
        case 4: launch<uint32_t, 32>(src, dst, na, nb, nc, byteswap, s); break;
        case 8: launch<uint64_t, 32>(src, dst, na, nb, nc, byteswap, s); break;
        default:
            ct::set_error("ct_transpose_xz: element size %d", (int)elem_bytes);
            return CT_ERR_PARAM;
    }
    return ct::check_launch("ct_transpose_xz");
}
