// k_synth.cu -- synthetic frames generated on the device.
//
// Counter-based: every voxel's value is a pure function of (seed, linear
// index, scene lists), identical to oracle/ct_oracle.c (ora_synth_*), so a
// GPU-generated frame equals the CPU oracle's without storing stacks.
//   base  = bg ramp (0.08 vmax + 0.04 vmax (x/nx + y/ny)) + Irwin-Hall noise
//   tubes = x-aligned cylinders, balls = spheres (1/16-voxel fixed point);
// inside voxels take clamp(base + amp): idempotent, so overlapping objects
// and launch order cannot change the result.
#include "ct_common.cuh"

namespace {

__device__ __forceinline__ u64 sm64(u64 x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ i64 floordiv(i64 a, i64 b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ i64 base_val(u64 key, i64 p, i64 i, i64 j, i64 nx, i64 ny, i64 vmax) {
    const u64 h = sm64(key ^ (u64)p);
    const i64 s = (i64)(h & 255) + (i64)((h >> 8) & 255) + (i64)((h >> 16) & 255) + (i64)((h >> 24) & 255);
    const i64 noise = floordiv((s - 510) * 13 * vmax, 65536);
    const i64 bg = (vmax * (8 * nx * ny + 4 * i * ny + 4 * j * nx)) / (100 * nx * ny);
    return bg + noise;
}

template <typename T>
__global__ void synth_base(T *out, i64 nx, i64 ny, i64 nz, u64 key, i64 vmax) {
    const i64 n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const i64 j = (p / nz) % ny, i = p / (ny * nz);
        out[p] = (T)ct::clampi(base_val(key, p, i, j, nx, ny, vmax), 0, vmax);
    }
}

template <typename T>
__global__ void synth_balls(T *out, i64 nx, i64 ny, i64 nz, u64 key, i64 vmax, const int64_t *balls, i64 amp) {
    const int64_t *b = balls + 4 * blockIdx.x;
    const i64 cx = b[0], cy = b[1], cz = b[2], r = b[3], r2 = r * r;
    const i64 i0 = ct::clampi(floordiv(cx - r, 16), 0, nx - 1), i1 = ct::clampi(floordiv(cx + r, 16) + 1, 0, nx - 1);
    const i64 j0 = ct::clampi(floordiv(cy - r, 16), 0, ny - 1), j1 = ct::clampi(floordiv(cy + r, 16) + 1, 0, ny - 1);
    const i64 k0 = ct::clampi(floordiv(cz - r, 16), 0, nz - 1), k1 = ct::clampi(floordiv(cz + r, 16) + 1, 0, nz - 1);
    const i64 bi = i1 - i0 + 1, bj = j1 - j0 + 1, bk = k1 - k0 + 1;
    for (i64 q = threadIdx.x; q < bi * bj * bk; q += blockDim.x) {
        const i64 k = k0 + q % bk, j = j0 + (q / bk) % bj, i = i0 + q / (bk * bj);
        const i64 a = 16 * i - cx, bb = 16 * j - cy, c = 16 * k - cz;
        if (a * a + bb * bb + c * c <= r2) {
            const i64 p = (i * ny + j) * nz + k;
            out[p] = (T)ct::clampi(base_val(key, p, i, j, nx, ny, vmax) + amp, 0, vmax);
        }
    }
}

template <typename T>
__global__ void synth_tubes(T *out, i64 nx, i64 ny, i64 nz, u64 key, i64 vmax, const int64_t *tubes, i64 amp) {
    const int64_t *t = tubes + 3 * blockIdx.y;
    const i64 cy = t[0], cz = t[1], r = t[2], r2 = r * r;
    const i64 j0 = ct::clampi(floordiv(cy - r, 16), 0, ny - 1), j1 = ct::clampi(floordiv(cy + r, 16) + 1, 0, ny - 1);
    const i64 k0 = ct::clampi(floordiv(cz - r, 16), 0, nz - 1), k1 = ct::clampi(floordiv(cz + r, 16) + 1, 0, nz - 1);
    const i64 bj = j1 - j0 + 1, bk = k1 - k0 + 1, n = nx * bj * bk;
    for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < n; q += (i64)gridDim.x * blockDim.x) {
        const i64 k = k0 + q % bk, j = j0 + (q / bk) % bj, i = q / (bk * bj);
        const i64 bb = 16 * j - cy, c = 16 * k - cz;
        if (bb * bb + c * c <= r2) {
            const i64 p = (i * ny + j) * nz + k;
            out[p] = (T)ct::clampi(base_val(key, p, i, j, nx, ny, vmax) + amp, 0, vmax);
        }
    }
}

template <typename T>
int synth(T *out, i64 nx, i64 ny, i64 nz, u64 seed, i64 vmax, const int64_t *balls, i64 nb, i64 ab,
          const int64_t *tubes, i64 nt, i64 at, cudaStream_t s) {
    // key = sm64(seed) computed on the host with the same mixer
    u64 x = seed + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    const u64 key = x ^ (x >> 31);
    const i64 n = nx * ny * nz;
    synth_base<T><<<ct::grid_for(n, 256), 256, 0, s>>>(out, nx, ny, nz, key, vmax);
    if (int st = ct::check_launch("synth_base")) return st;
    if (nt > 0) {
        synth_tubes<T><<<dim3(CT_NUM_SMS, (unsigned)nt), 256, 0, s>>>(out, nx, ny, nz, key, vmax, tubes, at);
        if (int st = ct::check_launch("synth_tubes")) return st;
    }
    if (nb > 0) {
        synth_balls<T><<<(unsigned)nb, 256, 0, s>>>(out, nx, ny, nz, key, vmax, balls, ab);
        if (int st = ct::check_launch("synth_balls")) return st;
    }
    return CT_OK;
}

}  // namespace

extern "C" int ct_synth_frame(void *out, int dtype, int64_t nx, int64_t ny, int64_t nz, uint64_t seed, int64_t vmax,
                              const int64_t *balls, int64_t n_balls, int64_t amp_ball, const int64_t *tubes,
                              int64_t n_tubes, int64_t amp_tube, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == CT_U8)
        return synth<uint8_t>((uint8_t *)out, nx, ny, nz, seed, vmax, balls, n_balls, amp_ball, tubes, n_tubes,
                              amp_tube, s);
    if (dtype == CT_U16)
        return synth<uint16_t>((uint16_t *)out, nx, ny, nz, seed, vmax, balls, n_balls, amp_ball, tubes, n_tubes,
                               amp_tube, s);
    ct::set_error("synthetic frames are U8 or U16");
    return CT_ERR_UNSUPPORTED;
}
