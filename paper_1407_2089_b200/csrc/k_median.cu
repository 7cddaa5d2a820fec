// k_median.cu -- K2: 3-D median filter (+ fused histogram) and the histogram.
//
// Replaces ref denoise.py:87-88 (ndimage.median_filter(size=2r+1,
// mode="nearest"): the size^3//2 order statistic of the clamp-to-edge cube)
// and ref segment.py:154-163 (intensity_histogram).
//
// r == 1, integer volumes: each thread filters two z-neighbours at once as a
// packed u16x2 pair (VIMNMX.U16x2 does min/max of both lanes in one op) with
// a forgetful-selection network: keep 15 candidates, repeatedly drop the
// minimum and maximum and admit the next window value; the survivor of the
// final three is the 14th smallest of 27.  The tile (with a clamped halo)
// is staged in SMEM as u16 with even alignment so the (k-1,k),(k,k+1),(k+1,k+2)
// pairs are one aligned LDS.32 plus one PRMT each.  The output histogram is
// accumulated per CTA in SMEM (warp-aggregated with __match_any_sync) and
// flushed once per persistent CTA.
#include "ct_common.cuh"

namespace {

constexpr int TK = 32;  // outputs along z per tile
constexpr int TJ = 8;
constexpr int TI = 2;
constexpr int SK = TK + 4;  // staged z extent: k0-2 .. k0+TK+1 (even-aligned)
constexpr int HBINS = 4096; // SMEM histogram bins (higher values go to global)

struct OpsU2 {
    typedef uint32_t T;
    static __device__ __forceinline__ T mn(T a, T b) { return __vminu2(a, b); }
    static __device__ __forceinline__ T mx(T a, T b) { return __vmaxu2(a, b); }
};
struct OpsF64 {
    typedef double T;
    static __device__ __forceinline__ T mn(T a, T b) { return b < a ? b : a; }
    static __device__ __forceinline__ T mx(T a, T b) { return b < a ? a : b; }
};

// 14th smallest of v[0..26]: forgetful selection, fully unrolled.
// Round with live set a[0..m-1]: order (a[0], a[m-1]); then for each pair of
// middle elements, the pair's low is exchanged against a[0] and its high
// against a[m-1] (an odd middle element goes through both), so a[0] ends
// as the minimum and a[m-1] as the maximum; both are dropped and the next
// window value is admitted into slot 0.  12 rounds take 15 -> 3 survivors.
template <class Ops>
__device__ __forceinline__ typename Ops::T median27(const typename Ops::T (&v)[27]) {
    typedef typename Ops::T T;
    T a[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) a[i] = v[i];
#pragma unroll
    for (int round = 0; round < 12; ++round) {
        const int m = 15 - round;
        {
            const T lo = Ops::mn(a[0], a[m - 1]), hi = Ops::mx(a[0], a[m - 1]);
            a[0] = lo;
            a[m - 1] = hi;
        }
#pragma unroll
        for (int i = 1; i + 1 < m - 1; i += 2) {
            const T lo = Ops::mn(a[i], a[i + 1]), hi = Ops::mx(a[i], a[i + 1]);
            a[i] = Ops::mx(a[0], lo);
            a[0] = Ops::mn(a[0], lo);
            a[i + 1] = Ops::mn(a[m - 1], hi);
            a[m - 1] = Ops::mx(a[m - 1], hi);
        }
        if ((m - 2) & 1) {
            const T x = a[m - 2];
            const T y = Ops::mx(a[0], x);
            a[0] = Ops::mn(a[0], x);
            a[m - 2] = Ops::mn(a[m - 1], y);
            a[m - 1] = Ops::mx(a[m - 1], y);
        }
        a[0] = v[15 + round];  // drop min (slot 0) and max (slot m-1)
    }
    const T lo = Ops::mn(a[0], a[1]), hi = Ops::mx(a[0], a[1]);
    return Ops::mx(lo, Ops::mn(hi, a[2]));
}

__device__ __forceinline__ void hist_add(uint32_t *sh, uint64_t *gh, int v) {
    const unsigned full = __activemask();
    const unsigned peers = __match_any_sync(full, v);
    const int leader = __ffs(peers) - 1;
    unsigned lane;
    asm("mov.u32 %0, %%laneid;" : "=r"(lane));
    if ((int)lane == leader) {
        const unsigned n = __popc(peers);
        if (v < HBINS) atomicAdd(&sh[v], n);
        else atomicAdd((unsigned long long *)&gh[v], (unsigned long long)n);
    }
}

// ---------------------------------------------------------------------------
// r == 1 on u8/u16 volumes.  Persistent CTAs of (TK/2, TJ, TI) threads.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(TK / 2 * TJ * TI) median3_int(const T *__restrict__ in, T *__restrict__ out,
                                                                i64 nx, i64 ny, i64 nz, uint64_t *__restrict__ ghist) {
    __shared__ __align__(16) uint16_t tile[TI + 2][TJ + 2][SK];
    __shared__ uint32_t sh[HBINS];
    const int tid = (threadIdx.z * TJ + threadIdx.y) * (TK / 2) + threadIdx.x;
    const int nth = TK / 2 * TJ * TI;
    if (ghist)
        for (int b = tid; b < HBINS; b += nth) sh[b] = 0;
    const i64 tk = (nz + TK - 1) / TK, tj = (ny + TJ - 1) / TJ, ti = (nx + TI - 1) / TI;
    const i64 ntiles = tk * tj * ti;
    for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const i64 k0 = (t % tk) * TK, j0 = ((t / tk) % tj) * TJ, i0 = (t / (tk * tj)) * TI;
        __syncthreads();
        for (int idx = tid; idx < (TI + 2) * (TJ + 2) * SK; idx += nth) {
            const int kk = idx % SK, jj = (idx / SK) % (TJ + 2), ii = idx / (SK * (TJ + 2));
            const i64 i = ct::clampi(i0 + ii - 1, 0, nx - 1), j = ct::clampi(j0 + jj - 1, 0, ny - 1),
                      k = ct::clampi(k0 + kk - 2, 0, nz - 1);
            tile[ii][jj][kk] = (uint16_t)in[(i * ny + j) * nz + k];
        }
        __syncthreads();
        const int lk = 2 * threadIdx.x, lj = threadIdx.y, li = threadIdx.z;
        const i64 i = i0 + li, j = j0 + lj, k = k0 + lk;
        if (i < nx && j < ny && k < nz) {
            uint32_t v[27];
            int e = 0;
#pragma unroll
            for (int di = 0; di < 3; ++di)
#pragma unroll
                for (int dj = 0; dj < 3; ++dj) {
                    const uint32_t *row = reinterpret_cast<const uint32_t *>(&tile[li + di][lj + dj][0]);
                    const uint32_t w0 = row[lk / 2], w1 = row[lk / 2 + 1], w2 = row[lk / 2 + 2];
                    // staged index of output k is lk+2 -> word lk/2+1 = (k, k+1)
                    v[e++] = __byte_perm(w0, w1, 0x5432);  // (k-1, k)
                    v[e++] = w1;                           // (k,   k+1)
                    v[e++] = __byte_perm(w1, w2, 0x5432);  // (k+1, k+2)
                }
            const uint32_t med = median27<OpsU2>(v);
            const i64 p = (i * ny + j) * nz + k;
            const T m0 = (T)(med & 0xFFFF), m1 = (T)(med >> 16);
            out[p] = m0;
            const bool two = k + 1 < nz;
            if (two) out[p + 1] = m1;
            if (ghist) {
                hist_add(sh, ghist, m0);
                if (two) hist_add(sh, ghist, m1);
            }
        }
    }
    if (ghist) {
        __syncthreads();
        for (int b = tid; b < HBINS; b += nth)
            if (sh[b]) atomicAdd((unsigned long long *)&ghist[b], (unsigned long long)sh[b]);
    }
}

// r == 1 on float64 (API path: denoise_cell_channel returns float64).
__global__ void __launch_bounds__(256) median3_f64(const double *__restrict__ in, double *__restrict__ out, i64 nx,
                                                   i64 ny, i64 nz) {
    const i64 n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
        double v[27];
        int e = 0;
#pragma unroll
        for (int di = -1; di <= 1; ++di)
#pragma unroll
            for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
                for (int dk = -1; dk <= 1; ++dk)
                    v[e++] = in[(ct::clampi(i + di, 0, nx - 1) * ny + ct::clampi(j + dj, 0, ny - 1)) * nz +
                                ct::clampi(k + dk, 0, nz - 1)];
        out[p] = median27<OpsF64>(v);
    }
}

// any radius, any dtype: window gathered into local memory, quickselect.
template <typename T>
__device__ T select_kth(T *a, int n, int k) {
    int lo = 0, hi = n - 1;
    while (hi > lo) {
        T x = a[lo], y = a[(lo + hi) / 2], z = a[hi], piv;
        if ((x <= y) == (y <= z)) piv = y;
        else if ((y <= x) == (x <= z)) piv = x;
        else piv = z;
        int i = lo, j = hi;
        while (i <= j) {
            while (a[i] < piv) ++i;
            while (a[j] > piv) --j;
            if (i <= j) { T t = a[i]; a[i] = a[j]; a[j] = t; ++i; --j; }
        }
        if (k <= j) hi = j;
        else if (k >= i) lo = i;
        else return a[k];
    }
    return a[k];
}

template <typename T>
__global__ void __launch_bounds__(128) median_generic(const T *__restrict__ in, T *__restrict__ out, i64 nx, i64 ny,
                                                      i64 nz, int rad, uint64_t *__restrict__ ghist) {
    T buf[343];  // rad <= 3
    const int size = 2 * rad + 1, win = size * size * size;
    const i64 n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
        int e = 0;
        for (int di = -rad; di <= rad; ++di)
            for (int dj = -rad; dj <= rad; ++dj)
                for (int dk = -rad; dk <= rad; ++dk)
                    buf[e++] = in[(ct::clampi(i + di, 0, nx - 1) * ny + ct::clampi(j + dj, 0, ny - 1)) * nz +
                                  ct::clampi(k + dk, 0, nz - 1)];
        const T m = select_kth(buf, win, win / 2);
        out[p] = m;
        if (ghist) atomicAdd((unsigned long long *)&ghist[ct::hist_bin(m)], 1ull);
    }
}

// intensity_histogram over any dtype (segment.py:154-163)
template <typename T>
__global__ void __launch_bounds__(512) histogram_kernel(const T *__restrict__ in, i64 n, uint64_t *__restrict__ ghist) {
    __shared__ uint32_t sh[HBINS];
    for (int b = threadIdx.x; b < HBINS; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
        hist_add(sh, ghist, ct::hist_bin(in[p]));
    __syncthreads();
    for (int b = threadIdx.x; b < HBINS; b += blockDim.x)
        if (sh[b]) atomicAdd((unsigned long long *)&ghist[b], (unsigned long long)sh[b]);
}

}  // namespace

extern "C" int ct_median(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, int radius, void *out,
                         uint64_t *hist, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || radius < 0) {
        ct::set_error("bad median arguments");
        return CT_ERR_PARAM;
    }
    if (radius > 3) {
        ct::set_error("median radius %d > 3 unsupported", radius);
        return CT_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    if (radius == 0) {
        const size_t es = dtype == CT_U8 ? 1 : (dtype == CT_U16 ? 2 : 8);
        cudaMemcpyAsync(out, in, n * es, cudaMemcpyDeviceToDevice, s);
        if (hist) return ct_histogram(out, dtype, n, hist, stream);
        return ct::check_launch("median copy");
    }
    if (radius == 1 && (dtype == CT_U8 || dtype == CT_U16)) {
        const i64 tiles = ((nz + TK - 1) / TK) * ((ny + TJ - 1) / TJ) * ((nx + TI - 1) / TI);
        const int grid = (int)min(tiles, (i64)CT_NUM_SMS * 8);
        dim3 block(TK / 2, TJ, TI);
        if (dtype == CT_U8)
            median3_int<uint8_t><<<grid, block, 0, s>>>((const uint8_t *)in, (uint8_t *)out, nx, ny, nz, hist);
        else
            median3_int<uint16_t><<<grid, block, 0, s>>>((const uint16_t *)in, (uint16_t *)out, nx, ny, nz, hist);
        return ct::check_launch("median3_int");
    }
    if (radius == 1 && dtype == CT_F64) {
        median3_f64<<<ct::grid_for(n, 256), 256, 0, s>>>((const double *)in, (double *)out, nx, ny, nz);
        if (int st = ct::check_launch("median3_f64")) return st;
        if (hist) return ct_histogram(out, dtype, n, hist, stream);
        return CT_OK;
    }
    CT_DISPATCH(dtype, T, {
        median_generic<T><<<ct::grid_for(n, 128), 128, 0, s>>>((const T *)in, (T *)out, nx, ny, nz, radius, hist);
    });
    return ct::check_launch("median_generic");
}

extern "C" int ct_histogram(const void *in, int dtype, int64_t n, uint64_t *hist, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n <= 0) return CT_OK;
    CT_DISPATCH(dtype, T, {
        histogram_kernel<T><<<ct::grid_for(n, 512, CT_NUM_SMS * 2), 512, 0, s>>>((const T *)in, n, hist);
    });
    return ct::check_launch("histogram");
}
