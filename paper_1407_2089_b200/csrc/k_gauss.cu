// k_gauss.cu -- K1: Gaussian background + residual + quantise.
//
// Replaces ref denoise.py:84-86:
//   background = ndimage.gaussian_filter(values, sigma, mode="nearest", truncate=4)
//   residual   = np.maximum(values - background, 0.0)
// scipy runs correlate1d along axis 0, 1, 2 with float64 intermediates; the
// symmetric branch of NI_Correlate1D accumulates
//   acc = x[i]*w[0];  for j = r..1: acc += (x[i-j] + x[i+j]) * w[j]
// with separately rounded multiply and add.  This file reproduces that order
// bit for bit (every op is __dmul_rn / __dadd_rn, so no DFMA can appear),
// which makes the kernel FP64-pipe bound: 3r+1 FP64 ops per voxel per axis.
//
// Layout: the volume is [nx][ny][nz] (z fastest).  Axes 0 and 1 are strided
// ("columns" = the contiguous inner index, lanes map to columns, coalesced);
// axis 2 is contiguous (lanes map to lines, each line staged whole in SMEM).
// Each thread computes B consecutive outputs along the filtered axis and keeps
// a left and a right window of B inputs in registers that slide one step per
// tap, so a tap costs 2 shared loads per B outputs (3B FP64 ops).
#include <cooperative_groups.h>
#include <cstdlib>
#include <type_traits>

#include "ct_common.cuh"

namespace {

constexpr int B = 8;      // outputs per thread along the filtered axis
constexpr int C = 32;     // columns per CTA (strided kernel) / lines per CTA (contig)
constexpr int TMAX = 128; // max tile length along the axis (strided kernel)
constexpr size_t SMEM_LIMIT = 200 * 1024;

// Sliding-window accumulation for outputs at local rows base..base+B-1 of a
// column whose element at local row q is col[q*stride].  Rows base-r .. base+B-1+r
// must be valid.  Exactly scipy's order per output.
template <bool FMA = false>
__device__ __forceinline__ void window_taps(const double *__restrict__ col, int stride, int base, int r,
                                            const double *__restrict__ w, double (&acc)[B]) {
    double Lw[B], Rw[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
        acc[b] = __dmul_rn(col[(base + b) * stride], w[0]);
        Lw[b] = col[(base - r + b) * stride];
        Rw[b] = col[(base + r + b) * stride];
    }
    int m = 0;
    // blocks of B taps: left slot (b+u)%B, right slot (b-u)%B are static
    for (; m + B <= r; m += B) {
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const double wj = w[r - m - u];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (FMA) {  // two independent FMAs: no add -> multiply dependency
                    acc[b] = __fma_rn(Lw[(b + u) % B], wj, acc[b]);
                    acc[b] = __fma_rn(Rw[(b - u + B) % B], wj, acc[b]);
                } else {
                    const double s = __dadd_rn(Lw[(b + u) % B], Rw[(b - u + B) % B]);
                    acc[b] = __dadd_rn(acc[b], __dmul_rn(s, wj));
                }
            }
            // slide to tap m+u+1: one new left element (row base-r+m+u+B),
            // one new right element (row base+r-(m+u+1)); both always in range.
            Lw[u] = col[(base - r + m + u + B) * stride];
            Rw[B - 1 - u] = col[(base + r - (m + u + 1)) * stride];
        }
    }
    // remaining taps (r % B of them, innermost): direct loads
    for (; m < r; ++m) {
        const int j = r - m;
        const double wj = w[j];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            if (FMA) {
                acc[b] = __fma_rn(col[(base + b - j) * stride], wj, acc[b]);
                acc[b] = __fma_rn(col[(base + b + j) * stride], wj, acc[b]);
            } else {
                const double s = __dadd_rn(col[(base + b - j) * stride], col[(base + b + j) * stride]);
                acc[b] = __dadd_rn(acc[b], __dmul_rn(s, wj));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Strided axis (0 or 1): volume viewed as [outer][L][inner].
// grid: x = column chunks of C, y = tiles of T along the axis, z = outer.
// block: (C, T/B).  SMEM: tile[T+2r][C] doubles + w[r+1].
// ---------------------------------------------------------------------------
// CH consecutive elements (one vector load: 4 x u8, 4 x u16, 2 x f64) -> doubles
template <typename Tin>
struct Chunk {
    static constexpr int CH = sizeof(Tin) == 8 ? 2 : 4;
    using V = typename std::conditional<sizeof(Tin) == 1, uint32_t,
                                        typename std::conditional<sizeof(Tin) == 2, uint2, double2>::type>::type;
    __device__ static __forceinline__ void to_f64(const V &v, double (&o)[CH]) {
        if constexpr (sizeof(Tin) == 1) {
#pragma unroll
            for (int e = 0; e < 4; ++e) o[e] = (double)((v >> (8 * e)) & 0xffu);
        } else if constexpr (sizeof(Tin) == 2) {
            o[0] = (double)(v.x & 0xffffu); o[1] = (double)(v.x >> 16);
            o[2] = (double)(v.y & 0xffffu); o[3] = (double)(v.y >> 16);
        } else {
            o[0] = v.x; o[1] = v.y;
        }
    }
};

template <typename Tin, bool FMA = false, int TT = TMAX, int MINB = 1>
__global__ void __launch_bounds__(C *TT / B, MINB) gauss_strided(const Tin *__restrict__ in, double *__restrict__ out,
                                                            i64 L, i64 inner, const double *__restrict__ w, int r,
                                                            int T) {
    extern __shared__ double smem[];
    const int R = T + 2 * r;
    double *tile = smem;
    double *ws = smem + (size_t)R * C;
    const i64 o = blockIdx.z;
    const i64 c0 = (i64)blockIdx.x * C;
    const i64 t0 = (i64)blockIdx.y * T;
    const int cw = (int)min((i64)C, inner - c0);
    const int tid = threadIdx.y * C + threadIdx.x, nth = C * blockDim.y;
    for (int j = tid; j <= r; j += nth) ws[j] = w[j];
    const Tin *src = in + o * L * inner + c0;
    using CK = Chunk<Tin>;
    constexpr int CH = CK::CH, CPR = C / CH;
    if (cw == C && (inner % CH) == 0 && ((uintptr_t)in % sizeof(typename CK::V)) == 0) {
        // vector loads, up to 8 in flight per thread, then convert + store
        const int total = R * CPR;
        for (int q0 = tid; q0 < total; q0 += 8 * nth) {
            typename CK::V buf[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + u * nth;
                if (q < total) {
                    const int row = q / CPR, h = q - row * CPR;
                    const i64 pos = ct::clampi(t0 - r + row, 0, L - 1);
                    buf[u] = __ldg((const typename CK::V *)(src + pos * inner) + h);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + u * nth;
                if (q < total) {
                    double v[CH];
                    CK::to_f64(buf[u], v);
#pragma unroll
                    for (int e = 0; e < CH; ++e) tile[q * CH + e] = v[e];
                }
            }
        }
    } else {
        for (int idx = tid; idx < R * C; idx += nth) {
            const int row = idx / C, c = idx - row * C;
            const i64 pos = ct::clampi(t0 - r + row, 0, L - 1);
            tile[idx] = c < cw ? ct::to_f64(src[pos * inner + c]) : 0.0;
        }
    }
    __syncthreads();
    const int c = threadIdx.x;
    const int ob = threadIdx.y * B;
    if (c >= cw || t0 + ob >= L) return;
    double acc[B];
    window_taps<FMA>(tile + c, C, r + ob, r, ws, acc);
    double *dst = out + o * L * inner + c0 + c;
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const i64 pos = t0 + ob + b;
        if (pos < L) dst[pos * inner] = acc[b];
    }
}

// ---------------------------------------------------------------------------
// Contiguous axis (2) with the fused epilogue of denoise.py:85-86.
// CTA = G lines (consecutive outer index) x whole line; lanes map to lines.
// SMEM line stride S = roundup(L,B) + 2r (+1 if even: conflict-free LDS.64).
// ---------------------------------------------------------------------------
// Certification of the FMA fast path (fused pipeline only): results within
// `cert` of a rounding boundary k+0.5 are appended to `fix` for the exact
// recompute (ct_gaussian_q); fix[0] = count, fix[1] = overflow, fix[2..] = p.
struct Cert {
    double eps;
    unsigned long long *fix;
    long long cap;
};

template <typename Traw, typename Tq, bool FMA = false, int LC = 0>  // LC > 0: L == LC at compile time
__global__ void __launch_bounds__(512) gauss_contig(const double *__restrict__ in, i64 nlines, int L_,
                                                      const double *__restrict__ w, int r, int S, int G,
                                                      const Traw *__restrict__ raw, double *__restrict__ bg_out,
                                                      double *__restrict__ res_out, Tq *__restrict__ q_out,
                                                      Cert cert = Cert{0.0, nullptr, 0}) {
    const int L = LC > 0 ? LC : L_;
    extern __shared__ double smem[];
    double *tile = smem;                  // [G][S]
    double *ws = smem + (size_t)G * S;    // [r+1]
    const i64 line0 = (i64)blockIdx.x * G;
    const int gl = (int)min((i64)G, nlines - line0);
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nth = blockDim.x * blockDim.y;
    for (int j = tid; j <= r; j += nth) ws[j] = w[j];
    const double *src = in + line0 * L;
#pragma unroll 4
    for (int idx = tid; idx < gl * L; idx += nth) {
        const int g = idx / L, k = idx - g * L;
        tile[g * S + r + k] = src[idx];
    }
    // clamped halos: rows [0, r) and [r+L, S); x = line, y strides the halo
    const int halo = S - L;
    if (threadIdx.x < gl) {
        const double lo = src[(i64)threadIdx.x * L], hi = src[(i64)threadIdx.x * L + L - 1];
        for (int h = threadIdx.y; h < halo; h += blockDim.y) {
            const int row = h < r ? h : h + L;
            tile[threadIdx.x * S + row] = h < r ? lo : hi;
        }
    }
    __syncthreads();
    const int g = threadIdx.x;
    const int ob = threadIdx.y * B;
    const bool active = g < gl && ob < L;
    double acc[B];
    if (active) window_taps<FMA>(tile + (size_t)g * S, 1, r + ob, r, ws, acc);
    __syncthreads();
    if (active) {
#pragma unroll
        for (int b = 0; b < B; ++b)
            if (ob + b < L) tile[g * S + ob + b] = acc[b];
    }
    __syncthreads();
    // coalesced epilogue over the G*L outputs of this CTA
    for (int idx = tid; idx < gl * L; idx += nth) {
        const int gg = idx / L, k = idx - gg * L;
        const i64 p = line0 * L + idx;
        const double bg = tile[gg * S + k];
        if (bg_out) bg_out[p] = bg;
        const double d = __dadd_rn(ct::to_f64(raw[p]), -bg);
        const double res = d < 0.0 ? 0.0 : d;  // np.maximum(x, 0.0)
        if (res_out) res_out[p] = res;
        if (q_out) q_out[p] = (Tq)rint(res);
        if (FMA && cert.fix) {
            const double fr = __dadd_rn(res, -floor(res));
            if (fabs(__dadd_rn(fr, -0.5)) <= cert.eps) {
                const unsigned long long at = atomicAdd(&cert.fix[0], 1ull);
                if ((long long)at < cert.cap) cert.fix[2 + at] = (unsigned long long)p;
                else cert.fix[1] = 1;
            }
        }
    }
}

// Fallback for any size / radius: one thread per output, global loads.
template <typename Tin>
__global__ void gauss_generic(const Tin *__restrict__ in, double *__restrict__ out, i64 outer, i64 L, i64 inner,
                              const double *__restrict__ w, int r) {
    const i64 n = outer * L * inner;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const i64 c = p % inner, pos = (p / inner) % L, o = p / (inner * L);
        const Tin *line = in + o * L * inner + c;
        double acc = __dmul_rn(ct::to_f64(line[pos * inner]), w[0]);
        for (int j = r; j >= 1; --j) {
            const double s = __dadd_rn(ct::to_f64(line[ct::clampi(pos - j, 0, L - 1) * inner]),
                                       ct::to_f64(line[ct::clampi(pos + j, 0, L - 1) * inner]));
            acc = __dadd_rn(acc, __dmul_rn(s, w[j]));
        }
        out[p] = acc;
    }
}

template <typename Traw, typename Tq>
__global__ void residual_generic(const double *__restrict__ bg, i64 n, const Traw *__restrict__ raw,
                                 double *__restrict__ bg_out, double *__restrict__ res_out, Tq *__restrict__ q_out) {
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const double b = bg[p];
        if (bg_out && bg_out != bg) bg_out[p] = b;
        const double d = __dadd_rn(ct::to_f64(raw[p]), -b);
        const double res = d < 0.0 ? 0.0 : d;
        if (res_out) res_out[p] = res;
        if (q_out) q_out[p] = (Tq)rint(res);
    }
}

template <typename Tin>
__global__ void to_f64_copy(const Tin *__restrict__ in, double *__restrict__ out, i64 n) {
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
        out[p] = ct::to_f64(in[p]);
}

// One pass along a strided axis; returns CT status.
template <typename Tin, bool FMA = false>
int pass_strided(const Tin *in, double *out, i64 outer, i64 L, i64 inner, const double *w, int r,
                 cudaStream_t s) {
    const i64 n = outer * L * inner;
    if (r < 0) {
        to_f64_copy<Tin><<<ct::grid_for(n, 256), 256, 0, s>>>(in, out, n);
        return ct::check_launch("gauss copy");
    }
    int T = (int)min((i64)TMAX, ((L + B - 1) / B) * B);
    size_t sm = ((size_t)(T + 2 * r) * C + r + 1) * sizeof(double);
    if (sm > SMEM_LIMIT || outer > 65535 || (L + T - 1) / T > 65535) {
        gauss_generic<Tin><<<ct::grid_for(n, 256), 256, 0, s>>>(in, out, outer, L, inner, w, r);
        return ct::check_launch("gauss_generic");
    }
    auto k = gauss_strided<Tin, FMA, TMAX, 2>;  // (64-row tiles at 2-3 CTAs/SM, or 1 CTA/SM: measured slower)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT);
    dim3 grid((unsigned)((inner + C - 1) / C), (unsigned)((L + T - 1) / T), (unsigned)outer);
    dim3 block(C, T / B);
    k<<<grid, block, sm, s>>>(in, out, L, inner, w, r, T);
    return ct::check_launch("gauss_strided");
}

template <typename Traw, typename Tq>
int pass_contig(const double *in, i64 nlines, i64 L, const double *w, int r, const Traw *raw, double *bg_out,
                double *res_out, Tq *q_out, double *scratch, cudaStream_t s) {
    const i64 n = nlines * L;
    if (r >= 0) {
        int S = (int)(((L + B - 1) / B) * B + 2 * r);
        if ((S & 1) == 0) S += 1;
        int G = C;
        while (G > 1 && ((size_t)G * S + r + 1) * sizeof(double) > SMEM_LIMIT) G >>= 1;
        const size_t sm = ((size_t)G * S + r + 1) * sizeof(double);
        const int nb = (int)((L + B - 1) / B);
        if (sm <= SMEM_LIMIT && nb * G <= 512 && G == C) {
            cudaFuncSetAttribute(gauss_contig<Traw, Tq>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM_LIMIT);
            dim3 block(G, nb);
            gauss_contig<Traw, Tq><<<(unsigned)((nlines + G - 1) / G), block, sm, s>>>(in, nlines, (int)L, w, r, S,
                                                                                  G, raw, bg_out, res_out, q_out);
            return ct::check_launch("gauss_contig");
        }
    }
    // generic: filter into bg_out, res_out or the caller's scratch (N doubles), then epilogue
    double *tmp = bg_out ? bg_out : res_out ? res_out : scratch;
    if (r < 0) {
        cudaMemcpyAsync(tmp, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
    } else {
        gauss_generic<double><<<ct::grid_for(n, 256), 256, 0, s>>>(in, tmp, nlines, L, 1, w, r);
        if (int st = ct::check_launch("gauss_generic z")) return st;
    }
    residual_generic<Traw, Tq><<<ct::grid_for(n, 256), 256, 0, s>>>(tmp, n, raw, bg_out, res_out, q_out);
    return ct::check_launch("residual_generic");
}

template <typename Traw, typename Tq>
int gaussian_residual(const Traw *raw, i64 nx, i64 ny, i64 nz, const double *w, int rx, int ry, int rz,
                      double *work, double *bg_out, double *res_out, Tq *q_out, cudaStream_t s) {
    const i64 N = nx * ny * nz;
    double *p1 = work, *p2 = work + N;
    const double *wx = w, *wy = w + (rx >= 0 ? rx + 1 : 0), *wz = wy + (ry >= 0 ? ry + 1 : 0);
    if (int st = pass_strided<Traw>(raw, p1, 1, nx, ny * nz, wx, rx, s)) return st;
    if (int st = pass_strided<double>(p1, p2, nx, ny, nz, wy, ry, s)) return st;
    return pass_contig<Traw, Tq>(p2, nx * ny, nz, wz, rz, raw, bg_out, res_out, q_out, p1, s);  // p1 is dead here
}

}  // namespace

extern "C" int ct_gaussian_residual(const void *raw, int raw_dtype, int64_t nx, int64_t ny, int64_t nz,
                                    const double *w, int rx, int ry, int rz, void *work, double *bg_out,
                                    double *residual_out, void *q_out, int q_dtype, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("empty grid");
        return CT_ERR_PARAM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    double *wk = (double *)work;
    if (q_out && raw_dtype != q_dtype) {
        ct::set_error("q dtype must equal the raw dtype");
        return CT_ERR_UNSUPPORTED;
    }
    switch (raw_dtype) {
        case CT_U8:
            return gaussian_residual<uint8_t, uint8_t>((const uint8_t *)raw, nx, ny, nz, w, rx, ry, rz, wk, bg_out,
                                                       residual_out, (uint8_t *)q_out, s);
        case CT_U16:
            return gaussian_residual<uint16_t, uint16_t>((const uint16_t *)raw, nx, ny, nz, w, rx, ry, rz, wk,
                                                         bg_out, residual_out, (uint16_t *)q_out, s);
        case CT_F64:
            if (q_out) {
                ct::set_error("q output needs integer raw");
                return CT_ERR_UNSUPPORTED;
            }
            return gaussian_residual<double, uint16_t>((const double *)raw, nx, ny, nz, w, rx, ry, rz, wk, bg_out,
                                                       residual_out, (uint16_t *)nullptr, s);
        default:
            ct::set_error("unsupported raw dtype %d", raw_dtype);
            return CT_ERR_UNSUPPORTED;
    }
}

// float64 copy of a U8/U16/F64 volume (the reference's astype(np.float64))
extern "C" int ct_to_f64(const void *in, int dtype, int64_t n, double *out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n <= 0) return CT_OK;
    CT_DISPATCH(dtype, T, { to_f64_copy<T><<<ct::grid_for(n, 256), 256, 0, s>>>((const T *)in, out, n); });
    return ct::check_launch("to_f64");
}

// ---------------------------------------------------------------------------
// Fused-pipeline fast path: q = rint(max(raw - bg, 0)) with the three passes
// accumulated by FMA chains (acc = fma(x[i-j], w_j, acc); acc = fma(x[i+j],
// w_j, acc): 2 FP64 ops per tap instead of 3, no add->multiply dependency),
// certified exact.  A pass of 2r+1 chained FMAs is within gamma_{2r+1} M of
// the real convolution and scipy's order within gamma_{r+3} M (u = 2^-53, M =
// max input, weights positive and summing to 1), so over three passes the two
// differ by at most (3(rx+ry+rz)+12) u M (+ the residual's rounding), which
// eps = 4(2(rx+ry+rz)+11) u M covers; q can differ only where the residual
// is that close to a half-integer; those voxels (fix list) are recomputed
// exactly from their full dependency cone: pass-x values for the (2ry+1) x nz
// rows around the voxel, pass y on its z-line, pass z at the voxel -- the same
// operations in the same order as ct_gaussian_residual.
// ---------------------------------------------------------------------------
namespace {

// Entries f >= start of the fix list, one CTA per entry (fallback for lists
// larger than the scratch of the grid-wide kernels below).
template <typename Traw, typename Tq>
__global__ void __launch_bounds__(256) gauss_fixup(const Traw *__restrict__ raw, i64 nx, i64 ny, i64 nz,
                                                   const double *__restrict__ w, int rx, int ry, int rz,
                                                   const unsigned long long *__restrict__ fix, long long cap,
                                                   Tq *__restrict__ q_out, long long start) {
    extern __shared__ double fsm[];
    const int RJ = 2 * ry + 1;
    double *P1 = fsm;                      // [RJ][nz]
    double *P2 = fsm + (size_t)RJ * nz;    // [nz]
    const double *wx = w, *wy = w + rx + 1, *wz = wy + ry + 1;
    const long long cnt = min((long long)fix[0], cap);
    for (long long f = start + blockIdx.x; f < cnt; f += gridDim.x) {
        const i64 p = (i64)fix[2 + f];
        const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
        __syncthreads();
        for (i64 e = threadIdx.x; e < (i64)RJ * nz; e += blockDim.x) {
            const i64 t = e / nz - ry, kk = e % nz;
            const i64 jj = ct::clampi(j + t, 0, ny - 1);
            const Traw *col = raw + jj * nz + kk;
            const i64 S = ny * nz;
            double acc = __dmul_rn(ct::to_f64(col[i * S]), wx[0]);
            for (int d = rx; d >= 1; --d) {
                const double sm = __dadd_rn(ct::to_f64(col[ct::clampi(i - d, 0, nx - 1) * S]),
                                            ct::to_f64(col[ct::clampi(i + d, 0, nx - 1) * S]));
                acc = __dadd_rn(acc, __dmul_rn(sm, wx[d]));
            }
            P1[e] = acc;
        }
        __syncthreads();
        for (i64 kk = threadIdx.x; kk < nz; kk += blockDim.x) {
            // row offset t lives at index (t + ry); clamping was applied when staging
            double acc = __dmul_rn(P1[(i64)ry * nz + kk], wy[0]);
            for (int d = ry; d >= 1; --d) {
                const double sm = __dadd_rn(P1[(i64)(ry - d) * nz + kk], P1[(i64)(ry + d) * nz + kk]);
                acc = __dadd_rn(acc, __dmul_rn(sm, wy[d]));
            }
            P2[kk] = acc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double acc = __dmul_rn(P2[k], wz[0]);
            for (int d = rz; d >= 1; --d) {
                const double sm = __dadd_rn(P2[ct::clampi(k - d, 0, nz - 1)], P2[ct::clampi(k + d, 0, nz - 1)]);
                acc = __dadd_rn(acc, __dmul_rn(sm, wz[d]));
            }
            const double dd = __dadd_rn(ct::to_f64(raw[p]), -acc);
            q_out[p] = (Tq)rint(dd < 0.0 ? 0.0 : dd);
        }
    }
}

// Exact recompute of the first F = min(count, capF) fix entries (scratch
// P1[F][2ry+1][nz] doubles): pass x at the (2ry+1) x nz positions of each
// entry's cone (grid-wide), then per entry pass y on its z-line and pass z +
// residual at the voxel -- the operations and order of ct_gaussian_residual.
template <typename Traw>
__global__ void fix_p1(const Traw *__restrict__ raw, i64 nx, i64 ny, i64 nz, const double *__restrict__ w, int rx,
                       int ry, const unsigned long long *__restrict__ fix, long long cap, long long capF,
                       double *__restrict__ P1) {
    const long long F = min(min((long long)fix[0], cap), capF);
    const i64 RJ = 2 * ry + 1, per = RJ * nz, S = ny * nz;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < F * per; e += (i64)gridDim.x * blockDim.x) {
        const i64 f = e / per, rem = e - f * per, tt = rem / nz, kk = rem - tt * nz;
        const i64 p = (i64)fix[2 + f];
        const i64 j = (p / nz) % ny, i = p / S;
        const i64 jj = ct::clampi(j + tt - ry, 0, ny - 1);
        const Traw *col = raw + jj * nz + kk;
        double acc = __dmul_rn(ct::to_f64(col[i * S]), w[0]);
        int d = rx;
        for (; d >= 8; d -= 8) {  // loads of 8 taps in flight, adds in scipy's order
            double lo[8], hi[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                lo[u] = ct::to_f64(__ldg(col + ct::clampi(i - (d - u), 0, nx - 1) * S));
                hi[u] = ct::to_f64(__ldg(col + ct::clampi(i + (d - u), 0, nx - 1) * S));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(lo[u], hi[u]), w[d - u]));
        }
        for (; d >= 1; --d) {
            const double sm = __dadd_rn(ct::to_f64(col[ct::clampi(i - d, 0, nx - 1) * S]),
                                        ct::to_f64(col[ct::clampi(i + d, 0, nx - 1) * S]));
            acc = __dadd_rn(acc, __dmul_rn(sm, w[d]));
        }
        P1[e] = acc;
    }
}

// Same phase 1 for nz % 32 == 0, rx <= 64: a warp's 32 values share (entry,
// tt) and read consecutive kk, so the warp first stages the (2rx+1) x 32 raw
// values of its taps in SMEM (one 32-element row chunk per lane and load
// round, all in flight together) and then runs scipy's accumulation from SMEM
// -- the per-thread form waited on one memory round trip per 8 taps.
constexpr int FXR = 64;  // max rx of the staged form
template <typename Traw>
__global__ void __launch_bounds__(128) fix_p1s(const Traw *__restrict__ raw, i64 nx, i64 ny, i64 nz,
                                               const double *__restrict__ w, int rx, int ry,
                                               const unsigned long long *__restrict__ fix, long long cap,
                                               long long capF, double *__restrict__ P1) {
    __shared__ Traw buf[4][(2 * FXR + 1) * 32];
    __shared__ double ws[FXR + 1];  // the taps, read by every lane at every step
    for (int d = threadIdx.x; d <= rx; d += blockDim.x) ws[d] = w[d];
    __syncthreads();
    const long long F = min(min((long long)fix[0], cap), capF);
    const i64 RJ = 2 * ry + 1, per = RJ * nz, S = ny * nz, tot = F * per;
    const unsigned lane = threadIdx.x & 31;
    Traw *b = buf[threadIdx.x >> 5];
    const int nr = 2 * rx + 1;
    for (i64 e0 = blockIdx.x * (i64)blockDim.x + (threadIdx.x & ~31u); e0 < tot; e0 += (i64)gridDim.x * blockDim.x) {
        const i64 f = e0 / per, rem = e0 - f * per, tt = rem / nz, kk0 = rem - tt * nz;  // kk0 % 32 == 0
        const i64 p = (i64)fix[2 + f];
        const i64 j = (p / nz) % ny, i = p / S;
        const i64 jj = ct::clampi(j + tt - ry, 0, ny - 1);
        const Traw *col = raw + jj * nz + kk0;
        // lane r stages tap row r (clamped), 32 consecutive values
        for (int r = (int)lane; r < nr; r += 32) {
            const Traw *src = col + ct::clampi(i - rx + r, 0, nx - 1) * S;
            if constexpr (sizeof(Traw) == 1) {
                const uint4 a = __ldg((const uint4 *)src), c = __ldg((const uint4 *)src + 1);
                *(uint4 *)(b + r * 32) = a;
                *(uint4 *)(b + r * 32 + 16) = c;
            } else {
#pragma unroll
                for (int q = 0; q < 32; ++q) b[r * 32 + q] = src[q];
            }
        }
        __syncwarp();
        const Traw *cb = b + lane;
        double acc = __dmul_rn(ct::u2d(cb[rx * 32]), ws[0]);
#pragma unroll 4
        for (int d = rx; d >= 1; --d)
            acc = __dadd_rn(acc, __dmul_rn(ct::pair_f64(cb[(rx - d) * 32], cb[(rx + d) * 32]), ws[d]));
        if (e0 + lane < tot) P1[e0 + lane] = acc;
        __syncwarp();
    }
}

// phases 2+3: one CTA (nz threads) per entry: P2 line in SMEM, then pass z +
// residual at the voxel
template <typename Traw, typename Tq>
__global__ void fix_p2q(const Traw *__restrict__ raw, i64 nz, const double *__restrict__ wy, int ry,
                        const double *__restrict__ wz, int rz, const unsigned long long *__restrict__ fix,
                        long long cap, long long capF, const double *__restrict__ P1, Tq *__restrict__ q_out) {
    __shared__ double line[128];
    const long long F = min(min((long long)fix[0], cap), capF);
    const int kk = threadIdx.x;
    for (long long f = blockIdx.x; f < F; f += gridDim.x) {
        __syncthreads();
        if (kk < nz) {
            const double *c = P1 + f * (2 * ry + 1) * nz + kk;
            double acc = __dmul_rn(c[(i64)ry * nz], wy[0]);
            int d = ry;
            for (; d >= 8; d -= 8) {  // 16 loads in flight, adds in scipy's order
                double lo[8], hi[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    lo[u] = c[(i64)(ry - (d - u)) * nz];
                    hi[u] = c[(i64)(ry + (d - u)) * nz];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(lo[u], hi[u]), wy[d - u]));
            }
            for (; d >= 1; --d)
                acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(c[(i64)(ry - d) * nz], c[(i64)(ry + d) * nz]), wy[d]));
            line[kk] = acc;
        }
        __syncthreads();
        if (kk == 0) {
            const i64 p = (i64)fix[2 + f], k = p % nz;
            double acc = __dmul_rn(line[k], wz[0]);
            for (int d = rz; d >= 1; --d)
                acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(line[ct::clampi(k - d, 0, nz - 1)],
                                                         line[ct::clampi(k + d, 0, nz - 1)]), wz[d]));
            const double dd = __dadd_rn(ct::to_f64(raw[p]), -acc);
            q_out[p] = (Tq)rint(dd < 0.0 ? 0.0 : dd);
        }
    }
}

// Same phases 2+3 with the entry's whole P1 cone ((2ry+1) x nz doubles)
// copied into SMEM by cp.async first (every load in flight at once; the
// per-thread form waited one L2 round trip per 8 taps), nz % 2 == 0.
// Entries past the scratch (f >= capF; gauss_fixup's job in the other
// configurations) build their cone here from raw, in the same order.
template <typename Traw, typename Tq>
__global__ void __launch_bounds__(128) fix_p2q_s(const Traw *__restrict__ raw, i64 nx, i64 ny, i64 nz,
                                                 const double *__restrict__ wx, int rx, const double *__restrict__ wy,
                                                 int ry, const double *__restrict__ wz, int rz,
                                                 const unsigned long long *__restrict__ fix, long long cap,
                                                 long long capF, const double *__restrict__ P1, Tq *__restrict__ q_out) {
    extern __shared__ __align__(16) double cone[];  // [(2ry+1) * nz], then line[nz]
    const long long cnt = min((long long)fix[0], cap), F = min(cnt, capF);
    const int per = (2 * ry + 1) * (int)nz;
    double *line = cone + per;
    const int kk = threadIdx.x;
    for (long long f = blockIdx.x; f < cnt; f += gridDim.x) {
        __syncthreads();
        if (f < F) {
            const double *src = P1 + f * per;
            for (int q = threadIdx.x; q < per / 2; q += blockDim.x) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(cone + 2 * q);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + 2 * q) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
        } else {
            const i64 p = (i64)fix[2 + f], j = (p / nz) % ny, i = p / (ny * nz), S = ny * nz;
            for (int e = threadIdx.x; e < per; e += blockDim.x) {
                const i64 jj = ct::clampi(j + e / nz - ry, 0, ny - 1);
                const Traw *col = raw + jj * nz + e % nz;
                double acc = __dmul_rn(ct::to_f64(col[i * S]), wx[0]);
                for (int d = rx; d >= 1; --d)
                    acc = __dadd_rn(acc, __dmul_rn(ct::pair_f64(col[ct::clampi(i - d, 0, nx - 1) * S],
                                                                col[ct::clampi(i + d, 0, nx - 1) * S]), wx[d]));
                cone[e] = acc;
            }
        }
        __syncthreads();
        if (kk < nz) {
            const double *c = cone + kk;
            double acc = __dmul_rn(c[ry * nz], wy[0]);
            for (int d = ry; d >= 1; --d)
                acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(c[(ry - d) * nz], c[(ry + d) * nz]), wy[d]));
            line[kk] = acc;
        }
        __syncthreads();
        if (kk == 0) {
            const i64 p = (i64)fix[2 + f], k = p % nz;
            double acc = __dmul_rn(line[k], wz[0]);
            for (int d = rz; d >= 1; --d)
                acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(line[ct::clampi(k - d, 0, nz - 1)],
                                                         line[ct::clampi(k + d, 0, nz - 1)]), wz[d]));
            const double dd = __dadd_rn(ct::to_f64(raw[p]), -acc);
            q_out[p] = (Tq)rint(dd < 0.0 ? 0.0 : dd);
        }
    }
}

// Fix-list overflow (fix[1] != 0: more voxels near a rounding boundary than
// the list holds -- adversarial inputs only): the whole q is recomputed in
// scipy's exact order, in stream, without a host round trip.  One cooperative
// launch; every CTA reads the same flag, so in the normal case all of them
// return at once.  Otherwise three grid-stride passes (x: raw -> p1, y: p1 ->
// p2, z: p2 -> residual -> q) separated by grid syncs, each voxel computed as
// ct_gaussian_residual does (ref denoise.py:84-86; the fast path's partial
// results in `work` are dead by now).
template <typename Traw>
__global__ void __launch_bounds__(256) k1_overflow_exact(const Traw *__restrict__ raw, i64 nx, i64 ny, i64 nz,
                                                         const double *__restrict__ w, int rx, int ry, int rz,
                                                         const unsigned long long *__restrict__ fix,
                                                         double *__restrict__ p1, double *__restrict__ p2,
                                                         Traw *__restrict__ q_out) {
    if (fix[1] == 0) return;
    namespace cg = cooperative_groups;
    const cg::grid_group grid = cg::this_grid();
    const double *wx = w, *wy = w + rx + 1, *wz = wy + ry + 1;
    const i64 N = nx * ny * nz, S = ny * nz;
    const i64 t0 = blockIdx.x * (i64)blockDim.x + threadIdx.x, dt = (i64)gridDim.x * blockDim.x;
    for (i64 p = t0; p < N; p += dt) {
        const i64 i = p / S;
        const Traw *col = raw + (p - i * S);
        double acc = __dmul_rn(ct::to_f64(col[i * S]), wx[0]);
        for (int d = rx; d >= 1; --d)
            acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(ct::to_f64(col[ct::clampi(i - d, 0, nx - 1) * S]),
                                                     ct::to_f64(col[ct::clampi(i + d, 0, nx - 1) * S])), wx[d]));
        p1[p] = acc;
    }
    grid.sync();
    for (i64 p = t0; p < N; p += dt) {
        const i64 j = (p / nz) % ny;
        const double *col = p1 + (p - j * nz);
        double acc = __dmul_rn(col[j * nz], wy[0]);
        for (int d = ry; d >= 1; --d)
            acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(col[ct::clampi(j - d, 0, ny - 1) * nz],
                                                     col[ct::clampi(j + d, 0, ny - 1) * nz]), wy[d]));
        p2[p] = acc;
    }
    grid.sync();
    for (i64 p = t0; p < N; p += dt) {
        const i64 k = p % nz;
        const double *line = p2 + (p - k);
        double acc = __dmul_rn(line[k], wz[0]);
        for (int d = rz; d >= 1; --d)
            acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(line[ct::clampi(k - d, 0, nz - 1)],
                                                     line[ct::clampi(k + d, 0, nz - 1)]), wz[d]));
        const double dd = __dadd_rn(ct::to_f64(raw[p]), -acc);
        q_out[p] = (Traw)rint(dd < 0.0 ? 0.0 : dd);
    }
}

// fix-up of a certified fast path: grid-wide phases for the first capF
// entries (scratch = the dead K1 workspace), per-CTA fallback for the rest
template <typename Traw>
int launch_fixup(const Traw *raw, i64 nx, i64 ny, i64 nz, const double *w, int rx, int ry, int rz, void *work,
                 size_t work_bytes, const unsigned long long *fix, long long cap, Traw *q, cudaStream_t s) {
    const double *wx = w, *wy = w + rx + 1, *wz = wy + ry + 1;
    const i64 per = (2 * (i64)ry + 1) * nz;
    const long long capF = nz <= 128 ? (long long)(work_bytes / ((size_t)per * sizeof(double))) : 0;
    double *P1 = (double *)work;
    if (nz % 32 == 0 && rx <= FXR && ((uintptr_t)raw & 15) == 0)
        fix_p1s<Traw><<<CT_NUM_SMS * 16, 128, 0, s>>>(raw, nx, ny, nz, wx, rx, ry, fix, cap, capF, P1);
    else
        fix_p1<Traw><<<CT_NUM_SMS * 8, 256, 0, s>>>(raw, nx, ny, nz, wx, rx, ry, fix, cap, capF, P1);
    const size_t csm = ((size_t)per + nz) * sizeof(double);
    if (nz % 2 == 0 && nz <= 128 && csm <= 200 * 1024) {
        // (also the entries past the scratch: no gauss_fixup launch)
        cudaFuncSetAttribute(fix_p2q_s<Traw, Traw>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
        fix_p2q_s<Traw, Traw><<<CT_NUM_SMS * 2, 128, csm, s>>>(raw, nx, ny, nz, wx, rx, wy, ry, wz, rz, fix, cap, capF,
                                                               P1, q);
        if (int st = ct::check_launch("fixup phases")) return st;
    } else {
        fix_p2q<Traw, Traw><<<CT_NUM_SMS * 2, 128, 0, s>>>(raw, nz, wy, ry, wz, rz, fix, cap, capF, P1, q);
        if (int st = ct::check_launch("fixup phases")) return st;
        const size_t fsm = ((size_t)(2 * ry + 1) * nz + nz) * sizeof(double);
        cudaFuncSetAttribute(gauss_fixup<Traw, Traw>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
        gauss_fixup<Traw, Traw><<<CT_NUM_SMS, 256, fsm, s>>>(raw, nx, ny, nz, w, rx, ry, rz, fix, cap, q, capF);
        if (int st = ct::check_launch("gauss_fixup")) return st;
    }
    // list overflow -> exact recompute in stream (returns at once otherwise)
    double *p1 = (double *)work, *p2 = p1 + nx * ny * nz;
    void *args[] = {(void *)&raw, (void *)&nx, (void *)&ny, (void *)&nz, (void *)&w, (void *)&rx, (void *)&ry,
                    (void *)&rz, (void *)&fix, (void *)&p1, (void *)&p2, (void *)&q};
    if (cudaLaunchCooperativeKernel((const void *)k1_overflow_exact<Traw>, dim3(CT_NUM_SMS * 2), dim3(256), args, 0,
                                    s) != cudaSuccess) {
        ct::set_error("k1_overflow_exact: cooperative launch failed (%s)", cudaGetErrorString(cudaGetLastError()));
        return CT_ERR_CUDA;
    }
    return CT_OK;
}

template <typename Traw>
int gaussian_q_fast(const Traw *raw, i64 nx, i64 ny, i64 nz, const double *w, int rx, int ry, int rz, double *work,
                    Traw *q, unsigned long long *fix, long long cap, double maxv, double eps_override,
                    cudaStream_t s) {
    const i64 N = nx * ny * nz;
    double *p1 = work, *p2 = work + N;
    const double *wx = w, *wy = w + rx + 1, *wz = wy + ry + 1;
    cudaMemsetAsync(fix, 0, 2 * sizeof(unsigned long long), s);
    if (int st = pass_strided<Traw, true>(raw, p1, 1, nx, ny * nz, wx, rx, s)) return st;
    if (int st = pass_strided<double, true>(p1, p2, nx, ny, nz, wy, ry, s)) return st;
    int S = (int)(((nz + B - 1) / B) * B + 2 * rz);
    if ((S & 1) == 0) S += 1;
    const size_t sm = ((size_t)C * S + rz + 1) * sizeof(double);
    const int nb = (int)((nz + B - 1) / B);
    const double u = 1.1102230246251565e-16;  // 2^-53
    Cert cert{eps_override > 0.0 ? eps_override : 4.0 * (2.0 * (rx + ry + rz) + 11.0) * u * maxv, fix, cap};
    auto kc = nz == 64 ? gauss_contig<Traw, Traw, true, 64>
              : nz == 32 ? gauss_contig<Traw, Traw, true, 32>
              : nz == 128 ? gauss_contig<Traw, Traw, true, 128> : gauss_contig<Traw, Traw, true, 0>;
    cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT);
    kc<<<(unsigned)((nx * ny + C - 1) / C), dim3(C, nb), sm, s>>>(p2, nx * ny, (int)nz, wz, rz, S, C, raw, nullptr,
                                                                 nullptr, q, cert);
    if (int st = ct::check_launch("gauss_contig fma")) return st;
    return launch_fixup<Traw>(raw, nx, ny, nz, w, rx, ry, rz, work, (size_t)2 * N * sizeof(double), fix, cap, q, s);
}

}  // namespace

int ct_gaussian_q_tc(const void *raw, int dtype, int64_t nx, int64_t ny, int64_t nz, const double *w, int rx, int ry,
                     int rz, void *work, void *q, unsigned long long *fix, int64_t cap, double eps_override,
                     cudaStream_t s);

bool ct_gaussian_q_tc_fits(int dtype, int64_t nx, int64_t ny, int64_t nz, int rx, int ry, int rz);

// K1 fast-path selection (per call): 0 auto (tensor cores when the shape
// fits, else FP64 FMA), 1 FP64 FMA, 2 tensor cores only.
extern "C" int ct_k1_path(int dtype, int64_t nx, int64_t ny, int64_t nz, int rx, int ry, int rz, int path) {
    if (path != 1 && ct_gaussian_q_tc_fits(dtype, nx, ny, nz, rx, ry, rz)) return 2;
    return 1;
}

extern "C" int ct_gaussian_q(const void *raw, int dtype, int64_t nx, int64_t ny, int64_t nz, const double *w, int rx,
                             int ry, int rz, void *work, void *q_out, unsigned long long *fix, int64_t fix_cap,
                             double eps_override, int path, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (path < 0 || path > 2) {
        ct::set_error("k1 path must be 0 (auto), 1 (FP64 FMA) or 2 (tensor cores)");
        return CT_ERR_PARAM;
    }
    // the fast kernels need the tiled paths (see pass_strided / pass_contig) and every axis filtered
    const bool fast = rx >= 0 && ry >= 0 && rz >= 0 && nz <= 128 &&
                      ((size_t)(TMAX + 2 * (rx > ry ? rx : ry)) * C + 64) * sizeof(double) <= SMEM_LIMIT &&
                      nx * ny <= (1ll << 31) && (((nz + B - 1) / B) * B + 2 * rz + 1) * C * 8 < (i64)SMEM_LIMIT &&
                      ((size_t)(2 * ry + 1) * nz + nz) * sizeof(double) <= SMEM_LIMIT && nx <= 65535 * 128 &&
                      ny <= 65535 * 128;
    if (!fast || (dtype != CT_U8 && dtype != CT_U16)) {
        if (fix) cudaMemsetAsync(fix, 0, 2 * sizeof(unsigned long long), s);
        return ct_gaussian_residual(raw, dtype, nx, ny, nz, w, rx, ry, rz, work, nullptr, nullptr, q_out, dtype,
                                    stream);
    }
    // tensor-core path (k_gauss_tc.cu) unless disabled or the shape does not fit
    if (path != 1) {
        const int st = ct_gaussian_q_tc(raw, dtype, nx, ny, nz, w, rx, ry, rz, work, q_out, fix, fix_cap,
                                        eps_override, s);
        if (st == CT_OK) {
            const size_t wb = (size_t)2 * nx * ny * nz * sizeof(double);
            return dtype == CT_U8 ? launch_fixup<uint8_t>((const uint8_t *)raw, nx, ny, nz, w, rx, ry, rz, work, wb,
                                                          fix, fix_cap, (uint8_t *)q_out, s)
                                  : launch_fixup<uint16_t>((const uint16_t *)raw, nx, ny, nz, w, rx, ry, rz, work,
                                                           wb, fix, fix_cap, (uint16_t *)q_out, s);
        }
        if (st != CT_ERR_UNSUPPORTED || path == 2) {
            if (st == CT_ERR_UNSUPPORTED) ct::set_error("tensor-core K1 does not support this shape");
            return st;
        }
    }
    if (dtype == CT_U8)
        return gaussian_q_fast<uint8_t>((const uint8_t *)raw, nx, ny, nz, w, rx, ry, rz, (double *)work,
                                        (uint8_t *)q_out, fix, fix_cap, 255.0, eps_override, s);
    return gaussian_q_fast<uint16_t>((const uint16_t *)raw, nx, ny, nz, w, rx, ry, rz, (double *)work,
                                     (uint16_t *)q_out, fix, fix_cap, 65535.0, eps_override, s);
}
