// k_morph.cu -- K4: threshold + morphological closing.
//
// Replaces ref segment.py:204 (mask = rint(v) > t) and segment.py:166-189
// (ball closing: pad r+1 zeros, binary_dilation, binary_erosion, crop), i.e.
// closing on the infinite zero domain:
//   D(q) = OR_{o in ball} M(q+o)   for q within r of the volume (M = 0 outside)
//   out(p) = AND_{o in ball} D(p+o)
// r == 1 (the default 6-cross): one fused tile kernel, halo 2 staged in SMEM,
// D computed for the tile + 1 shell, then the erosion.  r > 1: two passes
// through an extended (n+2r)^3 byte buffer.
#include "ct_common.cuh"

namespace {

constexpr int TK = 32, TJ = 8, TI = 4;

__device__ __forceinline__ i64 threshold_of(const int64_t *res, i64 t_host, bool &empty) {
    empty = false;
    if (!res) return t_host;
    if (res[CT_OTSU_STATUS] != 0) empty = true;
    return res[CT_OTSU_T];
}

template <typename T>
__global__ void __launch_bounds__(TK *TJ) close1_kernel(const T *__restrict__ in, i64 nx, i64 ny, i64 nz,
                                                        const int64_t *__restrict__ otsu, i64 t_host,
                                                        uint8_t *__restrict__ out) {
    __shared__ uint8_t m[TI + 4][TJ + 4][TK + 4];
    __shared__ uint8_t d[TI + 2][TJ + 2][TK + 2];
    bool empty;
    const i64 t = threshold_of(otsu, t_host, empty);
    const int tid = threadIdx.y * TK + threadIdx.x, nth = TK * TJ;
    const i64 tk = (nz + TK - 1) / TK, tj = (ny + TJ - 1) / TJ, ti = (nx + TI - 1) / TI;
    const i64 ntiles = tk * tj * ti;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 k0 = (tile % tk) * TK, j0 = ((tile / tk) % tj) * TJ, i0 = (tile / (tk * tj)) * TI;
        if (empty) {
            for (int idx = tid; idx < TI * TJ * TK; idx += nth) {
                const int kk = idx % TK, jj = (idx / TK) % TJ, ii = idx / (TK * TJ);
                const i64 i = i0 + ii, j = j0 + jj, k = k0 + kk;
                if (i < nx && j < ny && k < nz) out[(i * ny + j) * nz + k] = 0;
            }
            continue;
        }
        __syncthreads();
        for (int idx = tid; idx < (TI + 4) * (TJ + 4) * (TK + 4); idx += nth) {
            const int kk = idx % (TK + 4), jj = (idx / (TK + 4)) % (TJ + 4), ii = idx / ((TK + 4) * (TJ + 4));
            const i64 i = i0 + ii - 2, j = j0 + jj - 2, k = k0 + kk - 2;
            uint8_t v = 0;
            if (i >= 0 && i < nx && j >= 0 && j < ny && k >= 0 && k < nz) v = ct::above(in[(i * ny + j) * nz + k], t);
            m[ii][jj][kk] = v;
        }
        __syncthreads();
        for (int idx = tid; idx < (TI + 2) * (TJ + 2) * (TK + 2); idx += nth) {
            const int c = idx % (TK + 2), b = (idx / (TK + 2)) % (TJ + 2), a = idx / ((TK + 2) * (TJ + 2));
            const int A = a + 1, Bj = b + 1, Cc = c + 1;
            d[a][b][c] = m[A][Bj][Cc] | m[A - 1][Bj][Cc] | m[A + 1][Bj][Cc] | m[A][Bj - 1][Cc] | m[A][Bj + 1][Cc] |
                         m[A][Bj][Cc - 1] | m[A][Bj][Cc + 1];
        }
        __syncthreads();
        const int c = threadIdx.x, b = threadIdx.y;
        const i64 j = j0 + b, k = k0 + c;
        if (j < ny && k < nz) {
#pragma unroll
            for (int a = 0; a < TI; ++a) {
                const i64 i = i0 + a;
                if (i >= nx) break;
                const int A = a + 1, Bj = b + 1, Cc = c + 1;
                out[(i * ny + j) * nz + k] = d[A][Bj][Cc] & d[A - 1][Bj][Cc] & d[A + 1][Bj][Cc] & d[A][Bj - 1][Cc] &
                                             d[A][Bj + 1][Cc] & d[A][Bj][Cc - 1] & d[A][Bj][Cc + 1];
            }
        }
    }
}

template <typename T>
__global__ void threshold_kernel(const T *__restrict__ in, i64 n, const int64_t *__restrict__ otsu, i64 t_host,
                                 uint8_t *__restrict__ out) {
    bool empty;
    const i64 t = threshold_of(otsu, t_host, empty);
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
        out[p] = empty ? 0 : ct::above(in[p], t);
}

// r > 1: dilation into the extended domain, then erosion.
template <typename T>
__global__ void dilate_ext(const T *__restrict__ in, i64 nx, i64 ny, i64 nz, int r, const int64_t *__restrict__ otsu,
                           i64 t_host, uint8_t *__restrict__ ext) {
    bool empty;
    const i64 t = threshold_of(otsu, t_host, empty);
    const i64 ex = nx + 2 * r, ey = ny + 2 * r, ez = nz + 2 * r, n = ex * ey * ez;
    for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < n; q += (i64)gridDim.x * blockDim.x) {
        const i64 c = q % ez - r, b = (q / ez) % ey - r, a = q / (ey * ez) - r;
        uint8_t v = 0;
        if (!empty) {
            for (int da = -r; da <= r && !v; ++da)
                for (int db = -r; db <= r && !v; ++db)
                    for (int dc = -r; dc <= r && !v; ++dc) {
                        if (da * da + db * db + dc * dc > r * r) continue;
                        const i64 i = a + da, j = b + db, k = c + dc;
                        if (i >= 0 && i < nx && j >= 0 && j < ny && k >= 0 && k < nz)
                            v = ct::above(in[(i * ny + j) * nz + k], t);
                    }
        }
        ext[q] = v;
    }
}

__global__ void erode_ext(const uint8_t *__restrict__ ext, i64 nx, i64 ny, i64 nz, int r, uint8_t *__restrict__ out) {
    const i64 ey = ny + 2 * r, ez = nz + 2 * r, n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
        uint8_t v = 1;
        for (int da = -r; da <= r && v; ++da)
            for (int db = -r; db <= r && v; ++db)
                for (int dc = -r; dc <= r && v; ++dc) {
                    if (da * da + db * db + dc * dc > r * r) continue;
                    v = ext[((i + r + da) * ey + (j + r + db)) * ez + (k + r + dc)];
                }
        out[p] = v;
    }
}

// ---------------------------------------------------------------------------
// r == 1, nz <= 64: z-rows as 64-bit words.
//   pack_rows   : M(i,j) = threshold bits of row (i,j) (two ballots per row).
//   close1_bits : D(q) = OR of the 6-cross of M around q, E(p) = AND of the
//                 6-cross of D around p, with the out-of-volume D values of the
//                 infinite zero domain: D(i=-1,j) = M(0,j), D(i,j,k=-1) =
//                 M(i,j,0), ... (the only in-volume cross neighbour).  One
//                 thread per row, 13 word loads (L2-resident: N/8 bytes),
//                 bytes written through an SMEM transpose for coalescing.
// ---------------------------------------------------------------------------
template <typename T, typename R>
__global__ void __launch_bounds__(256) pack_rows(const T *__restrict__ in, i64 nrows, int nz,
                                                 const int64_t *__restrict__ otsu, i64 t_host,
                                                 R *__restrict__ rows) {
    bool empty;
    const i64 t = threshold_of(otsu, t_host, empty);
    const unsigned lane = threadIdx.x & 31;
    const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 r0 = warp * 32; r0 < nrows; r0 += nwarps * 32) {
        R mine = 0;
        const int nr = (int)min((i64)32, nrows - r0);
        for (int r = 0; r < nr; ++r) {
            const T *row = in + (r0 + r) * nz;
            R word = 0;
#pragma unroll
            for (int q = 0; q < ct::rbits<R>() / 32; ++q) {
                const int k = (int)lane + 32 * q;
                const bool a = !empty && k < nz && ct::above(row[k], t);
                word |= (R)__ballot_sync(0xffffffffu, a) << (32 * q);
            }
            if ((int)lane == r) mine = word;
        }
        if ((int)lane < nr) rows[r0 + lane] = mine;
    }
}

// u8, nz % 16 == 0 (<= 128): one thread per row, 16-byte loads, SIMD byte compares
// NZ > 0: compile-time row length (unrolled, constant shifts); v > t per byte
// as the carry out of v + (255 - t): an IADD and a majority LOP3 per 4 bytes
// (__vcmpgtu4 is emulated)
template <typename R, int NZ = 0>
__global__ void __launch_bounds__(256) pack_rows_u8v(const uint8_t *__restrict__ in, i64 nrows, int nz_,
                                                     const int64_t *__restrict__ otsu, i64 t_host,
                                                     R *__restrict__ rows) {
    const int nz = NZ > 0 ? NZ : nz_;
    bool empty;
    const i64 t = threshold_of(otsu, t_host, empty);
    const bool all = !empty && t < 0, none = empty || t >= 255;
    const uint32_t kb = (uint32_t)(255 - (all || none ? 0 : t)) * 0x01010101u;  // 255 - t per byte
    const uint32_t k7 = kb & 0x7f7f7f7fu;
    for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < nrows; r += (i64)gridDim.x * blockDim.x) {
        R w = 0;
        if (all) w = ct::rmask<R>(nz);
        else if (!none) {
            const uint4 *src = (const uint4 *)(in + r * nz);
#pragma unroll
            for (int c = 0; c < (NZ > 0 ? NZ / 16 : 8); ++c) {
                if (NZ == 0 && c >= nz / 16) break;
                const uint4 v = __ldg(src + c);
                const uint32_t x[4] = {v.x, v.y, v.z, v.w};
                uint32_t piece = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t cin = (x[q] & 0x7f7f7f7fu) + k7;  // bit 7 of each byte: the carry into bit 7
                    const uint32_t g = ((x[q] & kb) | ((x[q] | kb) & cin)) & 0x80808080u;  // carry out: v > t
                    piece |= (((g >> 7) * 0x10204080u) >> 28) << (4 * q);
                }
                w |= (R)piece << (16 * c);
            }
        }
        rows[r] = w;
    }
}

template <typename R>
__global__ void __launch_bounds__(256) close1_bits(const R *__restrict__ rows, i64 nx, i64 ny, int nz,
                                                   uint8_t *__restrict__ out, R *__restrict__ out_rows,
                                                   const ct::FastDiv fny) {
    __shared__ __align__(16) uint8_t stage[8][32 * ct::rbits<R>()];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const R kmask = ct::rmask<R>(nz);
    const R top = (R)1 << (nz - 1);
    const i64 nrows = nx * ny;
    const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
    // rows = nx ny < 2^31 (checked by the caller): 32-bit row coordinates by
    // multiply-shift (fny built on the host)
    const int inx = (int)nx, iny = (int)ny;
    auto M = [&](int ii, int jj) -> R {
        return (ii >= 0 && ii < inx && jj >= 0 && jj < iny) ? rows[(i64)ii * iny + jj] : (R)0;
    };
    auto sh = [](R w) { return w | (w << 1) | (w >> 1); };
    for (i64 r0 = warp * 32; r0 < nrows; r0 += nwarps * 32) {
        const i64 r = r0 + lane;
        R e = 0;
        if (r < nrows) {
            const int i = (int)fny.div((uint32_t)r), j = (int)r - i * iny;
            if (i >= 2 && i < inx - 2 && j >= 2 && j < iny - 2) {
                // interior (all but a 2-row rim): the 13 rows at fixed offsets, no bounds tests
                const R *p = rows + r;
                const R m = p[0], xm1 = p[-iny], xp1 = p[iny], ym1 = p[-1], yp1 = p[1];
                const R xm2 = p[-2 * iny], xp2 = p[2 * iny], ym2 = p[-2], yp2 = p[2];
                const R mm = p[-iny - 1], mp = p[-iny + 1], pm = p[iny - 1], pp = p[iny + 1];
                const R d = (sh(m) | xm1 | xp1 | ym1 | yp1) & kmask;
                const R dxm = (sh(xm1) | xm2 | m | mm | mp) & kmask, dxp = (sh(xp1) | xp2 | m | pm | pp) & kmask;
                const R dym = (sh(ym1) | ym2 | m | mm | pm) & kmask, dyp = (sh(yp1) | yp2 | m | mp | pp) & kmask;
                const R dkm = ((d << 1) | (m & (R)1)) & kmask, dkp = (d >> 1) | (m & top);
                e = d & dxm & dxp & dym & dyp & dkm & dkp;
                if (out_rows) out_rows[r] = e;
            } else {
            // the 13 distinct rows of the two-step cross, each loaded once
            const R m = rows[r];
            const R xm1 = M(i - 1, j), xp1 = M(i + 1, j), ym1 = M(i, j - 1), yp1 = M(i, j + 1);
            const R xm2 = M(i - 2, j), xp2 = M(i + 2, j), ym2 = M(i, j - 2), yp2 = M(i, j + 2);
            const R mm = M(i - 1, j - 1), mp = M(i - 1, j + 1), pm = M(i + 1, j - 1), pp = M(i + 1, j + 1);
            const R d = (sh(m) | xm1 | xp1 | ym1 | yp1) & kmask;
            // cross neighbours of D; outside the volume D equals the single in-volume M
            const R dxm = i > 0 ? (sh(xm1) | xm2 | m | mm | mp) & kmask : m;
            const R dxp = i < inx - 1 ? (sh(xp1) | xp2 | m | pm | pp) & kmask : m;
            const R dym = j > 0 ? (sh(ym1) | ym2 | m | mm | pm) & kmask : m;
            const R dyp = j < iny - 1 ? (sh(yp1) | yp2 | m | mp | pp) & kmask : m;
            const R dkm = ((d << 1) | (m & (R)1)) & kmask;    // D at k-1; k=-1 -> M(k=0)
            const R dkp = (d >> 1) | (m & top);               // D at k+1; k=nz -> M(k=nz-1)
            e = d & dxm & dxp & dym & dyp & dkm & dkp;
            if (out_rows) out_rows[r] = e;
            }
        }
        if (out) {
            // bits -> bytes via SMEM, then a coalesced copy of the warp's 32 rows
            uint8_t *st = stage[wid];
            if (nz % 16 == 0) {  // 16-byte SMEM stores (a plain 4-byte loop is 16-way bank conflicted)
                for (int k = 0; k < nz; k += 16) {
                    uint32_t b4[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) b4[q] = ((unsigned)((e >> (k + 4 * q)) & 0xF) * 0x00204081u) & 0x01010101u;
                    *reinterpret_cast<uint4 *>(st + lane * nz + k) = make_uint4(b4[0], b4[1], b4[2], b4[3]);
                }
            } else {
                for (int k = 0; k < nz; k += 4) {
                    const unsigned nib = (unsigned)((e >> k) & 0xF);
                    const uint32_t bytes = ((nib * 0x00204081u) & 0x01010101u);
                    *reinterpret_cast<uint32_t *>(st + lane * nz + k) = bytes;  // nz % 4 == 0 guaranteed by caller
                }
            }
            __syncwarp();
            const int nr = (int)min((i64)32, nrows - r0);
            const int nbytes = nr * nz;
            uint8_t *dst = out + r0 * nz;
            for (int b = lane * 16; b < nbytes; b += 32 * 16) {
                if (b + 16 <= nbytes) *reinterpret_cast<uint4 *>(dst + b) = *reinterpret_cast<const uint4 *>(st + b);
                else
                    for (int q = b; q < nbytes; ++q) dst[q] = st[q];
            }
            __syncwarp();
        }
    }
}

template <typename T>
int threshold_close(const T *in, i64 nx, i64 ny, i64 nz, const int64_t *otsu, i64 t_host, int r, uint8_t *out,
                    uint8_t *work, cudaStream_t s, void *rows_out = nullptr) {
    const i64 n = nx * ny * nz;
    if (r == 0) {
        threshold_kernel<T><<<ct::grid_for(n, 256), 256, 0, s>>>(in, n, otsu, t_host, out);
        return ct::check_launch("threshold");
    }
    if (r == 1 && nz <= 128 && nz % 4 == 0 && work && ((uintptr_t)out & 15) == 0 && nx * ny < (1ll << 31)) {
        const i64 nrows = nx * ny;
        auto run = [&](auto tag) -> int {
            using R = decltype(tag);
            R *rows = (R *)work;
            if (sizeof(T) == 1 && nz % 16 == 0 && ((uintptr_t)in & 15) == 0)
            {
                auto k = nz == 64 ? pack_rows_u8v<R, 64> : nz == 32 ? pack_rows_u8v<R, 32>
                         : nz == 128 ? pack_rows_u8v<R, 128> : pack_rows_u8v<R, 0>;
                k<<<ct::grid_for(nrows, 256, CT_NUM_SMS * 16), 256, 0, s>>>((const uint8_t *)in, nrows, (int)nz, otsu,
                                                                          t_host, rows);
            }
            else
                pack_rows<T, R><<<ct::grid_for(nrows, 256, CT_NUM_SMS * 16), 256, 0, s>>>(in, nrows, (int)nz, otsu,
                                                                                          t_host, rows);
            if (int st = ct::check_launch("pack_rows")) return st;
            close1_bits<R><<<ct::grid_for(nrows, 256, CT_NUM_SMS * 16), 256, 0, s>>>(rows, nx, ny, (int)nz, out,
                                                                                      (R *)rows_out,
                                                                                      ct::FastDiv((uint32_t)ny));
            return ct::check_launch("close1_bits");
        };
        return nz <= 64 ? run((u64)0) : run((ct::u128)0);
    }
    if (r == 1) {
        const i64 tiles = ((nz + TK - 1) / TK) * ((ny + TJ - 1) / TJ) * ((nx + TI - 1) / TI);
        const int grid = (int)min(tiles, (i64)CT_NUM_SMS * 8);
        close1_kernel<T><<<grid, dim3(TK, TJ), 0, s>>>(in, nx, ny, nz, otsu, t_host, out);
        return ct::check_launch("close1");
    }
    if (!work) {
        ct::set_error("closing radius %d needs a workspace", r);
        return CT_ERR_PARAM;
    }
    const i64 ne = (nx + 2 * r) * (ny + 2 * r) * (nz + 2 * r);
    dilate_ext<T><<<ct::grid_for(ne, 256), 256, 0, s>>>(in, nx, ny, nz, r, otsu, t_host, work);
    if (int st = ct::check_launch("dilate_ext")) return st;
    erode_ext<<<ct::grid_for(n, 256), 256, 0, s>>>(work, nx, ny, nz, r, out);
    return ct::check_launch("erode_ext");
}

}  // namespace

extern "C" int ct_threshold_close(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz,
                                  const int64_t *otsu_result, int64_t t_host, int radius, uint8_t *mask_out,
                                  void *work, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || radius < 0) {
        ct::set_error("bad closing arguments");
        return CT_ERR_PARAM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    CT_DISPATCH(dtype, T, {
        return threshold_close<T>((const T *)in, nx, ny, nz, otsu_result, t_host, radius, mask_out, (uint8_t *)work, s);
    });
    return CT_OK;
}

extern "C" int ct_threshold_close_rows(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz,
                                       const int64_t *otsu_result, int64_t t_host, uint8_t *mask_out, void *rows_out,
                                       void *work, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || !rows_out || !work) {
        ct::set_error("bad closing arguments");
        return CT_ERR_PARAM;
    }
    if (nz > 128 || nz % 4 != 0 || ((uintptr_t)mask_out & 15) || ((uintptr_t)rows_out & 15) ||
        nx * ny >= (1ll << 31)) {
        ct::set_error("ct_threshold_close_rows: needs nz <= 128, nz %% 4 == 0, nx ny < 2^31, 16-byte aligned outputs");
        return CT_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    CT_DISPATCH(dtype, T, {
        return threshold_close<T>((const T *)in, nx, ny, nz, otsu_result, t_host, 1, mask_out, (uint8_t *)work, s,
                                  rows_out);
    });
    return CT_OK;
}

extern "C" int ct_closing(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, int radius, uint8_t *out, void *work,
                          void *stream) {
    return ct_threshold_close(mask, CT_U8, nx, ny, nz, nullptr, 0, radius, out, work, stream);
}
