// k_edt.cu -- K8: exact anisotropic Euclidean distance transform.
//
// Replaces ref segment.py:292-304: ndimage.distance_transform_edt(~mask,
// sampling=(dx,dy,dz)) -- the distance (um) from every voxel to the nearest
// foreground voxel.  scipy forms it from an integer feature transform as
//   sqrt(((fi-i)dx)^2 + ((fj-j)dy)^2 + ((fk-k)dz)^2), summed axis 0 -> 2;
// here the nearest feature's integer offsets are carried through three
// separable passes and the distance is formed from them in exactly that order.
//
// Pass order x -> z -> y keeps every envelope sparse on vessel masks:
//   pass x : per (j,k) line along i: nearest foreground (two sweeps over a
//            register-prefetched stream).  Only columns holding foreground get
//            an offset.                                     1 B in, 2 B (di) out
//   pass z : per (i,j) line along the contiguous k: lower envelope (Felzenszwalb-
//            Huttenlocher) of (di*dx)^2 + ((k-q)*dz)^2; sites only where a
//            foreground column crosses the line.            2 B in, 4 B (dk,di) out
//   pass y : per (i,k) line along j, sites (di,dk): cost (di*dx)^2 + (dk*dz)^2,
//            output sqrt(((di*dx)^2 + (dj*dy)^2) + (dk*dz)^2).   4 B in, 8 B out
// Lines of passes x and y map to consecutive k across a warp (coalesced); pass
// z stages whole contiguous lines through SMEM.  Envelope stacks live in
// SMEM (global spill beyond the SMEM slots), top-of-stack in registers, and
// the predicates are division-free.  Arithmetic is identical to
// oracle/ct_oracle.c ora_edt, so results match it bit for bit; equidistant
// features may differ from scipy's choice in the last ulp, within the
// reference's 1e-9 um contract (ref test_acceptance.py:318-332).
#include "ct_common.cuh"

namespace {

constexpr int16_t NONE16 = INT16_MIN;
constexpr int32_t NONE32 = INT32_MIN;
constexpr int SCE = 96;  // SMEM stack entries (2 B positions) per thread (pass y)
constexpr int LT = 256;  // threads per pass-x / pass-y CTA
constexpr int PF = 16;   // prefetch depth (positions)
constexpr int ZL = 128;  // threads per pass-z CTA

__device__ __forceinline__ double sq(double x) { return __dmul_rn(x, x); }

// packed (dk, di): dk in the high half, di in the low half
__device__ __forceinline__ int32_t pack(int dk, int di) { return (int32_t)(((uint32_t)dk << 16) | (uint16_t)di); }
__device__ __forceinline__ int unpack_dk(int32_t p) { return p >> 16; }
__device__ __forceinline__ int unpack_di(int32_t p) { return (int)(int16_t)(p & 0xffff); }

// Division-free envelope predicates (same op order as oracle/ct_oracle.c).
// Sites b < p < q with costs gb, gp, gq; a = q - p, c = p - b:
//   pop p            iff c*(gq - gp) - a*(gp - gb) <= -(d2*a*c*(a + c))
//   x past p|q       iff gq - gp < d2*a*(2x - q - p)
__device__ __forceinline__ bool env_pop(int q, double gq, int p, double gp, int b, double gb, double d2) {
    const double a = (double)(q - p), c = (double)(p - b);
    const double lhs = __dadd_rn(__dmul_rn(c, __dadd_rn(gq, -gp)), -__dmul_rn(a, __dadd_rn(gp, -gb)));
    const double rhs = -__dmul_rn(__dmul_rn(__dmul_rn(d2, a), c), a + c);
    return lhs <= rhs;
}

__device__ __forceinline__ bool env_past(int x, int q, double gq, int p, double gp, double d2) {
    return __dadd_rn(gq, -gp) < __dmul_rn(__dmul_rn(d2, (double)(q - p)), (double)(2 * x - q - p));
}

// ---------------------------------------------------------------------------
// pass x: nearest foreground along i (ties -> lower i), di = fi - i
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(LT) edt_pass_x(const uint8_t *__restrict__ mask, i64 nlines, int nx,
                                                 int16_t *__restrict__ di) {
    const i64 l = blockIdx.x * (i64)LT + threadIdx.x;
    if (l >= nlines) return;
    const i64 S = nlines;  // ny * nz
    int last = -1;
    for (int x0 = 0; x0 < nx; x0 += PF) {
        uint8_t m[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) m[u] = x0 + u < nx ? mask[(i64)(x0 + u) * S + l] : 0;
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            if (x0 + u >= nx) break;
            if (m[u]) last = x0 + u;
            di[(i64)(x0 + u) * S + l] = last < 0 ? NONE16 : (int16_t)(last - (x0 + u));
        }
    }
    int next = -1;
    for (int x0 = nx - 1; x0 >= 0; x0 -= PF) {
        uint8_t m[PF];
        int16_t prevd[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int x = x0 - u;
            m[u] = x >= 0 ? mask[(i64)x * S + l] : 0;
            prevd[u] = x >= 0 ? di[(i64)x * S + l] : NONE16;
        }
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int x = x0 - u;
            if (x < 0) break;
            if (m[u]) next = x;
            const int prev = prevd[u] == NONE16 ? -1 : x + prevd[u];
            int best = prev;
            if (next >= 0 && (best < 0 || next - x < x - best)) best = next;
            di[(i64)x * S + l] = best < 0 ? NONE16 : (int16_t)(best - x);
        }
    }
}

// ---------------------------------------------------------------------------
// pass z: per (i,j) line along the contiguous k (nz <= 128); sites di != NONE,
// cost (di*dx)^2; output packed (dk, di).  A CTA stages ZL consecutive lines
// in SMEM (coalesced in and out); per-thread stacks hold (position, di).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double gx_of(int16_t d, double dx) { return sq(__dmul_rn((double)d, dx)); }

__global__ void __launch_bounds__(ZL) edt_pass_z(const int16_t *__restrict__ di, i64 nlines, int nz, double dx,
                                                 double dz, int32_t *__restrict__ out) {
    // CTA = ZL consecutive lines (contiguous in memory): staged in and out of
    // SMEM with coalesced copies; the envelope runs per thread on its line.
    extern __shared__ __align__(16) unsigned char zsm[];
    const int S = nz + 1;                          // padded stride
    int32_t *io = (int32_t *)zsm;                  // [ZL][S] in: di (as int32), out: packed
    int16_t *sdi = (int16_t *)(io + ZL * S);       // [nz][ZL] di of each stack entry
    uint8_t *stk = (uint8_t *)(sdi + ZL * nz);     // [nz][ZL] byte positions
    const i64 l0 = blockIdx.x * (i64)ZL;
    const int nl = (int)min((i64)ZL, nlines - l0);
    const int tot = nl * nz;
    const int16_t *src = di + l0 * nz;
    for (int idx = threadIdx.x; idx < tot; idx += ZL) {
        const int g = idx / nz, k = idx - g * nz;
        io[g * S + k] = src[idx];
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < nl) {
        int32_t *L = io + t * S;
        uint8_t *st = stk + t;
        int16_t *sd = sdi + t;
        const double d2 = __dmul_rn(dz, dz);
        int K = 0, tp = 0, bp = 0;
        double tg = 0.0, bg = 0.0;
        for (int x = 0; x < nz; ++x) {
            const int32_t v = L[x];
            if (v == NONE16) continue;
            const double gx = gx_of((int16_t)v, dx);
            while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
                --K;
                tp = bp;
                tg = bg;
                if (K >= 2) {
                    bp = st[(K - 2) * ZL];
                    bg = gx_of(sd[(K - 2) * ZL], dx);
                }
            }
            st[K * ZL] = (uint8_t)x;
            sd[K * ZL] = (int16_t)v;
            ++K;
            bp = tp; bg = tg; tp = x; tg = gx;
        }
        // results overwrite the staged line in place; stack entries keep
        // their own di, so no overwritten element is read again
        if (K == 0) {
            for (int x = 0; x < nz; ++x) L[x] = NONE32;
        } else {
            int e = 0;
            int cp = st[0], np = K > 1 ? st[ZL] : 0;
            int cdi = sd[0], ndi = K > 1 ? sd[ZL] : 0;
            double cg = gx_of((int16_t)cdi, dx), ng = K > 1 ? gx_of((int16_t)ndi, dx) : 0.0;
            for (int x = 0; x < nz; ++x) {
                while (e + 1 < K && env_past(x, np, ng, cp, cg, d2)) {
                    ++e;
                    cp = np; cdi = ndi; cg = ng;
                    if (e + 1 < K) {
                        np = st[(e + 1) * ZL];
                        ndi = sd[(e + 1) * ZL];
                        ng = gx_of((int16_t)ndi, dx);
                    }
                }
                L[x] = pack(cp - x, cdi);
            }
        }
    }
    __syncthreads();
    int32_t *dst = out + l0 * nz;
    for (int idx = threadIdx.x; idx < tot; idx += ZL) {
        const int g = idx / nz, k = idx - g * nz;
        dst[idx] = io[g * S + k];
    }
}

// ---------------------------------------------------------------------------
// pass y: envelope along j; sites (dk,di) != NONE, cost (di*dx)^2 + (dk*dz)^2;
// output the float64 distance in scipy's term order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double gxz(int32_t p, double dx, double dz) {
    return __dadd_rn(sq(__dmul_rn((double)unpack_di(p), dx)), sq(__dmul_rn((double)unpack_dk(p), dz)));
}

__global__ void __launch_bounds__(LT) edt_pass_y(const int32_t *__restrict__ in, i64 nlines, int ny, int nz, double dx,
                                                 double dy, double dz, double *__restrict__ out,
                                                 uint16_t *__restrict__ spill) {
    // stack of site positions (payloads are re-read from the input: L1-resident)
    __shared__ uint16_t stk[SCE][LT];
    const i64 l = blockIdx.x * (i64)LT + threadIdx.x;
    // lanes run data-dependent loops; reconverge (wm) before every batched
    // load and every store so the warp's accesses stay coalesced
    const unsigned wm = __ballot_sync(0xffffffffu, l < nlines);
    if (l >= nlines) return;
    const i64 base = (l / nz) * (i64)ny * nz + (l % nz);
    const double d2 = __dmul_rn(dy, dy);
    auto ent_ld = [&](int e) -> int {
        return e < SCE ? stk[e][threadIdx.x] : spill[(i64)(e - SCE) * nlines + l];
    };
    auto ent_st = [&](int e, int pos) {
        if (e < SCE) stk[e][threadIdx.x] = (uint16_t)pos;
        else spill[(i64)(e - SCE) * nlines + l] = (uint16_t)pos;
    };
    auto pay = [&](int pos) -> int32_t { return in[base + (i64)pos * nz]; };
    int K = 0, tp = 0, bp = 0;
    double tg = 0.0, bg = 0.0;
    for (int x0 = 0; x0 < ny; x0 += PF) {
        int32_t v[PF];
        __syncwarp(wm);
#pragma unroll
        for (int u = 0; u < PF; ++u) v[u] = x0 + u < ny ? in[base + (i64)(x0 + u) * nz] : NONE32;
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int x = x0 + u;
            if (x >= ny) break;
            if (v[u] == NONE32) continue;
            const double gx = gxz(v[u], dx, dz);
            while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
                --K;
                tp = bp;
                tg = bg;
                if (K >= 2) {
                    bp = ent_ld(K - 2);
                    bg = gxz(pay(bp), dx, dz);
                }
            }
            ent_st(K, x);
            bp = tp; bg = tg; tp = x; tg = gx;
            ++K;
        }
    }
    int e = 0, cp = 0, np = 0;
    int32_t cpl = 0, npl = 0;
    double cg = 0.0, ng = 0.0;
    if (K) {
        cp = ent_ld(0); cpl = pay(cp); cg = gxz(cpl, dx, dz);
        if (K > 1) { np = ent_ld(1); npl = pay(np); ng = gxz(npl, dx, dz); }
    }
    for (int x = 0; x < ny; ++x) {
        double r = INFINITY;
        if (K) {
            while (e + 1 < K && env_past(x, np, ng, cp, cg, d2)) {
                ++e;
                cp = np; cpl = npl; cg = ng;
                if (e + 1 < K) { np = ent_ld(e + 1); npl = pay(np); ng = gxz(npl, dx, dz); }
            }
            const double t0 = sq(__dmul_rn((double)unpack_di(cpl), dx));
            const double t1 = sq(__dmul_rn((double)(cp - x), dy));
            const double t2 = sq(__dmul_rn((double)unpack_dk(cpl), dz));
            r = __dsqrt_rn(__dadd_rn(__dadd_rn(t0, t1), t2));
        }
        __syncwarp(wm);
        out[base + (i64)x * nz] = r;
    }
}

}  // namespace

size_t ct_edt_workspace(int64_t nx, int64_t ny, int64_t nz) {
    const i64 N = nx * ny * nz;
    const i64 sp = nx * nz * (ny > SCE ? ny - SCE : 0);  // pass-y spill entries
    return (((size_t)N * 2 + 255) & ~(size_t)255) + (((size_t)N * 4 + 255) & ~(size_t)255) + (size_t)sp * 2 + 4096;
}

extern "C" int ct_edt(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, double dx, double dy, double dz,
                      void *work, double *out, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("mask has no voxels");
        return CT_ERR_PARAM;
    }
    if (nx > 32767 || ny > 32767 || nz > 128) {
        ct::set_error("EDT supports nx, ny < 32768 and nz <= 128 (packed int16 offsets, byte stacks)");
        return CT_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const i64 N = nx * ny * nz;
    int16_t *di = (int16_t *)work;
    int32_t *pk = (int32_t *)((char *)work + (((size_t)N * 2 + 255) & ~(size_t)255));
    uint16_t *spill = (uint16_t *)((char *)pk + (((size_t)N * 4 + 255) & ~(size_t)255));
    const i64 lx = ny * nz, lz = nx * ny, ly = nx * nz;
    edt_pass_x<<<(unsigned)((lx + LT - 1) / LT), LT, 0, s>>>(mask, lx, (int)nx, di);
    if (int st = ct::check_launch("edt_pass_x")) return st;
    const size_t zsm = (size_t)ZL * (nz + 1) * 4 + (size_t)ZL * nz * 3 + 16;
    cudaFuncSetAttribute(edt_pass_z, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);
    edt_pass_z<<<(unsigned)((lz + ZL - 1) / ZL), ZL, zsm, s>>>(di, lz, (int)nz, dx, dz, pk);
    if (int st = ct::check_launch("edt_pass_z")) return st;
    edt_pass_y<<<(unsigned)((ly + LT - 1) / LT), LT, 0, s>>>(pk, ly, (int)ny, (int)nz, dx, dy, dz, out, spill);
    return ct::check_launch("edt_pass_y");
}
