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
                                                 double dz, int32_t *__restrict__ out, uint8_t *__restrict__ rowflag) {
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
        rowflag[l0 + t] = K > 0;
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

// The sites of line (i,k) are the rows j whose z-line (i,j) had a site
// (pass z flags them); that row set does not depend on k.  A CTA owns plane i
// and KC consecutive k: it compacts the site rows once (ordered ballot scan),
// stages their payloads in SMEM, builds the KC envelopes (one thread each,
// stacks of row indices in SMEM), then all 256 threads write the KC x ny
// outputs -- thread (k, chunk) finds its chunk's first segment and streams.
constexpr int KC = 16;
constexpr int YT = 256;

__global__ void __launch_bounds__(YT) edt_pass_y(const int32_t *__restrict__ in, const uint8_t *__restrict__ rowflag,
                                                 int nx, int ny, int nz, double dx, double dy, double dz,
                                                 double *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char ysm[];
    uint16_t *J = (uint16_t *)ysm;                          // [ny] site rows
    int32_t *P = (int32_t *)(ysm + (((size_t)ny * 2 + 15) & ~(size_t)15));   // [nJ][KC] payloads
    uint16_t *st = (uint16_t *)(P + (size_t)ny * KC);       // [KC][ny] stack (indices into J)
    __shared__ int s_n, s_wsum[YT / 32], s_K[KC];
    const int kchunks = (nz + KC - 1) / KC;
    const int i = blockIdx.x / kchunks, k0 = (blockIdx.x % kchunks) * KC;
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const i64 plane = (i64)i * ny;
    // 1. ordered compaction of the flagged rows
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int j0 = 0; j0 < ny; j0 += YT) {
        const int j = j0 + threadIdx.x;
        const bool f = j < ny && rowflag[plane + j];
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_wsum[wid] = __popc(m);
        __syncthreads();
        int before = s_n;
        for (unsigned w = 0; w < wid; ++w) before += s_wsum[w];
        if (f) J[before + __popc(m & ((1u << lane) - 1))] = (uint16_t)j;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < YT / 32; ++w) t += s_wsum[w];
            s_n += t;
        }
        __syncthreads();
    }
    const int nJ = s_n;
    // 2. payloads of the site rows (rows of KC contiguous int32)
    for (int e = threadIdx.x; e < nJ * KC; e += YT) {
        const int r = e / KC, kk = e - r * KC;
        P[e] = k0 + kk < nz ? in[(plane + J[r]) * nz + k0 + kk] : NONE32;
    }
    __syncthreads();
    const double d2 = __dmul_rn(dy, dy);
    // 3. envelopes, one thread per k
    if (threadIdx.x < KC && k0 + (int)threadIdx.x < nz) {
        const int kk = threadIdx.x;
        uint16_t *S = st + kk * ny;
        int K = 0, tp = 0, bp = 0, tr = 0, br = 0;
        double tg = 0.0, bg = 0.0;
        for (int r = 0; r < nJ; ++r) {
            const int32_t v = P[r * KC + kk];
            if (v == NONE32) continue;
            const int x = J[r];
            const double gx = gxz(v, dx, dz);
            while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
                --K;
                tp = bp; tg = bg; tr = br;
                if (K >= 2) {
                    br = S[K - 2];
                    bp = J[br];
                    bg = gxz(P[br * KC + kk], dx, dz);
                }
            }
            S[K] = (uint16_t)r;
            ++K;
            bp = tp; bg = tg; br = tr;
            tp = x; tg = gx; tr = r;
        }
        s_K[kk] = K;
    }
    __syncthreads();
    // 4. outputs: thread = (k, chunk of rows)
    const int kk = threadIdx.x % KC, c = threadIdx.x / KC;
    const int nchunk = YT / KC, CH = (ny + nchunk - 1) / nchunk;
    const int ja = c * CH, jb = min(ny, ja + CH);
    if (k0 + kk >= nz || ja >= jb) return;
    const int K = s_K[kk];
    const uint16_t *S = st + kk * ny;
    double *o = out + (plane + ja) * nz + k0 + kk;
    if (K == 0) {
        for (int j = ja; j < jb; ++j, o += nz) *o = INFINITY;
        return;
    }
    int e = 0;
    int cr = S[0], cp = J[cr];
    int32_t cpl = P[cr * KC + kk];
    double cg = gxz(cpl, dx, dz);
    int nr = 0, np = 0;
    double ng = 0.0;
    if (K > 1) { nr = S[1]; np = J[nr]; ng = gxz(P[nr * KC + kk], dx, dz); }
    for (int j = ja; j < jb; ++j, o += nz) {
        while (e + 1 < K && env_past(j, np, ng, cp, cg, d2)) {
            ++e;
            cr = nr; cp = np; cg = ng;
            cpl = P[cr * KC + kk];
            if (e + 1 < K) { nr = S[e + 1]; np = J[nr]; ng = gxz(P[nr * KC + kk], dx, dz); }
        }
        const double t0 = sq(__dmul_rn((double)unpack_di(cpl), dx));
        const double t1 = sq(__dmul_rn((double)(cp - j), dy));
        const double t2 = sq(__dmul_rn((double)unpack_dk(cpl), dz));
        *o = __dsqrt_rn(__dadd_rn(__dadd_rn(t0, t1), t2));
    }
}

inline size_t ysmem(int ny) { return (((size_t)ny * 2 + 15) & ~(size_t)15) + (size_t)ny * KC * 4 + (size_t)KC * ny * 2; }

}  // namespace

size_t ct_edt_workspace(int64_t nx, int64_t ny, int64_t nz) {
    const i64 N = nx * ny * nz;
    return (((size_t)N * 2 + 255) & ~(size_t)255) + (((size_t)N * 4 + 255) & ~(size_t)255) + (size_t)nx * ny + 4096;
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
    uint8_t *rowflag = (uint8_t *)((char *)pk + (((size_t)N * 4 + 255) & ~(size_t)255));
    const i64 lx = ny * nz, lz = nx * ny;
    edt_pass_x<<<(unsigned)((lx + LT - 1) / LT), LT, 0, s>>>(mask, lx, (int)nx, di);
    if (int st = ct::check_launch("edt_pass_x")) return st;
    const size_t zsm = (size_t)ZL * (nz + 1) * 4 + (size_t)ZL * nz * 3 + 16;
    cudaFuncSetAttribute(edt_pass_z, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);
    edt_pass_z<<<(unsigned)((lz + ZL - 1) / ZL), ZL, zsm, s>>>(di, lz, (int)nz, dx, dz, pk, rowflag);
    if (int st = ct::check_launch("edt_pass_z")) return st;
    const size_t ysm = ysmem((int)ny);
    if (ysm > 220 * 1024) {
        ct::set_error("EDT: ny too large for the SMEM pass-y layout");
        return CT_ERR_UNSUPPORTED;
    }
    cudaFuncSetAttribute(edt_pass_y, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ysm);
    const i64 ychunks = nx * ((nz + KC - 1) / KC);
    edt_pass_y<<<(unsigned)ychunks, YT, ysm, s>>>(pk, rowflag, (int)nx, (int)ny, (int)nz, dx, dy, dz, out);
    return ct::check_launch("edt_pass_y");
}
