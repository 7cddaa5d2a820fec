// k_edt.cu -- K8: exact anisotropic Euclidean distance transform.
//
// Replaces ref segment.py:292-304: ndimage.distance_transform_edt(~mask,
// sampling=(dx,dy,dz)) -- the distance (um) from every voxel to the nearest
// foreground voxel.  scipy forms it from an integer feature transform as
//   sqrt(((fi-i)dx)^2 + ((fj-j)dy)^2 + ((fk-k)dz)^2), summed axis 0 -> 2;
// here the nearest feature's integer offsets are carried through three
// separable passes and the distance is formed from them in exactly that order.
//
//   pass x : per (j,k) line along i: nearest foreground (two sweeps over a
//            register-prefetched stream).                 1 B in, 2 B (di) out
//   pass y : per (i,k) line along j: lower envelope (Felzenszwalb-Huttenlocher)
//            of the parabolas (di*dx)^2 + ((j-q)*dy)^2 over the sites q; the
//            sites are sparse after pass x (only columns that hold foreground),
//            so each thread's stack lives in SMEM (global spill past 16).
//                                                           2 B in, 4 B (dj,di) out
//   pass z : per (i,j) line along the contiguous k (nz in {32, 64, 96, 128}): one
//            thread streams its line from global memory, builds the envelope
//            of (di*dx)^2 + (dj*dy)^2 + ((k-q)*dz)^2 with its stack in SMEM,
//            computes the switch points per entry, then sweeps the voxels
//            forming the float64 distances (32-byte stores; edt_pass_zr).
//            Other nz: SMEM-staged lines (edt_pass_z).      4 B in, 8 B out
// Lines of passes x and y map to consecutive k across a warp (coalesced).  The
// envelope uses division-free predicates; arithmetic is identical to
// oracle/ct_oracle.c ora_edt, so results match it bit for bit; equidistant
// features may differ from scipy's choice in the last ulp, within the
// reference's 1e-9 um contract (ref test_acceptance.py:318-332).
#include <climits>
#include <cstdlib>

#include "ct_common.cuh"

namespace {

constexpr int16_t NONE16 = INT16_MIN;
constexpr int32_t NONE32 = INT32_MIN;
constexpr int SC = 48;   // SMEM stack entries per thread (pass y)
constexpr int LT = 256;  // threads per pass-x / pass-y CTA
constexpr int PF = 16;   // prefetch depth (positions)
constexpr int ZL = 128;  // lines per pass-z CTA
constexpr int YSEG = 1;  // pass-y output segments per line (2 measured slower: the build dominates)

__device__ __forceinline__ double sq(double x) { return __dmul_rn(x, x); }


__device__ __forceinline__ int32_t pack(int dj, int di) { return (int32_t)(((uint32_t)dj << 16) | (uint16_t)di); }
__device__ __forceinline__ int unpack_dj(int32_t p) { return p >> 16; }
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

// smallest x in [xlo, xhi) with env_past(x, q, gq, p, gp) (xhi if none).  The
// predicate is monotone in x (its right side is a rounded increasing function
// of x), so a float estimate corrected by exact tests gives the same answer
// as testing every x in turn.
// The estimate is single precision (approximate reciprocal): a float64
// division was the largest instruction block of the pass-z sweep.
__device__ __forceinline__ int first_past(int xlo, int xhi, int q, double gq, int p, double gp, double d2) {
    const float xs = 0.5f * (__fdividef((float)(gq - gp), (float)d2 * (float)(q - p)) + (float)(q + p));
    int x = !(xs >= (float)xlo) ? xlo : (xs >= (float)xhi ? xhi : (int)xs + 1);
    while (x > xlo && env_past(x - 1, q, gq, p, gp, d2)) --x;
    while (x < xhi && !env_past(x, q, gq, p, gp, d2)) ++x;
    return x;
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

// Parallel pass x (nx <= 1024 * W): CTA = 32 consecutive lines x 32 segments
// of 32*W rows.  Each thread packs its segment's mask into W 32-bit words
// (bit u = row u); the last / first foreground of every segment goes through
// SMEM so each thread knows the nearest foreground left and right of its
// segment; then per row the nearest left / right foreground comes from the
// words by clz / ffs.  Same tie rule as the sweeps (equal distance -> lower i).
template <int W>
__global__ void __launch_bounds__(1024) edt_pass_x_seg(const uint8_t *__restrict__ mask, i64 nlines, int nx,
                                                        int16_t *__restrict__ di) {
    __shared__ int segL[32][33], segF[32][33];
    const int c = threadIdx.x, y = threadIdx.y;
    const i64 l = blockIdx.x * 32ll + c;
    const bool valid = l < nlines;
    const i64 S = nlines;
    const int row0 = y * 32 * W;
    uint32_t bits[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
        uint8_t m[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const int x = row0 + w * 32 + u;
            m[u] = (valid && x < nx) ? mask[(i64)x * S + l] : 0;
        }
        uint32_t b = 0;
#pragma unroll
        for (int u = 0; u < 32; ++u) b |= (m[u] ? 1u : 0u) << u;
        bits[w] = b;
    }
    int last = -1, first = -1;
#pragma unroll
    for (int w = W - 1; w >= 0; --w)
        if (last < 0 && bits[w]) last = row0 + w * 32 + 31 - __clz(bits[w]);
#pragma unroll
    for (int w = 0; w < W; ++w)
        if (first < 0 && bits[w]) first = row0 + w * 32 + __ffs(bits[w]) - 1;
    segL[y][c] = last;
    segF[y][c] = first;
    __syncthreads();
    int left = -1, right = -1;
    for (int yy = y - 1; yy >= 0; --yy)
        if (segL[yy][c] >= 0) { left = segL[yy][c]; break; }
    for (int yy = y + 1; yy < 32; ++yy)
        if (segF[yy][c] >= 0) { right = segF[yy][c]; break; }
    if (!valid) return;
    int rctx[W];
    {
        int r = right;
#pragma unroll
        for (int w = W - 1; w >= 0; --w) {
            rctx[w] = r;
            if (bits[w]) r = row0 + w * 32 + __ffs(bits[w]) - 1;
        }
    }
    int lc = left;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const int wb = row0 + w * 32;
        const uint32_t b = bits[w];
#pragma unroll 8
        for (int u = 0; u < 32; ++u) {
            const int x = wb + u;
            if (x >= nx) break;
            const uint32_t lo = b & ((2u << u) - 1u);  // rows <= x (u = 31: all)
            const uint32_t hi = b & ~((1u << u) - 1u);  // rows >= x
            const int lf = lo ? wb + 31 - __clz(lo) : lc;
            const int rf = hi ? wb + __ffs(hi) - 1 : rctx[w];
            int best = lf;
            if (rf >= 0 && (best < 0 || rf - x < x - best)) best = rf;
            di[(i64)x * S + l] = best < 0 ? NONE16 : (int16_t)(best - x);
        }
        if (b) lc = wb + 31 - __clz(b);
    }
}

// pass x for nx <= 1024 with 4 adjacent lines per thread (32-bit mask loads,
// 64-bit stores): CTA = 4 XG lines x 32 segments of 32 rows.
constexpr int XG = 8;
__global__ void __launch_bounds__(XG * 32) edt_pass_x_seg4(const uint8_t *__restrict__ mask, i64 nlines, int nx,
                                                           int16_t *__restrict__ di) {
    __shared__ int segL[32][4 * XG + 1], segF[32][4 * XG + 1];
    __shared__ uint32_t segM[4 * XG];  // per line: bit y = segment y holds foreground
    const int c = threadIdx.x, y = threadIdx.y;  // c: 4-line group, y: segment
    if (y == 0) for (int q = 0; q < 4; ++q) segM[4 * c + q] = 0u;
    __syncthreads();
    const i64 l0 = blockIdx.x * (4ll * XG) + 4 * c;
    const bool valid = l0 < nlines;             // nlines % 4 == 0
    const i64 S = nlines;
    const int row0 = y * 32;
    uint32_t bits[4] = {0, 0, 0, 0};
    uint32_t v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        const int x = row0 + u;
        v[u] = (valid && x < nx) ? __ldg((const uint32_t *)(mask + (i64)x * S + l0)) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 32; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) bits[q] |= (((v[u] >> (8 * q)) & 0xffu) ? 1u : 0u) << u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        segL[y][4 * c + q] = bits[q] ? row0 + 31 - __clz(bits[q]) : -1;
        segF[y][4 * c + q] = bits[q] ? row0 + __ffs(bits[q]) - 1 : -1;
        if (bits[q]) atomicOr(&segM[4 * c + q], 1u << y);
    }
    __syncthreads();
    if (!valid) return;
    // nearest segments with foreground left / right of this one from the
    // line's segment mask (a scan of the other 31 segments per line was most
    // of this kernel's instructions on sparse masks)
    int lc[4], rc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t sm = segM[4 * c + q];
        const uint32_t below = sm & ((1u << y) - 1u), above = sm & ~((2u << y) - 1u);
        lc[q] = below ? segL[31 - __clz(below)][4 * c + q] : -1;
        rc[q] = above ? segF[__ffs(above) - 1][4 * c + q] : -1;
    }
    // segments without foreground in their own rows (most of a sparse mask):
    // the nearest foreground is lc or rc for every row, no bit scans
    if (!(bits[0] | bits[1] | bits[2] | bits[3])) {
        if (max(max(lc[0], lc[1]), max(lc[2], lc[3])) < 0 && max(max(rc[0], rc[1]), max(rc[2], rc[3])) < 0) {
            const uint32_t none2 = (uint32_t)(uint16_t)NONE16 * 0x10001u;  // no foreground on the lines at all
#pragma unroll 8
            for (int u = 0; u < 32; ++u) {
                const int x = row0 + u;
                if (x >= nx) break;
                *(uint2 *)(di + (i64)x * S + l0) = make_uint2(none2, none2);
            }
            return;
        }
#pragma unroll 4
        for (int u = 0; u < 32; ++u) {
            const int x = row0 + u;
            if (x >= nx) break;
            uint32_t packed[2];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int best = lc[q];
                if (rc[q] >= 0 && (best < 0 || rc[q] - x < x - best)) best = rc[q];
                const uint32_t d = (uint16_t)(best < 0 ? NONE16 : (int16_t)(best - x));
                if (q & 1) packed[q >> 1] |= d << 16;
                else packed[q >> 1] = d;
            }
            *(uint2 *)(di + (i64)x * S + l0) = make_uint2(packed[0], packed[1]);
        }
        return;
    }
#pragma unroll 4
    for (int u = 0; u < 32; ++u) {
        const int x = row0 + u;
        if (x >= nx) break;
        uint32_t packed[2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t b = bits[q];
            const uint32_t lo = b & ((2u << u) - 1u), hi = b & ~((1u << u) - 1u);
            const int lf = lo ? row0 + 31 - __clz(lo) : lc[q];
            const int rf = hi ? row0 + __ffs(hi) - 1 : rc[q];
            int best = lf;
            if (rf >= 0 && (best < 0 || rf - x < x - best)) best = rf;
            const uint32_t d = (uint16_t)(best < 0 ? NONE16 : (int16_t)(best - x));
            if (q & 1) packed[q >> 1] |= d << 16;
            else packed[q >> 1] = d;
        }
        *(uint2 *)(di + (i64)x * S + l0) = make_uint2(packed[0], packed[1]);
    }
}

// ---------------------------------------------------------------------------
// pass y: envelope along j; sites di != NONE, cost (di*dx)^2; out (dj, di),
// in two kernels (parallelism: only nx*nz lines exist, too few threads
// for one-thread-per-line sweeps of ny outputs):
//   build  : thread per line (64-thread CTAs spread the lines evenly over the
//            SMs), loads PFB deep with compile-time strides; the envelope
//            stack (first SC entries in SMEM, the rest in the spill buffer) is
//            published to global, the switch points sw_e = first_past(sw_{e-1},
//            ...) -- exactly where the one-kernel sweep switches -- go to swh
//            (e-major) / over the line's consumed di entries, and est[s] = the
//            entry in force where output segment s starts.
//   output : YS threads per line, each starts at est[s] and sweeps its x
//            range with coalesced row stores.
// (Tried: YB scanners per line compacting the sparse sites into SMEM before a
// single-thread envelope, with the switch points in parallel -- slower: the
// envelope thread then runs in 2 of 16 warps.)
// ---------------------------------------------------------------------------
constexpr int LTB = 64;  // build CTA size: small CTAs spread the nx*nz lines evenly over the SMs
constexpr int YS = 8;    // output segments per line

template <int NZ, int PFB>
__global__ void __launch_bounds__(LTB) edt_y_build(int16_t *__restrict__ di, i64 nlines, int ny, int nz_, double dx,
                                                  double dy, uint32_t *__restrict__ head,
                                                  uint32_t *__restrict__ spill, int32_t *__restrict__ kc,
                                                  int16_t *__restrict__ swh, int16_t *__restrict__ est) {
    __shared__ uint32_t stk[SC][LTB];
    const int nz = NZ > 0 ? NZ : nz_;
    const i64 l = blockIdx.x * (i64)LTB + threadIdx.x;
    const unsigned wm = __ballot_sync(0xffffffffu, l < nlines);
    if (l >= nlines) return;
    int16_t *line = di + (l / nz) * (i64)ny * nz + (l % nz);
    const double d2 = __dmul_rn(dy, dy);
    auto ent_ld = [&](int e) -> uint32_t { return e < SC ? stk[e][threadIdx.x] : spill[(i64)(e - SC) * nlines + l]; };
    auto ent_st = [&](int e, uint32_t v) {
        if (e < SC) stk[e][threadIdx.x] = v;
        else spill[(i64)(e - SC) * nlines + l] = v;
    };
#define GOF(pl) sq(__dmul_rn((double)(int16_t)(pl), dx))
    int K = 0, tp = 0, bp = 0;
    double tg = 0.0, bg = 0.0;
    // batch x0 + PFB is loaded before batch x0 is consumed (double buffer)
    auto load = [&](int x0, int16_t (&v)[PFB]) {
        const int16_t *p = line + (i64)x0 * nz;
        if (x0 + PFB <= ny) {
#pragma unroll
            for (int u = 0; u < PFB; ++u) v[u] = __ldg(p + u * nz);
        } else {
#pragma unroll
            for (int u = 0; u < PFB; ++u) v[u] = x0 + u < ny ? __ldg(p + u * nz) : NONE16;
        }
    };
    int16_t vn[PFB];
    __syncwarp(wm);
    load(0, vn);
    for (int x0 = 0; x0 < ny; x0 += PFB) {
        int16_t v[PFB];
#pragma unroll
        for (int u = 0; u < PFB; ++u) v[u] = vn[u];
        __syncwarp(wm);
        if (x0 + PFB < ny) load(x0 + PFB, vn);
        // most (i, k) lines see no foreground in most x-columns after pass x:
        // skip a batch with no site in one test instead of one branch per entry
        uint32_t any = 0;
#pragma unroll
        for (int u = 0; u < PFB; ++u) any |= (uint32_t)(uint16_t)v[u] ^ 0x8000u;
        if (!any) continue;
#pragma unroll
        for (int u = 0; u < PFB; ++u) {
            if (v[u] == NONE16) continue;
            const int x = x0 + u;
            const double gx = GOF(v[u]);
            while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
                --K;
                tp = bp;
                tg = bg;
                if (K >= 2) {
                    const uint32_t e = ent_ld(K - 2);
                    bp = (int)(e >> 16);
                    bg = GOF(e & 0xffff);
                }
            }
            ent_st(K, ((uint32_t)x << 16) | (uint16_t)v[u]);
            bp = tp; bg = tg; tp = x; tg = gx;
            ++K;
        }
    }
    kc[l] = K;
    for (int e = 0; e < K && e < SC; ++e) head[(i64)e * nlines + l] = stk[e][threadIdx.x];
    // switch points: the envelope moves past entry e at x = sw_e (nondecreasing).
    // Entries < SC go to swh (e-major, coalesced across lines), the rest over
    // the line's own (already consumed) di entries.  est[s] = envelope entry
    // in force at the first x of output segment s.
    int s_next = 1, xs_next = (int)((i64)ny / YS);
    est[l] = 0;
    if (K > 1) {
        uint32_t c = ent_ld(0);
        int cp = (int)(c >> 16);
        double cg = GOF(c & 0xffff);
        int sw = 0;
        for (int e = 0; e + 1 < K; ++e) {
            const uint32_t nxt = ent_ld(e + 1);
            const int np = (int)(nxt >> 16);
            const double ng = GOF(nxt & 0xffff);
            sw = first_past(sw, ny, np, ng, cp, cg, d2);
            if (e < SC) swh[(i64)e * nlines + l] = (int16_t)sw;
            else line[(i64)e * nz] = (int16_t)sw;
            while (s_next < YS && xs_next < sw) {  // segments starting before sw keep entry e
                est[(i64)s_next * nlines + l] = (int16_t)e;
                ++s_next;
                xs_next = (int)((i64)ny * s_next / YS);
            }
            cp = np;
            cg = ng;
        }
    }
    for (; s_next < YS; ++s_next) est[(i64)s_next * nlines + l] = (int16_t)(K > 0 ? K - 1 : 0);
#undef GOF
}

template <int NZ>
__global__ void __launch_bounds__(LT) edt_y_out(const int16_t *__restrict__ swa, i64 nlines, int ny, int nz_,
                                                const uint32_t *__restrict__ head, const uint32_t *__restrict__ spill,
                                                const int32_t *__restrict__ kc, const int16_t *__restrict__ swh,
                                                const int16_t *__restrict__ est, int32_t *__restrict__ out) {
    const int nz = NZ > 0 ? NZ : nz_;
    const i64 l = blockIdx.x * (i64)LT + threadIdx.x;
    const unsigned wm = __ballot_sync(0xffffffffu, l < nlines);
    if (l >= nlines) return;
    const int seg = blockIdx.y;
    const int x0 = (int)((i64)ny * seg / YS), x1 = (int)((i64)ny * (seg + 1) / YS);
    const i64 base = (l / nz) * (i64)ny * nz + (l % nz);
    const int16_t *sw = swa + base;
    int32_t *o = out + base + (i64)x0 * nz;
    const int K = kc[l];
    auto ent = [&](int e) -> uint32_t { return e < SC ? head[(i64)e * nlines + l] : spill[(i64)(e - SC) * nlines + l]; };
    auto swv = [&](int e) -> int { return e < SC ? (int)swh[(i64)e * nlines + l] : (int)sw[(i64)e * nz]; };
    // lines without sites write NONE through the same (converged) loop
    int e = K ? est[(i64)seg * nlines + l] : 0;
    uint32_t c = K ? ent(e) : 0u;
    int nsw = e + 1 < K ? swv(e) : ny;
    const uint32_t step = K ? 1u << 16 : 0u;
    // packed (dj, di) drops by 1 << 16 per step in x while the feature is fixed
    uint32_t r = K ? (uint32_t)pack((int)(c >> 16) - x0, (int16_t)(c & 0xffff)) : (uint32_t)NONE32;
    for (int x = x0; x < x1; ++x, o += nz) {
        if (x >= nsw) {
            do {
                ++e;
                nsw = e + 1 < K ? swv(e) : ny;
            } while (x >= nsw);
            c = ent(e);
            r = (uint32_t)pack((int)(c >> 16) - x, (int16_t)(c & 0xffff));
        }
        __syncwarp(wm);  // lanes = consecutive k: keep the row store coalesced
        *o = (int32_t)r;
        r -= step;
    }
}

// ---------------------------------------------------------------------------
// pass z: CTA = ZL consecutive (i,j) lines of nz <= 128 elements.
//   phase 1 (all threads, coalesced): g = (di*dx)^2 + (dj*dy)^2 of every
//            element into SMEM (+inf for no site);
//   phase 2 (thread per line): envelope build with the top two costs in
//            registers, stack of uint8 positions in SMEM;
//   phase 3: distance sqrt(g_site + ((q-x)*dz)^2) -- g_site = t0 + t1, so this
//            is ((t0 + t1) + t2), scipy's order -- written straight out.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double gyz(int32_t pl, double dx, double dy) {
    return __dadd_rn(sq(__dmul_rn((double)unpack_di(pl), dx)), sq(__dmul_rn((double)unpack_dj(pl), dy)));
}

template <int NZ>  // NZ > 0: compile-time line length (== nz); 0: runtime
__global__ void __launch_bounds__(ZL) edt_pass_z(const int32_t *__restrict__ in, i64 nlines, int nz_, double dx,
                                                 double dy, double dz, double *__restrict__ out) {
    const int nz = NZ > 0 ? NZ : nz_;
    extern __shared__ __align__(16) unsigned char zsm[];
    const int S = nz + 1;                               // padded line stride (conflict-free)
    double *gs = (double *)zsm;                         // [ZL][S]
    uint8_t *stk = (uint8_t *)(gs + ZL * S);            // [ZL][nz] positions
    const i64 l0 = blockIdx.x * (i64)ZL;
    const int nl = (int)min((i64)ZL, nlines - l0);
    const int tot = nl * nz;
    const int32_t *src = in + l0 * nz;
    if (NZ > 0 && nl == ZL && ((uintptr_t)src & 15) == 0) {
        // 16-byte loads, 8 in flight per thread (two rounds for NZ = 64)
        constexpr int T4 = ZL * (NZ > 0 ? NZ : 4) / 4;
        for (int i0 = threadIdx.x; i0 < T4; i0 += 8 * ZL) {
            int4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (i0 + u * ZL < T4) v[u] = __ldg((const int4 *)src + i0 + u * ZL);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = i0 + u * ZL;
                if (q < T4) {
                    const int idx = q * 4, g = idx / nz, k = idx - g * nz;
                    double *d = gs + g * S + k;
                    d[0] = v[u].x == NONE32 ? INFINITY : gyz(v[u].x, dx, dy);
                    d[1] = v[u].y == NONE32 ? INFINITY : gyz(v[u].y, dx, dy);
                    d[2] = v[u].z == NONE32 ? INFINITY : gyz(v[u].z, dx, dy);
                    d[3] = v[u].w == NONE32 ? INFINITY : gyz(v[u].w, dx, dy);
                }
            }
        }
    } else {
        for (int idx = threadIdx.x; idx < tot; idx += ZL) {
            const int g = idx / nz, k = idx - g * nz;
            const int32_t pl = src[idx];
            gs[g * S + k] = pl == NONE32 ? INFINITY : gyz(pl, dx, dy);
        }
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t >= nl) return;
    const double *G = gs + t * S;
    uint8_t *st = stk + t * nz;
    const double d2 = __dmul_rn(dz, dz);
    int K = 0, tp = 0, bp = 0;
    double tg = 0.0, bg = 0.0;
    for (int x = 0; x < nz; ++x) {
        const double gx = G[x];
        if (gx == INFINITY) continue;
        while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
            --K;
            tp = bp;
            tg = bg;
            if (K >= 2) {
                bp = st[K - 2];
                bg = G[bp];
            }
        }
        st[K++] = (uint8_t)x;
        bp = tp; bg = tg; tp = x; tg = gx;
    }
    double *dst = out + (l0 + t) * nz;
    if (K == 0) {
        for (int x = 0; x < nz; ++x) dst[x] = INFINITY;
        return;
    }
    int e = 0;
    int cp = st[0], np = K > 1 ? st[1] : 0;
    double cg = G[cp], ng = K > 1 ? G[np] : 0.0;
    for (int x = 0; x < nz; ++x) {
        while (e + 1 < K && env_past(x, np, ng, cp, cg, d2)) {
            ++e;
            cp = np; cg = ng;
            if (e + 1 < K) { np = st[e + 1]; ng = G[np]; }
        }
        dst[x] = __dsqrt_rn(__dadd_rn(cg, sq(__dmul_rn((double)(cp - x), dz))));
    }
}

// Pass z, register-streamed form.  ncu on the SMEM-staged form (edt_pass_z):
// the thread-per-line envelope is latency bound (wait stalls, 16 warps/SM) and
// the SMEM staging of whole lines (396 B per line) is what caps the warps.  Here a thread streams
// its own line from global memory (one 32-byte load per 8 elements, the next
// chunk in flight), keeps only the envelope stack in SMEM (positions for all
// entries, packed offsets for the first SCZ; deeper entries re-read their
// offsets from the line, which stays in L1/L2), and forms the distances in the
// sweep itself, four voxels per 32-byte store (one full sector per lane).
// 192 B of SMEM per line (with the switch points): 32 warps per SM.  Same predicates and arithmetic
// as edt_pass_z (bit-identical output).
__device__ __forceinline__ void st_v4(double *p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// 8 elements of the line per lane in one 256-bit load that does not allocate
// in L1: the 1,024 lines' streams otherwise evict the L1 lines the envelope
// re-reads (C2: 298 -> 272 us, tools/micro/edtz_ab.cu; two 128-bit loads with
// allocation, or 256-bit with allocation: 297 / 300 us)
__device__ __forceinline__ void ld8_stream(const int32_t *p, int4 &a, int4 &b) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
}

constexpr int ZRT = 128;  // threads (lines) per CTA
template <int NZ, int SCZ>
__global__ void __launch_bounds__(ZRT, 8) edt_pass_zr(const int32_t *__restrict__ in, i64 nlines, double dx,
                                                      double dy, double dz, double *__restrict__ out) {
    __shared__ double czt[2 * NZ];          // czt[d + NZ] = sq(d * dz)
    __shared__ uint8_t posS[NZ][ZRT];       // stack positions
    __shared__ int32_t pkS[SCZ][ZRT];       // packed offsets of the first SCZ entries
    __shared__ uint8_t swS[NZ][ZRT];        // switch points of the envelope entries
    for (int d = threadIdx.x; d < 2 * NZ; d += ZRT) czt[d] = sq(__dmul_rn((double)(d - NZ), dz));
    __syncthreads();
    const i64 l = blockIdx.x * (i64)ZRT + threadIdx.x;
    if (l >= nlines) return;
    const int t = threadIdx.x;
    const int32_t *line = in + l * NZ;
    const double d2 = __dmul_rn(dz, dz);
    auto pk_ld = [&](int e, int pos) -> int32_t { return e < SCZ ? pkS[e][t] : __ldg(line + pos); };
    int K = 0, tp = 0, bp = 0;
    double tg = 0.0, bg = 0.0;
    int4 na, nb;
    ld8_stream(line, na, nb);
    for (int c = 0; c < NZ; c += 8) {
        const int32_t v[8] = {na.x, na.y, na.z, na.w, nb.x, nb.y, nb.z, nb.w};
        if (c + 8 < NZ) ld8_stream(line + c + 8, na, nb);
        // z-slices without foreground carry NONE32 in every line: skip such a
        // batch in one test
        uint32_t any = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) any |= (uint32_t)v[u] ^ 0x80000000u;
        if (!any) continue;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int32_t px = v[u];
            if (px == NONE32) continue;
            const int x = c + u;
            const double gx = gyz(px, dx, dy);
            while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
                --K;
                tp = bp;
                tg = bg;
                if (K >= 2) {
                    bp = posS[K - 2][t];
                    bg = gyz(pk_ld(K - 2, bp), dx, dy);
                }
            }
            CT_DCHECK(K < NZ);
            posS[K][t] = (uint8_t)x;
            if (K < SCZ) pkS[K][t] = px;
            ++K;
            bp = tp; bg = tg; tp = x; tg = gx;
        }
    }
    double *dst = out + l * NZ;
    if (K == 0) {
#pragma unroll 4
        for (int x = 0; x < NZ; x += 4) st_v4(dst + x, INFINITY, INFINITY, INFINITY, INFINITY);
        return;
    }
    int e = 0;
    int cp = posS[0][t];
    double cg = gyz(pk_ld(0, cp), dx, dy);
    // switch points first, per entry (a loop of at most K - 1 trips per lane
    // instead of a divergent test inside the voxel loop): the sweep moves past
    // entry e at sw_e = first_past(sw_{e-1}, ...), sw_{-1} = 0 -- exactly where
    // the voxel-by-voxel sweep of edt_pass_z switches
    {
        int p = cp, sw = 0;
        double pg = cg;
        for (int e2 = 0; e2 + 1 < K; ++e2) {
            const int q = posS[e2 + 1][t];
            const double qg = gyz(pk_ld(e2 + 1, q), dx, dy);
            sw = first_past(sw, NZ, q, qg, p, pg, d2);
            swS[e2][t] = (uint8_t)sw;
            p = q;
            pg = qg;
        }
    }
    int sw = K > 1 ? swS[0][t] : NZ;
    for (int x0 = 0; x0 < NZ; x0 += 4) {
        double r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int x = x0 + u;
            if (x >= sw) {
                do {
                    ++e;
                    sw = e + 1 < K ? swS[e][t] : NZ;
                } while (x >= sw);
                cp = posS[e][t];
                cg = gyz(pk_ld(e, cp), dx, dy);
            }
            CT_DCHECK(cp - x + NZ >= 0 && cp - x + NZ < 2 * NZ);
            r[u] = __dsqrt_rn(__dadd_rn(cg, czt[cp - x + NZ]));
        }
        st_v4(dst + x0, r[0], r[1], r[2], r[3]);
    }
}

// Pass z for long lines (nz > 128, up to 32767): the edt_pass_z envelope and
// sweep with the costs recomputed from the packed offsets on use and the
// stack in global memory (the int16 pass-x buffer, dead after pass y: one
// entry per voxel at most).  Thread per line; same predicates, same order.
__global__ void __launch_bounds__(128) edt_pass_z_long(const int32_t *__restrict__ in, i64 nlines, int nz, double dx,
                                                       double dy, double dz, int16_t *__restrict__ stack,
                                                       double *__restrict__ out) {
    const i64 l = blockIdx.x * (i64)blockDim.x + threadIdx.x;
    if (l >= nlines) return;
    const int32_t *line = in + l * nz;
    int16_t *st = stack + l * nz;
    auto G = [&](int x) { const int32_t pl = line[x]; return pl == NONE32 ? INFINITY : gyz(pl, dx, dy); };
    const double d2 = __dmul_rn(dz, dz);
    int K = 0, tp = 0, bp = 0;
    double tg = 0.0, bg = 0.0;
    for (int x = 0; x < nz; ++x) {
        const double gx = G(x);
        if (gx == INFINITY) continue;
        while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
            --K;
            tp = bp;
            tg = bg;
            if (K >= 2) {
                bp = st[K - 2];
                bg = G(bp);
            }
        }
        st[K++] = (int16_t)x;
        bp = tp; bg = tg; tp = x; tg = gx;
    }
    double *dst = out + l * nz;
    if (K == 0) {
        for (int x = 0; x < nz; ++x) dst[x] = INFINITY;
        return;
    }
    int e = 0;
    int cp = st[0], np = K > 1 ? st[1] : 0;
    double cg = G(cp), ng = K > 1 ? G(np) : 0.0;
    for (int x = 0; x < nz; ++x) {
        while (e + 1 < K && env_past(x, np, ng, cp, cg, d2)) {
            ++e;
            cp = np; cg = ng;
            if (e + 1 < K) { np = st[e + 1]; ng = G(np); }
        }
        dst[x] = __dsqrt_rn(__dadd_rn(cg, sq(__dmul_rn((double)(cp - x), dz))));
    }
}

inline size_t zsmem(int nz) {
    const int S = nz + 1;
    return (size_t)ZL * S * 8 + (size_t)ZL * nz + 16;
}

}  // namespace

size_t ct_edt_workspace(int64_t nx, int64_t ny, int64_t nz) {
    const i64 N = nx * ny * nz;
    const i64 sp = YSEG * nx * nz * (ny > SC ? ny - SC : 0);  // pass-y spill entries (per segment)
    const i64 ly = nx * nz;  // pass-y lines: published stack heads (SC each) + entry counts
    return (((size_t)N * 2 + 255) & ~(size_t)255) + (((size_t)N * 4 + 255) & ~(size_t)255) + (size_t)sp * 4 +
           (size_t)ly * (SC + 1) * 4 + (size_t)ly * (SC + YS) * 2 + 4096;
}

extern "C" int ct_edt(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, double dx, double dy, double dz,
                      void *work, double *out, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("mask has no voxels");
        return CT_ERR_PARAM;
    }
    if (nx > 32767 || ny > 32767 || nz > 32767) {
        ct::set_error("EDT supports extents < 32768 (packed int16 offsets); got (%lld, %lld, %lld)", (long long)nx,
                      (long long)ny, (long long)nz);
        return CT_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const i64 N = nx * ny * nz;
    int16_t *di = (int16_t *)work;
    int32_t *pk = (int32_t *)((char *)work + (((size_t)N * 2 + 255) & ~(size_t)255));
    uint32_t *spill = (uint32_t *)((char *)pk + (((size_t)N * 4 + 255) & ~(size_t)255));
    const i64 lx = ny * nz, ly = nx * nz, lz = nx * ny;
    if (nx <= 1024 && lx % 4 == 0 && ((uintptr_t)mask & 3) == 0 && ((uintptr_t)di & 7) == 0) {
        // (tried: bit scans only after passing a foreground, and a backward sweep
        // parking right distances in the output -- both slower, 137 / 105 us vs 99)
        edt_pass_x_seg4<<<(unsigned)((lx + 4 * XG - 1) / (4 * XG)), dim3(XG, 32), 0, s>>>(mask, lx, (int)nx, di);
    } else if (nx <= 1024) {
        edt_pass_x_seg<1><<<(unsigned)((lx + 31) / 32), dim3(32, 32), 0, s>>>(mask, lx, (int)nx, di);
    } else if (nx <= 4096) {
        edt_pass_x_seg<4><<<(unsigned)((lx + 31) / 32), dim3(32, 32), 0, s>>>(mask, lx, (int)nx, di);
    } else {
        edt_pass_x<<<(unsigned)((lx + LT - 1) / LT), LT, 0, s>>>(mask, lx, (int)nx, di);
    }
    if (int st = ct::check_launch("edt_pass_x")) return st;
    {
        uint32_t *head = spill + (size_t)YSEG * ly * (ny > SC ? ny - SC : 0);
        int32_t *kc = (int32_t *)(head + (size_t)SC * ly);
        int16_t *swh = (int16_t *)(kc + ly);
        int16_t *est = swh + (size_t)SC * ly;
        const unsigned gb = (unsigned)((ly + LT - 1) / LT);
        // build prefetch depth 16 (measured on C2: 8 -> 115 us, 16 -> 95, 32 -> 107, 64 -> 126)
        auto yb = nz == 64 ? edt_y_build<64, 16> : nz == 32 ? edt_y_build<32, 16> : nz == 96 ? edt_y_build<96, 16>
                  : nz == 128 ? edt_y_build<128, 16> : edt_y_build<0, 16>;
        auto yo = nz == 64 ? edt_y_out<64> : nz == 32 ? edt_y_out<32> : nz == 96 ? edt_y_out<96>
                  : nz == 128 ? edt_y_out<128> : edt_y_out<0>;
        yb<<<(unsigned)((ly + LTB - 1) / LTB), LTB, 0, s>>>(di, ly, (int)ny, (int)nz, dx, dy, head, spill, kc, swh, est);
        if (int st = ct::check_launch("edt_y_build")) return st;
        yo<<<dim3(gb, YS), LT, 0, s>>>(di, ly, (int)ny, (int)nz, head, spill, kc, swh, est, pk);
        if (int st = ct::check_launch("edt_y_out")) return st;
    }
    const size_t sm = zsmem((int)nz);
    if ((nz == 64 || nz == 32 || nz == 96 || nz == 128) && ((uintptr_t)pk & 31) == 0) {
        // (tried: the SMEM-staged thread-per-line form, and a 4-voxel distance phase over SMEM-staged lines
        // with packed offsets or float64 costs -- 468 / 490 / 654 us vs 307 for this register-streamed form)
        const unsigned g = (unsigned)((lz + ZRT - 1) / ZRT);
        if (nz == 64) edt_pass_zr<64, 16><<<g, ZRT, 0, s>>>(pk, lz, dx, dy, dz, out);
        else if (nz == 32) edt_pass_zr<32, 16><<<g, ZRT, 0, s>>>(pk, lz, dx, dy, dz, out);
        else if (nz == 96) edt_pass_zr<96, 16><<<g, ZRT, 0, s>>>(pk, lz, dx, dy, dz, out);
        else edt_pass_zr<128, 16><<<g, ZRT, 0, s>>>(pk, lz, dx, dy, dz, out);
        return ct::check_launch("edt_pass_z");
    }
    if (nz > 128) {
        edt_pass_z_long<<<(unsigned)((lz + 127) / 128), 128, 0, s>>>(pk, lz, (int)nz, dx, dy, dz, di, out);
        return ct::check_launch("edt_pass_z_long");
    }
    auto kz = nz == 64 ? edt_pass_z<64> : nz == 32 ? edt_pass_z<32> : nz == 128 ? edt_pass_z<128> : edt_pass_z<0>;
    cudaFuncSetAttribute(kz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kz<<<(unsigned)((lz + ZL - 1) / ZL), ZL, sm, s>>>(pk, lz, (int)nz, dx, dy, dz, out);
    return ct::check_launch("edt_pass_z");
}
