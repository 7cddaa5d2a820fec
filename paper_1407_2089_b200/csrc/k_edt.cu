// k_edt.cu -- K8: exact anisotropic Euclidean distance transform.
//
// Replaces ref segment.py:292-304: ndimage.distance_transform_edt(~mask,
// sampling=(dx,dy,dz)) -- the distance (um) from every voxel to the nearest
// foreground voxel.  scipy forms it from an integer feature transform as
//   sqrt(((fi-i)dx)^2 + ((fj-j)dy)^2 + ((fk-k)dz)^2), summed axis 0 -> 2;
// here the nearest feature's integer offsets are carried through three
// separable passes and the distance is formed from them in exactly that order.
//
//   pass z : per (i,j) line (contiguous, nz <= 128): the line's mask is four
//            warp ballots; each voxel's nearest set bit is one CLZ/FFS pair.
//            Output: dk (int8), or NONE.                       1 B in, 1 B out
//   pass y : per (i,k) line along j: lower envelope of the parabolas
//            (dk*dz)^2 + ((j-q)*dy)^2 over the sites q (Felzenszwalb-
//            Huttenlocher).  Output (dj, dk) packed in int32.   1 B in, 4 B out
//   pass x : per (j,k) line along i, site cost (dj*dy)^2 + (dk*dz)^2, output
//            the float64 distance.                              4 B in, 8 B out
// Lines map to consecutive k across a warp, so every load/store is coalesced.
// Each thread keeps its envelope stack (site position + payload) in SMEM
// (spilling to a global scratch beyond 16 entries); intersections are
// recomputed from the stack, so neither the build nor the output loop issues a
// dependent global load.  Arithmetic matches oracle/ct_oracle.c ora_edt bit for
// bit (separately rounded __d*_rn ops); equidistant features may differ from
// scipy's choice in the last ulp, within the reference's 1e-9 um contract
// (ref test_acceptance.py:318-332).
#include <type_traits>

#include "ct_common.cuh"

namespace {

constexpr int8_t NONE8 = -128;
constexpr int32_t NONE32 = INT32_MIN;
constexpr int SC = 16;       // SMEM stack entries per thread
constexpr int LT = 256;      // threads per envelope CTA

__device__ __forceinline__ double sq(double x) { return __dmul_rn(x, x); }

// ---------------------------------------------------------------------------
// pass z: nearest foreground along k, ties -> lower k
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) edt_pass_z(const uint8_t *__restrict__ mask, i64 nlines, int nz,
                                                  int8_t *__restrict__ dk) {
    const unsigned lane = threadIdx.x & 31;
    const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
    const int W = (nz + 31) >> 5;  // <= 4
    for (i64 l = warp; l < nlines; l += nwarps) {
        const uint8_t *m = mask + l * nz;
        uint32_t words[4] = {0, 0, 0, 0};
#pragma unroll
        for (int w = 0; w < 4; ++w)
            if (w < W) {
                const int k = 32 * w + lane;
                words[w] = __ballot_sync(0xffffffffu, k < nz && m[k] != 0);
            }
        const u64 lo = ((u64)words[1] << 32) | words[0], hi = ((u64)words[3] << 32) | words[2];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int k = 32 * w + lane;
            if (w >= W || k >= nz) continue;
            // previous set bit <= k
            int prev = -1, next = -1;
            if (k < 64) {
                const u64 x = lo & (k == 63 ? ~0ull : ((2ull << k) - 1));
                if (x) prev = 63 - __clzll((long long)x);
                const u64 y = lo & ~((1ull << k) - 1);
                if (y) next = __ffsll((long long)y) - 1;
                else if (hi) next = 64 + __ffsll((long long)hi) - 1;
            } else {
                const int kk = k - 64;
                const u64 x = hi & (kk == 63 ? ~0ull : ((2ull << kk) - 1));
                if (x) prev = 64 + 63 - __clzll((long long)x);
                else if (lo) prev = 63 - __clzll((long long)lo);
                const u64 y = hi & ~((1ull << kk) - 1);
                if (y) next = 64 + __ffsll((long long)y) - 1;
            }
            int best = prev;
            if (next >= 0 && (best < 0 || next - k < k - best)) best = next;
            dk[l * nz + k] = best < 0 ? NONE8 : (int8_t)(best - k);
        }
    }
}

// generic pass z for nz > 128 (one thread per line, two sweeps); offsets must fit int8
__global__ void edt_pass_z_generic(const uint8_t *__restrict__ mask, i64 nlines, int nz, int8_t *__restrict__ dk) {
    for (i64 l = blockIdx.x * (i64)blockDim.x + threadIdx.x; l < nlines; l += (i64)gridDim.x * blockDim.x) {
        const uint8_t *m = mask + l * nz;
        int8_t *o = dk + l * nz;
        int last = -1;
        for (int k = 0; k < nz; ++k) {
            if (m[k]) last = k;
            o[k] = last < 0 ? NONE8 : (int8_t)max(-127, last - k);
        }
        int next = -1;
        for (int k = nz - 1; k >= 0; --k) {
            if (m[k]) next = k;
            const int prev = o[k] == NONE8 ? -1 : k + o[k];
            int best = prev;
            if (next >= 0 && (best < 0 || next - k < k - best)) best = next;
            o[k] = best < 0 ? NONE8 : (int8_t)(best - k);
        }
    }
}

// ---------------------------------------------------------------------------
// envelope passes (AXIS 1: y, input int8 dk; AXIS 0: x, input packed (dj,dk))
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t pack(int dj, int dk) { return (int32_t)((dj << 8) | (uint8_t)(int8_t)dk); }
__device__ __forceinline__ int unpack_dj(int32_t p) { return p >> 8; }
__device__ __forceinline__ int unpack_dk(int32_t p) { return (int)(int8_t)(p & 0xff); }

template <int AXIS>
struct Env {
    // payload of a site (the feature's offsets along the already-done axes)
    typedef typename std::conditional<AXIS == 1, int8_t, int32_t>::type In;
    __device__ static bool site(In v) { return AXIS == 1 ? v != NONE8 : v != NONE32; }
    __device__ static int32_t payload(In v) { return (int32_t)v; }
    // cost of the site's feature on its own line position (previous axes only)
    __device__ static double g(int32_t pl, double dy, double dz) {
        if (AXIS == 1) return sq(__dmul_rn((double)pl, dz));
        return __dadd_rn(sq(__dmul_rn((double)unpack_dj(pl), dy)), sq(__dmul_rn((double)unpack_dk(pl), dz)));
    }
};

// Division-free envelope predicates (identical op order in oracle/ct_oracle.c).
// Sites b < p < q with costs gb, gp, gq; a = q - p, c = p - b.  The parabola
// of q overtakes p before p overtakes b (pop p) iff
//   c*(gq - gp) - a*(gp - gb) <= -(d2*a*c*(a + c))
// and position x has passed the p|q boundary iff
//   gq - gp < d2*a*(2x - q - p).
__device__ __forceinline__ bool env_pop(int q, double gq, int p, double gp, int b, double gb, double d2) {
    const double a = (double)(q - p), c = (double)(p - b);
    const double lhs = __dadd_rn(__dmul_rn(c, __dadd_rn(gq, -gp)), -__dmul_rn(a, __dadd_rn(gp, -gb)));
    const double rhs = -__dmul_rn(__dmul_rn(__dmul_rn(d2, a), c), a + c);
    return lhs <= rhs;
}

__device__ __forceinline__ bool env_past(int x, int q, double gq, int p, double gp, double d2) {
    return __dadd_rn(gq, -gp) < __dmul_rn(__dmul_rn(d2, (double)(q - p)), (double)(2 * x - q - p));
}

template <int AXIS>
__global__ void __launch_bounds__(LT) edt_pass_env(const typename Env<AXIS>::In *__restrict__ in, i64 nlines, int L,
                                                   i64 stride, double dx, double dy, double dz,
                                                   int32_t *__restrict__ out32, double *__restrict__ out64,
                                                   u64 *__restrict__ spill) {
    __shared__ u64 stk[SC][LT];  // entry = (position << 32) | payload
    typedef Env<AXIS> E;
    typedef typename E::In In;
    const double d = AXIS == 1 ? dy : dx, d2 = __dmul_rn(d, d);
    const i64 l = blockIdx.x * (i64)LT + threadIdx.x;
    if (l >= nlines) return;
    i64 base;
    if (AXIS == 1) {  // lines (i, k), position j, stride nz
        const i64 nz = stride, ny = L;
        base = (l / nz) * ny * nz + (l % nz);
    } else {          // lines (j, k) = flattened plane index, position i
        base = l;
    }
#define ENT(e) (*((e) < SC ? &stk[(e)][threadIdx.x] : &spill[((e) - SC) * nlines + l]))
    // build: stack entries 0..K-1 in memory; the top two also in registers
    int K = 0;
    int tp = 0, bp = 0;            // top / below positions
    double tg = 0.0, bg = 0.0;     // top / below costs
    In v = in[base];
    for (int x = 0; x < L; ++x) {
        const In cur = v;
        if (x + 1 < L) v = in[base + (i64)(x + 1) * stride];  // prefetch
        if (!E::site(cur)) continue;
        const int32_t pl = E::payload(cur);
        const double gx = E::g(pl, dy, dz);
        while (K >= 2 && env_pop(x, gx, tp, tg, bp, bg, d2)) {
            --K;
            tp = bp;
            tg = bg;
            if (K >= 2) {
                const u64 e = ENT(K - 2);
                bp = (int)(e >> 32);
                bg = E::g((int32_t)(e & 0xffffffffu), dy, dz);
            }
        }
        ENT(K) = ((u64)(uint32_t)x << 32) | (uint32_t)pl;
        bp = tp;
        bg = tg;
        tp = x;
        tg = gx;
        ++K;
    }
    // output: advance while x has passed the boundary to the next entry
    int e = 0;
    int cp = 0, np = 0;
    int32_t cpl = 0, npl = 0;
    double cg = 0.0, ng = 0.0;
    if (K) {
        const u64 c0 = ENT(0);
        cp = (int)(c0 >> 32); cpl = (int32_t)(c0 & 0xffffffffu); cg = E::g(cpl, dy, dz);
        if (K > 1) {
            const u64 c1 = ENT(1);
            np = (int)(c1 >> 32); npl = (int32_t)(c1 & 0xffffffffu); ng = E::g(npl, dy, dz);
        }
    }
    for (int x = 0; x < L; ++x) {
        const i64 o = base + (i64)x * stride;
        if (K == 0) {
            if (AXIS == 1) out32[o] = NONE32;
            else out64[o] = INFINITY;
            continue;
        }
        while (e + 1 < K && env_past(x, np, ng, cp, cg, d2)) {
            ++e;
            cp = np; cpl = npl; cg = ng;
            if (e + 1 < K) {
                const u64 c1 = ENT(e + 1);
                np = (int)(c1 >> 32); npl = (int32_t)(c1 & 0xffffffffu); ng = E::g(npl, dy, dz);
            }
        }
        if (AXIS == 1) {
            out32[o] = pack(cp - x, cpl);
        } else {
            const double t0 = sq(__dmul_rn((double)(cp - x), dx));
            const double t1 = sq(__dmul_rn((double)unpack_dj(cpl), dy));
            const double t2 = sq(__dmul_rn((double)unpack_dk(cpl), dz));
            out64[o] = __dsqrt_rn(__dadd_rn(__dadd_rn(t0, t1), t2));
        }
    }
#undef ENT
}

}  // namespace

size_t ct_edt_workspace(int64_t nx, int64_t ny, int64_t nz) {
    const i64 N = nx * ny * nz;
    // dk (1 B) + packed (4 B) + spill: (L - SC) entries per line, 8 B
    const i64 ly = nx * nz * (ny > SC ? ny - SC : 0), lx = ny * nz * (nx > SC ? nx - SC : 0);
    const i64 sp = ly > lx ? ly : lx;
    return (size_t)N * 5 + (size_t)sp * 8 + 4096;
}

extern "C" int ct_edt(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, double dx, double dy, double dz,
                      void *work, double *out, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("mask has no voxels");
        return CT_ERR_PARAM;
    }
    if (nz > 127 || ny > 32767 || nx > (1 << 30)) {
        // dk offsets are int8 and dj int24 in the packed payload
        if (nz > 127) {
            ct::set_error("EDT: nz > 127 unsupported by the packed feature format");
            return CT_ERR_UNSUPPORTED;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    const i64 N = nx * ny * nz;
    int8_t *dk = (int8_t *)work;
    int32_t *pk = (int32_t *)((char *)work + ((N + 255) & ~(i64)255));
    u64 *spill = (u64 *)((char *)pk + ((N * 4 + 255) & ~(i64)255));
    edt_pass_z<<<ct::grid_for(nx * ny * 32, 256, CT_NUM_SMS * 16), 256, 0, s>>>(mask, nx * ny, (int)nz, dk);
    if (int st = ct::check_launch("edt_pass_z")) return st;
    const i64 ly = nx * nz, lx = ny * nz;
    edt_pass_env<1><<<(unsigned)((ly + LT - 1) / LT), LT, 0, s>>>(dk, ly, (int)ny, nz, dx, dy, dz, pk, nullptr,
                                                                    spill);
    if (int st = ct::check_launch("edt_pass_y")) return st;
    edt_pass_env<0><<<(unsigned)((lx + LT - 1) / LT), LT, 0, s>>>(pk, lx, (int)nx, ny * nz, dx, dy, dz, nullptr, out,
                                                                    spill);
    return ct::check_launch("edt_pass_x");
}
