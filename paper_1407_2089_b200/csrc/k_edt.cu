// k_edt.cu -- K8: exact anisotropic Euclidean distance transform.
//
// Replaces ref segment.py:292-304: ndimage.distance_transform_edt(~mask,
// sampling=(dx,dy,dz)) -- the distance (um) from every voxel to the nearest
// foreground voxel, computed by scipy from an integer feature transform as
//   sqrt(((fi-i)dx)^2 + ((fj-j)dy)^2 + ((fk-k)dz)^2), summed axis 0 -> 2.
// Here the feature coordinates are carried through three separable passes
// (x: nearest foreground on the line; y, z: lower envelope of parabolas,
// Felzenszwalb-Huttenlocher) and the distance is formed from them in
// scipy's order, so distances agree bit for bit whenever the chosen feature
// is scipy's (equidistant features may differ in the last ulp; the
// reference's own contract is 1e-9 um, ref test_acceptance.py:318-332).
// Arithmetic is identical to oracle/ct_oracle.c (no FMA: __d*_rn).
#include "ct_common.cuh"

namespace {

constexpr int FB = 21;
constexpr i64 FM = (1ll << FB) - 1;

__device__ __forceinline__ i64 fpack(i64 a, i64 b, i64 c) { return (a << (2 * FB)) | (b << FB) | c; }

__device__ __forceinline__ double sq(double x) { return __dmul_rn(x, x); }

__device__ __forceinline__ double cost(i64 f, i64 i, i64 j, i64 k, int upto, double dx, double dy, double dz) {
    const i64 fi = (f >> (2 * FB)) & FM, fj = (f >> FB) & FM, fk = f & FM;
    const double t0 = sq(__dmul_rn((double)(fi - i), dx));
    if (upto == 0) return t0;
    const double t1 = sq(__dmul_rn((double)(fj - j), dy));
    if (upto == 1) return __dadd_rn(t0, t1);
    const double t2 = sq(__dmul_rn((double)(fk - k), dz));
    return __dadd_rn(__dadd_rn(t0, t1), t2);
}

// pass 0: per (j,k) line along x, nearest foreground (ties -> lower i)
__global__ void edt_pass_x(const uint8_t *__restrict__ mask, i64 nx, i64 ny, i64 nz, i64 *__restrict__ f) {
    const i64 nl = ny * nz, S = ny * nz;
    for (i64 l = blockIdx.x * (i64)blockDim.x + threadIdx.x; l < nl; l += (i64)gridDim.x * blockDim.x) {
        const i64 j = l / nz, k = l % nz;
        i64 last = -1;
        for (i64 i = 0; i < nx; ++i) {
            const i64 p = i * S + l;
            if (mask[p]) last = i;
            f[p] = last;
        }
        i64 next = -1;
        for (i64 i = nx - 1; i >= 0; --i) {
            const i64 p = i * S + l;
            if (mask[p]) next = i;
            i64 best = f[p];
            if (next >= 0 && (best < 0 || next - i < i - best)) best = next;
            f[p] = best < 0 ? -1 : fpack(best, j, k);
        }
    }
}

// passes 1 (axis y) and 2 (axis z): lower envelope per line; scratch laid
// out [position][line] so neighbouring threads (lines) coalesce.
template <int AXIS>
__global__ void edt_pass_env(const i64 *__restrict__ fin, i64 *__restrict__ fout, i64 nx, i64 ny, i64 nz, double dx,
                             double dy, double dz, int32_t *__restrict__ vs, double *__restrict__ zs,
                             double *__restrict__ gs) {
    const i64 nl = AXIS == 1 ? nx * nz : nx * ny;
    const i64 L = AXIS == 1 ? ny : nz;
    const double d = AXIS == 1 ? dy : dz, d2 = __dmul_rn(d, d);
    for (i64 l = blockIdx.x * (i64)blockDim.x + threadIdx.x; l < nl; l += (i64)gridDim.x * blockDim.x) {
        i64 ci, cj = 0, ck = 0, base, stride;
        if (AXIS == 1) {
            ci = l / nz; ck = l % nz; base = ci * ny * nz + ck; stride = nz;
        } else {
            ci = l / ny; cj = l % ny; base = l * nz; stride = 1;
        }
#define V(x) vs[(x) * nl + l]
#define Z(x) zs[(x) * nl + l]
#define G(x) gs[(x) * nl + l]
        i64 kk = -1;
        for (i64 q = 0; q < L; ++q) {
            const i64 f = fin[base + q * stride];
            if (f < 0) continue;
            const double gq = AXIS == 1 ? cost(f, ci, q, ck, 0, dx, dy, dz) : cost(f, ci, cj, q, 1, dx, dy, dz);
            G(q) = gq;
            if (kk < 0) {
                kk = 0; V(0) = (int32_t)q; Z(0) = -INFINITY; Z(1) = INFINITY;
                continue;
            }
            double s;
            for (;;) {
                const i64 p = V(kk);
                s = __dmul_rn(__dadd_rn(__ddiv_rn(__dadd_rn(gq, -G(p)), __dmul_rn(d2, (double)(q - p))),
                                        (double)(q + p)),
                              0.5);
                if (s <= Z(kk)) { --kk; continue; }
                break;
            }
            ++kk; V(kk) = (int32_t)q; Z(kk) = s; Z(kk + 1) = INFINITY;
        }
        if (kk < 0) {
            for (i64 x = 0; x < L; ++x) fout[base + x * stride] = -1;
            continue;
        }
        i64 e = 0;
        for (i64 x = 0; x < L; ++x) {
            while (Z(e + 1) < (double)x) ++e;
            fout[base + x * stride] = fin[base + (i64)V(e) * stride];
        }
#undef V
#undef Z
#undef G
    }
}

__global__ void edt_final(const i64 *__restrict__ f, i64 nx, i64 ny, i64 nz, double dx, double dy, double dz,
                          double *__restrict__ out) {
    const i64 n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
        const i64 fv = f[p];
        out[p] = fv < 0 ? INFINITY : __dsqrt_rn(cost(fv, i, j, k, 2, dx, dy, dz));
    }
}

}  // namespace

size_t ct_edt_workspace(int64_t nx, int64_t ny, int64_t nz) {
    const i64 N = nx * ny * nz;
    const i64 ly = nx * nz * (ny + 2), lz = nx * ny * (nz + 2);
    const i64 L = ly > lz ? ly : lz;
    return (size_t)(2 * N * 8) + (size_t)L * (4 + 8 + 8) + 1024;
}

extern "C" int ct_edt(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, double dx, double dy, double dz,
                      void *work, double *out, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("mask has no voxels");
        return CT_ERR_PARAM;
    }
    if (nx > FM || ny > FM || nz > FM) {
        ct::set_error("EDT supports extents below 2^21");
        return CT_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const i64 N = nx * ny * nz;
    i64 *fa = (i64 *)work, *fb = fa + N;
    const i64 ly = nx * nz * (ny + 2), lz = nx * ny * (nz + 2);
    const i64 L = ly > lz ? ly : lz;
    char *sp = (char *)(fb + N);
    double *zs = (double *)sp;
    double *gs = zs + L;
    int32_t *vs = (int32_t *)(gs + L);
    edt_pass_x<<<ct::grid_for(ny * nz, 128), 128, 0, s>>>(mask, nx, ny, nz, fa);
    if (int st = ct::check_launch("edt_pass_x")) return st;
    edt_pass_env<1><<<ct::grid_for(nx * nz, 128), 128, 0, s>>>(fa, fb, nx, ny, nz, dx, dy, dz, vs, zs, gs);
    if (int st = ct::check_launch("edt_pass_y")) return st;
    edt_pass_env<2><<<ct::grid_for(nx * ny, 128), 128, 0, s>>>(fb, fa, nx, ny, nz, dx, dy, dz, vs, zs, gs);
    if (int st = ct::check_launch("edt_pass_z")) return st;
    edt_final<<<ct::grid_for(N, 256), 256, 0, s>>>(fa, nx, ny, nz, dx, dy, dz, out);
    return ct::check_launch("edt_final");
}
