// A/B harness for the EDT pass z (k_edt.cu edt_pass_zr) on a real C2 input:
// tools/micro/edtz_dump.py writes the pass-y output (packed (dj, di)) and the
// production distance map; each variant runs on the same input, timed with CUDA
// events, and (exact variants) compared bit for bit with the production map.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -o edtz_ab edtz_ab.cu
//   ./edtz_ab DIR
// V bits: 1 = no sqrt (timing only), 2 = build only (timing only),
//         4 = envelope costs kept in SMEM for the first SCG entries,
//         8 = small-integer -> double by DADD (u2d) instead of I2F
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#include <vector>

typedef int64_t i64;
constexpr int32_t NONE32 = INT32_MIN;

__device__ __forceinline__ double sq(double x) { return __dmul_rn(x, x); }
__device__ __forceinline__ int unpack_dj(int32_t p) { return p >> 16; }
__device__ __forceinline__ int unpack_di(int32_t p) { return (int)(int16_t)(p & 0xffff); }
__device__ __forceinline__ double u2d(uint32_t v) {
    return __dadd_rn(__hiloint2double(0x43300000, (int)v), -4503599627370496.0);
}
template <int V> __device__ __forceinline__ double i2d(int v) {  // exact for |v| < 2^20
    if (V & 8) return __dadd_rn(__hiloint2double(0x43300000, v + (1 << 20)), -4503599628419072.0);
    return (double)v;
}
template <int V> __device__ __forceinline__ double gyz(int32_t pl, double dx, double dy) {
    return __dadd_rn(sq(__dmul_rn(i2d<V>(unpack_di(pl)), dx)), sq(__dmul_rn(i2d<V>(unpack_dj(pl)), dy)));
}
template <int V>
__device__ __forceinline__ bool env_pop(int q, double gq, int p, double gp, int b, double gb, double d2) {
    const double a = i2d<V>(q - p), c = i2d<V>(p - b);
    const double lhs = __dadd_rn(__dmul_rn(c, __dadd_rn(gq, -gp)), -__dmul_rn(a, __dadd_rn(gp, -gb)));
    const double rhs = -__dmul_rn(__dmul_rn(__dmul_rn(d2, a), c), a + c);
    return lhs <= rhs;
}
template <int V> __device__ __forceinline__ bool env_past(int x, int q, double gq, int p, double gp, double d2) {
    return __dadd_rn(gq, -gp) < __dmul_rn(__dmul_rn(d2, i2d<V>(q - p)), i2d<V>(2 * x - q - p));
}
template <int V>
__device__ __forceinline__ int first_past(int xlo, int xhi, int q, double gq, int p, double gp, double d2) {
    const float xs = 0.5f * (__fdividef((float)(gq - gp), (float)d2 * (float)(q - p)) + (float)(q + p));
    int x = !(xs >= (float)xlo) ? xlo : (xs >= (float)xhi ? xhi : (int)xs + 1);
    while (x > xlo && env_past<V>(x - 1, q, gq, p, gp, d2)) --x;
    while (x < xhi && !env_past<V>(x, q, gq, p, gp, d2)) ++x;
    return x;
}
__device__ __forceinline__ void st_v4(double *p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__device__ __noinline__ void line_global(const int32_t *__restrict__ line, int nz, double dx, double dy, double dz,
                                         int16_t *__restrict__ st, double *__restrict__ dst) {
    auto G = [&](int x) { const int32_t pl = line[x]; return pl == NONE32 ? INFINITY : gyz<0>(pl, dx, dy); };
    const double d2 = __dmul_rn(dz, dz);
    int K = 0, tp = 0, bp = 0;
    double tg = 0.0, bg = 0.0;
    for (int x = 0; x < nz; ++x) {
        const double gx = G(x);
        if (gx == INFINITY) continue;
        while (K >= 2 && env_pop<0>(x, gx, tp, tg, bp, bg, d2)) {
            --K; tp = bp; tg = bg;
            if (K >= 2) { bp = st[K - 2]; bg = G(bp); }
        }
        st[K++] = (int16_t)x;
        bp = tp; bg = tg; tp = x; tg = gx;
    }
    int e = 0;
    int cp = st[0], np = K > 1 ? st[1] : 0;
    double cg = G(cp), ng = K > 1 ? G(np) : 0.0;
    for (int x = 0; x < nz; ++x) {
        while (e + 1 < K && env_past<0>(x, np, ng, cp, cg, d2)) {
            ++e; cp = np; cg = ng;
            if (e + 1 < K) { np = st[e + 1]; ng = G(np); }
        }
        dst[x] = __dsqrt_rn(__dadd_rn(cg, sq(__dmul_rn((double)(cp - x), dz))));
    }
}

template <int V> __device__ __forceinline__ void ld8(const int32_t *p, int4 &a, int4 &b) {
    if (V & 4096) {
        asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p));
    } else if (V & 2048) {
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p));
    } else {
        a = __ldg((const int4 *)p);
        b = __ldg((const int4 *)p + 1);
    }
}

constexpr int ZRT = 128;
constexpr int NZ = 64, SCZ = 16;
static void *g_ovf = nullptr;

template <int V, int SCG, int SD = NZ, int MINB = 8, int SCZ = 16>
__global__ void __launch_bounds__(ZRT, MINB) passz(const int32_t *__restrict__ in, i64 nlines, double dx, double dy,
                                                double dz, double *__restrict__ out, int *__restrict__ kstat, void *kstat_ovf = nullptr) {
    __shared__ double czt[2 * NZ];
    __shared__ uint8_t posS[SD][ZRT];
    __shared__ int32_t pkS[(V & 4) ? 1 : SCZ][ZRT];
    __shared__ double gS[(V & 4) ? SCG : 1][ZRT];
    __shared__ uint8_t swS[SD][ZRT];
    for (int d = threadIdx.x; d < 2 * NZ; d += ZRT) czt[d] = sq(__dmul_rn((double)(d - NZ), dz));
    __syncthreads();
    const i64 l = blockIdx.x * (i64)ZRT + threadIdx.x;
    if (l >= nlines) return;
    const int t = threadIdx.x;
    const int32_t *line = in + l * NZ;
    const double d2 = __dmul_rn(dz, dz);
    uint16_t *ovf = (uint16_t *)kstat_ovf + l * NZ;
    auto pos_ld = [&](int e) -> int { return ((V & 128) && e >= SD) ? (int)(ovf[e] & 0xffu) : (int)posS[e][t]; };
    auto sw_ld = [&](int e) -> int { return ((V & 128) && e >= SD) ? (int)(ovf[e] >> 8) : (int)swS[e][t]; };
    // cost of stack entry e at position pos
    auto g_ld = [&](int e, int pos) -> double {
        if (V & 4) return e < SCG ? gS[e][t] : gyz<V>(__ldg(line + pos), dx, dy);
        return gyz<V>(e < SCZ ? pkS[e][t] : __ldg(line + pos), dx, dy);
    };
    int K = 0, tp = 0, bp = 0;
    double tg = 0.0, bg = 0.0;
    if (V & 32) {
        // one pop-or-push per iteration (all lanes run the same trip: the
        // warp's trips = max over lanes of pushes + pops instead of the sum
        // over sites of the per-site maximum)
        int x = 0;
        int4 w = __ldg((const int4 *)line);
        auto fetch = [&](int xx) -> int32_t {  // sequential per lane: 16-byte window
            if ((xx & 3) == 0 && xx < NZ) w = __ldg((const int4 *)(line + xx));
            const int u = xx & 3;
            return u == 0 ? w.x : u == 1 ? w.y : u == 2 ? w.z : w.w;
        };
        int32_t px = w.x;
        while (x < NZ && px == NONE32) { ++x; px = x < NZ ? fetch(x) : 0; }
        double gx = x < NZ ? gyz<0>(px, dx, dy) : 0.0;
        while (x < NZ) {
            if (K >= 2 && env_pop<0>(x, gx, tp, tg, bp, bg, d2)) {
                --K;
                tp = bp;
                tg = bg;
                if (K >= 2) {
                    bp = posS[K - 2][t];
                    bg = g_ld(K - 2, bp);
                }
            } else {
                posS[K][t] = (uint8_t)x;
                if (K < SCZ) pkS[K][t] = px;
                ++K;
                bp = tp; bg = tg; tp = x; tg = gx;
                do { ++x; px = x < NZ ? fetch(x) : 0; } while (x < NZ && px == NONE32);
                if (x < NZ) gx = gyz<0>(px, dx, dy);
            }
        }
    }
    int4 na, nb;
    ld8<V>(line, na, nb);
    bool deep = false;
    int32_t prevpx = NONE32;  // site at c - 1 (V & 64)
    double prevg = 0.0;
    int nrem = 0;
    for (int c = (V & 32) ? NZ : 0; c < NZ; c += 8) {
        const int32_t v[8] = {na.x, na.y, na.z, na.w, nb.x, nb.y, nb.z, nb.w};
        if (c + 8 < NZ) ld8<V>(line + c + 8, na, nb);
        uint32_t any = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) any |= (uint32_t)v[u] ^ 0x80000000u;
        if (!any) { prevpx = NONE32; continue; }
        double gv[8];
        bool keep[8];
        if (V & 64) {
            const int32_t nextpx = c + 8 < NZ ? na.x : NONE32;
            const double nextg = nextpx != NONE32 ? gyz<V>(nextpx, dx, dy) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) gv[u] = v[u] != NONE32 ? gyz<V>(v[u], dx, dy) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int32_t lp = u ? v[u - 1] : prevpx, rp = u < 7 ? v[u + 1] : nextpx;
                const double lg = u ? gv[u - 1] : prevg, rg = u < 7 ? gv[u + 1] : nextg;
                keep[u] = v[u] != NONE32 &&
                          !(lp != NONE32 && rp != NONE32 && env_pop<V>(c + u + 1, rg, c + u, gv[u], c + u - 1, lg, d2));
                nrem += v[u] != NONE32 && !keep[u];
            }
            prevpx = v[7];
            prevg = gv[7];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int32_t px = v[u];
            if ((V & 64) ? !keep[u] : px == NONE32) continue;
            const int x = c + u;
            const double gx = (V & 64) ? gv[u] : gyz<V>(px, dx, dy);
            while (K >= 2 && env_pop<V>(x, gx, tp, tg, bp, bg, d2)) {
                --K;
                tp = bp;
                tg = bg;
                if (K >= 2) {
                    bp = pos_ld(K - 2);
                    bg = g_ld(K - 2, bp);
                }
            }
            if (V & (256 | 512)) {
                if (K == SD) { deep = true; continue; }
                posS[K][t] = (uint8_t)x;
            } else if (!(V & 128) || K < SD) posS[K][t] = (uint8_t)x;
            else ovf[K] = (uint16_t)x;
            if (V & 4) {
                if (K < SCG) gS[K][t] = gx;
            } else if (K < SCZ) {
                pkS[K][t] = px;
            }
            ++K;
            bp = tp; bg = tg; tp = x; tg = gx;
        }
    }
    if ((V & (256 | 512)) && deep) {
        if (V & 256) line_global(line, NZ, dx, dy, dz, (int16_t *)kstat_ovf + l * NZ, out + l * NZ);
        else atomicAdd((int *)kstat_ovf, 1);
        return;
    }
    if (kstat) { atomicAdd(kstat + K, 1); if (V & 64) atomicAdd(kstat + NZ + 1, nrem); }
    double *dst = out + l * NZ;
    if (K == 0) {
        for (int x = 0; x < NZ; x += 4) st_v4(dst + x, INFINITY, INFINITY, INFINITY, INFINITY);
        return;
    }
    if (V & 2) {
        for (int x = 0; x < NZ; x += 4) st_v4(dst + x, tg, bg, tg, bg);
        return;
    }
    int e = 0;
    int cp = posS[0][t];
    double cg = g_ld(0, cp);
    {
        int p = cp, sw = 0;
        double pg = cg;
        for (int e2 = 0; e2 + 1 < K; ++e2) {
            const int q = pos_ld(e2 + 1);
            const double qg = g_ld(e2 + 1, q);
            sw = first_past<V>(sw, NZ, q, qg, p, pg, d2);
            if (!(V & 128) || e2 < SD) swS[e2][t] = (uint8_t)sw;
            else ovf[e2] = (uint16_t)(p | (sw << 8));
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
                    sw = e + 1 < K ? sw_ld(e) : NZ;
                } while (x >= sw);
                cp = pos_ld(e);
                cg = g_ld(e, cp);
            }
            const double s = __dadd_rn(cg, czt[cp - x + NZ]);
            r[u] = (V & 1) ? s : __dsqrt_rn(s);
        }
        st_v4(dst + x0, r[0], r[1], r[2], r[3]);
    }
}


// float-certified envelope build (V16): the pop test in FP32 with a rounding
// bound; only pops within the bound take the exact FP64 predicate
__device__ __forceinline__ float i2f(int v) {  // exact for |v| < 2^22: IADD + FADD, no XU
    return __fadd_rn(__int_as_float(0x4B400000 + v), -12582912.0f);
}
__device__ __forceinline__ float gyzf(int32_t pl, float dxf, float dyf) {
    return __fadd_rn(__fmul_rn(__fmul_rn(i2f(unpack_di(pl)), dxf), __fmul_rn(i2f(unpack_di(pl)), dxf)),
                     __fmul_rn(__fmul_rn(i2f(unpack_dj(pl)), dyf), __fmul_rn(i2f(unpack_dj(pl)), dyf)));
}
template <int V>
__global__ void __launch_bounds__(ZRT, 8) passz_f(const int32_t *__restrict__ in, i64 nlines, double dx, double dy,
                                                  double dz, double *__restrict__ out, int *__restrict__ nfall) {
    __shared__ double czt[2 * NZ];
    __shared__ uint8_t posS[NZ][ZRT];
    __shared__ int32_t pkS[SCZ][ZRT];
    __shared__ uint8_t swS[NZ][ZRT];
    for (int d = threadIdx.x; d < 2 * NZ; d += ZRT) czt[d] = sq(__dmul_rn((double)(d - NZ), dz));
    __syncthreads();
    const i64 l = blockIdx.x * (i64)ZRT + threadIdx.x;
    if (l >= nlines) return;
    const int t = threadIdx.x;
    const int32_t *line = in + l * NZ;
    const double d2 = __dmul_rn(dz, dz);
    const float dxf = (float)dx, dyf = (float)dy, d2f = (float)d2;
    auto pk_ld = [&](int e, int pos) -> int32_t { return e < SCZ ? pkS[e][t] : __ldg(line + pos); };
    int K = 0, tp = 0, bp = 0, fall = 0;
    int32_t tpk = 0, bpk = 0;
    float tgf = 0.f, bgf = 0.f;
    int4 na = __ldg((const int4 *)line), nb = __ldg((const int4 *)line + 1);
    for (int c = 0; c < NZ; c += 8) {
        const int32_t v[8] = {na.x, na.y, na.z, na.w, nb.x, nb.y, nb.z, nb.w};
        if (c + 8 < NZ) {
            na = __ldg((const int4 *)(line + c + 8));
            nb = __ldg((const int4 *)(line + c + 12));
        }
        uint32_t any = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) any |= (uint32_t)v[u] ^ 0x80000000u;
        if (!any) continue;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int32_t px = v[u];
            if (px == NONE32) continue;
            const int x = c + u;
            const float gxf = gyzf(px, dxf, dyf);
            while (K >= 2) {
                const float af = i2f(x - tp), cf = i2f(tp - bp);
                const float lhs = __fadd_rn(__fmul_rn(cf, __fadd_rn(gxf, -tgf)), -__fmul_rn(af, __fadd_rn(tgf, -bgf)));
                const float rm = __fmul_rn(__fmul_rn(__fmul_rn(d2f, af), cf), __fadd_rn(af, cf));
                const float m = __fadd_rn(lhs, rm);
                const float eb = __fmul_rn(1.9073486328125e-06f,  // 2^-19
                                           __fadd_rn(__fadd_rn(__fmul_rn(cf, __fadd_rn(gxf, tgf)),
                                                               __fmul_rn(af, __fadd_rn(tgf, bgf))), rm));
                bool pop;
                if (m < -eb) pop = true;
                else if (m > eb) pop = false;
                else {
                    ++fall;
                    pop = env_pop<0>(x, gyz<0>(px, dx, dy), tp, gyz<0>(tpk, dx, dy), bp, gyz<0>(bpk, dx, dy), d2);
                }
                if (!pop) break;
                --K;
                tp = bp;
                tpk = bpk;
                tgf = bgf;
                if (K >= 2) {
                    bp = posS[K - 2][t];
                    bpk = pk_ld(K - 2, bp);
                    bgf = gyzf(bpk, dxf, dyf);
                }
            }
            posS[K][t] = (uint8_t)x;
            if (K < SCZ) pkS[K][t] = px;
            ++K;
            bp = tp; bpk = tpk; bgf = tgf; tp = x; tpk = px; tgf = gxf;
        }
    }
    if (nfall && fall) atomicAdd(nfall, fall);
    double *dst = out + l * NZ;
    if (K == 0) {
        for (int x = 0; x < NZ; x += 4) st_v4(dst + x, INFINITY, INFINITY, INFINITY, INFINITY);
        return;
    }
    int e = 0;
    int cp = posS[0][t];
    double cg = gyz<0>(pk_ld(0, cp), dx, dy);
    {
        int p = cp, sw = 0;
        double pg = cg;
        for (int e2 = 0; e2 + 1 < K; ++e2) {
            const int q = posS[e2 + 1][t];
            const double qg = gyz<0>(pk_ld(e2 + 1, q), dx, dy);
            sw = first_past<0>(sw, NZ, q, qg, p, pg, d2);
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
                cg = gyz<0>(pk_ld(e, cp), dx, dy);
            }
            r[u] = __dsqrt_rn(__dadd_rn(cg, czt[cp - x + NZ]));
        }
        st_v4(dst + x0, r[0], r[1], r[2], r[3]);
    }
}

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

static std::vector<char> slurp(const char *path) {
    FILE *f = fopen(path, "rb");
    if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(1); }
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    std::vector<char> b(n);
    if (fread(b.data(), 1, n, f) != (size_t)n) exit(1);
    fclose(f);
    return b;
}

template <int V, int SCG, int SD = NZ, int MINB = 8, int SCZ = 16>
void run(const char *name, const int32_t *d_in, i64 lz, double *d_out, const std::vector<double> &ref, int reps) {
    const unsigned g = (unsigned)((lz + ZRT - 1) / ZRT);
    passz<V, SCG, SD, MINB, SCZ><<<g, ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, nullptr, g_ovf);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) passz<V, SCG, SD, MINB, SCZ><<<g, ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, nullptr, g_ovf);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<double> h(ref.size());
    CK(cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t i = 0; i < h.size(); ++i) bad += memcmp(&h[i], &ref[i], 8) != 0;
    printf("%-28s %8.1f us  mismatches %zu%s\n", name, 1000.0 * ms / reps, bad, (V & 3) ? " (timing only)" : "");
}

void run_f(const char *name, const int32_t *d_in, i64 lz, double *d_out, const std::vector<double> &ref, int reps, int *d_f) {
    const unsigned g = (unsigned)((lz + ZRT - 1) / ZRT);
    CK(cudaMemset(d_f, 0, 4));
    passz_f<16><<<g, ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, d_f);
    CK(cudaDeviceSynchronize());
    int nf = 0;
    CK(cudaMemcpy(&nf, d_f, 4, cudaMemcpyDeviceToHost));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) passz_f<16><<<g, ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, nullptr);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<double> h(ref.size());
    CK(cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t i = 0; i < h.size(); ++i) bad += memcmp(&h[i], &ref[i], 8) != 0;
    printf("%-28s %8.1f us  mismatches %zu  exact fallbacks %d\n", name, 1000.0 * ms / reps, bad, nf);
}

template <int V>
__global__ void __launch_bounds__(ZRT, 8) passz_h(const int32_t *__restrict__ in, i64 nlines, double dx, double dy,
                                                  double dz, double *__restrict__ out, int *__restrict__ dummy) {
    __shared__ double czt[2 * NZ];
    __shared__ uint8_t posS[NZ][ZRT];
    __shared__ int32_t pkS[SCZ][ZRT];
    __shared__ uint8_t swS[NZ][ZRT];
    for (int d = threadIdx.x; d < 2 * NZ; d += ZRT) czt[d] = sq(__dmul_rn((double)(d - NZ), dz));
    __syncthreads();
    const i64 l = blockIdx.x * (i64)ZRT + threadIdx.x;
    if (l >= nlines) return;
    const int t = threadIdx.x;
    const int32_t *line = in + l * NZ;
    const double d2 = __dmul_rn(dz, dz);
    auto pk_ld = [&](int e, int pos) -> int32_t { return e < SCZ ? pkS[e][t] : __ldg(line + pos); };
    auto hof = [&](int32_t pk, int pos) -> double { return __dadd_rn(gyz<0>(pk, dx, dy), czt[pos + NZ]); };
    int K = 0, tp = 0, bp = 0;
    double th = 0.0, bh = 0.0;  // h of the top and of the entry below it
    int4 na, nb;
    ld8<4096>(line, na, nb);
    for (int c = 0; c < NZ; c += 8) {
        const int32_t v[8] = {na.x, na.y, na.z, na.w, nb.x, nb.y, nb.z, nb.w};
        if (c + 8 < NZ) ld8<4096>(line + c + 8, na, nb);
        uint32_t any = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) any |= (uint32_t)v[u] ^ 0x80000000u;
        if (!any) continue;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int32_t px = v[u];
            if (px == NONE32) continue;
            const int x = c + u;
            const double hx = hof(px, x);
            while (K >= 2 && __dmul_rn(__dadd_rn(hx, -th), (double)(tp - bp)) <=
                                 __dmul_rn(__dadd_rn(th, -bh), (double)(x - tp))) {
                --K;
                tp = bp;
                th = bh;
                if (K >= 2) {
                    bp = posS[K - 2][t];
                    bh = hof(pk_ld(K - 2, bp), bp);
                }
            }
            posS[K][t] = (uint8_t)x;
            if (K < SCZ) pkS[K][t] = px;
            ++K;
            bp = tp; bh = th; tp = x; th = hx;
        }
    }
    double *dst = out + l * NZ;
    if (K == 0) {
        for (int x = 0; x < NZ; x += 4) st_v4(dst + x, INFINITY, INFINITY, INFINITY, INFINITY);
        return;
    }
    int e = 0;
    int cp = posS[0][t];
    double cg = gyz<0>(pk_ld(0, cp), dx, dy);
    {
        int p = cp, sw = 0;
        double pg = cg;
        for (int e2 = 0; e2 + 1 < K; ++e2) {
            const int q = posS[e2 + 1][t];
            const double qg = gyz<0>(pk_ld(e2 + 1, q), dx, dy);
            sw = first_past<0>(sw, NZ, q, qg, p, pg, d2);
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
                cg = gyz<0>(pk_ld(e, cp), dx, dy);
            }
            r[u] = __dsqrt_rn(__dadd_rn(cg, czt[cp - x + NZ]));
        }
        st_v4(dst + x0, r[0], r[1], r[2], r[3]);
    }
}

void run_h(const char *name, const int32_t *d_in, i64 lz, double *d_out, const std::vector<double> &ref, int reps) {
    const unsigned g = (unsigned)((lz + ZRT - 1) / ZRT);
    passz_h<0><<<g, ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, nullptr);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) passz_h<0><<<g, ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, nullptr);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<double> h(ref.size());
    CK(cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    double maxd = 0;
    for (size_t i = 0; i < h.size(); ++i) {
        if (memcmp(&h[i], &ref[i], 8) != 0) { ++bad; maxd = fmax(maxd, fabs(h[i] - ref[i])); }
    }
    printf("%-28s %8.1f us  mismatches %zu (max |d| %.3g)\n", name, 1000.0 * ms / reps, bad, maxd);
}

int main(int argc, char **argv) {
    const char *dir = argc > 1 ? argv[1] : "/tmp";
    char p[512];
    snprintf(p, sizeof p, "%s/edtz_pk.bin", dir);
    std::vector<char> pk = slurp(p);
    snprintf(p, sizeof p, "%s/edtz_out.bin", dir);
    std::vector<char> rb = slurp(p);
    const i64 N = (i64)pk.size() / 4, lz = N / NZ;
    std::vector<double> ref(N);
    memcpy(ref.data(), rb.data(), N * 8);
    int32_t *d_in;
    double *d_out;
    int *d_k;
    CK(cudaMalloc(&d_in, N * 4));
    CK(cudaMalloc(&d_out, N * 8));
    CK(cudaMalloc(&d_k, 4 * (NZ + 2)));
    CK(cudaMemcpy(d_in, pk.data(), N * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&g_ovf, N * 2));
    CK(cudaMemset(d_k, 0, 4 * (NZ + 2)));
    passz<0, 1><<<(unsigned)((lz + ZRT - 1) / ZRT), ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, d_k);
    int hk[NZ + 1];
    CK(cudaMemcpy(hk, d_k, sizeof hk, cudaMemcpyDeviceToHost));
    printf("lines %lld; envelope entries K histogram:", (long long)lz);
    double mean = 0;
    for (int k = 0; k <= NZ; ++k) {
        if (hk[k]) printf(" %d:%d", k, hk[k]);
        mean += (double)k * hk[k];
    }
    printf("\nmean K %.2f\n", mean / lz);
    {
        CK(cudaMemset(d_k, 0, 4 * (NZ + 2)));
        passz<64, 1><<<(unsigned)((lz + ZRT - 1) / ZRT), ZRT>>>(d_in, lz, 0.8, 0.8, 1.0, d_out, d_k);
        int hk2[NZ + 2];
        CK(cudaMemcpy(hk2, d_k, sizeof hk2, cudaMemcpyDeviceToHost));
        printf("prefilter removed %.2f sites per line\n", (double)hk2[NZ + 1] / lz);
    }
    const int reps = 20;
    run<0, 1>("V0 production", d_in, lz, d_out, ref, reps);
    run<1, 1>("V1 no sqrt", d_in, lz, d_out, ref, reps);
    run<2, 1>("V2 build only", d_in, lz, d_out, ref, reps);
    run<0, 1, 32, 10>("V0 stack 32, 10/SM", d_in, lz, d_out, ref, reps);
    run<2048, 1>("V2048 v8 loads", d_in, lz, d_out, ref, reps);
    run<4096, 1>("V4096 v8 no-allocate", d_in, lz, d_out, ref, reps);
    run<2048, 1, 64, 10>("V2048 v8, 10/SM cap", d_in, lz, d_out, ref, reps);
    run<4096 + 512, 1, 32, 10>("V4608 v8 na + stack32 list", d_in, lz, d_out, ref, reps);
    run<2048 + 512, 1, 32, 10>("V2560 v8 + stack32 list", d_in, lz, d_out, ref, reps);
    run<4096, 1>("V4096 v8 no-allocate", d_in, lz, d_out, ref, reps);
    run_h("V-h h-form pop, v8 na", d_in, lz, d_out, ref, reps);
    run_f("V16 float-certified build", d_in, lz, d_out, ref, reps, d_k);
    run<0, 1>("V0 production (again)", d_in, lz, d_out, ref, reps);
    return 0;
}
