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
#include <cudaTypedefs.h>

#include <cstring>
#include <type_traits>

#include "ct_common.cuh"
#include "tc_common.cuh"

PFN_cuTensorMapEncodeTiled_v12000 tma_encoder();  // k_gauss_tc.cu

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

// ---------------------------------------------------------------------------
// r == 1, integer volumes, nz <= 128: bit-sliced selection.
// A z-row of 32 voxels is kept as NB bit-plane words (bit lane = voxel), so
// one thread filters 32 voxels with word-wide logic: for each plane from the
// MSB, count (carry-save adder tree of LOP3s) the still-tied candidates among
// the 27 neighbour words that have a 0 bit, compare with the remaining rank,
// fix the median's bit and prune the candidates -- the 14th smallest of 27 in
// ~50 ALU ops per voxel for u8.  Neighbour rows come from SMEM planes built
// with warp ballots; the k+-1 neighbours are word shifts with clamp-to-edge
// fix-ups.  Output planes become bytes through 8x8 bit transposes; the u8
// histogram uses the per-thread byte counters (ByteHist256).
// ---------------------------------------------------------------------------
constexpr int BTI = 8, BTJ = 16;  // output rows per tile

__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t &s, uint32_t &cy) {
    s = a ^ b ^ c;
    cy = (a & b) | (c & (a ^ b));
}

// 5-bit sliced population count of 27 words
__device__ __forceinline__ void count27(const uint32_t (&t)[27], uint32_t (&c)[5]) {
    uint32_t s1[9], c2[13], c4[6], c8[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) fa(t[3 * i], t[3 * i + 1], t[3 * i + 2], s1[i], c2[i]);
    uint32_t s1b[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) fa(s1[3 * i], s1[3 * i + 1], s1[3 * i + 2], s1b[i], c2[9 + i]);
    fa(s1b[0], s1b[1], s1b[2], c[0], c2[12]);
    uint32_t s2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) fa(c2[3 * i], c2[3 * i + 1], c2[3 * i + 2], s2[i], c4[i]);
    uint32_t s2x;
    fa(s2[0], s2[1], s2[2], s2x, c4[4]);
    fa(s2x, s2[3], c2[12], c[1], c4[5]);
    uint32_t s4a, s4b;
    fa(c4[0], c4[1], c4[2], s4a, c8[0]);
    fa(c4[3], c4[4], c4[5], s4b, c8[1]);
    c[2] = s4a ^ s4b;
    c8[2] = s4a & s4b;
    fa(c8[0], c8[1], c8[2], c[3], c[4]);
}

// 8x8 bit transpose of a 64-bit matrix (byte r = row r)
__device__ __forceinline__ u64 transpose8(u64 x) {
    u64 t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull; x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull; x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull; x = x ^ t ^ (t << 28);
    return x;
}

// voxel values 8g..8g+7 of a word from 8 planes p[0..7] (bytes, little endian)
__device__ __forceinline__ u64 planes_to_bytes(uint32_t p0, uint32_t p1, uint32_t p2, uint32_t p3, uint32_t p4,
                                               uint32_t p5, uint32_t p6, uint32_t p7, int g) {
    const unsigned sel = (unsigned)g | ((unsigned)(4 + g) << 4);
    const uint32_t a01 = __byte_perm(p0, p1, sel), a23 = __byte_perm(p2, p3, sel);
    const uint32_t a45 = __byte_perm(p4, p5, sel), a67 = __byte_perm(p6, p7, sel);
    const uint32_t lo = __byte_perm(a01, a23, 0x5410), hi = __byte_perm(a45, a67, 0x5410);
    return transpose8(((u64)hi << 32) | lo);
}

// bit 8i+b of x (byte i, bit b) -> bit 4b+i: nibble b = plane b of 4 voxels
__device__ __forceinline__ uint32_t t4x8(uint32_t x) {
    uint32_t t;
    t = ((x >> 7) ^ x) & 0x00aa00aau; x ^= t ^ (t << 7);
    t = ((x >> 14) ^ x) & 0x0000ccccu; x ^= t ^ (t << 14);
    t = ((x >> 4) ^ x) & 0x00f000f0u; x ^= t ^ (t << 4);
    t = ((x >> 8) ^ x) & 0x0000ff00u; x ^= t ^ (t << 8);
    return x;
}

// Butterfly steps of the in-register transposes below.  Lane groups exchange
// halves with the partner lane (shfl xor s); a lane whose bit s is clear keeps
// its low parts and takes the partner's low parts shifted up, a lane with
// bit s set keeps its high parts and takes the partner's high parts shifted
// down.  Byte and half-word steps are one PRMT with a per-lane selector,
// nibble / 2-bit steps two SELs and a LOP3 -- no per-step branch (ncu: the
// select-by-branch form was 45% of the u16 median's stalls).
template <int SH, uint32_t M>
__device__ __forceinline__ uint32_t bfly_sel(uint32_t y, uint32_t o, bool hi) {  // SH-bit parts, mask M = low parts
    const uint32_t a = hi ? (o >> SH) : y, b = hi ? y : (o << SH);
    return (a & M) | (b & ~M);
}

// 8x8 nibble transpose across the 8 lanes of a group (lane s holds row s):
// afterwards lane s holds nibble s of every lane's row (row t at nibble t).
__device__ __forceinline__ uint32_t nib_transpose8(uint32_t y, unsigned sub) {
    uint32_t o = __shfl_xor_sync(0xffffffffu, y, 4);
    y = __byte_perm(y, o, (sub & 4) ? 0x3276 : 0x5410);  // 16-bit parts
    o = __shfl_xor_sync(0xffffffffu, y, 2);
    y = __byte_perm(y, o, (sub & 2) ? 0x3715 : 0x6240);  // bytes
    o = __shfl_xor_sync(0xffffffffu, y, 1);
    return bfly_sel<4, 0x0f0f0f0fu>(y, o, sub & 1);      // nibbles
}

// 16x16 transpose of 2-bit elements across the 16 lanes of a half warp (lane
// s holds row s; afterwards lane s holds element s of every lane's row, row t
// at element t)
__device__ __forceinline__ uint32_t pair_transpose16(uint32_t y, unsigned sub) {
    uint32_t o = __shfl_xor_sync(0xffffffffu, y, 8);
    y = __byte_perm(y, o, (sub & 8) ? 0x3276 : 0x5410);  // 16-bit parts
    o = __shfl_xor_sync(0xffffffffu, y, 4);
    y = __byte_perm(y, o, (sub & 4) ? 0x3715 : 0x6240);  // bytes
    o = __shfl_xor_sync(0xffffffffu, y, 2);
    y = bfly_sel<4, 0x0f0f0f0fu>(y, o, sub & 2);         // nibbles
    o = __shfl_xor_sync(0xffffffffu, y, 1);
    return bfly_sel<2, 0x33333333u>(y, o, sub & 1);      // 2-bit elements
}

// two u16 values (low half, high half) -> bit 2b + e = value e's bit b
__device__ __forceinline__ uint32_t zip16(uint32_t x) {
    x = (x & 0xff0000ffu) | ((x & 0x00ff0000u) >> 8) | ((x & 0x0000ff00u) << 8);
    x = (x & 0xf00ff00fu) | ((x & 0x0f000f00u) >> 4) | ((x & 0x00f000f0u) << 4);
    x = (x & 0xc3c3c3c3u) | ((x & 0x30303030u) >> 2) | ((x & 0x0c0c0c0cu) << 2);
    x = (x & 0x99999999u) | ((x & 0x44444444u) >> 1) | ((x & 0x22222222u) << 1);
    return x;
}

// WC > 0: nz == 32 * WC at compile time (planes built by in-register
// transposes from 32-bit loads instead of per-bit ballots: u8 4 voxels per
// lane, nibble transposes over 8 lanes; u16 2 voxels per lane, pair
// transposes over 16 lanes)
// TMA (WC > 0): the tile's (BTI+2) x (BTJ+2) input rows arrive as one 3-D
// cp.async.bulk.tensor box ([i][j][z], rows out of the volume zero-filled and
// then replaced by their clamped rows in SMEM), issued for the next tile as
// soon as this tile's planes are built, so the load overlaps phases B and C.
template <typename T, int NB, int WC = 0, bool TMA_IN = false>
__global__ void __launch_bounds__(256) median3_bits(const T *__restrict__ in, T *__restrict__ out, i64 nx, i64 ny,
                                                    int nz_, uint64_t *__restrict__ ghist,
                                                    const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char dsm[];
    const int nz = WC > 0 ? 32 * WC : nz_;
    const int W = WC > 0 ? WC : (nz + 31) >> 5;
    const int RI = BTI + 2, RJ = BTJ + 2;
    const int NW = RI * RJ * W;  // staged (row, word) units
    // planes stored [b][unit] so a warp's 32 units hit 32 banks; three
    // versions per word: value at k, at k-1 and at k+1 (clamped at the ends)
    uint32_t *pc = (uint32_t *)dsm;   // [NB][NW]
    uint32_t *pm = pc + NB * NW;      // [NB][NW]
    uint32_t *pp = pm + NB * NW;      // [NB][NW]
    uint32_t *s_any = pp + NB * NW;   // planes non-zero in this tile
    const size_t pbytes = ((size_t)3 * NB * NW * 4 + 16 + 15) & ~(size_t)15;
    constexpr bool BYTE = NB == 8;
    ct::ByteHist256 bh;
    uint32_t *sh16 = nullptr;
    if (ghist) {
        if (BYTE) bh.init(dsm + pbytes);
        else {
            sh16 = (uint32_t *)(dsm + pbytes);
            for (int b = threadIdx.x; b < 4096; b += 256) sh16[b] = 0;
        }
    }
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const i64 ti = (nx + BTI - 1) / BTI, tj = (ny + BTJ - 1) / BTJ, ntiles = ti * tj;
    const int units = BTI * BTJ * W;
    const int last_w = (nz - 1) >> 5, last_pos = (nz - 1) & 31;
    int since_flush = 0;
    // TMA input box: [RI][RJ][nz] elements after the planes and the histogram
    constexpr int TBOX = TMA_IN ? (BTI + 2) * (BTJ + 2) * 32 * WC * (int)sizeof(T) : 0;
    const T *tbuf = (const T *)(dsm + ((pbytes + (BYTE ? ct::ByteHist256::kBytes : 4096 * 4) + 127) & ~(size_t)127));
    __shared__ uint64_t tbar;
    uint32_t tphase = 0;
    auto tma_issue = [&](i64 tile) {  // one thread
        const int i0 = (int)((tile / tj) * BTI), j0 = (int)((tile % tj) * BTJ);
        tc::fence_async_smem();  // earlier generic reads of the buffer before the async-proxy write
        tc::mbar_expect_tx(&tbar, TBOX);
        tc::tma_load_3d((void *)tbuf, &tmap, 0, j0 - 1, i0 - 1, &tbar);
    };
    if constexpr (TMA_IN) {
        if (threadIdx.x == 0) {
            tc::mbar_init(&tbar, 1);
            tc::mbar_fence_init();
            tc::tma_prefetch_desc(&tmap);
            if ((i64)blockIdx.x < ntiles) tma_issue(blockIdx.x);
        }
        __syncthreads();
    }
    const int per_thread = (units + 255) / 256;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 i0 = (tile / tj) * BTI, j0 = (tile % tj) * BTJ;
        __syncthreads();
        if (threadIdx.x == 0) *s_any = 0;
        if constexpr (NB == 16 && WC > 0) {
            // clamped row offsets of the tile's input rows, once per tile (TMA:
            // rows in SMEM, out-of-volume rows replaced by their clamped rows)
            __shared__ long long roff16[(BTI + 2) * (BTJ + 2)];
            if constexpr (TMA_IN) {
                tc::mbar_wait(&tbar, tphase);
                tphase ^= 1;
                if (i0 == 0 || j0 == 0 || i0 + BTI >= nx || j0 + BTJ >= ny) {
                    constexpr int RWD = 32 * WC * (int)sizeof(T) / 4;  // words per row
                    uint32_t *tb = (uint32_t *)tbuf;
                    for (int e = threadIdx.x; e < RI * RJ * RWD; e += 256) {
                        const int r = e / RWD, wd = e - r * RWD, ri = r / RJ, rj = r - ri * RJ;
                        const int ci = (int)(ct::clampi(i0 + ri - 1, 0, nx - 1) - (i0 - 1));
                        const int cj = (int)(ct::clampi(j0 + rj - 1, 0, ny - 1) - (j0 - 1));
                        if (ci != ri || cj != rj) tb[r * RWD + wd] = tb[(ci * RJ + cj) * RWD + wd];
                    }
                }
                for (int r = threadIdx.x; r < RI * RJ; r += 256) roff16[r] = (long long)r * nz;
            } else {
                for (int r = threadIdx.x; r < RI * RJ; r += 256) {
                    const int ri = r / RJ, rj = r - ri * RJ;
                    const i64 i = ct::clampi(i0 + ri - 1, 0, nx - 1), j = ct::clampi(j0 + rj - 1, 0, ny - 1);
                    roff16[r] = (i * ny + j) * nz;
                }
            }
            __syncthreads();
            const T *src16 = TMA_IN ? tbuf : in;
            // phase A (u16): a half warp per (row, word) unit, lane s loads
            // voxels 2s, 2s+1 of the word; zip16 + pair_transpose16 leave lane
            // s with plane s of the word
            const unsigned sub = lane & 15;
            const int half = (int)(lane >> 4);
            unsigned anyw = 0;
            constexpr int UB = 4;  // units in flight per half warp
            for (int u0 = 2 * wid + half; u0 < NW; u0 += 16 * UB) {
                uint32_t x[UB];
#pragma unroll
                for (int qq = 0; qq < UB; ++qq) {
                    const int u = u0 + 16 * qq;
                    x[qq] = 0u;
                    if (u < NW) {
                        const int r = u / W, w = u - r * W;
                        x[qq] = TMA_IN ? *((const uint32_t *)(src16 + roff16[r] + 32 * w) + sub)
                                       : __ldg((const uint32_t *)(in + roff16[r] + 32 * w) + sub);
                    }
                }
#pragma unroll
                for (int qq = 0; qq < UB; ++qq) {
                    const int u = u0 + 16 * qq;
                    const uint32_t y = pair_transpose16(zip16(x[qq]), sub);
                    if (u < NW) {
                        pc[sub * NW + u] = y;
                        anyw |= y ? (1u << sub) : 0u;
                    }
                }
            }
            anyw = __reduce_or_sync(0xffffffffu, anyw);
            if (lane == 0 && anyw) atomicOr(s_any, anyw);
        } else if constexpr (NB == 8 && WC > 0) {
            // clamped row offsets of the tile's input rows, once per tile
            // (the per-load clamp / divide was a third of phase A); with TMA the
            // rows are in SMEM: wait for the box, replace the rows outside the
            // volume (zero-filled) by their clamped rows
            __shared__ long long roff[(BTI + 2) * (BTJ + 2)];
            if constexpr (TMA_IN) {
                tc::mbar_wait(&tbar, tphase);
                tphase ^= 1;
                if (i0 == 0 || j0 == 0 || i0 + BTI >= nx || j0 + BTJ >= ny) {
                    constexpr int RWD = 32 * WC * (int)sizeof(T) / 4;  // words per row
                    uint32_t *tb = (uint32_t *)tbuf;
                    for (int e = threadIdx.x; e < RI * RJ * RWD; e += 256) {
                        const int r = e / RWD, wd = e - r * RWD, ri = r / RJ, rj = r - ri * RJ;
                        const int ci = (int)(ct::clampi(i0 + ri - 1, 0, nx - 1) - (i0 - 1));
                        const int cj = (int)(ct::clampi(j0 + rj - 1, 0, ny - 1) - (j0 - 1));
                        if (ci != ri || cj != rj) tb[r * RWD + wd] = tb[(ci * RJ + cj) * RWD + wd];
                    }
                }
                for (int r = threadIdx.x; r < RI * RJ; r += 256) roff[r] = (long long)r * nz;
            } else {
                for (int r = threadIdx.x; r < RI * RJ; r += 256) {
                    const int ri = r / RJ, rj = r - ri * RJ;
                    const i64 i = ct::clampi(i0 + ri - 1, 0, nx - 1), j = ct::clampi(j0 + rj - 1, 0, ny - 1);
                    roff[r] = (i * ny + j) * nz;
                }
            }
            __syncthreads();
            const T *src = TMA_IN ? tbuf : in;
            // phase A (u8, nz = 32 WC): each lane loads 4 voxels (32 bits); a row
            // is 8 WC lanes; t4x8 + a nibble transpose over the 8 lanes of a
            // word leave lane s with plane s of that word
            constexpr int LPR = 8 * WC, RPW = 32 / LPR;
            const int NR = RI * RJ;
            const int lrow = lane / LPR, lw = (lane % LPR) >> 3;
            const unsigned sub = lane & 7;
            unsigned anyw = 0;
            for (int r0 = wid * RPW; r0 < NR; r0 += 8 * RPW * 4) {
                uint32_t x[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = r0 + q * 8 * RPW + lrow;
                    x[q] = 0u;
                    if (r < NR && lrow < RPW)  // (WC = 3: lanes 24-31 idle)
                        x[q] = TMA_IN ? *((const uint32_t *)(src + roff[r]) + (lane % LPR))
                                      : __ldg((const uint32_t *)(in + roff[r]) + (lane % LPR));
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = r0 + q * 8 * RPW + lrow;
                    const uint32_t y = nib_transpose8(t4x8(x[q]), sub);
                    if (r < NR && lrow < RPW) {
                        pc[sub * NW + r * W + lw] = y;
                        anyw |= y ? (1u << sub) : 0u;
                    }
                }
            }
            anyw = __reduce_or_sync(0xffffffffu, anyw);
            if (lane == 0 && anyw) atomicOr(s_any, anyw);
        } else {
            // phase A: planes of the (BTI+2) x (BTJ+2) input rows (clamped), one warp
            // per (row, word); loads batched 8 deep so their latencies overlap
            for (int u0 = wid; u0 < NW; u0 += 8 * 8) {
                unsigned vals[8];
    #pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int u = u0 + 8 * q;
                    vals[q] = 0u;
                    if (u < NW) {
                        const int w = u % W, row = u / W;
                        const int rj = row % RJ, ri = row / RJ;
                        const i64 i = ct::clampi(i0 + ri - 1, 0, nx - 1), j = ct::clampi(j0 + rj - 1, 0, ny - 1);
                        const int k = 32 * w + lane;
                        if (k < nz) vals[q] = (unsigned)in[(i * ny + j) * nz + k];
                    }
                }
                unsigned any = 0;
    #pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int u = u0 + 8 * q;
                    if (u >= NW) break;
                    uint32_t mine = 0;
    #pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        const uint32_t word = __ballot_sync(0xffffffffu, (vals[q] >> b) & 1u);
                        if ((int)lane == b) mine = word;
                    }
                    if ((int)lane < NB) {
                        pc[lane * NW + u] = mine;
                        any |= mine ? (1u << lane) : 0u;
                    }
                }
                if (any) atomicOr(s_any, any);
            }
        }
        __syncthreads();
        // the planes are built: the next tile's input box may overwrite the TMA buffer
        if constexpr (TMA_IN)
            if (threadIdx.x == 0 && tile + gridDim.x < ntiles) tma_issue(tile + gridDim.x);
        // phase B: shifted versions (k-1 and k+1 neighbours, clamp-to-edge)
        for (int e = threadIdx.x; e < NB * NW; e += 256) {
            const int u = e % NW;
            const int w = u % W;
            const uint32_t P = pc[e];
            const uint32_t Pm = w > 0 ? pc[e - 1] : 0u, Pn = w + 1 < W ? pc[e + 1] : 0u;
            uint32_t km1 = (P << 1) | (Pm >> 31);
            if (w == 0) km1 |= P & 1u;  // k = -1 clamps to k = 0
            uint32_t kp1 = (P >> 1) | (Pn << 31);
            if (w == last_w) {          // k = nz clamps to k = nz-1
                const uint32_t m = 1u << last_pos;
                kp1 = (kp1 & ~m) | (P & m);
            }
            pm[e] = km1;
            pp[e] = kp1;
        }
        __syncthreads();
        const uint32_t any = *s_any;
        for (int u = threadIdx.x; u < units; u += 256) {
            const int w = u % W, r = u / W;
            const int lj = r % BTJ, li = r / BTJ;
            const i64 i = i0 + li, j = j0 + lj;
            if (i >= nx || j >= ny) continue;
            int rows[9];
#pragma unroll
            for (int di = 0; di < 3; ++di)
#pragma unroll
                for (int dj = 0; dj < 3; ++dj) rows[di * 3 + dj] = ((li + di) * RJ + (lj + dj)) * W + w;
            uint32_t eq[27];
#pragma unroll
            for (int e = 0; e < 27; ++e) eq[e] = 0xffffffffu;
            uint32_t kr[5] = {0xffffffffu, 0u, 0xffffffffu, 0xffffffffu, 0u};  // rank 13
            uint32_t med[NB];
#pragma unroll
            for (int b = NB - 1; b >= 0; --b) {
                med[b] = 0u;
                if (!((any >> b) & 1u)) continue;  // all-zero plane: median bit 0, nothing pruned
                uint32_t wv[27];
#pragma unroll
                for (int r9 = 0; r9 < 9; ++r9) {
                    const int e = b * NW + rows[r9];
                    wv[3 * r9] = pm[e];
                    wv[3 * r9 + 1] = pc[e];
                    wv[3 * r9 + 2] = pp[e];
                }
                uint32_t t[27];
#pragma unroll
                for (int e = 0; e < 27; ++e) t[e] = eq[e] & ~wv[e];
                uint32_t c[5];
                count27(t, c);
                uint32_t gt = 0, same = 0xffffffffu;
#pragma unroll
                for (int q = 4; q >= 0; --q) {
                    gt |= same & c[q] & ~kr[q];
                    same &= ~(c[q] ^ kr[q]);
                }
                uint32_t br = 0;
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    const uint32_t d = kr[q] ^ c[q] ^ br;
                    br = (~kr[q] & c[q]) | (~(kr[q] ^ c[q]) & br);
                    kr[q] = (gt & kr[q]) | (~gt & d);
                }
                const uint32_t mb = ~gt;
                med[b] = mb;
#pragma unroll
                for (int e = 0; e < 27; ++e) eq[e] &= ~(wv[e] ^ mb);
            }
            const i64 p0 = (i * ny + j) * nz + 32 * w;
            CT_DCHECK(i < nx && j < ny && 32 * w < nz);
            const int nv = min(32, nz - 32 * w);
            if (NB == 8) {
                u64 g8[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) g8[g] = planes_to_bytes(med[0], med[1], med[2], med[3], med[4], med[5], med[6], med[7], g);
                if (nv == 32 && (p0 & 15) == 0) {
                    uint4 *dst = reinterpret_cast<uint4 *>(out + p0);
                    dst[0] = make_uint4((uint32_t)g8[0], (uint32_t)(g8[0] >> 32), (uint32_t)g8[1], (uint32_t)(g8[1] >> 32));
                    dst[1] = make_uint4((uint32_t)g8[2], (uint32_t)(g8[2] >> 32), (uint32_t)g8[3], (uint32_t)(g8[3] >> 32));
                    if (ghist) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) bh.add((int)((g8[q >> 3] >> (8 * (q & 7))) & 0xFF));
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        if (q >= nv) break;
                        const int v = (int)((g8[q >> 3] >> (8 * (q & 7))) & 0xFF);
                        out[p0 + q] = (T)v;
                        if (ghist) bh.add(v);
                    }
                }
            } else {
                u64 lo8[4], hi8[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    lo8[g] = planes_to_bytes(med[0], med[1], med[2], med[3], med[4], med[5], med[6], med[7], g);
                    hi8[g] = planes_to_bytes(med[8 % NB], med[9 % NB], med[10 % NB], med[11 % NB], med[12 % NB],
                                             med[13 % NB], med[14 % NB], med[15 % NB], g);
                }
                // 16-bit outputs: pairs packed into words, 16-byte stores when the
                // 32 voxels are whole and aligned; the histogram counts runs of
                // equal values along z (medians of residuals are mostly 0 and
                // smooth, and 32 lanes adding to one SMEM bin serialise)
                uint32_t pw[16];
#pragma unroll
                for (int q = 0; q < 32; q += 2) {
                    const uint32_t a = (uint32_t)(((lo8[q >> 3] >> (8 * (q & 7))) & 0xFF) |
                                                  (((hi8[q >> 3] >> (8 * (q & 7))) & 0xFF) << 8));
                    const uint32_t b = (uint32_t)(((lo8[q >> 3] >> (8 * ((q + 1) & 7))) & 0xFF) |
                                                  (((hi8[q >> 3] >> (8 * ((q + 1) & 7))) & 0xFF) << 8));
                    pw[q >> 1] = a | (b << 16);
                }
                if (nv == 32 && (p0 & 7) == 0) {
                    uint4 *dst = reinterpret_cast<uint4 *>(out + p0);
#pragma unroll
                    for (int c = 0; c < 4; ++c) dst[c] = make_uint4(pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
                } else {
#pragma unroll
                    for (int q = 0; q < 32; ++q)
                        if (q < nv) out[p0 + q] = (T)((pw[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                }
                if (ghist) {
                    int cur = -1;
                    unsigned run = 0;
                    auto add = [&](int v, unsigned c) {
                        if (v < 4096) atomicAdd(&sh16[v], c);
                        else atomicAdd((unsigned long long *)&ghist[v], (unsigned long long)c);
                    };
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        if (q >= nv) break;
                        const int v = (int)((pw[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                        if (v == cur) {
                            ++run;
                        } else {
                            if (run) add(cur, run);
                            cur = v;
                            run = 1;
                        }
                    }
                    if (run) add(cur, run);
                }
            }
        }
        if (BYTE && ghist) {
            since_flush += per_thread;
            if (since_flush + per_thread > 7) {  // <= 7 * 32 = 224 adds per thread
                bh.flush();
                since_flush = 0;
            }
        }
    }
    if (ghist) {
        if (BYTE) {
            bh.flush();
            bh.to_global((unsigned long long *)ghist);
        } else {
            __syncthreads();
            for (int b = threadIdx.x; b < 4096; b += 256)
                if (sh16[b]) atomicAdd((unsigned long long *)&ghist[b], (unsigned long long)sh16[b]);
        }
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

// ---------------------------------------------------------------------------
// r >= 2, integer volumes: sliding-window histograms (Huang's running median
// in 3-D).  A thread owns one (i, j) column and walks k = 0 .. nz-1: the
// window multiset {in[clamp(i+di), clamp(j+dj), clamp(k+dk)]} moves by one
// z-plane per step -- (2r+1)^2 values leave, (2r+1)^2 enter, and pairs that
// leave and enter with the same value (flat background) cost nothing.  The
// thread's private histogram (u16 counters in SMEM, [bin][thread] so a warp's
// accesses are conflict-free whatever the bins) and a running (m, #below m)
// pair give the size^3 // 2 order statistic after a few bin steps.
//   u8:  256 bins.
//   u16: the high byte in 256 coarse bins (running median bin h, rank rho
//        inside it) and a 256-bin fine histogram of the low bytes of the
//        values in bin h, rebuilt from the window when h moves (rare on
//        smooth data), with its own running position.
// A CTA owns NTC consecutive j of one i; the input rows it needs are staged
// in SMEM per z-chunk of ZC outputs with coalesced loads and an odd word
// stride per row (the per-thread reads of neighbouring columns hit distinct
// banks) -- direct global reads were one L1 wavefront per lane.  The output
// histogram is counted from runs of equal outputs along z.  Same order
// statistic as median_generic (scipy's rank filter, mode "nearest").
// ---------------------------------------------------------------------------
constexpr int SZC = 32;  // outputs per z-chunk

template <typename T, int R>
struct SlideCfg {
    static constexpr int D = 2 * R + 1;
    // counters: a bin holds at most (2r+1)^3 window values -- 125 at r = 2 fits
    // a byte (half the SMEM per column: more columns per SM), 343 at r = 3 not
    using CT = typename std::conditional<(D * D * D < 256), uint8_t, uint16_t>::type;
    static constexpr int NTC = sizeof(T) == 1 ? (sizeof(CT) == 1 ? 128 : 64) : (sizeof(CT) == 1 ? 64 : 32);
    static constexpr int ZS = SZC + 2 * R + 1;                   // staged z-extent per chunk
    static constexpr int W0 = (ZS * (int)sizeof(T) + 3) / 4;     // words per staged row
    static constexpr int RW = W0 | 1;                            // odd word stride
    static constexpr int ROWS = D * (NTC + 2 * R);               // staged rows
    static constexpr size_t HIST = (sizeof(T) == 2 ? 2 : 1) * 256 * NTC * sizeof(CT);
    static constexpr size_t SMEM = HIST + (size_t)ROWS * RW * 4;
};

template <typename T, int R>
__global__ void __launch_bounds__(SlideCfg<T, R>::NTC) median_slide(const T *__restrict__ in, T *__restrict__ out,
                                                                  i64 nx, i64 ny, i64 nz,
                                                                  uint64_t *__restrict__ ghist) {
    using C = SlideCfg<T, R>;
    constexpr int D = C::D, KTH = D * D * D / 2, NTC = C::NTC, ZS = C::ZS, RW = C::RW;
    constexpr bool U16 = sizeof(T) == 2;
    extern __shared__ __align__(16) unsigned char ssm[];
    using CT = typename C::CT;
    CT *hc = (CT *)ssm;                                         // [256][NTC] direct (u8) / coarse (u16)
    CT *hf = hc + 256 * NTC;                                    // [256][NTC] fine (u16)
    uint32_t *stg = (uint32_t *)(ssm + C::HIST);                // [ROWS][RW] words
    const int t = threadIdx.x;
    auto H = [&](int b) -> CT & { return hc[b * NTC + t]; };
    // +-1 on a counter.  u16 counters: a 32-bit shared-memory reduction on the
    // word that holds it (RED: the thread does not wait for it; program order
    // keeps the later reads of its own counters after it; counts never
    // underflow, so no borrow crosses into the neighbour's half).  u8 counters:
    // a plain byte read-modify-write (four columns share a word)
    auto hadd = [&](CT *h, int b, int d) {
        const int idx = b * NTC + t;
        if constexpr (sizeof(CT) == 2) atomicAdd((unsigned *)h + (idx >> 1), (unsigned)d << (16 * (idx & 1)));
        else h[idx] = (CT)(h[idx] + d);
    };
    auto F = [&](int b) -> CT & { return hf[b * NTC + t]; };
    const i64 jt = (ny + NTC - 1) / NTC, ntiles = nx * jt;
    auto flush_run = [&](int v, unsigned c) {
        if (ghist && c) atomicAdd((unsigned long long *)&ghist[v], (unsigned long long)c);
    };
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 i = tile / jt, j0 = (tile - i * jt) * NTC, j = j0 + t;
        const bool live = j < ny;
        // staged row (di, dj) of this thread: rows [di][NTC + 2R], column t + dj
        auto sval = [&](int di, int dj, int u) -> int {  // staged z offset u
            const T *row = (const T *)(stg + (di * (NTC + 2 * R) + t + dj) * RW);
            return (int)row[u];
        };
        for (int b = 0; b < 256; ++b) H(b) = 0;
        if constexpr (U16)
            for (int b = 0; b < 256; ++b) F(b) = 0;
        int m = 0, below = 0, hcur = 0, mf = 0, belowf = 0;
        int run_v = -1;
        unsigned run_n = 0;
        for (i64 k0 = 0; k0 < nz; k0 += SZC) {
            // stage z in [k0 - R - 1, k0 - R - 1 + ZS) (clamped) of the tile's rows
            __syncthreads();
            const i64 zb = k0 - R - 1;
            // a warp per staged row (clamped row pointer once per row), lanes
            // along z (coalesced), ROWS / (warps) rows per warp with the
            // loads of two rows in flight; per-element index math was ~30% of
            // this kernel's instructions
            {
                constexpr int NWARP = NTC / 32, RPW = 2;  // rows per warp iteration
                static_assert(ZS <= 64, "two lanes' worth of z per row");
                const int lane = t & 31, wid = t >> 5;
                const int k0c = (int)ct::clampi(zb + lane, 0, nz - 1), k1c = (int)ct::clampi(zb + 32 + lane, 0, nz - 1);
                for (int r0 = wid * RPW; r0 < C::ROWS; r0 += NWARP * RPW) {
                    T v[RPW][2];
#pragma unroll
                    for (int q = 0; q < RPW; ++q) {
                        const int r = r0 + q;
                        const int di = r / (NTC + 2 * R), dj = r - di * (NTC + 2 * R);
                        const T *row = in + (ct::clampi(i + di - R, 0, nx - 1) * ny +
                                             ct::clampi(j0 + dj - R, 0, ny - 1)) * nz;
                        v[q][0] = (r < C::ROWS && lane < ZS) ? row[k0c] : (T)0;
                        v[q][1] = (r < C::ROWS && 32 + lane < ZS) ? row[k1c] : (T)0;
                    }
#pragma unroll
                    for (int q = 0; q < RPW; ++q) {
                        const int r = r0 + q;
                        if (r < C::ROWS) {
                            T *dst = (T *)(stg + r * RW);
                            if (lane < ZS) dst[lane] = v[q][0];
                            if (32 + lane < ZS) dst[32 + lane] = v[q][1];
                        }
                    }
                }
            }
            __syncthreads();
            if (!live) continue;
            if (k0 == 0) {  // window of k = 0: z offsets R+1-R .. R+1+R in the chunk
                for (int dk = 0; dk < D; ++dk)
#pragma unroll
                    for (int e = 0; e < D * D; ++e) {
                        const int v = sval(e / D, e % D, 1 + dk);
                        ++H(U16 ? v >> 8 : v);
                        if (U16 && (v >> 8) == 0) ++F(v & 255);
                    }
            }
            const int kend = (int)min((i64)SZC, nz - k0);
            for (int kc = 0; kc < kend; ++kc) {
                const i64 k = k0 + kc;
                if (k > 0) {  // leaves: z = k - 1 - R (offset kc), enters: z = k + R (offset kc + 2R + 1)
#pragma unroll
                    for (int e = 0; e < D * D; ++e) {
                        const int vo = sval(e / D, e % D, kc), vn = sval(e / D, e % D, kc + 2 * R + 1);
                        if (vo == vn) continue;
                        const int bo = U16 ? vo >> 8 : vo, bn = U16 ? vn >> 8 : vn;
                        hadd(hc, bo, -1);
                        hadd(hc, bn, 1);
                        below += (bn < m) - (bo < m);
                        if constexpr (U16) {
                            if (bo == hcur) {
                                hadd(hf, vo & 255, -1);
                                belowf -= (vo & 255) < mf;
                            }
                            if (bn == hcur) {
                                hadd(hf, vn & 255, 1);
                                belowf += (vn & 255) < mf;
                            }
                        }
                    }
                }
                // the bin holding rank KTH: below <= KTH < below + H(m)
                while (below + (int)H(m) <= KTH) below += H(m++);
                while (below > KTH) below -= H(--m);
                int med = m;
                if constexpr (U16) {
                    if (m != hcur) {  // re-describe the fine histogram for the new bin (window z offsets kc+1 ..)
                        for (int b = 0; b < 256; ++b) F(b) = 0;
                        for (int dk = 0; dk < D; ++dk)
#pragma unroll
                            for (int e = 0; e < D * D; ++e) {
                                const int v = sval(e / D, e % D, kc + 1 + dk);
                                if ((v >> 8) == m) ++F(v & 255);
                            }
                        hcur = m;
                        mf = 0;
                        belowf = 0;
                    }
                    const int rho = KTH - below;
                    while (belowf + (int)F(mf) <= rho) belowf += F(mf++);
                    while (belowf > rho) belowf -= F(--mf);
                    med = (m << 8) | mf;
                }
                CT_DCHECK(med >= 0 && med < (U16 ? 65536 : 256) && i < nx && j < ny);
                out[(i * ny + j) * nz + k] = (T)med;
                if (med == run_v) {
                    ++run_n;
                } else {
                    flush_run(run_v, run_n);
                    run_v = med;
                    run_n = 1;
                }
            }
        }
        if (live) flush_run(run_v, run_n);
    }
}

// Any radius (> 3: the (2r+1)^3 window no longer fits a per-thread buffer):
// bitwise radix select of the k-th smallest order-preserving key, one pass
// over the clamped window per key bit (8 / 16 / 64 for u8 / u16 / f64).
// Same order statistic as select_kth (scipy's rank filter, rank = size^3 // 2).
template <typename T>
__device__ __forceinline__ unsigned long long okey(T v) {
    if constexpr (sizeof(T) == 8) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(v);
        return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    } else {
        return (unsigned long long)v;
    }
}

template <typename T>
__device__ __forceinline__ T from_okey(unsigned long long k) {
    if constexpr (sizeof(T) == 8) {
        return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
    } else {
        return (T)k;
    }
}

template <typename T>
__global__ void __launch_bounds__(128) median_radix(const T *__restrict__ in, T *__restrict__ out, i64 nx, i64 ny,
                                                    i64 nz, int rad, uint64_t *__restrict__ ghist) {
    constexpr int BITS = 8 * (int)sizeof(T);
    const int size = 2 * rad + 1;
    const int kth = size * size * size / 2;
    const i64 n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
        unsigned long long prefix = 0;
        int rank = kth;
        for (int b = BITS - 1; b >= 0; --b) {
            const unsigned long long hi = b == 63 ? 0ull : (~0ull << (b + 1));
            int c0 = 0;  // window keys matching the prefix above bit b with bit b clear
            for (int di = -rad; di <= rad; ++di)
                for (int dj = -rad; dj <= rad; ++dj) {
                    const T *row = in + (ct::clampi(i + di, 0, nx - 1) * ny + ct::clampi(j + dj, 0, ny - 1)) * nz;
                    for (int dk = -rad; dk <= rad; ++dk) {
                        const unsigned long long key = okey<T>(row[ct::clampi(k + dk, 0, nz - 1)]);
                        c0 += ((key & hi) == prefix) & !((key >> b) & 1ull);
                    }
                }
            if (rank >= c0) {
                rank -= c0;
                prefix |= 1ull << b;
            }
        }
        const T m = from_okey<T>(prefix);
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
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    if (radius == 0) {
        const size_t es = dtype == CT_U8 ? 1 : (dtype == CT_U16 ? 2 : 8);
        cudaMemcpyAsync(out, in, n * es, cudaMemcpyDeviceToDevice, s);
        if (hist) return ct_histogram(out, dtype, n, hist, stream);
        return ct::check_launch("median copy");
    }
    if (radius == 1 && (dtype == CT_U8 || dtype == CT_U16) && nz <= 128) {
        const int W = (int)((nz + 31) / 32);
        const size_t es = dtype == CT_U8 ? 1 : 2;
        const size_t NW = (size_t)(BTI + 2) * (BTJ + 2) * W;
        const size_t pbytes = ((size_t)3 * (dtype == CT_U8 ? 8 : 16) * NW * 4 + 16 + 15) & ~(size_t)15;
        size_t sm = pbytes + (dtype == CT_U8 ? ct::ByteHist256::kBytes : 4096 * 4);
        const i64 tiles = ((nx + BTI - 1) / BTI) * ((ny + BTJ - 1) / BTJ);
        const int grid = (int)min(tiles, (i64)CT_NUM_SMS * 2);
        const bool al4 = ((uintptr_t)in & 3) == 0;
        // nz = 32 WC: the tile's input rows by TMA (3-D box [BTI+2][BTJ+2][nz])
        CUtensorMap tm;
        memset(&tm, 0, sizeof(tm));
        bool tma = (nz == 32 || nz == 64 || nz == 96 || nz == 128) && ((uintptr_t)in & 15) == 0 &&
                   nx < (1 << 30) && ny < (1 << 30);
        if (tma) {
            PFN_cuTensorMapEncodeTiled_v12000 encode = tma_encoder();
            const cuuint64_t dims[3] = {(cuuint64_t)nz, (cuuint64_t)ny, (cuuint64_t)nx};
            const cuuint64_t strides[2] = {(cuuint64_t)(nz * es), (cuuint64_t)(ny * nz * es)};
            const cuuint32_t box[3] = {(cuuint32_t)nz, BTJ + 2, BTI + 2}, est[3] = {1, 1, 1};
            tma = encode && encode(&tm, es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                                   (void *)in, dims, strides, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        if (tma) sm = ((sm + 127) & ~(size_t)127) + (size_t)(BTI + 2) * (BTJ + 2) * nz * es;
        if (dtype == CT_U8) {
            auto k = !al4 ? median3_bits<uint8_t, 8, 0>
                     : !tma ? median3_bits<uint8_t, 8, 0>
                     : nz == 64 ? median3_bits<uint8_t, 8, 2, true>
                     : nz == 32 ? median3_bits<uint8_t, 8, 1, true>
                     : nz == 96 ? median3_bits<uint8_t, 8, 3, true> : median3_bits<uint8_t, 8, 4, true>;
            if (al4 && !tma && nz % 32 == 0)
                k = nz == 64 ? median3_bits<uint8_t, 8, 2> : nz == 32 ? median3_bits<uint8_t, 8, 1>
                    : nz == 96 ? median3_bits<uint8_t, 8, 3> : median3_bits<uint8_t, 8, 4>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k<<<grid, 256, sm, s>>>((const uint8_t *)in, (uint8_t *)out, nx, ny, (int)nz, hist, tm);
        } else {
            auto k = !al4 ? median3_bits<uint16_t, 16, 0>
                     : !tma ? median3_bits<uint16_t, 16, 0>
                     : nz == 64 ? median3_bits<uint16_t, 16, 2, true>
                     : nz == 32 ? median3_bits<uint16_t, 16, 1, true>
                     : nz == 96 ? median3_bits<uint16_t, 16, 3, true> : median3_bits<uint16_t, 16, 4, true>;
            if (al4 && !tma && nz % 32 == 0)
                k = nz == 64 ? median3_bits<uint16_t, 16, 2> : nz == 32 ? median3_bits<uint16_t, 16, 1>
                    : nz == 96 ? median3_bits<uint16_t, 16, 3> : median3_bits<uint16_t, 16, 4>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k<<<grid, 256, sm, s>>>((const uint16_t *)in, (uint16_t *)out, nx, ny, (int)nz, hist, tm);
        }
        return ct::check_launch("median3_bits");
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
    if (radius >= 2 && radius <= 3 && (dtype == CT_U8 || dtype == CT_U16)) {
        auto launch = [&](auto kern, size_t sm, int ntc, auto *typed_in) {
            using TT = std::remove_pointer_t<decltype(typed_in)>;
            const i64 tiles = nx * ((ny + ntc - 1) / ntc);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            kern<<<(unsigned)min(tiles, (i64)CT_NUM_SMS * 16), ntc, sm, s>>>((const TT *)in, (TT *)out, nx, ny, nz,
                                                                              hist);
        };
        if (dtype == CT_U8) {
            if (radius == 2) launch(median_slide<uint8_t, 2>, SlideCfg<uint8_t, 2>::SMEM, SlideCfg<uint8_t, 2>::NTC, (uint8_t *)nullptr);
            else launch(median_slide<uint8_t, 3>, SlideCfg<uint8_t, 3>::SMEM, SlideCfg<uint8_t, 3>::NTC, (uint8_t *)nullptr);
        } else {
            if (radius == 2) launch(median_slide<uint16_t, 2>, SlideCfg<uint16_t, 2>::SMEM, SlideCfg<uint16_t, 2>::NTC, (uint16_t *)nullptr);
            else launch(median_slide<uint16_t, 3>, SlideCfg<uint16_t, 3>::SMEM, SlideCfg<uint16_t, 3>::NTC, (uint16_t *)nullptr);
        }
        return ct::check_launch("median_slide");
    }
    if (radius > 3) {
        CT_DISPATCH(dtype, T, {
            median_radix<T><<<ct::grid_for(n, 128), 128, 0, s>>>((const T *)in, (T *)out, nx, ny, nz, radius, hist);
        });
        return ct::check_launch("median_radix");
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
