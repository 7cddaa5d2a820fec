// k_gauss_tc.cu -- K1 on the 5th-generation tensor cores (tcgen05, kind::i8).
//
// Certified fast path of ct_gaussian_q (ref denoise.py:84-86, see k_gauss.cu):
// q = rint(max(raw - gaussian_filter(raw), 0)) for u8 volumes.  Each 1-D pass
// is a banded integer GEMM: the double taps w_j are scaled to 35-bit integers
// Q_j = rint(w_j 2^35) (2^34, ... when a tap >= 1/8) split into four 8-bit limbs, intermediates are 32-bit
// fixed point (24 fractional bits) split into four byte planes, and every
// limb product is accumulated exactly in int32 by UTCIMMA.  The result S is
// the convolution in fixed point (scale 2^43 for the default 35-bit taps) with a rigorously bounded error
// (weight rounding, truncation of intermediates, dropped limb pairs of weight
// < 2^-43, and scipy's own float64 rounding); voxels whose residual lies
// within that bound of a rounding boundary go to the fix list and are
// recomputed in scipy's exact operation order (fix_p1s / fix_p2q_s in k_gauss.cu).
//
//   pass x, y (strided axes): D[out row][col] = A[out row][in row] * B[in row][col]
//       A = the tap band (128 x 256, Toeplitz, constant) held in TMEM;
//       B = 256 input rows (clamped at the edges = mode "nearest") x TN
//       columns of a byte plane, MN-major in shared memory.
//   pass z (contiguous axis, nz in {32, 64, 96}): D[line][out k] = A[line][in k] * B[in k][out k]
//       A = 128 lines x nz bytes, K-major; B = the taps that land inside the
//       line (nz x nz, constant), K-major; both in SMEM.  The taps beyond the
//       line ends (mode "nearest": the edge values) are one more K = 32
//       block: A = the lines' edge values in TMEM, B = the tail tap sums.
// All three passes are warp-specialised and persistent (one CTA per SM): a
// TMA producer warp stages the operand boxes (cp.async.bulk.tensor, mbarrier
// complete_tx) into a ring, one warp issues the MMAs, 16 epilogue warps drain
// TMEM, so each tile's epilogue overlaps the next tile's MMAs (passes x, y:
// tc_pass_xy_ws, with an edge-fixer warp for the clamped rows; pass z:
// tc_pass_z_ws).
//   Limb pairs (a, b) with a + b >= 2 (data limb a, weight limb b) are kept;
//   pairs of equal a + b share an accumulator (5 accumulators).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "ct_common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int FW = 40;         // max weight scale bits (lowered per axis so that every Q_j < 2^32)
constexpr int FD = 24;         // fractional bits of the intermediates
constexpr int TM = 128;        // output rows per tile (passes x, y) / lines per tile (pass z)
constexpr int TNX = 64;        // columns per tile, pass x (4 accumulators: 256 + 4*64 TMEM columns)
constexpr int TNY = 32;        // columns per tile, pass y (5 accumulators: 256 + 5*32)
constexpr int KXY = 256;       // input rows per tile (passes x, y): TM + 2r <= 256
constexpr int PMAX = 65;       // max taps per side + 1

// lowest kept limb-pair sum (data limb a + weight limb b) for NP data planes
// and NL weight limbs: u8 (4 planes, 24 fractional bits; 4 limbs, taps < 2^32)
// keeps a + b >= 2; u16 (5 planes: 40-bit intermediates, 24-28 fractional
// bits; 5 limbs: taps < 2^40, the weight rounding 2^8 finer) keeps a + b >= 4;
// always 5 accumulators (a + b = LOP .. LOP + 4)
__host__ __device__ constexpr int lo_pair(int np, int nl = 4) { return np == 1 ? 0 : np + nl - 6; }

// Tap band rows for TMEM: tb[b][128 + x] = limb b of Q_|x - r| for 0 <= x <= 2r
// (0 elsewhere), so band word c of row m (K bytes 4c .. 4c+3, tap index
// kk - r - m) is the 4 bytes at tb[b][128 + 4c - m]: two aligned loads and a
// funnel shift instead of four compare-and-lookup byte builds.
constexpr int TBW = 392;  // bytes per limb row (128 + 256 + pad)
__device__ __forceinline__ void tap_rows(uint8_t (*tb)[TBW], const long long *Q, int r, int nl) {
    for (int e = threadIdx.x; e < nl * TBW; e += blockDim.x) {
        const int b = e / TBW, x = e - b * TBW - 128;
        const int j = x - r;
        tb[b][e - b * TBW] = (x >= 0 && x <= 2 * r) ? (uint8_t)((Q[j < 0 ? -j : j] >> (8 * b)) & 0xff) : 0;
    }
}
__device__ __forceinline__ uint32_t band_word(const uint8_t *tbb, int c, int m) {
    const int o = 128 + 4 * c - m;  // 1 .. 380
    const uint32_t *w = (const uint32_t *)(tbb + (o & ~3));
    return __funnelshift_r(w[0], w[1], 8 * (o & 3));
}


struct TcParams {
    long long Q[3][PMAX];  // integer taps per axis (Q[axis][|j|] = rint(w_j 2^fw[axis]))
    int fw[3];             // weight scale bits per axis (<= FW, four 8-bit limbs)
    int fd;                // fractional bits of the 32-bit intermediates: 32 - bits(vmax), in [16, FD]
    long long eps;         // certification threshold in units of 2^-(fw[2] + fd - 16)
    unsigned vmax;         // u16: the frame's maximum (tc_vmax); u8: 255
};

// u16 frames: the maximum sets the intermediates' integer bits (P1, P2 <=
// vmax), so 12-bit data keeps 20 fractional bits instead of 16
__global__ void __launch_bounds__(256) tc_vmax(const uint4 *__restrict__ raw, long long n16, TcParams *prm) {
    uint32_t m = 0;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n16; i += (long long)gridDim.x * 256) {
        const uint4 v = raw[i];
        m = max(m, __vmaxu2(__vmaxu2(v.x, v.y), __vmaxu2(v.z, v.w)));
    }
    m = max(m & 0xffffu, m >> 16);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(&prm->vmax, m);
}

// ---------------------------------------------------------------------------
// Setup: integer taps and the certified error bound (one warp per axis).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(96) tc_prep(const double *__restrict__ w, int rx, int ry, int rz, int u8, int np,
                                               int nl, double eps_override, TcParams *prm) {
    // warp a handles axis a: lane-parallel taps, warp reductions
    const int a = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned vm = u8 ? 255u : prm->vmax;  // tc_vmax ran before (u16)
    const double vmax = (double)vm;
    // P <= vmax (1 + (2r+1) 2^-fw) < 2^bits(vmax): 8 np - bits integer bits left for the fraction
    // (4 planes: <= 24; 5 planes: <= 28 -- 12-bit data keeps 28, full 16-bit 24)
    const int fd = min(np == 4 ? FD : 28, max(16, 8 * np - (vm ? 32 - __clz(vm) : 0)));
    const int lop = lo_pair(np, nl);  // kept limb pairs a + b >= lop
    const int rr[3] = {rx, ry, rz};
    const double *ws = a == 0 ? w : (a == 1 ? w + rx + 1 : w + rx + 1 + ry + 1);
    const int r = rr[a];
    double wmax = 0.0;  // largest tap (w_0)
    for (int j = lane; j <= r; j += 32) wmax = fmax(wmax, ws[j]);
    for (int o = 16; o; o >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    wmax *= 1.0000001;
    // taps Q_j < 2^(8 nl); pass z: fw <= 36 + 8 (nl - 4) keeps the edge tail
    // sums < 16 * 2^(8 nl - 1) (16 pieces, see tc_pass_z_ws)
    const double qmax = ldexp(1.0, 8 * nl) - 1.0;
    int fw = a == 2 ? 36 + 8 * (nl - 4) : FW + 8 * (nl - 4);
    while (fw > 24 && wmax * ldexp(1.0, fw) >= qmax) --fw;
    const double scale = ldexp(1.0, fw);
    double dq = 0.0, qsum[4] = {0.0, 0.0, 0.0, 0.0};  // qsum[b] = sum_j limb b of Q_j over taps -r..r
    for (int j = lane; j < PMAX; j += 32) {
        long long q = 0;
        if (j <= r) {
            const double x = ws[j] * scale;     // exact (power-of-two scaling)
            q = __double2ll_rn(x);
            const double mult = j ? 2.0 : 1.0;  // taps -j and +j
            dq += mult * fabs((double)q - x);   // exact difference
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) qsum[bb] += mult * (double)((q >> (8 * bb)) & 0xff);
        }
        prm->Q[a][j] = q;
    }
    for (int o = 16; o; o >>= 1) {
        dq += __shfl_xor_sync(0xffffffffu, dq, o);
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) qsum[bb] += __shfl_xor_sync(0xffffffffu, qsum[bb], o);
    }
    // per-axis bound: weight rounding sum_j |Q_j 2^-fw - w_j| * max input (the
    // inputs of passes y, z are bounded by vmax up to the taps' sum rounding)
    // plus, for y and z, the dropped limb pairs a + b < lop (data limbs <= 255)
    double b = dq / scale * vmax * 1.001;
    if (a == 2)  // pass z: every output column also holds 32 edge-tap pieces (limbs <= 255)
        for (int bb = 0; bb < 4; ++bb) qsum[bb] += 32.0 * 255.0;
    if (a > 0)
        for (int da = 0; da < lop; ++da)
            for (int bb = 0; da + bb < lop && bb < nl; ++bb)
                b += 255.0 * qsum[bb] * ldexp(1.0, 8 * (da + bb) - fw - fd);
    __shared__ double bs[3];
    __shared__ int fws[3];
    if (lane == 0) {
        bs[a] = b;
        fws[a] = fw;
        prm->fw[a] = fw;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        prm->fd = fd;
        prm->vmax = vm;
        const int zs = fws[2] + fd - 8 * lop;  // scale bits of the final sum
        double bound = bs[0] + bs[1] + bs[2];
        bound += 2.0 * ldexp(1.0, -fd);                               // truncation of P1, P2
        bound += 4.0 * (rx + ry + rz + 12) * ldexp(1.0, -53) * vmax;  // scipy float64 order + residual
        prm->eps = (long long)ceil(bound * 1.25 * ldexp(1.0, zs)) + 16;
        if (eps_override > 0.0) prm->eps = (long long)ceil(eps_override * ldexp(1.0, zs));
    }
}



__device__ __forceinline__ uint32_t limb(long long q, int b) { return (uint32_t)((q >> (8 * b)) & 0xff); }

// S += v 2^k for a compile-time k (after unrolling): one IMAD.WIDE.U32 below
// 2^32, a high-word add above
__device__ __forceinline__ void acc_pow2(unsigned long long &S, uint32_t v, int k) {
    if (k < 32) S += (unsigned long long)v * (uint32_t)(1u << k);
    else S += (unsigned long long)v << k;
}

// Mixed-radix cursor over a CTA's tiles: tile t0 + k gs has digits (o, ti,
// cb) (cb fastest); advancing by gs adds gs's digits with carries, so the
// per-tile coordinates cost no division.
struct TileCur {
    int o, ti, cb, go, gti, gcb, nti, ncb;
    __device__ TileCur(long long t0, long long gs, int nti_, int ncb_) : nti(nti_), ncb(ncb_) {
        long long r = t0 / ncb;
        cb = (int)(t0 - r * ncb);
        ti = (int)(r % nti);
        o = (int)(r / nti);
        r = gs / ncb;
        gcb = (int)(gs - r * ncb);
        gti = (int)(r % nti);
        go = (int)(r / nti);
    }
    __device__ __forceinline__ void next() {
        cb += gcb;
        int c = cb >= ncb;
        if (c) cb -= ncb;
        ti += gti + c;
        c = ti >= nti;
        if (c) ti -= nti;
        o += go + c;
    }
};

// byte a of four u32 values -> one u32 (plane words), all four planes
__device__ __forceinline__ void planes4(uint32_t o0, uint32_t o1, uint32_t o2, uint32_t o3, uint32_t (&p)[4]) {
    const uint32_t l01 = __byte_perm(o0, o1, 0x5140), h01 = __byte_perm(o0, o1, 0x7362);
    const uint32_t l23 = __byte_perm(o2, o3, 0x5140), h23 = __byte_perm(o2, o3, 0x7362);
    p[0] = __byte_perm(l01, l23, 0x5410);
    p[1] = __byte_perm(l01, l23, 0x7632);
    p[2] = __byte_perm(h01, h23, 0x5410);
    p[3] = __byte_perm(h01, h23, 0x7632);
}

// ---------------------------------------------------------------------------
// Passes x and y, warp-specialised:
//   warp 0      TMA producer: one cp.async.bulk.tensor box per tile (256
//               input rows x TN columns of every byte plane) into a ring of
//               SSTG shared-memory stages (full / empty mbarriers);
//   warp 1      TMEM owner and MMA issuer: the tap band A lives in TMEM
//               columns [0, 256); ASTG accumulator sets follow, so MMA(k+1)
//               runs while the epilogue drains set k (afull / aempty);
//   warp 2      edge fixer: rows of a box that fall outside [0, L) arrive
//               zero-filled; it replaces them by the edge row (mode "nearest")
//               and releases the stage to the MMA warp (ready) -- off the MMA
//               warp's critical path (when the MMA warp did it, the 2 of 8
//               tiles per column at the volume's faces stalled the tensor pipe);
//   warps 3..18 epilogue: TMEM -> registers, combine the limb accumulators in
//               exact 64-bit integers, split into the next pass's byte planes,
//               staged in 64B / 32B-swizzled shared memory and stored by one
//               TMA tensor store per tile (warp w reads TMEM lane quarter
//               w % 4, column group (w - 3) / 4).
// ---------------------------------------------------------------------------
constexpr int WS_EPI = 16;                 // epilogue warps (4 per TMEM lane quarter)
constexpr int WS_NT = 32 * (2 + WS_EPI);   // 576 threads (pass z)
constexpr int WSX_NT = 32 * (3 + WS_EPI);  // 608 threads (passes x, y: + the edge fixer)

__device__ __forceinline__ void epi_bar() {  // named barrier 1: the epilogue warps only
    asm volatile("bar.sync 1, %0;" ::"n"(32 * WS_EPI) : "memory");
}

// DB = bytes per input voxel: 2 for raw u16 (pass x), read as a byte matrix
// of twice the width -- column 2c holds the low bytes of voxel c, column
// 2c + 1 the high bytes, so the MMA yields both limb sums and the epilogue
// combines S(c) = D[2c] + 256 D[2c + 1] (no de-interleave pass).
template <int NPIN, int TN, int SSTG, int ASTG, int DB = 1, int NPO = 4, int NL = 4>
__global__ void __launch_bounds__(WSX_NT, 1) tc_pass_xy_ws(const __grid_constant__ CUtensorMap tmap,
                                                          const __grid_constant__ CUtensorMap tmo, int L, int inner,
                                                          int outer, const TcParams *__restrict__ prm, int axis,
                                                          int r) {
    static_assert(DB == 1 || NPIN == 1, "u16 input only for the raw pass");
    constexpr int NACC = NPIN == 1 ? NL : 5;
    constexpr bool PERACC = NPIN == 1 && DB == 1;  // accumulators released one by one (pass x, u8)
    constexpr int AG = 3;                           // pass y: accumulators [0, AG) released first
    constexpr int AB = 64 * NL;  // TMEM columns of the tap band
    // operand stage: one TMA box per tile, [NPIN planes][KXY rows][TN bytes] in
    // the TMA's TN-byte swizzle = the MMA's MN-major SWIZZLE_32B / 64B
    // canonical layout (one atom across N; 8-row groups 8 TN bytes apart),
    // full 32-byte sectors per request
    static_assert(TN == 32 || TN == 64, "swizzled operand rows");
    constexpr int PB = KXY * TN;                    // bytes per plane
    constexpr int SB = NPIN * PB;                   // bytes per stage
    constexpr uint32_t LBO = PB, SBO = 8 * TN;
    constexpr int CW = TN / 4;                      // (byte) columns per epilogue thread (4 column groups)
    constexpr int TV = TN / DB;                     // voxels per tile row
    // staged output tile [NPO planes][128 rows][TV bytes], stored by one TMA
    // box per tile (tmo): rows of TV = 64 / 32 bytes in the TMA's 64B / 32B
    // swizzle (16-byte chunk c of row m at c ^ ((m >> 1) & 3) / c ^ ((m >> 2)
    // & 1)), so that the epilogue's row stores spread over the banks
    constexpr int OBUF = NPO * TM * TV;
    constexpr int VB = CW / DB;                     // output bytes per thread, row and plane (16, 8, 4)
    static_assert(TV == 64 || TV == 32 || TV == 16, "output row");
    auto soff = [](int m, int byte) {                // swizzled byte offset within a plane of the staged tile
        const int c = byte >> 4, key = TV == 64 ? (m >> 1) & 3 : TV == 32 ? (m >> 2) & 1 : 0;
        return m * TV + ((c ^ key) << 4) + (byte & 15);
    };
    static_assert(AB + ASTG * NACC * TN <= 512, "TMEM: band + accumulator sets");
    extern __shared__ __align__(1024) uint8_t sm[];  // [SSTG][SB] operand stages, [2][OBUF] output tiles
    uint8_t *sout = sm + SSTG * SB;
    // aempty[a][acc]: accumulator acc of set a drained -- pass x releases them one
    // by one, so the next tile's MMAs into accumulator 0 start while the others
    // drain (100 -> 90 us on C2); pass y releases the set at once (aempty[a][0])
    __shared__ uint64_t full[SSTG], ready[SSTG], empty[SSTG], afull[ASTG], aempty[ASTG][NACC];
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, wp = t >> 5, lane = t & 31;
    if (wp == 1) tc::tmem_alloc(&tbase, 512);
    if (t == 0) {
        for (int i = 0; i < SSTG; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&ready[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < ASTG; ++i) {
            tc::mbar_init(&afull[i], 1);
            for (int j = 0; j < NACC; ++j) tc::mbar_init(&aempty[i][j], WS_EPI);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap);
        tc::tma_prefetch_desc(&tmo);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t base = tbase;
    // epilogue warp e = wp - 3: TMEM lane quarter q = wp % 4 (hardware rule),
    // column group cg = e / 4; it writes band limb cg of its rows into TMEM
    const int e_w = wp - 3, q = wp & 3, cg = e_w >> 2, m = 32 * q + lane;
    const uint32_t la = base + ((uint32_t)(32 * q) << 16);
    {
        __shared__ __align__(16) uint8_t tb[NL][TBW];
        tap_rows(tb, prm->Q[axis], r, NL);
        __syncthreads();
        if (wp >= 3) {
            for (int b = cg; b < NL; b += 4)
                for (int c0 = 0; c0 < KXY / 4; c0 += 8) {
                    uint32_t v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = band_word(tb[b], c0 + i, m);
                    tc::tmem_st8(la + b * 64 + c0, v);
                }
            tc::tmem_st_wait();
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();

    const int nti = (L + TM - 1) / TM, ncb = inner / TN;
    const long long ntiles = (long long)outer * nti * ncb;
    const long long t0 = blockIdx.x, gs = gridDim.x;
    const long long nmine = t0 < ntiles ? (ntiles - 1 - t0) / gs + 1 : 0;
    TileCur cur(t0, gs, nti, ncb);  // each role walks its tiles k = 0, 1, ... in order
    if (wp == 0) {
        // ---- TMA producer ----
        for (long long k = 0; k < nmine; ++k) {
            const int s = (int)(k % SSTG);
            tc::mbar_wait(&empty[s], (uint32_t)((k / SSTG) & 1) ^ 1u);
            const int o = cur.o, ti = cur.ti, cb = cur.cb;
            cur.next();
            if (lane == 0) {
                tc::mbar_expect_tx(&full[s], SB);
                uint8_t *dst = sm + s * SB;
                if constexpr (NPIN == 1)
                    tc::tma_load_2d(dst, &tmap, cb * TN, ti * TM - r, &full[s]);
                else
                    tc::tma_load_4d(dst, &tmap, cb * TN, ti * TM - r, o, 0, &full[s]);
            }
            __syncwarp();
        }
    } else if (wp == 2) {
        // ---- edge fixer ----
        for (long long k = 0; k < nmine; ++k) {
            const int s = (int)(k % SSTG);
            tc::mbar_wait(&full[s], (uint32_t)((k / SSTG) & 1));
            const int ti = cur.ti;
            cur.next();
            const int g0 = ti * TM - r;  // global row of box row 0
            if (g0 < 0 || g0 + KXY > L) {
                // box rows outside [0, L) came back zero-filled: clamp to the edge rows
                // (16-byte chunk c of row kk sits at chunk c ^ key(kk) of the row)
                uint8_t *st = sm + s * SB;
                const int lo = -g0, hi = L - 1 - g0;
                constexpr int CPR = TN / 16;
                auto key = [](int kk) { return TN == 64 ? (kk >> 1) & 3 : (kk >> 2) & 1; };
                for (int e = lane; e < NPIN * KXY * CPR; e += 32) {
                    const int c = e % CPR, kk = (e / CPR) % KXY, pl = e / (CPR * KXY);
                    const int src = kk < lo ? lo : (kk > hi ? hi : -1);
                    if (src >= 0)
                        *(uint4 *)(st + pl * PB + kk * TN + 16 * (c ^ key(kk))) =
                            *(const uint4 *)(st + pl * PB + src * TN + 16 * (c ^ key(src)));
                }
                tc::fence_async_smem();
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&ready[s]);
        }
    } else if (wp == 1) {
        // ---- MMA issuer ----
        const uint32_t idesc = tc::idesc_i8(TM, TN, false, false, false, true);
        for (long long k = 0; k < nmine; ++k) {
            const int s = (int)(k % SSTG), a = (int)(k % ASTG);
            tc::mbar_wait(&ready[s], (uint32_t)((k / SSTG) & 1));
            const uint64_t d0 = tc::smem_desc_sw(tc::smem_u32(sm + s * SB), LBO, SBO, TN);
            if constexpr (PERACC) {
                // pass x: the MMAs grouped by accumulator (= weight limb), each group
                // issued as soon as its accumulator of the previous tile is drained
#pragma unroll
                for (int acc = 0; acc < NACC; ++acc) {
                    tc::mbar_wait(&aempty[a][acc], (uint32_t)((k / ASTG) & 1) ^ 1u);
                    tc::fence_after();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < KXY / 32; ++ks)
                            tc::mma_i8_ts(base + AB + (a * NACC + acc) * TN, base + acc * 64 + ks * 8,
                                          d0 + (uint64_t)((ks * 32 * TN) >> 4), idesc, ks == 0 ? 0u : 1u);
                    }
                    __syncwarp();
                }
            } else {
                // pass y: plane-major order (consecutive MMAs share the B plane); the
                // accumulators are released in two groups ([0, AG) and [AG, NACC)):
                // the pairs into the first group come first in this order
                tc::mbar_wait(&aempty[a][0], (uint32_t)((k / ASTG) & 1) ^ 1u);
                tc::fence_after();
                if (tc::elect_one()) {
                    bool first[NACC], g1 = NPIN == 1;
#pragma unroll
                    for (int s2 = 0; s2 < NACC; ++s2) first[s2] = true;
#pragma unroll
                    for (int da = 0; da < NPIN; ++da)
#pragma unroll
                        for (int b = 0; b < NL; ++b) {
                            const int acc = da + b - lo_pair(NPIN, NL);
                            if (acc < 0 || acc >= NACC) continue;
                            if (acc >= AG && !g1) {
                                tc::mbar_wait(&aempty[a][1], (uint32_t)((k / ASTG) & 1) ^ 1u);
                                tc::fence_after();
                                g1 = true;
                            }
#pragma unroll
                            for (int ks = 0; ks < KXY / 32; ++ks)
                                tc::mma_i8_ts(base + AB + (a * NACC + acc) * TN, base + b * 64 + ks * 8,
                                              d0 + (uint64_t)((da * PB + ks * 32 * TN) >> 4), idesc,
                                              first[acc] && ks == 0 ? 0u : 1u);
                            first[acc] = false;
                        }
                }
                __syncwarp();
            }
            if (tc::elect_one()) {
                tc::mma_commit(&empty[s]);  // stage s free once these MMAs have read it
                tc::mma_commit(&afull[a]);  // accumulator set a complete
            }
            __syncwarp();
        }
    } else {
        // ---- epilogue: row m, columns [h, h + CW) of every tile ----
        const int h = CW * cg;
        const int et = t - 96;  // 0 .. 32 * WS_EPI - 1
        // output = S >> shift: S has scale 2^fw (x) or 2^(FD + fw - 16) (y); P has FD bits
        const int shift_out = NPIN == 1 ? prm->fw[axis] - prm->fd : prm->fw[axis] - 8 * lo_pair(NPIN, NL);
        for (long long k = 0; k < nmine; ++k) {
            const int a = (int)(k % ASTG);
            tc::mbar_wait(&afull[a], (uint32_t)((k / ASTG) & 1));
            tc::fence_after();
            uint32_t v[NACC][CW];
#pragma unroll
            for (int acc = 0; acc < NACC; ++acc) {
                if constexpr (CW % 8 == 0) {
#pragma unroll
                    for (int g8 = 0; g8 < CW; g8 += 8)
                        tc::tmem_ld8(la + AB + (a * NACC + acc) * TN + h + g8,
                                     *reinterpret_cast<uint32_t(*)[8]>(&v[acc][g8]));
                } else {
                    tc::tmem_ld4(la + AB + (a * NACC + acc) * TN + h, *reinterpret_cast<uint32_t(*)[4]>(&v[acc][0]));
                }
                if constexpr (PERACC) {  // pass x: release accumulator by accumulator
                    tc::tmem_ld_wait();
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&aempty[a][acc]);  // MMA(k + ASTG) may overwrite accumulator acc
                }
                if constexpr (!PERACC && NPIN > 1) {  // pass y: first group released after its loads
                    if (acc == AG - 1) {
                        tc::tmem_ld_wait();
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&aempty[a][0]);
                    }
                }
            }
            if constexpr (!PERACC) {  // pass y: the second group; u16 pass x: the whole set (aempty[a][0])
                tc::tmem_ld_wait();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&aempty[a][NPIN > 1 ? 1 : 0]);
            }
            uint8_t *ob = sout + (int)(k & 1) * OBUF;
            uint32_t pw[NPO][VB / 4];  // the thread's VB output bytes of every plane
#pragma unroll
            for (int g4 = 0; g4 < CW; g4 += 4 * DB) {
                uint32_t ov[4], o4 = 0;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    unsigned long long S = 0;
#pragma unroll
                    for (int acc = 0; acc < NACC; ++acc) {
                        acc_pow2(S, v[acc][g4 + DB * c], 8 * acc);
                        if constexpr (DB == 2) acc_pow2(S, v[acc][g4 + 2 * c + 1], 8 * acc + 8);
                    }
                    const unsigned long long o = S >> shift_out;
                    ov[c] = (uint32_t)o;
                    if constexpr (NPO == 5) o4 |= (uint32_t)((o >> 32) & 0xff) << (8 * c);
                }
                uint32_t pl[4];
                planes4(ov[0], ov[1], ov[2], ov[3], pl);
#pragma unroll
                for (int pa = 0; pa < 4; ++pa) pw[pa][g4 / (4 * DB)] = pl[pa];
                if constexpr (NPO == 5) pw[4][g4 / (4 * DB)] = o4;
            }
#pragma unroll
            for (int pa = 0; pa < NPO; ++pa) {
                uint8_t *d = ob + pa * TM * TV + soff(m, h / DB);
                if constexpr (VB == 16) *(uint4 *)d = make_uint4(pw[pa][0], pw[pa][1], pw[pa][2], pw[pa][3]);
                else if constexpr (VB == 8) *(uint2 *)d = make_uint2(pw[pa][0], pw[pa][1]);
                else *(uint32_t *)d = pw[pa][0];
            }
            tc::fence_async_smem();                 // the staged tile -> visible to the TMA store
            if (et == 0) tc::bulk_wait_read<0>();  // tile k-1's store has read its buffer (reused by k+1)
            epi_bar();
            const int o = cur.o, ti = cur.ti, cb = cur.cb;
            cur.next();
            if (et == 0) {
                tc::tma_store_4d(&tmo, ob, cb * TV, ti * TM, o, 0);
                tc::bulk_commit();
            }
        }
        if (et == 0) tc::bulk_wait<0>();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (wp == 1) tc::tmem_dealloc(base, 512);
}

// The exact test and quantisation of one pass-z voxel from its accumulator
// sum S (scale 2^zs):  V = S - 2^(zs-1), q = max(raw - ceil(V / 2^zs), 0)
// (= rint(max(raw - bg, 0))), and the voxel goes to the fix list iff
// (eps - V) mod 2^zs <= 2 eps and raw 2^zs - V >= 2^zs - eps (a rounding
// boundary within the certified error, with raw - bg possibly >= 1/2).  Out
// of line, so the rare lanes that need it cost the fast epilogue no
// registers.
__device__ __noinline__ uint32_t qz_exact(const TcParams *__restrict__ prm, int spl, unsigned long long S, uint32_t rv,
                                          unsigned long long idx, unsigned long long *__restrict__ fix, long long cap) {
    const long long eps = prm->eps;
    const int zs = prm->fw[2] + prm->fd - spl;
    const long long half = 1ll << (zs - 1), one = 1ll << zs, fmask = one - 1;
    const long long V = (long long)S - half;
    const int qv = (int)rv - (int)((V + fmask) >> zs);
    if ((unsigned long long)((eps - V) & fmask) <= (unsigned long long)(2 * eps) && ((long long)rv << zs) - V >= one - eps) {
        const unsigned long long at = atomicAdd(&fix[0], 1ull);
        if ((long long)at < cap) fix[2 + at] = idx;
        else fix[1] = 1;
    }
    return qv > 0 ? (uint32_t)qv : 0u;
}

// RAWG: the epilogue reads raw straight from global memory (prefetched at the
// tile's start) instead of a staged copy, so that a 2-byte raw tile does not
// cost a pipeline stage (u16: 4 stages of 5 planes fit, 3 with staged raw)
template <int NZ, int SSTG, typename Traw = uint8_t, int NP = 4, int NL = 4, bool RAWG = false>
__global__ void __launch_bounds__(WS_NT, 1) tc_pass_z_ws(const __grid_constant__ CUtensorMap tmp,
                                                         const __grid_constant__ CUtensorMap tmr, long long nlines,
                                                         const TcParams *__restrict__ prm, int r,
                                                         const Traw *__restrict__ raw, Traw *__restrict__ q,
                                                         unsigned long long *__restrict__ fix, long long cap) {
    constexpr int RB = (int)sizeof(Traw);
    constexpr int LOP = lo_pair(NP, NL), SPL = 8 * LOP;
    constexpr int NCH = NZ / 16;
    constexpr uint32_t LBOB = 128, SBOB = NCH * 128, SBOE = 256;  // taps (K-major): in-line band, edge block
    constexpr uint32_t PLB = TM * 16;                                // bytes per plane per chunk
    constexpr uint32_t LBOA = NP * PLB, SBOA = 128;                  // staged data planes
    constexpr int DB = NCH * NP * PLB;                               // data bytes per stage
    constexpr int RBT = RAWG ? 0 : TM * NZ * RB;                     // raw bytes per stage
    constexpr int SB = DB + RBT;
    constexpr int BW = NZ * NZ, BE = NZ * 32;
    constexpr int ACOL = 5 * NZ;
    // edge blocks: two slots when they fit (tile k+2's block is written right
    // after afull(k), off the MMA's critical path; needs SSTG >= 3 so that its
    // stage is not the one the writer still holds), else one (tile k+1's)
    constexpr int ES = ACOL + 2 * NP * 8 <= 512 && SSTG >= 3 ? 2 : 1;
    static_assert(ACOL + ES * NP * 8 <= 512, "TMEM");
    static_assert(NZ % 32 == 0 && NZ <= 96, "pass z tile");
    constexpr int CW = NZ / 4;  // columns per epilogue thread
    extern __shared__ __align__(1024) uint8_t sm[];  // [SSTG][SB] stages, [NL][BW] taps, [NL][BE] edge taps
    uint8_t *sw = sm + SSTG * SB;
    uint8_t *swe = sw + NL * BW;
    __shared__ uint64_t full[SSTG], empty[SSTG], afull, aempty, efull[ES];
    __shared__ uint32_t tbase;
    __shared__ long long Qs[PMAX], Ts[PMAX + 1];
    const int t = threadIdx.x, wp = t >> 5, lane = t & 31;
    if (wp == 1) tc::tmem_alloc(&tbase, 512);
    for (int j = t; j < PMAX; j += WS_NT) Qs[j] = j <= r ? prm->Q[2][j] : 0;
    if (t == 0) {
        for (int i = 0; i < SSTG; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1 + WS_EPI);  // the MMA commit + every epilogue warp (raw read)
        }
        tc::mbar_init(&afull, 1);
        tc::mbar_init(&aempty, WS_EPI);
        for (int i = 0; i < ES; ++i) tc::mbar_init(&efull[i], 4);
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmp);
        tc::tma_prefetch_desc(&tmr);
    }
    __syncthreads();
    if (t == 0) {
        Ts[PMAX] = 0;
        for (int j = PMAX - 1; j >= 0; --j) Ts[j] = Ts[j + 1] + Qs[j];
    }
    __syncthreads();
    for (int e = t; e < NZ * NZ; e += WS_NT) {
        const int n = e / NZ, k = e - n * NZ;
        const int d = k > n ? k - n : n - k;
        const long long qv = d < PMAX ? Qs[d] : 0;
#pragma unroll
        for (int b = 0; b < NL; ++b) sw[b * BW + tc::kmajor_off(n, k, LBOB, SBOB)] = (uint8_t)limb(qv, b);
    }
    for (int e = t; e < NZ * 32; e += WS_NT) {
        const int n = e >> 5, sl = e & 31, s16 = sl & 15;
        const long long E = sl < 16 ? (n + 1 <= PMAX ? Ts[n + 1] : 0) : (NZ - n <= PMAX ? Ts[NZ - n] : 0);
        const long long pc = E / 16 + (s16 < E % 16 ? 1 : 0);
#pragma unroll
        for (int b = 0; b < NL; ++b) swe[b * BE + tc::kmajor_off(n, sl, LBOB, SBOE)] = (uint8_t)limb(pc, b);
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t base = tbase;
    const long long ntiles = (nlines + TM - 1) / TM;
    const long long t0 = blockIdx.x, gs = gridDim.x;
    const long long nmine = t0 < ntiles ? (ntiles - 1 - t0) / gs + 1 : 0;

    if (wp == 0) {
        // ---- TMA producer ----
        for (long long k = 0; k < nmine; ++k) {
            const int s = (int)(k % SSTG);
            tc::mbar_wait(&empty[s], (uint32_t)((k / SSTG) & 1) ^ 1u);
            if (lane == 0) {
                const int l0 = (int)((t0 + k * gs) * TM);
                uint8_t *dst = sm + s * SB;
                tc::mbar_expect_tx(&full[s], SB);
#pragma unroll
                for (int c = 0; c < NCH; ++c) tc::tma_load_3d(dst + c * NP * PLB, &tmp, 16 * c, l0, 0, &full[s]);
                if constexpr (!RAWG) tc::tma_load_2d(dst + DB, &tmr, 0, l0, &full[s]);
            }
            __syncwarp();
        }
    } else if (wp == 1) {
        // ---- MMA issuer ----
        const uint32_t idesc = tc::idesc_i8(TM, NZ, false, false, false, false);
        const uint64_t b0 = tc::smem_desc(tc::smem_u32(sw), LBOB, SBOB);
        const uint64_t be = tc::smem_desc(tc::smem_u32(swe), LBOB, SBOE);
        for (long long k = 0; k < nmine; ++k) {
            const int s = (int)(k % SSTG);
            tc::mbar_wait(&full[s], (uint32_t)((k / SSTG) & 1));
            tc::mbar_wait(&aempty, (uint32_t)(k & 1) ^ 1u);
            tc::mbar_wait(&efull[k % ES], (uint32_t)((k / ES) & 1));
            tc::fence_after();
            if (tc::elect_one()) {
                const uint64_t a0 = tc::smem_desc(tc::smem_u32(sm + s * SB), LBOA, SBOA);
                bool first[5] = {true, true, true, true, true};
#pragma unroll
                for (int a = 0; a < NP; ++a)
#pragma unroll
                    for (int b = 0; b < NL; ++b) {
                        const int acc = a + b - LOP;
                        if (acc < 0 || acc > 4) continue;
#pragma unroll
                        for (int ks = 0; ks < NZ / 32; ++ks)
                            tc::mma_i8_ss(base + NZ * acc, a0 + (uint64_t)((a * PLB + ks * 2 * LBOA) >> 4),
                                          b0 + (uint64_t)((b * BW + ks * 2 * LBOB) >> 4), idesc,
                                          first[acc] && ks == 0 ? 0u : 1u);
                        tc::mma_i8_ts(base + NZ * acc, base + ACOL + (int)(k % ES) * NP * 8 + a * 8,
                                      be + (uint64_t)((b * BE) >> 4), idesc, 1u);
                        first[acc] = false;
                    }
                tc::mma_commit(&empty[s]);
                tc::mma_commit(&afull);
            }
            __syncwarp();
        }
    } else {
        // ---- epilogue: line m of every tile, columns [h0, h0 + CW) ----
        const int qq = wp & 3, cg = (wp - 2) >> 2, m = 32 * qq + lane, h0 = cg * CW;
        const uint32_t la = base + ((uint32_t)(32 * qq) << 16);
        // Y = S + half + eps: the certification test is (Y mod 2^zs) <= 2 eps and,
        // when it fails, Y >> zs = ceil((S - half) / 2^zs) (no borrow from the low bits; qz_exact).  For
        // 32 <= zs < 64 and 2 eps < 2^32 the fast path reads bgq from Y's high
        // word and tests the top 32 fractional bits conservatively; otherwise
        // (fth = ~0) every voxel takes the exact path
        const long long eps = prm->eps;
        const int zs = prm->fw[2] + prm->fd - SPL;
        const bool fast = zs >= 32 && zs < 64 && 2 * eps < (1ll << 32);
        const unsigned long long Cy = (unsigned long long)((1ll << (zs - 1)) + eps);
        const uint32_t hsh = fast ? (uint32_t)(zs - 32) : 0u;
        const uint32_t fth = fast ? (uint32_t)((2 * eps) >> hsh) : 0xffffffffu;
        // the edge block of tile k (cg = 0 warps): staged edge bytes -> TMEM slots
        auto edge = [&](long long k) {
            const int s = (int)(k % SSTG);
            tc::mbar_wait(&full[s], (uint32_t)((k / SSTG) & 1));
            const uint8_t *st = sm + s * SB + m * 16;
#pragma unroll
            for (int a = 0; a < NP; ++a) {
                const uint32_t w0 = 0x01010101u * st[a * PLB], wl = 0x01010101u * st[(NCH - 1) * NP * PLB + a * PLB + 15];
                const uint32_t v[8] = {w0, w0, w0, w0, wl, wl, wl, wl};
                tc::tmem_st8(la + ACOL + (int)(k % ES) * NP * 8 + a * 8, v);
            }
            tc::tmem_st_wait();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&efull[k % ES]);
        };
        if (cg == 0)
            for (int k = 0; k < ES && k < nmine; ++k) edge(k);
        for (long long k = 0; k < nmine; ++k) {
            const int s = (int)(k % SSTG);
            const long long l = (t0 + k * gs) * TM + m;
            const bool live = l < nlines;
            // RAWG: the tile's raw words, in flight during the wait and the drain
            uint32_t rg[RAWG ? CW * RB / 4 : 1];
            if constexpr (RAWG) {
                static_assert(CW * RB % 16 == 0, "16-byte raw loads");
                const uint4 *src = (const uint4 *)((const uint8_t *)raw + ((live ? l : 0) * NZ + h0) * RB);
#pragma unroll
                for (int i = 0; i < CW * RB / 16; ++i) {
                    const uint4 x = __ldg(src + i);
                    rg[4 * i] = x.x; rg[4 * i + 1] = x.y; rg[4 * i + 2] = x.z; rg[4 * i + 3] = x.w;
                }
            }
            tc::mbar_wait(&afull, (uint32_t)(k & 1));
            tc::fence_after();
            // Y = S + half + eps per column.  CW <= 16: all accumulator words are
            // loaded, then released (MMA(k+1) waits only for the loads), then
            // combined; CW = 24 (NZ = 96): in 8-column groups (registers)
            uint32_t yh[CW], yl[CW];
            auto ycomb = [&](const uint32_t(&v)[5][8], int g8) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    unsigned long long Y = (((unsigned long long)v[4][c] << 32) | v[0][c]) + Cy;
                    Y += (unsigned long long)v[1][c] * 0x100u;
                    Y += (unsigned long long)v[2][c] * 0x10000u;
                    Y += (unsigned long long)v[3][c] * 0x1000000u;
                    yh[g8 + c] = (uint32_t)(Y >> 32);
                    yl[g8 + c] = (uint32_t)Y;
                }
            };
            if constexpr (CW <= 16) {
                uint32_t v[CW / 8][5][8];
#pragma unroll
                for (int g = 0; g < CW / 8; ++g)
#pragma unroll
                    for (int acc = 0; acc < 5; ++acc) tc::tmem_ld8(la + NZ * acc + h0 + 8 * g, v[g][acc]);
                tc::tmem_ld_wait();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&aempty);  // MMA(k+1) may overwrite the accumulators
#pragma unroll
                for (int g = 0; g < CW / 8; ++g) ycomb(v[g], 8 * g);
            } else {
#pragma unroll
                for (int g8 = 0; g8 < CW; g8 += 8) {
                    uint32_t v[5][8];
#pragma unroll
                    for (int acc = 0; acc < 5; ++acc) tc::tmem_ld8(la + NZ * acc + h0 + g8, v[acc]);
                    tc::tmem_ld_wait();
                    ycomb(v, g8);
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&aempty);
            }
            if (cg == 0 && k + ES < nmine) edge(k + ES);
            // raw of the tile (stage s, already landed: MMA(k) consumed it), then release the stage
            // the thread's CW * RB raw / q bytes move in 16-byte chunks (8-byte when
            // h0 * RB is not 16-aligned: NZ = 96)
            constexpr int QW = CW * RB / 4;  // 32-bit words
            static_assert(CW * RB % 8 == 0, "raw row chunk");
            uint32_t rw[QW];
            if constexpr (RAWG) {
#pragma unroll
                for (int i = 0; i < QW; ++i) rw[i] = rg[i];
            } else {
            tc::mbar_wait(&full[s], (uint32_t)((k / SSTG) & 1));
            const uint8_t *rl = sm + s * SB + DB + (m * NZ + h0) * RB;
            if constexpr (CW * RB % 16 == 0) {
#pragma unroll
                for (int i = 0; i < QW / 4; ++i) {
                    const uint4 x = *(const uint4 *)(rl + 16 * i);
                    rw[4 * i] = x.x; rw[4 * i + 1] = x.y; rw[4 * i + 2] = x.z; rw[4 * i + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < QW / 2; ++i) {
                    const uint2 x = *(const uint2 *)(rl + 8 * i);
                    rw[2 * i] = x.x; rw[2 * i + 1] = x.y;
                }
            }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[s]);
            // fast path for every column: bgq = Y >> zs, q = max(raw - bgq, 0) as
            // SIMD bytes (u8) / halves (u16); a conservative certification test on
            // the top 32 fractional bits (bits [zs - 32, zs) of Y, one funnel
            // shift) marks lanes that need the exact test below
            constexpr int VPW = 4 / RB;
            constexpr uint32_t VM = RB == 1 ? 0xffu : 0xffffu;
            uint32_t qw[QW];
            bool anyn = false;
#pragma unroll
            for (int i = 0; i < QW; ++i) {
                uint32_t bw;
                if constexpr (RB == 1) {
                    uint32_t b[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int c = 4 * i + u;
                        anyn |= __funnelshift_r(yl[c], yh[c], hsh) <= fth;
                        b[u] = yh[c] >> hsh;
                    }
                    bw = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
                    qw[i] = __vsubus4(rw[i], bw);
                } else {
                    uint32_t b[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int c = 2 * i + u;
                        anyn |= __funnelshift_r(yl[c], yh[c], hsh) <= fth;
                        b[u] = yh[c] >> hsh;
                    }
                    bw = __byte_perm(b[0], b[1], 0x5410);
                    qw[i] = __vsubus2(rw[i], bw);
                }
            }
            if (__builtin_expect(__any_sync(0xffffffffu, anyn && live), 0)) {
#pragma unroll
                for (int c = 0; c < CW; ++c) {
                    if (live && __funnelshift_r(yl[c], yh[c], hsh) <= fth) {
                        const uint32_t rv = (rw[c / VPW] >> (8 * RB * (c % VPW))) & VM;
                        const unsigned long long Y = ((unsigned long long)yh[c] << 32) | yl[c];
                        const uint32_t qv = qz_exact(prm, SPL, Y - Cy, rv, (unsigned long long)(l * NZ + h0 + c), fix, cap);
                        const int sh = 8 * RB * (c % VPW);
                        qw[c / VPW] = (qw[c / VPW] & ~(VM << sh)) | (qv << sh);
                    }
                }
            }
            if (live) {
                uint8_t *dst = (uint8_t *)q + (l * NZ + h0) * RB;
                if constexpr (CW * RB % 16 == 0) {
#pragma unroll
                    for (int i = 0; i < QW / 4; ++i)
                        *(uint4 *)(dst + 16 * i) = make_uint4(qw[4 * i], qw[4 * i + 1], qw[4 * i + 2], qw[4 * i + 3]);
                } else {
#pragma unroll
                    for (int i = 0; i < QW / 2; ++i) *(uint2 *)(dst + 8 * i) = make_uint2(qw[2 * i], qw[2 * i + 1]);
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (wp == 1) tc::tmem_dealloc(base, 512);
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda);
// the pointer is looked up once per process (idempotent)
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)p;
    }();
    return fn;
}

namespace {
// tensor map of an intermediate's NP byte planes [plane][outer][rows][row bytes]
// for the TMA store of 128-row x tv-byte output tiles (64B / 32B swizzle
// matching tc_pass_xy_ws's staging)
bool out_map(CUtensorMap *tm, PFN_cuTensorMapEncodeTiled_v12000 encode, uint8_t *base, long long row_bytes,
             long long rows, long long outer, int np, long long plane, int tv) {
    const cuuint64_t dims[4] = {(cuuint64_t)row_bytes, (cuuint64_t)rows, (cuuint64_t)outer, (cuuint64_t)np};
    const cuuint64_t strides[3] = {(cuuint64_t)row_bytes, (cuuint64_t)(row_bytes * rows), (cuuint64_t)plane};
    const cuuint32_t box[4] = {(cuuint32_t)tv, TM, 1, (cuuint32_t)np}, es[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw =
        tv == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : tv == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, (void *)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// TC path of ct_gaussian_q (u8, u16).  Returns CT_ERR_UNSUPPORTED when the
// shape does not fit (the caller then uses the SIMT FMA path).  work: >= 8 N
// bytes (byte planes of P1 and P2) + sizeof(TcParams).
bool ct_gaussian_q_tc_fits(int dtype, int64_t nx, int64_t ny, int64_t nz, int rx, int ry, int rz) {
    const bool u16 = dtype == CT_U16;
    if (dtype != CT_U8 && !u16) return false;
    return (nz == 32 || nz == 64 || (nz == 96 && !u16)) && rx >= 0 && ry >= 0 && rz >= 0 && rx <= (KXY - TM) / 2 &&
           ry <= (KXY - TM) / 2 && rz < PMAX && (ny * nz) % TNX == 0 && nz % TNY == 0 &&
           nx * ny * nz < (1ll << 31);
}

namespace {

// NP byte planes per intermediate: 4 for u8 (24 fractional bits), 5 for u16
// (40-bit intermediates: 28 fractional bits for 12-bit data, 24 at full range)
template <typename Traw>
int gaussian_q_tc(const Traw *raw, int64_t nx, int64_t ny, int64_t nz, int rx, int ry, int rz, uint8_t *p1,
                  uint8_t *p2, TcParams *prm, Traw *q, unsigned long long *fix, int64_t cap, cudaStream_t s) {
    constexpr int RB = (int)sizeof(Traw);
    constexpr int NP = RB == 1 ? 4 : 5, NL = NP;  // intermediate planes, weight limbs
    const long long N = nx * ny * nz;
    // persistent grids: one CTA per SM (capping it to leave SMs to the concurrent vessel stream measured
    // slower: 140 / 132 / 120 SMs -> 1.744 / 1.750 / 1.810 ms per C2 step vs 1.744)
    const int nsm = CT_NUM_SMS;
    PFN_cuTensorMapEncodeTiled_v12000 encode = tma_encoder();
    if (!encode) {
        ct::set_error("cuTensorMapEncodeTiled unavailable (driver entry point)");
        return CT_ERR_CUDA;
    }
    // pass x: warp-specialised, operands staged by TMA.  The raw volume as a
    // byte matrix [nx][ny nz RB]; one box of TX bytes x 256 x-rows per tile,
    // 64B / 32B-swizzled (u16: TX bytes = TX / 2 voxels, both byte limbs)
    {
        constexpr int TX = NL == 4 ? 64 : 32, SS = 6, AS = 1;  // TMEM: 64 NL band columns + NL TX accumulators (TX = 32 with two accumulator sets measured slower: 158 vs 138 us)
        CUtensorMap tm;
        const cuuint64_t dims[2] = {(cuuint64_t)(ny * nz * RB), (cuuint64_t)nx};
        const cuuint64_t strides[1] = {(cuuint64_t)(ny * nz * RB)};
        const cuuint32_t box[2] = {TX, KXY}, es[2] = {1, 1};
        if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void *)raw, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, TX == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            ct::set_error("tensor map (pass x) rejected");
            return CT_ERR_UNSUPPORTED;
        }
        CUtensorMap to;
        if (!out_map(&to, encode, p1, ny * nz, nx, 1, NP, N, TX / RB)) {
            ct::set_error("tensor map (pass x output) rejected");
            return CT_ERR_UNSUPPORTED;
        }
        auto kx = tc_pass_xy_ws<1, TX, SS, AS, RB, NP, NL>;
        const size_t sm = (size_t)SS * 1 * KXY * TX + 2 * NP * TM * (TX / RB) + 1024;
        cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const long long tiles = ((nx + TM - 1) / TM) * (ny * nz * RB / TX);
        kx<<<(unsigned)std::min<long long>(tiles, nsm), WSX_NT, sm, s>>>(tm, to, (int)nx, (int)(ny * nz * RB), 1, prm,
                                                                        0, rx);
        if (int st = ct::check_launch("tc_pass_x")) return st;
    }
    // pass y: [nx][ny][nz] x NP planes, warp-specialised like pass x: one 4-D
    // box {32 B, 256 rows, 1, NP planes} per tile (32B swizzle), the edge
    // fixer warp clamps the rows outside [0, ny)
    {
        constexpr int SS = NP == 4 ? 5 : 4;  // operand stages
        CUtensorMap tm;
        const cuuint64_t dims[4] = {(cuuint64_t)nz, (cuuint64_t)ny, (cuuint64_t)nx, (cuuint64_t)NP};
        const cuuint64_t strides[3] = {(cuuint64_t)nz, (cuuint64_t)(ny * nz), (cuuint64_t)N};
        const cuuint32_t box[4] = {TNY, KXY, 1, NP}, es[4] = {1, 1, 1, 1};
        if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, (void *)p1, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            ct::set_error("tensor map (pass y) rejected");
            return CT_ERR_UNSUPPORTED;
        }
        CUtensorMap to;
        if (!out_map(&to, encode, p2, nz, ny, nx, NP, N, TNY)) {
            ct::set_error("tensor map (pass y output) rejected");
            return CT_ERR_UNSUPPORTED;
        }
        auto ky = tc_pass_xy_ws<NP, TNY, SS, 1, 1, NP, NL>;
        const size_t sm = (size_t)SS * NP * KXY * TNY + 2 * NP * TM * TNY + 1024;
        cudaFuncSetAttribute(ky, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const long long tiles = nx * ((ny + TM - 1) / TM) * (nz / TNY);
        ky<<<(unsigned)std::min<long long>(tiles, nsm), WSX_NT, sm, s>>>(tm, to, (int)ny, (int)nz, (int)nx, prm, 1,
                                                                         ry);
        if (int st = ct::check_launch("tc_pass_y")) return st;
    }
    // pass z + epilogue: warp-specialised, operands by TMA
    {
        const long long lines = nx * ny, tiles = (lines + TM - 1) / TM;
        CUtensorMap tp, tr;
        const cuuint64_t pdims[3] = {(cuuint64_t)nz, (cuuint64_t)lines, (cuuint64_t)NP};
        const cuuint64_t pstr[2] = {(cuuint64_t)nz, (cuuint64_t)N};
        const cuuint32_t pbox[3] = {16, TM, NP}, es3[3] = {1, 1, 1};
        const cuuint64_t rdims[2] = {(cuuint64_t)(nz * RB), (cuuint64_t)lines};
        const cuuint64_t rstr[1] = {(cuuint64_t)(nz * RB)};
        const cuuint32_t rbox[2] = {(cuuint32_t)(nz * RB), TM}, es2[2] = {1, 1};
        if (encode(&tp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void *)p2, pdims, pstr, pbox, es3,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
            encode(&tr, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void *)raw, rdims, rstr, rbox, es2,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            ct::set_error("tensor map (pass z) rejected");
            return CT_ERR_UNSUPPORTED;
        }
        void (*kz)(const CUtensorMap, const CUtensorMap, long long, const TcParams *, int, const Traw *, Traw *,
                   unsigned long long *, long long);
        int stg;
        bool rawg = false;
        if constexpr (RB == 2) {  // u16: raw from global, 4 stages of 5 planes
            stg = 4;
            rawg = true;
            kz = nz == 64 ? tc_pass_z_ws<64, 4, Traw, 5, 5, true> : tc_pass_z_ws<32, 4, Traw, 5, 5, true>;
        } else {
            stg = nz == 96 ? 2 : 4;
            kz = nz == 64 ? tc_pass_z_ws<64, 4, Traw> : nz == 96 ? tc_pass_z_ws<96, 2, Traw> : tc_pass_z_ws<32, 4, Traw>;
        }
        const size_t sm = (size_t)stg * (NP * TM * nz + (rawg ? 0 : TM * nz * RB)) + NL * nz * nz + NL * nz * 32 + 1024;
        cudaFuncSetAttribute(kz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kz<<<(unsigned)std::min<long long>(tiles, nsm), WS_NT, sm, s>>>(tp, tr, lines, prm, rz, raw, q, fix, cap);
        if (int st = ct::check_launch("tc_pass_z")) return st;
    }
    return CT_OK;
}

}  // namespace

int ct_gaussian_q_tc(const void *raw, int dtype, int64_t nx, int64_t ny, int64_t nz, const double *w, int rx, int ry,
                     int rz, void *work, void *q, unsigned long long *fix, int64_t cap, double eps_override,
                     cudaStream_t s) {
    if (!ct_gaussian_q_tc_fits(dtype, nx, ny, nz, rx, ry, rz) || ((uintptr_t)raw & 15)) return CT_ERR_UNSUPPORTED;
    const long long N = nx * ny * nz;
    const int np = dtype == CT_U8 ? 4 : 5;
    uint8_t *p1 = (uint8_t *)work, *p2 = p1 + np * N;
    TcParams *prm = (TcParams *)(p2 + np * N);
    cudaMemsetAsync(fix, 0, 2 * sizeof(unsigned long long), s);
    const bool u8 = dtype == CT_U8;
    if (!u8) {
        cudaMemsetAsync(&prm->vmax, 0, sizeof(unsigned), s);
        tc_vmax<<<CT_NUM_SMS * 4, 256, 0, s>>>((const uint4 *)raw, N * 2 / 16, prm);  // N * 2 % 16 == 0 (nz % 32)
        if (int st = ct::check_launch("tc_vmax")) return st;
    }
    tc_prep<<<1, 96, 0, s>>>(w, rx, ry, rz, u8 ? 1 : 0, np, np, eps_override, prm);
    if (int st = ct::check_launch("tc_prep")) return st;
    if (u8)
        return gaussian_q_tc<uint8_t>((const uint8_t *)raw, nx, ny, nz, rx, ry, rz, p1, p2, prm, (uint8_t *)q, fix,
                                      cap, s);
    return gaussian_q_tc<uint16_t>((const uint16_t *)raw, nx, ny, nz, rx, ry, rz, p1, p2, prm, (uint16_t *)q, fix,
                                   cap, s);
}

size_t ct_gaussian_q_tc_work(int64_t nx, int64_t ny, int64_t nz) {  // <= the 16 N bytes ct_gaussian_q takes
    return (size_t)10 * nx * ny * nz + sizeof(TcParams) + 256;
}
