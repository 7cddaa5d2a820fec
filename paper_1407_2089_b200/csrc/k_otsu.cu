// k_otsu.cu -- K3: Otsu threshold with the reference's exact semantics.
//
// Replaces ref segment.py:99-151 (otsu_threshold) and the degenerate rules of
// binarize (segment.py:192-204).  The reference scores every t < nbins-1 as
//   num = float64(int64(s0*w1 - s1*w0))**2 ; den = float64(int64(w0*w1))
//   score = den > 0 ? num/den : 0
// with numpy int64 arrays (two's-complement wrap for huge N), keeps the
// candidates score >= best*(1-1e-9) (or every t when best <= 0), and decides
// among them exactly with Python integers (a^2/b compared cross-multiplied,
// strict improvement -> lowest t).  Here: one CTA of 1024 threads; each
// thread owns a contiguous chunk of bins (prefix sums via a block scan of
// chunk totals), pass A finds best, pass B applies the candidate filter and
// the exact comparison with 128-bit a and 384-bit products, and a block
// reduction keeps the lowest winning t.
#include "ct_common.cuh"

namespace {


struct U384 {
    u64 w[6];
};

__device__ __forceinline__ void mul64(u64 a, u64 b, u64 &lo, u64 &hi) {
    lo = a * b;
    hi = __umul64hi(a, b);
}

// r = a (n limbs) * b (2 limbs), result limbs up to 6
__device__ U384 mul_limbs(const u64 *a, int na, const u64 *b) {
    U384 r;
#pragma unroll
    for (int i = 0; i < 6; ++i) r.w[i] = 0;
    for (int i = 0; i < na; ++i) {
        u64 carry = 0;
        for (int j = 0; j < 2; ++j) {
            u64 lo, hi;
            mul64(a[i], b[j], lo, hi);
            u64 t = r.w[i + j] + lo;
            u64 c1 = t < lo;
            u64 t2 = t + carry;
            u64 c2 = t2 < t;
            r.w[i + j] = t2;
            carry = hi + c1 + c2;
        }
        // propagate
        for (int k = i + 2; k < 6 && carry; ++k) {
            u64 t = r.w[k] + carry;
            carry = t < carry;
            r.w[k] = t;
        }
    }
    return r;
}

__device__ int cmp384(const U384 &a, const U384 &b) {
    for (int i = 5; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] > b.w[i] ? 1 : -1;
    return 0;
}

struct Cand {
    i64 t;       // -1: none
    u64 a2[4];   // a^2 (256-bit)
    u64 b[2];    // w0*w1 (128-bit)
};

// is x strictly better than y (x.a2/x.b > y.a2/y.b)?
__device__ bool better(const Cand &x, const Cand &y) {
    if (y.t < 0) return x.t >= 0;
    if (x.t < 0) return false;
    U384 l = mul_limbs(x.a2, 4, y.b), r = mul_limbs(y.a2, 4, x.b);
    return cmp384(l, r) > 0;
}

// choose between two candidates: exact larger score, ties -> lower t
__device__ void merge(Cand &x, const Cand &y) {
    if (y.t < 0) return;
    if (x.t < 0) { x = y; return; }
    if (better(y, x)) x = y;
    else if (!better(x, y) && y.t < x.t) x = y;
}

template <int NT>  // threads (256 when the caller fixes 256 bins, else 1024)
__global__ void __launch_bounds__(NT) otsu_kernel(const uint64_t *__restrict__ hist, i64 nbins_given,
                                                  i64 *__restrict__ result) {
    constexpr int NW = NT / 32;
    __shared__ u64 s_w[NT], s_s[NT];
    __shared__ double s_best[NW];
    __shared__ i64 s_cnt[NW];
    __shared__ int s_hi;
    __shared__ Cand s_c[NW];
    const int tid = threadIdx.x;
    if (tid == 0) s_hi = 0;
    __syncthreads();
    i64 nb = nbins_given;
    if (nb <= 0) {
        for (int b = 256 + tid; b < 65536; b += NT)
            if (hist[b]) s_hi = 1;
        __syncthreads();
        nb = s_hi ? 65536 : 256;
    }
    const i64 chunk = (nb + NT - 1) / NT;
    const i64 b0 = min((i64)tid * chunk, nb), b1 = min(b0 + chunk, nb);
    // chunk totals
    u64 cw = 0, cs = 0;
    i64 nzc = 0;
    for (i64 b = b0; b < b1; ++b) {
        const u64 h = hist[b];
        cw += h;
        cs += h * (u64)b;
        nzc += h != 0;
    }
    s_w[tid] = cw;
    s_s[tid] = cs;
    // nonzero count
    for (int o = 16; o; o >>= 1) nzc += __shfl_xor_sync(0xffffffffu, nzc, o);
    if ((tid & 31) == 0) s_cnt[tid >> 5] = nzc;
    __syncthreads();
    // inclusive scan of chunk totals (Hillis-Steele on SMEM, wrap arithmetic)
    for (int off = 1; off < NT; off <<= 1) {
        u64 aw = 0, as = 0;
        if (tid >= off) { aw = s_w[tid - off]; as = s_s[tid - off]; }
        __syncthreads();
        s_w[tid] += aw;
        s_s[tid] += as;
        __syncthreads();
    }
    const u64 W = s_w[NT - 1], S = s_s[NT - 1];
    const u64 pre_w = tid ? s_w[tid - 1] : 0, pre_s = tid ? s_s[tid - 1] : 0;
    i64 nonzero = 0;
    for (int i = 0; i < NW; ++i) nonzero += s_cnt[i];
    if (nonzero < 2 || nb < 2) {
        if (tid == 0) {
            result[CT_OTSU_T] = 0;
            result[CT_OTSU_STATUS] = (nb >= 1 && hist[0] == W) ? 1 : 2;
            result[CT_OTSU_NBINS] = nb;
            result[CT_OTSU_NONZERO] = nonzero;
        }
        return;
    }
    // pass A: best float score over t in [0, nb-2]
    double best = -INFINITY;
    {
        u64 w0 = pre_w, s0 = pre_s;
        for (i64 t = b0; t < b1; ++t) {
            const u64 h = hist[t];
            w0 += h;
            s0 += h * (u64)t;
            if (t >= nb - 1) break;
            const u64 w1 = W - w0, s1 = S - s0;
            const i64 num_i = (i64)(s0 * w1 - s1 * w0);
            const i64 den_i = (i64)(w0 * w1);
            double num = (double)num_i;
            num = __dmul_rn(num, num);
            const double den = (double)den_i;
            const double sc = den > 0.0 ? __ddiv_rn(num, den) : 0.0;
            best = fmax(best, sc);
        }
    }
    for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((tid & 31) == 0) s_best[tid >> 5] = best;
    __syncthreads();
    best = s_best[0];
    for (int i = 1; i < NW; ++i) best = fmax(best, s_best[i]);
    const double cut = __dmul_rn(best, 1.0 - 1e-9);
    // pass B: candidates, exact comparison
    Cand mine;
    mine.t = -1;
    {
        u64 w0 = pre_w, s0 = pre_s;
        for (i64 t = b0; t < b1; ++t) {
            const u64 h = hist[t];
            w0 += h;
            s0 += h * (u64)t;
            if (t >= nb - 1) break;
            const u64 w1 = W - w0, s1 = S - s0;
            bool cand = true;
            if (!(best <= 0.0)) {
                const i64 num_i = (i64)(s0 * w1 - s1 * w0);
                const i64 den_i = (i64)(w0 * w1);
                double num = (double)num_i;
                num = __dmul_rn(num, num);
                const double den = (double)den_i;
                const double sc = den > 0.0 ? __ddiv_rn(num, den) : 0.0;
                cand = sc >= cut;
            }
            if (!cand) continue;
            // exact: a = s0*w1 - s1*w0 (Python ints), b = w0*w1
            const __int128 a = (__int128)(i64)s0 * (__int128)(i64)w1 - (__int128)(i64)s1 * (__int128)(i64)w0;
            const unsigned __int128 bb = (unsigned __int128)((__int128)(i64)w0 * (__int128)(i64)w1);
            if (bb == 0) continue;
            const unsigned __int128 ua = a < 0 ? (unsigned __int128)(-a) : (unsigned __int128)a;
            Cand c;
            c.t = t;
            const u64 al[2] = {(u64)ua, (u64)(ua >> 64)};
            U384 a2 = mul_limbs(al, 2, al);
            for (int i = 0; i < 4; ++i) c.a2[i] = a2.w[i];
            c.b[0] = (u64)bb;
            c.b[1] = (u64)(bb >> 64);
            if (better(c, mine)) mine = c;  // ascending t: strict improvement only
        }
    }
    // warp then block reduction (exact, ties -> lower t)
    for (int o = 16; o; o >>= 1) {
        Cand other;
        other.t = __shfl_xor_sync(0xffffffffu, mine.t, o);
        for (int i = 0; i < 4; ++i) other.a2[i] = __shfl_xor_sync(0xffffffffu, mine.a2[i], o);
        for (int i = 0; i < 2; ++i) other.b[i] = __shfl_xor_sync(0xffffffffu, mine.b[i], o);
        merge(mine, other);
    }
    if ((tid & 31) == 0) s_c[tid >> 5] = mine;
    __syncthreads();
    if (tid == 0) {
        Cand r = s_c[0];
        for (int i = 1; i < NW; ++i) merge(r, s_c[i]);
        result[CT_OTSU_T] = r.t < 0 ? 0 : r.t;
        result[CT_OTSU_STATUS] = 0;
        result[CT_OTSU_NBINS] = nb;
        result[CT_OTSU_NONZERO] = nonzero;
    }
}

}  // namespace

extern "C" int ct_otsu(const uint64_t *hist, int64_t nbins, int64_t *result, void *stream) {
    if (nbins > 65536) {
        ct::set_error("otsu supports at most 65536 bins (got %lld)", (long long)nbins);
        return CT_ERR_UNSUPPORTED;
    }
    if (nbins > 0 && nbins <= 256) otsu_kernel<256><<<1, 256, 0, (cudaStream_t)stream>>>(hist, nbins, result);
    else otsu_kernel<1024><<<1, 1024, 0, (cudaStream_t)stream>>>(hist, nbins, result);
    return ct::check_launch("otsu");
}
