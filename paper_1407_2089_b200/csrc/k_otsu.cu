// k_otsu.cu -- K3: Otsu threshold with the reference's exact semantics.
//
// Replaces ref segment.py:99-151 (otsu_threshold) and the degenerate rules of
// binarize (segment.py:192-204).  The reference scores every t < nbins-1 as
//   num = float64(int64(s0*w1 - s1*w0))**2 ; den = float64(int64(w0*w1))
//   score = den > 0 ? num/den : 0
// with numpy int64 arrays (two's-complement wrap for huge N), keeps the
// candidates score >= best*(1-1e-9) (or every t when best <= 0), and decides
// among them exactly with Python integers (a^2/b compared cross-multiplied,
// strict improvement -> lowest t).  Here: one CTA (256 or 1024 threads)
// visits the bins in rounds of consecutive bins (coalesced; prefix sums by a
// block scan per round plus a carry), pass A finds best, pass B applies the
// candidate filter and the exact comparison with 128-bit a and 384-bit
// products, and a block reduction keeps the lowest winning t.
#include <climits>

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

// candidate t (score within the reference's 1e-9 cut): exact a^2 / b against
// the best so far -- a = s0*w1 - s1*w0 (Python ints), b = w0*w1; ascending t,
// strict improvement only
__device__ __noinline__ void consider(Cand &mine, i64 t, u64 w0, u64 s0, u64 W, u64 S) {
    const u64 w1 = W - w0, s1 = S - s0;
    const __int128 a = (__int128)(i64)s0 * (__int128)(i64)w1 - (__int128)(i64)s1 * (__int128)(i64)w0;
    const unsigned __int128 bb = (unsigned __int128)((__int128)(i64)w0 * (__int128)(i64)w1);
    if (bb == 0) return;
    const unsigned __int128 ua = a < 0 ? (unsigned __int128)(-a) : (unsigned __int128)a;
    Cand c;
    c.t = t;
    const u64 al[2] = {(u64)ua, (u64)(ua >> 64)};
    U384 a2 = mul_limbs(al, 2, al);
    for (int i = 0; i < 4; ++i) c.a2[i] = a2.w[i];
    c.b[0] = (u64)bb;
    c.b[1] = (u64)(bb >> 64);
    if (better(c, mine)) mine = c;
}

// block-wide inclusive scan of (w, s) pairs (wrap arithmetic); returns the
// block totals.  Warp scans, then warp 0 scans the NT/32 warp totals; three
// barriers, two shared loads per thread.  Scratch: NT/32 pairs.
template <int NT>
__device__ __forceinline__ void block_scan2(u64 &w, u64 &s, u64 *sw, u64 *ss, u64 &tw, u64 &ts) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 a = __shfl_up_sync(0xffffffffu, w, o), b = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) {
            w += a;
            s += b;
        }
    }
    __syncthreads();  // previous round's readers of sw/ss are done
    if (lane == 31) {
        sw[wid] = w;
        ss[wid] = s;
    }
    __syncthreads();
    if (wid == 0) {
        u64 a = lane < NW ? sw[lane] : 0, b = lane < NW ? ss[lane] : 0;
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) {
            const u64 x = __shfl_up_sync(0xffffffffu, a, o), y = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) {
                a += x;
                b += y;
            }
        }
        if (lane < NW) {
            sw[lane] = a;  // inclusive prefix of the warp totals
            ss[lane] = b;
        }
    }
    __syncthreads();
    if (wid > 0) {
        w += sw[wid - 1];
        s += ss[wid - 1];
    }
    tw = sw[NW - 1];
    ts = ss[NW - 1];
}

// Bins are visited in rounds of NT consecutive bins (thread tid takes bin
// R*NT + tid: coalesced reads, no per-thread serial chain); the prefix sums
// w0, s0 at each bin come from a block scan per round plus the running carry.
template <int NT>  // threads (256 when the caller fixes 256 bins, else 1024)
__global__ void __launch_bounds__(NT) otsu_kernel(const uint64_t *__restrict__ hist, i64 nbins_given,
                                                  i64 *__restrict__ result) {
    constexpr int NW = NT / 32;
    __shared__ u64 s_w[NW], s_s[NW];
    __shared__ double s_best[NW];
    __shared__ i64 s_cnt[NW];
    __shared__ int s_hi;
    __shared__ Cand s_c[NW];
    const int tid = threadIdx.x;
    if (tid == 0) s_hi = 0;
    __syncthreads();
    i64 nb = nbins_given;
    if (nb <= 0) {
        int hi = 0;
        for (int b0 = 256; b0 < 65536; b0 += 8 * NT) {  // 8 independent loads in flight
            u64 hv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) hv[u] = b0 + u * NT + tid < 65536 ? hist[b0 + u * NT + tid] : 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) hi |= hv[u] != 0;
        }
        if (__any_sync(0xffffffffu, hi) && (tid & 31) == 0) s_hi = 1;
        __syncthreads();
        nb = s_hi ? 65536 : 256;
    }
    const i64 rounds = (nb + NT - 1) / NT;
    // totals, the non-empty bin count and the first / last non-empty bin.
    // Bins below the first or above the last non-empty one have w0 = 0 or
    // w1 = 0: score 0 and b = w0 w1 = 0, so they never win (nor change best
    // when a positive score exists) -- the scored rounds are [R_lo, R_hi]
    // (12-bit data in 65536 bins: 4 rounds instead of 64).
    u64 W = 0, S = 0;
    i64 nzc = 0, R_lo = 0, R_hi = -1;
    {
        u64 cw = 0, cs = 0;
        int lo = INT_MAX, hi = -1;
        for (i64 R0 = 0; R0 < rounds; R0 += 8) {  // 8 independent loads in flight (65536 bins: 64 rounds)
            u64 hv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const i64 b = (R0 + u) * NT + tid;
                hv[u] = (R0 + u < rounds && b < nb) ? hist[b] : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const i64 b = (R0 + u) * NT + tid;
                const u64 h = hv[u];
                cw += h;
                cs += h * (u64)b;
                nzc += h != 0;
                if (h) {
                    lo = min(lo, (int)b);
                    hi = (int)b;
                }
            }
        }
        for (int o = 16; o; o >>= 1) {
            cw += __shfl_xor_sync(0xffffffffu, cw, o);
            cs += __shfl_xor_sync(0xffffffffu, cs, o);
            nzc += __shfl_xor_sync(0xffffffffu, nzc, o);
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        __shared__ int s_lo[NW], s_hi2[NW];
        if ((tid & 31) == 0) {
            s_w[tid >> 5] = cw;
            s_s[tid >> 5] = cs;
            s_cnt[tid >> 5] = nzc;
            s_lo[tid >> 5] = lo;
            s_hi2[tid >> 5] = hi;
        }
        __syncthreads();
        nzc = 0;
        lo = INT_MAX;
        hi = -1;
        for (int i = 0; i < NW; ++i) {
            W += s_w[i];
            S += s_s[i];
            nzc += s_cnt[i];
            lo = min(lo, s_lo[i]);
            hi = max(hi, s_hi2[i]);
        }
        if (hi >= 0) {
            R_lo = lo / NT;
            R_hi = hi / NT;
        }
    }
    const i64 nonzero = nzc;
    if (nonzero < 2 || nb < 2) {
        if (tid == 0) {
            result[CT_OTSU_T] = 0;
            result[CT_OTSU_STATUS] = (nb >= 1 && hist[0] == W) ? 1 : 2;
            result[CT_OTSU_NBINS] = nb;
            result[CT_OTSU_NONZERO] = nonzero;
        }
        return;
    }
    auto score = [&](u64 w0, u64 s0) -> double {
        const u64 w1 = W - w0, s1 = S - s0;
        const i64 num_i = (i64)(s0 * w1 - s1 * w0);
        const i64 den_i = (i64)(w0 * w1);
        double num = (double)num_i;
        num = __dmul_rn(num, num);
        const double den = (double)den_i;
        return den > 0.0 ? __ddiv_rn(num, den) : 0.0;
    };
    // pass A: best float score over t in [0, nb-2]
    double best = -INFINITY;
    // the bins of RB rounds are loaded up front (independent loads in flight),
    // then scanned round by round: a load per barrier-separated round would
    // put its full latency on the critical path
    constexpr int RB = 8;
    u64 hb[RB];
    auto load_batch = [&](i64 R0) {
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const i64 t = (R0 + u) * NT + tid;
            hb[u] = (R0 + u < rounds && t < nb) ? hist[t] : 0;
        }
    };
    {
        u64 cw = 0, cs = 0;
        for (i64 R0 = R_lo; R0 <= R_hi; R0 += RB) {
            load_batch(R0);
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                if (R0 + u > R_hi) break;  // uniform
                const i64 t = (R0 + u) * NT + tid;
                u64 w0 = hb[u], s0 = hb[u] * (u64)t, tw, ts;
                block_scan2<NT>(w0, s0, s_w, s_s, tw, ts);
                w0 += cw;
                s0 += cs;
                cw += tw;
                cs += ts;
                // an empty bin t repeats bin t-1's (w0, s0), hence its score
                if (t < nb - 1 && (hb[u] != 0 || t == 0)) best = fmax(best, score(w0, s0));
            }
        }
    }
    for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((tid & 31) == 0) s_best[tid >> 5] = best;
    __syncthreads();
    best = s_best[0];
    for (int i = 1; i < NW; ++i) best = fmax(best, s_best[i]);
    const double cut = __dmul_rn(best, 1.0 - 1e-9);
    // pass B: candidates, exact comparison (each thread sees its bins in ascending t)
    Cand mine;
    mine.t = -1;
    {
        u64 cw = 0, cs = 0;
        auto visit = [&](i64 t, u64 w0, u64 s0, u64 h) {
            if (t >= nb - 1) return;
            // an empty bin t > 0 has bin t-1's (w0, s0): the same exact a^2/b,
            // and the lower t wins ties -- never a strict improvement
            if (h == 0 && t > 0) return;
            if (!(best <= 0.0) && !(score(w0, s0) >= cut)) return;
            consider(mine, t, w0, s0, W, S);  // rare: out of line
        };
        for (i64 R0 = R_lo; R0 <= R_hi; R0 += RB) {
            load_batch(R0);
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                if (R0 + u > R_hi) break;  // uniform
                const i64 t = (R0 + u) * NT + tid;
                u64 w0 = hb[u], s0 = hb[u] * (u64)t, tw, ts;
                block_scan2<NT>(w0, s0, s_w, s_s, tw, ts);
                w0 += cw;
                s0 += cs;
                cw += tw;
                cs += ts;
                visit(t, w0, s0, hb[u]);
            }
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
