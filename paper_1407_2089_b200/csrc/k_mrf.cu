// k_mrf.cu -- K7: vessel-channel MRF denoise (ref denoise.py:92-195).
//
//   delta     = intensity_step (denoise.py:135-144): min gap of the distinct
//               values.  Integer input: from the histogram's non-empty bins;
//               float input: radix-sorted copy (CUB), min positive gap.
//   sigma_hat = estimate_noise_variance (denoise.py:92-114) = np.std(lap)/sqrt(42)
//               over the interior 6-neighbour Laplacian.  np.std reduces with
//               numpy's pairwise summation (8-way unrolled leaves of <= 128,
//               halving splits rounded to multiples of 8).
//               * integer input: every Laplacian and every partial sum is an
//                 integer below 2^53, so the mean's sum is order-independent and
//                 is taken as an exact int64 reduction in the fused statistics
//                 pass; only sum((lap - mean)^2) needs numpy's tree.
//               * the tree: CTA b owns depth-D node b (D from the smallest path,
//                 so every depth-D node exists), stages its elements in SMEM
//                 with coalesced loads, sums its <= 128-element leaves (one
//                 thread each) and recombines them in recursion order; one CTA
//                 folds the 2^D partials pairwise.
//   first step (denoise.py:172-176): proposal = I0 + delta*sign(S), S the
//               edge-replicated sign sum (denoise.py:117-132).  For integer
//               input ||proposal - I0||^2 = delta^2 * #{S != 0} exactly, so the
//               statistics pass only counts non-zero sign sums.  On realistic
//               volumes the step is rejected (decision 0); further iterations
//               run through ct_mrf_step driven by the host.
#include <cub/device/device_radix_sort.cuh>

#include <cstdlib>
#include <type_traits>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ct_common.cuh"

namespace {

constexpr int PW_SUB = 4096;  // target minimum subtree size per CTA
constexpr int PT = 256;       // threads per subtree CTA
constexpr int MAX_LEAVES = 512;

__host__ __device__ inline i64 pw_left(i64 n) {
    i64 n2 = n / 2;
    return n2 - n2 % 8;
}

// depth D such that every node at depth D has size >= min(PW_SUB, n)
inline int pw_depth(i64 n) {
    int d = 0;
    i64 m = n;
    while (m > 128 && pw_left(m) >= PW_SUB && d < 24) {
        m = pw_left(m);
        ++d;
    }
    return d;
}

// largest node size at depth D (sizes per level form a tiny set)
inline i64 pw_max_node(i64 n, int D) {
    i64 sizes[64];
    int ns = 1;
    sizes[0] = n;
    for (int d = 0; d < D; ++d) {
        i64 nxt[64];
        int nn = 0;
        for (int i = 0; i < ns; ++i) {
            const i64 l = pw_left(sizes[i]), r = sizes[i] - l;
            const i64 c[2] = {l, r};
            for (int q = 0; q < 2; ++q) {
                bool seen = false;
                for (int u = 0; u < nn; ++u) seen |= nxt[u] == c[q];
                if (!seen && nn < 64) nxt[nn++] = c[q];
            }
        }
        ns = nn;
        for (int i = 0; i < ns; ++i) sizes[i] = nxt[i];
    }
    i64 m = 0;
    for (int i = 0; i < ns; ++i) m = sizes[i] > m ? sizes[i] : m;
    return m;
}

// node at depth D with path bits `idx` (MSB first = first split)
__device__ void pw_node(i64 n, int D, i64 idx, i64 &off, i64 &len) {
    off = 0;
    len = n;
    for (int d = D - 1; d >= 0; --d) {
        const i64 l = pw_left(len);
        if ((idx >> d) & 1) { off += l; len -= l; }
        else len = l;
    }
}

__device__ __forceinline__ int sgn(double x) { return (x > 0.0) - (x < 0.0); }

// Laplacian element e of the flattened C-order interior (nx-2, ny-2, nz-2);
// interior sizes fit 32 bits (volumes are < 2^31 voxels).
template <typename T>
__device__ __forceinline__ double lap_at(const T *v, uint32_t e, uint32_t my, uint32_t mz, i64 ny, i64 nz) {
    const uint32_t row = e / mz, c = e - row * mz;
    const uint32_t a = row / my, b = row - a * my;
    const i64 s0 = ny * nz;
    const i64 p = (i64)(a + 1) * s0 + (i64)(b + 1) * nz + (c + 1);
    double l = __dadd_rn(ct::to_f64(v[p - s0]), ct::to_f64(v[p + s0]));
    l = __dadd_rn(l, ct::to_f64(v[p - nz]));
    l = __dadd_rn(l, ct::to_f64(v[p + nz]));
    l = __dadd_rn(l, ct::to_f64(v[p - 1]));
    l = __dadd_rn(l, ct::to_f64(v[p + 1]));
    return __dadd_rn(l, -__dmul_rn(6.0, ct::to_f64(v[p])));
}

// element functors
template <typename T>
struct LapElem {  // lap (squared == 0) or (lap - mean)^2
    const T *v;
    i64 ny, nz;
    uint32_t my, mz;
    const double *mean;            // device, when squared == 1 and !int_sum
    const long long *int_sum;      // device exact sum of lap (integer input), mean = sum / n
    i64 n_interior;
    int squared;
    __device__ double operator()(i64 e) const {
        const double l = lap_at(v, (uint32_t)e, my, mz, ny, nz);
        if (!squared) return l;
        const double m = int_sum ? __ddiv_rn((double)*int_sum, (double)n_interior) : *mean;
        const double x = __dadd_rn(l, -m);
        return __dmul_rn(x, x);
    }
};

template <typename T>
__device__ __forceinline__ int sign_sum_at(const T *v, const double *cur, i64 nx, i64 ny, i64 nz, i64 p) {
    const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
    const i64 s0 = ny * nz;
#define VAL(q) (cur ? cur[q] : ct::to_f64(v[q]))
    const double c = VAL(p);
    int s = sgn(__dadd_rn(VAL(i > 0 ? p - s0 : p), -c)) + sgn(__dadd_rn(c, -VAL(i < nx - 1 ? p + s0 : p)));
    s += sgn(__dadd_rn(VAL(j > 0 ? p - nz : p), -c)) + sgn(__dadd_rn(c, -VAL(j < ny - 1 ? p + nz : p)));
    s += sgn(__dadd_rn(VAL(k > 0 ? p - 1 : p), -c)) + sgn(__dadd_rn(c, -VAL(k < nz - 1 ? p + 1 : p)));
#undef VAL
    return s;
}

template <typename T>
struct StepElem {  // (proposal - original)^2 for the step from `cur` (nullptr = original)
    const T *v;
    const double *cur;
    i64 nx, ny, nz;
    const double *delta;
    __device__ double operator()(i64 p) const {
        const double c = cur ? cur[p] : ct::to_f64(v[p]);
        const int s = sgn((double)sign_sum_at(v, cur, nx, ny, nz, p));
        const double prop = __dadd_rn(c, __dmul_rn(*delta, (double)s));
        const double d = __dadd_rn(prop, -ct::to_f64(v[p]));
        return __dmul_rn(d, d);
    }
};

// (lap - mean)^2 from the Laplacian array of the streaming pass (int16 for
// u8 input: |lap| <= 6*255; int32 for u16); mean = exact_sum / n (numpy's
// pairwise sum of integer-valued doubles is exact)
template <typename LT>
struct LapArrSq {
    const LT *lap;
    const double *mean;  // device: exact_sum / n, computed once (lap_mean)
    __device__ double operator()(i64 e) const {
        const double x = __dadd_rn((double)lap[e], -*mean);
        return __dmul_rn(x, x);
    }
};

// Leaf lookup inside a subtree without enumeration: node sizes at each depth
// of a subtree form a tiny set, so leaf counts per size are tabulated once per
// CTA (thread 0, a few dozen entries) and every thread descends to its leaf.
constexpr int PW_MAXD = 8;    // subtree depth (size <= ~16K elements -> <= 7 levels)
constexpr int PW_MAXS = 8;    // distinct sizes per level

struct PwShape {
    int ns[PW_MAXD + 1];                 // distinct sizes per depth
    int size[PW_MAXD + 1][PW_MAXS];
    int leaves[PW_MAXD + 1][PW_MAXS];
    int depth;                           // deepest level holding a leaf
};

__host__ __device__ inline int pw_lookup(const PwShape &sh, int d, int m) {
    for (int q = 0; q < sh.ns[d]; ++q)
        if (sh.size[d][q] == m) return sh.leaves[d][q];
    return 1;
}

__host__ __device__ inline void pw_shape(PwShape &sh, int m0) {
    sh.ns[0] = 1;
    sh.size[0][0] = m0;
    int d = 0;
    for (; d < PW_MAXD; ++d) {
        int nn = 0;
        for (int q = 0; q < sh.ns[d]; ++q) {
            const int m = sh.size[d][q];
            if (m <= 128) continue;
            const int c[2] = {(int)pw_left(m), m - (int)pw_left(m)};
            for (int h = 0; h < 2; ++h) {
                bool seen = false;
                for (int u = 0; u < nn; ++u) seen |= sh.size[d + 1][u] == c[h];
                if (!seen && nn < PW_MAXS) sh.size[d + 1][nn++] = c[h];
            }
        }
        sh.ns[d + 1] = nn;
        if (!nn) break;
    }
    sh.depth = d;
    for (int e = d; e >= 0; --e)
        for (int q = 0; q < sh.ns[e]; ++q) {
            const int m = sh.size[e][q];
            sh.leaves[e][q] = m <= 128 ? 1 : pw_lookup(sh, e + 1, (int)pw_left(m)) +
                                                 pw_lookup(sh, e + 1, m - (int)pw_left(m));
        }
}

// the distinct node sizes at depth D (a handful) with their shapes, tabulated
// on the host and passed by value (param space)
constexpr int PW_NSH = 4;
struct PwShapes {
    int count;
    int len[PW_NSH];
    PwShape sh[PW_NSH];
};

// CTA b: exact numpy-order sum of depth-D node b.  Elements are evaluated in
// place by the leaf lanes (f(e) reads global memory); leaf t found by descending with the tabulated leaf counts; internal nodes
// combined level by level (slot = path bits at that depth), so every add is
// left + right exactly as numpy's recursion performs it.
template <class F>
__global__ void __launch_bounds__(PT) pw_subtree(F f, i64 n, int D, double *__restrict__ partial,
                                                 const __grid_constant__ PwShapes shapes,
                                                 const unsigned long long *skip) {
    if (skip && *skip) return;  // decision certified earlier in the stream (mrf_quick)
    __shared__ PwShape shs;
    __shared__ double lv[2][1 << PW_MAXD];  // values per level slot (ping-pong)
    __shared__ double lval[MAX_LEAVES];
    __shared__ int lpos[MAX_LEAVES];  // depth << 16 | slot
    i64 off, len;
    pw_node(n, D, blockIdx.x, off, len);
    int si = -1;
    for (int q = 0; q < shapes.count; ++q)
        if (shapes.len[q] == (int)len) si = q;
    if (si < 0) {  // not tabulated: build it here
        if (threadIdx.x == 0) pw_shape(shs, (int)len);
        __syncthreads();
    }
    const PwShape &sh = si >= 0 ? shapes.sh[si] : shs;
    const int nleaves = sh.leaves[0][0];
    // leaves: 8 lanes per leaf; lane j accumulates numpy's r[j] (a[j], a[j+8],
    // ...), then the group combines ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by
    // shuffles and lane 0 adds the n % 8 tail -- numpy's leaf order exactly.
    const int grp = threadIdx.x >> 3, sub = threadIdx.x & 7;
    for (int base = 0; base < nleaves; base += PT / 8) {
        const int L = base + grp;
        int o = 0, m = 0, d = 0, slot = 0;
        if (L < nleaves) {
            int t = L;
            m = (int)len;
            while (m > 128) {
                const int l = (int)pw_left(m);
                const int nl = pw_lookup(sh, d + 1, l);
                slot <<= 1;
                if (t < nl) m = l;
                else { t -= nl; o += l; m -= l; slot |= 1; }
                ++d;
            }
        }
        const i64 a0 = off + o;  // leaf elements f(a0 .. a0+m-1), evaluated in place
        const int lim = m - (m & 7);
        double r = m >= 8 ? f(a0 + sub) : 0.0;
        for (int i = 8 + sub; i < lim; i += 8) r = __dadd_rn(r, f(a0 + i));
        double t = __shfl_down_sync(0xffffffffu, r, 1, 8);
        if ((sub & 1) == 0) r = __dadd_rn(r, t);
        t = __shfl_down_sync(0xffffffffu, r, 2, 8);
        if ((sub & 3) == 0) r = __dadd_rn(r, t);
        t = __shfl_down_sync(0xffffffffu, r, 4, 8);
        if (sub == 0 && L < nleaves) {
            double res;
            if (m < 8) {
                res = 0.0;
                for (int i = 0; i < m; ++i) res = __dadd_rn(res, f(a0 + i));
            } else {
                res = __dadd_rn(r, t);
                for (int i = lim; i < m; ++i) res = __dadd_rn(res, f(a0 + i));
            }
            lval[L] = res;
            lpos[L] = (d << 16) | slot;
        }
    }
    // combine bottom-up: at depth d, slots of existing nodes; a node at depth d
    // is a leaf (value from its thread) or internal (children at d+1)
    const int dmax = sh.depth;
    double *cur = lv[0], *nxt = lv[1];
    for (int d = dmax; d >= 0; --d) {
        // nodes at depth d: write leaves of this depth, combine internal ones
        __syncthreads();
        for (int L = threadIdx.x; L < nleaves; L += PT)
            if ((lpos[L] >> 16) == d) nxt[lpos[L] & 0xffff] = lval[L];
        // internal nodes at depth d combine children (depth d+1 values in cur)
        for (int sl = threadIdx.x; sl < (1 << d); sl += PT) {
            // descend the path of slot sl to learn whether it exists / is internal
            int m = (int)len;
            bool exists = true;
            for (int e = d - 1; e >= 0 && exists; --e) {
                if (m <= 128) exists = false;
                else m = ((sl >> e) & 1) ? m - (int)pw_left(m) : (int)pw_left(m);
            }
            if (exists && m > 128) nxt[sl] = __dadd_rn(cur[2 * sl], cur[2 * sl + 1]);
        }
        double *tmp = cur; cur = nxt; nxt = tmp;
    }
    __syncthreads();
    if (threadIdx.x == 0) partial[blockIdx.x] = cur[0];
}

// fold 2^D partials pairwise (complete binary tree above depth D); partial
// has room for 2 * 2^D values (ping-pong halves).
__global__ void __launch_bounds__(1024) pw_fold(double *partial, int D, double *out,
                                                const unsigned long long *skip = nullptr) {
    if (skip && *skip) return;
    const i64 m = 1ll << D;
    double *src = partial, *dst = partial + m;
    for (i64 w = m; w > 1; w >>= 1) {
        for (i64 i = threadIdx.x; i < w / 2; i += blockDim.x) dst[i] = __dadd_rn(src[2 * i], src[2 * i + 1]);
        __syncthreads();
        double *t = src; src = dst; dst = t;
    }
    if (threadIdx.x == 0) *out = src[0];
}

template <class F>
int pairwise_sum(const F &f, i64 n, double *partial, double *out, cudaStream_t s,
                 const unsigned long long *skip = nullptr) {
    if (n <= 0) {
        cudaMemsetAsync(out, 0, sizeof(double), s);
        return ct::check_launch("pairwise empty");
    }
    const int D = pw_depth(n);
    if (pw_max_node(n, D) > 64 * MAX_LEAVES) {
        ct::set_error("pairwise subtree too large");
        return CT_ERR_UNSUPPORTED;
    }
    // tabulate the shapes of the distinct node sizes at depth D
    PwShapes shapes;
    shapes.count = 0;
    {
        i64 sizes[64];
        int ns = 1;
        sizes[0] = n;
        for (int d = 0; d < D; ++d) {
            i64 nxt[64];
            int nn = 0;
            for (int i = 0; i < ns; ++i) {
                const i64 l = pw_left(sizes[i]), c2[2] = {l, sizes[i] - l};
                for (int q = 0; q < 2; ++q) {
                    bool seen = false;
                    for (int u = 0; u < nn; ++u) seen |= nxt[u] == c2[q];
                    if (!seen && nn < 64) nxt[nn++] = c2[q];
                }
            }
            ns = nn;
            for (int i = 0; i < ns; ++i) sizes[i] = nxt[i];
        }
        for (int i = 0; i < ns && shapes.count < PW_NSH; ++i) {
            shapes.len[shapes.count] = (int)sizes[i];
            pw_shape(shapes.sh[shapes.count], (int)sizes[i]);
            ++shapes.count;
        }
    }
    pw_subtree<F><<<(unsigned)(1ll << D), PT, 0, s>>>(f, n, D, partial, shapes, skip);
    if (int st = ct::check_launch("pw_subtree")) return st;
    pw_fold<<<1, 1024, 0, s>>>(partial, D, out, skip);
    return ct::check_launch("pw_fold");
}

// ---------------------------------------------------------------------------
// Vectorised numpy-order sum of (lap - mean)^2 over the Laplacian array.
// Same tree as pw_subtree, but each leaf (<= 128 elements, 8-aligned) is one
// thread: numpy's 8 accumulators are 8 independent FP64 chains fed by 16-byte
// loads, and the in-subtree combine follows a host-built schedule (internal
// nodes grouped by height, so every group is independent) instead of
// per-thread tree descents.
// ---------------------------------------------------------------------------
constexpr int PWV_SUB = 8192;   // nodes at depth D hold >= 8192 elements
constexpr int PWV_LEAVES = 256; // leaves per subtree (sizes < 2*PWV_SUB + 16)
constexpr int PWV_NSH = 4;
constexpr int PWV_MAXH = 16;
constexpr int PWV_T = 128;

struct PwvTabs {
    int count;
    int len[PWV_NSH], nleaves[PWV_NSH], nh[PWV_NSH];
    int hstart[PWV_NSH][PWV_MAXH + 1];       // internal nodes of height h: [hstart[h-1], hstart[h])
    uint32_t leaf[PWV_NSH][PWV_LEAVES];      // offset << 8 | length
    uint32_t node[PWV_NSH][PWV_LEAVES];      // left | right << 16 (indices into leaves ++ nodes)
};

inline int pwv_depth(i64 n) {
    int d = 0;
    i64 m = n;
    while (m > 128 && pw_left(m) >= PWV_SUB && d < 24) {
        m = pw_left(m);
        ++d;
    }
    return d;
}

// builds node m at offset off; returns (value index, height)
inline bool pwv_build(PwvTabs &t, int q, int m, int off, std::vector<std::pair<int, int>> &nodes,
                      std::vector<int> &heights, int &idx, int &h) {
    if (m <= 128) {
        if (t.nleaves[q] >= PWV_LEAVES) return false;
        t.leaf[q][t.nleaves[q]] = ((uint32_t)off << 8) | (uint32_t)m;
        idx = t.nleaves[q]++;
        h = 0;
        return true;
    }
    const int l = (int)pw_left(m);
    int ia, ha, ib, hb;
    if (!pwv_build(t, q, l, off, nodes, heights, ia, ha) || !pwv_build(t, q, m - l, off + l, nodes, heights, ib, hb))
        return false;
    nodes.push_back({ia, ib});
    h = (ha > hb ? ha : hb) + 1;
    heights.push_back(h);
    idx = -(int)nodes.size();  // internal: resolved after sorting
    return true;
}

inline bool pwv_table(PwvTabs &t, int q, int len) {
    t.len[q] = len;
    t.nleaves[q] = 0;
    std::vector<std::pair<int, int>> nodes;
    std::vector<int> heights;
    int idx, h;
    if (!pwv_build(t, q, len, 0, nodes, heights, idx, h) || h > PWV_MAXH) return false;
    const int nl = t.nleaves[q], ni = (int)nodes.size();
    // order internal nodes by height; value index of internal node = nl + position
    std::vector<int> order(ni), pos(ni);
    for (int i = 0; i < ni; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return heights[a] < heights[b]; });
    for (int i = 0; i < ni; ++i) pos[order[i]] = i;
    auto vidx = [&](int v) { return v >= 0 ? v : nl + pos[-v - 1]; };
    t.nh[q] = h;
    for (int hh = 0; hh <= PWV_MAXH; ++hh) t.hstart[q][hh] = 0;
    for (int i = 0; i < ni; ++i) {
        const int n = order[i];
        t.node[q][i] = (uint32_t)vidx(nodes[n].first) | ((uint32_t)vidx(nodes[n].second) << 16);
        t.hstart[q][heights[n]] = i + 1;
    }
    for (int hh = 1; hh <= h; ++hh)
        if (t.hstart[q][hh] < t.hstart[q][hh - 1]) t.hstart[q][hh] = t.hstart[q][hh - 1];
    return true;
}

template <typename LT>
__device__ __forceinline__ void load8(const LT *p, double (&x)[8]);
template <>
__device__ __forceinline__ void load8<int16_t>(const int16_t *p, double (&x)[8]) {
    const int4 v = __ldg((const int4 *)p);
    const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        x[2 * i] = (double)(int16_t)(w[i] & 0xffff);
        x[2 * i + 1] = (double)(int16_t)(w[i] >> 16);
    }
}
template <>
__device__ __forceinline__ void load8<int32_t>(const int32_t *p, double (&x)[8]) {
    const int4 a = __ldg((const int4 *)p), b = __ldg((const int4 *)p + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}

template <typename LT>
__global__ void __launch_bounds__(PWV_T) pw_subtree_lap(const LT *__restrict__ lap, const double *__restrict__ meanp,
                                                        i64 n, int D, double *__restrict__ partial,
                                                        const __grid_constant__ PwvTabs tabs,
                                                        const unsigned long long *skip) {
    if (skip && *skip) return;
    __shared__ double val[2 * PWV_LEAVES];
    i64 off, len;
    pw_node(n, D, blockIdx.x, off, len);
    int q = 0;
    for (int i = 1; i < tabs.count; ++i)
        if (tabs.len[i] == (int)len) q = i;
    const double mean = *meanp;
    const int nl = tabs.nleaves[q];
    auto sq = [&](double x) { const double d = __dadd_rn(x, -mean); return __dmul_rn(d, d); };
    for (int L = threadIdx.x; L < nl; L += PWV_T) {
        const uint32_t e = tabs.leaf[q][L];
        const int m = (int)(e & 0xff);
        const LT *a = lap + off + (e >> 8);
        double res;
        if (m < 8) {
            res = 0.0;
            for (int i = 0; i < m; ++i) res = __dadd_rn(res, sq((double)a[i]));
        } else {
            double r[8], x[8];
            load8<LT>(a, x);
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = sq(x[j]);
            const int lim = m - (m & 7);
            for (int i = 8; i < lim; i += 8) {
                load8<LT>(a + i, x);
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sq(x[j]));
            }
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (int i = lim; i < m; ++i) res = __dadd_rn(res, sq((double)a[i]));
        }
        val[L] = res;
    }
    for (int h = 1; h <= tabs.nh[q]; ++h) {
        __syncthreads();
        for (int i = tabs.hstart[q][h - 1] + threadIdx.x; i < tabs.hstart[q][h]; i += PWV_T) {
            const uint32_t nd = tabs.node[q][i];
            val[nl + i] = __dadd_rn(val[nd & 0xffff], val[nd >> 16]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) partial[blockIdx.x] = nl > 1 ? val[nl + tabs.hstart[q][tabs.nh[q]] - 1] : val[0];
}

// returns 1 when the shapes do not fit the tables (caller falls back)
template <typename LT>
int pairwise_sum_lap(const LT *lap, const double *mean, i64 n, double *partial, double *out, cudaStream_t s,
                     const unsigned long long *skip = nullptr) {
    if (n < 8 || ((uintptr_t)lap & 15) != 0 || n >= (1ll << 31)) return 1;
    const int D = pwv_depth(n);
    static thread_local i64 cached_n = -1;
    static thread_local PwvTabs tabs;
    static thread_local bool ok = false;
    if (cached_n != n) {
        cached_n = n;
        ok = true;
        i64 sizes[64];
        int ns = 1;
        sizes[0] = n;
        for (int d = 0; d < D && ok; ++d) {
            i64 nxt[64];
            int nn = 0;
            for (int i = 0; i < ns; ++i) {
                const i64 l = pw_left(sizes[i]), c2[2] = {l, sizes[i] - l};
                for (int k = 0; k < 2; ++k) {
                    bool seen = false;
                    for (int u = 0; u < nn; ++u) seen |= nxt[u] == c2[k];
                    if (!seen) {
                        if (nn == 64) { ok = false; break; }
                        nxt[nn++] = c2[k];
                    }
                }
            }
            ns = nn;
            for (int i = 0; i < ns; ++i) sizes[i] = nxt[i];
        }
        if (ns > PWV_NSH || sizes[0] >= (1 << 23)) ok = false;
        tabs.count = ns;
        for (int i = 0; i < ns && ok; ++i) ok = pwv_table(tabs, i, (int)sizes[i]);
    }
    if (!ok) return 1;
    pw_subtree_lap<LT><<<(unsigned)(1ll << D), PWV_T, 0, s>>>(lap, mean, n, D, partial, tabs, skip);
    if (int st = ct::check_launch("pw_subtree_lap")) return -st;
    pw_fold<<<1, 1024, 0, s>>>(partial, D, out, skip);
    if (int st = ct::check_launch("pw_fold")) return -st;
    return 0;
}

// state words
enum { S_DELTA = 0, S_SIGMA, S_SIGMA_STATUS, S_NNZ, S_NORM, S_DECISION, S_SUM1, S_SUM2, S_SUM3, S_WORDS };
// scalar words (u64) in the workspace
enum { W_NNZ = 0, W_BEST_BITS, W_MOVED, W_LAPSUM, W_LAPSQ, W_SKIP, W_WORDS = 8 };

// ---------------------------------------------------------------------------
// Streaming statistics pass (integer input): a CTA owns MJ rows (j) x all k
// and walks a chunk of planes along i with a 3-plane SMEM ring (the load of
// plane i+2 is issued before plane i is processed, so its latency hides
// behind compute; one barrier per plane).  Per voxel: histogram (byte
// counters for u8, SMEM atomics for u16), sign sum != 0, and for interior
// voxels the Laplacian -> exact int64 sum + int32 array in numpy's flattened
// interior order.
// ---------------------------------------------------------------------------
constexpr int MJ = 8;
constexpr int MIPER = 64;  // planes per CTA
constexpr int WIPER = 32;  // planes per CTA of the register walks (mrf_decide_walk*): 2+ waves on C2

template <typename T, typename LT>
__global__ void __launch_bounds__(256) mrf_stream_int(const T *__restrict__ v, i64 nx, i64 ny, int nz,
                                                      unsigned long long *__restrict__ ghist,
                                                      unsigned long long *__restrict__ scal,
                                                      LT *__restrict__ lap) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int PL = (MJ + 2) * nz;  // staged plane elements
    int *ring = (int *)dsm;        // [3][PL]
    unsigned char *hbase = dsm + ((3 * PL * 4 + 15) & ~15);
    constexpr bool BYTE = sizeof(T) == 1;
    // u8: one 256-bin u32 histogram per warp (8 KB); u16: 4096 shared bins
    uint32_t *sh16 = (uint32_t *)hbase;
    uint32_t *wh = sh16 + (threadIdx.x >> 5) * 256;
    for (int b = threadIdx.x; b < (BYTE ? 8 * 256 : 4096); b += 256) sh16[b] = 0;
    const i64 nJ = (ny + MJ - 1) / MJ;
    const i64 j0 = (blockIdx.x % nJ) * MJ;
    const i64 i0 = (blockIdx.x / nJ) * MIPER, i1 = min(i0 + MIPER, nx);
    const i64 my = ny - 2, mz = nz - 2;
    const int npos = MJ * nz;
    // thread positions (<= 4 per thread for nz <= 128)
    constexpr int MAXP = 4;
    int pj[MAXP], pk[MAXP];
    int np_ = 0;
    for (int p = threadIdx.x; p < npos && np_ < MAXP; p += 256, ++np_) {
        pj[np_] = p / nz;
        pk[np_] = p - pj[np_] * nz;
    }
    auto load_plane = [&](i64 i, int *regs) {
        const i64 ic = ct::clampi(i, 0, nx - 1);
        int q = 0;
        for (int e = threadIdx.x; e < PL; e += 256, ++q) {
            const int r = e / nz, k = e - r * nz;
            const i64 j = ct::clampi(j0 - 1 + r, 0, ny - 1);
            regs[q] = (int)v[(ic * ny + j) * nz + k];
        }
    };
    auto store_plane = [&](int slot, const int *regs) {
        int q = 0;
        for (int e = threadIdx.x; e < PL; e += 256, ++q) ring[slot * PL + e] = regs[q];
    };
    constexpr int MAXR = (MJ + 2) * 128 / 256 + 1;
    int regs[MAXR];
    // prologue: planes i0-1 (prev values) and i0, i0+1 into the ring
    load_plane(i0 - 1, regs);
    store_plane(2, regs);
    load_plane(i0, regs);
    store_plane(0, regs);
    load_plane(i0 + 1, regs);
    store_plane(1, regs);
    __syncthreads();
    int prev[MAXP];
    for (int q = 0; q < np_; ++q) prev[q] = ring[2 * PL + (pj[q] + 1) * nz + pk[q]];
    __syncthreads();  // plane i0-1 read by all before iteration i0 stores into its slot
    unsigned long long nnz = 0;
    long long lsum = 0;
    for (i64 i = i0; i < i1; ++i) {
        const int cs = (int)((i - i0) % 3), ns = (int)((i - i0 + 1) % 3), fs = (int)((i - i0 + 2) % 3);
        load_plane(i + 2, regs);  // in flight while plane i is processed
        const int *C = ring + cs * PL, *X = ring + ns * PL;
        const bool iint = i > 0 && i < nx - 1;
        for (int q = 0; q < np_; ++q) {
            const int jj = pj[q], k = pk[q];
            const i64 j = j0 + jj;
            if (j >= ny) continue;
            const int c = C[(jj + 1) * nz + k];
            const int xm = prev[q], xp = X[(jj + 1) * nz + k];
            const int ym = C[jj * nz + k], yp = C[(jj + 2) * nz + k];
            const int zm = k > 0 ? C[(jj + 1) * nz + k - 1] : c, zp = k < nz - 1 ? C[(jj + 1) * nz + k + 1] : c;
            const int sgs = ((xm > c) - (xm < c)) + ((c > xp) - (c < xp)) + ((ym > c) - (ym < c)) +
                            ((c > yp) - (c < yp)) + ((zm > c) - (zm < c)) + ((c > zp) - (c < zp));
            nnz += sgs != 0;
            if (iint && j > 0 && j < ny - 1 && k > 0 && k < nz - 1) {
                const int l = (xm + xp + ym + yp + zm + zp) - 6 * c;
                lsum += l;
                lap[((i - 1) * my + (j - 1)) * mz + (k - 1)] = (LT)l;
            }
            if (BYTE) atomicAdd(&wh[c], 1u);
            else if (c < 4096) atomicAdd(&sh16[c], 1u);
            else atomicAdd(&ghist[c], 1ull);
            prev[q] = c;
        }
        store_plane(fs, regs);
        __syncthreads();
    }
    for (int o = 16; o; o >>= 1) {
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&scal[W_NNZ], nnz);
        atomicAdd(&scal[W_LAPSUM], (unsigned long long)lsum);
    }
    __syncthreads();
    if (BYTE) {
        unsigned t = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += sh16[q * 256 + threadIdx.x];
        if (t) atomicAdd(&ghist[threadIdx.x], (unsigned long long)t);
    } else {
        for (int b = threadIdx.x; b < 4096; b += 256)
            if (sh16[b]) atomicAdd(&ghist[b], (unsigned long long)sh16[b]);
    }
}

// Same pass specialised for nz == NZ (32, 64, 128): thread t owns column
// k = t % NZ of rows t / NZ + p * (256 / NZ); planes staged as raw T in SMEM
// via 32-bit vector loads; 32-bit indexing (volumes < 2^31 voxels).
// MODE as in mrf_stream_v4: 0 = histogram, #{sign sum != 0}, Laplacian sum
// and Laplacians; 1 = histogram, #{sign sum != 0} and E = sum of squared
// forward differences (the certified decision's bound, ct_mrf_decide), no
// Laplacians; 2 = Laplacians and their sum only, nothing when certified.
template <typename T, typename LT, int NZ, int MODE = 0>
__global__ void __launch_bounds__(256) mrf_stream_nz(const T *__restrict__ v, int nx, int ny,
                                                     unsigned long long *__restrict__ ghist,
                                                     unsigned long long *__restrict__ scal,
                                                     LT *__restrict__ lap) {
    if (MODE == 2 && *(volatile unsigned long long *)&scal[W_SKIP]) return;
    constexpr int RP = 256 / NZ;           // rows per thread sweep
    constexpr int P = MJ / RP;             // positions per thread
    constexpr int PL = (MJ + 2) * NZ;      // staged plane elements
    constexpr int PW = PL * (int)sizeof(T) / 4;  // 32-bit words per plane
    constexpr int LW = (PW + 255) / 256;   // words per thread
    constexpr int RW = NZ * (int)sizeof(T) / 4;  // words per row
    constexpr bool BYTE = sizeof(T) == 1;
    __shared__ __align__(16) T ring[3][PL];
    __shared__ uint32_t hsm[BYTE ? 8 * 256 : 4096];
    uint32_t *wh = hsm + (BYTE ? (threadIdx.x >> 5) * 256 : 0);
    for (int b = threadIdx.x; b < (BYTE ? 8 * 256 : 4096); b += 256) hsm[b] = 0;
    const int nJ = (ny + MJ - 1) / MJ;
    const int j0 = (blockIdx.x % nJ) * MJ;
    const int i0 = (blockIdx.x / nJ) * MIPER, i1 = min(i0 + MIPER, nx);
    const int my = ny - 2, mz = NZ - 2;
    const int k = threadIdx.x % NZ, jt = threadIdx.x / NZ;
    // word w of a plane: row w / RW (clamped j), word w % RW
    int goff[LW];
#pragma unroll
    for (int q = 0; q < LW; ++q) {
        const int w = threadIdx.x + q * 256;
        const int row = w / RW, cw = w - row * RW;
        const int j = min(max(j0 - 1 + row, 0), ny - 1);
        goff[q] = w < PW ? j * RW + cw : 0;
    }
    const uint32_t *vw = (const uint32_t *)v;
    const size_t plane_w = (size_t)ny * RW;
    auto load_plane = [&](int i, uint32_t (&regs)[LW]) {
        const int ic = min(max(i, 0), nx - 1);
        const uint32_t *base = vw + (size_t)ic * plane_w;
#pragma unroll
        for (int q = 0; q < LW; ++q)
            if (threadIdx.x + q * 256 < PW) regs[q] = __ldg(base + goff[q]);
    };
    auto store_plane = [&](int slot, const uint32_t (&regs)[LW]) {
        uint32_t *dst = (uint32_t *)ring[slot];
#pragma unroll
        for (int q = 0; q < LW; ++q)
            if (threadIdx.x + q * 256 < PW) dst[threadIdx.x + q * 256] = regs[q];
    };
    uint32_t regs[LW];
    load_plane(i0 - 1, regs);
    store_plane(2, regs);
    load_plane(i0, regs);
    store_plane(0, regs);
    load_plane(i0 + 1, regs);
    store_plane(1, regs);
    __syncthreads();
    int prev[P];
#pragma unroll
    for (int p = 0; p < P; ++p) prev[p] = ring[2][(jt + p * RP + 1) * NZ + k];
    __syncthreads();  // plane i0-1 read by all before iteration i0 stores into its slot
    unsigned nnz = 0;
    long long lsum = 0;
    unsigned long long esq = 0;  // MODE 1 (clamped neighbours make boundary differences 0)
    int cs = 0, ns = 1, fs = 2;
    for (int i = i0; i < i1; ++i) {
        load_plane(i + 2, regs);  // in flight while plane i is processed
        const T *C = ring[cs], *X = ring[ns];
        const bool iint = i > 0 && i < nx - 1;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int jj = jt + p * RP, j = j0 + jj;
            if (j < ny) {
                const int o = (jj + 1) * NZ + k;
                const int c = C[o];
                const int xm = prev[p], xp = X[o];
                const int ym = C[o - NZ], yp = C[o + NZ];
                const int zm = k > 0 ? C[o - 1] : c, zp = k < NZ - 1 ? C[o + 1] : c;
                if (MODE != 2) {
                    const int sgs = ((xm > c) - (xm < c)) + ((c > xp) - (c < xp)) + ((ym > c) - (ym < c)) +
                                    ((c > yp) - (c < yp)) + ((zm > c) - (zm < c)) + ((c > zp) - (c < zp));
                    nnz += sgs != 0;
                    if (BYTE || c < 4096) atomicAdd(&wh[c], 1u);
                    else atomicAdd(&ghist[c], 1ull);
                }
                if (MODE == 1) {
                    const long long dx = xp - c, dy = yp - c, dz = zp - c;
                    esq += (unsigned long long)(dx * dx + dy * dy + dz * dz);
                } else if (iint && j > 0 && j < ny - 1 && k > 0 && k < NZ - 1) {
                    const int l = (xm + xp + ym + yp + zm + zp) - 6 * c;
                    lsum += l;
                    CT_DCHECK(i - 1 < nx - 2 && j - 1 < my && k - 1 < mz);
                    lap[((unsigned)(i - 1) * (unsigned)my + (unsigned)(j - 1)) * (unsigned)mz + (unsigned)(k - 1)] =
                        (LT)l;
                }
                prev[p] = c;
            }
        }
        store_plane(fs, regs);
        __syncthreads();
        const int t = cs; cs = ns; ns = fs; fs = t;
    }
    unsigned long long nnz64 = nnz;
    for (int o = 16; o; o >>= 1) {
        nnz64 += __shfl_xor_sync(0xffffffffu, nnz64, o);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        esq += __shfl_xor_sync(0xffffffffu, esq, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (MODE != 2) atomicAdd(&scal[W_NNZ], nnz64);
        if (MODE != 1) atomicAdd(&scal[W_LAPSUM], (unsigned long long)lsum);
        if (MODE == 1) atomicAdd(&scal[W_LAPSQ], esq);
    }
    if (MODE == 2) return;
    __syncthreads();
    if (BYTE) {
        unsigned t = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += hsm[q * 256 + threadIdx.x];
        if (t) atomicAdd(&ghist[threadIdx.x], (unsigned long long)t);
    } else {
        for (int b = threadIdx.x; b < 4096; b += 256)
            if (hsm[b]) atomicAdd(&ghist[b], (unsigned long long)hsm[b]);
    }
}

// per byte: bit 7 set iff a > b (unsigned), other bits clear.  s7 = [a_lo >
// b_lo] from (a & 0x7f) + (127 - b_lo); then a > b = (a7 & ~b7) | (a7 == b7 & s7).
__device__ __forceinline__ uint32_t gt_hi(uint32_t a, uint32_t b) {
    const uint32_t s = (a & 0x7f7f7f7fu) + (~b & 0x7f7f7f7fu);
    return ((a & ~b) | (~(a ^ b) & s)) & 0x80808080u;
}

// u8 input, nz == NZ: 4 voxels per thread as one 32-bit word (SIMD byte
// compares for the sign sum, packed 16-bit lanes for the Laplacian).  A CTA
// owns MJ4 = 256 / (NZ/4) rows and walks MIPER planes along i with the same
// 3-plane SMEM ring.  Edge neighbours are clamped exactly like the scalar
// kernels (j, i by the clamped row/plane loads; k by byte replication).
// MODE 0: histogram, #{sign sum != 0}, Laplacian sum and the Laplacians
// (lap) for the exact pairwise sigma_hat.  MODE 1 (certified quick decision,
// ct_mrf_decide): histogram, #{sign sum != 0} and the sum of squared forward
// differences E (W_LAPSQ) of the sigma bound -- no Laplacians.  MODE 2: the
// fallback of MODE 1 -- Laplacians and their sum only, and nothing at all
// when the quick decision certified (scal[W_SKIP]).
template <int NZ, int MODE = 0>
__global__ void __launch_bounds__(256) mrf_stream_v4(const uint8_t *__restrict__ v, int nx, int ny,
                                                     unsigned long long *__restrict__ ghist,
                                                     unsigned long long *__restrict__ scal,
                                                     int16_t *__restrict__ lap) {
    if (MODE == 2 && *(volatile unsigned long long *)&scal[W_SKIP]) return;
    constexpr int W = NZ / 4;               // words per row
    constexpr int MJ4 = 256 / W;            // rows per CTA
    constexpr int PW = (MJ4 + 2) * W;       // staged words per plane
    constexpr int LW = (PW + 255) / 256;
    // plane ring: i-1, i, i+1 and the slot plane i+2 is stored into.  When
    // rows do not tile the warps (NZ = 96) the Laplacian path reads plane i-1
    // from the ring (nb0 below), so the write slot must be a fourth one (the
    // store is not behind a barrier); otherwise it is plane i-1's slot.
    constexpr int NSLOT = (32 % W == 0) ? 3 : 4;
    __shared__ uint32_t ring[NSLOT][PW];
    __shared__ uint32_t hsm[8 * 256];
    uint32_t *wh = hsm + (threadIdx.x >> 5) * 256;
    for (int b = threadIdx.x; b < 8 * 256; b += 256) hsm[b] = 0;
    const int nJ = (ny + MJ4 - 1) / MJ4;
    const int j0 = (blockIdx.x % nJ) * MJ4;
    const int i0 = (blockIdx.x / nJ) * MIPER, i1 = min(i0 + MIPER, nx);
    const int my = ny - 2, mz = NZ - 2;
    const int jj = threadIdx.x / W, kw = threadIdx.x % W, j = j0 + jj;
    const bool own = jj < MJ4;  // (NZ = 96: 256 = 10 rows x 24 words + 16 idle threads)
    int goff[LW];
#pragma unroll
    for (int q = 0; q < LW; ++q) {
        const int w = threadIdx.x + q * 256;
        const int row = w / W, cw = w - row * W;
        goff[q] = w < PW ? min(max(j0 - 1 + row, 0), ny - 1) * W + cw : 0;
    }
    const uint32_t *vw = (const uint32_t *)v;
    const size_t plane_w = (size_t)ny * W;
    auto load_plane = [&](int i, uint32_t (&regs)[LW]) {
        const uint32_t *base = vw + (size_t)min(max(i, 0), nx - 1) * plane_w;
#pragma unroll
        for (int q = 0; q < LW; ++q)
            if (threadIdx.x + q * 256 < PW) regs[q] = __ldg(base + goff[q]);
    };
    auto store_plane = [&](int slot, const uint32_t (&regs)[LW]) {
#pragma unroll
        for (int q = 0; q < LW; ++q)
            if (threadIdx.x + q * 256 < PW) ring[slot][threadIdx.x + q * 256] = regs[q];
    };
    uint32_t regs[LW], regs2[LW];
    load_plane(i0 - 1, regs);
    store_plane(2, regs);
    load_plane(i0, regs);
    store_plane(0, regs);
    load_plane(i0 + 1, regs);
    store_plane(1, regs);
    load_plane(i0 + 2, regs2);  // two planes ahead from here on
    __syncthreads();
    const int o = own ? (jj + 1) * W + kw : W;
    uint32_t xm = ring[2][o];
    unsigned nnz = 0;
    long long lsum = 0;
    const bool jin = own && j < ny, jint = j > 0 && j < ny - 1;
    int cs = 0, ns = 1, fs = 2, ws = NSLOT == 4 ? 3 : 2;  // fs: plane i-1, ws: write slot
    // MODE 1: the x-direction comparisons of plane i against i+1 are reused
    // as plane i+1's comparisons against its i-1 neighbour (gxm, lxm)
    uint32_t gxm = 0, lxm = 0;
    if (MODE == 1) {
        const uint32_t c0 = ring[0][o];
        gxm = gt_hi(xm, c0);
        lxm = gt_hi(c0, xm);
    }
    // every thread has read plane i0-1 (slot 2) before the first iteration's
    // store may replace it (NSLOT = 3: the write slot of iteration i0 is slot 2)
    __syncthreads();
    unsigned esq = 0;  // MODE 1: sum of squared forward differences (edge term of the sigma bound)
    for (int i = i0; i < i1; ++i) {
        load_plane(i + 3, regs);  // planes i+2 (regs2) and i+3 (regs) in flight while plane i is processed
        const uint32_t c = ring[cs][o], xp = ring[ns][o];
        const uint32_t ym = ring[cs][o - W], yp = ring[cs][o + W];
        const uint32_t wl = kw > 0 ? ring[cs][o - 1] : c << 24, wr = kw < W - 1 ? ring[cs][o + 1] : c >> 24;
        const uint32_t zm = __funnelshift_l(wl, c, 8), zp = __funnelshift_r(c, wr, 8);
        if constexpr (MODE == 1) {
            // sign sum != 0 per byte <=> #(+1 terms) != #(-1 terms) <=> pos ^ neg != 0 (both <= 6)
            const uint32_t gxp = gt_hi(c, xp), lxp = gt_hi(xp, c);
            const uint32_t pos = ((gxm >> 7) + (gxp >> 7)) + ((gt_hi(ym, c) >> 7) + (gt_hi(c, yp) >> 7)) +
                                 ((gt_hi(zm, c) >> 7) + (gt_hi(c, zp) >> 7));
            const uint32_t neg = ((lxm >> 7) + (lxp >> 7)) + ((gt_hi(c, ym) >> 7) + (gt_hi(yp, c) >> 7)) +
                                 ((gt_hi(c, zm) >> 7) + (gt_hi(zp, c) >> 7));
            gxm = gxp;
            lxm = lxp;
            if (jin) {
                nnz += __popc(((pos ^ neg) + 0x7f7f7f7fu) & 0x80808080u);
                atomicAdd(&wh[c & 0xff], 1u);
                atomicAdd(&wh[(c >> 8) & 0xff], 1u);
                atomicAdd(&wh[(c >> 16) & 0xff], 1u);
                atomicAdd(&wh[c >> 24], 1u);
                // clamped neighbours make the boundary differences 0
                const uint32_t dx4 = __vabsdiffu4(c, xp), dy4 = __vabsdiffu4(c, yp), dz4 = __vabsdiffu4(c, zp);
                esq = __dp4a(dx4, dx4, esq);
                esq = __dp4a(dy4, dy4, esq);
                esq = __dp4a(dz4, dz4, esq);
            }
        } else {
        // sign sum != 0 per byte: #(+1 terms) != #(-1 terms)
        const uint32_t one = 0x01010101u;
        const uint32_t pos = (__vcmpgtu4(xm, c) & one) + (__vcmpgtu4(c, xp) & one) + (__vcmpgtu4(ym, c) & one) +
                             (__vcmpgtu4(c, yp) & one) + (__vcmpgtu4(zm, c) & one) + (__vcmpgtu4(c, zp) & one);
        const uint32_t neg = (__vcmpgtu4(c, xm) & one) + (__vcmpgtu4(xp, c) & one) + (__vcmpgtu4(c, ym) & one) +
                             (__vcmpgtu4(yp, c) & one) + (__vcmpgtu4(c, zm) & one) + (__vcmpgtu4(zp, c) & one);
        // Laplacian in 16-bit lanes: bytes 0, 2 (lo) and 1, 3 (hi)
        const uint32_t m16 = 0x00ff00ffu;
        const uint32_t sl = (xm & m16) + (xp & m16) + (ym & m16) + (yp & m16) + (zm & m16) + (zp & m16);
        const uint32_t sh = ((xm >> 8) & m16) + ((xp >> 8) & m16) + ((ym >> 8) & m16) + ((yp >> 8) & m16) +
                            ((zm >> 8) & m16) + ((zp >> 8) & m16);
        const uint32_t ll = __vsub2(sl, (c & m16) * 6u), lh = __vsub2(sh, ((c >> 8) & m16) * 6u);
        // voxel b's Laplacian: b0 = ll.lo, b1 = lh.lo, b2 = ll.hi, b3 = lh.hi
        const uint32_t w01 = __byte_perm(ll, lh, 0x5410), w23 = __byte_perm(ll, lh, 0x7632);
        // next word's b0 (voxel k = 4 kw + 4): from the neighbour lane when rows
        // are whole within warps, else recomputed from the ring (slot fs holds plane i-1)
        uint32_t nb0;
        if constexpr (32 % W == 0) {
            nb0 = __shfl_down_sync(0xffffffffu, w01 & 0xffffu, 1);
        } else {
            const int o1 = kw < W - 1 ? o + 1 : o;
            const int c1 = (int)(ring[cs][o1] & 0xffu);
            const int s6 = (int)(ring[fs][o1] & 0xffu) + (int)(ring[ns][o1] & 0xffu) + (int)(ring[cs][o1 - W] & 0xffu) +
                           (int)(ring[cs][o1 + W] & 0xffu) + (int)(c >> 24) + (int)((ring[cs][o1] >> 8) & 0xffu);
            nb0 = (uint32_t)(s6 - 6 * c1) & 0xffffu;
        }
        if (jin) {
            if (MODE == 0) {
                nnz += __popc(__vcmpne4(pos, neg)) >> 3;
                atomicAdd(&wh[c & 0xff], 1u);
                atomicAdd(&wh[(c >> 8) & 0xff], 1u);
                atomicAdd(&wh[(c >> 16) & 0xff], 1u);
                atomicAdd(&wh[c >> 24], 1u);
            }
            if (jint && i > 0 && i < nx - 1) {
                // elements k-1 for k = 4kw+1 .. 4kw+4 (two aligned 32-bit words)
                const uint32_t e0 = __byte_perm(w01, w23, 0x5432), e1 = __byte_perm(w23, nb0, 0x5432);
                uint32_t *dst = (uint32_t *)(lap + ((size_t)(i - 1) * my + (j - 1)) * mz + 4 * kw);
                dst[0] = e0;
                lsum += (int)(int16_t)(e0 & 0xffff) + (int)(int16_t)(e0 >> 16);
                if (kw < W - 1) {
                    dst[1] = e1;
                    lsum += (int)(int16_t)(e1 & 0xffff) + (int)(int16_t)(e1 >> 16);
                }
            }
        }
        }
        xm = c;
        store_plane(ws, regs2);
#pragma unroll
        for (int q = 0; q < LW; ++q) regs2[q] = regs[q];
        __syncthreads();
        const int t = fs;
        fs = cs; cs = ns; ns = ws;
        ws = NSLOT == 4 ? t : fs;
    }
    unsigned long long nnz64 = nnz, esq64 = esq;
    for (int q = 16; q; q >>= 1) {
        nnz64 += __shfl_xor_sync(0xffffffffu, nnz64, q);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, q);
        if (MODE == 1) esq64 += __shfl_xor_sync(0xffffffffu, esq64, q);
    }
    if ((threadIdx.x & 31) == 0) {
        if (MODE != 2) atomicAdd(&scal[W_NNZ], nnz64);
        if (MODE != 1) atomicAdd(&scal[W_LAPSUM], (unsigned long long)lsum);
        if (MODE == 1) atomicAdd(&scal[W_LAPSQ], esq64);
    }
    if (MODE == 2) return;
    __syncthreads();
    unsigned tt = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) tt += hsm[q * 256 + threadIdx.x];
    if (tt) atomicAdd(&ghist[threadIdx.x], (unsigned long long)tt);
}

// MODE 1 of mrf_stream_v4 without the shared-memory plane ring (NZ in {32,
// 64, 128}: a row is 8 / 16 / 32 lanes).  ncu on mrf_stream_v4<64, 1>: the
// per-plane __syncthreads of the ring and the ring loads were ~40% of the
// stall samples with one word per thread and plane.  Here a thread owns the
// word (j, kw) of every plane of its slab and walks i with the x-neighbours in
// registers; the y-neighbours (rows j -+ 1, clamped) are loaded from global
// memory (the rows of the neighbouring lanes' words: L1 hits), the
// z-neighbours come from the row's lanes by shuffles; plane i+1's loads are
// in flight while plane i is processed.  No barriers inside the walk.  Same
// per-byte arithmetic and results as mrf_stream_v4<NZ, 1>.
// Per byte lane, bit 7 only (the other bits are don't-care until the final
// mask): a > b is the carry out of a + ~b = maj(a7, ~b7, s7) with s = (a & 7f)
// + (~b & 7f); both orders of a pair share the masked operands.  The six +1
// and six -1 terms of a voxel's sign sum are counted in carry-save form (full
// adders on whole words), and the sum is nonzero iff the two 3-bit counts
// differ.
__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }
__device__ __forceinline__ void fadd(uint32_t a, uint32_t b, uint32_t c, uint32_t &s, uint32_t &cy) {
    s = a ^ b ^ c;
    cy = maj3(a, b, c);
}
// 3-bit count (b0, b1, b2) of six bit-7 flags
__device__ __forceinline__ void count6(uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3, uint32_t f4, uint32_t f5,
                                       uint32_t &b0, uint32_t &b1, uint32_t &b2) {
    uint32_t s1, c1, s2, c2;
    fadd(f0, f1, f2, s1, c1);
    fadd(f3, f4, f5, s2, c2);
    b0 = s1 ^ s2;
    const uint32_t c3 = s1 & s2;
    fadd(c1, c2, c3, b1, b2);
}

template <int NZ>
__global__ void __launch_bounds__(256) mrf_decide_walk(const uint8_t *__restrict__ v, int nx, int ny,
                                                       unsigned long long *__restrict__ ghist,
                                                       unsigned long long *__restrict__ scal) {
    constexpr int W = NZ / 4, RPC = 256 / W;  // words per row, rows per CTA
    static_assert(W == 8 || W == 16 || W == 32, "row = whole lane segment");
    constexpr uint32_t M7 = 0x7f7f7f7fu;
    __shared__ uint32_t hsm[8 * 256];
    uint32_t *wh = hsm + (threadIdx.x >> 5) * 256;
    for (int b = threadIdx.x; b < 8 * 256; b += 256) hsm[b] = 0;
    __syncthreads();
    const int nJ = (ny + RPC - 1) / RPC;
    const int j = (blockIdx.x % nJ) * RPC + (int)threadIdx.x / W, kw = (int)threadIdx.x % W;
    const int i0 = (blockIdx.x / nJ) * WIPER, i1 = min(i0 + WIPER, nx);
    const bool jin = j < ny;
    const int jc = min(j, ny - 1), jm = max(jc - 1, 0), jp = min(jc + 1, ny - 1);
    const size_t plane_w = (size_t)ny * W;
    // row pointers of plane i (ym, yp rows) and of plane i+2 (the centre row)
    const uint32_t *pm = (const uint32_t *)v + (size_t)i0 * plane_w + (size_t)jm * W + kw;
    const uint32_t *pp = pm + (size_t)(jp - jm) * W;
    const uint32_t *pc2 = pm + (size_t)(jc - jm) * W + (size_t)(min(i0 + 2, nx - 1) - i0) * plane_w;
    const uint32_t *pc = pm + (size_t)(jc - jm) * W;
    uint32_t xm = __ldg(pc - (i0 > 0 ? plane_w : 0)), c = __ldg(pc), xp = __ldg(pc + (i0 + 1 < nx ? plane_w : 0));
    uint32_t ym = __ldg(pm), yp = __ldg(pp);
    // x-pair flags of plane i against i-1: gt(xm, c) (+1) and gt(c, xm) (-1)
    uint32_t gxm, lxm;
    {
        const uint32_t cm = c & M7, nm = xm & M7;
        gxm = maj3(xm, ~c, nm + M7 - cm);
        lxm = maj3(c, ~xm, cm + M7 - nm);
    }
    unsigned nnz = 0, esq = 0;
    for (int i = i0; i < i1; ++i) {
        // plane i+1's loads in flight (rows clamped at the volume's faces)
        const bool more = i + 1 < nx;
        pm += more ? plane_w : 0;
        pp += more ? plane_w : 0;
        const uint32_t xp2 = __ldg(pc2), ym2 = __ldg(pm), yp2 = __ldg(pp);
        pc2 += i + 3 < nx ? plane_w : 0;
        const uint32_t wl0 = __shfl_up_sync(0xffffffffu, c, 1, W), wr0 = __shfl_down_sync(0xffffffffu, c, 1, W);
        const uint32_t wl = kw > 0 ? wl0 : c << 24, wr = kw < W - 1 ? wr0 : c >> 24;
        const uint32_t zm = __funnelshift_l(wl, c, 8), zp = __funnelshift_r(c, wr, 8);
        const uint32_t cm = c & M7;
        uint32_t gn[5], gc[5];  // gt(n, c), gt(c, n) for n = xp, ym, yp, zm, zp
        const uint32_t nb[5] = {xp, ym, yp, zm, zp};
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const uint32_t nm = nb[u] & M7;
            gn[u] = maj3(nb[u], ~c, nm + M7 - cm);
            gc[u] = maj3(c, ~nb[u], cm + M7 - nm);
        }
        // +1: gt(xm,c), gt(c,xp), gt(ym,c), gt(c,yp), gt(zm,c), gt(c,zp); -1: the reverses
        uint32_t p0, p1, p2, n0, n1, n2;
        count6(gxm, gc[0], gn[1], gc[2], gn[3], gc[4], p0, p1, p2);
        count6(lxm, gn[0], gc[1], gn[2], gc[3], gn[4], n0, n1, n2);
        gxm = gc[0];
        lxm = gn[0];
        if (jin) {
            nnz += __popc(((p0 ^ n0) | (p1 ^ n1) | (p2 ^ n2)) & 0x80808080u);
            atomicAdd(&wh[c & 0xff], 1u);
            atomicAdd(&wh[(c >> 8) & 0xff], 1u);
            atomicAdd(&wh[(c >> 16) & 0xff], 1u);
            atomicAdd(&wh[c >> 24], 1u);
            const uint32_t dx4 = __vabsdiffu4(c, xp), dy4 = __vabsdiffu4(c, yp), dz4 = __vabsdiffu4(c, zp);
            esq = __dp4a(dx4, dx4, esq);
            esq = __dp4a(dy4, dy4, esq);
            esq = __dp4a(dz4, dz4, esq);
        }
        xm = c;
        c = xp;
        xp = xp2;
        ym = ym2;
        yp = yp2;
    }
    unsigned long long nnz64 = nnz, esq64 = esq;
    for (int q = 16; q; q >>= 1) {
        nnz64 += __shfl_xor_sync(0xffffffffu, nnz64, q);
        esq64 += __shfl_xor_sync(0xffffffffu, esq64, q);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&scal[W_NNZ], nnz64);
        atomicAdd(&scal[W_LAPSQ], esq64);
    }
    __syncthreads();
    unsigned tt = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) tt += hsm[q * 256 + threadIdx.x];
    if (tt) atomicAdd(&ghist[threadIdx.x], (unsigned long long)tt);
}

// u16 form of mrf_decide_walk (nz in {32, 64}: a row is 16 / 32 lanes of
// 2-voxel words): the same walk, 16-bit lanes (a > b = carry-out majority at
// bit 15), carry-save counting, the 4096-bin SMEM histogram of mrf_stream_nz
// (values >= 4096 to global), E in 64-bit integers.  Results equal
// mrf_stream_nz<uint16_t, ., NZ, 1>'s.
template <int NZ>
__global__ void __launch_bounds__(256) mrf_decide_walk16(const uint16_t *__restrict__ v, int nx, int ny,
                                                         unsigned long long *__restrict__ ghist,
                                                         unsigned long long *__restrict__ scal) {
    constexpr int W = NZ / 2, RPC = 256 / W;  // words per row, rows per CTA
    static_assert(W == 16 || W == 32, "row = whole lane segment");
    constexpr uint32_t M15 = 0x7fff7fffu;
    __shared__ uint32_t hsm[4096];
    for (int b = threadIdx.x; b < 4096; b += 256) hsm[b] = 0;
    __syncthreads();
    const int nJ = (ny + RPC - 1) / RPC;
    const int j = (blockIdx.x % nJ) * RPC + (int)threadIdx.x / W, kw = (int)threadIdx.x % W;
    const int i0 = (blockIdx.x / nJ) * WIPER, i1 = min(i0 + WIPER, nx);
    const bool jin = j < ny;
    const int jc = min(j, ny - 1), jm = max(jc - 1, 0), jp = min(jc + 1, ny - 1);
    const size_t plane_w = (size_t)ny * W;
    const uint32_t *pm = (const uint32_t *)v + (size_t)i0 * plane_w + (size_t)jm * W + kw;
    const uint32_t *pp = pm + (size_t)(jp - jm) * W;
    const uint32_t *pc = pm + (size_t)(jc - jm) * W;
    const uint32_t *pc2 = pc + (size_t)(min(i0 + 2, nx - 1) - i0) * plane_w;
    uint32_t xm = __ldg(pc - (i0 > 0 ? plane_w : 0)), c = __ldg(pc), xp = __ldg(pc + (i0 + 1 < nx ? plane_w : 0));
    uint32_t ym = __ldg(pm), yp = __ldg(pp);
    uint32_t gxm, lxm;
    {
        const uint32_t cm = c & M15, nm = xm & M15;
        gxm = maj3(xm, ~c, nm + M15 - cm);
        lxm = maj3(c, ~xm, cm + M15 - nm);
    }
    unsigned nnz = 0;
    unsigned long long esq = 0;
    auto hadd = [&](uint32_t val) {
        if (val < 4096) atomicAdd(&hsm[val], 1u);
        else atomicAdd(&ghist[val], 1ull);
    };
    auto sq2 = [](uint32_t a, uint32_t b) {  // sum of the two lanes' squared differences
        const int d0 = (int)(a & 0xffffu) - (int)(b & 0xffffu), d1 = (int)(a >> 16) - (int)(b >> 16);
        return (unsigned long long)((long long)d0 * d0) + (unsigned long long)((long long)d1 * d1);
    };
    for (int i = i0; i < i1; ++i) {
        const bool more = i + 1 < nx;
        pm += more ? plane_w : 0;
        pp += more ? plane_w : 0;
        const uint32_t xp2 = __ldg(pc2), ym2 = __ldg(pm), yp2 = __ldg(pp);
        pc2 += i + 3 < nx ? plane_w : 0;
        const uint32_t wl0 = __shfl_up_sync(0xffffffffu, c, 1, W), wr0 = __shfl_down_sync(0xffffffffu, c, 1, W);
        const uint32_t wl = kw > 0 ? wl0 : c << 16, wr = kw < W - 1 ? wr0 : c >> 16;
        const uint32_t zm = __funnelshift_l(wl, c, 16), zp = __funnelshift_r(c, wr, 16);
        const uint32_t cm = c & M15;
        uint32_t gn[5], gc[5];
        const uint32_t nb[5] = {xp, ym, yp, zm, zp};
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const uint32_t nm = nb[u] & M15;
            gn[u] = maj3(nb[u], ~c, nm + M15 - cm);
            gc[u] = maj3(c, ~nb[u], cm + M15 - nm);
        }
        uint32_t p0, p1, p2, n0, n1, n2;
        count6(gxm, gc[0], gn[1], gc[2], gn[3], gc[4], p0, p1, p2);
        count6(lxm, gn[0], gc[1], gn[2], gc[3], gn[4], n0, n1, n2);
        gxm = gc[0];
        lxm = gn[0];
        if (jin) {
            nnz += __popc(((p0 ^ n0) | (p1 ^ n1) | (p2 ^ n2)) & 0x80008000u);
            hadd(c & 0xffffu);
            hadd(c >> 16);
            esq += sq2(c, xp) + sq2(c, yp) + sq2(c, zp);
        }
        xm = c;
        c = xp;
        xp = xp2;
        ym = ym2;
        yp = yp2;
    }
    unsigned long long nnz64 = nnz;
    for (int q = 16; q; q >>= 1) {
        nnz64 += __shfl_xor_sync(0xffffffffu, nnz64, q);
        esq += __shfl_xor_sync(0xffffffffu, esq, q);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&scal[W_NNZ], nnz64);
        atomicAdd(&scal[W_LAPSQ], esq);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 4096; b += 256)
        if (hsm[b]) atomicAdd(&ghist[b], (unsigned long long)hsm[b]);
}

// float input: #{sign sum != 0} only (delta via sort; sums via the tree)
template <typename T>
__global__ void mrf_nnz_generic(const T *__restrict__ v, i64 nx, i64 ny, i64 nz, unsigned long long *__restrict__ nnz) {
    const i64 n = nx * ny * nz;
    unsigned long long local = 0;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
        local += sign_sum_at<T>(v, nullptr, nx, ny, nz, p) != 0;
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(nnz, local);
}

// exact integer sum of the interior Laplacians (integer input of any shape;
// the stream kernels form it on the fly for nz <= 128)
template <typename T>
__global__ void lap_sum_int(const T *__restrict__ v, i64 ny, i64 nz, uint32_t my, uint32_t mz, i64 ni,
                            unsigned long long *__restrict__ sum) {
    long long local = 0;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < ni; e += (i64)gridDim.x * blockDim.x)
        local += (long long)lap_at(v, (uint32_t)e, my, mz, ny, nz);
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(sum, (unsigned long long)local);
}

// delta from the histogram of integer values (min gap of non-empty bins)
// (nbins: 256 for u8 input -- no other bin can be non-empty -- else 65536)
__global__ void delta_from_hist(const uint64_t *__restrict__ hist, int nbins, double *state) {
    __shared__ int prev_of[1024];
    __shared__ int wg[32], wlo[32], whi[32];
    const int t = threadIdx.x;
    // the non-empty span first (coalesced): 12-bit data in 65536 bins scans 4096
    int lo = INT32_MAX, hi = -1;
#pragma unroll 16
    for (int b = t; b < nbins; b += 1024)
        if (hist[b]) {
            lo = min(lo, b);
            hi = b;
        }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((t & 31) == 0) {
        wlo[t >> 5] = lo;
        whi[t >> 5] = hi;
    }
    __syncthreads();
    lo = INT32_MAX;
    hi = -1;
    for (int i = 0; i < 32; ++i) {
        lo = min(lo, wlo[i]);
        hi = max(hi, whi[i]);
    }
    const int span = hi >= lo ? hi - lo + 1 : 0;
    const int per = (span + 1023) / 1024, b0 = lo + t * per, b1 = min(b0 + per, hi + 1);
    int first = -1, last = -1, gap = INT32_MAX;
    for (int b = b0; b < b1; ++b) {
        if (!hist[b]) continue;
        if (last >= 0) gap = min(gap, b - last);
        if (first < 0) first = b;
        last = b;
    }
    prev_of[t] = last;
    __syncthreads();
    if (first >= 0) {
        for (int u = t - 1; u >= 0; --u)
            if (prev_of[u] >= 0) { gap = min(gap, first - prev_of[u]); break; }
    }
    for (int o = 16; o; o >>= 1) gap = min(gap, __shfl_xor_sync(0xffffffffu, gap, o));
    if ((t & 31) == 0) wg[t >> 5] = gap;
    __syncthreads();
    if (t == 0) {
        int g = INT32_MAX;
        for (int i = 0; i < 32; ++i) g = min(g, wg[i]);
        state[S_DELTA] = g == INT32_MAX ? 0.0 : (double)g;
    }
}

// delta from a sorted float64 copy: min positive gap between neighbours
__global__ void delta_from_sorted(const double *__restrict__ s, i64 n, unsigned long long *__restrict__ best_bits) {
    unsigned long long best = ~0ull;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x + 1; i < n; i += (i64)gridDim.x * blockDim.x) {
        if (s[i] != s[i - 1]) {
            const double d = __dadd_rn(s[i], -s[i - 1]);
            best = min(best, (unsigned long long)__double_as_longlong(d));  // d > 0: bit order == value order
        }
    }
    for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(best_bits, best);
}

__global__ void delta_store(const unsigned long long *best_bits, double *state) {
    state[S_DELTA] = *best_bits == ~0ull ? 0.0 : __longlong_as_double((long long)*best_bits);
}

__global__ void mean_from_sum(double *state, i64 n) { state[S_SUM1] = __ddiv_rn(state[S_SUM1], (double)n); }
__global__ void lap_mean(double *state, const long long *sum, i64 n, const unsigned long long *skip = nullptr) {
    if (skip && *skip) return;  // certified by mrf_quick: the Laplacian sums were not formed
    state[S_SUM1] = __ddiv_rn((double)*sum, (double)n);
}

// Certified first-step decision without sigma_hat (ct_mrf_decide).  The
// reference stops before its first step iff ||delta sign(S)|| > sigma_hat
// (denoise.py:172-176); for integer input the norm is sqrt(delta^2 nnz)
// exactly, and sigma_hat = std(L)/sqrt(42) <= sqrt(sum L^2 / n)/sqrt(42)
// (variance <= mean square) <= sqrt(12 E / n)/sqrt(42): L = sum of the six
// (neighbour - centre) differences, so L^2 <= 6 * sum of their squares
// (Cauchy-Schwarz), and over the interior every grid edge is counted at most
// twice -- E = sum over all forward edges of the squared difference.  When the
// norm beats that bound (with a 2^-20 relative margin for the reference's
// float64 rounding of std) the decision is 0 without the exact pairwise sum;
// a constant grid (delta 0) is decided too.  Otherwise scal[W_SKIP] stays 0
// and the exact kernels that follow (guarded by it) compute sigma_hat.
__global__ void mrf_quick(double *state, i64 n_interior, unsigned long long *scal) {
    const unsigned long long nnz = scal[W_NNZ];
    const double delta = state[S_DELTA];
    const double norm = __dsqrt_rn(__dmul_rn(__dmul_rn(delta, delta), (double)nnz));
    const double bound = __dmul_rn(__ddiv_rn(__dsqrt_rn(__ddiv_rn(12.0 * (double)scal[W_LAPSQ], (double)n_interior)),
                                             __dsqrt_rn(42.0)), 1.0 + 0x1p-20);
    if (n_interior >= 2 && (delta == 0.0 || norm > bound)) {
        state[S_NNZ] = (double)nnz;
        state[S_SUM3] = __dmul_rn(__dmul_rn(delta, delta), (double)nnz);
        state[S_NORM] = norm;
        state[S_SIGMA] = __longlong_as_double(0x7ff8000000000000ll);  // NaN: not computed
        state[S_SUM1] = state[S_SIGMA];                               // nor the Laplacian moments
        state[S_SUM2] = state[S_SIGMA];
        state[S_SIGMA_STATUS] = 2.0;                  // skipped (decision certified)
        state[S_DECISION] = delta == 0.0 ? 2.0 : 0.0;
        scal[W_SKIP] = 1;
    }
}

// int_path: norm^2 = delta^2 * nnz (exact); else state[S_SUM3] holds the tree sum
__global__ void mrf_decide(double *state, i64 n_interior, const unsigned long long *scal, int int_path) {
    if (scal[W_SKIP]) return;  // certified by mrf_quick
    if (n_interior < 2) {
        state[S_SIGMA] = 0.0;
        state[S_SIGMA_STATUS] = 1.0;
    } else {
        const double var = __ddiv_rn(state[S_SUM2], (double)n_interior);
        state[S_SIGMA] = __ddiv_rn(__dsqrt_rn(var), __dsqrt_rn(42.0));
        state[S_SIGMA_STATUS] = 0.0;
    }
    const unsigned long long nnz = scal[W_NNZ];
    state[S_NNZ] = (double)nnz;
    if (int_path) {
        state[S_SUM1] = n_interior > 0 ? __ddiv_rn((double)(long long)scal[W_LAPSUM], (double)n_interior) : 0.0;
        state[S_SUM3] = __dmul_rn(__dmul_rn(state[S_DELTA], state[S_DELTA]), (double)nnz);
    }
    const double norm = __dsqrt_rn(state[S_SUM3]);
    state[S_NORM] = norm;
    if (state[S_DELTA] == 0.0) state[S_DECISION] = 2.0;       // constant: input returned as is
    else if (norm > state[S_SIGMA]) state[S_DECISION] = 0.0;  // stop before the first step
    else if (nnz == 0) state[S_DECISION] = 0.0;               // fixed point
    else state[S_DECISION] = 1.0;                             // iterate (host loop)
}

template <typename T>
__global__ void mrf_apply(const T *__restrict__ v, const double *__restrict__ cur, i64 nx, i64 ny, i64 nz,
                          const double *__restrict__ delta_p, double *__restrict__ next,
                          unsigned long long *__restrict__ moved) {
    const i64 n = nx * ny * nz;
    const double delta = *delta_p;
    unsigned long long local = 0;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        const double c = cur ? cur[p] : ct::to_f64(v[p]);
        const int s = sgn((double)sign_sum_at(v, cur, nx, ny, nz, p));
        const double prop = __dadd_rn(c, __dmul_rn(delta, (double)s));
        next[p] = prop;
        local += prop != c;
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(moved, local);
}

template <typename T>
__global__ void sign_sum_kernel(const T *__restrict__ v, i64 nx, i64 ny, i64 nz, int64_t *__restrict__ out) {
    const i64 n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
        out[p] = sign_sum_at<T>(v, nullptr, nx, ny, nz, p);
}

__global__ void step_finish(double *out2, const unsigned long long *moved) {
    out2[0] = __dsqrt_rn(out2[0]);
    out2[1] = (double)*moved;
}

struct MrfWork {
    void *lap;                 // integer path: n_interior Laplacians (int16 for u8, int32 for u16)
    double *partial;           // 2 * 2^D
    unsigned long long *scal;  // W_WORDS
    double *sorted;            // float path: n
    void *cub_tmp;
    size_t cub_bytes;
};

size_t cub_sort_bytes(i64 n) {
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, (const double *)nullptr, (double *)nullptr, (int)n);
    return b;
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

inline i64 interior(i64 nx, i64 ny, i64 nz) {
    return (nx > 2 ? nx - 2 : 0) * (ny > 2 ? ny - 2 : 0) * (nz > 2 ? nz - 2 : 0);
}

MrfWork mrf_carve(void *work, i64 n, int dtype, i64 ni) {
    MrfWork w;
    char *p = (char *)work;
    w.lap = nullptr;
    if (dtype != CT_F64) {
        w.lap = p;
        p += al(ni * (dtype == CT_U8 ? 2 : 4));
    }
    const i64 parts = 1ll << pw_depth(n > 0 ? n : 1);
    w.partial = (double *)p; p += al(parts * 8 * 2 + 64);
    w.scal = (unsigned long long *)p; p += al(W_WORDS * 8);
    w.sorted = nullptr; w.cub_tmp = nullptr; w.cub_bytes = 0;
    if (dtype == CT_F64) {
        w.sorted = (double *)p; p += al(n * 8);
        w.cub_bytes = cub_sort_bytes(n);
        w.cub_tmp = p;
    }
    return w;
}

template <typename T>
int mrf_int(const T *v, i64 nx, i64 ny, i64 nz, MrfWork &w, double *state, uint64_t *hist, cudaStream_t s,
            bool quick = false) {
    const i64 mx = nx - 2 > 0 ? nx - 2 : 0, my = ny - 2 > 0 ? ny - 2 : 0, mz = nz - 2 > 0 ? nz - 2 : 0;
    const i64 ni = mx * my * mz;
    using LT = typename std::conditional<sizeof(T) == 1, int16_t, int32_t>::type;
    LT *lap = (LT *)w.lap;
    const i64 blocks = ((ny + MJ - 1) / MJ) * ((nx + MIPER - 1) / MIPER);
    if (sizeof(T) == 1 && (nz == 32 || nz == 64 || nz == 96 || nz == 128) && ((uintptr_t)v & 3) == 0 &&
        ((uintptr_t)lap & 3) == 0 &&
        nx * ny * nz < (1ll << 31)) {
        const i64 b4 = ((ny + 256 / (nz / 4) - 1) / (256 / (nz / 4))) * ((nx + MIPER - 1) / MIPER);
        auto launch = [&](auto kern) {
            kern<<<(unsigned)b4, 256, 0, s>>>((const uint8_t *)v, (int)nx, (int)ny, (unsigned long long *)hist,
                                              w.scal, (int16_t *)lap);
        };
        if (quick && ni >= 2) {
            // certified decision first; the Laplacians are stored (MODE 2) only if it fails
            const i64 bwk = ((ny + 256 / (nz / 4) - 1) / (256 / (nz / 4))) * ((nx + WIPER - 1) / WIPER);
            auto walk = [&](auto kern) {
                kern<<<(unsigned)bwk, 256, 0, s>>>((const uint8_t *)v, (int)nx, (int)ny, (unsigned long long *)hist,
                                                  w.scal);
            };
            if (nz == 32) walk(mrf_decide_walk<32>);
            else if (nz == 64) walk(mrf_decide_walk<64>);
            else if (nz == 96) launch(mrf_stream_v4<96, 1>);
            else walk(mrf_decide_walk<128>);
            if (int st = ct::check_launch("mrf_stream_v4")) return st;
            delta_from_hist<<<1, 1024, 0, s>>>(hist, 256, state);
            mrf_quick<<<1, 1, 0, s>>>(state, ni, w.scal);
            if (nz == 32) launch(mrf_stream_v4<32, 2>);
            else if (nz == 64) launch(mrf_stream_v4<64, 2>);
            else if (nz == 96) launch(mrf_stream_v4<96, 2>);
            else launch(mrf_stream_v4<128, 2>);
            if (int st = ct::check_launch("mrf_stream_v4 (exact sigma)")) return st;
            lap_mean<<<1, 1, 0, s>>>(state, (const long long *)&w.scal[W_LAPSUM], ni, &w.scal[W_SKIP]);
            const int vs = pairwise_sum_lap<LT>(lap, &state[S_SUM1], ni, w.partial, &state[S_SUM2], s, &w.scal[W_SKIP]);
            if (vs < 0) return -vs;
            if (vs == 1) {  // shapes outside the vectorised tables: the generic tree, same skip guard
                LapArrSq<LT> f{lap, &state[S_SUM1]};
                if (int st = pairwise_sum(f, ni, w.partial, &state[S_SUM2], s, &w.scal[W_SKIP])) return st;
            }
            mrf_decide<<<1, 1, 0, s>>>(state, ni, w.scal, 1);
            return ct::check_launch("mrf_decide");
        }
        if (nz == 32) launch(mrf_stream_v4<32>);
        else if (nz == 64) launch(mrf_stream_v4<64>);
        else if (nz == 96) launch(mrf_stream_v4<96>);
        else launch(mrf_stream_v4<128>);
        if (int st = ct::check_launch("mrf_stream_v4")) return st;
    } else if ((nz == 32 || nz == 64 || nz == 128) && ((uintptr_t)v & 3) == 0 && nx * ny * nz < (1ll << 31)) {
        if (quick && ni >= 2) {
            // certified decision first (MODE 1); Laplacians (MODE 2) only if it fails
            auto k1 = nz == 32 ? mrf_stream_nz<T, LT, 32, 1> : nz == 64 ? mrf_stream_nz<T, LT, 64, 1>
                                                                         : mrf_stream_nz<T, LT, 128, 1>;
            auto k2 = nz == 32 ? mrf_stream_nz<T, LT, 32, 2> : nz == 64 ? mrf_stream_nz<T, LT, 64, 2>
                                                                         : mrf_stream_nz<T, LT, 128, 2>;
            if (sizeof(T) == 2 && nz <= 64) {  // barrier-free walk (u16 words of two voxels)
                const int rpc = 256 / ((int)nz / 2);
                const unsigned bw = (unsigned)(((ny + rpc - 1) / rpc) * ((nx + WIPER - 1) / WIPER));
                auto kw = nz == 32 ? mrf_decide_walk16<32> : mrf_decide_walk16<64>;
                kw<<<bw, 256, 0, s>>>((const uint16_t *)v, (int)nx, (int)ny, (unsigned long long *)hist, w.scal);
            } else {
                k1<<<(unsigned)blocks, 256, 0, s>>>(v, (int)nx, (int)ny, (unsigned long long *)hist, w.scal, lap);
            }
            if (int st = ct::check_launch("mrf_stream_nz")) return st;
            delta_from_hist<<<1, 1024, 0, s>>>(hist, sizeof(T) == 1 ? 256 : 65536, state);
            mrf_quick<<<1, 1, 0, s>>>(state, ni, w.scal);
            k2<<<(unsigned)blocks, 256, 0, s>>>(v, (int)nx, (int)ny, (unsigned long long *)hist, w.scal, lap);
            if (int st = ct::check_launch("mrf_stream_nz (exact sigma)")) return st;
            lap_mean<<<1, 1, 0, s>>>(state, (const long long *)&w.scal[W_LAPSUM], ni, &w.scal[W_SKIP]);
            const int vs = pairwise_sum_lap<LT>(lap, &state[S_SUM1], ni, w.partial, &state[S_SUM2], s, &w.scal[W_SKIP]);
            if (vs < 0) return -vs;
            if (vs == 1) {
                LapArrSq<LT> f{lap, &state[S_SUM1]};
                if (int st = pairwise_sum(f, ni, w.partial, &state[S_SUM2], s, &w.scal[W_SKIP])) return st;
            }
            mrf_decide<<<1, 1, 0, s>>>(state, ni, w.scal, 1);
            return ct::check_launch("mrf_decide");
        }
        auto kern = nz == 32 ? mrf_stream_nz<T, LT, 32> : nz == 64 ? mrf_stream_nz<T, LT, 64> : mrf_stream_nz<T, LT, 128>;
        kern<<<(unsigned)blocks, 256, 0, s>>>(v, (int)nx, (int)ny, (unsigned long long *)hist, w.scal, lap);
        if (int st = ct::check_launch("mrf_stream_nz")) return st;
    } else if (nz <= 128) {
        const size_t hb = sizeof(T) == 1 ? 8 * 256 * sizeof(uint32_t) : 4096 * sizeof(uint32_t);
        const size_t sm = ((3 * (MJ + 2) * nz * 4 + 15) & ~(size_t)15) + hb;
        cudaFuncSetAttribute(mrf_stream_int<T, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        mrf_stream_int<T, LT><<<(unsigned)blocks, 256, sm, s>>>(v, nx, ny, (int)nz, (unsigned long long *)hist,
                                                               w.scal, lap);
        if (int st = ct::check_launch("mrf_stream_int")) return st;
    } else {
        // nz > 128: the same statistics from global memory, no stored Laplacians
        // (ct_workspace_bytes(4, ...) covers this path too): input histogram,
        // #{sign sum != 0}, the exact Laplacian sum, then numpy's pairwise tree
        // over (lap - mean)^2 with the Laplacians recomputed per element
        if (int st = ct_histogram(v, sizeof(T) == 1 ? CT_U8 : CT_U16, nx * ny * nz, hist, s)) return st;
        delta_from_hist<<<1, 1024, 0, s>>>(hist, sizeof(T) == 1 ? 256 : 65536, state);
        mrf_nnz_generic<T><<<ct::grid_for(nx * ny * nz, 256, CT_NUM_SMS * 4), 256, 0, s>>>(v, nx, ny, nz,
                                                                                           &w.scal[W_NNZ]);
        if (int st = ct::check_launch("mrf_nnz_generic")) return st;
        if (ni >= 2) {
            lap_sum_int<T><<<ct::grid_for(ni, 256, CT_NUM_SMS * 4), 256, 0, s>>>(v, ny, nz, (uint32_t)my,
                                                                                 (uint32_t)mz, ni,
                                                                                 &w.scal[W_LAPSUM]);
            if (int st = ct::check_launch("lap_sum_int")) return st;
            LapElem<T> f2{v, ny, nz, (uint32_t)my, (uint32_t)mz, nullptr, (const long long *)&w.scal[W_LAPSUM],
                          ni, 1};
            if (int st = pairwise_sum(f2, ni, w.partial, &state[S_SUM2], s)) return st;
        }
        mrf_decide<<<1, 1, 0, s>>>(state, ni, w.scal, 1);
        return ct::check_launch("mrf_decide");
    }
    delta_from_hist<<<1, 1024, 0, s>>>(hist, sizeof(T) == 1 ? 256 : 65536, state);
    if (int st = ct::check_launch("delta_from_hist")) return st;
    if (ni >= 2) {
        lap_mean<<<1, 1, 0, s>>>(state, (const long long *)&w.scal[W_LAPSUM], ni);
        const int vs = pairwise_sum_lap<LT>(lap, &state[S_SUM1], ni, w.partial, &state[S_SUM2], s);
        if (vs < 0) return -vs;
        if (vs == 1) {
            LapArrSq<LT> f{lap, &state[S_SUM1]};
            if (int st = pairwise_sum(f, ni, w.partial, &state[S_SUM2], s)) return st;
        }
    }
    mrf_decide<<<1, 1, 0, s>>>(state, ni, w.scal, 1);
    return ct::check_launch("mrf_decide");
}

int mrf_f64(const double *v, i64 nx, i64 ny, i64 nz, MrfWork &w, double *state, cudaStream_t s) {
    const i64 n = nx * ny * nz;
    const i64 mx = nx - 2 > 0 ? nx - 2 : 0, my = ny - 2 > 0 ? ny - 2 : 0, mz = nz - 2 > 0 ? nz - 2 : 0;
    const i64 ni = mx * my * mz;
    mrf_nnz_generic<double><<<ct::grid_for(n, 256, CT_NUM_SMS * 4), 256, 0, s>>>(v, nx, ny, nz, &w.scal[W_NNZ]);
    if (int st = ct::check_launch("mrf_nnz")) return st;
    size_t tb = w.cub_bytes;
    cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, v, w.sorted, (int)n, 0, 64, s);
    delta_from_sorted<<<ct::grid_for(n, 256, CT_NUM_SMS * 4), 256, 0, s>>>(w.sorted, n, &w.scal[W_BEST_BITS]);
    delta_store<<<1, 1, 0, s>>>(&w.scal[W_BEST_BITS], state);
    if (int st = ct::check_launch("mrf delta")) return st;
    if (ni >= 2) {
        LapElem<double> f1{v, ny, nz, (uint32_t)my, (uint32_t)mz, nullptr, nullptr, ni, 0};
        if (int st = pairwise_sum(f1, ni, w.partial, &state[S_SUM1], s)) return st;
        mean_from_sum<<<1, 1, 0, s>>>(state, ni);
        LapElem<double> f2{v, ny, nz, (uint32_t)my, (uint32_t)mz, &state[S_SUM1], nullptr, ni, 1};
        if (int st = pairwise_sum(f2, ni, w.partial, &state[S_SUM2], s)) return st;
    }
    StepElem<double> f3{v, nullptr, nx, ny, nz, &state[S_DELTA]};
    if (int st = pairwise_sum(f3, n, w.partial, &state[S_SUM3], s)) return st;
    mrf_decide<<<1, 1, 0, s>>>(state, ni, w.scal, 0);
    return ct::check_launch("mrf_decide");
}

}  // namespace

size_t ct_mrf_workspace(int64_t nx, int64_t ny, int64_t nz, int dtype) {
    const i64 n = nx * ny * nz;
    const i64 parts = 1ll << pw_depth(n > 0 ? n : 1);
    size_t b = al(parts * 8 * 2 + 64) + al(W_WORDS * 8);
    if (dtype != CT_F64) b += al(interior(nx, ny, nz) * (dtype == CT_U8 ? 2 : 4));
    if (dtype == CT_F64) b += al(n * 8) + al(cub_sort_bytes(n));
    return b + 1024;
}

extern "C" int ct_mrf(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, void *work, double *state,
                      uint64_t *hist, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("cannot denoise an empty grid");
        return CT_ERR_PARAM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    if (n >= (1ll << 31)) {
        ct::set_error("MRF limited to 2^31 voxels");
        return CT_ERR_UNSUPPORTED;
    }
    if (dtype != CT_F64 && !hist) {
        ct::set_error("integer MRF needs a (zeroed) histogram buffer");
        return CT_ERR_PARAM;
    }
    MrfWork w = mrf_carve(work, n, dtype, interior(nx, ny, nz));
    cudaMemsetAsync(state, 0, S_WORDS * sizeof(double), s);
    cudaMemsetAsync(w.scal, 0, W_WORDS * 8, s);
    cudaMemsetAsync(&w.scal[W_BEST_BITS], 0xff, 8, s);
    switch (dtype) {
        case CT_U8: return mrf_int<uint8_t>((const uint8_t *)in, nx, ny, nz, w, state, hist, s);
        case CT_U16: return mrf_int<uint16_t>((const uint16_t *)in, nx, ny, nz, w, state, hist, s);
        case CT_F64: return mrf_f64((const double *)in, nx, ny, nz, w, state, s);
        default:
            ct::set_error("unsupported dtype %d", dtype);
            return CT_ERR_UNSUPPORTED;
    }
}

// ct_mrf with a certified first-step decision (see mrf_quick): identical
// state except that sigma_hat (state[1]) is NaN with status state[2] = 2 when
// the decision was certified without it.  Non-u8 / unsupported shapes run the
// full ct_mrf.
extern "C" int ct_mrf_decide(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, void *work,
                             double *state, uint64_t *hist, void *stream) {
    if ((dtype != CT_U8 && dtype != CT_U16) || nx <= 0 || ny <= 0 || nz <= 0 || nx * ny * nz >= (1ll << 31) || !hist)
        return ct_mrf(in, dtype, nx, ny, nz, work, state, hist, stream);
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    MrfWork w = mrf_carve(work, n, dtype, interior(nx, ny, nz));
    cudaMemsetAsync(state, 0, S_WORDS * sizeof(double), s);
    cudaMemsetAsync(w.scal, 0, W_WORDS * 8, s);
    cudaMemsetAsync(&w.scal[W_BEST_BITS], 0xff, 8, s);
    if (dtype == CT_U16)
        return mrf_int<uint16_t>((const uint16_t *)in, nx, ny, nz, w, state, hist, s, true);
    return mrf_int<uint8_t>((const uint8_t *)in, nx, ny, nz, w, state, hist, s, true);
}

extern "C" int ct_mrf_step(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, const double *cur,
                           const double *state, double *next, void *work, double *out2, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    MrfWork w = mrf_carve(work, n, dtype, interior(nx, ny, nz));
    cudaMemsetAsync(&w.scal[W_MOVED], 0, 8, s);
    CT_DISPATCH(dtype, T, {
        const T *v = (const T *)in;
        StepElem<T> f{v, cur, nx, ny, nz, &state[S_DELTA]};
        if (int st = pairwise_sum(f, n, w.partial, &out2[0], s)) return st;
        mrf_apply<T><<<ct::grid_for(n, 256), 256, 0, s>>>(v, cur, nx, ny, nz, state + S_DELTA, next,
                                                          &w.scal[W_MOVED]);
        if (int st = ct::check_launch("mrf_apply")) return st;
    });
    step_finish<<<1, 1, 0, s>>>(out2, &w.scal[W_MOVED]);
    return ct::check_launch("mrf_step_finish");
}

// ref denoise.py:117-132 _neighbor_sign_sum: int64 sign sum, edges replicated.
extern "C" int ct_sign_sum(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, int64_t *out,
                           void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    if (n <= 0) return CT_OK;
    CT_DISPATCH(dtype, T, {
        sign_sum_kernel<T><<<ct::grid_for(n, 256), 256, 0, s>>>((const T *)in, nx, ny, nz, out);
    });
    return ct::check_launch("sign_sum");
}
