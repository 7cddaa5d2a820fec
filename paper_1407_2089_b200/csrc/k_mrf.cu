// k_mrf.cu -- K7: vessel-channel MRF denoise (ref denoise.py:92-195).
//
//   delta     = intensity_step: min gap of the distinct values (denoise.py:135-144)
//               integer input: from the histogram's non-empty bins;
//               float input: radix-sorted copy (CUB), min positive neighbour gap
//   sigma_hat = estimate_noise_variance (denoise.py:92-114) = np.std(lap)/sqrt(42)
//               over the interior 6-neighbour Laplacian.  np.std reduces with
//               numpy's pairwise summation (8-way unrolled leaves of <= 128,
//               halving splits rounded to multiples of 8); that tree is
//               reproduced exactly: CTA b sums the depth-D node b of the tree
//               (all depth-D nodes exist because D is chosen from the smallest
//               path), with the leaves below it enumerated and recombined in
//               recursion order, and one CTA folds the 2^D partials pairwise.
//   first step: proposal = I0 + delta*sign(S), S = edge-replicated sign sum
//               (denoise.py:117-132); stop when ||proposal - I0|| > sigma_hat
//               (denoise.py:173) or no voxel moves (denoise.py:175).  On
//               realistic volumes this stops at iteration 0; further iterations
//               run through ct_mrf_step driven by the host.
#include <cub/device/device_radix_sort.cuh>

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

// element functors over the flattened C-order interior (nx-2, ny-2, nz-2)
template <typename T>
struct LapElem {
    const T *v;
    i64 ny, nz, my, mz;
    const double *mean;  // device pointer (squared == 1)
    int squared;         // 0: lap, 1: (lap-mean)^2
    __device__ double operator()(i64 e) const {
        const i64 c = e % mz, b = (e / mz) % my, a = e / (mz * my);
        const i64 i = a + 1, j = b + 1, k = c + 1;
        const i64 s0 = ny * nz;
        const i64 p = i * s0 + j * nz + k;
        double l = __dadd_rn(ct::to_f64(v[p - s0]), ct::to_f64(v[p + s0]));
        l = __dadd_rn(l, ct::to_f64(v[p - nz]));
        l = __dadd_rn(l, ct::to_f64(v[p + nz]));
        l = __dadd_rn(l, ct::to_f64(v[p - 1]));
        l = __dadd_rn(l, ct::to_f64(v[p + 1]));
        l = __dadd_rn(l, -__dmul_rn(6.0, ct::to_f64(v[p])));
        if (!squared) return l;
        const double x = __dadd_rn(l, -*mean);
        return __dmul_rn(x, x);
    }
};

__device__ __forceinline__ int sgn(double x) { return (x > 0.0) - (x < 0.0); }

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

// (proposal - original)^2 for the step from `cur` (nullptr = original)
template <typename T>
struct StepElem {
    const T *v;
    const double *cur;
    i64 nx, ny, nz;
    const double *delta;  // device pointer
    __device__ double operator()(i64 p) const {
        const double c = cur ? cur[p] : ct::to_f64(v[p]);
        const int s = sgn((double)sign_sum_at(v, cur, nx, ny, nz, p));
        const double prop = __dadd_rn(c, __dmul_rn(*delta, (double)s));
        const double d = __dadd_rn(prop, -ct::to_f64(v[p]));
        return __dmul_rn(d, d);
    }
};

// numpy pairwise_sum leaf (n <= 128)
template <class F>
__device__ double pw_leaf(const F &f, i64 off, i64 n) {
    if (n < 8) {
        double res = 0.0;
        for (i64 i = 0; i < n; ++i) res = __dadd_rn(res, f(off + i));
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(off + j);
    i64 i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(off + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(off + i));
    return res;
}

// CTA b: exact numpy-order sum of depth-D node b.
template <class F>
__global__ void __launch_bounds__(PT) pw_subtree(F f, i64 n, int D, double *__restrict__ partial) {
    __shared__ i64 loff[MAX_LEAVES], llen[MAX_LEAVES];
    __shared__ double lsum[MAX_LEAVES];
    __shared__ int nleaves;
    i64 off, len;
    pw_node(n, D, blockIdx.x, off, len);
    if (threadIdx.x == 0) {
        // enumerate leaves in order (explicit DFS stack, right child pushed first)
        i64 so[64], sl[64];
        int sp = 0, nl = 0;
        so[sp] = off; sl[sp] = len; ++sp;
        while (sp) {
            --sp;
            const i64 o = so[sp], l = sl[sp];
            if (l <= 128) {
                loff[nl] = o; llen[nl] = l; ++nl;
            } else {
                const i64 h = pw_left(l);
                so[sp] = o + h; sl[sp] = l - h; ++sp;
                so[sp] = o; sl[sp] = h; ++sp;
            }
        }
        nleaves = nl;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nleaves; e += PT) lsum[e] = pw_leaf(f, loff[e], llen[e]);
    __syncthreads();
    if (threadIdx.x == 0) {
        // recombine in recursion order: post-order evaluation with a value stack
        i64 so[64], sl[64];
        int st[64];
        double vs[64];
        int sp = 0, vp = 0, leaf = 0;
        so[sp] = off; sl[sp] = len; st[sp] = 0; ++sp;
        while (sp) {
            const int top = sp - 1;
            const i64 o = so[top], l = sl[top];
            if (l <= 128) {
                vs[vp++] = lsum[leaf++];
                --sp;
            } else if (st[top] == 0) {
                st[top] = 1;
                const i64 h = pw_left(l);
                so[sp] = o; sl[sp] = h; st[sp] = 0; ++sp;
            } else if (st[top] == 1) {
                st[top] = 2;
                const i64 h = pw_left(l);
                so[sp] = o + h; sl[sp] = l - h; st[sp] = 0; ++sp;
            } else {
                const double b = vs[--vp], a = vs[--vp];
                vs[vp++] = __dadd_rn(a, b);
                --sp;
            }
        }
        partial[blockIdx.x] = vs[0];
    }
}

// fold 2^D partials pairwise (complete binary tree above depth D); partial
// has room for 2 * 2^D values (ping-pong halves).
__global__ void __launch_bounds__(1024) pw_fold(double *partial, int D, double *out) {
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
int pairwise_sum(const F &f, i64 n, double *partial, double *out, cudaStream_t s) {
    if (n <= 0) {
        cudaMemsetAsync(out, 0, sizeof(double), s);
        return ct::check_launch("pairwise empty");
    }
    const int D = pw_depth(n);
    pw_subtree<F><<<(unsigned)(1ll << D), PT, 0, s>>>(f, n, D, partial);
    if (int st = ct::check_launch("pw_subtree")) return st;
    pw_fold<<<1, 1024, 0, s>>>(partial, D, out);
    return ct::check_launch("pw_fold");
}

// state words
enum { S_DELTA = 0, S_SIGMA, S_SIGMA_STATUS, S_NNZ, S_NORM, S_DECISION, S_SUM1, S_SUM2, S_SUM3, S_WORDS };

template <typename T>
__global__ void mrf_stats(const T *__restrict__ v, i64 nx, i64 ny, i64 nz, uint64_t *__restrict__ hist,
                          unsigned long long *__restrict__ nnz) {
    __shared__ uint32_t sh[4096];
    __shared__ unsigned long long snz;
    for (int b = threadIdx.x; b < 4096; b += blockDim.x) sh[b] = 0;
    if (threadIdx.x == 0) snz = 0;
    __syncthreads();
    const i64 n = nx * ny * nz;
    unsigned long long local = 0;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
        local += sign_sum_at<T>(v, nullptr, nx, ny, nz, p) != 0;
        if (hist) {
            const int b = ct::hist_bin(v[p]);
            if (b < 4096) atomicAdd(&sh[b], 1u);
            else atomicAdd((unsigned long long *)&hist[b], 1ull);
        }
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&snz, local);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(nnz, snz);
    if (hist)
        for (int b = threadIdx.x; b < 4096; b += blockDim.x)
            if (sh[b]) atomicAdd((unsigned long long *)&hist[b], (unsigned long long)sh[b]);
}

// delta from the histogram of integer values (min gap of non-empty bins)
__global__ void delta_from_hist(const uint64_t *__restrict__ hist, double *state) {
    __shared__ int prev_of[1024];
    // each thread: first and last non-empty bin in its 64-bin chunk and its internal min gap
    const int t = threadIdx.x;
    int first = -1, last = -1, gap = INT32_MAX;
    for (int b = t * 64; b < t * 64 + 64; ++b) {
        if (!hist[b]) continue;
        if (last >= 0) gap = min(gap, b - last);
        if (first < 0) first = b;
        last = b;
    }
    prev_of[t] = last;
    __syncthreads();
    // gap to the previous non-empty chunk's last bin
    if (first >= 0) {
        for (int u = t - 1; u >= 0; --u)
            if (prev_of[u] >= 0) { gap = min(gap, first - prev_of[u]); break; }
    }
    for (int o = 16; o; o >>= 1) gap = min(gap, __shfl_xor_sync(0xffffffffu, gap, o));
    __shared__ int wg[32];
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

__global__ void mrf_decide(double *state, i64 n_interior, const unsigned long long *nnz) {
    const double n = (double)n_interior;
    if (n_interior < 2) {
        state[S_SIGMA] = 0.0;
        state[S_SIGMA_STATUS] = 1.0;
    } else {
        const double var = __ddiv_rn(state[S_SUM2], n);
        state[S_SIGMA] = __ddiv_rn(__dsqrt_rn(var), __dsqrt_rn(42.0));
        state[S_SIGMA_STATUS] = 0.0;
    }
    state[S_NNZ] = (double)*nnz;
    const double norm = __dsqrt_rn(state[S_SUM3]);
    state[S_NORM] = norm;
    if (state[S_DELTA] == 0.0) state[S_DECISION] = 2.0;             // constant: input returned as is
    else if (norm > state[S_SIGMA]) state[S_DECISION] = 0.0;        // stop before the first step
    else if (*nnz == 0) state[S_DECISION] = 0.0;                    // fixed point
    else state[S_DECISION] = 1.0;                                   // iterate (host loop)
}

__global__ void mean_from_sum(double *state, i64 n) { state[S_SUM1] = __ddiv_rn(state[S_SUM1], (double)n); }

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

struct MrfWork {
    double *partial;              // 2^D
    unsigned long long *scal;     // [4]: nnz, best_bits, moved, pad
    double *sorted;               // float path: n
    void *cub_tmp;
    size_t cub_bytes;
};

size_t cub_sort_bytes(i64 n) {
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, (const double *)nullptr, (double *)nullptr, (int)n);
    return b;
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

MrfWork mrf_carve(void *work, i64 n, int dtype) {
    MrfWork w;
    char *p = (char *)work;
    const i64 parts = 1ll << pw_depth(n > 0 ? n : 1);
    w.partial = (double *)p; p += al(parts * 8 * 2 + 64);
    w.scal = (unsigned long long *)p; p += al(64);
    w.sorted = nullptr; w.cub_tmp = nullptr; w.cub_bytes = 0;
    if (dtype == CT_F64) {
        w.sorted = (double *)p; p += al(n * 8);
        w.cub_bytes = cub_sort_bytes(n);
        w.cub_tmp = p;
    }
    return w;
}

}  // namespace

size_t ct_mrf_workspace(int64_t nx, int64_t ny, int64_t nz, int dtype) {
    const i64 n = nx * ny * nz;
    const i64 parts = 1ll << pw_depth(n > 0 ? n : 1);
    size_t b = al(parts * 8 * 2 + 64) + al(64);
    if (dtype == CT_F64) b += al(n * 8) + al(cub_sort_bytes(n));
    return b + 1024;
}

__global__ void step_finish(double *out2, const unsigned long long *moved) {
    out2[0] = __dsqrt_rn(out2[0]);
    out2[1] = (double)*moved;
}

extern "C" int ct_mrf(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, void *work, double *state,
                      uint64_t *hist, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("cannot denoise an empty grid");
        return CT_ERR_PARAM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    if (n >= (1ll << 31) && dtype == CT_F64) {
        ct::set_error("float MRF limited to 2^31 voxels");
        return CT_ERR_UNSUPPORTED;
    }
    if (dtype != CT_F64 && !hist) {
        ct::set_error("integer MRF needs a (zeroed) histogram buffer");
        return CT_ERR_PARAM;
    }
    MrfWork w = mrf_carve(work, n, dtype);
    cudaMemsetAsync(state, 0, S_WORDS * sizeof(double), s);
    cudaMemsetAsync(w.scal, 0, 64, s);
    cudaMemsetAsync(&w.scal[1], 0xff, 8, s);
    const i64 mx = nx - 2 > 0 ? nx - 2 : 0, my = ny - 2 > 0 ? ny - 2 : 0, mz = nz - 2 > 0 ? nz - 2 : 0;
    const i64 ni = mx * my * mz;
    CT_DISPATCH(dtype, T, {
        const T *v = (const T *)in;
        mrf_stats<T><<<ct::grid_for(n, 256, CT_NUM_SMS * 4), 256, 0, s>>>(v, nx, ny, nz,
                                                                          dtype == CT_F64 ? nullptr : hist, &w.scal[0]);
        if (int st = ct::check_launch("mrf_stats")) return st;
        if (dtype == CT_F64) {
            size_t tb = w.cub_bytes;
            cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, (const double *)in, w.sorted, (int)n, 0, 64, s);
            delta_from_sorted<<<ct::grid_for(n, 256, CT_NUM_SMS * 4), 256, 0, s>>>(w.sorted, n, &w.scal[1]);
            delta_store<<<1, 1, 0, s>>>(&w.scal[1], state);
        } else {
            delta_from_hist<<<1, 1024, 0, s>>>(hist, state);
        }
        if (int st = ct::check_launch("mrf delta")) return st;
        if (ni >= 2) {
            LapElem<T> f1{v, ny, nz, my, mz, nullptr, 0};
            if (int st = pairwise_sum(f1, ni, w.partial, &state[S_SUM1], s)) return st;
            mean_from_sum<<<1, 1, 0, s>>>(state, ni);
            LapElem<T> f2{v, ny, nz, my, mz, &state[S_SUM1], 1};
            if (int st = pairwise_sum(f2, ni, w.partial, &state[S_SUM2], s)) return st;
        }
        StepElem<T> f3{v, nullptr, nx, ny, nz, &state[S_DELTA]};
        if (int st = pairwise_sum(f3, n, w.partial, &state[S_SUM3], s)) return st;
        mrf_decide<<<1, 1, 0, s>>>(state, ni, &w.scal[0]);
    });
    return ct::check_launch("mrf_decide");
}

extern "C" int ct_mrf_step(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, const double *cur,
                           const double *state, double *next, void *work, double *out2, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const i64 n = nx * ny * nz;
    MrfWork w = mrf_carve(work, n, dtype);
    cudaMemsetAsync(&w.scal[2], 0, 8, s);
    CT_DISPATCH(dtype, T, {
        const T *v = (const T *)in;
        StepElem<T> f{v, cur, nx, ny, nz, &state[S_DELTA]};
        if (int st = pairwise_sum(f, n, w.partial, &out2[0], s)) return st;
        mrf_apply<T><<<ct::grid_for(n, 256), 256, 0, s>>>(v, cur, nx, ny, nz, state + S_DELTA, next, &w.scal[2]);
        if (int st = ct::check_launch("mrf_apply")) return st;
    });
    step_finish<<<1, 1, 0, s>>>(out2, &w.scal[2]);
    return ct::check_launch("mrf_step_finish");
}

namespace {
template <typename T>
__global__ void sign_sum_kernel(const T *__restrict__ v, i64 nx, i64 ny, i64 nz, int64_t *__restrict__ out) {
    const i64 n = nx * ny * nz;
    for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
        out[p] = sign_sum_at<T>(v, nullptr, nx, ny, nz, p);
}
}  // namespace

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
