// k_ccl.cu -- K5 26-connected component labelling and K6 the per-cell table.
//
// K5 replaces ref segment.py:254 (ndimage.label(mask, ones((3,3,3)))).  The
// label of a component is its minimum C-order linear index ("root"), which
// is exactly the key the reference orders components by after sizes
// (segment.py:257, v[0] of the C-ordered voxel list).  Union-find always
// links the larger root under the smaller one, so the final root is the
// component minimum regardless of the (non-deterministic) union order.
//   ccl_local   : per 4x8x32 tile, union-find in SMEM over the 13 backward
//                 neighbours inside the tile; writes labels (global index of the
//                 tile-local root) and appends foreground voxels to fg_list.
//   ccl_boundary: for foreground voxels on a tile face, unions with backward
//                 neighbours in other tiles (global atomicMin union-find).
//   ccl_flatten : labels[p] = find(p).
// K6 replaces ref segment.py:242-276 minus the hull (hull stays on the host):
//   tab_roots   : compact the roots (component index c, any order).
//   tab_stats   : per component count / bbox / intensity sum (warp-aggregated
//                 integer atomics: order-independent, deterministic).
//   tab_keep +  : volume filter in float64 (segment.py:253-255); then one warp
//   tab_rank_emit per kept cell: rank by (-count, root) (segment.py:257) = the
//                 number of smaller keys, voxel offset = their count sum, and
//                 the cell's table row (<= 4096 kept cells);
//   tab_rank    : above that, one CTA: stable LSD radix sort, ids, offsets.
//   tab_relabel : labels[p] = rank of p's kept cell or -1.
//   tab_voxels_w: one warp per kept cell walks its bbox in C order, emitting
//                 the ordered voxel list (segment.py:207-217) with ballots;
//                 lane 0 forms the centroid by the row-sequential float64
//                 sum numpy's mean(axis=0) performs (segment.py:260).
#include <algorithm>
#include <cstdlib>

#include "ct_common.cuh"

namespace {

constexpr int LI = 4, LJ = 8, LK = 32;
constexpr int LN = LI * LJ * LK;

// 13 backward neighbours (da, db, dc) of the 26-neighbourhood
__constant__ int8_t BACK[13][3] = {{-1, -1, -1}, {-1, -1, 0}, {-1, -1, 1}, {-1, 0, -1}, {-1, 0, 0},
                                   {-1, 0, 1},   {-1, 1, -1}, {-1, 1, 0},  {-1, 1, 1},  {0, -1, -1},
                                   {0, -1, 0},   {0, -1, 1},  {0, 0, -1}};

__device__ __forceinline__ unsigned lane_id() {
    unsigned l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

__device__ __forceinline__ int find_s(volatile int *L, int x) {
    int y = L[x];
    while (y != x) {
        x = y;
        y = L[x];
    }
    return x;
}

__device__ void union_s(int *L, int a, int b) {
    for (;;) {
        a = find_s(L, a);
        b = find_s(L, b);
        if (a == b) return;
        if (a > b) { const int t = a; a = b; b = t; }
        const int old = atomicMin(&L[b], a);
        if (old == b) return;
        b = old;
    }
}

__device__ __forceinline__ int find_g(volatile int32_t *L, int x) {
    int y = L[x];
    while (y != x) {
        x = y;
        y = L[x];
    }
    return x;
}

// find with path halving (x's parent becomes its grandparent): parents only
// ever move to ancestors, so concurrent unions (atomicMin on roots) stay valid
__device__ __forceinline__ int find_gh(volatile int32_t *L, int x) {
    int y = L[x];
    while (y != x) {
        const int z = L[y];
        if (z != y) L[x] = z;
        x = y;
        y = z;
    }
    return x;
}

__device__ void union_gh(int32_t *L, int a, int b) {
    for (;;) {
        a = find_gh(L, a);
        b = find_gh(L, b);
        if (a == b) return;
        if (a > b) { const int t = a; a = b; b = t; }
        const int old = atomicMin(&L[b], a);
        if (old == b) return;
        b = old;
    }
}

__device__ void union_g(int32_t *L, int a, int b) {
    for (;;) {
        a = find_g(L, a);
        b = find_g(L, b);
        if (a == b) return;
        if (a > b) { const int t = a; a = b; b = t; }
        const int old = atomicMin(&L[b], a);
        if (old == b) return;
        b = old;
    }
}

// warp-aggregated append of p to list (order within the list is irrelevant)
__device__ __forceinline__ void append(int32_t *list, unsigned long long *cnt, int32_t p, bool pred) {
    const unsigned m = __ballot_sync(__activemask(), pred);
    if (!pred) return;
    const unsigned lane = lane_id();
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if ((int)lane == leader) base = atomicAdd(cnt, (unsigned long long)__popc(m));
    base = __shfl_sync(m, base, leader);
    list[base + __popc(m & ((1u << lane) - 1))] = p;
}

__global__ void __launch_bounds__(LK *LJ) ccl_local(const uint8_t *__restrict__ mask, i64 nx, i64 ny, i64 nz,
                                                    int32_t *__restrict__ labels, int32_t *__restrict__ fg,
                                                    int64_t *__restrict__ counters) {
    __shared__ int L[LN];
    const i64 tk = (nz + LK - 1) / LK, tj = (ny + LJ - 1) / LJ, ti = (nx + LI - 1) / LI;
    const i64 ntiles = tk * tj * ti;
    const int c = threadIdx.x, b = threadIdx.y;
    // the next tile's mask bytes are loaded while the current tile is processed
    auto load = [&](i64 tile, uint8_t (&m)[LI]) {
        const i64 k0 = (tile % tk) * LK, j0 = ((tile / tk) % tj) * LJ, i0 = (tile / (tk * tj)) * LI;
        const i64 j = j0 + b, k = k0 + c;
#pragma unroll
        for (int a = 0; a < LI; ++a) {
            const i64 i = i0 + a;
            m[a] = (i < nx && j < ny && k < nz) ? __ldg(mask + (i * ny + j) * nz + k) : 0;
        }
    };
    uint8_t mnext[LI];
    if (blockIdx.x < ntiles) load(blockIdx.x, mnext);
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 k0 = (tile % tk) * LK, j0 = ((tile / tk) % tj) * LJ, i0 = (tile / (tk * tj)) * LI;
        __syncthreads();
        const i64 j = j0 + b, k = k0 + c;
        uint8_t mv[LI];
        bool any = false;
#pragma unroll
        for (int a = 0; a < LI; ++a) {
            mv[a] = mnext[a];
            any |= mv[a] != 0;
        }
        if (tile + gridDim.x < ntiles) load(tile + gridDim.x, mnext);
        // labels were pre-filled with -1: an all-background tile needs no work
        if (!__syncthreads_or(any)) continue;
#pragma unroll
        for (int a = 0; a < LI; ++a) {
            const int v = (a * LJ + b) * LK + c;
            L[v] = mv[a] ? v : -1;
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < LI; ++a) {
            const int v = (a * LJ + b) * LK + c;
            if (L[v] < 0) continue;
            for (int n = 0; n < 13; ++n) {
                const int aa = a + BACK[n][0], bb = b + BACK[n][1], cc = c + BACK[n][2];
                if (aa < 0 || bb < 0 || bb >= LJ || cc < 0 || cc >= LK) continue;
                const int u = (aa * LJ + bb) * LK + cc;
                if (L[u] >= 0) union_s(L, v, u);
            }
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < LI; ++a) {
            const int v = (a * LJ + b) * LK + c;
            if (L[v] >= 0) L[v] = find_s(L, v);
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < LI; ++a) {
            const i64 i = i0 + a;
            const int v = (a * LJ + b) * LK + c;
            const int r = L[v];
            const i64 p = (i * ny + j) * nz + k;
            if (r >= 0) {
                const int ra = r / (LJ * LK), rb = (r / LK) % LJ, rc = r % LK;
                labels[p] = (int32_t)(((i0 + ra) * ny + (j0 + rb)) * nz + (k0 + rc));
            }
            append(fg, (unsigned long long *)&counters[CT_CNT_FG], (int32_t)p, r >= 0);
        }
    }
}

__global__ void ccl_boundary(const uint8_t *__restrict__ mask, i64 nx, i64 ny, i64 nz, int32_t *labels,
                             const int32_t *__restrict__ fg, const int64_t *__restrict__ counters) {
    const i64 nfg = counters[CT_CNT_FG];
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < nfg; e += (i64)gridDim.x * blockDim.x) {
        const i64 p = fg[e];
        const i64 k = p % nz, j = (p / nz) % ny, i = p / (ny * nz);
        for (int n = 0; n < 13; ++n) {
            const i64 a = i + BACK[n][0], b = j + BACK[n][1], c = k + BACK[n][2];
            if (a < 0 || b < 0 || b >= ny || c < 0 || c >= nz) continue;
            if (a / LI == i / LI && b / LJ == j / LJ && c / LK == k / LK) continue;  // same tile
            const i64 q = (a * ny + b) * nz + c;
            if (mask[q]) union_g(labels, (int)p, (int)q);
        }
    }
}

__global__ void ccl_flatten(int32_t *labels, const int32_t *__restrict__ fg, const int64_t *__restrict__ counters) {
    const i64 nfg = counters[CT_CNT_FG];
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < nfg; e += (i64)gridDim.x * blockDim.x) {
        const int p = fg[e];
        labels[p] = find_g(labels, p);
    }
}

// ---------------------------------------------------------------------------
// Run-based labelling for nz <= 128: every z-row is one 64- or 128-bit word (packed on
// the fly from the mask bytes); union-find nodes are the runs of consecutive
// foreground voxels, identified by their first voxel's linear index (so the
// component root -- the minimum node -- is again its minimum voxel).
//   ccl_run_init  : labels[run start] = run start
//   ccl_run_union : each run unions with the runs of the 4 backward rows
//                   (i, j-1), (i-1, j-1..j+1) that touch it in z +- 1, except
//                   links already implied through row (i-1, j) (see the kernel)
//   ccl_run_roots : labels[run start] = find(run start) (compression to the root:
//                   concurrent finds only ever see ancestors)
//   ccl_run_emit  : labels of the run's other voxels = labels[run start]; fg list
// ---------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ R pack_row(const uint8_t *__restrict__ row, int nz) {
    R w = 0;
    if (nz % 16 == 0 && ((uintptr_t)row & 15) == 0) {
        for (int c = 0; c < nz / 16; ++c) {
            const uint4 v = __ldg((const uint4 *)row + c);
            const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t t = (x[q] | ((x[q] & 0x7f7f7f7fu) + 0x7f7f7f7fu)) & 0x80808080u;
                w |= (R)(((t >> 7) * 0x10204080u) >> 28) << (16 * c + 4 * q);
            }
        }
    } else {
        for (int k = 0; k < nz; ++k)
            if (row[k]) w |= (R)1 << k;
    }
    return w;
}

// z-row word r: from pre-packed rows (ct_threshold_close_rows) or packed
// on the fly from the mask bytes
template <typename R, bool BITS>
__device__ __forceinline__ R load_row(const uint8_t *__restrict__ mask, const R *__restrict__ rows, i64 r, int nz) {
    if constexpr (BITS) return rows[r];
    else return pack_row<R>(mask + r * nz, nz);
}

// run of w starting at bit s: mask of its bits
template <typename R>
__device__ __forceinline__ R run_mask(R w, int s) {
    const R above = ~(w >> s);  // first zero at or above s
    const int len = above ? ct::rffs(above) - 1 : ct::rbits<R>() - s;
    return ct::rmask<R>(len) << s;
}

template <typename R, bool BITS>
__global__ void ccl_run_init(const uint8_t *__restrict__ mask, const R *__restrict__ rows, i64 nrows, int nz,
                             int32_t *__restrict__ labels) {
    for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < nrows; r += (i64)gridDim.x * blockDim.x) {
        R st = load_row<R, BITS>(mask, rows, r, nz);
        st &= ~(st << 1);  // run starts
        while (st) {
            const int s = ct::rffs(st) - 1;
            st &= st - 1;
            labels[r * nz + s] = (int32_t)(r * nz + s);
        }
    }
}

// A run s unions with every run of row (i-1, j) it touches (F); a run of
// rows (i, j-1), (i-1, j-1), (i-1, j+1) that touches s is skipped when it also
// touches F: that link is implied -- s-F is made here, and the F-run link is
// owned by an earlier row ((i, j-1) against its (i-1, j); (i-1, j) against its
// (i-1, j-1); (i-1, j+1) against its (i-1, j)), itself made or implied by
// induction over the row order.  Same components, same roots (minimum index),
// fewer atomic unions on compact cells.
template <typename R, bool BITS>
__global__ void ccl_run_union(const uint8_t *__restrict__ mask, const R *__restrict__ rows, i64 nx, i64 ny, int nz,
                              int32_t *labels, const ct::FastDiv fny) {
    const i64 nrows = nx * ny;  // rows < 2^31 (labels are int32 voxel indices); fny built on the host
    for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < nrows; r += (i64)gridDim.x * blockDim.x) {
        const R w = load_row<R, BITS>(mask, rows, r, nz);
        if (!w) continue;
        const i64 i = fny.div((uint32_t)r), j = r - i * ny;
        // q = 0: (i-1, j) first (it defines F), then (i, j-1), (i-1, j-1), (i-1, j+1)
        const i64 nb[4] = {i > 0 ? r - ny : -1, j > 0 ? r - 1 : -1, (i > 0 && j > 0) ? r - ny - 1 : -1,
                           (i > 0 && j + 1 < ny) ? r - ny + 1 : -1};
        R u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = nb[q] >= 0 ? load_row<R, BITS>(mask, rows, nb[q], nz) : (R)0;
        R rem = w;
        while (rem) {
            const int s = ct::rffs(rem) - 1;
            const R mr = run_mask(w, s);
            rem &= ~mr;
            const R ds = mr | (mr << 1) | (mr >> 1);
            R dF = 0;  // F dilated by one along z
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!u[q]) continue;
                const R ustart = u[q] & ~(u[q] << 1);
                R o = ds & u[q];  // 26-neighbours in row nb[q]
                while (o) {
                    const int b = ct::rffs(o) - 1;
                    const R below = ustart & ct::rmask<R>(b + 1);
                    const int su = ct::rbits<R>() - 1 - ct::rclz(below);
                    const R um = run_mask(u[q], su);
                    o &= ~um;
                    if (q == 0) dF |= um | (um << 1) | (um >> 1);
                    else if (dF & um) continue;
                    union_gh(labels, (int)(r * nz + s), (int)(nb[q] * nz + su));
                }
            }
        }
    }
}

template <typename R, bool BITS>
__global__ void ccl_run_emit(const uint8_t *__restrict__ mask, const R *__restrict__ rows, i64 nrows, int nz,
                             int32_t *labels, int32_t *__restrict__ fg, int64_t *__restrict__ counters) {
    // the loop runs whole warps (trip count uniform per warp) so the fg-list
    // slots are claimed with one atomic per warp: a per-row atomic on the one
    // counter serialised ~10^5 non-empty rows
    const i64 stride = (i64)gridDim.x * blockDim.x;
    const unsigned lane = threadIdx.x & 31;
    for (i64 r0 = blockIdx.x * (i64)blockDim.x + (threadIdx.x & ~31u); r0 < nrows; r0 += stride) {
        const i64 r = r0 + lane;
        const R w = r < nrows ? load_row<R, BITS>(mask, rows, r, nz) : (R)0;
        const int n = ct::rpopc(w);
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += v;
        }
        unsigned long long wbase = 0;
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 31 && tot) wbase = atomicAdd((unsigned long long *)&counters[CT_CNT_FG], (unsigned long long)tot);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        if (!w) continue;
        const unsigned long long base = wbase + (unsigned long long)(incl - n);
        R rem = w;
        int e = 0;
        while (rem) {
            const int s = ct::rffs(rem) - 1;
            const R mr = run_mask(w, s);
            rem &= ~mr;
            const int32_t root = labels[r * nz + s];  // ccl_run_roots ran first: the start holds its root
            for (R m = mr; m; m &= m - 1) {
                CT_DCHECK(base + e < nrows * (i64)nz);
                fg[base + e++] = (int32_t)(r * nz + ct::rffs(m) - 1);
            }
            for (R m = mr & (mr - 1); m; m &= m - 1) labels[r * nz + ct::rffs(m) - 1] = root;
        }
    }
}

// run starts take their root (before ccl_run_emit, which copies it to the run)
template <typename R, bool BITS>
__global__ void ccl_run_roots(const uint8_t *__restrict__ mask, const R *__restrict__ rows, i64 nrows, int nz,
                              int32_t *labels) {
    for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < nrows; r += (i64)gridDim.x * blockDim.x) {
        R st = load_row<R, BITS>(mask, rows, r, nz);
        st &= ~(st << 1);
        while (st) {
            const int s = ct::rffs(st) - 1;
            st &= st - 1;
            labels[r * nz + s] = find_g(labels, (int)(r * nz + s));  // path compression to the root
        }
    }
}

// ---------------------------------------------------------------------------
// K6 -- table
// ---------------------------------------------------------------------------
struct TabWork {
    int32_t *root;      // [cap]
    uint32_t *count;    // [cap]
    int32_t *bbox;      // [cap][6] lo i,j,k then hi i,j,k
    uint64_t *isum;     // [cap]
    int32_t *rank;      // [cap]
    int32_t *sa, *sb;   // [cap] sort ping-pong (component indices)
    int32_t *comp;      // [N]   component index of fg_list[e]
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline size_t tab_bytes(i64 N, i64 cap) {
    return align_up(cap * 4) * 6 + align_up(cap * 24) + align_up(cap * 8) + align_up(N * 4);
}

__host__ TabWork tab_carve(void *work, i64 N, i64 cap) {
    char *p = (char *)work;
    TabWork w;
    w.root = (int32_t *)p; p += align_up(cap * 4);
    w.count = (uint32_t *)p; p += align_up(cap * 4);
    w.bbox = (int32_t *)p; p += align_up(cap * 24);
    w.isum = (uint64_t *)p; p += align_up(cap * 8);
    w.rank = (int32_t *)p; p += align_up(cap * 4);
    w.sa = (int32_t *)p; p += align_up(cap * 4);
    w.sb = (int32_t *)p; p += align_up(cap * 4);
    w.comp = (int32_t *)p; p += align_up(N * 4);
    return w;
}

__global__ void tab_roots(int32_t *labels, const int32_t *__restrict__ fg, int64_t *counters, TabWork w, i64 cap) {
    const i64 nfg = counters[CT_CNT_FG];
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < nfg; e += (i64)gridDim.x * blockDim.x) {
        const int p = fg[e];
        if (labels[p] != p) continue;
        const unsigned long long c = atomicAdd((unsigned long long *)&counters[CT_CNT_COMPONENTS], 1ull);
        if ((i64)c < cap) {
            w.root[c] = p;
            w.count[c] = 0;
            w.isum[c] = 0;
            w.bbox[6 * c + 0] = w.bbox[6 * c + 1] = w.bbox[6 * c + 2] = INT32_MAX;
            w.bbox[6 * c + 3] = w.bbox[6 * c + 4] = w.bbox[6 * c + 5] = -1;
            labels[p] = -(int32_t)(c + 2);
        } else {
            counters[CT_CNT_OVERFLOW] = 1;
        }
    }
}

template <typename TI>
__global__ void tab_stats(const int32_t *__restrict__ labels, i64 ny, i64 nz, const int32_t *__restrict__ fg,
                          const int64_t *__restrict__ counters, TabWork w, const TI *__restrict__ intensity,
                          const ct::FastDiv fnz, const ct::FastDiv fny) {
    const i64 nfg = counters[CT_CNT_FG];
    const bool over = counters[CT_CNT_OVERFLOW] != 0;
    // fnz, fny: built on the host (voxel indices are int32, N < 2^31)
    for (i64 e0 = blockIdx.x * (i64)blockDim.x; e0 < nfg; e0 += (i64)gridDim.x * blockDim.x) {
        const i64 e = e0 + threadIdx.x;
        int c = -1;
        int p = 0;
        if (e < nfg && !over) {
            p = fg[e];
            const int v = labels[p];
            const int rv = v < 0 ? v : labels[v];
            c = -(rv + 2);
            w.comp[e] = c;
        }
        const bool act = c >= 0;
        const unsigned full = __ballot_sync(0xffffffffu, act);
        if (!act) continue;
        const unsigned peers = __match_any_sync(full, c);
        const int leader = __ffs(peers) - 1;
        const uint32_t pz = fnz.div((uint32_t)p), pi = fny.div(pz);
        const int k = p - (int)(pz * (uint32_t)nz), j = (int)(pz - pi * (uint32_t)ny), i = (int)pi;
        const int imin = __reduce_min_sync(peers, i), jmin = __reduce_min_sync(peers, j),
                  kmin = __reduce_min_sync(peers, k);
        const int imax = __reduce_max_sync(peers, i), jmax = __reduce_max_sync(peers, j),
                  kmax = __reduce_max_sync(peers, k);
        unsigned isum = 0;
        if (intensity) isum = __reduce_add_sync(peers, (unsigned)intensity[p]);
        if ((int)lane_id() == leader) {
            atomicAdd(&w.count[c], (unsigned)__popc(peers));
            atomicMin(&w.bbox[6 * c + 0], imin);
            atomicMin(&w.bbox[6 * c + 1], jmin);
            atomicMin(&w.bbox[6 * c + 2], kmin);
            atomicMax(&w.bbox[6 * c + 3], imax);
            atomicMax(&w.bbox[6 * c + 4], jmax);
            atomicMax(&w.bbox[6 * c + 5], kmax);
            if (intensity) atomicAdd((unsigned long long *)&w.isum[c], (unsigned long long)isum);
        }
    }
}

// per-cell mean intensity: the numpy mean of the cell's integer intensities
// (raw[voxels].mean(): the float64 sum of integers < 2^53 is exact in any
// order, so the mean is one correctly rounded division); NaN without intensity
__device__ __forceinline__ double mean_intensity(u64 isum, u64 count, bool has_int) {
    return has_int ? __ddiv_rn((double)isum, (double)count) : __longlong_as_double(0x7ff8000000000000ll);
}

constexpr int RT = 512;    // tab_rank threads
constexpr int RK = 4096;   // kept cells ordered by the multi-CTA path (tab_keep / tab_rank_emit)
constexpr int RD = 16;     // radix digits (4 bits)

__device__ __forceinline__ u64 sort_key(const TabWork &w, int c, u64 maxc, int rbits) {
    return ((maxc - (u64)w.count[c]) << rbits) | (u64)(uint32_t)w.root[c];
}

// Block-wide exclusive scan of one value per thread; returns the total.
// sh must hold blockDim.x/32 + 1 entries.
__device__ u64 block_excl_scan(u64 &v, u64 *sh) {
    const unsigned lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    u64 x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if ((int)lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 acc = 0;
        for (unsigned i = 0; i < nw; ++i) { const u64 t = sh[i]; sh[i] = acc; acc += t; }
        sh[nw] = acc;
    }
    __syncthreads();
    const u64 res = sh[wid] + x - v;
    const u64 total = sh[nw];
    __syncthreads();
    v = res;
    return total;
}

__global__ void __launch_bounds__(RT) tab_rank(int64_t *counters, TabWork w, i64 cap, i64 N, double vv, bool has_int,
                                               double min_volume, i64 id_start, ct_cell *table) {
    __shared__ uint32_t hcnt[RD][RT];
    __shared__ u64 sh[RT / 32 + 1];
    __shared__ u64 s_maxc;
    const int tid = threadIdx.x;
    if (counters[CT_CNT_KEPT] <= RK) return;  // ordered by tab_rank_emit
    i64 nc = counters[CT_CNT_COMPONENTS];
    if (nc > cap) nc = cap;
    if (counters[CT_CNT_OVERFLOW]) nc = 0;
    // 1. kept components, compacted in component order; max count
    const i64 chunk = (nc + RT - 1) / RT;
    const i64 c0 = min((i64)tid * chunk, nc), c1 = min(c0 + chunk, nc);
    u64 kept = 0, maxc = 0;
    for (i64 c = c0; c < c1; ++c) {
        w.rank[c] = -1;
        const double vol = __dmul_rn((double)w.count[c], vv);
        if (!(vol < min_volume)) { ++kept; maxc = max(maxc, (u64)w.count[c]); }
    }
    for (int o = 16; o; o >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
    if (tid == 0) s_maxc = 0;
    __syncthreads();
    if ((tid & 31) == 0) atomicMax((unsigned long long *)&s_maxc, (unsigned long long)maxc);
    u64 off = kept;
    const u64 nk = block_excl_scan(off, sh);
    for (i64 c = c0; c < c1; ++c) {
        const double vol = __dmul_rn((double)w.count[c], vv);
        if (!(vol < min_volume)) w.sa[off++] = (int32_t)c;
    }
    __syncthreads();
    const u64 mc = s_maxc;
    int cbits = 0;
    while (cbits < 40 && (mc >> cbits)) ++cbits;
    int rbits = 1;
    while ((((u64)N - 1) >> rbits) && rbits < 40) ++rbits;
    const int passes = (cbits + rbits + 3) / 4;
    // 2. order sa[0..nk) by key (keys are unique: roots differ).  Few cells:
    //    rank by counting against all keys staged in SMEM (O(nk^2), no passes);
    //    many: stable LSD radix sort, 4-bit digits.
    int32_t *src = w.sa, *dst = w.sb;
    const i64 kchunk = ((i64)nk + RT - 1) / RT;
    const i64 e0 = min((i64)tid * kchunk, (i64)nk), e1 = min(e0 + kchunk, (i64)nk);
    __threadfence_block();
    __syncthreads();
    u64 *skey = reinterpret_cast<u64 *>(&hcnt[0][0]);  // RD*RT*4 bytes = 4096 keys
    if (nk <= (u64)(RD * RT / 2)) {
        for (i64 e = tid; e < (i64)nk; e += RT) skey[e] = sort_key(w, src[e], mc, rbits);
        __syncthreads();
        for (i64 e = tid; e < (i64)nk; e += RT) {
            const u64 k = skey[e];
            i64 r = 0;
            for (i64 f = 0; f < (i64)nk; ++f) r += skey[f] < k;
            dst[r] = src[e];
        }
        __threadfence_block();
        __syncthreads();
        int32_t *t = src; src = dst; dst = t;
    } else {
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = 4 * pass;
        uint32_t cnt[RD];
#pragma unroll
        for (int d = 0; d < RD; ++d) cnt[d] = 0;
        for (i64 e = e0; e < e1; ++e) {
            const int d = (int)((sort_key(w, src[e], mc, rbits) >> shift) & 15);
#pragma unroll
            for (int dd = 0; dd < RD; ++dd) cnt[dd] += (d == dd);
        }
#pragma unroll
        for (int d = 0; d < RD; ++d) hcnt[d][tid] = cnt[d];
        __syncthreads();
        // exclusive scan over (digit-major, thread-minor)
        u64 run = 0;
        for (int d = 0; d < RD; ++d) {
            u64 v = hcnt[d][tid];
            const u64 tot = block_excl_scan(v, sh);
            hcnt[d][tid] = (uint32_t)(run + v);
            run += tot;
        }
        __syncthreads();
        uint32_t pos[RD];
#pragma unroll
        for (int d = 0; d < RD; ++d) pos[d] = hcnt[d][tid];
        for (i64 e = e0; e < e1; ++e) {
            const int c = src[e];
            const int d = (int)((sort_key(w, c, mc, rbits) >> shift) & 15);
            uint32_t at = 0;
#pragma unroll
            for (int dd = 0; dd < RD; ++dd)
                if (d == dd) at = pos[dd]++;
            dst[at] = c;
        }
        __threadfence_block();
        __syncthreads();
        int32_t *t = src; src = dst; dst = t;
    }
    }
    // 3. ranks, ids, offsets
    u64 vox = 0;
    for (i64 e = e0; e < e1; ++e) vox += w.count[src[e]];
    u64 voff = vox;
    const u64 total_vox = block_excl_scan(voff, sh);
    for (i64 e = e0; e < e1; ++e) {
        const int c = src[e];
        w.rank[c] = (int32_t)e;
        ct_cell r;
        r.id = id_start + e;
        r.count = w.count[c];
        r.root = w.root[c];
        for (int a = 0; a < 3; ++a) {
            r.bbox_lo[a] = w.bbox[6 * c + a];
            r.bbox_hi[a] = w.bbox[6 * c + 3 + a];
        }
        r.intensity_sum = (int64_t)w.isum[c];
        r.centroid_um[0] = r.centroid_um[1] = r.centroid_um[2] = 0.0;
        r.volume_um3 = __dmul_rn((double)r.count, vv);
        r.voxel_offset = (int64_t)voff;
        r.mean_intensity = mean_intensity(w.isum[c], w.count[c], has_int);
        table[e] = r;
        voff += w.count[c];
    }
    if (tid == 0) {
        counters[CT_CNT_KEPT] = (int64_t)nk;
        counters[CT_CNT_KEPT_VOXELS] = (int64_t)total_vox;
    }
}

// Multi-CTA ordering for up to RK kept cells (the usual case); tab_rank
// (single CTA, radix sort) takes over above that.

__device__ __forceinline__ u64 order_key(const TabWork &w, int c) {  // (-count, root) ascending
    return ((u64)(0x7fffffffu - w.count[c]) << 32) | (u64)(uint32_t)w.root[c];
}

// kept components (volume filter in float64, segment.py:253-255), any order
__global__ void tab_keep(int64_t *counters, TabWork w, i64 cap, double vv, double min_volume) {
    i64 nc = counters[CT_CNT_COMPONENTS];
    if (nc > cap) nc = cap;
    if (counters[CT_CNT_OVERFLOW]) nc = 0;
    for (i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x; c < nc; c += (i64)gridDim.x * blockDim.x) {
        w.rank[c] = -1;
        const double vol = __dmul_rn((double)w.count[c], vv);
        const bool keep = !(vol < min_volume);
        const unsigned m = __ballot_sync(__activemask(), keep);
        if (!keep) continue;
        const unsigned lane = lane_id();
        const int leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if ((int)lane == leader) base = atomicAdd((unsigned long long *)&counters[CT_CNT_KEPT], (u64)__popc(m));
        base = __shfl_sync(m, base, leader);
        w.sa[base + __popc(m & ((1u << lane) - 1))] = (int32_t)c;
    }
}

// Rank + voxel offset + table row in one pass, one warp per kept cell (all
// SMs; replaces tab_rank_keys + the single-CTA tab_emit, which was bound by
// one SM's memory pipe): rank = #{keys < k}, voxel offset = sum of the counts
// of those keys (= the exclusive scan in rank order), lanes split the key
// range; the 128-byte row is written by 16 lanes, one field each.
__global__ void __launch_bounds__(256) tab_rank_emit(int64_t *counters, TabWork w, double vv, i64 id_start,
                                                     bool has_int, ct_cell *table) {
    __shared__ u64 key[RK];
    __shared__ uint32_t cnt[RK];
    const i64 nk = counters[CT_CNT_KEPT];
    if (nk > RK || (i64)blockIdx.x * 8 >= nk) return;
    for (i64 e = threadIdx.x; e < nk; e += 256) {
        const int c = w.sa[e];
        key[e] = order_key(w, c);
        cnt[e] = w.count[c];
    }
    __syncthreads();
    const unsigned lane = threadIdx.x & 31;
    const i64 e = (i64)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (e >= nk) return;
    const u64 k = key[e];
    unsigned r = 0;
    u64 v = 0;
    for (int f = (int)lane; f < (int)nk; f += 32) {
        const bool lt = key[f] < k;
        r += lt;
        v += lt ? cnt[f] : 0u;
    }
    for (int o = 16; o; o >>= 1) {
        r += __shfl_xor_sync(0xffffffffu, r, o);
        v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    const int c = w.sa[e];
    if (lane == 0) {
        w.rank[c] = (int32_t)r;
        w.sb[r] = c;
        if ((i64)r == nk - 1) counters[CT_CNT_KEPT_VOXELS] = (int64_t)(v + cnt[e]);
    }
    if (lane < 16) {
        int64_t f;
        switch (lane) {
            case 0: f = id_start + (i64)r; break;
            case 1: f = (int64_t)cnt[e]; break;
            case 2: f = w.root[c]; break;
            case 3: case 4: case 5: case 6: case 7: case 8: f = w.bbox[6 * c + (lane - 3)]; break;
            case 9: f = (int64_t)w.isum[c]; break;
            case 13: f = __double_as_longlong(__dmul_rn((double)cnt[e], vv)); break;
            case 14: f = (int64_t)v; break;
            case 15: f = __double_as_longlong(mean_intensity(w.isum[c], cnt[e], has_int)); break;
            default: f = 0; break;  // centroid (tab_voxels_w)
        }
        reinterpret_cast<int64_t *>(table + r)[lane] = f;
    }
}

__global__ void tab_relabel(int32_t *labels, const int32_t *__restrict__ fg, const int64_t *__restrict__ counters,
                            TabWork w) {
    const i64 nfg = counters[CT_CNT_FG];
    const bool over = counters[CT_CNT_OVERFLOW] != 0;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < nfg; e += (i64)gridDim.x * blockDim.x) {
        CT_DCHECK(over || (w.comp[e] >= 0 && w.comp[e] < counters[CT_CNT_COMPONENTS]));
        labels[fg[e]] = over ? -1 : w.rank[w.comp[e]];
    }
}

// One warp per kept cell: bbox scan in C order with ballots (no block
// barriers); the centroid is the row-sequential float64 sum of numpy's
// mean(axis=0), accumulated by lane 0 in list order via shuffles.
constexpr int TVB = 8;  // chunks of 32 candidates per round; the next round's labels are in flight
__global__ void __launch_bounds__(256) tab_voxels_w(const int32_t *__restrict__ labels, i64 ny, i64 nz,
                                                    const int64_t *__restrict__ counters, ct_cell *table,
                                                    int32_t *__restrict__ voxels, double dx, double dy, double dz) {
    __shared__ double csm[8][32 * 3];
    const unsigned lane = threadIdx.x & 31;
    double *cs = csm[threadIdx.x >> 5];
    const i64 nk = counters[CT_CNT_KEPT];
    const i64 w0 = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((i64)gridDim.x * blockDim.x) >> 5;
    const ct::FastDiv fyz((uint32_t)(ny * nz)), fz((uint32_t)nz);  // voxel index -> (i, j, k); N < 2^31
    for (i64 r = w0; r < nk; r += nw) {
        const int lo0 = table[r].bbox_lo[0], lo1 = table[r].bbox_lo[1], lo2 = table[r].bbox_lo[2];
        const unsigned bi = table[r].bbox_hi[0] - lo0 + 1, bj = table[r].bbox_hi[1] - lo1 + 1,
                       bk = table[r].bbox_hi[2] - lo2 + 1;
        const i64 off = table[r].voxel_offset;
        const unsigned nbox = bi * bj * bk;  // < 2^31 (volumes < 2^31 voxels)
        const unsigned bjk = bj * bk;
        const ct::FastDiv fjk(bjk), fk(bk);
        i64 written = 0;
        double sx = 0.0, sy = 0.0, sz = 0.0;
        // candidate q -> linear index (32-bit index math; q < nbox)
        auto lin = [&](unsigned q) -> int32_t {
            const unsigned a = fjk.div(q), rem = q - a * bjk, b = fk.div(rem), c = rem - b * bk;
            return (int32_t)(((i64)(lo0 + (int)a) * ny + (lo1 + (int)b)) * nz + (lo2 + (int)c));
        };
        int32_t pn[TVB], ln[TVB];  // next round: linear indices and labels in flight
        auto fetch = [&](unsigned q0, int32_t (&pv)[TVB], int32_t (&lv)[TVB]) {
#pragma unroll
            for (int u = 0; u < TVB; ++u) {
                const unsigned q = q0 + 32 * u + lane;
                pv[u] = 0;
                lv[u] = -2;
                if (q < nbox) {
                    pv[u] = lin(q);
                    lv[u] = __ldg(labels + pv[u]);
                }
            }
        };
        fetch(0, pn, ln);
        for (unsigned q00 = 0; q00 < nbox; q00 += 32 * TVB) {
            int32_t pv[TVB], lv[TVB];
#pragma unroll
            for (int u = 0; u < TVB; ++u) { pv[u] = pn[u]; lv[u] = ln[u]; }
            if (q00 + 32 * TVB < nbox) fetch(q00 + 32 * TVB, pn, ln);
#pragma unroll
            for (int u = 0; u < TVB; ++u) {
                const bool hit = lv[u] == (int32_t)r;
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                CT_DCHECK(!hit || written + __popc(m) <= table[r].count);  // a cell's list never outgrows its count
                if (hit) voxels[off + written + __popc(m & ((1u << lane) - 1))] = pv[u];
                written += __popc(m);
            }
        }
        // centroid: the row-sequential float64 sum numpy's mean(axis=0) performs,
        // over the list just written (C order), 32 voxels per step: the lanes form
        // the coordinates, lane 0 runs the three addition chains from SMEM (the
        // chains inside the walk, per 32 candidates with two warp barriers,
        // were ~half of this kernel's instructions and stalls)
        __syncwarp();  // the warp's list writes are visible to its lanes
        for (i64 c0 = 0; c0 < written; c0 += 32) {
            const i64 e = c0 + lane;
            if (e < written) {
                const uint32_t p = (uint32_t)voxels[off + e];
                const uint32_t a = fyz.div(p), rem = p - a * (uint32_t)(ny * nz);
                const uint32_t b = fz.div(rem), c = rem - b * (uint32_t)nz;
                cs[3 * lane] = __dmul_rn((double)a, dx);
                cs[3 * lane + 1] = __dmul_rn((double)b, dy);
                cs[3 * lane + 2] = __dmul_rn((double)c, dz);
            }
            __syncwarp();
            if (lane == 0) {
                const int n = (int)min((i64)32, written - c0);
                if (n == 32) {
#pragma unroll
                    for (int h = 0; h < 32; ++h) {
                        sx = __dadd_rn(sx, cs[3 * h]);
                        sy = __dadd_rn(sy, cs[3 * h + 1]);
                        sz = __dadd_rn(sz, cs[3 * h + 2]);
                    }
                } else {
                    for (int h = 0; h < n; ++h) {
                        sx = __dadd_rn(sx, cs[3 * h]);
                        sy = __dadd_rn(sy, cs[3 * h + 1]);
                        sz = __dadd_rn(sz, cs[3 * h + 2]);
                    }
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            const double n = (double)table[r].count;
            table[r].centroid_um[0] = __ddiv_rn(sx, n);
            table[r].centroid_um[1] = __ddiv_rn(sy, n);
            table[r].centroid_um[2] = __ddiv_rn(sz, n);
        }
    }
}

}  // namespace

size_t ct_table_workspace(int64_t N, int64_t cap) { return tab_bytes(N, cap); }

extern "C" int ct_ccl26(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, int32_t *labels, int32_t *fg_list,
                        int64_t *counters, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("empty mask");
        return CT_ERR_PARAM;
    }
    if (nx * ny * nz >= (1ll << 31)) {
        ct::set_error("volume of %lld voxels exceeds int32 labels", (long long)(nx * ny * nz));
        return CT_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(counters, 0, CT_CNT_WORDS * sizeof(int64_t), s);
    cudaMemsetAsync(labels, 0xff, (size_t)(nx * ny * nz) * sizeof(int32_t), s);  // background = -1
    if (nz <= 128) {  // run-based union-find on z-rows; the tile form covers nz > 128
        const i64 nrows = nx * ny;
        const int g = (int)min((nrows + 255) / 256, (i64)CT_NUM_SMS * 16);
        auto run = [&](auto tag) -> int {
            using R = decltype(tag);
            ccl_run_init<R, false><<<g, 256, 0, s>>>(mask, nullptr, nrows, (int)nz, labels);
            ccl_run_union<R, false><<<g, 256, 0, s>>>(mask, nullptr, nx, ny, (int)nz, labels,
                                                      ct::FastDiv((uint32_t)ny));
            ccl_run_roots<R, false><<<g, 256, 0, s>>>(mask, nullptr, nrows, (int)nz, labels);
            ccl_run_emit<R, false><<<g, 256, 0, s>>>(mask, nullptr, nrows, (int)nz, labels, fg_list, counters);
            return ct::check_launch("ccl_run");
        };
        return nz <= 64 ? run((unsigned long long)0) : run((ct::u128)0);
    }
    const i64 tiles = ((nz + LK - 1) / LK) * ((ny + LJ - 1) / LJ) * ((nx + LI - 1) / LI);
    ccl_local<<<(int)min(tiles, (i64)CT_NUM_SMS * 8), dim3(LK, LJ), 0, s>>>(mask, nx, ny, nz, labels, fg_list,
                                                                            counters);
    if (int st = ct::check_launch("ccl_local")) return st;
    ccl_boundary<<<CT_NUM_SMS * 4, 256, 0, s>>>(mask, nx, ny, nz, labels, fg_list, counters);
    if (int st = ct::check_launch("ccl_boundary")) return st;
    ccl_flatten<<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, fg_list, counters);
    return ct::check_launch("ccl_flatten");
}

// CT_LABELS_RESET: the previous frame's foreground (its fg list, count in
// counters[CT_CNT_FG]) goes back to -1 -- the only voxels ccl / cell table
// wrote -- before the counters are cleared
__global__ void __launch_bounds__(256) ccl_reset_prev(int32_t *__restrict__ labels,
                                                      const int32_t *__restrict__ fg_list,
                                                      const int64_t *__restrict__ counters) {
    const i64 n = counters[CT_CNT_FG];
    for (i64 e = blockIdx.x * 256ll + threadIdx.x; e < n; e += (i64)gridDim.x * 256) {
        CT_DCHECK(fg_list[e] >= 0);
        labels[fg_list[e]] = -1;
    }
}

extern "C" int ct_ccl26_rows(const void *rows, int64_t nx, int64_t ny, int64_t nz, int32_t *labels,
                             int32_t *fg_list, int64_t *counters, int flags, void *stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0) {
        ct::set_error("empty mask");
        return CT_ERR_PARAM;
    }
    if (nx * ny * nz >= (1ll << 31) || nz > 128) {
        ct::set_error("ct_ccl26_rows: needs nz <= 128 and < 2^31 voxels");
        return CT_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (flags & CT_LABELS_RESET) {
        ccl_reset_prev<<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, fg_list, counters);
        if (int st = ct::check_launch("ccl_reset_prev")) return st;
    }
    cudaMemsetAsync(counters, 0, CT_CNT_WORDS * sizeof(int64_t), s);
    if (!(flags & (CT_LABELS_PREFILLED | CT_LABELS_RESET)))  // else labels hold -1 already / after the reset
        cudaMemsetAsync(labels, 0xff, (size_t)(nx * ny * nz) * sizeof(int32_t), s);  // background = -1
    const i64 nrows = nx * ny;
    const int g = (int)min((nrows + 255) / 256, (i64)CT_NUM_SMS * 16);
    auto run = [&](auto tag) -> int {
        using R = decltype(tag);
        const R *rw = (const R *)rows;
        ccl_run_init<R, true><<<g, 256, 0, s>>>(nullptr, rw, nrows, (int)nz, labels);
        ccl_run_union<R, true><<<g, 256, 0, s>>>(nullptr, rw, nx, ny, (int)nz, labels,
                                                 ct::FastDiv((uint32_t)ny));
        ccl_run_roots<R, true><<<g, 256, 0, s>>>(nullptr, rw, nrows, (int)nz, labels);
        ccl_run_emit<R, true><<<g, 256, 0, s>>>(nullptr, rw, nrows, (int)nz, labels, fg_list, counters);
        return ct::check_launch("ccl_run_rows");
    };
    return nz <= 64 ? run((unsigned long long)0) : run((ct::u128)0);
}

extern "C" int ct_cell_table(int32_t *labels, int64_t nx, int64_t ny, int64_t nz, const int32_t *fg_list,
                             int64_t *counters, const void *intensity, int intensity_dtype, double dx, double dy,
                             double dz, double min_volume_um3, int64_t id_start, int64_t cap, void *work,
                             ct_cell *table, int32_t *voxels, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const i64 N = nx * ny * nz;
    if (cap <= 0 || !work) {
        ct::set_error("cell table needs a workspace with positive capacity");
        return CT_ERR_PARAM;
    }
    TabWork w = tab_carve(work, N, cap);
    const double vv = (dx * dy) * dz;  // VoxelSpacing.voxel_volume_um3 (imaging.py:41-43)
    tab_roots<<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, fg_list, counters, w, cap);
    if (int st = ct::check_launch("tab_roots")) return st;
    const ct::FastDiv fnz((uint32_t)nz), fny((uint32_t)ny);  // built once here, not per thread
    if (!intensity) {
        tab_stats<uint8_t><<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, ny, nz, fg_list, counters, w, nullptr, fnz, fny);
    } else if (intensity_dtype == CT_U8) {
        tab_stats<uint8_t><<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, ny, nz, fg_list, counters, w,
                                                          (const uint8_t *)intensity, fnz, fny);
    } else if (intensity_dtype == CT_U16) {
        tab_stats<uint16_t><<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, ny, nz, fg_list, counters, w,
                                                           (const uint16_t *)intensity, fnz, fny);
    } else {
        ct::set_error("intensity must be U8 or U16");
        return CT_ERR_UNSUPPORTED;
    }
    if (int st = ct::check_launch("tab_stats")) return st;
    cudaMemsetAsync(&counters[CT_CNT_KEPT], 0, sizeof(int64_t), s);
    tab_keep<<<CT_NUM_SMS * 2, 256, 0, s>>>(counters, w, cap, vv, min_volume_um3);
    const bool has_int = intensity != nullptr;
    tab_rank_emit<<<(unsigned)((std::min<i64>(cap, RK) + 7) / 8), 256, 0, s>>>(counters, w, vv, id_start, has_int,
                                                                              table);
    tab_rank<<<1, RT, 0, s>>>(counters, w, cap, N, vv, has_int, min_volume_um3, id_start, table);
    if (int st = ct::check_launch("tab_rank")) return st;
    tab_relabel<<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, fg_list, counters, w);
    if (int st = ct::check_launch("tab_relabel")) return st;
    tab_voxels_w<<<CT_NUM_SMS * 4, 256, 0, s>>>(labels, ny, nz, counters, table, voxels, dx, dy, dz);
    return ct::check_launch("tab_voxels");
}
