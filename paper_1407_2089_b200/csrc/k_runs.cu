// k_runs.cu -- z-run-length encoding of every kept cell's voxel list on the
// device (the results on-disk format).
//
// Replaces ref segment.py:321-337 encode_voxel_runs(det.voxels), which
// session._detection_to_dict (session.py:668) calls per detection: runs
// [i, j, k0, length] of consecutive k inside one (i, j) row, in the
// lexicographic (i, j, k) order of the voxels -- the C order ct_cell_table
// already lists them in.  Three kernels: per-cell run counts (warp per cell,
// ballots over the voxel list), an exclusive scan over cells, per-cell run
// emission.
#include "ct_common.cuh"

namespace {

// run breaks: first voxel of the cell, a gap in the linear index, or a new row
__device__ __forceinline__ bool run_break(const int32_t *__restrict__ v, i64 e, int64_t nz) {
    if (e == 0) return true;
    const int32_t p = v[e], q = v[e - 1];
    return p != q + 1 || (p % nz) == 0;
}

__global__ void __launch_bounds__(256) runs_count(const int32_t *__restrict__ voxels, const ct_cell *__restrict__ table,
                                                  const int64_t *__restrict__ counters, int64_t nz,
                                                  int64_t *__restrict__ run_offset) {
    const unsigned lane = threadIdx.x & 31;
    const i64 nk = counters[CT_CNT_KEPT];
    const i64 w0 = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 r = w0; r < nk; r += nw) {
        const int32_t *v = voxels + table[r].voxel_offset;
        const i64 n = table[r].count;
        i64 cnt = 0;
        for (i64 e0 = 0; e0 < n; e0 += 32) {
            const i64 e = e0 + lane;
            cnt += __popc(__ballot_sync(0xffffffffu, e < n && run_break(v, e, nz)));
        }
        if (lane == 0) run_offset[r + 1] = cnt;
    }
}

__global__ void __launch_bounds__(1024) runs_scan(const int64_t *__restrict__ counters, int64_t *run_offset,
                                                  int64_t cap_runs, int64_t *__restrict__ nruns_out) {
    __shared__ long long part[1024];
    const i64 nk = counters[CT_CNT_KEPT];
    const int t = threadIdx.x;
    const i64 chunk = (nk + 1023) / 1024, c0 = min((i64)t * chunk, nk), c1 = min(c0 + chunk, nk);
    long long s = 0;
    for (i64 c = c0; c < c1; ++c) s += run_offset[c + 1];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const long long x = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += x;
        __syncthreads();
    }
    // entry c + 1 (this thread's count of cell c) becomes the inclusive prefix,
    // i.e. the first run of cell c + 1: each entry is read and written by one thread
    long long acc = t ? part[t - 1] : 0;
    for (i64 c = c0; c < c1; ++c) {
        acc += run_offset[c + 1];
        run_offset[c + 1] = acc;
    }
    if (t == 0) {
        run_offset[0] = 0;
        nruns_out[0] = part[1023];
        nruns_out[1] = part[1023] > cap_runs ? 1 : 0;
    }
}

__global__ void __launch_bounds__(256) runs_write(const int32_t *__restrict__ voxels, const ct_cell *__restrict__ table,
                                                  const int64_t *__restrict__ counters, int64_t ny, int64_t nz,
                                                  const int64_t *__restrict__ run_offset, int64_t cap_runs,
                                                  int32_t *__restrict__ runs) {
    const unsigned lane = threadIdx.x & 31;
    const i64 nk = counters[CT_CNT_KEPT];
    if (run_offset[nk] > cap_runs) return;  // overflow reported by runs_scan
    const i64 w0 = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 r = w0; r < nk; r += nw) {
        const int32_t *v = voxels + table[r].voxel_offset;
        const i64 n = table[r].count;
        int32_t *out = runs + 4 * run_offset[r];
        i64 o = 0;
        // starts: [i, j, k0, index of the first voxel]
        for (i64 e0 = 0; e0 < n; e0 += 32) {
            const i64 e = e0 + lane;
            const bool b = e < n && run_break(v, e, nz);
            const unsigned m = __ballot_sync(0xffffffffu, b);
            if (b) {
                const int32_t p = v[e];
                const i64 k = p % nz, row = p / nz;
                int32_t *q = out + 4 * (o + __popc(m & ((1u << lane) - 1)));
                q[0] = (int32_t)(row / ny);
                q[1] = (int32_t)(row % ny);
                q[2] = (int32_t)k;
                q[3] = (int32_t)e;
            }
            o += __popc(m);
        }
        __syncwarp();
        // lengths from consecutive starts
        for (i64 u = lane; u < o; u += 32) {
            const i64 s = out[4 * u + 3], nxt = u + 1 < o ? out[4 * (u + 1) + 3] : n;
            __syncwarp(__activemask());
            out[4 * u + 3] = (int32_t)(nxt - s);
        }
    }
}

}  // namespace

extern "C" int ct_voxel_runs(const int32_t *voxels, const ct_cell *table, const int64_t *counters, int64_t ny,
                             int64_t nz, int64_t cap_runs, int32_t *runs, int64_t *run_offset, int64_t *nruns,
                             void *stream) {
    if (ny <= 0 || nz <= 0 || cap_runs < 0) {
        ct::set_error("ct_voxel_runs: bad sizes");
        return CT_ERR_PARAM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    runs_count<<<CT_NUM_SMS * 4, 256, 0, s>>>(voxels, table, counters, nz, run_offset);
    runs_scan<<<1, 1024, 0, s>>>(counters, run_offset, cap_runs, nruns);
    runs_write<<<CT_NUM_SMS * 4, 256, 0, s>>>(voxels, table, counters, ny, nz, run_offset, cap_runs, runs);
    return ct::check_launch("ct_voxel_runs");
}
