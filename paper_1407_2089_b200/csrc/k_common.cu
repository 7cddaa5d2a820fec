// k_common.cu -- error reporting, version and workspace sizing for libct.
#include <stdarg.h>
#include <string.h>

#include "ct_common.cuh"

size_t ct_table_workspace(int64_t N, int64_t cap);
size_t ct_edt_workspace(int64_t nx, int64_t ny, int64_t nz);
size_t ct_mrf_workspace(int64_t nx, int64_t ny, int64_t nz, int dtype);

namespace ct {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return CT_ERR_CUDA;
    }
    return CT_OK;
}

}  // namespace ct

extern "C" const char *ct_version(void) { return "libct 0.1 sm_100a"; }

extern "C" const char *ct_last_error(void) { return ct::g_err; }

extern "C" int ct_memset(void *dst, int value, int64_t bytes, void *stream) {
    if (bytes < 0 || (bytes > 0 && !dst)) {
        ct::set_error("ct_memset: bad destination");
        return CT_ERR_PARAM;
    }
    if (bytes && cudaMemsetAsync(dst, value, (size_t)bytes, (cudaStream_t)stream) != cudaSuccess)
        return ct::check_launch("ct_memset");
    return CT_OK;
}

extern "C" size_t ct_workspace_bytes(int which, int64_t nx, int64_t ny, int64_t nz, int64_t cap) {
    const int64_t N = nx * ny * nz;
    switch (which) {
        case 0: return (size_t)(2 * N) * sizeof(double);                                // gaussian
        case 1: {                                                                      // closing, cap = radius
            const size_t ext = (size_t)((nx + 2 * cap) * (ny + 2 * cap) * (nz + 2 * cap));
            const size_t rows = (size_t)(nx * ny) * 16 + 256;  // z-row words (u64 / u128)
            return ext > rows ? ext : rows;
        }
        case 2: return ct_table_workspace(N, cap);                                      // table
        case 3: return ct_edt_workspace(nx, ny, nz);                                    // edt
        case 4: return ct_mrf_workspace(nx, ny, nz, (int)cap);                          // mrf, cap = dtype
        default: return 0;
    }
}

// Measurement helper for the K1 roofline: throughput of separately rounded
// FP64 multiply and add (what the Gaussian issues), 8 independent chains.
__global__ void fp64_peak_kernel(double *out, int iters) {
    double x[8];
    const double m = 0.9999999, c = 1e-7 * (threadIdx.x + 1);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1.0 + i * 1e-3 + blockIdx.x * 1e-6;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(__dmul_rn(x[i], m), c);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

extern "C" int ct_fp64_peak(double *out, int iters, void *stream) {
    fp64_peak_kernel<<<CT_NUM_SMS * 8, 256, 0, (cudaStream_t)stream>>>(out, iters);
    return ct::check_launch("fp64_peak");
}
