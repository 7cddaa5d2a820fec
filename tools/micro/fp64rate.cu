// FP64 instruction throughput microbenchmark: DADD / DMUL / DFMA chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double *out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = __dadd_rn(x[i], a);
            else if (OP == 1) x[i] = __dmul_rn(x[i], b);
            else if (OP == 2) x[i] = __fma_rn(x[i], b, a);
            else x[i] = __fma_rn(__dadd_rn(x[i], a), b, x[i]);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
int main() {
    double *o; cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000, blocks = 148 * 8, threads = 256;
    const char *names[4] = {"DADD", "DMUL", "DFMA", "DADD+DFMA(2 instr)"};
    for (int op = 0; op < 4; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, threads>>>(o, iters, 1e-9, 1.0000001);
            if (op == 1) k<1><<<blocks, threads>>>(o, iters, 1e-9, 1.0000001);
            if (op == 2) k<2><<<blocks, threads>>>(o, iters, 1e-9, 1.0000001);
            if (op == 3) k<3><<<blocks, threads>>>(o, iters, 1e-9, 1.0000001);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)blocks * threads * iters * 8 * (op == 3 ? 2 : 1);
            if (rep) printf("%s: %.2f T instr/s (%.3f ms)\n", names[op], ops / ms / 1e9, ms);
        }
    }
    return 0;
}
