// Layout check for the int8 tcgen05 path (tc_common.cuh): A from TMEM with an
// MN-major B, and A/B both K-major from shared memory; compared with a CPU GEMM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1407_2089_b200/csrc tc_i8_test.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace tc;

// A [128][256] u8 (TMEM), B [256][32] u8 MN-major (SMEM), D [128][32]
__global__ void test_ts(const uint8_t *A, const uint8_t *B, int32_t *D, int swap) {
    constexpr int N = 32, K = 256;
    __shared__ __align__(1024) uint8_t sm[K * N];
    __shared__ uint32_t tbase;
    __shared__ uint64_t mbar;
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tmem_alloc(&tbase, 512);
    const uint32_t lbo = (N / 16) * 128, sbo = 128;
    for (int e = t; e < K * N; e += 128) sm[mnmajor_off(e / N, e % N, lbo, sbo)] = B[e];
    if (t == 0) {
        mbar_init(&mbar, 1);
        mbar_fence_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t base = tbase;
    const uint32_t lane_addr = base + ((uint32_t)(w * 32) << 16);
    for (int cc = 0; cc < K / 4; cc += 8) {
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) {
            const uint8_t *p = A + t * K + 4 * (cc + i);
            v[i] = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
        }
        tmem_st8(lane_addr + cc, v);
    }
    tmem_st_wait();
    fence_before();
    __syncthreads();
    fence_after();
    if (t == 0) {
        const uint32_t id = idesc_i8(128, N, false, false, false, true);
        for (int ks = 0; ks < K / 32; ++ks) {
            const uint64_t bd = smem_desc(smem_u32(sm) + ks * 4 * lbo, swap ? sbo : lbo, swap ? lbo : sbo);
            mma_i8_ts(base + 256, base + ks * 8, bd, id, ks > 0);
        }
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    fence_after();
    for (int h = 0; h < N; h += 16) {
        uint32_t v[16];
        tmem_ld16(lane_addr + 256 + h, v);
        tmem_ld_wait();
        for (int i = 0; i < 16; ++i) D[t * N + h + i] = (int32_t)v[i];
    }
    fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc(base, 512);
}

// A [128][160] u8 K-major (SMEM), B [64][160] u8 K-major (SMEM), D [128][64]
__global__ void test_ss(const uint8_t *A, const uint8_t *B, int32_t *D, int swap) {
    constexpr int M = 128, N = 64, K = 160;
    __shared__ __align__(1024) uint8_t sa[M * K];
    __shared__ __align__(1024) uint8_t sb[N * K];
    __shared__ uint32_t tbase;
    __shared__ uint64_t mbar;
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tmem_alloc(&tbase, 512);
    const uint32_t lbo = 128, sbo = (K / 16) * 128;
    for (int e = t; e < M * K; e += 128) sa[kmajor_off(e / K, e % K, lbo, sbo)] = A[e];
    for (int e = t; e < N * K; e += 128) sb[kmajor_off(e / K, e % K, lbo, sbo)] = B[e];
    if (t == 0) {
        mbar_init(&mbar, 1);
        mbar_fence_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t base = tbase;
    const uint32_t lane_addr = base + ((uint32_t)(w * 32) << 16);
    if (t == 0) {
        const uint32_t id = idesc_i8(M, N, false, false, false, false);
        for (int ks = 0; ks < K / 32; ++ks) {
            const uint32_t L = swap ? sbo : lbo, S = swap ? lbo : sbo;
            const uint64_t ad = smem_desc(smem_u32(sa) + ks * 2 * lbo, L, S);
            const uint64_t bd = smem_desc(smem_u32(sb) + ks * 2 * lbo, L, S);
            mma_i8_ss(base, ad, bd, id, ks > 0);
        }
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    fence_after();
    for (int h = 0; h < N; h += 16) {
        uint32_t v[16];
        tmem_ld16(lane_addr + h, v);
        tmem_ld_wait();
        for (int i = 0; i < 16; ++i) D[t * N + h + i] = (int32_t)v[i];
    }
    fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc(base, 512);
}

int main() {
    srand(1);
    {
        const int M = 128, N = 32, K = 256;
        std::vector<uint8_t> A(M * K), B(K * N);
        for (auto &x : A) x = rand() & 255;
        for (auto &x : B) x = rand() & 255;
        std::vector<int32_t> ref(M * N, 0), got(M * N);
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                int s = 0;
                for (int k = 0; k < K; ++k) s += A[m * K + k] * B[k * N + n];
                ref[m * N + n] = s;
            }
        uint8_t *dA, *dB;
        int32_t *dD;
        cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, got.size() * 4);
        cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
        for (int swap = 0; swap < 2; ++swap) {
            cudaMemset(dD, 0, got.size() * 4);
            test_ts<<<1, 128>>>(dA, dB, dD, swap);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int i = 0; i < M * N; ++i) bad += got[i] != ref[i];
            printf("TS (A tmem, B MN-major) swap=%d: %s, mismatches %d / %d (got[0]=%d ref[0]=%d)\n", swap,
                   cudaGetErrorString(e), bad, M * N, got[0], ref[0]);
        }
    }
    {
        const int M = 128, N = 64, K = 160;
        std::vector<uint8_t> A(M * K), B(N * K);
        for (auto &x : A) x = rand() & 255;
        for (auto &x : B) x = rand() & 255;
        std::vector<int32_t> ref(M * N, 0), got(M * N);
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                int s = 0;
                for (int k = 0; k < K; ++k) s += A[m * K + k] * B[n * K + k];
                ref[m * N + n] = s;
            }
        uint8_t *dA, *dB;
        int32_t *dD;
        cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, got.size() * 4);
        cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
        for (int swap = 0; swap < 2; ++swap) {
            cudaMemset(dD, 0, got.size() * 4);
            test_ss<<<1, 128>>>(dA, dB, dD, swap);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int i = 0; i < M * N; ++i) bad += got[i] != ref[i];
            printf("SS (A,B K-major) swap=%d: %s, mismatches %d / %d (got[0]=%d ref[0]=%d)\n", swap,
                   cudaGetErrorString(e), bad, M * N, got[0], ref[0]);
        }
    }
    return 0;
}
