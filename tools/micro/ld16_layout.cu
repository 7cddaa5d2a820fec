// Probe of the tcgen05.ld 16xNb shapes: which (lane, column) each thread of a
// warp receives.  TMEM cell (lane, col) holds lane * 1000 + col.
#include <cstdio>
#include <cstdint>
#include "../../paper_1407_2089_b200/csrc/tc_common.cuh"

__device__ __forceinline__ void ld16x64(uint32_t a, uint32_t &r0) {
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(a) : "memory");
}
__device__ __forceinline__ void ld16x128(uint32_t a, uint32_t (&r)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(a) : "memory");
}
__device__ __forceinline__ void ld16x256(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a) : "memory");
}

__global__ void probe(int *out) {
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, wp = t >> 5, lane = t & 31;
    if (wp == 0) tc::tmem_alloc(&tbase, 32);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t base = tbase;
    uint32_t v[8];
    for (int c = 0; c < 16; c += 8) {
        for (int i = 0; i < 8; ++i) v[i] = (uint32_t)((32 * wp + lane) * 1000 + c + i);
        tc::tmem_st8(base + ((uint32_t)(32 * wp) << 16) + c, v);
    }
    tc::tmem_st_wait();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (wp == 0) {
        for (int lb = 0; lb <= 16; lb += 16) {
            const uint32_t a = base + ((uint32_t)lb << 16);
            uint32_t r1, r2[2], r4[4];
            ld16x64(a, r1);
            ld16x128(a, r2);
            ld16x256(a, r4);
            tc::tmem_ld_wait();
            int *o = out + (lb / 16) * 32 * 7 + lane * 7;
            o[0] = r1; o[1] = r2[0]; o[2] = r2[1]; o[3] = r4[0]; o[4] = r4[1]; o[5] = r4[2]; o[6] = r4[3];
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (wp == 0) tc::tmem_dealloc(base, 32);
}

int main() {
    int *d, h[2 * 32 * 7];
    cudaMalloc(&d, sizeof(h));
    probe<<<1, 128>>>(d);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int lb = 0; lb < 2; ++lb) {
        printf("lane base %d (value = lane*1000 + col)\n thr | 16x64b | 16x128b       | 16x256b\n", 16 * lb);
        for (int t = 0; t < 32; ++t) {
            const int *o = h + lb * 32 * 7 + t * 7;
            printf("%3d | %6d | %6d %6d | %6d %6d %6d %6d\n", t, o[0], o[1], o[2], o[3], o[4], o[5], o[6]);
        }
    }
    return 0;
}
