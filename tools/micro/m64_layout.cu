// Probe of the tcgen05 kind::i8 M = 64 (cta_group::1) TMEM layout: which
// lanes an M = 64 accumulator occupies, and whether A / D at a lane offset of
// 16 select the other half.  A[m][k] = (k == m % 32), B[k][n] = (k * 3 + n) & 127
// => D[m][n] = B[m % 32][n].  Prints, for each TMEM lane, the row it holds.
#include <cstdio>
#include <cstdint>
#include "../../paper_1407_2089_b200/csrc/tc_common.cuh"

__global__ void probe(int lane_off, int *out) {
    __shared__ __align__(1024) uint8_t sb[32 * 32];
    __shared__ uint32_t tbase;
    __shared__ uint64_t mbar;
    const int t = threadIdx.x, wp = t >> 5, lane = t & 31;
    if (wp == 0) tc::tmem_alloc(&tbase, 512);
    for (int e = t; e < 32 * 32; e += blockDim.x) {
        const int n = e / 32, k = e % 32;
        sb[tc::kmajor_off(n, k, 128, 256)] = (uint8_t)((k * 3 + n) & 127);
    }
    if (t == 0) { tc::mbar_init(&mbar, 1); tc::mbar_fence_init(); }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t base = tbase;
    // A rows: lane L of quarter wp; guess row m = (L % 16) + 16 * wp for L % 32 < 16 (half 0), same + 64 for half 1
    {
        const int half = lane >= 16, m = (lane & 15) + 16 * wp;
        uint32_t v[8];
        for (int c = 0; c < 8; ++c) {  // 8 columns x 4 bytes = K 32
            uint32_t w = 0;
            for (int b = 0; b < 4; ++b) w |= (uint32_t)((4 * c + b) == (m % 32) ? (half ? 2 : 1) : 0) << (8 * b);
            v[c] = w;
        }
        tc::tmem_st8(base + ((uint32_t)(32 * wp) << 16) + 0, v);
        tc::tmem_st_wait();
    }
    // zero the D region
    {
        uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c = 0; c < 32; c += 8) tc::tmem_st8(base + ((uint32_t)(32 * wp) << 16) + 256 + c, z);
        tc::tmem_st_wait();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (wp == 0) {
        if (tc::elect_one()) {
            const uint32_t idesc = tc::idesc_i8(64, 32, false, false, false, false);
            const uint64_t bd = tc::smem_desc(tc::smem_u32(sb), 128, 256);
            const uint32_t loff = (uint32_t)lane_off << 16;
            tc::mma_i8_ts(base + loff + 256, base + loff + 0, bd, idesc, 0u);
            tc::mma_commit(&mbar);
        }
        __syncwarp();
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    uint32_t d[8];
    for (int c = 0; c < 32; c += 8) {
        tc::tmem_ld8(base + ((uint32_t)(32 * wp) << 16) + 256 + c, d);
        tc::tmem_ld_wait();
        for (int i = 0; i < 8; ++i) out[(32 * wp + lane) * 32 + c + i] = (int)d[i];
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (wp == 0) tc::tmem_dealloc(base, 512);
}

int main() {
    int *d, h[128 * 32];
    cudaMalloc(&d, sizeof(h));
    for (int lo = 0; lo <= 16; lo += 16) {
        cudaMemset(d, 0xff, sizeof(h));
        probe<<<1, 128>>>(lo, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("lane_off %d: %s\n", lo, cudaGetErrorString(e));
        for (int L = 0; L < 128; ++L) {
            // identify row: D[L][n] should be s * B[r][n] = s * ((r*3+n)&127) for some r, s in {1,2}
            int found = -1, sc = 0;
            for (int s = 1; s <= 2 && found < 0; ++s)
                for (int r = 0; r < 32 && found < 0; ++r) {
                    bool ok = true;
                    for (int n = 0; n < 32; ++n) ok &= h[L * 32 + n] == s * ((r * 3 + n) & 127);
                    if (ok) { found = r; sc = s; }
                }
            int zero = 1;
            for (int n = 0; n < 32; ++n) zero &= h[L * 32 + n] == 0;
            printf("%s%3d:%s", L % 8 ? "" : "\n", L, found >= 0 ? (sc == 1 ? "a" : "b") : (zero ? " z" : " ?"));
            if (found >= 0) printf("%-2d", found); else printf("  ");
            printf(" ");
        }
        printf("\n");
    }
    return 0;
}
