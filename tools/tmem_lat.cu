
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../paper_2602_20191_b200/csrc/sm100.cuh"
using namespace mobi::sm100;
__global__ void __launch_bounds__(512, 1) st_lat(int iters, int nwarps, unsigned long long* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    uint32_t v[16];
    for (int k = 0; k < 16; ++k) v[k] = k * 77 + threadIdx.x;
    const uint32_t lb = (uint32_t)(32 * (warp % 4)) << 16;
    if (warp < nwarps) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) { tmem_st16(lb + (i & 31) * 16, v); tmem_st_wait(); }
        long long t1 = clock64();
        for (int i = 0; i < iters; ++i) { tmem_st16(lb + (i & 31) * 16, v); }
        tmem_st_wait();
        long long t2 = clock64();
        uint32_t r[16];
        for (int i = 0; i < iters; ++i) { tmem_ld16(lb + (i & 31) * 16, r); tmem_ld_wait(); v[0] += r[3]; }
        long long t3 = clock64();
        uint32_t r2[16], r3[16], r4[16];
        for (int i = 0; i < iters; i += 4) {
            tmem_ld16(lb + (i & 31) * 16, r); tmem_ld16(lb + ((i + 1) & 31) * 16, r2);
            tmem_ld16(lb + ((i + 2) & 31) * 16, r3); tmem_ld16(lb + ((i + 3) & 31) * 16, r4);
            tmem_ld_wait(); v[0] += r[3] + r2[5] + r3[7] + r4[1];
        }
        long long t4 = clock64();
        uint32_t w[32];
        for (int i = 0; i < iters; ++i) { tmem_ld32(lb + (i & 15) * 32, w); tmem_ld_wait(); v[0] += w[3] + w[30]; }
        long long t5 = clock64();
        if ((threadIdx.x & 31) == 0) { out[warp * 8] = t1 - t0; out[warp * 8 + 1] = t2 - t1; out[warp * 8 + 2] = t3 - t2; out[warp*8+3] = v[0]; out[warp*8+4] = t4 - t3; out[warp*8+5] = t5 - t4; }
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc(0, 512);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 64 * 8 * 8);
    for (int nw : {1, 4, 8, 16}) {
        st_lat<<<148, 512>>>(2000, nw, d);
        { cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; } }
        unsigned long long h[64 * 8]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("warps %2d: st16+wait %.1f cyc, st16 pipelined %.1f cyc, ld16+wait %.1f cyc, ld16x4+wait %.1f cyc/ld, ld32+wait %.1f cyc\n", nw, h[0] / 2000.0, h[1] / 2000.0, h[2] / 2000.0, h[4] / 2000.0, h[5] / 2000.0);
    }
    return 0;
}
