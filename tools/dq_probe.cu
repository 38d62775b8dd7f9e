// dq_probe.cu -- development microbenchmark: the CTA-pair GEMM's dequantizer loop alone (16 warps = 4
// TMEM lane quarters x 4 k-block phases; per k-block: 4 x LDS.128 codes + 2 group constants from smem,
// 16 dequant4, one 32-column tcgen05.st, wait::st, fence, arrive) -- how many cycles per k-block can the
// dequantizers sustain with nothing else on the SM?
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2602_20191_b200/csrc/mobi_internal.cuh"
#include "../paper_2602_20191_b200/csrc/sm100.cuh"
using namespace mobi;
using namespace mobi::sm100;

template <int V>
__global__ void __launch_bounds__(512, 1) dq(int nkb, unsigned long long* out, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t full[5];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 4 * 20480 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 5; ++s) mbar_init(&full[s], 4);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int q = warp % 4, ph4 = warp / 4, sub = ph4 & 1, jpar = ph4 >> 1;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int c_off = sub * 8192 + (32 * q + lane) * 16;
    const uint32_t mw = 0xffffffffu;
    const float kc = 0.3f, inv2p = 1.f / 64;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int j = jpar; 2 * j < nkb; j += 2) {
        const int kb = 2 * j + sub;
        const uint8_t* dc = smem + (j % 4) * 20480 + c_off;
        uint4 c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = *reinterpret_cast<const uint4*>(dc + u * 128 * 16);
        float2 g[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) g[hh] = *reinterpret_cast<const float2*>(smem + (j % 4) * 20480 + 16384 + (32 * q + lane) * 8);
        uint32_t v[32];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const __half2 S2 = __float2half2_rn(g[hh].x * inv2p);
            const __half2 C2 = __float2half2_rn(fmaf(g[hh].x, kc, -g[hh].y));
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const uint32_t* w = reinterpret_cast<const uint32_t*>(&c[hh * 2 + cc]);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int o = hh * 16 + cc * 8 + 2 * u;
                    dequant4(w[u], mw, S2, C2, v[o], v[o + 1]);
                }
            }
        }
        const int s = kb % 5;
        if (V == 0) {
            tc_fence_after();
            tmem_st32(lane_base + 256 + s * 32, v);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&full[s]);
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc ^= v[i];
        }
    }
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
    sink[blockIdx.x * 512 + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(0, 512);
}

int main() {
    unsigned long long* d;
    uint32_t* sink;
    cudaMalloc(&d, 148 * 16 * 8);
    cudaMalloc(&sink, 148 * 512 * 4);
    const int nkb = 256;
    auto run = [&](auto k, const char* name) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 20480 + 1024);
        k<<<148, 512, 4 * 20480 + 1024>>>(nkb, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
        unsigned long long h[16];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int w = 0; w < 16; ++w) mx = h[w] > mx ? h[w] : mx;
        printf("%-24s %d k-blocks: %.0f cycles per k-block (max over warps)\n", name, nkb, mx / nkb);
    };
    run(dq<0>, "dequant + TMEM store");
    run(dq<1>, "dequant only");
    return 0;
}
