// drain_probe.cu -- development microbenchmark: the tc2 epilogue's TMEM drain (8 warps, 2 per lane
// quarter, 16-column tcgen05.ld chunks, x 2^e, bf16 pack, two 16-byte smem stores per chunk) in isolation.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2602_20191_b200/csrc/sm100.cuh"
using namespace mobi::sm100;

template <int V>
__global__ void __launch_bounds__(256, 1) drain(int reps, unsigned long long* out, float* sink, __nv_bfloat16* Y) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    float* tok_es = reinterpret_cast<float*>(smem + 65536);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) tmem_alloc(&slot, 512);
    for (int i = threadIdx.x; i < 256; i += 256) tok_es[i] = 1.0f + i;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int q = warp % 4, half = warp / 4;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    auto swz = [](int r) { return (r ^ (r >> 3)) & 7; };
    const int my_r = 32 * q + lane;
    uint8_t* my_row = smem + my_r * 512;
    const int my_g = swz(my_r);
    const int n = 256;
    uint32_t acc_sink = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        uint32_t va[16], vb[16];
        tmem_ld16(lane_base + 16 * half, va);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int c = 2 * i + half;
            const int c0 = 16 * c;
            if (c0 >= n) break;
            tmem_ld_wait();
            uint32_t(&cur)[16] = (i & 1) ? vb : va;
            uint32_t(&nxt)[16] = (i & 1) ? va : vb;
            if (c0 + 32 < n) tmem_ld16(lane_base + c0 + 32, nxt);
            uint32_t w[8];
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
                const float4 es = V & 1 ? make_float4(1.f, 2.f, 3.f, 4.f) : reinterpret_cast<const float4*>(tok_es + c0)[j4];
                const __nv_bfloat162 lo = __floats2bfloat162_rn(__uint_as_float(cur[4 * j4]) * es.x,
                                                                __uint_as_float(cur[4 * j4 + 1]) * es.y);
                const __nv_bfloat162 hi = __floats2bfloat162_rn(__uint_as_float(cur[4 * j4 + 2]) * es.z,
                                                                __uint_as_float(cur[4 * j4 + 3]) * es.w);
                w[2 * j4] = *reinterpret_cast<const uint32_t*>(&lo);
                w[2 * j4 + 1] = *reinterpret_cast<const uint32_t*>(&hi);
            }
            const int ch = 2 * c;
            if (V & 2) {
                acc_sink ^= w[0] ^ w[1] ^ w[2] ^ w[3] ^ w[4] ^ w[5] ^ w[6] ^ w[7];
            } else {
                *reinterpret_cast<uint4*>(my_row + ((ch ^ my_g) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
                *reinterpret_cast<uint4*>(my_row + (((ch + 1) ^ my_g) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    __syncthreads();
    if (lane == 0) out[blockIdx.x * 8 + warp] = (t1 - t0) / reps;
    // the scatter: thread = (8-row chunk et%16, token pair), 8 four-byte reads -> 8 rows x 2 tokens
    int32_t* tok_src = reinterpret_cast<int32_t*>(smem + 65536 + 1024);
    for (int i = threadIdx.x; i < 256; i += 256) tok_src[i] = (i * 37) % 256;
    __syncthreads();
    long long t2 = clock64();
    const int et = threadIdx.x;
    for (int rep = 0; rep < reps; ++rep) {
        const int rc0 = 8 * (et % 16);
        const int64_t r0 = (int64_t)blockIdx.x * 128 + rc0;
        for (int t = 2 * (et / 16); t < n; t += 32) {
            uint32_t wv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int r = rc0 + u;
                wv[u] = *reinterpret_cast<const uint32_t*>(smem + r * 512 + (((t >> 3) ^ swz(r)) << 4) + (t & 7) * 2);
            }
            const float e0 = tok_es[t], e1 = tok_es[t + 1];
            uint32_t o0[4], o1[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t a = wv[2 * u], b = wv[2 * u + 1];
                const __nv_bfloat162 lo = __floats2bfloat162_rn(__uint_as_float(a << 16) * e0, __uint_as_float(b << 16) * e0);
                const __nv_bfloat162 hi = __floats2bfloat162_rn(__uint_as_float(a & 0xffff0000u) * e1,
                                                                __uint_as_float(b & 0xffff0000u) * e1);
                o0[u] = *reinterpret_cast<const uint32_t*>(&lo);
                o1[u] = *reinterpret_cast<const uint32_t*>(&hi);
            }
            const uint4 y0 = make_uint4(o0[0], o0[1], o0[2], o0[3]);
            const uint4 y1 = make_uint4(o1[0], o1[1], o1[2], o1[3]);
            *reinterpret_cast<uint4*>(Y + (int64_t)tok_src[t] * 148 * 128 + r0) = y0;
            *reinterpret_cast<uint4*>(Y + (int64_t)tok_src[t + 1] * 148 * 128 + r0) = y1;
        }
    }
    __syncthreads();
    long long t3 = clock64();
    if (lane == 0) out[1184 + blockIdx.x * 8 + warp] = (t3 - t2) / reps;
    if (threadIdx.x == 0) sink[blockIdx.x] = reinterpret_cast<float*>(smem)[blockIdx.x] + (float)acc_sink;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(0, 512);
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8 * 148 * 8 * 2);
    __nv_bfloat16* Y;
    cudaMalloc(&Y, (size_t)256 * 148 * 128 * 2);
    cudaMalloc(&sink, 148 * 4);
    auto run = [&](auto k, const char* name) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
        k<<<148, 256, 70 * 1024>>>(100, d, sink, Y);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
        unsigned long long h[8];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%-28s cycles per drain per warp:", name);
        for (int w = 0; w < 8; ++w) printf(" %llu", h[w]);
        unsigned long long h2[8];
        cudaMemcpy(h2, d + 1184, sizeof(h2), cudaMemcpyDeviceToHost);
        printf("   scatter:");
        for (int w = 0; w < 8; ++w) printf(" %llu", h2[w]);
        printf("\n");
    };
    run(drain<0>, "full");
    run(drain<1>, "no tok_es LDS");
    run(drain<2>, "no STS");
    run(drain<3>, "no LDS, no STS");
    return 0;
}
