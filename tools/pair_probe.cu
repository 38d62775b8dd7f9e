// pair_probe.cu -- development microbenchmark (not product): tcgen05.mma.cta_group::2 (M = 256) issue
// rate in the shapes the CTA-pair GEMM uses, alone and with the producers it runs beside:
//   TS  = A (weights) in TMEM, B (tokens) in shared memory   (gemm_tc2.cu)
//   SS  = both operands in shared memory
// optional concurrent tcgen05.st streams into the A columns (the dequantizers) and a per-k-block
// commit + barrier wait (the MMA thread's real loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/pair_probe tools/pair_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2602_20191_b200/csrc/sm100.cuh"

using namespace mobi::sm100;

// MODE bit 0: SS (A from smem) instead of TS; bit 1: commit per k-block; bit 2: wait the previous
// k-block's commit before issuing (serialised ring of 1 = worst case), bit 3: 4-deep ring waits
template <int MODE, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256 + 512, 1)
    pair_probe(int iters, int store_warps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 192 * 1024);
    __shared__ uint32_t slot;
    __shared__ int done;
    const int warp = warp_idx_uniform();
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(bar + i, 1);
        fence_barrier_init();
        done = 0;
    }
    // operands: zeros, or random fp16 in [-1, 1) (data-dependent power) when store_warps < 0
    const bool rnd = store_warps < 0;
    for (int i = threadIdx.x; i < 192 * 1024 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        reinterpret_cast<uint32_t*>(smem)[i] = rnd ? (h & 0xbbffbbffu) : 0u;
    }
    if (warp == 0) tmem_alloc_2sm(&slot, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    constexpr uint32_t idesc = idesc_f16(256, N, 0);
    if (rnd && warp >= 4 && warp < 8) {
        uint32_t v[16];
        for (int c = 0; c < 256; c += 16) {
            for (int k = 0; k < 16; ++k) {
                uint32_t h = (threadIdx.x * 977u + c * 131u + k * 7919u + blockIdx.x) * 2654435761u;
                h ^= h >> 16;
                v[k] = h & 0xbbffbbffu;
            }
            tmem_st16(((uint32_t)(32 * (warp % 4)) << 16) + 256 + c, v);
        }
        tmem_st_wait();
    }
    if (rnd) {
        tc_fence_before();
        __syncthreads();
        cluster_sync();
        tc_fence_after();
    }
    if (warp == 0) {
        if (rank == 0 && elect_one_sync()) {
            const uint64_t adesc = sdesc_sw128(smem_u32(smem));
            const uint64_t bdesc = sdesc_sw128(smem_u32(smem + 65536));
            long long t0 = clock64();
            unsigned long long g0, g1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
            for (int i = 0; i < iters; ++i) {
                const int s = i & 3;
                if (MODE & 4) {
                    if (i >= 1) mbar_wait(bar + ((i - 1) & 3), ((i - 1) >> 2) & 1);
                } else if (MODE & 8) {
                    if (i >= 4) {
                        if (MODE & 16)
                            mbar_wait_cluster(bar + s, ((i - 4) >> 2) & 1);
                        else
                            mbar_wait(bar + s, ((i - 4) >> 2) & 1);
                    }
                }
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (MODE & 1)
                        mma_ss_f16_2sm(0u, adesc + (uint64_t)(s * 1024 + j * 2), bdesc + (uint64_t)(s * 1024 + j * 2),
                                       idesc, 1u);
                    else
                        mma_ts_f16_2sm(0u, 256u + (uint32_t)(s * 32 + j * 8), bdesc + (uint64_t)(s * 1024 + j * 2),
                                       idesc, 1u);
                }
                if (MODE & 14) mma_commit_2sm_mc(bar + s, (uint16_t)0x3);
            }
            mma_commit_2sm_mc(bar + 4, (uint16_t)0x3);
            mbar_wait(bar + 4, 0);
            long long t1 = clock64();
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
            out[blockIdx.x / 2] = (unsigned long long)(t1 - t0);
            out[128 + blockIdx.x / 2] = g1 - g0;
            done = 1;
        }
        __syncwarp();
    } else if (warp >= 4 && warp < 4 + store_warps) {
        uint32_t v[16];
        for (int k = 0; k < 16; ++k) v[k] = 0x3c003c00u ^ (k * 0x01230321u) ^ threadIdx.x;
        const uint32_t lb = (uint32_t)(32 * (warp % 4)) << 16;
        long long t0 = clock64();
        int i = 0;
        for (; i < iters * 4 && !*(volatile int*)&done; ++i) {
            tmem_st16(lb + 256 + (i & 15) * 16, v);
            tmem_st_wait();
            if (rank == 1 && i > iters * 2) break;
        }
        if ((threadIdx.x & 31) == 0 && warp == 4 && rank == 0 && blockIdx.x == 0)
            printf("  st16+wait::st: %d iters, %.1f cycles each (store warps %d)\n", i, (double)(clock64() - t0) / i,
                   store_warps);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 0) tmem_dealloc_2sm(0, 512);
}

int main(int argc, char** argv) {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned long long* d_out;
    cudaMalloc(&d_out, sizeof(unsigned long long) * 256);
    int iters = 4000;
    const size_t sm = 192 * 1024 + 128;
    auto run = [&](auto kern, int N, int store, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const int grid = 2 * (nsm / 2);
        kern<<<grid, 256 + 512, sm>>>(iters, store, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: %s\n", name, cudaGetErrorString(e));
            exit(1);
        }
        unsigned long long h[256];
        cudaMemcpy(h, d_out, sizeof(unsigned long long) * 256, cudaMemcpyDeviceToHost);
        double avg = 0, ns = 0;
        for (int i = 0; i < grid / 2; ++i) avg += h[i], ns += h[128 + i];
        avg /= grid / 2;
        ns /= grid / 2;
        const double per = avg / (iters * 4.0);
        printf("%-34s N=%3d st=%2d it=%6d cycles/MMA %7.1f (ideal %5.1f) eff.MHz %6.0f  TFLOP/s(wall) %7.1f\n", name, N,
               store, iters, per, 128.0 * N / 256, avg / ns * 1e3,
               2.0 * 256 * N * 16 * iters * 4.0 * (grid / 2) / (ns * 1e-9) / 1e12);
    };
    if (argc > 1) {  // small-N per-k-block overhead study
        run(pair_probe<0, 32>, 32, 0, "TS pair N32 no commit");
        run(pair_probe<2, 32>, 32, 0, "TS pair N32 commit/kb");
        run(pair_probe<8, 32>, 32, 0, "TS pair N32 commit/kb ring4 wait");
        run(pair_probe<24, 32>, 32, 0, "TS pair N32 commit ring4 wait.cluster");
        run(pair_probe<2, 64>, 64, 0, "TS pair N64 commit/kb");
        run(pair_probe<8, 64>, 64, 0, "TS pair N64 commit/kb ring4 wait");
        run(pair_probe<8, 128>, 128, 0, "TS pair N128 commit/kb ring4 wait");
        run(pair_probe<24, 128>, 128, 0, "TS pair N128 commit ring4 wait.cluster");
        return 0;
    }
    run(pair_probe<0, 256>, 256, 0, "TS pair");
    run(pair_probe<0, 256>, 256, 8, "TS pair + st");
    run(pair_probe<0, 256>, 256, 16, "TS pair + st");
    run(pair_probe<1, 256>, 256, 0, "SS pair");
    run(pair_probe<1, 256>, 256, 16, "SS pair + st (other cols)");
    run(pair_probe<0, 128>, 128, 0, "TS pair");
    run(pair_probe<0, 64>, 64, 0, "TS pair");
    run(pair_probe<0, 32>, 32, 0, "TS pair");
    run(pair_probe<2, 256>, 256, 0, "TS pair commit/kb");
    run(pair_probe<8, 256>, 256, 0, "TS pair commit/kb ring4 wait");
    run(pair_probe<8, 256>, 256, 16, "TS pair commit/kb ring4 wait + st");
    run(pair_probe<4, 256>, 256, 0, "TS pair commit/kb serial wait");
    run(pair_probe<9, 256>, 256, 0, "SS pair commit/kb ring4 wait");
    run(pair_probe<9, 256>, 256, 16, "SS pair commit/kb ring4 wait + st");
    for (int it2 : {4000, 40000, 400000}) {
        iters = it2;
        run(pair_probe<0, 256>, 256, -1, "TS pair RANDOM data");
        run(pair_probe<0, 256>, 256, 0, "TS pair zeros");
    }
    iters = 4000;
    for (int rep = 0; rep < 1; ++rep) {
        run(pair_probe<0, 256>, 256, -1, "TS pair RANDOM data");
        run(pair_probe<1, 256>, 256, -1, "SS pair RANDOM data");
        run(pair_probe<0, 128>, 128, -1, "TS pair RANDOM data");
    }
    return 0;
}
