// mma_probe.cu -- microbenchmark of the sm_100a primitives the MoBi kernels are built on
// (development tool, not part of the product).  One CTA per SM; thread 0 issues a stream of
// tcgen05.mma (kind::f16, M=128) with operands resident in shared memory / TMEM and measures
// cycles per instruction; optional concurrent TMA streaming and TMEM stores emulate the GEMM's
// producers.  Prints cycles/MMA and the implied chip TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe tools/mma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#include "../paper_2602_20191_b200/csrc/sm100.cuh"

using namespace mobi::sm100;

template <int MODE, int N>
__device__ __forceinline__ void issue_loop(int iters, uint64_t adesc, uint64_t bdesc, uint64_t* sink, uint64_t* done_bar) {
    constexpr uint32_t idesc = idesc_f16(128, N, 0);
    for (int i = 0; i < iters; ++i) {
        if (MODE >= 3) tc_fence_after();
        if (MODE >= 4) mbar_wait(done_bar, 0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (MODE == 0)
                mma_ss_f16(0u, adesc + j * 2, bdesc + j * 2, idesc, 1u);
            else
                mma_ts_f16(0u, 256u + j * 8, bdesc + j * 2, idesc, 1u);
        }
        if (MODE == 7) mma_commit_mc(sink, (uint16_t)0x3);
        else if (MODE >= 2) mma_commit(sink);
    }
}

// cluster-of-2 variant for the multicast commit
template <int MODE, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) probe_cl(int iters, int store_warps,
                                                                             unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 160 * 1024);
    __shared__ uint32_t slot;
    const int warp = warp_idx_uniform();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        mbar_arrive(bar + 1);
        mbar_init(bar + 2, 2 * 1000000);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    if (warp == 0 && elect_one_sync()) {
        const uint64_t adesc = sdesc_sw128(smem_u32(smem));
        const uint64_t bdesc = sdesc_sw128(smem_u32(smem + 32768));
        long long t0 = clock64();
        issue_loop<MODE, N>(iters, adesc, bdesc, bar + 2, bar + 1);
        mma_commit(bar);
        mbar_wait(bar, 0);
        out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 0) tmem_dealloc(0, 512);
}

template <int MODE, int N>
__global__ void __launch_bounds__(256, 1) probe(int iters, int store_warps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 160 * 1024);
    __shared__ uint32_t slot;
    __shared__ int done;
    const int warp = warp_idx_uniform(), lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        mbar_arrive(bar + 1);  // phase 0 complete
        mbar_init(bar + 2, 1);
        fence_barrier_init();
        done = 0;
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        if (elect_one_sync()) {
            const uint64_t adesc = sdesc_sw128(smem_u32(smem));
            const uint64_t bdesc = sdesc_sw128(smem_u32(smem + 32768));
            long long t0 = clock64();
            issue_loop<MODE, N>(iters, adesc, bdesc, bar + 2, bar + 1);
            mma_commit(bar);
            mbar_wait(bar, 0);
            long long t1 = clock64();
            out[blockIdx.x] = (unsigned long long)(t1 - t0);
            done = 1;
        }
        __syncwarp();
    } else if (warp >= 2 && warp < 2 + store_warps) {
        uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const uint32_t lb = (uint32_t)(32 * (warp % 4)) << 16;
        for (int i = 0; i < iters * 4 && !*(volatile int*)&done; ++i) {
            tmem_st8(lb + 256 + 128 + (i & 7) * 8, v);
            tmem_st_wait();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(0, 512);
}

// L2 -> SM streaming bandwidth with TMA: each CTA keeps `depth` 32 KiB loads in flight over a
// buffer of `rows` x 64 fp16 (L2 resident when small), cycling through distinct tiles.
__global__ void __launch_bounds__(32, 1) tma_bw(const __grid_constant__ CUtensorMap tmap, int rows, int iters,
                                                int depth, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * 32768);
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) mbar_init(&bars[i], 1);
        fence_barrier_init();
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const int ntiles = rows / 256;
    long long t0 = clock64();
    for (int i = 0; i < iters + depth; ++i) {
        const int s = i % depth;
        if (i >= depth) mbar_wait(&bars[s], ((i / depth) - 1) & 1);
        if (i < iters) {
            mbar_arrive_expect_tx(&bars[s], 32768);
            tma_load_2d(smem + s * 32768, &tmap, &bars[s], 0, ((blockIdx.x * 7 + i) % ntiles) * 256);
        }
    }
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned long long* d_out;
    cudaMalloc(&d_out, sizeof(unsigned long long) * nsm);
    void* buf;
    cudaMalloc(&buf, 8192 * 64 * 2);
    cudaMemset(buf, 0, 8192 * 64 * 2);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    CUtensorMap hmap;
    cuuint64_t dims[2] = {64, 8192};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 256};
    cuuint32_t es[2] = {1, 1};
    ((PFN_encodeTiled)f)(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* dmap;
    cudaMalloc(&dmap, sizeof(hmap));
    cudaMemcpy(dmap, &hmap, sizeof(hmap), cudaMemcpyHostToDevice);
    const int iters = 2000;
    auto runp = [&](auto kern, int N, int store, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024 + 64);
        kern<<<nsm, 256, 161 * 1024 + 64>>>(iters, store, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
        unsigned long long h[256];
        cudaMemcpy(h, d_out, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < nsm; ++i) avg += h[i];
        avg /= nsm;
        double per = avg / (iters * 4.0);
        printf("%-30s N=%3d cycles/MMA %7.1f (ideal %5.1f)  chip TFLOP/s @%d MHz: %7.1f\n", name, N, per, 128.0 * N / 256,
               clk / 1000, 2.0 * 128 * N * 16 / per * (clk * 1e3) * nsm / 1e12);
    };
    runp(probe<0, 16>, 16, 0, "SS");  runp(probe<0, 64>, 64, 0, "SS");  runp(probe<0, 128>, 128, 0, "SS");
    runp(probe<0, 256>, 256, 0, "SS");
    runp(probe<1, 16>, 16, 0, "TS");  runp(probe<1, 64>, 64, 0, "TS");  runp(probe<1, 128>, 128, 0, "TS");
    runp(probe<1, 256>, 256, 0, "TS");
    runp(probe<1, 256>, 256, 8, "TS + 8 st warps");
    runp(probe<2, 16>, 16, 0, "TS +commit/kblk"); runp(probe<2, 256>, 256, 0, "TS +commit/kblk");
    runp(probe<3, 16>, 16, 0, "TS +commit+fence"); runp(probe<3, 256>, 256, 0, "TS +commit+fence");
    runp(probe<4, 16>, 16, 0, "TS +c+f+trywait"); runp(probe<4, 256>, 256, 0, "TS +c+f+trywait");
    runp(probe_cl<2, 16>, 16, 0, "TS cluster2 +commit");
    runp(probe_cl<7, 16>, 16, 0, "TS cluster2 +commit multicast");
    runp(probe_cl<7, 256>, 256, 0, "TS cluster2 +commit multicast");
    // L2 bandwidth: 64 MiB buffer (L2 resident) and 1 GiB (HBM)
    for (long long rows : std::initializer_list<long long>{}) {
        void* big;
        cudaMalloc(&big, rows * 128);
        cudaMemset(big, 1, rows * 128);
        CUtensorMap bmap;
        cuuint64_t d2[2] = {64, (cuuint64_t)rows};
        ((PFN_encodeTiled)f)(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, big, d2, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(tma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 64);
        for (int depth : {2, 4, 6}) {
            const int it = 400;
            tma_bw<<<nsm, 32, 6 * 32768 + 64>>>(bmap, (int)rows, it, depth, d_out);
            cudaDeviceSynchronize();
            unsigned long long h[256];
            cudaMemcpy(h, d_out, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < nsm; ++i) avg += h[i];
            avg /= nsm;
            double bpc = 32768.0 * it / avg;
            printf("TMA stream %5lld MiB depth %d: %.1f B/cycle/SM  chip %.2f TB/s\n", rows * 128 >> 20, depth, bpc,
                   bpc * nsm * clk * 1e3 / 1e12);
        }
        cudaFree(big);
    }
    return 0;
}
