// l2_probe.cu -- development microbenchmark: chip-wide L2->SM streaming bandwidth with bulk async
// copies (cp.async.bulk, the TMA path), one CTA per SM, NS-stage ring of CHUNK-byte copies.
//   mode 0: every CTA streams its own distinct slice of an L2-resident buffer
//   mode 1: CTAs in pairs read the same addresses (no multicast)
//   mode 2: clusters of 2, each CTA issues half of the chunks multicast to both
//   mode 3: all CTAs read the same addresses
// Prints bytes delivered into shared memory per cycle per SM and chip TB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2602_20191_b200/csrc/sm100.cuh"
using namespace mobi::sm100;


__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}

template <int MODE, int CHUNK, int NS, int BOXR = 32, int V = 0>
__global__ void __launch_bounds__(96, 1) probe(const uint8_t* buf, size_t buf_bytes, int iters, unsigned long long* out, const __grid_constant__ CUtensorMap tm) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[NS], empty[NS];
    const int warp = threadIdx.x / 32;
    const uint32_t rank = MODE == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MODE == 2 ? 2 : 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (MODE == 2) cluster_sync();
    int src_cta = blockIdx.x;
    if (MODE == 1 || MODE == 2) src_cta = blockIdx.x / 2;
    if (MODE == 3) src_cta = 0;
    const size_t per_cta = (buf_bytes / gridDim.x / CHUNK) * CHUNK;
    const size_t nchunk = per_cta / CHUNK;
    long long t0 = clock64();
    if ((warp == 0 || (V == 2 && warp == 2)) && threadIdx.x % 32 == 0) {
        for (int it = (V == 2 && warp == 2) ? 1 : 0; it < iters; it += (V == 2 ? 2 : 1)) {
            const int s = it % NS;
            long long ta = clock64();
            mbar_wait(&empty[s], ((it / NS) & 1) ^ 1);
            long long tb = clock64();
            if (blockIdx.x == 0 && it < 64 && V == 9) out[1024 + it] = tb - ta;
            const uint8_t* src = buf + (size_t)src_cta * per_cta + (size_t)(it % nchunk) * CHUNK;
            if (MODE == 5) {
                // strided 2D: matrix [rows][4096] fp16 (8 KB pitch), box {64 cols, BOXR rows}; walk k then rows
                mbar_arrive_expect_tx(&full[s], CHUNK);
                const int nrows = (int)(buf_bytes / 8192);
                const int kc = (it % 64) * 64;
                const int rb = (int)(((size_t)blockIdx.x * 7 + it / 64) % (size_t)(nrows / (CHUNK / 128))) * (CHUNK / 128);
                for (int b = 0; b < CHUNK / (BOXR * 128); ++b)
                    tma_load_2d(sm + s * CHUNK + b * BOXR * 128, &tm, &full[s], kc, rb + b * BOXR);
            } else if (MODE == 4) {
                // 2D tensor TMA: rows of 128 B (64 fp16), BOXR-row boxes, CHUNK bytes per stage
                mbar_arrive_expect_tx(&full[s], CHUNK);
                const int row0 = (int)(((size_t)src_cta * per_cta + (size_t)(it % nchunk) * CHUNK) / 128);
                for (int b = 0; b < CHUNK / (BOXR * 128); ++b)
                    tma_load_2d(sm + s * CHUNK + b * BOXR * 128, &tm, &full[s], 0, row0 + b * BOXR);
            } else if (MODE == 2) {
                mbar_arrive_expect_tx(&full[s], CHUNK);
                bulk_mc(sm + s * CHUNK + rank * (CHUNK / 2), src + rank * (CHUNK / 2), CHUNK / 2, &full[s], 0x3);
            } else {
                if (V == 1)
                    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(CHUNK) : "memory");
                else
                    mbar_arrive_expect_tx(&full[s], CHUNK);
                long long tc = clock64();
                bulk(sm + s * CHUNK, src, CHUNK, &full[s]);
                long long td = clock64();
                if (blockIdx.x == 0 && it < 64 && V == 9) out[1024 + 64 + it] = (td - tc) * 100000 + (tc - tb);
            }
        }
    } else if (warp == 1 && threadIdx.x == 32) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % NS;
            mbar_wait(&full[s], (it / NS) & 1);

            if (MODE == 2) {
                mbar_arrive(&empty[s]);
                mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), rank ^ 1));
            } else {
                mbar_arrive(&empty[s]);
            }
        }
    }
    __syncthreads();
    if (MODE == 2) cluster_sync();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

CUtensorMap g_tm[8];
template <int MODE, int CHUNK, int NS, int BOXR = 32, int V = 0>
void run(const char* name, const uint8_t* buf, size_t bytes, unsigned long long* d_out, int nsm) {
    auto k = probe<MODE, CHUNK, NS, BOXR, V>;
    const CUtensorMap& tm = g_tm[(BOXR == 32 ? 0 : BOXR == 64 ? 1 : BOXR == 128 ? 2 : 3) + (MODE == 5 ? 4 : 0)];
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * CHUNK);
    const int iters = 2000;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm);
    cfg.blockDim = dim3(96);
    cfg.dynamicSmemBytes = NS * CHUNK;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = MODE == 2 ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k, (const uint8_t*)buf, bytes, iters, d_out, tm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, (const uint8_t*)buf, bytes, iters, d_out, tm);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[1024 + 128];
    cudaMemcpy(h, d_out, (1024 + 128) * 8, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 0; ++i) printf("  it %2d wait %8llu issue*1e5+expect %8llu\n", i, h[1024 + i], h[1024 + 64 + i]);
    double cyc = 0;
    for (int i = 0; i < nsm; ++i) cyc += h[i];
    cyc /= nsm;
    const double per_sm = (double)iters * CHUNK;
    printf("%-32s NS %2d boxr %3d chunk %6d  %6.1f B/cyc/SM  chip %6.2f TB/s (delivered to smem)  %.1f us\n", name, NS, BOXR, CHUNK,
           per_sm / cyc, per_sm * nsm / (ms * 1e-3) / 1e12, ms * 1e3);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    size_t bytes = 48ull << 20;  // L2 resident
    uint8_t* buf;
    cudaMalloc(&buf, 1ull << 30);
    cudaMemset(buf, 1, 1ull << 30);
    {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(f);
        const int br[4] = {32, 64, 128, 256};
        for (int i = 0; i < 4; ++i) {
            cuuint64_t dims[2] = {64, (1ull << 30) / 128};
            cuuint64_t str[1] = {128};
            cuuint32_t box[2] = {64, (cuuint32_t)br[i]};
            cuuint32_t es[2] = {1, 1};
            CUresult r = enc(&g_tm[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r) printf("enc fail %d\n", (int)r);
            cuuint64_t d2[2] = {4096, (1ull << 30) / 8192};
            cuuint64_t s2[1] = {8192};
            r = enc(&g_tm[4 + i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, d2, s2, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r) printf("enc2 fail %d\n", (int)r);
        }
    }
    unsigned long long* d_out;
    cudaMalloc(&d_out, 8 * 2048);
    run<0, 16384, 8>("bulk distinct 148 SMs", buf, bytes, d_out, nsm);
    run<0, 16384, 4>("bulk distinct 148 SMs", buf, bytes, d_out, nsm);
    run<0, 8192, 8>("bulk distinct 148 SMs", buf, bytes, d_out, nsm);
    run<0, 16384, 8, 32, 2>("bulk distinct 2 producers 148", buf, bytes, d_out, nsm);
    run<1, 16384, 8>("bulk pairs-same 148", buf, bytes, d_out, nsm);
    run<3, 16384, 8>("bulk all-same 148", buf, bytes, d_out, nsm);
    run<4, 16384, 6, 128>("tensor contiguous 148 box128", buf, bytes, d_out, nsm);
    run<4, 32768, 6, 256>("tensor contiguous 148 box256", buf, bytes, d_out, nsm);
    return 0;
}
