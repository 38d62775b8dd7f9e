// pipe_probe.cu -- development microbenchmark of the GEMM's producer/consumer choreography:
// NW "dequant" warps (4 lane quarters x NW/4) write A stages into TMEM and arrive on full[s];
// one MMA warp waits full[s], issues 4 TS MMAs (N), commits to empty[s]; NS stages.
// Variants: ST=0 skips tcgen05.st, WST=0 skips tcgen05.wait::st, PAR=1 splits warps by k parity.
#include <cuda_runtime.h>
#include <stdio.h>
#include "../paper_2602_20191_b200/csrc/sm100.cuh"
using namespace mobi::sm100;

template <int NS, int NW, int ST, int WST, int PAR, int N, int TMA = 0, int BOXR = 32, int NPROD = 1, int CONTIG = 0>
__global__ void __launch_bounds__(32 * (1 + NPROD + NW), 1) pipe(int kblocks, unsigned long long* out,
                                                         const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* bsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[NS], empty[NS], fullb[NS], done;
    __shared__ uint32_t slot;
    const int warp = warp_idx_uniform(), lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < NS * 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(bsm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], PAR ? NW / 2 : NW);
            mbar_init(&empty[s], TMA ? 2 : 1);
            mbar_init(&fullb[s], 1);
        }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        long long t0 = clock64();
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % NS;
            mbar_wait(&full[s], (kb / NS) & 1);
            if (TMA) mbar_wait(&fullb[s], (kb / NS) & 1);
            tc_fence_after();
            if (elect_one_sync()) {
                constexpr uint32_t idesc = idesc_f16(128, N, 0);
                const uint64_t bdesc = sdesc_sw128(smem_u32(bsm + (TMA ? s * 32768 : 0)));
#pragma unroll
                for (int j = 0; j < 4; ++j) mma_ts_f16(0u, 256u + s * 32 + j * 8, bdesc + j * 2, idesc, 1u);
                mma_commit(&empty[s]);
                if (TMA) mma_commit(&empty[s]);  // (count 2 when TMA shares the barrier)
                if (kb == kblocks - 1) mma_commit(&done);
            }
            __syncwarp();
        }
        mbar_wait(&done, 0);
        if (lane == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    } else if (warp >= 1 + NW) {
        if (TMA) {
            for (int kb = warp - 1 - NW; kb < kblocks; kb += NPROD) {
                const int s = kb % NS;
                mbar_wait(&empty[s], ((kb / NS) & 1) ^ 1);
                if (lane == 0) {
                    constexpr int nbox = (N + BOXR - 1) / BOXR;
                    mbar_arrive_expect_tx(&fullb[s], nbox * BOXR * 128);
                    for (int j = 0; j < nbox; ++j)
                        if (CONTIG)
                            tma_load_2d(bsm + s * 32768 + j * BOXR * 128, &tmap, &fullb[s], 0,
                                        ((blockIdx.x * 13 + kb) % 1024) * 256 + j * BOXR);
                        else
                        tma_load_2d(bsm + s * 32768 + j * BOXR * 128, &tmap, &fullb[s], (kb % 64) * 64,
                                    ((blockIdx.x * 13 + kb) % 64) * 256 + j * BOXR);
                }
                __syncwarp();
            }
        }
    } else {
        const int w = warp - 1, q = warp % 4;
        const int grp = w / 4;                 // 0..NW/4-1
        const int par = PAR ? grp % 2 : 0;
        const int ncol = PAR ? 16 : 32 / (NW / 4);
        const int col0 = PAR ? (grp / 2) * 16 : grp * ncol;
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0x3c003c00u;
        for (int kb = par; kb < kblocks; kb += PAR ? 2 : 1) {
            const int s = kb % NS;
            mbar_wait(&empty[s], ((kb / NS) & 1) ^ 1);
            tc_fence_after();
            if (ST) {
                const uint32_t ta = ((uint32_t)(32 * q) << 16) + 256 + s * 32 + col0;
                if (ncol == 16) tmem_st16(ta, v);
                else tmem_st8(ta, *reinterpret_cast<uint32_t(*)[8]>(v));
            }
            if (WST) tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(0, 512);
}


// router-like: TMA loads A (128 rows) and B (NB rows) boxes per stage, one thread issues SS MMAs M=128 N=NB
template <int NS, int NB>
__global__ void __launch_bounds__(64, 1) ss_pipe(int kblocks, unsigned long long* out, const __grid_constant__ CUtensorMap tma,
                                                 const __grid_constant__ CUtensorMap tmb) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[NS], empty[NS], done;
    __shared__ uint32_t slot;
    constexpr int SA = 128 * 128, SB = NB * 128, ST = SA + SB;
    const int warp = warp_idx_uniform();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    long long t0 = clock64();
    if (warp == 0) {
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % NS;
            mbar_wait(&full[s], (kb / NS) & 1);
            tc_fence_after();
            if (elect_one_sync()) {
                constexpr uint32_t idesc = idesc_f16(128, NB, 1);
                const uint32_t a = smem_u32(sm + s * ST);
                const uint64_t ad = sdesc_sw128(a), bd = sdesc_sw128(a + SA);
#pragma unroll
                for (int j = 0; j < 4; ++j) mma_ss_f16(0u, ad + j * 2, bd + j * 2, idesc, (kb | j) != 0);
                mma_commit(&empty[s]);
                if (kb == kblocks - 1) mma_commit(&done);
            }
            __syncwarp();
        }
        mbar_wait(&done, 0);
        if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    } else {
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % NS;
            mbar_wait(&empty[s], ((kb / NS) & 1) ^ 1);
            if (elect_one_sync()) {
                mbar_arrive_expect_tx(&full[s], ST);
                tma_load_2d(sm + s * ST, &tma, &full[s], (kb % 64) * 64, (blockIdx.x % 16) * 128);
                tma_load_2d(sm + s * ST + SA, &tmb, &full[s], (kb % 64) * 64, (blockIdx.x / 16) * NB);
            }
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(0, 512);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned long long* d;
    cudaMalloc(&d, 8 * nsm);
    const int kb = 4096;
    void* buf;
    const long long rows = 64 * 256;
    cudaMalloc(&buf, rows * 4096 * 2);
    cudaMemset(buf, 0, rows * 4096 * 2);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    CUtensorMap tm, tm256, tmc;
    cuuint64_t dims[2] = {4096, (cuuint64_t)rows};
    cuuint64_t strides[1] = {4096 * 2};
    cuuint32_t box[2] = {64, 32};
    cuuint32_t es[2] = {1, 1};
    ((PFN_encodeTiled)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint32_t box256[2] = {64, 256};
    {
        cuuint64_t dc[2] = {64, (cuuint64_t)rows * 64};
        cuuint64_t sc[1] = {128};
        ((PFN_encodeTiled)f)(&tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dc, sc, box256, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    ((PFN_encodeTiled)f)(&tm256, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box256, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto run = [&](auto k, int nthreads, const char* name, int big = 0) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
        k<<<nsm, nthreads + 32, 6 * 32768 + 1024>>>(kb, d, big == 2 ? tmc : big ? tm256 : tm);
        cudaError_t e = cudaGetLastError(); if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
        unsigned long long h[256];
        cudaMemcpy(h, d, 8 * nsm, cudaMemcpyDeviceToHost);
        double a = 0;
        for (int i = 0; i < nsm; ++i) a += h[i];
        printf("%-44s cycles/k-block %7.1f\n", name, a / nsm / kb);
    };
    {
        // X-like [2048][4096] bf16 and w1t-like [1024][4096] bf16, 128-row boxes, strided rows (8 KB pitch)
        CUtensorMap ta, tb, tb256;
        cuuint64_t da[2] = {4096, 2048}, db[2] = {4096, 1024}, st[1] = {8192};
        cuuint32_t b128[2] = {64, 128}, b256[2] = {64, 256};
        auto E = (PFN_encodeTiled)f;
        E(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, da, st, b128, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        E(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (char*)buf + (32 << 20), db, st, b128, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        E(&tb256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (char*)buf + (32 << 20), db, st, b256, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        auto rs = [&](auto k, int smem, const CUtensorMap& b, const char* name, int grid) {
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int w = 0; w < 2; ++w) k<<<grid, 64, smem>>>(64, d, ta, b);
            k<<<grid, 64, smem>>>(64, d, ta, b);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
            unsigned long long h[256];
            cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
            double a = 0;
            for (int i = 0; i < grid; ++i) a += h[i];
            printf("%-44s cycles/k-block %7.1f\n", name, a / grid / 64);
        };
        rs(ss_pipe<6, 128>, 6 * 32768 + 1024, tb, "SS router-like NS6 N128 grid128", 128);
        rs(ss_pipe<4, 256>, 4 * 49152 + 1024, tb256, "SS router-like NS4 N256 grid64", 64);
        rs(ss_pipe<6, 128>, 6 * 32768 + 1024, tb, "SS router-like NS6 N128 grid16", 16);
    }
    return 0;
}
