// hbm_probe.cu -- development microbenchmark: how fast can G CTAs stream S bytes each from HBM (cold,
// buffer >> L2) with one producer thread issuing cp.async.bulk copies of C bytes into a D-deep ring?
// This is the decode GEMV's streaming pattern (one CTA per 32-row tile, a few tens of KiB each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/hbm_probe tools/hbm_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2602_20191_b200/csrc/sm100.cuh"
using namespace mobi::sm100;

__global__ void __launch_bounds__(64, 1) stream(const uint8_t* buf, size_t per_cta, int chunk, int depth, int nprod,
                                                unsigned long long* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[16], empty[16];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < depth; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const uint8_t* src = buf + (size_t)blockIdx.x * per_cta;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int n = (int)(per_cta / chunk);
    if (warp == 0) {
        // producers: lanes 0..nprod-1 each own items it = lane (mod nprod)
        if (lane < nprod)
            for (int it = lane; it < n; it += nprod) {
                const int s = it % depth;
                mbar_wait(&empty[s], ((it / depth) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], chunk);
                bulk_g2s(sm + (size_t)s * chunk, src + (size_t)it * chunk, chunk, &full[s]);
            }
    } else if (lane == 0) {
        for (int it = 0; it < n; ++it) {
            const int s = it % depth;
            mbar_wait(&full[s], (it / depth) & 1);
            mbar_arrive(&empty[s]);
        }
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[2 * blockIdx.x] = t0;
        out[2 * blockIdx.x + 1] = t1;
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t big = 4ull << 30;
    uint8_t* buf;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 1, big);
    uint8_t* flush;
    cudaMalloc(&flush, 512 << 20);
    unsigned long long* d;
    cudaMalloc(&d, 16384);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { int grid; size_t per; int chunk, depth, nprod; };
    const Cfg cfgs[] = {
        {128, 64 << 10, 16 << 10, 4, 1}, {128, 64 << 10, 8 << 10, 8, 1}, {128, 64 << 10, 16 << 10, 4, 2},
        {128, 64 << 10, 16 << 10, 4, 4}, {128, 64 << 10, 4 << 10, 16, 4}, {148, 64 << 10, 16 << 10, 4, 4},
        {296, 32 << 10, 16 << 10, 2, 2}, {128, 128 << 10, 16 << 10, 8, 4}, {148, 1 << 20, 32 << 10, 6, 2},
        {148, 1 << 20, 16 << 10, 12, 4}, {128, 32 << 10, 16 << 10, 2, 2}, {128, 32 << 10, 8 << 10, 4, 4},
    };
    for (const Cfg& c : cfgs) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemsetAsync(flush, rep, 512 << 20);  // evict the buffer from L2
            const size_t off = (size_t)(rep % 4) * (big / 4);
            cudaEventRecord(e0);
            stream<<<c.grid, 64, (size_t)c.chunk * c.depth>>>(buf + off, c.per, c.chunk, c.depth, c.nprod, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            unsigned long long h[1024];
            cudaMemcpy(h, d, 16 * c.grid, cudaMemcpyDeviceToHost);
            unsigned long long lo = ~0ull, hi = 0;
            for (int i = 0; i < c.grid; ++i) lo = h[2 * i] < lo ? h[2 * i] : lo, hi = h[2 * i + 1] > hi ? h[2 * i + 1] : hi;
            const float ms = (hi - lo) * 1e-6f;
            if (ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        const double bytes = (double)c.grid * c.per;
        printf("grid %3d x %7zu B, chunk %6d, depth %2d, producers %d: %7.2f us  %6.2f TB/s\n", c.grid, c.per, c.chunk,
               c.depth, c.nprod, best * 1e3, bytes / (best * 1e-3) / 1e12);
    }
    return 0;
}
