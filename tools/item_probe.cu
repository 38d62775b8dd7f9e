// item_probe.cu -- development microbenchmark: cycles per item of the decode slice-plane GEMV's inner
// body (decode2.cu) with 16 warps per SM: one 16-byte ring read, 4 SHF + 32 LOP3 fragment builds,
// two 16-byte B-fragment reads and 8 mma.sync m16n8k16 in two chains of four.  MODE 0: full body,
// 1: no HMMA, 2: no LOP3 (fragments reused), 3: 4 chains of 2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/item_probe tools/item_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int SS>
__device__ __forceinline__ uint32_t frag(uint32_t w, uint32_t magic) {
    uint32_t r;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "n"(0x00030003u << (2 * SS)), "r"(magic));
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) body(uint32_t* out, int iters) {
    __shared__ uint4 ring[16][4][32];
    __shared__ uint4 xs[16][16];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 16 * 4 * 32; i += 512) (&ring[0][0][0])[i] = make_uint4(i, i * 3, i * 5, i * 7);
    for (int i = threadIdx.x; i < 16 * 16; i += 512) (&xs[0][0])[i] = make_uint4(0x3c003c00u, 0x3c003c00u, i, i);
    __syncthreads();
    float D0[4] = {}, D1[4] = {}, D2[4] = {}, D3[4] = {};
    const uint32_t magic = 0x64006400u;
    long long t0 = clock64();
    int slot = 0;
    for (int it = 0; it < iters; ++it) {
        const uint4 q = ring[warp][slot][lane];
        slot = slot + 1 == 4 ? 0 : slot + 1;
        const uint4 b0 = xs[warp][(lane % 4) * 2 + (it & 1) * 8], b1 = xs[warp][(lane % 4) * 2 + 1 + (it & 1) * 8];
        const uint32_t w0[4] = {q.x, q.y, q.z, q.w};
        const uint32_t w1[4] = {q.x >> 8, q.y >> 8, q.z >> 8, q.w >> 8};
        auto ks = [&](auto SSc, uint32_t bb0, uint32_t bb1) {
            constexpr int S = decltype(SSc)::value;
            uint32_t a[8];
            if (MODE == 2) {
                for (int i = 0; i < 4; ++i) a[i] = w0[i], a[4 + i] = w1[i];
            } else {
                for (int i = 0; i < 4; ++i) a[i] = frag<S>(w0[i], magic), a[4 + i] = frag<S>(w1[i], magic);
            }
            if (MODE == 1) {
                D0[0] += __uint_as_float(a[0] ^ a[1] ^ a[2] ^ a[3] ^ bb0);
                D1[0] += __uint_as_float(a[4] ^ a[5] ^ a[6] ^ a[7] ^ bb1);
            } else if (MODE == 3 && (S & 1)) {
                mma(D2, a[0], a[1], a[2], a[3], bb0, bb1);
                mma(D3, a[4], a[5], a[6], a[7], bb0, bb1);
            } else {
                mma(D0, a[0], a[1], a[2], a[3], bb0, bb1);
                mma(D1, a[4], a[5], a[6], a[7], bb0, bb1);
            }
        };
        ks(std::integral_constant<int, 0>{}, b0.x, b0.y);
        ks(std::integral_constant<int, 1>{}, b0.z, b0.w);
        ks(std::integral_constant<int, 2>{}, b1.x, b1.y);
        ks(std::integral_constant<int, 3>{}, b1.z, b1.w);
    }
    long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < 4; ++j) s += D0[j] + D1[j] + D2[j] + D3[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(s);
    if (threadIdx.x == 0) out[(1 << 20) + blockIdx.x] = (uint32_t)(t1 - t0);
}

template <int MODE>
void run(const char* name, uint32_t* d) {
    const int iters = 2048;
    body<MODE><<<148, 512>>>(d, iters);
    cudaDeviceSynchronize();
    body<MODE><<<148, 512>>>(d, iters);
    cudaDeviceSynchronize();
    uint32_t cyc;
    cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
    printf("%-40s %7.1f cycles per item per warp (16 warps/SM), %s\n", name, (double)cyc / iters,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, (2 << 20) * 4);
    run<0>("full body (2 chains x 4 HMMA)", d);
    run<1>("no HMMA", d);
    run<2>("no LOP3", d);
    run<3>("4 chains x 2 HMMA", d);
    return 0;
}
