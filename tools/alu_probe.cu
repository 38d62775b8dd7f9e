// alu_probe.cu -- development microbenchmark: SM throughput of PRMT (__byte_perm) vs LOP3/SHF byte
// extraction, FADD/FFMA, and mma.sync m16n8k16, in warp-instructions per cycle per SM.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

template <int OP>
__global__ void __launch_bounds__(256) k(uint32_t* out, int iters) {
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7919u + i * 104729u;
    float f[8];
    for (int i = 0; i < 8; ++i) f[i] = (float)a[i];
    float acc[4] = {0, 0, 0, 0}, acc2[4][4] = {};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = __byte_perm(a[i], 0x64646464u, 0x4140 + (i & 1));
            if (OP == 1) a[i] = (a[i] & 0x00FF00FFu) | 0x64006400u ^ it;
            if (OP == 2) a[i] = ((a[i] >> 8) & 0x00FF00FFu) | 0x64006400u;
            if (OP == 3) f[i] = fmaf(f[i], 1.0001f, 0.5f);
        }
        if (OP == 4) {
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]));
        }
        if (OP == 5) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(acc2[c][0]), "+f"(acc2[c][1]), "+f"(acc2[c][2]), "+f"(acc2[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]));
        }
    }
    long long t1 = clock64();
    for (int c = 0; c < 4; ++c) acc[c] += acc2[c][0] + acc2[c][1] + acc2[c][2] + acc2[c][3];
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + __float_as_uint(f[i]);
    s += __float_as_uint(acc[0] + acc[1] + acc[2] + acc[3]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) out[1 << 20 | blockIdx.x] = (uint32_t)(t1 - t0);
}

template <int OP>
void run(const char* name, uint32_t* d, int per_instr) {
    const int iters = 4096;
    k<OP><<<148, 256>>>(d, iters);
    cudaDeviceSynchronize();
    k<OP><<<148, 256>>>(d, iters);
    cudaDeviceSynchronize();
    uint32_t cyc;
    cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
    const double warp_instr = 8.0 * iters * per_instr;  // per warp, 8 warps per SM
    printf("%-34s %8.2f warp-instr/cycle/SM\n", name, warp_instr * 8 / cyc);
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, (2 << 20) * 4);
    run<0>("PRMT", d, 1);
    run<1>("LOP3 (and|or)", d, 1);
    run<2>("SHF+LOP3", d, 2);
    run<3>("FFMA", d, 1);
    cudaError_t e = cudaGetLastError();
    k<4><<<148, 256>>>(d, 4096);
    cudaDeviceSynchronize();
    uint32_t cyc;
    cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
    printf("%-34s %8.2f HMMA/cycle/SM (dependent chain per warp, 8 warps)\n", "mma.sync m16n8k16", 4096.0 * 8 / cyc);
    k<5><<<148, 256>>>(d, 1024);
    cudaDeviceSynchronize();
    cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
    printf("%-34s %8.2f HMMA/cycle/SM (4 independent chains per warp, 8 warps)\n", "mma.sync m16n8k16", 1024.0 * 4 * 8 / cyc);
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
