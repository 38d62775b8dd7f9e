// router.cu -- K1: the MoBiRoute scorer S = silu(X w1 + b1) w2 + b2 (router.hpp:63-76).
//
// The hidden GEMM X[T,in] x w1[in,h] runs on bf16 operands with fp32 accumulation; the SiLU
// and the tiny second layer (h x (E-1)) are fused into the epilogue, which writes one fp32
// partial score per (hidden tile, token, routed slice).  K2 (bucket.cu) reduces the partials
// in a fixed order, so the scores are deterministic run to run and rank to rank (no atomics).
#include "mobi_internal.cuh"

namespace mobi {
namespace {

constexpr int RT_TOK = 64, RT_HID = 64, RT_K = 32;

__global__ void __launch_bounds__(256) router_simt_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t T, int64_t in, const __nv_bfloat16* __restrict__ w1t,
    int64_t in_pad, int64_t h, const float* __restrict__ b1, const float* __restrict__ w2, int nr,
    float* __restrict__ s_part) {
    __shared__ float xs[RT_K][RT_TOK + 4];
    __shared__ float ws[RT_K][RT_HID + 4];
    __shared__ float red[RT_TOK][16][MOBI_MAX_SLICES - 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t t0 = (int64_t)blockIdx.x * RT_TOK;
    const int64_t h0 = (int64_t)blockIdx.y * RT_HID;
    float acc[4][4] = {};
    for (int64_t k0 = 0; k0 < in; k0 += RT_K) {
        for (int i = threadIdx.x; i < RT_TOK * RT_K; i += 256) {
            const int tt = i / RT_K, kk = i % RT_K;
            const int64_t t = t0 + tt, k = k0 + kk;
            xs[kk][tt] = (t < T && k < in) ? __bfloat162float(x[t * in + k]) : 0.f;
            const int64_t j = h0 + tt;
            ws[kk][tt] = (j < h && k < in) ? __bfloat162float(w1t[j * in_pad + k]) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < RT_K; ++kk) {
            float a[4], bb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) a[q] = xs[kk][ty * 4 + q];
#pragma unroll
            for (int q = 0; q < 4; ++q) bb[q] = ws[kk][tx * 4 + q];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
        __syncthreads();
    }
    // epilogue: silu(acc + b1) . w2 over this thread's 4 hidden units
    for (int i = 0; i < 4; ++i) {
        float p[MOBI_MAX_SLICES - 1] = {};
        for (int j = 0; j < 4; ++j) {
            const int64_t hj = h0 + tx * 4 + j;
            if (hj >= h) continue;
            const float v = silu_f(acc[i][j] + b1[hj]);
            for (int k = 0; k < nr; ++k) p[k] = fmaf(v, w2[hj * nr + k], p[k]);
        }
        for (int k = 0; k < nr; ++k) red[ty * 4 + i][tx][k] = p[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < RT_TOK * nr; i += 256) {
        const int tt = i / nr, k = i % nr;
        const int64_t t = t0 + tt;
        if (t >= T) continue;
        float s = 0.f;
        for (int q = 0; q < 16; ++q) s += red[tt][q][k];
        s_part[((int64_t)blockIdx.y * T + t) * nr + k] = s;
    }
}

}  // namespace

int launch_router(mobi_layer* L, const __nv_bfloat16* x, int64_t T, cudaStream_t st) {
    dim3 grid((unsigned)cdiv(T, RT_TOK), (unsigned)cdiv(L->h, RT_HID));
    L->htiles = grid.y;
    router_simt_kernel<<<grid, 256, 0, st>>>(x, T, L->in, L->w1t, L->in_pad, L->h, L->b1, L->w2,
                                             L->nr, L->s_part);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    L->plan[0] = MOBI_K_ROUTER_SIMT;
    return MOBI_OK;
}

}  // namespace mobi
