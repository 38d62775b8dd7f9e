// gemm_generic.cu -- forward_elastic (router.hpp:105-132) for slice layouts the folded-weight kernels
// cannot take: non-uniform widths or more than kFastSlices slices (any widths with sum <= 8 bits,
// config.hpp:143-182).  With unequal widths the merged code INT is not the sum of the slices' scaled
// codes, so there is no single AND-masked effective weight per bucket; instead every slice is
// dequantized on its own (slice_params, slicer.hpp:51-61; reconstruct_frame, slicer.hpp:118-131):
//     W_1 = s ((c_1 + 1/2) - z)
//     W_e = s 2^-P_e (c_e - 2^(b_e - 1) + 1/2),   P_e = b_1 + ... + b_(e-1)
// and contracted on CUDA cores, each slice's contribution added only for the tokens whose mask has
// it:  Y = X W_1^T + sum_(e>=2) diag(G[:, e-2]) X W_e^T  (gating applied to the activations).
// fp32 arithmetic throughout; one CTA per (64 rows, 64 tokens) tile, no bucketing or permutation.
#include "mobi_internal.cuh"

namespace mobi {
namespace {

constexpr int GT_ROWS = 64, GT_TOK = 64, GT_K = 32;

__global__ void __launch_bounds__(256) gemm_generic_kernel(
    const uint8_t* __restrict__ codes8, const float2* __restrict__ gconst, int64_t out_pad, int64_t out, int64_t in,
    int64_t kblocks, int64_t gs, int single_group, SliceLayout sl, const __nv_bfloat16* __restrict__ x, int64_t T,
    const uint8_t* __restrict__ masks, __nv_bfloat16* __restrict__ y) {
    __shared__ float ws[GT_K][GT_ROWS + 4];
    __shared__ float xs[GT_K][GT_TOK + 4];
    __shared__ int tmask[GT_TOK];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int64_t R0 = (int64_t)blockIdx.x * GT_ROWS, t0 = (int64_t)blockIdx.y * GT_TOK;
    if (tid < GT_TOK) tmask[tid] = t0 + tid < T ? masks[t0 + tid] : 0;
    float acc[4][4] = {};
    int P = 0;  // bits of the slices before e
    for (int e = 0; e < sl.E; ++e) {
        const float pe = ldexpf(1.f, -P);
        const float ze = e == 0 ? 0.f : (float)(1 << (sl.b[e] - 1)) - 0.5f;
        const unsigned fm = (1u << sl.b[e]) - 1u;
        for (int64_t k0 = 0; k0 < in; k0 += GT_K) {
            __syncthreads();  // the previous k-chunk's tiles are consumed
            for (int i = tid; i < GT_ROWS * GT_K; i += 256) {
                const int r = i / GT_K, kk = i % GT_K;
                const int64_t R = R0 + r, k = k0 + kk;
                float w = 0.f;
                if (R < out && k < in) {
                    const unsigned c = (codes8[code_offset(R, k, kblocks)] >> sl.off[e]) & fm;
                    const float2 sc = gconst[(single_group ? 0 : k / gs) * out_pad + R];  // (s, s z)
                    w = e == 0 ? fmaf(sc.x, (float)c + 0.5f, -sc.y) : sc.x * pe * ((float)c - ze);
                }
                ws[kk][r] = w;
            }
            for (int i = tid; i < GT_TOK * GT_K; i += 256) {
                const int tt = i / GT_K, kk = i % GT_K;
                const int64_t t = t0 + tt, k = k0 + kk;
                const bool on = t < T && k < in && (e == 0 || ((tmask[tt] >> e) & 1));
                xs[kk][tt] = on ? __bfloat162float(x[t * in + k]) : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int kk = 0; kk < GT_K; ++kk) {
                float a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = ws[kk][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = xs[kk][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
        }
        P += sl.b[e];
    }
    for (int j = 0; j < 4; ++j) {
        const int64_t t = t0 + tx * 4 + j;
        if (t >= T) continue;
        for (int i = 0; i < 4; ++i) {
            const int64_t R = R0 + ty * 4 + i;
            if (R < out) y[t * out + R] = __float2bfloat16_rn(acc[i][j]);
        }
    }
}

}  // namespace

int launch_gemm_generic(mobi_layer* L, const __nv_bfloat16* x, int64_t T, const uint8_t* masks, __nv_bfloat16* y,
                        cudaStream_t st) {
    if (T <= 0) return MOBI_OK;
    dim3 grid((unsigned)cdiv(L->out, (int64_t)GT_ROWS), (unsigned)cdiv(T, (int64_t)GT_TOK));
    gemm_generic_kernel<<<grid, 256, 0, st>>>(L->codes8, L->gconst, L->out_pad, L->out, L->in, L->kblocks, L->gs,
                                              L->single_group ? 1 : 0, L->sl, x, T, masks, y);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    L->plan[1] = MOBI_K_GEMM_GENERIC;
    L->plan[2] = (int32_t)(grid.x * grid.y);
    return MOBI_OK;
}

}  // namespace mobi
