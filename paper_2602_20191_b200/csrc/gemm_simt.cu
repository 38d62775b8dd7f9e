// gemm_simt.cu -- CUDA-core reference version of the nested residual GEMM (K3), used only by
// the test-suite as a second implementation to cross-check the tcgen05 kernel (gemm_tc.cu).
// Same inputs (tiled merged codes, fp16 permuted activations), same fp16 dequantization
// (mobi::dequant4), fp32 accumulation, same fused un-permute epilogue.
#include "mobi_internal.cuh"

namespace mobi {
namespace {

constexpr int SM_ROWS = 64, SM_TOK = 64;

__global__ void __launch_bounds__(256) gemm_simt_kernel(
    const uint8_t* __restrict__ codes8, const float2* __restrict__ gconst, int64_t out_pad,
    MaskTable mt, int64_t out, int64_t G, int64_t gs,
    bool single_group, int64_t kblocks, int64_t tpad, const __half* __restrict__ xperm,
    const float* __restrict__ escale, const int32_t* __restrict__ perm,
    const TokTile* __restrict__ tiles, const int32_t* __restrict__ meta,
    __nv_bfloat16* __restrict__ y) {
    if ((int)blockIdx.y >= meta[0]) return;
    const TokTile tile = tiles[blockIdx.y];
    const int sub0 = blockIdx.z * SM_TOK;
    if (sub0 >= tile.n) return;
    __shared__ float ws[kKBlock][SM_ROWS + 4];
    __shared__ float xs[kKBlock][SM_TOK + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t R0 = (int64_t)blockIdx.x * SM_ROWS;
    const int rl = tid % SM_ROWS, q = tid / SM_ROWS;  // loader: row, 16-code chunk
    const int64_t R = R0 + rl;
    const uint32_t mw = mt.maskword[tile.mask];
    const float kc = mt.kc[tile.mask];
    float acc[4][4] = {};
    for (int64_t kb = 0; kb < kblocks; ++kb) {
        {  // weights: 16 codes of row R -> ws[k][row]
            const int64_t k0 = kb * kKBlock + q * 16;
            uint4 c4 = *reinterpret_cast<const uint4*>(codes8 + code_offset(R, k0, kblocks));
            float s = 0.f, sz = 0.f;
            if (R < out) {
                const int64_t g = single_group ? 0 : k0 / gs;
                const float2 c = gconst[g * out_pad + R];
                s = c.x;
                sz = c.y;
            }
            const __half2 S2 = __float2half2_rn(s * mt.inv_2p);
            const __half2 C2 = __float2half2_rn(fmaf(s, kc, -sz));
            const uint32_t* cw = reinterpret_cast<const uint32_t*>(&c4);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                uint32_t w01, w23;
                dequant4(cw[w], mw, S2, C2, w01, w23);
                float2 f01 = __half22float2(*reinterpret_cast<__half2*>(&w01));
                float2 f23 = __half22float2(*reinterpret_cast<__half2*>(&w23));
                ws[q * 16 + w * 4 + 0][rl] = f01.x;
                ws[q * 16 + w * 4 + 1][rl] = f01.y;
                ws[q * 16 + w * 4 + 2][rl] = f23.x;
                ws[q * 16 + w * 4 + 3][rl] = f23.y;
            }
        }
        for (int i = tid; i < SM_TOK * kKBlock; i += 256) {  // activations
            const int tt = i / kKBlock, kk = i % kKBlock;
            const int64_t row = tile.row0 + sub0 + tt;
            xs[kk][tt] = (sub0 + tt < tile.n) ? __half2float(xperm[(kb * tpad + row) * kKBlock + kk]) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < kKBlock; ++kk) {
            float a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = ws[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = xs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
        __syncthreads();
    }
    for (int j = 0; j < 4; ++j) {
        const int tt = sub0 + tx * 4 + j;
        if (tt >= tile.n) continue;
        const int64_t row = tile.row0 + tt;
        const int32_t src = perm[row];
        if (src < 0) continue;
        const float es = escale[row];
        for (int i = 0; i < 4; ++i) {
            const int64_t Rr = R0 + ty * 4 + i;
            if (Rr < out) y[(int64_t)src * out + Rr] = __float2bfloat16_rn(acc[i][j] * es);
        }
    }
}

}  // namespace

int launch_gemm_simt(mobi_layer* L, __nv_bfloat16* y, int64_t T, cudaStream_t st) {
    dim3 grid((unsigned)(L->out_pad / SM_ROWS), (unsigned)L->max_tiles, kTokTile / SM_TOK);
    gemm_simt_kernel<<<grid, 256, 0, st>>>(L->codes8, L->gconst, L->out_pad, L->mtab, L->out, L->G, L->gs,
                                           L->single_group, L->kblocks, L->tpad_max, L->xperm, L->escale,
                                           L->perm, L->tiles, L->meta, y);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    L->plan[1] = MOBI_K_GEMM_SIMT;
    L->plan[2] = (int32_t)(grid.x * grid.y * grid.z);
    return MOBI_OK;
}

}  // namespace mobi
