// bucket.cu -- K2: route decisions + stable bucketing + permuted activation gather.
//
//   gate_hard (router.hpp:93-97):   G[t,j] = 1((S[t,j] - delta) > 0), strict
//   mask convention (bitplane.hpp:203-206): mask_t = 1 | sum_j G[t,j] << (j+1)
//   permute_by_slice (bitplane.hpp:178-201): stable sort of tokens by mask, ascending
//
// bucket_kernel: one CTA of 1024 threads; a stable counting sort (key histogram, then ranks
// of equal keys in token order), so every token gets exactly std::stable_sort's position.
// Two orders are written: the compact one (the reference's `perm`/`inverse`) and the padded
// one the GEMM consumes, where every bucket starts on a kBucketAlign boundary so a token
// tile never mixes masks.  It also emits the GEMM's token-tile list (bucket mask, first row,
// valid rows), so no host round trip is needed between routing and the GEMM.
//
// gather_kernel: one CTA per token copies X[t] (bf16) into xperm[pinv[t]] (fp16) scaled
// by a per-row power of two 2^-e (max|x| lands in [2^14, 2^15)); the GEMM epilogue multiplies
// by 2^e.  The scaling is exact, so fp16 operands lose nothing against the bf16 input.
#include "mobi_internal.cuh"

namespace mobi {
namespace {

constexpr int BK_THREADS = 1024;
constexpr int NKEY_ALL = 256;              // generic uint8 keys (permute_by_slice API)
constexpr int NKEY_MASK = 2 * kMaxBuckets;  // slice masks on the GEMM path (< 2^MOBI_MAX_SLICES)

// Stable counting sort on one CTA.  Keys are processed in chunks of 1024 tokens in token
// order; inside a chunk, __match_any_sync ranks equal keys within a warp and a per-key scan
// over the 32 warps orders the warps, so every token's position equals std::stable_sort's.
template <int NKEY>
__global__ void __launch_bounds__(BK_THREADS) bucket_kernel(
    const float* __restrict__ s_part, int htiles, int64_t T, int nr, const float* __restrict__ b2,
    float delta, const uint8_t* __restrict__ given_masks, int sanitize, float* __restrict__ scores_out,
    uint8_t* __restrict__ keys, uint8_t* __restrict__ masks_out, int32_t* __restrict__ perm,
    int64_t tpad_max, int32_t* __restrict__ cperm_out, int32_t* __restrict__ inverse_out,
    int32_t* __restrict__ counts_out, TokTile* __restrict__ tiles, int32_t* __restrict__ meta,
    int32_t* __restrict__ pinv) {
    __shared__ int hist[NKEY], cstart[NKEY], run[NKEY], pstart[NKEY_MASK];
    __shared__ int warp_hist[BK_THREADS / 32][NKEY];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int vmask = (1 << (nr + 1)) - 1;
    if (perm)
        for (int64_t i = tid; i < tpad_max; i += BK_THREADS) perm[i] = -1;
    if (tid < NKEY) {
        hist[tid] = 0;
        run[tid] = 0;
    }
    __syncthreads();
    // phase 1: decisions (gate_hard strict '>' on delta) and the key histogram
    for (int64_t t = tid; t < T; t += BK_THREADS) {
        int m;
        if (given_masks) {
            m = given_masks[t];
            if (sanitize) m = (m & vmask) | 1;
        } else {
            m = 1;
            for (int k = 0; k < nr; ++k) {
                float s = 0.f;
                for (int q = 0; q < htiles; ++q) s += s_part[((int64_t)q * T + t) * nr + k];
                s += b2[k];
                if (scores_out) scores_out[t * nr + k] = s;
                if ((s - delta) > 0.f) m |= 1 << (k + 1);
            }
        }
        keys[t] = (uint8_t)m;
        if (masks_out) masks_out[t] = (uint8_t)m;
        atomicAdd(&hist[m], 1);
    }
    __syncthreads();
    // phase 2: bucket starts (compact = reference order; padded = GEMM order) and token tiles
    if (tid == 0) {
        int c = 0;
        for (int v = 0; v < NKEY; ++v) {
            cstart[v] = c;
            c += hist[v];
            if (counts_out) counts_out[v] = hist[v];
        }
        if (perm) {
            // token tiles, largest first (the GEMM claims them dynamically in this order)
            int a = 0, n = 0;
            for (int v = 0; v < NKEY_MASK && v < NKEY; ++v) {
                pstart[v] = a;
                for (int j = 0; j < hist[v]; j += kTokTile) {
                    TokTile tt;
                    tt.row0 = a + j;
                    tt.n = min(kTokTile, hist[v] - j);
                    tt.mask = v;
                    tt.pad = 0;
                    int i = n++;
                    while (i > 0 && tiles[i - 1].n < tt.n) {
                        tiles[i] = tiles[i - 1];
                        --i;
                    }
                    tiles[i] = tt;
                }
                a += (int)round_up(hist[v], kBucketAlign);
            }
            meta[0] = n;
            meta[1] = a;
            for (int v = 0; v < NKEY_MASK && v < NKEY; ++v) meta[2 + v] = hist[v];
            meta[32] = 0;  // GEMM dynamic tile counter
            meta[33] = 1;  // GEMM split count (the GEMM overwrites it when it splits K)
        }
    }
    __syncthreads();
    // phase 3: stable positions
    for (int64_t base = 0; base < T; base += BK_THREADS) {
        for (int i = tid; i < (BK_THREADS / 32) * NKEY; i += BK_THREADS) (&warp_hist[0][0])[i] = 0;
        __syncthreads();
        const int64_t t = base + tid;
        const bool valid = t < T;
        const int key = valid ? keys[t] : NKEY;  // NKEY never matches a real key
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && rank == 0) warp_hist[wid][key] = __popc(peers);
        __syncthreads();
        if (tid < NKEY) {
            int r = run[tid];
            for (int w = 0; w < BK_THREADS / 32; ++w) {
                const int cnt = warp_hist[w][tid];
                warp_hist[w][tid] = r;
                r += cnt;
            }
            run[tid] = r;
        }
        __syncthreads();
        if (valid) {
            const int off = warp_hist[wid][key] + rank;
            const int cpos = cstart[key] + off;
            if (perm && key < NKEY_MASK) {
                perm[pstart[key] + off] = (int32_t)t;
                pinv[t] = pstart[key] + off;
            }
            if (cperm_out) cperm_out[cpos] = (int32_t)t;
            if (inverse_out) inverse_out[t] = cpos;
        }
        __syncthreads();
    }
}

// One CTA per token t: write its permuted row pinv[t].  Padding rows between buckets are never
// written: the GEMM only ever reads them as B columns whose outputs it discards.
__global__ void __launch_bounds__(128) gather_kernel(const __nv_bfloat16* __restrict__ x, int64_t in,
                                                     int64_t in_pad, int64_t tpad, const int32_t* __restrict__ pinv,
                                                     __half* __restrict__ xperm, float* __restrict__ escale,
                                                     bool vec) {
    __shared__ float red[4];
    const int64_t src = blockIdx.x;
    const int64_t i = pinv[src];
    // k-block slab layout [in_pad/64][tpad][64]: element k of permuted row i at (k/64*tpad + i)*64 + k%64
    __half* dst = xperm + i * kKBlock;
    auto at = [&](int64_t k) { return dst + (k / kKBlock) * tpad * kKBlock + (k % kKBlock); };
    const __nv_bfloat16* row = x + (int64_t)src * in;
    float m = 0.f;
    if (vec) {
        for (int64_t k = threadIdx.x * 8; k < in; k += 128 * 8) {
            uint4 q = __ldg(reinterpret_cast<const uint4*>(row + k));
            const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float2 f = __bfloat1622float2(p[j]);
                m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
            }
        }
    } else {
        for (int64_t k = threadIdx.x; k < in; k += 128) m = fmaxf(m, fabsf(__bfloat162float(row[k])));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    int e = 0;
    if (m > 0.f && isfinite(m)) e = ilogbf(m) - 14;
    const float sc = ldexpf(1.f, -e);
    if (threadIdx.x == 0) escale[i] = ldexpf(1.f, e);
    if (vec) {
        for (int64_t k = threadIdx.x * 8; k < in_pad; k += 128 * 8) {
            uint4 o = make_uint4(0, 0, 0, 0);
            if (k < in) {
                uint4 q = __ldg(reinterpret_cast<const uint4*>(row + k));
                const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q);
                __half2* h = reinterpret_cast<__half2*>(&o);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float2 f = __bfloat1622float2(p[j]);
                    h[j] = __floats2half2_rn(f.x * sc, f.y * sc);
                }
            }
            *reinterpret_cast<uint4*>(at(k)) = o;
        }
    } else {
        for (int64_t k = threadIdx.x; k < in_pad; k += 128)
            *at(k) = __float2half_rn(k < in ? __bfloat162float(row[k]) * sc : 0.f);
    }
}

}  // namespace

int launch_bucket(mobi_layer* L, int64_t T, float delta, const uint8_t* given_masks,
                  float* scores_out, uint8_t* masks_out, int32_t* cperm_out, int32_t* inverse_out,
                  int32_t* counts_out, cudaStream_t st) {
    bucket_kernel<NKEY_MASK><<<1, BK_THREADS, 0, st>>>(L->s_part, (int)L->htiles, T, L->nr, L->b2, delta,
                                             given_masks, 1, scores_out, L->masks, masks_out, L->perm,
                                             L->tpad_max, cperm_out, inverse_out, counts_out, L->tiles,
                                             L->meta, L->pinv);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    return MOBI_OK;
}

int launch_permute(const uint8_t* masks, int64_t T, uint8_t* keys_tmp, int32_t* cperm, int32_t* inverse,
                   int32_t* hist256, cudaStream_t st) {
    bucket_kernel<NKEY_ALL><<<1, BK_THREADS, 0, st>>>(nullptr, 0, T, 0, nullptr, 0.f, masks, 0, nullptr, keys_tmp,
                                             nullptr, nullptr, 0, cperm, inverse, hist256, nullptr, nullptr, nullptr);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

int launch_gather(mobi_layer* L, const __nv_bfloat16* x, int64_t T, cudaStream_t st) {
    const bool vec = (L->in % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    gather_kernel<<<(unsigned)T, 128, 0, st>>>(x, L->in, L->in_pad, L->tpad_max, L->pinv, L->xperm, L->escale, vec);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    return MOBI_OK;
}

}  // namespace mobi
