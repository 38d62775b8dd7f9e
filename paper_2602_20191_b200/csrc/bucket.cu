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
// by 2^e.  The scaling is exact for every element within 2^29 of the row's maximum (fp16's normal
// range below 2^15); smaller elements become fp16 subnormals or zero, a perturbation below 2^-24 of the
// row's largest term.
#include "mobi_internal.cuh"
#include "sm100.cuh"

namespace mobi {
namespace {

constexpr int BK_THREADS = 1024;
constexpr int NKEY_ALL = 256;              // generic uint8 keys (permute_by_slice API)
constexpr int NKEY_MASK = 2 * kMaxBuckets;  // slice masks on the GEMM path (< 2^MOBI_MAX_SLICES)
constexpr int kMaxTilesSmem = 1024;          // token tiles (T <= ~256K tokens per call)

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
    __shared__ int4 s_tiles[NKEY == NKEY_MASK ? kMaxTilesSmem : 1];
    __shared__ int s_ntiles;
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
    for (int64_t t0 = 0; t0 < T; t0 += BK_THREADS) {
        const int64_t t = t0 + tid;
        int m = NKEY;  // out of range: never counted
        if (t >= T) {
        } else if (given_masks) {
            m = given_masks[t];
            if (sanitize) m = (m & vmask) | 1;
        } else {
            m = 1;
            for (int k = 0; k < nr; ++k) {
                // fixed hidden-tile order (the same sum the router's fused decision computes)
                float s = 0.f;
#pragma unroll 8
                for (int j = 0; j < htiles; ++j) s += s_part[((int64_t)j * T + t) * nr + k];
                s += b2[k];
                if (scores_out) scores_out[t * nr + k] = s;
                if ((s - delta) > 0.f) m |= 1 << (k + 1);
            }
        }
        if (t < T) {
            keys[t] = (uint8_t)m;
            if (masks_out) masks_out[t] = (uint8_t)m;
        }
        // warp-aggregated histogram update (most tokens share a handful of masks)
        const unsigned peers = __match_any_sync(0xffffffffu, m);
        if (m < NKEY && lane == __ffs(peers) - 1) atomicAdd(&hist[m], __popc(peers));
    }
    __syncthreads();
    // phase 2: bucket starts (compact = reference order; padded = GEMM order) and the token-tile
    // list, built in shared memory by warp 0: full tiles in key order, then the partial last tiles of
    // each bucket largest first (the GEMM schedules tiles in list order)
    if (wid == 0) {
        // exclusive scans over the keys, 32 keys per step
        int c = 0, a = 0;
        for (int v0 = 0; v0 < NKEY; v0 += 32) {
            const int v = v0 + lane;
            const int h = v < NKEY ? hist[v] : 0;
            const int hp = (v < NKEY_MASK) ? (int)round_up(h, kBucketAlign) : 0;
            int incl = h, inclp = hp;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o), yp = __shfl_up_sync(0xffffffffu, inclp, o);
                if (lane >= o) incl += y, inclp += yp;
            }
            if (v < NKEY) {
                cstart[v] = c + incl - h;
                if (counts_out) counts_out[v] = h;
            }
            if (v < NKEY_MASK) pstart[v] = a + inclp - hp;
            c += __shfl_sync(0xffffffffu, incl, 31);
            a += __shfl_sync(0xffffffffu, inclp, 31);
        }
        __syncwarp();  // lane 0 reads every lane's pstart[] below (racecheck: intra-warp hazard)
        if (perm && lane == 0) {
            int n = 0;
            for (int v = 0; v < NKEY_MASK && v < NKEY; ++v)
                for (int j = 0; j + kTokTile <= hist[v]; j += kTokTile) s_tiles[n++] = make_int4(pstart[v] + j, kTokTile, v, 0);
            const int nfull = n;
            for (int v = 0; v < NKEY_MASK && v < NKEY; ++v) {
                const int r = hist[v] % kTokTile;
                if (!r) continue;
                int i = n++;
                while (i > nfull && s_tiles[i - 1].y < r) {
                    s_tiles[i] = s_tiles[i - 1];
                    --i;
                }
                s_tiles[i] = make_int4(pstart[v] + hist[v] - r, r, v, 0);
            }
            s_ntiles = n;
            meta[0] = n;
            meta[1] = a;
            meta[32] = 0;  // GEMM dynamic tile counter
            meta[33] = 1;  // GEMM split count (the GEMM overwrites it when it splits K)
        }
        if (perm && lane < NKEY_MASK && lane < NKEY) meta[2 + lane] = hist[lane];
    }
    __syncthreads();
    if (perm)
        for (int i = tid; i < s_ntiles; i += BK_THREADS) {
            const int4 v = s_tiles[i];
            TokTile tt;
            tt.row0 = v.x;
            tt.n = v.y;
            tt.mask = v.z;
            tt.pad = 0;
            tiles[i] = tt;
        }
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
// Padded bucket starts from the mask histogram (every bucket on a kBucketAlign boundary).
__device__ __forceinline__ int bucket_start(const int* hist, int m) {
    int a = 0;
    for (int v = 0; v < m; ++v) a += (int)round_up(__ldg(hist + v), kBucketAlign);
    return a;
}

// One thread: the GEMM token-tile list (full tiles in mask order, then each bucket's partial last
// tile, largest first) and meta -- the same layout bucket_kernel produces.
__device__ void build_tiles(const int* hist, TokTile* tiles, int32_t* meta) {
    int h[2 * kMaxBuckets], st[2 * kMaxBuckets];
    int a = 0;
    for (int v = 0; v < 2 * kMaxBuckets; ++v) {
        h[v] = __ldg(hist + v);
        st[v] = a;
        a += (int)round_up(h[v], kBucketAlign);
    }
    int n = 0;
    for (int v = 0; v < 2 * kMaxBuckets; ++v)
        for (int j = 0; j + kTokTile <= h[v]; j += kTokTile) tiles[n++] = TokTile{st[v] + j, kTokTile, v, 0};
    unsigned done = 0;
    for (;;) {  // partial tiles, largest first (ties: lower mask first)
        int best = -1, br = 0;
        for (int v = 0; v < 2 * kMaxBuckets; ++v) {
            const int r = h[v] % kTokTile;
            if (r && !(done >> v & 1u) && r > br) best = v, br = r;
        }
        if (best < 0) break;
        done |= 1u << best;
        tiles[n++] = TokTile{st[best] + h[best] - br, br, best, 0};
    }
    for (int v = 0; v < 2 * kMaxBuckets; ++v) meta[2 + v] = h[v];
    meta[0] = n;
    meta[1] = a;
    meta[32] = 0;  // GEMM dynamic tile counter
    meta[33] = 1;  // GEMM split count
}

__global__ void __launch_bounds__(128, 16) gather_kernel(const __nv_bfloat16* __restrict__ x, int64_t in,
                                                     int64_t in_pad, int64_t tpad, int32_t* __restrict__ pinv,
                                                     __half* __restrict__ xperm, float* __restrict__ escale,
                                                     bool vec, const uint8_t* __restrict__ masks,
                                                     const int* __restrict__ hist, int* __restrict__ fill,
                                                     int32_t* __restrict__ perm, TokTile* __restrict__ tiles,
                                                     int32_t* __restrict__ meta) {
    __shared__ float red[4];
    __shared__ int s_row;
    __shared__ uint64_t s_bar;
    // vec: the row (bf16, in % 8 == 0) lands in shared memory with one bulk copy issued before the grid
    // dependency resolves (an input, not a router output).  Staging in shared memory instead of registers
    // keeps the kernel at ~30 registers, so the whole batch's CTAs are resident in one wave (2048 tokens:
    // 14 per SM) and every row read is in flight at once.
    extern __shared__ __align__(16) uint8_t g_row[];
    const int64_t src = blockIdx.x;
    sm100::pdl_trigger();
    const __nv_bfloat16* row = x + (int64_t)src * in;
    const __nv_bfloat16* srow = reinterpret_cast<const __nv_bfloat16*>(g_row);
    float m = 0.f;
    if (vec) {
        if (threadIdx.x == 0) {
            sm100::mbar_init(&s_bar, 1);
            sm100::fence_barrier_init();
            sm100::mbar_arrive_expect_tx(&s_bar, (uint32_t)(in * 2));
            sm100::bulk_g2s(g_row, row, (uint32_t)(in * 2), &s_bar);
        }
        __syncthreads();  // the barrier is initialised before anyone waits on it
        sm100::mbar_wait(&s_bar, 0);
        // the row's max (and so its 2^-e scale) does not depend on the router either
        for (int64_t k = (int64_t)threadIdx.x * 8; k < in; k += 128 * 8) {
            const uint4 q = *reinterpret_cast<const uint4*>(srow + k);
            const __nv_bfloat162* pp = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(pp[j]);
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
    sm100::pdl_wait();  // the router's masks / histogram (PDL launch; a no-op otherwise)
    if (hist) {
        // fused bucketing (the router decided the masks and counted the buckets): claim the next slot
        // of this token's bucket.  The slot order inside a bucket is arbitrary, which cannot change
        // any output: a token's result depends only on its own row and its bucket's effective weight.
        if (threadIdx.x == 0) {
            if (src == 0) build_tiles(hist, tiles, meta);
            const int mk = masks[src];
            const int i = bucket_start(hist, mk) + atomicAdd(&fill[mk], 1);
            perm[i] = (int32_t)src;
            pinv[src] = i;
            s_row = i;
        }
    }
    __syncthreads();  // publishes s_row
    const int64_t i = hist ? s_row : pinv[src];
    // k-block slab layout [in_pad/64][tpad][64]: element k of permuted row i at (k/64*tpad + i)*64 + k%64
    __half* dst = xperm + i * kKBlock;
    auto at = [&](int64_t k) { return dst + (k / kKBlock) * tpad * kKBlock + (k % kKBlock); };
    int e = 0;
    if (m > 0.f && isfinite(m)) e = ilogbf(m) - 14;
    const float sc = ldexpf(1.f, -e);
    if (threadIdx.x == 0) escale[i] = ldexpf(1.f, e);
    if (vec) {
        for (int64_t k = (int64_t)threadIdx.x * 8; k < in_pad; k += 128 * 8) {  // the in..in_pad tail: zeros
            const uint4 q = k < in ? *reinterpret_cast<const uint4*>(srow + k) : make_uint4(0, 0, 0, 0);
            uint4 o;
            const __nv_bfloat162* pp = reinterpret_cast<const __nv_bfloat162*>(&q);
            __half2* h = reinterpret_cast<__half2*>(&o);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(pp[j]);
                h[j] = __floats2half2_rn(f.x * sc, f.y * sc);
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
                  int32_t* counts_out, cudaStream_t st, bool sanitize) {
    if (L->max_tiles > kMaxTilesSmem)
        return set_error(MOBI_EINVAL, "bucket: " + std::to_string(L->max_tiles) + " token tiles exceed " +
                                          std::to_string(kMaxTilesSmem) + " per call");
    bucket_kernel<NKEY_MASK><<<1, BK_THREADS, 0, st>>>(L->s_part, (int)L->htiles, T, L->nr, L->b2, delta,
                                             given_masks, sanitize ? 1 : 0, scores_out, L->masks, masks_out, L->perm,
                                             L->tpad_max, cperm_out, inverse_out, counts_out, L->tiles,
                                             L->meta, L->pinv);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    return MOBI_OK;
}

int launch_bucket_generic(mobi_layer* L, int64_t T, float delta, const uint8_t* given_masks, float* scores_out,
                          uint8_t* masks_out, int32_t* cperm_out, int32_t* inverse_out, int32_t* counts_out,
                          cudaStream_t st, bool sanitize) {
    // every mask value (up to 2^8) is a key; counts land in a 256-entry scratch, 2^E are returned
    int32_t* counts = nullptr;
    if (counts_out) {
        if (!L->hist256) MOBI_CUDA(cudaMalloc(&L->hist256, 256 * sizeof(int32_t)));
        counts = L->hist256;
    }
    bucket_kernel<NKEY_ALL><<<1, BK_THREADS, 0, st>>>(L->s_part, (int)L->htiles, T, L->nr, L->b2, delta, given_masks,
                                                      sanitize ? 1 : 0, scores_out, L->masks, masks_out, nullptr, 0,
                                                      cperm_out, inverse_out, counts, nullptr, nullptr, nullptr);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    if (counts_out)
        MOBI_CUDA(cudaMemcpyAsync(counts_out, counts, sizeof(int32_t) * ((size_t)1 << L->E), cudaMemcpyDeviceToDevice, st));
    return MOBI_OK;
}

int launch_permute(const uint8_t* masks, int64_t T, uint8_t* keys_tmp, int32_t* cperm, int32_t* inverse,
                   int32_t* hist256, cudaStream_t st) {
    bucket_kernel<NKEY_ALL><<<1, BK_THREADS, 0, st>>>(nullptr, 0, T, 0, nullptr, 0.f, masks, 0, nullptr, keys_tmp,
                                             nullptr, nullptr, 0, cperm, inverse, hist256, nullptr, nullptr, nullptr);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

int launch_gather(mobi_layer* L, const __nv_bfloat16* x, int64_t T, cudaStream_t st, bool claim, bool pdl) {
    const bool vec = (L->in % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && L->in * 2 <= 200 * 1024;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)T);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = vec ? (size_t)L->in * 2 : 0;
    cfg.stream = st;
    if (vec && cfg.dynamicSmemBytes > 48 * 1024)
        MOBI_TRY(func_attr_once(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    MOBI_CUDA(cudaLaunchKernelEx(&cfg, gather_kernel, x, L->in, L->in_pad, L->tpad_max, L->pinv, L->xperm, L->escale,
                                 vec, (const uint8_t*)L->masks, claim ? (const int*)L->bk_hist : (const int*)nullptr,
                                 L->bk_hist + 32, L->perm, L->tiles, L->meta));
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    return MOBI_OK;
}

}  // namespace mobi
