// decode.cu -- the decode-size MoBi-linear path (T <= kDecMaxT tokens per call).
//
// At decode batch sizes the layer is HBM-bound on its weight bytes (merged codes: 1 B/weight,
// router w1: 2 B per in x h), not tensor-bound, and the bucketed tcgen05 path's per-k-block
// pipeline cost (TMEM round trip + commit/barrier chain, ~700 cycles per 8 KiB block) caps its
// code streaming near 3 TB/s.  This path instead streams codes with TMA bulk copies and keeps the
// whole dequant -> MMA -> fold chain in registers (mma.sync m16n8k16, fp32 accumulate):
//
//   router_dec_kernel   score() for T tokens: H = X W1 (bf16 mma.sync, split-K over the grid),
//                       then silu(H + b1) . w2 + b2 and gate_hard(delta) -> slice masks, all in
//                       one launch via deterministic last-arriver reductions (router.hpp:63-88,
//                       router.hpp:92-103).  It triggers the dependent launch immediately.
//   decode_gemm_kernel  forward_elastic (router.hpp:105-133) for the same tokens, per-token
//                       masks applied directly (no bucket / permutation at this size): persistent
//                       stream-K over (row tile, k-block) units; a producer warp streams the
//                       8 KiB code blocks (prefetch starts before the router has finished: PDL),
//                       eight MMA warps turn code bytes into exact fp16 integers 1024 + (INT &
//                       maskbyte) with two PRMT + one LOP3 per four weights and multiply them with
//                       the token-scaled fp16 activations; each k-block's fp32 result is folded
//                       with the group constants into W = S*(INT & mask) + C exactly as the
//                       bucketed path does (mobi_internal.cuh), the 1024 offset cancelled with the
//                       block's activation sum.  Row tiles shared by several CTAs are reduced in
//                       CTA order by the last CTA to finish (deterministic).
#include "mobi_internal.cuh"
#include "sm100.cuh"

namespace mobi {
namespace {

using namespace sm100;

constexpr int kDecWarps = 8;                     // MMA warps, 16 weight rows each
constexpr int kDecThreads = 32 * kDecWarps;      // thread 0 doubles as the TMA producer (a 9th warp
                                                 // would put 3 warps on one SM sub-partition and cap
                                                 // registers at 168)
constexpr int kDecStages = 8;                    // 8 KiB code blocks in flight per CTA
constexpr int kRdWarps = 4;                      // router: warps per CTA (split K inside the CTA)
constexpr int kRdRows = 16;                      // router: hidden units per CTA (one m16 tile)

__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void bar_mma() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kDecWarps) : "memory"); }
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 v;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// ============================================================================================
// router
// ============================================================================================
struct RDParams {
    const __nv_bfloat16* x;   // [T][in]
    const __nv_bfloat16* w1t; // [h_pad][in_pad]
    const float* b1;          // [h_pad]
    const float* w2;          // [h_pad][nr]
    const float* b2;          // [nr]
    float* hpart;             // [ks][T][h_pad]
    float* spart;             // [n_mt][T][nr]
    int* cnt;                 // [n_mt + 1] arrival counters (zero between launches)
    uint8_t* masks;           // [T]
    uint8_t* masks_out;       // optional
    float* scores_out;        // optional [T][nr]
    int64_t in, in_pad, h, h_pad;
    int T, nr, ks, cpw;       // cpw: 32-wide k chunks per warp
    float delta;
};

// Lane (g, c) of a warp owns hidden rows g and g+8 of the CTA's m16 tile and, inside each 32-wide
// k chunk, the 8 contiguous k at 8c: two 16-byte loads per row, each feeding two m16n8k16 steps
// (MMA k order is a permutation of memory order; X uses the same permutation, so the dot products
// are unchanged).
template <int NT>
__global__ void __launch_bounds__(32 * kRdWarps) router_dec_kernel(const __grid_constant__ RDParams p) {
    grid_dep_launch();  // the decode GEMM may start prefetching codes right away
    __shared__ float red[kRdWarps][kRdRows][8 * NT + 1];
    __shared__ float act[8 * NT][kRdRows];
    __shared__ int s_last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, c = lane & 3;
    const int mt = blockIdx.x, split = blockIdx.y;
    const int64_t nchunks = p.in_pad / 32;
    const int64_t q0 = ((int64_t)split * kRdWarps + warp) * p.cpw;
    const int64_t q1 = q0 + p.cpw < nchunks ? q0 + p.cpw : nchunks;
    float acc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    const __nv_bfloat16* ar0 = p.w1t + ((int64_t)mt * kRdRows + g) * p.in_pad + 8 * c;
    const __nv_bfloat16* ar1 = ar0 + 8 * p.in_pad;
    constexpr int U = 4;
    for (int64_t q = q0; q < q1; q += U) {
        uint4 a0[U], a1[U], b[U][NT];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = (q + u) * 32;
            const bool ok = q + u < q1;
            a0[u] = ok ? ldg_stream(ar0 + k) : make_uint4(0, 0, 0, 0);
            a1[u] = ok ? ldg_stream(ar1 + k) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const int tok = 8 * n + g;
                b[u][n] = (ok && tok < p.T && k + 8 * c < p.in)
                              ? __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)tok * p.in + k + 8 * c))
                              : make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                mma_bf16(acc[n], a0[u].x, a1[u].x, a0[u].y, a1[u].y, b[u][n].x, b[u][n].y);
                mma_bf16(acc[n], a0[u].z, a1[u].z, a0[u].w, a1[u].w, b[u][n].z, b[u][n].w);
            }
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        red[warp][g][8 * n + 2 * c] = acc[n][0];
        red[warp][g][8 * n + 2 * c + 1] = acc[n][1];
        red[warp][g + 8][8 * n + 2 * c] = acc[n][2];
        red[warp][g + 8][8 * n + 2 * c + 1] = acc[n][3];
    }
    __syncthreads();
    for (int i = tid; i < kRdRows * 8 * NT; i += 32 * kRdWarps) {
        const int row = i % kRdRows, tok = i / kRdRows;
        if (tok >= p.T) continue;
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kRdWarps; ++w) s += red[w][row][tok];
        p.hpart[((int64_t)split * p.T + tok) * p.h_pad + (int64_t)mt * kRdRows + row] = s;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&p.cnt[mt], 1) == p.ks - 1;
    __syncthreads();
    if (!s_last) return;
    // ---- last split of hidden tile mt: silu(H + b1) . w2 for its 16 hidden units ----
    __threadfence();
    for (int i = tid; i < kRdRows * p.T; i += 32 * kRdWarps) {
        const int row = i % kRdRows, tok = i / kRdRows;
        const int64_t j = (int64_t)mt * kRdRows + row;
        float v = 0.f;
        if (j < p.h) {
            float H = 0.f;
            for (int s = 0; s < p.ks; ++s) H += __ldcg(p.hpart + ((int64_t)s * p.T + tok) * p.h_pad + j);
            const float a = H + p.b1[j];
            v = a * __fdividef(1.f, 1.f + __expf(-a));
        }
        act[tok][row] = v;
    }
    __syncthreads();
    for (int i = tid; i < p.T * p.nr; i += 32 * kRdWarps) {
        const int tok = i / p.nr, k = i % p.nr;
        float s = 0.f;
#pragma unroll
        for (int row = 0; row < kRdRows; ++row) s += act[tok][row] * p.w2[((int64_t)mt * kRdRows + row) * p.nr + k];
        p.spart[((int64_t)mt * p.T + tok) * p.nr + k] = s;
    }
    if (tid == 0) p.cnt[mt] = 0;
    __threadfence();
    __syncthreads();
    const int n_mt = gridDim.x;
    if (tid == 0) s_last = atomicAdd(&p.cnt[n_mt], 1) == n_mt - 1;
    __syncthreads();
    if (!s_last) return;
    // ---- last hidden tile overall: scores, gate_hard(delta) (strict '>', router.hpp:92-103) ----
    __threadfence();
    for (int tok = tid; tok < p.T; tok += 32 * kRdWarps) {
        int m = 1;
        for (int k = 0; k < p.nr; ++k) {
            float s = 0.f;
            for (int q = 0; q < n_mt; ++q) s += __ldcg(p.spart + ((int64_t)q * p.T + tok) * p.nr + k);
            s += p.b2[k];
            if (p.scores_out) p.scores_out[(int64_t)tok * p.nr + k] = s;
            if ((s - p.delta) > 0.f) m |= 1 << (k + 1);
        }
        p.masks[tok] = (uint8_t)m;
        if (p.masks_out) p.masks_out[tok] = (uint8_t)m;
    }
    if (tid == 0) p.cnt[n_mt] = 0;
}

// ============================================================================================
// decode GEMM
// ============================================================================================
struct DParams {
    const uint8_t* codes8;    // tiled merged codes [out_pad/128][kblocks][8192]
    const float2* gconst;     // [G][out_pad] (s, s*z)
    const __nv_bfloat16* x;   // [T][in]
    const uint8_t* masks;     // [T]
    __nv_bfloat16* y;         // [T][out]
    float* part;              // [(n_cta + n_rt)][T][128] row-tile partials
    int* cnt;                 // [n_rt] arrival counters (zero between launches)
    MaskTable mt;
    int64_t out, out_pad, in, kblocks, gs, U;
    int T, n_cta, len_max, xs_stride, single_group, vmask;
};

struct DecSmem {
    size_t ring, full, empty, xs, x16, total;
};
__host__ __device__ inline DecSmem dec_smem(int T, int len_max, int xs_stride) {
    DecSmem s;
    s.ring = 0;
    s.full = s.ring + (size_t)kDecStages * kBlockBytes;
    s.empty = s.full + kDecStages * 8;
    s.xs = s.empty + kDecStages * 8;
    s.x16 = s.xs + ((size_t)len_max * (T + 1) * 4 + 15) / 16 * 16;
    s.total = s.x16 + (size_t)(T + 1) * xs_stride * 2;
    return s;
}

// first CTA whose unit range contains unit u (ranges are [i*U/n, (i+1)*U/n))
__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int n) { return (int)(((u + 1) * n + U - 1) / U) - 1; }

template <int MAXT>
__global__ void __launch_bounds__(kDecThreads, 1) decode_gemm_kernel(const __grid_constant__ DParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ float s_escale[kDecMaxT + 1], s_scl[kDecMaxT + 1];
    __shared__ int s_max[kDecMaxT + 1];
    __shared__ int s_tmask[MAXT], s_ttok[MAXT][8];
    __shared__ int s_ntiles, s_flag;
    const int T = p.T;
    const DecSmem L = dec_smem(T, p.len_max, p.xs_stride);
    uint8_t* ring = smem + L.ring;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.full);
    uint64_t* empty = reinterpret_cast<uint64_t*>(smem + L.empty);
    float* xs = reinterpret_cast<float*>(smem + L.xs);
    __half* x16 = reinterpret_cast<__half*>(smem + L.x16);

    const int warp = warp_idx_uniform(), lane = threadIdx.x & 31;
    const int cta = blockIdx.x;
    const int64_t u0 = (int64_t)cta * p.U / p.n_cta, u1 = (int64_t)(cta + 1) * p.U / p.n_cta;
    const int64_t kbn = p.kblocks;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kDecStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kDecWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();

    // thread 0 streams this CTA's code blocks (independent of the router: starts before the
    // grid dependency resolves); the first kDecStages now, the rest as stages are released
    const int64_t nblk = u1 - u0;
    uint64_t pol = 0;
    if (threadIdx.x == 0) {
        pol = policy_evict_first();
        for (int64_t it = 0; it < nblk && it < kDecStages; ++it) {
            mbar_arrive_expect_tx(&full[it], kBlockBytes);
            bulk_load(ring + (size_t)it * kBlockBytes, p.codes8 + (u0 + it) * kBlockBytes, kBlockBytes, &full[it], pol);
        }
    }

    // ---------------- MMA warps ----------------
    const int tid = threadIdx.x;  // 0 .. 32*kDecWarps-1
    const int kb_start = (int)(u0 % kbn);
    const int len = (int)(u1 - u0 < kbn ? u1 - u0 : kbn);
    // (1) activations of the k-blocks this CTA touches -> fp16, scaled per token by 2^-e so that
    //     max|x| lands in [2^14, 2^15) (exact, as the bucketed path's gather); X was produced before
    //     the router started, so this overlaps the router.
    for (int t = tid; t <= T; t += 32 * kDecWarps) s_max[t] = 0;
    bar_mma();
    const int nvec = len * 8;  // 16-byte vectors per token
    for (int v = tid; v < T * nvec; v += 32 * kDecWarps) {
        const int t = v / nvec, r = v % nvec;
        const int64_t k = (int64_t)((kb_start + r / 8) % kbn) * kKBlock + (r % 8) * 8;
        if (k < p.in) {
            uint4 q = __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.in + k));
            const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
            float m = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float2 f = __bfloat1622float2(b[j]);
                m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
            }
            atomicMax(&s_max[t], __float_as_int(m));
        }
    }
    bar_mma();
    for (int t = tid; t <= T; t += 32 * kDecWarps) {
        const float m = __int_as_float(s_max[t]);
        int e = 0;
        if (t < T && m > 0.f && isfinite(m)) e = ilogbf(m) - 14;
        s_escale[t] = t < T ? ldexpf(1.f, e) : 0.f;
        s_scl[t] = ldexpf(1.f, -e);
    }
    bar_mma();
    for (int v = tid; v < (T + 1) * nvec; v += 32 * kDecWarps) {
        const int t = v / nvec, r = v % nvec;
        const int64_t k = (int64_t)((kb_start + r / 8) % kbn) * kKBlock + (r % 8) * 8;
        uint4 o = make_uint4(0, 0, 0, 0);
        if (t < T && k < p.in) {
            uint4 q = __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.in + k));
            const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
            __half2* h = reinterpret_cast<__half2*>(&o);
            const float sc = s_scl[t];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float2 f = __bfloat1622float2(b[j]);
                h[j] = __floats2half2_rn(f.x * sc, f.y * sc);
            }
        }
        *reinterpret_cast<uint4*>(x16 + (size_t)t * p.xs_stride + r * 8) = o;
    }
    bar_mma();
    // per (k-block, token) sums of the fp16 activations (cancel the 1024 offset of the weights)
    for (int i = tid; i < len * (T + 1); i += 32 * kDecWarps) {
        const int slot = i / (T + 1), t = i % (T + 1);
        const __half2* r = reinterpret_cast<const __half2*>(x16 + (size_t)t * p.xs_stride + slot * kKBlock);
        float s = 0.f;
#pragma unroll 8
        for (int j = 0; j < kKBlock / 2; ++j) {
            float2 f = __half22float2(r[j]);
            s += f.x;
            s += f.y;
        }
        xs[i] = s;
    }
    // (2) token tiles: tokens grouped by slice mask (ascending), 8 per MMA n-tile; empty columns
    //     point at the zero row T.  Needs the router's masks.
    grid_dep_wait();
    if (warp == 0) {
        for (int i = lane; i < MAXT * 8; i += 32) s_ttok[i / 8][i % 8] = T;
        __syncwarp();
        int m = -1;
        if (lane < T) {
            m = p.masks[lane];
            if (p.vmask) m = (m & p.vmask) | 1;
        }
        int base = 0;
        for (int v = 0; v < 2 * kMaxBuckets; ++v) {
            const unsigned bal = __ballot_sync(0xffffffffu, m == v);
            if (!bal) continue;
            if (m == v) {
                const int r = __popc(bal & ((1u << lane) - 1u));
                s_ttok[base + r / 8][r % 8] = lane;
            }
            const int nt = (__popc(bal) + 7) / 8;
            if (lane < nt) s_tmask[base + lane] = v;
            base += nt;
        }
        if (lane == 0) s_ntiles = base;
    }
    bar_mma();

    const int w = warp, g = lane >> 2, c = lane & 3;
    const int ntiles = s_ntiles;
    // per-lane tile constants: B row offset, output tokens (2c, 2c+1), their scales
    int xoff[MAXT], tk0[MAXT], tk1[MAXT], tmask[MAXT];
    float es0[MAXT], es1[MAXT];
#pragma unroll
    for (int i = 0; i < MAXT; ++i) {
        const int ii = i < ntiles ? i : 0;
        xoff[i] = s_ttok[ii][g] * p.xs_stride + 16 * c;
        tk0[i] = s_ttok[ii][2 * c];
        tk1[i] = s_ttok[ii][2 * c + 1];
        tmask[i] = s_tmask[ii];
        es0[i] = s_escale[tk0[i]];
        es1[i] = s_escale[tk1[i]];
    }
    float yp[MAXT][4];
    const float inv2p = p.mt.inv_2p;
    const int rl0 = 16 * w + g, rl1 = rl0 + 8;

    auto gc_load = [&](int64_t u, float2& a, float2& b) {
        const int64_t rt = u / kbn, kb = u % kbn;
        const int64_t grp = p.single_group ? 0 : (kb * kKBlock) / p.gs;
        const float2* gp = p.gconst + grp * p.out_pad + rt * kRowTile;
        a = __ldg(gp + rl0);
        b = __ldg(gp + rl1);
    };
    auto flush = [&](int64_t rt) {
        const int lo = cta_of(rt * kbn, p.U, p.n_cta), hi = cta_of(rt * kbn + kbn - 1, p.U, p.n_cta);
        const int64_t R0 = rt * kRowTile + rl0, R1 = rt * kRowTile + rl1;
        if (lo == hi) {
#pragma unroll
            for (int i = 0; i < MAXT; ++i) {
                if (i >= ntiles) break;
                if (tk0[i] < T) {
                    if (R0 < p.out) p.y[(int64_t)tk0[i] * p.out + R0] = __float2bfloat16_rn(yp[i][0]);
                    if (R1 < p.out) p.y[(int64_t)tk0[i] * p.out + R1] = __float2bfloat16_rn(yp[i][2]);
                }
                if (tk1[i] < T) {
                    if (R0 < p.out) p.y[(int64_t)tk1[i] * p.out + R0] = __float2bfloat16_rn(yp[i][1]);
                    if (R1 < p.out) p.y[(int64_t)tk1[i] * p.out + R1] = __float2bfloat16_rn(yp[i][3]);
                }
            }
            return;
        }
        float* mine = p.part + ((int64_t)cta + rt) * T * kRowTile;
#pragma unroll
        for (int i = 0; i < MAXT; ++i) {
            if (i >= ntiles) break;
            if (tk0[i] < T) {
                mine[tk0[i] * kRowTile + rl0] = yp[i][0];
                mine[tk0[i] * kRowTile + rl1] = yp[i][2];
            }
            if (tk1[i] < T) {
                mine[tk1[i] * kRowTile + rl0] = yp[i][1];
                mine[tk1[i] * kRowTile + rl1] = yp[i][3];
            }
        }
        __threadfence();
        bar_mma();
        if (tid == 0) s_flag = atomicAdd(&p.cnt[rt], 1) == hi - lo;
        bar_mma();
        if (s_flag) {
            __threadfence();
            for (int i = tid; i < T * kRowTile; i += 32 * kDecWarps) {
                const int t = i / kRowTile, rl = i % kRowTile;
                const int64_t R = rt * kRowTile + rl;
                if (R >= p.out) continue;
                float s = 0.f;
                for (int j = lo; j <= hi; ++j) s += __ldcg(p.part + (((int64_t)j + rt) * T + t) * kRowTile + rl);
                p.y[(int64_t)t * p.out + R] = __float2bfloat16_rn(s);
            }
            if (tid == 0) p.cnt[rt] = 0;
        }
        bar_mma();
    };

    int64_t cur_rt = -1;
    float2 gn0, gn1;
    if (u0 < u1) gc_load(u0, gn0, gn1);
    for (int64_t u = u0; u < u1; ++u) {
        const int64_t it = u - u0;
        const int64_t rt = u / kbn;
        const int kb = (int)(u % kbn);
        if (rt != cur_rt) {
            if (cur_rt >= 0) flush(cur_rt);
            cur_rt = rt;
#pragma unroll
            for (int i = 0; i < MAXT; ++i) yp[i][0] = yp[i][1] = yp[i][2] = yp[i][3] = 0.f;
        }
        if (threadIdx.x == 0 && it >= 1 && it - 1 + kDecStages < nblk) {
            // refill the stage every warp released in the previous iteration
            const int64_t j = it - 1;
            const int sj = (int)(j % kDecStages);
            mbar_wait(&empty[sj], (uint32_t)((j / kDecStages) & 1));
            mbar_arrive_expect_tx(&full[sj], kBlockBytes);
            bulk_load(ring + (size_t)sj * kBlockBytes, p.codes8 + (u0 + j + kDecStages) * kBlockBytes, kBlockBytes,
                      &full[sj], pol);
        }
        const float2 g0 = gn0, g1 = gn1;
        if (u + 1 < u1) gc_load(u + 1, gn0, gn1);
        const int slot = (int)((kb - kb_start + kbn) % kbn);
        const int s = (int)(it % kDecStages);
        mbar_wait(&full[s], (uint32_t)((it / kDecStages) & 1));
        const uint8_t* blk = ring + (size_t)s * kBlockBytes;
        const uint4 q0 = *reinterpret_cast<const uint4*>(blk + (c * kRowTile + rl0) * 16);
        const uint4 q1 = *reinterpret_cast<const uint4*>(blk + (c * kRowTile + rl1) * 16);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        // bytes -> {0x64, byte} half pairs (1024 + byte); lane's bytes are k = kb*64 + 16c + 0..15
        uint32_t s0[8], s1[8];
        {
            const uint32_t w0[4] = {q0.x, q0.y, q0.z, q0.w}, w1[4] = {q1.x, q1.y, q1.z, q1.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                s0[2 * j] = __byte_perm(w0[j], 0x64646464u, 0x4140);
                s0[2 * j + 1] = __byte_perm(w0[j], 0x64646464u, 0x4342);
                s1[2 * j] = __byte_perm(w1[j], 0x64646464u, 0x4140);
                s1[2 * j + 1] = __byte_perm(w1[j], 0x64646464u, 0x4342);
            }
        }
        const float* xsb = xs + slot * (T + 1);
        const int xb = slot * kKBlock;
        const float a0 = g0.x * inv2p, a1 = g1.x * inv2p;
        int cur_mask = -1;
        uint32_t A[16];
        float br0 = 0.f, br1 = 0.f;
#pragma unroll
        for (int i = 0; i < MAXT; ++i) {
            if (i >= ntiles) break;
            if (tmask[i] != cur_mask) {
                cur_mask = tmask[i];
                const uint32_t pat = 0xFF00FF00u | ((p.mt.maskword[cur_mask] & 0xFFu) * 0x00010001u);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    A[j] = s0[j] & pat;
                    A[8 + j] = s1[j] & pat;
                }
                const float kcm = p.mt.kc[cur_mask] - 1024.f * inv2p;
                br0 = fmaf(g0.x, kcm, -g0.y);
                br1 = fmaf(g1.x, kcm, -g1.y);
            }
            const uint4 b0 = *reinterpret_cast<const uint4*>(x16 + xoff[i] + xb);
            const uint4 b1 = *reinterpret_cast<const uint4*>(x16 + xoff[i] + xb + 8);
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            mma_f16(acc, A[0], A[8], A[1], A[9], b0.x, b0.y);
            mma_f16(acc, A[2], A[10], A[3], A[11], b0.z, b0.w);
            mma_f16(acc, A[4], A[12], A[5], A[13], b1.x, b1.y);
            mma_f16(acc, A[6], A[14], A[7], A[15], b1.z, b1.w);
            const float x0 = xsb[tk0[i]], x1 = xsb[tk1[i]];
            yp[i][0] = fmaf(fmaf(a0, acc[0], br0 * x0), es0[i], yp[i][0]);
            yp[i][1] = fmaf(fmaf(a0, acc[1], br0 * x1), es1[i], yp[i][1]);
            yp[i][2] = fmaf(fmaf(a1, acc[2], br1 * x0), es0[i], yp[i][2]);
            yp[i][3] = fmaf(fmaf(a1, acc[3], br1 * x1), es1[i], yp[i][3]);
        }
    }
    if (cur_rt >= 0) flush(cur_rt);
}

int sm_count_dec() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

struct DecPlan {
    int n_cta = 0, len_max = 0, xs_stride = 0;
    int64_t U = 0;
    size_t smem = 0;
};

DecPlan plan_decode(const mobi_layer* L, int64_t T) {
    DecPlan d;
    const int64_t n_rt = cdiv(L->out, kRowTile);
    d.U = n_rt * L->kblocks;
    d.n_cta = (int)std::min<int64_t>(sm_count_dec(), d.U);
    d.len_max = (int)std::min<int64_t>(cdiv(d.U, d.n_cta), L->kblocks);
    d.xs_stride = d.len_max * kKBlock + 8;  // row stride = 16 mod 128 bytes: conflict-free B loads
    d.smem = dec_smem((int)T, d.len_max, d.xs_stride).total;
    return d;
}

constexpr size_t kDecSmemMax = 200 * 1024;

template <int MAXT>
int launch_decode_gemm_t(mobi_layer* L, const DParams& p, size_t smem, bool pdl, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        MOBI_CUDA(cudaFuncSetAttribute(decode_gemm_kernel<MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kDecSmemMax));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.n_cta);
    cfg.blockDim = dim3(kDecThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    MOBI_CUDA(cudaLaunchKernelEx(&cfg, decode_gemm_kernel<MAXT>, p));
    ++L->last_launches;
    return MOBI_OK;
}

}  // namespace

bool decode_supported(const mobi_layer* L, const void* x, int64_t T) {
    if (T < 1 || T > kDecMaxT) return false;
    if (L->in % 8 != 0 || (reinterpret_cast<uintptr_t>(x) & 15u) != 0) return false;
    if (!L->single_group && L->gs % kKBlock != 0) return false;
    return plan_decode(L, T).smem <= kDecSmemMax;
}

int launch_router_dec(mobi_layer* L, const __nv_bfloat16* x, int64_t T, float delta, uint8_t* masks_out,
                      float* scores_out, cudaStream_t st) {
    RDParams p{};
    p.x = x;
    p.w1t = L->w1t;
    p.b1 = L->b1;
    p.w2 = L->w2;
    p.b2 = L->b2;
    p.hpart = L->hpart;
    p.spart = L->dec_spart;
    p.cnt = L->dec_cnt + cdiv(L->out, kRowTile);
    p.masks = L->masks;
    p.masks_out = masks_out;
    p.scores_out = scores_out;
    p.in = L->in;
    p.in_pad = L->in_pad;
    p.h = L->h;
    p.h_pad = L->h_pad;
    p.T = (int)T;
    p.nr = L->nr;
    p.delta = delta;
    const int n_mt = (int)(L->h_pad / kRdRows);
    const int64_t nchunks = L->in_pad / 32;
    int ks = std::max(1, std::min(16, (2 * sm_count_dec() + n_mt - 1) / n_mt));
    ks = (int)std::max<int64_t>(1, std::min<int64_t>(ks, nchunks / (kRdWarps * 2)));
    p.cpw = (int)cdiv(nchunks, (int64_t)ks * kRdWarps);
    ks = (int)cdiv(nchunks, (int64_t)p.cpw * kRdWarps);  // no empty splits
    p.ks = ks;
    const dim3 grid((unsigned)n_mt, (unsigned)ks);
    if (T <= 8)
        router_dec_kernel<1><<<grid, 32 * kRdWarps, 0, st>>>(p);
    else if (T <= 16)
        router_dec_kernel<2><<<grid, 32 * kRdWarps, 0, st>>>(p);
    else
        router_dec_kernel<4><<<grid, 32 * kRdWarps, 0, st>>>(p);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    return MOBI_OK;
}

int launch_decode_gemm(mobi_layer* L, const __nv_bfloat16* x, int64_t T, const uint8_t* given_masks,
                       __nv_bfloat16* y, bool pdl, cudaStream_t st) {
    const DecPlan d = plan_decode(L, T);
    DParams p{};
    p.codes8 = L->codes8;
    p.gconst = L->gconst;
    p.x = x;
    p.masks = given_masks ? given_masks : L->masks;
    p.vmask = given_masks ? (1 << (L->nr + 1)) - 1 : 0;
    p.y = y;
    p.part = L->dec_part;
    p.cnt = L->dec_cnt;
    p.mt = L->mtab;
    p.out = L->out;
    p.out_pad = L->out_pad;
    p.in = L->in;
    p.kblocks = L->kblocks;
    p.gs = L->gs;
    p.single_group = L->single_group ? 1 : 0;
    p.U = d.U;
    p.T = (int)T;
    p.n_cta = d.n_cta;
    p.len_max = d.len_max;
    p.xs_stride = d.xs_stride;
    if (T == 1) return launch_decode_gemm_t<1>(L, p, d.smem, pdl, st);
    if (T <= 8) return launch_decode_gemm_t<8>(L, p, d.smem, pdl, st);
    if (T <= 16) return launch_decode_gemm_t<9>(L, p, d.smem, pdl, st);
    return launch_decode_gemm_t<11>(L, p, d.smem, pdl, st);
}

}  // namespace mobi
