// decode2.cu -- decode GEMV on slice planes (T <= kD2MaxT tokens): stream only the slices a batch uses.
//
// At one to four tokens the layer is bound by the bytes it streams.  The merged 8-bit codes hold all
// four 2-bit slices, so a token that only needs slice 1 would still pay 1 B/weight.  Here every slice
// has its own plane (layer.cu: pack_dplanes_kernel), already arranged as mma.sync A fragments, and the
// kernel reads slice 1 (always on) while the router is still running, then -- once the masks are
// known (griddepcontrol.wait) -- only the planes of the union of the batch's slices.
//
// The contraction is split per slice (router.hpp:105-132 is exactly this sum):
//     y_t = sum_{e in m_t} sum_g (s_g / 64) 4^(4-e) (x_t . c_e)_g  +  kc[m_t] A_t - B_t
//     A_t = sum_g s_g sum_{k in g} x_t,   B_t = sum_g s_g z_g sum_{k in g} x_t
// which is the folded weight W_m = S (INT & maskbyte(m)) + C_m of the prefill GEMM
// (mobi_internal.cuh) regrouped per slice.  (x_t . c_e)_g runs on mma.sync m16n8k16 with the
// fragment-ordered 2-bit codes expanded to exact fp16 (1024 + c, the offset cancelled with the
// group's activation sum) and x scaled per token by 2^-e into fp16 (exact).
//
// One CTA owns R 32-row tiles (R = 1 while the tiles fit one wave, else 2/4/8) over the whole K (no
// cross-CTA reduction); each tile's 16/R warps split K and are summed in warp order at the end
// (deterministic).  With R > 1 the first 16/R warps convert X for everyone.
#include "mobi_internal.cuh"
#include "sm100.cuh"

namespace mobi {
namespace {

using namespace sm100;

constexpr int kD2Warps = 16, kD2Threads = 32 * kD2Warps;  // 16 warps: 4 per scheduler (latency hiding)
constexpr int kD2MaxT = 16;       // tokens per launch: two groups of 8 (the m16n8k16 N dimension)
constexpr int kD2MaxLaunchT = 32;  // larger decode batches: one launch per 16 tokens
constexpr int kD2Acc = 2 * 2 * 4;  // per lane: y over the token's slices (B folded in), A  ([2][4] each)

struct D2Params {
    const uint4* dplanes;     // [E][n_rt32][kblocks][32] 16 B
    const float2* gconst;     // [G][out_pad] (s, s*z)
    const __nv_bfloat16* x;   // [T][in]
    const uint8_t* masks;     // given masks (forward_masked) or null
    const float* spart;       // [n_mt][T][nr] router tile partial scores
    const float* b2;
    uint8_t* masks_dev;
    uint8_t* masks_out;
    float* scores_out;
    __nv_bfloat16* y;
    MaskTable mt;
    int64_t out, out_pad, in, in_pad, kblocks, gs;
    float delta;
    int single_group, T, E, nr, n_mt, vmask, n_rt32, xs_stride;
    int t0, t_all;    // this launch's first token and the batch size (router partials are [n_mt][t_all][nr])
    int gpw;          // groups per warp (bound) for the staged constants
    int R, wpt;       // 32-row tiles per CTA, warps per tile (R * wpt = kD2Warps)
    int64_t gcs_off;  // byte offset of the staged constants in dynamic smem
    int64_t ring_off; // byte offset of the per-lane cp.async rings
    int64_t xgs_off;  // byte offset of the per-(k range, token, group) activation sums
    unsigned long long* trace;  // debug: per-CTA globaltimer marks [2048 + cta][8]
};
__device__ __forceinline__ unsigned long long gtimer2() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void mma_f16_acc(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                            uint32_t b0, uint32_t b1) {
#ifdef MOBI_D2_NOMMA  // dev: what the stream costs without the tensor instructions (wrong results)
    d[0] = fmaf(__uint_as_float((a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1) & 0x3fffffffu), 1e-30f, d[0]);
    return;
#endif
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void grid_dep_wait2() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 2-bit fields i and i+8 of a fragment word -> half2 (1024 + lo, 1024 + hi)
// Field ss of a (pre-shifted) plane word -> half2 (1024 + 4^ss lo, 1024 + 4^ss hi): one LOP3 (a & b) | c,
// the magic in a register so the mask can be the immediate (layer.cu: pack_dplanes_kernel)
template <int SS>
__device__ __forceinline__ uint32_t frag(uint32_t w, uint32_t magic) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "n"(0x00030003u << (2 * SS)), "r"(magic));
    return r;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kD2Ring = 6;  // (slice, k-block) items in flight per lane (16 B each): 48 KiB per CTA
                            // (sized so the router's ring fits on the same SM at T = 8)

// NG token groups of 8 per launch: 1 (T <= 8, capped at 80 registers so the router's CTAs stay
// co-resident) or 2 (9..16 tokens: the A fragments of every item serve both groups)
template <int NG>
__global__ void __maxnreg__(NG == 1 ? 96 : 128) decode_planes_kernel(const __grid_constant__ D2Params p) {
    extern __shared__ __align__(16) uint8_t smem[];
    __half* x16 = reinterpret_cast<__half*>(smem);                                   // [T + 1][xs_stride]
    // [T][kblocks] {sum of the k-step-scaled fp16 X (offset cancellation), unscaled sum (A, B)}
    float2* xsum = reinterpret_cast<float2*>(smem + (size_t)(p.T + 1) * p.xs_stride * 2);  // rows 0..T-1 + zeros
    float* red = reinterpret_cast<float*>(smem);  // [warps][kD2Acc][32], aliases x16 after the passes
    __shared__ float es_s[kD2Warps][8 * NG];
    __shared__ float s_score[8 * NG][kFastSlices - 1];
    __shared__ int s_mask[8 * NG];
    const int tid = threadIdx.x, warp = warp_idx_uniform(), lane = tid & 31;
    float2* gcs = reinterpret_cast<float2*>(smem + p.gcs_off) + (size_t)warp * p.gpw * 32;  // [groups][32 rows]
    uint4* ring = reinterpret_cast<uint4*>(smem + p.ring_off) + (size_t)warp * kD2Ring * 32;   // [slots][32 lanes]
    const int wl = warp % p.wpt;                    // warp index inside its tile (K split)
    const int rt = blockIdx.x * p.R + warp / p.wpt;  // this warp's 32-row tile
    const bool conv = warp < p.wpt;                 // converts X (k range of wl) for the whole CTA
    auto TRM = [&](int i) {
        if (p.trace && tid == 0) p.trace[(size_t)(2048 + blockIdx.x) * 8 + i] = gtimer2();
    };
    TRM(0);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next router may prefetch its w1
    const int T = p.T;
    // k-block range of this warp; warps of a tile past the last have none (they still take part in
    // the CTA barriers)
    const int kw0 = (int)((int64_t)wl * p.kblocks / p.wpt);
    const int kw1 = rt < p.n_rt32 ? (int)((int64_t)(wl + 1) * p.kblocks / p.wpt) : kw0;
    // streamed items (see (2)-(4) below): item i = (slice slist[i / nk], k-block kw0 + i % nk); issued in
    // order, one cp.async group each, into ring slot i % kD2Ring; slice 1's first items go out now so
    // their latency hides behind the activation prologue
    int pi = 0;
    uint32_t slist = 0;  // the stream's slices, 2 bits each: slice 1 (e0 = 0), then the union's others
    int psi = 0, pkb = kw0;  // issue cursor: (slice index, k-block) of item pi
    const uint4* rt_planes = p.dplanes + (int64_t)rt * p.kblocks * 32 + lane;
    const int plane_stride = p.n_rt32 * (int)p.kblocks * 32;  // uint4s per slice plane
    const uint4* ip = rt_planes + kw0 * 32;  // source of item pi
    auto seek = [&]() { ip = rt_planes + ((int)(slist >> (2 * psi)) & 3) * plane_stride + pkb * 32; };
    // every prologue step and every loop iteration commits exactly one cp.async group (empty when there
    // is nothing to issue), so item ci is always followed by kD2Ring - 2 newer groups and one constant
    // wait_group covers every position of the stream
    int pslot = 0;  // ring slot of item pi (= pi % kD2Ring)
    auto issue = [&]() {
        cp_async16(ring + pslot * 32 + lane, ip, true);
        ++pi;
        pslot = pslot + 1 == kD2Ring ? 0 : pslot + 1;
        if (++pkb == kw1) {
            pkb = kw0, ++psi;
            seek();
        } else {
            ip += 32;
        }
    };
    // (0) stage, as one cp.async group: this warp's k range of every token's bf16 X into its x16 rows
    //     (converted in place below) and the group constants (s, s*z) of the warp's groups for the
    //     tile's 32 rows (read once for all slices); slice 1's first items follow as their own groups
    const int64_t k_lo = (int64_t)kw0 * kKBlock, k_hi = conv ? (int64_t)kw1 * kKBlock : k_lo;
    for (int t = 0; t < T; ++t)
        for (int64_t k = k_lo + lane * 8; k < k_hi; k += 256) {
            const bool ok = k < p.in;
            cp_async16(x16 + (size_t)t * p.xs_stride + k, ok ? (const void*)(p.x + (int64_t)t * p.in + k) : (const void*)p.x,
                       ok);
        }
    {
        const int64_t g0 = p.single_group ? 0 : (int64_t)kw0 * kKBlock / p.gs;
        const int64_t g1 = p.single_group ? 1 : ((int64_t)kw1 * kKBlock + p.gs - 1) / p.gs;
        if (kw1 > kw0)
            for (int i = lane; i < (int)(g1 - g0) * 16; i += 32)
                cp_async16(gcs + (i / 16) * 32 + (i % 16) * 2,
                           p.gconst + (g0 + i / 16) * p.out_pad + (int64_t)rt * 32 + (i % 16) * 2, true);
    }
    cp_commit();
    for (int j = 0; j < kD2Ring - 1; ++j) {
        if (pi < kw1 - kw0) issue();
        cp_commit();
    }
    cp_wait<kD2Ring - 1>();  // the staging group has landed (slice 1's items may still be in flight)
    __syncwarp();

    // (1) X in place: bf16 -> per-token 2^-e scale (max over the warp's range) x 4^-ss per k-step ->
    //     fp16, and per-(token, k-block) sums of the fp16 values (scaled, and rescaled by 4^ss)
    // k-step of a value: ss = (k % 16) / 4 (pack_dplanes_kernel's fragment order), so a lane's 8
    // values are 4 of k-step ss0 and 4 of ss0 + 1
    const int ss0 = 2 * (lane & 1);
    // four tokens at a time: their max-reductions and conversions proceed side by side
    // (independent shuffle chains)
    for (int tb = 0; tb < T; tb += 4) {
        float sc[4];
        {
            float m[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int t = tb + i;
                m[i] = 0.f;
                if (t < T)
                    for (int64_t k = k_lo + lane * 8; k < k_hi; k += 256) {
                        const uint4 q = *reinterpret_cast<const uint4*>(x16 + (size_t)t * p.xs_stride + k);
                        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float2 f2 = __bfloat1622float2(b[j]);
                            m[i] = fmaxf(m[i], fmaxf(fabsf(f2.x), fabsf(f2.y)));
                        }
                    }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int i = 0; i < 4; ++i) m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], o));
            if (tb == 0) TRM(6);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                // e = exponent(max) - 14 (the max lands in [2^14, 2^15)), clamped so 2^-e stays a
                // normal float for tiny activations; powers of two from exponent bits (no libm calls)
                int e = 0;
                if (m[i] > 0.f && m[i] <= 3.0e38f) e = max(((__float_as_int(m[i]) >> 23) & 0xff) - 127 - 14, -100);
                sc[i] = __int_as_float((127 - e - 2 * ss0) << 23);
                if (lane == 0 && tb + i < T) es_s[warp][tb + i] = __int_as_float((127 + e) << 23);
            }
        }
        for (int64_t k0 = k_lo; k0 < k_hi; k0 += 256) {  // warp-uniform trip count
            const int64_t k = k0 + lane * 8;
            float sacc[4], uacc[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int t = tb + i;
                float s_lo = 0.f, s_hi = 0.f;  // values of k-steps ss0 and ss0 + 1
                if (t < T && k < k_hi) {
                    __half* xp = x16 + (size_t)t * p.xs_stride + k;
                    const uint4 q = *reinterpret_cast<const uint4*>(xp);
                    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
                    uint4 o;
                    __half2* hh = reinterpret_cast<__half2*>(&o);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float scj = j < 2 ? sc[i] : sc[i] * 0.25f;  // 4^-ss, exact
                        const float2 f2 = __bfloat1622float2(b[j]);
                        hh[j] = __floats2half2_rn(f2.x * scj, f2.y * scj);
                        const float2 h2 = __half22float2(hh[j]);
                        (j < 2 ? s_lo : s_hi) += h2.x + h2.y;
                    }
                    *reinterpret_cast<uint4*>(xp) = o;
                }
                sacc[i] = s_lo + s_hi;
                uacc[i] = s_lo * (float)(1 << (2 * ss0)) + s_hi * (float)(4 << (2 * ss0));  // exact rescales
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    sacc[i] += __shfl_xor_sync(0xffffffffu, sacc[i], o);
                    uacc[i] += __shfl_xor_sync(0xffffffffu, uacc[i], o);
                }
            if (k < k_hi && (lane & 7) == 0)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (tb + i < T) xsum[(tb + i) * p.kblocks + k / kKBlock] = make_float2(sacc[i], uacc[i]);
        }
    }
    TRM(7);
    for (int64_t k = k_lo + lane * 8; k < k_hi; k += 256)
        *reinterpret_cast<uint4*>(x16 + (size_t)T * p.xs_stride + k) = make_uint4(0, 0, 0, 0);
    // per (token, group of this warp's k range) sums of the k-block sums, read once per group fold
    // instead of once per item: xgs[(wl * T + t) * gpw + lg], lg = local group (the first may be partial)
    const int kpg = p.single_group ? (1 << 30) : (int)(p.gs / kKBlock);  // k-blocks per group
    float2* xgs = reinterpret_cast<float2*>(smem + p.xgs_off);
    if (conv && kw1 > kw0) {
        __syncwarp();
        const int g_first = kw0 / kpg, n_lg = (kw1 - 1) / kpg - g_first + 1;
        for (int i = lane; i < T * n_lg; i += 32) {
            const int t = i / n_lg, lg = i % n_lg;
            const int b0 = max(kw0, (g_first + lg) * kpg), b1 = min(kw1, (g_first + lg + 1) * kpg);
            float sx = 0.f, su = 0.f;
            for (int b = b0; b < b1; ++b) {
                const float2 v = xsum[t * p.kblocks + b];
                sx += v.x, su += v.y;
            }
            xgs[(wl * T + t) * p.gpw + lg] = make_float2(sx, su);
        }
    }
    if (p.R > 1) __syncthreads();  // X, its sums and scales come from the first tile's warps
    else __syncwarp();

    // yt: this lane's outputs (rows g/g+8 of both row groups, tokens 8gi+2c / 8gi+2c+1 of token group
    // gi) over the slices each token uses; ys: the current slice's partials
    // A = sum_g s_g sum_k x (times kc[m] at the end, in units of the token scale); B = sum_g s_g z_g
    // sum_k x goes straight into slice 1's partials (slice 1 is every token's, scaled by the token scale)
    float yt[NG][2][4], ys[NG][2][4], A[NG][2][4], D[NG][2][4];
#pragma unroll
    for (int gi = 0; gi < NG; ++gi)
#pragma unroll
        for (int rg = 0; rg < 2; ++rg)
#pragma unroll
            for (int j = 0; j < 4; ++j) yt[gi][rg][j] = ys[gi][rg][j] = A[gi][rg][j] = D[gi][rg][j] = 0.f;
    TRM(1);
    const int g = lane >> 2, c = lane & 3;
    const __half* xr[NG];  // B-fragment token rows (row T is zeros)
    int tk0[NG], tk1[NG];  // this lane's D columns (tokens) per token group
    float es0[NG], es1[NG];
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
        const int tg = 8 * gi + g < T ? 8 * gi + g : T;
        xr[gi] = x16 + (size_t)tg * p.xs_stride + 16 * c;  // the lane's 16 values of every k-block
        tk0[gi] = 8 * gi + 2 * c;
        tk1[gi] = 8 * gi + 2 * c + 1;
        es0[gi] = tk0[gi] < T ? es_s[wl][tk0[gi]] : 0.f;
        es1[gi] = tk1[gi] < T ? es_s[wl][tk1[gi]] : 0.f;
    }
    int grp = 0, gleft = 0;
    // (2)-(4) one stream of (slice, k-block) items: slice 1's k-blocks (already in flight since the
    // prologue), then -- once the masks are known -- those of every other slice in the batch's union
    const int nk = kw1 - kw0;
    const int gleft0 = p.single_group ? (1 << 30) : kpg - (kw0 % kpg);  // k-blocks left in the first group
    const uint32_t magic = 0x64006400u;  // fp16 1024: (1024 + c) halves
    int n_items = nk, uni = 1;
    int mt0[NG], mt1[NG];
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) mt0[gi] = mt1[gi] = 0;
    int csi = 0, ckb = kw0, cslot = 0;  // consume cursor
    for (int ci = 0;; ++ci) {
        if (ci == nk) {
            TRM(2);
            // slice masks: gate_hard(delta) on S = sum over hidden tiles + b2 (router.hpp:92-103)
            grid_dep_wait2();
            TRM(3);
            if (p.masks) {
                if (tid < T) s_mask[tid] = (p.masks[tid] & p.vmask) | 1;
            } else {
                for (int i = warp; i < T * p.nr; i += kD2Warps) {
                    const int t = i / p.nr, k = i % p.nr;
                    float sc = 0.f;
                    for (int q = lane; q < p.n_mt; q += 32)
                        sc += __ldcg(p.spart + ((int64_t)q * p.t_all + p.t0 + t) * p.nr + k);
#pragma unroll
                    for (int o = 16; o; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
                    if (lane == 0) s_score[t][k] = sc + __ldg(p.b2 + k);
                }
                __syncthreads();
                if (tid < T) {
                    int m = 1;
                    for (int k = 0; k < p.nr; ++k) {
                        if ((s_score[tid][k] - p.delta) > 0.f) m |= 1 << (k + 1);
                        if (blockIdx.x == 0 && p.scores_out) p.scores_out[tid * p.nr + k] = s_score[tid][k];
                    }
                    s_mask[tid] = m;
                    if (blockIdx.x == 0) {
                        p.masks_dev[tid] = (uint8_t)m;
                        if (p.masks_out) p.masks_out[tid] = (uint8_t)m;
                    }
                }
            }
            __syncthreads();
            for (int t = 0; t < T; ++t) uni |= s_mask[t];
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                mt0[gi] = tk0[gi] < T ? s_mask[tk0[gi]] : 0;
                mt1[gi] = tk1[gi] < T ? s_mask[tk1[gi]] : 0;
            }
            int ns = 1;
            for (int e0 = 1; e0 < p.E; ++e0)
                if (uni >> e0 & 1) slist |= (uint32_t)e0 << (2 * ns++);
            n_items = nk * ns;
            seek();  // the issue cursor's slice is known now
            // burst: the union's first items (kD2Ring - 1 groups, padded with empty ones)
            for (int j = 0; j < kD2Ring - 1; ++j) {
                if (pi < n_items) issue();
                cp_commit();
            }
        }
        if (ci >= n_items) break;
        const int si = csi, kb = ckb, e0 = (int)(slist >> (2 * si)) & 3;
        if (++ckb == kw1) ckb = kw0, ++csi;
        // debug: per-item globaltimer marks of CTA 0's warps (before the wait, data in, issued)
        const bool tri = p.trace && blockIdx.x == 0 && lane == 0 && ci < 32;
        if (tri) p.trace[24576 + warp * 128 + ci * 4 + 0] = gtimer2();
        cp_wait<kD2Ring - 2>();
        const uint4 q = ring[cslot * 32 + lane];
        if (tri) p.trace[24576 + warp * 128 + ci * 4 + 1] = gtimer2() + (q.x & 0);
        cslot = cslot + 1 == kD2Ring ? 0 : cslot + 1;
        const uint32_t w0[4] = {q.x, q.y, q.z, q.w};
        const uint32_t w1[4] = {q.x >> 8, q.y >> 8, q.z >> 8, q.w >> 8};  // row group 1's fields
        uint4 xb[NG][2];  // B fragments of the four k-steps: (b0, b1) of k-step ss = words 2ss, 2ss + 1
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
            const uint4* xk = reinterpret_cast<const uint4*>(xr[gi] + (size_t)kb * kKBlock);
            xb[gi][0] = xk[0];
            xb[gi][1] = xk[1];
        }
        auto kstep = [&](auto SSc) {
            constexpr int SS = decltype(SSc)::value;
            const uint32_t a00 = frag<SS>(w0[0], magic), a01 = frag<SS>(w0[1], magic), a02 = frag<SS>(w0[2], magic),
                           a03 = frag<SS>(w0[3], magic);
            const uint32_t a10 = frag<SS>(w1[0], magic), a11 = frag<SS>(w1[1], magic), a12 = frag<SS>(w1[2], magic),
                           a13 = frag<SS>(w1[3], magic);
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {  // the A fragments serve every token group
                const uint4& v = xb[gi][SS / 2];
                const uint32_t b0 = SS % 2 ? v.z : v.x, b1 = SS % 2 ? v.w : v.y;
                mma_f16_acc(D[gi][0], a00, a01, a02, a03, b0, b1);
                mma_f16_acc(D[gi][1], a10, a11, a12, a13, b0, b1);
            }
        };
        kstep(std::integral_constant<int, 0>{});
        kstep(std::integral_constant<int, 1>{});
        kstep(std::integral_constant<int, 2>{});
        kstep(std::integral_constant<int, 3>{});
        // refill: item ci + R - 1 goes into the slot just consumed (its data is in registers)
        if (tri) p.trace[24576 + warp * 128 + ci * 4 + 2] = gtimer2() + (uint32_t)(D[0][0][0] != 0.f) * 0;
        if (pi < n_items && pi <= ci + kD2Ring - 1) issue();
        cp_commit();
        if (tri) p.trace[24576 + warp * 128 + ci * 4 + 3] = gtimer2();
        if (kb == kw0) {  // a slice starts: its group cursor
            grp = 0;
            gleft = gleft0;
        }
        const bool slice_end = kb + 1 == kw1;
        if (slice_end || --gleft == 0) {
            float xg0[NG], xg1[NG], xu0[NG], xu1[NG];  // the group's activation sums of the lane's tokens
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                const float2 s0 = tk0[gi] < T ? xgs[(wl * T + tk0[gi]) * p.gpw + grp] : make_float2(0.f, 0.f);
                const float2 s1 = tk1[gi] < T ? xgs[(wl * T + tk1[gi]) * p.gpw + grp] : make_float2(0.f, 0.f);
                xg0[gi] = s0.x, xu0[gi] = s0.y;
                xg1[gi] = s1.x, xu1[gi] = s1.y;
            }
#pragma unroll
            for (int rg = 0; rg < 2; ++rg) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // rows g and g+8 of the row group
                    const float2 sc = gcs[grp * 32 + 16 * rg + g + 8 * h];
#pragma unroll
                    for (int gi = 0; gi < NG; ++gi) {
                        ys[gi][rg][2 * h] = fmaf(D[gi][rg][2 * h] - 1024.f * xg0[gi], sc.x, ys[gi][rg][2 * h]);
                        ys[gi][rg][2 * h + 1] = fmaf(D[gi][rg][2 * h + 1] - 1024.f * xg1[gi], sc.x, ys[gi][rg][2 * h + 1]);
                        if (si == 0) {
                            A[gi][rg][2 * h] = fmaf(sc.x, xu0[gi], A[gi][rg][2 * h]);
                            A[gi][rg][2 * h + 1] = fmaf(sc.x, xu1[gi], A[gi][rg][2 * h + 1]);
                            ys[gi][rg][2 * h] = fmaf(-sc.y, xu0[gi], ys[gi][rg][2 * h]);
                            ys[gi][rg][2 * h + 1] = fmaf(-sc.y, xu1[gi], ys[gi][rg][2 * h + 1]);
                        }
                    }
                }
#pragma unroll
                for (int gi = 0; gi < NG; ++gi) D[gi][rg][0] = D[gi][rg][1] = D[gi][rg][2] = D[gi][rg][3] = 0.f;
            }
            ++grp;
            gleft = kpg;
        }
        if (slice_end) {  // the slice's partials go to the tokens that use it (slice 1: every token)
            const float fs = __int_as_float((127 - 2 * e0) << 23);  // 4^-e0: S 4^(4-e), S = s / 2^6, e = e0 + 1
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                const bool u0 = si == 0 || (mt0[gi] >> e0 & 1), u1 = si == 0 || (mt1[gi] >> e0 & 1);
                const float f0 = u0 ? fs * es0[gi] : 0.f, f1 = u1 ? fs * es1[gi] : 0.f;
#pragma unroll
                for (int rg = 0; rg < 2; ++rg) {
                    yt[gi][rg][0] = fmaf(ys[gi][rg][0], f0, yt[gi][rg][0]);
                    yt[gi][rg][2] = fmaf(ys[gi][rg][2], f0, yt[gi][rg][2]);
                    yt[gi][rg][1] = fmaf(ys[gi][rg][1], f1, yt[gi][rg][1]);
                    yt[gi][rg][3] = fmaf(ys[gi][rg][3], f1, yt[gi][rg][3]);
                    ys[gi][rg][0] = ys[gi][rg][1] = ys[gi][rg][2] = ys[gi][rg][3] = 0.f;
                }
            }
        }
    }
    cp_wait<0>();
    TRM(4);
    __syncthreads();  // x16 is dead: the reduction buffer aliases it

    // (5) warps' partials -> smem, then each (row, token) combines its slices in warp order
    {
        float* r = red + (size_t)warp * (NG * kD2Acc) * 32 + lane;
        int i = 0;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi)
#pragma unroll
            for (int rg = 0; rg < 2; ++rg)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    r[(i++) * 32] = yt[gi][rg][j];
                    r[(i++) * 32] = A[gi][rg][j] * (j & 1 ? es1[gi] : es0[gi]);  // exact: power of two
                }
    }
    __syncthreads();
    for (int i = tid; i < p.R * 32 * 8 * NG; i += kD2Threads) {
        const int rl = i % 32, t = (i / 32) % (8 * NG), j_tile = i / (32 * 8 * NG);
        const int64_t row = ((int64_t)blockIdx.x * p.R + j_tile) * 32 + rl;
        if (t < T && row < p.out) {
            const int gi = t / 8, tl = t % 8;
            const int rg = rl / 16, rr = rl % 16, g = rr % 8, hi = rr / 8;
            const int ln = g * 4 + tl / 2, j = hi * 2 + (tl & 1);
            const int base = ((gi * 2 + rg) * 4 + j) * 2;
            const float kc = p.mt.kc[s_mask[t]];
            float acc = 0.f;
            for (int w = j_tile * p.wpt; w < (j_tile + 1) * p.wpt; ++w) {
                const float* r = red + (size_t)w * (NG * kD2Acc) * 32 + ln;
                acc += r[(base + 0) * 32] + kc * r[(base + 1) * 32];
            }
            p.y[(int64_t)t * p.out + row] = __float2bfloat16_rn(acc);
        }
    }
    TRM(5);
}

}  // namespace

// 32-row tiles per CTA: the smallest R in {1, 2, 4, 8} whose CTAs fit one wave (a CTA's latency chain
// is serial, so a second wave costs as much as the first); 0 = the layer is too tall for this kernel
static int d2_tiles_per_cta(const mobi_layer* L) {
    const int64_t n_rt = cdiv(L->out, (int64_t)32);
    for (int r = 1; r <= 8; r *= 2)
        if (cdiv(n_rt, (int64_t)r) <= L->n_sm) return r;
    return 0;
}

static int d2_groups_per_warp(const mobi_layer* L, int wpt) {
    if (L->single_group) return 1;
    const int64_t kpw = cdiv(L->kblocks, (int64_t)wpt) * kKBlock;  // k per warp (upper bound)
    return (int)(kpw / L->gs + 2);
}

// dynamic shared memory: x16 rows 0..T (row T zeros) + per-(token, k-block) sums, aliased after the
// item loop by the warps' reduction buffer; then the staged group constants and the per-lane rings
struct D2Smem {
    size_t gcs_off, ring_off, xgs_off, total;
};
static D2Smem d2_smem(const mobi_layer* L, int64_t T, int R) {
    const int ng = T > 8 ? 2 : 1;
    const size_t xs = (size_t)(T + 1) * (L->in_pad + 8) * 2 + (size_t)T * L->kblocks * 8;
    D2Smem m;
    m.gcs_off = (std::max(xs, (size_t)kD2Warps * ng * kD2Acc * 32 * 4) + 15) / 16 * 16;
    m.ring_off = m.gcs_off + (size_t)kD2Warps * d2_groups_per_warp(L, kD2Warps / R) * 32 * 8;
    m.xgs_off = m.ring_off + (size_t)kD2Warps * kD2Ring * 32 * 16;
    m.total = m.xgs_off + (size_t)(kD2Warps / R) * T * d2_groups_per_warp(L, kD2Warps / R) * 8;
    return m;
}
// up to 8 tokens the kernel must leave room for the router's CTAs (co-residency under PDL)
constexpr size_t kD2SmemCoRes = 200 * 1024, kD2SmemMax = 225 * 1024;  // + static smem <= 227 KiB

bool decode_planes_supported(const mobi_layer* L, const void* x, int64_t T) {
    if (T < 1 || T > kD2MaxLaunchT || !L->dplanes || L->E > 4) return false;
    if (L->in % 8 != 0 || (reinterpret_cast<uintptr_t>(x) & 15u) != 0) return false;
    if (!L->single_group && L->gs % kKBlock != 0) return false;
    const int R = d2_tiles_per_cta(L);
    if (R == 0) return false;
    const int64_t Tg = std::min<int64_t>(T, kD2MaxT);
    return d2_smem(L, Tg, R).total <= (Tg > 8 ? kD2SmemMax : kD2SmemCoRes);
}

int launch_decode_planes(mobi_layer* L, const __nv_bfloat16* x, int64_t T, const uint8_t* given_masks, float delta,
                         uint8_t* masks_out, float* scores_out, __nv_bfloat16* y, bool pdl, cudaStream_t st,
                         unsigned long long* trace) {
    // one launch per <= kD2MaxT tokens (one or two m16n8k16 N groups); each decides its tokens' masks
    // from the router partials and streams only its own union of slices.  Under PDL the later groups'
    // prologue (activation staging, slice 1) overlaps the previous group's tail.
    {
        MOBI_TRY(func_attr_once(decode_planes_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kD2SmemMax));
        MOBI_TRY(func_attr_once(decode_planes_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kD2SmemMax));
    }
    for (int64_t t0 = 0; t0 < T; t0 += kD2MaxT) {
        const int64_t Tg = std::min<int64_t>(kD2MaxT, T - t0);
        D2Params p{};
        p.trace = t0 == 0 ? trace : nullptr;
        p.dplanes = reinterpret_cast<const uint4*>(L->dplanes);
        p.gconst = L->gconst;
        p.x = x + t0 * L->in;
        p.masks = given_masks ? given_masks + t0 : nullptr;
        p.spart = L->dec_spart;
        p.b2 = L->b2;
        p.masks_dev = L->masks + t0;
        p.masks_out = masks_out ? masks_out + t0 : nullptr;
        p.scores_out = scores_out ? scores_out + t0 * L->nr : nullptr;
        p.y = y + t0 * L->out;
        p.mt = L->mtab;
        p.out = L->out;
        p.out_pad = L->out_pad;
        p.in = L->in;
        p.in_pad = L->in_pad;
        p.kblocks = L->kblocks;
        p.gs = L->gs;
        p.delta = delta;
        p.single_group = L->single_group ? 1 : 0;
        p.T = (int)Tg;
        p.t0 = (int)t0;
        p.t_all = (int)T;
        p.E = L->E;
        p.nr = L->nr;
        p.n_mt = (int)(L->h_pad / 16);
        p.vmask = (1 << (L->nr + 1)) - 1;
        p.n_rt32 = (int)(L->out_pad / 32);
        p.xs_stride = (int)(L->in_pad + 8);
        p.R = d2_tiles_per_cta(L);
        p.wpt = kD2Warps / p.R;
        p.gpw = d2_groups_per_warp(L, p.wpt);
        const D2Smem sm = d2_smem(L, Tg, p.R);
        p.gcs_off = (int64_t)sm.gcs_off;
        p.ring_off = (int64_t)sm.ring_off;
        p.xgs_off = (int64_t)sm.xgs_off;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)cdiv(cdiv(L->out, (int64_t)32), (int64_t)p.R));
        cfg.blockDim = dim3(kD2Threads);
        cfg.dynamicSmemBytes = sm.total;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        if (Tg > 8)
            MOBI_CUDA(cudaLaunchKernelEx(&cfg, decode_planes_kernel<2>, p));
        else
            MOBI_CUDA(cudaLaunchKernelEx(&cfg, decode_planes_kernel<1>, p));
        ++L->last_launches;
        L->plan[1] = MOBI_K_GEMM_DECODE_PLANES;
        L->plan[2] = (int32_t)cfg.gridDim.x;
    }
    return MOBI_OK;
}

}  // namespace mobi
