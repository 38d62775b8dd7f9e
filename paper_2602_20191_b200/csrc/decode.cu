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
#ifndef MOBI_DEC_STAGES
#define MOBI_DEC_STAGES 8
#endif
constexpr int kDecStages = MOBI_DEC_STAGES;                    // 8 KiB code blocks in flight per CTA
constexpr int kRdWarps = 8;                      // router: warps per CTA (split K inside the CTA)
constexpr int kRdCluster = 2;                    // router: CTAs per hidden tile (split K across the cluster)
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
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
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
    unsigned long long* trace;  // debug: per-CTA globaltimer marks [cta][8]
};

// score() for T <= 32 tokens, no global synchronisation: a cluster of two CTAs owns one m16 tile of
// hidden units (rows of w1t) and splits K in halves; inside a CTA eight warps split the half again.
// Lane (g, c) of a warp owns hidden rows g and g+8 and, inside each 32-wide k chunk, the 8
// contiguous k at 8c: two 16-byte loads per row, each feeding two m16n8k16 steps (MMA k order is a
// permutation of memory order; X uses the same permutation, so the dot products are unchanged).
// Warp partials are summed in warp order in smem, the peer CTA's half is added through distributed
// shared memory (rank 0 + rank 1, fixed order), then silu(H + b1) . w2 over the tile's 16 hidden
// units gives the tile's partial scores spart[mt][t][k] (router.hpp:63-76).  The decode GEMM sums
// the tiles in order, adds b2 and applies gate_hard(delta).
// router: 32-k chunks in flight per lane -- 6, or fewer when that keeps every CTA of a tall router
// (down: 448 CTAs) in one wave (launch_router_dec)
__device__ __forceinline__ void rd_cp16(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
template <int NT, int kRdRing>
__global__ void __cluster_dims__(kRdCluster, 1, 1) __launch_bounds__(32 * kRdWarps)
    router_dec_kernel(const __grid_constant__ RDParams p) {
    static_assert(kRdRing >= 2, "ring");
    extern __shared__ __align__(16) uint8_t rd_ring[];  // [warps][kRdRing][32 lanes][2 + NT] x 16 B
    const int tcta = blockIdx.x;
    auto TRM = [&](int i) {
        if (p.trace && threadIdx.x == 0) p.trace[(size_t)tcta * 8 + i] = gtimer();
    };
    TRM(0);
    __shared__ float red[kRdWarps][kRdRows][8 * NT + 1];
    __shared__ float hsum[8 * NT][kRdRows];
    __shared__ float act[8 * NT][kRdRows];
    __shared__ float sb1[kRdRows], sw2[kRdRows * (kFastSlices - 1)];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, c = lane & 3;
    const uint32_t rank = cluster_ctarank();
    const int mt = blockIdx.x / kRdCluster;
    // the tile's b1 and w2 go out first: the epilogue must not wait on dependent global loads
    float pb1 = 0.f, pw2 = 0.f;
    if (tid < kRdRows) pb1 = __ldg(p.b1 + (int64_t)mt * kRdRows + tid);
    if (tid < kRdRows * p.nr) pw2 = __ldg(p.w2 + (int64_t)mt * kRdRows * p.nr + tid);
    const int64_t nchunks = p.in_pad / 32;
    const int64_t per_cta = (nchunks + kRdCluster - 1) / kRdCluster;
    const int64_t per_warp = (per_cta + kRdWarps - 1) / kRdWarps;
    const int64_t cta0 = rank * per_cta, cta1 = min(nchunks, cta0 + per_cta);
    const int64_t q0 = cta0 + warp * per_warp;
    const int64_t q1 = min(cta1, q0 + per_warp);
    float acc4[4][NT][4];  // four independent accumulator chains (HMMA dependent-issue latency)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc4[a][n][0] = acc4[a][n][1] = acc4[a][n][2] = acc4[a][n][3] = 0.f;
    const __nv_bfloat16* ar0 = p.w1t + ((int64_t)mt * kRdRows + g) * p.in_pad + 8 * c;
    const __nv_bfloat16* ar1 = ar0 + 8 * p.in_pad;
    // Per-lane cp.async ring: chunk q's two w1 vectors (rows g, g+8) and the X vectors of the lane's
    // tokens (8n + g) go into the lane's own slot, so kRdRing chunks are in flight per lane whatever
    // the register budget (the kernel shares the SM with the decode GEMM) and no lane reads another's.
    constexpr int kSlot = 2 + NT;  // 16-byte vectors per lane per chunk
    uint4* ring = reinterpret_cast<uint4*>(rd_ring) + ((size_t)warp * kRdRing * 32 + lane) * kSlot;
    int64_t qi = q0;  // next chunk to issue
    auto issue_w = [&](int64_t qq) {
        uint4* d = ring + (size_t)((qq - q0) % kRdRing) * 32 * kSlot;
        rd_cp16(d, ar0 + qq * 32, true);
        rd_cp16(d + 1, ar1 + qq * 32, true);
    };
    auto issue_x = [&](int64_t qq) {
        uint4* d = ring + (size_t)((qq - q0) % kRdRing) * 32 * kSlot;
        const int64_t k = qq * 32;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const int tok = 8 * n + g;
            const bool ok = tok < p.T && k + 8 * c < p.in;
            rd_cp16(d + 2 + n, ok ? (const void*)(p.x + (int64_t)tok * p.in + k + 8 * c) : (const void*)p.x, ok);
        }
    };
    auto issue = [&]() {
        issue_w(qi);
        issue_x(qi);
        asm volatile("cp.async.commit_group;" ::: "memory");
        ++qi;
    };
    // w1 is a constant: the first chunks stream in before the previous kernel in the stream has
    // finished (PDL); X -- possibly that kernel's output -- and every write wait for it
    while (qi < q1 && qi < q0 + kRdRing - 1) {
        issue_w(qi++);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    grid_dep_wait();
    // only now may the decode GEMM launch: it reads X before its own wait, and X may be the output of
    // the kernel this one just waited for
    grid_dep_launch();
    for (int64_t qq = q0; qq < qi; ++qq) issue_x(qq);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // the prologue chunks (w1 + X) have landed
    for (int64_t q = q0; q < q1; ++q) {
        const int64_t pend = qi - 1 - q;  // groups allowed to stay in flight
        if (pend >= kRdRing - 2) asm volatile("cp.async.wait_group %0;" ::"n"(kRdRing - 2) : "memory");
        else if (pend >= 2 && kRdRing > 4) asm volatile("cp.async.wait_group 2;" ::: "memory");
        else if (pend >= 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        const uint4* d = ring + (size_t)((q - q0) % kRdRing) * 32 * kSlot;
        const uint4 a0 = d[0], a1 = d[1];
        auto step = [&](float (&c0)[NT][4], float (&c1)[NT][4]) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const uint4 b = d[2 + n];
                mma_bf16(c0[n], a0.x, a1.x, a0.y, a1.y, b.x, b.y);
                mma_bf16(c1[n], a0.z, a1.z, a0.w, a1.w, b.z, b.w);
            }
        };
        if (((q - q0) & 1) == 0) step(acc4[0], acc4[1]);
        else step(acc4[2], acc4[3]);
        if (qi < q1) issue();  // refills the slot just read (its data is in registers)
    }
    TRM(1);
    if (tid < kRdRows) sb1[tid] = pb1;
    if (tid < kRdRows * p.nr) sw2[tid] = pw2;
    float acc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[n][j] = (acc4[0][n][j] + acc4[1][n][j]) + (acc4[2][n][j] + acc4[3][n][j]);
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
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kRdWarps; ++w) s += red[w][row][tok];
        hsum[tok][row] = s;
    }
    cluster_sync();  // both halves of K summed in their CTA
    if (rank == 0) {
        const uint32_t peer = mapa_shared(smem_u32(&hsum[0][0]), 1);
        for (int i = tid; i < kRdRows * 8 * NT; i += 32 * kRdWarps) {
            const int row = i % kRdRows, tok = i / kRdRows;
            float other;
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(other) : "r"(peer + (uint32_t)(tok * kRdRows + row) * 4u));
            const int64_t j = (int64_t)mt * kRdRows + row;
            float v = 0.f;
            if (j < p.h && tok < p.T) {
                const float a = hsum[tok][row] + other + sb1[row];
                v = a * __fdividef(1.f, 1.f + __expf(-a));
            }
            act[tok][row] = v;
        }
    }
    cluster_sync();  // the peer's smem stays alive until rank 0 has read it
    if (rank != 0) return;
    for (int i = tid; i < p.T * p.nr; i += 32 * kRdWarps) {
        const int tok = i / p.nr, k = i % p.nr;
        float s = 0.f;
#pragma unroll
        for (int row = 0; row < kRdRows; ++row) s += act[tok][row] * sw2[row * p.nr + k];
        p.spart[((int64_t)mt * p.T + tok) * p.nr + k] = s;
    }
    TRM(2);
}

// ============================================================================================
// decode GEMM
// ============================================================================================
struct DParams {
    const uint8_t* codes8;    // tiled merged codes [out_pad/128][kblocks][8192]
    const float2* gconst;     // [G][out_pad] (s, s*z)
    const __nv_bfloat16* x;   // [T][in]
    const uint8_t* masks;     // [T] given masks (forward_masked), else null: decided here from spart
    const float* spart;       // [n_mt][T][nr] router tile partial scores (router_dec_kernel)
    const float* b2;          // [nr]
    float delta;
    int n_mt, nr;
    uint8_t* masks_dev;       // decided masks -> L->masks (CTA 0)
    uint8_t* masks_out;       // optional
    float* scores_out;        // optional [T][nr]
    __nv_bfloat16* y;         // [T][out]
    float* part;              // [(n_cta + n_rt)][T][128] row-tile partials
    int* cnt;                 // [n_rt] arrival counters (zero between launches)
    MaskTable mt;
    int64_t out, out_pad, in, kblocks, gs, U;
    int T, n_cta, len_max, xs_stride, single_group, vmask;
    unsigned long long* trace;  // debug: per-CTA globaltimer marks [cta][8] (after the router's 2048)
};

struct DecSmem {
    size_t ring, full, empty, xs, x16, total;
};
constexpr int kDecStageBytes = kBlockBytes + kRowTile * 8;  // 8 KiB codes + the block's 128 (s, s*z) pairs
__host__ __device__ inline DecSmem dec_smem(int T, int len_max, int xs_stride) {
    DecSmem s;
    s.ring = 0;
    s.full = s.ring + (size_t)kDecStages * kDecStageBytes;
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
    __shared__ float s_escale[kDecMaxT + 1];
    __shared__ float s_score[kDecMaxT][kFastSlices - 1];
    __shared__ int s_mask[kDecMaxT];
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
    auto TRM = [&](int i) {
        if (p.trace && threadIdx.x == 0) p.trace[(size_t)(2048 + cta) * 8 + i] = gtimer();
    };
    TRM(0);
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
    // one stage = the 8 KiB code block of unit u plus its 128 rows' group constants (1 KiB, contiguous
    // in the [G][out_pad] layout)
    // producer cursor (unit u = rt * kbn + kb), advanced incrementally: no 64-bit divisions per block
    int64_t pu = u0, prt = u0 / kbn;
    int pkb = (int)(u0 - prt * kbn);
    auto issue = [&](int sidx) {
        const int64_t grp = p.single_group ? 0 : ((int64_t)pkb * kKBlock) / p.gs;
        uint8_t* dst = ring + (size_t)sidx * kDecStageBytes;
        fence_proxy_async_smem();  // the MMA warps' reads of a recycled stage precede the copy into it
        mbar_arrive_expect_tx(&full[sidx], kDecStageBytes);
        bulk_load(dst, p.codes8 + pu * kBlockBytes, kBlockBytes, &full[sidx], pol);
        bulk_load(dst + kBlockBytes, p.gconst + grp * p.out_pad + prt * kRowTile, kRowTile * 8, &full[sidx], pol);
        ++pu;
        if (++pkb == kbn) pkb = 0, ++prt;
    };
    if (threadIdx.x == 0) {
        pol = policy_evict_first();
        for (int64_t it = 0; it < nblk && it < kDecStages; ++it) issue((int)it);
    }

    // ---------------- MMA warps ----------------
    const int tid = threadIdx.x;  // 0 .. 32*kDecWarps-1
    const int kb_start = (int)(u0 % kbn);
    const int len = (int)(u1 - u0 < kbn ? u1 - u0 : kbn);
    // (1) activations of the k-blocks this CTA touches -> fp16, scaled per token by 2^-e so that
    //     max|x| lands in [2^14, 2^15) (exact, as the bucketed path's gather); X was produced before
    //     the router started, so this overlaps the router.
    // (a) raw bf16 rows of X for the k-blocks this CTA touches -> smem (one global round trip), zero
    //     row T (empty MMA columns) and zero tails past `in`
    const int nvec = len * 8;  // 16-byte vectors per token
    {
        constexpr int UX = 4;
        for (int v0 = tid; v0 < (T + 1) * nvec; v0 += UX * 32 * kDecWarps) {
            uint4 q[UX];
#pragma unroll
            for (int u = 0; u < UX; ++u) {
                const int v = v0 + u * 32 * kDecWarps;
                const int t = v / nvec, r = v % nvec;
                const int64_t k = (int64_t)((kb_start + r / 8) % kbn) * kKBlock + (r % 8) * 8;
                q[u] = (v < (T + 1) * nvec && t < T && k < p.in)
                           ? __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.in + k))
                           : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < UX; ++u) {
                const int v = v0 + u * 32 * kDecWarps;
                if (v < (T + 1) * nvec)
                    *reinterpret_cast<uint4*>(x16 + (size_t)(v / nvec) * p.xs_stride + (v % nvec) * 8) = q[u];
            }
        }
    }
    bar_mma();
    // (b) one warp per token: max|x| over the CTA's k range -> 2^-e so that it lands in [2^14, 2^15)
    //     (exact, as the bucketed path's gather), converted to fp16 in place
    for (int t = warp; t < T; t += kDecWarps) {
        uint4* row = reinterpret_cast<uint4*>(x16 + (size_t)t * p.xs_stride);
        float m = 0.f;
        for (int r = lane; r < nvec; r += 32) {
            const uint4 q = row[r];
            const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(b[j]);
                m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        int e = 0;
        if (m > 0.f && isfinite(m)) e = ilogbf(m) - 14;
        const float sc = ldexpf(1.f, -e);
        if (lane == 0) s_escale[t] = ldexpf(1.f, e);
        for (int r = lane; r < nvec; r += 32) {
            const uint4 q = row[r];
            const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
            uint4 o;
            __half2* h = reinterpret_cast<__half2*>(&o);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(b[j]);
                h[j] = __floats2half2_rn(f.x * sc, f.y * sc);
            }
            row[r] = o;
        }
    }
    if (tid == 0) s_escale[T] = 0.f;
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
    TRM(1);
    grid_dep_wait();
    TRM(2);
    // (3) slice masks: gate_hard(delta) on S = sum over hidden tiles (fixed order) + b2
    //     (router.hpp:92-103), or the caller's masks
    if (p.masks) {
        for (int t = tid; t < T; t += 32 * kDecWarps) s_mask[t] = (p.masks[t] & p.vmask) | 1;
    } else {
        // one warp per (token, slice): lane-strided partial sums over the hidden tiles, then a fixed
        // butterfly (deterministic)
        for (int i = warp; i < T * p.nr; i += kDecWarps) {
            const int t = i / p.nr, k = i % p.nr;
            float sc = 0.f;
            for (int q = lane; q < p.n_mt; q += 32) sc += __ldcg(p.spart + ((int64_t)q * T + t) * p.nr + k);
#pragma unroll
            for (int o = 16; o; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
            if (lane == 0) s_score[t][k] = sc + __ldg(p.b2 + k);
        }
        bar_mma();
        for (int t = tid; t < T; t += 32 * kDecWarps) {
            int m = 1;
            for (int k = 0; k < p.nr; ++k) {
                if ((s_score[t][k] - p.delta) > 0.f) m |= 1 << (k + 1);
                if (cta == 0 && p.scores_out) p.scores_out[t * p.nr + k] = s_score[t][k];
            }
            s_mask[t] = m;
            if (cta == 0) {
                p.masks_dev[t] = (uint8_t)m;
                if (p.masks_out) p.masks_out[t] = (uint8_t)m;
            }
        }
    }
    bar_mma();
    if (warp == 0) {
        for (int i = lane; i < MAXT * 8; i += 32) s_ttok[i / 8][i % 8] = T;
        __syncwarp();
        const int m = lane < T ? s_mask[lane] : -1;
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
    int64_t rt = u0 / kbn;
    int kb = (int)(u0 - rt * kbn), slot = 0;
    for (int it = 0; it < (int)nblk; ++it) {
        if (it > 0) {  // advance the consumer cursor
            if (++kb == kbn) kb = 0, ++rt;
            if (++slot == kbn) slot = 0;
        }
        if (rt != cur_rt) {
            if (cur_rt >= 0) flush(cur_rt);
            cur_rt = rt;
#pragma unroll
            for (int i = 0; i < MAXT; ++i) yp[i][0] = yp[i][1] = yp[i][2] = yp[i][3] = 0.f;
        }
        if (threadIdx.x == 0 && it >= 1 && it - 1 + kDecStages < nblk) {
            // refill the stage every warp released in the previous iteration
            const int j = it - 1;
            const int sj = j % kDecStages;
            mbar_wait(&empty[sj], (uint32_t)((j / kDecStages) & 1));
            issue(sj);
        }
        const int s = it % kDecStages;
        if (p.trace && threadIdx.x == 32 * (kDecWarps - 1) && cta < 4 && it < 32) p.trace[24576 + cta * 64 + it] = gtimer();
        mbar_wait(&full[s], (uint32_t)((it / kDecStages) & 1));
        if (p.trace && threadIdx.x == 32 * (kDecWarps - 1) && cta < 4 && it < 32) p.trace[24576 + cta * 64 + 32 + it] = gtimer();
        const uint8_t* blk = ring + (size_t)s * kDecStageBytes;
        const float2* gst = reinterpret_cast<const float2*>(blk + kBlockBytes);
        const float2 g0 = gst[rl0], g1 = gst[rl1];
        const uint4 q0 = *reinterpret_cast<const uint4*>(blk + (c * kRowTile + rl0) * 16);
        const uint4 q1 = *reinterpret_cast<const uint4*>(blk + (c * kRowTile + rl1) * 16);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // g0/g1 and q0/q1 are in registers
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
            // four independent accumulators: the legacy HMMA path has a long dependent-issue latency
            float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
            float c2[4] = {0.f, 0.f, 0.f, 0.f}, c3[4] = {0.f, 0.f, 0.f, 0.f};
            mma_f16(c0, A[0], A[8], A[1], A[9], b0.x, b0.y);
            mma_f16(c1, A[2], A[10], A[3], A[11], b0.z, b0.w);
            mma_f16(c2, A[4], A[12], A[5], A[13], b1.x, b1.y);
            mma_f16(c3, A[6], A[14], A[7], A[15], b1.z, b1.w);
            float acc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = (c0[j] + c1[j]) + (c2[j] + c3[j]);
            const float x0 = xsb[tk0[i]], x1 = xsb[tk1[i]];
            yp[i][0] = fmaf(fmaf(a0, acc[0], br0 * x0), es0[i], yp[i][0]);
            yp[i][1] = fmaf(fmaf(a0, acc[1], br0 * x1), es1[i], yp[i][1]);
            yp[i][2] = fmaf(fmaf(a1, acc[2], br1 * x0), es0[i], yp[i][2]);
            yp[i][3] = fmaf(fmaf(a1, acc[3], br1 * x1), es1[i], yp[i][3]);
        }
    }
    TRM(3);
    if (cur_rt >= 0) flush(cur_rt);
    TRM(4);
}


// ============================================================================================
// decode GEMV (T <= kFmaMaxT): CUDA-core FMAs on exact integer codes
// ============================================================================================
// At one to four tokens the contraction is far below any tensor-core tile, and the layer is bound by
// streaming the code bytes.  Thread (h, row) of a CTA owns one weight row of the 128-row tile and
// one 32-k half of every 64-k block: per block it turns its 32 merged codes into exact fp32 integers
// v = INT & maskbyte(m_t) (PRMT into 2^23 + v, FADD -2^23), accumulates x_t . v in fp32 (products
// of bf16 x and 8-bit v are exact) and folds the group constants
//      y_t += S_g * acc + (s_g * kc[m_t] - s_g * z_g) * sum_x        (mobi_internal.cuh)
// Code blocks and their group constants stream through the same TMA ring as decode_gemm_kernel;
// row tiles shared by several CTAs are reduced in CTA order by the last one to finish.
constexpr int kFmaMaxT = 4;

struct FmaSmem {
    size_t ring, full, empty, x32, xsum, total;
};
// a stage holds kFmaGroup consecutive code blocks (contiguous in codes8) and their constants, so
// the barrier round trips (each mbarrier wait/arrive costs hundreds of cycles of issue latency) are
// paid once per kFmaGroup blocks
#ifndef MOBI_FMA_CPS
#define MOBI_FMA_CPS 2
#endif
constexpr int kFmaCps = MOBI_FMA_CPS;  // CTAs per SM
constexpr int kFmaGroup = 4, kFmaStages = kFmaCps == 1 ? 4 : 2;
constexpr int kFmaWarps = 8, kFmaThreads = 32 * kFmaWarps;  // (small enough to co-reside with the router under PDL)
constexpr int kFmaParts = kFmaWarps / 4;                       // threads per weight row (k parts of a block)
constexpr int kFmaK = kKBlock / kFmaParts;                     // k per thread per block
constexpr int kFmaStageBytes = kFmaGroup * kDecStageBytes;
__host__ __device__ inline FmaSmem fma_smem(int T, int len_max) {
    FmaSmem s;
    s.ring = 0;
    s.full = s.ring + (size_t)kFmaStages * kFmaStageBytes;
    s.empty = s.full + kFmaStages * 8;
    s.x32 = s.empty + kFmaStages * 8;
    s.xsum = s.x32 + (size_t)T * len_max * kKBlock * 4;
    s.total = s.xsum + (size_t)T * len_max * kFmaParts * 4;
    return s;
}

template <int NT>
__global__ void __launch_bounds__(kFmaThreads, kFmaCps) decode_fma_kernel(const __grid_constant__ DParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ float s_score[kDecMaxT][kFastSlices - 1];
    __shared__ int s_mask[kDecMaxT];
    __shared__ float red[kFmaParts - 1][NT][kRowTile];
    __shared__ int s_flag;
    const int T = p.T;  // <= NT
    const FmaSmem L = fma_smem(NT, p.len_max);
    uint8_t* ring = smem + L.ring;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.full);
    uint64_t* empty = reinterpret_cast<uint64_t*>(smem + L.empty);
    float* x32 = reinterpret_cast<float*>(smem + L.x32);
    float* xsum = reinterpret_cast<float*>(smem + L.xsum);

    const int tid = threadIdx.x, warp = warp_idx_uniform(), lane = tid & 31;
    const int qq = warp / 4;            // k part of each 64-k block (warp-uniform): kFmaK consecutive k
    const int row = tid % kRowTile;     // weight row inside the tile
    const int cta = blockIdx.x;
    auto TRM = [&](int i) {
        if (p.trace && tid == 0) p.trace[(size_t)(2048 + cta) * 8 + i] = gtimer();
    };
    TRM(0);
    if (p.trace && tid == 0) p.trace[(size_t)(2048 + cta) * 8 + 7] = (unsigned long long)clock64();
    const int64_t u0 = (int64_t)cta * p.U / p.n_cta, u1 = (int64_t)(cta + 1) * p.U / p.n_cta;
    const int64_t kbn = p.kblocks;
    if (tid == 0) {
        for (int s = 0; s < kFmaStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kFmaWarps);
        }
        fence_barrier_init();
    }
    const int nblk = (int)(u1 - u0);
    const int nstage = (nblk + kFmaGroup - 1) / kFmaGroup;
    // (1a) issue this CTA's X loads before the code prefetch so they are not queued behind it
    const int kb_start = (int)(u0 % kbn);
    const int len = (int)(u1 - u0 < kbn ? u1 - u0 : kbn);
    const int nvec = len * 8;  // 8-element vectors per token
    constexpr int kXV = 4;     // vectors per thread held in registers (T * nvec <= kXV * 256 covered here)
    uint4 xq[kXV];
#pragma unroll
    for (int j = 0; j < kXV; ++j) {
        const int v = tid + j * kFmaThreads;
        const int t = v / nvec, r = v % nvec;
        const int64_t k = (int64_t)((kb_start + r / 8) % kbn) * kKBlock + (r % 8) * 8;
        xq[j] = (v < NT * nvec && t < T && k < p.in) ? __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.in + k))
                                                      : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    uint64_t pol = 0;
    int64_t pu = u0, prt = u0 / kbn;
    int pkb = (int)(u0 - prt * kbn);
    auto issue = [&](int sidx, int nb) {  // nb consecutive blocks: one code copy + one constants copy each
        uint8_t* dst = ring + (size_t)sidx * kFmaStageBytes;
        fence_proxy_async_smem();  // the FMA warps' reads of a recycled stage precede the copy into it
        mbar_arrive_expect_tx(&full[sidx], nb * kDecStageBytes);
        bulk_load(dst, p.codes8 + pu * kBlockBytes, nb * kBlockBytes, &full[sidx], pol);
        for (int j = 0; j < nb; ++j) {
            const int64_t grp = p.single_group ? 0 : ((int64_t)pkb * kKBlock) / p.gs;
            bulk_load(dst + kFmaGroup * kBlockBytes + j * kRowTile * 8, p.gconst + grp * p.out_pad + prt * kRowTile,
                      kRowTile * 8, &full[sidx], pol);
            ++pu;
            if (++pkb == kbn) pkb = 0, ++prt;
        }
    };
    if (tid == 0) {
        pol = policy_evict_first();
        for (int st = 0; st < nstage && st < kFmaStages; ++st) issue(st, min(kFmaGroup, nblk - st * kFmaGroup));
    }
    // (1b) X (bf16 -> fp32, exact) for the k-blocks this CTA touches; zero past `in`
    for (int v = tid; v < NT * nvec; v += kFmaThreads) {
        const int t = v / nvec, r = v % nvec;
        const int64_t k = (int64_t)((kb_start + r / 8) % kbn) * kKBlock + (r % 8) * 8;
        uint4 q = make_uint4(0, 0, 0, 0);
        const int j = (v - tid) / (kFmaThreads);
        if (j < kXV) {
#pragma unroll
            for (int jj = 0; jj < kXV; ++jj)
                if (jj == j) q = xq[jj];
        } else if (t < T && k < p.in) {
            q = __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.in + k));
        }
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
        float4 lo, hi;
        float2 f;
        f = __bfloat1622float2(b[0]); lo.x = f.x; lo.y = f.y;
        f = __bfloat1622float2(b[1]); lo.z = f.x; lo.w = f.y;
        f = __bfloat1622float2(b[2]); hi.x = f.x; hi.y = f.y;
        f = __bfloat1622float2(b[3]); hi.z = f.x; hi.w = f.y;
        float4* dst = reinterpret_cast<float4*>(x32 + (size_t)t * len * kKBlock + r * 8);
        dst[0] = lo;
        dst[1] = hi;
    }
    __syncthreads();
    for (int i = tid; i < NT * len * kFmaParts; i += kFmaThreads) {  // per (token, block, part) sums
        const float* r = x32 + (size_t)i * kFmaK;  // [t][slot][part][kFmaK] is contiguous
        float sacc = 0.f;
#pragma unroll
        for (int j = 0; j < kFmaK; ++j) sacc += r[j];
        xsum[i] = sacc;
    }
    TRM(1);
    grid_dep_wait();
    TRM(2);
    // (2) slice masks (as decode_gemm_kernel)
    if (p.masks) {
        if (tid < T) s_mask[tid] = (p.masks[tid] & p.vmask) | 1;
    } else {
        for (int i = warp; i < T * p.nr; i += kFmaWarps) {
            const int t = i / p.nr, k = i % p.nr;
            float sc = 0.f;
            for (int q = lane; q < p.n_mt; q += 32) sc += __ldcg(p.spart + ((int64_t)q * T + t) * p.nr + k);
#pragma unroll
            for (int o = 16; o; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
            if (lane == 0) s_score[t][k] = sc + __ldg(p.b2 + k);
        }
        __syncthreads();
        if (tid < T) {
            int m = 1;
            for (int k = 0; k < p.nr; ++k) {
                if ((s_score[tid][k] - p.delta) > 0.f) m |= 1 << (k + 1);
                if (cta == 0 && p.scores_out) p.scores_out[tid * p.nr + k] = s_score[tid][k];
            }
            s_mask[tid] = m;
            if (cta == 0) {
                p.masks_dev[tid] = (uint8_t)m;
                if (p.masks_out) p.masks_out[tid] = (uint8_t)m;
            }
        }
    }
    __syncthreads();
    uint32_t mw[NT];
    float kcm[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int m = t < T ? s_mask[t] : 1;
        mw[t] = p.mt.maskword[m];
        kcm[t] = p.mt.kc[m];
    }
    const float inv2p = p.mt.inv_2p;
    float yp[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) yp[t] = 0.f;

    auto flush = [&](int64_t rt) {
        // the k parts of each row: parts 1.. hand their partials to part 0 (fixed order)
        if (qq > 0)
#pragma unroll
            for (int t = 0; t < NT; ++t) red[qq - 1][t][row] = yp[t];
        __syncthreads();
        const int lo = cta_of(rt * kbn, p.U, p.n_cta), hi = cta_of(rt * kbn + kbn - 1, p.U, p.n_cta);
        const int64_t R = rt * kRowTile + row;
        if (qq == 0) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (t >= T) break;
                float v = yp[t];
#pragma unroll
                for (int q = 0; q < kFmaParts - 1; ++q) v += red[q][t][row];
                if (lo == hi) {
                    if (R < p.out) p.y[(int64_t)t * p.out + R] = __float2bfloat16_rn(v);
                } else {
                    p.part[(((int64_t)cta + rt) * T + t) * kRowTile + row] = v;
                }
            }
        }
        if (lo != hi) {
            __threadfence();
            __syncthreads();
            if (tid == 0) s_flag = atomicAdd(&p.cnt[rt], 1) == hi - lo;
            __syncthreads();
            if (s_flag) {
                __threadfence();
                for (int i = tid; i < T * kRowTile; i += kFmaThreads) {
                    const int t = i / kRowTile, rl = i % kRowTile;
                    const int64_t Rr = rt * kRowTile + rl;
                    if (Rr >= p.out) continue;
                    float sacc = 0.f;
                    for (int j = lo; j <= hi; ++j) sacc += __ldcg(p.part + (((int64_t)j + rt) * T + t) * kRowTile + rl);
                    p.y[(int64_t)t * p.out + Rr] = __float2bfloat16_rn(sacc);
                }
                if (tid == 0) p.cnt[rt] = 0;
            }
        }
        __syncthreads();
    };

    int64_t rt = u0 / kbn, cur_rt = -1;
    int kb = (int)(u0 - rt * kbn), slot = 0;
    for (int st = 0; st < nstage; ++st) {
        if (tid == 0 && st >= 1 && st - 1 + kFmaStages < nstage) {
            // refill the stage every warp released after the previous group
            const int j = st - 1;
            const int sj = j % kFmaStages;
            mbar_wait(&empty[sj], (uint32_t)((j / kFmaStages) & 1));
            if (p.trace && cta < 4 && st < 32) p.trace[24576 + 256 + cta * 64 + st] = gtimer();
            const int jn = j + kFmaStages;
            issue(sj, min(kFmaGroup, nblk - jn * kFmaGroup));
        }
        const int s = st % kFmaStages;
        if (p.trace && tid == 32 * (kFmaWarps - 1) && cta < 4 && st < 32) p.trace[24576 + cta * 64 + st] = gtimer();
        mbar_wait(&full[s], (uint32_t)((st / kFmaStages) & 1));
        if (p.trace && tid == 32 * (kFmaWarps - 1) && cta < 4 && st < 32) p.trace[24576 + cta * 64 + 32 + st] = gtimer();
        const uint8_t* stage = ring + (size_t)s * kFmaStageBytes;
        const int nb = min(kFmaGroup, nblk - st * kFmaGroup);
        for (int jb = 0; jb < nb; ++jb) {
            if (st > 0 || jb > 0) {  // advance the block cursor
                if (++kb == kbn) kb = 0, ++rt;
                if (++slot == kbn) slot = 0;
            }
            if (rt != cur_rt) {
                if (cur_rt >= 0) flush(cur_rt);
                cur_rt = rt;
#pragma unroll
                for (int t = 0; t < NT; ++t) yp[t] = 0.f;
            }
            const uint8_t* blk = stage + jb * kBlockBytes;
            const float2 g = reinterpret_cast<const float2*>(stage + kFmaGroup * kBlockBytes + jb * kRowTile * 8)[row];
            uint32_t w[kFmaK / 4];
#pragma unroll
            for (int c = 0; c < kFmaK / 16; ++c) {
                const uint4 qv = *reinterpret_cast<const uint4*>(blk + ((qq * (kFmaK / 16) + c) * kRowTile + row) * 16);
                w[4 * c] = qv.x, w[4 * c + 1] = qv.y, w[4 * c + 2] = qv.z, w[4 * c + 3] = qv.w;
            }
            const float S = g.x * inv2p;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (t >= T) break;
                const float4* xr = reinterpret_cast<const float4*>(x32 + ((size_t)t * len + slot) * kKBlock + qq * kFmaK);
                float a0 = 0.f, a1 = 0.f;  // two chains
#pragma unroll
                for (int wi = 0; wi < kFmaK / 4; ++wi) {
                    const uint32_t v = w[wi] & mw[t];
                    const float4 xv = xr[wi];
                    const float f0 = __int_as_float(__byte_perm(v, 0x4B000000u, 0x7540)) - 8388608.f;
                    const float f1 = __int_as_float(__byte_perm(v, 0x4B000000u, 0x7541)) - 8388608.f;
                    const float f2 = __int_as_float(__byte_perm(v, 0x4B000000u, 0x7542)) - 8388608.f;
                    const float f3 = __int_as_float(__byte_perm(v, 0x4B000000u, 0x7543)) - 8388608.f;
                    a0 = fmaf(xv.x, f0, a0);
                    a1 = fmaf(xv.y, f1, a1);
                    a0 = fmaf(xv.z, f2, a0);
                    a1 = fmaf(xv.w, f3, a1);
                }
                const float xs = xsum[((size_t)t * len + slot) * kFmaParts + qq];
                yp[t] = fmaf(S, a0 + a1, fmaf(fmaf(g.x, kcm[t], -g.y), xs, yp[t]));
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    TRM(3);
    if (cur_rt >= 0) flush(cur_rt);
    TRM(4);
    if (p.trace && tid == 0) {  // SM clock: cycles and ns over the whole CTA
        p.trace[(size_t)(2048 + cta) * 8 + 5] = (unsigned long long)clock64();
        p.trace[(size_t)(2048 + cta) * 8 + 6] = gtimer();
    }
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
    d.n_cta = (int)std::min<int64_t>(L->n_sm, d.U);
    d.len_max = (int)std::min<int64_t>(cdiv(d.U, d.n_cta), L->kblocks);
    d.xs_stride = d.len_max * kKBlock + 8;  // row stride = 16 mod 128 bytes: conflict-free B loads
    d.smem = dec_smem((int)T, d.len_max, d.xs_stride).total;
    return d;
}

constexpr size_t kDecSmemMax = 200 * 1024;
int g_dec_fma = 1;  // development switch: 0 = mma.sync decode kernel for every T

template <int NT>
int launch_decode_fma_t(mobi_layer* L, const DParams& p, size_t smem, bool pdl, cudaStream_t st) {
    {
        MOBI_TRY(func_attr_once(decode_fma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kDecSmemMax));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.n_cta);
    cfg.blockDim = dim3(kFmaThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    MOBI_CUDA(cudaLaunchKernelEx(&cfg, decode_fma_kernel<NT>, p));
    ++L->last_launches;
    L->plan[1] = MOBI_K_GEMM_DECODE_MERGED;
    L->plan[2] = p.n_cta;
    return MOBI_OK;
}

template <int MAXT>
int launch_decode_gemm_t(mobi_layer* L, const DParams& p, size_t smem, bool pdl, cudaStream_t st) {
    {
        MOBI_TRY(func_attr_once(decode_gemm_kernel<MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kDecSmemMax));
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
    L->plan[1] = MOBI_K_GEMM_DECODE_MERGED;
    L->plan[2] = p.n_cta;
    return MOBI_OK;
}

}  // namespace

bool decode_supported(const mobi_layer* L, const void* x, int64_t T) {
    if (L->generic || T < 1 || T > kDecMaxT) return false;
    if (L->in % 8 != 0 || (reinterpret_cast<uintptr_t>(x) & 15u) != 0) return false;
    if (!L->single_group && L->gs % kKBlock != 0) return false;
    return plan_decode(L, T).smem <= kDecSmemMax;
}

int launch_router_dec(mobi_layer* L, const __nv_bfloat16* x, int64_t T, float delta, uint8_t* masks_out,
                      float* scores_out, cudaStream_t st, unsigned long long* trace) {
    RDParams p{};
    p.trace = trace;
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
    const dim3 grid((unsigned)(n_mt * kRdCluster));
    auto smem_of = [](int nt, int ring) { return (size_t)kRdWarps * ring * 32 * (2 + nt) * 16; };
    // PDL: the router's CTAs may launch while the previous kernel (e.g. the last layer's decode GEMM)
    // drains and prefetch their first w1 chunks; griddepcontrol.wait guards X and every write
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(32 * kRdWarps);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int nt = T <= 8 ? 1 : T <= 16 ? 2 : 4;
    // the deepest ring whose occupancy keeps the whole grid in one wave: a CTA streams its share of w1
    // as one latency chain, so a second wave (4 CTAs past 3 per SM on down) doubles the router
    static int occ[3][3] = {};  // [nt 1/2/4][ring 6/4/2] CTAs per SM, queried once
    const int nti = nt == 1 ? 0 : nt == 2 ? 1 : 2;
    int ring = 6;
    for (int ri = 0; ri < 3; ++ri) {
        const int r = ri == 0 ? 6 : ri == 1 ? 4 : 2;
        const void* fn = nullptr;
        switch (nti * 3 + ri) {
#define RD_FN(i, N, R) case i: fn = reinterpret_cast<const void*>(router_dec_kernel<N, R>); break;
            RD_FN(0, 1, 6) RD_FN(1, 1, 4) RD_FN(2, 1, 2) RD_FN(3, 2, 6) RD_FN(4, 2, 4) RD_FN(5, 2, 2)
            RD_FN(6, 4, 6) RD_FN(7, 4, 4) RD_FN(8, 4, 2)
#undef RD_FN
        }
        // run with the SM configured for maximum shared memory, so the decode GEMV that follows (PDL)
        // can be co-resident while the router streams w1 (per device, once)
        MOBI_TRY(func_attr_once(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared));
        MOBI_TRY(func_attr_once(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_of(nt, r)));
        if (!occ[nti][ri]) {
            int n = 0;
            MOBI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, 32 * kRdWarps, smem_of(nt, r)));
            occ[nti][ri] = std::max(n, 1);
        }
        if ((int64_t)occ[nti][ri] * L->n_sm >= (int64_t)grid.x) {
            ring = r;
            break;
        }
    }
    cfg.dynamicSmemBytes = smem_of(nt, ring);
    auto go = [&](auto kern) { return cudaLaunchKernelEx(&cfg, kern, p); };
    cudaError_t e = cudaSuccess;
    if (nt == 1) e = ring == 6 ? go(router_dec_kernel<1, 6>) : ring == 4 ? go(router_dec_kernel<1, 4>) : go(router_dec_kernel<1, 2>);
    else if (nt == 2) e = ring == 6 ? go(router_dec_kernel<2, 6>) : ring == 4 ? go(router_dec_kernel<2, 4>) : go(router_dec_kernel<2, 2>);
    else e = ring == 6 ? go(router_dec_kernel<4, 6>) : ring == 4 ? go(router_dec_kernel<4, 4>) : go(router_dec_kernel<4, 2>);
    MOBI_CUDA(e);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    L->plan[0] = MOBI_K_ROUTER_DECODE;
    return MOBI_OK;
}

int launch_decode_gemm(mobi_layer* L, const __nv_bfloat16* x, int64_t T, const uint8_t* given_masks, float delta,
                       uint8_t* masks_out, float* scores_out, __nv_bfloat16* y, bool pdl, cudaStream_t st,
                       unsigned long long* trace) {
    const DecPlan d = plan_decode(L, T);
    DParams p{};
    p.trace = trace;
    p.spart = L->dec_spart;
    p.b2 = L->b2;
    p.delta = delta;
    p.n_mt = (int)(L->h_pad / kRdRows);
    p.nr = L->nr;
    p.masks_dev = L->masks;
    p.masks_out = masks_out;
    p.scores_out = scores_out;
    p.codes8 = L->codes8;
    p.gconst = L->gconst;
    p.x = x;
    p.masks = given_masks;
    p.vmask = (1 << (L->nr + 1)) - 1;
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
    if (g_dec_fma && T <= kFmaMaxT) {
        p.n_cta = (int)std::min<int64_t>((int64_t)kFmaCps * L->n_sm, d.U);
        p.len_max = (int)std::min<int64_t>(cdiv(d.U, p.n_cta), L->kblocks);
        const size_t sm = fma_smem(kFmaMaxT, p.len_max).total;
        if (T == 1) return launch_decode_fma_t<1>(L, p, fma_smem(1, p.len_max).total, pdl, st);
        if (T == 2) return launch_decode_fma_t<2>(L, p, fma_smem(2, p.len_max).total, pdl, st);
        return launch_decode_fma_t<kFmaMaxT>(L, p, sm, pdl, st);
    }
    if (T == 1) return launch_decode_gemm_t<1>(L, p, d.smem, pdl, st);
    if (T <= 8) return launch_decode_gemm_t<8>(L, p, d.smem, pdl, st);
    if (T <= 16) return launch_decode_gemm_t<9>(L, p, d.smem, pdl, st);
    return launch_decode_gemm_t<11>(L, p, d.smem, pdl, st);
}

}  // namespace mobi
