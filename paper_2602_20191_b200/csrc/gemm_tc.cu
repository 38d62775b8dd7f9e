// gemm_tc.cu -- K3/K5: the nested residual MoBi GEMM on 5th-generation tensor cores (tcgen05),
// with the un-permute scatter fused into the epilogue.
//
// Math (router.hpp:105-132 regrouped per bucket, SURVEY Appendix A "equivalent group form"):
// every token in a bucket with slice mask m sees the effective weight
//      W_m[r,c] = s_g * (F_m(r,c) - z_g),   F_m = (c1+.5) + sum_{e in m, e>=2} (c_e-1.5) 4^-(e-1)
//             = S_g * (INT & maskbyte(m)) + C_{g,m},   S_g = s_g/2^P, C = s_g K_m/2^(P+1) - s_g z_g
// so slice e is read and contracted only for tiles whose bucket contains e, and one MMA per
// k-step covers all of a bucket's active slices.
//
// Roles (one persistent CTA per SM, 704 threads):
//   warp 20     TMA producer: the pair's token tile as 32-row fp16 boxes (128-byte swizzle), half
//               issued by each CTA of the cluster and multicast to both
//   warp 21     TMEM allocator + single-thread tcgen05.mma issuer
//   (the two issuer warps have the highest ids: the warp arbiter favours them over ALU warps)
//   warps 0-15  dequantizers: each thread owns one weight row (= one TMEM lane) and 32 k of every
//               other 64-k block (two k-blocks in flight); coalesced 16-byte code loads, two of
//               its k-blocks ahead -> fp16 W_m -> tcgen05.st into the A stage in TMEM (the A operand
//               never touches shared memory)
//   warps 16-19 epilogue: tcgen05.ld the fp32 accumulator, x 2^e row scale, bf16 into a smem
//               staging tile, release TMEM, then scatter 256-byte token rows to Y[perm[i]]
//               (the un-permute, bitplane.hpp:171-172, fused)
// MMA: M=128 weight rows (TMEM lanes), N=tile tokens (<=256, multiple of 16), K=16 per
// instruction, D fp32 in TMEM columns [0,256); A stages at columns 256 + 32*s.
#include "mobi_internal.cuh"
#include "sm100.cuh"

#ifndef MOBI_RELAXED
#define MOBI_RELAXED 1
#endif
namespace mobi {
namespace {

using namespace sm100;

#ifndef MOBI_ABLATE
#define MOBI_ABLATE 0  // development ablations: 1 = no code loads, 2 = no dequantization
#endif
#ifndef MOBI_EV_MAX
#define MOBI_EV_MAX 4
#endif
#ifndef MOBI_NSTAGE
#define MOBI_NSTAGE 5
#endif
constexpr int NSTAGE = MOBI_NSTAGE;  // B stages (smem, 32 KiB each)
#ifndef MOBI_UNIFIED
#define MOBI_UNIFIED 1  // 1: one full/empty barrier pair per stage for both A (TMEM) and B (smem)
#endif
constexpr int NSA = MOBI_UNIFIED ? NSTAGE : 8;  // A stages (TMEM, 32 columns each)
constexpr int kSplitMaxT = 64;   // split-K only for decode-size batches
constexpr int kMaxSplit = 8;
#ifndef MOBI_BOXR
#define MOBI_BOXR 128
#endif
constexpr int kBoxRows = MOBI_BOXR;               // TMA box: token rows x 64 k (contiguous in xperm)
constexpr int kBoxBytes = kBoxRows * kKBlock * 2;
#ifndef MOBI_MC
#define MOBI_MC 1  // 1: the CTA pair multicasts the shared token tile; 0: every CTA loads its own copy
#endif
#ifndef MOBI_NPROD
#define MOBI_NPROD 1
#endif
constexpr int kNProd = MOBI_NPROD;                 // TMA producer warps (alternating k-blocks)
constexpr int kDqWarps = 16;                       // 4 per TMEM lane quarter
constexpr int kThreads = 32 * (1 + kNProd + kDqWarps + 4);  // dequant, epilogue, TMA, MMA
// Warp roles, ordered by scheduling priority (the SM's warp arbiter favours higher warp ids):
// the single-thread TMA and MMA issuers get the top ids so ALU-heavy dequant warps never starve them.
constexpr int kWarpDq0 = 0;                  // 16 dequantizer warps
constexpr int kWarpEpi0 = kDqWarps;          // 4 epilogue warps
constexpr int kWarpTma = kDqWarps + 4;       // TMA producer(s)
constexpr int kWarpMma = kDqWarps + 4 + kNProd;  // TMEM allocator + MMA issuer
constexpr int kStageBytes = kTokTile * kKBlock * 2;  // 32 KiB
constexpr int kAccCols = 256;
constexpr int kACol0 = 256;
constexpr int kYStageBytes = kTokTile * kRowTile * 2;  // 64 KiB bf16 output staging
constexpr int kSmemBytes = NSTAGE * kStageBytes + 1024 /*align*/ + 256 /*barriers*/ + kYStageBytes + kTokTile * 4;

struct Params {
    const uint8_t* codes8;
    const float2* gconst;  // [G][out_pad]
    int64_t out_pad;
    MaskTable mt;
    int64_t out, G, gs, kblocks;
    int64_t tpad;       // rows per k-block slab of xperm
    int single_group;
    int n_row_tiles;
    const float* escale;
    const int32_t* perm;
    const TokTile* tiles;
    const int32_t* meta;
    __nv_bfloat16* y;
    int vec_y;
    int* tile_counter;  // zeroed by the bucket kernel before every launch
    int* bk_hist;       // fused-bucketing histogram + slot counters: zeroed here for the next forward
    int max_split;      // split-K allowed (small T only): partials go to gpart, reduced by splitk_reduce
    int T;
    float* gpart;       // [split][T][out] fp32 (x 2^e applied)
    unsigned long long* trace;
};

// One 64-k block: four K=16 MMAs, D at TMEM column 0, A (fp16 weights) at TMEM column acol,
// B (fp16 tokens) from the 128B-swizzled smem stage; N is a compile-time constant so the
// instruction descriptor is an immediate.
template <uint32_t N>
__device__ __forceinline__ void issue_kblock_ts(uint32_t acol, uint64_t bdesc, bool first) {
    constexpr uint32_t idesc = idesc_f16(128, N, 0);
#pragma unroll
    for (int j = 0; j < kKBlock / 16; ++j)
        mma_ts_f16(0u, acol + j * 8, bdesc + (uint64_t)(j * 2), idesc, (!first || j != 0) ? 1u : 0u);
}

// TRACE=true: clock64 accounting of each role's barrier waits (debug hook impl 2), written to
// p.trace[cta][0..15]: 0 tma wait empty | 1 mma wait acc_empty | 2 mma wait full_b | 3 mma wait
// full_a | 4 mma loop | 5 dequant(w2) wait empty | 6 dequant(w2) loop | 7 epi(w18) wait acc_full |
// 8 epi(w18) loop | 9 tiles
template <bool TRACE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    mobi_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params p) {
    long long tr[6] = {0, 0, 0, 0, 0, 0};
    // per-k-block event timeline (CTA 0, first tile): trace[20480 + ev*64 + kb]
    auto EV = [&](int ev, int kb, uint32_t tile_idx) {
        if (TRACE && ev < MOBI_EV_MAX && blockIdx.x == 0 && tile_idx == 0 && kb < 64 && (threadIdx.x % 32) == 0)
            p.trace[20480 + ev * 64 + kb] = (unsigned long long)clock64();
    };
#define TW(i, stmt)                                   \
    do {                                              \
        if (TRACE) {                                  \
            long long t0_ = clock64();                \
            stmt;                                     \
            tr[i] += clock64() - t0_;                 \
        } else {                                      \
            stmt;                                     \
        }                                             \
    } while (0)
    long long tstart = TRACE ? clock64() : 0;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_b = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSTAGE * kStageBytes);
    uint64_t* full_b = bars;                  // [NSTAGE] TMA landed
    uint64_t* empty = bars + NSTAGE;          // [NSTAGE] MMAs of BOTH CTAs done with the B stage
    uint64_t* full_a = bars + 2 * NSTAGE;     // [NSA] A stage written to TMEM (8 warps)
    uint64_t* empty_a = full_a + NSA;         // [NSA] local MMAs done with the A stage
    uint64_t* acc_full = empty_a + NSA;       // accumulator ready for the epilogue
    // unified stages: the dequantizers arrive on the TMA's full barrier and wait on the MMA's empty one
    uint64_t* a_full = MOBI_UNIFIED ? full_b : full_a;
    uint64_t* a_empty = MOBI_UNIFIED ? empty : empty_a;
    uint64_t* acc_empty = acc_full + 1;       // epilogue drained the accumulator (4 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
    __nv_bfloat16* stage_y = reinterpret_cast<__nv_bfloat16*>(smem + NSTAGE * kStageBytes + 256);
    int32_t* tok_src = reinterpret_cast<int32_t*>(smem + NSTAGE * kStageBytes + 256 + kYStageBytes);
    auto epi_bar_sync = [] { asm volatile("bar.sync 1, 128;" ::: "memory"); };

    const int warp = warp_idx_uniform(), lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full_b[s], MOBI_UNIFIED ? 1 + kDqWarps / 2 : 1);
            mbar_init(&empty[s], MOBI_MC ? 2 : 1);  // MMA completion of BOTH CTAs of the pair (shared B stages)
        }
        for (int s = 0; s < NSA; ++s) {
            mbar_init(&full_a[s], kDqWarps / 2);
            mbar_init(&empty_a[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 4);
        fence_barrier_init();
        prefetch_tmap(&tmap_x);
    }
    if (warp == kWarpMma) tmem_alloc(tmem_slot, 512);
    if (blockIdx.x == 0 && threadIdx.x < 48 && p.bk_hist) p.bk_hist[threadIdx.x] = 0;  // gather consumed it
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // peer barriers initialised before any multicast lands
    tc_fence_after();
    // the CTA owns all 512 TMEM columns, so the allocation base is column 0 / lane 0; using the
    // constant keeps every tcgen05 operand in uniform registers (no per-instruction R2UR waterfall)
    if (*tmem_slot != 0) __trap();
    constexpr uint32_t tmem = 0;

    // Static schedule over CTA pairs (clusters of 2): a pair works on one token tile and two
    // adjacent 128-row weight tiles; each CTA TMA-loads half of the token tile's 32-row boxes and
    // multicasts them to both, so every CTA receives the full B tile for half the L2 traffic.
    const uint32_t rank = cluster_ctarank();
    const int n_tok_tiles = p.meta[0];
    const int n_pairs_row = p.n_row_tiles / 2;
    const int kb_n = (int)p.kblocks;
    const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
    // split-K when the (token tile x row pair) grid cannot fill the clusters (decode-size T):
    // every CTA derives the same split count from the device-side tile count
    int nsplit = 1;
    if (p.max_split > 1) nsplit = max(1, min(min(p.max_split, kb_n), ncl / max(1, n_tok_tiles * n_pairs_row)));
    const int kb_per = (kb_n + nsplit - 1) / nsplit;
    nsplit = (kb_n + kb_per - 1) / kb_per;  // every split owns at least one k-block (no empty ranges)
    if (blockIdx.x == 0 && threadIdx.x == 0 && p.max_split > 1) p.tile_counter[1] = nsplit;  // for the reduce
    const int total = n_tok_tiles * n_pairs_row * nsplit;
    // pair -> (token tile, this CTA's 128-row tile, k-block range [kb0, kb1))
    auto tile_of = [&](int pair, TokTile& tt, int& rt, int& ks, int& kb0, int& kb1) {
        ks = pair % nsplit;
        const int q = pair / nsplit;
        tt = uniform_tile(p.tiles[q / n_pairs_row]);
        rt = (q % n_pairs_row) * 2 + (int)rank;
        kb0 = ks * kb_per;
        kb1 = min(kb_n, kb0 + kb_per);
    };

    if (warp >= kWarpTma && warp < kWarpTma + kNProd) {
        // ---------------- TMA producer(s): producer w owns the k-block iterations it % kNProd == w ----------------
        const uint32_t pw = (uint32_t)(warp - kWarpTma);
        uint32_t it = 0;
        for (int pair = cid; pair < total; pair += ncl) {
            TokTile tt;
            int rt, ks, kb0, kb1;
            tile_of(pair, tt, rt, ks, kb0, kb1);
            if (TRACE && lane == 0) ++tr[3];
            const int nbox = (tt.n + kBoxRows - 1) / kBoxRows;
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                if (kNProd > 1 && it % kNProd != pw) continue;
                const int s = it % NSTAGE;
                const uint32_t ph = (it / NSTAGE) & 1;
                TW(0, mbar_wait(&empty[s], ph ^ 1));
                EV(0, kb, (uint32_t)(pair != cid));
                if (elect_one_sync()) {
                    mbar_arrive_expect_tx(&full_b[s], nbox * kBoxBytes);
                    if (MOBI_MC) {
                        for (int j = (int)rank; j < nbox; j += 2)
                            tma_load_2d_mc(stage_b + s * kStageBytes + j * kBoxBytes, &tmap_x, &full_b[s], 0,
                                           (int)(kb * p.tpad) + tt.row0 + j * kBoxRows, (uint16_t)0x3);
                    } else {
                        for (int j = 0; j < nbox; ++j)
                            tma_load_2d(stage_b + s * kStageBytes + j * kBoxBytes, &tmap_x, &full_b[s], 0,
                                        (int)(kb * p.tpad) + tt.row0 + j * kBoxRows);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == kWarpMma) {
        // ---------------- MMA issuer ----------------
        uint32_t it = 0, tc = 0;
        for (int pair = cid; pair < total; pair += ncl, ++tc) {
            TokTile tt;
            int rt, ks, kb0, kb1;
            tile_of(pair, tt, rt, ks, kb0, kb1);
            // N class: 16, or a multiple of 32 (constant instruction descriptors per class)
            const uint32_t n_mma = tt.n <= 16 ? 16u : (uint32_t)round_up(tt.n, 32);
            TW(0, mbar_wait(acc_empty, (tc & 1) ^ 1));
            tc_fence_after();
            long long t_tile0 = TRACE ? clock64() : 0;
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                const int s = it % NSTAGE;
                const uint32_t ph = (it / NSTAGE) & 1;
                const int sa = it % NSA;
                const uint32_t pha = (it / NSA) & 1;
                TW(1, mbar_wait(&full_b[s], ph));
                EV(1, kb, tc);
                if (!MOBI_UNIFIED) TW(2, mbar_wait(&full_a[sa], pha));
                EV(2, kb, tc);
                tc_fence_after();
                if (elect_one_sync()) {
                    const uint64_t bdesc = sdesc_sw128(smem_u32(stage_b + s * kStageBytes));
                    const uint32_t acol = tmem + kACol0 + sa * 32;
                    const bool first = kb == kb0;
                    switch (n_mma) {
                        case 16: issue_kblock_ts<16>(acol, bdesc, first); break;
                        case 32: issue_kblock_ts<32>(acol, bdesc, first); break;
                        case 64: issue_kblock_ts<64>(acol, bdesc, first); break;
                        case 96: issue_kblock_ts<96>(acol, bdesc, first); break;
                        case 128: issue_kblock_ts<128>(acol, bdesc, first); break;
                        case 160: issue_kblock_ts<160>(acol, bdesc, first); break;
                        case 192: issue_kblock_ts<192>(acol, bdesc, first); break;
                        case 224: issue_kblock_ts<224>(acol, bdesc, first); break;
                        default: issue_kblock_ts<256>(acol, bdesc, first); break;
                    }
                    if (MOBI_MC)
                        mma_commit_mc(&empty[s], (uint16_t)0x3);  // frees the shared B stage in both CTAs
                    else
                        mma_commit(&empty[s]);
                    if (!MOBI_UNIFIED) mma_commit(&empty_a[sa]);  // frees the local A stage
                    if (kb == kb1 - 1) mma_commit(acc_full);
                }
                __syncwarp();
                EV(3, kb, tc);
            }
            if (TRACE && lane == 0 && tc < 8) {  // per-tile: N and cycles from first wait to last issue
                p.trace[16 * 1024 + (blockIdx.x * 8 + tc) * 2] = (unsigned long long)n_mma;
                p.trace[16 * 1024 + (blockIdx.x * 8 + tc) * 2 + 1] = (unsigned long long)(clock64() - t_tile0);
            }
        }
    } else if (warp < kWarpEpi0) {
        // ---------------- dequantizers ----------------
        // 16 warps = 4 TMEM lane quarters x 2 k-halves x 2 k-block parities: a warp dequantizes
        // 32 codes of its row for every other k-block, so two k-blocks are in flight at once.
        const int idx = warp - kWarpDq0;
        const int q = warp % 4;
        const int par = (idx / 4) & 1;
        const int hh = idx / 8;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        uint32_t base = 0;  // global k-block counter at the start of the tile (stage/phase)
        for (int pair = cid; pair < total; pair += ncl) {
            TokTile tt;
            int rt, ks, kb0, kb1;
            tile_of(pair, tt, rt, ks, kb0, kb1);
            const int kb_lim = kb1;  // this tile's k-blocks are [kb0, kb1); stage index = base + kb - kb0
            const int64_t R = (int64_t)rt * kRowTile + 32 * q + lane;
            const bool rv = R < p.out;
            const uint32_t mw = p.mt.maskword[tt.mask];
            const float kc = p.mt.kc[tt.mask];
            const uint8_t* cbase =
                p.codes8 + (int64_t)rt * p.kblocks * kBlockBytes + ((hh * 2) * kRowTile + 32 * q + lane) * 16;
            const float2* gcol = p.gconst + (rv ? R : 0);
            auto ldc = [&](int gg) { return rv ? __ldg(gcol + (int64_t)gg * p.out_pad) : make_float2(0.f, 0.f); };
            auto ld = [&](int kb, uint4& c0, uint4& c1) {
                const uint8_t* b0 = cbase + (int64_t)kb * kBlockBytes;
                c0 = *reinterpret_cast<const uint4*>(b0);
                c1 = *reinterpret_cast<const uint4*>(b0 + kRowTile * 16);
            };
            // group of k = kb*64 + 32*hh, tracked incrementally (k advances by 128 per step)
            auto dq = [&](const uint4& c0, const uint4& c1, float2 gcst, uint32_t (&v)[16]) {
                const __half2 S2 = __float2half2_rn(gcst.x * p.mt.inv_2p);
                const __half2 C2 = __float2half2_rn(fmaf(gcst.x, kc, -gcst.y));
                const uint32_t* w0 = reinterpret_cast<const uint32_t*>(&c0);
                const uint32_t* w1 = reinterpret_cast<const uint32_t*>(&c1);
#pragma unroll
                for (int u = 0; u < 4; ++u) dequant4(w0[u], mw, S2, C2, v[2 * u], v[2 * u + 1]);
#pragma unroll
                for (int u = 0; u < 4; ++u) dequant4(w1[u], mw, S2, C2, v[8 + 2 * u], v[8 + 2 * u + 1]);
            };
            // Ring of three static slots (codes + group constants), unrolled so a slot is refilled
            // right after it was consumed and each load has two iterations of lead time; no
            // register moves touch a pending load.
            uint4 c00, c01, c10, c11, c20, c21;
            float2 g0 = make_float2(0.f, 0.f), g1 = g0, g2 = g0;
            int gp = 0, kinp = 0;  // group cursor at the next k-block to prefetch
            if (!p.single_group) {
                const int k0 = (kb0 + par) * kKBlock + hh * 32;
                gp = k0 / (int)p.gs;
                kinp = k0 - gp * (int)p.gs;
            }
            auto fetch = [&](int kb, uint4& c0, uint4& c1, float2& gc) {
#if MOBI_ABLATE >= 1
                c0 = make_uint4(kb, kb, kb, kb); c1 = c0; gc = make_float2(1.f, 0.f);
                return;
#endif
                if (kb < kb_lim) {
                    ld(kb, c0, c1);
                    gc = ldc(gp);
                }
                if (!p.single_group) {
                    kinp += 2 * kKBlock;
                    while (kinp >= p.gs) kinp -= (int)p.gs, ++gp;
                }
            };
            fetch(kb0 + par, c00, c01, g0);
            fetch(kb0 + par + 2, c10, c11, g1);
            fetch(kb0 + par + 4, c20, c21, g2);
            uint32_t v[16];
            auto step = [&](int kb, uint4& ca, uint4& cb, float2& ga, uint4& na, uint4& nb, float2& gn) -> bool {
                // v holds k-block kb (dequantized from the slot (ca, cb)); (na, nb) holds kb+2
                if (kb >= kb_lim) return false;
                const uint32_t itk = base + (kb - kb0);
                const int s = itk % NSA;
                const uint32_t ph = (itk / NSA) & 1;
                TW(0, mbar_wait(&a_empty[s], ph ^ 1));
                if (warp == 0 || warp == 4) EV(4, kb, base);
                tc_fence_after();
                TW(3, tmem_st16(tmem + lane_base + kACol0 + s * 32 + hh * 16, v));
                TW(4, fetch(kb + 6, ca, cb, ga));  // refill the consumed slot three of this warp's k-blocks ahead
#if MOBI_ABLATE >= 2
                (void)na; (void)nb; (void)gn;
#else
                if (kb + 2 < kb_lim) TW(1, dq(na, nb, gn, v));
#endif
                if (warp == 0 || warp == 4) EV(5, kb, base);
                TW(2, tmem_st_wait());
                tc_fence_before();
                __syncwarp();
                if (warp == 0 || warp == 4) EV(6, kb, base);
                if (lane == 0) {
#if MOBI_RELAXED
                    mbar_arrive_relaxed(&a_full[s]);
#else
                    mbar_arrive(&a_full[s]);
#endif
                }
                return true;
            };
            if (kb0 + par < kb_lim) dq(c00, c01, g0, v);
            for (int kb = kb0 + par; kb < kb_lim; kb += 6) {
                if (!step(kb, c00, c01, g0, c10, c11, g1)) break;
                if (!step(kb + 2, c10, c11, g1, c20, c21, g2)) break;
                if (!step(kb + 4, c20, c21, g2, c00, c01, g0)) break;
            }
            base += kb1 - kb0;
        }
    } else {
        // ---------------- epilogue ----------------
        // drain TMEM -> (x 2^e) -> bf16 -> smem tile [token][128 rows], release the accumulator,
        // then scatter whole 256-byte token rows into Y[perm[i]] with 16-byte stores
        const int q = warp % 4;
        const int et = threadIdx.x - 32 * kWarpEpi0;  // 0..127
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        uint32_t tc = 0;
        for (int pair = cid; pair < total; pair += ncl, ++tc) {
            TokTile tt;
            int rt, ks, kb0, kb1;
            tile_of(pair, tt, rt, ks, kb0, kb1);
            // the tile's token sources and row scales, fetched while the MMAs run (not per drained chunk)
            int32_t src_r[kTokTile / 32];
            float es_r[kTokTile / 32];
#pragma unroll
            for (int c = 0; c < kTokTile / 32; ++c) {
                const bool ok = 32 * c + lane < tt.n;
                src_r[c] = ok ? __ldg(p.perm + tt.row0 + 32 * c + lane) : -1;
                es_r[c] = ok ? __ldg(p.escale + tt.row0 + 32 * c + lane) : 0.f;
            }
            TW(0, mbar_wait(acc_full, tc & 1));
            tc_fence_after();
            if (nsplit > 1) {
                // split-K partial: fp32 x 2^e straight to gpart[ks][token][row] (coalesced over rows)
                const int64_t R = (int64_t)rt * kRowTile + 32 * q + lane;
                for (int c0 = 0; c0 < tt.n; c0 += 32) {
                    const int nn = min(32, tt.n - c0);
                    int32_t my_src = -1;
                    float my_es = 0.f;
                    if (lane < nn) {
                        my_src = __ldg(p.perm + tt.row0 + c0 + lane);
                        my_es = __ldg(p.escale + tt.row0 + c0 + lane);
                    }
                    uint32_t v[32];
                    tmem_ld32(tmem + lane_base + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int32_t src = __shfl_sync(0xffffffffu, my_src, j);
                        const float es = __shfl_sync(0xffffffffu, my_es, j);
                        if (src >= 0 && R < p.out)
                            p.gpart[((int64_t)ks * p.T + src) * p.out + R] = __uint_as_float(v[j]) * es;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(acc_empty);
                continue;
            }
            epi_bar_sync();  // the previous tile's scatter has finished reading the staging tile
            // 16-column TMEM loads, the next one in flight while the current one is converted
            uint32_t va[16], vb[16];
            tmem_ld16(tmem + lane_base, va);
#pragma unroll
            for (int c = 0; c < kTokTile / 16; ++c) {
                const int c0 = 16 * c;
                if (c0 >= tt.n) break;
                tmem_ld_wait();
                uint32_t(&cur)[16] = (c & 1) ? vb : va;
                uint32_t(&nxt)[16] = (c & 1) ? va : vb;
                if (c0 + 16 < tt.n) tmem_ld16(tmem + lane_base + c0 + 16, nxt);
                const float my_es = es_r[c / 2];
                if (q == 0 && (c & 1) == 0) tok_src[c0 + lane] = src_r[c / 2];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float es = __shfl_sync(0xffffffffu, my_es, (c & 1) * 16 + j);
                    stage_y[(c0 + j) * kRowTile + 32 * q + lane] = __float2bfloat16_rn(__uint_as_float(cur[j]) * es);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
            epi_bar_sync();  // staging tile complete
            const int64_t r0 = (int64_t)rt * kRowTile + 8 * (et % 16);
            for (int t = et / 16; t < tt.n; t += 8) {
                const int32_t src = tok_src[t];
                if (src < 0 || r0 >= p.out) continue;
                const __nv_bfloat16* sp = stage_y + t * kRowTile + 8 * (et % 16);
                __nv_bfloat16* dp = p.y + (int64_t)src * p.out + r0;
                if (p.vec_y && r0 + 8 <= p.out) {
                    *reinterpret_cast<uint4*>(dp) = *reinterpret_cast<const uint4*>(sp);
                } else {
                    for (int u = 0; u < 8 && r0 + u < p.out; ++u) dp[u] = sp[u];
                }
            }
        }
    }
    if (TRACE && lane == 0) {
        unsigned long long* o = p.trace + blockIdx.x * 16;
        const long long tot = clock64() - tstart;
        if (warp == kWarpTma) o[0] = tr[0];
        if (warp == kWarpMma) { o[1] = tr[0]; o[2] = tr[1]; o[3] = tr[2]; o[4] = tot; }
        if (warp == 0) {
            o[5] = tr[0]; o[6] = tot; o[10] = tr[1]; o[11] = tr[2]; o[12] = tr[3]; o[13] = tr[4]; o[14] = tr[5];
        }
        if (warp == kWarpEpi0) { o[7] = tr[0]; o[8] = tot; }
        if (warp == kWarpTma) o[9] = tr[3];
    }
#undef TW
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no CTA leaves while its peer may still multicast into it
    if (warp == kWarpMma) tmem_dealloc(tmem, 512);
}

// y[t][r] = bf16( sum_{ks < nsplit} gpart[ks][t][r] ) in a fixed order (deterministic)
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ gpart, const int* __restrict__ meta,
                                                            int T, int64_t out, __nv_bfloat16* __restrict__ y) {
    const int nsplit = meta[33];
    if (nsplit <= 1) return;  // the GEMM epilogue already wrote bf16
    const int t = blockIdx.x;
    for (int64_t r = threadIdx.x; r < out; r += blockDim.x) {
        float acc = 0.f;
        for (int ks = 0; ks < nsplit; ++ks) acc += gpart[((int64_t)ks * T + t) * out + r];
        y[(int64_t)t * out + r] = __float2bfloat16_rn(acc);
    }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(f);
    }
    return fn;
}


}  // namespace

// 2-D fp16 tensor map over a [rows][cols] row-major buffer, box {64 cols, box_rows rows},
// 128-byte swizzle.  Shared with the tcgen05 router (router_tc.cu).
int make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int64_t rows, int64_t cols,
                 int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return set_error(MOBI_ERUNTIME, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(cols * 2)};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(MOBI_ERUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return MOBI_OK;
}

int launch_gemm_tc(mobi_layer* L, __nv_bfloat16* y, int64_t T, cudaStream_t st, unsigned long long* trace) {
    {
        MOBI_TRY(func_attr_once(mobi_gemm_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBytes));
        MOBI_TRY(func_attr_once(mobi_gemm_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBytes));
    }
    if (!L->tmap_x) {
        L->tmap_x = new CUtensorMap;
        int rc = make_tmap_2d(L->tmap_x, L->xperm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, L->kblocks * L->tpad_max, kKBlock,
                              kBoxRows);
        if (rc) {
            delete L->tmap_x;
            L->tmap_x = nullptr;
            return rc;
        }
    }
    Params p;
    p.codes8 = L->codes8;
    p.gconst = L->gconst;
    p.out_pad = L->out_pad;
    p.mt = L->mtab;
    p.out = L->out;
    p.G = L->G;
    p.gs = L->gs;
    p.kblocks = L->kblocks;
    p.tpad = L->tpad_max;
    p.single_group = L->single_group;
    p.n_row_tiles = (int)(L->out_pad / kRowTile);
    p.escale = L->escale;
    p.perm = L->perm;
    p.tiles = L->tiles;
    p.meta = L->meta;
    p.y = y;
    p.vec_y = (L->out % 8 == 0) && ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
    const int64_t max_pairs = (int64_t)(p.n_row_tiles / 2) * L->max_tiles;
    const int grid = 2 * (int)std::min<int64_t>(L->n_sm / 2, max_pairs);
    p.trace = trace;
    p.tile_counter = L->meta + 32;
    p.T = (int)T;
    p.max_split = (T <= kSplitMaxT && L->gpart) ? kMaxSplit : 1;
    p.gpart = L->gpart;
    p.bk_hist = L->bk_hist;
    if (trace)
        mobi_gemm_tc_kernel<true><<<grid, kThreads, kSmemBytes, st>>>(*L->tmap_x, p);
    else
        mobi_gemm_tc_kernel<false><<<grid, kThreads, kSmemBytes, st>>>(*L->tmap_x, p);
    L->plan[1] = MOBI_K_GEMM_SPLITK;
    L->plan[2] = grid;
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    if (p.max_split > 1) {
        splitk_reduce_kernel<<<(unsigned)T, 256, 0, st>>>(L->gpart, L->meta, (int)T, L->out, y);
        MOBI_LAUNCH_CHECK();
        ++L->last_launches;
    }
    return MOBI_OK;
}

}  // namespace mobi
