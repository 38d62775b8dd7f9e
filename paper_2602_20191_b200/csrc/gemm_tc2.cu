// gemm_tc2.cu -- K3/K5 on CTA PAIRS: the nested residual MoBi GEMM with tcgen05.mma.cta_group::2
// (M = 256 weight rows per pair instruction), un-permute scatter fused in the epilogue.
//
// Same math and per-thread roles as gemm_tc.cu (see its header); what changes with cta_group::2:
//   * A (dequantized fp16 weights, 128 rows) is written by each CTA's dequantizers into its OWN
//     TMEM; the leader CTA's single MMA thread issues M=256 MMAs that read both CTAs' A;
//   * B (the bucket's token tile, N tokens) is split: each CTA TMA-loads N/2 token rows into its
//     own smem and the pair instruction reads both halves -> half the L2->SM bytes and half the
//     smem operand traffic per SM compared with the 1-CTA kernel (which was B-bandwidth bound);
//   * D: each CTA's TMEM holds its 128 rows x all N tokens;
//   * barriers: the peer's TMA completes on the leader's full_b, the peer's dequantizers and
//     epilogue arrive on the leader's full_a / acc_empty (mapa addresses, release.cluster); the
//     leader's MMA commits are multicast to both CTAs' empty / acc_full.
// With half-height B stages (16 KiB) the ring is 8 deep in both smem (B) and TMEM (A).
#include <algorithm>

#include "mobi_internal.cuh"
#include "sm100.cuh"

#ifndef MOBI_MMA_WAIT
#define MOBI_MMA_WAIT 0
#endif
#ifndef MOBI_RELAXED
#define MOBI_RELAXED 1
#endif
// bottleneck experiments (development only; all 0 in the product): drop one producer's real work
#ifndef MOBI_X_NOLOAD
#define MOBI_X_NOLOAD 0  // dequantizers skip the code / constant loads
#endif
#ifndef MOBI_X_NOTMA
#define MOBI_X_NOTMA 0   // the TMA warp arrives without loading B
#endif
#ifndef MOBI_X_NODQ
#define MOBI_X_NODQ 0    // dequantizers store the raw code words (no ALU work)
#endif
#ifndef MOBI_TRACE_UNIT
#define MOBI_TRACE_UNIT 0  // which of cluster 0's units the per-k-block trace records
#endif
#ifndef MOBI_X_NOWAIT
#define MOBI_X_NOWAIT 0  // the MMA thread issues without waiting for the stage (timing only: garbage output)
#endif
#ifndef MOBI_X_NOEPI
#define MOBI_X_NOEPI 0   // the epilogue releases TMEM without draining or storing
#endif
namespace mobi {
int make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int64_t rows, int64_t cols,
                 int box_rows);
namespace {

using namespace sm100;

constexpr int NSTAGE = 8;
constexpr int kDqWarps = 16;
constexpr int kThreads = 32 * (2 + kDqWarps + 4);
constexpr int kWarpDq0 = 0, kWarpEpi0 = kDqWarps, kWarpTma = kDqWarps + 4, kWarpMma = kDqWarps + 5;
// dynamic unit schedule: the leader's TMA warp claims units (atomic counter, units in decreasing
// size order) and publishes them through a small ring to every role of both CTAs
constexpr int kURing = 4;
constexpr int kUnitConsumers = 1 + kDqWarps + 4;  // per CTA: MMA (leader) or TMA (peer) + dequant + epilogue
constexpr int kHalfRows = kTokTile / 2;                  // token rows per CTA per stage
constexpr int kStageBytes = kHalfRows * kKBlock * 2;     // 16 KiB
constexpr int kBoxRows = 16;
constexpr int kBoxBytes = kBoxRows * kKBlock * 2;        // 2 KiB
constexpr int kACol0 = 256;
constexpr int kYStageBytes = kTokTile * kRowTile * 2;    // 64 KiB
constexpr int kSmemBytes = NSTAGE * kStageBytes + 1024 + 512 + kYStageBytes + kTokTile * 4;
constexpr int kBigBoxRows = kHalfRows;  // one TMA box per full half-tile

struct Params {
    const uint8_t* codes8;
    const float2* gconst;
    int64_t out_pad;
    MaskTable mt;
    int64_t out, G, gs, kblocks;
    int64_t tpad;
    int single_group;
    int n_row_tiles;
    const float* escale;
    const int32_t* perm;
    const TokTile* tiles;
    const int32_t* meta;
    OutDesc od;   // Y row t of this layer -> od.dst[k] + t*ldy + col0 (k < n_dst: local and peer buffers)
    int vec_y;
    int* bk_hist;  // fused-bucketing histogram + slot counters: zeroed here for the next forward
    int* unit_ctr;  // dynamic unit counter (meta[32]), zeroed by the kernel that builds the tile list
    unsigned long long* trace;
};

template <bool TRACE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    mobi_gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_big,
                         const Params p) {
    // per-k-block event timeline (cluster 0, first tile): trace[20480 + (rank*8+ev)*64 + kb]
    auto EV = [&](int ev, int kb, uint32_t tile_idx) {
        if (TRACE && blockIdx.x < 2 && tile_idx == MOBI_TRACE_UNIT && kb < 64 && (threadIdx.x % 32) == 0)
            p.trace[20480 + (cluster_ctarank() * 8 + ev) * 64 + kb] = (unsigned long long)clock64();
    };
    // per-unit events (cluster 0, first 16 units, globaltimer ns): trace[24576 + (rank*8+ev)*16 + u]
    auto EVU = [&](int ev, uint32_t u) {
        if (TRACE && blockIdx.x < 2 && u < 16 && (threadIdx.x % 32) == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.trace[24576 + (cluster_ctarank() * 8 + ev) * 16 + u] = t;
        }
    };
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_b = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSTAGE * kStageBytes);
    // one full barrier per stage, in the leader: both halves' TMA bytes (one expect_tx arrival) and the
    // 8 + 8 dequant warps of the pair (the peer's arrive remotely)
    uint64_t* full_b = bars;                 // [NSTAGE] leader: stage complete (A in both TMEMs, B in both smems)
    uint64_t* empty = bars + NSTAGE;         // [NSTAGE] each CTA: pair MMAs done with the stage
    uint64_t* acc_full = bars + 2 * NSTAGE;  // each CTA
    uint64_t* acc_empty = acc_full + 1;      // leader: both CTAs drained TMEM
    uint64_t* u_full = acc_empty + 1;        // [kURing] each CTA: unit slot published
    uint64_t* u_empty = u_full + kURing;     // [kURing] leader: every consumer of both CTAs read the slot
    int32_t* uring = reinterpret_cast<int32_t*>(u_empty + kURing);  // [kURing] unit index (-1 = done)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uring + kURing);
    __nv_bfloat16* stage_y = reinterpret_cast<__nv_bfloat16*>(smem + NSTAGE * kStageBytes + 512);
    int32_t* tok_src = reinterpret_cast<int32_t*>(smem + NSTAGE * kStageBytes + 512 + kYStageBytes);
    auto epi_bar_sync = [] { asm volatile("bar.sync 1, 128;" ::: "memory"); };

    const int warp = warp_idx_uniform(), lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full_b[s], 1 + kDqWarps);  // TMA expect_tx + 8 dequant warps per CTA x 2
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 8);  // 4 epilogue warps x 2 CTAs
        for (int s = 0; s < kURing; ++s) {
            mbar_init(&u_full[s], 1);
            mbar_init(&u_empty[s], 2 * kUnitConsumers);
        }
        fence_barrier_init();
        prefetch_tmap(&tmap_x);
        prefetch_tmap(&tmap_big);
    }
    if (warp == kWarpMma) tmem_alloc_2sm(tmem_slot, 512);
    pdl_wait();  // PDL launch: everything above overlapped the gather; its outputs are visible from here
    if (blockIdx.x == 0 && threadIdx.x < 48 && p.bk_hist) p.bk_hist[threadIdx.x] = 0;  // gather consumed it
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    if (*tmem_slot != 0) __trap();
    constexpr uint32_t tmem = 0;

    const int n_tok_tiles = p.meta[0];
    const int n_pairs_row = p.n_row_tiles / 2;
    const int total = n_tok_tiles * n_pairs_row;
    const int kb_n = (int)p.kblocks;
    const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
    // pair -> (token tile, this CTA's 128-row weight tile, N class: a multiple of 32 >= 32)
    auto tile_of = [&](int pair, TokTile& tt, int& rt, int& nc) {
        tt = uniform_tile(p.tiles[pair / n_pairs_row]);
        rt = (pair % n_pairs_row) * 2 + (int)rank;
        nc = max(32, (int)round_up(tt.n, 32));
    };
    // unit ring: consumers read slot ui % kURing, then release it on the leader's u_empty
    auto unit_get = [&](uint32_t ui) -> int {
        const int s = (int)(ui % kURing);
        const uint32_t ph = (ui / kURing) & 1;
        if (rank == 0)
            mbar_wait(&u_full[s], ph);
        else
            mbar_wait_cluster(&u_full[s], ph);  // published by the leader's thread (remote store + release)
        const int u = *reinterpret_cast<volatile int32_t*>(&uring[s]);
        __syncwarp();
        if (lane == 0) {
            if (rank == 0)
                mbar_arrive(&u_empty[s]);
            else
                mbar_arrive_cluster(mapa_shared(smem_u32(&u_empty[s]), 0));
        }
        return u;
    };
    // producer (the leader's TMA warp): the first unit of cluster c is c, later ones come from the
    // counter (claimed when this pair's TMA runs out of work, i.e. ~NSTAGE k-blocks ahead of its MMAs)
    auto unit_put = [&](uint32_t ui) -> int {
        const int s = (int)(ui % kURing);
        mbar_wait_cluster(&u_empty[s], ((ui / kURing) & 1) ^ 1);
        int u = 0;
        if (lane == 0) {
            u = ui == 0 ? cid : atomicAdd(p.unit_ctr, 1) + ncl;
            if (u >= total) u = -1;
            *reinterpret_cast<volatile int32_t*>(&uring[s]) = u;
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa_shared(smem_u32(&uring[s]), 1)), "r"(u)
                         : "memory");
            mbar_arrive(&u_full[s]);
            mbar_arrive_cluster(mapa_shared(smem_u32(&u_full[s]), 1));
        }
        return __shfl_sync(0xffffffffu, u, 0);
    };

    if (warp == kWarpTma) {
        // ---------------- TMA producer (both CTAs: own half of the token tile) ----------------
        const uint32_t full_b_leader = mapa_shared(smem_u32(full_b), 0);
        uint32_t it = 0;
        bool trig = false;
        for (uint32_t ui = 0;; ++ui) {
            const int pair = rank == 0 ? unit_put(ui) : unit_get(ui);
            // the last wave of units: the next kernel (the next layer's router, PDL) may launch its CTAs
            // onto SMs as this grid drains (it waits for this grid before touching anything we write)
            if (!trig && (pair < 0 || pair + ncl >= total)) {
                trig = true;
                if (elect_one_sync()) pdl_trigger();
                __syncwarp();
            }
            if (pair < 0) break;
            TokTile tt;
            int rt, nc;
            tile_of(pair, tt, rt, nc);
            const bool big = nc == kTokTile;  // full tile: one 128-row box per CTA
            const int nbox = big ? 1 : nc / 2 / kBoxRows;
            const int row_half = tt.row0 + (int)rank * (nc / 2);
            for (int kb = 0; kb < kb_n; ++kb, ++it) {
                const int s = it % NSTAGE;
                const uint32_t ph = (it / NSTAGE) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                EV(0, kb, ui);
                if (MOBI_X_NOTMA) {
                    if (elect_one_sync() && rank == 0) mbar_arrive_expect_tx(&full_b[s], 0);
                } else if (elect_one_sync()) {
                    if (rank == 0) mbar_arrive_expect_tx(&full_b[s], 2 * (big ? kStageBytes : nbox * kBoxBytes));
                    if (big)
                        tma_load_2d_2sm(stage_b + s * kStageBytes, &tmap_big, full_b_leader + s * 8, 0,
                                        (int)(kb * p.tpad) + row_half);
                    else
                        for (int j = 0; j < nbox; ++j)
                            tma_load_2d_2sm(stage_b + s * kStageBytes + j * kBoxBytes, &tmap_x, full_b_leader + s * 8,
                                            0, (int)(kb * p.tpad) + row_half + j * kBoxRows);
                }
                __syncwarp();
            }
        }
    } else if (warp == kWarpMma) {
        // ---------------- MMA issuer (leader, one thread) ----------------
        // A tight single-thread loop: per k-block one CTA-scope wait, four MMAs and a commit with every
        // operand in uniform registers (the per-unit N goes into a runtime instruction descriptor).  The
        // peer's dequantizers and TMA signal the leader's full barrier; TMEM ordering comes from their
        // tcgen05 fences, so no cluster-scope acquire (and its L1 invalidation) is needed per k-block.
        if (rank == 0 && elect_one_sync()) {
            const uint64_t bdesc0 = sdesc_sw128(smem_u32(stage_b));
            uint32_t it = 0;
            for (uint32_t tc = 0;; ++tc) {
                const int s0 = (int)(tc % kURing);
                mbar_wait(&u_full[s0], (tc / kURing) & 1);
                const int pair = *reinterpret_cast<volatile int32_t*>(&uring[s0]);
                mbar_arrive(&u_empty[s0]);
                if (pair < 0) break;
                const int tn = __ldg(&p.tiles[pair / n_pairs_row].n);
                const uint32_t nc = (uint32_t)max(32, (int)round_up(tn, 32));
                const uint32_t idesc = idesc_f16(256, nc, 0);
                mbar_wait_cluster(acc_empty, (tc & 1) ^ 1);  // both CTAs' epilogues drained the accumulator
                EVU(0, tc);
                if (TRACE && blockIdx.x < 2 && tc < 16) p.trace[24576 + 6 * 16 + tc] = nc;
                tc_fence_after();
                for (int kb = 0; kb < kb_n; ++kb, ++it) {
                    const uint32_t s = it % NSTAGE;
                    mbar_wait(&full_b[s], (it / NSTAGE) & 1);
                    EV(1, kb, tc);
                    tc_fence_after();
                    const uint32_t acol = kACol0 + s * 32;
                    const uint64_t bdesc = bdesc0 + (uint64_t)(s * (kStageBytes >> 4));
#pragma unroll
                    for (int j = 0; j < kKBlock / 16; ++j)
                        mma_ts_f16_2sm(0u, acol + j * 8, bdesc + (uint64_t)(j * 2), idesc, (kb | j) != 0 ? 1u : 0u);
                    mma_commit_2sm_mc(&empty[s], (uint16_t)0x3);
                    EV(3, kb, tc);
                }
                mma_commit_2sm_mc(acc_full, (uint16_t)0x3);
                EVU(1, tc);
            }
        }
        __syncwarp();
    } else if (warp < kWarpEpi0) {
        // ---------------- dequantizers ----------------
        // 16 warps = 4 TMEM lane quarters x 2 k-halves x 2 k-block parities: a warp dequantizes
        // 32 codes of its row for every other k-block, so two k-blocks are in flight at once.
        const int idx = warp - kWarpDq0;
        const int q = warp % 4;
        const int par = (idx / 4) & 1;
        const int hh = idx / 8;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        const uint32_t full_leader = mapa_shared(smem_u32(full_b), 0);
        uint32_t base = 0;  // global k-block counter at the start of the tile (stage/phase)
        for (uint32_t ui = 0;; ++ui, base += kb_n) {
            const int pair = unit_get(ui);
            if (pair < 0) break;
            TokTile tt;
            int rt, nc;
            tile_of(pair, tt, rt, nc);
            const int64_t R = (int64_t)rt * kRowTile + 32 * q + lane;
            const bool rv = R < p.out;
            const uint32_t mw = p.mt.maskword[tt.mask];
            const float kc = p.mt.kc[tt.mask];
            const uint8_t* cbase =
                p.codes8 + (int64_t)rt * p.kblocks * kBlockBytes + ((hh * 2) * kRowTile + 32 * q + lane) * 16;
            const float2* gcol = p.gconst + (rv ? R : 0);
            auto ldc = [&](int gg) {
                if (MOBI_X_NOLOAD) return make_float2(0.01f * gg, 0.02f);
                return rv ? __ldg(gcol + (int64_t)gg * p.out_pad) : make_float2(0.f, 0.f);
            };
            auto ld = [&](int kb, uint4& c0, uint4& c1) {
                if (MOBI_X_NOLOAD) {
                    c0 = make_uint4(kb, kb * 3, kb * 5, kb * 7);
                    c1 = make_uint4(kb * 11, kb, kb * 13, kb);
                    return;
                }
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
                if (MOBI_X_NODQ) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[2 * u] = v[2 * u + 1] = w0[u];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[8 + 2 * u] = v[8 + 2 * u + 1] = w1[u];
                    return;
                }
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
                kinp = par * kKBlock + hh * 32;
                while (kinp >= p.gs) kinp -= (int)p.gs, ++gp;
            }
            auto fetch = [&](int kb, uint4& c0, uint4& c1, float2& gc) {
                if (kb < kb_n) {
                    ld(kb, c0, c1);
                    gc = ldc(gp);
                }
                if (!p.single_group) {
                    kinp += 2 * kKBlock;
                    while (kinp >= p.gs) kinp -= (int)p.gs, ++gp;
                }
            };
            fetch(par, c00, c01, g0);
            fetch(par + 2, c10, c11, g1);
            fetch(par + 4, c20, c21, g2);
            uint32_t v[16];
            auto step = [&](int kb, uint4& ca, uint4& cb, float2& ga, uint4& na, uint4& nb, float2& gn) -> bool {
                // v holds k-block kb (dequantized from the slot (ca, cb)); (na, nb) holds kb+2
                if (kb >= kb_n) return false;
                const uint32_t itk = base + kb;
                const int s = itk % NSTAGE;
                const uint32_t ph = (itk / NSTAGE) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                if (warp == 0 || warp == 4) EV(4, kb, ui);
                tc_fence_after();
                tmem_st16(tmem + lane_base + kACol0 + s * 32 + hh * 16, v);
                fetch(kb + 6, ca, cb, ga);  // refill the consumed slot three of this warp's k-blocks ahead
                if (warp == 0 || warp == 4) EV(6, kb, ui);
                if (kb + 2 < kb_n) dq(na, nb, gn, v);
                if (warp == 0 || warp == 4) EV(7, kb, ui);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (warp == 0 || warp == 4) EV(5, kb, ui);
                if (lane == 0) {
#if MOBI_RELAXED
                    if (rank == 0)
                        mbar_arrive_relaxed(&full_b[s]);
                    else
                        mbar_arrive_relaxed_cluster(full_leader + s * 8);
#else
                    if (rank == 0)
                        mbar_arrive(&full_b[s]);
                    else
                        mbar_arrive_cluster(full_leader + s * 8);
#endif
                }
                return true;
            };
            if (par < kb_n) dq(c00, c01, g0, v);
            for (int kb = par; kb < kb_n; kb += 6) {
                if (!step(kb, c00, c01, g0, c10, c11, g1)) break;
                if (!step(kb + 2, c10, c11, g1, c20, c21, g2)) break;
                if (!step(kb + 4, c20, c21, g2, c00, c01, g0)) break;
            }
        }
    } else {
        // ---------------- epilogue ----------------
        // drain TMEM -> (x 2^e) -> bf16 -> smem tile [token][128 rows], release the accumulator,
        // then scatter whole 256-byte token rows into Y[perm[i]] with 16-byte stores
        const int q = warp % 4;
        const int et = threadIdx.x - 32 * kWarpEpi0;  // 0..127
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        for (uint32_t tc = 0;; ++tc) {
            const int pair = unit_get(tc);
            if (pair < 0) break;
            TokTile tt;
            int rt, nc;
            tile_of(pair, tt, rt, nc);
            int32_t src_r[kTokTile / 32];
            float es_r[kTokTile / 32];
#pragma unroll
            for (int c = 0; c < kTokTile / 32; ++c) {
                const bool ok = 32 * c + lane < tt.n;
                src_r[c] = ok ? __ldg(p.perm + tt.row0 + 32 * c + lane) : -1;
                es_r[c] = ok ? __ldg(p.escale + tt.row0 + 32 * c + lane) : 0.f;
            }
            // CTA-scope wait: the arrival is the tensor core's commit and TMEM visibility comes from
            // tcgen05.fence (a cluster-scope acquire would invalidate L1 on every poll)
            mbar_wait(acc_full, tc & 1);
            if (warp == kWarpEpi0) EVU(2, tc);
            tc_fence_after();
            if (MOBI_X_NOEPI) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(acc_empty), 0));
                continue;
            }
            epi_bar_sync();  // the previous tile's scatter has finished reading the staging tile
            if (warp == kWarpEpi0) EVU(5, tc);
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
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(acc_empty), 0));  // leader's barrier
            if (warp == kWarpEpi0) EVU(3, tc);
            epi_bar_sync();  // staging tile complete
            const int64_t r0 = (int64_t)rt * kRowTile + 8 * (et % 16);
            for (int t = et / 16; t < tt.n; t += 8) {
                const int32_t src = tok_src[t];
                if (src < 0 || r0 >= p.out) continue;
                const __nv_bfloat16* sp = stage_y + t * kRowTile + 8 * (et % 16);
                const int64_t off = (int64_t)src * p.od.ldy + p.od.col0 + r0;
                if (p.vec_y && r0 + 8 <= p.out) {
                    const uint4 v = *reinterpret_cast<const uint4*>(sp);
                    for (int k = 0; k < p.od.n_dst; ++k) *reinterpret_cast<uint4*>(p.od.dst[k] + off) = v;
                } else {
                    for (int k = 0; k < p.od.n_dst; ++k)
                        for (int u = 0; u < 8 && r0 + u < p.out; ++u) p.od.dst[k][off + u] = sp[u];
                }
            }
            if (warp == kWarpEpi0) EVU(4, tc);
        }
        // peer destinations: make this CTA's stores to other GPUs' memory visible system-wide before the
        // kernel completes (the caller orders the peers' reads after it with a collective)
        if (p.od.n_dst > 1) __threadfence_system();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == kWarpMma) tmem_dealloc_2sm(tmem, 512);
}


}  // namespace

int launch_gemm_tc2(mobi_layer* L, __nv_bfloat16* y, int64_t T, cudaStream_t st, unsigned long long* trace,
                    bool pdl) {
    {
        MOBI_TRY(func_attr_once(mobi_gemm_tc2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBytes));
        MOBI_TRY(func_attr_once(mobi_gemm_tc2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBytes));
    }
    if (!L->tmap_x2) {
        L->tmap_x2 = new CUtensorMap[2];
        const int64_t rows = L->kblocks * L->tpad_max;
        int rc = make_tmap_2d(&L->tmap_x2[0], L->xperm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, kKBlock, kBoxRows);
        if (!rc) rc = make_tmap_2d(&L->tmap_x2[1], L->xperm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, kKBlock, kBigBoxRows);
        if (rc) {
            delete[] L->tmap_x2;
            L->tmap_x2 = nullptr;
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
    if (L->od.n_dst > 0) {
        p.od = L->od;
    } else {
        p.od = OutDesc{};
        p.od.dst[0] = y;
        p.od.n_dst = 1;
        p.od.ldy = L->out;
        p.od.col0 = 0;
    }
    bool al = L->out % 8 == 0 && p.od.ldy % 8 == 0 && p.od.col0 % 8 == 0;
    for (int k = 0; k < p.od.n_dst; ++k) al = al && (reinterpret_cast<uintptr_t>(p.od.dst[k]) & 15) == 0;
    p.vec_y = al;
    const int64_t max_pairs = (int64_t)(p.n_row_tiles / 2) * L->max_tiles;
    const int grid = 2 * (int)std::min<int64_t>(L->n_sm / 2, max_pairs);
    p.trace = trace;
    p.bk_hist = L->bk_hist;
    p.unit_ctr = L->meta + 32;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];  // (cluster shape from __cluster_dims__)
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    if (trace)
        MOBI_CUDA(cudaLaunchKernelEx(&cfg, mobi_gemm_tc2_kernel<true>, *(&L->tmap_x2[0]), *(&L->tmap_x2[1]), p));
    else
        MOBI_CUDA(cudaLaunchKernelEx(&cfg, mobi_gemm_tc2_kernel<false>, *(&L->tmap_x2[0]), *(&L->tmap_x2[1]), p));
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    L->plan[1] = MOBI_K_GEMM_PAIR;
    L->plan[2] = grid;
    return MOBI_OK;
}

}  // namespace mobi
