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
// With half-height B stages (16 KiB) the ring is 6 deep in both smem (B) and TMEM (A).
//
// Codes reach the dequantizers through shared memory: a code warp per CTA bulk-copies each
// k-block's 8 KiB code block and the 1 KiB (s, s*z) slices of its groups into a 6-deep ring that the
// dequantizers release as soon as they have read it (not when the MMAs finish), so a copy is issued
// up to 8 + 5 k-blocks ahead of the MMA that consumes it.  A stage is two k-blocks (16 KiB of codes, one
// bulk copy) plus the constants of the groups they touch (one 1 KiB copy per group: one for gs >= 128):
// a single producer thread pays ~200 cycles of issue latency per bulk/TMA instruction, so per-k-block
// instruction counts, not bytes, bound the producers.  Likewise the B tile of a stage is ONE TMA box
// (16/32/64/128 rows, the smallest >= N/2; rows past the tile are loaded and ignored).  (Per-lane LDG
// prefetch rings of codes were bound by load issue and L2 latency: ~700 cycles per k-block whatever N.)
#include <algorithm>

#include "mobi_internal.cuh"
#include "sm100.cuh"

#ifndef MOBI_MMA_WAIT
#define MOBI_MMA_WAIT 0
#endif
// bottleneck experiments (development only; all 0 in the product): drop one producer's real work
#ifndef MOBI_X_NOTMA
#define MOBI_X_NOTMA 0   // the TMA warp arrives without loading B
#endif
#ifndef MOBI_X_NOCODE
#define MOBI_X_NOCODE 0  // the code warp arrives without copying (codes/constants garbage)
#endif
#ifndef MOBI_X_NOST
#define MOBI_X_NOST 0    // dequantizers skip the TMEM store (garbage A)
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
#ifndef MOBI_WAIT_SLEEP
#define MOBI_WAIT_SLEEP 1
#endif
namespace mobi {
int make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int64_t rows, int64_t cols,
                 int box_rows);
namespace {

using namespace sm100;
#if MOBI_WAIT_SLEEP
#define WAITX mbar_wait_sleep
#else
#define WAITX mbar_wait
#endif

constexpr int NSTAGE = 5;   // B (smem) / A (TMEM) stages
constexpr int NCS = 4;      // code stages (smem, 2 k-blocks each), released by the dequantizers, not by the MMAs
constexpr int kCodeKb = 2;  // k-blocks per code stage: one 16 KiB bulk copy (a row tile's k-blocks are contiguous)
constexpr int kDqWarps = 16;
constexpr int kEpiWarps = 8;  // two per TMEM lane quarter (alternate 16-column chunks)
constexpr int kThreads = 32 * (4 + kDqWarps + kEpiWarps);
constexpr int kWarpDq0 = 0, kWarpEpi0 = kDqWarps, kWarpTma = kDqWarps + kEpiWarps, kWarpMma = kWarpTma + 1;
constexpr int kWarpCode = kWarpTma + 2;  // 2 warps bulk-copy the code stages (alternating) into smem
constexpr int kCodeWarps = 2;
// dynamic unit schedule: the leader's TMA warp claims units (atomic counter, units in decreasing
// size order) and publishes them through a small ring to every role of both CTAs
constexpr int kURing = 4;
constexpr int kUnitConsumers = 1 + kCodeWarps + kDqWarps + kEpiWarps;  // per CTA: MMA (leader) or TMA (peer) + code + dequant + epilogue
constexpr int kHalfRows = kTokTile / 2;                  // token rows per CTA per stage
constexpr int kStageBytes = kHalfRows * kKBlock * 2;     // 16 KiB
constexpr int kACol0 = 256;
constexpr int kYStageBytes = kTokTile * kRowTile * 2;    // 64 KiB
constexpr int kConstOff = kCodeKb * kBlockBytes;
constexpr int kCodeStage = kConstOff + 2 * kCodeKb * kRowTile * 8;  // codes + (s, s*z) of up to 4 groups x 128 rows
// (no alignment slack: the dynamic smem base is declared 1024-aligned; checked at run time)
constexpr int kSmemBytes = NSTAGE * kStageBytes + 512 + kYStageBytes + 2 * kTokTile * 4 + NCS * kCodeStage;
static_assert(kSmemBytes <= 232448, "tc2 shared memory");
static_assert(NCS % kCodeWarps == 0, "each code warp owns fixed ring slots");

struct Params {
    const uint8_t* codes8;
    const float2* gconst;
    int64_t out_pad;
    MaskTable mt;
    int64_t out, G, gs, kblocks;
    int64_t tpad;
    int single_group;
    int g_uniform;  // every code stage (128 columns) lies in one group: single group or gs % 128 == 0
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
    mobi_gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmap16, const __grid_constant__ CUtensorMap tmap32,
                         const __grid_constant__ CUtensorMap tmap64, const __grid_constant__ CUtensorMap tmap128,
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
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    uint8_t* stage_b = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSTAGE * kStageBytes);
    // one full barrier per stage, in the leader: both halves' TMA bytes (one expect_tx arrival) and the
    // 8 + 8 dequant warps of the pair (the peer's arrive remotely)
    uint64_t* full_b = bars;                 // [NSTAGE] leader: B in both CTAs' smem (TMA bytes) + A in both TMEMs
    uint64_t* empty = bars + NSTAGE;         // [NSTAGE] each CTA: pair MMAs done with the stage
    uint64_t* acc_full = bars + 2 * NSTAGE;  // each CTA
    uint64_t* acc_empty = acc_full + 1;      // leader: both CTAs drained TMEM
    uint64_t* u_full = acc_empty + 1;        // [kURing] each CTA: unit slot published
    uint64_t* u_empty = u_full + kURing;     // [kURing] leader: every consumer of both CTAs read the slot
    int32_t* uring = reinterpret_cast<int32_t*>(u_empty + kURing + 2 * NCS + NSTAGE);  // [kURing] unit (-1 = done)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uring + kURing);
    uint8_t* stage_y = smem + NSTAGE * kStageBytes + 512;  // [128 rows][256 tokens] bf16, 16-byte chunks swizzled
    float* tok_es = reinterpret_cast<float*>(smem + NSTAGE * kStageBytes + 512 + kYStageBytes);  // [kTokTile]
    int32_t* tok_src = reinterpret_cast<int32_t*>(tok_es + kTokTile);                               // [kTokTile]
    uint8_t* stage_c = smem + NSTAGE * kStageBytes + 512 + kYStageBytes + 2 * kTokTile * 4;  // [NCS][kCodeStage]
    uint64_t* c_full = u_empty + kURing;   // [NCS] each CTA: the stage's codes + constants landed
    uint64_t* c_empty = c_full + NCS;      // [NCS] each CTA: the 256 lanes of its two k-blocks' 8 dequant warps read them
    uint64_t* full_a = full_b;             // one full barrier per stage: the A stores join the B bytes
    auto epi_bar_sync = [] { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); };

    const int warp = warp_idx_uniform(), lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023) __trap();  // SW128 B stages need 1024-byte alignment
        for (int s = 0; s < NSTAGE; ++s) {
            // the leader's TMA expect_tx + its 4 dequant warps' lanes (each after its own TMEM store) + the
            // peer's 4 dequant warps (one remote arrival each)
            mbar_init(&full_b[s], 1 + kDqWarps / 4 * 32 + kDqWarps / 4);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 2 * kEpiWarps);  // every epilogue warp of both CTAs
        for (int s = 0; s < kURing; ++s) {
            mbar_init(&u_full[s], 1);
            mbar_init(&u_empty[s], 2 * kUnitConsumers);
        }
        for (int s = 0; s < NCS; ++s) {
            mbar_init(&c_full[s], 1);
            mbar_init(&c_empty[s], kDqWarps / 2 * 32);  // every lane of the stage's 8 dequant warps
        }
        fence_barrier_init();
        prefetch_tmap(&tmap16);
        prefetch_tmap(&tmap32);
        prefetch_tmap(&tmap64);
        prefetch_tmap(&tmap128);
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
            WAITX(&u_full[s], ph);
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
            // one box per CTA per stage: the smallest of 16/32/64/128 rows covering N/2
            const int half = nc / 2;
            const int bx = half <= 16 ? 16 : half <= 32 ? 32 : half <= 64 ? 64 : 128;
            const CUtensorMap* tm = bx == 16 ? &tmap16 : bx == 32 ? &tmap32 : bx == 64 ? &tmap64 : &tmap128;
            const int row_half = tt.row0 + (int)rank * half;
            for (int kb = 0; kb < kb_n; ++kb, ++it) {
                const int s = it % NSTAGE;
                const uint32_t ph = (it / NSTAGE) & 1;
                WAITX(&empty[s], ph ^ 1);
                EV(0, kb, ui);
                if (MOBI_X_NOTMA) {
                    if (elect_one_sync() && rank == 0) mbar_arrive_expect_tx(&full_b[s], 0);
                } else if (elect_one_sync()) {
                    if (rank == 0) mbar_arrive_expect_tx(&full_b[s], 2 * bx * kKBlock * 2);
                    tma_load_2d_2sm(stage_b + s * kStageBytes, tm, full_b_leader + s * 8, 0,
                                    (int)(kb * p.tpad) + row_half);
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
                WAITX(&u_full[s0], (tc / kURing) & 1);
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
                    WAITX(&full_b[s], (it / NSTAGE) & 1);
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
    } else if (warp >= kWarpCode) {
        // ---------------- code producers (each CTA: its own 128-row tile) ----------------
        // two warps alternate code stages (global stage parity): a single thread needs ~1000 cycles to
        // issue one stage's expect_tx + bulk copies, longer than the MMAs of two k-blocks at N <= 128
        // per k-block: the 8 KiB code block and, for each k-half, the 1 KiB (s, s*z) row slice of its
        // group; the ring slot is released by the dequantizers as soon as they have read it
        uint32_t it = 0;
        for (uint32_t ui = 0;; ++ui) {
            const int pair = unit_get(ui);
            if (pair < 0) break;
            TokTile tt;
            int rt, nc;
            tile_of(pair, tt, rt, nc);
            const uint8_t* csrc = p.codes8 + (int64_t)rt * p.kblocks * kBlockBytes;
            const float2* gsrc = p.gconst + (int64_t)rt * kRowTile;
            for (int kb0 = 0; kb0 < kb_n; kb0 += kCodeKb, ++it) {
                if ((int)(it % kCodeWarps) != warp - kWarpCode) continue;
                const int s = (int)(it % NCS);
                WAITX(&c_empty[s], ((it / NCS) & 1) ^ 1);
                fence_proxy_async_smem();  // the dequantizers' reads of the slot precede the next copy into it
                EV(6, kb0, ui);
#ifndef MOBI_LANE_ISSUE
#define MOBI_LANE_ISSUE 1
#endif
                if (MOBI_X_NOCODE) {
                    if (elect_one_sync()) mbar_arrive_expect_tx(&c_full[s], 0);
                } else {
                    uint8_t* dc = stage_c + s * kCodeStage;
                    const int nkb = min(kCodeKb, kb_n - kb0);
                    // groups of the stage's first and last 32-column chunks (gs is a multiple of 32 or >= in)
                    const int g0 = p.single_group ? 0 : (int)((uint32_t)(kb0 * kKBlock) / (uint32_t)p.gs);
                    const int g1 = p.single_group ? 0 : (int)((uint32_t)((kb0 + nkb) * kKBlock - 32) / (uint32_t)p.gs);
                    if (lane == 0)
                        mbar_arrive_expect_tx(&c_full[s], nkb * kBlockBytes + (uint32_t)(g1 - g0 + 1) * kRowTile * 8);
                    __syncwarp();
                    if (MOBI_LANE_ISSUE) {
                        // one instruction, one copy per lane: lane 0 the codes, lane 1 + j group g0 + j
                        if (lane <= g1 - g0 + 1) {
                            const bool cl = lane == 0;
                            const int g = g0 + lane - 1;
                            bulk_g2s(cl ? dc : dc + kConstOff + (g - g0) * kRowTile * 8,
                                     cl ? (const void*)(csrc + (int64_t)kb0 * kBlockBytes)
                                        : (const void*)(gsrc + (int64_t)g * p.out_pad),
                                     cl ? nkb * kBlockBytes : kRowTile * 8, &c_full[s]);
                        }
                    } else if (lane == 0) {
                        bulk_g2s(dc, csrc + (int64_t)kb0 * kBlockBytes, nkb * kBlockBytes, &c_full[s]);
                        for (int g = g0; g <= g1; ++g)
                            bulk_g2s(dc + kConstOff + (g - g0) * kRowTile * 8, gsrc + (int64_t)g * p.out_pad,
                                     kRowTile * 8, &c_full[s]);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp < kWarpEpi0) {
        // ---------------- dequantizers ----------------
        // 16 warps = 4 TMEM lane quarters x 4 k-block phases: a warp dequantizes the 64 codes of its
        // row in every fourth k-block (one 32-column TMEM store), so each warp has four k-blocks of MMA
        // time to cover its smem reads, ALU work and the TMEM store latency.  Code stage j (k-blocks 2j,
        // 2j+1) is read by the 8 warps of phases 2(j%2), 2(j%2)+1.  Per k-block: dequantize (codes
        // already in registers), release the code stage, read the next k-block's codes, then -- once
        // the MMAs are done with the A stage -- store into TMEM and arrive on the stage's full barrier.
        const int idx = warp - kWarpDq0;
        const int q = idx % 4;
        const int ph4 = idx / 4;            // (code-stage parity, k-block inside the stage)
        const int jpar = ph4 >> 1;          // code stages j with j % 2 == jpar
        const int sub = ph4 & 1;            // k-block inside the stage
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        const uint32_t full_leader = mapa_shared(smem_u32(full_a), 0);
        const int c_off = sub * kBlockBytes + (32 * q + lane) * 16;  // + (h*2 + c) * kRowTile * 16
        uint32_t base = 0;   // global k-block counter at the start of the unit (A/B stage and phase)
        uint32_t cbase = 0;  // global code-stage counter at the start of the unit
        for (uint32_t ui = 0;; ++ui) {
            const int pair = unit_get(ui);
            if (pair < 0) break;
            TokTile tt;
            int rt, nc;
            tile_of(pair, tt, rt, nc);
            const uint32_t mw = p.mt.maskword[tt.mask];
            const float kc = p.mt.kc[tt.mask];
            const int ncs_u = (kb_n + kCodeKb - 1) / kCodeKb;
            // this warp's code stages: j = j0, j0 + 2, ... (global stage parity, so both phases of a
            // stage agree on which warps read it across units with an odd stage count)
            const int j0 = (int)((jpar - (int)(cbase & 1) + 2) & 1);
            uint4 c[4];
            float2 g[2];
            auto load = [&](int j) {
                const uint32_t cit = cbase + j;
                const int cs = (int)(cit % NCS);
                WAITX(&c_full[cs], (cit / NCS) & 1);
                const int kb = kCodeKb * j + sub;
                if (kb < kb_n) {
                    const uint8_t* dc = stage_c + cs * kCodeStage + c_off;
#pragma unroll
                    for (int u = 0; u < 4; ++u) c[u] = *reinterpret_cast<const uint4*>(dc + u * kRowTile * 16);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        // group slot inside the stage: 0 whenever a stage's 128 columns are one group
                        const int gslot = p.g_uniform ? 0
                                                      : (int)((uint32_t)(kb * kKBlock + 32 * hh) / (uint32_t)p.gs -
                                                              (uint32_t)(kCodeKb * j * kKBlock) / (uint32_t)p.gs);
                        g[hh] = *reinterpret_cast<const float2*>(stage_c + cs * kCodeStage + kConstOff +
                                                                  (gslot * kRowTile + 32 * q + lane) * 8);
                    }
                }
            };
            uint32_t v[32];
            if (j0 < ncs_u) load(j0);
            for (int j = j0; j < ncs_u; j += 2) {
                const int kb = kCodeKb * j + sub;
                const bool valid = kb < kb_n;
                if (valid) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const __half2 S2 = __float2half2_rn(g[hh].x * p.mt.inv_2p);
                        const __half2 C2 = __float2half2_rn(fmaf(g[hh].x, kc, -g[hh].y));
#pragma unroll
                        for (int cc = 0; cc < 2; ++cc) {
                            const uint32_t* w = reinterpret_cast<const uint32_t*>(&c[hh * 2 + cc]);
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int o = hh * 16 + cc * 8 + 2 * u;
                                if (MOBI_X_NODQ)
                                    v[o] = v[o + 1] = w[u];
                                else
                                    dequant4(w[u], mw, S2, C2, v[o], v[o + 1]);
                            }
                        }
                    }
                }
                // the stage's data is in registers (consumed above): release the slot to the code warp,
                // every lane for its own reads (the next bulk copy into the slot is an async-proxy write)
                mbar_arrive(&c_empty[(cbase + j) % NCS]);
                if (valid) {
                    const uint32_t itk = base + kb;
                    const int s = (int)(itk % NSTAGE);
                    WAITX(&empty[s], ((itk / NSTAGE) & 1) ^ 1);
                    if (warp == 0) EV(4, kb, ui);
                    tc_fence_after();
                    if (!MOBI_X_NOST) {
                        tmem_st32(tmem + lane_base + kACol0 + s * 32, v);
                        tmem_st_wait();
                    }
                    tc_fence_before();
                    if (warp == 0) EV(5, kb, ui);
                    if (warp == 3) EV(2, kb, ui);
                    if (rank == 0) {
                        mbar_arrive_relaxed(&full_a[s]);  // every lane, after its own wait::st
                    } else {
                        __syncwarp();
                        if (lane == 0) mbar_arrive_relaxed_cluster(full_leader + s * 8);
                    }
                }
                // the next code stage only after this k-block's A is in TMEM: a late code copy must not
                // hold back the MMAs of the stage already dequantized
                if (j + 2 < ncs_u) load(j + 2);
            }
            base += kb_n;
            cbase += ncs_u;
        }
    } else {
        // ---------------- epilogue ----------------
        // The accumulator is released as soon as it is drained into a TRANSPOSED staging tile
        // [row][token] (each thread: its TMEM lane = weight row, 16 tokens per load, two 16-byte smem
        // stores); the un-permute scatter of whole 256-byte token rows into Y[perm[i]] reads that tile
        // back transposed (8 rows x 2 tokens per thread) while the next unit's MMAs run.  16-byte chunks
        // of a row are XOR-swizzled by g(r) so both the drain stores and the scatter reads spread over
        // the banks.
        const int q = warp % 4;                       // TMEM lane quarter (hardware: warp id % 4)
        const int half = (warp - kWarpEpi0) / 4;      // 16-column chunks c with c % 2 == half
        const int et = threadIdx.x - 32 * kWarpEpi0;  // 0 .. 32*kEpiWarps-1
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        auto swz = [](int r) { return (r ^ (r >> 3)) & 7; };
        const int my_r = 32 * q + lane;
        uint8_t* my_row = stage_y + my_r * (kTokTile * 2);
        const int my_g = swz(my_r);
        for (uint32_t tc = 0;; ++tc) {
            const int pair = unit_get(tc);
            if (pair < 0) break;
            TokTile tt;
            int rt, nc;
            tile_of(pair, tt, rt, nc);
            epi_bar_sync();  // the previous unit's scatter has finished reading the staging tile
            for (int t = et; t < nc; t += 32 * kEpiWarps) {
                const bool ok = t < tt.n;
                tok_es[t] = ok ? __ldg(p.escale + tt.row0 + t) : 0.f;
                tok_src[t] = ok ? __ldg(p.perm + tt.row0 + t) : -1;
            }
            epi_bar_sync();
            // CTA-scope wait: the arrival is the tensor core's commit and TMEM visibility comes from
            // tcgen05.fence (a cluster-scope acquire would invalidate L1 on every poll)
            WAITX(acc_full, tc & 1);
            if (warp == kWarpEpi0) EVU(2, tc);
            tc_fence_after();
            if (MOBI_X_NOEPI) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(acc_empty), 0));
                continue;
            }
            if (warp == kWarpEpi0) EVU(5, tc);
            uint32_t va[16], vb[16];
            if (16 * half < tt.n) tmem_ld16(tmem + lane_base + 16 * half, va);
#pragma unroll
            for (int i = 0; i < kTokTile / 32; ++i) {
                const int c = 2 * i + half;
                const int c0 = 16 * c;
                if (c0 >= tt.n) break;
                if (TRACE && warp == kWarpEpi0 && lane == 0 && blockIdx.x < 2 && tc == MOBI_TRACE_UNIT)
                    p.trace[28672 + rank * 64 + 2 * i] = (unsigned long long)clock64();
                tmem_ld_wait();
                if (TRACE && warp == kWarpEpi0 && lane == 0 && blockIdx.x < 2 && tc == MOBI_TRACE_UNIT)
                    p.trace[28672 + rank * 64 + 2 * i + 1] = (unsigned long long)clock64();
                uint32_t(&cur)[16] = (i & 1) ? vb : va;
                uint32_t(&nxt)[16] = (i & 1) ? va : vb;
                if (c0 + 32 < tt.n) tmem_ld16(tmem + lane_base + c0 + 32, nxt);
                // bf16 of the raw accumulator; the token's 2^e comes in the scatter (a power-of-two
                // scale of a bf16 value is exact, so the result equals rounding acc * 2^e)
                uint32_t w[8];
#pragma unroll
                for (int j2 = 0; j2 < 8; ++j2) {
                    const __nv_bfloat162 h2 =
                        __floats2bfloat162_rn(__uint_as_float(cur[2 * j2]), __uint_as_float(cur[2 * j2 + 1]));
                    w[j2] = *reinterpret_cast<const uint32_t*>(&h2);
                }
                const int ch = 2 * c;  // 16-byte chunk (8 tokens) index
                *reinterpret_cast<uint4*>(my_row + ((ch ^ my_g) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
                *reinterpret_cast<uint4*>(my_row + (((ch + 1) ^ my_g) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(acc_empty), 0));  // leader's barrier
            if (warp == kWarpEpi0) EVU(3, tc);
            epi_bar_sync();  // staging tile complete
            // scatter: thread = (8-row chunk et%16, token pair); 8 four-byte reads give 8 rows x 2 tokens
            const int rc0 = 8 * (et % 16);
            const int64_t r0 = (int64_t)rt * kRowTile + rc0;
            for (int t = 2 * (et / 16); t < tt.n; t += 2 * (32 * kEpiWarps / 16)) {
                uint32_t wv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int r = rc0 + u;
                    wv[u] = *reinterpret_cast<const uint32_t*>(stage_y + r * (kTokTile * 2) +
                                                              (((t >> 3) ^ swz(r)) << 4) + (t & 7) * 2);
                }
                // token t: the low halves (x 2^e of t), token t+1: the high halves (x 2^e of t+1), in fp32
                const float e0 = tok_es[t], e1 = tok_es[t + 1];
                uint32_t o0[4], o1[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t a = wv[2 * u], b = wv[2 * u + 1];  // rows 2u, 2u+1: (t, t+1) each
                    const __nv_bfloat162 lo = __floats2bfloat162_rn(__uint_as_float(a << 16) * e0,
                                                                    __uint_as_float(b << 16) * e0);
                    const __nv_bfloat162 hi = __floats2bfloat162_rn(__uint_as_float(a & 0xffff0000u) * e1,
                                                                    __uint_as_float(b & 0xffff0000u) * e1);
                    o0[u] = *reinterpret_cast<const uint32_t*>(&lo);
                    o1[u] = *reinterpret_cast<const uint32_t*>(&hi);
                }
                const uint4 y0 = make_uint4(o0[0], o0[1], o0[2], o0[3]);
                const uint4 y1 = make_uint4(o1[0], o1[1], o1[2], o1[3]);
                if (r0 >= p.out) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (t + h >= tt.n) break;
                    const int32_t src = tok_src[t + h];
                    const uint4 v = h ? y1 : y0;
                    const int64_t off = (int64_t)src * p.od.ldy + p.od.col0 + r0;
                    if (p.vec_y && r0 + 8 <= p.out) {
                        for (int k = 0; k < p.od.n_dst; ++k) *reinterpret_cast<uint4*>(p.od.dst[k] + off) = v;
                    } else {
                        const __nv_bfloat16* e8 = reinterpret_cast<const __nv_bfloat16*>(&v);
                        for (int k = 0; k < p.od.n_dst; ++k)
                            for (int u = 0; u < 8 && r0 + u < p.out; ++u) p.od.dst[k][off + u] = e8[u];
                    }
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
        L->tmap_x2 = new CUtensorMap[4];
        const int64_t rows = L->kblocks * L->tpad_max;
        int rc = 0;
        for (int i = 0; i < 4 && !rc; ++i)
            rc = make_tmap_2d(&L->tmap_x2[i], L->xperm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, kKBlock, 16 << i);
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
    p.g_uniform = L->single_group || L->gs % (kCodeKb * kKBlock) == 0;
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
        MOBI_CUDA(cudaLaunchKernelEx(&cfg, mobi_gemm_tc2_kernel<true>, L->tmap_x2[0], L->tmap_x2[1], L->tmap_x2[2],
                                     L->tmap_x2[3], p));
    else
        MOBI_CUDA(cudaLaunchKernelEx(&cfg, mobi_gemm_tc2_kernel<false>, L->tmap_x2[0], L->tmap_x2[1], L->tmap_x2[2],
                                     L->tmap_x2[3], p));
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    L->plan[1] = MOBI_K_GEMM_PAIR;
    L->plan[2] = grid;
    return MOBI_OK;
}

}  // namespace mobi
