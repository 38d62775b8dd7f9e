// router_tc.cu -- K1 on tcgen05: H = X[T,in] . w1[in,h] (bf16 operands, fp32 accumulate in TMEM),
// with silu(H + b1) . w2 fused into the epilogue (router.hpp:63-76).
//
// Tile: M = 128 tokens (TMEM lanes) x N = 128 hidden units, K-blocks of 64.  Both operands are
// TMA-loaded (128-byte swizzle) into a 6-stage shared-memory ring; one thread issues the MMAs;
// the accumulator is double-buffered in TMEM (2 x 128 columns) so the epilogue of tile i overlaps
// the MMAs of tile i+1.  Each epilogue thread owns one token and reduces its 128 hidden units to
// E-1 partial scores, written to s_part[hidden tile][token][j] and summed in a fixed order by the
// bucket kernel (deterministic, no atomics).
#include <algorithm>
#include <utility>
#include <cstdlib>

#include "mobi_internal.cuh"
#include "sm100.cuh"

namespace mobi {
int make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int64_t rows, int64_t cols,
                 int box_rows);
namespace {

using namespace sm100;

constexpr int RS = 6;                       // smem stages
constexpr int RM = 128, RN = 128;           // tokens x hidden per tile
constexpr int kAB = RM * kKBlock * 2;       // 16 KiB per operand per stage
#ifndef MOBI_RTMA2
#define MOBI_RTMA2 1
#endif
// 4 epilogue warps, TMA, MMA [, second TMA]: one thread's TMA issue chain (~350 cycles per stage,
// tools/pipe_probe.cu) is slower than the 4 N=128 MMAs a stage feeds, so two producer warps take
// alternate stages
constexpr int kRProducers = MOBI_RTMA2 ? 2 : 1;
constexpr int kRThreads = 192 + 32 * (kRProducers - 1);
constexpr int kRWarpTma = 4, kRWarpMma = 5, kRWarpTma2 = 6;
constexpr int kRSmem = RS * 2 * kAB + 1024 + 256 + 2 * RN * 16;  // + per-tile {b1, w2} staging
constexpr int kRecvBytes = RM * RN * 4;  // one peer's partial H tile, [RN/4][RM][4] floats
constexpr int kMaxCsplit = 1 + (RS * 2 * kAB) / kRecvBytes;  // the peers' partials fit rank 0's ring
static_assert(kMaxCsplit >= 3, "ring too small for a 3-way cluster split");

struct RParams {
    int64_t T, h, h_pad;
    int kblocks, n_mt, n_nt, nr;
    int nsplit, kb_per;  // split-K (decode-size T): raw hidden partials to hpart, reduced below
    int csplit;          // > 1: the nsplit (= csplit) CTAs of a tile form a cluster; ranks 1.. ship their
                         // partial H to rank 0 through DSMEM and rank 0 runs the fused epilogue
    const float* b1;
    const float* w2;
    float* s_part;
    float* hpart;        // [nsplit][T][h_pad]
    unsigned long long* trace;  // debug: CTA 0 timeline (null = off)
    // fused route decision (nsplit == 1): the last hidden tile of a token tile to finish sums the
    // partial scores in hidden-tile order (+ b2) and applies gate_hard(delta) (router.hpp:92-103)
    int* cnt;                   // [n_mt] arrival counters, zero between launches
    const float* b2;
    float delta;
    uint8_t* masks;             // [T]
    uint8_t* masks_out;         // optional
    float* scores_out;          // optional [T][nr]
    // fused bucketing: mask histogram (the gather lays the buckets out and claims slots; the GEMM
    // zeroes it again)
    int* hist;                  // [16] zero between launches
};

__global__ void __launch_bounds__(kRThreads, 1) router_tc_kernel(const __grid_constant__ CUtensorMap tmap_a,
                                                                 const __grid_constant__ CUtensorMap tmap_b,
                                                                 const RParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RS * 2 * kAB);
    uint64_t* full = bars;              // [RS]
    uint64_t* empty = bars + RS;        // [RS]
    uint64_t* acc_full = bars + 2 * RS; // [2]
    uint64_t* acc_empty = acc_full + 2; // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    uint64_t* peer_go = acc_empty + 4;    // cluster split-K: rank 0's ring is free for the peers' partials
    uint64_t* recv_full = acc_empty + 5;  // cluster split-K (rank 0): the peers' partials have landed
    // [2][RN] {b1[j], w2[j][0..2]} of the tile's hidden units, staged by the epilogue warps while the
    // mainloop runs so the SiLU.w2 epilogue reads them as smem broadcasts (not dependent global loads)
    float4* cst = reinterpret_cast<float4*>(smem + RS * 2 * kAB + 256);
    const int warp = warp_idx_uniform(), lane = threadIdx.x % 32;
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        for (int s = 0; s < RS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        mbar_init(peer_go, 1);
        mbar_init(recv_full, 1);
        fence_barrier_init();
        // rank 0 expects the peers' partials as bulk-copy bytes (complete_tx may land before or after)
        if (p.csplit > 1 && cluster_ctarank() == 0) mbar_arrive_expect_tx(recv_full, (p.csplit - 1) * kRecvBytes);
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
    }
    const long long t_start = clock64();
    unsigned long long g_start = 0;
    if (p.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_start));
    auto TR = [&](int i) {
        if (p.trace && blockIdx.x < 2 && (threadIdx.x % 32) == 0)
            p.trace[blockIdx.x * 1024 + i] = (unsigned long long)(clock64() - t_start);
    };
    if (warp == kRWarpMma) tmem_alloc(tmem_slot, 512);  // all columns: base is the constant 0
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (p.csplit > 1) cluster_sync();  // peers' barriers initialised before any remote arrive
    if (*tmem_slot != 0) __trap();
    // PDL: the prologue above overlapped the previous kernel; X (possibly its output) and every write
    // wait for it.  Only then may the gather launch: it reads X before its own wait.
    pdl_wait();
    pdl_trigger();
    constexpr uint32_t tmem = 0;
    const int total = p.n_mt * p.n_nt * p.nsplit;
    // tile -> (token tile mt, hidden tile nt, k-split ks)
    auto tile_of = [&](int tile, int& mt, int& nt, int& ks, int& kb0, int& kb1) {
        ks = tile % p.nsplit;
        const int q = tile / p.nsplit;
        mt = q % p.n_mt;
        nt = q / p.n_mt;
        kb0 = ks * p.kb_per;
        kb1 = min(p.kblocks, kb0 + p.kb_per);
    };

    if (warp == kRWarpTma || (kRProducers == 2 && warp == kRWarpTma2)) {
        const uint32_t mine = warp == kRWarpTma ? 0u : 1u;
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
            int mt, nt, ks, kb0, kb1;
            tile_of(tile, mt, nt, ks, kb0, kb1);
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                if ((it & (kRProducers - 1)) != mine) continue;
                const int s = it % RS;
                mbar_wait(&empty[s], ((it / RS) & 1) ^ 1);
                if (kb < 64) TR(128 + kb);
                if (elect_one_sync()) {
                    uint8_t* a = smem + s * 2 * kAB;
                    mbar_arrive_expect_tx(&full[s], 2 * kAB);
                    tma_load_2d(a, &tmap_a, &full[s], kb * kKBlock, mt * RM);
                    tma_load_2d(a + kAB, &tmap_b, &full[s], kb * kKBlock, nt * RN);
                }
                __syncwarp();
            }
        }
    } else if (warp == kRWarpMma) {
        if (elect_one_sync()) {  // one thread, operands in uniform registers (see router_tc2_kernel)
            uint32_t it = 0, tc = 0;
            const uint64_t desc0 = sdesc_sw128(smem_u32(smem));
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
                int mt, nt, ks, kb0, kb1;
                tile_of(tile, mt, nt, ks, kb0, kb1);
                const uint32_t n_mma = (uint32_t)std::min<int64_t>(RN, round_up(p.h - (int64_t)nt * RN, 16));
                const uint32_t idesc = idesc_f16(RM, n_mma, 1);
                const int buf = tc & 1;
                mbar_wait(&acc_empty[buf], ((tc >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + buf * RN;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t s = it % RS;
                    mbar_wait(&full[s], (it / RS) & 1);
                    if (kb < 64) TR(kb);
                    tc_fence_after();
                    const uint64_t adesc = desc0 + (uint64_t)((s * 2 * kAB) >> 4), bdesc = adesc + (uint64_t)(kAB >> 4);
#pragma unroll
                    for (int j = 0; j < kKBlock / 16; ++j)
                        mma_ss_f16(d, adesc + (uint64_t)(j * 2), bdesc + (uint64_t)(j * 2), idesc,
                                   (kb != kb0 || j != 0) ? 1u : 0u);
                    mma_commit(&empty[s]);
                }
                mma_commit(&acc_full[buf]);
            }
        }
        __syncwarp();
    } else {
        const int q = warp % 4;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        uint32_t tc = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
            int mt, nt, ks, kb0, kb1;
            tile_of(tile, mt, nt, ks, kb0, kb1);
            const int buf = tc & 1;
            const int64_t t = (int64_t)mt * RM + 32 * q + lane;
            const int64_t h0 = (int64_t)nt * RN;
            const int nh = (int)std::min<int64_t>(RN, p.h - h0);
            const bool clus = p.csplit > 1;
            const uint32_t crank = clus ? cluster_ctarank() : 0u;
            if (p.nsplit == 1 || (clus && crank == 0)) {
                const int et = 32 * q + lane;  // epilogue warps are 0..3
                float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
                if (et < nh) {
                    const int64_t hj = h0 + et;
                    c.x = __ldg(p.b1 + hj);
                    c.y = __ldg(p.w2 + hj * p.nr);
                    if (p.nr > 1) c.z = __ldg(p.w2 + hj * p.nr + 1);
                    if (p.nr > 2) c.w = __ldg(p.w2 + hj * p.nr + 2);
                }
                cst[buf * RN + et] = c;
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
            mbar_wait(&acc_full[buf], (tc >> 1) & 1);
            if (q == 0) TR(200);
            tc_fence_after();
            // cluster split-K receive buffer: rank 0's (idle) stage ring, [peer][column / 4][token row][4]
            const uint32_t recv0 = smem_u32(smem);
            if (clus && crank != 0) {  // peer: ship this K-range's H[128 x RN] to rank 0
                // stage it in this CTA's own (idle) ring as [column / 4][token row][4] floats, then one
                // bulk copy into rank 0's ring once rank 0 has released it
                for (int c0 = 0; c0 < RN; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + lane_base + buf * RN + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<uint4*>(smem + ((size_t)((c0 + j) / 4) * RM + 32 * q + lane) * 16) =
                            make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                }
                tc_fence_before();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> bulk copy
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (q == 0) TR(210);
                if (q == 0 && lane == 0) {
                    mbar_arrive(&acc_empty[buf]);
                    mbar_wait_cluster(peer_go, 0);
                    TR(211);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            mapa_shared(recv0 + (crank - 1) * (uint32_t)kRecvBytes, 0)),
                        "r"(recv0), "r"((uint32_t)kRecvBytes), "r"(mapa_shared(smem_u32(recv_full), 0))
                        : "memory");
                }
                continue;
            }
            if (clus) {  // rank 0: every MMA of this CTA has completed (acc_full), so no stage of the ring
                         // is read or written any more -- hand it to the peers, wait for their partials
                if (q == 0 && lane > 0 && lane < p.csplit)
                    mbar_arrive_cluster(mapa_shared(smem_u32(peer_go), (uint32_t)lane));
                mbar_wait_cluster(recv_full, 0);
                if (q == 0) TR(212);
            }
            if (p.nsplit > 1 && !clus) {  // raw hidden partial H[t, h0..h0+nh) for this k-split
                for (int c0 = 0; c0 < nh; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + lane_base + buf * RN + c0, v);
                    tmem_ld_wait();
                    if (t < p.T) {
                        float* dst = p.hpart + ((int64_t)ks * p.T + t) * p.h_pad + h0 + c0;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c0 + j < nh) dst[j] = __uint_as_float(v[j]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[buf]);
                continue;
            }
            float part0 = 0.f, part1 = 0.f, part2 = 0.f;
            for (int c0 = 0; c0 < nh; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + lane_base + buf * RN + c0, v);
                tmem_ld_wait();
                for (int r = 1; r < p.csplit; ++r) {  // H = rank 0 + rank 1 + ... (fixed order)
                    const uint8_t* src = smem + (size_t)(r - 1) * kRecvBytes;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 f = *reinterpret_cast<const float4*>(
                            src + ((size_t)((c0 + j) / 4) * RM + 32 * q + lane) * 16);
                        v[j] = __float_as_uint(__uint_as_float(v[j]) + f.x);
                        v[j + 1] = __float_as_uint(__uint_as_float(v[j + 1]) + f.y);
                        v[j + 2] = __float_as_uint(__uint_as_float(v[j + 2]) + f.z);
                        v[j + 3] = __float_as_uint(__uint_as_float(v[j + 3]) + f.w);
                    }
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float4 c = cst[buf * RN + c0 + j];
                    // TMEM columns past the tile's hidden units are undefined: clamp them to 0
                    const float a = (c0 + j < nh ? __uint_as_float(v[j]) : 0.f) + c.x;
                    const float sv = a * __fdividef(1.f, 1.f + __expf(-a));
                    part0 = fmaf(sv, c.y, part0);
                    part1 = fmaf(sv, c.z, part1);
                    part2 = fmaf(sv, c.w, part2);
                }
            }
            const float part[3] = {part0, part1, part2};
            tc_fence_before();
            __syncwarp();
            if (q == 0) TR(201);
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
            if (t < p.T) {
#pragma unroll
                for (int k = 0; k < kFastSlices - 1; ++k)
                    if (k < p.nr) p.s_part[((int64_t)nt * p.T + t) * p.nr + k] = part[k];
            }
            // last hidden tile of token tile mt: scores and slice masks for its tokens
            __threadfence();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (q == 0 && lane == 0) s_last = atomicAdd(&p.cnt[mt], 1) == p.n_nt - 1;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (s_last) {
                __threadfence();
                int mk = 2 * kMaxBuckets;  // no token
                if (t < p.T) {
                    int m = 1;
                    for (int k = 0; k < p.nr; ++k) {
                        float sc = 0.f;
                        for (int j = 0; j < p.n_nt; ++j) sc += __ldcg(p.s_part + ((int64_t)j * p.T + t) * p.nr + k);
                        sc += __ldg(p.b2 + k);
                        if (p.scores_out) p.scores_out[t * p.nr + k] = sc;
                        if ((sc - p.delta) > 0.f) m |= 1 << (k + 1);
                    }
                    p.masks[t] = (uint8_t)m;
                    if (p.masks_out) p.masks_out[t] = (uint8_t)m;
                    mk = m;
                }
                if (q == 0 && lane == 0) p.cnt[mt] = 0;
                if (p.hist) {  // bucket sizes for the gather (which lays the buckets out)
                    const unsigned peers = __match_any_sync(0xffffffffu, mk);
                    if (mk < 2 * kMaxBuckets && lane == __ffs(peers) - 1) atomicAdd(&p.hist[mk], __popc(peers));
                }
            }
        }
    }
    TR(202 + (warp == kRWarpMma) + 2 * (warp == kRWarpTma));
    tc_fence_before();
    __syncthreads();
    if (p.csplit > 1) cluster_sync();  // no CTA leaves while a peer may still address its shared memory
    if (warp == kRWarpMma) tmem_dealloc(tmem, 512);
    TR(205);
    if (p.trace && threadIdx.x == 0) {  // per-CTA wall marks (ns) + SM id
        unsigned long long g_end;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_end));
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        p.trace[4096 + 4 * blockIdx.x] = g_start;
        p.trace[4096 + 4 * blockIdx.x + 1] = g_end;
        p.trace[4096 + 4 * blockIdx.x + 2] = smid;
        p.trace[4096 + 4 * blockIdx.x + 3] = (unsigned long long)(clock64() - t_start);
    }
}

// CTA-pair router tile (cta_group::2): M = 256 tokens (128 per CTA, each CTA TMA-loads its own X
// rows) x N = PN hidden units (each CTA TMA-loads PN/2 rows of w1, the tensor cores exchange the
// halves), fp32 D in each CTA's TMEM for its own 128 tokens.  Per k-block a CTA takes in 16 KiB of X
// + PN/4 KiB of w1 for 128 x PN outputs, against 32 KiB for 128 x 128 in the 1-CTA kernel, whose
// tiles sit at the measured ~71 B/cycle/SM L2->SMEM limit.  The leader's MMA thread issues for the
// pair; both CTAs run the same fused SiLU.w2 / gate / histogram epilogue on their own tokens.
// 8 epilogue warps (two per TMEM lane quarter, each taking half of the tile's hidden units), TMA, MMA
// two TMA warps (X and w1): one thread issues a TMA about every 250-430 cycles, the pair's MMAs for a
// k-block take 256 (N = 128)
constexpr int k2WarpTma = 8, k2WarpMma = 9, k2WarpTmaB = 10, k2Threads = 352;
template <int PN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(k2Threads, 1)
    router_tc2_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                      const RParams p) {
    constexpr int kBB = PN / 2 * kKBlock * 2;  // w1 half per stage
    constexpr int kStg = kAB + kBB;
    constexpr int NS = (RS * 2 * kAB) / kStg;   // stages in the same ring footprint
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RS * 2 * kAB);
    uint64_t* full = bars;                 // [NS] leader: both CTAs' bytes of the stage
    uint64_t* empty = bars + NS;           // [NS] each CTA: the pair's MMAs are done with the stage
    uint64_t* acc_full = bars + 2 * NS;    // [2] each CTA
    uint64_t* acc_empty = acc_full + 2;    // [2] leader: 8 epilogue warps x 2 CTAs drained the buffer
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    float4* cst = reinterpret_cast<float4*>(smem + RS * 2 * kAB + 1024);  // [2][PN] {b1, w2[0..2]}
    const int warp = warp_idx_uniform(), lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    __shared__ int s_last;
    __shared__ float s_pp[RM][3];  // the second column half's partial scores per token
    unsigned long long g_start = 0, c_start = clock64();
    if (p.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_start));
    auto MARK = [&](int i) {  // debug: per-CTA cycle marks [4096 + 8*cta + i]
        if (p.trace && (threadIdx.x % 32) == 0 && blockIdx.x < 148)
            p.trace[4096 + 8 * blockIdx.x + i] = (unsigned long long)(clock64() - c_start);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 16);
        }
        fence_barrier_init();
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
    }
    if (warp == k2WarpMma) tmem_alloc_2sm(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    if (*tmem_slot != 0) __trap();
    pdl_wait();     // PDL: X (possibly the previous kernel's output) and every write wait for it
    pdl_trigger();  // the gather may launch and start loading its rows
    if (warp == 0) MARK(1);  // prologue done
    constexpr uint32_t tmem = 0;
    const int n_mp = (p.n_mt + 1) / 2;
    const int total = n_mp * p.n_nt;
    const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
    auto tile_of = [&](int pair, int& mp, int& nt) {
        mp = pair % n_mp;
        nt = pair / n_mp;
    };
    if (warp == k2WarpTma || warp == k2WarpTmaB) {
        // X rows (warp k2WarpTma, which also posts the stage's expected bytes) and w1 rows (k2WarpTmaB)
        // of every stage; a w1 box may land before the expect_tx (the tx-count goes transiently negative)
        const bool xw = warp == k2WarpTma;
        const uint32_t full_leader = mapa_shared(smem_u32(full), 0);
        uint32_t it = 0;
        for (int pair = cid; pair < total; pair += ncl) {
            int mp, nt;
            tile_of(pair, mp, nt);
            for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
                const int s = it % NS;
                mbar_wait(&empty[s], ((it / NS) & 1) ^ 1);
                if (elect_one_sync()) {
                    uint8_t* a = smem + s * kStg;
                    if (xw) {
                        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kStg);
                        tma_load_2d_2sm(a, &tmap_a, full_leader + s * 8, kb * kKBlock, (2 * mp + (int)rank) * RM);
                    } else {
                        tma_load_2d_2sm(a + kAB, &tmap_b, full_leader + s * 8, kb * kKBlock,
                                        nt * PN + (int)rank * (PN / 2));
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == k2WarpMma) {
        // one thread, CTA-scope stage waits, operands in uniform registers (a whole-warp loop with a
        // cluster-scope acquire per k-block cost ~700 cycles per k-block, 2.7x the N = 128 MMAs)
        if (rank == 0 && elect_one_sync()) {
            uint32_t it = 0, tc = 0;
            constexpr uint32_t idesc = idesc_f16(2 * RM, PN, 1);
            const uint64_t desc0 = sdesc_sw128(smem_u32(smem));
            for (int pair = cid; pair < total; pair += ncl, ++tc) {
                const int buf = tc & 1;
                mbar_wait_cluster(&acc_empty[buf], ((tc >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
                    const uint32_t s = it % NS;
                    mbar_wait(&full[s], (it / NS) & 1);
                    if (p.trace && blockIdx.x == 0 && tc == 0 && kb < 64)
                        p.trace[8192 + kb] = (unsigned long long)(clock64() - c_start);
                    tc_fence_after();
                    const uint64_t adesc = desc0 + (uint64_t)((s * kStg) >> 4), bdesc = adesc + (uint64_t)(kAB >> 4);
#pragma unroll
                    for (int j = 0; j < kKBlock / 16; ++j)
                        mma_ss_f16_2sm(tmem + buf * PN, adesc + (uint64_t)(j * 2), bdesc + (uint64_t)(j * 2), idesc,
                                       (kb | j) != 0 ? 1u : 0u);
                    mma_commit_2sm_mc(&empty[s], (uint16_t)0x3);
                }
                mma_commit_2sm_mc(&acc_full[buf], (uint16_t)0x3);
            }
        }
        __syncwarp();
    } else {
        const int q = warp % 4, half = warp / 4;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        const uint32_t acc_empty_leader = mapa_shared(smem_u32(acc_empty), 0);
        uint32_t tc = 0;
        for (int pair = cid; pair < total; pair += ncl, ++tc) {
            int mp, nt;
            tile_of(pair, mp, nt);
            const int mt = 2 * mp + (int)rank;
            const int buf = tc & 1;
            const int64_t t = (int64_t)mt * RM + 32 * q + lane;
            const int64_t h0 = (int64_t)nt * PN;
            for (int et = threadIdx.x; et < PN; et += 256) {
                float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
                const int64_t hj = h0 + et;
                c.x = __ldg(p.b1 + hj);
                c.y = __ldg(p.w2 + hj * p.nr);
                if (p.nr > 1) c.z = __ldg(p.w2 + hj * p.nr + 1);
                if (p.nr > 2) c.w = __ldg(p.w2 + hj * p.nr + 2);
                cst[buf * PN + et] = c;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            mbar_wait(&acc_full[buf], (tc >> 1) & 1);
            if (warp == 0 && tc == 0) MARK(2);  // first tile's accumulator complete
            tc_fence_after();
            float part0 = 0.f, part1 = 0.f, part2 = 0.f;
            for (int c0 = half * (PN / 2); c0 < (half + 1) * (PN / 2); c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + lane_base + buf * PN + c0, v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float4 c = cst[buf * PN + c0 + j];
                    const float a = __uint_as_float(v[j]) + c.x;
                    const float sv = a * __fdividef(1.f, 1.f + __expf(-a));
                    part0 = fmaf(sv, c.y, part0);
                    part1 = fmaf(sv, c.z, part1);
                    part2 = fmaf(sv, c.w, part2);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0)
                    mbar_arrive(&acc_empty[buf]);
                else
                    mbar_arrive_cluster(acc_empty_leader + buf * 8);
            }
            // the two column halves' partial scores, summed in a fixed order by the first half
            if (half == 1) {
                s_pp[32 * q + lane][0] = part0;
                s_pp[32 * q + lane][1] = part1;
                s_pp[32 * q + lane][2] = part2;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (half == 1) continue;
            const float part[3] = {part0 + s_pp[32 * q + lane][0], part1 + s_pp[32 * q + lane][1],
                                   part2 + s_pp[32 * q + lane][2]};
            if (t < p.T) {
#pragma unroll
                for (int k = 0; k < kFastSlices - 1; ++k)
                    if (k < p.nr) p.s_part[((int64_t)nt * p.T + t) * p.nr + k] = part[k];
            }
            // last hidden tile of token tile mt: scores and slice masks for its tokens
            __threadfence();
            asm volatile("bar.sync 2, 128;" ::: "memory");
            if (q == 0 && lane == 0) s_last = (int64_t)mt * RM < p.T && atomicAdd(&p.cnt[mt], 1) == p.n_nt - 1;
            asm volatile("bar.sync 2, 128;" ::: "memory");
            if (s_last) {
                __threadfence();
                int mk = 2 * kMaxBuckets;  // no token
                if (t < p.T) {
                    int m = 1;
                    for (int k = 0; k < p.nr; ++k) {
                        float sc = 0.f;
                        for (int j = 0; j < p.n_nt; ++j) sc += __ldcg(p.s_part + ((int64_t)j * p.T + t) * p.nr + k);
                        sc += __ldg(p.b2 + k);
                        if (p.scores_out) p.scores_out[t * p.nr + k] = sc;
                        if ((sc - p.delta) > 0.f) m |= 1 << (k + 1);
                    }
                    p.masks[t] = (uint8_t)m;
                    if (p.masks_out) p.masks_out[t] = (uint8_t)m;
                    mk = m;
                }
                if (q == 0 && lane == 0) p.cnt[mt] = 0;
                if (p.hist) {
                    const unsigned peers = __match_any_sync(0xffffffffu, mk);
                    if (mk < 2 * kMaxBuckets && lane == __ffs(peers) - 1) atomicAdd(&p.hist[mk], __popc(peers));
                }
            }
        }
    }
    if (warp == 0) MARK(3);  // epilogue done
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the peer's remote arrivals and TMEM use are over before either CTA releases it
    if (warp == k2WarpMma) tmem_dealloc_2sm(tmem, 512);
    if (p.trace && threadIdx.x == 0 && blockIdx.x < 148) {
        unsigned long long g_end;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_end));
        p.trace[4096 + 8 * blockIdx.x + 4] = g_start;
        p.trace[4096 + 8 * blockIdx.x + 5] = g_end;
        p.trace[4096 + 8 * blockIdx.x + 6] = (unsigned long long)(clock64() - c_start);
    }
}

// split-K finish: H = sum_ks hpart (fixed order) -> silu(H + b1) . w2 -> s_part[nt][t][k]
__global__ void __launch_bounds__(RN) router_reduce_kernel(const float* __restrict__ hpart, int nsplit, int64_t T,
                                                           int64_t h, int64_t h_pad, const float* __restrict__ b1,
                                                           const float* __restrict__ w2, int nr,
                                                           float* __restrict__ s_part) {
    __shared__ float red[kFastSlices - 1][RN];
    const int64_t t = blockIdx.x;
    const int nt = blockIdx.y;
    const int64_t j = (int64_t)nt * RN + threadIdx.x;
    float sv = 0.f;
    if (j < h) {
        float H = 0.f;
        for (int ks = 0; ks < nsplit; ++ks) H += hpart[((int64_t)ks * T + t) * h_pad + j];
        const float a = H + b1[j];
        sv = a * __fdividef(1.f, 1.f + __expf(-a));
    }
    for (int k = 0; k < nr; ++k) red[k][threadIdx.x] = j < h ? sv * w2[j * nr + k] : 0.f;
    __syncthreads();
    for (int w = RN / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int k = 0; k < nr; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < nr; ++k) s_part[((int64_t)nt * T + t) * nr + k] = red[k][0];
}


}  // namespace

bool router_tc_supported(const mobi_layer* L, const void* x) {
    return !L->generic && (L->in % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
}

// Launch with programmatic stream serialization (PDL) and, when cluster > 0, a runtime cluster size.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              int cluster, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int n = 0;
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n++].val.programmaticStreamSerializationAllowed = 1;
    if (cluster > 0) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = (unsigned)cluster;
        at[n].val.clusterDim.y = 1;
        at[n++].val.clusterDim.z = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// development switch (MOBI_ROUTER_PAIR): 0 = never use the CTA-pair router, 2 = N = 256 tiles whenever h allows
int g_router_pair = [] {
    const char* e = std::getenv("MOBI_ROUTER_PAIR");
    return e ? std::atoi(e) : 1;
}();
constexpr int r2_smem(int pn) { return RS * 2 * kAB + 1024 + 1024 + 2 * pn * 16; }

// development switch (MOBI_ROUTER_CSPLIT): 0 = no cluster split-K in the prefill router, 1 = by tile count
int g_router_csplit = [] {
    const char* e = std::getenv("MOBI_ROUTER_CSPLIT");
    return e ? std::atoi(e) : 1;
}();

int launch_router_tc(mobi_layer* L, const __nv_bfloat16* x, int64_t T, float delta, float* scores_out,
                     uint8_t* masks_out, bool* masks_ready, cudaStream_t st, unsigned long long* trace,
                     bool fuse_bucket) {
    {
        MOBI_TRY(func_attr_once(router_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRSmem));
    }
    if (!L->tmap_w1) {
        L->tmap_w1 = new CUtensorMap;
        int rc = make_tmap_2d(L->tmap_w1, L->w1t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, L->h_pad, L->in_pad, RN);
        if (rc) {
            delete L->tmap_w1;
            L->tmap_w1 = nullptr;
            return rc;
        }
    }
    CUtensorMap tmap_x;
    int rc = make_tmap_2d(&tmap_x, x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, T, L->in, RM);
    if (rc) return rc;
    RParams p;
    p.T = T;
    p.h = L->h;
    p.h_pad = L->h_pad;
    p.hpart = L->hpart;
    p.kblocks = (int)L->kblocks;
    p.n_mt = (int)cdiv(T, RM);
    p.n_nt = (int)cdiv(L->h, RN);
    p.nr = L->nr;
    p.b1 = L->b1;
    p.w2 = L->w2;
    p.s_part = L->s_part;
    p.trace = trace;
    p.cnt = L->rt_cnt;
    p.b2 = L->b2;
    p.delta = delta;
    p.masks = L->masks;
    p.masks_out = masks_out;
    p.scores_out = scores_out;
    p.hist = fuse_bucket ? L->bk_hist : nullptr;
    L->htiles = p.n_nt;
    // split K when the tile grid cannot fill the SMs (decode-size T)
    p.nsplit = 1;
    p.csplit = 1;
    // CTA-pair tiles when they alone fill the SMs (fewer w1 bytes per SM per flop, see the kernel).
    // The variant (and the cluster K-split below) is chosen from the plan size Tp -- the whole batch
    // when mobi_forward_host runs it in chunks -- so every chunk sums each token's score in the same
    // order as the whole-batch call.
    const int64_t Tp = std::max(T, L->plan_T);
    const int n_mp = (int)cdiv(T, 2 * RM);
    const int n_mp_plan = (int)cdiv(Tp, 2 * RM);
    int pn = 0;
    if (g_router_pair && Tp > 64 && L->h % 256 == 0 &&
        (n_mp_plan * (int)(L->h / 256) * 2 >= L->n_sm || g_router_pair == 2))
        pn = 256;
    else if (g_router_pair && Tp > 64 && L->h % 128 == 0 && n_mp_plan * (int)(L->h / 128) * 2 >= L->n_sm * 3 / 4)
        pn = 128;
    if (pn == 128 && !L->tmap_w1_64) {
        L->tmap_w1_64 = new CUtensorMap;
        int rc2 = make_tmap_2d(L->tmap_w1_64, L->w1t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, L->h_pad, L->in_pad, 64);
        if (rc2) {
            delete L->tmap_w1_64;
            L->tmap_w1_64 = nullptr;
            return rc2;
        }
    }
    if (pn) {
        L->plan[0] = pn == 256 ? MOBI_K_ROUTER_PAIR256 : MOBI_K_ROUTER_PAIR128;
        p.n_nt = (int)(L->h / pn);
        L->htiles = p.n_nt;
        if (masks_ready) *masks_ready = true;
        const int grid = 2 * std::min(n_mp * p.n_nt, L->n_sm / 2);
        if (pn == 256) {
            {
                MOBI_TRY(func_attr_once(router_tc2_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               r2_smem(256)));
            }
            MOBI_CUDA(launch_pdl(router_tc2_kernel<256>, dim3(grid), dim3(k2Threads), r2_smem(256), st, 0, tmap_x,
                                 *L->tmap_w1, p));
        } else {
            {
                MOBI_TRY(func_attr_once(router_tc2_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               r2_smem(128)));
            }
            MOBI_CUDA(launch_pdl(router_tc2_kernel<128>, dim3(grid), dim3(k2Threads), r2_smem(128), st, 0, tmap_x,
                                 *L->tmap_w1_64, p));
        }
        MOBI_LAUNCH_CHECK();
        ++L->last_launches;
        return MOBI_OK;
    }
    const int tiles = p.n_mt * p.n_nt;
    const int tiles_plan = (int)cdiv(Tp, RM) * p.n_nt;
    if (g_router_csplit == 2 && p.kblocks >= 8) {  // experiment: fixed 2-way split at every T
        p.csplit = 2;
        p.nsplit = 2;
    } else if (g_router_csplit == 1 && 2 * tiles_plan <= L->n_sm && p.kblocks >= 8) {
        // too few tiles to fill the SMs: split K over a cluster of 2-3 CTAs per tile (DSMEM reduction
        // into rank 0, which keeps the fused gate/histogram epilogue).  The split depends on the tile
        // count only, so outputs are identical for every T of the same regime.
        p.csplit = std::min(kMaxCsplit, std::min(3, L->n_sm / tiles_plan));
        p.nsplit = p.csplit;
    } else if (Tp <= 64 && L->hpart) {  // small K: global split-K partials + a reduce kernel
        p.nsplit = std::max(1, std::min(16, L->n_sm / tiles));
    }
    p.kb_per = (p.kblocks + p.nsplit - 1) / p.nsplit;
    p.nsplit = (p.kblocks + p.kb_per - 1) / p.kb_per;  // no empty splits
    if (p.csplit > 1) p.csplit = p.nsplit;
    const int total = tiles * p.nsplit;
    const bool clus = p.csplit > 1;
    if (masks_ready) *masks_ready = p.nsplit == 1 || clus;
    if (p.nsplit != 1 && !clus) p.hist = nullptr;
    L->plan[0] = clus ? MOBI_K_ROUTER_TC_CLUSTER : (p.nsplit > 1 ? MOBI_K_ROUTER_TC_SPLITK : MOBI_K_ROUTER_TC);
    if (clus) {
        MOBI_CUDA(launch_pdl(router_tc_kernel, dim3((unsigned)total), dim3(kRThreads), (size_t)kRSmem, st, p.csplit,
                             tmap_x, *L->tmap_w1, p));
        ++L->last_launches;
        return MOBI_OK;
    }
    const int grid = std::min(total, L->n_sm);
    MOBI_CUDA(launch_pdl(router_tc_kernel, dim3(grid), dim3(kRThreads), (size_t)kRSmem, st, 0, tmap_x, *L->tmap_w1, p));
    ++L->last_launches;
    if (p.nsplit > 1) {
        router_reduce_kernel<<<dim3((unsigned)T, (unsigned)p.n_nt), RN, 0, st>>>(L->hpart, p.nsplit, T, L->h, L->h_pad,
                                                                                L->b1, L->w2, L->nr, L->s_part);
        MOBI_LAUNCH_CHECK();
        ++L->last_launches;
    }
    return MOBI_OK;
}

}  // namespace mobi
