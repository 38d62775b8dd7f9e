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
//   warp 0      TMA producer: X_perm tile [256 tokens x 64 k] fp16, 128-byte swizzle -> smem stage
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-17  dequantizers: each thread owns one weight row (= one TMEM lane) and 16 k of the
//               64-k block; coalesced 16-byte code loads (3 k-blocks in flight) -> fp16 W_m ->
//               tcgen05.st into the A stage in TMEM (A operand never touches shared memory)
//   warps 18-21 epilogue: tcgen05.ld the fp32 accumulator, x 2^e row scale, bf16, scatter
//               Y[perm[i], r] (the un-permute, bitplane.hpp:171-172, fused)
// MMA: M=128 weight rows (TMEM lanes), N=tile tokens (<=256, multiple of 16), K=16 per
// instruction, D fp32 in TMEM columns [0,256); A stages at columns 256 + 32*s.
#include "mobi_internal.cuh"
#include "sm100.cuh"

namespace mobi {
namespace {

using namespace sm100;

constexpr int NSTAGE = 4;
constexpr int kDqWarps = 16;                       // 4 per TMEM lane quarter
constexpr int kThreads = 32 * (2 + kDqWarps + 4);  // TMA, MMA, dequant, epilogue
constexpr int kStageBytes = kTokTile * kKBlock * 2;  // 32 KiB
constexpr int kAccCols = 256;
constexpr int kACol0 = 256;
constexpr int kSmemBytes = NSTAGE * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

struct Params {
    const uint8_t* codes8;
    const float* gscale;
    const float* gsz;
    MaskTable mt;
    int64_t out, G, gs, kblocks;
    int single_group;
    int n_row_tiles;
    const float* escale;
    const int32_t* perm;
    const TokTile* tiles;
    const int32_t* meta;
    __nv_bfloat16* y;
    unsigned long long* trace;
};

// TRACE=true: clock64 accounting of each role's barrier waits (debug hook impl 2), written to
// p.trace[cta][0..15]: 0 tma wait empty | 1 mma wait acc_empty | 2 mma wait full_b | 3 mma wait
// full_a | 4 mma loop | 5 dequant(w2) wait empty | 6 dequant(w2) loop | 7 epi(w18) wait acc_full |
// 8 epi(w18) loop | 9 tiles
template <bool TRACE>
__global__ void __launch_bounds__(kThreads, 1) mobi_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x,
                                                                   const Params p) {
    long long tr[4] = {0, 0, 0, 0};
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
    uint64_t* full_a = bars + NSTAGE;         // [NSTAGE] A stage written to TMEM (8 warps)
    uint64_t* empty = bars + 2 * NSTAGE;      // [NSTAGE] MMAs reading the stage completed
    uint64_t* acc_full = bars + 3 * NSTAGE;   // accumulator ready for the epilogue
    uint64_t* acc_empty = acc_full + 1;       // epilogue drained the accumulator (4 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full_b[s], 1);
            mbar_init(&full_a[s], kDqWarps);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 4);
        fence_barrier_init();
        prefetch_tmap(&tmap_x);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int n_tok_tiles = p.meta[0];
    const int total = n_tok_tiles * p.n_row_tiles;
    const int kb_n = (int)p.kblocks;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
            const TokTile tt = p.tiles[tile / p.n_row_tiles];
            for (int kb = 0; kb < kb_n; ++kb, ++it) {
                const int s = it % NSTAGE;
                const uint32_t ph = (it / NSTAGE) & 1;
                TW(0, mbar_wait(&empty[s], ph ^ 1));
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full_b[s], kStageBytes);
                    tma_load_2d(stage_b + s * kStageBytes, &tmap_x, &full_b[s], kb * kKBlock, tt.row0);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        uint32_t it = 0, tc = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
            const TokTile tt = p.tiles[tile / p.n_row_tiles];
            const uint32_t n_mma = (uint32_t)round_up(tt.n, 16);
            const uint32_t idesc = idesc_f16(128, n_mma, 0);
            TW(0, mbar_wait(acc_empty, (tc & 1) ^ 1));
            tc_fence_after();
            for (int kb = 0; kb < kb_n; ++kb, ++it) {
                const int s = it % NSTAGE;
                const uint32_t ph = (it / NSTAGE) & 1;
                TW(1, mbar_wait(&full_b[s], ph));
                TW(2, mbar_wait(&full_a[s], ph));
                tc_fence_after();
                if (lane == 0) {
                    const uint64_t bdesc = sdesc_sw128(smem_u32(stage_b + s * kStageBytes));
#pragma unroll
                    for (int j = 0; j < kKBlock / 16; ++j) {
                        mma_ts_f16(tmem, tmem + kACol0 + s * 32 + j * 8, bdesc + (uint64_t)(j * 2), idesc,
                                   (kb | j) != 0);
                    }
                    mma_commit(&empty[s]);
                    if (kb == kb_n - 1) mma_commit(acc_full);
                }
                __syncwarp();
            }
        }
    } else if (warp < 2 + kDqWarps) {
        // ---------------- dequantizers ----------------
        // warp -> (TMEM lane quarter q, 16-code chunk j of the 64-k block); 4 warps per quarter
        const int q = warp % 4;
        const int j = (warp - 2) / 4;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
            const TokTile tt = p.tiles[tile / p.n_row_tiles];
            const int rt = tile % p.n_row_tiles;
            const int64_t R = (int64_t)rt * kRowTile + 32 * q + lane;
            const bool rv = R < p.out;
            const uint32_t mw = p.mt.maskword[tt.mask];
            const float kc = p.mt.kc[tt.mask];
            const uint8_t* cbase = p.codes8 + (int64_t)rt * p.kblocks * kBlockBytes + (j * kRowTile + 32 * q + lane) * 16;
            const float* srow = p.gscale + (rv ? R : 0) * p.G;
            const float* zrow = p.gsz + (rv ? R : 0) * p.G;
            // codes ring, 3 k-blocks ahead
            uint4 ca = *reinterpret_cast<const uint4*>(cbase);
            uint4 cb = kb_n > 1 ? *reinterpret_cast<const uint4*>(cbase + kBlockBytes) : ca;
            uint4 cc = kb_n > 2 ? *reinterpret_cast<const uint4*>(cbase + 2 * kBlockBytes) : ca;
            // group tracking without division: k = kb*64 + 16j
            int g = 0, kin = 16 * j;
            if (!p.single_group)
                while (kin >= p.gs) kin -= (int)p.gs, ++g;
            __half2 S2, C2;
            auto group_consts = [&](int gg) {
                const float sc = rv ? __ldg(srow + gg) : 0.f;
                const float sz = rv ? __ldg(zrow + gg) : 0.f;
                S2 = __float2half2_rn(sc * p.mt.inv_2p);
                C2 = __float2half2_rn(fmaf(sc, kc, -sz));
            };
            group_consts(g);
            uint32_t v[8];
            {
                const uint32_t* w = reinterpret_cast<const uint32_t*>(&ca);
#pragma unroll
                for (int u = 0; u < 4; ++u) dequant4(w[u], mw, S2, C2, v[2 * u], v[2 * u + 1]);
            }
            for (int kb = 0; kb < kb_n; ++kb, ++it) {
                const int s = it % NSTAGE;
                const uint32_t ph = (it / NSTAGE) & 1;
                TW(0, mbar_wait(&empty[s], ph ^ 1));
                tc_fence_after();
                tmem_st8(tmem + lane_base + kACol0 + s * 32 + j * 8, v);
                // overlap the TMEM store with the next k-block's loads and dequantization
                ca = cb;
                cb = cc;
                if (kb + 3 < kb_n) cc = *reinterpret_cast<const uint4*>(cbase + (int64_t)(kb + 3) * kBlockBytes);
                uint32_t vn[8];
                if (kb + 1 < kb_n) {
                    if (!p.single_group) {
                        kin += kKBlock;
                        bool ch = false;
                        while (kin >= p.gs) kin -= (int)p.gs, ++g, ch = true;
                        if (ch) group_consts(g);
                    }
                    const uint32_t* w = reinterpret_cast<const uint32_t*>(&ca);
#pragma unroll
                    for (int u = 0; u < 4; ++u) dequant4(w[u], mw, S2, C2, vn[2 * u], vn[2 * u + 1]);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full_a[s]);
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = vn[u];
            }
        }
    } else {
        // ---------------- epilogue ----------------
        const int q = warp % 4;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        uint32_t tc = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
            const TokTile tt = p.tiles[tile / p.n_row_tiles];
            const int rt = tile % p.n_row_tiles;
            const int64_t R = (int64_t)rt * kRowTile + 32 * q + lane;
            const bool rv = R < p.out;
            TW(0, mbar_wait(acc_full, tc & 1));
            tc_fence_after();
            for (int c0 = 0; c0 < tt.n; c0 += 32) {
                // lane j fetches the destination row and scale of token c0+j; issued before the
                // TMEM load so their latency overlaps it, then broadcast with shuffles
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
                    if (rv && src >= 0)
                        p.y[(int64_t)src * p.out + R] = __float2bfloat16_rn(__uint_as_float(v[j]) * es);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
        }
    }
    if (TRACE && lane == 0) {
        unsigned long long* o = p.trace + blockIdx.x * 16;
        const long long tot = clock64() - tstart;
        if (warp == 0) o[0] = tr[0];
        if (warp == 1) { o[1] = tr[0]; o[2] = tr[1]; o[3] = tr[2]; o[4] = tot; }
        if (warp == 2) { o[5] = tr[0]; o[6] = tot; }
        if (warp == 2 + kDqWarps) { o[7] = tr[0]; o[8] = tot; }
        if (warp == 0) o[9] = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
    }
#undef TW
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
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

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
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
    static bool attr = false;
    if (!attr) {
        MOBI_CUDA(cudaFuncSetAttribute(mobi_gemm_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBytes));
        MOBI_CUDA(cudaFuncSetAttribute(mobi_gemm_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBytes));
        attr = true;
    }
    if (!L->tmap_x) {
        L->tmap_x = new CUtensorMap;
        int rc = make_tmap_2d(L->tmap_x, L->xperm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, L->tpad_max, L->in_pad, kTokTile);
        if (rc) {
            delete L->tmap_x;
            L->tmap_x = nullptr;
            return rc;
        }
    }
    Params p;
    p.codes8 = L->codes8;
    p.gscale = L->gscale;
    p.gsz = L->gsz;
    p.mt = L->mtab;
    p.out = L->out;
    p.G = L->G;
    p.gs = L->gs;
    p.kblocks = L->kblocks;
    p.single_group = L->single_group;
    p.n_row_tiles = (int)(L->out_pad / kRowTile);
    p.escale = L->escale;
    p.perm = L->perm;
    p.tiles = L->tiles;
    p.meta = L->meta;
    p.y = y;
    const int64_t max_total = (int64_t)p.n_row_tiles * L->max_tiles;
    const int grid = (int)std::min<int64_t>(sm_count(), max_total);
    p.trace = trace;
    if (trace)
        mobi_gemm_tc_kernel<true><<<grid, kThreads, kSmemBytes, st>>>(*L->tmap_x, p);
    else
        mobi_gemm_tc_kernel<false><<<grid, kThreads, kSmemBytes, st>>>(*L->tmap_x, p);
    MOBI_LAUNCH_CHECK();
    ++L->last_launches;
    return MOBI_OK;
}

}  // namespace mobi
