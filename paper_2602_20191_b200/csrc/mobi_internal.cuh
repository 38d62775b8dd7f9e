// mobi_internal.cuh -- device layout, workspace and launcher declarations shared by the
// MoBi-linear kernels (sm_100a).  See DESIGN.md for the layouts and their rationale.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/mobi_b200.h"

namespace mobi {

// ---------------------------------------------------------------------------------------------
// Geometry of the device weight layout ("tiled merged codes").
//   kRowTile rows x kKBlock input columns form one 8 KiB block; inside a block the bytes are
//   ordered [half h (2)][chunk c (2)][row r (128)][16 codes], so the 32 lanes of a warp that
//   own 32 consecutive rows read 512 contiguous bytes per 16-byte load (coalesced), and each
//   thread receives the 32 consecutive K-codes of its row that it dequantizes into one TMEM
//   lane.  Rows are padded to kRowTile, K to kKBlock (padding codes are 0; padded X columns
//   are 0, so padded weights never contribute).
// ---------------------------------------------------------------------------------------------
constexpr int kRowTile = 128;
constexpr int kKBlock = 64;
constexpr int kBlockBytes = kRowTile * kKBlock;  // 8192
constexpr int kBucketAlign = 16;                 // bucket starts in the permuted token order
constexpr int kTokTile = 256;                    // tokens per GEMM tile (MMA N <= 256)
constexpr int kFastSlices = 4;  // uniform-width layers up to 4 slices take the tcgen05 / slice-plane paths
constexpr int kMaxBuckets = 1 << (kFastSlices - 1);  // 8 masks (slice-1 bit always set)
constexpr int kDecMaxT = 32;                     // decode path (decode.cu): up to 32 tokens per call

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return cdiv(a, b) * b; }

// byte offset of code (row R, col k) in the tiled layout
__host__ __device__ inline int64_t code_offset(int64_t R, int64_t k, int64_t kblocks) {
    int64_t rt = R / kRowTile, r = R % kRowTile;
    int64_t kb = k / kKBlock, kk = k % kKBlock;
    int64_t h = kk / 32, c = (kk % 32) / 16, b = kk % 16;
    return (rt * kblocks + kb) * kBlockBytes + ((h * 2 + c) * kRowTile + r) * 16 + b;
}

// One GEMM tile of the token dimension: a run of <= kTokTile permuted rows of one bucket.
struct TokTile {
    int32_t row0;   // first permuted row
    int32_t n;      // valid rows (1..kTokTile)
    int32_t mask;   // bucket slice mask (bit0 always set)
    int32_t pad;
};

// Tile record read from global memory, broadcast from lane 0 so the compiler can prove the
// fields warp-uniform (keeps TMA / tcgen05 operands derived from them in uniform registers).
__device__ __forceinline__ TokTile uniform_tile(const TokTile& t) {
    TokTile u;
    u.row0 = __shfl_sync(0xffffffffu, t.row0, 0);
    u.n = __shfl_sync(0xffffffffu, t.n, 0);
    u.mask = __shfl_sync(0xffffffffu, t.mask, 0);
    u.pad = 0;
    return u;
}

// Where a layer's Y [T, out] goes: n_dst buffers (device pointers, peer-mapped for the fused
// all-gather of column-parallel shards), row stride ldy, this layer's first output column col0.
struct OutDesc {
    __nv_bfloat16* dst[MOBI_MAX_DST];
    int32_t n_dst;
    int64_t ldy;
    int64_t col0;
};

// Per-mask dequant constants (uniform b-bit slices): W = S*INT_m + C with
//   INT_m = merged & maskbyte[m],  S = s / 2^P,  C = s*K[m]/2^(P+1) - s*z
struct MaskTable {
    uint32_t maskword[kMaxBuckets * 2];  // maskbyte replicated x4, indexed by mask value (<16)
    float kc[kMaxBuckets * 2];           // K[m] / 2^(P+1)
    float inv_2p;                        // 1 / 2^P
};

}  // namespace mobi

namespace mobi {
// Bit layout of the merged code INT = ((c1 << b2 | c2) << b3 | c3) ... (slicer.hpp:150-161) for any
// widths: slice e (0-based) occupies bits [off[e], off[e] + b[e]).
struct SliceLayout {
    int E;
    int b[MOBI_MAX_SLICES];
    int off[MOBI_MAX_SLICES];
};
}  // namespace mobi

struct mobi_layer {
    int device = 0;
    int n_sm = 148;                          // SMs of `device` (grid sizing)
    int64_t out = 0, in = 0, gs = 0, G = 0;  // G = groups per row
    int32_t E = 0, b = 0;                    // slices, bits per slice (0: non-uniform widths)
    bool generic = false;                    // non-uniform widths or E > kFastSlices: per-slice CUDA-core path
    mobi::SliceLayout sl{};
    int32_t* hist256 = nullptr;              // generic layers: per-mask counts scratch (mobi_route)
    int32_t nr = 0;                          // routed slices = E-1
    int64_t h = 0;                           // router hidden
    int64_t out_pad = 0, in_pad = 0, kblocks = 0, h_pad = 0;
    int64_t group_shift = -1;                // log2(gs) when gs is a power of two >= 32
    bool single_group = false;               // gs >= in: one group per row

    // device weights
    uint8_t* codes8 = nullptr;        // tiled merged codes [out_pad/128][kblocks][8192]
    uint8_t* dplanes = nullptr;       // decode slice planes [E][out_pad/32][kblocks][32 lanes][16 B] (2-bit slices)
    float2* gconst = nullptr;         // [G][out_pad] (s, s*z) per group: coalesced across rows
    __nv_bfloat16* w1t = nullptr;     // [h_pad][in_pad] bf16, K-major (router B operand)
    float* b1 = nullptr;              // [h_pad]
    float* w2 = nullptr;              // [h_pad][nr]
    float* b2 = nullptr;              // [nr]
    mobi::MaskTable mtab{};

    // workspace (sized for ws_T tokens)
    int64_t ws_T = -1;
    int64_t tpad_max = 0, max_tiles = 0, htiles = 0;
    float* s_part = nullptr;   // [htiles][T][nr]
    float* scores = nullptr;   // [T][nr]
    uint8_t* masks = nullptr;  // [T]
    int32_t* perm = nullptr;   // [tpad_max] permuted row -> token (-1 pad)
    int32_t* pinv = nullptr;   // [T] token -> permuted row
    int32_t* inverse = nullptr;// [T]
    int32_t* cperm = nullptr;  // [T] compact (unpadded) permutation
    float* escale = nullptr;   // [tpad_max] per-row power-of-two scale
    __half* xperm = nullptr;   // [kblocks][tpad_max][64] fp16 permuted, scaled activations: k-block slabs,
                               // so a TMA box of consecutive permuted rows is one contiguous span
    std::shared_ptr<void> xperm_shared;  // set: xperm is a block shared with other handles
                                         // (mobi_layers_share_activations), freed with its last user
    mobi::TokTile* tiles = nullptr;  // [max_tiles]
    float* gpart = nullptr;    // [8][64][out] split-K partials (decode-size T)
    float* hpart = nullptr;    // [16][64][h_pad] router split-K partials
    float* dec_part = nullptr; // decode path: [(sm + n_rt)][kDecMaxT][128] row-tile partials
    float* dec_spart = nullptr;// decode router: [h_pad/16][kDecMaxT][nr] score partials
    int32_t* dec_cnt = nullptr;// decode arrival counters [n_rt + h_pad/16 + 1], zero between launches
    int32_t* rt_cnt = nullptr; // [T/128 + 1] router arrival counters (per token tile, then all), zero between launches
    int32_t* bk_hist = nullptr;// [48] fused bucketing: mask histogram | padded starts | slot counters
    int32_t* meta = nullptr;   // [0]=n_tiles [1]=total padded rows [2..2+16) bucket counts
    void* x_dev = nullptr;     // staging for mobi_forward_host
    void* y_dev = nullptr;
    void* h_x = nullptr;       // pinned host staging
    void* h_y = nullptr;
    int64_t h_cap = 0;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // mobi_forward_host pipeline (created on first use)
    cudaEvent_t ev_pipe[17] = {};  // e2e pipeline: [0..7] chunk copied in, [8..15] computed, [16] prior work
    CUtensorMap* tmap_x = nullptr;  // host copies, rebuilt when the workspace changes
    CUtensorMap* tmap_w1 = nullptr; // router w1t (fixed for the layer's lifetime), 128-row boxes
    CUtensorMap* tmap_w1_64 = nullptr;  // the same with 64-row boxes (CTA-pair router, N = 128)
    CUtensorMap* tmap_x2 = nullptr; // xperm, 16/32/64/128-row boxes (CTA-pair GEMM)
    int32_t last_launches = 0;
    int64_t device_bytes = 0;
    // profiling: event pairs around each launch, resolved lazily
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<int, int>>> ev_marks;  // (kernel id, (start ev, stop ev))
    size_t ev_next = 0;
    double prof_ms[4] = {0, 0, 0, 0};
    int64_t prof_n[4] = {0, 0, 0, 0};

    // Per-call state.  The handle's own workspace serves the first stream it is called on; every
    // other stream gets a context -- a mobi_layer that shares the handle's weights and owns its own
    // workspace -- so concurrent forwards on distinct streams never share scratch memory.  A
    // context's call_mu keeps one forward's launch sequence contiguous on its stream when several
    // host threads use the same stream.
    mobi_layer* owner = nullptr;         // set on per-stream contexts
    void* ctx_stream = nullptr;          // the stream this workspace serves
    bool ctx_bound = false;
    std::vector<mobi_layer*> ctxs;       // handle: contexts of the other streams
    std::mutex* ctx_mu = nullptr;        // handle: guards ctxs
    std::mutex* call_mu = nullptr;       // every context
    int64_t reserved_T = 0;              // handle: mobi_layer_reserve (applied to new contexts)
    int64_t plan_T = 0;                  // > T: choose kernels as for a batch of plan_T tokens (chunked calls)
    int32_t impl = 0;                    // development hook (mobi_layer_debug_impl): kernel override
    int32_t plan[8] = {};                // the last call's kernels (mobi_layer_last_plan)
    mobi::OutDesc od{};                  // this call's output placement (n_dst == 0: plain y)
    // multi-GPU (mobi_layer_create_sharded, shard.cu)
    int32_t shard_mode = 0, shard_rank = 0, shard_nranks = 1;
    void* shard_comm = nullptr;          // ncclComm_t of the caller
    int64_t shard_per = 0, shard_out = 0;  // rows per rank (128-aligned), the unsharded out
    __nv_bfloat16* gather_buf = nullptr;  // [P][T][per] rank-major all-gather buffer
    int64_t gather_T = 0;
    __nv_bfloat16* y_tmp = nullptr;      // staging for non-default placements on the small-T paths
    int64_t y_tmp_T = 0;
    mobi_layer* plan_ctx = nullptr;      // handle: the context that ran the last call
};

namespace mobi {

// error plumbing (abi.cu)
int set_error(int code, const std::string& msg);
#define MOBI_CUDA(call)                                                                       \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return ::mobi::set_error(MOBI_ERUNTIME, std::string(#call) + ": " +              \
                                                         cudaGetErrorString(e_));              \
    } while (0)
#define MOBI_TRY(call)              \
    do {                            \
        const int rc_ = (call);     \
        if (rc_) return rc_;        \
    } while (0)
// cudaFuncSetAttribute once per (current device, kernel, attribute): function attributes are
// per-device state, so a process driving several GPUs sets them on each (abi.cu)
int func_attr_once_impl(const void* fn, cudaFuncAttribute attr, int value);
template <class F>
inline int func_attr_once(F* fn, cudaFuncAttribute attr, int value) {
    return func_attr_once_impl(reinterpret_cast<const void*>(fn), attr, value);
}
#define MOBI_LAUNCH_CHECK()                                                                   \
    do {                                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess)                                                                \
            return ::mobi::set_error(MOBI_ERUNTIME, std::string("kernel launch: ") +         \
                                                         cudaGetErrorString(e_));              \
    } while (0)

// ---- launchers (each returns MOBI_OK or an error code; each counts its launches) ----
// layer.cu
int launch_pack_dplanes(mobi_layer* L, cudaStream_t st);
// decode2.cu
bool decode_planes_supported(const mobi_layer* L, const void* x, int64_t T);
int launch_decode_planes(mobi_layer* L, const __nv_bfloat16* x, int64_t T, const uint8_t* given_masks, float delta,
                         uint8_t* masks_out, float* scores_out, __nv_bfloat16* y, bool pdl, cudaStream_t st,
                         unsigned long long* trace = nullptr);
int check_codes_device(const uint8_t* codes_dev, int64_t n, int qmax, int64_t* bad);
int launch_pack_codes(mobi_layer* L, const uint8_t* codes_dev, cudaStream_t st);
int launch_pack_planes(mobi_layer* L, const uint64_t* planes_dev, int bits, int64_t wpr,
                       cudaStream_t st);
int launch_unpack_codes(const mobi_layer* L, uint8_t* codes_dev, cudaStream_t st);
// router.cu
int launch_router(mobi_layer* L, const __nv_bfloat16* x, int64_t T, cudaStream_t st);      // CUDA cores
// router_tc.cu (tcgen05; needs in % 8 == 0 and a 16-byte aligned X for TMA)
bool router_tc_supported(const mobi_layer* L, const void* x);
int launch_router_tc(mobi_layer* L, const __nv_bfloat16* x, int64_t T, float delta, float* scores_out,
                     uint8_t* masks_out, bool* masks_ready, cudaStream_t st, unsigned long long* trace,
                     bool fuse_bucket = false);
// bucket.cu
int launch_bucket(mobi_layer* L, int64_t T, float delta, const uint8_t* given_masks,
                  float* scores_out, uint8_t* masks_out, int32_t* cperm_out,
                  int32_t* inverse_out, int32_t* counts_out, cudaStream_t st, bool sanitize = true);
int launch_gather(mobi_layer* L, const __nv_bfloat16* x, int64_t T, cudaStream_t st, bool claim = false,
                  bool pdl = false);
// gemm_tc.cu (tcgen05) / gemm_simt.cu (reference kernel, tests only)
int launch_gemm_tc(mobi_layer* L, __nv_bfloat16* y, int64_t T, cudaStream_t st,
                   unsigned long long* trace = nullptr);
int launch_gemm_simt(mobi_layer* L, __nv_bfloat16* y, int64_t T, cudaStream_t st);
// generic slice layouts (non-uniform widths, E > kFastSlices): per-slice CUDA-core GEMM on the
// original token order, and the mask decision / stable permutation over all 2^E keys
int launch_gemm_generic(mobi_layer* L, const __nv_bfloat16* x, int64_t T, const uint8_t* masks, __nv_bfloat16* y,
                        cudaStream_t st);
int launch_bucket_generic(mobi_layer* L, int64_t T, float delta, const uint8_t* given_masks, float* scores_out,
                          uint8_t* masks_out, int32_t* cperm_out, int32_t* inverse_out, int32_t* counts_out,
                          cudaStream_t st, bool sanitize);
int launch_gemm_tc2(mobi_layer* L, __nv_bfloat16* y, int64_t T, cudaStream_t st, unsigned long long* trace = nullptr,
                    bool pdl = false);  // gemm_tc2.cu (CTA pairs)
// decode.cu (T <= kDecMaxT: router GEMV + stream-K decode GEMM, PDL-chained)
bool decode_supported(const mobi_layer* L, const void* x, int64_t T);
int launch_router_dec(mobi_layer* L, const __nv_bfloat16* x, int64_t T, float delta, uint8_t* masks_out,
                      float* scores_out, cudaStream_t st, unsigned long long* trace = nullptr);
int launch_decode_gemm(mobi_layer* L, const __nv_bfloat16* x, int64_t T, const uint8_t* given_masks, float delta,
                       uint8_t* masks_out, float* scores_out, __nv_bfloat16* y, bool pdl, cudaStream_t st,
                       unsigned long long* trace = nullptr);
// layer.cu: copy Y rows [T, out] (ldy = out) to every destination of an output descriptor
int launch_scatter_out(const __nv_bfloat16* y, int64_t T, int64_t out, const OutDesc& od, cudaStream_t st);
// select.cu: the score of descending rank k (exact fp32) -> host (synchronous on `st`)
int launch_select_desc(const float* scores, int64_t n, int64_t k, float* out_host, cudaStream_t st);
int launch_avg_bits(const uint8_t* masks, int64_t T, const int32_t* slice_bits, int32_t E, double* avg, cudaStream_t st);
// decompose.cu
int launch_decompose(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* bits,
                     int32_t E, double gamma, uint8_t* codes, double* scale, double* zero,
                     int64_t* clamp_counts_host, cudaStream_t st);

// ---- small device helpers ----
__device__ __forceinline__ float silu_f(float x) {
    // common.hpp:125-133 sigmoid with the sign split; silu = x * sigmoid(x)
    float s = x >= 0.f ? 1.f / (1.f + expf(-x)) : expf(x) / (1.f + expf(x));
    return x * s;
}

// Dequantize 4 merged codes (one 32-bit word) of a bucket with mask word `mw` into two half2
// words (elements 0,1 and 2,3):  W = S * (codes & mask) + C, exact INT->fp16 via the 0x6400
// magic (1024 + n), exact subtraction of 1024, one HFMA2.
__device__ __forceinline__ void dequant4(uint32_t codes4, uint32_t mw, __half2 S2, __half2 C2,
                                         uint32_t& w01, uint32_t& w23) {
    const uint32_t v = codes4 & mw;
    uint32_t lo = __byte_perm(v, 0x64646464u, 0x4140);
    uint32_t hi = __byte_perm(v, 0x64646464u, 0x4342);
    const __half2 k1024 = __half2half2(__ushort_as_half((unsigned short)0x6400));
    __half2 a = __hsub2(*reinterpret_cast<__half2*>(&lo), k1024);
    __half2 c = __hsub2(*reinterpret_cast<__half2*>(&hi), k1024);
    a = __hfma2(a, S2, C2);
    c = __hfma2(c, S2, C2);
    w01 = *reinterpret_cast<uint32_t*>(&a);
    w23 = *reinterpret_cast<uint32_t*>(&c);
}

}  // namespace mobi
