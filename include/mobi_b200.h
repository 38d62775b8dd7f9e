/*
 * mobi_b200.h -- C ABI of the B200-native MoBi linear layer (the drop-in for the
 * MoBiQuant inference hot path: route -> bucket -> nested residual GEMM -> un-permute).
 *
 * Plain C, plain pointers and sizes; no CUDA or torch types.  Streams are passed as
 * `void*` (a cudaStream_t, NULL = the legacy default stream).  Device pointers are
 * CUDA device memory on the layer's device.
 *
 * Reference interfaces replaced (paths under /root/reference/proj/include/mobi):
 *   mobi_layer_create        slicer::SliceStack (slicer.hpp:25-66) + qcore::QuantParams
 *                            (qcore.hpp:22-49) + router::RouterState (router.hpp:32-60), or
 *                            bench::LayerRecord (bench/checkpoint.hpp:30-74) -- the reference is
 *                            stateless, so its per-call inputs become a persistent device handle
 *   mobi_score               router::score            (router.hpp:63-76)
 *   mobi_route               router::score + router::gate_hard (router.hpp:63-97) + mask convention
 *                            (bitplane.hpp:203-206) + bitplane::permute_by_slice (bitplane.hpp:178-201)
 *   mobi_forward             score -> gate_hard(delta) -> forward_elastic(kHard) as called by
 *                            bench::eval_at_ratio (pipeline.hpp:146-183) and trainer::calibrate_model
 *                            (trainer.hpp:804-812)
 *   mobi_forward_masked      router::forward_elastic (router.hpp:105-132) with given hard gates
 *   mobi_forward_host        mobi_forward from/to host buffers (the call a CPU caller makes)
 *   mobi_permute_by_slice    bitplane::permute_by_slice (bitplane.hpp:178-201), index part
 *   mobi_calibrate_threshold router::calibrate_threshold (router.hpp:167-174)
 *   mobi_layer_unpack_codes  bench::LayerRecord::stack() (checkpoint.hpp:54-73) / bitplane::unpack
 *                            (bitplane.hpp:75-84), read back from the device layout (bit-exact check)
 *   mobi_decompose           slicer::decompose (slicer.hpp:69-113) + qcore::params_from_clip
 *                            (qcore.hpp:122-146), on the GPU
 *   mobi_joint_step          trainer::joint_forward (trainer.hpp:203-263) + trainer::joint_backward
 *                            (trainer.hpp:341-396): one stage-2 calibration step, fp64, on the GPU
 *   mobi_msb_step            trainer::msb_forward + msb_backward (trainer.hpp:404-426): the stage-1 step
 *
 * Error convention (mirrors MOBI_CHECK, common.hpp:13-24): every entry point returns
 * MOBI_OK, MOBI_EINVAL (the reference would throw std::invalid_argument; message names the
 * offending dim/index like the reference's) or MOBI_ERUNTIME (CUDA/NCCL failure,
 * std::runtime_error).  mobi_last_error() returns the thread-local message of the last failure.
 *
 * Threading: a layer handle's weights are immutable after create.  Each stream a handle is called
 * on gets its own workspace (created on first use), so calls on distinct streams may run
 * concurrently from any threads; calls on one stream are serialised by the handle (one call's
 * launch sequence is contiguous on the stream).  Handles on different devices are independent.
 */
#ifndef MOBI_B200_H
#define MOBI_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MOBI_API __attribute__((visibility("default")))
#else
#define MOBI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MOBI_OK 0
#define MOBI_EINVAL 1
#define MOBI_ERUNTIME 2

#define MOBI_MAX_SLICES 8 /* slice 1 + up to 7 routed residual slices (sum of widths <= 8 bits) */
#define MOBI_MAX_DST 8    /* destinations of one output descriptor (ranks of a column-parallel layer) */

typedef struct mobi_layer* mobi_layer_t;

/* Host-side description of one MoBi linear layer.  All arrays are host memory, row-major,
 * in the reference's own layouts and dtypes (double / uint8 / uint64). */
typedef struct {
    int64_t out;        /* output rows of W (QuantParams::rows)                         */
    int64_t in;         /* input dim (QuantParams::cols)                                 */
    int64_t group_size; /* qcore::kDefaultGroupSize = 128; group = r*ceil(in/gs) + c/gs   */
    int32_t n_slices;   /* E (SliceStack::num_slices), 2..MOBI_MAX_SLICES                */
    const int32_t* slice_bits; /* [E] widths >= 1, sum <= 8 (slice.bits = 2 2 2 2); uniform widths
                                  with E <= 4 run the tcgen05 / slice-plane kernels, any other
                                  layout the generic per-slice CUDA-core kernels */
    const double* scale; /* [out*ceil(in/gs)] base (slice-1) scales, > 0               */
    const double* zero;  /* [out*ceil(in/gs)] base (slice-1) continuous zeros          */
    /* slice payload, exactly one of: */
    const uint8_t* codes;     /* [E][out][in] slice codes c_e (SliceStack::slices)      */
    const uint64_t* planes;   /* [plane_bits][out][words_per_row] merged-code bit-planes,
                                 MSB plane first (LayerRecord::planes, bitplane.hpp:21-36) */
    int32_t plane_bits;
    int64_t words_per_row;
    /* router (RouterState): hidden width h, n_routed = E-1 */
    int64_t router_hidden;
    const double* w1; /* [in][h]     */
    const double* b1; /* [h]         */
    const double* w2; /* [h][E-1]    */
    const double* b2; /* [E-1]       */
} mobi_layer_desc;

/* Upload, validate and repack a layer onto `device`.  The handle owns its device weights. */
MOBI_API int mobi_layer_create(const mobi_layer_desc* desc, int device, mobi_layer_t* out);
/* Same as mobi_layer_create, but desc->codes ([n_slices][out][in] uint8 slice codes) already resides in
 * device memory on `device` (e.g. the output of mobi_decompose): validated and repacked on the GPU,
 * no host staging.  Every other descriptor array stays on the host.  No reference counterpart: it is
 * the device-resident ingest for model-scale stacks (hundreds of matrices). */
MOBI_API int mobi_layer_create_device(const mobi_layer_desc* desc, int device, mobi_layer_t* out);
/* Column-parallel shard: a layer holding weight rows [row0, row1) of `desc` (every slice or
 * bit-plane and the rows' group parameters -- groups never span rows, qcore.hpp:30-34) and the full
 * router, so every rank decides the same masks.  Rank p of P creates rows [p*ceil(out/P), ...) and
 * all-gathers the [T, row1-row0] outputs (NCCL) into [T, out]; the shards' outputs are bit-identical
 * to the corresponding columns of the unsharded layer's.  No reference counterpart (single process). */
MOBI_API int mobi_layer_create_rows(const mobi_layer_desc* desc, int64_t row0, int64_t row1, int device,
                                    mobi_layer_t* out);
MOBI_API int mobi_layer_destroy(mobi_layer_t layer);
/* Pre-size the internal workspace for up to max_tokens tokens (avoids allocation inside
 * forward, required before stream capture into a CUDA graph). */
MOBI_API int mobi_layer_reserve(mobi_layer_t layer, int64_t max_tokens);
/* Shape queries. */
/* Model stacks: let layers that run one after another on one stream share one permuted-activation
 * buffer (the largest workspace part, T_pad x in_pad fp16 per layer -- ~5 GiB over a 224-layer
 * LLaMA3-8B stack at 2048 tokens).  Each layer must be reserved (mobi_layer_reserve) first; the block
 * is sized for the largest and freed with its last user.  Shares the handles' primary workspace only;
 * layers whose calls can overlap in time (different streams) must not share.  A later reserve or call
 * beyond a layer's reserved size gives that layer a private buffer again.  Synchronises the device. */
MOBI_API int mobi_layers_share_activations(mobi_layer_t* layers, int32_t n);
MOBI_API int mobi_layer_info(mobi_layer_t layer, int64_t* out, int64_t* in, int32_t* n_slices,
                    int64_t* router_hidden, int64_t* device_bytes);

/* The router parameters exactly as the device uses them, widened to float (w1 is stored
 * bf16 on the device, b1/w2/b2 fp32): lets a checker feed the oracle identical inputs. */
MOBI_API int mobi_layer_export_router(mobi_layer_t layer, float* w1 /*[in][h]*/, float* b1, float* w2,
                             float* b2);
/* K6: read the device weight layout back as slice codes [E][out][in] (host). */
MOBI_API int mobi_layer_unpack_codes(mobi_layer_t layer, uint8_t* codes_host);

/* router::score: S[T][E-1] fp32 (device) from X[T][in] bf16 (device). */
MOBI_API int mobi_score(mobi_layer_t layer, const void* x_bf16, int64_t T, float* scores, void* stream);

/* score -> gate_hard(delta) -> mask_t = 1 | sum_j 1(S[t,j]-delta>0) << (j+1) -> stable bucket
 * permutation.  All outputs device, each nullable.  perm[i] = source token of permuted row i,
 * inverse[t] = permuted row of token t; bucket_count[m] = tokens with mask m (m < 2^E). */
MOBI_API int mobi_route(mobi_layer_t layer, const void* x_bf16, int64_t T, float delta, float* scores,
               uint8_t* masks, int32_t* perm, int32_t* inverse, int32_t* bucket_count,
               void* stream);

/* Full layer: Y[T][out] bf16 (device) = forward_elastic(X, stack, gate_hard(score(X), delta)).
 * masks (device, nullable) receives the per-token slice masks. */
MOBI_API int mobi_forward(mobi_layer_t layer, const void* x_bf16, int64_t T, float delta, void* y_bf16,
                 uint8_t* masks, void* stream);

/* forward_elastic with given per-token masks (device uint8, bit0 must be set; bit e-1 = slice e):
 * isolates GEMM parity from router decisions. */
MOBI_API int mobi_forward_masked(mobi_layer_t layer, const void* x_bf16, int64_t T, const uint8_t* masks,
                        void* y_bf16, void* stream);

/* Output placement: Y row t of this layer is written at dst[k] + t*ldy + col0 (bf16 elements) for
 * every k < n_dst.  Column-parallel shards use it to write their columns straight into the full
 * [T, out] buffers of every rank (dst = local + peer-mapped buffers, see mobi_ipc_open): the
 * all-gather happens in the GEMM epilogue, tile by tile.  After the call, order the peers' reads
 * behind a collective on the same stream (stores to peers are fenced system-wide by the kernel). */
typedef struct {
    int32_t n_dst;              /* 1..MOBI_MAX_DST */
    void* dst[MOBI_MAX_DST];    /* device pointers (local or peer-mapped) */
    int64_t ldy;                /* row stride of every destination, elements (>= col0 + out) */
    int64_t col0;               /* column of this layer's first output */
} mobi_out_desc;
MOBI_API int mobi_forward_out(mobi_layer_t layer, const void* x_bf16, int64_t T, float delta,
                              const mobi_out_desc* out, uint8_t* masks, void* stream);

/* Multi-GPU entry, one process per GPU, `nccl_comm` an ncclComm_t over nranks ranks
 * (NULL allowed when nranks == 1):
 *   MOBI_SHARD_COLUMN: rank p owns weight rows [p*per, (p+1)*per) (per = ceil(out/P) rounded up to
 *     128) and the full router; mobi_forward_sharded takes the full X [T, in] on every rank and
 *     returns the full Y [T, out] on every rank (the epilogue writes this rank's block into a
 *     rank-major buffer, one in-place ncclAllGather, one interleave pass).  Bit-identical to the
 *     unsharded layer.
 *   MOBI_SHARD_TOKEN: replicated weights; each rank passes its own tokens, no collective. */
#define MOBI_SHARD_COLUMN 1
#define MOBI_SHARD_TOKEN 2
MOBI_API int mobi_layer_create_sharded(const mobi_layer_desc* desc, void* nccl_comm, int rank, int nranks,
                                       int mode, int device, mobi_layer_t* out);
MOBI_API int mobi_forward_sharded(mobi_layer_t layer, const void* x_bf16, int64_t T, float delta, void* y_bf16,
                                  uint8_t* masks, void* stream);

/* CUDA IPC plumbing for peer destinations (one process per GPU): export the allocation holding
 * dev_ptr as a 64-byte handle (+ dev_ptr's offset in it), open a peer's handle on `device` (peer
 * access enabled lazily; the peer's pointer is *dev_ptr + offset), close the mapping. */
MOBI_API int mobi_ipc_export(void* dev_ptr, void* handle64, int64_t* offset);
MOBI_API int mobi_ipc_open(const void* handle64, int device, void** dev_ptr);
MOBI_API int mobi_ipc_close(void* dev_ptr);

/* mobi_forward from HOST buffers: x_host bf16 [T][in] -> y_host bf16 [T][out] (+ masks_host,
 * nullable); copies go through the layer's pinned staging buffers on `stream`; synchronous. */
MOBI_API int mobi_forward_host(mobi_layer_t layer, const void* x_host, int64_t T, float delta,
                      void* y_host, uint8_t* masks_host, void* stream);

/* bitplane::permute_by_slice index part on the GPU: masks (device, [T]) -> perm, inverse
 * (device int32 [T]), groups (host: group_mask[<=256], group_len[<=256], *n_groups). */
MOBI_API int mobi_permute_by_slice(const uint8_t* masks, int64_t T, int32_t* perm, int32_t* inverse,
                          uint8_t* group_mask, int64_t* group_len, int64_t* n_groups, void* stream);

/* router::calibrate_threshold over n device fp32 scores: delta = sort_desc(s)[floor(rho*n+1e-9)],
 * or min-1 if that index is >= n.  Synchronous; result to host. */
MOBI_API int mobi_calibrate_threshold(const float* scores, int64_t n, double rho, double* delta,
                             void* stream);

/* router::avg_bits (router.hpp:135-150) from device masks [T] (bit e-1 <-> slice e): mean over tokens
 * of the active slices' widths (exact integer sum on the device, one division).  Synchronous. */
MOBI_API int mobi_avg_bits(const uint8_t* masks, int64_t T, const int32_t* slice_bits, int32_t n_slices,
                           double* avg, void* stream);

/* slicer::decompose on the GPU, with base params from params_from_clip(identity clip gamma):
 * w (device fp64 [out][in]) -> codes (device uint8 [E][out][in]), scale/zero (device fp64
 * [out*ceil(in/gs)]), clamp_counts (host int64 [E], nullable).  Bit-exact with the reference. */
MOBI_API int mobi_decompose(const double* w, int64_t out, int64_t in, int64_t group_size,
                   const int32_t* slice_bits, int32_t n_slices, double gamma, uint8_t* codes,
                   double* scale, double* zero, int64_t* clamp_counts, void* stream);

/* Stage-2 calibration step (offline PTQ).  BudgetSchedule (trainer.hpp:45-51):
 * shape 0 log / 1 linear / 2 cosine / 3 exp. */
typedef struct mobi_budget_schedule {
    double b_init;
    double b_target;
    int64_t total_steps;
    int32_t shape;
    double reg_weight;
} mobi_budget_schedule;

/* JointForward's scalars (trainer.hpp:186-199) */
typedef struct mobi_joint_scalars {
    double data_term;
    double reg_term; /* unweighted (AvgBits - b(t)) * ||G||_1 */
    double avg_bits;
    double sched_b;
    double loss;
    double tau; /* 0 at t = L (indicator gate) and with force_gates_on */
} mobi_joint_scalars;

/* trainer::joint_forward (+ joint_backward when d_gamma_lo is non-null) of one QuantLayer, fp64:
 *   w [out][in], x [T][in], y_fp [T][out], router w1 [in][h], b1 [h], w2 [h][n_slices-1], b2 [n_slices-1],
 *   y_hat [T][out] (nullable) and the router gradients (same shapes) are DEVICE memory;
 *   slice_bits, the per-group clip gammas gamma_lo / gamma_hi [out*ceil(in/gs)] and their gradients are
 *   HOST memory (the clip squash runs on the host with the reference's libm; groups are few).
 * Synchronous on `stream`.  Errors as the reference's MOBI_CHECKs (shape mismatch, t outside [1, L]). */
MOBI_API int mobi_joint_step(const double* w, int64_t out, int64_t in, int64_t group_size, const int32_t* slice_bits,
                             int32_t n_slices, const double* gamma_lo, const double* gamma_hi, const double* w1,
                             const double* b1, const double* w2, const double* b2, int64_t hidden, const double* x,
                             const double* y_fp, int64_t T, const mobi_budget_schedule* sched, int64_t t,
                             int32_t force_gates_on, double* y_hat, mobi_joint_scalars* scalars, double* d_gamma_lo,
                             double* d_gamma_hi, double* d_w1, double* d_b1, double* d_w2, double* d_b2,
                             void* stream);

/* Stage-1 calibration step: trainer::msb_forward + msb_backward (trainer.hpp:404-426), fp64 -- slice 1
 * alone (quantize_floor with the clip's base params), y_msb = X·W_1ᵀ, loss = MSE, clip gradients.
 * Same memory conventions as mobi_joint_step; y_msb and the gradients are nullable. */
MOBI_API int mobi_msb_step(const double* w, int64_t out, int64_t in, int64_t group_size, int32_t msb_bits,
                           const double* gamma_lo, const double* gamma_hi, const double* x, const double* y_fp,
                           int64_t T, double* y_msb, double* loss, double* d_gamma_lo, double* d_gamma_hi,
                           void* stream);

/* Per-kernel device timing (CUDA events recorded on the launch stream around every kernel the
 * layer launches).  enable=1 starts a fresh accumulation; mobi_layer_profile_read synchronises
 * and returns, per kernel id (0 router, 1 bucket, 2 gather, 3 gemm), the summed milliseconds and
 * the number of launches since enabling. */
#define MOBI_PROF_KERNELS 4
MOBI_API int mobi_layer_profile(mobi_layer_t layer, int enable);
MOBI_API int mobi_layer_profile_read(mobi_layer_t layer, double* ms /*[MOBI_PROF_KERNELS]*/,
                                     int64_t* launches /*[MOBI_PROF_KERNELS]*/);

/* Number of kernels the last forward on this layer launched (for launch accounting). */
MOBI_API int mobi_layer_last_launches(mobi_layer_t layer, int32_t* launches);

/* Kernel ids reported by mobi_layer_last_plan. */
#define MOBI_K_NONE 0
#define MOBI_K_ROUTER_DECODE 1      /* decode GEMV router (router_dec_kernel, T <= 32)               */
#define MOBI_K_ROUTER_TC 2          /* 1-CTA tcgen05 router tiles (128 tokens x 128 hidden)          */
#define MOBI_K_ROUTER_TC_CLUSTER 3  /* the same with K split over a 2-3 CTA cluster (DSMEM sum)     */
#define MOBI_K_ROUTER_TC_SPLITK 4   /* the same with global split-K partials + a reduce kernel       */
#define MOBI_K_ROUTER_PAIR128 5     /* CTA-pair tcgen05 router, 256 tokens x 128 hidden per pair    */
#define MOBI_K_ROUTER_PAIR256 6     /* CTA-pair tcgen05 router, 256 tokens x 256 hidden per pair    */
#define MOBI_K_ROUTER_SIMT 7        /* CUDA-core router (inputs the tcgen05 router cannot take)      */
#define MOBI_K_GEMM_DECODE_PLANES 11 /* decode GEMV over the union's 2-bit slice planes              */
#define MOBI_K_GEMM_DECODE_MERGED 12 /* decode stream-K GEMV over the merged 8-bit codes             */
#define MOBI_K_GEMM_SPLITK 13       /* 1-CTA tcgen05 nested residual GEMM with split-K (T <= 64)     */
#define MOBI_K_GEMM_PAIR 14         /* CTA-pair tcgen05 nested residual GEMM (prefill)              */
#define MOBI_K_GEMM_SIMT 15         /* CUDA-core reference GEMM (test hook only)                     */
#define MOBI_K_GEMM_GENERIC 16      /* per-slice CUDA-core GEMM: non-uniform widths or > 4 slices    */
/* The last call's plan: plan[0] router kernel id, [1] GEMM kernel id, [2] GEMM grid (CTAs),
 * [3] kernels launched, [4] token tiles of the bucketed GEMM (-1 for the decode kernels),
 * [5] 256-row weight-tile pairs, [6] GEMM units = [4] x [5] (-1 for decode), [7] tokens.
 * Synchronises the call's stream to read the device-side tile count. */
MOBI_API int mobi_layer_last_plan(mobi_layer_t layer, int32_t* plan /*[8]*/);

MOBI_API const char* mobi_last_error(void);

/* Test hook (not part of the drop-in surface), per layer: impl 1 routes the GEMM through the
 * CUDA-core reference kernel (gemm_simt.cu) so the test-suite can cross-check the tcgen05 kernel;
 * 5 = the 1-CTA split-K GEMM, 10 = the decode kernels for every batch they support (T <= 32);
 * other values select traced / alternative kernels for development tools.  0 = production. */
MOBI_API int mobi_layer_debug_impl(mobi_layer_t layer, int impl);
MOBI_API const char* mobi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOBI_B200_H */
