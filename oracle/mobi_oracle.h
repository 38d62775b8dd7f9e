/*
 * mobi_oracle.h -- CPU restatement of the MoBiQuant reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This header and mobi_oracle.c are the parity
 * checker for the B200 product path (paper_2602_20191_b200/csrc).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * Nothing in the product links or calls it.
 *
 * Every function restates one reference function in plain C99 with the same
 * loop order and the same double-precision operation order, so its results are
 * bit-identical to the reference (pinned by tests/test_oracle.py against the
 * reference itself compiled into oracle/_ref/ and against the golden vectors in
 * tests/golden/).  File:line citations are into /root/reference/proj/include/mobi.
 *
 * Conventions: all matrices are dense row-major; sizes are int64_t; every
 * function returns 0 on success or 1 on an invalid argument, with the message
 * (worded like the reference's MOBI_CHECK text) available from
 * orc_last_error().
 */
#ifndef MOBI_ORACLE_H
#define MOBI_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* ---- common.hpp:140-201  xoshiro256++ seeded by splitmix64, Box-Muller normal ---- */
typedef struct {
    uint64_t s[4];
    double spare;
    int has_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n);
double orc_rng_normal(orc_rng* r);
/* Fill n normals / uniform indices in sequence (convenience for fixture generation). */
void orc_rng_fill_normal(orc_rng* r, double* out, int64_t n, double scale);

/* ---- bench/calibset.hpp:20-47  gen_calibset: out[nsamples][seqlen][dim] ---- */
int orc_gen_calibset(int64_t nsamples, int64_t seqlen, int64_t dim, double outlier_frac,
                     double outlier_scale, uint64_t seed, double* out,
                     int64_t* outlier_channels /* nullable, length round(frac*dim) */,
                     int64_t* n_outlier /* nullable */);

/* ---- bench/calibset.hpp:56-66  gen_model: out[depth][dim][dim] ---- */
int orc_gen_model(int64_t dim, int64_t depth, uint64_t seed, double weight_scale, double* out);

/* ---- router.hpp:47-60  RouterState::init (w1 ~ N(0,1/d), b1 = 0, w2 = 0, b2 = 0) ---- */
int orc_router_init(int64_t d, int64_t n_routed, int64_t hidden, orc_rng* rng, double* w1,
                    double* b1, double* w2, double* b2);

/* ---- qcore.hpp:75-146  GroupStats + params_from_clip ---- */
int orc_params_from_clip(const double* w, int64_t rows, int64_t cols, int64_t group_size,
                         const double* gamma_lo, const double* gamma_hi, int bits,
                         double* scale, double* zero);

/* ---- qcore.hpp:159-197  quantize_floor / dequantize_centered ---- */
int orc_quantize_floor(const double* x, int64_t rows, int64_t cols, int64_t group_size, int bits,
                       const double* scale, const double* zero, uint8_t* codes);
int orc_dequantize_centered(const uint8_t* codes, int64_t rows, int64_t cols, int64_t group_size,
                            int bits, const double* scale, const double* zero, double* out);

/* ---- slicer.hpp:69-113  decompose: codes[n_slices][rows*cols] ---- */
int orc_decompose(const double* w, int64_t rows, int64_t cols, int64_t group_size,
                  const double* scale, const double* zero, const int32_t* slice_bits,
                  int32_t n_slices, uint8_t* codes, uint8_t* clamp_mask /* nullable */,
                  int64_t* clamp_counts /* nullable */);

/* ---- slicer.hpp:118-146  reconstruct_frame / reconstruct(st, k) ---- */
int orc_reconstruct(const uint8_t* codes, int64_t rows, int64_t cols, int64_t group_size,
                    const int32_t* slice_bits, int32_t n_slices, const double* scale,
                    const double* zero, int32_t k, double* out);

/* ---- slicer.hpp:150-161  merge_codes(st, k) ---- */
int orc_merge_codes(const uint8_t* codes, int64_t n, const int32_t* slice_bits, int32_t n_slices,
                    int32_t k, uint8_t* merged);

/* ---- router.hpp:63-76  score: S = silu(X w1 + b1) w2 + b2 ---- */
int orc_score(const double* x, int64_t T, int64_t d, const double* w1, const double* b1,
              int64_t h, const double* w2, const double* b2, int64_t n_routed, double* s);

/* ---- router.hpp:93-97  gate_hard: G = 1((S - delta) > 0) ---- */
void orc_gate_hard(const double* s, int64_t n, double delta, double* g);

/* ---- router.hpp:105-132  forward_elastic (hard=1 checks binary gates) ---- */
int orc_forward_elastic(const double* x, int64_t T, int64_t in, const uint8_t* codes,
                        int32_t n_slices, const int32_t* slice_bits, const double* scale,
                        const double* zero, int64_t out, int64_t group_size,
                        const double* gates, int hard, double* y);

/* ---- router.hpp:135-192 ---- */
int orc_avg_bits(const double* gates, int64_t T, int64_t n_routed, const int32_t* slice_bits,
                 int32_t n_slices, double* result);
int orc_ratio_from_target_bits(double target, const int32_t* slice_bits, int32_t n_slices,
                               double* rho);
int orc_calibrate_threshold(const double* scores, int64_t n, double rho, double* delta);

/* ---- mask convention (bitplane.hpp:203-206): bit e-1 <-> slice e; slice 1 always on ---- */
void orc_masks_from_gates(const double* gates, int64_t T, int64_t n_routed, uint8_t* masks);

/* ---- bitplane.hpp:48-84  pack_bit_major / unpack; planes[bits][rows*wpr] MSB plane first ---- */
int64_t orc_words_for(int64_t n);
int orc_pack_bit_major(const uint8_t* codes, int64_t rows, int64_t cols, int bits,
                       uint64_t* planes);
int orc_unpack(const uint64_t* planes, int64_t rows, int64_t cols, int bits, int64_t wpr,
               uint8_t* codes);

/* ---- bench/checkpoint.hpp:54-73  LayerRecord::stack(): merged codes -> slice codes ---- */
int orc_split_merged(const uint8_t* merged, int64_t n, const int32_t* slice_bits,
                     int32_t n_slices, uint8_t* codes);

/* ---- bitplane.hpp:89-167  preaffine_accumulate / bitplane_matmul (epilogue oracle) ---- */
int orc_preaffine_accumulate(const double* x, int64_t T, const uint64_t* planes, int64_t out,
                             int64_t in, int bits, int64_t wpr, const int32_t* active,
                             int32_t n_active, double* acc);
int orc_bitplane_matmul(const double* x, int64_t T, const uint64_t* planes, int64_t out,
                        int64_t in, int bits, int64_t wpr, int64_t group_size,
                        const double* scale, const double* zero, const int32_t* active,
                        int32_t n_active, double* y);

/* ---- bitplane.hpp:178-201  permute_by_slice (stable, ascending mask) ---- */
int orc_permute_by_slice(const double* tokens, int64_t T, int64_t cols, const uint8_t* masks,
                         double* permuted /* nullable */, int64_t* perm, int64_t* inverse,
                         uint8_t* group_mask, int64_t* group_len, int64_t* n_groups);

#ifdef __cplusplus
}
#endif
#endif
