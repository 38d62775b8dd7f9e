/*
 * mobi_oracle.c -- CPU restatement of the MoBiQuant reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see mobi_oracle.h).  Compiled with
 * -ffp-contract=off so no multiply-add is fused, matching the reference's
 * -O3 build on x86-64 (no FMA).  Each function cites the reference
 * function it restates; loop order and double operation order are kept so
 * the results are bit-identical to the reference.
 */
#include "mobi_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return 1;
}

#define CHECK(cond, ...)                      \
    do {                                      \
        if (!(cond)) return fail(__VA_ARGS__); \
    } while (0)

/* common.hpp:125-133 */
static double sigmoid(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}
static double silu(double x) { return x * sigmoid(x); }

/* ---------------- common.hpp:140-201 Rng ---------------- */
static uint64_t splitmix64(uint64_t* x) {
    *x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

void orc_rng_init(orc_rng* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
    r->spare = 0.0;
    r->has_spare = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n) { return orc_rng_next_u64(r) % n; }

double orc_rng_normal(orc_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = 0.0;
    do {
        u1 = orc_rng_uniform(r);
    } while (u1 <= 0.0);
    double u2 = orc_rng_uniform(r);
    double rad = sqrt(-2.0 * log(u1));
    double theta = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(theta);
    r->has_spare = 1;
    return rad * cos(theta);
}

void orc_rng_fill_normal(orc_rng* r, double* out, int64_t n, double scale) {
    for (int64_t i = 0; i < n; ++i) out[i] = scale * orc_rng_normal(r);
}

/* ---------------- bench/calibset.hpp:20-47 ---------------- */
int orc_gen_calibset(int64_t nsamples, int64_t seqlen, int64_t dim, double outlier_frac,
                     double outlier_scale, uint64_t seed, double* out,
                     int64_t* outlier_channels, int64_t* n_outlier) {
    CHECK(dim > 0, "gen_calibset: dim must be positive");
    orc_rng rng;
    orc_rng_init(&rng, seed ^ 0x9e3779b97f4a7c15ULL);
    int64_t n_out = 0;
    if (outlier_frac > 0.0) {
        n_out = (int64_t)llround(outlier_frac * (double)dim);
        if (n_out < 1) n_out = 1;
    }
    double* channel_scale = (double*)malloc(sizeof(double) * (size_t)dim);
    unsigned char* taken = (unsigned char*)calloc((size_t)dim, 1);
    for (int64_t c = 0; c < dim; ++c) channel_scale[c] = 1.0;
    int64_t have = 0;
    while (have < n_out) {
        int64_t c = (int64_t)orc_rng_uniform_index(&rng, (uint64_t)dim);
        if (taken[c]) continue;
        taken[c] = 1;
        if (outlier_channels) outlier_channels[have] = c;
        ++have;
        channel_scale[c] = outlier_scale;
    }
    if (n_outlier) *n_outlier = n_out;
    for (int64_t i = 0; i < nsamples; ++i)
        for (int64_t t = 0; t < seqlen; ++t)
            for (int64_t c = 0; c < dim; ++c)
                out[(i * seqlen + t) * dim + c] = channel_scale[c] * orc_rng_normal(&rng);
    free(channel_scale);
    free(taken);
    return 0;
}

/* ---------------- bench/calibset.hpp:56-66 ---------------- */
int orc_gen_model(int64_t dim, int64_t depth, uint64_t seed, double weight_scale, double* out) {
    orc_rng rng;
    orc_rng_init(&rng, seed ^ 0xd1b54a32d192ed03ULL);
    for (int64_t i = 0; i < depth * dim * dim; ++i) out[i] = weight_scale * orc_rng_normal(&rng);
    return 0;
}

/* ---------------- router.hpp:47-60 ---------------- */
int orc_router_init(int64_t d, int64_t n_routed, int64_t hidden, orc_rng* rng, double* w1,
                    double* b1, double* w2, double* b2) {
    int64_t h = hidden ? hidden : (d / 4 > 1 ? d / 4 : 1);
    double sd = 1.0 / sqrt((double)d);
    for (int64_t i = 0; i < d * h; ++i) w1[i] = sd * orc_rng_normal(rng);
    for (int64_t i = 0; i < h; ++i) b1[i] = 0.0;
    for (int64_t i = 0; i < h * n_routed; ++i) w2[i] = 0.0;
    for (int64_t i = 0; i < n_routed; ++i) b2[i] = 0.0;
    return 0;
}

/* ---------------- qcore.hpp ---------------- */
static int64_t groups_per_row(int64_t cols, int64_t gs) { return (cols + gs - 1) / gs; }

/* qcore.hpp:43-54 QuantParams::validate */
static int validate_params(int64_t rows, int64_t cols, int64_t gs, int bits, const double* scale,
                           const double* zero) {
    CHECK(bits >= 1 && bits <= 8, "QuantParams: bits must be in [1,8], got %d", bits);
    CHECK(gs >= 1, "QuantParams: group_size must be >= 1");
    int64_t n = rows * groups_per_row(cols, gs);
    for (int64_t g = 0; g < n; ++g) {
        CHECK(isfinite(scale[g]) && scale[g] > 0.0, "QuantParams: non-positive scale at group %lld",
              (long long)g);
        CHECK(isfinite(zero[g]), "QuantParams: non-finite zero at group %lld", (long long)g);
    }
    return 0;
}

/* qcore.hpp:75-118 GroupStats::from_weights + clip_lo_of/clip_hi_of, 122-146 params_from_clip */
int orc_params_from_clip(const double* w, int64_t rows, int64_t cols, int64_t gs,
                         const double* gamma_lo, const double* gamma_hi, int bits, double* scale,
                         double* zero) {
    CHECK(rows * cols > 0, "params_from_clip: empty weight");
    CHECK(bits >= 1 && bits <= 8, "params_from_clip: bits must be in [1,8], got %d", bits);
    int64_t gpr = groups_per_row(cols, gs);
    int64_t n = rows * gpr;
    double* mn = (double*)malloc(sizeof(double) * (size_t)n);
    double* mx = (double*)malloc(sizeof(double) * (size_t)n);
    unsigned char* seen = (unsigned char*)calloc((size_t)n, 1);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int64_t g = r * gpr + c / gs;
            double v = w[r * cols + c];
            if (!isfinite(v)) {
                free(mn);
                free(mx);
                free(seen);
                return fail("GroupStats: non-finite weight at (%lld,%lld)", (long long)r,
                            (long long)c);
            }
            if (!seen[g]) {
                mn[g] = v;
                mx[g] = v;
                seen[g] = 1;
            } else {
                if (v < mn[g]) mn[g] = v;
                if (v > mx[g]) mx[g] = v;
            }
        }
    double qmax = (double)((1 << bits) - 1);
    for (int64_t g = 0; g < n; ++g) {
        double lo0 = mn[g] > 0.0 ? mn[g] : 0.0;             /* std::max(0.0, min) */
        double ref = lo0 < mx[g] ? lo0 : mx[g];                /* std::min(.., max) */
        double lo = ref + sigmoid(gamma_lo[g]) * (mn[g] - ref);
        double hi = ref + sigmoid(gamma_hi[g]) * (mx[g] - ref);
        double s = (hi - lo) / qmax;
        if (!(s > 1e-8)) s = 1e-8;
        scale[g] = s;
        zero[g] = -lo / s;
    }
    free(mn);
    free(mx);
    free(seen);
    return 0;
}

/* qcore.hpp:159-177 quantize_floor */
int orc_quantize_floor(const double* x, int64_t rows, int64_t cols, int64_t gs, int bits,
                       const double* scale, const double* zero, uint8_t* codes) {
    if (validate_params(rows, cols, gs, bits, scale, zero)) return 1;
    int64_t gpr = groups_per_row(cols, gs);
    const double qmax = (double)((1 << bits) - 1);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            double v = x[r * cols + c];
            CHECK(isfinite(v), "quantize_floor: non-finite input at (%lld,%lld)", (long long)r,
                  (long long)c);
            int64_t g = r * gpr + c / gs;
            double u = floor(v / scale[g] + zero[g]);
            u = fmin(fmax(u, 0.0), qmax);
            codes[r * cols + c] = (uint8_t)u;
        }
    return 0;
}

/* qcore.hpp:180-197 dequantize_centered */
int orc_dequantize_centered(const uint8_t* codes, int64_t rows, int64_t cols, int64_t gs, int bits,
                            const double* scale, const double* zero, double* out) {
    if (validate_params(rows, cols, gs, bits, scale, zero)) return 1;
    int64_t gpr = groups_per_row(cols, gs);
    const int qmax = (1 << bits) - 1;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int code = codes[r * cols + c];
            CHECK(code >= 0 && code <= qmax,
                  "dequantize_centered: code %d out of [0,%d] at (%lld,%lld)", code, qmax,
                  (long long)r, (long long)c);
            int64_t g = r * gpr + c / gs;
            out[r * cols + c] = scale[g] * ((double)code - zero[g] + 0.5);
        }
    return 0;
}

/* ---------------- slicer.hpp ---------------- */
static int bits_before(const int32_t* slice_bits, int32_t e) {
    int acc = 0;
    for (int32_t j = 0; j + 1 < e; ++j) acc += slice_bits[j];
    return acc;
}

/* slicer.hpp:69-113 decompose (slice_params 51-61 inlined: s_e = s*2^-bb, z_e = 2^(b_e-1)) */
int orc_decompose(const double* w, int64_t rows, int64_t cols, int64_t gs, const double* scale,
                  const double* zero, const int32_t* slice_bits, int32_t n_slices, uint8_t* codes,
                  uint8_t* clamp_mask, int64_t* clamp_counts) {
    CHECK(n_slices > 0, "decompose: slice_bits is empty");
    int total = 0;
    for (int32_t e = 0; e < n_slices; ++e) {
        CHECK(slice_bits[e] >= 1 && slice_bits[e] <= 8, "decompose: slice bit width %d out of [1,8]",
              slice_bits[e]);
        total += slice_bits[e];
    }
    CHECK(total <= 8, "decompose: total bits %d exceed the 8-bit code budget", total);
    if (validate_params(rows, cols, gs, slice_bits[0], scale, zero)) return 1;
    const int64_t n = rows * cols;
    const int64_t gpr = groups_per_row(cols, gs);
    const int64_t ng = rows * gpr;
    double* resid = (double*)malloc(sizeof(double) * (size_t)n);
    double* sc = (double*)malloc(sizeof(double) * (size_t)ng);
    memcpy(resid, w, sizeof(double) * (size_t)n);
    if (clamp_mask) memset(clamp_mask, 0, (size_t)n);
    for (int32_t e = 1; e <= n_slices; ++e) {
        double f = ldexp(1.0, -bits_before(slice_bits, e));
        for (int64_t g = 0; g < ng; ++g) sc[g] = e == 1 ? scale[g] : scale[g] * f;
        const double mid = ldexp(1.0, slice_bits[e - 1] - 1);
        const double qmax = (double)((1 << slice_bits[e - 1]) - 1);
        int64_t clamped = 0;
        uint8_t* ce = codes + (int64_t)(e - 1) * n;
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t c = 0; c < cols; ++c) {
                int64_t g = r * gpr + c / gs;
                double z = e == 1 ? zero[g] : mid;
                double v = resid[r * cols + c];
                if (!isfinite(v)) {
                    free(resid);
                    free(sc);
                    return fail("decompose: non-finite residual at (%lld,%lld)", (long long)r,
                                (long long)c);
                }
                double u = floor(v / sc[g] + z);
                if (u < 0.0 || u > qmax) {
                    if (clamp_mask) clamp_mask[r * cols + c] |= (uint8_t)(1u << (e - 1));
                    ++clamped;
                    u = fmin(fmax(u, 0.0), qmax);
                }
                ce[r * cols + c] = (uint8_t)u;
                resid[r * cols + c] = v - sc[g] * (u - z + 0.5);
            }
        if (clamp_counts) clamp_counts[e - 1] = clamped;
    }
    free(resid);
    free(sc);
    return 0;
}

/* slicer.hpp:118-146 reconstruct_frame + reconstruct */
int orc_reconstruct(const uint8_t* codes, int64_t rows, int64_t cols, int64_t gs,
                    const int32_t* slice_bits, int32_t n_slices, const double* scale,
                    const double* zero, int32_t k, double* out) {
    CHECK(k >= 1 && k <= n_slices, "reconstruct: k = %d out of [1,%d]", k, n_slices);
    const int64_t n = rows * cols;
    const int64_t gpr = groups_per_row(cols, gs);
    for (int64_t i = 0; i < n; ++i) out[i] = codes[i] + 0.5;
    for (int32_t e = 2; e <= k; ++e) {
        double unit = ldexp(1.0, -bits_before(slice_bits, e));
        double mid = ldexp(1.0, slice_bits[e - 1] - 1);
        const uint8_t* ce = codes + (int64_t)(e - 1) * n;
        for (int64_t i = 0; i < n; ++i) out[i] += (ce[i] - mid + 0.5) * unit;
    }
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int64_t g = r * gpr + c / gs;
            out[r * cols + c] = scale[g] * (out[r * cols + c] - zero[g]);
        }
    return 0;
}

/* slicer.hpp:150-161 merge_codes */
int orc_merge_codes(const uint8_t* codes, int64_t n, const int32_t* slice_bits, int32_t n_slices,
                    int32_t k, uint8_t* merged) {
    CHECK(k >= 1 && k <= n_slices, "merge_codes: k = %d out of range", k);
    memcpy(merged, codes, (size_t)n);
    for (int32_t e = 2; e <= k; ++e) {
        int b = slice_bits[e - 1];
        const uint8_t* ce = codes + (int64_t)(e - 1) * n;
        for (int64_t i = 0; i < n; ++i) merged[i] = (uint8_t)((merged[i] << b) + ce[i]);
    }
    return 0;
}

/* ---------------- common.hpp:84-123 naive matmuls (fixed k order) ---------------- */
/* C = A * B^T, A (m x k), B (n x k) */
static void matmul_nt(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* c) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            const double* ar = a + i * k;
            const double* br = b + j * k;
            for (int64_t q = 0; q < k; ++q) acc += ar[q] * br[q];
            c[i * n + j] = acc;
        }
}
/* C = A * B, A (m x k), B (k x n) */
static void matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* c) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int64_t q = 0; q < k; ++q) acc += a[i * k + q] * b[q * n + j];
            c[i * n + j] = acc;
        }
}

/* ---------------- router.hpp ---------------- */
/* router.hpp:63-76 score */
int orc_score(const double* x, int64_t T, int64_t d, const double* w1, const double* b1, int64_t h,
              const double* w2, const double* b2, int64_t n_routed, double* s) {
    for (int64_t i = 0; i < T * d; ++i)
        CHECK(isfinite(x[i]), "score: non-finite input at flat index %lld", (long long)i);
    double* hidden = (double*)malloc(sizeof(double) * (size_t)(T * h > 0 ? T * h : 1));
    matmul(x, T, d, w1, h, hidden);
    for (int64_t r = 0; r < T; ++r)
        for (int64_t c = 0; c < h; ++c) hidden[r * h + c] = silu(hidden[r * h + c] + b1[c]);
    matmul(hidden, T, h, w2, n_routed, s);
    for (int64_t r = 0; r < T; ++r)
        for (int64_t c = 0; c < n_routed; ++c) s[r * n_routed + c] += b2[c];
    free(hidden);
    return 0;
}

/* router.hpp:93-97 gate_hard */
void orc_gate_hard(const double* s, int64_t n, double delta, double* g) {
    for (int64_t i = 0; i < n; ++i) g[i] = (s[i] - delta) > 0.0 ? 1.0 : 0.0;
}

/* router.hpp:105-132 forward_elastic (reconstruct(st,1) for slice 1, dequantize_centered with
 * slice_params(e) for e >= 2, each contracted over ALL tokens, gate skips/copies/scales rows) */
int orc_forward_elastic(const double* x, int64_t T, int64_t in, const uint8_t* codes,
                        int32_t n_slices, const int32_t* slice_bits, const double* scale,
                        const double* zero, int64_t out, int64_t gs, const double* gates,
                        int hard, double* y) {
    const int64_t nr = n_slices - 1;
    if (hard) {
        for (int64_t i = 0; i < T * nr; ++i)
            CHECK(gates[i] == 0.0 || gates[i] == 1.0, "forward_elastic: hard gate not binary");
    }
    if (validate_params(out, in, gs, slice_bits[0], scale, zero)) return 1;
    const int64_t n = out * in;
    const int64_t gpr = groups_per_row(in, gs);
    double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* pe = (double*)malloc(sizeof(double) * (size_t)(T * out > 0 ? T * out : 1));
    double* sc = (double*)malloc(sizeof(double) * (size_t)(out * gpr));
    /* W_1 = reconstruct(st, 1): s * ((c_1 + 0.5) - z) (frame form, slicer.hpp:121,142) */
    for (int64_t r = 0; r < out; ++r)
        for (int64_t c = 0; c < in; ++c) {
            int64_t g = r * gpr + c / gs;
            double frame = codes[r * in + c] + 0.5;
            w[r * in + c] = scale[g] * (frame - zero[g]);
        }
    matmul_nt(x, T, in, w, out, y);
    for (int32_t e = 2; e <= n_slices; ++e) {
        double f = ldexp(1.0, -bits_before(slice_bits, e));
        double mid = ldexp(1.0, slice_bits[e - 1] - 1);
        int qmax = (1 << slice_bits[e - 1]) - 1;
        for (int64_t g = 0; g < out * gpr; ++g) sc[g] = scale[g] * f;
        const uint8_t* ce = codes + (int64_t)(e - 1) * n;
        for (int64_t r = 0; r < out; ++r)
            for (int64_t c = 0; c < in; ++c) {
                int code = ce[r * in + c];
                if (code > qmax) {
                    free(w);
                    free(pe);
                    free(sc);
                    return fail("dequantize_centered: code %d out of [0,%d] at (%lld,%lld)", code,
                                qmax, (long long)r, (long long)c);
                }
                int64_t g = r * gpr + c / gs;
                w[r * in + c] = sc[g] * ((double)code - mid + 0.5);
            }
        matmul_nt(x, T, in, w, out, pe);
        for (int64_t i = 0; i < T; ++i) {
            double gv = gates[i * nr + (e - 2)];
            if (gv == 0.0) continue;
            if (gv == 1.0) {
                for (int64_t j = 0; j < out; ++j) y[i * out + j] += pe[i * out + j];
            } else {
                for (int64_t j = 0; j < out; ++j) y[i * out + j] += gv * pe[i * out + j];
            }
        }
    }
    free(w);
    free(pe);
    free(sc);
    return 0;
}

/* router.hpp:135-150 avg_bits */
int orc_avg_bits(const double* gates, int64_t T, int64_t nr, const int32_t* slice_bits,
                 int32_t n_slices, double* result) {
    CHECK(n_slices > 0, "avg_bits: empty slice_bits");
    CHECK(T > 0, "avg_bits: no tokens");
    CHECK(nr + 1 == n_slices, "avg_bits: gate columns %lld != residual slices %d", (long long)nr,
          n_slices - 1);
    for (int64_t i = 0; i < T * nr; ++i)
        CHECK(gates[i] >= 0.0 && gates[i] <= 1.0, "avg_bits: gate outside [0,1]");
    double total = 0.0;
    for (int64_t i = 0; i < T; ++i) {
        double bits = (double)slice_bits[0];
        for (int64_t j = 0; j < nr; ++j)
            if (gates[i * nr + j] > 0.5) bits += (double)slice_bits[j + 1];
        total += bits;
    }
    *result = total / (double)T;
    return 0;
}

/* router.hpp:153-162 ratio_from_target_bits */
int orc_ratio_from_target_bits(double target, const int32_t* slice_bits, int32_t n_slices,
                               double* rho) {
    CHECK(n_slices >= 2, "ratio_from_target_bits: need at least one residual slice");
    double b_msb = (double)slice_bits[0];
    double resid = 0.0;
    for (int32_t e = 1; e < n_slices; ++e) resid += (double)slice_bits[e];
    CHECK(target >= b_msb && target <= b_msb + resid,
          "ratio_from_target_bits: target %g outside [%g,%g]", target, b_msb, b_msb + resid);
    *rho = (target - b_msb) / resid;
    return 0;
}

static int cmp_desc(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}

/* router.hpp:167-174 calibrate_threshold */
int orc_calibrate_threshold(const double* scores, int64_t n, double rho, double* delta) {
    CHECK(n > 0, "calibrate_threshold: empty score sample");
    CHECK(rho >= 0.0 && rho <= 1.0, "calibrate_threshold: rho %g outside [0,1]", rho);
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(s, scores, sizeof(double) * (size_t)n);
    qsort(s, (size_t)n, sizeof(double), cmp_desc);
    int64_t k = (int64_t)floor(rho * (double)n + 1e-9);
    *delta = k >= n ? s[n - 1] - 1.0 : s[k];
    free(s);
    return 0;
}

void orc_masks_from_gates(const double* gates, int64_t T, int64_t nr, uint8_t* masks) {
    for (int64_t t = 0; t < T; ++t) {
        unsigned m = 1u;
        for (int64_t j = 0; j < nr; ++j)
            if (gates[t * nr + j] > 0.5) m |= 1u << (j + 1);
        masks[t] = (uint8_t)m;
    }
}

/* ---------------- bitplane.hpp ---------------- */
int64_t orc_words_for(int64_t n) { return (n + 63) / 64; }

/* bitplane.hpp:48-73 */
int orc_pack_bit_major(const uint8_t* codes, int64_t rows, int64_t cols, int bits,
                       uint64_t* planes) {
    CHECK(bits >= 1 && bits <= 8, "pack_bit_major: bits %d out of [1,8]", bits);
    const unsigned qmax = (1u << bits) - 1u;
    const int64_t wpr = orc_words_for(cols);
    memset(planes, 0, sizeof(uint64_t) * (size_t)(bits * rows * wpr));
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            unsigned code = codes[r * cols + c];
            CHECK(code <= qmax, "pack_bit_major: code %u exceeds %d bits at (%lld,%lld)", code, bits,
                  (long long)r, (long long)c);
            for (int b = 0; b < bits; ++b)
                if ((code >> b) & 1u)
                    planes[(int64_t)(bits - 1 - b) * rows * wpr + r * wpr + c / 64] |=
                        (uint64_t)1 << (c % 64);
        }
    return 0;
}

/* bitplane.hpp:75-84 */
int orc_unpack(const uint64_t* planes, int64_t rows, int64_t cols, int bits, int64_t wpr,
               uint8_t* codes) {
    CHECK(bits >= 1 && bits <= 8, "unpack: bits %d out of [1,8]", bits);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            unsigned code = 0;
            for (int b = 0; b < bits; ++b) {
                uint64_t word = planes[(int64_t)(bits - 1 - b) * rows * wpr + r * wpr + c / 64];
                code |= (unsigned)((word >> (c % 64)) & 1u) << b;
            }
            codes[r * cols + c] = (uint8_t)code;
        }
    return 0;
}

/* bench/checkpoint.hpp:54-73 LayerRecord::stack() split of merged codes */
int orc_split_merged(const uint8_t* merged, int64_t n, const int32_t* slice_bits, int32_t n_slices,
                     uint8_t* codes) {
    int total = 0;
    for (int32_t e = 0; e < n_slices; ++e) total += slice_bits[e];
    int shift = total;
    for (int32_t e = 0; e < n_slices; ++e) {
        shift -= slice_bits[e];
        unsigned mask = (1u << slice_bits[e]) - 1u;
        for (int64_t i = 0; i < n; ++i) codes[(int64_t)e * n + i] = (uint8_t)((merged[i] >> shift) & mask);
    }
    return 0;
}

/* bitplane.hpp:89-111 */
int orc_preaffine_accumulate(const double* x, int64_t T, const uint64_t* planes, int64_t out,
                             int64_t in, int bits, int64_t wpr, const int32_t* active,
                             int32_t n_active, double* acc) {
    CHECK(n_active > 0, "bitplane_matmul: active plane set is empty");
    for (int32_t i = 0; i < n_active; ++i)
        CHECK(active[i] >= 0 && active[i] < bits, "bitplane_matmul: plane %d out of [0,%d]",
              active[i], bits - 1);
    for (int64_t i = 0; i < T * out; ++i) acc[i] = 0.0;
    for (int32_t ai = 0; ai < n_active; ++ai) {
        int p = active[ai];
        const uint64_t* plane = planes + (int64_t)(bits - 1 - p) * out * wpr;
        const double weight = ldexp(1.0, p);
        for (int64_t t = 0; t < T; ++t)
            for (int64_t r = 0; r < out; ++r) {
                double dot = 0.0;
                const uint64_t* row = plane + r * wpr;
                for (int64_t c = 0; c < in; ++c)
                    if ((row[c / 64] >> (c % 64)) & 1u) dot += x[t * in + c];
                acc[t * out + r] += weight * dot;
            }
    }
    return 0;
}

/* bitplane.hpp:122-167 */
int orc_bitplane_matmul(const double* x, int64_t T, const uint64_t* planes, int64_t out, int64_t in,
                        int bits, int64_t wpr, int64_t gs, const double* scale, const double* zero,
                        const int32_t* active, int32_t n_active, double* y) {
    CHECK(n_active > 0, "bitplane_matmul: active plane set is empty");
    for (int32_t i = 0; i < n_active; ++i)
        CHECK(active[i] >= 0 && active[i] < bits, "bitplane_matmul: plane %d out of range", active[i]);
    const int64_t gpr = groups_per_row(in, gs);
    double* xsum = (double*)calloc((size_t)(T * gpr > 0 ? T * gpr : 1), sizeof(double));
    for (int64_t t = 0; t < T; ++t)
        for (int64_t c = 0; c < in; ++c) xsum[t * gpr + c / gs] += x[t * in + c];
    for (int64_t t = 0; t < T; ++t)
        for (int64_t r = 0; r < out; ++r) {
            double out_val = 0.0;
            for (int64_t gc = 0; gc < gpr; ++gc) {
                const int64_t c0 = gc * gs;
                const int64_t c1 = in < c0 + gs ? in : c0 + gs;
                double acc = 0.0;
                for (int32_t ai = 0; ai < n_active; ++ai) {
                    int p = active[ai];
                    const uint64_t* row = planes + (int64_t)(bits - 1 - p) * out * wpr + r * wpr;
                    double dot = 0.0;
                    for (int64_t c = c0; c < c1; ++c)
                        if ((row[c / 64] >> (c % 64)) & 1u) dot += x[t * in + c];
                    acc += ldexp(1.0, p) * dot;
                }
                const int64_t g = r * gpr + gc;
                out_val += scale[g] * (acc - (zero[g] - 0.5) * xsum[t * gpr + gc]);
            }
            y[t * out + r] = out_val;
        }
    free(xsum);
    return 0;
}

/* bitplane.hpp:178-201 permute_by_slice: std::stable_sort by mask == counting sort */
int orc_permute_by_slice(const double* tokens, int64_t T, int64_t cols, const uint8_t* masks,
                         double* permuted, int64_t* perm, int64_t* inverse, uint8_t* group_mask,
                         int64_t* group_len, int64_t* n_groups) {
    int64_t count[256] = {0};
    int64_t start[256];
    for (int64_t t = 0; t < T; ++t) ++count[masks[t]];
    int64_t acc = 0;
    for (int m = 0; m < 256; ++m) {
        start[m] = acc;
        acc += count[m];
    }
    for (int64_t t = 0; t < T; ++t) perm[start[masks[t]]++] = t;
    for (int64_t i = 0; i < T; ++i) {
        inverse[perm[i]] = i;
        if (permuted)
            for (int64_t c = 0; c < cols; ++c) permuted[i * cols + c] = tokens[perm[i] * cols + c];
    }
    int64_t ng = 0;
    for (int m = 0; m < 256; ++m)
        if (count[m]) {
            group_mask[ng] = (uint8_t)m;
            group_len[ng] = count[m];
            ++ng;
        }
    *n_groups = ng;
    return 0;
}
