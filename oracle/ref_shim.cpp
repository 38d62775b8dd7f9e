// ref_shim.cpp -- extern "C" wrappers over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file against
// /root/reference/proj/include (the reference sources where they lie; nothing
// is copied) into oracle/_ref/libmobi_ref.so.  It is used (a) to pin the C
// restatement in mobi_oracle.c bit-for-bit, (b) to mint the golden fixtures in
// tests/golden/, and (c) as the timed CPU baseline (bench.py cpu_baseline /
// --impl reference, kind "reference").  It is never linked into the product.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "mobi/bench/checkpoint.hpp"
#include "mobi/bitplane.hpp"
#include "mobi/common.hpp"
#include "mobi/qcore.hpp"
#include "mobi/router.hpp"
#include "mobi/slicer.hpp"
#include "mobi/trainer.hpp"

using namespace mobi;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Matrix mat(const double* p, int64_t r, int64_t c) {
    Matrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));
    if (r * c) std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(r * c));
    return m;
}

void put(const Matrix& m, double* out) {
    if (m.size()) std::memcpy(out, m.data(), sizeof(double) * m.size());
}

qcore::QuantParams params(int64_t rows, int64_t cols, int64_t gs, int bits, const double* scale,
                          const double* zero) {
    qcore::QuantParams qp;
    qp.rows = static_cast<std::size_t>(rows);
    qp.cols = static_cast<std::size_t>(cols);
    qp.group_size = static_cast<std::size_t>(gs);
    qp.bits = bits;
    std::size_t n = qp.num_groups();
    qp.scale.assign(scale, scale + n);
    qp.zero.assign(zero, zero + n);
    return qp;
}

slicer::SliceStack stack_of(const uint8_t* codes, int32_t n_slices, const int32_t* slice_bits,
                            int64_t out, int64_t in, int64_t gs, const double* scale,
                            const double* zero) {
    slicer::SliceStack st;
    st.slice_bits.assign(slice_bits, slice_bits + n_slices);
    st.base = params(out, in, gs, slice_bits[0], scale, zero);
    const std::size_t n = static_cast<std::size_t>(out * in);
    for (int32_t e = 0; e < n_slices; ++e) {
        Codes c(static_cast<std::size_t>(out), static_cast<std::size_t>(in));
        std::memcpy(c.vec().data(), codes + e * n, n);
        st.slices.push_back(std::move(c));
    }
    st.clamp_mask = Codes(static_cast<std::size_t>(out), static_cast<std::size_t>(in), 0);
    st.clamp_counts.assign(static_cast<std::size_t>(n_slices), 0);
    return st;
}

router::RouterState router_of(int64_t d, int64_t h, int64_t nr, const double* w1, const double* b1,
                              const double* w2, const double* b2) {
    router::RouterState rs;
    rs.w1 = mat(w1, d, h);
    rs.b1.assign(b1, b1 + h);
    rs.w2 = mat(w2, h, nr);
    rs.b2.assign(b2, b2 + nr);
    return rs;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// router.hpp:63
int ref_score(const double* x, int64_t T, int64_t d, const double* w1, const double* b1, int64_t h,
              const double* w2, const double* b2, int64_t nr, double* s) {
    return guard([&] { put(router::score(mat(x, T, d), router_of(d, h, nr, w1, b1, w2, b2)), s); });
}

// router.hpp:93
int ref_gate_hard(const double* s, int64_t T, int64_t nr, double delta, double* g) {
    return guard([&] { put(router::gate_hard(mat(s, T, nr), delta), g); });
}

// router.hpp:105
int ref_forward_elastic(const double* x, int64_t T, int64_t in, const uint8_t* codes,
                        int32_t n_slices, const int32_t* slice_bits, const double* scale,
                        const double* zero, int64_t out, int64_t gs, const double* gates, int hard,
                        double* y) {
    return guard([&] {
        slicer::SliceStack st = stack_of(codes, n_slices, slice_bits, out, in, gs, scale, zero);
        Matrix r = router::forward_elastic(mat(x, T, in), st, mat(gates, T, n_slices - 1),
                                           hard ? router::GateMode::kHard : router::GateMode::kSoft);
        put(r, y);
    });
}

// router.hpp:167
int ref_calibrate_threshold(const double* scores, int64_t n, double rho, double* delta) {
    return guard([&] {
        std::vector<double> v(scores, scores + n);
        *delta = router::calibrate_threshold(std::move(v), rho);
    });
}

// router.hpp:135
int ref_avg_bits(const double* gates, int64_t T, int64_t nr, const int32_t* slice_bits,
                 int32_t n_slices, double* result) {
    return guard([&] {
        *result = router::avg_bits(mat(gates, T, nr), std::vector<int>(slice_bits, slice_bits + n_slices));
    });
}

// router.hpp:153
int ref_ratio_from_target_bits(double target, const int32_t* slice_bits, int32_t n_slices,
                               double* rho) {
    return guard([&] {
        *rho = router::ratio_from_target_bits(target, std::vector<int>(slice_bits, slice_bits + n_slices));
    });
}

// router.hpp:47 RouterState::init with a fresh Rng(seed) (fixture generation)
int ref_router_init(int64_t d, int64_t nr, int64_t hidden, uint64_t seed, double* w1, double* b1,
                    double* w2, double* b2) {
    return guard([&] {
        Rng rng(seed);
        router::RouterState rs = router::RouterState::init(static_cast<std::size_t>(d), static_cast<std::size_t>(nr), 1000, rng,
                                                           static_cast<std::size_t>(hidden));
        put(rs.w1, w1);
        std::copy(rs.b1.begin(), rs.b1.end(), b1);
        put(rs.w2, w2);
        std::copy(rs.b2.begin(), rs.b2.end(), b2);
    });
}

// qcore.hpp:122 params_from_clip (GroupStats::from_weights + ClipParams)
int ref_params_from_clip(const double* w, int64_t rows, int64_t cols, int64_t gs,
                         const double* gamma_lo, const double* gamma_hi, int bits, double* scale,
                         double* zero) {
    return guard([&] {
        Matrix m = mat(w, rows, cols);
        qcore::GroupStats gst = qcore::GroupStats::from_weights(m, static_cast<std::size_t>(gs));
        qcore::ClipParams cp;
        cp.gamma_lo.assign(gamma_lo, gamma_lo + gst.min.size());
        cp.gamma_hi.assign(gamma_hi, gamma_hi + gst.min.size());
        qcore::QuantParams qp = qcore::params_from_clip(m, gst, cp, bits, static_cast<std::size_t>(gs));
        std::copy(qp.scale.begin(), qp.scale.end(), scale);
        std::copy(qp.zero.begin(), qp.zero.end(), zero);
    });
}

// slicer.hpp:69 decompose
int ref_decompose(const double* w, int64_t rows, int64_t cols, int64_t gs, const double* scale,
                  const double* zero, const int32_t* slice_bits, int32_t n_slices, uint8_t* codes,
                  uint8_t* clamp_mask, int64_t* clamp_counts) {
    return guard([&] {
        qcore::QuantParams base = params(rows, cols, gs, slice_bits[0], scale, zero);
        slicer::SliceStack st = slicer::decompose(mat(w, rows, cols), base,
                                                  std::vector<int>(slice_bits, slice_bits + n_slices));
        const std::size_t n = static_cast<std::size_t>(rows * cols);
        for (int32_t e = 0; e < n_slices; ++e) std::memcpy(codes + e * n, st.slices[e].vec().data(), n);
        if (clamp_mask) std::memcpy(clamp_mask, st.clamp_mask.vec().data(), n);
        if (clamp_counts)
            for (int32_t e = 0; e < n_slices; ++e) clamp_counts[e] = static_cast<int64_t>(st.clamp_counts[e]);
    });
}

// slicer.hpp:135 reconstruct
int ref_reconstruct(const uint8_t* codes, int64_t rows, int64_t cols, int64_t gs,
                    const int32_t* slice_bits, int32_t n_slices, const double* scale,
                    const double* zero, int32_t k, double* out) {
    return guard([&] {
        put(slicer::reconstruct(stack_of(codes, n_slices, slice_bits, rows, cols, gs, scale, zero),
                                static_cast<std::size_t>(k)),
            out);
    });
}

// slicer.hpp:150 merge_codes
int ref_merge_codes(const uint8_t* codes, int64_t rows, int64_t cols, const int32_t* slice_bits,
                    int32_t n_slices, int32_t k, uint8_t* merged) {
    return guard([&] {
        std::vector<double> dummy(static_cast<std::size_t>(rows * ((cols + 127) / 128)), 1.0);
        slicer::SliceStack st = stack_of(codes, n_slices, slice_bits, rows, cols, 128, dummy.data(), dummy.data());
        Codes m = slicer::merge_codes(st, static_cast<std::size_t>(k));
        std::memcpy(merged, m.vec().data(), m.size());
    });
}

// bitplane.hpp:48 pack_bit_major; planes out[bits][rows*wpr]
int ref_pack_bit_major(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint64_t* planes) {
    return guard([&] {
        Codes c(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
        std::memcpy(c.vec().data(), codes, static_cast<std::size_t>(rows * cols));
        bitplane::PackedPlanes pp = bitplane::pack_bit_major(c, bits);
        std::size_t off = 0;
        for (const auto& p : pp.planes) {
            std::memcpy(planes + off, p.data(), p.size() * sizeof(uint64_t));
            off += p.size();
        }
    });
}

// checkpoint.hpp:54 LayerRecord::stack() from merged bit planes -> slice codes [n_slices][rows*cols]
int ref_layer_stack(const uint64_t* planes, int64_t rows, int64_t cols, int bits, int64_t wpr,
                    const int32_t* slice_bits, int32_t n_slices, uint8_t* codes) {
    return guard([&] {
        bench::LayerRecord rec;
        rec.rows = static_cast<std::size_t>(rows);
        rec.cols = static_cast<std::size_t>(cols);
        rec.group_size = 128;
        rec.slice_bits.assign(slice_bits, slice_bits + n_slices);
        rec.planes.out = rec.rows;
        rec.planes.in = rec.cols;
        rec.planes.bits = bits;
        rec.planes.words_per_row = static_cast<std::size_t>(wpr);
        const std::size_t np = static_cast<std::size_t>(rows * wpr);
        for (int p = 0; p < bits; ++p) rec.planes.planes.emplace_back(planes + p * np, planes + (p + 1) * np);
        slicer::SliceStack st = rec.stack();
        const std::size_t n = static_cast<std::size_t>(rows * cols);
        for (int32_t e = 0; e < n_slices; ++e) std::memcpy(codes + e * n, st.slices[e].vec().data(), n);
    });
}

// bitplane.hpp:122 bitplane_matmul
int ref_bitplane_matmul(const double* x, int64_t T, const uint64_t* planes, int64_t out, int64_t in,
                        int bits, int64_t wpr, int64_t gs, const double* scale, const double* zero,
                        const int32_t* active, int32_t n_active, double* y) {
    return guard([&] {
        bitplane::PackedPlanes pp;
        pp.out = static_cast<std::size_t>(out);
        pp.in = static_cast<std::size_t>(in);
        pp.bits = bits;
        pp.words_per_row = static_cast<std::size_t>(wpr);
        const std::size_t np = static_cast<std::size_t>(out * wpr);
        for (int p = 0; p < bits; ++p) pp.planes.emplace_back(planes + p * np, planes + (p + 1) * np);
        auto res = bitplane::bitplane_matmul(mat(x, T, in), pp, params(out, in, gs, bits, scale, zero),
                                             std::vector<int>(active, active + n_active));
        put(res.out, y);
    });
}

// bitplane.hpp:178 permute_by_slice
int ref_permute_by_slice(const double* tokens, int64_t T, int64_t cols, const uint8_t* masks,
                         double* permuted, int64_t* perm, int64_t* inverse, uint8_t* group_mask,
                         int64_t* group_len, int64_t* n_groups) {
    return guard([&] {
        auto p = bitplane::permute_by_slice(mat(tokens, T, cols), std::vector<std::uint8_t>(masks, masks + T));
        if (permuted) put(p.permuted, permuted);
        for (int64_t i = 0; i < T; ++i) {
            perm[i] = static_cast<int64_t>(p.perm[i]);
            inverse[i] = static_cast<int64_t>(p.inverse[i]);
        }
        for (std::size_t g = 0; g < p.groups.size(); ++g) {
            group_mask[g] = p.groups[g].first;
            group_len[g] = static_cast<int64_t>(p.groups[g].second);
        }
        *n_groups = static_cast<int64_t>(p.groups.size());
    });
}

// The timed CPU baseline: the reference's own per-layer inference sequence
// score -> gate_hard(delta) -> forward_elastic (pipeline.hpp:146-183, with delta
// given), token-sharded over `threads` std::threads (the functions are pure and
// re-entrant).  Returns the hard gates and outputs.
int ref_layer_forward_threaded(const double* x, int64_t T, int64_t in, const uint8_t* codes,
                               int32_t n_slices, const int32_t* slice_bits, const double* scale,
                               const double* zero, int64_t out, int64_t gs, int64_t h,
                               const double* w1, const double* b1, const double* w2,
                               const double* b2, double delta, int threads, double* gates_out,
                               double* y) {
    return guard([&] {
        const int64_t nr = n_slices - 1;
        slicer::SliceStack st = stack_of(codes, n_slices, slice_bits, out, in, gs, scale, zero);
        router::RouterState rs = router_of(in, h, nr, w1, b1, w2, b2);
        int nt = std::max(1, std::min<int>(threads, static_cast<int>(T)));
        std::vector<std::thread> pool;
        std::vector<std::string> errs(static_cast<std::size_t>(nt));
        for (int w = 0; w < nt; ++w) {
            pool.emplace_back([&, w] {
                try {
                    int64_t t0 = T * w / nt, t1 = T * (w + 1) / nt;
                    if (t1 <= t0) return;
                    Matrix xs = mat(x + t0 * in, t1 - t0, in);
                    Matrix s = router::score(xs, rs);
                    Matrix g = router::gate_hard(s, delta);
                    Matrix ys = router::forward_elastic(xs, st, g, router::GateMode::kHard);
                    if (gates_out) std::memcpy(gates_out + t0 * nr, g.data(), sizeof(double) * g.size());
                    std::memcpy(y + t0 * out, ys.data(), sizeof(double) * ys.size());
                } catch (const std::exception& e) {
                    errs[static_cast<std::size_t>(w)] = e.what();
                }
            });
        }
        for (auto& t : pool) t.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
    });
}

// Same sequence, sharded for small token counts: score is token-sharded, forward_elastic is
// ROW-sharded -- each thread runs the reference forward_elastic on the SliceStack of a block of
// output rows (groups never span rows, qcore.hpp:30-34, so the split is exact and the output
// columns are bit-identical to the unsharded call).  This amortises the reference's per-call
// re-dequantization (router.hpp:115-120) across threads.
int ref_layer_forward_rowsharded(const double* x, int64_t T, int64_t in, const uint8_t* codes,
                                 int32_t n_slices, const int32_t* slice_bits, const double* scale,
                                 const double* zero, int64_t out, int64_t gs, int64_t h,
                                 const double* w1, const double* b1, const double* w2,
                                 const double* b2, double delta, int threads, double* gates_out,
                                 double* y) {
    return guard([&] {
        const int64_t nr = n_slices - 1;
        const int64_t gpr = (in + gs - 1) / gs;
        router::RouterState rs = router_of(in, h, nr, w1, b1, w2, b2);
        Matrix xs = mat(x, T, in);
        // score, token-sharded
        Matrix g(static_cast<std::size_t>(T), static_cast<std::size_t>(nr));
        {
            int nt = std::max(1, std::min<int>(threads, static_cast<int>(T)));
            std::vector<std::thread> pool;
            for (int w = 0; w < nt; ++w)
                pool.emplace_back([&, w] {
                    int64_t t0 = T * w / nt, t1 = T * (w + 1) / nt;
                    if (t1 <= t0) return;
                    Matrix s = router::score(mat(x + t0 * in, t1 - t0, in), rs);
                    Matrix gg = router::gate_hard(s, delta);
                    std::memcpy(g.data() + t0 * nr, gg.data(), sizeof(double) * gg.size());
                });
            for (auto& t : pool) t.join();
        }
        if (gates_out) std::memcpy(gates_out, g.data(), sizeof(double) * g.size());
        // forward_elastic, row-sharded over sub-stacks
        int nt = std::max(1, std::min<int>(threads, static_cast<int>(out)));
        std::vector<std::thread> pool;
        std::vector<std::string> errs(static_cast<std::size_t>(nt));
        for (int w = 0; w < nt; ++w)
            pool.emplace_back([&, w] {
                try {
                    int64_t r0 = out * w / nt, r1 = out * (w + 1) / nt, nrow = r1 - r0;
                    if (nrow <= 0) return;
                    std::vector<uint8_t> sub(static_cast<std::size_t>(n_slices * nrow * in));
                    for (int32_t e = 0; e < n_slices; ++e)
                        std::memcpy(sub.data() + e * nrow * in, codes + e * out * in + r0 * in,
                                    static_cast<std::size_t>(nrow * in));
                    slicer::SliceStack st = stack_of(sub.data(), n_slices, slice_bits, nrow, in, gs,
                                                     scale + r0 * gpr, zero + r0 * gpr);
                    Matrix ys = router::forward_elastic(xs, st, g, router::GateMode::kHard);
                    for (int64_t t = 0; t < T; ++t)
                        std::memcpy(y + t * out + r0, ys.data() + t * nrow, sizeof(double) * nrow);
                } catch (const std::exception& e) {
                    errs[static_cast<std::size_t>(w)] = e.what();
                }
            });
        for (auto& t : pool) t.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
    });
}

// trainer.hpp:203-263 joint_forward + 341-396 joint_backward (one stage-2 calibration step).
// scalars[6] = data_term, reg_term, avg_bits, sched_b, loss, tau.  Gradients are written only when
// d_gamma_lo is non-null.
int ref_joint_step(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* slice_bits,
                   int32_t n_slices, const double* gamma_lo, const double* gamma_hi, const double* w1,
                   const double* b1, const double* w2, const double* b2, int64_t h, const double* x,
                   const double* y_fp, int64_t T, double b_init, double b_target, int64_t total_steps,
                   int32_t shape, double reg_weight, int64_t t, int32_t force_gates_on, double* y_hat,
                   double* scalars, double* d_gamma_lo, double* d_gamma_hi, double* d_w1, double* d_b1,
                   double* d_w2, double* d_b2) {
    return guard([&] {
        trainer::QuantLayer L;
        L.w = mat(w, out, in);
        L.group_size = static_cast<std::size_t>(gs);
        L.slice_bits.assign(slice_bits, slice_bits + n_slices);
        L.stats = qcore::GroupStats::from_weights(L.w, L.group_size);
        const std::size_t ng = L.stats.min.size();
        L.clip.gamma_lo.assign(gamma_lo, gamma_lo + ng);
        L.clip.gamma_hi.assign(gamma_hi, gamma_hi + ng);
        L.rs = router_of(in, h, n_slices - 1, w1, b1, w2, b2);
        trainer::BudgetSchedule sc;
        sc.b_init = b_init;
        sc.b_target = b_target;
        sc.total_steps = static_cast<std::size_t>(total_steps);
        sc.shape = static_cast<trainer::ScheduleShape>(shape);
        sc.reg_weight = reg_weight;
        trainer::JointOptions opt;
        opt.force_gates_on = force_gates_on != 0;
        const Matrix X = mat(x, T, in), Y = mat(y_fp, T, out);
        trainer::JointForward f = trainer::joint_forward(L, X, Y, sc, static_cast<std::size_t>(t), opt);
        if (y_hat) put(f.y_hat, y_hat);
        const double sv[6] = {f.data_term, f.reg_term, f.avg_bits, f.sched_b, f.loss, f.tau};
        std::copy(sv, sv + 6, scalars);
        if (!d_gamma_lo) return;
        trainer::JointGrads g = trainer::joint_backward(L, f, X, Y, sc);
        std::copy(g.d_gamma_lo.begin(), g.d_gamma_lo.end(), d_gamma_lo);
        std::copy(g.d_gamma_hi.begin(), g.d_gamma_hi.end(), d_gamma_hi);
        put(g.d_w1, d_w1);
        std::copy(g.d_b1.begin(), g.d_b1.end(), d_b1);
        put(g.d_w2, d_w2);
        std::copy(g.d_b2.begin(), g.d_b2.end(), d_b2);
    });
}

// trainer.hpp:404-426 msb_forward + msb_backward (the stage-1 step)
int ref_msb_step(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* slice_bits, int32_t n_slices,
                 const double* gamma_lo, const double* gamma_hi, const double* x, const double* y_fp, int64_t T,
                 double* y_msb, double* loss, double* d_gamma_lo, double* d_gamma_hi) {
    return guard([&] {
        trainer::QuantLayer L;
        L.w = mat(w, out, in);
        L.group_size = static_cast<std::size_t>(gs);
        L.slice_bits.assign(slice_bits, slice_bits + n_slices);
        L.stats = qcore::GroupStats::from_weights(L.w, L.group_size);
        const std::size_t ng = L.stats.min.size();
        L.clip.gamma_lo.assign(gamma_lo, gamma_lo + ng);
        L.clip.gamma_hi.assign(gamma_hi, gamma_hi + ng);
        const Matrix X = mat(x, T, in), Y = mat(y_fp, T, out);
        trainer::MsbForward f = trainer::msb_forward(L, X, Y);
        put(f.y_msb, y_msb);
        *loss = f.loss;
        std::vector<double> lo, hi;
        trainer::msb_backward(L, f, X, Y, lo, hi);
        std::copy(lo.begin(), lo.end(), d_gamma_lo);
        std::copy(hi.begin(), hi.end(), d_gamma_hi);
    });
}

}  // extern "C"
