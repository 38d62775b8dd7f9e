// dropin_test.cpp -- the reference's own hot-path calls next to the drop-in (include/mobi_b200.hpp):
// builds a layer with the reference's decompose/RouterState, runs router::score + gate_hard +
// forward_elastic from the reference and the same calls through the B200 shim, and compares
// (scores within 2e-3+1e-4|S|, masks equal outside a 1e-2 margin, outputs rel-L2 per token <= 1e-2).
// Built by tests/cpp/Makefile against /root/reference (test infrastructure), run by
// tests/test_cpp_dropin.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <vector>

#include "mobi/bench/calibset.hpp"
#include "mobi/bitplane.hpp"
#include "mobi/router.hpp"
#include "mobi/slicer.hpp"
#include "mobi/trainer.hpp"
#include "mobi_b200.hpp"

using namespace mobi;

static int fails = 0;
#define EXPECT(c, ...)                 \
    do {                               \
        if (!(c)) {                    \
            std::printf("FAIL: " __VA_ARGS__); \
            std::printf("\n");         \
            ++fails;                   \
        }                              \
    } while (0)

int run_case(size_t out, size_t in, size_t gs, size_t T, unsigned seed) {
    Rng rng(seed);
    Matrix w(out, in);
    for (size_t i = 0; i < w.size(); ++i) w[i] = 0.02 * rng.normal();
    qcore::GroupStats gst = qcore::GroupStats::from_weights(w, gs);
    qcore::ClipParams cp = qcore::ClipParams::identity_init(gst.min.size(), 4.0);
    qcore::QuantParams base = qcore::params_from_clip(w, gst, cp, 2, gs);
    slicer::SliceStack st = slicer::decompose(w, base, {2, 2, 2, 2});
    router::RouterState rs = router::RouterState::init(in, 3, 1000, rng);
    for (auto& v : rs.w2.vec()) v = 0.3 * rng.normal();
    for (auto& v : rs.b2) v = 0.1 * rng.normal();
    bench::CalibSet cs = bench::gen_calibset(1, T, in, 0.05, 8.0, seed + 1);
    Matrix x = cs.batches[0];
    // feed both sides the same bf16-representable inputs and device-rounded router weights
    for (size_t i = 0; i < x.size(); ++i) x[i] = mobi_b200::from_bf16(mobi_b200::to_bf16(x[i]));
    for (size_t i = 0; i < rs.w1.size(); ++i) rs.w1[i] = mobi_b200::from_bf16(mobi_b200::to_bf16(rs.w1[i]));
    for (auto& v : rs.w2.vec()) v = static_cast<float>(v);
    for (auto& v : rs.b2) v = static_cast<float>(v);

    mobi_b200::Layer layer(st, rs);
    Matrix s_ref = router::score(x, rs);
    Matrix s_gpu = layer.score(x);
    double max_ds = 0;
    for (size_t i = 0; i < s_ref.size(); ++i) {
        double d = std::fabs(s_ref[i] - s_gpu[i]);
        max_ds = std::max(max_ds, d);
        EXPECT(d <= 2e-3 + 1e-4 * std::fabs(s_ref[i]), "score %zu: %g vs %g", i, s_ref[i], s_gpu[i]);
    }
    double delta = router::calibrate_threshold(s_ref.vec(), 1.0 / 6.0);
    Matrix g_ref = router::gate_hard(s_ref, delta);
    Matrix g_gpu;
    Matrix y_full = layer.forward(x, delta, &g_gpu);
    size_t flips = 0;
    for (size_t t = 0; t < T; ++t) {
        bool near = false;
        for (size_t j = 0; j < 3; ++j) near |= std::fabs(s_ref(t, j) - delta) <= 1e-2;
        for (size_t j = 0; j < 3; ++j)
            if (g_ref(t, j) != g_gpu(t, j)) {
                ++flips;
                EXPECT(near, "gate flip outside margin at token %zu", t);
            }
    }
    // forward_elastic with the GPU's own gates: reference vs drop-in
    Matrix y_ref = router::forward_elastic(x, st, g_gpu, router::GateMode::kHard);
    Matrix y_gpu = layer.forward_elastic(x, g_gpu);
    double worst = 0;
    for (size_t t = 0; t < T; ++t) {
        double num = 0, den = 0, num2 = 0;
        for (size_t r = 0; r < out; ++r) {
            double d = y_gpu(t, r) - y_ref(t, r), d2 = y_full(t, r) - y_ref(t, r);
            num += d * d;
            num2 += d2 * d2;
            den += y_ref(t, r) * y_ref(t, r);
        }
        double rel = std::sqrt(num / den), rel2 = std::sqrt(num2 / den);
        worst = std::max(worst, std::max(rel, rel2));
        EXPECT(rel <= 1e-2 && rel2 <= 1e-2, "token %zu rel-L2 %g / %g", t, rel, rel2);
    }
    // column-parallel shards (mobi_layer_create_rows): two halves of the rows concatenate to the full
    // layer's output bit-for-bit (same kernels, same per-row arithmetic)
    if (out >= 64) {
        const int64_t half = static_cast<int64_t>(out / 2);
        mobi_b200::Layer s0(st, rs, 0, 0, half), s1(st, rs, 0, half, static_cast<int64_t>(out));
        Matrix y0 = s0.forward_elastic(x, g_gpu), y1 = s1.forward_elastic(x, g_gpu);
        for (size_t t = 0; t < T; ++t)
            for (size_t r = 0; r < out; ++r) {
                const double v = r < static_cast<size_t>(half) ? y0(t, r) : y1(t, r - half);
                EXPECT(v == y_gpu(t, r), "shard output (%zu,%zu) %g != %g", t, r, v, y_gpu(t, r));
            }
    }
    // the remaining hot-path calls of the reference next to the shim's GPU versions
    {
        std::vector<float> sf(s_ref.size());
        std::vector<double> s_f(s_ref.size());
        for (size_t i = 0; i < s_ref.size(); ++i) s_f[i] = sf[i] = static_cast<float>(s_ref[i]);
        for (double rho : {0.0, 1.0 / 12, 1.0 / 6, 1.0 / 3, 1.0})
            EXPECT(mobi_b200::calibrate_threshold(s_f, rho) == router::calibrate_threshold(s_f, rho),
                   "calibrate_threshold rho=%g", rho);
        EXPECT(mobi_b200::avg_bits(g_gpu, {2, 2, 2, 2}) == router::avg_bits(g_gpu, {2, 2, 2, 2}), "avg_bits");
        std::vector<uint8_t> masks(T, 1);
        for (size_t t = 0; t < T; ++t)
            for (size_t j = 0; j < 3; ++j)
                if (g_gpu(t, j) > 0.5) masks[t] |= static_cast<uint8_t>(1u << (j + 1));
        bitplane::Permutation pr = bitplane::permute_by_slice(x, masks);
        Matrix xp;
        mobi_b200::Permutation pg = mobi_b200::permute_by_slice(x, masks, &xp);
        EXPECT(pg.perm == pr.perm && pg.inverse == pr.inverse, "permute_by_slice perm/inverse");
        EXPECT(pg.groups == pr.groups, "permute_by_slice groups");
        bool same = xp.size() == pr.permuted.size();
        for (size_t i = 0; same && i < xp.size(); ++i) same = xp[i] == pr.permuted[i];
        EXPECT(same, "permute_by_slice permuted tokens");
    }
    // the multi-GPU entry at world size 1 (COLUMN: one shard owning every row; TOKEN: replicas)
    for (int mode : {MOBI_SHARD_COLUMN, MOBI_SHARD_TOKEN}) {
        mobi_b200::ShardedLayer sl(st, rs, nullptr, 0, 1, mode, 0);
        Matrix ys = sl.forward(x, delta);
        bool same = ys.size() == y_full.size();
        for (size_t i = 0; same && i < ys.size(); ++i) same = ys[i] == y_full[i];
        EXPECT(same, "sharded forward (mode %d, world 1) == forward", mode);
    }
    // error behaviour mirrors MOBI_CHECK
    bool threw = false;
    try {
        layer.forward_elastic(x, Matrix(T, 2, 1.0));
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "gate shape mismatch must throw std::invalid_argument");
    std::printf("case %zux%zu gs=%zu T=%zu: max|dS| %.2e, gate flips %zu, worst rel-L2 %.2e\n", out, in, gs, T, max_ds,
                flips, worst);
    return 0;
}

// trainer::joint_forward / joint_backward (the stage-2 calibration step) next to mobi_b200::joint_step
int run_joint(size_t out, size_t in, size_t T, unsigned seed) {
    Rng rng(seed);
    Matrix w(out, in);
    for (size_t i = 0; i < w.size(); ++i) w[i] = 0.02 * rng.normal();
    trainer::QuantLayer L = trainer::QuantLayer::init(w, {2, 2, 2, 2}, 128, 10, rng, 4.0);
    for (auto& v : L.rs.w2.vec()) v = 0.5 * rng.normal();
    for (size_t g = 0; g < L.clip.gamma_lo.size(); ++g) {
        L.clip.gamma_lo[g] = 1.0 + 4.0 * rng.uniform();
        L.clip.gamma_hi[g] = 1.0 + 4.0 * rng.uniform();
    }
    Matrix x(T, in);
    for (size_t i = 0; i < x.size(); ++i) x[i] = rng.normal();
    Matrix y = matmul_nt(x, w);
    trainer::BudgetSchedule sc;
    sc.total_steps = 10;
    sc.reg_weight = 1e-3;
    trainer::JointOptions opt;
    for (size_t t : {3u, 10u}) {
        trainer::JointForward f = trainer::joint_forward(L, x, y, sc, t, opt);
        trainer::JointGrads g = trainer::joint_backward(L, f, x, y, sc);
        auto r = mobi_b200::joint_step(L, x, y, sc, t, opt);
        auto rel = [](const double* a, const double* b, size_t n) {
            double m = 0, d = 0;
            for (size_t i = 0; i < n; ++i) {
                m = std::max(m, std::fabs(b[i]));
                d = std::max(d, std::fabs(a[i] - b[i]));
            }
            return m > 0 ? d / m : d;
        };
        EXPECT(std::fabs(r.loss - f.loss) <= 1e-9 * std::fabs(f.loss), "joint loss t=%zu", t);
        EXPECT(r.avg_bits == f.avg_bits && r.sched_b == f.sched_b && r.tau == f.tau, "joint scalars t=%zu", t);
        EXPECT(rel(r.y_hat.data(), f.y_hat.data(), f.y_hat.size()) <= 1e-9, "joint y_hat t=%zu", t);
        EXPECT(rel(r.d_gamma_lo.data(), g.d_gamma_lo.data(), g.d_gamma_lo.size()) <= 1e-9, "d_gamma_lo t=%zu", t);
        EXPECT(rel(r.d_gamma_hi.data(), g.d_gamma_hi.data(), g.d_gamma_hi.size()) <= 1e-9, "d_gamma_hi t=%zu", t);
        EXPECT(rel(r.d_w1.data(), g.d_w1.data(), g.d_w1.size()) <= 1e-9, "d_w1 t=%zu", t);
        EXPECT(rel(r.d_w2.data(), g.d_w2.data(), g.d_w2.size()) <= 1e-9, "d_w2 t=%zu", t);
        EXPECT(rel(r.d_b1.data(), g.d_b1.data(), g.d_b1.size()) <= 1e-9, "d_b1 t=%zu", t);
        std::printf("joint step %zux%zu T=%zu t=%zu: loss %.6e (ref %.6e)\n", out, in, T, t, r.loss, f.loss);
    }
    {  // stage 1
        trainer::MsbForward f = trainer::msb_forward(L, x, y);
        std::vector<double> lo, hi;
        trainer::msb_backward(L, f, x, y, lo, hi);
        auto r = mobi_b200::msb_step(L, x, y);
        double dl = 0, ml = 0;
        for (size_t g = 0; g < lo.size(); ++g) {
            dl = std::max(dl, std::max(std::fabs(r.d_lo[g] - lo[g]), std::fabs(r.d_hi[g] - hi[g])));
            ml = std::max(ml, std::max(std::fabs(lo[g]), std::fabs(hi[g])));
        }
        EXPECT(std::fabs(r.loss - f.loss) <= 1e-9 * f.loss, "msb loss");
        EXPECT(dl <= 1e-9 * ml, "msb clip gradients");
        std::printf("msb step %zux%zu T=%zu: loss %.6e (ref %.6e)\n", out, in, T, r.loss, f.loss);
    }
    return 0;
}

int main() {
    run_case(256, 512, 128, 64, 3);
    run_case(130, 96, 32, 37, 5);
    run_case(32, 32, 128, 128, 1);
    run_joint(192, 320, 48, 7);
    std::printf(fails ? "DROPIN FAIL (%d)\n" : "DROPIN OK\n", fails);
    return fails ? 1 : 0;
}
