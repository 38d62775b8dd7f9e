// mobi_b200.hpp -- header-only C++ shim over the C ABI (mobi_b200.h) with the reference's
// hot-path signatures, for a C++ caller of the MoBiQuant reference (proj/include/mobi).
//
// It is templated on the reference's own types (mobi::Matrix, mobi::slicer::SliceStack,
// mobi::router::RouterState) so it does not depend on the reference headers; include it after
// them.  Errors are rethrown with the reference's exception types: MOBI_EINVAL ->
// std::invalid_argument (what MOBI_CHECK throws), anything else -> std::runtime_error.
//
//   reference call (router.hpp)                       drop-in
//   router::score(x, rs)                        ->    mobi_b200::Layer(stack, rs).score(x)
//   router::forward_elastic(x, st, G, kHard)    ->    layer.forward_elastic(x, G)
//   score -> calibrate_threshold -> gate_hard -> forward_elastic (pipeline.hpp:146-183)
//                                               ->    layer.forward(x, delta, &gates)
//   router::calibrate_threshold(scores, rho)    ->    mobi_b200::calibrate_threshold(scores, rho)
//   router::avg_bits(gates, slice_bits)         ->    mobi_b200::avg_bits(gates, slice_bits)
//   bitplane::permute_by_slice(tokens, masks)   ->    mobi_b200::permute_by_slice(tokens, masks)
//   (multi-GPU)                    ->    mobi_b200::ShardedLayer(stack, rs, comm, rank, P, mode)
//   trainer::joint_forward + joint_backward     ->    mobi_b200::joint_step(layer, x, y_fp, sched, t, opt)
//   (trainer.hpp:203-263, 341-396)                    (one stage-2 calibration step, fp64, on the GPU)
//   trainer::msb_forward + msb_backward         ->    mobi_b200::msb_step(layer, x, y_fp)  (stage 1)
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "mobi_b200.h"

namespace mobi_b200 {

inline void check(int rc) {
    if (rc == MOBI_OK) return;
    if (rc == MOBI_EINVAL) throw std::invalid_argument(mobi_last_error());
    throw std::runtime_error(mobi_last_error());
}

inline uint16_t to_bf16(double d) {
    float f = static_cast<float>(d);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
inline double from_bf16(uint16_t b) {
    uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// Device-resident MoBi layer built from the reference's SliceStack + RouterState.
class Layer {
public:
    // Column-parallel shard: weight rows [row0, row1) of the stack (and their group parameters), full router.
    template <class SliceStack, class RouterState>
    Layer(const SliceStack& st, const RouterState& rs, int device, int64_t row0, int64_t row1)
        : Layer(st, rs, device, row0, row1, 0) {}

    template <class SliceStack, class RouterState>
    Layer(const SliceStack& st, const RouterState& rs, int device = 0) : Layer(st, rs, device, -1, -1, 0) {}

private:
    template <class SliceStack, class RouterState>
    Layer(const SliceStack& st, const RouterState& rs, int device, int64_t row0, int64_t row1, int)
        : device_(device) {
        mobi_layer_desc d{};
        d.out = static_cast<int64_t>(st.rows());
        d.in = static_cast<int64_t>(st.cols());
        d.group_size = static_cast<int64_t>(st.base.group_size);
        d.n_slices = static_cast<int32_t>(st.num_slices());
        bits_.assign(st.slice_bits.begin(), st.slice_bits.end());
        d.slice_bits = bits_.data();
        d.scale = st.base.scale.data();
        d.zero = st.base.zero.data();
        const size_t n = st.rows() * st.cols();
        codes_.resize(n * st.num_slices());
        for (size_t e = 0; e < st.num_slices(); ++e) std::memcpy(codes_.data() + e * n, st.slices[e].vec().data(), n);
        d.codes = codes_.data();
        d.router_hidden = static_cast<int64_t>(rs.hidden_dim());
        d.w1 = rs.w1.data();
        d.b1 = rs.b1.data();
        d.w2 = rs.w2.data();
        d.b2 = rs.b2.data();
        if (row0 >= 0) {
            check(mobi_layer_create_rows(&d, row0, row1, device, &h_));
            d.out = row1 - row0;
        } else {
            check(mobi_layer_create(&d, device, &h_));
        }
        out_ = d.out;
        in_ = d.in;
        nr_ = d.n_slices - 1;
        codes_.clear();
        codes_.shrink_to_fit();
    }

public:
    ~Layer() { mobi_layer_destroy(h_); }
    Layer(const Layer&) = delete;
    Layer& operator=(const Layer&) = delete;

    // router::score (router.hpp:63): S [T, E-1]
    template <class Matrix>
    Matrix score(const Matrix& x) {
        Dev<uint16_t> dx(upload_bf16(x));
        Dev<float> ds(x.rows() * nr_);
        check(mobi_score(h_, dx.p, static_cast<int64_t>(x.rows()), ds.p, nullptr));
        std::vector<float> s = ds.download();
        Matrix out(x.rows(), static_cast<size_t>(nr_));
        for (size_t i = 0; i < s.size(); ++i) out[i] = s[i];
        return out;
    }

    // router::forward_elastic(x, st, gates, kHard) (router.hpp:105): gates [T, E-1] binary
    template <class Matrix>
    Matrix forward_elastic(const Matrix& x, const Matrix& gates) {
        if (gates.rows() != x.rows() || static_cast<int64_t>(gates.cols()) != nr_)
            throw std::invalid_argument("forward_elastic: gate shape " + std::to_string(gates.rows()) + "x" +
                                        std::to_string(gates.cols()) + " != " + std::to_string(x.rows()) + "x" +
                                        std::to_string(nr_));
        std::vector<uint8_t> m(x.rows(), 1);
        for (size_t t = 0; t < x.rows(); ++t)
            for (int64_t j = 0; j < nr_; ++j) {
                const double g = gates(t, static_cast<size_t>(j));
                if (g != 0.0 && g != 1.0) throw std::invalid_argument("forward_elastic: hard gate not binary");
                if (g == 1.0) m[t] |= static_cast<uint8_t>(1u << (j + 1));
            }
        Dev<uint16_t> dx(upload_bf16(x));
        Dev<uint8_t> dm(m);
        Dev<uint16_t> dy(x.rows() * static_cast<size_t>(out_));
        check(mobi_forward_masked(h_, dx.p, static_cast<int64_t>(x.rows()), dm.p, dy.p, nullptr));
        return to_matrix<Matrix>(dy.download(), x.rows());
    }

    // score -> gate_hard(delta) -> forward_elastic(kHard); optionally returns the hard gates
    template <class Matrix>
    Matrix forward(const Matrix& x, double delta, Matrix* gates_out = nullptr) {
        std::vector<uint16_t> hx = to_bf16_vec(x);
        std::vector<uint16_t> hy(x.rows() * static_cast<size_t>(out_));
        std::vector<uint8_t> hm(x.rows());
        check(mobi_forward_host(h_, hx.data(), static_cast<int64_t>(x.rows()), static_cast<float>(delta), hy.data(),
                                hm.data(), nullptr));
        if (gates_out) {
            *gates_out = Matrix(x.rows(), static_cast<size_t>(nr_));
            for (size_t t = 0; t < x.rows(); ++t)
                for (int64_t j = 0; j < nr_; ++j) (*gates_out)(t, static_cast<size_t>(j)) = (hm[t] >> (j + 1)) & 1u;
        }
        return to_matrix<Matrix>(hy, x.rows());
    }

    mobi_layer_t handle() const { return h_; }

private:
    template <class T>
    struct Dev {
        T* p = nullptr;
        size_t n = 0;
        explicit Dev(size_t n_) : n(n_) {
            if (cudaMalloc(&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
        }
        explicit Dev(const std::vector<T>& h) : Dev(h.size()) {
            if (n && cudaMemcpy(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
                throw std::runtime_error("cudaMemcpy failed");
        }
        ~Dev() { cudaFree(p); }
        std::vector<T> download() const {
            std::vector<T> h(n);
            if (n && cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess)
                throw std::runtime_error("cudaMemcpy failed");
            return h;
        }
    };
    template <class Matrix>
    static std::vector<uint16_t> to_bf16_vec(const Matrix& x) {
        std::vector<uint16_t> v(x.size());
        for (size_t i = 0; i < x.size(); ++i) v[i] = to_bf16(x[i]);
        return v;
    }
    template <class Matrix>
    std::vector<uint16_t> upload_bf16(const Matrix& x) {
        if (static_cast<int64_t>(x.cols()) != in_)
            throw std::invalid_argument("score: token dim " + std::to_string(x.cols()) + " != router input dim " +
                                        std::to_string(in_));
        return to_bf16_vec(x);
    }
    template <class Matrix>
    Matrix to_matrix(const std::vector<uint16_t>& y, size_t T) const {
        Matrix out(T, static_cast<size_t>(out_));
        for (size_t i = 0; i < y.size(); ++i) out[i] = from_bf16(y[i]);
        return out;
    }

    mobi_layer_t h_ = nullptr;
    int device_ = 0;
    int64_t out_ = 0, in_ = 0, nr_ = 0;
    std::vector<int32_t> bits_;
    std::vector<uint8_t> codes_;
    friend class ShardedLayer;
};

namespace detail {
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t n_) : n(n_) {
        if (cudaMalloc(&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    }
    explicit DevBuf(const std::vector<T>& h) : DevBuf(h.size()) {
        if (n && cudaMemcpy(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
            throw std::runtime_error("cudaMemcpy failed");
    }
    ~DevBuf() { cudaFree(p); }
    std::vector<T> download() const {
        std::vector<T> h(n);
        if (n && cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess)
            throw std::runtime_error("cudaMemcpy failed");
        return h;
    }
};
}  // namespace detail

// router::calibrate_threshold (router.hpp:167-174) on the GPU (device radix select): scores are taken
// as fp32 -- what the device router produces -- so doubles that are not float-representable go
// through the reference's own host algorithm instead, keeping the result identical.
inline double calibrate_threshold(const std::vector<double>& scores, double rho) {
    if (scores.empty()) throw std::invalid_argument("calibrate_threshold: empty score sample");
    std::vector<float> f(scores.size());
    bool exact = true;
    for (size_t i = 0; i < scores.size(); ++i) {
        f[i] = static_cast<float>(scores[i]);
        exact = exact && static_cast<double>(f[i]) == scores[i];
    }
    if (!exact) {
        if (rho < 0.0 || rho > 1.0) throw std::invalid_argument("calibrate_threshold: rho outside [0,1]");
        std::vector<double> s(scores);
        const size_t k = static_cast<size_t>(rho * static_cast<double>(s.size()) + 1e-9);
        if (k >= s.size()) return *std::min_element(s.begin(), s.end()) - 1.0;
        std::nth_element(s.begin(), s.begin() + static_cast<std::ptrdiff_t>(k), s.end(), std::greater<double>());
        return s[k];
    }
    detail::DevBuf<float> d(f);
    double delta = 0.0;
    check(mobi_calibrate_threshold(d.p, static_cast<int64_t>(f.size()), rho, &delta, nullptr));
    return delta;
}

// router::avg_bits (router.hpp:135-150): mean over tokens of b_1 + sum_j 1(G[t,j] > 0.5) * b_{j+1}
template <class Matrix>
double avg_bits(const Matrix& gates, const std::vector<int>& slice_bits) {
    if (slice_bits.size() != gates.cols() + 1)
        throw std::invalid_argument("avg_bits: " + std::to_string(gates.cols()) + " gate columns for " +
                                    std::to_string(slice_bits.size()) + " slices");
    if (gates.rows() == 0) return static_cast<double>(slice_bits[0]);
    std::vector<uint8_t> m(gates.rows(), 1);
    for (size_t t = 0; t < gates.rows(); ++t)
        for (size_t j = 0; j < gates.cols(); ++j)
            if (gates(t, j) > 0.5) m[t] |= static_cast<uint8_t>(1u << (j + 1));
    detail::DevBuf<uint8_t> dm(m);
    std::vector<int32_t> b(slice_bits.begin(), slice_bits.end());
    double out = 0.0;
    check(mobi_avg_bits(dm.p, static_cast<int64_t>(m.size()), b.data(), static_cast<int32_t>(b.size()), &out, nullptr));
    return out;
}

// trainer::joint_forward + trainer::joint_backward (trainer.hpp:203-263, 341-396) on the GPU, fp64.
// QuantLayer / BudgetSchedule / JointOptions are the reference's types (trainer.hpp:45-51, 136-169,
// 182-184); the result carries JointForward's scalars and y_hat and JointGrads' fields.
template <class Matrix>
struct JointStep {
    double data_term = 0, reg_term = 0, avg_bits = 0, sched_b = 0, loss = 0, tau = 0;
    bool hard = false;
    Matrix y_hat;
    std::vector<double> d_gamma_lo, d_gamma_hi, d_b1, d_b2;
    Matrix d_w1, d_w2;
};

template <class QuantLayer, class Matrix, class Schedule, class Options>
JointStep<Matrix> joint_step(const QuantLayer& L, const Matrix& x, const Matrix& y_fp, const Schedule& sc, size_t t,
                             const Options& opt, bool backward = true) {
    const int64_t out = (int64_t)L.w.rows(), in = (int64_t)L.w.cols(), T = (int64_t)x.rows();
    if (x.cols() != L.w.cols()) throw std::invalid_argument("joint_forward: input dim mismatch");
    if (y_fp.rows() != x.rows() || y_fp.cols() != L.w.rows())
        throw std::invalid_argument("joint_forward: reference output shape mismatch");
    const int64_t h = (int64_t)L.rs.w1.cols(), nr = (int64_t)L.rs.w2.cols();
    std::vector<int32_t> bits(L.slice_bits.begin(), L.slice_bits.end());
    auto vec = [](const Matrix& m) { return std::vector<double>(m.data(), m.data() + m.size()); };
    detail::DevBuf<double> w(vec(L.w)), dx(vec(x)), dy(vec(y_fp)), w1(vec(L.rs.w1)), b1(L.rs.b1), w2(vec(L.rs.w2)),
        b2(L.rs.b2), yh(static_cast<size_t>(T * out)), gw1(static_cast<size_t>(in * h)), gb1(static_cast<size_t>(h)),
        gw2(static_cast<size_t>(h * nr)), gb2(static_cast<size_t>(nr));
    mobi_budget_schedule bs{sc.b_init, sc.b_target, (int64_t)sc.total_steps, (int32_t)sc.shape, sc.reg_weight};
    mobi_joint_scalars r{};
    JointStep<Matrix> o;
    const size_t ng = L.clip.gamma_lo.size();
    o.d_gamma_lo.assign(ng, 0.0);
    o.d_gamma_hi.assign(ng, 0.0);
    check(mobi_joint_step(w.p, out, in, (int64_t)L.group_size, bits.data(), (int32_t)bits.size(), L.clip.gamma_lo.data(),
                          L.clip.gamma_hi.data(), w1.p, b1.p, w2.p, b2.p, h, dx.p, dy.p, T, &bs, (int64_t)t,
                          opt.force_gates_on ? 1 : 0, yh.p, &r, backward ? o.d_gamma_lo.data() : nullptr,
                          o.d_gamma_hi.data(), gw1.p, gb1.p, gw2.p, gb2.p, nullptr));
    o.data_term = r.data_term;
    o.reg_term = r.reg_term;
    o.avg_bits = r.avg_bits;
    o.sched_b = r.sched_b;
    o.loss = r.loss;
    o.tau = r.tau;
    o.hard = opt.force_gates_on || t == sc.total_steps;
    auto mat = [](const std::vector<double>& v, size_t rows, size_t cols) {
        Matrix m(rows, cols);
        std::copy(v.begin(), v.end(), m.data());
        return m;
    };
    o.y_hat = mat(yh.download(), (size_t)T, (size_t)out);
    if (backward) {
        o.d_w1 = mat(gw1.download(), (size_t)in, (size_t)h);
        o.d_w2 = mat(gw2.download(), (size_t)h, (size_t)nr);
        o.d_b1 = gb1.download();
        o.d_b2 = gb2.download();
    }
    return o;
}

// trainer::msb_forward + trainer::msb_backward (trainer.hpp:404-426) on the GPU, fp64: loss, y_msb and
// the clip gradients of the stage-1 step
template <class Matrix>
struct MsbStep {
    double loss = 0;
    Matrix y_msb;
    std::vector<double> d_lo, d_hi;
};

template <class QuantLayer, class Matrix>
MsbStep<Matrix> msb_step(const QuantLayer& L, const Matrix& x, const Matrix& y_fp) {
    const int64_t out = (int64_t)L.w.rows(), in = (int64_t)L.w.cols(), T = (int64_t)x.rows();
    auto vec = [](const Matrix& m) { return std::vector<double>(m.data(), m.data() + m.size()); };
    detail::DevBuf<double> w(vec(L.w)), dx(vec(x)), dy(vec(y_fp)), y(static_cast<size_t>(T * out));
    MsbStep<Matrix> o;
    o.d_lo.assign(L.clip.gamma_lo.size(), 0.0);
    o.d_hi.assign(L.clip.gamma_hi.size(), 0.0);
    check(mobi_msb_step(w.p, out, in, (int64_t)L.group_size, (int32_t)L.slice_bits[0], L.clip.gamma_lo.data(),
                        L.clip.gamma_hi.data(), dx.p, dy.p, T, y.p, &o.loss, o.d_lo.data(), o.d_hi.data(), nullptr));
    const std::vector<double> h = y.download();
    o.y_msb = Matrix((size_t)T, (size_t)out);
    std::copy(h.begin(), h.end(), o.y_msb.data());
    return o;
}

// bitplane::permute_by_slice (bitplane.hpp:178-201): stable sort of tokens by mask
struct Permutation {
    std::vector<size_t> perm, inverse;                    // perm[i] = source row, inverse[src] = i
    std::vector<std::pair<uint8_t, size_t>> groups;      // (mask, run length), ascending mask
};
template <class Matrix>
Permutation permute_by_slice(const Matrix& tokens, const std::vector<uint8_t>& masks, Matrix* permuted = nullptr) {
    if (tokens.rows() != masks.size())
        throw std::invalid_argument("permute_by_slice: " + std::to_string(masks.size()) + " masks for " +
                                    std::to_string(tokens.rows()) + " tokens");
    const int64_t T = static_cast<int64_t>(masks.size());
    Permutation out;
    if (T == 0) return out;
    detail::DevBuf<uint8_t> dm(masks);
    detail::DevBuf<int32_t> dp(masks.size()), di(masks.size());
    std::vector<uint8_t> gm(256);
    std::vector<int64_t> gl(256);
    int64_t ng = 0;
    check(mobi_permute_by_slice(dm.p, T, dp.p, di.p, gm.data(), gl.data(), &ng, nullptr));
    const std::vector<int32_t> p = dp.download(), iv = di.download();
    out.perm.assign(p.begin(), p.end());
    out.inverse.assign(iv.begin(), iv.end());
    for (int64_t g = 0; g < ng; ++g) out.groups.emplace_back(gm[g], static_cast<size_t>(gl[g]));
    if (permuted) {
        *permuted = Matrix(tokens.rows(), tokens.cols());
        for (size_t i = 0; i < out.perm.size(); ++i)
            for (size_t c = 0; c < tokens.cols(); ++c) (*permuted)(i, c) = tokens(out.perm[i], c);
    }
    return out;
}

// A layer partitioned over the ranks of an NCCL communicator (mobi_layer_create_sharded): COLUMN mode
// returns the full [T, out] on every rank, TOKEN mode this rank's tokens.
class ShardedLayer {
public:
    template <class SliceStack, class RouterState>
    ShardedLayer(const SliceStack& st, const RouterState& rs, void* nccl_comm, int rank, int nranks,
                 int mode = MOBI_SHARD_COLUMN, int device = 0)
        : mode_(mode) {
        mobi_layer_desc d{};
        d.out = static_cast<int64_t>(st.rows());
        d.in = static_cast<int64_t>(st.cols());
        d.group_size = static_cast<int64_t>(st.base.group_size);
        d.n_slices = static_cast<int32_t>(st.num_slices());
        std::vector<int32_t> bits(st.slice_bits.begin(), st.slice_bits.end());
        d.slice_bits = bits.data();
        d.scale = st.base.scale.data();
        d.zero = st.base.zero.data();
        const size_t n = st.rows() * st.cols();
        std::vector<uint8_t> codes(n * st.num_slices());
        for (size_t e = 0; e < st.num_slices(); ++e) std::memcpy(codes.data() + e * n, st.slices[e].vec().data(), n);
        d.codes = codes.data();
        d.router_hidden = static_cast<int64_t>(rs.hidden_dim());
        d.w1 = rs.w1.data();
        d.b1 = rs.b1.data();
        d.w2 = rs.w2.data();
        d.b2 = rs.b2.data();
        check(mobi_layer_create_sharded(&d, nccl_comm, rank, nranks, mode, device, &h_));
        out_ = d.out;
        in_ = d.in;
    }
    ~ShardedLayer() { mobi_layer_destroy(h_); }
    ShardedLayer(const ShardedLayer&) = delete;
    ShardedLayer& operator=(const ShardedLayer&) = delete;

    // score -> gate_hard(delta) -> forward_elastic on this rank's rows, then the all-gather (COLUMN)
    template <class Matrix>
    Matrix forward(const Matrix& x, double delta) {
        if (static_cast<int64_t>(x.cols()) != in_)
            throw std::invalid_argument("score: token dim " + std::to_string(x.cols()) + " != router input dim " +
                                        std::to_string(in_));
        std::vector<uint16_t> hx(x.size());
        for (size_t i = 0; i < x.size(); ++i) hx[i] = to_bf16(x[i]);
        detail::DevBuf<uint16_t> dx(hx), dy(x.rows() * static_cast<size_t>(out_));
        check(mobi_forward_sharded(h_, dx.p, static_cast<int64_t>(x.rows()), static_cast<float>(delta), dy.p, nullptr,
                                   nullptr));
        const std::vector<uint16_t> hy = dy.download();
        Matrix y(x.rows(), static_cast<size_t>(out_));
        for (size_t i = 0; i < hy.size(); ++i) y[i] = from_bf16(hy[i]);
        return y;
    }

private:
    mobi_layer_t h_ = nullptr;
    int mode_ = MOBI_SHARD_COLUMN;
    int64_t out_ = 0, in_ = 0;
};

}  // namespace mobi_b200
