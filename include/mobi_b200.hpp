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
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
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
};

}  // namespace mobi_b200
