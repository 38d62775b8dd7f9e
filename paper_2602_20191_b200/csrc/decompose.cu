// decompose.cu -- GPU slice decomposition: base params from clipping
// (qcore.hpp:75-146, GroupStats + params_from_clip) and the recursive residual decomposition
// (slicer.hpp:69-113), bit-exact with the reference.
//
// Exactness: every double operation is an explicit round-to-nearest intrinsic (no FMA
// contraction; the file is also compiled with -fmad=false), the operation order is the
// reference's, and the only transcendental (sigmoid of the clip gamma) is evaluated on the
// host with the same libm the reference uses and passed in.
#include <cmath>

#include "mobi_internal.cuh"

namespace mobi {
namespace {

// one warp per (row, group): stats (warp min / max) -> params -> all slices of the group's elements,
// lanes striding the group (coalesced); per-element arithmetic is the reference's, in its order
__global__ void decompose_kernel(const double* __restrict__ w, int64_t out, int64_t in, int64_t gs,
                                 int64_t G, const int32_t* __restrict__ bits_dev, int E, double sq_lo,
                                 double sq_hi, const double* __restrict__ sq_lo_g,
                                 const double* __restrict__ sq_hi_g, uint8_t* __restrict__ codes,
                                 double* __restrict__ scale, double* __restrict__ zero,
                                 double* __restrict__ stats, unsigned long long* __restrict__ clamp_counts) {
    const int lane = threadIdx.x & 31;
    const int64_t gi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // warp-uniform
    if (gi >= out * G) return;
    const int64_t r = gi / G, g = gi % G;
    const int64_t c0 = g * gs, c1 = min(in, c0 + gs);
    const double* row = w + r * in;
    double mn = row[c0], mx = row[c0];
    for (int64_t c = c0 + lane; c < c1; c += 32) {
        const double v = row[c];
        mn = fmin(mn, v);
        mx = fmax(mx, v);
    }
    for (int o = 16; o; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    // GroupStats::ref = min(max(0, min), max); clip_lo/hi; params_from_clip
    const double lo0 = mn > 0.0 ? mn : 0.0;
    const double ref = mx < lo0 ? mx : lo0;
    if (sq_lo_g) {  // per-group clip (a calibration step's gammas)
        sq_lo = sq_lo_g[gi];
        sq_hi = sq_hi_g[gi];
    }
    if (stats && lane == 0) {  // GroupStats min / max / ref, [3][out*G]
        stats[gi] = mn;
        stats[out * G + gi] = mx;
        stats[2 * out * G + gi] = ref;
    }
    const double lo = __dadd_rn(ref, __dmul_rn(sq_lo, __dsub_rn(mn, ref)));
    const double hi = __dadd_rn(ref, __dmul_rn(sq_hi, __dsub_rn(mx, ref)));
    const int b1 = bits_dev[0];
    double s = __ddiv_rn(__dsub_rn(hi, lo), (double)((1 << b1) - 1));
    if (!(s > 1e-8)) s = 1e-8;
    const double z1 = __ddiv_rn(-lo, s);
    if (lane == 0) {
        scale[gi] = s;
        zero[gi] = z1;
    }
    unsigned cl[MOBI_MAX_SLICES] = {};
    for (int64_t c = c0 + lane; c < c1; c += 32) {
        double v = row[c];
        int bb = 0;
        for (int e = 0; e < E; ++e) {
            const int be = bits_dev[e];
            const double sc = e == 0 ? s : s * ldexp(1.0, -bb);  // exact power-of-two scaling
            const double z = e == 0 ? z1 : ldexp(1.0, be - 1);
            const double qmax = (double)((1 << be) - 1);
            double u = floor(__dadd_rn(__ddiv_rn(v, sc), z));
            if (u < 0.0 || u > qmax) {
                ++cl[e];
                u = fmin(fmax(u, 0.0), qmax);
            }
            codes[(int64_t)e * out * in + r * in + c] = (uint8_t)u;
            v = __dsub_rn(v, __dmul_rn(sc, __dadd_rn(__dsub_rn(u, z), 0.5)));
            bb += be;
        }
    }
    for (int e = 0; e < E; ++e) {
        unsigned n = cl[e];
        for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        if (lane == 0 && n) atomicAdd(&clamp_counts[e], (unsigned long long)n);
    }
}

}  // namespace

int launch_decompose(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* bits, int32_t E,
                     double gamma, uint8_t* codes, double* scale, double* zero, int64_t* clamp_counts_host,
                     cudaStream_t st) {
    if (E < 1 || E > MOBI_MAX_SLICES) return set_error(MOBI_EINVAL, "decompose: slice_bits is empty or too long");
    int total = 0;
    for (int e = 0; e < E; ++e) {
        if (bits[e] < 1 || bits[e] > 8)
            return set_error(MOBI_EINVAL, "decompose: slice bit width " + std::to_string(bits[e]) + " out of [1,8]");
        total += bits[e];
    }
    if (total > 8)
        return set_error(MOBI_EINVAL, "decompose: total bits " + std::to_string(total) + " exceed the 8-bit code budget");
    if (out <= 0 || in <= 0 || gs <= 0) return set_error(MOBI_EINVAL, "decompose: empty weight");
    // squash(gamma) = sigmoid(gamma) on the host (common.hpp:125-131), identical libm to the reference
    const double sq = gamma >= 0.0 ? 1.0 / (1.0 + std::exp(-gamma)) : std::exp(gamma) / (1.0 + std::exp(gamma));
    const int64_t G = cdiv(in, gs);
    int32_t* bits_dev = nullptr;
    unsigned long long* cc = nullptr;
    MOBI_CUDA(cudaMallocAsync(&bits_dev, sizeof(int32_t) * E, st));
    MOBI_CUDA(cudaMallocAsync(&cc, sizeof(unsigned long long) * MOBI_MAX_SLICES, st));
    MOBI_CUDA(cudaMemcpyAsync(bits_dev, bits, sizeof(int32_t) * E, cudaMemcpyHostToDevice, st));
    MOBI_CUDA(cudaMemsetAsync(cc, 0, sizeof(unsigned long long) * MOBI_MAX_SLICES, st));
    decompose_kernel<<<(unsigned)cdiv(out * G * 32, 128), 128, 0, st>>>(w, out, in, gs, G, bits_dev, E, sq, sq, nullptr,
                                                                   nullptr, codes, scale, zero, nullptr, cc);
    MOBI_LAUNCH_CHECK();
    unsigned long long h[MOBI_MAX_SLICES];
    MOBI_CUDA(cudaMemcpyAsync(h, cc, sizeof(h), cudaMemcpyDeviceToHost, st));
    MOBI_CUDA(cudaStreamSynchronize(st));
    if (clamp_counts_host)
        for (int e = 0; e < E; ++e) clamp_counts_host[e] = (int64_t)h[e];
    cudaFreeAsync(bits_dev, st);
    cudaFreeAsync(cc, st);
    return MOBI_OK;
}

// The calibration step's decomposition (trainer.hpp:166-168 QuantLayer::decompose): per-group clip
// squashes sq_lo_g / sq_hi_g (device, evaluated on the host with the reference's libm), the group
// statistics written to stats [3][out*G].  bits_dev is device memory; asynchronous.
int launch_decompose_clip(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* bits_dev, int32_t E,
                          const double* sq_lo_g, const double* sq_hi_g, uint8_t* codes, double* scale, double* zero,
                          double* stats, unsigned long long* clamp_counts, cudaStream_t st) {
    const int64_t G = cdiv(in, gs);
    decompose_kernel<<<(unsigned)cdiv(out * G * 32, 128), 128, 0, st>>>(w, out, in, gs, G, bits_dev, E, 0.0, 0.0, sq_lo_g,
                                                                   sq_hi_g, codes, scale, zero, stats, clamp_counts);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

}  // namespace mobi
