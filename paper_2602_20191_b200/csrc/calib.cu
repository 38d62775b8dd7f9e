// calib.cu -- SURVEY 8(f)-4: one stage-2 calibration step on the GPU, in fp64 like the reference:
// trainer.hpp:203-263 joint_forward (decompose -> per-slice dequant + X·W_eᵀ -> router MLP ->
// gate_soft -> gated sum -> MSE + budget regulariser) and trainer.hpp:341-396 joint_backward
// (slice cotangents -> per-group clip gradients, accumulate_clip_grads trainer.hpp:276-339; router
// gradients through gate_soft / SiLU).
//
// This is offline calibration, not the inference hot path: it runs once per layer per optimiser
// step.  The matrix products are a shared-memory tiled fp64 tensor-core GEMM (DMMA m8n8k4, 128x64
// CTA tiles, 3-stage cp.async ring; a fixed k order -> deterministic); the reductions the reference performs in a fixed order
// (per-group clip sums, column sums of the bias gradients) keep that order (one thread per group /
// column), every other reduction is a fixed two-level tree, so repeated steps are bit-identical.
// The per-group sigmoid of the clip gammas is evaluated on the host with the reference's libm
// (decompose.cu), the decomposition itself is decompose.cu's bit-exact kernel.
#include <cmath>
#include <vector>

#include "mobi_internal.cuh"

namespace mobi {

int launch_decompose_clip(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* bits_dev, int32_t E,
                          const double* sq_lo_g, const double* sq_hi_g, uint8_t* codes, double* scale, double* zero,
                          double* stats, unsigned long long* clamp_counts, cudaStream_t st);

namespace {

constexpr int kBM = 128, kBN = 64, kTk = 16, kStages = 3, kGemmThreads = 256, kRedThreads = 256;

__device__ __forceinline__ double sigmoid_d(double v) {  // common.hpp:125-131
    if (v >= 0.0) return 1.0 / (1.0 + exp(-v));
    const double e = exp(v);
    return e / (1.0 + e);
}

// C[i][j] = Σ_k A(i,k)·B(k,j) (+ bias[j]); A(i,k) = A[i·sai + k·sak], B(k,j) = B[k·sbk + j·sbj].
// fp64 tensor cores: mma.sync m8n8k4 (DMMA), 128x64 CTA tile, 8 warps of 32x32 (4x4 MMA tiles each);
// k staged 16 at a time through a kStages-deep cp.async ring (8-byte element copies, so any operand
// stride lands in the same k-major tile; out-of-range elements are zero-filled by the copy).
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}

// +8 doubles per row: a fragment load's four k rows take two bank halves (two wavefronts, the minimum
// for 32 doubles); the column index is XOR-swizzled by (k >> 1) & 7 inside each 8-column group so the
// k-fast copies of a k-contiguous operand also spread over all banks
constexpr int kAStride = kBM + 8, kBStride = kBN + 8;
constexpr int kStageDoubles = kTk * (kAStride + kBStride);
constexpr size_t kGemmSmem = (size_t)kStages * kStageDoubles * sizeof(double);

__global__ void __launch_bounds__(kGemmThreads, 1) dgemm_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A,
                                                                int64_t sai, int64_t sak, const double* __restrict__ B,
                                                                int64_t sbk, int64_t sbj, const double* __restrict__ bias,
                                                                double* __restrict__ C, int64_t ldc) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
    const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
    const int64_t i0 = (int64_t)blockIdx.y * kBM, j0 = (int64_t)blockIdx.x * kBN;
    const int64_t nkt = (K + kTk - 1) / kTk;
    // a thread's copies in one stage differ by a fixed step along one dimension: (row, k) of copy l is
    // (r0 + l·dr, k0 + c0 + l·dc), with the unit-stride dimension walked by consecutive threads
    const bool a_kf = sak == 1, b_kf = sbk == 1 && sbj != 1;
    const int a_r0 = a_kf ? tid / kTk : tid % kBM, a_c0 = a_kf ? tid % kTk : tid / kBM;
    const int a_dr = a_kf ? kGemmThreads / kTk : 0, a_dc = a_kf ? 0 : kGemmThreads / kBM;
    const int b_r0 = b_kf ? tid / kTk : tid % kBN, b_c0 = b_kf ? tid % kTk : tid / kBN;
    const int b_dr = b_kf ? kGemmThreads / kTk : 0, b_dc = b_kf ? 0 : kGemmThreads / kBN;
    auto load = [&](int64_t kt) {
        double* As = smem + (kt % kStages) * kStageDoubles;
        double* Bs = As + kTk * kAStride;
        const int64_t k0 = kt * kTk;
#pragma unroll
        for (int l = 0; l < kBM * kTk / kGemmThreads; ++l) {
            const int ii = a_r0 + l * a_dr, kk = a_c0 + l * a_dc;
            const int64_t i = i0 + ii, k = k0 + kk;
            const bool ok = i < M && k < K;
            cp_async8(As + kk * kAStride + (ii ^ ((kk >> 1) & 7)), ok ? A + i * sai + k * sak : A, ok);
        }
#pragma unroll
        for (int l = 0; l < kBN * kTk / kGemmThreads; ++l) {
            const int jj = b_r0 + l * b_dr, kb = b_c0 + l * b_dc;
            const int64_t j = j0 + jj, k = k0 + kb;
            const bool ok = j < N && k < K;
            cp_async8(Bs + kb * kBStride + (jj ^ ((kb >> 1) & 7)), ok ? B + k * sbk + j * sbj : B, ok);
        }
    };
    double acc[4][4][2] = {};
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nkt) load(s);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int64_t kt = 0; kt < nkt; ++kt) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kStages - 2));
        __syncthreads();  // stage kt landed for every thread; stage kt-1 is free to refill
        if (kt + kStages - 1 < nkt) load(kt + kStages - 1);
        asm volatile("cp.async.commit_group;\n" ::);
        const double* As = smem + (kt % kStages) * kStageDoubles;
        const double* Bs = As + kTk * kAStride;
#pragma unroll
        for (int ks = 0; ks < kTk; ks += 4) {
            double a[4], b[4];
            const int sw = ((ks + q) >> 1) & 7;
#pragma unroll
            for (int m = 0; m < 4; ++m) a[m] = As[(ks + q) * kAStride + ((wm + m * 8 + g) ^ sw)];  // A: row g, col q
#pragma unroll
            for (int n = 0; n < 4; ++n) b[n] = Bs[(ks + q) * kBStride + ((wn + n * 8 + g) ^ sw)];  // B: row q, col g
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int n = 0; n < 4; ++n) dmma(acc[m][n], a[m], b[n]);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int64_t i = i0 + wm + m * 8 + g;
        if (i >= M) continue;
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // C frag: row g, cols 2q, 2q+1
                const int64_t j = j0 + wn + n * 8 + 2 * q + h;
                if (j < N) C[i * ldc + j] = bias ? acc[m][n][h] + bias[j] : acc[m][n][h];
            }
    }
}

// dP_e = diag(g_e)·resid (trainer.hpp:351-357): the gate-scaled operand of dL/dW_e
__global__ void row_scale_kernel(const double* __restrict__ resid, const double* __restrict__ gates, int nr, int col,
                                 int64_t T, int64_t out, double* __restrict__ dst) {
    const int64_t n = T * out;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = resid[i] * gates[(i / out) * nr + col];
}

// W_e = slice_params(e) dequantize_centered: s·2^{-before}·(code − z + ½), z = zero[g] for e = 1,
// 2^{b_e−1} otherwise (qcore.hpp:180-197, slicer.hpp:51-61)
__global__ void dequant_slice_kernel(const uint8_t* __restrict__ codes, const double* __restrict__ scale,
                                     const double* __restrict__ zero, int64_t out, int64_t in, int64_t gs, int64_t G,
                                     double unit, double mid, int first, double* __restrict__ W) {
    const int64_t n = out * in;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / in, c = idx % in, g = r * G + c / gs;
        const double z = first ? zero[g] : mid;
        W[idx] = (scale[g] * unit) * ((double)codes[idx] - z + 0.5);
    }
}

__global__ void silu_kernel(const double* __restrict__ pre, double* __restrict__ act, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        act[i] = pre[i] * sigmoid_d(pre[i]);
}

// gate_soft (router.hpp:79-90): sigmoid(tau·S), or the indicator 1(S > 0) at t = L; all-ones for the
// force_gates_on ablation (trainer.hpp:221-226)
__global__ void gates_kernel(const double* __restrict__ s, double* __restrict__ g, int64_t n, double tau, int mode) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        g[i] = mode == 2 ? 1.0 : (mode == 1 ? (s[i] > 0.0 ? 1.0 : 0.0) : sigmoid_d(tau * s[i]));
}

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += red[i];
    return t;
}

// ŷ = P_1 + Σ_e g_e ⊙ P_e with the reference's skip / plain-add / scaled-add branches
// (trainer.hpp:246-258); per-block partial sums of (ŷ − y)² (one block per token row)
__global__ void __launch_bounds__(kRedThreads) combine_kernel(const double* __restrict__ P, int64_t TO, int E,
                                                              const double* __restrict__ gates, int nr, int64_t out,
                                                              const double* __restrict__ y_fp, double* __restrict__ y_hat,
                                                              double* __restrict__ partial) {
    __shared__ double red[kRedThreads / 32];
    const int64_t i = blockIdx.x;
    double sq = 0.0;
    for (int64_t j = threadIdx.x; j < out; j += blockDim.x) {
        const int64_t o = i * out + j;
        double y = P[o];
        for (int e = 2; e <= E; ++e) {
            const double g = gates[i * nr + e - 2];
            if (g == 0.0) continue;
            y += g == 1.0 ? P[(int64_t)(e - 1) * TO + o] : g * P[(int64_t)(e - 1) * TO + o];
        }
        y_hat[o] = y;
        const double d = y - y_fp[o];
        sq += d * d;
    }
    const double t = block_sum(sq, red);
    if (threadIdx.x == 0) partial[i] = t;
}

// one block: Σ partial (data term), ||G||₁, Σ_i bits_i (router::avg_bits, router.hpp:135-150)
__global__ void __launch_bounds__(kRedThreads) scalars_kernel(const double* __restrict__ partial, int64_t T,
                                                              const double* __restrict__ gates, int nr,
                                                              const int32_t* __restrict__ bits, double* __restrict__ out3) {
    __shared__ double red[kRedThreads / 32];
    double a = 0.0, l1 = 0.0, nb = 0.0;
    for (int64_t i = threadIdx.x; i < T; i += blockDim.x) {
        a += partial[i];
        double b = (double)bits[0];
        for (int e = 0; e < nr; ++e) {
            const double g = gates[i * nr + e];
            l1 += g;
            if (g > 0.5) b += (double)bits[e + 1];
        }
        nb += b;
    }
    a = block_sum(a, red);
    l1 = block_sum(l1, red);
    nb = block_sum(nb, red);
    if (threadIdx.x == 0) {
        out3[0] = a;
        out3[1] = l1;
        out3[2] = nb;
    }
}

__global__ void resid_kernel(const double* __restrict__ y_hat, const double* __restrict__ y_fp, double c,
                             double* __restrict__ resid, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        resid[i] = c * (y_hat[i] - y_fp[i]);
}

// accumulate_clip_grads (trainer.hpp:276-301) for slice e: one thread per (row, group), the group's
// elements in the reference's order, slices accumulated in order across launches
__global__ void clip_accum_kernel(const double* __restrict__ dm, const uint8_t* __restrict__ codes, int64_t out,
                                  int64_t in, int64_t gs, int64_t G, double unit, double mid, double qmax1, int first,
                                  double* __restrict__ d_lo, double* __restrict__ d_hi, double* __restrict__ s1) {
    const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= out * G) return;
    const int64_t r = gi / G, c0 = (gi % G) * gs, c1 = min(in, c0 + gs);
    double lo = d_lo[gi], hi = d_hi[gi], s = 0.0;
    for (int64_t c = c0; c < c1; ++c) {
        const double d = dm[r * in + c];
        if (first) s += d;
        if (d == 0.0) continue;
        const double frame = ((double)codes[r * in + c] - mid + 0.5) * unit;
        hi += d * frame / qmax1;
        if (first)
            lo += d * (1.0 - frame / qmax1);
        else
            lo -= d * frame / qmax1;
    }
    d_lo[gi] = lo;
    d_hi[gi] = hi;
    if (first) s1[gi] = s;
}

// d(clip)/d(gamma) (trainer.hpp:303-338), epsilon-floored groups through slice 1 only
__global__ void gamma_grad_kernel(const double* __restrict__ stats, int64_t n, const double* __restrict__ sq_lo,
                                  const double* __restrict__ sq_hi, const double* __restrict__ sg_lo,
                                  const double* __restrict__ sg_hi, double qmax1, const double* __restrict__ d_lo,
                                  const double* __restrict__ d_hi, const double* __restrict__ s1,
                                  double* __restrict__ dg_lo, double* __restrict__ dg_hi) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const double mn = stats[g], mx = stats[n + g], ref = stats[2 * n + g];
    const double lo = ref + sq_lo[g] * (mn - ref), hi = ref + sq_hi[g] * (mx - ref);
    if ((hi - lo) / qmax1 > 1e-8) {
        dg_lo[g] = d_lo[g] * sg_lo[g] * (mn - ref);
        dg_hi[g] = d_hi[g] * sg_hi[g] * (mx - ref);
    } else {
        dg_lo[g] = s1[g] * sg_lo[g] * (mn - ref);
        dg_hi[g] = 0.0;
    }
}

// dL/dG (data coupling + detached budget pressure) -> dL/dS through the soft gate
// (trainer.hpp:361-373); one block per token row
__global__ void __launch_bounds__(kRedThreads) dscore_kernel(const double* __restrict__ resid, const double* __restrict__ P,
                                                             int64_t TO, int64_t out, int nr,
                                                             const double* __restrict__ gates, double reg_coeff,
                                                             double tau, double* __restrict__ d_score) {
    __shared__ double red[kRedThreads / 32];
    const int64_t i = blockIdx.x;
    for (int e = 0; e < nr; ++e) {
        const double* pe = P + (int64_t)(e + 1) * TO + i * out;
        double dot = 0.0;
        for (int64_t j = threadIdx.x; j < out; j += blockDim.x) dot += resid[i * out + j] * pe[j];
        dot = block_sum(dot, red);
        if (threadIdx.x == 0) {
            const double gv = gates[i * nr + e];
            d_score[i * nr + e] = (dot + reg_coeff) * tau * gv * (1.0 - gv);
        }
    }
}

// column sums in row order (the bias gradients, trainer.hpp:377-378, 393-394)
__global__ void colsum_kernel(const double* __restrict__ m, int64_t rows, int64_t cols, double* __restrict__ out) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    double s = 0.0;
    for (int64_t r = 0; r < rows; ++r) s += m[r * cols + c];
    out[c] = s;
}

__global__ void silu_grad_mul_kernel(double* __restrict__ d_act, const double* __restrict__ pre, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double s = sigmoid_d(pre[i]);
        d_act[i] *= s * (1.0 + pre[i] * (1.0 - s));
    }
}

inline unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 16); }

int dgemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t sai, int64_t sak, const double* B, int64_t sbk,
          int64_t sbj, const double* bias, double* C, int64_t ldc, cudaStream_t st) {
    if (M <= 0 || N <= 0) return MOBI_OK;
    // per device, cached (mobi_internal.cuh): 3 stages x 26 KB of dynamic shared memory
    const int rc = func_attr_once_impl(reinterpret_cast<const void*>(dgemm_kernel),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
    if (rc) return rc;
    dim3 grid((unsigned)cdiv(N, kBN), (unsigned)cdiv(M, kBM));
    dgemm_kernel<<<grid, kGemmThreads, kGemmSmem, st>>>(M, N, K, A, sai, sak, B, sbk, sbj, bias, C, ldc);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

double host_sigmoid(double v) { return v >= 0.0 ? 1.0 / (1.0 + std::exp(-v)) : std::exp(v) / (1.0 + std::exp(v)); }

// trainer.hpp:52-73
double schedule_value(const mobi_budget_schedule& s, int64_t t) {
    const double bi = s.b_init, bt = s.b_target, frac = (double)t / (double)s.total_steps;
    switch (s.shape) {
        case 0:
            if (t == s.total_steps) return bt;
            return bi - (bi - bt) * std::log((double)t) / std::log((double)s.total_steps);
        case 1: return bi - (bi - bt) * frac;
        case 2: return bt + (bi - bt) * (1.0 + std::cos(M_PI * frac)) / 2.0;
        default: return bi * std::pow(bt / bi, frac);
    }
}

struct DevBuf {  // stream-ordered scratch, freed on every exit path
    cudaStream_t st;
    std::vector<void*> ptrs;
    ~DevBuf() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
    template <class T>
    int get(T** p, int64_t n) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), (size_t)std::max<int64_t>(n, 1) * sizeof(T), st);
        if (e != cudaSuccess) return set_error(MOBI_ERUNTIME, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        ptrs.push_back(*p);
        return MOBI_OK;
    }
};

#define TRY(x)                  \
    do {                        \
        int rc_ = (x);          \
        if (rc_) return rc_;    \
    } while (0)

}  // namespace

int joint_step(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* slice_bits, int32_t E,
               const double* gamma_lo, const double* gamma_hi, const double* w1, const double* b1, const double* w2,
               const double* b2, int64_t h, const double* x, const double* y_fp, int64_t T,
               const mobi_budget_schedule* sched, int64_t t, int32_t force_on, double* y_hat_out,
               mobi_joint_scalars* res, double* d_gamma_lo, double* d_gamma_hi, double* d_w1, double* d_b1,
               double* d_w2, double* d_b2, cudaStream_t st, bool msb) {
    const int nr = E - 1;  // 0 for the stage-1 MSB step (slice 1 alone, no router)
    const int64_t G = cdiv(in, gs), NG = out * G, TO = T * out;
    {  // keep the stream-ordered scratch (hundreds of MB at LLaMA shapes) mapped between steps: the
       // default pool would otherwise return it to the OS at every synchronize and re-map it next step
        int dev = 0;
        cudaMemPool_t pool;
        MOBI_CUDA(cudaGetDevice(&dev));
        MOBI_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = UINT64_MAX;
        MOBI_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    DevBuf buf{st, {}};
    // host side: per-group squash / squash' with the reference's libm; schedule, temperature
    std::vector<double> hq(4 * NG);
    for (int64_t g = 0; g < NG; ++g) {
        const double a = host_sigmoid(gamma_lo[g]), b = host_sigmoid(gamma_hi[g]);
        hq[g] = a;
        hq[NG + g] = b;
        hq[2 * NG + g] = a * (1.0 - a);
        hq[3 * NG + g] = b * (1.0 - b);
    }
    const bool hard = force_on || t == sched->total_steps;
    double tau = 0.0;
    if (!hard) {
        const double ll = std::log((double)sched->total_steps);
        tau = ll / (ll - std::log((double)t));
    }
    double *sq, *scale, *zero, *stats, *W, *P, *hpre = nullptr, *hact = nullptr, *S = nullptr, *gates, *y_hat, *partial,
                                                *sc3;
    int32_t* bits_dev;
    uint8_t* codes;
    unsigned long long* cc;
    TRY(buf.get(&sq, 4 * NG));
    TRY(buf.get(&bits_dev, E));
    TRY(buf.get(&codes, (int64_t)E * out * in));
    TRY(buf.get(&scale, NG));
    TRY(buf.get(&zero, NG));
    TRY(buf.get(&stats, 3 * NG));
    TRY(buf.get(&cc, MOBI_MAX_SLICES));
    TRY(buf.get(&W, out * in));
    TRY(buf.get(&P, (int64_t)E * TO));
    TRY(buf.get(&gates, T * std::max(nr, 1)));
    TRY(buf.get(&partial, T));
    TRY(buf.get(&sc3, 3));
    if (y_hat_out) {
        y_hat = y_hat_out;
    } else {
        TRY(buf.get(&y_hat, TO));
    }
    MOBI_CUDA(cudaMemcpyAsync(sq, hq.data(), sizeof(double) * 4 * NG, cudaMemcpyHostToDevice, st));
    MOBI_CUDA(cudaMemcpyAsync(bits_dev, slice_bits, sizeof(int32_t) * E, cudaMemcpyHostToDevice, st));
    MOBI_CUDA(cudaMemsetAsync(cc, 0, sizeof(unsigned long long) * MOBI_MAX_SLICES, st));
    // f.stack = layer.decompose() (trainer.hpp:210)
    TRY(launch_decompose_clip(w, out, in, gs, bits_dev, E, sq, sq + NG, codes, scale, zero, stats, cc, st));
    // P_e = X · dequant(slice e)ᵀ (trainer.hpp:213-217)
    std::vector<double> unit(E), mid(E);
    for (int e = 0, before = 0; e < E; before += slice_bits[e], ++e) {
        unit[e] = std::ldexp(1.0, -before);
        mid[e] = e == 0 ? 0.0 : std::ldexp(1.0, slice_bits[e] - 1);
        dequant_slice_kernel<<<grid_for(out * in), 256, 0, st>>>(codes + (int64_t)e * out * in, scale, zero, out, in,
                                                                 gs, G, unit[e], mid[e], e == 0, W);
        MOBI_LAUNCH_CHECK();
        TRY(dgemm(T, out, in, x, in, 1, W, 1, in, nullptr, P + (int64_t)e * TO, out, st));
    }
    // router MLP + gate_soft (trainer.hpp:220-243)
    if (!force_on) {
        TRY(buf.get(&hpre, T * h));
        TRY(buf.get(&hact, T * h));
        TRY(buf.get(&S, T * nr));
        TRY(dgemm(T, h, in, x, in, 1, w1, h, 1, b1, hpre, h, st));
        silu_kernel<<<grid_for(T * h), 256, 0, st>>>(hpre, hact, T * h);
        MOBI_LAUNCH_CHECK();
        TRY(dgemm(T, nr, h, hact, h, 1, w2, nr, 1, b2, S, nr, st));
    }
    if (nr > 0) {
        gates_kernel<<<grid_for(T * nr), 256, 0, st>>>(S, gates, T * nr, tau, force_on ? 2 : (hard ? 1 : 0));
        MOBI_LAUNCH_CHECK();
    }
    combine_kernel<<<(unsigned)T, kRedThreads, 0, st>>>(P, TO, E, gates, nr, out, y_fp, y_hat, partial);
    MOBI_LAUNCH_CHECK();
    scalars_kernel<<<1, kRedThreads, 0, st>>>(partial, T, gates, nr, bits_dev, sc3);
    MOBI_LAUNCH_CHECK();
    double h3[3];
    MOBI_CUDA(cudaMemcpyAsync(h3, sc3, sizeof(h3), cudaMemcpyDeviceToHost, st));
    MOBI_CUDA(cudaStreamSynchronize(st));
    res->data_term = h3[0] / (double)TO;
    res->avg_bits = h3[2] / (double)T;
    res->sched_b = schedule_value(*sched, t);
    res->reg_term = (res->avg_bits - res->sched_b) * h3[1];
    res->loss = res->data_term + sched->reg_weight * res->reg_term;
    res->tau = tau;
    if (!d_gamma_lo) return MOBI_OK;

    // ---- joint_backward (trainer.hpp:341-396) ----
    double *resid, *dpe, *d_lo, *d_hi, *s1;
    TRY(buf.get(&resid, TO));
    TRY(buf.get(&dpe, TO));
    TRY(buf.get(&d_lo, NG));
    TRY(buf.get(&d_hi, NG));
    TRY(buf.get(&s1, NG));
    resid_kernel<<<grid_for(TO), 256, 0, st>>>(y_hat, y_fp, 2.0 * (1.0 / (double)TO), resid, TO);
    MOBI_LAUNCH_CHECK();
    MOBI_CUDA(cudaMemsetAsync(d_lo, 0, sizeof(double) * NG, st));
    MOBI_CUDA(cudaMemsetAsync(d_hi, 0, sizeof(double) * NG, st));
    const double qmax1 = (double)((1 << slice_bits[0]) - 1);
    for (int e = 0; e < E; ++e) {
        // dL/dW_e = (g_e ⊙ resid)ᵀ X  [out][in]   (W's buffer is free after the forward)
        const double* dp = resid;
        if (e > 0) {  // the reference materialises dpe = resid * gate, then multiplies (trainer.hpp:351-358)
            row_scale_kernel<<<grid_for(TO), 256, 0, st>>>(resid, gates, nr, e - 1, T, out, dpe);
            MOBI_LAUNCH_CHECK();
            dp = dpe;
        }
        TRY(dgemm(out, in, T, dp, 1, out, x, in, 1, nullptr, W, in, st));
        clip_accum_kernel<<<(unsigned)cdiv(NG, 128), 128, 0, st>>>(W, codes + (int64_t)e * out * in, out, in, gs, G,
                                                                   unit[e], mid[e], qmax1, e == 0, d_lo, d_hi, s1);
        MOBI_LAUNCH_CHECK();
    }
    double* dg;
    TRY(buf.get(&dg, 2 * NG));
    gamma_grad_kernel<<<(unsigned)cdiv(NG, 128), 128, 0, st>>>(stats, NG, sq, sq + NG, sq + 2 * NG, sq + 3 * NG, qmax1,
                                                               d_lo, d_hi, s1, dg, dg + NG);
    MOBI_LAUNCH_CHECK();
    MOBI_CUDA(cudaMemcpyAsync(d_gamma_lo, dg, sizeof(double) * NG, cudaMemcpyDeviceToHost, st));
    MOBI_CUDA(cudaMemcpyAsync(d_gamma_hi, dg + NG, sizeof(double) * NG, cudaMemcpyDeviceToHost, st));
    if (msb) {  // msb_backward (trainer.hpp:417-426): clip gradients only
    } else if (hard) {  // indicator gate: zero router gradient (trainer.hpp:364)
        MOBI_CUDA(cudaMemsetAsync(d_w1, 0, sizeof(double) * in * h, st));
        MOBI_CUDA(cudaMemsetAsync(d_b1, 0, sizeof(double) * h, st));
        MOBI_CUDA(cudaMemsetAsync(d_w2, 0, sizeof(double) * h * nr, st));
        MOBI_CUDA(cudaMemsetAsync(d_b2, 0, sizeof(double) * nr, st));
    } else {
        double *d_score, *d_act;
        TRY(buf.get(&d_score, T * nr));
        TRY(buf.get(&d_act, T * h));
        const double reg_coeff = sched->reg_weight * (res->avg_bits - res->sched_b);
        dscore_kernel<<<(unsigned)T, kRedThreads, 0, st>>>(resid, P, TO, out, nr, gates, reg_coeff, tau, d_score);
        MOBI_LAUNCH_CHECK();
        TRY(dgemm(h, nr, T, hact, 1, h, d_score, nr, 1, nullptr, d_w2, nr, st));  // hactᵀ d_score
        colsum_kernel<<<1, 32, 0, st>>>(d_score, T, nr, d_b2);
        MOBI_LAUNCH_CHECK();
        TRY(dgemm(T, h, nr, d_score, nr, 1, w2, 1, nr, nullptr, d_act, h, st));  // d_score w2ᵀ
        silu_grad_mul_kernel<<<grid_for(T * h), 256, 0, st>>>(d_act, hpre, T * h);
        MOBI_LAUNCH_CHECK();
        TRY(dgemm(in, h, T, x, 1, in, d_act, h, 1, nullptr, d_w1, h, st));  // Xᵀ d_act
        colsum_kernel<<<(unsigned)cdiv(h, 128), 128, 0, st>>>(d_act, T, h, d_b1);
        MOBI_LAUNCH_CHECK();
    }
    MOBI_CUDA(cudaStreamSynchronize(st));
    return MOBI_OK;
}

}  // namespace mobi
