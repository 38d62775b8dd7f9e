// select.cu -- router::calibrate_threshold (router.hpp:167-174) on the device: the threshold is the
// element of rank k = floor(rho*N + 1e-9) of the scores sorted in descending order (min - 1 when
// k >= N).  A 4-pass MSB-first radix select over order-preserving 32-bit keys: each pass histograms
// one byte of the keys that share the prefix found so far and narrows to the byte value holding rank
// k.  The result is the exact fp32 score (bit-identical to sorting), so nothing but the one value
// crosses to the host.
#include <algorithm>
#include <cstring>

#include "mobi_internal.cuh"

namespace mobi {
namespace {

constexpr int kSelThreads = 256;

// order-preserving map float -> uint32 (larger float <=> larger key; -0 sorts just below +0)
__device__ __forceinline__ uint32_t f2key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float key2f(uint32_t k) {
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

struct SelState {
    uint32_t prefix;  // key bits fixed so far
    uint32_t mask;    // which bits of the prefix are fixed
    int64_t rank;     // rank still sought among the keys matching the prefix (descending)
};

// histogram of key byte `shift` over the keys matching the current prefix
__global__ void __launch_bounds__(kSelThreads) sel_hist_kernel(const float* __restrict__ s, int64_t n,
                                                               const SelState* __restrict__ st, int shift,
                                                               unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t prefix = st->prefix, mask = st->mask;
    for (int64_t i = (int64_t)blockIdx.x * kSelThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kSelThreads) {
        const uint32_t k = f2key(__ldg(s + i));
        if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

// one warp: walk the byte values from 255 down, find the one holding the sought rank, narrow the
// prefix, and clear the histogram for the next pass
__global__ void sel_pick_kernel(SelState* __restrict__ st, int shift, unsigned long long* __restrict__ hist) {
    __shared__ unsigned long long cnt[256];
    for (int i = threadIdx.x; i < 256; i += 32) {
        cnt[i] = hist[i];
        hist[i] = 0;
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        int64_t r = st->rank;
        int d = 255;
        for (; d > 0; --d) {
            if (r < (int64_t)cnt[d]) break;
            r -= (int64_t)cnt[d];
        }
        st->prefix |= (uint32_t)d << shift;
        st->mask |= 0xffu << shift;
        st->rank = r;
    }
}

__global__ void __launch_bounds__(256) avg_bits_kernel(const uint8_t* __restrict__ m, int64_t T, uint4 bits_lo,
                                                       uint4 bits_hi, int E, unsigned long long* __restrict__ sum) {
    const uint32_t b[8] = {bits_lo.x, bits_lo.y, bits_lo.z, bits_lo.w, bits_hi.x, bits_hi.y, bits_hi.z, bits_hi.w};
    unsigned long long acc = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t mk = m[t] | 1u;  // slice 1 is always on (router.hpp:141)
        for (int e = 0; e < E && e < 8; ++e)
            if ((mk >> e) & 1u) acc += b[e];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(sum, acc);
}

}  // namespace

int launch_avg_bits(const uint8_t* masks, int64_t T, const int32_t* slice_bits, int32_t E, double* avg,
                    cudaStream_t stream) {
    uint32_t b[8] = {};
    for (int e = 0; e < E && e < 8; ++e) b[e] = (uint32_t)slice_bits[e];
    unsigned long long* d = nullptr;
    MOBI_CUDA(cudaMallocAsync(&d, sizeof(unsigned long long), stream));
    MOBI_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), stream));
    const int blocks = (int)std::min<int64_t>(cdiv(T, 256), 296);
    avg_bits_kernel<<<blocks, 256, 0, stream>>>(masks, T, make_uint4(b[0], b[1], b[2], b[3]),
                                                make_uint4(b[4], b[5], b[6], b[7]), E, d);
    MOBI_LAUNCH_CHECK();
    unsigned long long h = 0;
    MOBI_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    MOBI_CUDA(cudaStreamSynchronize(stream));
    cudaFreeAsync(d, stream);
    *avg = (double)h / (double)T;
    return MOBI_OK;
}

int launch_select_desc(const float* scores, int64_t n, int64_t k, float* out_host, cudaStream_t stream) {
    SelState* st = nullptr;
    unsigned long long* hist = nullptr;
    MOBI_CUDA(cudaMallocAsync(&st, sizeof(SelState), stream));
    MOBI_CUDA(cudaMallocAsync(&hist, 256 * sizeof(unsigned long long), stream));
    const SelState init{0u, 0u, k};
    int rc = MOBI_OK;
    auto fail = [&](cudaError_t e) {
        if (e != cudaSuccess && !rc) rc = set_error(MOBI_ERUNTIME, std::string("calibrate_threshold: ") + cudaGetErrorString(e));
    };
    fail(cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, stream));
    fail(cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), stream));
    const int blocks = (int)std::min<int64_t>(cdiv(n, kSelThreads), 1184);  // 8 per SM on 148 SMs
    for (int shift = 24; shift >= 0 && !rc; shift -= 8) {
        sel_hist_kernel<<<blocks, kSelThreads, 0, stream>>>(scores, n, st, shift, hist);
        sel_pick_kernel<<<1, 32, 0, stream>>>(st, shift, hist);
        fail(cudaGetLastError());
    }
    SelState res{};
    fail(cudaMemcpyAsync(&res, st, sizeof(res), cudaMemcpyDeviceToHost, stream));
    fail(cudaStreamSynchronize(stream));
    cudaFreeAsync(st, stream);
    cudaFreeAsync(hist, stream);
    if (!rc) *out_host = key2f(res.prefix);
    return rc;
}

}  // namespace mobi
