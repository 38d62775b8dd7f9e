// layer.cu -- device repacking of a layer's slice payload into the tiled merged-code layout
// (mobi_internal.cuh) and the K6 read-back used for bit-exact verification.
//
// Reference layouts consumed:
//   SliceStack::slices     [E][out][in] uint8 codes            (slicer.hpp:25-30)
//   LayerRecord::planes    merged code INT = c1<<(E-1)b | ... | cE (slicer.hpp:150-161) as
//                          `bits` planes of uint64 words, plane 0 = MSB, word r*wpr + c/64,
//                          bit c%64 (bitplane.hpp:21-36, 48-73)
#include "mobi_internal.cuh"

namespace mobi {
namespace {

// one thread = one (row, 16-column chunk): merge E slice codes, store 16 bytes
__global__ void pack_codes_kernel(const uint8_t* __restrict__ codes, int64_t out, int64_t in,
                                  int64_t out_pad, int64_t kblocks, SliceLayout sl,
                                  uint8_t* __restrict__ dst) {
    const int64_t nchunks = kblocks * (kKBlock / 16);
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= out_pad * nchunks) return;
    const int64_t R = idx / nchunks, ch = idx % nchunks;
    const int64_t k0 = ch * 16;
    uint8_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int64_t k = k0 + j;
        unsigned m = 0;
        if (R < out && k < in) {
            for (int e = 0; e < sl.E; ++e) m |= (unsigned)codes[(int64_t)e * out * in + R * in + k] << sl.off[e];
        }
        v[j] = (uint8_t)m;
    }
    uint4 w;
    memcpy(&w, v, 16);
    *reinterpret_cast<uint4*>(dst + code_offset(R, k0, kblocks)) = w;
}

// one thread = one (row, 64-bit word): gather `bits` plane bits of 64 columns
__global__ void pack_planes_kernel(const uint64_t* __restrict__ planes, int bits, int64_t wpr,
                                   int64_t out, int64_t in, int64_t out_pad, int64_t kblocks,
                                   uint8_t* __restrict__ dst) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= out_pad * kblocks) return;
    const int64_t R = idx / kblocks, w = idx % kblocks;  // kKBlock == 64 == bits per word
    uint64_t pw[8];
    for (int p = 0; p < 8; ++p)
        pw[p] = (p < bits && R < out && w < wpr) ? planes[(int64_t)p * out * wpr + R * wpr + w] : 0ull;
    for (int c = 0; c < 4; ++c) {
        uint8_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int col = c * 16 + j;
            unsigned code = 0;
            for (int bit = 0; bit < bits; ++bit)  // bit `bit` lives in plane bits-1-bit
                code |= (unsigned)((pw[bits - 1 - bit] >> col) & 1ull) << bit;
            if (w * 64 + col >= in) code = 0;
            v[j] = (uint8_t)code;
        }
        uint4 q;
        memcpy(&q, v, 16);
        *reinterpret_cast<uint4*>(dst + code_offset(R, w * 64 + c * 16, kblocks)) = q;
    }
}

// K6: tiled merged codes -> slice codes [E][out][in]  (LayerRecord::stack() split)
__global__ void unpack_codes_kernel(const uint8_t* __restrict__ src, int64_t out, int64_t in,
                                    int64_t kblocks, SliceLayout sl, uint8_t* __restrict__ codes) {
    const int64_t nchunks = kblocks * (kKBlock / 16);
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= out * nchunks) return;
    const int64_t R = idx / nchunks, k0 = (idx % nchunks) * 16;
    uint4 q = *reinterpret_cast<const uint4*>(src + code_offset(R, k0, kblocks));
    uint8_t v[16];
    memcpy(v, &q, 16);
    for (int j = 0; j < 16; ++j) {
        const int64_t k = k0 + j;
        if (k >= in) break;
        for (int e = 0; e < sl.E; ++e)
            codes[(int64_t)e * out * in + R * in + k] = (uint8_t)((v[j] >> sl.off[e]) & ((1u << sl.b[e]) - 1u));
    }
}

__global__ void check_codes_kernel(const uint8_t* __restrict__ codes, int64_t n, int qmax,
                                   unsigned long long* __restrict__ first_bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (codes[i] > qmax) atomicMin(first_bad, (unsigned long long)i);
}

}  // namespace

// index of the first slice code above qmax, or -1 (device-resident SliceStack ingest)
int check_codes_device(const uint8_t* codes_dev, int64_t n, int qmax, int64_t* bad) {
    unsigned long long* d = nullptr;
    MOBI_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
    unsigned long long init = ~0ull, h = 0;
    MOBI_CUDA(cudaMemcpy(d, &init, sizeof(init), cudaMemcpyHostToDevice));
    check_codes_kernel<<<592, 256>>>(codes_dev, n, qmax, d);
    cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return set_error(MOBI_ERUNTIME, std::string("check_codes: ") + cudaGetErrorString(e));
    *bad = h == ~0ull ? -1 : (int64_t)h;
    return MOBI_OK;
}

// Decode slice planes (decode2.cu): per slice e, 32-row tile rt, 64-k block kb: 32 lanes x 16 bytes
// holding the lane's m16n8k16 A fragments.  Lane (g = lane/4, c = lane%4): word q is fragment register
// a_q (a0: row g, MMA k 2c|2c+1; a1: row g+8; a2: row g, MMA k 2c+8|2c+9; a3: row g+8) of all eight
// MMAs of the block.  MMA k of k-step ss maps to memory k 16c + 4ss + {0,1 | 2,3} (a0 | a2), so the
// activations a lane feeds as B fragments over the block's four k-steps are 16 contiguous values (two
// 16-byte shared loads).  Row group rg (16 rows) x k-step ss sits in field i = 4 rg + ss, low half at
// bits 2i..2i+1, high half at bits 16+2i.  A field masked in place (rg 0) or after one shift by 8
// (rg 1) reads as the fp16 1024 + c 4^ss with a single LOP3, so the kernel scales the activations of
// k-step ss by 4^-ss instead of shifting every field down.  A kernel reads only the planes it needs.
__global__ void pack_dplanes_kernel(const uint8_t* __restrict__ codes8, int64_t kblocks, int64_t n_rt32, int E,
                                    int b, uint4* __restrict__ dplanes) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)E * n_rt32 * kblocks * 32;
    if (idx >= total) return;
    const int lane = (int)(idx % 32);
    const int64_t kb = (idx / 32) % kblocks;
    const int64_t rt = (idx / 32 / kblocks) % n_rt32;
    const int e = (int)(idx / 32 / kblocks / n_rt32);  // 0-based slice
    const int g = lane / 4, c = lane % 4;
    const int shift = (E - 1 - e) * b;
    uint32_t wv[4];
    for (int q = 0; q < 4; ++q) {
        uint32_t word = 0;
        for (int i = 0; i < 8; ++i) {
            const int rg = i / 4, ss = i % 4;
            const int64_t row = rt * 32 + 16 * rg + g + ((q & 1) ? 8 : 0);
            const int64_t k0 = kb * kKBlock + 16 * c + 4 * ss + ((q & 2) ? 2 : 0);
            const uint32_t lo = (codes8[code_offset(row, k0, kblocks)] >> shift) & 3u;
            const uint32_t hi = (codes8[code_offset(row, k0 + 1, kblocks)] >> shift) & 3u;
            word |= lo << (2 * i) | hi << (16 + 2 * i);
        }
        wv[q] = word;
    }
    dplanes[idx] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
}

int launch_pack_dplanes(mobi_layer* L, cudaStream_t st) {
    const int64_t n_rt32 = L->out_pad / 32;
    const int64_t total = (int64_t)L->E * n_rt32 * L->kblocks * 32;
    pack_dplanes_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(L->codes8, L->kblocks, n_rt32, L->E, L->b,
                                                                   reinterpret_cast<uint4*>(L->dplanes));
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

int launch_pack_codes(mobi_layer* L, const uint8_t* codes_dev, cudaStream_t st) {
    const int64_t n = L->out_pad * L->kblocks * (kKBlock / 16);
    pack_codes_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(codes_dev, L->out, L->in, L->out_pad,
                                                             L->kblocks, L->sl, L->codes8);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

int launch_pack_planes(mobi_layer* L, const uint64_t* planes_dev, int bits, int64_t wpr,
                       cudaStream_t st) {
    const int64_t n = L->out_pad * L->kblocks;
    pack_planes_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(planes_dev, bits, wpr, L->out, L->in,
                                                              L->out_pad, L->kblocks, L->codes8);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

int launch_unpack_codes(const mobi_layer* L, uint8_t* codes_dev, cudaStream_t st) {
    const int64_t n = L->out * L->kblocks * (kKBlock / 16);
    unpack_codes_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(L->codes8, L->out, L->in, L->kblocks,
                                                               L->sl, codes_dev);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

// Y [T, out] (row stride out) -> every destination of an output descriptor (row stride ldy, column
// offset col0): the small-T paths compute into a staging buffer and place it with this copy
__global__ void scatter_out_kernel(const __nv_bfloat16* __restrict__ y, int64_t out, OutDesc od) {
    const int64_t t = blockIdx.x;
    const __nv_bfloat16* src = y + t * out;
    for (int64_t c = threadIdx.x; c < out; c += blockDim.x) {
        const __nv_bfloat16 v = src[c];
        for (int k = 0; k < od.n_dst; ++k) od.dst[k][t * od.ldy + od.col0 + c] = v;
    }
    if (od.n_dst > 1) __threadfence_system();
}

int launch_scatter_out(const __nv_bfloat16* y, int64_t T, int64_t out, const OutDesc& od, cudaStream_t st) {
    if (T <= 0) return MOBI_OK;
    scatter_out_kernel<<<(unsigned)T, 256, 0, st>>>(y, out, od);
    MOBI_LAUNCH_CHECK();
    return MOBI_OK;
}

}  // namespace mobi
