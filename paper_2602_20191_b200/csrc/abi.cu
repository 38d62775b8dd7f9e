// abi.cu -- host side of the C ABI (include/mobi_b200.h): validation with the reference's
// MOBI_CHECK wording, upload + device repack of a layer, workspace management, and the
// route -> bucket -> gather -> GEMM launch sequence.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>
#include <string>
#include <vector>

#include "mobi_internal.cuh"

namespace mobi {

static thread_local std::string g_err;
static unsigned long long* g_trace_buf = nullptr;

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int func_attr_once_impl(const void* fn, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::set<std::tuple<int, const void*, int>> done;
    int dev = 0;
    MOBI_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (done.count(std::make_tuple(dev, fn, (int)attr))) return MOBI_OK;
    MOBI_CUDA(cudaFuncSetAttribute(fn, attr, value));
    done.insert(std::make_tuple(dev, fn, (int)attr));
    return MOBI_OK;
}

int joint_step(const double* w, int64_t out, int64_t in, int64_t gs, const int32_t* slice_bits, int32_t E,
               const double* gamma_lo, const double* gamma_hi, const double* w1, const double* b1, const double* w2,
               const double* b2, int64_t h, const double* x, const double* y_fp, int64_t T,
               const mobi_budget_schedule* sched, int64_t t, int32_t force_on, double* y_hat_out,
               mobi_joint_scalars* res, double* d_gamma_lo, double* d_gamma_hi, double* d_w1, double* d_b1,
               double* d_w2, double* d_b2, cudaStream_t st, bool msb = false);
int launch_permute(const uint8_t* masks, int64_t T, uint8_t* keys_tmp, int32_t* cperm, int32_t* inverse,
                   int32_t* hist256, cudaStream_t st);

namespace {

#define CHECK_ARG(cond, msg)                            \
    do {                                                \
        if (!(cond)) {                                  \
            std::ostringstream o_;                      \
            o_ << msg;                                  \
            return set_error(MOBI_EINVAL, o_.str());    \
        }                                               \
    } while (0)

inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

template <class T>
int dmalloc(T** p, size_t n, mobi_layer* L) {
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
    if (e != cudaSuccess) return set_error(MOBI_ERUNTIME, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    if (L) L->device_bytes += (int64_t)(n * sizeof(T));
    return MOBI_OK;
}

template <class T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

uint16_t f2bf(float f) {  // round-to-nearest-even, NaN-preserving
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
float bf2f(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

void free_ws(mobi_layer* L) {
    if (L->hist256) cudaFree(L->hist256);
    L->hist256 = nullptr;
    dfree(L->s_part);
    dfree(L->scores);
    dfree(L->masks);
    dfree(L->perm);
    dfree(L->pinv);
    dfree(L->inverse);
    dfree(L->cperm);
    dfree(L->escale);
    if (L->xperm_shared) {
        L->xperm_shared.reset();
        L->xperm = nullptr;
    } else {
        dfree(L->xperm);
    }
    dfree(L->tiles);
    dfree(L->meta);
    dfree(L->rt_cnt);
    dfree(L->bk_hist);
    if (L->tmap_x) delete L->tmap_x;
    L->tmap_x = nullptr;
    if (L->tmap_x2) delete[] L->tmap_x2;
    L->tmap_x2 = nullptr;
    L->ws_T = -1;
}

int ensure_ws(mobi_layer* L, int64_t T) {
    if (T <= L->ws_T) return MOBI_OK;
    if (L->ws_T >= 0) {  // the old workspace may still be in use by work queued on this context's stream
        if (L->ctx_bound)
            MOBI_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(L->ctx_stream)));
        else
            MOBI_CUDA(cudaDeviceSynchronize());
    }
    free_ws(L);
    const int64_t Tc = round_up(std::max<int64_t>(T, 1), 256);
    L->tpad_max = round_up(Tc + 2 * kMaxBuckets * (kBucketAlign - 1), kBucketAlign);
    L->max_tiles = cdiv(Tc, kTokTile) + 2 * kMaxBuckets;
    const int64_t htiles_max = cdiv(L->h, 64);
    int rc;
    if ((rc = dmalloc(&L->s_part, (size_t)(htiles_max * Tc * L->nr), nullptr))) return rc;
    if ((rc = dmalloc(&L->scores, (size_t)(Tc * L->nr), nullptr))) return rc;
    if ((rc = dmalloc(&L->masks, (size_t)Tc, nullptr))) return rc;
    if ((rc = dmalloc(&L->perm, (size_t)L->tpad_max, nullptr))) return rc;
    if ((rc = dmalloc(&L->pinv, (size_t)Tc, nullptr))) return rc;
    if ((rc = dmalloc(&L->inverse, (size_t)Tc, nullptr))) return rc;
    if ((rc = dmalloc(&L->cperm, (size_t)Tc, nullptr))) return rc;
    if ((rc = dmalloc(&L->escale, (size_t)L->tpad_max, nullptr))) return rc;
    if ((rc = dmalloc(&L->xperm, (size_t)(L->tpad_max * L->in_pad), nullptr))) return rc;
    if ((rc = dmalloc(&L->tiles, (size_t)L->max_tiles, nullptr))) return rc;
    if ((rc = dmalloc(&L->meta, 64, nullptr))) return rc;
    if ((rc = dmalloc(&L->rt_cnt, (size_t)(Tc / 128 + 1), nullptr))) return rc;
    MOBI_CUDA(cudaMemset(L->rt_cnt, 0, (size_t)(Tc / 128 + 1) * sizeof(int32_t)));
    if ((rc = dmalloc(&L->bk_hist, 48, nullptr))) return rc;
    MOBI_CUDA(cudaMemset(L->bk_hist, 0, 48 * sizeof(int32_t)));
    if (!L->gpart && (rc = dmalloc(&L->gpart, (size_t)(8 * 64 * L->out_pad), nullptr))) return rc;
    if (!L->hpart && (rc = dmalloc(&L->hpart, (size_t)(16 * 64 * L->h_pad), nullptr))) return rc;
    if (!L->dec_cnt) {
        int nsm = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int64_t n_rt = cdiv(L->out, kRowTile), n_mt = L->h_pad / 16;
        if ((rc = dmalloc(&L->dec_part, (size_t)((std::max(nsm, 1) + n_rt) * kDecMaxT * kRowTile), nullptr))) return rc;
        if ((rc = dmalloc(&L->dec_spart, (size_t)(n_mt * kDecMaxT * L->nr), nullptr))) return rc;
        if ((rc = dmalloc(&L->dec_cnt, (size_t)(n_rt + n_mt + 1), nullptr))) return rc;
        MOBI_CUDA(cudaMemset(L->dec_cnt, 0, (size_t)(n_rt + n_mt + 1) * sizeof(int32_t)));
    }
    L->ws_T = Tc;
    return MOBI_OK;
}

int validate_and_fill(const mobi_layer_desc* d, mobi_layer* L, bool codes_on_device = false) {
    CHECK_ARG(d != nullptr, "mobi_layer_create: null descriptor");
    CHECK_ARG(d->out > 0 && d->in > 0, "mobi_layer_create: empty weight " << d->out << "x" << d->in);
    CHECK_ARG(d->group_size >= 1, "QuantParams: group_size must be >= 1");
    CHECK_ARG(d->n_slices >= 2 && d->n_slices <= MOBI_MAX_SLICES,
              "mobi_layer_create: " << d->n_slices << " slices; supported 2.." << MOBI_MAX_SLICES);
    CHECK_ARG(d->slice_bits != nullptr, "decompose: slice_bits is empty");
    int total = 0;
    bool uniform = true;
    for (int e = 0; e < d->n_slices; ++e) {
        CHECK_ARG(d->slice_bits[e] >= 1 && d->slice_bits[e] <= 8,
                  "decompose: slice bit width " << d->slice_bits[e] << " out of [1,8]");
        uniform = uniform && d->slice_bits[e] == d->slice_bits[0];
        total += d->slice_bits[e];
    }
    CHECK_ARG(total <= 8, "decompose: total bits " << total << " exceed the 8-bit code budget");
    CHECK_ARG(d->group_size >= d->in || d->group_size % 32 == 0,
              "mobi_layer_create: group_size " << d->group_size
                                               << " must be a multiple of 32 or cover the whole row (in=" << d->in << ")");
    CHECK_ARG(d->scale && d->zero, "QuantParams: missing scales/zeros");
    L->out = d->out;
    L->in = d->in;
    L->gs = d->group_size;
    L->G = cdiv(d->in, d->group_size);
    L->single_group = d->group_size >= d->in;
    L->E = d->n_slices;
    // uniform widths with E <= 4: the folded-weight kernels (W_m = S (INT & maskbyte(m)) + C_m needs
    // equal widths, see mobi_internal.cuh); anything else: the generic per-slice kernels (gemm_generic.cu)
    L->generic = !uniform || d->n_slices > kFastSlices;
    L->b = uniform ? d->slice_bits[0] : 0;
    L->nr = d->n_slices - 1;
    L->sl.E = L->E;
    for (int e = L->E - 1, off = 0; e >= 0; --e) {  // INT = ((c1 << b2 | c2) << b3 | c3) ...
        L->sl.b[e] = d->slice_bits[e];
        L->sl.off[e] = off;
        off += d->slice_bits[e];
    }
    const int64_t ng = L->out * L->G;
    for (int64_t g = 0; g < ng; ++g) {
        CHECK_ARG(std::isfinite(d->scale[g]) && d->scale[g] > 0.0, "QuantParams: non-positive scale at group " << g);
        CHECK_ARG(std::isfinite(d->zero[g]), "QuantParams: non-finite zero at group " << g);
    }
    CHECK_ARG((d->codes != nullptr) != (d->planes != nullptr),
              "mobi_layer_create: give exactly one of codes (SliceStack) or planes (LayerRecord)");
    if (d->codes && !codes_on_device) {
        const int64_t n = L->out * L->in;
        for (int e = 0; e < L->E; ++e) {
            const int qmax = (1 << L->sl.b[e]) - 1;
            for (int64_t i = 0; i < n; ++i)
                if (d->codes[(int64_t)e * n + i] > qmax)
                    return set_error(MOBI_EINVAL, "dequantize_centered: code " + std::to_string(d->codes[e * n + i]) +
                                                      " out of [0," + std::to_string(qmax) + "] at (" +
                                                      std::to_string(i / L->in) + "," + std::to_string(i % L->in) +
                                                      ")");
        }
    } else if (!d->codes) {
        CHECK_ARG(d->plane_bits == total, "bitplane: planes carry " << d->plane_bits << " bits, slices need " << total);
        CHECK_ARG(d->words_per_row == cdiv(d->in, 64),
                  "bitplane: words_per_row " << d->words_per_row << " != ceil(in/64) = " << cdiv(d->in, 64));
    }
    CHECK_ARG(d->router_hidden >= 1, "RouterState: hidden width must be >= 1");
    CHECK_ARG(d->w1 && d->b1 && d->w2 && d->b2, "RouterState: missing router weights");
    L->h = d->router_hidden;
    L->out_pad = round_up(L->out, 2 * kRowTile);  // row tiles come in pairs (GEMM CTA clusters)
    L->in_pad = round_up(L->in, kKBlock);
    L->kblocks = L->in_pad / kKBlock;
    L->h_pad = round_up(L->h, 128);
    if (L->generic) return MOBI_OK;
    // per-mask dequant constants (uniform b-bit slices, see mobi_internal.cuh)
    const int P = (L->E - 1) * L->b;
    const unsigned fm = (1u << L->b) - 1u;
    for (int m = 0; m < 2 * kMaxBuckets; ++m) {
        unsigned mb = 0;
        double K = std::ldexp(1.0, P);
        for (int e = 1; e <= L->E; ++e) {
            if (!((m >> (e - 1)) & 1)) continue;
            mb |= fm << ((L->E - e) * L->b);
            if (e >= 2) K -= (double)fm * std::ldexp(1.0, P - (e - 1) * L->b);
        }
        L->mtab.maskword[m] = mb * 0x01010101u;
        L->mtab.kc[m] = (float)(K / std::ldexp(1.0, P + 1));
    }
    L->mtab.inv_2p = (float)std::ldexp(1.0, -P);
    return MOBI_OK;
}

int upload_layer(const mobi_layer_desc* d, mobi_layer* L, bool codes_on_device = false) {
    int rc;
    const int64_t ng = L->out * L->G;
    // weights: tiled merged codes (repacked on the device)
    if ((rc = dmalloc(&L->codes8, (size_t)(L->out_pad * L->in_pad), L))) return rc;
    if (d->codes && codes_on_device) {
        const int64_t n = L->out * L->in;
        for (int e = 0; e < L->E; ++e) {
            int64_t bad = -1;
            const int qmax = (1 << L->sl.b[e]) - 1;
            if ((rc = check_codes_device(d->codes + (int64_t)e * n, n, qmax, &bad))) return rc;
            if (bad >= 0)
                return set_error(MOBI_EINVAL, "dequantize_centered: code out of [0," + std::to_string(qmax) + "] at (" +
                                                  std::to_string(bad / L->in) + "," + std::to_string(bad % L->in) + ")");
        }
        rc = launch_pack_codes(L, d->codes, 0);
        cudaDeviceSynchronize();
        if (rc) return rc;
    } else if (d->codes) {
        uint8_t* tmp = nullptr;
        const size_t n = (size_t)(L->E * L->out * L->in);
        if ((rc = dmalloc(&tmp, n, nullptr))) return rc;
        MOBI_CUDA(cudaMemcpy(tmp, d->codes, n, cudaMemcpyHostToDevice));
        rc = launch_pack_codes(L, tmp, 0);
        cudaDeviceSynchronize();
        dfree(tmp);
        if (rc) return rc;
    } else {
        uint64_t* tmp = nullptr;
        const size_t n = (size_t)(d->plane_bits * L->out * d->words_per_row);
        if ((rc = dmalloc(&tmp, n, nullptr))) return rc;
        MOBI_CUDA(cudaMemcpy(tmp, d->planes, n * 8, cudaMemcpyHostToDevice));
        rc = launch_pack_planes(L, tmp, d->plane_bits, d->words_per_row, 0);
        cudaDeviceSynchronize();
        dfree(tmp);
        if (rc) return rc;
    }
    // decode slice planes (2-bit slices only): the decode GEMV streams just the slices a batch uses
    if (L->b == 2 && !L->generic) {
        if ((rc = dmalloc(&L->dplanes, (size_t)(L->E * (L->out_pad / 32) * L->kblocks * 512), L))) return rc;
        if ((rc = launch_pack_dplanes(L, 0))) return rc;
        MOBI_CUDA(cudaDeviceSynchronize());
    }
    // group constants transposed to [G][out_pad] (s, s*z): a warp's 32 rows read 256 contiguous bytes
    std::vector<float2> gc((size_t)(L->G * L->out_pad), make_float2(0.f, 0.f));
    for (int64_t r = 0; r < L->out; ++r)
        for (int64_t g = 0; g < L->G; ++g) {
            const double sc = d->scale[r * L->G + g];
            gc[(size_t)(g * L->out_pad + r)] = make_float2((float)sc, (float)(sc * d->zero[r * L->G + g]));
        }
    (void)ng;
    if ((rc = dmalloc(&L->gconst, gc.size(), L))) return rc;
    MOBI_CUDA(cudaMemcpy(L->gconst, gc.data(), gc.size() * sizeof(float2), cudaMemcpyHostToDevice));
    // router: w1 transposed to [h_pad][in_pad] bf16 (K-major B operand), zero padded
    std::vector<uint16_t> w1t((size_t)(L->h_pad * L->in_pad), 0);
    for (int64_t k = 0; k < L->in; ++k)
        for (int64_t j = 0; j < L->h; ++j) w1t[(size_t)(j * L->in_pad + k)] = f2bf((float)d->w1[k * L->h + j]);
    std::vector<float> b1((size_t)L->h_pad, 0.f), w2((size_t)(L->h_pad * L->nr), 0.f), b2((size_t)L->nr);
    for (int64_t j = 0; j < L->h; ++j) {
        b1[j] = (float)d->b1[j];
        for (int k = 0; k < L->nr; ++k) w2[j * L->nr + k] = (float)d->w2[j * L->nr + k];
    }
    for (int k = 0; k < L->nr; ++k) b2[k] = (float)d->b2[k];
    if ((rc = dmalloc(&L->w1t, w1t.size(), L))) return rc;
    if ((rc = dmalloc(&L->b1, b1.size(), L))) return rc;
    if ((rc = dmalloc(&L->w2, w2.size(), L))) return rc;
    if ((rc = dmalloc(&L->b2, b2.size(), L))) return rc;
    MOBI_CUDA(cudaMemcpy(L->w1t, w1t.data(), w1t.size() * 2, cudaMemcpyHostToDevice));
    MOBI_CUDA(cudaMemcpy(L->b1, b1.data(), b1.size() * 4, cudaMemcpyHostToDevice));
    MOBI_CUDA(cudaMemcpy(L->w2, w2.data(), w2.size() * 4, cudaMemcpyHostToDevice));
    MOBI_CUDA(cudaMemcpy(L->b2, b2.data(), b2.size() * 4, cudaMemcpyHostToDevice));
    MOBI_CUDA(cudaDeviceSynchronize());
    return MOBI_OK;
}

// score (router.hpp:63-76); the tcgen05 router also applies gate_hard(delta) for prefill sizes and
// then reports *masks_ready (L->masks, scores_out, masks_out written)
int route_scores(mobi_layer* L, const __nv_bfloat16* x, int64_t T, float delta, float* scores_out, uint8_t* masks_out,
                 bool* masks_ready, cudaStream_t st, bool fuse_bucket = false) {
    *masks_ready = false;
    if (L->generic) return launch_router(L, x, T, st);  // more than 3 routed scores: CUDA-core router
    if (L->impl == 7 && router_tc_supported(L, x)) {  // traced router (development hook)
        static unsigned long long* tbuf = nullptr;
        if (!tbuf) MOBI_CUDA(cudaMalloc(&tbuf, (16 * 1024 + 16 * 1024) * sizeof(unsigned long long)));
        MOBI_CUDA(cudaMemsetAsync(tbuf, 0, (16 * 1024 + 16 * 1024) * sizeof(unsigned long long), st));
        g_trace_buf = tbuf;
        return launch_router_tc(L, x, T, delta, scores_out, masks_out, masks_ready, st, tbuf);
    }
    if (L->impl != 1 && router_tc_supported(L, x))
        return launch_router_tc(L, x, T, delta, scores_out, masks_out, masks_ready, st, nullptr, fuse_bucket);
    return launch_router(L, x, T, st);
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ---- per-stream contexts (re-entrancy, see mobi_layer in mobi_internal.cuh) ----
mobi_layer* new_context(mobi_layer* H, void* stream) {
    mobi_layer* c = new mobi_layer;
    c->device = H->device;
    c->n_sm = H->n_sm;
    c->out = H->out, c->in = H->in, c->gs = H->gs, c->G = H->G;
    c->E = H->E, c->b = H->b, c->nr = H->nr, c->h = H->h;
    c->generic = H->generic, c->sl = H->sl;
    c->out_pad = H->out_pad, c->in_pad = H->in_pad, c->kblocks = H->kblocks, c->h_pad = H->h_pad;
    c->group_shift = H->group_shift;
    c->single_group = H->single_group;
    c->codes8 = H->codes8, c->dplanes = H->dplanes, c->gconst = H->gconst;
    c->w1t = H->w1t, c->b1 = H->b1, c->w2 = H->w2, c->b2 = H->b2;
    c->mtab = H->mtab;
    c->owner = H;
    c->ctx_stream = stream;
    c->ctx_bound = true;
    c->call_mu = new std::mutex;
    return c;
}

// the context serving `stream` (created on first use); call with the handle
mobi_layer* context_for(mobi_layer* H, void* stream, int* rc) {
    *rc = MOBI_OK;
    std::lock_guard<std::mutex> g(*H->ctx_mu);
    if (!H->ctx_bound) {
        H->ctx_bound = true;
        H->ctx_stream = stream;
    }
    if (H->ctx_stream == stream) return H;
    for (mobi_layer* c : H->ctxs)
        if (c->ctx_stream == stream) return c;
    // a stream being captured into a CUDA graph cannot allocate a workspace: it records the handle's
    // own (reserved) workspace, which the graph then uses wherever it is replayed
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(reinterpret_cast<cudaStream_t>(stream), &cap) != cudaSuccess) cudaGetLastError();
    if (cap != cudaStreamCaptureStatusNone) return H;
    mobi_layer* c = new_context(H, stream);
    if (H->reserved_T > 0) *rc = ensure_ws(c, H->reserved_T);
    H->ctxs.push_back(c);
    return c;
}

// entry-point prologue: device guard + the stream's context, locked for the whole launch sequence
struct CallScope {
    DeviceGuard dg;
    mobi_layer* C = nullptr;
    std::unique_lock<std::mutex> lk;
    int rc = MOBI_OK;
    CallScope(mobi_layer* H, void* stream) : dg(H->device) {
        C = context_for(H, stream, &rc);
        lk = std::unique_lock<std::mutex>(*C->call_mu);
        C->impl = H->impl;
    }
    // the handle reports the last call's launch accounting whichever context ran it
    void publish(mobi_layer* H) {
        H->last_launches = C->last_launches;
        for (int i = 0; i < 8; ++i) H->plan[i] = C->plan[i];
        H->plan_ctx = C;
    }
};

// ---- profiling: event pairs around launches, resolved when the pool wraps or on read ----
constexpr size_t kEvPool = 4096;

void prof_resolve(mobi_layer* L) {
    if (L->ev_marks.empty()) return;
    cudaEventSynchronize(L->ev_pool[L->ev_marks.back().second.second]);
    for (auto& m : L->ev_marks) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, L->ev_pool[m.second.first], L->ev_pool[m.second.second]) == cudaSuccess) {
            L->prof_ms[m.first] += ms;
            L->prof_n[m.first] += 1;
        }
    }
    L->ev_marks.clear();
    L->ev_next = 0;
}

int prof_event(mobi_layer* L) {
    if (L->ev_next >= L->ev_pool.size()) prof_resolve(L);
    return (int)L->ev_next++;
}

struct ProfScope {
    mobi_layer* L;
    int id, a = -1;
    cudaStream_t st;
    ProfScope(mobi_layer* L_, int id_, cudaStream_t st_) : L(L_), id(id_), st(st_) {
        if (L->prof) {
            a = prof_event(L);
            cudaEventRecord(L->ev_pool[a], st);
        }
    }
    ~ProfScope() {
        if (L->prof && a >= 0) {
            int b = prof_event(L);
            if (b < a) return;  // pool wrapped between the pair: drop this sample
            cudaEventRecord(L->ev_pool[b], st);
            L->ev_marks.push_back({id, {a, b}});
        }
    }
};

int run_layer_y(mobi_layer* L, const void* x, int64_t T, float delta, const uint8_t* given_masks, void* y,
                uint8_t* masks_out, cudaStream_t st);

// Decode kernels (router GEMV + slice-plane / stream-K GEMV) for batches up to kDecodePreferT tokens (one
// slice-plane launch) when the slice-plane GEMV takes the batch, and below kDecodeMergedT tokens when only
// the stream-K merged-code GEMV does (it streams all four slices); above, the prefill path (tcgen05 router
// + gather + CTA-pair GEMM) is faster.  Measured eager, tools/small_t_probe.py, decode vs prefill path:
// q/o T=16 43.8 vs 42.8 us, T=17 51.4 vs 42.7; gate/up (merged at 16) 107.1 vs 102.7; down (merged from
// T=3) T=4 95.7 vs 111.6, T=8 113.3 vs 99.3, T=16 165.6 vs 99.5; k/v T=16 32.9 vs 41.4.  Debug impls 6 (no
// PDL), 9 (traced) and 10 run the decode kernels whenever they support the batch (T <= 32).
constexpr int64_t kDecodePreferT = 16, kDecodeMergedT = 8;
bool uses_decode(const mobi_layer* L, const void* x, int64_t Tp) {
    if (!decode_supported(L, x, Tp)) return false;
    if (L->impl == 6 || L->impl == 9 || L->impl == 10) return true;
    if (L->impl != 0 || Tp > kDecodePreferT) return false;
    return Tp < kDecodeMergedT || decode_planes_supported(L, x, Tp);
}

// the layer forward with an output descriptor: the CTA-pair GEMM places Y itself (every destination,
// from its epilogue); the small-T paths compute into a staging buffer and scatter it
int run_layer(mobi_layer* L, const void* x, int64_t T, float delta, const uint8_t* given_masks, void* y,
              uint8_t* masks_out, cudaStream_t st, const OutDesc* od = nullptr) {
    if (!od) return run_layer_y(L, x, T, delta, given_masks, y, masks_out, st);
    CHECK_ARG(od->n_dst >= 1 && od->n_dst <= MOBI_MAX_DST, "mobi_out_desc: n_dst " << od->n_dst << " outside [1,"
                                                                                    << MOBI_MAX_DST << "]");
    CHECK_ARG(od->ldy >= od->col0 + L->out && od->col0 >= 0,
              "mobi_out_desc: columns [" << od->col0 << "," << od->col0 + L->out << ") exceed ldy " << od->ldy);
    for (int k = 0; k < od->n_dst; ++k) CHECK_ARG(od->dst[k], "mobi_out_desc: null destination " << k);
    const int64_t Tp = std::max(T, L->plan_T);
    const bool pair = L->impl == 0 && !L->generic && !uses_decode(L, x, Tp);
    if (pair) {
        L->od = *od;
        const int rc = run_layer_y(L, x, T, delta, given_masks, nullptr, masks_out, st);
        L->od = OutDesc{};
        return rc;
    }
    if (T > L->y_tmp_T) {
        if (L->y_tmp) MOBI_CUDA(cudaFree(L->y_tmp));
        L->y_tmp = nullptr;
        L->y_tmp_T = 0;
        MOBI_CUDA(cudaMalloc(&L->y_tmp, (size_t)(T * L->out * 2)));
        L->y_tmp_T = T;
    }
    int rc = run_layer_y(L, x, T, delta, given_masks, L->y_tmp, masks_out, st);
    if (!rc) rc = launch_scatter_out(L->y_tmp, T, L->out, *od, st);
    if (!rc) ++L->last_launches;
    return rc;
}

int run_layer_y(mobi_layer* L, const void* x, int64_t T, float delta, const uint8_t* given_masks, void* y,
                uint8_t* masks_out, cudaStream_t st) {
    CHECK_ARG(T >= 0, "forward_elastic: negative token count " << T);
    L->last_launches = 0;
    for (int i = 0; i < 8; ++i) L->plan[i] = 0;
    L->plan[7] = (int32_t)T;
    if (T == 0) return MOBI_OK;
    int rc;
    if ((rc = ensure_ws(L, T))) return rc;
    const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(x);
    if (L->generic) {  // non-uniform widths / more than 4 slices: router -> masks -> per-slice GEMM
        if (!given_masks) {
            ProfScope p(L, 0, st);
            if ((rc = launch_router(L, xb, T, st))) return rc;
        }
        {
            ProfScope p(L, 1, st);
            if ((rc = launch_bucket_generic(L, T, delta, given_masks, nullptr, masks_out, nullptr, nullptr, nullptr, st,
                                            given_masks != nullptr)))
                return rc;
        }
        ProfScope p(L, 3, st);
        return launch_gemm_generic(L, xb, T, L->masks, reinterpret_cast<__nv_bfloat16*>(y), st);
    }
    // kernel choices follow the plan size (the whole batch when mobi_forward_host runs it in chunks)
    const int64_t Tp = std::max(T, L->plan_T);
    if (uses_decode(L, x, Tp)) {
        // decode-size batch: router GEMV -> (PDL) stream-K decode GEMM, no bucketing
        unsigned long long* tbuf = nullptr;
        if (L->impl == 9) {  // traced (development hook): per-CTA globaltimer marks
            static unsigned long long* buf = nullptr;
            if (!buf) MOBI_CUDA(cudaMalloc(&buf, (16 * 1024 + 16 * 1024) * sizeof(unsigned long long)));
            MOBI_CUDA(cudaMemsetAsync(buf, 0, (16 * 1024 + 16 * 1024) * sizeof(unsigned long long), st));
            g_trace_buf = tbuf = buf;
        }
        if (!given_masks) {  // partial scores per hidden tile; the GEMM sums them and applies gate_hard
            ProfScope p(L, 0, st);
            if ((rc = launch_router_dec(L, xb, T, delta, masks_out, nullptr, st, tbuf))) return rc;
        }
        ProfScope p(L, 3, st);
        const bool pdl = !given_masks && L->impl != 6 && !L->prof;
        if (decode_planes_supported(L, x, T))  // slice planes: stream only the slices the batch uses
            return launch_decode_planes(L, xb, T, given_masks, delta, masks_out, nullptr,
                                        reinterpret_cast<__nv_bfloat16*>(y), pdl, st, tbuf);
        return launch_decode_gemm(L, xb, T, given_masks, delta, masks_out, nullptr, reinterpret_cast<__nv_bfloat16*>(y),
                                  pdl, st, tbuf);
    }
    bool ready = false;
    if (!given_masks) {
        ProfScope p(L, 0, st);
        if ((rc = route_scores(L, xb, T, delta, nullptr, masks_out, &ready, st, L->impl != 8))) return rc;
    }
    // the tcgen05 router (prefill sizes) has already decided the masks and laid out the buckets;
    // otherwise (given masks, fallback router) the bucket kernel does it
    const bool fused = ready && L->impl != 8;
    if (!fused) {
        ProfScope p(L, 1, st);
        if ((rc = launch_bucket(L, T, delta, ready ? L->masks : given_masks, nullptr, ready ? nullptr : masks_out,
                                nullptr, nullptr, nullptr, st, !ready)))
            return rc;
    }
    {
        ProfScope p(L, 2, st);
        if ((rc = launch_gather(L, xb, T, st, fused, fused && !L->prof))) return rc;
    }
    __nv_bfloat16* yb = reinterpret_cast<__nv_bfloat16*>(y);
    if (fused && L->impl != 0 && L->impl != 3 && L->impl != 5)  // the tcgen05 GEMMs clear them
        MOBI_CUDA(cudaMemsetAsync(L->bk_hist, 0, 48 * sizeof(int32_t), st));
    ProfScope p(L, 3, st);
    if (L->impl == 1) return launch_gemm_simt(L, yb, T, st);
    if (L->impl == 2 || L->impl == 4) {  // traced tcgen05 kernels (development hook)
        static unsigned long long* tbuf = nullptr;
        if (!tbuf) MOBI_CUDA(cudaMalloc(&tbuf, (16 * 1024 + 16 * 1024) * sizeof(unsigned long long)));
        MOBI_CUDA(cudaMemsetAsync(tbuf, 0, (16 * 1024 + 16 * 1024) * sizeof(unsigned long long), st));
        g_trace_buf = tbuf;
        if (L->impl == 4) return launch_gemm_tc2(L, yb, T, st, tbuf);
        return launch_gemm_tc(L, yb, T, st, tbuf);
    }
    if (L->impl == 3) return launch_gemm_tc2(L, yb, T, st);  // CTA-pair kernel
    if (L->impl == 5) return launch_gemm_tc(L, yb, T, st);   // 1-CTA kernel (comparison)
    // production: the CTA-pair kernel (B split across the pair: half the smem operand traffic per SM) for
    // every batch above the decode sizes; at 33..64 tokens it beats the 1-CTA split-K kernel too
    // (56 vs 72-74 us at q/o 4096x4096, tools/small_t_probe.py), which stays as a comparison path
    return launch_gemm_tc2(L, yb, T, st, nullptr, !L->prof);
}

}  // namespace
}  // namespace mobi

using namespace mobi;

extern "C" {

const char* mobi_last_error(void) { return g_err.c_str(); }
const char* mobi_version(void) { return "mobi_b200 0.1 (sm_100a)"; }

int mobi_layer_debug_impl(mobi_layer_t L, int impl) {
    CHECK_ARG(L, "null layer");
    L->impl = impl;
    return MOBI_OK;
}

/* development hook: copy the last traced GEMM's per-CTA counters (16 x u64 per CTA) to host */
MOBI_API int mobi_debug_read_trace(unsigned long long* host, int n_cta) {
    if (!g_trace_buf) return set_error(MOBI_EINVAL, "no trace recorded");
    MOBI_CUDA(cudaDeviceSynchronize());
    MOBI_CUDA(cudaMemcpy(host, g_trace_buf, (size_t)(16 * 1024 + 16 * 1024) * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost));
    (void)n_cta;
    return MOBI_OK;
}

static int create_impl(const mobi_layer_desc* desc, int device, mobi_layer_t* out, bool codes_on_device) {
    CHECK_ARG(out != nullptr, "mobi_layer_create: null output handle");
    *out = nullptr;
    int ndev = 0;
    MOBI_CUDA(cudaGetDeviceCount(&ndev));
    CHECK_ARG(device >= 0 && device < ndev, "mobi_layer_create: device " << device << " out of [0," << ndev << ")");
    DeviceGuard g(device);
    int n_sm = 0;
    MOBI_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
    mobi_layer* L = new mobi_layer;
    L->device = device;
    L->n_sm = n_sm;
    L->ctx_mu = new std::mutex;
    L->call_mu = new std::mutex;
    int rc = validate_and_fill(desc, L, codes_on_device);
    if (!rc && codes_on_device) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, desc->codes) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
            pa.device != device) {
            cudaGetLastError();
            rc = set_error(MOBI_EINVAL, "mobi_layer_create_device: codes must be device memory on device " +
                                            std::to_string(device));
        }
    }
    if (!rc) rc = upload_layer(desc, L, codes_on_device);
    if (rc) {
        std::string keep = g_err;
        mobi_layer_destroy(L);
        g_err = keep;
        return rc;
    }
    *out = L;
    return MOBI_OK;
}

int mobi_layer_create(const mobi_layer_desc* desc, int device, mobi_layer_t* out) {
    return create_impl(desc, device, out, false);
}

int mobi_layer_create_rows(const mobi_layer_desc* desc, int64_t row0, int64_t row1, int device, mobi_layer_t* out) {
    CHECK_ARG(desc != nullptr && out != nullptr, "mobi_layer_create_rows: null argument");
    CHECK_ARG(0 <= row0 && row0 < row1 && row1 <= desc->out,
              "mobi_layer_create_rows: rows [" << row0 << "," << row1 << ") outside [0," << desc->out << ")");
    CHECK_ARG(desc->group_size >= 1 && desc->scale && desc->zero, "QuantParams: missing scales/zeros");
    CHECK_ARG((desc->codes != nullptr) != (desc->planes != nullptr),
              "mobi_layer_create: give exactly one of codes (SliceStack) or planes (LayerRecord)");
    // column-parallel shard: rows [row0, row1) of every slice and their groups (groups never span rows,
    // qcore.hpp:30-34); the router is the full one (replicated on every rank)
    const int64_t n = row1 - row0, G = cdiv(desc->in, desc->group_size);
    mobi_layer_desc d = *desc;
    d.out = n;
    std::vector<double> sc(desc->scale + row0 * G, desc->scale + row1 * G), ze(desc->zero + row0 * G, desc->zero + row1 * G);
    d.scale = sc.data();
    d.zero = ze.data();
    std::vector<uint8_t> codes;
    std::vector<uint64_t> planes;
    if (desc->codes) {
        CHECK_ARG(desc->n_slices >= 1, "mobi_layer_create: bad slice count");
        codes.resize((size_t)(desc->n_slices * n * desc->in));
        for (int e = 0; e < desc->n_slices; ++e)
            std::memcpy(codes.data() + (size_t)e * n * desc->in, desc->codes + ((int64_t)e * desc->out + row0) * desc->in,
                        (size_t)(n * desc->in));
        d.codes = codes.data();
    } else {
        CHECK_ARG(desc->plane_bits >= 1 && desc->words_per_row >= 1, "bitplane: bad plane geometry");
        planes.resize((size_t)(desc->plane_bits * n * desc->words_per_row));
        for (int b = 0; b < desc->plane_bits; ++b)
            std::memcpy(planes.data() + (size_t)b * n * desc->words_per_row,
                        desc->planes + ((int64_t)b * desc->out + row0) * desc->words_per_row,
                        (size_t)(n * desc->words_per_row) * 8);
        d.planes = planes.data();
    }
    return create_impl(&d, device, out, false);
}

int mobi_layer_create_device(const mobi_layer_desc* desc, int device, mobi_layer_t* out) {
    CHECK_ARG(desc && desc->codes && !desc->planes, "mobi_layer_create_device: give device slice codes");
    return create_impl(desc, device, out, true);
}

static void destroy_context(mobi_layer* c) {  // workspace + lazily built host objects; weights are the handle's
    free_ws(c);
    if (c->y_tmp) cudaFree(c->y_tmp);
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    for (auto& e : c->ev_pipe)
        if (e) cudaEventDestroy(e);
    dfree(c->gpart);
    dfree(c->hpart);
    dfree(c->dec_part);
    dfree(c->dec_spart);
    dfree(c->dec_cnt);
    if (c->tmap_w1) delete c->tmap_w1;
    if (c->tmap_w1_64) delete c->tmap_w1_64;
    if (c->x_dev) cudaFree(c->x_dev);
    if (c->y_dev) cudaFree(c->y_dev);
    if (c->h_x) cudaFreeHost(c->h_x);
    if (c->h_y) cudaFreeHost(c->h_y);
    for (auto& e : c->ev_pool) cudaEventDestroy(e);
    delete c->call_mu;
    delete c;
}

int mobi_layer_destroy(mobi_layer_t L) {
    if (!L) return MOBI_OK;
    DeviceGuard g(L->device);
    cudaDeviceSynchronize();
    for (mobi_layer* c : L->ctxs) destroy_context(c);
    L->ctxs.clear();
    if (L->y_tmp) cudaFree(L->y_tmp);
    if (L->gather_buf) cudaFree(L->gather_buf);
    delete L->ctx_mu;
    delete L->call_mu;
    free_ws(L);
    dfree(L->codes8);
    dfree(L->dplanes);
    if (L->s_h2d) cudaStreamDestroy(L->s_h2d);
    if (L->s_d2h) cudaStreamDestroy(L->s_d2h);
    for (auto& e : L->ev_pipe)
        if (e) cudaEventDestroy(e);
    dfree(L->gconst);
    dfree(L->gpart);
    dfree(L->hpart);
    dfree(L->dec_part);
    dfree(L->dec_spart);
    dfree(L->dec_cnt);
    dfree(L->w1t);
    dfree(L->b1);
    dfree(L->w2);
    dfree(L->b2);
    if (L->tmap_w1) delete L->tmap_w1;
    if (L->tmap_w1_64) delete L->tmap_w1_64;
    if (L->x_dev) cudaFree(L->x_dev);
    if (L->y_dev) cudaFree(L->y_dev);
    if (L->h_x) cudaFreeHost(L->h_x);
    if (L->h_y) cudaFreeHost(L->h_y);
    for (auto& e : L->ev_pool) cudaEventDestroy(e);
    delete L;
    return MOBI_OK;
}

int mobi_layer_reserve(mobi_layer_t L, int64_t max_tokens) {
    CHECK_ARG(L, "null layer");
    CHECK_ARG(max_tokens >= 0, "mobi_layer_reserve: negative token count");
    DeviceGuard g(L->device);
    std::lock_guard<std::mutex> lk(*L->ctx_mu);
    L->reserved_T = std::max(L->reserved_T, max_tokens);
    int rc = ensure_ws(L, max_tokens);
    for (mobi_layer* c : L->ctxs)
        if (!rc) rc = ensure_ws(c, max_tokens);
    return rc;
}

int mobi_layers_share_activations(mobi_layer_t* layers, int32_t n) {
    CHECK_ARG(layers && n >= 1, "mobi_layers_share_activations: no layers");
    size_t bytes = 0;
    for (int32_t i = 0; i < n; ++i) {
        CHECK_ARG(layers[i], "mobi_layers_share_activations: null layer " << i);
        CHECK_ARG(layers[i]->device == layers[0]->device, "mobi_layers_share_activations: layers on different devices");
        CHECK_ARG(layers[i]->ws_T > 0, "mobi_layers_share_activations: layer " << i << " not reserved");
        bytes = std::max(bytes, (size_t)(layers[i]->tpad_max * layers[i]->in_pad) * sizeof(__half));
    }
    DeviceGuard g(layers[0]->device);
    MOBI_CUDA(cudaDeviceSynchronize());  // queued work may still use the buffers being replaced
    void* p = nullptr;
    MOBI_CUDA(cudaMalloc(&p, bytes));
    std::shared_ptr<void> blk(p, [](void* q) { cudaFree(q); });
    for (int32_t i = 0; i < n; ++i) {
        mobi_layer* L = layers[i];
        std::lock_guard<std::mutex> lk(*L->ctx_mu);
        if (L->xperm_shared)
            L->xperm_shared.reset();
        else
            dfree(L->xperm);
        L->xperm = reinterpret_cast<__half*>(p);
        L->xperm_shared = blk;
        if (L->tmap_x) delete L->tmap_x;  // tensor maps encode the old address
        L->tmap_x = nullptr;
        if (L->tmap_x2) delete[] L->tmap_x2;
        L->tmap_x2 = nullptr;
    }
    return MOBI_OK;
}

int mobi_layer_info(mobi_layer_t L, int64_t* out, int64_t* in, int32_t* n_slices, int64_t* router_hidden,
                    int64_t* device_bytes) {
    CHECK_ARG(L, "null layer");
    if (out) *out = L->out;
    if (in) *in = L->in;
    if (n_slices) *n_slices = L->E;
    if (router_hidden) *router_hidden = L->h;
    if (device_bytes) *device_bytes = L->device_bytes;
    return MOBI_OK;
}

int mobi_layer_export_router(mobi_layer_t L, float* w1, float* b1, float* w2, float* b2) {
    CHECK_ARG(L, "null layer");
    DeviceGuard g(L->device);
    std::vector<uint16_t> w1t((size_t)(L->h_pad * L->in_pad));
    MOBI_CUDA(cudaMemcpy(w1t.data(), L->w1t, w1t.size() * 2, cudaMemcpyDeviceToHost));
    if (w1)
        for (int64_t k = 0; k < L->in; ++k)
            for (int64_t j = 0; j < L->h; ++j) w1[k * L->h + j] = bf2f(w1t[(size_t)(j * L->in_pad + k)]);
    if (b1) MOBI_CUDA(cudaMemcpy(b1, L->b1, L->h * 4, cudaMemcpyDeviceToHost));
    if (w2) MOBI_CUDA(cudaMemcpy(w2, L->w2, L->h * L->nr * 4, cudaMemcpyDeviceToHost));
    if (b2) MOBI_CUDA(cudaMemcpy(b2, L->b2, L->nr * 4, cudaMemcpyDeviceToHost));
    return MOBI_OK;
}

int mobi_layer_unpack_codes(mobi_layer_t L, uint8_t* codes_host) {
    CHECK_ARG(L && codes_host, "mobi_layer_unpack_codes: null argument");
    DeviceGuard g(L->device);
    uint8_t* tmp = nullptr;
    const size_t n = (size_t)(L->E * L->out * L->in);
    int rc;
    if ((rc = dmalloc(&tmp, n, nullptr))) return rc;
    rc = launch_unpack_codes(L, tmp, 0);
    if (!rc) {
        cudaError_t e = cudaMemcpy(codes_host, tmp, n, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = set_error(MOBI_ERUNTIME, cudaGetErrorString(e));
    }
    dfree(tmp);
    return rc;
}

int mobi_score(mobi_layer_t H, const void* x, int64_t T, float* scores, void* stream) {
    CHECK_ARG(H, "null layer");
    CHECK_ARG(T >= 0, "score: negative token count");
    if (T == 0) return MOBI_OK;
    CallScope cs(H, stream);
    if (cs.rc) return cs.rc;
    mobi_layer* L = cs.C;
    int rc;
    if ((rc = ensure_ws(L, T))) return rc;
    L->last_launches = 0;
    bool ready = false;
    if ((rc = route_scores(L, reinterpret_cast<const __nv_bfloat16*>(x), T, INFINITY, scores, nullptr, &ready, S(stream))))
        return rc;
    if (L->generic)
        rc = launch_bucket_generic(L, T, INFINITY, nullptr, scores, nullptr, nullptr, nullptr, nullptr, S(stream), false);
    else if (!ready)
        rc = launch_bucket(L, T, INFINITY, nullptr, scores, nullptr, nullptr, nullptr, nullptr, S(stream));
    cs.publish(H);
    return rc;
}

int mobi_route(mobi_layer_t H, const void* x, int64_t T, float delta, float* scores, uint8_t* masks, int32_t* perm,
               int32_t* inverse, int32_t* bucket_count, void* stream) {
    CHECK_ARG(H, "null layer");
    CHECK_ARG(T >= 0, "score: negative token count");
    if (T == 0) return MOBI_OK;
    CallScope cs(H, stream);
    if (cs.rc) return cs.rc;
    mobi_layer* L = cs.C;
    int rc;
    if ((rc = ensure_ws(L, T))) return rc;
    L->last_launches = 0;
    bool ready = false;
    if ((rc = route_scores(L, reinterpret_cast<const __nv_bfloat16*>(x), T, delta, scores, masks, &ready, S(stream))))
        return rc;
    if (L->generic) {
        rc = launch_bucket_generic(L, T, delta, nullptr, scores, masks, perm, inverse, bucket_count, S(stream), false);
        cs.publish(H);
        return rc;
    }
    rc = launch_bucket(L, T, delta, ready ? L->masks : nullptr, ready ? nullptr : scores, ready ? nullptr : masks, perm,
                       inverse, bucket_count, S(stream), !ready);
    cs.publish(H);
    return rc;
}

int mobi_forward(mobi_layer_t H, const void* x, int64_t T, float delta, void* y, uint8_t* masks, void* stream) {
    CHECK_ARG(H, "null layer");
    CallScope cs(H, stream);
    if (cs.rc) return cs.rc;
    const int rc = run_layer(cs.C, x, T, delta, nullptr, y, masks, S(stream));
    cs.publish(H);
    return rc;
}

int mobi_forward_masked(mobi_layer_t H, const void* x, int64_t T, const uint8_t* masks, void* y, void* stream) {
    CHECK_ARG(H, "null layer");
    CHECK_ARG(masks != nullptr || T == 0, "forward_elastic: null gate masks");
    CallScope cs(H, stream);
    if (cs.rc) return cs.rc;
    const int rc = run_layer(cs.C, x, T, 0.f, masks, y, nullptr, S(stream));
    cs.publish(H);
    return rc;
}

}  // extern "C"
namespace mobi {
int run_layer_entry(mobi_layer* H, const void* x, int64_t T, float delta, void* y, uint8_t* masks, cudaStream_t st,
                    const OutDesc* od) {
    CallScope cs(H, st);
    if (cs.rc) return cs.rc;
    const int rc = run_layer(cs.C, x, T, delta, nullptr, y, masks, st, od);
    cs.publish(H);
    return rc;
}
}  // namespace mobi
extern "C" {

int mobi_forward_out(mobi_layer_t H, const void* x, int64_t T, float delta, const mobi_out_desc* out, uint8_t* masks,
                     void* stream) {
    CHECK_ARG(H && out, "mobi_forward_out: null argument");
    OutDesc od{};
    CHECK_ARG(out->n_dst >= 1 && out->n_dst <= MOBI_MAX_DST,
              "mobi_out_desc: n_dst " << out->n_dst << " outside [1," << MOBI_MAX_DST << "]");
    od.n_dst = out->n_dst;
    for (int k = 0; k < od.n_dst; ++k) od.dst[k] = reinterpret_cast<__nv_bfloat16*>(out->dst[k]);
    od.ldy = out->ldy;
    od.col0 = out->col0;
    CallScope cs(H, stream);
    if (cs.rc) return cs.rc;
    const int rc = run_layer(cs.C, x, T, delta, nullptr, nullptr, masks, S(stream), &od);
    cs.publish(H);
    return rc;
}

int mobi_forward_host(mobi_layer_t H, const void* x_host, int64_t T, float delta, void* y_host, uint8_t* masks_host,
                      void* stream) {
    CHECK_ARG(H && x_host && y_host, "mobi_forward_host: null argument");
    CHECK_ARG(T >= 0, "forward_elastic: negative token count " << T);
    if (T == 0) return MOBI_OK;
    CallScope cs(H, stream);
    if (cs.rc) return cs.rc;
    mobi_layer* L = cs.C;
    cudaStream_t st = S(stream);
    const size_t xb = (size_t)(T * L->in * 2), yb = (size_t)(T * L->out * 2);
    if (T > L->h_cap) {
        if (L->x_dev) cudaFree(L->x_dev);
        if (L->y_dev) cudaFree(L->y_dev);
        if (L->h_x) cudaFreeHost(L->h_x);
        if (L->h_y) cudaFreeHost(L->h_y);
        L->x_dev = L->y_dev = L->h_x = L->h_y = nullptr;
        MOBI_CUDA(cudaMalloc(&L->x_dev, xb + T));
        MOBI_CUDA(cudaMalloc(&L->y_dev, yb));
        MOBI_CUDA(cudaMallocHost(&L->h_x, xb));
        MOBI_CUDA(cudaMallocHost(&L->h_y, yb + T));
        L->h_cap = T;
    }
    auto pinned = [](const void* p) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    };
    const bool xp = pinned(x_host), yp = pinned(y_host);
    const void* xsrc = x_host;
    if (!xp) {
        std::memcpy(L->h_x, x_host, xb);
        xsrc = L->h_x;
    }
    uint8_t* mdev = masks_host ? reinterpret_cast<uint8_t*>(L->x_dev) + xb : nullptr;
    void* ydst = yp ? y_host : L->h_y;
    // token chunks pipelined over three streams: the host->device copy of chunk i+1 and the
    // device->host copy of chunk i-1 overlap the forward of chunk i.  Tokens are independent and
    // every chunk runs the kernels the whole batch would (plan_T = T: router variant, cluster K-split
    // and GEMM path are chosen from the batch size; no chunk is shorter than 256 tokens), so the
    // chunked result is bit-identical to one whole-batch mobi_forward.
    static const int nch_env = [] {  // development knob: MOBI_E2E_CHUNKS overrides the chunk count
        const char* e = std::getenv("MOBI_E2E_CHUNKS");
        return e ? std::max(1, std::min(8, std::atoi(e))) : 0;
    }();
    const int nch = nch_env ? (int)std::min<int64_t>(nch_env, std::max<int64_t>(1, T / 256))
                            : (T >= 2048 ? 4 : (T >= 1024 ? 2 : 1));
    if (nch > 1 && !L->s_h2d) {
        MOBI_CUDA(cudaStreamCreateWithFlags(&L->s_h2d, cudaStreamNonBlocking));
        MOBI_CUDA(cudaStreamCreateWithFlags(&L->s_d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 17; ++i) MOBI_CUDA(cudaEventCreateWithFlags(&L->ev_pipe[i], cudaEventDisableTiming));
    }
    if (nch == 1) {
        MOBI_CUDA(cudaMemcpyAsync(L->x_dev, xsrc, xb, cudaMemcpyHostToDevice, st));
        int rc = run_layer(L, L->x_dev, T, delta, nullptr, L->y_dev, mdev, st);
        if (rc) return rc;
        MOBI_CUDA(cudaMemcpyAsync(ydst, L->y_dev, yb, cudaMemcpyDeviceToHost, st));
        if (masks_host) MOBI_CUDA(cudaMemcpyAsync(masks_host, mdev, (size_t)T, cudaMemcpyDeviceToHost, st));
    } else {
        const int64_t step = round_up(cdiv(T, (int64_t)nch), 256);
        cudaEvent_t* ev = L->ev_pipe;  // [0..7] copied in, [8..15] computed, [16] prior work
        MOBI_CUDA(cudaEventRecord(ev[16], st));  // prior work on the caller's stream
        MOBI_CUDA(cudaStreamWaitEvent(L->s_h2d, ev[16], 0));
        struct PlanScope {  // kernels chosen for the whole batch while the chunks run
            mobi_layer* L;
            ~PlanScope() { L->plan_T = 0; }
        } ps{L};
        L->plan_T = T;
        int rc = ensure_ws(L, step + 256);  // the largest chunk (a folded tail adds < 256 tokens)
        if (rc) return rc;
        int c = 0;
        for (int64_t t0 = 0; t0 < T && !rc; ++c) {
            int64_t n = std::min(step, T - t0);
            if (T - (t0 + n) < 256) n = T - t0;  // fold a short tail into this chunk
            const size_t xo = (size_t)(t0 * L->in * 2), yo = (size_t)(t0 * L->out * 2);
            MOBI_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(L->x_dev) + xo,
                                      reinterpret_cast<const uint8_t*>(xsrc) + xo, (size_t)(n * L->in * 2),
                                      cudaMemcpyHostToDevice, L->s_h2d));
            MOBI_CUDA(cudaEventRecord(ev[c], L->s_h2d));
            MOBI_CUDA(cudaStreamWaitEvent(st, ev[c], 0));
            rc = run_layer(L, reinterpret_cast<uint8_t*>(L->x_dev) + xo, n, delta, nullptr,
                           reinterpret_cast<uint8_t*>(L->y_dev) + yo, mdev ? mdev + t0 : nullptr, st);
            if (rc) break;
            MOBI_CUDA(cudaEventRecord(ev[8 + c], st));
            MOBI_CUDA(cudaStreamWaitEvent(L->s_d2h, ev[8 + c], 0));
            MOBI_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(ydst) + yo,
                                      reinterpret_cast<const uint8_t*>(L->y_dev) + yo, (size_t)(n * L->out * 2),
                                      cudaMemcpyDeviceToHost, L->s_d2h));
            if (masks_host)
                MOBI_CUDA(cudaMemcpyAsync(masks_host + t0, mdev + t0, (size_t)n, cudaMemcpyDeviceToHost, L->s_d2h));
            t0 += n;
        }
        if (rc) return rc;
        MOBI_CUDA(cudaStreamSynchronize(L->s_d2h));
    }
    MOBI_CUDA(cudaStreamSynchronize(st));
    if (!yp) std::memcpy(y_host, L->h_y, yb);
    return MOBI_OK;
}

int mobi_ipc_export(void* dev_ptr, void* handle64, int64_t* offset) {
    CHECK_ARG(dev_ptr && handle64 && offset, "mobi_ipc_export: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    // the handle names the whole allocation (e.g. a caching allocator's block): report dev_ptr's offset
    typedef CUresult (*PFN_range)(CUdeviceptr*, size_t*, CUdeviceptr);
    static PFN_range range = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
        return reinterpret_cast<PFN_range>(f);
    }();
    CUdeviceptr base = 0;
    size_t size = 0;
    if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return set_error(MOBI_ERUNTIME, "mobi_ipc_export: cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    MOBI_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle64, &h, sizeof(h));
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    return MOBI_OK;
}

int mobi_ipc_open(const void* handle64, int device, void** dev_ptr) {
    CHECK_ARG(handle64 && dev_ptr, "mobi_ipc_open: null argument");
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    MOBI_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return MOBI_OK;
}

int mobi_ipc_close(void* dev_ptr) {
    CHECK_ARG(dev_ptr, "mobi_ipc_close: null argument");
    MOBI_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return MOBI_OK;
}

int mobi_permute_by_slice(const uint8_t* masks, int64_t T, int32_t* perm, int32_t* inverse, uint8_t* group_mask,
                          int64_t* group_len, int64_t* n_groups, void* stream) {
    CHECK_ARG(T >= 0, "permute_by_slice: negative token count");
    if (n_groups) *n_groups = 0;
    if (T == 0) return MOBI_OK;
    cudaStream_t st = S(stream);
    uint8_t* keys = nullptr;
    int32_t* hist = nullptr;
    MOBI_CUDA(cudaMallocAsync(&keys, (size_t)T, st));
    MOBI_CUDA(cudaMallocAsync(&hist, 256 * sizeof(int32_t), st));
    int rc = launch_permute(masks, T, keys, perm, inverse, hist, st);
    int32_t h[256];
    if (!rc) {
        cudaError_t e = cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = set_error(MOBI_ERUNTIME, cudaGetErrorString(e));
    }
    cudaFreeAsync(keys, st);
    cudaFreeAsync(hist, st);
    if (rc) return rc;
    int64_t ng = 0;
    for (int v = 0; v < 256; ++v)
        if (h[v]) {
            if (group_mask) group_mask[ng] = (uint8_t)v;
            if (group_len) group_len[ng] = h[v];
            ++ng;
        }
    if (n_groups) *n_groups = ng;
    return MOBI_OK;
}

int mobi_calibrate_threshold(const float* scores, int64_t n, double rho, double* delta, void* stream) {
    CHECK_ARG(n > 0, "calibrate_threshold: empty score sample");
    CHECK_ARG(rho >= 0.0 && rho <= 1.0, "calibrate_threshold: rho " << rho << " outside [0,1]");
    CHECK_ARG(delta && scores, "calibrate_threshold: null argument");
    // router.hpp:167-174: sort descending, delta = s[floor(rho*N + 1e-9)], or min - 1 past the end;
    // the rank is selected on the device (radix select, select.cu), bit-identical to sorting
    const int64_t k = (int64_t)std::floor(rho * (double)n + 1e-9);
    float v = 0.f;
    MOBI_TRY(launch_select_desc(scores, n, std::min(k, n - 1), &v, S(stream)));
    *delta = k >= n ? (double)v - 1.0 : (double)v;
    return MOBI_OK;
}

int mobi_avg_bits(const uint8_t* masks, int64_t T, const int32_t* slice_bits, int32_t n_slices, double* avg,
                  void* stream) {
    CHECK_ARG(avg && slice_bits, "avg_bits: null argument");
    CHECK_ARG(n_slices >= 1 && n_slices <= 8, "avg_bits: " << n_slices << " slices");
    CHECK_ARG(T >= 0 && (T == 0 || masks), "avg_bits: bad gate matrix");
    if (T == 0) {
        *avg = (double)slice_bits[0];
        return MOBI_OK;
    }
    return launch_avg_bits(masks, T, slice_bits, n_slices, avg, S(stream));
}

int mobi_decompose(const double* w, int64_t out, int64_t in, int64_t group_size, const int32_t* slice_bits,
                   int32_t n_slices, double gamma, uint8_t* codes, double* scale, double* zero, int64_t* clamp_counts,
                   void* stream) {
    CHECK_ARG(w && codes && scale && zero && slice_bits, "decompose: null argument");
    return launch_decompose(w, out, in, group_size, slice_bits, n_slices, gamma, codes, scale, zero, clamp_counts,
                            S(stream));
}

int mobi_joint_step(const double* w, int64_t out, int64_t in, int64_t group_size, const int32_t* slice_bits,
                    int32_t n_slices, const double* gamma_lo, const double* gamma_hi, const double* w1, const double* b1,
                    const double* w2, const double* b2, int64_t hidden, const double* x, const double* y_fp, int64_t T,
                    const mobi_budget_schedule* sched, int64_t t, int32_t force_gates_on, double* y_hat,
                    mobi_joint_scalars* scalars, double* d_gamma_lo, double* d_gamma_hi, double* d_w1, double* d_b1,
                    double* d_w2, double* d_b2, void* stream) {
    CHECK_ARG(w && slice_bits && gamma_lo && gamma_hi && x && y_fp && sched && scalars, "joint_step: null argument");
    CHECK_ARG(force_gates_on || (w1 && b1 && w2 && b2), "joint_step: null router argument");
    CHECK_ARG(!d_gamma_lo || (d_gamma_hi && d_w1 && d_b1 && d_w2 && d_b2), "joint_step: null gradient argument");
    CHECK_ARG(out > 0 && in > 0 && group_size > 0 && T > 0 && hidden > 0, "joint_step: empty dimension");
    CHECK_ARG(n_slices >= 2 && n_slices <= MOBI_MAX_SLICES, "joint_step: need 2.." << MOBI_MAX_SLICES << " slices");
    int total = 0;
    for (int e = 0; e < n_slices; ++e) {
        CHECK_ARG(slice_bits[e] >= 1 && slice_bits[e] <= 8, "joint_step: slice bit width " << slice_bits[e]);
        total += slice_bits[e];
    }
    CHECK_ARG(total <= 8, "joint_step: total bits " << total << " exceed the 8-bit code budget");
    CHECK_ARG(sched->total_steps >= 1 && sched->shape >= 0 && sched->shape <= 3, "joint_step: bad schedule");
    CHECK_ARG(t >= 1 && t <= sched->total_steps,
              "schedule_value: step " << t << " outside [1," << sched->total_steps << "]");
    CHECK_ARG(sched->shape != 3 || (sched->b_init > 0.0 && sched->b_target > 0.0),
              "schedule_value: exponential shape needs positive bits");
    return joint_step(w, out, in, group_size, slice_bits, n_slices, gamma_lo, gamma_hi, w1, b1, w2, b2, hidden, x,
                      y_fp, T, sched, t, force_gates_on, y_hat, scalars, d_gamma_lo, d_gamma_hi, d_w1, d_b1, d_w2,
                      d_b2, S(stream));
}

int mobi_msb_step(const double* w, int64_t out, int64_t in, int64_t group_size, int32_t msb_bits,
                  const double* gamma_lo, const double* gamma_hi, const double* x, const double* y_fp, int64_t T,
                  double* y_msb, double* loss, double* d_gamma_lo, double* d_gamma_hi, void* stream) {
    CHECK_ARG(w && gamma_lo && gamma_hi && x && y_fp && loss, "msb_step: null argument");
    CHECK_ARG(!d_gamma_lo == !d_gamma_hi, "msb_step: null gradient argument");
    CHECK_ARG(out > 0 && in > 0 && group_size > 0 && T > 0, "msb_step: empty dimension");
    CHECK_ARG(msb_bits >= 1 && msb_bits <= 8, "msb_step: slice bit width " << msb_bits);
    // stage 1 = the joint step's machinery on slice 1 alone: decompose's first slice is
    // quantize_floor(w, base) (slicer.hpp:86-100 vs qcore.hpp:157-176), no router, loss = MSE
    const mobi_budget_schedule one{0.0, 0.0, 1, 0, 0.0};
    mobi_joint_scalars r{};
    const int rc = joint_step(w, out, in, group_size, &msb_bits, 1, gamma_lo, gamma_hi, nullptr, nullptr, nullptr,
                              nullptr, 1, x, y_fp, T, &one, 1, 1, y_msb, &r, d_gamma_lo, d_gamma_hi, nullptr, nullptr,
                              nullptr, nullptr, S(stream), true);
    *loss = r.data_term;
    return rc;
}

int mobi_layer_profile(mobi_layer_t L, int enable) {
    CHECK_ARG(L, "null layer");
    DeviceGuard g(L->device);
    if (L->ev_pool.empty() && enable) {
        L->ev_pool.resize(kEvPool);
        for (auto& e : L->ev_pool) MOBI_CUDA(cudaEventCreate(&e));
    }
    if (L->prof) prof_resolve(L);
    L->ev_marks.clear();
    L->ev_next = 0;
    for (int i = 0; i < MOBI_PROF_KERNELS; ++i) {
        L->prof_ms[i] = 0.0;
        L->prof_n[i] = 0;
    }
    L->prof = enable != 0;
    return MOBI_OK;
}

int mobi_layer_profile_read(mobi_layer_t L, double* ms, int64_t* launches) {
    CHECK_ARG(L, "null layer");
    DeviceGuard g(L->device);
    prof_resolve(L);
    for (int i = 0; i < MOBI_PROF_KERNELS; ++i) {
        if (ms) ms[i] = L->prof_ms[i];
        if (launches) launches[i] = L->prof_n[i];
    }
    return MOBI_OK;
}

int mobi_layer_last_launches(mobi_layer_t L, int32_t* launches) {
    CHECK_ARG(L && launches, "null argument");
    *launches = L->last_launches;
    return MOBI_OK;
}

int mobi_layer_last_plan(mobi_layer_t L, int32_t* plan) {
    CHECK_ARG(L && plan, "null argument");
    DeviceGuard g(L->device);
    for (int i = 0; i < 8; ++i) plan[i] = L->plan[i];
    plan[3] = L->last_launches;
    plan[4] = plan[6] = -1;
    plan[5] = (int32_t)(L->out_pad / (2 * kRowTile));
    mobi_layer* c = L->plan_ctx ? L->plan_ctx : L;
    if ((plan[1] == MOBI_K_GEMM_PAIR || plan[1] == MOBI_K_GEMM_SPLITK || plan[1] == MOBI_K_GEMM_SIMT) && c->meta) {
        int32_t n = 0;
        MOBI_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(c->ctx_stream)));
        MOBI_CUDA(cudaMemcpy(&n, c->meta, sizeof(n), cudaMemcpyDeviceToHost));
        plan[4] = n;
        plan[6] = n * plan[5];
    }
    return MOBI_OK;
}

}  // extern "C"
