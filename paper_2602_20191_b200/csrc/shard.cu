// shard.cu -- the multi-GPU entry of the C ABI: a layer partitioned over the ranks of
// a caller-provided NCCL communicator, one process per GPU.
//
//   COLUMN: rank p owns weight rows [p*per, min(out, (p+1)*per)) of every slice and their groups
//           (groups never span rows, qcore.hpp:30-34; per = ceil(out/P) rounded to 128) and the full
//           router (every rank decides the same masks).  The GEMM epilogue writes the rank's
//           [T, per] block straight into its slot of a rank-major [P][T][per] buffer, one in-place
//           ncclAllGather fills the other slots, and one pass interleaves it into the caller's
//           [T, out].  (The fused alternative -- epilogue stores into every rank's [T, out] over
//           NVLink -- is mobi_forward_out with peer destinations, sharding.py "peer" mode.)
//   TOKEN:  replicated weights; every rank forwards its own tokens, no collective.
//
// NCCL is resolved at run time (the process's libnccl if one is loaded -- e.g. torch's -- else
// libnccl.so.2), so the library itself carries no NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <sstream>

#include "mobi_internal.cuh"

namespace mobi {
int run_layer_entry(mobi_layer* H, const void* x, int64_t T, float delta, void* y, uint8_t* masks, cudaStream_t st,
                    const OutDesc* od);

namespace {

typedef ncclResult_t (*PFN_allgather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
typedef const char* (*PFN_errstr)(ncclResult_t);

struct Nccl {
    PFN_allgather allgather = nullptr;
    PFN_errstr errstr = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* a = dlsym(RTLD_DEFAULT, "ncclAllGather");
        void* e = dlsym(RTLD_DEFAULT, "ncclGetErrorString");
        if (!a) {
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (h) {
                a = dlsym(h, "ncclAllGather");
                e = dlsym(h, "ncclGetErrorString");
            }
        }
        n.allgather = reinterpret_cast<PFN_allgather>(a);
        n.errstr = reinterpret_cast<PFN_errstr>(e);
    });
    return n;
}

// gathered [P][T][per] (rank-major) -> y [T][out]
__global__ void interleave_kernel(const __nv_bfloat16* __restrict__ g, int64_t T, int64_t per, int64_t out,
                                  __nv_bfloat16* __restrict__ y) {
    const int64_t t = blockIdx.x;
    const int p = blockIdx.y;
    const int64_t c0 = (int64_t)p * per;
    const int64_t n = std::min<int64_t>(per, out - c0);
    if (n <= 0) return;
    const __nv_bfloat16* src = g + ((int64_t)p * T + t) * per;
    __nv_bfloat16* dst = y + t * out + c0;
    if ((per % 8) == 0 && (out % 8) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (n % 8) == 0) {
        for (int64_t c = 8 * threadIdx.x; c < n; c += 8 * blockDim.x)
            *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(src + c);
    } else {
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) dst[c] = src[c];
    }
}

}  // namespace
}  // namespace mobi

using namespace mobi;

extern "C" {

int mobi_layer_create_sharded(const mobi_layer_desc* desc, void* nccl_comm, int rank, int nranks, int mode,
                              int device, mobi_layer_t* out) {
    if (!desc || !out) return set_error(MOBI_EINVAL, "mobi_layer_create_sharded: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(MOBI_EINVAL, "mobi_layer_create_sharded: rank " + std::to_string(rank) + " outside [0," +
                                          std::to_string(nranks) + ")");
    if (mode != MOBI_SHARD_COLUMN && mode != MOBI_SHARD_TOKEN)
        return set_error(MOBI_EINVAL, "mobi_layer_create_sharded: unknown mode " + std::to_string(mode));
    if (nranks > 1 && !nccl_comm) return set_error(MOBI_EINVAL, "mobi_layer_create_sharded: null NCCL communicator");
    if (nranks > 1 && !nccl().allgather)
        return set_error(MOBI_ERUNTIME, "mobi_layer_create_sharded: NCCL (libnccl.so.2) not found");
    *out = nullptr;
    mobi_layer_t L = nullptr;
    int64_t per = desc->out, r0 = 0, r1 = desc->out;
    int rc;
    if (mode == MOBI_SHARD_COLUMN) {
        per = round_up(cdiv(desc->out, nranks), kRowTile);
        r0 = std::min<int64_t>(desc->out, (int64_t)rank * per);
        r1 = std::min<int64_t>(desc->out, r0 + per);
        if (r1 <= r0)
            return set_error(MOBI_EINVAL, "column-parallel: rank " + std::to_string(rank) + " of " +
                                              std::to_string(nranks) + " owns no rows of " + std::to_string(desc->out));
        rc = mobi_layer_create_rows(desc, r0, r1, device, &L);
    } else {
        rc = mobi_layer_create(desc, device, &L);
    }
    if (rc) return rc;
    L->shard_mode = mode;
    L->shard_rank = rank;
    L->shard_nranks = nranks;
    L->shard_comm = nccl_comm;
    L->shard_per = per;
    L->shard_out = desc->out;
    *out = L;
    return MOBI_OK;
}

int mobi_forward_sharded(mobi_layer_t L, const void* x, int64_t T, float delta, void* y, uint8_t* masks,
                         void* stream) {
    if (!L || (T > 0 && (!x || !y))) return set_error(MOBI_EINVAL, "mobi_forward_sharded: null argument");
    if (L->shard_mode == 0) return set_error(MOBI_EINVAL, "mobi_forward_sharded: layer was not created sharded");
    if (T < 0) return set_error(MOBI_EINVAL, "forward_elastic: negative token count " + std::to_string(T));
    if (T == 0) return MOBI_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (L->shard_mode == MOBI_SHARD_TOKEN)  // this rank's tokens, no collective
        return run_layer_entry(L, x, T, delta, y, masks, st, nullptr);
    const int P = L->shard_nranks, p = L->shard_rank;
    const int64_t per = L->shard_per;
    {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != L->device) cudaSetDevice(L->device);
        if (T > L->gather_T) {
            if (L->gather_buf) cudaFree(L->gather_buf);
            L->gather_buf = nullptr;
            L->gather_T = 0;
            MOBI_CUDA(cudaMalloc(&L->gather_buf, (size_t)(P * T * per) * 2));
            MOBI_CUDA(cudaMemset(L->gather_buf, 0, (size_t)(P * T * per) * 2));  // shard padding stays 0
            L->gather_T = T;
        }
        if (cur != L->device) cudaSetDevice(cur);
    }
    __nv_bfloat16* g = L->gather_buf;
    OutDesc od{};
    od.n_dst = 1;
    od.dst[0] = g + (int64_t)p * T * per;  // this rank's slot of the rank-major buffer
    od.ldy = per;
    od.col0 = 0;
    int rc = run_layer_entry(L, x, T, delta, nullptr, masks, st, &od);
    if (rc) return rc;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != L->device) cudaSetDevice(L->device);
    if (P > 1) {
        const ncclResult_t r = nccl().allgather(g + (int64_t)p * T * per, g, (size_t)(T * per), ncclBfloat16,
                                                reinterpret_cast<ncclComm_t>(L->shard_comm), st);
        if (r != ncclSuccess) {
            if (cur != L->device) cudaSetDevice(cur);
            return set_error(MOBI_ERUNTIME, std::string("ncclAllGather: ") +
                                                (nccl().errstr ? nccl().errstr(r) : std::to_string((int)r)));
        }
    }
    interleave_kernel<<<dim3((unsigned)T, (unsigned)P), 256, 0, st>>>(g, T, per, L->shard_out,
                                                                      reinterpret_cast<__nv_bfloat16*>(y));
    const cudaError_t e = cudaGetLastError();
    if (cur != L->device) cudaSetDevice(cur);
    if (e != cudaSuccess) return set_error(MOBI_ERUNTIME, std::string("interleave: ") + cudaGetErrorString(e));
    return MOBI_OK;
}

}  // extern "C"
