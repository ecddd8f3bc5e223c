// adop_comm.cu -- the library's own NCCL communicator (include/adop.h "Multi-GPU"): the collectives of the
// two partitionings of the north star, run by adop_rasterize_forward / _backward between
// their phases when a communicator is passed:
//   ADOP_SHARD_POINTS (BASELINE configs[3]): after the depth pass a MIN all-reduce of every view's 64-bit keys
//     (R8: the int64 order equals the uint64 order) -- or, with ADOP_COMM_KEYS32, of only the 32-bit depth
//     words (packed into a contiguous scratch buffer by k_hi_pack) --, after the blend a SUM all-reduce of
//     accum and count; the backward sums d_pose (and d_intrinsics) over the shards.
//   ADOP_SHARD_VIEWS (BASELINE configs[4]): the forward is local; the backward sums d_feat, d_pos (and d_env)
//     over the ranks (each rank owns a range of views of the batch; d_pose rows stay with their view's rank).
// NCCL is resolved at run time (dlopen of libnccl.so.2, the library a torch process has already loaded), so
// libadop.so does not depend on it unless a communicator is created.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <mutex>
#include <new>
#include <nccl.h>

#include "adop_internal.h"

struct adop_comm {
    ncclComm_t nccl;
    int32_t nranks, rank, mode, flags, device;
    void *scratch;          // ADOP_COMM_KEYS32: contiguous depth words of one view
    size_t scratch_bytes;
};

namespace adop {
namespace {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId *);
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*commDestroy)(ncclComm_t);
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*groupStart)();
    ncclResult_t (*groupEnd)();
    const char *(*getErrorString)(ncclResult_t);
    bool ok;
};

const NcclApi &nccl() {
    static NcclApi api{};
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
        api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
        api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.groupStart &&
                 api.groupEnd && api.getErrorString;
    });
    return api;
}

adop_status nccl_fail(ncclResult_t r, const char *what) {
    char msg[256];
    std::snprintf(msg, sizeof(msg), "%s: %s", what, nccl().ok ? nccl().getErrorString(r) : "NCCL unavailable");
    return set_status(ADOP_ERR_NCCL, msg);
}

// bits(z) word (high half, little endian) of every key <-> a contiguous int32 buffer
__global__ void k_hi_pack(const uint32_t *keys32, int32_t *hi, int64_t P) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P; q += (int64_t)gridDim.x * blockDim.x)
        hi[q] = (int32_t)keys32[2 * q + 1];
}
__global__ void k_hi_unpack(uint32_t *keys32, const int32_t *hi, int64_t P) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P; q += (int64_t)gridDim.x * blockDim.x)
        keys32[2 * q + 1] = (uint32_t)hi[q];
}

}  // namespace

adop_status comm_check(const adop_comm *comm) {
    if (!comm) return ADOP_OK;
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != comm->device) return set_status(ADOP_ERR_INVALID_ARGUMENT, "comm belongs to another device");
    return ADOP_OK;
}

// After the depth pass (point sharding): keys MIN over the shards.
adop_status comm_keys(adop_comm *comm, const adop_pyramid *views, const int64_t *pixels, int32_t n_views,
                      void *stream) {
    if (!comm || comm->mode != ADOP_SHARD_POINTS) return ADOP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const NcclApi &n = nccl();
    if (comm->flags & ADOP_COMM_KEYS32) {
        int64_t maxP = 0;
        for (int v = 0; v < n_views; ++v) maxP = pixels[v] > maxP ? pixels[v] : maxP;
        const size_t need = (size_t)maxP * sizeof(int32_t);
        if (comm->scratch_bytes < need) {
            if (comm->scratch) cudaFree(comm->scratch);
            comm->scratch = nullptr;
            comm->scratch_bytes = 0;
            if (cudaMalloc(&comm->scratch, need) != cudaSuccess) {
                cudaGetLastError();
                return set_status(ADOP_ERR_CUDA, "comm: scratch allocation failed");
            }
            comm->scratch_bytes = need;
        }
        int32_t *hi = static_cast<int32_t *>(comm->scratch);
        for (int v = 0; v < n_views; ++v) {  // one view at a time through the scratch buffer (same stream)
            const int64_t P = pixels[v];
            const unsigned g = (unsigned)((P + 255) / 256 < 1184 ? (P + 255) / 256 : 1184);
            k_hi_pack<<<g, 256, 0, s>>>(reinterpret_cast<const uint32_t *>(views[v].keys), hi, P);
            ncclResult_t r = n.allReduce(hi, hi, (size_t)P, ncclInt32, ncclMin, comm->nccl, s);
            if (r != ncclSuccess) return nccl_fail(r, "comm: MIN of the depth words");
            k_hi_unpack<<<g, 256, 0, s>>>(reinterpret_cast<uint32_t *>(views[v].keys), hi, P);
        }
        if (cudaGetLastError() != cudaSuccess) return set_status(ADOP_ERR_CUDA, "comm: depth-word pack launch");
        return ADOP_OK;
    }
    n.groupStart();
    for (int v = 0; v < n_views; ++v) {
        ncclResult_t r = n.allReduce(views[v].keys, views[v].keys, (size_t)pixels[v], ncclInt64, ncclMin, comm->nccl, s);
        if (r != ncclSuccess) {
            n.groupEnd();
            return nccl_fail(r, "comm: MIN of the keys");
        }
    }
    ncclResult_t r = n.groupEnd();
    return r == ncclSuccess ? ADOP_OK : nccl_fail(r, "comm: MIN of the keys");
}

// After the blend (point sharding): accum and count SUM over the shards.
adop_status comm_sums(adop_comm *comm, const adop_pyramid *views, const int64_t *pixels, int32_t n_views, int32_t C,
                      void *stream) {
    if (!comm || comm->mode != ADOP_SHARD_POINTS) return ADOP_OK;
    const NcclApi &n = nccl();
    cudaStream_t s = (cudaStream_t)stream;
    n.groupStart();
    for (int v = 0; v < n_views; ++v) {
        ncclResult_t r = n.allReduce(views[v].accum, views[v].accum, (size_t)pixels[v] * C, ncclFloat32, ncclSum,
                                     comm->nccl, s);
        if (r == ncclSuccess)
            r = n.allReduce(views[v].count, views[v].count, (size_t)pixels[v], ncclFloat32, ncclSum, comm->nccl, s);
        if (r != ncclSuccess) {
            n.groupEnd();
            return nccl_fail(r, "comm: SUM of accum / count");
        }
    }
    ncclResult_t r = n.groupEnd();
    return r == ncclSuccess ? ADOP_OK : nccl_fail(r, "comm: SUM of accum / count");
}

// After the backward: point sharding sums the per-view pose / intrinsics gradients, view sharding the point
// gradients (and the environment map's).
adop_status comm_grads(adop_comm *comm, int64_t n, int32_t C, int32_t n_views, float *d_feat, float *d_pos,
                       double *d_pose, double *d_intr, float *d_env, int64_t n_env, void *stream) {
    if (!comm) return ADOP_OK;
    const NcclApi &nc = nccl();
    cudaStream_t s = (cudaStream_t)stream;
    struct Item {
        void *p;
        size_t count;
        ncclDataType_t t;
    } items[4];
    int k = 0;
    if (comm->mode == ADOP_SHARD_POINTS) {
        if (d_pose) items[k++] = {d_pose, (size_t)n_views * 6, ncclFloat64};
        if (d_intr) items[k++] = {d_intr, (size_t)n_views * 12, ncclFloat64};
    } else {
        if (d_feat) items[k++] = {d_feat, (size_t)n * C, ncclFloat32};
        if (d_pos) items[k++] = {d_pos, (size_t)n * 3, ncclFloat32};
        if (d_env && n_env > 0) items[k++] = {d_env, (size_t)n_env, ncclFloat32};
    }
    if (k == 0) return ADOP_OK;
    nc.groupStart();
    for (int i = 0; i < k; ++i) {
        ncclResult_t r = nc.allReduce(items[i].p, items[i].p, items[i].count, items[i].t, ncclSum, comm->nccl, s);
        if (r != ncclSuccess) {
            nc.groupEnd();
            return nccl_fail(r, "comm: SUM of the gradients");
        }
    }
    ncclResult_t r = nc.groupEnd();
    return r == ncclSuccess ? ADOP_OK : nccl_fail(r, "comm: SUM of the gradients");
}

}  // namespace adop

using namespace adop;

extern "C" {

adop_status adop_comm_unique_id(uint8_t id[128]) {
    if (!id) return set_status(ADOP_ERR_INVALID_ARGUMENT, "id is NULL");
    const NcclApi &n = nccl();
    if (!n.ok) return set_status(ADOP_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    ncclResult_t r = n.getUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, &u, 128);
    return set_status(ADOP_OK, "");
}

adop_status adop_comm_init(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t mode, int32_t flags,
                           adop_comm **out) {
    if (!id || !out) return set_status(ADOP_ERR_INVALID_ARGUMENT, "NULL argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_status(ADOP_ERR_INVALID_ARGUMENT, "rank not in [0, nranks)");
    if (mode != ADOP_SHARD_POINTS && mode != ADOP_SHARD_VIEWS)
        return set_status(ADOP_ERR_INVALID_ARGUMENT, "mode must be ADOP_SHARD_POINTS or ADOP_SHARD_VIEWS");
    if (flags & ~ADOP_COMM_KEYS32) return set_status(ADOP_ERR_INVALID_ARGUMENT, "unknown comm flags");
    const NcclApi &n = nccl();
    if (!n.ok) return set_status(ADOP_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return set_status(ADOP_ERR_CUDA, "no current CUDA device");
    }
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclComm_t c = nullptr;
    ncclResult_t r = n.commInitRank(&c, nranks, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    adop_comm *m = new (std::nothrow) adop_comm{c, nranks, rank, mode, flags, dev, nullptr, 0};
    if (!m) {
        n.commDestroy(c);
        return set_status(ADOP_ERR_INVALID_ARGUMENT, "out of host memory");
    }
    *out = m;
    return set_status(ADOP_OK, "");
}

adop_status adop_comm_destroy(adop_comm *comm) {
    if (!comm) return set_status(ADOP_OK, "");
    if (comm->scratch) cudaFree(comm->scratch);
    ncclResult_t r = nccl().ok ? nccl().commDestroy(comm->nccl) : ncclSuccess;
    delete comm;
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return set_status(ADOP_OK, "");
}

}  // extern "C"
