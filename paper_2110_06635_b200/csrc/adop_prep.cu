// adop_prep.cu -- preprocessing before the hot path, sm_100a:
//
//   adop_blocked_morton_order  the blocked Morton shuffle of PAPER.md L360 (§4.5), reading R34:
//                              bounding box (block reduction), 63-bit Morton codes from 21-bit fp32
//                              quantization (pinned order, bit-identical to the oracle), stable radix sort
//                              of (code, index) (CUB), blocks of B points ordered by (h(seed, b), b)
//   adop_apply_order           gather of positions / radii / descriptors / normals into the new order
//   adop_knn_radius            r_world of §4.4 (L338) "inside its local neighborhood", reading R33: median
//                              distance to the k nearest neighbours, exact, by ring search over the cells of
//                              the Morton-sorted cloud (cells = Morton prefixes at a level chosen from n / k)
//
// The sort is a library primitive (cub::DeviceRadixSort, like a GEMM would be cuBLAS); everything else is
// written here.  Scratch comes from the caller's workspace (adop_prep_workspace_size).
#include <cstdint>
#include <cstdio>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "adop_internal.h"

namespace adop {
namespace {

constexpr int kT = 256;
constexpr uint32_t kQMax = 2097151u;  // 2^21 - 1

// order-preserving float <-> uint (for atomic min / max of floats)
__device__ __forceinline__ uint32_t f2o(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t u) { return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u); }

struct PrepHdr {
    uint32_t lo[3], hi[3];  // ordered-uint bounding box
    int32_t short_slot;     // position of the (short) last Morton block in the block order
};

__global__ void k_bbox_init(PrepHdr *h) {
    if (threadIdx.x < 3) {
        h->lo[threadIdx.x] = 0xFFFFFFFFu;
        h->hi[threadIdx.x] = 0u;
    }
}

__global__ void __launch_bounds__(kT) k_bbox(const float *pos, int64_t stride, int64_t n, PrepHdr *h) {
    uint32_t lo[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, hi[3] = {0u, 0u, 0u};
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
        for (int a = 0; a < 3; ++a) {
            const uint32_t o = f2o(pos[a * stride + i]);
            lo[a] = min(lo[a], o);
            hi[a] = max(hi[a], o);
        }
    for (int a = 0; a < 3; ++a) {
        const uint32_t l = __reduce_min_sync(0xffffffffu, lo[a]), u = __reduce_max_sync(0xffffffffu, hi[a]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&h->lo[a], l);
            atomicMax(&h->hi[a], u);
        }
    }
}

__device__ __forceinline__ uint64_t split3(uint32_t v) {
    uint64_t x = v & 0x1FFFFF;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

// R34 quantization: q = trunc(fl(fl(fl(x - lo) / fl(hi - lo)) * (2^21 - 1))), 0 on a degenerate axis.
__device__ __forceinline__ uint32_t quant(float x, float lo, float hi) {
    const float ext = __fsub_rn(hi, lo);
    if (!(ext > 0.0f)) return 0u;
    const float t = __fdiv_rn(__fsub_rn(x, lo), ext);
    const float q = __fmul_rn(t, 2097151.0f);
    const uint32_t u = (uint32_t)q;
    return u > kQMax ? kQMax : u;
}

__global__ void __launch_bounds__(kT) k_codes(const float *pos, int64_t stride, int64_t n, const PrepHdr *h,
                                              uint64_t *codes, uint32_t *idx) {
    const float lo[3] = {o2f(h->lo[0]), o2f(h->lo[1]), o2f(h->lo[2])};
    const float hi[3] = {o2f(h->hi[0]), o2f(h->hi[1]), o2f(h->hi[2])};
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
        uint64_t c = 0;
        for (int a = 0; a < 3; ++a) c |= split3(quant(pos[a * stride + i], lo[a], hi[a])) << a;
        codes[i] = c;
        idx[i] = (uint32_t)i;
    }
}

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// block keys (h(seed, b) << 32 | b), h = mix32(b ^ mix32(lo32(seed) + 0x9E3779B9 * 4)) (R34)
__global__ void k_block_keys(int64_t nb, uint64_t seed, uint64_t *keys) {
    const uint32_t salt = mix32((uint32_t)seed + 0x9E3779B9u * 4u);
    for (int64_t b = (int64_t)blockIdx.x * kT + threadIdx.x; b < nb; b += (int64_t)gridDim.x * kT)
        keys[b] = ((uint64_t)mix32((uint32_t)b ^ salt) << 32) | (uint64_t)(uint32_t)b;
}

__global__ void k_find_short(const uint64_t *bkeys, int64_t nb, PrepHdr *h) {
    for (int64_t j = (int64_t)blockIdx.x * kT + threadIdx.x; j < nb; j += (int64_t)gridDim.x * kT)
        if ((int64_t)(uint32_t)bkeys[j] == nb - 1) h->short_slot = (int32_t)j;
}

// perm[out] = order[b_j * B + t] for the j-th block in block order, t < len(b_j)
__global__ void __launch_bounds__(kT) k_assemble(const uint32_t *order, const uint64_t *bkeys, int64_t n, int64_t nb,
                                                 int32_t B, const PrepHdr *h, int64_t *perm) {
    const int64_t last_len = n - (nb - 1) * (int64_t)B;
    const int64_t s = h->short_slot;
    for (int64_t g = (int64_t)blockIdx.x * kT + threadIdx.x; g < nb * (int64_t)B; g += (int64_t)gridDim.x * kT) {
        const int64_t j = g / B, t = g % B;
        const int64_t b = (int64_t)(uint32_t)bkeys[j];
        const int64_t len = b == nb - 1 ? last_len : B;
        if (t >= len) continue;
        const int64_t out = j * (int64_t)B - (j > s ? (int64_t)B - last_len : 0) + t;
        perm[out] = (int64_t)order[b * (int64_t)B + t];
    }
}

__global__ void __launch_bounds__(kT) k_gather(adop_points src, adop_points dst, const int64_t *perm) {
    const int C = src.channels;
    for (int64_t j = (int64_t)blockIdx.x * kT + threadIdx.x; j < src.n; j += (int64_t)gridDim.x * kT) {
        const int64_t i = perm[j];
        for (int a = 0; a < 3; ++a) const_cast<float *>(dst.pos)[a * dst.pos_stride + j] = src.pos[a * src.pos_stride + i];
        if (src.radius && dst.radius) const_cast<float *>(dst.radius)[j] = src.radius[i];
        if (src.normal && dst.normal)
            for (int a = 0; a < 3; ++a)
                const_cast<float *>(dst.normal)[a * dst.pos_stride + j] = src.normal[a * src.pos_stride + i];
        if (src.feat && dst.feat)
            for (int c = 0; c < C; ++c) const_cast<float *>(dst.feat)[j * C + c] = src.feat[i * C + c];
    }
}

// ---- kNN radius (R33) ----
constexpr int kKMax = 32;

__device__ __forceinline__ uint32_t part1by2_inv(uint64_t x) {  // compact every third bit
    x &= 0x1249249249249249ull;
    x = (x ^ (x >> 2)) & 0x10C30C30C30C30C3ull;
    x = (x ^ (x >> 4)) & 0x100F00F00F00F00Full;
    x = (x ^ (x >> 8)) & 0x1F0000FF0000FFull;
    x = (x ^ (x >> 16)) & 0x1F00000000FFFFull;
    x = (x ^ (x >> 32)) & 0x1FFFFFull;
    return (uint32_t)x;
}

// first index in sorted[0, n) with (sorted >> sh) >= key
__device__ __forceinline__ int64_t lower(const uint64_t *sorted, int64_t n, int sh, uint64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((sorted[mid] >> sh) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One thread per point (in Morton order): top-k smallest squared distances over rings of level-c cells.
__global__ void __launch_bounds__(kT) k_knn(const float *pos, int64_t stride, int64_t n, int k, const uint64_t *codes,
                                            const uint32_t *order, const PrepHdr *h, int c, float *radius) {
    const int sh = 3 * (21 - c);
    const int64_t cells = (int64_t)1 << c;
    float lo[3], side[3], diag2 = 0.f;
    for (int a = 0; a < 3; ++a) {
        lo[a] = o2f(h->lo[a]);
        const float ext = o2f(h->hi[a]) - lo[a];
        side[a] = ext > 0.f ? ext / (float)cells : INFINITY;  // degenerate axis: one slab
        diag2 += ext * ext;
    }
    const float smin = fminf(side[0], fminf(side[1], side[2]));
    for (int64_t s = (int64_t)blockIdx.x * kT + threadIdx.x; s < n; s += (int64_t)gridDim.x * kT) {
        const int64_t i = order[s];
        const float p[3] = {pos[i], pos[stride + i], pos[2 * stride + i]};
        const uint64_t me = codes[s] >> sh;
        const int cx = (int)part1by2_inv(me), cy = (int)part1by2_inv(me >> 1), cz = (int)part1by2_inv(me >> 2);
        float best[kKMax];
        int cnt = 0;
        for (int r = 0;; ++r) {
            for (int dz = -r; dz <= r; ++dz)
                for (int dy = -r; dy <= r; ++dy)
                    for (int dx = -r; dx <= r; ++dx) {
                        if (max(abs(dx), max(abs(dy), abs(dz))) != r) continue;  // the shell only
                        const int x = cx + dx, y = cy + dy, z = cz + dz;
                        if (x < 0 || y < 0 || z < 0 || x >= cells || y >= cells || z >= cells) continue;
                        const uint64_t key = split3(x) | (split3(y) << 1) | (split3(z) << 2);
                        for (int64_t t = lower(codes, n, sh, key); t < n && (codes[t] >> sh) == key; ++t) {
                            const int64_t jj = order[t];
                            if (jj == i) continue;
                            const float ddx = pos[jj] - p[0], ddy = pos[stride + jj] - p[1], ddz = pos[2 * stride + jj] - p[2];
                            const float d2 = ddx * ddx + ddy * ddy + ddz * ddz;
                            if (cnt == k && !(d2 < best[k - 1])) continue;
                            int m = cnt < k ? cnt++ : k - 1;  // insertion into the sorted top-k
                            while (m > 0 && best[m - 1] > d2) {
                                best[m] = best[m - 1];
                                --m;
                            }
                            best[m] = d2;
                        }
                    }
            // every point of ring r + 1 or beyond is at least r * side_min away
            const float reach = (float)r * smin;
            if (cnt == k && best[k - 1] <= reach * reach) break;
            if (r >= cells) break;  // the whole grid has been searched
        }
        float med;
        if (cnt == 0) med = 0.f;
        else if (cnt & 1) med = sqrtf(best[cnt / 2]);
        else med = 0.5f * (sqrtf(best[cnt / 2 - 1]) + sqrtf(best[cnt / 2]));
        radius[i] = fmaxf(med, 1e-9f * sqrtf(diag2));
    }
}

struct PrepWs {
    PrepHdr *hdr;
    uint64_t *codes_in, *codes_out, *bkeys_in, *bkeys_out;
    uint32_t *idx_in, *idx_out;
    void *temp;
    size_t temp_bytes;
};

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

size_t cub_temp(int64_t n, int64_t nb) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)n, 0, 63);
    cub::DeviceRadixSort::SortKeys(nullptr, b, (const uint64_t *)nullptr, (uint64_t *)nullptr, (int)nb, 0, 64);
    return a > b ? a : b;
}

size_t prep_bytes(int64_t n, int64_t nb, size_t *temp) {
    *temp = cub_temp(n, nb);
    return align256(sizeof(PrepHdr)) + 2 * align256(8 * n) + 2 * align256(8 * nb) + 2 * align256(4 * n) +
           align256(*temp);
}

adop_status carve(void *ws, size_t bytes, int64_t n, int64_t nb, PrepWs &w) {
    size_t temp = 0;
    const size_t need = prep_bytes(n, nb, &temp);
    if (!ws) return set_status(ADOP_ERR_INVALID_ARGUMENT, "prep workspace is NULL");
    if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0)
        return set_status(ADOP_ERR_INVALID_ARGUMENT, "prep workspace must be 256-byte aligned");
    if (bytes < need) return set_status(ADOP_ERR_WORKSPACE_TOO_SMALL, "prep workspace too small");
    char *b = static_cast<char *>(ws);
    auto take = [&](size_t s) { char *r = b; b += align256(s); return r; };
    w.hdr = reinterpret_cast<PrepHdr *>(take(sizeof(PrepHdr)));
    w.codes_in = reinterpret_cast<uint64_t *>(take(8 * n));
    w.codes_out = reinterpret_cast<uint64_t *>(take(8 * n));
    w.bkeys_in = reinterpret_cast<uint64_t *>(take(8 * nb));
    w.bkeys_out = reinterpret_cast<uint64_t *>(take(8 * nb));
    w.idx_in = reinterpret_cast<uint32_t *>(take(4 * n));
    w.idx_out = reinterpret_cast<uint32_t *>(take(4 * n));
    w.temp = take(temp);
    w.temp_bytes = temp;
    return ADOP_OK;
}

int grid_for(int64_t n) {
    int64_t g = (n + kT - 1) / kT;
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

adop_status check_pts(const adop_points *p) {
    if (!p) return set_status(ADOP_ERR_INVALID_ARGUMENT, "points is NULL");
    if (p->n < 1 || p->n >= ((int64_t)1 << 31)) return set_status(ADOP_ERR_INVALID_ARGUMENT, "n not in [1, 2^31)");
    if (!p->pos || p->pos_stride < p->n) return set_status(ADOP_ERR_INVALID_ARGUMENT, "bad positions");
    return ADOP_OK;
}

// bbox + codes + (code, index) radix sort -> w.codes_out / w.idx_out sorted
adop_status sort_codes(const adop_points *p, PrepWs &w, cudaStream_t s) {
    k_bbox_init<<<1, 32, 0, s>>>(w.hdr);
    k_bbox<<<grid_for(p->n), kT, 0, s>>>(p->pos, p->pos_stride, p->n, w.hdr);
    k_codes<<<grid_for(p->n), kT, 0, s>>>(p->pos, p->pos_stride, p->n, w.hdr, w.codes_in, w.idx_in);
    size_t tb = w.temp_bytes;
    if (cub::DeviceRadixSort::SortPairs(w.temp, tb, w.codes_in, w.codes_out, w.idx_in, w.idx_out, (int)p->n, 0, 63, s) !=
        cudaSuccess)
        return set_status(ADOP_ERR_CUDA, "radix sort failed");
    return ADOP_OK;
}

}  // namespace
}  // namespace adop

using namespace adop;

extern "C" {

adop_status adop_prep_workspace_size(int64_t n, int32_t block, size_t *bytes) {
    if (!bytes || n < 1 || block < 1) return set_status(ADOP_ERR_INVALID_ARGUMENT, "bad arguments");
    size_t temp = 0;
    *bytes = prep_bytes(n, (n + block - 1) / block, &temp);
    return ADOP_OK;
}

adop_status adop_blocked_morton_order(const adop_points *points, int32_t block, uint64_t seed, int64_t *perm,
                                      void *workspace, size_t workspace_bytes, void *stream) {
    adop_status st = check_pts(points);
    if (st) return st;
    if (block < 1 || !perm) return set_status(ADOP_ERR_INVALID_ARGUMENT, "block < 1 or perm is NULL");
    const int64_t n = points->n, nb = (n + block - 1) / block;
    PrepWs w;
    if ((st = carve(workspace, workspace_bytes, n, nb, w))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = sort_codes(points, w, s))) return st;
    k_block_keys<<<grid_for(nb), kT, 0, s>>>(nb, seed, w.bkeys_in);
    size_t tb = w.temp_bytes;
    if (cub::DeviceRadixSort::SortKeys(w.temp, tb, w.bkeys_in, w.bkeys_out, (int)nb, 0, 64, s) != cudaSuccess)
        return set_status(ADOP_ERR_CUDA, "block sort failed");
    k_find_short<<<grid_for(nb), kT, 0, s>>>(w.bkeys_out, nb, w.hdr);
    k_assemble<<<grid_for(nb * block), kT, 0, s>>>(w.idx_out, w.bkeys_out, n, nb, block, w.hdr, perm);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_status(ADOP_ERR_CUDA, cudaGetErrorString(e));
    return set_status(ADOP_OK, "");
}

adop_status adop_apply_order(const adop_points *src, const int64_t *perm, const adop_points *dst, void *stream) {
    adop_status st = check_pts(src);
    if (st) return st;
    if (!dst || !perm || dst->n != src->n || dst->channels != src->channels || !dst->pos || dst->pos_stride < dst->n ||
        dst->pos_stride != src->pos_stride)
        return set_status(ADOP_ERR_INVALID_ARGUMENT, "dst must match src (n, channels, pos_stride)");
    k_gather<<<grid_for(src->n), kT, 0, (cudaStream_t)stream>>>(*src, *dst, perm);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_status(ADOP_ERR_CUDA, cudaGetErrorString(e));
    return set_status(ADOP_OK, "");
}

adop_status adop_knn_radius(const adop_points *points, int32_t k, float *radius, void *workspace,
                            size_t workspace_bytes, void *stream) {
    adop_status st = check_pts(points);
    if (st) return st;
    if (k < 1 || k > kKMax || points->n < k + 1 || !radius)
        return set_status(ADOP_ERR_INVALID_ARGUMENT, "need 1 <= k <= 32, n >= k + 1 and radius");
    const int64_t n = points->n;
    PrepWs w;
    if ((st = carve(workspace, workspace_bytes, n, 1, w))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = sort_codes(points, w, s))) return st;
    // grid level: ~k..2k points per occupied cell for surface-like clouds (n / 4^c ~ k), 1..12
    int level = 1;
    while (level < 12 && ((int64_t)1 << (2 * (level + 1))) * k <= n) ++level;
    k_knn<<<grid_for(n), kT, 0, s>>>(points->pos, points->pos_stride, n, k, w.codes_out, w.idx_out, w.hdr, level,
                                     radius);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_status(ADOP_ERR_CUDA, cudaGetErrorString(e));
    return set_status(ADOP_OK, "");
}

}  // extern "C"
