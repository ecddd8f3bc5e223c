// adop_kernels.cu -- sm_100a kernels of the ADOP one-pixel point rasterizer.
//
//   k_clear          keys <- sentinel + header / plane / layer tables (phase 1); accum, count <- 0 (phase 2)
//   k_depth_pool     the depth-only pass (§4.5, min_z of Eq. 6) -- the hot kernel: TMA-streamed warp tiles from
//                    a CTA-wide pool of stages; lane-box cull, hash-first discard prefilter (Eq. 12), exact
//                    projection (Eqs. 2-4), 64-bit red.min of the packed keys (R8), survivor records
//   k_depth_async    the same pass with per-warp 2-stage rings (tile culling / dynamic claiming; A/B reference)
//   k_stream         fallback sweep for unaligned inputs <DEPTH>, the blend's overflow re-stream <BLEND>,
//                    the per-point masks <MASKS>
//   k_chunk_hist / k_chunk_scatter   view-major order of the multi-view lists' 64-slot chunks
//   k_blend          survivor records: fuzzy test (Eq. 6) + vector red.add of tau and the count (§4.5)
//   k_resolve        per pixel: Eq. 7 mean or background (constant or environment map), planar NCHW output
//   k_fill / k_bwd_prep / k_bwd_sweep / k_bwd_tex / k_bwd_ghost / k_pose_reduce   the backward: zero fill and
//                    mode choice, per-pixel tables, the re-render sweep (ghost list; texture list only when the
//                    forward's records cannot be reused), texture gradient (R24), ghost gradient (Eqs. 9-11 +
//                    chain rule, Eq. 8, Eq. 17), fixed-order fp64 pose reduction
//   k_backward       fused planar backward for unaligned inputs
//
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdlib>

#include "adop_device.cuh"

namespace adop {

// Bounds-checked build (ADOP_CHECKS=1, scripts/build_variants.py chk=ADOP_CHECKS=1): every index into a pyramid,
// a point array, the record region, the chunk tables or a shared-memory list is checked on the device; a
// violation prints the check and traps (the run fails).  compute-sanitizer is closed on this GPU pool; the GPU
// test suite runs against this build instead.
#ifndef ADOP_CHECKS
#define ADOP_CHECKS 0
#endif
#if ADOP_CHECKS
#define ADOP_CHECK(cond)                                                                                         \
    do {                                                                                                         \
        if (!(cond)) {                                                                                           \
            printf("ADOP_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x);                                                                                 \
            __trap();                                                                                            \
        }                                                                                                        \
    } while (0)
#else
#define ADOP_CHECK(cond) \
    do {                 \
    } while (0)
#endif

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kCap = 256;  // records buffered per warp in shared memory before a flush
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxBwdBlocks = 2048;

enum { MODE_DEPTH = 0, MODE_BLEND = 1, MODE_MASKS = 2 };

// --------------------------------------------------------------------------- //
// clear
// --------------------------------------------------------------------------- //
// CLEAR_KEYS (phase 1): keys <- sentinel, workspace header reset.
// CLEAR_ACC  (phase 2): accum, count <- 0 right before the blend, so the blend's reductions and the
//                        resolve find these 55 MB (configs[3]) still in L2.
enum { CLEAR_KEYS = 0, CLEAR_ACC = 1 };
#ifndef ADOP_CLEAR_REVERSE
#define ADOP_CLEAR_REVERSE 1
#endif
template <int WHAT>
__global__ void __launch_bounds__(kThreads) k_clear(const __grid_constant__ RasterArgs a) {
    // CLEAR_ACC clears the views last-to-first (blocks are scheduled in blockIdx.y order): the view-major blend
    // starts on view 0, whose freshly zeroed lines are then the ones still in L2
    const ViewDesc &v = a.v[WHAT == CLEAR_ACC && ADOP_CLEAR_REVERSE ? gridDim.y - 1 - blockIdx.y : blockIdx.y];
    const int64_t P = v.pixels;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (WHAT == CLEAR_KEYS) {
        const unsigned long long sentinel = 0x7FFFFFFFFFFFFFFFull;
        unsigned long long *k = reinterpret_cast<unsigned long long *>(v.keys);
        if (!a.clear_pyr) {  // shared pyramid: the owner's adop_clear_pyramid reset it
        } else if ((reinterpret_cast<uintptr_t>(k) & 15) == 0) {
            for (int64_t q = tid; q < P / 2; q += stride)
                reinterpret_cast<ulonglong2 *>(k)[q] = make_ulonglong2(sentinel, sentinel);
            for (int64_t q = (P / 2) * 2 + tid; q < P; q += stride) k[q] = sentinel;
        } else {
            for (int64_t q = tid; q < P; q += stride) k[q] = sentinel;
        }
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
            a.hdr->resv = 0ull;
            a.hdr->front_ok = 0ull;
            a.hdr->back_ok = 0ull;
            a.hdr->overflow = 0;
            a.hdr->tag = a.tag;
            a.hdr->tiles_fwd = 0ull;
            a.hdr->tiles_read = 0ull;
            a.hdr->ghosts_fwd = a.ghost_fwd;  // cleared by the depth pass if a ghost did not fit the list
        }
        if (blockIdx.x == 0 && threadIdx.x < 5) {  // this view's frustum planes for tile_views
            const int k = threadIdx.x;
            a.planes[blockIdx.y].pl[k] = make_float4(v.pl[k][0], v.pl[k][1], v.pl[k][2], v.pl[k][3]);
            a.planes[blockIdx.y].pm[k] = make_float2(v.pm[k][0], v.pm[k][1]);
        }
        if (blockIdx.x == 0 && threadIdx.x < ADOP_MAX_LAYERS) {  // this view's layer table for the drain
            LayerDesc &d = a.ldesc[blockIdx.y];
            const int l = threadIdx.x;
            d.off[l] = v.off[l];
            d.wl[l] = v.wl[l];
            d.hl[l] = v.hl[l];
            if (l == 0) d.keys = v.keys;
        }
        return;
    }
    float *bufs[2] = {v.accum, v.count};
    const int64_t lens[2] = {P * a.channels, P};
    for (int b = 0; b < 2; ++b) {
        float *acc = bufs[b];
        const int64_t n = lens[b];
        if ((reinterpret_cast<uintptr_t>(acc) & 15) == 0) {
            for (int64_t q = tid; q < n / 4; q += stride) reinterpret_cast<float4 *>(acc)[q] = make_float4(0, 0, 0, 0);
            for (int64_t q = (n / 4) * 4 + tid; q < n; q += stride) acc[q] = 0.0f;
        } else {
            for (int64_t q = tid; q < n; q += stride) acc[q] = 0.0f;
        }
    }
}

// --------------------------------------------------------------------------- //
// point loads for one warp chunk: lane owns points i0..i0+3
// --------------------------------------------------------------------------- //
template <bool VEC>
__device__ __forceinline__ void load_points(const RasterArgs &a, int64_t i0, float (&px)[4], float (&py)[4],
                                            float (&pz)[4], float (&pr)[4]) {
    if (VEC && i0 + 3 < a.n) {
        float4 X = ld_stream4(a.x + i0), Y = ld_stream4(a.y + i0), Z = ld_stream4(a.z + i0);
        px[0] = X.x; px[1] = X.y; px[2] = X.z; px[3] = X.w;
        py[0] = Y.x; py[1] = Y.y; py[2] = Y.z; py[3] = Y.w;
        pz[0] = Z.x; pz[1] = Z.y; pz[2] = Z.z; pz[3] = Z.w;
        if (a.radius) {
            float4 Rw = ld_stream4(a.radius + i0);
            pr[0] = Rw.x; pr[1] = Rw.y; pr[2] = Rw.z; pr[3] = Rw.w;
        } else {
            pr[0] = pr[1] = pr[2] = pr[3] = a.radius_uniform;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = i0 + j;
            if (i < a.n) {
                px[j] = ld_stream(a.x + i);
                py[j] = ld_stream(a.y + i);
                pz[j] = ld_stream(a.z + i);
                pr[j] = a.radius ? ld_stream(a.radius + i) : a.radius_uniform;
            } else {
                px[j] = py[j] = pz[j] = __int_as_float(0x7fc00000);  // NaN: culled by the validity test
                pr[j] = 0.0f;
            }
        }
    }
}

// ---- record-region reservations (WsHeader::resv: front slots | back chunks << 40) ----
#ifndef ADOP_CHUNK
#define ADOP_CHUNK 256
#endif
constexpr int kChunk = ADOP_CHUNK;  // record slots reserved per warp at a time (back list: kChunk / 2 ghost entries)
static_assert(kChunk % kListChunk == 0, "list chunks are reserved in units of the chunk table's kListChunk slots");
constexpr int kPoolLane = 31;  // multi-view lists: the lane holding the warp's pool of reserved list chunks (views <= 16)
constexpr unsigned long long kFrontMask = (1ull << kResvBackShift) - 1ull;
constexpr unsigned long long kNoSlot = ~0ull;

__device__ __forceinline__ unsigned long long resv_front_used(unsigned long long r) { return r & kFrontMask; }
__device__ __forceinline__ unsigned long long resv_back_slots(unsigned long long r) {
    return (r >> kResvBackShift) * (unsigned long long)kChunk;
}
// Reserve k front slots (BACK = false) or one back chunk of kChunk slots (BACK = true).  One atomicAdd on
// `resv` orders every reservation of both lists; a reservation succeeds if, counting everything reserved
// before it on either side, the two lists do not collide.  Failures are monotone (both counts only grow),
// so the successful ones form a prefix of each list: [0, front_ok) and [capacity - back_ok, capacity).
// Returns the first slot, or kNoSlot (then `overflow` is set when `flag`: the depth pass's list is
// incomplete).
template <bool BACK>
__device__ __forceinline__ unsigned long long resv_take(const RasterArgs &a, unsigned long long k, bool flag) {
    const unsigned long long cap = (unsigned long long)a.rec_capacity;
    const unsigned long long o = atomicAdd(&a.hdr->resv, BACK ? (1ull << kResvBackShift) : k);
    const unsigned long long f = resv_front_used(o), b = resv_back_slots(o);
    if ((BACK ? f + b + kChunk : f + k + b) > cap) {
        if (flag) atomicExch(&a.hdr->overflow, 1);
        return kNoSlot;
    }
    if (BACK) {
        atomicMax(&a.hdr->back_ok, b + kChunk);
        return cap - b - kChunk;
    }
    atomicMax(&a.hdr->front_ok, f + k);
    return f;
}

// Warp-level flush of the shared-memory record buffer into the global survivor list.
__device__ __forceinline__ void flush_records(const RasterArgs &a, Record *buf, int &wcount, int lane) {
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) base = resv_take<false>(a, (unsigned long long)wcount, true);
    base = __shfl_sync(kFull, base, 0);
    if (base != kNoSlot)
        for (int k = lane; k < wcount; k += 32)
            reinterpret_cast<uint4 *>(a.records)[base + k] = reinterpret_cast<const uint4 *>(buf)[k];
    __syncwarp();
    wcount = 0;
}

template <bool VEC4>
__device__ __forceinline__ void accumulate_feature(const RasterArgs &a, const ViewDesc &v, int64_t idx,
                                                   uint32_t pix) {
    ADOP_CHECK(idx >= 0 && idx < a.n && pix < (uint32_t)v.pixels);
    const int C = a.channels;
    const float *f = a.feat + idx * C;
    float *acc = v.accum + (int64_t)pix * C;
    if (VEC4) {
        const uint64_t pol = policy_evict_first();
        for (int c = 0; c < C; c += 4) {
            float4 t = ld_once4(f + c, pol);
            if (a.log_desc) t = make_float4(expf(t.x), expf(t.y), expf(t.z), expf(t.w));
            red_add_v4(acc + c, t);
        }
    } else {
        for (int c = 0; c < C; ++c) red_add(acc + c, desc_lin(a, __ldg(f + c)));
    }
    red_add(v.count + pix, 1.0f);
}

// --------------------------------------------------------------------------- //
// streaming sweep over all points (depth pass / blend fallback / masks)
// --------------------------------------------------------------------------- //
template <int MODEL, bool VEC, int MODE, bool VEC4>
__device__ __forceinline__ void stream_sweep(const RasterArgs &a) {
    __shared__ __align__(16) Record sbuf[MODE == MODE_DEPTH ? kWarps : 1][MODE == MODE_DEPTH ? kCap : 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    int wcount = 0;
    const int64_t nchunks = (a.n + 127) / 128;
    for (int64_t ch = (int64_t)blockIdx.x * kWarps + wid; ch < nchunks; ch += (int64_t)gridDim.x * kWarps) {
        const int64_t i0 = ch * 128 + lane * 4;
        float px[4], py[4], pz[4], pr[4];
        load_points<VEC>(a, i0, px, py, pz, pr);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = i0 + j;
            const bool in = i < a.n;
            const uint32_t gi = a.goff + (uint32_t)i;
            const bool ghost = in && a.ghost_thr != 0u && h24(a.ghost_salt, gi) < a.ghost_thr;
            const bool live = MODE == MODE_MASKS ? in : (in && !ghost);
            if (!__any_sync(kFull, live)) continue;
            for (int vs = 0; vs < a.nviews; ++vs) {
                const ViewDesc &v = a.v[vs];
                Proj p;
                const bool ok = live && project_point<MODEL>(v, a.z_near, px[j], py[j], pz[j], p) &&
                                normal_keep(a, v, i, p.X, p.Y, p.Z);
                if (MODE == MODE_MASKS) {
                    unsigned m = ghost ? 0x80u : 0u;
                    if (ok) {
                        const int nk = keep_layers(a, v, pr[j], p.iz, gi);
                        for (int l = 0; l < a.layers; ++l) {
                            int pu, pv;
                            if (l < nk && layer_pixel(v, p, l, pu, pv) >= 0) m |= 1u << l;
                        }
                    }
                    if (in) a.mask[(int64_t)vs * a.n + i] = (uint8_t)m;
                    continue;
                }
                if (!__any_sync(kFull, ok)) continue;
                const int nk = ok ? keep_layers(a, v, pr[j], p.iz, gi) : 0;
                const uint64_t key = depth_key(p.D, gi);
#pragma unroll
                for (int l = 0; l < ADOP_MAX_LAYERS; ++l) {
                    if (l >= a.layers) break;
                    int pu, pv;
                    const int loc = l < nk ? layer_pixel(v, p, l, pu, pv) : -1;
                    const bool hit = loc >= 0;
                    const uint32_t pix = (uint32_t)(v.off[l] + loc);
                    if (MODE == MODE_DEPTH) {
                        if (hit) red_min_u64(v.keys + pix, key);
                        const unsigned b = __ballot_sync(kFull, hit);
                        if (b) {
                            if (wcount + 32 > kCap) flush_records(a, sbuf[wid], wcount, lane);
                            if (hit) {
                                Record r;
                                r.pix = pix;
                                r.zbits = __float_as_uint(p.D);
                                r.idx = (uint32_t)i;
                                r.view = (uint32_t)vs;
                                sbuf[wid][wcount + __popc(b & lt)] = r;
                            }
                            wcount += __popc(b);
                        }
                    } else {  // MODE_BLEND: re-streamed accumulate (only after a record overflow)
                        if (hit && fuzzy_pass(p.D, v.keys[pix], a.onepa)) accumulate_feature<VEC4>(a, v, i, pix);
                    }
                }
            }
        }
    }
    if (MODE == MODE_DEPTH && wcount > 0) flush_records(a, sbuf[wid], wcount, lane);
}

template <int MODEL, bool VEC, int MODE, bool VEC4>
__global__ void __launch_bounds__(kThreads) k_stream(const __grid_constant__ RasterArgs a) {
    stream_sweep<MODEL, VEC, MODE, VEC4>(a);
}

// --------------------------------------------------------------------------- //
// depth pass, TMA pipelined (k_depth_pool; k_depth_async with per-warp rings)
//
// Work unit = a warp tile of 256 consecutive (blocked-Morton ordered) points.  Lane 0 of a warp streams a
// tile's x, y, z rows with one 2-D TMA tensor copy (cp.async.bulk.tensor; 1-D bulk copies without a tensor
// map) and the r_world row with a 1-D bulk copy (L2 evict-first) into a shared-memory stage guarded by an
// mbarrier; the lane owns points h*128 + 4*lane + j so every LDS.128 of a row is one contiguous 512-B access.
// k_depth_pool: the CTA's tiles k G + b cycle through a pool of kPool stages (see there); k_depth_async:
// warp w of the grid takes tiles w, w + W, ... through a private 2-stage ring.  Per tile and view:
//   1. lane-box cull: a lane whose 8-point bounding box lies outside one of 5 conservative world-space
//      half-spaces (pinhole frustum, or the OpenCV8 image window in normalized coordinates) skips its points;
//      a warp whose lanes all agree skips the tile;
//   2. discard on: the hash-first prefilter (Eq. 12 on the lane box's depth bound: one hash compare per
//      point); discard off: a branch-free FMA pre-cull per point -> candidate bit mask, compacted per warp;
//   3. candidates, 32 per iteration: pinned transform (R1), validity (R7), OpenCV8 window test, exact discard
//      (R10), exact projection (R2/R6); kept points go to a warp queue;
//   4. the queue is drained 32 at a time: per layer round + bounds (Eqs. 3-4), 64-bit red.min of the
//      packed key (§4.5, R8) and survivor records written straight to global memory into per-warp chunks
//      (multi-view launches: per-view 64-slot chunks from a warp pool; unused slots are marked dead).
// --------------------------------------------------------------------------- //
constexpr int kStages = 2;   // backward sweep ring depth
#ifndef ADOP_DSTAGES
#define ADOP_DSTAGES 2
#endif
#ifndef ADOP_DCTAS
#define ADOP_DCTAS 3
#endif
constexpr int kDStages = ADOP_DSTAGES;  // depth sweep ring depth (tiles in flight per warp)
#ifndef ADOP_PREFILTER
#define ADOP_PREFILTER 1
#endif
#ifndef ADOP_LAYER_UNROLL
#define ADOP_LAYER_UNROLL 0  // measured: the rolled layer loop halves the kernel (icache) and is faster
#endif
#ifndef ADOP_DRAIN_NOINLINE
#define ADOP_DRAIN_NOINLINE 0
#endif
#ifndef ADOP_PREREDUCE
#define ADOP_PREREDUCE 0
#endif
#ifndef ADOP_COUNTERS  // profiling build only: per-stage work counts of the depth sweep (scripts/depth_counters.py)
#define ADOP_COUNTERS 0
#endif
#if ADOP_COUNTERS
__device__ unsigned long long g_depth_counts[8];  // tiles, view-tiles kept by the box test, candidates, kept, hits
extern "C" __attribute__((visibility("default"))) int adop_debug_depth_counts(unsigned long long *out, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out, g_depth_counts, sizeof(g_depth_counts));
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_depth_counts, z, sizeof(z));
    }
    return (int)e;
}
#define CNT(k, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_depth_counts[k], (unsigned long long)(v)); } while (0)
#else
#define CNT(k, v) do { } while (0)
#endif
#ifndef ADOP_CHUNK_PREFETCH
#define ADOP_CHUNK_PREFETCH 0
#endif
constexpr bool kPrefilter = ADOP_PREFILTER;  // depth sweep: hash-first discard prefilter (see depth_lane8)
constexpr int kDCTAs = ADOP_DCTAS;      // depth sweep CTAs per SM
constexpr int kSW = 8;               // warps per CTA of the TMA sweeps (3 CTAs x 8 warps per SM)
constexpr int kST = kSW * 32;
constexpr int kWTile = 256;  // points per warp tile (8 per lane)
constexpr int kQCap = 64;
constexpr uint32_t kDeadView = 0xFFFFFFFFu;

__device__ __forceinline__ void cp_async16(void *dst, const void *src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct WarpQueue {
    float4 e[kQCap];      // u0, v0, bits(z), shard-local index
    uint8_t meta[kQCap];  // kept layers (low 4 bits) | view slot << 4
};

// Dynamic tile scheduling: lane 0 of a warp claims batches of `kc` consecutive tiles from a global
// counter, one batch ahead (the atomic's latency overlaps the current batch); kc is sized so every warp
// gets several batches (load balance) while keeping the single-address atomics few.
struct TileClaim {
    long long cur, end, next, stride;
    int kc;
    bool dyn;
    __device__ __forceinline__ void init(unsigned long long *ctr, long long ntiles, long long warps, long long wglobal,
                                         bool dynamic) {
        dyn = dynamic;
        if (!dyn) {  // static round-robin: warp w takes tiles w, w + W, ... (contiguous front through memory)
            cur = wglobal;
            stride = warps;
            return;
        }
        long long k = ntiles / (warps * 4);
        kc = (int)(k < 1 ? 1 : (k > 16 ? 16 : k));
        cur = (long long)atomicAdd(ctr, (unsigned long long)kc);
        end = cur + kc;
        next = (long long)atomicAdd(ctr, (unsigned long long)kc);
    }
    __device__ __forceinline__ long long take(unsigned long long *ctr) {
        if (!dyn) {
            const long long t = cur;
            cur += stride;
            return t;
        }
        if (cur >= end) {
            cur = next;
            end = cur + kc;
            next = (long long)atomicAdd(ctr, (unsigned long long)kc);
        }
        return cur++;
    }
};

// Bounding box of a lane's points (see box_culled).
struct Box {
    float c[3], e[3], B;  // centre, half extent, sum_a max|p_a|
};

// float <-> int with the same order (for REDUX min/max of floats)
__device__ __forceinline__ int f2ord(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// The drain indexes the per-view layer table (LayerDesc, adop_internal.h) with a per-lane view slot:
// divergent constant-bank loads would serialise, so it reads the workspace copy through L1.



struct DepthSmem {
    float pos[kDStages][kSW][4][kWTile];  // stage, warp, row (x, y, z, r_world), point of the warp tile
    uint64_t bar[kSW][kDStages];          // per-warp TMA completion barriers
    uint64_t rbar[kSW][kDStages];         // per-warp barriers of the lazily loaded r_world row (kLazyR)
    int tile[kSW][kDStages];              // tile claimed into each stage (dynamic claiming / tile culling)
    uint32_t tviews[kSW][kDStages];       // tile culling: views whose frustum meets the tile's bounds
    WarpQueue q[kSW];
    uint8_t cand[kSW][kWTile];           // compacted candidate list of the warp tile (tile offsets)
};

// Tile culling, per lane: the views whose frustum may meet tile t (all views tested by this lane).
__device__ __forceinline__ uint32_t bounds_views_lane(const RasterArgs &a, int t) {
    const float4 lo = __ldg(reinterpret_cast<const float4 *>(a.tbounds) + 2 * t);
    const float4 hi = __ldg(reinterpret_cast<const float4 *>(a.tbounds) + 2 * t + 1);
    const float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
    if (!(l[0] <= h[0])) return 0u;
    Box w;
    float ext = 0.0f;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        w.c[ax] = 0.5f * (l[ax] + h[ax]);
        w.e[ax] = 0.5f * (h[ax] - l[ax]) * 1.0000002f;
        ext += fmaxf(fabsf(l[ax]), fabsf(h[ax]));
    }
    w.B = ext;
    uint32_t mask = 0u;
    for (int vv = 0; vv < a.nviews; ++vv) {
        const PlaneTab &v = a.planes[vv];
        bool out = false;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const float4 P = __ldg(&v.pl[k]);
            const float2 M = __ldg(&v.pm[k]);
            float val = P.w;
            val = fmaf(P.x, w.c[0], val);
            val = fmaf(fabsf(P.x), w.e[0], val);
            val = fmaf(P.y, w.c[1], val);
            val = fmaf(fabsf(P.y), w.e[1], val);
            val = fmaf(P.z, w.c[2], val);
            val = fmaf(fabsf(P.z), w.e[2], val);
            out |= val < -fmaf(M.x, w.B, M.y);
        }
        mask |= (out ? 0u : 1u) << vv;
    }
    return mask;
}

// Tile culling with precomputed per-tile bounds (adop_tile_bounds): the views whose (widened) frustum may
// contain a point of tile t, as a warp-uniform mask (lane v tests view v; the same conservative half-space
// test as the per-lane boxes).  Tiles without any view are neither loaded nor processed.
__device__ __forceinline__ uint32_t bounds_views(const RasterArgs &a, int t, int lane) {
    const float4 lo = __ldg(reinterpret_cast<const float4 *>(a.tbounds) + 2 * t);
    const float4 hi = __ldg(reinterpret_cast<const float4 *>(a.tbounds) + 2 * t + 1);
    const float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
    if (!(l[0] <= h[0])) return 0u;  // no valid point in the tile
    Box w;
    float ext = 0.0f;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        w.c[ax] = 0.5f * (l[ax] + h[ax]);
        w.e[ax] = 0.5f * (h[ax] - l[ax]) * 1.0000002f;  // covers the rounding of c -+ e
        ext += fmaxf(fabsf(l[ax]), fabsf(h[ax]));
    }
    w.B = ext;
    bool in = false;
    if (lane < a.nviews) {
        const PlaneTab &v = a.planes[lane];
        bool out = false;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const float4 P = __ldg(&v.pl[k]);
            const float2 M = __ldg(&v.pm[k]);
            float val = P.w;
            val = fmaf(P.x, w.c[0], val);
            val = fmaf(fabsf(P.x), w.e[0], val);
            val = fmaf(P.y, w.c[1], val);
            val = fmaf(fabsf(P.y), w.e[1], val);
            val = fmaf(P.z, w.c[2], val);
            val = fmaf(fabsf(P.z), w.e[2], val);
            out |= val < -fmaf(M.x, w.B, M.y);
        }
        in = !out;
    }
    return __ballot_sync(kFull, in);
}

__device__ __forceinline__ void init_layer_descs(const RasterArgs &a, LayerDesc *ld) {
    constexpr int F = 3 * ADOP_MAX_LAYERS + 1;
    for (int t = threadIdx.x; t < a.nviews * F; t += blockDim.x) {
        const int v = t / F, f = t % F;
        if (f < ADOP_MAX_LAYERS) ld[v].off[f] = a.v[v].off[f];
        else if (f < 2 * ADOP_MAX_LAYERS) ld[v].wl[f - ADOP_MAX_LAYERS] = a.v[v].wl[f - ADOP_MAX_LAYERS];
        else if (f < 3 * ADOP_MAX_LAYERS) ld[v].hl[f - 2 * ADOP_MAX_LAYERS] = a.v[v].hl[f - 2 * ADOP_MAX_LAYERS];
        else ld[v].keys = a.v[v].keys;
    }
}

// Views whose (widened) frustum may contain a point of the warp's tile, as a warp-uniform bit mask.
// With more than 2 views the warp's union box is tested against all views at once (lane v tests
// view v from the shared-memory table); otherwise every view is returned.
__device__ __forceinline__ uint32_t tile_views(const RasterArgs &a, const Box &b, int lane) {
    if (a.nviews <= 2) return (1u << a.nviews) - 1u;
    float lo[3], hi[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const bool valid = b.B >= 0.0f;
        const float l0 = valid ? b.c[ax] - b.e[ax] : __int_as_float(0x7f800000);
        const float h0 = valid ? b.c[ax] + b.e[ax] : -__int_as_float(0x7f800000);
        lo[ax] = ord2f(__reduce_min_sync(kFull, f2ord(l0)));
        hi[ax] = ord2f(__reduce_max_sync(kFull, f2ord(h0)));
    }
    if (!(lo[0] <= hi[0])) return 0u;  // no valid point in the tile
    Box w;
    float ext = 0.0f;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        w.c[ax] = 0.5f * (lo[ax] + hi[ax]);
        w.e[ax] = 0.5f * (hi[ax] - lo[ax]) * 1.0000002f;  // covers the rounding of c -+ e
        ext += fmaxf(fabsf(lo[ax]), fabsf(hi[ax]));
    }
    w.B = ext;
    bool in = false;
    if (lane < a.nviews) {
        const PlaneTab &v = a.planes[lane];
        bool out = false;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const float4 P = __ldg(&v.pl[k]);
            const float2 M = __ldg(&v.pm[k]);
            float val = P.w;
            val = fmaf(P.x, w.c[0], val);
            val = fmaf(fabsf(P.x), w.e[0], val);
            val = fmaf(P.y, w.c[1], val);
            val = fmaf(fabsf(P.y), w.e[1], val);
            val = fmaf(P.z, w.c[2], val);
            val = fmaf(fabsf(P.z), w.e[2], val);
            out |= val < -fmaf(M.x, w.B, M.y);
        }
        in = !out;
    }
    return __ballot_sync(kFull, in);
}

struct RecChunk {  // warp-uniform (pend: lane 0)
    unsigned long long base;
    int left;
#if ADOP_CHUNK_PREFETCH
    unsigned long long pend;  // old value of the next chunk's reservation, issued one chunk ahead
    bool has;
#endif
};

// A chunk that could not be reserved has base = capacity: its records are dropped (overflow is set).
__device__ __forceinline__ void put_record(const RasterArgs &a, unsigned long long slot, uint4 r) {
    ADOP_CHECK(r.w == 0xFFFFFFFFu || (r.w < (uint32_t)a.nviews && r.x < (uint32_t)a.v[r.w].pixels && r.z < (uint64_t)a.n));
    if (slot < (unsigned long long)a.rec_capacity) reinterpret_cast<uint4 *>(a.records)[slot] = r;
}

// mark the chunk's unused slots dead, then reserve a fresh chunk (one atomic per kChunk slots)
#if ADOP_CHUNK_PREFETCH
// validation of a front reservation whose atomicAdd returned o (see resv_take)
__device__ __forceinline__ unsigned long long front_validate(const RasterArgs &a, unsigned long long o) {
    const unsigned long long f = resv_front_used(o);
    if (f + kChunk + resv_back_slots(o) <= (unsigned long long)a.rec_capacity) {
        atomicMax(&a.hdr->front_ok, f + kChunk);
        return f;
    }
    atomicExch(&a.hdr->overflow, 1);
    return kNoSlot;
}
#endif

__device__ __forceinline__ void rec_reserve(const RasterArgs &a, RecChunk &c, int lane, bool fresh) {
    for (int k = lane; k < c.left; k += 32) put_record(a, c.base + k, make_uint4(0u, 0u, 0u, kDeadView));
#if ADOP_CHUNK_PREFETCH
    // the next chunk is reserved one chunk ahead, so the atomic's latency is not waited for
    unsigned long long b = 0;
    if (!fresh) {  // end of the sweep: the prefetched chunk is never used -- mark it dead
        if (!c.has) return;
        if (lane == 0) b = front_validate(a, c.pend);
        b = __shfl_sync(kFull, b, 0);
        if (b != kNoSlot)
            for (int k = lane; k < kChunk; k += 32) put_record(a, b + k, make_uint4(0u, 0u, 0u, kDeadView));
        return;
    }
    if (lane == 0) {
        const unsigned long long o = c.has ? c.pend : atomicAdd(&a.hdr->resv, (unsigned long long)kChunk);
        b = front_validate(a, o);
        c.pend = atomicAdd(&a.hdr->resv, (unsigned long long)kChunk);
    }
    c.has = true;
#else
    if (!fresh) return;
    unsigned long long b = 0;
    if (lane == 0) b = resv_take<false>(a, kChunk, true);
#endif
    b = __shfl_sync(kFull, b, 0);
    c.base = b == kNoSlot ? (unsigned long long)a.rec_capacity : b;
    c.left = kChunk;
}

// ---- work lists shared by the sweeps (front: records; back: ghost entries / depth candidates) ----
constexpr uint32_t kDead = 0xFFFFFFFFu;

struct ListChunk {  // warp-uniform per-warp chunk of a work list
    unsigned long long base;  // slot of the next free item
    int left;                 // items left in the chunk; -1: the list is full (process inline)
};

// Mark the chunk's unused items dead (front: Record.view, back: GhostEntry.vsnk).
template <bool BACK>
__device__ __forceinline__ void list_close(const RasterArgs &a, const ListChunk &c, int lane) {
    uint4 *r = reinterpret_cast<uint4 *>(a.records);
    for (int k = lane; k < c.left; k += 32) {
        if (BACK)
            r[c.base + 2ull * k + 1] = make_uint4(0u, 0u, kDead, kDead);
        else
            r[c.base + k] = make_uint4(0u, 0u, 0u, kDead);
    }
}

// Slots for the lanes in ballot b (front: 1 slot per item, back: 2); returns the lane's slot, or kNoSlot
// when the record region is full (the caller processes its item inline).  Warp-collective.
template <bool BACK>
__device__ __forceinline__ unsigned long long list_take(const RasterArgs &a, ListChunk &c, unsigned b, bool mine,
                                                        int lane, unsigned lt) {
    constexpr int W = BACK ? 2 : 1;
    const int nb = __popc(b);
    if (c.left >= 0 && nb > c.left) {
        list_close<BACK>(a, c, lane);
        unsigned long long s = 0;
        if (lane == 0) s = resv_take<BACK>(a, kChunk, false);
        s = __shfl_sync(kFull, s, 0);
        if (s == kNoSlot) {
            c.left = -1;
        } else {
            c.base = s;
            c.left = kChunk / W;
        }
    }
    if (c.left < 0) return kNoSlot;
    const unsigned long long slot = c.base + (unsigned long long)W * __popc(b & lt);
    c.base += (unsigned long long)W * nb;
    c.left -= nb;
    return mine ? slot : kNoSlot;
}


// Multi-view lists (RasterArgs::mv_lists): every kListChunk-slot chunk of the survivor list holds one view's
// records.  Lane w of the warp keeps view w's open chunk in c.base (the next free slot; a multiple of
// kListChunk means no room left).  The lanes of ballot b (record `rec` each, view `vs`) append to their
// views' chunks, one view at a time (a drain usually holds one or two views); a chunk that fills up is
// continued in a fresh one, whose view is written to the chunk table.  Warp-collective.
__device__ __forceinline__ void mv_put(const RasterArgs &a, RecChunk &c, unsigned b, bool hit, int vs, uint4 rec,
                                       int lane, unsigned lt) {
    unsigned pend = b;
    while (pend) {
        const int w = __shfl_sync(kFull, vs, __ffs(pend) - 1);
        const unsigned grp = __ballot_sync(kFull, hit && vs == w);
        const int cnt = __popc(grp);
        const unsigned long long st = __shfl_sync(kFull, c.base, w);
        const int used = (int)(st & (kListChunk - 1));
        const int room = used ? kListChunk - used : 0;
        unsigned long long nb = 0;
        if (cnt > room) {  // a fresh list chunk from the warp's pool (lane kPoolLane), refilled kChunk slots at a time
            unsigned long long pb = __shfl_sync(kFull, c.base, kPoolLane);
            int pl = __shfl_sync(kFull, c.left, kPoolLane);
            if (pl <= 0) {
                if (lane == 0) pb = resv_take<false>(a, kChunk, true);
                pb = __shfl_sync(kFull, pb, 0);
                pl = pb == kNoSlot ? 0 : kChunk / kListChunk;
            }
            if (pl > 0) {
                nb = pb;
                pb += kListChunk;
                --pl;
                if (lane == 0) a.cview[nb / kListChunk] = (uint8_t)w;
            } else {
                nb = (unsigned long long)a.rec_capacity;  // region full: dropped (overflow is set)
            }
            if (lane == kPoolLane) {
                c.base = pb;
                c.left = pl;
            }
        }
        if (hit && vs == w) {
            const int off = __popc(grp & lt);
            put_record(a, off < room ? st + off : nb + (off - room), rec);
        }
        if (lane == w) c.base = cnt <= room ? st + cnt : nb + (cnt - room);
        pend &= ~grp;
    }
}

// End of a multi-view sweep: lane w marks the rest of view w's open chunk dead; the pool lane marks its unused
// chunks dead (their chunk-table entry: no view).
__device__ __forceinline__ void mv_close(const RasterArgs &a, const RecChunk &c, int lane) {
    if (lane == kPoolLane) {
        for (int k = 0; k < c.left; ++k) {
            const unsigned long long b = c.base + (unsigned long long)k * kListChunk;
            a.cview[b / kListChunk] = 0xFF;
            for (int j = 0; j < kListChunk; ++j) put_record(a, b + j, make_uint4(0u, 0u, 0u, kDeadView));
        }
        return;
    }
    for (unsigned long long s = c.base; (s & (kListChunk - 1)) != 0; ++s) put_record(a, s, make_uint4(0u, 0u, 0u, kDeadView));
}

// Multi-view ghost list (RasterArgs::mv_lists): like mv_put for the back list -- lane vs keeps view vs's open
// chunk in c.base (next free slot; 2 slots per ghost entry); all items of a call share the warp-uniform view
// slot vs.  Returns the lane's slot or kNoSlot (region full: processed inline).  Warp-collective.
__device__ __forceinline__ unsigned long long mv_take_back(const RasterArgs &a, ListChunk &c, unsigned b, bool mine,
                                                           int vs, int lane, unsigned lt) {
    const int nb = __popc(b);
    const unsigned long long st = __shfl_sync(kFull, c.base, vs);
    const int used = (int)(st & (kListChunk - 1));
    const int room = used ? (kListChunk - used) / 2 : 0;
    unsigned long long nbase = 0;
    if (nb > room) {  // a fresh list chunk from the warp's pool (lane kPoolLane), refilled one back reservation at a time
        unsigned long long pb = __shfl_sync(kFull, c.base, kPoolLane);
        int pl = __shfl_sync(kFull, c.left, kPoolLane);
        if (pl <= 0) {
            if (lane == 0) pb = resv_take<true>(a, kChunk, false);
            pb = __shfl_sync(kFull, pb, 0);
            pl = pb == kNoSlot ? 0 : kChunk / kListChunk;
        }
        if (pl > 0) {
            nbase = pb;
            pb += kListChunk;
            --pl;
            if (lane == 0) a.cview[nbase / kListChunk] = (uint8_t)vs;
        } else {
            nbase = kNoSlot;  // region full: the items are processed inline
        }
        if (lane == kPoolLane) {
            c.base = pb;
            c.left = pl;
        }
    }
    const int off = __popc(b & lt);
    const unsigned long long slot =
        off < room ? st + 2ull * off : (nbase == kNoSlot ? kNoSlot : nbase + 2ull * (off - room));
    if (lane == vs) c.base = nb <= room ? st + 2ull * nb : (nbase == kNoSlot ? 0ull : nbase + 2ull * (nb - room));
    return mine ? slot : kNoSlot;
}

// End of a multi-view backward sweep: lane w marks the rest of view w's ghost chunk dead.
__device__ __forceinline__ void mv_close_back(const RasterArgs &a, const ListChunk &c, int lane) {
    uint4 *r = reinterpret_cast<uint4 *>(a.records);
    if (lane == kPoolLane) {
        for (int k = 0; k < c.left; ++k) {
            const unsigned long long b = c.base + (unsigned long long)k * kListChunk;
            a.cview[b / kListChunk] = 0xFF;
            for (int j = 0; j < kListChunk; j += 2) r[b + j + 1] = make_uint4(0u, 0u, kDead, kDead);
        }
        return;
    }
    for (unsigned long long s = c.base; (s & (kListChunk - 1)) != 0; s += 2) r[s + 1] = make_uint4(0u, 0u, kDead, kDead);
}

// Layers of one kept point per lane (nk = 0: idle lane).  Warp-collective.
template <bool MV>
__device__ __forceinline__ void depth_layers(const RasterArgs &a, const LayerDesc &v, int vs, int nk, float u0,
                                             float v0, uint32_t zbits, uint32_t idx, RecChunk &c, int lane,
                                             unsigned lt) {
    const uint64_t key = ((uint64_t)zbits << 32) | (a.goff + idx);
    Proj p;
    p.u0 = u0;
    p.v0 = v0;
#if ADOP_LAYER_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int l = 0; l < ADOP_MAX_LAYERS; ++l) {
        if (l >= a.layers) break;
        int pu, pv;
        const int loc = l < nk ? layer_pixel(v, p, l, pu, pv) : -1;
        const bool hit = loc >= 0;
        const uint32_t pix = (uint32_t)(v.off[l] + loc);
#if ADOP_PREREDUCE
        // warp-level pre-reduction (measured, see profiles/r02/evolution.md): lanes hitting the same (view, pixel)
        // min-reduce their keys with two 32-bit REDUX steps and only the group's winner issues the L2 reduction
        {
            const unsigned grp = __match_any_sync(kFull, hit ? (((unsigned long long)vs << 32) | pix) : ~0ull);
            const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
            const unsigned mhi = __reduce_min_sync(grp, hi);
            const unsigned mlo = __reduce_min_sync(grp, hi == mhi ? lo : 0xFFFFFFFFu);
            if (hit && hi == mhi && lo == mlo) red_min_u64_keep(v.keys + pix, key, policy_evict_last());
        }
#else
        ADOP_CHECK(!hit || (loc < v.wl[l] * v.hl[l] && (l + 1 >= ADOP_MAX_LAYERS || pix < (uint32_t)v.off[l + 1] ||
                                                         l + 1 >= a.layers)));
        if (hit) red_min_u64_keep(v.keys + pix, key, policy_evict_last());
#endif
        const unsigned b = __ballot_sync(kFull, hit);
        if (b == 0u) {
            if (!__any_sync(kFull, l + 1 < nk)) break;
            continue;
        }
        const int nb = __popc(b);
        CNT(4, nb);
        if (MV && a.mv_lists) {
            mv_put(a, c, b, hit, vs, make_uint4(pix, zbits, idx, (uint32_t)vs), lane, lt);
            continue;
        }
        if (nb > c.left) rec_reserve(a, c, lane, true);
        if (hit) put_record(a, c.base + __popc(b & lt), make_uint4(pix, zbits, idx, (uint32_t)vs));
        c.base += nb;
        c.left -= nb;
    }
}

// Process `cnt` (<= 32) entries from the top of the queue, one per lane (each with its own view slot).
template <bool MV>
#if ADOP_DRAIN_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void drain(const RasterArgs &a, const LayerDesc *ld, WarpQueue &q, int &qn, int cnt, RecChunk &c, int lane, unsigned lt) {
    __syncwarp();
    int nk = 0, vs = 0;
    float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane < cnt) {
        e = q.e[qn - cnt + lane];
        const int meta = q.meta[qn - cnt + lane];
        nk = meta & 15;
        vs = meta >> 4;
    }
    __syncwarp();
    qn -= cnt;
    depth_layers<MV>(a, ld[vs], vs, nk, e.x, e.y, __float_as_uint(e.z), __float_as_uint(e.w), c, lane, lt);
}

// Candidate part for one point and view: pinned Xc = R x + t (R1), validity (R7), exact discard (Eq. 12,
// R10) BEFORE the projection, exact projection (R2/R6); kept points are appended to the warp queue,
// which is drained 32 at a time.  Warp-collective.
// PRECHECK (multi-view launches, distortion / fisheye cameras): kept points outside the image at every layer
// are dropped before the queue (configs[4]: a quarter of the kept point-views; with distortion the pre-cull
// planes bound the whole valid cone, well beyond the image).  On the single-view pinhole headline the extra
// compares cost more than the few out-of-image points they save.
//
// Forward ghost listing (RasterArgs::ghost_fwd, R13 / R22): a candidate that is a ghost (`ghost`) takes the same exact
// test -- plus the in-bounds test of some kept layer, as the backward sweep's ghost emission (bwd_emit) -- and, if it
// passes, goes to the ghost list at the back of the record region instead of the depth test, so the backward
// consumes it without re-streaming the cloud.  A ghost whose slot cannot be reserved clears hdr->ghosts_fwd (the
// backward then re-finds every ghost with its sweep).  One exact path for both (a second inlined copy of it doubled
// the configs[4] depth pass: instruction-cache misses, 26% of the stall samples).
template <int MODEL, bool PRECHECK, bool MV>
__device__ __forceinline__ void depth_candidate(const RasterArgs &a, const ViewDesc &v, int vs, bool ok, float x,
                                                float y, float z, float rw, int64_t i, uint32_t gi, const LayerDesc *ld,
                                                WarpQueue &q, int &qn, RecChunk &c, int lane, unsigned lt,
                                                bool ghost = false, ListChunk *cg = nullptr) {
    Proj p;
    int nk = 0;
#if ADOP_COUNTERS
    bool c_valid = false, c_proj = false;
#endif
    if (ok) {
        to_camera(v, x, y, z, p.X, p.Y, p.Z);
        if (depth_valid<MODEL>(p, a.z_near) && (MODEL != 1 || !v.wn_on || in_window(v, p.X, p.Y, p.Z)) &&
            normal_keep(a, v, i, p.X, p.Y, p.Z)) {
            nk = keep_layers(a, v, rw, p.iz, gi);
#if ADOP_COUNTERS
            c_valid = true;
#endif
        }
    }
#if ADOP_COUNTERS
    {  // (ballots outside CNT: its argument is evaluated by lane 0 only)
        const unsigned b_valid = __ballot_sync(kFull, c_valid), b_disc = __ballot_sync(kFull, nk > 0);
        if (nk > 0) c_proj = project_uv<MODEL>(v, p);
        const unsigned b_proj = __ballot_sync(kFull, c_proj);
        CNT(5, __popc(b_valid));
        CNT(6, __popc(b_disc));
        CNT(7, __popc(b_proj));
    }
#endif
    if (nk > 0 && !(project_uv<MODEL>(v, p) && ((!PRECHECK && !ghost) || any_layer_in_bounds(v, p, nk)))) nk = 0;
    if (cg && __any_sync(kFull, ghost)) {  // ghost candidates: to the ghost list (GhostEntry, as bwd_emit)
        const bool gh = ghost && nk > 0;
        const unsigned bg = __ballot_sync(kFull, gh);
        if (bg != 0u) {
            const unsigned long long slot = (MV && a.mv_lists) ? mv_take_back(a, *cg, bg, gh, vs, lane, lt)
                                                               : list_take<true>(a, *cg, bg, gh, lane, lt);
            if (gh) {
                if (slot != kNoSlot) {
                    uint4 *r = reinterpret_cast<uint4 *>(a.records) + slot;
                    r[0] = make_uint4(__float_as_uint(p.u0), __float_as_uint(p.v0), __float_as_uint(p.X),
                                      __float_as_uint(p.Y));
                    r[1] = make_uint4(__float_as_uint(p.Z), (uint32_t)i, (uint32_t)(vs | (nk << 8)), __float_as_uint(p.D));
                } else {
                    *(volatile int32_t *)&a.hdr->ghosts_fwd = 0;
                }
            }
        }
        if (ghost) nk = 0;  // ghosts take no part in the depth test (§4.3)
    }
    const unsigned b = __ballot_sync(kFull, nk > 0);
    if (b == 0u) return;
    if (nk > 0) {
        const int slot = qn + __popc(b & lt);
        ADOP_CHECK(slot < kQCap && vs < 16);
        q.e[slot] = make_float4(p.u0, p.v0, p.D, __uint_as_float((uint32_t)i));
        q.meta[slot] = (uint8_t)(nk | (vs << 4));
    }
    qn += __popc(b);
    CNT(3, __popc(b));
    if (qn >= 32) drain<MV>(a, ld, q, qn, 32, c, lane, lt);
}


// The lane owns points e = h*128 + 4*lane + j (h = 0, 1; j = 0..3) of the warp tile: every LDS.128
// of a row is then one contiguous 512-byte warp access.
__device__ __forceinline__ float4 lane_row(const float *row, int lane, int h) {
    return *reinterpret_cast<const float4 *>(row + h * 128 + 4 * lane);
}

__device__ __forceinline__ Box lane_box(const float *const *rows, int lane, int valid) {
    Box b;
    float ext = 0.0f;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const float4 A = lane_row(rows[ax], lane, 0), Bv = lane_row(rows[ax], lane, 1);
        const float c[8] = {A.x, A.y, A.z, A.w, Bv.x, Bv.y, Bv.z, Bv.w};
        float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
        if (valid == 0xFF) {  // full tile: branch-free 3-input min/max trees
            // 3-input FMNMX3 chains: 8 values in 4 ops
            lo = fminf(fminf(fminf(fminf(fminf(fminf(c[0], c[1]), c[2]), c[3]), c[4]), fminf(c[5], c[6])), c[7]);
            hi = fmaxf(fmaxf(fmaxf(fmaxf(fmaxf(fmaxf(c[0], c[1]), c[2]), c[3]), c[4]), fmaxf(c[5], c[6])), c[7]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if ((valid >> j) & 1) {
                    lo = fminf(lo, c[j]);
                    hi = fmaxf(hi, c[j]);
                }
        }
        b.c[ax] = 0.5f * (lo + hi);
        b.e[ax] = 0.5f * (hi - lo);
        ext += fmaxf(fabsf(lo), fabsf(hi));
    }
    b.B = ext;
    if (!(b.e[0] >= 0.0f)) b.B = -1.0f;  // no valid point in the lane
    return b;
}

// true if no point of the lane's box can pass the exact projection test of view v (conservative:
// the planes hold with slack for every passing point; margins in adop_api.cu fill_args).
__device__ __forceinline__ bool box_culled(const ViewDesc &v, const Box &b) {
    if (b.B < 0.0f) return true;
    bool out = false;
#pragma unroll
    for (int k = 4; k >= 0; --k) {
        float val = v.pl[k][3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            val = fmaf(v.pl[k][ax], b.c[ax], val);
            val = fmaf(fabsf(v.pl[k][ax]), b.e[ax], val);
        }
        out |= val < -fmaf(v.pm[k][0], b.B, v.pm[k][1]);
    }
    return out;
}

// Early discard test (Eq. 12 at layer 0) on an upper bound of the projected radius: z >= Zf - m (the
// pre-cull's margin bounds |Zf - Zp|), r_screen <= gamma r_w f_eff / (Zf - m).  Returns false only if
// the exact test (R10) cannot keep the point at layer 0 -- and so at no layer (nested keep sets).
__device__ __forceinline__ bool maybe_kept(const RasterArgs &a, const ViewDesc &v, float rw, float Zf, float m,
                                           uint32_t gi) {
    const float zl = Zf - m;
    const float r = a.gamma * rw * v.feff * __fdividef(1.0f, zl);
    const uint32_t h = h24(v.discard_salt, gi);
    const float om = (float)(16777216u - h) * 5.9604644775390625e-8f;
    return !(zl > 0.0f) || r * r * 1.002f > om;
}

// Lazily loaded r_world row (kLazyR): the x, y, z rows of a warp tile are streamed for every tile, the r_world
// row only for a tile that some view's box test keeps (21% of the tiles on configs[3]; r_world is only read
// by the discard test of Eq. 12).  ensure_r issues its 1 KB bulk copy into the stage's row 3 and waits for it.
#ifndef ADOP_LAZY_R
#define ADOP_LAZY_R 0  // measured: no gain on configs[3] (0.3225 vs 0.3210 ms depth), slower tile culling
#endif
constexpr bool kLazyR = ADOP_LAZY_R;
struct LazyR {
    uint32_t bar, dst;  // the stage's r barrier and row-3 shared-memory address
    const float *src;   // global r_world of the tile, or nullptr when row 3 already holds it
    uint32_t parity;
};
__device__ __forceinline__ void ensure_r(LazyR &r, int lane) {
    if (!r.src) return;
    if (lane == 0) {
        mbar_expect_tx_a(r.bar, kWTile * sizeof(float));
        bulk_g2s_a(r.dst, r.src, kWTile * sizeof(float), r.bar, policy_evict_first());
    }
    mbar_wait_a(r.bar, r.parity);
    r.src = nullptr;
}

// The lane's 8 points of one warp tile (tile base index `base`, valid-point bit mask `vmask`), all views,
// read from the warp tile's shared-memory rows.
struct NoRelease {
    __device__ __forceinline__ void operator()() const {}
};
// EARLY (single-view pool kernel): a tile with at most kCBuf candidates copies their x, y, z, r_world into the warp's
// candidate buffer `cbuf` and calls release() -- the stage is refilled while the exact path runs from the copy, so a
// visible tile no longer holds its stage through the latency-bound exact path and drains.  Returns true if
// release() was called.
constexpr int kCBuf = 64;
template <int MODEL, int VM, bool DISC, bool SPLIT = false, bool EARLY = false, typename Rel = NoRelease>
__device__ __forceinline__ bool depth_lane8(const RasterArgs &a, const float *const *rows, int64_t base, int vmask,
                                            bool staged_r, const LayerDesc *ld, WarpQueue &q, int &qn, RecChunk &c,
                                            uint8_t *cl, int lane, unsigned lt, uint32_t pre_views, LazyR &lr,
                                            ListChunk *cc = nullptr, float4 *cbuf = nullptr, Rel &&release = Rel()) {
    auto pidx = [&](int j) { return base + (j >> 2) * 128 + 4 * lane + (j & 3); };
    // ghosts take no part in the depth test (§4.3): their mask is hashed at the tile's first visible view
    uint32_t live = (uint32_t)vmask;
    const bool gf = !SPLIT && !EARLY && a.ghost_fwd;  // this pass lists the ghosts (ghost_thr != 0)
    bool live_done = a.ghost_thr == 0u || gf;
    const Box box = lane_box(rows, lane, vmask);
    uint32_t views = pre_views != 0xFFFFFFFFu ? pre_views
                     : (VM == 2 ? tile_views(a, box, lane) : (VM == 0 ? 1u : (1u << a.nviews) - 1u));
#pragma unroll 1
    while (views) {
        const int vs = VM == 0 ? 0 : __ffs(views) - 1;  // VM 0: compile-time view 0 (constant-bank operands)
        views &= views - 1u;
        const ViewDesc &v = a.v[vs];
        const bool lane_out = box_culled(v, box);
        if (__all_sync(kFull, lane_out)) continue;  // every lane's box is outside (warp-uniform)
        CNT(1, 1);
        if (kLazyR && staged_r) ensure_r(lr, lane);
        uint32_t m = 0u;
        // DISC = stochastic discarding on (a separate instance: each keeps only the code it runs)
        if (kPrefilter && DISC && (MODEL != 2 || v.zplane)) {
            // Discard prefilter (Eq. 12 on a lane bound): the near plane's minimum over the lane box bounds every
            // point's depth from below (margins as box_culled), so r_screen <= r_max = gamma r_w,max f_eff / z_lo
            // and a point can be kept at layer 0 -- hence at any layer -- only if 1 - beta < r_max^2, i.e. its
            // hash h > H = 2^24 (1 - r_max^2) (with slack).  Only those go to the exact path; no per-point
            // frustum pre-cull (the exact path's bounds test decides).
            float vmin = v.pl[4][3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                vmin = fmaf(v.pl[4][ax], box.c[ax], vmin);
                vmin = fmaf(-fabsf(v.pl[4][ax]), box.e[ax], vmin);
            }
            const float zlo = (vmin - fmaf(v.pm[4][0], box.B, v.pm[4][1])) * 0.9999f + v.zoff;
            float rwmax = a.radius_uniform;
            if (staged_r) {
                const float4 R0 = lane_row(rows[3], lane, 0), R1 = lane_row(rows[3], lane, 1);
                rwmax = fmaxf(fmaxf(fmaxf(R0.x, R0.y), fmaxf(R0.z, R0.w)), fmaxf(fmaxf(R1.x, R1.y), fmaxf(R1.z, R1.w)));
            }
            bool all = true;
            uint32_t H = 0u;
            if (zlo > 0.0f) {
                const float rmax = a.gamma * rwmax * v.feff / zlo;
                const float qk = rmax * rmax * 1.004f;
                if (qk < 1.0f) {
                    const float hf = 16777216.0f * (1.0f - qk);
                    if (hf > 4.0f) {
                        H = (uint32_t)hf - 2u;
                        all = false;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                m |= ((all || h24(v.discard_salt, a.goff + (uint32_t)pidx(j)) > H) ? 1u : 0u) << j;
            if (lane_out) m = 0u;
        } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 X = lane_row(rows[0], lane, h), Y = lane_row(rows[1], lane, h), Z = lane_row(rows[2], lane, h);
            const float4 Rw = staged_r ? lane_row(rows[3], lane, h)
                                       : make_float4(a.radius_uniform, a.radius_uniform, a.radius_uniform,
                                                     a.radius_uniform);
            const float xs[4] = {X.x, X.y, X.z, X.w}, ys[4] = {Y.x, Y.y, Y.z, Y.w}, zs[4] = {Z.x, Z.y, Z.z, Z.w};
            const float rs[4] = {Rw.x, Rw.y, Rw.z, Rw.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float Zf, mz;
                bool cand = precull_fma_z<MODEL>(v, xs[j], ys[j], zs[j], Zf, mz);
                if (DISC) cand &= maybe_kept(a, v, rs[j], Zf, mz, a.goff + (uint32_t)pidx(4 * h + j));
                m |= (cand ? 1u : 0u) << (4 * h + j);
            }
        }
        }
        if (!live_done) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (h24(a.ghost_salt, a.goff + (uint32_t)pidx(j)) < a.ghost_thr) live &= ~(1u << j);
            live_done = true;
        }
        m &= gf ? (uint32_t)vmask : live;  // (listing ghosts: they stay candidates, flagged per candidate below)
        if (!__any_sync(kFull, m != 0u)) continue;
        // compact the warp's candidates into a list of tile offsets, then run the exact path 32 at a time
        // with every lane busy (a per-lane loop would idle the lanes whose points are all rejected)
        int cn = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const bool bit = (m >> j) & 1u;
            const unsigned b = __ballot_sync(kFull, bit);
            ADOP_CHECK(!bit || cn + __popc(b & lt) < kWTile);
            if (bit) cl[cn + __popc(b & lt)] = (uint8_t)((j >> 2) * 128 + 4 * lane + (j & 3));
            cn += __popc(b);
        }
        __syncwarp();
        CNT(2, cn);
        if constexpr (EARLY && VM == 0) {
            if (cn <= kCBuf) {
                for (int k = lane; k < cn; k += 32) {
                    const int e = cl[k];
                    cbuf[k] = make_float4(rows[0][e], rows[1][e], rows[2][e], staged_r ? rows[3][e] : a.radius_uniform);
                }
                __syncwarp();
                release();  // the stage is free: refilled while the exact path runs from the copy
                for (int i0 = 0; i0 < cn; i0 += 32) {
                    const bool ok = i0 + lane < cn;
                    const int e = ok ? cl[i0 + lane] : 0;
                    const float4 pc = cbuf[ok ? i0 + lane : 0];
                    depth_candidate<MODEL, MODEL != 0, false>(a, v, vs, ok, pc.x, pc.y, pc.z, pc.w, base + e,
                                                              a.goff + (uint32_t)(base + e), ld, q, qn, c, lane, lt);
                }
                __syncwarp();
                return true;
            }
        }
        for (int i0 = 0; i0 < cn; i0 += 32) {
            bool ok = i0 + lane < cn;
            const int e = ok ? cl[i0 + lane] : 0;
            const float rw = staged_r ? rows[3][e] : a.radius_uniform;
            if (SPLIT) {  // hand the candidate to k_depth_exact: {x, y, z, r_world}, {index, view, live} in the back list
                const unsigned long long slot = list_take<true>(a, *cc, __ballot_sync(kFull, ok), ok, lane, lt);
                if (ok && slot != kNoSlot) {
                    uint4 *r = reinterpret_cast<uint4 *>(a.records) + slot;
                    r[0] = make_uint4(__float_as_uint(rows[0][e]), __float_as_uint(rows[1][e]), __float_as_uint(rows[2][e]),
                                      __float_as_uint(rw));
                    r[1] = make_uint4((uint32_t)(base + e), (uint32_t)vs, 0u, 0u);
                    ok = false;
                }
                if (!__any_sync(kFull, ok)) continue;  // (the region is full: the rest is processed here)
            }
            const uint32_t gi = a.goff + (uint32_t)(base + e);
            const bool ghost = gf && ok && h24(a.ghost_salt, gi) < a.ghost_thr;
            depth_candidate<MODEL, VM != 0 || MODEL != 0, VM == 2>(a, v, vs, ok, rows[0][e], rows[1][e], rows[2][e], rw, base + e,
                                   gi, ld, q, qn, c, lane, lt, ghost, gf ? cc : nullptr);
        }
        __syncwarp();  // the list is rewritten by the next view / tile
    }
    return false;
}

static_assert(sizeof(DepthSmem) + 1024 <= 228 * 1024 / kDCTAs, "depth sweep: kDCTAs CTAs per SM must fit in shared memory");

template <int MODEL, int VM, bool DISC>
__global__ void __launch_bounds__(kST, kDCTAs) k_depth_async(const __grid_constant__ RasterArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DepthSmem &sm = *reinterpret_cast<DepthSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned lt = lanemask_lt();
    static_assert(kWTile == 256, "RasterArgs::ntiles / nfull are counted in 256-point tiles");
    const int ntiles = a.ntiles, nfull = a.nfull;  // tiles [0, nfull) are full: TMA-streamed
    const bool staged_r = a.discard && a.radius != nullptr;
    const int rows = staged_r ? 4 : 3;
    const bool dyn = a.dyn_tiles & 1;
    const bool tcull = a.tbounds != nullptr;  // the claimed tile goes through shared memory (sm.tile)
    if (lane == 0) {
        for (int st = 0; st < kDStages; ++st) {
            mbar_init(&sm.bar[wid][st], 1);
            mbar_init(&sm.rbar[wid][st], 1);
        }
        fence_mbar_init();
    }
    __syncwarp();
    // per-warp constants of the issue path: shared-window addresses, L2 policy, tile sequence
    constexpr uint32_t kStageBytes = sizeof(sm.pos[0]), kRowBytes = kWTile * sizeof(float);
    const uint32_t bar_s = smem_addr(&sm.bar[wid][0]);
    const uint32_t rbar_s = smem_addr(&sm.rbar[wid][0]);
    const uint32_t pos_s = smem_addr(&sm.pos[0][wid][0][0]);
    const int streamed = kLazyR ? 3 : rows;  // rows every tile streams (r_world lazily with kLazyR)
    const uint32_t txb = (uint32_t)streamed * kRowBytes;
    const uint64_t pol = policy_evict_first();
    const int stride = (int)gridDim.x * kSW;
    int t_next = (int)blockIdx.x * kSW + wid;  // static order: warp w takes tiles w, w + W, ...
    TileClaim tc;
    if (dyn && lane == 0) tc.init(&a.hdr->tiles_fwd, ntiles, stride, t_next, true);
    uint32_t win_rem = 0u, win_lmask = 0u;  // tile culling window (static claiming)
    int win_t0 = 0;
    // lane 0 claims the stage's next tile and streams its rows with the TMA engine (L2 evict-first):
    // x, y, z in one 2-D tensor copy (or three 1-D bulk copies), r_world in a 1-D bulk copy
    auto issue = [&](int st) {
        int t;
        if (tcull && !dyn) {
            // warp-collective window scan: lane i tests tile t_next + i * stride (one round trip for 32 tiles),
            // the visible ones are then issued one by one
            uint32_t views = 0u;
            for (;;) {
                if (win_rem == 0u) {
                    if (t_next >= ntiles) {
                        t = ntiles;
                        break;
                    }
                    const int ti = t_next + lane * stride;
                    win_lmask = ti < ntiles ? bounds_views_lane(a, ti) : 0u;
                    win_t0 = t_next;
                    t_next += 32 * stride;
                    win_rem = __ballot_sync(kFull, win_lmask != 0u);
                    continue;
                }
                const int i = __ffs(win_rem) - 1;
                win_rem &= win_rem - 1u;
                t = win_t0 + i * stride;
                views = __shfl_sync(kFull, win_lmask, i);
                break;
            }
            if (lane != 0) return;
            sm.tile[wid][st] = t;
            sm.tviews[wid][st] = views;
            if (t < ntiles) atomicAdd(&a.hdr->tiles_read, 1ull);
        } else if (tcull) {  // dynamic claiming: tile by tile (lane v tests view v)
            uint32_t views;
            for (;;) {
                if (lane == 0) {
                    if (dyn) {
                        t = (int)tc.take(&a.hdr->tiles_fwd);
                    } else {
                        t = t_next;
                        t_next += stride;
                    }
                }
                t = __shfl_sync(kFull, t, 0);
                if (t >= ntiles) {
                    views = 0u;
                    break;
                }
                views = bounds_views(a, t, lane);
                if (views) break;
            }
            if (lane != 0) return;
            sm.tile[wid][st] = t;
            sm.tviews[wid][st] = views;
            if (t < ntiles) atomicAdd(&a.hdr->tiles_read, 1ull);
        } else {
            if (lane != 0) return;
            if (dyn) {
                t = (int)tc.take(&a.hdr->tiles_fwd);
                sm.tile[wid][st] = t;
            } else {
                t = t_next;
                t_next += stride;
            }
        }
        if (t < nfull) {
            const uint32_t bar = bar_s + 8u * st, dst = pos_s + kStageBytes * st;
            mbar_expect_tx_a(bar, txb);
            if (a.use_tmap) {
                tensor_g2s_2d_a(dst, &a.tmap, t * kWTile, 0, bar, pol);
            } else {
                for (int r = 0; r < 3; ++r) {
                    const float *src = r == 0 ? a.x : (r == 1 ? a.y : a.z);
                    bulk_g2s_a(dst + r * kRowBytes, src + (int64_t)t * kWTile, kRowBytes, bar, pol);
                }
            }
            if (streamed == 4) bulk_g2s_a(dst + 3 * kRowBytes, a.radius + (int64_t)t * kWTile, kRowBytes, bar, pol);
        }
    };
    for (int st = 0; st < kDStages; ++st) issue(st);
    __syncwarp();
    WarpQueue &q = sm.q[wid];
    int qn = 0;
    RecChunk c;
    c.base = 0;
    c.left = 0;
#if ADOP_CHUNK_PREFETCH
    c.has = false;
    c.pend = 0;
#endif
    uint32_t phase = 0u, rphase = 0u;
    int t_cons = (int)blockIdx.x * kSW + wid;
    for (int st = 0;; st = st + 1 == kDStages ? 0 : st + 1) {
        int t;
        uint32_t pre_views = 0xFFFFFFFFu;
        if (dyn || tcull) {
            t = *(volatile int *)&sm.tile[wid][st];
            if (tcull) pre_views = *(volatile uint32_t *)&sm.tviews[wid][st];
        } else {
            t = t_cons;
            t_cons += stride;
        }
        if (t >= ntiles) break;
        const int64_t base = (int64_t)t * kWTile;
        const float *rp[4] = {sm.pos[st][wid][0], sm.pos[st][wid][1], sm.pos[st][wid][2], sm.pos[st][wid][3]};
        int vmask = 0xFF;
        if (t < nfull) {
            mbar_wait_a(bar_s + 8u * st, (phase >> st) & 1u);
            phase ^= 1u << st;
        } else {  // ragged last tile: guarded loads into this stage (no copy was issued for it)
            const float *src[4] = {a.x, a.y, a.z, a.radius};
            vmask = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int e = (j >> 2) * 128 + 4 * lane + (j & 3);
                const bool in = base + e < a.n;
                for (int r = 0; r < 4; ++r)
                    sm.pos[st][wid][r][e] = (in && r < rows) ? src[r][base + e] : 0.f;
                vmask |= (in ? 1 : 0) << j;
            }
            __syncwarp();
        }
        CNT(0, 1);
        LazyR lr;
        lr.bar = rbar_s + 8u * st;
        lr.dst = pos_s + kStageBytes * st + 3 * kRowBytes;
        lr.src = (kLazyR && staged_r && t < nfull) ? a.radius + base : nullptr;  // (a ragged tile loaded row 3)
        lr.parity = (rphase >> st) & 1u;
        const bool r_pending = lr.src != nullptr;
        depth_lane8<MODEL, VM, DISC>(a, rp, base, vmask, staged_r, a.ldesc, q, qn, c, sm.cand[wid], lane, lt, pre_views,
                                     lr);
        if (r_pending && !lr.src) rphase ^= 1u << st;
        __syncwarp();  // every lane is done with stage st
        issue(st);
        __syncwarp();
    }
    if (qn > 0) drain<VM == 2>(a, a.ldesc, q, qn, qn, c, lane, lt);
    if (VM == 2 && a.mv_lists)
        mv_close(a, c, lane);        // lane w: the rest of view w's chunk
    else
        rec_reserve(a, c, lane, false);  // mark this warp's unused slots dead
}

// --------------------------------------------------------------------------- //
// depth pass with a CTA-wide pool of stages (launches without tile culling or dynamic claiming): the CTA's k-th
// warp tile is tile k G + b (G CTAs; all CTAs sweep the cloud as one
// front) and lands in stage k mod kPool.  A warp claims the next k of its CTA, waits for that stage, processes
// the tile and refills the stage with tile k + kPool.  Unlike the per-warp rings, a loaded stage never waits
// for a particular warp: a warp busy with a visible tile holds one stage, every other loaded stage goes to the
// next free warp (the per-warp rings left the busy warp's prefetched tile idle).
// --------------------------------------------------------------------------- //
#ifndef ADOP_POOL_STAGES
#define ADOP_POOL_STAGES 16  // (14 with the early-release candidate buffers)
#endif
#ifndef ADOP_EARLY_RELEASE
#define ADOP_EARLY_RELEASE 0  // measured: no gain (profiles/r02/evolution.md)
#endif
constexpr int kPool = ADOP_POOL_STAGES;
#ifndef ADOP_PCTAS
#define ADOP_PCTAS 3  // pooled depth sweep CTAs per SM
#endif
constexpr int kPCTAs = ADOP_PCTAS;
#ifndef ADOP_POOL_SLEEP
#define ADOP_POOL_SLEEP 64  // ns between polls of a stage whose refill is not issued yet
#endif
constexpr int kPoolSV = 11, kPoolMV = kPool;
template <int NP>
struct PoolSmemT {
    float pos[NP][4][kWTile];
    uint64_t bar[NP];
    int filled[NP];  // the k whose copy into the stage was issued last (phase-unambiguous waits)
    int next;
    WarpQueue q[kSW];
    uint8_t cand[kSW][kWTile];
#if ADOP_EARLY_RELEASE
    float4 cbuf[kSW][kCBuf];  // early release: the warp's candidates of its current tile
#endif
};
// Single-view launches: 4 CTAs x 11 stages per SM (32 warps; headline depth -2%); multi-view ones keep 3 x 16
// (configs[4] forward +5% with 4 x 11): profiles/r02/evolution.md.
template <int NP> constexpr int pool_ctas() { return NP == kPoolSV ? 4 : kPCTAs; }
static_assert(sizeof(PoolSmemT<kPoolSV>) + 1024 <= 228 * 1024 / 4, "pooled depth sweep: 4 CTAs x 11 stages per SM");
static_assert(sizeof(PoolSmemT<kPoolMV>) + 1024 <= 228 * 1024 / kPCTAs, "pooled depth sweep: kPCTAs CTAs per SM must fit");

template <int MODEL, int VM, bool DISC, bool SPLIT, int NP>
__global__ void __launch_bounds__(kST, pool_ctas<NP>()) k_depth_pool(const __grid_constant__ RasterArgs a) {
    constexpr int kPool = NP;
    using PoolSmem = PoolSmemT<NP>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PoolSmem &sm = *reinterpret_cast<PoolSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned lt = lanemask_lt();
    const int ntiles = a.ntiles, nfull = a.nfull;
    const bool staged_r = a.discard && a.radius != nullptr;
    const int rows = staged_r ? 4 : 3;
    const int G = (int)gridDim.x, b = (int)blockIdx.x;
    if (tid < kPool) {
        mbar_init(&sm.bar[tid], 1);
        sm.filled[tid] = -1;
    }
    if (tid == 0) sm.next = 0;
    fence_mbar_init();
    __syncthreads();
    constexpr uint32_t kStageBytes = sizeof(sm.pos[0]), kRowBytes = kWTile * sizeof(float);
    const uint32_t bar0 = smem_addr(&sm.bar[0]), pos0 = smem_addr(&sm.pos[0][0][0]);
    const uint32_t txb = (uint32_t)rows * kRowBytes;
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int k) {  // lane 0: stream the CTA's k-th tile into stage k mod kPool
        const int t = k * G + b;
        if (t >= ntiles) return;
        const int s = k % kPool;
        const uint32_t bar = bar0 + 8u * s, dst = pos0 + kStageBytes * s;
        *(volatile int *)&sm.filled[s] = k;
        if (t >= nfull) {  // ragged last tile: its consumer loads it; the arrival only releases the stage
            mbar_arrive_a(bar);
            return;
        }
        mbar_expect_tx_a(bar, txb);
        if (a.use_tmap) {
            tensor_g2s_2d_a(dst, &a.tmap, t * kWTile, 0, bar, pol);
        } else {
            for (int r = 0; r < 3; ++r) {
                const float *src = r == 0 ? a.x : (r == 1 ? a.y : a.z);
                bulk_g2s_a(dst + r * kRowBytes, src + (int64_t)t * kWTile, kRowBytes, bar, pol);
            }
        }
        if (rows == 4) bulk_g2s_a(dst + 3 * kRowBytes, a.radius + (int64_t)t * kWTile, kRowBytes, bar, pol);
    };
    if (lane == 0)
        for (int k0 = wid; k0 < kPool; k0 += kSW) issue(k0);
    __syncwarp();
    WarpQueue &q = sm.q[wid];
    int qn = 0;
    RecChunk c;
    c.base = 0;
    c.left = 0;
#if ADOP_CHUNK_PREFETCH
    c.has = false;
    c.pend = 0;
#endif
    LazyR lr;
    lr.src = nullptr;
    ListChunk cc;  // SPLIT: this warp's chunk of the candidate list
    cc.base = 0;
    cc.left = 0;
    for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(&sm.next, 1);
        k = __shfl_sync(kFull, k, 0);
        const int t = k * G + b;
        if (t >= ntiles) break;
        const int s = k % kPool;
        const int64_t base = (int64_t)t * kWTile;
        const float *rp[4] = {sm.pos[s][0], sm.pos[s][1], sm.pos[s][2], sm.pos[s][3]};
        // the stage's barrier alternates parity per use: wait until tile k's copy was issued (tile k - kPool is then
        // done with the stage), so the parity names tile k's phase and not a later or earlier one
        while (*(volatile int *)&sm.filled[s] != k) __nanosleep(ADOP_POOL_SLEEP);
        mbar_wait_a(bar0 + 8u * s, (uint32_t)(k / kPool) & 1u);
        int vmask = 0xFF;
        if (t >= nfull) {  // ragged last tile: guarded loads into the released stage
            const float *src[4] = {a.x, a.y, a.z, a.radius};
            vmask = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int e = (j >> 2) * 128 + 4 * lane + (j & 3);
                const bool in = base + e < a.n;
                for (int r = 0; r < 4; ++r) sm.pos[s][r][e] = (in && r < rows) ? src[r][base + e] : 0.f;
                vmask |= (in ? 1 : 0) << j;
            }
            __syncwarp();
        }
        CNT(0, 1);
        constexpr bool kEarly = ADOP_EARLY_RELEASE && VM == 0 && !SPLIT;
        auto rel = [&]() {
            if (lane == 0) issue(k + kPool);
            __syncwarp();
        };
        const bool released = depth_lane8<MODEL, VM, DISC, SPLIT, kEarly>(
            a, rp, base, vmask, staged_r, a.ldesc, q, qn, c, sm.cand[wid], lane, lt, 0xFFFFFFFFu, lr, &cc,
#if ADOP_EARLY_RELEASE
            sm.cbuf[wid],
#else
            nullptr,
#endif
            rel);
        __syncwarp();  // every lane is done with stage s
        if (!released) rel();
    }
    if (SPLIT) list_close<true>(a, cc, lane);
    if (!SPLIT && a.ghost_fwd) {  // the rest of this warp's ghost-list chunk(s)
        if (VM == 2 && a.mv_lists)
            mv_close_back(a, cc, lane);
        else
            list_close<true>(a, cc, lane);
    }
    if (qn > 0) drain<VM == 2>(a, a.ldesc, q, qn, qn, c, lane, lt);
    if (VM == 2 && a.mv_lists)
        mv_close(a, c, lane);
    else
        rec_reserve(a, c, lane, false);
}

// The exact part of a split depth pass (ADOP_DEPTH_SPLIT): the candidates k_depth_pool<SPLIT> compacted into the
// back list -- 32 per warp iteration, every warp busy -- through the same exact path, queue and drains.  The cull
// kernel then streams the cloud with little per-tile work and no long visible-tile latency chains, which kept
// its loaded stages waiting; the candidates (1.57M on configs[3]) cost 32 B written and read each.
struct ExactSmem {
    WarpQueue q[kWarps];
};
template <int MODEL, int VM>
__global__ void __launch_bounds__(kThreads) k_depth_exact(const __grid_constant__ RasterArgs a) {
    __shared__ ExactSmem sm;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const unsigned long long back = *(volatile unsigned long long *)&a.hdr->back_ok;
    const uint4 *list = reinterpret_cast<const uint4 *>(a.records) + ((unsigned long long)a.rec_capacity - back);
    const unsigned long long total = back / 2;
    WarpQueue &q = sm.q[wid];
    int qn = 0;
    RecChunk c;
    c.base = 0;
    c.left = 0;
#if ADOP_CHUNK_PREFETCH
    c.has = false;
    c.pend = 0;
#endif
    const unsigned long long W = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long gw = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // global warp
    for (unsigned long long j0 = gw * 32; j0 < total; j0 += W * 32) {
        const unsigned long long j = j0 + lane;
        bool ok = j < total;
        uint4 e0 = make_uint4(0u, 0u, 0u, 0u), e1 = make_uint4(0u, 0u, kDead, 0u);
        if (ok) {
            e1 = __ldcs(list + 2 * j + 1);
            ok = e1.z != kDead;
            if (ok) e0 = __ldcs(list + 2 * j);
        }
        const int vs = ok ? (int)e1.y : 0;
        ADOP_CHECK(!ok || (vs < a.nviews && e1.x < (uint64_t)a.n));
        // (single-view instances: vs = 0 for every candidate, so the warp-uniform view argument holds)
        depth_candidate<MODEL, VM != 0 || MODEL != 0, VM == 2>(a, a.v[VM == 0 ? 0 : vs], vs, ok, __uint_as_float(e0.x),
                                                               __uint_as_float(e0.y), __uint_as_float(e0.z),
                                                               __uint_as_float(e0.w), (int64_t)e1.x, a.goff + e1.x,
                                                               a.ldesc, q, qn, c, lane, lt);
    }
    if (qn > 0) drain<VM == 2>(a, a.ldesc, q, qn, qn, c, lane, lt);
    rec_reserve(a, c, lane, false);
}

// Shared-pyramid reset (adop_clear_pyramid): keys <- sentinel, accum / count <- 0.
__global__ void __launch_bounds__(kThreads) k_clear_pyr(unsigned long long *keys, float *accum, float *count, int64_t P,
                                                        int C) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P; q += stride) {
        keys[q] = 0x7FFFFFFFFFFFFFFFull;
        count[q] = 0.0f;
        for (int c = 0; c < C; ++c) accum[q * C + c] = 0.0f;
    }
}

int launch_clear_pyr(uint64_t *keys, float *accum, float *count, int64_t P, int C, void *stream) {
    int64_t g = (P + kThreads - 1) / kThreads;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    k_clear_pyr<<<(unsigned)g, kThreads, 0, (cudaStream_t)stream>>>(reinterpret_cast<unsigned long long *>(keys), accum,
                                                                   count, P, C);
    return (int)cudaGetLastError();
}

// Per-tile bounds for tile culling: warp per 256-point tile, AABB of its finite points (lo.xyz, -, hi.xyz, -).
__global__ void __launch_bounds__(kThreads) k_tile_bounds(const float *x, const float *y, const float *z, int64_t n,
                                                          float4 *out) {
    const int lane = threadIdx.x & 31;
    const int64_t ntiles = (n + kWTile - 1) / kWTile;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; t < ntiles;
         t += (int64_t)gridDim.x * blockDim.x / 32) {
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int k = lane; k < kWTile; k += 32) {
            const int64_t i = t * kWTile + k;
            if (i >= n) break;
            const float p[3] = {x[i], y[i], z[i]};
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                lo[ax] = fminf(lo[ax], p[ax]);  // NaN coordinates are ignored (such points are invalid, R7)
                hi[ax] = fmaxf(hi[ax], p[ax]);
            }
        }
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            lo[ax] = ord2f(__reduce_min_sync(kFull, f2ord(lo[ax])));
            hi[ax] = ord2f(__reduce_max_sync(kFull, f2ord(hi[ax])));
        }
        if (lane == 0) {
            out[2 * t] = make_float4(lo[0], lo[1], lo[2], 0.f);
            out[2 * t + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
        }
    }
}

int launch_tile_bounds(const float *x, const float *y, const float *z, int64_t n, float *out, void *stream) {
    const int64_t ntiles = (n + kWTile - 1) / kWTile;
    int64_t g = (ntiles * 32 + kThreads - 1) / kThreads;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    k_tile_bounds<<<(unsigned)g, kThreads, 0, (cudaStream_t)stream>>>(x, y, z, n, reinterpret_cast<float4 *>(out));
    return (int)cudaGetLastError();
}

// --------------------------------------------------------------------------- //
// blend over survivor records (§4.5 accumulate pass)
// --------------------------------------------------------------------------- //
// (Measured: a separate low-register record kernel at higher occupancy moved more DRAM bytes and ran
// slower on configs[4]; the L2 reductions, not latency, bound this pass.)
// HOCC: 6 blocks per SM (40 registers; the overflow fallback spills, it is the slow path anyway) -- one
// view: blend phase 63 -> 58 us on configs[3]; with 16 views (configs[4]) the extra concurrency thrashes
// L2 (forward 4.73 -> 5.17 ms), so multi-view launches keep 4 blocks per SM.
// ---- view-major order of a multi-view list's chunks (list 0: survivor records, 1: ghost entries) ----
// Chunk range of a list in the chunk table: the front list [0, front_ok) grows from slot 0, the back list
// [capacity - back_ok, capacity) from the top; both consist of whole kListChunk-slot chunks.
__device__ __forceinline__ void list_chunks(const RasterArgs &a, int list, unsigned long long &c0,
                                            unsigned long long &c1) {
    const unsigned long long cap = (unsigned long long)a.rec_capacity;
    if (list == 0) {
        c0 = 0;
        c1 = *(volatile unsigned long long *)&a.hdr->front_ok / kListChunk;
    } else {
        c1 = cap / kListChunk;
        c0 = (cap - *(volatile unsigned long long *)&a.hdr->back_ok) / kListChunk;
    }
}
__device__ __forceinline__ int chunk_bucket(const RasterArgs &a, unsigned long long c) {
    const unsigned v = a.cview[c];
    return v < (unsigned)a.nviews ? (int)v : ADOP_MAX_VIEWS_PER_LAUNCH;  // 16: not a per-view chunk
}
// Per-view chunk counts (ccount[list][0..16], zeroed by the launcher).
__global__ void __launch_bounds__(kThreads) k_chunk_hist(const __grid_constant__ RasterArgs a, int list) {
    __shared__ unsigned h[ADOP_MAX_VIEWS_PER_LAUNCH + 1];
    if (threadIdx.x <= ADOP_MAX_VIEWS_PER_LAUNCH) h[threadIdx.x] = 0u;
    __syncthreads();
    unsigned long long c0, c1;
    list_chunks(a, list, c0, c1);
    for (unsigned long long c = c0 + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; c < c1;
         c += (unsigned long long)gridDim.x * blockDim.x)
        atomicAdd(&h[chunk_bucket(a, c)], 1u);
    __syncthreads();
    if (threadIdx.x <= ADOP_MAX_VIEWS_PER_LAUNCH && h[threadIdx.x])
        atomicAdd(&a.ccount[list * 64 + threadIdx.x], h[threadIdx.x]);
}
// Scatter every chunk index to its view's segment of corder[list] (segments in view order; the order inside a
// segment is arbitrary -- the consumers' results do not depend on it beyond fp32 summation order).
__global__ void __launch_bounds__(kThreads) k_chunk_scatter(const __grid_constant__ RasterArgs a, int list) {
    constexpr int NB = ADOP_MAX_VIEWS_PER_LAUNCH + 1;
    __shared__ unsigned start[NB], h[NB], base[NB];
    unsigned *cnt = a.ccount + list * 64;
    if (threadIdx.x == 0) {
        unsigned s0 = 0;
        for (int b = 0; b < NB; ++b) {
            start[b] = s0;
            s0 += cnt[b];
        }
    }
    unsigned long long c0, c1;
    list_chunks(a, list, c0, c1);
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long r0 = c0 + (unsigned long long)blockIdx.x * blockDim.x; r0 < c1; r0 += stride) {
        if (threadIdx.x < NB) h[threadIdx.x] = 0u;
        __syncthreads();
        const unsigned long long c = r0 + threadIdx.x;
        int bk = -1;
        unsigned rank = 0u;
        if (c < c1) {
            bk = chunk_bucket(a, c);
            rank = atomicAdd(&h[bk], 1u);
        }
        __syncthreads();
        if (threadIdx.x < NB && h[threadIdx.x]) base[threadIdx.x] = atomicAdd(&cnt[32 + threadIdx.x], h[threadIdx.x]);
        __syncthreads();
        if (bk >= 0) a.corder[list][start[bk] + base[bk] + rank] = (uint32_t)c;
        __syncthreads();
    }
}

// Visit the slots of a multi-view list in view-major chunk order: warp w takes ordered chunks w, w + W, ...
// (so the chunks in flight at any time are a narrow window of the order, mostly one view), lane k of the warp
// takes items k, k + 32, ... of the chunk, STEP slots per item (STEP = 2 for ghost entries: one entry per lane).
template <int STEP, typename F>
__device__ __forceinline__ void for_ordered(const RasterArgs &a, int list, F &&f) {
    unsigned long long c0, c1;
    list_chunks(a, list, c0, c1);
    const unsigned long long nch = c1 - c0;
    const unsigned long long W = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (unsigned long long j = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < nch; j += W) {
        const unsigned long long base = (unsigned long long)a.corder[list][j] * kListChunk;
        ADOP_CHECK(base + kListChunk <= (unsigned long long)a.rec_capacity);
#pragma unroll
        for (int k = 0; k < kListChunk / (32 * STEP); ++k) f(base + (unsigned long long)STEP * (k * 32 + lane));
    }
}

template <bool VEC4>
__device__ __forceinline__ void blend_record(const RasterArgs &a, unsigned long long r) {
    ADOP_CHECK(r < (unsigned long long)a.rec_capacity);
    const uint4 rec = __ldcs(reinterpret_cast<const uint4 *>(a.records) + r);
    if (rec.w == kDeadView) return;
    ADOP_CHECK(rec.w < (uint32_t)a.nviews && rec.x < (uint32_t)a.v[rec.w].pixels && rec.z < (uint64_t)a.n);
    const ViewDesc &v = a.v[rec.w];
    const uint64_t key = __ldcg(reinterpret_cast<const unsigned long long *>(v.keys) + rec.x);
    if (fuzzy_pass(__uint_as_float(rec.y), key, a.onepa)) accumulate_feature<VEC4>(a, v, rec.z, rec.x);
}

// The record list's overflow fallback out of line: its registers do not weigh on the record path's allocation.
template <int MODEL, bool VEC, bool VEC4>
__device__ __noinline__ void blend_overflow(const RasterArgs &a) {
    stream_sweep<MODEL, VEC, MODE_BLEND, VEC4>(a);
}

template <int MODEL, bool VEC, bool VEC4, bool HOCC>
__global__ void __launch_bounds__(kThreads, HOCC ? 6 : 1) k_blend(const __grid_constant__ RasterArgs a) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && !*(volatile int32_t *)&a.hdr->ghosts_fwd) {
        // a split depth pass's candidate list is consumed: drop it (a ghost list of the depth pass stays)
        a.hdr->back_ok = 0ull;
        a.hdr->resv = *(volatile unsigned long long *)&a.hdr->front_ok;
    }
    if (*(volatile int32_t *)&a.hdr->overflow) {  // record list overflowed: re-stream every point instead
        blend_overflow<MODEL, VEC, VEC4>(a);
        return;
    }
    if (a.mv_lists) {  // multi-view: the survivor chunks view by view (keys and accumulators stay in L2)
        for_ordered<1>(a, 0, [&](unsigned long long r) { blend_record<VEC4>(a, r); });
        return;
    }
    const unsigned long long total = *(volatile unsigned long long *)&a.hdr->front_ok;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long r = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; r < total; r += stride)
        blend_record<VEC4>(a, r);
}

// Environment-map background of channels c0..c0+3 at layer-l pixel j (NEXT-2, R29).
__device__ __forceinline__ void env_bg4(const RasterArgs &a, const ViewDesc &v, int l, int j, int c0, float out[4]) {
    int idx[4];
    float w[4];
    env_taps(a, v, l, j % v.wl[l], j / v.wl[l], idx, w);
    const int C = a.channels;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        float e = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) e = fmaf(w[k], __ldg(a.env + (int64_t)idx[k] * C + c0 + cc), e);
        out[cc] = e;
    }
}

// --------------------------------------------------------------------------- //
// resolve: Eq. 7 (mean or background), planar per-layer output
// --------------------------------------------------------------------------- //
// Groups of 4 consecutive pixels of one layer (host guarantees off_l and h_l*w_l are multiples of 4
// when VEC4): one 16-B count load, accum read only for covered pixels, one 16-B store per channel plane.
// ENV: empty pixels sample the environment map (NEXT-2); a separate instance keeps the plain path lean.
#ifndef ADOP_RESOLVE_SPARSE
#define ADOP_RESOLVE_SPARSE 1
#endif
template <bool VEC4, bool ENV>
__global__ void __launch_bounds__(kThreads) k_resolve(const __grid_constant__ RasterArgs a) {
    const ViewDesc &v = a.v[blockIdx.y];
    const int C = a.channels;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (VEC4) {
        // Multi-view launches: the views' accumulators do not stay in L2 after the blend (configs[1]: 4 x 55 MB), so
        // a pixel's accumulator is read only if its count is non-zero -- an empty pixel's 32-B sector is never
        // fetched (configs[1]: ~6% of the pixels are covered).  One view: loaded with the counts (L2 hits).
        const bool sparse = a.nviews > 1 && ADOP_RESOLVE_SPARSE;
        const int64_t g0 = a.res_p0 / 4, g1 = (a.res_p1 < v.pixels ? a.res_p1 : v.pixels) / 4;  // (range: multiples of 4)
        for (int64_t g = g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < g1; g += stride) {
            const int64_t p = 4 * g;
            int l = 0;
#pragma unroll
            for (int k = 1; k < ADOP_MAX_LAYERS; ++k)
                if (k < a.layers && p >= v.off[k]) l = k;
            const int64_t j = p - v.off[l];
            const int64_t hw = (int64_t)v.wl[l] * v.hl[l];
            const float4 cnt = __ldcs(reinterpret_cast<const float4 *>(v.count + p));
            const float cn[4] = {cnt.x, cnt.y, cnt.z, cnt.w};
            float *img = v.image + (int64_t)C * v.off[l] + j;
            for (int c0 = 0; c0 < C; c0 += 4) {
                float o[4][4];  // [channel][pixel]
#pragma unroll
                float4 acc[4];  // loaded with the counts (L2-resident after the blend): one round trip
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    acc[q] = (!sparse || cn[q] > 0.0f) ? __ldcs(reinterpret_cast<const float4 *>(v.accum + (p + q) * C + c0))
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float av[4] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w};
                    float bgv[4] = {a.bg[c0], a.bg[c0 + 1], a.bg[c0 + 2], a.bg[c0 + 3]};
                    if (ENV && !(cn[q] > 0.0f)) env_bg4(a, v, l, (int)(j + q), c0, bgv);
                    const float inv = __frcp_rn(cn[q]);  // Eq. 7 mean as sum x (1/n): within 1 ulp of the quotient
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) o[cc][q] = cn[q] > 0.0f ? __fmul_rn(av[cc], inv) : bgv[cc];
                }
#pragma unroll
                for (int cc = 0; cc < 4; ++cc)
                    __stcs(reinterpret_cast<float4 *>(img + (c0 + cc) * hw), make_float4(o[cc][0], o[cc][1], o[cc][2], o[cc][3]));
            }
        }
        return;
    }
    const int64_t p1 = a.res_p1 < v.pixels ? a.res_p1 : v.pixels;
    for (int64_t p = a.res_p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p1; p += stride) {
        int l = 0;
#pragma unroll
        for (int k = 1; k < ADOP_MAX_LAYERS; ++k)
            if (k < a.layers && p >= v.off[k]) l = k;
        const int64_t j = p - v.off[l];
        const int64_t hw = (int64_t)v.wl[l] * v.hl[l];
        const float cnt = __ldcs(v.count + p);
        float *img = v.image + (int64_t)C * v.off[l] + j;
        const float *acc = v.accum + p * C;
        if (ENV && !(cnt > 0.0f)) {  // Eq. 7 first case: E(R^T C^-1(u, v)) (NEXT-2)
            int idx[4];
            float w[4];
            env_taps(a, v, l, (int)(j % v.wl[l]), (int)(j / v.wl[l]), idx, w);
            for (int c = 0; c < C; ++c) {
                float e = 0.f;
                for (int k = 0; k < 4; ++k) e = fmaf(w[k], __ldg(a.env + (int64_t)idx[k] * C + c), e);
                __stcs(img + c * hw, e);
            }
            continue;
        }
        const float inv = __frcp_rn(cnt);  // as the vector path: sum x (1/n), so any pixel range resolves identically
        for (int c = 0; c < C; ++c) __stcs(img + c * hw, cnt > 0.0f ? __fmul_rn(acc[c], inv) : a.bg[c]);
    }
}

// --------------------------------------------------------------------------- //
// backward
// --------------------------------------------------------------------------- //
// Image-space gradient contribution of one neighbour q (Eq. 11 as R14, times G as R16), planar reads
// (fallback sweep for unaligned inputs).
template <int CT>
__device__ __forceinline__ float neighbour_term(const RasterArgs &a, const ViewDesc &v, int l, int qu, int qv,
                                                float z, const float *tau) {
    if (qu < 0 || qv < 0 || qu >= v.wl[l] || qv >= v.hl[l]) return 0.0f;  // outside: no term
    const int j = qv * v.wl[l] + qu;
    const int q = v.off[l] + j;
    const float nq = v.count[q];
    float factor;
    if (nq == 0.0f) {
        factor = 1.0f;                                     // case 1: background neighbour
    } else {
        const float m = __uint_as_float((uint32_t)(v.keys[q] >> 32));
        if (z > fmul(a.onepa, m)) return 0.0f;             // case 2: behind
        factor = fmul(z, a.onepa) < m ? 1.0f : __frcp_rn(nq + 1.0f);  // case 3 / case 4
    }
    const int C = CT > 0 ? CT : a.channels;
    const int64_t hw = (int64_t)v.wl[l] * v.hl[l];
    const float *G = v.grad + (int64_t)C * v.off[l] + j;
    const float *I = v.image + (int64_t)C * v.off[l] + j;
    float d = 0.0f;
#pragma unroll
    for (int c = 0; c < (CT > 0 ? CT : ADOP_MAX_CHANNELS); ++c) {
        if (CT == 0 && c >= C) break;
        d = fmaf(__ldg(G + c * hw), tau[c] - __ldg(I + c * hw), d);
    }
    return factor * d;
}

// Backward pixel table of one view (workspace scratch), built once per call: one row of a.prow floats per
// pixel, {bits(m_p), count_p, S_p, 0, G_0(p) .. G_{C-1}(p)}, m_p = the pixel's min depth (key >> 32),
// S_p = sum_c G_c(p) I_c(p) with I exactly as k_resolve computes it (accum/count, or the background).
// A gather of one neighbour (Eq. 11) or texture hit then touches ONE row -- one 32-B sector at C = 4 --
// and Delta . G = factor (tau . G - S).
__global__ void __launch_bounds__(kThreads) k_bwd_prep(const __grid_constant__ RasterArgs a) {
    const ViewDesc &v = a.v[blockIdx.y];
    if (blockIdx.x == 0 && threadIdx.x < 5) {  // this view's frustum planes for the sweep's tile_views
        const int k = threadIdx.x;
        a.planes[blockIdx.y].pl[k] = make_float4(v.pl[k][0], v.pl[k][1], v.pl[k][2], v.pl[k][3]);
        a.planes[blockIdx.y].pm[k] = make_float2(v.pm[k][0], v.pm[k][1]);
    }
    const int C = a.channels, RS = a.prow;
    float *rows = const_cast<float *>(v.prow);
    const bool v4 = (C & 3) == 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < v.pixels; p += stride) {
        int l = 0;
#pragma unroll
        for (int k = 1; k < ADOP_MAX_LAYERS; ++k)
            if (k < a.layers && p >= v.off[k]) l = k;
        const int64_t j = p - v.off[l];
        const int64_t hw = (int64_t)v.wl[l] * v.hl[l];
        const float *G = v.grad + (int64_t)C * v.off[l] + j;
        float *row = rows + p * RS;
        const float cnt = __ldcs(v.count + p);
        const unsigned long long key = __ldcs(reinterpret_cast<const unsigned long long *>(v.keys) + p);
        const float *Iv = v.image + (int64_t)C * v.off[l] + j;  // I exactly as k_resolve wrote it
        float S = 0.0f;
        if (v4) {  // 16-B row writes (C % 4 == 0)
            for (int c = 0; c < C; c += 4) {
                const float4 g = make_float4(__ldcs(G + c * hw), __ldcs(G + (c + 1) * hw), __ldcs(G + (c + 2) * hw),
                                             __ldcs(G + (c + 3) * hw));
                S = fmaf(g.x, __ldcs(Iv + c * hw), S);
                S = fmaf(g.y, __ldcs(Iv + (c + 1) * hw), S);
                S = fmaf(g.z, __ldcs(Iv + (c + 2) * hw), S);
                S = fmaf(g.w, __ldcs(Iv + (c + 3) * hw), S);
                __stcg(reinterpret_cast<float4 *>(row + 4 + c), g);
            }
        } else {
            for (int c = 0; c < C; ++c) {
                const float g = __ldcs(G + c * hw);
                S = fmaf(g, __ldcs(Iv + c * hw), S);
                row[4 + c] = g;
            }
        }
        if (a.d_env && !(cnt > 0.0f)) {  // NEXT-2: dL/dE of the empty pixel's bilinear taps
            int idx[4];
            float w[4];
            env_taps(a, v, l, (int)(j % v.wl[l]), (int)(j / v.wl[l]), idx, w);
            for (int c = 0; c < C; ++c) {
                const float g = row[4 + c];
#pragma unroll
                for (int k = 0; k < 4; ++k) red_add(a.d_env + (int64_t)idx[k] * C + c, w[k] * g);
            }
        }
        __stcg(reinterpret_cast<uint4 *>(row),
               make_uint4((uint32_t)(key >> 32), __float_as_uint(cnt), __float_as_uint(S), 0u));
    }
}

// R35 equidistant fisheye: g = theta / rho (u0 = fx g X + cx), and A = dg/dX / X = dg/dY / Y.  For
// t = rho / Z < 0.3 A uses the series of (t - (1 + t^2) atan t) / t^3 (the direct form cancels in fp32).
__device__ __forceinline__ void fisheye_gA(const Proj &p, float &g, float &A) {
    const float X = p.X, Y = p.Y, Z = p.Z;
    const float rho2 = X * X + Y * Y, rho = sqrtf(rho2), d2 = rho2 + Z * Z;
    const float th = atan2f(rho, Z);
    g = rho > 0.f ? th / rho : 1.f / Z;
    if (Z > 0.f && rho < 0.3f * Z) {
        const float t2 = rho2 / (Z * Z);
        const float h = -2.f / 3.f + t2 * (2.f / 15.f + t2 * (-2.f / 35.f + t2 * (2.f / 63.f)));
        A = h / (Z * d2);
    } else {
        A = (Z * rho - th * d2) / (rho2 * rho * d2);
    }
}

template <int MODEL>
__device__ __forceinline__ void jacobian(const ViewDesc &v, const Proj &p, float J[6]) {
    if (MODEL == 2) {
        float g, A;
        fisheye_gA(p, g, A);
        const float X = p.X, Y = p.Y, d2 = X * X + Y * Y + p.Z * p.Z;
        J[0] = v.fx * (g + X * X * A); J[1] = v.fx * X * Y * A; J[2] = -v.fx * X / d2;
        J[3] = v.fy * X * Y * A; J[4] = v.fy * (g + Y * Y * A); J[5] = -v.fy * Y / d2;
        return;
    }
    const float iz = p.iz, xn = p.X * iz, yn = p.Y * iz;
    // dn/dXc = [[iz, 0, -xn iz], [0, iz, -yn iz]]
    float D00 = 1.f, D01 = 0.f, D10 = 0.f, D11 = 1.f;
    if (MODEL == 1) {
        const float r2 = xn * xn + yn * yn;
        const float num = 1.f + r2 * (v.k[0] + r2 * (v.k[1] + r2 * v.k[2]));
        const float den = 1.f + r2 * (v.k[3] + r2 * (v.k[4] + r2 * v.k[5]));
        const float dnum = v.k[0] + r2 * (2.f * v.k[1] + 3.f * r2 * v.k[2]);
        const float dden = v.k[3] + r2 * (2.f * v.k[4] + 3.f * r2 * v.k[5]);
        const float rad = num / den;
        const float drad = (dnum * den - num * dden) / (den * den);
        const float p1 = v.p[0], p2 = v.p[1];
        D00 = rad + 2.f * xn * xn * drad + 2.f * p1 * yn + 6.f * p2 * xn;
        D01 = 2.f * xn * yn * drad + 2.f * p1 * xn + 2.f * p2 * yn;
        D10 = D01;
        D11 = rad + 2.f * yn * yn * drad + 6.f * p1 * yn + 2.f * p2 * xn;
    }
    const float a0 = v.fx * iz, a1 = v.fy * iz;
    // J = diag(f) D N, N = [[1, 0, -xn], [0, 1, -yn]] * iz
    J[0] = a0 * D00; J[1] = a0 * D01; J[2] = -a0 * (D00 * xn + D01 * yn);
    J[3] = a1 * D10; J[4] = a1 * D11; J[5] = -a1 * (D10 * xn + D11 * yn);
}

// w = J^T g = dL/dXc (R21).  The distortion model's Jacobian is evaluated in fp64: near the edge of the
// camera's valid radius (R6) the radial derivative rad + 2 r^2 drad/dr^2 nearly cancels, and an fp32 J there
// errs by ~eps |rad| instead of ~eps |J| (measured on configs[4]: d_pos 2.4x over the R20 tolerance).
template <int MODEL>
__device__ __forceinline__ void chain_w(const ViewDesc &v, const Proj &p, float gu, float gv, double w[3]) {
    if (MODEL != 1) {
        float J[6];
        jacobian<MODEL>(v, p, J);
        w[0] = (double)(J[0] * gu + J[3] * gv);
        w[1] = (double)(J[1] * gu + J[4] * gv);
        w[2] = (double)(J[2] * gu + J[5] * gv);
        return;
    }
    const double iz = 1.0 / (double)p.Z, xn = (double)p.X * iz, yn = (double)p.Y * iz;
    const double r2 = xn * xn + yn * yn;
    const double k0 = v.k[0], k1 = v.k[1], k2 = v.k[2], k3 = v.k[3], k4 = v.k[4], k5 = v.k[5];
    const double num = 1.0 + r2 * (k0 + r2 * (k1 + r2 * k2));
    const double den = 1.0 + r2 * (k3 + r2 * (k4 + r2 * k5));
    const double dnum = k0 + r2 * (2.0 * k1 + 3.0 * r2 * k2);
    const double dden = k3 + r2 * (2.0 * k4 + 3.0 * r2 * k5);
    const double rad = num / den;
    const double drad = (dnum * den - num * dden) / (den * den);
    const double p1 = v.p[0], p2 = v.p[1];
    const double D00 = rad + 2.0 * xn * xn * drad + 2.0 * p1 * yn + 6.0 * p2 * xn;
    const double D01 = 2.0 * xn * yn * drad + 2.0 * p1 * xn + 2.0 * p2 * yn;
    const double D11 = rad + 2.0 * yn * yn * drad + 6.0 * p1 * yn + 2.0 * p2 * xn;
    const double a0 = (double)v.fx * iz * gu, a1 = (double)v.fy * iz * gv;  // g scaled by f / Z
    // J = diag(f) D N, N = [[1, 0, -xn], [0, 1, -yn]] / Z  ->  w = N^T D^T diag(f) g
    const double e0 = D00 * a0 + D01 * a1, e1 = D01 * a0 + D11 * a1;
    w[0] = e0;
    w[1] = e1;
    w[2] = -(e0 * xn + e1 * yn);
}

// Structural terms of one ghost in one view, per view accumulated in fp64 (R20): t[0..6) = the tangent
// pose terms (w, Xc x w) (Eq. 17 left increment, R19); with nt = kNT, t[6..18) = the camera-intrinsics
// terms (d(u0,v0)/d theta)^T g (NEXT-1), theta = (fx, fy, cx, cy, k1..k6, p1, p2), g = (g_u, g_v) in
// layer-0 pixels (R17); the pinhole model has no distortion parameters (those terms are 0).
constexpr int kNI = 12;
constexpr int kNT = 6 + kNI;
template <int MODEL>
__device__ __forceinline__ void struct_terms(const ViewDesc &v, const Proj &p, float gu, float gv, const double *w,
                                             int nt, double *t) {
    t[0] = w[0]; t[1] = w[1]; t[2] = w[2];
    t[3] = (double)p.Y * w[2] - (double)p.Z * w[1];
    t[4] = (double)p.Z * w[0] - (double)p.X * w[2];
    t[5] = (double)p.X * w[1] - (double)p.Y * w[0];
    if (nt <= 6) return;
    float xn = p.X * p.iz, yn = p.Y * p.iz;
    if (MODEL == 2) {  // R35: xd = g X, yd = g Y; no distortion parameters
        float g, A;
        fisheye_gA(p, g, A);
        xn = g * p.X;
        yn = g * p.Y;
    }
    float xd = xn, yd = yn;
#pragma unroll
    for (int k = 4; k < kNI; ++k) t[6 + k] = 0.0;
    if (MODEL == 1) {  // camera model R6: u0 = fx xd + cx, xd = xn rad + 2 p1 xn yn + p2 (r2 + 2 xn^2), ...
        const float r2 = xn * xn + yn * yn, r4 = r2 * r2, r6 = r4 * r2;
        const float num = 1.f + v.k[0] * r2 + v.k[1] * r4 + v.k[2] * r6;
        const float den = 1.f + v.k[3] * r2 + v.k[4] * r4 + v.k[5] * r6;
        const float idn = 1.f / den, rad = num * idn;
        xd = xn * rad + 2.f * v.p[0] * xn * yn + v.p[1] * (r2 + 2.f * xn * xn);
        yd = yn * rad + v.p[0] * (r2 + 2.f * yn * yn) + 2.f * v.p[1] * xn * yn;
        const float a = gu * v.fx, b = gv * v.fy, s = a * xn + b * yn;  // g . d(u0,v0)/d rad
        const float q = -s * num * idn * idn;
        t[10] = (double)(s * r2 * idn); t[11] = (double)(s * r4 * idn); t[12] = (double)(s * r6 * idn);  // k1..k3
        t[13] = (double)(q * r2); t[14] = (double)(q * r4); t[15] = (double)(q * r6);                   // k4..k6
        t[16] = (double)(a * 2.f * xn * yn + b * (r2 + 2.f * yn * yn));                                 // p1
        t[17] = (double)(a * (r2 + 2.f * xn * xn) + b * 2.f * xn * yn);                                 // p2
    }
    t[6] = (double)(gu * xd);  // fx
    t[7] = (double)(gv * yd);  // fy
    t[8] = gu;                 // cx
    t[9] = gv;                 // cy
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    return x;
}

template <int MODEL, bool VEC, int CT>
__global__ void __launch_bounds__(kThreads) k_backward(const __grid_constant__ RasterArgs a) {
    __shared__ double spose[ADOP_MAX_VIEWS_PER_LAUNCH * kNT];
    const int NT = a.nterms;
    for (int t = threadIdx.x; t < a.nviews * NT; t += blockDim.x) spose[t] = 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int C = CT > 0 ? CT : a.channels;
    constexpr int CR = CT > 0 ? CT : 1;  // register accumulators (generic C works in global memory)
    const int64_t nchunks = (a.n + 127) / 128;
    for (int64_t ch = (int64_t)blockIdx.x * kWarps + wid; ch < nchunks; ch += (int64_t)gridDim.x * kWarps) {
        const int64_t i0 = ch * 128 + lane * 4;
        float px[4], py[4], pz[4], pr[4];
        load_points<VEC>(a, i0, px, py, pz, pr);
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
            const int64_t i = i0 + j;
            const bool in = i < a.n;
            const uint32_t gi = a.goff + (uint32_t)i;
            const bool ghost = in && a.ghost_thr != 0u && h24(a.ghost_salt, gi) < a.ghost_thr;
            float dt[CR];
#pragma unroll
            for (int c = 0; c < CR; ++c) dt[c] = 0.0f;
            if (CT == 0 && in && a.d_feat && !a.grad_accumulate)
                for (int c = 0; c < C; ++c) a.d_feat[i * C + c] = 0.0f;
            float dxx = 0.f, dxy = 0.f, dxz = 0.f;
            float tau[CT > 0 ? CT : ADOP_MAX_CHANNELS];
            bool tau_loaded = false;
            for (int vs = 0; vs < a.nviews; ++vs) {
                const ViewDesc &v = a.v[vs];
                Proj p;
                const bool ok = in && project_point<MODEL>(v, a.z_near, px[j], py[j], pz[j], p) &&
                                normal_keep(a, v, i, p.X, p.Y, p.Z);
                if (!__any_sync(kFull, ok)) continue;
                const int nk = ok ? keep_layers(a, v, pr[j], p.iz, gi) : 0;
                float gu = 0.f, gv = 0.f;
                bool gc = false;
                for (int l = 0; l < a.layers; ++l) {
                    if (l >= nk) break;
                    int pu, pv;
                    const int loc = layer_pixel(v, p, l, pu, pv);
                    if (loc < 0) continue;
                    if (!ghost) {
                        // texture gradient: dI/dtau = 1/|Lambda| for members of Lambda (R24)
                        const int q = v.off[l] + loc;
                        const float cnt = v.count[q];
                        if (fuzzy_pass(p.D, v.keys[q], a.onepa)) {
                        const int64_t hw = (int64_t)v.wl[l] * v.hl[l];
                        const float *G = v.grad + (int64_t)C * v.off[l] + loc;
                        if (CT > 0) {
#pragma unroll
                            for (int c = 0; c < CR; ++c)
                                dt[c] += __fdiv_rn(__ldg(G + c * hw), cnt) * (a.log_desc ? expf(__ldg(a.feat + i * C + c)) : 1.0f);
                        } else if (a.d_feat) {
                            for (int c = 0; c < C; ++c)
                                a.d_feat[i * C + c] += __fdiv_rn(__ldg(G + c * hw), cnt) *
                                                       (a.log_desc ? expf(__ldg(a.feat + i * C + c)) : 1.0f);
                        }
                        }
                    }
                    if (a.spatial_rendered ? !ghost : ghost) {  // spatial gradient (R22 / R31)
                        if (!tau_loaded) {
                            for (int c = 0; c < C; ++c) tau[c] = desc_lin(a, __ldg(a.feat + i * C + c));
                            tau_loaded = true;
                        }
                        // Eqs. 9-11: signed central differences over the 4-neighbourhood (R14, R15)
                        const float dup = neighbour_term<CT>(a, v, l, pu + 1, pv, p.D, tau);
                        const float dum = neighbour_term<CT>(a, v, l, pu - 1, pv, p.D, tau);
                        const float dvp = neighbour_term<CT>(a, v, l, pu, pv + 1, p.D, tau);
                        const float dvm = neighbour_term<CT>(a, v, l, pu, pv - 1, p.D, tau);
                        const float s = 0.5f * pow2_neg(l);  // layer-l pixels -> layer-0 pixels (R17)
                        gu += s * (dup - dum);
                        gv += s * (dvp - dvm);
                        gc = true;
                    }
                }
                if (!__any_sync(kFull, gc)) continue;
                double tt[kNT];
#pragma unroll
                for (int k = 0; k < kNT; ++k) tt[k] = 0.0;
                if (gc) {
                    double w[3];
                    chain_w<MODEL>(v, p, gu, gv, w);  // w = J^T g = dL/dXc
                    dxx += (float)(v.R[0] * w[0] + v.R[3] * w[1] + v.R[6] * w[2]);  // dx = R^T w
                    dxy += (float)(v.R[1] * w[0] + v.R[4] * w[1] + v.R[7] * w[2]);
                    dxz += (float)(v.R[2] * w[0] + v.R[5] * w[1] + v.R[8] * w[2]);
                    struct_terms<MODEL>(v, p, gu, gv, w, NT, tt);
                }
                // pose (+ intrinsics) terms: warp sum in fp64
                for (int k = 0; k < NT; ++k) {
                    const double s = warp_sum(tt[k]);
                    if (lane == 0) atomicAdd(&spose[vs * NT + k], s);
                }
            }
            if (in) {
                if (CT > 0 && a.d_feat) {
                    float *df = a.d_feat + i * C;
#pragma unroll
                    for (int c = 0; c < CR; ++c) df[c] = a.grad_accumulate ? df[c] + dt[c] : dt[c];
                }
                if (a.d_pos) {
                    float *dp = a.d_pos;
                    if (a.grad_accumulate) {
                        if (dxx != 0.f || dxy != 0.f || dxz != 0.f) {
                            dp[i] += dxx; dp[a.n + i] += dxy; dp[2 * a.n + i] += dxz;
                        }
                    } else {
                        dp[i] = dxx; dp[a.n + i] = dxy; dp[2 * a.n + i] = dxz;
                    }
                }
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.nviews * NT; t += blockDim.x)
        a.pose_partials[(int64_t)blockIdx.x * a.nviews * NT + t] = spose[t];
}

// --------------------------------------------------------------------------- //
// backward, TMA-pipelined (same tiling as k_depth_async)
//
// Overwrite mode first zero-fills d_feat / d_pos (k_fill, write bandwidth); the sweep then only
// touches points that are rendered or ghosts at some layer of some view: per tile and view the
// lane-box cull, the branch-free FMA pre-cull + early discard mask, then one candidate per lane per
// iteration: exact projection and discard (bit-identical to the forward), the texture gradient of
// rendered points (fuzzy membership against the forward's keys, G / |Lambda|, R24) and, for ghosts,
// the 4-neighbour Eq. 11 terms (R14-R16) -> g (R17) -> w = J^T g (R21) -> dx = R^T w and the tangent
// pose terms (w, Xc x w) (R19), warp-reduced in fp64.  Each point belongs to one lane, so its gradient
// rows are updated with plain read-modify-writes (no atomics).
// --------------------------------------------------------------------------- //
// Thread 0 also picks the backward's mode: the depth pass's survivor records are exactly the re-render's
// rendered hits when they were written by a call with the same inputs (tag) and did not
// overflow -> the texture gradient consumes them and the sweep only collects ghosts (mode 1); otherwise
// the sweep re-renders every point into fresh lists (mode 0).  Either way the ghost list starts empty.
__global__ void __launch_bounds__(kThreads) k_fill(float *p, int64_t n, float *q, int64_t m, float *r, int64_t rn,
                                                   WsHeader *hdr,
                                                   double *inline_row, int inline_len, unsigned long long tag,
                                                   int fwd_ghosts_ok) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid == 0 && hdr) {
        const bool reuse = tag != 0ull && hdr->tag == tag && hdr->overflow == 0;
        // mode 2: the depth pass also listed every ghost (and nothing has replaced its list since): no sweep
        const bool ghosts = reuse && fwd_ghosts_ok && hdr->ghosts_fwd == 1;
        hdr->mode = ghosts ? 2 : (reuse ? 1 : 0);
        if (!ghosts) {
            if (reuse) {  // keep the survivor records, drop the ghost list (an earlier backward's or the depth pass's)
                hdr->resv = hdr->front_ok;
            } else {      // the sweep's lists overwrite the record region
                hdr->tag = 0ull;
                hdr->resv = 0ull;
                hdr->front_ok = 0ull;
                hdr->overflow = 0;
            }
            hdr->back_ok = 0ull;
            hdr->ghosts_fwd = 0;
        }
        hdr->tiles_bwd = 0ull;
    }
    if (inline_row && tid < inline_len) inline_row[tid] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float *bufs[3] = {p, q, r};
    const int64_t lens[3] = {n, m, rn};
    for (int b = 0; b < 3; ++b) {
        float *x = bufs[b];
        const int64_t len = lens[b];
        if (!x) continue;
        const int64_t head = (int64_t)(((16 - (reinterpret_cast<uintptr_t>(x) & 15)) & 15) / 4);
        const int64_t h = head < len ? head : len;
        for (int64_t k = tid; k < h; k += stride) x[k] = 0.0f;
        float4 *x4 = reinterpret_cast<float4 *>(x + h);
        const int64_t n4 = (len - h) / 4;
        for (int64_t k = tid; k < n4; k += stride) x4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t k = h + 4 * n4 + tid; k < len; k += stride) x[k] = 0.0f;
    }
}

template <int CT>
__device__ __forceinline__ float row_dot(const float *row, const float *tau, int C) {
    float d = 0.0f;
    if (CT > 0 && CT % 4 == 0) {
#pragma unroll
        for (int c = 0; c < CT; c += 4) {
            const float4 g = __ldcg(reinterpret_cast<const float4 *>(row + c));
            d = fmaf(g.x, tau[c], d);
            d = fmaf(g.y, tau[c + 1], d);
            d = fmaf(g.z, tau[c + 2], d);
            d = fmaf(g.w, tau[c + 3], d);
        }
    } else {
        for (int c = 0; c < C; ++c) d = fmaf(__ldcg(row + c), tau[c], d);
    }
    return d;
}

// Ghost image-space gradient at one layer (Eqs. 9-11, R14-R16) from the pixel tables: the four
// neighbours' table entries are loaded together, then their G rows.
template <int CT>
__device__ __forceinline__ void ghost_layer(const RasterArgs &a, const ViewDesc &v, int l, int pu, int pv, float z,
                                           const float *tau, float &gu, float &gv) {
    const int C = CT > 0 ? CT : a.channels;
    const int du[4] = {1, -1, 0, 0}, dv[4] = {0, 0, 1, -1};
    int q[4];
    uint4 e[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int qu = pu + du[k], qv = pv + dv[k];
        const bool in = qu >= 0 && qv >= 0 && qu < v.wl[l] && qv < v.hl[l];
        q[k] = in ? v.off[l] + qv * v.wl[l] + qu : -1;
        e[k] = in ? __ldcg(reinterpret_cast<const uint4 *>(v.prow + (int64_t)q[k] * a.prow)) : make_uint4(0u, 0u, 0u, 0u);
    }
    float d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        d[k] = 0.0f;
        if (q[k] < 0) continue;  // outside: no term
        const float nq = __uint_as_float(e[k].y);
        float factor;
        if (nq == 0.0f) {
            factor = 1.0f;                                            // case 1: background
        } else {
            const float m = __uint_as_float(e[k].x);
            if (z > fmul(a.onepa, m)) continue;                       // case 2: behind
            factor = fmul(z, a.onepa) < m ? 1.0f : __frcp_rn(nq + 1.0f);  // case 3 / case 4
        }
        ADOP_CHECK(q[k] < v.pixels);
        d[k] = factor * (row_dot<CT>(v.prow + (int64_t)q[k] * a.prow + 4, tau, C) - __uint_as_float(e[k].z));
    }
    const float sc = 0.5f * pow2_neg(l);  // layer-l pixels -> layer-0 pixels (R17)
    gu += sc * (d[0] - d[1]);
    gv += sc * (d[2] - d[3]);
}

// ---- record-driven backward: work lists in the record region, two balanced kernels consume them ----
// Texture list = the front list (Record layout): the depth pass's survivor records (mode 1) or the
// sweep's rendered hits (mode 0).  Ghost list = the back list (GhostEntry layout), written by the sweep.
__device__ __forceinline__ void red_add_row(float *dst, const float *src, int C, float scale) {
    if ((C & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        for (int c = 0; c < C; c += 4) {
            const float4 g = __ldcg(reinterpret_cast<const float4 *>(src + c));
            red_add_v4(dst + c, make_float4(__fdiv_rn(g.x, scale), __fdiv_rn(g.y, scale), __fdiv_rn(g.z, scale),
                                            __fdiv_rn(g.w, scale)));
        }
    } else {
        for (int c = 0; c < C; ++c) red_add(dst + c, __fdiv_rn(__ldcg(src + c), scale));
    }
}

// texture gradient of one rendered hit (R24): fuzzy membership against the forward's key, G / |Lambda|
__device__ __forceinline__ void tex_hit(const RasterArgs &a, const ViewDesc &v, uint32_t q, float z, int64_t idx) {
    ADOP_CHECK(q < (uint32_t)v.pixels && idx >= 0 && idx < a.n);
    const float *row = v.prow + (int64_t)q * a.prow;
    const uint4 e = __ldcg(reinterpret_cast<const uint4 *>(row));
    if (!(z <= fmul(a.onepa, __uint_as_float(e.x)))) return;  // fuzzy test (Eq. 6, R9)
    const int C = a.channels;
    if (a.log_desc) {  // d exp(tau)/d tau = exp(tau) (NEXT-2)
        for (int c = 0; c < C; ++c)
            red_add(a.d_feat + idx * C + c, __fdiv_rn(__ldcg(row + 4 + c), __uint_as_float(e.y)) * expf(__ldg(a.feat + idx * C + c)));
        return;
    }
    red_add_row(a.d_feat + idx * C, row + 4, C, __uint_as_float(e.y));
}

// ghost: image gradient over its kept layers (Eqs. 9-11), chain rule (Eq. 8) -> dx (atomics), and the
// nt structural terms (struct_terms) returned for the caller's reduction.
template <int MODEL, int CT>
__device__ __forceinline__ bool ghost_point(const RasterArgs &a, const ViewDesc &v, const Proj &p, int nk,
                                            int64_t idx, int nt, double *tt, float *g = nullptr) {
    const int C = CT > 0 ? CT : a.channels;
    float tau[CT > 0 ? CT : ADOP_MAX_CHANNELS];
    for (int c = 0; c < C; ++c) tau[c] = desc_lin(a, __ldg(a.feat + idx * C + c));  // linear space
    float gu = 0.f, gv = 0.f;
    bool gc = false;
    for (int l = 0; l < nk; ++l) {
        int pu, pv;
        if (layer_pixel(v, p, l, pu, pv) < 0) continue;
        ghost_layer<CT>(a, v, l, pu, pv, p.D, tau, gu, gv);
        gc = true;
    }
    if (!gc) return false;
    double w[3];
    chain_w<MODEL>(v, p, gu, gv, w);  // w = J^T g = dL/dXc
    if (a.d_pos) {
        red_add(a.d_pos + idx, (float)(v.R[0] * w[0] + v.R[3] * w[1] + v.R[6] * w[2]));  // dx = R^T w
        red_add(a.d_pos + a.n + idx, (float)(v.R[1] * w[0] + v.R[4] * w[1] + v.R[7] * w[2]));
        red_add(a.d_pos + 2 * a.n + idx, (float)(v.R[2] * w[0] + v.R[5] * w[1] + v.R[8] * w[2]));
    }
    struct_terms<MODEL>(v, p, gu, gv, w, nt, tt);
    if (g) {
        g[0] = gu;
        g[1] = gv;
    }
    return true;
}

// A ghost whose list slot could not be reserved (record region full) is processed by the sweep itself.
// The pose terms stay inline as before; the intrinsics terms (NEXT-1, only when requested) are added
// out of line so their registers do not weigh on the sweep.
template <int MODEL>
__device__ __forceinline__ void intr_inline(const RasterArgs &a, const ViewDesc &v, int vs, const Proj &p, float gu,
                                            float gv) {
    double *row = a.pose_partials + ((int64_t)a.inline_row * a.nviews + vs) * kNT + 6;
    float xn = p.X * p.iz, yn = p.Y * p.iz;
    if (MODEL == 2) {
        float g, A;
        fisheye_gA(p, g, A);
        xn = g * p.X;
        yn = g * p.Y;
    }
    float xd = xn, yd = yn;
    if (MODEL == 1) {  // as struct_terms, one term at a time (no term array in the sweep's registers)
        const float r2 = xn * xn + yn * yn, r4 = r2 * r2, r6 = r4 * r2;
        const float num = 1.f + v.k[0] * r2 + v.k[1] * r4 + v.k[2] * r6;
        const float den = 1.f + v.k[3] * r2 + v.k[4] * r4 + v.k[5] * r6;
        const float idn = 1.f / den, rad = num * idn;
        xd = xn * rad + 2.f * v.p[0] * xn * yn + v.p[1] * (r2 + 2.f * xn * xn);
        yd = yn * rad + v.p[0] * (r2 + 2.f * yn * yn) + 2.f * v.p[1] * xn * yn;
        const float a0 = gu * v.fx, b0 = gv * v.fy, s = a0 * xn + b0 * yn, q = -s * num * idn * idn;
        atomicAdd(row + 4, (double)(s * r2 * idn));
        atomicAdd(row + 5, (double)(s * r4 * idn));
        atomicAdd(row + 6, (double)(s * r6 * idn));
        atomicAdd(row + 7, (double)(q * r2));
        atomicAdd(row + 8, (double)(q * r4));
        atomicAdd(row + 9, (double)(q * r6));
        atomicAdd(row + 10, (double)(a0 * 2.f * xn * yn + b0 * (r2 + 2.f * yn * yn)));
        atomicAdd(row + 11, (double)(a0 * (r2 + 2.f * xn * xn) + b0 * 2.f * xn * yn));
    }
    atomicAdd(row + 0, (double)(gu * xd));
    atomicAdd(row + 1, (double)(gv * yd));
    atomicAdd(row + 2, (double)gu);
    atomicAdd(row + 3, (double)gv);
}
template <int MODEL, int CT>
__device__ __forceinline__ void ghost_inline(const RasterArgs &a, const ViewDesc &v, int vs, const Proj &p, int nk,
                                             int64_t i) {
    double t6[6];
    float g[2];
    if (!ghost_point<MODEL, CT>(a, v, p, nk, i, 6, t6, g)) return;
    const int NT = a.nterms;
    for (int k = 0; k < 6; ++k) atomicAdd(&a.pose_partials[((int64_t)a.inline_row * a.nviews + vs) * NT + k], t6[k]);
    if (NT == kNT) intr_inline<MODEL>(a, v, vs, p, g[0], g[1]);
}

// Sweep candidate: exact projection and discard, then emit the rendered hits to the texture list (mode 0
// only) and the ghost to the ghost list (inline processing when the region is full).  Warp-collective.
template <int MODEL, int CT, bool MV>
__device__ __forceinline__ void bwd_emit(const RasterArgs &a, const ViewDesc &v, int vs, bool ok, bool ghost, float x,
                                         float y, float z, float rw, int64_t i, uint32_t gi, ListChunk &ct,
                                         ListChunk &cg, bool tex_on, int lane, unsigned lt) {
    Proj p;
    int nk = 0;
    if (ok) {
        to_camera(v, x, y, z, p.X, p.Y, p.Z);
        if (depth_valid<MODEL>(p, a.z_near) && (MODEL != 1 || !v.wn_on || in_window(v, p.X, p.Y, p.Z)) &&
            normal_keep(a, v, i, p.X, p.Y, p.Z)) {
            nk = keep_layers(a, v, rw, p.iz, gi);
            if (nk > 0 && !(project_uv<MODEL>(v, p) && any_layer_in_bounds(v, p, nk))) nk = 0;  // R14: no term
        }
    }
    const bool rend = tex_on && nk > 0 && !ghost && a.d_feat;
    if (__any_sync(kFull, rend)) {
#pragma unroll 1
        for (int l = 0; l < a.layers; ++l) {
            int pu, pv;
            const int loc = (rend && l < nk) ? layer_pixel(v, p, l, pu, pv) : -1;
            const bool hit = loc >= 0;
            const unsigned b = __ballot_sync(kFull, hit);
            if (b == 0u) {
                if (!__any_sync(kFull, rend && l + 1 < nk)) break;
                continue;
            }
            const uint32_t q = (uint32_t)(v.off[l] + loc);
            const unsigned long long slot = list_take<false>(a, ct, b, hit, lane, lt);
            if (hit) {
                if (slot != kNoSlot)
                    reinterpret_cast<uint4 *>(a.records)[slot] =
                        make_uint4(q, __float_as_uint(p.D), (uint32_t)i, (uint32_t)vs);  // Record
                else
                    tex_hit(a, v, q, p.D, i);
            }
        }
    }
    const bool gh = nk > 0 && (a.spatial_rendered ? !ghost : ghost);  // spatial-gradient list (R22 / R31)
    const unsigned bg = __ballot_sync(kFull, gh);
    if (bg == 0u) return;
    const unsigned long long slot = (MV && a.mv_lists) ? mv_take_back(a, cg, bg, gh, vs, lane, lt)
                                                       : list_take<true>(a, cg, bg, gh, lane, lt);
    if (!gh) return;
    if (slot != kNoSlot) {  // GhostEntry
        uint4 *r = reinterpret_cast<uint4 *>(a.records) + slot;
        r[0] = make_uint4(__float_as_uint(p.u0), __float_as_uint(p.v0), __float_as_uint(p.X), __float_as_uint(p.Y));
        r[1] = make_uint4(__float_as_uint(p.Z), (uint32_t)i, (uint32_t)(vs | (nk << 8)), __float_as_uint(p.D));
    } else {
        ghost_inline<MODEL, CT>(a, v, vs, p, nk, i);
    }
}

// texture list consumer: one thread per hit (balanced), vector reductions into d_feat.
__global__ void __launch_bounds__(kThreads) k_bwd_tex(const __grid_constant__ RasterArgs a) {
    const uint4 *list = reinterpret_cast<const uint4 *>(a.records);
    if ((a.mv_lists & 2) && *(volatile int32_t *)&a.hdr->mode >= 1) {  // the forward's per-view chunks, view by view
        for_ordered<1>(a, 0, [&](unsigned long long r) {
            const uint4 e = __ldcs(list + r);
            if (e.w != kDead) tex_hit(a, a.v[e.w], e.x, __uint_as_float(e.y), (int64_t)e.z);
        });
        return;
    }
    const unsigned long long total = *(volatile unsigned long long *)&a.hdr->front_ok;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long r = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; r < total; r += stride) {
        const uint4 e = __ldcs(list + r);
        if (e.w == kDead) continue;
        tex_hit(a, a.v[e.w], e.x, __uint_as_float(e.y), (int64_t)e.z);
    }
}

// ghost list consumer: one thread per (ghost, view) (balanced); pose terms warp-reduced in fp64 into
// per-warp shared slots, per-block partials reduced by k_pose_reduce in a fixed order.
// NT = 6 (pose) or kNT (pose + intrinsics).
template <int MODEL, int CT, int NT>
__global__ void __launch_bounds__(kThreads, 4) k_bwd_ghost(const __grid_constant__ RasterArgs a) {
    __shared__ double wpose[kWarps][ADOP_MAX_VIEWS_PER_LAUNCH * NT];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < kWarps * ADOP_MAX_VIEWS_PER_LAUNCH * NT; t += blockDim.x) (&wpose[0][0])[t] = 0.0;
    __syncthreads();
    // one ghost entry per lane (ent = NULL: none), then the warp's fp64 reduction per distinct view present
    // (usually one: with multi-view lists every chunk holds one view).  Warp-collective.
    auto entry = [&](const uint4 *ent) {
        double t6[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) t6[k] = 0.0;
        int vs = -1;
        if (ent) {
            const uint4 e1 = __ldcs(ent + 1);
            if (e1.z != kDead) {
                const uint4 e0 = __ldcs(ent);
                vs = (int)(e1.z & 0xFF);
                const int nk = (int)(e1.z >> 8);
                ADOP_CHECK(vs < a.nviews && nk >= 1 && nk <= a.layers && e1.y < (uint64_t)a.n);
                const ViewDesc &v = a.v[vs];
                Proj p;
                p.u0 = __uint_as_float(e0.x);
                p.v0 = __uint_as_float(e0.y);
                p.X = __uint_as_float(e0.z);
                p.Y = __uint_as_float(e0.w);
                p.Z = __uint_as_float(e1.x);
                p.D = __uint_as_float(e1.w);  // the depth of Eq. 6 (R4 / R35)
                p.iz = __frcp_rn(p.D);
                if (!ghost_point<MODEL, CT>(a, v, p, nk, (int64_t)e1.y, NT, t6)) vs = -1;
            }
        }
        unsigned pending = __ballot_sync(kFull, vs >= 0);
        while (pending) {
            const int leader = __ffs(pending) - 1;
            const int vv = __shfl_sync(kFull, vs, leader);
            const bool mine = vs == vv;
#pragma unroll
            for (int k = 0; k < NT; ++k) {
                const double sum = warp_sum(mine ? t6[k] : 0.0);
                if (lane == 0) wpose[wid][vv * NT + k] += sum;
            }
            pending &= ~__ballot_sync(kFull, mine);
        }
    };
    const uint4 *rec = reinterpret_cast<const uint4 *>(a.records);
    if (a.mv_lists & 4) {  // the per-view ghost chunks, view by view (one view's pixel tables stay in L2)
        for_ordered<2>(a, 1, [&](unsigned long long slot) { entry(rec + slot); });
    } else {  // the sweep's ghost list: the back of the record region
        const unsigned long long back = *(volatile unsigned long long *)&a.hdr->back_ok;
        const uint4 *list = rec + ((unsigned long long)a.rec_capacity - back);
        const unsigned long long total = back / 2;
        const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
        for (unsigned long long r0 = (unsigned long long)blockIdx.x * blockDim.x; r0 < total; r0 += stride) {
            const unsigned long long r = r0 + threadIdx.x;
            entry(r < total ? list + 2 * r : nullptr);
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.nviews * NT; t += blockDim.x) {
        double acc = 0.0;
        for (int w = 0; w < kWarps; ++w) acc += wpose[w][t];
        a.pose_partials[(int64_t)blockIdx.x * a.nviews * NT + t] = acc;
    }
}

constexpr int kBPool = 2 * kSW;  // backward sweep stage pool
struct BwdSmem {  // CTA-wide pool of kBPool stages, claimed like k_depth_pool's
    float pos[kBPool][4][kWTile];
    uint64_t bar[kBPool];
    int filled[kBPool];
    int next;
    LayerDesc ld[ADOP_MAX_VIEWS_PER_LAUNCH];
    uint8_t gl[kSW][kWTile];  // mode 1: compacted ghost points of the warp tile (tile offsets)
};

static_assert(sizeof(BwdSmem) + 1024 <= 228 * 1024 / 3, "backward sweep: 3 CTAs per SM must fit in shared memory");
static_assert(kBPool >= kSW && kBPool <= 3 * kSW, "the sweeps' initial fills issue at most three stages per warp");

// GO (ghosts only) is launched for mode 1, !GO for mode 0; the instance not matching the mode exits.
template <int MODEL, int CT, bool MV, bool GO>
__global__ void __launch_bounds__(kST, 3) k_bwd_sweep(const __grid_constant__ RasterArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BwdSmem &sm = *reinterpret_cast<BwdSmem *>(smem_raw);
    const int32_t mode = *(volatile int32_t *)&a.hdr->mode;
    if (mode == 2 || (mode == 1) != GO) return;  // mode 2: the depth pass listed the ghosts
    constexpr bool tex_on = !GO;  // mode 1: the survivor records are the texture list
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned lt = lanemask_lt();
    ListChunk ct, cg;
    ct.base = cg.base = 0;
    ct.left = cg.left = 0;
    const long long ntiles = (a.n + kWTile - 1) / kWTile;
    const bool staged_r = a.discard && a.radius != nullptr;
    const int rows = staged_r ? 4 : 3;
    const float *src[4] = {a.x, a.y, a.z, a.radius};
    init_layer_descs(a, sm.ld);
    if (tid < kBPool) {
        mbar_init(&sm.bar[tid], 1);
        sm.filled[tid] = -1;
    }
    if (tid == 0) sm.next = 0;
    fence_mbar_init();
    __syncthreads();
    const long long G = gridDim.x, bk = blockIdx.x;
    auto full_tile = [&](long long t) { return (t + 1) * kWTile <= a.n; };
    auto issue = [&](int k) {  // lane 0: the CTA's k-th tile (k G + b) into stage k mod kBPool
        const long long t = (long long)k * G + bk;
        if (t >= ntiles) return;
        const int st = k % kBPool;
        *(volatile int *)&sm.filled[st] = k;
        if (!full_tile(t)) {  // ragged last tile: its consumer loads it; the arrival only releases the stage
            mbar_arrive_a(smem_addr(&sm.bar[st]));
            return;
        }
        const uint64_t pol = policy_evict_first();
        mbar_expect_tx(&sm.bar[st], (uint32_t)(rows * kWTile * sizeof(float)));
        if (a.use_tmap) {  // x, y, z rows in one 2-D tensor copy, r_world in a 1-D bulk copy
            tensor_g2s_2d(sm.pos[st][0], &a.tmap, (int)(t * kWTile), 0, &sm.bar[st], pol);
            if (rows == 4) bulk_g2s(sm.pos[st][3], src[3] + t * kWTile, kWTile * sizeof(float), &sm.bar[st], pol);
        } else {
            for (int r = 0; r < rows; ++r)
                bulk_g2s(sm.pos[st][r], src[r] + t * kWTile, kWTile * sizeof(float), &sm.bar[st], pol);
        }
    };
    if (lane == 0)
        for (int k0 = wid; k0 < kBPool; k0 += kSW) issue(k0);
    __syncwarp();
    for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(&sm.next, 1);
        k = __shfl_sync(kFull, k, 0);
        const long long t = (long long)k * G + bk;
        if (t >= ntiles) break;
        const int st = k % kBPool;
        const int64_t base = t * kWTile;
        const float *rp[4] = {sm.pos[st][0], sm.pos[st][1], sm.pos[st][2], sm.pos[st][3]};
        while (*(volatile int *)&sm.filled[st] != k) __nanosleep(ADOP_POOL_SLEEP);  // (see k_depth_pool)
        mbar_wait(&sm.bar[st], (uint32_t)(k / kBPool) & 1u);
        int vmask = 0xFF;
        if (!full_tile(t)) {
            vmask = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int e = (j >> 2) * 128 + 4 * lane + (j & 3);
                const bool in = base + e < a.n;
                for (int r = 0; r < 4; ++r) sm.pos[st][r][e] = (in && r < rows) ? src[r][base + e] : 0.f;
                vmask |= (in ? 1 : 0) << j;
            }
            __syncwarp();
        }
        auto pidx = [&](int j) { return base + (j >> 2) * 128 + 4 * lane + (j & 3); };
        uint32_t ghosts = 0u;
        auto hash_ghosts = [&]() {
            if (a.ghost_thr != 0u) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (h24(a.ghost_salt, a.goff + (uint32_t)pidx(j)) < a.ghost_thr) ghosts |= 1u << j;
            }
        };
        if (GO) {
            // mode 1: only ghosts (~rho of the points) are left to find.  The tile's visible views come first (a
            // culled tile costs no hashing); then the ghosts are compacted and only they are pre-culled and
            // projected, 32 per warp iteration (every lane busy)
            const Box box = lane_box(rp, lane, vmask);
            uint32_t views = MV ? tile_views(a, box, lane) : (1u << a.nviews) - 1u, vis = 0u;
#pragma unroll 1
            for (uint32_t vv = views; vv; vv &= vv - 1u) {
                const int vs = __ffs(vv) - 1;
                if (!__all_sync(kFull, box_culled(a.v[vs], box))) vis |= 1u << vs;
            }
            int gn = 0;
            if (vis) {
                hash_ghosts();
                const uint32_t gm = (a.spatial_rendered ? ~ghosts : ghosts) & (uint32_t)vmask;  // R22 / R31
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const bool bit = (gm >> j) & 1u;
                    const unsigned b = __ballot_sync(kFull, bit);
                    if (bit) sm.gl[wid][gn + __popc(b & lt)] = (uint8_t)((j >> 2) * 128 + 4 * lane + (j & 3));
                    gn += __popc(b);
                }
                __syncwarp();
            }
            if (gn > 0) {
#pragma unroll 1
                while (vis) {
                    const int vs = __ffs(vis) - 1;
                    vis &= vis - 1u;
                    const ViewDesc &v = a.v[vs];
                    for (int i0 = 0; i0 < gn; i0 += 32) {
                        const bool in = i0 + lane < gn;
                        const int e = in ? sm.gl[wid][i0 + lane] : 0;
                        const float x = rp[0][e], y = rp[1][e], z = rp[2][e];
                        const float rw = staged_r ? rp[3][e] : a.radius_uniform;
                        const uint32_t gi = a.goff + (uint32_t)(base + e);
                        float Zf, mz;
                        bool cand = in && precull_fma_z<MODEL>(v, x, y, z, Zf, mz);
                        if (a.discard) cand = cand && maybe_kept(a, v, rw, Zf, mz, gi);
                        if (__any_sync(kFull, cand))
                            bwd_emit<MODEL, CT, MV>(a, v, vs, cand, !a.spatial_rendered, x, y, z, rw, base + e, gi, ct, cg,
                                                false, lane, lt);
                    }
                }
            }
            __syncwarp();  // the ghost list is rewritten by the next tile; every lane is done with the stage
            if (lane == 0) issue(k + kBPool);
            __syncwarp();
            continue;
        }
        hash_ghosts();
        const Box box = lane_box(rp, lane, vmask);
        uint32_t views = MV ? tile_views(a, box, lane) : (1u << a.nviews) - 1u;
#pragma unroll 1
        while (views) {
            const int vs = __ffs(views) - 1;
            views &= views - 1u;
            const ViewDesc &v = a.v[vs];
            if (__all_sync(kFull, box_culled(v, box))) continue;
            uint32_t m = 0u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float4 X = lane_row(rp[0], lane, h), Y = lane_row(rp[1], lane, h), Z = lane_row(rp[2], lane, h);
                const float4 Rw = staged_r ? lane_row(rp[3], lane, h)
                                           : make_float4(a.radius_uniform, a.radius_uniform, a.radius_uniform,
                                                         a.radius_uniform);
                const float xs[4] = {X.x, X.y, X.z, X.w}, ys[4] = {Y.x, Y.y, Y.z, Y.w}, zs[4] = {Z.x, Z.y, Z.z, Z.w};
                const float rs[4] = {Rw.x, Rw.y, Rw.z, Rw.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float Zf, mz;
                    bool cand = precull_fma_z<MODEL>(v, xs[j], ys[j], zs[j], Zf, mz);
                    if (a.discard) cand &= maybe_kept(a, v, rs[j], Zf, mz, a.goff + (uint32_t)pidx(4 * h + j));
                    m |= (cand ? 1u : 0u) << (4 * h + j);
                }
            }
            m &= (uint32_t)vmask;
            while (__any_sync(kFull, m != 0u)) {
                const bool ok = m != 0u;
                const int j = ok ? __ffs(m) - 1 : 0;
                m &= m - 1u;
                const int e = (j >> 2) * 128 + 4 * lane + (j & 3);
                const float rw = staged_r ? rp[3][e] : a.radius_uniform;
                bwd_emit<MODEL, CT, MV>(a, v, vs, ok, (ghosts >> j) & 1u, rp[0][e], rp[1][e], rp[2][e], rw, base + e,
                                    a.goff + (uint32_t)(base + e), ct, cg, tex_on, lane, lt);
            }
        }
        __syncwarp();
        if (lane == 0) issue(k + kBPool);
        __syncwarp();
    }
    list_close<false>(a, ct, lane);
    if (MV && a.mv_lists)
        mv_close_back(a, cg, lane);
    else
        list_close<true>(a, cg, lane);
}

// Column t = view * nt + j of the per-block partials, summed over blocks in a fixed order (deterministic):
// j < 6 -> d_pose[view][j], else d_intr[view][j - 6]; a NULL output is skipped.
__global__ void __launch_bounds__(256) k_pose_reduce(const double *partials, int nblocks, int nviews, int nt,
                                                     double *d_pose, double *d_intr, int accumulate) {
    __shared__ double s[256];
    const int t = blockIdx.x, view = t / nt, j = t % nt;
    double *out = j < 6 ? (d_pose ? d_pose + view * 6 + j : nullptr) : (d_intr ? d_intr + view * kNI + (j - 6) : nullptr);
    if (!out) return;
    const int nvals = nviews * nt;
    double acc = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) acc += partials[(int64_t)b * nvals + t];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = accumulate ? *out + s[0] : s[0];
}

// --------------------------------------------------------------------------- //
// launchers
// --------------------------------------------------------------------------- //
template <typename K>
static int resident_grid(K kernel, int sms, int64_t work_items_per_block, int64_t items) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t need = (items + work_items_per_block - 1) / work_items_per_block;
    int64_t g = (int64_t)sms * per_sm;
    if (need < g) g = need;
    return (int)(g < 1 ? 1 : g);
}

static bool feat_vec4(const RasterArgs &a) {
    return a.channels % 4 == 0 && (reinterpret_cast<uintptr_t>(a.feat) & 15) == 0;
}

static bool accum_vec4(const RasterArgs &a) {
    if (a.channels % 4 != 0) return false;
    for (int v = 0; v < a.nviews; ++v)
        if (reinterpret_cast<uintptr_t>(a.v[v].accum) & 15) return false;
    return true;
}

int launch_clear(const RasterArgs &a, int what, void *stream) {
    int64_t maxP = 1;
    for (int v = 0; v < a.nviews; ++v) maxP = a.v[v].pixels > maxP ? a.v[v].pixels : maxP;
    int64_t bx = (maxP + kThreads * 4 - 1) / (kThreads * 4);
    if (bx > 1184) bx = 1184;
    dim3 grid((unsigned)bx, (unsigned)a.nviews);
    if (what == CLEAR_KEYS)
        k_clear<CLEAR_KEYS><<<grid, kThreads, 0, (cudaStream_t)stream>>>(a);
    else
        k_clear<CLEAR_ACC><<<grid, kThreads, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

static bool depth_pool_enabled() {  // ADOP_DEPTH_POOL=0: the per-warp-ring depth sweep instead (A/B)
    static int env = -1;
    if (env < 0) {
        const char *e = std::getenv("ADOP_DEPTH_POOL");
        env = e ? std::atoi(e) : 1;
    }
    return env != 0;
}

static bool depth_split_enabled() {  // ADOP_DEPTH_SPLIT=1: cull kernel + exact kernel (single-view launches)
    static int env = -1;
    if (env < 0) {
        const char *e = std::getenv("ADOP_DEPTH_SPLIT");
        env = e ? std::atoi(e) : 0;
    }
    return env != 0;
}

static bool ghost_fwd_enabled() {  // ADOP_GHOST_FWD=0: ghosts found by the backward's sweep instead (A/B)
    static int env = -1;
    if (env < 0) {
        const char *e = std::getenv("ADOP_GHOST_FWD");
        env = e ? std::atoi(e) : 1;
    }
    return env != 0;
}

// The depth launch for `a` is the pooled, unsplit sweep (launch_depth_async's first branch on the vector path),
// the only one that lists ghosts.
bool depth_lists_ghosts(const RasterArgs &a) {
    return ghost_fwd_enabled() && depth_pool_enabled() && !a.tbounds && !(a.dyn_tiles & 1) &&
           !(a.nviews == 1 && depth_split_enabled()) && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 &&
           !ADOP_EARLY_RELEASE;
}

template <int MODEL, int VM>
static int launch_depth_async(const RasterArgs &a, int sms, void *stream) {
    if (depth_pool_enabled() && !a.tbounds && !(a.dyn_tiles & 1)) {
        constexpr int NP = VM == 0 ? kPoolSV : kPoolMV;
        using PoolSmem = PoolSmemT<NP>;
        const bool split = VM == 0 && depth_split_enabled();
        auto kp = split ? (a.discard ? k_depth_pool<MODEL, VM, true, true, NP> : k_depth_pool<MODEL, VM, false, true, NP>)
                        : (a.discard ? k_depth_pool<MODEL, VM, true, false, NP> : k_depth_pool<MODEL, VM, false, false, NP>);
        if (cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PoolSmem)) !=
            cudaSuccess)
            return (int)cudaGetLastError();
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, kST, sizeof(PoolSmem));
        if (per_sm < 1) per_sm = 1;
        int64_t g = (int64_t)sms * per_sm;
        const int64_t tiles = (a.n + kWTile - 1) / kWTile;
        if ((tiles + kSW - 1) / kSW < g) g = (tiles + kSW - 1) / kSW;
        if (g < 1) g = 1;
        kp<<<(unsigned)g, kST, sizeof(PoolSmem), (cudaStream_t)stream>>>(a);
        if (split) {
            if constexpr (VM == 0) {
                int pe = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pe, k_depth_exact<MODEL, VM>, kThreads, 0);
                k_depth_exact<MODEL, VM><<<(unsigned)(sms * (pe < 1 ? 1 : pe)), kThreads, 0, (cudaStream_t)stream>>>(a);
            }
        }
        return (int)cudaGetLastError();
    }
    auto k = a.discard ? k_depth_async<MODEL, VM, true> : k_depth_async<MODEL, VM, false>;
    // the dynamic shared-memory limit is a per-device (context) attribute: raised once per device and
    // instance (two threads racing here both set the same value)
    static std::atomic<unsigned long long> attr_set[2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_set[a.discard ? 1 : 0].load(std::memory_order_acquire) & bit)) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DepthSmem)) !=
            cudaSuccess)
            return (int)cudaGetLastError();
        attr_set[a.discard ? 1 : 0].fetch_or(bit, std::memory_order_acq_rel);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kST, sizeof(DepthSmem));
    if (per_sm < 1) per_sm = 1;
    int64_t tiles = (a.n + kWTile - 1) / kWTile;
    int64_t g = (int64_t)sms * per_sm;
    if ((tiles + kSW - 1) / kSW < g) g = (tiles + kSW - 1) / kSW;
    if (g < 1) g = 1;
    k<<<(unsigned)g, kST, sizeof(DepthSmem), (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

template <int MODEL, bool VEC>
static int launch_depth_t(const RasterArgs &a, int sms, void *stream) {
    if (VEC && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0)
        return a.nviews > 2 ? launch_depth_async<MODEL, 2>(a, sms, stream)
               : (a.nviews == 1 ? launch_depth_async<MODEL, 0>(a, sms, stream) : launch_depth_async<MODEL, 1>(a, sms, stream));
    auto k = k_stream<MODEL, VEC, MODE_DEPTH, false>;
    int g = resident_grid(k, sms, kWarps * 128, a.n);
    k<<<g, kThreads, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

int launch_depth(const RasterArgs &a, int model, bool vec, int sms, void *stream) {
    if (model == 0) return vec ? launch_depth_t<0, true>(a, sms, stream) : launch_depth_t<0, false>(a, sms, stream);
    if (model == 2) return vec ? launch_depth_t<2, true>(a, sms, stream) : launch_depth_t<2, false>(a, sms, stream);
    return vec ? launch_depth_t<1, true>(a, sms, stream) : launch_depth_t<1, false>(a, sms, stream);
}

template <int MODEL, bool VEC, bool VEC4>
static int launch_blend_t(const RasterArgs &a, int sms, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    auto k = k_blend<MODEL, VEC, VEC4, false>;
    if constexpr (VEC && VEC4)
        if (a.nviews == 1) k = k_blend<MODEL, VEC, VEC4, true>;
    int g = resident_grid(k, sms, kWarps * 128, a.n > 0 ? a.n : 1);
    if (a.clear_pyr) {  // a shared pyramid was reset by its owner (adop_clear_pyramid)
        int e = launch_clear(a, CLEAR_ACC, stream);
        if (e) return e;
    }
    k<<<g, kThreads, 0, s>>>(a);
    return (int)cudaGetLastError();
}

int launch_blend(const RasterArgs &a, int model, bool vec, int sms, void *stream) {
    const bool v4 = feat_vec4(a) && accum_vec4(a);
    if (model == 0) {
        if (vec) return v4 ? launch_blend_t<0, true, true>(a, sms, stream) : launch_blend_t<0, true, false>(a, sms, stream);
        return v4 ? launch_blend_t<0, false, true>(a, sms, stream) : launch_blend_t<0, false, false>(a, sms, stream);
    }
    if (model == 2) {
        if (vec) return v4 ? launch_blend_t<2, true, true>(a, sms, stream) : launch_blend_t<2, true, false>(a, sms, stream);
        return v4 ? launch_blend_t<2, false, true>(a, sms, stream) : launch_blend_t<2, false, false>(a, sms, stream);
    }
    if (vec) return v4 ? launch_blend_t<1, true, true>(a, sms, stream) : launch_blend_t<1, true, false>(a, sms, stream);
    return v4 ? launch_blend_t<1, false, true>(a, sms, stream) : launch_blend_t<1, false, false>(a, sms, stream);
}

// View-major order of list 0 (survivor records) or 1 (ghost entries) of a multi-view launch.
int launch_chunk_order(const RasterArgs &a, int list, int sms, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int e = (int)cudaMemsetAsync(a.ccount + list * 64, 0, 64 * sizeof(uint32_t), s);
    if (e) return e;
    k_chunk_hist<<<sms, kThreads, 0, s>>>(a, list);
    k_chunk_scatter<<<sms, kThreads, 0, s>>>(a, list);
    return (int)cudaGetLastError();
}

int launch_resolve(const RasterArgs &a, void *stream) {
    int64_t maxP = 1;
    for (int v = 0; v < a.nviews; ++v) maxP = a.v[v].pixels > maxP ? a.v[v].pixels : maxP;
    int64_t bx = (maxP + kThreads - 1) / kThreads;
    if (bx > 4096) bx = 4096;
    dim3 grid((unsigned)bx, (unsigned)a.nviews);
    bool v4 = accum_vec4(a);
    for (int v = 0; v < a.nviews && v4; ++v) {
        if (reinterpret_cast<uintptr_t>(a.v[v].count) & 15) v4 = false;
        if (reinterpret_cast<uintptr_t>(a.v[v].image) & 15) v4 = false;
        for (int l = 0; l < a.layers; ++l)
            if ((a.v[v].off[l] & 3) || (((int64_t)a.v[v].wl[l] * a.v[v].hl[l]) & 3)) v4 = false;
        if (a.v[v].pixels & 3) v4 = false;
    }
    if ((a.res_p0 & 3) || ((a.res_p1 & 3) && a.res_p1 < maxP)) v4 = false;  // a range resolved 4 pixels at a time
    cudaStream_t s = (cudaStream_t)stream;
    if (a.env) {
        if (v4) k_resolve<true, true><<<grid, kThreads, 0, s>>>(a);
        else k_resolve<false, true><<<grid, kThreads, 0, s>>>(a);
    } else {
        if (v4) k_resolve<true, false><<<grid, kThreads, 0, s>>>(a);
        else k_resolve<false, false><<<grid, kThreads, 0, s>>>(a);
    }
    return (int)cudaGetLastError();
}

// The argument block with the backward's pixel-table pointers (workspace table region).
static RasterArgs with_tables(const RasterArgs &a) {
    RasterArgs b = a;
    char *base = reinterpret_cast<char *>(a.tables);
    int64_t off = 0;
    b.prow = 4 + ((a.channels + 3) & ~3);  // row stride in floats (16-B multiple)
    for (int v = 0; v < a.nviews; ++v) {
        b.v[v].prow = reinterpret_cast<const float *>(base + off);
        off += (int64_t)a.v[v].pixels * b.prow * (int64_t)sizeof(float);
    }
    return b;
}

int launch_env_grad(const RasterArgs &a, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!a.d_env || !a.tables) return (int)cudaErrorInvalidValue;
    if (!a.grad_accumulate)
        cudaMemsetAsync(a.d_env, 0, sizeof(float) * (size_t)a.env_w * a.env_h * a.channels, s);
    int64_t maxP = 1;
    for (int v = 0; v < a.nviews; ++v) maxP = a.v[v].pixels > maxP ? a.v[v].pixels : maxP;
    int64_t bx = (maxP + kThreads - 1) / kThreads;
    if (bx > 2048) bx = 2048;
    k_bwd_prep<<<dim3((unsigned)bx, (unsigned)a.nviews), kThreads, 0, s>>>(with_tables(a));
    return (int)cudaGetLastError();
}

int backward_grid(int sms) {
    int g = sms * 8;
    return g > kMaxBwdBlocks ? kMaxBwdBlocks : g;
}

// Per-thread, per-device side stream and fork / join events of the backward (created on first use, never
// destroyed; thread-local so concurrent callers never share a fork event).  NULL if creation failed: the
// caller's stream is used alone.
#ifndef ADOP_BWD_SIDE_STREAM
#define ADOP_BWD_SIDE_STREAM 1
#endif
constexpr int kMaxDevices = 64;
static cudaStream_t side_stream() {
    if (!ADOP_BWD_SIDE_STREAM) return nullptr;
    static thread_local cudaStream_t streams[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        streams[dev] = nullptr;
    }
    return streams[dev];
}
static cudaEvent_t side_event(int which) {
    static thread_local cudaEvent_t events[kMaxDevices][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) return nullptr;
    if (!events[dev][which] && cudaEventCreateWithFlags(&events[dev][which], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        events[dev][which] = nullptr;
    }
    return events[dev][which];
}

template <int MODEL, bool VEC, int CT>
static int launch_backward_t(const RasterArgs &a, int sms, int grid_cap, double *d_pose, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t maxP = 1;
    for (int v = 0; v < a.nviews; ++v) maxP = a.v[v].pixels > maxP ? a.v[v].pixels : maxP;
    const bool fast = VEC && a.tables != nullptr && a.rec_capacity >= 4 * kChunk &&
                      (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 &&
                      (!a.radius || (reinterpret_cast<uintptr_t>(a.radius) & 15) == 0);
    RasterArgs b = with_tables(a);
    b.grad_accumulate = 1;  // every kernel below adds into the (zeroed or caller's) gradients
    const int64_t n_env = a.d_env ? (int64_t)a.env_w * a.env_h * a.channels : 0;
    if (!fast) {  // planar fused sweep (unaligned inputs or a small workspace)
        if (a.d_env) {  // the environment-map gradient comes from the pixel-table pass
            int e = launch_env_grad(a, stream);
            if (e) return e;
        }
        auto k = k_backward<MODEL, VEC, CT>;
        int g = resident_grid(k, sms, kWarps * 128, a.n);
        if (g > grid_cap) g = grid_cap;
        k<<<g, kThreads, 0, s>>>(a);
        if (d_pose || a.d_intr)
            k_pose_reduce<<<a.nviews * a.nterms, 256, 0, s>>>(a.pose_partials, g, a.nviews, a.nterms, d_pose, a.d_intr,
                                                              a.grad_accumulate);
        return (int)cudaGetLastError();
    }
    // ghost-list kernel grid (its per-block pose partials) and the inline-overflow row after them
    int gg = sms * 4;
    if (gg > grid_cap - 1) gg = grid_cap - 1;
    b.inline_row = gg;
    {   // zero-fill (overwrite mode), reset the work-list counters and the inline pose row
        const bool fill = !a.grad_accumulate;
        int64_t nf = (fill && a.d_feat) ? a.n * a.channels : 0, np = (fill && a.d_pos) ? 3 * a.n : 0;
        int64_t mx = nf > np ? nf : np;
        int64_t bx = (mx / 4 + kThreads - 1) / kThreads;
        if (bx > (int64_t)sms * 8) bx = (int64_t)sms * 8;
        if (bx < 1) bx = 1;
        const int64_t ne = fill ? n_env : 0;
        k_fill<<<(unsigned)bx, kThreads, 0, s>>>(nf ? a.d_feat : nullptr, nf, np ? a.d_pos : nullptr, np,
                                                ne ? a.d_env : nullptr, ne, a.hdr,
                                                a.pose_partials + (int64_t)gg * a.nviews * a.nterms, a.nviews * a.nterms,
                                                a.tag, a.spatial_rendered ? 0 : 1);
    }
    {   // per-pixel tables
        int64_t bx = (maxP + kThreads - 1) / kThreads;
        if (bx > 2048) bx = 2048;
        k_bwd_prep<<<dim3((unsigned)bx, (unsigned)a.nviews), kThreads, 0, s>>>(b);
    }
    {   // sweep: emit work lists
        for (int go = 0; go < 2; ++go) {  // the instance not matching the device-side mode exits at once
            auto k = a.nviews > 2 ? (go ? k_bwd_sweep<MODEL, CT, true, true> : k_bwd_sweep<MODEL, CT, true, false>)
                                  : (go ? k_bwd_sweep<MODEL, CT, false, true> : k_bwd_sweep<MODEL, CT, false, false>);
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BwdSmem));
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kST, sizeof(BwdSmem));
            if (per_sm < 1) per_sm = 1;
            int64_t tiles = (a.n + kWTile - 1) / kWTile;
            int64_t g = (int64_t)sms * per_sm;
            if ((tiles + kSW - 1) / kSW < g) g = (tiles + kSW - 1) / kSW;
            if (g < 1) g = 1;
            k<<<(unsigned)g, kST, sizeof(BwdSmem), s>>>(b);
        }
    }
    if (b.mv_lists) {  // the ghost list's per-view chunks in view-major order
        int e = launch_chunk_order(b, 1, sms, stream);
        if (e) return e;
    }
    // the two list consumers are independent (d_feat from the texture list; d_pos and the pose / intrinsics
    // partials from the ghost list) and both latency-bound: the texture kernel runs on a side stream forked
    // from and joined back into the caller's (event fork / join, CUDA-graph capturable).
    // Measured: configs[2] backward 0.387 -> 0.351 ms; with 16 views (configs[4], 0.7 GB of pixel tables) the
    // two consumers thrash L2 together (+1.5%), so large launches keep them in sequence.
    int64_t tbytes = 0;
    for (int v = 0; v < a.nviews; ++v) tbytes += a.v[v].pixels * b.prow * (int64_t)sizeof(float);
    cudaStream_t side = (a.d_feat && tbytes <= (256ll << 20)) ? side_stream() : nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (side) {
        fork = side_event(0);
        join = side_event(1);
        if (!fork || !join) side = nullptr;  // no events: stay on the caller's stream
    }
    if (side) {
        cudaEventRecord(fork, s);
        cudaStreamWaitEvent(side, fork, 0);
    }
    if (a.d_feat) k_bwd_tex<<<sms * 8, kThreads, 0, side ? side : s>>>(b);
    if (a.nterms == kNT)  // the intrinsics terms cost 12 more fp64 warp sums per ghost: only when requested
        k_bwd_ghost<MODEL, CT, kNT><<<gg, kThreads, 0, s>>>(b);
    else
        k_bwd_ghost<MODEL, CT, 6><<<gg, kThreads, 0, s>>>(b);
    if (side) {
        cudaEventRecord(join, side);
        cudaStreamWaitEvent(s, join, 0);
    }
    if (d_pose || a.d_intr)
        k_pose_reduce<<<a.nviews * a.nterms, 256, 0, s>>>(a.pose_partials, gg + 1, a.nviews, a.nterms, d_pose, a.d_intr,
                                                          a.grad_accumulate);
    return (int)cudaGetLastError();
}

template <int MODEL, bool VEC>
static int launch_backward_c(const RasterArgs &a, int sms, int grid_cap, double *d_pose, void *stream) {
    if (a.channels == 4) return launch_backward_t<MODEL, VEC, 4>(a, sms, grid_cap, d_pose, stream);
    if (a.channels == 8) return launch_backward_t<MODEL, VEC, 8>(a, sms, grid_cap, d_pose, stream);
    return launch_backward_t<MODEL, VEC, 0>(a, sms, grid_cap, d_pose, stream);
}

int launch_backward(const RasterArgs &a, int model, bool vec, int sms, int grid_cap, double *d_pose, void *stream) {
    if (model == 0) return vec ? launch_backward_c<0, true>(a, sms, grid_cap, d_pose, stream)
                               : launch_backward_c<0, false>(a, sms, grid_cap, d_pose, stream);
    if (model == 2) return vec ? launch_backward_c<2, true>(a, sms, grid_cap, d_pose, stream)
                               : launch_backward_c<2, false>(a, sms, grid_cap, d_pose, stream);
    return vec ? launch_backward_c<1, true>(a, sms, grid_cap, d_pose, stream)
               : launch_backward_c<1, false>(a, sms, grid_cap, d_pose, stream);
}

int launch_masks(const RasterArgs &a, int model, void *stream) {
    const int64_t nchunks = (a.n + 127) / 128;
    int64_t g = (nchunks + kWarps - 1) / kWarps;
    if (g < 1) g = 1;
    if (g > 65535) g = 65535;
    if (model == 0)
        k_stream<0, false, MODE_MASKS, false><<<(unsigned)g, kThreads, 0, (cudaStream_t)stream>>>(a);
    else if (model == 2)
        k_stream<2, false, MODE_MASKS, false><<<(unsigned)g, kThreads, 0, (cudaStream_t)stream>>>(a);
    else
        k_stream<1, false, MODE_MASKS, false><<<(unsigned)g, kThreads, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace adop
