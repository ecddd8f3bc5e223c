// adop_internal.h -- kernel argument blocks shared by the host API (adop_api.cu)
// and the kernels (adop_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda.h>

#include "../../include/adop.h"

#define ADOP_MAX_VIEWS_PER_LAUNCH 16

namespace adop {

// Per-view constants, passed by value in the __grid_constant__ kernel argument block.
struct ViewDesc {
    float R[9];
    float t[3];
    float fx, fy, cx, cy;
    float k[6];
    float p[2];
    float r2_max;
    int32_t model;         // ADOP_PINHOLE / ADOP_OPENCV8 (runtime use: C^-1 of the environment map)
    float feff;            // fl(fl(fx + fy) * 0.5): focal length of the discard radius (R10)
    float ulo, uhi, vlo, vhi;  // conservative pre-cull window (pixels, all layers)
    float r2cull;          // OpenCV8 pre-cull on X^2+Y^2 <= r2cull Z^2
    float fk, fkt;         // FMA pre-cull margin: m = fk * (|x|+|y|+|z|) + fkt
    float pl[5][4];        // conservative world-space frustum planes n.p + d >= 0 (warp-box cull)
    float pm[5][2];        // their margins: m = pm0 * sum_a max|p_a| + pm1 (+ 2^-16 |terms|)
    int32_t zplane;        // plane 4 is the depth half-space Z + (pl[4][3] - t_z) >= 0 (all but the wide fisheye)
    float zoff;            // Z = plane-4 value + zoff (z_near; 0 for the fisheye)
    uint32_t discard_salt; // hash salt of (seed, DISCARD, view id) (R11)
    int32_t wl[ADOP_MAX_LAYERS], hl[ADOP_MAX_LAYERS], off[ADOP_MAX_LAYERS];
    int32_t pixels;        // P
    uint64_t *keys;
    float *accum, *count, *image;
    const float *grad;     // backward: dL/dI (image layout)
    const float *prow;     // backward pixel table: [P] rows of RasterArgs::prow floats (k_bwd_prep)
    float wn[4];           // OpenCV8: image window in undistorted normalized coordinates (xlo, xhi, ylo, yhi):
    int32_t wn_on;         // every point landing in some layer has xlo Z <= X <= xhi Z, ylo Z <= Y <= yhi Z
};

struct Record {  // one (point, view, layer) hit of the render set, 16 bytes
    uint32_t pix;   // pixel index within the view's pyramid (off_l + local)
    uint32_t zbits; // bits of the point's camera-space z
    uint32_t idx;   // shard-local point index
    uint32_t view;  // view slot within the launch (0xFFFFFFFF: dead slot)
};

struct GhostEntry {  // one (ghost point, view) kept at >= 1 layer (§4.3), 32 bytes = 2 record slots
    float u0, v0;    // layer-0 continuous pixel coordinates (R2/R6)
    float X, Y;      // camera-space point (R1)
    float Z;
    uint32_t idx;    // shard-local point index
    uint32_t vsnk;   // view slot | kept layers << 8 (0xFFFFFFFF: dead entry)
    float D;         // depth of keys / Eq. 6: Z, or the distance for the fisheye (R35)
};
constexpr int kResvBackShift = 40;

// The record region of the workspace holds two lists: survivor records (16-B Record slots) growing
// from the front -- written by the depth pass, read by the blend and by the backward's texture gradient
// -- and ghost entries (GhostEntry, two slots each) growing from the back, written by the backward
// sweep.  (When the backward cannot reuse the survivor records it re-renders them into the front list.)
// Both are reserved per warp in chunks through ONE 64-bit counter `resv` (front slots in the low 40
// bits, back chunks of 256 slots in the high 24); the successful reservations form the prefixes
// [0, front_ok) and [capacity - back_ok, capacity) (see resv_take in adop_kernels.cu).
struct WsHeader {
    unsigned long long resv;       // front slots | back chunks << 40 (see above)
    int32_t overflow;              // set when a reservation did not fit (the lists are incomplete)
    int32_t mode;                  // backward: 1 = texture list = the depth pass's records, 0 = full re-render
    unsigned long long tag;        // fingerprint of the call that wrote the lists (0: not reusable)
    unsigned long long front_ok;   // slots of the front list (survivor / texture records)
    unsigned long long back_ok;    // slots of the back list (ghost entries, 2 slots each)
    unsigned long long tiles_read; // tile culling: tiles the depth pass loaded
    unsigned long long tiles_fwd;  // dynamic tile counters of the depth and backward sweeps
    unsigned long long tiles_bwd;
    int32_t ghosts_fwd;            // 1: the depth pass listed every ghost (back list), the backward needs no sweep
    int32_t pad_;
};

// Frustum half-spaces of every view in the workspace (written by k_clear<KEYS> of the depth phase;
// the backward sweep writes its own copy): tile_views reads them with a per-lane view index through L1.
struct PlaneTab {
    float4 pl[5];  // (n, d)
    float2 pm[5];  // margins (see box_culled)
};

// Layer table of one view (read with a per-lane view slot by the depth drain; in the workspace header,
// written by k_clear<KEYS>, and in shared memory for the backward sweep).
struct LayerDesc {
    int32_t off[ADOP_MAX_LAYERS], wl[ADOP_MAX_LAYERS], hl[ADOP_MAX_LAYERS];
    uint64_t *keys;
};

struct RasterArgs {
    CUtensorMap tmap;      // 2-D TMA descriptor of the x/y/z rows ([3][pos_stride] fp32), box 256 x 3
    int32_t use_tmap;
    const float *x, *y, *z;
    const float *radius;
    float radius_uniform;
    const float *feat;
    int64_t n;
    int32_t ntiles, nfull; // depth sweep: ceil(n / 256) tiles, of which the first n / 256 are full
    uint32_t goff;
    int32_t channels;
    int32_t layers;
    int32_t nviews;
    int32_t view_slot0;    // view slot of views[0] in the record's view field (multi-launch chunks)
    float onepa;           // fl(1 + alpha)
    float gamma;
    float z_near;
    int32_t discard;
    uint32_t ghost_thr;    // floor(rho * 2^24); 0 = no ghosts
    uint32_t ghost_salt;
    int32_t grad_accumulate;
    float bg[ADOP_MAX_CHANNELS];
    int32_t spatial_rendered;  // NEXT-3 (R31): spatial gradients for rendered points instead of ghosts
    int32_t normal_cull;   // NEXT-3, Eq. 5 (R32): 0 off, +1 / -1 sign of (R n).Xc that is kept
    const float *nrm;      // normals SoA [3][nrm_stride] (device) when normal_cull != 0
    int64_t nrm_stride;
    int32_t log_desc;      // NEXT-2: descriptors stored as log, linearized with exp()
    int32_t clear_pyr;     // 1: the phases clear keys / accum / count; 0: shared pyramid (adop_clear_pyramid)
                           // (placed in the padding after log_desc: the other fields keep their offsets)
    const float *env;      // NEXT-2: environment map [env_h][env_w][C] (device) or NULL (R18 constant bg)
    int32_t env_w, env_h;
    float *d_env;          // backward: [env_h][env_w][C] environment-map gradient or NULL
    WsHeader *hdr;
    Record *records;       // record region: survivor records (front) + ghost list (back), see WsHeader
    int64_t rec_capacity;  // in 16-B slots
    void *tables;          // backward pixel tables, per view [P][prow] floats
    int32_t prow;          // pixel-table row stride in floats: 4 + C rounded up to a multiple of 4
    double *pose_partials; // [gridDim.x][nviews][nterms]
    int32_t nterms;        // structural terms per view: 6 (pose) or 18 (pose + 12 intrinsics, NEXT-1)
    double *d_intr;        // backward: [V][12] intrinsics gradient or NULL
    int32_t inline_row;    // pose-partials row for inline (list overflow) ghost contributions
    int32_t dyn_tiles;     // bit 0: depth sweep, bit 1: backward sweep use dynamic tile claiming
    unsigned long long tag;// fingerprint of this call's inputs (host); 0 = records not reusable by the backward
    const float *tbounds;  // tile culling: per-256-point-tile AABBs [ntiles][8] (adop_tile_bounds) or NULL
    PlaneTab *planes;      // [nviews] in the workspace header area
    LayerDesc *ldesc;      // [nviews] in the workspace header area
    float *d_feat;
    float *d_pos;          // [3][n]
    uint8_t *mask;         // point-mask debug output [V][n]
    ViewDesc v[ADOP_MAX_VIEWS_PER_LAUNCH];
    // Multi-view work lists (nviews > 2; appended after v[] so the fields above keep their offsets): the record
    // region is cut into kListChunk-slot chunks, every chunk of the depth pass's survivor list and of the
    // backward's ghost list holds ONE view's items, and the consumers walk the chunks in view-major order
    // (k_chunk_hist / k_chunk_scatter), so one view's keys, accumulators and pixel tables stay in L2.
    uint8_t *cview;        // [rec_capacity / kListChunk] view of each chunk (written when it is reserved)
    uint32_t *corder[2];   // view-major chunk order of the front (survivor) and back (ghost) list
    uint32_t *ccount;      // [2][64]: per-view chunk counts [0..16], cursors [32..48], total [63]
    int32_t mv_lists;      // bit 0: the sweeps write per-view chunks (the blend walks them view-major);
                           // bit 1: the texture consumer walks them view-major too; bit 2: the ghost consumer
    int32_t ghost_fwd;     // the depth pass also lists the ghosts (back of the record region) for the backward
    int64_t res_p0, res_p1;  // resolve only pyramid pixels [res_p0, res_p1) of every view (adop_forward_resolve_range)
};
constexpr int kListChunk = 64;  // record slots per chunk of the chunk table (a 64-aligned unit of every list)

// Launchers (adop_kernels.cu).  Return cudaError_t as int.
int launch_clear(const RasterArgs &a, int what, void *stream);  // 0 keys+header, 1 accum+count
int launch_depth(const RasterArgs &a, int model, bool vec, int sms, void *stream);
bool depth_lists_ghosts(const RasterArgs &a);  // the depth launch for `a` runs k_depth_pool (it can list ghosts)
int launch_blend(const RasterArgs &a, int model, bool vec, int sms, void *stream);
int launch_resolve(const RasterArgs &a, void *stream);
int launch_chunk_order(const RasterArgs &a, int list, int sms, void *stream);  // multi-view lists (mv_lists)
int launch_backward(const RasterArgs &a, int model, bool vec, int sms, int grid, double *d_pose, void *stream);
int launch_masks(const RasterArgs &a, int model, void *stream);
int launch_env_grad(const RasterArgs &a, void *stream);  // d_env only (zeroed first unless grad_accumulate)
int launch_clear_pyr(uint64_t *keys, float *accum, float *count, int64_t P, int C, void *stream);
int launch_tile_bounds(const float *x, const float *y, const float *z, int64_t n, float *out, void *stream);
adop_status set_status(adop_status s, const char *msg);  // thread-local last-error message (adop_api.cu)
// collectives of a communicator between the fused entry points' phases (adop_comm.cu; comm NULL: no-ops)
adop_status comm_check(const adop_comm *comm);
adop_status comm_keys(adop_comm *comm, const adop_pyramid *views, const int64_t *pixels, int32_t n_views, void *stream);
adop_status comm_sums(adop_comm *comm, const adop_pyramid *views, const int64_t *pixels, int32_t n_views, int32_t C,
                      void *stream);
adop_status comm_grads(adop_comm *comm, int64_t n, int32_t C, int32_t n_views, float *d_feat, float *d_pos,
                       double *d_pose, double *d_intr, float *d_env, int64_t n_env, void *stream);
int backward_grid(int sms);

}  // namespace adop
