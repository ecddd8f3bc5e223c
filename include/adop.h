/*
 * adop.h -- C-ABI of the B200-native ADOP one-pixel point rasterizer
 * (Rückert, Franke, Stamminger, "ADOP: Approximate Differentiable One-Pixel
 * Point Rendering", arXiv 2110.06635).  Library: libadop.so (sm_100a).
 *
 * The entry points are the render function of Eq. 1 (PAPER.md L171-177,
 * §4 "I_l = Phi_l(C, R, t, x, n, E, tau)") split into the three passes of
 * §4.5 (L356-359: depth-only pass, accumulate with counts, normalize), and
 * its backward (§4.2-4.3: texture gradient, ghost-geometry
 * position and tangent-space pose gradients, Eq. 8, Eq. 17).
 *
 * Conventions (all entry points):
 *  - Every pointer inside adop_points / adop_pyramid and every gradient
 *    pointer is DEVICE memory (cudaMalloc / torch CUDA tensor) on the current
 *    device; camera, pose and params descriptors (and params->background)
 *    are HOST memory read during the call.
 *  - The caller owns every buffer.  The library allocates no device memory;
 *    scratch comes from the caller's workspace (adop_workspace_size).
 *  - Work is enqueued on `stream` (a cudaStream_t passed as void*, NULL =
 *    legacy default stream).  No entry point synchronizes the host.
 *  - All argument checks run on the host before anything is enqueued; on
 *    any error nothing runs and adop_last_error() describes it.  Points that
 *    are behind the camera or non-finite are NOT errors: they are culled
 *    (PAPER.md L205-207 bounds test; R7).
 *  - No C++ exception crosses this boundary.
 *
 * Layouts:
 *  - positions: SoA rows x, y, z: pos[0..n), pos[stride..stride+n),
 *    pos[2*stride..2*stride+n).  Rows 16-byte aligned with stride % 4 == 0
 *    select the vectorized load path (any 4-byte aligned layout works).
 *  - features tau: [n][C] fp32 row-major (C contiguous).
 *  - pyramid of one view, L layers, layer l of size w_l x h_l with
 *    w_l = ceil(w / 2^l), h_l = ceil(h / 2^l) (R5), pixel offset
 *    off_l = sum_{k<l} w_k h_k, P = off_L:
 *      keys  [P]    uint64 packed depth keys (bits(z) << 32 | global index),
 *                   empty pixel = 0x7FFFFFFFFFFFFFFF (R8)
 *      count [P]    float, |Lambda_{l,u,v}| (exact integers)
 *      accum [P][C] float, sum of tau over Lambda (shard-reducible scratch)
 *      image [C*P]  float, layer l stored planar [C][h_l][w_l] at C*off_l
 *                   (an NCHW tensor per layer), Eq. 7 output.
 *  - upstream gradient dL/dI: same layout as image.
 *  - d_feat [n][C], d_pos [3][n] (SoA rows, stride n), d_pose [V][6] double
 *    ordered (translation, rotation) of the left tangent increment of Eq. 17.
 */
#ifndef ADOP_H
#define ADOP_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ADOP_API __attribute__((visibility("default")))
#else
#define ADOP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ADOP_OK = 0,
    ADOP_ERR_INVALID_ARGUMENT = 1,
    ADOP_ERR_SHAPE_MISMATCH = 2,
    ADOP_ERR_UNSUPPORTED = 3,
    ADOP_ERR_WORKSPACE_TOO_SMALL = 4,
    ADOP_ERR_CUDA = 5,
    ADOP_ERR_NCCL = 6
} adop_status;

enum { ADOP_PINHOLE = 0, ADOP_OPENCV8 = 1, ADOP_FISHEYE = 2 };

/* Multi-GPU communicator (adop_comm_init; NULL everywhere = single GPU).  The two partitionings of the
 * north star ("well over 100M points"; the paper itself is single-GPU, L811):
 *  ADOP_SHARD_POINTS: every rank renders its shard of one cloud (disjoint global_offset ranges) into a full
 *    local pyramid; adop_rasterize_forward MIN-reduces the keys after the depth pass (64-bit keys, or only
 *    the 32-bit depth words with ADOP_COMM_KEYS32 -- the blend reads only those; the winner indices then
 *    stay shard-local) and SUM-reduces accum and count after the blend, so every rank resolves the image
 *    of the whole cloud; adop_rasterize_backward sums d_pose and d_intrinsics over the shards.
 *  ADOP_SHARD_VIEWS: every rank renders the whole cloud for its range of the batch's views (params
 *    view_id_base = the range's first view, so the discard draws equal the unsharded batch's); the forward
 *    is local and adop_rasterize_backward sums d_feat, d_pos and d_env over the ranks (d_pose rows stay
 *    with their view's rank).
 * Collectives are NCCL (libnccl.so.2 loaded at run time) on the call's stream; NCCL errors return
 * ADOP_ERR_NCCL. */
typedef struct adop_comm adop_comm;
enum { ADOP_SHARD_POINTS = 0, ADOP_SHARD_VIEWS = 1 };
enum { ADOP_COMM_KEYS32 = 1 };

#define ADOP_MAX_LAYERS 8
#define ADOP_MAX_CHANNELS 32

/* One shard of the point cloud (x, tau and r_world of Eq. 1 / §4.4). */
typedef struct {
    int64_t n;              /* points in this shard, >= 0                                  */
    int64_t global_offset;  /* global index of point 0; keys and hashes use it (R25);
                               global_offset + n <= 2^32                                  */
    int64_t pos_stride;     /* elements between the x, y, z rows, >= n                      */
    const float *pos;       /* device, SoA [3][pos_stride]                                  */
    const float *radius;    /* device [n] world radius r_world (§4.4), or NULL         */
    float radius_uniform;   /* used when radius == NULL                                     */
    const float *feat;      /* device [n][C] neural descriptor tau -- or pinned HOST memory
                               (cudaHostAlloc / torch pin_memory, device-accessible through
                               UVA): the forward then reads only the survivors' descriptors
                               over PCIe, in place (zero-copy; bench.py's e2e)             */
    int32_t channels;       /* C, 1..32                                                     */
    const float *normal;    /* device SoA [3][pos_stride] normals n of Eq. 1 (Eq. 5 culling),
                               or NULL; required when params->normal_culling != 0        */
    const float *tile_bounds;/* device [ceil(n/256)][8] per-256-point-tile bounding boxes
                               (adop_tile_bounds) or NULL.  When given, the depth pass
                               neither loads nor processes tiles whose box meets no view's
                               frustum (results are identical; for static clouds rendered
                               many times).  Must describe the current positions.          */
} adop_points;

/* Camera model C of Eq. 2 (R6): pinhole, or OpenCV rational 8-coefficient distortion
 * on normalized coordinates; points with r^2 > r2_max or a non-positive radial
 * denominator are culled.  Host memory. */
typedef struct {
    int32_t width, height;  /* layer-0 image size, >= 1                                     */
    int32_t model;          /* ADOP_PINHOLE, ADOP_OPENCV8, or ADOP_FISHEYE: equidistant
                               r_d = f theta with the distance |Xc| as depth (L214; DESIGN.md
                               R35), r2_max = theta_max in (0, pi]                          */
    float fx, fy, cx, cy;   /* pixels; pixel centres at integer coordinates                 */
    float k[6];             /* k1..k6 (OpenCV8)                                             */
    float p[2];             /* p1, p2 (OpenCV8)                                             */
    float r2_max;           /* validity radius in normalized r^2 (OpenCV8; +inf allowed)   */
} adop_camera;

/* World -> camera rigid transform (R, t) of Eq. 2: Xc = R x + t, R row-major.  Host. */
typedef struct {
    float R[9];
    float t[3];
} adop_pose;

/* Method parameters.  Host memory. */
typedef struct {
    int32_t layers;         /* L, 1..8 (Eq. 1 l in {0..L-1})                                */
    float alpha;            /* fuzzy depth threshold of Eq. 6, >= 0 (paper: 0.01, L217)     */
    int32_t discard;        /* stochastic point discarding of §4.4 on/off                   */
    float gamma;            /* Eq. 12 gamma > 0 (paper: 1.5, L349)                          */
    float ghost_rate;       /* rho in [0,1): fraction of points in the ghost set (§4.3)    */
    float z_near;           /* near plane >= 0; points with z <= z_near are culled (R7)     */
    uint64_t seed;          /* seeds the ghost split and the per-(view, point) beta (R11)   */
    int32_t view_id_base;   /* global id of view 0 of this call (beta is keyed by it)       */
    const float *background;/* host [C] constant environment colour E (R18), NULL = zeros   */
    int32_t grad_accumulate;/* backward: 0 overwrite d_feat/d_pos/d_pose, 1 add into them   */
    int32_t log_descriptors;/* tau stored as log, exp() when rasterized (NEXT-2) */
    const float *env_map;   /* DEVICE [env_height][env_width][C] equirectangular environment
                               map E of Eq. 7 sampled for empty pixels
                               (R29), or NULL -> constant `background`          */
    int32_t env_width, env_height;
    int32_t spatial_rendered;/* backward: 0 = ghost gradients (spatial gradients for ghosts only,
                               §4.3, Fig. 4); 1 = ghost gradients disabled, the §6.2 baseline
                               (L584-590): Eqs. 9-11 for the rendered points (R31)  */
    int32_t normal_culling; /* Eq. 5 (L208) normal culling, R32: 0 off; +1 keep points
                               with (R n).(R x + t) > 0 as printed; -1 keep < 0 (the flipped
                               orientation: outward normals facing the camera)              */
    int32_t shared_pyramid; /* point sharding over peer memory: 1 = the
                               keys / accum / count buffers of `views` are ONE pyramid shared by
                               every shard (e.g. the owner's, opened with adop_ipc_open); the
                               phases then do not clear them -- the owner calls
                               adop_clear_pyramid once per frame and the caller orders the
                               phases of all shards (depth of every shard before any blend,
                               every blend before the owner's resolve).  0 = private pyramid. */
} adop_params;

/* Buffers of one view (device).  See layouts above. */
typedef struct {
    float *image;
    float *count;
    uint64_t *keys;
    float *accum;
} adop_pyramid;

/* Pixels of one pyramid: sum_l ceil(w/2^l) * ceil(h/2^l).  Returns 0 on invalid sizes. */
ADOP_API int64_t adop_pyramid_pixels(int32_t width, int32_t height, int32_t layers);

/* Workspace bytes for calls over `n_views` views (cameras: host [n_views]) of `points`.
 * Layout: 4 KiB header | pose partials | backward pixel tables (per view and pixel one
 * row {min depth, count, sum_c G I, 0, G[C]} of 16 + 4 * roundup4(C) bytes) | record region |
 * chunk tables.
 * record_capacity: 16-byte slots of the record region (rounded up to 64-slot chunks).  The depth
 * pass fills it from the front with survivor records (one per (point, view, layer) hit of the
 * render set) and the backward sweep, when params->ghost_rate > 0, from the back with ghost
 * entries (2 slots per kept (ghost, view)); both are reserved per warp in chunks of 64 slots whose
 * unused slots are marked dead.  With more than 2 views every chunk holds one view's items and the
 * chunk tables (per chunk: 1 view byte + 2 x 4-byte order entries; plus 1 KiB) let the consumers
 * walk the lists view by view.  < 0 selects the worst case n * n_views * max(layers, 2) plus chunk
 * slack.  If the lists do not fit, the blend pass re-streams all points and the backward
 * re-renders them (correct, slower).
 * Bytes = 4096 + 2048 * 16 * 18 * 8 + tables + ceil(capacity / 64) * 1033 + 1024.
 * Errors: ADOP_ERR_INVALID_ARGUMENT (NULL pointers, n_views not in [1, 16], bad layers,
 * channels or camera sizes). */
ADOP_API adop_status adop_workspace_size(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                const adop_params *params, int64_t record_capacity, size_t *bytes);

/* Phase 1, depth-only render pass (§4.5; Eqs. 2-4, 12, min_z of Eq. 6):
 * sets keys to the sentinel for every view, then
 * atomically min-reduces the packed key of every render-set point into every
 * layer it lands on, and records the survivors in the workspace.
 * Caller-run collectives (point sharding) may min-reduce keys (as int64 or
 * uint64: the sentinel keeps both orders equal) before phase 2.
 * Errors: ADOP_ERR_INVALID_ARGUMENT, ADOP_ERR_WORKSPACE_TOO_SMALL, ADOP_ERR_CUDA. */
ADOP_API adop_status adop_forward_depth(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                               const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                               void *workspace, size_t workspace_bytes, void *stream);

/* Phase 2, accumulate (§4.5; fuzzy test Eq. 6, sums of Eq. 7):
 * sets accum and count to zero, then for every survivor of phase 1 that passes
 * z <= (1+alpha) * min_z against the (possibly globally reduced) keys, adds tau
 * to accum and 1 to count.  Caller-run collectives (point sharding) may
 * sum-reduce accum and count before phase 3.
 * Must follow adop_forward_depth with the same arguments and workspace. */
ADOP_API adop_status adop_forward_blend(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                               const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                               void *workspace, size_t workspace_bytes, void *stream);

/* Phase 3, normalize (Eq. 7): image = accum / count where count > 0,
 * else the background colour; writes the planar image of every layer. */
ADOP_API adop_status adop_forward_resolve(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                 const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                                 void *workspace, size_t workspace_bytes, void *stream);

/* Phase 3 over a pixel range (point sharding with a reduce-scatter, DESIGN.md section 8;
 * SURVEY §8(e)): as adop_forward_resolve, but only pyramid pixels [p0, p1) of every
 * view -- pixel p of the concatenated layers 0..L-1 (layout above) -- are normalized
 * and written; the rest of the image is left untouched.  p1 is clipped to each view's
 * pixel count.  After a reduce-scatter of accum and count, rank r resolves its own
 * slice.  Ranges whose ends are multiples of 4 (or p1 >= P) take the vector path.
 * Errors: ADOP_ERR_INVALID_ARGUMENT (p0 < 0 or p1 < p0), as adop_forward_resolve. */
ADOP_API adop_status adop_forward_resolve_range(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                       const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                                       int64_t p0, int64_t p1, void *workspace, size_t workspace_bytes, void *stream);

/* Phases 1-3 in order (single GPU). */
ADOP_API adop_status adop_rasterize_forward(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                   const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                                   void *workspace, size_t workspace_bytes, adop_comm *comm, void *stream);

/* Backward (§4.2-4.5): re-renders every point (L361) against the forward's
 * keys/count/accum/image (which must be unmodified) and the upstream gradient
 * grad_image[v] (device, image layout).  The re-render's work lists (rendered hits,
 * kept ghosts) are exactly the survivor records and ghost list the depth pass left in
 * the workspace: when the workspace still holds them for the same inputs (a
 * fingerprint of points, cameras, poses, params and pyramids), they are consumed
 * directly; otherwise (different inputs, an overflowed record region, or a forward on
 * the unaligned path) every point is re-projected.  Results are the same either way.
 * It produces
 *   d_feat [n][C]: sum over views/layers of G/|Lambda| for rendered points (ghosts 0),
 *   d_pos  [3][n]: ghost points only: R^T J^T g, g from Eqs. 9-11 (R14-R17) (rendered points
 *                  instead with params->spatial_rendered),
 *   d_pose [V][6]: sum over ghosts of (w, Xc x w), w = J^T g (Eq. 17 left increment),
 *   d_intrinsics [V][12]: sum over ghosts of (d(u0,v0)/d theta)^T g, theta = (fx, fy, cx, cy,
 *                 k1..k6, p1, p2) of the view's camera (the camera model C of Eq. 2, optimized by
 *                 the paper: Fig. 4); 0 for the distortion entries of a pinhole camera,
 *   d_env [env_height][env_width][C]: environment-map gradient, every empty pixel's G
 *                 scattered to its bilinear taps ("straightforward"); requires env_map.
 * With log_descriptors the texture gradient includes d exp(tau)/d tau and the ghosts' Eq. 11
 * uses the linear descriptor exp(tau).
 * Any of d_feat / d_pos / d_pose / d_intrinsics / d_env may be NULL.  params->grad_accumulate selects
 * overwrite or add.  Points, cameras, poses and params must equal the forward's.
 * Errors: ADOP_ERR_INVALID_ARGUMENT, ADOP_ERR_WORKSPACE_TOO_SMALL, ADOP_ERR_CUDA. */
ADOP_API adop_status adop_rasterize_backward(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                    const adop_pose *poses, const adop_params *params,
                                    const adop_pyramid *fwd_views, const float *const *grad_image,
                                    float *d_feat, float *d_pos, double *d_pose, double *d_intrinsics,
                                    float *d_env, void *workspace, size_t workspace_bytes, adop_comm *comm,
                                    void *stream);

/* Debug / parity: per point and view, bit l (l < L) = valid, in bounds and kept
 * by the discard test at layer l; bit 7 = ghost.  mask: device uint8 [V][n]. */
ADOP_API adop_status adop_point_masks(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                             const adop_pose *poses, const adop_params *params, uint8_t *mask, void *stream);

/* List statistics of `workspace` (synchronizes `stream`); any output may be NULL:
 * records: survivor-record slots of the last depth pass (including dead chunk tails),
 * ghost_entries: ghost-list entries of the last backward (including dead chunk tails),
 * overflowed: whether the depth pass's records did not fit the record region,
 * tiles_read: with tile_bounds, the 256-point tiles the last depth pass loaded. */
ADOP_API adop_status adop_workspace_stats(const void *workspace, size_t workspace_bytes, void *stream,
                                 int64_t *records, int64_t *ghost_entries, int32_t *overflowed,
                                 int64_t *tiles_read);

/* Bounding box of every 256-point tile of `points` (lo x, y, z, 0, hi x, y, z, 0; NaN coordinates
 * ignored): bounds = device float [ceil(n/256)][8], 16-byte aligned.  Enqueued on `stream`. */
ADOP_API adop_status adop_tile_bounds(const adop_points *points, float *bounds, void *stream);

/* A fresh NCCL unique id (128 bytes) on one rank, to be broadcast to the others (e.g. with
 * torch.distributed.broadcast_object_list).  Errors: ADOP_ERR_INVALID_ARGUMENT, ADOP_ERR_NCCL. */
ADOP_API adop_status adop_comm_unique_id(uint8_t id[128]);

/* Collective over nranks processes (one per GPU, the CURRENT device of the calling thread): mode
 * ADOP_SHARD_POINTS or ADOP_SHARD_VIEWS, flags 0 or ADOP_COMM_KEYS32.  Every rank calls it with the same
 * id.  The communicator owns its NCCL communicator and (with ADOP_COMM_KEYS32) a device scratch buffer of
 * the largest view's P int32 -- the only device memory the library allocates.  Errors:
 * ADOP_ERR_INVALID_ARGUMENT (rank not in [0, nranks), bad mode or flags), ADOP_ERR_CUDA, ADOP_ERR_NCCL. */
ADOP_API adop_status adop_comm_init(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t mode, int32_t flags,
                                    adop_comm **comm);

/* Frees the communicator (NULL: no-op).  The caller ensures no enqueued call still uses it. */
ADOP_API adop_status adop_comm_destroy(adop_comm *comm);

/* Host-only diagnostic of the OpenCV8 candidate window (no GPU work): the box [xlo, xhi] x [ylo, yhi]
 * in undistorted normalized coordinates that contains every point n with |n|^2 <= r2_max whose
 * distorted pixel (Eq. 2 with R6) lies in the all-layer window (-2^(L-1) - 2, w + 2^(L-1) + 2) x
 * (same for h); points outside it cannot land in any layer, so the depth and backward sweeps cull
 * them before the distortion model.  out[4] = (xlo, xhi, ylo, yhi); *valid = 0 when no window is
 * used for this camera (pinhole / fisheye, no finite r2_max, or an edge point failed to invert).
 * Errors: ADOP_ERR_INVALID_ARGUMENT (NULL pointers, bad camera or layers). */
ADOP_API adop_status adop_camera_window(const adop_camera *camera, int32_t layers, float out[4], int32_t *valid);

/* ---- Point sharding over peer memory (NVLink P2P / CUDA IPC) ---------- */

/* keys <- sentinel, accum <- 0, count <- 0 for every view of `views` (device buffers of
 * adop_pyramid_pixels(w, h, layers) pixels, C channels): the owner's once-per-frame reset of a
 * shared pyramid.  Enqueued on `stream`.  Errors: ADOP_ERR_INVALID_ARGUMENT, ADOP_ERR_CUDA. */
ADOP_API adop_status adop_clear_pyramid(int32_t n_views, const adop_camera *cameras, int32_t layers, int32_t channels,
                               const adop_pyramid *views, void *stream);

/* Export device memory to another process: `handle` (64 bytes, host) names the allocation that
 * contains `ptr`, `offset` is ptr's byte offset in it (cudaIpcGetMemHandle + the allocation base). */
ADOP_API adop_status adop_ipc_export(const void *ptr, unsigned char handle[64], uint64_t *offset);

/* Map an exported allocation into this process (peer access enabled lazily): *base = the mapped
 * allocation (pass it to adop_ipc_close), *ptr = base + offset.  One mapping per allocation and
 * process: the caller caches it (opening the same handle twice fails). */
ADOP_API adop_status adop_ipc_open(const unsigned char handle[64], uint64_t offset, void **base, void **ptr);

/* Unmap an allocation mapped by adop_ipc_open. */
ADOP_API adop_status adop_ipc_close(void *base);

/* ---- Preprocessing before the hot path (untimed setup) ------------- */

/* Scratch bytes of the preprocessing calls for n points and Morton blocks of `block` points. */
ADOP_API adop_status adop_prep_workspace_size(int64_t n, int32_t block, size_t *bytes);

/* Blocked Morton shuffle (§4.5; R34): positions quantized to 21 bits per
 * axis over the cloud's bounding box (fp32, pinned order), 63-bit Morton codes, stable sort by
 * (code, index), blocks of `block` points ordered by (hash(seed, block), block).  perm: device
 * int64 [n], perm[j] = the old index of the point that goes to position j.  points->n in [1, 2^31).
 * workspace: 256-byte aligned, adop_prep_workspace_size bytes.  Enqueued on `stream`. */
ADOP_API adop_status adop_blocked_morton_order(const adop_points *points, int32_t block, uint64_t seed, int64_t *perm,
                                      void *workspace, size_t workspace_bytes, void *stream);

/* dst.x[j] = src.x[perm[j]] for positions, radii, descriptors and normals present in both
 * (device buffers; dst must match src's n, channels and pos_stride; dst->pos etc. are written). */
ADOP_API adop_status adop_apply_order(const adop_points *src, const int64_t *perm, const adop_points *dst,
                             void *stream);

/* World radius r_world of every point "inside its local neighborhood" (§4.4; R33):
 * the median distance to its k nearest other points (1 <= k <= 32, n >= k + 1), floored at
 * 1e-9 x the bounding-box diagonal; exact (ring search over Morton cells).  radius: device [n]. */
ADOP_API adop_status adop_knn_radius(const adop_points *points, int32_t k, float *radius, void *workspace,
                            size_t workspace_bytes, void *stream);

/* Thread-local description of the last non-OK status ("" if none). */
ADOP_API const char *adop_last_error(void);

/* Library version string. */
ADOP_API const char *adop_version(void);

#ifdef __cplusplus
}
#endif

#endif /* ADOP_H */
