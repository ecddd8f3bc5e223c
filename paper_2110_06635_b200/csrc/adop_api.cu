// adop_api.cu -- host side of the C-ABI (include/adop.h): argument validation,
// kernel argument blocks, workspace layout and launch sequencing.
// No exception crosses the ABI; errors are reported as adop_status plus a
// thread-local message (adop_last_error).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <vector>

#include "adop_internal.h"

using namespace adop;

namespace {
thread_local char g_err[512] = "";
}  // namespace

// shared with adop_prep.cu: record the last error message (thread-local) and return s
adop_status adop::set_status(adop_status s, const char *msg) {
    std::snprintf(g_err, sizeof(g_err), "%s", msg ? msg : "");
    return s;
}

namespace {

adop_status fail(adop_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

adop_status ok() {
    g_err[0] = '\0';
    return ADOP_OK;
}

// hash salt (R11, R13): mix of (seed, stream, view)
uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
uint32_t salt_of(uint64_t seed, uint32_t stream, uint32_t view) {
    uint32_t s = mix32((uint32_t)seed + 0x9E3779B9U * (stream + 1U));
    s = mix32(s ^ (uint32_t)(seed >> 32));
    return mix32(s + 0x85EBCA6BU * (view + 1U));
}
constexpr uint32_t kStreamGhost = 1, kStreamDiscard = 2;

constexpr size_t kHeaderBytes = 4096;  // WsHeader at 0, PlaneTab[16] at 256, LayerDesc[16] at 2304
constexpr int64_t kRecordSlack = 1 << 20;  // >= resident warps x 256-slot record chunks
constexpr int kMaxBwdBlocks = 2048;
constexpr size_t kPartialBytes = (size_t)kMaxBwdBlocks * ADOP_MAX_VIEWS_PER_LAUNCH * 18 * sizeof(double);

int32_t layer_size(int32_t s, int l) { return (int32_t)((s + (1 << l) - 1) >> l); }

int device_sms() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = sms > 0 ? sms : 148;
    }
    return cached[dev];
}

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

adop_status check_points(const adop_points *pts, bool need_feat) {
    if (!pts) return fail(ADOP_ERR_INVALID_ARGUMENT, "points is NULL");
    if (pts->n < 0) return fail(ADOP_ERR_INVALID_ARGUMENT, "points->n = %lld < 0", (long long)pts->n);
    if (pts->global_offset < 0 || pts->global_offset + pts->n > (int64_t)4294967296LL)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "global_offset + n must be in [0, 2^32]");
    if (pts->channels < 1 || pts->channels > ADOP_MAX_CHANNELS)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "channels = %d not in [1, %d]", pts->channels, ADOP_MAX_CHANNELS);
    if (pts->n == 0) return ok();
    if (!pts->pos) return fail(ADOP_ERR_INVALID_ARGUMENT, "points->pos is NULL");
    if (!aligned(pts->pos, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "points->pos not 4-byte aligned");
    if (pts->pos_stride < pts->n) return fail(ADOP_ERR_INVALID_ARGUMENT, "pos_stride < n");
    if (pts->radius && !aligned(pts->radius, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "radius not aligned");
    if (!pts->radius && !(pts->radius_uniform >= 0.0f && std::isfinite(pts->radius_uniform)))
        return fail(ADOP_ERR_INVALID_ARGUMENT, "radius_uniform must be finite and >= 0");
    if (need_feat && !pts->feat) return fail(ADOP_ERR_INVALID_ARGUMENT, "points->feat is NULL");
    if (pts->feat && !aligned(pts->feat, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "feat not aligned");
    if (pts->normal && !aligned(pts->normal, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "normal not aligned");
    if (pts->tile_bounds && !aligned(pts->tile_bounds, 16))
        return fail(ADOP_ERR_INVALID_ARGUMENT, "tile_bounds not 16-byte aligned");
    return ok();
}

adop_status check_culling(const adop_points *pts, const adop_params *pr) {
    if (pr->normal_culling && pts->n > 0 && !pts->normal)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "normal_culling needs points->normal");
    return ok();
}

adop_status check_params(const adop_params *pr) {
    if (!pr) return fail(ADOP_ERR_INVALID_ARGUMENT, "params is NULL");
    if (pr->layers < 1 || pr->layers > ADOP_MAX_LAYERS)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "layers = %d not in [1, %d]", pr->layers, ADOP_MAX_LAYERS);
    if (!(pr->alpha >= 0.0f) || !std::isfinite(pr->alpha)) return fail(ADOP_ERR_INVALID_ARGUMENT, "alpha must be >= 0");
    if (pr->discard && (!(pr->gamma > 0.0f) || !std::isfinite(pr->gamma)))
        return fail(ADOP_ERR_INVALID_ARGUMENT, "gamma must be > 0 with discard on");
    if (!(pr->ghost_rate >= 0.0f && pr->ghost_rate < 1.0f))
        return fail(ADOP_ERR_INVALID_ARGUMENT, "ghost_rate must be in [0, 1)");
    if (!(pr->z_near >= 0.0f) || !std::isfinite(pr->z_near))
        return fail(ADOP_ERR_INVALID_ARGUMENT, "z_near must be finite and >= 0");
    if (pr->view_id_base < 0) return fail(ADOP_ERR_INVALID_ARGUMENT, "view_id_base < 0");
    if (pr->env_map) {
        if (pr->env_width < 1 || pr->env_height < 1)
            return fail(ADOP_ERR_INVALID_ARGUMENT, "env_map: width/height < 1");
        if ((int64_t)pr->env_width * pr->env_height >= (int64_t)1 << 31)
            return fail(ADOP_ERR_INVALID_ARGUMENT, "env_map too large");
        if (!aligned(pr->env_map, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "env_map misaligned");
    }
    return ok();
}

adop_status check_camera(const adop_camera *c, int v, int layers) {
    if (c->width < 1 || c->height < 1) return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: width/height < 1", v);
    if (c->model == ADOP_FISHEYE && !(c->r2_max > 0.0f && c->r2_max <= 3.14159265f))
        return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: fisheye theta_max (r2_max) must be in (0, pi]", v);
    if (c->model != ADOP_PINHOLE && c->model != ADOP_OPENCV8 && c->model != ADOP_FISHEYE)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: unknown camera model %d", v, c->model);
    if (!std::isfinite(c->fx) || !std::isfinite(c->fy) || !std::isfinite(c->cx) || !std::isfinite(c->cy))
        return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: non-finite intrinsics", v);
    if (c->model == ADOP_OPENCV8) {
        for (int i = 0; i < 6; ++i)
            if (!std::isfinite(c->k[i])) return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: non-finite k", v);
        if (!std::isfinite(c->p[0]) || !std::isfinite(c->p[1]))
            return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: non-finite p", v);
        if (!(c->r2_max > 0.0f)) return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: r2_max must be > 0", v);
    }
    int64_t P = adop_pyramid_pixels(c->width, c->height, layers);
    if (P <= 0 || P >= (int64_t)1 << 31) return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: pyramid too large", v);
    return ok();
}

adop_status check_views(int32_t n_views, const adop_camera *cams, const adop_pose *poses, const adop_params *pr,
                        const adop_pyramid *views, int C, bool need_pyr) {
    if (n_views < 1 || n_views > ADOP_MAX_VIEWS_PER_LAUNCH)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "n_views = %d not in [1, %d]", n_views, ADOP_MAX_VIEWS_PER_LAUNCH);
    if (!cams || !poses) return fail(ADOP_ERR_INVALID_ARGUMENT, "cameras/poses is NULL");
    if (need_pyr && !views) return fail(ADOP_ERR_INVALID_ARGUMENT, "views is NULL");
    for (int v = 0; v < n_views; ++v) {
        adop_status s = check_camera(&cams[v], v, pr->layers);
        if (s) return s;
        for (int i = 0; i < 9; ++i)
            if (!std::isfinite(poses[v].R[i])) return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: non-finite R", v);
        for (int i = 0; i < 3; ++i)
            if (!std::isfinite(poses[v].t[i])) return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: non-finite t", v);
        if (!need_pyr) continue;
        const adop_pyramid &py = views[v];
        if (!py.image || !py.count || !py.keys || !py.accum)
            return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: NULL pyramid buffer", v);
        if (!aligned(py.keys, 8) || !aligned(py.count, 4) || !aligned(py.image, 4) || !aligned(py.accum, 4))
            return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: misaligned pyramid buffer", v);
    }
    (void)C;
    return ok();
}

struct Ws {
    WsHeader *hdr;
    double *partials;
    void *tables;
    Record *records;
    int64_t capacity;   // record slots, a multiple of kListChunk
    uint8_t *cview;     // chunk tables of the multi-view lists (after the record region)
    uint32_t *corder0, *corder1, *ccount;
};

// Bytes of the record region per kListChunk-slot chunk: the slots, the chunk's view byte and its two order
// entries (front / back list); plus a fixed tail for the counts and alignment.
constexpr size_t kChunkBytes = (size_t)kListChunk * sizeof(Record) + 1 + 2 * sizeof(uint32_t);
constexpr size_t kListTail = 1024;

// Backward pixel tables: per view and pixel one row {m, count, S, 0, G[C]} of 16 + 4 * roundup4(C)
// bytes (k_bwd_prep), 256-B rounded.
size_t table_bytes(int32_t n_views, const adop_camera *cams, int32_t layers, int32_t channels) {
    size_t t = 0;
    const size_t row = 16u + 4u * (size_t)((channels + 3) & ~3);
    for (int v = 0; v < n_views; ++v) t += (size_t)adop_pyramid_pixels(cams[v].width, cams[v].height, layers) * row;
    return (t + 255) / 256 * 256;
}

// Workspace layout: [header 4 KiB | pose partials | backward pixel tables | record region (16-B slots)].
adop_status carve_workspace(void *ws, size_t bytes, size_t tbytes, Ws &out) {
    if (!ws) return fail(ADOP_ERR_INVALID_ARGUMENT, "workspace is NULL");
    if (!aligned(ws, 256)) return fail(ADOP_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
    const size_t fixed = kHeaderBytes + kPartialBytes + tbytes;
    if (bytes < fixed)
        return fail(ADOP_ERR_WORKSPACE_TOO_SMALL, "workspace of %zu bytes < minimum %zu for these views", bytes, fixed);
    char *b = static_cast<char *>(ws);
    out.hdr = reinterpret_cast<WsHeader *>(b);
    out.partials = reinterpret_cast<double *>(b + kHeaderBytes);
    out.tables = b + kHeaderBytes + kPartialBytes;
    out.records = reinterpret_cast<Record *>(b + fixed);
    const size_t avail = bytes - fixed;
    const int64_t nch = avail > kListTail ? (int64_t)((avail - kListTail) / kChunkBytes) : 0;
    out.capacity = nch * kListChunk;
    char *t = b + fixed + (size_t)out.capacity * sizeof(Record);
    out.cview = reinterpret_cast<uint8_t *>(t);
    t += (nch + 15) / 16 * 16;
    out.corder0 = reinterpret_cast<uint32_t *>(t);
    out.corder1 = out.corder0 + nch;
    t += (size_t)nch * 2 * sizeof(uint32_t);
    t = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(t) + 255) & ~(uintptr_t)255);
    out.ccount = reinterpret_cast<uint32_t *>(t);  // 2 x 64 u32, within kListTail
    return ok();
}

// Fingerprint of a call's inputs: the backward consumes the depth pass's lists only if its own
// fingerprint equals the one the depth pass stored in the workspace header (FNV-1a, never 0).
struct Fnv {
    uint64_t h = 1469598103934665603ull;
    void add(const void *p, size_t n) {
        const unsigned char *c = static_cast<const unsigned char *>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
    }
    template <typename T>
    void put(const T &v) { add(&v, sizeof(v)); }
};
uint64_t call_tag(const adop_points *pts, int32_t n_views, const adop_camera *cams, const adop_pose *poses,
                  const adop_params *pr, const adop_pyramid *views, size_t ws_bytes) {
    Fnv f;
    f.put(pts->n); f.put(pts->global_offset); f.put(pts->pos_stride); f.put(pts->pos); f.put(pts->radius);
    f.put(pts->radius_uniform); f.put(pts->channels); f.put(n_views); f.put(ws_bytes);
    f.add(cams, sizeof(adop_camera) * (size_t)n_views);
    f.add(poses, sizeof(adop_pose) * (size_t)n_views);
    f.put(pr->layers); f.put(pr->alpha); f.put(pr->discard); f.put(pr->gamma); f.put(pr->ghost_rate);
    f.put(pr->z_near); f.put(pr->seed); f.put(pr->view_id_base); f.put(pr->log_descriptors);
    f.put(pr->env_map); f.put(pr->env_width); f.put(pr->env_height); f.put(pr->normal_culling);
    f.put(pts->normal);
    for (int v = 0; views && v < n_views; ++v) f.put(views[v].keys);
    return f.h | 1ull;
}

// ---- OpenCV8 image window in undistorted normalized coordinates (the candidate window test) ----
// W = { n : |n|^2 <= r2_max, the distortion map d(n) of R6 lands in the pixel window (ulo, uhi) x (vlo, vhi) }.
// Its bounding box [xlo, xhi] x [ylo, yhi] is found from W's boundary, which lies on the valid circle
// |n|^2 = r2_max (sampled, kept where d(n) is in the window) and on the preimages of the window's four edges
// (sampled, inverted by Newton's method, kept inside the disk); the box is widened by the largest distance
// between consecutive boundary samples.  Every point whose exact projection lands in some layer satisfies
// xlo Z <= X <= xhi Z, ylo Z <= Y <= yhi Z (the pixel window already holds a 2-pixel margin over the fp32
// projection's rounding).  ok = false (no window test) if an edge point inside the distorted disk fails to
// invert, or the camera has no finite valid radius.
struct NormWindow {
    double xlo, xhi, ylo, yhi;
    bool ok;
};

static void distort_jac(const adop_camera &c, double xn, double yn, double &xd, double &yd, double J[2][2]) {
    const double k1 = c.k[0], k2 = c.k[1], k3 = c.k[2], k4 = c.k[3], k5 = c.k[4], k6 = c.k[5];
    const double p1 = c.p[0], p2 = c.p[1];
    const double r2 = xn * xn + yn * yn;
    const double num = 1.0 + r2 * (k1 + r2 * (k2 + r2 * k3)), den = 1.0 + r2 * (k4 + r2 * (k5 + r2 * k6));
    const double rad = num / den;
    const double dnum = k1 + r2 * (2.0 * k2 + 3.0 * r2 * k3), dden = k4 + r2 * (2.0 * k5 + 3.0 * r2 * k6);
    const double drad = (dnum * den - num * dden) / (den * den);  // d rad / d r^2
    xd = xn * rad + 2.0 * p1 * xn * yn + p2 * (r2 + 2.0 * xn * xn);
    yd = yn * rad + p1 * (r2 + 2.0 * yn * yn) + 2.0 * p2 * xn * yn;
    J[0][0] = rad + 2.0 * xn * xn * drad + 2.0 * p1 * yn + 6.0 * p2 * xn;
    J[0][1] = 2.0 * xn * yn * drad + 2.0 * p1 * xn + 2.0 * p2 * yn;
    J[1][0] = J[0][1];
    J[1][1] = rad + 2.0 * yn * yn * drad + 6.0 * p1 * yn + 2.0 * p2 * xn;
}

// d(n) = q by damped Newton from (x, y); true if it converged (the result may lie outside the valid disk).
static bool newton_inverse(const adop_camera &c, double qx, double qy, double R, double R2, double &x, double &y) {
    for (int it = 0; it < 60; ++it) {
        double xd, yd, J[2][2];
        distort_jac(c, x, y, xd, yd, J);
        const double rx = xd - qx, ry = yd - qy;
        if (std::hypot(rx, ry) <= 1e-12 * (1.0 + std::hypot(qx, qy))) return true;
        const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        if (!(std::fabs(det) > 1e-300)) return false;
        double sx = (J[1][1] * rx - J[0][1] * ry) / det, sy = (-J[1][0] * rx + J[0][0] * ry) / det;
        const double sn = std::hypot(sx, sy), lim = 0.25 * (1.0 + R);
        if (sn > lim) {  // damped step
            sx *= lim / sn;
            sy *= lim / sn;
        }
        x -= sx;
        y -= sy;
        if (!(x * x + y * y <= 16.0 * R2)) return false;  // left the model's domain
    }
    return false;
}

static NormWindow compute_window(const adop_camera &c, double ulo, double uhi, double vlo, double vhi) {
    NormWindow w{0, 0, 0, 0, false};
    const double R2 = c.r2_max;
    if (!(R2 > 0.0) || !std::isfinite(R2)) return w;
    double ax = (ulo - c.cx) / c.fx, bx = (uhi - c.cx) / c.fx, ay = (vlo - c.cy) / c.fy, by = (vhi - c.cy) / c.fy;
    if (ax > bx) std::swap(ax, bx);
    if (ay > by) std::swap(ay, by);
    double lo[2] = {INFINITY, INFINITY}, hi[2] = {-INFINITY, -INFINITY}, gap = 0.0;
    auto add = [&](double x, double y) {
        lo[0] = std::fmin(lo[0], x); hi[0] = std::fmax(hi[0], x);
        lo[1] = std::fmin(lo[1], y); hi[1] = std::fmax(hi[1], y);
    };
    // the valid circle: kept where it maps into the window
    const int NC = 4096;
    const double R = std::sqrt(R2);
    std::vector<double> cx(NC), cy(NC);  // the distorted circle, a closed polygon around the distorted disk
    for (int i = 0; i < NC; ++i) {
        const double th = 2.0 * M_PI * i / NC, x = R * std::cos(th), y = R * std::sin(th);
        double xd, yd, J[2][2];
        distort_jac(c, x, y, xd, yd, J);
        cx[i] = xd;
        cy[i] = yd;
        if (xd >= ax && xd <= bx && yd >= ay && yd <= by) add(x, y);
    }
    // q inside the distorted disk (even-odd test against the polygon scaled by 1 + 1e-5 about the origin)
    auto in_image_of_disk = [&](double qx, double qy) {
        const double s = 1.0 / (1.0 + 1e-5);
        qx *= s;
        qy *= s;
        bool in = false;
        for (int i = 0, j = NC - 1; i < NC; j = i++)
            if ((cy[i] > qy) != (cy[j] > qy) && qx < (cx[j] - cx[i]) * (qy - cy[i]) / (cy[j] - cy[i]) + cx[i]) in = !in;
        return in;
    };
    gap = 2.0 * M_PI * R / NC;
    // the window's edges, inverted point by point (continuation from the previous solution)
    const int NE = 1024;
    for (int e = 0; e < 4; ++e) {
        double px = 0, py = 0;
        bool prev = false;
        for (int i = 0; i <= NE; ++i) {
            const double t = (double)i / NE;
            const double qx = e == 0 ? ax + t * (bx - ax) : (e == 1 ? ax + t * (bx - ax) : (e == 2 ? ax : bx));
            const double qy = e == 0 ? ay : (e == 1 ? by : ay + t * (by - ay));
            // Newton from the previous edge point's preimage, then (near the fold at the valid radius, where a
            // second preimage outside the disk exists) from q itself and from points pulled towards the centre
            double x = 0.0, y = 0.0;
            bool conv = false;
            for (int start = 0; start < 4 && !(conv && x * x + y * y <= R2 * (1.0 + 1e-3)); ++start) {
                if (start == 0 && !prev) continue;
                const double sc = start <= 1 ? 1.0 : (start == 2 ? 0.9 : 0.6);
                x = start == 0 ? px : sc * qx;
                y = start == 0 ? py : sc * qy;
                conv = newton_inverse(c, qx, qy, R, R2, x, y);
            }
            // at the fold (the valid radius is where the radial map stops increasing) a window point just inside
            // the distorted disk can have its inner preimage numerically indistinguishable from the outer one:
            // an outer preimage within 1e-3 of the circle is taken, and the box widened by twice its distance
            const double r2 = x * x + y * y;
            const bool in = conv && r2 <= R2 * (1.0 + 1e-3);
            if (in && r2 > R2) gap = std::fmax(gap, 2.0 * (std::sqrt(r2) - R));
            if (in) {
                add(x, y);
                if (prev) gap = std::fmax(gap, std::hypot(x - px, y - py));
                px = x;
                py = y;
            } else if (in_image_of_disk(qx, qy)) {
                return w;  // inside the distorted disk but not inverted: no window test for this camera
            }
            prev = in;
        }
    }
    if (!(lo[0] <= hi[0])) {  // nothing of the valid disk lands in the window: an empty window
        w.xlo = w.ylo = 1.0;
        w.xhi = w.yhi = -1.0;
        w.ok = true;
        return w;
    }
    const double m = 2.0 * gap + 1e-6;
    w.xlo = lo[0] - m;
    w.xhi = hi[0] + m;
    w.ylo = lo[1] - m;
    w.yhi = hi[1] + m;
    w.ok = true;
    return w;
}

// compute_window of a camera, cached by the camera's bytes and the window (refined intrinsics recompute it)
static NormWindow camera_window(const adop_camera &c, float ulo, float uhi, float vlo, float vhi) {
    struct Entry {
        adop_camera cam;
        float win[4];
        NormWindow w;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    const float win[4] = {ulo, uhi, vlo, vhi};
    {
        std::lock_guard<std::mutex> g(mu);
        for (const Entry &e : cache)
            if (!std::memcmp(&e.cam, &c, sizeof(c)) && !std::memcmp(e.win, win, sizeof(win))) return e.w;
    }
    const NormWindow w = compute_window(c, ulo, uhi, vlo, vhi);
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() >= 256) cache.erase(cache.begin());
    cache.push_back(Entry{c, {ulo, uhi, vlo, vhi}, w});
    return w;
}

// ADOP_WINDOW=0 disables the OpenCV8 window test (A/B measurements)
static bool window_test_enabled() {
    static int env = -1;
    if (env < 0) {
        const char *e = std::getenv("ADOP_WINDOW");
        env = e ? std::atoi(e) : 1;
    }
    return env != 0;
}

bool vec_path(const adop_points *pts) {
    return pts->n > 0 && aligned(pts->pos, 16) && pts->pos_stride % 4 == 0 && (!pts->radius || aligned(pts->radius, 16));
}

void fill_args(RasterArgs &a, const adop_points *pts, int32_t n_views, const adop_camera *cams,
               const adop_pose *poses, const adop_params *pr, const adop_pyramid *views, const Ws *ws) {
    std::memset(&a, 0, sizeof(a));
    a.res_p0 = 0;
    a.res_p1 = INT64_MAX;  // adop_forward_resolve: every pixel
    a.x = pts->pos;
    a.y = pts->pos ? pts->pos + pts->pos_stride : nullptr;
    a.z = pts->pos ? pts->pos + 2 * pts->pos_stride : nullptr;
    a.radius = pts->radius;
    a.radius_uniform = pts->radius_uniform;
    a.feat = pts->feat;
    a.n = pts->n;
    a.ntiles = (int32_t)((pts->n + 255) / 256);
    a.nfull = (int32_t)(pts->n / 256);
    a.goff = (uint32_t)pts->global_offset;
    a.channels = pts->channels;
    a.layers = pr->layers;
    a.nviews = n_views;
    a.onepa = 1.0f + pr->alpha;
    a.gamma = pr->gamma;
    a.z_near = pr->z_near;
    a.discard = pr->discard ? 1 : 0;
    a.ghost_thr = (uint32_t)std::floor((double)pr->ghost_rate * 16777216.0);
    a.ghost_salt = salt_of(pr->seed, kStreamGhost, 0u);
    a.grad_accumulate = pr->grad_accumulate ? 1 : 0;
    {   // tile scheduling of the sweeps (bit 0 depth, bit 1 backward): static round-robin streams the cloud
        // as one contiguous front; dynamic claiming balances irregular (backward) work.  ADOP_TILES overrides.
        static int mode = -1;
        if (mode < 0) {
            const char *e = std::getenv("ADOP_TILES");
            mode = e ? std::atoi(e) : 0;
        }
        a.dyn_tiles = mode;
    }
    for (int c = 0; c < pts->channels; ++c) a.bg[c] = pr->background ? pr->background[c] : 0.0f;
    a.log_desc = pr->log_descriptors ? 1 : 0;
    a.spatial_rendered = pr->spatial_rendered ? 1 : 0;
    a.normal_cull = pr->normal_culling > 0 ? 1 : (pr->normal_culling < 0 ? -1 : 0);
    a.clear_pyr = pr->shared_pyramid ? 0 : 1;
    a.nrm = pts->normal;
    a.tbounds = pts->tile_bounds;
    a.nrm_stride = pts->pos_stride;
    if (!pts->normal) a.normal_cull = 0;
    a.env = pr->env_map;
    a.env_w = pr->env_map ? pr->env_width : 0;
    a.env_h = pr->env_map ? pr->env_height : 0;
    if (ws) {
        a.hdr = ws->hdr;
        a.planes = reinterpret_cast<PlaneTab *>(reinterpret_cast<char *>(ws->hdr) + 256);
        a.ldesc = reinterpret_cast<LayerDesc *>(reinterpret_cast<char *>(ws->hdr) + 2304);
        static_assert(256 + ADOP_MAX_VIEWS_PER_LAUNCH * sizeof(PlaneTab) <= 2304, "header layout");
        static_assert(2304 + ADOP_MAX_VIEWS_PER_LAUNCH * sizeof(LayerDesc) <= kHeaderBytes, "header layout");
        a.records = ws->records;
        a.rec_capacity = ws->capacity;
        a.cview = ws->cview;
        a.corder[0] = ws->corder0;
        a.corder[1] = ws->corder1;
        a.ccount = ws->ccount;
        // per-view chunk lists for multi-view launches (the chunk slot index must fit 32 bits)
        // (only for large launches: the chunk ordering costs three small launches, more than the view-major
        // consumers save on configs[1]'s 4M point-views; configs[4] has 800M)
        const bool large = pts->n * (int64_t)n_views >= ((int64_t)1 << 26);
        a.mv_lists = (n_views > 2 && vec_path(pts) && ws->capacity >= 64 * kListChunk &&
                      ws->capacity < ((int64_t)1 << 32) - 256) ? (large ? 1 : 2) : 0;  // 2: small launch
        {
            // ADOP_MV_LISTS (A/B measurements, tests): bit 0 lists on, bit 1 view-major texture consumer, bit 2
            // view-major ghost consumer, bit 3 also for small launches.  Default 5: the texture gradient keeps the
            // lists' chunk order, in which a point's records of different views sit close together (its d_feat
            // row is reused), while the blend and the ghost consumer gain more from one view's pixel state
            // staying in L2.
            static int env = -1;
            if (env < 0) {
                const char *e = std::getenv("ADOP_MV_LISTS");
                env = e ? std::atoi(e) : 5;
            }
            const bool on = a.mv_lists == 1 || (a.mv_lists == 2 && (env & 8));
            a.mv_lists = (on && (env & 1)) ? (env & 7) : 0;
        }
        a.tables = ws->tables;
        a.pose_partials = ws->partials;
    }
    const float lmax = (float)(1 << (pr->layers - 1));
    for (int v = 0; v < n_views; ++v) {
        ViewDesc &d = a.v[v];
        const adop_camera &c = cams[v];
        std::memcpy(d.R, poses[v].R, sizeof(d.R));
        std::memcpy(d.t, poses[v].t, sizeof(d.t));
        d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy;
        d.model = c.model;
        if (c.model == ADOP_OPENCV8) {
            std::memcpy(d.k, c.k, sizeof(d.k));
            std::memcpy(d.p, c.p, sizeof(d.p));
            d.r2_max = c.r2_max;
            d.r2cull = std::isinf(c.r2_max) ? c.r2_max : (float)((double)c.r2_max * (1.0 + 1.0 / 4096.0));
        } else if (c.model == ADOP_FISHEYE) {
            // R35: r2_max holds theta_max; up to 1.5 rad the pre-cull is the cone X^2 + Y^2 <= tan^2 Z^2 (with
            // slack for the 1e-7-accurate atan), beyond it (a field of view near or over 180 degrees) none
            d.r2_max = c.r2_max;
            const double tt = std::tan((double)c.r2_max);
            d.r2cull = c.r2_max <= 1.5f ? (float)(tt * tt * (1.0 + 1.0 / 1024.0)) : INFINITY;
        } else {
            d.r2_max = INFINITY;
            d.r2cull = INFINITY;
        }
        d.feff = (c.fx + c.fy) * 0.5f;
        // conservative window over all layers: u0 in (-2^(L-1)/2, w + 2^(L-1)) plus margin
        d.ulo = -lmax - 2.0f;
        d.uhi = (float)c.width + lmax + 2.0f;
        d.vlo = -lmax - 2.0f;
        d.vhi = (float)c.height + lmax + 2.0f;
        d.wn_on = 0;
        if (c.model == ADOP_OPENCV8 && window_test_enabled()) {
            // OpenCV8: the image window in undistorted normalized coordinates (camera_window), widened by 1e-4
            // relative so the fp32 test X <= xhi Z of the candidate path is conservative
            const NormWindow w = camera_window(c, d.ulo, d.uhi, d.vlo, d.vhi);
            if (w.ok) {
                const double b[4] = {w.xlo, w.xhi, w.ylo, w.yhi};
                for (int k = 0; k < 4; ++k)
                    d.wn[k] = (float)(b[k] + (k & 1 ? 1.0 : -1.0) * 1e-4 * (1.0 + std::fabs(b[k])));
                d.wn_on = 1;
            }
        }
        // Margin of the FMA-evaluated pre-cull: |Xf - Xp| <= 2^-20 (|x|+|y|+|z| + max|t|) for the FMA and
        // the pinned evaluations of R x + t (|R| <= 1); the pre-cull combinations add at most
        // (|f| + |c| + |bound|) times that plus their own rounding, so 2^-18 (...) is conservative.
        {
            const double T = std::fmax(std::fabs((double)poses[v].t[0]),
                                       std::fmax(std::fabs((double)poses[v].t[1]), std::fabs((double)poses[v].t[2])));
            double S = 1.0;
            if (c.model == ADOP_PINHOLE) {
                S = std::fmax(std::fabs((double)c.fx), std::fabs((double)c.fy)) +
                    std::fmax(std::fabs((double)c.cx), std::fabs((double)c.cy)) +
                    std::fmax(std::fmax(std::fabs((double)d.ulo), std::fabs((double)d.uhi)),
                              std::fmax(std::fabs((double)d.vlo), std::fabs((double)d.vhi)));
            }
            const double K = std::ldexp(1.0, -18) * S * 1.02;
            d.fk = (float)K;
            d.fkt = (float)(K * (T + 1e-30) * 1.02);
        }
        // World-space planes for the per-warp bounding-box cull: camera-space
        // half-spaces ncam . Xc + dc >= 0 that every point passing the exact test satisfies with slack,
        // mapped to world space n = R^T ncam, d = ncam . t + dc.
        {
            double nc[5][3] = {{0}}, dc[5] = {0, 0, 0, 0, -(double)pr->z_near};
            if (c.model == ADOP_PINHOLE) {
                const double fx = c.fx, fy = c.fy, cx = c.cx, cy = c.cy;
                const double ncam[4][3] = {{fx, 0, cx - d.ulo}, {-fx, 0, d.uhi - cx},
                                           {0, fy, cy - d.vlo}, {0, -fy, d.vhi - cy}};
                std::memcpy(nc, ncam, sizeof(ncam));
            } else if (!std::isinf(d.r2cull)) {
                const double sr = std::sqrt((double)d.r2cull) * (1.0 + 1.0 / 1024.0);
                // the valid cone |X|, |Y| <= sr Z, tightened to the image window in normalized coordinates
                double xlo = -sr, xhi = sr, ylo = -sr, yhi = sr;
                if (c.model == ADOP_OPENCV8 && d.wn_on) {
                    xlo = std::fmax(xlo, (double)d.wn[0]);
                    xhi = std::fmin(xhi, (double)d.wn[1]);
                    ylo = std::fmax(ylo, (double)d.wn[2]);
                    yhi = std::fmin(yhi, (double)d.wn[3]);
                }
                const double ncam[4][3] = {{1, 0, -xlo}, {-1, 0, xhi}, {0, 1, -ylo}, {0, -1, yhi}};
                std::memcpy(nc, ncam, sizeof(ncam));
            } else {
                for (int k = 0; k < 4; ++k) dc[k] = 1.0;  // no lateral bound
            }
            nc[4][2] = 1.0;
            d.zplane = 1;
            d.zoff = pr->z_near;
            if (c.model == ADOP_FISHEYE) {  // the depth is the distance: valid points only have Z >= 0 (narrow)
                dc[4] = 0.0;
                d.zoff = 0.0f;
                if (std::isinf(d.r2cull)) {  // wide: no half-space at all
                    nc[4][2] = 0.0;
                    dc[4] = 1.0;
                    d.zplane = 0;
                }
            }
            const double T = std::fabs((double)poses[v].t[0]) + std::fabs((double)poses[v].t[1]) +
                             std::fabs((double)poses[v].t[2]);
            const float *R = poses[v].R;
            for (int k = 0; k < 5; ++k) {
                double n[3], dd = dc[k], l1 = 0.0;
                for (int ax = 0; ax < 3; ++ax)
                    n[ax] = (double)R[0 + ax] * nc[k][0] + (double)R[3 + ax] * nc[k][1] + (double)R[6 + ax] * nc[k][2];
                for (int r = 0; r < 3; ++r) {
                    dd += nc[k][r] * (double)poses[v].t[r];
                    l1 += std::fabs(nc[k][r]);
                }
                for (int ax = 0; ax < 3; ++ax) d.pl[k][ax] = (float)n[ax];
                d.pl[k][3] = (float)dd;
                // margin m = kb0 * B + kb1, B = sum_a max|p_a| over the box: the pinned-vs-real deviation
                // of Xc (2^-18 |ncam|_1 (B + T), x4 slack) plus the fp32 evaluation of the plane (2^-16 |n|_1 B
                // + 2^-16 |d|, ~10x the rounding bound)
                const double n1 = std::fabs(n[0]) + std::fabs(n[1]) + std::fabs(n[2]);
                const double ck = std::ldexp(1.0, -18) * l1 * 1.02;
                d.pm[k][0] = (float)((ck + std::ldexp(1.0, -16) * n1) * 1.02);
                d.pm[k][1] = (float)((ck * T + std::ldexp(1.0, -16) * std::fabs(dd)) * 1.02 + 1e-30);
            }
        }
        d.discard_salt = salt_of(pr->seed, kStreamDiscard, (uint32_t)(pr->view_id_base + v));
        int32_t off = 0;
        for (int l = 0; l < ADOP_MAX_LAYERS; ++l) {
            if (l < pr->layers) {
                d.wl[l] = layer_size(c.width, l);
                d.hl[l] = layer_size(c.height, l);
                d.off[l] = off;
                off += d.wl[l] * d.hl[l];
            } else {
                d.wl[l] = d.hl[l] = 0;
                d.off[l] = off;
            }
        }
        d.pixels = off;
        if (views) {
            d.keys = views[v].keys;
            d.accum = views[v].accum;
            d.count = views[v].count;
            d.image = views[v].image;
        }
    }
}

// 2-D TMA descriptor over the x/y/z rows (dims {n, 3}, row stride pos_stride * 4 bytes, box 256 x 3).
// Resolved through the runtime's driver entry point (no libcuda link); on any failure the kernels fall
// back to one 1-D bulk copy per row.
void encode_pos_tmap(RasterArgs &a, const adop_points *pts) {
    a.use_tmap = 0;
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
        else
            cudaGetLastError();
    }
    if (!encode || pts->n < 256 || pts->n >= ((int64_t)1 << 31)) return;
    const cuuint64_t dims[2] = {(cuuint64_t)pts->n, 3};
    const cuuint64_t strides[1] = {(cuuint64_t)pts->pos_stride * sizeof(float)};
    const cuuint32_t box[2] = {256, 3};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(pts->pos), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.use_tmap = r == CUDA_SUCCESS ? 1 : 0;
}


adop_status cuda_status(int err, const char *what) {
    if (err != cudaSuccess) return fail(ADOP_ERR_CUDA, "%s: %s", what, cudaGetErrorString((cudaError_t)err));
    return ok();
}

adop_status prologue(const adop_points *points, int32_t n_views, const adop_camera *cameras, const adop_pose *poses,
                     const adop_params *params, const adop_pyramid *views, void *workspace, size_t workspace_bytes,
                     bool need_feat, Ws &ws) {
    adop_status s;
    if ((s = check_params(params))) return s;
    if ((s = check_points(points, need_feat))) return s;
    if ((s = check_culling(points, params))) return s;
    if ((s = check_views(n_views, cameras, poses, params, views, points->channels, true))) return s;
    if ((s = carve_workspace(workspace, workspace_bytes,
                             table_bytes(n_views, cameras, params->layers, points->channels), ws)))
        return s;
    cudaError_t pending = cudaGetLastError();
    if (pending != cudaSuccess) return fail(ADOP_ERR_CUDA, "pending CUDA error: %s", cudaGetErrorString(pending));
    return ok();
}

bool uniform_model(int32_t n_views, const adop_camera *cams, int &model) {
    model = cams[0].model;
    for (int v = 1; v < n_views; ++v)
        if (cams[v].model != model) return false;
    return true;
}

}  // namespace

extern "C" {

int64_t adop_pyramid_pixels(int32_t width, int32_t height, int32_t layers) {
    if (width < 1 || height < 1 || layers < 1 || layers > ADOP_MAX_LAYERS) return 0;
    int64_t t = 0;
    for (int l = 0; l < layers; ++l) t += (int64_t)layer_size(width, l) * layer_size(height, l);
    return t;
}

adop_status adop_workspace_size(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                const adop_params *params, int64_t record_capacity, size_t *bytes) {
    if (!points || !params || !bytes || !cameras) return fail(ADOP_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_views < 1 || n_views > ADOP_MAX_VIEWS_PER_LAUNCH)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "n_views = %d not in [1, %d]", n_views, ADOP_MAX_VIEWS_PER_LAUNCH);
    if (params->layers < 1 || params->layers > ADOP_MAX_LAYERS) return fail(ADOP_ERR_INVALID_ARGUMENT, "bad layers");
    if (points->n < 0) return fail(ADOP_ERR_INVALID_ARGUMENT, "n < 0");
    if (points->channels < 1 || points->channels > ADOP_MAX_CHANNELS)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "channels = %d not in [1, %d]", points->channels, ADOP_MAX_CHANNELS);
    for (int v = 0; v < n_views; ++v)
        if (adop_pyramid_pixels(cameras[v].width, cameras[v].height, params->layers) <= 0)
            return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: bad width/height", v);
    // worst case n*V*max(L, 2) (a ghost entry takes 2 slots) plus slack for partially filled per-warp chunks
    const int64_t per = params->layers > 2 ? params->layers : 2;
    int64_t cap = record_capacity >= 0 ? record_capacity : points->n * (int64_t)n_views * per + kRecordSlack;
    const size_t nch = (size_t)((cap + kListChunk - 1) / kListChunk);
    *bytes = kHeaderBytes + kPartialBytes + table_bytes(n_views, cameras, params->layers, points->channels) +
             nch * kChunkBytes + kListTail;
    return ok();
}

adop_status adop_forward_depth(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                               const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                               void *workspace, size_t workspace_bytes, void *stream) {
    Ws ws;
    adop_status s = prologue(points, n_views, cameras, poses, params, views, workspace, workspace_bytes, false, ws);
    if (s) return s;
    int model;
    if (!uniform_model(n_views, cameras, model))
        return fail(ADOP_ERR_UNSUPPORTED, "all views of one call must use the same camera model");
    static thread_local RasterArgs a;
    fill_args(a, points, n_views, cameras, poses, params, views, &ws);
    if (vec_path(points)) encode_pos_tmap(a, points);
    // only the pipelined depth kernel (vector path) writes the ghost list the backward can consume
    a.tag = vec_path(points) ? call_tag(points, n_views, cameras, poses, params, views, workspace_bytes) : 0ull;
    // with ghosts (rho > 0) the pooled depth pass also lists them for the backward, which then needs no sweep
    a.ghost_fwd = (a.tag != 0ull && a.ghost_thr != 0u && depth_lists_ghosts(a)) ? 1 : 0;
    int e = launch_clear(a, 0, stream);
    if (e) return cuda_status(e, "clear launch");
    if (points->n > 0) {
        e = launch_depth(a, model, vec_path(points), device_sms(), stream);
        if (e) return cuda_status(e, "depth launch");
    }
    if (a.mv_lists) {  // multi-view: the survivor chunks in view-major order (blend, and the backward's texture list)
        e = launch_chunk_order(a, 0, device_sms(), stream);
        if (e) return cuda_status(e, "chunk order launch");
    }
    return ok();
}

adop_status adop_forward_blend(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                               const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                               void *workspace, size_t workspace_bytes, void *stream) {
    Ws ws;
    adop_status s = prologue(points, n_views, cameras, poses, params, views, workspace, workspace_bytes, true, ws);
    if (s) return s;
    int model;
    if (!uniform_model(n_views, cameras, model))
        return fail(ADOP_ERR_UNSUPPORTED, "all views of one call must use the same camera model");
    static thread_local RasterArgs a;
    fill_args(a, points, n_views, cameras, poses, params, views, &ws);
    int e = launch_blend(a, model, vec_path(points), device_sms(), stream);  // also clears accum/count
    if (e) return cuda_status(e, "blend launch");
    return ok();
}

adop_status adop_forward_resolve(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                 const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                                 void *workspace, size_t workspace_bytes, void *stream) {
    Ws ws;
    adop_status s = prologue(points, n_views, cameras, poses, params, views, workspace, workspace_bytes, false, ws);
    if (s) return s;
    static thread_local RasterArgs a;
    fill_args(a, points, n_views, cameras, poses, params, views, &ws);
    int e = launch_resolve(a, stream);
    if (e) return cuda_status(e, "resolve launch");
    return ok();
}

adop_status adop_forward_resolve_range(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                       const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                                       int64_t p0, int64_t p1, void *workspace, size_t workspace_bytes, void *stream) {
    if (p0 < 0 || p1 < p0) return fail(ADOP_ERR_INVALID_ARGUMENT, "resolve range: need 0 <= p0 <= p1");
    Ws ws;
    adop_status s = prologue(points, n_views, cameras, poses, params, views, workspace, workspace_bytes, false, ws);
    if (s) return s;
    static thread_local RasterArgs a;
    fill_args(a, points, n_views, cameras, poses, params, views, &ws);
    a.res_p0 = p0;
    a.res_p1 = p1;
    if (p0 == p1) return ok();
    int e = launch_resolve(a, stream);
    if (e) return cuda_status(e, "resolve launch");
    return ok();
}

adop_status adop_rasterize_forward(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                   const adop_pose *poses, const adop_params *params, const adop_pyramid *views,
                                   void *workspace, size_t workspace_bytes, adop_comm *comm, void *stream) {
    adop_status s;
    if ((s = check_points(points, true))) return s;
    if ((s = comm_check(comm))) return s;
    if (comm && params && params->shared_pyramid)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "a communicator and a shared pyramid exclude each other");
    if ((s = adop_forward_depth(points, n_views, cameras, poses, params, views, workspace, workspace_bytes, stream)))
        return s;
    int64_t pixels[ADOP_MAX_VIEWS_PER_LAUNCH];
    for (int v = 0; v < n_views; ++v) pixels[v] = adop_pyramid_pixels(cameras[v].width, cameras[v].height, params->layers);
    if ((s = comm_keys(comm, views, pixels, n_views, stream))) return s;  // point sharding: MIN of the keys
    if ((s = adop_forward_blend(points, n_views, cameras, poses, params, views, workspace, workspace_bytes, stream)))
        return s;
    if ((s = comm_sums(comm, views, pixels, n_views, points->channels, stream))) return s;  // SUM of accum, count
    return adop_forward_resolve(points, n_views, cameras, poses, params, views, workspace, workspace_bytes, stream);
}

adop_status adop_rasterize_backward(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                                    const adop_pose *poses, const adop_params *params,
                                    const adop_pyramid *fwd_views, const float *const *grad_image, float *d_feat,
                                    float *d_pos, double *d_pose, double *d_intrinsics, float *d_env,
                                    void *workspace, size_t workspace_bytes, adop_comm *comm, void *stream) {
    Ws ws;
    adop_status cs = comm_check(comm);
    if (cs) return cs;
    adop_status s = prologue(points, n_views, cameras, poses, params, fwd_views, workspace, workspace_bytes, true, ws);
    if (s) return s;
    if (!grad_image) return fail(ADOP_ERR_INVALID_ARGUMENT, "grad_image is NULL");
    for (int v = 0; v < n_views; ++v)
        if (!grad_image[v] || !aligned(grad_image[v], 4))
            return fail(ADOP_ERR_INVALID_ARGUMENT, "grad_image[%d] is NULL or misaligned", v);
    if (d_feat && !aligned(d_feat, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "d_feat misaligned");
    if (d_pos && !aligned(d_pos, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "d_pos misaligned");
    if (d_pose && !aligned(d_pose, 8)) return fail(ADOP_ERR_INVALID_ARGUMENT, "d_pose misaligned");
    if (d_intrinsics && !aligned(d_intrinsics, 8)) return fail(ADOP_ERR_INVALID_ARGUMENT, "d_intrinsics misaligned");
    if (d_env && !params->env_map) return fail(ADOP_ERR_INVALID_ARGUMENT, "d_env given without an env_map");
    if (d_env && !aligned(d_env, 4)) return fail(ADOP_ERR_INVALID_ARGUMENT, "d_env misaligned");
    int model;
    if (!uniform_model(n_views, cameras, model))
        return fail(ADOP_ERR_UNSUPPORTED, "all views of one call must use the same camera model");
    static thread_local RasterArgs a;
    fill_args(a, points, n_views, cameras, poses, params, fwd_views, &ws);
    for (int v = 0; v < n_views; ++v) a.v[v].grad = grad_image[v];
    if (vec_path(points)) encode_pos_tmap(a, points);
    a.tag = call_tag(points, n_views, cameras, poses, params, fwd_views, workspace_bytes);
    a.d_feat = d_feat;
    a.d_pos = d_pos;
    a.d_intr = d_intrinsics;
    a.nterms = d_intrinsics ? 18 : 6;
    a.d_env = d_env;
    if (points->n == 0) {
        if (d_pose && !params->grad_accumulate) {
            int e = (int)cudaMemsetAsync(d_pose, 0, sizeof(double) * 6 * n_views, (cudaStream_t)stream);
            if (e) return cuda_status(e, "memset d_pose");
        }
        if (d_intrinsics && !params->grad_accumulate) {
            int e = (int)cudaMemsetAsync(d_intrinsics, 0, sizeof(double) * 12 * n_views, (cudaStream_t)stream);
            if (e) return cuda_status(e, "memset d_intrinsics");
        }
        if (d_env) {  // every pixel is background: E still gets its gradient
            int e = launch_env_grad(a, stream);
            if (e) return cuda_status(e, "env gradient launch");
        }
    } else {
        int e = launch_backward(a, model, vec_path(points), device_sms(), kMaxBwdBlocks, d_pose, stream);
        if (e) return cuda_status(e, "backward launch");
    }
    const int64_t n_env = d_env ? (int64_t)params->env_width * params->env_height * points->channels : 0;
    adop_status st = comm_grads(comm, points->n, points->channels, n_views, d_feat, d_pos, d_pose, d_intrinsics, d_env,
                                n_env, stream);
    if (st) return st;
    return ok();
}

adop_status adop_point_masks(const adop_points *points, int32_t n_views, const adop_camera *cameras,
                             const adop_pose *poses, const adop_params *params, uint8_t *mask, void *stream) {
    adop_status s;
    if ((s = check_params(params))) return s;
    if ((s = check_points(points, false))) return s;
    if ((s = check_culling(points, params))) return s;
    if ((s = check_views(n_views, cameras, poses, params, nullptr, points->channels, false))) return s;
    if (!mask && points->n > 0) return fail(ADOP_ERR_INVALID_ARGUMENT, "mask is NULL");
    int model;
    if (!uniform_model(n_views, cameras, model))
        return fail(ADOP_ERR_UNSUPPORTED, "all views of one call must use the same camera model");
    if (points->n == 0) return ok();
    static thread_local RasterArgs a;
    fill_args(a, points, n_views, cameras, poses, params, nullptr, nullptr);
    a.mask = mask;
    int e = launch_masks(a, model, stream);
    if (e) return cuda_status(e, "mask launch");
    return ok();
}

adop_status adop_tile_bounds(const adop_points *points, float *bounds, void *stream) {
    adop_status s;
    if ((s = check_points(points, false))) return s;
    if (points->n > 0 && !bounds) return fail(ADOP_ERR_INVALID_ARGUMENT, "bounds is NULL");
    if (bounds && !aligned(bounds, 16)) return fail(ADOP_ERR_INVALID_ARGUMENT, "bounds not 16-byte aligned");
    if (points->n == 0) return ok();
    int e = launch_tile_bounds(points->pos, points->pos + points->pos_stride, points->pos + 2 * points->pos_stride,
                               points->n, bounds, stream);
    if (e) return cuda_status(e, "tile bounds launch");
    return ok();
}

adop_status adop_camera_window(const adop_camera *camera, int32_t layers, float out[4], int32_t *valid) {
    if (!camera || !out || !valid) return fail(ADOP_ERR_INVALID_ARGUMENT, "NULL argument");
    if (layers < 1 || layers > ADOP_MAX_LAYERS) return fail(ADOP_ERR_INVALID_ARGUMENT, "bad layers");
    adop_status st = check_camera(camera, 0, layers);
    if (st) return st;
    *valid = 0;
    if (camera->model != ADOP_OPENCV8 || !window_test_enabled()) return ok();
    // the same window and widening as fill_args
    const float lmax = (float)(1 << (layers - 1));
    const NormWindow w = camera_window(*camera, -lmax - 2.0f, (float)camera->width + lmax + 2.0f, -lmax - 2.0f,
                                       (float)camera->height + lmax + 2.0f);
    if (!w.ok) return ok();
    const double b[4] = {w.xlo, w.xhi, w.ylo, w.yhi};
    for (int k = 0; k < 4; ++k) out[k] = (float)(b[k] + (k & 1 ? 1.0 : -1.0) * 1e-4 * (1.0 + std::fabs(b[k])));
    *valid = 1;
    return ok();
}

adop_status adop_clear_pyramid(int32_t n_views, const adop_camera *cameras, int32_t layers, int32_t channels,
                               const adop_pyramid *views, void *stream) {
    if (!cameras || !views) return fail(ADOP_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_views < 1 || n_views > ADOP_MAX_VIEWS_PER_LAUNCH)
        return fail(ADOP_ERR_INVALID_ARGUMENT, "n_views = %d not in [1, %d]", n_views, ADOP_MAX_VIEWS_PER_LAUNCH);
    if (layers < 1 || layers > ADOP_MAX_LAYERS) return fail(ADOP_ERR_INVALID_ARGUMENT, "bad layers");
    if (channels < 1 || channels > ADOP_MAX_CHANNELS) return fail(ADOP_ERR_INVALID_ARGUMENT, "bad channels");
    for (int v = 0; v < n_views; ++v) {
        const int64_t P = adop_pyramid_pixels(cameras[v].width, cameras[v].height, layers);
        if (P <= 0) return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: bad width/height", v);
        if (!views[v].keys || !views[v].accum || !views[v].count)
            return fail(ADOP_ERR_INVALID_ARGUMENT, "view %d: NULL pyramid buffer", v);
        int e = launch_clear_pyr(views[v].keys, views[v].accum, views[v].count, P, channels, stream);
        if (e) return cuda_status(e, "clear pyramid launch");
    }
    return ok();
}

adop_status adop_ipc_export(const void *ptr, unsigned char handle[64], uint64_t *offset) {
    if (!ptr || !handle || !offset) return fail(ADOP_ERR_INVALID_ARGUMENT, "NULL argument");
    static PFN_cuMemGetAddressRange_v3020 range = nullptr;
    if (!range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return fail(ADOP_ERR_CUDA, "cuMemGetAddressRange unavailable");
        }
        range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return fail(ADOP_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)base);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
    *offset = (uint64_t)((CUdeviceptr)ptr - base);
    return ok();
}

adop_status adop_ipc_open(const unsigned char handle[64], uint64_t offset, void **base, void **ptr) {
    if (!handle || !base || !ptr) return fail(ADOP_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void *b = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcOpenMemHandle");
    *base = b;
    *ptr = static_cast<char *>(b) + offset;
    return ok();
}

adop_status adop_ipc_close(void *base) {
    if (!base) return fail(ADOP_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcCloseMemHandle");
    return ok();
}

adop_status adop_workspace_stats(const void *workspace, size_t workspace_bytes, void *stream, int64_t *records,
                                 int64_t *ghost_entries, int32_t *overflowed, int64_t *tiles_read) {
    if (!workspace || workspace_bytes < kHeaderBytes) return fail(ADOP_ERR_INVALID_ARGUMENT, "bad workspace");
    WsHeader h;
    cudaError_t e = cudaMemcpyAsync(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status((int)e, "workspace stats");
    if (records) *records = (int64_t)h.front_ok;
    if (ghost_entries) *ghost_entries = (int64_t)(h.back_ok / 2);
    if (tiles_read) *tiles_read = (int64_t)h.tiles_read;
    if (overflowed) *overflowed = h.overflow;
    return ok();
}

const char *adop_last_error(void) { return g_err; }

#if defined(ADOP_CHECKS) && ADOP_CHECKS
const char *adop_version(void) { return "adop-b200 0.2 (sm_100a, bounds-checked)"; }
#else
const char *adop_version(void) { return "adop-b200 0.2 (sm_100a)"; }
#endif

}  // extern "C"
