/*
 * adop_oracle.c -- plain, slow, single-threaded CPU oracle of ADOP's one-pixel
 * point rasterizer (Rückert, Franke, Stamminger: "ADOP: Approximate
 * Differentiable One-Pixel Point Rendering", arXiv 2110.06635).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path may import, link or
 * execute this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant generator with paper_2110_06635_b200/csrc/; the CUDA path
 * and this file were written separately against the readings R1..R27 listed
 * in DESIGN.md.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (section/equation
 * named alongside).  Readings "Rnn" = DESIGN.md §Readings.
 *
 * Precision: every quantity that DECIDES an integer (pixel index, bounds,
 * depth key, discard/ghost bits, fuzzy-test and Eq. 11 case choices) is
 * computed in IEEE fp32 with the pinned operation order of R1/R2/R6/R9/R10/R14
 * (compile with -ffp-contract=off, no fast-math), because the task requires
 * both sides to take such decisions in the same precision.  Every continuous
 * result (blend sums, means, gradients, Jacobians) is accumulated in fp64.
 *
 * Loops follow the paper's order: per view, per layer/point: project (Eq. 2),
 * round (Eq. 3), bounds (Eq. 4), stochastic discard (Eq. 12), depth-only pass
 * (§4.5), fuzzy test (Eq. 6), blend mean (Eq. 7); backward: texture gradient
 * (§4.2 "straightforward"), ghost image-space gradient (Eqs. 9-11, §4.3),
 * chain rule to points and tangent-space pose (Eq. 8, Eq. 17).
 *
 * Threads: OpenMP over points in chunks of ORC_CHUNK.  Every
 * per-point quantity (projection, masks, pixels, per-point gradients) is
 * computed in parallel into per-point slots of the chunk; every quantity that
 * is a reduction over points (depth keys, blend sums and counts, pose and
 * intrinsics gradients) is then reduced SERIALLY in point order.  The results
 * are therefore bit-identical to the single-threaded program for any thread
 * count (tests/test_oracle_threads.py checks it).
 *
 * Parity pins: tests/test_oracle_*.py (closed forms, brute force, finite
 * differences, worked values).  Parity unpinned: none of the functions below
 * is unpinned; the *usefulness* of ghost gradients (paper §6.2) is not a
 * parity claim.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_CHUNK ((int64_t)1 << 18) /* points per parallel chunk */

static int orc_threads = 1;

/* Thread count of every parallel loop below (>= 1); returns the count in effect. */
int orc_set_threads(int n)
{
#ifdef _OPENMP
    orc_threads = n >= 1 ? n : omp_get_num_procs();
#else
    (void)n;
    orc_threads = 1;
#endif
    return orc_threads;
}

int orc_get_threads(void) { return orc_threads; }

typedef struct {
    int32_t width, height, model; /* model 0 = pinhole, 1 = OpenCV rational 8-coefficient (R6),
                                     2 = equidistant fisheye with distance depth (R35; r2_max holds theta_max) */
    float fx, fy, cx, cy;
    float k[6];
    float p[2];
    float r2_max;
} orc_camera;

typedef struct {
    float R[9]; /* world -> camera rotation, row-major: Xc = R x + t (Eq. 2) */
    float t[3];
} orc_pose;

typedef struct {
    int32_t layers;
    float alpha;        /* fuzzy depth threshold, Eq. 6 */
    int32_t discard;    /* stochastic point discarding on/off, §4.4 */
    float gamma;        /* Eq. 12 */
    float ghost_rate;   /* dropout rate of the ghost split, §4.3 (R13) */
    float z_near;       /* R7 */
    uint64_t seed;
    int32_t view_id_base;
    int32_t log_descriptors; /* NEXT-2: tau stored as log, linearized by exp() when rasterized */
    int32_t spatial_rendered;/* NEXT-3 (R31): 0 = ghost gradients (spatial gradients for ghosts only, §4.3);
                                1 = ghost gradients disabled (the §6.2 baseline): Eqs. 9-11
                                for the rendered points, none for ghosts */
    int32_t normal_culling;  /* NEXT-3, Eq. 5, R32: 0 off; +1 keep iff (Rn).Xc > 0 (as printed);
                                -1 keep iff (Rn).Xc < 0 (the flipped orientation) */
} orc_params;

typedef struct {             /* NEXT-2: spherical environment map E of Eq. 7, R29 */
    const float *data;       /* [height][width][C] equirectangular, NULL = constant background (R18) */
    int32_t width, height;
} orc_env;

typedef struct {
    int64_t n;
    int64_t global_offset; /* global index of point 0 (R25) */
    int64_t pos_stride;    /* x row at pos[0..n), y row at pos[stride..], z row at pos[2*stride..] */
    const float *pos;
    const float *radius;   /* [n] or NULL -> radius_uniform */
    float radius_uniform;
    const float *feat;     /* [n][C] */
    int32_t channels;
    const float *normal;   /* NEXT-3: SoA [3][pos_stride] point normals n of Eq. 1, or NULL */
} orc_points;

#define ORC_SENTINEL 0x7FFFFFFFFFFFFFFFULL /* R8: empty pixel */
#define ORC_STREAM_GHOST 1u
#define ORC_STREAM_DISCARD 2u

/* ------------------------------------------------------------------------- */
/* Layer geometry (R5): w_l = ceil(w / 2^l), h_l = ceil(h / 2^l).             */
/* ------------------------------------------------------------------------- */
static int32_t layer_w(int32_t w, int l) { return (int32_t)((w + (1 << l) - 1) >> l); }

int64_t orc_pyramid_pixels(int32_t w, int32_t h, int32_t layers)
{
    int64_t total = 0;
    for (int l = 0; l < layers; ++l) total += (int64_t)layer_w(w, l) * layer_w(h, l);
    return total;
}

static int64_t layer_offset(int32_t w, int32_t h, int l)
{
    return orc_pyramid_pixels(w, h, l);
}

/* ------------------------------------------------------------------------- */
/* Counter-based hash (R11, R13).  Both sides implement this same published  */
/* integer finalizer independently (the task allows "each side implements    */
/* the same counter-based generator").                                       */
/* ------------------------------------------------------------------------- */
static uint32_t mix32(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

static uint32_t stream_salt(uint64_t seed, uint32_t stream, uint32_t view)
{
    uint32_t s = mix32((uint32_t)seed + 0x9E3779B9U * (stream + 1U));
    s = mix32(s ^ (uint32_t)(seed >> 32));
    return mix32(s + 0x85EBCA6BU * (view + 1U));
}

/* Top 24 bits of the hash of global point index i for (seed, stream, view). */
uint32_t orc_h24(uint64_t seed, uint32_t stream, uint32_t view, uint32_t i)
{
    return mix32(i ^ stream_salt(seed, stream, view)) >> 8;
}

static uint32_t ghost_threshold(float rate)
{
    /* floor(rho * 2^24); rho in [0,1) */
    return (uint32_t)floor((double)rate * 16777216.0);
}

/* R13: point is a ghost (dropout set of §4.3). */
int orc_is_ghost(const orc_params *pr, uint32_t gi)
{
    uint32_t thr = ghost_threshold(pr->ghost_rate);
    return thr != 0 && orc_h24(pr->seed, ORC_STREAM_GHOST, 0u, gi) < thr;
}

/* ------------------------------------------------------------------------- */
/* Projection P_0 = C(R x + t)   (Eq. 2; camera model R6)        */
/* Pinned fp32 order (R1, R2, R6).  Returns 1 if the point is valid (R7).    */
/* out: [0..2] = Xc, [3] = u0, [4] = v0, [5] = 1/z                            */
/* ------------------------------------------------------------------------- */
/* R35: atan(t) for t in [0, 1] as t * P(t^2), a fixed degree-9 polynomial (max error 1e-7 rad) evaluated
 * by Horner in fp32 with one rounding per operation -- the GPU evaluates the same operations, so the
 * fisheye's pixel decisions stay bit-identical. */
static float atan01(float t)
{
    static const float c[10] = {-0.0015244261594489217f, 0.009669913910329342f, -0.028764614835381508f,
                                0.05541255697607994f, -0.08245089650154114f, 0.10893233865499496f,
                                -0.14251546561717987f, 0.1999710500240326f, -0.33333227038383484f, 1.0f};
    float u = t * t, p = c[0];
    for (int k = 1; k < 10; ++k) p = p * u + c[k];
    return t * p;
}
/* angle in [0, pi] of (x, y) with y >= 0 (R35) */
float orc_atan2p(float y, float x)
{
    const float PI = 3.14159265358979f, HALF_PI = 1.57079632679490f;
    float ax = fabsf(x), a;
    if (y <= ax) a = ax > 0.0f ? atan01(y / ax) : 0.0f;
    else a = HALF_PI - atan01(ax / y);
    return x >= 0.0f ? a : PI - a;
}

int orc_project(const orc_camera *c, const orc_pose *P, float x, float y, float z, float z_near, float *out)
{
    const float *R = P->R, *t = P->t;
    float X = ((R[0] * x + R[1] * y) + R[2] * z) + t[0];
    float Y = ((R[3] * x + R[4] * y) + R[5] * z) + t[1];
    float Z = ((R[6] * x + R[7] * y) + R[8] * z) + t[2];
    out[0] = X; out[1] = Y; out[2] = Z;
    out[6] = Z;  /* the depth of keys / Eq. 6 (R4): camera z, or the distance for the fisheye */
    if (c->model == 2) {
        /* R35 equidistant fisheye: theta = angle to the optical axis, r_d = f theta, depth = |Xc| */
        float rho2 = X * X + Y * Y;
        float d = sqrtf(rho2 + Z * Z);
        out[6] = d;
        if (!(d > z_near && d <= FLT_MAX)) return 0;
        float rho = sqrtf(rho2);
        float th = orc_atan2p(rho, Z);
        if (!(th <= c->r2_max)) return 0;  /* outside the field of view theta_max */
        float s = rho > 0.0f ? th / rho : 0.0f;
        float xd = X * s, yd = Y * s;
        out[3] = c->fx * xd + c->cx;
        out[4] = c->fy * yd + c->cy;
        out[5] = 1.0f / d;
        return 1;
    }
    if (!(Z > z_near && Z <= FLT_MAX)) return 0; /* behind camera / non-finite: culled (R7) */
    float iz = 1.0f / Z;
    float xn = X * iz, yn = Y * iz;
    float xd = xn, yd = yn;
    if (c->model == 1) {
        float xx = xn * xn, yy = yn * yn, xy = xn * yn;
        float r2 = xx + yy;
        if (!(r2 <= c->r2_max)) return 0; /* outside the camera's valid radius (R6) */
        float r4 = r2 * r2, r6 = r4 * r2;
        float num = ((1.0f + c->k[0] * r2) + c->k[1] * r4) + c->k[2] * r6;
        float den = ((1.0f + c->k[3] * r2) + c->k[4] * r4) + c->k[5] * r6;
        if (!(den > 0.0f)) return 0;
        float radial = num / den;
        float a1 = 2.0f * xy;
        float a2 = r2 + 2.0f * xx;
        float a3 = r2 + 2.0f * yy;
        xd = (xn * radial + c->p[0] * a1) + c->p[1] * a2;
        yd = (yn * radial + c->p[0] * a3) + c->p[1] * a1;
    }
    out[3] = c->fx * xd + c->cx;
    out[4] = c->fy * yd + c->cy;
    out[5] = iz;
    return 1;
}

/* Eq. 3 + Eq. 4: round half away from zero (R3) and
 * bounds-test the rounded float.  Returns the layer-local linear index or -1. */
static int64_t layer_pixel(const orc_camera *c, float u0, float v0, int l)
{
    float s = ldexpf(1.0f, -l);         /* 1/2^l of Eq. 2 */
    float ru = roundf(u0 * s), rv = roundf(v0 * s);
    int32_t wl = layer_w(c->width, l), hl = layer_w(c->height, l);
    if (!(ru >= 0.0f && ru < (float)wl && rv >= 0.0f && rv < (float)hl)) return -1;
    return (int64_t)rv * wl + (int64_t)ru;
}

/* Eq. 12, R10/R11: number of leading layers at which the point is
 * kept.  keep_l <=> (gamma * r_screen_l)^2 > 1 - beta, beta per (view, point). */
static int keep_layers(const orc_params *pr, const orc_camera *c, float rw, float iz, uint32_t view, uint32_t gi)
{
    if (!pr->discard) return pr->layers;
    float feff = (c->fx + c->fy) * 0.5f;
    float rs0 = (rw * feff) * iz;                      /* r_world projected to pixels, layer 0 */
    uint32_t h = orc_h24(pr->seed, ORC_STREAM_DISCARD, view, gi);
    float one_minus_beta = (float)(16777216u - h) * (1.0f / 16777216.0f);
    int l;
    for (l = 0; l < pr->layers; ++l) {
        float rl = rs0 * ldexpf(1.0f, -l);
        float a = pr->gamma * rl;
        if (!(a * a > one_minus_beta)) break;
    }
    return l;
}

static float point_radius(const orc_points *pts, int64_t i)
{
    return pts->radius ? pts->radius[i] : pts->radius_uniform;
}

/* Per point, per view: bit l = valid & in-bounds at l & kept at l (discard);
 * bit 7 = ghost.  The render set at layer l is bit l and not bit 7. */
static unsigned point_mask(const orc_points *pts, int64_t i, const orc_camera *c, const orc_pose *P,
                           const orc_params *pr, uint32_t view, int64_t *pix /*[layers]*/, float *proj /*[6]*/)
{
    uint32_t gi = (uint32_t)(pts->global_offset + i);
    const float *pos = pts->pos;
    float x = pos[i], y = pos[pts->pos_stride + i], z = pos[2 * pts->pos_stride + i];
    unsigned m = orc_is_ghost(pr, gi) ? 0x80u : 0u;
    if (!orc_project(c, P, x, y, z, pr->z_near, proj)) return m;
    if (pr->normal_culling && pts->normal) {
        /* Eq. 5 as R32: sign of (R n) . Xc in the pinned fp32 order of R1 (|Xc| > 0 drops out) */
        const float *nv = pts->normal;
        float nx = nv[i], ny = nv[pts->pos_stride + i], nz = nv[2 * pts->pos_stride + i];
        float ncx = (P->R[0] * nx + P->R[1] * ny) + P->R[2] * nz;
        float ncy = (P->R[3] * nx + P->R[4] * ny) + P->R[5] * nz;
        float ncz = (P->R[6] * nx + P->R[7] * ny) + P->R[8] * nz;
        float dot = (ncx * proj[0] + ncy * proj[1]) + ncz * proj[2];
        if (!(pr->normal_culling > 0 ? dot > 0.0f : dot < 0.0f)) return m;
    }
    int nk = keep_layers(pr, c, point_radius(pts, i), proj[5], view, gi);
    for (int l = 0; l < pr->layers; ++l) {
        pix[l] = layer_pixel(c, proj[3], proj[4], l);
        if (l < nk && pix[l] >= 0) m |= 1u << l;
    }
    return m;
}

void orc_point_masks(const orc_points *pts, int32_t n_views, const orc_camera *cams, const orc_pose *poses,
                     const orc_params *pr, uint8_t *mask /*[V][n]*/)
{
    for (int v = 0; v < n_views; ++v) {
        #pragma omp parallel for schedule(static) num_threads(orc_threads)
        for (int64_t i = 0; i < pts->n; ++i) {
            int64_t pix[8];
            float proj[7];
            mask[(int64_t)v * pts->n + i] =
                (uint8_t)point_mask(pts, i, &cams[v], &poses[v], pr, (uint32_t)(pr->view_id_base + v), pix, proj);
        }
    }
}

/* Per-point slots of one chunk [i0, i0 + cnt): mask, pixels per layer and projection of every point, computed
 * in parallel (a map: each point writes only its own slot).  The callers reduce over the slots serially. */
typedef struct {
    uint8_t *mask;  /* [ORC_CHUNK] */
    int64_t *pix;   /* [ORC_CHUNK][8] */
    float *proj;    /* [ORC_CHUNK][8] (orc_project's 7 outputs) */
} orc_chunk;

static int chunk_alloc(orc_chunk *ch)
{
    ch->mask = (uint8_t *)malloc((size_t)ORC_CHUNK);
    ch->pix = (int64_t *)malloc(sizeof(int64_t) * 8 * (size_t)ORC_CHUNK);
    ch->proj = (float *)malloc(sizeof(float) * 8 * (size_t)ORC_CHUNK);
    return ch->mask && ch->pix && ch->proj;
}

static void chunk_free(orc_chunk *ch)
{
    free(ch->mask);
    free(ch->pix);
    free(ch->proj);
}

static void chunk_masks(const orc_points *pts, int64_t i0, int64_t cnt, const orc_camera *c, const orc_pose *P,
                        const orc_params *pr, uint32_t view, orc_chunk *ch)
{
    #pragma omp parallel for schedule(static) num_threads(orc_threads)
    for (int64_t j = 0; j < cnt; ++j)
        ch->mask[j] = (uint8_t)point_mask(pts, i0 + j, c, P, pr, view, ch->pix + 8 * j, ch->proj + 8 * j);
}

static uint64_t depth_key(float Z, uint32_t gi)
{
    uint32_t zb;
    memcpy(&zb, &Z, 4);
    return ((uint64_t)zb << 32) | gi; /* R8 */
}

static float key_depth(uint64_t key)
{
    uint32_t zb = (uint32_t)(key >> 32);
    float m;
    memcpy(&m, &zb, 4);
    return m;
}

/* Linear-space descriptor channel (logarithmic descriptors are converted to linear space
 * during rasterization): exp(tau) in fp64 for log descriptors, tau otherwise. */
static double desc_lin(const orc_params *pr, float t) { return pr->log_descriptors ? exp((double)t) : (double)t; }

/* ------------------------------------------------------------------------- */
/* Environment map (NEXT-2), reading R29.                                    */
/* C^{-1}: layer-l pixel centre (u, v) -> layer-0 continuous pixel (u 2^l,   */
/* v 2^l) (inverse of Eq. 2's 2^-l) -> normalized camera coordinates: the    */
/* pinhole inverse, then for OpenCV8 8 Newton steps on the distortion map    */
/* of R6 started at the distorted coordinates.  World direction d = R^T      */
/* (xn, yn, 1) (Eq. 7's E(R^T C^{-1}(u, v))).  Equirectangular lookup:       */
/* lon = atan2(d_x, d_z), lat = atan2(d_y, hypot(d_x, d_z)),                 */
/* s = (lon / 2pi + 1/2) W - 1/2, t = (lat / pi + 1/2) H - 1/2, bilinear,    */
/* columns wrapped, rows clamped.                                            */
/* ------------------------------------------------------------------------- */
static void distort_f64(const orc_camera *c, double xn, double yn, double *xd, double *yd, double D[2][2])
{
    const double k1 = c->k[0], k2 = c->k[1], k3 = c->k[2], k4 = c->k[3], k5 = c->k[4], k6 = c->k[5];
    const double p1 = c->p[0], p2 = c->p[1];
    double r2 = xn * xn + yn * yn;
    double num = 1.0 + k1 * r2 + k2 * r2 * r2 + k3 * r2 * r2 * r2;
    double den = 1.0 + k4 * r2 + k5 * r2 * r2 + k6 * r2 * r2 * r2;
    double rad = num / den;
    *xd = xn * rad + 2.0 * p1 * xn * yn + p2 * (r2 + 2.0 * xn * xn);
    *yd = yn * rad + p1 * (r2 + 2.0 * yn * yn) + 2.0 * p2 * xn * yn;
    double dnum = k1 + 2.0 * k2 * r2 + 3.0 * k3 * r2 * r2;
    double dden = k4 + 2.0 * k5 * r2 + 3.0 * k6 * r2 * r2;
    double drad = (dnum * den - num * dden) / (den * den);
    D[0][0] = rad + 2.0 * xn * xn * drad + 2.0 * p1 * yn + 6.0 * p2 * xn;
    D[0][1] = 2.0 * xn * yn * drad + 2.0 * p1 * xn + 2.0 * p2 * yn;
    D[1][0] = D[0][1];
    D[1][1] = rad + 2.0 * yn * yn * drad + 6.0 * p1 * yn + 2.0 * p2 * xn;
}

void orc_unproject(const orc_camera *c, double u0, double v0, double *xn, double *yn)
{
    double xd = (u0 - (double)c->cx) / (double)c->fx, yd = (v0 - (double)c->cy) / (double)c->fy;
    double x = xd, y = yd;
    if (c->model == 1) {
        for (int it = 0; it < 8; ++it) {
            double fx_, fy_, D[2][2];
            distort_f64(c, x, y, &fx_, &fy_, D);
            double rx = fx_ - xd, ry = fy_ - yd;
            double det = D[0][0] * D[1][1] - D[0][1] * D[1][0];
            x -= (D[1][1] * rx - D[0][1] * ry) / det;
            y -= (-D[1][0] * rx + D[0][0] * ry) / det;
        }
    }
    *xn = x;
    *yn = y;
}

/* Bilinear lookup of E in world direction d: 4 texel indices (texel = row * W + col) and weights. */
void orc_env_taps(const orc_env *e, const double *d, int64_t *idx, double *w)
{
    const double PI = 3.14159265358979323846;
    double lon = atan2(d[0], d[2]), lat = atan2(d[1], sqrt(d[0] * d[0] + d[2] * d[2]));
    double s = (lon / (2.0 * PI) + 0.5) * e->width - 0.5, t = (lat / PI + 0.5) * e->height - 0.5;
    double s0 = floor(s), t0 = floor(t), fs = s - s0, ft = t - t0;
    int64_t c0 = (int64_t)s0, r0 = (int64_t)t0;
    int64_t cols[2] = {((c0 % e->width) + e->width) % e->width, (((c0 + 1) % e->width) + e->width) % e->width};
    int64_t rows[2] = {r0 < 0 ? 0 : (r0 >= e->height ? e->height - 1 : r0),
                       r0 + 1 < 0 ? 0 : (r0 + 1 >= e->height ? e->height - 1 : r0 + 1)};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            idx[a * 2 + b] = rows[a] * e->width + cols[b];
            w[a * 2 + b] = (a ? ft : 1.0 - ft) * (b ? fs : 1.0 - fs);
        }
}

/* World direction of layer-l pixel (u, v) of a view (R29). */
void orc_env_dir(const orc_camera *c, const orc_pose *P, int l, int64_t u, int64_t v, double *d)
{
    double xn, yn;
    double dc[3];
    if (c->model == 2) {  /* R35: theta = |(xd, yd)|, direction (sin theta xd / theta, sin theta yd / theta, cos theta) */
        double xd = (ldexp((double)u, l) - (double)c->cx) / (double)c->fx;
        double yd = (ldexp((double)v, l) - (double)c->cy) / (double)c->fy;
        double th = sqrt(xd * xd + yd * yd), s = th > 0.0 ? sin(th) / th : 1.0;
        dc[0] = s * xd; dc[1] = s * yd; dc[2] = cos(th);
    } else {
        orc_unproject(c, ldexp((double)u, l), ldexp((double)v, l), &xn, &yn);
        dc[0] = xn; dc[1] = yn; dc[2] = 1.0;
    }
    for (int k = 0; k < 3; ++k)  /* R^T dc */
        d[k] = (double)P->R[0 + k] * dc[0] + (double)P->R[3 + k] * dc[1] + (double)P->R[6 + k] * dc[2];
}

/* ------------------------------------------------------------------------- */
/* Forward pass 1: depth-only render pass (§4.5) = per-pixel min of  */
/* the packed keys over the render set (Eq. 6's min_z with R8 tie rule).     */
/* keys: [V][P], set to the sentinel first.                                  */
/* ------------------------------------------------------------------------- */
void orc_forward_depth(const orc_points *pts, int32_t n_views, const orc_camera *cams, const orc_pose *poses,
                       const orc_params *pr, uint64_t *keys)
{
    orc_chunk ch;
    if (!chunk_alloc(&ch)) abort();
    for (int v = 0; v < n_views; ++v) {
        const orc_camera *c = &cams[v];
        int64_t P = orc_pyramid_pixels(c->width, c->height, pr->layers);
        uint64_t *kv = keys + (int64_t)v * P;
        for (int64_t p = 0; p < P; ++p) kv[p] = ORC_SENTINEL;
        for (int64_t i0 = 0; i0 < pts->n; i0 += ORC_CHUNK) {
            int64_t cnt = pts->n - i0 < ORC_CHUNK ? pts->n - i0 : ORC_CHUNK;
            chunk_masks(pts, i0, cnt, c, &poses[v], pr, (uint32_t)(pr->view_id_base + v), &ch);
            for (int64_t j = 0; j < cnt; ++j) {  /* serial, point order */
                unsigned m = ch.mask[j];
                if (m & 0x80u) continue; /* ghosts are not rendered */
                uint64_t key = depth_key(ch.proj[8 * j + 6], (uint32_t)(pts->global_offset + i0 + j));
                for (int l = 0; l < pr->layers; ++l) {
                    if (!(m & (1u << l))) continue;
                    int64_t q = layer_offset(c->width, c->height, l) + ch.pix[8 * j + l];
                    if (key < kv[q]) kv[q] = key;
                }
            }
        }
    }
    chunk_free(&ch);
}

/* Fuzzy depth test, Eq. 6, pinned as R9: z <= fl(fl(1+alpha) * m). */
static int fuzzy_pass(float z, uint64_t key, float alpha)
{
    float onepa = 1.0f + alpha;
    float thr = onepa * key_depth(key);
    return z <= thr;
}

/* ------------------------------------------------------------------------- */
/* Forward pass 2: accumulate tau and |Lambda| for points passing the fuzzy  */
/* test (§4.5).  accum [V][P][C] fp64, count [V][P] fp64; both   */
/* are zeroed first.                                                         */
/* ------------------------------------------------------------------------- */
void orc_forward_blend(const orc_points *pts, int32_t n_views, const orc_camera *cams, const orc_pose *poses,
                       const orc_params *pr, const uint64_t *keys, double *accum, double *count)
{
    const int C = pts->channels;
    orc_chunk ck;
    if (!chunk_alloc(&ck)) abort();
    for (int v = 0; v < n_views; ++v) {
        const orc_camera *c = &cams[v];
        int64_t P = orc_pyramid_pixels(c->width, c->height, pr->layers);
        const uint64_t *kv = keys + (int64_t)v * P;
        double *av = accum + (int64_t)v * P * C;
        double *cv = count + (int64_t)v * P;
        memset(av, 0, sizeof(double) * (size_t)(P * C));
        memset(cv, 0, sizeof(double) * (size_t)P);
        for (int64_t i0 = 0; i0 < pts->n; i0 += ORC_CHUNK) {
            int64_t cnt = pts->n - i0 < ORC_CHUNK ? pts->n - i0 : ORC_CHUNK;
            chunk_masks(pts, i0, cnt, c, &poses[v], pr, (uint32_t)(pr->view_id_base + v), &ck);
            for (int64_t j = 0; j < cnt; ++j) {  /* serial, point order */
                unsigned m = ck.mask[j];
                if (m & 0x80u) continue;
                int64_t i = i0 + j;
                for (int l = 0; l < pr->layers; ++l) {
                    if (!(m & (1u << l))) continue;
                    int64_t q = layer_offset(c->width, c->height, l) + ck.pix[8 * j + l];
                    if (!fuzzy_pass(ck.proj[8 * j + 6], kv[q], pr->alpha)) continue;
                    for (int ch = 0; ch < C; ++ch) av[q * C + ch] += desc_lin(pr, pts->feat[i * C + ch]);
                    cv[q] += 1.0;
                }
            }
        }
    }
    chunk_free(&ck);
}

/* ------------------------------------------------------------------------- */
/* Forward pass 3: Eq. 7: mean of tau over Lambda, or the       */
/* background E (constant vector, R18) when Lambda is empty.  image layout:  */
/* [V][C*P], layer l planar [C][h_l][w_l] starting at C*off_l.               */
/* ------------------------------------------------------------------------- */
void orc_forward_resolve(int32_t n_views, const orc_camera *cams, const orc_pose *poses, const orc_params *pr,
                         int32_t C, const double *accum, const double *count, const float *bg, const orc_env *env,
                         double *image)
{
    for (int v = 0; v < n_views; ++v) {
        const orc_camera *c = &cams[v];
        int64_t P = orc_pyramid_pixels(c->width, c->height, pr->layers);
        for (int l = 0; l < pr->layers; ++l) {
            int64_t off = layer_offset(c->width, c->height, l);
            int32_t wl = layer_w(c->width, l);
            int64_t hw = (int64_t)wl * layer_w(c->height, l);
            #pragma omp parallel for schedule(static) num_threads(orc_threads)
            for (int64_t j = 0; j < hw; ++j) {  /* each pixel writes only its own outputs */
                int64_t q = off + j;
                double n = count[(int64_t)v * P + q];
                double bgv[32];
                if (n == 0.0) {  /* Eq. 7 first case: E(R^T C^{-1}(u, v)), or the constant E of R18 */
                    for (int ch = 0; ch < C; ++ch) bgv[ch] = bg ? (double)bg[ch] : 0.0;
                    if (env && env->data) {
                        double d[3], w[4];
                        int64_t idx[4];
                        orc_env_dir(c, &poses[v], l, j % wl, j / wl, d);
                        orc_env_taps(env, d, idx, w);
                        for (int ch = 0; ch < C; ++ch) {
                            bgv[ch] = 0.0;
                            for (int k = 0; k < 4; ++k) bgv[ch] += w[k] * (double)env->data[idx[k] * C + ch];
                        }
                    }
                }
                for (int ch = 0; ch < C; ++ch) {
                    double val = n > 0.0 ? accum[((int64_t)v * P + q) * C + ch] / n : bgv[ch];
                    image[(int64_t)v * C * P + C * off + ch * hw + j] = val;
                }
            }
        }
    }
}

/* Full forward: Eq. 1 I_l = Phi_l(...) for all layers and views. */
void orc_forward(const orc_points *pts, int32_t n_views, const orc_camera *cams, const orc_pose *poses,
                 const orc_params *pr, const float *bg, const orc_env *env, uint64_t *keys, double *accum,
                 double *count, double *image)
{
    orc_forward_depth(pts, n_views, cams, poses, pr, keys);
    orc_forward_blend(pts, n_views, cams, poses, pr, keys, accum, count);
    orc_forward_resolve(n_views, cams, poses, pr, pts->channels, accum, count, bg, env, image);
}

/* ------------------------------------------------------------------------- */
/* Eq. 11 with reading R14: induced change of neighbour pixel q */
/* when the ghost (descriptor tau, depth z) is virtually shifted onto q.     */
/* Returns the case number 1..4.                                             */
/* ------------------------------------------------------------------------- */
static int induced_change_d(int32_t C, const double *tau, float z, float alpha, double n_q, uint64_t key_q,
                            const double *I_q, double *delta)
{
    float onepa = 1.0f + alpha;
    float m_q = key_depth(key_q);
    int kase;
    if (n_q == 0.0) kase = 1;                       /* background neighbour */
    else if (z > onepa * m_q) kase = 2;             /* shifted point fully behind */
    else if (z * onepa < m_q) kase = 3;             /* shifted point fully in front */
    else kase = 4;                                  /* fuzzy co-visible: blend mean changes */
    for (int ch = 0; ch < C; ++ch) {
        double t = tau[ch];
        switch (kase) {
        case 1: case 3: delta[ch] = t - I_q[ch]; break;
        case 2: delta[ch] = 0.0; break;
        default: delta[ch] = (n_q * I_q[ch] + t) / (n_q + 1.0) - I_q[ch]; break;
        }
    }
    return kase;
}

int orc_induced_change(int32_t C, const float *tau, float z, float alpha, double n_q, uint64_t key_q,
                       const double *I_q, double *delta)
{
    double t[32];
    for (int ch = 0; ch < C; ++ch) t[ch] = (double)tau[ch];
    return induced_change_d(C, t, z, alpha, n_q, key_q, I_q, delta);
}

/* Projection Jacobian d(u0,v0)/dXc (R21), fp64 at the fp32 camera point.   */
void orc_jacobian(const orc_camera *c, const float *Xc, double *J /* 2x3 row-major */)
{
    double X = Xc[0], Y = Xc[1], Z = Xc[2];
    if (c->model == 2) {
        /* R35 equidistant: u0 = fx g X + cx, v0 = fy g Y + cy, g = theta / rho, theta = atan2(rho, Z) */
        double rho2 = X * X + Y * Y, rho = sqrt(rho2), d2 = rho2 + Z * Z;
        double g, A;
        if (rho < 1e-6 * fabs(Z) && Z > 0) {  /* series at the optical axis */
            g = (1.0 - rho2 / (3.0 * Z * Z)) / Z;
            A = -2.0 / (3.0 * Z * Z * Z);
        } else {
            double th = atan2(rho, Z);
            g = th / rho;
            A = Z / (rho2 * d2) - th / (rho2 * rho);
        }
        J[0] = c->fx * (g + X * X * A); J[1] = c->fx * X * Y * A; J[2] = -c->fx * X / d2;
        J[3] = c->fy * X * Y * A; J[4] = c->fy * (g + Y * Y * A); J[5] = -c->fy * Y / d2;
        return;
    }
    double xn = X / Z, yn = Y / Z;
    /* dn/dXc = [[1/Z, 0, -X/Z^2], [0, 1/Z, -Y/Z^2]] */
    double N[2][3] = {{1.0 / Z, 0.0, -X / (Z * Z)}, {0.0, 1.0 / Z, -Y / (Z * Z)}};
    double D[2][2] = {{1.0, 0.0}, {0.0, 1.0}};
    if (c->model == 1) {
        const double k1 = c->k[0], k2 = c->k[1], k3 = c->k[2], k4 = c->k[3], k5 = c->k[4], k6 = c->k[5];
        const double p1 = c->p[0], p2 = c->p[1];
        double r2 = xn * xn + yn * yn;
        double num = 1.0 + k1 * r2 + k2 * r2 * r2 + k3 * r2 * r2 * r2;
        double den = 1.0 + k4 * r2 + k5 * r2 * r2 + k6 * r2 * r2 * r2;
        double dnum = k1 + 2.0 * k2 * r2 + 3.0 * k3 * r2 * r2;
        double dden = k4 + 2.0 * k5 * r2 + 3.0 * k6 * r2 * r2;
        double rad = num / den;
        double drad = (dnum * den - num * dden) / (den * den); /* d radial / d r2 */
        D[0][0] = rad + 2.0 * xn * xn * drad + 2.0 * p1 * yn + 6.0 * p2 * xn;
        D[0][1] = 2.0 * xn * yn * drad + 2.0 * p1 * xn + 2.0 * p2 * yn;
        D[1][0] = 2.0 * xn * yn * drad + 2.0 * p1 * xn + 2.0 * p2 * yn;
        D[1][1] = rad + 2.0 * yn * yn * drad + 6.0 * p1 * yn + 2.0 * p2 * xn;
    }
    double f[2] = {c->fx, c->fy};
    for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k)
            J[r * 3 + k] = f[r] * (D[r][0] * N[0][k] + D[r][1] * N[1][k]);
}

/* Continuous fp64 projection (same camera model) -- used only to check the
 * Jacobian by finite differences. */
void orc_project_f64(const orc_camera *c, const double *Xc, double *uv)
{
    if (c->model == 2) {
        double rho = sqrt(Xc[0] * Xc[0] + Xc[1] * Xc[1]), th = atan2(rho, Xc[2]);
        double g = rho > 0.0 ? th / rho : 1.0 / Xc[2];
        uv[0] = c->fx * g * Xc[0] + c->cx;
        uv[1] = c->fy * g * Xc[1] + c->cy;
        return;
    }
    double xn = Xc[0] / Xc[2], yn = Xc[1] / Xc[2];
    double xd = xn, yd = yn;
    if (c->model == 1) {
        double r2 = xn * xn + yn * yn;
        double num = 1.0 + c->k[0] * r2 + c->k[1] * r2 * r2 + c->k[2] * r2 * r2 * r2;
        double den = 1.0 + c->k[3] * r2 + c->k[4] * r2 * r2 + c->k[5] * r2 * r2 * r2;
        double rad = num / den;
        xd = xn * rad + 2.0 * c->p[0] * xn * yn + c->p[1] * (r2 + 2.0 * xn * xn);
        yd = yn * rad + c->p[0] * (r2 + 2.0 * yn * yn) + 2.0 * c->p[1] * xn * yn;
    }
    uv[0] = c->fx * xd + c->cx;
    uv[1] = c->fy * yd + c->cy;
}

/* Intrinsics Jacobian d(u0,v0)/d theta (NEXT-1; Eq. 8's chain rule continued into the camera model C
 * of Eq. 2, which the paper optimizes: Fig. 4), fp64 at the fp32 camera point.
 * theta = (fx, fy, cx, cy, k1..k6, p1, p2); Jt row-major [2][12].  Camera model R6:
 *   u0 = fx xd + cx, v0 = fy yd + cy;
 *   xd = xn rad + 2 p1 xn yn + p2 (r2 + 2 xn^2),  yd = yn rad + p1 (r2 + 2 yn^2) + 2 p2 xn yn,
 *   rad = num / den, num = 1 + k1 r2 + k2 r2^2 + k3 r2^3, den = 1 + k4 r2 + k5 r2^2 + k6 r2^3.
 * Pinhole: xd = xn, yd = yn and the distortion columns are 0 (the model has no such parameters). */
void orc_intrinsics_jacobian(const orc_camera *c, const float *Xc, double *Jt)
{
    double xn = (double)Xc[0] / (double)Xc[2], yn = (double)Xc[1] / (double)Xc[2];
    for (int k = 0; k < 24; ++k) Jt[k] = 0.0;
    double xd = xn, yd = yn;
    if (c->model == 2) {  /* R35: xd = g X, yd = g Y (no distortion parameters) */
        double X = Xc[0], Y = Xc[1], rho = sqrt(X * X + Y * Y), th = atan2(rho, (double)Xc[2]);
        double g = rho > 0.0 ? th / rho : 1.0 / (double)Xc[2];
        xd = g * X;
        yd = g * Y;
    }
    if (c->model == 1) {
        double r2 = xn * xn + yn * yn;
        double r[3] = {r2, r2 * r2, r2 * r2 * r2};
        double num = 1.0 + c->k[0] * r[0] + c->k[1] * r[1] + c->k[2] * r[2];
        double den = 1.0 + c->k[3] * r[0] + c->k[4] * r[1] + c->k[5] * r[2];
        double rad = num / den;
        xd = xn * rad + 2.0 * c->p[0] * xn * yn + c->p[1] * (r2 + 2.0 * xn * xn);
        yd = yn * rad + c->p[0] * (r2 + 2.0 * yn * yn) + 2.0 * c->p[1] * xn * yn;
        for (int i = 0; i < 3; ++i) {
            double drad_num = r[i] / den;                 /* d rad / d k_{i+1} */
            double drad_den = -num * r[i] / (den * den);  /* d rad / d k_{i+4} */
            Jt[0 * 12 + 4 + i] = c->fx * xn * drad_num;
            Jt[1 * 12 + 4 + i] = c->fy * yn * drad_num;
            Jt[0 * 12 + 7 + i] = c->fx * xn * drad_den;
            Jt[1 * 12 + 7 + i] = c->fy * yn * drad_den;
        }
        Jt[0 * 12 + 10] = c->fx * 2.0 * xn * yn;          /* p1 */
        Jt[1 * 12 + 10] = c->fy * (r2 + 2.0 * yn * yn);
        Jt[0 * 12 + 11] = c->fx * (r2 + 2.0 * xn * xn);   /* p2 */
        Jt[1 * 12 + 11] = c->fy * 2.0 * xn * yn;
    }
    Jt[0 * 12 + 0] = xd;   /* fx */
    Jt[1 * 12 + 1] = yd;   /* fy */
    Jt[0 * 12 + 2] = 1.0;  /* cx */
    Jt[1 * 12 + 3] = 1.0;  /* cy */
}

/* Ghost image-space gradient at layer l, pixel (u,v) (Eqs. 9-11, R14-R16):
 * g = (g_u, g_v) in layer-l pixels; gabs = per-direction sums of |G.Delta|/2. */
static void ghost_layer_grad(const orc_camera *c, const orc_params *pr, int l, int64_t local, int32_t C,
                             const double *tau, float z, const uint64_t *kv, const double *cv, const double *img,
                             const float *Gv, int64_t P, double *g, double *gabs)
{
    int32_t wl = layer_w(c->width, l), hl = layer_w(c->height, l);
    int64_t off = layer_offset(c->width, c->height, l);
    int64_t hw = (int64_t)wl * hl;
    int64_t u = local % wl, vv = local / wl;
    static const int du[4] = {+1, -1, 0, 0}, dv[4] = {0, 0, +1, -1};
    double d[4], dabs[4];
    double Iq[32], delta[32];
    (void)P;
    for (int k = 0; k < 4; ++k) {
        int64_t qu = u + du[k], qv = vv + dv[k];
        d[k] = 0.0; dabs[k] = 0.0;
        if (qu < 0 || qu >= wl || qv < 0 || qv >= hl) continue; /* neighbour outside: no term (R14) */
        int64_t qj = qv * wl + qu;
        for (int ch = 0; ch < C; ++ch) Iq[ch] = img[C * off + ch * hw + qj];
        int kase = induced_change_d(C, tau, z, pr->alpha, cv[off + qj], kv[off + qj], Iq, delta);
        /* magnitude scale for tolerances: sum_c |G| (|tau| + |I|) times the case factor */
        double fac = kase == 2 ? 0.0 : (kase == 4 ? 1.0 / (cv[off + qj] + 1.0) : 1.0);
        for (int ch = 0; ch < C; ++ch) {
            double gq = (double)Gv[C * off + ch * hw + qj];
            d[k] += gq * delta[ch];
            dabs[k] += fabs(gq) * (fabs(tau[ch]) + fabs(Iq[ch])) * fac;
        }
    }
    g[0] = 0.5 * (d[0] - d[1]);   /* Eq. 10 with the signed central difference (R15) */
    g[1] = 0.5 * (d[2] - d[3]);
    gabs[0] = 0.5 * dabs[0]; gabs[1] = 0.5 * dabs[1];
    gabs[2] = 0.5 * dabs[2]; gabs[3] = 0.5 * dabs[3];
}

/* One point of the backward in one view (the loop body of orc_backward): texture gradient of a rendered point
 * into dtau[i] (R24), spatial gradient (ghost, or rendered point with spatial_rendered) into dx[i] (R17, R21),
 * and its pose / intrinsics terms into slot: [0] = 1 if any, [1..6] d_pose, [7..12] their scales,
 * [13..24] d_intrinsics, [25..36] their scales.  Writes only point i's entries and its own slot. */
#define SLOT 37
static void backward_point(const orc_points *pts, int64_t i, unsigned m, const int64_t *pix, const float *proj,
                           const orc_camera *c, const orc_pose *Pz, const orc_params *pr, const uint64_t *kv,
                           const double *cv, const double *img, const float *Gv, int64_t P, double *dtau,
                           double *dx, double *dtau_abs, double *dx_abs, int want_intr, double *slot)
{
    const int C = pts->channels;
    const int64_t n = pts->n;
    slot[0] = 0.0;
    if (!(m & 0x7Fu)) return;
    double tau[32];  /* linear-space descriptor */
    for (int ch = 0; ch < C; ++ch) tau[ch] = desc_lin(pr, pts->feat[i * C + ch]);
    if (!(m & 0x80u)) {
        /* rendered point: texture gradient of Eq. 7, dI/dtau = 1/|Lambda| (R24) */
        for (int l = 0; l < pr->layers; ++l) {
            if (!(m & (1u << l))) continue;
            int64_t off = layer_offset(c->width, c->height, l);
            int64_t q = off + pix[l];
            if (!fuzzy_pass(proj[6], kv[q], pr->alpha)) continue;
            int64_t hw = (int64_t)layer_w(c->width, l) * layer_w(c->height, l);
            for (int ch = 0; ch < C; ++ch) {
                /* d tau_lin / d tau = exp(tau) = tau_lin for log descriptors, 1 otherwise */
                double t = (double)Gv[C * off + ch * hw + pix[l]] / cv[q] * (pr->log_descriptors ? tau[ch] : 1.0);
                if (dtau) dtau[i * C + ch] += t;
                if (dtau_abs) dtau_abs[i * C + ch] += fabs(t);
            }
        }
        if (!pr->spatial_rendered) return;
    } else if (pr->spatial_rendered) {
        return;  /* ghost gradients disabled: ghosts take no part at all */
    }
    /* spatial gradient (ghost point, or a rendered point with ghost gradients disabled): image-space
     * gradient of Eqs. 9-11 summed over layers in layer-0 pixels (R17) */
    double gu = 0.0, gv = 0.0, ga[4] = {0, 0, 0, 0};
    for (int l = 0; l < pr->layers; ++l) {
        if (!(m & (1u << l))) continue;
        double g[2], gabs[4];
        ghost_layer_grad(c, pr, l, pix[l], C, tau, proj[6], kv, cv, img, Gv, P, g, gabs);
        double s = ldexp(1.0, -l);
        gu += s * g[0]; gv += s * g[1];
        for (int k = 0; k < 4; ++k) ga[k] += s * gabs[k];
    }
    double J[6];
    orc_jacobian(c, proj, J);
    /* w = J^T g = dL/dXc */
    double w[3], wu[3], wv[3];
    for (int k = 0; k < 3; ++k) {
        w[k] = J[k] * gu + J[3 + k] * gv;
        wu[k] = J[k];
        wv[k] = J[3 + k];
    }
    const float *R = Pz->R;
    double X[3] = {proj[0], proj[1], proj[2]};
    /* tolerance scale: rounding errors of w live in camera space and R^T mixes them into every
     * component, so each component's scale is the 2-norm of the term vectors R^T J^T e. */
    double nu = sqrt(wu[0] * wu[0] + wu[1] * wu[1] + wu[2] * wu[2]);
    double nv = sqrt(wv[0] * wv[0] + wv[1] * wv[1] + wv[2] * wv[2]);
    for (int k = 0; k < 3; ++k) {
        /* dx = R^T w (Xc = R x + t) */
        double a = R[0 + k] * w[0] + R[3 + k] * w[1] + R[6 + k] * w[2];
        if (dx) dx[k * n + i] += a;
        if (dx_abs) dx_abs[k * n + i] += (ga[0] + ga[1]) * nu + (ga[2] + ga[3]) * nv;
    }
    slot[0] = 1.0;
    if (want_intr) {
        /* NEXT-1: d theta = Jt^T g (layer-0 pixel gradient, R17) */
        double Jt[24];
        orc_intrinsics_jacobian(c, proj, Jt);
        for (int k = 0; k < 12; ++k) {
            slot[13 + k] = Jt[k] * gu + Jt[12 + k] * gv;
            slot[25 + k] = (ga[0] + ga[1]) * fabs(Jt[k]) + (ga[2] + ga[3]) * fabs(Jt[12 + k]);
        }
    } else {
        for (int k = 13; k < SLOT; ++k) slot[k] = 0.0;
    }
    /* Eq. 17 left perturbation: dXc/dxi = [I | -[Xc]x] -> (w, Xc x w) (R19) */
    double cr[3] = {X[1] * w[2] - X[2] * w[1], X[2] * w[0] - X[0] * w[2], X[0] * w[1] - X[1] * w[0]};
    double cu[3] = {X[1] * wu[2] - X[2] * wu[1], X[2] * wu[0] - X[0] * wu[2], X[0] * wu[1] - X[1] * wu[0]};
    double cvv[3] = {X[1] * wv[2] - X[2] * wv[1], X[2] * wv[0] - X[0] * wv[2], X[0] * wv[1] - X[1] * wv[0]};
    double ncu = sqrt(cu[0] * cu[0] + cu[1] * cu[1] + cu[2] * cu[2]);
    double ncv = sqrt(cvv[0] * cvv[0] + cvv[1] * cvv[1] + cvv[2] * cvv[2]);
    for (int k = 0; k < 3; ++k) {
        slot[1 + k] = w[k];
        slot[4 + k] = cr[k];
        slot[7 + k] = (ga[0] + ga[1]) * nu + (ga[2] + ga[3]) * nv;
        slot[10 + k] = (ga[0] + ga[1]) * ncu + (ga[2] + ga[3]) * ncv;
    }
}

/* ------------------------------------------------------------------------- */
/* Backward.  Inputs: the forward's keys/count/image (re-render) and */
/* the upstream gradient G = dL/dI (image layout).  Outputs (overwritten):   */
/*   dtau [n][C]   texture gradient of rendered points (R24; ghosts 0)       */
/*   dx   [3][n]   position gradient of ghost points (R17, R22; others 0)    */
/*   dpose [V][6]  tangent-space pose gradient (w, Xc x w) (R19)             */
/*   dintr [V][12] intrinsics gradient (NEXT-1): sum over ghosts of          */
/*                 (d(u0,v0)/d theta)^T (g_u, g_v), theta as in              */
/*                 orc_intrinsics_jacobian                                   */
/*   denv [H][W][C] environment-map gradient (NEXT-2; "straightforward",     */
/*                 P:L253): every empty pixel's G scattered to its 4         */
/*                 bilinear taps (R29); only with env                        */
/* and the per-element sums of |terms| used to scale tolerances (R20).       */
/* Log descriptors (NEXT-2): the texture gradient carries d exp(tau)/d tau   */
/* and the ghosts' Eq. 11 uses the linear descriptor exp(tau).               */
/* Any output pointer may be NULL.                                           */
/* ------------------------------------------------------------------------- */
void orc_backward(const orc_points *pts, int32_t n_views, const orc_camera *cams, const orc_pose *poses,
                  const orc_params *pr, const orc_env *env, const uint64_t *keys, const double *count,
                  const double *image, const float *G, double *dtau, double *dx, double *dpose, double *dintr,
                  double *denv, double *dtau_abs, double *dx_abs, double *dpose_abs, double *dintr_abs,
                  double *denv_abs)
{
    const int C = pts->channels;
    const int64_t n = pts->n;
    orc_chunk ck;
    double *slot = (double *)malloc(sizeof(double) * SLOT * (size_t)ORC_CHUNK);
    if (!chunk_alloc(&ck) || !slot) abort();
    if (dtau) memset(dtau, 0, sizeof(double) * (size_t)(n * C));
    if (dtau_abs) memset(dtau_abs, 0, sizeof(double) * (size_t)(n * C));
    if (dx) memset(dx, 0, sizeof(double) * (size_t)(3 * n));
    if (dx_abs) memset(dx_abs, 0, sizeof(double) * (size_t)(3 * n));
    if (dpose) memset(dpose, 0, sizeof(double) * (size_t)(6 * n_views));
    if (dpose_abs) memset(dpose_abs, 0, sizeof(double) * (size_t)(6 * n_views));
    if (dintr) memset(dintr, 0, sizeof(double) * (size_t)(12 * n_views));
    if (dintr_abs) memset(dintr_abs, 0, sizeof(double) * (size_t)(12 * n_views));
    const int64_t nenv = (env && env->data) ? (int64_t)env->width * env->height * C : 0;
    if (denv) memset(denv, 0, sizeof(double) * (size_t)nenv);
    if (denv_abs) memset(denv_abs, 0, sizeof(double) * (size_t)nenv);
    int64_t Gbase = 0;
    for (int v = 0; v < n_views; ++v) {
        const orc_camera *c = &cams[v];
        const orc_pose *Pz = &poses[v];
        int64_t P = orc_pyramid_pixels(c->width, c->height, pr->layers);
        const uint64_t *kv = keys + (int64_t)v * P;
        const double *cv = count + (int64_t)v * P;
        const double *img = image + Gbase;
        const float *Gv = G + Gbase;
        Gbase += (int64_t)C * P;
        if (nenv && (denv || denv_abs)) {
            /* environment map: I = sum_k w_k E[idx_k] on empty pixels -> dE[idx_k] += w_k G */
            for (int l = 0; l < pr->layers; ++l) {
                int64_t off = layer_offset(c->width, c->height, l);
                int32_t wl = layer_w(c->width, l);
                int64_t hw = (int64_t)wl * layer_w(c->height, l);
                for (int64_t j = 0; j < hw; ++j) {
                    if (cv[off + j] != 0.0) continue;
                    double d[3], w[4];
                    int64_t idx[4];
                    orc_env_dir(c, Pz, l, j % wl, j / wl, d);
                    orc_env_taps(env, d, idx, w);
                    for (int k = 0; k < 4; ++k)
                        for (int ch = 0; ch < C; ++ch) {
                            double t = w[k] * (double)Gv[C * off + ch * hw + j];
                            if (denv) denv[idx[k] * C + ch] += t;
                            /* tolerance scale: |G| per tap (the fp32 lookup's weights err by ~(W + H) 2^-22) */
                            if (denv_abs) denv_abs[idx[k] * C + ch] += fabs((double)Gv[C * off + ch * hw + j]);
                        }
                }
            }
        }
        for (int64_t i0 = 0; i0 < n; i0 += ORC_CHUNK) {
            int64_t cnt = n - i0 < ORC_CHUNK ? n - i0 : ORC_CHUNK;
            chunk_masks(pts, i0, cnt, c, Pz, pr, (uint32_t)(pr->view_id_base + v), &ck);
            /* map: every point writes its own d_tau / d_x entries and its pose / intrinsics terms into its slot */
            #pragma omp parallel for schedule(static) num_threads(orc_threads)
            for (int64_t j = 0; j < cnt; ++j)
                backward_point(pts, i0 + j, ck.mask[j], ck.pix + 8 * j, ck.proj + 8 * j, c, Pz, pr, kv, cv, img, Gv,
                               P, dtau, dx, dtau_abs, dx_abs, dintr || dintr_abs, slot + SLOT * j);
            /* reduce: per-view sums over points, serially in point order */
            for (int64_t j = 0; j < cnt; ++j) {
                const double *sl = slot + SLOT * j;
                if (sl[0] == 0.0) continue;
                for (int k = 0; k < 6; ++k) {
                    if (dpose) dpose[v * 6 + k] += sl[1 + k];
                    if (dpose_abs) dpose_abs[v * 6 + k] += sl[7 + k];
                }
                for (int k = 0; k < 12; ++k) {
                    if (dintr) dintr[v * 12 + k] += sl[13 + k];
                    if (dintr_abs) dintr_abs[v * 12 + k] += sl[25 + k];
                }
            }
        }
    }
    chunk_free(&ck);
    free(slot);
}
