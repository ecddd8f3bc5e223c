// adop_device.cuh -- device-side building blocks of the sm_100a rasterizer.
//
// Every operation that decides an integer (pixel index, bounds, depth key,
// discard / ghost bits, fuzzy and Eq. 11 case choices) uses explicitly
// rounded fp32 intrinsics (__fmul_rn / __fadd_rn / __frcp_rn / __fdiv_rn) in
// the operation order fixed by DESIGN.md R1-R14, so nvcc cannot contract it
// into FMAs; this is what makes keys and masks bit-identical to the CPU oracle.
// Citations: PAPER.md line numbers (Lnnn) with the equation they belong to.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "adop_internal.h"

namespace adop {

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }

// Round half away from zero (Eq. 3, reading R3).  x - trunc(x) is exact.
__device__ __forceinline__ float round_away(float x) {
    float t = truncf(x);
    float d = __fsub_rn(x, t);
    return fabsf(d) >= 0.5f ? __fadd_rn(t, copysignf(1.0f, x)) : t;
}

// 2^-l as an exact float (Eq. 2's 1/2^l).
__device__ __forceinline__ float pow2_neg(int l) { return __int_as_float((127 - l) << 23); }

// Counter-based hash (R11, R13): integer finalizer with two odd multipliers.
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t h24(uint32_t salt, uint32_t gi) { return mix32(gi ^ salt) >> 8; }

// Projection result of one point in one view (Eq. 2 with camera model R6).
struct Proj {
    float X, Y, Z;  // camera-space point (R1)
    float u0, v0;   // layer-0 continuous pixel coordinates
    float iz;       // 1 / D (IEEE)
    float D;        // depth of keys and Eq. 6 (R4): Z, or the distance |Xc| for the fisheye (R35)
};

// R35: atan(t), t in [0, 1], as t * P(t^2) with the fixed degree-9 polynomial of DESIGN.md R35, Horner in fp32
// with one rounding per operation (identical to the oracle's), and the angle in [0, pi] of (x, y), y >= 0.
__device__ __forceinline__ float atan01(float t) {
    const float c[10] = {-0.0015244261594489217f, 0.009669913910329342f, -0.028764614835381508f,
                         0.05541255697607994f, -0.08245089650154114f, 0.10893233865499496f,
                         -0.14251546561717987f, 0.1999710500240326f, -0.33333227038383484f, 1.0f};
    const float u = __fmul_rn(t, t);
    float p = c[0];
#pragma unroll
    for (int k = 1; k < 10; ++k) p = __fadd_rn(__fmul_rn(p, u), c[k]);
    return __fmul_rn(t, p);
}
__device__ __forceinline__ float atan2p(float y, float x) {
    const float ax = fabsf(x);
    float a;
    if (y <= ax) a = ax > 0.0f ? atan01(__fdiv_rn(y, ax)) : 0.0f;
    else a = __fsub_rn(1.57079632679490f, atan01(__fdiv_rn(ax, y)));
    return x >= 0.0f ? a : __fsub_rn(3.14159265358979f, a);
}

// Validity (R7 / R35) and the depth D of a camera point; sets p.D and p.iz = 1/D.  Pinned fp32.
template <int MODEL>
__device__ __forceinline__ bool depth_valid(Proj &p, float z_near) {
    if (MODEL == 2) {
        const float rho2 = __fadd_rn(__fmul_rn(p.X, p.X), __fmul_rn(p.Y, p.Y));
        p.D = __fsqrt_rn(__fadd_rn(rho2, __fmul_rn(p.Z, p.Z)));
    } else {
        p.D = p.Z;
    }
    if (!(p.D > z_near && p.D <= 3.402823466e38f)) return false;
    p.iz = __frcp_rn(p.D);
    return true;
}

// Xc = R x + t in the pinned order ((r0 x + r1 y) + r2 z) + t (R1).
__device__ __forceinline__ void to_camera(const ViewDesc &v, float x, float y, float z, float &X, float &Y,
                                          float &Z) {
    X = fadd(fadd(fadd(fmul(v.R[0], x), fmul(v.R[1], y)), fmul(v.R[2], z)), v.t[0]);
    Y = fadd(fadd(fadd(fmul(v.R[3], x), fmul(v.R[4], y)), fmul(v.R[5], z)), v.t[1]);
    Z = fadd(fadd(fadd(fmul(v.R[6], x), fmul(v.R[7], y)), fmul(v.R[8], z)), v.t[2]);
}

// OpenCV8 image window in undistorted normalized coordinates (ViewDesc::wn, computed and widened on the host):
// false only if the pinned camera point (Z > 0) cannot land in any layer.
__device__ __forceinline__ bool in_window(const ViewDesc &v, float X, float Y, float Z) {
    return X >= v.wn[0] * Z && X <= v.wn[1] * Z && Y >= v.wn[2] * Z && Y <= v.wn[3] * Z;
}
// The same test on the FMA-evaluated point with the pre-cull margin m (|Xf - Xp|, |Zf - Zp| <= m).
__device__ __forceinline__ bool in_window_fma(const ViewDesc &v, float X, float Y, float Z, float m) {
    return X >= fmaf(v.wn[0], Z, -m * (1.0f + fabsf(v.wn[0]))) && X <= fmaf(v.wn[1], Z, m * (1.0f + fabsf(v.wn[1]))) &&
           Y >= fmaf(v.wn[2], Z, -m * (1.0f + fabsf(v.wn[2]))) && Y <= fmaf(v.wn[3], Z, m * (1.0f + fabsf(v.wn[3])));
}

// Conservative, division-free frustum test (never rejects a point the exact
// per-layer test would accept).  Z > z_near already holds.
template <int MODEL>
__device__ __forceinline__ bool precull_pass(const ViewDesc &v, float X, float Y, float Z) {
    if (MODEL == 2 && !(v.r2cull <= 3.402823466e38f)) return true;  // fisheye wider than 180 degrees
    if (MODEL == 0) {
        float su = fmaf(v.fx, X, v.cx * Z);
        float sv = fmaf(v.fy, Y, v.cy * Z);
        return su >= v.ulo * Z && su <= v.uhi * Z && sv >= v.vlo * Z && sv <= v.vhi * Z;
    } else {
        float r2z = fmaf(X, X, Y * Y);
        if (MODEL == 1 && v.wn_on && !in_window(v, X, Y, Z)) return false;
        return r2z <= v.r2cull * (Z * Z);
    }
}

// Conservative pre-cull evaluated with FMAs straight from the world point (no pinned ops):
// never rejects a point whose pinned projection lands in some layer (margin fk*B + fkt covers the
// difference between the FMA and the pinned evaluation of R x + t).
template <int MODEL>
__device__ __forceinline__ bool precull_fma(const ViewDesc &v, float x, float y, float z) {
    const float X = fmaf(v.R[0], x, fmaf(v.R[1], y, fmaf(v.R[2], z, v.t[0])));
    const float Y = fmaf(v.R[3], x, fmaf(v.R[4], y, fmaf(v.R[5], z, v.t[1])));
    const float Z = fmaf(v.R[6], x, fmaf(v.R[7], y, fmaf(v.R[8], z, v.t[2])));
    const float m = fmaf(v.fk, fabsf(x) + fabsf(y) + fabsf(z), v.fkt);
    if (MODEL == 0) {
        const float su = fmaf(v.fx, X, v.cx * Z);
        const float sv = fmaf(v.fy, Y, v.cy * Z);
        const float d0 = fmaf(-v.ulo, Z, su), d1 = fmaf(v.uhi, Z, -su);
        const float d2 = fmaf(-v.vlo, Z, sv), d3 = fmaf(v.vhi, Z, -sv);
        return fminf(fminf(d0, d1), fminf(d2, d3)) >= -m;
    } else if (MODEL == 2 && !(v.r2cull <= 3.402823466e38f)) {
        return true;  // fisheye wider than 180 degrees: no cone
    } else {
        // |Xp| >= |Xf| - m etc.: (|Xf|-m)+^2 + (|Yf|-m)+^2 <= r2cull (|Zf|+m)^2 is implied by the exact test
        const float ax = fmaxf(fabsf(X) - m, 0.0f), ay = fmaxf(fabsf(Y) - m, 0.0f), az = fabsf(Z) + m;
        if (MODEL == 1 && v.wn_on && !in_window_fma(v, X, Y, Z, m)) return false;
        return Z >= -m && fmaf(ax, ax, ay * ay) <= v.r2cull * (az * az);
    }
}

// Same test, also returning the FMA depth and the margin (for the early discard test).
template <int MODEL>
__device__ __forceinline__ bool precull_fma_z(const ViewDesc &v, float x, float y, float z, float &Zo, float &mo) {
    const float X = fmaf(v.R[0], x, fmaf(v.R[1], y, fmaf(v.R[2], z, v.t[0])));
    const float Y = fmaf(v.R[3], x, fmaf(v.R[4], y, fmaf(v.R[5], z, v.t[1])));
    const float Z = fmaf(v.R[6], x, fmaf(v.R[7], y, fmaf(v.R[8], z, v.t[2])));
    const float m = fmaf(v.fk, fabsf(x) + fabsf(y) + fabsf(z), v.fkt);
    Zo = Z;
    mo = m;
    if (MODEL == 2 && !(v.r2cull <= 3.402823466e38f)) return true;  // fisheye wider than 180 degrees
    if (MODEL == 0) {
        const float su = fmaf(v.fx, X, v.cx * Z);
        const float sv = fmaf(v.fy, Y, v.cy * Z);
        const float d0 = fmaf(-v.ulo, Z, su), d1 = fmaf(v.uhi, Z, -su);
        const float d2 = fmaf(-v.vlo, Z, sv), d3 = fmaf(v.vhi, Z, -sv);
        return fminf(fminf(d0, d1), fminf(d2, d3)) >= -m;
    } else {
        const float ax = fmaxf(fabsf(X) - m, 0.0f), ay = fmaxf(fabsf(Y) - m, 0.0f), az = fabsf(Z) + m;
        if (MODEL == 1 && v.wn_on && !in_window_fma(v, X, Y, Z, m)) return false;
        return Z >= -m && fmaf(ax, ax, ay * ay) <= v.r2cull * (az * az);
    }
}

// Exact projection to layer-0 pixels given p.X, p.Y, p.Z (pinned) and p.iz = 1/Z (R2, R6).
template <int MODEL>
__device__ __forceinline__ bool project_uv(const ViewDesc &v, Proj &p) {
    if (MODEL == 2) {  // R35 equidistant: theta = atan2(rho, Z) <= theta_max, r_d = f theta
        const float rho = __fsqrt_rn(__fadd_rn(__fmul_rn(p.X, p.X), __fmul_rn(p.Y, p.Y)));
        const float th = atan2p(rho, p.Z);
        if (!(th <= v.r2_max)) return false;
        const float s = rho > 0.0f ? __fdiv_rn(th, rho) : 0.0f;
        p.u0 = fadd(fmul(v.fx, fmul(p.X, s)), v.cx);
        p.v0 = fadd(fmul(v.fy, fmul(p.Y, s)), v.cy);
        return true;
    }
    float xn = fmul(p.X, p.iz), yn = fmul(p.Y, p.iz);
    float xd = xn, yd = yn;
    if (MODEL == 1) {
        float xx = fmul(xn, xn), yy = fmul(yn, yn), xy = fmul(xn, yn);
        float r2 = fadd(xx, yy);
        if (!(r2 <= v.r2_max)) return false;
        float r4 = fmul(r2, r2), r6 = fmul(r4, r2);
        float num = fadd(fadd(fadd(1.0f, fmul(v.k[0], r2)), fmul(v.k[1], r4)), fmul(v.k[2], r6));
        float den = fadd(fadd(fadd(1.0f, fmul(v.k[3], r2)), fmul(v.k[4], r4)), fmul(v.k[5], r6));
        if (!(den > 0.0f)) return false;
        float radial = __fdiv_rn(num, den);
        float a1 = fmul(2.0f, xy);
        float a2 = fadd(r2, fmul(2.0f, xx));
        float a3 = fadd(r2, fmul(2.0f, yy));
        xd = fadd(fadd(fmul(xn, radial), fmul(v.p[0], a1)), fmul(v.p[1], a2));
        yd = fadd(fadd(fmul(yn, radial), fmul(v.p[0], a3)), fmul(v.p[1], a1));
    }
    p.u0 = fadd(fmul(v.fx, xd), v.cx);
    p.v0 = fadd(fmul(v.fy, yd), v.cy);
    return true;
}

// Full projection of a point: validity (R7 / R35), pre-cull, exact projection.
template <int MODEL>
__device__ __forceinline__ bool project_point(const ViewDesc &v, float z_near, float x, float y, float z, Proj &p) {
    to_camera(v, x, y, z, p.X, p.Y, p.Z);
    if (!depth_valid<MODEL>(p, z_near)) return false;
    if (!precull_pass<MODEL>(v, p.X, p.Y, p.Z)) return false;
    return project_uv<MODEL>(v, p);
}

// Eq. 12 (L344) as R10/R11: number of leading layers at which the point is kept.
__device__ __forceinline__ int keep_layers(const RasterArgs &a, const ViewDesc &v, float rw, float iz, uint32_t gi) {
    if (!a.discard) return a.layers;
    float rs0 = fmul(fmul(rw, v.feff), iz);
    uint32_t h = h24(v.discard_salt, gi);
    float om = fmul((float)(16777216u - h), 5.9604644775390625e-8f);  // 1 - beta, exact
    int l = 0;
#pragma unroll
    for (int k = 0; k < ADOP_MAX_LAYERS; ++k) {
        if (k < a.layers) {
            float al = fmul(a.gamma, fmul(rs0, pow2_neg(k)));
            if (l == k && fmul(al, al) > om) l = k + 1;
        }
    }
    return l;
}

// True unless the point is outside the image at every layer l < nk (then no layer_pixel call can hit):
// round_away(u0 2^-l) is in [0, w_l) only if -2^(l-1) < u0 < (w_l - 1/2) 2^l <= w + 2^(l-1), and the widest
// of these over l < nk is l = nk - 1.  Exact (power-of-two scalings), so dropping the point changes nothing.
template <typename VD>
__device__ __forceinline__ bool any_layer_in_bounds(const VD &v, const Proj &p, int nk) {
    const float hs = __int_as_float((126 + nk) << 23);  // 2^(nk - 2) = 0.5 * 2^(nk - 1)
    return p.u0 > -hs && p.u0 < (float)v.wl[0] + hs && p.v0 > -hs && p.v0 < (float)v.hl[0] + hs;
}

// Eqs. 3-4: layer-local pixel (u, v) and bounds.  Returns layer-local linear index or -1.
template <typename VD>
__device__ __forceinline__ int layer_pixel(const VD &v, const Proj &p, int l, int &pu, int &pv) {
    float s = pow2_neg(l);
    float ru = round_away(fmul(p.u0, s));
    float rv = round_away(fmul(p.v0, s));
    if (!(ru >= 0.0f && ru < (float)v.wl[l] && rv >= 0.0f && rv < (float)v.hl[l])) return -1;
    pu = (int)ru;
    pv = (int)rv;
    return pv * v.wl[l] + pu;
}

// Normal culling, Eq. 5 with reading R32: sign of (R n) . Xc in the pinned fp32 order of R1
// (|Xc| > 0 drops out); normal_cull +1 keeps (Rn).Xc > 0 as printed, -1 keeps < 0.  The normal is gathered
// only here, on the exact path of the points that survived the pre-cull.
__device__ __forceinline__ bool normal_keep(const RasterArgs &a, const ViewDesc &v, int64_t i, float X, float Y,
                                            float Z) {
    if (a.normal_cull == 0) return true;
    const float nx = __ldg(a.nrm + i), ny = __ldg(a.nrm + a.nrm_stride + i), nz = __ldg(a.nrm + 2 * a.nrm_stride + i);
    const float ncx = fadd(fadd(fmul(v.R[0], nx), fmul(v.R[1], ny)), fmul(v.R[2], nz));
    const float ncy = fadd(fadd(fmul(v.R[3], nx), fmul(v.R[4], ny)), fmul(v.R[5], nz));
    const float ncz = fadd(fadd(fmul(v.R[6], nx), fmul(v.R[7], ny)), fmul(v.R[8], nz));
    const float dot = fadd(fadd(fmul(ncx, X), fmul(ncy, Y)), fmul(ncz, Z));
    return a.normal_cull > 0 ? dot > 0.0f : dot < 0.0f;
}

// Linear-space descriptor channel (NEXT-2): exp(tau) for log descriptors.
__device__ __forceinline__ float desc_lin(const RasterArgs &a, float t) { return a.log_desc ? expf(t) : t; }

// Environment map E of Eq. 7 (NEXT-2, reading R29): bilinear taps (texel = row * W + col) and weights of
// layer-l pixel (u, v): layer-0 (u 2^l, v 2^l), C^-1 (pinhole inverse; OpenCV8: 8 Newton steps on R6's
// distortion map from the distorted coordinates), d = R^T (xn, yn, 1), lon = atan2(dx, dz),
// lat = atan2(dy, hypot(dx, dz)), s = (lon / 2pi + 1/2) W - 1/2, t = (lat / pi + 1/2) H - 1/2; columns
// wrap, rows clamp.  Continuous in (u, v) -> compared with the oracle's fp64 within tolerance.
__device__ __forceinline__ void env_taps(const RasterArgs &a, const ViewDesc &v, int l, int u, int vv, int idx[4],
                                         float w[4]) {
    const float u0 = ldexpf((float)u, l), v0 = ldexpf((float)vv, l);
    const float xd = (u0 - v.cx) / v.fx, yd = (v0 - v.cy) / v.fy;
    float x = xd, y = yd, zc = 1.f;
    if (v.model == 2) {  // R35: theta = |(xd, yd)|, direction (sin theta xd / theta, sin theta yd / theta, cos theta)
        const float th = sqrtf(xd * xd + yd * yd), s = th > 0.f ? sinf(th) / th : 1.f;
        x = s * xd;
        y = s * yd;
        zc = cosf(th);
    } else if (v.model == ADOP_OPENCV8) {
        for (int it = 0; it < 8; ++it) {
            const float r2 = x * x + y * y;
            const float num = 1.f + r2 * (v.k[0] + r2 * (v.k[1] + r2 * v.k[2]));
            const float den = 1.f + r2 * (v.k[3] + r2 * (v.k[4] + r2 * v.k[5]));
            const float dnum = v.k[0] + r2 * (2.f * v.k[1] + 3.f * r2 * v.k[2]);
            const float dden = v.k[3] + r2 * (2.f * v.k[4] + 3.f * r2 * v.k[5]);
            const float rad = num / den, drad = (dnum * den - num * dden) / (den * den);
            const float fx_ = x * rad + 2.f * v.p[0] * x * y + v.p[1] * (r2 + 2.f * x * x);
            const float fy_ = y * rad + v.p[0] * (r2 + 2.f * y * y) + 2.f * v.p[1] * x * y;
            const float D00 = rad + 2.f * x * x * drad + 2.f * v.p[0] * y + 6.f * v.p[1] * x;
            const float D01 = 2.f * x * y * drad + 2.f * v.p[0] * x + 2.f * v.p[1] * y;
            const float D11 = rad + 2.f * y * y * drad + 6.f * v.p[0] * y + 2.f * v.p[1] * x;
            const float rx = fx_ - xd, ry = fy_ - yd, idet = 1.f / (D00 * D11 - D01 * D01);
            x -= (D11 * rx - D01 * ry) * idet;
            y -= (-D01 * rx + D00 * ry) * idet;
        }
    }
    const float dx = v.R[0] * x + v.R[3] * y + v.R[6] * zc, dy = v.R[1] * x + v.R[4] * y + v.R[7] * zc;
    const float dz = v.R[2] * x + v.R[5] * y + v.R[8] * zc;
    const float lon = atan2f(dx, dz), lat = atan2f(dy, sqrtf(dx * dx + dz * dz));
    const float s = (lon * 0.15915494309189535f + 0.5f) * (float)a.env_w - 0.5f;
    const float t = (lat * 0.3183098861837907f + 0.5f) * (float)a.env_h - 0.5f;
    const float s0 = floorf(s), t0 = floorf(t), fs = s - s0, ft = t - t0;
    int c0 = (int)s0 % a.env_w;
    if (c0 < 0) c0 += a.env_w;
    const int c1 = c0 + 1 == a.env_w ? 0 : c0 + 1;
    const int r0i = (int)t0;
    const int r0 = r0i < 0 ? 0 : (r0i >= a.env_h ? a.env_h - 1 : r0i);
    const int r1 = r0i + 1 < 0 ? 0 : (r0i + 1 >= a.env_h ? a.env_h - 1 : r0i + 1);
    idx[0] = r0 * a.env_w + c0; w[0] = (1.f - ft) * (1.f - fs);
    idx[1] = r0 * a.env_w + c1; w[1] = (1.f - ft) * fs;
    idx[2] = r1 * a.env_w + c0; w[2] = ft * (1.f - fs);
    idx[3] = r1 * a.env_w + c1; w[3] = ft * fs;
}

__device__ __forceinline__ uint64_t depth_key(float Z, uint32_t gi) {
    return ((uint64_t)__float_as_uint(Z) << 32) | gi;  // R8
}

// Fuzzy depth test Eq. 6 (L209) as R9: z <= fl(fl(1+alpha) * m).
__device__ __forceinline__ bool fuzzy_pass(float z, uint64_t key, float onepa) {
    return z <= fmul(onepa, __uint_as_float((uint32_t)(key >> 32)));
}

// Streaming loads for the point arrays (read once: evict-first in L1 and L2).
__device__ __forceinline__ float4 ld_stream4(const float *p) { return __ldcs(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ float ld_stream(const float *p) { return __ldcs(p); }

// sm_90+ vector reduction: accum[0..3] += v in one L2 atomic.
__device__ __forceinline__ void red_add_v4(float *addr, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void red_add(float *addr, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(v) : "memory");
}
// Keys are re-read by the blend and the backward: keep their lines in L2 while the cloud streams past.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void red_min_u64_keep(uint64_t *addr, uint64_t v, uint64_t pol) {
    asm volatile("red.global.min.u64.L2::cache_hint [%0], %1, %2;" ::"l"(addr), "l"(v), "l"(pol) : "memory");
}
// Features of blended points are read once: do not let them evict the accumulators.
__device__ __forceinline__ float4 ld_once4(const float *p, uint64_t pol) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void red_min_u64(uint64_t *addr, uint64_t v) {
    asm volatile("red.global.min.u64 [%0], %1;" ::"l"(addr), "l"(v) : "memory");
}

// ---- TMA bulk copies + mbarriers (sm_90+/sm_100a async proxy) ----
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 1-D bulk copy global -> shared (TMA engine, no tensor map), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

// 2-D tensor copy (TMA with a tensor map): box at element coordinates (c0, c1) -> dst, complete_tx on bar.
__device__ __forceinline__ void tensor_g2s_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

// Same, on precomputed shared-window addresses (the depth sweep's per-tile issue path).
__device__ __forceinline__ void mbar_expect_tx_a(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tensor_g2s_2d_a(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t bar,
                                                uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
        : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace adop
