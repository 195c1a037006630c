// ges_device.cuh -- device math shared by the GES kernels (sm_100a).
//
// KEYSPEC: the per-particle geometry that decides keys, rects and
// order is a fixed fp32 op sequence -- every sum of products a left-to-right
// fma chain, every other operation one IEEE-rounded op -- written here with
// explicit round-to-nearest intrinsics so that nvcc can neither contract nor
// reassociate.  The CPU oracle implements the same sequence independently;
// the parity tests require bit equality.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ges {

constexpr int kTile = 16;                 // 16x16 pixel tiles (north_star)
constexpr int kBlock = kTile * kTile;     // one thread per pixel
constexpr float kDilation = 0.3f;         // low-pass dilation of Sigma2D (R7)
constexpr float kAlphaMin = 1.0f / 255.0f;// skip threshold (R7)
constexpr float kAlphaMax = 0.99f;        // alpha clamp (R7)
constexpr float kTMin = 1e-4f;            // transmittance stop (R7, R12)

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float fsqrt(float a) { return __fsqrt_rn(a); }

// KEYSPEC exp: clamp to [-87, 88]; k = rint(x log2e); Cody-Waite r = x - k ln2
// (ln2_hi = 0x3f317200, ln2_lo = 0x35bfbe8e); degree-7 Taylor Horner chain
// with fp32-rounded 1/n!; times 2^k.  <= 2 ulp vs exp over the range.
__device__ __forceinline__ float exp_spec(float x) {
    x = fminf(88.0f, fmaxf(-87.0f, x));
    const float log2e = __uint_as_float(0x3fb8aa3bu);
    const float ln2_hi = __uint_as_float(0x3f317200u);
    const float ln2_lo = __uint_as_float(0x35bfbe8eu);
    const float k = rintf(fmul(x, log2e));
    float r = ffma(-k, ln2_hi, x);
    r = ffma(-k, ln2_lo, r);
    float p = (float)(1.0 / 5040.0);
    p = ffma(p, r, (float)(1.0 / 720.0));
    p = ffma(p, r, (float)(1.0 / 120.0));
    p = ffma(p, r, (float)(1.0 / 24.0));
    p = ffma(p, r, (float)(1.0 / 6.0));
    p = ffma(p, r, 0.5f);
    p = ffma(p, r, 1.0f);
    p = ffma(p, r, 1.0f);
    const int ki = (int)k;
    return fmul(p, __uint_as_float((uint32_t)(ki + 127) << 23));
}

// KEYSPEC log for normal x > 1: x = m 2^e, m folded into [sqrt(1/2), sqrt(2)];
// ln m = 2 atanh(s), s = (m-1)/(m+1), odd Horner chain to s^9; + e ln2.
__device__ __forceinline__ float log_spec(float x) {
    const uint32_t bits = __float_as_uint(x);
    int e = (int)(bits >> 23) - 127;
    float m = __uint_as_float((bits & 0x7fffffu) | 0x3f800000u);
    if (m > 1.41421354f) { m = fmul(m, 0.5f); e += 1; }
    const float s = fdiv(fsub(m, 1.0f), fadd(m, 1.0f));
    const float s2 = fmul(s, s);
    float p = (float)(1.0 / 9.0);
    p = ffma(p, s2, (float)(1.0 / 7.0));
    p = ffma(p, s2, (float)(1.0 / 5.0));
    p = ffma(p, s2, (float)(1.0 / 3.0));
    p = ffma(p, s2, 1.0f);
    float t = fmul(s, p);
    t = fadd(t, t);
    return ffma((float)e, (float)0.69314718055994531, t);
}

// Real spherical harmonics up to degree 3 (Condon-Shortley phase), index
// k = l^2 + l + m, KEYSPEC op order.
struct SHConst {
    static constexpr float C0 = 0.28209479177387814f;
    static constexpr float C1 = 0.48860251190291987f;
    static constexpr float C2a = 1.0925484305920792f;
    static constexpr float C2b = 0.31539156525252005f;
    static constexpr float C2c = 0.54627421529603959f;
    static constexpr float C3a = -0.59004358992664352f;
    static constexpr float C3b = 2.8906114426405538f;
    static constexpr float C3c = -0.45704579946446572f;
    static constexpr float C3d = 0.3731763325901154f;
    static constexpr float C3e = 1.4453057213202769f;
};

template <int K>
__device__ __forceinline__ void sh_basis(float x, float y, float z, float Y[16]) {
    using S = SHConst;
    Y[0] = S::C0;
    if (K <= 1) return;
    Y[1] = fmul(-S::C1, y);
    Y[2] = fmul(S::C1, z);
    Y[3] = fmul(-S::C1, x);
    if (K <= 4) return;
    const float xx = fmul(x, x), yy = fmul(y, y), zz = fmul(z, z);
    const float xy = fmul(x, y), yz = fmul(y, z), xz = fmul(x, z);
    Y[4] = fmul(S::C2a, xy);
    Y[5] = fmul(-S::C2a, yz);
    float t6 = fadd(zz, zz); t6 = fsub(t6, xx); t6 = fsub(t6, yy);
    Y[6] = fmul(S::C2b, t6);
    Y[7] = fmul(-S::C2a, xz);
    const float xmy = fsub(xx, yy);
    Y[8] = fmul(S::C2c, xmy);
    if (K <= 9) return;
    const float xx3 = fmul(3.0f, xx), yy3 = fmul(3.0f, yy);
    float t9 = fsub(xx3, yy); t9 = fmul(y, t9);
    Y[9] = fmul(S::C3a, t9);
    Y[10] = fmul(S::C3b, fmul(xy, z));
    float q4 = fmul(4.0f, zz); q4 = fsub(q4, xx); q4 = fsub(q4, yy);
    Y[11] = fmul(S::C3c, fmul(y, q4));
    float t12 = fadd(zz, zz); t12 = fsub(t12, xx3); t12 = fsub(t12, yy3); t12 = fmul(z, t12);
    Y[12] = fmul(S::C3d, t12);
    Y[13] = fmul(S::C3c, fmul(x, q4));
    Y[14] = fmul(S::C3e, fmul(z, xmy));
    float t15 = fsub(xx, yy3); t15 = fmul(x, t15);
    Y[15] = fmul(S::C3a, t15);
}

// Gradient of each basis function w.r.t. the unit direction (derivatives of
// the polynomials above), accumulated as sum_k w_k dY_k.
template <int K>
__device__ __forceinline__ void sh_basis_grad_dot(float x, float y, float z, const float w[16], float& gx, float& gy,
                                                  float& gz) {
    using S = SHConst;
    gx = gy = gz = 0.0f;
    if (K <= 1) return;
    gy += -S::C1 * w[1];
    gz += S::C1 * w[2];
    gx += -S::C1 * w[3];
    if (K <= 4) return;
    gx += S::C2a * y * w[4];
    gy += S::C2a * x * w[4];
    gy += -S::C2a * z * w[5];
    gz += -S::C2a * y * w[5];
    gx += -2.0f * S::C2b * x * w[6];
    gy += -2.0f * S::C2b * y * w[6];
    gz += 4.0f * S::C2b * z * w[6];
    gx += -S::C2a * z * w[7];
    gz += -S::C2a * x * w[7];
    gx += 2.0f * S::C2c * x * w[8];
    gy += -2.0f * S::C2c * y * w[8];
    if (K <= 9) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    gx += 6.0f * S::C3a * x * y * w[9];
    gy += S::C3a * (3.0f * xx - 3.0f * yy) * w[9];
    gx += S::C3b * y * z * w[10];
    gy += S::C3b * x * z * w[10];
    gz += S::C3b * x * y * w[10];
    gx += -2.0f * S::C3c * x * y * w[11];
    gy += S::C3c * (4.0f * zz - xx - 3.0f * yy) * w[11];
    gz += 8.0f * S::C3c * y * z * w[11];
    gx += -6.0f * S::C3d * x * z * w[12];
    gy += -6.0f * S::C3d * y * z * w[12];
    gz += S::C3d * (6.0f * zz - 3.0f * xx - 3.0f * yy) * w[12];
    gx += S::C3c * (4.0f * zz - 3.0f * xx - yy) * w[13];
    gy += -2.0f * S::C3c * x * y * w[13];
    gz += 8.0f * S::C3c * x * z * w[13];
    gx += 2.0f * S::C3e * x * z * w[14];
    gy += -2.0f * S::C3e * y * z * w[14];
    gz += S::C3e * (xx - yy) * w[14];
    gx += S::C3a * (3.0f * xx - 3.0f * yy) * w[15];
    gy += -6.0f * S::C3a * x * y * w[15];
}

// Camera constants derived on the device (KEYSPEC order), uniform per launch.
struct CamDerived {
    float limx, limy;  // Jacobian clamp: 1.3 * tan(half fov)
    float c0, c1, c2;  // camera centre -R^T t
};

struct CamParams {
    int W, H, tiles_x, tiles_y;
    float fx, fy, cx, cy, near_z;
    float R[9];
    float t[3];
};

__device__ __forceinline__ CamDerived derive_camera(const CamParams& c) {
    CamDerived d;
    d.limx = fmul(1.3f, fdiv(fmul(0.5f, (float)c.W), c.fx));
    d.limy = fmul(1.3f, fdiv(fmul(0.5f, (float)c.H), c.fy));
    float p;
    p = fmul(c.R[0], c.t[0]); p = ffma(c.R[3], c.t[1], p); p = ffma(c.R[6], c.t[2], p); d.c0 = -p;
    p = fmul(c.R[1], c.t[0]); p = ffma(c.R[4], c.t[1], p); p = ffma(c.R[7], c.t[2], p); d.c1 = -p;
    p = fmul(c.R[2], c.t[0]); p = ffma(c.R[5], c.t[1], p); p = ffma(c.R[8], c.t[2], p); d.c2 = -p;
    return d;
}

// Compositing math shared bit-for-bit by the forward and backward kernels.
// The conic is pre-scaled by -log2(e) so that G = 2^(A dx^2 + B dx dy + C dy^2):
//   A = -0.5 a log2e, B = -b log2e, C = -0.5 c log2e.
struct Splat2D {
    float u, v, A, B, C, kappa, r, g, b;
};

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float exponent2(const Splat2D& s, float dx, float dy) {
    // p2 = dx (A dx + B dy) + C dy^2, fixed op order (no contraction freedom)
    const float t1 = __fmaf_rn(s.A, dx, __fmul_rn(s.B, dy));
    const float t2 = __fmul_rn(__fmul_rn(s.C, dy), dy);
    return fminf(__fmaf_rn(dx, t1, t2), 0.0f);
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

}  // namespace ges
