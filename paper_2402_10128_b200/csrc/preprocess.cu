// preprocess.cu -- S1: per-particle projection of GES
// particles and the depth keys of the following radix sort.
//
// Paper: Eq. 2 kernel and Sigma; PAPER.md:249-254 EWA
// Sigma' = J W Sigma W^T J^T with Sigma = R S S^T R^T and S "modified by"
// phi(beta); Eq. 4 (:268-270) effective variance; Eq. 6 (:291-293)
// phi-bar_rho(beta) = 2 / (1 + exp(-(rho beta - 2 rho))); PAPER.md:247 opacity
// and SH colour.  Inherited constants: DESIGN.md R7.  Op order: KEYSPEC
// -- bit-identical to oracle/ges_geom.inc (REAL=float).
//
// HBM-bound: reads 48 B/particle (mean, log-scale, quat, logit, beta) plus 12K
// bytes of SH for visible particles only; coalesced planar loads (lane i of a
// warp reads element i of each plane).
#include <algorithm>

#include "ges_device.cuh"
#include "ges_internal.h"

namespace ges {

struct PreOut {
    float depth, u, v, ca, cb, cc, kappa, r, g, b;
    float hb;    // beta / 2 (exact kernel payload)
    float J[9];  // d rgb / d unit direction, 0 unless visible and unclamped
    int radius, x0, y0, x1, y1;
    uint8_t status, flags;
};

// The 12 per-particle scalars every particle needs (one memory round trip).
struct ParamIn {
    float mx, my, mz, qw, qx, qy, qz, ls0, ls1, ls2, beta, logit;
};

__device__ __forceinline__ ParamIn load_params(const PreprocessArgs& a, int i) {
    const int P = a.P;
    ParamIn p;
    p.mx = __ldg(a.mean + i); p.my = __ldg(a.mean + P + i); p.mz = __ldg(a.mean + 2 * P + i);
    p.qw = __ldg(a.quat + i); p.qx = __ldg(a.quat + P + i); p.qy = __ldg(a.quat + 2 * P + i);
    p.qz = __ldg(a.quat + 3 * P + i);
    p.ls0 = __ldg(a.log_scale + i); p.ls1 = __ldg(a.log_scale + P + i); p.ls2 = __ldg(a.log_scale + 2 * P + i);
    p.beta = __ldg(a.beta + i);
    p.logit = __ldg(a.opacity_logit + i);
    return p;
}

// SH coefficient (plane 3k + ch) of this particle: sh[(3k + ch) * stride]
// (global planes: sh = a.sh + i, stride P; a staged tile: its smem column, stride 128).
template <int K>
__device__ __forceinline__ PreOut preprocess_one(const PreprocessArgs& a, const CamDerived& cd, int i,
                                                 const ParamIn& in, const float* sh, int sh_stride) {
    const int P = a.P;
    const CamParams& c = a.cam;
    PreOut o;
    o.u = o.v = o.ca = o.cb = o.cc = o.kappa = o.r = o.g = o.b = o.hb = 0.0f;
    o.radius = o.x0 = o.y0 = o.x1 = o.y1 = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) o.J[k] = 0.0f;
    o.flags = 0;
    const float mx = in.mx, my = in.my, mz = in.mz;
    // camera space t = W mu + t
    float tx = fmul(c.R[0], mx); tx = ffma(c.R[1], my, tx); tx = ffma(c.R[2], mz, tx); tx = fadd(tx, c.t[0]);
    float ty = fmul(c.R[3], mx); ty = ffma(c.R[4], my, ty); ty = ffma(c.R[5], mz, ty); ty = fadd(ty, c.t[1]);
    float tz = fmul(c.R[6], mx); tz = ffma(c.R[7], my, tz); tz = ffma(c.R[8], mz, tz); tz = fadd(tz, c.t[2]);
    o.depth = tz;
    if (!(tz > c.near_z)) { o.status = GES_CULL_NEAR; return o; }

    // normalised quaternion -> rotation
    float qw = in.qw, qx = in.qx, qy = in.qy, qz = in.qz;
    float n2 = fmul(qw, qw); n2 = ffma(qx, qx, n2); n2 = ffma(qy, qy, n2); n2 = ffma(qz, qz, n2);
    if (!(n2 > 0.0f) || !isfinite(n2)) { o.status = GES_DEGENERATE; return o; }
    const float nq = fsqrt(n2);
    qw = fdiv(qw, nq); qx = fdiv(qx, nq); qy = fdiv(qy, nq); qz = fdiv(qz, nq);
    const float xx = fmul(qx, qx), yy = fmul(qy, qy), zz = fmul(qz, qz);
    const float xy = fmul(qx, qy), xz = fmul(qx, qz), yz = fmul(qy, qz);
    const float wx = fmul(qw, qx), wy = fmul(qw, qy), wz = fmul(qw, qz);
    float r[3][3];
    r[0][0] = fsub(1.0f, fmul(2.0f, fadd(yy, zz)));
    r[0][1] = fmul(2.0f, fsub(xy, wz));
    r[0][2] = fmul(2.0f, fadd(xz, wy));
    r[1][0] = fmul(2.0f, fadd(xy, wz));
    r[1][1] = fsub(1.0f, fmul(2.0f, fadd(xx, zz)));
    r[1][2] = fmul(2.0f, fsub(yz, wx));
    r[2][0] = fmul(2.0f, fsub(xz, wy));
    r[2][1] = fmul(2.0f, fadd(yz, wx));
    r[2][2] = fsub(1.0f, fmul(2.0f, fadd(xx, yy)));

    // exact GEF kernel (Eq. 2) needs beta > 0
    if (a.kernel == GES_KERNEL_EXACT_BETA && !(in.beta > 0.0f)) { o.status = GES_DEGENERATE; return o; }
    o.hb = fmul(0.5f, in.beta);
    // phi-bar (Eq. 6) -> effective scale (R1); none in the exact kernel
    float mfac = 1.0f;
    if (!a.gaussian_only && a.kernel == GES_KERNEL_PHI_GAUSS) {
        const float d = fsub(in.beta, 2.0f);
        const float ar = fmul(a.rho, d);
        const float e = exp_spec(-ar);
        const float phi = fdiv(2.0f, fadd(1.0f, e));
        mfac = (a.phi_mode == GES_PHI_VARIANCE) ? fsqrt(phi) : phi;
    }
    float se[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) se[k] = fmul(exp_spec(k == 0 ? in.ls0 : (k == 1 ? in.ls1 : in.ls2)), mfac);

    // Sigma = M M^T, M = R diag(se)
    float M[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k) M[j][k] = fmul(r[j][k], se[k]);
    float S[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int l = j; l < 3; ++l) {
            float p = fmul(M[j][0], M[l][0]); p = ffma(M[j][1], M[l][1], p); p = ffma(M[j][2], M[l][2], p);
            S[j][l] = p; S[l][j] = p;
        }

    // EWA Jacobian at the clamped mean; T = J W
    const float xn = fdiv(tx, tz), yn = fdiv(ty, tz);
    uint8_t fl = 0;
    const float xc = fminf(cd.limx, fmaxf(-cd.limx, xn));
    const float yc = fminf(cd.limy, fmaxf(-cd.limy, yn));
    if (xn > cd.limx || xn < -cd.limx) fl |= 8;
    if (yn > cd.limy || yn < -cd.limy) fl |= 16;
    const float txc = fmul(xc, tz), tyc = fmul(yc, tz);
    const float tz2 = fmul(tz, tz);
    const float j00 = fdiv(c.fx, tz), j02 = fdiv(-fmul(c.fx, txc), tz2);
    const float j11 = fdiv(c.fy, tz), j12 = fdiv(-fmul(c.fy, tyc), tz2);
    float T[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T[0][k] = ffma(j02, c.R[6 + k], fmul(j00, c.R[0 + k]));
        T[1][k] = ffma(j12, c.R[6 + k], fmul(j11, c.R[3 + k]));
    }
    float U[2][3];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float p = fmul(T[j][0], S[0][k]); p = ffma(T[j][1], S[1][k], p); p = ffma(T[j][2], S[2][k], p);
            U[j][k] = p;
        }
    float c00 = fmul(U[0][0], T[0][0]); c00 = ffma(U[0][1], T[0][1], c00); c00 = ffma(U[0][2], T[0][2], c00);
    float c01 = fmul(U[0][0], T[1][0]); c01 = ffma(U[0][1], T[1][1], c01); c01 = ffma(U[0][2], T[1][2], c01);
    float c11 = fmul(U[1][0], T[1][0]); c11 = ffma(U[1][1], T[1][1], c11); c11 = ffma(U[1][2], T[1][2], c11);
    const float A = fadd(c00, kDilation), B = c01, C = fadd(c11, kDilation);
    const float bb = fmul(B, B);
    const float det = ffma(A, C, -bb);
    o.flags = fl;
    if (!(det > 0.0f) || !isfinite(det)) { o.status = GES_DEGENERATE; return o; }
    const float ca = fdiv(C, det), cb = fdiv(-B, det), ccn = fdiv(A, det);
    const float mid = fmul(0.5f, fadd(A, C));
    float d2 = ffma(mid, mid, -det);
    d2 = fmaxf(0.1f, d2);
    const float lam = fadd(mid, fsqrt(d2));
    const float rad = ceilf(fmul(3.0f, fsqrt(lam)));
    const float u = ffma(c.fx, xn, c.cx), v = ffma(c.fy, yn, c.cy);
    if (!isfinite(u) || !isfinite(v) || !isfinite(rad)) { o.status = GES_DEGENERATE; return o; }
    // rect (R10): tiles whose pixel centres meet the bounding box of
    // the ellipse kappa exp(-Q/2) >= 0.98/255: half-extents sqrt(Q_thr A),
    // sqrt(Q_thr C) with Q_thr = 2 ln(255 kappa / 0.98).
    const float kap = fdiv(1.0f, fadd(1.0f, exp_spec(-in.logit)));
    const float kr = fdiv(fmul(kap, 255.0f), 0.98f);
    float qthr = 0.0f;
    if (kr > 1.0f) { qthr = log_spec(kr); qthr = fadd(qthr, qthr); }
    if (a.kernel == GES_KERNEL_EXACT_BETA && kr > 1.0f) {
        // exact GEF: kappa exp(-1/2 Q^(beta/2)) >= 0.98/255 <=> Q <= exp((2/beta) ln(2 ln(255 kappa/0.98)))
        const float hbi = fdiv(2.0f, in.beta);
        qthr = exp_spec(fmul(hbi, log_spec(qthr)));
    }
    const float ex = fsqrt(fmul(qthr, A)), ey = fsqrt(fmul(qthr, C));
    const float fx0 = ceilf(fmul(fsub(fsub(u, ex), 15.5f), 0.0625f));
    const float fx1 = fadd(floorf(fmul(fsub(fadd(u, ex), 0.5f), 0.0625f)), 1.0f);
    const float fy0 = ceilf(fmul(fsub(fsub(v, ey), 15.5f), 0.0625f));
    const float fy1 = fadd(floorf(fmul(fsub(fadd(v, ey), 0.5f), 0.0625f)), 1.0f);
    const float ftx = (float)c.tiles_x, fty = (float)c.tiles_y;
    o.x0 = (int)fminf(fmaxf(fx0, 0.0f), ftx);
    o.x1 = (int)fminf(fmaxf(fx1, 0.0f), ftx);
    o.y0 = (int)fminf(fmaxf(fy0, 0.0f), fty);
    o.y1 = (int)fminf(fmaxf(fy1, 0.0f), fty);
    if (o.x1 < o.x0) o.x1 = o.x0;
    if (o.y1 < o.y0) o.y1 = o.y0;
    if (!(kr > 1.0f)) o.x1 = o.x0;
    if (a.band_step > 1) {  // image tile rows -> band rows: row r = begin + k step <-> k
        const int b = a.band_begin, n = a.band_step;
        o.y0 = o.y0 > b ? (o.y0 - b + n - 1) / n : 0;
        o.y1 = o.y1 > b ? (o.y1 - b + n - 1) / n : 0;
    }
    o.u = u; o.v = v; o.ca = ca; o.cb = cb; o.cc = ccn;
    o.kappa = kap;
    o.radius = (int)rad;
    if ((o.x1 - o.x0) * (o.y1 - o.y0) == 0) { o.status = GES_OFFSCREEN; return o; }

    // view-dependent colour: rgb = sum_k Y_k(dir) sh_k + 0.5, >= 0
    const float dx = fsub(mx, cd.c0), dy = fsub(my, cd.c1), dz = fsub(mz, cd.c2);
    float dn2 = fmul(dx, dx); dn2 = ffma(dy, dy, dn2); dn2 = ffma(dz, dz, dn2);
    const float dn = fsqrt(dn2);
    const float ux = fdiv(dx, dn), uy = fdiv(dy, dn), uz = fdiv(dz, dn);
    float Y[16];
    sh_basis<K>(ux, uy, uz, Y);
    float rgb[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        float w[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = (k < K) ? sh[(size_t)(3 * k + ch) * sh_stride] : 0.0f;
        float acc = fmul(Y[0], w[0]);
#pragma unroll
        for (int k = 1; k < K; ++k) acc = ffma(Y[k], w[k], acc);
        acc = fadd(acc, 0.5f);
        const bool clamped = acc < 0.0f;
        if (clamped) { acc = 0.0f; fl |= (uint8_t)(1u << ch); }
        rgb[ch] = acc;
        // d rgb_ch / d u for S5b (so the backward need not re-read the SH planes)
        float gx, gy, gz;
        sh_basis_grad_dot<K>(ux, uy, uz, w, gx, gy, gz);
        o.J[3 * ch] = clamped ? 0.0f : gx;
        o.J[3 * ch + 1] = clamped ? 0.0f : gy;
        o.J[3 * ch + 2] = clamped ? 0.0f : gz;
    }
    o.r = rgb[0]; o.g = rgb[1]; o.b = rgb[2];
    o.flags = fl;
    o.status = GES_VISIBLE;
    return o;
}

constexpr int kPreThreads = 256;

// Per-thread counts of the non-visible statuses (ges_counts: culled_near, degenerate,
// offscreen), summed over the warp once at the end; status -1 = no particle.
struct StatusCounts {
    uint32_t near = 0, degen = 0, off = 0;
    __device__ __forceinline__ void add(int status) {
        near += status == GES_CULL_NEAR;
        degen += status == GES_DEGENERATE;
        off += status == GES_OFFSCREEN;
    }
    __device__ __forceinline__ void flush(unsigned long long* ctr) const {  // whole warp; lane 0 adds
        const uint32_t n = __reduce_add_sync(0xffffffffu, near), d = __reduce_add_sync(0xffffffffu, degen),
                       o = __reduce_add_sync(0xffffffffu, off);
        if ((threadIdx.x & 31) == 0) {
            if (n) atomicAdd(&ctr[GES_CTR_CULLED_NEAR], (unsigned long long)n);
            if (d) atomicAdd(&ctr[GES_CTR_DEGENERATE], (unsigned long long)d);
            if (o) atomicAdd(&ctr[GES_CTR_OFFSCREEN], (unsigned long long)o);
        }
    }
};

// Writes particle i's S1 state and its sort key (fp32 depth bits, or 0xffffffff
// when not visible -- dropped by depth pass 0, which thereby compacts the
// visible set).  Returns visibility.
#ifndef GES_PRE_L2_KEEP
#define GES_PRE_L2_KEEP 1
#endif
__device__ __forceinline__ bool store_out(const PreprocessArgs& a, int i, const PreOut& o) {
    a.depth[i] = o.depth;
    a.pay0[i] = make_float4(o.u, o.v, o.ca, o.cb);
    a.pay1[i] = make_float4(o.cc, o.kappa, o.r, o.g);
    a.pay2[i] = o.b;
    if (a.kernel == GES_KERNEL_EXACT_BETA) a.pay3[i] = o.hb;
    a.radius[i] = o.radius;
#if GES_PRE_L2_KEEP
    {   // the rects the depth sort's last pass gathers by particle: stored with an L2
        // evict_last policy (measured: S5b -3 us, the rest unchanged)
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        const uint64_t r = (uint64_t)(uint16_t)o.x0 | ((uint64_t)(uint16_t)o.y0 << 16) |
                           ((uint64_t)(uint16_t)o.x1 << 32) | ((uint64_t)(uint16_t)o.y1 << 48);
        asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(a.rect + i), "l"(r), "l"(pol) : "memory");
    }
#else
    a.rect[i] = make_ushort4((uint16_t)o.x0, (uint16_t)o.y0, (uint16_t)o.x1, (uint16_t)o.y1);
#endif
    a.status[i] = o.status;
    a.flags[i] = o.flags;
#pragma unroll
    for (int k = 0; k < 9; ++k) a.drgb_ddir[(size_t)k * a.P + i] = o.J[k];
    const bool vis = o.status == GES_VISIBLE;
    a.vis_key[i] = vis ? __float_as_uint(o.depth) : 0xffffffffu;
    return vis;
}

// Grid-stride over particles: no cross-CTA dependency.  Every particle writes
// its S1 state and its sort key (fp32 depth bits, or 0xffffffff when not
// visible -- dropped by depth pass 0, which thereby compacts the visible set).
template <int K>
#ifndef GES_PRE_MINB  // tuning knob: min resident CTAs per SM (register cap)
#define GES_PRE_MINB 3
#endif
__global__ void __launch_bounds__(kPreThreads, GES_PRE_MINB) preprocess_kernel(PreprocessArgs a) {
    const int tid = threadIdx.x, lane = tid & 31;
    const CamDerived cd = derive_camera(a.cam);
    uint32_t nvis = 0, kmax = 0;  // visible count, largest visible depth key (depth sort pass plan)
    StatusCounts sc;
    for (int base = blockIdx.x * kPreThreads; base < a.P; base += gridDim.x * kPreThreads) {
        const int i = base + tid;
        bool vis = false;
        int status = -1;
        if (i < a.P) {
            const ParamIn in = load_params(a, i);
            const PreOut o = preprocess_one<K>(a, cd, i, in, a.sh + i, a.P);
            vis = store_out(a, i, o);
            status = o.status;
        }
        nvis += __popc(__ballot_sync(0xffffffffu, vis));
        sc.add(status);
        if (vis) kmax = max(kmax, a.vis_key[i]);
    }
    if (lane == 0 && nvis) atomicAdd(&a.counters[GES_CTR_VISIBLE], (unsigned long long)nvis);
    sc.flush(a.counters);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0 && kmax) atomicMax(&a.counters[GES_CTR_KEYMAX], (unsigned long long)kmax);
}

// --- TMA-staged variant -------------------------------------------------------
// One producer warp streams every input plane of a 128-particle tile (12 + 3K
// planes x 512 B) into a 2-stage shared-memory ring with cp.async.bulk
// (mbarrier completion); four consumer warps run S1 on the staged tile, one
// particle per thread, and write the outputs directly.  The HBM reads of the
// next tile overlap this tile's arithmetic without any loads held in registers.
// Needs 16-B aligned planes (P % 4 == 0 and aligned base pointers); the last
// partial tile is processed from global memory.
#ifndef GES_PRE_TILE
#define GES_PRE_TILE 128
#endif
#ifndef GES_PRE_STAGES
#define GES_PRE_STAGES 2
#endif
// experiment knob GES_PRE_TMA_MINB: min blocks per SM (unset: no second launch-bounds
// argument -- spelling out 1 lets ptxas take 121 registers instead of 96)
#ifdef GES_PRE_TMA_MINB
#define GES_PRE_TMA_LB __launch_bounds__(kPreTmaThreads, GES_PRE_TMA_MINB)
#else
#define GES_PRE_TMA_LB __launch_bounds__(kPreTmaThreads)
#endif
constexpr int kPreTile = GES_PRE_TILE;
constexpr int kPreStages = GES_PRE_STAGES;
constexpr int kPreTmaThreads = kPreTile + 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int K>
__device__ __forceinline__ const float* pre_plane(const PreprocessArgs& a, int p) {
    if (p < 3) return a.mean + (size_t)p * a.P;
    if (p < 6) return a.log_scale + (size_t)(p - 3) * a.P;
    if (p < 10) return a.quat + (size_t)(p - 6) * a.P;
    if (p == 10) return a.opacity_logit;
    if (p == 11) return a.beta;
    return a.sh + (size_t)(p - 12) * a.P;
}

template <int K>
__global__ void GES_PRE_TMA_LB preprocess_tma_kernel(PreprocessArgs a) {
    constexpr int NPL = 12 + 3 * K;
    extern __shared__ __align__(128) float s_st[];  // [kPreStages][NPL][kPreTile]
    __shared__ __align__(8) uint64_t s_full[kPreStages], s_empty[kPreStages];
    __shared__ uint32_t s_nvis, s_kmax;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntiles = a.P / kPreTile;
    if (tid == 0) {
        for (int st = 0; st < kPreStages; ++st) {
            mbar_init(&s_full[st], 1);
            mbar_init(&s_empty[st], kPreTile / 32);
        }
        s_nvis = 0;
        s_kmax = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kPreTile / 32) {  // producer
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int st = it % kPreStages;
                if (it >= kPreStages) mbar_wait(&s_empty[st], ((it / kPreStages) - 1) & 1);
                mbar_expect_tx(&s_full[st], NPL * kPreTile * 4);
                float* dst = s_st + (size_t)st * NPL * kPreTile;
                for (int p = 0; p < NPL; ++p)
                    bulk_g2s(dst + p * kPreTile, pre_plane<K>(a, p) + (size_t)t * kPreTile, kPreTile * 4, &s_full[st]);
            }
        }
        return;
    }
    const CamDerived cd = derive_camera(a.cam);
    uint32_t nvis = 0, kmax = 0;  // visible count, largest visible depth key (depth sort pass plan)
    StatusCounts sc;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % kPreStages;
        mbar_wait(&s_full[st], (it / kPreStages) & 1);
        const float* sp = s_st + (size_t)st * NPL * kPreTile + tid;
        ParamIn in;
        in.mx = sp[0 * kPreTile]; in.my = sp[1 * kPreTile]; in.mz = sp[2 * kPreTile];
        in.ls0 = sp[3 * kPreTile]; in.ls1 = sp[4 * kPreTile]; in.ls2 = sp[5 * kPreTile];
        in.qw = sp[6 * kPreTile]; in.qx = sp[7 * kPreTile]; in.qy = sp[8 * kPreTile]; in.qz = sp[9 * kPreTile];
        in.logit = sp[10 * kPreTile];
        in.beta = sp[11 * kPreTile];
        const int i = t * kPreTile + tid;
        const PreOut o = preprocess_one<K>(a, cd, i, in, sp + 12 * kPreTile, kPreTile);
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[st]);  // the warp is done reading the stage
        const bool vis = store_out(a, i, o);
        nvis += __popc(__ballot_sync(0xffffffffu, vis));
        sc.add(o.status);
        if (vis) kmax = max(kmax, __float_as_uint(o.depth));
    }
    // the partial last tile, from global memory
    if (blockIdx.x == 0) {
        const int i = ntiles * kPreTile + tid;
        bool vis = false;
        int status = -1;
        if (i < a.P) {
            const ParamIn in = load_params(a, i);
            const PreOut o = preprocess_one<K>(a, cd, i, in, a.sh + i, a.P);
            vis = store_out(a, i, o);
            status = o.status;
            if (vis) kmax = max(kmax, __float_as_uint(o.depth));
        }
        nvis += __popc(__ballot_sync(0xffffffffu, vis));
        sc.add(status);
    }
    sc.flush(a.counters);
    if (lane == 0 && nvis) atomicAdd(&s_nvis, nvis);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0 && kmax) atomicMax(&s_kmax, kmax);
    asm volatile("bar.sync 1, %0;" ::"r"(kPreTile) : "memory");  // consumer warps only
    if (tid == 0 && s_nvis) atomicAdd(&a.counters[GES_CTR_VISIBLE], (unsigned long long)s_nvis);
    if (tid == 0 && s_kmax) atomicMax(&a.counters[GES_CTR_KEYMAX], (unsigned long long)s_kmax);
}

template <int K>
static cudaError_t launch_preprocess_tma(const PreprocessArgs& a, cudaStream_t stream) {
    constexpr int NPL = 12 + 3 * K;
    const int smem = kPreStages * NPL * kPreTile * 4;
    static int grids[kMaxDevices] = {0};
    int& grid = grids[current_device()];
    if (grid == 0) {
        cudaFuncSetAttribute(preprocess_tma_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, preprocess_tma_kernel<K>, kPreTmaThreads, smem);
        grid = std::max(1, per_sm) * num_sms();
    }
    const int ntiles = a.P / kPreTile;
    const int g = std::max(1, std::min(grid, ntiles));
    preprocess_tma_kernel<K><<<g, kPreTmaThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

static bool planes_aligned(const PreprocessArgs& a) {
    auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    return (a.P % 4) == 0 && a.P >= kPreTile && al(a.mean) && al(a.log_scale) && al(a.quat) &&
           al(a.opacity_logit) && al(a.beta) && al(a.sh);
}

cudaError_t launch_preprocess(const PreprocessArgs& a, cudaStream_t stream) {
#ifndef GES_PRE_NO_TMA
    if (planes_aligned(a)) {
        switch (a.sh_degree) {
            case 0: return launch_preprocess_tma<1>(a, stream);
            case 1: return launch_preprocess_tma<4>(a, stream);
            case 2: return launch_preprocess_tma<9>(a, stream);
            case 3: return launch_preprocess_tma<16>(a, stream);
            default: return cudaErrorInvalidValue;
        }
    }
#endif
    const int64_t need = (a.P + kPreThreads - 1) / kPreThreads;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)num_sms() * 6));
    dim3 g((unsigned)grid), block(kPreThreads);
    switch (a.sh_degree) {
        case 0: preprocess_kernel<1><<<g, block, 0, stream>>>(a); break;
        case 1: preprocess_kernel<4><<<g, block, 0, stream>>>(a); break;
        case 2: preprocess_kernel<9><<<g, block, 0, stream>>>(a); break;
        case 3: preprocess_kernel<16><<<g, block, 0, stream>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace ges
