// particle_bwd.cu -- S5b: per-particle chain rule from the
// 2-D gradients (u, v, conic, kappa, rgb) to the raw parameters: mean,
// log-scale, quaternion, opacity logit, SH coefficients and the shape beta
// ("This optimization strategy encompasses the beta parameter as
// well as the splat's position x, opacity kappa, covariance matrix Sigma, and
// color representation through spherical harmonics coefficients").
//
//   conic (a,b,c) = (C, -B, A)/det of the dilated Sigma2D (A, B, C)
//   Sigma2D = T Sigma T^T (entries 00, 01, 11), T = J W
//   Sigma = M M^T, M = R(q/|q|) diag(s_eff), s_eff = exp(log s) m(beta)
//   m = phi-bar (SCALE) or sqrt(phi-bar) (VARIANCE), phi-bar of Eq. 6:
//     d phi-bar / d beta = rho phi-bar (1 - phi-bar / 2)
//   J: exact piecewise derivative (zero through the clamped components, R13)
//   u = fx x/z + cx, v = fy y/z + cy;  rgb = sum_k Y_k(dir) sh_k + 0.5 (>= 0)
// HBM-bound: reads the parameters and 36 B of 2-D gradients, writes
// (14 + 3K) * 4 B per visible particle.
#include <algorithm>

#include "ges_internal.h"

namespace ges {

#ifndef GES_PBWD_MINB  // tuning knob: min resident CTAs per SM (register cap)
#define GES_PBWD_MINB 4
#endif

// The inputs S5b reads for one particle (from global memory or a staged tile).
struct PbIn {
    float m0, m1, m2, q0, q1, q2, q3, ls0, ls1, ls2, beta, logit;
    float4 r0, r1, r2;  // the 12-float 2-D gradient record
    float J[9];         // d rgb / d unit direction (S1)
    int status, flags;
};

__device__ __forceinline__ PbIn pb_load_global(const ParticleBwdArgs& a, int i) {
    const int P = a.P;
    PbIn in;
    in.status = a.status[i];
    in.flags = a.flags[i];
    in.m0 = __ldg(a.mean + i); in.m1 = __ldg(a.mean + P + i); in.m2 = __ldg(a.mean + 2 * P + i);
    in.q0 = __ldg(a.quat + i); in.q1 = __ldg(a.quat + P + i); in.q2 = __ldg(a.quat + 2 * P + i);
    in.q3 = __ldg(a.quat + 3 * P + i);
    in.ls0 = __ldg(a.log_scale + i); in.ls1 = __ldg(a.log_scale + P + i); in.ls2 = __ldg(a.log_scale + 2 * P + i);
    in.beta = __ldg(a.beta + i);
    in.logit = __ldg(a.opacity_logit + i);
    const float4* rrec = reinterpret_cast<const float4*>(a.grad2d) + (size_t)i * (kGrad2dStride / 4);
    in.r0 = rrec[0]; in.r1 = rrec[1]; in.r2 = rrec[2];
#pragma unroll
    for (int k = 0; k < 9; ++k) in.J[k] = __ldg(a.drgb_ddir + (size_t)k * P + i);
    return in;
}

template <int K>
__device__ __forceinline__ void particle_bwd_one(const ParticleBwdArgs& a, int i, const PbIn& in) {
    const int P = a.P;
    const bool acc = a.accumulate != 0;
    auto put = [&](float* base, int plane, float val) {
        float* p = base + (size_t)plane * P + i;
        *p = acc ? (*p + val) : val;
    };
    // Every thread of a warp stores every plane in the same instruction (zeros
    // for particles that are not visible): full 32-B sectors, no partial-sector
    // read-modify-write in DRAM.
    const bool vis = in.status == GES_VISIBLE;
    float o_mean[3] = {0.f, 0.f, 0.f}, o_ls[3] = {0.f, 0.f, 0.f}, o_q[4] = {0.f, 0.f, 0.f, 0.f};
    float o_op = 0.f, o_beta = 0.f, o_m2d[2] = {0.f, 0.f};
    float Y[16], drgb[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 16; ++k) Y[k] = 0.f;
    if (vis) {
        const CamParams& cam = a.cam;
        const CamDerived cd = derive_camera(cam);
        const float W[9] = {cam.R[0], cam.R[1], cam.R[2], cam.R[3], cam.R[4], cam.R[5], cam.R[6], cam.R[7], cam.R[8]};
        const int fl = in.flags;
        // ---- forward recompute ----
        const float m0 = in.m0, m1 = in.m1, m2 = in.m2;
        const float tx = W[0] * m0 + W[1] * m1 + W[2] * m2 + cam.t[0];
        const float ty = W[3] * m0 + W[4] * m1 + W[5] * m2 + cam.t[1];
        const float tz = W[6] * m0 + W[7] * m1 + W[8] * m2 + cam.t[2];
        const float q0 = in.q0, q1 = in.q1, q2 = in.q2, q3 = in.q3;
        const float nq = sqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
        const float inq = 1.0f / nq;
        const float w = q0 * inq, x = q1 * inq, y = q2 * inq, z = q3 * inq;
        const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                            2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                            2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
        float phi = 1.f, mfac = 1.f, dm_dbeta = 0.f;
        if (!a.gaussian_only && a.kernel == GES_KERNEL_PHI_GAUSS) {
            phi = 2.f / (1.f + expf(-(a.rho * (in.beta - 2.f))));
            const float dphi = a.rho * phi * (1.f - 0.5f * phi);
            if (a.phi_mode == GES_PHI_VARIANCE) { mfac = sqrtf(phi); dm_dbeta = 0.5f * dphi / mfac; }
            else { mfac = phi; dm_dbeta = dphi; }
        }
        float s[3], se[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) { s[k] = expf(k == 0 ? in.ls0 : (k == 1 ? in.ls1 : in.ls2)); se[k] = s[k] * mfac; }
        float M[9];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) M[j * 3 + k] = R[j * 3 + k] * se[k];
        float Sig[9];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int l = 0; l < 3; ++l) Sig[j * 3 + l] = M[j * 3] * M[l * 3] + M[j * 3 + 1] * M[l * 3 + 1] + M[j * 3 + 2] * M[l * 3 + 2];
        const bool clx = (fl >> 3) & 1, cly = (fl >> 4) & 1;
        const float Lx = (tx / tz > 0.f) ? cd.limx : -cd.limx, Ly = (ty / tz > 0.f) ? cd.limy : -cd.limy;
        const float txc = clx ? Lx * tz : tx, tyc = cly ? Ly * tz : ty;
        const float itz = 1.f / tz, itz2 = itz * itz;
        const float j00 = cam.fx * itz, j02 = -cam.fx * txc * itz2, j11 = cam.fy * itz, j12 = -cam.fy * tyc * itz2;
        float Tm[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            Tm[k] = j00 * W[k] + j02 * W[6 + k];
            Tm[3 + k] = j11 * W[3 + k] + j12 * W[6 + k];
        }
        float TS[6];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                TS[j * 3 + k] = Tm[j * 3] * Sig[k] + Tm[j * 3 + 1] * Sig[3 + k] + Tm[j * 3 + 2] * Sig[6 + k];
        const float A = TS[0] * Tm[0] + TS[1] * Tm[1] + TS[2] * Tm[2] + kDilation;
        const float B = TS[0] * Tm[3] + TS[1] * Tm[4] + TS[2] * Tm[5];
        const float C = TS[3] * Tm[3] + TS[4] * Tm[4] + TS[5] * Tm[5] + kDilation;
        const float det = A * C - B * B;
        const float idet = 1.f / det, idet2 = idet * idet;

        // ---- incoming 2-D gradients ----
        // 12-float record of S5a's raw moments over the particle's composited pixels,
        // (sum m dx, sum m dy, sum m dx^2, sum m dx dy | sum m dy^2, K, dr, dg | db, Sb, -, -),
        // zeroed after reading so the buffer is clean for the next frame's backward.
        // Gaussian kernel: m = kappa G dL/dalpha, dL/dp2 = ln2 m, K = kappa dL/dkappa;
        // exact kernel: m = G dL/dalpha Q^hb / qp, dL/dp2 = kappa beta / 4 m, K = dL/dkappa.
        // With p2 = A' dx^2 + B' dx dy + C' dy^2 (the log2-scaled conic A' = -1/2 log2e a,
        // B' = -log2e b, C' = -1/2 log2e c) and dL/dp2 = kl m:
        // dL/du = kl (2 A' sum m dx + B' sum m dy), dL/dv = kl (B' sum m dx + 2 C' sum m dy),
        // dL/dA' = kl sum m dx^2, dL/dB' = kl sum m dx dy, dL/dC' = kl sum m dy^2.
        const float4 r0 = in.r0, r1 = in.r1, r2 = in.r2;
        const float kap = 1.f / (1.f + expf(-in.logit));
        const bool exact = a.kernel == GES_KERNEL_EXACT_BETA;
        const float kl = exact ? kap * (0.25f * in.beta) : 0.69314718055994531f;
        const float cA = (C * idet) * (-0.5f * kLog2e), cB = (-B * idet) * (-kLog2e), cC = (A * idet) * (-0.5f * kLog2e);
        const float E = kl * r0.x, F = kl * r0.y;
        const float du = 2.f * cA * E + cB * F, dv = cB * E + 2.f * cC * F;
        o_m2d[0] = du;
        o_m2d[1] = dv;
        const float da = (kl * r0.z) * (-0.5f * kLog2e);
        const float db = (kl * r0.w) * (-kLog2e);
        const float dc = (kl * r1.x) * (-0.5f * kLog2e);
        const float dk = exact ? r1.y : r1.y / kap;
        drgb[0] = r1.z; drgb[1] = r1.w; drgb[2] = r2.x;

        // conic -> (A, B, C)
        const float gA = da * (-C * C * idet2) + db * (B * C * idet2) + dc * (idet - A * C * idet2);
        const float gB = da * (2.f * B * C * idet2) + db * (-idet - 2.f * B * B * idet2) + dc * (2.f * A * B * idet2);
        const float gC = da * (idet - A * C * idet2) + db * (A * B * idet2) + dc * (-A * A * idet2);
        // dSig = T^T Gc T with Gc = [[gA, gB], [0, gC]]
        float dSig[9];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int l = 0; l < 3; ++l)
                dSig[k * 3 + l] = Tm[k] * (gA * Tm[l] + gB * Tm[3 + l]) + Tm[3 + k] * (gC * Tm[3 + l]);
        // dT = (Gc + Gc^T) T Sig
        float dT[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            dT[k] = 2.f * gA * TS[k] + gB * TS[3 + k];
            dT[3 + k] = gB * TS[k] + 2.f * gC * TS[3 + k];
        }
        // Sig = M M^T -> dM = (dSig + dSig^T) M
        float dM[9];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                float acc2 = 0.f;
#pragma unroll
                for (int l = 0; l < 3; ++l) acc2 += (dSig[j * 3 + l] + dSig[l * 3 + j]) * M[l * 3 + k];
                dM[j * 3 + k] = acc2;
            }
        float dR[9], dse[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) { dR[j * 3 + k] = dM[j * 3 + k] * se[k]; dse[k] += dM[j * 3 + k] * R[j * 3 + k]; }
        float dbeta = 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            o_ls[k] = dse[k] * se[k];
            dbeta += dse[k] * s[k] * dm_dbeta;
        }
        // exact GEF kernel: beta enters through Eq. 2's exponent only,
        // dL/dbeta = -1/4 kappa ln2 Sb (record[9])
        o_beta = exact ? (-0.25f * 0.69314718055994531f) * kap * r2.y : dbeta;
        float dq[4];
        dq[0] = dR[1] * (-2.f * z) + dR[2] * (2.f * y) + dR[3] * (2.f * z) + dR[5] * (-2.f * x) + dR[6] * (-2.f * y) + dR[7] * (2.f * x);
        dq[1] = dR[1] * (2.f * y) + dR[2] * (2.f * z) + dR[3] * (2.f * y) + dR[4] * (-4.f * x) + dR[5] * (-2.f * w) +
                dR[6] * (2.f * z) + dR[7] * (2.f * w) + dR[8] * (-4.f * x);
        dq[2] = dR[0] * (-4.f * y) + dR[1] * (2.f * x) + dR[2] * (2.f * w) + dR[3] * (2.f * x) + dR[5] * (2.f * z) +
                dR[6] * (-2.f * w) + dR[7] * (2.f * z) + dR[8] * (-4.f * y);
        dq[3] = dR[0] * (-4.f * z) + dR[1] * (-2.f * w) + dR[2] * (2.f * x) + dR[3] * (2.f * w) + dR[4] * (-4.f * z) +
                dR[5] * (2.f * y) + dR[6] * (2.f * x) + dR[7] * (2.f * y);
        const float qh[4] = {w, x, y, z};
        const float dotq = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
#pragma unroll
        for (int k = 0; k < 4; ++k) o_q[k] = (dq[k] - qh[k] * dotq) * inq;
        // T = J W -> dJ = dT W^T (entries 00, 02, 11, 12)
        const float dj00 = dT[0] * W[0] + dT[1] * W[1] + dT[2] * W[2];
        const float dj02 = dT[0] * W[6] + dT[1] * W[7] + dT[2] * W[8];
        const float dj11 = dT[3] * W[3] + dT[4] * W[4] + dT[5] * W[5];
        const float dj12 = dT[3] * W[6] + dT[4] * W[7] + dT[5] * W[8];
        float dtx = 0.f, dty = 0.f, dtz = 0.f;
        dtz += dj00 * (-cam.fx * itz2) + dj11 * (-cam.fy * itz2);
        if (!clx) { dtx += dj02 * (-cam.fx * itz2); dtz += dj02 * (2.f * cam.fx * tx * itz2 * itz); }
        else { dtz += dj02 * (cam.fx * Lx * itz2); }
        if (!cly) { dty += dj12 * (-cam.fy * itz2); dtz += dj12 * (2.f * cam.fy * ty * itz2 * itz); }
        else { dtz += dj12 * (cam.fy * Ly * itz2); }
        dtx += du * cam.fx * itz; dtz += du * (-cam.fx * tx * itz2);
        dty += dv * cam.fy * itz; dtz += dv * (-cam.fy * ty * itz2);
        float dmean[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) dmean[k] = W[k] * dtx + W[3 + k] * dty + W[6 + k] * dtz;
        // colour
        const float d0 = m0 - cd.c0, d1 = m1 - cd.c1, d2 = m2 - cd.c2;
        const float dn = sqrtf(d0 * d0 + d1 * d1 + d2 * d2), idn = 1.f / dn;
        const float ux = d0 * idn, uy = d1 * idn, uz = d2 * idn;
        sh_basis<K>(ux, uy, uz, Y);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            if ((fl >> ch) & 1) drgb[ch] = 0.f;
        // d L / d u = sum_ch dL/drgb_ch * d rgb_ch / d u (S1 stored the Jacobian, zero rows
        // where the channel was clamped)
        float gx = 0.f, gy = 0.f, gz = 0.f;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            gx += drgb[ch] * in.J[3 * ch];
            gy += drgb[ch] * in.J[3 * ch + 1];
            gz += drgb[ch] * in.J[3 * ch + 2];
        }
        const float dotd = ux * gx + uy * gy + uz * gz;
        dmean[0] += (gx - ux * dotd) * idn;
        dmean[1] += (gy - uy * dotd) * idn;
        dmean[2] += (gz - uz * dotd) * idn;
#pragma unroll
        for (int k = 0; k < 3; ++k) o_mean[k] = dmean[k];
        o_op = dk * kap * (1.f - kap);
    }  // vis
#pragma unroll
    for (int k = 0; k < 3; ++k) put(a.g_mean, k, o_mean[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) put(a.g_log_scale, k, o_ls[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) put(a.g_quat, k, o_q[k]);
    put(a.g_opacity_logit, 0, o_op);
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) put(a.g_sh, 3 * k + ch, Y[k] * drgb[ch]);
    put(a.g_beta, 0, o_beta);
    if (a.g_mean2d) {
        put(a.g_mean2d, 0, o_m2d[0]);
        put(a.g_mean2d, 1, o_m2d[1]);
    }
    if (a.g_drgb) {  // the per-view colour gradient the SH gradient factors through
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) put(a.g_drgb, ch, drgb[ch]);
    }
    // leave the 2-D record zeroed for the next backward (ges.h); every particle's
    // record is written so the 48-B records cover whole sectors
    float4* rec = reinterpret_cast<float4*>(a.grad2d) + (size_t)i * (kGrad2dStride / 4);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    rec[0] = z4; rec[1] = z4; rec[2] = z4;
}

template <int K>
__global__ void __launch_bounds__(256, GES_PBWD_MINB) particle_bwd_kernel(ParticleBwdArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.P) return;
    particle_bwd_one<K>(a, i, pb_load_global(a, i));
}

// --- TMA-staged variant (as S1's): a producer warp streams each 128-particle
// tile's inputs -- 12 parameter planes, the 48-B 2-D gradient records, the 9
// d rgb / d dir planes, status and flags (~17 KB) -- into a 2-stage ring
// (cp.async.bulk, mbarriers); four consumer warps run the chain rule and store
// the gradients.  Needs P % 4 == 0 and 16-B aligned planes; the partial last
// tile goes through global loads.
#ifndef GES_PB_TILE
#define GES_PB_TILE 128
#endif
#ifndef GES_PB_STAGES
#define GES_PB_STAGES 2
#endif
constexpr int kPbTile = GES_PB_TILE;
constexpr int kPbStages = GES_PB_STAGES;
constexpr int kPbThreads = kPbTile + 32;
constexpr int kPbPlanes = 12 + 9;
struct PbStage {
    float plane[kPbPlanes][kPbTile];       // mean 0-2, quat 3-6, log-scale 7-9, beta 10, logit 11, J 12-20
    float4 rec[kPbTile * 3];               // grad2d records
    uint8_t status[kPbTile], flags[kPbTile];
};

__device__ __forceinline__ uint32_t pb_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void pb_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(pb_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void pb_mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(pb_smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void pb_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(pb_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void pb_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pb_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void pb_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            pb_smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(pb_smem_u32(bar))
        : "memory");
}

template <int K>
// experiment knob GES_PB_TMA_MINB: min resident CTAs per SM (register cap); unset = none
#ifdef GES_PB_TMA_MINB
#define GES_PB_TMA_LB __launch_bounds__(kPbThreads, GES_PB_TMA_MINB)
#else
#define GES_PB_TMA_LB __launch_bounds__(kPbThreads)
#endif
__global__ void GES_PB_TMA_LB particle_bwd_tma_kernel(ParticleBwdArgs a) {
    extern __shared__ __align__(128) unsigned char s_raw[];
    PbStage* stg = reinterpret_cast<PbStage*>(s_raw);
    __shared__ __align__(8) uint64_t s_full[kPbStages], s_empty[kPbStages];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = a.P, ntiles = P / kPbTile;
    if (tid == 0) {
        for (int st = 0; st < kPbStages; ++st) {
            pb_mbar_init(&s_full[st], 1);
            pb_mbar_init(&s_empty[st], kPbTile / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kPbTile / 32) {  // producer
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int st = it % kPbStages;
                if (it >= kPbStages) pb_mbar_wait(&s_empty[st], ((it / kPbStages) - 1) & 1);
                constexpr uint32_t kBytes = kPbPlanes * kPbTile * 4 + kPbTile * 48 + 2 * kPbTile;
                pb_mbar_expect_tx(&s_full[st], kBytes);
                PbStage& S = stg[st];
                const size_t i0 = (size_t)t * kPbTile;
                const float* src[12] = {a.mean, a.mean + P, a.mean + 2 * (size_t)P, a.quat, a.quat + P,
                                        a.quat + 2 * (size_t)P, a.quat + 3 * (size_t)P, a.log_scale,
                                        a.log_scale + P, a.log_scale + 2 * (size_t)P, a.beta, a.opacity_logit};
#pragma unroll
                for (int p = 0; p < 12; ++p) pb_bulk(S.plane[p], src[p] + i0, kPbTile * 4, &s_full[st]);
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    pb_bulk(S.plane[12 + k], a.drgb_ddir + (size_t)k * P + i0, kPbTile * 4, &s_full[st]);
                pb_bulk(S.rec, a.grad2d + i0 * kGrad2dStride, kPbTile * 48, &s_full[st]);
                pb_bulk(S.status, a.status + i0, kPbTile, &s_full[st]);
                pb_bulk(S.flags, a.flags + i0, kPbTile, &s_full[st]);
            }
        }
        return;
    }
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % kPbStages;
        pb_mbar_wait(&s_full[st], (it / kPbStages) & 1);
        const PbStage& S = stg[st];
        PbIn in;
        in.m0 = S.plane[0][tid]; in.m1 = S.plane[1][tid]; in.m2 = S.plane[2][tid];
        in.q0 = S.plane[3][tid]; in.q1 = S.plane[4][tid]; in.q2 = S.plane[5][tid]; in.q3 = S.plane[6][tid];
        in.ls0 = S.plane[7][tid]; in.ls1 = S.plane[8][tid]; in.ls2 = S.plane[9][tid];
        in.beta = S.plane[10][tid]; in.logit = S.plane[11][tid];
#pragma unroll
        for (int k = 0; k < 9; ++k) in.J[k] = S.plane[12 + k][tid];
        in.r0 = S.rec[3 * tid]; in.r1 = S.rec[3 * tid + 1]; in.r2 = S.rec[3 * tid + 2];
        in.status = S.status[tid]; in.flags = S.flags[tid];
        __syncwarp();
        if (lane == 0) pb_mbar_arrive(&s_empty[st]);  // the warp has its inputs in registers
        particle_bwd_one<K>(a, t * kPbTile + tid, in);
    }
    if (blockIdx.x == 0) {  // the partial last tile
        const int i = ntiles * kPbTile + tid;
        if (i < P) particle_bwd_one<K>(a, i, pb_load_global(a, i));
    }
}

template <int K>
static cudaError_t launch_particle_bwd_tma(const ParticleBwdArgs& a, cudaStream_t stream) {
    const int smem = kPbStages * (int)sizeof(PbStage);
    static int grids[kMaxDevices] = {0};
    int& grid = grids[current_device()];
    if (grid == 0) {
        cudaFuncSetAttribute(particle_bwd_tma_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, particle_bwd_tma_kernel<K>, kPbThreads, smem);
        grid = std::max(1, per_sm) * num_sms();
    }
    const int g = std::max(1, std::min(grid, a.P / kPbTile));
    particle_bwd_tma_kernel<K><<<g, kPbThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

static bool pb_aligned(const ParticleBwdArgs& a) {
    auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    return (a.P % 4) == 0 && a.P >= kPbTile && al(a.mean) && al(a.log_scale) && al(a.quat) &&
           al(a.opacity_logit) && al(a.beta) && al(a.drgb_ddir) && al(a.grad2d) && al(a.status) && al(a.flags);
}

// SH gradient from per-view colour gradients (view DP): S5b's SH term is
// dL/dsh[3k + ch] = Y_k(u_v) dL/drgb_v[ch] per view v (u_v the unit direction from
// view v's camera centre to the mean), so the SH gradient of any set of views follows
// from their 3-float dL/drgb and their cameras -- the same expressions S5b evaluates.
struct ShFromColourArgs {
    const float* mean;       // [3][P]
    int P;
    const float* cams;       // [n][12]: R (9, world -> camera, row-major), t (3)
    int n_views;
    const float* drgb;       // [n][3][P]
    float* g_sh;             // [3K][P]
    int accumulate;
};

template <int K>
__global__ void __launch_bounds__(128) sh_from_colour_kernel(ShFromColourArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.P) return;
    const int P = a.P;
    const float m0 = __ldg(a.mean + i), m1 = __ldg(a.mean + P + i), m2 = __ldg(a.mean + 2 * P + i);
    float acc[3 * K];
#pragma unroll
    for (int q = 0; q < 3 * K; ++q) acc[q] = 0.f;
    for (int v = 0; v < a.n_views; ++v) {
        const float* dv = a.drgb + (size_t)v * 3 * P + i;
        const float r[3] = {__ldg(dv), __ldg(dv + P), __ldg(dv + 2 * P)};
        if (r[0] == 0.f && r[1] == 0.f && r[2] == 0.f) continue;  // not visible in view v
        CamParams cam;
        for (int k = 0; k < 9; ++k) cam.R[k] = __ldg(a.cams + 12 * v + k);
        for (int k = 0; k < 3; ++k) cam.t[k] = __ldg(a.cams + 12 * v + 9 + k);
        cam.W = cam.H = 1; cam.fx = cam.fy = 1.f;
        const CamDerived cd = derive_camera(cam);
        const float d0 = m0 - cd.c0, d1 = m1 - cd.c1, d2 = m2 - cd.c2;
        const float dn = sqrtf(d0 * d0 + d1 * d1 + d2 * d2), idn = 1.f / dn;
        float Y[16];
        sh_basis<K>(d0 * idn, d1 * idn, d2 * idn, Y);
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) acc[3 * k + ch] += Y[k] * r[ch];
    }
#pragma unroll
    for (int q = 0; q < 3 * K; ++q) {
        float* o = a.g_sh + (size_t)q * P + i;
        *o = a.accumulate ? *o + acc[q] : acc[q];
    }
}

cudaError_t launch_sh_from_colour(const float* mean, int64_t P, int sh_degree, const float* cams, int n_views,
                                  const float* drgb, float* g_sh, int accumulate, cudaStream_t stream) {
    ShFromColourArgs a{mean, (int)P, cams, n_views, drgb, g_sh, accumulate};
    const unsigned grid = (unsigned)((P + 127) / 128);
    switch (sh_degree) {
        case 0: sh_from_colour_kernel<1><<<grid, 128, 0, stream>>>(a); break;
        case 1: sh_from_colour_kernel<4><<<grid, 128, 0, stream>>>(a); break;
        case 2: sh_from_colour_kernel<9><<<grid, 128, 0, stream>>>(a); break;
        case 3: sh_from_colour_kernel<16><<<grid, 128, 0, stream>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_particle_bwd(const ParticleBwdArgs& a, cudaStream_t stream) {
#ifndef GES_PBWD_NO_TMA
    if (pb_aligned(a)) {
        switch (a.sh_degree) {
            case 0: return launch_particle_bwd_tma<1>(a, stream);
            case 1: return launch_particle_bwd_tma<4>(a, stream);
            case 2: return launch_particle_bwd_tma<9>(a, stream);
            case 3: return launch_particle_bwd_tma<16>(a, stream);
            default: return cudaErrorInvalidValue;
        }
    }
#endif
    const int grid = (a.P + 255) / 256;
    switch (a.sh_degree) {
        case 0: particle_bwd_kernel<1><<<grid, 256, 0, stream>>>(a); break;
        case 1: particle_bwd_kernel<4><<<grid, 256, 0, stream>>>(a); break;
        case 2: particle_bwd_kernel<9><<<grid, 256, 0, stream>>>(a); break;
        case 3: particle_bwd_kernel<16><<<grid, 256, 0, stream>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace ges
