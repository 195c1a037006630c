// loss.cu -- the image-loss front end: the
// frequency mask M_omega (Eq. 7), L1, SSIM and L_omega (Eq. 8) combined as
// Eq. 9 (PAPER.md:305-358; Appendix :1226, :1252-1263), forward value and
// dL/dimage -- the upstream gradient S5a consumes.  Readings R22-R28
// (DESIGN.md): luminance DoG on a 0.2 bilinear downsample, |DoG| min-max
// normalised, > 0.5, complement for omega <= 0.5, nearest upsample; SSIM with
// an 11 x 11 Gaussian window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, zero
// padding; every term a mean over pixels and channels.
//
// HBM/stencil-bound; no tensor cores.  Per call:
//   mask:  lum_down -> blur_h (both sigmas) -> blur_v + |DoG| + min/max ->
//          threshold (all on the ~HW/25 downsampled grid)
//   loss:  ssim_fwd (per 32 x 16 tile and channel: x, y with a 5-px halo in
//          shared memory, separable 11-tap blurs of x, y, x^2, y^2, xy, the
//          SSIM map and its three partials d_mu, d_E2, d_Exy, block sums of
//          SSIM, |I - I_gt| and |I - I_gt| M) -> ssim_bwd (the partials'
//          blurs = the window's adjoint, combined with the L1 and L_omega
//          subgradients into dL/dI) -> reduce (fixed order, fp64).
#include <algorithm>
#include <cmath>

#include "ges_internal.h"

namespace ges {

constexpr int kLTX = 32, kLTY = 16;             // loss tile
constexpr int kWin = 11, kWr = kWin / 2;        // SSIM window
constexpr int kLThreads = kLTX * kLTY;          // one pixel per thread
constexpr float kC1 = 0.0001f, kC2 = 0.0009f;   // (0.01)^2, (0.03)^2

__device__ __forceinline__ void ssim_taps(float* w) {
    if (threadIdx.x < kWin) {
        float s = 0.0f;
        for (int i = 0; i < kWin; ++i) {
            const float d = (float)(i - kWr);
            s += expf(-d * d / (2.0f * 1.5f * 1.5f));
        }
        const float d = (float)((int)threadIdx.x - kWr);  // signed: threadIdx.x is unsigned
        w[threadIdx.x] = expf(-d * d / (2.0f * 1.5f * 1.5f)) / s;
    }
}

__device__ __forceinline__ float block_sum(float v, float* s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    float t = 0.0f;
    if (threadIdx.x == 0)
        for (int w = 0; w < kLThreads / 32; ++w) t += s_red[w];
    return t;  // valid in thread 0
}

__device__ __forceinline__ uint8_t mask_at(const uint8_t* mask_lo, int Hd, int Wd, int H, int W, int y, int x) {
    const int iy = min((int)(((int64_t)y * Hd) / H), Hd - 1), ix = min((int)(((int64_t)x * Wd) / W), Wd - 1);
    return mask_lo[iy * Wd + ix];
}

// ---- SSIM forward: 5 blurred moments, the map and its partials ------------
__global__ void __launch_bounds__(kLThreads) ssim_fwd_kernel(LossArgs a) {
    __shared__ float s_w[kWin];
    __shared__ float s_x[kLTY + 2 * kWr][kLTX + 2 * kWr];
    __shared__ float s_y[kLTY + 2 * kWr][kLTX + 2 * kWr];
    __shared__ float s_h[5][kLTY + 2 * kWr][kLTX];
    __shared__ float s_red[kLThreads / 32];
    const int c = blockIdx.z, W = a.W, H = a.H;
    const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY;
    const float* X = a.image + (size_t)c * W * H;
    const float* Y = a.gt + (size_t)c * W * H;
    ssim_taps(s_w);
    for (int i = threadIdx.x; i < (kLTY + 2 * kWr) * (kLTX + 2 * kWr); i += kLThreads) {
        const int r = i / (kLTX + 2 * kWr), q = i - r * (kLTX + 2 * kWr);
        const int gy = y0 + r - kWr, gx = x0 + q - kWr;
        const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;  // zero padding
        s_x[r][q] = in ? __ldg(X + (size_t)gy * W + gx) : 0.0f;
        s_y[r][q] = in ? __ldg(Y + (size_t)gy * W + gx) : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (kLTY + 2 * kWr) * kLTX; i += kLThreads) {
        const int r = i / kLTX, q = i - r * kLTX;
        float m1 = 0.f, m2 = 0.f, e11 = 0.f, e22 = 0.f, e12 = 0.f;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const float w = s_w[k], xv = s_x[r][q + k], yv = s_y[r][q + k];
            m1 += w * xv; m2 += w * yv; e11 += w * xv * xv; e22 += w * yv * yv; e12 += w * xv * yv;
        }
        s_h[0][r][q] = m1; s_h[1][r][q] = m2; s_h[2][r][q] = e11; s_h[3][r][q] = e22; s_h[4][r][q] = e12;
    }
    __syncthreads();
    const int ty = threadIdx.x / kLTX, tx = threadIdx.x - ty * kLTX;
    const int gx = x0 + tx, gy = y0 + ty;
    float S = 0.0f, ad = 0.0f, adm = 0.0f;
    if (gx < W && gy < H) {
        float mx = 0.f, my = 0.f, exx = 0.f, eyy = 0.f, exy = 0.f;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const float w = s_w[k];
            mx += w * s_h[0][ty + k][tx]; my += w * s_h[1][ty + k][tx];
            exx += w * s_h[2][ty + k][tx]; eyy += w * s_h[3][ty + k][tx]; exy += w * s_h[4][ty + k][tx];
        }
        const float A1 = 2.f * mx * my + kC1, A2 = 2.f * (exy - mx * my) + kC2;
        const float B1 = mx * mx + my * my + kC1, B2 = (exx - mx * mx) + (eyy - my * my) + kC2;
        const float iB = 1.0f / (B1 * B2);
        S = A1 * A2 * iB;
        const size_t pix = (size_t)c * W * H + (size_t)gy * W + gx;
        a.d_mu[pix] = (2.f * my * A2 - 2.f * my * A1) * iB - S * (2.f * mx / B1 - 2.f * mx / B2);
        a.d_e2[pix] = -S / B2;
        a.d_exy[pix] = 2.f * A1 * iB;
#ifdef GES_LOSS_DEBUG
        if (c == 0) {
            const size_t q = (size_t)gy * W + gx, n = (size_t)W * H;
            a.d_mu[q] = mx; a.d_mu[n + q] = my; a.d_mu[2 * n + q] = exx; a.d_e2[q] = eyy; a.d_e2[n + q] = exy;
            a.d_e2[2 * n + q] = s_w[threadIdx.x % kWin];
        }
#endif
        const float d = s_x[ty + kWr][tx + kWr] - s_y[ty + kWr][tx + kWr];
        ad = fabsf(d);
        adm = a.mask_lo && mask_at(a.mask_lo, a.Hd, a.Wd, H, W, gy, gx) ? ad : 0.0f;
    }
    const int blk = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const float sS = block_sum(S, s_red);
    if (threadIdx.x == 0) a.partial[3 * blk] = sS;
    const float sA = block_sum(ad, s_red);
    if (threadIdx.x == 0) a.partial[3 * blk + 1] = sA;
    const float sM = block_sum(adm, s_red);
    if (threadIdx.x == 0) a.partial[3 * blk + 2] = sM;
}

// ---- backward: the window's adjoint on the partials + L1 / L_omega ---------
__global__ void __launch_bounds__(kLThreads) ssim_bwd_kernel(LossArgs a) {
    __shared__ float s_w[kWin];
    __shared__ float s_p[3][kLTY + 2 * kWr][kLTX + 2 * kWr];
    __shared__ float s_h[3][kLTY + 2 * kWr][kLTX];
    const int c = blockIdx.z, W = a.W, H = a.H;
    const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY;
    const size_t base = (size_t)c * W * H;
    ssim_taps(s_w);
    for (int i = threadIdx.x; i < (kLTY + 2 * kWr) * (kLTX + 2 * kWr); i += kLThreads) {
        const int r = i / (kLTX + 2 * kWr), q = i - r * (kLTX + 2 * kWr);
        const int gy = y0 + r - kWr, gx = x0 + q - kWr;
        const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;  // no window centred off the image
        const size_t p = base + (size_t)gy * W + gx;
        s_p[0][r][q] = in ? a.d_mu[p] : 0.0f;
        s_p[1][r][q] = in ? a.d_e2[p] : 0.0f;
        s_p[2][r][q] = in ? a.d_exy[p] : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (kLTY + 2 * kWr) * kLTX; i += kLThreads) {
        const int r = i / kLTX, q = i - r * kLTX;
        float b0 = 0.f, b1 = 0.f, b2 = 0.f;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const float w = s_w[k];
            b0 += w * s_p[0][r][q + k]; b1 += w * s_p[1][r][q + k]; b2 += w * s_p[2][r][q + k];
        }
        s_h[0][r][q] = b0; s_h[1][r][q] = b1; s_h[2][r][q] = b2;
    }
    __syncthreads();
    const int ty = threadIdx.x / kLTX, tx = threadIdx.x - ty * kLTX;
    const int gx = x0 + tx, gy = y0 + ty;
    if (gx >= W || gy >= H) return;
    float g0 = 0.f, g1 = 0.f, g2 = 0.f;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
        const float w = s_w[k];
        g0 += w * s_h[0][ty + k][tx]; g1 += w * s_h[1][ty + k][tx]; g2 += w * s_h[2][ty + k][tx];
    }
    const size_t p = base + (size_t)gy * W + gx;
    const float xv = __ldg(a.image + p), yv = __ldg(a.gt + p);
    const float dS = g0 + 2.f * xv * g1 + yv * g2;          // N d mean SSIM / dx
    const float d = xv - yv;
    const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    const float m = a.mask_lo && mask_at(a.mask_lo, a.Hd, a.Wd, H, W, gy, gx) ? 1.f : 0.f;
    const float lam_l1 = 1.0f - a.lambda_ssim - a.lambda_omega;
    a.dL_dimage[p] = (lam_l1 * sg - a.lambda_ssim * dS + a.lambda_omega * sg * m) * a.inv_n;
}

// one CTA: fixed-order fp64 sums of the block partials -> total, L1, SSIM, L_omega
__global__ void __launch_bounds__(256) loss_reduce_kernel(LossArgs a) {
    __shared__ double s[3][256];
    double t[3] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < a.nblocks; b += 256)
        for (int k = 0; k < 3; ++k) t[k] += (double)a.partial[3 * b + k];
    for (int k = 0; k < 3; ++k) s[k][threadIdx.x] = t[k];
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int k = 0; k < 3; ++k) s[k][threadIdx.x] += s[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double inv = (double)a.inv_n;
        const double ss = s[0][0] * inv, l1 = s[1][0] * inv, lw = s[2][0] * inv;
        const double lam_l1 = 1.0 - (double)a.lambda_ssim - (double)a.lambda_omega;
        a.loss_out[0] = (float)(lam_l1 * l1 + (double)a.lambda_ssim * (1.0 - ss) + (double)a.lambda_omega * lw);
        a.loss_out[1] = (float)l1;
        a.loss_out[2] = (float)ss;
        a.loss_out[3] = (float)lw;
    }
}

cudaError_t launch_loss(const LossArgs& a0, cudaStream_t stream) {
    LossArgs a = a0;
    const dim3 grid((a.W + kLTX - 1) / kLTX, (a.H + kLTY - 1) / kLTY, 3);
    a.nblocks = (int)(grid.x * grid.y * grid.z);
    cudaError_t e;
    ssim_fwd_kernel<<<grid, kLThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ssim_bwd_kernel<<<grid, kLThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    loss_reduce_kernel<<<1, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

int64_t loss_partials(int W, int H) {
    return (int64_t)((W + kLTX - 1) / kLTX) * ((H + kLTY - 1) / kLTY) * 3;
}

// ---- the frequency mask M_omega (Eq. 7) on the downsampled grid -------------
// Bilinear downsample of the luminance (output centre i samples
// (i + 0.5) H / Hd - 0.5, clamped), as the oracle.
__global__ void mask_lum_down_kernel(MaskArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.Hd * a.Wd) return;
    const int oy = i / a.Wd, ox = i - oy * a.Wd;
    auto coord = [](int o, int n_out, int n_in, int& i0, int& i1, float& f) {
        float cc = ((float)o + 0.5f) * ((float)n_in / (float)n_out) - 0.5f;
        cc = fminf(fmaxf(cc, 0.0f), (float)(n_in - 1));
        i0 = (int)floorf(cc);
        i1 = min(i0 + 1, n_in - 1);
        f = cc - (float)i0;
    };
    int y0, y1, x0, x1;
    float fy, fx;
    coord(oy, a.Hd, a.H, y0, y1, fy);
    coord(ox, a.Wd, a.W, x0, x1, fx);
    const size_t P = (size_t)a.W * a.H;
    auto lum = [&](int y, int x) {
        const size_t p = (size_t)y * a.W + x;
        return 0.299f * __ldg(a.gt + p) + 0.587f * __ldg(a.gt + P + p) + 0.114f * __ldg(a.gt + 2 * P + p);
    };
    const float top = lum(y0, x0) * (1.f - fx) + lum(y0, x1) * fx;
    const float bot = lum(y1, x0) * (1.f - fx) + lum(y1, x1) * fx;
    a.lo[i] = top * (1.f - fy) + bot * fy;
}

__device__ __forceinline__ int reflect_idx(int i, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    i %= period;
    if (i < 0) i += period;
    return i < n ? i : period - i;
}

// taps of both sigmas (normalised in fp32): w_s[k], k in [0, 2 r_s]
__device__ __forceinline__ void dog_taps(const MaskArgs& a, float* w1, float* w2) {
    for (int s = 0; s < 2; ++s) {
        const int r = s ? a.r2 : a.r1;
        const float ih = s ? a.ih2 : a.ih1;
        float* w = s ? w2 : w1;
        for (int k = threadIdx.x; k <= 2 * r; k += blockDim.x) w[k] = expf(-(float)((k - r) * (k - r)) * ih);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            const int r = s ? a.r2 : a.r1;
            float* w = s ? w2 : w1;
            float t = 0.f;
            for (int k = 0; k <= 2 * r; ++k) t += w[k];
            for (int k = 0; k <= 2 * r; ++k) w[k] /= t;
        }
    }
    __syncthreads();
}

// Each blur is evaluated as the value plus a small deviation, G*f = f + sum_k
// w_k (f[x+k] - f[x]) (the taps sum to 1), so that DoG -- a difference of two
// nearly equal blurs at small omega -- keeps its relative precision in fp32:
//   h pass:  dh_s(x) = sum_k w_k (lo[x+k] - lo[x])          (deviation of G_x * lo)
//   v pass:  G_y G_x lo - lo = dv_s(lo) + G_y * dh_s,  DoG = (G1 - lo) - (G2 - lo)
constexpr int kMaxTaps = 2 * 64 + 1;
__global__ void mask_blur_h_kernel(MaskArgs a) {
    __shared__ float w1[kMaxTaps], w2[kMaxTaps];
    dog_taps(a, w1, w2);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.Hd * a.Wd) return;
    const int y = i / a.Wd, x = i - y * a.Wd;
    const float* row = a.lo + (size_t)y * a.Wd;
    const float c = row[x];
    float s1 = 0.f, s2 = 0.f;
    for (int k = 0; k <= 2 * a.r1; ++k) s1 += w1[k] * (row[reflect_idx(x + k - a.r1, a.Wd)] - c);
    for (int k = 0; k <= 2 * a.r2; ++k) s2 += w2[k] * (row[reflect_idx(x + k - a.r2, a.Wd)] - c);
    a.h1[i] = s1;
    a.h2[i] = s2;
}

__global__ void mask_blur_v_kernel(MaskArgs a) {
    __shared__ float w1[kMaxTaps], w2[kMaxTaps];
    dog_taps(a, w1, w2);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = i < a.Hd * a.Wd;
    float d = 0.f;
    if (ok) {
        const int y = i / a.Wd, x = i - y * a.Wd;
        const float c = a.lo[i];
        float s1 = 0.f, s2 = 0.f;
        for (int k = 0; k <= 2 * a.r1; ++k) {
            const size_t q = (size_t)reflect_idx(y + k - a.r1, a.Hd) * a.Wd + x;
            s1 += w1[k] * ((a.lo[q] - c) + a.h1[q]);
        }
        for (int k = 0; k <= 2 * a.r2; ++k) {
            const size_t q = (size_t)reflect_idx(y + k - a.r2, a.Hd) * a.Wd + x;
            s2 += w2[k] * ((a.lo[q] - c) + a.h2[q]);
        }
        d = fabsf(s1 - s2);
        a.dog[i] = d;
    }
    // min / max of |DoG| >= 0: float bits are monotone
    unsigned mn = ok ? __float_as_uint(d) : 0xffffffffu, mx = ok ? __float_as_uint(d) : 0u;
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(a.minmax, mn);
        atomicMax(a.minmax + 1, mx);
    }
}

__global__ void mask_threshold_kernel(MaskArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.Hd * a.Wd) return;
    const float mn = __uint_as_float(a.minmax[0]), mx = __uint_as_float(a.minmax[1]);
    const float nrm = mx > mn ? (a.dog[i] - mn) / (mx - mn) : 0.0f;
    bool m = nrm > a.eps;
    if (a.complement) m = !m;
    a.mask_lo[i] = m ? 1 : 0;
}

cudaError_t launch_mask(const MaskArgs& a, cudaStream_t stream) {
    const int n = a.Hd * a.Wd, blocks = (n + 255) / 256;
    cudaError_t e;
    if ((e = cudaMemsetAsync(a.minmax, 0xff, sizeof(unsigned), stream)) != cudaSuccess) return e;   // min
    if ((e = cudaMemsetAsync(a.minmax + 1, 0, sizeof(unsigned), stream)) != cudaSuccess) return e;  // max
    mask_lum_down_kernel<<<blocks, 256, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    mask_blur_h_kernel<<<blocks, 256, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    mask_blur_v_kernel<<<blocks, 256, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    mask_threshold_kernel<<<blocks, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
