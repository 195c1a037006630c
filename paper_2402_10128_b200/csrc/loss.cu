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
//   loss:  ssim_fwd (per 32 x 32 tile and channel: x, y with a 5-px halo in
//          shared memory, separable 11-tap blurs of x, y, x^2, y^2, xy -- each
//          thread two vertically adjacent pixels sharing 10 window rows --, the
//          SSIM map and its three partials d_mu, d_E2, d_Exy, block sums of
//          SSIM, |I - I_gt| and |I - I_gt| M) -> ssim_bwd (the partials'
//          blurs = the window's adjoint, combined with the L1 and L_omega
//          subgradients into dL/dI) -> reduce (fixed order, fp64).
#include <algorithm>
#include <cmath>

#include "ges_internal.h"

namespace ges {

constexpr int kLTX = 32, kLTY = 32;             // loss tile
constexpr int kWin = 11, kWr = kWin / 2;        // SSIM window
constexpr int kLThreads = 512;                  // 2 pixels per thread
constexpr int kHX = kLTX + 2 * kWr, kHY = kLTY + 2 * kWr;
constexpr float kC1 = 0.0001f, kC2 = 0.0009f;   // (0.01)^2, (0.03)^2
// exp(-(k - 5)^2 / (2 1.5^2)) / sum, k = 0..10 (the SSIM window of R27), fp32
__constant__ float kSsimW[kWin] = {0.00102838008f, 0.00759875814f, 0.0360007721f, 0.10936069f, 0.213005538f,
                                   0.266011725f,   0.213005538f,   0.10936069f,   0.0360007721f, 0.00759875814f,
                                   0.00102838008f};

// Thread 0 gets the block sums of three values.
__device__ __forceinline__ void block_sum3(float& a0, float& a1, float& a2, float (*s_red)[kLThreads / 32]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) { s_red[0][warp] = a0; s_red[1][warp] = a1; s_red[2][warp] = a2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        a0 = a1 = a2 = 0.0f;
        for (int w = 0; w < kLThreads / 32; ++w) { a0 += s_red[0][w]; a1 += s_red[1][w]; a2 += s_red[2][w]; }
    }
}

// full-resolution pixel (y, x) reads mask_lo[floor(y Hd / H), floor(x Wd / W)] (32-bit: sizes <= 4096)
__device__ __forceinline__ uint8_t mask_at(const uint8_t* mask_lo, int Hd, int Wd, int H, int W, int y, int x) {
    const int iy = min((int)((unsigned)(y * Hd) / (unsigned)H), Hd - 1);
    const int ix = min((int)((unsigned)(x * Wd) / (unsigned)W), Wd - 1);
    return mask_lo[iy * Wd + ix];
}

// ---- SSIM forward: 5 blurred moments, the map and its partials ------------
// Per 32 x 32 tile and channel: x, y with a 5-px halo in shared memory (zero
// outside the image), the horizontal 11-tap pass of x, y, x^2, y^2, xy for the
// 42 rows, then the vertical pass for two pixels per thread.
__global__ void __launch_bounds__(kLThreads) ssim_fwd_kernel(LossArgs a) {
    __shared__ float s_in[2][kHY][kHX];   // x, y
    __shared__ float s_h[5][kHY][kLTX];
    __shared__ float s_red[3][kLThreads / 32];
    const int c = blockIdx.z, W = a.W, H = a.H;
    const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY;
    const float* X = a.image + (size_t)c * W * H;
    const float* Y = a.gt + (size_t)c * W * H;
    constexpr int kLoadIt = (kHY * kHX + kLThreads - 1) / kLThreads;
    float lx[kLoadIt], ly[kLoadIt];
#pragma unroll
    for (int u = 0; u < kLoadIt; ++u) {  // every load in flight before any store
        const int i = threadIdx.x + u * kLThreads;
        const int r = i / kHX, q = i - r * kHX;
        const int gy = y0 + r - kWr, gx = x0 + q - kWr;
        const bool in = i < kHY * kHX && gx >= 0 && gx < W && gy >= 0 && gy < H;  // zero padding
        lx[u] = in ? __ldg(X + (size_t)gy * W + gx) : 0.0f;
        ly[u] = in ? __ldg(Y + (size_t)gy * W + gx) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kLoadIt; ++u) {
        const int i = threadIdx.x + u * kLThreads;
        if (i < kHY * kHX) {
            const int r = i / kHX, q = i - r * kHX;
            s_in[0][r][q] = lx[u]; s_in[1][r][q] = ly[u];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHY * kLTX; i += kLThreads) {
        const int r = i / kLTX, q = i - r * kLTX;
        float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const float xv = s_in[0][r][q + k], yv = s_in[1][r][q + k];
            const float wx = kSsimW[k] * xv, wy = kSsimW[k] * yv;
            m[0] += wx; m[1] += wy;
            m[2] = fmaf(wx, xv, m[2]); m[3] = fmaf(wy, yv, m[3]); m[4] = fmaf(wx, yv, m[4]);
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) s_h[j][r][q] = m[j];
    }
    __syncthreads();
    float sS = 0.0f, sA = 0.0f, sM = 0.0f;
    // two vertically adjacent pixels per thread: their windows share 10 of 12 rows
    const int tx = threadIdx.x & (kLTX - 1), ty0 = 2 * (threadIdx.x / kLTX);
    float m[2][5] = {{0.f, 0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int k = 0; k <= kWin; ++k) {
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const float v = s_h[j][ty0 + k][tx];
            if (k < kWin) m[0][j] = fmaf(kSsimW[k], v, m[0][j]);
            if (k > 0) m[1][j] = fmaf(kSsimW[k - 1], v, m[1][j]);
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int ty = ty0 + h;
        const int gx = x0 + tx, gy = y0 + ty;
        if (gx >= W || gy >= H) continue;
        const float mx = m[h][0], my = m[h][1], exx = m[h][2], eyy = m[h][3], exy = m[h][4];
        const float A1 = 2.f * mx * my + kC1, A2 = 2.f * (exy - mx * my) + kC2;
        const float B1 = mx * mx + my * my + kC1, B2 = (exx - mx * mx) + (eyy - my * my) + kC2;
        const float iB1 = __frcp_rn(B1), iB2 = __frcp_rn(B2);
        const float S = A1 * A2 * iB1 * iB2;
        const size_t pix = (size_t)c * W * H + (size_t)gy * W + gx;
        a.d_mu[pix] = 2.f * my * (A2 - A1) * iB1 * iB2 - S * 2.f * mx * (iB1 - iB2);
        a.d_e2[pix] = -S * iB2;
        a.d_exy[pix] = 2.f * A1 * iB1 * iB2;
        const float d = fabsf(s_in[0][ty + kWr][tx + kWr] - s_in[1][ty + kWr][tx + kWr]);
        sS += S;
        sA += d;
        if (a.mask_lo && mask_at(a.mask_lo, a.Hd, a.Wd, H, W, gy, gx)) sM += d;
    }
    block_sum3(sS, sA, sM, s_red);
    if (threadIdx.x == 0) {
        const int blk = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        a.partial[3 * blk] = sS;
        a.partial[3 * blk + 1] = sA;
        a.partial[3 * blk + 2] = sM;
    }
}

// ---- backward: the window's adjoint on the partials + L1 / L_omega ---------
__global__ void __launch_bounds__(kLThreads) ssim_bwd_kernel(LossArgs a) {
    __shared__ float s_p[3][kHY][kHX];
    __shared__ float s_h[3][kHY][kLTX];
    const int c = blockIdx.z, W = a.W, H = a.H;
    const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY;
    const size_t base = (size_t)c * W * H;
    constexpr int kLoadIt = (kHY * kHX + kLThreads - 1) / kLThreads;
    float l0[kLoadIt], l1[kLoadIt], l2[kLoadIt];
#pragma unroll
    for (int u = 0; u < kLoadIt; ++u) {  // every load in flight before any store
        const int i = threadIdx.x + u * kLThreads;
        const int r = i / kHX, q = i - r * kHX;
        const int gy = y0 + r - kWr, gx = x0 + q - kWr;
        const bool in = i < kHY * kHX && gx >= 0 && gx < W && gy >= 0 && gy < H;  // no window off the image
        const size_t p = base + (size_t)gy * W + gx;
        l0[u] = in ? a.d_mu[p] : 0.0f;
        l1[u] = in ? a.d_e2[p] : 0.0f;
        l2[u] = in ? a.d_exy[p] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kLoadIt; ++u) {
        const int i = threadIdx.x + u * kLThreads;
        if (i < kHY * kHX) {
            const int r = i / kHX, q = i - r * kHX;
            s_p[0][r][q] = l0[u]; s_p[1][r][q] = l1[u]; s_p[2][r][q] = l2[u];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHY * kLTX; i += kLThreads) {
        const int r = i / kLTX, q = i - r * kLTX;
        float b[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const float w = kSsimW[k];
#pragma unroll
            for (int j = 0; j < 3; ++j) b[j] = fmaf(w, s_p[j][r][q + k], b[j]);
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) s_h[j][r][q] = b[j];
    }
    __syncthreads();
    const float lam_l1 = 1.0f - a.lambda_ssim - a.lambda_omega;
    const int tx = threadIdx.x & (kLTX - 1), ty0 = 2 * (threadIdx.x / kLTX);
    float g[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
#pragma unroll
    for (int k = 0; k <= kWin; ++k) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float v = s_h[j][ty0 + k][tx];
            if (k < kWin) g[0][j] = fmaf(kSsimW[k], v, g[0][j]);
            if (k > 0) g[1][j] = fmaf(kSsimW[k - 1], v, g[1][j]);
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int gx = x0 + tx, gy = y0 + ty0 + h;
        if (gx >= W || gy >= H) continue;
        const size_t p = base + (size_t)gy * W + gx;
        const float xv = __ldg(a.image + p), yv = __ldg(a.gt + p);
        const float dS = g[h][0] + 2.f * xv * g[h][1] + yv * g[h][2];   // N d mean SSIM / dx
        const float d = xv - yv;
        const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        const float m = a.mask_lo && mask_at(a.mask_lo, a.Hd, a.Wd, H, W, gy, gx) ? 1.f : 0.f;
        a.dL_dimage[p] = (lam_l1 * sg - a.lambda_ssim * dS + a.lambda_omega * sg * m) * a.inv_n;
    }
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
