// mix1d.cu -- SURVEY.md §8(f) NEXT-4: the paper's 1-D mixture simulation
// (PAPER.md Appendix :606-745) and the Theorem-1 error integrals (:555-603).
//
// ges_mix_fit runs a whole sweep of independent fits in one launch: one CTA
// per run (model, weight mode, N components, target signal), parameters and
// Adam moments in shared memory, `steps` Adam steps on the MSE of the mixture
// over the n-sample grid.  Each step is two passes over the samples:
//   pass 1  (thread per sample)      prediction h(x_j) = sum_i w_i phi_i(x_j) and
//                                    the residual r_j = h(x_j) - y_j (shared memory)
//   pass 2  (warp per component)     the few sample sums the component's gradient
//                                    needs (e.g. GMM: sum r e d, sum r e d^2, sum r e),
//                                    warp-reduced; the per-component constants
//                                    (w, 1/(2 s^2 + eps), 4 s, ...) are applied once.
// Models (d = x - mu, D = 2 s^2 + eps, eps = 1e-8, nu = 4):
//   GMM  e^{-d^2/D}            DoG  e^{-d^2/D} - e^{-d^2/(2 s^2/nu + eps)}
//   LoG  (1 - d^2/s^2) e^{-d^2/D}                GEF  e^{-|d|^beta / D}  (one beta)
// weights w = omega (real) or exp(omega) (positive; R35).  The
// exponentials are MUFU ex2 of pre-scaled arguments, |d|^beta = ex2(beta lg2|d|).
//
// ges_theorem1_errors evaluates E_GEF(alpha, beta) = int |S - f| for the square
// wave S (amplitude A, width L) by quadrature, one warp per (alpha, beta):
// E = A L + 2 A I_total - 4 A I_1, I_total = alpha Gamma(1 + 1/beta), and
// I_1 = int_0^{L/2} e^{-(t/alpha)^beta} dt by composite Simpson after
// t = (L/2) s^m, m = ceil(2 / beta) (smooth at 0 for every beta).
#include <cmath>

#include "ges_internal.h"

namespace ges {

constexpr int kMixThreads = 256;
constexpr int kMixWarps = kMixThreads / 32;
constexpr float kMixEps = 1e-8f;
constexpr float kMixNu = 4.0f;
constexpr float kMixLog2e = 1.4426950408889634f;

__device__ __forceinline__ float mix_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float mix_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float mix_signal(int kind, float x, float width) {
    const float half = 0.5f * width;
    const bool inside = x > -half && x < half;
    switch (kind) {
        case GES_SIG_SQUARE: return inside ? 1.0f : 0.0f;
        case GES_SIG_TRIANGLE: return inside ? half - fabsf(x) : 0.0f;
        case GES_SIG_PARABOLIC: return inside ? half * half - x * x : 0.0f;
        case GES_SIG_HALF_SINUSOID: return inside ? sinf((x + half) * 3.14159265358979f / width) : 0.0f;
        case GES_SIG_EXPONENTIAL: return inside ? expf(-fabsf(x)) : 0.0f;
        default: return expf(-x * x / (2.0f * width * width));  // GES_SIG_GAUSSIAN
    }
}

__global__ void mix_signal_kernel(int kind, float width, float x_lo, float h, int n, float* y) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) y[j] = mix_signal(kind, fmaf((float)j, h, x_lo), width);
}

// Per-component constants of one step.
struct MixComp {
    float mu, w, dw;  // mean, weight, d weight / d omega
    float k1, k2;     // -log2e / D (and the DoG's narrow -log2e / D2, LoG's 1 / s^2)
    float s4;         // 4 s
};

template <int MODEL>
__device__ __forceinline__ float mix_phi(const MixComp& c, float x, float beta) {
    const float d = x - c.mu, d2 = d * d;
    if (MODEL == GES_MIX_GMM) return mix_ex2(d2 * c.k1);
    if (MODEL == GES_MIX_DOG) return mix_ex2(d2 * c.k1) - mix_ex2(d2 * c.k2);
    if (MODEL == GES_MIX_LOG) return (1.0f - d2 * c.k2) * mix_ex2(d2 * c.k1);
    const float ad = fabsf(d);
    const float p = ad > 0.0f ? mix_ex2(beta * mix_lg2(ad)) : 0.0f;
    return mix_ex2(p * c.k1);
}

__device__ __forceinline__ float mix_warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}


// shared-memory block: th | m | v | grad | comp | residuals
struct MixSmem {
    float th[3 * GES_MIX_MAX_N + 1];
    float m[3 * GES_MIX_MAX_N + 1];
    float v[3 * GES_MIX_MAX_N + 1];
    float g[3 * GES_MIX_MAX_N + 1];
    float gb[GES_MIX_MAX_N];  // per-component beta-gradient parts (GEF)
    MixComp comp[GES_MIX_MAX_N];
    float red[kMixWarps];
};

template <int MODEL>
__device__ void mix_run(const MixArgs& a, MixSmem& S, float* r, int N, bool positive, const float* y, bool fit,
                        float* loss_out, float* grad_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int np = 3 * N + 1;
    const float inv_n2 = 2.0f / (float)a.n;
    const int steps = fit ? a.steps : 0;
    for (int step = 0; step <= steps; ++step) {
        const bool last = step == steps;  // the final pass: loss (and eval gradient) only
        // per-component constants
        for (int i = tid; i < N; i += kMixThreads) {
            MixComp c;
            c.mu = S.th[i];
            const float s = S.th[N + i], om = S.th[2 * N + i];
            c.w = positive ? expf(om) : om;
            c.dw = positive ? c.w : 1.0f;
            const float D = 2.0f * s * s + kMixEps;
            c.k1 = -kMixLog2e / D;
            c.k2 = MODEL == GES_MIX_DOG ? -kMixLog2e / (2.0f * s * s / kMixNu + kMixEps)
                                        : (MODEL == GES_MIX_LOG ? 1.0f / (s * s) : 0.0f);
            c.s4 = 4.0f * s;
            S.comp[i] = c;
        }
        __syncthreads();
        const float beta = S.th[3 * N];
        // pass 1: residuals (and the loss)
        float lsum = 0.0f;
        for (int j = tid; j < a.n; j += kMixThreads) {
            const float x = fmaf((float)j, a.h, a.x_lo);
            float pred = 0.0f;
            for (int i = 0; i < N; ++i) {
                const MixComp c = S.comp[i];
                pred = fmaf(c.w, mix_phi<MODEL>(c, x, beta), pred);
            }
            const float rj = pred - y[j];
            r[j] = rj;
            lsum = fmaf(rj, rj, lsum);
        }
        if (last) {
            lsum = mix_warp_sum(lsum);
            if (lane == 0) S.red[warp] = lsum;
        }
        __syncthreads();
        if (last && tid == 0) {
            float t = 0.0f;
            for (int w = 0; w < kMixWarps; ++w) t += S.red[w];
            *loss_out = t / (float)a.n;
        }
        if (last && !grad_out) break;
        // pass 2: per-component sample sums, warp per component
        for (int i = warp; i < N; i += kMixWarps) {
            const MixComp c = S.comp[i];
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
            for (int j = lane; j < a.n; j += 32) {
                const float x = fmaf((float)j, a.h, a.x_lo);
                const float rj = r[j];
                const float d = x - c.mu, d2 = d * d;
                if (MODEL == GES_MIX_GMM) {
                    const float e = mix_ex2(d2 * c.k1) * rj;
                    s0 += e * d; s1 += e * d2; s2 += e;
                } else if (MODEL == GES_MIX_DOG) {
                    const float e1 = mix_ex2(d2 * c.k1) * rj, e2 = mix_ex2(d2 * c.k2) * rj;
                    s0 += e1 * d; s1 += e2 * d; s2 += e1 * d2; s3 += e2 * d2; s4 += e1 - e2;
                } else if (MODEL == GES_MIX_LOG) {
                    const float e = mix_ex2(d2 * c.k1) * rj, ae = (1.0f - d2 * c.k2) * e;
                    s0 += e * d; s1 += ae * d; s2 += e * d2; s3 += ae * d2; s4 += ae;
                } else {
                    const float ad = fabsf(d);
                    if (ad > 0.0f) {  // every |d|^beta term is 0 at d = 0 (oracle/mix1d.py)
                        const float l2 = mix_lg2(ad);
                        const float p = mix_ex2(beta * l2);
                        const float e = mix_ex2(p * c.k1) * rj, ep = e * p;
                        s0 += __fdividef(ep, d); s1 += ep; s2 += e; s3 += ep * l2;
                    } else {
                        s2 += rj;  // phi = 1 at the mean
                    }
                }
            }
            s0 = mix_warp_sum(s0); s1 = mix_warp_sum(s1); s2 = mix_warp_sum(s2);
            if (MODEL != GES_MIX_GMM) { s3 = mix_warp_sum(s3); s4 = mix_warp_sum(s4); }
            if (lane == 0) {
                const float s = S.th[N + i];
                const float iD = 1.0f / (2.0f * s * s + kMixEps);
                float gmu, gs, gom, gbe = 0.0f;
                if (MODEL == GES_MIX_GMM) {
                    gmu = 2.0f * iD * s0; gs = c.s4 * iD * iD * s1; gom = s2;
                } else if (MODEL == GES_MIX_DOG) {
                    const float iD2 = 1.0f / (2.0f * s * s / kMixNu + kMixEps);
                    gmu = 2.0f * iD * s0 - 2.0f * iD2 * s1;
                    gs = c.s4 * iD * iD * s2 - (c.s4 / kMixNu) * iD2 * iD2 * s3;
                    gom = s4;
                } else if (MODEL == GES_MIX_LOG) {
                    const float ig2 = c.k2;
                    gmu = 2.0f * ig2 * s0 + 2.0f * iD * s1;
                    gs = 2.0f * ig2 / s * s2 + c.s4 * iD * iD * s3;
                    gom = s4;
                } else {
                    gmu = beta * iD * s0;
                    gs = c.s4 * iD * iD * s1;
                    gom = s2;
                    gbe = -0.69314718055994531f * iD * s3;  // ln|d| = ln2 lg2|d|
                }
                S.g[i] = c.w * gmu * inv_n2;
                S.g[N + i] = c.w * gs * inv_n2;
                S.g[2 * N + i] = c.dw * gom * inv_n2;
                S.gb[i] = c.w * gbe * inv_n2;
            }
        }
        __syncthreads();
        if (tid == 0) {
            float t = 0.0f;
            if (MODEL == GES_MIX_GEF)
                for (int i = 0; i < N; ++i) t += S.gb[i];
            S.g[3 * N] = t;
        }
        __syncthreads();
        if (last) {  // eval: the gradient at the given parameters
            for (int k = tid; k < np; k += kMixThreads) grad_out[k] = S.g[k];
            break;
        }
        // Adam (torch.optim.Adam): bias corrections in double, once per step
        const int t = a.t0 + step + 1;
        const float bc1 = (float)(1.0 / (1.0 - pow((double)a.b1, (double)t)));
        const float bc2 = (float)(1.0 / (1.0 - pow((double)a.b2, (double)t)));
        for (int k = tid; k < np; k += kMixThreads) {
            const float g = S.g[k];
            const float m = a.b1 * S.m[k] + (1.0f - a.b1) * g;
            const float v = a.b2 * S.v[k] + (1.0f - a.b2) * g * g;
            S.m[k] = m;
            S.v[k] = v;
            S.th[k] -= a.lr * (m * bc1) / (sqrtf(v * bc2) + a.eps);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kMixThreads) mix_kernel(MixArgs a, int fit) {
    extern __shared__ float s_r[];  // [n] residuals
    __shared__ MixSmem S;
    const int run = blockIdx.x;
    if (run >= a.n_runs) return;
    const ges_mix_run R = a.runs[run];
    const int N = R.n_comp;
    float* loss = a.loss + run;
    if (N < 1 || N > GES_MIX_MAX_N || 3 * N + 1 > a.stride || R.model < 0 || R.model > 3 || R.target < 0) {
        if (threadIdx.x == 0) *loss = __int_as_float(0x7fc00000);  // invalid run: NaN
        return;
    }
    const int np = 3 * N + 1;
    float* th = a.params + (size_t)run * a.stride;
    for (int k = threadIdx.x; k < np; k += kMixThreads) {
        S.th[k] = th[k];
        S.m[k] = fit ? a.m[(size_t)run * a.stride + k] : 0.0f;
        S.v[k] = fit ? a.v[(size_t)run * a.stride + k] : 0.0f;
    }
    __syncthreads();
    const float* y = a.targets + (size_t)R.target * a.n;
    float* gout = (!fit && a.grad) ? a.grad + (size_t)run * a.stride : nullptr;
    const bool pos = R.positive != 0;
    switch (R.model) {
        case GES_MIX_GMM: mix_run<GES_MIX_GMM>(a, S, s_r, N, pos, y, fit, loss, gout); break;
        case GES_MIX_DOG: mix_run<GES_MIX_DOG>(a, S, s_r, N, pos, y, fit, loss, gout); break;
        case GES_MIX_LOG: mix_run<GES_MIX_LOG>(a, S, s_r, N, pos, y, fit, loss, gout); break;
        default: mix_run<GES_MIX_GEF>(a, S, s_r, N, pos, y, fit, loss, gout); break;
    }
    if (fit) {
        __syncthreads();
        for (int k = threadIdx.x; k < np; k += kMixThreads) {
            th[k] = S.th[k];
            a.m[(size_t)run * a.stride + k] = S.m[k];
            a.v[(size_t)run * a.stride + k] = S.v[k];
        }
    }
}

// ---- Theorem 1 --------------------------------------------------------------------
__global__ void theorem1_kernel(const float* alpha, int na, const float* beta, int nb, float A, float L, int n,
                                float* E) {
    const int lane = threadIdx.x & 31;
    const int64_t pair = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (pair >= (int64_t)na * nb) return;
    const float al = alpha[pair / nb], be = beta[pair % nb];
    if (!(al > 0.0f) || !(be > 0.0f)) {
        if (lane == 0) E[pair] = __int_as_float(0x7fc00000);
        return;
    }
    const int m = max(1, (int)ceilf(2.0f / be));
    const float c = powf(0.5f * L / al, be);   // (L / (2 alpha))^beta
    const float mb = (float)m * be;
    const float hs = 1.0f / (float)n;
    // Simpson on s in [0, 1]: f(s) = m s^(m-1) exp(-c s^(m beta)), times L/2
    float acc = 0.0f;
    for (int k = lane; k <= n; k += 32) {
        const float s = (float)k * hs;
        const float sm1 = m == 1 ? 1.0f : (k == 0 ? 0.0f : powf(s, (float)(m - 1)));
        const float ex = k == 0 ? 1.0f : expf(-c * exp2f(mb * log2f(s)));  // (c may be inf)
        const float f = (float)m * sm1 * ex;
        const float wgt = (k == 0 || k == n) ? 1.0f : ((k & 1) ? 4.0f : 2.0f);
        acc = fmaf(wgt, f, acc);
    }
    acc = mix_warp_sum(acc);
    if (lane == 0) {
        const float I1 = 0.5f * L * acc * hs / 3.0f;
        const float It = al * tgammaf(1.0f + 1.0f / be);
        E[pair] = A * L + 2.0f * A * It - 4.0f * A * I1;
    }
}

// MUFU issue-rate probe (the mix1d roofline's denominator): 8 independent ex2
// chains per thread; out[tid] keeps the chains live.
__global__ void __launch_bounds__(256) mufu_probe_kernel(float* out, int iters) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = -1e-3f * (float)(threadIdx.x + k);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = mix_ex2(v[k]) - 1.0f;
    }
    float t = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += v[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

cudaError_t launch_mufu_probe(float* out, int iters, int blocks, cudaStream_t stream) {
    mufu_probe_kernel<<<blocks, 256, 0, stream>>>(out, iters);
    return cudaGetLastError();
}

cudaError_t launch_mix_signal(int kind, float width, float x_lo, float h, int n, float* y, cudaStream_t stream) {
    mix_signal_kernel<<<(n + 255) / 256, 256, 0, stream>>>(kind, width, x_lo, h, n, y);
    return cudaGetLastError();
}

cudaError_t launch_mix(const MixArgs& a, bool fit, cudaStream_t stream) {
    const size_t smem = sizeof(float) * (size_t)a.n;
    static size_t configured_dev[kMaxDevices] = {0};
    size_t& configured = configured_dev[current_device()];
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    mix_kernel<<<a.n_runs, kMixThreads, smem, stream>>>(a, fit ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_theorem1(const float* alpha, int na, const float* beta, int nb, float A, float L, int n, float* E,
                            cudaStream_t stream) {
    const int64_t threads = (int64_t)na * nb * 32;
    theorem1_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(alpha, na, beta, nb, A, L, n, E);
    return cudaGetLastError();
}

}  // namespace ges
