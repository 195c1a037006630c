// train.cu -- the optimizer and shape-aware density control (SURVEY.md §8(f)
// NEXT-2; §4.4 :348-358 and Appendix :1227-1271; readings DESIGN.md
// R29-R33): a fused bias-corrected Adam step over the planar parameter buffer
// with per-plane learning rates, the opacity / shape resets, the densification
// statistic (view-space gradient norms, between S5a and S5b), and one
// densify+prune pass that writes the new particle set in a fixed order
//   [kept particles, split parents replaced by their first child] ++ [clones]
//   ++ [second split children]
// through three exclusive scans (keep, clone, split flags).  Split children
// sit at mu + R (s . z), z from splitmix64 + Box-Muller on (seed, particle,
// child) -- the generator the oracle implements independently.
// Everything HBM-bound: coalesced plane-major loads and stores.
#include <algorithm>
#include <cmath>

#include "ges_internal.h"

namespace ges {

// ---- Adam -------------------------------------------------------------------
__device__ __forceinline__ float plane_lr(const AdamArgs& a, int plane) {
    const int K3 = a.n_planes - 12;  // 3K SH planes
    if (plane < 3) return a.lr_position;
    if (plane < 6) return a.lr_scaling;
    if (plane < 10) return a.lr_rotation;
    if (plane == 10) return a.lr_opacity;
    if (plane < 14) return a.lr_feature_dc;
    if (plane < 11 + K3) return a.lr_feature_rest;
    return a.lr_shape;
}

__device__ __forceinline__ void adam1(const AdamArgs& a, float lr, float g, float& p, float& m, float& v) {
    m = a.beta1 * m + (1.0f - a.beta1) * g;
    v = a.beta2 * v + (1.0f - a.beta2) * g * g;
    p -= lr * (m * a.inv_bc1) / (sqrtf(v * a.inv_bc2) + a.eps);
}

__global__ void adam_kernel(AdamArgs a) {
    const int plane = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.P) return;
    const float lr = plane_lr(a, plane);
    const size_t q = (size_t)plane * a.P + i;
    float p = a.params[q], m = a.m[q], v = a.v[q];
    adam1(a, lr, a.grads[q], p, m, v);
    a.params[q] = p; a.m[q] = m; a.v[q] = v;
}

// P % 4 == 0 and 16-B aligned buffers: four elements per thread, float4 loads/stores
__global__ void adam4_kernel(AdamArgs a) {
    const int plane = blockIdx.y;
    const int64_t i4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * i4 >= a.P) return;
    const float lr = plane_lr(a, plane);
    const size_t q = ((size_t)plane * a.P) / 4 + i4;
    float4 p = reinterpret_cast<float4*>(a.params)[q];
    float4 m = reinterpret_cast<float4*>(a.m)[q];
    float4 v = reinterpret_cast<float4*>(a.v)[q];
    const float4 g = reinterpret_cast<const float4*>(a.grads)[q];
    adam1(a, lr, g.x, p.x, m.x, v.x);
    adam1(a, lr, g.y, p.y, m.y, v.y);
    adam1(a, lr, g.z, p.z, m.z, v.z);
    adam1(a, lr, g.w, p.w, m.w, v.w);
    reinterpret_cast<float4*>(a.params)[q] = p;
    reinterpret_cast<float4*>(a.m)[q] = m;
    reinterpret_cast<float4*>(a.v)[q] = v;
}

// A contiguous range [begin, begin + count) of the flattened [C][P] buffer (a
// ZeRO-1 shard: dist.ShardedAdam); the gradient holds the range only.  Four
// elements per thread when begin, P are multiples of 4 (a float4 never straddles
// a plane), else one.
template <bool VEC>
__global__ void adam_range_kernel(AdamArgs a, int64_t begin, int64_t count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (VEC) {
        for (int64_t i4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 4 * i4 < count; i4 += stride) {
            const int64_t q = begin + 4 * i4;
            const float lr = plane_lr(a, (int)(q / a.P));
            float4 p = *reinterpret_cast<float4*>(a.params + q);
            float4 m = *reinterpret_cast<float4*>(a.m + q);
            float4 v = *reinterpret_cast<float4*>(a.v + q);
            const float4 g = *reinterpret_cast<const float4*>(a.grads + 4 * i4);
            adam1(a, lr, g.x, p.x, m.x, v.x);
            adam1(a, lr, g.y, p.y, m.y, v.y);
            adam1(a, lr, g.z, p.z, m.z, v.z);
            adam1(a, lr, g.w, p.w, m.w, v.w);
            *reinterpret_cast<float4*>(a.params + q) = p;
            *reinterpret_cast<float4*>(a.m + q) = m;
            *reinterpret_cast<float4*>(a.v + q) = v;
        }
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
            const int64_t q = begin + i;
            const float lr = plane_lr(a, (int)(q / a.P));
            float p = a.params[q], m = a.m[q], v = a.v[q];
            adam1(a, lr, a.grads[i], p, m, v);
            a.params[q] = p; a.m[q] = m; a.v[q] = v;
        }
    }
}

cudaError_t launch_adam_range(const AdamArgs& a, int64_t begin, int64_t count, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    const bool vec = begin % 4 == 0 && count % 4 == 0 && a.P % 4 == 0 && al(a.params) && al(a.grads) && al(a.m) &&
                     al(a.v);
    const int64_t work = vec ? count / 4 : count;
    const int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)num_sms() * 16);
    if (vec) adam_range_kernel<true><<<grid, 256, 0, stream>>>(a, begin, count);
    else adam_range_kernel<false><<<grid, 256, 0, stream>>>(a, begin, count);
    return cudaGetLastError();
}

cudaError_t launch_adam(const AdamArgs& a, cudaStream_t stream) {
    auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    if (a.P % 4 == 0 && al(a.params) && al(a.grads) && al(a.m) && al(a.v)) {
        const dim3 grid((unsigned)((a.P / 4 + 255) / 256), (unsigned)a.n_planes);
        adam4_kernel<<<grid, 256, 0, stream>>>(a);
    } else {
        const dim3 grid((unsigned)((a.P + 255) / 256), (unsigned)a.n_planes);
        adam_kernel<<<grid, 256, 0, stream>>>(a);
    }
    return cudaGetLastError();
}

// ---- resets -------------------------------------------------------------------
__global__ void reset_kernel(float* params, int64_t P, int plane, float cap, int mode) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    float* p = params + (size_t)plane * P + i;
    *p = mode == 0 ? fminf(*p, cap) : cap;  // 0: opacity cap, 1: shape := cap (beta 2)
}

cudaError_t launch_reset(float* params, int64_t P, int plane, float cap, int mode, cudaStream_t stream) {
    reset_kernel<<<(unsigned)((P + 255) / 256), 256, 0, stream>>>(params, P, plane, cap, mode);
    return cudaGetLastError();
}

// ---- densification statistic ------------------------------------------------------
__global__ void densify_stats_kernel(DensifyStatsArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.P || a.status[i] != GES_VISIBLE) return;
    // dL/du, dL/dv from S5a's raw moments (record layout: ges.h, particle_bwd.cu)
    const float m1 = a.grad2d[(size_t)i * kGrad2dStride], s1 = a.grad2d[(size_t)i * kGrad2dStride + 1];
    const float4 p0 = a.pay0[i], p1 = a.pay1[i];
    const float kl = a.kernel == GES_KERNEL_EXACT_BETA ? p1.y * 0.5f * a.pay3[i] : 0.69314718055994531f;
    const float cA = p0.z * (-0.5f * kLog2e), cB = p0.w * (-kLog2e), cC = p1.x * (-0.5f * kLog2e);
    const float E = kl * m1, F = kl * s1;
    const float du = 2.f * cA * E + cB * F, dv = cB * E + 2.f * cC * F;
    const float gx = du * 0.5f * (float)a.W, gy = dv * 0.5f * (float)a.H;  // NDC units
    a.accum[i] += sqrtf(gx * gx + gy * gy);
    a.count[i] += 1.0f;
}

cudaError_t launch_densify_stats(const DensifyStatsArgs& a, cudaStream_t stream) {
    densify_stats_kernel<<<(unsigned)((a.P + 255) / 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

// ---- densify + prune ------------------------------------------------------------
constexpr int kDpThreads = 256, kDpItems = 8, kDpBlock = kDpThreads * kDpItems;

__device__ __forceinline__ int dp_action(const DensifyArgs& a, int64_t i) {
    const float logit = a.params[(size_t)10 * a.P + i];
    const float kappa = 1.0f / (1.0f + expf(-logit));
    const float beta = a.params[(size_t)(a.n_planes - 1) * a.P + i];
    const float phib = 2.0f / (1.0f + expf(-a.rho * (beta - 2.0f)));
    if (kappa < a.opacity_prune || phib < a.shape_prune) return 0;
    const float c = a.count[i];
    const float avg = c > 0.0f ? a.accum[i] / c : 0.0f;
    if (!(avg >= a.grad_threshold)) return 1;
    float smax = 0.0f;
    for (int k = 0; k < 3; ++k) smax = fmaxf(smax, expf(a.params[(size_t)(3 + k) * a.P + i]));
    return smax <= a.percent_dense * a.extent ? 2 : 3;
}

// per block: counts of (keep, clone, split) -> block_cnt[3 b + k]
__global__ void __launch_bounds__(kDpThreads) dp_count_kernel(DensifyArgs a) {
    __shared__ int s[3][kDpThreads / 32];
    const int64_t b0 = (int64_t)blockIdx.x * kDpBlock;
    int c[3] = {0, 0, 0};
    for (int j = 0; j < kDpItems; ++j) {
        const int64_t i = b0 + j * kDpThreads + threadIdx.x;
        if (i < a.P) {
            const int act = dp_action(a, i);
            a.action[i] = (uint8_t)act;
            c[0] += act > 0; c[1] += act == 2; c[2] += act == 3;
        }
    }
    for (int k = 0; k < 3; ++k) {
        int v = c[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) s[k][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        int t = 0;
        for (int w = 0; w < kDpThreads / 32; ++w) t += s[threadIdx.x][w];
        a.block_cnt[3 * blockIdx.x + threadIdx.x] = t;
    }
}

// one CTA: exclusive scan of the block counts per kind; totals -> new size
__global__ void dp_scan_kernel(DensifyArgs a) {
    __shared__ long long s_tot[3];
    const int k = threadIdx.x;
    if (k < 3) {
        long long run = 0;
        for (int b = 0; b < a.nblocks; ++b) {
            const int v = a.block_cnt[3 * b + k];
            a.block_cnt[3 * b + k] = (int)run;
            run += v;
        }
        a.totals[k] = run;
        s_tot[k] = run;
    }
    __syncthreads();
    if (k == 0) *a.P_out = s_tot[0] + s_tot[1] + s_tot[2];
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform24(uint64_t seed, uint64_t particle, int child, int k) {
    const uint64_t key = seed * 0x100000001B3ull + particle * 16ull + (uint64_t)child * 4ull + (uint64_t)k;
    return ((double)(splitmix64(key) >> 40) + 0.5) / 16777216.0;
}

__device__ void copy_particle(const DensifyArgs& a, int64_t src, int64_t dst, bool zero_moments) {
    for (int p = 0; p < a.n_planes; ++p) {
        const size_t s = (size_t)p * a.P + src, d = (size_t)p * a.cap_out + dst;
        a.params_out[d] = a.params[s];
        a.m_out[d] = zero_moments ? 0.0f : a.m[s];
        a.v_out[d] = zero_moments ? 0.0f : a.v[s];
    }
}

// a split child: the parent's planes with mean mu + R (s . z), log-scales - ln 1.6, zero moments
__device__ void write_child(const DensifyArgs& a, int64_t src, int64_t dst, int child) {
    copy_particle(a, src, dst, true);
    const float* P0 = a.params;
    const size_t P = (size_t)a.P, C = (size_t)a.cap_out;
    float q[4];
    for (int k = 0; k < 4; ++k) q[k] = P0[(6 + k) * P + src];
    const float n = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const float w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                        2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                        2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
    double u[4];
    for (int k = 0; k < 4; ++k) u[k] = uniform24(a.seed, (uint64_t)src, child, k);
    const double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
    const double pi2 = 6.283185307179586;
    const float zz[3] = {(float)(r0 * cos(pi2 * u[1])), (float)(r0 * sin(pi2 * u[1])), (float)(r1 * cos(pi2 * u[3]))};
    float sz[3];
    for (int k = 0; k < 3; ++k) sz[k] = expf(P0[(3 + k) * P + src]) * zz[k];
    for (int r = 0; r < 3; ++r)
        a.params_out[r * C + dst] = P0[r * P + src] + (R[3 * r] * sz[0] + R[3 * r + 1] * sz[1] + R[3 * r + 2] * sz[2]);
    for (int k = 0; k < 3; ++k) a.params_out[(3 + k) * C + dst] = P0[(3 + k) * P + src] - 0.47000363f;  // ln 1.6
}

__global__ void __launch_bounds__(kDpThreads) dp_scatter_kernel(DensifyArgs a) {
    __shared__ int s_off[3][kDpThreads];
    const int64_t b0 = (int64_t)blockIdx.x * kDpBlock;
    // block-local exclusive ranks: each thread owns kDpItems consecutive particles
    int cnt[3] = {0, 0, 0}, act[kDpItems];
    for (int j = 0; j < kDpItems; ++j) {
        const int64_t i = b0 + (int64_t)threadIdx.x * kDpItems + j;
        act[j] = i < a.P ? (int)a.action[i] : 0;
        cnt[0] += act[j] > 0; cnt[1] += act[j] == 2; cnt[2] += act[j] == 3;
    }
    for (int k = 0; k < 3; ++k) s_off[k][threadIdx.x] = cnt[k];
    __syncthreads();
    if (threadIdx.x < 3) {  // serial exclusive scan of 256 values per kind (small)
        int run = 0;
        for (int t = 0; t < kDpThreads; ++t) { const int v = s_off[threadIdx.x][t]; s_off[threadIdx.x][t] = run; run += v; }
    }
    __syncthreads();
    int64_t pk = (int64_t)a.block_cnt[3 * blockIdx.x] + s_off[0][threadIdx.x];
    int64_t pc = a.totals[0] + a.block_cnt[3 * blockIdx.x + 1] + s_off[1][threadIdx.x];
    int64_t ps = a.totals[0] + a.totals[1] + a.block_cnt[3 * blockIdx.x + 2] + s_off[2][threadIdx.x];
    for (int j = 0; j < kDpItems; ++j) {
        const int64_t i = b0 + (int64_t)threadIdx.x * kDpItems + j;
        if (i >= a.P || act[j] == 0) continue;
        if (act[j] == 3) {
            write_child(a, i, pk++, 0);
            write_child(a, i, ps++, 1);
        } else {
            copy_particle(a, i, pk++, false);
            if (act[j] == 2) copy_particle(a, i, pc++, true);
        }
    }
}

int64_t densify_blocks(int64_t P) { return (P + kDpBlock - 1) / kDpBlock; }

cudaError_t launch_densify_prune(const DensifyArgs& a0, cudaStream_t stream) {
    DensifyArgs a = a0;
    a.nblocks = (int)densify_blocks(a.P);
    cudaError_t e;
    dp_count_kernel<<<a.nblocks, kDpThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    dp_scan_kernel<<<1, 32, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    dp_scatter_kernel<<<a.nblocks, kDpThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
