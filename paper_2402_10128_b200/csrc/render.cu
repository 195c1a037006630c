// render.cu -- S4 and S5a: per-16x16-tile front-to-back
// alpha compositing (Eq. 3, discretised as
// C = sum_i c_i alpha_i prod_{j<i} (1 - alpha_j) + T_final * bg) and its
// adjoint.  Inherited rules (R7, R12): alpha = min(0.99, kappa G),
// entries with alpha < 1/255 skipped, a pixel stops -- without compositing --
// at the first entry that would take T below 1e-4.  The per-pixel kernel is
// the Gaussian of the phi-bar-scaled covariance (the paper's approximate
// rasterization "without taking the beta exponent"; R6).
//
// One CTA per tile, one thread per pixel.  Each batch of 256 list entries is
// gathered once into shared memory (payload of the particle: 36 B) and then
// evaluated by all 256 pixels; __syncthreads_count retires a tile as soon as
// every pixel has terminated.  The backward walks the same lists back to
// front from the last composited entry and reduces the nine per-pair
// gradients across each warp with a recursive-halving shuffle (16 SHFL per
// warp and entry instead of 45) into shared accumulators that are flushed
// with one global atomic per (particle, tile, component).
#include "ges_internal.h"

namespace ges {

__device__ __forceinline__ Splat2D load_splat(const float4* pay0, const float4* pay1, const float* pay2, uint32_t p) {
    const float4 a = __ldg(pay0 + p);
    const float4 b = __ldg(pay1 + p);
    Splat2D s;
    s.u = a.x; s.v = a.y;
    s.A = __fmul_rn(__fmul_rn(-0.5f, a.z), kLog2e);
    s.B = __fmul_rn(-a.w, kLog2e);
    s.C = __fmul_rn(__fmul_rn(-0.5f, b.x), kLog2e);
    s.kappa = b.y; s.r = b.z; s.g = b.w;
    s.b = __ldg(pay2 + p);
    return s;
}

// exact same instruction sequence in forward and backward
__device__ __forceinline__ float raw_exponent(const Splat2D& s, float dx, float dy) {
    const float t1 = __fmaf_rn(s.A, dx, __fmul_rn(s.B, dy));
    const float t2 = __fmul_rn(__fmul_rn(s.C, dy), dy);
    return __fmaf_rn(dx, t1, t2);
}

__global__ void __launch_bounds__(kBlock) render_fwd_kernel(RenderFwdArgs a) {
    __shared__ float4 s_g0[kBlock];
    __shared__ float4 s_g1[kBlock];
    __shared__ float s_b[kBlock];
    const int tile = blockIdx.x;
    const int tid = threadIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int px = tx * kTile + (tid & (kTile - 1)), py = ty * kTile + (tid >> 4);
    const bool inside = px < a.W && py < a.H;
    const float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;
    uint32_t start = a.ranges[tile], end = a.ranges[tile + 1];
    if (a.counters[GES_CTR_OVERFLOW]) start = end = 0;
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;
    uint32_t last = 0, n_eval = end - start;
    for (uint32_t b0 = start; b0 < end; b0 += kBlock) {
        if (__syncthreads_count(done) == kBlock) break;
        const uint32_t k = b0 + tid;
        if (k < end) {
            const Splat2D s = load_splat(a.pay0, a.pay1, a.pay2, __ldg(a.list + k));
            s_g0[tid] = make_float4(s.u, s.v, s.A, s.B);
            s_g1[tid] = make_float4(s.C, s.kappa, s.r, s.g);
            s_b[tid] = s.b;
        }
        __syncthreads();
        if (!done) {
            const int n = (int)min((uint32_t)kBlock, end - b0);
            for (int j = 0; j < n; ++j) {
                const float4 g0 = s_g0[j];
                const float4 g1 = s_g1[j];
                Splat2D s;
                s.u = g0.x; s.v = g0.y; s.A = g0.z; s.B = g0.w; s.C = g1.x;
                const float dx = __fsub_rn(s.u, fpx), dy = __fsub_rn(s.v, fpy);
                const float p2 = fminf(raw_exponent(s, dx, dy), 0.0f);
                const float alpha = fminf(kAlphaMax, __fmul_rn(g1.y, fast_exp2(p2)));
                if (alpha < kAlphaMin) continue;
                const float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                if (Tn < kTMin) {
                    done = true;
                    n_eval = b0 - start + j + 1;
                    break;
                }
                const float w = __fmul_rn(alpha, T);
                cr = __fmaf_rn(g1.z, w, cr);
                cg = __fmaf_rn(g1.w, w, cg);
                cb = __fmaf_rn(s_b[j], w, cb);
                T = Tn;
                last = b0 - start + j + 1;
            }
        }
    }
    if (inside) {
        const int pix = py * a.W + px;
        const int plane = a.W * a.H;
        a.image[pix] = __fmaf_rn(T, a.bg[0], cr);
        a.image[plane + pix] = __fmaf_rn(T, a.bg[1], cg);
        a.image[2 * plane + pix] = __fmaf_rn(T, a.bg[2], cb);
        a.final_T[pix] = T;
        a.n_contrib[pix] = last;
        if (a.n_eval) a.n_eval[pix] = n_eval;
    }
}

cudaError_t launch_render_fwd(const RenderFwdArgs& a, cudaStream_t stream) {
    render_fwd_kernel<<<a.tiles_x * a.tiles_y, kBlock, 0, stream>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// S5a backward
// ---------------------------------------------------------------------------
// Recursive-halving warp reduction of 9 (padded to 16) values.  On return
// lane L holds the warp sum of component (L >> 1) (valid for L>>1 < 9, even L).
__device__ __forceinline__ float warp_reduce9(float v[16]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int step = 0; step < 4; ++step) {
        const int o = 16 >> step;      // 16, 8, 4, 2
        const int half = 8 >> step;    // 8, 4, 2, 1
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = upper ? v[i] : v[i + half];
            const float keep = upper ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__global__ void __launch_bounds__(kBlock) render_bwd_kernel(RenderBwdArgs a) {
    __shared__ float4 s_g0[kBlock];
    __shared__ float4 s_g1[kBlock];
    __shared__ float s_b[kBlock];
    __shared__ uint32_t s_pid[kBlock];
    __shared__ float s_acc[9][kBlock];
    __shared__ uint32_t s_max;
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int px = tx * kTile + (tid & (kTile - 1)), py = ty * kTile + (tid >> 4);
    const bool inside = px < a.W && py < a.H;
    const float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;
    uint32_t start = a.ranges[tile], end = a.ranges[tile + 1];
    if (a.counters[GES_CTR_OVERFLOW]) start = end = 0;
    const int pix = py * a.W + px;
    const int plane = a.W * a.H;
    float T = 1.0f, gr = 0.0f, gg = 0.0f, gb = 0.0f, Tfin = 1.0f;
    uint32_t last = 0;
    if (inside) {
        Tfin = a.final_T[pix];
        T = Tfin;
        last = a.n_contrib[pix];
        gr = a.dL_dimage[pix];
        gg = a.dL_dimage[plane + pix];
        gb = a.dL_dimage[2 * plane + pix];
    }
    if (tid == 0) s_max = 0;
    for (int c = 0; c < 9; ++c) s_acc[c][tid] = 0.0f;
    __syncthreads();
    if (last) atomicMax(&s_max, last);
    __syncthreads();
    const uint32_t max_last = s_max;
    const float gbg = gr * a.bg[0] + gg * a.bg[1] + gb * a.bg[2];
    const float bg_term = Tfin * gbg;
    float suffix = 0.0f;  // sum_{j > k} (rgb_j . g) alpha_j T_j
    for (int32_t b_end = (int32_t)max_last; b_end > 0; b_end -= kBlock) {
        const int32_t b_begin = max(0, b_end - kBlock);
        const int n = b_end - b_begin;
        if (tid < n) {
            const uint32_t p = __ldg(a.list + start + b_begin + tid);
            const Splat2D s = load_splat(a.pay0, a.pay1, a.pay2, p);
            s_g0[tid] = make_float4(s.u, s.v, s.A, s.B);
            s_g1[tid] = make_float4(s.C, s.kappa, s.r, s.g);
            s_b[tid] = s.b;
            s_pid[tid] = p;
        }
        __syncthreads();
        for (int j = n - 1; j >= 0; --j) {
            const uint32_t pos = (uint32_t)(b_begin + j);
            float v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = 0.0f;
            bool contrib = false;
            if (pos < last) {
                const float4 g0 = s_g0[j];
                const float4 g1 = s_g1[j];
                Splat2D s;
                s.u = g0.x; s.v = g0.y; s.A = g0.z; s.B = g0.w; s.C = g1.x;
                const float dx = __fsub_rn(s.u, fpx), dy = __fsub_rn(s.v, fpy);
                const float p2raw = raw_exponent(s, dx, dy);
                const float p2 = fminf(p2raw, 0.0f);
                const float G = fast_exp2(p2);
                const float araw = __fmul_rn(g1.y, G);
                const float alpha = fminf(kAlphaMax, araw);
                if (alpha >= kAlphaMin) {
                    contrib = true;
                    const float om = __fsub_rn(1.0f, alpha);
                    const float inv_om = 1.0f / om;
                    const float Tk = T * inv_om;  // transmittance before entry k
                    const float rb = s_b[j];
                    const float cgk = g1.z * gr + g1.w * gg + rb * gb;
                    const float dalpha = Tk * cgk - (suffix + bg_term) * inv_om;
                    suffix += cgk * alpha * Tk;
                    const float w = alpha * Tk;
                    v[6] = w * gr;
                    v[7] = w * gg;
                    v[8] = w * gb;
                    if (araw < kAlphaMax) {
                        v[5] = G * dalpha;
                        // dL/dp2 with G = 2^p2: alpha = kappa 2^p2 -> d alpha / d p2 = alpha ln 2
                        const float dp2 = (p2raw <= 0.0f) ? araw * dalpha * 0.69314718055994531f : 0.0f;
                        v[0] = dp2 * (2.0f * s.A * dx + s.B * dy);   // d p2 / d u
                        v[1] = dp2 * (s.B * dx + 2.0f * s.C * dy);   // d p2 / d v
                        v[2] = dp2 * dx * dx;                        // d p2 / d A
                        v[3] = dp2 * dx * dy;                        // d p2 / d B
                        v[4] = dp2 * dy * dy;                        // d p2 / d C
                    }
                    T = Tk;
                }
            }
            if (__any_sync(0xffffffffu, contrib)) {
                const float r = warp_reduce9(v);
                const int c = lane >> 1;
                if (!(lane & 1) && c < 9) atomicAdd(&s_acc[c][j], r);
            }
        }
        __syncthreads();
        if (tid < n) {
            const uint32_t p = s_pid[tid];
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                const float x = s_acc[c][tid];
                if (x != 0.0f) atomicAdd(a.grad2d + (size_t)c * a.P + p, x);
                s_acc[c][tid] = 0.0f;
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_render_bwd(const RenderBwdArgs& a, cudaStream_t stream) {
    render_bwd_kernel<<<a.tiles_x * a.tiles_y, kBlock, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
