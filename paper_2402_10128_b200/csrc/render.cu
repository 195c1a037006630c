// render.cu -- S4 and S5a: per-16x16-tile front-to-back
// alpha compositing (Eq. 3, discretised as
// C = sum_i c_i alpha_i prod_{j<i} (1 - alpha_j) + T_final * bg) and its
// adjoint.  Inherited rules (R7, R12): alpha = min(0.99, kappa G),
// entries with alpha < 1/255 skipped, a pixel stops -- without compositing --
// at the first entry that would take T below 1e-4.  The per-pixel kernel is
// the Gaussian of the phi-bar-scaled covariance (the paper's approximate
// rasterization "without taking the beta exponent"; R6).
//
// One CTA per tile, PPT pixels per thread (2 forward, 4 backward); warp w owns
// the 8 x (4 PPT)-pixel region (x0 = 8 (w & 1), y0 = 4 PPT (w >> 1)) of the tile.
// Each batch of kBatchFwd (128, S4) / kBatch (256, S5a) list entries is gathered once into shared memory
// (its list ids prefetched one batch early by cp.async); while gathering, each
// thread tests its entry against the warp regions with an exact lower bound of the
// Mahalanobis form over the region (the minimum of a positive-definite
// quadratic over a box) and marks the regions where alpha >= 1/255 is
// possible.  Each warp then walks only its own compacted entry list.  The
// test is conservative (a margin of 0.01 in log2 units), so culled entries are
// exactly the ones every pixel of the region would skip: results are
// identical to the unculled loop.  __syncthreads_count retires the tile once
// all pixels have terminated.  The backward walks the same lists back to
// front from the last composited entry of each warp and reduces the per-pair
// gradient moments across the warp with a column-aware recursive-halving
// shuffle (9 SHFL per warp and entry, grad_reduce), then nine lanes add them
// (red.global.add.f32) into the particle's 12-float raw-moment record.
#include <cstddef>
#include <cstdlib>
#include <type_traits>

#include "ges_internal.h"

namespace ges {

#ifdef GES_TILE_CLOCK
// Debug (GES_TILE_CLOCK builds only): per tile, the first warp start and the last warp
// end (%globaltimer ns) and the SM of the forward [0] and backward [1] kernels.
__device__ unsigned long long g_tile_clk[2][16384][3];
// and an optional launch order (block -> tile) per kernel, to measure schedules
__device__ int g_tile_order[2][16384];
__device__ int g_tile_order_on[2];
struct TileClock {
    unsigned long long* rec;
    __device__ TileClock(int which, int tile) {
        rec = g_tile_clk[which][tile & 16383];
        unsigned long long t, sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(*(unsigned*)&sm));
        if ((threadIdx.x & 31) == 0) { atomicMin(rec, t); rec[2] = sm & 0xffffffffull; }
    }
    __device__ ~TileClock() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if ((threadIdx.x & 31) == 0) atomicMax(rec + 1, t);
    }
};
#define GES_CLOCK(which, tile) TileClock tile_clock_(which, tile)
#define GES_TILE(which) (g_tile_order_on[which] ? g_tile_order[which][blockIdx.x] : (int)blockIdx.x)
#else
#define GES_CLOCK(which, tile)
#define GES_TILE(which) ((int)blockIdx.x)
#endif

#ifndef GES_BATCH
#define GES_BATCH 256
#endif
constexpr int kBatch = GES_BATCH;  // list entries staged per barrier (S5a)
#ifndef GES_BATCH_FWD
#define GES_BATCH_FWD 128
#endif
constexpr int kBatchFwd = GES_BATCH_FWD;  // (S4)
// tuning knobs: min resident CTAs per SM (register cap); unset = ptxas's choice
// forward: 9 resident CTAs per SM (PPT 2: 128 threads, a 56-register cap met
// without spills) measured 2 % faster than ptxas's own 64 registers
#ifndef GES_RFWD_MINB
#define GES_RFWD_MINB 9
#endif
#define GES_RFWD_LB(t) __launch_bounds__(t, GES_RFWD_MINB)
// backward: 9 resident 64-thread CTAs per SM (PPT 4; a 113-register cap, which
// ptxas meets at 91 without spills) measured 2 % faster than ptxas's own 121
#ifdef GES_RBWD_MINB
#define GES_RBWD_LB(t, ppt) __launch_bounds__(t, GES_RBWD_MINB)
#else
#define GES_RBWD_LB(t, ppt) __launch_bounds__(t, (ppt) == 4 ? 9 : 1)
#endif
constexpr float kCullMargin = 0.01f;      // log2 units (0.7% in alpha)
#ifdef GES_BWD_HALF
constexpr bool kBwdHalf = true;
#else
constexpr bool kBwdHalf = false;
#endif

struct Splat {
    float u, v, A, B, C, kappa, r, g, b;
};

__device__ __forceinline__ Splat load_splat(const float4* pay0, const float4* pay1, const float* pay2, uint32_t p) {
    const float4 a = __ldg(pay0 + p);
    const float4 b = __ldg(pay1 + p);
    Splat s;
    s.u = a.x; s.v = a.y;
    s.A = __fmul_rn(__fmul_rn(-0.5f, a.z), kLog2e);
    s.B = __fmul_rn(-a.w, kLog2e);
    s.C = __fmul_rn(__fmul_rn(-0.5f, b.x), kLog2e);
    s.kappa = b.y; s.r = b.z; s.g = b.w;
    s.b = __ldg(pay2 + p);
    return s;
}

// p2 = A dx^2 + B dx dy + C dy^2 (log2 units) as c0 + dy (c1 + C dy) with the
// per-(entry, thread) constants c0 = A dx^2, c1 = B dx (a thread's pixels share
// their column, so dx): two FMAs per pixel.  Fixed op order: the forward and
// the backward evaluate exactly this sequence, so their decisions agree.
struct ExpCol {
    float c0, c1;
};
__device__ __forceinline__ ExpCol exp_col(float A, float B, float dx) {
    return ExpCol{__fmul_rn(__fmul_rn(A, dx), dx), __fmul_rn(B, dx)};
}
__device__ __forceinline__ float raw_exponent(ExpCol e, float C, float dy) {
    return __fmaf_rn(dy, __fmaf_rn(C, dy, e.c1), e.c0);
}

// 1 / x for x in [0.01, 1] (x = 1 - alpha): one MUFU.RCP, no range fix-up.
__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Two fp32 values in one 64-bit register pair, for the packed sm_100 instructions
// (FADD2 / FMUL2 / FFMA2: one issue slot for two IEEE round-to-nearest operations, each
// lane's result identical to the scalar instruction's).  A scalar operand broadcast with
// f2_bc costs nothing: ptxas folds it into the instruction's .F32 operand form.
typedef unsigned long long f2;
#if !defined(GES_F32X2) && !defined(GES_NO_F32X2)
#define GES_F32X2 1  // S5a's Gaussian entry loop on pixel pairs (GES_NO_F32X2: scalar)
#endif
#ifdef GES_F32X2
constexpr bool kF32x2 = true;
#else
constexpr bool kF32x2 = false;
#endif
__device__ __forceinline__ f2 f2_pk(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2 f2_bc(float a) { return f2_pk(a, a); }
__device__ __forceinline__ float f2_lo(f2 r) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return a;
}
__device__ __forceinline__ float f2_hi(f2 r) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return b;
}
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_sub(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_fma(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Minimum of Q = a x^2 + b x y + c y^2 (a, c > 0, 4ac > b^2) over the box
// [x0, x1] x [y0, y1]: 0 if the box holds the origin, else on an edge.
__device__ __forceinline__ float box_min_quadratic(float a, float b, float c, float ia2, float ic2, float x0, float x1,
                                                   float y0, float y1) {
    if (x0 <= 0.0f && x1 >= 0.0f && y0 <= 0.0f && y1 >= 0.0f) return 0.0f;
    float m = 3.0e38f;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const float X = e ? x1 : x0;
        const float y = fminf(fmaxf(-b * X * ic2, y0), y1);
        m = fminf(m, (a * X + b * y) * X + c * y * y);
        const float Y = e ? y1 : y0;
        const float x = fminf(fmaxf(-b * Y * ia2, x0), x1);
        m = fminf(m, (a * x + b * Y) * x + c * Y * Y);
    }
    return m;
}

// Thread/pixel layout: PPT pixels per thread; warp w owns the 8 x (4 PPT)
// region (x0 = 8 (w & 1), y0 = 4 PPT (w >> 1)) of the 16x16 tile; lane l
// holds pixels (x0 + (l & 7), y0 + (l >> 3) + 4k), k < PPT.
template <int PPT>
struct Layout {
    static constexpr int kThreads = kBlock / PPT;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kRegionH = 4 * PPT;
};

// Bit w set if some pixel of warp region w may get alpha >= 1/255 from s.
// The bound on -p2 (log2 units): Gaussian kernel log2(255 kappa); exact GEF
// kernel (hb = beta/2) 1/2 log2e Qc with Qc = (2 ln(255 kappa))^(1/hb), here
// from fast intrinsics with a 2 % relative margin on top of the additive one.
template <int PPT, bool EXACT>
__device__ __forceinline__ uint32_t region_mask(const Splat& s, float hb, int tile_x0, int tile_y0) {
    using Lt = Layout<PPT>;
    const float k255 = s.kappa * 255.0f;
    if (!(k255 > 1.0f)) return 0u;
    float thr = __log2f(k255) + kCullMargin;  // cull if min(-p2) > thr
    if (EXACT) {
        const float lq = __log2f(2.0f * __logf(k255)) * __fdividef(1.0f, hb);  // log2 Qc
        thr = 0.5f * kLog2e * exp2f(lq) * 1.02f + kCullMargin;
    }
    const float a = -s.A, b = -s.B, c = -s.C;
    const float ia2 = 0.5f / a, ic2 = 0.5f / c;
    uint32_t mask = 0;
#pragma unroll
    for (int w = 0; w < Lt::kWarps; ++w) {
        const float rx = (float)(tile_x0 + 8 * (w & 1)), ry = (float)(tile_y0 + Lt::kRegionH * (w >> 1));
        const float x0 = s.u - (rx + 7.5f), x1 = s.u - (rx + 0.5f);
        const float y0 = s.v - (ry + (float)Lt::kRegionH - 0.5f), y1 = s.v - (ry + 0.5f);
        if (box_min_quadratic(a, b, c, ia2, ic2, x0, x1, y0, y1) <= thr) mask |= 1u << w;
    }
    return mask;
}

// The exact GEF kernel (Eq. 2) from the log2-scaled Gaussian exponent p2 =
// -1/2 log2e Q:  Q = 2 ln2 qp (qp = -p2), log2 Q = log2 qp + kC0,
// Q^hb = 2^(hb log2 Q), G = exp(-1/2 Q^hb) = 2^(kC1 Q^hb).  qp is floored at
// 1e-30 so that log2 and Q^(hb-1) stay finite at a pixel on the mean.
constexpr float kGefC0 = 0.47123362f;    // log2(2 ln 2)
constexpr float kGefC1 = -0.72134752f;   // -1/2 log2 e
__device__ __forceinline__ float fast_log2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
struct Gef {
    float G, Qb, L, qp;  // G, Q^hb, log2 Q, -p2
};
__device__ __forceinline__ Gef gef_eval(float p2, float hb) {
    Gef r;
    r.qp = fmaxf(-p2, 1e-30f);
    r.L = fast_log2(r.qp) + kGefC0;
    r.Qb = fast_exp2(hb * r.L);
    r.G = fast_exp2(kGefC1 * r.Qb);
    return r;
}

// Shared-memory loads from 32-bit shared-window addresses computed once per
// CTA (the compiler otherwise rebuilds each array's address from the CTA id in
// every iteration of the entry loops).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int OFF>
__device__ __forceinline__ float4 lds_f4_at(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ float lds_f_at(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ uint32_t lds_u32_at(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
    return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_f(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Per-warp compaction of the batch entries whose mask has this warp's bit.
template <int NB = kBatch>
__device__ __forceinline__ int compact_warp_list(const uint8_t* s_mask, int n, int warp, uint16_t* out) {
    const int lane = threadIdx.x & 31;
    int cnt = 0;
#ifdef GES_COMPACT_BOUNDED
#pragma unroll 4
    for (int c = 0; c < (n + 31) / 32; ++c) {
#else
#pragma unroll
    for (int c = 0; c < NB / 32; ++c) {
#endif
        const int j = c * 32 + lane;
        const bool bit = j < n && ((s_mask[j] >> warp) & 1u);
        const uint32_t ball = __ballot_sync(0xffffffffu, bit);
        if (bit) out[cnt + __popc(ball & ((1u << lane) - 1u))] = (uint16_t)j;
        cnt += __popc(ball);
    }
    __syncwarp();
    return cnt;
}

// Band tile t = k tiles_x + tx is image tile (tx, band_begin + k band_step).
__device__ __forceinline__ void tile_origin(int tile, int tiles_x, int band_begin, int band_step, int& x0, int& y0) {
    x0 = (tile % tiles_x) * kTile;
    y0 = (band_begin + (tile / tiles_x) * band_step) * kTile;
}

// Bucket of a backward tile cost on a log scale, 4 buckets per octave (exact below 4),
// saturating at kTileBuckets - 1.
__device__ __forceinline__ uint32_t cost_bucket(uint32_t c) {
    if (c < 4u) return c;
    const int e = 31 - __clz(c);
    return min((uint32_t)(kTileBuckets - 1), 4u * (uint32_t)(e - 1) + ((c >> (e - 2)) & 3u));
}

// S5a: tile number b (of T) in descending cost order (the forward's buckets), or b itself
// when the buckets do not hold exactly T tiles.  Every warp computes it.
__device__ __forceinline__ int ordered_tile(const uint32_t* bucket, const uint32_t* order, uint32_t b, uint32_t T) {
    static_assert(kTileBuckets == 64, "two buckets per lane");
    const int lane = threadIdx.x & 31;
    // lane l holds buckets 63 - l (first half) and 31 - l (second half): descending cost
    const uint32_t c0 = bucket[63 - lane], c1 = bucket[31 - lane];
    uint32_t i0 = c0, i1 = c1;  // inclusive scans of each half
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t x0 = __shfl_up_sync(0xffffffffu, i0, d), x1 = __shfl_up_sync(0xffffffffu, i1, d);
        if (lane >= d) { i0 += x0; i1 += x1; }
    }
    const uint32_t h0 = __shfl_sync(0xffffffffu, i0, 31);
    if (h0 + __shfl_sync(0xffffffffu, i1, 31) != T) return (int)b;
    const unsigned m0 = __ballot_sync(0xffffffffu, i0 > b);
    int q;
    uint32_t excl;
    if (m0) {
        q = __ffs(m0) - 1;
        excl = __shfl_sync(0xffffffffu, i0 - c0, q);
        return (int)__ldg(order + (size_t)(63 - q) * T + (b - excl));
    }
    const unsigned m1 = __ballot_sync(0xffffffffu, h0 + i1 > b);
    q = __ffs(m1) - 1;
    excl = h0 + __shfl_sync(0xffffffffu, i1 - c1, q);
    return (int)__ldg(order + (size_t)(31 - q) * T + (b - excl));
}

template <int PPT>
__device__ __forceinline__ void pixel_base(int tile_x0, int tile_y0, int tid, int& px, int& py0) {
    const int warp = tid >> 5, lane = tid & 31;
    px = tile_x0 + 8 * (warp & 1) + (lane & 7);
    py0 = tile_y0 + Layout<PPT>::kRegionH * (warp >> 1) + (lane >> 3);
}

struct StagedBatch {
    float4* g0;  // u, v, A, B
    float4* g1;  // C, kappa, r, g
    float* b;
    uint32_t* pid;
    uint8_t* mask;
    float* hb;   // beta / 2 (exact kernel)
};

// The list ids of a batch arrive in shared memory ahead of time (cp.async, one
// batch early): staging then waits for the payload gathers only, not for the
// id load that addresses them.
__device__ __forceinline__ void prefetch_ids(uint32_t* dst, const uint32_t* list, uint32_t first, int n) {
    for (int q = threadIdx.x; q < n; q += blockDim.x)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst + q)), "l"(list + first + q)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void wait_ids() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int PPT, bool EXACT, int NT = Layout<PPT>::kThreads, int NB = kBatch>
__device__ __forceinline__ void stage_batch(const float4* pay0, const float4* pay1, const float* pay2,
                                            const float* pay3, const uint32_t* ids, int n,
                                            int tile_x0, int tile_y0, StagedBatch sb) {
    static_assert(NB % NT == 0 && NB % 32 == 0, "a batch is whole rounds of the CTA's threads");
#pragma unroll
    for (int h = 0; h < NB / NT; ++h) {
        const int q = threadIdx.x + h * NT;
        if (q < n) {
            const uint32_t p = ids[q];
            const Splat s = load_splat(pay0, pay1, pay2, p);
            sb.g0[q] = make_float4(s.u, s.v, s.A, s.B);
            sb.g1[q] = make_float4(s.C, s.kappa, s.r, s.g);
            sb.b[q] = s.b;
            if (sb.pid) sb.pid[q] = p;
            const float hb = EXACT ? __ldg(pay3 + p) : 1.0f;
            if (EXACT) sb.hb[q] = hb;
            sb.mask[q] = (uint8_t)region_mask<PPT, EXACT>(s, hb, tile_x0, tile_y0);
        }
    }
}

// One shared-memory block per CTA: the staged batch at compile-time offsets, so
// an entry's fields are one base register + an immediate (ld.shared [r+imm]).
template <int PPT, bool EXACT, int NB = kBatch>
struct RenderSmem {
    float4 g0[NB];  // u, v, A, B
    float4 g1[NB];  // C, kappa, r, g
    float b[NB];
    uint32_t pid[NB];
    float hb[EXACT ? NB : 1];
    uint16_t list[Layout<PPT>::kWarps][NB];
    uint32_t ids[2][NB];  // list ids of this and the next batch
    uint8_t mask[NB];
    uint32_t max;
    uint32_t wmax[Layout<PPT>::kWarps];  // forward: each warp's largest n_contrib (tile cost)
    static constexpr int kG1 = NB * 16, kB = NB * 32, kPid = NB * 36, kHb = NB * 40;
};

template <int PPT, bool DIAG, bool EXACT>
__global__ void GES_RFWD_LB(Layout<PPT>::kThreads) render_fwd_kernel(RenderFwdArgs a) {
    using Lt = Layout<PPT>;
    using Sm = RenderSmem<PPT, EXACT, kBatchFwd>;
    __shared__ Sm S;
    static_assert(offsetof(Sm, g1) == Sm::kG1 && offsetof(Sm, b) == Sm::kB && offsetof(Sm, pid) == Sm::kPid &&
                  offsetof(Sm, hb) == Sm::kHb, "smem layout");
    const int tile = GES_TILE(0);
    GES_CLOCK(0, tile);
    const int tid = threadIdx.x, warp = tid >> 5;
    int px, py0;
    int tile_x0, tile_y0;
    tile_origin(tile, a.tiles_x, a.band_begin, a.band_step, tile_x0, tile_y0);
    pixel_base<PPT>(tile_x0, tile_y0, tid, px, py0);
    const float fpx = (float)px + 0.5f;
    uint32_t start = a.ranges[tile], end = a.ranges[tile + 1];
    if (a.counters[GES_CTR_OVERFLOW]) start = end = 0;
    // per pixel: T, colour, last composited position; thr = the alpha skip
    // threshold, 2 (never reached) once the pixel has stopped or lies outside
    float T[PPT], cr[PPT], cg[PPT], cb[PPT], thr[PPT];
    uint32_t last[PPT], n_eval[PPT], n_comp[PPT];
    uint32_t done = 0;  // bit k: pixel k finished (or outside the image)
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        T[k] = 1.0f; cr[k] = cg[k] = cb[k] = 0.0f; last[k] = 0; n_eval[k] = end - start; n_comp[k] = 0;
        thr[k] = kAlphaMin;
        if (!(px < a.W && py0 + 4 * k < a.H)) { done |= 1u << k; thr[k] = 2.0f; }
    }
    constexpr uint32_t kAll = (1u << PPT) - 1u;
    // the plain Gaussian instance runs a thread's two pixels as one register pair with the
    // packed FP32 instructions (same per-lane results: the image is bit-identical)
    constexpr bool kPk = kF32x2 && !EXACT && !DIAG && PPT == 2;
    f2 Tp = f2_pk(T[0], T[PPT - 1]), crp = 0ull, cgp = 0ull, cbp = 0ull;
    const f2 pyp = f2_pk((float)py0 + 0.5f, (float)(py0 + 4) + 0.5f);
    StagedBatch sb{S.g0, S.g1, S.b, nullptr, S.mask, S.hb};
    uint32_t sbase = smem_addr(&S);
    uint32_t a_list = smem_addr(S.list[warp]);
    // opaque: kept in registers instead of rebuilt from the CTA's shared window
    // (S2UR SR_CgaCtaId + ULEA) in every iteration of the entry loop
    asm volatile("" : "+r"(sbase), "+r"(a_list));
    if (start < end) prefetch_ids(S.ids[0], a.list, start, (int)min((uint32_t)kBatchFwd, end - start));
    int buf = 0;
    for (uint32_t b0 = start; b0 < end; b0 += kBatchFwd, buf ^= 1) {
        wait_ids();
        if (__syncthreads_count(done == kAll) == Lt::kThreads) break;
        const int n = (int)min((uint32_t)kBatchFwd, end - b0);
        if (b0 + kBatchFwd < end) prefetch_ids(S.ids[buf ^ 1], a.list, b0 + kBatchFwd, (int)min((uint32_t)kBatchFwd, end - b0 - kBatchFwd));
        stage_batch<PPT, EXACT, Lt::kThreads, kBatchFwd>(a.pay0, a.pay1, a.pay2, a.pay3, S.ids[buf], n, tile_x0, tile_y0, sb);
        __syncthreads();
        if (__all_sync(0xffffffffu, done == kAll)) continue;  // the barrier above retires the tile
        const int nw = compact_warp_list<kBatchFwd>(S.mask, n, warp, S.list[warp]);
        for (int i = 0; i < nw; ++i) {
            const int j = (int)lds_u16(a_list + 2u * (uint32_t)i);
            const uint32_t r16 = sbase + 16u * (uint32_t)j, r4 = sbase + 4u * (uint32_t)j;
            const float4 g0 = lds_f4_at<0>(r16);
            const float4 g1 = lds_f4_at<Sm::kG1>(r16);
            const float gbl = lds_f_at<Sm::kB>(r4);
            const float hb = EXACT ? lds_f_at<Sm::kHb>(r4) : 1.0f;
            const float dx = __fsub_rn(g0.x, fpx);
            const ExpCol ec = exp_col(g0.z, g0.w, dx);
            const uint32_t pos1 = b0 - start + j + 1;
            // per-pixel kernel value: Gaussian 2^p2, or Eq. 2's exp(-1/2 Q^(beta/2))
            auto kern = [&](float dy) {
                const float p2 = raw_exponent(ec, g1.x, dy);
                if constexpr (EXACT) return gef_eval(p2, hb).G;
                else return fast_exp2(p2);
            };
            const bool clampk = g1.y > kAlphaMax;  // warp-uniform: only then can alpha reach 0.99
            // alpha' = alpha if alpha >= thr (the skip test; thr = 2 for stopped pixels), else 0;
            // the would-be transmittance T (1 - alpha') decides the stop.  (The exponent is not
            // clamped at 0: the form is >= 0 up to rounding, G exceeds 1 by <= 2^-22 -- R19b.)
            float al[PPT], w[PPT], Tn[PPT];
            float tmin = 1.0f;
            if constexpr (kPk) {
                const f2 dy = f2_sub(f2_bc(g0.y), pyp);
                const f2 p2 = f2_fma(dy, f2_fma(f2_bc(g1.x), dy, f2_bc(ec.c1)), f2_bc(ec.c0));
                const f2 araw = f2_mul(f2_bc(g1.y), f2_pk(fast_exp2(f2_lo(p2)), fast_exp2(f2_hi(p2))));
                float a0 = f2_lo(araw), a1 = f2_hi(araw);
                if (clampk) { a0 = fminf(kAlphaMax, a0); a1 = fminf(kAlphaMax, a1); }
                al[0] = a0 >= thr[0] ? a0 : 0.0f;
                al[1] = a1 >= thr[1] ? a1 : 0.0f;
                const f2 wp = f2_mul(f2_pk(al[0], al[1]), Tp);
                const f2 Tnp = f2_sub(Tp, wp);
                tmin = fminf(tmin, fminf(f2_lo(Tnp), f2_hi(Tnp)));
                if (!__any_sync(0xffffffffu, tmin < kTMin)) {
                    crp = f2_fma(f2_bc(g1.z), wp, crp);
                    cgp = f2_fma(f2_bc(g1.w), wp, cgp);
                    cbp = f2_fma(f2_bc(gbl), wp, cbp);
#pragma unroll
                    for (int k = 0; k < PPT; ++k) last[k] = al[k] > 0.0f ? pos1 : last[k];
                    Tp = Tnp;
                } else {
                    const bool st0 = f2_lo(Tnp) < kTMin, st1 = f2_hi(Tnp) < kTMin;
                    const f2 wk = f2_pk(st0 ? 0.0f : f2_lo(wp), st1 ? 0.0f : f2_hi(wp));
                    crp = f2_fma(f2_bc(g1.z), wk, crp);
                    cgp = f2_fma(f2_bc(g1.w), wk, cgp);
                    cbp = f2_fma(f2_bc(gbl), wk, cbp);
                    last[0] = (!st0 && al[0] > 0.0f) ? pos1 : last[0];
                    last[1] = (!st1 && al[1] > 0.0f) ? pos1 : last[1];
                    Tp = f2_pk(st0 ? f2_lo(Tp) : f2_lo(Tnp), st1 ? f2_hi(Tp) : f2_hi(Tnp));
                    thr[0] = st0 ? 2.0f : thr[0];
                    thr[1] = st1 ? 2.0f : thr[1];
                    done |= (st0 ? 1u : 0u) | (st1 ? 2u : 0u);
                    if (__all_sync(0xffffffffu, done == kAll)) break;  // done changes only here
                }
                continue;
            }
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const float dy = __fsub_rn(g0.y, (float)(py0 + 4 * k) + 0.5f);
                float alpha = __fmul_rn(g1.y, kern(dy));
                if (clampk) alpha = fminf(kAlphaMax, alpha);
                al[k] = alpha >= thr[k] ? alpha : 0.0f;
                w[k] = __fmul_rn(al[k], T[k]);
                Tn[k] = __fsub_rn(T[k], w[k]);
                tmin = fminf(tmin, Tn[k]);
            }
            if (!__any_sync(0xffffffffu, tmin < kTMin)) {
                // common case: no pixel of the warp stops at this entry
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    cr[k] = __fmaf_rn(g1.z, w[k], cr[k]);
                    cg[k] = __fmaf_rn(g1.w, w[k], cg[k]);
                    cb[k] = __fmaf_rn(gbl, w[k], cb[k]);
                    if (DIAG) n_comp[k] += al[k] > 0.0f ? 1u : 0u;
                    last[k] = al[k] > 0.0f ? pos1 : last[k];
                    T[k] = Tn[k];
                }
            } else {
                // some pixel stops: it composites nothing more (R12)
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const bool stop = Tn[k] < kTMin;  // implies alpha' > 0 (T >= 1e-4 before)
                    const float wk = stop ? 0.0f : w[k];
                    cr[k] = __fmaf_rn(g1.z, wk, cr[k]);
                    cg[k] = __fmaf_rn(g1.w, wk, cg[k]);
                    cb[k] = __fmaf_rn(gbl, wk, cb[k]);
                    const bool comp = !stop && al[k] > 0.0f;
                    if (DIAG) { n_comp[k] += comp ? 1u : 0u; n_eval[k] = stop ? pos1 : n_eval[k]; }
                    last[k] = comp ? pos1 : last[k];
                    T[k] = stop ? T[k] : Tn[k];
                    thr[k] = stop ? 2.0f : thr[k];
                    done |= (stop ? 1u : 0u) << k;
                }
                if (__all_sync(0xffffffffu, done == kAll)) break;  // done changes only here
            }
        }
    }
    wait_ids();  // no copy into shared memory outlives the CTA
    if constexpr (kPk) {
        T[0] = f2_lo(Tp); T[PPT - 1] = f2_hi(Tp);
        cr[0] = f2_lo(crp); cr[PPT - 1] = f2_hi(crp);
        cg[0] = f2_lo(cgp); cg[PPT - 1] = f2_hi(cgp);
        cb[0] = f2_lo(cbp); cb[PPT - 1] = f2_hi(cbp);
    }
    {
        // S5a's launch order (ges_frame.tile_order): a backward CTA lasts as long as its
        // longer walk, so the tile's cost is its largest n_contrib (measured against the
        // sum over the two backward warp regions and the list length: tools/tile_clock.py)
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < PPT; ++k) m = max(m, last[k]);
        m = __reduce_max_sync(0xffffffffu, m);
        if ((tid & 31) == 0) S.wmax[warp] = m;
        __syncthreads();
        if (tid == 0) {
            uint32_t c = 0u;
#pragma unroll
            for (int w = 0; w < Lt::kWarps; ++w) c = max(c, S.wmax[w]);
            const uint32_t b = cost_bucket(c);
            const uint32_t slot = atomicAdd(a.tile_bucket + b, 1u);
            a.tile_order[(size_t)b * gridDim.x + slot] = (uint32_t)tile;
        }
    }
    const int plane = a.W * a.H;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int py = py0 + 4 * k;
        if (px < a.W && py < a.H) {
            const int pix = py * a.W + px;
            a.image[pix] = __fmaf_rn(T[k], a.bg[0], cr[k]);
            a.image[plane + pix] = __fmaf_rn(T[k], a.bg[1], cg[k]);
            a.image[2 * plane + pix] = __fmaf_rn(T[k], a.bg[2], cb[k]);
            a.final_T[pix] = T[k];
            a.n_contrib[pix] = last[k];
            if (DIAG && a.n_eval) a.n_eval[pix] = n_eval[k];
            if (DIAG && a.n_comp) a.n_comp[pix] = n_comp[k];
        }
    }
}

// Pixels per thread (tuning knob; GES_PPT_FWD / GES_PPT_BWD = 2 or 4 override for experiments).
static int ppt_from_env(const char* name, int dflt) {
    const char* e = getenv(name);
    const int v = e ? atoi(e) : dflt;
    return (v == 2 || v == 4) ? v : dflt;
}

// Experiment knob: GES_CARVEOUT = preferred shared-memory carveout (percent) of the
// render kernels; unset = the driver's choice.
template <typename K>
static void apply_carveout(K kernel) {
    static const int pct = [] {
        const char* e = getenv("GES_CARVEOUT");
        return e ? atoi(e) : -1;
    }();
    if (pct >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

template <int PPT, bool EXACT>
static void launch_fwd_ppt(const RenderFwdArgs& a, int grid, bool diag, cudaStream_t stream) {
    apply_carveout(render_fwd_kernel<PPT, false, EXACT>);
    if (diag) render_fwd_kernel<PPT, true, EXACT><<<grid, Layout<PPT>::kThreads, 0, stream>>>(a);
    else render_fwd_kernel<PPT, false, EXACT><<<grid, Layout<PPT>::kThreads, 0, stream>>>(a);
}

cudaError_t launch_render_fwd(const RenderFwdArgs& a, cudaStream_t stream) {
    static const int ppt = ppt_from_env("GES_PPT_FWD", 2);
    const int grid = a.tiles_x * a.tiles_y;
    if (grid == 0) return cudaSuccess;  // a band without tile rows renders nothing
    const bool diag = a.n_eval || a.n_comp;  // the counters cost issue slots: only when asked
    if (a.exact) {
        if (ppt == 4) launch_fwd_ppt<4, true>(a, grid, diag, stream);
        else launch_fwd_ppt<2, true>(a, grid, diag, stream);
    } else {
        if (ppt == 4) launch_fwd_ppt<4, false>(a, grid, diag, stream);
        else launch_fwd_ppt<2, false>(a, grid, diag, stream);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// S5a backward
// ---------------------------------------------------------------------------
// Warp sum of the per-pair gradient terms.  Each lane holds its pixels' sums
// S0 = sum q, S1 = sum q dy, S2 = sum q dy^2 and the colour terms (exact
// kernel: + dk, Sb); the record wants sum q dx and sum q dx^2, sum q dx dy too.
// Lanes l, l^8, l^16, l^24 share a pixel column (dx), so the first two
// recursive-halving levels (xor 16, xor 8) sum the column's lanes, the column
// moments are formed once per column (dx S0, dx^2 S0, dx S1), and the last three
// levels (xor 4, 2, 1) sum the 8 columns:
//   xor 16: lo {S0, S1, S2, dk} | hi {db, dr, dg, Sb}        4 SHFL (Gaussian 3)
//   xor 8:  lo {., dk | db, Sb} | hi {S1, S2 | dr, dg}       2
//   groups (bit 16, bit 8): 00 {dk, dx S0, dx^2 S0}, 01 {S1, S2, dx S1},
//           10 {db, Sb}, 11 {dr, dg}   (Gaussian: dk = S0, no Sb)
//   xor 4: {slot 0, 1 | slot 2} 2, xor 2: 1, xor 1: 1  -> 10 SHFL (Gaussian 9)
// Afterwards lanes l and l^1 hold the full sum of record component
// record_component<EXACT>(l) (or -1: none).
template <bool EXACT>
__device__ __forceinline__ int record_component(int lane) {
    const int g = ((lane >> 3) & 3);           // bit 16 -> 2, bit 8 -> 1
    const int slot = ((lane & 4) ? 2 : 0) + ((lane & 2) ? 1 : 0);
    // record: 0 sum q dx, 1 sum q dy, 2 sum q dx^2, 3 sum q dx dy, 4 sum q dy^2,
    //         5 dL/dkappa, 6 dr, 7 dg, 8 db, 9 Sb
    constexpr int kMap[4][4] = {{5, 0, 2, -1}, {1, 4, 3, -1}, {8, EXACT ? 9 : -1, -1, -1}, {6, 7, -1, -1}};
    return kMap[g][slot];
}

template <bool EXACT>
__device__ __forceinline__ float grad_reduce(float S0, float S1, float S2, float dk, float Sb, float dr, float dg,
                                             float db, float dx) {
    const int lane = threadIdx.x & 31;
    const bool u16 = (lane & 16) != 0, u8 = (lane & 8) != 0, u4 = (lane & 4) != 0, u2 = (lane & 2) != 0;
    constexpr unsigned kAll = 0xffffffffu;
    const float a0 = (u16 ? db : S0) + __shfl_xor_sync(kAll, u16 ? S0 : db, 16);
    const float a1 = (u16 ? dr : S1) + __shfl_xor_sync(kAll, u16 ? S1 : dr, 16);
    const float a2 = (u16 ? dg : S2) + __shfl_xor_sync(kAll, u16 ? S2 : dg, 16);
    float a3 = 0.0f;
    if (EXACT) a3 = (u16 ? Sb : dk) + __shfl_xor_sync(kAll, u16 ? dk : Sb, 16);
    const float b0 = (u8 ? a1 : a0) + __shfl_xor_sync(kAll, u8 ? a0 : a1, 8);
    const float b1 = (u8 ? a2 : a3) + __shfl_xor_sync(kAll, u8 ? a3 : a2, 8);
    const bool g00 = !u16 && !u8, g01 = !u16 && u8;
    const float t = dx * b0;  // column moment dx S (S0 in group 00, S1 in 01)
    const float c0 = (EXACT && g00) ? b1 : b0;
    const float c1 = g00 ? t : b1;
    const float c2 = g00 ? dx * t : (g01 ? t : 0.0f);
    const float d0 = (u4 ? c2 : c0) + __shfl_xor_sync(kAll, u4 ? c0 : c2, 4);
    const float d1 = (u4 ? 0.0f : c1) + __shfl_xor_sync(kAll, u4 ? c1 : 0.0f, 4);
    float e = (u2 ? d1 : d0) + __shfl_xor_sync(kAll, u2 ? d0 : d1, 2);
    e += __shfl_xor_sync(kAll, e, 1);
    return e;
}

__device__ __forceinline__ void red_add(float* addr, float x) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(x) : "memory");
}

template <int PPT, bool EXACT>
__global__ void GES_RBWD_LB(kBwdHalf ? 32 : Layout<PPT>::kThreads, PPT) render_bwd_kernel(RenderBwdArgs a) {
    using Sm = RenderSmem<PPT, EXACT>;
    // kBwdHalf (experiment): one warp per CTA, CTA 2b + h walks warp region h of tile b
    constexpr int kNT = kBwdHalf ? 32 : Layout<PPT>::kThreads;
    __shared__ Sm S;
    const uint32_t b_ = kBwdHalf ? blockIdx.x >> 1 : blockIdx.x, T_ = kBwdHalf ? gridDim.x >> 1 : gridDim.x;
#ifdef GES_TILE_CLOCK
    const int tile = g_tile_order_on[1] ? GES_TILE(1) : (a.use_order ? ordered_tile(a.tile_bucket, a.tile_order, b_, T_) : (int)b_);
#else
    const int tile = a.use_order ? ordered_tile(a.tile_bucket, a.tile_order, b_, T_) : (int)b_;
#endif
    GES_CLOCK(1, tile);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int vw = kBwdHalf ? (int)(blockIdx.x & 1u) : warp;  // the warp region walked
    int px, py0;
    int tile_x0, tile_y0;
    tile_origin(tile, a.tiles_x, a.band_begin, a.band_step, tile_x0, tile_y0);
    pixel_base<PPT>(tile_x0, tile_y0, vw * 32 + lane, px, py0);
    const float fpx = (float)px + 0.5f;
    const bool ovf = a.counters[GES_CTR_OVERFLOW] != 0;
    const uint32_t start = ovf ? 0u : a.ranges[tile];
    const int plane = a.W * a.H;
    // U = T_final bg . g + sum over entries behind of c_j . g alpha_j T_j
    float T[PPT], gr[PPT], gg[PPT], gb[PPT], U[PPT], thr[PPT];
    uint32_t last[PPT];
    uint32_t my_max = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int py = py0 + 4 * k;
        T[k] = 1.0f; gr[k] = gg[k] = gb[k] = 0.0f; last[k] = 0;
        thr[k] = 2.0f;  // inactive until the walk passes below the pixel's last entry
        float Tfin = 1.0f;
        if (px < a.W && py < a.H && !ovf) {
            const int pix = py * a.W + px;
            Tfin = a.final_T[pix];
            last[k] = a.n_contrib[pix];
            gr[k] = a.dL_dimage[pix];
            gg[k] = a.dL_dimage[plane + pix];
            gb[k] = a.dL_dimage[2 * plane + pix];
        }
        T[k] = Tfin;
        U[k] = Tfin * (gr[k] * a.bg[0] + gg[k] * a.bg[1] + gb[k] * a.bg[2]);
        my_max = max(my_max, last[k]);
    }
#ifdef GES_F32X2
    // pixels 2h, 2h + 1 of the thread as register pairs (the Gaussian entry loop)
    f2 Tp[PPT / 2], Up[PPT / 2], grp[PPT / 2], ggp[PPT / 2], gbp[PPT / 2], pyp[PPT / 2];
#pragma unroll
    for (int h = 0; h < PPT / 2; ++h) {
        Tp[h] = f2_pk(T[2 * h], T[2 * h + 1]);
        Up[h] = f2_pk(U[2 * h], U[2 * h + 1]);
        grp[h] = f2_pk(gr[2 * h], gr[2 * h + 1]);
        ggp[h] = f2_pk(gg[2 * h], gg[2 * h + 1]);
        gbp[h] = f2_pk(gb[2 * h], gb[2 * h + 1]);
        pyp[h] = f2_pk((float)(py0 + 8 * h) + 0.5f, (float)(py0 + 8 * h + 4) + 0.5f);
    }
#endif
    if (tid == 0) S.max = 0;
    __syncthreads();
    const uint32_t warp_max = __reduce_max_sync(0xffffffffu, my_max);
    if (lane == 0 && warp_max) atomicMax(&S.max, warp_max);
    __syncthreads();
    const uint32_t max_last = S.max;
    // the largest `last` among the warp's inactive pixels: the walk (positions
    // descending) activates them when it passes below it
    uint32_t nxt = warp_max;
    const int red_comp = record_component<EXACT>(lane);
    StagedBatch sb{S.g0, S.g1, S.b, S.pid, S.mask, S.hb};
    uint32_t sbase = smem_addr(&S);
    uint32_t a_list = smem_addr(S.list[warp]);
    // opaque: kept in registers instead of rebuilt from the CTA's shared window
    // (S2UR SR_CgaCtaId + ULEA) in every iteration of the entry loop
    asm volatile("" : "+r"(sbase), "+r"(a_list));
    if (max_last > 0) {
        const int32_t b0 = max(0, (int32_t)max_last - kBatch);
        prefetch_ids(S.ids[0], a.list, start + (uint32_t)b0, (int)max_last - b0);
    }
    int buf = 0;
    for (int32_t b_end = (int32_t)max_last; b_end > 0; b_end -= kBatch, buf ^= 1) {
        const int32_t b_begin = max(0, b_end - kBatch);
        const int n = b_end - b_begin;
        wait_ids();
        __syncthreads();  // previous batch fully consumed; this batch's ids visible
        if (b_begin > 0) {
            const int32_t nb = max(0, b_begin - kBatch);
            prefetch_ids(S.ids[buf ^ 1], a.list, start + (uint32_t)nb, b_begin - nb);
        }
        stage_batch<PPT, EXACT, kNT>(a.pay0, a.pay1, a.pay2, a.pay3, S.ids[buf], n, tile_x0, tile_y0, sb);
        __syncthreads();
        // this warp's pixels composite nothing at or behind list position warp_max
        const int nw_lim = (int)min((int64_t)n, max((int64_t)0, (int64_t)warp_max - b_begin));
        const int nw = compact_warp_list(S.mask, nw_lim, vw, S.list[warp]);
        for (int i = nw - 1; i >= 0; --i) {
            const int j = (int)lds_u16(a_list + 2u * (uint32_t)i);
            const uint32_t pos = (uint32_t)(b_begin + j);
            if (pos < nxt) {  // warp-uniform: some pixels start compositing here
                uint32_t m = 0;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if (pos < last[k]) thr[k] = kAlphaMin;
                    else m = max(m, last[k]);
                }
                nxt = __reduce_max_sync(0xffffffffu, m);
            }
            const uint32_t r16 = sbase + 16u * (uint32_t)j, r4 = sbase + 4u * (uint32_t)j;
            const float4 g0 = lds_f4_at<0>(r16);
            const float4 g1 = lds_f4_at<Sm::kG1>(r16);
            const float rb = lds_f_at<Sm::kB>(r4);
            const float dx = __fsub_rn(g0.x, fpx);
            const ExpCol ec = exp_col(g0.z, g0.w, dx);
            // Per pixel only the sums the chain rule needs: with q = G dalpha (kappa
            // factored out) and dp2 = kappa ln2 q, the conic/mean terms are
            // sum dp2 (dx, dy) and sum dp2 (dx^2, dx dy, dy^2); dx is the thread's
            // column, so S0 = sum q (= d alpha-part of dL/dkappa), S1 = sum q dy,
            // S2 = sum q dy^2 suffice.  alpha' = alpha where the pixel composites
            // this entry (alpha >= thr: active and not skipped), else 0; then every
            // term below vanishes without a select.  (No exponent clamp: R19b.)
            bool contrib = false;
            float S0 = 0.0f, S1 = 0.0f, S2 = 0.0f, dk = 0.0f, Sb = 0.0f, dr = 0.0f, dgc = 0.0f, dbc = 0.0f;
            if constexpr (EXACT) {
            const float hb = lds_f_at<Sm::kHb>(r4);
            const bool clampk = g1.y > kAlphaMax;  // warp-uniform
            const float rk = fast_rcp(g1.y);
            // Eq. 2: G = exp(-1/2 Q^hb).  dG/dp2 = G hb Q^hb / (2 qp) (Q = 2 ln2 qp),
            // dG/dbeta = -1/4 G Q^hb ln Q; with Gd = G dL/dalpha where composited:
            // dL/dkappa += Gd, the moments take wm = Gd Q^hb / qp (factor kappa hb / 2),
            // Sb = sum Gd Q^hb log2 Q (factor -1/4 kappa ln2).
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const float dy = __fsub_rn(g0.y, (float)(py0 + 4 * k) + 0.5f);
                const Gef ge = gef_eval(raw_exponent(ec, g1.x, dy), hb);
                const float araw = __fmul_rn(g1.y, ge.G);
                const float alpha = clampk ? fminf(kAlphaMax, araw) : araw;
                const float al = alpha >= thr[k] ? alpha : 0.0f;
                contrib |= al > 0.0f;
                const float inv_om = fast_rcp(__fsub_rn(1.0f, al));
                const float Tk = T[k] * inv_om;
                const float cgk = g1.z * gr[k] + g1.w * gg[k] + rb * gb[k];
                const float w = al * Tk;
                const float dalpha = Tk * cgk - U[k] * inv_om;
                U[k] += cgk * w;
                dr += w * gr[k];
                dgc += w * gg[k];
                dbc += w * gb[k];
                float Gd = (al * rk) * dalpha;  // G dL/dalpha where composited
                if (clampk) Gd = (al > 0.0f && araw < kAlphaMax) ? ge.G * dalpha : 0.0f;
                dk += Gd;
                const float GQ = Gd * ge.Qb;
                const float wm = GQ * fast_rcp(ge.qp);
                S0 += wm;
                const float t = wm * dy;
                S1 += t;
                S2 += t * dy;
                Sb += GQ * ge.L;
                T[k] = Tk;
            }
            // (dL/dp2 = kappa hb / 2 wm, dL/dbeta = -1/4 kappa ln2 Sb: S5b applies the
            // per-particle factors)
            } else {
            // The Gaussian path accumulates kappa q = alpha' dL/dalpha (kappa, a
            // per-particle constant, is divided out in S5b).
            float amax = 0.0f;
#ifdef GES_F32X2
            // the same per-pixel arithmetic on pixel pairs with FADD2 / FMUL2 / FFMA2 (the
            // exponent, alpha and the skip decision bit-identical to the scalar form and the
            // forward's); the sums accumulate per pair half and are added at the end
            {
                const f2 kap = f2_bc(g1.y), C2 = f2_bc(g1.x), c1 = f2_bc(ec.c1), c0 = f2_bc(ec.c0);
                const f2 gy = f2_bc(g0.y), one = f2_bc(1.0f);
                const f2 cz = f2_bc(g1.z), cw = f2_bc(g1.w), cb = f2_bc(rb);
                f2 s0 = 0ull, s1 = 0ull, s2 = 0ull, sr = 0ull, sg = 0ull, sb = 0ull;
                auto pairs = [&](auto clamp_tag) {
                    constexpr bool CLAMP = decltype(clamp_tag)::value;
#pragma unroll
                    for (int h = 0; h < PPT / 2; ++h) {
                        const f2 dy = f2_sub(gy, pyp[h]);
                        const f2 p2 = f2_fma(dy, f2_fma(C2, dy, c1), c0);
                        const f2 araw = f2_mul(kap, f2_pk(fast_exp2(f2_lo(p2)), fast_exp2(f2_hi(p2))));
                        float a0 = f2_lo(araw), a1 = f2_hi(araw);
                        if (CLAMP) { a0 = fminf(kAlphaMax, a0); a1 = fminf(kAlphaMax, a1); }
                        a0 = a0 >= thr[2 * h] ? a0 : 0.0f;
                        a1 = a1 >= thr[2 * h + 1] ? a1 : 0.0f;
                        amax = fmaxf(amax, fmaxf(a0, a1));
                        const f2 al = f2_pk(a0, a1);
                        const f2 om = f2_sub(one, al);
                        const f2 inv = f2_pk(fast_rcp(f2_lo(om)), fast_rcp(f2_hi(om)));
                        const f2 Tk = f2_mul(Tp[h], inv);  // transmittance before this entry
                        const f2 cg = f2_fma(cz, grp[h], f2_fma(cw, ggp[h], f2_mul(cb, gbp[h])));
                        const f2 w = f2_mul(al, Tk);
                        const f2 dal = f2_sub(f2_mul(Tk, cg), f2_mul(Up[h], inv));
                        Up[h] = f2_fma(cg, w, Up[h]);
                        sr = f2_fma(w, grp[h], sr);
                        sg = f2_fma(w, ggp[h], sg);
                        sb = f2_fma(w, gbp[h], sb);
                        f2 q;
                        if (CLAMP) {  // no gradient through the clamp (R13): q = araw dL/dalpha
                            const f2 qr = f2_mul(araw, dal);
                            const float q0 = (a0 > 0.0f && f2_lo(araw) < kAlphaMax) ? f2_lo(qr) : 0.0f;
                            const float q1 = (a1 > 0.0f && f2_hi(araw) < kAlphaMax) ? f2_hi(qr) : 0.0f;
                            q = f2_pk(q0, q1);
                        } else {
                            q = f2_mul(al, dal);  // kappa G dL/dalpha where composited
                        }
                        s0 = f2_add(s0, q);
                        const f2 t = f2_mul(q, dy);
                        s1 = f2_add(s1, t);
                        s2 = f2_fma(t, dy, s2);
                        Tp[h] = Tk;
                    }
                };
                if (!(g1.y > kAlphaMax)) pairs(std::false_type{});  // warp-uniform
                else pairs(std::true_type{});
                S0 = f2_lo(s0) + f2_hi(s0);
                S1 = f2_lo(s1) + f2_hi(s1);
                S2 = f2_lo(s2) + f2_hi(s2);
                dr = f2_lo(sr) + f2_hi(sr);
                dgc = f2_lo(sg) + f2_hi(sg);
                dbc = f2_lo(sb) + f2_hi(sb);
            }
            if (false) {
#else
            if (!(g1.y > kAlphaMax)) {  // warp-uniform: alpha cannot reach the 0.99 clamp
#endif
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const float dy = __fsub_rn(g0.y, (float)(py0 + 4 * k) + 0.5f);
                    const float G = fast_exp2(raw_exponent(ec, g1.x, dy));
                    const float alpha = __fmul_rn(g1.y, G);
                    const float al = alpha >= thr[k] ? alpha : 0.0f;
                    amax = fmaxf(amax, al);
                    const float inv_om = fast_rcp(__fsub_rn(1.0f, al));
                    const float Tk = T[k] * inv_om;  // transmittance before this entry
                    const float cgk = g1.z * gr[k] + g1.w * gg[k] + rb * gb[k];
                    const float w = al * Tk;
                    const float dalpha = Tk * cgk - U[k] * inv_om;
                    U[k] += cgk * w;
                    dr += w * gr[k];
                    dgc += w * gg[k];
                    dbc += w * gb[k];
                    const float q = al * dalpha;  // kappa G dL/dalpha where composited
                    S0 += q;
                    const float t = q * dy;
                    S1 += t;
                    S2 += t * dy;
                    T[k] = Tk;
                }
            } else if (!kF32x2) {  // alpha = min(0.99, kappa G): no gradient through the clamp (R13)
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const float dy = __fsub_rn(g0.y, (float)(py0 + 4 * k) + 0.5f);
                    const float G = fast_exp2(raw_exponent(ec, g1.x, dy));
                    const float araw = __fmul_rn(g1.y, G);
                    const float alpha = fminf(kAlphaMax, araw);
                    const float al = alpha >= thr[k] ? alpha : 0.0f;
                    amax = fmaxf(amax, al);
                    const float inv_om = fast_rcp(__fsub_rn(1.0f, al));
                    const float Tk = T[k] * inv_om;
                    const float cgk = g1.z * gr[k] + g1.w * gg[k] + rb * gb[k];
                    const float w = al * Tk;
                    const float dalpha = Tk * cgk - U[k] * inv_om;
                    U[k] += cgk * w;
                    dr += w * gr[k];
                    dgc += w * gg[k];
                    dbc += w * gb[k];
                    const float q = (al > 0.0f && araw < kAlphaMax) ? araw * dalpha : 0.0f;
                    S0 += q;
                    const float t = q * dy;
                    S1 += t;
                    S2 += t * dy;
                    T[k] = Tk;
                }
            }
            // alpha = kappa 2^p2: d alpha / d p2 = alpha ln 2, so dL/dp2 = ln2 (kappa q).
            // The record takes the raw moments sum kappa q (dx, dy, dx^2, dx dy, dy^2):
            // every factor that turns them into dL/d(u, v, A, B, C, kappa) is constant
            // per particle (kappa, the conic), so S5b applies it once after the sum.
            contrib = amax > 0.0f;
            }
            if (__any_sync(0xffffffffu, contrib)) {  // (measured: skipping beats always reducing)
                const float r = grad_reduce<EXACT>(S0, S1, S2, dk, Sb, dr, dgc, dbc, dx);
                if (red_comp >= 0 && (lane & 1) == 0)
                    red_add(a.grad2d + (size_t)lds_u32_at<Sm::kPid>(r4) * kGrad2dStride + red_comp, r);
            }
        }
    }
}

cudaError_t launch_render_bwd(const RenderBwdArgs& args, cudaStream_t stream) {
    static const int ppt = ppt_from_env("GES_PPT_BWD", 4);
    // experiment knob: GES_BWD_ORDER=0 launches the tiles in index order
    static const int use_order = [] {
        const char* e = getenv("GES_BWD_ORDER");
        return e ? atoi(e) : 1;
    }();
    RenderBwdArgs a = args;
    a.use_order = use_order && a.tile_bucket && a.tile_order;
    const int grid = a.tiles_x * a.tiles_y * (kBwdHalf ? 2 : 1);
    if (grid == 0) return cudaSuccess;  // a band without tile rows: no 2-D gradients
    if (a.exact) {
        if (ppt == 4) render_bwd_kernel<4, true><<<grid, kBwdHalf ? 32 : Layout<4>::kThreads, 0, stream>>>(a);
        else render_bwd_kernel<2, true><<<grid, kBwdHalf ? 32 : Layout<2>::kThreads, 0, stream>>>(a);
    } else {
        if (ppt == 4) {
            apply_carveout(render_bwd_kernel<4, false>);
            render_bwd_kernel<4, false><<<grid, kBwdHalf ? 32 : Layout<4>::kThreads, 0, stream>>>(a);
        } else {
            render_bwd_kernel<2, false><<<grid, kBwdHalf ? 32 : Layout<2>::kThreads, 0, stream>>>(a);
        }
    }
    return cudaGetLastError();
}

}  // namespace ges

#ifdef GES_TILE_CLOCK
extern "C" void ges_debug_tile_order(int which, const int* order, int n) {  // n = 0: off
    int on = n > 0;
    if (on) cudaMemcpyToSymbol(ges::g_tile_order, order, sizeof(int) * n, sizeof(int) * 16384 * which);
    cudaMemcpyToSymbol(ges::g_tile_order_on, &on, sizeof(int), sizeof(int) * which);
}
extern "C" void ges_debug_tile_clock(unsigned long long* out, int reset) {
    if (reset) {
        static unsigned long long init[2][16384][3];
        for (int w = 0; w < 2; ++w)
            for (int i = 0; i < 16384; ++i) { init[w][i][0] = ~0ull; init[w][i][1] = 0; init[w][i][2] = 0; }
        cudaMemcpyToSymbol(ges::g_tile_clk, init, sizeof(init));
    } else {
        cudaMemcpyFromSymbol(out, ges::g_tile_clk, sizeof(unsigned long long) * 2 * 16384 * 3);
    }
}
#endif
