// bin.cu -- S2 pair generation and S3 ranges by row-then-column binning
// (DESIGN.md "Sort").
//
// Input: the visible particles in (depth bits, index) order as item records
// (particle, packed tile rect; sort.cu) and the number of items covering each
// band tile row.  Output: the per-tile lists list[ranges[t] .. ranges[t+1]) in
// (depth bits, index) order -- exactly the order of a stable sort of the
// (tile << 32 | depth) keys -- without sorting any pair.
//
// A tile's list is the subsequence of the depth-ordered items covering it.
// Two 1-D binnings produce it:
//   bin_rows       items -> per-row lists (row r: the items covering r, in
//                  order; entries (particle, x0 | (x1 - 1) << 8));
//   bin_cols_count per chunk of a row list: the column counts, their prefix
//                  over the row's earlier chunks, and (last chunk) the tile
//                  totals of the row;
//   bin_cols       per chunk of a row list: entries -> the tiles' lists; the
//                  ranges (S3) from the tile totals.
// Both binnings work the same way on a chunk of records held by 16 warps: a
// warp's per-bin counts from a difference array in shared memory (2 atomics
// per record), exclusive over the warps, the chunk's offsets over the earlier
// chunks (published vectors, two levels of 16-chunk groups, no grid barrier),
// then per group of 32 records the LANE MASK of every bin (the records covering
// it) from a XOR difference array -- a lane owning bin b writes the records of
// mask(b) in lane order at its own cursor: no two lanes share a cursor and no
// ranking is needed.  Each chunk's output is staged in shared memory and
// copied out as one contiguous run per bin.  Work is O(V + rows V + M); the
// pairs are written once, in coalesced runs.
#include <algorithm>

#include "ges_internal.h"

namespace ges {

constexpr int kBinThreads = 512;     // column kernels
constexpr int kBinWarps = kBinThreads / 32;
#ifndef GES_ROW_THREADS
#define GES_ROW_THREADS 512
#endif
constexpr int kRowThreads = GES_ROW_THREADS;  // row kernel
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kRowItems = kRowChunk / kRowThreads;  // items per lane
constexpr int kColItems = kColChunk / kBinThreads;  // entries per lane
#ifndef GES_ROW_STAGE
#define GES_ROW_STAGE 8192
#endif
#ifndef GES_COL_STAGE
#define GES_COL_STAGE 16384
#endif
constexpr int kRowStage = GES_ROW_STAGE;  // staged row-list entries (8 B) per chunk
constexpr int kColStage = GES_COL_STAGE;  // staged list entries (4 B) per chunk
constexpr uint32_t kPub = 0x80000000u;  // published word flag (values < 2^31)
constexpr int kGroup = 16;
constexpr int kScanRows = kMaxBandRows / 32;  // rows per lane of a one-warp row scan
static_assert(kRowItems * kRowThreads == kRowChunk && kColItems * kBinThreads == kColChunk, "chunk sizes");

__device__ __forceinline__ uint32_t lb_load(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void lb_store(uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lb_wait(const uint32_t* p) {
    uint32_t v = lb_load(p);
    while (!(v & kPub)) v = lb_load(p);
    return v & ~kPub;
}

// One warp: out[i] = sum of get(j) for j < i (i < n), out[n] = the total.
template <int BPL, class F>
__device__ __forceinline__ void warp_excl(F get, uint32_t* out, int n) {
    const int lane = threadIdx.x & 31;
    uint32_t v[BPL], run = 0;
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        const int i = lane * BPL + j;
        v[j] = i < n ? get(i) : 0u;
        run += v[j];
    }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    uint32_t ex = incl - run;
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        const int i = lane * BPL + j;
        if (i < n) out[i] = ex;
        ex += v[j];
    }
    if (lane == 31) out[n] = ex;
}

// Bin of staged slot / chunk g: the last r with first[r] <= g (bins without
// entries share their first value with the next bin).
__device__ __forceinline__ int row_of(const uint32_t* first, int rows, uint32_t g) {
    int lo = 0, hi = rows - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (first[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Exclusive prefix over the earlier chunks of a sequence of published n-vectors,
// in two levels of kGroup chunks (as sort.cu's pass prefix): the words of the
// earlier chunks of this chunk's group, plus the group totals of the earlier
// groups, each published by its group's last chunk after its in-group sum.  st:
// the sequence's chunk words [chunks][n]; gt: its group words (indexed by the
// group's first chunk); k: this chunk, nk: the sequence's chunks; agg (shared):
// this chunk's vector; out (shared) = the sum over chunks < k.  Chunks are
// claimed in order (tickets), so every awaited word has a running or finished
// writer.
__device__ __forceinline__ void chunk_publish(uint32_t* st, int64_t k, int n, const uint32_t* agg) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) lb_store(st + k * n + i, kPub | agg[i]);
}
__device__ void chunk_wait(uint32_t* st, uint32_t* gt, int64_t k, int64_t nk, int n, const uint32_t* agg,
                           uint32_t* out) {
    const int tid = threadIdx.x;
    const int nt = blockDim.x;
    for (int i = tid; i < n; i += nt) out[i] = 0;
    __syncthreads();
    const int64_t first = k / kGroup * kGroup, glast = (first + kGroup < nk ? first + kGroup : nk) - 1;
    const int m = (int)(k - first);
    for (int t = tid; t < n * m; t += nt) {
        const int i = t % n, j = t / n;
        atomicAdd(&out[i], lb_wait(st + (first + j) * n + i));
    }
    __syncthreads();
    if (k == glast)
        for (int i = tid; i < n; i += nt) lb_store(gt + first * n + i, kPub | (out[i] + agg[i]));
    const int ng = (int)(first / kGroup);
    for (int t = tid; t < n * ng; t += nt) {
        const int i = t % n, gg = t / n;
        atomicAdd(&out[i], lb_wait(gt + (int64_t)gg * kGroup * n + i));
    }
    __syncthreads();
}
__device__ void chunk_prefix(uint32_t* st, uint32_t* gt, int64_t k, int64_t nk, int n, const uint32_t* agg,
                             uint32_t* out) {
    chunk_publish(st, k, n, agg);
    chunk_wait(st, gt, k, nk, n, agg, out);
}

// Per-warp bin counts of this lane's records (difference array in shared memory,
// then a prefix over the bins; lane owns bins [lane BPL, lane BPL + BPL)).
template <int BPL, int N>
__device__ __forceinline__ void warp_counts(uint32_t* sc, const int (&lo)[N], const int (&hi)[N], uint32_t valid) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int g = 0; g < N; ++g)
        if ((valid >> g) & 1u) {
            atomicAdd(&sc[lo[g]], 1u);
            atomicSub(&sc[hi[g]], 1u);
        }
    __syncwarp();
    uint32_t v[BPL], run = 0;
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        run += sc[lane * BPL + j];
        v[j] = run;
    }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    const uint32_t ex = incl - run;
#pragma unroll
    for (int j = 0; j < BPL; ++j) sc[lane * BPL + j] = v[j] + ex;
    if (lane == 0) sc[32 * BPL] = 0;
    __syncwarp();
}

// Lane masks of one group of 32 records: m[j] = the lanes whose record covers bin
// lane + 32 j, from a XOR difference array (sx: the warp's [32 BPL + 1] words,
// all zero on entry and on return).  The prefix runs over contiguous bins per
// lane; the masks are handed out strided so that a lane's bins lie far apart
// (the records of a group cluster in neighbouring bins: the emission loop runs
// max over lanes of the records per bin, per j).
template <int BPL>
__device__ __forceinline__ void group_masks(uint32_t* sx, bool valid, int lo, int hi, uint32_t (&m)[BPL]) {
    const int lane = threadIdx.x & 31;
    if (valid) {
        atomicXor(&sx[lo], 1u << lane);
        atomicXor(&sx[hi], 1u << lane);
    }
    __syncwarp();
    uint32_t c[BPL], run = 0;
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        run ^= sx[lane * BPL + j];
        c[j] = run;
    }
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x ^= nn;
    }
    const uint32_t ex = x ^ run;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < BPL; ++j) sx[lane * BPL + j] = c[j] ^ ex;
    if (lane == 0) sx[32 * BPL] = 0u;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        m[j] = sx[lane + 32 * j];
        sx[lane + 32 * j] = 0u;
    }
    __syncwarp();
}

// Emission of one group: the lane owning bin b = lane + 32 j writes the payloads
// of the records in m[j] (lane order) at dst[cur[j]++].  No warp collective per
// trip (VOTE and SHFL issue at a fraction of the ALU rate): the trip count is the
// warp's largest popcount (one REDUX per j), the payloads come from shared memory.
#ifdef GES_BIN_STATS
__device__ unsigned long long g_bin_trips[2];  // emission loop trips: [0] rows, [1] columns
__device__ unsigned long long g_bin_direct[4]; // chunks: [0] rows direct, [1] rows, [2] columns direct, [3] columns
#endif
template <int BPL, class T>
__device__ __forceinline__ void emit_group(T* dst, const uint32_t (&m)[BPL], uint32_t (&cur)[BPL], const T* pay) {
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        uint32_t bits = m[j];
        const int n = (int)__reduce_max_sync(0xffffffffu, (unsigned)__popc(bits));
#ifdef GES_BIN_STATS
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_bin_trips[sizeof(T) == 4], (unsigned long long)n);
#endif
        for (int t = 0; t < n; ++t) {
            if (bits) {
                dst[cur[j]++] = pay[__ffs(bits) - 1];
                bits &= bits - 1u;
            }
        }
    }
}

// The same into a shared-memory stage, branch-free: a lane with no record left
// in this bin writes to the stage's spare slot stage[spare].
template <int BPL, class T>
__device__ __forceinline__ void emit_group_staged(T* stage, uint32_t spare, const uint32_t (&m)[BPL],
                                                  uint32_t (&cur)[BPL], const T* pay) {
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        uint32_t bits = m[j];
        const int n = (int)__reduce_max_sync(0xffffffffu, (unsigned)__popc(bits));
        uint32_t c = cur[j];
#pragma unroll 2
        for (int t = 0; t < n; ++t) {
            const uint32_t act = bits != 0u;
            const T v = pay[(__ffs(bits) - 1) & 31];
            stage[act ? c : spare] = v;
            c += act;
            bits &= bits - 1u;
        }
        cur[j] = c;
    }
}

// Copy-out of a staged chunk: bin x's run stage[lbase[x], lbase[x+1]) goes to
// out[gbase[x] ...) (one warp per bin, coalesced).
template <class T>
__device__ __forceinline__ void copy_runs(const T* stage, T* out, const uint32_t* lbase, const uint32_t* gbase, int n) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int x = warp; x < n; x += (int)(blockDim.x >> 5)) {
        const uint32_t l0 = lbase[x], len = lbase[x + 1] - l0, g0 = gbase[x];
        for (uint32_t i = lane; i < len; i += 32) out[g0 + i] = stage[l0 + i];
    }
}

// ---- rows: items -> per-row lists ------------------------------------------
template <int BPL>
__global__ void __launch_bounds__(kRowThreads) bin_rows_kernel(BinArgs a) {
    constexpr int NB = 32 * BPL;
    __shared__ uint32_t s_cnt[kRowWarps][NB + 1];
    __shared__ uint32_t s_msk[kRowWarps][NB + 1];
    __shared__ uint32_t s_agg[NB], s_excl[NB], s_lbase[NB + 1], s_gbase[kMaxBandRows + 1];
    __shared__ uint2 s_pay[kRowWarps][32];
    __shared__ unsigned long long s_k;
    extern __shared__ __align__(16) uint2 s_rstage[];  // [kRowStage + 1] (+ the spare slot)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = a.rows;
    if ((int64_t)a.counters[GES_CTR_SLOTS] > a.capacity) {  // the lists would not fit: nothing is binned
        if (blockIdx.x == 0 && tid == 0) a.counters[GES_CTR_OVERFLOW] = 1ull;
        return;
    }
    const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
    if (tid == 0) s_k = atomicAdd(&a.counters[GES_CTR_TICKET], 1ull);
    for (int i = tid; i < kRowWarps * (NB + 1); i += kRowThreads) {
        (&s_cnt[0][0])[i] = 0u;
        (&s_msk[0][0])[i] = 0u;
    }
    __syncthreads();
    const int64_t k = (int64_t)s_k, s0 = k * kRowChunk;
    if (s0 >= V) return;
    const int64_t nk = (V + kRowChunk - 1) / kRowChunk;
    // this warp's 32 x kRowItems items, groups of 32 in order
    uint32_t pid[kRowItems], xp[kRowItems];
    int y0[kRowItems], y1[kRowItems];
    uint32_t valid = 0;
    const int64_t wb = s0 + (int64_t)warp * 32 * kRowItems;
#pragma unroll
    for (int g = 0; g < kRowItems; ++g) {
        const int64_t idx = wb + g * 32 + lane;
        const uint2 it = idx < V ? a.items[idx] : make_uint2(0u, 0u);
        if (idx < V) valid |= 1u << g;
        pid[g] = it.x;
        xp[g] = it.y & 0xffffu;
        y0[g] = (int)((it.y >> 16) & 255u);
        y1[g] = (int)(it.y >> 24) + 1;
    }
    warp_counts<BPL>(s_cnt[warp], y0, y1, valid);
    __syncthreads();
    if (tid < rows) {  // exclusive over the warps; the chunk's row counts
        uint32_t run = 0;
        for (int w = 0; w < kRowWarps; ++w) {
            const uint32_t x = s_cnt[w][tid];
            s_cnt[w][tid] = run;
            run += x;
        }
        s_agg[tid] = run;
    }
    __syncthreads();
    // publish this chunk's row counts now; the prefix over the earlier chunks is awaited only
    // after the emission into the stage (which needs the local offsets alone)
    uint32_t* lbw = a.lb_rows;
    uint32_t* lbg = a.lb_rows + a.row_chunks * rows;
    chunk_publish(lbw, k, rows, s_agg);
    if (warp == 1) warp_excl<BPL>([&](int i) { return s_agg[i]; }, s_lbase, rows);  // staging offsets
    __syncthreads();
    const uint32_t total = s_lbase[rows];
    const bool staged = total <= (uint32_t)kRowStage;
#ifdef GES_BIN_STATS
    if (tid == 0) { atomicAdd(&g_bin_direct[0], staged ? 0ull : 1ull); atomicAdd(&g_bin_direct[1], 1ull); }
#endif
    auto global_base = [&]() {  // global first slot of this chunk's entries in each row
        chunk_wait(lbw, lbg, k, nk, rows, s_agg, s_excl);
        if (warp == 0) {
            warp_excl<kScanRows>([&](int i) { return a.row_count[i]; }, s_gbase, rows);
            __syncwarp();
            for (int i = lane; i < rows; i += 32) s_gbase[i] += s_excl[i];
        }
        __syncthreads();
    };
    if (!staged) global_base();
    uint32_t cur[BPL];
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
        const int y = lane + 32 * j;
        cur[j] = y < rows ? (staged ? s_lbase[y] : s_gbase[y]) + s_cnt[warp][y] : 0u;
    }
#pragma unroll
    for (int g = 0; g < kRowItems; ++g) {
        uint32_t m[BPL];
        s_pay[warp][lane] = make_uint2(pid[g], xp[g]);
        group_masks<BPL>(s_msk[warp], (valid >> g) & 1u, y0[g], y1[g], m);  // (syncs the warp)
        if (staged) emit_group_staged<BPL>(s_rstage, kRowStage, m, cur, s_pay[warp]);
        else emit_group<BPL>(a.rowlist, m, cur, s_pay[warp]);
        __syncwarp();
    }
    if (staged) {
        global_base();  // (its barriers also order the emission before the copy)
        copy_runs(s_rstage, a.rowlist, s_lbase, s_gbase, rows);
    }
}

// Row scans shared by the column kernels: s_rb = first row-list entry of each
// row, s_cf = first column chunk of each row ([rows] = the totals).
__device__ __forceinline__ void row_tables(const BinArgs& a, uint32_t* s_rb, uint32_t* s_cf) {
    const int warp = threadIdx.x >> 5;
    if (warp == 0) warp_excl<kScanRows>([&](int i) { return a.row_count[i]; }, s_rb, a.rows);
    else if (warp == 1)
        warp_excl<kScanRows>([&](int i) { return (a.row_count[i] + (uint32_t)kColChunk - 1u) / (uint32_t)kColChunk; },
                             s_cf, a.rows);
}

// ---- columns, pass 1: per-chunk column counts and their prefix ---------------
template <int BPL>
__global__ void __launch_bounds__(kBinThreads) bin_cols_count_kernel(BinArgs a) {
    constexpr int NB = 32 * BPL;
    __shared__ uint32_t s_rb[kMaxBandRows + 1], s_cf[kMaxBandRows + 1];
    __shared__ uint32_t s_d[NB + 1], s_excl[NB];
    __shared__ uint32_t s_sum;
    __shared__ unsigned long long s_g;
    if (a.counters[GES_CTR_OVERFLOW]) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = a.rows, tx = a.tiles_x;
    row_tables(a, s_rb, s_cf);
    __syncthreads();
    const uint32_t G2 = s_cf[rows];
    for (;;) {
        if (tid == 0) { s_g = atomicAdd(&a.counters[GES_CTR_TICKET_COLS], 1ull); s_sum = 0; }
        for (int i = tid; i <= NB; i += kBinThreads) s_d[i] = 0u;
        __syncthreads();
        const uint64_t g = s_g;
        if (g >= G2) break;
        const int y = row_of(s_cf, rows, (uint32_t)g);
        const int64_t k = (int64_t)g - s_cf[y], nk = (int64_t)s_cf[y + 1] - s_cf[y];
        const uint32_t e0 = s_rb[y] + (uint32_t)k * kColChunk, e1 = min(e0 + (uint32_t)kColChunk, s_rb[y + 1]);
        uint32_t r[kColItems];
#pragma unroll
        for (int u = 0; u < kColItems; ++u) {
            const uint32_t e = e0 + u * kBinThreads + tid;
            r[u] = e < e1 ? a.rowlist[e].y : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < kColItems; ++u)
            if (r[u] != 0xffffffffu) {
                atomicAdd(&s_d[r[u] & 255u], 1u);
                atomicSub(&s_d[((r[u] >> 8) & 255u) + 1u], 1u);
            }
        __syncthreads();
        if (warp == 0) {  // column counts (inclusive prefix of the difference array)
            uint32_t v[BPL], run = 0;
#pragma unroll
            for (int j = 0; j < BPL; ++j) { run += s_d[lane * BPL + j]; v[j] = run; }
            uint32_t incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += nn;
            }
            const uint32_t ex = incl - run;
#pragma unroll
            for (int j = 0; j < BPL; ++j) s_d[lane * BPL + j] = v[j] + ex;
        }
        __syncthreads();
        const int64_t g0 = (int64_t)g - k;  // the row's first chunk
        chunk_prefix(a.lb_cols + g0 * tx, a.lb_cols + (a.col_chunks + g0) * tx, k, nk, tx, s_d, s_excl);
        for (int x = tid; x < tx; x += kBinThreads) a.col_excl[g * tx + x] = s_excl[x];
        if (k == nk - 1) {  // the row's tile totals
            uint32_t part = 0;
            for (int x = tid; x < tx; x += kBinThreads) {
                const uint32_t t = s_excl[x] + s_d[x];
                a.tile_count[(int64_t)y * tx + x] = t;
                part += t;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (lane == 0 && part) atomicAdd(&s_sum, part);
            __syncthreads();
            if (tid == 0) a.row_pairs[y] = s_sum;
        }
        __syncthreads();
    }
}

// ---- columns, pass 2: row-list entries -> tile lists; the ranges -------------
template <int BPL>
__global__ void __launch_bounds__(kBinThreads) bin_cols_kernel(BinArgs a) {
    constexpr int NB = 32 * BPL;
    __shared__ uint32_t s_cnt[kBinWarps][NB + 1];
    __shared__ uint32_t s_msk[kBinWarps][NB + 1];
    __shared__ uint32_t s_rb[kMaxBandRows + 1], s_cf[kMaxBandRows + 1], s_rp[kMaxBandRows + 1];
    __shared__ uint32_t s_lbase[NB + 1], s_gbase[NB + 1];
    __shared__ uint32_t s_pay[kBinWarps][32];
    __shared__ unsigned long long s_g;
    extern __shared__ __align__(16) uint32_t s_cstage[];  // [kColStage + 1] (+ the spare slot)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = a.rows, tx = a.tiles_x;
    const bool ovf = a.counters[GES_CTR_OVERFLOW] != 0;
    row_tables(a, s_rb, s_cf);
    if (warp == 2) warp_excl<kScanRows>([&](int i) { return a.row_pairs[i]; }, s_rp, rows);
    for (int i = tid; i < kBinWarps * (NB + 1); i += kBinThreads) (&s_msk[0][0])[i] = 0u;
    __syncthreads();
    // S3: ranges of the rows y = blockIdx.x (mod gridDim.x); on overflow every count is 0
    if (warp == 0) {
        for (int y = blockIdx.x; y < rows; y += gridDim.x) {
            warp_excl<BPL>([&](int i) { return a.tile_count[(int64_t)y * tx + i]; }, s_gbase, tx);
            __syncwarp();
            for (int x = lane; x < tx; x += 32) a.ranges[(int64_t)y * tx + x] = s_rp[y] + s_gbase[x];
            __syncwarp();
        }
        if (blockIdx.x == 0 && lane == 0) {
            a.ranges[(int64_t)rows * tx] = s_rp[rows];
            a.counters[GES_CTR_PAIRS] = s_rp[rows];
        }
    }
    if (ovf) return;
    const uint32_t G2 = s_cf[rows];
    for (;;) {
        if (tid == 0) s_g = atomicAdd(&a.counters[GES_CTR_TICKET_EMIT], 1ull);
        for (int i = tid; i < kBinWarps * (NB + 1); i += kBinThreads) (&s_cnt[0][0])[i] = 0u;
        __syncthreads();
        const uint64_t g = s_g;
        if (g >= G2) break;
        const int y = row_of(s_cf, rows, (uint32_t)g);
        const uint32_t k = (uint32_t)g - s_cf[y];
        const uint32_t e0 = s_rb[y] + k * kColChunk, e1 = min(e0 + (uint32_t)kColChunk, s_rb[y + 1]);
        if (warp == 0) {  // first list slot of this chunk's entries in each tile of the row
            warp_excl<BPL>([&](int i) { return a.tile_count[(int64_t)y * tx + i]; }, s_gbase, tx);
            __syncwarp();
            for (int x = lane; x < tx; x += 32) s_gbase[x] += s_rp[y] + a.col_excl[g * tx + x];
        }
        // this warp's entries [e0 + warp 32 kColItems, ...), groups of 32 in order
        uint32_t pid[kColItems];
        int x0[kColItems], x1[kColItems];
        uint32_t valid = 0;
        const uint32_t wb = e0 + (uint32_t)warp * 32 * kColItems;
#pragma unroll
        for (int g2 = 0; g2 < kColItems; ++g2) {
            const uint32_t e = wb + g2 * 32 + lane;
            const uint2 r = e < e1 ? a.rowlist[e] : make_uint2(0u, 0u);
            if (e < e1) valid |= 1u << g2;
            pid[g2] = r.x;
            x0[g2] = (int)(r.y & 255u);
            x1[g2] = (int)((r.y >> 8) & 255u) + 1;
        }
        warp_counts<BPL>(s_cnt[warp], x0, x1, valid);
        __syncthreads();
        if (tid < tx) {  // exclusive over the warps; the chunk's column counts
            uint32_t run = 0;
            for (int w = 0; w < kBinWarps; ++w) {
                const uint32_t x = s_cnt[w][tid];
                s_cnt[w][tid] = run;
                run += x;
            }
            s_lbase[tid] = run;
        }
        __syncthreads();
        if (warp == 0) {  // staging offsets
            uint32_t v[BPL];
#pragma unroll
            for (int j = 0; j < BPL; ++j) v[j] = lane * BPL + j < tx ? s_lbase[lane * BPL + j] : 0u;
            __syncwarp();
            warp_excl<BPL>([&](int i) {
                uint32_t r = 0;
#pragma unroll
                for (int j = 0; j < BPL; ++j) r = (i == lane * BPL + j) ? v[j] : r;
                return r;
            }, s_lbase, tx);
        }
        __syncthreads();
        const uint32_t total = s_lbase[tx];
        const bool staged = total <= (uint32_t)kColStage;
#ifdef GES_BIN_STATS
        if (tid == 0) { atomicAdd(&g_bin_direct[2], staged ? 0ull : 1ull); atomicAdd(&g_bin_direct[3], 1ull); }
#endif
        uint32_t cur[BPL];
#pragma unroll
        for (int j = 0; j < BPL; ++j) {
            const int x = lane + 32 * j;
            cur[j] = x < tx ? (staged ? s_lbase[x] : s_gbase[x]) + s_cnt[warp][x] : 0u;
        }
#pragma unroll
        for (int g2 = 0; g2 < kColItems; ++g2) {
            uint32_t m[BPL];
            s_pay[warp][lane] = pid[g2];
            group_masks<BPL>(s_msk[warp], (valid >> g2) & 1u, x0[g2], x1[g2], m);  // (syncs the warp)
            if (staged) emit_group_staged<BPL>(s_cstage, kColStage, m, cur, s_pay[warp]);
            else emit_group<BPL>(a.list, m, cur, s_pay[warp]);
            __syncwarp();
        }
        __syncthreads();
        if (staged) copy_runs(s_cstage, a.list, s_lbase, s_gbase, tx);
        __syncthreads();
    }
}

template <class K>
static cudaError_t set_smem(K kernel, int bytes, int* done) {
    int& d = done[current_device()];
    if (d) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) d = 1;
    return e;
}

template <int BR>
static cudaError_t launch_rows(const BinArgs& a, cudaStream_t stream) {
    static int done[kMaxDevices] = {0};
    const int smem = (kRowStage + 1) * (int)sizeof(uint2);
    cudaError_t e = set_smem(bin_rows_kernel<BR>, smem, done);
    if (e != cudaSuccess) return e;
    bin_rows_kernel<BR><<<(unsigned)std::max<int64_t>(1, a.row_chunks), kRowThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

template <int BC>
static cudaError_t launch_cols(const BinArgs& a, cudaStream_t stream) {
    static int done[kMaxDevices] = {0};
    const int smem = (kColStage + 1) * (int)sizeof(uint32_t);
    cudaError_t e = set_smem(bin_cols_kernel<BC>, smem, done);
    if (e != cudaSuccess) return e;
    bin_cols_count_kernel<BC><<<num_sms() * 4, kBinThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    bin_cols_kernel<BC><<<num_sms() * 2, kBinThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

static int bins_per_lane(int n) {
    const int b = std::max(1, (n + 31) / 32);
    return b <= 4 ? b : 8;
}

cudaError_t launch_bin(const BinArgs& a, cudaStream_t stream) {
    cudaError_t e;
    switch (bins_per_lane(a.rows)) {
        case 1: e = launch_rows<1>(a, stream); break;
        case 2: e = launch_rows<2>(a, stream); break;
        case 3: e = launch_rows<3>(a, stream); break;
        case 4: e = launch_rows<4>(a, stream); break;
        default: e = launch_rows<8>(a, stream); break;
    }
    if (e != cudaSuccess) return e;
    switch (bins_per_lane(a.tiles_x)) {
        case 1: return launch_cols<1>(a, stream);
        case 2: return launch_cols<2>(a, stream);
        case 3: return launch_cols<3>(a, stream);
        case 4: return launch_cols<4>(a, stream);
        default: return launch_cols<8>(a, stream);
    }
}

}  // namespace ges

#ifdef GES_BIN_STATS
extern "C" void ges_debug_bin_trips(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, ges::g_bin_trips, sizeof(unsigned long long) * 2);
    cudaMemcpyFromSymbol(out + 2, ges::g_bin_direct, sizeof(unsigned long long) * 4);
}
#endif
