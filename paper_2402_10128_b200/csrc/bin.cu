// bin.cu -- S2 pair generation and S3 ranges by direct tile binning
// (DESIGN.md "Sort").
//
// Input: the visible particles in (depth bits, index) order as packed item
// records (E = first pair slot, particle, x0|y0<<16, x1|y1<<16 of the R10
// rect; written by the item scan in sort.cu).  Output: the per-tile lists
// list[ranges[t] .. ranges[t+1]) in (depth bits, index) order -- exactly the
// order of a stable sort of the (tile << 32 | depth) keys -- without sorting
// any pair.
//
// The depth-ordered items are cut into chunks of equal cost, cost = pairs +
// kBinItemCost x items (the item scan records the first item of every chunk).  A tile's list is then the concatenation, in
// chunk order, of each chunk's items covering the tile, in item order:
//   bin_count     per (chunk, window of tile rows): per-tile counts of the
//                 chunk's items from a 2-D difference array of their rects in
//                 shared memory (4 atomics per item) -> table[chunk][t];
//   bin_colscan   per 32-tile column block: exclusive prefix of table[.][t]
//                 over the chunks (32 warps split the chunks), tile total ->
//                 ranges[t];
//   bin_tilescan  exclusive prefix of the tile totals -> ranges, M;
//   bin_scatter   per (chunk, window): cursors = ranges[t] + table[chunk][t]
//                 in shared memory; the chunk's item records stream into a
//                 4-stage shared-memory ring by TMA bulk copies (one producer
//                 warp, mbarriers); consumer warp w owns the window's tile rows
//                 ly = w (mod 8), so no two warps ever touch one cursor.  The
//                 warp expands 32 items at a time into its pairs (a warp scan
//                 of their pair counts, a 5-step shuffle search per pair) in
//                 (item, row, column) order; pairs of one round that hit the
//                 same tile are ranked in lane order (a conflict test in
//                 shared memory, then a ballot multisplit only when needed),
//                 so every tile receives its items in item order.
// Work is O(V + M) with no pass over the pairs other than writing them once.
#include <algorithm>

#include "ges_internal.h"

namespace ges {

constexpr int kBinThreads = 256;
constexpr int kBinWarps = kBinThreads / 32;  // row classes of the scatter
constexpr int kDiffMax = kBinWinTiles + 2 * 256 + 1;  // (rows + 1) x (tiles_x + 1)
static_assert(kBinWarps == 8, "row classes are ly mod 8");

__device__ __forceinline__ int64_t bin_chunks(const BinArgs& a) { return (int64_t)a.counters[GES_CTR_CHUNKS]; }

__device__ __forceinline__ void unpack_rect(const uint4 r, int& x0, int& y0, int& x1, int& y1) {
    x0 = (int)(r.z & 0xffffu); y0 = (int)(r.z >> 16); x1 = (int)(r.w & 0xffffu); y1 = (int)(r.w >> 16);
}

__global__ void __launch_bounds__(kBinThreads) bin_count_kernel(BinArgs a) {
    __shared__ int s_diff[kDiffMax];
    if (a.counters[GES_CTR_OVERFLOW]) return;
    const int64_t c = blockIdx.x;
    if (c >= bin_chunks(a)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R0 = (int)blockIdx.y * a.win_rows, R1 = min(a.rows, R0 + a.win_rows);
    const int nr = R1 - R0, tx = a.tiles_x, pitch = tx + 1;
    for (int i = tid; i < (nr + 1) * pitch; i += kBinThreads) s_diff[i] = 0;
    __syncthreads();
    const uint32_t f = a.chunk_first[c], e = a.chunk_first[c + 1];
    constexpr int kU = 8;  // record loads in flight per thread
    for (uint32_t s0 = f; s0 < e; s0 += kU * kBinThreads) {
        uint4 rec[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t s = s0 + u * kBinThreads + tid;
            rec[u] = s < e ? __ldg(a.items + s) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            int x0, y0, x1, y1;
            unpack_rect(rec[u], x0, y0, x1, y1);
            const int ya = max(y0, R0) - R0, yb = min(y1, R1) - R0;
            if (ya >= yb) continue;  // also the padding records (empty rects)
            atomicAdd(&s_diff[ya * pitch + x0], 1);
            atomicAdd(&s_diff[ya * pitch + x1], -1);
            atomicAdd(&s_diff[yb * pitch + x0], -1);
            atomicAdd(&s_diff[yb * pitch + x1], 1);
        }
    }
    __syncthreads();
    // prefix along x: one warp per row
    for (int y = warp; y < nr; y += kBinWarps) {
        int run = 0;
        for (int x0 = 0; x0 < tx; x0 += 32) {
            const int x = x0 + lane;
            const int v = x < tx ? s_diff[y * pitch + x] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int nn = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += nn;
            }
            if (x < tx) s_diff[y * pitch + x] = run + incl;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    // prefix along y, one thread per column (shared memory only) ...
    for (int x = tid; x < tx; x += kBinThreads) {
        int run = 0;
        for (int y = 0; y < nr; ++y) {
            run += s_diff[y * pitch + x];
            s_diff[y * pitch + x] = run;
        }
    }
    __syncthreads();
    // ... then table[c][t] (one coalesced row per chunk)
    for (int i = tid; i < nr * tx; i += kBinThreads) {
        const int y = i / tx, x = i - y * tx;
        a.table[c * a.T + R0 * tx + i] = (uint32_t)s_diff[y * pitch + x];
    }
}

// Per block of 32 tiles (lane = tile): 32 warps split the chunks into
// contiguous ranges; pass 1 sums each range, the ranges are scanned in shared
// memory, pass 2 rewrites each count as its exclusive prefix.  The tile totals
// become the ranges (S3) in the same kernel: warp 0 scans its block's 32 totals
// and finds the pairs of all earlier blocks by a decoupled look-back over their
// published (flagged) sums -- no separate scan launch over the tiles.
constexpr int kColThreads = 1024;
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = (1ull << 62) - 1;
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__global__ void __launch_bounds__(kColThreads) bin_colscan_kernel(BinArgs a) {
    __shared__ uint32_t s_sum[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int blk = blockIdx.x, nblk = gridDim.x;
    const int64_t t = (int64_t)blk * 32 + lane;
    const bool ok = t < a.T;
    if (a.counters[GES_CTR_OVERFLOW]) {  // nothing was binned: empty ranges
        if (warp == 0 && ok) a.ranges[t] = 0;
        if (warp == 0 && blk == nblk - 1 && lane == 0) { a.ranges[a.T] = 0; a.counters_w[GES_CTR_PAIRS] = 0; }
        return;
    }
    const int C = (int)bin_chunks(a);
    const int per = (C + 31) / 32;
    const int c0 = min(C, warp * per), c1 = min(C, c0 + per);
    uint32_t sum = 0;
    constexpr int kU = 8;
    for (int c = c0; c < c1; c += kU) {
        uint32_t v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = (ok && c + u < c1) ? a.table[(int64_t)(c + u) * a.T + t] : 0u;
#pragma unroll
        for (int u = 0; u < kU; ++u) sum += v[u];
    }
    s_sum[warp][lane] = sum;
    __syncthreads();
    if (warp == 0) {
        uint32_t run = 0;  // this tile's total
        for (int w = 0; w < 32; ++w) {
            const uint32_t x = s_sum[w][lane];
            s_sum[w][lane] = run;
            run += x;
        }
        // the block's exclusive prefix over its 32 tiles, its aggregate
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += nn;
        }
        const unsigned long long agg = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long* st = a.lookback;
        if (lane == 0) lb_store(st + blk, (blk == 0 ? kLbInc : kLbAgg) | agg);
        // decoupled look-back over the earlier blocks, 32 at a time
        unsigned long long excl = 0;
        for (int j = blk - 1; j >= 0; j -= 32) {
            const int idx = j - lane;
            unsigned long long s = idx >= 0 ? lb_load(st + idx) : kLbInc;
            while (__any_sync(0xffffffffu, (s & ~kLbVal) == 0ull)) {
                if ((s & ~kLbVal) == 0ull) s = lb_load(st + idx);
            }
            const uint32_t inc = __ballot_sync(0xffffffffu, (s & kLbInc) != 0ull);
            const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest inclusive predecessor (or this window)
            unsigned long long v = lane <= stop ? (s & kLbVal) : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            excl += v;
            if (inc) break;
        }
        if (lane == 0 && blk > 0) lb_store(st + blk, kLbInc | (excl + agg));
        if (ok) a.ranges[t] = (uint32_t)(excl + incl - run);
        if (blk == nblk - 1 && lane == 31) {
            a.ranges[a.T] = (uint32_t)(excl + incl);
            a.counters_w[GES_CTR_PAIRS] = excl + incl;
        }
    }
    __syncthreads();
    uint32_t run = s_sum[warp][lane];
    for (int c = c0; c < c1; c += kU) {
        uint32_t v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = (ok && c + u < c1) ? a.table[(int64_t)(c + u) * a.T + t] : 0u;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (ok && c + u < c1) a.table[(int64_t)(c + u) * a.T + t] = run;
            run += v[u];
        }
    }
}

// An item's pairs in the rows ly = warp (mod 8) of the window: count, and the
// packed geometry (x0, w - 1, first row of the class).
__device__ __forceinline__ uint32_t class_pairs(const uint4 r, int R0, int R1, int warp, uint32_t& geo) {
    int x0, y0, x1, y1;
    unpack_rect(r, x0, y0, x1, y1);
    const int ya = max(y0, R0) - R0, yb = min(y1, R1) - R0;
    if (ya >= yb) return 0u;
    const int nrows = ((yb + 7 - warp) >> 3) - ((ya + 7 - warp) >> 3);
    const int w = x1 - x0;
    const int afirst = ya + ((warp - ya) & 7);  // first row of the class
    geo = (uint32_t)x0 | ((uint32_t)(w - 1) << 8) | ((uint32_t)afirst << 16);
    return (uint32_t)(nrows * w);
}

constexpr int kQueue = 64;  // per-warp FIFO of item records (power of 2, >= 63)

// --- mbarrier / TMA bulk-copy helpers (PTX) ---------------------------------
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

// Warps 0-7 consume the chunk's item records from a 4-stage ring that warp 8
// fills with TMA bulk copies; each consumer appends the records with pairs in
// its rows to a private FIFO and expands every 32 queued items into pairs.
constexpr int kStageRec = 512;  // item records per stage (8 KB)
constexpr int kStages = 4;
constexpr int kScatThreads = kBinThreads + 32;
__global__ void __launch_bounds__(kScatThreads) bin_scatter_kernel(BinArgs a) {
    extern __shared__ __align__(128) uint4 s_ring[];  // [kStages][kStageRec]
    __shared__ uint32_t s_cur[kBinWinTiles];
    __shared__ uint8_t s_own[kBinWinTiles];
    __shared__ uint4 s_q[kBinWarps][kQueue];
    __shared__ uint8_t s_mark[kBinWarps][32];
    __shared__ __align__(8) uint64_t s_full[kStages], s_empty[kStages];
    if (a.counters[GES_CTR_OVERFLOW]) return;
    const int64_t c = blockIdx.x;
    if (c >= bin_chunks(a)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int R0 = (int)blockIdx.y * a.win_rows, R1 = min(a.rows, R0 + a.win_rows);
    const int tx = a.tiles_x, wt = (R1 - R0) * tx;
    const int64_t tbase = (int64_t)R0 * tx;
    const uint32_t f = a.chunk_first[c], e = a.chunk_first[c + 1];
    const uint32_t nb = (e - f + kStageRec - 1) / kStageRec;
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], kBinWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < wt; i += kScatThreads) s_cur[i] = a.ranges[tbase + i] + a.table[c * a.T + tbase + i];
    if (warp < kBinWarps) s_mark[warp][lane] = 0;
    __syncthreads();
    if (warp == kBinWarps) {  // producer
        if (lane == 0) {
            for (uint32_t b = 0; b < nb; ++b) {
                const int st = (int)(b % kStages);
                if (b >= kStages) mbar_wait(&s_empty[st], ((b / kStages) - 1) & 1);
                const uint32_t n = min((uint32_t)kStageRec, e - f - b * kStageRec);
                mbar_expect_tx(&s_full[st], n * 16u);
                bulk_g2s(s_ring + st * kStageRec, a.items + f + b * kStageRec, n * 16u, &s_full[st]);
            }
        }
        return;
    }
    int qhead = 0, qn = 0;  // FIFO state (warp-uniform)
    // Expands the next `ng` queued items (FIFO head) into their pairs in the
    // warp's rows, in (item, row, column) order, 32 pairs per round: the source
    // item of each lane from the item starts marked in shared memory, the tile by
    // an exact float division, the stable rank among equal tiles of the round by
    // a conflict test (owner bytes) and MATCH only when needed.
    auto expand_group = [&](int ng) {
    uint32_t cnt = 0, geo = 0, pid = 0;
    float rw = 0.0f;
    if (lane < ng) {
        const uint4 r = s_q[warp][(qhead + lane) & (kQueue - 1)];
        cnt = class_pairs(r, R0, R1, warp, geo);
        pid = r.y;
        rw = __fdividef(1.0f, (float)(((geo >> 8) & 255u) + 1u));
    }
    qhead = (qhead + ng) & (kQueue - 1);
    qn -= ng;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    const uint32_t excl = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    int carry = 0;  // source lane of the pair before this round
    for (uint32_t base = 0; base < total; base += 32) {
        // source lane of pair base + lane: the last item starting at or before it
        if (cnt && excl >= base && excl < base + 32) s_mark[warp][excl - base] = (uint8_t)(lane + 1);
        __syncwarp();
        const uint32_t m = s_mark[warp][lane];
        s_mark[warp][lane] = 0;
        const uint32_t starts = __ballot_sync(0xffffffffu, m != 0u) & (0xffffffffu >> (31 - lane));
        const int sm = (int)__shfl_sync(0xffffffffu, m, starts ? 31 - __clz(starts) : 0) - 1;
        const int src = starts ? sm : carry;  // no start at or before this lane: the carried item
        const uint32_t gi = base + lane;
        const bool valid = gi < total;
        const uint32_t s_excl = __shfl_sync(0xffffffffu, excl, src);
        const uint32_t s_geo = __shfl_sync(0xffffffffu, geo, src);
        const uint32_t s_pid = __shfl_sync(0xffffffffu, pid, src);
        const float s_rw = __shfl_sync(0xffffffffu, rw, src);
        carry = __shfl_sync(0xffffffffu, src, 31);
        const uint32_t k = gi - s_excl;
        const uint32_t w = ((s_geo >> 8) & 255u) + 1u;
        // k / w exactly: k < 32 w, w <= 256, so the quotient (<= 31) is >= 0.5 / w from an
        // integer while a few-ulp reciprocal errs by < 1e-5
        const uint32_t ri = __float2uint_rz(__fmaf_rn((float)k, s_rw, 0.5f * s_rw));
        const uint32_t xx = k - ri * w;
        const uint32_t ly = (s_geo >> 16) + 8u * ri;
        const uint32_t lt = ly * (uint32_t)tx + (s_geo & 255u) + xx;
        // lanes of this round that hit the same tile: ranked in lane order
        if (valid) s_own[lt] = (uint8_t)lane;
        __syncwarp();
        const bool lost = valid && s_own[lt] != (uint8_t)lane;
        uint32_t peers = 1u << lane;
        if (__any_sync(0xffffffffu, lost)) {
#ifndef GES_BIN_BALLOT
            peers = __match_any_sync(0xffffffffu, valid ? lt : 0xffffffffu);
#else
            const uint32_t cid = (ly >> 3) * (uint32_t)tx + (s_geo & 255u) + xx;
            peers = __ballot_sync(0xffffffffu, valid);
            for (int b = 0; b < a.rank_bits; ++b) {
                const uint32_t bit = (cid >> b) & 1u;
                const uint32_t bal = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bal : ~bal;
            }
#endif
        }
        uint32_t cur = 0;
        if (valid) cur = s_cur[lt];
        __syncwarp();
        if (valid) {
            a.list[cur + __popc(peers & lt_mask)] = s_pid;
            if ((peers >> lane) == 1u) s_cur[lt] = cur + __popc(peers);
        }
        __syncwarp();
    }
};
    for (uint32_t b = 0; b < nb || qn > 0;) {
        if (b < nb) {
            // enqueue this stage's records with pairs in the warp's rows
            const int st = (int)(b % kStages);
            mbar_wait(&s_full[st], (b / kStages) & 1);
            const uint4* rec = s_ring + st * kStageRec;
            const int n = (int)min((uint32_t)kStageRec, e - f - b * kStageRec);
            for (int q0 = 0; q0 < n; q0 += 32) {
                const int qi = q0 + lane;
                uint4 r = make_uint4(0, 0, 0, 0);
                if (qi < n) r = rec[qi];
                // the record's row-class mask (sort.cu); an item whose class rows all lie
                // outside this window is dropped later (class_pairs = 0 in expand_group)
                const int y0 = (int)(r.z >> 16), y1 = (int)(r.w >> 16);
                const bool rel = qi < n && ((r.x >> warp) & 1u) && y1 > R0 && y0 < R1;
                const uint32_t bal = __ballot_sync(0xffffffffu, rel);
                if (rel) s_q[warp][(qhead + qn + __popc(bal & lt_mask)) & (kQueue - 1)] = r;
                qn += __popc(bal);
                __syncwarp();
                if (qn >= 32) {  // expand a full group
                    expand_group(32);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[st]);
            ++b;
        } else {
            expand_group(min(qn, 32));
        }
    }
}

cudaError_t launch_bin(const BinArgs& a, cudaStream_t stream) {
    const int T = a.tiles_x * a.rows;
    const unsigned nwin = (unsigned)((a.rows + a.win_rows - 1) / a.win_rows);
    const dim3 grid((unsigned)std::max(1, a.cmax), std::max(1u, nwin));
    cudaError_t e;
    bin_count_kernel<<<grid, kBinThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    bin_colscan_kernel<<<(unsigned)((T + 31) / 32), kColThreads, 0, stream>>>(a);  // + the ranges (S3)
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int smem = kStages * kStageRec * 16;  // the record ring
    static int configured_dev[kMaxDevices] = {0};
    int& configured = configured_dev[current_device()];
    if (smem > configured) {
        if ((e = cudaFuncSetAttribute(bin_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) !=
            cudaSuccess)
            return e;
        configured = smem;
    }
    bin_scatter_kernel<<<grid, kScatThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
