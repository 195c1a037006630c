// bin.cu -- S2 pair generation and S3 ranges by direct tile binning
// (DESIGN.md "Sort").
//
// Input: the visible particles in (depth bits, index) order as packed item
// records (E = first pair slot, particle, x0|y0<<16, x1|y1<<16 of the R10
// rect; written by item_scan_kernel in sort.cu).  Output: the per-tile lists
// list[ranges[t] .. ranges[t+1]) in (depth bits, index) order -- exactly the
// order of a stable sort of the (tile << 32 | depth) keys -- without sorting
// any pair.
//
// The depth-ordered items are cut into chunks of equal cost, cost = pairs +
// kBinItemCost x items (the item scan records the first item of every chunk).  A tile's list is then the concatenation, in
// chunk order, of each chunk's items covering the tile, in item order:
//   bin_count     per (chunk, window of tile rows): per-tile counts of the
//                 chunk's items from a 2-D difference array of their rects in
//                 shared memory (4 atomics per item) -> table[t][chunk];
//   bin_colscan   one warp per tile: exclusive prefix of table[t][.] over the
//                 chunks, tile total -> ranges[t];
//   bin_tilescan  exclusive prefix of the tile totals -> ranges, M;
//   bin_scatter   per (chunk, window): cursors = ranges[t] + table[t][chunk]
//                 in shared memory; warp w owns the window's tile rows
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
constexpr int kBinStage = 256;               // item records staged per round
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
    for (uint32_t s = f + tid; s < e; s += kBinThreads) {
        int x0, y0, x1, y1;
        unpack_rect(__ldg(a.items + s), x0, y0, x1, y1);
        const int ya = max(y0, R0) - R0, yb = min(y1, R1) - R0;
        if (ya >= yb) continue;
        atomicAdd(&s_diff[ya * pitch + x0], 1);
        atomicAdd(&s_diff[ya * pitch + x1], -1);
        atomicAdd(&s_diff[yb * pitch + x0], -1);
        atomicAdd(&s_diff[yb * pitch + x1], 1);
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
    // prefix along y, one thread per column; table[t][c] (chunk-minor)
    for (int x = tid; x < tx; x += kBinThreads) {
        int run = 0;
        for (int y = 0; y < nr; ++y) {
            run += s_diff[y * pitch + x];
            a.table[(int64_t)((R0 + y) * tx + x) * a.cmax + c] = (uint32_t)run;
        }
    }
}

// One warp per tile: exclusive prefix of the tile's chunk counts (in place),
// the tile total into ranges[t].
__global__ void __launch_bounds__(kBinThreads) bin_colscan_kernel(BinArgs a) {
    const int64_t t = ((int64_t)blockIdx.x * kBinThreads + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t T = (int64_t)a.tiles_x * a.rows;
    if (t >= T || a.counters[GES_CTR_OVERFLOW]) return;
    const int C = (int)bin_chunks(a);
    uint32_t* col = a.table + t * a.cmax;
    uint32_t run = 0;
    for (int c0 = 0; c0 < C; c0 += 128) {
        uint32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + 32 * u + lane;
            v[u] = c < C ? col[c] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + 32 * u + lane;
            uint32_t incl = v[u];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += nn;
            }
            if (c < C) col[c] = run + incl - v[u];
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    if (lane == 0) a.ranges[t] = run;
}

// One CTA: exclusive prefix of the tile totals -> ranges[0..T], M.
constexpr int kTileScanThreads = 1024;
__global__ void __launch_bounds__(kTileScanThreads) bin_tilescan_kernel(BinArgs a) {
    __shared__ uint32_t s_warp[kTileScanThreads / 32 + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = a.tiles_x * a.rows;
    if (a.counters[GES_CTR_OVERFLOW]) {
        for (int t = tid; t <= T; t += kTileScanThreads) a.ranges[t] = 0;
        if (tid == 0) a.counters_w[GES_CTR_PAIRS] = 0;
        return;
    }
    const int per = (T + kTileScanThreads - 1) / kTileScanThreads;
    const int t0 = min(T, tid * per), t1 = min(T, t0 + per);
    uint32_t sum = 0;
    for (int t = t0; t < t1; ++t) sum += a.ranges[t];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t wv = s_warp[lane];
        uint32_t wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += nn;
        }
        s_warp[lane] = wi - wv;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    uint32_t run = s_warp[warp] + incl - sum;
    for (int t = t0; t < t1; ++t) {
        const uint32_t v = a.ranges[t];
        a.ranges[t] = run;
        run += v;
    }
    if (tid == 0) {
        a.ranges[T] = s_warp[32];
        a.counters_w[GES_CTR_PAIRS] = s_warp[32];
    }
}

// Item q of the staged batch has rows of the warp's class w (ly = w mod 8)
// inside the window: its pair count there, packed geometry (x0, w - 1, first
// row of the class) and particle.
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

__global__ void __launch_bounds__(kBinThreads) bin_scatter_kernel(BinArgs a) {
    __shared__ uint32_t s_cur[kBinWinTiles];
    __shared__ uint8_t s_own[kBinWinTiles];
    __shared__ uint4 s_rec[kBinStage];
    __shared__ uint8_t s_idx[kBinWarps][kBinStage];
    if (a.counters[GES_CTR_OVERFLOW]) return;
    const int64_t c = blockIdx.x;
    if (c >= bin_chunks(a)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int R0 = (int)blockIdx.y * a.win_rows, R1 = min(a.rows, R0 + a.win_rows);
    const int tx = a.tiles_x, wt = (R1 - R0) * tx;
    const int64_t tbase = (int64_t)R0 * tx;
    for (int i = tid; i < wt; i += kBinThreads) s_cur[i] = a.ranges[tbase + i] + a.table[(tbase + i) * a.cmax + c];
    const uint32_t f = a.chunk_first[c], e = a.chunk_first[c + 1];
    for (uint32_t b0 = f; b0 < e; b0 += kBinStage) {
        const int n = (int)min((uint32_t)kBinStage, e - b0);
        __syncthreads();  // previous records consumed (and the cursors written, first time)
        for (int i = tid; i < n; i += kBinThreads) s_rec[i] = __ldg(a.items + b0 + i);
        __syncthreads();
        // the batch's items with pairs in this warp's rows, in item order
        int nrel = 0;
        for (int q0 = 0; q0 < n; q0 += 32) {
            const int q = q0 + lane;
            uint32_t geo;
            const bool rel = q < n && class_pairs(s_rec[q], R0, R1, warp, geo) != 0u;
            const uint32_t bal = __ballot_sync(0xffffffffu, rel);
            if (rel) s_idx[warp][nrel + __popc(bal & lt_mask)] = (uint8_t)q;
            nrel += __popc(bal);
        }
        __syncwarp();
        for (int g0 = 0; g0 < nrel; g0 += 32) {
            // this lane's item: its pairs in the warp's rows
            uint32_t cnt = 0, geo = 0, pid = 0;
            if (g0 + lane < nrel) {
                const uint4 r = s_rec[s_idx[warp][g0 + lane]];
                cnt = class_pairs(r, R0, R1, warp, geo);
                pid = r.y;
            }
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += nn;
            }
            const uint32_t excl = incl - cnt;
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            for (uint32_t base = 0; base < total; base += 32) {
                const uint32_t gi = base + lane;
                const bool valid = gi < total;
                // source lane = number of lanes whose inclusive count is <= gi
                int src = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const uint32_t v = __shfl_sync(0xffffffffu, incl, src + step - 1);
                    if (v <= gi) src += step;
                }
                const uint32_t s_excl = __shfl_sync(0xffffffffu, excl, src);
                const uint32_t s_geo = __shfl_sync(0xffffffffu, geo, src);
                const uint32_t s_pid = __shfl_sync(0xffffffffu, pid, src);
                const uint32_t k = gi - s_excl;
                const uint32_t w = ((s_geo >> 8) & 255u) + 1u;
                // k / w exactly: k < 32 w, w <= 256 (quotient <= 31, far from rounding trouble)
                const uint32_t ri = __float2uint_rz(((float)k + 0.5f) * __frcp_rn((float)w));
                const uint32_t xx = k - ri * w;
                const uint32_t ly = (s_geo >> 16) + 8u * ri;
                const uint32_t lt = ly * (uint32_t)tx + (s_geo & 255u) + xx;
                // lanes of this round that hit the same tile: ranked in lane order
                if (valid) s_own[lt] = (uint8_t)lane;
                __syncwarp();
                const bool lost = valid && s_own[lt] != (uint8_t)lane;
                uint32_t peers = 1u << lane;
                if (__any_sync(0xffffffffu, lost)) {
                    const uint32_t cid = (ly >> 3) * (uint32_t)tx + (s_geo & 255u) + xx;
                    peers = __ballot_sync(0xffffffffu, valid);
                    for (int b = 0; b < a.rank_bits; ++b) {
                        const uint32_t bit = (cid >> b) & 1u;
                        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
                        peers &= bit ? bal : ~bal;
                    }
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
    bin_colscan_kernel<<<(unsigned)((T * 32 + kBinThreads - 1) / kBinThreads), kBinThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    bin_tilescan_kernel<<<1, kTileScanThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    bin_scatter_kernel<<<grid, kBinThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
