// sort.cu -- S2: depth radix sort of the visible particles
// and the item scan that turns the depth-sorted particles into pair slots.
//
// Design: instead of a 64-bit LSD sort of
// (tile_id << 32 | depth) keys over all pairs, the depth order is established
// once on the V visible particles (4 LSD passes over V << M; pass 0 also
// compacts the visible set), then bin.cu writes every tile's list directly in
// that order -- exactly the order of the 64-bit keys.
//   depth passes  reduce-then-scan (per-tile digit histograms, one column scan
//                 per digit, scatter): no CTA ever waits for another; ranking
//                 is a warp multisplit with one ballot per digit bit;
//   item scan     exclusive prefix E[s] of the rect areas of the sorted
//                 particles (decoupled look-back), packed item records, the
//                 first item of every binning chunk, the slot count M.
// Hand-written; no CUB.
#include <algorithm>

#include "ges_internal.h"
#include "ges_scan.cuh"

namespace ges {

// ---------------------------------------------------------------------------
// Item scan
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

int64_t item_scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }
constexpr uint64_t kItemCost = kBinItemCost;

__device__ __forceinline__ uint32_t rect_count(ushort4 r) { return (uint32_t)(r.z - r.x) * (uint32_t)(r.w - r.y); }

__global__ void __launch_bounds__(kScanThreads) item_scan_kernel(ItemScanArgs a) {
    __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
    __shared__ uint32_t s_tile, s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
    if (V == 0) {
        if (blockIdx.x == 0 && tid == 0) { a.counters[GES_CTR_SLOTS] = 0; a.counters[GES_CTR_CHUNKS] = 0; }
        return;
    }
    if (tid == 0) s_tile = (uint32_t)atomicAdd(a.tile_counter, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile * kScanTile >= V) return;  // tickets are ordered: nobody waits on this one
    const int64_t first = tile * kScanTile + (int64_t)tid * kScanItems;
    uint32_t c[kScanItems], ids[kScanItems];
    ushort4 rc[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) ids[j] = (first + j < V) ? __ldg(a.sorted_vis + first + j) : 0u;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) rc[j] = (first + j < V) ? __ldg(a.rect + ids[j]) : make_ushort4(0, 0, 0, 0);
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) { c[j] = rect_count(rc[j]); sum += c[j]; }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t wv = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
        uint32_t wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += nn;
        }
        if (lane < kScanThreads / 32) s_warp[lane] = wi - wv;
        const uint32_t total = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
        const uint32_t prefix = lookback_warp(a.lookback, (uint32_t)tile, total);
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    uint32_t e = s_prefix + s_warp[warp] + incl - sum;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t s = first + j;
        if (s < V) {
            a.E[s] = e;
            // packed item record for the pair expansion: one coalesced 16-B load there
            a.items[s] = make_uint4(e, ids[j], (uint32_t)rc[j].x | ((uint32_t)rc[j].y << 16),
                                    (uint32_t)rc[j].z | ((uint32_t)rc[j].w << 16));
            // binning chunk k = the items whose cost W[s] = E[s] + kItemCost s lies in
            // [k S, (k+1) S) (a pair costs 1, an item kItemCost: bin.cu's work per
            // item), i.e. chunk_first[k] = min{s : W[s] >= k S}; item s + 1 is that
            // minimum for every k with k S in (W[s], W[s+1]].  Item 0 opens chunk 0.
            const uint64_t S = (uint64_t)a.chunk_slots, e1 = (uint64_t)e + c[j];
            const uint64_t w0 = (uint64_t)e + kItemCost * (uint64_t)s, w1 = e1 + kItemCost * (uint64_t)(s + 1);
            const bool ovf = (int64_t)e1 > a.capacity;
            if (s == 0) a.chunk_first[0] = 0;
            if (!ovf)
                for (uint64_t k = w0 / S + 1; k * S <= w1; ++k) a.chunk_first[k] = (uint32_t)(s + 1);
            if (s == V - 1) {  // total pair slots, capacity check, chunk count and closing entry
                a.counters[GES_CTR_SLOTS] = e1;
                a.counters[GES_CTR_OVERFLOW] = ovf ? 1ull : 0ull;
                const uint64_t C = (w1 + S - 1) / S;
                a.counters[GES_CTR_CHUNKS] = ovf ? 0ull : C;
                if (!ovf) a.chunk_first[C] = (uint32_t)V;
            }
        }
        e += c[j];
    }
}

cudaError_t launch_item_scan(const ItemScanArgs& a, int64_t max_items, cudaStream_t stream) {
    const int64_t grid = std::max<int64_t>(1, item_scan_tiles(max_items));
    item_scan_kernel<<<(unsigned)grid, kScanThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// LSD radix passes of the depth sort, reduce-then-scan (no inter-CTA waiting):
//   radix_hist_kernel     per 4096-key tile: digit histogram -> H[d][tile]
//   radix_scan_kernel     per digit: exclusive scan of H[d][.] over the tiles,
//                         column total -> T[d]
//   radix_scatter_kernel  per tile: stable warp-multisplit ranking, shared-memory
//                         reorder, scatter to off(d) + H[d][tile] + local rank
// ---------------------------------------------------------------------------
constexpr int kRadixThreads = 256;
#ifndef GES_SCAT_MINB  // tuning knob: min resident CTAs per SM for the scatter kernels
#define GES_SCAT_MINB 3
#endif
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr uint32_t kInvalidKey = 0xffffffffu;

int64_t radix_tiles(int64_t n) { return (n + kRadixTile - 1) / kRadixTile; }

__device__ __forceinline__ int64_t pass_count(const RadixPassArgs& a) {
    return a.count ? min((int64_t)*a.count, a.max_items) : a.max_items;
}

// Loads the tile's keys/values in warp-striped order: item j of lane l of
// warp w is element w*512 + j*32 + l of the tile.  valid bit j marks items
// that take part.
__device__ __forceinline__ void load_tile(const RadixPassArgs& a, int64_t tile, int64_t n,
                                          uint32_t (&k)[kRadixItems], uint32_t (&v)[kRadixItems], uint32_t& valid,
                                          bool need_vals) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = tile * kRadixTile + warp * (kRadixItems * 32);
    valid = 0;
    // issue every load before any use (all in flight together)
#pragma unroll
    for (int j = 0; j < kRadixItems; ++j) {
        const int64_t idx = base + j * 32 + lane;
        k[j] = (idx < n) ? __ldg(a.keys_in + idx) : kInvalidKey;
    }
    if (need_vals) {
        if (a.vals_in) {
#pragma unroll
            for (int j = 0; j < kRadixItems; ++j) {
                const int64_t idx = base + j * 32 + lane;
                v[j] = (idx < n) ? __ldg(a.vals_in + idx) : 0u;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kRadixItems; ++j) v[j] = (uint32_t)(base + j * 32 + lane);
        }
    }
#pragma unroll
    for (int j = 0; j < kRadixItems; ++j) {
        const int64_t idx = base + j * 32 + lane;
        if (idx < n && !(a.drop_invalid && k[j] == kInvalidKey)) valid |= 1u << j;
    }
}

__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(RadixPassArgs a) {
    __shared__ uint32_t s_hist[kRadixDigits];
    const int64_t n = pass_count(a);
    const int64_t tile = blockIdx.x;
    if (tile * kRadixTile >= n) return;
    s_hist[threadIdx.x] = 0;
    uint32_t k[kRadixItems], v[kRadixItems], valid;
    load_tile(a, tile, n, k, v, valid, false);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRadixItems; ++j)
        if (valid & (1u << j)) atomicAdd(&s_hist[(k[j] >> a.shift) & 255u], 1u);
    __syncthreads();
    a.tile_hist[(int64_t)threadIdx.x * a.hist_stride + tile] = s_hist[threadIdx.x];
}

// One CTA per digit: exclusive scan of H[d][.] over the tiles (in place).
__global__ void __launch_bounds__(256) radix_scan_kernel(RadixPassArgs a) {
    __shared__ uint32_t s_warp[9];
    const int d = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = pass_count(a);
    const int nt = (int)((n + kRadixTile - 1) / kRadixTile);
    const int per = (nt + 255) / 256;
    const int t0 = min(nt, tid * per), t1 = min(nt, t0 + per);
    uint32_t* col = a.tile_hist + (int64_t)d * a.hist_stride;  // digit-major: contiguous over tiles
    uint32_t sum = 0;
    for (int t = t0; t < t1; ++t) sum += col[t];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        uint32_t r = 0;
        for (int w = 0; w < 8; ++w) { const uint32_t c = s_warp[w]; s_warp[w] = r; r += c; }
        s_warp[8] = r;
    }
    __syncthreads();
    uint32_t run = s_warp[warp] + incl - sum;
    for (int t = t0; t < t1; ++t) {
        const uint32_t c = col[t];
        col[t] = run;
        run += c;
    }
    if (tid == 0) a.digit_total[d] = s_warp[8];
}

__global__ void __launch_bounds__(kRadixThreads, GES_SCAT_MINB) radix_scatter_kernel(RadixPassArgs a) {
    __shared__ uint32_t s_keys[kRadixTile];
    __shared__ uint32_t s_vals[kRadixTile];
    __shared__ uint32_t s_whist[kRadixWarps][kRadixDigits];
    __shared__ uint32_t s_local[kRadixDigits];
    __shared__ uint32_t s_global[kRadixDigits];
    __shared__ uint32_t s_warp[kRadixWarps + 1];
    const int64_t n = pass_count(a);
    const int64_t tile = blockIdx.x;
    if (tile * kRadixTile >= n) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // keys first: their loads overlap the offset computation below
    uint32_t k[kRadixItems], v[kRadixItems], rank[kRadixItems], valid;
    load_tile(a, tile, n, k, v, valid, true);
    for (int d = tid; d < kRadixWarps * kRadixDigits; d += kRadixThreads) (&s_whist[0][0])[d] = 0;
    // global digit offsets: exclusive scan of the column totals + this tile's prefix
    {
        const uint32_t tot = a.digit_total[tid];
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += nn;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (tid == 0) {
            uint32_t r = 0;
            for (int w = 0; w < kRadixWarps; ++w) { const uint32_t c = s_warp[w]; s_warp[w] = r; r += c; }
        }
        __syncthreads();
        s_global[tid] = s_warp[warp] + incl - tot + a.tile_hist[(int64_t)tid * a.hist_stride + tile];
        __syncthreads();
    }
    // warp multisplit ranking, items in (j, lane) = index order.  The lanes
    // holding the same digit are found with one ballot per digit bit (only the
    // bits this pass can hold), which issues at full rate, unlike MATCH.
    const int nbits = a.digit_bits;
#pragma unroll
    for (int j = 0; j < kRadixItems; ++j) {
        const bool ok = (valid >> j) & 1u;
        const uint32_t d = (k[j] >> a.shift) & 255u;
        uint32_t peers = __ballot_sync(0xffffffffu, ok);
        for (int b = 0; b < nbits; ++b) {
            const uint32_t bit = (d >> b) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
        uint32_t cnt = 0;
        if (ok) cnt = s_whist[warp][d];
        __syncwarp();
        rank[j] = cnt + __popc(peers & lt_mask);
        if (ok && (peers >> lane) == 1u) s_whist[warp][d] = cnt + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive over warps, block total; block-local exclusive scan
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
        const uint32_t c = s_whist[w][tid];
        s_whist[w][tid] = tot;
        tot += c;
    }
    {
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += nn;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (tid == 0) {
            uint32_t r = 0;
            for (int w = 0; w < kRadixWarps; ++w) { const uint32_t c = s_warp[w]; s_warp[w] = r; r += c; }
            s_warp[kRadixWarps] = r;
        }
        __syncthreads();
        s_local[tid] = s_warp[warp] + incl - tot;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRadixItems; ++j) {
        if ((valid >> j) & 1u) {
            const uint32_t dd = (k[j] >> a.shift) & 255u;
            const uint32_t pos = s_local[dd] + s_whist[warp][dd] + rank[j];
            s_keys[pos] = k[j];
            s_vals[pos] = v[j];
        }
    }
    __syncthreads();
    const int nvalid = (int)s_warp[kRadixWarps];
    for (int s = tid; s < nvalid; s += kRadixThreads) {
        const uint32_t key = s_keys[s];
        const uint32_t dd = (key >> a.shift) & 255u;
        const uint32_t out = s_global[dd] + (uint32_t)s - s_local[dd];
        if (a.keys_out) a.keys_out[out] = key;
        a.vals_out[out] = s_vals[s];
    }
}

cudaError_t launch_radix_pass(const RadixPassArgs& a, cudaStream_t stream) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, radix_tiles(a.max_items));
    cudaError_t e;
    radix_hist_kernel<<<grid, kRadixThreads, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    radix_scan_kernel<<<kRadixDigits, 256, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    radix_scatter_kernel<<<grid, kRadixThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
