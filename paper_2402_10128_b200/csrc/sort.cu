// sort.cu -- S2/S3: depth radix sort of the visible
// particles, generation of the (tile, particle) pairs in depth order (every
// tile of each particle's R10 rect), stable radix sort of the pairs by tile id,
// per-tile ranges.
//
// Design: instead of a 64-bit LSD sort of
// (tile_id << 32 | depth) keys (6 x 8-bit passes over all pairs), the depth
// order is established once on the V visible particles (4 passes over
// V << M; pass 0 also compacts the visible set), then the pairs are generated
// in that order and sorted STABLY by tile id alone (2 passes for <= 65536
// tiles): every tile's list comes out in (depth bits, particle index) order --
// exactly the order of the 64-bit keys.
//   item scan   exclusive prefix E[s] of the rect areas of the sorted particles
//               (decoupled look-back), packed item records, the particle that
//               holds the first slot of each 4096-slot tile, the slot count;
//   pass 1      each CTA owns 4096 consecutive pair SLOTS (balanced however
//               unequal the footprints are), stages the particles covering
//               them in shared memory, expands its slots by a load-balanced
//               search, ranks and scatters them by the low tile digit -- no unsorted pair array is ever written;
//   pass 2      the high tile digit;
//   ranges      the boundaries of the sorted tile ids.
// Each pass is reduce-then-scan (per-tile digit histograms, one column scan
// per digit, scatter): no CTA ever waits for another.  Ranking is a warp
// multisplit with one ballot per digit bit.  Hand-written; no CUB.
#include <algorithm>

#include "ges_internal.h"
#include "ges_scan.cuh"

namespace ges {

constexpr int kSlotTile = 4096;  // pair slots per CTA == radix tile

// ---------------------------------------------------------------------------
// Item scan
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

int64_t item_scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }
int64_t slot_tiles(int64_t cap) { return (cap + kSlotTile - 1) / kSlotTile + 2; }

__device__ __forceinline__ uint32_t rect_count(ushort4 r) { return (uint32_t)(r.z - r.x) * (uint32_t)(r.w - r.y); }

__global__ void __launch_bounds__(kScanThreads) item_scan_kernel(ItemScanArgs a) {
    __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
    __shared__ uint32_t s_tile, s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
    if (V == 0) {
        if (blockIdx.x == 0 && tid == 0) a.counters[GES_CTR_SLOTS] = 0;
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
            // slot tiles whose first slot lies in [e, e + c)
            for (uint32_t st = (e + kSlotTile - 1) / kSlotTile; st * (uint64_t)kSlotTile < (uint64_t)e + c[j]; ++st)
                a.tile_first[st] = (uint32_t)s;
            if (s == V - 1) {  // total pair slots, capacity check
                const uint64_t slots = (uint64_t)e + c[j];
                a.counters[GES_CTR_SLOTS] = slots;
                a.counters[GES_CTR_OVERFLOW] = (int64_t)slots > a.capacity ? 1ull : 0ull;
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
// LSD radix passes, reduce-then-scan (no inter-CTA waiting):
//   radix_hist_kernel     per 4096-key tile: digit histogram -> H[d][tile]
//   radix_scan_kernel     per digit: exclusive scan of H[d][.] over the tiles,
//                         column total -> T[d]
//   radix_scatter_kernel  per tile: stable warp-multisplit ranking, shared-memory
//                         reorder, scatter to off(d) + H[d][tile] + local rank
// GEN = true: a tile's keys (ty << 8 | tx) and values (particle ids) are
// generated from the depth-sorted particles (load-balanced search over pair
// slots); its digit is the tile column tx, whose histogram gen_hist_kernel
// computes from the items alone.
// ---------------------------------------------------------------------------
constexpr int kRadixThreads = 256;
#ifndef GES_SCAT_MINB  // tuning knob: min resident CTAs per SM for the scatter kernels
#define GES_SCAT_MINB 3
#endif
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr uint32_t kInvalidKey = 0xffffffffu;
static_assert(kRadixTile == kSlotTile, "slot tiles are radix tiles");

int64_t radix_tiles(int64_t n) { return (n + kRadixTile - 1) / kRadixTile; }

// Particles covering a CTA's 4096 slots are staged in shared memory when
// there are at most kStageMax of them (the common case: a particle touches
// ~20 tiles); tiles of many tiny particles read them from L2 instead.
constexpr int kStageMax = 1024;
struct GenSmem {
    uint32_t E[kStageMax];
    uint32_t pid[kStageMax];
    ushort4 rect[kStageMax];
};

__device__ __forceinline__ int64_t pass_count(const RadixPassArgs& a) {
    return a.count ? min((int64_t)*a.count, a.max_items) : a.max_items;
}

// Loads (or generates) the tile's keys/values in warp-striped order: item j of
// lane l of warp w is element w*512 + j*32 + l of the tile.  valid bit j marks
// items that take part.
template <bool GEN>
__device__ __forceinline__ void load_tile(const RadixPassArgs& a, int64_t tile, int64_t n,
                                          uint32_t (&k)[kRadixItems], uint32_t (&v)[kRadixItems], uint32_t& valid,
                                          uint32_t* s_keys, uint32_t* s_vals, unsigned char* s_dyn,
                                          bool need_vals) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = tile * kRadixTile + warp * (kRadixItems * 32);
    valid = 0;
    if constexpr (GEN) {
        GenSmem& g = *reinterpret_cast<GenSmem*>(s_dyn);
        const int64_t slot0 = tile * kRadixTile;
        const int nslots = (int)min((int64_t)kRadixTile, n - slot0);
        const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
        const int64_t f = a.tile_first[tile];
        const int64_t last_item = (slot0 + kRadixTile < n) ? (int64_t)a.tile_first[tile + 1] : V - 1;
        const int nit = (int)(last_item - f + 1);
        const bool staged = nit <= kStageMax;
        if (staged) {
            constexpr int kU = kStageMax / kRadixThreads;
            uint4 rec[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int q = tid + u * kRadixThreads;
                if (q < nit) rec[u] = __ldg(a.items + f + q);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int q = tid + u * kRadixThreads;
                if (q < nit) {
                    g.E[q] = rec[u].x;
                    g.pid[q] = rec[u].y;
                    g.rect[q] = make_ushort4((uint16_t)(rec[u].z & 0xffffu), (uint16_t)(rec[u].z >> 16),
                                             (uint16_t)(rec[u].w & 0xffffu), (uint16_t)(rec[u].w >> 16));
                }
            }
        }
        __syncthreads();
        auto itemE = [&](int q) -> uint32_t { return staged ? g.E[q] : __ldg(a.E + f + q); };
        auto itemPid = [&](int q) -> uint32_t { return staged ? g.pid[q] : __ldg(a.sorted_vis + f + q); };
        auto itemRect = [&](int q) -> ushort4 { return staged ? g.rect[q] : __ldg(a.rect + itemPid(q)); };
        // thread-contiguous slots, then an exchange to the warp-striped order
        const int ls0 = tid * kRadixItems;
        int it = 0;
        if (ls0 < nslots) {
            const uint32_t s0 = (uint32_t)(slot0 + ls0);
            int lo = 0, hi = nit - 1;  // last item with E <= s0
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (itemE(mid) <= s0) lo = mid; else hi = mid - 1;
            }
            it = lo;
        }
        // walk the thread's 16 consecutive slots: one division per item start, then
        // the tile advances along the rect's rows incrementally
        ushort4 r = itemRect(it);
        uint32_t pid = itemPid(it), E1 = (it + 1 < nit) ? itemE(it + 1) : 0xffffffffu;
        uint32_t w = r.z - r.x;
        uint32_t xx = 0, yy = 0;
        if (ls0 < nslots) {
            const uint32_t li = (uint32_t)(slot0 + ls0) - itemE(it);
            // li / w exactly: the quotient is < 2^16, far from rounding trouble
            yy = __float2uint_rz(((float)li + 0.5f) * __fdividef(1.0f, (float)w));
            xx = li - yy * w;
        }
#pragma unroll
        for (int j = 0; j < kRadixItems; ++j) {
            const int ls = ls0 + j;
            const uint32_t s = (uint32_t)(slot0 + ls);
            if (ls < nslots) {
                if (s >= E1) {  // next item(s); items are never empty
                    do {
                        ++it;
                        E1 = (it + 1 < nit) ? itemE(it + 1) : 0xffffffffu;
                    } while (s >= E1);
                    r = itemRect(it);
                    pid = itemPid(it);
                    w = r.z - r.x;
                    xx = 0;
                    yy = 0;
                }
                const uint32_t tx = r.x + xx, ty = r.y + yy;
                const uint32_t key = (ty << 8) | tx;
                const int pad = ls + (ls >> 5);  // +1 word per 32: conflict-free both ways
                s_keys[pad] = key;
                s_vals[pad] = pid;
                if (++xx == w) { xx = 0; ++yy; }
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kRadixItems; ++j) {
            const int ls = warp * (kRadixItems * 32) + j * 32 + lane;
            if (ls < nslots) {
                const int pad = ls + (ls >> 5);
                k[j] = s_keys[pad];
                if (need_vals) v[j] = s_vals[pad];
                valid |= 1u << j;
            }
        }
        __syncthreads();
    } else {
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
}

template <bool GEN>
__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(RadixPassArgs a) {
    __shared__ uint32_t s_keys[GEN ? kRadixTile + kRadixTile / 32 : 1];
    __shared__ uint32_t s_vals[GEN ? kRadixTile + kRadixTile / 32 : 1];
    __shared__ uint32_t s_hist[kRadixDigits];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    if (a.overflow && *a.overflow) return;
    const int64_t n = pass_count(a);
    const int64_t tile = blockIdx.x;
    if (tile * kRadixTile >= n) return;
    s_hist[threadIdx.x] = 0;
    uint32_t k[kRadixItems], v[kRadixItems], valid;
    load_tile<GEN>(a, tile, n, k, v, valid, s_keys, s_vals, s_dyn, false);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRadixItems; ++j)
        if (valid & (1u << j)) atomicAdd(&s_hist[(k[j] >> a.shift) & 255u], 1u);
    __syncthreads();
    a.tile_hist[(int64_t)threadIdx.x * a.hist_stride + tile] = s_hist[threadIdx.x];
}

// GEN pass histogram without generating the pairs: the digit of a pair is
// its tile column tx, so the slots an item holds inside this CTA's 4096-slot
// window add +1 over column ranges -- at most three range updates per item
// (partial first row, full rows, partial last row) in a 257-entry difference
// array -- followed by a prefix sum over the 256 columns.
__global__ void __launch_bounds__(kRadixThreads) gen_hist_kernel(RadixPassArgs a) {
    __shared__ int s_diff[kRadixDigits + 1];
    __shared__ int s_warp[kRadixWarps];
    if (a.overflow && *a.overflow) return;
    const int64_t n = pass_count(a);
    const int64_t tile = blockIdx.x;
    if (tile * kRadixTile >= n) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    s_diff[tid] = 0;
    if (tid == 0) s_diff[kRadixDigits] = 0;
    __syncthreads();
    const int64_t slot0 = tile * kRadixTile, slot1 = min(slot0 + kRadixTile, n);
    const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
    const int64_t f = a.tile_first[tile];
    const int64_t last_item = (slot1 < n) ? (int64_t)a.tile_first[tile + 1] : V - 1;
    for (int64_t q = f + tid; q <= last_item; q += kRadixThreads) {
        const uint4 rec = __ldg(a.items + q);
        const int x0 = (int)(rec.z & 0xffffu), y0 = (int)(rec.z >> 16);
        const int x1 = (int)(rec.w & 0xffffu), y1 = (int)(rec.w >> 16);
        const int64_t e0 = rec.x;
        const uint32_t w = (uint32_t)(x1 - x0), area = w * (uint32_t)(y1 - y0);
        const int64_t lo = max(slot0, e0) - e0, hi = min(slot1, e0 + (int64_t)area) - e0;  // slots [lo, hi) of the item
        if (lo >= hi) continue;
        const uint32_t ra = (uint32_t)lo / w, ca = (uint32_t)lo - ra * w;
        const uint32_t rb = (uint32_t)hi / w, cb = (uint32_t)hi - rb * w;
        if (ra == rb) {
            atomicAdd(&s_diff[x0 + ca], 1); atomicAdd(&s_diff[x0 + cb], -1);
        } else {
            atomicAdd(&s_diff[x0 + ca], 1); atomicAdd(&s_diff[x1], -1);          // row ra from column ca
            if (rb > ra + 1) { atomicAdd(&s_diff[x0], (int)(rb - ra - 1)); atomicAdd(&s_diff[x1], -(int)(rb - ra - 1)); }
            if (cb > 0) { atomicAdd(&s_diff[x0], 1); atomicAdd(&s_diff[x0 + cb], -1); }  // row rb up to cb
        }
    }
    __syncthreads();
    // inclusive prefix over the columns
    const int d = s_diff[tid];
    int incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int base = 0;
    for (int w2 = 0; w2 < warp; ++w2) base += s_warp[w2];
    a.tile_hist[(int64_t)tid * a.hist_stride + tile] = (uint32_t)(base + incl);
}

// One CTA per digit: exclusive scan of H[d][.] over the tiles (in place).
__global__ void __launch_bounds__(256) radix_scan_kernel(RadixPassArgs a) {
    __shared__ uint32_t s_warp[9];
    const int d = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.overflow && *a.overflow) return;
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

template <bool GEN>
__global__ void __launch_bounds__(kRadixThreads, GES_SCAT_MINB) radix_scatter_kernel(RadixPassArgs a) {
    __shared__ uint32_t s_keys[kRadixTile + kRadixTile / 32];
    __shared__ uint32_t s_vals[kRadixTile + kRadixTile / 32];
    __shared__ uint32_t s_whist[kRadixWarps][kRadixDigits];
    __shared__ uint32_t s_local[kRadixDigits];
    __shared__ uint32_t s_global[kRadixDigits];
    __shared__ uint32_t s_warp[kRadixWarps + 1];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    if (a.overflow && *a.overflow) return;
    const int64_t n = pass_count(a);
    const int64_t tile = blockIdx.x;
    if (tile * kRadixTile >= n) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // keys first: their loads overlap the offset computation below
    uint32_t k[kRadixItems], v[kRadixItems], rank[kRadixItems], valid;
    load_tile<GEN>(a, tile, n, k, v, valid, s_keys, s_vals, s_dyn, true);
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
    if (a.gen) {
        static bool configured = false;
        if (!configured) {
            cudaFuncSetAttribute(radix_scatter_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(GenSmem));
            configured = true;
        }
        gen_hist_kernel<<<grid, kRadixThreads, 0, stream>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        radix_scan_kernel<<<kRadixDigits, 256, 0, stream>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        radix_scatter_kernel<true><<<grid, kRadixThreads, sizeof(GenSmem), stream>>>(a);
    } else {
        radix_hist_kernel<false><<<grid, kRadixThreads, 0, stream>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        radix_scan_kernel<<<kRadixDigits, 256, 0, stream>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        radix_scatter_kernel<false><<<grid, kRadixThreads, 0, stream>>>(a);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// S3: per-tile ranges from the sorted tile ids
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ranges_kernel(RangesArgs a) {
    const int T = a.tiles_x * a.tiles_y;
    if (a.counters[GES_CTR_OVERFLOW]) {
        for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= T; t += gridDim.x * blockDim.x) a.ranges[t] = 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) a.counters[GES_CTR_PAIRS] = 0;
        return;
    }
    const uint32_t M = (uint32_t)min((int64_t)a.counters[GES_CTR_SLOTS], a.max_pairs);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.counters[GES_CTR_PAIRS] = M;
    // entry m opens every tile in (tile[m-1], tile[m]]; the end closes (tile[M-1], T];
    // tile(key) = ty * tiles_x + tx for key = ty << 8 | tx (monotone in the key)
    auto tile_of = [&](uint32_t k) { return (int)(k >> 8) * a.tiles_x + (int)(k & 255u); };
    // four entries per thread (one 16-B load) plus the entry before them
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 4 * g <= (int64_t)M;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m0 = 4 * g;
        uint32_t k[4];
        if (m0 + 4 <= (int64_t)M) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(a.keys + m0));
            k[0] = q.x; k[1] = q.y; k[2] = q.z; k[3] = q.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) k[j] = (m0 + j < (int64_t)M) ? __ldg(a.keys + m0 + j) : 0u;
        }
        int prev = m0 > 0 ? tile_of(__ldg(a.keys + m0 - 1)) : -1;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t m = m0 + j;
            if (m > (int64_t)M) break;
            const int cur = m < (int64_t)M ? tile_of(k[j]) : T;
            for (int t = prev + 1; t <= cur; ++t) a.ranges[t] = (uint32_t)m;
            prev = cur;
        }
    }
}

cudaError_t launch_ranges(const RangesArgs& a, cudaStream_t stream) {
    const int grid = std::max(1, std::min(num_sms() * 8, (int)((a.max_pairs / 4 + 256) / 256)));
    ranges_kernel<<<grid, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
