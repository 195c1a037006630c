// sort.cu -- S2/S3: per-tile ranges, depth radix sort of
// the visible particles, (tile, particle) duplication in depth order, and the
// stable radix sort of the pairs by tile id.
//
// Design: instead of a 64-bit LSD sort of
// (tile_id << 32 | depth) keys (6 x 8-bit passes over M pairs), the depth order
// is established once on the V visible particles (4 passes over V << M), the
// pairs are emitted in that order, and a STABLE sort on the tile id alone (2
// passes over M for <= 65536 tiles) yields exactly the (tile, depth, index)
// order of the 64-bit keys.  The per-tile pair counts -- hence the ranges and
// the tile-digit histograms -- come from a 2-D difference grid of the rects
// built in S1, so no pass over the pairs is spent on counting.
//
// Every pass is a single-pass "onesweep" LSD step: 4096 keys per CTA,
// warp-level multisplit ranking with __match_any_sync, decoupled look-back
// across CTAs per digit, reordering through shared memory for coalesced
// scatter.  Hand-written; no CUB.
#include <algorithm>

#include "ges_internal.h"
#include "ges_scan.cuh"

namespace ges {

// ---------------------------------------------------------------------------
// S3: ranges and digit offsets (one CTA)
// ---------------------------------------------------------------------------
constexpr int kRangesThreads = 1024;

__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t v, uint32_t* s_warp, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_warp[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += n;
        }
        s_warp[lane] = wi - w;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    const uint32_t res = s_warp[warp] + incl - v;
    total = s_warp[32];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kRangesThreads) ranges_kernel(RangesArgs a) {
    extern __shared__ int32_t s_grid[];  // (tiles_y + 1) x (tiles_x + 1)
    __shared__ uint32_t s_warp[33];
    __shared__ uint32_t s_th[2][256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = a.tiles_x, ty = a.tiles_y, sx = tx + 1;
    const int G = sx * (ty + 1);
    for (int k = tid; k < 512; k += kRangesThreads) (&s_th[0][0])[k] = 0;
    for (int k = tid; k < G; k += kRangesThreads) s_grid[k] = a.tile_diff[k];
    __syncthreads();
    // 2-D prefix sum of the difference grid: rows (warp per row), then columns
    for (int y = warp; y <= ty; y += kRangesThreads / 32) {
        int32_t carry = 0;
        for (int x0 = 0; x0 <= tx; x0 += 32) {
            const int x = x0 + lane;
            int32_t v = (x <= tx) ? s_grid[y * sx + x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t nn = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += nn;
            }
            if (x <= tx) s_grid[y * sx + x] = v + carry;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    for (int x = warp; x <= tx; x += kRangesThreads / 32) {
        int32_t carry = 0;
        for (int y0 = 0; y0 <= ty; y0 += 32) {
            const int y = y0 + lane;
            int32_t v = (y <= ty) ? s_grid[y * sx + x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t nn = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += nn;
            }
            if (y <= ty) s_grid[y * sx + x] = v + carry;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    // exclusive scan of the per-tile counts in tile order (t = y * tx + x)
    const int T = tx * ty;
    const int per = (T + kRangesThreads - 1) / kRangesThreads;
    const int t0 = min(T, tid * per), t1 = min(T, t0 + per);
    uint32_t local = 0;
    for (int t = t0; t < t1; ++t) {
        const uint32_t c = (uint32_t)s_grid[(t / tx) * sx + (t % tx)];
        local += c;
        atomicAdd(&s_th[0][t & 255], c);
        atomicAdd(&s_th[1][(t >> 8) & 255], c);
    }
    uint32_t total;
    uint32_t run = block_excl_scan_1024(local, s_warp, total);
    for (int t = t0; t < t1; ++t) {
        a.ranges[t] = run;
        run += (uint32_t)s_grid[(t / tx) * sx + (t % tx)];
    }
    if (tid == 0) {
        a.ranges[T] = total;
        a.counters[GES_CTR_PAIRS] = total;
        a.counters[GES_CTR_OVERFLOW] = (int64_t)total > a.capacity ? 1ull : 0ull;
    }
    __syncthreads();
    // exclusive digit offsets: 4 depth digit histograms (from S1) + 2 tile digits
    if (tid < 6 * 32) {
        const int h = tid >> 5;
        uint32_t* src = (h < 4) ? (a.hist + h * 256) : s_th[h - 4];
        uint32_t* dst = a.hist + h * 256;
        uint32_t vals[8], s = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { vals[q] = src[lane * 8 + q]; s += vals[q]; }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        uint32_t run2 = incl - s;
#pragma unroll
        for (int q = 0; q < 8; ++q) { dst[lane * 8 + q] = run2; run2 += vals[q]; }
    }
}

int ranges_smem_bytes(int tiles_x, int tiles_y) { return (tiles_x + 1) * (tiles_y + 1) * 4; }

cudaError_t launch_ranges(const RangesArgs& a, cudaStream_t stream) {
    const int smem = ranges_smem_bytes(a.tiles_x, a.tiles_y);
    static int configured = 0;
    if (smem > 48 * 1024 && configured < smem) {
        cudaFuncSetAttribute(ranges_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = 200 * 1024;
    }
    ranges_kernel<<<1, kRangesThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// One onesweep LSD pass: 8-bit digit at `shift`, 256 threads x 16 keys.
// ---------------------------------------------------------------------------
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096
constexpr int kRadixWarps = kRadixThreads / 32;

int64_t radix_tiles(int64_t n) { return (n + kRadixTile - 1) / kRadixTile; }

__global__ void __launch_bounds__(kRadixThreads) radix_pass_kernel(RadixPassArgs a) {
    __shared__ uint32_t s_keys[kRadixTile];
    __shared__ uint32_t s_vals[kRadixTile];
    __shared__ uint32_t s_whist[kRadixWarps][kRadixDigits];
    __shared__ uint32_t s_local[kRadixDigits];
    __shared__ uint32_t s_global[kRadixDigits];
    __shared__ uint32_t s_warp[kRadixWarps + 1];
    __shared__ uint32_t s_tile;
    if (a.overflow && *a.overflow) return;
    const int64_t n = min((int64_t)*a.count, a.max_items);
    const int64_t num_tiles = (n + kRadixTile - 1) / kRadixTile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    while (true) {
        if (tid == 0) s_tile = (uint32_t)atomicAdd(a.tile_counter, 1ull);
        for (int d = tid; d < kRadixWarps * kRadixDigits; d += kRadixThreads) (&s_whist[0][0])[d] = 0;
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= num_tiles) break;
        const int64_t base = tile * kRadixTile + warp * (kRadixItems * 32);
        uint32_t k[kRadixItems], v[kRadixItems], rank[kRadixItems];
#pragma unroll
        for (int j = 0; j < kRadixItems; ++j) {
            const int64_t idx = base + j * 32 + lane;
            if (idx < n) { k[j] = a.keys_in[idx]; v[j] = a.vals_in[idx]; }
        }
        // warp multisplit ranking, items in (j, lane) = index order
#pragma unroll
        for (int j = 0; j < kRadixItems; ++j) {
            const int64_t idx = base + j * 32 + lane;
            const bool valid = idx < n;
            const uint32_t d = valid ? ((k[j] >> a.shift) & 255u) : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            uint32_t cnt = 0;
            if (valid) cnt = s_whist[warp][d];
            __syncwarp();
            rank[j] = cnt + __popc(peers & lt_mask);
            if (valid && lane == __ffs(peers) - 1) s_whist[warp][d] = cnt + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // per digit (thread = digit): exclusive over warps, block total
        uint32_t tot = 0;
        {
            const int d = tid;
#pragma unroll
            for (int w = 0; w < kRadixWarps; ++w) {
                const uint32_t c = s_whist[w][d];
                s_whist[w][d] = tot;
                tot += c;
            }
            // publish + look back (serial per digit)
            uint32_t* st = a.lookback + tile * kRadixDigits;
            uint32_t excl = 0;
            if (tile == 0) {
                st_volatile(&st[d], kFlagPrefix | tot);
            } else {
                st_volatile(&st[d], kFlagAgg | tot);
                int64_t p = tile - 1;
                while (true) {
                    const uint32_t w = ld_volatile(a.lookback + p * kRadixDigits + d);
                    if (w == 0) continue;
                    excl += w & kValueMask;
                    if (w & kFlagPrefix) break;
                    --p;
                }
                st_volatile(&st[d], kFlagPrefix | (excl + tot));
            }
            s_global[d] = a.digit_offset[d] + excl;
        }
        // block-local exclusive scan of the digit totals (for the smem reorder)
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
            }
            __syncthreads();
            s_local[tid] = s_warp[warp] + incl - tot;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kRadixItems; ++j) {
            const int64_t idx = base + j * 32 + lane;
            if (idx < n) {
                const uint32_t d = (k[j] >> a.shift) & 255u;
                const uint32_t pos = s_local[d] + s_whist[warp][d] + rank[j];
                s_keys[pos] = k[j];
                s_vals[pos] = v[j];
            }
        }
        __syncthreads();
        const int nvalid = (int)min((int64_t)kRadixTile, n - tile * kRadixTile);
        for (int s = tid; s < nvalid; s += kRadixThreads) {
            const uint32_t key = s_keys[s];
            const uint32_t d = (key >> a.shift) & 255u;
            const uint32_t out = s_global[d] + (uint32_t)s - s_local[d];
            if (a.keys_out) a.keys_out[out] = key;
            a.vals_out[out] = s_vals[s];
        }
        __syncthreads();
    }
}

cudaError_t launch_radix_pass(const RadixPassArgs& a, cudaStream_t stream) {
    const int sms = num_sms();
    const int64_t tiles = radix_tiles(a.max_items);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * 4));
    radix_pass_kernel<<<(unsigned)grid, kRadixThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// S2 duplication: visible particles in depth order -> (tile, particle) pairs
// ---------------------------------------------------------------------------
constexpr int kDupThreads = 256;
constexpr int kDupItems = 4;
constexpr int kDupTile = kDupThreads * kDupItems;

int64_t duplicate_tiles(int64_t P) { return (P + kDupTile - 1) / kDupTile; }

__global__ void __launch_bounds__(kDupThreads) duplicate_kernel(DuplicateArgs a) {
    __shared__ uint32_t s_start[kDupTile + 1];  // inclusive-prefix form: item q covers [s_start[q], s_start[q+1])
    __shared__ uint32_t s_pid[kDupTile];
    __shared__ ushort4 s_rect[kDupTile];
    __shared__ uint32_t s_warp[kDupItems][kDupThreads / 32];
    __shared__ uint32_t s_tile, s_base, s_total;
    if (a.counters[GES_CTR_OVERFLOW]) return;
    const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (uint32_t)atomicAdd(a.tile_counter, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile * kDupTile >= V) return;  // tiles are claimed in order: nobody waits on this one
    // items in order q = j * 256 + tid (coalesced loads, index order j-major)
    uint32_t cnt[kDupItems];
#pragma unroll
    for (int j = 0; j < kDupItems; ++j) {
        const int q = j * kDupThreads + tid;
        const int64_t s = tile * kDupTile + q;
        cnt[j] = 0;
        if (s < V) {
            const uint32_t p = a.sorted_vis[s];
            const ushort4 r = a.rect[p];
            s_pid[q] = p;
            s_rect[q] = r;
            cnt[j] = (uint32_t)(r.z - r.x) * (uint32_t)(r.w - r.y);
        }
    }
    // block exclusive scan over q
    uint32_t incl[kDupItems];
#pragma unroll
    for (int j = 0; j < kDupItems; ++j) {
        uint32_t x = cnt[j];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += nn;
        }
        incl[j] = x;
        if (lane == 31) s_warp[j][warp] = x;
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t v = (&s_warp[0][0])[lane];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += nn;
        }
        (&s_warp[0][0])[lane] = x - v;
        const uint32_t total = __shfl_sync(0xffffffffu, x, 31);
        const uint32_t prefix = lookback_warp(a.lookback, (uint32_t)tile, total);
        if (lane == 0) { s_base = prefix; s_total = total; }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kDupItems; ++j) {
        const int q = j * kDupThreads + tid;
        s_start[q] = s_warp[j][warp] + incl[j] - cnt[j];
    }
    if (tid == 0) s_start[kDupTile] = s_total;
    __syncthreads();
    // load-balanced emission: one pair slot per thread per round
    const uint32_t total = s_total, gbase = s_base;
    for (uint32_t s = tid; s < total; s += kDupThreads) {
        // largest q with s_start[q] <= s (items with zero pairs are skipped naturally)
        int lo = 0, hi = kDupTile - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_start[mid] <= s) lo = mid; else hi = mid - 1;
        }
        const ushort4 r = s_rect[lo];
        const uint32_t li = s - s_start[lo];
        const uint32_t w = (uint32_t)(r.z - r.x);
        const uint32_t ty = r.y + li / w, tx = r.x + li % w;
        a.pair_tile[gbase + s] = ty * (uint32_t)a.tiles_x + tx;
        a.pair_val[gbase + s] = s_pid[lo];
    }
}

cudaError_t launch_duplicate(const DuplicateArgs& a, cudaStream_t stream) {
    const int64_t tiles = duplicate_tiles(a.max_items);
    duplicate_kernel<<<(unsigned)std::max<int64_t>(1, tiles), kDupThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace ges
