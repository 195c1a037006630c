// sort.cu -- S2: depth radix sort of the visible particles
// and the item scan that turns the depth-sorted particles into pair slots.
//
// Design: instead of a 64-bit LSD sort of
// (tile_id << 32 | depth) keys over all pairs, the depth order is established
// once on the V visible particles (LSD passes over V << M; pass 0 also
// compacts the visible set), then bin.cu writes every tile's list directly in
// that order -- exactly the order of the 64-bit keys.  The keys are sorted
// as key - bits(near_z) (every visible z > near_z > 0, fp32 bits monotone)
// in 9-bit digits; S1 records the largest visible key, so only
// ceil(bits(max - base) / 9) passes run (3 for the bench scene).
//
// ONE persistent cooperative kernel (one 1024-thread CTA per SM): at V ~ 1e6
// the passes are latency-bound, so every phase boundary that is not a true
// data dependency is removed.
//   phase H  CTA c zeroes its published words and counts pass 0's digits of
//            its range [c P / G, (c+1) P / G) of the S1 keys.  Grid barrier.
//   pass p   CTA c owns [c n / G, (c+1) n / G) of the pass input (n = P for
//            pass 0, then V): it ranks its keys stably by digit (a 8192-key
//            tile: warp match_any multisplit, shared-memory reorder), publishes
//            its digit counts (flagged words), and finds its starting position
//            per digit without a grid barrier, in two levels of 16-CTA groups
//            (the earlier CTAs of its group + the earlier groups' totals, each
//            group total published by the group's last CTA; the digit totals
//            are the sums of all group totals), then writes the reordered
//            keys in coalesced runs.  One grid barrier between passes.  (A
//            range longer than one tile is counted by a separate sweep.)
//   last     the same, plus the item scan fused in: the first pair slot of
//            a particle, E = exclusive prefix of the rect areas in sorted
//            order, is the digit's area base (the area totals of the smaller
//            digits + the earlier CTAs' published area sums of this digit) +
//            a segmented block scan of the reordered tile; the item records,
//            the binning chunk starts and the slot count follow from E.
// 3 grid barriers for 3 passes (was 11).  Hand-written; no CUB.
#include <cooperative_groups.h>

#include <algorithm>

#include "ges_internal.h"

namespace cg = cooperative_groups;

namespace ges {

constexpr int kDsThreads = 1024;
constexpr int kDsWarps = kDsThreads / 32;
constexpr int kDsItems = 8;
constexpr int kDsTile = kDsThreads * kDsItems;  // 8192 keys
constexpr uint32_t kInvalidKey = 0xffffffffu;
constexpr uint64_t kItemCost = kBinItemCost;
constexpr int kDsDigits = kRadixDigits;  // 9-bit digits
constexpr int kDsBits = 9;
constexpr uint32_t kCntFlag = 0x80000000u;            // published count word
constexpr unsigned long long kAreaFlag = 1ull << 63;  // published area word

struct DsSmem {
    uint32_t whist[kDsWarps][kDsDigits];  // per-warp digit counts -> offsets; last pass: the tile's rects
    uint32_t keys[kDsTile];
    uint32_t vals[kDsTile];
    uint32_t xs[kDsTile + 1];            // last pass: exclusive block scan of the tile's areas
    uint32_t base[kDsDigits];            // running global position of each digit
    uint32_t local[kDsDigits];           // tile-local exclusive digit offsets
    uint32_t cnt[kDsDigits];             // tile (or range) digit counts
    unsigned long long abase[kDsDigits]; // last pass: running area base of each digit
    unsigned long long acnt[kDsDigits];  // last pass: range area sums per digit
    unsigned long long atot[kDsDigits];  // last pass: global area totals per digit
    uint32_t warp[kDsWarps + 1];
    unsigned long long warp64[kDsWarps + 1];
};

__device__ __forceinline__ uint32_t ds_digit(uint32_t key, uint32_t kmin, int shift) {
    return ((key - kmin) >> shift) & (kDsDigits - 1);
}
__device__ __forceinline__ int64_t range_lo(int64_t n, int c, int G) { return n * c / G; }
__device__ __forceinline__ uint32_t rect_area(ushort4 r) {
    return (uint32_t)(r.z - r.x) * (uint32_t)(r.w - r.y);
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exclusive scan of v over the first 512 threads (16 warps); returns the
// exclusive value; *total (optional) gets the sum.  All threads must call.
template <typename T>
__device__ __forceinline__ T scan512(T v, T* s_warp, T* total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    if (tid < kDsDigits && lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const T wv = lane < kDsDigits / 32 ? s_warp[lane] : T(0);
        T wi = wv;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const T nn = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += nn;
        }
        if (lane < kDsDigits / 32) s_warp[lane] = wi - wv;
        if (lane == kDsDigits / 32 - 1) s_warp[kDsDigits / 32] = wi;
    }
    __syncthreads();
    const T ex = tid < kDsDigits ? s_warp[warp] + incl - v : T(0);
    if (total) *total = s_warp[kDsDigits / 32];
    __syncthreads();
    return ex;
}

// This CTA's digit counts (and, in the last pass, rect-area sums) of its range
// of a pass input (pass >= 1: V visible keys with particle ids).
__device__ void ds_range_hist(const DepthSortArgs& a, DsSmem& sm, const uint32_t* kin, const uint32_t* vin,
                              int64_t r0, int64_t r1, int shift, bool last, bool drop = false) {
    const int tid = threadIdx.x;
    uint32_t* apart = sm.local;  // u32 area partials of one 8192-key tile (< 2^29: areas <= 2^16)
    if (tid < kDsDigits) { sm.cnt[tid] = 0; sm.acnt[tid] = 0; apart[tid] = 0; }
    __syncthreads();
    for (int64_t t0 = r0; t0 < r1; t0 += kDsTile) {
        uint32_t k[kDsItems], v[kDsItems];
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const int64_t idx = t0 + j * kDsThreads + tid;
            k[j] = idx < r1 ? __ldcg(kin + idx) : kInvalidKey;
            v[j] = (last && idx < r1) ? (vin ? __ldcg(vin + idx) : (uint32_t)idx) : 0u;
        }
        uint32_t ar[kDsItems];
        if (last) {
#pragma unroll
            for (int j = 0; j < kDsItems; ++j)
                ar[j] = t0 + j * kDsThreads + tid < r1 && !(drop && k[j] == kInvalidKey) ? rect_area(__ldg(a.rect + v[j])) : 0u;
        }
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            if (t0 + j * kDsThreads + tid < r1 && !(drop && k[j] == kInvalidKey)) {
                const uint32_t d = ds_digit(k[j], a.key_base, shift);
                atomicAdd(&sm.cnt[d], 1u);
                if (last) atomicAdd(&apart[d], ar[j]);
            }
        }
        if (last) {
            __syncthreads();
            if (tid < kDsDigits) { sm.acnt[tid] += apart[tid]; apart[tid] = 0; }
        }
    }
    __syncthreads();
}

// Publishes this CTA's counts (and area sums) of pass p, then finds the sums
// over the CTAs before it without a grid barrier, in two levels of groups of
// kDsGroup CTAs: the published words of the earlier CTAs of its group, plus the
// published totals of the earlier groups (each written by its group's last CTA
// after its own in-group sum) -- three dependent rounds of loads whatever c is.
// Leaves in sm.base / sm.abase the CTA's first position / area base per digit.
constexpr int kDsGroup = 16;
// Sum of the n flagged words base[0], base[stride], ... (spinning until each is
// published), U loads in flight.
template <typename T, T FLAG, int U>
__device__ __forceinline__ T ds_sum_published(const T* base, size_t stride, int n) {
    T s = 0;
    for (int j0 = 0; j0 < n; j0 += U) {
        T v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = j0 + j < n ? ld_volatile(base + (j0 + j) * stride) : FLAG;
#pragma unroll
        for (int j = 0; j < U; ++j) {
            while (!(v[j] & FLAG)) v[j] = ld_volatile(base + (j0 + j) * stride);
            s += v[j] & ~FLAG;
        }
    }
    return s;
}

__device__ void ds_prefix(const DepthSortArgs& a, DsSmem& sm, int p, bool last, bool publish) {
    const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
    const int g = c / kDsGroup, first = g * kDsGroup, glast = min(first + kDsGroup, G) - 1;
    uint32_t* stc = a.st_cnt + ((size_t)p * kDsMaxGrid) * kDsDigits;
    uint32_t* gtc = a.gt_cnt + ((size_t)p * kDsMaxGroups) * kDsDigits;
    if (publish && tid < kDsDigits) {
        if (last) st_volatile(a.st_area + (size_t)c * kDsDigits + tid, kAreaFlag | sm.acnt[tid]);
        st_volatile(stc + (size_t)c * kDsDigits + tid, kCntFlag | sm.cnt[tid]);
    }
    // threads 0..511: the counts of digit tid; threads 512..1023: the area sums (last
    // pass).  The digit totals are the sums of ALL group totals (every CTA has then
    // published: the pass's implicit barrier).
    const int d = tid & (kDsDigits - 1);
    const int ng = (G + kDsGroup - 1) / kDsGroup;
    uint32_t tot = 0;
    unsigned long long atot = 0;
    if (tid < kDsDigits) {
        const uint32_t in = ds_sum_published<uint32_t, kCntFlag, kDsGroup - 1>(stc + (size_t)first * kDsDigits + d,
                                                                               kDsDigits, c - first);
        if (c == glast) st_volatile(gtc + (size_t)g * kDsDigits + d, kCntFlag | (in + sm.cnt[d]));
        const uint32_t out = ds_sum_published<uint32_t, kCntFlag, 16>(gtc + d, kDsDigits, g);
        tot = out + ds_sum_published<uint32_t, kCntFlag, 16>(gtc + (size_t)g * kDsDigits + d, kDsDigits, ng - g);
        sm.base[d] = in + out;
    } else if (last) {
        const unsigned long long in = ds_sum_published<unsigned long long, kAreaFlag, 8>(
            a.st_area + (size_t)first * kDsDigits + d, kDsDigits, c - first);
        if (c == glast) st_volatile(a.gt_area + (size_t)g * kDsDigits + d, kAreaFlag | (in + sm.acnt[d]));
        const unsigned long long out =
            ds_sum_published<unsigned long long, kAreaFlag, 8>(a.gt_area + d, kDsDigits, g);
        atot = out + ds_sum_published<unsigned long long, kAreaFlag, 8>(a.gt_area + (size_t)g * kDsDigits + d,
                                                                         kDsDigits, ng - g);
        sm.abase[d] = in + out;
    }
    if (last && tid >= kDsDigits) sm.atot[d] = atot;
    __syncthreads();
    // + the totals of the smaller digits
    {
        const uint32_t ex = scan512<uint32_t>(tot, sm.warp, nullptr);
        if (tid < kDsDigits) sm.base[tid] += ex;
    }
    if (last) {
        const unsigned long long t = tid < kDsDigits ? sm.atot[tid] : 0ull;
        const unsigned long long ex = scan512<unsigned long long>(t, sm.warp64, nullptr);
        if (tid < kDsDigits) sm.abase[tid] += ex;
    }
    __syncthreads();
}

// --- one 8192-key tile of a pass: rank, (last pass) areas, write -------------
// ds_tile_rank: loads the tile [t0, min(t0 + kDsTile, r1)), ranks it stably by
// digit (warp multisplit: one ballot per digit bit), and reorders it in shared
// memory (sm.keys / sm.vals in digit order); sm.cnt = the tile's digit counts,
// sm.local = their exclusive offsets.  Returns the number of valid keys.
__device__ uint32_t ds_tile_rank(DsSmem& sm, const uint32_t* kin, const uint32_t* vin, int64_t t0, int64_t r1,
                                 int shift, bool drop, uint32_t kmin) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // warp-striped: item j of lane l of warp w is element t0 + w 256 + j 32 + l
    const int64_t wb = t0 + warp * (kDsItems * 32);
    uint32_t k[kDsItems], v[kDsItems], rank[kDsItems], valid = 0;
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const int64_t idx = wb + j * 32 + lane;
        k[j] = idx < r1 ? __ldcg(kin + idx) : kInvalidKey;
    }
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const int64_t idx = wb + j * 32 + lane;
        v[j] = vin ? (idx < r1 ? __ldcg(vin + idx) : 0u) : (uint32_t)idx;
        if (idx < r1 && !(drop && k[j] == kInvalidKey)) valid |= 1u << j;
    }
#pragma unroll
    for (int j = 0; j < kDsDigits / 32; ++j) sm.whist[warp][j * 32 + lane] = 0;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const bool ok = (valid >> j) & 1u;
        const uint32_t d = ds_digit(k[j], kmin, shift);
#ifdef GES_DS_BALLOT
        uint32_t peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
        for (int b = 0; b < kDsBits; ++b) {
            const uint32_t bit = (d >> b) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
#else
        // lanes with the same digit (invalid lanes share the out-of-range value 512)
        const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : (uint32_t)kDsDigits);
#endif
        uint32_t cn = 0;
        if (ok) cn = sm.whist[warp][d];
        __syncwarp();
        rank[j] = cn + __popc(peers & lt_mask);
        if (ok && (peers >> lane) == 1u) sm.whist[warp][d] = cn + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive over warps, tile count, tile-local exclusive offsets
    uint32_t tc = 0;
    if (tid < kDsDigits) {
#pragma unroll 8
        for (int w = 0; w < kDsWarps; ++w) {
            const uint32_t x = sm.whist[w][tid];
            sm.whist[w][tid] = tc;
            tc += x;
        }
        sm.cnt[tid] = tc;
    }
    uint32_t nvalid;
    const uint32_t loc = scan512<uint32_t>(tc, sm.warp, &nvalid);
    if (tid < kDsDigits) sm.local[tid] = loc;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        if ((valid >> j) & 1u) {
            const uint32_t d = ds_digit(k[j], kmin, shift);
            const uint32_t pos = sm.local[d] + sm.whist[warp][d] + rank[j];
            sm.keys[pos] = k[j];
            sm.vals[pos] = v[j];
        }
    }
    __syncthreads();
    return nvalid;
}

// Last pass: the rect of every reordered key staged in shared memory (over the
// free rank histograms) and sm.xs = the exclusive scan of their areas over the
// tile (xs[nvalid] = the total); sm.acnt (if tile_sums) = the digit area sums.
__device__ void ds_tile_areas(const DepthSortArgs& a, DsSmem& sm, uint32_t nvalid, bool tile_sums) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint2* rs = reinterpret_cast<uint2*>(&sm.whist[0][0]);
    // thread tid owns the positions [8 tid, 8 tid + 8)
    const int s0 = tid * kDsItems;
    uint32_t ar[kDsItems], sum = 0;
    uint2 rc[kDsItems];
#pragma unroll
    for (int j = 0; j < kDsItems; ++j)
        rc[j] = s0 + j < (int)nvalid ? __ldg(reinterpret_cast<const uint2*>(a.rect) + sm.vals[s0 + j]) : make_uint2(0, 0);
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        rs[s0 + j] = rc[j];
        ar[j] = ((rc[j].y & 0xffffu) - (rc[j].x & 0xffffu)) * ((rc[j].y >> 16) - (rc[j].x >> 16));
        sum += ar[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    if (lane == 31) sm.warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t wv = sm.warp[lane];
        uint32_t wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += nn;
        }
        sm.warp[lane] = wi - wv;
    }
    __syncthreads();
    uint32_t x = sm.warp[warp] + incl - sum;
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        if (s0 + j <= (int)nvalid) sm.xs[s0 + j] = x;
        x += ar[j];
    }
    if (tid == kDsThreads - 1) sm.xs[kDsTile] = x;   // (a full tile: nvalid = kDsTile)
    __syncthreads();
    if (tile_sums && tid < kDsDigits) sm.acnt[tid] = sm.xs[sm.local[tid] + sm.cnt[tid]] - sm.xs[sm.local[tid]];
}

// Writes the reordered tile at its sorted positions (sm.base): the next pass's
// keys and ids, or (last pass) the sorted ids, E, the item records and the
// binning chunk starts.  Then advances sm.base (and sm.abase) past the tile.
__device__ void ds_tile_write(const DepthSortArgs& a, DsSmem& sm, uint32_t nvalid, uint32_t* kout, uint32_t* vout,
                              int shift, bool last, int64_t V) {
    const int tid = threadIdx.x;
    const uint32_t kmin = a.key_base;
    if (!last) {
        for (int s = tid; s < (int)nvalid; s += kDsThreads) {
            const uint32_t key = sm.keys[s];
            const uint32_t d = ds_digit(key, kmin, shift);
            const uint32_t out = sm.base[d] + (uint32_t)s - sm.local[d];
            vout[out] = sm.vals[s];
            if (kout) kout[out] = key;
        }
    } else {
        const uint2* rs = reinterpret_cast<const uint2*>(&sm.whist[0][0]);
        const uint64_t S = (uint64_t)a.chunk_slots;
        const double invS = 1.0 / (double)S;
        for (int s = tid; s < (int)nvalid; s += kDsThreads) {
            const uint32_t d = ds_digit(sm.keys[s], kmin, shift);
            const uint32_t seg = sm.local[d];
            const int64_t out = (int64_t)sm.base[d] + s - seg;
            const uint64_t e = sm.abase[d] + (sm.xs[s] - sm.xs[seg]);
            const uint64_t e1 = e + (sm.xs[s + 1] - sm.xs[s]);
            const uint32_t pid = sm.vals[s];
            const uint2 rc = rs[s];
            vout[out] = pid;
            a.E[out] = (uint32_t)e;
            a.items[out] = make_uint4(row_class_mask(rc.x >> 16, rc.y >> 16), pid, rc.x, rc.y);
            // binning chunk k = the items whose cost W[s] = E[s] + kItemCost s lies in
            // [k S, (k+1) S) (bin.cu): chunk_first[k] = min{s : W[s] >= k S}; item s + 1
            // is that minimum for every k with k S in (W[s], W[s+1]].  Item 0 opens chunk 0.
            const uint64_t w0 = e + kItemCost * (uint64_t)out;
            const uint64_t w1 = e1 + kItemCost * (uint64_t)(out + 1);
            const bool ovf = (int64_t)e1 > a.capacity;
            if (out == 0) a.chunk_first[0] = 0;
            if (!ovf) {
                // floor(w0 / S) + 1 from a double quotient (exact after the correction; w < 2^53)
                uint64_t kn = (uint64_t)((double)w0 * invS);
                if (kn * S > w0) --kn;
                else if ((kn + 1) * S <= w0) ++kn;
                for (++kn; kn * S <= w1; ++kn) a.chunk_first[kn] = (uint32_t)(out + 1);
            }
            if (out == V - 1) {  // total pair slots, capacity check, chunk count and closing entry
                a.counters[GES_CTR_SLOTS] = e1;
                a.counters[GES_CTR_OVERFLOW] = ovf ? 1ull : 0ull;
                const uint64_t C = (w1 + S - 1) / S;
                a.counters[GES_CTR_CHUNKS] = ovf ? 0ull : C;
                if (!ovf) a.chunk_first[C] = (uint32_t)V;
            }
        }
        __syncthreads();
        if (tid < kDsDigits) sm.abase[tid] += sm.xs[sm.local[tid] + sm.cnt[tid]] - sm.xs[sm.local[tid]];
    }
    __syncthreads();
    if (tid < kDsDigits) sm.base[tid] += sm.cnt[tid];
    __syncthreads();
}

// One pass over the CTA's range [r0, r1) of the pass input.  A range of one
// tile (V <= G x 8192 after pass 0) is ranked first and its digit counts (and
// area sums) taken from the ranking; otherwise a counting sweep precedes.
__device__ void ds_pass(const DepthSortArgs& a, DsSmem& sm, const uint32_t* kin, const uint32_t* vin, uint32_t* kout,
                        uint32_t* vout, int64_t r0, int64_t r1, int p, bool last_pass, int64_t V) {
    // the item scan rides on the last pass of a frame's sort (a plain sort -- items == null,
    // ges_reorder -- writes the sorted ids only)
    const bool last = last_pass && a.items != nullptr;
    const int shift = kDsBits * p;
    const bool drop = p == 0;  // pass 0 reads the S1 keys: drops the non-visible ones
    if (p > 0 && r1 - r0 <= kDsTile) {
        const uint32_t nvalid = ds_tile_rank(sm, kin, vin, r0, r1, shift, drop, a.key_base);
        if (last) ds_tile_areas(a, sm, nvalid, true);
        ds_prefix(a, sm, p, last, true);
        ds_tile_write(a, sm, nvalid, kout, vout, shift, last, V);
        return;
    }
    if (p > 0) ds_range_hist(a, sm, kin, vin, r0, r1, shift, last);
    ds_prefix(a, sm, p, last, p > 0);   // pass 0: counted and published by phase H
    for (int64_t t0 = r0; t0 < r1; t0 += kDsTile) {
        const uint32_t nvalid = ds_tile_rank(sm, kin, vin, t0, r1, shift, drop, a.key_base);
        if (last) ds_tile_areas(a, sm, nvalid, false);
        ds_tile_write(a, sm, nvalid, kout, vout, shift, last, V);
    }
}

// GES_DS_TIMING: CTA 0 records %globaltimer at phase boundaries in counters[8..15]
__device__ __forceinline__ void ds_mark(const DepthSortArgs& a, int slot) {
#ifdef GES_DS_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.counters[8 + slot] = t;
    }
#endif
}

__global__ void __launch_bounds__(kDsThreads, 1) depth_sort_kernel(DepthSortArgs a) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    DsSmem& sm = *reinterpret_cast<DsSmem*>(s_raw);
    cg::grid_group grid = cg::this_grid();
    const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
    const int64_t P = a.P;
    const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
    const uint32_t kmin = a.key_base;
    // passes: 9-bit digits over bits(max visible key - base) (S1 records the max)
    const uint32_t span = V ? (uint32_t)a.counters[GES_CTR_KEYMAX] - kmin : 0u;
    const int npass = max(1, ((span ? 32 - __clz(span) : 0) + kDsBits - 1) / kDsBits);
    ds_mark(a, 0);
    // ---- phase H: zero this CTA's published words, count pass 0 of its range ----
    for (int i = tid; i < kDsMaxPasses * kDsDigits; i += kDsThreads)
        a.st_cnt[((size_t)(i / kDsDigits) * kDsMaxGrid + c) * kDsDigits + (i % kDsDigits)] = 0u;
    if (tid < kDsDigits) { a.st_area[(size_t)c * kDsDigits + tid] = 0ull; sm.cnt[tid] = 0; sm.acnt[tid] = 0; }
    if (c == min((c / kDsGroup + 1) * kDsGroup, G) - 1) {  // the group's last CTA: its group totals
        const int g = c / kDsGroup;
        for (int i = tid; i < kDsMaxPasses * kDsDigits; i += kDsThreads)
            a.gt_cnt[((size_t)(i / kDsDigits) * kDsMaxGroups + g) * kDsDigits + (i % kDsDigits)] = 0u;
        if (tid < kDsDigits) a.gt_area[(size_t)g * kDsDigits + tid] = 0ull;
    }
    __syncthreads();
    {
        const int64_t h0 = range_lo(P, c, G), h1 = range_lo(P, c + 1, G);
        if (npass == 1 && a.items) {   // pass 0 is the last: its area sums too
            ds_range_hist(a, sm, a.key0, nullptr, h0, h1, 0, true, true);
        } else {
            for (int64_t t0 = h0; t0 < h1; t0 += kDsTile) {
                uint32_t k[kDsItems];
#pragma unroll
                for (int j = 0; j < kDsItems; ++j) {
                    const int64_t idx = t0 + j * kDsThreads + tid;
                    k[j] = idx < h1 ? __ldcg(a.key0 + idx) : kInvalidKey;
                }
#pragma unroll
                for (int j = 0; j < kDsItems; ++j)
                    if (k[j] != kInvalidKey) atomicAdd(&sm.cnt[ds_digit(k[j], kmin, 0)], 1u);
            }
            __syncthreads();
        }
    }
    if (tid < kDsDigits) {  // pass 0 of this CTA's range is counted: publish it
        if (npass == 1 && a.items) a.st_area[(size_t)c * kDsDigits + tid] = kAreaFlag | sm.acnt[tid];
        a.st_cnt[(size_t)c * kDsDigits + tid] = kCntFlag | sm.cnt[tid];
    }
    grid.sync();
    ds_mark(a, 1);
    if (V == 0) {
        if (c == 0 && tid == 0) {
            a.counters[GES_CTR_SLOTS] = 0;
            a.counters[GES_CTR_CHUNKS] = 0;
        }
        return;
    }
    // ---- the passes ----
    const uint32_t* kin = a.key0;
    const uint32_t* vin = nullptr;
    int64_t n = P;
    for (int p = 0; p < npass; ++p) {
        const bool last = p == npass - 1;
        const int64_t r0 = range_lo(n, c, G), r1 = range_lo(n, c + 1, G);
        uint32_t* kout = last ? nullptr : a.keys[p & 1];
        uint32_t* vout = last ? a.sorted_vis : a.vals[p & 1];
        ds_pass(a, sm, kin, vin, kout, vout, r0, r1, p, last, V);
        if (!last) grid.sync();
        ds_mark(a, last ? 6 : 2 + p);
        kin = kout;
        vin = vout;
        n = V;
    }
}

int depth_sort_grid() {
    static int grid[kMaxDevices] = {0};
    const int dev = current_device();
    if (grid[dev] == 0) {
        int per_sm = 0;
        cudaFuncSetAttribute(depth_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DsSmem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, depth_sort_kernel, kDsThreads, sizeof(DsSmem));
        grid[dev] = std::min(kDsMaxGrid, std::max(1, std::min(per_sm, 1)) * num_sms());
    }
    return grid[dev];
}

cudaError_t launch_depth_sort(const DepthSortArgs& a, cudaStream_t stream) {
    DepthSortArgs args = a;
    args.G = depth_sort_grid();
    void* params[] = {&args};
    return cudaLaunchCooperativeKernel((const void*)depth_sort_kernel, dim3(args.G), dim3(kDsThreads), params,
                                       sizeof(DsSmem), stream);
}

}  // namespace ges
