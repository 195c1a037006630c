// sort.cu -- S2: depth radix sort of the visible particles;
// its last pass writes the depth-ordered item records the binning (bin.cu)
// turns into the per-tile lists.
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
//   phase H  CTA c zeroes its published words, counts pass 0's digits of its
//            range [c P / G, (c+1) P / G) of the S1 keys and compacts the
//            visible ones (with their indices, in index order) into shared
//            memory, from where pass 0 ranks them as one tile.  Grid barrier.
//   pass p   CTA c owns [c n / G, (c+1) n / G) of the pass input (n = P for
//            pass 0, then V): it ranks its keys stably by digit (a 8192-key
//            tile: stable warp ranks by owner-slot rounds, shared-memory
//            reorder), publishes its digit counts (flagged words; a range of
//            one tile before ranking), and finds its starting position
//            per digit without a grid barrier, in two levels of 16-CTA groups
//            (the earlier CTAs of its group + the earlier groups' totals, each
//            group total published by the group's last CTA; the digit totals
//            are the sums of all group totals), then writes the reordered
//            keys in coalesced runs.  One grid barrier between passes.  (A
//            range longer than one tile is counted by a separate sweep.)
//   last     the same, writing the item records (particle, packed rect) of
//            the depth-ordered visible particles for the binning (bin.cu),
//            and per CTA: the pair slots (sum of rect areas) and the items
//            covering each band row (a row difference array in shared memory)
//            are added to SLOTS and row_count.
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
constexpr int kDsDigits = kRadixDigits;  // 9-bit digits
constexpr int kDsBits = 9;
constexpr uint32_t kCntFlag = 0x80000000u;            // published count word

struct DsSmem {
    uint32_t whist[kDsWarps][kDsDigits];  // per-warp digit counts -> offsets; last pass: the tile's rects
    uint32_t keys[kDsTile];
    uint32_t vals[kDsTile];
    uint32_t base[kDsDigits];            // running global position of each digit
    uint32_t local[kDsDigits];           // tile-local exclusive digit offsets
    uint32_t cnt[kDsDigits];             // tile (or range) digit counts
    int rowd[kMaxBandRows + 1];          // last pass: row difference counts of the CTA's items
    unsigned long long area;             // last pass: the CTA's pair slots
    uint32_t warp[kDsWarps + 1];
    uint32_t hn;                         // phase H's compacted count (> kDsTile: did not fit)
    // phase H keeps the visible keys of the CTA's range of the S1 keys (and their
    // indices), compacted in index order, for pass 0 when they fit one tile -- over
    // whist, which pass 0's ranking overwrites only after loading them
    __device__ uint32_t* hkeys() { return &whist[0][0]; }
    __device__ uint32_t* hvals() { return &whist[0][0] + kDsTile; }
};
static_assert(sizeof(uint32_t) * kDsWarps * kDsDigits >= sizeof(uint32_t) * 2 * kDsTile, "hkeys/hvals fit whist");

__device__ __forceinline__ uint32_t ds_digit(uint32_t key, uint32_t kmin, int shift) {
    return ((key - kmin) >> shift) & (kDsDigits - 1);
}
__device__ __forceinline__ int64_t range_lo(int64_t n, int c, int G) { return n * c / G; }
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

// This CTA's digit counts of its range of a pass input.
__device__ void ds_range_hist(const DepthSortArgs& a, DsSmem& sm, const uint32_t* kin, int64_t r0, int64_t r1,
                              int shift, bool drop) {
    const int tid = threadIdx.x;
    if (tid < kDsDigits) sm.cnt[tid] = 0;
    __syncthreads();
    for (int64_t t0 = r0; t0 < r1; t0 += kDsTile) {
        uint32_t k[kDsItems];
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const int64_t idx = t0 + j * kDsThreads + tid;
            k[j] = idx < r1 ? __ldcg(kin + idx) : kInvalidKey;
        }
#pragma unroll
        for (int j = 0; j < kDsItems; ++j)
            if (t0 + j * kDsThreads + tid < r1 && !(drop && k[j] == kInvalidKey))
                atomicAdd(&sm.cnt[ds_digit(k[j], a.key_base, shift)], 1u);
    }
    __syncthreads();
}

#if defined(GES_DS_TIMING) && GES_DS_TIMING == 3
__device__ unsigned long long g_ds_t[8];
__device__ long long g_ds_q[6];
#ifndef GES_DS_TIMING_SHIFT
#define GES_DS_TIMING_SHIFT 9  // the pass whose rank phases are timed (digit shift)
#endif
#define DS_RMARK(k) do { __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0 && shift == GES_DS_TIMING_SHIFT) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_ds_t[k] = t_; } } while (0)
#else
#define DS_RMARK(k) do {} while (0)
#endif
#if defined(GES_DS_TIMING) && GES_DS_TIMING == 4
// per pass p and phase k (0 start, 1 ranked, 2 prefix known, 3 written, 4 after the grid
// barrier): %globaltimer of thread 0 of CTA 0 [0] and of the last CTA [1]
__device__ unsigned long long g_ds_p[2][4][5];
#define DS_PMARK(p, k) do { if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && (p) < 4) { \
    unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
    g_ds_p[blockIdx.x == 0 ? 0 : 1][p][k] = t_; } } while (0)
#else
#define DS_PMARK(p, k) do {} while (0)
#endif
// Publishes this CTA's digit counts of pass p, then finds the sums over the
// CTAs before it without a grid barrier, in two levels of groups of kDsGroup
// CTAs: the published words of the earlier CTAs of its group, plus the
// published totals of the earlier groups (each written by its group's last CTA
// after its own in-group sum) -- three dependent rounds of loads whatever c is.
// Leaves in sm.base the CTA's first position per digit.
constexpr int kDsGroup = 16;
// Sum of the n flagged words base[0], base[stride], ... (spinning until each is
// published), U loads in flight.
template <int U>
__device__ __forceinline__ uint32_t ds_sum_published(const uint32_t* base, size_t stride, int n) {
    uint32_t s = 0;
    for (int j0 = 0; j0 < n; j0 += U) {
        uint32_t v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = j0 + j < n ? ld_volatile(base + (j0 + j) * stride) : kCntFlag;
#pragma unroll
        for (int j = 0; j < U; ++j) {
            while (!(v[j] & kCntFlag)) v[j] = ld_volatile(base + (j0 + j) * stride);
            s += v[j] & ~kCntFlag;
        }
    }
    return s;
}

__device__ void ds_prefix(const DepthSortArgs& a, DsSmem& sm, int p, bool publish) {
    const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
    const int g = c / kDsGroup, first = g * kDsGroup, glast = min(first + kDsGroup, G) - 1;
    uint32_t* stc = a.st_cnt + ((size_t)p * kDsMaxGrid) * kDsDigits;
    uint32_t* gtc = a.gt_cnt + ((size_t)p * kDsMaxGroups) * kDsDigits;
    if (publish && tid < kDsDigits) st_volatile(stc + (size_t)c * kDsDigits + tid, kCntFlag | sm.cnt[tid]);
    // the digit totals are the sums of ALL group totals (every CTA has then published:
    // the pass's implicit barrier)
    const int ng = (G + kDsGroup - 1) / kDsGroup;
    uint32_t tot = 0;
#if defined(GES_DS_TIMING) && GES_DS_TIMING == 3
    long long q0 = clock64(), q1 = 0, q2 = 0, q3 = 0;
#endif
    if (tid < kDsDigits) {
        const int d = tid;
        const uint32_t in = ds_sum_published<kDsGroup - 1>(stc + (size_t)first * kDsDigits + d, kDsDigits, c - first);
        if (c == glast)  // + this CTA's own published count (sm.cnt may hold a tile's by now)
            st_volatile(gtc + (size_t)g * kDsDigits + d,
                        kCntFlag | (in + (ld_volatile(stc + (size_t)c * kDsDigits + d) & ~kCntFlag)));
#if defined(GES_DS_TIMING) && GES_DS_TIMING == 3
        q1 = clock64();
#endif
        const uint32_t out = ds_sum_published<16>(gtc + d, kDsDigits, g);
#if defined(GES_DS_TIMING) && GES_DS_TIMING == 3
        q2 = clock64();
#endif
        tot = out + ds_sum_published<16>(gtc + (size_t)g * kDsDigits + d, kDsDigits, ng - g);
#if defined(GES_DS_TIMING) && GES_DS_TIMING == 3
        q3 = clock64();
        if (p == 1 && tid == 0 && (c == 0 || c == G - 1)) { g_ds_q[(c ? 3 : 0) + 0] = q1 - q0; g_ds_q[(c ? 3 : 0) + 1] = q2 - q1; g_ds_q[(c ? 3 : 0) + 2] = q3 - q2; }
#endif
        sm.base[d] = in + out;
    }
    __syncthreads();
    // + the totals of the smaller digits
    const uint32_t ex = scan512<uint32_t>(tot, sm.warp, nullptr);
    if (tid < kDsDigits) sm.base[tid] += ex;
    __syncthreads();
}

// --- one 8192-key tile of a pass: rank, (last pass) areas, write -------------
// ds_tile_rank: loads the tile [t0, min(t0 + kDsTile, r1)), ranks it stably by
// digit (per-warp counters, owner-slot rounds: below), and reorders it in shared
// memory (sm.keys / sm.vals in digit order); sm.cnt = the tile's digit counts,
// sm.local = their exclusive offsets.  Returns the number of valid keys.
template <bool SMEM_IN = false>  // the tile's keys / ids come from shared memory (phase H's compaction)
__device__ uint32_t ds_tile_rank(DsSmem& sm, const uint32_t* kin, const uint32_t* vin, int64_t t0, int64_t r1,
                                 int shift, bool drop, uint32_t kmin, uint32_t* publish = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    DS_RMARK(0);
    const uint32_t lt_mask = (1u << lane) - 1u;
    // warp-striped: item j of lane l of warp w is element t0 + w 256 + j 32 + l
    const int64_t wb = t0 + warp * (kDsItems * 32);
    uint32_t k[kDsItems], v[kDsItems], rank[kDsItems], valid = 0;
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const int64_t idx = wb + j * 32 + lane;
        k[j] = idx < r1 ? (SMEM_IN ? kin[idx] : __ldcg(kin + idx)) : kInvalidKey;
    }
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const int64_t idx = wb + j * 32 + lane;
        v[j] = vin ? (idx < r1 ? (SMEM_IN ? vin[idx] : __ldcg(vin + idx)) : 0u) : (uint32_t)idx;
        if (idx < r1 && !(drop && k[j] == kInvalidKey)) valid |= 1u << j;
    }
    if (SMEM_IN) __syncthreads();  // the inputs alias whist: every thread has loaded them
    if (publish) {  // the tile is the CTA's whole range: publish its digit counts before ranking,
                    // so that the pass prefix's loads find the other CTAs' words already set
        if (tid < kDsDigits) sm.cnt[tid] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kDsItems; ++j)
            if ((valid >> j) & 1u) atomicAdd(&sm.cnt[ds_digit(k[j], kmin, shift)], 1u);
        __syncthreads();
        if (tid < kDsDigits) st_volatile(publish + tid, kCntFlag | sm.cnt[tid]);
    }
#pragma unroll
    for (int j = 0; j < kDsDigits / 32; ++j) sm.whist[warp][j * 32 + lane] = 0;
    __syncwarp();
#if defined(GES_DS_TIMING) && GES_DS_TIMING == 3
    { uint32_t x = 0; for (int j = 0; j < kDsItems; ++j) x ^= k[j] ^ v[j]; if (x == 0x12345678u) sm.warp[0] = x; }
    DS_RMARK(1);
#endif
#ifndef GES_DS_MATCH
    // Stable ranks without MATCH or per-bit ballots (both issue far below the ALU rate):
    // per item, rounds in which the lowest unranked lane of every digit (atomicMin on a
    // per-warp owner slot) takes the digit's next count.  Rounds = the largest digit
    // multiplicity among the warp's 32 keys (mostly 1-3).  The owner slots borrow
    // sm.keys / sm.vals (free until the reorder below), 512 per warp, all ~0 between uses.
    uint32_t* own = sm.keys + warp * kDsDigits;
#pragma unroll
    for (int j = 0; j < kDsDigits / 32; ++j) own[j * 32 + lane] = 0xffffffffu;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const uint32_t d = ds_digit(k[j], kmin, shift);
        bool pending = (valid >> j) & 1u;
        rank[j] = 0;
        while (__any_sync(0xffffffffu, pending)) {
            if (pending) atomicMin(&own[d], (uint32_t)lane);
            __syncwarp();
            const bool win = pending && own[d] == (uint32_t)lane;
            __syncwarp();
            if (win) {
                const uint32_t c = sm.whist[warp][d];
                rank[j] = c;
                sm.whist[warp][d] = c + 1u;
                own[d] = 0xffffffffu;
                pending = false;
            }
            __syncwarp();
        }
    }
#else
    // the peers (lanes with the same digit) of all items first, then the serial
    // per-warp counter updates
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t peers[kDsItems];
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const bool ok = (valid >> j) & 1u;
        const uint32_t d = ds_digit(k[j], kmin, shift);
        peers[j] = __match_any_sync(0xffffffffu, ok ? d : (uint32_t)kDsDigits);
    }
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        const bool ok = (valid >> j) & 1u;
        const uint32_t d = ds_digit(k[j], kmin, shift);
        uint32_t cn = 0;
        if (ok) cn = sm.whist[warp][d];
        __syncwarp();
        rank[j] = cn + __popc(peers[j] & lt_mask);
        if (ok && (peers[j] >> lane) == 1u) sm.whist[warp][d] = cn + __popc(peers[j]);
        __syncwarp();
    }
#endif
    __syncthreads();
    DS_RMARK(2);
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
    DS_RMARK(3);
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
    DS_RMARK(4);
    return nvalid;
}

// Last pass: the rect of every reordered key staged in shared memory (over the
// free rank histograms); the tile's rect areas and row coverage accumulate into
// sm.area and sm.rowd.
// Last pass: gathers the ranked tile's rects (8 B each) into shared memory over whist
// (free once the tile is ranked) with cp.async, so that the gathers' latency overlaps the
// prefix look-back that follows; ds_tile_rects consumes them.
__device__ void ds_rect_prefetch(const DepthSortArgs& a, DsSmem& sm, uint32_t nvalid) {
    const int s0 = threadIdx.x * kDsItems;  // thread tid owns the positions [8 tid, 8 tid + 8)
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm.whist[0][0]) + 8u * (uint32_t)s0;
    const uint2* src = reinterpret_cast<const uint2*>(a.rect);
#pragma unroll
    for (int j = 0; j < kDsItems; ++j)
        if (s0 + j < (int)nvalid)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * j), "l"(src + sm.vals[s0 + j])
                         : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ void ds_tile_rects(const DepthSortArgs& a, DsSmem& sm, uint32_t nvalid) {
    const int tid = threadIdx.x;
    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's gathers (ds_rect_prefetch)
    uint2* rs = reinterpret_cast<uint2*>(&sm.whist[0][0]);
    const int s0 = tid * kDsItems;
    uint2 rc[kDsItems];
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) rc[j] = s0 + j < (int)nvalid ? rs[s0 + j] : make_uint2(0, 0);
    unsigned long long ar = 0;
#pragma unroll
    for (int j = 0; j < kDsItems; ++j) {
        if (s0 + j < (int)nvalid) {
            const uint32_t y0 = rc[j].x >> 16, y1 = rc[j].y >> 16;
            ar += (unsigned long long)((rc[j].y & 0xffffu) - (rc[j].x & 0xffffu)) * (y1 - y0);
            atomicAdd(&sm.rowd[y0], 1);
            atomicSub(&sm.rowd[y1], 1);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ar += __shfl_xor_sync(0xffffffffu, ar, o);
    if ((tid & 31) == 0 && ar) atomicAdd(&sm.area, ar);
    __syncthreads();
}

// Writes the reordered tile at its sorted positions (sm.base): the next pass's
// keys and ids, or (last pass) the sorted ids and the item records.  Then
// advances sm.base past the tile.
__device__ void ds_tile_write(const DepthSortArgs& a, DsSmem& sm, uint32_t nvalid, uint32_t* kout, uint32_t* vout,
                              int shift, bool last) {
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
        for (int s = tid; s < (int)nvalid; s += kDsThreads) {
            const uint32_t d = ds_digit(sm.keys[s], kmin, shift);
            const uint32_t out = sm.base[d] + (uint32_t)s - sm.local[d];
            const uint32_t pid = sm.vals[s];
            const uint2 rc = rs[s];
            vout[out] = pid;
            a.items[out] = make_uint2(pid, pack_rect(rc.x & 0xffffu, rc.x >> 16, rc.y & 0xffffu, rc.y >> 16));
        }
    }
    __syncthreads();
    if (tid < kDsDigits) sm.base[tid] += sm.cnt[tid];
    __syncthreads();
}

// One pass over the CTA's range [r0, r1) of the pass input.  A range of one
// tile (V <= G x 8192 after pass 0) is ranked first and its digit counts taken
// from the ranking; otherwise a counting sweep precedes.
__device__ void ds_pass(const DepthSortArgs& a, DsSmem& sm, const uint32_t* kin, const uint32_t* vin, uint32_t* kout,
                        uint32_t* vout, int64_t r0, int64_t r1, int p, bool last_pass) {
    // the item records ride on the last pass of a frame's sort (a plain sort -- items ==
    // null, ges_reorder -- writes the sorted ids only)
    const bool last = last_pass && a.items != nullptr;
    const int shift = kDsBits * p;
    const bool drop = p == 0;  // pass 0 reads the S1 keys: drops the non-visible ones
    const int tid = threadIdx.x;
    if (last) {
        for (int i = tid; i <= a.rows; i += kDsThreads) sm.rowd[i] = 0;
        if (tid == 0) sm.area = 0;
        __syncthreads();
    }
    DS_PMARK(p, 0);
    if (p == 0 && sm.hn <= (uint32_t)kDsTile) {
        // pass 0 from phase H's compacted visible keys: one tile, counted and published there
        const uint32_t nvalid = ds_tile_rank<true>(sm, sm.hkeys(), sm.hvals(), 0, sm.hn, shift, false, a.key_base);
        if (last) ds_rect_prefetch(a, sm, nvalid);
        DS_PMARK(p, 1);
        ds_prefix(a, sm, p, false);
        if (last) ds_tile_rects(a, sm, nvalid);
        DS_PMARK(p, 2);
        ds_tile_write(a, sm, nvalid, kout, vout, shift, last);
        DS_PMARK(p, 3);
    } else if (p > 0 && r1 - r0 <= kDsTile) {
        uint32_t* pub = a.st_cnt + ((size_t)p * kDsMaxGrid + blockIdx.x) * kDsDigits;
        const uint32_t nvalid = ds_tile_rank(sm, kin, vin, r0, r1, shift, drop, a.key_base, pub);
        if (last) ds_rect_prefetch(a, sm, nvalid);
        DS_PMARK(p, 1);
        ds_prefix(a, sm, p, false);  // (published before the ranking)
        if (last) ds_tile_rects(a, sm, nvalid);
        DS_PMARK(p, 2);
        ds_tile_write(a, sm, nvalid, kout, vout, shift, last);
        DS_PMARK(p, 3);
    } else {
        if (p > 0) ds_range_hist(a, sm, kin, r0, r1, shift, false);
        if (p > 0) ds_prefix(a, sm, p, true);
        for (int64_t t0 = r0; t0 < r1; t0 += kDsTile) {
            const uint32_t nvalid = ds_tile_rank(sm, kin, vin, t0, r1, shift, drop, a.key_base);
            if (last) {
                ds_rect_prefetch(a, sm, nvalid);
                ds_tile_rects(a, sm, nvalid);
            }
            // pass 0 (counted and published by phase H): the prefix after the first tile's ranking
            if (p == 0 && t0 == r0) ds_prefix(a, sm, p, false);
            ds_tile_write(a, sm, nvalid, kout, vout, shift, last);
        }
        if (p == 0 && r1 <= r0) ds_prefix(a, sm, p, false);  // (an empty range still takes part)
    }
    if (last) {  // the CTA's pair slots and row coverage
        uint32_t v = tid < a.rows ? (uint32_t)sm.rowd[tid] : 0u;
        const uint32_t ex = scan512<uint32_t>(v, sm.warp, nullptr);  // (rows <= 256 < 512)
        if (tid < a.rows && ex + v) atomicAdd(a.row_count + tid, ex + v);
        if (tid == 0 && sm.area) atomicAdd(&a.counters[GES_CTR_SLOTS], sm.area);
    }
}

// GES_DS_TIMING: CTA 0 records %globaltimer at phase boundaries in counters[16..23]
__device__ __forceinline__ void ds_mark(const DepthSortArgs& a, int slot) {
#ifdef GES_DS_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.counters[16 + slot] = t;
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
    if (tid < kDsDigits) sm.cnt[tid] = 0;
    if (c == min((c / kDsGroup + 1) * kDsGroup, G) - 1) {  // the group's last CTA: its group totals
        const int g = c / kDsGroup;
        for (int i = tid; i < kDsMaxPasses * kDsDigits; i += kDsThreads)
            a.gt_cnt[((size_t)(i / kDsDigits) * kDsMaxGroups + g) * kDsDigits + (i % kDsDigits)] = 0u;
    }
    __syncthreads();
    {
        // count pass 0's digits of the range and compact its visible keys (with their
        // indices, in index order) into sm.hkeys / sm.hvals while they fit one tile
        const int64_t h0 = range_lo(P, c, G), h1 = range_lo(P, c + 1, G);
        const int lane = tid & 31, warp = tid >> 5;
        const uint32_t lt_mask = (1u << lane) - 1u;
        uint32_t hn = 0;  // (uniform)
        for (int64_t t0 = h0; t0 < h1; t0 += kDsTile) {
            // warp-striped as in ds_tile_rank: item j of lane l of warp w is t0 + w 256 + j 32 + l
            const int64_t wb = t0 + warp * (kDsItems * 32);
            uint32_t k[kDsItems], bal[kDsItems], wcnt = 0;
#pragma unroll
            for (int j = 0; j < kDsItems; ++j) {
                const int64_t idx = wb + j * 32 + lane;
                k[j] = idx < h1 ? __ldcg(a.key0 + idx) : kInvalidKey;
            }
#pragma unroll
            for (int j = 0; j < kDsItems; ++j) {
                bal[j] = __ballot_sync(0xffffffffu, k[j] != kInvalidKey);
                wcnt += __popc(bal[j]);
                if (k[j] != kInvalidKey) atomicAdd(&sm.cnt[ds_digit(k[j], kmin, 0)], 1u);
            }
            if (lane == 0) sm.warp[warp] = wcnt;
            __syncthreads();
            if (warp == 0) {  // exclusive scan of the 32 warp counts
                const uint32_t x = sm.warp[lane];
                uint32_t incl = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += nn;
                }
                sm.warp[lane] = incl - x;
                if (lane == 31) sm.warp[kDsWarps] = incl;
            }
            __syncthreads();
            uint32_t pos = hn + sm.warp[warp];
            const uint32_t tile_total = sm.warp[kDsWarps];
#pragma unroll
            for (int j = 0; j < kDsItems; ++j) {
                if (k[j] != kInvalidKey) {
                    const uint32_t q = pos + __popc(bal[j] & lt_mask);
                    if (q < (uint32_t)kDsTile) {
                        sm.hkeys()[q] = k[j];
                        sm.hvals()[q] = (uint32_t)(wb + j * 32 + lane);
                    }
                }
                pos += __popc(bal[j]);
            }
            hn += tile_total;
            __syncthreads();  // (sm.warp is reused by the next tile)
        }
        if (tid == 0) sm.hn = hn;
        __syncthreads();
    }
    if (tid < kDsDigits) a.st_cnt[(size_t)c * kDsDigits + tid] = kCntFlag | sm.cnt[tid];  // pass 0 counted
    grid.sync();
    ds_mark(a, 1);
    if (V == 0) return;
    // ---- the passes ----
    const uint32_t* kin = a.key0;
    const uint32_t* vin = nullptr;
    int64_t n = P;
    for (int p = 0; p < npass; ++p) {
        const bool last = p == npass - 1;
        const int64_t r0 = range_lo(n, c, G), r1 = range_lo(n, c + 1, G);
        uint32_t* kout = last ? nullptr : a.keys[p & 1];
        uint32_t* vout = last ? a.sorted_vis : a.vals[p & 1];
        ds_pass(a, sm, kin, vin, kout, vout, r0, r1, p, last);
        if (!last) grid.sync();
        DS_PMARK(p, 4);
        ds_mark(a, last ? 6 : 2 + p);
        kin = kout;
        vin = vout;
        n = V;
    }
}

#if defined(GES_DS_TIMING) && GES_DS_TIMING == 3
}  // namespace ges
extern "C" void ges_debug_ds_times(unsigned long long* out) { cudaMemcpyFromSymbol(out, ges::g_ds_t, 64); }
extern "C" void ges_debug_ds_q(long long* out) { cudaMemcpyFromSymbol(out, ges::g_ds_q, 48); }
namespace ges {
#endif
#if defined(GES_DS_TIMING) && GES_DS_TIMING == 4
}  // namespace ges
extern "C" void ges_debug_ds_pass_times(unsigned long long* out) { cudaMemcpyFromSymbol(out, ges::g_ds_p, 320); }
namespace ges {
#endif
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
