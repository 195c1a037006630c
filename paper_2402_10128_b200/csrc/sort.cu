// sort.cu -- S2: depth radix sort of the visible particles
// and the item scan that turns the depth-sorted particles into pair slots.
//
// Design: instead of a 64-bit LSD sort of
// (tile_id << 32 | depth) keys over all pairs, the depth order is established
// once on the V visible particles (LSD passes over V << M; pass 0 also
// compacts the visible set), then bin.cu writes every tile's list directly in
// that order -- exactly the order of the 64-bit keys.  The keys are sorted
// as key - bits(near_z) (every visible z > near_z > 0, fp32 bits monotone)
// in 9-bit digits; pass 0's histogram phase also finds the largest key, so
// only ceil(bits(max - base) / 9) passes run (3 for the bench scene).
//
// Everything here is ONE persistent cooperative kernel (one 1024-thread CTA
// per SM, grid-wide barriers between phases) because at V ~ 1e6 the passes
// are launch- and latency-bound, not bandwidth-bound.  Per pass, CTA c owns
// the contiguous input range [c n / G, (c+1) n / G):
//   hist     digit histogram of its range -> H[d][c]
//   colscan  CTA c scans the digits d = c (mod G) over the CTAs (in place),
//            digit totals -> Tot[d]
//   scatter  bases = exclusive scan of Tot + H[d][c]; its range in 8192-key
//            tiles, in order: stable warp-multisplit ranking (one ballot per
//            digit bit), shared-memory reorder, coalesced-run writes; the
//            last pass writes the particle ids and their item records
//            (particle, packed rect) in sorted order.
// Then the item scan: exclusive prefix E[s] of the rect areas of the sorted
// particles (per-CTA sums, a barrier, then each CTA's scan), the first item
// of every binning chunk, the slot count M.
// Hand-written; no CUB.
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

constexpr int kDsDigits = 512;  // up to 9-bit digits

struct DsSmem {
    uint32_t whist[kDsWarps][kDsDigits];  // per-warp digit counts -> offsets
    uint32_t keys[kDsTile];
    uint32_t vals[kDsTile];
    uint32_t base[kDsDigits];   // running global position of each digit
    uint32_t local[kDsDigits];  // tile-local exclusive digit offsets
    uint32_t cnt[kDsDigits];    // tile digit counts
    uint32_t warp[kDsWarps + 1];
};

// The digit of pass `shift` of a visible key, relative to the smallest key.
__device__ __forceinline__ uint32_t ds_digit(uint32_t key, uint32_t kmin, int shift, uint32_t mask) {
    return ((key - kmin) >> shift) & mask;
}

__device__ __forceinline__ int64_t range_lo(int64_t n, int c, int G) { return n * c / G; }

// Exclusive scan of v over the first 512 threads (16 warps); returns the
// exclusive value; *total (optional) gets the sum.  All threads must call.
__device__ __forceinline__ uint32_t scan512(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nn;
    }
    if (tid < kDsDigits && lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        uint32_t r = 0;
        for (int w = 0; w < kDsDigits / 32; ++w) { const uint32_t x = s_warp[w]; s_warp[w] = r; r += x; }
        s_warp[kDsDigits / 32] = r;
    }
    __syncthreads();
    const uint32_t ex = tid < kDsDigits ? s_warp[warp] + incl - v : 0u;
    if (total) *total = s_warp[kDsDigits / 32];
    __syncthreads();
    return ex;
}

__device__ void ds_hist(const DepthSortArgs& a, DsSmem& sm, const uint32_t* in, int64_t n, int shift, bool drop,
                        uint32_t kmin, uint32_t mask) {
    const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
    if (tid < kDsDigits) sm.cnt[tid] = 0;
    __syncthreads();
    const int64_t r0 = range_lo(n, c, G), r1 = range_lo(n, c + 1, G);
    uint32_t kmax = 0;
    for (int64_t t0 = r0; t0 < r1; t0 += kDsTile) {
        uint32_t k[kDsItems];
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const int64_t idx = t0 + j * kDsThreads + tid;
            k[j] = idx < r1 ? __ldcg(in + idx) : kInvalidKey;
        }
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const int64_t idx = t0 + j * kDsThreads + tid;
            if (idx < r1 && !(drop && k[j] == kInvalidKey)) {
                atomicAdd(&sm.cnt[ds_digit(k[j], kmin, shift, mask)], 1u);
                kmax = max(kmax, k[j]);
            }
        }
    }
    if (drop) {  // pass 0: the largest visible key (plan of the remaining passes)
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if ((tid & 31) == 0 && kmax) atomicMax(&a.counters[GES_CTR_KEYMAX], (unsigned long long)kmax);
    }
    __syncthreads();
    if (tid <= (int)mask) a.hist[(int64_t)tid * G + c] = sm.cnt[tid];
}

// CTA c scans digits d = c, c + G, ... over the CTAs (one warp per digit).
__device__ void ds_colscan(const DepthSortArgs& a, int nd) {
    const int c = blockIdx.x, G = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = c + warp * G; d < nd; d += kDsWarps * G) {
        uint32_t* col = a.hist + (int64_t)d * G;
        uint32_t run = 0;
        for (int c0 = 0; c0 < G; c0 += 32) {
            const int cc = c0 + lane;
            const uint32_t v = cc < G ? __ldcg(col + cc) : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nn = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += nn;
            }
            if (cc < G) col[cc] = run + incl - v;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) a.tot[d] = run;
    }
}

template <int D>
__device__ void ds_scatter(const DepthSortArgs& a, DsSmem& sm, const uint32_t* kin, const uint32_t* vin,
                           uint32_t* kout, uint32_t* vout, int64_t n, int shift, bool drop, uint32_t kmin,
                           bool last) {
    const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    constexpr int ND = 1 << D;
    constexpr uint32_t kMask = ND - 1;
    {
        const uint32_t t = tid < ND ? __ldcg(a.tot + tid) : 0u;
        const uint32_t ex = scan512(t, sm.warp, nullptr);
        if (tid < ND) sm.base[tid] = ex + __ldcg(a.hist + (int64_t)tid * G + c);
    }
    const int64_t r0 = range_lo(n, c, G), r1 = range_lo(n, c + 1, G);
    for (int64_t t0 = r0; t0 < r1; t0 += kDsTile) {
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
        for (int j = 0; j < ND / 32; ++j) sm.whist[warp][j * 32 + lane] = 0;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const bool ok = (valid >> j) & 1u;
            const uint32_t d = ds_digit(k[j], kmin, shift, kMask);
            uint32_t peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
            for (int b = 0; b < D; ++b) {
                const uint32_t bit = (d >> b) & 1u;
                const uint32_t bal = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bal : ~bal;
            }
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
        if (tid < ND) {
#pragma unroll 8
            for (int w = 0; w < kDsWarps; ++w) {
                const uint32_t x = sm.whist[w][tid];
                sm.whist[w][tid] = tc;
                tc += x;
            }
            sm.cnt[tid] = tc;
        }
        uint32_t nvalid;
        const uint32_t loc = scan512(tc, sm.warp, &nvalid);
        if (tid < ND) sm.local[tid] = loc;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            if ((valid >> j) & 1u) {
                const uint32_t d = ds_digit(k[j], kmin, shift, kMask);
                const uint32_t pos = sm.local[d] + sm.whist[warp][d] + rank[j];
                sm.keys[pos] = k[j];
                sm.vals[pos] = v[j];
            }
        }
        __syncthreads();
        for (int s = tid; s < (int)nvalid; s += kDsThreads) {
            const uint32_t key = sm.keys[s];
            const uint32_t d = ds_digit(key, kmin, shift, kMask);
            const uint32_t out = sm.base[d] + (uint32_t)s - sm.local[d];
            const uint32_t pid = sm.vals[s];
            vout[out] = pid;
            if (!last) {
                kout[out] = key;
            } else {  // item record: row-class mask, particle, rect
                const ushort4 rc = __ldg(a.rect + pid);
                a.items[out] = make_uint4(row_class_mask(rc.y, rc.w), pid, (uint32_t)rc.x | ((uint32_t)rc.y << 16),
                                          (uint32_t)rc.z | ((uint32_t)rc.w << 16));
            }
        }
        __syncthreads();
        if (tid < ND) sm.base[tid] += sm.cnt[tid];
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t rec_count(uint4 r) {
    return ((r.w & 0xffffu) - (r.z & 0xffffu)) * ((r.w >> 16) - (r.z >> 16));
}

// Item scan over the V sorted particles: CTA c owns [V c / G, V (c+1) / G),
// thread t a contiguous run of it (all its records loaded at once).  PASS 0
// sums the CTA's areas into part[c]; PASS 1 (after a barrier) scans and
// writes E, the item records' slot field, the chunk starts and the counts.
constexpr int kDsRun = 8;  // records per thread per round
template <int PASS>
__device__ void ds_items(const DepthSortArgs& a, DsSmem& sm, int64_t V) {
    const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = range_lo(V, c, G), r1 = range_lo(V, c + 1, G);
    uint64_t run = 0;  // slots before this round
    if (PASS == 1) {   // this CTA's base: sum of the preceding CTAs' areas
        unsigned long long s = 0;
        for (int cc = tid; cc < c; cc += kDsThreads) s += __ldcg(a.part + cc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        uint64_t* s64 = reinterpret_cast<uint64_t*>(sm.keys);
        if (lane == 0) s64[warp] = s;
        __syncthreads();
        for (int w = 0; w < kDsWarps; ++w) run += s64[w];
        __syncthreads();
    }
    for (int64_t t0 = r0; t0 < r1; t0 += (int64_t)kDsThreads * kDsRun) {
        const int64_t s0 = t0 + (int64_t)tid * kDsRun;
        uint4 rec[kDsRun];
        uint32_t sum = 0;
#pragma unroll
        for (int j = 0; j < kDsRun; ++j) rec[j] = s0 + j < r1 ? __ldcg(a.items + s0 + j) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < kDsRun; ++j) sum += rec_count(rec[j]);
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
            if (lane == 31) sm.warp[32] = wi;
        }
        __syncthreads();
        const uint32_t round_total = sm.warp[32];
        if (PASS == 1) {
            uint64_t e = run + sm.warp[warp] + incl - sum;
            const uint64_t S = (uint64_t)a.chunk_slots;
            // the next chunk boundary after this thread's first item (one division per run)
            uint64_t kn = (e + kItemCost * (uint64_t)s0) / S + 1;
#pragma unroll
            for (int j = 0; j < kDsRun; ++j) {
                const int64_t s = s0 + j;
                if (s >= r1) break;
                const uint64_t e1 = e + rec_count(rec[j]);
                a.E[s] = (uint32_t)e;
                // binning chunk k = the items whose cost W[s] = E[s] + kItemCost s lies in
                // [k S, (k+1) S) (bin.cu): chunk_first[k] = min{s : W[s] >= k S}; item s + 1
                // is that minimum for every k with k S in (W[s], W[s+1]].  Item 0 opens chunk 0.
                const uint64_t w1 = e1 + kItemCost * (uint64_t)(s + 1);
                const bool ovf = (int64_t)e1 > a.capacity;
                if (s == 0) a.chunk_first[0] = 0;
                for (; kn * S <= w1; ++kn)
                    if (!ovf) a.chunk_first[kn] = (uint32_t)(s + 1);
                if (s == V - 1) {  // total pair slots, capacity check, chunk count and closing entry
                    a.counters[GES_CTR_SLOTS] = e1;
                    a.counters[GES_CTR_OVERFLOW] = ovf ? 1ull : 0ull;
                    const uint64_t C = (w1 + S - 1) / S;
                    a.counters[GES_CTR_CHUNKS] = ovf ? 0ull : C;
                    if (!ovf) a.chunk_first[C] = (uint32_t)V;
                }
                e = e1;
            }
        }
        run += round_total;
        __syncthreads();
    }
    if (PASS == 0 && tid == 0) a.part[c] = run;
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
    const int64_t P = a.P;
    const int64_t V = (int64_t)a.counters[GES_CTR_VISIBLE];
    // pass d: pass 0 reads the preprocess keys (indices as values) and drops
    // the non-visible ones; the last pass writes sorted_vis and the item records.
    // keys are sorted as key - kbase in 9-bit digits; the pass count follows
    // from the largest key, found by pass 0's histogram phase
    const uint32_t kmin = a.key_base;
    constexpr int D = 9;
    int npass = 4;
    const uint32_t* kin = a.key0;
    const uint32_t* vin = nullptr;
    int64_t n = P;
    ds_mark(a, 1);
    for (int d = 0; d < npass; ++d) {
        const bool drop = d == 0;
        const int shift = D * d;
        ds_hist(a, sm, kin, n, shift, drop, kmin, (1u << D) - 1);
        grid.sync();
        if (d == 0) {
            const uint32_t span = V ? (uint32_t)__ldcg(a.counters + GES_CTR_KEYMAX) - kmin : 0u;
            const int b = span ? 32 - __clz(span) : 0;
            npass = max(1, (b + D - 1) / D);
        }
        const bool last = d == npass - 1;
        uint32_t* kout = last ? nullptr : a.keys[d & 1];
        uint32_t* vout = last ? a.sorted_vis : a.vals[d & 1];
        ds_colscan(a, 1 << D);
        grid.sync();
        ds_scatter<D>(a, sm, kin, vin, kout, vout, n, shift, drop, kmin, last);
        grid.sync();
        ds_mark(a, 2 + d);
        kin = kout;
        vin = vout;
        n = V;
    }
    if (V == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.counters[GES_CTR_SLOTS] = 0;
            a.counters[GES_CTR_CHUNKS] = 0;
        }
        return;
    }
    ds_items<0>(a, sm, V);
    grid.sync();
    ds_mark(a, 6);
    ds_items<1>(a, sm, V);
    grid.sync();
    ds_mark(a, 7);
}

int depth_sort_grid() {
    static int grid = 0;
    if (grid == 0) {
        int per_sm = 0;
        cudaFuncSetAttribute(depth_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DsSmem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, depth_sort_kernel, kDsThreads, sizeof(DsSmem));
        grid = std::max(1, std::min(per_sm, 1)) * num_sms();
    }
    return grid;
}

cudaError_t launch_depth_sort(const DepthSortArgs& a, cudaStream_t stream) {
    DepthSortArgs args = a;
    args.G = depth_sort_grid();
    void* params[] = {&args};
    return cudaLaunchCooperativeKernel((const void*)depth_sort_kernel, dim3(args.G), dim3(kDsThreads), params,
                                       sizeof(DsSmem), stream);
}

}  // namespace ges
