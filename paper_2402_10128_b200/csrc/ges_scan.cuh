// ges_scan.cuh -- decoupled look-back prefix (single-pass scan across CTAs).
//
// A CTA that owns tile `tile` publishes its aggregate, then walks back over
// its predecessors' published words until it meets an inclusive prefix.
// Status word: bit31 = inclusive prefix available, bit30 = aggregate
// available, bits 0..29 = value.  Tiles must be claimed in increasing order
// (an atomic ticket), so every predecessor is resident or finished: no
// deadlock.  The caller zeroes the status array once per pass.
#pragma once
#include <cstdint>

namespace ges {

constexpr uint32_t kFlagPrefix = 0x80000000u;
constexpr uint32_t kFlagAgg = 0x40000000u;
constexpr uint32_t kValueMask = 0x3fffffffu;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Warp-cooperative look-back: all 32 lanes of the calling warp participate;
// returns the exclusive prefix of `tile` (same value in every lane) and
// publishes the inclusive prefix.  `agg` must be uniform across the warp.
__device__ __forceinline__ uint32_t lookback_warp(uint32_t* status, uint32_t tile, uint32_t agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_volatile(&status[0], kFlagPrefix | agg);
        return 0;
    }
    if (lane == 0) st_volatile(&status[tile], kFlagAgg | agg);
    uint32_t prefix = 0;
    int64_t base = (int64_t)tile - 1;  // highest predecessor still to examine
    while (true) {
        const int64_t p = base - lane;  // lane 0 looks at the nearest predecessor
        uint32_t v = kFlagPrefix;       // beyond tile 0: behaves as a 0 prefix
        if (p >= 0) {
            do { v = ld_volatile(&status[p]); } while (v == 0);
        }
        // lanes up to (and including) the first one holding an inclusive prefix count
        const uint32_t pre_mask = __ballot_sync(0xffffffffu, (v & kFlagPrefix) != 0);
        const int stop = pre_mask ? (__ffs(pre_mask) - 1) : 31;
        uint32_t val = (lane <= stop) ? (v & kValueMask) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (pre_mask) break;
        base -= 32;
    }
    if (lane == 0) st_volatile(&status[tile], kFlagPrefix | (prefix + agg));
    return prefix;
}

}  // namespace ges
