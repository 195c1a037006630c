// reorder.cu -- particle storage order: the
// planar particle buffers permuted into the Morton (Z-curve) order of the
// particle means, once after loading a scene and after every densify/prune.
// Off the per-step hot path; what it buys on it: particles that a camera culls
// (outside the frustum, behind the near plane) then come in runs, so S1 skips
// the 192 B of SH of a whole 128-particle tile with nothing visible and S5b the
// inputs of such a tile, instead of touching every 32-B sector of every plane
// (with the particles in random order nearly every sector holds a visible one).
//   bounds   the axis-aligned box of the means (order-preserving int atomics)
//   morton   30-bit codes: each axis quantised to 1024 cells of the box,
//            bits interleaved (x lowest)
//   sort     the depth-sort kernel of sort.cu in its plain mode: a stable LSD
//            sort of the codes with the particle index as value -- equal codes
//            keep index order, so the permutation is deterministic
//   gather   out[c][j] = in[c][perm[j]] for every plane (params, optional Adam
//            moments)
#include <algorithm>
#include <climits>

#include "ges_internal.h"

namespace ges {

__device__ __forceinline__ int ord_int(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord_float(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__global__ void reorder_bounds_kernel(const float* mean, int64_t P, int* box) {
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float f = mean[(size_t)k * P + i];
            if (f == f) {  // NaN means sort last (code 0 is fine too; they are excluded from the box)
                mn[k] = min(mn[k], ord_int(f));
                mx[k] = max(mx[k], ord_int(f));
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        mn[k] = __reduce_min_sync(0xffffffffu, mn[k]);
        mx[k] = __reduce_max_sync(0xffffffffu, mx[k]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(box + k, mn[k]);
            atomicMax(box + 3 + k, mx[k]);
        }
    }
}

__global__ void reorder_init_kernel(int* box, unsigned long long* counters) {
    const int t = threadIdx.x;
    if (t < 3) { box[t] = INT_MAX; box[3 + t] = INT_MIN; }
    if (t < GES_CTR_N) counters[t] = 0ull;
}

__device__ __forceinline__ uint32_t spread10(uint32_t x) {
    x = (x | (x << 16)) & 0x030000FFu;
    x = (x | (x << 8)) & 0x0300F00Fu;
    x = (x | (x << 4)) & 0x030C30C3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__global__ void reorder_morton_kernel(const float* mean, int64_t P, const int* box, uint32_t* keys,
                                      unsigned long long* counters) {
    float lo[3], scale[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = ord_float(box[k]);
        const float ext = ord_float(box[3 + k]) - lo[k];
        scale[k] = ext > 0.0f ? 1024.0f / ext : 0.0f;
    }
    uint32_t kmax = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t code = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float f = (mean[(size_t)k * P + i] - lo[k]) * scale[k];
            const uint32_t q = f == f ? (uint32_t)fminf(fmaxf(f, 0.0f), 1023.0f) : 1023u;
            code |= spread10(q) << k;
        }
        keys[i] = code + 1u;  // the sort's keys must exceed its base (0); 0xffffffff stays "invalid"
        kmax = max(kmax, code + 1u);
    }
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if ((threadIdx.x & 31) == 0) atomicMax(counters + GES_CTR_KEYMAX, (unsigned long long)kmax);
    if (blockIdx.x == 0 && threadIdx.x == 0) counters[GES_CTR_VISIBLE] = (unsigned long long)P;
}

__global__ void reorder_gather_kernel(const float* in, float* out, int64_t P, int n_planes, const uint32_t* perm) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < P; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t src = __ldg(perm + j);
        for (int c = 0; c < n_planes; ++c) out[(size_t)c * P + j] = __ldg(in + (size_t)c * P + src);
    }
}

// Workspace: box (8 ints) | counters | keys0 [P] | keys [2][P] | vals [2][P] | the
// depth sort's published words.
static size_t carve(char* base, int64_t P, DepthSortArgs* ds, int** box) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        char* p = base ? base + off : nullptr;
        off = (off + bytes + 255) / 256 * 256;
        return p;
    };
    int* b = (int*)take(8 * sizeof(int));
    unsigned long long* ctr = (unsigned long long*)take(GES_CTR_N * sizeof(unsigned long long));
    uint32_t* k0 = (uint32_t*)take(4 * (size_t)P);
    uint32_t* k1 = (uint32_t*)take(4 * (size_t)P);
    uint32_t* k2 = (uint32_t*)take(4 * (size_t)P);
    uint32_t* v1 = (uint32_t*)take(4 * (size_t)P);
    uint32_t* v2 = (uint32_t*)take(4 * (size_t)P);
    uint32_t* stc = (uint32_t*)take(sizeof(uint32_t) * kRadixDigits * (size_t)kDsMaxGrid * kDsMaxPasses);
    uint32_t* gtc = (uint32_t*)take(sizeof(uint32_t) * kRadixDigits * (size_t)kDsMaxGroups * kDsMaxPasses);
    if (ds) {
        *ds = DepthSortArgs{};
        ds->key0 = k0;
        ds->keys[0] = k1; ds->keys[1] = k2;
        ds->vals[0] = v1; ds->vals[1] = v2;
        ds->st_cnt = stc; ds->gt_cnt = gtc;
        ds->P = P; ds->key_base = 0u;
        ds->counters = ctr;
    }
    if (box) *box = b;
    return off;
}

size_t reorder_workspace_bytes(int64_t P) { return carve(nullptr, P, nullptr, nullptr); }

cudaError_t launch_reorder(const float* const* in, float* const* out, int n_buffers, int64_t P, int n_planes,
                           uint32_t* perm, void* workspace, cudaStream_t stream) {
    DepthSortArgs ds;
    int* box = nullptr;
    carve((char*)workspace, P, &ds, &box);
    ds.sorted_vis = perm;
    cudaError_t e;
    reorder_init_kernel<<<1, 32, 0, stream>>>(box, ds.counters);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((P + 255) / 256, (int64_t)num_sms() * 8));
    reorder_bounds_kernel<<<grid, 256, 0, stream>>>(in[0], P, box);
    reorder_morton_kernel<<<grid, 256, 0, stream>>>(in[0], P, box, const_cast<uint32_t*>(ds.key0), ds.counters);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_depth_sort(ds, stream)) != cudaSuccess) return e;
    for (int b = 0; b < n_buffers; ++b) {
        if (!in[b] || !out[b]) continue;
        reorder_gather_kernel<<<grid, 256, 0, stream>>>(in[b], out[b], P, n_planes, perm);
    }
    return cudaGetLastError();
}

}  // namespace ges
