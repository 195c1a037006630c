// grad_pack.cu -- SURVEY.md §8(e) view data parallelism: visible-union
// compaction of the gradient allreduce.  A particle that no view of any rank
// saw has a zero gradient on every rank, so only the planes of the union of the
// ranks' visible sets need to cross NVLink:
//   ges_mask_visible   mask[i] |= (S1 status of the frame's view == VISIBLE)
//   (the caller ORs the masks over the ranks: a MAX allreduce of P bytes)
//   ges_grad_index     idx = { i : mask[i] } ascending (block counts, one-CTA
//                      scan, in-order ballot scatter), U = |idx|
//   ges_grad_pack      packed[c][k] = grads[c][idx[k]] (planar [C][U])
//   (the caller allreduces the C U floats)
//   ges_grad_unpack    grads[c][idx[k]] = packed[c][k]
// Rows of `packed` are U apart, U read from device memory by the kernels, so
// nothing here synchronises; the host reads U once to size the allreduce.
#include <algorithm>

#include "ges_internal.h"

namespace ges {

constexpr int kGpThreads = 256;
constexpr int kGpItems = 8;
constexpr int kGpBlock = kGpThreads * kGpItems;  // mask bytes per CTA

__global__ void mask_visible_kernel(const uint8_t* status, int64_t P, uint8_t* mask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P && status[i] == GES_VISIBLE) mask[i] = 1;
}

__global__ void __launch_bounds__(kGpThreads) gp_count_kernel(const uint8_t* mask, int64_t P, int* counts) {
    __shared__ int s_w[kGpThreads / 32];
    const int64_t b0 = (int64_t)blockIdx.x * kGpBlock;
    int c = 0;
#pragma unroll
    for (int j = 0; j < kGpItems; ++j) {
        const int64_t i = b0 + j * kGpThreads + threadIdx.x;
        c += (i < P && mask[i]) ? 1 : 0;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kGpThreads / 32; ++w) t += s_w[w];
        counts[blockIdx.x] = t;
    }
}

// One CTA: exclusive scan of the block counts in place, total -> *U.
__global__ void __launch_bounds__(1024) gp_scan_kernel(int* counts, int nblocks, long long* U) {
    __shared__ int s_w[33];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int carry = 0;
    for (int base = 0; base < nblocks; base += 1024) {
        const int i = base + tid;
        const int v = i < nblocks ? counts[i] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const int wv = s_w[lane];
            int wi = wv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int n = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += n;
            }
            s_w[lane] = wi - wv;
            if (lane == 31) s_w[32] = wi;
        }
        __syncthreads();
        if (i < nblocks) counts[i] = carry + s_w[warp] + incl - v;
        carry += s_w[32];
        __syncthreads();
    }
    if (tid == 0) *U = carry;
}

// In-order scatter of the selected indices: thread-contiguous runs of kGpItems.
__global__ void __launch_bounds__(kGpThreads) gp_index_kernel(const uint8_t* mask, int64_t P, const int* offsets,
                                                             int* idx) {
    __shared__ int s_w[kGpThreads / 32 + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * kGpBlock + (int64_t)tid * kGpItems;
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < kGpItems; ++j) {
        const int64_t i = r0 + j;
        if (i < P && mask[i]) bits |= 1u << j;
    }
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        int t = 0;
        for (int w = 0; w < kGpThreads / 32; ++w) { const int x = s_w[w]; s_w[w] = t; t += x; }
    }
    __syncthreads();
    int pos = offsets[blockIdx.x] + s_w[warp] + incl - c;
#pragma unroll
    for (int j = 0; j < kGpItems; ++j)
        if ((bits >> j) & 1u) idx[pos++] = (int)(r0 + j);
}

// packed[c][k] = grads[c][idx[k]] (pack) or the reverse (unpack), k < U; plane c
// = blockIdx.y (one element per thread: every load in flight at once).
template <bool PACK>
__global__ void gp_move_kernel(float* grads, int64_t P, const int* idx, const long long* U, float* packed) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t u = *U;
    if (k >= u) return;
    const int64_t c = blockIdx.y;
    const int64_t i = __ldg(idx + k);
    if (PACK) packed[c * u + k] = __ldg(grads + c * P + i);
    else grads[c * P + i] = __ldg(packed + c * u + k);
}

int64_t grad_pack_blocks(int64_t P) { return (P + kGpBlock - 1) / kGpBlock; }

// Failure detection: *count += the number of NaN / Inf values among x[0, n).
__global__ void count_nonfinite_kernel(const float* x, int64_t n, unsigned long long* count) {
    uint32_t c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += !isfinite(__ldg(x + i));
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

cudaError_t launch_count_nonfinite(const float* x, int64_t n, unsigned long long* count, cudaStream_t stream) {
    const int64_t want = (n + 255) / 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * 8));
    count_nonfinite_kernel<<<grid, 256, 0, stream>>>(x, n, count);
    return cudaGetLastError();
}

cudaError_t launch_mask_visible(const uint8_t* status, int64_t P, uint8_t* mask, cudaStream_t stream) {
    mask_visible_kernel<<<(unsigned)((P + 255) / 256), 256, 0, stream>>>(status, P, mask);
    return cudaGetLastError();
}

cudaError_t launch_grad_index(int64_t P, const uint8_t* mask, int* counts, int* idx, long long* U,
                              cudaStream_t stream) {
    const int nb = (int)grad_pack_blocks(P);
    gp_count_kernel<<<nb, kGpThreads, 0, stream>>>(mask, P, counts);
    gp_scan_kernel<<<1, 1024, 0, stream>>>(counts, nb, U);
    gp_index_kernel<<<nb, kGpThreads, 0, stream>>>(mask, P, counts, idx);
    return cudaGetLastError();
}

cudaError_t launch_grad_pack(const float* grads, int64_t P, int C, const int* idx, const long long* U, float* packed,
                             cudaStream_t stream) {
    gp_move_kernel<true><<<dim3((unsigned)((P + 255) / 256), (unsigned)C), 256, 0, stream>>>(const_cast<float*>(grads),
                                                                                           P, idx, U, packed);
    return cudaGetLastError();
}

cudaError_t launch_grad_unpack(const float* packed, int64_t P, int C, const int* idx, const long long* U,
                               float* grads, cudaStream_t stream) {
    gp_move_kernel<false><<<dim3((unsigned)((P + 255) / 256), (unsigned)C), 256, 0, stream>>>(grads, P, idx, U,
                                                                                            const_cast<float*>(packed));
    return cudaGetLastError();
}

}  // namespace ges
