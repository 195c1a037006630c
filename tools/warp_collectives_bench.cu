// Issue cost of warp collectives on the B200 (cycles per dependent iteration of warp 0
// with 1-32 resident warps per SM): ballot, shfl, match_any (plus the LCG that feeds them).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wc tools/warp_collectives_bench.cu && /tmp/wc
// Measured: profiles/r2d_warp_collectives.txt
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ballot(unsigned* out, int iters) {
    unsigned x = threadIdx.x * 2654435761u, acc = 0;
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = x * 1664525u + 1013904223u;
        acc += __ballot_sync(0xffffffffu, x & 0x100u);
    }
    long long c1 = clock64();
    if (acc == 7) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (unsigned)(c1 - c0);
}
__global__ void k_match(unsigned* out, int iters) {
    unsigned x = threadIdx.x * 2654435761u, acc = 0;
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = x * 1664525u + 1013904223u;
        acc += __match_any_sync(0xffffffffu, (x >> 10) & 511u);
    }
    long long c1 = clock64();
    if (acc == 7) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (unsigned)(c1 - c0);
}
__global__ void k_shfl(unsigned* out, int iters) {
    unsigned x = threadIdx.x * 2654435761u, acc = 0;
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = x * 1664525u + 1013904223u;
        acc += __shfl_sync(0xffffffffu, x, (x >> 7) & 31);
    }
    long long c1 = clock64();
    if (acc == 7) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (unsigned)(c1 - c0);
}
__global__ void k_alu(unsigned* out, int iters) {
    unsigned x = threadIdx.x * 2654435761u, acc = 0;
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = x * 1664525u + 1013904223u;
        acc += x & 0x100u;
    }
    long long c1 = clock64();
    if (acc == 7) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (unsigned)(c1 - c0);
}
int main() {
    unsigned* d; cudaMalloc(&d, 8); unsigned h[2];
    int iters = 4096;
    for (int warps : {1, 4, 8, 32}) {
        void (*ks[4])(unsigned*, int) = {k_alu, k_ballot, k_shfl, k_match};
        const char* nm[4] = {"alu", "ballot", "shfl", "match"};
        for (int k = 0; k < 4; ++k) {
            ks[k]<<<148, warps * 32>>>(d, iters);
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
            printf("warps/SM %2d %-6s cycles/iter (warp 0) %.1f\n", warps, nm[k], h[1] / (double)iters);
        }
    }
}
