// ges_internal.h -- launch-argument structs shared by the kernels and the C
// ABI layer (ges_api.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ges.h"
#include "ges_device.cuh"

namespace ges {

struct PreprocessArgs {
    const float *mean, *log_scale, *quat, *opacity_logit, *sh, *beta;
    int P, sh_degree;
    float rho;
    int phi_mode, gaussian_only;
    CamParams cam;
    float* depth;
    float4* pay0;
    float4* pay1;
    float* pay2;
    int32_t* radius;
    ushort4* rect;
    uint8_t* status;
    uint8_t* flags;
    uint32_t* vis_key;
    uint32_t* vis_val;
    int32_t* tile_diff;
    uint32_t* hist;       // [4][256] depth digits
    uint32_t* lookback;   // [tiles]
    unsigned long long* counters;
};

cudaError_t launch_preprocess(const PreprocessArgs& a, cudaStream_t stream);
int64_t preprocess_lookback_words(int64_t P);

// --- sort / ranges ---------------------------------------------------------
struct RangesArgs {
    const int32_t* tile_diff;
    int tiles_x, tiles_y, tile_bits;
    uint32_t* ranges;                 // [T+1]
    uint32_t* hist;                   // [8][256]: 0-3 depth digits (in: counts, out: offsets), 4-5 tile digits
    unsigned long long* counters;
    int64_t capacity;
};
cudaError_t launch_ranges(const RangesArgs& a, cudaStream_t stream);
int ranges_smem_bytes(int tiles_x, int tiles_y);  // must be <= 200 KB
int num_sms();

struct RadixPassArgs {
    const uint32_t* keys_in;
    const uint32_t* vals_in;
    uint32_t* keys_out;               // may be null (last pass)
    uint32_t* vals_out;
    const unsigned long long* count;  // device item count
    int64_t max_items;                // upper bound (grid sizing); items beyond are ignored
    const uint32_t* digit_offset;     // [256] exclusive offsets of this pass's digits
    uint32_t* lookback;               // [tiles][256], zeroed
    unsigned long long* tile_counter; // zeroed
    int shift;
    const unsigned long long* overflow;  // if non-null and *overflow != 0: do nothing
};
cudaError_t launch_radix_pass(const RadixPassArgs& a, cudaStream_t stream);
int64_t radix_tiles(int64_t n);
constexpr int kRadixDigits = 256;

struct DuplicateArgs {
    const uint32_t* sorted_vis;       // [V] particle ids in depth order
    const ushort4* rect;
    const unsigned long long* counters;  // visible count, overflow flag
    int tiles_x;
    uint32_t* pair_tile;
    uint32_t* pair_val;
    uint32_t* lookback;               // [tiles]
    unsigned long long* tile_counter;
    int64_t max_items;
};
cudaError_t launch_duplicate(const DuplicateArgs& a, cudaStream_t stream);
int64_t duplicate_tiles(int64_t P);

// --- render ----------------------------------------------------------------
struct RenderFwdArgs {
    const float4* pay0;
    const float4* pay1;
    const float* pay2;
    const uint32_t* list;
    const uint32_t* ranges;
    const unsigned long long* counters;
    int W, H, tiles_x, tiles_y;
    float bg[3];
    float* image;
    float* final_T;
    uint32_t* n_contrib;
    uint32_t* n_eval;
};
cudaError_t launch_render_fwd(const RenderFwdArgs& a, cudaStream_t stream);

struct RenderBwdArgs {
    const float4* pay0;
    const float4* pay1;
    const float* pay2;
    const uint32_t* list;
    const uint32_t* ranges;
    const unsigned long long* counters;
    int W, H, tiles_x, tiles_y;
    float bg[3];
    const float* final_T;
    const uint32_t* n_contrib;
    const float* dL_dimage;
    float* grad2d;  // [9][P]: du, dv, dA, dB, dC (pre-scaled conic), dkappa, dr, dg, db
    int P;
};
cudaError_t launch_render_bwd(const RenderBwdArgs& a, cudaStream_t stream);

struct ParticleBwdArgs {
    const float *mean, *log_scale, *quat, *opacity_logit, *sh, *beta;
    int P, sh_degree;
    float rho;
    int phi_mode, gaussian_only;
    CamParams cam;
    const uint8_t* status;
    const uint8_t* flags;
    const float* grad2d;
    float *g_mean, *g_log_scale, *g_quat, *g_opacity_logit, *g_sh, *g_beta;
    int accumulate;
};
cudaError_t launch_particle_bwd(const ParticleBwdArgs& a, cudaStream_t stream);

}  // namespace ges
