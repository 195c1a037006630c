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
    float* drgb_ddir;     // [9][P] d rgb / d unit direction (for S5b)
    uint32_t* vis_key;    // [P] depth bits, 0xffffffff if not visible
    int band_begin, band_step;  // rect rows become band rows (ges_settings tile band)
    unsigned long long* counters;
};

cudaError_t launch_preprocess(const PreprocessArgs& a, cudaStream_t stream);

// --- sort / ranges ---------------------------------------------------------
int num_sms();
constexpr int kRadixDigits = 256;

struct RadixPassArgs {
    const uint32_t* keys_in;
    const uint32_t* vals_in;          // null: the value is the input index
    uint32_t* keys_out;               // may be null
    uint32_t* vals_out;
    const unsigned long long* count;  // device item count (null: max_items)
    int64_t max_items;                // upper bound (grid sizing); items beyond are ignored
    uint32_t* tile_hist;              // [256][hist_stride] per-tile digit counts -> offsets (digit-major)
    int64_t hist_stride;              // >= number of tiles
    uint32_t* digit_total;            // [256] column totals of this pass
    int shift;
    int digit_bits;                   // bits of the digit that can be non-zero (1..8)
    int drop_invalid;                 // 1: keys == 0xffffffff are dropped (compaction)
};
cudaError_t launch_radix_pass(const RadixPassArgs& a, cudaStream_t stream);
int64_t radix_tiles(int64_t n);

struct ItemScanArgs {
    const uint32_t* sorted_vis;
    const ushort4* rect;
    unsigned long long* counters;     // reads VISIBLE; writes SLOTS, OVERFLOW
    int64_t capacity;
    uint32_t* E;                      // [P]
    uint4* items;                     // [P] packed (E, particle, rect x0|y0<<16, x1|y1<<16)
    uint32_t* chunk_first;            // [cap/chunk_slots + 1] first item of every binning chunk
    int64_t chunk_slots;              // pair slots per binning chunk (bin.cu)
    uint32_t* lookback;               // [tiles]
    unsigned long long* tile_counter;
};
cudaError_t launch_item_scan(const ItemScanArgs& a, int64_t max_items, cudaStream_t stream);
int64_t item_scan_tiles(int64_t n);

// --- direct tile binning (bin.cu) -------------------------------------------
constexpr int kBinWinTiles = 6144;    // tiles of one binning window (shared-memory cursors)
constexpr int kBinItemCost = 4;       // chunk cost of an item, in pair slots
struct BinArgs {
    const uint4* items;               // [V] item records in depth order (item scan)
    const uint32_t* chunk_first;      // [chunks + 1]
    const unsigned long long* counters;  // reads CHUNKS, OVERFLOW
    unsigned long long* counters_w;   // writes PAIRS
    uint32_t* table;                  // [cmax][T] per-(chunk, tile) counts -> offsets
    uint32_t* ranges;                 // [T+1]
    uint32_t* list;                   // [cap]
    int tiles_x, rows;                // band tiles: T = tiles_x * rows
    int64_t T;
    int win_rows;                     // tile rows per window (win_rows * tiles_x <= kBinWinTiles)
    int cmax;                         // chunk capacity (table row length, grid.x)
    int64_t chunk_slots;
    int rank_bits;                    // bits of a warp-local tile id (ballot ranking)
};
cudaError_t launch_bin(const BinArgs& a, cudaStream_t stream);

// --- render ----------------------------------------------------------------
constexpr int kGrad2dStride = 12;  // floats per particle in grad2d (3 x float4)
struct RenderFwdArgs {
    const float4* pay0;
    const float4* pay1;
    const float* pay2;
    const uint32_t* list;
    const uint32_t* ranges;
    const unsigned long long* counters;
    int W, H, tiles_x, tiles_y;       // tiles_y = the band's rows (ges_frame.band_rows)
    int band_begin, band_step;        // band tile row k is image tile row band_begin + k band_step
    float bg[3];
    float* image;
    float* final_T;
    uint32_t* n_contrib;
    uint32_t* n_eval;
    uint32_t* n_comp;
};
cudaError_t launch_render_fwd(const RenderFwdArgs& a, cudaStream_t stream);

struct RenderBwdArgs {
    const float4* pay0;
    const float4* pay1;
    const float* pay2;
    const uint32_t* list;
    const uint32_t* ranges;
    const unsigned long long* counters;
    int W, H, tiles_x, tiles_y;       // tiles_y = the band's rows (ges_frame.band_rows)
    int band_begin, band_step;        // band tile row k is image tile row band_begin + k band_step
    float bg[3];
    const float* final_T;
    const uint32_t* n_contrib;
    const float* dL_dimage;
    float* grad2d;  // [P][12]: du, dv, dA, dB | dC (pre-scaled conic), dkappa, dr, dg | db, 0, 0, 0
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
    const float* drgb_ddir;           // [9][P] from S1
    float* grad2d;
    float *g_mean, *g_log_scale, *g_quat, *g_opacity_logit, *g_sh, *g_beta;
    int accumulate;
};
cudaError_t launch_particle_bwd(const ParticleBwdArgs& a, cudaStream_t stream);

}  // namespace ges
