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
    int kernel;                       // ges_kernel: 1 = exact GEF of Eq. 2 (no phi-bar, exact rect)
    CamParams cam;
    float* depth;
    float4* pay0;
    float4* pay1;
    float* pay2;
    float* pay3;                      // [P] beta / 2 (exact kernel)
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

// Launch setup (function attributes, occupancy-derived grids) is per device: the
// memos below are indexed by the current device.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & (kMaxDevices - 1);
}

// --- sort / ranges ---------------------------------------------------------
int num_sms();
constexpr int kRadixDigits = 512;  // max digits of a depth-sort pass (9 bits)

constexpr int kDsMaxGrid = 1024;      // max CTAs of the cooperative depth sort
constexpr int kDsMaxPasses = 4;       // 9-bit digits of a 32-bit key
constexpr int kDsMaxGroups = kDsMaxGrid / 16;  // CTA groups of the two-level pass prefix (sort.cu)

constexpr int kMaxBandRows = 256;     // tile rows of a frame (ges_frame_init: <= 256 per axis)

// Item record of a depth-sorted visible particle (sort.cu -> bin.cu): particle
// index, and its nonempty tile rect [x0, x1) x [y0, y1) packed as
// x0 | (x1 - 1) << 8 | y0 << 16 | (y1 - 1) << 24 (tile coordinates < 256).
__device__ __forceinline__ uint32_t pack_rect(uint32_t x0, uint32_t y0, uint32_t x1, uint32_t y1) {
    return x0 | ((x1 - 1u) << 8) | (y0 << 16) | ((y1 - 1u) << 24);
}

struct DepthSortArgs {
    const uint32_t* key0;             // [P] preprocess keys: depth bits, 0xffffffff = not visible
    uint32_t* keys[2];                // [P] ping-pong (keys[0] may not alias key0; keys[1] may)
    uint32_t* vals[2];                // [P] ping-pong
    uint32_t* sorted_vis;             // [V] out: visible particles in (depth bits, index) order
    uint32_t* st_cnt;                 // [kDsMaxPasses][kDsMaxGrid][512] published per-CTA digit counts
    uint32_t* gt_cnt;                 // [kDsMaxPasses][kDsMaxGroups][512] published group totals
    int64_t P;
    int G;                            // grid (set by the launcher)
    uint32_t key_base;                // fp32 bits of near_z: every visible key is larger
    const ushort4* rect;
    uint2* items;                     // [V] out: (particle, pack_rect) in depth order (null: plain sort)
    uint32_t* row_count;              // [rows] out (+=): items covering each band row (zeroed per frame)
    int rows;                         // band rows (<= kMaxBandRows)
    unsigned long long* counters;     // reads VISIBLE, KEYMAX; adds SLOTS
};
cudaError_t launch_depth_sort(const DepthSortArgs& a, cudaStream_t stream);

// --- particle storage order (reorder.cu) --------------------------------------
size_t reorder_workspace_bytes(int64_t P);
cudaError_t launch_reorder(const float* const* in, float* const* out, int n_buffers, int64_t P, int n_planes,
                           uint32_t* perm, void* workspace, cudaStream_t stream);

// --- row-then-column binning (bin.cu) ----------------------------------------
#ifndef GES_ROW_CHUNK
#define GES_ROW_CHUNK 2048
#endif
constexpr int kRowChunk = GES_ROW_CHUNK;  // items per row-binning CTA
constexpr int kTileBuckets = 64;          // S5a launch-order cost buckets (ges_frame.tile_order)
#ifndef GES_COL_CHUNK
#define GES_COL_CHUNK 3072
#endif
constexpr int kColChunk = GES_COL_CHUNK;  // row-list entries per column-binning CTA
struct BinArgs {
    const uint2* items;               // [V] depth-ordered item records (sort.cu)
    const uint32_t* row_count;        // [rows] items covering each row (sort.cu)
    uint2* rowlist;                   // [cap] per-row lists of (particle, x0 | (x1 - 1) << 8)
    uint32_t* lb_rows;                // [2][row_chunks][rows] published words (zeroed per frame)
    uint32_t* lb_cols;                // [2][col_chunks][tiles_x] published words (zeroed per frame)
    uint32_t* col_excl;               // [col_chunks][tiles_x] per-chunk exclusive column offsets
    uint32_t* tile_count;             // [rows][tiles_x] pairs per tile (zeroed per frame)
    uint32_t* row_pairs;              // [rows] pairs per row (zeroed per frame)
    uint32_t* ranges;                 // [T+1]
    uint32_t* list;                   // [cap]
    unsigned long long* counters;     // reads VISIBLE, SLOTS; writes OVERFLOW, PAIRS; tickets
    int tiles_x, rows;                // band tiles: T = tiles_x * rows
    int64_t capacity;                 // pair capacity
    int64_t row_chunks, col_chunks;   // capacities of the look-back words
};
cudaError_t launch_bin(const BinArgs& a, cudaStream_t stream);
cudaError_t launch_count_nonfinite(const float* x, int64_t n, unsigned long long* count, cudaStream_t stream);

// --- render ----------------------------------------------------------------
constexpr int kGrad2dStride = 12;  // floats per particle in grad2d (3 x float4)
struct RenderFwdArgs {
    const float4* pay0;
    const float4* pay1;
    const float* pay2;
    const float* pay3;                // beta / 2 (exact kernel)
    int exact;                        // 1: exact GEF kernel of Eq. 2
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
    uint32_t* tile_bucket;            // [kTileBuckets] (ges_frame.tile_order)
    uint32_t* tile_order;             // [kTileBuckets][gridDim]
};
cudaError_t launch_render_fwd(const RenderFwdArgs& a, cudaStream_t stream);

struct RenderBwdArgs {
    const float4* pay0;
    const float4* pay1;
    const float* pay2;
    const float* pay3;                // beta / 2 (exact kernel)
    int exact;                        // 1: exact GEF kernel of Eq. 2
    const uint32_t* list;
    const uint32_t* ranges;
    const unsigned long long* counters;
    int W, H, tiles_x, tiles_y;       // tiles_y = the band's rows (ges_frame.band_rows)
    int band_begin, band_step;        // band tile row k is image tile row band_begin + k band_step
    float bg[3];
    const float* final_T;
    const uint32_t* n_contrib;
    const float* dL_dimage;
    float* grad2d;  // [P][12]: du, dv, dA, dB | dC (pre-scaled conic), dkappa, dr, dg | db, dbeta*, 0, 0
                    // (* exact kernel: Eq. 2's direct dL/dbeta)
    int P;
    const uint32_t* tile_bucket;      // S4's cost buckets: launch the costliest tiles first
    const uint32_t* tile_order;
    int use_order;
};
cudaError_t launch_render_bwd(const RenderBwdArgs& a, cudaStream_t stream);

struct ParticleBwdArgs {
    const float *mean, *log_scale, *quat, *opacity_logit, *sh, *beta;
    int P, sh_degree;
    float rho;
    int phi_mode, gaussian_only;
    int kernel;                       // 1: exact GEF (no phi-bar; record[9] = direct dL/dbeta)
    CamParams cam;
    const uint8_t* status;
    const uint8_t* flags;
    const float* drgb_ddir;           // [9][P] from S1
    float* grad2d;
    float *g_mean, *g_log_scale, *g_quat, *g_opacity_logit, *g_sh, *g_beta;
    float* g_mean2d;                  // optional [2][P] dL/d(u, v)
    float* g_drgb;                    // optional [3][P] dL/d rgb (clamped channels 0)
    int accumulate;
};
cudaError_t launch_particle_bwd(const ParticleBwdArgs& a, cudaStream_t stream);
cudaError_t launch_sh_from_colour(const float* mean, int64_t P, int sh_degree, const float* cams, int n_views,
                                  const float* drgb, float* g_sh, int accumulate, cudaStream_t stream);

// --- loss front end (loss.cu) ------------------------
struct LossArgs {
    const float* image;               // [3][H][W]
    const float* gt;                  // [3][H][W]
    const uint8_t* mask_lo;           // [Hd][Wd] M_omega on the downsampled grid (null: no L_omega term)
    int W, H, Hd, Wd;
    float lambda_ssim, lambda_omega;
    float inv_n;                      // 1 / (3 H W)
    float *d_mu, *d_e2, *d_exy;       // [3][H][W] SSIM partials (workspace)
    float* partial;                   // [blocks][3] block sums (workspace)
    int nblocks;
    float* dL_dimage;                 // [3][H][W] out
    float* loss_out;                  // [4] out: total, L1, SSIM, L_omega
};
cudaError_t launch_loss(const LossArgs& a, cudaStream_t stream);
int64_t loss_partials(int W, int H);

struct MaskArgs {
    const float* gt;                  // [3][H][W]
    int W, H, Hd, Wd;
    int r1, r2;                       // blur radii ceil(3 sigma) of sigma1 = 0.2 + 20 w, sigma2 = 0.1 + 10 w
    float ih1, ih2;                   // 1 / (2 sigma^2)
    float eps;
    int complement;                   // omega <= 0.5
    float *lo, *h1, *h2, *dog;        // [Hd][Wd] workspace
    unsigned* minmax;                 // [2] workspace
    uint8_t* mask_lo;                 // [Hd][Wd] out
};
cudaError_t launch_mask(const MaskArgs& a, cudaStream_t stream);

// --- optimizer and density control (train.cu) ----------
struct AdamArgs {
    float* params;                    // [n_planes][P]
    const float* grads;
    float *m, *v;
    int64_t P;
    int n_planes;
    float lr_position, lr_scaling, lr_rotation, lr_opacity, lr_feature_dc, lr_feature_rest, lr_shape;
    float beta1, beta2, eps, inv_bc1, inv_bc2;
};
cudaError_t launch_adam(const AdamArgs& a, cudaStream_t stream);
cudaError_t launch_adam_range(const AdamArgs& a, int64_t begin, int64_t count, cudaStream_t stream);
cudaError_t launch_reset(float* params, int64_t P, int plane, float cap, int mode, cudaStream_t stream);

struct DensifyStatsArgs {
    const uint8_t* status;
    const float* grad2d;              // the frame's [P][12] raw-moment records after S5a
    const float4 *pay0, *pay1;        // S1 payload: conic a, b (pay0.zw), c, kappa (pay1.xy)
    const float* pay3;                // beta / 2 (exact kernel)
    float *accum, *count;             // [P]
    int64_t P;
    int W, H, kernel;
};
cudaError_t launch_densify_stats(const DensifyStatsArgs& a, cudaStream_t stream);

struct DensifyArgs {
    const float *params, *m, *v;      // [n_planes][P]
    const float *accum, *count;       // [P]
    int64_t P, cap_out;
    int n_planes;
    float grad_threshold, percent_dense, extent, opacity_prune, shape_prune, rho;
    unsigned long long seed;
    float *params_out, *m_out, *v_out;  // [n_planes][cap_out]
    uint8_t* action;                  // [P] workspace
    int* block_cnt;                   // [3 blocks] workspace
    long long* totals;                // [3] workspace
    long long* P_out;                 // device: the new particle count
    int nblocks;
};
cudaError_t launch_densify_prune(const DensifyArgs& a, cudaStream_t stream);
int64_t densify_blocks(int64_t P);

// --- NEXT-4: 1-D mixtures and Theorem 1 (mix1d.cu) ------------------------
struct MixArgs {
    const ges_mix_run* runs;
    int n_runs, stride;
    float* params;
    float *m, *v;            // Adam moments (fit)
    float* grad;             // eval: [R][stride] or null
    float* loss;             // [R]
    const float* targets;    // [T][n]
    float x_lo, h;
    int n;
    int steps, t0;
    float lr, b1, b2, eps;
};
cudaError_t launch_mix_signal(int kind, float width, float x_lo, float h, int n, float* y, cudaStream_t stream);
cudaError_t launch_mix(const MixArgs& a, bool fit, cudaStream_t stream);
cudaError_t launch_mufu_probe(float* out, int iters, int blocks, cudaStream_t stream);
cudaError_t launch_theorem1(const float* alpha, int na, const float* beta, int nb, float A, float L, int n, float* E,
                            cudaStream_t stream);

// --- view-DP gradient compaction (grad_pack.cu) -----------------------------
int64_t grad_pack_blocks(int64_t P);
cudaError_t launch_mask_visible(const uint8_t* status, int64_t P, uint8_t* mask, cudaStream_t stream);
cudaError_t launch_grad_index(int64_t P, const uint8_t* mask, int* counts, int* idx, long long* U,
                              cudaStream_t stream);
cudaError_t launch_grad_pack(const float* grads, int64_t P, int C, const int* idx, const long long* U, float* packed,
                             cudaStream_t stream);
cudaError_t launch_grad_unpack(const float* packed, int64_t P, int C, const int* idx, const long long* U,
                               float* grads, cudaStream_t stream);

}  // namespace ges
