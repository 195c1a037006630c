/* include/ges.h -- C ABI of the B200-native GES tile rasterizer (libges.so).
 *
 * GES = Generalized Exponential Splatting, arXiv 2402.10128 (/root/reference/
 * PAPER.md).  The library implements the data-parallel hot path named by
 * BASELINE.json:north_star, every stage as hand-written sm_100a CUDA:
 *
 *   ges_preprocess  S1  per particle: Sigma = R S S^T R^T with S scaled by
 *                       phi-bar(beta) (Eq. 4 :268-270;
 *                       Eq. 6 :291-293), EWA projection Sigma' = J W Sigma W^T J^T
 *                       (PAPER.md:249-253), SH colour and opacity kappa
 *                       (PAPER.md:247), screen radius and 16x16-tile rect;
 *                       depth keys, digit histograms and the per-tile pair
 *                       counts (2-D difference grid of the rects).
 *   ges_sort        S2  depth radix sort of the visible particles (pass 0
 *                       compacts them), then every (tile, particle) pair is
 *                       written once into its tile's list; each list is in
 *                       the order of the keys (tile_id << 32 | fp32 bits of
 *                       depth), ties by particle index.
 *                   S3  per-tile ranges [ranges[t], ranges[t+1]).
 *   ges_render_fwd  S4  per 16x16 tile front-to-back alpha compositing with
 *                       early termination on transmittance (Eq. 3,
 *                       PAPER.md:259-266; constants DESIGN.md R7).
 *   ges_render_bwd  S5  adjoint of S4 per tile, then the per-particle chain
 *                       to mean, log-scale, quaternion, opacity logit, SH and
 *                       beta ("optimization ... encompasses the beta parameter
 *                       as well as position, opacity, covariance, SH",
 *                       PAPER.md:351).
 *
 * Conventions (every entry point):
 *   - Pointers are DEVICE pointers unless the name says *_host.  The caller
 *     owns every buffer; the library never allocates or frees and keeps no
 *     global state (re-entrant across distinct frames).  All work is
 *     stream-ordered on `stream` (a cudaStream_t passed as void*; NULL = the
 *     legacy default stream) and CUDA-graph capturable; only ges_counts_get
 *     synchronises.
 *   - Particles: planar SoA fp32 [C][P] (plane c of particle i at ptr[c*P+i]):
 *       mean[3][P]; log_scale[3][P]; quat[4][P] (w,x,y,z; any non-zero norm);
 *       opacity_logit[P] (kappa = sigmoid); sh[3K][P] (plane 3k+channel,
 *       K = (sh_degree+1)^2, real SH, Condon-Shortley phase, rgb = sum + 0.5,
 *       clamped >= 0); beta[P] = the TRUE shape parameter (the paper stores
 *       beta - 2: a storage shift only).
 *   - Camera: world->camera rotation R (row-major) and translation t, OpenCV
 *     axes (x right, y down, z forward), pinhole fx, fy, cx, cy in pixels;
 *     pixel (row i, col j) samples the point (j+0.5, i+0.5).
 *   - Images are planar fp32 [3][H][W], linear, unclamped.
 *   - Errors: argument errors return GES_ERR_INVALID_ARG before any launch;
 *     launch failures return GES_ERR_CUDA.  A frame whose pair-slot count
 *     (sum of rect areas) exceeds its capacity sets counts.overflow;
 *     ges_sort then writes no pairs and the renders draw nothing: the caller
 *     regrows the workspace (ges_workspace_bytes with a larger capacity) and
 *     re-runs.
 */
#ifndef GES_H_
#define GES_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GES_OK = 0,
    GES_ERR_INVALID_ARG = 1,
    GES_ERR_CAPACITY = 2,
    GES_ERR_CUDA = 3,
    GES_ERR_UNSUPPORTED = 4
} ges_status;

/* DESIGN.md R1: phi-bar scales the 3-D scale vector (SCALE: s_eff = phi s,
 * following "the scales matrix ... modified by phi") or
 * the variance (VARIANCE: s_eff = sqrt(phi) s, following Eq. 4's "effective
 * variance").  Both are the identity at beta = 2. */
typedef enum { GES_PHI_SCALE = 0, GES_PHI_VARIANCE = 1 } ges_phi_mode;

/* Per-particle status written by ges_preprocess into frame.status. */
typedef enum { GES_VISIBLE = 0, GES_CULL_NEAR = 1, GES_DEGENERATE = 2, GES_OFFSCREEN = 3 } ges_particle_status;

typedef struct {
    int64_t P;          /* number of particles, 1 <= P <= 2^31 - 1           */
    int32_t sh_degree;  /* 0..3                                              */
    int32_t _pad;
    const float *mean, *log_scale, *quat, *opacity_logit, *sh, *beta;
} ges_particles;

typedef struct {
    int32_t width, height;      /* pixels, each <= 4096 (16x16 tiles, <= 256 per axis) */
    float fx, fy, cx, cy;       /* pinhole intrinsics (pixels)               */
    float near_z;               /* particles with camera z <= near_z culled  */
    float R[9];                 /* world -> camera rotation, row-major       */
    float t[3];
} ges_camera;

typedef struct {
    float rho;                  /* shape strength of Eq. 6 (paper: 0.1); >= 0 */
    int32_t phi_mode;           /* ges_phi_mode                                              */
    int32_t gaussian_only;      /* 1: beta ignored (phi = 1) -- the equivalent Gaussian rasterizer */
    float background[3];
    /* Screen-tile band (BASELINE config 3 "the 8 GPUs splitting
     * screen-tile bands of one frame"): render only the tile rows
     * r = tile_row_begin + k * tile_row_step.  (0, 0) and (0, 1) = the full frame;
     * otherwise 0 <= tile_row_begin < tile_row_step.  ges_preprocess records the band
     * in the frame; ges_render_* require the same band.  Per-tile lists and pixels
     * of a band are identical to the full frame's; pixels outside it are untouched;
     * the S5 gradients of all bands sum to the full frame's. */
    int32_t tile_row_begin, tile_row_step;
    /* Per-pixel kernel (ges_kernel).  GES_KERNEL_PHI_GAUSS (0): the paper's
     * rasterization -- a Gaussian of the phi-bar-scaled covariance
     * (R6).  GES_KERNEL_EXACT_BETA (1): Eq. 2 itself
     * (SURVEY.md §8(f) NEXT-3): no phi-bar, per pixel
     * alpha = min(0.99, kappa exp(-1/2 Q^(beta/2))), Q the Mahalanobis form of the
     * dilated Sigma2D; rects bound Q <= (2 ln(255 kappa / 0.98))^(2/beta); the
     * backward adds Eq. 2's direct dL/dbeta.  beta must be > 0 (else the particle
     * is GES_DEGENERATE).  gaussian_only is ignored in this mode. */
    int32_t kernel;
} ges_settings;

typedef enum { GES_KERNEL_PHI_GAUSS = 0, GES_KERNEL_EXACT_BETA = 1 } ges_kernel;

/* Gradients, planar [C][P] fp32 in the parameter layout.  accumulate = 1 adds
 * into the buffers (several views before one allreduce), 0 overwrites. */
typedef struct {
    float *mean, *log_scale, *quat, *opacity_logit, *sh, *beta;
    float *mean2d;          /* optional (NULL: not written): [2][P] dL/d(u, v), the gradient of
                               the projected mean in pixels (the view-space gradient of 3DGS's
                               densification; 0 for particles that are not visible) */
    float *drgb;            /* optional (NULL: not written): [3][P] dL/d rgb of the view (0 for a
                               clamped channel or a particle that is not visible): with the camera
                               it determines this view's SH gradient (ges_sh_grad_from_colour);
                               = or += with accumulate like every other output */
    int32_t accumulate;
    int32_t _pad;
} ges_grads;

typedef struct {
    int64_t visible;    /* particles with status GES_VISIBLE                        */
    int64_t pairs;      /* M = (tile, particle) pairs in the per-tile lists          */
    int64_t slots;      /* sum over visible particles of their rect areas (>= M)     */
    int64_t capacity;   /* pair capacity of the frame                               */
    int64_t culled_near;/* particles with status GES_CULL_NEAR                       */
    int64_t degenerate; /* particles with status GES_DEGENERATE                      */
    int64_t offscreen;  /* particles with status GES_OFFSCREEN                       */
    int32_t overflow;   /* 1 if slots > capacity: lists and images are invalid       */
    int32_t _pad;
} ges_counts;

/* Counter slots inside frame.counters (uint64). */
enum {
    GES_CTR_VISIBLE = 0,  /* V: visible particles                                 */
    GES_CTR_PAIRS = 1,    /* M: (tile, particle) pairs in the lists (R8/R10)        */
    GES_CTR_OVERFLOW = 2, /* 1 if SLOTS > pair capacity                             */
    GES_CTR_SLOTS = 3,    /* rect pairs = sum of rect areas (pair-slot count)       */
    GES_CTR_TICKET = 4,   /* scratch: chunk tickets of the row binning              */
    GES_CTR_TICKET_COLS = 5, /* scratch: chunk tickets of the column counts         */
    GES_CTR_TICKET_EMIT = 6, /* scratch: chunk tickets of the column binning        */
    GES_CTR_KEYMAX = 7,   /* largest visible depth key (depth sort pass plan)       */
    GES_CTR_CULLED_NEAR = 8, /* particles behind the near plane                      */
    GES_CTR_DEGENERATE = 9,  /* non-finite / singular particles                      */
    GES_CTR_OFFSCREEN = 10,  /* particles whose rect misses the frame (or band)      */
    GES_CTR_N = 24           /* (slots 16-23: debug timers of instrumented builds)   */
};

/* A frame: every per-frame device array, carved by ges_frame_init out of ONE
 * caller-owned device workspace.  The struct lives in caller (host) memory;
 * its fields are public so that tests can read the intermediate arrays. */
typedef struct {
    int64_t P, pair_capacity;
    int32_t width, height, tiles_x, tiles_y, num_tiles, tile_bits;
    int32_t sh_degree_max;
    int32_t kernel;                /* ges_kernel of the last ges_preprocess (renders must match) */
    int32_t band_begin, band_step; /* tile rows of this frame: band_begin + k band_step (ges_settings) */
    int32_t band_rows;             /* k < band_rows; the lists and ranges index band tiles
                                      t = k * tiles_x + tx, and rect rows are band rows k  */
    uint32_t depth_key_base;       /* fp32 bits of the last ges_preprocess camera's near_z: every
                                      visible depth key is larger (depth sort digit base)  */
    /* ---- S1 per-particle state ---- */
    float *depth;          /* [P] camera-space z                                       */
    float *pay0;           /* [P][4] (u, v, a, b): projected mean, conic a, b           */
    float *pay1;           /* [P][4] (c, kappa, r, g): conic c, opacity, colour r, g    */
    float *pay2;           /* [P]    colour b                                           */
    float *pay3;           /* [P]    beta / 2 (exact GEF kernel only)                    */
    int32_t *radius;       /* [P] screen radius (pixels)                                */
    uint16_t *rect;        /* [P][4] tile rect x0, y0, x1, y1 (exclusive ends)           */
    uint8_t *status;       /* [P] ges_particle_status                                   */
    uint8_t *flags;        /* [P] bit0-2 rgb clamped at 0, bit3/4 Jacobian x/y clamped   */
    float *drgb_ddir;      /* [9][P] d rgb_c / d u_d (u: unit view direction, dY/du of the
                              SH polynomials), plane 3c + d; 0 where rgb_c is clamped
                              or the particle is not visible (read by S5b)            */
    /* ---- S2 depth sort of the visible particles ---- */
    uint32_t *vis_key[2];  /* [P] depth bits (0xffffffff = not visible), ping-pong */
    uint32_t *vis_val[2];  /* [P] particle index, ping-pong                      */
    uint32_t *sorted_vis;  /* [V] visible particles in (depth, index) order             */
    /* ---- S2 radix scratch (depth passes) ---- */
    uint32_t *radix_hist;  /* [4][1024][512] u32 per-CTA digit counts of each pass, then
                              [4][64][512] group totals, published with a flag bit       */
    /* ---- S2 pairs and S3 ranges: row-then-column binning ---- */
    uint32_t *items;       /* [P][2] depth-ordered visible particles: (particle,
                              x0 | (x1-1) << 8 | y0 << 16 | (y1-1) << 24) of the rect */
    uint32_t *row_count;   /* [tiles_y] items covering each band row (zeroed per frame) */
    uint32_t *rowlist;     /* [cap][2] row lists: row r = the items covering r in depth
                              order, at the exclusive prefix of row_count; entries
                              (particle, x0 | (x1-1) << 8)                            */
    uint32_t *tile_count;  /* [T] pairs per tile (zeroed per frame)                   */
    uint32_t *row_pairs;   /* [tiles_y] pairs per band row (zeroed per frame)         */
    uint32_t *tile_bucket; /* [64] tiles per backward-cost bucket, appended by S4 (zeroed
                              per frame; see tile_order)                             */
    uint32_t *lb_rows;     /* [2][row_chunks][tiles_y] published chunk / group words of
                              the row binning (zeroed per frame)                      */
    uint32_t *lb_cols;     /* [2][col_chunks][tiles_x] published words of the column
                              counts (zeroed per frame)                               */
    uint32_t *col_excl;    /* [col_chunks][tiles_x] offset of each column chunk inside
                              its tiles' lists                                        */
    int64_t row_chunks;    /* ceil(P / 2048): item chunks of the row binning           */
    int64_t col_chunks;    /* ceil(cap / 3072) + tiles_y: row-list chunks (bound)      */
    uint32_t *list;        /* [cap] per-tile lists: tile t = list[ranges[t] .. ranges[t+1]) */
    uint32_t *ranges;      /* [T+1]                                               */
    uint64_t *counters;    /* [GES_CTR_N]                                         */
    size_t zero_bytes;     /* bytes from `counters` zeroed at the start of a frame */
    /* ---- S4 / S5 ---- */
    float *final_T;        /* [H*W] transmittance after the last composited particle   */
    uint32_t *n_contrib;   /* [H*W] list position of the last composited particle + 1  */
    uint32_t *tile_order;  /* [64][T] S5a launch order: S4 appends each tile to the bucket
                              of its backward cost (the longest backward walk: the tile's
                              largest n_contrib, on a 4-per-octave log scale); S5a's
                              CTA b takes the b-th tile of the
                              buckets in descending cost (costliest first: a shorter tail),
                              or tile b when the buckets do not hold exactly T tiles
                              (S4 run twice on one frame).  Only an order: any permutation
                              gives the same sums up to float atomics order             */
    float *grad2d;         /* [P][12] per-particle S5a record: raw moments over the
                              particle's composited pixels (dx = u - px, dy = v - py),
                              (sum m dx, sum m dy, sum m dx^2, sum m dx dy |
                              sum m dy^2, K, dr, dg | db, Sb, 0, 0); Gaussian kernel
                              m = kappa G dL/dalpha, K = kappa dL/dkappa; exact kernel
                              m = G dL/dalpha Q^(beta/2) / qp, K = dL/dkappa, Sb =
                              sum G dL/dalpha Q^(beta/2) log2 Q.  S5b turns them into
                              dL/d(u, v, conic, kappa) with the per-particle factors
                              (kappa, beta, the conic).  Kept all-zero between backward
                              passes */
    size_t workspace_bytes;
} ges_frame;

/* Bytes of device workspace a frame needs (256-byte aligned base). */
size_t ges_workspace_bytes(int64_t P, int32_t width, int32_t height, int64_t pair_capacity);

/* Carve `frame` out of `workspace` (device, >= ges_workspace_bytes(...) bytes,
 * 256-byte aligned).  Host-only; no device work.  The workspace must be
 * zero-filled once before the frame's first ges_render_bwd (the backward
 * keeps frame.grad2d zero between calls instead of clearing it per frame). */
ges_status ges_frame_init(void *workspace, size_t bytes, int64_t P, int32_t width, int32_t height,
                          int64_t pair_capacity, ges_frame *frame);

/* The frame's sub-arrays as (byte offset from the workspace base, bytes) pairs,
 * extents[2 i], extents[2 i + 1], in carving order: counters, row_count,
 * tile_count, row_pairs, lb_rows, lb_cols (the zero-per-frame region), depth, pay0, pay1, pay2, pay3, radius, rect, status, flags,
 * drgb_ddir, vis_key[0], vis_val[0], vis_key[1], vis_val[1], sorted_vis,
 * radix_hist, items, rowlist, col_excl, list, ranges, final_T, n_contrib,
 * grad2d.  Each array starts 256-byte aligned; the bytes
 * between one array's end and the next one's start are padding that no
 * kernel touches (tests poison them to detect out-of-bounds writes).  Host-only.
 * *count = the number of arrays; GES_ERR_CAPACITY if it exceeds `capacity`
 * (extents then holds the first `capacity`).  extents may be NULL when
 * capacity is 0 (query the count). */
ges_status ges_frame_layout(const ges_frame *frame, int64_t *extents, int32_t capacity, int32_t *count);

/* S1.  Writes the per-particle state, the visible list and the tile
 * histogram of `frame`.  particles/camera/settings are host structs whose
 * array pointers are device pointers; camera must match the frame size. */
ges_status ges_preprocess(const ges_particles *particles, const ges_camera *camera, const ges_settings *settings,
                          ges_frame *frame, void *stream);

/* S2 + S3.  Depth sort, pair duplication, tile sort, ranges. */
ges_status ges_sort(ges_frame *frame, void *stream);

/* S4.  image: [3][H][W] fp32 (device).  Also writes frame.final_T and
 * frame.n_contrib.  Optional diagnostics ([H*W] u32 each, may be NULL):
 * n_eval = list entries each pixel evaluated (up to and including the one that
 * stopped it), n_comp = entries it composited (alpha >= 1/255, before the stop)
 * -- the algorithmic work of S4 and S5. */
ges_status ges_render_fwd(ges_frame *frame, const ges_settings *settings, float *image, uint32_t *n_eval,
                          uint32_t *n_comp, void *stream);

/* S5 = S5a then S5b.  dL_dimage: [3][H][W] fp32 (device); gradients of
 * L = <dL_dimage, image> w.r.t. every particle parameter go to `grads`.
 * Needs the frame's S1-S4 state (same particles, camera, settings). */
ges_status ges_render_bwd(const ges_particles *particles, const ges_camera *camera, const ges_settings *settings,
                          ges_frame *frame, const float *dL_dimage, const ges_grads *grads, void *stream);

/* S5a alone: the per-tile adjoint of S4 (Eq. 3); adds the 2-D gradients
 * into frame.grad2d. */
ges_status ges_render_bwd_tiles(const ges_settings *settings, ges_frame *frame, const float *dL_dimage,
                                void *stream);

/* S5b alone: chain frame.grad2d to the parameters (mean, log-scale,
 * quaternion, opacity logit, SH, beta through phi-bar, Eq. 6) and reset
 * frame.grad2d to zero. */
ges_status ges_backward_particles(const ges_particles *particles, const ges_camera *camera,
                                  const ges_settings *settings, ges_frame *frame, const ges_grads *grads,
                                  void *stream);

/* Copies the frame's counts to host memory.  Synchronises `stream`. */
ges_status ges_counts_get(const ges_frame *frame, ges_counts *host_out, void *stream);

const char *ges_status_string(ges_status s);

/* Library version / build id (static string). */
const char *ges_version(void);

/* ------------------------------------------------------------------------
 * Image-loss front end: Eq. 9
 *   L = l_L1 L1 + l_ssim (1 - SSIM) + l_w L_omega,  l_L1 = 1 - l_ssim - l_w,
 * with L_omega = ||(I - I_gt) . M_omega||_1 (Eq. 8) and the
 * frequency mask M_omega of Eq. 7 (complement for omega <= 0.5
 * :327, computed on a downsampled ground truth :1226).  Readings (DESIGN.md
 * R22-R28): every term a mean over pixels and channels; SSIM with an 11 x 11
 * Gaussian window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, zero padding; the mask
 * from the luminance 0.299 R + 0.587 G + 0.114 B, bilinear downsample to
 * max(1, floor(n s + 1/2)) per axis, DoG = G(., 0.2 + 20 w) - G(., 0.1 + 10 w)
 * (separable, radius ceil(3 sigma), reflect padding), |DoG| min-max normalised
 * (a constant response gives 0), > eps_omega; nearest upsample (full-res pixel
 * (i, j) reads mask_lo[floor(i Hd / H), floor(j Wd / W)]).
 * Images are [3][H][W] fp32 device arrays; the caller owns every buffer and a
 * device workspace of ges_loss_workspace_bytes(); stream-ordered, no sync.
 * ------------------------------------------------------------------------ */
typedef struct {
    float lambda_ssim;   /* 0.2 */
    float lambda_omega;  /* 0.5        */
    float eps_omega;     /* 0.5         */
    float downsample;    /* 0.2        */
} ges_loss_settings;

/* Downsampled mask grid of a W x H image: Wd = max(1, floor(W s + 1/2)), same for H. */
ges_status ges_loss_mask_dims(int32_t width, int32_t height, float downsample, int32_t *Wd, int32_t *Hd);

/* Device workspace bytes for ges_loss_mask and ges_loss on a W x H image. */
size_t ges_loss_workspace_bytes(int32_t width, int32_t height, float downsample);

/* M_omega of `gt` for normalised frequency omega in [0, 1] (the schedule
 * omega = iteration / iterations) into mask_lo [Hd][Wd] (u8 0/1).
 * Errors: null pointers, W/H < 1, omega outside [0, 1], workspace too small. */
ges_status ges_loss_mask(const float *gt, int32_t width, int32_t height, float omega, const ges_loss_settings *settings,
                         void *workspace, size_t workspace_bytes, uint8_t *mask_lo, void *stream);

/* ------------------------------------------------------------------------
 * Optimizer and shape-aware density control (
 * PAPER.md §4.4 :348-358, Appendix :1227-1271; readings DESIGN.md R29-R33).
 * Parameter, gradient and Adam-moment buffers are planar fp32 [C][P] in the
 * ges_particles order (mean 3, log_scale 3, quat 4, opacity_logit 1, sh 3K,
 * beta 1; C = 12 + 3K), device, caller-owned; stream-ordered.
 * ------------------------------------------------------------------------ */
typedef struct {
    int32_t step;                 /* 1-based Adam step (bias correction)                          */
    float lr_position;            /* ges_lr_position(step, ...) (:1232-1236)                      */
    float lr_scaling, lr_rotation, lr_opacity; /* 0.005, 0.001, 0.05 (:1238-1242)                */
    float lr_feature_dc, lr_feature_rest;      /* 0.0025 and 0.0025 / 20 (SH DC / higher bands)  */
    float lr_shape;               /* 0.001 (:1242; :397 says 0.0015, R20)                          */
    float beta1, beta2, eps;      /* 0.9, 0.999, 1e-15                                             */
} ges_adam_settings;

/* Log-linear position learning rate init -> final over max_steps (delay multiplier
 * ramp over delay_steps; none for 0), the schedule of PAPER.md:1232-1236.  Host. */
double ges_lr_position(int64_t step, double init, double final_, double delay_mult, int64_t max_steps,
                       int64_t delay_steps);

/* One bias-corrected Adam step of every plane (params, m, v updated in place). */
ges_status ges_adam_step(float *params, const float *grads, float *m, float *v, int64_t P, int32_t sh_degree,
                         const ges_adam_settings *settings, void *stream);

/* The same step on the contiguous range [begin, begin + count) of the flattened
 * [C][P] buffers only (a ZeRO-1 optimizer shard of data-parallel training, each
 * rank updating 1/N of the parameters after a reduce-scatter of the gradients):
 * params, m, v are the FULL buffers, grads_range holds the range's count gradient
 * values (element i <-> flat index begin + i).  Elementwise identical to
 * ges_adam_step on those entries.  begin + count must not exceed C P. */
ges_status ges_adam_step_range(float *params, const float *grads_range, float *m, float *v, int64_t P,
                               int32_t sh_degree, const ges_adam_settings *settings, int64_t begin, int64_t count,
                               void *stream);

/* Particle storage order (not a step of the hot path):
 * permutes the planar [C][P] parameter buffer (and, if given, the Adam moments
 * m, v) into the Morton order of the particle means -- each axis quantised to
 * 1024 cells of the means' bounding box, bits interleaved, ties in index order
 * (a stable sort: the permutation is deterministic).  Call after loading a
 * scene and after every ges_densify_prune: culled particles then come in runs,
 * which S1 and S5b skip a 128-particle tile at a time.  perm_out[j] = the old
 * index of the particle now at j (device, [P]).  Out-of-place (in != out).
 * workspace: device, >= ges_reorder_workspace_bytes(P), 256-B aligned. */
size_t ges_reorder_workspace_bytes(int64_t P);
ges_status ges_reorder(const float *params, float *params_out, const float *m, float *m_out, const float *v,
                       float *v_out, int64_t P, int32_t sh_degree, uint32_t *perm_out, void *workspace, size_t bytes,
                       void *stream);

/* Opacity reset (what = 0): logit <- min(logit, logit(0.01)); shape reset (what = 1):
 * beta <- 2 (PAPER.md:1253 intervals; targets R30). */
ges_status ges_reset(float *params, int64_t P, int32_t sh_degree, int32_t what, void *stream);

/* Densification statistic of one view, between ges_render_bwd_tiles (S5a) and
 * ges_backward_particles (S5b): for every visible particle accum += |(du W/2,
 * dv H/2)| (the view-space gradient in NDC units) and count += 1 (R32). */
ges_status ges_densify_stats(const ges_frame *frame, float *accum, float *count, void *stream);

typedef struct {
    float grad_threshold;   /* 3e-4 (:1250)                                */
    float percent_dense;    /* 0.01 (:1246)                                */
    float scene_extent;     /* clone if max exp(log s) <= percent_dense x this */
    float opacity_prune;    /* 0.005 (:1248)                               */
    float shape_prune;      /* prune if phi-bar_rho(beta) < this: 0.5 (:397; :1248 says 0.005, R20/R31) */
    float rho;              /* of phi-bar (Eq. 6)                          */
    uint64_t seed;          /* split positions: splitmix64 + Box-Muller on (seed, particle, child) */
} ges_density_settings;

/* Bytes of device workspace for ges_densify_prune on P particles. */
size_t ges_densify_workspace_bytes(int64_t P);

/* Prune / clone / split (R31-R33) into *_out planar [C][capacity_out] buffers,
 * capacity_out >= 2 P (the largest possible set); the new count goes to the
 * device int64 *P_out.  New order: kept particles in index order (a split parent
 * replaced by its first child), then clones, then second split children; kept
 * particles keep their Adam moments, new ones start at zero. */
ges_status ges_densify_prune(const float *params, const float *m, const float *v, const float *accum,
                             const float *count, int64_t P, int32_t sh_degree, const ges_density_settings *settings,
                             float *params_out, float *m_out, float *v_out, int64_t capacity_out, void *workspace,
                             size_t workspace_bytes, int64_t *P_out, void *stream);

/* Eq. 9 on (image, gt): dL_dimage [3][H][W] (overwritten) and loss_out[4] =
 * (L, L1, SSIM, L_omega) on the device.  mask_lo = NULL drops the L_omega
 * term (its weight still enters l_L1).  Errors as ges_loss_mask. */
ges_status ges_loss(const float *image, const float *gt, const uint8_t *mask_lo, int32_t width, int32_t height,
                    const ges_loss_settings *settings, void *workspace, size_t workspace_bytes, float *dL_dimage,
                    float *loss_out, void *stream);


/* ======================================================================
 * NEXT-4: the 1-D mixture simulation of the Appendix
 * (PAPER.md :606-745) and the Theorem-1 error integrals (:555-603).
 * ====================================================================== */
#define GES_MIX_MAX_N 128      /* components per run                       */
#define GES_MIX_MAX_SAMPLES 49152 /* grid samples (residuals in shared memory) */
typedef enum { GES_MIX_GMM = 0, GES_MIX_DOG = 1, GES_MIX_LOG = 2, GES_MIX_GEF = 3 } ges_mix_model;
typedef enum {
    GES_SIG_SQUARE = 0, GES_SIG_TRIANGLE = 1, GES_SIG_PARABOLIC = 2,
    GES_SIG_HALF_SINUSOID = 3, GES_SIG_EXPONENTIAL = 4, GES_SIG_GAUSSIAN = 5
} ges_signal;

/* One independent fit (device array element, 16 bytes). */
typedef struct {
    int32_t model;      /* ges_mix_model                                              */
    int32_t positive;   /* 1: w = exp(omega) (positive weights, R35); 0: w = omega    */
    int32_t n_comp;     /* N in [1, GES_MIX_MAX_N]; params need stride >= 3 N + 1     */
    int32_t target;     /* row of the target table                                   */
} ges_mix_run;

/* The sample grid x_j = x_lo + j (x_hi - x_lo) / (n - 1), 2 <= n <= GES_MIX_MAX_SAMPLES. */
typedef struct { float x_lo, x_hi; int32_t n; } ges_mix_grid;

typedef struct { float lr, beta1, beta2, eps; } ges_mix_adam;   /* torch.optim.Adam semantics */

/* y[j] = signal(x_j) of width `width` (:662-745; zero outside (-width/2, width/2)
 * except the Gaussian).  y: device [n]. */
ges_status ges_mix_signal(int32_t kind, float width, const ges_mix_grid *grid, float *y, void *stream);

/* Per run r: loss[r] = mean_j (h(x_j) - y_j)^2 of the mixture at params[r]
 * (device [R][stride]: mu[N], s[N], omega[N], beta) against targets[run.target]
 * (device [T][n]); grad (device [R][stride], may be NULL) = d loss / d params.
 * A run with an invalid descriptor gets loss NaN. */
ges_status ges_mix_eval(const ges_mix_run *runs, int32_t n_runs, const float *params, int32_t stride,
                        const ges_mix_grid *grid, const float *targets, float *loss, float *grad, void *stream);

/* `steps` Adam steps per run, in place on params and the moments m, v (device
 * [R][stride], zero before a run's first step); step t uses bias corrections of
 * t0 + 1 .. t0 + steps.  loss[r] = the MSE at the final parameters.  The beta
 * slot changes only for GEF runs (its gradient is 0 otherwise).  One CTA per run:
 * order heavy runs (large N) first. */
ges_status ges_mix_fit(const ges_mix_run *runs, int32_t n_runs, float *params, float *m, float *v, int32_t stride,
                       const ges_mix_grid *grid, const float *targets, const ges_mix_adam *adam, int32_t steps,
                       int32_t t0, float *loss, void *stream);

/* Theorem 1: E[a][b] = int |S(t) - A e^{-(|t|/alpha_a)^beta_b}| dt for the square
 * wave S of amplitude A and width L, by composite Simpson with `intervals` (even,
 * >= 2) panels on the substituted inner integral (see mix1d.cu); beta = 2 is the
 * Gaussian's E_G.  alpha [na], beta [nb], E [na][nb]: device.  Non-positive
 * alpha or beta give NaN. */
ges_status ges_theorem1_errors(const float *alpha, int32_t na, const float *beta, int32_t nb, float A, float L,
                               int32_t intervals, float *E, void *stream);

/* View data parallelism, SH-factorised exchange: the SH gradient of a
 * view is Y_k(u) dL/drgb per particle (u the unit direction from the view's camera
 * centre to the mean), so ranks can exchange the 3-float dL/drgb of their views
 * (ges_grads.drgb) instead of reducing the 3K SH planes.  g_sh [3K][P] (=, or += with
 * accumulate) <- sum over the n views of Y_k(u_v) drgb[v][ch] (drgb: device [n][3][P];
 * cams: device [n][12] = R (world -> camera, row-major 3x3) then t, as ges_camera;
 * mean: device [3][P]). */
ges_status ges_sh_grad_from_colour(const float *mean, int64_t P, int32_t sh_degree, const float *cams,
                                   int32_t n_views, const float *drgb, float *g_sh, int32_t accumulate, void *stream);

/* Failure detection (debug): *count (device uint64, accumulated --
 * zero it first) += the number of NaN / Inf values among x[0, n) (device fp32: an
 * image, a gradient buffer, the parameters).  No synchronisation. */
ges_status ges_count_nonfinite(const float *x, int64_t n, uint64_t *count, void *stream);

/* ---- view data parallelism: visible-union compaction of the gradient allreduce
 * (SURVEY.md §8(e)).  A particle no view of any rank saw has a zero gradient on
 * every rank, so only the union of the ranks' visible sets is reduced:
 *   ges_mask_visible per view (mask |= visible), a MAX allreduce of the P-byte
 *   mask, ges_grad_index, then (when U is small enough) ges_grad_pack, an
 *   allreduce of the C * U packed floats and ges_grad_unpack. */

/* mask[i] = 1 for every particle the frame's last ges_preprocess marked visible
 * (other entries untouched).  mask: device uint8 [P]. */
ges_status ges_mask_visible(const ges_frame *frame, uint8_t *mask, void *stream);

/* Bytes of device workspace for ges_grad_index on P particles. */
size_t ges_grad_pack_workspace_bytes(int64_t P);

/* idx (device int32 [P]) <- the i with mask[i] != 0 in ascending order, *U (device
 * int64) <- their count.  No synchronisation; read *U on the host to decide and to
 * size the allreduce (compaction pays when U is well below P). */
ges_status ges_grad_index(int64_t P, const uint8_t *mask, void *workspace, size_t workspace_bytes, int32_t *idx,
                          int64_t *U, void *stream);

/* packed (device float, >= C U) <- planar [C][U], packed[c U + k] = grads[c P + idx[k]]
 * for k < *U.  grads: the planar [C][P] buffer. */
ges_status ges_grad_pack(const float *grads, int64_t P, int32_t C, const int32_t *idx, const int64_t *U,
                         float *packed, void *stream);

/* grads[c P + idx[k]] = packed[c U + k] for k < *U (the reduced rows back into
 * the planar buffer; the other entries are left as they are -- zero). */
ges_status ges_grad_unpack(const float *packed, int64_t P, int32_t C, const int32_t *idx, const int64_t *U,
                           float *grads, void *stream);

/* Diagnostic: `blocks` x 256 threads each run 8 independent chains of `iters`
 * MUFU ex2 (8 iters blocks 256 results in total); out: device [blocks * 256].
 * The caller times it: the measured special-function rate is the roofline
 * denominator of the ex2-bound kernels (mix1d). */
ges_status ges_probe_mufu(float *out, int32_t iters, int32_t blocks, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GES_H_ */
