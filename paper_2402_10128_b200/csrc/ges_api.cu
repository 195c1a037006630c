// ges_api.cu -- the C ABI (include/ges.h): workspace layout, argument checks
// and the launch sequence of each stage.  Host code only; every kernel lives
// in preprocess.cu / sort.cu / render.cu / particle_bwd.cu.
#include <algorithm>
#include <cmath>
#include <cstring>

#include <nvtx3/nvToolsExt.h>  // header-only: the ranges cost nothing without a tool attached

#include "ges_internal.h"
#include "ges_scan.cuh"

namespace ges {

int num_sms() {
    static int sms[kMaxDevices] = {0};
    const int d = current_device();
    if (sms[d] == 0) {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        sms[d] = n > 0 ? n : 148;
    }
    return sms[d];
}

namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }


int tiles_of(int px) { return (px + kTile - 1) / kTile; }

int bits_for(int64_t n) {
    int b = 0;
    while (((int64_t)1 << b) < n) ++b;
    return b;
}

// Carves the frame; returns the total size.  base == nullptr => size only.
size_t layout(char* base, int64_t P, int32_t W, int32_t H, int64_t cap, ges_frame* f, int64_t* extents = nullptr,
              int32_t max_extents = 0, int32_t* n_extents = nullptr) {
    const int tx = tiles_of(W), ty = tiles_of(H);
    const int64_t T = (int64_t)tx * ty;
    const int64_t HW = (int64_t)W * H;
    size_t off = 0;
    int32_t ne = 0;
    auto take = [&](size_t bytes) -> char* {
        char* p = base ? base + off : nullptr;
        if (extents && ne < max_extents) { extents[2 * ne] = (int64_t)off; extents[2 * ne + 1] = (int64_t)bytes; }
        ++ne;
        off = align_up(off + bytes);
        return p;
    };
    ges_frame g;
    std::memset(&g, 0, sizeof(g));
    g.P = P; g.pair_capacity = cap; g.width = W; g.height = H; g.tiles_x = tx; g.tiles_y = ty;
    g.num_tiles = (int32_t)T; g.tile_bits = std::max(1, bits_for(T)); g.sh_degree_max = 3;
    g.band_begin = 0; g.band_step = 1; g.band_rows = ty;
    // --- zero-per-frame region (one memset in ges_preprocess) ---
    g.row_chunks = (P + kRowChunk - 1) / kRowChunk;
    g.col_chunks = (cap + kColChunk - 1) / kColChunk + ty;
    g.counters = (uint64_t*)take(sizeof(uint64_t) * GES_CTR_N);
    g.row_count = (uint32_t*)take(sizeof(uint32_t) * ty);
    g.tile_count = (uint32_t*)take(sizeof(uint32_t) * (size_t)T);
    g.row_pairs = (uint32_t*)take(sizeof(uint32_t) * ty);
    g.tile_bucket = (uint32_t*)take(sizeof(uint32_t) * kTileBuckets);
    g.lb_rows = (uint32_t*)take(sizeof(uint32_t) * 2 * (size_t)g.row_chunks * ty);
    g.lb_cols = (uint32_t*)take(sizeof(uint32_t) * 2 * (size_t)g.col_chunks * tx);
    g.zero_bytes = off;  // bytes of the zero region from the workspace base
    // --- per particle ---
    g.depth = (float*)take(sizeof(float) * P);
    g.pay0 = (float*)take(16 * (size_t)P);
    g.pay1 = (float*)take(16 * (size_t)P);
    g.pay2 = (float*)take(sizeof(float) * P);
    g.pay3 = (float*)take(sizeof(float) * P);
    g.radius = (int32_t*)take(sizeof(int32_t) * P);
    g.rect = (uint16_t*)take(8 * (size_t)P);
    g.status = (uint8_t*)take((size_t)P);
    g.flags = (uint8_t*)take((size_t)P);
    g.drgb_ddir = (float*)take(sizeof(float) * 9 * (size_t)P);
    for (int k = 0; k < 2; ++k) {
        g.vis_key[k] = (uint32_t*)take(sizeof(uint32_t) * P);
        g.vis_val[k] = (uint32_t*)take(sizeof(uint32_t) * P);
    }
    g.sorted_vis = (uint32_t*)take(sizeof(uint32_t) * P);
    // depth-sort published words: [kDsMaxPasses][kDsMaxGrid][512] u32, then [kDsMaxPasses][kDsMaxGroups][512]
    g.radix_hist = (uint32_t*)take(sizeof(uint32_t) * kRadixDigits * (size_t)kDsMaxGrid * kDsMaxPasses +
                                   sizeof(uint32_t) * kRadixDigits * (size_t)kDsMaxGroups * kDsMaxPasses);
    g.items = (uint32_t*)take(8 * (size_t)P);
    g.rowlist = (uint32_t*)take(8 * (size_t)cap);
    g.col_excl = (uint32_t*)take(sizeof(uint32_t) * (size_t)g.col_chunks * tx);
    g.list = (uint32_t*)take(sizeof(uint32_t) * (size_t)cap);
    g.ranges = (uint32_t*)take(sizeof(uint32_t) * (size_t)(T + 1));
    g.final_T = (float*)take(sizeof(float) * HW);
    g.n_contrib = (uint32_t*)take(sizeof(uint32_t) * HW);
    g.tile_order = (uint32_t*)take(sizeof(uint32_t) * kTileBuckets * (size_t)T);
    g.grad2d = (float*)take(sizeof(float) * kGrad2dStride * (size_t)P);
    g.workspace_bytes = off;
    if (n_extents) *n_extents = ne;
    if (f) *f = g;
    return off;
}

CamParams cam_params(const ges_camera* c) {
    CamParams p;
    p.W = c->width; p.H = c->height;
    p.tiles_x = tiles_of(c->width); p.tiles_y = tiles_of(c->height);
    p.fx = c->fx; p.fy = c->fy; p.cx = c->cx; p.cy = c->cy; p.near_z = c->near_z;
    for (int k = 0; k < 9; ++k) p.R[k] = c->R[k];
    for (int k = 0; k < 3; ++k) p.t[k] = c->t[k];
    return p;
}

bool particles_ok(const ges_particles* p) {
    return p && p->P >= 1 && p->P <= 0x7fffffff && p->sh_degree >= 0 && p->sh_degree <= 3 && p->mean &&
           p->log_scale && p->quat && p->opacity_logit && p->sh && p->beta;
}

// Band of a settings struct: (begin, step), validated; rows = #{r < tiles_y : r = begin + k step}.
bool band_of(const ges_settings* s, int tiles_y, int* begin, int* step, int* rows) {
    int b = s->tile_row_begin, n = s->tile_row_step;
    if (n == 0 && b == 0) n = 1;
    if (n < 1 || b < 0 || b >= n) return false;
    *begin = b; *step = n; *rows = b < tiles_y ? (tiles_y - b + n - 1) / n : 0;
    return true;
}

bool band_matches(const ges_settings* s, const ges_frame* f) {
    int b, n, r;
    return band_of(s, f->tiles_y, &b, &n, &r) && b == f->band_begin && n == f->band_step && s->kernel == f->kernel;
}

bool camera_ok(const ges_camera* c, const ges_frame* f) {
    return c && c->width == f->width && c->height == f->height && c->near_z > 0.0f && c->fx > 0.0f && c->fy > 0.0f;
}

ges_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GES_OK : GES_ERR_CUDA; }

// NVTX range around each entry point (nsys / ncu --nvtx timelines by stage).
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

}  // namespace
}  // namespace ges

using namespace ges;

extern "C" {

size_t ges_workspace_bytes(int64_t P, int32_t width, int32_t height, int64_t pair_capacity) {
    if (P < 1 || width < 1 || height < 1 || pair_capacity < 1) return 0;
    return layout(nullptr, P, width, height, pair_capacity, nullptr);
}

ges_status ges_frame_layout(const ges_frame* frame, int64_t* extents, int32_t capacity, int32_t* count) {
    if (!frame || !count || (capacity > 0 && !extents) || capacity < 0) return GES_ERR_INVALID_ARG;
    layout(nullptr, frame->P, frame->width, frame->height, frame->pair_capacity, nullptr, extents, capacity, count);
    return *count > capacity ? GES_ERR_CAPACITY : GES_OK;
}

ges_status ges_frame_init(void* workspace, size_t bytes, int64_t P, int32_t width, int32_t height,
                          int64_t pair_capacity, ges_frame* frame) {
    if (!workspace || !frame || P < 1 || P > 0x7fffffff || width < 1 || height < 1 || pair_capacity < 1 ||
        pair_capacity >= (int64_t)kValueMask)
        return GES_ERR_INVALID_ARG;
    if (((uintptr_t)workspace) % kAlign) return GES_ERR_INVALID_ARG;
    const int tx = tiles_of(width), ty = tiles_of(height);
    if (tx > 256 || ty > 256) return GES_ERR_INVALID_ARG;
    if (bytes < layout(nullptr, P, width, height, pair_capacity, nullptr)) return GES_ERR_CAPACITY;
    layout((char*)workspace, P, width, height, pair_capacity, frame);
    return GES_OK;
}

ges_status ges_preprocess(const ges_particles* particles, const ges_camera* camera, const ges_settings* settings,
                          ges_frame* frame, void* stream) {
    Nvtx nvtx_("ges_preprocess");
    if (!frame || !settings || !particles_ok(particles) || !camera_ok(camera, frame) || particles->P != frame->P ||
        !(settings->rho >= 0.0f) || (settings->phi_mode != GES_PHI_SCALE && settings->phi_mode != GES_PHI_VARIANCE) ||
        (settings->kernel != GES_KERNEL_PHI_GAUSS && settings->kernel != GES_KERNEL_EXACT_BETA))
        return GES_ERR_INVALID_ARG;
    int band_begin, band_step, band_rows;
    if (!band_of(settings, frame->tiles_y, &band_begin, &band_step, &band_rows)) return GES_ERR_INVALID_ARG;
    frame->band_begin = band_begin; frame->band_step = band_step; frame->band_rows = band_rows;
    frame->kernel = settings->kernel;
    std::memcpy(&frame->depth_key_base, &camera->near_z, sizeof(uint32_t));
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(frame->counters, 0, frame->zero_bytes, s);
    if (e != cudaSuccess) return GES_ERR_CUDA;
    PreprocessArgs a;
    a.mean = particles->mean; a.log_scale = particles->log_scale; a.quat = particles->quat;
    a.opacity_logit = particles->opacity_logit; a.sh = particles->sh; a.beta = particles->beta;
    a.P = (int)particles->P; a.sh_degree = particles->sh_degree;
    a.rho = settings->rho; a.phi_mode = settings->phi_mode; a.gaussian_only = settings->gaussian_only ? 1 : 0;
    a.kernel = settings->kernel;
    a.cam = cam_params(camera);
    a.depth = frame->depth; a.pay0 = (float4*)frame->pay0; a.pay1 = (float4*)frame->pay1; a.pay2 = frame->pay2;
    a.pay3 = frame->pay3;
    a.radius = frame->radius; a.rect = (ushort4*)frame->rect; a.status = frame->status; a.flags = frame->flags;
    a.drgb_ddir = frame->drgb_ddir;
    a.vis_key = frame->vis_key[0];
    a.band_begin = band_begin; a.band_step = band_step;
    a.counters = (unsigned long long*)frame->counters;
    return cuda_status(launch_preprocess(a, s));
}

ges_status ges_sort(ges_frame* frame, void* stream) {
    Nvtx nvtx_("ges_sort");
    if (!frame) return GES_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* ctr = (unsigned long long*)frame->counters;
    cudaError_t e;
    // depth sort (<= 4 passes; pass 0 compacts the visible set; the last one writes the
    // item records): one cooperative kernel.  Keys: vis_key[0] -> [1] -> [0] -> [1] ->
    // (values only) sorted_vis
    DepthSortArgs ds;
    ds.key0 = frame->vis_key[0];
    ds.keys[0] = frame->vis_key[1]; ds.keys[1] = frame->vis_key[0];
    ds.vals[0] = frame->vis_val[1]; ds.vals[1] = frame->vis_val[0];
    ds.sorted_vis = frame->sorted_vis;
    ds.st_cnt = frame->radix_hist;
    ds.gt_cnt = frame->radix_hist + (size_t)kRadixDigits * kDsMaxGrid * kDsMaxPasses;
    ds.P = frame->P; ds.G = 0; ds.key_base = frame->depth_key_base;
    ds.rect = (const ushort4*)frame->rect;
    ds.items = (uint2*)frame->items;
    ds.row_count = frame->row_count;
    ds.rows = frame->band_rows;
    ds.counters = ctr;
    if ((e = launch_depth_sort(ds, s)) != cudaSuccess) return GES_ERR_CUDA;
    // rows, then columns: every (tile, particle) pair written once, in depth order
    BinArgs b;
    b.items = (const uint2*)frame->items; b.row_count = frame->row_count;
    b.rowlist = (uint2*)frame->rowlist;
    b.lb_rows = frame->lb_rows; b.lb_cols = frame->lb_cols; b.col_excl = frame->col_excl;
    b.tile_count = frame->tile_count; b.row_pairs = frame->row_pairs;
    b.ranges = frame->ranges; b.list = frame->list;
    b.counters = ctr;
    b.tiles_x = frame->tiles_x; b.rows = frame->band_rows;
    b.capacity = frame->pair_capacity;
    b.row_chunks = frame->row_chunks; b.col_chunks = frame->col_chunks;
    if ((e = launch_bin(b, s)) != cudaSuccess) return GES_ERR_CUDA;
    return GES_OK;
}

ges_status ges_render_fwd(ges_frame* frame, const ges_settings* settings, float* image, uint32_t* n_eval,
                          uint32_t* n_comp, void* stream) {
    Nvtx nvtx_("ges_render_fwd");
    if (!frame || !settings || !image || !band_matches(settings, frame)) return GES_ERR_INVALID_ARG;
    RenderFwdArgs a;
    a.pay0 = (const float4*)frame->pay0; a.pay1 = (const float4*)frame->pay1; a.pay2 = frame->pay2;
    a.pay3 = frame->pay3; a.exact = frame->kernel == GES_KERNEL_EXACT_BETA;
    a.list = frame->list; a.ranges = frame->ranges; a.counters = (const unsigned long long*)frame->counters;
    a.W = frame->width; a.H = frame->height; a.tiles_x = frame->tiles_x; a.tiles_y = frame->band_rows;
    a.band_begin = frame->band_begin; a.band_step = frame->band_step;
    for (int k = 0; k < 3; ++k) a.bg[k] = settings->background[k];
    a.image = image; a.final_T = frame->final_T; a.n_contrib = frame->n_contrib; a.n_eval = n_eval;
    a.n_comp = n_comp;
    a.tile_bucket = frame->tile_bucket; a.tile_order = frame->tile_order;
    return cuda_status(launch_render_fwd(a, (cudaStream_t)stream));
}

ges_status ges_render_bwd_tiles(const ges_settings* settings, ges_frame* frame, const float* dL_dimage,
                                void* stream) {
    Nvtx nvtx_("ges_render_bwd_tiles");
    if (!frame || !settings || !dL_dimage || !band_matches(settings, frame)) return GES_ERR_INVALID_ARG;
    RenderBwdArgs b;
    b.pay0 = (const float4*)frame->pay0; b.pay1 = (const float4*)frame->pay1; b.pay2 = frame->pay2;
    b.pay3 = frame->pay3; b.exact = frame->kernel == GES_KERNEL_EXACT_BETA;
    b.list = frame->list; b.ranges = frame->ranges; b.counters = (const unsigned long long*)frame->counters;
    b.W = frame->width; b.H = frame->height; b.tiles_x = frame->tiles_x; b.tiles_y = frame->band_rows;
    b.band_begin = frame->band_begin; b.band_step = frame->band_step;
    for (int k = 0; k < 3; ++k) b.bg[k] = settings->background[k];
    b.final_T = frame->final_T; b.n_contrib = frame->n_contrib; b.dL_dimage = dL_dimage; b.grad2d = frame->grad2d;
    b.P = (int)frame->P;
    b.tile_bucket = frame->tile_bucket; b.tile_order = frame->tile_order;
    return cuda_status(launch_render_bwd(b, (cudaStream_t)stream));
}

ges_status ges_backward_particles(const ges_particles* particles, const ges_camera* camera,
                                  const ges_settings* settings, ges_frame* frame, const ges_grads* grads,
                                  void* stream) {
    Nvtx nvtx_("ges_backward_particles");
    if (!frame || !settings || !grads || !particles_ok(particles) || !camera_ok(camera, frame) ||
        particles->P != frame->P || !grads->mean || !grads->log_scale || !grads->quat || !grads->opacity_logit ||
        !grads->sh || !grads->beta)
        return GES_ERR_INVALID_ARG;
    ParticleBwdArgs q;
    q.mean = particles->mean; q.log_scale = particles->log_scale; q.quat = particles->quat;
    q.opacity_logit = particles->opacity_logit; q.sh = particles->sh; q.beta = particles->beta;
    q.P = (int)particles->P; q.sh_degree = particles->sh_degree;
    q.rho = settings->rho; q.phi_mode = settings->phi_mode; q.gaussian_only = settings->gaussian_only ? 1 : 0;
    q.kernel = frame->kernel;
    q.cam = cam_params(camera);
    q.status = frame->status; q.flags = frame->flags; q.grad2d = frame->grad2d; q.drgb_ddir = frame->drgb_ddir;
    q.g_mean = grads->mean; q.g_log_scale = grads->log_scale; q.g_quat = grads->quat;
    q.g_opacity_logit = grads->opacity_logit; q.g_sh = grads->sh; q.g_beta = grads->beta;
    q.g_mean2d = grads->mean2d;
    q.g_drgb = grads->drgb;
    q.accumulate = grads->accumulate;
    return cuda_status(launch_particle_bwd(q, (cudaStream_t)stream));
}

ges_status ges_render_bwd(const ges_particles* particles, const ges_camera* camera, const ges_settings* settings,
                          ges_frame* frame, const float* dL_dimage, const ges_grads* grads, void* stream) {
    if (!frame || !settings || !dL_dimage || !grads || !particles_ok(particles) || !camera_ok(camera, frame) ||
        particles->P != frame->P || !grads->mean || !grads->log_scale || !grads->quat || !grads->opacity_logit ||
        !grads->sh || !grads->beta)
        return GES_ERR_INVALID_ARG;
    const ges_status st = ges_render_bwd_tiles(settings, frame, dL_dimage, stream);
    if (st != GES_OK) return st;
    return ges_backward_particles(particles, camera, settings, frame, grads, stream);
}

ges_status ges_counts_get(const ges_frame* frame, ges_counts* host_out, void* stream) {
    if (!frame || !host_out) return GES_ERR_INVALID_ARG;
    uint64_t c[GES_CTR_N];
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemcpyAsync(c, frame->counters, sizeof(c), cudaMemcpyDeviceToHost, s) != cudaSuccess) return GES_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return GES_ERR_CUDA;
    host_out->visible = (int64_t)c[GES_CTR_VISIBLE];
    host_out->pairs = (int64_t)c[GES_CTR_PAIRS];
    host_out->slots = (int64_t)c[GES_CTR_SLOTS];
    host_out->capacity = frame->pair_capacity;
    host_out->culled_near = (int64_t)c[GES_CTR_CULLED_NEAR];
    host_out->degenerate = (int64_t)c[GES_CTR_DEGENERATE];
    host_out->offscreen = (int64_t)c[GES_CTR_OFFSCREEN];
    host_out->overflow = (int32_t)c[GES_CTR_OVERFLOW];
    host_out->_pad = 0;
    return GES_OK;
}

const char* ges_status_string(ges_status st) {
    switch (st) {
        case GES_OK: return "ok";
        case GES_ERR_INVALID_ARG: return "invalid argument";
        case GES_ERR_CAPACITY: return "workspace or pair capacity too small";
        case GES_ERR_CUDA: return "CUDA error";
        case GES_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown";
}

const char* ges_version(void) { return "ges-b200 0.1 (sm_100a)"; }

// ---------------------------------------------------------------------------
// loss front end
// ---------------------------------------------------------------------------
namespace {
int down_dim(int n, float s) { return std::max(1, (int)std::floor((double)n * (double)s + 0.5)); }

struct LossLayout {
    size_t d_mu, d_e2, d_exy, partial, lo, h1, h2, dog, minmax, total;
};
LossLayout loss_layout(int W, int H, float s) {
    LossLayout L;
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off = align_up(off + bytes); return o; };
    const size_t n3 = (size_t)3 * W * H, nd = (size_t)down_dim(W, s) * down_dim(H, s);
    L.d_mu = take(4 * n3); L.d_e2 = take(4 * n3); L.d_exy = take(4 * n3);
    L.partial = take(4 * 3 * (size_t)loss_partials(W, H));
    L.lo = take(4 * nd); L.h1 = take(4 * nd); L.h2 = take(4 * nd); L.dog = take(4 * nd);
    L.minmax = take(8);
    L.total = off;
    return L;
}
bool loss_settings_ok(const ges_loss_settings* s) {
    return s && s->lambda_ssim >= 0.0f && s->lambda_omega >= 0.0f && s->lambda_ssim + s->lambda_omega <= 1.0f &&
           s->eps_omega >= 0.0f && s->eps_omega <= 1.0f && s->downsample > 0.0f && s->downsample <= 1.0f;
}
}  // namespace

ges_status ges_loss_mask_dims(int32_t width, int32_t height, float downsample, int32_t* Wd, int32_t* Hd) {
    if (width < 1 || height < 1 || !(downsample > 0.0f && downsample <= 1.0f) || !Wd || !Hd)
        return GES_ERR_INVALID_ARG;
    *Wd = down_dim(width, downsample);
    *Hd = down_dim(height, downsample);
    return GES_OK;
}

size_t ges_loss_workspace_bytes(int32_t width, int32_t height, float downsample) {
    if (width < 1 || height < 1 || !(downsample > 0.0f && downsample <= 1.0f)) return 0;
    return loss_layout(width, height, downsample).total;
}

ges_status ges_loss_mask(const float* gt, int32_t width, int32_t height, float omega, const ges_loss_settings* settings,
                         void* workspace, size_t workspace_bytes, uint8_t* mask_lo, void* stream) {
    Nvtx nvtx_("ges_loss_mask");
    if (!gt || !mask_lo || !workspace || width < 1 || height < 1 || !loss_settings_ok(settings) ||
        !(omega >= 0.0f && omega <= 1.0f))
        return GES_ERR_INVALID_ARG;
    const LossLayout L = loss_layout(width, height, settings->downsample);
    if (workspace_bytes < L.total) return GES_ERR_CAPACITY;
    char* ws = (char*)workspace;
    MaskArgs m;
    m.gt = gt; m.W = width; m.H = height;
    m.Wd = down_dim(width, settings->downsample); m.Hd = down_dim(height, settings->downsample);
    const double w = (double)omega, s1 = 0.2 + 20.0 * w, s2 = 0.1 + 10.0 * w;  // Eq. 7 sigmas
    m.r1 = (int)std::ceil(3.0 * s1); m.r2 = (int)std::ceil(3.0 * s2);
    m.ih1 = (float)(1.0 / (2.0 * s1 * s1)); m.ih2 = (float)(1.0 / (2.0 * s2 * s2));
    m.eps = settings->eps_omega;
    m.complement = omega <= 0.5f;
    m.lo = (float*)(ws + L.lo); m.h1 = (float*)(ws + L.h1); m.h2 = (float*)(ws + L.h2); m.dog = (float*)(ws + L.dog);
    m.minmax = (unsigned*)(ws + L.minmax);
    m.mask_lo = mask_lo;
    return cuda_status(launch_mask(m, (cudaStream_t)stream));
}

ges_status ges_loss(const float* image, const float* gt, const uint8_t* mask_lo, int32_t width, int32_t height,
                    const ges_loss_settings* settings, void* workspace, size_t workspace_bytes, float* dL_dimage,
                    float* loss_out, void* stream) {
    Nvtx nvtx_("ges_loss");
    if (!image || !gt || !workspace || !dL_dimage || !loss_out || width < 1 || height < 1 ||
        !loss_settings_ok(settings))
        return GES_ERR_INVALID_ARG;
    const LossLayout L = loss_layout(width, height, settings->downsample);
    if (workspace_bytes < L.total) return GES_ERR_CAPACITY;
    char* ws = (char*)workspace;
    LossArgs a;
    a.image = image; a.gt = gt; a.mask_lo = mask_lo;
    a.W = width; a.H = height;
    a.Wd = down_dim(width, settings->downsample); a.Hd = down_dim(height, settings->downsample);
    a.lambda_ssim = settings->lambda_ssim; a.lambda_omega = settings->lambda_omega;
    a.inv_n = (float)(1.0 / (3.0 * width * (double)height));
    a.d_mu = (float*)(ws + L.d_mu); a.d_e2 = (float*)(ws + L.d_e2); a.d_exy = (float*)(ws + L.d_exy);
    a.partial = (float*)(ws + L.partial);
    a.nblocks = 0;
    a.dL_dimage = dL_dimage; a.loss_out = loss_out;
    return cuda_status(launch_loss(a, (cudaStream_t)stream));
}


// ---------------------------------------------------------------------------
// optimizer and density control
// ---------------------------------------------------------------------------
double ges_lr_position(int64_t step, double init, double final_, double delay_mult, int64_t max_steps,
                       int64_t delay_steps) {
    if (step < 0 || (init == 0.0 && final_ == 0.0) || max_steps <= 0) return 0.0;
    double delay = 1.0;
    if (delay_steps > 0) {
        const double t = std::min(std::max((double)step / (double)delay_steps, 0.0), 1.0);
        delay = delay_mult + (1.0 - delay_mult) * std::sin(0.5 * 3.14159265358979323846 * t);
    }
    const double t = std::min(std::max((double)step / (double)max_steps, 0.0), 1.0);
    return delay * std::exp(std::log(init) * (1.0 - t) + std::log(final_) * t);
}

ges_status ges_adam_step(float* params, const float* grads, float* m, float* v, int64_t P, int32_t sh_degree,
                         const ges_adam_settings* s, void* stream) {
    Nvtx nvtx_("ges_adam_step");
    if (!params || !grads || !m || !v || !s || P < 1 || sh_degree < 0 || sh_degree > 3 || s->step < 1)
        return GES_ERR_INVALID_ARG;
    const int K = (sh_degree + 1) * (sh_degree + 1);
    AdamArgs a;
    a.params = params; a.grads = grads; a.m = m; a.v = v; a.P = P; a.n_planes = 12 + 3 * K;
    a.lr_position = s->lr_position; a.lr_scaling = s->lr_scaling; a.lr_rotation = s->lr_rotation;
    a.lr_opacity = s->lr_opacity; a.lr_feature_dc = s->lr_feature_dc; a.lr_feature_rest = s->lr_feature_rest;
    a.lr_shape = s->lr_shape; a.beta1 = s->beta1; a.beta2 = s->beta2; a.eps = s->eps;
    a.inv_bc1 = (float)(1.0 / (1.0 - std::pow((double)s->beta1, (double)s->step)));
    a.inv_bc2 = (float)(1.0 / (1.0 - std::pow((double)s->beta2, (double)s->step)));
    return cuda_status(launch_adam(a, (cudaStream_t)stream));
}

ges_status ges_adam_step_range(float* params, const float* grads_range, float* m, float* v, int64_t P,
                               int32_t sh_degree, const ges_adam_settings* s, int64_t begin, int64_t count,
                               void* stream) {
    Nvtx nvtx_("ges_adam_step_range");
    const int K = (sh_degree + 1) * (sh_degree + 1);
    if (!params || !grads_range || !m || !v || !s || P < 1 || sh_degree < 0 || sh_degree > 3 || s->step < 1 ||
        begin < 0 || count < 0 || begin + count > (int64_t)(12 + 3 * K) * P)
        return GES_ERR_INVALID_ARG;
    AdamArgs a;
    a.params = params; a.grads = grads_range; a.m = m; a.v = v; a.P = P; a.n_planes = 12 + 3 * K;
    a.lr_position = s->lr_position; a.lr_scaling = s->lr_scaling; a.lr_rotation = s->lr_rotation;
    a.lr_opacity = s->lr_opacity; a.lr_feature_dc = s->lr_feature_dc; a.lr_feature_rest = s->lr_feature_rest;
    a.lr_shape = s->lr_shape; a.beta1 = s->beta1; a.beta2 = s->beta2; a.eps = s->eps;
    a.inv_bc1 = (float)(1.0 / (1.0 - std::pow((double)s->beta1, (double)s->step)));
    a.inv_bc2 = (float)(1.0 / (1.0 - std::pow((double)s->beta2, (double)s->step)));
    return cuda_status(launch_adam_range(a, begin, count, (cudaStream_t)stream));
}

size_t ges_reorder_workspace_bytes(int64_t P) { return P < 1 ? 0 : reorder_workspace_bytes(P); }

ges_status ges_reorder(const float* params, float* params_out, const float* m, float* m_out, const float* v,
                       float* v_out, int64_t P, int32_t sh_degree, uint32_t* perm_out, void* workspace, size_t bytes,
                       void* stream) {
    Nvtx nvtx_("ges_reorder");
    if (!params || !params_out || !perm_out || !workspace || P < 1 || P > 0x7fffffff || sh_degree < 0 ||
        sh_degree > 3 || (!m != !m_out) || (!v != !v_out) || params == params_out || (m && m == m_out) ||
        (v && v == v_out))
        return GES_ERR_INVALID_ARG;
    if (bytes < reorder_workspace_bytes(P)) return GES_ERR_CAPACITY;
    if (((uintptr_t)workspace) % kAlign) return GES_ERR_INVALID_ARG;
    const int K = (sh_degree + 1) * (sh_degree + 1);
    const float* in[3] = {params, m, v};
    float* out[3] = {params_out, m_out, v_out};
    return cuda_status(launch_reorder(in, out, 3, P, 12 + 3 * K, perm_out, workspace, (cudaStream_t)stream));
}

ges_status ges_reset(float* params, int64_t P, int32_t sh_degree, int32_t what, void* stream) {
    if (!params || P < 1 || sh_degree < 0 || sh_degree > 3 || (what != 0 && what != 1)) return GES_ERR_INVALID_ARG;
    const int K = (sh_degree + 1) * (sh_degree + 1);
    if (what == 0)
        return cuda_status(launch_reset(params, P, 10, (float)std::log(0.01 / 0.99), 0, (cudaStream_t)stream));
    return cuda_status(launch_reset(params, P, 11 + 3 * K, 2.0f, 1, (cudaStream_t)stream));
}

ges_status ges_densify_stats(const ges_frame* frame, float* accum, float* count, void* stream) {
    Nvtx nvtx_("ges_densify_stats");
    if (!frame || !accum || !count) return GES_ERR_INVALID_ARG;
    DensifyStatsArgs a;
    a.status = frame->status; a.grad2d = frame->grad2d; a.accum = accum; a.count = count;
    a.pay0 = (const float4*)frame->pay0; a.pay1 = (const float4*)frame->pay1; a.pay3 = frame->pay3;
    a.P = frame->P; a.W = frame->width; a.H = frame->height; a.kernel = frame->kernel;
    return cuda_status(launch_densify_stats(a, (cudaStream_t)stream));
}

size_t ges_densify_workspace_bytes(int64_t P) {
    if (P < 1) return 0;
    return align_up((size_t)P) + align_up(sizeof(int) * 3 * (size_t)densify_blocks(P)) + align_up(3 * sizeof(long long));
}

ges_status ges_densify_prune(const float* params, const float* m, const float* v, const float* accum,
                             const float* count, int64_t P, int32_t sh_degree, const ges_density_settings* s,
                             float* params_out, float* m_out, float* v_out, int64_t capacity_out, void* workspace,
                             size_t workspace_bytes, int64_t* P_out, void* stream) {
    Nvtx nvtx_("ges_densify_prune");
    if (!params || !m || !v || !accum || !count || !s || !params_out || !m_out || !v_out || !workspace || !P_out ||
        P < 1 || sh_degree < 0 || sh_degree > 3 || capacity_out < 2 * P)
        return GES_ERR_INVALID_ARG;
    if (workspace_bytes < ges_densify_workspace_bytes(P)) return GES_ERR_CAPACITY;
    const int K = (sh_degree + 1) * (sh_degree + 1);
    char* ws = (char*)workspace;
    DensifyArgs a;
    a.params = params; a.m = m; a.v = v; a.accum = accum; a.count = count;
    a.P = P; a.cap_out = capacity_out; a.n_planes = 12 + 3 * K;
    a.grad_threshold = s->grad_threshold; a.percent_dense = s->percent_dense; a.extent = s->scene_extent;
    a.opacity_prune = s->opacity_prune; a.shape_prune = s->shape_prune; a.rho = s->rho; a.seed = s->seed;
    a.params_out = params_out; a.m_out = m_out; a.v_out = v_out;
    a.action = (uint8_t*)ws;
    a.block_cnt = (int*)(ws + align_up((size_t)P));
    a.totals = (long long*)(ws + align_up((size_t)P) + align_up(sizeof(int) * 3 * (size_t)densify_blocks(P)));
    a.P_out = (long long*)P_out;
    a.nblocks = 0;
    return cuda_status(launch_densify_prune(a, (cudaStream_t)stream));
}

// ---- NEXT-4: 1-D mixtures and Theorem 1 --------------------------------------
static bool grid_ok(const ges_mix_grid* g) {
    return g && g->n >= 2 && g->n <= GES_MIX_MAX_SAMPLES && std::isfinite(g->x_lo) && std::isfinite(g->x_hi) &&
           g->x_hi > g->x_lo;
}

ges_status ges_mix_signal(int32_t kind, float width, const ges_mix_grid* grid, float* y, void* stream) {
    if (!grid_ok(grid) || !y || kind < 0 || kind > 5 || !(width > 0.0f)) return GES_ERR_INVALID_ARG;
    const float h = (grid->x_hi - grid->x_lo) / (float)(grid->n - 1);
    return cuda_status(launch_mix_signal(kind, width, grid->x_lo, h, grid->n, y, (cudaStream_t)stream));
}

static ges_status mix_common(const ges_mix_run* runs, int32_t n_runs, float* params, int32_t stride,
                             const ges_mix_grid* grid, const float* targets, float* loss, MixArgs& a) {
    if (!runs || n_runs < 1 || !params || stride < 4 || !grid_ok(grid) || !targets || !loss) return GES_ERR_INVALID_ARG;
    a.runs = runs; a.n_runs = n_runs; a.stride = stride; a.params = params; a.m = a.v = nullptr; a.grad = nullptr;
    a.loss = loss; a.targets = targets; a.x_lo = grid->x_lo; a.n = grid->n;
    a.h = (grid->x_hi - grid->x_lo) / (float)(grid->n - 1);
    a.steps = 0; a.t0 = 0; a.lr = 0.0f; a.b1 = 0.9f; a.b2 = 0.999f; a.eps = 1e-8f;
    return GES_OK;
}

ges_status ges_mix_eval(const ges_mix_run* runs, int32_t n_runs, const float* params, int32_t stride,
                        const ges_mix_grid* grid, const float* targets, float* loss, float* grad, void* stream) {
    MixArgs a;
    const ges_status st = mix_common(runs, n_runs, const_cast<float*>(params), stride, grid, targets, loss, a);
    if (st != GES_OK) return st;
    a.grad = grad;
    return cuda_status(launch_mix(a, false, (cudaStream_t)stream));
}

ges_status ges_mix_fit(const ges_mix_run* runs, int32_t n_runs, float* params, float* m, float* v, int32_t stride,
                       const ges_mix_grid* grid, const float* targets, const ges_mix_adam* adam, int32_t steps,
                       int32_t t0, float* loss, void* stream) {
    MixArgs a;
    const ges_status st = mix_common(runs, n_runs, params, stride, grid, targets, loss, a);
    if (st != GES_OK) return st;
    if (!m || !v || !adam || steps < 0 || t0 < 0 || !(adam->lr >= 0.0f) || !(adam->beta1 >= 0.0f && adam->beta1 < 1.0f) ||
        !(adam->beta2 >= 0.0f && adam->beta2 < 1.0f) || !(adam->eps >= 0.0f))
        return GES_ERR_INVALID_ARG;
    a.m = m; a.v = v; a.steps = steps; a.t0 = t0;
    a.lr = adam->lr; a.b1 = adam->beta1; a.b2 = adam->beta2; a.eps = adam->eps;
    return cuda_status(launch_mix(a, true, (cudaStream_t)stream));
}

ges_status ges_theorem1_errors(const float* alpha, int32_t na, const float* beta, int32_t nb, float A, float L,
                               int32_t intervals, float* E, void* stream) {
    if (!alpha || !beta || !E || na < 1 || nb < 1 || intervals < 2 || (intervals & 1) || !(L > 0.0f) ||
        !std::isfinite(A) || (int64_t)na * nb > (int64_t)1 << 26)
        return GES_ERR_INVALID_ARG;
    return cuda_status(launch_theorem1(alpha, na, beta, nb, A, L, intervals, E, (cudaStream_t)stream));
}

ges_status ges_probe_mufu(float* out, int32_t iters, int32_t blocks, void* stream) {
    if (!out || iters < 1 || blocks < 1) return GES_ERR_INVALID_ARG;
    return cuda_status(launch_mufu_probe(out, iters, blocks, (cudaStream_t)stream));
}

// ---- view-DP gradient compaction -----------------------------
ges_status ges_sh_grad_from_colour(const float* mean, int64_t P, int32_t sh_degree, const float* cams,
                                   int32_t n_views, const float* drgb, float* g_sh, int32_t accumulate, void* stream) {
    Nvtx nvtx_("ges_sh_grad_from_colour");
    if (!mean || !g_sh || P < 1 || P > 0x7fffffff || sh_degree < 0 || sh_degree > 3 || n_views < 0 ||
        (n_views > 0 && (!cams || !drgb)))
        return GES_ERR_INVALID_ARG;
    return cuda_status(launch_sh_from_colour(mean, P, sh_degree, cams, n_views, drgb, g_sh, accumulate ? 1 : 0,
                                             (cudaStream_t)stream));
}

ges_status ges_count_nonfinite(const float* x, int64_t n, uint64_t* count, void* stream) {
    if (!x || !count || n < 0) return GES_ERR_INVALID_ARG;
    if (n == 0) return GES_OK;
    return cuda_status(launch_count_nonfinite(x, n, (unsigned long long*)count, (cudaStream_t)stream));
}

ges_status ges_mask_visible(const ges_frame* frame, uint8_t* mask, void* stream) {
    Nvtx nvtx_("ges_mask_visible");
    if (!frame || !mask) return GES_ERR_INVALID_ARG;
    return cuda_status(launch_mask_visible(frame->status, frame->P, mask, (cudaStream_t)stream));
}

size_t ges_grad_pack_workspace_bytes(int64_t P) {
    if (P < 1) return 0;
    return align_up(sizeof(int) * (size_t)grad_pack_blocks(P));
}

ges_status ges_grad_index(int64_t P, const uint8_t* mask, void* workspace, size_t workspace_bytes, int32_t* idx,
                          int64_t* U, void* stream) {
    Nvtx nvtx_("ges_grad_index");
    if (P < 1 || P > 0x7fffffff || !mask || !workspace || !idx || !U) return GES_ERR_INVALID_ARG;
    if (workspace_bytes < ges_grad_pack_workspace_bytes(P)) return GES_ERR_CAPACITY;
    return cuda_status(launch_grad_index(P, mask, (int*)workspace, idx, (long long*)U, (cudaStream_t)stream));
}

ges_status ges_grad_pack(const float* grads, int64_t P, int32_t C, const int32_t* idx, const int64_t* U,
                         float* packed, void* stream) {
    Nvtx nvtx_("ges_grad_pack");
    if (!grads || P < 1 || P > 0x7fffffff || C < 1 || !idx || !U || !packed) return GES_ERR_INVALID_ARG;
    return cuda_status(launch_grad_pack(grads, P, C, idx, (const long long*)U, packed, (cudaStream_t)stream));
}

ges_status ges_grad_unpack(const float* packed, int64_t P, int32_t C, const int32_t* idx, const int64_t* U,
                           float* grads, void* stream) {
    Nvtx nvtx_("ges_grad_unpack");
    if (!packed || P < 1 || P > 0x7fffffff || C < 1 || !idx || !U || !grads) return GES_ERR_INVALID_ARG;
    return cuda_status(launch_grad_unpack(packed, P, C, idx, (const long long*)U, grads, (cudaStream_t)stream));
}

}  // extern "C"
