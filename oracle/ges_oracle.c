/* oracle/ges_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The parity oracle for the GES tile rasterizer: a plain, slow, CPU
 * implementation of what the hot path computes, written from the paper
 * (arXiv 2402.10128, /root/reference/PAPER.md) and SURVEY.md §8(a)/(c).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, constant
 * table or helper with the CUDA path (paper_2402_10128_b200/csrc).
 *
 * Contents
 *   S1  preprocess_f32 / preprocess_f64      (ges_geom.inc; KEYSPEC fp32 / fp64)
 *       exp_spec                              (KEYSPEC exp)
 *   S2  or_pairs_sorted: brute-force (tile, depth) keys + qsort
 *       or_tile_lists:   per-tile membership (tile in rect_i and the tile
 *                        reaches alpha >= 0.98/255, tile_member), sorted by
 *                        (depth bits, index)                          (R8, R11)
 *   S4  or_render_fwd:   per pixel, front-to-back alpha compositing of its
 *                        tile's list in fp64 (Eq. 3; R7, R12)
 *   S5a or_render_bwd:   per pixel hand-derived adjoint of Eq. 3 in fp64
 *   S5b or_backward_particles: chain 2D -> 3D parameters in fp64, incl. beta
 *                        through phi-bar (Eq. 6)
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC
 *        (contraction OFF: KEYSPEC fixes every rounding).
 * Threads: OpenMP over tiles; every reduction is done serially in a fixed
 * order, so results do not depend on the thread count.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum { OR_VISIBLE = 0, OR_CULL_NEAR = 1, OR_DEGENERATE = 2, OR_OFFSCREEN = 3 };
enum { OR_PHI_SCALE = 0, OR_PHI_VARIANCE = 1 };

typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy, near_z;
    float R[9]; /* world -> camera rotation, row-major */
    float t[3];
} OrCamera;

typedef struct {
    float rho;
    int32_t phi_mode;
    int32_t gaussian_only;
    float bg[3];
    int32_t kernel; /* 0: phi-bar-scaled Gaussian (R6); 1: exact GEF of Eq. 2 (NEXT-3) */
} OrSettings;

/* ------------------------------------------------------------------ */
/* KEYSPEC exp: Cody-Waite reduction + degree-7 Taylor (fp32).          */
/* ------------------------------------------------------------------ */
static float f32_from_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }

float or_exp_spec(float x) {
    x = fminf(88.0f, fmaxf(-87.0f, x));
    const float log2e = f32_from_bits(0x3fb8aa3bu);
    const float ln2_hi = f32_from_bits(0x3f317200u);
    const float ln2_lo = f32_from_bits(0x35bfbe8eu);
    float k = rintf(x * log2e);
    float r = fmaf(-k, ln2_hi, x);
    r = fmaf(-k, ln2_lo, r);
    /* 1/n! rounded to fp32 */
    const float c7 = (float)(1.0 / 5040.0), c6 = (float)(1.0 / 720.0), c5 = (float)(1.0 / 120.0);
    const float c4 = (float)(1.0 / 24.0), c3 = (float)(1.0 / 6.0), c2 = 0.5f, c1 = 1.0f, c0 = 1.0f;
    float p = c7;
    p = fmaf(p, r, c6);
    p = fmaf(p, r, c5);
    p = fmaf(p, r, c4);
    p = fmaf(p, r, c3);
    p = fmaf(p, r, c2);
    p = fmaf(p, r, c1);
    p = fmaf(p, r, c0);
    int ki = (int)k;
    float two_k = f32_from_bits((uint32_t)(ki + 127) << 23);
    return p * two_k;
}

/* KEYSPEC log for x > 1 (normal): x = m 2^e with m in [sqrt(1/2), sqrt(2));
 * ln m = 2 atanh(s), s = (m-1)/(m+1), odd series to s^9; + e ln2. */
float or_log_spec(float x) {
    uint32_t bits;
    memcpy(&bits, &x, 4);
    int e = (int)(bits >> 23) - 127;
    float m = f32_from_bits((bits & 0x7fffffu) | 0x3f800000u);
    if (m > 1.41421354f) { m = m * 0.5f; e += 1; }
    const float s = (m - 1.0f) / (m + 1.0f);
    const float s2 = s * s;
    float p = (float)(1.0 / 9.0);
    p = fmaf(p, s2, (float)(1.0 / 7.0));
    p = fmaf(p, s2, (float)(1.0 / 5.0));
    p = fmaf(p, s2, (float)(1.0 / 3.0));
    p = fmaf(p, s2, 1.0f);
    float t = s * p;
    t = t + t;
    return fmaf((float)e, (float)0.69314718055994531, t);
}

/* ---------------- fp32 KEYSPEC instantiation ---------------- */
#define REAL float
#define PREAL float
#define SFX(n) n##_f32
#define FMA fmaf
#define EXPF or_exp_spec
#define LOGF or_log_spec
#define SQRTF sqrtf
#define FLOORF floorf
#define CEILF ceilf
#define FMINF fminf
#define FMAXF fmaxf
#include "ges_geom.inc"
#undef REAL
#undef PREAL
#undef SFX
#undef FMA
#undef EXPF
#undef LOGF
#undef SQRTF
#undef FLOORF
#undef CEILF
#undef FMINF
#undef FMAXF

/* ---------------- fp64 instantiation ---------------- */
#define REAL double
#define PREAL double
#define SFX(n) n##_f64
#define FMA fma
#define EXPF exp
#define LOGF log
#define SQRTF sqrt
#define FLOORF floor
#define CEILF ceil
#define FMINF fmin
#define FMAXF fmax
#include "ges_geom.inc"
#undef REAL
#undef PREAL
#undef SFX
#undef FMA
#undef EXPF
#undef LOGF
#undef SQRTF
#undef FLOORF
#undef CEILF
#undef FMINF
#undef FMAXF

void or_preprocess_f32(const OrParticles_f32 *pp, const OrCamera *cam, const OrSettings *st, OrPre_f32 *out) {
    preprocess_f32(pp, cam, st, out);
}
void or_preprocess_f64(const OrParticles_f64 *pp, const OrCamera *cam, const OrSettings *st, OrPre_f64 *out) {
    preprocess_f64(pp, cam, st, out);
}
void or_sh_basis_f64(double x, double y, double z, int K, double *Y) { sh_basis_f64(x, y, z, K, Y); }
void or_sh_basis_f32(float x, float y, float z, int K, float *Y) { sh_basis_f32(x, y, z, K, Y); }

/* ------------------------------------------------------------------ */
/* S2: keys and per-tile lists                                         */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t key; int32_t idx; } OrPair;

static int cmp_pair(const void *a, const void *b) {
    const OrPair *x = (const OrPair *)a, *y = (const OrPair *)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/* Geometry for the tile-membership test (NULL: plain rect membership). */
typedef struct {
    int32_t precision;  /* 0: fp32 KEYSPEC arrays, 1: fp64 */
    int32_t _pad;
    int64_t P;
    const void *uv, *conic, *kappa; /* [2][P], [3][P], [P] */
} OrGeom;

static int or_member(const OrGeom *g, int64_t i, int tx, int ty) {
    if (!g) return 1;
    const int64_t P = g->P;
    if (g->precision == 0) {
        const float *uv = (const float *)g->uv, *cn = (const float *)g->conic, *k = (const float *)g->kappa;
        return tile_member_f32(uv[i], uv[P + i], cn[i], cn[P + i], cn[2 * P + i], k[i], tx, ty);
    }
    const double *uv = (const double *)g->uv, *cn = (const double *)g->conic, *k = (const double *)g->kappa;
    return tile_member_f64(uv[i], uv[P + i], cn[i], cn[P + i], cn[2 * P + i], k[i], tx, ty);
}

int or_tile_member_f32(float u, float v, float a, float b, float c, float kappa, int tx, int ty) {
    return tile_member_f32(u, v, a, b, c, kappa, tx, ty);
}

/* Number of (particle, tile) pairs. */
int64_t or_count_pairs(int64_t P, const int32_t *status, const int32_t *tiles) {
    int64_t M = 0;
    for (int64_t i = 0; i < P; ++i)
        if (status[i] == OR_VISIBLE) M += tiles[i];
    return M;
}

/* Brute force: enumerate every (visible particle, tile in its rect) pair, build
 * key = (tile_id << 32) | depth_bits, sort ascending by (key, particle index).
 * depth_bits[i] = the fp32 bit pattern of the depth (positive => monotone). */
int64_t or_pairs_sorted(int64_t P, const int32_t *status, const int32_t *rect, const uint32_t *depth_bits,
                        const OrGeom *geom, int32_t tiles_x, uint64_t *keys_out, int32_t *vals_out, int64_t cap) {
    int64_t M = 0;
    for (int64_t i = 0; i < P; ++i) {
        if (status[i] != OR_VISIBLE) continue;
        for (int ty = rect[P + i]; ty < rect[3 * P + i]; ++ty)
            for (int tx = rect[i]; tx < rect[2 * P + i]; ++tx) M += or_member(geom, i, tx, ty);
    }
    if (M > cap) return -M;
    OrPair *pr = (OrPair *)malloc(sizeof(OrPair) * (size_t)(M > 0 ? M : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < P; ++i) {
        if (status[i] != OR_VISIBLE) continue;
        for (int ty = rect[P + i]; ty < rect[3 * P + i]; ++ty)
            for (int tx = rect[i]; tx < rect[2 * P + i]; ++tx) {
                if (!or_member(geom, i, tx, ty)) continue;
                uint64_t tile = (uint64_t)ty * (uint64_t)tiles_x + (uint64_t)tx;
                pr[m].key = (tile << 32) | (uint64_t)depth_bits[i];
                pr[m].idx = (int32_t)i;
                ++m;
            }
    }
    qsort(pr, (size_t)M, sizeof(OrPair), cmp_pair);
    for (int64_t k = 0; k < M; ++k) { keys_out[k] = pr[k].key; vals_out[k] = pr[k].idx; }
    free(pr);
    return M;
}

/* Per-tile membership S(tile) = { i visible : tile in rect_i }, sorted by
 * (order[i], i).  tile_mask (may be NULL) restricts which tiles get lists.
 * offsets has T+1 entries.  If list == NULL only offsets are produced.
 * Returns the total list length. */
int64_t or_tile_lists(int64_t P, const int32_t *status, const int32_t *rect, const uint64_t *order,
                      const OrGeom *geom, int32_t tiles_x, int32_t tiles_y, const uint8_t *tile_mask,
                      int64_t *offsets, int32_t *list, int64_t cap) {
    const int64_t T = (int64_t)tiles_x * tiles_y;
    int64_t *cnt = (int64_t *)calloc((size_t)T + 1, sizeof(int64_t));
    for (int64_t i = 0; i < P; ++i) {
        if (status[i] != OR_VISIBLE) continue;
        for (int ty = rect[P + i]; ty < rect[3 * P + i]; ++ty)
            for (int tx = rect[i]; tx < rect[2 * P + i]; ++tx) {
                int64_t tile = (int64_t)ty * tiles_x + tx;
                if ((!tile_mask || tile_mask[tile]) && or_member(geom, i, tx, ty)) cnt[tile]++;
            }
    }
    offsets[0] = 0;
    for (int64_t t = 0; t < T; ++t) offsets[t + 1] = offsets[t] + cnt[t];
    const int64_t total = offsets[T];
    if (!list) { free(cnt); return total; }
    if (total > cap) { free(cnt); return -total; }
    OrPair *pr = (OrPair *)malloc(sizeof(OrPair) * (size_t)(total > 0 ? total : 1));
    for (int64_t t = 0; t < T; ++t) cnt[t] = offsets[t];
    for (int64_t i = 0; i < P; ++i) {
        if (status[i] != OR_VISIBLE) continue;
        for (int ty = rect[P + i]; ty < rect[3 * P + i]; ++ty)
            for (int tx = rect[i]; tx < rect[2 * P + i]; ++tx) {
                int64_t tile = (int64_t)ty * tiles_x + tx;
                if (tile_mask && !tile_mask[tile]) continue;
                if (!or_member(geom, i, tx, ty)) continue;
                pr[cnt[tile]].key = order[i];
                pr[cnt[tile]].idx = (int32_t)i;
                cnt[tile]++;
            }
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t t = 0; t < T; ++t)
        qsort(pr + offsets[t], (size_t)(offsets[t + 1] - offsets[t]), sizeof(OrPair), cmp_pair);
    for (int64_t k = 0; k < total; ++k) list[k] = pr[k].idx;
    free(pr);
    free(cnt);
    return total;
}

/* ------------------------------------------------------------------ */
/* S4 / S5a: compositing in fp64                                       */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t width, height, tiles_x, tiles_y;
    double bg[3];
} OrScreen;

typedef struct {
    int64_t P;
    const double *uv, *conic, *kappa, *rgb; /* planar [2][P], [3][P], [P], [3][P] */
    const double *hbeta;                    /* [P] beta / 2 of the exact GEF kernel, or NULL (Gaussian) */
} OrSplat2D;

/* Decision thresholds are the fp32 constants of R7 (what the kernel compares
 * against), promoted exactly to fp64. */
#define OR_ALPHA_MIN ((double)(1.0f / 255.0f))
#define OR_ALPHA_MAX ((double)0.99f)
#define OR_T_MIN ((double)1e-4f)

/* Extra relative margin added to the ambiguity bound (tests widen it to mask
 * pixels whose decisions a finite-difference step could flip). */
static double g_amb_margin = 0.0;
void or_set_amb_margin(double m) { g_amb_margin = m; }

typedef struct {
    int32_t k;      /* position in the tile list */
    int32_t idx;    /* particle */
    double alpha, T, G, araw, dx, dy;
    double Q, Qb;   /* exact kernel: Mahalanobis^2 Q and Q^(beta/2) */
    int clamped;    /* araw >= 0.99 -> alpha = 0.99, no gradient to kappa/power */
    int pos_power;  /* raw power > 0 was clamped to 0 */
    double ea, eT;  /* fp32 error bounds (R18 model): alpha relative, T_k relative */
} OrComp;

/* Front-to-back compositing of one pixel (Eq. 3 discretised: C = sum c_i a_i T_i,
 * T_i = prod_{j<i} (1 - a_j)), with the inherited rules (R7, R12):
 *   power = -1/2 (a dx^2 + c dy^2) - b dx dy, clamped to <= 0
 *   [exact GEF kernel (Eq. 2): Q = -2 power, power = -1/2 Q^(beta/2)];
 *   alpha = min(0.99, kappa exp(power)); skip if alpha < 1/255;
 *   if T (1 - alpha) < 1e-4 stop WITHOUT compositing this particle.
 * Returns the number of composited entries written to rec (if rec != NULL).
 * amb: bit0 = a skip/stop decision lies within the fp32 error bound (the
 * image may legitimately differ), bit1 = a 0.99-clamp decision does. */
/* flip_at >= 0 (R18, both branches): the flip_at-th ambiguous decision of the pixel
 * (0-based, in list order) takes its other outcome; every other decision is made
 * as usual.  Returns -1 (and leaves C untouched) if the pixel has no such decision. */
static int composite_pixel_flip(const OrSplat2D *s, const int32_t *lst, int64_t n, double px, double py,
                                double C[3], double *T_out, int32_t *n_contrib, int32_t *n_eval, uint8_t *amb,
                                OrComp *rec, double *errT_out, int flip_at);
static int composite_pixel(const OrSplat2D *s, const int32_t *lst, int64_t n, double px, double py,
                           double C[3], double *T_out, int32_t *n_contrib, int32_t *n_eval, uint8_t *amb,
                           OrComp *rec, double *errT_out) {
    return composite_pixel_flip(s, lst, n, px, py, C, T_out, n_contrib, n_eval, amb, rec, errT_out, -1);
}
static int composite_pixel_flip(const OrSplat2D *s, const int32_t *lst, int64_t n, double px, double py,
                                double C[3], double *T_out, int32_t *n_contrib, int32_t *n_eval, uint8_t *amb,
                                OrComp *rec, double *errT_out, int flip_at) {
    int na = 0, flipped = 0;  /* ambiguous decisions met so far; whether flip_at was reached */
    const int64_t P = s->P;
    double T = 1.0, errT = 0.0;
    int nrec = 0;
    int32_t last = 0, ne = (int32_t)n;
    uint8_t a = 0;
    C[0] = C[1] = C[2] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        const int32_t i = lst[k];
        const double ca = s->conic[i], cb = s->conic[P + i], cc = s->conic[2 * P + i];
        const double dx = s->uv[i] - px, dy = s->uv[P + i] - py;
        const double qa = 0.5 * (ca * dx * dx + cc * dy * dy), qb = cb * dx * dy;
        double power = -qa - qb;
        int pos = 0;
        if (power > 0.0) { power = 0.0; pos = 1; }
        /* fp32 error bound of alpha relative to itself (R18) */
        double erel = 2e-6 + 6e-7 * (fabs(qa) + fabs(qb)) + g_amb_margin;
        double Q = 0.0, Qb = 0.0;
        if (s->hbeta) {
            const double hb = s->hbeta[i];
            Q = -2.0 * power;
            Qb = Q > 0.0 ? pow(Q, hb) : 0.0;
            power = -0.5 * Qb;
            /* R18 for the kernel's fp32 path Q^(beta/2) = 2^(hb (log2 q + c)), G = 2^(c' Q^hb):
             * q carries the quadratic form's relative error dq (the Gaussian bound's 6e-7),
             * lg2.approx adds <= 2.4e-7 absolute, hb (log2 Q) one rounding, ex2.approx <= 2.4e-7
             * relative; G's relative error is Q^hb / 2 times Qb's.  Safety factor 2. */
            const double dq = 6e-7 * (fabs(qa) + fabs(qb)) / (qa + qb > 1e-30 ? qa + qb : 1e-30);
            const double l2 = Q > 0.0 ? fabs(log2(Q)) : 0.0;
            const double eL = 2.4e-7 + dq / 0.6931;
            const double eQb = 0.6931 * (hb * eL + 6e-8 * hb * l2) + 2.4e-7;
            erel = 2.0 * (0.5 * Qb * eQb + 2.4e-7) + 2e-6 + g_amb_margin;
        }
        const double G = exp(power);
        const double araw = s->kappa[i] * G;
        int clamp = !(araw < OR_ALPHA_MAX);
        if (fabs(araw - OR_ALPHA_MAX) <= erel * araw) {
            a |= 2;
            if (na++ == flip_at) { clamp = !clamp; flipped = 1; }
        }
        const double alpha = clamp ? OR_ALPHA_MAX : araw;
        int skip = alpha < OR_ALPHA_MIN;
        if (fabs(araw - OR_ALPHA_MIN) <= erel * araw) {
            a |= 1;
            if (na++ == flip_at) { skip = !skip; flipped = 1; }
        }
        if (skip) continue;
        const double Tn = T * (1.0 - alpha);
        const double errTn = errT + erel * alpha / (1.0 - alpha) + 2.4e-7;
        int stop = Tn < OR_T_MIN;
        if (fabs(Tn - OR_T_MIN) <= OR_T_MIN * (errTn + 1e-6 + g_amb_margin)) {
            a |= 1;
            if (na++ == flip_at) { stop = !stop; flipped = 1; }
        }
        if (stop) { ne = (int32_t)(k + 1); break; }
        for (int ch = 0; ch < 3; ++ch) C[ch] += s->rgb[(int64_t)ch * P + i] * alpha * T;
        if (rec) {
            OrComp *r = &rec[nrec];
            r->k = (int32_t)k; r->idx = i; r->alpha = alpha; r->T = T; r->G = G; r->araw = araw;
            r->dx = dx; r->dy = dy; r->clamped = !(araw < OR_ALPHA_MAX); r->pos_power = pos;
            r->Q = Q; r->Qb = Qb;
            r->ea = erel; r->eT = errT;
        }
        ++nrec;
        T = Tn;
        errT = errTn;
        last = (int32_t)(k + 1);
    }
    *T_out = T;
    if (errT_out) *errT_out = errT;
    *n_contrib = last;
    *n_eval = ne;
    *amb = a;
    if (flip_at >= 0 && !flipped) return -1;
    return nrec;
}

/* R18 both branches: for every pixel with amb != 0, alt[f] = the image when the f-th
 * ambiguous decision of the pixel (list order) takes its other outcome, f < n_alt;
 * NaN where the pixel has fewer than f + 1 such decisions (or amb == 0). */
int or_render_fwd_alternatives(const OrScreen *sc, const OrSplat2D *s, const int64_t *offsets, const int32_t *list,
                               const uint8_t *amb_in, int n_alt, double *alt) {
    const int W = sc->width, H = sc->height;
    const int64_t T = (int64_t)sc->tiles_x * sc->tiles_y, HW = (int64_t)W * H;
    for (int64_t q = 0; q < (int64_t)n_alt * 3 * HW; ++q) alt[q] = NAN;
#pragma omp parallel for schedule(dynamic, 2)
    for (int64_t t = 0; t < T; ++t) {
        const int tx = (int)(t % sc->tiles_x), ty = (int)(t / sc->tiles_x);
        const int32_t *lst = list + offsets[t];
        const int64_t n = offsets[t + 1] - offsets[t];
        for (int yy = 0; yy < 16; ++yy)
            for (int xx = 0; xx < 16; ++xx) {
                const int px = tx * 16 + xx, py = ty * 16 + yy;
                if (px >= W || py >= H) continue;
                const int64_t pix = (int64_t)py * W + px;
                if (!amb_in[pix]) continue;
                for (int f = 0; f < n_alt; ++f) {
                    double C[3], Tf;
                    int32_t nc, ne;
                    uint8_t am;
                    if (composite_pixel_flip(s, lst, n, px + 0.5, py + 0.5, C, &Tf, &nc, &ne, &am, NULL, NULL, f) < 0)
                        break;
                    for (int ch = 0; ch < 3; ++ch) alt[((int64_t)f * 3 + ch) * HW + pix] = C[ch] + Tf * sc->bg[ch];
                }
            }
    }
    return 0;
}

int or_render_fwd(const OrScreen *sc, const OrSplat2D *s, const int64_t *offsets, const int32_t *list,
                  const uint8_t *tile_mask, double *image, double *final_T, int32_t *n_contrib, int32_t *n_eval,
                  int32_t *n_comp, uint8_t *amb) {
    const int W = sc->width, H = sc->height;
    const int64_t T = (int64_t)sc->tiles_x * sc->tiles_y;
#pragma omp parallel for schedule(dynamic, 2)
    for (int64_t t = 0; t < T; ++t) {
        if (tile_mask && !tile_mask[t]) continue;
        const int tx = (int)(t % sc->tiles_x), ty = (int)(t / sc->tiles_x);
        const int32_t *lst = list + offsets[t];
        const int64_t n = offsets[t + 1] - offsets[t];
        for (int yy = 0; yy < 16; ++yy)
            for (int xx = 0; xx < 16; ++xx) {
                const int px = tx * 16 + xx, py = ty * 16 + yy;
                if (px >= W || py >= H) continue;
                const int64_t pix = (int64_t)py * W + px;
                double C[3], Tf;
                n_comp[pix] = composite_pixel(s, lst, n, px + 0.5, py + 0.5, C, &Tf, &n_contrib[pix], &n_eval[pix],
                                              &amb[pix], NULL, NULL);
                for (int ch = 0; ch < 3; ++ch) image[(int64_t)ch * W * H + pix] = C[ch] + Tf * sc->bg[ch];
                final_T[pix] = Tf;
            }
    }
    return 0;
}

/* S5a: per pixel adjoint of the compositing.  With g = dL/dC(p):
 *   dL/drgb_k   += alpha_k T_k g
 *   dL/dalpha_k  = T_k (rgb_k . g) - (sum_{j>k} (rgb_j . g) alpha_j T_j + T_final (bg . g)) / (1 - alpha_k)
 *   unclamped:  dL/dkappa += G dL/dalpha ;  dL/dpower = kappa G dL/dalpha
 *   dL/d(a,b,c) += dL/dpower (-dx^2/2, -dx dy, -dy^2/2)
 *   dL/d(u,v)   += dL/dpower (-(a dx + b dy), -(b dx + c dy))
 * exact GEF kernel: power = -1/2 Q^h, h = beta/2, Q = -2 power_g (the Gaussian
 * power above), so the conic/mean chain takes dL/dpower_g = dL/dpower h Q^(h-1)
 * and dL/dbeta += dL/dpower (-1/4 Q^h ln Q) (0 at Q = 0).
 * Output g2d planar [10][P]: du, dv, da, db, dc, dkappa, dr, dg, db, dbeta. */
/* (Gaussian kernel: the dbeta plane is 0; beta enters through phi-bar in S5b.)
 * Accumulation order is fixed: tiles ascending, pixels row-major within the
 * tile, list order -- independent of the thread count. */
int or_render_bwd(const OrScreen *sc, const OrSplat2D *s, const int64_t *offsets, const int32_t *list,
                  const uint8_t *tile_mask, const double *dL_dimg, double *g2d, double *g2d_mag) {
    const int W = sc->width, H = sc->height;
    const int64_t P = s->P;
    const int64_t T = (int64_t)sc->tiles_x * sc->tiles_y;
    const int64_t total = offsets[T];
    double *acc = (double *)calloc((size_t)(total > 0 ? total : 1) * 10, sizeof(double));
    if (!acc) return -1;
    /* R19 (g2d_mag, [20][P], may be NULL):
     *   planes 0-9:  the same sums with every operand replaced by its magnitude
     *                and every difference by a sum -- sum over terms of |term|,
     *                the scale of fp32 rounding in the sums;
     *   planes 10-19: sum over terms of |term| x (its first-order relative
     *                sensitivity to the fp32 error of the alphas it depends on:
     *                eps_alpha of the pair and the accumulated eps_T of T_k, the
     *                error model of R18) -- how far any fp32 evaluation of the
     *                forward quantities moves the sum. */
    double *aab = NULL;
    if (g2d_mag) {
        aab = (double *)calloc((size_t)(total > 0 ? total : 1) * 20, sizeof(double));
        if (!aab) { free(acc); return -1; }
    }
#pragma omp parallel
    {
        int64_t maxn = 0;
        for (int64_t t = 0; t < T; ++t) if (offsets[t + 1] - offsets[t] > maxn) maxn = offsets[t + 1] - offsets[t];
        OrComp *rec = (OrComp *)malloc(sizeof(OrComp) * (size_t)(maxn > 0 ? maxn : 1));
#pragma omp for schedule(dynamic, 2)
        for (int64_t t = 0; t < T; ++t) {
            if (tile_mask && !tile_mask[t]) continue;
            const int tx = (int)(t % sc->tiles_x), ty = (int)(t / sc->tiles_x);
            const int32_t *lst = list + offsets[t];
            const int64_t n = offsets[t + 1] - offsets[t];
            double *a9 = acc + offsets[t] * 10;
            for (int yy = 0; yy < 16; ++yy)
                for (int xx = 0; xx < 16; ++xx) {
                    const int px = tx * 16 + xx, py = ty * 16 + yy;
                    if (px >= W || py >= H) continue;
                    const int64_t pix = (int64_t)py * W + px;
                    double C[3], Tf, eTf;
                    int32_t nc, ne;
                    uint8_t am;
                    const int nr = composite_pixel(s, lst, n, px + 0.5, py + 0.5, C, &Tf, &nc, &ne, &am, rec, &eTf);
                    const double g[3] = {dL_dimg[pix], dL_dimg[(int64_t)W * H + pix], dL_dimg[2 * (int64_t)W * H + pix]};
                    const double gbg = g[0] * sc->bg[0] + g[1] * sc->bg[1] + g[2] * sc->bg[2];
                    const double gbg_abs = fabs(g[0] * sc->bg[0]) + fabs(g[1] * sc->bg[1]) + fabs(g[2] * sc->bg[2]);
                    double suffix = 0.0, suffix_abs = 0.0, suffix_sens = 0.0;
                    for (int r = nr - 1; r >= 0; --r) {
                        const OrComp *c = &rec[r];
                        const int32_t i = c->idx;
                        const double cg = s->rgb[i] * g[0] + s->rgb[P + i] * g[1] + s->rgb[2 * P + i] * g[2];
                        const double dalpha = c->T * cg - (suffix + Tf * gbg) / (1.0 - c->alpha);
                        suffix += cg * c->alpha * c->T;
                        double *o = a9 + (int64_t)c->k * 10;
                        for (int ch = 0; ch < 3; ++ch) o[6 + ch] += c->alpha * c->T * g[ch];
                        /* R19 magnitudes: the same expressions over |operands| (ob[0..9]) and
                         * their fp32 sensitivities (ob[10..19]) */
                        double *ob = aab ? aab + (offsets[t] + c->k) * 20 : NULL;
                        double dalpha_abs = 0.0, dalpha_sens = 0.0;
                        if (ob) {
                            const double cg_abs = fabs(s->rgb[i] * g[0]) + fabs(s->rgb[P + i] * g[1]) +
                                                  fabs(s->rgb[2 * P + i] * g[2]);
                            const double amp = c->ea * c->alpha / (1.0 - c->alpha); /* rel. error of 1 - alpha */
                            const double tail = (suffix_abs + Tf * gbg_abs) / (1.0 - c->alpha);
                            dalpha_abs = c->T * cg_abs + tail;
                            dalpha_sens = c->T * cg_abs * c->eT + (suffix_sens + Tf * gbg_abs * eTf) / (1.0 - c->alpha) +
                                          tail * amp;
                            suffix_abs += cg_abs * c->alpha * c->T;
                            suffix_sens += cg_abs * c->alpha * c->T * (c->ea + c->eT);
                            for (int ch = 0; ch < 3; ++ch) {
                                ob[6 + ch] += fabs(c->alpha * c->T * g[ch]);
                                ob[16 + ch] += fabs(c->alpha * c->T * g[ch]) * (c->ea + c->eT);
                            }
                        }
                        if (c->clamped) continue;
                        o[5] += c->G * dalpha;
                        double dpow = c->pos_power ? 0.0 : c->araw * dalpha;
                        double dpow_abs = c->pos_power ? 0.0 : c->araw * dalpha_abs;
                        double dpow_sens = c->pos_power ? 0.0 : c->araw * (dalpha_sens + dalpha_abs * c->ea);
                        if (ob) {
                            ob[5] += c->G * dalpha_abs;
                            ob[15] += c->G * (dalpha_sens + dalpha_abs * c->ea);
                        }
                        if (s->hbeta) {
                            const double hb = s->hbeta[i];
                            const double d_all = c->araw * dalpha;  /* dL/dpower of the GEF power */
                            o[9] += c->Q > 0.0 ? d_all * (-0.25 * c->Qb * log(c->Q)) : 0.0;
                            dpow = c->Q > 0.0 ? d_all * hb * pow(c->Q, hb - 1.0) : 0.0;
                            if (ob) {
                                const double d_all_abs = c->araw * dalpha_abs;
                                const double d_all_sens = c->araw * (dalpha_sens + dalpha_abs * c->ea);
                                const double f9 = c->Q > 0.0 ? fabs(0.25 * c->Qb * log(c->Q)) : 0.0;
                                const double fp = c->Q > 0.0 ? hb * pow(c->Q, hb - 1.0) : 0.0;
                                ob[9] += d_all_abs * f9;
                                ob[19] += (d_all_sens + d_all_abs * c->ea) * f9;
                                dpow_abs = d_all_abs * fp;
                                dpow_sens = (d_all_sens + d_all_abs * c->ea) * fp;
                            }
                        }
                        const double ca = s->conic[i], cb = s->conic[P + i], cc = s->conic[2 * P + i];
                        const double dx = c->dx, dy = c->dy;
                        o[0] += dpow * (-(ca * dx + cb * dy));
                        o[1] += dpow * (-(cb * dx + cc * dy));
                        o[2] += dpow * (-0.5 * dx * dx);
                        o[3] += dpow * (-dx * dy);
                        o[4] += dpow * (-0.5 * dy * dy);
                        if (ob) {
                            const double geo[5] = {fabs(ca * dx) + fabs(cb * dy), fabs(cb * dx) + fabs(cc * dy),
                                                   0.5 * dx * dx, fabs(dx * dy), 0.5 * dy * dy};
                            for (int q = 0; q < 5; ++q) { ob[q] += dpow_abs * geo[q]; ob[10 + q] += dpow_sens * geo[q]; }
                        }
                    }
                }
        }
        free(rec);
    }
    memset(g2d, 0, sizeof(double) * 10 * (size_t)P);
    for (int64_t t = 0; t < T; ++t) {
        if (tile_mask && !tile_mask[t]) continue;
        for (int64_t k = offsets[t]; k < offsets[t + 1]; ++k) {
            const int32_t i = list[k];
            for (int c = 0; c < 10; ++c) g2d[c * P + i] += acc[k * 10 + c];
        }
    }
    if (g2d_mag) {
        memset(g2d_mag, 0, sizeof(double) * 20 * (size_t)P);
        for (int64_t t = 0; t < T; ++t) {
            if (tile_mask && !tile_mask[t]) continue;
            for (int64_t k = offsets[t]; k < offsets[t + 1]; ++k) {
                const int32_t i = list[k];
                for (int c = 0; c < 20; ++c) g2d_mag[c * P + i] += aab[k * 20 + c];
            }
        }
        free(aab);
    }
    free(acc);
    return 0;
}

/* ------------------------------------------------------------------ */
/* S5b: per-particle chain rule to the raw parameters (fp64)           */
/* ------------------------------------------------------------------ */
static void mat_mul(int n, int m, int p, const double *A, const double *B, double *C) {
    /* C[n][p] = A[n][m] B[m][p] */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < p; ++j) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += A[i * m + k] * B[k * p + j];
            C[i * p + j] = s;
        }
}
static void mat_T(int n, int m, const double *A, double *AT) {
    for (int i = 0; i < n; ++i) for (int j = 0; j < m; ++j) AT[j * n + i] = A[i * m + j];
}

/* Gradient of each real SH basis function with respect to the unit direction,
 * dY[k][0..2] (derivatives of the polynomials in sh_basis). */
static void sh_basis_grad(double x, double y, double z, int K, double dY[16][3]) {
    const double C1 = sqrt(3.0 / (4.0 * M_PI));
    const double C2a = 0.5 * sqrt(15.0 / M_PI), C2b = 0.25 * sqrt(5.0 / M_PI), C2c = 0.25 * sqrt(15.0 / M_PI);
    const double C3a = -0.25 * sqrt(35.0 / (2.0 * M_PI)), C3b = 0.5 * sqrt(105.0 / M_PI);
    const double C3c = -0.25 * sqrt(21.0 / (2.0 * M_PI)), C3d = 0.25 * sqrt(7.0 / M_PI), C3e = 0.25 * sqrt(105.0 / M_PI);
    memset(dY, 0, sizeof(double) * 16 * 3);
    if (K <= 1) return;
    dY[1][1] = -C1;
    dY[2][2] = C1;
    dY[3][0] = -C1;
    if (K <= 4) return;
    dY[4][0] = C2a * y;  dY[4][1] = C2a * x;
    dY[5][1] = -C2a * z; dY[5][2] = -C2a * y;
    dY[6][0] = -2 * C2b * x; dY[6][1] = -2 * C2b * y; dY[6][2] = 4 * C2b * z;
    dY[7][0] = -C2a * z; dY[7][2] = -C2a * x;
    dY[8][0] = 2 * C2c * x; dY[8][1] = -2 * C2c * y;
    if (K <= 9) return;
    dY[9][0] = 6 * C3a * x * y; dY[9][1] = C3a * (3 * x * x - 3 * y * y);
    dY[10][0] = C3b * y * z; dY[10][1] = C3b * x * z; dY[10][2] = C3b * x * y;
    dY[11][0] = -2 * C3c * x * y; dY[11][1] = C3c * (4 * z * z - x * x - 3 * y * y); dY[11][2] = 8 * C3c * y * z;
    dY[12][0] = -6 * C3d * x * z; dY[12][1] = -6 * C3d * y * z; dY[12][2] = C3d * (6 * z * z - 3 * x * x - 3 * y * y);
    dY[13][0] = C3c * (4 * z * z - 3 * x * x - y * y); dY[13][1] = -2 * C3c * x * y; dY[13][2] = 8 * C3c * x * z;
    dY[14][0] = 2 * C3e * x * z; dY[14][1] = -2 * C3e * y * z; dY[14][2] = C3e * (x * x - y * y);
    dY[15][0] = C3a * (3 * x * x - 3 * y * y); dY[15][1] = -6 * C3a * x * y;
}

/* grads: planar [n_planes][P] in ABI order: mean 3, log_scale 3, quat 4,
 * opacity_logit 1, sh 3K, beta 1.  status/flags (may be NULL) take the
 * visibility and clamp decisions from the fp32 path (the kernel's precision);
 * otherwise they are recomputed in fp64. */
static void mat_abs(int n, const double *A, double *out) {
    for (int i = 0; i < n; ++i) out[i] = fabs(A[i]);
}

/* absmode = 0: the gradients.  absmode = 1 (R19): the same chain evaluated over
 * magnitudes -- g2d holds the S5a sums of |terms|, every coefficient and matrix
 * is replaced by its absolute value (AB), every difference of terms by their
 * sum -- giving sum|terms| of each parameter gradient, the denominator of its
 * condition number.  AB() is the identity when absmode = 0, and every wrapped
 * expression is written so that its value there is bit-identical to the plain
 * chain (a - b == a + (-b)). */
static int backward_particles_impl(const OrParticles_f64 *pp, const OrCamera *cam, const OrSettings *st,
                                   const double *g2d, const int32_t *status_in, const int32_t *flags_in,
                                   double *grads, const int absmode) {
#define AB(x) (absmode ? fabs(x) : (x))
    const int64_t P = pp->P;
    const int K = (pp->sh_degree + 1) * (pp->sh_degree + 1);
    const int n_planes = 3 + 3 + 4 + 1 + 3 * K + 1;
    memset(grads, 0, sizeof(double) * (size_t)n_planes * (size_t)P);
    double *gmean = grads, *gls = grads + 3 * P, *gq = grads + 6 * P, *glogit = grads + 10 * P;
    double *gsh = grads + 11 * P, *gbeta = grads + (11 + 3 * K) * P;
    const double Wm[9] = {cam->R[0], cam->R[1], cam->R[2], cam->R[3], cam->R[4], cam->R[5], cam->R[6], cam->R[7], cam->R[8]};
    const double tc[3] = {cam->t[0], cam->t[1], cam->t[2]};
    const double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
    const double limx = 1.3 * (0.5 * cam->width / fx), limy = 1.3 * (0.5 * cam->height / fy);
    double ccen[3];
    for (int k = 0; k < 3; ++k) ccen[k] = -(Wm[0 * 3 + k] * tc[0] + Wm[1 * 3 + k] * tc[1] + Wm[2 * 3 + k] * tc[2]);
    const double rho = st->rho;
    (void)cx; (void)cy;

    /* fp64 geometry for visibility when no fp32 decisions are given */
    int32_t *st64 = NULL, *fl64 = NULL;
    if (!status_in || !flags_in) {
        OrPre_f64 pre;
        double *buf = (double *)calloc((size_t)P * 16, sizeof(double));
        int32_t *ib = (int32_t *)calloc((size_t)P * 13, sizeof(int32_t));
        pre.depth = buf; pre.uv = buf + P; pre.conic = buf + 3 * P; pre.cov2d = buf + 6 * P;
        pre.kappa = buf + 9 * P; pre.rgb = buf + 10 * P;
        pre.radius = ib; pre.rect = ib + P; pre.tiles = ib + 5 * P; pre.status = ib + 6 * P; pre.flags = ib + 7 * P;
        pre.rect3 = ib + 8 * P;
        preprocess_f64(pp, cam, st, &pre);
        st64 = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
        fl64 = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
        memcpy(st64, pre.status, sizeof(int32_t) * (size_t)P);
        memcpy(fl64, pre.flags, sizeof(int32_t) * (size_t)P);
        free(buf); free(ib);
    }
    const int32_t *status = status_in ? status_in : st64;
    const int32_t *flags = flags_in ? flags_in : fl64;

#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < P; ++i) {
        if (status[i] != OR_VISIBLE) continue;
        const int fl = flags[i];
        /* ---- forward recompute (fp64) ---- */
        const double m[3] = {pp->mean[i], pp->mean[P + i], pp->mean[2 * P + i]};
        double t[3];
        for (int j = 0; j < 3; ++j) t[j] = Wm[j * 3 + 0] * m[0] + Wm[j * 3 + 1] * m[1] + Wm[j * 3 + 2] * m[2] + tc[j];
        const double q[4] = {pp->quat[i], pp->quat[P + i], pp->quat[2 * P + i], pp->quat[3 * P + i]};
        const double nq = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        const double w = q[0] / nq, x = q[1] / nq, y = q[2] / nq, z = q[3] / nq;
        const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                             2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                             2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
        double s[3], se[3];
        double phi = 1.0, mfac = 1.0, dm_dbeta = 0.0;
        if (!st->gaussian_only && st->kernel == 0) {
            phi = 2.0 / (1.0 + exp(-(rho * (pp->beta[i] - 2.0))));
            const double dphi = rho * phi * (1.0 - 0.5 * phi); /* d phi-bar / d beta */
            if (st->phi_mode == OR_PHI_VARIANCE) { mfac = sqrt(phi); dm_dbeta = 0.5 * dphi / mfac; }
            else { mfac = phi; dm_dbeta = dphi; }
        }
        for (int k = 0; k < 3; ++k) { s[k] = exp(pp->log_scale[k * P + i]); se[k] = s[k] * mfac; }
        double M[9], MT[9], Sig[9];
        for (int j = 0; j < 3; ++j) for (int k = 0; k < 3; ++k) M[j * 3 + k] = R[j * 3 + k] * se[k];
        mat_T(3, 3, M, MT);
        mat_mul(3, 3, 3, M, MT, Sig);
        const double tx = t[0], ty = t[1], tz = t[2];
        const int clx = (fl >> 3) & 1, cly = (fl >> 4) & 1;
        const double Lx = (tx / tz > 0 ? limx : -limx), Ly = (ty / tz > 0 ? limy : -limy);
        const double txc = clx ? Lx * tz : tx, tyc = cly ? Ly * tz : ty;
        const double J[6] = {fx / tz, 0.0, -fx * txc / (tz * tz), 0.0, fy / tz, -fy * tyc / (tz * tz)};
        double Tm[6], TmT[6];
        mat_mul(2, 3, 3, J, Wm, Tm);
        mat_T(2, 3, Tm, TmT);
        double TS[6], cov[4];
        mat_mul(2, 3, 3, Tm, Sig, TS);
        mat_mul(2, 3, 2, TS, TmT, cov);
        const double A = cov[0] + 0.3, B = cov[1], C = cov[3] + 0.3;
        const double det = A * C - B * B, det2 = det * det;

        /* ---- incoming 2D gradients ---- */
        const double du = g2d[i], dv = g2d[P + i], da = g2d[2 * P + i], db = g2d[3 * P + i], dc = g2d[4 * P + i];
        const double dk = g2d[5 * P + i];
        double drgb[3] = {g2d[6 * P + i], g2d[7 * P + i], g2d[8 * P + i]};

        /* conic (a,b,c) = (C, -B, A) / det  ->  (A, B, C) */
        const double gA = da * AB(-C * C / det2) + db * AB(B * C / det2) + dc * (AB(1.0 / det) + AB(-A * C / det2));
        const double gB = da * AB(2.0 * B * C / det2) + db * (AB(-1.0 / det) + AB(-2.0 * B * B / det2)) +
                          dc * AB(2.0 * A * B / det2);
        const double gC = da * (AB(1.0 / det) + AB(-A * C / det2)) + db * AB(A * B / det2) + dc * AB(-A * A / det2);
        /* magnitudes of the forward matrices the adjoint multiplies by */
        double aTm[6], aTmT[6], aSig[9], aM[9], aMT[9];
        if (absmode) {
            mat_abs(9, M, aM);
            mat_T(3, 3, aM, aMT);
            mat_mul(3, 3, 3, aM, aMT, aSig);
            double aJ[6], aW[9];
            mat_abs(6, J, aJ);
            mat_abs(9, Wm, aW);
            mat_mul(2, 3, 3, aJ, aW, aTm);
            mat_T(2, 3, aTm, aTmT);
        } else {
            memcpy(aTm, Tm, sizeof aTm); memcpy(aTmT, TmT, sizeof aTmT);
            memcpy(aSig, Sig, sizeof aSig); memcpy(aM, M, sizeof aM);
        }
        /* cov = T Sig T^T, read entries (0,0), (0,1), (1,1) */
        const double Gc[4] = {gA, gB, 0.0, gC};
        double GcT[4], Gs[4];
        mat_T(2, 2, Gc, GcT);
        for (int k = 0; k < 4; ++k) Gs[k] = Gc[k] + GcT[k];
        double tmp6[6], dSig[9], dT[6];
        mat_mul(2, 2, 3, Gc, aTm, tmp6);     /* Gc T      */
        mat_mul(3, 2, 3, aTmT, tmp6, dSig);  /* T^T Gc T  */
        double GsT[6];
        mat_mul(2, 2, 3, Gs, aTm, GsT);      /* (Gc+Gc^T) T */
        mat_mul(2, 3, 3, GsT, aSig, dT);     /* ... Sig     */
        /* Sig = M M^T */
        double dSigS[9], dM[9];
        for (int j = 0; j < 3; ++j) for (int k = 0; k < 3; ++k) dSigS[j * 3 + k] = dSig[j * 3 + k] + dSig[k * 3 + j];
        mat_mul(3, 3, 3, dSigS, aM, dM);
        /* M = R diag(se) */
        double dR[9], dse[3] = {0, 0, 0};
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k) { dR[j * 3 + k] = dM[j * 3 + k] * se[k]; dse[k] += dM[j * 3 + k] * AB(R[j * 3 + k]); }
        double dbeta = 0.0;
        for (int k = 0; k < 3; ++k) {
            gls[k * P + i] = dse[k] * se[k];
            dbeta += dse[k] * s[k] * AB(dm_dbeta);
        }
        gbeta[i] = dbeta + (st->kernel == 1 ? g2d[9 * P + i] : 0.0);  /* exact GEF: the direct term */
        /* R(q-hat) partials */
        double dqh[4];
        dqh[0] = dR[1] * AB(-2 * z) + dR[2] * AB(2 * y) + dR[3] * AB(2 * z) + dR[5] * AB(-2 * x) +
                 dR[6] * AB(-2 * y) + dR[7] * AB(2 * x);
        dqh[1] = dR[1] * AB(2 * y) + dR[2] * AB(2 * z) + dR[3] * AB(2 * y) + dR[4] * AB(-4 * x) + dR[5] * AB(-2 * w) +
                 dR[6] * AB(2 * z) + dR[7] * AB(2 * w) + dR[8] * AB(-4 * x);
        dqh[2] = dR[0] * AB(-4 * y) + dR[1] * AB(2 * x) + dR[2] * AB(2 * w) + dR[3] * AB(2 * x) + dR[5] * AB(2 * z) +
                 dR[6] * AB(-2 * w) + dR[7] * AB(2 * z) + dR[8] * AB(-4 * y);
        dqh[3] = dR[0] * AB(-4 * z) + dR[1] * AB(-2 * w) + dR[2] * AB(2 * x) + dR[3] * AB(2 * w) + dR[4] * AB(-4 * z) +
                 dR[5] * AB(2 * y) + dR[6] * AB(2 * x) + dR[7] * AB(2 * y);
        const double qh[4] = {w, x, y, z};
        const double dotq = AB(qh[0]) * dqh[0] + AB(qh[1]) * dqh[1] + AB(qh[2]) * dqh[2] + AB(qh[3]) * dqh[3];
        for (int k = 0; k < 4; ++k) gq[k * P + i] = (dqh[k] + AB(-qh[k]) * dotq) / nq;
        /* T = J W  ->  dJ = dT W^T */
        double WT[9], dJ[6];
        mat_T(3, 3, Wm, WT);
        if (absmode) mat_abs(9, WT, WT);
        mat_mul(2, 3, 3, dT, WT, dJ);
        double dt[3] = {0, 0, 0};
        const double tz2 = tz * tz, tz3 = tz2 * tz;
        dt[2] += dJ[0] * AB(-fx / tz2) + dJ[4] * AB(-fy / tz2);
        if (!clx) { dt[0] += dJ[2] * AB(-fx / tz2); dt[2] += dJ[2] * AB(2.0 * fx * tx / tz3); }
        else { dt[2] += dJ[2] * AB(fx * Lx / tz2); }
        if (!cly) { dt[1] += dJ[5] * AB(-fy / tz2); dt[2] += dJ[5] * AB(2.0 * fy * ty / tz3); }
        else { dt[2] += dJ[5] * AB(fy * Ly / tz2); }
        /* projection u = fx tx/tz + cx, v = fy ty/tz + cy */
        dt[0] += AB(du * fx / tz); dt[2] += du * AB(-fx * tx / tz2);
        dt[1] += AB(dv * fy / tz); dt[2] += dv * AB(-fy * ty / tz2);
        double dmean[3];
        for (int k = 0; k < 3; ++k)
            dmean[k] = AB(Wm[0 * 3 + k]) * dt[0] + AB(Wm[1 * 3 + k]) * dt[1] + AB(Wm[2 * 3 + k]) * dt[2];
        /* colour: rgb = sum_k Y_k(dir) sh_k + 0.5, clamped at 0 */
        const double d[3] = {m[0] - ccen[0], m[1] - ccen[1], m[2] - ccen[2]};
        const double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        const double dir[3] = {d[0] / dn, d[1] / dn, d[2] / dn};
        double Y[16], dY[16][3];
        sh_basis_f64(dir[0], dir[1], dir[2], K, Y);
        sh_basis_grad(dir[0], dir[1], dir[2], K, dY);
        for (int ch = 0; ch < 3; ++ch) if ((fl >> ch) & 1) drgb[ch] = 0.0;
        double ddir[3] = {0, 0, 0};
        for (int k = 0; k < K; ++k)
            for (int ch = 0; ch < 3; ++ch) {
                gsh[(int64_t)(3 * k + ch) * P + i] = AB(Y[k]) * drgb[ch];
                const double shv = pp->sh[(int64_t)(3 * k + ch) * P + i];
                for (int e = 0; e < 3; ++e) ddir[e] += AB(drgb[ch] * shv * dY[k][e]);
            }
        const double dotd = AB(dir[0]) * ddir[0] + AB(dir[1]) * ddir[1] + AB(dir[2]) * ddir[2];
        for (int e = 0; e < 3; ++e) dmean[e] += (ddir[e] + AB(-dir[e]) * dotd) / dn;
        for (int e = 0; e < 3; ++e) gmean[e * P + i] = dmean[e];
        /* opacity */
        const double kap = 1.0 / (1.0 + exp(-pp->opacity_logit[i]));
        glogit[i] = dk * kap * (1.0 - kap);
    }
    free(st64);
    free(fl64);
    return 0;
#undef AB
}

int or_backward_particles(const OrParticles_f64 *pp, const OrCamera *cam, const OrSettings *st,
                          const double *g2d, const int32_t *status_in, const int32_t *flags_in, double *grads) {
    return backward_particles_impl(pp, cam, st, g2d, status_in, flags_in, grads, 0);
}

/* R19: sum|terms| of every parameter gradient entry, from the S5a magnitudes
 * g2d_abs of or_render_bwd (same layout as g2d). */
int or_backward_particles_abs(const OrParticles_f64 *pp, const OrCamera *cam, const OrSettings *st,
                              const double *g2d_abs, const int32_t *status_in, const int32_t *flags_in,
                              double *bound) {
    return backward_particles_impl(pp, cam, st, g2d_abs, status_in, flags_in, bound, 1);
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Vectorised helpers for the pins. */
void or_exp_spec_array(const float *x, float *y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = or_exp_spec(x[i]);
}

void or_log_spec_array(const float *x, float *y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = or_log_spec(x[i]);
}
