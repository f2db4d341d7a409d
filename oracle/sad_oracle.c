/* sad_oracle.c — TEST INFRASTRUCTURE ONLY (see sad_oracle.h).
 *
 * Plain-C restatement of the reference SAD fitting loop.  Each function names the reference
 * file:line it restates (paths relative to /root/reference/proj).  Built with
 * -O2 -ffp-contract=off like the reference (CMakeLists.txt:15-17) so float/double operations
 * round exactly as the reference's do; libm is the same glibc on the build and GPU hosts.
 */
#define _GNU_SOURCE
#include "sad_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* sado_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng.hpp:12-45 */
static inline uint32_t mix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h;
}

static uint32_t seeded_state(uint64_t seed, uint32_t a, uint32_t b) {
    uint32_t h = mix32((uint32_t)seed ^ 0x9e3779b9u);
    h ^= mix32((uint32_t)(seed >> 32) + 0x85ebca6bu);
    h = mix32(h + mix32(a ^ 0x27d4eb2fu));
    h = mix32(h ^ mix32(b + 0x165667b1u));
    return h ? h : 0x6b33a1c9u;
}

static inline uint32_t xs_next(uint32_t* s) {
    uint32_t x = *s;
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    *s = x;
    return x;
}

static inline double xs_unit(uint32_t* s) { return (xs_next(s) >> 8) * (1.0 / 16777216.0); }
static inline uint32_t xs_below(uint32_t* s, uint32_t n) { return n ? xs_next(s) % n : 0; }

uint32_t sado_seeded_state(uint64_t seed, uint32_t a, uint32_t b) { return seeded_state(seed, a, b); }

/* ------------------------------------------------------------------ half.hpp:10-64
 * Restated with the compiler's IEEE binary16 type (round-to-nearest-even conversions). */
uint16_t sado_float_to_half(float f) {
    _Float16 h = (_Float16)f;
    uint16_t b;
    memcpy(&b, &h, 2);
    return b;
}

float sado_half_to_float(uint16_t b) {
    _Float16 h;
    memcpy(&h, &b, 2);
    return (float)h;
}

static inline double half_rt(double v) { return (double)(float)(_Float16)(float)v; }

/* ------------------------------------------------------------------ accum.hpp:10-31 */
typedef struct {
    double hi, lo;
} accum_t;

static inline void accum_add(accum_t* a, double x) {
    double s = a->hi + x;
    double bb = s - a->hi;
    double err = (a->hi - (s - bb)) + (x - bb);
    a->hi = s;
    a->lo += err;
}

static inline void accum_merge(accum_t* a, const accum_t* o) {
    accum_add(a, o->hi);
    accum_add(a, o->lo);
}

static inline double accum_value(const accum_t* a) { return a->hi + a->lo; }

/* ------------------------------------------------------------------ types.hpp / score.cpp */
typedef struct {
    double x, y, log_tau, radius, cr, cg, cb, dx, dy, aniso;
    int active, frozen;
} site_t;

static site_t site_get(const sad_sites_view* s, size_t i) {
    site_t p = {s->x[i], s->y[i], s->log_tau[i], s->radius[i], s->col_r[i], s->col_g[i],
                s->col_b[i], s->dir_x[i], s->dir_y[i], s->aniso[i], s->active[i], s->frozen[i]};
    return p;
}

static void site_set(sad_sites_view* s, size_t i, const site_t* p) {
    s->x[i] = p->x; s->y[i] = p->y; s->log_tau[i] = p->log_tau; s->radius[i] = p->radius;
    s->col_r[i] = p->cr; s->col_g[i] = p->cg; s->col_b[i] = p->cb;
    s->dir_x[i] = p->dx; s->dir_y[i] = p->dy; s->aniso[i] = p->aniso;
    s->active[i] = p->active ? 1 : 0;
    s->frozen[i] = p->frozen ? 1 : 0;
    s->generation++;
}

/* half_packed (score.cpp:9-22) */
static site_t site_half(site_t p) {
    p.x = half_rt(p.x); p.y = half_rt(p.y); p.log_tau = half_rt(p.log_tau);
    p.radius = half_rt(p.radius); p.dx = half_rt(p.dx); p.dy = half_rt(p.dy);
    p.aniso = half_rt(p.aniso);
    return p;
}

/* site_logit = -exp(log_tau) * d_mix (score.cpp:24-46), all double */
static double site_logit_d(double px, double py, const site_t* s, double scale) {
    double ea = exp(s->aniso), ia = exp(-s->aniso);
    double ux = s->dx, uy = s->dy, vx = -uy, vy = ux;
    double gxx = ea * ux * ux + ia * vx * vx;
    double gxy = ea * ux * uy + ia * vx * vy;
    double gyy = ea * uy * uy + ia * vy * vy;
    double dx = px - s->x, dy = py - s->y;
    double q = gxx * dx * dx + 2.0 * gxy * dx * dy + gyy * dy * dy;
    if (q < 0) q = 0;
    double d = sqrt(q) * scale - s->radius * scale;
    return -exp(s->log_tau) * d;
}

/* normalization_scale (types.hpp:178-181) */
static double norm_scale(int w, int h) { return 1.0 / (double)(w > h ? w : h); }

/* SiteStore::active_ids (types.cpp:71-80) */
static uint32_t* active_list(const sad_sites_view* s, uint32_t* n) {
    uint32_t* a = (uint32_t*)malloc(4 * (s->size + 1));
    uint32_t c = 0;
    for (size_t i = 0; i < s->size; i++)
        if (s->active[i]) a[c++] = (uint32_t)i;
    *n = c;
    return a;
}

static int check_synced(const sad_sites_view* s, const sad_field_view* f) {
    if (f->synced_generation != s->generation)
        return fail(SAD_ESTALE, "candidate field is stale for this store");
    if (f->gw < 1 || f->gh < 1) return fail(SAD_EINVAL, "candidate field not sized");
    return SAD_OK;
}

/* ------------------------------------------------------------------ generic kernels */
#define T float
#define SFX f
#define EXPT expf
#define SQRTT sqrtf
#define TINY 1e-12f
#include "sad_oracle_t.inc"
#undef T
#undef SFX
#undef EXPT
#undef SQRTT
#undef TINY
#define T double
#define SFX d
#define EXPT exp
#define SQRTT sqrt
#define TINY 1e-18
#include "sad_oracle_t.inc"
#undef T
#undef SFX
#undef EXPT
#undef SQRTT
#undef TINY

/* ------------------------------------------------------------------ candidates.cpp */
static uint32_t ceil_log2(uint32_t v) {
    uint32_t e = 0;
    while ((1u << e) < v) e++;
    return e;
}

/* jump_step (candidates.cpp:27-33) */
int sado_jump_step(uint32_t t, uint32_t b, uint32_t* out) {
    if (b < 2 || (b & (b - 1)) != 0) return fail(SAD_EINVAL, "jump_step: b must be a power of two >= 2");
    uint32_t lg = ceil_log2(b);
    uint32_t e = (t < lg - 1 ? t : lg - 1) + 1;
    uint32_t s = b >> e;
    *out = s < 1 ? 1 : s;
    return SAD_OK;
}

/* JumpSchedule::for_extent + full_refresh_passes (candidates.cpp:13-46) */
int sado_full_refresh_passes(int gw, int gh, int extra, sad_pass_spec* out, int* n) {
    if (gw < 1 || gh < 1) return fail(SAD_EINVAL, "JumpSchedule: empty extent");
    uint32_t m = (uint32_t)(gw > gh ? gw : gh);
    uint32_t b = 1u << ceil_log2(m);
    if (b < 2) b = 2;
    uint32_t events = ceil_log2(m);
    int total = (int)events + (extra > 0 ? extra : 0);
    if (total > *n) return fail(SAD_EINVAL, "pass buffer too small");
    int c = 0;
    for (uint32_t t = 0; t < events; t++) {
        uint32_t s;
        sado_jump_step(t, b, &s);
        out[c].step = s;
        out[c++].stencil = 1;
    }
    for (int i = 0; i < extra; i++) {
        out[c].step = 1;
        out[c++].stencil = 0;
    }
    *n = c;
    return SAD_OK;
}

/* jfa_seed (candidates.cpp:64-84) */
int sado_jfa_seed(const sad_sites_view* s, sad_field_view* f) {
    size_t cells = (size_t)f->gw * f->gh * f->k;
    for (size_t i = 0; i < cells; i++) f->ids[i] = SAD_EMPTY_ID;
    double scale = norm_scale(f->width, f->height);
    for (size_t id = 0; id < s->size; id++) {
        if (!s->active[id]) continue;
        long px = lround(s->x[id]), py = lround(s->y[id]);
        if (px < 0) px = 0;
        if (px > f->width - 1) px = f->width - 1;
        if (py < 0) py = 0;
        if (py > f->height - 1) py = f->height - 1;
        int gx = (int)px / f->cell, gy = (int)py / f->cell;
        uint32_t* slot = f->ids + (size_t)f->k * ((size_t)gy * f->gw + gx);
        if (slot[0] == SAD_EMPTY_ID) {
            slot[0] = (uint32_t)id;
            continue;
        }
        double cx = gx * (double)f->cell + (f->cell - 1) * 0.5;
        double cy = gy * (double)f->cell + (f->cell - 1) * 0.5;
        site_t a = site_half(site_get(s, slot[0])), b = site_half(site_get(s, id));
        double cur = site_logit_d(cx, cy, &a, scale), cand = site_logit_d(cx, cy, &b, scale);
        if (cand > cur || (cand == cur && (uint32_t)id < slot[0])) slot[0] = (uint32_t)id;
    }
    f->synced_generation = s->generation;
    return SAD_OK;
}

int sado_run_passes(const sad_sites_view* s, sad_field_view* f, const sad_pass_spec* seq, int n_pass,
                    int inject, uint64_t seed, int fp64) {
    if (f->gw < 1 || f->gh < 1) return fail(SAD_EINVAL, "run_passes: field not sized");
    if (fp64)
        run_passes_d(s, f, seq, n_pass, inject, seed);
    else
        run_passes_f(s, f, seq, n_pass, inject, seed);
    return SAD_OK;
}

/* refresh (candidates.cpp:183-194) */
int sado_refresh(const sad_sites_view* s, sad_field_view* f, int mode, int passes, int inject,
                 uint64_t seed, int fp64) {
    int rc;
    if (mode == SAD_REFRESH_FULL) {
        sad_pass_spec seq[64 + 4096];
        int n = (int)(sizeof seq / sizeof seq[0]);
        if ((rc = sado_full_refresh_passes(f->gw, f->gh, passes, seq, &n))) return rc;
        sado_jfa_seed(s, f);
        rc = sado_run_passes(s, f, seq, n, inject, seed, fp64);
    } else {
        int n = passes < 0 ? 0 : passes;
        sad_pass_spec* seq = (sad_pass_spec*)malloc(sizeof(sad_pass_spec) * (n + 1));
        for (int i = 0; i < n; i++) {
            seq[i].step = 1;
            seq[i].stencil = 0;
        }
        rc = sado_run_passes(s, f, seq, n, inject, seed, fp64);
        free(seq);
    }
    if (rc) return rc;
    f->refresh_count++;
    return SAD_OK;
}

/* ------------------------------------------------------------------ render.cpp */
int sado_render_image(const sad_sites_view* s, const sad_field_view* f, int fp64, double* out) {
    int rc = check_synced(s, f);
    if (rc) return rc;
    return fp64 ? render_d(s, f, out) : render_f(s, f, out);
}

/* render_id_map (render.cpp:118-154): argmax of the double ScoreTable logit, ties to lower id */
int sado_render_id_map(const sad_sites_view* s, const sad_field_view* f, uint32_t* out) {
    int rc = check_synced(s, f);
    if (rc) return rc;
    score_tab_d tab;
    score_tab_build_d(&tab, s, norm_scale(f->width, f->height), 0);
    int empty = 0;
    for (int py = 0; py < f->height; py++)
        for (int px = 0; px < f->width; px++) {
            const uint32_t* lst = f->ids + (size_t)f->k * ((size_t)(py / f->cell) * f->gw + px / f->cell);
            uint32_t best = SAD_EMPTY_ID;
            double bl = 0;
            for (int i = 0; i < f->k; i++) {
                uint32_t id = lst[i];
                if (id == SAD_EMPTY_ID) break;
                if (!s->active[id]) continue;
                double l = score_logit_d(&tab, px, py, id);
                if (best == SAD_EMPTY_ID || l > bl || (l == bl && id < best)) {
                    best = id;
                    bl = l;
                }
            }
            out[(size_t)py * f->width + px] = best;
            if (best == SAD_EMPTY_ID) empty = 1;
        }
    score_tab_free_d(&tab);
    return empty ? fail(SAD_EEMPTY, "render: empty candidate list at a pixel") : SAD_OK;
}

/* ------------------------------------------------------------------ grad.cpp */
static int backward_common(const sad_sites_view* s, const sad_field_view* f, const double* tgt,
                           const double* pg, int fp64, int with_removal, double* grads,
                           uint64_t* nonfinite, double* loss) {
    int rc = check_synced(s, f);
    if (rc) return rc;
    accum_t* acc = (accum_t*)calloc(s->size * 11 + 1, sizeof(accum_t));
    uint64_t nf = 0;
    double l = 0;
    rc = fp64 ? backward_d(s, f, tgt, pg, with_removal, acc, &nf, &l)
              : backward_f(s, f, tgt, pg, with_removal, acc, &nf, &l);
    if (!rc) {
        for (size_t i = 0; i < s->size * 11; i++) grads[i] = accum_value(&acc[i]);
        if (nonfinite) *nonfinite = nf;
        if (loss) *loss = l;
    }
    free(acc);
    return rc;
}

int sado_backward_image(const sad_sites_view* s, const sad_field_view* f, const double* tgt, int fp64,
                        int with_removal, double* grads, uint64_t* nonfinite, double* loss) {
    return backward_common(s, f, tgt, NULL, fp64, with_removal, grads, nonfinite, loss);
}

int sado_image_loss(const sad_sites_view* s, const sad_field_view* f, const double* tgt, int fp64,
                    double* loss) {
    int rc = check_synced(s, f);
    if (rc) return rc;
    return fp64 ? loss_d(s, f, tgt, loss) : loss_f(s, f, tgt, loss);
}

/* tau_diffusion (train.cpp:171-213): every pixel owner's logtau gradient becomes
 * (1 - lambda) g0[o] + lambda * (sequential ascending-id sum of g0 over its unique co-candidates) / count,
 * stored through a reset Accum (reset + add). */
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y);
}

int sado_tau_diffusion(const sad_sites_view* s, const sad_field_view* f, double lambda, double* grads) {
    if (lambda == 0) return SAD_OK;
    if (lambda < 0 || lambda > 1) return fail(SAD_EINVAL, "tau_diffusion: lambda out of [0,1]");
    size_t np = (size_t)f->width * f->height;
    uint32_t* owner = (uint32_t*)malloc(4 * np + 4);
    int rc = sado_render_id_map(s, f, owner);
    if (rc) {
        free(owner);
        return rc;
    }
    uint64_t* e = (uint64_t*)malloc(8 * np * f->k + 8);
    size_t ne = 0;
    for (int py = 0; py < f->height; py++)
        for (int px = 0; px < f->width; px++) {
            uint64_t o = owner[(size_t)py * f->width + px];
            const uint32_t* lst = f->ids + (size_t)f->k * ((size_t)(py / f->cell) * f->gw + px / f->cell);
            for (int i = 0; i < f->k; i++) {
                uint32_t id = lst[i];
                if (id == SAD_EMPTY_ID) break;
                if (!s->active[id]) continue;
                e[ne++] = (o << 32) | id;
            }
        }
    qsort(e, ne, 8, cmp_u64); /* (owner, id) pair order == u64 order */
    size_t nu = 0;
    for (size_t i = 0; i < ne; i++)
        if (nu == 0 || e[nu - 1] != e[i]) e[nu++] = e[i];
    double* g0 = (double*)malloc(8 * s->size + 8);
    for (size_t i = 0; i < s->size; i++) g0[i] = grads[i * 11 + 2];
    size_t i = 0;
    while (i < nu) {
        uint32_t o = (uint32_t)(e[i] >> 32);
        double sum = 0;
        int cnt = 0;
        while (i < nu && (uint32_t)(e[i] >> 32) == o) {
            sum += g0[(uint32_t)e[i]];
            cnt++;
            i++;
        }
        double mixed = (1.0 - lambda) * g0[o] + lambda * (sum / cnt);
        accum_t a = {0.0, 0.0};
        accum_add(&a, mixed);
        grads[(size_t)o * 11 + 2] = accum_value(&a);
    }
    free(g0);
    free(e);
    free(owner);
    return SAD_OK;
}

/* ------------------------------------------------------------------ train.cpp */
static inline double mx(double a, double b) { return (a < b) ? b : a; } /* std::max */
static inline double mn(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* clamp_project (train.cpp:113-137) */
int sado_clamp_project(sad_sites_view* s, int w, int h, const sad_train_config* c) {
    for (size_t i = 0; i < s->size; i++) {
        if (!s->active[i] || s->frozen[i]) continue;
        s->x[i] = mn(mx(s->x[i], 0.0), w - 1.0);
        s->y[i] = mn(mx(s->y[i], 0.0), h - 1.0);
        s->log_tau[i] = mn(mx(s->log_tau[i], c->log_tau_min), c->log_tau_max);
        s->radius[i] = mn(mx(s->radius[i], c->radius_min), c->radius_max);
        s->aniso[i] = mn(mx(s->aniso[i], c->aniso_min), c->aniso_max);
        if (c->clamp_color) {
            s->col_r[i] = mn(mx(s->col_r[i], 0.0), 1.0);
            s->col_g[i] = mn(mx(s->col_g[i], 0.0), 1.0);
            s->col_b[i] = mn(mx(s->col_b[i], 0.0), 1.0);
        }
        double nx = s->dir_x[i], ny = s->dir_y[i];
        double nrm = sqrt(nx * nx + ny * ny);
        if (!(nrm > 1e-12) || !isfinite(nrm)) {
            s->dir_x[i] = 1.0;
            s->dir_y[i] = 0.0;
        } else {
            s->dir_x[i] = nx / nrm;
            s->dir_y[i] = ny / nrm;
        }
    }
    s->generation++;
    return SAD_OK;
}

/* adam_step (train.cpp:139-169) */
int sado_adam_step(sad_sites_view* s, const double* grads, sad_adam_view* a, int w, int h,
                   const sad_train_config* c) {
    if (a->sites != s->size) {
        if (s->size > a->capacity) return fail(SAD_ENOMEM, "adam capacity");
        for (size_t i = a->sites * 10; i < s->size * 10; i++) a->m[i] = a->v[i] = 0.0; /* resize */
        a->sites = s->size;
    }
    a->t++;
    double bc1 = 1.0 - pow(c->beta1, (double)a->t);
    double bc2 = 1.0 - pow(c->beta2, (double)a->t);
    const double lrs[10] = {c->lr_pos, c->lr_pos, c->lr_log_tau, c->lr_radius, c->lr_color,
                            c->lr_color, c->lr_color, c->lr_dir, c->lr_dir, c->lr_aniso};
    for (size_t id = 0; id < s->size; id++) {
        if (!s->active[id] || s->frozen[id]) continue;
        double* p[10] = {&s->x[id], &s->y[id], &s->log_tau[id], &s->radius[id], &s->col_r[id],
                         &s->col_g[id], &s->col_b[id], &s->dir_x[id], &s->dir_y[id], &s->aniso[id]};
        for (int k = 0; k < 10; k++) {
            double gv = grads[id * 11 + k];
            if (!isfinite(gv)) {
                a->skipped++;
                continue;
            }
            size_t mi = id * 10 + k;
            double m = a->m[mi] = c->beta1 * a->m[mi] + (1.0 - c->beta1) * gv;
            double v = a->v[mi] = c->beta2 * a->v[mi] + (1.0 - c->beta2) * gv * gv;
            *p[k] -= lrs[k] * (m / bc1) / (sqrt(v / bc2) + c->adam_eps);
        }
    }
    s->generation++;
    return sado_clamp_project(s, w, h, c);
}

/* sobel_magnitude (train.cpp:33-57) */
static double* sobel(const double* img, int w, int h) {
    size_t n = (size_t)w * h;
    double* l = (double*)malloc(n * 8);
    double* m = (double*)malloc(n * 8);
    for (size_t i = 0; i < n; i++) l[i] = 0.2126 * img[3 * i] + 0.7152 * img[3 * i + 1] + 0.0722 * img[3 * i + 2];
#define LA(X, Y) l[(size_t)((Y) < 0 ? 0 : (Y) > h - 1 ? h - 1 : (Y)) * w + ((X) < 0 ? 0 : (X) > w - 1 ? w - 1 : (X))]
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) {
            double gx = (LA(x + 1, y - 1) + 2 * LA(x + 1, y) + LA(x + 1, y + 1)) -
                        (LA(x - 1, y - 1) + 2 * LA(x - 1, y) + LA(x - 1, y + 1));
            double gy = (LA(x - 1, y + 1) + 2 * LA(x, y + 1) + LA(x + 1, y + 1)) -
                        (LA(x - 1, y - 1) + 2 * LA(x, y - 1) + LA(x + 1, y - 1));
            m[(size_t)y * w + x] = sqrt(gx * gx + gy * gy);
        }
#undef LA
    free(l);
    return m;
}

typedef struct {
    double key;
    uint32_t idx;
} keyed_t;

/* (key desc, idx asc) — the `better` order of train.cpp:86-88 */
static int cmp_better(const void* a, const void* b) {
    const keyed_t* x = (const keyed_t*)a;
    const keyed_t* y = (const keyed_t*)b;
    if (x->key > y->key) return -1;
    if (x->key < y->key) return 1;
    return (x->idx < y->idx) ? -1 : (x->idx > y->idx);
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* init_sites (train.cpp:59-111): exponential-key weighted sampling without replacement.  The
 * reference's nth_element + sort yields the n best (key desc, idx asc) cells in raster order;
 * a full sort under the same strict order selects the identical set. */
int sado_init_sites(sad_sites_view* s, const double* img, int w, int h, int n, const sad_train_config* c) {
    size_t np = (size_t)w * h;
    if (n < 1 || (size_t)n > np) return fail(SAD_EINVAL, "init_sites: count out of range");
    if ((size_t)n > s->capacity) return fail(SAD_ENOMEM, "sites capacity");
    double* g = sobel(img, w, h);
    accum_t tot = {0, 0};
    for (size_t i = 0; i < np; i++) accum_add(&tot, g[i]);
    double gsum = accum_value(&tot);
    double lambda = c->lambda_init;
    if (gsum <= 0) lambda = 1.0;
    double uni = 1.0 / (double)np;
    uint32_t rs = seeded_state(c->seed, 0x1717, 0);
    keyed_t* k = (keyed_t*)malloc(np * sizeof(keyed_t));
    for (size_t i = 0; i < np; i++) {
        double wgt = lambda * uni + (gsum > 0 ? (1.0 - lambda) * g[i] / gsum : 0.0);
        if (wgt < 1e-300) wgt = 1e-300;
        double u = xs_unit(&rs);
        if (u < 1e-12) u = 1e-12;
        k[i].key = log(u) / wgt;
        k[i].idx = (uint32_t)i;
    }
    qsort(k, np, sizeof(keyed_t), cmp_better);
    uint32_t* cells = (uint32_t*)malloc(4 * (size_t)n);
    for (int i = 0; i < n; i++) cells[i] = k[i].idx;
    qsort(cells, (size_t)n, 4, cmp_u32);
    double r0 = c->init_radius > 0 ? c->init_radius : sqrt((double)w * h / (double)n);
    uint32_t os = seeded_state(c->seed, 0x1717, 1);
    s->size = 0;
    s->generation++;
    for (int i = 0; i < n; i++) {
        int cx = (int)(cells[i] % (uint32_t)w), cy = (int)(cells[i] / (uint32_t)w);
        site_t p;
        p.x = mn(cx + 0.25 + 0.5 * xs_unit(&os), w - 1.0);
        p.y = mn(cy + 0.25 + 0.5 * xs_unit(&os), h - 1.0);
        p.log_tau = c->init_log_tau;
        p.radius = r0;
        p.aniso = c->init_aniso;
        p.dx = 1.0;
        p.dy = 0.0;
        const double* col = img + 3 * ((size_t)cy * w + cx);
        p.cr = col[0]; p.cg = col[1]; p.cb = col[2];
        p.active = 1;
        p.frozen = 0;
        site_set(s, s->size, &p);
        s->size++;
    }
    free(cells);
    free(k);
    free(g);
    return SAD_OK;
}

/* ------------------------------------------------------------------ budget.cpp */
/* accumulate_stats (budget.cpp:39-155): always double, ScoreTable (unpacked) logits. */
int sado_accumulate_stats(const sad_sites_view* s, const sad_field_view* f, const double* tgt,
                          double* stats, uint64_t* valid) {
    if (f->synced_generation != s->generation) return fail(SAD_ESTALE, "stats: candidate field is stale");
    score_tab_d tab;
    score_tab_build_d(&tab, s, norm_scale(f->width, f->height), 0);
    accum_t* acc = (accum_t*)calloc(s->size * 8 + 1, sizeof(accum_t));
    uint64_t nv = 0;
    for (int py = 0; py < f->height; py++)
        for (int px = 0; px < f->width; px++) {
            const uint32_t* lst = f->ids + (size_t)f->k * ((size_t)(py / f->cell) * f->gw + px / f->cell);
            uint32_t ids[16];
            double lg[16], w[16];
            int n = 0;
            double best = 0;
            for (int i = 0; i < f->k; i++) {
                uint32_t id = lst[i];
                if (id == SAD_EMPTY_ID) break;
                if (!s->active[id]) continue;
                double l = score_logit_d(&tab, (double)px, (double)py, id);
                if (!isfinite(l)) continue;
                ids[n] = id;
                lg[n] = l;
                if (n == 0 || l > best) best = l;
                n++;
            }
            if (n == 0) continue;
            nv++;
            double wsum = 0;
            for (int i = 0; i < n; i++) {
                w[i] = exp(lg[i] - best);
                wsum += w[i];
            }
            double invw = 1.0 / wsum;
            double ch[3] = {0, 0, 0};
            for (int i = 0; i < n; i++) {
                w[i] *= invw;
                ch[0] += w[i] * s->col_r[ids[i]];
                ch[1] += w[i] * s->col_g[ids[i]];
                ch[2] += w[i] * s->col_b[ids[i]];
            }
            const double* tp = tgt + 3 * ((size_t)py * f->width + px);
            double e0 = ch[0] - tp[0], e1 = ch[1] - tp[1], e2 = ch[2] - tp[2];
            double r2 = e0 * e0 + e1 * e1 + e2 * e2;
            double fx = px, fy = py;
            for (int i = 0; i < n; i++) {
                double rho = w[i] * r2, c[8];
                c[0] = w[i];
                c[1] = rho;
                c[2] = rho * fx;
                c[3] = rho * fy;
                c[4] = rho * fx * fx;
                c[5] = rho * fx * fy;
                c[6] = rho * fy * fy;
                if (w[i] >= 1.0 - 1e-6) {
                    c[7] = 1e6;
                } else {
                    double ir = 1.0 / (1.0 - w[i]);
                    double r0 = (ch[0] - w[i] * s->col_r[ids[i]]) * ir - tp[0];
                    double r1 = (ch[1] - w[i] * s->col_g[ids[i]]) * ir - tp[1];
                    double rk = (ch[2] - w[i] * s->col_b[ids[i]]) * ir - tp[2];
                    c[7] = r0 * r0 + r1 * r1 + rk * rk - r2;
                }
                for (int t = 0; t < 8; t++) {
                    if (!isfinite(c[t])) c[t] = 0;
                    accum_add(&acc[(size_t)ids[i] * 8 + t], c[t]);
                }
            }
        }
    for (size_t i = 0; i < s->size * 8; i++) stats[i] = accum_value(&acc[i]);
    *valid = nv;
    free(acc);
    score_tab_free_d(&tab);
    return SAD_OK;
}

static int cmp_key_asc(const void* a, const void* b) {
    const keyed_t* x = (const keyed_t*)a;
    const keyed_t* y = (const keyed_t*)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/* prune (budget.cpp:286-305) */
int sado_prune(sad_sites_view* s, const double* stats, uint64_t valid, double pct, int* removed) {
    *removed = 0;
    if (pct <= 0) return SAD_OK;
    if (pct > 1) return fail(SAD_EINVAL, "prune: percentile out of (0,1]");
    keyed_t* e = (keyed_t*)malloc(sizeof(keyed_t) * (s->size + 1));
    size_t ne = 0;
    double norm = (double)(valid > 1 ? valid : 1);
    for (size_t id = 0; id < s->size; id++)
        if (s->active[id] && !s->frozen[id]) {
            e[ne].key = stats[id * 8 + 7] / norm;
            e[ne++].idx = (uint32_t)id;
        }
    int want = (int)((double)ne * pct);
    if (want >= 1) {
        qsort(e, ne, sizeof(keyed_t), cmp_key_asc);
        for (int i = 0; i < want; i++) {
            uint32_t id = e[i].idx;
            s->active[id] = 0;
            s->x[id] = -1.0;
            s->y[id] = -1.0;
            s->generation++;
        }
        *removed = want;
    }
    free(e);
    return SAD_OK;
}

static double luma_at(const double* img, int w, int h, int x, int y) {
    x = x < 0 ? 0 : x > w - 1 ? w - 1 : x;
    y = y < 0 ? 0 : y > h - 1 ? h - 1 : y;
    const double* p = img + 3 * ((size_t)y * w + x);
    return 0.2126 * p[0] + 0.7152 * p[1] + 0.0722 * p[2];
}

/* split_axis (budget.cpp:170-215) */
static void split_axis(const double* st, const site_t* par, const double* img, int w, int h,
                       const sad_train_config* c, double* ax, double* ay, double* an) {
    *ax = 1; *ay = 0; *an = 0;
    int fallback = 1;
    double mass = st[0], energy = st[1];
    if (mass >= 4.0 && energy > 0) {
        double wv = energy, mxv = st[2] / wv, myv = st[3] / wv;
        double cxx = st[4] / wv - mxv * mxv, cyy = st[6] / wv - myv * myv, cxy = st[5] / wv - mxv * myv;
        double half = 0.5 * (cxx - cyy);
        double root = sqrt(half * half + cxy * cxy);
        double mid = 0.5 * (cxx + cyy);
        double l1 = mid + root, l2 = mid - root;
        if (l1 > 0 && (l2 <= 0 || l1 > 1.05 * l2)) {
            double vx = cxy, vy = l1 - cxx;
            double n = sqrt(vx * vx + vy * vy);
            if (n < 1e-18 * l1) {
                vx = l1 - cyy;
                vy = cxy;
                n = sqrt(vx * vx + vy * vy);
            }
            if (n > 0 && isfinite(n)) {
                *ax = vx / n;
                *ay = vy / n;
                double ratio = l2 > 0 ? l1 / l2 : 1e18;
                double a = -0.5 * log(ratio);
                *an = a < c->aniso_min ? c->aniso_min : (a > c->aniso_max ? c->aniso_max : a);
                fallback = 0;
            }
        }
    }
    if (fallback) {
        int px = (int)lround(par->x), py = (int)lround(par->y);
        double gx = (luma_at(img, w, h, px + 1, py - 1) + 2 * luma_at(img, w, h, px + 1, py) +
                     luma_at(img, w, h, px + 1, py + 1)) -
                    (luma_at(img, w, h, px - 1, py - 1) + 2 * luma_at(img, w, h, px - 1, py) +
                     luma_at(img, w, h, px - 1, py + 1));
        double gy = (luma_at(img, w, h, px - 1, py + 1) + 2 * luma_at(img, w, h, px, py + 1) +
                     luma_at(img, w, h, px + 1, py + 1)) -
                    (luma_at(img, w, h, px - 1, py - 1) + 2 * luma_at(img, w, h, px, py - 1) +
                     luma_at(img, w, h, px + 1, py - 1));
        double n = sqrt(gx * gx + gy * gy);
        if (n > 1e-12) {
            *ax = gx / n;
            *ay = gy / n;
        }
        double a = 0.8 * par->aniso;
        *an = a < c->aniso_min ? c->aniso_min : (a > c->aniso_max ? c->aniso_max : a);
    }
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* densify (budget.cpp:219-284) */
int sado_densify(sad_sites_view* s, sad_adam_view* a, const double* stats, const double* img, int w,
                 int h, double pct, const sad_train_config* c, int* done) {
    *done = 0;
    if (pct <= 0) return SAD_OK;
    if (pct > 1) return fail(SAD_EINVAL, "densify: percentile out of (0,1]");
    size_t n0 = s->size;
    keyed_t* e = (keyed_t*)malloc(sizeof(keyed_t) * (n0 + 1));
    size_t ne = 0;
    for (size_t id = 0; id < n0; id++)
        if (s->active[id] && !s->frozen[id] && stats[id * 8] > 1.0) {
            /* densify_score (budget.cpp:157-159); descending -> sort on the negated key */
            double sc = stats[id * 8 + 1] / pow(mx(stats[id * 8], c->stats_eps), c->alpha);
            e[ne].key = -sc;
            e[ne++].idx = (uint32_t)id;
        }
    int want = (int)((double)ne * pct);
    if (want < 1) {
        free(e);
        return SAD_OK;
    }
    qsort(e, ne, sizeof(keyed_t), cmp_key_asc);
    uint32_t* fr = (uint32_t*)malloc(4 * (n0 + 1));
    size_t nf = 0, next = 0;
    for (size_t id = 0; id < n0; id++)
        if (!s->active[id]) fr[nf++] = (uint32_t)id;
    int cnt = 0;
    for (int i = 0; i < want; i++) {
        uint32_t p = e[i].idx;
        int have = next < nf;
        if (!have && c->max_sites > 0 && s->size >= c->max_sites) break;
        if (!have && s->size >= s->capacity) {
            free(e);
            free(fr);
            return fail(SAD_ENOMEM, "densify: sites capacity");
        }
        const double* st = stats + (size_t)p * 8;
        site_t par = site_get(s, p);
        double ax, ay, an;
        split_axis(st, &par, img, w, h, c, &ax, &ay, &an);
        double mag = clampd(0.5 * sqrt(mx(st[0], 0.0)), 1.5, 48.0);
        site_t ch = par;
        ch.log_tau = mx(par.log_tau - 0.25, c->log_tau_min);
        ch.radius = mx(par.radius * 0.85, c->radius_min);
        ch.aniso = an;
        ch.dx = ax;
        ch.dy = ay;
        for (int side = 0; side < 2; side++) {
            site_t q = ch;
            double sg = side == 0 ? 1.0 : -1.0;
            q.x = clampd(par.x + sg * ax * mag, 0.0, w - 1.0);
            q.y = clampd(par.y + sg * ay * mag, 0.0, h - 1.0);
            int cx = (int)lround(q.x), cy = (int)lround(q.y);
            const double* col = img + 3 * ((size_t)cy * w + cx);
            q.cr = col[0]; q.cg = col[1]; q.cb = col[2];
            size_t slot;
            if (side == 0) {
                slot = p;
            } else if (have) {
                slot = fr[next++];
            } else {
                slot = s->size++;
            }
            site_set(s, slot, &q);
            if (slot >= a->sites) {
                if (slot >= a->capacity) {
                    free(e);
                    free(fr);
                    return fail(SAD_ENOMEM, "densify: adam capacity");
                }
                for (size_t r = a->sites * 10; r < (slot + 1) * 10; r++) a->m[r] = a->v[r] = 0.0;
                a->sites = slot + 1;
            }
            for (int k = 0; k < 10; k++) a->m[slot * 10 + k] = a->v[slot * 10 + k] = 0.0;
        }
        cnt++;
    }
    *done = cnt;
    free(e);
    free(fr);
    return SAD_OK;
}

/* bpp_target_count (budget.cpp:307-310) */
int sado_bpp_target_count(double bpp, int w, int h, uint64_t* out) {
    if (bpp < 0 || w < 1 || h < 1) return fail(SAD_EINVAL, "bpp target: bad inputs");
    *out = (uint64_t)(bpp * (double)w * h / 128.0);
    return SAD_OK;
}

/* simulate_schedule (budget.cpp:312-332) */
int sado_simulate_schedule(int n0, double scale, const sad_train_config* c, int* out) {
    int n = n0;
    for (int t = 1; t <= c->iters; t++) {
        int ev_d = t >= c->densify_start && t <= c->densify_end && t % c->densify_every == 0;
        int ev_p = t >= c->prune_start && t <= c->prune_end && t % c->prune_every == 0;
        if (ev_p && !c->prune_during_densify && t <= c->densify_end) ev_p = 0;
        if (ev_p) {
            int p = (int)(n * c->prune_pct * scale);
            if (p >= n) p = n - 1;
            if (p > 0) n -= p;
        }
        if (ev_d) {
            int d = (int)(n * c->densify_pct * scale);
            if (c->max_sites > 0 && (size_t)(n + d) > c->max_sites) d = (int)c->max_sites - n;
            if (d > 0) n += d;
        }
    }
    *out = n;
    return SAD_OK;
}

/* plan_schedule (budget.cpp:334-374) */
int sado_plan_schedule(int n0, uint64_t target, const sad_train_config* c, double* out) {
    double cap = c->budget_scale_cap, tgt = (double)target;
    int mnf = n0, mxf = n0;
#define MISS(S, M)                                  \
    do {                                            \
        int fin;                                    \
        sado_simulate_schedule(n0, (S), c, &fin);   \
        if (fin < mnf) mnf = fin;                   \
        if (fin > mxf) mxf = fin;                   \
        (M) = fabs((double)fin - tgt);              \
    } while (0)
    double best_s = 0, best_m, m;
    MISS(0.0, best_m);
    for (int i = 1; i <= 96; i++) {
        double sc = cap * i / 96;
        MISS(sc, m);
        if (m < best_m) {
            best_m = m;
            best_s = sc;
        }
    }
    double lo = mx(0.0, best_s - cap / 96), hi = mn(cap, best_s + cap / 96);
    for (int i = 0; i <= 256; i++) {
        double sc = lo + (hi - lo) * i / 256;
        MISS(sc, m);
        if (m < best_m) {
            best_m = m;
            best_s = sc;
        }
    }
#undef MISS
    *out = (tgt < mnf || tgt > mxf) ? cap : best_s;
    return SAD_OK;
}

/* ------------------------------------------------------------------ quality.cpp:68-73 */
double sado_psnr_from_loss(double loss) {
    double m = loss / 3.0;
    if (m <= 0) return 99.0;
    double v = 10.0 * log10(1.0 / m);
    return v > 99.0 ? 99.0 : v;
}

/* ------------------------------------------------------------------ TrainConfig defaults / validate */
void sado_default_config(sad_train_config* c) {
    memset(c, 0, sizeof *c);
    c->iters = 4000; c->seed = 1; c->k = 8; c->inject = 4; c->lambda_init = 0.3;
    c->lr_pos = 0.5; c->lr_color = 0.05; c->lr_log_tau = 0.05; c->lr_radius = 0.25;
    c->lr_dir = 0.025; c->lr_aniso = 0.025;
    c->beta1 = 0.9; c->beta2 = 0.999; c->adam_eps = 1e-8;
    c->refresh_every = 1; c->refresh_passes = 1; c->final_passes = 16;
    c->densify_every = 20; c->densify_start = 20; c->densify_end = 3000;
    c->densify_pct = 0.01; c->alpha = 0.7; c->stats_eps = 1e-8;
    c->prune_every = 40; c->prune_start = 100; c->prune_end = 3000; c->prune_pct = 0.033;
    c->prune_during_densify = 1; c->budget_scale_cap = 0.95;
    c->init_log_tau = 7.5; c->log_tau_min = 2.0; c->log_tau_max = 20.0;
    c->radius_min = 1.0; c->radius_max = 512.0; c->aniso_min = -2.0; c->aniso_max = 2.0;
    c->clamp_color = 1; c->fp64 = 1; c->threads = 1;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* TrainConfig::validate (types.cpp:103-126) */
static int validate(sad_train_config* c, int w, int h) {
    if (w < 1 || h < 1) return fail(SAD_EINVAL, "config: empty image");
    if (c->iters < 0) return fail(SAD_EINVAL, "config: negative iters");
    if (c->k < 1 || c->k > 16) return fail(SAD_EINVAL, "config: k out of [1,16]");
    if (c->inject < 0) return fail(SAD_EINVAL, "config: negative inject");
    if (c->lambda_init < 0 || c->lambda_init > 1) return fail(SAD_EINVAL, "config: lambda_init out of [0,1]");
    if (c->densify_every < 1 || c->prune_every < 1) return fail(SAD_EINVAL, "config: event period < 1");
    if (c->densify_pct < 0 || c->densify_pct > 1 || c->prune_pct < 0 || c->prune_pct > 1)
        return fail(SAD_EINVAL, "config: percentile out of [0,1]");
    if (c->refresh_every < 1) return fail(SAD_EINVAL, "config: refresh period < 1");
    if (c->refresh_passes < 0 || c->final_passes < 0) return fail(SAD_EINVAL, "config: negative passes");
    if (c->target_bpp < 0) return fail(SAD_EINVAL, "config: negative bpp");
    if (c->n_sites < 0) return fail(SAD_EINVAL, "config: negative site count");
    if (c->log_tau_min > c->log_tau_max || c->radius_min > c->radius_max || c->aniso_min > c->aniso_max)
        return fail(SAD_EINVAL, "config: inverted clamp range");
    if (c->threads < 1) c->threads = 1;
    c->densify_start = clampi(c->densify_start, 0, c->iters);
    c->densify_end = clampi(c->densify_end, 0, c->iters);
    c->prune_start = clampi(c->prune_start, 0, c->iters);
    c->prune_end = clampi(c->prune_end, 0, c->iters);
    if (c->densify_end < c->densify_start || c->prune_end < c->prune_start)
        return fail(SAD_EINVAL, "config: inverted schedule window");
    return SAD_OK;
}

/* ------------------------------------------------------------------ fit (train.cpp:221-311) */
static int initial_count(const sad_train_config* c, int w, int h, int* n) {
    *n = c->n_sites;
    if (*n == 0 && c->target_bpp > 0) {
        uint64_t want;
        sado_bpp_target_count(c->target_bpp, w, h, &want);
        if (want < 1) return fail(SAD_EINVAL, "fit: bpp target below one site");
        size_t n0 = (size_t)ceil((double)want * 1.6), cap = (size_t)w * h;
        *n = (int)(n0 < cap ? n0 : cap);
    }
    if (*n < 1) return fail(SAD_EINVAL, "fit: site count unset");
    return SAD_OK;
}

/* Upper bound on SiteStore::size over a fit: every densify event may append at most
 * floor(active * pct * scale) <= floor(size * pct) slots (budget.cpp:230, 277). */
int sado_fit_capacity(int w, int h, const sad_train_config* cfg, size_t n_init, size_t* cap) {
    sad_train_config c = *cfg;
    int rc = validate(&c, w, h);
    if (rc) return rc;
    size_t n = n_init;
    if (n == 0) {
        int n0;
        if ((rc = initial_count(&c, w, h, &n0))) return rc;
        n = (size_t)n0;
    }
    if (c.target_bpp > 0)
        for (int t = 1; t <= c.iters; t++)
            if (t >= c.densify_start && t <= c.densify_end && t % c.densify_every == 0)
                n += (size_t)((double)n * c.densify_pct);
    *cap = n;
    return SAD_OK;
}

int sado_fit(const double* tgt, int w, int h, const sad_train_config* cfg, const sad_sites_view* init,
             sad_sites_view* st, sad_field_view* f, sad_history_row* hist, double* sched) {
    sad_train_config c = *cfg;
    int rc = validate(&c, w, h);
    if (rc) return rc;
    if (init) {
        if (init->size > st->capacity) return fail(SAD_ENOMEM, "sites capacity");
        st->size = init->size;
        memcpy(st->x, init->x, 8 * init->size); memcpy(st->y, init->y, 8 * init->size);
        memcpy(st->log_tau, init->log_tau, 8 * init->size); memcpy(st->radius, init->radius, 8 * init->size);
        memcpy(st->col_r, init->col_r, 8 * init->size); memcpy(st->col_g, init->col_g, 8 * init->size);
        memcpy(st->col_b, init->col_b, 8 * init->size); memcpy(st->dir_x, init->dir_x, 8 * init->size);
        memcpy(st->dir_y, init->dir_y, 8 * init->size); memcpy(st->aniso, init->aniso, 8 * init->size);
        memcpy(st->active, init->active, init->size); memcpy(st->frozen, init->frozen, init->size);
        st->generation = init->generation;
    } else {
        int n;
        if ((rc = initial_count(&c, w, h, &n))) return rc;
        if ((rc = sado_init_sites(st, tgt, w, h, n, &c))) return rc;
    }
    int fp64 = c.fp64;
    int budget = c.target_bpp > 0;
    double scale = 1.0;
    *sched = 0;
    if (budget) {
        uint64_t want;
        sado_bpp_target_count(c.target_bpp, w, h, &want);
        uint32_t na;
        free(active_list(st, &na));
        sado_plan_schedule((int)na, want, &c, &scale);
        *sched = scale;
    }
    sad_adam_view ad;
    ad.capacity = st->capacity;
    ad.sites = st->size;
    ad.m = (double*)calloc(ad.capacity * 10 + 1, 8);
    ad.v = (double*)calloc(ad.capacity * 10 + 1, 8);
    ad.t = 0;
    ad.skipped = 0;
    double* gb = (double*)malloc(8 * (st->capacity * 11 + 1));
    double* stats = (double*)malloc(8 * (st->capacity * 8 + 1));
    if ((rc = sado_refresh(st, f, SAD_REFRESH_FULL, 4, c.inject, c.seed, fp64))) goto done;
    for (int t = 1; t <= c.iters; t++) {
        if ((t - 1) % c.refresh_every == 0)
            if ((rc = sado_refresh(st, f, SAD_REFRESH_WARM, c.refresh_passes, c.inject, c.seed, fp64))) goto done;
        double loss;
        uint64_t nf;
        if ((rc = sado_backward_image(st, f, tgt, fp64, 0, gb, &nf, &loss))) goto done;
        if (!isfinite(loss)) {
            rc = fail(SAD_ENUMERIC, "fit: non-finite loss");
            goto done;
        }
        if (c.tau_diffusion_lambda > 0)
            if ((rc = sado_tau_diffusion(st, f, c.tau_diffusion_lambda, gb))) goto done;
        int ev_d = budget && t >= c.densify_start && t <= c.densify_end && t % c.densify_every == 0;
        int ev_p = budget && t >= c.prune_start && t <= c.prune_end && t % c.prune_every == 0;
        if (ev_p && !c.prune_during_densify && t <= c.densify_end) ev_p = 0;
        uint64_t valid = 0;
        if (ev_d || ev_p)
            if ((rc = sado_accumulate_stats(st, f, tgt, stats, &valid))) goto done;
        sado_adam_step(st, gb, &ad, w, h, &c);
        int cnt;
        if (ev_p) sado_prune(st, stats, valid, c.prune_pct * scale, &cnt);
        if (ev_d)
            if ((rc = sado_densify(st, &ad, stats, tgt, w, h, c.densify_pct * scale, &c, &cnt))) goto done;
        if (ev_d || ev_p) {
            for (size_t r = ad.sites * 10; r < st->size * 10; r++) ad.m[r] = ad.v[r] = 0.0;
            ad.sites = st->size;
            if ((rc = sado_refresh(st, f, SAD_REFRESH_FULL, 4, c.inject, c.seed, fp64))) goto done;
        } else {
            f->synced_generation = st->generation;
        }
        uint32_t na;
        free(active_list(st, &na));
        hist[t - 1].iter = t;
        hist[t - 1].loss = loss;
        hist[t - 1].psnr = sado_psnr_from_loss(loss);
        hist[t - 1].active_sites = (int)na;
        hist[t - 1].ms = 0;
    }
    rc = sado_refresh(st, f, SAD_REFRESH_FULL, c.final_passes, c.inject, c.seed, fp64);
done:
    free(ad.m);
    free(ad.v);
    free(gb);
    free(stats);
    return rc;
}

/* ------------------------------------------------------------------ codec.cpp (decode path) */
static double cclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static uint32_t un_enc(double v, double lo, double sc, uint32_t mx) {
    return (uint32_t)lround(cclamp((v - lo) / sc, 0.0, 1.0) * mx);
}
static double un_dec(uint32_t c, double lo, double sc, uint32_t mx) { return lo + ((double)c / mx) * sc; }
static void le32w(uint8_t* p, uint32_t v) { for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i)); }
static uint32_t le32r(const uint8_t* p) { return p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24); }
static void f32w(uint8_t* p, double v) { float f = (float)v; uint32_t u; memcpy(&u, &f, 4); le32w(p, u); }
static double f32r(const uint8_t* p) { uint32_t u = le32r(p); float f; memcpy(&f, &u, 4); return f; }

/* compute_ranges (codec.cpp:53-88) */
static void cover(double lo, double hi, double* mn_o, double* sc_o) {
    float mn = (float)lo;
    if ((double)mn > lo) mn = nextafterf(mn, -INFINITY);
    double span = hi - (double)mn;
    float sc = (float)(span < 1e-6 ? 1e-6 : span);
    while ((double)mn + (double)sc < hi) sc = nextafterf(sc, INFINITY);
    *mn_o = mn;
    *sc_o = sc;
}

/* write_file (codec.cpp:147-177) into memory */
int sado_encode(const sad_sites_view* s, int w, int h, uint8_t* out, size_t cap, size_t* nbytes) {
    if (w < 1 || h < 1) return fail(SAD_EINVAL, "write: empty extent");
    size_t cnt = 0;
    for (size_t i = 0; i < s->size; i++) cnt += s->active[i] != 0;
    *nbytes = 58 + 16 * cnt;
    if (!out) return SAD_OK;
    if (cap < *nbytes) return fail(SAD_ENOMEM, "encode: buffer too small");
    double q[10] = {0, 1e-6, 0, 1e-6, 0, 0, 0, 1e-6, 1e-6, 1e-6}; /* lt min/scale, r min/scale, cmin[3], cscale[3] */
    double lo[5], hi[5];
    int any = 0;
    for (size_t i = 0; i < s->size; i++) {
        if (!s->active[i]) continue;
        double v[5] = {s->log_tau[i], s->radius[i], s->col_r[i], s->col_g[i], s->col_b[i]};
        for (int k = 0; k < 5; k++) {
            if (!any) lo[k] = hi[k] = v[k];
            else { if (v[k] < lo[k]) lo[k] = v[k]; if (hi[k] < v[k]) hi[k] = v[k]; }
        }
        any = 1;
    }
    if (any) {
        cover(lo[0], hi[0], &q[0], &q[1]);
        cover(lo[1], hi[1], &q[2], &q[3]);
        for (int c = 0; c < 3; c++) cover(lo[2 + c], hi[2 + c], &q[4 + c], &q[7 + c]);
    }
    memcpy(out, "SADF", 4);
    out[4] = 1; out[5] = 0;
    le32w(out + 6, (uint32_t)w); le32w(out + 10, (uint32_t)h); le32w(out + 14, (uint32_t)cnt);
    for (int k = 0; k < 10; k++) f32w(out + 18 + 4 * k, q[k]);
    double wd = w > 1 ? w - 1.0 : 1.0, hd = h > 1 ? h - 1.0 : 1.0;
    uint8_t* r = out + 58;
    for (size_t i = 0; i < s->size; i++) {
        if (!s->active[i]) continue;
        le32w(r, un_enc(s->x[i], 0, wd, 32767) | (un_enc(s->y[i], 0, hd, 32767) << 15) | (1u << 31));
        le32w(r + 4, un_enc(s->col_r[i], q[4], q[7], 2047) | (un_enc(s->col_g[i], q[5], q[8], 2047) << 11) |
                         (un_enc(s->col_b[i], q[6], q[9], 1023) << 22));
        le32w(r + 8, un_enc(s->log_tau[i], q[0], q[1], 65535) | (un_enc(s->radius[i], q[2], q[3], 65535) << 16));
        double ang = atan2(s->dir_y[i], s->dir_x[i]);
        le32w(r + 12, un_enc(ang, -3.14159265358979323846, 2.0 * 3.14159265358979323846, 65535) |
                          ((uint32_t)sado_float_to_half((float)s->aniso[i]) << 16));
        r += 16;
    }
    return SAD_OK;
}

/* read_file + unpack_site (codec.cpp:115-140, 179-222) */
int sado_decode(const uint8_t* b, size_t n, sad_sites_view* s, int* w, int* h) {
    char msg[96];
    if (n < 18) { snprintf(msg, sizeof msg, "file truncated at byte %zu, need %zu", n, (size_t)18); return fail(SAD_EFORMAT, msg); }
    if (memcmp(b, "SADF", 4)) return fail(SAD_EFORMAT, "bad magic, not a site file");
    if ((b[4] | (b[5] << 8)) != 1) return fail(SAD_EFORMAT, "unknown format version");
    uint32_t ww = le32r(b + 6), hh = le32r(b + 10), cnt = le32r(b + 14);
    if (ww < 1 || hh < 1 || ww > (1u << 24) || hh > (1u << 24)) return fail(SAD_EFORMAT, "unreasonable image extent in header");
    size_t need = 58 + 16 * (size_t)cnt;
    if (n != need) { snprintf(msg, sizeof msg, "file truncated at byte %zu, need %zu", n, need); return fail(SAD_EFORMAT, msg); }
    if (s->capacity < cnt) return fail(SAD_ENOMEM, "decode: capacity");
    double q[10];
    for (int k = 0; k < 10; k++) q[k] = f32r(b + 18 + 4 * k);
    *w = (int)ww; *h = (int)hh;
    double wd = ww > 1 ? ww - 1.0 : 1.0, hd = hh > 1 ? hh - 1.0 : 1.0;
    for (uint32_t i = 0; i < cnt; i++) {
        const uint8_t* r = b + 58 + 16 * (size_t)i;
        uint32_t w0 = le32r(r), w1 = le32r(r + 4), w2 = le32r(r + 8), w3 = le32r(r + 12);
        site_t p = {0, 0, 7.5, 1.0, 0, 0, 0, 1.0, 0, 0, 1, 0};
        if (!(w0 >> 31)) {
            p.active = 0; p.x = -1.0; p.y = -1.0;
        } else {
            p.x = un_dec(w0 & 0x7fffu, 0, wd, 32767);
            p.y = un_dec((w0 >> 15) & 0x7fffu, 0, hd, 32767);
            p.cr = cclamp(un_dec(w1 & 0x7ffu, q[4], q[7], 2047), 0, 1);
            p.cg = cclamp(un_dec((w1 >> 11) & 0x7ffu, q[5], q[8], 2047), 0, 1);
            p.cb = cclamp(un_dec(w1 >> 22, q[6], q[9], 1023), 0, 1);
            p.log_tau = un_dec(w2 & 0xffffu, q[0], q[1], 65535);
            p.radius = un_dec(w2 >> 16, q[2], q[3], 65535);
            double ang = un_dec(w3 & 0xffffu, -3.14159265358979323846, 2.0 * 3.14159265358979323846, 65535);
            p.dx = cos(ang); p.dy = sin(ang);
            p.aniso = (double)sado_half_to_float((uint16_t)(w3 >> 16));
        }
        site_set(s, i, &p);
    }
    s->size = cnt;
    return SAD_OK;
}
