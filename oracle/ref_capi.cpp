// ref_capi.cpp — TEST INFRASTRUCTURE ONLY (oracle). Never linked into the product.
//
// A C-ABI wrapper over the *unmodified* reference library compiled from /root/reference/proj/src
// (see oracle/Makefile).  It exposes the same host-view entry points as include/sad_b200.h with a
// `sadref_` prefix so the parity tests can run the reference and the CUDA path side by side on the
// same buffers.  The fit entry point is a replica of fit_impl (train.cpp:221-291) that pre-warms
// SiteStore::active_ids() single-threaded before every refresh: the reference's lazy cache races
// when threads > 1 (types.cpp:71-80 vs candidates.cpp:99); results are thread-count invariant
// (test_candidates.cpp:294-303), so the replica returns exactly what sad::fit returns.
#include "sad/budget.hpp"
#include "sad/codec.hpp"
#include "sad/candidates.hpp"
#include "sad/grad.hpp"
#include "sad/half.hpp"
#include "sad/quality.hpp"
#include "sad/render.hpp"
#include "sad/rng.hpp"
#include "sad/score.hpp"
#include "sad/train.hpp"

#include "../include/sad_b200.h"

#include <chrono>
#include <cstdio>
#include <unistd.h>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

using namespace sad;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
    g_err = what;
    return code;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return SAD_OK;
    } catch (const numeric_error& e) {
        return fail(SAD_ENUMERIC, e.what());
    } catch (const format_error& e) {
        return fail(SAD_EFORMAT, e.what());
    } catch (const std::invalid_argument& e) {
        std::string m = e.what();
        if (m.find("stale") != std::string::npos) return fail(SAD_ESTALE, e.what());
        if (m.find("empty candidate") != std::string::npos) return fail(SAD_EEMPTY, e.what());
        return fail(SAD_EINVAL, e.what());
    } catch (const std::exception& e) {
        return fail(SAD_EINVAL, e.what());
    }
}

SiteStore to_store(const sad_sites_view* v) {
    SiteStore st;
    size_t n = v->size;
    st.x.assign(v->x, v->x + n);
    st.y.assign(v->y, v->y + n);
    st.log_tau.assign(v->log_tau, v->log_tau + n);
    st.radius.assign(v->radius, v->radius + n);
    st.col_r.assign(v->col_r, v->col_r + n);
    st.col_g.assign(v->col_g, v->col_g + n);
    st.col_b.assign(v->col_b, v->col_b + n);
    st.dir_x.assign(v->dir_x, v->dir_x + n);
    st.dir_y.assign(v->dir_y, v->dir_y + n);
    st.aniso.assign(v->aniso, v->aniso + n);
    st.active.assign(v->active, v->active + n);
    st.frozen.assign(v->frozen, v->frozen + n);
    st.generation = v->generation;
    return st;
}

int from_store(const SiteStore& st, sad_sites_view* v) {
    size_t n = st.size();
    if (n > v->capacity) return fail(SAD_ENOMEM, "sites view capacity too small");
    auto cp = [n](double* dst, const std::vector<double>& s) { std::memcpy(dst, s.data(), n * 8); };
    cp(v->x, st.x); cp(v->y, st.y); cp(v->log_tau, st.log_tau); cp(v->radius, st.radius);
    cp(v->col_r, st.col_r); cp(v->col_g, st.col_g); cp(v->col_b, st.col_b);
    cp(v->dir_x, st.dir_x); cp(v->dir_y, st.dir_y); cp(v->aniso, st.aniso);
    std::memcpy(v->active, st.active.data(), n);
    std::memcpy(v->frozen, st.frozen.data(), n);
    v->size = n;
    v->generation = st.generation;
    return SAD_OK;
}

CandidateField to_field(const sad_field_view* f) {
    CandidateField c;
    c.resize(f->width, f->height, f->k, f->cell);
    std::memcpy(c.ids.data(), f->ids, c.ids.size() * 4);
    c.synced_generation = f->synced_generation;
    c.refresh_count = f->refresh_count;
    c.pass_index = f->pass_index;
    return c;
}

void from_field(const CandidateField& c, sad_field_view* f) {
    f->width = c.width; f->height = c.height; f->cell = c.cell;
    f->gw = c.gw; f->gh = c.gh; f->k = c.k;
    std::memcpy(f->ids, c.ids.data(), c.ids.size() * 4);
    f->synced_generation = c.synced_generation;
    f->refresh_count = c.refresh_count;
    f->pass_index = c.pass_index;
}

ImageBuffer to_image(const double* rgb, int w, int h) {
    ImageBuffer img;
    img.resize(w, h);
    std::memcpy(img.data.data(), rgb, img.data.size() * 8);
    return img;
}

TrainConfig to_cfg(const sad_train_config* c) {
    TrainConfig t;
    t.iters = c->iters; t.n_sites = c->n_sites; t.target_bpp = c->target_bpp; t.seed = c->seed;
    t.k = c->k; t.inject = c->inject; t.lambda_init = c->lambda_init;
    t.lr.pos = c->lr_pos; t.lr.color = c->lr_color; t.lr.log_tau = c->lr_log_tau;
    t.lr.radius = c->lr_radius; t.lr.dir = c->lr_dir; t.lr.aniso = c->lr_aniso;
    t.beta1 = c->beta1; t.beta2 = c->beta2; t.adam_eps = c->adam_eps;
    t.refresh_every = c->refresh_every; t.refresh_passes = c->refresh_passes;
    t.final_passes = c->final_passes; t.tau_diffusion_lambda = c->tau_diffusion_lambda;
    t.densify_every = c->densify_every; t.densify_start = c->densify_start;
    t.densify_end = c->densify_end; t.densify_pct = c->densify_pct; t.alpha = c->alpha;
    t.stats_eps = c->stats_eps; t.prune_every = c->prune_every; t.prune_start = c->prune_start;
    t.prune_end = c->prune_end; t.prune_pct = c->prune_pct;
    t.prune_during_densify = c->prune_during_densify != 0;
    t.budget_scale_cap = c->budget_scale_cap; t.max_sites = c->max_sites;
    t.init_log_tau = c->init_log_tau; t.init_radius = c->init_radius; t.init_aniso = c->init_aniso;
    t.log_tau_min = c->log_tau_min; t.log_tau_max = c->log_tau_max;
    t.radius_min = c->radius_min; t.radius_max = c->radius_max;
    t.aniso_min = c->aniso_min; t.aniso_max = c->aniso_max;
    t.clamp_color = c->clamp_color != 0; t.fp64 = c->fp64 != 0; t.threads = c->threads;
    return t;
}

struct RefFit {
    FitResult res;
    double seconds = 0;
    double phase[8] = {0};
};

// fit_impl replica (train.cpp:221-291) with single-threaded active_ids() pre-warm and phase timers.
FitResult fit_replica(SiteStore st, const ImageBuffer& target, TrainConfig cfg, double* phase) {
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a) {
        return std::chrono::duration<double, std::milli>(clk::now() - a).count();
    };
    const int kEventRefreshPasses = 4;
    int w = target.width, h = target.height;
    cfg.validate(w, h);
    RunOpts opts = run_opts(cfg);
    bool budget_on = cfg.target_bpp > 0;
    FitResult out;
    double scale = 1.0;
    if (budget_on) {
        size_t want = bpp_target_count(cfg.target_bpp, w, h);
        scale = plan_schedule(static_cast<int>(st.active_count()), want, cfg);
        out.schedule_scale = scale;
    }
    AdamState adam;
    adam.resize(st.size());
    CandidateField field;
    field.resize(w, h, cfg.k);
    st.active_ids();
    auto t0 = clk::now();
    refresh(st, field, RefreshMode::Full, kEventRefreshPasses, cfg.inject, cfg.seed, opts);
    phase[4] += ms(t0);
    GradBuffer gb;
    // SAD_REF_STOP_AT=t (divergence hunting): stop after iteration t, keep the field as it is then
    const char* stop_env = std::getenv("SAD_REF_STOP_AT");
    const int stop_at = stop_env ? std::atoi(stop_env) : 0;
    for (int t = 1; t <= cfg.iters; t++) {
        auto tick = clk::now();
        if ((t - 1) % cfg.refresh_every == 0) {
            st.active_ids();
            auto a = clk::now();
            refresh(st, field, RefreshMode::WarmStart, cfg.refresh_passes, cfg.inject, cfg.seed, opts);
            phase[0] += ms(a);
        }
        auto b = clk::now();
        double loss = backward_image(st, field, target, gb, opts, false);
        phase[1] += ms(b);
        if (!std::isfinite(loss)) throw numeric_error("fit: non-finite loss");
        if (cfg.tau_diffusion_lambda > 0) tau_diffusion(st, field, cfg.tau_diffusion_lambda, gb, opts);
        bool ev_d = budget_on && t >= cfg.densify_start && t <= cfg.densify_end &&
                    t % cfg.densify_every == 0;
        bool ev_p = budget_on && t >= cfg.prune_start && t <= cfg.prune_end &&
                    t % cfg.prune_every == 0;
        if (ev_p && !cfg.prune_during_densify && t <= cfg.densify_end) ev_p = false;
        StatsResult stats;
        auto c = clk::now();
        if (ev_d || ev_p) stats = accumulate_stats(st, field, target, opts);
        phase[3] += ms(c);
        auto d = clk::now();
        adam_step(st, gb, adam, w, h, cfg);
        phase[2] += ms(d);
        auto e = clk::now();
        if (ev_p) prune(st, stats, cfg.prune_pct * scale);
        if (ev_d) densify(st, adam, stats, target, cfg.densify_pct * scale, cfg);
        if (ev_d || ev_p) {
            adam.resize(st.size());
            st.active_ids();
            refresh(st, field, RefreshMode::Full, kEventRefreshPasses, cfg.inject, cfg.seed, opts);
        } else {
            field.synced_generation = st.generation;
        }
        phase[3] += ms(e);
        HistoryRow row;
        row.iter = t;
        row.loss = loss;
        row.psnr = psnr_from_loss(loss);
        row.active_sites = static_cast<int>(st.active_count());
        row.ms = ms(tick);
        out.history.push_back(row);
        if (stop_at == t) break;
    }
    st.active_ids();
    auto f = clk::now();
    if (!stop_at) refresh(st, field, RefreshMode::Full, cfg.final_passes, cfg.inject, cfg.seed, opts);
    phase[4] += ms(f);
    out.sites = std::move(st);
    out.field = std::move(field);
    return out;
}

} // namespace

extern "C" {

const char* sadref_last_error(void) { return g_err.c_str(); }

void sadref_default_config(sad_train_config* c) {
    TrainConfig t;
    std::memset(c, 0, sizeof(*c));
    c->iters = t.iters; c->n_sites = t.n_sites; c->target_bpp = t.target_bpp; c->seed = t.seed;
    c->k = t.k; c->inject = t.inject; c->lambda_init = t.lambda_init;
    c->lr_pos = t.lr.pos; c->lr_color = t.lr.color; c->lr_log_tau = t.lr.log_tau;
    c->lr_radius = t.lr.radius; c->lr_dir = t.lr.dir; c->lr_aniso = t.lr.aniso;
    c->beta1 = t.beta1; c->beta2 = t.beta2; c->adam_eps = t.adam_eps;
    c->refresh_every = t.refresh_every; c->refresh_passes = t.refresh_passes;
    c->final_passes = t.final_passes; c->tau_diffusion_lambda = t.tau_diffusion_lambda;
    c->densify_every = t.densify_every; c->densify_start = t.densify_start;
    c->densify_end = t.densify_end; c->densify_pct = t.densify_pct; c->alpha = t.alpha;
    c->stats_eps = t.stats_eps; c->prune_every = t.prune_every; c->prune_start = t.prune_start;
    c->prune_end = t.prune_end; c->prune_pct = t.prune_pct;
    c->prune_during_densify = t.prune_during_densify; c->budget_scale_cap = t.budget_scale_cap;
    c->max_sites = t.max_sites; c->init_log_tau = t.init_log_tau; c->init_radius = t.init_radius;
    c->init_aniso = t.init_aniso; c->log_tau_min = t.log_tau_min; c->log_tau_max = t.log_tau_max;
    c->radius_min = t.radius_min; c->radius_max = t.radius_max; c->aniso_min = t.aniso_min;
    c->aniso_max = t.aniso_max; c->clamp_color = t.clamp_color; c->fp64 = t.fp64;
    c->threads = t.threads;
}

// ---- core helpers exposed for golden-vector generation
uint32_t sadref_seeded_state(uint64_t seed, uint32_t a, uint32_t b) { return seeded_stream(seed, a, b).s; }
uint16_t sadref_float_to_half(float f) { return float_to_half(f); }
float sadref_half_to_float(uint16_t h) { return half_to_float(h); }
double sadref_psnr_from_loss(double loss) { return psnr_from_loss(loss); }

int sadref_jump_step(uint32_t t, uint32_t b, uint32_t* out) {
    return guard([&] { *out = jump_step(t, b); });
}

int sadref_full_refresh_passes(int gw, int gh, int extra, sad_pass_spec* out, int* n) {
    return guard([&] {
        auto seq = full_refresh_passes(gw, gh, extra);
        if (static_cast<int>(seq.size()) > *n) throw std::invalid_argument("pass buffer too small");
        for (size_t i = 0; i < seq.size(); i++)
            out[i] = {seq[i].step, seq[i].stencil == Stencil::Box3 ? 1 : 0};
        *n = static_cast<int>(seq.size());
    });
}

int sadref_jfa_seed(const sad_sites_view* sv, sad_field_view* fv) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        jfa_seed(st, f);
        from_field(f, fv);
    });
}

int sadref_run_passes(const sad_sites_view* sv, sad_field_view* fv, const sad_pass_spec* seq,
                      int n_pass, int inject, uint64_t seed, int fp64, int threads) {
    return guard([&] {
        SiteStore st = to_store(sv);
        st.active_ids();
        CandidateField f = to_field(fv);
        std::vector<PassSpec> v;
        for (int i = 0; i < n_pass; i++)
            v.push_back({seq[i].step, seq[i].stencil ? Stencil::Box3 : Stencil::Axial});
        run_passes(st, f, v, inject, seed, RunOpts{fp64 != 0, threads});
        from_field(f, fv);
    });
}

int sadref_refresh(const sad_sites_view* sv, sad_field_view* fv, int mode, int passes, int inject,
                   uint64_t seed, int fp64, int threads) {
    return guard([&] {
        SiteStore st = to_store(sv);
        st.active_ids();
        CandidateField f = to_field(fv);
        refresh(st, f, mode == SAD_REFRESH_FULL ? RefreshMode::Full : RefreshMode::WarmStart, passes,
                inject, seed, RunOpts{fp64 != 0, threads});
        from_field(f, fv);
    });
}

int sadref_exact_topk_batch(const sad_sites_view* sv, const int32_t* xy, size_t n, int k,
                            double scale, int fp64, uint32_t* out) {
    return guard([&] {
        SiteStore st = to_store(sv);
        std::vector<std::pair<int, int>> px;
        for (size_t i = 0; i < n; i++) px.push_back({xy[2 * i], xy[2 * i + 1]});
        auto res = exact_topk_batch(st, px, k, scale, fp64 != 0);
        for (size_t i = 0; i < n; i++)
            for (int j = 0; j < k; j++)
                out[i * k + j] = j < static_cast<int>(res[i].size()) ? res[i][j] : SAD_EMPTY_ID;
    });
}

int sadref_render_image(const sad_sites_view* sv, const sad_field_view* fv, int fp64, int threads,
                        double* out) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        ImageBuffer img = render_image(st, f, RunOpts{fp64 != 0, threads});
        std::memcpy(out, img.data.data(), img.data.size() * 8);
    });
}

int sadref_pixel_weights(const sad_sites_view* sv, const sad_field_view* fv, const int32_t* xy,
                         size_t n_q, uint32_t* ids, double* w, int32_t* n) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        for (size_t q = 0; q < n_q; q++) {
            PixelMix m = pixel_weights(st, f, xy[2 * q], xy[2 * q + 1]);
            n[q] = m.n;
            for (int i = 0; i < 16; i++) {
                ids[q * 16 + i] = i < m.n ? m.ids[i] : SAD_EMPTY_ID;
                w[q * 16 + i] = i < m.n ? m.w[i] : 0.0;
            }
        }
    });
}

int sadref_render_id_map(const sad_sites_view* sv, const sad_field_view* fv, uint32_t* out) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        auto m = render_id_map(st, f);
        std::memcpy(out, m.data(), m.size() * 4);
    });
}

static void grads_out(const GradBuffer& gb, size_t n, double* grads) {
    for (size_t id = 0; id < n; id++) {
        for (int s = 0; s < kGradSlots; s++) grads[id * 11 + s] = gb.grad(s, static_cast<uint32_t>(id));
        grads[id * 11 + 10] = gb.removal_delta(static_cast<uint32_t>(id));
    }
}

int sadref_backward_image(const sad_sites_view* sv, const sad_field_view* fv, const double* tgt,
                          int fp64, int with_removal, int threads, double* grads,
                          uint64_t* nonfinite, double* loss) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        ImageBuffer t = to_image(tgt, f.width, f.height);
        GradBuffer gb;
        *loss = backward_image(st, f, t, gb, RunOpts{fp64 != 0, threads}, with_removal != 0);
        grads_out(gb, st.size(), grads);
        *nonfinite = gb.nonfinite;
    });
}

int sadref_tau_diffusion(const sad_sites_view* sv, const sad_field_view* fv, double lambda, double* grads) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        size_t n = st.size();
        GradBuffer gb;
        gb.resize(n);
        for (size_t id = 0; id < n; id++)
            for (int s = 0; s < kChannels; s++) {
                Accum a;
                a.add(grads[id * 11 + s]);
                gb.at(s, static_cast<uint32_t>(id)) = a;
            }
        tau_diffusion(st, f, lambda, gb, RunOpts{});
        grads_out(gb, n, grads);
    });
}

int sadref_image_loss(const sad_sites_view* sv, const sad_field_view* fv, const double* tgt, int fp64,
                      double* loss) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        ImageBuffer t = to_image(tgt, f.width, f.height);
        *loss = image_loss(st, f, t, RunOpts{fp64 != 0, 1});
    });
}

int sadref_backward_pixel_grad(const sad_sites_view* sv, const sad_field_view* fv,
                               const double* dl, int dl_w, int dl_h, int fp64, double* grads, uint64_t* nonfinite) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        ImageBuffer t = to_image(dl, dl_w, dl_h);
        GradBuffer gb;
        backward_pixel_grad(st, f, t, gb, RunOpts{fp64 != 0, 1});
        grads_out(gb, st.size(), grads);
        *nonfinite = gb.nonfinite;
    });
}

int sadref_adam_step(sad_sites_view* sv, const double* grads, sad_adam_view* av, int w, int h,
                     const sad_train_config* c) {
    return guard([&] {
        SiteStore st = to_store(sv);
        size_t n = st.size();
        GradBuffer gb;
        gb.resize(n);
        for (size_t id = 0; id < n; id++)
            for (int s = 0; s < kChannels; s++) {
                Accum a;
                a.add(grads[id * 11 + s]);
                gb.at(s, static_cast<uint32_t>(id)) = a;
            }
        AdamState a;
        a.m.assign(av->m, av->m + av->sites * kGradSlots);
        a.v.assign(av->v, av->v + av->sites * kGradSlots);
        a.t = av->t;
        a.skipped = av->skipped;
        adam_step(st, gb, a, w, h, to_cfg(c));
        if (a.sites() > av->capacity) throw std::invalid_argument("adam capacity");
        std::memcpy(av->m, a.m.data(), a.m.size() * 8);
        std::memcpy(av->v, a.v.data(), a.v.size() * 8);
        av->sites = a.sites();
        av->t = a.t;
        av->skipped = a.skipped;
        if (from_store(st, sv)) throw std::invalid_argument(g_err);
    });
}

int sadref_clamp_project(sad_sites_view* sv, int w, int h, const sad_train_config* c) {
    return guard([&] {
        SiteStore st = to_store(sv);
        clamp_project(st, w, h, to_cfg(c));
        if (from_store(st, sv)) throw std::invalid_argument(g_err);
    });
}

int sadref_init_sites(sad_sites_view* sv, const double* tgt, int w, int h, int n,
                      const sad_train_config* c) {
    return guard([&] {
        SiteStore st;
        ImageBuffer t = to_image(tgt, w, h);
        init_sites(st, t, n, to_cfg(c));
        if (from_store(st, sv)) throw std::invalid_argument(g_err);
    });
}

int sadref_sobel_magnitude(const double* tgt, int w, int h, double* out) {
    return guard([&] {
        auto m = sobel_magnitude(to_image(tgt, w, h));
        std::memcpy(out, m.data(), m.size() * 8);
    });
}

static StatsResult stats_in(const double* s, uint64_t valid, size_t n) {
    StatsResult r;
    r.site.resize(n);
    for (size_t i = 0; i < n; i++) {
        const double* p = s + i * 8;
        r.site[i] = SiteStats{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7]};
    }
    r.valid_pixels = valid;
    return r;
}

int sadref_accumulate_stats(const sad_sites_view* sv, const sad_field_view* fv, const double* tgt,
                            int threads, double* stats, uint64_t* valid) {
    return guard([&] {
        SiteStore st = to_store(sv);
        CandidateField f = to_field(fv);
        ImageBuffer t = to_image(tgt, f.width, f.height);
        StatsResult r = accumulate_stats(st, f, t, RunOpts{true, threads});
        for (size_t i = 0; i < st.size(); i++) {
            const SiteStats& s = r.site[i];
            double row[8] = {s.mass, s.energy, s.sx, s.sy, s.sxx, s.sxy, s.syy, s.removal};
            std::memcpy(stats + i * 8, row, sizeof row);
        }
        *valid = r.valid_pixels;
    });
}

int sadref_prune(sad_sites_view* sv, const double* stats, uint64_t valid, double pct, int* removed) {
    return guard([&] {
        SiteStore st = to_store(sv);
        *removed = prune(st, stats_in(stats, valid, st.size()), pct);
        if (from_store(st, sv)) throw std::invalid_argument(g_err);
    });
}

int sadref_densify(sad_sites_view* sv, sad_adam_view* av, const double* stats, const double* tgt,
                   int w, int h, double pct, const sad_train_config* c, int* done) {
    return guard([&] {
        SiteStore st = to_store(sv);
        AdamState a;
        a.m.assign(av->m, av->m + av->sites * kGradSlots);
        a.v.assign(av->v, av->v + av->sites * kGradSlots);
        a.t = av->t;
        a.skipped = av->skipped;
        ImageBuffer t = to_image(tgt, w, h);
        *done = densify(st, a, stats_in(stats, 0, st.size()), t, pct, to_cfg(c));
        if (a.sites() > av->capacity) throw std::invalid_argument("adam capacity");
        std::memcpy(av->m, a.m.data(), a.m.size() * 8);
        std::memcpy(av->v, a.v.data(), a.v.size() * 8);
        av->sites = a.sites();
        if (from_store(st, sv)) throw std::invalid_argument(g_err);
    });
}

int sadref_bpp_target_count(double bpp, int w, int h, uint64_t* out) {
    return guard([&] { *out = bpp_target_count(bpp, w, h); });
}

int sadref_simulate_schedule(int n0, double scale, const sad_train_config* c, int* out) {
    return guard([&] {
        TrainConfig t = to_cfg(c);
        *out = simulate_schedule(n0, scale, t);
    });
}

int sadref_plan_schedule(int n0, uint64_t target, const sad_train_config* c, double* out) {
    return guard([&] {
        TrainConfig t = to_cfg(c);
        *out = plan_schedule(n0, target, t);
    });
}

double sadref_mse(const double* a, const double* b, int w, int h) {
    return mse(to_image(a, w, h), to_image(b, w, h));
}

// ---- codec (write_file / read_file go through a temporary file: the reference API is file based)
int sadref_encode(const sad_sites_view* sv, int w, int h, uint8_t* out, size_t cap, size_t* nbytes) {
    return guard([&] {
        SiteStore st = to_store(sv);
        char path[] = "/tmp/sadref_XXXXXX";
        int fd = mkstemp(path);
        if (fd < 0) throw std::runtime_error("mkstemp");
        close(fd);
        write_file(path, st, w, h);
        FILE* f = std::fopen(path, "rb");
        std::vector<uint8_t> b;
        int ch;
        while ((ch = std::fgetc(f)) != EOF) b.push_back(static_cast<uint8_t>(ch));
        std::fclose(f);
        std::remove(path);
        *nbytes = b.size();
        if (out) {
            if (cap < b.size()) throw std::invalid_argument("encode: buffer too small");
            std::memcpy(out, b.data(), b.size());
        }
    });
}

int sadref_decode(const uint8_t* buf, size_t n, sad_sites_view* sv, int* w, int* h) {
    return guard([&] {
        char path[] = "/tmp/sadref_XXXXXX";
        int fd = mkstemp(path);
        if (fd < 0) throw std::runtime_error("mkstemp");
        FILE* f = fdopen(fd, "wb");
        std::fwrite(buf, 1, n, f);
        std::fclose(f);
        try {
            DecodedFile d = read_file(path);
            std::remove(path);
            *w = d.width;
            *h = d.height;
            if (from_store(d.sites, sv)) throw std::invalid_argument(g_err);
        } catch (...) {
            std::remove(path);
            throw;
        }
    });
}

// ---- fit: always the pre-warmed fit_impl replica above (tests/cpp/compat_check pins it to the library sad::fit)
int sadref_fit(const double* tgt, int w, int h, const sad_train_config* c, const sad_sites_view* init,
               void** handle) {
    return guard([&] {
        auto* r = new RefFit();
        ImageBuffer t = to_image(tgt, w, h);
        TrainConfig cfg = to_cfg(c);
        auto t0 = std::chrono::steady_clock::now();
        if (init) {
            r->res = fit_replica(to_store(init), t, cfg, r->phase);
        } else {
            TrainConfig v = cfg;
            v.validate(w, h);
            int n = v.n_sites;
            if (n == 0 && v.target_bpp > 0) {
                size_t want = bpp_target_count(v.target_bpp, w, h);
                if (want < 1) throw std::invalid_argument("fit: bpp target below one site");
                size_t n0 = static_cast<size_t>(std::ceil(static_cast<double>(want) * 1.6));
                n = static_cast<int>(std::min(n0, static_cast<size_t>(w) * h));
            }
            if (n < 1) throw std::invalid_argument("fit: site count unset");
            SiteStore st;
            auto ti = std::chrono::steady_clock::now();
            init_sites(st, t, n, v);
            r->phase[5] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ti).count();
            r->res = fit_replica(std::move(st), t, cfg, r->phase);
        }
        r->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *handle = r;
    });
}

int sadref_fit_info(void* handle, size_t* n_sites, int* n_hist, double* scale, double* seconds,
                    double* phase8) {
    auto* r = static_cast<RefFit*>(handle);
    *n_sites = r->res.sites.size();
    *n_hist = static_cast<int>(r->res.history.size());
    *scale = r->res.schedule_scale;
    *seconds = r->seconds;
    if (phase8) std::memcpy(phase8, r->phase, sizeof r->phase);
    return SAD_OK;
}

int sadref_fit_download(void* handle, sad_sites_view* sv, sad_field_view* fv, sad_history_row* hist) {
    auto* r = static_cast<RefFit*>(handle);
    int rc = from_store(r->res.sites, sv);
    if (rc) return rc;
    from_field(r->res.field, fv);
    for (size_t i = 0; i < r->res.history.size(); i++) {
        const HistoryRow& h = r->res.history[i];
        hist[i] = {h.iter, h.loss, h.psnr, h.active_sites, h.ms};
    }
    return SAD_OK;
}

void sadref_fit_free(void* handle) { delete static_cast<RefFit*>(handle); }

} // extern "C"
