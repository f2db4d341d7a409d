// sad_b200_compat.hpp — drop-in C++ shim for code written against the reference library.
//
// Include this after the reference headers ("sad/types.hpp", ...) and link libsad_b200.so: every
// function below has the signature of the reference function it replaces (cited), takes the
// reference's own value types, and runs on the B200 through the C ABI (sad_b200.h).  Errors come
// back as the reference's exception types (std::invalid_argument, sad::numeric_error, ...).
//
//   sad::b200::Context gpu;                          // one per device/thread
//   sad::b200::refresh(gpu, st, field, sad::RefreshMode::Full, 4, 4, seed, opts);
//   double loss = sad::b200::backward_image(gpu, st, field, target, grads, opts, false);
//   sad::FitResult r = sad::b200::fit(gpu, target, cfg);
#pragma once
#include "sad/budget.hpp"
#include "sad/candidates.hpp"
#include "sad/grad.hpp"
#include "sad/render.hpp"
#include "sad/train.hpp"
#include "sad/types.hpp"
#include "sad_b200.h"

#include <stdexcept>
#include <string>
#include <cstring>
#include <vector>

namespace sad::b200 {

inline void check(sad_status rc) {
    if (rc == SAD_OK) return;
    std::string m = sad_last_error();
    switch (rc) {
    case SAD_ENUMERIC: throw sad::numeric_error(m);
    case SAD_EFORMAT: throw sad::format_error(m);
    case SAD_ECUDA:
    case SAD_ENOMEM: throw std::runtime_error(m);
    default: throw std::invalid_argument(m);
    }
}

class Context {
public:
    explicit Context(int device = 0, void* stream = nullptr) { check(sad_ctx_create(device, stream, &ctx_)); }
    ~Context() { sad_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    sad_ctx* get() const { return ctx_; }

private:
    sad_ctx* ctx_ = nullptr;
};

namespace detail {

// SiteStore (types.hpp:37-63) <-> sad_sites_view; `extra` reserves room for densify appends.
struct SitesView {
    sad_sites_view v{};
    std::vector<double> buf[10];
    std::vector<uint8_t> act, frz;
    SitesView(const SiteStore& st, size_t extra = 0) {
        size_t n = st.size(), cap = n + extra + 1;
        const std::vector<double>* src[10] = {&st.x, &st.y, &st.log_tau, &st.radius, &st.col_r,
                                              &st.col_g, &st.col_b, &st.dir_x, &st.dir_y, &st.aniso};
        double** dst[10] = {&v.x, &v.y, &v.log_tau, &v.radius, &v.col_r, &v.col_g, &v.col_b, &v.dir_x, &v.dir_y, &v.aniso};
        for (int k = 0; k < 10; k++) {
            buf[k].assign(cap, 0.0);
            std::copy(src[k]->begin(), src[k]->end(), buf[k].begin());
            *dst[k] = buf[k].data();
        }
        act.assign(cap, 0);
        frz.assign(cap, 0);
        std::copy(st.active.begin(), st.active.end(), act.begin());
        std::copy(st.frozen.begin(), st.frozen.end(), frz.begin());
        v.active = act.data();
        v.frozen = frz.data();
        v.size = n;
        v.capacity = cap;
        v.generation = st.generation;
    }
    void store_into(SiteStore& st) const {
        size_t n = v.size;
        std::vector<double>* dst[10] = {&st.x, &st.y, &st.log_tau, &st.radius, &st.col_r,
                                        &st.col_g, &st.col_b, &st.dir_x, &st.dir_y, &st.aniso};
        for (int k = 0; k < 10; k++) dst[k]->assign(buf[k].begin(), buf[k].begin() + n);
        st.active.assign(act.begin(), act.begin() + n);
        st.frozen.assign(frz.begin(), frz.begin() + n);
        st.generation = v.generation;
    }
};

inline sad_field_view field_view(const CandidateField& f) {
    sad_field_view v{};
    v.width = f.width;
    v.height = f.height;
    v.cell = f.cell;
    v.gw = f.gw;
    v.gh = f.gh;
    v.k = f.k;
    v.ids = const_cast<uint32_t*>(f.ids.data());
    v.synced_generation = f.synced_generation;
    v.refresh_count = f.refresh_count;
    v.pass_index = f.pass_index;
    return v;
}

inline void field_back(const sad_field_view& v, CandidateField& f) {
    f.synced_generation = v.synced_generation;
    f.refresh_count = v.refresh_count;
    f.pass_index = v.pass_index;
}

inline sad_train_config config(const TrainConfig& t) {
    sad_train_config c{};
    c.iters = t.iters; c.n_sites = t.n_sites; c.target_bpp = t.target_bpp; c.seed = t.seed;
    c.k = t.k; c.inject = t.inject; c.lambda_init = t.lambda_init;
    c.lr_pos = t.lr.pos; c.lr_color = t.lr.color; c.lr_log_tau = t.lr.log_tau;
    c.lr_radius = t.lr.radius; c.lr_dir = t.lr.dir; c.lr_aniso = t.lr.aniso;
    c.beta1 = t.beta1; c.beta2 = t.beta2; c.adam_eps = t.adam_eps;
    c.refresh_every = t.refresh_every; c.refresh_passes = t.refresh_passes; c.final_passes = t.final_passes;
    c.tau_diffusion_lambda = t.tau_diffusion_lambda;
    c.densify_every = t.densify_every; c.densify_start = t.densify_start; c.densify_end = t.densify_end;
    c.densify_pct = t.densify_pct; c.alpha = t.alpha; c.stats_eps = t.stats_eps;
    c.prune_every = t.prune_every; c.prune_start = t.prune_start; c.prune_end = t.prune_end;
    c.prune_pct = t.prune_pct; c.prune_during_densify = t.prune_during_densify;
    c.budget_scale_cap = t.budget_scale_cap; c.max_sites = t.max_sites;
    c.init_log_tau = t.init_log_tau; c.init_radius = t.init_radius; c.init_aniso = t.init_aniso;
    c.log_tau_min = t.log_tau_min; c.log_tau_max = t.log_tau_max; c.radius_min = t.radius_min;
    c.radius_max = t.radius_max; c.aniso_min = t.aniso_min; c.aniso_max = t.aniso_max;
    c.clamp_color = t.clamp_color; c.fp64 = t.fp64; c.threads = t.threads;
    return c;
}

}  // namespace detail

// jfa_seed (candidates.hpp:47)
inline void jfa_seed(Context& g, const SiteStore& st, CandidateField& f) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    check(sad_jfa_seed(g.get(), &s.v, &v));
    detail::field_back(v, f);
}

// run_passes / propagate_pass (candidates.hpp:55-60)
inline void run_passes(Context& g, const SiteStore& st, CandidateField& f, const std::vector<PassSpec>& seq,
                       int inject, uint64_t seed, const RunOpts& o) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    std::vector<sad_pass_spec> p;
    for (const PassSpec& ps : seq) p.push_back({ps.step, ps.stencil == Stencil::Box3 ? 1 : 0});
    check(sad_run_passes(g.get(), &s.v, &v, p.data(), static_cast<int>(p.size()), inject, seed, o.fp64));
    detail::field_back(v, f);
}

inline void propagate_pass(Context& g, const SiteStore& st, CandidateField& f, const PassSpec& pass, int inject,
                           uint64_t seed, const RunOpts& o) {
    run_passes(g, st, f, {pass}, inject, seed, o);
}

// refresh (candidates.hpp:67-68)
inline void refresh(Context& g, const SiteStore& st, CandidateField& f, RefreshMode mode, int passes, int inject,
                    uint64_t seed, const RunOpts& o) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    check(sad_refresh(g.get(), &s.v, &v, mode == RefreshMode::Full ? SAD_REFRESH_FULL : SAD_REFRESH_WARM, passes,
                      inject, seed, o.fp64));
    detail::field_back(v, f);
}

// exact_topk_batch / exact_topk (candidates.hpp:66-72) on the device brute force (k_exact_topk); probes
// are pixel centres (integers), as every caller of the reference passes
inline std::vector<std::vector<uint32_t>> exact_topk_batch(Context& g, const SiteStore& st,
                                                           const std::vector<std::pair<int, int>>& pixels, int k,
                                                           double scale, bool fp64 = true) {
    if (k < 1 || k > 16) throw std::invalid_argument("exact_topk: k out of range");
    detail::SitesView s(st);
    std::vector<int32_t> xy(2 * pixels.size() + 2);
    for (size_t i = 0; i < pixels.size(); i++) {
        xy[2 * i] = pixels[i].first;
        xy[2 * i + 1] = pixels[i].second;
    }
    std::vector<uint32_t> out(std::max<size_t>(pixels.size(), 1) * k, 0xffffffffu);
    check(sad_exact_topk_batch(g.get(), &s.v, xy.data(), pixels.size(), k, scale, fp64 ? 1 : 0, out.data()));
    std::vector<std::vector<uint32_t>> res(pixels.size());
    for (size_t i = 0; i < pixels.size(); i++)
        for (int j = 0; j < k && out[i * k + j] != 0xffffffffu; j++) res[i].push_back(out[i * k + j]);
    return res;
}

inline std::vector<uint32_t> exact_topk(Context& g, const SiteStore& st, double px, double py, int k, double scale,
                                        bool fp64 = true) {
    if (k < 1 || k > 16) throw std::invalid_argument("exact_topk: k out of range");
    const int ix = static_cast<int>(px), iy = static_cast<int>(py);
    if (ix != px || iy != py) throw std::invalid_argument("exact_topk: the device path takes pixel-centre probes");
    return exact_topk_batch(g, st, {{ix, iy}}, k, scale, fp64)[0];
}

// pixel_weights (render.hpp:18), one query through the batched device kernel
inline PixelMix pixel_weights(Context& g, const SiteStore& st, const CandidateField& f, int px, int py) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    int32_t xy[2] = {px, py};
    uint32_t ids[16];
    double w[16];
    int32_t n = 0;
    check(sad_pixel_weights(g.get(), &s.v, &v, xy, 1, ids, w, &n));
    PixelMix m;
    m.n = n;
    for (int i = 0; i < n; i++) {
        m.ids[i] = ids[i];
        m.w[i] = w[i];
    }
    return m;
}

// render_image (render.hpp:21-22)
inline ImageBuffer render_image(Context& g, const SiteStore& st, const CandidateField& f, const RunOpts& o = {}) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    ImageBuffer out;
    out.resize(f.width, f.height);
    check(sad_render_image(g.get(), &s.v, &v, o.fp64, out.data.data()));
    return out;
}

// render_id_map (render.hpp:26-27)
inline std::vector<uint32_t> render_id_map(Context& g, const SiteStore& st, const CandidateField& f) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    std::vector<uint32_t> out(static_cast<size_t>(f.width) * f.height);
    check(sad_render_id_map(g.get(), &s.v, &v, out.data()));
    return out;
}

inline void grads_back(const std::vector<double>& g, size_t n, GradBuffer& out) {
    out.resize(n);
    for (size_t id = 0; id < n; id++)
        for (int c = 0; c < kChannels; c++) {
            Accum& a = out.at(c, static_cast<uint32_t>(id));
            a.reset();
            a.add(g[id * kChannels + c]);
        }
}

// backward_image (grad.hpp:96-98)
inline double backward_image(Context& g, const SiteStore& st, const CandidateField& f, const ImageBuffer& target,
                             GradBuffer& out, const RunOpts& o = {}, bool with_removal = true) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    std::vector<double> buf(std::max<size_t>(st.size(), 1) * kChannels);
    uint64_t nf = 0;
    double loss = 0;
    check(sad_backward_image(g.get(), &s.v, &v, target.data.data(), o.fp64, with_removal, buf.data(), &nf, &loss));
    grads_back(buf, st.size(), out);
    out.nonfinite = nf;
    return loss;
}

// image_loss (grad.hpp:101-102)
inline double image_loss(Context& g, const SiteStore& st, const CandidateField& f, const ImageBuffer& target,
                         const RunOpts& o = {}) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    double loss = 0;
    check(sad_image_loss(g.get(), &s.v, &v, target.data.data(), o.fp64, &loss));
    return loss;
}

// backward_pixel_grad (grad.hpp:106-107)
inline void backward_pixel_grad(Context& g, const SiteStore& st, const CandidateField& f, const ImageBuffer& dl,
                                GradBuffer& out, const RunOpts& o = {}) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    std::vector<double> buf(std::max<size_t>(st.size(), 1) * kChannels);
    uint64_t nf = 0;
    check(sad_backward_pixel_grad(g.get(), &s.v, &v, dl.data.data(), dl.width, dl.height, o.fp64, buf.data(), &nf));
    grads_back(buf, st.size(), out);
    out.nonfinite = nf;
}

// clamp_project (train.hpp:38)
inline void clamp_project(Context& g, SiteStore& st, int w, int h, const TrainConfig& cfg) {
    detail::SitesView s(st);
    sad_train_config c = detail::config(cfg);
    check(sad_clamp_project(g.get(), &s.v, w, h, &c));
    s.store_into(st);
}

// init_sites (train.hpp:29): replaces the store's contents (clear + n appends: generation + 1 + n)
inline void init_sites(Context& g, SiteStore& st, const ImageBuffer& target, int n, const TrainConfig& cfg) {
    const uint64_t gen = st.generation;
    SiteStore tmp;
    tmp.resize(static_cast<size_t>(std::max(n, 0)));
    detail::SitesView s(tmp);
    sad_train_config c = detail::config(cfg);
    check(sad_init_sites(g.get(), &s.v, target.data.data(), target.width, target.height, n, &c));
    s.store_into(st);
    st.generation = gen + 1 + static_cast<uint64_t>(std::max(n, 0));
}

// bpp_target_count / plan_schedule / simulate_schedule (budget.hpp:51-60): host arithmetic of the library
inline size_t bpp_target_count(double bpp, int w, int h) {
    uint64_t out = 0;
    check(sad_bpp_target_count(bpp, w, h, &out));
    return static_cast<size_t>(out);
}
inline double plan_schedule(int n0, size_t target, const TrainConfig& cfg) {
    sad_train_config c = detail::config(cfg);
    double out = 0;
    check(sad_plan_schedule(n0, target, &c, &out));
    return out;
}
inline int simulate_schedule(int n0, double scale, const TrainConfig& cfg) {
    sad_train_config c = detail::config(cfg);
    int out = 0;
    check(sad_simulate_schedule(n0, scale, &c, &out));
    return out;
}

// adam_step (train.hpp:33-34)
inline void adam_step(Context& g, SiteStore& st, const GradBuffer& gb, AdamState& a, int w, int h,
                      const TrainConfig& cfg) {
    if (gb.size() != st.size()) throw std::invalid_argument("adam_step: gradient size mismatch");
    detail::SitesView s(st);
    std::vector<double> buf(std::max<size_t>(st.size(), 1) * kChannels);
    for (size_t id = 0; id < st.size(); id++)
        for (int c = 0; c < kChannels; c++) buf[id * kChannels + c] = gb.grad(c, static_cast<uint32_t>(id));
    a.resize(st.size());
    sad_adam_view av{a.sites(), a.sites(), a.m.data(), a.v.data(), a.t, a.skipped};
    sad_train_config c = detail::config(cfg);
    check(sad_adam_step(g.get(), &s.v, buf.data(), &av, w, h, &c));
    s.store_into(st);
    a.t = av.t;
    a.skipped = av.skipped;
}

// tau_diffusion (train.hpp:43-44): owners' logtau accumulators are reset to the mixed value
inline void tau_diffusion(Context& g, const SiteStore& st, const CandidateField& f, double lambda, GradBuffer& gb,
                          const RunOpts& = {}) {
    if (lambda == 0) return;
    if (lambda < 0 || lambda > 1) throw std::invalid_argument("tau_diffusion: lambda out of [0,1]");
    if (gb.size() != st.size()) throw std::invalid_argument("tau_diffusion: size mismatch");
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    std::vector<double> buf(std::max<size_t>(st.size(), 1) * kChannels);
    for (size_t id = 0; id < st.size(); id++)
        for (int c = 0; c < kChannels; c++) buf[id * kChannels + c] = gb.grad(c, static_cast<uint32_t>(id));
    std::vector<double> before(buf);
    check(sad_tau_diffusion(g.get(), &s.v, &v, lambda, buf.data()));
    for (size_t id = 0; id < st.size(); id++) {
        const size_t i = id * kChannels + kGradLogTau;
        if (std::memcmp(&buf[i], &before[i], sizeof(double)) == 0) continue;
        Accum& a = gb.at(kGradLogTau, static_cast<uint32_t>(id));
        a.reset();
        a.add(buf[i]);
    }
}

// accumulate_stats (budget.hpp:29-30)
inline StatsResult accumulate_stats(Context& g, const SiteStore& st, const CandidateField& f,
                                    const ImageBuffer& target, const RunOpts& = {}) {
    detail::SitesView s(st);
    sad_field_view v = detail::field_view(f);
    std::vector<double> buf(std::max<size_t>(st.size(), 1) * 8);
    uint64_t valid = 0;
    check(sad_accumulate_stats(g.get(), &s.v, &v, target.data.data(), buf.data(), &valid));
    StatsResult r;
    r.site.resize(st.size());
    for (size_t i = 0; i < st.size(); i++) {
        const double* p = &buf[i * 8];
        r.site[i] = SiteStats{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7]};
    }
    r.valid_pixels = valid;
    return r;
}

inline std::vector<double> stats_flat(const StatsResult& s) {
    std::vector<double> out(std::max<size_t>(s.site.size(), 1) * 8);
    for (size_t i = 0; i < s.site.size(); i++) {
        const SiteStats& t = s.site[i];
        double row[8] = {t.mass, t.energy, t.sx, t.sy, t.sxx, t.sxy, t.syy, t.removal};
        std::copy(row, row + 8, out.begin() + i * 8);
    }
    return out;
}

// prune (budget.hpp:48)
inline int prune(Context& g, SiteStore& st, const StatsResult& stats, double pct) {
    // the C ABI takes n*8 doubles for n sites: a StatsResult of another size is refused here (budget.cpp:287)
    if (stats.site.size() != st.size()) throw std::invalid_argument("prune: stats size mismatch");
    detail::SitesView s(st);
    std::vector<double> sf = stats_flat(stats);
    int removed = 0;
    check(sad_prune(g.get(), &s.v, sf.data(), stats.valid_pixels, pct, &removed));
    s.store_into(st);
    return removed;
}

// densify (budget.hpp:43-44)
inline int densify(Context& g, SiteStore& st, AdamState& adam, const StatsResult& stats, const ImageBuffer& target,
                   double pct, const TrainConfig& cfg) {
    if (stats.site.size() != st.size()) throw std::invalid_argument("densify: stats size mismatch");  // budget.cpp:221
    size_t n = st.size();
    detail::SitesView s(st, n);
    adam.resize(n);
    std::vector<double> m(2 * n * kGradSlots + kGradSlots), v(2 * n * kGradSlots + kGradSlots);
    std::copy(adam.m.begin(), adam.m.end(), m.begin());
    std::copy(adam.v.begin(), adam.v.end(), v.begin());
    sad_adam_view av{n, 2 * n + 1, m.data(), v.data(), adam.t, adam.skipped};
    std::vector<double> sf = stats_flat(stats);
    sad_train_config c = detail::config(cfg);
    int done = 0;
    check(sad_densify(g.get(), &s.v, &av, sf.data(), target.data.data(), target.width, target.height, pct, &c, &done));
    s.store_into(st);
    adam.m.assign(m.begin(), m.begin() + av.sites * kGradSlots);
    adam.v.assign(v.begin(), v.begin() + av.sites * kGradSlots);
    return done;
}

// fit / fit_store (train.hpp:64-68), resident on the device.
inline FitResult fit_impl(Context& g, const ImageBuffer& target, const TrainConfig& cfg, const SiteStore* init) {
    sad_train_config c = detail::config(cfg);
    sad_fit_run* run = nullptr;
    check(sad_fit_create(g.get(), target.width, target.height, &c, &run));
    struct Guard {
        sad_fit_run* r;
        ~Guard() { sad_fit_destroy(r); }
    } guard{run};
    check(sad_fit_set_target(run, target.data.data()));
    if (init) {
        detail::SitesView s(*init);
        check(sad_fit_run_store(run, &s.v));
    } else {
        check(sad_fit_run_init(run));
    }
    size_t n = 0;
    int nh = 0;
    double scale = 0;
    check(sad_fit_info(run, &n, &nh, &scale));
    FitResult r;
    SiteStore tmp;
    tmp.resize(n);
    detail::SitesView s(tmp);
    r.field.resize(target.width, target.height, cfg.k);
    sad_field_view fv = detail::field_view(r.field);
    std::vector<sad_history_row> hist(static_cast<size_t>(nh));
    check(sad_fit_download(run, &s.v, &fv, hist.data()));
    s.store_into(r.sites);
    detail::field_back(fv, r.field);
    r.field.synced_generation = r.sites.generation;
    for (const sad_history_row& h : hist) r.history.push_back(HistoryRow{h.iter, h.loss, h.psnr, h.active_sites, h.ms});
    r.schedule_scale = scale;
    return r;
}

inline FitResult fit(Context& g, const ImageBuffer& target, const TrainConfig& cfg) {
    return fit_impl(g, target, cfg, nullptr);
}

inline FitResult fit_store(Context& g, SiteStore st, const ImageBuffer& target, const TrainConfig& cfg) {
    return fit_impl(g, target, cfg, &st);
}

}  // namespace sad::b200
