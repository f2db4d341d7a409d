// Link shim: the reference library's hot-path functions, with the exact signatures of its
// headers (candidates.hpp, render.hpp, grad.hpp, train.hpp, budget.hpp), defined in namespace `sad` over
// the B200 library's C ABI (include/sad_b200.h via include/sad_b200_compat.hpp) on one device context
// per host thread.  Linked into the reference's own, unmodified test sources (tests/reftests/Makefile)
// in place of the reference's CPU definitions, so those tests run against libsad_b200.so.
//
// Replaced: jfa_seed, propagate_pass, run_passes, refresh, exact_topk(_batch) | pixel_weights,
// render_image, render_id_map, render_tau_map | backward_image, image_loss, backward_pixel_grad | init_sites, adam_step,
// clamp_project, tau_diffusion, fit, fit_store | accumulate_stats, densify, prune, bpp_target_count,
// plan_schedule, simulate_schedule.  Everything else (value types, codec, quality, GradBuffer,
// TileReducer, for_each_contribution, the jump schedule helpers, boundary_map, ...) is the reference's
// own code, built from its sources.
#include "sad_b200_compat.hpp"

namespace sad {

namespace {
b200::Context& gpu() {
    thread_local b200::Context ctx(0);
    return ctx;
}
}  // namespace

// ---------------------------------------------------------------- candidates.hpp
void jfa_seed(const SiteStore& sites, CandidateField& field) { b200::jfa_seed(gpu(), sites, field); }

void propagate_pass(const SiteStore& sites, CandidateField& field, const PassSpec& pass, int inject, uint64_t seed,
                    const RunOpts& opts) {
    b200::propagate_pass(gpu(), sites, field, pass, inject, seed, opts);
}

void run_passes(const SiteStore& sites, CandidateField& field, const std::vector<PassSpec>& seq, int inject,
                uint64_t seed, const RunOpts& opts) {
    if (field.gw < 1 || field.gh < 1) throw std::invalid_argument("run_passes: field not sized");
    b200::run_passes(gpu(), sites, field, seq, inject, seed, opts);
}

void refresh(const SiteStore& sites, CandidateField& field, RefreshMode mode, int passes, int inject, uint64_t seed,
             const RunOpts& opts) {
    b200::refresh(gpu(), sites, field, mode, passes, inject, seed, opts);
}

std::vector<uint32_t> exact_topk(const SiteStore& sites, double px, double py, int k, double scale, bool fp64) {
    return b200::exact_topk(gpu(), sites, px, py, k, scale, fp64);
}

std::vector<std::vector<uint32_t>> exact_topk_batch(const SiteStore& sites,
                                                    const std::vector<std::pair<int, int>>& pixels, int k,
                                                    double scale, bool fp64) {
    return b200::exact_topk_batch(gpu(), sites, pixels, k, scale, fp64);
}

// ---------------------------------------------------------------- render.hpp
PixelMix pixel_weights(const SiteStore& sites, const CandidateField& field, int px, int py) {
    return b200::pixel_weights(gpu(), sites, field, px, py);
}

ImageBuffer render_image(const SiteStore& sites, const CandidateField& field, const RunOpts& opts) {
    return b200::render_image(gpu(), sites, field, opts);
}

std::vector<uint32_t> render_id_map(const SiteStore& sites, const CandidateField& field, const RunOpts&) {
    return b200::render_id_map(gpu(), sites, field);
}

// render_tau_map (render.cpp:157-163): the owner's log-temperature per pixel, owners from the device id map
std::vector<double> render_tau_map(const SiteStore& sites, const CandidateField& field, const RunOpts& opts) {
    std::vector<uint32_t> owners = render_id_map(sites, field, opts);
    std::vector<double> out(owners.size());
    for (size_t i = 0; i < owners.size(); i++) out[i] = sites.log_tau[owners[i]];
    return out;
}

// ---------------------------------------------------------------- grad.hpp
double backward_image(const SiteStore& sites, const CandidateField& field, const ImageBuffer& target, GradBuffer& out,
                      const RunOpts& opts, bool with_removal) {
    if (target.width != field.width || target.height != field.height)
        throw std::invalid_argument("backward: target size mismatch");
    return b200::backward_image(gpu(), sites, field, target, out, opts, with_removal);
}

double image_loss(const SiteStore& sites, const CandidateField& field, const ImageBuffer& target,
                  const RunOpts& opts) {
    if (target.width != field.width || target.height != field.height)
        throw std::invalid_argument("loss: target size mismatch");
    return b200::image_loss(gpu(), sites, field, target, opts);
}

void backward_pixel_grad(const SiteStore& sites, const CandidateField& field, const ImageBuffer& dl_dvalue,
                         GradBuffer& out, const RunOpts& opts) {
    b200::backward_pixel_grad(gpu(), sites, field, dl_dvalue, out, opts);
}

// ---------------------------------------------------------------- train.hpp
void init_sites(SiteStore& st, const ImageBuffer& target, int n, const TrainConfig& cfg) {
    b200::init_sites(gpu(), st, target, n, cfg);
}

void adam_step(SiteStore& st, const GradBuffer& g, AdamState& a, int width, int height, const TrainConfig& cfg) {
    b200::adam_step(gpu(), st, g, a, width, height, cfg);
}

void clamp_project(SiteStore& st, int width, int height, const TrainConfig& cfg) {
    b200::clamp_project(gpu(), st, width, height, cfg);
}

void tau_diffusion(const SiteStore& st, const CandidateField& field, double lambda, GradBuffer& g,
                   const RunOpts& opts) {
    b200::tau_diffusion(gpu(), st, field, lambda, g, opts);
}

FitResult fit(const ImageBuffer& target, const TrainConfig& cfg) { return b200::fit(gpu(), target, cfg); }

FitResult fit_store(SiteStore st, const ImageBuffer& target, const TrainConfig& cfg) {
    return b200::fit_store(gpu(), std::move(st), target, cfg);
}

// ---------------------------------------------------------------- budget.hpp
StatsResult accumulate_stats(const SiteStore& sites, const CandidateField& field, const ImageBuffer& target,
                             const RunOpts& opts) {
    if (target.width != field.width || target.height != field.height)
        throw std::invalid_argument("stats: target size mismatch");
    return b200::accumulate_stats(gpu(), sites, field, target, opts);
}

int densify(SiteStore& st, AdamState& adam, const StatsResult& stats, const ImageBuffer& target, double percentile,
            const TrainConfig& cfg) {
    return b200::densify(gpu(), st, adam, stats, target, percentile, cfg);
}

int prune(SiteStore& st, const StatsResult& stats, double percentile) {
    return b200::prune(gpu(), st, stats, percentile);
}

size_t bpp_target_count(double bpp, int width, int height) { return b200::bpp_target_count(bpp, width, height); }

double plan_schedule(int n0, size_t target, const TrainConfig& cfg) { return b200::plan_schedule(n0, target, cfg); }

int simulate_schedule(int n0, double scale, const TrainConfig& cfg) { return b200::simulate_schedule(n0, scale, cfg); }

}  // namespace sad
