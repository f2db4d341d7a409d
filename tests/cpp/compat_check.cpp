// compat_check.cpp — the reference's own API driving the B200 library through sad_b200_compat.hpp,
// checked against the reference implementation (libsadref.so, compiled from /root/reference) in
// the same process.  Mirrors the reference tests' fixtures (test_candidates.cpp:15-33,
// test_grad.cpp:16-41).  Built by oracle/Makefile (needs the reference headers), run by
// tests/test_compat_cpp.py on a GPU.  Prints one line per check and exits non-zero on failure.
#include "sad/rng.hpp"
#include "sad_b200_compat.hpp"

#include <cmath>
#include <cstdio>

using namespace sad;

static int failures = 0;
static void expect(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) failures++;
}

static SiteStore random_model(int w, int h, int n, uint64_t seed) {
    SiteStore st;
    RngState rng = seeded_stream(seed, 0xbeef, 1);
    for (int i = 0; i < n; i++) {
        Site s;
        s.x = rng.next_unit() * (w - 1);
        s.y = rng.next_unit() * (h - 1);
        s.log_tau = 6.0 + rng.next_unit() * 3.0;
        s.radius = 1.0 + rng.next_unit() * 8.0;
        for (int c = 0; c < 3; c++) s.color[c] = rng.next_unit();
        double th = rng.next_unit() * 6.283185307179586;
        s.dir[0] = std::cos(th);
        s.dir[1] = std::sin(th);
        s.aniso = (rng.next_unit() - 0.5) * 2.0;
        st.append(s);
    }
    return st;
}

static ImageBuffer random_target(int w, int h, uint64_t seed) {
    ImageBuffer img;
    img.resize(w, h);
    RngState rng = seeded_stream(seed, 0x515, 2);
    for (double& v : img.data) v = rng.next_unit();
    return img;
}

int main() {
    b200::Context gpu;
    const int W = 64, H = 48;
    SiteStore st = random_model(W, H, 90, 7);
    ImageBuffer tgt = random_target(W, H, 8);
    RunOpts f32{false, 1};

    CandidateField a, b;
    a.resize(W, H, 8);
    b.resize(W, H, 8);
    refresh(st, a, RefreshMode::Full, 4, 4, 7, f32);
    b200::refresh(gpu, st, b, RefreshMode::Full, 4, 4, 7, f32);
    expect(a.ids == b.ids && a.pass_index == b.pass_index, "refresh(Full) maps identical");
    refresh(st, a, RefreshMode::WarmStart, 3, 4, 9, f32);
    b200::refresh(gpu, st, b, RefreshMode::WarmStart, 3, 4, 9, f32);
    expect(a.ids == b.ids, "refresh(WarmStart) maps identical");

    ImageBuffer ra = render_image(st, a, f32), rb = b200::render_image(gpu, st, b, f32);
    expect(ra.data == rb.data, "render_image fp32 bit-identical");

    GradBuffer ga, gb;
    double la = backward_image(st, a, tgt, ga, f32, true);
    double lb = b200::backward_image(gpu, st, b, tgt, gb, f32, true);
    bool same = la == lb;
    for (uint32_t id = 0; id < st.size(); id++)
        for (int c = 0; c < kChannels; c++) same = same && ga.grad(c, id) == gb.grad(c, id);
    expect(same, "backward_image fp32 loss and gradients bit-identical");

    GradBuffer ta = ga, tb = ga;
    tau_diffusion(st, a, 0.4, ta);
    b200::tau_diffusion(gpu, st, b, 0.4, tb);
    bool tsame = true;
    for (uint32_t id = 0; id < st.size(); id++)
        for (int c = 0; c < kChannels; c++) tsame = tsame && ta.grad(c, id) == tb.grad(c, id);
    expect(tsame, "tau_diffusion bit-identical");

    SiteStore sa = st, sb = st;
    AdamState ma, mb;
    TrainConfig cfg;
    adam_step(sa, ga, ma, W, H, cfg);
    b200::adam_step(gpu, sb, ga, mb, W, H, cfg);
    expect(sa.x == sb.x && sa.dir_y == sb.dir_y && ma.t == mb.t, "adam_step bit-identical");

    CandidateField fa;
    fa.resize(W, H, 8);
    refresh(st, fa, RefreshMode::Full, 4, 4, 7, RunOpts{});
    StatsResult s1 = accumulate_stats(st, fa, tgt), s2 = b200::accumulate_stats(gpu, st, fa, tgt);
    bool sclose = s1.valid_pixels == s2.valid_pixels;
    for (size_t i = 0; i < st.size(); i++)
        sclose = sclose && std::abs(s1.site[i].removal - s2.site[i].removal) <= 1e-12 * (1 + std::abs(s1.site[i].removal));
    expect(sclose, "accumulate_stats within 1e-12");
    SiteStore pa = st, pb = st;
    expect(prune(pa, s1, 0.2) == b200::prune(gpu, pb, s1, 0.2) && pa.active == pb.active, "prune identical");
    AdamState da, db;
    da.resize(pa.size());
    db.resize(pb.size());
    int na = densify(pa, da, s1, tgt, 0.5, cfg), nb = b200::densify(gpu, pb, db, s1, tgt, 0.5, cfg);
    expect(na == nb && pa.x == pb.x && pa.size() == pb.size(), "densify identical");

    TrainConfig fc;
    fc.iters = 60;
    fc.target_bpp = 4.0;
    fc.fp64 = false;
    fc.seed = 5;
    ImageBuffer small = random_target(32, 24, 3);
    FitResult r1 = fit(small, fc), r2 = b200::fit(gpu, small, fc);
    bool hist = r1.history.size() == r2.history.size();
    for (size_t i = 0; hist && i < r1.history.size(); i++) hist = history_line(r1.history[i]) == history_line(r2.history[i]);
    expect(hist && r1.field.ids == r2.field.ids, "fit(): history lines and final map bit-identical");
    std::printf("%d failure(s)\n", failures);
    return failures ? 1 : 0;
}
