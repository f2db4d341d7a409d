// sad_runtime.cu — host runtime of the B200 SAD library: context, device workspace, the C ABI of
// include/sad_b200.h (per-call entry points that mirror the reference functions), and the resident
// fit loop (train.cpp:221-311) that keeps every buffer in HBM between the target upload and the
// result download.
#include "../../include/sad_b200.h"
#include "sad_kernels.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <cstring>
#include <stdexcept>
#include <string>
#include <limits>
#include <dlfcn.h>
#include <functional>
#include <nccl.h>
#include <memory>
#include <vector>

using sadk::DevState;

namespace {

thread_local std::string g_err;
bool g_cuda_used = false;  // a context exists: launch errors are worth checking

struct SadFail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw SadFail{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SAD_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
sad_status guard(F&& f) {
    try {
        f();
        if (g_cuda_used) {
            cudaError_t le = cudaGetLastError();  // kernel launch failures (no synchronisation)
            if (le != cudaSuccess) fail(SAD_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(le));
        }
        return SAD_OK;
    } catch (const SadFail& e) {
        g_err = e.msg;
        return static_cast<sad_status>(e.code);
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SAD_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SAD_EINVAL;
    }
}

// ------------------------------------------------------------------ device buffers
// Bumped by every device allocation: cached CUDA graphs hold raw buffer addresses and are dropped
// when it moves (sad_fit_run::plain).
static std::atomic<uint64_t> g_alloc_epoch{0};

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void ensure(size_t m) {
        if (m <= n && p) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        if (m == 0) m = 1;
        ck(cudaMalloc(&p, m * sizeof(T)), "cudaMalloc");
        g_alloc_epoch.fetch_add(1, std::memory_order_relaxed);
        n = m;
    }
};

// ------------------------------------------------------------------ host-side reference arithmetic
uint32_t ceil_log2(uint32_t v) {
    uint32_t e = 0;
    while ((1u << e) < v) e++;
    return e;
}

// jump_step (candidates.cpp:27-33)
uint32_t jump_step(uint32_t t, uint32_t b) {
    if (b < 2 || (b & (b - 1)) != 0) fail(SAD_EINVAL, "jump_step: b must be a power of two >= 2");
    uint32_t lg = ceil_log2(b);
    uint32_t e = (t < lg - 1 ? t : lg - 1) + 1;
    uint32_t s = b >> e;
    return s < 1 ? 1 : s;
}

std::vector<sad_pass_spec> full_refresh_passes(int gw, int gh, int extra) {
    if (gw < 1 || gh < 1) fail(SAD_EINVAL, "JumpSchedule: empty extent");
    uint32_t m = static_cast<uint32_t>(gw > gh ? gw : gh);
    uint32_t b = 1u << ceil_log2(m);
    if (b < 2) b = 2;
    uint32_t events = ceil_log2(m);
    std::vector<sad_pass_spec> seq;
    for (uint32_t t = 0; t < events; t++) seq.push_back({jump_step(t, b), 1});
    for (int i = 0; i < extra; i++) seq.push_back({1, 0});
    return seq;
}

std::vector<sad_pass_spec> schedule_passes(int gw, int gh, int total) {
    if (gw < 1 || gh < 1) fail(SAD_EINVAL, "JumpSchedule: empty extent");
    uint32_t m = static_cast<uint32_t>(gw > gh ? gw : gh);
    uint32_t b = 1u << ceil_log2(m);
    if (b < 2) b = 2;
    uint32_t events = ceil_log2(m);
    std::vector<sad_pass_spec> seq;
    for (int t = 0; t < total; t++) {
        uint32_t tu = static_cast<uint32_t>(t);
        seq.push_back(tu < events ? sad_pass_spec{jump_step(tu, b), 1} : sad_pass_spec{1, 0});
    }
    return seq;
}

double norm_scale(int w, int h) {
    if (w < 1 || h < 1) fail(SAD_EINVAL, "normalization_scale: empty extent");
    return 1.0 / static_cast<double>(w > h ? w : h);
}

// TrainConfig::validate (types.cpp:103-126)
void validate(sad_train_config& c, int w, int h) {
    auto bad = [](const char* m) { fail(SAD_EINVAL, m); };
    if (w < 1 || h < 1) bad("config: empty image");
    if (c.iters < 0) bad("config: negative iters");
    if (c.k < 1 || c.k > 16) bad("config: k out of [1,16]");
    if (c.inject < 0) bad("config: negative inject");
    if (c.lambda_init < 0 || c.lambda_init > 1) bad("config: lambda_init out of [0,1]");
    if (c.densify_every < 1 || c.prune_every < 1) bad("config: event period < 1");
    if (c.densify_pct < 0 || c.densify_pct > 1 || c.prune_pct < 0 || c.prune_pct > 1)
        bad("config: percentile out of [0,1]");
    if (c.refresh_every < 1) bad("config: refresh period < 1");
    if (c.refresh_passes < 0 || c.final_passes < 0) bad("config: negative passes");
    if (c.target_bpp < 0) bad("config: negative bpp");
    if (c.n_sites < 0) bad("config: negative site count");
    if (c.log_tau_min > c.log_tau_max || c.radius_min > c.radius_max || c.aniso_min > c.aniso_max)
        bad("config: inverted clamp range");
    if (c.threads < 1) c.threads = 1;
    c.densify_start = std::clamp(c.densify_start, 0, c.iters);
    c.densify_end = std::clamp(c.densify_end, 0, c.iters);
    c.prune_start = std::clamp(c.prune_start, 0, c.iters);
    c.prune_end = std::clamp(c.prune_end, 0, c.iters);
    if (c.densify_end < c.densify_start || c.prune_end < c.prune_start) bad("config: inverted schedule window");
}

uint64_t bpp_target_count(double bpp, int w, int h) {
    if (bpp < 0 || w < 1 || h < 1) fail(SAD_EINVAL, "bpp target: bad inputs");
    return static_cast<uint64_t>(bpp * static_cast<double>(w) * h / 128.0);
}

// simulate_schedule (budget.cpp:312-332)
int simulate_schedule(int n0, double scale, const sad_train_config& c) {
    int n = n0;
    for (int t = 1; t <= c.iters; t++) {
        bool ev_d = t >= c.densify_start && t <= c.densify_end && t % c.densify_every == 0;
        bool ev_p = t >= c.prune_start && t <= c.prune_end && t % c.prune_every == 0;
        if (ev_p && !c.prune_during_densify && t <= c.densify_end) ev_p = false;
        if (ev_p) {
            int p = static_cast<int>(n * c.prune_pct * scale);
            if (p >= n) p = n - 1;
            if (p > 0) n -= p;
        }
        if (ev_d) {
            int d = static_cast<int>(n * c.densify_pct * scale);
            if (c.max_sites > 0 && static_cast<size_t>(n + d) > c.max_sites) d = static_cast<int>(c.max_sites) - n;
            if (d > 0) n += d;
        }
    }
    return n;
}

// plan_schedule (budget.cpp:334-374)
double plan_schedule(int n0, uint64_t target, const sad_train_config& c) {
    double cap = c.budget_scale_cap, tgt = static_cast<double>(target);
    int mn = n0, mx = n0;
    auto miss = [&](double s) {
        int fin = simulate_schedule(n0, s, c);
        mn = std::min(mn, fin);
        mx = std::max(mx, fin);
        return std::abs(static_cast<double>(fin) - tgt);
    };
    double best_s = 0, best_m = miss(0);
    for (int i = 1; i <= 96; i++) {
        double s = cap * i / 96;
        double m = miss(s);
        if (m < best_m) {
            best_m = m;
            best_s = s;
        }
    }
    double lo = std::max(0.0, best_s - cap / 96), hi = std::min(cap, best_s + cap / 96);
    for (int i = 0; i <= 256; i++) {
        double s = lo + (hi - lo) * i / 256;
        double m = miss(s);
        if (m < best_m) {
            best_m = m;
            best_s = s;
        }
    }
    if (tgt < mn || tgt > mx) {
        std::fprintf(stderr, "schedule: target %llu outside reachable range [%d, %d], using scale cap\n",
                     static_cast<unsigned long long>(target), mn, mx);
        return cap;
    }
    return best_s;
}

// ------------------------------------------------------------------ xorshift32 jump-ahead (GF(2) matrices)
struct Gf2 {
    uint32_t col[32];
};

uint32_t gf2_apply(const Gf2& m, uint32_t s) {
    uint32_t r = 0;
    for (int i = 0; i < 32; i++)
        if (s >> i & 1u) r ^= m.col[i];
    return r;
}

Gf2 gf2_mul(const Gf2& a, const Gf2& b) {
    Gf2 r;
    for (int i = 0; i < 32; i++) r.col[i] = gf2_apply(a, b.col[i]);
    return r;
}

Gf2 xs_matrix_pow(uint64_t e) {
    Gf2 base, acc;
    for (int i = 0; i < 32; i++) {
        uint32_t x = 1u << i;
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        base.col[i] = x;
        acc.col[i] = 1u << i;
    }
    while (e) {
        if (e & 1) acc = gf2_mul(base, acc);
        base = gf2_mul(base, base);
        e >>= 1;
    }
    return acc;
}

uint32_t mix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h;
}

uint32_t seeded_state(uint64_t seed, uint32_t a, uint32_t b) {
    uint32_t h = mix32(static_cast<uint32_t>(seed) ^ 0x9e3779b9u);
    h ^= mix32(static_cast<uint32_t>(seed >> 32) + 0x85ebca6bu);
    h = mix32(h + mix32(a ^ 0x27d4eb2fu));
    h = mix32(h ^ mix32(b + 0x165667b1u));
    return h ? h : 0x6b33a1c9u;
}

// states[c] = stream state after c * stride draws.
std::vector<uint32_t> jump_states(uint32_t s0, uint64_t stride, size_t count) {
    Gf2 m = xs_matrix_pow(stride);
    std::vector<uint32_t> out(count);
    uint32_t s = s0;
    for (size_t c = 0; c < count; c++) {
        out[c] = s;
        s = gf2_apply(m, s);
    }
    return out;
}

// ------------------------------------------------------------------ workspace
struct Workspace {
    cudaStream_t stream = nullptr;
    int cap = 0;
    int w = 0, h = 0;
    sadk::FieldDims fd{};
    DBuf<double> params;
    DBuf<uint8_t> active, frozen;
    DBuf<uint32_t> ids[2];
    int cur = 0;
    DBuf<char> pack, gtab, rtab, rtab_d;
    DBuf<double2> grads, stats;       // RedTarget.over: [11][cap] / [8][cap]
    DBuf<double2> gpart, spart;       // RedTarget.part records
    DBuf<int32_t> gcnt, scnt;         // RedTarget.cnt
    DBuf<double2> loss_part;          // per-block loss partials
    int maxt = getenv("SAD_MAXT") ? atoi(getenv("SAD_MAXT")) : 16;  // record slots per site and pass
    // Test knobs (read at context / run creation): force the overflow-record pool and the adaptive
    // record pool down to a fixed size, so tests reach the exhausted-pool fallbacks (exact DD CAS).
    int ocap_force = getenv("SAD_OCAP") ? std::max(1, atoi(getenv("SAD_OCAP"))) : 0;
    long long apsize_force = getenv("SAD_APSIZE") ? std::max(1ll, atoll(getenv("SAD_APSIZE"))) : 0;
    DBuf<double> m, v;
    DBuf<uint32_t> act, free_list;
    DBuf<uint8_t> flags;
    DBuf<unsigned long long> keys[2];
    DBuf<uint32_t> vals[2];
    DBuf<char> cub_tmp;
    DBuf<double> tgt_d, px_d;
    DBuf<float> tgt_f, px_f;
    DBuf<DevState> st;
    DevState* hst = nullptr;  // pinned mirror
    // init_sites scratch (train.cpp:59-111 on the device), sized for W*H pixels
    struct InitBufs {
        size_t np = 0;
        DBuf<double> mag;
        DBuf<double2> gsum;
        DBuf<unsigned long long> k0, k1;
        DBuf<uint32_t> v0, v1, cells, jk, jo;
        DBuf<uint8_t> fl;
        DBuf<int32_t> nsel;
        DBuf<char> tmp;
    } ib;
    // tau_diffusion scratch (train.cpp:171-213): W*H*k edge keys, owner map, per-site totals
    struct TauBufs {
        size_t ne = 0;
        int nb = 0, tcap = 0;
        DBuf<uint64_t> k0, k1;
        DBuf<int32_t> count;
        DBuf<uint32_t> owner;
        DBuf<double> tot, g0;
        DBuf<char> tmp;
        size_t tmp_bytes = 0;
    } tb;

    ~Workspace() {
        if (hst) cudaFreeHost(hst);
    }

    sadk::SitesDev sites() { return sadk::SitesDev{params.p, active.p, frozen.p, cap}; }
    DBuf<int32_t> ghead, shead, gnext, snext, otops;  // overflow lists (otops: [0] grads, [1] stats)
    DBuf<double2> gopart, sopart;
    int ocap = 0;
    sadk::RedTarget gred() {
        return sadk::RedTarget{grads.p, gpart.p, gcnt.p, cap, maxt, 11, ghead.p, gnext.p, gopart.p, otops.p, ocap,
                               nullptr, nullptr, 0};
    }
    sadk::RedTarget sred() {
        return sadk::RedTarget{stats.p, spart.p, scnt.p, cap, maxt, 8, shead.p, snext.p, sopart.p, otops.p + 1, ocap,
                               nullptr, nullptr, 0};
    }
    // Adaptive stats-record layout of the resident fit's events: capacities from the gradient record counts
    // of the same pass (k_stats_plan), offsets by an exclusive scan; a pool of `spsize` 8-channel records
    DBuf<double2> spool;
    DBuf<int32_t> sroff, srcap;
    long long spsize = 0;
    sadk::RedTarget sred_adaptive() {
        sadk::RedTarget t = sred();
        t.roff = sroff.p;
        t.rcap = srcap.p;
        t.part = spool.p;
        t.psize = spsize;
        return t;
    }
    // Adaptive gradient-record layout of the resident fit (see RedTarget): per-site capacity planned
    // from the previous pass, offsets by an exclusive scan, one pool.
    DBuf<double2> apool;
    DBuf<int32_t> roff, rcap;
    long long apsize = 0;
    sadk::RedTarget gred_adaptive() {
        sadk::RedTarget t = gred();
        t.roff = roff.p;
        t.rcap = rcap.p;
        t.part = apool.p;
        t.psize = apsize;
        return t;
    }
    // order tags of the fp64 reference-order reduction (sadk::fp64_ordered): per record of gpart
    // (cap * maxt), of the adaptive pool and of the overflow pool; per-site values for Adam
    DBuf<uint32_t> gtag, atag, otag;
    DBuf<double> otot;
    sadk::RedTarget gred_ord() {
        sadk::RedTarget t = gred();
        gtag.ensure(static_cast<size_t>(cap) * maxt);
        otag.ensure(static_cast<size_t>(ocap));
        t.tag = gtag.p;
        t.otag = otag.p;
        return t;
    }
    sadk::RedTarget gred_adaptive_ord() {
        sadk::RedTarget t = gred_adaptive();
        atag.ensure(static_cast<size_t>(apsize));
        otag.ensure(static_cast<size_t>(ocap));
        t.tag = atag.p;
        t.otag = otag.p;
        return t;
    }
    void ensure_adaptive(size_t tiles) {
        long long want = apsize_force ? apsize_force : 16ll * cap + 64ll * static_cast<long long>(tiles);
        if (apsize < want || !apool.p) {
            apool.ensure(static_cast<size_t>(want) * 11);
            apsize = want;
        }
        roff.ensure(cap);
        rcap.ensure(cap);
    }
    void plan_records() {  // roff = exclusive_scan(rcap)
        size_t bytes = cub_tmp.n;
        ck(cub::DeviceScan::ExclusiveSum(cub_tmp.p, bytes, rcap.p, roff.p, cap, stream), "DeviceScan");
    }
    // overflow pool sized from the number of reduction tiles (each tile adds at most its bucket count)
    void ensure_pool(size_t tiles) {
        size_t want = ocap_force ? static_cast<size_t>(ocap_force) : std::max<size_t>(tiles * 16, 4096);
        if (static_cast<size_t>(ocap) >= want && otops.p) return;
        gnext.ensure(want);
        snext.ensure(want);
        gopart.ensure(want * 11);
        sopart.ensure(want * 8);
        otops.ensure(3);  // [0] gradient overflow top, [1] stats overflow top, [2] gradient record pool top
        ck(cudaMemsetAsync(otops.p, 0, 3 * sizeof(int32_t), stream), "memset otop");
        ocap = static_cast<int>(want);
    }
    void zero_red(bool g) {
        if (g) {
            ck(cudaMemsetAsync(grads.p, 0, sizeof(double2) * 11 * cap, stream), "memset grads");
            ck(cudaMemsetAsync(gcnt.p, 0, sizeof(int32_t) * cap, stream), "memset gcnt");
            ck(cudaMemsetAsync(ghead.p, 0xff, sizeof(int32_t) * cap, stream), "memset ghead");
            ck(cudaMemsetAsync(otops.p, 0, sizeof(int32_t), stream), "memset otop");
        } else {
            ck(cudaMemsetAsync(stats.p, 0, sizeof(double2) * 8 * cap, stream), "memset stats");
            ck(cudaMemsetAsync(scnt.p, 0, sizeof(int32_t) * cap, stream), "memset scnt");
            ck(cudaMemsetAsync(shead.p, 0xff, sizeof(int32_t) * cap, stream), "memset shead");
            ck(cudaMemsetAsync(otops.p + 1, 0, sizeof(int32_t), stream), "memset otop");
        }
    }

    void ensure_state() {
        if (!st.p) {
            st.ensure(1);
            ck(cudaMallocHost(&hst, sizeof(DevState)), "cudaMallocHost");
            std::memset(hst, 0, sizeof(DevState));
            ck(cudaMemsetAsync(st.p, 0, sizeof(DevState), stream), "memset state");
        }
    }

    // Grows every per-site buffer to `c` slots (contents of params/flags/adam preserved).
    void ensure_cap(int c) {
        ensure_state();
        if (c <= cap && params.p) return;
        int nc = std::max(c, 1);
        auto grow_d = [&](DBuf<double>& b, size_t per) {
            DBuf<double> nb;
            nb.ensure(per * nc);
            ck(cudaMemsetAsync(nb.p, 0, per * nc * sizeof(double), stream), "memset");
            if (b.p && cap > 0)
                for (size_t k = 0; k < per; k++)
                    ck(cudaMemcpyAsync(nb.p + k * nc, b.p + k * cap, cap * sizeof(double), cudaMemcpyDeviceToDevice,
                                       stream),
                       "grow copy");
            std::swap(b.p, nb.p);
            std::swap(b.n, nb.n);
        };
        auto grow_u8 = [&](DBuf<uint8_t>& b) {
            DBuf<uint8_t> nb;
            nb.ensure(nc);
            ck(cudaMemsetAsync(nb.p, 0, nc, stream), "memset");
            if (b.p && cap > 0) ck(cudaMemcpyAsync(nb.p, b.p, cap, cudaMemcpyDeviceToDevice, stream), "grow copy");
            std::swap(b.p, nb.p);
            std::swap(b.n, nb.n);
        };
        ck(cudaStreamSynchronize(stream), "sync");
        grow_d(params, 10);
        grow_d(m, 10);
        grow_d(v, 10);
        grow_u8(active);
        grow_u8(frozen);
        cap = nc;
        pack.ensure(static_cast<size_t>(nc) * 64);
        gtab.ensure(static_cast<size_t>(nc) * 96);
        rtab.ensure(static_cast<size_t>(nc) * 96);
        rtab_d.ensure(static_cast<size_t>(nc) * 96);
        grads.ensure(static_cast<size_t>(nc) * 11);
        stats.ensure(static_cast<size_t>(nc) * 8);
        gpart.ensure(static_cast<size_t>(nc) * maxt * 11);
        spart.ensure(static_cast<size_t>(nc) * maxt * 8);
        gcnt.ensure(nc);
        scnt.ensure(nc);
        ghead.ensure(nc);
        shead.ensure(nc);
        ck(cudaMemsetAsync(ghead.p, 0xff, ghead.n * sizeof(int32_t), stream), "memset ghead");
        ck(cudaMemsetAsync(shead.p, 0xff, shead.n * sizeof(int32_t), stream), "memset shead");
        ck(cudaMemsetAsync(grads.p, 0, grads.n * sizeof(double2), stream), "memset grads");
        ck(cudaMemsetAsync(gcnt.p, 0, gcnt.n * sizeof(int32_t), stream), "memset gcnt");
        ck(cudaMemsetAsync(scnt.p, 0, scnt.n * sizeof(int32_t), stream), "memset scnt");
        act.ensure(nc);
        free_list.ensure(nc);
        flags.ensure(nc);
        for (int i = 0; i < 2; i++) {
            keys[i].ensure(nc);
            vals[i].ensure(nc);
        }
        ensure_cub(nc);
    }

    void ensure_cub(size_t items) {
        size_t a = 0, b = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, a, keys[0].p, keys[1].p, vals[0].p, vals[1].p, static_cast<int>(items),
                                        0, 64, stream);
        thrust::counting_iterator<uint32_t> it(0);
        cub::DeviceSelect::Flagged(nullptr, b, it, flags.p, act.p, &st.p->n_active, static_cast<int>(items), stream);
        size_t c = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, c, static_cast<int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                      static_cast<int>(items), stream);
        cub_tmp.ensure(std::max({a, b, c}) + 256);
    }

    void ensure_field(int w_, int h_, int k, int cell) {
        w = w_;
        h = h_;
        fd.width = w_;
        fd.height = h_;
        fd.cell = cell;
        fd.gw = (w_ + cell - 1) / cell;
        fd.gh = (h_ + cell - 1) / cell;
        fd.k = k;
        size_t n = static_cast<size_t>(fd.gw) * fd.gh * k;
        ids[0].ensure(n);
        ids[1].ensure(n);
        loss_part.ensure(static_cast<size_t>(std::max({sadk::backward_blocks(false, fd), sadk::backward_blocks(true, fd),
                                                       sadk::loss_blocks(fd)})));
        ensure_pool(static_cast<size_t>(std::max(sadk::backward_blocks(false, fd),
                                                 ((w_ + 7) / 8) * ((h_ + 7) / 8))));
    }

    void ensure_target(size_t px) {
        tgt_d.ensure(3 * px);
        tgt_f.ensure(3 * px);
    }

    // ---- state scalars
    void set_state(const DevState& s) {
        *hst = s;
        ck(cudaMemcpyAsync(st.p, hst, sizeof(DevState), cudaMemcpyHostToDevice, stream), "H2D state");
    }
    DevState get_state() {
        ck(cudaMemcpyAsync(hst, st.p, sizeof(DevState), cudaMemcpyDeviceToHost, stream), "D2H state");
        ck(cudaStreamSynchronize(stream), "sync");
        return *hst;
    }
    template <typename F>
    void patch_state(size_t off, const F& val) {
        ck(cudaMemcpyAsync(reinterpret_cast<char*>(st.p) + off, &val, sizeof(F), cudaMemcpyHostToDevice, stream),
           "patch state");
    }
    void zero_state_field(size_t off, size_t bytes) {
        ck(cudaMemsetAsync(reinterpret_cast<char*>(st.p) + off, 0, bytes, stream), "memset state");
    }

    // ---- active list (SiteStore::active_ids, types.cpp:71-80)
    void compute_active() {
        sadk::launch_flag_active(sites(), st.p, flags.p, stream);
        size_t bytes = cub_tmp.n;
        thrust::counting_iterator<uint32_t> it(0);
        ck(cub::DeviceSelect::Flagged(cub_tmp.p, bytes, it, flags.p, act.p, &st.p->n_active, cap, stream),
           "DeviceSelect active");
    }

    void sort_pairs(int n) {
        size_t bytes = cub_tmp.n;
        ck(cub::DeviceRadixSort::SortPairs(cub_tmp.p, bytes, keys[0].p, keys[1].p, vals[0].p, vals[1].p, n, 0, 64,
                                           stream),
           "DeviceRadixSort");
    }
};

// host view -> device
void upload_sites(Workspace& ws, const sad_sites_view* v, int extra_cap = 0) {
    if (!v) fail(SAD_EINVAL, "null sites view");
    size_t n = v->size;
    if (n > static_cast<size_t>(INT32_MAX / 2)) fail(SAD_EINVAL, "too many sites");
    ws.ensure_cap(static_cast<int>(n) + extra_cap);
    const double* src[10] = {v->x, v->y, v->log_tau, v->radius, v->col_r, v->col_g, v->col_b, v->dir_x, v->dir_y,
                             v->aniso};
    if (n) {
        for (int k = 0; k < 10; k++)
            ck(cudaMemcpyAsync(ws.params.p + static_cast<size_t>(k) * ws.cap, src[k], n * 8, cudaMemcpyHostToDevice,
                               ws.stream),
               "H2D sites");
        ck(cudaMemcpyAsync(ws.active.p, v->active, n, cudaMemcpyHostToDevice, ws.stream), "H2D active");
        ck(cudaMemcpyAsync(ws.frozen.p, v->frozen, n, cudaMemcpyHostToDevice, ws.stream), "H2D frozen");
    }
    ws.patch_state(offsetof(DevState, n_sites), static_cast<int32_t>(n));
}

void download_sites(Workspace& ws, sad_sites_view* v, size_t n) {
    if (n > v->capacity) fail(SAD_ENOMEM, "sites view capacity too small");
    double* dst[10] = {v->x, v->y, v->log_tau, v->radius, v->col_r, v->col_g, v->col_b, v->dir_x, v->dir_y, v->aniso};
    if (n) {
        for (int k = 0; k < 10; k++)
            ck(cudaMemcpyAsync(dst[k], ws.params.p + static_cast<size_t>(k) * ws.cap, n * 8, cudaMemcpyDeviceToHost,
                               ws.stream),
               "D2H sites");
        ck(cudaMemcpyAsync(v->active, ws.active.p, n, cudaMemcpyDeviceToHost, ws.stream), "D2H active");
        ck(cudaMemcpyAsync(v->frozen, ws.frozen.p, n, cudaMemcpyDeviceToHost, ws.stream), "D2H frozen");
    }
    ck(cudaStreamSynchronize(ws.stream), "sync");
    v->size = n;
}

void check_field(const sad_field_view* f) {
    if (!f) fail(SAD_EINVAL, "null field view");
    if (f->gw < 1 || f->gh < 1) fail(SAD_EINVAL, "candidate field not sized");
    if (f->k < 1 || f->k > 16) fail(SAD_EINVAL, "CandidateField: k out of range");
    if (f->cell < 1) fail(SAD_EINVAL, "CandidateField: bad cell size");
}

void upload_field(Workspace& ws, const sad_field_view* f) {
    check_field(f);
    ws.ensure_field(f->width, f->height, f->k, f->cell);
    size_t n = static_cast<size_t>(f->gw) * f->gh * f->k;
    ws.cur = 0;
    ck(cudaMemcpyAsync(ws.ids[0].p, f->ids, n * 4, cudaMemcpyHostToDevice, ws.stream), "H2D field");
}

void download_field(Workspace& ws, sad_field_view* f) {
    size_t n = static_cast<size_t>(f->gw) * f->gh * f->k;
    ck(cudaMemcpyAsync(f->ids, ws.ids[ws.cur].p, n * 4, cudaMemcpyDeviceToHost, ws.stream), "D2H field");
    ck(cudaStreamSynchronize(ws.stream), "sync");
}

void upload_target(Workspace& ws, const double* rgb, int w, int h) {
    size_t n = 3 * static_cast<size_t>(w) * h;
    ws.ensure_target(n / 3);
    ck(cudaMemcpyAsync(ws.tgt_d.p, rgb, n * 8, cudaMemcpyHostToDevice, ws.stream), "H2D target");
    sadk::launch_f64_to_f32(ws.tgt_d.p, ws.tgt_f.p, n, ws.stream);
}

void check_synced(const sad_sites_view* s, const sad_field_view* f) {
    if (f->synced_generation != s->generation) fail(SAD_ESTALE, "candidate field is stale for this store");
    if (f->gw < 1 || f->gh < 1) fail(SAD_EINVAL, "candidate field not sized");
}

void check_err(Workspace& ws, const char* what) {
    DevState s = ws.get_state();
    if (s.err & 1) {
        ws.zero_state_field(offsetof(DevState, err), sizeof(int32_t));
        fail(SAD_EEMPTY, std::string(what) + ": empty candidate list at a pixel");
    }
    if (s.err & 2) {
        ws.zero_state_field(offsetof(DevState, err), sizeof(int32_t));
        fail(SAD_ENOMEM, std::string(what) + ": site capacity exhausted");
    }
}

// ------------------------------------------------------------------ stream-ordered operations
// Propagation passes on the device field starting from ids[cur]; pass i uses pass index
// st->pass_index + pass_base + i.  Tables must already hold the packed snapshot.
void passes_device(Workspace& ws, const std::vector<sad_pass_spec>& seq, int inject, uint64_t seed, bool fp64,
                   uint32_t pass_base) {
    double scale = norm_scale(ws.fd.width, ws.fd.height);
    for (size_t i = 0; i < seq.size(); i++) {
        sadk::launch_propagate(fp64, ws.ids[ws.cur].p, ws.ids[1 - ws.cur].p, ws.pack.p, ws.act.p, ws.st.p, ws.fd,
                               seq[i].step, seq[i].stencil, inject, seed, pass_base + static_cast<uint32_t>(i), scale,
                               ws.stream);
        ws.cur = 1 - ws.cur;
    }
}

void build_tables(Workspace& ws, bool fp64, bool pack, bool gtab, bool rtab) {
    sadk::launch_tables(fp64, ws.sites(), ws.st.p, norm_scale(ws.fd.width, ws.fd.height), pack ? ws.pack.p : nullptr,
                        gtab ? ws.gtab.p : nullptr, rtab ? (fp64 ? ws.rtab_d.p : ws.rtab.p) : nullptr, ws.stream);
}

// ------------------------------------------------------------------ tau_diffusion (train.cpp:171-213)
// Sizes are fixed per (W, H, k, capacity): W*H*k edge keys of 2*nb bits, with nb such that every
// valid id is below the all-ones id field.  Everything stays on the stream (graph capturable).
void ensure_tau(Workspace& ws) {
    auto& tb = ws.tb;
    const size_t np = static_cast<size_t>(ws.fd.width) * ws.fd.height;
    const size_t ne = np * static_cast<size_t>(ws.fd.k);
    int nb = 1;
    while (nb < 32 && ((1ull << nb) - 1) < static_cast<unsigned long long>(ws.cap)) nb++;
    if (tb.ne == ne && tb.nb == nb && tb.tcap == ws.cap) return;
    if (ne > static_cast<size_t>(INT32_MAX)) fail(SAD_EINVAL, "tau_diffusion: too many edges");
    tb.k0.ensure(ne);
    tb.k1.ensure(ne);
    tb.owner.ensure(np);
    tb.count.ensure(1);
    tb.tot.ensure(10 * static_cast<size_t>(ws.cap));
    tb.g0.ensure(ws.cap);
    size_t b1 = 0, b2 = 0;
    ck(cub::DeviceRadixSort::SortKeys(nullptr, b1, tb.k0.p, tb.k1.p, static_cast<int>(ne), 0, 2 * nb, ws.stream),
       "tau sort size");
    ck(cub::DeviceSelect::Unique(nullptr, b2, tb.k1.p, tb.k0.p, tb.count.p, static_cast<int>(ne), ws.stream),
       "tau unique size");
    tb.tmp_bytes = std::max<size_t>(std::max(b1, b2), 16);
    tb.tmp.ensure(tb.tmp_bytes);
    tb.ne = ne;
    tb.nb = nb;
    tb.tcap = ws.cap;
}

// Owner map (render_id_map, double ScoreTable) -> edge keys -> radix sort -> unique -> per-owner mix
// into out[] (non-owners keep what out already holds).  g0 is the logtau column before mixing.
void tau_device(Workspace& ws, double lambda, double* out, const double* g0) {
    auto& tb = ws.tb;
    build_tables(ws, true, false, false, true);
    sadk::launch_id_map(ws.ids[ws.cur].p, ws.rtab_d.p, ws.fd, norm_scale(ws.fd.width, ws.fd.height), tb.owner.p,
                        ws.st.p, ws.stream);
    sadk::launch_tau_edges(ws.ids[ws.cur].p, tb.owner.p, ws.active.p, ws.fd, tb.nb, tb.k0.p, ws.stream);
    size_t bytes = tb.tmp_bytes;
    ck(cub::DeviceRadixSort::SortKeys(tb.tmp.p, bytes, tb.k0.p, tb.k1.p, static_cast<int>(tb.ne), 0, 2 * tb.nb,
                                      ws.stream),
       "tau sort");
    bytes = tb.tmp_bytes;
    ck(cub::DeviceSelect::Unique(tb.tmp.p, bytes, tb.k1.p, tb.k0.p, tb.count.p, static_cast<int>(tb.ne), ws.stream),
       "tau unique");
    sadk::launch_tau_mix(tb.k0.p, tb.count.p, static_cast<int>(tb.ne), tb.nb, g0, lambda, out, ws.stream);
}

sadk::AdamHyper adam_hyper(const sad_train_config& c, int w, int h) {
    sadk::AdamHyper hp{};
    const double lrs[10] = {c.lr_pos,   c.lr_pos,   c.lr_log_tau, c.lr_radius, c.lr_color,
                            c.lr_color, c.lr_color, c.lr_dir,     c.lr_dir,    c.lr_aniso};
    for (int i = 0; i < 10; i++) hp.lr[i] = lrs[i];
    hp.beta1 = c.beta1;
    hp.beta2 = c.beta2;
    hp.eps = c.adam_eps;
    hp.log_tau_min = c.log_tau_min;
    hp.log_tau_max = c.log_tau_max;
    hp.radius_min = c.radius_min;
    hp.radius_max = c.radius_max;
    hp.aniso_min = c.aniso_min;
    hp.aniso_max = c.aniso_max;
    hp.clamp_color = c.clamp_color;
    hp.width = w;
    hp.height = h;
    return hp;
}

// accumulate_stats on the device.  from_grads: the gradient record counts of this pass are still live (the
// resident fit's event iterations, between the backward and Adam), so the stats records get a planned
// per-site layout instead of the fixed 16 slots + linked overflow records (long chains at 8x8 tiles).
void stats_device(Workspace& ws, bool from_grads = false) {
    build_tables(ws, true, false, false, true);
    ws.zero_red(false);
    ws.zero_state_field(offsetof(DevState, valid), sizeof(uint64_t));
    sadk::RedTarget red = ws.sred();
    if (from_grads && ws.apsize > 0) {
        const long long want = ws.apsize;  // >= the gradient records of a pass, typically 2-4x them
        if (ws.spsize < want || !ws.spool.p) {
            ws.spool.ensure(static_cast<size_t>(want) * 8);
            ws.spsize = want;
        }
        ws.sroff.ensure(ws.cap);
        ws.srcap.ensure(ws.cap);
        sadk::launch_stats_plan(ws.gcnt.p, ws.st.p, ws.cap, ws.srcap.p, ws.stream);
        size_t bytes = ws.cub_tmp.n;
        ck(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, bytes, ws.srcap.p, ws.sroff.p, ws.cap, ws.stream), "DeviceScan");
        red = ws.sred_adaptive();
    }
    sadk::launch_stats(ws.ids[ws.cur].p, ws.rtab_d.p, ws.tgt_d.p, ws.fd, norm_scale(ws.fd.width, ws.fd.height), red,
                       ws.st.p, ws.stream);
    sadk::launch_finalize(red, 8, ws.st.p, ws.stream);
}

void prune_device(Workspace& ws, double pct) {
    ws.zero_state_field(offsetof(DevState, n_elig), sizeof(int32_t));
    ws.zero_state_field(offsetof(DevState, done), sizeof(int32_t));
    if (pct <= 0) return;
    sadk::launch_prune_keys(ws.sites(), ws.st.p, ws.stats.p, ws.cap, ws.keys[0].p, ws.vals[0].p, ws.stream);
    ws.sort_pairs(ws.cap);
    sadk::launch_prune_apply(ws.sites(), ws.st.p, ws.vals[1].p, pct, ws.stream);
}

void densify_device(Workspace& ws, double pct, const sad_train_config& c) {
    ws.zero_state_field(offsetof(DevState, n_elig), sizeof(int32_t));
    ws.zero_state_field(offsetof(DevState, done), sizeof(int32_t));
    if (pct <= 0) return;
    sadk::launch_densify_keys(ws.sites(), ws.st.p, ws.stats.p, ws.cap, c.alpha, c.stats_eps, ws.keys[0].p,
                              ws.vals[0].p, ws.flags.p, ws.stream);
    {
        size_t bytes = ws.cub_tmp.n;
        thrust::counting_iterator<uint32_t> it(0);
        ck(cub::DeviceSelect::Flagged(ws.cub_tmp.p, bytes, it, ws.flags.p, ws.free_list.p, &ws.st.p->n_free, ws.cap,
                                      ws.stream),
           "DeviceSelect free");
    }
    ws.sort_pairs(ws.cap);
    sadk::SplitHyper hp{c.log_tau_min, c.radius_min, c.aniso_min, c.aniso_max, ws.fd.width, ws.fd.height, c.max_sites};
    sadk::launch_densify_apply(ws.sites(), ws.st.p, ws.stats.p, ws.cap, ws.vals[1].p, ws.free_list.p, ws.tgt_d.p, pct,
                               hp, ws.m.p, ws.v.p, ws.stream);
}

// Scratch for init_sites_device, allocated once per image size.
void ensure_init_bufs(Workspace& ws, int w, int h, int n) {
    auto& b = ws.ib;
    size_t np = static_cast<size_t>(w) * h;
    if (b.np < np) {
        b.mag.ensure(np);
        b.gsum.ensure(1);
        b.k0.ensure(np);
        b.k1.ensure(np);
        b.v0.ensure(np);
        b.v1.ensure(np);
        b.fl.ensure(np);
        b.nsel.ensure(1);
        b.jk.ensure(np / 64 + 2);
        size_t a = 0, c = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, a, b.k0.p, b.k1.p, b.v0.p, b.v1.p, static_cast<int>(np), 0, 64,
                                        ws.stream);
        thrust::counting_iterator<uint32_t> it(0);
        cub::DeviceSelect::Flagged(nullptr, c, it, b.fl.p, b.v1.p, b.nsel.p, static_cast<int>(np), ws.stream);
        b.tmp.ensure(std::max(a, c) + 256);
        b.np = np;
    }
    b.cells.ensure(static_cast<size_t>(n));
    b.jo.ensure(static_cast<size_t>(n) / 32 + 2);
}

// init_sites (train.cpp:59-111) on the device.
void init_sites_device(Workspace& ws, int w, int h, int n, const sad_train_config& c) {
    size_t np = static_cast<size_t>(w) * h;
    if (n < 1 || static_cast<size_t>(n) > np) fail(SAD_EINVAL, "init_sites: count out of range");
    if (n > ws.cap) fail(SAD_ENOMEM, "init_sites: capacity");
    ensure_init_bufs(ws, w, h, n);
    auto& b = ws.ib;
    sadk::launch_sobel(ws.tgt_d.p, w, h, b.mag.p, ws.stream);
    ck(cudaMemsetAsync(b.gsum.p, 0, sizeof(double2), ws.stream), "memset");
    sadk::launch_dd_sum(b.mag.p, np, b.gsum.p, ws.stream);
    const int chunk = 64;
    auto js = jump_states(seeded_state(c.seed, 0x1717, 0), chunk, (np + chunk - 1) / chunk);
    ck(cudaMemcpyAsync(b.jk.p, js.data(), js.size() * 4, cudaMemcpyHostToDevice, ws.stream), "H2D jump");
    sadk::launch_init_keys(b.mag.p, w, h, b.gsum.p, c.lambda_init, b.jk.p, chunk, b.k0.p, b.v0.p, ws.stream);
    size_t bytes = b.tmp.n;
    ck(cub::DeviceRadixSort::SortPairs(b.tmp.p, bytes, b.k0.p, b.k1.p, b.v0.p, b.v1.p, static_cast<int>(np), 0, 64,
                                       ws.stream),
       "init sort");
    ck(cudaMemsetAsync(b.fl.p, 0, np, ws.stream), "memset");
    sadk::launch_mark_cells(b.v1.p, n, b.fl.p, ws.stream);
    bytes = b.tmp.n;
    thrust::counting_iterator<uint32_t> it(0);
    ck(cub::DeviceSelect::Flagged(b.tmp.p, bytes, it, b.fl.p, b.cells.p, b.nsel.p, static_cast<int>(np), ws.stream),
       "init select");
    const int chunk2 = 32;
    auto jo_h = jump_states(seeded_state(c.seed, 0x1717, 1), 2 * chunk2, (n + chunk2 - 1) / chunk2);
    ck(cudaMemcpyAsync(b.jo.p, jo_h.data(), jo_h.size() * 4, cudaMemcpyHostToDevice, ws.stream), "H2D jump");
    double r0 = c.init_radius > 0 ? c.init_radius : std::sqrt(static_cast<double>(w) * h / static_cast<double>(n));
    sadk::launch_init_sites(ws.sites(), ws.st.p, b.cells.p, n, ws.tgt_d.p, w, h, r0, c.init_log_tau, c.init_aniso,
                            b.jo.p, chunk2, ws.stream);
}

}  // namespace

// ====================================================================== context
// Device-resident SiteStore / CandidateField of a context: uploaded once, used by the
// per-call functions when they get NULL views, downloaded on request.  A call with a host view
// replaces the workspace copy and so invalidates the corresponding resident object.
struct Resident {
    bool sites = false, field = false;
    size_t n = 0, capacity = 0;
    uint64_t generation = 0;
    sad_field_view fmeta{};  // ids unused
};

struct sad_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own = false;
    Workspace ws;
    uint64_t launches0 = 0;
    Resident res;
};

// Resolve a sites argument: a host view is uploaded; NULL selects the resident store (its size and
// generation are returned through `meta` for the staleness checks).
static const sad_sites_view* sites_arg(sad_ctx* c, const sad_sites_view* s, sad_sites_view& meta, int extra_cap = 0) {
    if (s) {
        upload_sites(c->ws, s, extra_cap);
        c->res.sites = false;
        return s;
    }
    if (!c->res.sites) fail(SAD_EINVAL, "no resident sites: pass a view or call sad_sites_upload first");
    if (extra_cap > 0) c->ws.ensure_cap(static_cast<int>(c->res.n) + extra_cap);
    meta = sad_sites_view{};
    meta.size = c->res.n;
    meta.capacity = c->res.capacity;
    meta.generation = c->res.generation;
    return &meta;
}

// Resolve a field argument: a host view is (optionally) uploaded; NULL selects the resident field.
static sad_field_view* field_arg(sad_ctx* c, sad_field_view* f, bool upload);
static const sad_field_view* field_arg(sad_ctx* c, const sad_field_view* f) {
    return field_arg(c, const_cast<sad_field_view*>(f), true);
}
static sad_field_view* field_arg(sad_ctx* c, sad_field_view* f, bool upload) {
    if (f) {
        check_field(f);
        if (upload) upload_field(c->ws, f);
        c->res.field = false;
        return f;
    }
    if (!c->res.field) fail(SAD_EINVAL, "no resident field: pass a view or call sad_field_upload / sad_field_alloc");
    return &c->res.fmeta;
}

struct sad_fit_run {
    sad_ctx* ctx = nullptr;
    int w = 0, h = 0;
    sad_train_config cfg{};
    Workspace ws;
    bool have_target = false;
    bool done = false;
    std::vector<sad_history_row> hist;
    double schedule_scale = 0;
    size_t n_sites = 0;
    double total_ms = 0;
    double phase_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    DBuf<double2> loss_hist;
    DBuf<int32_t> active_hist;
    DBuf<double2> bc_table;
    bool bc_ready = false;
    int planned_n0 = -1;  // plan_schedule is a pure function of (n0, target, cfg): cached
    double planned_scale = 0;
    // CUDA graphs of runs of n plain iterations, keyed by (field buffer parity, warm refresh flag, n);
    // value: the executable graph and the kernel launches it holds
    std::map<int, std::pair<cudaGraphExec_t, uint64_t>> plain;
    uint64_t graph_epoch = ~0ull;  // g_alloc_epoch when the cached graphs were captured
    sad_train_config graph_cfg{};  // and the config whose scalars they hold
    void drop_graphs() {
        for (auto& g : plain)
            if (g.second.first) cudaGraphExecDestroy(g.second.first);
        plain.clear();
    }
    bool profile = false;  // per-phase CUDA-event timing (disables graphs)
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    // row-strip multi-GPU fit (config 5): this run's rank, the world size, every rank's first row
    // (world + 1 bounds), and the buffers of the exact cross-rank merges
    int rank = 0, world = 1;
    std::vector<int> strip;
    DBuf<double2> gpart_self, loss_self, loss_all;
    DBuf<double> tot;
    DBuf<unsigned long long> valid_all;
    // owner-merged exchange: per-destination record counts (and the gathered R x R matrix), send /
    // receive records, the owned range of the active list, parameter / stats slice staging
    DBuf<unsigned long long> own_counts, own_matrix;
    DBuf<sadk::OwnRec> own_send, own_recv;
    DBuf<sadk::OwnRec> ord_send, ord_recv;  // fp64 reference-order strips: tagged records
    DBuf<int32_t> own_range;
    DBuf<double> slice_p, slice_all_p;
    DBuf<double2> slice_s, slice_all_s;
    long long xfer_records = 0;  // gradient records this rank sent to owners over the fit
    ~sad_fit_run() {
        drop_graphs();
    }
};

// plain iterations per graph launch (SAD_GRAPH_ITERS overrides; 1 = one graph per iteration)
static const int g_graph_iters = getenv("SAD_GRAPH_ITERS") ? std::max(1, atoi(getenv("SAD_GRAPH_ITERS"))) : 8;

extern "C" {

const char* sad_last_error(void) { return g_err.c_str(); }
void sad_internal_set_error(const char* msg) { g_err = msg; }
int sad_abi_version(void) { return SAD_ABI_VERSION; }

void sad_default_config(sad_train_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->iters = 4000; c->n_sites = 0; c->target_bpp = 0; c->seed = 1; c->k = 8; c->inject = 4; c->lambda_init = 0.3;
    c->lr_pos = 0.5; c->lr_color = 0.05; c->lr_log_tau = 0.05; c->lr_radius = 0.25; c->lr_dir = 0.025;
    c->lr_aniso = 0.025; c->beta1 = 0.9; c->beta2 = 0.999; c->adam_eps = 1e-8;
    c->refresh_every = 1; c->refresh_passes = 1; c->final_passes = 16; c->tau_diffusion_lambda = 0.0;
    c->densify_every = 20; c->densify_start = 20; c->densify_end = 3000; c->densify_pct = 0.01; c->alpha = 0.7;
    c->stats_eps = 1e-8; c->prune_every = 40; c->prune_start = 100; c->prune_end = 3000; c->prune_pct = 0.033;
    c->prune_during_densify = 1; c->budget_scale_cap = 0.95; c->max_sites = 0;
    c->init_log_tau = 7.5; c->init_radius = 0; c->init_aniso = 0;
    c->log_tau_min = 2.0; c->log_tau_max = 20.0; c->radius_min = 1.0; c->radius_max = 512.0;
    c->aniso_min = -2.0; c->aniso_max = 2.0; c->clamp_color = 1; c->fp64 = 1; c->threads = 1;
}

sad_status sad_ctx_create(int device, void* stream, sad_ctx** out) {
    return guard([&] {
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) fail(SAD_ECUDA, "no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10) fail(SAD_ECUDA, "libsad_b200 is built for sm_100a (B200); device is sm_" +
                                                  std::to_string(prop.major) + std::to_string(prop.minor));
        auto* c = new sad_ctx();
        g_cuda_used = true;
        c->device = device;
        if (stream) {
            c->stream = static_cast<cudaStream_t>(stream);
        } else {
            ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            c->own = true;
        }
        c->ws.stream = c->stream;
        sadk::prepare_kernels();
        c->ws.ensure_state();
        c->launches0 = sadk::launch_counter();
        *out = c;
    });
}

void sad_ctx_destroy(sad_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    cudaStream_t s = c->stream;
    bool own = c->own;
    delete c;
    if (own) cudaStreamDestroy(s);
}

sad_status sad_ctx_synchronize(sad_ctx* c) {
    return guard([&] { ck(cudaStreamSynchronize(c->stream), "sync"); });
}

long long sad_debug_check_failures(void) { return sadk::debug_check_failures(); }

uint64_t sad_ctx_launch_count(const sad_ctx* c) { return sadk::launch_counter() - (c ? c->launches0 : 0); }

// ====================================================================== candidates
// ====================================================================== device-resident objects
sad_status sad_sites_alloc(sad_ctx* c, size_t capacity) {
    return guard([&] {
        if (capacity > static_cast<size_t>(INT32_MAX / 2)) fail(SAD_EINVAL, "too many sites");
        c->ws.ensure_cap(static_cast<int>(std::max<size_t>(capacity, 1)));
        c->ws.patch_state(offsetof(DevState, n_sites), 0);
        c->res.sites = true;
        c->res.n = 0;
        c->res.capacity = capacity;
        c->res.generation = 0;
    });
}

sad_status sad_sites_upload(sad_ctx* c, const sad_sites_view* s) {
    return guard([&] {
        if (!s) fail(SAD_EINVAL, "null sites view");
        upload_sites(c->ws, s, static_cast<int>(s->capacity > s->size ? s->capacity - s->size : 0));
        c->res.sites = true;
        c->res.n = s->size;
        c->res.capacity = std::max(s->capacity, s->size);
        c->res.generation = s->generation;
    });
}

sad_status sad_sites_download(sad_ctx* c, sad_sites_view* s) {
    return guard([&] {
        if (!s) fail(SAD_EINVAL, "null sites view");
        if (!c->res.sites) fail(SAD_EINVAL, "no resident sites");
        download_sites(c->ws, s, c->res.n);
        s->generation = c->res.generation;
    });
}

sad_status sad_sites_info(sad_ctx* c, size_t* size, size_t* capacity, uint64_t* generation) {
    return guard([&] {
        if (!c->res.sites) fail(SAD_EINVAL, "no resident sites");
        if (size) *size = c->res.n;
        if (capacity) *capacity = c->res.capacity;
        if (generation) *generation = c->res.generation;
    });
}

sad_status sad_field_alloc(sad_ctx* c, int width, int height, int k, int cell) {
    return guard([&] {
        if (width < 1 || height < 1) fail(SAD_EINVAL, "CandidateField: empty image");
        if (k < 1 || k > 16) fail(SAD_EINVAL, "CandidateField: k out of range");
        if (cell < 1) fail(SAD_EINVAL, "CandidateField: bad cell size");
        Workspace& ws = c->ws;
        ws.ensure_field(width, height, k, cell);
        ws.cur = 0;
        const size_t n = static_cast<size_t>(ws.fd.gw) * ws.fd.gh * k;
        ck(cudaMemsetAsync(ws.ids[0].p, 0xff, 4 * n, ws.stream), "memset field");
        sad_field_view& m = c->res.fmeta;  // CandidateField::resize (types.cpp:89-101)
        m = sad_field_view{};
        m.width = width;
        m.height = height;
        m.cell = cell;
        m.gw = ws.fd.gw;
        m.gh = ws.fd.gh;
        m.k = k;
        m.synced_generation = ~0ull;
        c->res.field = true;
    });
}

sad_status sad_field_upload(sad_ctx* c, const sad_field_view* f) {
    return guard([&] {
        upload_field(c->ws, f);
        c->res.fmeta = *f;
        c->res.fmeta.ids = nullptr;
        c->res.field = true;
    });
}

sad_status sad_field_download(sad_ctx* c, sad_field_view* f) {
    return guard([&] {
        if (!f) fail(SAD_EINVAL, "null field view");
        if (!c->res.field) fail(SAD_EINVAL, "no resident field");
        const sad_field_view& m = c->res.fmeta;
        f->width = m.width;
        f->height = m.height;
        f->cell = m.cell;
        f->gw = m.gw;
        f->gh = m.gh;
        f->k = m.k;
        if (f->ids) download_field(c->ws, f);  // ids == NULL: metadata only
        f->synced_generation = m.synced_generation;
        f->refresh_count = m.refresh_count;
        f->pass_index = m.pass_index;
    });
}

sad_status sad_math_exp(sad_ctx* c, const double* x, double* y, size_t n, int single) {
    return guard([&] {
        DBuf<double> dx, dy;
        dx.ensure(std::max<size_t>(n, 1));
        dy.ensure(std::max<size_t>(n, 1));
        ck(cudaMemcpyAsync(dx.p, x, 8 * n, cudaMemcpyHostToDevice, c->stream), "H2D");
        sadk::launch_math(dx.p, dy.p, n, single, c->stream);  // 0 exp, 1 expf, 2 log
        ck(cudaMemcpyAsync(y, dy.p, 8 * n, cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaStreamSynchronize(c->stream), "math");
    });
}

sad_status sad_jump_step(uint32_t t, uint32_t b, uint32_t* out) {
    return guard([&] { *out = jump_step(t, b); });
}

sad_status sad_full_refresh_passes(int gw, int gh, int extra, sad_pass_spec* out, int* n) {
    return guard([&] {
        auto seq = full_refresh_passes(gw, gh, extra);
        if (static_cast<int>(seq.size()) > *n) fail(SAD_EINVAL, "pass buffer too small");
        std::copy(seq.begin(), seq.end(), out);
        *n = static_cast<int>(seq.size());
    });
}

sad_status sad_schedule_passes(int gw, int gh, int total, sad_pass_spec* out, int* n) {
    return guard([&] {
        auto seq = schedule_passes(gw, gh, total);
        if (static_cast<int>(seq.size()) > *n) fail(SAD_EINVAL, "pass buffer too small");
        std::copy(seq.begin(), seq.end(), out);
        *n = static_cast<int>(seq.size());
    });
}

sad_status sad_jfa_seed(sad_ctx* c, const sad_sites_view* s_in, sad_field_view* f_in) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        sad_field_view* f = field_arg(c, f_in, false);
        ws.ensure_field(f->width, f->height, f->k, f->cell);
        ws.cur = 0;
        sadk::launch_jfa_seed(ws.sites(), ws.st.p, ws.ids[0].p, ws.fd, norm_scale(f->width, f->height), ws.stream);
        if (f_in) download_field(ws, f);
        f->synced_generation = s->generation;
    });
}

static void run_passes_call(sad_ctx* c, const sad_sites_view* s_in, sad_field_view* f_in,
                            const std::vector<sad_pass_spec>& seq, int inject, uint64_t seed, int fp64, bool full) {
    Workspace& ws = c->ws;
    sad_sites_view sm;
    const sad_sites_view* s = sites_arg(c, s_in, sm);
    sad_field_view* f = field_arg(c, f_in, !full);
    if (full) {
        ws.ensure_field(f->width, f->height, f->k, f->cell);
        ws.cur = 0;
        sadk::launch_jfa_seed(ws.sites(), ws.st.p, ws.ids[0].p, ws.fd, norm_scale(f->width, f->height), ws.stream);
    }
    ws.patch_state(offsetof(DevState, pass_index), f->pass_index);
    ws.compute_active();
    build_tables(ws, fp64 != 0, true, false, false);
    passes_device(ws, seq, inject, seed, fp64 != 0, 0);
    if (f_in) download_field(ws, f);
    f->pass_index += static_cast<uint32_t>(seq.size());
    f->synced_generation = s->generation;
}

sad_status sad_run_passes(sad_ctx* c, const sad_sites_view* s, sad_field_view* f, const sad_pass_spec* seq, int n_pass,
                          int inject, uint64_t seed, int fp64) {
    return guard([&] {
        std::vector<sad_pass_spec> v(seq, seq + std::max(n_pass, 0));
        run_passes_call(c, s, f, v, inject, seed, fp64, false);
    });
}

sad_status sad_refresh(sad_ctx* c, const sad_sites_view* s, sad_field_view* f_in, int mode, int passes, int inject,
                       uint64_t seed, int fp64) {
    return guard([&] {
        sad_field_view* f = f_in ? f_in : field_arg(c, nullptr, false);
        if (f_in) check_field(f_in);
        if (mode == SAD_REFRESH_FULL) {
            run_passes_call(c, s, f_in, full_refresh_passes(f->gw, f->gh, passes), inject, seed, fp64, true);
        } else {
            std::vector<sad_pass_spec> v(static_cast<size_t>(passes < 0 ? 0 : passes), sad_pass_spec{1, 0});
            run_passes_call(c, s, f_in, v, inject, seed, fp64, false);
        }
        f->refresh_count++;
    });
}

sad_status sad_exact_topk_batch(sad_ctx* c, const sad_sites_view* s, const int32_t* xy, size_t n_pix, int k,
                                double scale, int fp64, uint32_t* out) {
    return guard([&] {
        if (k < 1 || k > 16) fail(SAD_EINVAL, "exact_topk: k out of range");
        Workspace& ws = c->ws;
        sad_sites_view sm;
        sites_arg(c, s, sm);
        ws.compute_active();
        // tables use the probe scale supplied by the caller
        sadk::launch_tables(fp64 != 0, ws.sites(), ws.st.p, scale, nullptr, nullptr, fp64 ? ws.rtab_d.p : ws.rtab.p,
                            ws.stream);
        DevState st = ws.get_state();
        DBuf<int32_t> dxy;
        DBuf<uint32_t> dout;
        dxy.ensure(2 * n_pix);
        dout.ensure(n_pix * k);
        ck(cudaMemcpyAsync(dxy.p, xy, 8 * n_pix, cudaMemcpyHostToDevice, ws.stream), "H2D");
        sadk::launch_exact_topk(fp64 != 0, fp64 ? ws.rtab_d.p : ws.rtab.p, ws.act.p, st.n_active, dxy.p,
                                static_cast<int>(n_pix), k, scale, dout.p, ws.stream);
        ck(cudaMemcpyAsync(out, dout.p, 4 * n_pix * k, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        ck(cudaStreamSynchronize(ws.stream), "sync");
    });
}

// ====================================================================== render
sad_status sad_render_image(sad_ctx* c, const sad_sites_view* s_in, const sad_field_view* f_in, int fp64, double* out) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        const sad_field_view* f = field_arg(c, f_in);
        check_synced(s, f);
        build_tables(ws, fp64 != 0, false, false, true);
        size_t n = 3 * static_cast<size_t>(f->width) * f->height;
        if (fp64) {
            ws.px_d.ensure(n);
            sadk::launch_render(true, ws.ids[ws.cur].p, ws.rtab_d.p, ws.fd, norm_scale(f->width, f->height), ws.px_d.p,
                                ws.st.p, ws.stream);
            ck(cudaMemcpyAsync(out, ws.px_d.p, n * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H render");
            check_err(ws, "render");
        } else {
            ws.px_f.ensure(n);
            sadk::launch_render(false, ws.ids[ws.cur].p, ws.rtab.p, ws.fd, norm_scale(f->width, f->height), ws.px_f.p,
                                ws.st.p, ws.stream);
            std::vector<float> tmp(n);
            ck(cudaMemcpyAsync(tmp.data(), ws.px_f.p, n * 4, cudaMemcpyDeviceToHost, ws.stream), "D2H render");
            check_err(ws, "render");
            for (size_t i = 0; i < n; i++) out[i] = tmp[i];
        }
    });
}

sad_status sad_pixel_weights(sad_ctx* c, const sad_sites_view* s_in, const sad_field_view* f_in, const int32_t* xy,
                             size_t n_q, uint32_t* ids, double* w, int32_t* n) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        const sad_field_view* f = field_arg(c, f_in);
        check_synced(s, f);
        for (size_t q = 0; q < n_q; q++)
            if (xy[2 * q] < 0 || xy[2 * q + 1] < 0 || xy[2 * q] >= f->width || xy[2 * q + 1] >= f->height)
                fail(SAD_EINVAL, "pixel_weights: pixel out of bounds");
        build_tables(ws, true, false, false, true);
        DBuf<int32_t> dxy, dn;
        DBuf<uint32_t> did;
        DBuf<double> dw;
        dxy.ensure(2 * n_q);
        dn.ensure(n_q);
        did.ensure(16 * n_q);
        dw.ensure(16 * n_q);
        ck(cudaMemcpyAsync(dxy.p, xy, 8 * n_q, cudaMemcpyHostToDevice, ws.stream), "H2D");
        sadk::launch_pixel_weights(ws.ids[ws.cur].p, ws.rtab_d.p, ws.fd, norm_scale(f->width, f->height), dxy.p,
                                   static_cast<int>(n_q), did.p, dw.p, dn.p, ws.stream);
        ck(cudaMemcpyAsync(ids, did.p, 64 * n_q, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        ck(cudaMemcpyAsync(w, dw.p, 128 * n_q, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        ck(cudaMemcpyAsync(n, dn.p, 4 * n_q, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        ck(cudaStreamSynchronize(ws.stream), "sync");
        for (size_t q = 0; q < n_q; q++)
            if (n[q] == 0) fail(SAD_EEMPTY, "pixel_weights: empty candidate list");
    });
}

sad_status sad_render_id_map(sad_ctx* c, const sad_sites_view* s_in, const sad_field_view* f_in, uint32_t* out) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        const sad_field_view* f = field_arg(c, f_in);
        check_synced(s, f);
        build_tables(ws, true, false, false, true);
        DBuf<uint32_t> d;
        size_t n = static_cast<size_t>(f->width) * f->height;
        d.ensure(n);
        sadk::launch_id_map(ws.ids[ws.cur].p, ws.rtab_d.p, ws.fd, norm_scale(f->width, f->height), d.p, ws.st.p,
                            ws.stream);
        ck(cudaMemcpyAsync(out, d.p, 4 * n, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        check_err(ws, "render");
    });
}

sad_status sad_tau_diffusion(sad_ctx* c, const sad_sites_view* s_in, const sad_field_view* f_in, double lambda,
                             double* grads) {
    return guard([&] {
        if (lambda == 0) return;
        if (lambda < 0 || lambda > 1) fail(SAD_EINVAL, "tau_diffusion: lambda out of [0,1]");
        if (!grads) fail(SAD_EINVAL, "tau_diffusion: null gradient buffer");
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        const sad_field_view* f = field_arg(c, f_in);
        check_synced(s, f);
        ensure_tau(ws);
        const size_t n = s->size;
        std::vector<double> g0(n + 1), o(n + 1);
        for (size_t i = 0; i < n; i++) g0[i] = grads[i * 11 + 2];
        ck(cudaMemcpyAsync(ws.tb.g0.p, g0.data(), 8 * n, cudaMemcpyHostToDevice, ws.stream), "H2D g0");
        ck(cudaMemcpyAsync(ws.tb.tot.p, g0.data(), 8 * n, cudaMemcpyHostToDevice, ws.stream), "H2D g0");
        tau_device(ws, lambda, ws.tb.tot.p, ws.tb.g0.p);
        ck(cudaMemcpyAsync(o.data(), ws.tb.tot.p, 8 * n, cudaMemcpyDeviceToHost, ws.stream), "D2H tau");
        ck(cudaStreamSynchronize(ws.stream), "tau_diffusion");
        check_err(ws, "render");
        for (size_t i = 0; i < n; i++) grads[i * 11 + 2] = o[i];
    });
}

// fp64 per-site gradient sums in the reference's summation order (sadk::fp64_ordered).  The
// record tags hold the reference tile's raster index in 23 bits: beyond 2^23 tiles (an image over ~46k^2
// pixels) the double-double reduction is used.
static bool use_ordered(bool fp64, const sadk::FieldDims& fd) {
    const long long tiles = ((fd.width + 15ll) / 16) * ((fd.height + 15ll) / 16);
    return fp64 && sadk::fp64_ordered() && tiles < (1ll << 23);
}

// ====================================================================== grad
static void backward_call(sad_ctx* c, const sad_sites_view* s_in, const sad_field_view* f_in, const double* img,
                          int fp64, int mode, double* grads, uint64_t* nonfinite, double* loss) {
    Workspace& ws = c->ws;
    sad_sites_view sm;
    const sad_sites_view* s = sites_arg(c, s_in, sm);
    const sad_field_view* f = field_arg(c, f_in);
    check_synced(s, f);
    size_t npx = static_cast<size_t>(f->width) * f->height;
    ws.ensure_target(npx);
    ck(cudaMemcpyAsync(ws.tgt_d.p, img, 24 * npx, cudaMemcpyHostToDevice, ws.stream), "H2D target");
    if (!fp64) sadk::launch_f64_to_f32(ws.tgt_d.p, ws.tgt_f.p, 3 * npx, ws.stream);
    build_tables(ws, fp64 != 0, false, true, false);
    ws.zero_red(true);
    ws.zero_state_field(offsetof(DevState, nonfinite), sizeof(uint64_t));
    ws.zero_state_field(offsetof(DevState, loss), sizeof(double2));
    const bool ordered = use_ordered(fp64 != 0, ws.fd);
    const sadk::RedTarget red = ordered ? ws.gred_ord() : ws.gred();
    sadk::launch_backward(fp64 != 0, mode, ws.ids[ws.cur].p, ws.gtab.p,
                          fp64 ? static_cast<const void*>(ws.tgt_d.p) : static_cast<const void*>(ws.tgt_f.p), ws.fd,
                          norm_scale(f->width, f->height), red, ws.loss_part.p, ws.st.p, ws.stream);
    // channel 10 only with removal
    if (ordered) sadk::launch_ordered_totals(red, mode == 1 ? 11 : 10, ws.st.p, nullptr, nullptr, true, ws.stream);
    else sadk::launch_finalize(red, mode == 1 ? 11 : 10, ws.st.p, ws.stream);
    if (mode != 2)
        sadk::launch_loss_reduce(ws.loss_part.p, sadk::backward_blocks(fp64 != 0, ws.fd, ordered), &ws.st.p->loss,
                                 ws.stream);
    DBuf<double> out;
    size_t n = s->size;
    out.ensure(std::max<size_t>(n, 1) * 11);
    if (n) sadk::launch_scatter_grads_out(ws.grads.p, ws.cap, static_cast<int>(n), out.p, ws.stream);
    if (n) ck(cudaMemcpyAsync(grads, out.p, n * 11 * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H grads");
    DevState st = ws.get_state();
    if (st.err & 8) {
        ws.zero_state_field(offsetof(DevState, err), sizeof(int32_t));
        std::fprintf(stderr, "sad: fp64 ordered reduction: record pools full, some sums merged as double-doubles "
                             "(raise SAD_OCAP)\n");
    }
    if (st.err & 1) {
        ws.zero_state_field(offsetof(DevState, err), sizeof(int32_t));
        fail(SAD_EEMPTY, "backward: empty candidate list at a pixel");
    }
    if (nonfinite) *nonfinite = st.nonfinite;
    if (loss) *loss = (st.loss.x + st.loss.y) / (static_cast<double>(f->width) * f->height);
}

sad_status sad_backward_image(sad_ctx* c, const sad_sites_view* s, const sad_field_view* f, const double* tgt, int fp64,
                              int with_removal, double* grads, uint64_t* nonfinite, double* loss) {
    return guard([&] { backward_call(c, s, f, tgt, fp64, with_removal ? 1 : 0, grads, nonfinite, loss); });
}

sad_status sad_backward_pixel_grad(sad_ctx* c, const sad_sites_view* s, const sad_field_view* f, const double* dl,
                                   int dl_width, int dl_height, int fp64, double* grads, uint64_t* nonfinite) {
    return guard([&] {
        const sad_field_view* fv = field_arg(c, f);
        if (!dl || dl_width != fv->width || dl_height != fv->height)  // grad.cpp:383-384
            fail(SAD_EINVAL, "backward: adjoint size mismatch");
        backward_call(c, s, f, dl, fp64, 2, grads, nonfinite, nullptr);
    });
}

sad_status sad_image_loss(sad_ctx* c, const sad_sites_view* s_in, const sad_field_view* f_in, const double* tgt,
                          int fp64, double* loss) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        const sad_field_view* f = field_arg(c, f_in);
        check_synced(s, f);
        upload_target(ws, tgt, f->width, f->height);
        build_tables(ws, fp64 != 0, false, true, false);
        ws.zero_state_field(offsetof(DevState, loss), sizeof(double2));
        sadk::launch_loss(fp64 != 0, ws.ids[ws.cur].p, ws.gtab.p,
                          fp64 ? static_cast<const void*>(ws.tgt_d.p) : static_cast<const void*>(ws.tgt_f.p), ws.fd,
                          norm_scale(f->width, f->height), ws.loss_part.p, ws.st.p, ws.stream);
        sadk::launch_loss_reduce(ws.loss_part.p, sadk::loss_blocks(ws.fd), &ws.st.p->loss, ws.stream);
        DevState st = ws.get_state();
        if (st.err & 1) {
            ws.zero_state_field(offsetof(DevState, err), sizeof(int32_t));
            fail(SAD_EEMPTY, "loss: empty candidate list at a pixel");
        }
        *loss = (st.loss.x + st.loss.y) / (static_cast<double>(f->width) * f->height);
    });
}

// ====================================================================== train
sad_status sad_adam_step(sad_ctx* c, sad_sites_view* s_in, const double* grads, sad_adam_view* a, int w, int h,
                         const sad_train_config* cfg) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        size_t n = s->size;
        if (a->sites != n && n > a->capacity) fail(SAD_ENOMEM, "adam capacity");
        // grads (n*11 values) -> (hi=value, lo=0) accumulators; moments -> slot-major
        std::vector<double2> g(static_cast<size_t>(11) * ws.cap, make_double2(0, 0));
        std::vector<double> m(static_cast<size_t>(10) * ws.cap, 0.0), v(static_cast<size_t>(10) * ws.cap, 0.0);
        for (size_t id = 0; id < n; id++) {
            for (int k = 0; k < 11; k++) g[k * ws.cap + id] = make_double2(grads[id * 11 + k], 0.0);
            if (id < a->sites)
                for (int k = 0; k < 10; k++) {
                    m[k * ws.cap + id] = a->m[id * 10 + k];
                    v[k * ws.cap + id] = a->v[id * 10 + k];
                }
        }
        ck(cudaMemcpyAsync(ws.grads.p, g.data(), g.size() * sizeof(double2), cudaMemcpyHostToDevice, ws.stream), "H2D");
        ck(cudaMemsetAsync(ws.gcnt.p, 0, sizeof(int32_t) * ws.cap, ws.stream), "memset gcnt");
        ck(cudaMemcpyAsync(ws.m.p, m.data(), m.size() * 8, cudaMemcpyHostToDevice, ws.stream), "H2D");
        ck(cudaMemcpyAsync(ws.v.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, ws.stream), "H2D");
        ws.zero_state_field(offsetof(DevState, skipped), sizeof(uint64_t));
        int64_t t = a->t + 1;
        double2 bc = make_double2(1.0 - std::pow(cfg->beta1, static_cast<double>(t)),
                                  1.0 - std::pow(cfg->beta2, static_cast<double>(t)));
        sadk::launch_adam(false, ws.sites(), ws.st.p, ws.gred(), ws.m.p, ws.v.p, adam_hyper(*cfg, w, h), nullptr, bc,
                          false, 1.0, nullptr, nullptr, nullptr, ws.stream);
        ck(cudaMemcpyAsync(m.data(), ws.m.p, m.size() * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        ck(cudaMemcpyAsync(v.data(), ws.v.p, v.size() * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        DevState st = ws.get_state();
        if (s_in) download_sites(ws, s_in, n);
        for (size_t id = 0; id < n; id++)
            for (int k = 0; k < 10; k++) {
                a->m[id * 10 + k] = m[k * ws.cap + id];
                a->v[id * 10 + k] = v[k * ws.cap + id];
            }
        a->sites = n;
        a->t = t;
        a->skipped += st.skipped;
        // adam_step and clamp_project each bump (train.cpp:167, 136)
        if (s_in) s_in->generation += 2;
        else c->res.generation += 2;
    });
}

sad_status sad_clamp_project(sad_ctx* c, sad_sites_view* s_in, int w, int h, const sad_train_config* cfg) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        sites_arg(c, s_in, sm);
        sadk::launch_clamp(ws.sites(), ws.st.p, adam_hyper(*cfg, w, h), ws.stream);
        if (s_in) {
            download_sites(ws, s_in, s_in->size);
            s_in->generation += 1;
        } else {
            ck(cudaStreamSynchronize(ws.stream), "clamp");
            c->res.generation += 1;
        }
    });
}

sad_status sad_init_sites(sad_ctx* c, sad_sites_view* s, const double* tgt, int w, int h, int n,
                          const sad_train_config* cfg) {
    return guard([&] {
        size_t np = static_cast<size_t>(w) * h;
        if (w < 1 || h < 1) fail(SAD_EINVAL, "init_sites: empty image");
        if (n < 1 || static_cast<size_t>(n) > np) fail(SAD_EINVAL, "init_sites: count out of range");
        if (s && static_cast<size_t>(n) > s->capacity) fail(SAD_ENOMEM, "sites view capacity too small");
        Workspace& ws = c->ws;
        ws.ensure_cap(n);
        upload_target(ws, tgt, w, h);
        init_sites_device(ws, w, h, n, *cfg);
        if (s) {  // host view
            download_sites(ws, s, static_cast<size_t>(n));
            s->generation += 1 + static_cast<uint64_t>(n);
            c->res.sites = false;
        } else {  // into the resident store
            ck(cudaStreamSynchronize(ws.stream), "init_sites");
            c->res.generation += 1 + static_cast<uint64_t>(n);
            c->res.n = static_cast<size_t>(n);
            c->res.capacity = std::max(c->res.capacity, static_cast<size_t>(ws.cap));
            c->res.sites = true;
        }
    });
}

// ====================================================================== budget
sad_status sad_accumulate_stats(sad_ctx* c, const sad_sites_view* s_in, const sad_field_view* f_in,
                                const double* tgt, double* stats, uint64_t* valid) {
    return guard([&] {
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        const sad_field_view* f = field_arg(c, f_in);
        if (f->synced_generation != s->generation) fail(SAD_ESTALE, "stats: candidate field is stale");
        upload_target(ws, tgt, f->width, f->height);
        stats_device(ws);
        size_t n = s->size;
        std::vector<double2> h(static_cast<size_t>(8) * ws.cap);
        ck(cudaMemcpyAsync(h.data(), ws.stats.p, h.size() * sizeof(double2), cudaMemcpyDeviceToHost, ws.stream), "D2H");
        DevState st = ws.get_state();
        for (size_t id = 0; id < n; id++)
            for (int k = 0; k < 8; k++) stats[id * 8 + k] = h[k * ws.cap + id].x + h[k * ws.cap + id].y;
        *valid = st.valid;
    });
}

static void upload_stats(Workspace& ws, const double* stats, size_t n, uint64_t valid) {
    std::vector<double2> h(static_cast<size_t>(8) * ws.cap, make_double2(0, 0));
    for (size_t id = 0; id < n; id++)
        for (int k = 0; k < 8; k++) h[k * ws.cap + id] = make_double2(stats[id * 8 + k], 0.0);
    ck(cudaMemcpyAsync(ws.stats.p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, ws.stream), "H2D");
    ck(cudaMemsetAsync(ws.scnt.p, 0, sizeof(int32_t) * ws.cap, ws.stream), "memset scnt");
    ws.patch_state(offsetof(DevState, valid), valid);
}

sad_status sad_prune(sad_ctx* c, sad_sites_view* s_in, const double* stats, uint64_t valid, double pct,
                     int* removed) {
    return guard([&] {
        *removed = 0;
        if (pct <= 0) return;
        if (pct > 1) fail(SAD_EINVAL, "prune: percentile out of (0,1]");
        Workspace& ws = c->ws;
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm);
        upload_stats(ws, stats, s->size, valid);
        prune_device(ws, pct);
        DevState st = ws.get_state();
        *removed = st.done;
        if (s_in) {
            download_sites(ws, s_in, s_in->size);
            s_in->generation += static_cast<uint64_t>(st.done);
        } else {
            c->res.generation += static_cast<uint64_t>(st.done);
        }
    });
}

sad_status sad_densify(sad_ctx* c, sad_sites_view* s_in, sad_adam_view* a, const double* stats, const double* tgt,
                       int w, int h, double pct, const sad_train_config* cfg, int* done) {
    return guard([&] {
        *done = 0;
        if (pct <= 0) return;
        if (pct > 1) fail(SAD_EINVAL, "densify: percentile out of (0,1]");
        Workspace& ws = c->ws;
        const size_t cap_s = s_in ? s_in->capacity : c->res.capacity;
        size_t n = s_in ? s_in->size : c->res.n;
        int room = static_cast<int>(std::min(cap_s, a->capacity)) - static_cast<int>(n);
        sad_sites_view sm;
        const sad_sites_view* s = sites_arg(c, s_in, sm, std::max(room, 0));
        upload_stats(ws, stats, n, 0);
        upload_target(ws, tgt, w, h);
        std::vector<double> m(static_cast<size_t>(10) * ws.cap, 0.0), v(static_cast<size_t>(10) * ws.cap, 0.0);
        for (size_t id = 0; id < std::min(n, a->sites); id++)
            for (int k = 0; k < 10; k++) {
                m[k * ws.cap + id] = a->m[id * 10 + k];
                v[k * ws.cap + id] = a->v[id * 10 + k];
            }
        ck(cudaMemcpyAsync(ws.m.p, m.data(), m.size() * 8, cudaMemcpyHostToDevice, ws.stream), "H2D");
        ck(cudaMemcpyAsync(ws.v.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, ws.stream), "H2D");
        ws.fd.width = w;
        ws.fd.height = h;
        // densify only ever appends into [n, n + room); slots beyond the caller's capacity flag ENOMEM
        densify_device(ws, pct, *cfg);
        DevState st = ws.get_state();
        if (st.err & 2) {
            ws.zero_state_field(offsetof(DevState, err), sizeof(int32_t));
            fail(SAD_ENOMEM, "densify: sites capacity");
        }
        size_t nn = static_cast<size_t>(st.n_sites);
        if (nn > s->capacity || nn > a->capacity) fail(SAD_ENOMEM, "densify: sites capacity");
        ck(cudaMemcpyAsync(m.data(), ws.m.p, m.size() * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        ck(cudaMemcpyAsync(v.data(), ws.v.p, v.size() * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
        if (s_in) download_sites(ws, s_in, nn);
        else ck(cudaStreamSynchronize(ws.stream), "densify");
        size_t rows = std::max(nn, a->sites);
        for (size_t id = 0; id < rows; id++)
            for (int k = 0; k < 10; k++) {
                a->m[id * 10 + k] = id < nn ? m[k * ws.cap + id] : a->m[id * 10 + k];
                a->v[id * 10 + k] = id < nn ? v[k * ws.cap + id] : a->v[id * 10 + k];
            }
        a->sites = rows;
        *done = st.done;
        if (s_in) {
            s_in->generation += 2 * static_cast<uint64_t>(st.done);
        } else {
            c->res.generation += 2 * static_cast<uint64_t>(st.done);
            c->res.n = nn;
        }
    });
}

sad_status sad_bpp_target_count(double bpp, int w, int h, uint64_t* out) {
    return guard([&] { *out = bpp_target_count(bpp, w, h); });
}

sad_status sad_simulate_schedule(int n0, double scale, const sad_train_config* cfg, int* out) {
    return guard([&] { *out = simulate_schedule(n0, scale, *cfg); });
}

sad_status sad_plan_schedule(int n0, uint64_t target, const sad_train_config* cfg, double* out) {
    return guard([&] { *out = plan_schedule(n0, target, *cfg); });
}

// ====================================================================== resident fit
static int initial_count(const sad_train_config& c, int w, int h);
static int capacity_bound(const sad_train_config& c, int n0, double scale, bool budget);

sad_status sad_fit_create(sad_ctx* c, int w, int h, const sad_train_config* cfg, sad_fit_run** out) {
    return guard([&] {
        sad_train_config v = *cfg;
        validate(v, w, h);
        auto* r = new sad_fit_run();
        try {
            r->ctx = c;
            r->w = w;
            r->h = h;
            r->cfg = v;
            r->ws.stream = c->stream;
            r->ws.ensure_state();
            r->ws.ensure_field(w, h, v.k, 1);
            r->ws.ensure_target(static_cast<size_t>(w) * h);
            // Pre-size everything fit() needs so the run itself never allocates.
            if (v.n_sites > 0 || v.target_bpp > 0) {
                int n0 = initial_count(v, w, h);
                double sched = v.target_bpp > 0 ? plan_schedule(n0, bpp_target_count(v.target_bpp, w, h), v) : 1.0;
                r->planned_n0 = n0;
                r->planned_scale = sched;
                r->ws.ensure_cap(capacity_bound(v, n0, sched, v.target_bpp > 0));
                ensure_init_bufs(r->ws, w, h, n0);
            }
            r->loss_hist.ensure(std::max(v.iters, 1));
            r->active_hist.ensure(std::max(v.iters, 1));
            std::vector<double2> bc(static_cast<size_t>(v.iters) + 2);
            for (int t = 1; t <= v.iters + 1; t++)
                bc[t] = make_double2(1.0 - std::pow(v.beta1, static_cast<double>(t)),
                                     1.0 - std::pow(v.beta2, static_cast<double>(t)));
            r->bc_table.ensure(bc.size());
            ck(cudaMemcpy(r->bc_table.p, bc.data(), bc.size() * sizeof(double2), cudaMemcpyHostToDevice), "H2D bc");
            r->bc_ready = true;
            ck(cudaStreamSynchronize(r->ws.stream), "sync");
        } catch (...) {
            delete r;
            throw;
        }
        *out = r;
    });
}

void sad_fit_destroy(sad_fit_run* r) {
    if (!r) return;
    cudaStreamSynchronize(r->ws.stream);
    delete r;
}

sad_status sad_fit_set_target(sad_fit_run* r, const double* rgb) {
    return guard([&] {
        upload_target(r->ws, rgb, r->w, r->h);
        r->have_target = true;
    });
}

sad_status sad_fit_set_target_device(sad_fit_run* r, const double* drgb) {
    return guard([&] {
        size_t n = 3 * static_cast<size_t>(r->w) * r->h;
        ck(cudaMemcpyAsync(r->ws.tgt_d.p, drgb, n * 8, cudaMemcpyDeviceToDevice, r->ws.stream), "D2D target");
        sadk::launch_f64_to_f32(r->ws.tgt_d.p, r->ws.tgt_f.p, n, r->ws.stream);
        r->have_target = true;
    });
}

static int initial_count(const sad_train_config& c, int w, int h) {
    int n = c.n_sites;
    if (n == 0 && c.target_bpp > 0) {
        uint64_t want = bpp_target_count(c.target_bpp, w, h);
        if (want < 1) fail(SAD_EINVAL, "fit: bpp target below one site");
        size_t n0 = static_cast<size_t>(std::ceil(static_cast<double>(want) * 1.6));
        n = static_cast<int>(std::min(n0, static_cast<size_t>(w) * h));
    }
    if (n < 1) fail(SAD_EINVAL, "fit: site count unset");
    return n;
}

// Upper bound of SiteStore::size over the run: each densify event appends at most
// floor(size * pct * scale) slots (budget.cpp:230, 277).
static int capacity_bound(const sad_train_config& c, int n0, double scale, bool budget) {
    double n = n0;
    if (budget)
        for (int t = 1; t <= c.iters; t++)
            if (t >= c.densify_start && t <= c.densify_end && t % c.densify_every == 0)
                n += std::floor(n * c.densify_pct * std::max(scale, 0.0));
    if (c.max_sites > 0) n = std::min(n, static_cast<double>(std::max<uint64_t>(c.max_sites, n0)));
    return static_cast<int>(n) + 1;
}

// History rows and the end-of-fit checks of a finished run (device loss partials -> HistoryRow).
static void finish_run(sad_fit_run* r, float ms, int n_rows) {
    Workspace& ws = r->ws;
    const sad_train_config& c = r->cfg;
    DevState fs = ws.get_state();
    r->n_sites = static_cast<size_t>(fs.n_sites);
    std::vector<double2> lh(std::max(c.iters, 1));
    std::vector<int32_t> ah(std::max(c.iters, 1));
    ck(cudaMemcpy(lh.data(), r->loss_hist.p, lh.size() * sizeof(double2), cudaMemcpyDeviceToHost), "D2H hist");
    ck(cudaMemcpy(ah.data(), r->active_hist.p, ah.size() * 4, cudaMemcpyDeviceToHost), "D2H hist");
    r->hist.resize(n_rows);
    const double npx = static_cast<double>(r->w) * r->h;
    for (int t = 0; t < n_rows; t++) {
        double loss = (lh[t].x + lh[t].y) / npx;
        double m = loss / 3.0;
        double ps = m <= 0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / m));
        r->hist[t] = sad_history_row{t + 1, loss, ps, ah[t], ms / std::max(c.iters, 1)};
    }
    r->done = true;
    if (fs.err & 1) fail(SAD_EEMPTY, "backward: empty candidate list at a pixel");
    if (fs.err & 2) fail(SAD_ENOMEM, "fit: site capacity exhausted");
    if (fs.err & 8)
        std::fprintf(stderr, "sad: fp64 ordered reduction: record pools full, some sums merged as double-doubles "
                             "(raise SAD_OCAP)\n");
    for (int t = 0; t < n_rows; t++)
        if (!std::isfinite(r->hist[t].loss)) fail(SAD_ENUMERIC, "fit: non-finite loss");
}

// SAD_ADAM_ALL=1: plain-iteration Adam over every slot (A/B)
static const bool g_adam_all = getenv("SAD_ADAM_ALL") != nullptr;
static const bool g_stats_adaptive = getenv("SAD_STATS_FIXED") == nullptr;  // A/B: fixed stats record layout

// fit_impl (train.cpp:221-291), resident in HBM.
static void fit_loop(sad_fit_run* r) {
    Workspace& ws = r->ws;
    const sad_train_config& c = r->cfg;
    const int w = r->w, h = r->h;
    const bool fp64 = c.fp64 != 0;
    const bool budget = c.target_bpp > 0;
    const double scale_n = norm_scale(w, h);
    cudaStream_t s = ws.stream;

    DevState st0 = ws.get_state();
    ws.compute_active();
    DevState sta = ws.get_state();
    double sched = 1.0;
    r->schedule_scale = 0;
    if (budget) {
        if (sta.n_active != r->planned_n0) {
            r->planned_scale = plan_schedule(sta.n_active, bpp_target_count(c.target_bpp, w, h), c);
            r->planned_n0 = sta.n_active;
        }
        sched = r->planned_scale;
        r->schedule_scale = sched;
    }
    int capn = capacity_bound(c, st0.n_sites, sched, budget);
    if (capn > ws.cap) {
        ws.ensure_cap(capn);  // reallocates the active list: rebuild it
        ws.compute_active();
        sta = ws.get_state();
    }
    // fresh optimiser and accumulators
    ck(cudaMemsetAsync(ws.m.p, 0, sizeof(double) * 10 * ws.cap, s), "memset m");
    ck(cudaMemsetAsync(ws.v.p, 0, sizeof(double) * 10 * ws.cap, s), "memset v");
    ws.zero_red(true);
    DevState init{};
    init.n_sites = st0.n_sites;
    init.n_active = sta.n_active;
    ws.set_state(init);
    ws.ensure_adaptive(static_cast<size_t>(sadk::backward_blocks(fp64, ws.fd)));
    // tau_diffusion (train.cpp:251-252): only lambda > 0 runs it, and lambda > 1 fails on iteration 1
    const bool tau = c.tau_diffusion_lambda > 0;
    if (tau && c.iters >= 1 && c.tau_diffusion_lambda > 1) fail(SAD_EINVAL, "tau_diffusion: lambda out of [0,1]");
    if (tau) ensure_tau(ws);
    // fp64: per-site sums in the reference's order (sadk::fp64_ordered): tagged records, then the ordered
    // totals (values) for Adam; tau_diffusion then works on those values as on the double-double ones
    const bool ordered = use_ordered(fp64, ws.fd);
    if (ordered) ws.otot.ensure(10 * static_cast<size_t>(ws.cap));
    auto gred = [&] { return ordered ? ws.gred_adaptive_ord() : ws.gred_adaptive(); };
    if (ordered) (void)gred();  // the tag arrays exist before any graph capture
    const double* totals = tau ? ws.tb.tot.p : ordered ? ws.otot.p : nullptr;
    auto tau_step = [&] {
        if (ordered)
            sadk::launch_ordered_totals(gred(), 10, ws.st.p, const_cast<double*>(totals), tau ? ws.tb.g0.p : nullptr,
                                        false, s);
        if (!tau) return;
        if (!ordered) sadk::launch_site_totals(gred(), ws.st.p, ws.cap, ws.tb.tot.p, ws.tb.g0.p, s);
        tau_device(ws, c.tau_diffusion_lambda, ws.tb.tot.p + 2 * static_cast<size_t>(ws.cap), ws.tb.g0.p);
    };
    sadk::launch_fill_i32(ws.rcap.p, ws.cap, 16, s);
    ws.plan_records();
    ck(cudaMemsetAsync(ws.gcnt.p, 0, sizeof(int32_t) * ws.cap, s), "memset gcnt");
    ck(cudaMemsetAsync(ws.ghead.p, 0xff, sizeof(int32_t) * ws.cap, s), "memset ghead");

    const sadk::AdamHyper hp = adam_hyper(c, w, h);
    const auto full4 = full_refresh_passes(ws.fd.gw, ws.fd.gh, 4);
    const std::vector<sad_pass_spec> warm(static_cast<size_t>(c.refresh_passes), sad_pass_spec{1, 0});
    const void* tgt = fp64 ? static_cast<const void*>(ws.tgt_d.p) : static_cast<const void*>(ws.tgt_f.p);

    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    // phase timing: 0 propagate (warm + event refresh passes), 1 fwd+bwd, 2 Adam + bookkeeping,
    // 3 events (stats, selection, compaction, seeding), 4 init refresh + final refresh
    for (auto& m : r->marks) {
        cudaEventDestroy(m.second.first);
        cudaEventDestroy(m.second.second);
    }
    r->marks.clear();
    const bool prof = r->profile;
    auto mark = [&](int ph, auto&& fn) {
        if (!prof) {
            fn();
            return;
        }
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        fn();
        cudaEventRecord(b, s);
        r->marks.push_back({ph, {a, b}});
    };

    // initial full refresh (train.cpp:238-239)
    build_tables(ws, fp64, true, true, false);
    ws.cur = 0;
    sadk::launch_jfa_seed(ws.sites(), ws.st.p, ws.ids[0].p, ws.fd, scale_n, s);
    passes_device(ws, full4, c.inject, c.seed, fp64, 0);
    const int nbw = sadk::backward_blocks(fp64, ws.fd, ordered);
    sadk::launch_advance(ws.st.p, static_cast<int>(full4.size()), 0, nullptr, nullptr, nullptr, 0, ws.otops.p, s);

    const bool use_graphs = getenv("SAD_NO_GRAPHS") == nullptr && !prof;
    const bool fold_advance = getenv("SAD_NO_FOLD") == nullptr;
    // One plain iteration: warm pass(es) -> fused fwd+bwd -> Adam (+ tables for the next pass) ->
    // bookkeeping.  All per-iteration scalars live in DevState, so the sequence is replayable.
    auto plain_iteration = [&](bool rf) {
        int np = 0;
        if (rf) {
            mark(0, [&] { passes_device(ws, warm, c.inject, c.seed, fp64, 0); });
            np = static_cast<int>(warm.size());
        }
        mark(1, [&] {
            sadk::launch_backward(fp64, 0, ws.ids[ws.cur].p, ws.gtab.p, tgt, ws.fd, scale_n, gred(),
                                  ws.loss_part.p, ws.st.p, s);
            tau_step();
        });
        // the iteration's bookkeeping rides in Adam's grid (AdvanceArgs) unless SAD_NO_FOLD is set
        sadk::AdvanceArgs adv;
        if (fold_advance) {
            adv.loss_hist = r->loss_hist.p;
            adv.active_hist = r->active_hist.p;
            adv.loss_part = ws.loss_part.p;
            adv.n_part = nbw;
            adv.passes = np;
            adv.otop = ws.otops.p;
        }
        mark(2, [&] {
            // plain iterations: active sites only (event iterations below run every slot, which also
            // zeroes the record capacity of pruned slots before densify can reuse them)
            sadk::launch_adam(fp64, ws.sites(), ws.st.p, gred(), ws.m.p, ws.v.p, hp, r->bc_table.p,
                              make_double2(0, 0), true, scale_n, ws.pack.p, ws.gtab.p, ws.rcap.p, s, totals,
                              ws.roff.p, ws.otops.p + 2, g_adam_all ? nullptr : ws.act.p, nullptr, adv);
        });
        if (!fold_advance)
            mark(5, [&] {
                sadk::launch_advance(ws.st.p, np, 1, r->loss_hist.p, r->active_hist.p, ws.loss_part.p, nbw,
                                     ws.otops.p, s);
            });
    };
    // SAD_STOP_AT=t (divergence hunting): stop after iteration t without the final refresh
    const int stop_at = getenv("SAD_STOP_AT") ? atoi(getenv("SAD_STOP_AT")) : 0;
    auto refresh_at = [&](int t) { return (t - 1) % c.refresh_every == 0; };
    auto event_d = [&](int t) { return budget && t >= c.densify_start && t <= c.densify_end && t % c.densify_every == 0; };
    auto event_p = [&](int t) {
        bool e = budget && t >= c.prune_start && t <= c.prune_end && t % c.prune_every == 0;
        return e && !(!c.prune_during_densify && t <= c.densify_end);
    };
    for (int t = 1; t <= c.iters; t++) {
        if (stop_at && t > stop_at) break;
        const bool rf = refresh_at(t);
        bool ev_d = event_d(t);
        bool ev_p = event_p(t);
        bool ev = ev_d || ev_p;
        if (!ev && use_graphs) {
            // a run of n plain iterations with the same refresh flag, replayed as one graph
            int n = 1;
            const int last = stop_at ? std::min(stop_at, c.iters) : c.iters;
            while (n < g_graph_iters && t + n <= last && refresh_at(t + n) == rf && !event_d(t + n) && !event_p(t + n)) n++;
            if (r->graph_epoch != g_alloc_epoch.load() || std::memcmp(&r->graph_cfg, &c, sizeof c) != 0) {
                r->drop_graphs();
                r->graph_epoch = g_alloc_epoch.load();
                r->graph_cfg = c;
            }
            const int c0 = ws.cur;
            const int key = c0 | (rf ? 2 : 0) | (n << 2);
            auto& gx = r->plain[key];
            if (!gx.first) {
                cudaGraph_t g = nullptr;
                uint64_t l0 = sadk::launch_counter();
                ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
                for (int i = 0; i < n; i++) plain_iteration(rf);
                ck(cudaStreamEndCapture(s, &g), "end capture");
                ck(cudaGraphInstantiate(&gx.first, g, 0), "graph instantiate");
                cudaGraphDestroy(g);
                gx.second = sadk::launch_counter() - l0;
                ws.cur = c0;
            }
            ck(cudaGraphLaunch(gx.first, s), "graph launch");
            sadk::add_launches(gx.second);
            if (rf && (warm.size() & 1) && (n & 1)) ws.cur = 1 - c0;
            t += n - 1;
            continue;
        }
        if (!ev) {
            plain_iteration(rf);
            continue;
        }
        int npass = 0;
        if (rf) {
            mark(0, [&] { passes_device(ws, warm, c.inject, c.seed, fp64, 0); });
            npass += static_cast<int>(warm.size());
        }
        mark(1, [&] {
            sadk::launch_backward(fp64, 0, ws.ids[ws.cur].p, ws.gtab.p, tgt, ws.fd, scale_n, gred(),
                                  ws.loss_part.p, ws.st.p, s);
            tau_step();
        });
        mark(3, [&] { stats_device(ws, g_stats_adaptive); });
        mark(2, [&] {
            sadk::launch_adam(fp64, ws.sites(), ws.st.p, gred(), ws.m.p, ws.v.p, hp, r->bc_table.p,
                              make_double2(0, 0), true, scale_n, nullptr, nullptr, ws.rcap.p, s, totals,
                              ws.roff.p, ws.otops.p + 2);
        });
        mark(3, [&] {
            if (ev_p) prune_device(ws, c.prune_pct * sched);
            if (ev_d) densify_device(ws, c.densify_pct * sched, c);
            ws.compute_active();
            build_tables(ws, fp64, true, true, false);
            ws.cur = 0;
            sadk::launch_jfa_seed(ws.sites(), ws.st.p, ws.ids[0].p, ws.fd, scale_n, s);
        });
        mark(0, [&] { passes_device(ws, full4, c.inject, c.seed, fp64, static_cast<uint32_t>(npass)); });
        npass += static_cast<int>(full4.size());
        mark(2, [&] {
            sadk::launch_advance(ws.st.p, npass, 1, r->loss_hist.p, r->active_hist.p, ws.loss_part.p, nbw, ws.otops.p,
                                 s);
        });
    }
    // final full refresh (train.cpp:287)
    if (!stop_at) {
        const auto fin = full_refresh_passes(ws.fd.gw, ws.fd.gh, c.final_passes);
        ws.cur = 0;
        sadk::launch_jfa_seed(ws.sites(), ws.st.p, ws.ids[0].p, ws.fd, scale_n, s);
        passes_device(ws, fin, c.inject, c.seed, fp64, 0);
        sadk::launch_advance(ws.st.p, static_cast<int>(fin.size()), 0, nullptr, nullptr, nullptr, 0, ws.otops.p, s);
    }
    cudaEventRecord(e1, s);
    ck(cudaStreamSynchronize(s), "fit");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    r->total_ms = ms;
    for (double& p : r->phase_ms) p = 0;
    for (auto& m : r->marks) {
        float pm = 0;
        cudaEventElapsedTime(&pm, m.second.first, m.second.second);
        if (m.first < 8) r->phase_ms[m.first] += pm;
    }
    if (r->profile)
        std::fprintf(stderr, "phases ms: propagate %.1f fwd_bwd %.1f adam %.1f events %.1f advance %.1f\n",
                     r->phase_ms[0], r->phase_ms[1], r->phase_ms[2], r->phase_ms[3], r->phase_ms[5]);

    finish_run(r, ms, stop_at ? std::min(c.iters, stop_at) : c.iters);
}

// ====================================================================== row-strip multi-GPU fit (config 5)
// one large image split into row strips.  Every rank holds the sites, the tables, the target
// and the whole candidate field, but computes only its strip: propagation rows, backward and stats tiles
// (FieldDims row range; strips are multiples of the tile heights).  Sites are OWNED by id slice: rank q
// owns ids [q*slice, (q+1)*slice), slice = ceil(cap / R); init_sites numbers sites in raster order, so
// slices start out as row bands close to the strips.  Exchanges per iteration:
//   * before every propagation pass at jump s: the rows within s of the strip (owner -> reader); at the
//     end, all strips, so every rank holds the whole final field;
//   * after the backward (owner merge): each rank's double-double partial totals of the sites it touched
//     but does not own travel to their owners as (id, 10 double-doubles) records (counts first: one R x R
//     all-gather and one host read, then grouped point-to-point), and the owner merges them exactly;
//   * Adam runs on the owned slice only (moments live with the owner), then the updated parameters of
//     every slice are all-gathered (10 doubles per site) and each rank rebuilds its tables;
//   * at events: stats partials take the same owner merge, then the owned stats totals are all-gathered
//     (8 double-doubles per site) so prune / densify (and the seeding) run replicated and deterministically.
// Every sum is an exact double-double merge, so the strip fit is bit-identical to the single-GPU fit.
// Transports: NCCL (one process per GPU; loaded with dlopen), a loopback of R virtual ranks on one device,
// and a host-staged transport whose collectives are callbacks (the Python binding runs them over a
// torch.distributed process group, e.g. gloo: two processes can share one GPU).
struct XferPlan {  // one local rank's point-to-point exchange: peer i gets send[i], we get recv[i] from it
    std::vector<int> peer;
    std::vector<const void*> send;
    std::vector<size_t> sbytes;
    std::vector<void*> recv;
    std::vector<size_t> rbytes;
    void add(int q, const void* s, size_t sb, void* r, size_t rb) {
        peer.push_back(q);
        send.push_back(s);
        sbytes.push_back(sb);
        recv.push_back(r);
        rbytes.push_back(rb);
    }
};

struct StripComm {
    virtual ~StripComm() = default;
    virtual int world() const = 0;
    // rows [strip[q], strip[q+1]) of ids[b] (cell rows of gw*k u32) from rank q to every rank
    virtual void gather_rows(std::vector<sad_fit_run*>& runs, int b) = 0;
    // before a pass at jump `step`: every rank fetches the rows it will read outside its strip,
    // [row0 - step, row0) and [row1, row1 + step), from their owners (buffer ids[b])
    virtual void halo_rows(std::vector<sad_fit_run*>& runs, int b, int step) = 0;
    // slice q (bytes each) of every rank's `all` <- rank q's `self`
    virtual void gather(std::vector<sad_fit_run*>& runs, const std::function<const void*(sad_fit_run*)>& self,
                        const std::function<void*(sad_fit_run*)>& all, size_t bytes) = 0;
    // grouped point-to-point transfers, plans[i] for runs[i] (device pointers; sizes agree pairwise)
    virtual void exchange(std::vector<sad_fit_run*>& runs, std::vector<XferPlan>& plans) = 0;
};

// Rows rank `r` reads outside its strip at jump `step` that rank `q` owns: up to two [lo, hi) ranges.
// A pass at jump s reads rows y - s, y, y + s for the strip's rows y: the bands [row0 - s, row1 - s) and
// [row0 + s, row1 + s) outside the strip (for s >= the strip height, a strip-sized band, not s rows).
static int halo_ranges(const std::vector<int>& strip, int r, int q, int step, int out[4]) {
    const int rows = strip.back();
    const int r0 = strip[r], r1 = strip[r + 1];
    const int need[2][2] = {{std::max(0, r0 - step), std::min(r0, r1 - step)},
                            {std::max(r1, r0 + step), std::min(rows, r1 + step)}};
    int n = 0;
    for (const auto& nd : need) {
        const int lo = std::max(nd[0], strip[q]), hi = std::min(nd[1], strip[q + 1]);
        if (hi > lo) {
            out[2 * n] = lo;
            out[2 * n + 1] = hi;
            n++;
        }
    }
    return n;
}

// The rows rank `r` must receive from rank `q` (and, symmetrically, send) for a halo at jump `step`.
static void halo_plan(std::vector<sad_fit_run*>& runs, int b, int step, std::vector<XferPlan>& plans, int world) {
    const size_t row = static_cast<size_t>(runs[0]->ws.fd.gw) * runs[0]->ws.fd.k;
    plans.assign(runs.size(), XferPlan{});
    for (size_t i = 0; i < runs.size(); i++) {
        sad_fit_run* r = runs[i];
        const int me = r->rank;
        for (int q = 0; q < world; q++) {
            if (q == me) continue;
            int sr[4], rr[4];
            const int ms = halo_ranges(r->strip, q, me, step, sr);  // rows q needs that I own
            const int mr = halo_ranges(r->strip, me, q, step, rr);  // rows I need that q owns
            for (int j = 0; j < std::max(ms, mr); j++) {
                const uint32_t* sp = j < ms ? r->ws.ids[b].p + row * sr[2 * j] : nullptr;
                uint32_t* rp = j < mr ? r->ws.ids[b].p + row * rr[2 * j] : nullptr;
                plans[i].add(q, sp, j < ms ? 4 * row * (sr[2 * j + 1] - sr[2 * j]) : 0, rp,
                             j < mr ? 4 * row * (rr[2 * j + 1] - rr[2 * j]) : 0);
            }
        }
    }
}

// Every rank's strip to every other rank.
static void rows_plan(std::vector<sad_fit_run*>& runs, int b, std::vector<XferPlan>& plans, int world) {
    const size_t row = static_cast<size_t>(runs[0]->ws.fd.gw) * runs[0]->ws.fd.k;
    plans.assign(runs.size(), XferPlan{});
    for (size_t i = 0; i < runs.size(); i++) {
        sad_fit_run* r = runs[i];
        const int me = r->rank;
        for (int q = 0; q < world; q++) {
            if (q == me) continue;
            plans[i].add(q, r->ws.ids[b].p + row * r->strip[me], 4 * row * (r->strip[me + 1] - r->strip[me]),
                         r->ws.ids[b].p + row * r->strip[q], 4 * row * (r->strip[q + 1] - r->strip[q]));
        }
    }
}

struct LoopbackComm : StripComm {
    int n;
    explicit LoopbackComm(int world) : n(world) {}
    int world() const override { return n; }
    void gather_rows(std::vector<sad_fit_run*>& runs, int b) override {
        std::vector<XferPlan> plans;
        rows_plan(runs, b, plans, n);
        exchange(runs, plans);
    }
    void halo_rows(std::vector<sad_fit_run*>& runs, int b, int step) override {
        std::vector<XferPlan> plans;
        halo_plan(runs, b, step, plans, n);
        exchange(runs, plans);
    }
    void gather(std::vector<sad_fit_run*>& runs, const std::function<const void*(sad_fit_run*)>& self,
                const std::function<void*(sad_fit_run*)>& all, size_t bytes) override {
        for (int q = 0; q < n; q++)
            for (int r = 0; r < n; r++)
                ck(cudaMemcpyAsync(static_cast<char*>(all(runs[r])) + bytes * q, self(runs[q]), bytes,
                                   cudaMemcpyDeviceToDevice, runs[r]->ws.stream),
                   "loopback gather");
    }
    void exchange(std::vector<sad_fit_run*>& runs, std::vector<XferPlan>& plans) override {
        // every local rank holds both ends: the j-th non-empty send of r to q pairs with the j-th non-empty
        // receive of q from r (the order NCCL and the host transport pair them in)
        for (int r = 0; r < n; r++)
            for (int q = 0; q < n; q++) {
                if (q == r) continue;
                std::vector<size_t> si, ri;
                for (size_t i = 0; i < plans[r].peer.size(); i++)
                    if (plans[r].peer[i] == q && plans[r].sbytes[i]) si.push_back(i);
                for (size_t i = 0; i < plans[q].peer.size(); i++)
                    if (plans[q].peer[i] == r && plans[q].rbytes[i]) ri.push_back(i);
                if (si.size() != ri.size()) fail(SAD_ECUDA, "strips loopback: unmatched transfers");
                for (size_t j = 0; j < si.size(); j++) {
                    if (plans[r].sbytes[si[j]] != plans[q].rbytes[ri[j]]) fail(SAD_ECUDA, "strips loopback: size mismatch");
                    ck(cudaMemcpyAsync(plans[q].recv[ri[j]], plans[r].send[si[j]], plans[r].sbytes[si[j]],
                                       cudaMemcpyDeviceToDevice, runs[q]->ws.stream),
                       "loopback exchange");
                }
            }
    }
};

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    static NcclApi& get() {
        static NcclApi a;
        if (!a.lib) {
            a.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!a.lib) fail(SAD_EINVAL, std::string("strips: cannot load libnccl.so.2: ") + dlerror());
            auto sym = [&](const char* n) {
                void* f = dlsym(a.lib, n);
                if (!f) fail(SAD_EINVAL, std::string("strips: NCCL symbol missing: ") + n);
                return f;
            };
            a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(sym("ncclGetUniqueId"));
            a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(sym("ncclCommInitRank"));
            a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(sym("ncclCommDestroy"));
            a.allGather = reinterpret_cast<decltype(a.allGather)>(sym("ncclAllGather"));
            a.broadcast = reinterpret_cast<decltype(a.broadcast)>(sym("ncclBroadcast"));
            a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
            a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
            a.groupStart = reinterpret_cast<decltype(a.groupStart)>(sym("ncclGroupStart"));
            a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(sym("ncclGroupEnd"));
            a.errorString = reinterpret_cast<decltype(a.errorString)>(sym("ncclGetErrorString"));
        }
        return a;
    }
    void check(ncclResult_t rc, const char* what) const {
        if (rc != ncclSuccess) fail(SAD_ECUDA, std::string(what) + ": " + errorString(rc));
    }
};

struct NcclComm : StripComm {
    NcclApi& api;
    ncclComm_t comm = nullptr;
    int n;
    NcclComm(int rank, int world, const uint8_t* id) : api(NcclApi::get()), n(world) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        api.check(api.commInitRank(&comm, world, uid, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm) api.commDestroy(comm);
    }
    int world() const override { return n; }
    void gather_rows(std::vector<sad_fit_run*>& runs, int b) override {
        sad_fit_run* r = runs[0];
        const size_t row = static_cast<size_t>(r->ws.fd.gw) * r->ws.fd.k;
        api.check(api.groupStart(), "ncclGroupStart");
        for (int q = 0; q < n; q++) {
            const size_t off = row * r->strip[q], cnt = row * (r->strip[q + 1] - r->strip[q]);
            if (cnt)
                api.check(api.broadcast(r->ws.ids[b].p + off, r->ws.ids[b].p + off, cnt, ncclUint32, q, comm, r->ws.stream),
                          "ncclBroadcast");
        }
        api.check(api.groupEnd(), "ncclGroupEnd");
    }
    void halo_rows(std::vector<sad_fit_run*>& runs, int b, int step) override {
        std::vector<XferPlan> plans;
        halo_plan(runs, b, step, plans, n);
        exchange(runs, plans);
    }
    void gather(std::vector<sad_fit_run*>& runs, const std::function<const void*(sad_fit_run*)>& self,
                const std::function<void*(sad_fit_run*)>& all, size_t bytes) override {
        sad_fit_run* r = runs[0];
        api.check(api.allGather(self(r), all(r), bytes, ncclChar, comm, r->ws.stream), "ncclAllGather");
    }
    void exchange(std::vector<sad_fit_run*>& runs, std::vector<XferPlan>& plans) override {
        sad_fit_run* r = runs[0];
        const XferPlan& pl = plans[0];
        api.check(api.groupStart(), "ncclGroupStart");
        for (size_t i = 0; i < pl.peer.size(); i++) {
            if (pl.sbytes[i])
                api.check(api.send(pl.send[i], pl.sbytes[i], ncclChar, pl.peer[i], comm, r->ws.stream), "ncclSend");
            if (pl.rbytes[i])
                api.check(api.recv(pl.recv[i], pl.rbytes[i], ncclChar, pl.peer[i], comm, r->ws.stream), "ncclRecv");
        }
        api.check(api.groupEnd(), "ncclGroupEnd");
    }
};

// Host-staged transport: device data goes through pinned host buffers and the caller's collective
// callbacks (sad_host_allgather_fn / sad_host_exchange_fn, include/sad_b200.h).
struct HostComm : StripComm {
    int n, me;
    sad_host_allgather_fn ag;
    sad_host_exchange_fn ex;
    void* user;
    std::vector<char*> pin;
    std::vector<size_t> pin_n;
    HostComm(int rank, int world, sad_host_allgather_fn a, sad_host_exchange_fn e, void* u)
        : n(world), me(rank), ag(a), ex(e), user(u), pin(8, nullptr), pin_n(8, 0) {}
    ~HostComm() override {
        for (char* p : pin)
            if (p) cudaFreeHost(p);
    }
    char* stage(int i, size_t bytes) {
        if (pin_n[i] < bytes) {
            if (pin[i]) cudaFreeHost(pin[i]);
            pin[i] = nullptr;
            ck(cudaMallocHost(&pin[i], std::max<size_t>(bytes, 1)), "cudaMallocHost");
            pin_n[i] = bytes;
        }
        return pin[i];
    }
    int world() const override { return n; }
    void gather_rows(std::vector<sad_fit_run*>& runs, int b) override {
        std::vector<XferPlan> plans;
        rows_plan(runs, b, plans, n);
        exchange(runs, plans);
    }
    void halo_rows(std::vector<sad_fit_run*>& runs, int b, int step) override {
        std::vector<XferPlan> plans;
        halo_plan(runs, b, step, plans, n);
        exchange(runs, plans);
    }
    void gather(std::vector<sad_fit_run*>& runs, const std::function<const void*(sad_fit_run*)>& self,
                const std::function<void*(sad_fit_run*)>& all, size_t bytes) override {
        sad_fit_run* r = runs[0];
        char* hs = stage(0, bytes);
        char* ha = stage(1, bytes * n);
        ck(cudaMemcpyAsync(hs, self(r), bytes, cudaMemcpyDeviceToHost, r->ws.stream), "D2H gather");
        ck(cudaStreamSynchronize(r->ws.stream), "host gather");
        if (ag(user, hs, ha, bytes) != 0) fail(SAD_ECUDA, "strips: host all-gather callback failed");
        ck(cudaMemcpyAsync(all(r), ha, bytes * n, cudaMemcpyHostToDevice, r->ws.stream), "H2D gather");
        ck(cudaStreamSynchronize(r->ws.stream), "host gather");
    }
    void exchange(std::vector<sad_fit_run*>& runs, std::vector<XferPlan>& plans) override {
        sad_fit_run* r = runs[0];
        const XferPlan& pl = plans[0];
        const size_t m = pl.peer.size();
        size_t st = 0, rt = 0;
        for (size_t i = 0; i < m; i++) {
            st += pl.sbytes[i];
            rt += pl.rbytes[i];
        }
        char* hs = stage(2, st);
        char* hr = stage(3, rt);
        std::vector<const void*> sp(m);
        std::vector<void*> rp(m);
        size_t so = 0, ro = 0;
        for (size_t i = 0; i < m; i++) {
            if (pl.sbytes[i])
                ck(cudaMemcpyAsync(hs + so, pl.send[i], pl.sbytes[i], cudaMemcpyDeviceToHost, r->ws.stream), "D2H xfer");
            sp[i] = hs + so;
            rp[i] = hr + ro;
            so += pl.sbytes[i];
            ro += pl.rbytes[i];
        }
        ck(cudaStreamSynchronize(r->ws.stream), "host exchange");
        if (m && ex(user, static_cast<int>(m), pl.peer.data(), sp.data(), pl.sbytes.data(), rp.data(), pl.rbytes.data()) != 0)
            fail(SAD_ECUDA, "strips: host exchange callback failed");
        for (size_t i = 0; i < m; i++)
            if (pl.rbytes[i])
                ck(cudaMemcpyAsync(pl.recv[i], rp[i], pl.rbytes[i], cudaMemcpyHostToDevice, r->ws.stream), "H2D xfer");
        ck(cudaStreamSynchronize(r->ws.stream), "host exchange");
    }
};

// Row bounds of `world` strips over `rows` rows, each a multiple of the backward/stats tile heights
// (sadk::tile_row_quantum), so no tile straddles two strips.
static std::vector<int> strip_bounds(int rows, int world, bool ordered) {
    // the fp64 reference-order backward works on the reference's 16-row tiles
    const int qr = ordered ? std::max(16, sadk::tile_row_quantum()) : sadk::tile_row_quantum();
    const int tiles = (rows + qr - 1) / qr;
    std::vector<int> b(static_cast<size_t>(world) + 1);
    for (int q = 0; q <= world; q++)
        b[q] = std::min(rows, qr * static_cast<int>(static_cast<long long>(tiles) * q / world));
    return b;
}

// Owner merge of one reduction (gradients: nch 10 from `part`; stats: 8): every rank sends the partials
// of the touched sites it does not own to their owners, who merge them into `part` exactly.  Returns the
// records each rank sent (for the exchange-volume report).
static long long owner_merge(std::vector<sad_fit_run*>& runs, StripComm& T, int R, int slice, int nch,
                             const std::function<double2*(sad_fit_run*)>& part,
                             const std::function<sadk::RedTarget(sad_fit_run*)>& red, bool grads) {
    const int send_cap = slice;
    for (sad_fit_run* r : runs) {
        Workspace& ws = r->ws;
        ck(cudaMemsetAsync(r->own_counts.p, 0, sizeof(unsigned long long) * R, ws.stream), "memset counts");
        sadk::launch_owner_pack(part(r), nch, red(r), ws.st.p, ws.active.p, slice, r->rank, R, r->own_send.p, send_cap,
                                r->own_counts.p, grads ? ws.rcap.p : nullptr, grads, ws.stream);
    }
    T.gather(runs, [](sad_fit_run* r) { return static_cast<const void*>(r->own_counts.p); },
             [](sad_fit_run* r) { return static_cast<void*>(r->own_matrix.p); }, sizeof(unsigned long long) * R);
    long long sent = 0;
    std::vector<XferPlan> plans(runs.size());
    std::vector<std::vector<unsigned long long>> mats(runs.size(), std::vector<unsigned long long>(size_t(R) * R));
    for (size_t i = 0; i < runs.size(); i++) {
        ck(cudaMemcpyAsync(mats[i].data(), runs[i]->own_matrix.p, sizeof(unsigned long long) * R * R,
                           cudaMemcpyDeviceToHost, runs[i]->ws.stream),
           "D2H counts");
        ck(cudaStreamSynchronize(runs[i]->ws.stream), "counts");
    }
    std::vector<long long> nrecv(runs.size(), 0);
    for (size_t i = 0; i < runs.size(); i++) {
        sad_fit_run* r = runs[i];
        const int me = r->rank;
        const auto& M = mats[i];  // M[src * R + dst]
        long long roff = 0;
        for (int q = 0; q < R; q++) {
            if (q == me) continue;
            const long long ns = std::min<long long>(M[static_cast<size_t>(me) * R + q], send_cap);
            const long long nr = std::min<long long>(M[static_cast<size_t>(q) * R + me], send_cap);
            plans[i].add(q, r->own_send.p + static_cast<size_t>(q) * send_cap, ns * sizeof(sadk::OwnRec),
                         r->own_recv.p + roff, nr * sizeof(sadk::OwnRec));
            roff += nr;
            sent += ns;
            if (grads) r->xfer_records += ns;
        }
        nrecv[i] = roff;
    }
    T.exchange(runs, plans);
    for (size_t i = 0; i < runs.size(); i++)
        sadk::launch_owner_merge(runs[i]->own_recv.p, nrecv[i], nch, runs[i]->ws.cap, part(runs[i]), runs[i]->ws.stream);
    return sent;
}

// fp64 reference-order strips: every rank sends the tagged records of the sites it touched but does not own to
// their owners (counts first), who link them into the sites' overflow lists; the ordered merge then replays
// each owned site's records from all strips in the reference's tile order.  Returns the records sent.
static long long owner_merge_ord(std::vector<sad_fit_run*>& runs, StripComm& T, int R, int slice) {
    for (sad_fit_run* r : runs) {
        Workspace& ws = r->ws;
        ck(cudaMemsetAsync(r->own_counts.p, 0, sizeof(unsigned long long) * R, ws.stream), "memset counts");
        sadk::launch_owner_count_ord(ws.gred_adaptive_ord(), ws.st.p, slice, r->rank, R, r->own_counts.p, ws.stream);
    }
    T.gather(runs, [](sad_fit_run* r) { return static_cast<const void*>(r->own_counts.p); },
             [](sad_fit_run* r) { return static_cast<void*>(r->own_matrix.p); }, sizeof(unsigned long long) * R);
    std::vector<std::vector<unsigned long long>> mats(runs.size(), std::vector<unsigned long long>(size_t(R) * R));
    for (size_t i = 0; i < runs.size(); i++) {
        ck(cudaMemcpyAsync(mats[i].data(), runs[i]->own_matrix.p, sizeof(unsigned long long) * R * R,
                           cudaMemcpyDeviceToHost, runs[i]->ws.stream),
           "D2H counts");
        ck(cudaStreamSynchronize(runs[i]->ws.stream), "counts");
    }
    long long sent = 0;
    std::vector<XferPlan> plans(runs.size());
    std::vector<long long> nrecv(runs.size(), 0);
    for (size_t i = 0; i < runs.size(); i++) {
        sad_fit_run* r = runs[i];
        Workspace& ws = r->ws;
        const int me = r->rank;
        const auto& M = mats[i];  // M[src * R + dst]
        long long send_cap = 1, recv_n = 0;
        for (int q = 0; q < R; q++) {
            send_cap = std::max<long long>(send_cap, static_cast<long long>(M[static_cast<size_t>(me) * R + q]));
            if (q != me) recv_n += static_cast<long long>(M[static_cast<size_t>(q) * R + me]);
        }
        r->ord_send.ensure(static_cast<size_t>(R) * send_cap);
        r->ord_recv.ensure(static_cast<size_t>(std::max<long long>(recv_n, 1)));
        ck(cudaMemsetAsync(r->own_counts.p, 0, sizeof(unsigned long long) * R, ws.stream), "memset cursors");
        sadk::launch_owner_pack_ord(ws.gred_adaptive_ord(), ws.st.p, slice, me, R, r->ord_send.p, send_cap,
                                    r->own_counts.p, ws.stream);
        long long roff = 0;
        for (int q = 0; q < R; q++) {
            if (q == me) continue;
            const long long ns = static_cast<long long>(M[static_cast<size_t>(me) * R + q]);
            const long long nr = static_cast<long long>(M[static_cast<size_t>(q) * R + me]);
            plans[i].add(q, r->ord_send.p + static_cast<size_t>(q) * send_cap, ns * sizeof(sadk::OwnRec),
                         r->ord_recv.p + roff, nr * sizeof(sadk::OwnRec));
            roff += nr;
            sent += ns;
            r->xfer_records += ns;
        }
        nrecv[i] = roff;
    }
    T.exchange(runs, plans);
    for (size_t i = 0; i < runs.size(); i++)
        sadk::launch_owner_merge_ord(runs[i]->ord_recv.p, nrecv[i], runs[i]->ws.gred_adaptive_ord(), runs[i]->ws.st.p,
                                     runs[i]->ws.stream);
    return sent;
}

static void fit_loop_strips(std::vector<sad_fit_run*>& runs, StripComm& T) {
    // every exit (including an exception mid-fit) leaves the runs' field views on the whole image
    struct RowRestore {
        std::vector<sad_fit_run*>& rs;
        ~RowRestore() {
            for (sad_fit_run* r : rs) {
                r->ws.fd.row0 = 0;
                r->ws.fd.row1 = 1 << 30;
            }
        }
    } restore_rows{runs};
    const int R = T.world();
    sad_fit_run* r0 = runs[0];
    const sad_train_config& c = r0->cfg;
    const int w = r0->w, h = r0->h;
    const bool fp64 = c.fp64 != 0;
    const bool ordered = use_ordered(fp64, r0->ws.fd);  // fp64: the reference's summation order (§3)
    const bool budget = c.target_bpp > 0;
    const double scale_n = norm_scale(w, h);
    if (c.tau_diffusion_lambda > 0) fail(SAD_EINVAL, "strips: tau_diffusion is not supported");
    if (c.k > 16 || r0->ws.fd.cell != 1) fail(SAD_EINVAL, "strips: cell size 1 only");
    double sched = 1.0;
    // prologue, per rank (as fit_loop)
    for (sad_fit_run* r : runs) {
        Workspace& ws = r->ws;
        cudaStream_t s = ws.stream;
        DevState st0 = ws.get_state();
        ws.compute_active();
        DevState sta = ws.get_state();
        r->schedule_scale = 0;
        if (budget) {
            if (sta.n_active != r->planned_n0) {
                r->planned_scale = plan_schedule(sta.n_active, bpp_target_count(c.target_bpp, w, h), c);
                r->planned_n0 = sta.n_active;
            }
            sched = r->planned_scale;
            r->schedule_scale = sched;
        }
        int capn = capacity_bound(c, st0.n_sites, sched, budget);
        if (capn > ws.cap) {
            ws.ensure_cap(capn);
            ws.compute_active();
            sta = ws.get_state();
        }
        ck(cudaMemsetAsync(ws.m.p, 0, sizeof(double) * 10 * ws.cap, s), "memset m");
        ck(cudaMemsetAsync(ws.v.p, 0, sizeof(double) * 10 * ws.cap, s), "memset v");
        ws.zero_red(true);
        DevState init{};
        init.n_sites = st0.n_sites;
        init.n_active = sta.n_active;
        ws.set_state(init);
        r->strip = strip_bounds(h, R, ordered);
        ws.fd.row0 = r->strip[r->rank];
        ws.fd.row1 = r->strip[r->rank + 1];
        ws.ensure_adaptive(static_cast<size_t>(sadk::backward_blocks(fp64, ws.fd)));
        if (ordered) (void)ws.gred_adaptive_ord();  // tag arrays
        sadk::launch_fill_i32(ws.rcap.p, ws.cap, 16, s);
        ws.plan_records();
        ck(cudaMemsetAsync(ws.gcnt.p, 0, sizeof(int32_t) * ws.cap, s), "memset gcnt");
        ck(cudaMemsetAsync(ws.ghead.p, 0xff, sizeof(int32_t) * ws.cap, s), "memset ghead");
    }
    const int cap = r0->ws.cap;
    for (sad_fit_run* r : runs)
        if (r->ws.cap != cap) fail(SAD_EINVAL, "strips: ranks disagree on the site capacity");
    const int slice = (cap + R - 1) / R;
    for (sad_fit_run* r : runs) {
        const size_t sc = static_cast<size_t>(slice);
        r->gpart_self.ensure(10 * static_cast<size_t>(cap));
        r->loss_self.ensure(1);
        r->loss_all.ensure(R);
        r->tot.ensure(10 * static_cast<size_t>(cap));
        r->valid_all.ensure(R);
        r->own_counts.ensure(R);
        r->own_matrix.ensure(static_cast<size_t>(R) * R);
        r->own_send.ensure(static_cast<size_t>(R) * sc);
        r->own_recv.ensure(static_cast<size_t>(R) * sc);
        r->own_range.ensure(2);
        r->slice_p.ensure(10 * sc);
        r->slice_all_p.ensure(static_cast<size_t>(R) * 10 * sc);
        r->slice_s.ensure(8 * sc);
        r->slice_all_s.ensure(static_cast<size_t>(R) * 8 * sc);
        r->xfer_records = 0;
    }
    const sadk::AdamHyper hp = adam_hyper(c, w, h);
    const auto full4 = full_refresh_passes(r0->ws.fd.gw, r0->ws.fd.gh, 4);
    const std::vector<sad_pass_spec> warm(static_cast<size_t>(c.refresh_passes), sad_pass_spec{1, 0});
    auto tgt_of = [&](sad_fit_run* r) {
        return fp64 ? static_cast<const void*>(r->ws.tgt_d.p) : static_cast<const void*>(r->ws.tgt_f.p);
    };
    // Each pass reads rows [row0 - step, row1 + step) of the current buffer: those outside the strip are
    // fetched from their owners right before the pass; the pass writes the strip of the other buffer.
    auto passes = [&](const std::vector<sad_pass_spec>& seq, uint32_t base) {
        for (size_t i = 0; i < seq.size(); i++) {
            T.halo_rows(runs, r0->ws.cur, static_cast<int>(seq[i].step));
            for (sad_fit_run* r : runs) {
                Workspace& ws = r->ws;
                sadk::launch_propagate(fp64, ws.ids[ws.cur].p, ws.ids[1 - ws.cur].p, ws.pack.p, ws.act.p, ws.st.p, ws.fd,
                                       seq[i].step, seq[i].stencil, c.inject, c.seed, base + static_cast<uint32_t>(i),
                                       scale_n, ws.stream);
            }
            for (sad_fit_run* r : runs) r->ws.cur = 1 - r->ws.cur;
        }
    };
    auto reseed = [&] {
        for (sad_fit_run* r : runs) {
            r->ws.cur = 0;
            sadk::launch_jfa_seed(r->ws.sites(), r->ws.st.p, r->ws.ids[0].p, r->ws.fd, scale_n, r->ws.stream);
        }
    };
    // all-gather of the owned parameter slices (10 doubles per site)
    auto gather_params = [&] {
        for (sad_fit_run* r : runs)
            sadk::launch_slice_pack<double>(r->ws.params.p, 10, cap, r->rank * slice, slice, r->slice_p.p, r->ws.stream);
        T.gather(runs, [](sad_fit_run* r) { return static_cast<const void*>(r->slice_p.p); },
                 [](sad_fit_run* r) { return static_cast<void*>(r->slice_all_p.p); }, sizeof(double) * 10 * slice);
        for (sad_fit_run* r : runs)
            sadk::launch_slice_unpack<double>(r->slice_all_p.p, 10, cap, slice, R, r->ws.params.p, r->ws.stream);
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, r0->ws.stream);
    // initial full refresh
    for (sad_fit_run* r : runs) build_tables(r->ws, fp64, true, true, false);
    reseed();
    passes(full4, 0);
    for (sad_fit_run* r : runs)
        sadk::launch_advance(r->ws.st.p, static_cast<int>(full4.size()), 0, nullptr, nullptr, nullptr, 0,
                             r->ws.otops.p, r->ws.stream);
    for (int t = 1; t <= c.iters; t++) {
        const bool rf = (t - 1) % c.refresh_every == 0;
        bool ev_d = budget && t >= c.densify_start && t <= c.densify_end && t % c.densify_every == 0;
        bool ev_p = budget && t >= c.prune_start && t <= c.prune_end && t % c.prune_every == 0;
        if (ev_p && !c.prune_during_densify && t <= c.densify_end) ev_p = false;
        const bool ev = ev_d || ev_p;
        int npass = 0;
        if (rf) {
            passes(warm, 0);
            npass += static_cast<int>(warm.size());
        }
        // backward on the strips; each rank's partial totals of the sites it touched
        for (sad_fit_run* r : runs) {
            Workspace& ws = r->ws;
            sadk::launch_backward(fp64, 0, ws.ids[ws.cur].p, ws.gtab.p, tgt_of(r), ws.fd, scale_n,
                                  ordered ? ws.gred_adaptive_ord() : ws.gred_adaptive(), ws.loss_part.p, ws.st.p,
                                  ws.stream);
            sadk::launch_loss_reduce(ws.loss_part.p, sadk::backward_blocks(fp64, ws.fd, ordered), r->loss_self.p,
                                     ws.stream);
            if (!ordered) sadk::launch_site_partials(ws.gred_adaptive(), ws.st.p, cap, r->gpart_self.p, ws.stream);
        }
        T.gather(runs, [](sad_fit_run* r) { return static_cast<const void*>(r->loss_self.p); },
                 [](sad_fit_run* r) { return static_cast<void*>(r->loss_all.p); }, sizeof(double2));
        // owner merge of the gradient partials; the owned totals' values feed Adam
        if (ordered) {
            owner_merge_ord(runs, T, R, slice);
            for (sad_fit_run* r : runs) {
                Workspace& ws = r->ws;
                const sadk::RedTarget red = ws.gred_adaptive_ord();
                sadk::launch_ordered_totals(red, 10, ws.st.p, r->tot.p, nullptr, false, ws.stream);
                sadk::launch_ord_finish(red, ws.st.p, ws.active.p, ws.rcap.p, ws.stream);
                ws.plan_records();
            }
        } else {
            owner_merge(
                runs, T, R, slice, 10, [](sad_fit_run* r) { return r->gpart_self.p; },
                [](sad_fit_run* r) { return r->ws.gred_adaptive(); }, true);
            for (sad_fit_run* r : runs) {
                sadk::launch_dd_values(r->gpart_self.p, 10ll * cap, r->tot.p, r->ws.stream);
                r->ws.plan_records();  // next pass's record slices from the capacities owner_pack planned
            }
        }
        if (ev) {  // stats (budget.cpp:39-155) on the strips: owner merge, then every rank gets all totals
            for (sad_fit_run* r : runs) stats_device(r->ws);
            owner_merge(
                runs, T, R, slice, 8, [](sad_fit_run* r) { return r->ws.stats.p; },
                [](sad_fit_run* r) { return r->ws.sred(); }, false);
            for (sad_fit_run* r : runs)
                sadk::launch_slice_pack<double2>(r->ws.stats.p, 8, cap, r->rank * slice, slice, r->slice_s.p, r->ws.stream);
            T.gather(runs, [](sad_fit_run* r) { return static_cast<const void*>(r->slice_s.p); },
                     [](sad_fit_run* r) { return static_cast<void*>(r->slice_all_s.p); }, sizeof(double2) * 8 * slice);
            for (sad_fit_run* r : runs)
                sadk::launch_slice_unpack<double2>(r->slice_all_s.p, 8, cap, slice, R, r->ws.stats.p, r->ws.stream);
            T.gather(runs, [](sad_fit_run* r) { return static_cast<const void*>(&r->ws.st.p->valid); },
                     [](sad_fit_run* r) { return static_cast<void*>(r->valid_all.p); }, sizeof(unsigned long long));
            for (sad_fit_run* r : runs) {
                std::vector<unsigned long long> va(R);
                ck(cudaMemcpyAsync(va.data(), r->valid_all.p, 8 * R, cudaMemcpyDeviceToHost, r->ws.stream), "D2H valid");
                ck(cudaStreamSynchronize(r->ws.stream), "valid");
                uint64_t vt = 0;
                for (unsigned long long v : va) vt += v;
                r->ws.patch_state(offsetof(DevState, valid), vt);
            }
        }
        // Adam on the owned slice of the active list, then every rank receives every slice
        for (sad_fit_run* r : runs) {
            Workspace& ws = r->ws;
            sadk::launch_owned_range(ws.act.p, ws.st.p, r->rank * slice, std::min(cap, (r->rank + 1) * slice),
                                     r->own_range.p, ws.stream);
            sadk::launch_adam(fp64, ws.sites(), ws.st.p, ws.gred_adaptive(), ws.m.p, ws.v.p, hp, r->bc_table.p,
                              make_double2(0, 0), false, scale_n, nullptr, nullptr, nullptr, ws.stream, r->tot.p, nullptr,
                              nullptr, ws.act.p, r->own_range.p);
        }
        gather_params();
        if (ev) {
            for (sad_fit_run* r : runs) {
                Workspace& ws = r->ws;
                if (ev_p) prune_device(ws, c.prune_pct * sched);
                if (ev_d) densify_device(ws, c.densify_pct * sched, c);
                ws.compute_active();
                build_tables(ws, fp64, true, true, false);
            }
            reseed();
            passes(full4, static_cast<uint32_t>(npass));
            npass += static_cast<int>(full4.size());
        } else {
            for (sad_fit_run* r : runs) build_tables(r->ws, fp64, true, true, false);
        }
        for (sad_fit_run* r : runs)
            sadk::launch_advance(r->ws.st.p, npass, 1, r->loss_hist.p, r->active_hist.p, r->loss_all.p, R,
                                 r->ws.otops.p, r->ws.stream);
    }
    // final full refresh (train.cpp:287)
    reseed();
    passes(full_refresh_passes(r0->ws.fd.gw, r0->ws.fd.gh, c.final_passes), 0);
    for (sad_fit_run* r : runs)
        sadk::launch_advance(r->ws.st.p, static_cast<int>(full_refresh_passes(r0->ws.fd.gw, r0->ws.fd.gh, c.final_passes).size()),
                             0, nullptr, nullptr, nullptr, 0, r->ws.otops.p, r->ws.stream);
    T.gather_rows(runs, r0->ws.cur);  // every rank ends with the whole final field
    cudaEventRecord(e1, r0->ws.stream);
    for (sad_fit_run* r : runs) ck(cudaStreamSynchronize(r->ws.stream), "fit strips");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (sad_fit_run* r : runs) {
        r->total_ms = ms;
        r->ws.fd.row0 = 0;  // downloads / renders of the finished run see the whole image
        r->ws.fd.row1 = 1 << 30;
        finish_run(r, ms, c.iters);
    }
}

static void strips_prepare(sad_fit_run* r, bool init_sites) {
    if (!r->have_target) fail(SAD_EINVAL, "fit: target not set");
    if (init_sites) {
        int n = initial_count(r->cfg, r->w, r->h);
        r->ws.ensure_cap(n);
        init_sites_device(r->ws, r->w, r->h, n, r->cfg);
    }
}

sad_status sad_nccl_unique_id(uint8_t* out) {
    return guard([&] {
        NcclApi& api = NcclApi::get();
        ncclUniqueId uid;
        api.check(api.getUniqueId(&uid), "ncclGetUniqueId");
        std::memcpy(out, &uid, sizeof(uid));
    });
}

struct sad_strip_comm {
    std::unique_ptr<StripComm> comm;
    int rank = 0, world = 1;
};

sad_status sad_strip_comm_create(int rank, int world, const uint8_t* nccl_id, sad_strip_comm** out) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(SAD_EINVAL, "strips: bad rank / world");
        if (!nccl_id || !out) fail(SAD_EINVAL, "strips: null argument");
        auto* c = new sad_strip_comm();
        try {
            c->comm.reset(new NcclComm(rank, world, nccl_id));
        } catch (...) {
            delete c;
            throw;
        }
        c->rank = rank;
        c->world = world;
        *out = c;
    });
}

sad_status sad_strip_comm_create_host(int rank, int world, sad_host_allgather_fn allgather,
                                      sad_host_exchange_fn exchange, void* user, sad_strip_comm** out) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(SAD_EINVAL, "strips: bad rank / world");
        if (!allgather || !exchange || !out) fail(SAD_EINVAL, "strips: null argument");
        auto* c = new sad_strip_comm();
        c->comm.reset(new HostComm(rank, world, allgather, exchange, user));
        c->rank = rank;
        c->world = world;
        *out = c;
    });
}

void sad_strip_comm_destroy(sad_strip_comm* c) { delete c; }

sad_status sad_fit_strip_exchange(sad_fit_run* r, long long* records_sent) {
    return guard([&] {
        if (!records_sent) fail(SAD_EINVAL, "strips: null argument");
        *records_sent = r->xfer_records;
    });
}

sad_status sad_fit_run_strips(sad_fit_run* r, sad_strip_comm* comm, const sad_sites_view* init) {
    return guard([&] {
        if (!comm) fail(SAD_EINVAL, "strips: null communicator");
        if (init) upload_sites(r->ws, init);
        strips_prepare(r, !init);
        r->rank = comm->rank;
        r->world = comm->world;
        std::vector<sad_fit_run*> runs{r};
        fit_loop_strips(runs, *comm->comm);
    });
}

sad_status sad_fit_run_strips_loopback(sad_fit_run* const* rs, int world) {
    return guard([&] {
        if (world < 1 || !rs) fail(SAD_EINVAL, "strips: bad world");
        std::vector<sad_fit_run*> runs(rs, rs + world);
        for (int q = 0; q < world; q++) {
            if (!runs[q] || runs[q]->ws.stream != runs[0]->ws.stream)
                fail(SAD_EINVAL, "strips loopback: runs must share one context (stream)");
            strips_prepare(runs[q], true);
            runs[q]->rank = q;
            runs[q]->world = world;
        }
        LoopbackComm comm(world);
        fit_loop_strips(runs, comm);
    });
}

sad_status sad_fit_run_init(sad_fit_run* r) {
    return guard([&] {
        if (!r->have_target) fail(SAD_EINVAL, "fit: target not set");
        int n = initial_count(r->cfg, r->w, r->h);
        r->ws.ensure_cap(n);
        init_sites_device(r->ws, r->w, r->h, n, r->cfg);
        fit_loop(r);
    });
}

sad_status sad_fit_run_store(sad_fit_run* r, const sad_sites_view* s) {
    return guard([&] {
        if (!r->have_target) fail(SAD_EINVAL, "fit: target not set");
        upload_sites(r->ws, s);
        fit_loop(r);
    });
}

sad_status sad_fit_info(sad_fit_run* r, size_t* n, int* nh, double* sc) {
    return guard([&] {
        if (!r->done) fail(SAD_EINVAL, "fit: not run");
        *n = r->n_sites;
        *nh = static_cast<int>(r->hist.size());
        *sc = r->schedule_scale;
    });
}

sad_status sad_fit_download(sad_fit_run* r, sad_sites_view* s, sad_field_view* f, sad_history_row* hist) {
    return guard([&] {
        if (!r->done) fail(SAD_EINVAL, "fit: not run");
        download_sites(r->ws, s, r->n_sites);
        if (f) {
            f->width = r->w;
            f->height = r->h;
            f->cell = 1;
            f->gw = r->ws.fd.gw;
            f->gh = r->ws.fd.gh;
            f->k = r->ws.fd.k;
            download_field(r->ws, f);
            DevState st = r->ws.get_state();
            f->pass_index = st.pass_index;
            f->synced_generation = s->generation;
            f->refresh_count = 0;
        }
        if (hist) std::copy(r->hist.begin(), r->hist.end(), hist);
    });
}

// ---- one-shot fit / fit_store (train.hpp:62-68, train.cpp:295-311) over the resident run
sad_status sad_fit_capacity(int w, int h, const sad_train_config* cfg, size_t n_init, size_t* cap) {
    return guard([&] {
        if (!cfg || !cap) fail(SAD_EINVAL, "null argument");
        sad_train_config v = *cfg;
        validate(v, w, h);
        const int n0 = n_init ? static_cast<int>(n_init) : initial_count(v, w, h);
        *cap = static_cast<size_t>(capacity_bound(v, n0, 1.0, v.target_bpp > 0));  // schedule scale <= 1
    });
}

static void fit_once(sad_ctx* c, const double* rgb, int w, int h, const sad_train_config* cfg,
                     const sad_sites_view* init, sad_sites_view* out_sites, sad_field_view* out_field,
                     sad_history_row* hist, double* scale) {
    auto chk = [](sad_status st) {
        if (st != SAD_OK) fail(st, sad_last_error());
    };
    if (!rgb || !cfg || !out_sites) fail(SAD_EINVAL, "null argument");
    sad_fit_run* r = nullptr;
    chk(sad_fit_create(c, w, h, cfg, &r));
    std::unique_ptr<sad_fit_run, void (*)(sad_fit_run*)> hold(r, sad_fit_destroy);
    chk(sad_fit_set_target(r, rgb));
    chk(init ? sad_fit_run_store(r, init) : sad_fit_run_init(r));
    size_t n = 0;
    int nh = 0;
    double sc = 0;
    chk(sad_fit_info(r, &n, &nh, &sc));
    if (out_sites->capacity < n) fail(SAD_ENOMEM, "fit: output sites capacity (see sad_fit_capacity)");
    chk(sad_fit_download(r, out_sites, out_field, hist));
    if (scale) *scale = sc;
}

sad_status sad_fit(sad_ctx* c, const double* rgb, int w, int h, const sad_train_config* cfg, sad_sites_view* out_sites,
                   sad_field_view* out_field, sad_history_row* hist, double* scale) {
    return guard([&] { fit_once(c, rgb, w, h, cfg, nullptr, out_sites, out_field, hist, scale); });
}

sad_status sad_fit_store(sad_ctx* c, const double* rgb, int w, int h, const sad_sites_view* init,
                         const sad_train_config* cfg, sad_sites_view* out_sites, sad_field_view* out_field,
                         sad_history_row* hist, double* scale) {
    return guard([&] {
        if (!init) fail(SAD_EINVAL, "fit_store: null initial sites");
        fit_once(c, rgb, w, h, cfg, init, out_sites, out_field, hist, scale);
    });
}

sad_status sad_fit_render_device(sad_fit_run* r, float* out) {
    return guard([&] {
        Workspace& ws = r->ws;
        build_tables(ws, false, false, false, true);
        sadk::launch_render(false, ws.ids[ws.cur].p, ws.rtab.p, ws.fd, norm_scale(r->w, r->h), out, ws.st.p, ws.stream);
    });
}

// Micro-benchmark of one kernel on the fitted, device-resident state (roofline evidence).
// which: 0 warm propagate pass, 1 fused fwd+bwd, 2 render, 3 Box3 flood pass (step 16), 4 Adam, 5 stats,
// 6 record-counter memsets, 7 event full refresh (seed + floods + 4 Axial passes).
sad_status sad_fit_bench(sad_fit_run* r, int which, int reps, double* ms_per_launch) {
    return guard([&] {
        if (!r->done) fail(SAD_EINVAL, "fit: not run");
        Workspace& ws = r->ws;
        const sad_train_config& c = r->cfg;
        const bool fp64 = c.fp64 != 0;
        const double sn = norm_scale(r->w, r->h);
        cudaStream_t s = ws.stream;
        build_tables(ws, fp64, true, true, false);
        build_tables(ws, false, false, false, true);
        ws.px_f.ensure(3 * static_cast<size_t>(r->w) * r->h);
        const void* tgt = fp64 ? static_cast<const void*>(ws.tgt_d.p) : static_cast<const void*>(ws.tgt_f.p);
        sadk::AdamHyper hp = adam_hyper(c, r->w, r->h);
        auto once = [&]() {
            switch (which) {
            case 0: passes_device(ws, {sad_pass_spec{1, 0}}, c.inject, c.seed, fp64, 0); break;
            case 1:  // record counters reset each launch as Adam does in the fit (memsets timed separately)
                ck(cudaMemsetAsync(ws.gcnt.p, 0, sizeof(int32_t) * ws.cap, s), "memset");
                ck(cudaMemsetAsync(ws.ghead.p, 0xff, sizeof(int32_t) * ws.cap, s), "memset");
                ck(cudaMemsetAsync(ws.otops.p, 0, sizeof(int32_t), s), "memset");
                sadk::launch_backward(fp64, 0, ws.ids[ws.cur].p, ws.gtab.p, tgt, ws.fd, sn, ws.gred_adaptive(),
                                      ws.loss_part.p, ws.st.p, s);
                break;
            case 6:
                ck(cudaMemsetAsync(ws.gcnt.p, 0, sizeof(int32_t) * ws.cap, s), "memset");
                ck(cudaMemsetAsync(ws.ghead.p, 0xff, sizeof(int32_t) * ws.cap, s), "memset");
                ck(cudaMemsetAsync(ws.otops.p, 0, sizeof(int32_t), s), "memset");
                break;
            case 2: sadk::launch_render(false, ws.ids[ws.cur].p, ws.rtab.p, ws.fd, sn, ws.px_f.p, ws.st.p, s); break;
            case 3: passes_device(ws, {sad_pass_spec{16, 1}}, c.inject, c.seed, fp64, 0); break;
            case 8: {  // one Box3 pass at SAD_BENCH_STEP (default 1) on the fitted field
                const char* e = getenv("SAD_BENCH_STEP");
                passes_device(ws, {sad_pass_spec{static_cast<uint32_t>(e ? atoi(e) : 1), 1}}, c.inject, c.seed, fp64, 0);
                break;
            }
            case 4:
                // one fwd+bwd then Adam, as in the fit (records present); the fwd+bwd share is timed apart
                sadk::launch_backward(fp64, 0, ws.ids[ws.cur].p, ws.gtab.p, tgt, ws.fd, sn, ws.gred_adaptive(),
                                      ws.loss_part.p, ws.st.p, s);
                sadk::launch_adam(fp64, ws.sites(), ws.st.p, ws.gred_adaptive(), ws.m.p, ws.v.p, hp, nullptr,
                                  make_double2(1.0, 1.0), true, sn, ws.pack.p, ws.gtab.p, ws.rcap.p, s);
                ws.plan_records();
                break;
            case 5: stats_device(ws); break;
            case 9:  // plain-iteration Adam over the active list on unchanged records (no reset, no claims)
                sadk::launch_adam(fp64, ws.sites(), ws.st.p, ws.gred_adaptive(), ws.m.p, ws.v.p, hp, nullptr,
                                  make_double2(1.0, 1.0), false, sn, ws.pack.p, ws.gtab.p, nullptr, s, nullptr,
                                  nullptr, nullptr, ws.act.p);
                break;
            case 10:  // k_advance alone (loss partials of the last backward)
                sadk::launch_advance(ws.st.p, 0, 0, nullptr, nullptr, ws.loss_part.p, sadk::backward_blocks(fp64, ws.fd),
                                     nullptr, s);
                break;
            case 7:  // one event refresh: seed + ceil(log2) Box3 floods + 4 Axial passes
                ws.cur = 0;
                sadk::launch_jfa_seed(ws.sites(), ws.st.p, ws.ids[0].p, ws.fd, sn, s);
                passes_device(ws, full_refresh_passes(ws.fd.gw, ws.fd.gh, 4), c.inject, c.seed, fp64, 0);
                break;
            default: fail(SAD_EINVAL, "bench: unknown kernel");
            }
        };
        once();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int i = 0; i < reps; i++) once();
        cudaEventRecord(b, s);
        ck(cudaEventSynchronize(b), "bench");
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *ms_per_launch = ms / std::max(reps, 1);
        if (which == 1) {  // subtract the counter reset
            double base = 0;
            sad_status rc = sad_fit_bench(r, 6, reps, &base);
            if (rc == SAD_OK) *ms_per_launch = std::max(0.0, *ms_per_launch - base);
        }
        if (which == 4) {  // Adam (+ record plan) = (fwd+bwd, Adam, plan) - fwd+bwd
            double base = 0;
            sad_status rc = sad_fit_bench(r, 1, reps, &base);
            if (rc == SAD_OK) *ms_per_launch = std::max(0.0, *ms_per_launch - base);
        }
    });
}

// Batched random-access decode against the fitted, device-resident field (pixel_weights semantics,
// render.cpp:93-105, with the table built once instead of per query).  xy/ids/w/n are DEVICE
// pointers (n_q queries; ids/w hold 16 entries per query).
sad_status sad_fit_point_query(sad_fit_run* r, const int32_t* d_xy, size_t n_q, uint32_t* d_ids, double* d_w,
                               int32_t* d_n) {
    return guard([&] {
        if (!r->done) fail(SAD_EINVAL, "fit: not run");
        Workspace& ws = r->ws;
        build_tables(ws, true, false, false, true);
        sadk::launch_pixel_weights(ws.ids[ws.cur].p, ws.rtab_d.p, ws.fd, norm_scale(r->w, r->h), d_xy,
                                   static_cast<int>(n_q), d_ids, d_w, d_n, ws.stream);
    });
}

// Decode pipeline (SPEC decode: read_file -> refresh(Full, passes) -> render_image): bytes -> sites on
// the host (exact) -> device full refresh -> device render into out_rgb (host, 3*W*H doubles).
sad_status sad_decode_render(sad_ctx* c, const uint8_t* buf, size_t n, int k, int passes, int inject, uint64_t seed,
                             int fp64, double* out_rgb, sad_sites_view* out_sites) {
    return guard([&] {
        int w = 0, h = 0;
        uint32_t count = 0;
        sad_status rc = sad_decode_header(buf, n, &w, &h, &count);
        if (rc != SAD_OK) fail(rc, sad_last_error());
        std::vector<double> p(10 * static_cast<size_t>(count) + 10);
        std::vector<uint8_t> fl(2 * static_cast<size_t>(count) + 2);
        sad_sites_view v{};
        v.capacity = count + 1;
        double** arr[10] = {&v.x, &v.y, &v.log_tau, &v.radius, &v.col_r, &v.col_g, &v.col_b, &v.dir_x, &v.dir_y, &v.aniso};
        for (int i = 0; i < 10; i++) *arr[i] = p.data() + static_cast<size_t>(i) * (count + 1);
        v.active = fl.data();
        v.frozen = fl.data() + count + 1;
        rc = sad_decode(buf, n, &v, &w, &h);
        if (rc != SAD_OK) fail(rc, sad_last_error());
        Workspace& ws = c->ws;
        upload_sites(ws, &v);
        ws.ensure_field(w, h, k, 1);
        ws.cur = 0;
        ws.patch_state(offsetof(DevState, pass_index), static_cast<uint32_t>(0));
        ws.compute_active();
        build_tables(ws, fp64 != 0, true, false, fp64 == 0);
        double sn = norm_scale(w, h);
        sadk::launch_jfa_seed(ws.sites(), ws.st.p, ws.ids[0].p, ws.fd, sn, ws.stream);
        passes_device(ws, full_refresh_passes(ws.fd.gw, ws.fd.gh, passes), inject, seed, fp64 != 0, 0);
        size_t npx = 3 * static_cast<size_t>(w) * h;
        if (fp64) {
            build_tables(ws, true, false, false, true);
            ws.px_d.ensure(npx);
            sadk::launch_render(true, ws.ids[ws.cur].p, ws.rtab_d.p, ws.fd, sn, ws.px_d.p, ws.st.p, ws.stream);
            ck(cudaMemcpyAsync(out_rgb, ws.px_d.p, npx * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H render");
        } else {
            ws.px_f.ensure(npx);
            sadk::launch_render(false, ws.ids[ws.cur].p, ws.rtab.p, ws.fd, sn, ws.px_f.p, ws.st.p, ws.stream);
            std::vector<float> tmp(npx);
            ck(cudaMemcpyAsync(tmp.data(), ws.px_f.p, npx * 4, cudaMemcpyDeviceToHost, ws.stream), "D2H render");
            ck(cudaStreamSynchronize(ws.stream), "sync");
            for (size_t i = 0; i < npx; i++) out_rgb[i] = tmp[i];
        }
        check_err(ws, "render");
        if (out_sites) {
            if (out_sites->capacity < count) fail(SAD_ENOMEM, "decode: sites view capacity too small");
            double** dst[10] = {&out_sites->x, &out_sites->y, &out_sites->log_tau, &out_sites->radius,
                                &out_sites->col_r, &out_sites->col_g, &out_sites->col_b, &out_sites->dir_x,
                                &out_sites->dir_y, &out_sites->aniso};
            for (int i = 0; i < 10; i++) std::memcpy(*dst[i], *arr[i], 8 * count);
            std::memcpy(out_sites->active, v.active, count);
            std::memcpy(out_sites->frozen, v.frozen, count);
            out_sites->size = count;
            out_sites->generation = v.generation;
        }
    });
}

void* sad_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}

void sad_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

sad_status sad_fit_set_profiling(sad_fit_run* r, int on) {
    return guard([&] { r->profile = on != 0; });
}

sad_status sad_fit_timing(sad_fit_run* r, double* total, double* ph) {
    return guard([&] {
        *total = r->total_ms;
        for (int i = 0; i < 4; i++) ph[i] = r->phase_ms[i];  // ph holds 4 phases (header contract)
    });
}

}  // extern "C"
