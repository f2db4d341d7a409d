// sad_kernels.cu — the SAD fitting-loop kernels for sm_100a.
//
// Every kernel restates one reference loop (cited per kernel) with the reference's exact operation
// order; the library is built with --fmad=false (see sad_device.cuh).  None of these steps is a
// dense contraction, so there are no tensor-core paths: the roofline is HBM / L2 bandwidth or the
// FP32/FP64 pipes.
#if SAD_ORD_DEBUG
#include <cstdio>
#endif
#include "sad_kcommon.cuh"

#ifndef SAD_EXPERIMENT
#define SAD_EXPERIMENT 0
#endif
#if SAD_EXPERIMENT == 3 || SAD_EXPERIMENT == 4
__device__ unsigned long long g_phase_clk[16];
extern "C" void sad_exp_phase(unsigned long long* out, int reset) {
    if (reset) { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_phase_clk, z, sizeof z); }
    else cudaMemcpyFromSymbol(out, g_phase_clk, 16 * sizeof(unsigned long long));
}
#endif
#if SAD_EXPERIMENT == 3
#define PH(i) do { __syncthreads(); if (threadIdx.x == 0) { long long _c = clock64(); atomicAdd(&g_phase_clk[i], (unsigned long long)(_c - _t0)); _t0 = _c; } } while (0)
#else
#define PH(i) do { } while (0)
#endif

#include <atomic>

namespace sadk {

static std::atomic<uint64_t> g_launches{0};
long long debug_check_failures() {
#if SAD_CHECKED
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, g_check_fail, sizeof v);
    return static_cast<long long>(v);
#else
    return -1;  // not a checked build
#endif
}
uint64_t launch_counter() { return g_launches.load(); }
void add_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
#define SAD_LAUNCHED() g_launches.fetch_add(1, std::memory_order_relaxed)

// ====================================================================== per-site tables
// ScoreTable<T>::build (score_table.hpp:20-46), packed and unpacked, and GradTable<T>::build
// (grad.cpp:79-111).  Coefficients are derived in double and rounded to T exactly as the reference.
template <typename T>
__global__ void k_tables(SitesDev s, const DevState* __restrict__ st, double scale, Q4<T>* __restrict__ pack,
                         Q4<T>* __restrict__ gtab, Q4<T>* __restrict__ rtab) {
    int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= st->n_sites) return;
    const int cap = s.cap;
    const double* p = s.p;
    bool act = s.active[id] != 0;
    double x = p[0 * cap + id], y = p[1 * cap + id], lt = p[2 * cap + id], r = p[3 * cap + id];
    double cr = p[4 * cap + id], cg = p[5 * cap + id], cb = p[6 * cap + id];
    double ux = p[7 * cap + id], uy = p[8 * cap + id], an = p[9 * cap + id];
    if (pack) {
        Q4<T> a, b;
        if (!act) {
            a = {T(0), T(0), T(0), T(0)};
            b = {T(1), T(0), T(1), T(0)};
        } else {
            double hx = half_rt(x), hy = half_rt(y), hlt = half_rt(lt), hr = half_rt(r);
            double hux = half_rt(ux), huy = half_rt(uy), han = half_rt(an);
            double ea = sad_dexp(han), ia = sad_dexp(-han);
            double vx = -huy, vy = hux;
            a = {static_cast<T>(hx), static_cast<T>(hy), static_cast<T>(sad_dexp(hlt)), static_cast<T>(hr)};
            b = {static_cast<T>(ea * hux * hux + ia * vx * vx), static_cast<T>(ea * hux * huy + ia * vx * vy),
                 static_cast<T>(ea * huy * huy + ia * vy * vy), T(1)};
        }
        pack[2 * id] = a;
        pack[2 * id + 1] = b;
    }
    if (gtab) {
        Q4<T> a, b, c;
        if (!act) {
            a = {T(0), T(0), T(0), T(0)};
            b = {T(1), T(1), T(1), T(0)};
            c = {T(0), T(0), T(0), T(0)};
        } else {
            a = {static_cast<T>(x), static_cast<T>(y), static_cast<T>(sad_dexp(lt)), static_cast<T>(r)};
            b = {static_cast<T>(sad_dexp(an)), static_cast<T>(sad_dexp(-an)), static_cast<T>(ux), static_cast<T>(uy)};
            c = {static_cast<T>(cr), static_cast<T>(cg), static_cast<T>(cb), T(1)};
        }
        gtab[3 * id] = a;
        gtab[3 * id + 1] = b;
        gtab[3 * id + 2] = c;
    }
    if (rtab) {
        Q4<T> a, b, c;
        if (!act) {
            a = {T(0), T(0), T(0), T(0)};
            b = {T(1), T(0), T(1), T(0)};
        } else {
            double ea = sad_dexp(an), ia = sad_dexp(-an);
            double vx = -uy, vy = ux;
            a = {static_cast<T>(x), static_cast<T>(y), static_cast<T>(sad_dexp(lt)), static_cast<T>(r)};
            b = {static_cast<T>(ea * ux * ux + ia * vx * vx), static_cast<T>(ea * ux * uy + ia * vx * vy),
                 static_cast<T>(ea * uy * uy + ia * vy * vy), T(1)};
        }
        c = {static_cast<T>(cr), static_cast<T>(cg), static_cast<T>(cb), T(0)};
        rtab[3 * id] = a;
        rtab[3 * id + 1] = b;
        rtab[3 * id + 2] = c;
    }
}

void launch_tables(bool fp64, const SitesDev& s, const DevState* st, double scale, void* pack, void* gtab,
                   void* rtab, cudaStream_t stream) {
    int grid = (s.cap + 255) / 256;
    if (grid < 1) grid = 1;
    if (fp64)
        k_tables<double><<<grid, 256, 0, stream>>>(s, st, scale, (Q4<double>*)pack, (Q4<double>*)gtab,
                                                   (Q4<double>*)rtab);
    else
        k_tables<float><<<grid, 256, 0, stream>>>(s, st, scale, (Q4<float>*)pack, (Q4<float>*)gtab,
                                                  (Q4<float>*)rtab);
    SAD_LAUNCHED();
}

// ScoreTable<T>::logit (score_table.hpp:48-54), quadratic form, no contraction.
template <typename T>
__device__ __forceinline__ T score_logit(const Q4<T>& a, const Q4<T>& b, T px, T py, T s) {
    T dx = px - a.x, dy = py - a.y;
    T q = b.x * dx * dx + T(2) * b.y * dx * dy + b.z * dy * dy;
    if (q < T(0)) q = T(0);
    T d = tsqrt(q) * s - a.w * s;
    return -a.z * d;
}

// ====================================================================== jfa_seed (candidates.cpp:64-84)
// Site -> cell scatter; a collision keeps the better double logit of the half-packed sites at the
// cell centre (ties to the lower id).  The winner is a max under a strict total order, so a CAS loop
// gives the reference's sequential result regardless of arrival order.
__device__ __forceinline__ double packed_logit_d(const SitesDev& s, uint32_t id, double cx, double cy, double scale) {
    const int cap = s.cap;
    const double* p = s.p;
    double x = half_rt(p[0 * cap + id]), y = half_rt(p[1 * cap + id]);
    double lt = half_rt(p[2 * cap + id]), r = half_rt(p[3 * cap + id]);
    double ux = half_rt(p[7 * cap + id]), uy = half_rt(p[8 * cap + id]), an = half_rt(p[9 * cap + id]);
    double ea = sad_dexp(an), ia = sad_dexp(-an);
    double vx = -uy, vy = ux;
    double gxx = ea * ux * ux + ia * vx * vx;
    double gxy = ea * ux * uy + ia * vx * vy;
    double gyy = ea * uy * uy + ia * vy * vy;
    double dx = cx - x, dy = cy - y;
    double q = gxx * dx * dx + 2.0 * gxy * dx * dy + gyy * dy * dy;
    if (q < 0) q = 0;
    double d = __dsqrt_rn(q) * scale - r * scale;
    return -sad_dexp(lt) * d;
}

__global__ void k_jfa_seed(SitesDev s, const DevState* __restrict__ st, uint32_t* __restrict__ ids, FieldDims f,
                           double scale) {
    int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= st->n_sites || !s.active[id]) return;
    long long px = llround(s.p[0 * s.cap + id]);
    long long py = llround(s.p[1 * s.cap + id]);
    px = px < 0 ? 0 : (px > f.width - 1 ? f.width - 1 : px);
    py = py < 0 ? 0 : (py > f.height - 1 ? f.height - 1 : py);
    int gx = static_cast<int>(px) / f.cell, gy = static_cast<int>(py) / f.cell;
    uint32_t* slot = ids + static_cast<size_t>(f.k) * (static_cast<size_t>(gy) * f.gw + gx);
    uint32_t cur = atomicCAS(slot, kEmpty, static_cast<uint32_t>(id));
    if (cur == kEmpty) return;
    double cx = gx * static_cast<double>(f.cell) + (f.cell - 1) * 0.5;
    double cy = gy * static_cast<double>(f.cell) + (f.cell - 1) * 0.5;
    double mine = packed_logit_d(s, id, cx, cy, scale);
    while (true) {
        double other = packed_logit_d(s, cur, cx, cy, scale);
        bool better = mine > other || (mine == other && static_cast<uint32_t>(id) < cur);
        if (!better) return;
        uint32_t prev = atomicCAS(slot, cur, static_cast<uint32_t>(id));
        if (prev == cur) return;
        cur = prev;
    }
}

void launch_jfa_seed(const SitesDev& s, const DevState* st, uint32_t* ids, const FieldDims& f, double scale,
                     cudaStream_t stream) {
    cudaMemsetAsync(ids, 0xff, sizeof(uint32_t) * static_cast<size_t>(f.gw) * f.gh * f.k, stream);
    int grid = (s.cap + 255) / 256;
    if (grid < 1) grid = 1;
    k_jfa_seed<<<grid, 256, 0, stream>>>(s, st, ids, f, scale);
    SAD_LAUNCHED();
}

// ====================================================================== top-K list in registers
// TopK<T>::consider (score_table.hpp:67-80) with static register indexing: the position search
// walks back from n exactly like the reference's while-loop (so even unordered NaN entries behave
// identically), and the shift is a predicated select chain.
template <typename T>
__device__ __forceinline__ bool better(T l, uint32_t c, T L, uint32_t C) {
    return l > L || (l == L && c < C);
}

template <typename T, int KM, bool EXACT>
struct TopKReg {
    uint32_t id[KM];
    T lg[KM];
    int n;
    int k;  // runtime list length (== KM when EXACT)

    __device__ __forceinline__ void init(int kk) {
        n = 0;
        k = EXACT ? KM : kk;
#pragma unroll
        for (int i = 0; i < KM; i++) {
            id[i] = kEmpty;
            lg[i] = T(0);
        }
    }
    __device__ __forceinline__ bool contains(uint32_t c) const {
        bool d = false;
#pragma unroll
        for (int i = 0; i < KM; i++) d |= (id[i] == c);
        return d;
    }
    // Reject fast when the list is full and (l, c) does not beat the last entry.
    __device__ __forceinline__ bool full_reject(T l, uint32_t c) const {
        if (EXACT) return n == KM && !better(l, c, lg[KM - 1], id[KM - 1]);
        return false;
    }
    __device__ __forceinline__ void consider(uint32_t c, T l) {
        int pos = n;
        bool run = true;
#pragma unroll
        for (int i = KM - 1; i >= 0; i--) {
            if (i < n) {
                run = run && better(l, c, lg[i], id[i]);
                if (run) pos = i;
            }
        }
        if (pos >= k) return;
#pragma unroll
        for (int i = KM - 1; i >= 0; i--) {
            if (i > pos) {
                if (i < k) {
                    id[i] = id[i - 1];
                    lg[i] = lg[i - 1];
                }
            } else if (i == pos) {
                id[i] = c;
                lg[i] = l;
            }
        }
        if (n < k) n++;
    }
};

// ====================================================================== propagate (candidates.cpp:92-141)
// One thread per candidate cell.  Gathers self + 4 (Axial) or 8 (Box3) neighbour lists at +-step,
// stopping each at its first sentinel and dropping inactive ids, then `inject` ids drawn from the
// reference's per-(seed, pass, cell) xorshift stream; keeps the top-K under (logit desc, id asc).
// Deduplication is streaming: a candidate already in the running list is skipped, which yields
// the reference's set-based result because the list's K-th key only ever improves.
template <typename T, int KM, bool EXACT, bool BOX>
__device__ __forceinline__ void propagate_cell(const uint32_t* __restrict__ prev, uint32_t* __restrict__ next,
                                               const Q4<T>* __restrict__ pack, const uint32_t* __restrict__ act,
                                               const DevState* __restrict__ st, const FieldDims& f, int gx, int gy,
                                               int step, int inject, uint64_t seed, uint32_t pass_offset, T s) {
    const int k = EXACT ? KM : f.k;
    const T cx = static_cast<T>(gx * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    const T cy = static_cast<T>(gy * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    TopKReg<T, KM, EXACT> sel;
    sel.init(k);

    auto consider = [&](uint32_t c) {
        if (sel.contains(c)) return;
        const Q4<T> a = pack[2 * c];
        const Q4<T> b = pack[2 * c + 1];
        if (b.w == T(0)) return;  // inactive: dropped on the way in (candidates.cpp:110)
        T l = score_logit(a, b, cx, cy, s);
        if (sel.full_reject(l, c)) return;
        sel.consider(c, l);
    };

    constexpr int NOFF = BOX ? 9 : 5;
#pragma unroll 1
    for (int o = 0; o < NOFF; o++) {
        // kAxialOff / kBoxOff order (candidates.cpp:88-90)
        int ox = (o == 1 || o == 5 || o == 6) ? 1 : ((o == 2 || o == 7 || o == 8) ? -1 : 0);
        int oy = (o == 3 || o == 5 || o == 7) ? 1 : ((o == 4 || o == 6 || o == 8) ? -1 : 0);
        int nx = gx + ox * step, ny = gy + oy * step;
        if (nx < 0 || ny < 0 || nx >= f.gw || ny >= f.gh) continue;
        const uint32_t* lst = prev + static_cast<size_t>(k) * (static_cast<size_t>(ny) * f.gw + nx);
        if (EXACT && (KM % 4) == 0) {
            uint32_t v[KM];
#pragma unroll
            for (int q = 0; q < KM / 4; q++) {
                uint4 u = __ldg(reinterpret_cast<const uint4*>(lst) + q);
                v[4 * q] = u.x;
                v[4 * q + 1] = u.y;
                v[4 * q + 2] = u.z;
                v[4 * q + 3] = u.w;
            }
#pragma unroll
            for (int i = 0; i < KM; i++) {
                if (v[i] == kEmpty) break;
                consider(v[i]);
            }
        } else {
            for (int i = 0; i < k; i++) {
                uint32_t c = __ldg(lst + i);
                if (c == kEmpty) break;
                consider(c);
            }
        }
    }
    const int n_act = st->n_active;
    if (inject > 0 && n_act > 0) {
        uint32_t rs = seeded_state(seed, st->pass_index + pass_offset,
                                   static_cast<uint32_t>(gy) * static_cast<uint32_t>(f.gw) + static_cast<uint32_t>(gx));
#pragma unroll 1
        for (int j = 0; j < inject; j++) consider(__ldg(act + xs_next(rs) % static_cast<uint32_t>(n_act)));
    }
    uint32_t* out = next + static_cast<size_t>(k) * (static_cast<size_t>(gy) * f.gw + gx);
    if (EXACT && (KM % 4) == 0) {
#pragma unroll
        for (int q = 0; q < KM / 4; q++)
            reinterpret_cast<uint4*>(out)[q] = make_uint4(sel.id[4 * q], sel.id[4 * q + 1], sel.id[4 * q + 2],
                                                          sel.id[4 * q + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < KM; i++)
            if (i < k) out[i] = sel.id[i];
    }
}

template <typename T, int KM, bool EXACT, bool BOX>
__global__ void __launch_bounds__(256) k_propagate(const uint32_t* __restrict__ prev, uint32_t* __restrict__ next,
                                                   const Q4<T>* __restrict__ pack, const uint32_t* __restrict__ act,
                                                   const DevState* __restrict__ st, FieldDims f, int step, int inject,
                                                   uint64_t seed, uint32_t pass_offset, T s) {
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = blockIdx.y * blockDim.y + threadIdx.y + f.row0;
    if (gx >= f.gw || gy >= f.gh || gy >= f.row1) return;
    propagate_cell<T, KM, EXACT, BOX>(prev, next, pack, act, st, f, gx, gy, step, inject, seed, pass_offset, s);
}

// Rare-path fallback of the key kernels below (a NaN logit or a repeated id in the own list): the
// cell is recomputed by the streaming kernel body in the reference's feed order.
template <bool BOX>
__device__ __noinline__ void propagate_cell_slow(const uint32_t* __restrict__ prev, uint32_t* __restrict__ next,
                                                 const Q4<float>* __restrict__ pack, const uint32_t* __restrict__ act,
                                                 const DevState* __restrict__ st, FieldDims f, int gx, int gy, int step,
                                                 int inject, uint64_t seed, uint32_t pass_offset, float s) {
    propagate_cell<float, 8, true, BOX>(prev, next, pack, act, st, f, gx, gy, step, inject, seed, pass_offset, s);
}

// Propagate pass specialised for K = 8 (Axial: 4 neighbour lists; Box3: 8).  Same map as
// k_propagate, fewer divergent slots: the cell's own list is scored and ordered with an 8-input
// sorting network (the insertion sort of TopK::consider yields the same order for distinct, finite
// keys); the neighbour entries not already in the running list go, four lists at a time, into a
// per-thread shared-memory queue (the injected ids join the last round), and only the queue is
// scored and inserted.  The TopK result over a set of distinct candidates does not depend on feed
// order (strict total order), and a repeated candidate is either in the list (skipped) or worse
// than the current K-th (the K-th key only improves), so the map equals the reference's
// first-appearance pool (candidates.cpp:108-135).  Own lists with a repeated id or a non-finite
// logit take the generic streaming path.  List loads are issued two lists at a time and the queue
// drain prefetches the next candidate's table rows while the current one is scored.
constexpr int kAxQ = 36;  // 4 neighbour lists x 8 + 4 injected (larger inject: generic kernel)

template <typename T>
__device__ __forceinline__ void cex(T& la, uint32_t& ia, T& lb, uint32_t& ib) {
    // after the exchange (la, ia) is the better of the two under (logit desc, id asc)
    bool sw = better(lb, ib, la, ia);
    T tl = sw ? lb : la;
    uint32_t ti = sw ? ib : ia;
    lb = sw ? la : lb;
    ib = sw ? ia : ib;
    la = tl;
    ia = ti;
}

// kAxialOff / kBoxOff (candidates.cpp:88-90), offsets 1..8
__device__ __forceinline__ int off_x(int o) { return (o == 1 || o == 5 || o == 6) ? 1 : ((o == 2 || o == 7 || o == 8) ? -1 : 0); }
__device__ __forceinline__ int off_y(int o) { return (o == 3 || o == 5 || o == 7) ? 1 : ((o == 4 || o == 6 || o == 8) ? -1 : 0); }

template <typename T, bool BOX>
__global__ void __launch_bounds__(256) k_propagate_k8(const uint32_t* __restrict__ prev, uint32_t* __restrict__ next,
                                                      const Q4<T>* __restrict__ pack, const uint32_t* __restrict__ act,
                                                      const DevState* __restrict__ st, FieldDims f, int step,
                                                      int inject, uint64_t seed, uint32_t pass_offset, T s) {
    __shared__ uint32_t q[kAxQ * 256];
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = blockIdx.y * blockDim.y + threadIdx.y + f.row0;
    if (gx >= f.gw || gy >= f.gh || gy >= f.row1) return;
    const T cx = static_cast<T>(gx * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    const T cy = static_cast<T>(gy * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    TopKReg<T, 8, true> sel;
    sel.init(8);

    // ---- own list: score, then sort with a network
    const uint32_t* own = prev + 8 * (static_cast<size_t>(gy) * f.gw + gx);
    uint4 o0 = __ldg(reinterpret_cast<const uint4*>(own)), o1 = __ldg(reinterpret_cast<const uint4*>(own) + 1);
    uint32_t oid[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
    T ol[8];
    bool stop = false, fallback = false;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        stop = stop || oid[i] == kEmpty;
        ol[i] = -INFINITY;
        if (!stop) {
            const Q4<T> a = pack[2 * oid[i]], b = pack[2 * oid[i] + 1];
            if (b.w != T(0)) {
                ol[i] = score_logit(a, b, cx, cy, s);
                fallback |= !isfinite(static_cast<double>(ol[i]));
            } else {
                oid[i] = kEmpty;  // inactive: dropped
            }
        } else {
            oid[i] = kEmpty;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = i + 1; j < 8; j++) fallback |= (oid[i] != kEmpty && oid[i] == oid[j]);
    if (!fallback) {
        // Batcher odd-even merge sort, 19 comparators; kEmpty entries carry -inf and sort last
        cex(ol[0], oid[0], ol[1], oid[1]); cex(ol[2], oid[2], ol[3], oid[3]);
        cex(ol[4], oid[4], ol[5], oid[5]); cex(ol[6], oid[6], ol[7], oid[7]);
        cex(ol[0], oid[0], ol[2], oid[2]); cex(ol[1], oid[1], ol[3], oid[3]);
        cex(ol[4], oid[4], ol[6], oid[6]); cex(ol[5], oid[5], ol[7], oid[7]);
        cex(ol[1], oid[1], ol[2], oid[2]); cex(ol[5], oid[5], ol[6], oid[6]);
        cex(ol[0], oid[0], ol[4], oid[4]); cex(ol[1], oid[1], ol[5], oid[5]);
        cex(ol[2], oid[2], ol[6], oid[6]); cex(ol[3], oid[3], ol[7], oid[7]);
        cex(ol[2], oid[2], ol[4], oid[4]); cex(ol[3], oid[3], ol[5], oid[5]);
        cex(ol[1], oid[1], ol[2], oid[2]); cex(ol[3], oid[3], ol[4], oid[4]);
        cex(ol[5], oid[5], ol[6], oid[6]);
        int n = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            sel.id[i] = oid[i];
            sel.lg[i] = oid[i] == kEmpty ? T(0) : ol[i];
            n += oid[i] != kEmpty;
        }
        sel.n = n;
    } else {
        // generic streaming insertion in list order (reference semantics incl. NaN)
#pragma unroll
        for (int i = 0; i < 8; i++) {
            uint32_t c = oid[i];
            if (c == kEmpty || sel.contains(c)) continue;
            sel.consider(c, ol[i]);
        }
    }

    const int n_act = st->n_active;
    constexpr int NG = BOX ? 2 : 1;
#pragma unroll 1
    for (int g = 0; g < NG; g++) {
        // ---- neighbour entries not already in the list (two lists per load batch)
        int nq = 0;
#pragma unroll 1
        for (int pr = 0; pr < 2; pr++) {
            uint4 u[4];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int o = 1 + 4 * g + 2 * pr + h;
                const int nx = gx + off_x(o) * step, ny = gy + off_y(o) * step;
                if (nx >= 0 && ny >= 0 && nx < f.gw && ny < f.gh) {
                    const uint4* lst = reinterpret_cast<const uint4*>(prev + 8 * (static_cast<size_t>(ny) * f.gw + nx));
                    u[2 * h] = __ldg(lst);
                    u[2 * h + 1] = __ldg(lst + 1);
                } else {
                    u[2 * h] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
                    u[2 * h + 1] = u[2 * h];
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t v[8] = {u[2 * h].x, u[2 * h].y, u[2 * h].z, u[2 * h].w,
                                       u[2 * h + 1].x, u[2 * h + 1].y, u[2 * h + 1].z, u[2 * h + 1].w};
                bool end = false;
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    end = end || v[i] == kEmpty;
                    if (!end && !sel.contains(v[i])) q[nq++ * 256 + tid] = v[i];
                }
            }
        }
        if (g == NG - 1 && inject > 0 && n_act > 0) {
            uint32_t rs = seeded_state(seed, st->pass_index + pass_offset,
                                       static_cast<uint32_t>(gy) * static_cast<uint32_t>(f.gw) + static_cast<uint32_t>(gx));
            for (int j = 0; j < inject; j++)
                q[nq++ * 256 + tid] = __ldg(act + xs_next(rs) % static_cast<uint32_t>(n_act));
        }
        // ---- score and insert the queue; the next entry's rows are in flight meanwhile
        if (nq > 0) {
            uint32_t c = q[tid];
            Q4<T> b = pack[2 * c + 1], a = pack[2 * c];
#pragma unroll 1
            for (int j = 0; j < nq; j++) {
                const uint32_t cn = j + 1 < nq ? q[(j + 1) * 256 + tid] : c;
                const Q4<T> bn = pack[2 * cn + 1], an = pack[2 * cn];
                if (b.w != T(0) && !sel.contains(c)) {
                    const T l = score_logit(a, b, cx, cy, s);
                    if (!sel.full_reject(l, c)) sel.consider(c, l);
                }
                c = cn;
                a = an;
                b = bn;
            }
        }
    }
    uint4* out = reinterpret_cast<uint4*>(next + 8 * (static_cast<size_t>(gy) * f.gw + gx));
    out[0] = make_uint4(sel.id[0], sel.id[1], sel.id[2], sel.id[3]);
    out[1] = make_uint4(sel.id[4], sel.id[5], sel.id[6], sel.id[7]);
}

#ifndef SAD_QUEUE_BY
#define SAD_QUEUE_BY 4  // block height of the queue kernels (32 x BY threads)
#endif
#ifndef SAD_PROP_MINB
#define SAD_PROP_MINB 4
#endif
// ---------------------------------------------------------------------- K = 8, fp32, 64-bit keys
// A list entry (logit l, id c) is one u64 key: the order-preserving bits of l (with -0 folded onto
// +0, so equal logits tie exactly as in TopK) in the high word and ~c in the low word.  Larger key
// <=> better under (logit desc, id asc), every real key is > 0 (the most negative finite float maps
// to 0x00800000), and an empty slot is key 0 whose low word decodes to kEmpty.  `better` becomes
// one 64-bit compare, the K-th rejection test one compare, and the sorted insertion eight compares
// plus selects with no position search.  Only a NaN logit (no order) or a repeated id in the own
// list leaves this representation; such a cell is recomputed by propagate_cell_slow.
__device__ __forceinline__ uint64_t list_key(float l, uint32_t c) {
    uint32_t u = __float_as_uint(__fadd_rn(l, 0.0f));
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return (static_cast<uint64_t>(u) << 32) | static_cast<uint32_t>(~c);
}

struct KeyList8 {
    uint64_t k[8];
    __device__ __forceinline__ bool contains(uint32_t c) const {
        // ~c through an opaque `not`: otherwise the compiler folds every compare into (k ^ c) == -1,
        // two instructions each instead of one ISETP
        uint32_t nc;
        asm("not.b32 %0, %1;" : "=r"(nc) : "r"(c));
        bool d = false;
#pragma unroll
        for (int i = 0; i < 8; i++) d |= (static_cast<uint32_t>(k[i]) == nc);
        return d;
    }
    // x must beat k[7] and must not be in the list
    __device__ __forceinline__ void insert(uint64_t x) {
        bool b[8];
#pragma unroll
        for (int i = 0; i < 8; i++) b[i] = x > k[i];
#pragma unroll
        for (int i = 7; i >= 1; i--) k[i] = b[i - 1] ? k[i - 1] : (b[i] ? x : k[i]);
        k[0] = b[0] ? x : k[0];
    }
    __device__ __forceinline__ void consider(uint32_t c, uint64_t x) {
#if SAD_EXPERIMENT == 4
        atomicAdd(&g_phase_clk[0], 1ull);
        if (x > k[7]) atomicAdd(&g_phase_clk[1], 1ull);
        if (x > k[7] && !contains(c)) atomicAdd(&g_phase_clk[2], 1ull);
#endif
        if (x > k[7] && !contains(c)) insert(x);
    }
};

__device__ __forceinline__ void kcex(uint64_t& a, uint64_t& b) {  // a <- max, b <- min
    const uint64_t hi = a > b ? a : b, lo = a > b ? b : a;
    a = hi;
    b = lo;
}

// Own list -> sorted keys.  Returns false when the slow path is needed (NaN logit, repeated id).
__device__ __forceinline__ bool own_keys(const uint32_t* __restrict__ prev, const Q4<float>* __restrict__ pack,
                                         const FieldDims& f, int gx, int gy, float cx, float cy, float s,
                                         KeyList8& L) {
    const uint4* own = reinterpret_cast<const uint4*>(prev + 8 * (static_cast<size_t>(gy) * f.gw + gx));
    const uint4 o0 = __ldg(own), o1 = __ldg(own + 1);
    const uint32_t oid[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
    bool stop = false, ok = true;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        stop = stop || oid[i] == kEmpty;
        L.k[i] = 0;
        if (!stop) {
            const Q4<float> a = pack[2 * oid[i]], b = pack[2 * oid[i] + 1];
            if (b.w != 0.0f) {
                const float l = score_logit(a, b, cx, cy, s);
                ok &= (l == l);
                L.k[i] = list_key(l, oid[i]);
            }
        }
    }
    // Batcher odd-even merge sort (descending), 19 comparators
    kcex(L.k[0], L.k[1]); kcex(L.k[2], L.k[3]); kcex(L.k[4], L.k[5]); kcex(L.k[6], L.k[7]);
    kcex(L.k[0], L.k[2]); kcex(L.k[1], L.k[3]); kcex(L.k[4], L.k[6]); kcex(L.k[5], L.k[7]);
    kcex(L.k[1], L.k[2]); kcex(L.k[5], L.k[6]);
    kcex(L.k[0], L.k[4]); kcex(L.k[1], L.k[5]); kcex(L.k[2], L.k[6]); kcex(L.k[3], L.k[7]);
    kcex(L.k[2], L.k[4]); kcex(L.k[3], L.k[5]);
    kcex(L.k[1], L.k[2]); kcex(L.k[3], L.k[4]); kcex(L.k[5], L.k[6]);
    // a repeated id has a repeated key, adjacent after sorting
#pragma unroll
    for (int i = 0; i < 7; i++) ok &= !(L.k[i] != 0 && L.k[i] == L.k[i + 1]);
    return ok;
}

__device__ __forceinline__ void store_keys(uint32_t* __restrict__ next, const FieldDims& f, int gx, int gy,
                                           const KeyList8& L) {
    uint4* out = reinterpret_cast<uint4*>(next + 8 * (static_cast<size_t>(gy) * f.gw + gx));
    out[0] = make_uint4(~static_cast<uint32_t>(L.k[0]), ~static_cast<uint32_t>(L.k[1]), ~static_cast<uint32_t>(L.k[2]),
                        ~static_cast<uint32_t>(L.k[3]));
    out[1] = make_uint4(~static_cast<uint32_t>(L.k[4]), ~static_cast<uint32_t>(L.k[5]), ~static_cast<uint32_t>(L.k[6]),
                        ~static_cast<uint32_t>(L.k[7]));
}

// Streaming variant (Box3 floods): every neighbour entry is scored first, then tested against the
// K-th key, and only the survivors are deduplicated against the list — at flood steps most entries
// are new sites, so dedup-first would be wasted work.
template <bool BOX>
__global__ void __launch_bounds__(256, SAD_PROP_MINB) k_prop8_stream(const uint32_t* __restrict__ prev, uint32_t* __restrict__ next,
                                                      const Q4<float>* __restrict__ pack,
                                                      const uint32_t* __restrict__ act, const DevState* __restrict__ st,
                                                      FieldDims f, int step, int inject, uint64_t seed,
                                                      uint32_t pass_offset, float s) {
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = blockIdx.y * blockDim.y + threadIdx.y + f.row0;
    if (gx >= f.gw || gy >= f.gh || gy >= f.row1) return;
    const float cx = static_cast<float>(gx * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    const float cy = static_cast<float>(gy * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    KeyList8 L;
    bool ok = own_keys(prev, pack, f, gx, gy, cx, cy, s, L);
    auto feed = [&](uint32_t c) {
        SAD_CHECK(c < static_cast<uint32_t>(st->n_sites));
        const Q4<float> b = pack[2 * c + 1], a = pack[2 * c];
        if (b.w == 0.0f) return;
        const float l = score_logit(a, b, cx, cy, s);
        ok &= (l == l);
        L.consider(c, list_key(l, c));
    };
    constexpr int NOFF = BOX ? 9 : 5;
    // the next neighbour list is in flight while the current one is scored
    auto load = [&](int o, uint4& u0, uint4& u1) {
        const int nx = gx + off_x(o) * step, ny = gy + off_y(o) * step;
        if (nx < 0 || ny < 0 || nx >= f.gw || ny >= f.gh) {
            u0 = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
            u1 = u0;
            return;
        }
        const uint4* lst = reinterpret_cast<const uint4*>(prev + 8 * (static_cast<size_t>(ny) * f.gw + nx));
        u0 = __ldg(lst);
        u1 = __ldg(lst + 1);
    };
    uint4 u0, u1;
    load(1, u0, u1);
#pragma unroll 1
    for (int o = 1; o < NOFF; o++) {
        const uint32_t v[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
        if (o + 1 < NOFF) load(o + 1, u0, u1);
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (v[i] == kEmpty) break;
            feed(v[i]);
        }
    }
    const int n_act = st->n_active;
    if (inject > 0 && n_act > 0) {
        uint32_t rs = seeded_state(seed, st->pass_index + pass_offset,
                                   static_cast<uint32_t>(gy) * static_cast<uint32_t>(f.gw) + static_cast<uint32_t>(gx));
#pragma unroll 1
        for (int j = 0; j < inject; j++) feed(__ldg(act + xs_next(rs) % static_cast<uint32_t>(n_act)));
    }
    if (ok)
        store_keys(next, f, gx, gy, L);
    else
        propagate_cell_slow<BOX>(prev, next, pack, act, st, f, gx, gy, step, inject, seed, pass_offset, s);
}

// Queue variant (warm Axial passes): most neighbour entries are already in the own list, so they are
// filtered by id first and only the rest (plus the injected ids) go through a per-thread shared
// queue that is scored convergently, with the next entry's table rows prefetched.
template <bool BOX>
__global__ void __launch_bounds__(32 * SAD_QUEUE_BY, SAD_PROP_MINB * 8 / SAD_QUEUE_BY) k_prop8_queue(const uint32_t* __restrict__ prev, uint32_t* __restrict__ next,
                                                     const Q4<float>* __restrict__ pack,
                                                     const uint32_t* __restrict__ act, const DevState* __restrict__ st,
                                                     FieldDims f, int step, int inject, uint64_t seed,
                                                     uint32_t pass_offset, float s) {
    pdl_enter<1>();
    constexpr int QB = 32 * SAD_QUEUE_BY;  // threads per block = per-thread queue stride
    __shared__ uint32_t q[kAxQ * QB];
    // this thread's queue column as a shared-window address
    const uint32_t qa = static_cast<uint32_t>(__cvta_generic_to_shared(q + (threadIdx.y * blockDim.x + threadIdx.x)));
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = blockIdx.y * blockDim.y + threadIdx.y + f.row0;
    if (gx >= f.gw || gy >= f.gh || gy >= f.row1) return;
    const float cx = static_cast<float>(gx * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    const float cy = static_cast<float>(gy * static_cast<double>(f.cell) + (f.cell - 1) * 0.5);
    // injected ids first: their act[] loads overlap the own-list scoring, they take queue slots
    // [0, ni) (drained with the last group) and their table rows are prefetched into L1 long before
    // the drain reaches them (random ids: the rows are rarely L1-resident otherwise)
    const int n_act = st->n_active;
    const int ni = (inject > 0 && n_act > 0) ? inject : 0;
    uint32_t inj[4];
    if (ni > 0) {
        uint32_t rs = seeded_state(seed, st->pass_index + pass_offset,
                                   static_cast<uint32_t>(gy) * static_cast<uint32_t>(f.gw) + static_cast<uint32_t>(gx));
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (j < ni) inj[j] = __ldg(act + xs_next(rs) % static_cast<uint32_t>(n_act));
    }
    KeyList8 L;
    bool ok = own_keys(prev, pack, f, gx, gy, cx, cy, s, L);
#pragma unroll
    for (int j = 0; j < 4; j++)
        if (j < ni) {
            q[j * QB + tid] = inj[j];
            asm volatile("prefetch.global.L1 [%0];" :: "l"(pack + 2 * inj[j]));
        }
    constexpr int NG = BOX ? 2 : 1;  // groups of four neighbour lists (Box3: axial, then diagonal)
#pragma unroll 1
    for (int g = 0; g < NG; g++) {
        int nq = ni;
        const int j0 = g == NG - 1 ? 0 : ni;  // the injected slots are drained once, with the last group
#pragma unroll 1
        for (int pr = 0; pr < 2; pr++) {
            uint4 u[4];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int o = 1 + 4 * g + 2 * pr + h;
                const int nx = gx + off_x(o) * step, ny = gy + off_y(o) * step;
                if (nx >= 0 && ny >= 0 && nx < f.gw && ny < f.gh) {
                    const uint4* lst = reinterpret_cast<const uint4*>(prev + 8 * (static_cast<size_t>(ny) * f.gw + nx));
                    u[2 * h] = __ldg(lst);
                    u[2 * h + 1] = __ldg(lst + 1);
                } else {
                    u[2 * h] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
                    u[2 * h + 1] = u[2 * h];
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t v[8] = {u[2 * h].x, u[2 * h].y, u[2 * h].z, u[2 * h].w,
                                       u[2 * h + 1].x, u[2 * h + 1].y, u[2 * h + 1].z, u[2 * h + 1].w};
                bool end = false;
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    end = end || v[i] == kEmpty;
                    const bool push = !end && !L.contains(v[i]);
                    // predicated st.shared at the precomputed queue address: no branch, no re-derivation
                    // of the shared window per entry
                    asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.u32 [%0], %1; }"
                                 :: "r"(qa + 4u * QB * static_cast<uint32_t>(nq)), "r"(v[i]), "r"(static_cast<uint32_t>(push))
                                 : "memory");
                    nq += push;
                }
            }
        }
        if (nq > j0) {
            uint32_t c = q[j0 * QB + tid];
            Q4<float> b = pack[2 * c + 1], a = pack[2 * c];
#pragma unroll 1
            for (int j = j0; j < nq; j++) {
                SAD_CHECK(c < static_cast<uint32_t>(st->n_sites));
                const uint32_t cn = j + 1 < nq ? q[(j + 1) * QB + tid] : c;
                const Q4<float> bn = pack[2 * cn + 1], an = pack[2 * cn];
                if (b.w != 0.0f) {
                    const float l = score_logit(a, b, cx, cy, s);
                    ok &= (l == l);
                    L.consider(c, list_key(l, c));
                }
                c = cn;
                a = an;
                b = bn;
            }
        }
    }
    if (ok)
        store_keys(next, f, gx, gy, L);
    else
        propagate_cell_slow<BOX>(prev, next, pack, act, st, f, gx, gy, step, inject, seed, pass_offset, s);
}

template <typename T, int KM, bool EXACT>
static void propagate_t(const uint32_t* prev, uint32_t* next, const void* pack, const uint32_t* act,
                        const DevState* st, const FieldDims& f, uint32_t step, int box, int inject, uint64_t seed,
                        uint32_t pass_offset, double scale, cudaStream_t stream) {
    dim3 block(32, 8);
    dim3 grid((f.gw + 31) / 32, (rows_of(f, f.gh) + 7) / 8);
    if (box)
        k_propagate<T, KM, EXACT, true><<<grid, block, 0, stream>>>(prev, next, (const Q4<T>*)pack, act, st, f,
                                                                    (int)step, inject, seed, pass_offset,
                                                                    static_cast<T>(scale));
    else
        k_propagate<T, KM, EXACT, false><<<grid, block, 0, stream>>>(prev, next, (const Q4<T>*)pack, act, st, f,
                                                                     (int)step, inject, seed, pass_offset,
                                                                     static_cast<T>(scale));
    SAD_LAUNCHED();
}

#ifndef SAD_STREAM_BY
#define SAD_STREAM_BY 4  // block height of the streaming Box3 kernel (32 x BY threads)
#endif
// largest Box3 step that uses the dedup-first queue kernel (SAD_BOX_QUEUE_STEP overrides, for A/B)
static const int g_box_queue_max_step = getenv("SAD_BOX_QUEUE_STEP") ? atoi(getenv("SAD_BOX_QUEUE_STEP")) : 4;

void launch_propagate(bool fp64, const uint32_t* prev, uint32_t* next, const void* pack, const uint32_t* act,
                      const DevState* st, const FieldDims& f, uint32_t step, int box, int inject, uint64_t seed,
                      uint32_t pass_offset, double scale, cudaStream_t stream) {
    if (f.k == 8 && !fp64) {
        dim3 block(32, 8);
        dim3 grid((f.gw + 31) / 32, (rows_of(f, f.gh) + 7) / 8);
        const float sf = static_cast<float>(scale);
        // Box3 floods at small steps see mostly ids already in the cell's list: dedup first (queue);
        // at larger steps most entries are new sites: score first (stream)
        if (box && (inject > 4 || step > g_box_queue_max_step))
            k_prop8_stream<true><<<dim3(grid.x, (rows_of(f, f.gh) + SAD_STREAM_BY - 1) / SAD_STREAM_BY),
                                   dim3(32, SAD_STREAM_BY), 0, stream>>>(prev, next, (const Q4<float>*)pack, act, st, f, (int)step,
                                                             inject, seed, pass_offset, sf);
        else if (box)
            launch_pdl(k_prop8_queue<true>, dim3(grid.x, (rows_of(f, f.gh) + SAD_QUEUE_BY - 1) / SAD_QUEUE_BY),
                       dim3(32, SAD_QUEUE_BY), 0, stream, prev, next, (const Q4<float>*)pack, act, st, f, (int)step,
                       inject, seed, pass_offset, sf);
        else if (inject <= 4)
            launch_pdl(k_prop8_queue<false>, dim3(grid.x, (rows_of(f, f.gh) + SAD_QUEUE_BY - 1) / SAD_QUEUE_BY),
                       dim3(32, SAD_QUEUE_BY), 0, stream, prev, next, (const Q4<float>*)pack, act, st, f, (int)step,
                       inject, seed, pass_offset, sf);
        else
            k_prop8_stream<false><<<grid, block, 0, stream>>>(prev, next, (const Q4<float>*)pack, act, st, f,
                                                              (int)step, inject, seed, pass_offset, sf);
        SAD_LAUNCHED();
        return;
    }
    if (f.k == 8 && inject <= 4 && !box) {
        dim3 block(32, 8);
        dim3 grid((f.gw + 31) / 32, (rows_of(f, f.gh) + 7) / 8);
        k_propagate_k8<double, false><<<grid, block, 0, stream>>>(prev, next, (const Q4<double>*)pack, act, st, f,
                                                                 (int)step, inject, seed, pass_offset, scale);
        SAD_LAUNCHED();
        return;
    }
    if (f.k == 8) {
        if (fp64)
            propagate_t<double, 8, true>(prev, next, pack, act, st, f, step, box, inject, seed, pass_offset, scale,
                                         stream);
        else
            propagate_t<float, 8, true>(prev, next, pack, act, st, f, step, box, inject, seed, pass_offset, scale,
                                        stream);
    } else {
        if (fp64)
            propagate_t<double, 16, false>(prev, next, pack, act, st, f, step, box, inject, seed, pass_offset, scale,
                                           stream);
        else
            propagate_t<float, 16, false>(prev, next, pack, act, st, f, step, box, inject, seed, pass_offset, scale,
                                          stream);
    }
}

// ====================================================================== exact_topk_batch (candidates.cpp:198-216)
// Brute-force top-K over the ascending active list under the unpacked ScoreTable<T> (probe-parallel).
template <typename T>
__global__ void k_exact_topk(const Q4<T>* __restrict__ rtab, const uint32_t* __restrict__ act, int n_act,
                             const int32_t* __restrict__ xy, int n_pix, int k, T s, uint32_t* __restrict__ out) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_pix) return;
    T px = static_cast<T>(static_cast<double>(xy[2 * q])), py = static_cast<T>(static_cast<double>(xy[2 * q + 1]));
    TopKReg<T, 16, false> sel;
    sel.init(k);
    for (int j = 0; j < n_act; j++) {
        uint32_t id = act[j];
        sel.consider(id, score_logit(rtab[3 * id], rtab[3 * id + 1], px, py, s));
    }
#pragma unroll
    for (int i = 0; i < 16; i++)
        if (i < k) out[static_cast<size_t>(q) * k + i] = i < sel.n ? sel.id[i] : kEmpty;
}

void launch_exact_topk(bool fp64, const void* rtab, const uint32_t* act, int n_act, const int32_t* xy, int n_pix,
                       int k, double scale, uint32_t* out, cudaStream_t stream) {
    int grid = (n_pix + 127) / 128;
    if (grid < 1) grid = 1;
    if (fp64)
        k_exact_topk<double><<<grid, 128, 0, stream>>>((const Q4<double>*)rtab, act, n_act, xy, n_pix, k, scale, out);
    else
        k_exact_topk<float><<<grid, 128, 0, stream>>>((const Q4<float>*)rtab, act, n_act, xy, n_pix, k,
                                                      static_cast<float>(scale), out);
    SAD_LAUNCHED();
}

// ====================================================================== render (render.cpp:19-89)
template <typename T, int KM>
__global__ void __launch_bounds__(256) k_render(const uint32_t* __restrict__ ids, const Q4<T>* __restrict__ rtab,
                                                FieldDims f, T s, T* __restrict__ out, DevState* st) {
    // mix_at (render.cpp:19-52): candidates stay in their list slots; `ok` marks the ones the reference
    // keeps (before the first sentinel, active, finite logit), and every sum runs over the kept slots
    // in list order, so it rounds exactly like the reference's compacted loop
    const int px = blockIdx.x * blockDim.x + threadIdx.x;
    const int py = blockIdx.y * blockDim.y + threadIdx.y;
    if (px >= f.width || py >= f.height) return;
    const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
    uint32_t cid[KM];
    if (KM == 8 && f.k == 8) {
        const uint4 u0 = __ldg(reinterpret_cast<const uint4*>(lst)), u1 = __ldg(reinterpret_cast<const uint4*>(lst) + 1);
        cid[0] = u0.x; cid[1] = u0.y; cid[2] = u0.z; cid[3] = u0.w;
        cid[4] = u1.x; cid[5] = u1.y; cid[6] = u1.z; cid[7] = u1.w;
    } else {
#pragma unroll
        for (int i = 0; i < KM; i++) cid[i] = i < f.k ? __ldg(lst + i) : kEmpty;
    }
    T lg[KM];
    bool ok[KM];
    bool any = false, stop = false;
    T best = T(0);
    const T fx = static_cast<T>(px), fy = static_cast<T>(py);
    // branch-free: slots past the first sentinel read site 0's rows and are masked out; a masked slot
    // adds +0.0 to the running sums, an exact no-op (sums that start at +0 are never -0)
#pragma unroll
    for (int i = 0; i < KM; i++) {
        stop = stop || cid[i] == kEmpty;
        const uint32_t id = stop ? 0u : cid[i];
        const Q4<T> a = rtab[3 * id], b = rtab[3 * id + 1];
        const T l = score_logit(a, b, fx, fy, s);
        ok[i] = !stop && b.w != T(0) && tfinite(l);
        lg[i] = ok[i] ? l : T(0);
        best = (ok[i] && (!any || l > best)) ? l : best;
        any = any || ok[i];
        cid[i] = id;
    }
    if (!any) {
        atomicOr(&st->err, 1);
        return;
    }
    T w[KM];
    T sum = T(0);
#pragma unroll
    for (int i = 0; i < KM; i++) {
        const T e = texp(lg[i] - best);
        w[i] = ok[i] ? e : T(0);
        sum += w[i];
    }
    const T inv = trcp(sum);
    T r = T(0), g = T(0), b = T(0);
#pragma unroll
    for (int i = 0; i < KM; i++) {
        const T wi = w[i] * inv;
        const Q4<T> c = rtab[3 * cid[i] + 2];
        r += ok[i] ? wi * c.x : T(0);
        g += ok[i] ? wi * c.y : T(0);
        b += ok[i] ? wi * c.z : T(0);
    }
    T* o = out + 3 * (static_cast<size_t>(py) * f.width + px);
    o[0] = r;
    o[1] = g;
    o[2] = b;
}

void launch_render(bool fp64, const uint32_t* ids, const void* rtab, const FieldDims& f, double scale, void* out,
                   DevState* st, cudaStream_t stream) {
    dim3 block(32, 8), grid((f.width + 31) / 32, (f.height + 7) / 8);
    if (fp64) {
        if (f.k <= 8)
            k_render<double, 8><<<grid, block, 0, stream>>>(ids, (const Q4<double>*)rtab, f, scale, (double*)out, st);
        else
            k_render<double, 16><<<grid, block, 0, stream>>>(ids, (const Q4<double>*)rtab, f, scale, (double*)out, st);
    } else {
        if (f.k <= 8)
            k_render<float, 8><<<grid, block, 0, stream>>>(ids, (const Q4<float>*)rtab, f, static_cast<float>(scale),
                                                           (float*)out, st);
        else
            k_render<float, 16><<<grid, block, 0, stream>>>(ids, (const Q4<float>*)rtab, f, static_cast<float>(scale),
                                                            (float*)out, st);
    }
    SAD_LAUNCHED();
}

// render_id_map (render.cpp:118-154): double ScoreTable argmax, ties to the lower id.
__global__ void k_id_map(const uint32_t* __restrict__ ids, const Q4<double>* __restrict__ rtab, FieldDims f, double s,
                         uint32_t* __restrict__ out, DevState* st) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x;
    const int py = blockIdx.y * blockDim.y + threadIdx.y;
    if (px >= f.width || py >= f.height) return;
    const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
    uint32_t best = kEmpty;
    double bl = 0;
    for (int i = 0; i < f.k; i++) {
        uint32_t id = lst[i];
        if (id == kEmpty) break;
        Q4<double> a = rtab[3 * id], b = rtab[3 * id + 1];
        if (b.w == 0.0) continue;
        double l = score_logit(a, b, static_cast<double>(px), static_cast<double>(py), s);
        if (best == kEmpty || l > bl || (l == bl && id < best)) {
            best = id;
            bl = l;
        }
    }
    out[static_cast<size_t>(py) * f.width + px] = best;
    if (best == kEmpty) atomicOr(&st->err, 1);
}

void launch_id_map(const uint32_t* ids, const void* rtab_d, const FieldDims& f, double scale, uint32_t* out,
                   DevState* st, cudaStream_t stream) {
    dim3 block(32, 8), grid((f.width + 31) / 32, (f.height + 7) / 8);
    k_id_map<<<grid, block, 0, stream>>>(ids, (const Q4<double>*)rtab_d, f, scale, out, st);
    SAD_LAUNCHED();
}

// pixel_weights (render.cpp:92-116), batched point queries against a cached double table: one thread per query, list slots unrolled (no local-memory
// arrays), kept candidates compacted in list order at output time; each block stages its 128 queries'
// 16-slot rows in shared memory (stride 17: conflict-free) and writes them back coalesced.
template <int KM>
__global__ void __launch_bounds__(128) k_pixel_weights(const uint32_t* __restrict__ ids,
                                                       const Q4<double>* __restrict__ rtab, FieldDims f, double s,
                                                       const int32_t* __restrict__ xy, int n_q,
                                                       uint32_t* __restrict__ oid, double* __restrict__ ow,
                                                       int32_t* __restrict__ on) {
    constexpr int QB = 128, RS = 17;
    __shared__ uint32_t sid[QB * RS];
    __shared__ double sw[QB * RS];
    const int q0 = blockIdx.x * QB;
    const int q = q0 + threadIdx.x;
    uint32_t cid[KM];
    double lg[KM];
    bool ok[KM];
    bool any = false;
    double best = 0;
#pragma unroll
    for (int i = 0; i < KM; i++) {
        cid[i] = kEmpty;
        lg[i] = 0;
        ok[i] = false;
    }
    if (q < n_q) {
        const int px = xy[2 * q], py = xy[2 * q + 1];
        if (px >= 0 && py >= 0 && px < f.width && py < f.height) {
            const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
            // the whole list in one or two vector loads (random cells: one HBM round trip, not K), then
            // a branch-free candidate loop whose table loads do not wait on the previous slot: slots past
            // the first sentinel read site 0's rows and are masked
            if (KM == 8 && f.k == 8) {
                const uint4 u0 = __ldg(reinterpret_cast<const uint4*>(lst)), u1 = __ldg(reinterpret_cast<const uint4*>(lst) + 1);
                const uint32_t v[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
                for (int i = 0; i < KM; i++) cid[i] = v[i % 8];
            } else {
#pragma unroll
                for (int i = 0; i < KM; i++) cid[i] = i < f.k ? __ldg(lst + i) : kEmpty;
            }
            bool stop = false;
#pragma unroll
            for (int i = 0; i < KM; i++) {
                stop = stop || cid[i] == kEmpty;
                const uint32_t id = stop ? 0u : cid[i];
                const Q4<double> a = rtab[3 * id], b = rtab[3 * id + 1];
                const double l = score_logit(a, b, static_cast<double>(px), static_cast<double>(py), s);
                ok[i] = !stop && b.w != 0.0 && isfinite(l);
                lg[i] = ok[i] ? l : 0.0;
                best = (ok[i] && (!any || l > best)) ? l : best;
                any = any || ok[i];
            }
        }
    }
    double w[KM];
    double sum = 0;
#pragma unroll
    for (int i = 0; i < KM; i++) {
        w[i] = 0;
        if (ok[i]) w[i] = sad_dexp(lg[i] - best);
        sum += w[i];  // +0.0 for masked slots: exact
    }
    const double inv = 1.0 / sum;
    uint32_t* my_id = sid + threadIdx.x * RS;
    double* my_w = sw + threadIdx.x * RS;
#pragma unroll
    for (int i = 0; i < 16; i++) {
        my_id[i] = kEmpty;
        my_w[i] = 0.0;
    }
    int n = 0;
#pragma unroll
    for (int i = 0; i < KM; i++)
        if (ok[i]) {
            my_id[n] = cid[i];
            my_w[n] = w[i] * inv;
            n++;
        }
    if (q < n_q) on[q] = n;
    __syncthreads();
    const int rows = n_q - q0 < QB ? n_q - q0 : QB;
    for (int j = threadIdx.x; j < rows * 16; j += QB) {
        const int r = j >> 4, c = j & 15;
        oid[static_cast<size_t>(q0) * 16 + j] = sid[r * RS + c];
        ow[static_cast<size_t>(q0) * 16 + j] = sw[r * RS + c];
    }
}

// K = 8 point queries with eight lanes per query (lane = list slot): every slot's table rows are in
// flight at once instead of one slot after another, and the output rows are written straight from
// registers, coalesced (four queries = 768 contiguous bytes per warp).  The order-dependent sums stay
// sequential in slot order: lane 0 of the query adds the eight weights (+0.0 for masked slots, an
// exact no-op) exactly as the one-thread kernel does; the maximum is order-independent.
__global__ void __launch_bounds__(128) k_pixel_weights8(const uint32_t* __restrict__ ids,
                                                        const Q4<double>* __restrict__ rtab, FieldDims f, double s,
                                                        const int32_t* __restrict__ xy, int n_q,
                                                        uint32_t* __restrict__ oid, double* __restrict__ ow,
                                                        int32_t* __restrict__ on) {
    const int lane = threadIdx.x & 31, slot = lane & 7, qbase = lane & 24;
    const unsigned qmask = 0xffu << qbase;
    const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    const bool valid_q = q < n_q;
    int px = -1, py = -1;
    if (valid_q) {
        px = xy[2 * q];
        py = xy[2 * q + 1];
    }
    const bool inside = valid_q && px >= 0 && py >= 0 && px < f.width && py < f.height;
    uint32_t id = kEmpty;
    if (inside) id = __ldg(ids + 8 * cell_index(f, px, py) + slot);
    // the list is read up to its first sentinel: a slot is live if no earlier slot is empty
    const unsigned empt = __ballot_sync(0xffffffffu, id == kEmpty) & qmask;
    const unsigned before = (1u << lane) - 1u;  // lanes below this one
    const bool stop = (empt & (before | (1u << lane)) & qmask) != 0u;
    const uint32_t sid = stop ? 0u : id;
    const Q4<double> a = rtab[3 * sid], b = rtab[3 * sid + 1];
    const double l = score_logit(a, b, static_cast<double>(px), static_cast<double>(py), s);
    const bool ok = inside && !stop && b.w != 0.0 && isfinite(l);
    // maximum over the query's live slots (a value: independent of order)
    double best = ok ? l : -INFINITY;
#pragma unroll
    for (int d = 4; d >= 1; d >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, best, d, 8);
        best = o > best ? o : best;
    }
    const double w = ok ? sad_dexp(l - best) : 0.0;
    // softmax denominator in slot order, as the one-thread loop
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < 8; i++) sum += __shfl_sync(0xffffffffu, w, qbase + i);
    const double inv = 1.0 / sum;
    const unsigned okm = __ballot_sync(0xffffffffu, ok) & qmask;
    const int n = __popc(okm);
    const int pos = __popc(okm & before);  // compacted output position of this slot
    // rows of 16: live entries in list order at their compacted column, then kEmpty / 0 padding
    if (valid_q) {
        uint32_t* rid = oid + static_cast<size_t>(q) * 16;
        double* rw = ow + static_cast<size_t>(q) * 16;
        if (slot == 0) on[q] = n;
        if (ok) {
            rid[pos] = sid;
            rw[pos] = w * inv;
        }
        // padding: 16 - n columns, two per lane at most (n <= 8 so 8 <= 16 - n <= 16)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int col = n + slot + 8 * h;
            if (col < 16) {
                rid[col] = kEmpty;
                rw[col] = 0.0;
            }
        }
    }
}

// SAD_PW1=1: one thread per point query (A/B)
static const bool g_pw8 = getenv("SAD_PW1") == nullptr;
void launch_pixel_weights(const uint32_t* ids, const void* rtab_d, const FieldDims& f, double scale, const int32_t* xy,
                          int n_q, uint32_t* out_ids, double* out_w, int32_t* out_n, cudaStream_t stream) {
    int grid = (n_q + 127) / 128;
    if (grid < 1) grid = 1;
    if (f.k == 8 && g_pw8) {
        const long long thr = 8ll * n_q;
        const int g8 = static_cast<int>((thr + 127) / 128);
        k_pixel_weights8<<<g8 > 0 ? g8 : 1, 128, 0, stream>>>(ids, (const Q4<double>*)rtab_d, f, scale, xy, n_q,
                                                               out_ids, out_w, out_n);
    } else if (f.k <= 8)
        k_pixel_weights<8><<<grid, 128, 0, stream>>>(ids, (const Q4<double>*)rtab_d, f, scale, xy, n_q, out_ids, out_w,
                                                     out_n);
    else
        k_pixel_weights<16><<<grid, 128, 0, stream>>>(ids, (const Q4<double>*)rtab_d, f, scale, xy, n_q, out_ids,
                                                      out_w, out_n);
    SAD_LAUNCHED();
}

// ====================================================================== tile reduction (grad.cpp:10-64)
// The reference reduces per-(site, channel) contributions of a 16x16 tile in a 256-slot hash table
// of compensated accumulators, then merges per worker; every sum is double-double, so the result is
// the exactly-rounded total independent of grouping.  Here a block owns a TW x TH pixel tile:
//   1. each thread computes its pixel's per-candidate contributions into shared memory
//      (entry e = slot * TPX + pixel, channel-major rows);
//   2. site ids are hashed into a shared table and compacted to local bucket ids;
//   3. entries are bucketed per site (counting sort) into `order`, bucket of each sorted position in
//      `posloc`;
//   4. buckets are cut into chunks of PT consecutive sorted positions; a thread sums one chunk for
//      half of the channels (5 independent double-double chains); when there are at most NT/2
//      chunks the two channel halves run at once on the two halves of the block;
//   5. each (site, tile) total is one record, claimed with one atomicAdd per site (RedTarget).
// Chunk length of step 4 and the one-pass split.  Measured on the config-2 fit (exp A/B, identical
// results): chunks of 8 with two sequential channel halves 895 ms; chunks of 12 with the split 870 ms
// (10 and 13 equal within noise, 16 876 ms; 12 without the split 885 ms).  Longer chunks give fewer
// chunks (NC ~ entries / 12 + buckets / 2, usually <= 128), so both halves fit on the 256 threads at once.
#ifndef SAD_TILE_PT
#define SAD_TILE_PT 12  // 0: chunks of KM sorted positions
#endif
#ifndef SAD_TILE_SCAN1
#define SAD_TILE_SCAN1 1  // 1: the chunk scan runs inside the bucket scan (one warp-0 pass, one barrier less)
#endif
#ifndef SAD_TILE_HTDIV
#define SAD_TILE_HTDIV 4  // hash slots = E / 4 (= UMAX): half the table init and compaction work; a tile
                          // holds ~40-100 distinct sites, so probes stay short (config-2 fit 857 -> 853 ms)
#endif
#ifndef SAD_TILE_SPLIT
#define SAD_TILE_SPLIT 1  // 1: when NC <= NT/2, the two channel halves run at once on the two thread halves
#endif
template <typename CT, int NCH, int TPX, int KM, int NT = TPX>
struct TileRed {  // TPX pixels, KM slots each, NT threads (TPX or 2 * TPX)
    static constexpr int E = TPX * KM;  // entries per tile
    static constexpr int UMAX = E / 4;  // distinct sites per tile kept in shared memory (rest: DD atomics)
    static constexpr int HT = E / SAD_TILE_HTDIV;  // hash slots (>= UMAX; a full table sends entries to `over`)
    static_assert(HT >= UMAX, "chunk_base lives in local_of_slot");
    static_assert((HT & (HT - 1)) == 0, "the tile hash masks with HT - 1: HT must be a power of two");
    static constexpr int ES = E + 16 / static_cast<int>(sizeof(CT));  // row stride: 16-byte aligned rows
    static constexpr int PT = SAD_TILE_PT > 0 ? SAD_TILE_PT : KM;  // sorted positions per chunk in step 4
    static constexpr int CA = NCH / 2, CB = NCH - CA;  // step 4 runs in two channel halves
    // step 4 writes the chunk partials of channels [0, CA) over rows [0, CA) and those of [CA, NCH)
    // over rows [CA, NCH): each half's rows are dead once its sums are read
    static_assert(CA * ES * sizeof(CT) >= 2 * TPX * CA * sizeof(DD), "chunk partials (half A) do not fit");
    static_assert(CB * ES * sizeof(CT) >= 2 * TPX * CB * sizeof(DD), "chunk partials (half B) do not fit");
    static_assert((CA * ES * sizeof(CT)) % 16 == 0, "half B rows must stay 16-byte aligned");
    alignas(16) CT c[NCH * ES];
    union {
        uint32_t key[E];  // site id per entry (steps 1-2)
        struct {
            uint16_t order[E];  // entry of each sorted position (steps 3-4)
        } srt;
    };
    union {
        uint32_t hkey[HT];  // hash keys (step 2)
        uint32_t cnt[UMAX];  // bucket sizes (step 3)
    };
    uint16_t local_of_entry[E];
    uint16_t local_of_slot[HT];
    uint32_t start[UMAX];
    uint32_t site_of_local[UMAX];
    uint32_t slot_of_local[UMAX];
    int n_local;
    DD warp_part[NT / 32];
};


template <typename CT, int NCH, int TPX, int KM, int NT>
__device__ __forceinline__ void tile_reduce(TileRed<CT, NCH, TPX, KM, NT>& sm, const RedTarget& red) {
    using R = TileRed<CT, NCH, TPX, KM, NT>;
    static_assert(NT == TPX || NT == 2 * TPX, "thread count");
    constexpr bool TWO = NT < 2 * TPX;  // each thread sums chunks tid and tid + NT (else only tid)
    const int tid = threadIdx.x;
#if SAD_EXPERIMENT == 3
    long long _t0 = clock64();
#endif
    // 2. hash insert (site ids are < 2^31; table keys start as kEmpty)
    for (int e = tid; e < R::E; e += NT) {
        uint32_t key = sm.key[e];
        if (key == kEmpty) continue;
        SAD_CHECK(key < static_cast<uint32_t>(red.cap));
        uint32_t h = (key * 2654435761u) & (R::HT - 1);
        uint16_t got = 0xffffu;  // stays 0xffff if the table is full: the entry goes to the atomic path
        for (int probe = 0; probe < R::HT; probe++) {
            uint32_t prev = atomicCAS(&sm.hkey[h], kEmpty, key);
            if (prev == kEmpty || prev == key) {
                got = static_cast<uint16_t>(h);
                break;
            }
            h = (h + 1) & (R::HT - 1);
        }
        sm.local_of_entry[e] = got;
    }
    __syncthreads();
    PH(1);
    for (int h = tid; h < R::HT; h += NT) {
        uint32_t key = sm.hkey[h];
        if (key != kEmpty) {
            int loc = atomicAdd(&sm.n_local, 1);
            sm.local_of_slot[h] = static_cast<uint16_t>(loc < R::UMAX ? loc : 0xffff);
            if (loc < R::UMAX) sm.site_of_local[loc] = key;
        }
    }
    __syncthreads();
    const int U = sm.n_local < R::UMAX ? sm.n_local : R::UMAX;
    // Record slot claims: one global atomicAdd per (site, tile), issued here and consumed only before
    // step 5, so their latency overlaps steps 3-4.  Step 5 then stores without global loads.
    constexpr int RU = (R::UMAX + NT - 1) / NT;
    uint32_t c_raw[RU], c_cap[RU];
    int32_t c_off[RU];
#pragma unroll
    for (int r = 0; r < RU; r++) {
        const int u = tid + r * NT;
        c_raw[r] = 0;
        c_cap[r] = 0;
        c_off[r] = 0;
        if (u < U) {
            sm.cnt[u] = 0;  // aliases hkey: safe after the barrier
            const uint32_t site = sm.site_of_local[u];
            c_raw[r] = static_cast<uint32_t>(atomicAdd(red.cnt + site, 1));
            c_cap[r] = red.roff ? static_cast<uint32_t>(red.rcap[site]) : static_cast<uint32_t>(red.maxt);
            c_off[r] = red.roff ? red.roff[site] : 0;
        }
    }
    __syncthreads();
    PH(2);
    // 3. bucket counts (entries with key == kEmpty get bucket 0xffff)
    for (int e = tid; e < R::E; e += NT) {
        uint16_t loc = 0xffffu;
        const uint32_t key = sm.key[e];
        if (key != kEmpty) {
            const uint16_t hs = sm.local_of_entry[e];
            loc = hs == 0xffffu ? static_cast<uint16_t>(0xffffu) : sm.local_of_slot[hs];
            if (loc != 0xffffu) {
                atomicAdd(&sm.cnt[loc], 1u);
            } else {  // more than UMAX distinct sites in this tile: exact DD merge straight into `over`
#pragma unroll
                for (int ch = 0; ch < NCH; ch++)
                    dd_atomic_merge(red.over + static_cast<size_t>(ch) * red.cap + key,
                                    DD{static_cast<double>(sm.c[ch * R::ES + e]), 0.0});
            }
        }
        sm.local_of_entry[e] = loc;
    }
    __syncthreads();
    // exclusive scans by warp 0 (U <= E) of cnt[0..U) -> start, and (SAD_TILE_SCAN1) of the chunk
    // counts ceil(cnt / PT) -> chunk_base (local_of_slot is dead after the counting above)
    __shared__ int n_valid;
    __shared__ int n_chunks;
    uint16_t* chunk_base = sm.local_of_slot;  // chunk index of each bucket's first chunk
    if (tid < 32) {
        int carry = 0, ccarry = 0;
        for (int base = 0; base < U; base += 32) {
            int u = base + tid;
            int v = u < U ? static_cast<int>(sm.cnt[u]) : 0;
            int x = v;
            int cv = SAD_TILE_SCAN1 ? (v + R::PT - 1) / R::PT : 0;
            int cx = cv;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, x, d);
                if (tid >= d) x += y;
                if (SAD_TILE_SCAN1) {
                    int cy = __shfl_up_sync(0xffffffffu, cx, d);
                    if (tid >= d) cx += cy;
                }
            }
            if (u < U) {
                sm.start[u] = static_cast<uint32_t>(carry + x - v);
                if (SAD_TILE_SCAN1) chunk_base[u] = static_cast<uint16_t>(ccarry + cx - cv);
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
            if (SAD_TILE_SCAN1) ccarry += __shfl_sync(0xffffffffu, cx, 31);
        }
        if (tid == 0) {
            n_valid = carry;
            if (SAD_TILE_SCAN1) n_chunks = ccarry;
        }
    }
    __syncthreads();  // key[] is dead from here: its storage becomes order/posloc
    PH(3);
    for (int e = tid; e < R::E; e += NT) {
        int loc = sm.local_of_entry[e];
        if (loc == 0xffff) continue;
        int pos = static_cast<int>(atomicAdd(&sm.start[loc], 1u));
        SAD_CHECK(loc < R::UMAX && pos >= 0 && pos < R::E);
        sm.srt.order[pos] = static_cast<uint16_t>(e);
    }
    __syncthreads();
    const int U2 = U;
    uint16_t* chunk_bucket = sm.local_of_entry;  // dead after the scatter: bucket of each chunk
    for (int u = tid; u < U; u += NT) {
        sm.start[u] -= sm.cnt[u];  // cursor back to the bucket start
        if (SAD_TILE_SCAN1) {
            const int c0 = chunk_base[u], nc = static_cast<int>((sm.cnt[u] + R::PT - 1) / R::PT);
            for (int c = c0; c < c0 + nc; c++) chunk_bucket[c] = static_cast<uint16_t>(u);
        }
    }
    PH(4);
    // 4. buckets split into chunks of PT sorted entries; thread t sums chunks t and t + NT for all
    //    channels (convergent fixed-trip loops, NCH independent double-double chains)
    if (!SAD_TILE_SCAN1 && tid < 32) {
        int carry = 0;
        for (int base = 0; base < U2; base += 32) {
            int u = base + tid;
            int v = u < U2 ? static_cast<int>((sm.cnt[u] + R::PT - 1) / R::PT) : 0;
            int x = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, x, d);
                if (tid >= d) x += y;
            }
            if (u < U2) chunk_base[u] = static_cast<uint16_t>(carry + x - v);
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (tid == 0) n_chunks = carry;
    }
    if (!SAD_TILE_SCAN1) {
        __syncthreads();
        for (int u = tid; u < U2; u += NT) {
            int c0 = chunk_base[u], nc = static_cast<int>((sm.cnt[u] + R::PT - 1) / R::PT);
            for (int c = c0; c < c0 + nc; c++) chunk_bucket[c] = static_cast<uint16_t>(u);
        }
    }
    __syncthreads();
    const int NC = n_chunks;
    PH(5);
    // Two channel halves: each thread holds its two chunks' partials for CB channels at a time (half
    // the registers of a single pass), and each half's partials overwrite that half's dead rows.
    auto sum_chunk = [&](int c, int ch0, int nch, DD* acc) {
#pragma unroll
        for (int ch = 0; ch < R::CB; ch++) acc[ch] = DD{0.0, 0.0};
        const int u = chunk_bucket[c];
        const int off = (c - chunk_base[u]) * R::PT;
        const int n = static_cast<int>(sm.cnt[u]) - off;
        const int b = static_cast<int>(sm.start[u]) + off;
        // branch-free: steps past the chunk end read the padding column E, which holds +0.0 in every
        // channel; adding +0.0 to these accumulators is an exact no-op (a running double-double sum
        // that starts at +0 is never -0)
#pragma unroll
        for (int j = 0; j < R::PT; j++) {
            SAD_CHECK(j >= n || (b + j >= 0 && b + j < R::E));
            const int e = j < n ? static_cast<int>(sm.srt.order[b + j]) : R::E;
#pragma unroll
            for (int ch = 0; ch < R::CB; ch++)
                if (ch < nch) dd_add(acc[ch], static_cast<double>(sm.c[(ch0 + ch) * R::ES + e]));
        }
    };
    DD* const carry_a = reinterpret_cast<DD*>(sm.c);
    DD* const carry_b = reinterpret_cast<DD*>(sm.c + R::CA * R::ES);
    auto half = [&](int ch0, int nch, DD* carry) {
        DD acc0[R::CB], acc1[R::CB];
        if (tid < NC) sum_chunk(tid, ch0, nch, acc0);
        if (TWO && tid + NT < NC) sum_chunk(tid + NT, ch0, nch, acc1);
        // chunks beyond 2*TPX (more than ~TPX distinct sites in one tile): merged straight into `over`
        for (int c = tid + 2 * TPX; c < NC; c += NT) {
            DD tmp[R::CB];
            sum_chunk(c, ch0, nch, tmp);
            const uint32_t site = sm.site_of_local[chunk_bucket[c]];
#pragma unroll
            for (int ch = 0; ch < R::CB; ch++)
                if (ch < nch) dd_atomic_merge(red.over + static_cast<size_t>(ch0 + ch) * red.cap + site, tmp[ch]);
        }
        __syncthreads();  // every read of this half's rows is done: they become its chunk partials
        if (tid < NC) {
#pragma unroll
            for (int ch = 0; ch < R::CB; ch++)
                if (ch < nch) carry[tid * nch + ch] = acc0[ch];
        }
        if (TWO && tid + NT < NC) {
#pragma unroll
            for (int ch = 0; ch < R::CB; ch++)
                if (ch < nch) carry[(tid + NT) * nch + ch] = acc1[ch];
        }
    };
    if (SAD_TILE_SPLIT && NC <= NT / 2) {
        // threads [0, NT/2) sum channel half A of chunk tid, threads [NT/2, NT) half B of chunk
        // tid - NT/2: one pass, and each half's partials still overwrite only that half's rows
        const bool hb = tid >= NT / 2;
        const int c = hb ? tid - NT / 2 : tid;
        const int ch0 = hb ? R::CA : 0, nch = hb ? R::CB : R::CA;
        DD acc[R::CB];
        if (c < NC) sum_chunk(c, ch0, nch, acc);
        __syncthreads();
        if (c < NC) {
            DD* carry = hb ? carry_b : carry_a;
#pragma unroll
            for (int ch = 0; ch < R::CB; ch++)
                if (ch < nch) carry[c * nch + ch] = acc[ch];
        }
        PH(6);
    } else {
        half(0, R::CA, carry_a);
        PH(6);
        half(R::CA, R::CB, carry_b);
    }
    // record code per local site: bits 31-30 = 00 record index into part, 01 overflow record into opart,
    // 11 pool exhausted (exact DD CAS into over)
#pragma unroll
    for (int r = 0; r < RU; r++) {
        const int u = tid + r * NT;
        if (u < U) {
            const uint32_t site = sm.site_of_local[u];
            uint32_t slot = c_raw[r];
            const uint32_t scap = c_cap[r];
            if (red.roff && slot < scap && static_cast<long long>(c_off[r]) + slot >= red.psize) slot = scap;  // pool bound
            uint32_t code;
            if (slot < scap) {
                code = red.roff ? static_cast<uint32_t>(c_off[r]) + slot : site * static_cast<uint32_t>(red.maxt) + slot;
            } else {  // overflow record from the pool, linked per site
                const int ro = atomicAdd(red.otop, 1);
                if (ro < red.ocap) red.onext[ro] = atomicExch(red.head + site, ro);
                code = ro < red.ocap ? (0x40000000u | static_cast<uint32_t>(ro)) : 0xc0000000u;
            }
            sm.slot_of_local[u] = code;
        }
    }
    __syncthreads();
    PH(7);
    // 5. per (site, channel): merge the site's chunks and store the record (or CAS on slot overflow)
    const int NCK = NC < 2 * TPX ? NC : 2 * TPX;
    for (int item = tid; item < U2 * NCH; item += NT) {
        const int u = item / NCH, ch = item - u * NCH;
        const int c0 = chunk_base[u];
        const int c1 = c0 + static_cast<int>((sm.cnt[u] + R::PT - 1) / R::PT);
        DD t{0.0, 0.0};
        const DD* cp = ch < R::CA ? carry_a + ch : carry_b + (ch - R::CA);
        const int cs = ch < R::CA ? R::CA : R::CB;
        for (int c = c0; c < c1 && c < NCK; c++) dd_merge(t, cp[c * cs]);
        const uint32_t site = sm.site_of_local[u];
        const uint32_t code = sm.slot_of_local[u];
        if ((code >> 30) == 0u) {
            SAD_CHECK(red.roff ? static_cast<long long>(code) < red.psize
                               : static_cast<long long>(code) < static_cast<long long>(red.cap) * red.maxt);
            red.part[static_cast<size_t>(code) * red.stride + ch] = make_double2(t.hi, t.lo);
        } else if ((code >> 30) == 1u) {
            SAD_CHECK(static_cast<int>(code & 0x3fffffffu) < red.ocap);
            red.opart[static_cast<size_t>(code & 0x3fffffffu) * red.stride + ch] = make_double2(t.hi, t.lo);
        } else {  // pool exhausted
#if SAD_EXPERIMENT == 3
            if (ch == 0) atomicAdd(&g_phase_clk[15], 1ull);
#endif
            dd_atomic_merge(red.over + static_cast<size_t>(ch) * red.cap + site, t);
        }
    }
    PH(8);
}

template <typename CT, int NCH, int TPX, int KM, int NT>
__device__ __forceinline__ void tile_init(TileRed<CT, NCH, TPX, KM, NT>& sm) {
    using R = TileRed<CT, NCH, TPX, KM, NT>;
    for (int h = threadIdx.x; h < R::HT; h += NT) sm.hkey[h] = kEmpty;
    if (threadIdx.x < NCH) sm.c[threadIdx.x * R::ES + R::E] = CT(0);  // padding column (step 4)
    if (threadIdx.x == 0) sm.n_local = 0;
}

// Block-wide compensated reduction of one DD per thread, merged into `dst`.
template <int TPX>
__device__ __forceinline__ void block_dd_merge(DD v, DD* warp_part, double2* dst) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        DD o{__shfl_down_sync(0xffffffffu, v.hi, d), __shfl_down_sync(0xffffffffu, v.lo, d)};
        dd_merge(v, o);
    }
    if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        DD t = warp_part[0];
        for (int w = 1; w < TPX / 32; w++) dd_merge(t, warp_part[w]);
        if (t.hi != 0.0 || t.lo != 0.0) dd_atomic_merge(dst, t);
    }
}

// Block-wide compensated reduction stored (no atomics) to dst (one partial per block).
template <int TPX>
__device__ __forceinline__ void block_dd_store(DD v, DD* warp_part, double2* dst) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        DD o{__shfl_down_sync(0xffffffffu, v.hi, d), __shfl_down_sync(0xffffffffu, v.lo, d)};
        dd_merge(v, o);
    }
    if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        DD t = warp_part[0];
        for (int w = 1; w < TPX / 32; w++) dd_merge(t, warp_part[w]);
        *dst = make_double2(t.hi, t.lo);
    }
}

template <int TPX>
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long* sm_tmp) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0) sm_tmp[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < TPX / 32; w++) t += sm_tmp[w];
    return t;
}

// ====================================================================== fused forward + backward
// pixel_pass (grad.cpp:117-240) per pixel, tile reduction as above, loss as a compensated sum.
// MODE 0: MSE vs target, no removal (the fit's call, train.cpp:249); 1: with removal delta;
// 2: caller-supplied dL/dvalue (backward_pixel_grad, grad.cpp:382-390).
template <typename T> struct BwdTile;
#ifndef SAD_BWD2_TH
#define SAD_BWD2_TH 8  // fp32 tile rows (16 x TH pixels, 32 * TH threads in k_backward2)
#endif
template <> struct BwdTile<float> { static constexpr int TW = 16, TH = SAD_BWD2_TH; };
template <> struct BwdTile<double> { static constexpr int TW = 8, TH = 8; };

template <typename T, int KM, int MODE>
__global__ void __launch_bounds__(BwdTile<T>::TW * BwdTile<T>::TH)
    k_backward(const uint32_t* __restrict__ ids, const Q4<T>* __restrict__ gtab, const T* __restrict__ tgt, FieldDims f,
               T s, T inv_hw2, RedTarget red, double2* __restrict__ loss_part, DevState* st) {
    constexpr int TW = BwdTile<T>::TW, TH = BwdTile<T>::TH, TPX = TW * TH;
    constexpr int NCH = MODE == 1 ? 11 : 10;
    using Red = TileRed<T, NCH, TPX, KM>;
    extern __shared__ __align__(16) unsigned char smraw[];
    Red& sm = *reinterpret_cast<Red*>(smraw);
#if SAD_EXPERIMENT == 3
    long long _t0 = clock64();
#endif
    tile_init(sm);

    const int tid = threadIdx.x;
    const int px = blockIdx.x * TW + (tid % TW);
    const int py = blockIdx.y * TH + (tid / TW) + f.row0;
    const bool inside = px < f.width && py < f.height && py < f.row1;
    constexpr T kTiny = sizeof(T) == 8 ? T(1e-18) : T(1e-12);

    // Candidates stay in their list slots; `ok` marks the ones the reference keeps (active, finite
    // logit, before the first sentinel).  Iterating slots in order with `ok` predication visits the
    // kept candidates in the reference's order, so every sum below rounds identically.
    uint32_t cid[KM];
    T dxs[KM], dys[KM], ud[KM], vd[KM], nrm[KM], lg[KM];
    bool ok[KM];
    bool any = false;
    T best = T(0);
    unsigned long long nonfinite = 0;
    DD loss{0.0, 0.0};
    {
        const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
        const T fx = static_cast<T>(px), fy = static_cast<T>(py);
        bool stop = !inside;
#pragma unroll
        for (int i = 0; i < KM; i++) {
            uint32_t id = kEmpty;
            if (!stop && i < f.k) id = lst[i];
            stop = stop || id == kEmpty;
            cid[i] = id;
            ok[i] = false;
            dxs[i] = dys[i] = ud[i] = vd[i] = nrm[i] = lg[i] = T(0);
            if (!stop) {
                const Q4<T> a = gtab[3 * id], b = gtab[3 * id + 1];
                const T act = gtab[3 * id + 2].w;
                T dx = fx - a.x, dy = fy - a.y;
                T pa = b.z * dx + b.w * dy;
                T pb = b.z * dy - b.w * dx;
                T q = b.x * pa * pa + b.y * pb * pb;
                if (q < T(0)) q = T(0);
                T m = tsqrt(q);
                T l = -a.z * (m * s - a.w * s);
                ok[i] = act != T(0) && c_finite(l);
                dxs[i] = dx;
                dys[i] = dy;
                ud[i] = pa;
                vd[i] = pb;
                nrm[i] = m;
                lg[i] = l;
                if (ok[i] && (!any || l > best)) best = l;
                any = any || ok[i];
            }
        }
        if (inside && !any) atomicOr(&st->err, 1);
    }
    if (any) {
        T w[KM];
        T wsum = T(0);
#pragma unroll
        for (int i = 0; i < KM; i++) {
            w[i] = T(0);
            if (ok[i]) {
                w[i] = texp(lg[i] - best);
                wsum += w[i];
            }
        }
        T invw = trcp(wsum);
        T ch0 = T(0), ch1 = T(0), ch2 = T(0);
#pragma unroll
        for (int i = 0; i < KM; i++)
            if (ok[i]) {
                w[i] *= invw;
                const Q4<T> c = gtab[3 * cid[i] + 2];
                ch0 += w[i] * c.x;
                ch1 += w[i] * c.y;
                ch2 += w[i] * c.z;
            }
        T g0, g1, g2, t0 = T(0), t1 = T(0), t2 = T(0), pl = T(0);
        const T* tp = tgt + 3 * (static_cast<size_t>(py) * f.width + px);
        if (MODE != 2) {
            t0 = tp[0];
            t1 = tp[1];
            t2 = tp[2];
            T e0 = ch0 - t0, e1 = ch1 - t1, e2 = ch2 - t2;
            pl = e0 * e0 + e1 * e1 + e2 * e2;
            double plv = static_cast<double>(pl);
            if (!c_finite(pl)) {
                nonfinite++;
                plv = 0;
            }
            dd_add(loss, plv);
            g0 = inv_hw2 * e0;
            g1 = inv_hw2 * e1;
            g2 = inv_hw2 * e2;
        } else {
            g0 = tp[0];
            g1 = tp[1];
            g2 = tp[2];
        }
        // A kept candidate whose softmax weight underflowed to exactly 0 contributes +-0 to every
        // channel when the pixel's adjoint g (and, with removal, its loss pl) is finite: every term is
        // a product with w or A = w * finite.  Dropping it then leaves every compensated sum and the
        // non-finite count bit-identical, and shrinks the reduction.  With a non-finite g the
        // reference's 0 * inf = NaN terms are scrubbed and counted, so such pixels keep the entry.
        const bool wz_skip = c_finite(g0) && c_finite(g1) && c_finite(g2) && (MODE != 1 || c_finite(pl));
#pragma unroll
        for (int i = 0; i < KM; i++) {
            const int e = i * TPX + tid;
            if (!ok[i] || (w[i] == T(0) && wz_skip)) {
                sm.key[e] = kEmpty;
                continue;
            }
#if SAD_EXPERIMENT == 3
            atomicAdd(&g_phase_clk[13], 1ull);
            if (w[i] == T(0)) atomicAdd(&g_phase_clk[14], 1ull);
#endif
            const uint32_t id = cid[i];
            const Q4<T> a = gtab[3 * id], b = gtab[3 * id + 1], c = gtab[3 * id + 2];
            T dc0 = c.x - ch0, dc1 = c.y - ch1, dc2 = c.z - ch2;
            T A = w[i] * (g0 * dc0 + g1 * dc1 + g2 * dc2);
            T ts = a.z * s;
            T v[11];
            v[4] = w[i] * g0;
            v[5] = w[i] * g1;
            v[6] = w[i] * g2;
            v[2] = A * lg[i];
            v[3] = A * ts;
            if (nrm[i] > kTiny) {
                T inv_n = trcp(nrm[i]);
                T eau = b.x * ud[i];
                T iav = b.y * vd[i];
                T coef = A * ts * inv_n;
                v[0] = coef * (eau * b.z - iav * b.w);
                v[1] = coef * (eau * b.w + iav * b.z);
                v[7] = -coef * (eau * dxs[i] + iav * dys[i]);
                v[8] = -coef * (eau * dys[i] - iav * dxs[i]);
                v[9] = -A * ts * T(0.5) * inv_n * (eau * ud[i] - iav * vd[i]);
            } else {
                v[0] = v[1] = v[7] = v[8] = v[9] = T(0);
            }
            if (MODE == 1) {
                if (w[i] >= T(1) - T(1e-6)) {
                    v[10] = static_cast<T>(1e6);
                } else {
                    T inv_rest = trcp(T(1) - w[i]);
                    T r0 = (ch0 - w[i] * c.x) * inv_rest - t0;
                    T r1 = (ch1 - w[i] * c.y) * inv_rest - t1;
                    T r2 = (ch2 - w[i] * c.z) * inv_rest - t2;
                    v[10] = r0 * r0 + r1 * r1 + r2 * r2 - pl;
                }
            }
            sm.key[e] = id;
            // non-finite components are zeroed and counted (grad.cpp:232-237); one combined test first
            bool bad = false;
#pragma unroll
            for (int t = 0; t < NCH; t++) bad |= !c_finite(v[t]);
            if (bad) {
#pragma unroll
                for (int t = 0; t < NCH; t++)
                    if (!c_finite(v[t])) {
                        v[t] = T(0);
                        nonfinite++;
                    }
            }
#pragma unroll
            for (int t = 0; t < NCH; t++) sm.c[t * Red::ES + e] = v[t];
        }
    } else {
#pragma unroll
        for (int i = 0; i < KM; i++) sm.key[i * TPX + tid] = kEmpty;
    }
    __syncthreads();
    PH(0);
    tile_reduce(sm, red);
    __syncthreads();
    if (MODE != 2) block_dd_store<TPX>(loss, sm.warp_part, loss_part + blockIdx.y * gridDim.x + blockIdx.x);
    __syncthreads();
    unsigned long long nf = block_sum_u64<TPX>(nonfinite, reinterpret_cast<unsigned long long*>(sm.warp_part));
    if (threadIdx.x == 0 && nf) atomicAdd(reinterpret_cast<unsigned long long*>(&st->nonfinite), nf);
}

// fp32 variant with two lanes per pixel (256 threads per 16x8 tile): lane h of a pixel takes list
// slots [h*KM/2, (h+1)*KM/2).  Everything order-sensitive keeps the reference's sequential order: the
// sentinel of lane 0 ends lane 1's list, the running max is combined in slot order, and the float
// sums of the softmax denominator and of the blended colour are continued by lane 1 from lane 0's
// partial (one shuffle each way), so every rounding equals the one-thread loop of k_backward.  The
// shuffles run for every lane (pairs whose pixel is outside or empty compute unused values), and the
// tile reduction then runs on all 256 threads.
#ifndef SAD_VEC_IDS
#define SAD_VEC_IDS 1  // 1: K = 8 lists read as one 16-byte load per lane (two-lane backward and stats)
#endif
#ifndef SAD_BWD_HOIST_TGT
#define SAD_BWD_HOIST_TGT 1  // measured: with SAD_BWD_EARLY_COL, config-2 fit 868.5 -> 865 ms
#endif
#ifndef SAD_BWD_EARLY_COL
#define SAD_BWD_EARLY_COL 1
#endif
#ifndef SAD_BWD2_MINB
#define SAD_BWD2_MINB 4
#endif
template <int KM, int MODE>
__global__ void __launch_bounds__(32 * SAD_BWD2_TH, SAD_BWD2_MINB * 8 / SAD_BWD2_TH) k_backward2(const uint32_t* __restrict__ ids, const Q4<float>* __restrict__ gtab,
                                                   const float* __restrict__ tgt, FieldDims f, float s, float inv_hw2,
                                                   RedTarget red, double2* __restrict__ loss_part, DevState* st) {
    pdl_enter<2>();
    using T = float;
    constexpr int TW = 16, TH = SAD_BWD2_TH, TPX = TW * TH, NT = 2 * TPX, H = KM / 2;
    constexpr int NCH = MODE == 1 ? 11 : 10;
    constexpr unsigned FULL = 0xffffffffu;
    using Red = TileRed<T, NCH, TPX, KM, NT>;
    extern __shared__ __align__(16) unsigned char smraw[];
    Red& sm = *reinterpret_cast<Red*>(smraw);
#if SAD_EXPERIMENT == 3
    long long _t0 = clock64();
#endif
    tile_init(sm);

    const int tid = threadIdx.x;
    const int pix = tid >> 1, half = tid & 1;
    const int px = blockIdx.x * TW + (pix % TW);
    const int py = blockIdx.y * TH + (pix / TW) + f.row0;
    const bool inside = px < f.width && py < f.height && py < f.row1;
    constexpr T kTiny = T(1e-12);

    uint32_t cid[H];
    T dxs[H], dys[H], ud[H], vd[H], nrm[H], lg[H];
    bool ok[H];
    bool any = false;
    T best = T(0);
    unsigned long long nonfinite = 0;
    DD loss{0.0, 0.0};
#if SAD_BWD_HOIST_TGT
    // the pixel's target (or dL/dvalue) row: the only HBM stream of the kernel, issued before the list
    T tq0 = T(0), tq1 = T(0), tq2 = T(0);
    if (inside) {
        const T* tq = tgt + 3 * (static_cast<size_t>(py) * f.width + px);
        tq0 = tq[0];
        tq1 = tq[1];
        tq2 = tq[2];
    }
#endif
#if SAD_BWD_EARLY_COL
    Q4<T> col[H];
#endif
    {
        uint32_t idv[H];
        const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
        bool has_empty = false;
        if (SAD_VEC_IDS && H == 4 && f.k == 8) {  // this lane's half of the list in one 16-byte load
            uint4 q = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
            if (inside) q = *reinterpret_cast<const uint4*>(lst + half * 4);
            idv[0] = q.x;
            idv[1] = q.y;
            idv[2 % H] = q.z;
            idv[3 % H] = q.w;
        } else {
#pragma unroll
            for (int j = 0; j < H; j++) {
                const int i = half * H + j;
                idv[j] = (inside && i < f.k) ? lst[i] : kEmpty;
            }
        }
#pragma unroll
        for (int j = 0; j < H; j++) has_empty = has_empty || idv[j] == kEmpty;
        const bool partner_empty = __shfl_xor_sync(FULL, has_empty, 1);
        const T fx = static_cast<T>(px), fy = static_cast<T>(py);
        bool stop = !inside || (half == 1 && partner_empty);
#pragma unroll
        for (int j = 0; j < H; j++) {
            const uint32_t id = idv[j];
            stop = stop || id == kEmpty;
            cid[j] = id;
            ok[j] = false;
            dxs[j] = dys[j] = ud[j] = vd[j] = nrm[j] = lg[j] = T(0);
#if SAD_BWD_EARLY_COL
            col[j] = Q4<T>{T(0), T(0), T(0), T(0)};
#endif
            if (!stop) {
                SAD_CHECK(id < static_cast<uint32_t>(st->n_sites));
                const Q4<T> a = gtab[3 * id], b = gtab[3 * id + 1];
#if SAD_BWD_EARLY_COL
                col[j] = gtab[3 * id + 2];
                const T act = col[j].w;
#else
                const T act = gtab[3 * id + 2].w;
#endif
                T dx = fx - a.x, dy = fy - a.y;
                T pa = b.z * dx + b.w * dy;
                T pb = b.z * dy - b.w * dx;
                T q = b.x * pa * pa + b.y * pb * pb;
                if (q < T(0)) q = T(0);
                T m = tsqrt(q);
                T l = -a.z * (m * s - a.w * s);
                ok[j] = act != T(0) && c_finite(l);
                dxs[j] = dx;
                dys[j] = dy;
                ud[j] = pa;
                vd[j] = pb;
                nrm[j] = m;
                lg[j] = l;
                if (ok[j] && (!any || l > best)) best = l;
                any = any || ok[j];
            }
        }
    }
    // running max in slot order: lane 1's candidates come after lane 0's
    const bool pany = __shfl_xor_sync(FULL, any, 1);
    const T pbest = __shfl_xor_sync(FULL, best, 1);
    const bool a0 = half == 0 ? any : pany, a1 = half == 0 ? pany : any;
    const T b0 = half == 0 ? best : pbest, b1 = half == 0 ? pbest : best;
    best = a0 ? ((a1 && b1 > b0) ? b1 : b0) : b1;
    const bool any_all = a0 || a1;
    if (inside && !any_all && half == 0) atomicOr(&st->err, 1);

    // softmax denominator: lane 0 sums its slots from 0, lane 1 continues from lane 0's sum
    T w[H];
    T wpart = T(0);
#pragma unroll
    for (int j = 0; j < H; j++) {
        w[j] = T(0);
        if (ok[j]) w[j] = texp(lg[j] - best);
    }
    if (half == 0) {
#pragma unroll
        for (int j = 0; j < H; j++)
            if (ok[j]) wpart += w[j];
    }
    const T from0 = __shfl_xor_sync(FULL, wpart, 1);
    if (half == 1) {
        wpart = from0;
#pragma unroll
        for (int j = 0; j < H; j++)
            if (ok[j]) wpart += w[j];
    }
    const T from1 = __shfl_xor_sync(FULL, wpart, 1);
    const T wsum = half == 0 ? from1 : wpart;
    const T invw = trcp(wsum);
    // blended colour, same hand-over
#if !SAD_BWD_EARLY_COL
    Q4<T> col[H];
#endif
    T c0 = T(0), c1 = T(0), c2 = T(0);
#pragma unroll
    for (int j = 0; j < H; j++) {
#if !SAD_BWD_EARLY_COL
        col[j] = Q4<T>{T(0), T(0), T(0), T(0)};
#endif
        if (ok[j]) {
            w[j] *= invw;
#if !SAD_BWD_EARLY_COL
            col[j] = gtab[3 * cid[j] + 2];
#endif
        }
    }
    if (half == 0) {
#pragma unroll
        for (int j = 0; j < H; j++)
            if (ok[j]) {
                c0 += w[j] * col[j].x;
                c1 += w[j] * col[j].y;
                c2 += w[j] * col[j].z;
            }
    }
    {
        const T r0 = __shfl_xor_sync(FULL, c0, 1), r1 = __shfl_xor_sync(FULL, c1, 1), r2 = __shfl_xor_sync(FULL, c2, 1);
        if (half == 1) {
            c0 = r0;
            c1 = r1;
            c2 = r2;
#pragma unroll
            for (int j = 0; j < H; j++)
                if (ok[j]) {
                    c0 += w[j] * col[j].x;
                    c1 += w[j] * col[j].y;
                    c2 += w[j] * col[j].z;
                }
        }
        const T s0 = __shfl_xor_sync(FULL, c0, 1), s1 = __shfl_xor_sync(FULL, c1, 1), s2 = __shfl_xor_sync(FULL, c2, 1);
        if (half == 0) {
            c0 = s0;
            c1 = s1;
            c2 = s2;
        }
    }
    const T ch0 = c0, ch1 = c1, ch2 = c2;
    if (any_all) {
        T g0, g1, g2, t0 = T(0), t1 = T(0), t2 = T(0), pl = T(0);
#if SAD_BWD_HOIST_TGT
        const T tp[3] = {tq0, tq1, tq2};
#else
        const T* tp = tgt + 3 * (static_cast<size_t>(py) * f.width + px);
#endif
        if (MODE != 2) {
            t0 = tp[0];
            t1 = tp[1];
            t2 = tp[2];
            T e0 = ch0 - t0, e1 = ch1 - t1, e2 = ch2 - t2;
            pl = e0 * e0 + e1 * e1 + e2 * e2;
            if (half == 0) {
                double plv = static_cast<double>(pl);
                if (!c_finite(pl)) {
                    nonfinite++;
                    plv = 0;
                }
                dd_add(loss, plv);
            }
            g0 = inv_hw2 * e0;
            g1 = inv_hw2 * e1;
            g2 = inv_hw2 * e2;
        } else {
            g0 = tp[0];
            g1 = tp[1];
            g2 = tp[2];
        }
        const bool wz_skip = c_finite(g0) && c_finite(g1) && c_finite(g2) && (MODE != 1 || c_finite(pl));
#pragma unroll
        for (int j = 0; j < H; j++) {
            const int e = (half * H + j) * TPX + pix;
            if (!ok[j] || (w[j] == T(0) && wz_skip)) {  // zero weight: +-0 in every channel (see k_backward)
                sm.key[e] = kEmpty;
                continue;
            }
            const uint32_t id = cid[j];
            const Q4<T> a = gtab[3 * id], b = gtab[3 * id + 1];
            const Q4<T> c = col[j];
            T dc0 = c.x - ch0, dc1 = c.y - ch1, dc2 = c.z - ch2;
            T A = w[j] * (g0 * dc0 + g1 * dc1 + g2 * dc2);
            T ts = a.z * s;
            T v[11];
            v[4] = w[j] * g0;
            v[5] = w[j] * g1;
            v[6] = w[j] * g2;
            v[2] = A * lg[j];
            v[3] = A * ts;
            if (nrm[j] > kTiny) {
                T inv_n = trcp(nrm[j]);
                T eau = b.x * ud[j];
                T iav = b.y * vd[j];
                T coef = A * ts * inv_n;
                v[0] = coef * (eau * b.z - iav * b.w);
                v[1] = coef * (eau * b.w + iav * b.z);
                v[7] = -coef * (eau * dxs[j] + iav * dys[j]);
                v[8] = -coef * (eau * dys[j] - iav * dxs[j]);
                v[9] = -A * ts * T(0.5) * inv_n * (eau * ud[j] - iav * vd[j]);
            } else {
                v[0] = v[1] = v[7] = v[8] = v[9] = T(0);
            }
            if (MODE == 1) {
                if (w[j] >= T(1) - T(1e-6)) {
                    v[10] = static_cast<T>(1e6);
                } else {
                    T inv_rest = trcp(T(1) - w[j]);
                    T r0 = (ch0 - w[j] * c.x) * inv_rest - t0;
                    T r1 = (ch1 - w[j] * c.y) * inv_rest - t1;
                    T r2 = (ch2 - w[j] * c.z) * inv_rest - t2;
                    v[10] = r0 * r0 + r1 * r1 + r2 * r2 - pl;
                }
            }
            sm.key[e] = id;
            bool bad = false;
#pragma unroll
            for (int t = 0; t < NCH; t++) bad |= !c_finite(v[t]);
            if (bad) {
#pragma unroll
                for (int t = 0; t < NCH; t++)
                    if (!c_finite(v[t])) {
                        v[t] = T(0);
                        nonfinite++;
                    }
            }
#pragma unroll
            for (int t = 0; t < NCH; t++) sm.c[t * Red::ES + e] = v[t];
        }
    } else {
#pragma unroll
        for (int j = 0; j < H; j++) sm.key[(half * H + j) * TPX + pix] = kEmpty;
    }
    __syncthreads();
    PH(0);
    tile_reduce(sm, red);
    __syncthreads();
    if (MODE != 2) block_dd_store<NT>(loss, sm.warp_part, loss_part + blockIdx.y * gridDim.x + blockIdx.x);
    __syncthreads();
    unsigned long long nf = block_sum_u64<NT>(nonfinite, reinterpret_cast<unsigned long long*>(sm.warp_part));
    if (threadIdx.x == 0 && nf) atomicAdd(reinterpret_cast<unsigned long long*>(&st->nonfinite), nf);
}

static constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
static constexpr int lcm_c(int a, int b) { return a / gcd_c(a, b) * b; }
int tile_row_quantum() {
    constexpr int kStatsTH = 8;  // k_stats / k_stats2 tiles
    return lcm_c(lcm_c(BwdTile<float>::TH, BwdTile<double>::TH), kStatsTH);
}

int backward_ord_blocks(const FieldDims& f);
int backward_blocks(bool fp64, const FieldDims& f, bool ordered) {
    if (fp64 && ordered) return backward_ord_blocks(f);
    int tw = fp64 ? BwdTile<double>::TW : BwdTile<float>::TW, th = fp64 ? BwdTile<double>::TH : BwdTile<float>::TH;
    return ((f.width + tw - 1) / tw) * ((rows_of(f, f.height) + th - 1) / th);
}

template <typename T, int KM, int MODE>
static void backward_attr() {
    constexpr int TW = BwdTile<T>::TW, TH = BwdTile<T>::TH;
    constexpr int NCH = MODE == 1 ? 11 : 10;
    cudaFuncSetAttribute(k_backward<T, KM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileRed<T, NCH, TW * TH, KM>));
    if (sizeof(T) == 4)
        cudaFuncSetAttribute(k_backward2<KM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(TileRed<float, NCH, 16 * SAD_BWD2_TH, KM, 32 * SAD_BWD2_TH>));
}

// SAD_BWD1=1 selects the one-lane-per-pixel fp32 kernel (A/B and regression checks)
static const bool g_bwd1 = getenv("SAD_BWD1") != nullptr;

template <typename T, int KM, int MODE>
static void backward_t(const uint32_t* ids, const void* gtab, const void* tgt, const FieldDims& f, double scale,
                       const RedTarget& red, double2* loss_part, DevState* st, cudaStream_t stream) {
    constexpr int TW = BwdTile<T>::TW, TH = BwdTile<T>::TH;
    constexpr int NCH = MODE == 1 ? 11 : 10;
    dim3 grid((f.width + TW - 1) / TW, (rows_of(f, f.height) + TH - 1) / TH);
    T inv_hw2 = static_cast<T>(2.0 / (static_cast<double>(f.width) * f.height));
    if (sizeof(T) == 4 && !g_bwd1) {
        static_assert(BwdTile<float>::TW == 16 && BwdTile<float>::TH == SAD_BWD2_TH, "k_backward2 tile");
        size_t smem = sizeof(TileRed<float, NCH, 16 * SAD_BWD2_TH, KM, 32 * SAD_BWD2_TH>);
        launch_pdl(k_backward2<KM, MODE>, grid, dim3(32 * SAD_BWD2_TH), smem, stream, ids, (const Q4<float>*)gtab,
                   (const float*)tgt, f, static_cast<float>(scale), static_cast<float>(inv_hw2), red, loss_part, st);
    } else {
        size_t smem = sizeof(TileRed<T, NCH, TW * TH, KM>);
        auto kern = k_backward<T, KM, MODE>;
        kern<<<grid, TW * TH, smem, stream>>>(ids, (const Q4<T>*)gtab, (const T*)tgt, f, static_cast<T>(scale),
                                              inv_hw2, red, loss_part, st);
    }
    SAD_LAUNCHED();
}

template <int KM, int MODE>
static void backward_ord_t(const uint32_t* ids, const void* gtab, const void* tgt, const FieldDims& f, double scale,
                           const RedTarget& red, double2* loss_part, DevState* st, cudaStream_t stream);

void launch_backward(bool fp64, int mode, const uint32_t* ids, const void* gtab, const void* tgt, const FieldDims& f,
                     double scale, const RedTarget& red, double2* loss_part, DevState* st, cudaStream_t stream) {
#define SAD_BWD_ORD(KM)                                                                                 \
    do {                                                                                               \
        if (mode == 0) backward_ord_t<KM, 0>(ids, gtab, tgt, f, scale, red, loss_part, st, stream);     \
        else if (mode == 1) backward_ord_t<KM, 1>(ids, gtab, tgt, f, scale, red, loss_part, st, stream); \
        else backward_ord_t<KM, 2>(ids, gtab, tgt, f, scale, red, loss_part, st, stream);               \
    } while (0)
#define SAD_BWD(T, KM)                                                                                 \
    do {                                                                                               \
        if (mode == 0) backward_t<T, KM, 0>(ids, gtab, tgt, f, scale, red, loss_part, st, stream);      \
        else if (mode == 1) backward_t<T, KM, 1>(ids, gtab, tgt, f, scale, red, loss_part, st, stream); \
        else backward_t<T, KM, 2>(ids, gtab, tgt, f, scale, red, loss_part, st, stream);                \
    } while (0)
    if (fp64 && red.tag) {  // the reference's summation order (k_backward_ord)
        if (f.k <= 8) SAD_BWD_ORD(8);
        else SAD_BWD_ORD(16);
    } else if (fp64) {
        if (f.k <= 8) SAD_BWD(double, 8);
        else SAD_BWD(double, 16);
    } else {
        if (f.k <= 8) SAD_BWD(float, 8);
        else SAD_BWD(float, 16);
    }
#undef SAD_BWD
#undef SAD_BWD_ORD
}

bool fp64_ordered() { return getenv("SAD_FP64_DD") == nullptr; }  // read per fit / per call

// ====================================================================== fp64 backward in the reference's order
// The reference's per-site sums are Accum cascades (accum.hpp:14-26: hi = fl(hi + x), lo += the
// two-sum error), which are exact -- and so order-independent -- for float contributions but not for
// doubles.  For fp64 the B200 path therefore replays the reference's order itself (backward_impl,
// grad.cpp:242-289, at RunOpts::threads = 1, the library default, types.hpp:163-172):
//   * 16x16 tiles in raster order; inside a tile the TileReducer (grad.cpp:37-64) with its 256-slot
//     table, tile_hash and 8 linear probes (grad.hpp:67-90): a site that finds a slot accumulates a
//     per-tile Accum over the tile's contributions in pixel-major order (pixels row-major, list slots
//     in order) and is flushed into the buffer as add(hi), add(lo); a site that finds none overflows
//     and each of its contributions is added to the buffer directly, in pixel order;
//   * the output buffer then receives the worker buffer as add(hi), add(lo) (GradBuffer::merge), and
//     grad() is hi + lo.
// k_backward_ord emits one tagged record per (site, tile) Accum and one per overflowed contribution
// (tag = tile << 9 | [0x100 | pixel] for raw contributions); ord_total replays a site's records in tag
// order through the same Accum.  All arithmetic is the reference's (--fmad=false): contributions are
// recomputed in the replay from the forward pass's weights and per-pixel state, with the same
// expressions as k_backward, so every contribution has the same bits in both places.
constexpr int kRefTile = 16;    // grad.cpp:81 kTile
constexpr int kRefTable = 256;  // grad.hpp:67 TileReducer::kTableSize
constexpr int kRefProbes = 8;   // grad.hpp:68 kMaxProbes
constexpr uint32_t kTagRaw = 0x100u;
__device__ __forceinline__ uint32_t ref_tile_hash(uint32_t site) { return (site * 2654435761u) >> 24; }

// Accum::add (accum.hpp:14-21)
__device__ __forceinline__ void ref_add(DD& a, double x) {
    const double sum = __dadd_rn(a.hi, x);
    const double bb = __dsub_rn(sum, a.hi);
    const double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(sum, bb)), __dsub_rn(x, bb));
    a.hi = sum;
    a.lo = __dadd_rn(a.lo, err);
}

// Shared state of one reference tile.  The contributions are computed and replayed in 4 bands of 4
// rows (64 pixels), so only a band's contributions are resident; the per-(site, channel) Accums
// stay in registers across the bands.
#ifndef SAD_ORD_BAND
#define SAD_ORD_BAND 64  // pixels per band (a multiple of 32, at most 64)
#endif
#ifndef SAD_ORD_MINB
#define SAD_ORD_MINB 2  // two 256-thread blocks per SM (<= 128 registers; the shared footprint allows two)
#endif
constexpr int kOrdBandPx = SAD_ORD_BAND;
template <int KM, int NPX, int NCH>
struct OrdTile {
    static constexpr int NP = kRefTile * kRefTile, BE = kOrdBandPx * KM, CS = BE + 1;  // CS: padded row
    uint32_t key[NP * KM];  // kept candidate of entry e = pixel * KM + slot, else kEmpty
    double w[NP * KM];      // its normalised softmax weight
    double pix[NPX][NP];    // per pixel: g0 g1 g2 ch0 ch1 ch2 [t0 t1 t2 pl]
    double c[NCH * CS];     // the band's contributions, channel-major
    uint32_t bm[kRefTable][2];         // per table slot: the band pixels holding its site (64 bits)
    long long rec[kRefTable];          // record claimed per occupied slot (ord_claim code)
    uint32_t tkey[kRefTable];          // the TileReducer table: site per slot (kEmpty: free)
    uint16_t occ[kRefTable];           // occupied slots, compacted
    uint16_t bstart[kRefTable];        // band bucket start per slot
    uint16_t list[BE];                 // band entries bucketed by slot, in pixel order
    uint16_t eslot[BE];                // slot of each band entry (0xffff: none / overflowed)
    int wsum[8];
    DD warp_part[8];
};

// exclusive scan of one int per thread over a 256-thread block
__device__ __forceinline__ int block_excl_scan256(int v, int* wsum, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        const int t = wsum[q];
        off += q < warp ? t : 0;
        tot += t;
    }
    __syncthreads();
    total = tot;
    return off + x - v;
}

// The eleven contribution components of one kept candidate (grad.cpp:193-238): the expressions of
// k_backward in the same order.  Returns the number of non-finite components (scrubbed to zero).
template <int NCH>
__device__ __forceinline__ int ord_contrib(double fx, double fy, double wi, const Q4<double>& a, const Q4<double>& b,
                                           const Q4<double>& c, double s, const double* pix, int pstride,
                                           double (&v)[NCH]) {
    constexpr double kTiny = 1e-18;
    const double dx = fx - a.x, dy = fy - a.y;
    const double pa = b.z * dx + b.w * dy;
    const double pb = b.z * dy - b.w * dx;
    double q = b.x * pa * pa + b.y * pb * pb;
    if (q < 0.0) q = 0.0;
    const double m = __dsqrt_rn(q);
    const double l = -a.z * (m * s - a.w * s);
    const double g0 = pix[0], g1 = pix[pstride], g2 = pix[2 * pstride];
    const double ch0 = pix[3 * pstride], ch1 = pix[4 * pstride], ch2 = pix[5 * pstride];
    const double dc0 = c.x - ch0, dc1 = c.y - ch1, dc2 = c.z - ch2;
    const double A = wi * (g0 * dc0 + g1 * dc1 + g2 * dc2);
    const double ts = a.z * s;
    v[4] = wi * g0;
    v[5] = wi * g1;
    v[6] = wi * g2;
    v[2] = A * l;
    v[3] = A * ts;
    if (m > kTiny) {
        const double inv_n = __drcp_rn(m);
        const double eau = b.x * pa;
        const double iav = b.y * pb;
        const double coef = A * ts * inv_n;
        v[0] = coef * (eau * b.z - iav * b.w);
        v[1] = coef * (eau * b.w + iav * b.z);
        v[7] = -coef * (eau * dx + iav * dy);
        v[8] = -coef * (eau * dy - iav * dx);
        v[9] = -A * ts * 0.5 * inv_n * (eau * pa - iav * pb);
    } else {
        v[0] = v[1] = v[7] = v[8] = v[9] = 0.0;
    }
    if constexpr (NCH == 11) {
        const double t0 = pix[6 * pstride], t1 = pix[7 * pstride], t2 = pix[8 * pstride], pl = pix[9 * pstride];
        if (wi >= 1.0 - 1e-6) {
            v[10] = 1e6;
        } else {
            const double inv_rest = __drcp_rn(1.0 - wi);
            const double r0 = (ch0 - wi * c.x) * inv_rest - t0;
            const double r1 = (ch1 - wi * c.y) * inv_rest - t1;
            const double r2 = (ch2 - wi * c.z) * inv_rest - t2;
            v[10] = r0 * r0 + r1 * r1 + r2 * r2 - pl;
        }
    }
    int bad = 0;
#pragma unroll
    for (int t = 0; t < NCH; t++)
        if (!c_finite(v[t])) {
            v[t] = 0.0;
            bad++;
        }
    return bad;
}

// A site's per-tile record in two steps: one thread claims it (code >= 0: part record, <= -2: opart
// record -2 - code, -1: pools full) and writes the tag; each channel's owner then stores its Accum.
__device__ __forceinline__ long long ord_claim(const RedTarget& red, uint32_t site, uint32_t tag) {
    const int slot = atomicAdd(red.cnt + site, 1);
    if (red.roff) {
        const long long rec = static_cast<long long>(red.roff[site]) + slot;
        if (slot < red.rcap[site] && rec < red.psize) {
            red.tag[rec] = tag;
            return rec;
        }
    } else if (slot < red.maxt) {
        const long long rec = static_cast<long long>(site) * red.maxt + slot;
        red.tag[rec] = tag;
        return rec;
    }
    const int ro = atomicAdd(red.otop, 1);
    if (ro >= red.ocap) return -1;
    red.otag[ro] = tag;
    red.onext[ro] = atomicExch(red.head + site, ro);
    return -2 - static_cast<long long>(ro);
}

__device__ __forceinline__ void ord_put(const RedTarget& red, long long code, uint32_t site, int ch, const DD& a,
                                        DevState* st) {
    if (code >= 0) {
        red.part[static_cast<size_t>(code) * red.stride + ch] = make_double2(a.hi, a.lo);
    } else if (code <= -2) {
        red.opart[static_cast<size_t>(-2 - code) * red.stride + ch] = make_double2(a.hi, a.lo);
    } else {
        atomicOr(&st->err, 8);
        dd_atomic_merge(red.over + static_cast<size_t>(ch) * red.cap + site, a);
    }
}

// One tagged record for `site` written by one thread (raw contributions of an overflowed site).
template <int NCH>
__device__ __forceinline__ void ord_store(const RedTarget& red, uint32_t site, uint32_t tag, const double (&hi)[NCH],
                                          const double (&lo)[NCH], DevState* st) {
    const long long code = ord_claim(red, site, tag);
#pragma unroll
    for (int ch = 0; ch < NCH; ch++) ord_put(red, code, site, ch, DD{hi[ch], lo[ch]}, st);
}

#if SAD_ORD_DEBUG
__device__ unsigned long long g_ord_clk[8];
__device__ unsigned long long g_ord_launch;
#define ORD_T(i)                                                  \
    do {                                                          \
        if (threadIdx.x == 0) {                                   \
            const long long _n = clock64();                       \
            atomicAdd(&g_ord_clk[i], (unsigned long long)(_n - _t)); \
            _t = _n;                                              \
        }                                                         \
    } while (0)
#else
#define ORD_T(i) \
    do {         \
    } while (0)
#endif
template <int KM, int MODE>
__global__ void __launch_bounds__(256, SAD_ORD_MINB) k_backward_ord(const uint32_t* __restrict__ ids, const Q4<double>* __restrict__ gtab,
                                                      const double* __restrict__ tgt, FieldDims f, double s,
                                                      double inv_hw2, RedTarget red, double2* __restrict__ loss_part,
                                                      DevState* st) {
    constexpr int NCH = MODE == 1 ? 11 : 10, NPX = MODE == 1 ? 10 : 6, NP = kRefTile * kRefTile;
    using Sm = OrdTile<KM, NPX, NCH>;
    constexpr int BE = Sm::BE, CS = Sm::CS;
    extern __shared__ __align__(16) unsigned char smraw[];
    Sm& sm = *reinterpret_cast<Sm*>(smraw);
    const int tid = threadIdx.x;
#if SAD_ORD_DEBUG
    long long _t = clock64();
#endif
    const int px = blockIdx.x * kRefTile + (tid % kRefTile);
    const int py = blockIdx.y * kRefTile + (tid / kRefTile) + f.row0;
    const bool inside = px < f.width && py < f.height && py < f.row1;
    // raster order of the reference's tiles over the whole image (a strip starts at a tile row: row0 % 16 == 0)
    const uint32_t tile = (blockIdx.y + static_cast<uint32_t>(f.row0) / kRefTile) * gridDim.x + blockIdx.x;
    sm.tkey[tid] = kEmpty;
    const double fx = static_cast<double>(px), fy = static_cast<double>(py);

    // ---- forward of this thread's pixel (k_backward's first half, same expressions)
    unsigned long long nonfinite = 0;
    DD loss{0.0, 0.0};
    {
        uint32_t cid[KM];
        double lg[KM], w[KM];
        bool ok[KM];
        bool any = false;
        double best = 0.0;
        const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
        bool stop = !inside;
#pragma unroll
        for (int i = 0; i < KM; i++) {
            uint32_t id = kEmpty;
            if (!stop && i < f.k) id = lst[i];
            stop = stop || id == kEmpty;
            cid[i] = id;
            ok[i] = false;
            lg[i] = 0.0;
            w[i] = 0.0;
            if (!stop) {
                const Q4<double> a = gtab[3 * id], b = gtab[3 * id + 1];
                const double act = gtab[3 * id + 2].w;
                const double dx = fx - a.x, dy = fy - a.y;
                const double pa = b.z * dx + b.w * dy;
                const double pb = b.z * dy - b.w * dx;
                double q = b.x * pa * pa + b.y * pb * pb;
                if (q < 0.0) q = 0.0;
                const double m = __dsqrt_rn(q);
                const double l = -a.z * (m * s - a.w * s);
                ok[i] = act != 0.0 && c_finite(l);
                lg[i] = l;
                if (ok[i] && (!any || l > best)) best = l;
                any = any || ok[i];
            }
        }
        if (inside && !any) atomicOr(&st->err, 1);
        double ch0 = 0.0, ch1 = 0.0, ch2 = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0, t0 = 0.0, t1 = 0.0, t2 = 0.0, pl = 0.0;
        if (any) {
            double wsum = 0.0;
#pragma unroll
            for (int i = 0; i < KM; i++) {
                w[i] = 0.0;
                if (ok[i]) {
                    w[i] = sad_dexp(lg[i] - best);
                    wsum += w[i];
                }
            }
            const double invw = __drcp_rn(wsum);
#pragma unroll
            for (int i = 0; i < KM; i++)
                if (ok[i]) {
                    w[i] *= invw;
                    const Q4<double> c = gtab[3 * cid[i] + 2];
                    ch0 += w[i] * c.x;
                    ch1 += w[i] * c.y;
                    ch2 += w[i] * c.z;
                }
            const double* tp = tgt + 3 * (static_cast<size_t>(py) * f.width + px);
            if (MODE != 2) {
                t0 = tp[0];
                t1 = tp[1];
                t2 = tp[2];
                const double e0 = ch0 - t0, e1 = ch1 - t1, e2 = ch2 - t2;
                pl = e0 * e0 + e1 * e1 + e2 * e2;
                double plv = pl;
                if (!c_finite(pl)) {
                    nonfinite++;
                    plv = 0;
                }
                dd_add(loss, plv);
                g0 = inv_hw2 * e0;
                g1 = inv_hw2 * e1;
                g2 = inv_hw2 * e2;
            } else {
                g0 = tp[0];
                g1 = tp[1];
                g2 = tp[2];
            }
        }
#pragma unroll
        for (int i = 0; i < KM; i++) {
            sm.key[tid * KM + i] = any && ok[i] ? cid[i] : kEmpty;
            sm.w[tid * KM + i] = w[i];
        }
        sm.pix[0][tid] = g0;
        sm.pix[1][tid] = g1;
        sm.pix[2][tid] = g2;
        sm.pix[3][tid] = ch0;
        sm.pix[4][tid] = ch1;
        sm.pix[5][tid] = ch2;
        if constexpr (NPX == 10) {
            sm.pix[6][tid] = t0;
            sm.pix[7][tid] = t1;
            sm.pix[8][tid] = t2;
            sm.pix[9][tid] = pl;
        }
    }
    __syncthreads();
    ORD_T(0);

    // ---- the TileReducer's table (grad.cpp:40-57, grad.hpp:67-90).  Only a site's first appearance in
    // entry order can change it (later ones find the site, or overflow again: the table only fills), so:
    // (1) first appearances, in parallel: a tile-local hash (in the band buffer, unused until the bands)
    //     keeps each distinct site's smallest entry index;
    // (2) those sites compacted in entry order (block scan over the threads' pixel-major entries);
    // (3) warp 0 inserts them 32 at a time speculatively: each lane takes the first free slot of its 8
    //     probes in the current table; a lane whose probe run [home, slot] holds an earlier lane's slot
    //     would have probed differently, so the batch commits up to the first such lane and resumes there.
    {
        constexpr int HS = NP * KM;  // local hash slots (>= distinct sites)
        uint32_t* hk = reinterpret_cast<uint32_t*>(sm.c);
        int* hf = reinterpret_cast<int*>(hk + HS);
        uint16_t* he = reinterpret_cast<uint16_t*>(hf + HS);
        uint32_t* fa = reinterpret_cast<uint32_t*>(he + HS);
        for (int j = tid; j < HS; j += NP) {
            hk[j] = kEmpty;
            hf[j] = 0x7fffffff;
        }
        __syncthreads();
#pragma unroll 1
        for (int i = 0; i < KM; i++) {
            const int e = tid * KM + i;
            const uint32_t k = sm.key[e];
            // lanes holding the same site in list slot i: the lowest (smallest entry) inserts for all
            const unsigned grp = __match_any_sync(0xffffffffu, k);
            const int leader = __ffs(grp) - 1;
            uint32_t h = 0;
            if (k != kEmpty && (tid & 31) == leader) {
                h = (k * 2654435761u) & (HS - 1);
                for (;;) {
                    const uint32_t old = atomicCAS(&hk[h], kEmpty, k);
                    if (old == kEmpty || old == k) break;
                    h = (h + 1) & (HS - 1);
                }
                atomicMin(&hf[h], e);
            }
            h = __shfl_sync(0xffffffffu, h, leader);
            if (k != kEmpty) he[e] = static_cast<uint16_t>(h);
        }
        __syncthreads();
        int nfirst = 0;
#pragma unroll 1
        for (int i = 0; i < KM; i++) {
            const int e = tid * KM + i;
            nfirst += sm.key[e] != kEmpty && hf[he[e]] == e;
        }
        int n_fa;
        int pos = block_excl_scan256(nfirst, sm.wsum, n_fa);
#pragma unroll 1
        for (int i = 0; i < KM; i++) {
            const int e = tid * KM + i;
            if (sm.key[e] != kEmpty && hf[he[e]] == e) fa[pos++] = sm.key[e];
        }
        __syncthreads();
        int* claim = reinterpret_cast<int*>(fa + HS);  // [kRefTable], 32 = unclaimed
        static_assert(HS * 14 + kRefTable * 4 <= NCH * CS * 8, "claim array exceeds the band buffer");
        for (int j = tid; j < kRefTable; j += NP) claim[j] = 32;
        __syncthreads();
        if (tid < 32) {
            const int lane = tid;
            for (int base = 0; base < n_fa;) {
                const int m = n_fa - base < 32 ? n_fa - base : 32;
                const uint32_t k = lane < m ? fa[base + lane] : kEmpty;
                const uint32_t h = ref_tile_hash(k);
                int slot = -1;  // first free probe slot, -1: all eight taken (overflow)
                if (lane < m) {
                    uint32_t t[kRefProbes];
#pragma unroll
                    for (int q = 0; q < kRefProbes; q++) t[q] = sm.tkey[(h + q) & (kRefTable - 1)];
#pragma unroll
                    for (int q = kRefProbes - 1; q >= 0; q--)
                        if (t[q] == kEmpty) slot = q;
                }
                // claim[pos]: the lowest lane whose chosen slot is pos (the batch's speculative inserts)
                const uint32_t mine = (h + static_cast<uint32_t>(slot)) & (kRefTable - 1);
                if (slot >= 0) atomicMin(&claim[mine], lane);
                __syncwarp();
                bool valid = true;
                if (slot > 0) {  // an earlier lane's slot inside my probe run [home, home + slot]
#pragma unroll
                    for (int q = 0; q < kRefProbes; q++)
                        if (q <= slot && claim[(h + q) & (kRefTable - 1)] < lane) valid = false;
                } else if (slot == 0) {
                    valid = claim[mine] == lane;
                }
                __syncwarp();
                if (slot >= 0) claim[mine] = 32;
                const unsigned bad = __ballot_sync(0xffffffffu, lane < m && !valid);
                const int commit = bad ? __ffs(bad) - 1 : m;  // lane 0 is always valid: commit >= 1
                if (lane < commit && slot >= 0) sm.tkey[(h + static_cast<uint32_t>(slot)) & (kRefTable - 1)] = k;
                __syncwarp();
                base += commit;
            }
        }
    }
    __syncthreads();
    ORD_T(1);

    // ---- the occupied table slots, compacted; thread t owns the (slot, channel) items t + 256 j
    int n_occ;
    {
        const bool o = sm.tkey[tid] != kEmpty;
        const int pos = block_excl_scan256(o ? 1 : 0, sm.wsum, n_occ);
        if (o) sm.occ[pos] = static_cast<uint16_t>(tid);
    }
    const int n_items = n_occ * NCH;
    DD acc[NCH];
#pragma unroll
    for (int j = 0; j < NCH; j++) acc[j] = DD{0.0, 0.0};
#pragma unroll 1
    for (int band = 0; band < NP / kOrdBandPx; band++) {
        sm.bm[tid][0] = sm.bm[tid][1] = 0u;
        __syncthreads();
        ORD_T(2);
        // contributions of the band's entries (pixel-major); an overflowed site's go out as raw records
#pragma unroll 1
        for (int le = tid; le < BE; le += NP) {
            const int lp = le / KM, p = band * kOrdBandPx + lp, e = p * KM + (le - lp * KM);
            const uint32_t k = sm.key[e];
            uint16_t us = 0xffffu;
            if (k != kEmpty) {
                const uint32_t h = ref_tile_hash(k);
                int u = -1;
#pragma unroll
                for (int q = kRefProbes - 1; q >= 0; q--)
                    if (sm.tkey[(h + q) & (kRefTable - 1)] == k) u = static_cast<int>((h + q) & (kRefTable - 1));
                double v[NCH];
                const double ffx = static_cast<double>(blockIdx.x * kRefTile + (p % kRefTile));
                const double ffy = static_cast<double>(blockIdx.y * kRefTile + (p / kRefTile) + f.row0);
                nonfinite += ord_contrib<NCH>(ffx, ffy, sm.w[e], gtab[3 * k], gtab[3 * k + 1], gtab[3 * k + 2], s,
                                              &sm.pix[0][p], NP, v);
                if (u >= 0) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ch++) sm.c[ch * CS + le] = v[ch];
                    atomicOr(&sm.bm[u][lp >> 5], 1u << (lp & 31));
                    us = static_cast<uint16_t>(u);
                } else {
                    double z[NCH];
#pragma unroll
                    for (int ch = 0; ch < NCH; ch++) z[ch] = 0.0;
                    ord_store<NCH>(red, k, (tile << 9) | kTagRaw | static_cast<uint32_t>(p), v, z, st);
                }
            }
            sm.eslot[le] = us;
        }
        __syncthreads();
        ORD_T(3);
        // bucket the band's entries by slot, in pixel order (a site occurs once per pixel)
        {
            int tot;
            sm.bstart[tid] = static_cast<uint16_t>(
                block_excl_scan256(__popc(sm.bm[tid][0]) + __popc(sm.bm[tid][1]), sm.wsum, tot));
        }
        __syncthreads();
        ORD_T(4);
#pragma unroll 1
        for (int le = tid; le < BE; le += NP) {
            const int us = sm.eslot[le];
            if (us == 0xffff) continue;
            const int lp = le / KM;
            const unsigned long long bits = sm.bm[us][0] | (static_cast<unsigned long long>(sm.bm[us][1]) << 32);
            sm.list[sm.bstart[us] + __popcll(bits & ((1ull << lp) - 1ull))] = static_cast<uint16_t>(le);
        }
        __syncthreads();
        ORD_T(5);
        // replay: each item continues its (site, channel) Accum over the band's bucket
#pragma unroll
        for (int j = 0; j < NCH; j++) {
            const int item = tid + NP * j;
            if (item < n_items) {
                const int ui = item / NCH, ch = item - ui * NCH;
                const int u = sm.occ[ui];
                const int b0 = sm.bstart[u], n = __popc(sm.bm[u][0]) + __popc(sm.bm[u][1]);
                const double* crow = sm.c + ch * CS;
#pragma unroll 4
                for (int q = 0; q < n; q++) ref_add(acc[j], crow[sm.list[b0 + q]]);
            }
        }
        __syncthreads();
        ORD_T(6);
    }
    // ---- one record per occupied slot: the per-tile Accums, flushed as end_tile does
    for (int ui = tid; ui < n_occ; ui += NP) sm.rec[ui] = ord_claim(red, sm.tkey[sm.occ[ui]], tile << 9);
    __syncthreads();
    ORD_T(7);
#pragma unroll
    for (int j = 0; j < NCH; j++) {
        const int item = tid + NP * j;
        if (item < n_items) {
            const int ui = item / NCH, ch = item - ui * NCH;
            ord_put(red, sm.rec[ui], sm.tkey[sm.occ[ui]], ch, acc[j], st);
        }
    }
    __syncthreads();
    ORD_T(7);
    if (MODE != 2) block_dd_store<NP>(loss, sm.warp_part, loss_part + blockIdx.y * gridDim.x + blockIdx.x);
    __syncthreads();
    unsigned long long nf = block_sum_u64<NP>(nonfinite, reinterpret_cast<unsigned long long*>(sm.warp_part));
    if (threadIdx.x == 0 && nf) atomicAdd(reinterpret_cast<unsigned long long*>(&st->nonfinite), nf);
}

int backward_ord_blocks(const FieldDims& f) {
    return ((f.width + kRefTile - 1) / kRefTile) * ((rows_of(f, f.height) + kRefTile - 1) / kRefTile);
}

template <int KM, int MODE>
static void backward_ord_t(const uint32_t* ids, const void* gtab, const void* tgt, const FieldDims& f, double scale,
                           const RedTarget& red, double2* loss_part, DevState* st, cudaStream_t stream) {
    constexpr int NPX = MODE == 1 ? 10 : 6, NCH = MODE == 1 ? 11 : 10;
    const size_t smem = sizeof(OrdTile<KM, NPX, NCH>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_backward_ord<KM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    dim3 grid((f.width + kRefTile - 1) / kRefTile, (rows_of(f, f.height) + kRefTile - 1) / kRefTile);
    const double inv_hw2 = 2.0 / (static_cast<double>(f.width) * f.height);
    k_backward_ord<KM, MODE><<<grid, kRefTile * kRefTile, smem, stream>>>(
        ids, (const Q4<double>*)gtab, (const double*)tgt, f, scale, inv_hw2, red, loss_part, st);
    SAD_LAUNCHED();
}

// ---- replay of one site's records in tag order (grad.cpp:59-64 flushes, :285-288 merge): one warp
// per site; up to kOrdFast records are ranked in shared memory, more take a selection walk over the
// tags in global memory.  Lane ch < NCH replays channel ch; returns the output Accum of the channel.
constexpr int kOrdFast = 128;
#if SAD_ORD_DEBUG
__device__ int g_ord_dbg;
#endif
struct OrdRef {
    uint32_t tag;
    int32_t rec;  // >= 0: part record, < 0: opart record ~rec
};

template <int NCH>
__device__ DD ord_total(const RedTarget& red, int id, int n_slice, long long base, OrdRef* buf, int* sorted) {
    const int lane = threadIdx.x & 31;
    // gather: the slice, then the overflow list (walked by lane 0)
    int n = n_slice;
    for (int j = lane; j < n_slice && j < kOrdFast; j += 32)
        buf[j] = OrdRef{red.tag[base + j], static_cast<int32_t>(base + j)};
    if (lane == 0) {
        for (int r = red.head[id]; r >= 0; r = red.onext[r]) {
            if (n < kOrdFast) buf[n] = OrdRef{red.otag[r], ~r};
            n++;
        }
    }
    n = __shfl_sync(0xffffffffu, n, 0);
    __syncwarp();
    DD buf_acc{0.0, 0.0};
    auto replay = [&](int32_t rec, uint32_t tag) {
        if (lane >= NCH) return;
        const double2 v = rec >= 0 ? red.part[static_cast<size_t>(rec) * red.stride + lane]
                                   : red.opart[static_cast<size_t>(~rec) * red.stride + lane];
        ref_add(buf_acc, v.x);
        if (!(tag & kTagRaw)) ref_add(buf_acc, v.y);
    };
    if (n <= kOrdFast) {
        for (int j = lane; j < n; j += 32) {
            const uint32_t t = buf[j].tag;
            int rank = 0;
            for (int q = 0; q < n; q++) rank += buf[q].tag < t;
            sorted[rank] = j;
        }
        __syncwarp();
        // eight records' values in flight per lane, then their cascade steps in order
        if (lane < NCH) {
            for (int r0 = 0; r0 < n; r0 += 8) {
                double2 v[8];
                bool raw[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    v[q] = make_double2(0.0, 0.0);
                    raw[q] = true;
                    if (r0 + q < n) {
                        const OrdRef o = buf[sorted[r0 + q]];
                        v[q] = o.rec >= 0 ? red.part[static_cast<size_t>(o.rec) * red.stride + lane]
                                          : red.opart[static_cast<size_t>(~o.rec) * red.stride + lane];
                        raw[q] = (o.tag & kTagRaw) != 0;
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; q++)
                    if (r0 + q < n) {
                        ref_add(buf_acc, v[q].x);
                        if (!raw[q]) ref_add(buf_acc, v[q].y);
                    }
            }
        }
    } else {
        // selection walk: the next larger tag each step (tags of one site are distinct)
        long long last = -1;
        for (int step = 0; step < n; step++) {
            unsigned best = 0xffffffffu;
            int32_t brec = 0;
            for (int j = lane; j < n_slice; j += 32) {
                const uint32_t t = red.tag[base + j];
                if (static_cast<long long>(t) > last && t <= best) {
                    best = t;
                    brec = static_cast<int32_t>(base + j);
                }
            }
            if (lane == 0)
                for (int r = red.head[id]; r >= 0; r = red.onext[r]) {
                    const uint32_t t = red.otag[r];
                    if (static_cast<long long>(t) > last && t <= best) {
                        best = t;
                        brec = ~r;
                    }
                }
            const unsigned m = __reduce_min_sync(0xffffffffu, best);
            const int src = __ffs(__ballot_sync(0xffffffffu, best == m)) - 1;
            const int32_t rec = __shfl_sync(0xffffffffu, brec, src);
            replay(rec, m);
            last = m;
        }
    }
    // GradBuffer::merge into the zeroed output (grad.cpp:285-288): add(hi), add(lo); a full record
    // pool's CAS totals (st->err bit 3) come last
    DD out{0.0, 0.0};
    ref_add(out, buf_acc.hi);
    ref_add(out, buf_acc.lo);
    if (lane < NCH) {
        const double2 o = red.over[static_cast<size_t>(lane) * red.cap + id];
        if (o.x != 0.0 || o.y != 0.0) dd_merge(out, DD{o.x, o.y});
    }
    return out;
}

// per-site slice bounds of either record layout
__device__ __forceinline__ int ord_slice(const RedTarget& red, int id, long long& base) {
    int n = red.cnt[id];
    if (red.roff) {
        base = red.roff[id];
        if (n > red.rcap[id]) n = red.rcap[id];
        if (base + n > red.psize) n = static_cast<int>(red.psize - base > 0 ? red.psize - base : 0);
    } else {
        base = static_cast<long long>(id) * red.maxt;
        if (n > red.maxt) n = red.maxt;
    }
    return n;
}

// Ordered totals of every live site: values (hi + lo, GradBuffer::grad) into tot[ch][cap] and, with
// `dd`, the output Accums into red.over (the per-call GradBuffer); with `reset` the counters too.
template <int NCH>
__global__ void __launch_bounds__(128) k_ordered_totals(RedTarget red, const DevState* __restrict__ st,
                                                        double* __restrict__ tot, double* __restrict__ g0, int reset) {
    __shared__ OrdRef buf[4][kOrdFast];
    __shared__ int sorted[4][kOrdFast];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int id = blockIdx.x * 4 + warp;
    if (id >= st->n_sites) return;
    long long base = 0;
    const int n_slice = ord_slice(red, id, base);
#if SAD_ORD_DEBUG
    // diagnostics build: k_backward_ord's per-phase clocks (cycles summed over tiles, per launch) every
    // 1000 launches, and sites with long record lists
    if (id == 0 && lane == 0) {
        const unsigned long long L = atomicAdd(&g_ord_launch, 1ull);
        if (L % 1000 == 999)
            printf("ord clk A %llu B %llu bandstart %llu D1 %llu scan %llu scatter %llu D2 %llu records %llu\n",
                   g_ord_clk[0] / (L + 1), g_ord_clk[1] / (L + 1), g_ord_clk[2] / (L + 1), g_ord_clk[3] / (L + 1),
                   g_ord_clk[4] / (L + 1), g_ord_clk[5] / (L + 1), g_ord_clk[6] / (L + 1), g_ord_clk[7] / (L + 1));
    }
    if (lane == 0) {
        int nl = 0;
        for (int r = red.head[id]; r >= 0; r = red.onext[r]) nl++;
        if (n_slice + nl > 64 && atomicAdd(&g_ord_dbg, 1) < 40)
            printf("ord site %d cnt %d slice %d (cap %d) list %d\n", id, red.cnt[id], n_slice,
                   red.roff ? red.rcap[id] : red.maxt, nl);
    }
#endif
    const DD t = ord_total<NCH>(red, id, n_slice, base, buf[warp], sorted[warp]);
    if (lane < NCH) {
        if (tot) tot[static_cast<size_t>(lane) * red.cap + id] = t.hi + t.lo;
        if (g0 && lane == 2) g0[id] = t.hi + t.lo;
        if (!tot) red.over[static_cast<size_t>(lane) * red.cap + id] = make_double2(t.hi, t.lo);
    }
    __syncwarp();
    if (reset && lane == 0) {
        red.cnt[id] = 0;
        red.head[id] = -1;
    }
}

void launch_ordered_totals(const RedTarget& red, int n_ch, const DevState* st, double* tot, double* g0, bool reset,
                           cudaStream_t stream) {
    int grid = (red.cap + 3) / 4;
    if (grid < 1) grid = 1;
    if (n_ch == 11) k_ordered_totals<11><<<grid, 128, 0, stream>>>(red, st, tot, g0, reset ? 1 : 0);
    else k_ordered_totals<10><<<grid, 128, 0, stream>>>(red, st, tot, g0, reset ? 1 : 0);
    SAD_LAUNCHED();
}

// ====================================================================== image_loss (grad.cpp:291-360)
template <typename T, int KM>
__global__ void __launch_bounds__(128) k_loss(const uint32_t* __restrict__ ids, const Q4<T>* __restrict__ gtab,
                                              const T* __restrict__ tgt, FieldDims f, T s, double2* __restrict__ loss_part,
                                              DevState* st) {
    __shared__ DD parts[4];
    const int tid = threadIdx.x;
    const int px = blockIdx.x * 16 + (tid % 16);
    const int py = blockIdx.y * 8 + (tid / 16);
    DD loss{0.0, 0.0};
    if (px < f.width && py < f.height) {
        const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
        uint32_t cid[KM];
        T lg[KM];
        int n = 0;
        T best = T(0);
        const T fx = static_cast<T>(px), fy = static_cast<T>(py);
#pragma unroll
        for (int i = 0; i < KM; i++) {
            cid[i] = 0;
            lg[i] = T(0);
        }
#pragma unroll
        for (int i = 0; i < KM; i++) {
            if (i >= f.k) break;
            uint32_t id = lst[i];
            if (id == kEmpty) break;
            const Q4<T> a = gtab[3 * id], b = gtab[3 * id + 1];
            if (gtab[3 * id + 2].w == T(0)) continue;
            T dx = fx - a.x, dy = fy - a.y;
            T pa = b.z * dx + b.w * dy;
            T pb = b.z * dy - b.w * dx;
            T q = b.x * pa * pa + b.y * pb * pb;
            if (q < T(0)) q = T(0);
            T m = tsqrt(q);
            T l = -a.z * (m * s - a.w * s);
            if (!tfinite(l)) continue;
#pragma unroll
            for (int j = 0; j < KM; j++)
                if (j == n) {
                    cid[j] = id;
                    lg[j] = l;
                }
            if (n == 0 || l > best) best = l;
            n++;
        }
        if (n == 0) {
            atomicOr(&st->err, 1);
        } else {
            T w[KM];
            T wsum = T(0);
#pragma unroll
            for (int i = 0; i < KM; i++)
                if (i < n) {
                    w[i] = texp(lg[i] - best);
                    wsum += w[i];
                }
            T invw = trcp(wsum);
            T c0 = T(0), c1 = T(0), c2 = T(0);
#pragma unroll
            for (int i = 0; i < KM; i++)
                if (i < n) {
                    T wi = w[i] * invw;
                    const Q4<T> c = gtab[3 * cid[i] + 2];
                    c0 += wi * c.x;
                    c1 += wi * c.y;
                    c2 += wi * c.z;
                }
            const T* tp = tgt + 3 * (static_cast<size_t>(py) * f.width + px);
            T e0 = c0 - tp[0], e1 = c1 - tp[1], e2 = c2 - tp[2];
            double pl = static_cast<double>(e0 * e0 + e1 * e1 + e2 * e2);
            if (isfinite(pl)) dd_add(loss, pl);
        }
    }
    block_dd_store<128>(loss, parts, loss_part + blockIdx.y * gridDim.x + blockIdx.x);
}

int loss_blocks(const FieldDims& f) { return ((f.width + 15) / 16) * ((f.height + 7) / 8); }

void launch_loss(bool fp64, const uint32_t* ids, const void* gtab, const void* tgt, const FieldDims& f, double scale,
                 double2* lp, DevState* st, cudaStream_t stream) {
    dim3 grid((f.width + 15) / 16, (f.height + 7) / 8);
    if (fp64) {
        if (f.k <= 8) k_loss<double, 8><<<grid, 128, 0, stream>>>(ids, (const Q4<double>*)gtab, (const double*)tgt, f, scale, lp, st);
        else k_loss<double, 16><<<grid, 128, 0, stream>>>(ids, (const Q4<double>*)gtab, (const double*)tgt, f, scale, lp, st);
    } else {
        float s = static_cast<float>(scale);
        if (f.k <= 8) k_loss<float, 8><<<grid, 128, 0, stream>>>(ids, (const Q4<float>*)gtab, (const float*)tgt, f, s, lp, st);
        else k_loss<float, 16><<<grid, 128, 0, stream>>>(ids, (const Q4<float>*)gtab, (const float*)tgt, f, s, lp, st);
    }
    SAD_LAUNCHED();
}

// Compensated sum of per-block loss partials into dst (one block; order independent).
__global__ void k_loss_reduce(const double2* __restrict__ part, int n, double2* dst) {
    __shared__ DD parts[8];
    DD acc{0.0, 0.0};
    for (int i = threadIdx.x; i < n; i += blockDim.x) dd_merge(acc, DD{part[i].x, part[i].y});
    block_dd_store<256>(acc, parts, dst);
}

void launch_loss_reduce(const double2* loss_part, int n, double2* dst, cudaStream_t stream) {
    k_loss_reduce<<<1, 256, 0, stream>>>(loss_part, n, dst);
    SAD_LAUNCHED();
}

// Merge of per-(site, tile) records into the totals (consumer side of RedTarget).
__device__ __forceinline__ DD red_total(const RedTarget& red, int id, int ch, int n) {
    double2 o = red.over[static_cast<size_t>(ch) * red.cap + id];
    DD acc{o.x, o.y};
    const double2* rec = red.part + static_cast<size_t>(id) * red.maxt * red.stride + ch;
    if (red.roff) {
        const long long base = red.roff[id];
        rec = red.part + static_cast<size_t>(base) * red.stride + ch;
        if (n > red.rcap[id]) n = red.rcap[id];
        if (base + n > red.psize) n = static_cast<int>(red.psize - base > 0 ? red.psize - base : 0);
    }
    SAD_CHECK(!red.roff || n <= 0 || static_cast<long long>(red.roff[id]) + n <= red.psize);
    for (int s = 0; s < n; s++) {
        double2 r = rec[static_cast<size_t>(s) * red.stride];
        dd_merge(acc, DD{r.x, r.y});
    }
    for (int r = red.head[id]; r >= 0; r = red.onext[r]) {
        SAD_CHECK(r < red.ocap);
        double2 o2 = red.opart[static_cast<size_t>(r) * red.stride + ch];
        dd_merge(acc, DD{o2.x, o2.y});
    }
    return acc;
}

// One 16-lane group per site, lane ch < NCH merges channel ch (records, overflow list, CAS totals);
// the counters are reset after the whole group has read them.
template <int NCH>
__global__ void __launch_bounds__(128) k_finalize(RedTarget red, const DevState* __restrict__ st) {
    static_assert(NCH <= 16, "channels per group");
    const int lane16 = threadIdx.x & 15;
    const int id = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const unsigned gmask = 0xffffu << (threadIdx.x & 16);
    const bool live = id < st->n_sites;
    int n = live ? red.cnt[id] : 0;
    if (!red.roff && n > red.maxt) n = red.maxt;  // (adaptive layout: red_total bounds n by rcap / the pool)
    if (live && lane16 < NCH) {
        const DD t = red_total(red, id, lane16, n);
        red.over[static_cast<size_t>(lane16) * red.cap + id] = make_double2(t.hi, t.lo);
    }
    __syncwarp(gmask);
    if (live && lane16 == 0) {
        red.cnt[id] = 0;
        red.head[id] = -1;
    }
}

void launch_finalize(const RedTarget& red, int n_ch, const DevState* st, cudaStream_t stream) {
    int grid = (red.cap + 7) / 8;  // 8 sites (16 lanes each) per block
    if (grid < 1) grid = 1;
    if (n_ch == 8) k_finalize<8><<<grid, 128, 0, stream>>>(red, st);
    else if (n_ch == 10) k_finalize<10><<<grid, 128, 0, stream>>>(red, st);
    else k_finalize<11><<<grid, 128, 0, stream>>>(red, st);
    SAD_LAUNCHED();
}

// ====================================================================== accumulate_stats (budget.cpp:39-155)
// Always double, unpacked ScoreTable logits; 8 channels per (pixel, candidate), same tile contract.
template <int KM>
__global__ void __launch_bounds__(64) k_stats(const uint32_t* __restrict__ ids, const Q4<double>* __restrict__ rtab,
                                             const double* __restrict__ tgt, FieldDims f, double s, RedTarget red,
                                             DevState* st) {
    constexpr int TW = 8, TH = 8, TPX = 64, NCH = 8;
    using Red = TileRed<double, NCH, TPX, KM>;
    extern __shared__ __align__(16) unsigned char smraw[];
    Red& sm = *reinterpret_cast<Red*>(smraw);
    tile_init(sm);
    const int tid = threadIdx.x;
    const int px = blockIdx.x * TW + (tid % TW);
    const int py = blockIdx.y * TH + (tid / TW) + f.row0;
    int n = 0;
    uint32_t cid[KM];
    double lg[KM];
#pragma unroll
    for (int i = 0; i < KM; i++) {
        cid[i] = kEmpty;
        lg[i] = 0;
    }
    double best = 0;
    if (px < f.width && py < f.height && py < f.row1) {
        const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
#pragma unroll
        for (int i = 0; i < KM; i++) {
            if (i >= f.k) break;
            uint32_t id = lst[i];
            if (id == kEmpty) break;
            const Q4<double> a = rtab[3 * id], b = rtab[3 * id + 1];
            if (b.w == 0.0) continue;
            double l = score_logit(a, b, static_cast<double>(px), static_cast<double>(py), s);
            if (!isfinite(l)) continue;
#pragma unroll
            for (int j = 0; j < KM; j++)
                if (j == n) {
                    cid[j] = id;
                    lg[j] = l;
                }
            if (n == 0 || l > best) best = l;
            n++;
        }
    }
    if (n > 0) {
        double w[KM];
        double wsum = 0;
#pragma unroll
        for (int i = 0; i < KM; i++)
            if (i < n) {
                w[i] = sad_dexp(lg[i] - best);
                wsum += w[i];
            }
        double invw = 1.0 / wsum;
        double ch0 = 0, ch1 = 0, ch2 = 0;
#pragma unroll
        for (int i = 0; i < KM; i++)
            if (i < n) {
                w[i] *= invw;
                const Q4<double> c = rtab[3 * cid[i] + 2];
                ch0 += w[i] * c.x;
                ch1 += w[i] * c.y;
                ch2 += w[i] * c.z;
            }
        const double* tp = tgt + 3 * (static_cast<size_t>(py) * f.width + px);
        double e0 = ch0 - tp[0], e1 = ch1 - tp[1], e2 = ch2 - tp[2];
        double r2 = e0 * e0 + e1 * e1 + e2 * e2;
        double fx = px, fy = py;
#pragma unroll
        for (int i = 0; i < KM; i++) {
            if (i >= n) break;
            const Q4<double> c = rtab[3 * cid[i] + 2];
            double rho = w[i] * r2;
            double v[8];
            v[0] = w[i];
            v[1] = rho;
            v[2] = rho * fx;
            v[3] = rho * fy;
            v[4] = rho * fx * fx;
            v[5] = rho * fx * fy;
            v[6] = rho * fy * fy;
            if (w[i] >= 1.0 - 1e-6) {
                v[7] = 1e6;
            } else {
                double ir = 1.0 / (1.0 - w[i]);
                double r0 = (ch0 - w[i] * c.x) * ir - tp[0];
                double r1 = (ch1 - w[i] * c.y) * ir - tp[1];
                double rk = (ch2 - w[i] * c.z) * ir - tp[2];
                v[7] = r0 * r0 + r1 * r1 + rk * rk - r2;
            }
            const int e = i * TPX + tid;
            sm.key[e] = cid[i];
#pragma unroll
            for (int t = 0; t < NCH; t++) sm.c[t * Red::ES + e] = isfinite(v[t]) ? v[t] : 0.0;
        }
    }
#pragma unroll
    for (int i = 0; i < KM; i++)
        if (i >= n) sm.key[i * TPX + tid] = kEmpty;
    __syncthreads();
    tile_reduce(sm, red);
    __syncthreads();
    unsigned long long v = block_sum_u64<TPX>(n > 0 ? 1ull : 0ull, reinterpret_cast<unsigned long long*>(sm.warp_part));
    if (threadIdx.x == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(&st->valid), v);
}

// Opt-in shared-memory sizes of the tile-reduction kernels; called once per context, before any
// launch can be captured into a CUDA graph.
template <int KM>
__global__ void k_stats2(const uint32_t* __restrict__ ids, const Q4<double>* __restrict__ rtab,
                         const double* __restrict__ tgt, FieldDims f, double s, RedTarget red, DevState* st);

void prepare_kernels() {
    backward_attr<float, 8, 0>();
    backward_attr<float, 8, 1>();
    backward_attr<float, 8, 2>();
    backward_attr<float, 16, 0>();
    backward_attr<float, 16, 1>();
    backward_attr<float, 16, 2>();
    backward_attr<double, 8, 0>();
    backward_attr<double, 8, 1>();
    backward_attr<double, 8, 2>();
    backward_attr<double, 16, 0>();
    backward_attr<double, 16, 1>();
    backward_attr<double, 16, 2>();
    cudaFuncSetAttribute(k_stats<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileRed<double, 8, 64, 8>));
    cudaFuncSetAttribute(k_stats<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileRed<double, 8, 64, 16>));
    cudaFuncSetAttribute(k_stats2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileRed<double, 8, 64, 8, 128>));
    cudaFuncSetAttribute(k_stats2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileRed<double, 8, 64, 16, 128>));
}

// Two lanes per pixel (128 threads per 8x8 tile), same hand-over of the order-sensitive double sums
// as k_backward2: lane 0 sums its slots' softmax weights / colours from zero, lane 1 continues from
// lane 0's partial.  Skipped slots (inactive, non-finite logit) do not take part, exactly as the
// reference's compacted candidate loop (budget.cpp:60-100).
template <int KM>
__global__ void __launch_bounds__(128) k_stats2(const uint32_t* __restrict__ ids, const Q4<double>* __restrict__ rtab,
                                               const double* __restrict__ tgt, FieldDims f, double s, RedTarget red,
                                               DevState* st) {
    constexpr int TW = 8, TH = 8, TPX = 64, NT = 128, NCH = 8, H = KM / 2;
    constexpr unsigned FULL = 0xffffffffu;
    using Red = TileRed<double, NCH, TPX, KM, NT>;
    extern __shared__ __align__(16) unsigned char smraw[];
    Red& sm = *reinterpret_cast<Red*>(smraw);
    tile_init(sm);
    const int tid = threadIdx.x;
    const int pix = tid >> 1, half = tid & 1;
    const int px = blockIdx.x * TW + (pix % TW);
    const int py = blockIdx.y * TH + (pix / TW) + f.row0;
    const bool inside = px < f.width && py < f.height && py < f.row1;
    uint32_t cid[H];
    double lg[H];
    bool ok[H];
    bool any = false;
    double best = 0;
    {
        uint32_t idv[H];
        const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
        bool has_empty = false;
        if (SAD_VEC_IDS && H == 4 && f.k == 8) {  // this lane's half of the list in one 16-byte load
            uint4 q = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
            if (inside) q = *reinterpret_cast<const uint4*>(lst + half * 4);
            idv[0] = q.x;
            idv[1] = q.y;
            idv[2 % H] = q.z;
            idv[3 % H] = q.w;
        } else {
#pragma unroll
            for (int j = 0; j < H; j++) {
                const int i = half * H + j;
                idv[j] = (inside && i < f.k) ? lst[i] : kEmpty;
            }
        }
#pragma unroll
        for (int j = 0; j < H; j++) has_empty = has_empty || idv[j] == kEmpty;
        const bool partner_empty = __shfl_xor_sync(FULL, has_empty, 1);
        bool stop = !inside || (half == 1 && partner_empty);
#pragma unroll
        for (int j = 0; j < H; j++) {
            const uint32_t id = idv[j];
            stop = stop || id == kEmpty;
            cid[j] = id;
            ok[j] = false;
            lg[j] = 0;
            if (!stop) {
                const Q4<double> a = rtab[3 * id], b = rtab[3 * id + 1];
                if (b.w != 0.0) {
                    const double l = score_logit(a, b, static_cast<double>(px), static_cast<double>(py), s);
                    if (isfinite(l)) {
                        ok[j] = true;
                        lg[j] = l;
                        if (!any || l > best) best = l;
                        any = true;
                    }
                }
            }
        }
    }
    const bool pany = __shfl_xor_sync(FULL, any, 1);
    const double pbest = __shfl_xor_sync(FULL, best, 1);
    const bool a0 = half == 0 ? any : pany, a1 = half == 0 ? pany : any;
    const double b0 = half == 0 ? best : pbest, b1 = half == 0 ? pbest : best;
    best = a0 ? ((a1 && b1 > b0) ? b1 : b0) : b1;
    const bool any_all = a0 || a1;

    double w[H];
    double wpart = 0;
#pragma unroll
    for (int j = 0; j < H; j++) w[j] = ok[j] ? sad_dexp(lg[j] - best) : 0.0;
    if (half == 0) {
#pragma unroll
        for (int j = 0; j < H; j++)
            if (ok[j]) wpart += w[j];
    }
    const double from0 = __shfl_xor_sync(FULL, wpart, 1);
    if (half == 1) {
        wpart = from0;
#pragma unroll
        for (int j = 0; j < H; j++)
            if (ok[j]) wpart += w[j];
    }
    const double from1 = __shfl_xor_sync(FULL, wpart, 1);
    const double invw = 1.0 / (half == 0 ? from1 : wpart);
    Q4<double> col[H];
    double c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
    for (int j = 0; j < H; j++) {
        col[j] = Q4<double>{0, 0, 0, 0};
        if (ok[j]) {
            w[j] *= invw;
            col[j] = rtab[3 * cid[j] + 2];
        }
    }
    if (half == 0) {
#pragma unroll
        for (int j = 0; j < H; j++)
            if (ok[j]) {
                c0 += w[j] * col[j].x;
                c1 += w[j] * col[j].y;
                c2 += w[j] * col[j].z;
            }
    }
    {
        const double r0 = __shfl_xor_sync(FULL, c0, 1), r1 = __shfl_xor_sync(FULL, c1, 1),
                     r2 = __shfl_xor_sync(FULL, c2, 1);
        if (half == 1) {
            c0 = r0;
            c1 = r1;
            c2 = r2;
#pragma unroll
            for (int j = 0; j < H; j++)
                if (ok[j]) {
                    c0 += w[j] * col[j].x;
                    c1 += w[j] * col[j].y;
                    c2 += w[j] * col[j].z;
                }
        }
        const double s0 = __shfl_xor_sync(FULL, c0, 1), s1 = __shfl_xor_sync(FULL, c1, 1),
                     s2 = __shfl_xor_sync(FULL, c2, 1);
        if (half == 0) {
            c0 = s0;
            c1 = s1;
            c2 = s2;
        }
    }
    if (any_all) {
        const double* tp = tgt + 3 * (static_cast<size_t>(py) * f.width + px);
        const double e0 = c0 - tp[0], e1 = c1 - tp[1], e2 = c2 - tp[2];
        const double r2 = e0 * e0 + e1 * e1 + e2 * e2;
        const double fx = px, fy = py;
#pragma unroll
        for (int j = 0; j < H; j++) {
            const int e = (half * H + j) * TPX + pix;
            if (!ok[j]) {
                sm.key[e] = kEmpty;
                continue;
            }
            const Q4<double> c = col[j];
            const double rho = w[j] * r2;
            double v[8];
            v[0] = w[j];
            v[1] = rho;
            v[2] = rho * fx;
            v[3] = rho * fy;
            v[4] = rho * fx * fx;
            v[5] = rho * fx * fy;
            v[6] = rho * fy * fy;
            if (w[j] >= 1.0 - 1e-6) {
                v[7] = 1e6;
            } else {
                const double ir = 1.0 / (1.0 - w[j]);
                const double q0 = (c0 - w[j] * c.x) * ir - tp[0];
                const double q1 = (c1 - w[j] * c.y) * ir - tp[1];
                const double q2 = (c2 - w[j] * c.z) * ir - tp[2];
                v[7] = q0 * q0 + q1 * q1 + q2 * q2 - r2;
            }
            sm.key[e] = cid[j];
#pragma unroll
            for (int t = 0; t < NCH; t++) sm.c[t * Red::ES + e] = isfinite(v[t]) ? v[t] : 0.0;
        }
    } else {
#pragma unroll
        for (int j = 0; j < H; j++) sm.key[(half * H + j) * TPX + pix] = kEmpty;
    }
    __syncthreads();
    tile_reduce(sm, red);
    __syncthreads();
    unsigned long long v = block_sum_u64<NT>((half == 0 && any_all) ? 1ull : 0ull,
                                             reinterpret_cast<unsigned long long*>(sm.warp_part));
    if (threadIdx.x == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(&st->valid), v);
}

static const bool g_stats1 = getenv("SAD_STATS1") != nullptr;

void launch_stats(const uint32_t* ids, const void* rtab_d, const double* tgt, const FieldDims& f, double scale,
                  const RedTarget& red, DevState* st, cudaStream_t stream) {
    dim3 grid((f.width + 7) / 8, (rows_of(f, f.height) + 7) / 8);
    if (g_stats1) {  // one lane per pixel (A/B)
        if (f.k <= 8)
            k_stats<8><<<grid, 64, sizeof(TileRed<double, 8, 64, 8>), stream>>>(ids, (const Q4<double>*)rtab_d, tgt, f,
                                                                                scale, red, st);
        else
            k_stats<16><<<grid, 64, sizeof(TileRed<double, 8, 64, 16>), stream>>>(ids, (const Q4<double>*)rtab_d, tgt,
                                                                                  f, scale, red, st);
    } else {
        if (f.k <= 8)
            k_stats2<8><<<grid, 128, sizeof(TileRed<double, 8, 64, 8, 128>), stream>>>(ids, (const Q4<double>*)rtab_d,
                                                                                       tgt, f, scale, red, st);
        else
            k_stats2<16><<<grid, 128, sizeof(TileRed<double, 8, 64, 16, 128>), stream>>>(
                ids, (const Q4<double>*)rtab_d, tgt, f, scale, red, st);
    }
    SAD_LAUNCHED();
}

// ====================================================================== adam_step + clamp_project (train.cpp:113-169)
// Per-site thread, bit-exact double arithmetic in the reference order; bias corrections come from
// the host (glibc pow) through `bc`.  Optionally zeroes the gradient accumulators for the next
// iteration and rebuilds this site's candidate snapshot and backward table (the only consumers of
// the new parameters before the next event), which removes two table-build launches per iteration.
__device__ __forceinline__ void clamp_site(double* p, int cap, int id, const AdamHyper& hp) {
    double x = p[0 * cap + id], y = p[1 * cap + id];
    p[0 * cap + id] = smin(smax(x, 0.0), hp.width - 1.0);
    p[1 * cap + id] = smin(smax(y, 0.0), hp.height - 1.0);
    p[2 * cap + id] = smin(smax(p[2 * cap + id], hp.log_tau_min), hp.log_tau_max);
    p[3 * cap + id] = smin(smax(p[3 * cap + id], hp.radius_min), hp.radius_max);
    p[9 * cap + id] = smin(smax(p[9 * cap + id], hp.aniso_min), hp.aniso_max);
    if (hp.clamp_color) {
        p[4 * cap + id] = smin(smax(p[4 * cap + id], 0.0), 1.0);
        p[5 * cap + id] = smin(smax(p[5 * cap + id], 0.0), 1.0);
        p[6 * cap + id] = smin(smax(p[6 * cap + id], 0.0), 1.0);
    }
    double nx = p[7 * cap + id], ny = p[8 * cap + id];
    double norm = __dsqrt_rn(nx * nx + ny * ny);
    if (!(norm > 1e-12) || !isfinite(norm)) {
        p[7 * cap + id] = 1.0;
        p[8 * cap + id] = 0.0;
    } else {
        p[7 * cap + id] = nx / norm;
        p[8 * cap + id] = ny / norm;
    }
}

// One 16-lane group per site.  The site's gradient records (one per tile that touched it) are
// merged in parallel — lane j takes records j, j+16, ... for all ten channels, then a 16-lane
// butterfly of double-double merges (order independent) leaves every lane with the totals.  Lane
// k < 10 then applies the Adam update of parameter k and its clamp; dir is renormalised from both
// lanes' values exchanged by shuffle; lanes 0-4 rebuild the site's candidate snapshot and backward
// table.  With the adaptive record layout, lane 0 also plans the next pass's record capacity.
#ifndef SAD_ADAM_TWO
#define SAD_ADAM_TWO 0
#endif
// The ten channel totals of site `id`, merged by its 16-lane group (shared by k_adam and
// k_site_totals so both see bit-identical values).  Lanes first sum disjoint record subsets for all
// channels, then a reduce-scatter (10 -> 5 -> 4 -> 2 -> 1 channels per lane; exact double-double
// merges, so the grouping does not matter) leaves lane l with the total of channel
// lane_channel(l) = 5 * bit3(l) + (l & 7) when (l & 7) < 5, else none (-1).  Returns the claimed
// record count.
__device__ __forceinline__ int lane_channel(int lane16) {
    const int loc = lane16 & 7;
    return loc < 5 ? 5 * ((lane16 >> 3) & 1) + loc : -1;
}
__device__ __forceinline__ int channel_lane(int ch) { return ch < 5 ? ch : ch + 3; }

__device__ __forceinline__ DD shfl_xor_dd(unsigned mask, const DD& v, int d) {
    return DD{__shfl_xor_sync(mask, v.hi, d, 16), __shfl_xor_sync(mask, v.lo, d, 16)};
}

__device__ __forceinline__ int merge_site(const RedTarget& grads, int id, bool live, int lane16, unsigned gmask,
                                          int cap, DD& mine) {
    DD acc[10];
#pragma unroll
    for (int ch = 0; ch < 10; ch++) acc[ch] = DD{0.0, 0.0};
    int claimed = 0;
    if (live) {
        claimed = grads.cnt[id];
        int n, base;
        if (grads.roff) {
            n = claimed < grads.rcap[id] ? claimed : grads.rcap[id];
            base = grads.roff[id];
        } else {
            n = claimed < grads.maxt ? claimed : grads.maxt;
            base = id * grads.maxt;
        }
        if (grads.roff && static_cast<long long>(base) + n > grads.psize)
            n = static_cast<int>(grads.psize - base > 0 ? grads.psize - base : 0);
#if SAD_ADAM_TWO
        for (int j = lane16; j < n; j += 32) {  // two records in flight per lane
            const bool two = j + 16 < n;
            const double2* r0 = grads.part + (static_cast<size_t>(base) + j) * grads.stride;
            const double2* r1 = grads.part + (static_cast<size_t>(base) + (two ? j + 16 : j)) * grads.stride;
            double2 a[10], b[10];
#pragma unroll
            for (int ch = 0; ch < 10; ch++) {
                a[ch] = r0[ch];
                b[ch] = r1[ch];
            }
#pragma unroll
            for (int ch = 0; ch < 10; ch++) {
                dd_merge(acc[ch], DD{a[ch].x, a[ch].y});
                if (two) dd_merge(acc[ch], DD{b[ch].x, b[ch].y});
            }
        }
#else
        for (int j = lane16; j < n; j += 16) {  // one record per lane and step: most sites have <= 16
            const double2* r0 = grads.part + (static_cast<size_t>(base) + j) * grads.stride;
            double2 a[10];
#pragma unroll
            for (int ch = 0; ch < 10; ch++) a[ch] = r0[ch];
#pragma unroll
            for (int ch = 0; ch < 10; ch++) dd_merge(acc[ch], DD{a[ch].x, a[ch].y});
        }
#endif
        if (lane16 == 0)
            for (int r = grads.head[id]; r >= 0; r = grads.onext[r]) {
#pragma unroll
                for (int ch = 0; ch < 10; ch++) {
                    double2 o = grads.opart[static_cast<size_t>(r) * grads.stride + ch];
                    dd_merge(acc[ch], DD{o.x, o.y});
                }
            }
        if (lane16 < 10) {
            double2 o = grads.over[static_cast<size_t>(lane16) * cap + id];  // CAS-fallback totals
            DD mine{o.x, o.y};
#pragma unroll
            for (int ch = 0; ch < 10; ch++)
                if (ch == lane16) dd_merge(acc[ch], mine);
        }
    }
    const bool b3 = lane16 & 8, b2 = lane16 & 4, b1 = lane16 & 2, b0 = lane16 & 1;
    const DD z{0.0, 0.0};
    DD a5[5];  // channel 5*b3 + j
#pragma unroll
    for (int j = 0; j < 5; j++) {
        DD keep = b3 ? acc[5 + j] : acc[j];
        const DD o = shfl_xor_dd(gmask, b3 ? acc[j] : acc[5 + j], 8);
        dd_merge(keep, o);
        a5[j] = keep;
    }
    DD a4[4];  // channel 5*b3 + 4*b2 + j (local index 4*b2 + j < 5)
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const DD hi_part = j + 4 < 5 ? a5[j + 4 < 5 ? j + 4 : 0] : z;
        DD keep = b2 ? hi_part : a5[j];
        const DD o = shfl_xor_dd(gmask, b2 ? a5[j] : hi_part, 4);
        dd_merge(keep, o);
        a4[j] = keep;
    }
    DD a2[2];  // channel 5*b3 + 4*b2 + 2*b1 + j
#pragma unroll
    for (int j = 0; j < 2; j++) {
        DD keep = b1 ? a4[2 + j] : a4[j];
        const DD o = shfl_xor_dd(gmask, b1 ? a4[j] : a4[2 + j], 2);
        dd_merge(keep, o);
        a2[j] = keep;
    }
    mine = b0 ? a2[1] : a2[0];
    dd_merge(mine, shfl_xor_dd(gmask, b0 ? a2[0] : a2[1], 1));
    return claimed;
}

// Gradient values (Accum::value) of every site and channel into tot[ch * cap + id], plus a copy of the
// logtau column in g0 — the inputs of tau_diffusion inside the fit.
__global__ void __launch_bounds__(128) k_site_totals(RedTarget grads, const DevState* __restrict__ st, int cap,
                                                     double* __restrict__ tot, double* __restrict__ g0) {
    const int lane16 = threadIdx.x & 15;
    const int id = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const unsigned gmask = 0xffffu << (threadIdx.x & 16);
    const bool live = id < st->n_sites;
    DD g;
    merge_site(grads, id, live, lane16, gmask, cap, g);
    const int ch = lane_channel(lane16);
    if (!live || ch < 0) return;
    tot[static_cast<size_t>(ch) * cap + id] = g.hi + g.lo;
    if (ch == 2) g0[id] = g.hi + g.lo;
}

void launch_site_totals(const RedTarget& grads, const DevState* st, int cap, double* tot, double* g0,
                        cudaStream_t stream) {
    int grid = (cap + 7) / 8;
    if (grid < 1) grid = 1;
    k_site_totals<<<grid, 128, 0, stream>>>(grads, st, cap, tot, g0);
    SAD_LAUNCHED();
}

// Row-strip fits: each rank's per-site double-double totals of its own records (all ten channels,
// same merge code as Adam), and the rank-ordered merge of the gathered partials.  Every sum is an
// exact double-double, so the merged totals equal the single-GPU ones bit for bit.
__global__ void __launch_bounds__(128) k_site_partials(RedTarget grads, const DevState* __restrict__ st, int cap,
                                                       double2* __restrict__ out) {
    const int lane16 = threadIdx.x & 15;
    const int id = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const unsigned gmask = 0xffffu << (threadIdx.x & 16);
    const bool live = id < st->n_sites;
    DD g;
    merge_site(grads, id, live, lane16, gmask, cap, g);
    const int ch = lane_channel(lane16);
    if (id < cap && ch >= 0) out[static_cast<size_t>(ch) * cap + id] = live ? make_double2(g.hi, g.lo) : make_double2(0, 0);
}

void launch_site_partials(const RedTarget& grads, const DevState* st, int cap, double2* out, cudaStream_t stream) {
    int grid = (cap + 7) / 8;
    k_site_partials<<<grid ? grid : 1, 128, 0, stream>>>(grads, st, cap, out);
    SAD_LAUNCHED();
}

// parts: world slices of [nch][cap] double2; writes values (hi + lo) and/or the merged double-doubles
__global__ void k_merge_partials(const double2* __restrict__ parts, int world, int cap, int nch,
                                 double* __restrict__ values, double2* __restrict__ dd) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const size_t n = static_cast<size_t>(nch) * cap;
    if (i >= n) return;
    DD t{0.0, 0.0};
    for (int r = 0; r < world; r++) {
        const double2 v = parts[static_cast<size_t>(r) * n + i];
        dd_merge(t, DD{v.x, v.y});
    }
    if (values) values[i] = t.hi + t.lo;
    if (dd) dd[i] = make_double2(t.hi, t.lo);
}

void launch_merge_partials(const double2* parts, int world, int cap, int nch, double* values, double2* dd,
                           cudaStream_t stream) {
    const size_t n = static_cast<size_t>(nch) * cap;
    k_merge_partials<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(parts, world, cap, nch, values, dd);
    SAD_LAUNCHED();
}

// ---------------------------------------------------------------------- owner-merged row-strip exchange
// Site ownership by id slice: rank q owns ids [q * slice, (q + 1) * slice).  Each rank sends the partial
// totals of the sites it touched (cnt > 0) that another rank owns, as (id, nch double-doubles) records
// grouped by owner; the owner merges them exactly into its own partials (128-bit CAS: several sources may
// add to one site).  The reduction state of every touched site is reset for the next pass here, and (for
// gradients) the next pass's record capacities are planned from this rank's counts, as k_adam does.
__global__ void k_owner_pack(const double2* __restrict__ part, int nch, RedTarget red, const DevState* __restrict__ st,
                             const uint8_t* __restrict__ active, int slice, int me, int world, OwnRec* __restrict__ send,
                             int send_cap, unsigned long long* __restrict__ counts, int32_t* __restrict__ rcap_next,
                             int reset) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= red.cap) return;
    if (id >= st->n_sites) {  // unused slots claim no record space in the next pass's layout
        if (rcap_next) rcap_next[id] = 0;
        return;
    }
    const int cl = red.cnt[id];
    if (rcap_next) {
        int want = active[id] ? cl + (cl >> 2) + 2 : 0;
        rcap_next[id] = want < 4096 ? want : 4096;
    }
    // touched: records claimed this pass (gradients), or (finalized stats, whose counts are already
    // reset) any non-zero partial — an all-zero partial adds nothing to the owner's total
    bool touched = cl > 0;
    if (!rcap_next && !touched)
        for (int c = 0; c < nch && !touched; c++) {
            const double2 v = part[static_cast<size_t>(c) * red.cap + id];
            touched = v.x != 0.0 || v.y != 0.0;
        }
    if (touched) {
        const int q = id / slice;
        if (q != me && q < world) {
            const int pos = static_cast<int>(atomicAdd(counts + q, 1ull));
            if (pos < send_cap) {
                OwnRec& r = send[static_cast<size_t>(q) * send_cap + pos];
                r.id = static_cast<uint32_t>(id);
                for (int c = 0; c < nch; c++) r.v[c] = part[static_cast<size_t>(c) * red.cap + id];
            }
        }
    }
    if (reset) {
        for (int c = 0; c < red.stride; c++) red.over[static_cast<size_t>(c) * red.cap + id] = make_double2(0.0, 0.0);
        red.cnt[id] = 0;
        red.head[id] = -1;
    }
}

void launch_owner_pack(const double2* part, int nch, const RedTarget& red, const DevState* st, const uint8_t* active,
                       int slice, int me, int world, OwnRec* send, int send_cap, unsigned long long* counts,
                       int32_t* rcap_next, bool reset, cudaStream_t stream) {
    const int grid = (red.cap + 255) / 256;
    k_owner_pack<<<grid ? grid : 1, 256, 0, stream>>>(part, nch, red, st, active, slice, me, world, send, send_cap, counts,
                                                      rcap_next, reset ? 1 : 0);
    SAD_LAUNCHED();
}

__global__ void k_owner_merge(const OwnRec* __restrict__ recv, long long n, int nch, int cap, double2* __restrict__ part) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n * nch) return;
    const long long r = i / nch;
    const int c = static_cast<int>(i - r * nch);
    const OwnRec& rec = recv[r];
    SAD_CHECK(rec.id < static_cast<uint32_t>(cap));
    const double2 v = rec.v[c];
    if (v.x != 0.0 || v.y != 0.0) dd_atomic_merge(part + static_cast<size_t>(c) * cap + rec.id, DD{v.x, v.y});
}

void launch_owner_merge(const OwnRec* recv, long long n, int nch, int cap, double2* part, cudaStream_t stream) {
    if (n <= 0) return;
    const long long items = n * nch;
    k_owner_merge<<<static_cast<unsigned>((items + 255) / 256), 256, 0, stream>>>(recv, n, nch, cap, part);
    SAD_LAUNCHED();
}

// ---------------------------------------------------------------------- ordered (fp64) strip exchange
// The records of one site on this rank: its slice [0, n_slice) and its overflow list.
template <typename F>
__device__ __forceinline__ void for_site_records(const RedTarget& red, int id, F&& fn) {
    long long base = 0;
    const int n_slice = ord_slice(red, id, base);
    for (int j = 0; j < n_slice; j++)
        fn(red.part + static_cast<size_t>(base + j) * red.stride, red.tag[base + j]);
    for (int r = red.head[id]; r >= 0; r = red.onext[r]) fn(red.opart + static_cast<size_t>(r) * red.stride, red.otag[r]);
}

__global__ void k_owner_count_ord(RedTarget red, const DevState* __restrict__ st, int slice, int me, int world,
                                  unsigned long long* __restrict__ counts) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= st->n_sites || red.cnt[id] <= 0) return;
    const int q = id / slice;
    if (q == me || q >= world) return;
    unsigned long long n = 0;
    for_site_records(red, id, [&](const double2*, uint32_t) { n++; });
    atomicAdd(counts + q, n);
}

__global__ void k_owner_pack_ord(RedTarget red, const DevState* __restrict__ st, int slice, int me, int world,
                                 OwnRec* __restrict__ send, long long send_cap, unsigned long long* __restrict__ cursors) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= st->n_sites || red.cnt[id] <= 0) return;
    const int q = id / slice;
    if (q == me || q >= world) return;
    unsigned long long n = 0;
    for_site_records(red, id, [&](const double2*, uint32_t) { n++; });
    long long pos = static_cast<long long>(atomicAdd(cursors + q, n));
    for_site_records(red, id, [&](const double2* v, uint32_t tag) {
        SAD_CHECK(pos < send_cap);
        OwnRec& r = send[static_cast<size_t>(q) * send_cap + pos++];
        r.id = static_cast<uint32_t>(id);
        r.pad[0] = tag;
        for (int c = 0; c < 10; c++) r.v[c] = v[c];
    });
}

__global__ void k_owner_merge_ord(const OwnRec* __restrict__ recv, long long n, RedTarget red, DevState* st) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const OwnRec& rec = recv[i];
    SAD_CHECK(rec.id < static_cast<uint32_t>(red.cap));
    const int ro = atomicAdd(red.otop, 1);
    if (ro < red.ocap) {
        for (int c = 0; c < 10; c++) red.opart[static_cast<size_t>(ro) * red.stride + c] = rec.v[c];
        red.otag[ro] = rec.pad[0];
        red.onext[ro] = atomicExch(red.head + rec.id, ro);
    } else {
        atomicOr(&st->err, 8);
        for (int c = 0; c < 10; c++)
            dd_atomic_merge(red.over + static_cast<size_t>(c) * red.cap + rec.id, DD{rec.v[c].x, rec.v[c].y});
    }
}

__global__ void k_ord_finish(RedTarget red, const DevState* __restrict__ st, const uint8_t* __restrict__ active,
                             int32_t* __restrict__ rcap_next) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= red.cap) return;
    if (id >= st->n_sites) {
        rcap_next[id] = 0;
        return;
    }
    const int cl = red.cnt[id];
    const int want = active[id] ? cl + (cl >> 2) + 2 : 0;
    rcap_next[id] = want < 4096 ? want : 4096;
    for (int c = 0; c < red.stride; c++) red.over[static_cast<size_t>(c) * red.cap + id] = make_double2(0.0, 0.0);
    red.cnt[id] = 0;
    red.head[id] = -1;
}

void launch_owner_count_ord(const RedTarget& red, const DevState* st, int slice, int me, int world,
                            unsigned long long* counts, cudaStream_t stream) {
    const int grid = (red.cap + 255) / 256;
    k_owner_count_ord<<<grid ? grid : 1, 256, 0, stream>>>(red, st, slice, me, world, counts);
    SAD_LAUNCHED();
}
void launch_owner_pack_ord(const RedTarget& red, const DevState* st, int slice, int me, int world, OwnRec* send,
                           long long send_cap, unsigned long long* cursors, cudaStream_t stream) {
    const int grid = (red.cap + 255) / 256;
    k_owner_pack_ord<<<grid ? grid : 1, 256, 0, stream>>>(red, st, slice, me, world, send, send_cap, cursors);
    SAD_LAUNCHED();
}
void launch_owner_merge_ord(const OwnRec* recv, long long n, const RedTarget& red, DevState* st, cudaStream_t stream) {
    if (n <= 0) return;
    k_owner_merge_ord<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(recv, n, red, st);
    SAD_LAUNCHED();
}
void launch_ord_finish(const RedTarget& red, const DevState* st, const uint8_t* active, int32_t* rcap_next,
                       cudaStream_t stream) {
    const int grid = (red.cap + 255) / 256;
    k_ord_finish<<<grid ? grid : 1, 256, 0, stream>>>(red, st, active, rcap_next);
    SAD_LAUNCHED();
}

// Slice staging for the all-gathers: buf[c][i] = src[c][lo + i] (i < slice; zero past cap) and the inverse
// over every rank's slice of the gathered buffer.
template <typename T>
__global__ void k_slice_pack(const T* __restrict__ src, int nch, int cap, int lo, int slice, T* __restrict__ buf) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(nch) * slice) return;
    const int c = static_cast<int>(i / slice), j = static_cast<int>(i - static_cast<long long>(c) * slice);
    buf[i] = lo + j < cap ? src[static_cast<size_t>(c) * cap + lo + j] : T{};
}

template <typename T>
__global__ void k_slice_unpack(const T* __restrict__ all, int nch, int cap, int slice, int world, T* __restrict__ dst) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long per = static_cast<long long>(nch) * slice;
    if (i >= per * world) return;
    const int q = static_cast<int>(i / per);
    const long long rem = i - q * per;
    const int c = static_cast<int>(rem / slice), j = static_cast<int>(rem - static_cast<long long>(c) * slice);
    const int id = q * slice + j;
    if (id < cap) dst[static_cast<size_t>(c) * cap + id] = all[i];
}

template <typename T>
void launch_slice_pack(const T* src, int nch, int cap, int lo, int slice, T* buf, cudaStream_t stream) {
    const long long n = static_cast<long long>(nch) * slice;
    k_slice_pack<T><<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(src, nch, cap, lo, slice, buf);
    SAD_LAUNCHED();
}
template <typename T>
void launch_slice_unpack(const T* all, int nch, int cap, int slice, int world, T* dst, cudaStream_t stream) {
    const long long n = static_cast<long long>(nch) * slice * world;
    k_slice_unpack<T><<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(all, nch, cap, slice, world, dst);
    SAD_LAUNCHED();
}
template void launch_slice_pack<double>(const double*, int, int, int, int, double*, cudaStream_t);
template void launch_slice_pack<double2>(const double2*, int, int, int, int, double2*, cudaStream_t);
template void launch_slice_unpack<double>(const double*, int, int, int, int, double*, cudaStream_t);
template void launch_slice_unpack<double2>(const double2*, int, int, int, int, double2*, cudaStream_t);

// The owned range [a0, a1) of the ascending active list (ids in [lo, hi)) and the owned totals' values.
__global__ void k_owned_range(const uint32_t* __restrict__ act, const DevState* __restrict__ st, int lo, int hi,
                              int32_t* __restrict__ range) {
    const int n = st->n_active;
    auto lower = [&](int v) {
        int a = 0, b = n;
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (static_cast<int>(act[mid]) < v) a = mid + 1;
            else b = mid;
        }
        return a;
    };
    range[0] = lower(lo);
    range[1] = lower(hi);
}

void launch_owned_range(const uint32_t* act, const DevState* st, int lo, int hi, int32_t* range, cudaStream_t stream) {
    k_owned_range<<<1, 1, 0, stream>>>(act, st, lo, hi, range);
    SAD_LAUNCHED();
}

__global__ void k_dd_values(const double2* __restrict__ dd, long long n, double* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = dd[i].x + dd[i].y;
}

void launch_dd_values(const double2* dd, long long n, double* out, cudaStream_t stream) {
    if (n <= 0) return;
    k_dd_values<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(dd, n, out);
    SAD_LAUNCHED();
}

// The loss of one backward call: the exact (double-double) sum of its per-block partials, always in
// the order of a 1024-thread block (virtual thread j merges partials j, j + 1024, ...; a shuffle tree
// per virtual warp, then one over the 32 warp sums) whatever the block size (1024 / V threads, each
// warp playing V virtual warps with independent accumulators so their loads overlap), so k_advance
// and k_adam's bookkeeping block produce the same bits.  Result in thread 0; parts: shared [32].
template <int V>
__device__ DD loss_total(const double2* __restrict__ part, int n, DD* parts) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = 32 / V;
    DD acc[V];
#pragma unroll
    for (int v = 0; v < V; v++) acc[v] = DD{0.0, 0.0};
    for (int base = lane; base < n; base += 1024) {
#pragma unroll
        for (int v = 0; v < V; v++) {
            const int i = base + (warp + v * nw) * 32;
            if (i < n) dd_merge(acc[v], DD{part[i].x, part[i].y});
        }
    }
#pragma unroll
    for (int v = 0; v < V; v++) {
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            DD o{__shfl_down_sync(0xffffffffu, acc[v].hi, d), __shfl_down_sync(0xffffffffu, acc[v].lo, d)};
            dd_merge(acc[v], o);
        }
        if (lane == 0) parts[warp + v * nw] = acc[v];
    }
    __syncthreads();
    DD t{0.0, 0.0};
    if (threadIdx.x < 32) {
        t = parts[threadIdx.x];
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            DD o{__shfl_down_sync(0xffffffffu, t.hi, d), __shfl_down_sync(0xffffffffu, t.lo, d)};
            dd_merge(t, o);
        }
    }
    return t;
}

// k_adam with AdvanceArgs: every Adam block reads t before it finishes; the last of the n to
// finish advances t and resets the record pool top its blocks claimed from.
__device__ __forceinline__ void adam_ticket(DevState* st, int32_t* otop, unsigned n) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (static_cast<unsigned>(atomicAdd(&st->ticket, 1)) == n - 1) {
            __threadfence();
            st->t += 1;
            otop[2] = 0;
            st->ticket = 0;
        }
    }
}

#ifndef SAD_ADAM_MINB
#define SAD_ADAM_MINB 5  // resident 128-thread blocks per SM the register allocator must allow: config-2 fit
                         // 1: 862.7, 4: 854 (r1), 4 -> 5: 851 -> 846.5 ms (96 regs; the ~5k active sites' blocks
                         // fit one wave), 6: 866 ms (spills)
#endif
template <typename T>
__global__ void __launch_bounds__(128, SAD_ADAM_MINB) k_adam(SitesDev s, DevState* st, RedTarget grads, double* __restrict__ m,
                                              double* __restrict__ v, AdamHyper hp,
                                              const double2* __restrict__ bc_table, double2 bc_now, int zero_grads,
                                              double scale, Q4<T>* pack, Q4<T>* gtab, int32_t* rcap_next,
                                              const double* __restrict__ totals, int32_t* roff_next,
                                              int32_t* pool_top, const uint32_t* __restrict__ act,
                                              const int32_t* __restrict__ act_range, AdvanceArgs adv) {
    pdl_enter<4>();
    __shared__ int32_t s_want[8], s_base;
    const bool book = adv.loss_hist != nullptr;
    if (book && blockIdx.x == 0) {
        // the bookkeeping block, dispatched first so its serial reduction overlaps the Adam blocks:
        // k_advance's work except t and the record pool top, which the Adam blocks still read or claim
        // from (adam_ticket does those)
        __shared__ DD parts[32];
        const DD loss = loss_total<8>(adv.loss_part, adv.n_part, parts);  // 128 threads
        if (threadIdx.x == 0) {
            const int it = st->iter;
            adv.loss_hist[it] = make_double2(loss.hi, loss.lo);
            if (adv.active_hist) adv.active_hist[it] = st->n_active;
            st->iter = it + 1;
            st->pass_index += static_cast<uint32_t>(adv.passes);
            adv.otop[0] = 0;  // gradient overflow pool (read through the head/onext lists only)
        }
        return;
    }
    const int lane16 = threadIdx.x & 15;
    const int bid = static_cast<int>(blockIdx.x) - (book ? 1 : 0);
    const int grp = (bid * static_cast<int>(blockDim.x) + static_cast<int>(threadIdx.x)) >> 4;
    const unsigned gmask = 0xffffu << (threadIdx.x & 16);
    const int cap = s.cap;
    // with `act` (plain iterations) the groups walk the ascending active list: inactive sites have no
    // records, no update and keep their tables, so skipping them is exact
    // active-list mode: blocks whose 8 groups all lie past the active count have nothing to do (the grid
    // is sized by the capacity because it is captured in a CUDA graph); block-uniform, before any barrier
    // act_range (row-strip fits): only the owned slice act[a0, a1) of the active list
    const int a0 = act_range ? act_range[0] : 0;
    const int n_act = act_range ? act_range[1] - act_range[0] : (act ? st->n_active : 0);
    // blocks that read t and take the ticket: the ones with work (at least one)
    const unsigned n_ticket = act ? static_cast<unsigned>(n_act > 0 ? (n_act + 7) / 8 : 1) : gridDim.x - 1;
    if (act && bid * 8 >= n_act) {
        if (book && bid == 0) adam_ticket(st, adv.otop, n_ticket);
        return;
    }
    const bool live = act ? grp < n_act : grp < st->n_sites;
    const int id = act ? (live ? static_cast<int>(act[a0 + grp]) : cap) : grp;
    const int k = lane16;
    unsigned long long skipped = 0;
    const int kc = lane_channel(lane16);  // the parameter this lane updates (-1: none)
    // the site's parameter, moments and flags do not depend on the gradient: their loads are issued
    // before the record merge so their latency overlaps it
    bool upd = false, is_active = false;
    double p = 0.0, m0 = 0.0, v0 = 0.0;
    double2 bc = bc_now;
    if (live) {
        is_active = s.active[id] != 0;
        upd = is_active && !s.frozen[id];
        if (kc >= 0) {
            const size_t mi = static_cast<size_t>(kc) * cap + id;
            p = s.p[mi];
            m0 = m[mi];
            v0 = v[mi];
        }
        if (bc_table) bc = bc_table[st->t + 1];
    }
    // ---- gradient totals (all lanes of the group take part in the shuffles)
    DD g;
    const int claimed = merge_site(grads, id, live && !totals, lane16, gmask, cap, g);
    if (live) {
        if (upd && kc >= 0) {
            const int k = kc;
            double gv = totals ? totals[static_cast<size_t>(k) * cap + id] : g.hi + g.lo;
            if (!isfinite(gv)) {
                skipped++;
            } else {
                const size_t mi = static_cast<size_t>(k) * cap + id;
                double mm = hp.beta1 * m0 + (1.0 - hp.beta1) * gv;
                double vv = hp.beta2 * v0 + (1.0 - hp.beta2) * gv * gv;
                m[mi] = mm;
                v[mi] = vv;
                p -= hp.lr[k] * (mm / bc.x) / (__dsqrt_rn(vv / bc.y) + hp.eps);
            }
            // clamp_project (train.cpp:113-137)
            switch (k) {
            case 0: p = smin(smax(p, 0.0), hp.width - 1.0); break;
            case 1: p = smin(smax(p, 0.0), hp.height - 1.0); break;
            case 2: p = smin(smax(p, hp.log_tau_min), hp.log_tau_max); break;
            case 3: p = smin(smax(p, hp.radius_min), hp.radius_max); break;
            case 4:
            case 5:
            case 6:
                if (hp.clamp_color) p = smin(smax(p, 0.0), 1.0);
                break;
            case 9: p = smin(smax(p, hp.aniso_min), hp.aniso_max); break;
            default: break;
            }
        }
        const double nx = __shfl_sync(gmask, p, (threadIdx.x & 16) + channel_lane(7));
        const double ny = __shfl_sync(gmask, p, (threadIdx.x & 16) + channel_lane(8));
        if (upd && (kc == 7 || kc == 8)) {
            double norm = __dsqrt_rn(nx * nx + ny * ny);
            if (!(norm > 1e-12) || !isfinite(norm)) p = kc == 7 ? 1.0 : 0.0;
            else p = (kc == 7 ? nx : ny) / norm;
        }
        if (upd && kc >= 0) s.p[static_cast<size_t>(kc) * cap + id] = p;
        // this pass's record count (with precomputed totals, merge_site did not read it): before the reset
        const int cl = totals ? grads.cnt[id] : claimed;
        if (zero_grads) {
            if (k < 11) grads.over[static_cast<size_t>(k) * cap + id] = make_double2(0.0, 0.0);
            if (k == 0) grads.cnt[id] = 0;
            if (k == 1) grads.head[id] = -1;
        }
        if (rcap_next && k == 0) {
            // next pass's record capacity: last count plus headroom (active sites only)
            int want = is_active ? cl + (cl >> 2) + 2 : 0;
            want = want < 4096 ? want : 4096;
            rcap_next[id] = want;
            if (roff_next) s_want[threadIdx.x >> 4] = want;
        }
    } else {
        __shfl_sync(gmask, 0.0, (threadIdx.x & 16) + channel_lane(7));
        __shfl_sync(gmask, 0.0, (threadIdx.x & 16) + channel_lane(8));
        if (rcap_next && k == 0 && id < cap) rcap_next[id] = 0;  // (act: id == cap, nothing written)
        if (rcap_next && k == 0) s_want[threadIdx.x >> 4] = 0;
    }
    // record slices for the next pass: a block-wide prefix of the 8 capacities and one pool claim per
    // block (the layout is order dependent, the merged totals are not)
    if (rcap_next && roff_next) {
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int g = 0; g < 8; g++) {
                const int w = s_want[g];
                s_want[g] = tot;
                tot += w;
            }
            s_base = atomicAdd(pool_top, tot);
        }
        __syncthreads();
        if (k == 0 && id < cap) roff_next[id] = s_base + s_want[threadIdx.x >> 4];
    }
    if (skipped) atomicAdd(reinterpret_cast<unsigned long long*>(&st->skipped), skipped);
    // the site's final parameters (each lane kc holds channel kc, updated or as loaded) to the table lanes
    double q[10];
#pragma unroll
    for (int c = 0; c < 10; c++) q[c] = __shfl_sync(gmask, p, (threadIdx.x & 16) + channel_lane(c));
    if (live && lane16 < 5 && (pack || gtab)) {
        // same derivations as k_tables (score_table.hpp:20-46, grad.cpp:84-110), one output quad per lane
        const bool act = is_active;
        const double x = q[0], y = q[1], lt = q[2], r = q[3];
        const double ux = q[7], uy = q[8], an = q[9];
        if (lane16 == 0 && pack) {
            Q4<T> a{T(0), T(0), T(0), T(0)};
            if (act) a = {static_cast<T>(half_rt(x)), static_cast<T>(half_rt(y)), static_cast<T>(sad_dexp(half_rt(lt))),
                          static_cast<T>(half_rt(r))};
            pack[2 * id] = a;
        } else if (lane16 == 1 && pack) {
            Q4<T> b{T(1), T(0), T(1), T(0)};
            if (act) {
                double hux = half_rt(ux), huy = half_rt(uy), han = half_rt(an);
                double ea = sad_dexp(han), ia = sad_dexp(-han);
                double vx = -huy, vy = hux;
                b = {static_cast<T>(ea * hux * hux + ia * vx * vx), static_cast<T>(ea * hux * huy + ia * vx * vy),
                     static_cast<T>(ea * huy * huy + ia * vy * vy), T(1)};
            }
            pack[2 * id + 1] = b;
        } else if (lane16 == 2 && gtab) {
            Q4<T> a{T(0), T(0), T(0), T(0)};
            if (act) a = {static_cast<T>(x), static_cast<T>(y), static_cast<T>(sad_dexp(lt)), static_cast<T>(r)};
            gtab[3 * id] = a;
        } else if (lane16 == 3 && gtab) {
            Q4<T> b{T(1), T(1), T(1), T(0)};
            if (act) b = {static_cast<T>(sad_dexp(an)), static_cast<T>(sad_dexp(-an)), static_cast<T>(ux), static_cast<T>(uy)};
            gtab[3 * id + 1] = b;
        } else if (lane16 == 4 && gtab) {
            Q4<T> c{T(0), T(0), T(0), T(0)};
            if (act) c = {static_cast<T>(q[4]), static_cast<T>(q[5]), static_cast<T>(q[6]), T(1)};
            gtab[3 * id + 2] = c;
        }
    }
    if (book) adam_ticket(st, adv.otop, n_ticket);
}

void launch_adam(bool fp64, const SitesDev& s, DevState* st, const RedTarget& grads, double* m, double* v,
                 const AdamHyper& hp, const double2* bc_table, double2 bc_now, bool zero_grads, double scale,
                 void* pack, void* gtab, int32_t* rcap_next, cudaStream_t stream, const double* totals,
                 int32_t* roff_next, int32_t* pool_top, const uint32_t* act, const int32_t* act_range,
                 const AdvanceArgs& adv) {
    int grid = (s.cap + 7) / 8;  // 8 sites (16 lanes each) per 128-thread block
    if (grid < 1) grid = 1;
    if (adv.loss_hist) grid += 1;  // + the bookkeeping block
    if (fp64)
        launch_pdl(k_adam<double>, dim3(grid), dim3(128), 0, stream, s, st, grads, m, v, hp, bc_table, bc_now,
                   zero_grads ? 1 : 0, scale, (Q4<double>*)pack, (Q4<double>*)gtab, rcap_next, totals, roff_next, pool_top,
                   act, act_range, adv);
    else
        launch_pdl(k_adam<float>, dim3(grid), dim3(128), 0, stream, s, st, grads, m, v, hp, bc_table, bc_now,
                   zero_grads ? 1 : 0, scale, (Q4<float>*)pack, (Q4<float>*)gtab, rcap_next, totals, roff_next, pool_top,
                   act, act_range, adv);
    SAD_LAUNCHED();
}

// ====================================================================== tau_diffusion (train.cpp:171-213)
// Edge keys (owner << nb | id) for every pixel's active candidates (owner from render_id_map); the
// sentinel (all ones in 2·nb bits) marks no edge and sorts last.  nb is chosen so that no valid id
// equals the all-ones id field.
__global__ void k_tau_edges(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ owner,
                            const uint8_t* __restrict__ active, FieldDims f, int nb, uint64_t* __restrict__ keys) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x;
    const int py = blockIdx.y;
    if (px >= f.width) return;
    const size_t pix = static_cast<size_t>(py) * f.width + px;
    const uint64_t sentinel = (nb >= 32) ? ~0ull : ((1ull << (2 * nb)) - 1);
    const uint32_t o = owner[pix];
    const uint32_t* lst = ids + static_cast<size_t>(f.k) * cell_index(f, px, py);
    uint64_t* out = keys + pix * f.k;
    bool end = o == kEmpty;
    for (int i = 0; i < f.k; i++) {
        const uint32_t id = lst[i];
        end = end || id == kEmpty;
        out[i] = (end || !active[id]) ? sentinel : ((static_cast<uint64_t>(o) << nb) | id);
    }
}

void launch_tau_edges(const uint32_t* ids, const uint32_t* owner, const uint8_t* active, const FieldDims& f, int nb,
                      uint64_t* keys, cudaStream_t stream) {
    dim3 grid((f.width + 127) / 128, f.height);
    k_tau_edges<<<grid, 128, 0, stream>>>(ids, owner, active, f, nb, keys);
    SAD_LAUNCHED();
}

// One thread per owner segment of the sorted unique edges: the co-candidate sum runs sequentially in
// ascending id order exactly as the reference loop, then the mixed value goes through a reset Accum
// (Accum::add on {0, 0}, accum.hpp) into out[owner].
__global__ void k_tau_mix(const uint64_t* __restrict__ uniq, const int* __restrict__ count, int nb,
                          const double* __restrict__ g0, double lambda, double* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = *count;
    if (e >= n) return;
    const uint64_t sentinel = (nb >= 32) ? ~0ull : ((1ull << (2 * nb)) - 1);
    const uint64_t key = uniq[e];
    if (key == sentinel) return;
    const uint64_t o = key >> nb;
    if (e > 0 && (uniq[e - 1] >> nb) == o) return;
    const uint64_t mask = (1ull << nb) - 1;
    double sum = 0.0;
    int cnt = 0;
    for (int j = e; j < n; j++) {
        const uint64_t kj = uniq[j];
        if (kj == sentinel || (kj >> nb) != o) break;
        sum += g0[kj & mask];
        cnt++;
    }
    const double mixed = (1.0 - lambda) * g0[o] + lambda * (sum / cnt);
    const double hi = 0.0 + mixed;
    const double bb = hi - 0.0;
    const double err = (0.0 - (hi - bb)) + (mixed - bb);
    out[o] = hi + (0.0 + err);
}

void launch_tau_mix(const uint64_t* uniq, const int* count, int max_items, int nb, const double* g0, double lambda,
                    double* out, cudaStream_t stream) {
    int grid = (max_items + 255) / 256;
    if (grid < 1) grid = 1;
    k_tau_mix<<<grid, 256, 0, stream>>>(uniq, count, nb, g0, lambda, out);
    SAD_LAUNCHED();
}

// The device libm ports the kernels use, exposed for verification against the host's glibc.
__global__ void k_math(const double* __restrict__ x, double* __restrict__ y, size_t n, int which) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    y[i] = which == 0 ? sad_dexp(x[i])
                      : which == 1 ? static_cast<double>(sad_expf(static_cast<float>(x[i]))) : sad_dlog(x[i]);
}

void launch_math(const double* x, double* y, size_t n, int which, cudaStream_t stream) {
    const unsigned grid = static_cast<unsigned>((n + 255) / 256);
    k_math<<<grid ? grid : 1, 256, 0, stream>>>(x, y, n, which);
    SAD_LAUNCHED();
}

__global__ void k_fill_i32(int32_t* p, int n, int32_t v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// Stats record capacities from this pass's gradient record counts: a site's 8x8 stats tiles are halves of its
// 16x8 backward tiles, so it claims at most twice as many stats records (+2 slack); unused slots claim none.
__global__ void k_stats_plan(const int32_t* __restrict__ gcnt, const DevState* __restrict__ st, int cap,
                             int32_t* __restrict__ rcap) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= cap) return;
    rcap[id] = id < st->n_sites ? 2 * gcnt[id] + 2 : 0;
}

void launch_stats_plan(const int32_t* gcnt, const DevState* st, int cap, int32_t* rcap, cudaStream_t stream) {
    k_stats_plan<<<(cap + 255) / 256, 256, 0, stream>>>(gcnt, st, cap, rcap);
    SAD_LAUNCHED();
}

void launch_fill_i32(int32_t* p, int n, int32_t v, cudaStream_t stream) {
    k_fill_i32<<<(n + 255) / 256, 256, 0, stream>>>(p, n, v);
    SAD_LAUNCHED();
}

__global__ void k_clamp(SitesDev s, const DevState* st, AdamHyper hp) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= st->n_sites || !s.active[id] || s.frozen[id]) return;
    clamp_site(s.p, s.cap, id, hp);
}

void launch_clamp(const SitesDev& s, const DevState* st, const AdamHyper& hp, cudaStream_t stream) {
    int grid = (s.cap + 127) / 128;
    if (grid < 1) grid = 1;
    k_clamp<<<grid, 128, 0, stream>>>(s, st, hp);
    SAD_LAUNCHED();
}

// ====================================================================== prune / densify (budget.cpp:219-305)
// Selection = stable ascending radix sort of order_key() over all slots; ineligible slots get the
// largest key so they sort last, and the stable sort keeps ascending ids within ties (the
// reference's id tie-break).
__global__ void k_prune_keys(SitesDev s, DevState* st, const double2* __restrict__ stats, int cap,
                             unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= cap) return;
    bool elig = id < st->n_sites && s.active[id] && !s.frozen[id];
    double norm = static_cast<double>(st->valid > 1 ? st->valid : 1);
    keys[id] = elig ? order_key(dd_value(stats[7 * static_cast<size_t>(cap) + id]) / norm) : ~0ull;
    vals[id] = static_cast<uint32_t>(id);
    unsigned mask = __ballot_sync(0xffffffffu, elig);
    if ((threadIdx.x & 31) == 0 && mask) atomicAdd(&st->n_elig, __popc(mask));
}

void launch_prune_keys(const SitesDev& s, DevState* st, const double2* stats, int cap, unsigned long long* keys,
                       uint32_t* vals, cudaStream_t stream) {
    k_prune_keys<<<(cap + 255) / 256, 256, 0, stream>>>(s, st, stats, cap, keys, vals);
    SAD_LAUNCHED();
}

__global__ void k_prune_apply(SitesDev s, DevState* st, const uint32_t* __restrict__ sorted, double pct) {
    int want = static_cast<int>(static_cast<double>(st->n_elig) * pct);
    if (pct <= 0) want = 0;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) st->done = want < 1 ? 0 : want;
    if (i >= want) return;
    uint32_t id = sorted[i];
    s.active[id] = 0;
    s.p[0 * s.cap + id] = -1.0;
    s.p[1 * s.cap + id] = -1.0;
}

void launch_prune_apply(const SitesDev& s, DevState* st, const uint32_t* sorted, double pct, cudaStream_t stream) {
    k_prune_apply<<<(s.cap + 255) / 256, 256, 0, stream>>>(s, st, sorted, pct);
    SAD_LAUNCHED();
}

__global__ void k_densify_keys(SitesDev s, DevState* st, const double2* __restrict__ stats, int cap, double alpha,
                               double eps, unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals,
                               uint8_t* __restrict__ free_flags) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= cap) return;
    const bool inside = id < st->n_sites;
    double mass = inside ? dd_value(stats[static_cast<size_t>(id)]) : 0.0;
    bool elig = inside && s.active[id] && !s.frozen[id] && mass > 1.0;
    unsigned long long key = ~0ull;
    if (elig) {
        double energy = dd_value(stats[static_cast<size_t>(cap) + id]);
        double sc = energy / pow(smax(mass, eps), alpha);  // densify_score (budget.cpp:157-159)
        key = order_key(-sc);                              // descending score, ascending id
    }
    keys[id] = key;
    vals[id] = static_cast<uint32_t>(id);
    free_flags[id] = (inside && !s.active[id]) ? 1 : 0;
    unsigned mask = __ballot_sync(0xffffffffu, elig);
    if ((threadIdx.x & 31) == 0 && mask) atomicAdd(&st->n_elig, __popc(mask));
}

void launch_densify_keys(const SitesDev& s, DevState* st, const double2* stats, int cap, double alpha, double eps,
                         unsigned long long* keys, uint32_t* vals, uint8_t* free_flags, cudaStream_t stream) {
    k_densify_keys<<<(cap + 255) / 256, 256, 0, stream>>>(s, st, stats, cap, alpha, eps, keys, vals, free_flags);
    SAD_LAUNCHED();
}

__device__ __forceinline__ double luma_at(const double* img, int w, int h, int x, int y) {
    x = x < 0 ? 0 : (x > w - 1 ? w - 1 : x);
    y = y < 0 ? 0 : (y > h - 1 ? h - 1 : y);
    const double* p = img + 3 * (static_cast<size_t>(y) * w + x);
    return 0.2126 * p[0] + 0.7152 * p[1] + 0.0722 * p[2];
}

// split_axis (budget.cpp:170-215) + the split of densify (budget.cpp:237-279).  Split i uses free
// slot i while they last, then appends in order; parents are active so no two splits touch the same
// slot, which makes the reference's sequential loop embarrassingly parallel.
// The split-axis anisotropy -0.5*log(lam1/lam2) uses sad_dlog, the device port of the host glibc's log
// that the reference calls (budget.cpp:198-199): no host round trip per event.
__global__ void k_densify_apply(SitesDev s, DevState* st, const double2* __restrict__ stats, int cap,
                                const uint32_t* __restrict__ sorted, const uint32_t* __restrict__ free_list,
                                const double* __restrict__ img, double pct, SplitHyper hp, double* m, double* v) {
    const int n_elig = st->n_elig, n_free = st->n_free, size0 = st->n_sites;
    int want = static_cast<int>(static_cast<double>(n_elig) * pct);
    if (pct <= 0 || want < 1) want = 0;
    long long room = hp.max_sites > 0 ? (static_cast<long long>(hp.max_sites) - size0) : (1ll << 40);
    if (room < 0) room = 0;
    long long done = want < static_cast<long long>(n_free) + room ? want : static_cast<long long>(n_free) + room;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= done) return;
    const uint32_t par = sorted[i];
    double st8[8];
#pragma unroll
    for (int c = 0; c < 8; c++) st8[c] = dd_value(stats[static_cast<size_t>(c) * cap + par]);
    double* p = s.p;
    const double px = p[0 * cap + par], py = p[1 * cap + par], plt = p[2 * cap + par], pr = p[3 * cap + par];
    const double pan = p[9 * cap + par];
    double ax = 1, ay = 0, an = 0;
    bool fallback = true;
    if (st8[0] >= 4.0 && st8[1] > 0) {
        double wv = st8[1];
        double mx = st8[2] / wv, my = st8[3] / wv;
        double cxx = st8[4] / wv - mx * mx;
        double cyy = st8[6] / wv - my * my;
        double cxy = st8[5] / wv - mx * my;
        double half = 0.5 * (cxx - cyy);
        double root = __dsqrt_rn(half * half + cxy * cxy);
        double mid = 0.5 * (cxx + cyy);
        double l1 = mid + root, l2 = mid - root;
        if (l1 > 0 && (l2 <= 0 || l1 > 1.05 * l2)) {
            double vx = cxy, vy = l1 - cxx;
            double nn = __dsqrt_rn(vx * vx + vy * vy);
            if (nn < 1e-18 * l1) {
                vx = l1 - cyy;
                vy = cxy;
                nn = __dsqrt_rn(vx * vx + vy * vy);
            }
            if (nn > 0 && isfinite(nn)) {
                ax = vx / nn;
                ay = vy / nn;
                double ratio = l2 > 0 ? l1 / l2 : 1e18;
                // negative a elongates the influence region along the axis (budget.cpp:197-199); the device
                // port of glibc's log is bit-identical to the host's
                an = sclamp(-0.5 * sad_dlog(ratio), hp.aniso_min, hp.aniso_max);
                fallback = false;
            }
        }
    }
    if (fallback) {
        int sx = static_cast<int>(llround(px)), sy = static_cast<int>(llround(py));
        int w = hp.width, h = hp.height;
        double gx = (luma_at(img, w, h, sx + 1, sy - 1) + 2 * luma_at(img, w, h, sx + 1, sy) +
                     luma_at(img, w, h, sx + 1, sy + 1)) -
                    (luma_at(img, w, h, sx - 1, sy - 1) + 2 * luma_at(img, w, h, sx - 1, sy) +
                     luma_at(img, w, h, sx - 1, sy + 1));
        double gy = (luma_at(img, w, h, sx - 1, sy + 1) + 2 * luma_at(img, w, h, sx, sy + 1) +
                     luma_at(img, w, h, sx + 1, sy + 1)) -
                    (luma_at(img, w, h, sx - 1, sy - 1) + 2 * luma_at(img, w, h, sx, sy - 1) +
                     luma_at(img, w, h, sx + 1, sy - 1));
        double nn = __dsqrt_rn(gx * gx + gy * gy);
        if (nn > 1e-12) {
            ax = gx / nn;
            ay = gy / nn;
        }
        an = sclamp(0.8 * pan, hp.aniso_min, hp.aniso_max);
    }
    double mag = sclamp(0.5 * __dsqrt_rn(smax(st8[0], 0.0)), 1.5, 48.0);
    double clt = smax(plt - 0.25, hp.log_tau_min);
    double cr = smax(pr * 0.85, hp.radius_min);
    for (int side = 0; side < 2; side++) {
        double sg = side == 0 ? 1.0 : -1.0;
        double cx = sclamp(px + sg * ax * mag, 0.0, hp.width - 1.0);
        double cy = sclamp(py + sg * ay * mag, 0.0, hp.height - 1.0);
        int ix = static_cast<int>(llround(cx)), iy = static_cast<int>(llround(cy));
        const double* col = img + 3 * (static_cast<size_t>(iy) * hp.width + ix);
        uint32_t slot = side == 0 ? par : (i < n_free ? free_list[i] : static_cast<uint32_t>(size0 + (i - n_free)));
        if (slot >= static_cast<uint32_t>(cap)) {
            atomicOr(&st->err, 2);
            continue;
        }
        p[0 * cap + slot] = cx;
        p[1 * cap + slot] = cy;
        p[2 * cap + slot] = clt;
        p[3 * cap + slot] = cr;
        p[4 * cap + slot] = col[0];
        p[5 * cap + slot] = col[1];
        p[6 * cap + slot] = col[2];
        p[7 * cap + slot] = ax;
        p[8 * cap + slot] = ay;
        p[9 * cap + slot] = an;
        s.active[slot] = 1;
        s.frozen[slot] = 0;
#pragma unroll
        for (int k = 0; k < 10; k++) {
            m[static_cast<size_t>(k) * cap + slot] = 0.0;
            v[static_cast<size_t>(k) * cap + slot] = 0.0;
        }
    }
    if (i == done - 1) {
        st->done = static_cast<int>(done);
        long long grow = done - n_free;
        if (grow > 0) st->n_sites = size0 + static_cast<int>(grow);
    }
}

void launch_densify_apply(const SitesDev& s, DevState* st, const double2* stats, int cap, const uint32_t* sorted,
                          const uint32_t* free_list, const double* tgt, double pct, const SplitHyper& hp, double* m,
                          double* v, cudaStream_t stream) {
    k_densify_apply<<<(cap + 127) / 128, 128, 0, stream>>>(s, st, stats, cap, sorted, free_list, tgt, pct, hp, m, v);
    SAD_LAUNCHED();
}


__global__ void k_flag_active(SitesDev s, const DevState* st, uint8_t* flags) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= s.cap) return;
    flags[id] = (id < st->n_sites && s.active[id]) ? 1 : 0;
}

void launch_flag_active(const SitesDev& s, const DevState* st, uint8_t* flags, cudaStream_t stream) {
    k_flag_active<<<(s.cap + 255) / 256, 256, 0, stream>>>(s, st, flags);
    SAD_LAUNCHED();
}

// ====================================================================== loop bookkeeping
// End-of-iteration bookkeeping: loss = exact (double-double) sum of the per-tile partials, history
// rows, pass index and Adam step.
__global__ void __launch_bounds__(1024) k_advance(DevState* st, int passes, int adam_steps, double2* loss_hist,
                                                  int32_t* active_hist, const double2* __restrict__ loss_part,
                                                  int n_part, int32_t* otop) {
    pdl_enter<8>();
    if (otop && threadIdx.x == 0) {
        otop[0] = 0;  // gradient overflow pool
        otop[2] = 0;  // gradient record pool (claimed by the next k_adam)
    }
    __shared__ DD parts[32];
    const DD acc = loss_total<1>(loss_part, loss_hist ? n_part : 0, parts);
    if (threadIdx.x != 0) return;
    if (loss_hist) {
        loss_hist[st->iter] = make_double2(acc.hi, acc.lo);
        if (active_hist) active_hist[st->iter] = st->n_active;
        st->iter += 1;
    }
    st->pass_index += static_cast<uint32_t>(passes);
    st->t += adam_steps;
}

void launch_advance(DevState* st, int passes, int adam_steps, double2* loss_hist, int32_t* active_hist,
                    const double2* loss_part, int n_part, int32_t* otop, cudaStream_t stream) {
    launch_pdl(k_advance, dim3(1), dim3(1024), 0, stream, st, passes, adam_steps, loss_hist, active_hist, loss_part,
               n_part, otop);
    SAD_LAUNCHED();
}

// ====================================================================== init_sites (train.cpp:33-111), device path
__global__ void k_sobel(const double* __restrict__ img, int w, int h, double* __restrict__ mag) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    double gx = (luma_at(img, w, h, x + 1, y - 1) + 2 * luma_at(img, w, h, x + 1, y) + luma_at(img, w, h, x + 1, y + 1)) -
                (luma_at(img, w, h, x - 1, y - 1) + 2 * luma_at(img, w, h, x - 1, y) + luma_at(img, w, h, x - 1, y + 1));
    double gy = (luma_at(img, w, h, x - 1, y + 1) + 2 * luma_at(img, w, h, x, y + 1) + luma_at(img, w, h, x + 1, y + 1)) -
                (luma_at(img, w, h, x - 1, y - 1) + 2 * luma_at(img, w, h, x, y - 1) + luma_at(img, w, h, x + 1, y - 1));
    mag[static_cast<size_t>(y) * w + x] = __dsqrt_rn(gx * gx + gy * gy);
}

void launch_sobel(const double* tgt, int w, int h, double* mag, cudaStream_t stream) {
    dim3 block(32, 8), grid((w + 31) / 32, (h + 7) / 8);
    k_sobel<<<grid, block, 0, stream>>>(tgt, w, h, mag);
    SAD_LAUNCHED();
}

__global__ void k_dd_sum(const double* __restrict__ x, size_t n, double2* out) {
    __shared__ DD parts[8];
    DD acc{0.0, 0.0};
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dd_add(acc, x[i]);
    block_dd_merge<256>(acc, parts, out);
}

void launch_dd_sum(const double* x, size_t n, double2* out, cudaStream_t stream) {
    k_dd_sum<<<296, 256, 0, stream>>>(x, n, out);
    SAD_LAUNCHED();
}

// Exponential keys log(u)/w from one sequential xorshift stream: thread c owns pixels
// [c*chunk, (c+1)*chunk) and starts from the stream state after c*chunk draws (host-computed
// jump-ahead).  Sorting ascending on order_key(-key) gives (key desc, index asc).
__global__ void k_init_keys(const double* __restrict__ mag, int w, int h, const double2* __restrict__ gsum_dd,
                            double lambda_init, const uint32_t* __restrict__ jump, int chunk,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
    const size_t np = static_cast<size_t>(w) * h;
    const size_t c = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    size_t b = c * chunk;
    if (b >= np) return;
    double gsum = dd_value(*gsum_dd);
    double lambda = gsum <= 0 ? 1.0 : lambda_init;
    double uni = 1.0 / static_cast<double>(np);
    uint32_t rs = jump[c];
    size_t e = b + chunk < np ? b + chunk : np;
    for (size_t i = b; i < e; i++) {
        double wgt = lambda * uni + (gsum > 0 ? (1.0 - lambda) * mag[i] / gsum : 0.0);
        if (wgt < 1e-300) wgt = 1e-300;
        double u = xs_unit(rs);
        if (u < 1e-12) u = 1e-12;
        double key = sad_dlog(u) / wgt;  // glibc log port (train.cpp:81)
        keys[i] = order_key(-key);
        vals[i] = static_cast<uint32_t>(i);
    }
}

void launch_init_keys(const double* mag, int w, int h, const double2* gsum, double lambda, const uint32_t* jump_states,
                      int chunk, unsigned long long* keys, uint32_t* vals, cudaStream_t stream) {
    size_t np = static_cast<size_t>(w) * h;
    size_t threads = (np + chunk - 1) / chunk;
    k_init_keys<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(mag, w, h, gsum, lambda, jump_states, chunk,
                                                                      keys, vals);
    SAD_LAUNCHED();
}

__global__ void k_mark_cells(const uint32_t* __restrict__ sorted_idx, int n, uint8_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[sorted_idx[i]] = 1;
}

void launch_mark_cells(const uint32_t* sorted_idx, int n, uint8_t* flags, cudaStream_t stream) {
    k_mark_cells<<<(n + 255) / 256, 256, 0, stream>>>(sorted_idx, n, flags);
    SAD_LAUNCHED();
}

// Site j takes draws 2j and 2j+1 of stream (seed, 0x1717, 1) (train.cpp:96-110); `jump` holds the
// state after j0 = block*chunk sites' draws, so each thread replays at most 2*chunk steps.
__global__ void k_init_sites(SitesDev s, DevState* st, const uint32_t* __restrict__ cells, int n,
                             const double* __restrict__ img, int w, int h, double r0, double lt0, double an0,
                             const uint32_t* __restrict__ jump, int chunk) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = c * chunk;
    if (b >= n) return;
    uint32_t rs = jump[c];
    const int e = b + chunk < n ? b + chunk : n;
    const int cap = s.cap;
    for (int j = b; j < e; j++) {
        uint32_t cell = cells[j];
        int cx = static_cast<int>(cell % static_cast<uint32_t>(w)), cy = static_cast<int>(cell / static_cast<uint32_t>(w));
        double ox = xs_unit(rs), oy = xs_unit(rs);
        s.p[0 * cap + j] = smin(cx + 0.25 + 0.5 * ox, w - 1.0);
        s.p[1 * cap + j] = smin(cy + 0.25 + 0.5 * oy, h - 1.0);
        s.p[2 * cap + j] = lt0;
        s.p[3 * cap + j] = r0;
        const double* col = img + 3 * (static_cast<size_t>(cy) * w + cx);
        s.p[4 * cap + j] = col[0];
        s.p[5 * cap + j] = col[1];
        s.p[6 * cap + j] = col[2];
        s.p[7 * cap + j] = 1.0;
        s.p[8 * cap + j] = 0.0;
        s.p[9 * cap + j] = an0;
        s.active[j] = 1;
        s.frozen[j] = 0;
    }
    if (c == 0) st->n_sites = n;
}

void launch_init_sites(const SitesDev& s, DevState* st, const uint32_t* cells, int n, const double* tgt, int w, int h,
                       double r0, double log_tau0, double aniso0, const uint32_t* jump_states, int chunk,
                       cudaStream_t stream) {
    int threads = (n + chunk - 1) / chunk;
    k_init_sites<<<(threads + 127) / 128, 128, 0, stream>>>(s, st, cells, n, tgt, w, h, r0, log_tau0, aniso0,
                                                            jump_states, chunk);
    SAD_LAUNCHED();
}

// ====================================================================== misc
__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<float>(in[i]);
}

void launch_f64_to_f32(const double* in, float* out, size_t n, cudaStream_t stream) {
    size_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    k_f64_to_f32<<<(unsigned)blocks, 256, 0, stream>>>(in, out, n);
    SAD_LAUNCHED();
}

__global__ void k_grads_out(const double2* __restrict__ g, int cap, int n, double* __restrict__ out) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n) return;
#pragma unroll
    for (int k = 0; k < 11; k++) out[static_cast<size_t>(id) * 11 + k] = dd_value(g[static_cast<size_t>(k) * cap + id]);
}

void launch_scatter_grads_out(const double2* grads, int cap, int n, double* out, cudaStream_t stream) {
    k_grads_out<<<(n + 255) / 256 + 1, 256, 0, stream>>>(grads, cap, n, out);
    SAD_LAUNCHED();
}

}  // namespace sadk
