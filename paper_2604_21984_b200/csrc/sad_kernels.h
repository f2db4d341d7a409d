// sad_kernels.h — host-visible launch interface of the SAD CUDA kernels (sad_kernels.cu).
//
// Device data layouts:
//   sites   : double p[10][cap] slot-major (x, y, log_tau, radius, R, G, B, dir_x, dir_y, aniso —
//             the GradSlot order of grad.hpp:13-26), u8 active[cap], frozen[cap]
//   field   : u32 ids[(gy*gw+gx)*k + i], two buffers (ping-pong per propagation pass)
//   pack    : per-site candidate snapshot, 2 x Q4<T>  {x, y, tau, r}, {gxx, gxy, gyy, active}
//   gtab    : per-site backward constants, 3 x Q4<T> {x, y, tau, r}, {e^a, e^-a, ux, uy}, {R, G, B, active}
//   rtab    : per-site render constants,   3 x Q4<T> {x, y, tau, r}, {gxx, gxy, gyy, active}, {R, G, B, 0}
//   grads   : double2 g[11][cap]   (hi, lo) compensated accumulators, channel-major
//   stats   : double2 s[8][cap]
//   adam    : double m[10][cap], v[10][cap]
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sadk {

// Per-fit scalars that live in device memory so CUDA graphs can replay iterations unchanged.
struct DevState {
    uint32_t pass_index;  // CandidateField::pass_index
    int32_t n_sites;      // SiteStore::size
    int64_t t;            // AdamState::t
    int32_t iter;         // history row being produced (0-based)
    int32_t n_active;     // |active_ids|
    int32_t n_elig;       // eligible count of the current prune/densify selection
    int32_t n_free;       // inactive slots below n_sites (densify free list)
    int32_t done;         // splits / removals performed by the last event
    int32_t err;          // bit 0: empty candidate list, bit 1: capacity, bit 2: non-finite loss
    uint64_t nonfinite;   // GradBuffer::nonfinite
    uint64_t valid;       // StatsResult::valid_pixels
    uint64_t skipped;     // AdamState::skipped
    double2 loss;         // compensated loss sum of the current backward call
    int32_t ticket;       // k_adam blocks finished (the last one advances t; reset by it)
};

// The end-of-iteration bookkeeping k_advance does, folded into a plain iteration's k_adam (one
// extra block): history row, iter, pass_index and the overflow pool top; the last Adam block to
// finish advances t and resets the record pool top.  loss_hist == nullptr: none.
struct AdvanceArgs {
    double2* loss_hist = nullptr;
    int32_t* active_hist = nullptr;
    const double2* loss_part = nullptr;
    int n_part = 0;
    int passes = 0;
    int32_t* otop = nullptr;
};

struct SitesDev {
    double* p;  // 10 * cap
    uint8_t* active;
    uint8_t* frozen;
    int cap;
};

// Destination of a tile reduction (grad.cpp:37-64 semantics): each tile that touches a site claims
// one record slot for it with a single atomicAdd and stores its compensated per-channel partials
// there; the consumer merges the records in any order (double-double is order independent).  A
// site that collects more than `maxt` tiles in one pass falls back to a 128-bit CAS merge into
// `over`.  Consumers also merge `over`.
struct RedTarget {
    double2* over;  // [nch][cap]   (hi, lo) accumulators, CAS fallback and finalized totals
    double2* part;  // [cap][maxt][stride] records
    int32_t* cnt;   // [cap] records claimed per site
    int cap;
    int maxt;
    int stride;     // channels per record (11 for gradients, 8 for stats)
    // overflow pool: records beyond maxt per site go to opart[r], linked per site from head[site]
    int32_t* head;  // [cap] first overflow record of the site, -1 = none
    int32_t* onext; // [ocap] next record of the same site
    double2* opart; // [ocap][stride]
    int32_t* otop;  // pool allocation counter (reset per pass)
    int ocap;
    // adaptive layout (when roff != nullptr): site records live at part[roff[site] + slot] for
    // slot < rcap[site] (capacity planned from the previous pass's count), pool of `psize` records
    const int32_t* roff;
    int32_t* rcap;
    long long psize;
    // fp64 backward in the reference's summation order (k_backward_ord): one order tag per record
    // (tag[rec] for part, otag[r] for opart); nullptr: the double-double path
    uint32_t* tag = nullptr;
    uint32_t* otag = nullptr;
};

struct FieldDims {
    int width, height, cell, gw, gh, k;
    // Optional row range (pixel rows for the pixel kernels, cell rows for propagation; equal at cell 1):
    // the row-strip partition of a multi-GPU fit computes [row0, row1) only.  Defaults: everything.
    int row0 = 0, row1 = 1 << 30;
};

struct AdamHyper {
    double lr[10];
    double beta1, beta2, eps;
    double log_tau_min, log_tau_max, radius_min, radius_max, aniso_min, aniso_max;
    int clamp_color;
    int width, height;
};

struct SplitHyper {
    double log_tau_min, radius_min, aniso_min, aniso_max;
    int width, height;
    uint64_t max_sites;
};

// ---------------------------------------------------------------- tables
// which: bit0 pack (half snapshot), bit1 gtab, bit2 rtab.  T = float or double.
void launch_tables(bool fp64, const SitesDev& s, const DevState* st, double scale, void* pack, void* gtab,
                   void* rtab, cudaStream_t stream);

// ---------------------------------------------------------------- candidates
void launch_jfa_seed(const SitesDev& s, const DevState* st, uint32_t* ids, const FieldDims& f, double scale,
                     cudaStream_t stream);
void launch_propagate(bool fp64, const uint32_t* prev, uint32_t* next, const void* pack, const uint32_t* act,
                      const DevState* st, const FieldDims& f, uint32_t step, int box, int inject, uint64_t seed,
                      uint32_t pass_offset, double scale, cudaStream_t stream);
void launch_exact_topk(bool fp64, const void* rtab, const uint32_t* act, int n_act, const int32_t* xy, int n_pix,
                       int k, double scale, uint32_t* out, cudaStream_t stream);

// ---------------------------------------------------------------- render
void launch_render(bool fp64, const uint32_t* ids, const void* rtab, const FieldDims& f, double scale, void* out_rgb,
                   DevState* st, cudaStream_t stream);
void launch_id_map(const uint32_t* ids, const void* rtab_d, const FieldDims& f, double scale, uint32_t* out,
                   DevState* st, cudaStream_t stream);
void launch_pixel_weights(const uint32_t* ids, const void* rtab_d, const FieldDims& f, double scale,
                          const int32_t* xy, int n_q, uint32_t* out_ids, double* out_w, int32_t* out_n,
                          cudaStream_t stream);

// ---------------------------------------------------------------- backward / loss / stats
// mode: 0 = MSE target, 1 = MSE target + removal delta, 2 = caller adjoint (pixgrad)
// Per-block loss partials go to loss_part[block]; launch_loss_reduce / launch_advance reduce them.
int backward_blocks(bool fp64, const FieldDims& f, bool ordered = false);
// fp64 in the reference's summation order (default; SAD_FP64_DD=1 selects the double-double path):
// the runtime then passes RedTargets with order tags, launch_backward runs k_backward_ord, and the
// totals come from launch_ordered_totals (GradBuffer Accums into red.over with tot == nullptr, else
// values into tot[ch][cap], g0 = channel 2) instead of k_finalize / the Adam merge.
bool fp64_ordered();
void launch_ordered_totals(const RedTarget& red, int n_ch, const DevState* st, double* tot, double* g0, bool reset,
                           cudaStream_t stream);
// Row quantum of the per-tile kernels (least common multiple of the fp32/fp64 backward and the stats
// tile heights): row strips that are multiples of it never split a tile.
int tile_row_quantum();
void launch_backward(bool fp64, int mode, const uint32_t* ids, const void* gtab, const void* tgt_or_pixgrad,
                     const FieldDims& f, double scale, const RedTarget& red, double2* loss_part, DevState* st,
                     cudaStream_t stream);
int loss_blocks(const FieldDims& f);
void launch_loss(bool fp64, const uint32_t* ids, const void* gtab, const void* tgt, const FieldDims& f, double scale,
                 double2* loss_part, DevState* st, cudaStream_t stream);
void launch_loss_reduce(const double2* loss_part, int n, double2* dst, cudaStream_t stream);
void launch_stats(const uint32_t* ids, const void* rtab_d, const double* tgt, const FieldDims& f, double scale,
                  const RedTarget& red, DevState* st, cudaStream_t stream);
// Merges records into red.over (n_ch channels) for sites < n_sites and resets the record counters.
void launch_finalize(const RedTarget& red, int n_ch, const DevState* st, cudaStream_t stream);

// ---------------------------------------------------------------- optimiser
// Adam (+ clamp_project) over all slots < n_sites; optionally zeroes grads and rebuilds pack/gtab.
// bc: (1 - beta1^t, 1 - beta2^t) table indexed by the new t, or nullptr to use bc_now.
// With grads.roff set, Adam also writes next pass's record capacities to rcap_next (then
// launch_plan_records turns them into offsets).
void launch_adam(bool fp64, const SitesDev& s, DevState* st, const RedTarget& grads, double* m, double* v,
                 const AdamHyper& hp, const double2* bc_table, double2 bc_now, bool zero_grads, double scale,
                 void* pack, void* gtab, int32_t* rcap_next, cudaStream_t stream, const double* totals = nullptr,
                 int32_t* roff_next = nullptr, int32_t* pool_top = nullptr, const uint32_t* act = nullptr,
                 const int32_t* act_range = nullptr, const AdvanceArgs& adv = AdvanceArgs());
void launch_math(const double* x, double* y, size_t n, int which, cudaStream_t stream);
// row-strip fits (multi-GPU config 5)
void launch_site_partials(const RedTarget& grads, const DevState* st, int cap, double2* out, cudaStream_t stream);
void launch_merge_partials(const double2* parts, int world, int cap, int nch, double* values, double2* dd,
                           cudaStream_t stream);
// owner-merged exchange of the row-strip fit: ids [q*slice, (q+1)*slice) belong to rank q
struct OwnRec {
    uint32_t id, pad[3];
    double2 v[11];
};
void launch_owner_pack(const double2* part, int nch, const RedTarget& red, const DevState* st, const uint8_t* active,
                       int slice, int me, int world, OwnRec* send, int send_cap, unsigned long long* counts,
                       int32_t* rcap_next, bool reset, cudaStream_t stream);
void launch_owner_merge(const OwnRec* recv, long long n, int nch, int cap, double2* part, cudaStream_t stream);
// fp64 reference-order strips: the tagged records themselves travel to the owners (OwnRec.pad[0] = tag).
// count: records per destination rank; pack: writes them at per-destination cursors (send + q * send_cap);
// merge: the owner links each received record into the site's overflow list; finish: next pass's record
// capacities from this rank's own counts, then the per-site reduction state is reset.
void launch_owner_count_ord(const RedTarget& red, const DevState* st, int slice, int me, int world,
                            unsigned long long* counts, cudaStream_t stream);
void launch_owner_pack_ord(const RedTarget& red, const DevState* st, int slice, int me, int world, OwnRec* send,
                           long long send_cap, unsigned long long* cursors, cudaStream_t stream);
void launch_owner_merge_ord(const OwnRec* recv, long long n, const RedTarget& red, DevState* st, cudaStream_t stream);
void launch_ord_finish(const RedTarget& red, const DevState* st, const uint8_t* active, int32_t* rcap_next,
                       cudaStream_t stream);
template <typename T>
void launch_slice_pack(const T* src, int nch, int cap, int lo, int slice, T* buf, cudaStream_t stream);
template <typename T>
void launch_slice_unpack(const T* all, int nch, int cap, int slice, int world, T* dst, cudaStream_t stream);
void launch_owned_range(const uint32_t* act, const DevState* st, int lo, int hi, int32_t* range, cudaStream_t stream);
void launch_dd_values(const double2* dd, long long n, double* out, cudaStream_t stream);
// tau_diffusion pieces (train.cpp:171-213)
void launch_site_totals(const RedTarget& grads, const DevState* st, int cap, double* tot, double* g0,
                        cudaStream_t stream);
void launch_tau_edges(const uint32_t* ids, const uint32_t* owner, const uint8_t* active, const FieldDims& f, int nb,
                      uint64_t* keys, cudaStream_t stream);
void launch_tau_mix(const uint64_t* uniq, const int* count, int max_items, int nb, const double* g0, double lambda,
                    double* out, cudaStream_t stream);
// Initial record plan: rcap = per_site for every slot (offsets follow from a scan).
void launch_fill_i32(int32_t* p, int n, int32_t v, cudaStream_t stream);
void launch_stats_plan(const int32_t* gcnt, const DevState* st, int cap, int32_t* rcap, cudaStream_t stream);
void launch_clamp(const SitesDev& s, const DevState* st, const AdamHyper& hp, cudaStream_t stream);

// ---------------------------------------------------------------- budget events
void launch_prune_keys(const SitesDev& s, DevState* st, const double2* stats, int cap,
                       unsigned long long* keys, uint32_t* vals, cudaStream_t stream);
void launch_prune_apply(const SitesDev& s, DevState* st, const uint32_t* sorted, double pct, cudaStream_t stream);
void launch_densify_keys(const SitesDev& s, DevState* st, const double2* stats, int cap, double alpha, double eps,
                         unsigned long long* keys, uint32_t* vals, uint8_t* free_flags, cudaStream_t stream);
void launch_densify_apply(const SitesDev& s, DevState* st, const double2* stats, int cap, const uint32_t* sorted,
                          const uint32_t* free_list, const double* tgt, double pct, const SplitHyper& hp, double* m,
                          double* v, cudaStream_t stream);
void launch_flag_active(const SitesDev& s, const DevState* st, uint8_t* flags, cudaStream_t stream);

// ---------------------------------------------------------------- loop bookkeeping
// pass_index += passes; t and iter advance; records loss/active history row `iter`.
// With loss_hist: reduces loss_part[0..n_part) into history row `iter` and advances iter.
void launch_advance(DevState* st, int passes, int adam_steps, double2* loss_hist, int32_t* active_hist,
                    const double2* loss_part, int n_part, int32_t* otop, cudaStream_t stream);

// ---------------------------------------------------------------- init (train.cpp:33-111) device path
void launch_sobel(const double* tgt, int w, int h, double* mag, cudaStream_t stream);
void launch_init_keys(const double* mag, int w, int h, const double2* gsum, double lambda, const uint32_t* jump_states,
                      int chunk, unsigned long long* keys, uint32_t* vals, cudaStream_t stream);
void launch_init_sites(const SitesDev& s, DevState* st, const uint32_t* cells, int n, const double* tgt, int w, int h,
                       double r0, double log_tau0, double aniso0, const uint32_t* jump_states, int chunk,
                       cudaStream_t stream);
void launch_dd_sum(const double* x, size_t n, double2* out, cudaStream_t stream);
void launch_mark_cells(const uint32_t* sorted_idx, int n, uint8_t* flags, cudaStream_t stream);

// ---------------------------------------------------------------- misc
void launch_f64_to_f32(const double* in, float* out, size_t n, cudaStream_t stream);
void launch_scatter_grads_out(const double2* grads, int cap, int n, double* out /* n*11 */, cudaStream_t stream);

// Number of kernel launches issued through these wrappers (process-wide; evidence counter).
uint64_t launch_counter();
// checked builds (-DSAD_CHECKED=1): kernel bound-check violations so far; -1 in the product build
long long debug_check_failures();
// Graph replays re-run captured launches without passing through the wrappers: account for them.
void add_launches(uint64_t n);
// Sets per-kernel attributes (opt-in shared memory); call once per device before launching.
void prepare_kernels();

}  // namespace sadk
