/*
 * sad_b200.h — C ABI of the B200-native SAD (Soft Anisotropic Diagrams) fitting loop.
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json:north_star.  Every entry
 * point replaces one function of the reference C++ library (namespace `sad`, /root/reference/proj);
 * the replaced declaration is cited beside each prototype.  Nothing here uses C++ or torch types:
 * plain pointers, sizes and POD structs only, so cgo / JNI / ctypes / C++ can bind it directly.
 *
 * Data model (identical to the reference, so buffers can be passed through unchanged):
 *   - Sites: structure-of-arrays of ten doubles + u8 active/frozen flags      (types.hpp:37-63)
 *   - Candidate field: u32 ids[(gy*gw + gx)*k + i], sentinel 0xffffffff         (types.hpp:84-110)
 *   - Images: interleaved RGB doubles, row-major [py][px][c]                    (types.hpp:67-79)
 *   - Gradients: n x 11 doubles, slot order x,y,log_tau,r,R,G,B,dir_x,dir_y,a,removal (grad.hpp:13-26)
 *   - Adam moments: n x 10 doubles [id*10 + slot]                               (train.hpp:13-21)
 *   - Stats: n x 8 doubles (mass, energy, sx, sy, sxx, sxy, syy, removal)       (budget.hpp:14-25)
 *
 * Two layers:
 *   1. Per-call functions (sad_refresh, sad_render_image, sad_backward_image, ...) take HOST views,
 *      copy them to the device, run the CUDA kernels, and copy results back.  They reproduce the
 *      reference call-by-call (parity tests use them).
 *   2. The resident fit (sad_fit_*) keeps every buffer in HBM for the whole optimisation and only
 *      crosses PCIe for the target upload and the result download (sad::fit, train.cpp:295-311).
 *
 * Errors: every function returns a sad_status; sad_last_error() gives the thread-local message.
 * The reference throws std::invalid_argument / sad::numeric_error / sad::format_error; the codes
 * below map one to one (SAD_ESTALE and SAD_EEMPTY are invalid_argument in the reference).
 *
 * Precision: `fp64 = 0` selects the float32 kernels (RunOpts{fp64=false}); results then match the
 * reference's float path, which is the parity target.  `fp64 = 1` selects double kernels.
 */
#ifndef SAD_B200_H
#define SAD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAD_ABI_VERSION 1

typedef enum sad_status {
    SAD_OK = 0,
    SAD_EINVAL = 1,   /* std::invalid_argument: bad shapes / config / arguments */
    SAD_ESTALE = 2,   /* std::invalid_argument("candidate field is stale ...") render.cpp:11-15 */
    SAD_EEMPTY = 3,   /* std::invalid_argument("... empty candidate list ...") render.cpp:87-88 */
    SAD_ENUMERIC = 4, /* sad::numeric_error (train.cpp:250) */
    SAD_EFORMAT = 5,  /* sad::format_error */
    SAD_ECUDA = 6,    /* CUDA runtime failure (no reference equivalent) */
    SAD_ENOMEM = 7    /* capacity exhausted (caller must grow the view) */
} sad_status;

#define SAD_EMPTY_ID 0xffffffffu /* CandidateField::kEmpty (types.hpp:85) */

/* SiteStore (types.hpp:37-63).  `capacity` is the allocated length of every array; `size` the
 * number of slots in use.  Only densify may grow `size` (budget.cpp:277). */
typedef struct sad_sites_view {
    size_t size;
    size_t capacity;
    double *x, *y, *log_tau, *radius, *col_r, *col_g, *col_b, *dir_x, *dir_y, *aniso;
    uint8_t *active, *frozen;
    uint64_t generation;
} sad_sites_view;

/* CandidateField (types.hpp:84-110). */
typedef struct sad_field_view {
    int width, height; /* image extent */
    int cell;          /* integer downscale of the candidate grid */
    int gw, gh;        /* grid extent */
    int k;             /* list length, 1..16 */
    uint32_t* ids;     /* gw*gh*k */
    uint64_t synced_generation;
    uint64_t refresh_count;
    uint32_t pass_index;
} sad_field_view;

/* PassSpec (candidates.hpp:33-36). stencil: 0 = Axial, 1 = Box3. */
typedef struct sad_pass_spec {
    uint32_t step;
    int32_t stencil;
} sad_pass_spec;

/* RefreshMode (candidates.hpp:62-65). */
typedef enum sad_refresh_mode { SAD_REFRESH_FULL = 0, SAD_REFRESH_WARM = 1 } sad_refresh_mode;

/* AdamState (train.hpp:13-21): m, v are n x 10 doubles laid out [id*10 + slot]. */
typedef struct sad_adam_view {
    size_t sites;    /* rows in use */
    size_t capacity; /* rows allocated */
    double *m, *v;
    int64_t t;
    uint64_t skipped;
} sad_adam_view;

/* TrainConfig (types.hpp:112-167), field for field. */
typedef struct sad_train_config {
    int32_t iters;
    int32_t n_sites;
    double target_bpp;
    uint64_t seed;
    int32_t k;
    int32_t inject;
    double lambda_init;
    double lr_pos, lr_color, lr_log_tau, lr_radius, lr_dir, lr_aniso;
    double beta1, beta2, adam_eps;
    int32_t refresh_every, refresh_passes, final_passes;
    double tau_diffusion_lambda;
    int32_t densify_every, densify_start, densify_end;
    double densify_pct, alpha, stats_eps;
    int32_t prune_every, prune_start, prune_end;
    double prune_pct;
    int32_t prune_during_densify;
    double budget_scale_cap;
    uint64_t max_sites;
    double init_log_tau, init_radius, init_aniso;
    double log_tau_min, log_tau_max, radius_min, radius_max, aniso_min, aniso_max;
    int32_t clamp_color;
    int32_t fp64;
    int32_t threads; /* accepted for ABI parity with RunOpts; the GPU ignores it */
} sad_train_config;

/* HistoryRow (train.hpp:46-52). */
typedef struct sad_history_row {
    int32_t iter;
    double loss;
    double psnr;
    int32_t active_sites;
    double ms;
} sad_history_row;

typedef struct sad_ctx sad_ctx;
typedef struct sad_fit_run sad_fit_run;

/* ---------------------------------------------------------------- context / errors */
const char* sad_last_error(void);
int sad_abi_version(void);
/* Fills `cfg` with the reference defaults (types.hpp:121-167). */
void sad_default_config(sad_train_config* cfg);
/* Creates a context bound to CUDA `device`; `stream` is a cudaStream_t or NULL for a private one. */
sad_status sad_ctx_create(int device, void* stream, sad_ctx** out);
void sad_ctx_destroy(sad_ctx* ctx);
sad_status sad_ctx_synchronize(sad_ctx* ctx);
/* Number of kernel launches this context issued so far (evidence for the bench's gpu_launches). */
/* Bound-check violations counted by the kernels of a checked build (libsad_b200_checked.so, built with
 * -DSAD_CHECKED=1 by __graft_entry__.build_checked); -1 for the product build. */
long long sad_debug_check_failures(void);
uint64_t sad_ctx_launch_count(const sad_ctx* ctx);

/* ---------------------------------------------------------------- device-resident objects
 * A context can hold one SiteStore and one CandidateField in HBM.  Every per-call function below
 * that takes a sites or field view also accepts NULL, meaning "the context's resident object": it is
 * used in place (no host copy) and results stay on the device (fields produced by jfa_seed /
 * run_passes / refresh, sites changed by adam_step / clamp_project / init_sites / prune / densify),
 * with generation, pass_index, synced_generation and refresh_count tracked exactly as for views.
 * Passing a host view instead replaces the workspace copy and invalidates that resident object. */
sad_status sad_sites_alloc(sad_ctx* ctx, size_t capacity);            /* empty resident store */
sad_status sad_sites_upload(sad_ctx* ctx, const sad_sites_view* sites); /* size/generation from the view */
sad_status sad_sites_download(sad_ctx* ctx, sad_sites_view* sites);     /* capacity must hold `size` */
sad_status sad_sites_info(sad_ctx* ctx, size_t* size, size_t* capacity, uint64_t* generation);
sad_status sad_field_alloc(sad_ctx* ctx, int width, int height, int k, int cell); /* CandidateField::resize */
sad_status sad_field_upload(sad_ctx* ctx, const sad_field_view* field);
sad_status sad_field_download(sad_ctx* ctx, sad_field_view* field); /* ids: gw*gh*k or NULL (metadata only) */

/* The device ports of glibc's math the kernels use, applied to n host values -- exposed so their
 * bit-identity with the host libm can be verified.  single: 0 exp (double), 1 expf, 2 log (double). */
sad_status sad_math_exp(sad_ctx* ctx, const double* x, double* y, size_t n, int single);

/* ---------------------------------------------------------------- candidates.hpp */
/* jump_step (candidates.cpp:27-33) */
sad_status sad_jump_step(uint32_t t, uint32_t b, uint32_t* out);
/* full_refresh_passes / schedule_passes (candidates.cpp:37-62); `out` holds >= *n entries on entry */
sad_status sad_full_refresh_passes(int gw, int gh, int extra_step1, sad_pass_spec* out, int* n);
sad_status sad_schedule_passes(int gw, int gh, int total, sad_pass_spec* out, int* n);
/* jfa_seed (candidates.hpp:47, candidates.cpp:64-84) */
sad_status sad_jfa_seed(sad_ctx* ctx, const sad_sites_view* sites, sad_field_view* field);
/* run_passes / propagate_pass (candidates.hpp:55-60, candidates.cpp:143-181) */
sad_status sad_run_passes(sad_ctx* ctx, const sad_sites_view* sites, sad_field_view* field,
                          const sad_pass_spec* seq, int n_pass, int inject, uint64_t seed, int fp64);
/* refresh (candidates.hpp:67-68, candidates.cpp:183-194) */
sad_status sad_refresh(sad_ctx* ctx, const sad_sites_view* sites, sad_field_view* field,
                       int mode, int passes, int inject, uint64_t seed, int fp64);
/* exact_topk_batch (candidates.hpp:75-77, candidates.cpp:198-248): out is n_pix*k, sentinel-padded */
sad_status sad_exact_topk_batch(sad_ctx* ctx, const sad_sites_view* sites, const int32_t* pixels_xy,
                                size_t n_pix, int k, double scale, int fp64, uint32_t* out);

/* ---------------------------------------------------------------- render.hpp */
/* render_image (render.hpp:21-22, render.cpp:107-116): out is 3*W*H doubles */
sad_status sad_render_image(sad_ctx* ctx, const sad_sites_view* sites, const sad_field_view* field,
                            int fp64, double* out_rgb);
/* pixel_weights (render.hpp:18, render.cpp:93-105), batched: ids/w are n_q*16, n is n_q */
sad_status sad_pixel_weights(sad_ctx* ctx, const sad_sites_view* sites, const sad_field_view* field,
                             const int32_t* pixels_xy, size_t n_q, uint32_t* ids, double* w,
                             int32_t* n);
/* render_id_map (render.hpp:26-27, render.cpp:118-154) */
sad_status sad_render_id_map(sad_ctx* ctx, const sad_sites_view* sites, const sad_field_view* field,
                             uint32_t* out);

/* tau_diffusion (train.hpp:43-44, train.cpp:171-213).  grads: n*11 doubles in/out; only the logtau
 * column (slot 2) of pixel owners changes.  lambda == 0 is a no-op; lambda outside [0,1] -> EINVAL;
 * a stale field -> ESTALE; an empty candidate list -> EEMPTY (render_id_map). */
sad_status sad_tau_diffusion(sad_ctx* ctx, const sad_sites_view* sites, const sad_field_view* field, double lambda,
                             double* grads);

/* ---------------------------------------------------------------- grad.hpp */
/* backward_image (grad.hpp:96-98, grad.cpp:364-372).  grads: n*11 doubles (value of each Accum). */
sad_status sad_backward_image(sad_ctx* ctx, const sad_sites_view* sites, const sad_field_view* field,
                              const double* target_rgb, int fp64, int with_removal, double* grads,
                              uint64_t* nonfinite, double* loss);
/* image_loss (grad.hpp:101-102, grad.cpp:374-380) */
sad_status sad_image_loss(sad_ctx* ctx, const sad_sites_view* sites, const sad_field_view* field,
                          const double* target_rgb, int fp64, double* loss);
/* backward_pixel_grad (grad.hpp:106-107, grad.cpp:382-390).  dl_width x dl_height is the adjoint
 * image's size; a size other than the field's -> EINVAL "backward: adjoint size mismatch"
 * (grad.cpp:383-384), checked before any byte of dl_dvalue_rgb is read. */
sad_status sad_backward_pixel_grad(sad_ctx* ctx, const sad_sites_view* sites,
                                   const sad_field_view* field, const double* dl_dvalue_rgb,
                                   int dl_width, int dl_height, int fp64, double* grads,
                                   uint64_t* nonfinite);

/* ---------------------------------------------------------------- train.hpp */
/* adam_step (train.hpp:33-34, train.cpp:139-169) incl. clamp_project; updates sites and adam */
sad_status sad_adam_step(sad_ctx* ctx, sad_sites_view* sites, const double* grads,
                         sad_adam_view* adam, int width, int height, const sad_train_config* cfg);
/* clamp_project (train.hpp:38, train.cpp:113-137) */
sad_status sad_clamp_project(sad_ctx* ctx, sad_sites_view* sites, int width, int height,
                             const sad_train_config* cfg);
/* init_sites (train.hpp:29, train.cpp:59-111): sites.capacity must be >= n */
sad_status sad_init_sites(sad_ctx* ctx, sad_sites_view* sites, const double* target_rgb, int width,
                          int height, int n, const sad_train_config* cfg);

/* ---------------------------------------------------------------- budget.hpp */
/* accumulate_stats (budget.hpp:29-30, budget.cpp:39-155): stats n*8 doubles */
sad_status sad_accumulate_stats(sad_ctx* ctx, const sad_sites_view* sites,
                                const sad_field_view* field, const double* target_rgb,
                                double* stats, uint64_t* valid_pixels);
/* prune (budget.hpp:48, budget.cpp:286-305) */
sad_status sad_prune(sad_ctx* ctx, sad_sites_view* sites, const double* stats,
                     uint64_t valid_pixels, double percentile, int* removed);
/* densify (budget.hpp:43-44, budget.cpp:219-284).  May append up to `want` slots: sites and adam
 * capacities must allow size + want rows (SAD_ENOMEM otherwise). */
sad_status sad_densify(sad_ctx* ctx, sad_sites_view* sites, sad_adam_view* adam, const double* stats,
                       const double* target_rgb, int width, int height, double percentile,
                       const sad_train_config* cfg, int* done);
/* bpp_target_count / simulate_schedule / plan_schedule (budget.cpp:307-374) — host arithmetic */
sad_status sad_bpp_target_count(double bpp, int width, int height, uint64_t* out);
sad_status sad_simulate_schedule(int n0, double scale, const sad_train_config* cfg, int* out);
sad_status sad_plan_schedule(int n0, uint64_t target, const sad_train_config* cfg, double* out);

/* ---------------------------------------------------------------- codec.hpp (decode path) */
/* write_file (codec.cpp:147-177) into memory: out NULL -> only *nbytes = required size. */
sad_status sad_encode(const sad_sites_view* sites, int width, int height, uint8_t* out, size_t cap, size_t* nbytes);
/* read_file header checks (codec.cpp:179-205): magic, version, extent, size equation. */
sad_status sad_decode_header(const uint8_t* buf, size_t n, int* width, int* height, uint32_t* count);
/* read_file + unpack_site (codec.cpp:115-140, 179-222); sites.capacity >= count. */
sad_status sad_decode(const uint8_t* buf, size_t n, sad_sites_view* sites, int* width, int* height);
/* bpp (codec.cpp:142-145) */
sad_status sad_bpp(size_t count, int width, int height, double* out);
/* Decode pipeline: bytes -> sites -> refresh(Full, passes) on the device -> render_image into out_rgb
 * (3*W*H host doubles); optionally returns the decoded sites (capacity >= count). */
sad_status sad_decode_render(sad_ctx* ctx, const uint8_t* buf, size_t n, int k, int passes, int inject,
                             uint64_t seed, int fp64, double* out_rgb, sad_sites_view* out_sites);

/* ---------------------------------------------------------------- row-strip multi-GPU fit (config 5)
 * One image split into row strips (multiples of the tile heights): each rank holds the sites and tables
 * and computes its strip of the propagation passes, backward and stats.  Sites are owned by id slice
 * (rank q: ids [q*slice, (q+1)*slice)): the partial totals of touched, non-owned sites travel to their
 * owners, who merge them exactly and run Adam on their slice; the parameter slices are then all-gathered
 * (events: stats totals too, and prune / densify run replicated).  Every merge is an exact double-double
 * merge, so the result is bit-identical to the single-GPU fit.  One process per GPU: rank 0 calls
 * sad_nccl_unique_id and shares the 128 bytes (e.g. torch.distributed), every rank creates one
 * communicator (sad_strip_comm_create; NCCL ids are single-use), then per fit its run (sad_fit_create,
 * sad_fit_set_target with the whole image) and calls sad_fit_run_strips (init NULL:
 * fit(), else fit_store() from `init`).  Results are read with sad_fit_info / sad_fit_download on any rank.
 * sad_fit_run_strips_loopback runs `world` virtual ranks (runs created on one context) on one device,
 * exchanging by device copies: the single-GPU check of the partition.
 * sad_strip_comm_create_host builds a host-staged communicator: device data is copied to pinned host
 * memory and moved by the caller's callbacks (return 0 on success) — e.g. a torch.distributed gloo group,
 * which lets several processes share one GPU:
 *   allgather(user, send, recv, bytes): recv[q*bytes, (q+1)*bytes) <- rank q's send;
 *   exchange(user, n, peer, send, send_bytes, recv, recv_bytes): for each i, send send[i] to peer[i] and
 *     receive recv[i] from it; transfers to one peer pair up in order, zero-byte entries are skipped.
 * sad_fit_strip_exchange reports the gradient records this rank sent to owners during the last fit. */
typedef struct sad_strip_comm sad_strip_comm; /* a communicator over the strip ranks (reusable) */
typedef int (*sad_host_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);
typedef int (*sad_host_exchange_fn)(void* user, int n, const int* peer, const void* const* send,
                                    const size_t* send_bytes, void* const* recv, const size_t* recv_bytes);
sad_status sad_nccl_unique_id(uint8_t* out128);
sad_status sad_strip_comm_create(int rank, int world, const uint8_t* nccl_id128, sad_strip_comm** out);
sad_status sad_strip_comm_create_host(int rank, int world, sad_host_allgather_fn allgather,
                                      sad_host_exchange_fn exchange, void* user, sad_strip_comm** out);
void sad_strip_comm_destroy(sad_strip_comm* comm);
sad_status sad_fit_run_strips(sad_fit_run* run, sad_strip_comm* comm, const sad_sites_view* init);
sad_status sad_fit_run_strips_loopback(sad_fit_run* const* runs, int world);
sad_status sad_fit_strip_exchange(sad_fit_run* run, long long* records_sent);

/* ---------------------------------------------------------------- fit / fit_store in one call
 * fit (train.hpp:62-63, train.cpp:295-311) and fit_store (train.hpp:66-68): target upload, the whole
 * resident loop, result download.  out_sites->capacity >= sad_fit_capacity(); out_field (optional)
 * needs an ids buffer of W*H*k (cell 1; metadata is filled in); history (optional) holds cfg->iters
 * rows; schedule_scale (optional) receives FitResult::schedule_scale. */
sad_status sad_fit_capacity(int width, int height, const sad_train_config* cfg, size_t n_init, size_t* capacity);
sad_status sad_fit(sad_ctx* ctx, const double* target_rgb, int width, int height, const sad_train_config* cfg,
                   sad_sites_view* out_sites, sad_field_view* out_field, sad_history_row* history,
                   double* schedule_scale);
sad_status sad_fit_store(sad_ctx* ctx, const double* target_rgb, int width, int height,
                         const sad_sites_view* initial_sites, const sad_train_config* cfg, sad_sites_view* out_sites,
                         sad_field_view* out_field, sad_history_row* history, double* schedule_scale);

/* ---------------------------------------------------------------- resident fit (train.cpp:221-311) */
/* Allocates every device buffer for a W x H fit.  `n_init` = 0 lets fit() choose (bpp / n_sites). */
sad_status sad_fit_create(sad_ctx* ctx, int width, int height, const sad_train_config* cfg,
                          sad_fit_run** out);
void sad_fit_destroy(sad_fit_run* run);
/* Target upload from host RGB doubles (H2D inside) or from a device pointer (already in HBM). */
sad_status sad_fit_set_target(sad_fit_run* run, const double* host_rgb);
sad_status sad_fit_set_target_device(sad_fit_run* run, const double* device_rgb);
/* fit(): init_sites on the device, then the loop.  fit_store(): start from caller sites. */
sad_status sad_fit_run_init(sad_fit_run* run);
sad_status sad_fit_run_store(sad_fit_run* run, const sad_sites_view* sites);
/* Results.  Sizes first, then a download into caller views sized from them. */
sad_status sad_fit_info(sad_fit_run* run, size_t* n_sites, int* n_history, double* schedule_scale);
sad_status sad_fit_download(sad_fit_run* run, sad_sites_view* sites, sad_field_view* field,
                            sad_history_row* history);
/* Device-side render of the fitted field into a device buffer (float32 RGB, 3*W*H), no copies. */
sad_status sad_fit_render_device(sad_fit_run* run, float* device_rgb);
/* Total kernel time of the last run in ms and per-phase split (propagate, fwd_bwd, adam, events). */
sad_status sad_fit_timing(sad_fit_run* run, double* total_ms, double* phase_ms4);
/* Enables per-phase CUDA-event timing for the next runs (propagate, fwd+bwd, Adam+bookkeeping,
 * events); costs a few microseconds per iteration and disables graph replay while on. */
sad_status sad_fit_set_profiling(sad_fit_run* run, int on);
/* Times `reps` launches of one kernel on the fitted, device-resident state with CUDA events on the
 * run's stream.  which: 0 warm propagate pass, 1 fused fwd+bwd, 2 render, 3 Box3 flood pass
 * (step 16), 4 Adam, 5 stats.  Evidence for the roofline numbers; not part of the reference API. */
sad_status sad_fit_bench(sad_fit_run* run, int which, int reps, double* ms_per_launch);
/* Batched point queries (pixel_weights, render.cpp:93-105) against the fitted field; all pointers
 * are DEVICE pointers: xy is n_q (x, y) pairs, ids/w receive 16 entries per query, n the counts. */
sad_status sad_fit_point_query(sad_fit_run* run, const int32_t* d_xy, size_t n_q, uint32_t* d_ids, double* d_w,
                               int32_t* d_n);
/* Pinned host memory for zero-staging transfers (cudaMallocHost / cudaFreeHost). */
void* sad_host_alloc(size_t bytes);
void sad_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* SAD_B200_H */
