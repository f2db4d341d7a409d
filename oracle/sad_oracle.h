/* sad_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, single-threaded restatement of the reference SAD fitting loop
 * (/root/reference/proj, C++20).  It is the CPU checker for the CUDA path: tests/, smoke() and the
 * bench's cpu_baseline leg may call it; the product never does.  Parity of this restatement is
 * pinned against the compiled reference (oracle/_ref/libsadref.so) by tests/test_oracle.py and
 * against committed golden vectors in tests/golden/ generated from that library.
 *
 * Entry points mirror include/sad_b200.h with a `sado_` prefix and take the same host views.
 */
#ifndef SAD_ORACLE_H
#define SAD_ORACLE_H
#include "../include/sad_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* sado_last_error(void);
void sado_default_config(sad_train_config* cfg);
uint32_t sado_seeded_state(uint64_t seed, uint32_t a, uint32_t b);
uint16_t sado_float_to_half(float f);
float sado_half_to_float(uint16_t h);
double sado_psnr_from_loss(double loss);

int sado_jump_step(uint32_t t, uint32_t b, uint32_t* out);
int sado_full_refresh_passes(int gw, int gh, int extra, sad_pass_spec* out, int* n);
int sado_jfa_seed(const sad_sites_view* s, sad_field_view* f);
int sado_run_passes(const sad_sites_view* s, sad_field_view* f, const sad_pass_spec* seq, int n_pass,
                    int inject, uint64_t seed, int fp64);
int sado_refresh(const sad_sites_view* s, sad_field_view* f, int mode, int passes, int inject,
                 uint64_t seed, int fp64);
int sado_render_image(const sad_sites_view* s, const sad_field_view* f, int fp64, double* out);
int sado_render_id_map(const sad_sites_view* s, const sad_field_view* f, uint32_t* out);
int sado_backward_image(const sad_sites_view* s, const sad_field_view* f, const double* tgt, int fp64,
                        int with_removal, double* grads, uint64_t* nonfinite, double* loss);
int sado_image_loss(const sad_sites_view* s, const sad_field_view* f, const double* tgt, int fp64,
                    double* loss);
int sado_tau_diffusion(const sad_sites_view* s, const sad_field_view* f, double lambda, double* grads);
int sado_adam_step(sad_sites_view* s, const double* grads, sad_adam_view* a, int w, int h,
                   const sad_train_config* cfg);
int sado_clamp_project(sad_sites_view* s, int w, int h, const sad_train_config* cfg);
int sado_init_sites(sad_sites_view* s, const double* tgt, int w, int h, int n,
                    const sad_train_config* cfg);
int sado_accumulate_stats(const sad_sites_view* s, const sad_field_view* f, const double* tgt,
                          double* stats, uint64_t* valid);
int sado_prune(sad_sites_view* s, const double* stats, uint64_t valid, double pct, int* removed);
int sado_densify(sad_sites_view* s, sad_adam_view* a, const double* stats, const double* tgt, int w,
                 int h, double pct, const sad_train_config* cfg, int* done);
int sado_bpp_target_count(double bpp, int w, int h, uint64_t* out);
int sado_simulate_schedule(int n0, double scale, const sad_train_config* cfg, int* out);
int sado_plan_schedule(int n0, uint64_t target, const sad_train_config* cfg, double* out);
/* fit: `init` NULL -> fit() (init_sites), else fit_store().  `out` sites/field must be sized by
 * the caller from sado_fit_capacity(); history holds cfg->iters rows. */
int sado_encode(const sad_sites_view* s, int w, int h, uint8_t* out, size_t cap, size_t* nbytes);
int sado_decode(const uint8_t* buf, size_t n, sad_sites_view* s, int* w, int* h);
int sado_fit_capacity(int w, int h, const sad_train_config* cfg, size_t n_init, size_t* cap);
int sado_fit(const double* tgt, int w, int h, const sad_train_config* cfg,
             const sad_sites_view* init, sad_sites_view* out_sites, sad_field_view* out_field,
             sad_history_row* history, double* schedule_scale);

#ifdef __cplusplus
}
#endif
#endif
