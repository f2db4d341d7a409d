// Forced include (TEST INFRASTRUCTURE ONLY) for the reference's hot-path translation units when they are
// linked beside tests/reftests/sad_link_shim.cpp: the functions the shim provides on the GPU are renamed
// to cpu_* here, so the reference's own definitions stay compiled (and internally consistent) but unused,
// and every call the unmodified tests make resolves to the shim.
#pragma once
#define jfa_seed cpu_jfa_seed
#define propagate_pass cpu_propagate_pass
#define run_passes cpu_run_passes
#define refresh cpu_refresh
#define exact_topk cpu_exact_topk
#define exact_topk_batch cpu_exact_topk_batch
#define pixel_weights cpu_pixel_weights
#define render_image cpu_render_image
#define render_id_map cpu_render_id_map
#define render_tau_map cpu_render_tau_map
#define backward_image cpu_backward_image
#define image_loss cpu_image_loss
#define backward_pixel_grad cpu_backward_pixel_grad
#define init_sites cpu_init_sites
#define adam_step cpu_adam_step
#define clamp_project cpu_clamp_project
#define tau_diffusion cpu_tau_diffusion
#define fit cpu_fit
#define fit_store cpu_fit_store
#define accumulate_stats cpu_accumulate_stats
#define densify cpu_densify
#define prune cpu_prune
#define bpp_target_count cpu_bpp_target_count
#define plan_schedule cpu_plan_schedule
#define simulate_schedule cpu_simulate_schedule
