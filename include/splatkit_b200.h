/*
 * splatkit_b200 — C ABI of the B200-native 3DGS training hot path.
 *
 * This is the drop-in boundary for the reference's header-only C++ API in
 * namespace splat (reference: proj/include/splatkit/ headers). The reference has
 * no FFI of its own; every entry point below names the reference function it
 * replaces (file:line, relative to proj/include/splatkit/). A C++ caller keeps
 * the splat:: surface through include/splatkit_b200.hpp, which is a thin
 * header-only layer over these symbols.
 *
 * Conventions
 *  - Every function returns an int status (SK_OK == 0). sk_last_error(ctx)
 *    returns the message of the last failure on that context. No C++ exception
 *    crosses this boundary; the C++ wrapper rethrows std::runtime_error /
 *    std::invalid_argument with the reference's message text
 *    (types.hpp:66-68, scene.hpp:89-92, raster.hpp:116).
 *  - A context owns one CUDA device and one stream. It is not thread-safe;
 *    callers synchronise externally (reference: single writer, parallel.hpp).
 *  - Host buffers are borrowed for the duration of the call. Device buffers
 *    returned by *_device_* accessors stay owned by the library.
 *  - Storage orders: images are row-major interleaved RGB float32 [H][W][3]
 *    (types.hpp:39-48 Image<T>); per-pixel scalar maps are row-major [H][W]
 *    (the reference's Eigen ScalarMap/MaskMap are column-major; the C++
 *    wrapper transposes). Scene parameters are planar fp32 [C][n] with the
 *    component order given by SK_COMP_* below.
 */
#ifndef SPLATKIT_B200_H_
#define SPLATKIT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_OK 0
#define SK_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define SK_ERR_RUNTIME 2          /* std::runtime_error (require()) */
#define SK_ERR_CUDA 3             /* CUDA runtime / launch failure */
#define SK_ERR_OUT_OF_MEMORY 4

/* ---- scene parameter layout: planar fp32 [SK_COMP_COUNT(deg)][n] ----------
 * Gaussian3D<T> (scene.hpp:18-27): mu(3) rot(4, w x y z) log_scale(3)
 * opacity_logit(1) sh((deg+1)^2 x 3). SH coefficient (k, c) — row k, RGB
 * column c of the reference ShMatrix — is component SK_COMP_SH + 3 k + c.   */
#define SK_COMP_MU 0
#define SK_COMP_ROT 3
#define SK_COMP_LOG_SCALE 7
#define SK_COMP_OPACITY 10
#define SK_COMP_SH 11
#define SK_COMP_COUNT(deg) (11 + 3 * ((deg) + 1) * ((deg) + 1))

/* Camera<T> (camera.hpp:23-57). world_to_cam is a row-major 4x4. */
typedef struct sk_camera {
  int32_t width, height;
  float fx, fy, cx, cy;
  float world_to_cam[16];
  float near_plane;
} sk_camera;

/* BinningConfig<T> (raster.hpp:41-46) plus the tile size that the reference
 * passes separately to build_tile_grid (raster.hpp:157). mode: 0 = AABB,
 * 1 = compact box. */
typedef struct sk_binning {
  int32_t mode;
  float beta;
  float tau_alpha;
  int32_t tile_size; /* 8, 16 or 32 */
} sk_binning;

/* ProjectedGaussian<T> (camera.hpp:60-68) as host SoA arrays of n entries.
 * Arrays may be NULL when not needed. cov2d / conic are row-major 2x2. */
typedef struct sk_projected {
  int32_t* visible;       /* [n] 1 if not culled (project() returned a value) */
  float* mu2d;            /* [n][2] */
  float* cov2d;           /* [n][4] */
  float* conic;           /* [n][4] cov2d_inv */
  float* depth;           /* [n] */
  float* color;           /* [n][3] */
  float* opacity;         /* [n] */
  int32_t* tiles_touched; /* [n] number of tiles the footprint bins into */
} sk_projected;

/* BlendGrads<T> (raster.hpp:251-275) as host SoA arrays of n entries. */
typedef struct sk_blend_grads {
  float* d_mu2d;    /* [n][2] */
  float* d_conic;   /* [n][4] full-matrix convention */
  float* d_color;   /* [n][3] */
  float* d_opacity; /* [n] */
  float* abs_grad;  /* [n][2] */
} sk_blend_grads;

/* LossResult<T> (loss.hpp:10-19) scalars, plus the PSNR the trainer logs. */
typedef struct sk_loss_values {
  double loss, l1, ssim, psnr;
} sk_loss_values;

typedef struct sk_ctx sk_ctx;
typedef struct sk_scene sk_scene;
typedef struct sk_frame sk_frame;

/* ---- context ------------------------------------------------------------ */
int sk_ctx_create(int device, sk_ctx** out);
int sk_ctx_destroy(sk_ctx* ctx);
const char* sk_last_error(const sk_ctx* ctx);
int sk_ctx_set_stream(sk_ctx* ctx, void* cuda_stream);
int sk_ctx_synchronize(sk_ctx* ctx);
/* Number of library kernels launched on this context so far. */
int sk_ctx_launch_count(const sk_ctx* ctx, int64_t* out);
/* Per-phase device timing of training steps (CUDA events on the context
 * stream). Phases: 0 preprocess (K1), 1 binning + sort (K2-K5), 2 forward
 * blend (K6), 3 loss (K7), 4 backward blend (K8), 5 project-backward (K9,
 * plus the gradient all-reduce on a view-parallel step), 6 Adam (K10).
 * ms[SK_NUM_PHASES] accumulates milliseconds, steps counts timed steps. */
#define SK_NUM_PHASES 7
int sk_ctx_enable_timing(sk_ctx* ctx, int on);
int sk_ctx_get_timing(const sk_ctx* ctx, double* ms, int64_t* steps);
int sk_ctx_reset_timing(sk_ctx* ctx);
/* Phase timing of density events (Trainer::density_event trainer.hpp:177-243)
 * while timing is on: 0 the K scored views (K1-K6 + K11 error maps + K7 SSIM
 * + K12 masked count blend per view, plus the C3 exchange), 1 K13 scores,
 * 2 K14 selection, 3 K15 compaction (+ Adam moment remap). */
#define SK_NUM_EVENT_PHASES 4
int sk_ctx_get_event_timing(const sk_ctx* ctx, double* ms, int64_t* events);
/* Kernel-only time inside phase 3 (sum over timed events): the K15 row-move
 * kernel, without the class scans and the host round trip for the split
 * normals (the phase time includes both). */
int sk_ctx_get_compact_kernel_ms(const sk_ctx* ctx, double* move_ms);
/* Training steps this context launched as the captured CUDA graph
 * (single-rank pipelined steps in steady state; SK_STEP_GRAPH=0 disables). */
int sk_ctx_graph_steps(const sk_ctx* ctx, int64_t* steps);
const char* sk_version(void);

/* ---- scene (Scene<T>, scene.hpp:30-52) ---------------------------------- */
int sk_scene_create(sk_ctx* ctx, int sh_degree, int64_t capacity, sk_scene** out);
int sk_scene_destroy(sk_scene* scene);
/* host_params: planar [SK_COMP_COUNT(deg)][n]. Resets Adam state and the
 * score table (SceneOptimizer::init adam.hpp:102-111, ScoreTable::reset
 * adc.hpp:33-42). */
int sk_scene_upload(sk_ctx* ctx, sk_scene* scene, const float* host_params, int64_t n);
int sk_scene_download(sk_ctx* ctx, const sk_scene* scene, float* host_params);
int sk_scene_size(const sk_scene* scene, int64_t* n);
int sk_scene_sh_degree(const sk_scene* scene, int* deg);
/* Device pointer to the planar parameters and their component stride. */
int sk_scene_device_params(const sk_scene* scene, float** params, int64_t* stride);

/* ---- per-view render state ---------------------------------------------- */
int sk_frame_create(sk_ctx* ctx, sk_frame** out);
int sk_frame_destroy(sk_frame* frame);

/* K1: project() for every Gaussian (camera.hpp:93-123, project_scene :137),
 * plus the per-Gaussian tile count of bin_aabb / bin_compact
 * (raster.hpp:61-141). */
int sk_preprocess(sk_ctx* ctx, const sk_scene* scene, const sk_camera* cam,
                  const sk_binning* binning, sk_frame* frame);
/* Injects n already-projected Gaussians (projected index i, source index i),
 * as the reference tests do with random_projected (tests/helpers.hpp:72-96). */
int sk_frame_set_projected(sk_ctx* ctx, sk_frame* frame, const sk_projected* pgs, int64_t n,
                           int width, int height, const sk_binning* binning);
/* K2-K5: build_tile_grid (raster.hpp:157-168): depth order (:146-154),
 * per-tile lists, count_pairs (:170-174). pairs may be NULL. */
int sk_bin_sort(sk_ctx* ctx, sk_frame* frame, int64_t* pairs);
/* K6 / K12: blend_forward (raster.hpp:194-248). mask_host ([H][W] u8) and
 * counts_host ([n_source] int32, accumulated +=) may both be NULL; if one is
 * given the other must be too. */
int sk_render_forward(sk_ctx* ctx, sk_frame* frame, const uint8_t* mask_host,
                      int32_t* counts_host);

/* A caller's TileGrid (raster.hpp:27-57, build_tile_grid :157-168) for the
 * frame's projected set: ranges [tiles][2] contiguous in tile order into
 * values [pairs] (projected indices). sk_render_forward then blends exactly
 * these lists in their given order (blend_forward raster.hpp:194-248). */
int sk_frame_set_tile_lists(sk_ctx* ctx, sk_frame* frame, const int32_t* ranges, const int32_t* values,
                            int64_t pairs);
/* A caller's rendered image ([H][W][3]) as the frame's render, so sk_loss
 * evaluates training_loss(rendered, gt, lambda) (loss.hpp:21-47) on it. */
int sk_frame_set_image(sk_ctx* ctx, sk_frame* frame, const float* hwc, int width, int height);

/* Workload counters of the last forward render (SURVEY 8(d) roofline units):
 * visited = pixel-Gaussian evaluations the reference loop performs
 * (raster.hpp:219-235: list entries up to and including the terminating one),
 * contributing = entries with alpha >= 1/255 (sum of contrib_count). */
int sk_frame_pge_counts(sk_ctx* ctx, sk_frame* frame, int64_t* visited, int64_t* contributing);

/* frame readback */
int sk_frame_num_projected(const sk_frame* frame, int64_t* n);
int sk_frame_dims(const sk_frame* frame, int* width, int* height);
int sk_frame_get_projected(sk_ctx* ctx, const sk_frame* frame, sk_projected* out);
int sk_frame_get_image(sk_ctx* ctx, const sk_frame* frame, float* hwc);
int sk_frame_get_transmittance(sk_ctx* ctx, const sk_frame* frame, float* hw);
int sk_frame_get_contrib_count(sk_ctx* ctx, const sk_frame* frame, int32_t* hw);
/* Tile lists: ranges [tiles][2] (begin, end) into values [pairs]. */
int sk_frame_num_tiles(const sk_frame* frame, int* tiles_x, int* tiles_y);
int sk_frame_get_tile_lists(sk_ctx* ctx, const sk_frame* frame, int32_t* ranges,
                            int32_t* values);

/* ---- loss (training_loss loss.hpp:21-47, ssim_with_grad metrics.hpp:93) --
 * gt_host: [H][W][3] float32 image. Leaves dL/dimage on the frame. */
int sk_loss(sk_ctx* ctx, sk_frame* frame, const float* gt_host, float lambda,
            sk_loss_values* out);
/* Same with an 8-bit GT already decoded as byte/255.0f (png_io.cpp:64). */
int sk_loss_u8(sk_ctx* ctx, sk_frame* frame, const uint8_t* gt_host, float lambda,
               sk_loss_values* out);
/* SSIM only (metrics.hpp:83-89), and PSNR (metrics.hpp:126-134). */
int sk_ssim(sk_ctx* ctx, const float* a_hwc, const float* b_hwc, int width, int height,
            double* ssim_out, double* psnr_out);
/* float64 value path (the reference's T = double instantiation,
 * tools/splatkit_main.cpp:31; used by its FD tests, acceptance.cpp:163-254):
 * project -> tile-binned blend_forward -> training_loss, all in double on the
 * device. params_host: planar [SK_COMP_COUNT(deg)][n] doubles (n <= 65536).
 * image_hwc (nullable): [H][W][3] rendered image. gt_hwc + loss3 (both
 * nullable): loss3 = {loss, l1, ssim}. A checking path for finite
 * differences, not a training path. */
int sk_fp64_render_loss(sk_ctx* ctx, const double* params_host, int64_t n, int sh_degree,
                        const sk_camera* cam, const sk_binning* binning, const double* gt_hwc,
                        double lambda, double* image_hwc, double* loss3);
int sk_frame_get_dimage(sk_ctx* ctx, const sk_frame* frame, float* hwc);
int sk_frame_set_dimage(sk_ctx* ctx, sk_frame* frame, const float* hwc);

/* ---- backward (blend_backward raster.hpp:281-355) ---------------------- */
int sk_render_backward(sk_ctx* ctx, sk_frame* frame);
int sk_frame_get_blend_grads(sk_ctx* ctx, const sk_frame* frame, sk_blend_grads* out);

/* ---- optimizer (adam.hpp) and score table (adc.hpp:23-45) ---------------- */
/* LearningRates<T> (adam.hpp:78-86). */
typedef struct sk_learning_rates {
  float position, position_final, sh_dc, sh_rest, opacity, scale, rotation;
} sk_learning_rates;
void sk_default_learning_rates(sk_learning_rates* out);
/* expon_lr (adam.hpp:23-26), evaluated in float exactly as the reference. */
float sk_expon_lr(float lr_init, float lr_final, int step, int max_steps);

/* ScoreTable<T> as host SoA arrays [n] (grad3d_acc [n][3]); NULL = skip. */
typedef struct sk_score_table {
  float* s_d;
  float* s_p_raw;
  float* s_p;
  float* grad_norm_acc;
  float* abs_grad_acc;
  float* grad3d_acc;
  int32_t* views_seen;
  float* max_radius2d;
} sk_score_table;
int sk_scene_get_score_table(sk_ctx* ctx, sk_scene* scene, sk_score_table* out);
int sk_scene_set_score_table(sk_ctx* ctx, sk_scene* scene, const sk_score_table* in);
int sk_scene_reset_score_table(sk_ctx* ctx, sk_scene* scene);

/* K9: cov_grad_from_inv_grad + project_backward (camera.hpp:148-213) for every
 * Gaussian the frame projected, into the scene's planar gradient buffer
 * (culled Gaussians get zeros, SceneGrads::init adam.hpp:90-97); with
 * accumulate_stats the ScoreTable statistics of trainer.hpp:139-156 are
 * updated. grads_host ([C][n]) may be NULL. */
int sk_project_backward(sk_ctx* ctx, sk_scene* scene, sk_frame* frame, int accumulate_stats, float* grads_host);
/* project_backward (camera.hpp:156-213) for every Gaussian of the scene
 * (no culling test, as the reference's per-Gaussian call) with explicit
 * upstream gradients: d_mu2d [n][2], d_cov2d [n][4] (row-major 2x2, the
 * output of cov_grad_from_inv_grad camera.hpp:148-150), d_color [n][3],
 * d_opacity [n]. Gradients go to the scene's gradient buffer and, if
 * grads_host != NULL, to planar [C][n] host memory. */
int sk_project_backward_explicit(sk_ctx* ctx, sk_scene* scene, const sk_camera* cam, const float* d_mu2d,
                                 const float* d_cov2d, const float* d_color, const float* d_opacity,
                                 float* grads_host);
/* Overwrites the parameters (planar [C][n], n = the scene size) keeping the
 * optimizer state (SceneOptimizer holds moments across steps, adam.hpp). */
int sk_scene_set_params(sk_ctx* ctx, sk_scene* scene, const float* host_params, int64_t n);
/* SceneOptimizer::remap (adam.hpp:113-120 / AdamGroup::remap :45-58):
 * old_to_new [n] (-1 = removed), the scene size becomes new_n; survivors keep
 * their moments, new slots start at zero, the step counters are kept. */
int sk_scene_remap_moments(sk_ctx* ctx, sk_scene* scene, const int32_t* old_to_new, int64_t new_n);
/* SceneOptimizer::step_sh_rest (adam.hpp:146-153): the SH-rest group alone,
 * from the gradient buffer. */
int sk_adam_step_sh_rest(sk_ctx* ctx, sk_scene* scene, const sk_learning_rates* lrs);
/* SceneOptimizer::reset_opacity_state (adam.hpp:157-160). */
int sk_adam_reset_opacity_state(sk_ctx* ctx, sk_scene* scene);
/* Overwrites the scene's gradient buffer (planar [C][n]). */
int sk_scene_set_grads(sk_ctx* ctx, sk_scene* scene, const float* grads_host);
/* K10: SceneOptimizer::step (adam.hpp:124-143) from the gradient buffer. */
int sk_adam_step(sk_ctx* ctx, sk_scene* scene, const sk_learning_rates* lrs, float position_lr, int update_sh_rest);
/* K9 + K10 fused: gradients stay in registers. */
int sk_project_backward_adam(sk_ctx* ctx, sk_scene* scene, sk_frame* frame, const sk_learning_rates* lrs,
                             float position_lr, int update_sh_rest, int accumulate_stats);
/* Adam moments (planar [C][n], may be NULL) and the six group step counters. */
int sk_scene_get_adam(sk_ctx* ctx, const sk_scene* scene, float* m, float* v, int64_t* t6);

/* ---- multi-view density control (adc.hpp, the paper's contribution) ------- */
/* accumulate_scores (adc.hpp:91-115): renders each of the k views, builds its
 * error maps (error_maps.hpp:22-43), counts per Gaussian the high-error pixels
 * it contributes to (second blend pass), and fills s_d / s_p_raw / s_p of
 * the scene's ScoreTable (scores_from_counts :69-84). images: k float32 HWC
 * images concatenated. counts_out ([k][n]) and photometric_out ([k]) may be
 * NULL. */
int sk_accumulate_scores(sk_ctx* ctx, sk_scene* scene, int k, const sk_camera* cams, const float* images, float tau,
                         float lambda, const sk_binning* binning, int32_t* counts_out, float* photometric_out);
/* build_error_maps (error_maps.hpp:22-43) on explicit [H][W][3] images:
 * raw and normalized maps and the strict mask ([H][W] row-major; any output
 * may be NULL) and the photometric term. */
int sk_error_maps(sk_ctx* ctx, const float* rendered, const float* gt, int width, int height, float tau,
                  float lambda, float* raw, float* normalized, uint8_t* mask, float* photometric);
/* scores_from_counts (adc.hpp:69-84) on explicit count rows counts [k][n]
 * and photometric [k]: s_d, s_p_raw and the min-max normalized s_p ([n]
 * each, any may be NULL). Raises the reference's message for k == 0. */
int sk_scores_from_counts(sk_ctx* ctx, const int32_t* counts, const float* photometric, int k, int64_t n, float* s_d,
                          float* s_p_raw, float* s_p);
/* select_densify (adc.hpp:135-153) over the scene's ScoreTable; flags [n]. */
int sk_select_densify(sk_ctx* ctx, sk_scene* scene, float tau_d, float grad_threshold, float percent_dense,
                      int use_vcd, float extent, uint8_t* clone, uint8_t* split);
/* PruneParams<T> (adc.hpp:208-217). */
typedef struct sk_prune_params {
  float tau_p, min_opacity, opacity_late, world_size_frac, screen_size;
  int32_t size_prune_from, densify_until, use_vcp;
} sk_prune_params;
void sk_default_prune_params(sk_prune_params* out);
/* select_prune (adc.hpp:224-270); flags [n]. */
int sk_select_prune(sk_ctx* ctx, sk_scene* scene, int iteration, const sk_prune_params* params, float extent,
                    uint8_t* prune);
/* apply_prune (adc.hpp:273-289), then apply_densify (:167-205), with the Adam
 * moment remaps (adam.hpp:45-58), sequenced as Trainer::density_event
 * (trainer.hpp:203-233). Flags are host arrays over the pre-event indices
 * (any may be NULL); clone/split entries whose prune flag is set are dropped.
 * eps: 6 standard normals per split Gaussian in ascending index order (child
 * 0 then child 1), drawn by the caller's Rng. old_to_new ([n], the final
 * index of every original Gaussian or -1) and new_size may be NULL. The score
 * table is reset afterwards (trainer.hpp:241). */
int sk_apply_prune_densify(sk_ctx* ctx, sk_scene* scene, const uint8_t* prune, const uint8_t* clone,
                           const uint8_t* split, float clone_step_lr, const float* eps, int32_t* old_to_new,
                           int64_t* new_size);

/* ---- training (trainer.hpp, config.hpp) ------------------------------------ */
/* TrainConfig (config.hpp:20-61); bin_mode "compact" <=> compact != 0. */
typedef struct sk_train_config {
  int32_t iterations, k;
  double lambda, tau, tau_d, tau_p, beta, tau_alpha;
  int32_t densify_from, densify_until, densify_every, prune_every_early, prune_every_late;
  double grad_threshold, percent_dense;
  double lr_position, lr_position_final, lr_sh_dc, lr_sh_rest, lr_opacity, lr_scale, lr_rotation;
  int32_t opacity_reset_every, lazy_opt_enabled, lazy_opt_interval_15k, lazy_opt_interval_20k;
  uint64_t seed;
  int32_t tile_size, workers, sh_degree, compact, vcd, vcp;
  double prune_min_opacity, prune_opacity_late, prune_world_size_frac, prune_screen_size;
  int32_t size_prune_from, schedule_dry_run;
} sk_train_config;
void sk_default_config(sk_train_config* out);
/* set_config_value (config.hpp:139-163): one `key = value` pair with the
 * reference's key names ("bin_mode" = aabb|compact sets `compact`); unknown
 * keys raise "config: unknown key '<key>'". ctx may be NULL. */
int sk_config_set(sk_ctx* ctx, sk_train_config* cfg, const char* key, const char* value);
/* load_config_file (config.hpp:167-196): flat key = value lines, '#' comments. */
int sk_config_load_file(sk_ctx* ctx, sk_train_config* cfg, const char* path);
/* TrainConfig::validate (config.hpp:63-80), same messages. */
int sk_validate_config(sk_ctx* ctx, const sk_train_config* cfg);

/* LogRow (trainer.hpp:21-28) plus the view drawn and an event flag. */
typedef struct sk_log_row {
  int32_t iteration, gaussians;
  int64_t tile_pairs;
  double loss, psnr, elapsed_ms;
  int32_t view, event; /* event: bit0 densify, bit1 prune */
} sk_log_row;

/* Dataset<T> (dataset.hpp:24-32): cameras + 8-bit GT images resident in HBM.
 * images: n_views images, each [H_v][W_v][3] u8, concatenated in view order. */
typedef struct sk_dataset sk_dataset;
int sk_dataset_create(sk_ctx* ctx, int n_views, const sk_camera* cams, const uint8_t* images,
                      const int32_t* train_indices, int n_train, float extent, sk_dataset** out);
int sk_dataset_destroy(sk_dataset* d);
int sk_dataset_num_views(const sk_dataset* d, int* n);
int sk_dataset_camera(const sk_dataset* d, int view, sk_camera* out);
/* Copies view `view`'s 8-bit GT image ([H][W][3]) to host memory. */
int sk_dataset_image_u8(sk_ctx* ctx, const sk_dataset* d, int view, uint8_t* out);
/* Train split (every 8th view is a test view, dataset.hpp:44-53). out may be
 * NULL to query the count. */
int sk_dataset_train_indices(const sk_dataset* d, int32_t* out, int* count);
int sk_dataset_extent(const sk_dataset* d, float* extent);
int sk_dataset_set_train_indices(sk_dataset* d, const int32_t* idx, int count);

/* ---- scene construction on the device ----------------- */
/* SynthSpec of generate_synthetic (dataset.hpp:178-250). width == height and
 * scale_mult = 1, focal <= 0 reproduce the reference generator; the
 * non-square size, (500/N)^(1/3) scale multiplier and focal override are the
 * large-config extensions of SURVEY §8(d). */
typedef struct sk_synth_spec {
  int32_t n_gaussians, n_views, width, height;
  uint64_t seed;
  double scale_mult;
  double focal; /* <= 0: 1.1 * height */
} sk_synth_spec;
/* generate_synthetic: GT Gaussians drawn with the reference Rng on the host
 * (same draw order), camera ring, every GT view rendered by K1-K6 on the GPU
 * and quantised through 8 bits into the dataset (device-resident), then the
 * init point cloud (GT mu + noise, DC colour) and the scene extent.
 * gt_out (SH degree 1), init_xyz / init_rgb ([n][3]) and extent_out may be
 * NULL. */
int sk_synthetic_create(sk_ctx* ctx, const sk_synth_spec* spec, sk_scene** gt_out, sk_dataset** data_out,
                        float* init_xyz, float* init_rgb, float* extent_out);
/* init_from_points (scene.hpp:117-141): log of the mean distance to the three
 * nearest neighbours as isotropic log-scale, identity rotation, opacity
 * logit(0.1), DC from the point colour, higher SH zero. Raises
 * "init_from_points: empty point cloud" for n == 0. */
int sk_init_from_points(sk_ctx* ctx, int64_t n, const float* xyz, const float* rgb, int sh_degree, int64_t capacity,
                        sk_scene** out);

/* ---- on-disk formats ----------------------------------
 * Host-side file I/O. ctx may be NULL for the pure file functions (points,
 * PNG, cameras.json); errors are then reported by status only. */
/* save_checkpoint (ply.hpp:217-248): binary little-endian PLY, float32 rows
 * x y z nx ny nz f_dc_0..2 f_rest_* (channel-major) opacity scale_0..2
 * rot_0..3. The planar device scene is gathered into rows on the GPU. */
int sk_checkpoint_save(sk_ctx* ctx, const sk_scene* scene, const char* path);
/* load_checkpoint (ply.hpp:251-315): SH degree from the f_rest count; missing
 * fields raise "checkpoint: missing property '<name>'". */
int sk_checkpoint_load(sk_ctx* ctx, const char* path, int64_t capacity, sk_scene** out);
/* read_points_ply (ply.hpp:179-196): xyz / rgb [count][3]; colours rescaled
 * by 1/255 when integer-typed. Pass xyz = rgb = NULL to query *count; else
 * *count is the buffer capacity on entry and the point count on return. */
int sk_points_read(sk_ctx* ctx, const char* path, float* xyz, float* rgb, int64_t* count);
/* write_points_ply (ply.hpp:198-212): float xyz + uchar rgb (lround). */
int sk_points_write(sk_ctx* ctx, const char* path, const float* xyz, const float* rgb, int64_t n);
/* read_png (png_io.cpp:25-72) as 8-bit RGB [H][W][3] (the reference's float
 * image is byte / 255.0f). rgb = NULL queries *width / *height. */
int sk_png_read(sk_ctx* ctx, const char* path, uint8_t* rgb, int* width, int* height);
/* write_png (png_io.cpp:74-104): lround(clamp(v, 0, 1) * 255) per channel. */
int sk_png_write(sk_ctx* ctx, const char* path, const float* rgb, int width, int height);
int sk_png_write_u8(sk_ctx* ctx, const char* path, const uint8_t* rgb, int width, int height);
/* cameras.json records (dataset.hpp:80-100, 127-150). cams = NULL queries
 * *count; cameras are validated (Camera::validate camera.hpp:34-42). */
int sk_cameras_read(sk_ctx* ctx, const char* path, sk_camera* cams, int32_t* ids, int* count);
int sk_cameras_write(sk_ctx* ctx, const char* path, const sk_camera* cams, const int32_t* ids, int n);
/* load_dataset (dataset.hpp:73-125): cameras.json, images/%05d.png and
 * points3d.ply into a device-resident dataset; every-8th test split; extent =
 * 1.1 x the radius around the mean camera centre. */
int sk_dataset_load(sk_ctx* ctx, const char* dir, sk_dataset** out);
/* Init point cloud of a loaded or synthetic dataset (Dataset::init_points). */
int sk_dataset_init_points(const sk_dataset* d, float* xyz, float* rgb, int64_t* count);
/* The files generate_synthetic writes (dataset.hpp:221-247): cameras.json,
 * images/%05d.png (device images, 8-bit) and points3d.ply. */
int sk_dataset_save(sk_ctx* ctx, const sk_dataset* d, const char* dir);

typedef struct sk_trainer sk_trainer;
/* Trainer(scene, data, cfg) (trainer.hpp:70-87). The trainer borrows scene and
 * dataset; both must outlive it. */
int sk_trainer_create(sk_ctx* ctx, sk_scene* scene, const sk_dataset* data, const sk_train_config* cfg,
                      sk_trainer** out);
int sk_trainer_destroy(sk_trainer* t);
/* Trainer::run (trainer.hpp:89-119) for `iterations` more iterations (clamped
 * to cfg.iterations); rows may be NULL. */
int sk_trainer_run(sk_trainer* t, int iterations, sk_log_row* rows);
int sk_trainer_iteration(const sk_trainer* t, int* it);
/* Resumes the schedule at iteration `it` (the next run() trains it + 1). */
int sk_trainer_set_iteration(sk_trainer* t, int it);
/* Trainer::density_event (trainer.hpp:177-243) now, outside the schedule:
 * samples cfg.k training views, scores, selects and compacts. */
int sk_trainer_density_event(sk_trainer* t, int iteration, int densify, int prune);
/* Density-event records (for parity checks): header [7] = iteration,
 * n_before, n_after, n_clone, n_split, n_prune, k; flags are [n_before] u8. */
int sk_trainer_record_events(sk_trainer* t, int on);
int sk_trainer_num_events(const sk_trainer* t, int* n);
int sk_trainer_event(const sk_trainer* t, int e, int32_t* header, uint8_t* clone, uint8_t* split, uint8_t* prune,
                     int32_t* sampled, float* photometric);

/* ---- multi-GPU view sharding over NCCL ------------------------
 * One process per GPU. Rank 0 creates the id and shares it (e.g. through
 * torch.distributed); every rank creates its communicator. A trainer with a
 * communicator of R ranks trains R views per step (one per rank, drawn from
 * the shared Rng in rank order), sums gradients before Adam (C1), reduces the
 * ScoreTable statistics at events (C2) and shards the K scored views
 * round-robin (C3); selection and compaction run identically on all ranks. */
#define SK_COMM_ID_BYTES 128
typedef struct sk_comm sk_comm;
int sk_comm_unique_id(uint8_t* id /* [SK_COMM_ID_BYTES] */);
int sk_comm_create(sk_ctx* ctx, const uint8_t* id, int nranks, int rank, sk_comm** out);
/* Host-callback collectives: the library stages its device buffers through
 * pinned host memory and calls these (e.g. torch.distributed over gloo, MPI),
 * so the same C1 / C2 / C3 code runs without NCCL (and with several ranks on
 * one GPU). Buffers are host pointers; dtype SK_DT_*, op SK_OP_*; each
 * returns 0 on success. reduce_scatter: send holds world * count elements
 * (rank-major), recv gets this rank's reduced count; all_gather: send holds
 * count elements, recv world * count (rank-major). */
#define SK_DT_F32 0
#define SK_DT_I32 1
#define SK_OP_SUM 0
#define SK_OP_MAX 1
typedef struct sk_comm_host_ops {
  void* user;
  int (*all_reduce)(void* user, void* buf, int64_t count, int dtype, int op);
  int (*reduce_scatter)(void* user, const void* send, void* recv, int64_t count, int dtype, int op);
  int (*all_gather)(void* user, const void* send, void* recv, int64_t count, int dtype);
} sk_comm_host_ops;
int sk_comm_create_host(sk_ctx* ctx, int nranks, int rank, const sk_comm_host_ops* ops, sk_comm** out);
int sk_comm_destroy(sk_comm* comm);
int sk_comm_rank(const sk_comm* comm, int* rank, int* world);
int sk_trainer_set_comm(sk_trainer* t, sk_comm* comm);
/* Round-robin ownership of n_items among world ranks (the score-pass
 * sharding): fills owned[] (may be NULL) and *n_owned. */
int sk_shard_assign(int n_items, int world, int rank, int32_t* owned, int* n_owned);

/* One train_iteration (trainer.hpp:124-175) on an explicit camera with the
 * GT image in HOST memory (copied in) — the end-to-end entry point. */
int sk_train_step_host(sk_ctx* ctx, sk_scene* scene, sk_frame* frame, const sk_camera* cam, const uint8_t* gt_host,
                       const sk_train_config* cfg, float extent, int iteration, sk_log_row* row);
/* The reference Rng (rng.hpp:18-69, mt19937_64 + Box-Muller with a cached
 * spare) as the density event draws the split noise: successive chunks of
 * normal() values from one generator seeded with `seed`, written back to back
 * into out. The batched draw (uniforms in order, transcendentals on worker
 * threads) is bit-identical to sequential normal() calls. */
int sk_rng_normals(uint64_t seed, const int64_t* chunks, int n_chunks, float* out);

/* Pipelined variant for streaming inputs: the GT upload runs on a copy
 * stream into one of two device buffers (overlapping the previous step), and
 * `row` (loss / PSNR / pairs) is written when the step completes — during the
 * next call on this frame, or at sk_train_step_host_flush. `row` and
 * `gt_host` (pinned memory for a truly asynchronous copy) must stay valid
 * until then. Parameters and results are those of sk_train_step_host; with
 * a communicator (view-parallel steps) the gradients are summed
 * over its ranks before Adam (C1), as in sk_trainer_run. comm may be NULL. */
int sk_train_step_host_async(sk_ctx* ctx, sk_scene* scene, sk_frame* frame, const sk_camera* cam,
                             const uint8_t* gt_host, const sk_train_config* cfg, float extent, int iteration,
                             sk_log_row* row, const sk_comm* comm);
int sk_train_step_host_flush(sk_ctx* ctx, sk_frame* frame);

#ifdef __cplusplus
}
#endif

#endif /* SPLATKIT_B200_H_ */
