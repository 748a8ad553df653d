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

/* frame readback */
int sk_frame_num_projected(const sk_frame* frame, int64_t* n);
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
int sk_frame_get_dimage(sk_ctx* ctx, const sk_frame* frame, float* hwc);
int sk_frame_set_dimage(sk_ctx* ctx, sk_frame* frame, const float* hwc);

/* ---- backward (blend_backward raster.hpp:281-355) ---------------------- */
int sk_render_backward(sk_ctx* ctx, sk_frame* frame);
int sk_frame_get_blend_grads(sk_ctx* ctx, const sk_frame* frame, sk_blend_grads* out);

#ifdef __cplusplus
}
#endif

#endif /* SPLATKIT_B200_H_ */
