// C ABI (include/splatkit_b200.h): context, scene, frame, and the
// reference-facing functional entry points. Every function traps C++
// exceptions and maps them to status codes (no exception crosses the ABI).
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>

#include "abi_util.h"

namespace sk {

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

uint32_t read_error_word(sk_ctx* ctx) {
  uint32_t bits = 0;
  SK_CUDA(cudaMemcpyAsync(&bits, ctx->err_word.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (bits) SK_CUDA(cudaMemsetAsync(ctx->err_word.ptr, 0, sizeof(uint32_t), ctx->stream));
  return bits;
}

// Device error bits -> the reference's exception types and messages
// (scene.hpp:89-92, raster.hpp:116).
void raise_device_errors(uint32_t bits) {
  if (bits & kErrCovNonFinite) throw std::invalid_argument("covariance_3d: non-finite rotation or scale");
  if (bits & kErrCovNonPositive) throw std::invalid_argument("covariance_3d: scale must be positive");
  if (bits & kErrCompactNotPD) throw std::runtime_error("bin_compact: cov2d must be positive definite");
}

namespace {

void set_device(sk_ctx* ctx) { SK_CUDA(cudaSetDevice(ctx->device)); }

}  // namespace

// planar [3][H][W] device -> interleaved [H][W][3] host
void planar_to_hwc(sk_ctx* ctx, const void* dev, float* hwc, int w, int h) {
  const size_t plane = (size_t)w * h;
  std::vector<float> tmp(3 * plane);
  d2h(ctx, tmp.data(), dev, 3 * plane);
  sync(ctx);
  for (size_t p = 0; p < plane; ++p)
    for (int c = 0; c < 3; ++c) hwc[p * 3 + c] = tmp[c * plane + p];
}

void hwc_to_planar(sk_ctx* ctx, void* dev, const float* hwc, int w, int h) {
  const size_t plane = (size_t)w * h;
  std::vector<float> tmp(3 * plane);
  for (size_t p = 0; p < plane; ++p)
    for (int c = 0; c < 3; ++c) tmp[c * plane + p] = hwc[p * 3 + c];
  h2d(ctx, dev, tmp.data(), 3 * plane);
  sync(ctx);
}


}  // namespace sk

using namespace sk;

extern "C" {

const char* sk_version(void) { return "splatkit_b200 0.1 (sm_100a)"; }

int sk_ctx_create(int device, sk_ctx** out) {
  if (!out) return SK_ERR_INVALID_ARGUMENT;
  auto ctx = std::make_unique<sk_ctx>();
  ctx->device = device;
  const int rc = guarded(ctx.get(), [&] {
    int count = 0;
    SK_CUDA(cudaGetDeviceCount(&count));
    arg(device >= 0 && device < count, "sk_ctx_create: no such CUDA device");
    SK_CUDA(cudaSetDevice(device));
    SK_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
    ensure<uint32_t>(ctx->err_word, 4);
    SK_CUDA(cudaMemsetAsync(ctx->err_word.ptr, 0, 16, ctx->stream));
    SK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
  if (rc != SK_OK) {
    *out = nullptr;
    return rc;
  }
  *out = ctx.release();
  return SK_OK;
}

int sk_ctx_destroy(sk_ctx* ctx) {
  if (!ctx) return SK_OK;
  cudaSetDevice(ctx->device);
  if (ctx->helper) {
    delete ctx->helper_frame;
    sk_ctx_destroy(ctx->helper);
    ctx->helper = nullptr;
    ctx->helper_frame = nullptr;
  }
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->count_stream) {
    cudaStreamSynchronize(ctx->count_stream);
    cudaStreamDestroy(ctx->count_stream);
  }
  if (ctx->count_ev) cudaEventDestroy(ctx->count_ev);
  if (ctx->step_graph) cudaGraphExecDestroy(ctx->step_graph);
  if (ctx->capture_stream) cudaStreamDestroy(ctx->capture_stream);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return SK_OK;
}

const char* sk_last_error(const sk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int sk_ctx_set_stream(sk_ctx* ctx, void* stream) {
  return guarded(ctx, [&] {
    set_device(ctx);
    SK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->own_stream) SK_CUDA(cudaStreamDestroy(ctx->stream));
    ctx->stream = static_cast<cudaStream_t>(stream);
    ctx->own_stream = false;
  });
}

int sk_ctx_synchronize(sk_ctx* ctx) {
  return guarded(ctx, [&] {
    SK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_ctx_launch_count(const sk_ctx*, int64_t* out) {
  if (out) *out = g_launches.load();
  return SK_OK;
}

int sk_ctx_enable_timing(sk_ctx* ctx, int on) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (on && !ctx->tev[0][0]) {
      for (auto& set : ctx->tev)
        for (auto& e : set) SK_CUDA(cudaEventCreate(&e));
      for (auto& e : ctx->ev.tev) SK_CUDA(cudaEventCreate(&e));
      for (auto& e : ctx->ev.move_ev) SK_CUDA(cudaEventCreate(&e));
    }
    ctx->timing = on != 0;
  });
}

int sk_ctx_get_timing(const sk_ctx* ctx, double* ms, int64_t* steps) {
  if (!ctx) return SK_ERR_INVALID_ARGUMENT;
  if (ms)
    for (int i = 0; i < SK_NUM_PHASES; ++i) ms[i] = ctx->phase_ms[i];
  if (steps) *steps = ctx->timed_steps;
  return SK_OK;
}

int sk_ctx_get_event_timing(const sk_ctx* ctx, double* ms, int64_t* events) {
  if (!ctx) return SK_ERR_INVALID_ARGUMENT;
  if (ms)
    for (int i = 0; i < SK_NUM_EVENT_PHASES; ++i) ms[i] = ctx->ev.phase_ms[i];
  if (events) *events = ctx->ev.timed_events;
  return SK_OK;
}

int sk_ctx_get_compact_kernel_ms(const sk_ctx* ctx, double* move_ms) {
  if (!ctx || !move_ms) return SK_ERR_INVALID_ARGUMENT;
  *move_ms = ctx->ev.move_ms;
  return SK_OK;
}

int sk_ctx_graph_steps(const sk_ctx* ctx, int64_t* steps) {
  if (!ctx || !steps) return SK_ERR_INVALID_ARGUMENT;
  *steps = ctx->graph_steps;
  return SK_OK;
}

int sk_ctx_reset_timing(sk_ctx* ctx) {
  if (!ctx) return SK_ERR_INVALID_ARGUMENT;
  for (auto& v : ctx->phase_ms) v = 0.0;
  ctx->timed_steps = 0;
  for (auto& v : ctx->ev.phase_ms) v = 0.0;
  ctx->ev.timed_events = 0;
  ctx->ev.move_ms = 0.0;
  return SK_OK;
}

// ---- scene -----------------------------------------------------------------
int sk_scene_create(sk_ctx* ctx, int sh_degree, int64_t capacity, sk_scene** out) {
  return guarded(ctx, [&] {
    arg(out != nullptr, "sk_scene_create: null output");
    arg(sh_degree >= 0 && sh_degree <= 3, "config: sh_degree must be in 0..3");
    arg(capacity >= 0, "sk_scene_create: negative capacity");
    set_device(ctx);
    auto s = std::make_unique<sk_scene>();
    s->sh_degree = sh_degree;
    s->comps = SK_COMP_COUNT(sh_degree);
    s->capacity = round_capacity(capacity);
    ensure<float>(s->params, (size_t)s->comps * s->capacity);
    *out = s.release();
  });
}

int sk_scene_destroy(sk_scene* s) {
  delete s;
  return SK_OK;
}

int sk_scene_upload(sk_ctx* ctx, sk_scene* s, const float* host, int64_t n) {
  return guarded(ctx, [&] {
    arg(s && (host || n == 0) && n >= 0, "sk_scene_upload: bad arguments");
    set_device(ctx);
    if (n > s->capacity) {
      s->capacity = round_capacity(n);
      s->params.release();
    }
    float* p = ensure<float>(s->params, (size_t)s->comps * s->capacity);
    if (n > 0)
      SK_CUDA(cudaMemcpy2DAsync(p, sizeof(float) * s->capacity, host, sizeof(float) * n, sizeof(float) * n, s->comps,
                                cudaMemcpyHostToDevice, ctx->stream));
    s->n = n;
    for (auto& t : s->adam_t) t = 0;
    const size_t cells = (size_t)s->comps * s->capacity;
    if (s->adam_m.ptr && s->adam_m.bytes >= cells * sizeof(float)) {
      // same capacity: zero the moments / statistics in place instead of
      // freeing and re-allocating them (SceneOptimizer::init, ScoreTable::reset)
      SK_CUDA(cudaMemsetAsync(s->adam_m.ptr, 0, cells * sizeof(float), ctx->stream));
      SK_CUDA(cudaMemsetAsync(s->adam_v.ptr, 0, cells * sizeof(float), ctx->stream));
    } else {
      s->grads.release();
      s->adam_m.release();
      s->adam_v.release();
    }
    if (s->grad_norm_acc.ptr && s->grad_norm_acc.bytes >= (size_t)s->capacity * sizeof(float)) {
      reset_score_table(ctx, s);
    } else {
      for (DevBuf* b : {&s->s_d, &s->s_p_raw, &s->s_p, &s->grad_norm_acc, &s->abs_grad_acc, &s->grad3d_acc,
                        &s->views_seen, &s->max_radius2d})
        b->release();
    }
    s->rest_n = -1;
    s->moments_sharded_over = nullptr;  // fresh moments: nothing left to gather
    sync(ctx);
  });
}

int sk_scene_download(sk_ctx* ctx, const sk_scene* s, float* host) {
  return guarded(ctx, [&] {
    arg(s && host, "sk_scene_download: bad arguments");
    set_device(ctx);
    if (s->n > 0)
      SK_CUDA(cudaMemcpy2DAsync(host, sizeof(float) * s->n, s->params.ptr, sizeof(float) * s->capacity,
                                sizeof(float) * s->n, s->comps, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
  });
}

int sk_scene_size(const sk_scene* s, int64_t* n) {
  if (!s || !n) return SK_ERR_INVALID_ARGUMENT;
  *n = s->n;
  return SK_OK;
}

int sk_scene_sh_degree(const sk_scene* s, int* deg) {
  if (!s || !deg) return SK_ERR_INVALID_ARGUMENT;
  *deg = s->sh_degree;
  return SK_OK;
}

int sk_scene_device_params(const sk_scene* s, float** params, int64_t* stride) {
  if (!s) return SK_ERR_INVALID_ARGUMENT;
  if (params) *params = s->params.as<float>();
  if (stride) *stride = s->capacity;
  return SK_OK;
}

// ---- frame -------------------------------------------------------------------
int sk_frame_create(sk_ctx* ctx, sk_frame** out) {
  return guarded(ctx, [&] {
    arg(out != nullptr, "sk_frame_create: null output");
    *out = new sk_frame();
  });
}

int sk_frame_destroy(sk_frame* f) {
  delete f;
  return SK_OK;
}

int sk_preprocess(sk_ctx* ctx, const sk_scene* s, const sk_camera* cam, const sk_binning* b, sk_frame* f) {
  return guarded(ctx, [&] {
    arg(s && cam && f, "sk_preprocess: bad arguments");
    arg(cam->fx > 0 && cam->fy > 0, "camera: focal lengths must be positive");
    set_device(ctx);
    frame_geometry(f, cam->width, cam->height, b);
    f->camera = *cam;
    ensure_projected(f, s->n);
    launch_preprocess(ctx, s, *cam, f);
    raise_device_errors(read_error_word(ctx));
  });
}

int sk_frame_set_projected(sk_ctx* ctx, sk_frame* f, const sk_projected* pg, int64_t n, int width, int height,
                           const sk_binning* b) {
  return guarded(ctx, [&] {
    arg(f && pg && n >= 0, "sk_frame_set_projected: bad arguments");
    arg(n == 0 || (pg->mu2d && pg->cov2d && pg->conic && pg->depth && pg->color && pg->opacity),
        "sk_frame_set_projected: missing arrays");
    set_device(ctx);
    frame_geometry(f, width, height, b);
    ensure_projected(f, n);
    f->extras_valid = true;  // the caller's covariances; tiles and a* from the injection kernel
    std::vector<float2> mu(n);
    std::vector<float4> co(n), rgb(n), cov(n), c4(n);
    for (int64_t i = 0; i < n; ++i) {
      mu[i] = make_float2(pg->mu2d[2 * i], pg->mu2d[2 * i + 1]);
      co[i] = make_float4(pg->conic[4 * i], pg->conic[4 * i + 1], pg->conic[4 * i + 3], pg->opacity[i]);
      rgb[i] = make_float4(pg->color[3 * i], pg->color[3 * i + 1], pg->color[3 * i + 2], pg->depth[i]);
      cov[i] = make_float4(pg->cov2d[4 * i], pg->cov2d[4 * i + 1], pg->cov2d[4 * i + 2], pg->cov2d[4 * i + 3]);
      c4[i] = make_float4(pg->conic[4 * i], pg->conic[4 * i + 1], pg->conic[4 * i + 2], pg->conic[4 * i + 3]);
    }
    if (n > 0) {
      h2d(ctx, f->mean2d.ptr, mu.data(), n);
      h2d(ctx, f->conic_op.ptr, co.data(), n);
      h2d(ctx, f->rgb_depth.ptr, rgb.data(), n);
      h2d(ctx, f->cov2d.ptr, cov.data(), n);
      h2d(ctx, f->conic4.ptr, c4.data(), n);
    }
    launch_inject_bin(ctx, f);
    raise_device_errors(read_error_word(ctx));
  });
}

// A caller's TileGrid (raster.hpp:27-57) as the frame's tile lists: ranges
// [tiles][2] into values [pairs] (projected indices); blend_forward then
// blends exactly these lists in their order, as the reference does.
int sk_frame_set_tile_lists(sk_ctx* ctx, sk_frame* f, const int32_t* ranges, const int32_t* values, int64_t pairs) {
  return guarded(ctx, [&] {
    arg(f && ranges && (values || pairs == 0) && pairs >= 0, "sk_frame_set_tile_lists: bad arguments");
    set_device(ctx);
    const int tiles = f->tiles_x * f->tiles_y;
    int64_t expect = 0;
    for (int t = 0; t < tiles; ++t) {
      arg(ranges[2 * t] == expect && ranges[2 * t + 1] >= ranges[2 * t],
          "sk_frame_set_tile_lists: ranges must be contiguous in tile order");
      expect = ranges[2 * t + 1];
    }
    arg(expect == pairs, "sk_frame_set_tile_lists: ranges do not cover the values");
    for (int64_t k = 0; k < pairs; ++k)
      arg(values[k] >= 0 && values[k] < f->n, "sk_frame_set_tile_lists: projected index out of range");
    ensure<int2>(f->ranges, (size_t)std::max(tiles, 1));
    if (tiles > 0) h2d(ctx, f->ranges.ptr, ranges, 2 * (size_t)tiles);
    const size_t pm = (size_t)std::max<int64_t>(pairs, 1);
    uint32_t* pv = ensure<uint32_t>(f->pval_a, pm);
    if (pairs > 0) h2d(ctx, pv, values, pairs);
    f->pair_val = pv;
    f->pairs = pairs;
    f->binned = true;
    f->rendered = false;
    f->cmask_valid = false;
    sync(ctx);
  });
}

// A caller's rendered image ([H][W][3]) as the frame's render, for
// training_loss (loss.hpp:21-47) on explicit images.
int sk_frame_set_image(sk_ctx* ctx, sk_frame* f, const float* hwc, int width, int height) {
  return guarded(ctx, [&] {
    arg(f && hwc, "sk_frame_set_image: bad arguments");
    set_device(ctx);
    frame_geometry(f, width, height, nullptr);
    ensure_image(f);
    hwc_to_planar(ctx, f->image.ptr, hwc, width, height);
    f->rendered = true;
  });
}

int sk_bin_sort(sk_ctx* ctx, sk_frame* f, int64_t* pairs) {
  return guarded(ctx, [&] {
    arg(f != nullptr, "sk_bin_sort: null frame");
    set_device(ctx);
    bin_sort(ctx, f);
    if (pairs) *pairs = f->pairs;
  });
}

int sk_render_forward(sk_ctx* ctx, sk_frame* f, const uint8_t* mask_host, int32_t* counts_host) {
  return guarded(ctx, [&] {
    arg(f != nullptr, "sk_render_forward: null frame");
    arg((mask_host == nullptr) == (counts_host == nullptr), "sk_render_forward: mask and counter go together");
    set_device(ctx);
    if (!f->binned) bin_sort(ctx, f);
    ensure_image(f);
    const size_t plane = (size_t)f->width * f->height;
    if (mask_host) {
      // blend_forward(grid, pgs, &mask, &counter): the image plus the K12 count pass
      uint8_t* m = ensure<uint8_t>(f->mask, plane);
      int32_t* c = ensure<int32_t>(f->counts, (size_t)std::max<int64_t>(f->n, 1));
      h2d(ctx, m, mask_host, plane);
      SK_CUDA(cudaMemsetAsync(c, 0, sizeof(int32_t) * f->n, ctx->stream));
      launch_blend_forward(ctx, f, nullptr, nullptr);
      launch_blend_forward(ctx, f, m, c);
      std::vector<int32_t> tmp(f->n);
      d2h(ctx, tmp.data(), c, f->n);
      sync(ctx);
      for (int64_t i = 0; i < f->n; ++i) counts_host[i] += tmp[i];
    } else {
      launch_blend_forward(ctx, f, nullptr, nullptr);
      sync(ctx);
    }
    f->rendered = true;
  });
}

int sk_frame_num_projected(const sk_frame* f, int64_t* n) {
  if (!f || !n) return SK_ERR_INVALID_ARGUMENT;
  *n = f->n;
  return SK_OK;
}

int sk_frame_dims(const sk_frame* f, int* w, int* h) {
  if (!f) return SK_ERR_INVALID_ARGUMENT;
  if (w) *w = f->width;
  if (h) *h = f->height;
  return SK_OK;
}

int sk_frame_get_projected(sk_ctx* ctx, const sk_frame* f, sk_projected* out) {
  return guarded(ctx, [&] {
    arg(f && out, "sk_frame_get_projected: bad arguments");
    arg(f->extras_valid || f->n == 0,
        "sk_frame_get_projected: the frame was last projected by a training step (no covariance / tile counts); "
        "run sk_preprocess on it first");
    set_device(ctx);
    const int64_t n = f->n;
    std::vector<float2> mu(n);
    std::vector<float4> rgb(n), cov(n), c4(n), co(n);
    std::vector<float> rad(n);
    std::vector<int> tiles(n);
    if (n > 0) {
      d2h(ctx, mu.data(), f->mean2d.ptr, n);
      d2h(ctx, rgb.data(), f->rgb_depth.ptr, n);
      d2h(ctx, cov.data(), f->cov2d.ptr, n);
      d2h(ctx, c4.data(), f->conic4.ptr, n);
      d2h(ctx, co.data(), f->conic_op.ptr, n);
      d2h(ctx, rad.data(), f->radius.ptr, n);
      d2h(ctx, tiles.data(), f->tiles.ptr, n);
    }
    sync(ctx);
    for (int64_t i = 0; i < n; ++i) {
      const bool vis = rad[i] > 0.0f;
      if (out->visible) out->visible[i] = vis ? 1 : 0;
      if (out->tiles_touched) out->tiles_touched[i] = tiles[i];
      if (!vis) continue;
      if (out->mu2d) {
        out->mu2d[2 * i] = mu[i].x;
        out->mu2d[2 * i + 1] = mu[i].y;
      }
      if (out->cov2d) {
        out->cov2d[4 * i] = cov[i].x;
        out->cov2d[4 * i + 1] = cov[i].y;
        out->cov2d[4 * i + 2] = cov[i].z;
        out->cov2d[4 * i + 3] = cov[i].w;
      }
      if (out->conic) {
        out->conic[4 * i] = c4[i].x;
        out->conic[4 * i + 1] = c4[i].y;
        out->conic[4 * i + 2] = c4[i].z;
        out->conic[4 * i + 3] = c4[i].w;
      }
      if (out->depth) out->depth[i] = rgb[i].w;
      if (out->color) {
        out->color[3 * i] = rgb[i].x;
        out->color[3 * i + 1] = rgb[i].y;
        out->color[3 * i + 2] = rgb[i].z;
      }
      if (out->opacity) out->opacity[i] = co[i].w;
    }
  });
}

int sk_frame_get_image(sk_ctx* ctx, const sk_frame* f, float* hwc) {
  return guarded(ctx, [&] {
    arg(f && hwc && f->rendered, "sk_frame_get_image: frame not rendered");
    set_device(ctx);
    planar_to_hwc(ctx, f->image.ptr, hwc, f->width, f->height);
  });
}

int sk_frame_pge_counts(sk_ctx* ctx, sk_frame* f, int64_t* visited, int64_t* contributing) {
  return guarded(ctx, [&] {
    arg(f && visited && contributing && f->rendered, "sk_frame_pge_counts: frame not rendered");
    set_device(ctx);
    frame_pge_counts(ctx, f, visited, contributing);
  });
}

int sk_frame_get_transmittance(sk_ctx* ctx, const sk_frame* f, float* hw) {
  return guarded(ctx, [&] {
    arg(f && hw && f->rendered, "sk_frame_get_transmittance: frame not rendered");
    set_device(ctx);
    d2h(ctx, hw, f->final_t.ptr, (size_t)f->width * f->height);
    sync(ctx);
  });
}

int sk_frame_get_contrib_count(sk_ctx* ctx, const sk_frame* f, int32_t* hw) {
  return guarded(ctx, [&] {
    arg(f && hw && f->rendered, "sk_frame_get_contrib_count: frame not rendered");
    set_device(ctx);
    d2h(ctx, hw, f->n_contrib.ptr, (size_t)f->width * f->height);
    sync(ctx);
  });
}

int sk_frame_num_tiles(const sk_frame* f, int* tx, int* ty) {
  if (!f) return SK_ERR_INVALID_ARGUMENT;
  if (tx) *tx = f->tiles_x;
  if (ty) *ty = f->tiles_y;
  return SK_OK;
}

int sk_frame_get_tile_lists(sk_ctx* ctx, const sk_frame* f, int32_t* ranges, int32_t* values) {
  return guarded(ctx, [&] {
    arg(f && f->binned, "sk_frame_get_tile_lists: frame not binned");
    set_device(ctx);
    if (ranges) d2h(ctx, ranges, f->ranges.ptr, 2 * (size_t)f->tiles_x * f->tiles_y);
    if (values && f->pairs > 0) d2h(ctx, values, f->pair_val, (size_t)f->pairs);
    sync(ctx);
  });
}

// ---- loss ----------------------------------------------------------------------
static int loss_common(sk_ctx* ctx, sk_frame* f, const void* gt_host, bool u8, float lambda, sk_loss_values* out) {
  return guarded(ctx, [&] {
    arg(f && gt_host && f->rendered, "training_loss: frame not rendered");
    arg(lambda >= 0.0f && lambda <= 1.0f, "config: lambda must be in [0,1]");
    set_device(ctx);
    const size_t plane = (size_t)f->width * f->height;
    const size_t bytes = plane * 3 * (u8 ? 1 : sizeof(float));
    void* gt = f->gt.ensure(bytes);
    SK_CUDA(cudaMemcpyAsync(gt, gt_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    LossSums sums{};
    launch_loss(ctx, f, gt, u8, lambda, true, &sums);
    if (out) finish_loss(f->width, f->height, lambda, sums, out);
  });
}

int sk_loss(sk_ctx* ctx, sk_frame* f, const float* gt, float lambda, sk_loss_values* out) {
  return loss_common(ctx, f, gt, false, lambda, out);
}

int sk_loss_u8(sk_ctx* ctx, sk_frame* f, const uint8_t* gt, float lambda, sk_loss_values* out) {
  return loss_common(ctx, f, gt, true, lambda, out);
}

int sk_ssim(sk_ctx* ctx, const float* a, const float* b, int w, int h, double* ssim_out, double* psnr_out) {
  return guarded(ctx, [&] {
    arg(a && b && w > 0 && h > 0, "ssim: image dimensions differ");
    set_device(ctx);
    sk_frame tmp;
    tmp.width = w;
    tmp.height = h;
    ensure<float>(tmp.image, 3 * (size_t)w * h);
    hwc_to_planar(ctx, tmp.image.ptr, a, w, h);
    void* gt = tmp.gt.ensure(sizeof(float) * 3 * (size_t)w * h);
    h2d(ctx, gt, b, 3 * (size_t)w * h);
    LossSums sums{};
    launch_loss(ctx, &tmp, gt, false, 0.0f, false, &sums);
    sk_loss_values v{};
    finish_loss(w, h, 0.0f, sums, &v);
    if (ssim_out) *ssim_out = v.ssim;
    if (psnr_out) *psnr_out = v.psnr;
  });
}

int sk_frame_get_dimage(sk_ctx* ctx, const sk_frame* f, float* hwc) {
  return guarded(ctx, [&] {
    arg(f && hwc && f->dimage.ptr, "sk_frame_get_dimage: no gradient image");
    set_device(ctx);
    planar_to_hwc(ctx, f->dimage.ptr, hwc, f->width, f->height);
  });
}

int sk_frame_set_dimage(sk_ctx* ctx, sk_frame* f, const float* hwc) {
  return guarded(ctx, [&] {
    arg(f && hwc, "sk_frame_set_dimage: bad arguments");
    set_device(ctx);
    ensure<float>(f->dimage, 3 * (size_t)f->width * f->height);
    hwc_to_planar(ctx, f->dimage.ptr, hwc, f->width, f->height);
  });
}

// ---- backward ---------------------------------------------------------------------
int sk_render_backward(sk_ctx* ctx, sk_frame* f) {
  return guarded(ctx, [&] {
    arg(f && f->rendered && f->dimage.ptr, "blend_backward: frame needs a forward render and dL/dimage");
    set_device(ctx);
    ensure<float>(f->bgrads, (size_t)kBGradFields * std::max<int64_t>(f->n, 1));
    launch_blend_backward(ctx, f);
    sync(ctx);
  });
}

int sk_frame_get_blend_grads(sk_ctx* ctx, const sk_frame* f, sk_blend_grads* out) {
  return guarded(ctx, [&] {
    arg(f && out && f->bgrads.ptr, "sk_frame_get_blend_grads: no gradients");
    set_device(ctx);
    const int64_t n = f->n;
    std::vector<float> g((size_t)kBGradFields * n);
    d2h(ctx, g.data(), f->bgrads.ptr, g.size());
    sync(ctx);
    auto F = [&](int field, int64_t i) { return g[(size_t)field * n + i]; };
    for (int64_t i = 0; i < n; ++i) {
      if (out->d_mu2d) {
        out->d_mu2d[2 * i] = F(0, i);
        out->d_mu2d[2 * i + 1] = F(1, i);
      }
      if (out->d_conic) {
        out->d_conic[4 * i] = F(2, i);
        out->d_conic[4 * i + 1] = F(3, i);
        out->d_conic[4 * i + 2] = F(3, i);
        out->d_conic[4 * i + 3] = F(4, i);
      }
      if (out->d_color) {
        out->d_color[3 * i] = F(5, i);
        out->d_color[3 * i + 1] = F(6, i);
        out->d_color[3 * i + 2] = F(7, i);
      }
      if (out->d_opacity) out->d_opacity[i] = F(8, i);
      if (out->abs_grad) {
        out->abs_grad[2 * i] = F(9, i);
        out->abs_grad[2 * i + 1] = F(10, i);
      }
    }
  });
}

}  // extern "C"
