// TEST INFRASTRUCTURE ONLY — extern "C" surface of the CPU oracle for ctypes
// (tests/, __graft_entry__.smoke(), bench.py cpu_baseline / --impl reference).
// Every function instantiates the restated reference code in splat_oracle.hpp.
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "../include/splatkit_b200.h"
#include "splat_oracle.hpp"

using namespace oracle;

namespace {

thread_local std::string g_err;
// pixel-Gaussian evaluations visited by the last or_render_* call (RenderOutputs::pge_visited)
thread_local int64_t g_pge_visited = 0;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SK_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SK_ERR_RUNTIME;
  }
}

template <typename T>
Camera<T> to_camera(const sk_camera* c) {
  Camera<T> cam;
  cam.width = c->width;
  cam.height = c->height;
  cam.fx = T(c->fx);
  cam.fy = T(c->fy);
  cam.cx = T(c->cx);
  cam.cy = T(c->cy);
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) cam.world_to_cam(r, k) = T(c->world_to_cam[r * 4 + k]);
  cam.near = T(c->near_plane);
  return cam;
}

template <typename T>
BinningConfig<T> to_binning(const sk_binning* b) {
  BinningConfig<T> cfg;
  if (b) {
    cfg.mode = b->mode == 1 ? BinMode::kCompact : BinMode::kAabb;
    cfg.beta = T(b->beta);
    cfg.tau_alpha = T(b->tau_alpha);
  }
  return cfg;
}

inline int tile_size_of(const sk_binning* b) { return b ? b->tile_size : 16; }

// planar [C][n] (SK_COMP_*) <-> Scene<T>
template <typename T>
Scene<T> scene_from_planar(const T* p, int64_t n, int deg) {
  Scene<T> s;
  s.sh_degree = deg;
  const int nsh = sh_coeff_count(deg);
  s.gaussians.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    auto& g = s.gaussians[i];
    for (int d = 0; d < 3; ++d) g.mu[d] = p[(SK_COMP_MU + d) * n + i];
    for (int d = 0; d < 4; ++d) g.rot[d] = p[(SK_COMP_ROT + d) * n + i];
    for (int d = 0; d < 3; ++d) g.log_scale[d] = p[(SK_COMP_LOG_SCALE + d) * n + i];
    g.opacity_logit = p[SK_COMP_OPACITY * n + i];
    g.sh = ShMatrix<T>(nsh);
    for (int k = 0; k < nsh; ++k)
      for (int c = 0; c < 3; ++c) g.sh(k, c) = p[(SK_COMP_SH + 3 * k + c) * n + i];
  }
  return s;
}

template <typename T>
void scene_to_planar(const Scene<T>& s, T* p) {
  const int64_t n = s.size();
  const int nsh = sh_coeff_count(s.sh_degree);
  for (int64_t i = 0; i < n; ++i) {
    const auto& g = s.gaussians[i];
    for (int d = 0; d < 3; ++d) p[(SK_COMP_MU + d) * n + i] = g.mu[d];
    for (int d = 0; d < 4; ++d) p[(SK_COMP_ROT + d) * n + i] = g.rot[d];
    for (int d = 0; d < 3; ++d) p[(SK_COMP_LOG_SCALE + d) * n + i] = g.log_scale[d];
    p[SK_COMP_OPACITY * n + i] = g.opacity_logit;
    for (int k = 0; k < nsh; ++k)
      for (int c = 0; c < 3; ++c) p[(SK_COMP_SH + 3 * k + c) * n + i] = g.sh(k, c);
  }
}

template <typename T>
Image<T> image_from(const T* hwc, int w, int h) {
  Image<T> img(w, h);
  for (size_t i = 0; i < img.pixels.size(); ++i)
    for (int c = 0; c < 3; ++c) img.pixels[i][c] = hwc[i * 3 + c];
  return img;
}

template <typename T>
void image_to(const Image<T>& img, T* hwc) {
  for (size_t i = 0; i < img.pixels.size(); ++i)
    for (int c = 0; c < 3; ++c) hwc[i * 3 + c] = img.pixels[i][c];
}

// Projected Gaussians passed across the oracle ABI: n entries in projected
// order. cov2d/conic row-major 2x2. source may be NULL (then source = i).
template <typename T>
struct PgIn {
  const T* mu2d;
  const T* cov2d;
  const T* conic;
  const T* depth;
  const T* color;
  const T* opacity;
};

template <typename T>
std::vector<ProjectedGaussian<T>> pgs_from(const PgIn<T>& in, int64_t n) {
  std::vector<ProjectedGaussian<T>> pgs(n);
  for (int64_t i = 0; i < n; ++i) {
    auto& pg = pgs[i];
    pg.mu2d[0] = in.mu2d[2 * i];
    pg.mu2d[1] = in.mu2d[2 * i + 1];
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) {
        pg.cov2d(r, c) = in.cov2d[4 * i + 2 * r + c];
        pg.cov2d_inv(r, c) = in.conic[4 * i + 2 * r + c];
      }
    pg.depth = in.depth[i];
    for (int c = 0; c < 3; ++c) pg.color[c] = in.color[3 * i + c];
    pg.opacity = in.opacity[i];
    pg.source_index = int(i);
  }
  return pgs;
}

// Render outputs for ctypes: any pointer may be NULL.
template <typename T>
struct RenderOut {
  T* image;           // [H][W][3]
  T* transmittance;   // [H][W]
  int32_t* contrib;   // [H][W]
  int32_t* ranges;    // [tiles][2]
  int32_t* values;    // [cap] tile-list entries as SOURCE indices
  int64_t values_cap;
  int64_t* pairs;
};

template <typename T>
void write_render(const TileGrid& grid, const std::vector<ProjectedGaussian<T>>& pgs, const RenderOutputs<T>& out,
                  const RenderOut<T>& o) {
  const int w = grid.width, h = grid.height;
  if (o.image) image_to(out.image, o.image);
  if (o.transmittance)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) o.transmittance[size_t(y) * w + x] = out.transmittance(y, x);
  if (o.contrib)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) o.contrib[size_t(y) * w + x] = out.contrib_count(y, x);
  const int64_t pairs = count_pairs(grid);
  if (o.pairs) *o.pairs = pairs;
  if (o.ranges || o.values) {
    int64_t off = 0;
    for (int t = 0; t < grid.tile_count(); ++t) {
      const auto& list = grid.tiles[t];
      if (o.ranges) {
        o.ranges[2 * t] = int32_t(off);
        o.ranges[2 * t + 1] = int32_t(off + list.size());
      }
      for (const int idx : list) {
        if (o.values && off < o.values_cap) o.values[off] = pgs[idx].source_index;
        ++off;
      }
    }
  }
}

template <typename T>
struct GradOut {
  T* d_mu2d;     // [n][2]
  T* d_conic;    // [n][4]
  T* d_color;    // [n][3]
  T* d_opacity;  // [n]
  T* abs_grad;   // [n][2]
};

template <typename T>
void write_grads(const BlendGrads<T>& g, const GradOut<T>& o) {
  for (size_t i = 0; i < g.d_mu2d.size(); ++i) {
    for (int d = 0; d < 2; ++d) {
      if (o.d_mu2d) o.d_mu2d[2 * i + d] = g.d_mu2d[i][d];
      if (o.abs_grad) o.abs_grad[2 * i + d] = g.abs_grad[i][d];
    }
    if (o.d_conic)
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) o.d_conic[4 * i + 2 * r + c] = g.d_conic[i](r, c);
    if (o.d_color)
      for (int c = 0; c < 3; ++c) o.d_color[3 * i + c] = g.d_color[i][c];
    if (o.d_opacity) o.d_opacity[i] = g.d_opacity[i];
  }
}

MaskMap mask_from(const uint8_t* m, int w, int h) {
  MaskMap mask(h, w);
  for (size_t i = 0; i < mask.d.size(); ++i) mask.d[i] = m[i];
  return mask;
}

// ---- templated bodies ------------------------------------------------------

template <typename T>
int project_scene_t(const T* params, int64_t n, int deg, const sk_camera* c, const sk_binning* b,
                    int32_t* visible, T* mu2d, T* cov2d, T* conic, T* depth, T* color, T* opacity,
                    int32_t* tiles_touched) {
  return guard([&] {
    const Scene<T> s = scene_from_planar(params, n, deg);
    const Camera<T> cam = to_camera<T>(c);
    const BinningConfig<T> bin = to_binning<T>(b);
    const TileGrid grid = make_tile_grid(cam.width, cam.height, tile_size_of(b));
    for (int64_t i = 0; i < n; ++i) {
      auto pg = project(s.gaussians[i], cam, deg, int(i));
      if (visible) visible[i] = pg ? 1 : 0;
      if (!pg) {
        if (tiles_touched) tiles_touched[i] = 0;
        continue;
      }
      if (mu2d) {
        mu2d[2 * i] = pg->mu2d[0];
        mu2d[2 * i + 1] = pg->mu2d[1];
      }
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 2; ++k) {
          if (cov2d) cov2d[4 * i + 2 * r + k] = pg->cov2d(r, k);
          if (conic) conic[4 * i + 2 * r + k] = pg->cov2d_inv(r, k);
        }
      if (depth) depth[i] = pg->depth;
      if (color)
        for (int k = 0; k < 3; ++k) color[3 * i + k] = pg->color[k];
      if (opacity) opacity[i] = pg->opacity;
      if (tiles_touched) tiles_touched[i] = int32_t(bin_one(*pg, grid, bin).size());
    }
  });
}

template <typename T>
int render_scene_t(const T* params, int64_t n, int deg, const sk_camera* c, const sk_binning* b, const uint8_t* mask,
                   int32_t* counts, int workers, const RenderOut<T>& o) {
  return guard([&] {
    const Scene<T> s = scene_from_planar(params, n, deg);
    const Camera<T> cam = to_camera<T>(c);
    const auto pgs = project_scene(s, cam);
    const TileGrid grid = build_tile_grid(pgs, cam.width, cam.height, to_binning<T>(b), tile_size_of(b));
    std::unique_ptr<MaskMap> mm;
    std::unique_ptr<FootprintCounter> fc;
    if (mask && counts) {
      mm = std::make_unique<MaskMap>(mask_from(mask, cam.width, cam.height));
      fc = std::make_unique<FootprintCounter>(int(n));
    }
    const auto out = blend_forward(grid, pgs, mm.get(), fc.get(), workers);
    if (fc)
      for (int64_t i = 0; i < n; ++i) counts[i] += fc->counts[i];
    g_pge_visited = out.pge_visited;
    write_render(grid, pgs, out, o);
  });
}

template <typename T>
int render_pg_t(const PgIn<T>& in, int64_t n, int w, int h, const sk_binning* b, const uint8_t* mask,
                int32_t* counts, int workers, const RenderOut<T>& o) {
  return guard([&] {
    const auto pgs = pgs_from(in, n);
    const TileGrid grid = build_tile_grid(pgs, w, h, to_binning<T>(b), tile_size_of(b));
    std::unique_ptr<MaskMap> mm;
    std::unique_ptr<FootprintCounter> fc;
    if (mask && counts) {
      mm = std::make_unique<MaskMap>(mask_from(mask, w, h));
      fc = std::make_unique<FootprintCounter>(int(n));
    }
    const auto out = blend_forward(grid, pgs, mm.get(), fc.get(), workers);
    if (fc)
      for (int64_t i = 0; i < n; ++i) counts[i] += fc->counts[i];
    g_pge_visited = out.pge_visited;
    write_render(grid, pgs, out, o);
  });
}

// Untiled brute-force renderer (tests/helpers.hpp:25-66): every Gaussian per
// pixel in global (depth, index) order, same cutoffs and expression order.
template <typename T>
int brute_render_pg_t(const PgIn<T>& in, int64_t n, int w, int h, const uint8_t* mask, int32_t* counts, T* image,
                      T* trans_out, int32_t* contrib) {
  return guard([&] {
    const auto pgs = pgs_from(in, n);
    const auto order = depth_order(pgs);
    for (int py = 0; py < h; ++py)
      for (int px = 0; px < w; ++px) {
        T trans = T(1);
        Vec3<T> c = Vec3<T>::zero();
        int cnt = 0;
        const bool masked = mask && mask[size_t(py) * w + px] != 0;
        for (const int idx : order) {
          const auto& pg = pgs[idx];
          const T dx = T(px) - pg.mu2d[0];
          const T dy = T(py) - pg.mu2d[1];
          const T q = pg.cov2d_inv(0, 0) * dx * dx + T(2) * pg.cov2d_inv(0, 1) * dx * dy + pg.cov2d_inv(1, 1) * dy * dy;
          if (q < T(0)) continue;
          const T alpha = min_ref(T(kAlphaCap), pg.opacity * ex(T(-0.5) * q));
          if (alpha < T(kAlphaMin)) continue;
          const T wgt = trans * alpha;
          for (int ch = 0; ch < 3; ++ch) c[ch] = c[ch] + wgt * pg.color[ch];
          ++cnt;
          if (masked && counts) ++counts[pg.source_index];
          trans = trans * (T(1) - alpha);
          if (trans < T(kTransmitMin)) break;
        }
        const size_t p = size_t(py) * w + px;
        if (image)
          for (int ch = 0; ch < 3; ++ch) image[p * 3 + ch] = c[ch];
        if (trans_out) trans_out[p] = trans;
        if (contrib) contrib[p] = cnt;
      }
  });
}

template <typename T>
int blend_backward_pg_t(const PgIn<T>& in, int64_t n, int w, int h, const sk_binning* b, const T* d_image,
                        int workers, const GradOut<T>& o) {
  return guard([&] {
    const auto pgs = pgs_from(in, n);
    const TileGrid grid = build_tile_grid(pgs, w, h, to_binning<T>(b), tile_size_of(b));
    const auto g = blend_backward(grid, pgs, image_from(d_image, w, h), workers);
    write_grads(g, o);
  });
}

template <typename T>
int training_loss_t(const T* r, const T* g, int w, int h, T lambda, T* loss, T* l1, T* ssim_v, T* d_image) {
  return guard([&] {
    const auto res = training_loss(image_from(r, w, h), image_from(g, w, h), lambda);
    if (loss) *loss = res.loss;
    if (l1) *l1 = res.l1;
    if (ssim_v) *ssim_v = res.ssim_value;
    if (d_image) image_to(res.d_image, d_image);
  });
}

// project_backward for every visible Gaussian of a scene, with upstream
// gradients indexed by SCENE index (d_conic: gradient on cov2d_inv, converted
// by cov_grad_from_inv_grad as the trainer does, trainer.hpp:141-146).
template <typename T>
int project_backward_t(const T* params, int64_t n, int deg, const sk_camera* c, const T* d_mu2d, const T* d_conic,
                       const T* d_color, const T* d_opacity, T* grads_planar) {
  return guard([&] {
    const Scene<T> s = scene_from_planar(params, n, deg);
    const Camera<T> cam = to_camera<T>(c);
    Scene<T> gs = s;  // reuse the planar writer for gradients
    for (auto& g : gs.gaussians) {
      g.mu = Vec3<T>::zero();
      g.rot = Vec4<T>::zero();
      g.log_scale = Vec3<T>::zero();
      g.opacity_logit = T(0);
      g.sh = ShMatrix<T>(g.sh.rows);
    }
    for (int64_t i = 0; i < n; ++i) {
      auto pg = project(s.gaussians[i], cam, deg, int(i));
      if (!pg) continue;
      Mat2<T> dinv;
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 2; ++k) dinv(r, k) = d_conic[4 * i + 2 * r + k];
      const Mat2<T> dcov = cov_grad_from_inv_grad(pg->cov2d_inv, dinv);
      Vec2<T> dm;
      dm[0] = d_mu2d[2 * i];
      dm[1] = d_mu2d[2 * i + 1];
      const auto g = project_backward(s.gaussians[i], cam, deg, dm, dcov, v3(d_color[3 * i], d_color[3 * i + 1], d_color[3 * i + 2]),
                                      d_opacity[i]);
      auto& o = gs.gaussians[i];
      o.mu = g.mu;
      o.rot = g.rot;
      o.log_scale = g.log_scale;
      o.opacity_logit = g.opacity_logit;
      o.sh = g.sh;
    }
    scene_to_planar(gs, grads_planar);
  });
}

}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }
int64_t or_last_pge_visited() { return g_pge_visited; }

// The reference Rng's normal() stream (rng.hpp:36-49), count draws cast to float.
int or_rng_normals(uint64_t seed, int64_t count, float* out) {
  Rng r(seed);
  for (int64_t k = 0; k < count; ++k) out[k] = static_cast<float>(r.normal());
  return 0;
}
void or_set_detmath(int on) { g_detmath = on != 0; }
float or_expf(float x) { return sk::det_expf(x); }
float or_logf(float x) { return sk::det_logf(x); }

// ---- projection --------------------------------------------------------------
int or_project_scene_f(const float* params, int64_t n, int deg, const sk_camera* cam, const sk_binning* bin,
                       int32_t* visible, float* mu2d, float* cov2d, float* conic, float* depth, float* color,
                       float* opacity, int32_t* tiles_touched) {
  return project_scene_t<float>(params, n, deg, cam, bin, visible, mu2d, cov2d, conic, depth, color, opacity,
                                tiles_touched);
}
int or_project_scene_d(const double* params, int64_t n, int deg, const sk_camera* cam, const sk_binning* bin,
                       int32_t* visible, double* mu2d, double* cov2d, double* conic, double* depth, double* color,
                       double* opacity, int32_t* tiles_touched) {
  return project_scene_t<double>(params, n, deg, cam, bin, visible, mu2d, cov2d, conic, depth, color, opacity,
                                 tiles_touched);
}

// ---- rendering -------------------------------------------------------------
int or_render_scene_f(const float* params, int64_t n, int deg, const sk_camera* cam, const sk_binning* bin,
                      const uint8_t* mask, int32_t* counts, int workers, float* image, float* trans, int32_t* contrib,
                      int32_t* ranges, int32_t* values, int64_t values_cap, int64_t* pairs) {
  return render_scene_t<float>(params, n, deg, cam, bin, mask, counts, workers,
                               {image, trans, contrib, ranges, values, values_cap, pairs});
}

int or_render_pg_f(const float* mu2d, const float* cov2d, const float* conic, const float* depth, const float* color,
                   const float* opacity, int64_t n, int w, int h, const sk_binning* bin, const uint8_t* mask,
                   int32_t* counts, int workers, float* image, float* trans, int32_t* contrib, int32_t* ranges,
                   int32_t* values, int64_t values_cap, int64_t* pairs) {
  return render_pg_t<float>({mu2d, cov2d, conic, depth, color, opacity}, n, w, h, bin, mask, counts, workers,
                            {image, trans, contrib, ranges, values, values_cap, pairs});
}
int or_render_pg_d(const double* mu2d, const double* cov2d, const double* conic, const double* depth,
                   const double* color, const double* opacity, int64_t n, int w, int h, const sk_binning* bin,
                   const uint8_t* mask, int32_t* counts, int workers, double* image, double* trans, int32_t* contrib,
                   int32_t* ranges, int32_t* values, int64_t values_cap, int64_t* pairs) {
  return render_pg_t<double>({mu2d, cov2d, conic, depth, color, opacity}, n, w, h, bin, mask, counts, workers,
                             {image, trans, contrib, ranges, values, values_cap, pairs});
}

int or_brute_render_pg_f(const float* mu2d, const float* cov2d, const float* conic, const float* depth,
                         const float* color, const float* opacity, int64_t n, int w, int h, const uint8_t* mask,
                         int32_t* counts, float* image, float* trans, int32_t* contrib) {
  return brute_render_pg_t<float>({mu2d, cov2d, conic, depth, color, opacity}, n, w, h, mask, counts, image, trans,
                                   contrib);
}
int or_brute_render_pg_d(const double* mu2d, const double* cov2d, const double* conic, const double* depth,
                         const double* color, const double* opacity, int64_t n, int w, int h, const uint8_t* mask,
                         int32_t* counts, double* image, double* trans, int32_t* contrib) {
  return brute_render_pg_t<double>({mu2d, cov2d, conic, depth, color, opacity}, n, w, h, mask, counts, image, trans,
                                    contrib);
}

// Tile ids of one projected Gaussian (bin_aabb / bin_compact), double or float.
int or_bin_one_d(const double* mu2d, const double* cov2d, const double* conic, double opacity, int w, int h,
                 const sk_binning* bin, int32_t* tiles, int cap, int* count) {
  return guard([&] {
    ProjectedGaussian<double> pg;
    pg.mu2d[0] = mu2d[0];
    pg.mu2d[1] = mu2d[1];
    for (int r = 0; r < 2; ++r)
      for (int k = 0; k < 2; ++k) {
        pg.cov2d(r, k) = cov2d[2 * r + k];
        pg.cov2d_inv(r, k) = conic[2 * r + k];
      }
    pg.opacity = opacity;
    const TileGrid grid = make_tile_grid(w, h, tile_size_of(bin));
    const auto t = bin_one(pg, grid, to_binning<double>(bin));
    *count = int(t.size());
    for (int i = 0; i < int(t.size()) && i < cap; ++i) tiles[i] = t[i];
  });
}
double or_compact_threshold_d(double sigma, double tau_alpha, double beta) {
  return compact_threshold(sigma, tau_alpha, beta);
}

// ---- backward ----------------------------------------------------------------
int or_blend_backward_pg_f(const float* mu2d, const float* cov2d, const float* conic, const float* depth,
                           const float* color, const float* opacity, int64_t n, int w, int h, const sk_binning* bin,
                           const float* d_image, int workers, float* d_mu2d, float* d_conic, float* d_color,
                           float* d_opacity, float* abs_grad) {
  return blend_backward_pg_t<float>({mu2d, cov2d, conic, depth, color, opacity}, n, w, h, bin, d_image, workers,
                                    {d_mu2d, d_conic, d_color, d_opacity, abs_grad});
}
int or_blend_backward_pg_d(const double* mu2d, const double* cov2d, const double* conic, const double* depth,
                           const double* color, const double* opacity, int64_t n, int w, int h, const sk_binning* bin,
                           const double* d_image, int workers, double* d_mu2d, double* d_conic, double* d_color,
                           double* d_opacity, double* abs_grad) {
  return blend_backward_pg_t<double>({mu2d, cov2d, conic, depth, color, opacity}, n, w, h, bin, d_image, workers,
                                     {d_mu2d, d_conic, d_color, d_opacity, abs_grad});
}

int or_project_backward_f(const float* params, int64_t n, int deg, const sk_camera* cam, const float* d_mu2d,
                          const float* d_conic, const float* d_color, const float* d_opacity, float* grads) {
  return project_backward_t<float>(params, n, deg, cam, d_mu2d, d_conic, d_color, d_opacity, grads);
}
int or_project_backward_d(const double* params, int64_t n, int deg, const sk_camera* cam, const double* d_mu2d,
                          const double* d_conic, const double* d_color, const double* d_opacity, double* grads) {
  return project_backward_t<double>(params, n, deg, cam, d_mu2d, d_conic, d_color, d_opacity, grads);
}

// Raw project_backward with a d_cov2d upstream (camera.hpp:156), one Gaussian.
int or_project_backward_raw_d(const double* params, int deg, const sk_camera* cam, const double* d_mu2d,
                              const double* d_cov2d, const double* d_color, double d_opacity, double* grads) {
  return guard([&] {
    const Scene<double> s = scene_from_planar(params, 1, deg);
    const Camera<double> c = to_camera<double>(cam);
    Mat2<double> dc;
    for (int r = 0; r < 2; ++r)
      for (int k = 0; k < 2; ++k) dc(r, k) = d_cov2d[2 * r + k];
    Vec2<double> dm;
    dm[0] = d_mu2d[0];
    dm[1] = d_mu2d[1];
    const auto g = project_backward(s.gaussians[0], c, deg, dm, dc, v3(d_color[0], d_color[1], d_color[2]), d_opacity);
    Scene<double> gs = s;
    auto& o = gs.gaussians[0];
    o.mu = g.mu;
    o.rot = g.rot;
    o.log_scale = g.log_scale;
    o.opacity_logit = g.opacity_logit;
    o.sh = g.sh;
    scene_to_planar(gs, grads);
  });
}

// Raw project() of one Gaussian in double (for finite differences).
int or_project_one_d(const double* params, int deg, const sk_camera* cam, int32_t* visible, double* mu2d,
                     double* cov2d, double* color, double* opacity) {
  return guard([&] {
    const Scene<double> s = scene_from_planar(params, 1, deg);
    auto pg = project(s.gaussians[0], to_camera<double>(cam), deg, 0);
    *visible = pg ? 1 : 0;
    if (!pg) return;
    mu2d[0] = pg->mu2d[0];
    mu2d[1] = pg->mu2d[1];
    for (int r = 0; r < 2; ++r)
      for (int k = 0; k < 2; ++k) cov2d[2 * r + k] = pg->cov2d(r, k);
    for (int k = 0; k < 3; ++k) color[k] = pg->color[k];
    *opacity = pg->opacity;
  });
}

int or_covariance_3d_d(const double* rot, const double* scale, double* sigma) {
  return guard([&] {
    Vec4<double> q;
    for (int i = 0; i < 4; ++i) q[i] = rot[i];
    const Mat3<double> s = covariance_3d(q, v3(scale[0], scale[1], scale[2]));
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) sigma[3 * r + k] = s(r, k);
  });
}
int or_covariance_3d_backward_d(const double* rot, const double* scale, const double* d_sigma, double* d_rot,
                                double* d_scale) {
  return guard([&] {
    Vec4<double> q;
    for (int i = 0; i < 4; ++i) q[i] = rot[i];
    Mat3<double> ds;
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) ds(r, k) = d_sigma[3 * r + k];
    Vec4<double> dr;
    Vec3<double> dsc;
    covariance_3d_backward(q, v3(scale[0], scale[1], scale[2]), ds, dr, dsc);
    for (int i = 0; i < 4; ++i) d_rot[i] = dr[i];
    for (int i = 0; i < 3; ++i) d_scale[i] = dsc[i];
  });
}
int or_evaluate_sh_d(const double* sh, int deg, const double* dir, double* rgb) {
  return guard([&] {
    ShMatrix<double> m(sh_coeff_count(deg));
    for (size_t i = 0; i < m.d.size(); ++i) m.d[i] = sh[i];
    const auto c = evaluate_sh(m, v3(dir[0], dir[1], dir[2]), deg);
    for (int i = 0; i < 3; ++i) rgb[i] = c[i];
  });
}
int or_evaluate_sh_backward_d(const double* sh, int deg, const double* dir, const double* d_color, double* d_sh,
                              double* d_dir) {
  return guard([&] {
    ShMatrix<double> m(sh_coeff_count(deg));
    for (size_t i = 0; i < m.d.size(); ++i) m.d[i] = sh[i];
    ShMatrix<double> dsh;
    Vec3<double> dd;
    evaluate_sh_backward(m, v3(dir[0], dir[1], dir[2]), deg, v3(d_color[0], d_color[1], d_color[2]), dsh, dd);
    for (size_t i = 0; i < dsh.d.size(); ++i) d_sh[i] = dsh.d[i];
    for (int i = 0; i < 3; ++i) d_dir[i] = dd[i];
  });
}

// ---- loss / metrics ---------------------------------------------------------
int or_training_loss_f(const float* r, const float* g, int w, int h, float lambda, float* loss, float* l1,
                       float* ssim_v, float* d_image) {
  return training_loss_t<float>(r, g, w, h, lambda, loss, l1, ssim_v, d_image);
}
int or_training_loss_d(const double* r, const double* g, int w, int h, double lambda, double* loss, double* l1,
                       double* ssim_v, double* d_image) {
  return training_loss_t<double>(r, g, w, h, lambda, loss, l1, ssim_v, d_image);
}
int or_ssim_f(const float* a, const float* b, int w, int h, float* out) {
  return guard([&] { *out = ssim(image_from(a, w, h), image_from(b, w, h)); });
}
int or_ssim_d(const double* a, const double* b, int w, int h, double* out) {
  return guard([&] { *out = ssim(image_from(a, w, h), image_from(b, w, h)); });
}
int or_psnr_f(const float* a, const float* b, int w, int h, double* out) {
  return guard([&] { *out = psnr(image_from(a, w, h), image_from(b, w, h)); });
}
int or_psnr_d(const double* a, const double* b, int w, int h, double* out) {
  return guard([&] { *out = psnr(image_from(a, w, h), image_from(b, w, h)); });
}

int or_error_maps_d(const double* r, const double* g, int w, int h, double tau, double lambda, double* raw,
                    double* normalized, uint8_t* mask, double* photometric) {
  return guard([&] {
    const auto m = build_error_maps(image_from(r, w, h), image_from(g, w, h), tau, lambda);
    for (size_t i = 0; i < m.raw.d.size(); ++i) {
      if (raw) raw[i] = m.raw.d[i];
      if (normalized) normalized[i] = m.normalized.d[i];
      if (mask) mask[i] = m.mask.d[i];
    }
    *photometric = m.photometric;
  });
}
int or_error_maps_f(const float* r, const float* g, int w, int h, float tau, float lambda, float* raw,
                    float* normalized, uint8_t* mask, float* photometric) {
  return guard([&] {
    const auto m = build_error_maps(image_from(r, w, h), image_from(g, w, h), tau, lambda);
    for (size_t i = 0; i < m.raw.d.size(); ++i) {
      if (raw) raw[i] = m.raw.d[i];
      if (normalized) normalized[i] = m.normalized.d[i];
      if (mask) mask[i] = m.mask.d[i];
    }
    *photometric = m.photometric;
  });
}

// ---- density control ----------------------------------------------------------
// counts: [k][n] int32 row-major; outputs s_d, s_p_raw, s_p [n].
int or_scores_from_counts_f(const int32_t* counts, const float* photometric, int k, int64_t n, float* s_d,
                            float* s_p_raw, float* s_p) {
  return guard([&] {
    std::vector<std::vector<int>> c(k, std::vector<int>(n));
    for (int j = 0; j < k; ++j)
      for (int64_t i = 0; i < n; ++i) c[j][i] = counts[j * n + i];
    ScoreTable<float> t;
    scores_from_counts(c, std::vector<float>(photometric, photometric + k), t);
    for (int64_t i = 0; i < n; ++i) {
      s_d[i] = t.s_d[i];
      s_p_raw[i] = t.s_p_raw[i];
      s_p[i] = t.s_p[i];
    }
  });
}

// Score-table view for selection calls (ScoreTable adc.hpp:23-45).
struct or_table_f {
  const float* s_d;
  const float* s_p;
  const float* grad_norm_acc;
  const float* abs_grad_acc;
  const float* grad3d_acc;  // [n][3]
  const int32_t* views_seen;
  const float* max_radius2d;
};

static ScoreTable<float> table_from(const or_table_f* t, int64_t n) {
  ScoreTable<float> s;
  s.reset(int(n));
  for (int64_t i = 0; i < n; ++i) {
    if (t->s_d) s.s_d[i] = t->s_d[i];
    if (t->s_p) s.s_p[i] = t->s_p[i];
    if (t->grad_norm_acc) s.grad_norm_acc[i] = t->grad_norm_acc[i];
    if (t->abs_grad_acc) s.abs_grad_acc[i] = t->abs_grad_acc[i];
    if (t->grad3d_acc)
      for (int d = 0; d < 3; ++d) s.grad3d_acc[i][d] = t->grad3d_acc[3 * i + d];
    if (t->views_seen) s.views_seen[i] = t->views_seen[i];
    if (t->max_radius2d) s.max_radius2d[i] = t->max_radius2d[i];
  }
  return s;
}

// flags out: clone[n], split[n] (0/1)
int or_select_densify_f(const float* params, int64_t n, int deg, const or_table_f* t, float tau_d,
                        float grad_threshold, float percent_dense, int use_vcd, float extent, uint8_t* clone,
                        uint8_t* split) {
  return guard([&] {
    const Scene<float> s = scene_from_planar(params, n, deg);
    DensifyParams<float> p;
    p.tau_d = tau_d;
    p.grad_threshold = grad_threshold;
    p.percent_dense = percent_dense;
    p.use_vcd = use_vcd != 0;
    const auto sel = select_densify(table_from(t, n), s, p, extent);
    std::memset(clone, 0, n);
    std::memset(split, 0, n);
    for (int i : sel.clone) clone[i] = 1;
    for (int i : sel.split) split[i] = 1;
  });
}

int or_select_prune_f(const float* params, int64_t n, int deg, const or_table_f* t, int iteration, float tau_p,
                      float min_opacity, float opacity_late, float world_size_frac, float screen_size,
                      int size_prune_from, int densify_until, int use_vcp, float extent, uint8_t* prune) {
  return guard([&] {
    const Scene<float> s = scene_from_planar(params, n, deg);
    PruneParams<float> p;
    p.tau_p = tau_p;
    p.min_opacity = min_opacity;
    p.opacity_late = opacity_late;
    p.world_size_frac = world_size_frac;
    p.screen_size = screen_size;
    p.size_prune_from = size_prune_from;
    p.densify_until = densify_until;
    p.use_vcp = use_vcp != 0;
    const auto pr = select_prune(table_from(t, n), s, iteration, p, extent);
    std::memset(prune, 0, n);
    for (int i : pr) prune[i] = 1;
  });
}

// accumulate_scores (adc.hpp:91-115) over k explicit views with float HWC
// images (concatenated); fills counts [k][n], photometric [k], s_d/s_p_raw/s_p.
int or_accumulate_scores_f(const float* params, int64_t n, int deg, int k, const sk_camera* cams,
                           const float* images, float tau, float lambda, const sk_binning* bin, int workers,
                           int32_t* counts_out, float* photo_out, float* s_d, float* s_p_raw, float* s_p) {
  return guard([&] {
    const Scene<float> s = scene_from_planar(params, n, deg);
    std::vector<Camera<float>> cv;
    std::vector<Image<float>> iv;
    size_t off = 0;
    for (int j = 0; j < k; ++j) {
      cv.push_back(to_camera<float>(&cams[j]));
      iv.push_back(image_from(images + off, cams[j].width, cams[j].height));
      off += size_t(cams[j].width) * cams[j].height * 3;
    }
    std::vector<ViewRef<float>> views;
    for (int j = 0; j < k; ++j) views.push_back({&cv[j], &iv[j]});
    ScoreTable<float> t;
    t.reset(int(n));
    std::vector<std::vector<int>> counts;
    std::vector<float> photo;
    accumulate_scores(s, views, tau, lambda, to_binning<float>(bin), tile_size_of(bin), t, workers, &counts, &photo);
    for (int j = 0; j < k; ++j) {
      if (photo_out) photo_out[j] = photo[j];
      if (counts_out)
        for (int64_t i = 0; i < n; ++i) counts_out[j * n + i] = counts[j][i];
    }
    for (int64_t i = 0; i < n; ++i) {
      if (s_d) s_d[i] = t.s_d[i];
      if (s_p_raw) s_p_raw[i] = t.s_p_raw[i];
      if (s_p) s_p[i] = t.s_p[i];
    }
  });
}

// Parameter gradients of one view (SceneGrads, trainer.hpp:128-147): render,
// training_loss, blend_backward, project_backward. grads planar [C][n].
int or_view_grads_f(const float* params, int64_t n, int deg, const sk_camera* cam, const float* gt_hwc, float lambda,
                    int workers, float* grads_planar, double* loss) {
  return guard([&] {
    const Scene<float> s = scene_from_planar(params, n, deg);
    const Camera<float> c = to_camera<float>(cam);
    const auto pgs = project_scene(s, c);
    const TileGrid grid = build_tile_grid(pgs, c.width, c.height, BinningConfig<float>{}, 16);
    const auto rendered = blend_forward(grid, pgs, nullptr, nullptr, workers);
    const auto lr = training_loss(rendered.image, image_from(gt_hwc, c.width, c.height), lambda);
    const auto bg = blend_backward(grid, pgs, lr.d_image, workers);
    Scene<float> gs = s;
    for (auto& g : gs.gaussians) {
      g.mu = Vec3<float>::zero();
      g.rot = Vec4<float>::zero();
      g.log_scale = Vec3<float>::zero();
      g.opacity_logit = 0.0f;
      g.sh = ShMatrix<float>(g.sh.rows);
    }
    for (size_t p = 0; p < pgs.size(); ++p) {
      const auto& pg = pgs[p];
      const Mat2<float> dcov = cov_grad_from_inv_grad(pg.cov2d_inv, bg.d_conic[p]);
      const auto g = project_backward(s.gaussians[pg.source_index], c, deg, bg.d_mu2d[p], dcov, bg.d_color[p],
                                      bg.d_opacity[p]);
      auto& o = gs.gaussians[pg.source_index];
      o.mu = g.mu;
      o.rot = g.rot;
      o.log_scale = g.log_scale;
      o.opacity_logit = g.opacity_logit;
      o.sh = g.sh;
    }
    scene_to_planar(gs, grads_planar);
    if (loss) *loss = lr.loss;
  });
}

// Trainer::density_event compaction (trainer.hpp:203-233) with explicit split
// normals: prune -> Adam remap -> densify -> Adam remap. m/v planar [C][n] in,
// [C][new_n] out (caller sizes them for n + clones + 2 splits).
int or_apply_prune_densify_f(const float* params, int64_t n, int deg, const uint8_t* prune, const uint8_t* clone,
                             const uint8_t* split, const float* grad3d, const int32_t* views_seen, float clone_lr,
                             const float* eps, const float* m_in, const float* v_in, float* params_out,
                             float* m_out, float* v_out, int64_t* new_n, int32_t* old_to_new) {
  return guard([&] {
    Scene<float> s = scene_from_planar(params, n, deg);
    const int comps = 11 + 3 * sh_coeff_count(deg);
    SceneOptimizer<float> opt;
    opt.init(s);
    AdamGroup<float>* groups[6] = {&opt.pos_, &opt.rot_, &opt.scale_, &opt.opacity_, &opt.sh_dc_, &opt.sh_rest_};
    auto locate = [&](int c, int& g, int& d) {
      if (c < 3) { g = 0; d = c; }
      else if (c < 7) { g = 1; d = c - 3; }
      else if (c < 10) { g = 2; d = c - 7; }
      else if (c < 11) { g = 3; d = 0; }
      else if (c < 14) { g = 4; d = c - 11; }
      else { g = 5; d = c - 14; }
    };
    if (m_in && v_in)
      for (int c = 0; c < comps; ++c) {
        int g, d;
        locate(c, g, d);
        for (int64_t i = 0; i < n; ++i) {
          groups[g]->m[i * groups[g]->dim + d] = m_in[c * n + i];
          groups[g]->v[i * groups[g]->dim + d] = v_in[c * n + i];
        }
      }
    std::vector<int> prune_set, cl, sp;
    for (int64_t i = 0; i < n; ++i) {
      if (prune && prune[i]) prune_set.push_back(int(i));
      else {
        if (clone && clone[i]) cl.push_back(int(i));
        if (split && split[i]) sp.push_back(int(i));
      }
    }
    ScoreTable<float> table;
    table.reset(int(n));
    for (int64_t i = 0; i < n; ++i) {
      table.views_seen[i] = views_seen ? views_seen[i] : 0;
      for (int d = 0; d < 3; ++d) table.grad3d_acc[i][d] = grad3d ? grad3d[3 * i + d] : 0.0f;
    }
    const IndexRemap pr = apply_prune(s, prune_set);
    opt.remap(pr);
    for (int& i : cl) i = pr.old_to_new[i];
    for (int& i : sp) i = pr.old_to_new[i];
    ScoreTable<float> mapped;
    mapped.reset(pr.new_size);
    for (size_t i = 0; i < pr.old_to_new.size(); ++i) {
      const int j = pr.old_to_new[i];
      if (j < 0) continue;
      mapped.grad3d_acc[j] = table.grad3d_acc[i];
      mapped.views_seen[j] = table.views_seen[i];
    }
    size_t e = 0;
    const IndexRemap dr = apply_densify_with(s, cl, sp, mapped, clone_lr, [&] { return double(eps[e++]); });
    opt.remap(dr);
    const int64_t nn = s.size();
    *new_n = nn;
    scene_to_planar(s, params_out);
    if (m_out && v_out)
      for (int c = 0; c < comps; ++c) {
        int g, d;
        locate(c, g, d);
        for (int64_t i = 0; i < nn; ++i) {
          m_out[c * nn + i] = groups[g]->m[i * groups[g]->dim + d];
          v_out[c * nn + i] = groups[g]->v[i * groups[g]->dim + d];
        }
      }
    if (old_to_new)
      for (int64_t i = 0; i < n; ++i) {
        const int a = pr.old_to_new[i];
        old_to_new[i] = a < 0 ? -1 : dr.old_to_new[a];
      }
  });
}

// ---- datasets / training ------------------------------------------------------
struct or_dataset {
  Dataset<float> data;
  Scene<float> gt;
};

or_dataset* or_synth_create(int n_gaussians, int n_views, int width, int height, uint64_t seed, double scale_mult,
                            double focal, int render) {
  auto* d = new or_dataset;
  SynthSpec spec;
  spec.n_gaussians = n_gaussians;
  spec.n_views = n_views;
  spec.width = width;
  spec.height = height;
  spec.seed = seed;
  spec.scale_mult = scale_mult;
  spec.focal = focal;
  try {
    d->gt = generate_synthetic(spec, d->data, render != 0);
  } catch (const std::exception& e) {
    g_err = e.what();
    delete d;
    return nullptr;
  }
  return d;
}
void or_dataset_destroy(or_dataset* d) { delete d; }
int or_dataset_num_views(const or_dataset* d) { return int(d->data.cameras.size()); }
float or_dataset_extent(const or_dataset* d) { return d->data.extent; }
int or_dataset_camera(const or_dataset* d, int v, sk_camera* out) {
  const auto& c = d->data.cameras[v];
  out->width = c.width;
  out->height = c.height;
  out->fx = c.fx;
  out->fy = c.fy;
  out->cx = c.cx;
  out->cy = c.cy;
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) out->world_to_cam[r * 4 + k] = c.world_to_cam(r, k);
  out->near_plane = c.near;
  return 0;
}
int or_dataset_image_u8(const or_dataset* d, int v, uint8_t* hwc) {
  if (v >= int(d->data.images_u8.size())) return SK_ERR_INVALID_ARGUMENT;
  std::memcpy(hwc, d->data.images_u8[v].data(), d->data.images_u8[v].size());
  return 0;
}
int or_dataset_num_points(const or_dataset* d) { return int(d->data.init_points.size()); }
int or_dataset_points(const or_dataset* d, float* xyz, float* rgb) {
  for (size_t i = 0; i < d->data.init_points.size(); ++i)
    for (int c = 0; c < 3; ++c) {
      xyz[3 * i + c] = d->data.init_points[i].first[c];
      rgb[3 * i + c] = d->data.init_points[i].second[c];
    }
  return 0;
}
int or_dataset_train_indices(const or_dataset* d, int32_t* out, int* count) {
  *count = int(d->data.train_indices.size());
  if (out)
    for (size_t i = 0; i < d->data.train_indices.size(); ++i) out[i] = d->data.train_indices[i];
  return 0;
}
int or_dataset_gt_scene(const or_dataset* d, float* params) {
  scene_to_planar(d->gt, params);
  return 0;
}
// Replace the views' images by externally rendered u8 images (e.g. GPU).
int or_dataset_set_image_u8(or_dataset* d, int v, const uint8_t* hwc) {
  const auto& c = d->data.cameras[v];
  const size_t sz = size_t(c.width) * c.height * 3;
  if (int(d->data.images_u8.size()) <= v) {
    d->data.images_u8.resize(d->data.cameras.size());
    d->data.images.resize(d->data.cameras.size());
  }
  d->data.images_u8[v].assign(hwc, hwc + sz);
  Image<float> img(c.width, c.height);
  for (size_t p = 0; p < img.pixels.size(); ++p)
    for (int k = 0; k < 3; ++k) img.pixels[p][k] = hwc[p * 3 + k] / 255.0f;
  d->data.images[v] = std::move(img);
  return 0;
}

int or_init_from_points(const float* xyz, const float* rgb, int64_t n, int deg, float* params) {
  return guard([&] {
    std::vector<std::pair<Vec3<float>, Vec3<float>>> pts(n);
    for (int64_t i = 0; i < n; ++i)
      pts[i] = {v3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]), v3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2])};
    scene_to_planar(init_from_points(pts, deg), params);
  });
}

// TrainConfig as a flat struct for ctypes (config.hpp:20-61).
struct or_train_config {
  int iterations, k;
  double lambda, tau, tau_d, tau_p, beta, tau_alpha;
  int densify_from, densify_until, densify_every, prune_every_early, prune_every_late;
  double grad_threshold, percent_dense;
  double lr_position, lr_position_final, lr_sh_dc, lr_sh_rest, lr_opacity, lr_scale, lr_rotation;
  int opacity_reset_every, lazy_opt_enabled, lazy_opt_interval_15k, lazy_opt_interval_20k;
  uint64_t seed;
  int tile_size, workers, sh_degree, compact, vcd, vcp;
  double prune_min_opacity, prune_opacity_late, prune_world_size_frac, prune_screen_size;
  int size_prune_from, schedule_dry_run;
};

static TrainConfig to_cfg(const or_train_config* c) {
  TrainConfig t;
  t.iterations = c->iterations;
  t.k = c->k;
  t.lambda = c->lambda;
  t.tau = c->tau;
  t.tau_d = c->tau_d;
  t.tau_p = c->tau_p;
  t.beta = c->beta;
  t.tau_alpha = c->tau_alpha;
  t.densify_from = c->densify_from;
  t.densify_until = c->densify_until;
  t.densify_every = c->densify_every;
  t.prune_every_early = c->prune_every_early;
  t.prune_every_late = c->prune_every_late;
  t.grad_threshold = c->grad_threshold;
  t.percent_dense = c->percent_dense;
  t.lr_position = c->lr_position;
  t.lr_position_final = c->lr_position_final;
  t.lr_sh_dc = c->lr_sh_dc;
  t.lr_sh_rest = c->lr_sh_rest;
  t.lr_opacity = c->lr_opacity;
  t.lr_scale = c->lr_scale;
  t.lr_rotation = c->lr_rotation;
  t.opacity_reset_every = c->opacity_reset_every;
  t.lazy_opt_enabled = c->lazy_opt_enabled != 0;
  t.lazy_opt_interval_15k = c->lazy_opt_interval_15k;
  t.lazy_opt_interval_20k = c->lazy_opt_interval_20k;
  t.seed = c->seed;
  t.tile_size = c->tile_size;
  t.workers = c->workers;
  t.sh_degree = c->sh_degree;
  t.compact = c->compact != 0;
  t.vcd = c->vcd != 0;
  t.vcp = c->vcp != 0;
  t.prune_min_opacity = c->prune_min_opacity;
  t.prune_opacity_late = c->prune_opacity_late;
  t.prune_world_size_frac = c->prune_world_size_frac;
  t.prune_screen_size = c->prune_screen_size;
  t.size_prune_from = c->size_prune_from;
  t.schedule_dry_run = c->schedule_dry_run != 0;
  return t;
}

void or_default_config(or_train_config* c) {
  TrainConfig t;
  c->iterations = t.iterations;
  c->k = t.k;
  c->lambda = t.lambda;
  c->tau = t.tau;
  c->tau_d = t.tau_d;
  c->tau_p = t.tau_p;
  c->beta = t.beta;
  c->tau_alpha = t.tau_alpha;
  c->densify_from = t.densify_from;
  c->densify_until = t.densify_until;
  c->densify_every = t.densify_every;
  c->prune_every_early = t.prune_every_early;
  c->prune_every_late = t.prune_every_late;
  c->grad_threshold = t.grad_threshold;
  c->percent_dense = t.percent_dense;
  c->lr_position = t.lr_position;
  c->lr_position_final = t.lr_position_final;
  c->lr_sh_dc = t.lr_sh_dc;
  c->lr_sh_rest = t.lr_sh_rest;
  c->lr_opacity = t.lr_opacity;
  c->lr_scale = t.lr_scale;
  c->lr_rotation = t.lr_rotation;
  c->opacity_reset_every = t.opacity_reset_every;
  c->lazy_opt_enabled = t.lazy_opt_enabled;
  c->lazy_opt_interval_15k = t.lazy_opt_interval_15k;
  c->lazy_opt_interval_20k = t.lazy_opt_interval_20k;
  c->seed = t.seed;
  c->tile_size = t.tile_size;
  c->workers = t.workers;
  c->sh_degree = t.sh_degree;
  c->compact = t.compact;
  c->vcd = t.vcd;
  c->vcp = t.vcp;
  c->prune_min_opacity = t.prune_min_opacity;
  c->prune_opacity_late = t.prune_opacity_late;
  c->prune_world_size_frac = t.prune_world_size_frac;
  c->prune_screen_size = t.prune_screen_size;
  c->size_prune_from = t.size_prune_from;
  c->schedule_dry_run = t.schedule_dry_run;
}

int or_densify_due(int it, const or_train_config* c) { return densify_due(it, to_cfg(c)); }
int or_prune_due(int it, const or_train_config* c) { return prune_due(it, to_cfg(c)); }
double or_expon_lr_f(float a, float b, int step, int max_steps) { return expon_lr(a, b, step, max_steps); }

struct or_trainer {
  std::unique_ptr<Dataset<float>> owned;  // single-view trainers own their dataset
  std::unique_ptr<Trainer<float>> t;
};

// A Trainer over a one-view dataset (camera + 8-bit GT): the CPU baseline of
// the config-2 training step (the Rng's view draw always picks view 0).
or_trainer* or_view_trainer_create(const float* params, int64_t n, int deg, const sk_camera* cam,
                                   const uint8_t* gt_hwc, const or_train_config* cfg, float extent) {
  try {
    auto* h = new or_trainer;
    h->owned = std::make_unique<Dataset<float>>();
    Dataset<float>& d = *h->owned;
    d.cameras.push_back(to_camera<float>(cam));
    const size_t px = size_t(cam->width) * cam->height;
    d.images_u8.emplace_back(gt_hwc, gt_hwc + 3 * px);
    Image<float> img(cam->width, cam->height);
    for (size_t p = 0; p < px; ++p)
      for (int c = 0; c < 3; ++c) img.pixels[p][c] = gt_hwc[3 * p + c] / 255.0f;
    d.images.push_back(std::move(img));
    d.train_indices = {0};
    d.extent = extent;
    h->t = std::make_unique<Trainer<float>>(scene_from_planar(params, n, deg), d, to_cfg(cfg));
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

or_trainer* or_trainer_create(const float* params, int64_t n, int deg, const or_dataset* d,
                              const or_train_config* cfg) {
  try {
    auto* h = new or_trainer;
    h->t = std::make_unique<Trainer<float>>(scene_from_planar(params, n, deg), d->data, to_cfg(cfg));
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void or_trainer_destroy(or_trainer* h) { delete h; }

// Runs `iters` iterations (steps + events); log rows: [iters][4] = loss, psnr,
// gaussians, tile_pairs. Returns wall seconds via *seconds.
int or_trainer_run(or_trainer* h, int iters, double* log_rows, double* seconds) {
  return guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const auto rows = h->t->run(iters);
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (log_rows)
      for (size_t i = 0; i < rows.size(); ++i) {
        log_rows[4 * i] = rows[i].loss;
        log_rows[4 * i + 1] = rows[i].psnr;
        log_rows[4 * i + 2] = rows[i].gaussians;
        log_rows[4 * i + 3] = double(rows[i].tile_pairs);
      }
  });
}
int64_t or_trainer_size(const or_trainer* h) { return h->t->scene().size(); }
void or_trainer_set_iteration(or_trainer* h, int it) { h->t->set_iteration(it); }
int or_trainer_scene(const or_trainer* h, float* params) {
  scene_to_planar(h->t->scene(), params);
  return 0;
}
int or_trainer_num_events(const or_trainer* h) { return int(h->t->events().size()); }

// Follow mode: decisions to replay at event `idx` (flags over n pre-event indices).
int or_trainer_force_event(or_trainer* h, int idx, int n, const uint8_t* clone, const uint8_t* split,
                           const uint8_t* prune) {
  auto& f = h->t->forced_;
  if (int(f.size()) <= idx) f.resize(idx + 1);
  f[idx].n = n;
  f[idx].clone.assign(clone, clone + n);
  f[idx].split.assign(split, split + n);
  f[idx].prune.assign(prune, prune + n);
  return 0;
}
// Event e: header [iteration, n_before, n_after, n_clone, n_split, n_prune, k]
int or_trainer_event(const or_trainer* h, int e, int32_t* header, int32_t* clone, int32_t* split, int32_t* prune,
                     int32_t* sampled, float* photometric) {
  const auto& ev = h->t->events()[e];
  header[0] = ev.iteration;
  header[1] = ev.n_before;
  header[2] = ev.n_after;
  header[3] = int(ev.clone.size());
  header[4] = int(ev.split.size());
  header[5] = int(ev.prune.size());
  header[6] = int(ev.sampled.size());
  if (clone) std::copy(ev.clone.begin(), ev.clone.end(), clone);
  if (split) std::copy(ev.split.begin(), ev.split.end(), split);
  if (prune) std::copy(ev.prune.begin(), ev.prune.end(), prune);
  if (sampled) std::copy(ev.sampled.begin(), ev.sampled.end(), sampled);
  if (photometric) std::copy(ev.photometric.begin(), ev.photometric.end(), photometric);
  return 0;
}

// One training iteration on an explicit view (no RNG), for per-step parity:
// returns loss/psnr and the updated scene plus the score table accumulators.
int or_train_step_view(const float* params, int64_t n, int deg, const sk_camera* cam, const float* gt_hwc,
                       const or_train_config* cfg, float extent, int iteration, int workers, float* params_out,
                       double* loss_psnr, int64_t* pairs, float* grad_norm_acc, float* abs_grad_acc,
                       float* grad3d_acc, int32_t* views_seen, float* max_radius2d) {
  return guard([&] {
    Dataset<float> d;
    d.cameras.push_back(to_camera<float>(cam));
    d.images.push_back(image_from(gt_hwc, cam->width, cam->height));
    d.train_indices = {0};
    d.extent = extent;
    TrainConfig c = to_cfg(cfg);
    c.workers = workers;
    Trainer<float> t(scene_from_planar(params, n, deg), d, c);
    const LogRow row = t.train_iteration(iteration);
    scene_to_planar(t.scene(), params_out);
    if (loss_psnr) {
      loss_psnr[0] = row.loss;
      loss_psnr[1] = row.psnr;
    }
    if (pairs) *pairs = row.tile_pairs;
    const auto& tb = t.table();
    for (int64_t i = 0; i < n; ++i) {
      if (grad_norm_acc) grad_norm_acc[i] = tb.grad_norm_acc[i];
      if (abs_grad_acc) abs_grad_acc[i] = tb.abs_grad_acc[i];
      if (grad3d_acc)
        for (int k = 0; k < 3; ++k) grad3d_acc[3 * i + k] = tb.grad3d_acc[i][k];
      if (views_seen) views_seen[i] = tb.views_seen[i];
      if (max_radius2d) max_radius2d[i] = tb.max_radius2d[i];
    }
  });
}

}  // extern "C"
