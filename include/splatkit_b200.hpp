// splatkit_b200.hpp — the reference's splat:: C++ surface (scene, camera,
// raster, train step, densify/prune) re-exposed over the C ABI in
// splatkit_b200.h, so a splatkit caller keeps its call sites.
//
// Differences from the reference headers (proj/include/splatkit):
//  * no Eigen: Vec2/Vec3/Vec4/Mat2/Mat4 are small POD arrays with operator[] /
//    operator(); ShMatrix is row-major (k, c) storage; ScalarMap/MaskMap are
//    row-major (y, x); Image<T> keeps the reference's row-major RGB pixels.
//  * fp32 only (the GPU path); the double instantiation the reference uses for
//    finite differences stays with the CPU oracle.
//  * every call runs on the GPU of a splat::Device (one context + stream);
//    errors come back as the reference's exception types and messages.
#pragma once

#include <array>
#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "splatkit_b200.h"

namespace splat {

using T = float;
struct Vec2 { T v[2] = {0, 0}; T& operator[](int i) { return v[i]; } const T& operator[](int i) const { return v[i]; } };
struct Vec3 { T v[3] = {0, 0, 0}; T& operator[](int i) { return v[i]; } const T& operator[](int i) const { return v[i]; } };
struct Vec4 { T v[4] = {1, 0, 0, 0}; T& operator[](int i) { return v[i]; } const T& operator[](int i) const { return v[i]; } };
struct Mat2 { T m[4] = {0, 0, 0, 0}; T& operator()(int r, int c) { return m[2 * r + c]; } const T& operator()(int r, int c) const { return m[2 * r + c]; } };
struct Mat4 {
  T m[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
  T& operator()(int r, int c) { return m[4 * r + c]; }
  const T& operator()(int r, int c) const { return m[4 * r + c]; }
};

struct ShMatrix {
  int rows = 0;
  std::vector<T> d;
  ShMatrix() = default;
  explicit ShMatrix(int r) : rows(r), d(size_t(r) * 3, 0) {}
  T& operator()(int k, int c) { return d[size_t(k) * 3 + c]; }
  const T& operator()(int k, int c) const { return d[size_t(k) * 3 + c]; }
};

inline constexpr int sh_coeff_count(int degree) { return (degree + 1) * (degree + 1); }

// Gaussian3D / Scene (scene.hpp:18-52)
struct Gaussian3D {
  Vec3 mu;
  Vec4 rot;
  Vec3 log_scale;
  T opacity_logit = 0;
  ShMatrix sh;
};
struct Scene {
  std::vector<Gaussian3D> gaussians;
  int sh_degree = 3;
  int size() const { return int(gaussians.size()); }
};

// Camera (camera.hpp:23-57)
struct Camera {
  int width = 0, height = 0;
  T fx = 0, fy = 0, cx = 0, cy = 0;
  Mat4 world_to_cam;
  T near = T(0.2);
};

struct ProjectedGaussian {
  Vec2 mu2d;
  Mat2 cov2d, cov2d_inv;
  T depth = 0;
  Vec3 color;
  T opacity = 0;
  int source_index = -1;
};

enum class BinMode { kAabb, kCompact };
struct BinningConfig {
  BinMode mode = BinMode::kAabb;
  T beta = 1;
  T tau_alpha = T(1.0 / 255);
};

template <typename U>
struct Map2D {
  int h = 0, w = 0;
  std::vector<U> d;
  Map2D() = default;
  Map2D(int h_, int w_, U fill = U()) : h(h_), w(w_), d(size_t(h_) * w_, fill) {}
  U& operator()(int y, int x) { return d[size_t(y) * w + x]; }
  const U& operator()(int y, int x) const { return d[size_t(y) * w + x]; }
};
using ScalarMap = Map2D<T>;
using MaskMap = Map2D<std::uint8_t>;

struct Image {
  int width = 0, height = 0;
  std::vector<Vec3> pixels;
  Image() = default;
  Image(int w, int h) : width(w), height(h), pixels(size_t(w) * h) {}
  Vec3& at(int x, int y) { return pixels[size_t(y) * width + x]; }
  const Vec3& at(int x, int y) const { return pixels[size_t(y) * width + x]; }
};

struct TileGrid {
  int width = 0, height = 0, tile_size = 16, tiles_x = 0, tiles_y = 0;
  std::vector<std::vector<int>> tiles;
  int tile_count() const { return tiles_x * tiles_y; }
};

struct RenderOutputs {
  Image image;
  ScalarMap transmittance;
  Map2D<int> contrib_count;
};

struct FootprintCounter {
  std::vector<int> counts;
  explicit FootprintCounter(int n = 0) : counts(n, 0) {}
};

struct BlendGrads {
  std::vector<Vec2> d_mu2d;
  std::vector<Mat2> d_conic;
  std::vector<Vec3> d_color;
  std::vector<T> d_opacity;
  std::vector<Vec2> abs_grad;
};

struct LossResult {
  T loss = 0, l1 = 0, ssim_value = 0;
  Image d_image;
};

namespace detail {

inline void raise(int rc, const char* msg) {
  if (rc == SK_OK) return;
  if (rc == SK_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

inline sk_camera to_c(const Camera& c) {
  sk_camera o{};
  o.width = c.width;
  o.height = c.height;
  o.fx = c.fx;
  o.fy = c.fy;
  o.cx = c.cx;
  o.cy = c.cy;
  for (int i = 0; i < 16; ++i) o.world_to_cam[i] = c.world_to_cam.m[i];
  o.near_plane = c.near;
  return o;
}

inline sk_binning to_c(const BinningConfig& b, int tile_size) {
  return sk_binning{b.mode == BinMode::kCompact ? 1 : 0, b.beta, b.tau_alpha, tile_size};
}

inline std::vector<float> planar(const Scene& s) {
  const int n = s.size(), nsh = sh_coeff_count(s.sh_degree);
  std::vector<float> p(size_t(SK_COMP_COUNT(s.sh_degree)) * n);
  for (int i = 0; i < n; ++i) {
    const auto& g = s.gaussians[i];
    for (int d = 0; d < 3; ++d) p[size_t(SK_COMP_MU + d) * n + i] = g.mu[d];
    for (int d = 0; d < 4; ++d) p[size_t(SK_COMP_ROT + d) * n + i] = g.rot[d];
    for (int d = 0; d < 3; ++d) p[size_t(SK_COMP_LOG_SCALE + d) * n + i] = g.log_scale[d];
    p[size_t(SK_COMP_OPACITY) * n + i] = g.opacity_logit;
    for (int k = 0; k < nsh; ++k)
      for (int c = 0; c < 3; ++c) p[size_t(SK_COMP_SH + 3 * k + c) * n + i] = g.sh(k, c);
  }
  return p;
}

inline void from_planar(const std::vector<float>& p, int n, Scene& s) {
  const int nsh = sh_coeff_count(s.sh_degree);
  s.gaussians.assign(n, Gaussian3D{});
  for (int i = 0; i < n; ++i) {
    auto& g = s.gaussians[i];
    for (int d = 0; d < 3; ++d) g.mu[d] = p[size_t(SK_COMP_MU + d) * n + i];
    for (int d = 0; d < 4; ++d) g.rot[d] = p[size_t(SK_COMP_ROT + d) * n + i];
    for (int d = 0; d < 3; ++d) g.log_scale[d] = p[size_t(SK_COMP_LOG_SCALE + d) * n + i];
    g.opacity_logit = p[size_t(SK_COMP_OPACITY) * n + i];
    g.sh = ShMatrix(nsh);
    for (int k = 0; k < nsh; ++k)
      for (int c = 0; c < 3; ++c) g.sh(k, c) = p[size_t(SK_COMP_SH + 3 * k + c) * n + i];
  }
}

}  // namespace detail

// One GPU: context + a scratch frame. Calls on a Device are not thread-safe.
class Device {
 public:
  explicit Device(int device = 0) {
    detail::raise(sk_ctx_create(device, &ctx_), "splat::Device: sk_ctx_create failed");
    check(sk_frame_create(ctx_, &frame_));
  }
  ~Device() {
    if (frame_) sk_frame_destroy(frame_);
    if (ctx_) sk_ctx_destroy(ctx_);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  sk_ctx* ctx() const { return ctx_; }
  sk_frame* frame() const { return frame_; }
  void check(int rc) const { detail::raise(rc, sk_last_error(ctx_)); }

 private:
  sk_ctx* ctx_ = nullptr;
  sk_frame* frame_ = nullptr;
};

// Device-resident copy of a Scene for the duration of a call sequence.
class DeviceScene {
 public:
  DeviceScene(const Device& dev, const Scene& s) : dev_(dev), deg_(s.sh_degree) {
    dev.check(sk_scene_create(dev.ctx(), s.sh_degree, s.size(), &h_));
    const auto p = detail::planar(s);
    dev.check(sk_scene_upload(dev.ctx(), h_, p.data(), s.size()));
  }
  ~DeviceScene() { sk_scene_destroy(h_); }
  DeviceScene(const DeviceScene&) = delete;
  DeviceScene& operator=(const DeviceScene&) = delete;
  sk_scene* handle() const { return h_; }
  Scene download() const {
    int64_t n = 0;
    sk_scene_size(h_, &n);
    std::vector<float> p(size_t(SK_COMP_COUNT(deg_)) * n);
    dev_.check(sk_scene_download(dev_.ctx(), h_, p.data()));
    Scene s;
    s.sh_degree = deg_;
    detail::from_planar(p, int(n), s);
    return s;
  }

 private:
  const Device& dev_;
  int deg_;
  sk_scene* h_ = nullptr;
};

// project_scene (camera.hpp:137-144): compacted, in scene order.
inline std::vector<ProjectedGaussian> project_scene(const Device& dev, const Scene& scene, const Camera& cam) {
  DeviceScene ds(dev, scene);
  const sk_camera c = detail::to_c(cam);
  const sk_binning b = detail::to_c(BinningConfig{}, 16);
  dev.check(sk_preprocess(dev.ctx(), ds.handle(), &c, &b, dev.frame()));
  const size_t n = size_t(scene.size());
  std::vector<int32_t> vis(n), tiles(n);
  std::vector<float> mu(2 * n), cov(4 * n), con(4 * n), depth(n), col(3 * n), op(n);
  sk_projected out{vis.data(), mu.data(), cov.data(), con.data(), depth.data(), col.data(), op.data(), tiles.data()};
  dev.check(sk_frame_get_projected(dev.ctx(), dev.frame(), &out));
  std::vector<ProjectedGaussian> pgs;
  for (size_t i = 0; i < n; ++i) {
    if (!vis[i]) continue;
    ProjectedGaussian pg;
    pg.mu2d[0] = mu[2 * i];
    pg.mu2d[1] = mu[2 * i + 1];
    for (int k = 0; k < 4; ++k) {
      pg.cov2d.m[k] = cov[4 * i + k];
      pg.cov2d_inv.m[k] = con[4 * i + k];
    }
    pg.depth = depth[i];
    for (int k = 0; k < 3; ++k) pg.color[k] = col[3 * i + k];
    pg.opacity = op[i];
    pg.source_index = int(i);
    pgs.push_back(pg);
  }
  return pgs;
}

namespace detail {
inline void inject(const Device& dev, const std::vector<ProjectedGaussian>& pgs, int w, int h, const sk_binning& b) {
  const size_t n = pgs.size();
  std::vector<float> mu(2 * n), cov(4 * n), con(4 * n), depth(n), col(3 * n), op(n);
  for (size_t i = 0; i < n; ++i) {
    const auto& pg = pgs[i];
    mu[2 * i] = pg.mu2d[0];
    mu[2 * i + 1] = pg.mu2d[1];
    for (int k = 0; k < 4; ++k) {
      cov[4 * i + k] = pg.cov2d.m[k];
      con[4 * i + k] = pg.cov2d_inv.m[k];
    }
    depth[i] = pg.depth;
    for (int k = 0; k < 3; ++k) col[3 * i + k] = pg.color[k];
    op[i] = pg.opacity;
  }
  sk_projected in{nullptr, mu.data(), cov.data(), con.data(), depth.data(), col.data(), op.data(), nullptr};
  dev.check(sk_frame_set_projected(dev.ctx(), dev.frame(), &in, int64_t(n), w, h, &b));
}
}  // namespace detail

// build_tile_grid (raster.hpp:157-168): per-tile lists of projected indices.
inline TileGrid build_tile_grid(const Device& dev, const std::vector<ProjectedGaussian>& pgs, int width, int height,
                                const BinningConfig& binning, int tile_size = 16) {
  const sk_binning b = detail::to_c(binning, tile_size);
  detail::inject(dev, pgs, width, height, b);
  int64_t pairs = 0;
  dev.check(sk_bin_sort(dev.ctx(), dev.frame(), &pairs));
  TileGrid g;
  g.width = width;
  g.height = height;
  g.tile_size = tile_size;
  sk_frame_num_tiles(dev.frame(), &g.tiles_x, &g.tiles_y);
  std::vector<int32_t> ranges(2 * size_t(g.tile_count())), values(size_t(pairs > 0 ? pairs : 1));
  dev.check(sk_frame_get_tile_lists(dev.ctx(), dev.frame(), ranges.data(), values.data()));
  g.tiles.resize(g.tile_count());
  for (int t = 0; t < g.tile_count(); ++t) g.tiles[t].assign(values.begin() + ranges[2 * t], values.begin() + ranges[2 * t + 1]);
  return g;
}

inline std::int64_t count_pairs(const TileGrid& grid) {
  std::int64_t total = 0;
  for (const auto& t : grid.tiles) total += std::int64_t(t.size());
  return total;
}

// blend_forward (raster.hpp:194-248) over the projected list; the tile lists
// are rebuilt on the device from `pgs` with the grid's geometry.
inline RenderOutputs blend_forward(const Device& dev, const TileGrid& grid, const std::vector<ProjectedGaussian>& pgs,
                                   const MaskMap* mask = nullptr, FootprintCounter* counter = nullptr,
                                   const BinningConfig& binning = BinningConfig{}) {
  detail::inject(dev, pgs, grid.width, grid.height, detail::to_c(binning, grid.tile_size));
  RenderOutputs out;
  std::vector<int32_t> counts;
  if (mask && counter) counts.assign(pgs.size(), 0);
  dev.check(sk_render_forward(dev.ctx(), dev.frame(), (mask && counter) ? mask->d.data() : nullptr,
                              (mask && counter) ? counts.data() : nullptr));
  if (mask && counter) {
    for (size_t i = 0; i < pgs.size(); ++i) {
      const int src = pgs[i].source_index;
      if (src >= 0 && src < int(counter->counts.size())) counter->counts[src] += counts[i];
    }
  }
  out.image = Image(grid.width, grid.height);
  std::vector<float> hwc(size_t(grid.width) * grid.height * 3);
  dev.check(sk_frame_get_image(dev.ctx(), dev.frame(), hwc.data()));
  for (size_t p = 0; p < out.image.pixels.size(); ++p)
    for (int c = 0; c < 3; ++c) out.image.pixels[p][c] = hwc[3 * p + c];
  out.transmittance = ScalarMap(grid.height, grid.width);
  dev.check(sk_frame_get_transmittance(dev.ctx(), dev.frame(), out.transmittance.d.data()));
  out.contrib_count = Map2D<int>(grid.height, grid.width);
  dev.check(sk_frame_get_contrib_count(dev.ctx(), dev.frame(), out.contrib_count.d.data()));
  return out;
}

// blend_backward (raster.hpp:281-355), after blend_forward on the same Device.
inline BlendGrads blend_backward(const Device& dev, const Image& d_image) {
  std::vector<float> hwc(d_image.pixels.size() * 3);
  for (size_t p = 0; p < d_image.pixels.size(); ++p)
    for (int c = 0; c < 3; ++c) hwc[3 * p + c] = d_image.pixels[p][c];
  dev.check(sk_frame_set_dimage(dev.ctx(), dev.frame(), hwc.data()));
  dev.check(sk_render_backward(dev.ctx(), dev.frame()));
  int64_t n = 0;
  sk_frame_num_projected(dev.frame(), &n);
  std::vector<float> dm(2 * n), dc(4 * n), dcol(3 * n), dop(n), ab(2 * n);
  sk_blend_grads g{dm.data(), dc.data(), dcol.data(), dop.data(), ab.data()};
  dev.check(sk_frame_get_blend_grads(dev.ctx(), dev.frame(), &g));
  BlendGrads out;
  out.d_mu2d.resize(n);
  out.d_conic.resize(n);
  out.d_color.resize(n);
  out.d_opacity.assign(dop.begin(), dop.end());
  out.abs_grad.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 2; ++k) {
      out.d_mu2d[i][k] = dm[2 * i + k];
      out.abs_grad[i][k] = ab[2 * i + k];
    }
    for (int k = 0; k < 4; ++k) out.d_conic[i].m[k] = dc[4 * i + k];
    for (int k = 0; k < 3; ++k) out.d_color[i][k] = dcol[3 * i + k];
  }
  return out;
}

// training_loss (loss.hpp:21-47) of the Device's last render against gt.
inline LossResult training_loss(const Device& dev, const Image& ground_truth, T lambda) {
  std::vector<float> gt(ground_truth.pixels.size() * 3);
  for (size_t p = 0; p < ground_truth.pixels.size(); ++p)
    for (int c = 0; c < 3; ++c) gt[3 * p + c] = ground_truth.pixels[p][c];
  sk_loss_values v{};
  dev.check(sk_loss(dev.ctx(), dev.frame(), gt.data(), lambda, &v));
  LossResult out;
  out.loss = T(v.loss);
  out.l1 = T(v.l1);
  out.ssim_value = T(v.ssim);
  out.d_image = Image(ground_truth.width, ground_truth.height);
  std::vector<float> d(gt.size());
  dev.check(sk_frame_get_dimage(dev.ctx(), dev.frame(), d.data()));
  for (size_t p = 0; p < out.d_image.pixels.size(); ++p)
    for (int c = 0; c < 3; ++c) out.d_image.pixels[p][c] = d[3 * p + c];
  return out;
}

// TrainConfig (config.hpp:20-61) — the C struct with the reference's field names.
using TrainConfig = sk_train_config;
inline TrainConfig default_train_config() {
  TrainConfig c;
  sk_default_config(&c);
  return c;
}

// Dataset (dataset.hpp:24-32): cameras + 8-bit GT images.
struct Dataset {
  std::vector<Camera> cameras;
  std::vector<int> camera_ids;
  std::vector<std::vector<std::uint8_t>> images_u8;  // HWC per view
  std::vector<std::pair<Vec3, Vec3>> init_points;    // xyz, rgb in 0..1
  std::vector<int> train_indices;
  std::vector<int> test_indices;
  T extent = 1;
};

// ---- on-disk formats (ply.hpp, png_io.cpp, dataset.hpp) ------------------
namespace detail {
inline void io_check(const Device* dev, int rc, const char* what) {
  if (dev) dev->check(rc);
  else raise(rc, what);
}
inline Camera from_c(const sk_camera& c) {
  Camera o;
  o.width = c.width;
  o.height = c.height;
  o.fx = c.fx;
  o.fy = c.fy;
  o.cx = c.cx;
  o.cy = c.cy;
  for (int i = 0; i < 16; ++i) o.world_to_cam.m[i] = c.world_to_cam[i];
  o.near = c.near_plane;
  return o;
}
}  // namespace detail

// save_checkpoint (ply.hpp:217-248)
inline void save_checkpoint(const Device& dev, const Scene& scene, const std::string& path) {
  DeviceScene ds(dev, scene);
  dev.check(sk_checkpoint_save(dev.ctx(), ds.handle(), path.c_str()));
}

// load_checkpoint (ply.hpp:251-315)
inline Scene load_checkpoint(const Device& dev, const std::string& path) {
  sk_scene* h = nullptr;
  dev.check(sk_checkpoint_load(dev.ctx(), path.c_str(), 0, &h));
  std::unique_ptr<sk_scene, int (*)(sk_scene*)> guard(h, sk_scene_destroy);
  int deg = 0;
  int64_t n = 0;
  sk_scene_sh_degree(h, &deg);
  sk_scene_size(h, &n);
  std::vector<float> p(size_t(SK_COMP_COUNT(deg)) * n);
  dev.check(sk_scene_download(dev.ctx(), h, p.data()));
  Scene s;
  s.sh_degree = deg;
  detail::from_planar(p, int(n), s);
  return s;
}

// read_png (png_io.cpp:25-72): float image = byte / 255.0f.
inline Image read_png(const std::string& path) {
  int w = 0, h = 0;
  detail::io_check(nullptr, sk_png_read(nullptr, path.c_str(), nullptr, &w, &h), ("png: cannot read " + path).c_str());
  std::vector<std::uint8_t> rgb(size_t(w) * h * 3);
  detail::io_check(nullptr, sk_png_read(nullptr, path.c_str(), rgb.data(), &w, &h), ("png: cannot read " + path).c_str());
  Image img(w, h);
  for (size_t i = 0; i < size_t(w) * h; ++i)
    for (int c = 0; c < 3; ++c) img.pixels[i][c] = rgb[3 * i + c] / 255.0f;
  return img;
}

// write_png (png_io.cpp:74-104)
inline void write_png(const std::string& path, const Image& image) {
  std::vector<float> rgb(size_t(image.width) * image.height * 3);
  for (size_t i = 0; i < image.pixels.size(); ++i)
    for (int c = 0; c < 3; ++c) rgb[3 * i + c] = image.pixels[i][c];
  detail::io_check(nullptr, sk_png_write(nullptr, path.c_str(), rgb.data(), image.width, image.height),
                   ("png: cannot write " + path).c_str());
}

// read_points_ply / write_points_ply (ply.hpp:179-212)
inline std::vector<std::pair<Vec3, Vec3>> read_points_ply(const std::string& path) {
  int64_t n = 0;
  detail::io_check(nullptr, sk_points_read(nullptr, path.c_str(), nullptr, nullptr, &n),
                   ("ply: cannot read " + path).c_str());
  std::vector<float> xyz(size_t(n) * 3), rgb(size_t(n) * 3);
  detail::io_check(nullptr, sk_points_read(nullptr, path.c_str(), xyz.data(), rgb.data(), &n),
                   ("ply: cannot read " + path).c_str());
  std::vector<std::pair<Vec3, Vec3>> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      out[i].first[d] = xyz[3 * i + d];
      out[i].second[d] = rgb[3 * i + d];
    }
  return out;
}

inline void write_points_ply(const std::string& path, const std::vector<std::pair<Vec3, Vec3>>& points) {
  std::vector<float> xyz, rgb;
  for (const auto& [p, c] : points)
    for (int d = 0; d < 3; ++d) {
      xyz.push_back(p[d]);
      rgb.push_back(c[d]);
    }
  detail::io_check(nullptr, sk_points_write(nullptr, path.c_str(), xyz.data(), rgb.data(), int64_t(points.size())),
                   ("ply: cannot write " + path).c_str());
}

// load_dataset (dataset.hpp:73-125)
inline Dataset load_dataset(const Device& dev, const std::string& path) {
  sk_dataset* d = nullptr;
  dev.check(sk_dataset_load(dev.ctx(), path.c_str(), &d));
  std::unique_ptr<sk_dataset, int (*)(sk_dataset*)> guard(d, sk_dataset_destroy);
  Dataset out;
  int nv = 0;
  sk_dataset_num_views(d, &nv);
  for (int v = 0; v < nv; ++v) {
    sk_camera c;
    sk_dataset_camera(d, v, &c);
    out.cameras.push_back(detail::from_c(c));
    std::vector<std::uint8_t> img(size_t(c.width) * c.height * 3);
    dev.check(sk_dataset_image_u8(dev.ctx(), d, v, img.data()));
    out.images_u8.push_back(std::move(img));
  }
  int cnt = 0;
  sk_dataset_train_indices(d, nullptr, &cnt);
  std::vector<int32_t> tr(static_cast<size_t>(cnt));
  sk_dataset_train_indices(d, tr.data(), &cnt);
  out.train_indices.assign(tr.begin(), tr.end());
  for (int v = 0; v < nv; ++v)
    if (std::find(tr.begin(), tr.end(), v) == tr.end()) out.test_indices.push_back(v);
  int64_t np = 0;
  sk_dataset_init_points(d, nullptr, nullptr, &np);
  std::vector<float> xyz(size_t(np) * 3), rgb(size_t(np) * 3);
  sk_dataset_init_points(d, xyz.data(), rgb.data(), &np);
  for (int64_t i = 0; i < np; ++i) {
    std::pair<Vec3, Vec3> pr;
    for (int k = 0; k < 3; ++k) {
      pr.first[k] = xyz[3 * i + k];
      pr.second[k] = rgb[3 * i + k];
    }
    out.init_points.push_back(pr);
  }
  std::vector<sk_camera> cams(static_cast<size_t>(nv));
  std::vector<int32_t> ids(static_cast<size_t>(nv));
  int cc = nv;
  if (nv > 0 && sk_cameras_read(nullptr, (path + "/cameras.json").c_str(), cams.data(), ids.data(), &cc) == SK_OK)
    out.camera_ids.assign(ids.begin(), ids.end());
  sk_dataset_extent(d, &out.extent);
  return out;
}

// save_cameras_json (dataset.hpp:127-150)
inline void save_cameras_json(const std::string& path, const std::vector<Camera>& cameras,
                              const std::vector<int>& ids) {
  std::vector<sk_camera> c;
  for (const auto& cam : cameras) c.push_back(detail::to_c(cam));
  std::vector<int32_t> i(ids.begin(), ids.end());
  detail::io_check(nullptr, sk_cameras_write(nullptr, path.c_str(), c.data(), i.data(), int(c.size())),
                   ("dataset: cannot write " + path).c_str());
}

struct LogRow {
  int iteration = 0;
  double loss = 0, psnr = 0;
  int gaussians = 0;
  std::int64_t tile_pairs = 0;
  double elapsed_ms = 0;
};

struct TrainResult {
  Scene scene;
  std::vector<LogRow> log;
};

// run_training (trainer.hpp:273-278) on the GPU.
inline TrainResult run_training(const Device& dev, const Scene& scene, const Dataset& data, const TrainConfig& cfg) {
  DeviceScene ds(dev, scene);
  std::vector<sk_camera> cams;
  std::vector<std::uint8_t> imgs;
  for (size_t v = 0; v < data.cameras.size(); ++v) {
    cams.push_back(detail::to_c(data.cameras[v]));
    imgs.insert(imgs.end(), data.images_u8[v].begin(), data.images_u8[v].end());
  }
  std::vector<int32_t> train(data.train_indices.begin(), data.train_indices.end());
  sk_dataset* d = nullptr;
  dev.check(sk_dataset_create(dev.ctx(), int(cams.size()), cams.data(), imgs.data(), train.data(), int(train.size()),
                              data.extent, &d));
  std::unique_ptr<sk_dataset, int (*)(sk_dataset*)> dguard(d, sk_dataset_destroy);
  sk_trainer* t = nullptr;
  dev.check(sk_trainer_create(dev.ctx(), ds.handle(), d, &cfg, &t));
  std::unique_ptr<sk_trainer, int (*)(sk_trainer*)> tguard(t, sk_trainer_destroy);
  std::vector<sk_log_row> rows(size_t(cfg.iterations > 0 ? cfg.iterations : 1));
  dev.check(sk_trainer_run(t, cfg.iterations, rows.data()));
  TrainResult out;
  for (int i = 0; i < cfg.iterations; ++i) {
    LogRow r;
    r.iteration = rows[i].iteration;
    r.loss = rows[i].loss;
    r.psnr = rows[i].psnr;
    r.gaussians = rows[i].gaussians;
    r.tile_pairs = rows[i].tile_pairs;
    r.elapsed_ms = rows[i].elapsed_ms;
    out.log.push_back(r);
  }
  out.scene = ds.download();
  return out;
}

}  // namespace splat
