// splatkit_b200.hpp — the reference's splat:: C++ surface (proj/include/
// splatkit: scene, camera, raster, loss, densify/prune, optimizer, trainer,
// dataset) re-exposed over the C ABI in splatkit_b200.h, so a splatkit caller
// keeps its call sites: the same type and function names, template parameter
// T, argument lists, storage orders and exception types / messages.
//
// What differs from the reference headers, and why:
//  * No Eigen (not a dependency of this library): Vec2/Vec3/Vec4/Mat2/Mat4,
//    ShMatrix and ScalarMap / MaskMap are small POD templates with the
//    reference's element accessors and storage orders (ShMatrix col-major,
//    maps col-major (y, x) -> x * H + y, Image row-major RGB pixels), not
//    Eigen expressions.
//  * Every computation runs on the GPU in fp32 (T = double is converted at
//    the boundary); the double instantiation the reference uses for finite
//    differences stays with the CPU oracle.
//  * Calls run on the current splat::Device (a process-wide Device(0) unless
//    a DeviceScope selects another), so no call site passes a device.
//  * apply_densify takes its clone / split lists in ascending index order
//    (as select_densify returns them); the children are appended in that
//    order, exactly as the reference does for such lists.
//  * Dataset images are held as float Image<T>; the trainer uploads them as
//    8-bit (lround(clamp(v) * 255), exact for images read from PNG).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "splatkit_b200.h"

namespace splat {

// ---- constants (raster.hpp:19-25, camera.hpp:17-20, sh.hpp, adam.hpp:16-18, adc.hpp:160)
inline constexpr double kAlphaCap = 0.99;
inline constexpr double kAlphaMin = 1.0 / 255;
inline constexpr double kTransmitMin = 1e-4;
inline constexpr double kBinSigma = 3.0;
inline constexpr double kBinMahaMax = kBinSigma * kBinSigma;
inline constexpr double kCov2dFloor = 0.3;
inline constexpr double kCullGuard = 1.3;
inline constexpr double kShC0 = 0.28209479177387814;
inline constexpr double kSplitScaleShrink = 1.6;
inline constexpr double kAdamBeta1 = 0.9;
inline constexpr double kAdamBeta2 = 0.999;
inline constexpr double kAdamEps = 1e-15;

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw std::runtime_error(msg);
}

template <typename T>
inline T sigmoid(T x) {
  return T(1) / (T(1) + std::exp(-x));
}
template <typename T>
inline T logit(T x) {
  return std::log(x / (T(1) - x));
}

// ---- small linear-algebra PODs (types.hpp:14-26 without Eigen) -------------
template <typename T, int N>
struct VecN {
  T v[N] = {};
  T& operator[](int i) { return v[i]; }
  const T& operator[](int i) const { return v[i]; }
  bool operator==(const VecN& o) const { return std::equal(v, v + N, o.v); }
  bool operator!=(const VecN& o) const { return !(*this == o); }
  T norm() const {
    T s = T(0);
    for (int i = 0; i < N; ++i) s += v[i] * v[i];
    return std::sqrt(s);
  }
};
template <typename T>
struct Vec2 : VecN<T, 2> {
  Vec2() = default;
  Vec2(T a, T b) { this->v[0] = a, this->v[1] = b; }
  static Vec2 Zero() { return Vec2(); }
};
template <typename T>
struct Vec3 : VecN<T, 3> {
  Vec3() = default;
  Vec3(T a, T b, T c) { this->v[0] = a, this->v[1] = b, this->v[2] = c; }
  static Vec3 Zero() { return Vec3(); }
  static Vec3 Constant(T x) { return Vec3(x, x, x); }
};
template <typename T>
struct Vec4 : VecN<T, 4> {
  Vec4() = default;
  Vec4(T a, T b, T c, T d) { this->v[0] = a, this->v[1] = b, this->v[2] = c, this->v[3] = d; }
  static Vec4 Zero() { return Vec4(); }
};

template <typename T, int R, int C>
struct MatRC {
  T m[R * C] = {};
  T& operator()(int r, int c) { return m[r * C + c]; }
  const T& operator()(int r, int c) const { return m[r * C + c]; }
  bool operator==(const MatRC& o) const { return std::equal(m, m + R * C, o.m); }
};
template <typename T>
struct Mat2 : MatRC<T, 2, 2> {
  static Mat2 Zero() { return Mat2(); }
  static Mat2 Identity() {
    Mat2 a;
    a(0, 0) = a(1, 1) = T(1);
    return a;
  }
  T determinant() const { return (*this)(0, 0) * (*this)(1, 1) - (*this)(0, 1) * (*this)(1, 0); }
};
template <typename T>
struct Mat4 : MatRC<T, 4, 4> {
  Mat4() {
    for (int i = 0; i < 4; ++i) (*this)(i, i) = T(1);
  }
  static Mat4 Identity() { return Mat4(); }
};

// SH coefficients: one row per basis function, RGB columns, column-major
// storage as Eigen's Matrix<T, Dynamic, 3>.
template <typename T>
struct ShMatrix {
  int rows_ = 0;
  std::vector<T> d;
  ShMatrix() = default;
  ShMatrix(int rows, int cols) : rows_(rows), d(size_t(rows) * 3, T(0)) { require(cols == 3, "ShMatrix: 3 columns"); }
  static ShMatrix Zero(int rows, int cols) { return ShMatrix(rows, cols); }
  int rows() const { return rows_; }
  int cols() const { return 3; }
  T& operator()(int k, int c) { return d[size_t(c) * rows_ + k]; }
  const T& operator()(int k, int c) const { return d[size_t(c) * rows_ + k]; }
  bool operator==(const ShMatrix& o) const { return rows_ == o.rows_ && d == o.d; }
};

// Per-pixel maps (H rows x W cols), column-major as Eigen::Array.
template <typename U>
struct Map2D {
  int h = 0, w = 0;
  std::vector<U> d;
  Map2D() = default;
  Map2D(int rows, int cols, U fill = U()) : h(rows), w(cols), d(size_t(rows) * cols, fill) {}
  static Map2D Zero(int rows, int cols) { return Map2D(rows, cols, U(0)); }
  static Map2D Ones(int rows, int cols) { return Map2D(rows, cols, U(1)); }
  static Map2D Constant(int rows, int cols, U v) { return Map2D(rows, cols, v); }
  int rows() const { return h; }
  int cols() const { return w; }
  U& operator()(int y, int x) { return d[size_t(x) * h + y]; }
  const U& operator()(int y, int x) const { return d[size_t(x) * h + y]; }
};
template <typename T>
using ScalarMap = Map2D<T>;
using MaskMap = Map2D<std::uint8_t>;
using IntMap = Map2D<int>;

// RGB image, row-major pixels (types.hpp:37-68).
template <typename T>
struct Image {
  int width = 0, height = 0;
  std::vector<Vec3<T>> pixels;
  Image() = default;
  Image(int w, int h) : width(w), height(h), pixels(size_t(w) * h) {}
  Vec3<T>& at(int x, int y) { return pixels[size_t(y) * width + x]; }
  const Vec3<T>& at(int x, int y) const { return pixels[size_t(y) * width + x]; }
  ScalarMap<T> channel(int c) const {
    ScalarMap<T> out(height, width);
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) out(y, x) = at(x, y)[c];
    return out;
  }
};

// ---- the GPU a call runs on ---------------------------------------------------
class Device {
 public:
  explicit Device(int device = 0) {
    const int rc = sk_ctx_create(device, &ctx_);
    if (rc != SK_OK) throw std::runtime_error("splat::Device: no CUDA device " + std::to_string(device));
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
  // Rethrows a C ABI status as the reference's exception type and message.
  void check(int rc) const {
    if (rc == SK_OK) return;
    const std::string msg = sk_last_error(ctx_);
    if (rc == SK_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }

 private:
  sk_ctx* ctx_ = nullptr;
  sk_frame* frame_ = nullptr;
};

namespace detail {
inline Device*& current_slot() {
  thread_local Device* d = nullptr;
  return d;
}
}  // namespace detail

// The device splat:: calls on this thread run on: the innermost DeviceScope,
// else a process-wide Device(0) created on first use (never destroyed, so no
// CUDA teardown runs from static destructors).
inline Device& current_device() {
  if (Device* d = detail::current_slot()) return *d;
  static Device* fallback = new Device(0);
  return *fallback;
}

class DeviceScope {
 public:
  explicit DeviceScope(Device& d) : prev_(detail::current_slot()) { detail::current_slot() = &d; }
  ~DeviceScope() { detail::current_slot() = prev_; }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;

 private:
  Device* prev_;
};

// ---- Rng (rng.hpp:18-69): mt19937_64 + the hand-rolled distributions ------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : eng_(seed) {}
  std::uint64_t next_u64() { return eng_(); }
  double uniform() { return double(eng_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  std::uint64_t bounded(std::uint64_t n) { return std::uint64_t((__uint128_t(eng_()) * n) >> 64); }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    const double u1 = std::max(uniform(), 0x1.0p-53);
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    spare_ = r * std::sin(a);
    spare_ok_ = true;
    return r * std::cos(a);
  }
  std::vector<int> sample_without_replacement(int n, int k) {
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    const int m = std::min(k, n);
    for (int i = 0; i < m; ++i) std::swap(idx[i], idx[i + int(bounded(std::uint64_t(n - i)))]);
    idx.resize(m);
    return idx;
  }

 private:
  std::mt19937_64 eng_;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

// ---- scene.hpp ------------------------------------------------------------------
inline constexpr int sh_coeff_count(int degree) { return (degree + 1) * (degree + 1); }

template <typename T>
struct Gaussian3D {
  Vec3<T> mu;
  Vec4<T> rot = Vec4<T>(T(1), T(0), T(0), T(0));  // w, x, y, z
  Vec3<T> log_scale;
  T opacity_logit = T(0);
  ShMatrix<T> sh;
  Vec3<T> scale() const { return Vec3<T>(std::exp(log_scale[0]), std::exp(log_scale[1]), std::exp(log_scale[2])); }
  T opacity() const { return sigmoid(opacity_logit); }
};

template <typename T>
struct Scene {
  std::vector<Gaussian3D<T>> gaussians;
  int sh_degree = 3;
  int size() const { return int(gaussians.size()); }
};

// ---- camera.hpp -----------------------------------------------------------------
template <typename T>
struct Camera {
  int width = 0, height = 0;
  T fx = T(0), fy = T(0), cx = T(0), cy = T(0);
  Mat4<T> world_to_cam;
  T near = T(0.2);
};

template <typename T>
struct ProjectedGaussian {
  Vec2<T> mu2d;
  Mat2<T> cov2d, cov2d_inv;
  T depth = T(0);
  Vec3<T> color;
  T opacity = T(0);
  int source_index = -1;
};

template <typename T>
struct GaussianGrads {
  Vec3<T> mu;
  Vec4<T> rot;
  Vec3<T> log_scale;
  T opacity_logit = T(0);
  ShMatrix<T> sh;
};

// ---- raster.hpp -----------------------------------------------------------------
enum class BinMode { kAabb, kCompact };

template <typename T>
struct BinningConfig {
  BinMode mode = BinMode::kAabb;
  T beta = T(1);
  T tau_alpha = T(1.0 / 255);
};

struct TileGrid {
  int width = 0, height = 0, tile_size = 16, tiles_x = 0, tiles_y = 0;
  std::vector<std::vector<int>> tiles;
  int tile_count() const { return tiles_x * tiles_y; }
};

inline TileGrid make_tile_grid(int width, int height, int tile_size = 16) {
  TileGrid g;
  g.width = width;
  g.height = height;
  g.tile_size = tile_size;
  g.tiles_x = (width + tile_size - 1) / tile_size;
  g.tiles_y = (height + tile_size - 1) / tile_size;
  g.tiles.assign(size_t(g.tile_count()), {});
  return g;
}

template <typename T>
struct RenderOutputs {
  Image<T> image;
  ScalarMap<T> transmittance;
  IntMap contrib_count;
};

struct FootprintCounter {
  std::vector<int> counts;
  explicit FootprintCounter(int n_gaussians = 0) : counts(n_gaussians, 0) {}
};

template <typename T>
struct BlendGrads {
  std::vector<Vec2<T>> d_mu2d;
  std::vector<Mat2<T>> d_conic;
  std::vector<Vec3<T>> d_color;
  std::vector<T> d_opacity;
  std::vector<Vec2<T>> abs_grad;
};

namespace detail {

inline Device& dev() { return current_device(); }

template <typename T>
inline sk_camera to_c(const Camera<T>& c) {
  sk_camera o{};
  o.width = c.width;
  o.height = c.height;
  o.fx = float(c.fx);
  o.fy = float(c.fy);
  o.cx = float(c.cx);
  o.cy = float(c.cy);
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) o.world_to_cam[4 * r + k] = float(c.world_to_cam(r, k));
  o.near_plane = float(c.near);
  return o;
}

template <typename T>
inline Camera<T> from_c(const sk_camera& c) {
  Camera<T> o;
  o.width = c.width;
  o.height = c.height;
  o.fx = T(c.fx);
  o.fy = T(c.fy);
  o.cx = T(c.cx);
  o.cy = T(c.cy);
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) o.world_to_cam(r, k) = T(c.world_to_cam[4 * r + k]);
  o.near = T(c.near_plane);
  return o;
}

template <typename T>
inline sk_binning to_c(const BinningConfig<T>& b, int tile_size) {
  return sk_binning{b.mode == BinMode::kCompact ? 1 : 0, float(b.beta), float(b.tau_alpha), tile_size};
}

// Scene<T> <-> planar fp32 [SK_COMP_COUNT(deg)][n] (SK_COMP_* order).
template <typename T>
inline std::vector<float> planar(const Scene<T>& s) {
  const int n = s.size(), nsh = sh_coeff_count(s.sh_degree);
  std::vector<float> p(size_t(SK_COMP_COUNT(s.sh_degree)) * n);
  for (int i = 0; i < n; ++i) {
    const auto& g = s.gaussians[i];
    require(g.sh.rows() >= nsh, "scene: sh has fewer rows than sh_degree needs");
    for (int d = 0; d < 3; ++d) p[size_t(SK_COMP_MU + d) * n + i] = float(g.mu[d]);
    for (int d = 0; d < 4; ++d) p[size_t(SK_COMP_ROT + d) * n + i] = float(g.rot[d]);
    for (int d = 0; d < 3; ++d) p[size_t(SK_COMP_LOG_SCALE + d) * n + i] = float(g.log_scale[d]);
    p[size_t(SK_COMP_OPACITY) * n + i] = float(g.opacity_logit);
    for (int k = 0; k < nsh; ++k)
      for (int c = 0; c < 3; ++c) p[size_t(SK_COMP_SH + 3 * k + c) * n + i] = float(g.sh(k, c));
  }
  return p;
}

template <typename T>
inline void from_planar(const std::vector<float>& p, int n, int sh_degree, Scene<T>& s) {
  const int nsh = sh_coeff_count(sh_degree);
  s.sh_degree = sh_degree;
  s.gaussians.assign(n, Gaussian3D<T>{});
  for (int i = 0; i < n; ++i) {
    auto& g = s.gaussians[i];
    for (int d = 0; d < 3; ++d) g.mu[d] = T(p[size_t(SK_COMP_MU + d) * n + i]);
    for (int d = 0; d < 4; ++d) g.rot[d] = T(p[size_t(SK_COMP_ROT + d) * n + i]);
    for (int d = 0; d < 3; ++d) g.log_scale[d] = T(p[size_t(SK_COMP_LOG_SCALE + d) * n + i]);
    g.opacity_logit = T(p[size_t(SK_COMP_OPACITY) * n + i]);
    g.sh = ShMatrix<T>::Zero(nsh, 3);
    for (int k = 0; k < nsh; ++k)
      for (int c = 0; c < 3; ++c) g.sh(k, c) = T(p[size_t(SK_COMP_SH + 3 * k + c) * n + i]);
  }
}

// A device-resident copy of a Scene for the duration of a call.
class DeviceScene {
 public:
  template <typename T>
  explicit DeviceScene(const Scene<T>& s, int64_t capacity = 0) : deg_(s.sh_degree) {
    Device& d = dev();
    d.check(sk_scene_create(d.ctx(), s.sh_degree, std::max<int64_t>(capacity, s.size()), &h_));
    const auto p = planar(s);
    d.check(sk_scene_upload(d.ctx(), h_, p.data(), s.size()));
  }
  ~DeviceScene() { sk_scene_destroy(h_); }
  DeviceScene(const DeviceScene&) = delete;
  DeviceScene& operator=(const DeviceScene&) = delete;
  sk_scene* handle() const { return h_; }
  int64_t size() const {
    int64_t n = 0;
    sk_scene_size(h_, &n);
    return n;
  }
  template <typename T>
  void download(Scene<T>& s) const {
    const int64_t n = size();
    std::vector<float> p(size_t(SK_COMP_COUNT(deg_)) * n);
    dev().check(sk_scene_download(dev().ctx(), h_, p.data()));
    from_planar(p, int(n), deg_, s);
  }
  // Writes the ScoreTable fields that are present (others left as reset).
  template <typename Table>
  void set_table(const Table& t) {
    const int64_t n = size();
    std::vector<float> s_d, s_p, gn, ag, g3, mr;
    std::vector<int32_t> vs;
    sk_score_table st{};
    auto put = [&](const auto& src, std::vector<float>& dst, float*& field) {
      if (int64_t(src.size()) != n) return;
      dst.assign(src.begin(), src.end());
      field = dst.data();
    };
    put(t.s_d, s_d, st.s_d);
    put(t.s_p, s_p, st.s_p);
    put(t.grad_norm_acc, gn, st.grad_norm_acc);
    put(t.abs_grad_acc, ag, st.abs_grad_acc);
    put(t.max_radius2d, mr, st.max_radius2d);
    if (int64_t(t.grad3d_acc.size()) == n) {
      g3.resize(3 * size_t(n));
      for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) g3[3 * i + d] = float(t.grad3d_acc[i][d]);
      st.grad3d_acc = g3.data();
    }
    if (int64_t(t.views_seen.size()) == n) {
      vs.assign(t.views_seen.begin(), t.views_seen.end());
      st.views_seen = vs.data();
    }
    dev().check(sk_scene_set_score_table(dev().ctx(), h_, &st));
  }

 private:
  int deg_;
  sk_scene* h_ = nullptr;
};

// A device scene handle with no ownership (SceneOptimizer's state scene).
struct DeviceSceneView {
  sk_scene* h;
  int deg;
  DeviceSceneView(sk_scene* h_, int d) : h(h_), deg(d) {}
  template <typename T>
  void download(Scene<T>& s) const {
    int64_t n = 0;
    sk_scene_size(h, &n);
    std::vector<float> p(size_t(SK_COMP_COUNT(deg)) * n);
    dev().check(sk_scene_download(dev().ctx(), h, p.data()));
    from_planar(p, int(n), deg, s);
  }
};

// File-only calls run without a device (ctx NULL): the message is built here.
inline void io(int rc, const std::string& what) {
  if (rc == SK_OK) return;
  if (rc == SK_ERR_INVALID_ARGUMENT) throw std::invalid_argument(what);
  throw std::runtime_error(what);
}

// Injects a projected set (projected index i = position i) into the frame.
template <typename T>
inline void inject(const std::vector<ProjectedGaussian<T>>& pgs, int w, int h, const sk_binning& b) {
  const size_t n = pgs.size();
  std::vector<float> mu(2 * n), cov(4 * n), con(4 * n), depth(n), col(3 * n), op(n);
  for (size_t i = 0; i < n; ++i) {
    const auto& pg = pgs[i];
    mu[2 * i] = float(pg.mu2d[0]);
    mu[2 * i + 1] = float(pg.mu2d[1]);
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) {
        cov[4 * i + 2 * r + c] = float(pg.cov2d(r, c));
        con[4 * i + 2 * r + c] = float(pg.cov2d_inv(r, c));
      }
    depth[i] = float(pg.depth);
    for (int k = 0; k < 3; ++k) col[3 * i + k] = float(pg.color[k]);
    op[i] = float(pg.opacity);
  }
  sk_projected in{nullptr, mu.data(), cov.data(), con.data(), depth.data(), col.data(), op.data(), nullptr};
  dev().check(sk_frame_set_projected(dev().ctx(), dev().frame(), &in, int64_t(n), w, h, &b));
}

// The grid's lists as the frame's tile lists (blend exactly these).
inline void set_lists(const TileGrid& grid) {
  std::vector<int32_t> ranges(2 * size_t(grid.tile_count()));
  std::vector<int32_t> values;
  for (int t = 0; t < grid.tile_count(); ++t) {
    ranges[2 * t] = int32_t(values.size());
    values.insert(values.end(), grid.tiles[t].begin(), grid.tiles[t].end());
    ranges[2 * t + 1] = int32_t(values.size());
  }
  dev().check(sk_frame_set_tile_lists(dev().ctx(), dev().frame(), ranges.data(), values.data(),
                                      int64_t(values.size())));
}

template <typename T>
inline std::vector<float> hwc(const Image<T>& img) {
  std::vector<float> out(img.pixels.size() * 3);
  for (size_t p = 0; p < img.pixels.size(); ++p)
    for (int c = 0; c < 3; ++c) out[3 * p + c] = float(img.pixels[p][c]);
  return out;
}

template <typename T>
inline Image<T> image_from(const std::vector<float>& hwc, int w, int h) {
  Image<T> img(w, h);
  for (size_t p = 0; p < img.pixels.size(); ++p)
    for (int c = 0; c < 3; ++c) img.pixels[p][c] = T(hwc[3 * p + c]);
  return img;
}

// row-major [H][W] (the C ABI) -> col-major map
template <typename U, typename V>
inline Map2D<U> map_from_rows(const std::vector<V>& rows, int h, int w) {
  Map2D<U> m(h, w);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) m(y, x) = U(rows[size_t(y) * w + x]);
  return m;
}

template <typename U>
inline std::vector<U> rows_from_map(const Map2D<U>& m) {
  std::vector<U> rows(size_t(m.h) * m.w);
  for (int y = 0; y < m.h; ++y)
    for (int x = 0; x < m.w; ++x) rows[size_t(y) * m.w + x] = m(y, x);
  return rows;
}

inline std::vector<uint8_t> flags(const std::vector<int>& idx, int n, const char* what) {
  std::vector<uint8_t> f(size_t(n), 0);
  for (const int i : idx) {
    if (i < 0 || i >= n) throw std::invalid_argument(std::string(what) + ": index out of range");
    f[size_t(i)] = 1;
  }
  return f;
}

inline std::vector<int> indices(const std::vector<uint8_t>& f) {
  std::vector<int> out;
  for (size_t i = 0; i < f.size(); ++i)
    if (f[i]) out.push_back(int(i));
  return out;
}

}  // namespace detail

// project (camera.hpp:93-123): nullopt when culled (near plane, guard band).
template <typename T>
inline std::optional<ProjectedGaussian<T>> project(const Gaussian3D<T>& g, const Camera<T>& cam, int sh_degree,
                                                   int source_index = -1) {
  Scene<T> one;
  one.sh_degree = sh_degree;
  one.gaussians.push_back(g);
  detail::DeviceScene ds(one);
  Device& d = detail::dev();
  const sk_camera c = detail::to_c(cam);
  const sk_binning b = detail::to_c(BinningConfig<T>{}, 16);
  d.check(sk_preprocess(d.ctx(), ds.handle(), &c, &b, d.frame()));
  int32_t vis = 0;
  float mu[2], cov[4], con[4], depth, col[3], op;
  sk_projected out{&vis, mu, cov, con, &depth, col, &op, nullptr};
  d.check(sk_frame_get_projected(d.ctx(), d.frame(), &out));
  if (!vis) return std::nullopt;
  ProjectedGaussian<T> pg;
  pg.mu2d = Vec2<T>(T(mu[0]), T(mu[1]));
  for (int r = 0; r < 2; ++r)
    for (int k = 0; k < 2; ++k) {
      pg.cov2d(r, k) = T(cov[2 * r + k]);
      pg.cov2d_inv(r, k) = T(con[2 * r + k]);
    }
  pg.depth = T(depth);
  pg.color = Vec3<T>(T(col[0]), T(col[1]), T(col[2]));
  pg.opacity = T(op);
  pg.source_index = source_index;
  return pg;
}

// project_scene (camera.hpp:137-144): the non-culled footprints in scene order.
template <typename T>
inline std::vector<ProjectedGaussian<T>> project_scene(const Scene<T>& scene, const Camera<T>& cam) {
  detail::DeviceScene ds(scene);
  Device& d = detail::dev();
  const sk_camera c = detail::to_c(cam);
  const sk_binning b = detail::to_c(BinningConfig<T>{}, 16);
  d.check(sk_preprocess(d.ctx(), ds.handle(), &c, &b, d.frame()));
  const size_t n = size_t(scene.size());
  std::vector<int32_t> vis(n);
  std::vector<float> mu(2 * n), cov(4 * n), con(4 * n), depth(n), col(3 * n), op(n);
  sk_projected out{vis.data(), mu.data(), cov.data(), con.data(), depth.data(), col.data(), op.data(), nullptr};
  d.check(sk_frame_get_projected(d.ctx(), d.frame(), &out));
  std::vector<ProjectedGaussian<T>> pgs;
  for (size_t i = 0; i < n; ++i) {
    if (!vis[i]) continue;
    ProjectedGaussian<T> pg;
    pg.mu2d = Vec2<T>(T(mu[2 * i]), T(mu[2 * i + 1]));
    for (int r = 0; r < 2; ++r)
      for (int k = 0; k < 2; ++k) {
        pg.cov2d(r, k) = T(cov[4 * i + 2 * r + k]);
        pg.cov2d_inv(r, k) = T(con[4 * i + 2 * r + k]);
      }
    pg.depth = T(depth[i]);
    pg.color = Vec3<T>(T(col[3 * i]), T(col[3 * i + 1]), T(col[3 * i + 2]));
    pg.opacity = T(op[i]);
    pg.source_index = int(i);
    pgs.push_back(pg);
  }
  return pgs;
}

// cov_grad_from_inv_grad (camera.hpp:148-150): -(inv * d_inv * inv).
template <typename T>
inline Mat2<T> cov_grad_from_inv_grad(const Mat2<T>& inv, const Mat2<T>& d_inv) {
  Mat2<T> a, out;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) a(r, c) = inv(r, 0) * d_inv(0, c) + inv(r, 1) * d_inv(1, c);
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) out(r, c) = -(a(r, 0) * inv(0, c) + a(r, 1) * inv(1, c));
  return out;
}

// project_backward (camera.hpp:156-213): the exact adjoint for one Gaussian.
template <typename T>
inline GaussianGrads<T> project_backward(const Gaussian3D<T>& g, const Camera<T>& cam, int sh_degree,
                                         const Vec2<T>& d_mu2d, const Mat2<T>& d_cov2d, const Vec3<T>& d_color,
                                         T d_opacity) {
  Scene<T> one;
  one.sh_degree = sh_degree;
  one.gaussians.push_back(g);
  detail::DeviceScene ds(one);
  Device& d = detail::dev();
  const sk_camera c = detail::to_c(cam);
  const float dm[2] = {float(d_mu2d[0]), float(d_mu2d[1])};
  const float dc[4] = {float(d_cov2d(0, 0)), float(d_cov2d(0, 1)), float(d_cov2d(1, 0)), float(d_cov2d(1, 1))};
  const float dcol[3] = {float(d_color[0]), float(d_color[1]), float(d_color[2])};
  const float dop = float(d_opacity);
  std::vector<float> grads(size_t(SK_COMP_COUNT(sh_degree)));
  d.check(sk_project_backward_explicit(d.ctx(), ds.handle(), &c, dm, dc, dcol, &dop, grads.data()));
  GaussianGrads<T> out;
  for (int k = 0; k < 3; ++k) out.mu[k] = T(grads[SK_COMP_MU + k]);
  for (int k = 0; k < 4; ++k) out.rot[k] = T(grads[SK_COMP_ROT + k]);
  for (int k = 0; k < 3; ++k) out.log_scale[k] = T(grads[SK_COMP_LOG_SCALE + k]);
  out.opacity_logit = T(grads[SK_COMP_OPACITY]);
  out.sh = ShMatrix<T>::Zero(g.sh.rows(), 3);
  for (int k = 0; k < sh_coeff_count(sh_degree); ++k)
    for (int ch = 0; ch < 3; ++ch) out.sh(k, ch) = T(grads[SK_COMP_SH + 3 * k + ch]);
  return out;
}

// build_tile_grid (raster.hpp:157-168): per-tile lists of projected indices
// in global (depth, index) order.
template <typename T>
inline TileGrid build_tile_grid(const std::vector<ProjectedGaussian<T>>& pgs, int width, int height,
                                const BinningConfig<T>& binning, int tile_size = 16) {
  Device& d = detail::dev();
  detail::inject(pgs, width, height, detail::to_c(binning, tile_size));
  int64_t pairs = 0;
  d.check(sk_bin_sort(d.ctx(), d.frame(), &pairs));
  TileGrid g = make_tile_grid(width, height, tile_size);
  std::vector<int32_t> ranges(2 * size_t(g.tile_count())), values(size_t(std::max<int64_t>(pairs, 1)));
  d.check(sk_frame_get_tile_lists(d.ctx(), d.frame(), ranges.data(), values.data()));
  for (int t = 0; t < g.tile_count(); ++t)
    g.tiles[t].assign(values.begin() + ranges[2 * t], values.begin() + ranges[2 * t + 1]);
  return g;
}

inline std::int64_t count_pairs(const TileGrid& grid) {
  std::int64_t total = 0;
  for (const auto& t : grid.tiles) total += std::int64_t(t.size());
  return total;
}

// blend_forward (raster.hpp:194-248) over exactly the grid's lists. With a
// mask and counter, every contribution on a masked pixel increments the
// counter of its source Gaussian. `workers` is accepted for API parity.
template <typename T>
inline RenderOutputs<T> blend_forward(const TileGrid& grid, const std::vector<ProjectedGaussian<T>>& pgs,
                                      const MaskMap* mask = nullptr, FootprintCounter* counter = nullptr,
                                      int workers = 1) {
  (void)workers;
  Device& d = detail::dev();
  detail::inject(pgs, grid.width, grid.height, detail::to_c(BinningConfig<T>{}, grid.tile_size));
  detail::set_lists(grid);
  std::vector<int32_t> counts;
  std::vector<uint8_t> mrows;
  const bool count = mask && counter;
  if (count) {
    require(mask->rows() == grid.height && mask->cols() == grid.width, "blend_forward: mask size mismatch");
    mrows = detail::rows_from_map(*mask);
    counts.assign(std::max<size_t>(pgs.size(), 1), 0);
  }
  d.check(sk_render_forward(d.ctx(), d.frame(), count ? mrows.data() : nullptr, count ? counts.data() : nullptr));
  if (count)
    for (size_t i = 0; i < pgs.size(); ++i)
      if (counts[i]) counter->counts.at(size_t(pgs[i].source_index)) += counts[i];
  RenderOutputs<T> out;
  const size_t npx = size_t(grid.width) * grid.height;
  std::vector<float> img(3 * npx), tr(npx);
  std::vector<int32_t> cc(npx);
  d.check(sk_frame_get_image(d.ctx(), d.frame(), img.data()));
  d.check(sk_frame_get_transmittance(d.ctx(), d.frame(), tr.data()));
  d.check(sk_frame_get_contrib_count(d.ctx(), d.frame(), cc.data()));
  out.image = detail::image_from<T>(img, grid.width, grid.height);
  out.transmittance = detail::map_from_rows<T>(tr, grid.height, grid.width);
  out.contrib_count = detail::map_from_rows<int>(cc, grid.height, grid.width);
  return out;
}

// blend_backward (raster.hpp:281-355) over the grid's lists: per projected
// Gaussian gradients of the image loss (full-matrix d_conic convention).
template <typename T>
inline BlendGrads<T> blend_backward(const TileGrid& grid, const std::vector<ProjectedGaussian<T>>& pgs,
                                    const Image<T>& d_image, int workers = 1) {
  (void)workers;
  require(d_image.width == grid.width && d_image.height == grid.height, "blend_backward: d_image size mismatch");
  Device& d = detail::dev();
  detail::inject(pgs, grid.width, grid.height, detail::to_c(BinningConfig<T>{}, grid.tile_size));
  detail::set_lists(grid);
  d.check(sk_render_forward(d.ctx(), d.frame(), nullptr, nullptr));
  const auto up = detail::hwc(d_image);
  d.check(sk_frame_set_dimage(d.ctx(), d.frame(), up.data()));
  d.check(sk_render_backward(d.ctx(), d.frame()));
  const size_t n = pgs.size();
  std::vector<float> dm(2 * n + 1), dc(4 * n + 1), dcol(3 * n + 1), dop(n + 1), ab(2 * n + 1);
  sk_blend_grads g{dm.data(), dc.data(), dcol.data(), dop.data(), ab.data()};
  d.check(sk_frame_get_blend_grads(d.ctx(), d.frame(), &g));
  BlendGrads<T> out;
  out.d_mu2d.resize(n);
  out.d_conic.resize(n);
  out.d_color.resize(n);
  out.d_opacity.resize(n);
  out.abs_grad.resize(n);
  for (size_t i = 0; i < n; ++i) {
    out.d_mu2d[i] = Vec2<T>(T(dm[2 * i]), T(dm[2 * i + 1]));
    out.abs_grad[i] = Vec2<T>(T(ab[2 * i]), T(ab[2 * i + 1]));
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) out.d_conic[i](r, c) = T(dc[4 * i + 2 * r + c]);
    out.d_color[i] = Vec3<T>(T(dcol[3 * i]), T(dcol[3 * i + 1]), T(dcol[3 * i + 2]));
    out.d_opacity[i] = T(dop[i]);
  }
  return out;
}

// ---- metrics.hpp / loss.hpp / error_maps.hpp --------------------------------------
template <typename T>
inline T ssim(const Image<T>& a, const Image<T>& b) {
  require(a.width == b.width && a.height == b.height, "ssim: image dimensions differ");
  Device& d = detail::dev();
  const auto x = detail::hwc(a), y = detail::hwc(b);
  double s = 0, p = 0;
  d.check(sk_ssim(d.ctx(), x.data(), y.data(), a.width, a.height, &s, &p));
  return T(s);
}

template <typename T>
inline double psnr(const Image<T>& a, const Image<T>& b) {
  require(a.width == b.width && a.height == b.height, "psnr: image dimensions differ");
  Device& d = detail::dev();
  const auto x = detail::hwc(a), y = detail::hwc(b);
  double s = 0, p = 0;
  d.check(sk_ssim(d.ctx(), x.data(), y.data(), a.width, a.height, &s, &p));
  return p;
}

template <typename T>
struct LossResult {
  T loss = T(0), l1 = T(0), ssim_value = T(0);
  Image<T> d_image;
};

// training_loss (loss.hpp:21-47): (1 - lambda) L1 + lambda (1 - SSIM) and dL/dimage.
template <typename T>
inline LossResult<T> training_loss(const Image<T>& rendered, const Image<T>& ground_truth, T lambda) {
  require(rendered.width == ground_truth.width && rendered.height == ground_truth.height,
          "ssim: image dimensions differ");
  Device& d = detail::dev();
  const auto r = detail::hwc(rendered), g = detail::hwc(ground_truth);
  d.check(sk_frame_set_image(d.ctx(), d.frame(), r.data(), rendered.width, rendered.height));
  sk_loss_values v{};
  d.check(sk_loss(d.ctx(), d.frame(), g.data(), float(lambda), &v));
  std::vector<float> dimg(r.size());
  d.check(sk_frame_get_dimage(d.ctx(), d.frame(), dimg.data()));
  LossResult<T> out;
  out.loss = T(v.loss);
  out.l1 = T(v.l1);
  out.ssim_value = T(v.ssim);
  out.d_image = detail::image_from<T>(dimg, rendered.width, rendered.height);
  return out;
}

template <typename T>
struct ErrorMaps {
  ScalarMap<T> raw, normalized;
  MaskMap mask;
  T photometric = T(0);
};

// build_error_maps (error_maps.hpp:22-43).
template <typename T>
inline ErrorMaps<T> build_error_maps(const Image<T>& rendered, const Image<T>& ground_truth, T tau, T lambda) {
  require(rendered.width == ground_truth.width && rendered.height == ground_truth.height,
          "ssim: image dimensions differ");
  Device& d = detail::dev();
  const int w = rendered.width, h = rendered.height;
  const auto r = detail::hwc(rendered), g = detail::hwc(ground_truth);
  std::vector<float> raw(size_t(w) * h), nrm(size_t(w) * h);
  std::vector<uint8_t> mask(size_t(w) * h);
  float photo = 0;
  d.check(sk_error_maps(d.ctx(), r.data(), g.data(), w, h, float(tau), float(lambda), raw.data(), nrm.data(),
                        mask.data(), &photo));
  ErrorMaps<T> out;
  out.raw = detail::map_from_rows<T>(raw, h, w);
  out.normalized = detail::map_from_rows<T>(nrm, h, w);
  out.mask = detail::map_from_rows<std::uint8_t>(mask, h, w);
  out.photometric = T(photo);
  return out;
}

// ---- adc.hpp ----------------------------------------------------------------------
template <typename T>
struct ScoreTable {
  std::vector<T> s_d, s_p_raw, s_p, grad_norm_acc, abs_grad_acc;
  std::vector<Vec3<T>> grad3d_acc;
  std::vector<int> views_seen;
  std::vector<T> max_radius2d;
  void reset(int n) {
    s_d.assign(n, T(0));
    s_p_raw.assign(n, T(0));
    s_p.assign(n, T(0));
    grad_norm_acc.assign(n, T(0));
    abs_grad_acc.assign(n, T(0));
    grad3d_acc.assign(n, Vec3<T>::Zero());
    views_seen.assign(n, 0);
    max_radius2d.assign(n, T(0));
  }
  int size() const { return int(s_d.size()); }
};

// minmax_normalize (adc.hpp:48-56): zeros for a degenerate population.
template <typename T>
inline std::vector<T> minmax_normalize(const std::vector<T>& v) {
  if (v.empty()) return {};
  const auto [lo_it, hi_it] = std::minmax_element(v.begin(), v.end());
  const T lo = *lo_it, hi = *hi_it;
  std::vector<T> out(v.size(), T(0));
  if (hi > lo)
    for (size_t i = 0; i < v.size(); ++i) out[i] = (v[i] - lo) / (hi - lo);
  return out;
}

template <typename T>
struct ViewRef {
  const Camera<T>* camera = nullptr;
  const Image<T>* image = nullptr;
};

// scores_from_counts (adc.hpp:69-84) on the GPU (K13).
template <typename T>
inline void scores_from_counts(const std::vector<std::vector<int>>& counts, const std::vector<T>& photometric,
                               ScoreTable<T>& table) {
  require(!counts.empty() && counts.size() == photometric.size(),
          "scores_from_counts: need one count row and one photometric value per view");
  const int k = int(counts.size());
  const size_t n = counts[0].size();
  std::vector<int32_t> rows;
  rows.reserve(k * n);
  for (const auto& r : counts) {
    require(r.size() == n, "scores_from_counts: count rows differ in length");
    rows.insert(rows.end(), r.begin(), r.end());
  }
  std::vector<float> ph(photometric.begin(), photometric.end()), sd(n), spr(n), sp(n);
  Device& d = detail::dev();
  d.check(sk_scores_from_counts(d.ctx(), rows.data(), ph.data(), k, int64_t(n), sd.data(), spr.data(), sp.data()));
  table.s_d.assign(sd.begin(), sd.end());
  table.s_p_raw.assign(spr.begin(), spr.end());
  table.s_p.assign(sp.begin(), sp.end());
}

// accumulate_scores (adc.hpp:91-115): per view render, error maps, masked
// footprint counts (K6 + K11 + K12), then K13. `workers` is accepted for API parity.
template <typename T>
inline void accumulate_scores(const Scene<T>& scene, const std::vector<ViewRef<T>>& views, T tau, T lambda,
                              const BinningConfig<T>& binning, int tile_size, ScoreTable<T>& table,
                              int workers = 1) {
  (void)workers;
  require(!views.empty(), "accumulate_scores: no training views");
  Device& d = detail::dev();
  detail::DeviceScene ds(scene);
  std::vector<sk_camera> cams;
  std::vector<float> images;
  for (const auto& v : views) {
    require(v.camera && v.image, "accumulate_scores: null view");
    require(v.image->width == v.camera->width && v.image->height == v.camera->height,
            "accumulate_scores: image size differs from its camera");
    cams.push_back(detail::to_c(*v.camera));
    const auto img = detail::hwc(*v.image);
    images.insert(images.end(), img.begin(), img.end());
  }
  const sk_binning b = detail::to_c(binning, tile_size);
  d.check(sk_accumulate_scores(d.ctx(), ds.handle(), int(views.size()), cams.data(), images.data(), float(tau),
                               float(lambda), &b, nullptr, nullptr));
  const size_t n = size_t(scene.size());
  std::vector<float> sd(n + 1), spr(n + 1), sp(n + 1);
  sk_score_table st{};
  st.s_d = sd.data();
  st.s_p_raw = spr.data();
  st.s_p = sp.data();
  d.check(sk_scene_get_score_table(d.ctx(), ds.handle(), &st));
  table.s_d.assign(sd.begin(), sd.begin() + n);
  table.s_p_raw.assign(spr.begin(), spr.begin() + n);
  table.s_p.assign(sp.begin(), sp.begin() + n);
}

template <typename T>
struct DensifyParams {
  T tau_d = T(5);
  T grad_threshold = T(2e-4);
  T percent_dense = T(0.01);
  bool use_vcd = true;
};

struct DensifySelection {
  std::vector<int> clone;
  std::vector<int> split;
};

// select_densify (adc.hpp:135-153) on the GPU (K14); ascending index lists.
template <typename T>
inline DensifySelection select_densify(const ScoreTable<T>& table, const Scene<T>& scene,
                                       const DensifyParams<T>& params, T scene_extent) {
  const int n = scene.size();
  require(table.size() == n || n == 0, "select_densify: score table size differs from the scene");
  DensifySelection sel;
  if (n == 0) return sel;
  Device& d = detail::dev();
  detail::DeviceScene ds(scene);
  ds.set_table(table);
  std::vector<uint8_t> clone(n), split(n);
  d.check(sk_select_densify(d.ctx(), ds.handle(), float(params.tau_d), float(params.grad_threshold),
                            float(params.percent_dense), params.use_vcd ? 1 : 0, float(scene_extent), clone.data(),
                            split.data()));
  sel.clone = detail::indices(clone);
  sel.split = detail::indices(split);
  return sel;
}

struct IndexRemap {
  std::vector<int> old_to_new;
  int new_size = 0;
};

namespace detail {
inline void check_ascending(const std::vector<int>& v, const char* what) {
  for (size_t i = 1; i < v.size(); ++i)
    if (!(v[i - 1] < v[i])) throw std::invalid_argument(std::string(what) + ": indices must be strictly ascending");
}

template <typename T>
inline IndexRemap compact(Scene<T>& scene, const std::vector<uint8_t>* prune, const std::vector<uint8_t>* clone,
                          const std::vector<uint8_t>* split, const ScoreTable<T>* table, T clone_step_lr,
                          const std::vector<float>& eps) {
  const int n = scene.size();
  const int64_t cap = int64_t(n) + (clone ? std::count(clone->begin(), clone->end(), 1) : 0) +
                      2 * (split ? std::count(split->begin(), split->end(), 1) : 0);
  DeviceScene ds(scene, cap);
  if (table) ds.set_table(*table);
  IndexRemap r;
  r.old_to_new.assign(size_t(n), -1);
  int64_t nn = 0;
  Device& d = dev();
  d.check(sk_apply_prune_densify(d.ctx(), ds.handle(), prune ? prune->data() : nullptr,
                                 clone ? clone->data() : nullptr, split ? split->data() : nullptr,
                                 float(clone_step_lr), eps.empty() ? nullptr : eps.data(),
                                 n ? r.old_to_new.data() : nullptr, &nn));
  ds.download(scene);
  r.new_size = int(nn);
  return r;
}
}  // namespace detail

// apply_densify (adc.hpp:166-205): non-split survivors, then clones (offset
// by one positional-gradient step), then split children in pairs with
// noise drawn from rng (6 normals per split, in order).
template <typename T>
inline IndexRemap apply_densify(Scene<T>& scene, const std::vector<int>& clone, const std::vector<int>& split,
                                const ScoreTable<T>& table, T clone_step_lr, Rng& rng) {
  detail::check_ascending(clone, "apply_densify");
  detail::check_ascending(split, "apply_densify");
  const auto fc = detail::flags(clone, scene.size(), "apply_densify");
  const auto fs = detail::flags(split, scene.size(), "apply_densify");
  std::vector<float> eps;
  eps.reserve(6 * split.size());
  for (size_t i = 0; i < 6 * split.size(); ++i) eps.push_back(float(T(rng.normal())));
  return detail::compact(scene, nullptr, &fc, &fs, &table, clone_step_lr, eps);
}

template <typename T>
struct PruneParams {
  T tau_p = T(0.9);
  T min_opacity = T(0.005);
  T opacity_late = T(0.1);
  T world_size_frac = T(0.1);
  T screen_size = T(20);
  int size_prune_from = 3000;
  int densify_until = 15000;
  bool use_vcp = true;
};

// select_prune (adc.hpp:223-270) on the GPU (K14 + the VCP ordering);
// ascending index list, never the whole scene.
template <typename T>
inline std::vector<int> select_prune(const ScoreTable<T>& table, const Scene<T>& scene, int iteration,
                                     const PruneParams<T>& params, T scene_extent) {
  const int n = scene.size();
  if (n == 0) return {};
  require(table.size() == n, "select_prune: score table size differs from the scene");
  Device& d = detail::dev();
  detail::DeviceScene ds(scene);
  ds.set_table(table);
  sk_prune_params pp{float(params.tau_p),      float(params.min_opacity), float(params.opacity_late),
                     float(params.world_size_frac), float(params.screen_size), params.size_prune_from,
                     params.densify_until,     params.use_vcp ? 1 : 0};
  std::vector<uint8_t> prune(n);
  d.check(sk_select_prune(d.ctx(), ds.handle(), iteration, &pp, float(scene_extent), prune.data()));
  return detail::indices(prune);
}

// apply_prune (adc.hpp:272-289): stable compaction.
template <typename T>
inline IndexRemap apply_prune(Scene<T>& scene, const std::vector<int>& prune) {
  const auto fp = detail::flags(prune, scene.size(), "apply_prune");
  return detail::compact<T>(scene, &fp, nullptr, nullptr, nullptr, T(0), {});
}

// ---- adam.hpp ---------------------------------------------------------------------
template <typename T>
inline T expon_lr(T lr_init, T lr_final, int step, int max_steps) {
  const T t = std::clamp(T(step) / T(std::max(1, max_steps)), T(0), T(1));
  return std::exp((T(1) - t) * std::log(lr_init) + t * std::log(lr_final));
}

template <typename T>
struct LearningRates {
  T position = T(1.6e-4);
  T position_final = T(1.6e-6);
  T sh_dc = T(2.5e-3);
  T sh_rest = T(2.5e-3 / 20);
  T opacity = T(5e-2);
  T scale = T(5e-3);
  T rotation = T(1e-3);
};

template <typename T>
struct SceneGrads {
  std::vector<GaussianGrads<T>> per_gaussian;
  void init(const Scene<T>& scene) {
    per_gaussian.assign(scene.size(), GaussianGrads<T>{});
    for (auto& g : per_gaussian) g.sh = ShMatrix<T>::Zero(sh_coeff_count(scene.sh_degree), 3);
  }
};

// SceneOptimizer (adam.hpp:99-164): the Adam moments of the six groups live
// on the GPU (K10); the scene passed to step() is read and written back.
template <typename T>
class SceneOptimizer {
 public:
  SceneOptimizer() = default;
  SceneOptimizer(const SceneOptimizer&) = delete;
  SceneOptimizer& operator=(const SceneOptimizer&) = delete;
  ~SceneOptimizer() {
    if (h_) sk_scene_destroy(h_);
  }

  void init(const Scene<T>& scene) {
    Device& d = detail::dev();
    if (h_) sk_scene_destroy(h_);
    h_ = nullptr;
    deg_ = scene.sh_degree;
    d.check(sk_scene_create(d.ctx(), deg_, scene.size(), &h_));
    const auto p = detail::planar(scene);
    d.check(sk_scene_upload(d.ctx(), h_, p.data(), scene.size()));
  }

  void remap(const IndexRemap& r) {
    Device& d = detail::dev();
    require(h_ && int64_t(r.old_to_new.size()) == size(), "SceneOptimizer::remap: remap size differs");
    d.check(sk_scene_remap_moments(d.ctx(), h_, r.old_to_new.data(), r.new_size));
  }

  void step(Scene<T>& scene, const SceneGrads<T>& grads, const LearningRates<T>& lrs, T position_lr,
            bool update_sh_rest = true) {
    prepare(scene);
    const int n = scene.size();
    std::vector<float> g(size_t(SK_COMP_COUNT(deg_)) * n, 0.0f);
    for (int i = 0; i < n; ++i) {
      const auto& gi = grads.per_gaussian.at(size_t(i));
      for (int k = 0; k < 3; ++k) g[size_t(SK_COMP_MU + k) * n + i] = float(gi.mu[k]);
      for (int k = 0; k < 4; ++k) g[size_t(SK_COMP_ROT + k) * n + i] = float(gi.rot[k]);
      for (int k = 0; k < 3; ++k) g[size_t(SK_COMP_LOG_SCALE + k) * n + i] = float(gi.log_scale[k]);
      g[size_t(SK_COMP_OPACITY) * n + i] = float(gi.opacity_logit);
      for (int k = 0; k < sh_coeff_count(deg_); ++k)
        for (int c = 0; c < 3; ++c) g[size_t(SK_COMP_SH + 3 * k + c) * n + i] = float(gi.sh(k, c));
    }
    Device& d = detail::dev();
    d.check(sk_scene_set_grads(d.ctx(), h_, g.data()));
    const sk_learning_rates l = c_lrs(lrs);
    d.check(sk_adam_step(d.ctx(), h_, &l, float(position_lr), update_sh_rest ? 1 : 0));
    detail::DeviceSceneView(h_, deg_).download(scene);
  }

  void step_sh_rest(Scene<T>& scene, const std::vector<ShMatrix<T>>& rest_grads, const LearningRates<T>& lrs) {
    if (sh_coeff_count(deg_) <= 1) return;
    prepare(scene);
    const int n = scene.size();
    std::vector<float> g(size_t(SK_COMP_COUNT(deg_)) * n, 0.0f);
    for (int i = 0; i < n; ++i)
      for (int k = 1; k < sh_coeff_count(deg_); ++k)
        for (int c = 0; c < 3; ++c) g[size_t(SK_COMP_SH + 3 * k + c) * n + i] = float(rest_grads.at(i)(k, c));
    Device& d = detail::dev();
    d.check(sk_scene_set_grads(d.ctx(), h_, g.data()));
    const sk_learning_rates l = c_lrs(lrs);
    d.check(sk_adam_step_sh_rest(d.ctx(), h_, &l));
    detail::DeviceSceneView(h_, deg_).download(scene);
  }

  void reset_opacity_state() {
    if (h_) detail::dev().check(sk_adam_reset_opacity_state(detail::dev().ctx(), h_));
  }

  // Moments (planar [C][n]) and the six group step counters, for inspection.
  void moments(std::vector<float>* m, std::vector<float>* v, int64_t t6[6]) const {
    const int64_t n = size();
    if (m) m->resize(size_t(SK_COMP_COUNT(deg_)) * n);
    if (v) v->resize(size_t(SK_COMP_COUNT(deg_)) * n);
    detail::dev().check(sk_scene_get_adam(detail::dev().ctx(), h_, m ? m->data() : nullptr,
                                          v ? v->data() : nullptr, t6));
  }

 private:
  int64_t size() const {
    int64_t n = 0;
    if (h_) sk_scene_size(h_, &n);
    return n;
  }
  void prepare(const Scene<T>& scene) {
    require(h_ != nullptr, "SceneOptimizer: init() first");
    require(scene.sh_degree == deg_ && int64_t(scene.size()) == size(),
            "SceneOptimizer: scene differs from the optimizer state (init / remap)");
    const auto p = detail::planar(scene);
    detail::dev().check(sk_scene_set_params(detail::dev().ctx(), h_, p.data(), scene.size()));
  }
  static sk_learning_rates c_lrs(const LearningRates<T>& l) {
    return sk_learning_rates{float(l.position), float(l.position_final), float(l.sh_dc), float(l.sh_rest),
                             float(l.opacity),  float(l.scale),          float(l.rotation)};
  }
  sk_scene* h_ = nullptr;
  int deg_ = 3;
};

// ---- config.hpp ---------------------------------------------------------------------
struct TrainConfig {
  int iterations = 30000;
  int k = 10;
  double lambda = 0.2;
  double tau = 0.5;
  double tau_d = 5.0;
  double tau_p = 0.9;
  double beta = 1.0;
  double tau_alpha = 1.0 / 255;
  int densify_from = 500;
  int densify_until = 15000;
  int densify_every = 500;
  int prune_every_early = 500;
  int prune_every_late = 3000;
  double grad_threshold = 2e-4;
  double percent_dense = 0.01;
  double lr_position = 1.6e-4;
  double lr_position_final = 1.6e-6;
  double lr_sh_dc = 2.5e-3;
  double lr_sh_rest = 2.5e-3 / 20;
  double lr_opacity = 5e-2;
  double lr_scale = 5e-3;
  double lr_rotation = 1e-3;
  int opacity_reset_every = 0;
  bool lazy_opt_enabled = false;
  int lazy_opt_interval_15k = 32;
  int lazy_opt_interval_20k = 64;
  std::uint64_t seed = 0;
  int tile_size = 16;
  int workers = 1;
  int sh_degree = 3;
  std::string bin_mode = "aabb";
  bool vcd = true;
  bool vcp = true;
  double prune_min_opacity = 0.005;
  double prune_opacity_late = 0.1;
  double prune_world_size_frac = 0.1;
  double prune_screen_size = 20.0;
  int size_prune_from = 3000;
  bool schedule_dry_run = false;

  sk_train_config to_c() const {
    sk_train_config c;
    sk_default_config(&c);
    c.iterations = iterations;
    c.k = k;
    c.lambda = lambda;
    c.tau = tau;
    c.tau_d = tau_d;
    c.tau_p = tau_p;
    c.beta = beta;
    c.tau_alpha = tau_alpha;
    c.densify_from = densify_from;
    c.densify_until = densify_until;
    c.densify_every = densify_every;
    c.prune_every_early = prune_every_early;
    c.prune_every_late = prune_every_late;
    c.grad_threshold = grad_threshold;
    c.percent_dense = percent_dense;
    c.lr_position = lr_position;
    c.lr_position_final = lr_position_final;
    c.lr_sh_dc = lr_sh_dc;
    c.lr_sh_rest = lr_sh_rest;
    c.lr_opacity = lr_opacity;
    c.lr_scale = lr_scale;
    c.lr_rotation = lr_rotation;
    c.opacity_reset_every = opacity_reset_every;
    c.lazy_opt_enabled = lazy_opt_enabled;
    c.lazy_opt_interval_15k = lazy_opt_interval_15k;
    c.lazy_opt_interval_20k = lazy_opt_interval_20k;
    c.seed = seed;
    c.tile_size = tile_size;
    c.workers = workers;
    c.sh_degree = sh_degree;
    c.compact = bin_mode == "compact" ? 1 : 0;
    c.vcd = vcd;
    c.vcp = vcp;
    c.prune_min_opacity = prune_min_opacity;
    c.prune_opacity_late = prune_opacity_late;
    c.prune_world_size_frac = prune_world_size_frac;
    c.prune_screen_size = prune_screen_size;
    c.size_prune_from = size_prune_from;
    c.schedule_dry_run = schedule_dry_run;
    return c;
  }
  void from_c(const sk_train_config& c) {
    iterations = c.iterations;
    k = c.k;
    lambda = c.lambda;
    tau = c.tau;
    tau_d = c.tau_d;
    tau_p = c.tau_p;
    beta = c.beta;
    tau_alpha = c.tau_alpha;
    densify_from = c.densify_from;
    densify_until = c.densify_until;
    densify_every = c.densify_every;
    prune_every_early = c.prune_every_early;
    prune_every_late = c.prune_every_late;
    grad_threshold = c.grad_threshold;
    percent_dense = c.percent_dense;
    lr_position = c.lr_position;
    lr_position_final = c.lr_position_final;
    lr_sh_dc = c.lr_sh_dc;
    lr_sh_rest = c.lr_sh_rest;
    lr_opacity = c.lr_opacity;
    lr_scale = c.lr_scale;
    lr_rotation = c.lr_rotation;
    opacity_reset_every = c.opacity_reset_every;
    lazy_opt_enabled = c.lazy_opt_enabled != 0;
    lazy_opt_interval_15k = c.lazy_opt_interval_15k;
    lazy_opt_interval_20k = c.lazy_opt_interval_20k;
    seed = c.seed;
    tile_size = c.tile_size;
    workers = c.workers;
    sh_degree = c.sh_degree;
    bin_mode = c.compact ? "compact" : "aabb";
    vcd = c.vcd != 0;
    vcp = c.vcp != 0;
    prune_min_opacity = c.prune_min_opacity;
    prune_opacity_late = c.prune_opacity_late;
    prune_world_size_frac = c.prune_world_size_frac;
    prune_screen_size = c.prune_screen_size;
    size_prune_from = c.size_prune_from;
    schedule_dry_run = c.schedule_dry_run != 0;
  }
  // TrainConfig::validate (config.hpp:63-80), same messages.
  void validate() const {
    if (bin_mode != "aabb" && bin_mode != "compact")
      throw std::invalid_argument("config: bin_mode must be 'aabb' or 'compact'");
    const sk_train_config c = to_c();
    detail::dev().check(sk_validate_config(detail::dev().ctx(), &c));
  }
};

// set_config_value (config.hpp:135-160) / load_config_file (:162-188).
inline void set_config_value(TrainConfig& cfg, const std::string& key, const std::string& value) {
  sk_train_config c = cfg.to_c();
  detail::dev().check(sk_config_set(detail::dev().ctx(), &c, key.c_str(), value.c_str()));
  cfg.from_c(c);
}
inline void load_config_file(TrainConfig& cfg, const std::string& path) {
  sk_train_config c = cfg.to_c();
  detail::dev().check(sk_config_load_file(detail::dev().ctx(), &c, path.c_str()));
  cfg.from_c(c);
}

// ---- dataset.hpp ----------------------------------------------------------------------
template <typename T>
struct Dataset {
  std::vector<Camera<T>> cameras;
  std::vector<int> camera_ids;
  std::vector<Image<T>> images;
  std::vector<std::pair<Vec3<T>, Vec3<T>>> init_points;
  std::vector<int> train_indices;
  std::vector<int> test_indices;
  T extent = T(1);
};

// ---- trainer.hpp ----------------------------------------------------------------------
struct LogRow {
  int iteration = 0;
  double loss = 0;
  double psnr = 0;
  int gaussians = 0;
  std::int64_t tile_pairs = 0;
  double elapsed_ms = 0;
};

struct TrainCallbacks {
  std::function<void(int)> on_densify_event;
  std::function<void(int)> on_prune_event;
  std::function<void(int)> on_iteration;
};

template <typename T>
struct TrainResult {
  Scene<T> scene;
  std::vector<LogRow> log;
};

inline bool densify_due(int iteration, const TrainConfig& cfg) {
  return iteration >= cfg.densify_from && iteration <= cfg.densify_until && iteration % cfg.densify_every == 0;
}
inline bool prune_due(int iteration, const TrainConfig& cfg) {
  if (iteration >= cfg.densify_from && iteration <= cfg.densify_until) return iteration % cfg.prune_every_early == 0;
  if (iteration > cfg.densify_until) return (iteration - cfg.densify_until) % cfg.prune_every_late == 0;
  return false;
}
inline bool lazy_update_due(int iteration, const TrainConfig& cfg) {
  if (!cfg.lazy_opt_enabled || iteration < 15000) return true;
  if (iteration < 20000) return iteration % cfg.lazy_opt_interval_15k == 0;
  return iteration % cfg.lazy_opt_interval_20k == 0;
}

namespace detail {
template <typename T>
inline uint8_t quantize(T v) {
  const double c = std::min(std::max(double(v), 0.0), 1.0);
  return uint8_t(std::lround(float(c) * 255.0f));
}
}  // namespace detail

// Trainer (trainer.hpp:67-261) on the GPU: the scene (held by value, as the
// reference) lives on the device between calls; the dataset is borrowed.
template <typename T>
class Trainer {
 public:
  Trainer(Scene<T> scene, const Dataset<T>& data, const TrainConfig& cfg) : cfg_(cfg), host_(std::move(scene)) {
    cfg_.validate();
    require(!data.cameras.empty(), "trainer: dataset has no views");
    require(!data.train_indices.empty(), "trainer: dataset has no training views");
    require(data.images.size() == data.cameras.size(), "trainer: one image per camera");
    Device& d = detail::dev();
    d.check(sk_scene_create(d.ctx(), host_.sh_degree, host_.size(), &scene_));
    const auto p = detail::planar(host_);
    d.check(sk_scene_upload(d.ctx(), scene_, p.data(), host_.size()));
    std::vector<sk_camera> cams;
    std::vector<uint8_t> imgs;
    for (size_t v = 0; v < data.cameras.size(); ++v) {
      cams.push_back(detail::to_c(data.cameras[v]));
      const auto& img = data.images[v];
      require(img.width == data.cameras[v].width && img.height == data.cameras[v].height,
              "trainer: image size differs from its camera");
      for (const auto& px : img.pixels)
        for (int c = 0; c < 3; ++c) imgs.push_back(detail::quantize(px[c]));
    }
    std::vector<int32_t> train(data.train_indices.begin(), data.train_indices.end());
    d.check(sk_dataset_create(d.ctx(), int(cams.size()), cams.data(), imgs.data(), train.data(), int(train.size()),
                              float(data.extent), &data_));
    const sk_train_config c = cfg_.to_c();
    d.check(sk_trainer_create(d.ctx(), scene_, data_, &c, &trainer_));
  }
  ~Trainer() {
    if (trainer_) sk_trainer_destroy(trainer_);
    if (data_) sk_dataset_destroy(data_);
    if (scene_) sk_scene_destroy(scene_);
  }
  Trainer(const Trainer&) = delete;
  Trainer& operator=(const Trainer&) = delete;

  // Trainer::run (trainer.hpp:89-119): every iteration's step, the due
  // density event, the opacity reset; the callbacks fire per iteration.
  TrainResult<T> run(const TrainCallbacks& callbacks = {}) {
    Device& d = detail::dev();
    TrainResult<T> result;
    const bool per_iteration = callbacks.on_densify_event || callbacks.on_prune_event || callbacks.on_iteration;
    std::vector<sk_log_row> rows(size_t(std::max(cfg_.iterations, 1)));
    int done = 0;
    int it0 = 0;
    sk_trainer_iteration(trainer_, &it0);
    while (it0 + done < cfg_.iterations) {
      const int chunk = per_iteration ? 1 : cfg_.iterations - it0 - done;
      d.check(sk_trainer_run(trainer_, chunk, rows.data() + done));
      for (int j = 0; j < chunk; ++j) {
        const sk_log_row& r = rows[size_t(done + j)];
        if (densify_due(r.iteration, cfg_) && callbacks.on_densify_event) callbacks.on_densify_event(r.iteration);
        if (prune_due(r.iteration, cfg_) && callbacks.on_prune_event) callbacks.on_prune_event(r.iteration);
        LogRow row;
        row.iteration = r.iteration;
        row.loss = r.loss;
        row.psnr = r.psnr;
        row.gaussians = r.gaussians;
        row.tile_pairs = r.tile_pairs;
        row.elapsed_ms = r.elapsed_ms;
        result.log.push_back(row);
        if (callbacks.on_iteration) callbacks.on_iteration(r.iteration);
      }
      done += chunk;
    }
    result.scene = scene();
    return result;
  }

  const Scene<T>& scene() {
    detail::DeviceSceneView(scene_, host_.sh_degree).download(host_);
    return host_;
  }

 private:
  TrainConfig cfg_;
  Scene<T> host_;
  sk_scene* scene_ = nullptr;
  sk_dataset* data_ = nullptr;
  sk_trainer* trainer_ = nullptr;
};

template <typename T>
inline TrainResult<T> run_training(Scene<T> scene, const Dataset<T>& data, const TrainConfig& cfg,
                                   const TrainCallbacks& callbacks = {}) {
  Trainer<T> trainer(std::move(scene), data, cfg);
  return trainer.run(callbacks);
}

// ---- scene construction, on-disk formats (scene.hpp:117, ply.hpp, png_io.hpp, dataset.hpp)
template <typename T>
inline Scene<T> init_from_points(const std::vector<std::pair<Vec3<T>, Vec3<T>>>& points, int sh_degree = 3) {
  std::vector<float> xyz, rgb;
  for (const auto& [p, c] : points)
    for (int k = 0; k < 3; ++k) {
      xyz.push_back(float(p[k]));
      rgb.push_back(float(c[k]));
    }
  Device& d = detail::dev();
  sk_scene* h = nullptr;
  d.check(sk_init_from_points(d.ctx(), int64_t(points.size()), xyz.data(), rgb.data(), sh_degree, 0, &h));
  std::unique_ptr<sk_scene, int (*)(sk_scene*)> guard(h, sk_scene_destroy);
  Scene<T> s;
  detail::DeviceSceneView(h, sh_degree).download(s);
  return s;
}

template <typename T>
inline void save_checkpoint(const Scene<T>& scene, const std::string& path) {
  detail::DeviceScene ds(scene);
  detail::dev().check(sk_checkpoint_save(detail::dev().ctx(), ds.handle(), path.c_str()));
}

template <typename T>
inline Scene<T> load_checkpoint(const std::string& path) {
  Device& d = detail::dev();
  sk_scene* h = nullptr;
  d.check(sk_checkpoint_load(d.ctx(), path.c_str(), 0, &h));
  std::unique_ptr<sk_scene, int (*)(sk_scene*)> guard(h, sk_scene_destroy);
  int deg = 0;
  sk_scene_sh_degree(h, &deg);
  Scene<T> s;
  detail::DeviceSceneView(h, deg).download(s);
  return s;
}

// read_png (png_io.cpp:25-72): byte / 255.0f. Host-only (no device needed).
inline Image<float> read_png(const std::string& path) {
  int w = 0, h = 0;
  detail::io(sk_png_read(nullptr, path.c_str(), nullptr, &w, &h), "png: cannot read '" + path + "'");
  std::vector<std::uint8_t> rgb(size_t(w) * h * 3);
  detail::io(sk_png_read(nullptr, path.c_str(), rgb.data(), &w, &h), "png: cannot read '" + path + "'");
  Image<float> img(w, h);
  for (size_t i = 0; i < size_t(w) * h; ++i)
    for (int c = 0; c < 3; ++c) img.pixels[i][c] = rgb[3 * i + c] / 255.0f;
  return img;
}

// write_png (png_io.cpp:74-104): lround(clamp(v) * 255). Host-only.
inline void write_png(const std::string& path, const Image<float>& image) {
  const auto rgb = detail::hwc(image);
  detail::io(sk_png_write(nullptr, path.c_str(), rgb.data(), image.width, image.height),
             "png: cannot write '" + path + "'");
}

// read_points_ply / write_points_ply (ply.hpp:196-233). Host-only.
template <typename T = float>
inline std::vector<std::pair<Vec3<T>, Vec3<T>>> read_points_ply(const std::string& path) {
  int64_t n = 0;
  detail::io(sk_points_read(nullptr, path.c_str(), nullptr, nullptr, &n), "ply: cannot read '" + path + "'");
  std::vector<float> xyz(size_t(n) * 3), rgb(size_t(n) * 3);
  detail::io(sk_points_read(nullptr, path.c_str(), xyz.data(), rgb.data(), &n), "ply: cannot read '" + path + "'");
  std::vector<std::pair<Vec3<T>, Vec3<T>>> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      out[i].first[k] = T(xyz[3 * i + k]);
      out[i].second[k] = T(rgb[3 * i + k]);
    }
  return out;
}

template <typename T>
inline void write_points_ply(const std::string& path, const std::vector<std::pair<Vec3<T>, Vec3<T>>>& points) {
  std::vector<float> xyz, rgb;
  for (const auto& [p, c] : points)
    for (int k = 0; k < 3; ++k) {
      xyz.push_back(float(p[k]));
      rgb.push_back(float(c[k]));
    }
  detail::io(sk_points_write(nullptr, path.c_str(), xyz.data(), rgb.data(), int64_t(points.size())),
             "ply: cannot write '" + path + "'");
}

// load_dataset (dataset.hpp:73-125): cameras.json, images/%05d.png, points3d.ply.
template <typename T = float>
inline Dataset<T> load_dataset(const std::string& path) {
  Device& d = detail::dev();
  sk_dataset* ds = nullptr;
  d.check(sk_dataset_load(d.ctx(), path.c_str(), &ds));
  std::unique_ptr<sk_dataset, int (*)(sk_dataset*)> guard(ds, sk_dataset_destroy);
  Dataset<T> out;
  int nv = 0;
  sk_dataset_num_views(ds, &nv);
  for (int v = 0; v < nv; ++v) {
    sk_camera c;
    sk_dataset_camera(ds, v, &c);
    out.cameras.push_back(detail::from_c<T>(c));
    std::vector<std::uint8_t> img(size_t(c.width) * c.height * 3);
    d.check(sk_dataset_image_u8(d.ctx(), ds, v, img.data()));
    Image<T> im(c.width, c.height);
    for (size_t i = 0; i < im.pixels.size(); ++i)
      for (int k = 0; k < 3; ++k) im.pixels[i][k] = T(img[3 * i + k] / 255.0f);
    out.images.push_back(std::move(im));
  }
  int cnt = 0;
  sk_dataset_train_indices(ds, nullptr, &cnt);
  std::vector<int32_t> tr(static_cast<size_t>(cnt));
  sk_dataset_train_indices(ds, tr.data(), &cnt);
  out.train_indices.assign(tr.begin(), tr.end());
  for (int v = 0; v < nv; ++v)
    if (std::find(tr.begin(), tr.end(), v) == tr.end()) out.test_indices.push_back(v);
  int64_t np = 0;
  sk_dataset_init_points(ds, nullptr, nullptr, &np);
  std::vector<float> xyz(size_t(np) * 3), rgb(size_t(np) * 3);
  sk_dataset_init_points(ds, xyz.data(), rgb.data(), &np);
  for (int64_t i = 0; i < np; ++i)
    out.init_points.emplace_back(Vec3<T>(T(xyz[3 * i]), T(xyz[3 * i + 1]), T(xyz[3 * i + 2])),
                                 Vec3<T>(T(rgb[3 * i]), T(rgb[3 * i + 1]), T(rgb[3 * i + 2])));
  std::vector<sk_camera> cams(static_cast<size_t>(nv));
  std::vector<int32_t> ids(static_cast<size_t>(nv));
  int cc = nv;
  if (nv > 0 && sk_cameras_read(nullptr, (path + "/cameras.json").c_str(), cams.data(), ids.data(), &cc) == SK_OK)
    out.camera_ids.assign(ids.begin(), ids.end());
  float ext = 1.0f;
  sk_dataset_extent(ds, &ext);
  out.extent = T(ext);
  return out;
}

// save_cameras_json (dataset.hpp:127-150)
template <typename T>
inline void save_cameras_json(const std::string& path, const std::vector<Camera<T>>& cameras,
                              const std::vector<int>& ids) {
  std::vector<sk_camera> c;
  for (const auto& cam : cameras) c.push_back(detail::to_c(cam));
  std::vector<int32_t> i(ids.begin(), ids.end());
  detail::io(sk_cameras_write(nullptr, path.c_str(), c.data(), i.data(), int(c.size())),
             "dataset: cannot write '" + path + "'");
}

}  // namespace splat
