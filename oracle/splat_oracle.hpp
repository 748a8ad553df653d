// =============================================================================
// TEST INFRASTRUCTURE ONLY — CPU ORACLE. Never linked into the product.
//
// Operation-by-operation C++ restatement of the reference splatkit hot path
// (arxiv 2511.04283; /root/reference/proj/include/splatkit/*.hpp). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
// load it, and only as the checker.
//
// Why a restatement: the reference cannot be compiled here (it needs Eigen3,
// libpng and vendored doctest/CLI11, none present).
// Eigen fixes the small-matrix evaluation order internally; this file fixes
// one explicit order (documented per function) and the CUDA kernels follow
// the same order, so binning keys, tile lists, forward images, transmittance
// and footprint counts are bit-comparable. The oracle is pinned against the
// reference's own known-answer tests (tests/test_oracle_kats.py).
//
// exp/log: the reference calls std::exp/std::log. With g_detmath=true (the
// default for float) the oracle calls sk::det_expf/det_logf instead — the
// deterministic routines the GPU uses — so GPU == oracle bit-for-bit. With
// g_detmath=false it calls std::exp/std::log exactly as the reference does;
// tests measure the (tiny) difference between the two modes.
//
// Compile with -O2 -ffp-contract=off and no -march (no FMA contraction).
// =============================================================================
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../paper_2511_04283_b200/csrc/detmath.h"

namespace oracle {

inline bool g_detmath = true;

template <typename T>
inline T ex(T x) {
  if constexpr (std::is_same_v<T, float>) {
    if (g_detmath) return sk::det_expf(x);
  }
  return std::exp(x);
}

template <typename T>
inline T lg(T x) {
  if constexpr (std::is_same_v<T, float>) {
    if (g_detmath) return sk::det_logf(x);
  }
  return std::log(x);
}

// ---------------------------------------------------------------------------
// Foundation (types.hpp). Small fixed-size vectors/matrices replacing Eigen.
// Matrix products are evaluated as sequential dot products over k:
//   (a0*b0 + a1*b1) + a2*b2
// ---------------------------------------------------------------------------
template <typename T, int N>
struct Vec {
  T v[N];
  T& operator[](int i) { return v[i]; }
  const T& operator[](int i) const { return v[i]; }
  static Vec zero() {
    Vec r;
    for (int i = 0; i < N; ++i) r.v[i] = T(0);
    return r;
  }
};
template <typename T> using Vec2 = Vec<T, 2>;
template <typename T> using Vec3 = Vec<T, 3>;
template <typename T> using Vec4 = Vec<T, 4>;

template <typename T, int N>
inline Vec<T, N> operator+(const Vec<T, N>& a, const Vec<T, N>& b) {
  Vec<T, N> r;
  for (int i = 0; i < N; ++i) r[i] = a[i] + b[i];
  return r;
}
template <typename T, int N>
inline Vec<T, N> operator-(const Vec<T, N>& a, const Vec<T, N>& b) {
  Vec<T, N> r;
  for (int i = 0; i < N; ++i) r[i] = a[i] - b[i];
  return r;
}
template <typename T, int N>
inline Vec<T, N> operator*(T s, const Vec<T, N>& a) {
  Vec<T, N> r;
  for (int i = 0; i < N; ++i) r[i] = s * a[i];
  return r;
}
template <typename T, int N>
inline Vec<T, N> operator/(const Vec<T, N>& a, T s) {
  Vec<T, N> r;
  for (int i = 0; i < N; ++i) r[i] = a[i] / s;
  return r;
}
template <typename T, int N>
inline Vec<T, N>& operator+=(Vec<T, N>& a, const Vec<T, N>& b) {
  for (int i = 0; i < N; ++i) a[i] = a[i] + b[i];
  return a;
}
template <typename T, int N>
inline Vec<T, N>& operator-=(Vec<T, N>& a, const Vec<T, N>& b) {
  for (int i = 0; i < N; ++i) a[i] = a[i] - b[i];
  return a;
}
template <typename T, int N>
inline T dot(const Vec<T, N>& a, const Vec<T, N>& b) {
  T s = a[0] * b[0];
  for (int i = 1; i < N; ++i) s = s + a[i] * b[i];
  return s;
}
template <typename T, int N>
inline T squared_norm(const Vec<T, N>& a) {
  return dot(a, a);
}
template <typename T, int N>
inline T norm(const Vec<T, N>& a) {
  return std::sqrt(squared_norm(a));
}
template <typename T, int N>
inline bool all_finite(const Vec<T, N>& a) {
  for (int i = 0; i < N; ++i)
    if (!std::isfinite(a[i])) return false;
  return true;
}

template <typename T, int R, int C>
struct Mat {
  T m[R][C];
  T& operator()(int r, int c) { return m[r][c]; }
  const T& operator()(int r, int c) const { return m[r][c]; }
  static Mat zero() {
    Mat o;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < C; ++c) o.m[r][c] = T(0);
    return o;
  }
  static Mat identity() {
    Mat o = zero();
    for (int i = 0; i < R && i < C; ++i) o.m[i][i] = T(1);
    return o;
  }
  Mat<T, C, R> transpose() const {
    Mat<T, C, R> o;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < C; ++c) o.m[c][r] = m[r][c];
    return o;
  }
};
template <typename T> using Mat2 = Mat<T, 2, 2>;
template <typename T> using Mat3 = Mat<T, 3, 3>;
template <typename T> using Mat4 = Mat<T, 4, 4>;
template <typename T> using Mat23 = Mat<T, 2, 3>;

template <typename T, int R, int K, int C>
inline Mat<T, R, C> operator*(const Mat<T, R, K>& a, const Mat<T, K, C>& b) {
  Mat<T, R, C> o;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) {
      T s = a.m[r][0] * b.m[0][c];
      for (int k = 1; k < K; ++k) s = s + a.m[r][k] * b.m[k][c];
      o.m[r][c] = s;
    }
  return o;
}
template <typename T, int R, int C>
inline Vec<T, R> operator*(const Mat<T, R, C>& a, const Vec<T, C>& x) {
  Vec<T, R> o;
  for (int r = 0; r < R; ++r) {
    T s = a.m[r][0] * x[0];
    for (int k = 1; k < C; ++k) s = s + a.m[r][k] * x[k];
    o[r] = s;
  }
  return o;
}
template <typename T, int R, int C>
inline Mat<T, R, C> operator+(const Mat<T, R, C>& a, const Mat<T, R, C>& b) {
  Mat<T, R, C> o;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) o.m[r][c] = a.m[r][c] + b.m[r][c];
  return o;
}
template <typename T, int R, int C>
inline Mat<T, R, C>& operator+=(Mat<T, R, C>& a, const Mat<T, R, C>& b) {
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) a.m[r][c] = a.m[r][c] + b.m[r][c];
  return a;
}
template <typename T, int R, int C>
inline Mat<T, R, C> operator*(T s, const Mat<T, R, C>& a) {
  Mat<T, R, C> o;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) o.m[r][c] = s * a.m[r][c];
  return o;
}
template <typename T, int R, int C>
inline Mat<T, R, C> operator-(const Mat<T, R, C>& a) {
  Mat<T, R, C> o;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) o.m[r][c] = -a.m[r][c];
  return o;
}

// types.hpp:28-35
template <typename T>
inline T sigmoid(T x) {
  return T(1) / (T(1) + ex(-x));
}
template <typename T>
inline T logit(T x) {
  return std::log(x / (T(1) - x));
}

// types.hpp:66-68
inline void require(bool cond, const std::string& msg) {
  if (!cond) throw std::runtime_error(msg);
}

// Image<T> (types.hpp:38-64): row-major interleaved RGB.
template <typename T>
struct Image {
  int width = 0, height = 0;
  std::vector<Vec3<T>> pixels;
  Image() = default;
  Image(int w, int h) : width(w), height(h), pixels(size_t(w) * h, Vec3<T>::zero()) {}
  Vec3<T>& at(int x, int y) { return pixels[size_t(y) * width + x]; }
  const Vec3<T>& at(int x, int y) const { return pixels[size_t(y) * width + x]; }
};

// Per-pixel scalar map (ScalarMap / MaskMap, types.hpp:24-25). Stored row-major
// here; the reference's Eigen arrays are column-major but are only ever
// addressed by (y, x), so the element values are the same.
template <typename T>
struct Map2D {
  int h = 0, w = 0;
  std::vector<T> d;
  Map2D() = default;
  Map2D(int h_, int w_, T fill = T(0)) : h(h_), w(w_), d(size_t(h_) * w_, fill) {}
  T& operator()(int y, int x) { return d[size_t(y) * w + x]; }
  const T& operator()(int y, int x) const { return d[size_t(y) * w + x]; }
};
using MaskMap = Map2D<std::uint8_t>;

// ---------------------------------------------------------------------------
// parallel.hpp:14-32
// ---------------------------------------------------------------------------
inline void parallel_chunks(int count, int workers, const std::function<void(int, int, int)>& fn) {
  if (count <= 0) return;
  if (workers <= 1 || count == 1) {
    fn(0, 0, count);
    return;
  }
  const int n = std::min(workers, count);
  std::vector<std::thread> threads;
  const int chunk = (count + n - 1) / n;
  for (int w = 0; w < n; ++w) {
    const int begin = w * chunk;
    const int end = std::min(count, begin + chunk);
    if (begin >= end) break;
    threads.emplace_back(fn, w, begin, end);
  }
  for (auto& t : threads) t.join();
}

// ---------------------------------------------------------------------------
// rng.hpp:18-69 — mt19937_64 is fully specified by the standard.
// ---------------------------------------------------------------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t next_u64() { return engine_(); }
  double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  std::uint64_t bounded(std::uint64_t n) {
    return static_cast<std::uint64_t>((static_cast<__uint128_t>(engine_()) * n) >> 64);
  }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    double u2 = uniform();
    u1 = std::max(u1, 0x1.0p-53);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * M_PI * u2;
    spare_ = r * std::sin(a);
    has_spare_ = true;
    return r * std::cos(a);
  }
  std::vector<int> sample_without_replacement(int n, int k) {
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    const int m = std::min(k, n);
    for (int i = 0; i < m; ++i) {
      const int j = i + static_cast<int>(bounded(static_cast<std::uint64_t>(n - i)));
      std::swap(idx[i], idx[j]);
    }
    idx.resize(m);
    return idx;
  }

 private:
  std::mt19937_64 engine_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ---------------------------------------------------------------------------
// sh.hpp:14-114
// ---------------------------------------------------------------------------
inline constexpr double kShC0 = 0.28209479177387814;
inline constexpr double kShC1 = 0.4886025119029199;
inline constexpr double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                    -1.0925484305920792, 0.5462742152960396};
inline constexpr double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                    0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                                    -0.5900435899266435};

inline constexpr int sh_coeff_count(int degree) { return (degree + 1) * (degree + 1); }

// ShMatrix<T> (types.hpp:22): n_sh rows x 3 columns.
template <typename T>
struct ShMatrix {
  int rows = 0;
  std::vector<T> d;  // row-major (k, c) -> 3k + c
  ShMatrix() = default;
  explicit ShMatrix(int r) : rows(r), d(size_t(r) * 3, T(0)) {}
  T& operator()(int k, int c) { return d[size_t(k) * 3 + c]; }
  const T& operator()(int k, int c) const { return d[size_t(k) * 3 + c]; }
};

template <typename T>
inline void sh_basis(const Vec3<T>& dir, int degree, T* basis) {
  const T x = dir[0], y = dir[1], z = dir[2];
  basis[0] = T(kShC0);
  if (degree < 1) return;
  basis[1] = T(-kShC1) * y;
  basis[2] = T(kShC1) * z;
  basis[3] = T(-kShC1) * x;
  if (degree < 2) return;
  const T xx = x * x, yy = y * y, zz = z * z;
  const T xy = x * y, yz = y * z, xz = x * z;
  basis[4] = T(kShC2[0]) * xy;
  basis[5] = T(kShC2[1]) * yz;
  basis[6] = T(kShC2[2]) * (T(2) * zz - xx - yy);
  basis[7] = T(kShC2[3]) * xz;
  basis[8] = T(kShC2[4]) * (xx - yy);
  if (degree < 3) return;
  basis[9] = T(kShC3[0]) * y * (T(3) * xx - yy);
  basis[10] = T(kShC3[1]) * xy * z;
  basis[11] = T(kShC3[2]) * y * (T(4) * zz - xx - yy);
  basis[12] = T(kShC3[3]) * z * (T(2) * zz - T(3) * xx - T(3) * yy);
  basis[13] = T(kShC3[4]) * x * (T(4) * zz - xx - yy);
  basis[14] = T(kShC3[5]) * z * (xx - yy);
  basis[15] = T(kShC3[6]) * x * (xx - T(3) * yy);
}

template <typename T>
inline Vec3<T> v3(T a, T b, T c) {
  Vec3<T> r;
  r[0] = a;
  r[1] = b;
  r[2] = c;
  return r;
}

template <typename T>
inline void sh_basis_jacobian(const Vec3<T>& dir, int degree, Vec3<T>* db) {
  const T x = dir[0], y = dir[1], z = dir[2];
  db[0] = Vec3<T>::zero();
  if (degree < 1) return;
  db[1] = v3(T(0), T(-kShC1), T(0));
  db[2] = v3(T(0), T(0), T(kShC1));
  db[3] = v3(T(-kShC1), T(0), T(0));
  if (degree < 2) return;
  db[4] = T(kShC2[0]) * v3(y, x, T(0));
  db[5] = T(kShC2[1]) * v3(T(0), z, y);
  db[6] = T(kShC2[2]) * v3(T(-2) * x, T(-2) * y, T(4) * z);
  db[7] = T(kShC2[3]) * v3(z, T(0), x);
  db[8] = T(kShC2[4]) * v3(T(2) * x, T(-2) * y, T(0));
  if (degree < 3) return;
  const T xx = x * x, yy = y * y, zz = z * z;
  db[9] = T(kShC3[0]) * v3(T(6) * x * y, T(3) * xx - T(3) * yy, T(0));
  db[10] = T(kShC3[1]) * v3(y * z, x * z, x * y);
  db[11] = T(kShC3[2]) * v3(T(-2) * x * y, T(4) * zz - xx - T(3) * yy, T(8) * y * z);
  db[12] = T(kShC3[3]) * v3(T(-6) * x * z, T(-6) * y * z, T(6) * zz - T(3) * xx - T(3) * yy);
  db[13] = T(kShC3[4]) * v3(T(4) * zz - T(3) * xx - yy, T(-2) * x * y, T(8) * x * z);
  db[14] = T(kShC3[5]) * v3(T(2) * x * z, T(-2) * y * z, xx - yy);
  db[15] = T(kShC3[6]) * v3(T(3) * xx - T(3) * yy, T(-6) * x * y, T(0));
}

// sh.hpp:80-88: rgb = sum_k basis_k sh.row(k), k ascending from a zero vector.
template <typename T>
inline Vec3<T> evaluate_sh(const ShMatrix<T>& sh, const Vec3<T>& dir, int degree) {
  const int n = sh_coeff_count(degree);
  T basis[16];
  sh_basis(dir, degree, basis);
  Vec3<T> rgb = Vec3<T>::zero();
  for (int k = 0; k < n; ++k)
    for (int c = 0; c < 3; ++c) rgb[c] = rgb[c] + basis[k] * sh(k, c);
  for (int c = 0; c < 3; ++c) {
    rgb[c] = rgb[c] + T(0.5);
    rgb[c] = (rgb[c] < T(0)) ? T(0) : rgb[c];
  }
  return rgb;
}

template <typename T>
inline void evaluate_sh_backward(const ShMatrix<T>& sh, const Vec3<T>& dir, int degree,
                                 const Vec3<T>& d_color, ShMatrix<T>& d_sh, Vec3<T>& d_dir) {
  const int n = sh_coeff_count(degree);
  T basis[16];
  Vec3<T> db[16];
  sh_basis(dir, degree, basis);
  sh_basis_jacobian(dir, degree, db);
  Vec3<T> raw = Vec3<T>::zero();
  for (int k = 0; k < n; ++k)
    for (int c = 0; c < 3; ++c) raw[c] = raw[c] + basis[k] * sh(k, c);
  for (int c = 0; c < 3; ++c) raw[c] = raw[c] + T(0.5);
  Vec3<T> d_raw = d_color;
  for (int c = 0; c < 3; ++c)
    if (raw[c] < T(0)) d_raw[c] = T(0);
  d_sh = ShMatrix<T>(sh.rows);
  d_dir = Vec3<T>::zero();
  for (int k = 0; k < n; ++k) {
    for (int c = 0; c < 3; ++c) d_sh(k, c) = basis[k] * d_raw[c];
    const T s = (sh(k, 0) * d_raw[0] + sh(k, 1) * d_raw[1]) + sh(k, 2) * d_raw[2];
    d_dir += s * db[k];
  }
}

// ---------------------------------------------------------------------------
// scene.hpp:18-154
// ---------------------------------------------------------------------------
template <typename T>
struct Gaussian3D {
  Vec3<T> mu = Vec3<T>::zero();
  Vec4<T> rot = [] {
    Vec4<T> q;
    q[0] = T(1);
    q[1] = q[2] = q[3] = T(0);
    return q;
  }();
  Vec3<T> log_scale = Vec3<T>::zero();
  T opacity_logit = T(0);
  ShMatrix<T> sh;
  Vec3<T> scale() const {
    Vec3<T> s;
    for (int i = 0; i < 3; ++i) s[i] = ex(log_scale[i]);
    return s;
  }
  T opacity() const { return sigmoid(opacity_logit); }
};

template <typename T>
struct Scene {
  std::vector<Gaussian3D<T>> gaussians;
  int sh_degree = 3;
  int size() const { return static_cast<int>(gaussians.size()); }
};

// scene.hpp:57-65; normalisation q / sqrt(((w^2 + x^2) + y^2) + z^2).
template <typename T>
inline Mat3<T> quat_to_rotation(const Vec4<T>& q_in) {
  const T n2 = squared_norm(q_in);
  Vec4<T> q = q_in;
  if (n2 > T(0)) q = q_in / std::sqrt(n2);
  const T w = q[0], x = q[1], y = q[2], z = q[3];
  Mat3<T> r;
  r(0, 0) = T(1) - T(2) * (y * y + z * z);
  r(0, 1) = T(2) * (x * y - w * z);
  r(0, 2) = T(2) * (x * z + w * y);
  r(1, 0) = T(2) * (x * y + w * z);
  r(1, 1) = T(1) - T(2) * (x * x + z * z);
  r(1, 2) = T(2) * (y * z - w * x);
  r(2, 0) = T(2) * (x * z - w * y);
  r(2, 1) = T(2) * (y * z + w * x);
  r(2, 2) = T(1) - T(2) * (x * x + y * y);
  return r;
}

template <typename T>
inline T mat_inner(const Mat3<T>& a, const Mat3<T>& b) {
  T s = T(0);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) s = s + a(r, c) * b(r, c);
  return s;
}

// scene.hpp:70-84
template <typename T>
inline Vec4<T> quat_rotation_backward(const Vec4<T>& q_in, const Mat3<T>& d_r) {
  const T nrm = norm(q_in);
  const Vec4<T> q = q_in / nrm;
  const T w = q[0], x = q[1], y = q[2], z = q[3];
  auto mk = [](T a, T b, T c, T d, T e, T f, T g, T h, T i) {
    Mat3<T> m;
    m(0, 0) = a; m(0, 1) = b; m(0, 2) = c;
    m(1, 0) = d; m(1, 1) = e; m(1, 2) = f;
    m(2, 0) = g; m(2, 1) = h; m(2, 2) = i;
    return m;
  };
  const Mat3<T> dw = mk(T(0), T(-2) * z, T(2) * y, T(2) * z, T(0), T(-2) * x, T(-2) * y, T(2) * x, T(0));
  const Mat3<T> dx = mk(T(0), T(2) * y, T(2) * z, T(2) * y, T(-4) * x, T(-2) * w, T(2) * z, T(2) * w, T(-4) * x);
  const Mat3<T> dy = mk(T(-4) * y, T(2) * x, T(2) * w, T(2) * x, T(0), T(2) * z, T(-2) * w, T(2) * z, T(-4) * y);
  const Mat3<T> dz = mk(T(-4) * z, T(-2) * w, T(2) * x, T(2) * w, T(-4) * z, T(2) * y, T(2) * x, T(2) * y, T(0));
  Vec4<T> du;
  du[0] = mat_inner(d_r, dw);
  du[1] = mat_inner(d_r, dx);
  du[2] = mat_inner(d_r, dy);
  du[3] = mat_inner(d_r, dz);
  const T qd = dot(q, du);
  Vec4<T> o;
  for (int i = 0; i < 4; ++i) o[i] = (du[i] - q[i] * qd) / nrm;
  return o;
}

// scene.hpp:88-96. Sigma = M M^T, M = R diag(s).
template <typename T>
inline Mat3<T> covariance_3d(const Vec4<T>& rot, const Vec3<T>& scale) {
  if (!all_finite(rot) || !all_finite(scale))
    throw std::invalid_argument("covariance_3d: non-finite rotation or scale");
  for (int i = 0; i < 3; ++i)
    if (scale[i] <= T(0)) throw std::invalid_argument("covariance_3d: scale must be positive");
  const Mat3<T> r = quat_to_rotation(rot);
  Mat3<T> m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m(i, j) = r(i, j) * scale[j];
  return m * m.transpose();
}

// scene.hpp:101-110
template <typename T>
inline void covariance_3d_backward(const Vec4<T>& rot, const Vec3<T>& scale, const Mat3<T>& d_sigma,
                                   Vec4<T>& d_rot, Vec3<T>& d_scale) {
  const Mat3<T> r = quat_to_rotation(rot);
  Mat3<T> m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m(i, j) = r(i, j) * scale[j];
  const Mat3<T> d_m = (d_sigma + d_sigma.transpose()) * m;
  Mat3<T> d_r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) d_r(i, j) = d_m(i, j) * scale[j];
  for (int j = 0; j < 3; ++j) d_scale[j] = (d_m(0, j) * r(0, j) + d_m(1, j) * r(1, j)) + d_m(2, j) * r(2, j);
  d_rot = quat_rotation_backward(rot, d_r);
}

// scene.hpp:117-154
template <typename T>
inline Scene<T> init_from_points(const std::vector<std::pair<Vec3<T>, Vec3<T>>>& points, int sh_degree) {
  if (points.empty()) throw std::invalid_argument("init_from_points: empty point cloud");
  const int n = static_cast<int>(points.size());
  Scene<T> scene;
  scene.sh_degree = sh_degree;
  scene.gaussians.reserve(n);
  for (int i = 0; i < n; ++i) {
    T d0 = std::numeric_limits<T>::max(), d1 = d0, d2 = d0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const T d = norm(points[j].first - points[i].first);
      if (d < d0) {
        d2 = d1; d1 = d0; d0 = d;
      } else if (d < d1) {
        d2 = d1; d1 = d;
      } else if (d < d2) {
        d2 = d;
      }
    }
    T mean = T(1);
    if (n == 2) mean = d0;
    else if (n == 3) mean = (d0 + d1) / T(2);
    else if (n > 3) mean = (d0 + d1 + d2) / T(3);
    mean = std::max(mean, T(1e-7));
    Gaussian3D<T> g;
    g.mu = points[i].first;
    const T ls = std::log(mean);
    g.log_scale = v3(ls, ls, ls);
    g.opacity_logit = logit(T(0.1));
    g.sh = ShMatrix<T>(sh_coeff_count(sh_degree));
    for (int c = 0; c < 3; ++c) g.sh(0, c) = (points[i].second[c] - T(0.5)) / T(kShC0);
    scene.gaussians.push_back(std::move(g));
  }
  return scene;
}

// ---------------------------------------------------------------------------
// camera.hpp:14-213
// ---------------------------------------------------------------------------
inline constexpr double kCov2dFloor = 0.3;
inline constexpr double kCullGuard = 1.3;

template <typename T>
struct Camera {
  int width = 0, height = 0;
  T fx = T(0), fy = T(0), cx = T(0), cy = T(0);
  Mat4<T> world_to_cam = Mat4<T>::identity();
  T near = T(0.2);
  Mat3<T> rotation() const {
    Mat3<T> r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r(i, j) = world_to_cam(i, j);
    return r;
  }
  Vec3<T> translation() const { return v3(world_to_cam(0, 3), world_to_cam(1, 3), world_to_cam(2, 3)); }
  // center = -(R^T t), evaluated (R_0i t0 + R_1i t1) + R_2i t2.
  Vec3<T> center() const {
    const Vec3<T> c = rotation().transpose() * translation();
    return v3(-c[0], -c[1], -c[2]);
  }
};

template <typename T>
struct ProjectedGaussian {
  Vec2<T> mu2d = Vec2<T>::zero();
  Mat2<T> cov2d = Mat2<T>::zero();
  Mat2<T> cov2d_inv = Mat2<T>::zero();
  T depth = T(0);
  Vec3<T> color = Vec3<T>::zero();
  T opacity = T(0);
  int source_index = -1;
};

template <typename T>
inline T max_eigenvalue_2x2(const Mat2<T>& m) {
  const T mid = (m(0, 0) + m(1, 1)) / T(2);
  const T h = (m(0, 0) - m(1, 1)) / T(2);
  return mid + std::sqrt(h * h + m(0, 1) * m(0, 1));
}

template <typename T>
inline Mat23<T> projection_jacobian(const Camera<T>& cam, const Vec3<T>& t) {
  const T iz = T(1) / t[2];
  const T iz2 = iz * iz;
  Mat23<T> j;
  j(0, 0) = cam.fx * iz;
  j(0, 1) = T(0);
  j(0, 2) = -cam.fx * t[0] * iz2;
  j(1, 0) = T(0);
  j(1, 1) = cam.fy * iz;
  j(1, 2) = -cam.fy * t[1] * iz2;
  return j;
}

template <typename T>
inline std::optional<ProjectedGaussian<T>> project(const Gaussian3D<T>& g, const Camera<T>& cam, int sh_degree,
                                                   int source_index = -1) {
  const Mat3<T> w_rot = cam.rotation();
  const Vec3<T> t = w_rot * g.mu + cam.translation();
  if (t[2] <= cam.near) return std::nullopt;
  const Mat23<T> j = projection_jacobian(cam, t);
  const Mat23<T> m = j * w_rot;
  const Mat3<T> sigma3 = covariance_3d(g.rot, g.scale());
  Mat2<T> cov2d = (m * sigma3) * m.transpose();
  cov2d(0, 0) = cov2d(0, 0) + T(kCov2dFloor);
  cov2d(1, 1) = cov2d(1, 1) + T(kCov2dFloor);

  ProjectedGaussian<T> pg;
  pg.mu2d[0] = cam.fx * t[0] / t[2] + cam.cx;
  pg.mu2d[1] = cam.fy * t[1] / t[2] + cam.cy;
  const T radius = T(3) * std::sqrt(max_eigenvalue_2x2(cov2d));
  const T guard = T(kCullGuard) * radius;
  if (pg.mu2d[0] < -guard || pg.mu2d[0] > T(cam.width - 1) + guard || pg.mu2d[1] < -guard ||
      pg.mu2d[1] > T(cam.height - 1) + guard)
    return std::nullopt;
  const T det = cov2d(0, 0) * cov2d(1, 1) - cov2d(0, 1) * cov2d(1, 0);
  pg.cov2d = cov2d;
  pg.cov2d_inv(0, 0) = cov2d(1, 1) / det;
  pg.cov2d_inv(0, 1) = -cov2d(0, 1) / det;
  pg.cov2d_inv(1, 0) = -cov2d(1, 0) / det;
  pg.cov2d_inv(1, 1) = cov2d(0, 0) / det;
  pg.depth = t[2];
  const Vec3<T> rel = g.mu - cam.center();
  pg.color = evaluate_sh(g.sh, rel / norm(rel), sh_degree);
  pg.opacity = sigmoid(g.opacity_logit);
  pg.source_index = source_index;
  return pg;
}

template <typename T>
struct GaussianGrads {
  Vec3<T> mu = Vec3<T>::zero();
  Vec4<T> rot = Vec4<T>::zero();
  Vec3<T> log_scale = Vec3<T>::zero();
  T opacity_logit = T(0);
  ShMatrix<T> sh;
};

template <typename T>
inline std::vector<ProjectedGaussian<T>> project_scene(const Scene<T>& scene, const Camera<T>& cam) {
  std::vector<ProjectedGaussian<T>> pgs;
  pgs.reserve(scene.gaussians.size());
  for (int i = 0; i < scene.size(); ++i)
    if (auto pg = project(scene.gaussians[i], cam, scene.sh_degree, i)) pgs.push_back(*pg);
  return pgs;
}

template <typename T>
inline Mat2<T> cov_grad_from_inv_grad(const Mat2<T>& cov2d_inv, const Mat2<T>& d_inv) {
  return -((cov2d_inv * d_inv) * cov2d_inv);
}

// camera.hpp:156-213
template <typename T>
inline GaussianGrads<T> project_backward(const Gaussian3D<T>& g, const Camera<T>& cam, int sh_degree,
                                         const Vec2<T>& d_mu2d, const Mat2<T>& d_cov2d, const Vec3<T>& d_color,
                                         T d_opacity) {
  GaussianGrads<T> out;
  out.sh = ShMatrix<T>(g.sh.rows);
  const Mat3<T> w_rot = cam.rotation();
  const Vec3<T> t = w_rot * g.mu + cam.translation();
  const Mat23<T> j = projection_jacobian(cam, t);
  const Mat23<T> m = j * w_rot;
  const Vec3<T> scale = g.scale();
  const Mat3<T> sigma3 = covariance_3d(g.rot, scale);

  const T sig = sigmoid(g.opacity_logit);
  out.opacity_logit = d_opacity * sig * (T(1) - sig);
  {
    const Vec3<T> rel = g.mu - cam.center();
    const T dist = norm(rel);
    const Vec3<T> dir = rel / dist;
    Vec3<T> d_dir;
    evaluate_sh_backward(g.sh, dir, sh_degree, d_color, out.sh, d_dir);
    const T dd = dot(dir, d_dir);
    for (int i = 0; i < 3; ++i) out.mu[i] = out.mu[i] + (d_dir[i] - dir[i] * dd) / dist;
  }
  const Mat23<T> d_m = ((d_cov2d + d_cov2d.transpose()) * m) * sigma3;
  const Mat3<T> d_sigma3 = (m.transpose() * d_cov2d) * m;
  {
    Vec4<T> d_rot;
    Vec3<T> d_scale;
    covariance_3d_backward(g.rot, scale, d_sigma3, d_rot, d_scale);
    out.rot += d_rot;
    for (int i = 0; i < 3; ++i) out.log_scale[i] = out.log_scale[i] + d_scale[i] * scale[i];
  }
  Vec3<T> d_t = Vec3<T>::zero();
  {
    const Mat23<T> d_j = d_m * w_rot.transpose();
    const T iz = T(1) / t[2];
    const T iz2 = iz * iz;
    const T iz3 = iz2 * iz;
    d_t[0] = d_t[0] + d_j(0, 2) * (-cam.fx * iz2);
    d_t[1] = d_t[1] + d_j(1, 2) * (-cam.fy * iz2);
    d_t[2] = d_t[2] + (((d_j(0, 0) * (-cam.fx * iz2) + d_j(0, 2) * (T(2) * cam.fx * t[0] * iz3)) +
                        d_j(1, 1) * (-cam.fy * iz2)) +
                       d_j(1, 2) * (T(2) * cam.fy * t[1] * iz3));
  }
  d_t += j.transpose() * d_mu2d;
  out.mu += w_rot.transpose() * d_t;
  return out;
}

// ---------------------------------------------------------------------------
// raster.hpp:19-355
// ---------------------------------------------------------------------------
inline constexpr double kAlphaCap = 0.99;
inline constexpr double kAlphaMin = 1.0 / 255;
inline constexpr double kTransmitMin = 1e-4;
inline constexpr double kBinSigma = 3.0;
inline constexpr double kBinMahaMax = kBinSigma * kBinSigma;

struct TileGrid {
  int width = 0, height = 0, tile_size = 16, tiles_x = 0, tiles_y = 0;
  std::vector<std::vector<int>> tiles;
  int tile_count() const { return tiles_x * tiles_y; }
};

enum class BinMode { kAabb, kCompact };

template <typename T>
struct BinningConfig {
  BinMode mode = BinMode::kAabb;
  T beta = T(1);
  T tau_alpha = T(1.0 / 255);
};

inline TileGrid make_tile_grid(int width, int height, int tile_size = 16) {
  TileGrid grid;
  grid.width = width;
  grid.height = height;
  grid.tile_size = tile_size;
  grid.tiles_x = (width + tile_size - 1) / tile_size;
  grid.tiles_y = (height + tile_size - 1) / tile_size;
  grid.tiles.assign(size_t(grid.tile_count()), {});
  return grid;
}

// static_cast<int>(std::floor(v)) in the reference is undefined for |v| >=
// 2^31 (huge footprints); both the oracle and the GPU saturate at +-2^30.
template <typename T>
inline int floor_to_int(T v) {
  T f = std::floor(v);
  if (!(f > T(-1073741824))) f = T(-1073741824);
  if (f > T(1073741824)) f = T(1073741824);
  return static_cast<int>(f);
}

template <typename T>
inline std::vector<int> bin_aabb(const ProjectedGaussian<T>& pg, const TileGrid& grid) {
  const T r = T(kBinSigma) * std::sqrt(max_eigenvalue_2x2(pg.cov2d));
  const int ts = grid.tile_size;
  const int tx0 = floor_to_int((pg.mu2d[0] - r) / T(ts));
  const int tx1 = floor_to_int((pg.mu2d[0] + r) / T(ts));
  const int ty0 = floor_to_int((pg.mu2d[1] - r) / T(ts));
  const int ty1 = floor_to_int((pg.mu2d[1] + r) / T(ts));
  std::vector<int> out;
  if (tx1 < 0 || ty1 < 0 || tx0 >= grid.tiles_x || ty0 >= grid.tiles_y) return out;
  for (int ty = std::max(ty0, 0); ty <= std::min(ty1, grid.tiles_y - 1); ++ty)
    for (int tx = std::max(tx0, 0); tx <= std::min(tx1, grid.tiles_x - 1); ++tx) out.push_back(ty * grid.tiles_x + tx);
  return out;
}

template <typename T>
inline T compact_threshold(T sigma, T tau_alpha, T beta) {
  return beta * (T(2) * lg(sigma / tau_alpha));
}

template <typename T>
inline T clamp_ref(T v, T lo, T hi) {  // std::clamp
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}
template <typename T>
inline T min_ref(T a, T b) {  // std::min(a, b)
  return (b < a) ? b : a;
}

template <typename T>
inline T min_mahalanobis_on_rect(const Mat2<T>& conic, const Vec2<T>& mu, T x0, T x1, T y0, T y1) {
  if (mu[0] >= x0 && mu[0] <= x1 && mu[1] >= y0 && mu[1] <= y1) return T(0);
  const T a = conic(0, 0), b = conic(0, 1), c = conic(1, 1);
  const auto q = [&](T dx, T dy) { return a * dx * dx + T(2) * b * dx * dy + c * dy * dy; };
  T best = std::numeric_limits<T>::max();
  for (const T x : {x0, x1}) {
    const T dx = x - mu[0];
    const T y = clamp_ref(mu[1] - b * dx / c, y0, y1);
    best = min_ref(best, q(dx, y - mu[1]));
  }
  for (const T y : {y0, y1}) {
    const T dy = y - mu[1];
    const T x = clamp_ref(mu[0] - b * dy / a, x0, x1);
    best = min_ref(best, q(x - mu[0], dy));
  }
  return best;
}

template <typename T>
inline std::vector<int> bin_compact(const ProjectedGaussian<T>& pg, const TileGrid& grid, T beta, T tau_alpha) {
  std::vector<int> out;
  if (pg.opacity <= tau_alpha) return out;
  const T det = pg.cov2d(0, 0) * pg.cov2d(1, 1) - pg.cov2d(1, 0) * pg.cov2d(0, 1);
  require(det > T(0) && pg.cov2d(0, 0) > T(0), "bin_compact: cov2d must be positive definite");
  const T a_star = min_ref(compact_threshold(pg.opacity, tau_alpha, beta), T(kBinMahaMax));
  const T ext_x = std::sqrt(a_star * pg.cov2d(0, 0));
  const T ext_y = std::sqrt(a_star * pg.cov2d(1, 1));
  const int ts = grid.tile_size;
  const int tx0 = std::max(0, floor_to_int((pg.mu2d[0] - ext_x) / T(ts)));
  const int tx1 = std::min(grid.tiles_x - 1, floor_to_int((pg.mu2d[0] + ext_x) / T(ts)));
  const int ty0 = std::max(0, floor_to_int((pg.mu2d[1] - ext_y) / T(ts)));
  const int ty1 = std::min(grid.tiles_y - 1, floor_to_int((pg.mu2d[1] + ext_y) / T(ts)));
  for (int ty = ty0; ty <= ty1; ++ty) {
    const T y0 = T(ty * ts);
    const T y1 = T(std::min((ty + 1) * ts, grid.height) - 1);
    for (int tx = tx0; tx <= tx1; ++tx) {
      const T x0 = T(tx * ts);
      const T x1 = T(std::min((tx + 1) * ts, grid.width) - 1);
      if (min_mahalanobis_on_rect(pg.cov2d_inv, pg.mu2d, x0, x1, y0, y1) <= a_star)
        out.push_back(ty * grid.tiles_x + tx);
    }
  }
  return out;
}

template <typename T>
inline std::vector<int> depth_order(const std::vector<ProjectedGaussian<T>>& pgs) {
  std::vector<int> order(pgs.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (pgs[a].depth != pgs[b].depth) return pgs[a].depth < pgs[b].depth;
    return a < b;
  });
  return order;
}

template <typename T>
inline std::vector<int> bin_one(const ProjectedGaussian<T>& pg, const TileGrid& grid, const BinningConfig<T>& b) {
  return b.mode == BinMode::kAabb ? bin_aabb(pg, grid) : bin_compact(pg, grid, b.beta, b.tau_alpha);
}

template <typename T>
inline TileGrid build_tile_grid(const std::vector<ProjectedGaussian<T>>& pgs, int width, int height,
                                const BinningConfig<T>& binning, int tile_size = 16) {
  TileGrid grid = make_tile_grid(width, height, tile_size);
  for (const int idx : depth_order(pgs))
    for (const int t : bin_one(pgs[idx], grid, binning)) grid.tiles[t].push_back(idx);
  return grid;
}

inline std::int64_t count_pairs(const TileGrid& grid) {
  std::int64_t total = 0;
  for (const auto& t : grid.tiles) total += static_cast<std::int64_t>(t.size());
  return total;
}

template <typename T>
struct RenderOutputs {
  Image<T> image;
  Map2D<T> transmittance;
  Map2D<int> contrib_count;
  // Workload counter (not in the reference; SURVEY 8(d) roofline units):
  // list entries the per-pixel loop examined, the terminating one included.
  std::int64_t pge_visited = 0;
};

struct FootprintCounter {
  std::vector<int> counts;
  explicit FootprintCounter(int n = 0) : counts(n, 0) {}
};

// raster.hpp:194-248. Per-pixel expression order is the reference's:
//   q = ((c00 dx) dx + ((2 c01) dx) dy) + (c11 dy) dy
//   C += (T alpha) color;  T *= 1 - alpha
template <typename T>
inline RenderOutputs<T> blend_forward(const TileGrid& grid, const std::vector<ProjectedGaussian<T>>& pgs,
                                      const MaskMap* mask = nullptr, FootprintCounter* counter = nullptr,
                                      int workers = 1) {
  RenderOutputs<T> out;
  out.image = Image<T>(grid.width, grid.height);
  out.transmittance = Map2D<T>(grid.height, grid.width, T(1));
  out.contrib_count = Map2D<int>(grid.height, grid.width, 0);
  const int n_workers = std::max(1, workers);
  std::vector<std::vector<int>> worker_counts;
  if (counter) worker_counts.assign(n_workers, std::vector<int>(counter->counts.size(), 0));
  std::vector<std::int64_t> worker_visited(n_workers, 0);
  parallel_chunks(grid.tile_count(), n_workers, [&](int worker, int begin, int end) {
    std::vector<int>* local = counter ? &worker_counts[worker] : nullptr;
    std::int64_t visited = 0;
    for (int tile = begin; tile < end; ++tile) {
      const auto& list = grid.tiles[tile];
      const int tx = tile % grid.tiles_x;
      const int ty = tile / grid.tiles_x;
      const int px1 = std::min((tx + 1) * grid.tile_size, grid.width);
      const int py1 = std::min((ty + 1) * grid.tile_size, grid.height);
      for (int py = ty * grid.tile_size; py < py1; ++py)
        for (int px = tx * grid.tile_size; px < px1; ++px) {
          T trans = T(1);
          Vec3<T> c = Vec3<T>::zero();
          int n = 0;
          const bool masked = mask && (*mask)(py, px) != 0;
          for (const int idx : list) {
            ++visited;
            const ProjectedGaussian<T>& pg = pgs[idx];
            const T dx = T(px) - pg.mu2d[0];
            const T dy = T(py) - pg.mu2d[1];
            const T q = pg.cov2d_inv(0, 0) * dx * dx + T(2) * pg.cov2d_inv(0, 1) * dx * dy +
                        pg.cov2d_inv(1, 1) * dy * dy;
            if (q < T(0)) continue;
            const T alpha = min_ref(T(kAlphaCap), pg.opacity * ex(T(-0.5) * q));
            if (alpha < T(kAlphaMin)) continue;
            const T w = trans * alpha;
            for (int ch = 0; ch < 3; ++ch) c[ch] = c[ch] + w * pg.color[ch];
            ++n;
            if (masked && local) ++(*local)[pg.source_index];
            trans = trans * (T(1) - alpha);
            if (trans < T(kTransmitMin)) break;
          }
          out.image.at(px, py) = c;
          out.transmittance(py, px) = trans;
          out.contrib_count(py, px) = n;
        }
    }
    worker_visited[worker] += visited;
  });
  for (const std::int64_t v : worker_visited) out.pge_visited += v;
  if (counter)
    for (const auto& wc : worker_counts)
      for (size_t i = 0; i < wc.size(); ++i) counter->counts[i] += wc[i];
  return out;
}

template <typename T>
struct BlendGrads {
  std::vector<Vec2<T>> d_mu2d;
  std::vector<Mat2<T>> d_conic;
  std::vector<Vec3<T>> d_color;
  std::vector<T> d_opacity;
  std::vector<Vec2<T>> abs_grad;
  explicit BlendGrads(size_t n = 0)
      : d_mu2d(n, Vec2<T>::zero()), d_conic(n, Mat2<T>::zero()), d_color(n, Vec3<T>::zero()),
        d_opacity(n, T(0)), abs_grad(n, Vec2<T>::zero()) {}
  void add(const BlendGrads& o) {
    for (size_t i = 0; i < d_mu2d.size(); ++i) {
      d_mu2d[i] += o.d_mu2d[i];
      d_conic[i] += o.d_conic[i];
      d_color[i] += o.d_color[i];
      d_opacity[i] = d_opacity[i] + o.d_opacity[i];
      abs_grad[i] += o.abs_grad[i];
    }
  }
};

// raster.hpp:281-355
template <typename T>
inline BlendGrads<T> blend_backward(const TileGrid& grid, const std::vector<ProjectedGaussian<T>>& pgs,
                                    const Image<T>& d_image, int workers = 1) {
  const int n_workers = std::max(1, workers);
  std::vector<BlendGrads<T>> worker_grads(n_workers, BlendGrads<T>(pgs.size()));
  struct Entry {
    int idx;
    T alpha, dx, dy, q, t_before;
    bool capped;
  };
  parallel_chunks(grid.tile_count(), n_workers, [&](int worker, int begin, int end) {
    BlendGrads<T>& acc = worker_grads[worker];
    std::vector<Entry> entries;
    for (int tile = begin; tile < end; ++tile) {
      const auto& list = grid.tiles[tile];
      if (list.empty()) continue;
      const int tx = tile % grid.tiles_x;
      const int ty = tile / grid.tiles_x;
      const int px1 = std::min((tx + 1) * grid.tile_size, grid.width);
      const int py1 = std::min((ty + 1) * grid.tile_size, grid.height);
      for (int py = ty * grid.tile_size; py < py1; ++py)
        for (int px = tx * grid.tile_size; px < px1; ++px) {
          entries.clear();
          T trans = T(1);
          for (const int idx : list) {
            const ProjectedGaussian<T>& pg = pgs[idx];
            const T dx = T(px) - pg.mu2d[0];
            const T dy = T(py) - pg.mu2d[1];
            const T q = pg.cov2d_inv(0, 0) * dx * dx + T(2) * pg.cov2d_inv(0, 1) * dx * dy +
                        pg.cov2d_inv(1, 1) * dy * dy;
            if (q < T(0)) continue;
            const T raw = pg.opacity * ex(T(-0.5) * q);
            const bool capped = raw > T(kAlphaCap);
            const T alpha = capped ? T(kAlphaCap) : raw;
            if (alpha < T(kAlphaMin)) continue;
            entries.push_back({idx, alpha, dx, dy, q, trans, capped});
            trans = trans * (T(1) - alpha);
            if (trans < T(kTransmitMin)) break;
          }
          if (entries.empty()) continue;
          const Vec3<T> dc = d_image.at(px, py);
          T suffix = T(0);
          for (auto it = entries.rbegin(); it != entries.rend(); ++it) {
            const ProjectedGaussian<T>& pg = pgs[it->idx];
            const T w = dot(pg.color, dc);
            const T d_alpha = it->t_before * w - suffix / (T(1) - it->alpha);
            suffix = suffix + it->t_before * it->alpha * w;
            const T ta = it->t_before * it->alpha;
            for (int ch = 0; ch < 3; ++ch) acc.d_color[it->idx][ch] = acc.d_color[it->idx][ch] + ta * dc[ch];
            if (it->capped) continue;
            const T g = ex(T(-0.5) * it->q);
            acc.d_opacity[it->idx] = acc.d_opacity[it->idx] + g * d_alpha;
            const T d_q = T(-0.5) * it->alpha * d_alpha;
            const T dx = it->dx, dy = it->dy;
            Mat2<T> outer;
            outer(0, 0) = dx * dx;
            outer(0, 1) = dx * dy;
            outer(1, 0) = dx * dy;
            outer(1, 1) = dy * dy;
            acc.d_conic[it->idx] += d_q * outer;
            Vec2<T> d_vec;
            d_vec[0] = pg.cov2d_inv(0, 0) * dx + pg.cov2d_inv(0, 1) * dy;
            d_vec[1] = pg.cov2d_inv(1, 0) * dx + pg.cov2d_inv(1, 1) * dy;
            const Vec2<T> d_mu = (T(-2) * d_q) * d_vec;
            acc.d_mu2d[it->idx] += d_mu;
            acc.abs_grad[it->idx][0] = acc.abs_grad[it->idx][0] + std::abs(d_mu[0]);
            acc.abs_grad[it->idx][1] = acc.abs_grad[it->idx][1] + std::abs(d_mu[1]);
          }
        }
    }
  });
  BlendGrads<T> total(pgs.size());
  for (const auto& wg : worker_grads) total.add(wg);
  return total;
}

// ---------------------------------------------------------------------------
// metrics.hpp:11-134
// ---------------------------------------------------------------------------
inline constexpr int kSsimWindow = 11;
inline constexpr double kSsimSigma = 1.5;
inline constexpr double kSsimC1 = 0.01 * 0.01;
inline constexpr double kSsimC2 = 0.03 * 0.03;

template <typename T>
inline std::array<T, kSsimWindow> ssim_kernel() {
  std::array<T, kSsimWindow> k;
  const int half = kSsimWindow / 2;
  T sum = T(0);
  for (int i = 0; i < kSsimWindow; ++i) {
    const T d = T(i - half);
    k[i] = std::exp(-(d * d) / (T(2) * T(kSsimSigma) * T(kSsimSigma)));
    sum = sum + k[i];
  }
  for (int i = 0; i < kSsimWindow; ++i) k[i] = k[i] / sum;
  return k;
}

template <typename T>
using ScalarMap = Map2D<T>;

// Separable blur with zero padding; not renormalised at borders (:30-52).
template <typename T>
inline ScalarMap<T> gauss_filter(const ScalarMap<T>& in) {
  static const std::array<T, kSsimWindow> k = ssim_kernel<T>();
  const int h = in.h, w = in.w;
  const int half = kSsimWindow / 2;
  ScalarMap<T> tmp(h, w);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      T s = T(0);
      const int o0 = std::max(-half, -x), o1 = std::min(half, w - 1 - x);
      for (int o = o0; o <= o1; ++o) s = s + k[o + half] * in(y, x + o);
      tmp(y, x) = s;
    }
  ScalarMap<T> out(h, w);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      T s = T(0);
      const int o0 = std::max(-half, -y), o1 = std::min(half, h - 1 - y);
      for (int o = o0; o <= o1; ++o) s = s + k[o + half] * tmp(y + o, x);
      out(y, x) = s;
    }
  return out;
}

template <typename T>
inline ScalarMap<T> channel(const Image<T>& img, int c) {
  ScalarMap<T> out(img.height, img.width);
  for (int y = 0; y < img.height; ++y)
    for (int x = 0; x < img.width; ++x) out(y, x) = img.at(x, y)[c];
  return out;
}

template <typename T, typename F>
inline ScalarMap<T> pointwise(const ScalarMap<T>& a, F f) {
  ScalarMap<T> o(a.h, a.w);
  for (size_t i = 0; i < a.d.size(); ++i) o.d[i] = f(i);
  return o;
}

template <typename T>
inline T map_mean(const ScalarMap<T>& m) {
  T s = T(0);
  for (const T v : m.d) s = s + v;
  return s / T(m.d.size());
}

template <typename T>
struct SsimChannelMaps {
  ScalarMap<T> mu_x, mu_y, mxx, myy, mxy, s;
};

template <typename T>
inline SsimChannelMaps<T> ssim_channel(const ScalarMap<T>& x, const ScalarMap<T>& y) {
  SsimChannelMaps<T> m;
  m.mu_x = gauss_filter(x);
  m.mu_y = gauss_filter(y);
  m.mxx = gauss_filter(pointwise(x, [&](size_t i) { return x.d[i] * x.d[i]; }));
  m.myy = gauss_filter(pointwise(y, [&](size_t i) { return y.d[i] * y.d[i]; }));
  m.mxy = gauss_filter(pointwise(x, [&](size_t i) { return x.d[i] * y.d[i]; }));
  m.s = pointwise(x, [&](size_t i) {
    const T mx = m.mu_x.d[i], my = m.mu_y.d[i];
    const T sxx = m.mxx.d[i] - mx * mx;
    const T syy = m.myy.d[i] - my * my;
    const T sxy = m.mxy.d[i] - mx * my;
    const T a1 = T(2) * mx * my + T(kSsimC1);
    const T a2 = T(2) * sxy + T(kSsimC2);
    const T b1 = mx * mx + my * my + T(kSsimC1);
    const T b2 = sxx + syy + T(kSsimC2);
    return (a1 * a2) / (b1 * b2);
  });
  return m;
}

template <typename T>
inline T ssim(const Image<T>& a, const Image<T>& b) {
  require(a.width == b.width && a.height == b.height, "ssim: image dimensions differ");
  T total = T(0);
  for (int c = 0; c < 3; ++c) total = total + map_mean(ssim_channel<T>(channel(a, c), channel(b, c)).s);
  return total / T(3);
}

template <typename T>
inline T ssim_with_grad(const Image<T>& a, const Image<T>& b, Image<T>& d_a) {
  require(a.width == b.width && a.height == b.height, "ssim: image dimensions differ");
  d_a = Image<T>(a.width, a.height);
  const T nrm = T(1) / (T(3) * T(a.width) * T(a.height));
  T total = T(0);
  for (int c = 0; c < 3; ++c) {
    const ScalarMap<T> x = channel(a, c);
    const ScalarMap<T> y = channel(b, c);
    const auto m = ssim_channel<T>(x, y);
    total = total + map_mean(m.s);
    ScalarMap<T> u_mu(x.h, x.w), u_mxy(x.h, x.w), u_mxx(x.h, x.w);
    for (size_t i = 0; i < x.d.size(); ++i) {
      const T mx = m.mu_x.d[i], my = m.mu_y.d[i];
      const T a1 = T(2) * mx * my + T(kSsimC1);
      const T a2 = T(2) * (m.mxy.d[i] - mx * my) + T(kSsimC2);
      const T b1 = mx * mx + my * my + T(kSsimC1);
      const T b2 = (m.mxx.d[i] - mx * mx) + (m.myy.d[i] - my * my) + T(kSsimC2);
      const T inv_bb = T(1) / (b1 * b2);
      const T s = m.s.d[i];
      u_mu.d[i] = nrm * (a2 * inv_bb * T(2) * my - a1 * inv_bb * T(2) * my - s / b1 * T(2) * mx +
                         s / b2 * T(2) * mx);
      u_mxy.d[i] = nrm * (a1 * inv_bb * T(2));
      u_mxx.d[i] = nrm * (-s / b2);
    }
    const ScalarMap<T> f_mu = gauss_filter(u_mu), f_mxy = gauss_filter(u_mxy), f_mxx = gauss_filter(u_mxx);
    for (int py = 0; py < a.height; ++py)
      for (int px = 0; px < a.width; ++px)
        d_a.at(px, py)[c] = f_mu(py, px) + f_mxy(py, px) * y(py, px) + f_mxx(py, px) * T(2) * x(py, px);
  }
  return total / T(3);
}

template <typename T>
inline double psnr(const Image<T>& a, const Image<T>& b) {
  require(a.width == b.width && a.height == b.height, "psnr: image dimensions differ");
  double mse = 0;
  // (a - b) in T, cast to double, squaredNorm = (d0^2 + d1^2) + d2^2
  for (size_t i = 0; i < a.pixels.size(); ++i) {
    const double d0 = double(a.pixels[i][0] - b.pixels[i][0]);
    const double d1 = double(a.pixels[i][1] - b.pixels[i][1]);
    const double d2 = double(a.pixels[i][2] - b.pixels[i][2]);
    mse += (d0 * d0 + d1 * d1) + d2 * d2;
  }
  mse /= 3.0 * a.pixels.size();
  if (mse < 1e-10) return 100.0;
  return 10.0 * std::log10(1.0 / mse);
}

// ---------------------------------------------------------------------------
// loss.hpp:21-47
// ---------------------------------------------------------------------------
template <typename T>
struct LossResult {
  T loss = T(0), l1 = T(0), ssim_value = T(0);
  Image<T> d_image;
};

template <typename T>
inline LossResult<T> training_loss(const Image<T>& rendered, const Image<T>& gt, T lambda) {
  require(rendered.width == gt.width && rendered.height == gt.height, "training_loss: image dimensions differ");
  LossResult<T> out;
  out.d_image = Image<T>(rendered.width, rendered.height);
  const T inv_n = T(1) / (T(3) * T(rendered.pixels.size()));
  T l1 = T(0);
  for (size_t i = 0; i < rendered.pixels.size(); ++i) {
    const Vec3<T> diff = rendered.pixels[i] - gt.pixels[i];
    l1 = l1 + ((std::abs(diff[0]) + std::abs(diff[1])) + std::abs(diff[2]));
    for (int c = 0; c < 3; ++c) {
      const T s = diff[c] > T(0) ? T(1) : (diff[c] < T(0) ? T(-1) : T(0));
      out.d_image.pixels[i][c] = (T(1) - lambda) * s * inv_n;
    }
  }
  out.l1 = l1 * inv_n;
  Image<T> d_ssim;
  out.ssim_value = ssim_with_grad(rendered, gt, d_ssim);
  for (size_t i = 0; i < rendered.pixels.size(); ++i)
    for (int c = 0; c < 3; ++c) out.d_image.pixels[i][c] = out.d_image.pixels[i][c] - lambda * d_ssim.pixels[i][c];
  out.loss = (T(1) - lambda) * out.l1 + lambda * (T(1) - out.ssim_value);
  return out;
}

// ---------------------------------------------------------------------------
// error_maps.hpp:14-43
// ---------------------------------------------------------------------------
template <typename T>
struct ErrorMaps {
  ScalarMap<T> raw, normalized;
  MaskMap mask;
  T photometric = T(0);
};

template <typename T>
inline ErrorMaps<T> build_error_maps(const Image<T>& rendered, const Image<T>& gt, T tau, T lambda) {
  require(rendered.width == gt.width && rendered.height == gt.height, "build_error_maps: image dimensions differ");
  const int w = rendered.width, h = rendered.height;
  ErrorMaps<T> out;
  out.raw = ScalarMap<T>(h, w);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const Vec3<T> d = rendered.at(x, y) - gt.at(x, y);
      out.raw(y, x) = ((std::abs(d[0]) + std::abs(d[1])) + std::abs(d[2])) / T(3);
    }
  T lo = out.raw.d[0], hi = out.raw.d[0];
  for (const T v : out.raw.d) {
    lo = std::min(lo, v);
    hi = std::max(hi, v);
  }
  out.normalized = ScalarMap<T>(h, w);
  if (hi > lo)
    for (size_t i = 0; i < out.raw.d.size(); ++i) out.normalized.d[i] = (out.raw.d[i] - lo) / (hi - lo);
  out.mask = MaskMap(h, w);
  for (size_t i = 0; i < out.raw.d.size(); ++i) out.mask.d[i] = out.normalized.d[i] > tau ? 1 : 0;
  const T l1 = map_mean(out.raw);
  out.photometric = (T(1) - lambda) * l1 + lambda * (T(1) - ssim(rendered, gt));
  return out;
}

// ---------------------------------------------------------------------------
// adc.hpp:18-289
// ---------------------------------------------------------------------------
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
    grad3d_acc.assign(n, Vec3<T>::zero());
    views_seen.assign(n, 0);
    max_radius2d.assign(n, T(0));
  }
  int size() const { return static_cast<int>(s_d.size()); }
};

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

template <typename T>
inline void scores_from_counts(const std::vector<std::vector<int>>& counts, const std::vector<T>& photometric,
                               ScoreTable<T>& table) {
  require(!counts.empty() && counts.size() == photometric.size(),
          "scores_from_counts: need one count row and one photometric value per view");
  const int k = static_cast<int>(counts.size());
  const int n = static_cast<int>(counts[0].size());
  table.s_d.assign(n, T(0));
  table.s_p_raw.assign(n, T(0));
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < n; ++i) {
      table.s_d[i] = table.s_d[i] + T(counts[j][i]);
      table.s_p_raw[i] = table.s_p_raw[i] + T(counts[j][i]) * photometric[j];
    }
  for (int i = 0; i < n; ++i) table.s_d[i] = table.s_d[i] / T(k);
  table.s_p = minmax_normalize(table.s_p_raw);
}

template <typename T>
inline void accumulate_scores(const Scene<T>& scene, const std::vector<ViewRef<T>>& views, T tau, T lambda,
                              const BinningConfig<T>& binning, int tile_size, ScoreTable<T>& table,
                              int workers = 1, std::vector<std::vector<int>>* counts_out = nullptr,
                              std::vector<T>* photometric_out = nullptr) {
  require(!views.empty(), "accumulate_scores: no training views");
  const int n = scene.size();
  const int k = static_cast<int>(views.size());
  std::vector<std::vector<int>> counts(k);
  std::vector<T> photometric(k, T(0));
  parallel_chunks(k, workers, [&](int, int begin, int end) {
    for (int j = begin; j < end; ++j) {
      const Camera<T>& cam = *views[j].camera;
      const auto pgs = project_scene(scene, cam);
      const TileGrid grid = build_tile_grid(pgs, cam.width, cam.height, binning, tile_size);
      const RenderOutputs<T> rendered = blend_forward(grid, pgs);
      const ErrorMaps<T> maps = build_error_maps(rendered.image, *views[j].image, tau, lambda);
      FootprintCounter counter(n);
      blend_forward(grid, pgs, &maps.mask, &counter);
      counts[j] = std::move(counter.counts);
      photometric[j] = maps.photometric;
    }
  });
  scores_from_counts(counts, photometric, table);
  if (counts_out) *counts_out = counts;
  if (photometric_out) *photometric_out = photometric;
}

template <typename T>
struct DensifyParams {
  T tau_d = T(5);
  T grad_threshold = T(2e-4);
  T percent_dense = T(0.01);
  bool use_vcd = true;
};

struct DensifySelection {
  std::vector<int> clone, split;
};

template <typename T>
inline T max_coeff(const Vec3<T>& v) {
  T m = v[0];
  if (v[1] > m) m = v[1];
  if (v[2] > m) m = v[2];
  return m;
}

template <typename T>
inline DensifySelection select_densify(const ScoreTable<T>& table, const Scene<T>& scene,
                                       const DensifyParams<T>& params, T scene_extent) {
  DensifySelection sel;
  for (int i = 0; i < scene.size(); ++i) {
    if (table.views_seen[i] == 0) continue;
    if (params.use_vcd && !(table.s_d[i] > params.tau_d)) continue;
    const T inv_seen = T(1) / T(table.views_seen[i]);
    const T mean_grad = table.grad_norm_acc[i] * inv_seen;
    const T mean_abs_grad = table.abs_grad_acc[i] * inv_seen;
    const bool small = max_coeff(scene.gaussians[i].scale()) <= params.percent_dense * scene_extent;
    if (small) {
      if (mean_grad >= params.grad_threshold) sel.clone.push_back(i);
    } else {
      if (mean_abs_grad >= params.grad_threshold) sel.split.push_back(i);
    }
  }
  return sel;
}

struct IndexRemap {
  std::vector<int> old_to_new;
  int new_size = 0;
};

inline constexpr double kSplitScaleShrink = 1.6;

// Split noise: Vec3(normal(), normal(), normal()) (adc.hpp:196). The order in
// which C++ evaluates those three constructor arguments is unspecified; this
// restatement (and the GPU trainer) draws them left to right.
template <typename T, typename NormalSource>
inline IndexRemap apply_densify_with(Scene<T>& scene, const std::vector<int>& clone, const std::vector<int>& split,
                                     const ScoreTable<T>& table, T clone_step_lr, NormalSource&& normal);

template <typename T>
inline IndexRemap apply_densify(Scene<T>& scene, const std::vector<int>& clone, const std::vector<int>& split,
                                const ScoreTable<T>& table, T clone_step_lr, Rng& rng) {
  return apply_densify_with(scene, clone, split, table, clone_step_lr, [&] { return rng.normal(); });
}

template <typename T, typename NormalSource>
inline IndexRemap apply_densify_with(Scene<T>& scene, const std::vector<int>& clone, const std::vector<int>& split,
                                     const ScoreTable<T>& table, T clone_step_lr, NormalSource&& normal) {
  const int n = scene.size();
  IndexRemap remap;
  remap.old_to_new.assign(n, -1);
  std::vector<bool> is_split(n, false);
  for (const int i : split) is_split[i] = true;
  std::vector<Gaussian3D<T>> next;
  next.reserve(n + clone.size() + 2 * split.size());
  for (int i = 0; i < n; ++i) {
    if (is_split[i]) continue;
    remap.old_to_new[i] = static_cast<int>(next.size());
    next.push_back(scene.gaussians[i]);
  }
  for (const int i : clone) {
    Gaussian3D<T> g = scene.gaussians[i];
    if (table.views_seen[i] > 0) {
      const T vs = T(table.views_seen[i]);
      for (int d = 0; d < 3; ++d) g.mu[d] = g.mu[d] - clone_step_lr * (table.grad3d_acc[i][d] / vs);
    }
    next.push_back(std::move(g));
  }
  for (const int i : split) {
    const Gaussian3D<T>& parent = scene.gaussians[i];
    const Mat3<T> rot = quat_to_rotation(parent.rot);
    const Vec3<T> scale = parent.scale();
    for (int c = 0; c < 2; ++c) {
      Gaussian3D<T> child = parent;
      Vec3<T> eps;
      eps[0] = T(normal());
      eps[1] = T(normal());
      eps[2] = T(normal());
      Vec3<T> es;
      for (int d = 0; d < 3; ++d) es[d] = eps[d] * scale[d];
      child.mu = parent.mu + rot * es;
      for (int d = 0; d < 3; ++d) child.log_scale[d] = parent.log_scale[d] - T(std::log(kSplitScaleShrink));
      next.push_back(std::move(child));
    }
  }
  scene.gaussians = std::move(next);
  remap.new_size = scene.size();
  return remap;
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

template <typename T>
inline std::vector<int> select_prune(const ScoreTable<T>& table, const Scene<T>& scene, int iteration,
                                     const PruneParams<T>& params, T scene_extent) {
  const int n = scene.size();
  std::vector<int> pruned;
  if (iteration < params.densify_until) {
    std::vector<int> candidates;
    for (int i = 0; i < n; ++i) {
      const Gaussian3D<T>& g = scene.gaussians[i];
      bool cand = g.opacity() < params.min_opacity;
      if (iteration > params.size_prune_from) {
        cand = cand || max_coeff(g.scale()) > params.world_size_frac * scene_extent;
        cand = cand || table.max_radius2d[i] > params.screen_size;
      }
      if (cand) candidates.push_back(i);
    }
    if (!params.use_vcp) {
      pruned = std::move(candidates);
    } else {
      std::sort(candidates.begin(), candidates.end(), [&](int a, int b) {
        if (table.s_p[a] != table.s_p[b]) return table.s_p[a] > table.s_p[b];
        return a < b;
      });
      const int take = (static_cast<int>(candidates.size()) + 1) / 2;
      pruned.assign(candidates.begin(), candidates.begin() + take);
      std::sort(pruned.begin(), pruned.end());
    }
  } else {
    const T opacity_cut = params.use_vcp ? params.opacity_late : params.min_opacity;
    for (int i = 0; i < n; ++i) {
      const bool low = scene.gaussians[i].opacity() < opacity_cut;
      const bool scored = params.use_vcp && table.s_p[i] > params.tau_p;
      if (low || scored) pruned.push_back(i);
    }
  }
  if (static_cast<int>(pruned.size()) == n && n > 0) {
    int keep = 0;
    for (int i = 1; i < n; ++i)
      if (table.s_p[i] < table.s_p[keep]) keep = i;
    pruned.erase(std::find(pruned.begin(), pruned.end(), keep));
  }
  return pruned;
}

template <typename T>
inline IndexRemap apply_prune(Scene<T>& scene, const std::vector<int>& prune) {
  const int n = scene.size();
  std::vector<bool> drop(n, false);
  for (const int i : prune) drop[i] = true;
  IndexRemap remap;
  remap.old_to_new.assign(n, -1);
  std::vector<Gaussian3D<T>> next;
  next.reserve(n - prune.size());
  for (int i = 0; i < n; ++i) {
    if (drop[i]) continue;
    remap.old_to_new[i] = static_cast<int>(next.size());
    next.push_back(std::move(scene.gaussians[i]));
  }
  scene.gaussians = std::move(next);
  remap.new_size = scene.size();
  return remap;
}

// ---------------------------------------------------------------------------
// adam.hpp:16-164
// ---------------------------------------------------------------------------
inline constexpr double kAdamBeta1 = 0.9;
inline constexpr double kAdamBeta2 = 0.999;
inline constexpr double kAdamEps = 1e-15;

template <typename T>
inline T expon_lr(T lr_init, T lr_final, int step, int max_steps) {
  const T t = clamp_ref(T(step) / T(std::max(1, max_steps)), T(0), T(1));
  return std::exp((T(1) - t) * std::log(lr_init) + t * std::log(lr_final));
}

template <typename T>
struct AdamGroup {
  int dim = 1;
  std::vector<T> m, v;
  std::int64_t t = 0;
  void init(int n, int d) {
    dim = d;
    m.assign(size_t(n) * d, T(0));
    v.assign(size_t(n) * d, T(0));
    t = 0;
  }
  void remap(const IndexRemap& r) {
    std::vector<T> nm(size_t(r.new_size) * dim, T(0)), nv(size_t(r.new_size) * dim, T(0));
    for (size_t i = 0; i < r.old_to_new.size(); ++i) {
      const int j = r.old_to_new[i];
      if (j < 0) continue;
      for (int d = 0; d < dim; ++d) {
        nm[size_t(j) * dim + d] = m[i * dim + d];
        nv[size_t(j) * dim + d] = v[i * dim + d];
      }
    }
    m = std::move(nm);
    v = std::move(nv);
  }
  // bias corrections are std::pow in T (adam.hpp:64-66)
  template <typename ParamAt, typename GradAt>
  void step(T lr, int n, ParamAt param_at, GradAt grad_at) {
    ++t;
    const T bc1 = T(1) - std::pow(T(kAdamBeta1), T(t));
    const T bc2 = T(1) - std::pow(T(kAdamBeta2), T(t));
    for (int i = 0; i < n; ++i)
      for (int d = 0; d < dim; ++d) {
        const size_t s = size_t(i) * dim + d;
        const T g = grad_at(i, d);
        m[s] = T(kAdamBeta1) * m[s] + (T(1) - T(kAdamBeta1)) * g;
        v[s] = T(kAdamBeta2) * v[s] + (T(1) - T(kAdamBeta2)) * g * g;
        param_at(i, d) = param_at(i, d) - lr * (m[s] / bc1) / (std::sqrt(v[s] / bc2) + T(kAdamEps));
      }
  }
};

template <typename T>
struct LearningRates {
  T position = T(1.6e-4), position_final = T(1.6e-6), sh_dc = T(2.5e-3), sh_rest = T(2.5e-3 / 20),
    opacity = T(5e-2), scale = T(5e-3), rotation = T(1e-3);
};

template <typename T>
struct SceneGrads {
  std::vector<GaussianGrads<T>> per_gaussian;
  void init(const Scene<T>& scene) {
    per_gaussian.assign(scene.size(), GaussianGrads<T>{});
    for (auto& g : per_gaussian) g.sh = ShMatrix<T>(sh_coeff_count(scene.sh_degree));
  }
};

template <typename T>
class SceneOptimizer {
 public:
  void init(const Scene<T>& scene) {
    const int n = scene.size();
    n_sh_ = sh_coeff_count(scene.sh_degree);
    pos_.init(n, 3);
    rot_.init(n, 4);
    scale_.init(n, 3);
    opacity_.init(n, 1);
    sh_dc_.init(n, 3);
    sh_rest_.init(n, 3 * std::max(0, n_sh_ - 1));
  }
  void remap(const IndexRemap& r) {
    pos_.remap(r);
    rot_.remap(r);
    scale_.remap(r);
    opacity_.remap(r);
    sh_dc_.remap(r);
    sh_rest_.remap(r);
  }
  void step(Scene<T>& scene, const SceneGrads<T>& grads, const LearningRates<T>& lrs, T position_lr,
            bool update_sh_rest = true) {
    const int n = scene.size();
    auto& gs = scene.gaussians;
    const auto& pg = grads.per_gaussian;
    pos_.step(position_lr, n, [&](int i, int d) -> T& { return gs[i].mu[d]; }, [&](int i, int d) { return pg[i].mu[d]; });
    rot_.step(lrs.rotation, n, [&](int i, int d) -> T& { return gs[i].rot[d]; }, [&](int i, int d) { return pg[i].rot[d]; });
    scale_.step(lrs.scale, n, [&](int i, int d) -> T& { return gs[i].log_scale[d]; },
                [&](int i, int d) { return pg[i].log_scale[d]; });
    opacity_.step(lrs.opacity, n, [&](int i, int) -> T& { return gs[i].opacity_logit; },
                  [&](int i, int) { return pg[i].opacity_logit; });
    sh_dc_.step(lrs.sh_dc, n, [&](int i, int d) -> T& { return gs[i].sh(0, d); }, [&](int i, int d) { return pg[i].sh(0, d); });
    if (update_sh_rest && n_sh_ > 1)
      sh_rest_.step(lrs.sh_rest, n, [&](int i, int d) -> T& { return gs[i].sh(1 + d / 3, d % 3); },
                    [&](int i, int d) { return pg[i].sh(1 + d / 3, d % 3); });
  }
  void step_sh_rest(Scene<T>& scene, const std::vector<ShMatrix<T>>& rest_grads, const LearningRates<T>& lrs) {
    if (n_sh_ <= 1) return;
    sh_rest_.step(lrs.sh_rest, scene.size(), [&](int i, int d) -> T& { return scene.gaussians[i].sh(1 + d / 3, d % 3); },
                  [&](int i, int d) { return rest_grads[i](1 + d / 3, d % 3); });
  }
  void reset_opacity_state() {
    std::fill(opacity_.m.begin(), opacity_.m.end(), T(0));
    std::fill(opacity_.v.begin(), opacity_.v.end(), T(0));
  }
  AdamGroup<T> pos_, rot_, scale_, opacity_, sh_dc_, sh_rest_;
  int n_sh_ = 16;
};

// ---------------------------------------------------------------------------
// config.hpp:20-81 (struct + validate only; the file parser is out of scope)
// ---------------------------------------------------------------------------
struct TrainConfig {
  int iterations = 30000;
  int k = 10;
  double lambda = 0.2, tau = 0.5, tau_d = 5.0, tau_p = 0.9, beta = 1.0, tau_alpha = 1.0 / 255;
  int densify_from = 500, densify_until = 15000, densify_every = 500, prune_every_early = 500, prune_every_late = 3000;
  double grad_threshold = 2e-4, percent_dense = 0.01;
  double lr_position = 1.6e-4, lr_position_final = 1.6e-6, lr_sh_dc = 2.5e-3, lr_sh_rest = 2.5e-3 / 20,
         lr_opacity = 5e-2, lr_scale = 5e-3, lr_rotation = 1e-3;
  int opacity_reset_every = 0;
  bool lazy_opt_enabled = false;
  int lazy_opt_interval_15k = 32, lazy_opt_interval_20k = 64;
  std::uint64_t seed = 0;
  int tile_size = 16, workers = 1, sh_degree = 3;
  bool compact = false;  // bin_mode == "compact"
  bool vcd = true, vcp = true;
  double prune_min_opacity = 0.005, prune_opacity_late = 0.1, prune_world_size_frac = 0.1, prune_screen_size = 20.0;
  int size_prune_from = 3000;
  bool schedule_dry_run = false;
  void validate() const {
    require(iterations >= 0, "config: iterations must be >= 0");
    require(k >= 1, "config: k must be >= 1");
    require(lambda >= 0 && lambda <= 1, "config: lambda must be in [0,1]");
    require(tau > 0 && tau < 1, "config: tau must be in (0,1)");
    require(tau_d >= 0, "config: tau_d must be >= 0");
    require(tau_p >= 0 && tau_p <= 1, "config: tau_p must be in [0,1]");
    require(beta > 0 && beta <= 1, "config: beta must be in (0,1]");
    require(tau_alpha > 0 && tau_alpha < 1, "config: tau_alpha must be in (0,1)");
    require(densify_every > 0 && prune_every_early > 0 && prune_every_late > 0, "config: event cadences must be positive");
    require((densify_until - densify_from) % densify_every == 0,
            "config: densify_every must divide densify_until - densify_from");
    require(tile_size > 0, "config: tile_size must be positive");
    require(sh_degree >= 0 && sh_degree <= 3, "config: sh_degree must be in 0..3");
  }
};

// ---------------------------------------------------------------------------
// dataset.hpp:24-250 (in-memory; PNG round trip emulated by 8-bit quantisation)
// ---------------------------------------------------------------------------
template <typename T>
struct Dataset {
  std::vector<Camera<T>> cameras;
  std::vector<Image<T>> images;
  std::vector<std::vector<std::uint8_t>> images_u8;  // the PNG bytes, HWC
  std::vector<std::pair<Vec3<T>, Vec3<T>>> init_points;
  std::vector<int> train_indices, test_indices;
  T extent = T(1);
};

inline void split_views(int n, std::vector<int>& train, std::vector<int>& test) {
  train.clear();
  test.clear();
  for (int i = 0; i < n; ++i) (i % 8 == 0 ? test : train).push_back(i);
  if (train.empty()) {
    train = std::move(test);
    test.clear();
  }
}

template <typename T>
inline T scene_extent(const std::vector<Camera<T>>& cameras, const std::vector<std::pair<Vec3<T>, Vec3<T>>>& points) {
  Vec3<T> center = Vec3<T>::zero();
  for (const auto& c : cameras) center += c.center();
  if (!cameras.empty()) center = center / T(cameras.size());
  T radius = T(0);
  for (const auto& c : cameras) radius = std::max(radius, norm(c.center() - center));
  for (const auto& p : points) radius = std::max(radius, norm(p.first - center));
  radius = radius * T(1.1);
  return radius > T(1e-9) ? radius : T(1);
}

template <typename T>
inline Vec3<T> cross(const Vec3<T>& a, const Vec3<T>& b) {
  return v3(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
}

template <typename T>
inline Mat4<T> look_at(const Vec3<T>& eye, const Vec3<T>& target, const Vec3<T>& up) {
  const Vec3<T> zd = target - eye;
  const Vec3<T> z = zd / norm(zd);
  const Vec3<T> xc = cross(z, up);
  const Vec3<T> x = xc / norm(xc);
  const Vec3<T> y = cross(z, x);
  Mat4<T> m = Mat4<T>::identity();
  for (int j = 0; j < 3; ++j) {
    m(0, j) = x[j];
    m(1, j) = y[j];
    m(2, j) = z[j];
  }
  Mat3<T> r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = m(i, j);
  const Vec3<T> t = r * eye;
  for (int i = 0; i < 3; ++i) m(i, 3) = -t[i];
  return m;
}

// PNG round trip: write lround(clamp(v,0,1)*255) (png_io.cpp:97-98), read byte/255.0f (:64).
inline std::uint8_t quantize_u8(float v) {
  const float c = std::min(1.0f, std::max(0.0f, v));
  return static_cast<std::uint8_t>(std::lround(c * 255.0f));
}

struct SynthSpec {
  int n_gaussians = 500;
  int n_views = 64;
  int width = 128;   // the reference has one image_size; width == height there
  int height = 128;
  std::uint64_t seed = 1;
  double scale_mult = 1.0;  // (500/N)^(1/3) for the large configs
  double focal = -1.0;      // <0: reference 1.1 * size
};

// dataset.hpp:178-250 without file output. Returns the GT scene; the views are
// rendered by this oracle's own rasterizer and quantised through 8 bits.
inline Scene<float> generate_synthetic(const SynthSpec& spec, Dataset<float>& data, bool render_images = true) {
  require(spec.n_views >= 2, "synthetic: n_views must be >= 2");
  require(spec.n_gaussians >= 1, "synthetic: n_gaussians must be >= 1");
  Rng rng(spec.seed);
  Scene<float> gt;
  gt.sh_degree = 1;
  gt.gaussians.reserve(spec.n_gaussians);
  for (int i = 0; i < spec.n_gaussians; ++i) {
    Gaussian3D<float> g;
    for (int d = 0; d < 3; ++d) g.mu[d] = static_cast<float>(rng.uniform(-0.5, 0.5));
    Vec4<float> q;
    for (int d = 0; d < 4; ++d) q[d] = static_cast<float>(rng.normal());
    const float qn = norm(q);
    if (qn > 1e-6f) {
      g.rot = q / qn;
    } else {
      g.rot[0] = 1; g.rot[1] = g.rot[2] = g.rot[3] = 0;
    }
    for (int d = 0; d < 3; ++d)
      g.log_scale[d] = std::log(static_cast<float>(rng.uniform(0.02, 0.075) * spec.scale_mult));
    g.opacity_logit = logit(static_cast<float>(rng.uniform(0.25, 0.95)));
    g.sh = ShMatrix<float>(sh_coeff_count(gt.sh_degree));
    for (int c = 0; c < 3; ++c) g.sh(0, c) = static_cast<float>((rng.uniform(0.05, 0.95) - 0.5) / kShC0);
    for (int m = 1; m < sh_coeff_count(gt.sh_degree); ++m)
      for (int c = 0; c < 3; ++c) g.sh(m, c) = static_cast<float>(rng.uniform(-0.1, 0.1));
    gt.gaussians.push_back(std::move(g));
  }
  data = Dataset<float>{};
  const float ring_radius = 2.4f, ring_height = 1.0f;
  for (int v = 0; v < spec.n_views; ++v) {
    const float angle = 2.0f * static_cast<float>(M_PI) * v / spec.n_views;
    Camera<float> cam;
    cam.width = spec.width;
    cam.height = spec.height;
    cam.fx = cam.fy = spec.focal > 0 ? static_cast<float>(spec.focal) : 1.1f * spec.height;
    cam.cx = (spec.width - 1) / 2.0f;
    cam.cy = (spec.height - 1) / 2.0f;
    cam.near = 0.2f;
    const Vec3<float> eye = v3(ring_radius * std::cos(angle), ring_radius * std::sin(angle), ring_height);
    cam.world_to_cam = look_at<float>(eye, Vec3<float>::zero(), v3(0.0f, 0.0f, 1.0f));
    data.cameras.push_back(cam);
  }
  if (render_images) {
    const BinningConfig<float> binning;
    for (int v = 0; v < spec.n_views; ++v) {
      const auto pgs = project_scene(gt, data.cameras[v]);
      const TileGrid grid = build_tile_grid(pgs, spec.width, spec.height, binning);
      const RenderOutputs<float> out = blend_forward(grid, pgs);
      std::vector<std::uint8_t> bytes(size_t(spec.width) * spec.height * 3);
      Image<float> img(spec.width, spec.height);
      for (size_t p = 0; p < out.image.pixels.size(); ++p)
        for (int c = 0; c < 3; ++c) {
          bytes[p * 3 + c] = quantize_u8(out.image.pixels[p][c]);
          img.pixels[p][c] = bytes[p * 3 + c] / 255.0f;
        }
      data.images_u8.push_back(std::move(bytes));
      data.images.push_back(std::move(img));
    }
  }
  const float extent = scene_extent<float>(data.cameras, {});
  const float noise = 0.05f * extent;
  for (const auto& g : gt.gaussians) {
    Vec3<float> p = g.mu;
    for (int d = 0; d < 3; ++d) p[d] = p[d] + noise * static_cast<float>(rng.normal());
    Vec3<float> color;
    for (int c = 0; c < 3; ++c) color[c] = std::clamp(0.5f + static_cast<float>(kShC0) * g.sh(0, c), 0.0f, 1.0f);
    data.init_points.push_back({p, color});
  }
  split_views(spec.n_views, data.train_indices, data.test_indices);
  data.extent = scene_extent(data.cameras, data.init_points);
  return gt;
}

// ---------------------------------------------------------------------------
// trainer.hpp:21-279
// ---------------------------------------------------------------------------
struct LogRow {
  int iteration = 0;
  double loss = 0, psnr = 0;
  int gaussians = 0;
  std::int64_t tile_pairs = 0;
  double elapsed_ms = 0;
};

inline bool densify_due(int it, const TrainConfig& cfg) {
  return it >= cfg.densify_from && it <= cfg.densify_until && it % cfg.densify_every == 0;
}
inline bool prune_due(int it, const TrainConfig& cfg) {
  if (it >= cfg.densify_from && it <= cfg.densify_until) return it % cfg.prune_every_early == 0;
  if (it > cfg.densify_until) return (it - cfg.densify_until) % cfg.prune_every_late == 0;
  return false;
}
inline bool lazy_update_due(int it, const TrainConfig& cfg) {
  if (!cfg.lazy_opt_enabled || it < 15000) return true;
  if (it < 20000) return it % cfg.lazy_opt_interval_15k == 0;
  return it % cfg.lazy_opt_interval_20k == 0;
}

// Event record exposed to the parity tests (masks compared per event).
struct EventRecord {
  int iteration = 0;
  std::vector<int> sampled;       // view indices (into cameras)
  std::vector<float> photometric;
  std::vector<int> clone, split, prune;  // pre-event indices (own selection)
  int n_before = 0, n_after = 0;
  bool forced = false;
};

// Decisions to replay at one event (flags over the pre-event indices).
struct ForcedEvent {
  int n = 0;
  std::vector<std::uint8_t> clone, split, prune;
};

template <typename T>
class Trainer {
 public:
  Trainer(Scene<T> scene, const Dataset<T>& data, const TrainConfig& cfg)
      : scene_(std::move(scene)), data_(data), cfg_(cfg), rng_(cfg.seed) {
    cfg_.validate();
    require(!data.cameras.empty(), "trainer: dataset has no views");
    require(!data.train_indices.empty(), "trainer: dataset has no training views");
    binning_.mode = cfg_.compact ? BinMode::kCompact : BinMode::kAabb;
    binning_.beta = T(cfg_.beta);
    binning_.tau_alpha = T(cfg_.tau_alpha);
    lrs_.position = T(cfg_.lr_position);
    lrs_.position_final = T(cfg_.lr_position_final);
    lrs_.sh_dc = T(cfg_.lr_sh_dc);
    lrs_.sh_rest = T(cfg_.lr_sh_rest);
    lrs_.opacity = T(cfg_.lr_opacity);
    lrs_.scale = T(cfg_.lr_scale);
    lrs_.rotation = T(cfg_.lr_rotation);
    optimizer_.init(scene_);
    table_.reset(scene_.size());
  }

  std::vector<LogRow> run(int iterations_to_run = -1) {
    std::vector<LogRow> log;
    const int last = iterations_to_run < 0 ? cfg_.iterations : std::min(cfg_.iterations, it_ + iterations_to_run);
    while (it_ < last) {
      const int it = ++it_;
      LogRow row;
      row.iteration = it;
      if (!cfg_.schedule_dry_run) row = train_iteration(it);
      const bool densify = densify_due(it, cfg_);
      const bool prune = prune_due(it, cfg_);
      if (!cfg_.schedule_dry_run && (densify || prune)) density_event(it, densify, prune);
      if (!cfg_.schedule_dry_run && cfg_.opacity_reset_every > 0 && it % cfg_.opacity_reset_every == 0) reset_opacity();
      row.iteration = it;
      row.gaussians = scene_.size();
      log.push_back(row);
    }
    return log;
  }

  const Scene<T>& scene() const { return scene_; }
  const ScoreTable<T>& table() const { return table_; }
  const std::vector<EventRecord>& events() const { return events_; }
  int iteration() const { return it_; }
  // Test hook: resume the schedule at iteration `it` (exercises the late
  // lazy SH-rest intervals without running 15000 iterations).
  void set_iteration(int it) { it_ = it; }
  const SceneOptimizer<T>& optimizer() const { return optimizer_; }

  LogRow train_iteration(int it) {
    LogRow row;
    const int view = data_.train_indices[size_t(rng_.bounded(std::uint64_t(data_.train_indices.size())))];
    const Camera<T>& cam = data_.cameras[view];
    const Image<T>& gt = data_.images[view];
    const auto pgs = project_scene(scene_, cam);
    const TileGrid grid = build_tile_grid(pgs, cam.width, cam.height, binning_, cfg_.tile_size);
    const RenderOutputs<T> rendered = blend_forward(grid, pgs, nullptr, nullptr, cfg_.workers);
    const LossResult<T> loss = training_loss(rendered.image, gt, T(cfg_.lambda));
    const BlendGrads<T> bg = blend_backward(grid, pgs, loss.d_image, cfg_.workers);
    SceneGrads<T> grads;
    grads.init(scene_);
    const T ndc_x = T(cam.width) / T(2);
    const T ndc_y = T(cam.height) / T(2);
    for (size_t p = 0; p < pgs.size(); ++p) {
      const ProjectedGaussian<T>& pg = pgs[p];
      const Mat2<T> d_cov2d = cov_grad_from_inv_grad(pg.cov2d_inv, bg.d_conic[p]);
      const int src = pg.source_index;
      grads.per_gaussian[src] = project_backward(scene_.gaussians[src], cam, scene_.sh_degree, bg.d_mu2d[p], d_cov2d,
                                                 bg.d_color[p], bg.d_opacity[p]);
      Vec2<T> g_ndc;
      g_ndc[0] = bg.d_mu2d[p][0] * ndc_x;
      g_ndc[1] = bg.d_mu2d[p][1] * ndc_y;
      table_.grad_norm_acc[src] = table_.grad_norm_acc[src] + norm(g_ndc);
      table_.abs_grad_acc[src] = table_.abs_grad_acc[src] + (bg.abs_grad[p][0] * ndc_x + bg.abs_grad[p][1] * ndc_y);
      table_.grad3d_acc[src] += grads.per_gaussian[src].mu;
      table_.views_seen[src] += 1;
      table_.max_radius2d[src] =
          std::max(table_.max_radius2d[src], T(kBinSigma) * std::sqrt(max_eigenvalue_2x2(pg.cov2d)));
    }
    const T pos_lr = expon_lr(T(cfg_.lr_position) * data_.extent, T(cfg_.lr_position_final) * data_.extent, it,
                              cfg_.iterations);
    if (!cfg_.lazy_opt_enabled) {
      optimizer_.step(scene_, grads, lrs_, pos_lr, true);
    } else {
      optimizer_.step(scene_, grads, lrs_, pos_lr, false);
      if (rest_accum_.size() != size_t(scene_.size())) clear_rest();
      for (int i = 0; i < scene_.size(); ++i)
        for (size_t e = 0; e < rest_accum_[i].d.size(); ++e)
          rest_accum_[i].d[e] = rest_accum_[i].d[e] + grads.per_gaussian[i].sh.d[e];
      if (lazy_update_due(it, cfg_)) {
        optimizer_.step_sh_rest(scene_, rest_accum_, lrs_);
        clear_rest();
      }
    }
    row.loss = double(loss.loss);
    row.psnr = psnr(rendered.image, gt);
    row.tile_pairs = count_pairs(grid);
    last_view_ = view;
    return row;
  }

  void density_event(int it, bool densify, bool prune) {
    EventRecord rec;
    rec.iteration = it;
    rec.n_before = scene_.size();
    const std::vector<int> sampled =
        rng_.sample_without_replacement(static_cast<int>(data_.train_indices.size()), cfg_.k);
    std::vector<ViewRef<T>> views;
    for (const int s : sampled) {
      const int v = data_.train_indices[s];
      views.push_back({&data_.cameras[v], &data_.images[v]});
      rec.sampled.push_back(v);
    }
    std::vector<T> photo;
    accumulate_scores(scene_, views, T(cfg_.tau), T(cfg_.lambda), binning_, cfg_.tile_size, table_, cfg_.workers,
                      nullptr, &photo);
    for (const T p : photo) rec.photometric.push_back(float(p));
    DensifySelection sel;
    if (densify) {
      DensifyParams<T> dp;
      dp.tau_d = T(cfg_.tau_d);
      dp.grad_threshold = T(cfg_.grad_threshold);
      dp.percent_dense = T(cfg_.percent_dense);
      dp.use_vcd = cfg_.vcd;
      sel = select_densify(table_, scene_, dp, data_.extent);
    }
    std::vector<int> prune_set;
    if (prune) {
      PruneParams<T> pp;
      pp.tau_p = T(cfg_.tau_p);
      pp.min_opacity = T(cfg_.prune_min_opacity);
      pp.opacity_late = T(cfg_.prune_opacity_late);
      pp.world_size_frac = T(cfg_.prune_world_size_frac);
      pp.screen_size = T(cfg_.prune_screen_size);
      pp.size_prune_from = cfg_.size_prune_from;
      pp.densify_until = cfg_.densify_until;
      pp.use_vcp = cfg_.vcp;
      prune_set = select_prune(table_, scene_, it, pp, data_.extent);
    }
    if (!prune_set.empty()) {
      std::vector<bool> dropped(scene_.size(), false);
      for (const int i : prune_set) dropped[i] = true;
      std::erase_if(sel.clone, [&](int i) { return dropped[i]; });
      std::erase_if(sel.split, [&](int i) { return dropped[i]; });
    }
    rec.clone = sel.clone;
    rec.split = sel.split;
    rec.prune = prune_set;
    // Parity "follow" mode: replay another run's decisions (e.g. the GPU's) so
    // both runs keep consuming the shared Rng identically; the oracle's own
    // selection stays in the record for flip reporting.
    const size_t ev_index = events_.size();
    if (ev_index < forced_.size() && forced_[ev_index].n == scene_.size()) {
      const auto& f = forced_[ev_index];
      sel.clone.clear();
      sel.split.clear();
      prune_set.clear();
      for (int i = 0; i < f.n; ++i) {
        if (f.prune[i]) prune_set.push_back(i);
        else {
          if (f.clone[i]) sel.clone.push_back(i);
          if (f.split[i]) sel.split.push_back(i);
        }
      }
      rec.forced = true;
    }
    const IndexRemap prune_remap = apply_prune(scene_, prune_set);
    optimizer_.remap(prune_remap);
    for (int& i : sel.clone) i = prune_remap.old_to_new[i];
    for (int& i : sel.split) i = prune_remap.old_to_new[i];
    ScoreTable<T> mapped;
    mapped.reset(prune_remap.new_size);
    for (size_t i = 0; i < prune_remap.old_to_new.size(); ++i) {
      const int j = prune_remap.old_to_new[i];
      if (j < 0) continue;
      mapped.grad3d_acc[j] = table_.grad3d_acc[i];
      mapped.views_seen[j] = table_.views_seen[i];
    }
    const T pos_lr = expon_lr(T(cfg_.lr_position) * data_.extent, T(cfg_.lr_position_final) * data_.extent, it,
                              cfg_.iterations);
    const IndexRemap densify_remap = apply_densify(scene_, sel.clone, sel.split, mapped, pos_lr, rng_);
    optimizer_.remap(densify_remap);
    table_.reset(scene_.size());
    clear_rest();
    rec.n_after = scene_.size();
    events_.push_back(std::move(rec));
  }

  void reset_opacity() {
    const T cap = logit(T(0.01));
    for (auto& g : scene_.gaussians) g.opacity_logit = std::min(g.opacity_logit, cap);
    optimizer_.reset_opacity_state();
  }

  void clear_rest() {
    rest_accum_.assign(scene_.size(), ShMatrix<T>(sh_coeff_count(scene_.sh_degree)));
  }

  Scene<T> scene_;
  const Dataset<T>& data_;
  TrainConfig cfg_;
  Rng rng_;
  BinningConfig<T> binning_;
  LearningRates<T> lrs_;
  SceneOptimizer<T> optimizer_;
  ScoreTable<T> table_;
  std::vector<ShMatrix<T>> rest_accum_;
  std::vector<EventRecord> events_;
  std::vector<ForcedEvent> forced_;
  int it_ = 0;
  int last_view_ = -1;
};

}  // namespace oracle
