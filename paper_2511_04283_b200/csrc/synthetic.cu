// Scene construction on the device:
//
// * sk_synthetic_create restates generate_synthetic (reference
//   dataset.hpp:178-250): the GT Gaussians are drawn on the host with the
//   reference Rng in its exact draw order (mu, q, scale, opacity, DC, rest
//   per Gaussian; then the init-point noise), the camera ring is built with
//   look_at (dataset.hpp:207-219), and every GT view is rendered on the GPU by
//   the bit-exact K1-K6 path and quantised through 8 bits as the PNG path does
//   (lround(clamp(v)·255), png_io.cpp:97-98) straight into the dataset's
//   device images. The CPU reference renders each view with its CPU
//   rasterizer, which is what makes configs 3-5 (1M-8M Gaussians, 200-512
//   views) impractical there.
// * sk_init_from_points restates init_from_points (scene.hpp:117-141): the
//   mean distance to the three nearest neighbours is an O(n^2) brute-force
//   scan in the reference; here it is a shared-memory-tiled all-pairs kernel
//   (same fp32 distance expression, compiled without FMA contraction), and
//   the per-point log / logit / DC terms are evaluated on the host with the
//   same libm calls as the reference.
//
// Host arithmetic in this file is compiled with -ffp-contract=off (builder.py),
// so every value matches the CPU oracle bit for bit.
#include <cmath>
#include <memory>
#include <vector>

#include "abi_util.h"
#include "trainer.h"

namespace sk {
namespace {

constexpr double kShC0 = 0.28209479177387814;

struct V3 {
  float v[3];
  float& operator[](int i) { return v[i]; }
  float operator[](int i) const { return v[i]; }
};
V3 v3(float a, float b, float c) { return V3{{a, b, c}}; }
V3 sub(const V3& a, const V3& b) { return v3(a[0] - b[0], a[1] - b[1], a[2] - b[2]); }
float dot(const V3& a, const V3& b) {
  float s = a[0] * b[0];
  s = s + a[1] * b[1];
  s = s + a[2] * b[2];
  return s;
}
float norm(const V3& a) { return std::sqrt(dot(a, a)); }
V3 divs(const V3& a, float s) { return v3(a[0] / s, a[1] / s, a[2] / s); }
V3 cross(const V3& a, const V3& b) {
  return v3(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
}

// look_at (dataset.hpp:162-176): rows x, y, z of the rotation, t = -R eye.
void look_at(const V3& eye, float* m /*row-major 4x4*/) {
  const V3 zd = sub(v3(0.0f, 0.0f, 0.0f), eye);
  const V3 z = divs(zd, norm(zd));
  const V3 xc = cross(z, v3(0.0f, 0.0f, 1.0f));
  const V3 x = divs(xc, norm(xc));
  const V3 y = cross(z, x);
  for (int i = 0; i < 16; ++i) m[i] = (i % 5 == 0) ? 1.0f : 0.0f;
  for (int j = 0; j < 3; ++j) {
    m[0 * 4 + j] = x[j];
    m[1 * 4 + j] = y[j];
    m[2 * 4 + j] = z[j];
  }
  for (int i = 0; i < 3; ++i) {
    float s = m[i * 4 + 0] * eye[0];
    s = s + m[i * 4 + 1] * eye[1];
    s = s + m[i * 4 + 2] * eye[2];
    m[i * 4 + 3] = -s;
  }
}

// Camera::center (camera.hpp:32): -R^T t.
V3 camera_center(const sk_camera& c) {
  V3 o;
  for (int r = 0; r < 3; ++r) {
    float s = c.world_to_cam[0 * 4 + r] * c.world_to_cam[0 * 4 + 3];
    for (int k = 1; k < 3; ++k) s = s + c.world_to_cam[k * 4 + r] * c.world_to_cam[k * 4 + 3];
    o[r] = s;
  }
  return v3(-o[0], -o[1], -o[2]);
}

// scene_extent (dataset.hpp:56-66).
float scene_extent(const std::vector<sk_camera>& cams, const std::vector<V3>& points) {
  V3 center = v3(0.0f, 0.0f, 0.0f);
  for (const auto& c : cams) {
    const V3 cc = camera_center(c);
    for (int i = 0; i < 3; ++i) center[i] = center[i] + cc[i];
  }
  if (!cams.empty()) center = divs(center, (float)cams.size());
  float radius = 0.0f;
  for (const auto& c : cams) radius = std::max(radius, norm(sub(camera_center(c), center)));
  for (const auto& p : points) radius = std::max(radius, norm(sub(p, center)));
  radius = radius * 1.1f;
  return radius > 1e-9f ? radius : 1.0f;
}

float logit(float x) { return std::log(x / (1.0f - x)); }

// lround(clamp(v, 0, 1) * 255) of the planar render into 8-bit HWC.
__global__ void quantize_kernel(const float* __restrict__ img, int64_t plane, uint8_t* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= plane) return;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float v = fminf(1.0f, fmaxf(0.0f, img[c * plane + p]));
    out[p * 3 + c] = (uint8_t)lroundf(v * 255.0f);
  }
}

// Three smallest squared distances to the other points (strictly-less
// insertion, as the reference's scan), shared-memory tiles of the cloud.
constexpr int kKnnThreads = 256;
constexpr int kKnnTile = 1024;
__global__ void __launch_bounds__(kKnnThreads) knn3_kernel(const float* __restrict__ xyz, int n,
                                                           float* __restrict__ d3) {
  __shared__ float s_p[kKnnTile][3];
  const int i = blockIdx.x * kKnnThreads + threadIdx.x;
  float px = 0.0f, py = 0.0f, pz = 0.0f;
  if (i < n) {
    px = xyz[3 * i];
    py = xyz[3 * i + 1];
    pz = xyz[3 * i + 2];
  }
  const float inf = 3.40282347e38f;
  float d0 = inf, d1 = inf, d2 = inf;
  for (int t0 = 0; t0 < n; t0 += kKnnTile) {
    __syncthreads();
    for (int k = threadIdx.x; k < kKnnTile * 3; k += kKnnThreads) {
      const int g = t0 * 3 + k;
      (&s_p[0][0])[k] = g < 3 * n ? xyz[g] : 0.0f;
    }
    __syncthreads();
    const int cnt = min(kKnnTile, n - t0);
    for (int k = 0; k < cnt; ++k) {
      if (t0 + k == i) continue;
      const float ax = s_p[k][0] - px, ay = s_p[k][1] - py, az = s_p[k][2] - pz;
      float s = ax * ax;
      s = s + ay * ay;
      s = s + az * az;
      if (s < d0) {
        d2 = d1;
        d1 = d0;
        d0 = s;
      } else if (s < d1) {
        d2 = d1;
        d1 = s;
      } else if (s < d2) {
        d2 = s;
      }
    }
  }
  if (i < n) {
    d3[3 * i] = d0;
    d3[3 * i + 1] = d1;
    d3[3 * i + 2] = d2;
  }
}

}  // namespace
}  // namespace sk

using namespace sk;

extern "C" {

int sk_init_from_points(sk_ctx* ctx, int64_t n, const float* xyz, const float* rgb, int sh_degree, int64_t capacity,
                        sk_scene** out) {
  return guarded(ctx, [&] {
    arg(out && xyz && rgb, "init_from_points: null argument");
    if (n <= 0) throw std::invalid_argument("init_from_points: empty point cloud");
    arg(n < (1ll << 31), "init_from_points: too many points");
    arg(sh_degree >= 0 && sh_degree <= 3, "config: sh_degree must be in 0..3");
    SK_CUDA(cudaSetDevice(ctx->device));
    DevBuf dxyz, dd;
    dxyz.ensure(sizeof(float) * 3 * n);
    dd.ensure(sizeof(float) * 3 * n);
    h2d(ctx, dxyz.ptr, xyz, (size_t)3 * n);
    knn3_kernel<<<(unsigned)((n + kKnnThreads - 1) / kKnnThreads), kKnnThreads, 0, ctx->stream>>>(
        dxyz.as<float>(), (int)n, dd.as<float>());
    note_launch();
    SK_CUDA(cudaGetLastError());
    std::vector<float> d3((size_t)3 * n);
    d2h(ctx, d3.data(), dd.ptr, (size_t)3 * n);
    sync(ctx);
    const int comps = SK_COMP_COUNT(sh_degree);
    std::vector<float> p((size_t)comps * n, 0.0f);
    const float op = logit(0.1f);
    for (int64_t i = 0; i < n; ++i) {
      const float d0 = std::sqrt(d3[3 * i]), d1 = std::sqrt(d3[3 * i + 1]), d2 = std::sqrt(d3[3 * i + 2]);
      float mean = 1.0f;
      if (n == 2) mean = d0;
      else if (n == 3) mean = (d0 + d1) / 2.0f;
      else if (n > 3) mean = (d0 + d1 + d2) / 3.0f;
      mean = std::max(mean, 1e-7f);
      const float ls = std::log(mean);
      for (int d = 0; d < 3; ++d) p[(SK_COMP_MU + d) * n + i] = xyz[3 * i + d];
      p[SK_COMP_ROT * n + i] = 1.0f;
      for (int d = 0; d < 3; ++d) p[(SK_COMP_LOG_SCALE + d) * n + i] = ls;
      p[SK_COMP_OPACITY * n + i] = op;
      for (int c = 0; c < 3; ++c) p[(SK_COMP_SH + c) * n + i] = (rgb[3 * i + c] - 0.5f) / (float)kShC0;
    }
    sk_scene* s = nullptr;
    const int rc = sk_scene_create(ctx, sh_degree, std::max<int64_t>(capacity, n), &s);
    if (rc != SK_OK) throw std::runtime_error(ctx->err);
    std::unique_ptr<sk_scene> holder(s);
    if (sk_scene_upload(ctx, s, p.data(), n) != SK_OK) throw std::runtime_error(ctx->err);
    *out = holder.release();
  });
}

int sk_synthetic_create(sk_ctx* ctx, const sk_synth_spec* spec, sk_scene** gt_out, sk_dataset** data_out,
                        float* init_xyz, float* init_rgb, float* extent_out) {
  return guarded(ctx, [&] {
    arg(spec && data_out, "synthetic: null argument");
    arg(spec->n_views >= 2, "synthetic: n_views must be >= 2");
    arg(spec->n_gaussians >= 1, "synthetic: n_gaussians must be >= 1");
    arg(spec->width > 0 && spec->height > 0, "camera: empty image");
    SK_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = spec->n_gaussians;
    const int deg = 1;  // dataset.hpp:185
    const int comps = SK_COMP_COUNT(deg);
    HostRng rng;
    rng.seed(spec->seed);
    auto uni = [&](double lo, double hi) { return lo + (hi - lo) * rng.uniform(); };
    std::vector<float> p((size_t)comps * n);
    auto at = [&](int comp, int64_t i) -> float& { return p[(size_t)comp * n + i]; };
    for (int64_t i = 0; i < n; ++i) {
      for (int d = 0; d < 3; ++d) at(SK_COMP_MU + d, i) = (float)uni(-0.5, 0.5);
      float q[4];
      for (int d = 0; d < 4; ++d) q[d] = (float)rng.normal();
      float qs = q[0] * q[0];
      for (int d = 1; d < 4; ++d) qs = qs + q[d] * q[d];
      const float qn = std::sqrt(qs);
      for (int d = 0; d < 4; ++d) at(SK_COMP_ROT + d, i) = qn > 1e-6f ? q[d] / qn : (d == 0 ? 1.0f : 0.0f);
      for (int d = 0; d < 3; ++d) at(SK_COMP_LOG_SCALE + d, i) = std::log((float)(uni(0.02, 0.075) * spec->scale_mult));
      at(SK_COMP_OPACITY, i) = logit((float)uni(0.25, 0.95));
      for (int c = 0; c < 3; ++c) at(SK_COMP_SH + c, i) = (float)((uni(0.05, 0.95) - 0.5) / kShC0);
      for (int m = 1; m < (deg + 1) * (deg + 1); ++m)
        for (int c = 0; c < 3; ++c) at(SK_COMP_SH + 3 * m + c, i) = (float)uni(-0.1, 0.1);
    }
    // camera ring (dataset.hpp:207-219)
    std::vector<sk_camera> cams(spec->n_views);
    const float ring_radius = 2.4f, ring_height = 1.0f;
    for (int v = 0; v < spec->n_views; ++v) {
      const float angle = 2.0f * (float)M_PI * (float)v / (float)spec->n_views;
      sk_camera& c = cams[v];
      c.width = spec->width;
      c.height = spec->height;
      c.fx = c.fy = spec->focal > 0 ? (float)spec->focal : 1.1f * (float)spec->height;
      c.cx = (float)(spec->width - 1) / 2.0f;
      c.cy = (float)(spec->height - 1) / 2.0f;
      c.near_plane = 0.2f;
      look_at(v3(ring_radius * std::cos(angle), ring_radius * std::sin(angle), ring_height), c.world_to_cam);
    }
    // GT scene on the device, views rendered and quantised there
    sk_scene* gs = nullptr;
    if (sk_scene_create(ctx, deg, n, &gs) != SK_OK) throw std::runtime_error(ctx->err);
    std::unique_ptr<sk_scene> gt(gs);
    if (sk_scene_upload(ctx, gs, p.data(), n) != SK_OK) throw std::runtime_error(ctx->err);
    auto d = std::make_unique<sk_dataset>();
    d->cams = cams;
    sk_frame f;
    const sk_binning bin{0, 1.0f, (float)(1.0 / 255), 16};
    for (int v = 0; v < spec->n_views; ++v) {
      frame_geometry(&f, cams[v].width, cams[v].height, &bin);
      f.camera = cams[v];
      ensure_projected(&f, gs->n);
      ensure_image(&f);
      launch_preprocess(ctx, gs, cams[v], &f);
      bin_sort(ctx, &f);
      launch_blend_forward(ctx, &f, nullptr, nullptr);
      const int64_t plane = (int64_t)cams[v].width * cams[v].height;
      auto buf = std::make_unique<DevBuf>();
      buf->ensure((size_t)plane * 3);
      quantize_kernel<<<(unsigned)((plane + 255) / 256), 256, 0, ctx->stream>>>(f.image.as<float>(), plane,
                                                                                buf->as<uint8_t>());
      note_launch();
      SK_CUDA(cudaGetLastError());
      d->images.push_back(std::move(buf));
    }
    raise_device_errors(read_error_word(ctx));
    // init points: GT mu + N(0, (0.05 extent_cams)^2), colour from the DC term
    const float noise = 0.05f * scene_extent(cams, {});
    std::vector<V3> pts((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      V3 q3 = v3(at(SK_COMP_MU, i), at(SK_COMP_MU + 1, i), at(SK_COMP_MU + 2, i));
      for (int k = 0; k < 3; ++k) q3[k] = q3[k] + noise * (float)rng.normal();
      pts[i] = q3;
      for (int k = 0; k < 3; ++k) d->init_xyz.push_back(q3[k]);
      for (int c = 0; c < 3; ++c)
        d->init_rgb.push_back(std::min(1.0f, std::max(0.0f, 0.5f + (float)kShC0 * at(SK_COMP_SH + c, i))));
      if (init_xyz)
        for (int k = 0; k < 3; ++k) init_xyz[3 * i + k] = q3[k];
      if (init_rgb)
        for (int c = 0; c < 3; ++c)
          init_rgb[3 * i + c] = std::min(1.0f, std::max(0.0f, 0.5f + (float)kShC0 * at(SK_COMP_SH + c, i)));
    }
    for (int i = 0; i < spec->n_views; ++i) d->ids.push_back(i);
    for (int i = 0; i < spec->n_views; ++i)
      if (i % 8 != 0) d->train.push_back(i);
    if (d->train.empty())
      for (int i = 0; i < spec->n_views; ++i) d->train.push_back(i);
    d->extent = scene_extent(cams, pts);
    if (extent_out) *extent_out = d->extent;
    sync(ctx);
    *data_out = d.release();
    if (gt_out) *gt_out = gt.release();
  });
}

}  // extern "C"
