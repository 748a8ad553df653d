// float64 value path: project + tile-binned blend + training loss in double
// on the device, for finite-difference checks of the float32 analytic
// gradients at the GPU level. The reference templates everything on T and
// runs Trainer<double> behind `--float64` (tools/splatkit_main.cpp:31); its
// gradient tests difference the double loss (tests/acceptance.cpp:163-254,
// tests/test_raster.cpp:230-297). This file is that double forward chain:
//
//   project            camera.hpp:93-123 (+ sh.hpp:80-88, scene.hpp:57-96)
//   bin_aabb/compact   raster.hpp:61-150 (tile membership, evaluated per tile)
//   depth_order        raster.hpp:152-160 (depth, then index)
//   blend_forward      raster.hpp:194-248
//   training_loss      loss.hpp:21-47 with ssim (metrics.hpp:30-89)
//
// It is a checking path, not a training path: one thread per Gaussian, an
// O(n^2) rank sort, one CTA per tile walking the whole depth-sorted list, a
// direct separable SSIM. Sizes are capped (n <= 65536, W*H <= 4 Mpx).
#include <cmath>

#include "abi_util.h"

namespace sk {
namespace {

constexpr double kShC0d = 0.28209479177387814;
constexpr double kShC1d = 0.4886025119029199;
__device__ constexpr double kShC2d[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                         -1.0925484305920792, 0.5462742152960396};
__device__ constexpr double kShC3d[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                         0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                                         -0.5900435899266435};
constexpr int kMaxN = 65536;
constexpr int kThreads = 256;
constexpr int kPixPerThread = 4;  // a 32x32 tile on 256 threads

struct CamD {
  int w, h;
  double fx, fy, cx, cy, near;
  double R[9], t[3], center[3];
};

struct BinD {
  int compact, ts, tiles_x, tiles_y;
  double beta, tau;
};

struct PgD {
  double mx, my, c00, c01, c11, i00, i01, i11, depth, op, a_star;
  double col[3];
  int tx0, tx1, ty0, ty1;  // clamped tile rectangle (empty when tx0 > tx1)
  int visible;
};

struct Kern11 {
  double k[11];
};

__device__ __forceinline__ int floor_to_int_d(double v) {  // oracle floor_to_int
  double f = floor(v);
  if (!(f > -1073741824.0)) f = -1073741824.0;
  if (f > 1073741824.0) f = 1073741824.0;
  return (int)f;
}

__device__ __forceinline__ double max_eig(double a, double b, double d) {  // camera.hpp max_eigenvalue_2x2
  const double mid = (a + d) / 2.0, h = (a - d) / 2.0;
  return mid + sqrt(h * h + b * b);
}

// project() (camera.hpp:93-123) plus the tile rectangle of bin_aabb /
// bin_compact (raster.hpp:61-150) for one Gaussian.
__global__ void fp64_project_kernel(const double* __restrict__ p, int n, int deg, CamD cam, BinD bin,
                                    PgD* __restrict__ out, uint32_t* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  PgD pg{};
  pg.tx0 = 1;
  pg.tx1 = 0;
  auto P = [&](int c) { return p[(int64_t)c * n + i]; };
  const double mu[3] = {P(SK_COMP_MU), P(SK_COMP_MU + 1), P(SK_COMP_MU + 2)};
  double t[3];
  for (int r = 0; r < 3; ++r) {
    double s = 0.0;
    for (int k = 0; k < 3; ++k) s = s + cam.R[3 * r + k] * mu[k];
    t[r] = s + cam.t[r];
  }
  if (t[2] <= cam.near) {
    out[i] = pg;
    return;
  }
  const double iz = 1.0 / t[2], iz2 = iz * iz;
  const double J[2][3] = {{cam.fx * iz, 0.0, -cam.fx * t[0] * iz2}, {0.0, cam.fy * iz, -cam.fy * t[1] * iz2}};
  double m[2][3];
  for (int a = 0; a < 2; ++a)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s = s + J[a][k] * cam.R[3 * k + j];
      m[a][j] = s;
    }
  // covariance_3d (scene.hpp:88-96)
  double q[4] = {P(SK_COMP_ROT), P(SK_COMP_ROT + 1), P(SK_COMP_ROT + 2), P(SK_COMP_ROT + 3)};
  double sc[3];
  bool ok = true;
  for (int k = 0; k < 4; ++k) ok = ok && isfinite(q[k]);
  for (int k = 0; k < 3; ++k) {
    sc[k] = exp(P(SK_COMP_LOG_SCALE + k));
    ok = ok && isfinite(sc[k]);
  }
  if (!ok || !(sc[0] > 0.0 && sc[1] > 0.0 && sc[2] > 0.0)) {
    atomicOr(err, ok ? kErrCovNonPositive : kErrCovNonFinite);
    out[i] = pg;
    return;
  }
  const double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
  if (n2 > 0.0) {
    const double nq = sqrt(n2);
    for (int k = 0; k < 4; ++k) q[k] = q[k] / nq;
  }
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double r[3][3] = {{1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)},
                          {2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)},
                          {2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)}};
  double M[3][3], S[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) M[a][b] = r[a][b] * sc[b];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s = s + M[a][k] * M[b][k];
      S[a][b] = s;
    }
  double mS[2][3], cov[2][2];
  for (int a = 0; a < 2; ++a)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s = s + m[a][k] * S[k][j];
      mS[a][j] = s;
    }
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s = s + mS[a][k] * m[b][k];
      cov[a][b] = s;
    }
  cov[0][0] = cov[0][0] + 0.3;  // kCov2dFloor
  cov[1][1] = cov[1][1] + 0.3;
  pg.mx = cam.fx * t[0] / t[2] + cam.cx;
  pg.my = cam.fy * t[1] / t[2] + cam.cy;
  const double lmax = max_eig(cov[0][0], cov[0][1], cov[1][1]);
  const double guard = 1.3 * (3.0 * sqrt(lmax));  // kCullGuard * radius
  if (pg.mx < -guard || pg.mx > (double)(cam.w - 1) + guard || pg.my < -guard || pg.my > (double)(cam.h - 1) + guard) {
    out[i] = pg;
    return;
  }
  const double det = cov[0][0] * cov[1][1] - cov[0][1] * cov[1][0];
  pg.c00 = cov[0][0];
  pg.c01 = cov[0][1];
  pg.c11 = cov[1][1];
  pg.i00 = cov[1][1] / det;
  pg.i01 = -cov[0][1] / det;
  pg.i11 = cov[0][0] / det;
  pg.depth = t[2];
  // colour: evaluate_sh (sh.hpp:80-88) along (mu - centre) / |mu - centre|
  {
    const double rel[3] = {mu[0] - cam.center[0], mu[1] - cam.center[1], mu[2] - cam.center[2]};
    const double nr = sqrt((rel[0] * rel[0] + rel[1] * rel[1]) + rel[2] * rel[2]);
    const double dx = rel[0] / nr, dy = rel[1] / nr, dz = rel[2] / nr;
    double basis[16];
    basis[0] = kShC0d;
    if (deg >= 1) {
      basis[1] = -kShC1d * dy;
      basis[2] = kShC1d * dz;
      basis[3] = -kShC1d * dx;
    }
    if (deg >= 2) {
      const double xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yz = dy * dz, xz = dx * dz;
      basis[4] = kShC2d[0] * xy;
      basis[5] = kShC2d[1] * yz;
      basis[6] = kShC2d[2] * (2.0 * zz - xx - yy);
      basis[7] = kShC2d[3] * xz;
      basis[8] = kShC2d[4] * (xx - yy);
      if (deg >= 3) {
        basis[9] = kShC3d[0] * dy * (3.0 * xx - yy);
        basis[10] = kShC3d[1] * xy * dz;
        basis[11] = kShC3d[2] * dy * (4.0 * zz - xx - yy);
        basis[12] = kShC3d[3] * dz * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        basis[13] = kShC3d[4] * dx * (4.0 * zz - xx - yy);
        basis[14] = kShC3d[5] * dz * (xx - yy);
        basis[15] = kShC3d[6] * dx * (xx - 3.0 * yy);
      }
    }
    const int nsh = (deg + 1) * (deg + 1);
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int k = 0; k < nsh; ++k) s = s + basis[k] * P(SK_COMP_SH + 3 * k + c);
      s = s + 0.5;
      pg.col[c] = s < 0.0 ? 0.0 : s;
    }
  }
  pg.op = 1.0 / (1.0 + exp(-P(SK_COMP_OPACITY)));
  pg.visible = 1;
  // tile rectangle
  const int ts = bin.ts;
  if (!bin.compact) {  // bin_aabb
    const double rr = 3.0 * sqrt(lmax);
    const int tx0 = floor_to_int_d((pg.mx - rr) / ts), tx1 = floor_to_int_d((pg.mx + rr) / ts);
    const int ty0 = floor_to_int_d((pg.my - rr) / ts), ty1 = floor_to_int_d((pg.my + rr) / ts);
    if (!(tx1 < 0 || ty1 < 0 || tx0 >= bin.tiles_x || ty0 >= bin.tiles_y)) {
      pg.tx0 = max(tx0, 0);
      pg.tx1 = min(tx1, bin.tiles_x - 1);
      pg.ty0 = max(ty0, 0);
      pg.ty1 = min(ty1, bin.tiles_y - 1);
    }
  } else if (pg.op > bin.tau) {  // bin_compact
    if (!(det > 0.0 && cov[0][0] > 0.0)) {
      atomicOr(err, kErrCompactNotPD);
    } else {
      const double th = bin.beta * (2.0 * log(pg.op / bin.tau));
      pg.a_star = (9.0 < th) ? 9.0 : th;
      const double ex = sqrt(pg.a_star * cov[0][0]), ey = sqrt(pg.a_star * cov[1][1]);
      pg.tx0 = max(0, floor_to_int_d((pg.mx - ex) / ts));
      pg.tx1 = min(bin.tiles_x - 1, floor_to_int_d((pg.mx + ex) / ts));
      pg.ty0 = max(0, floor_to_int_d((pg.my - ey) / ts));
      pg.ty1 = min(bin.tiles_y - 1, floor_to_int_d((pg.my + ey) / ts));
    }
  }
  out[i] = pg;
}

// depth_order (raster.hpp:152-160): rank by (depth, index) among the visible.
__global__ void fp64_rank_kernel(const PgD* __restrict__ pg, int n, int* __restrict__ order) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !pg[i].visible) return;
  const double d = pg[i].depth;
  int rank = 0;
  for (int j = 0; j < n; ++j) {
    if (!pg[j].visible) continue;
    const double dj = pg[j].depth;
    rank += (dj < d || (dj == d && j < i)) ? 1 : 0;
  }
  order[rank] = i;
}

__device__ __forceinline__ double clamp_d(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
__device__ __forceinline__ double min_d(double a, double b) { return (b < a) ? b : a; }

// min_mahalanobis_on_rect (raster.hpp:96-112)
__device__ double min_maha_rect(const PgD& g, double x0, double x1, double y0, double y1) {
  if (g.mx >= x0 && g.mx <= x1 && g.my >= y0 && g.my <= y1) return 0.0;
  const double a = g.i00, b = g.i01, c = g.i11;
  auto qf = [&](double dx, double dy) { return a * dx * dx + 2.0 * b * dx * dy + c * dy * dy; };
  double best = 1.7976931348623157e308;
  const double xs[2] = {x0, x1}, ys[2] = {y0, y1};
  for (int k = 0; k < 2; ++k) {
    const double dx = xs[k] - g.mx;
    const double yy = clamp_d(g.my - b * dx / c, y0, y1);
    best = min_d(best, qf(dx, yy - g.my));
  }
  for (int k = 0; k < 2; ++k) {
    const double dy = ys[k] - g.my;
    const double xx = clamp_d(g.mx - b * dy / a, x0, x1);
    best = min_d(best, qf(xx - g.mx, dy));
  }
  return best;
}

// blend_forward (raster.hpp:194-248): one CTA per tile walks the depth-sorted
// visible list in chunks; membership in the tile's list is re-derived per
// chunk from the tile rectangle (and the compact box test), so every pixel
// sees exactly its tile's list in the reference's order.
__global__ void __launch_bounds__(kThreads) fp64_blend_kernel(const PgD* __restrict__ pg, const int* __restrict__ order,
                                                              int nvis, BinD bin, int W, int H,
                                                              double* __restrict__ image) {
  __shared__ PgD s_pg[kThreads];
  __shared__ int s_member[kThreads];
  const int tx = blockIdx.x, ty = blockIdx.y, ts = bin.ts;
  const int npx = ts * ts;
  double tr[kPixPerThread], c[kPixPerThread][3];
  bool done[kPixPerThread];
  for (int k = 0; k < kPixPerThread; ++k) {
    tr[k] = 1.0;
    c[k][0] = c[k][1] = c[k][2] = 0.0;
    const int l = threadIdx.x + k * kThreads;
    const int px = tx * ts + l % ts, py = ty * ts + l / ts;
    done[k] = l >= npx || px >= W || py >= H;
  }
  const double x0 = (double)(tx * ts), y0 = (double)(ty * ts);
  const double x1 = (double)(min((tx + 1) * ts, W) - 1), y1 = (double)(min((ty + 1) * ts, H) - 1);
  for (int base = 0; base < nvis; base += kThreads) {
    __syncthreads();
    const int j = base + threadIdx.x;
    int mem = 0;
    if (j < nvis) {
      const PgD g = pg[order[j]];
      mem = tx >= g.tx0 && tx <= g.tx1 && ty >= g.ty0 && ty <= g.ty1;
      if (mem && bin.compact) mem = min_maha_rect(g, x0, x1, y0, y1) <= g.a_star;
      s_pg[threadIdx.x] = g;
    }
    s_member[threadIdx.x] = mem;
    __syncthreads();
    const int cnt = min(kThreads, nvis - base);
    for (int k = 0; k < kPixPerThread; ++k) {
      if (done[k]) continue;
      const int l = threadIdx.x + k * kThreads;
      const double px = (double)(tx * ts + l % ts), py = (double)(ty * ts + l / ts);
      for (int e = 0; e < cnt; ++e) {
        if (!s_member[e]) continue;
        const PgD& g = s_pg[e];
        const double dx = px - g.mx, dy = py - g.my;
        const double q = g.i00 * dx * dx + 2.0 * g.i01 * dx * dy + g.i11 * dy * dy;
        if (q < 0.0) continue;
        const double alpha = min_d(0.99, g.op * exp(-0.5 * q));
        if (alpha < 1.0 / 255.0) continue;
        const double w = tr[k] * alpha;
        for (int ch = 0; ch < 3; ++ch) c[k][ch] = c[k][ch] + w * g.col[ch];
        tr[k] = tr[k] * (1.0 - alpha);
        if (tr[k] < 1e-4) {
          done[k] = true;
          break;
        }
      }
    }
  }
  for (int k = 0; k < kPixPerThread; ++k) {
    const int l = threadIdx.x + k * kThreads;
    const int px = tx * ts + l % ts, py = ty * ts + l / ts;
    if (l >= npx || px >= W || py >= H) continue;
    for (int ch = 0; ch < 3; ++ch) image[((int64_t)py * W + px) * 3 + ch] = c[k][ch];
  }
}

// gauss_filter (metrics.hpp:30-52), horizontal pass of the five SSIM inputs
// x, y, x*x, y*y, x*y of channel ch (zero padding, taps ascending).
__global__ void fp64_ssim_h_kernel(const double* __restrict__ a, const double* __restrict__ b, int W, int H, int ch,
                                   Kern11 kern, double* __restrict__ tmp) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)W * H) return;
  const int x = (int)(idx % W), y = (int)(idx / W);
  const int o0 = max(-5, -x), o1 = min(5, W - 1 - x);
  double s[5] = {0, 0, 0, 0, 0};
  for (int o = o0; o <= o1; ++o) {
    const double k = kern.k[o + 5];
    const double xv = a[((int64_t)y * W + x + o) * 3 + ch], yv = b[((int64_t)y * W + x + o) * 3 + ch];
    s[0] += k * xv;
    s[1] += k * yv;
    s[2] += k * (xv * xv);
    s[3] += k * (yv * yv);
    s[4] += k * (xv * yv);
  }
  for (int m = 0; m < 5; ++m) tmp[(int64_t)m * W * H + idx] = s[m];
}

// vertical pass + ssim_channel's per-pixel S (metrics.hpp:61-78); also the
// L1 term of training_loss (loss.hpp:27-33) for this channel.
__global__ void fp64_ssim_v_kernel(const double* __restrict__ tmp, const double* __restrict__ a,
                                   const double* __restrict__ b, int W, int H, int ch, Kern11 kern,
                                   double* __restrict__ s_map, double* __restrict__ l1_map) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)W * H) return;
  const int x = (int)(idx % W), y = (int)(idx / W);
  const int o0 = max(-5, -y), o1 = min(5, H - 1 - y);
  double m[5];
  for (int q = 0; q < 5; ++q) {
    double s = 0.0;
    for (int o = o0; o <= o1; ++o) s += kern.k[o + 5] * tmp[(int64_t)q * W * H + (int64_t)(y + o) * W + x];
    m[q] = s;
  }
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  const double mx = m[0], my = m[1];
  const double sxx = m[2] - mx * mx, syy = m[3] - my * my, sxy = m[4] - mx * my;
  const double a1 = 2.0 * mx * my + C1, a2 = 2.0 * sxy + C2;
  const double b1 = mx * mx + my * my + C1, b2 = sxx + syy + C2;
  s_map[(int64_t)ch * W * H + idx] = (a1 * a2) / (b1 * b2);
  l1_map[(int64_t)ch * W * H + idx] = fabs(a[idx * 3 + ch] - b[idx * 3 + ch]);
}

// Deterministic sum of `count` doubles per segment (one CTA per segment,
// fixed striding and a fixed tree).
__global__ void fp64_sum_kernel(const double* __restrict__ v, int64_t count, double* __restrict__ out) {
  __shared__ double sh[kThreads];
  const double* seg = v + (int64_t)blockIdx.x * count;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += kThreads) s += seg[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

}  // namespace
}  // namespace sk

using namespace sk;

extern "C" int sk_fp64_render_loss(sk_ctx* ctx, const double* params_host, int64_t n, int sh_degree,
                                   const sk_camera* cam, const sk_binning* binning, const double* gt_hwc,
                                   double lambda, double* image_hwc, double* loss3) {
  return guarded(ctx, [&] {
    arg(ctx && cam && (n == 0 || params_host), "fp64_render_loss: null argument");
    arg(n >= 0 && n <= kMaxN, "fp64_render_loss: n must be in [0, 65536] (a checking path)");
    arg(sh_degree >= 0 && sh_degree <= 3, "fp64_render_loss: sh_degree must be 0..3");
    const int W = cam->width, H = cam->height;
    arg(W > 0 && H > 0 && (int64_t)W * H <= (4 << 20), "fp64_render_loss: image must be 1..4 Mpx");
    const int ts = binning ? binning->tile_size : 16;
    arg(ts == 8 || ts == 16 || ts == 32, "fp64_render_loss: tile_size must be 8, 16 or 32");
    SK_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    // camera in double (the oracle's to_camera<double>): centre = -(R^T t),
    // evaluated (R_0i t0 + R_1i t1) + R_2i t2
    CamD cd{};
    cd.w = W;
    cd.h = H;
    cd.fx = cam->fx;
    cd.fy = cam->fy;
    cd.cx = cam->cx;
    cd.cy = cam->cy;
    cd.near = cam->near_plane;
    for (int r = 0; r < 3; ++r) {
      for (int k = 0; k < 3; ++k) cd.R[3 * r + k] = cam->world_to_cam[4 * r + k];
      cd.t[r] = cam->world_to_cam[4 * r + 3];
    }
    for (int i = 0; i < 3; ++i) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s = s + cd.R[3 * k + i] * cd.t[k];
      cd.center[i] = -s;
    }
    BinD bd{};
    bd.compact = binning && binning->mode == 1;
    bd.beta = binning ? binning->beta : 1.0;
    bd.tau = binning ? binning->tau_alpha : 1.0 / 255;
    bd.ts = ts;
    bd.tiles_x = (W + ts - 1) / ts;
    bd.tiles_y = (H + ts - 1) / ts;
    const int comps = SK_COMP_COUNT(sh_degree);
    const int64_t px = (int64_t)W * H;
    DevBuf d_params, d_pg, d_order, d_err, d_img, d_gt, d_tmp, d_maps, d_sums;
    ensure<uint32_t>(d_err, 1);
    ensure<double>(d_img, 3 * px);
    SK_CUDA(cudaMemsetAsync(d_err.ptr, 0, sizeof(uint32_t), st));
    SK_CUDA(cudaMemsetAsync(d_img.ptr, 0, sizeof(double) * 3 * px, st));
    int nvis = 0;
    if (n > 0) {
      ensure<double>(d_params, (size_t)comps * n);
      d_pg.ensure(sizeof(PgD) * n);
      ensure<int>(d_order, (size_t)n);
      h2d(ctx, d_params.ptr, params_host, (size_t)comps * n);
      const unsigned g = (unsigned)((n + kThreads - 1) / kThreads);
      fp64_project_kernel<<<g, kThreads, 0, st>>>(d_params.as<double>(), (int)n, sh_degree, cd, bd,
                                                  static_cast<PgD*>(d_pg.ptr), d_err.as<uint32_t>());
      note_launch();
      SK_CUDA(cudaGetLastError());
      uint32_t e = 0;
      d2h(ctx, &e, d_err.ptr, 1);
      sync(ctx);
      raise_device_errors(e);
      fp64_rank_kernel<<<g, kThreads, 0, st>>>(static_cast<const PgD*>(d_pg.ptr), (int)n, d_order.as<int>());
      note_launch();
      SK_CUDA(cudaGetLastError());
      // the visible count: every visible Gaussian holds one rank slot
      std::vector<PgD> host(n);
      d2h(ctx, host.data(), d_pg.ptr, (size_t)n);
      sync(ctx);
      for (const PgD& q : host) nvis += q.visible;
      fp64_blend_kernel<<<dim3(bd.tiles_x, bd.tiles_y), kThreads, 0, st>>>(
          static_cast<const PgD*>(d_pg.ptr), d_order.as<int>(), nvis, bd, W, H, d_img.as<double>());
      note_launch();
      SK_CUDA(cudaGetLastError());
    }
    if (image_hwc) d2h(ctx, image_hwc, d_img.ptr, (size_t)(3 * px));
    if (gt_hwc && loss3) {
      Kern11 kern;
      double ksum = 0.0;
      for (int i = 0; i < 11; ++i) {
        const double d = (double)(i - 5);
        kern.k[i] = std::exp(-(d * d) / (2.0 * 1.5 * 1.5));
        ksum += kern.k[i];
      }
      for (double& k : kern.k) k /= ksum;
      ensure<double>(d_gt, 3 * px);
      ensure<double>(d_tmp, 5 * px);
      ensure<double>(d_maps, 6 * px);  // [3] SSIM maps, [3] |diff| maps
      ensure<double>(d_sums, 6);
      h2d(ctx, d_gt.ptr, gt_hwc, (size_t)(3 * px));
      const unsigned g = (unsigned)((px + kThreads - 1) / kThreads);
      for (int ch = 0; ch < 3; ++ch) {
        fp64_ssim_h_kernel<<<g, kThreads, 0, st>>>(d_img.as<double>(), d_gt.as<double>(), W, H, ch, kern,
                                                   d_tmp.as<double>());
        fp64_ssim_v_kernel<<<g, kThreads, 0, st>>>(d_tmp.as<double>(), d_img.as<double>(), d_gt.as<double>(), W, H,
                                                   ch, kern, d_maps.as<double>(), d_maps.as<double>() + 3 * px);
        note_launch();
        note_launch();
      }
      fp64_sum_kernel<<<6, kThreads, 0, st>>>(d_maps.as<double>(), px, d_sums.as<double>());
      note_launch();
      SK_CUDA(cudaGetLastError());
      double sums[6];
      d2h(ctx, sums, d_sums.ptr, 6);
      sync(ctx);
      const double npx = (double)px;
      const double ssim = ((sums[0] / npx + sums[1] / npx) + sums[2] / npx) / 3.0;
      const double l1 = ((sums[3] + sums[4]) + sums[5]) * (1.0 / (3.0 * npx));
      loss3[0] = (1.0 - lambda) * l1 + lambda * (1.0 - ssim);
      loss3[1] = l1;
      loss3[2] = ssim;
    }
    sync(ctx);
  });
}
