// K1 preprocess and K3 duplicate-with-keys.
//
// K1 follows project() (reference camera.hpp:93-123) with covariance_3d
// (scene.hpp:88-96), quat_to_rotation (scene.hpp:57-65), evaluate_sh
// (sh.hpp:28-51, 80-88) and the tile count of bin_aabb / bin_compact
// (raster.hpp:61-141), in the oracle's fixed operation order. This file is
// compiled with -fmad=false and uses IEEE division/sqrt plus the shared
// deterministic exp/log (detmath.h), so every projected field and every tile
// rectangle is bit-identical to the CPU oracle.
//
// Layout: one thread per Gaussian; all parameter reads are planar
// ([component][capacity]) and therefore fully coalesced; outputs are float2 /
// float4 SoA records.
#include "state.h"

namespace sk {
namespace {

__device__ __forceinline__ int floor_to_int(float v) {
  float f = floorf(v);
  if (!(f > -1073741824.0f)) f = -1073741824.0f;
  if (f > 1073741824.0f) f = 1073741824.0f;
  return (int)f;
}

__device__ __forceinline__ float min_ref(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ float clamp_ref(float v, float lo, float hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// raster.hpp:89-106
__device__ __forceinline__ float min_mahalanobis_on_rect(float a, float b, float c, float mx, float my, float x0,
                                                         float x1, float y0, float y1) {
  if (mx >= x0 && mx <= x1 && my >= y0 && my <= y1) return 0.0f;
  float best = 3.40282347e38f;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float x = e == 0 ? x0 : x1;
    const float dx = x - mx;
    const float y = clamp_ref(my - b * dx / c, y0, y1);
    const float dy = y - my;
    best = min_ref(best, a * dx * dx + 2.0f * b * dx * dy + c * dy * dy);
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float y = e == 0 ? y0 : y1;
    const float dy = y - my;
    const float x = clamp_ref(mx - b * dy / a, x0, x1);
    const float dx = x - mx;
    best = min_ref(best, a * dx * dx + 2.0f * b * dx * dy + c * dy * dy);
  }
  return best;
}

struct BinOut {
  int4 rect;
  int count;
  float a_star;
};

// Tile rectangle + count for one footprint (bin_aabb raster.hpp:61-74,
// bin_compact :111-141). Returns false if the compact-box PD check fails.
__device__ __forceinline__ bool bin_footprint(float mx, float my, float c00, float c01, float c10, float c11,
                                              float inv00, float inv01, float inv11, float opacity, int mode,
                                              float beta, float tau_alpha, int ts, int tiles_x, int tiles_y, int W,
                                              int H, BinOut& out) {
  out.count = 0;
  out.a_star = 0.0f;
  out.rect = make_int4(0, 0, -1, -1);
  const float fts = (float)ts;
  if (mode == 0) {
    const float mid = (c00 + c11) / 2.0f;
    const float h = (c00 - c11) / 2.0f;
    const float lam = mid + sqrtf(h * h + c01 * c01);
    const float rr = kBinSigma * sqrtf(lam);
    const int tx0 = floor_to_int((mx - rr) / fts);
    const int tx1 = floor_to_int((mx + rr) / fts);
    const int ty0 = floor_to_int((my - rr) / fts);
    const int ty1 = floor_to_int((my + rr) / fts);
    if (tx1 < 0 || ty1 < 0 || tx0 >= tiles_x || ty0 >= tiles_y) return true;
    const int x0 = max(tx0, 0), x1 = min(tx1, tiles_x - 1);
    const int y0 = max(ty0, 0), y1 = min(ty1, tiles_y - 1);
    out.rect = make_int4(x0, y0, x1, y1);
    out.count = (x1 - x0 + 1) * (y1 - y0 + 1);
    return true;
  }
  if (opacity <= tau_alpha) return true;
  const float det = c00 * c11 - c10 * c01;
  if (!(det > 0.0f && c00 > 0.0f)) return false;
  const float a_star = min_ref(beta * (2.0f * det_logf(opacity / tau_alpha)), kBinMahaMax);
  const float ext_x = sqrtf(a_star * c00);
  const float ext_y = sqrtf(a_star * c11);
  const int x0 = max(0, floor_to_int((mx - ext_x) / fts));
  const int x1 = min(tiles_x - 1, floor_to_int((mx + ext_x) / fts));
  const int y0 = max(0, floor_to_int((my - ext_y) / fts));
  const int y1 = min(tiles_y - 1, floor_to_int((my + ext_y) / fts));
  out.a_star = a_star;
  out.rect = make_int4(x0, y0, x1, y1);
  int cnt = 0;
  for (int ty = y0; ty <= y1; ++ty) {
    const float ry0 = (float)(ty * ts);
    const float ry1 = (float)(min((ty + 1) * ts, H) - 1);
    for (int tx = x0; tx <= x1; ++tx) {
      const float rx0 = (float)(tx * ts);
      const float rx1 = (float)(min((tx + 1) * ts, W) - 1);
      if (min_mahalanobis_on_rect(inv00, inv01, inv11, mx, my, rx0, rx1, ry0, ry1) <= a_star) ++cnt;
    }
  }
  out.count = cnt;
  return true;
}

// Orderable bits of a float (ascending float order == ascending uint order).
__device__ __forceinline__ uint32_t depth_key_bits(float d) {
  const uint32_t u = __float_as_uint(d);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct BinParams {
  int mode;
  float beta, tau_alpha;
  int ts, tiles_x, tiles_y, W, H;
};


template <int DEG>
__global__ void __launch_bounds__(256) preprocess_kernel(const float* __restrict__ p, int64_t stride, int64_t n,
                                                         CamParams cam, BinParams bp, float2* __restrict__ mean2d,
                                                         float4* __restrict__ conic_op, float4* __restrict__ rgbd,
                                                         float4* __restrict__ cov_out, float4* __restrict__ conic4,
                                                         float* __restrict__ radius_out, int* __restrict__ tiles_out,
                                                         int4* __restrict__ rect_out, float* __restrict__ astar_out,
                                                         uint32_t* __restrict__ key_out, uint32_t* __restrict__ val_out,
                                                         uint32_t* __restrict__ err) {
  __shared__ float s_exp2[64];
  stage_exp2_table(s_exp2);
  const SmemPinnedTable tab(s_exp2);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  val_out[i] = (uint32_t)i;  // the depth sort's payload (projected index)
  auto culled = [&]() {
    radius_out[i] = 0.0f;
    tiles_out[i] = 0;
    key_out[i] = 0xffffffffu;
  };
  const float mu0 = p[0 * stride + i], mu1 = p[1 * stride + i], mu2 = p[2 * stride + i];
  // rotation / scale / opacity loads issued with mu's, before the near test,
  // so their latency overlaps the projection arithmetic
  const float pf_q0 = p[3 * stride + i], pf_q1 = p[4 * stride + i], pf_q2 = p[5 * stride + i],
              pf_q3 = p[6 * stride + i], pf_s0 = p[7 * stride + i], pf_s1 = p[8 * stride + i],
              pf_s2 = p[9 * stride + i], pf_op = p[SK_COMP_OPACITY * stride + i];
#define SK_P(c, v) (v)
  const float* R = cam.r;
  // t = R mu + t  (Mat * Vec: ((R_k0 mu0 + R_k1 mu1) + R_k2 mu2), then + t_k)
  const float t0 = ((R[0] * mu0 + R[1] * mu1) + R[2] * mu2) + cam.t[0];
  const float t1 = ((R[3] * mu0 + R[4] * mu1) + R[5] * mu2) + cam.t[1];
  const float t2 = ((R[6] * mu0 + R[7] * mu1) + R[8] * mu2) + cam.t[2];
  if (t2 <= cam.near_plane) {
    culled();
    return;
  }
  // projection_jacobian (camera.hpp:80-87)
  const float iz = 1.0f / t2;
  const float iz2 = iz * iz;
  const float J00 = cam.fx * iz, J01 = 0.0f, J02 = -cam.fx * t0 * iz2;
  const float J10 = 0.0f, J11 = cam.fy * iz, J12 = -cam.fy * t1 * iz2;
  float m[2][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    m[0][j] = (J00 * R[0 * 3 + j] + J01 * R[1 * 3 + j]) + J02 * R[2 * 3 + j];
    m[1][j] = (J10 * R[0 * 3 + j] + J11 * R[1 * 3 + j]) + J12 * R[2 * 3 + j];
  }
  // covariance_3d (scene.hpp:88-96)
  const float qw_in = SK_P(3, pf_q0), qx_in = SK_P(4, pf_q1), qy_in = SK_P(5, pf_q2), qz_in = SK_P(6, pf_q3);
  constexpr int NSH = (DEG + 1) * (DEG + 1);
#define SK_SH(k) p[(SK_COMP_SH + (k)) * stride + i]
  const float s0 = det_expf(SK_P(7, pf_s0), tab), s1 = det_expf(SK_P(8, pf_s1), tab),
              s2 = det_expf(SK_P(9, pf_s2), tab);
  if (!(isfinite(qw_in) && isfinite(qx_in) && isfinite(qy_in) && isfinite(qz_in) && isfinite(s0) && isfinite(s1) &&
        isfinite(s2))) {
    atomicOr(err, kErrCovNonFinite);
    culled();
    return;
  }
  if (s0 <= 0.0f || s1 <= 0.0f || s2 <= 0.0f) {
    atomicOr(err, kErrCovNonPositive);
    culled();
    return;
  }
  float qw = qw_in, qx = qx_in, qy = qy_in, qz = qz_in;
  const float n2 = ((qw * qw + qx * qx) + qy * qy) + qz * qz;
  if (n2 > 0.0f) {
    const float nq = sqrtf(n2);
    qw = qw / nq;
    qx = qx / nq;
    qy = qy / nq;
    qz = qz / nq;
  }
  float r[3][3];
  r[0][0] = 1.0f - 2.0f * (qy * qy + qz * qz);
  r[0][1] = 2.0f * (qx * qy - qw * qz);
  r[0][2] = 2.0f * (qx * qz + qw * qy);
  r[1][0] = 2.0f * (qx * qy + qw * qz);
  r[1][1] = 1.0f - 2.0f * (qx * qx + qz * qz);
  r[1][2] = 2.0f * (qy * qz - qw * qx);
  r[2][0] = 2.0f * (qx * qz - qw * qy);
  r[2][1] = 2.0f * (qy * qz + qw * qx);
  r[2][2] = 1.0f - 2.0f * (qx * qx + qy * qy);
  float M[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    M[a][0] = r[a][0] * s0;
    M[a][1] = r[a][1] * s1;
    M[a][2] = r[a][2] * s2;
  }
  float S[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) S[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];
  // cov2d = (m Sigma) m^T + floor
  float A[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) A[a][b] = (m[a][0] * S[0][b] + m[a][1] * S[1][b]) + m[a][2] * S[2][b];
  float c[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) c[a][b] = (A[a][0] * m[b][0] + A[a][1] * m[b][1]) + A[a][2] * m[b][2];
  c[0][0] = c[0][0] + kCov2dFloor;
  c[1][1] = c[1][1] + kCov2dFloor;
  const float mx = cam.fx * t0 / t2 + cam.cx;
  const float my = cam.fy * t1 / t2 + cam.cy;
  // max_eigenvalue_2x2 (camera.hpp:71-75)
  const float mid = (c[0][0] + c[1][1]) / 2.0f;
  const float hh = (c[0][0] - c[1][1]) / 2.0f;
  const float radius = 3.0f * sqrtf(mid + sqrtf(hh * hh + c[0][1] * c[0][1]));
  const float guard = kCullGuard * radius;
  if (mx < -guard || mx > (float)(cam.width - 1) + guard || my < -guard || my > (float)(cam.height - 1) + guard) {
    culled();
    return;
  }
  const float det = c[0][0] * c[1][1] - c[0][1] * c[1][0];
  const float inv00 = c[1][1] / det, inv01 = -c[0][1] / det, inv10 = -c[1][0] / det, inv11 = c[0][0] / det;
  // colour: evaluate_sh along (mu - C) / |mu - C|
  const float rel0 = mu0 - cam.center[0], rel1 = mu1 - cam.center[1], rel2 = mu2 - cam.center[2];
  const float dn = sqrtf((rel0 * rel0 + rel1 * rel1) + rel2 * rel2);
  const float x = rel0 / dn, y = rel1 / dn, z = rel2 / dn;
  float basis[NSH];
  basis[0] = (float)0.28209479177387814;
  if (DEG >= 1) {
    basis[1] = (float)(-0.4886025119029199) * y;
    basis[2] = (float)(0.4886025119029199) * z;
    basis[3] = (float)(-0.4886025119029199) * x;
  }
  if (DEG >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    const float xy = x * y, yz = y * z, xz = x * z;
    basis[4] = (float)1.0925484305920792 * xy;
    basis[5] = (float)(-1.0925484305920792) * yz;
    basis[6] = (float)0.31539156525252005 * (2.0f * zz - xx - yy);
    basis[7] = (float)(-1.0925484305920792) * xz;
    basis[8] = (float)0.5462742152960396 * (xx - yy);
    if (DEG >= 3) {
      basis[9] = (float)(-0.5900435899266435) * y * (3.0f * xx - yy);
      basis[10] = (float)2.890611442640554 * xy * z;
      basis[11] = (float)(-0.4570457994644658) * y * (4.0f * zz - xx - yy);
      basis[12] = (float)0.3731763325901154 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
      basis[13] = (float)(-0.4570457994644658) * x * (4.0f * zz - xx - yy);
      basis[14] = (float)1.445305721320277 * z * (xx - yy);
      basis[15] = (float)(-0.5900435899266435) * x * (xx - 3.0f * yy);
    }
  }
  float rgb[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < NSH; ++k)
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) rgb[ch] = rgb[ch] + basis[k] * SK_SH(3 * k + ch);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    rgb[ch] = rgb[ch] + 0.5f;
    rgb[ch] = (rgb[ch] < 0.0f) ? 0.0f : rgb[ch];
  }
  const float opacity = det_sigmoidf(SK_P(SK_COMP_OPACITY, pf_op), tab);
#undef SK_P
#undef SK_SH

  BinOut bo;
  if (!bin_footprint(mx, my, c[0][0], c[0][1], c[1][0], c[1][1], inv00, inv01, inv11, opacity, bp.mode, bp.beta,
                     bp.tau_alpha, bp.ts, bp.tiles_x, bp.tiles_y, bp.W, bp.H, bo)) {
    atomicOr(err, kErrCompactNotPD);
  }
  mean2d[i] = make_float2(mx, my);
  conic_op[i] = make_float4(inv00, inv01, inv11, opacity);
  rgbd[i] = make_float4(rgb[0], rgb[1], rgb[2], t2);
  cov_out[i] = make_float4(c[0][0], c[0][1], c[1][0], c[1][1]);
  conic4[i] = make_float4(inv00, inv01, inv10, inv11);
  radius_out[i] = radius;
  tiles_out[i] = bo.count;
  rect_out[i] = bo.rect;
  astar_out[i] = bo.a_star;
  key_out[i] = bo.count > 0 ? depth_key_bits(t2) : 0xffffffffu;
}

// Binning for injected projected Gaussians (sk_frame_set_projected).
__global__ void inject_bin_kernel(int64_t n, BinParams bp, const float2* __restrict__ mean2d,
                                  const float4* __restrict__ conic_op, const float4* __restrict__ rgbd,
                                  const float4* __restrict__ cov, float* __restrict__ radius_out,
                                  int* __restrict__ tiles_out, int4* __restrict__ rect_out,
                                  float* __restrict__ astar_out, uint32_t* __restrict__ key_out,
                                  uint32_t* __restrict__ val_out, uint32_t* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  val_out[i] = (uint32_t)i;
  const float2 mu = mean2d[i];
  const float4 co = conic_op[i];
  const float4 cv = cov[i];
  const float mid = (cv.x + cv.w) / 2.0f;
  const float hh = (cv.x - cv.w) / 2.0f;
  radius_out[i] = 3.0f * sqrtf(mid + sqrtf(hh * hh + cv.y * cv.y));
  BinOut bo;
  if (!bin_footprint(mu.x, mu.y, cv.x, cv.y, cv.z, cv.w, co.x, co.y, co.z, co.w, bp.mode, bp.beta, bp.tau_alpha,
                     bp.ts, bp.tiles_x, bp.tiles_y, bp.W, bp.H, bo))
    atomicOr(err, kErrCompactNotPD);
  tiles_out[i] = bo.count;
  rect_out[i] = bo.rect;
  astar_out[i] = bo.a_star;
  key_out[i] = bo.count > 0 ? depth_key_bits(rgbd[i].w) : 0xffffffffu;
}

// K3: one thread per depth-sorted position; writes the Gaussian's tile ids
// (row-major within its rectangle, as bin_aabb / bin_compact enumerate them)
// at its scanned offset. Pair order = (depth, index) order, which the
// stable tile sort then preserves inside each tile.
// K3: pairs (tile, Gaussian) in (depth, index) order, plus the digit
// histograms of the following tile-id radix sort (hist[p][256], p < passes).
// A warp takes 32 consecutive depth-ordered slots; their pair runs are
// adjacent in the output, so in AABB mode the warp writes the whole range
// cooperatively (lane e writes pair e: owner found by a shuffle binary search
// over the lanes' offsets, tile from the owner's rectangle) and every store
// is coalesced. Compact mode keeps one thread per Gaussian (its tiles are a
// filtered subset of the rectangle).
constexpr int kDupThreads = 256;
__global__ void __launch_bounds__(kDupThreads) duplicate_kernel(int64_t n, BinParams bp,
                                                                const uint32_t* __restrict__ order,
                                                                const int32_t* __restrict__ offsets,
                                                                const int* __restrict__ tiles,
                                                                const int4* __restrict__ rect,
                                                                const float2* __restrict__ mean2d,
                                                                const float4* __restrict__ conic_op,
                                                                const float* __restrict__ a_star,
                                                                uint32_t* __restrict__ pair_tile,
                                                                uint32_t* __restrict__ pair_val, int passes,
                                                                int width, uint32_t* __restrict__ hist,
                                                                int64_t cap) {
  __shared__ uint32_t s_hist[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += kDupThreads) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  auto count_digits = [&](uint32_t t) {
    for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(t >> (width * p)) & ((1u << width) - 1u)], 1u);
  };
  const int64_t warps = (int64_t)gridDim.x * (kDupThreads / 32);
  for (int64_t wi = (int64_t)blockIdx.x * (kDupThreads / 32) + (threadIdx.x >> 5); wi * 32 < n; wi += warps) {
    const int64_t s = wi * 32 + lane;
    const bool valid = s < n;
    const uint32_t g = valid ? order[s] : 0u;
    const int cnt = valid ? tiles[g] : 0;
    const int off = valid ? offsets[s] : 0x7fffffff;
    if (bp.mode != 0) {
      if (cnt == 0) continue;
      int64_t o = off;
      const float2 mu = mean2d[g];
      const float4 co = conic_op[g];
      const float as = a_star[g];
      const int4 rc = rect[g];
      for (int ty = rc.y; ty <= rc.w; ++ty) {
        const float ry0 = (float)(ty * bp.ts);
        const float ry1 = (float)(min((ty + 1) * bp.ts, bp.H) - 1);
        for (int tx = rc.x; tx <= rc.z; ++tx) {
          const float rx0 = (float)(tx * bp.ts);
          const float rx1 = (float)(min((tx + 1) * bp.ts, bp.W) - 1);
          if (min_mahalanobis_on_rect(co.x, co.y, co.z, mu.x, mu.y, rx0, rx1, ry0, ry1) <= as) {
            const uint32_t t = (uint32_t)(ty * bp.tiles_x + tx);
            if (o < cap) {
              pair_tile[o] = t;
              pair_val[o] = g;
            }
            count_digits(t);
            ++o;
          }
        }
      }
      continue;
    }
    const int4 rc = cnt ? rect[g] : make_int4(0, 0, 0, 0);
    const int w = rc.z - rc.x + 1;
    const float inv_w = 1.0f / (float)w;  // row split of the pair index: estimate + exact fix-up
    // the warp's pairs occupy [first, last) contiguously
    const int first = __reduce_min_sync(0xffffffffu, valid ? off : 0x7fffffff);
    const int last = __reduce_max_sync(0xffffffffu, valid ? off + cnt : 0);
    const int total = last - first;
    for (int e0 = 0; e0 < total; e0 += 32) {
      const int pos = first + e0 + lane;
      // owner = the highest lane whose offset is <= pos (zero-count lanes
      // share the next lane's offset, so they are never chosen for a pair)
      int L = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int o = __shfl_sync(0xffffffffu, off, L + step);
        if (o <= pos) L += step;
      }
      const int k = pos - __shfl_sync(0xffffffffu, off, L);
      const int ox = __shfl_sync(0xffffffffu, rc.x, L);
      const int oy = __shfl_sync(0xffffffffu, rc.y, L);
      const int ow = __shfl_sync(0xffffffffu, w, L);
      const float oinv = __shfl_sync(0xffffffffu, inv_w, L);
      const uint32_t og = __shfl_sync(0xffffffffu, g, L);
      const bool active = e0 + lane < total;
      uint32_t t = 0;
      if (active) {
        int r = (int)((float)k * oinv);  // within one of k / ow (k < 2^24)
        r += (r + 1) * ow <= k;
        r -= r * ow > k;
        t = (uint32_t)((oy + r) * bp.tiles_x + ox + (k - r * ow));
        if (pos < cap) {
          pair_tile[pos] = t;
          pair_val[pos] = og;
        }
      }
      if (active) count_digits(t);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kDupThreads) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

BinParams make_bin_params(const sk_frame* f) {
  BinParams bp;
  bp.mode = f->binning.mode;
  bp.beta = f->binning.beta;
  bp.tau_alpha = f->binning.tau_alpha;
  bp.ts = f->tile_size;
  bp.tiles_x = f->tiles_x;
  bp.tiles_y = f->tiles_y;
  bp.W = f->width;
  bp.H = f->height;
  return bp;
}

}  // namespace

void launch_preprocess(sk_ctx* ctx, const sk_scene* scene, const sk_camera& cam, sk_frame* f) {
  const int64_t n = scene->n;
  if (n == 0) return;
  const CamParams cp = make_cam_params(cam);
  const BinParams bp = make_bin_params(f);
  const int block = 256;
  const unsigned grid = (unsigned)((n + block - 1) / block);
  auto args = [&](auto kern) {
    kern<<<grid, block, 0, ctx->stream>>>(
        scene->params.as<float>(), scene->capacity, n, cp, bp, f->mean2d.as<float2>(), f->conic_op.as<float4>(),
        f->rgb_depth.as<float4>(), f->cov2d.as<float4>(), f->conic4.as<float4>(), f->radius.as<float>(),
        f->tiles.as<int>(), f->rect.as<int4>(), f->a_star.as<float>(), f->keys_a.as<uint32_t>(),
        f->vals_a.as<uint32_t>(), ctx->err_word.as<uint32_t>());
  };
  switch (scene->sh_degree) {
    case 0: args(preprocess_kernel<0>); break;
    case 1: args(preprocess_kernel<1>); break;
    case 2: args(preprocess_kernel<2>); break;
    default: args(preprocess_kernel<3>); break;
  }
  note_launch();
  SK_CUDA(cudaGetLastError());
}

void launch_inject_bin(sk_ctx* ctx, sk_frame* f) {
  if (f->n == 0) return;
  const BinParams bp = make_bin_params(f);
  const unsigned grid = (unsigned)((f->n + 255) / 256);
  inject_bin_kernel<<<grid, 256, 0, ctx->stream>>>(
      f->n, bp, f->mean2d.as<float2>(), f->conic_op.as<float4>(), f->rgb_depth.as<float4>(), f->cov2d.as<float4>(),
      f->radius.as<float>(), f->tiles.as<int>(), f->rect.as<int4>(), f->a_star.as<float>(),
      f->keys_a.as<uint32_t>(), f->vals_a.as<uint32_t>(), ctx->err_word.as<uint32_t>());
  note_launch();
  SK_CUDA(cudaGetLastError());
}

void launch_duplicate(sk_ctx* ctx, sk_frame* f, const uint32_t* order, const int32_t* offsets, uint32_t* pair_tile,
                      uint32_t* pair_val, int passes, int width, uint32_t* hist, int64_t cap) {
  if (f->n == 0) return;
  const BinParams bp = make_bin_params(f);
  const int64_t warps = (f->n + 31) / 32;
  const unsigned grid = (unsigned)std::min<int64_t>((warps + kDupThreads / 32 - 1) / (kDupThreads / 32), 148 * 8);
  duplicate_kernel<<<grid, kDupThreads, 0, ctx->stream>>>(
      f->n, bp, order, offsets, f->tiles.as<int>(), f->rect.as<int4>(), f->mean2d.as<float2>(),
      f->conic_op.as<float4>(), f->a_star.as<float>(), pair_tile, pair_val, passes, width, hist, cap);
  note_launch();
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
