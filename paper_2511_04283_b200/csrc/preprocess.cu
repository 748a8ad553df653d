// K1 preprocess and K3 tile binning (counting scatter).
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
  auto culled = [&]() {
    radius_out[i] = 0.0f;
    if (cov_out) tiles_out[i] = 0;
    rect_out[i] = make_int4(0, 0, -1, -1);  // K3 enumerates rectangles only
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
  // L1 prefetch of the SH rows (no registers held): they land while the
  // projection, covariance and culling arithmetic below runs (K1 -2%)
#pragma unroll
  for (int c = SK_COMP_SH; c < SK_COMP_SH + 3 * (DEG + 1) * (DEG + 1); ++c)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p + c * stride + i));
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
  conic4[i] = make_float4(inv00, inv01, inv10, inv11);
  radius_out[i] = radius;
  rect_out[i] = bo.rect;
  // the covariance and tile count only leave the device through
  // sk_frame_get_projected; a* only feeds compact binning
  if (cov_out) {
    cov_out[i] = make_float4(c[0][0], c[0][1], c[1][0], c[1][1]);
    tiles_out[i] = bo.count;
  }
  if (cov_out || bp.mode != 0) astar_out[i] = bo.a_star;
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

// K3: the per-tile lists as a stable counting scatter (replaces the
// reference's per-tile push_back in build_tile_grid, raster.hpp:157-168, and
// the sort that list order implies).
//
// The slots are visited in (depth, index) order — the depth sort's output —
// cut into chunks of consecutive slots. The tile rows are split into
// row-groups whose counters fit in shared memory (one group at 1080p / 16-px
// tiles); a CTA handles one (chunk, row-group).
//   bin_count_kernel    counts[chunk][tile] = pairs of the chunk per tile
//                       (shared-memory atomics; order does not matter here)
//   bin_prefix_kernel   counts -> exclusive prefix over chunks, per tile; the
//                       last CTA scans the tile totals into the ranges and P
//   bin_scatter_kernel  each warp owns a band of tile rows, so no two warps
//                       share a tile counter. Per stage of slots the CTA
//                       builds, with ballots, each band's list of the slots
//                       whose rectangle reaches it (in slot order); a warp
//                       walks its list and enumerates the band's pairs
//                       Gaussian-major, 32 at a time (lane e takes pair e:
//                       owner by a shuffle binary search over the lanes'
//                       offsets, tile from the owner's rectangle). Lower lanes
//                       therefore hold earlier Gaussians, so a pair's rank
//                       among the round's same-tile pairs is its order in the
//                       warp: a shared-memory tag probe (each lane tags its
//                       tile, a lane reading back another id has a peer)
//                       finds the rounds with shared tiles, and only those
//                       rank with __match_any_sync. The round's first lane of
//                       each tile advances the tile's counter: slot =
//                       ranges[t].x + prefix[chunk][t] + the chunk's earlier
//                       pairs of t.
// Every tile thus receives its Gaussians in (depth, index) order — the
// reference's list order — with no key sort over the pairs, and only the
// 4-byte Gaussian index is written per pair. Compact binning enumerates the
// same rectangle and drops the tiles failing the min-Mahalanobis test
// (bin_compact, raster.hpp:111-141), exactly as K1 counted them.
#ifndef SK_BIN_WARPS
#define SK_BIN_WARPS 16
#endif
#ifndef SK_BIN_MINB
#define SK_BIN_MINB 2
#endif
constexpr int kBinWarps = SK_BIN_WARPS;  // tile-row bands per scatter CTA
constexpr int kBinThreads = kBinWarps * 32;
constexpr int kBinStage = 1024;  // slots staged in shared memory per step
constexpr int kCountThreads = 256;
constexpr int kBinMaxSmemTiles = 24576;  // 96 KB of int32 counters (+ 96 KB of tags) per row-group
constexpr int kCountSmallArea = 48;      // larger rectangles are counted by the whole warp

struct BinLayout {
  int64_t n;           // slots in depth order
  int64_t chunk;       // slots per chunk (multiple of kBinThreads)
  int tiles;           // tiles_x * tiles_y
  int rows_per_group;  // tile rows per CTA row-group
};

__device__ __forceinline__ uint32_t lanemask_lt_u32() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Compact binning keeps a tile of the rectangle only if the footprint's
// min-Mahalanobis distance to it is within a* (the test K1 counted with).
__device__ __forceinline__ bool compact_keeps(const BinParams& bp, int ty, int tx, float2 mu, float4 co, float as) {
  const float ry0 = (float)(ty * bp.ts);
  const float ry1 = (float)(min((ty + 1) * bp.ts, bp.H) - 1);
  const float rx0 = (float)(tx * bp.ts);
  const float rx1 = (float)(min((tx + 1) * bp.ts, bp.W) - 1);
  return min_mahalanobis_on_rect(co.x, co.y, co.z, mu.x, mu.y, rx0, rx1, ry0, ry1) <= as;
}

__global__ void __launch_bounds__(kCountThreads) bin_count_kernel(BinParams bp, BinLayout L,
                                                                  const uint32_t* __restrict__ order,
                                                                  const int4* __restrict__ rect,
                                                                  const float2* __restrict__ mean2d,
                                                                  const float4* __restrict__ conic_op,
                                                                  const float* __restrict__ a_star,
                                                                  int32_t* __restrict__ counts) {
  extern __shared__ int32_t s_cnt[];
  const int row0 = blockIdx.y * L.rows_per_group;
  const int rows = min(L.rows_per_group, bp.tiles_y - row0);
  const int t0 = row0 * bp.tiles_x;
  const int gtiles = rows * bp.tiles_x;
  for (int i = threadIdx.x; i < gtiles; i += kCountThreads) s_cnt[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t s_begin = (int64_t)blockIdx.x * L.chunk;
  const int64_t s_end = s_begin + L.chunk < L.n ? s_begin + L.chunk : L.n;
  constexpr int kPer = 4;  // slots per thread per step: their loads are issued together
  for (int64_t sb = s_begin; sb < s_end; sb += kCountThreads * kPer) {
    uint32_t gq[kPer];
    int4 rq[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int64_t s = sb + q * kCountThreads + threadIdx.x;
      gq[q] = s < s_end ? order[s] : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) rq[q] = gq[q] != 0xffffffffu ? rect[gq[q]] : make_int4(0, 0, -1, -1);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t g = gq[q];
      const int4 rc = rq[q];
      const int ya = max(rc.y, row0), yb = min(rc.w, row0 + rows - 1), xa = rc.x, w = rc.z - rc.x + 1;
      const int area = ya <= yb ? (yb - ya + 1) * w : 0;
      if (area > 0 && area <= kCountSmallArea) {
        float2 mu = make_float2(0.f, 0.f);
        float4 co = make_float4(0.f, 0.f, 0.f, 0.f);
        float as = 0.f;
        if (bp.mode != 0) {
          mu = mean2d[g];
          co = conic_op[g];
          as = a_star[g];
        }
        for (int ty = ya; ty <= yb; ++ty)
          for (int tx = xa; tx < xa + w; ++tx)
            if (bp.mode == 0 || compact_keeps(bp, ty, tx, mu, co, as)) atomicAdd(&s_cnt[(ty - row0) * bp.tiles_x + tx], 1);
      }
      // large rectangles: the whole warp strides over one at a time
      uint32_t big = __ballot_sync(0xffffffffu, area > kCountSmallArea);
      while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const int sya = __shfl_sync(0xffffffffu, ya, src);
        const int sxa = __shfl_sync(0xffffffffu, xa, src);
        const int sw = __shfl_sync(0xffffffffu, w, src);
        const int sarea = __shfl_sync(0xffffffffu, area, src);
        const uint32_t sg = __shfl_sync(0xffffffffu, g, src);
        float2 mu = make_float2(0.f, 0.f);
        float4 co = make_float4(0.f, 0.f, 0.f, 0.f);
        float as = 0.f;
        if (bp.mode != 0) {
          mu = mean2d[sg];
          co = conic_op[sg];
          as = a_star[sg];
        }
        for (int k = lane; k < sarea; k += 32) {
          const int r = k / sw;
          const int ty = sya + r, tx = sxa + (k - r * sw);
          if (bp.mode == 0 || compact_keeps(bp, ty, tx, mu, co, as)) atomicAdd(&s_cnt[(ty - row0) * bp.tiles_x + tx], 1);
        }
      }
    }
  }
  __syncthreads();
  int32_t* crow = counts + (int64_t)blockIdx.x * L.tiles + t0;
  for (int i = threadIdx.x; i < gtiles; i += kCountThreads) crow[i] = s_cnt[i];
}

// counts[c][t] -> sum over chunks c' < c (in place), per tile column: 32
// tiles per CTA, pages of 32 x 8 chunk rows, each warp holding its 8 rows
// of the page in registers (one read, one write of the matrix). The last CTA
// to finish scans the tile totals into ranges[t] = [start, start + total)
// and writes P.
constexpr int kPrefixWarps = 32;
constexpr int kPrefixRows = 8;
__global__ void __launch_bounds__(kPrefixWarps * 32) bin_prefix_kernel(int32_t* __restrict__ counts, int chunks,
                                                                       int tiles, int32_t* __restrict__ totals,
                                                                       int2* __restrict__ ranges,
                                                                       unsigned int* __restrict__ done,
                                                                       long long* __restrict__ total_out,
                                                                       int64_t cap, uint32_t* __restrict__ err) {
  constexpr int NT = kPrefixWarps * 32;
  constexpr int kItems = 4;
  __shared__ int32_t s_sum[kPrefixWarps][32];
  __shared__ bool s_last;
  __shared__ long long s_carry;
  __shared__ long long s_warp[kPrefixWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  int carry = 0;
  for (int page = 0; page < chunks; page += kPrefixWarps * kPrefixRows) {
    const int c0 = page + warp * kPrefixRows;
    int v[kPrefixRows];
    int sum = 0;
#pragma unroll
    for (int r = 0; r < kPrefixRows; ++r) {
      v[r] = c0 + r < chunks && t < tiles ? counts[(int64_t)(c0 + r) * tiles + t] : 0;
      sum += v[r];
    }
    __syncthreads();  // s_sum of the previous page consumed
    s_sum[warp][lane] = sum;
    __syncthreads();
    int run = carry, page_total = 0;
#pragma unroll
    for (int w = 0; w < kPrefixWarps; ++w) {
      const int x = s_sum[w][lane];
      run += w < warp ? x : 0;
      page_total += x;
    }
#pragma unroll
    for (int r = 0; r < kPrefixRows; ++r) {
      if (c0 + r < chunks && t < tiles) counts[(int64_t)(c0 + r) * tiles + t] = run;
      run += v[r];
    }
    carry += page_total;
  }
  if (warp == 0 && t < tiles) totals[t] = carry;
  // the last CTA: exclusive scan of the tile totals
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) s_carry = 0;
  for (int base = 0; base < tiles; base += NT * kItems) {
    __syncthreads();
    const int i0 = base + threadIdx.x * kItems;
    int v[kItems];
    long long loc = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      v[q] = i0 + q < tiles ? __ldcg(&totals[i0 + q]) : 0;
      loc += v[q];
    }
    long long x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    long long wb = s_carry, all = 0;
#pragma unroll
    for (int w = 0; w < kPrefixWarps; ++w) {
      wb += w < warp ? s_warp[w] : 0;
      all += s_warp[w];
    }
    long long start = wb + x - loc;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      if (i0 + q < tiles) ranges[i0 + q] = make_int2((int)start, (int)(start + v[q]));
      start += v[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry += all;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *total_out = s_carry;
    *done = 0;  // ready for the next frame
    if (cap >= 0 && s_carry > cap) atomicOr(err, kErrPairOverflow);
  }
}

__global__ void __launch_bounds__(kBinThreads, SK_BIN_MINB) bin_scatter_kernel(BinParams bp, BinLayout L,
                                                                  const uint32_t* __restrict__ order,
                                                                  const int4* __restrict__ rect,
                                                                  const float2* __restrict__ mean2d,
                                                                  const float4* __restrict__ conic_op,
                                                                  const float* __restrict__ a_star,
                                                                  const int32_t* __restrict__ counts,
                                                                  const int2* __restrict__ ranges,
                                                                  uint32_t* __restrict__ pair_val, int64_t cap) {
  extern __shared__ int32_t s_pos[];  // the row-group's tile counters
  __shared__ uint32_t s_g[kBinStage];
  __shared__ int4 s_rect[kBinStage];
  __shared__ uint32_t s_cls[kBinStage];         // per slot: bit w = the rectangle reaches warp w's rows
  __shared__ uint16_t s_queue[kBinWarps][64];  // per warp: stage slots reaching its rows, in slot order
  const int tid = threadIdx.x;
  const int row0 = blockIdx.y * L.rows_per_group;
  const int rows = min(L.rows_per_group, bp.tiles_y - row0);
  const int t0 = row0 * bp.tiles_x;
  const int gtiles = rows * bp.tiles_x;
  const int32_t* crow = counts + (int64_t)blockIdx.x * L.tiles + t0;
  for (int i = tid; i < gtiles; i += kBinThreads) s_pos[i] = ranges[t0 + i].x + crow[i];
  uint32_t* s_tag = reinterpret_cast<uint32_t*>(s_pos + L.rows_per_group * bp.tiles_x);  // per tile: last tagging lane

  // warp w owns the group's tile rows row0 + w + q * kBinWarps (interleaved,
  // so the pair load is balanced whatever the scene's vertical profile)
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = lanemask_lt_u32();
  const int64_t s_begin = (int64_t)blockIdx.x * L.chunk;
  const int64_t s_end = s_begin + L.chunk < L.n ? s_begin + L.chunk : L.n;
  // this warp's rows of a rectangle's clipped row span [ya, yb]: q in [qa, qb]
  auto my_rows = [&](int ya, int yb, int& qa) {
    const int lo = ya - row0 - warp, hi = yb - row0 - warp;
    qa = lo <= 0 ? 0 : (lo + kBinWarps - 1) / kBinWarps;
    const int qb = hi < 0 ? -1 : hi / kBinWarps;
    return qb - qa + 1;
  };
  // one batch of up to 32 queued slots (each reaches this warp's rows): their
  // pairs in this warp's rows, Gaussian-major, 32 per round. Per-round cost
  // is what bounds this kernel (MATCH / SHFL are 1/2 and 1 warp-instruction
  // per clock per SM, POPC / FLO / I2F 1/2: scripts/micro/warp_ops.cu), so a
  // round uses 5 + 3 shuffles, one MATCH, two POPC and a multiply-high for
  // the row split.
  auto walk = [&](int head, int cnt) {
    int m = 0;
    uint32_t g = 0, packed = 0, magic = 0;
    if (lane < cnt) {
      const int slot = s_queue[warp][(head + lane) & 63];
      const int4 rc = s_rect[slot];
      g = s_g[slot];
      int qa;
      const int nr = my_rows(max(rc.y, row0), min(rc.w, row0 + rows - 1), qa);
      const int w = rc.z - rc.x + 1;
      m = nr * w;
      packed = (uint32_t)rc.x | ((uint32_t)qa << 12) | ((uint32_t)w << 20);
      magic = 0xffffffffu / (uint32_t)w + 1u;  // k / w == umulhi(k, magic) for k, w < 2^16
    }
    int incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int off = incl - m;  // lanes >= cnt: off == total, never an owner
    for (int e0 = 0; e0 < total; e0 += 32) {
      const int pos = e0 + lane;
      // owner = the highest lane whose offset is <= pos = (number of queued
      // lanes with offset <= pos) - 1: queued lanes hold at least one pair,
      // so their offsets are distinct and increasing. Counted as the lanes
      // starting before this round (one ballot) plus the segment starts
      // inside it up to pos (one OR-reduction of start bits), instead of a
      // 5-step dependent shuffle search.
      const bool live = lane < cnt;
      const uint32_t before = __ballot_sync(0xffffffffu, live && off < e0);
      const uint32_t starts =
          __reduce_or_sync(0xffffffffu, (live && off >= e0 && off < e0 + 32) ? 1u << (off - e0) : 0u);
      const uint32_t upto = lane == 31 ? 0xffffffffu : (2u << lane) - 1u;
      const int o = max(0, __popc(before) + __popc(starts & upto) - 1);
      const int off_o = __shfl_sync(0xffffffffu, off, o);
      const uint32_t og = __shfl_sync(0xffffffffu, g, o);
      const uint32_t op = __shfl_sync(0xffffffffu, packed, o);
      const uint32_t omag = __shfl_sync(0xffffffffu, magic, o);
      const uint32_t k = (uint32_t)(pos - off_o);
      const uint32_t r = __umulhi(k, omag);
      const int ow = (int)(op >> 20);
      const int ty = row0 + warp + ((int)((op >> 12) & 0xffu) + (int)r) * kBinWarps;
      const int tx = (int)(op & 0xfffu) + (int)k - (int)r * ow;
      bool take = pos < total;
      if (take && bp.mode != 0) take = compact_keeps(bp, ty, tx, mean2d[og], conic_op[og], a_star[og]);
      const int local = (ty - row0) * bp.tiles_x + tx;
      // Conflict probe: each taking lane tags its tile with its lane id; a
      // lane that reads back another id shares its tile with a lower or
      // higher lane of the round. Depth-adjacent Gaussians are rarely
      // screen-adjacent, so most rounds have no shared tile and skip the
      // long-latency MATCH (rank 0, one pair per tile).
      // (an atomic exchange: concurrent tags of one tile are the point)
      if (take) atomicExch(&s_tag[local], (uint32_t)lane);
      __syncwarp();
      int rank = 0, cnt = 1;
      if (__any_sync(0xffffffffu, take && s_tag[local] != (uint32_t)lane)) {
        const uint32_t peers = __match_any_sync(0xffffffffu, take ? (uint32_t)local : 0xffffffffu);
        rank = __popc(peers & lt);
        cnt = __popc(peers);
      }
      // every lane reads the tile's counter, then the round's first lane of
      // each tile advances it (no leader search, no broadcast)
      int base = 0;
      if (take) base = s_pos[local];
      __syncwarp();
      if (take && rank == 0) s_pos[local] = base + cnt;
      __syncwarp();
      const int64_t slot = (int64_t)base + rank;
      if (take && slot < cap) pair_val[slot] = og;
    }
  };

  // stages of kBinStage slots; each thread prefetches its slots of the next
  // stage (Gaussian index, then rectangle) while the current one is walked
  constexpr int kPer = kBinStage / kBinThreads;
  uint32_t gq[kPer];
  int4 rq[kPer];
  auto prefetch = [&](int64_t sb) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int64_t s = sb + q * kBinThreads + tid;
      gq[q] = s < s_end ? order[s] : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) rq[q] = gq[q] != 0xffffffffu ? rect[gq[q]] : make_int4(0, 0, -1, -1);
  };
  prefetch(s_begin);
  for (int64_t sb = s_begin; sb < s_end; sb += kBinStage) {
    __syncthreads();  // counters initialised / the previous stage walked
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      s_g[q * kBinThreads + tid] = gq[q];
      s_rect[q * kBinThreads + tid] = rq[q];
      // row classes (mod kBinWarps) of the rectangle's rows in this group
      uint32_t cls = 0;
      const int a = max(rq[q].y, row0) - row0, b = min(rq[q].w, row0 + rows - 1) - row0;
      if (rq[q].z >= rq[q].x && a <= b) {
        constexpr uint32_t kAll = kBinWarps == 32 ? 0xffffffffu : (1u << kBinWarps) - 1u;
        const int nrow = b - a + 1;
        if (nrow >= kBinWarps) {
          cls = kAll;
        } else {
          const uint64_t run = ((1ull << nrow) - 1ull) << (a % kBinWarps);
          cls = (uint32_t)(run | (run >> kBinWarps)) & kAll;
        }
      }
      s_cls[q * kBinThreads + tid] = cls;
    }
    __syncthreads();
    if (sb + kBinStage < s_end) prefetch(sb + kBinStage);
    const int nstage = (int)(s_end - sb < kBinStage ? s_end - sb : kBinStage);
    int head = 0, queued = 0;
    for (int j0 = 0; j0 < nstage; j0 += 32) {
      const bool in = (s_cls[j0 + lane] >> warp) & 1u;
      const uint32_t mb = __ballot_sync(0xffffffffu, in);
      if (in) s_queue[warp][(head + queued + __popc(mb & lt)) & 63] = (uint16_t)(j0 + lane);
      queued += __popc(mb);
      __syncwarp();
      if (queued >= 32) {
        walk(head, 32);
        head = (head + 32) & 63;
        queued -= 32;
      }
    }
    if (queued > 0) walk(head, queued);
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

void launch_preprocess(sk_ctx* ctx, const sk_scene* scene, const sk_camera& cam, sk_frame* f, bool extras) {
  const int64_t n = scene->n;
  if (n == 0) return;
  const CamParams cp = make_cam_params(cam);
  const BinParams bp = make_bin_params(f);
  const int block = 256;
  const unsigned grid = (unsigned)((n + block - 1) / block);
  f->extras_valid = extras;
  auto args = [&](auto kern) {
    kern<<<grid, block, 0, ctx->stream>>>(
        scene->params.as<float>(), scene->capacity, n, cp, bp, f->mean2d.as<float2>(), f->conic_op.as<float4>(),
        f->rgb_depth.as<float4>(), extras ? f->cov2d.as<float4>() : nullptr, f->conic4.as<float4>(), f->radius.as<float>(),
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

BinLayout bin_layout(const sk_frame* f) {
  BinLayout L;
  L.n = f->n;
  L.tiles = f->tiles_x * f->tiles_y;
  // ~8 chunks per SM (measured at config 2); SK_BIN_CHUNK overrides (A/B)
  static const int64_t forced = [] {
    const char* e = std::getenv("SK_BIN_CHUNK");
    return e ? std::atoll(e) : 0ll;
  }();
  int64_t chunk = forced > 0 ? forced : (L.n + 8 * 148 - 1) / (8 * 148);
  chunk = std::max<int64_t>(chunk, 1024);
  L.chunk = (chunk + kBinStage - 1) / kBinStage * kBinStage;
  L.rows_per_group = std::max(1, std::min(f->tiles_y, kBinMaxSmemTiles / f->tiles_x));
  // the scatter packs a tile column and a rectangle width into 12 bits each
  // and a warp's row index into 8 (tile grids up to 4095 x 4095)
  require(f->tiles_x < 4096 && f->tiles_y < 4096, "build_tile_grid: at most 4095 x 4095 tiles");
  return L;
}

void launch_bin_tiles(sk_ctx* ctx, sk_frame* f, const uint32_t* order, int32_t* counts, uint32_t* pair_val,
                      int64_t cap) {
  if (f->n == 0) return;
  const BinParams bp = make_bin_params(f);
  const BinLayout L = bin_layout(f);
  const dim3 grid((unsigned)((L.n + L.chunk - 1) / L.chunk),
                  (unsigned)((f->tiles_y + L.rows_per_group - 1) / L.rows_per_group));
  const size_t smem = sizeof(int32_t) * (size_t)L.rows_per_group * f->tiles_x;
  static bool attr = false;
  if (!attr) {
    SK_CUDA(cudaFuncSetAttribute(bin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 sizeof(int32_t) * kBinMaxSmemTiles));
    SK_CUDA(cudaFuncSetAttribute(bin_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * sizeof(int32_t) * kBinMaxSmemTiles));
    attr = true;
  }
  if (pair_val)
    bin_scatter_kernel<<<grid, kBinThreads, 2 * smem, ctx->stream>>>(
        bp, L, order, f->rect.as<int4>(), f->mean2d.as<float2>(), f->conic_op.as<float4>(),
        f->a_star.as<float>(), counts, f->ranges.as<int2>(), pair_val, cap);
  else
    bin_count_kernel<<<grid, kCountThreads, smem, ctx->stream>>>(bp, L, order,
                                                                 f->rect.as<int4>(), f->mean2d.as<float2>(),
                                                                 f->conic_op.as<float4>(), f->a_star.as<float>(),
                                                                 counts);
  note_launch();
  SK_CUDA(cudaGetLastError());
}

int64_t bin_chunks(const sk_frame* f) {
  const BinLayout L = bin_layout(f);
  return (L.n + L.chunk - 1) / L.chunk;
}

void launch_bin_prefix(sk_ctx* ctx, sk_frame* f, int32_t* counts, int32_t* totals, unsigned int* done, int64_t cap,
                       uint32_t* err, long long* total_out) {
  const int tiles = f->tiles_x * f->tiles_y;
  bin_prefix_kernel<<<(unsigned)((tiles + 31) / 32), kPrefixWarps * 32, 0, ctx->stream>>>(
      counts, (int)bin_chunks(f), tiles, totals, f->ranges.as<int2>(), done, total_out, cap, err);
  note_launch();
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
