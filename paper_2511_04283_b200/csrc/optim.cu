// K9 project-backward + ScoreTable statistics and K10 dense Adam.
//
// K9 restates cov_grad_from_inv_grad and project_backward (reference
// camera.hpp:148-213) with evaluate_sh_backward (sh.hpp:93-114) and
// covariance_3d_backward / quat_rotation_backward (scene.hpp:70-110), plus the
// per-render statistics of Trainer::train_iteration (trainer.hpp:139-156).
// K10 restates AdamGroup::step (adam.hpp:62-74) for all six groups of
// SceneOptimizer::step (:124-143): dense over every Gaussian, a per-group
// step counter and bias correction, eps outside the sqrt.
//
// K9 runs one thread per Gaussian (zero gradients when culled) and writes the
// gradients through a shared-memory tile; K10 streams params / m / v / grads
// with float4 accesses at ~92% of the HBM copy roof. On one GPU with dense
// Adam the two run fused (project_bwd_adam_kernel): the gradients never
// leave the CTA's tile.
#include "state.h"

namespace sk {
namespace {

constexpr float kC0 = 0.28209479177387814f;
constexpr float kC1 = 0.4886025119029199f;
__device__ constexpr float kC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                                     -1.0925484305920792f, 0.5462742152960396f};
__device__ constexpr float kC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                                     0.3731763325901154f,  -0.4570457994644658f, 1.445305721320277f,
                                     -0.5900435899266435f};

struct Stats {
  float* grad_norm_acc;
  float* abs_grad_acc;
  float* grad3d_acc;  // [3][stride]
  int* views_seen;
  float* max_radius2d;
};

// Computes all parameter gradients of one visible Gaussian (camera.hpp:156-213).
// grad[] is indexed by SK_COMP_*.
// grad[c * GS] receives the gradient of component c.
template <int DEG, int GS>
__device__ __forceinline__ void project_backward_one(const float* __restrict__ p, int64_t stride, int64_t i,
                                                     const CamParams& cam, const float dmu2d[2], const float dcov[2][2],
                                                     const float dcol[3], float dop, float* grad,
                                                     const float* s_exp2) {
  constexpr int NSH = (DEG + 1) * (DEG + 1);
  const float mu[3] = {p[0 * stride + i], p[1 * stride + i], p[2 * stride + i]};
  const float* R = cam.r;
  float t[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = ((R[3 * k] * mu[0] + R[3 * k + 1] * mu[1]) + R[3 * k + 2] * mu[2]) + cam.t[k];
  const float iz = 1.0f / t[2];
  const float iz2 = iz * iz;
  const float iz3 = iz2 * iz;
  const float J[2][3] = {{cam.fx * iz, 0.0f, -cam.fx * t[0] * iz2}, {0.0f, cam.fy * iz, -cam.fy * t[1] * iz2}};
  float m[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) m[a][j] = (J[a][0] * R[j] + J[a][1] * R[3 + j]) + J[a][2] * R[6 + j];
  // rotation / scale
  const float q_in[4] = {p[3 * stride + i], p[4 * stride + i], p[5 * stride + i], p[6 * stride + i]};
  const float s[3] = {det_expf(p[7 * stride + i], s_exp2), det_expf(p[8 * stride + i], s_exp2),
                      det_expf(p[9 * stride + i], s_exp2)};
  const float n2 = ((q_in[0] * q_in[0] + q_in[1] * q_in[1]) + q_in[2] * q_in[2]) + q_in[3] * q_in[3];
  const float nq = sqrtf(n2);
  const float w = q_in[0] / nq, x = q_in[1] / nq, y = q_in[2] / nq, z = q_in[3] / nq;
  float r[3][3];
  r[0][0] = 1.0f - 2.0f * (y * y + z * z);
  r[0][1] = 2.0f * (x * y - w * z);
  r[0][2] = 2.0f * (x * z + w * y);
  r[1][0] = 2.0f * (x * y + w * z);
  r[1][1] = 1.0f - 2.0f * (x * x + z * z);
  r[1][2] = 2.0f * (y * z - w * x);
  r[2][0] = 2.0f * (x * z - w * y);
  r[2][1] = 2.0f * (y * z + w * x);
  r[2][2] = 1.0f - 2.0f * (x * x + y * y);
  float M[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) M[a][b] = r[a][b] * s[b];
  float S[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) S[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];

  // opacity (camera.hpp:171-172)
  const float sig = det_sigmoidf(p[SK_COMP_OPACITY * stride + i], s_exp2);
  grad[SK_COMP_OPACITY * GS] = dop * sig * (1.0f - sig);

  // colour (camera.hpp:175-182, sh.hpp:93-114)
  float gmu[3];
  {
    const float rel[3] = {mu[0] - cam.center[0], mu[1] - cam.center[1], mu[2] - cam.center[2]};
    const float dist = sqrtf((rel[0] * rel[0] + rel[1] * rel[1]) + rel[2] * rel[2]);
    const float dx = rel[0] / dist, dy = rel[1] / dist, dz = rel[2] / dist;
    float basis[NSH];
    float db[NSH][3];
    basis[0] = kC0;
    db[0][0] = db[0][1] = db[0][2] = 0.0f;
    if (DEG >= 1) {
      basis[1] = -kC1 * dy;
      basis[2] = kC1 * dz;
      basis[3] = -kC1 * dx;
      db[1][0] = 0.f, db[1][1] = -kC1, db[1][2] = 0.f;
      db[2][0] = 0.f, db[2][1] = 0.f, db[2][2] = kC1;
      db[3][0] = -kC1, db[3][1] = 0.f, db[3][2] = 0.f;
    }
    if (DEG >= 2) {
      const float xx = dx * dx, yy = dy * dy, zz = dz * dz;
      basis[4] = kC2[0] * (dx * dy);
      basis[5] = kC2[1] * (dy * dz);
      basis[6] = kC2[2] * (2.0f * zz - xx - yy);
      basis[7] = kC2[3] * (dx * dz);
      basis[8] = kC2[4] * (xx - yy);
      db[4][0] = kC2[0] * dy, db[4][1] = kC2[0] * dx, db[4][2] = 0.f;
      db[5][0] = 0.f, db[5][1] = kC2[1] * dz, db[5][2] = kC2[1] * dy;
      db[6][0] = kC2[2] * (-2.0f * dx), db[6][1] = kC2[2] * (-2.0f * dy), db[6][2] = kC2[2] * (4.0f * dz);
      db[7][0] = kC2[3] * dz, db[7][1] = 0.f, db[7][2] = kC2[3] * dx;
      db[8][0] = kC2[4] * (2.0f * dx), db[8][1] = kC2[4] * (-2.0f * dy), db[8][2] = 0.f;
      if (DEG >= 3) {
        basis[9] = kC3[0] * dy * (3.0f * xx - yy);
        basis[10] = kC3[1] * (dx * dy) * dz;
        basis[11] = kC3[2] * dy * (4.0f * zz - xx - yy);
        basis[12] = kC3[3] * dz * (2.0f * zz - 3.0f * xx - 3.0f * yy);
        basis[13] = kC3[4] * dx * (4.0f * zz - xx - yy);
        basis[14] = kC3[5] * dz * (xx - yy);
        basis[15] = kC3[6] * dx * (xx - 3.0f * yy);
        db[9][0] = kC3[0] * (6.0f * dx * dy), db[9][1] = kC3[0] * (3.0f * xx - 3.0f * yy), db[9][2] = 0.f;
        db[10][0] = kC3[1] * (dy * dz), db[10][1] = kC3[1] * (dx * dz), db[10][2] = kC3[1] * (dx * dy);
        db[11][0] = kC3[2] * (-2.0f * dx * dy), db[11][1] = kC3[2] * (4.0f * zz - xx - 3.0f * yy),
        db[11][2] = kC3[2] * (8.0f * dy * dz);
        db[12][0] = kC3[3] * (-6.0f * dx * dz), db[12][1] = kC3[3] * (-6.0f * dy * dz),
        db[12][2] = kC3[3] * (6.0f * zz - 3.0f * xx - 3.0f * yy);
        db[13][0] = kC3[4] * (4.0f * zz - 3.0f * xx - yy), db[13][1] = kC3[4] * (-2.0f * dx * dy),
        db[13][2] = kC3[4] * (8.0f * dx * dz);
        db[14][0] = kC3[5] * (2.0f * dx * dz), db[14][1] = kC3[5] * (-2.0f * dy * dz), db[14][2] = kC3[5] * (xx - yy);
        db[15][0] = kC3[6] * (3.0f * xx - 3.0f * yy), db[15][1] = kC3[6] * (-6.0f * dx * dy), db[15][2] = 0.f;
      }
    }
    // the SH coefficients are read twice (L1-resident) instead of being held
    // in 48 registers across both passes
    float raw[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < NSH; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) raw[c] += basis[k] * p[(SK_COMP_SH + 3 * k + c) * stride + i];
    float draw[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) draw[c] = (raw[c] + 0.5f < 0.0f) ? 0.0f : dcol[c];
    float ddir[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < NSH; ++k) {
#pragma unroll
      for (int c = 0; c < 3; ++c) grad[(SK_COMP_SH + 3 * k + c) * GS] = basis[k] * draw[c];
      const float s0 = p[(SK_COMP_SH + 3 * k + 0) * stride + i];
      const float s1 = p[(SK_COMP_SH + 3 * k + 1) * stride + i];
      const float s2 = p[(SK_COMP_SH + 3 * k + 2) * stride + i];
      const float sd = (s0 * draw[0] + s1 * draw[1]) + s2 * draw[2];
#pragma unroll
      for (int c = 0; c < 3; ++c) ddir[c] += sd * db[k][c];
    }
    const float dd = (dx * ddir[0] + dy * ddir[1]) + dz * ddir[2];
    gmu[0] = (ddir[0] - dx * dd) / dist;
    gmu[1] = (ddir[1] - dy * dd) / dist;
    gmu[2] = (ddir[2] - dz * dd) / dist;
  }

  // covariance: d_m = ((G + G^T) m) Sigma, d_Sigma3 = (m^T G) m
  float Gs[2][2] = {{dcov[0][0] + dcov[0][0], dcov[0][1] + dcov[1][0]},
                    {dcov[1][0] + dcov[0][1], dcov[1][1] + dcov[1][1]}};
  float Gm[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) Gm[a][j] = Gs[a][0] * m[0][j] + Gs[a][1] * m[1][j];
  float dm[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) dm[a][j] = (Gm[a][0] * S[0][j] + Gm[a][1] * S[1][j]) + Gm[a][2] * S[2][j];
  float mG[3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) mG[a][b] = m[0][a] * dcov[0][b] + m[1][a] * dcov[1][b];
  float dS[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) dS[a][b] = mG[a][0] * m[0][b] + mG[a][1] * m[1][b];
  // covariance_3d_backward (scene.hpp:101-110)
  {
    float dM[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) acc += (dS[a][k] + dS[k][a]) * M[k][b];
        dM[a][b] = acc;
      }
    float dr[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) dr[a][b] = dM[a][b] * s[b];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const float ds = (dM[0][b] * r[0][b] + dM[1][b] * r[1][b]) + dM[2][b] * r[2][b];
      grad[(SK_COMP_LOG_SCALE + b) * GS] = ds * s[b];
    }
    // quat_rotation_backward (scene.hpp:70-84)
    const float du_w = dr[0][1] * (-2.0f * z) + dr[0][2] * (2.0f * y) + dr[1][0] * (2.0f * z) +
                       dr[1][2] * (-2.0f * x) + dr[2][0] * (-2.0f * y) + dr[2][1] * (2.0f * x);
    const float du_x = dr[0][1] * (2.0f * y) + dr[0][2] * (2.0f * z) + dr[1][0] * (2.0f * y) +
                       dr[1][1] * (-4.0f * x) + dr[1][2] * (-2.0f * w) + dr[2][0] * (2.0f * z) +
                       dr[2][1] * (2.0f * w) + dr[2][2] * (-4.0f * x);
    const float du_y = dr[0][0] * (-4.0f * y) + dr[0][1] * (2.0f * x) + dr[0][2] * (2.0f * w) +
                       dr[1][0] * (2.0f * x) + dr[1][2] * (2.0f * z) + dr[2][0] * (-2.0f * w) +
                       dr[2][1] * (2.0f * z) + dr[2][2] * (-4.0f * y);
    const float du_z = dr[0][0] * (-4.0f * z) + dr[0][1] * (-2.0f * w) + dr[0][2] * (2.0f * x) +
                       dr[1][0] * (2.0f * w) + dr[1][1] * (-4.0f * z) + dr[1][2] * (2.0f * y) +
                       dr[2][0] * (2.0f * x) + dr[2][1] * (2.0f * y);
    const float qd = ((w * du_w + x * du_x) + y * du_y) + z * du_z;
    grad[(SK_COMP_ROT + 0) * GS] = (du_w - w * qd) / nq;
    grad[(SK_COMP_ROT + 1) * GS] = (du_x - x * qd) / nq;
    grad[(SK_COMP_ROT + 2) * GS] = (du_y - y * qd) / nq;
    grad[(SK_COMP_ROT + 3) * GS] = (du_z - z * qd) / nq;
  }
  // d_j = d_m R^T ; d_t (camera.hpp:197-207) ; + J^T d_mu2d ; mu += R^T d_t
  float dj[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) dj[a][j] = (dm[a][0] * R[3 * j] + dm[a][1] * R[3 * j + 1]) + dm[a][2] * R[3 * j + 2];
  float dt[3];
  dt[0] = dj[0][2] * (-cam.fx * iz2);
  dt[1] = dj[1][2] * (-cam.fy * iz2);
  dt[2] = ((dj[0][0] * (-cam.fx * iz2) + dj[0][2] * (2.0f * cam.fx * t[0] * iz3)) + dj[1][1] * (-cam.fy * iz2)) +
          dj[1][2] * (2.0f * cam.fy * t[1] * iz3);
#pragma unroll
  for (int k = 0; k < 3; ++k) dt[k] += J[0][k] * dmu2d[0] + J[1][k] * dmu2d[1];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    grad[(SK_COMP_MU + k) * GS] = gmu[k] + ((R[k] * dt[0] + R[3 + k] * dt[1]) + R[6 + k] * dt[2]);
}

struct AdamParams {
  float lr[6];
  float bc1[6];
  float bc2[6];
  int active[6];
};

__device__ __forceinline__ int comp_group(int c) {
  return c < 3 ? 0 : (c < 7 ? 1 : (c < 10 ? 2 : (c < 11 ? 3 : (c < 14 ? 4 : 5))));
}

// Correctly rounded a / b for b > 0 finite. A zero dividend takes the IEEE
// division's slow path (FCHK) on sm_100; +-0 / b == a, so select it instead.
__device__ __forceinline__ float div_pos(float a, float b) {
  const float q = __fdiv_rn(a == 0.0f ? 1.0f : a, b);
  return a == 0.0f ? a : q;
}

// AdamGroup::step element update (adam.hpp:70-73), exactly in the reference's order.
__device__ __forceinline__ void adam_update(float& param, float& m, float& v, float g, float lr, float bc1, float bc2) {
  const float b1 = (float)0.9, b2 = (float)0.999;
  m = __fadd_rn(__fmul_rn(b1, m), __fmul_rn(__fsub_rn(1.0f, b1), g));
  v = __fadd_rn(__fmul_rn(b2, v), __fmul_rn(__fmul_rn(__fsub_rn(1.0f, b2), g), g));
  const float num = __fmul_rn(lr, div_pos(m, bc1));
  const float vh = div_pos(v, bc2);
  const float root = __fsqrt_rn(vh == 0.0f ? 1.0f : vh);
  const float den = __fadd_rn(vh == 0.0f ? vh : root, (float)1e-15);
  param = __fsub_rn(param, div_pos(num, den));
}

__device__ __forceinline__ void load_blend(const float* __restrict__ bg, int64_t gstride, int64_t i, float dmu2d[2],
                                           float dcov[2][2], const float4 conic4, float dcol[3], float& dop,
                                           float absg[2]) {
  dmu2d[0] = bg[0 * gstride + i];
  dmu2d[1] = bg[1 * gstride + i];
  const float dc00 = bg[2 * gstride + i], dc01 = bg[3 * gstride + i], dc11 = bg[4 * gstride + i];
  dcol[0] = bg[5 * gstride + i];
  dcol[1] = bg[6 * gstride + i];
  dcol[2] = bg[7 * gstride + i];
  dop = bg[8 * gstride + i];
  absg[0] = bg[9 * gstride + i];
  absg[1] = bg[10 * gstride + i];
  // cov_grad_from_inv_grad: -(inv dinv) inv, dinv = [[dc00, dc01], [dc01, dc11]]
  const float inv[2][2] = {{conic4.x, conic4.y}, {conic4.z, conic4.w}};
  const float dinv[2][2] = {{dc00, dc01}, {dc01, dc11}};
  float A[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) A[a][b] = inv[a][0] * dinv[0][b] + inv[a][1] * dinv[1][b];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) dcov[a][b] = -(A[a][0] * inv[0][b] + A[a][1] * inv[1][b]);
}

__device__ __forceinline__ void accumulate_stats(const Stats& st, int64_t i, int64_t stride, const float dmu2d[2],
                                                 const float absg[2], const float gmu[3], float radius, float ndc_x,
                                                 float ndc_y) {
  const float gx = dmu2d[0] * ndc_x, gy = dmu2d[1] * ndc_y;
  st.grad_norm_acc[i] += sqrtf(gx * gx + gy * gy);
  st.abs_grad_acc[i] += absg[0] * ndc_x + absg[1] * ndc_y;
#pragma unroll
  for (int k = 0; k < 3; ++k) st.grad3d_acc[k * stride + i] += gmu[k];
  st.views_seen[i] += 1;
  st.max_radius2d[i] = fmaxf(st.max_radius2d[i], radius);
}

constexpr int kPbThreads = 128;
constexpr int kK9MinBlocks = 4;  // resident CTAs per SM the register budget is sized for (5 / 6 spill)

// K9: one thread per Gaussian computes all parameter gradients into its
// column of a shared-memory tile (conflict-free: column = threadIdx.x, so no
// 59-register live range) and the tile is written back as coalesced rows of the
// planar gradient buffer; culled Gaussians get zeros (SceneGrads::init).
template <int DEG>
__global__ void __launch_bounds__(kPbThreads, kK9MinBlocks) project_bwd_kernel(
    const float* __restrict__ params, int64_t stride, int64_t n, CamParams cam, const float* __restrict__ radius,
    const float4* __restrict__ conic4, const float* __restrict__ bg, int64_t gstride, float* __restrict__ grads,
    Stats st, bool do_stats, const uint32_t* __restrict__ err) {
  constexpr int NC = 11 + 3 * (DEG + 1) * (DEG + 1);
  // A step whose K1 raised a device error (covariance_3d's throw,
  // scene.hpp:89-92) mutates no persistent state: the reference throws
  // before any update. The word is block-uniform.
  if (__ldg(err)) return;
  __shared__ float s_grad[NC * kPbThreads];
  __shared__ float s_exp2[64];
  stage_exp2_table(s_exp2);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kPbThreads + threadIdx.x;
  if (i >= n) return;
  float* g = s_grad + threadIdx.x;  // component c at g[c * kPbThreads]
  // L1 prefetches (no registers held) of everything the visible path reads
  // first, issued before the radius test so the latency overlaps it
#pragma unroll
  for (int c = 0; c < 11; ++c) asm volatile("prefetch.global.L1 [%0];" ::"l"(bg + c * gstride + i));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(conic4 + i));
#pragma unroll
  for (int c = 0; c < NC; ++c)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(params + c * stride + i));
  if (do_stats) {  // the statistics read-modify-write at the end
    asm volatile("prefetch.global.L1 [%0];" ::"l"(st.grad_norm_acc + i));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(st.abs_grad_acc + i));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(st.views_seen + i));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(st.max_radius2d + i));
#pragma unroll
    for (int k = 0; k < 3; ++k) asm volatile("prefetch.global.L1 [%0];" ::"l"(st.grad3d_acc + k * stride + i));
  }
  const float rad = radius[i];
  if (rad > 0.0f) {
    float dmu2d[2], dcov[2][2], dcol[3], dop, absg[2];
    load_blend(bg, gstride, i, dmu2d, dcov, conic4[i], dcol, dop, absg);
    project_backward_one<DEG, kPbThreads>(params, stride, i, cam, dmu2d, dcov, dcol, dop, g, s_exp2);
    if (do_stats) {
      const float gmu[3] = {g[0], g[kPbThreads], g[2 * kPbThreads]};
      accumulate_stats(st, i, stride, dmu2d, absg, gmu, rad, (float)cam.width / 2.0f, (float)cam.height / 2.0f);
    }
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) g[c * kPbThreads] = 0.0f;
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) grads[c * stride + i] = g[c * kPbThreads];
}

// project_backward (camera.hpp:156-213) with explicit per-Gaussian upstream
// gradients (d_mu2d [n][2], d_cov2d [n][4] row-major, d_color [n][3],
// d_opacity [n]) for every Gaussian, as the reference's per-Gaussian call:
// no culling test (the C++ API's project_backward).
template <int DEG>
__global__ void __launch_bounds__(kPbThreads, kK9MinBlocks) project_bwd_explicit_kernel(
    const float* __restrict__ params, int64_t stride, int64_t n, CamParams cam, const float* __restrict__ up_mu,
    const float* __restrict__ up_cov, const float* __restrict__ up_col, const float* __restrict__ up_op,
    float* __restrict__ grads) {
  constexpr int NC = 11 + 3 * (DEG + 1) * (DEG + 1);
  __shared__ float s_grad[NC * kPbThreads];
  __shared__ float s_exp2[64];
  stage_exp2_table(s_exp2);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kPbThreads + threadIdx.x;
  if (i >= n) return;
  float* g = s_grad + threadIdx.x;
  float dmu2d[2] = {up_mu[2 * i], up_mu[2 * i + 1]};
  float dcov[2][2] = {{up_cov[4 * i], up_cov[4 * i + 1]}, {up_cov[4 * i + 2], up_cov[4 * i + 3]}};
  float dcol[3] = {up_col[3 * i], up_col[3 * i + 1], up_col[3 * i + 2]};
  project_backward_one<DEG, kPbThreads>(params, stride, i, cam, dmu2d, dcov, dcol, up_op[i], g, s_exp2);
#pragma unroll
  for (int c = 0; c < NC; ++c) grads[c * stride + i] = g[c * kPbThreads];
}

// AdamGroup::remap (adam.hpp:45-58) for every group: survivors keep their
// moments at their new index, new slots start at zero (zeroed by the caller).
__global__ void remap_moments_kernel(const float* __restrict__ m, const float* __restrict__ v, int64_t stride, int64_t n,
                                     const int32_t* __restrict__ old_to_new, float* __restrict__ m2,
                                     float* __restrict__ v2, int64_t stride2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = old_to_new[i];
  if (j < 0) return;
  const int c = blockIdx.y;
  m2[c * stride2 + j] = m[c * stride + i];
  v2[c * stride2 + j] = v[c * stride + i];
}

// K10: dense Adam over every component of every Gaussian (SceneOptimizer::step
// adam.hpp:124-143), float4-vectorised along the Gaussian axis (capacity is a
// multiple of 4, rows are 16-byte aligned). blockIdx.y is the component, so
// the group's learning rate and bias corrections are block-uniform.
// HBM-bound: 28 B per scalar (params, m, v read + written, gradient read).
constexpr int kAdamThreads = 256;
__global__ void __launch_bounds__(kAdamThreads) adam_kernel(float* __restrict__ params, const float* __restrict__ grads,
                                                            float* __restrict__ am, float* __restrict__ av,
                                                            int64_t stride, int64_t gstride, int64_t n,
                                                            AdamParams ap, const uint32_t* __restrict__ err) {
  if (__ldg(err)) return;  // see project_bwd_kernel
  const int c = blockIdx.y;
  const int gidx = comp_group(c);
  if (!ap.active[gidx]) return;
  const float lr = ap.lr[gidx], bc1 = ap.bc1[gidx], bc2 = ap.bc2[gidx];
  const int64_t row = (int64_t)c * stride, grow = (int64_t)c * gstride;
  const int64_t nq = n >> 2;
  for (int64_t q = (int64_t)blockIdx.x * kAdamThreads + threadIdx.x; q < nq; q += (int64_t)gridDim.x * kAdamThreads) {
    const int64_t o = row + q * 4;
    float4 p = __ldcs(reinterpret_cast<const float4*>(params + o));
    float4 m = __ldcs(reinterpret_cast<const float4*>(am + o));
    float4 v = __ldcs(reinterpret_cast<const float4*>(av + o));
    const float4 g = __ldcs(reinterpret_cast<const float4*>(grads + grow + q * 4));
    adam_update(p.x, m.x, v.x, g.x, lr, bc1, bc2);
    adam_update(p.y, m.y, v.y, g.y, lr, bc1, bc2);
    adam_update(p.z, m.z, v.z, g.z, lr, bc1, bc2);
    adam_update(p.w, m.w, v.w, g.w, lr, bc1, bc2);
    __stcs(reinterpret_cast<float4*>(params + o), p);
    __stcs(reinterpret_cast<float4*>(am + o), m);
    __stcs(reinterpret_cast<float4*>(av + o), v);
  }
  // ragged tail (n % 4 scalars), one thread per component
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t o = row + nq * 4 + threadIdx.x;
    float p = params[o], m = am[o], v = av[o];
    adam_update(p, m, v, grads[grow + nq * 4 + threadIdx.x], lr, bc1, bc2);
    params[o] = p;
    am[o] = m;
    av[o] = v;
  }
}

// The step's readback (loss sums, pair count, error word) written straight
// into the pinned host slot by the step's last kernel: no copy-engine
// transfers queued behind the step on the stream.
__device__ __forceinline__ void write_readback(const StepReadback& rb) {
  rb.dst[0] = __ldcg(rb.sums);
  rb.dst[1] = __ldcg(rb.sums + 1);
  rb.dst[2] = __ldcg(rb.sums + 2);
  rb.dst[3] = __longlong_as_double(__ldcg(rb.pairs));
  rb.dst[4] = __longlong_as_double((long long)__ldcg(rb.err));
}

// K9 + K10 fused (one GPU, dense Adam): the gradients of a CTA's 128
// Gaussians stay in its shared-memory tile and are consumed there by the
// Adam update of the same Gaussians, so the 59-component gradient buffer is
// neither written nor re-read (2 x 236 B per Gaussian) and the parameters
// the projection backward just read are re-read from L2. Phase 2 streams
// params / m / v as float4 rows (32 lanes x 4 Gaussians = one component row
// of the tile; the four warps take four components, kAdamUnroll rows in
// flight each), so the Adam half runs at HBM rate while the latency-bound
// gradient half of the other resident CTAs overlaps it. Bit-identical to
// K9 followed by K10: the same per-Gaussian gradient code and the same
// adam_update in the same order.
constexpr int kAdamUnroll = 4;  // rows in flight per warp (measured: 2 and 6 slower)
template <int DEG>
__global__ void __launch_bounds__(kPbThreads, kK9MinBlocks) project_bwd_adam_kernel(
    float* __restrict__ params, int64_t stride, int64_t n, CamParams cam, const float* __restrict__ radius,
    const float4* __restrict__ conic4, const float* __restrict__ bg, int64_t gstride, float* __restrict__ am,
    float* __restrict__ av, AdamParams ap, Stats st, bool do_stats, const uint32_t* __restrict__ err,
    StepReadback rb) {
  constexpr int NC = 11 + 3 * (DEG + 1) * (DEG + 1);
  if (rb.dst && blockIdx.x == 0 && threadIdx.x == 0) write_readback(rb);
  if (__ldg(err)) return;  // see project_bwd_kernel
  __shared__ __align__(16) float s_grad[NC * kPbThreads];
  __shared__ float s_exp2[64];
  // per component: (lr, bc1, bc2, active): group lookups off the param struct
  __shared__ float4 s_adam[NC];
  if (threadIdx.x < NC) {
    const int gi = comp_group(threadIdx.x);
    s_adam[threadIdx.x] = make_float4(ap.lr[gi], ap.bc1[gi], ap.bc2[gi], ap.active[gi] ? 1.0f : 0.0f);
  }
  const int64_t i0 = (int64_t)blockIdx.x * kPbThreads;
  const int64_t i = i0 + threadIdx.x;
  stage_exp2_table(s_exp2);
  __syncthreads();
  float* g = s_grad + threadIdx.x;
  if (i < n) {
#pragma unroll
    for (int c = 0; c < 11; ++c) asm volatile("prefetch.global.L1 [%0];" ::"l"(bg + c * gstride + i));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(conic4 + i));
#pragma unroll
    for (int c = 0; c < NC; ++c) asm volatile("prefetch.global.L1 [%0];" ::"l"(params + c * stride + i));
    if (do_stats) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(st.grad_norm_acc + i));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(st.abs_grad_acc + i));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(st.views_seen + i));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(st.max_radius2d + i));
#pragma unroll
      for (int k = 0; k < 3; ++k) asm volatile("prefetch.global.L1 [%0];" ::"l"(st.grad3d_acc + k * stride + i));
    }
    const float rad = radius[i];
    if (rad > 0.0f) {
      float dmu2d[2], dcov[2][2], dcol[3], dop, absg[2];
      load_blend(bg, gstride, i, dmu2d, dcov, conic4[i], dcol, dop, absg);
      project_backward_one<DEG, kPbThreads>(params, stride, i, cam, dmu2d, dcov, dcol, dop, g, s_exp2);
      if (do_stats) {
        const float gmu[3] = {g[0], g[kPbThreads], g[2 * kPbThreads]};
        accumulate_stats(st, i, stride, dmu2d, absg, gmu, rad, (float)cam.width / 2.0f, (float)cam.height / 2.0f);
      }
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) g[c * kPbThreads] = 0.0f;
    }
  }
  __syncthreads();
  // phase 2: Adam over the tile, component rows as float4 along the Gaussians
  const int nloc = (int)(n - i0 < kPbThreads ? n - i0 : kPbThreads);
  const int q = threadIdx.x & 31, wq = threadIdx.x >> 5;  // float4 column, warp
  const int e0 = q * 4;                                     // first Gaussian of the column
  const bool full = e0 + 3 < nloc;
  constexpr int kWarps = kPbThreads / 32;
  for (int cb = 0; cb < NC; cb += kWarps * kAdamUnroll) {
    float4 P[kAdamUnroll], M[kAdamUnroll], V[kAdamUnroll];
#pragma unroll
    for (int u = 0; u < kAdamUnroll; ++u) {
      const int c = cb + wq + kWarps * u;
      if (c < NC && full && s_adam[c].w != 0.0f) {
        const int64_t o = (int64_t)c * stride + i0 + e0;
        P[u] = *reinterpret_cast<const float4*>(params + o);
        M[u] = __ldcs(reinterpret_cast<const float4*>(am + o));
        V[u] = __ldcs(reinterpret_cast<const float4*>(av + o));
      }
    }
#pragma unroll
    for (int u = 0; u < kAdamUnroll; ++u) {
      const int c = cb + wq + kWarps * u;
      if (c >= NC) continue;
      const float4 hp = s_adam[c];
      if (hp.w == 0.0f) continue;
      const float lr = hp.x, bc1 = hp.y, bc2 = hp.z;
      const int64_t o = (int64_t)c * stride + i0 + e0;
      if (full) {
        const float4 G = *reinterpret_cast<const float4*>(s_grad + c * kPbThreads + e0);
        adam_update(P[u].x, M[u].x, V[u].x, G.x, lr, bc1, bc2);
        adam_update(P[u].y, M[u].y, V[u].y, G.y, lr, bc1, bc2);
        adam_update(P[u].z, M[u].z, V[u].z, G.z, lr, bc1, bc2);
        adam_update(P[u].w, M[u].w, V[u].w, G.w, lr, bc1, bc2);
        *reinterpret_cast<float4*>(params + o) = P[u];
        __stcs(reinterpret_cast<float4*>(am + o), M[u]);
        __stcs(reinterpret_cast<float4*>(av + o), V[u]);
      } else {
        for (int e = 0; e < 4 && e0 + e < nloc; ++e) {
          float p = params[o + e], m = am[o + e], v = av[o + e];
          adam_update(p, m, v, s_grad[c * kPbThreads + e0 + e], lr, bc1, bc2);
          params[o + e] = p;
          am[o + e] = m;
          av[o + e] = v;
        }
      }
    }
  }
}

AdamParams make_adam(sk_scene* s, const LearningRates& lrs, float position_lr, bool update_sh_rest) {
  AdamParams ap;
  const float lr[6] = {position_lr, lrs.rotation, lrs.scale, lrs.opacity, lrs.sh_dc, lrs.sh_rest};
  for (int g = 0; g < 6; ++g) {
    const bool active = g < 5 || (update_sh_rest && s->sh_degree > 0);
    ap.active[g] = active ? 1 : 0;
    ap.lr[g] = lr[g];
    if (active) s->adam_t[g] += 1;
    const float t = (float)s->adam_t[g];
    // adam.hpp:64-66: T(1) - std::pow(T(beta), T(t)) in float
    ap.bc1[g] = 1.0f - std::pow((float)0.9, t);
    ap.bc2[g] = 1.0f - std::pow((float)0.999, t);
  }
  return ap;
}

Stats make_stats(sk_scene* s) {
  Stats st;
  st.grad_norm_acc = s->grad_norm_acc.as<float>();
  st.abs_grad_acc = s->abs_grad_acc.as<float>();
  st.grad3d_acc = s->grad3d_acc.as<float>();
  st.views_seen = s->views_seen.as<int>();
  st.max_radius2d = s->max_radius2d.as<float>();
  return st;
}

void launch_pb(sk_ctx* ctx, sk_scene* s, sk_frame* f, bool do_stats) {
  const CamParams cp = make_cam_params(f->camera);
  const unsigned grid = (unsigned)((s->n + kPbThreads - 1) / kPbThreads);
  auto go = [&](auto kern) {
    kern<<<grid, kPbThreads, 0, ctx->stream>>>(s->params.as<float>(), s->capacity, s->n, cp, f->radius.as<float>(),
                                               f->conic4.as<float4>(), f->bgrads.as<float>(), f->n,
                                               s->grads.as<float>(), make_stats(s), do_stats,
                                               ctx->err_word.as<uint32_t>());
  };
  switch (s->sh_degree) {
    case 0: go(project_bwd_kernel<0>); break;
    case 1: go(project_bwd_kernel<1>); break;
    case 2: go(project_bwd_kernel<2>); break;
    default: go(project_bwd_kernel<3>); break;
  }
  note_launch();
  SK_CUDA(cudaGetLastError());
}

}  // namespace

void ensure_optimizer_state(sk_ctx* ctx, sk_scene* s) {
  const size_t cells = (size_t)s->comps * s->capacity;
  if (!s->adam_m.ptr || s->adam_m.bytes < cells * sizeof(float)) {
    ensure<float>(s->adam_m, cells);
    ensure<float>(s->adam_v, cells);
    SK_CUDA(cudaMemsetAsync(s->adam_m.ptr, 0, cells * sizeof(float), ctx->stream));
    SK_CUDA(cudaMemsetAsync(s->adam_v.ptr, 0, cells * sizeof(float), ctx->stream));
  }
  ensure<float>(s->grads, cells);
  ensure_score_table(ctx, s);
}

void ensure_score_table(sk_ctx* ctx, sk_scene* s) {
  const size_t cap = (size_t)s->capacity;
  if (s->grad_norm_acc.ptr && s->grad_norm_acc.bytes >= cap * sizeof(float)) return;
  ensure<float>(s->s_d, cap);
  ensure<float>(s->s_p_raw, cap);
  ensure<float>(s->s_p, cap);
  ensure<float>(s->grad_norm_acc, cap);
  ensure<float>(s->abs_grad_acc, cap);
  ensure<float>(s->grad3d_acc, 3 * cap);
  ensure<int>(s->views_seen, cap);
  ensure<float>(s->max_radius2d, cap);
  reset_score_table(ctx, s);
}

// ScoreTable::reset (adc.hpp:33-42): the ten per-Gaussian rows in one launch.
struct TableRows {
  float4* row[10];
};
__global__ void reset_table_kernel(TableRows t, int64_t quads) {
  const int r = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < quads; i += (int64_t)gridDim.x * blockDim.x)
    t.row[r][i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
}

void reset_score_table(sk_ctx* ctx, sk_scene* s) {
  const int64_t cap = s->capacity;  // a multiple of 32: whole float4s
  TableRows t;
  float4* g3 = s->grad3d_acc.as<float4>();
  DevBuf* rows[7] = {&s->s_d, &s->s_p_raw, &s->s_p, &s->grad_norm_acc, &s->abs_grad_acc, &s->views_seen,
                     &s->max_radius2d};
  for (int k = 0; k < 7; ++k) t.row[k] = rows[k]->as<float4>();
  for (int d = 0; d < 3; ++d) t.row[7 + d] = g3 + d * (cap / 4);
  const int64_t quads = cap / 4;
  reset_table_kernel<<<dim3((unsigned)std::min<int64_t>((quads + 255) / 256, 148), 10), 256, 0, ctx->stream>>>(t, quads);
  note_launch();
  SK_CUDA(cudaGetLastError());
}

void launch_project_backward(sk_ctx* ctx, sk_scene* s, sk_frame* f, bool do_stats) {
  ensure_optimizer_state(ctx, s);
  launch_pb(ctx, s, f, do_stats);
}

namespace {
// K10 over Gaussians [first, first + count) of every component; the
// gradients of that range are row c of `grads` with stride gstride.
void adam_range(sk_ctx* ctx, sk_scene* s, const AdamParams& ap, const float* grads, int64_t gstride, int64_t first,
                int64_t count) {
  if (count <= 0) return;
  // ~16 resident 256-thread blocks per SM spread over the components
  const int64_t per_comp = std::max<int64_t>(1, (int64_t)148 * 16 / s->comps);
  const int64_t need = (count / 4 + kAdamThreads - 1) / kAdamThreads;
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min(need, per_comp)), (unsigned)s->comps);
  adam_kernel<<<grid, kAdamThreads, 0, ctx->stream>>>(s->params.as<float>() + first, grads, s->adam_m.as<float>() + first,
                                                      s->adam_v.as<float>() + first, s->capacity, gstride, count, ap,
                                                      ctx->err_word.as<uint32_t>());
  note_launch();
  SK_CUDA(cudaGetLastError());
}
}  // namespace

void launch_adam(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs, float position_lr, bool update_sh_rest) {
  ensure_optimizer_state(ctx, s);
  require(s->capacity % 4 == 0, "adam: scene capacity must be a multiple of 4");
  const AdamParams ap = make_adam(s, lrs, position_lr, update_sh_rest);
  adam_range(ctx, s, ap, s->grads.as<float>(), s->capacity, 0, s->n);
}

void launch_adam_shard(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs, float position_lr, bool update_sh_rest,
                       const float* gshard, int64_t chunk, int rank) {
  ensure_optimizer_state(ctx, s);
  const AdamParams ap = make_adam(s, lrs, position_lr, update_sh_rest);
  const int64_t first = (int64_t)rank * chunk;
  adam_range(ctx, s, ap, gshard, chunk, first, std::min(chunk, s->n - first));
}

__global__ void accumulate_rest_kernel(float* __restrict__ acc, const float* __restrict__ g, int64_t stride,
                                       int64_t n, int c0, int c1, const uint32_t* __restrict__ err) {
  if (__ldg(err)) return;  // see project_bwd_kernel
  const int c = c0 + blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)c * stride + i;
    acc[o] = acc[o] + g[o];
  }
}

__global__ void reset_opacity_kernel(float* __restrict__ op, float* __restrict__ m, float* __restrict__ v, int64_t n,
                                     float cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = op[i];
  op[i] = (cap < x) ? cap : x;  // std::min(x, cap)
  m[i] = 0.0f;
  v[i] = 0.0f;
}

void lazy_sh_rest(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs, bool due) {
  if (s->sh_degree == 0 || s->n == 0) return;
  const int c0 = SK_COMP_SH + 3, c1 = s->comps;
  const size_t bytes = sizeof(float) * (size_t)s->comps * s->capacity;
  if (s->rest_n != s->n) {  // clear_rest() when the scene size changed
    s->rest_accum.ensure(bytes);
    SK_CUDA(cudaMemsetAsync(s->rest_accum.ptr, 0, bytes, ctx->stream));
    s->rest_n = s->n;
    s->rest_stride = s->capacity;
  } else if (s->rest_stride != s->capacity) {  // same size, re-strided buffers: keep the values
    DevBuf nb;
    nb.ensure(bytes);
    SK_CUDA(cudaMemsetAsync(nb.ptr, 0, bytes, ctx->stream));
    SK_CUDA(cudaMemcpy2DAsync(nb.ptr, sizeof(float) * s->capacity, s->rest_accum.ptr, sizeof(float) * s->rest_stride,
                              sizeof(float) * s->n, s->comps, cudaMemcpyDeviceToDevice, ctx->stream));
    s->rest_accum.swap(nb);
    s->rest_stride = s->capacity;
  }
  const dim3 grid((unsigned)std::min<int64_t>((s->n + 255) / 256, 64), (unsigned)(c1 - c0));
  accumulate_rest_kernel<<<grid, 256, 0, ctx->stream>>>(s->rest_accum.as<float>(), s->grads.as<float>(), s->capacity,
                                                        s->n, c0, c1, ctx->err_word.as<uint32_t>());
  note_launch();
  SK_CUDA(cudaGetLastError());
  if (!due) return;
  // SceneOptimizer::step_sh_rest: the SH-rest group alone, on the accumulator
  AdamParams ap = make_adam(s, lrs, 0.0f, true);
  for (int g = 0; g < 5; ++g) {
    if (ap.active[g]) s->adam_t[g] -= 1;  // make_adam counted every group; only SH-rest steps here
    ap.active[g] = 0;
  }
  adam_range(ctx, s, ap, s->rest_accum.as<float>(), s->capacity, 0, s->n);
  SK_CUDA(cudaMemsetAsync(s->rest_accum.ptr, 0, bytes, ctx->stream));
}

void reset_opacity(sk_ctx* ctx, sk_scene* s) {
  ensure_optimizer_state(ctx, s);
  if (s->n == 0) return;
  const float cap = std::log(0.01f / (1.0f - 0.01f));  // logit(T(0.01)), host libm as the reference
  const int64_t o = (int64_t)SK_COMP_OPACITY * s->capacity;
  reset_opacity_kernel<<<(unsigned)((s->n + 255) / 256), 256, 0, ctx->stream>>>(
      s->params.as<float>() + o, s->adam_m.as<float>() + o, s->adam_v.as<float>() + o, s->n, cap);
  note_launch();
  SK_CUDA(cudaGetLastError());
}

void launch_project_backward_explicit(sk_ctx* ctx, sk_scene* s, const sk_camera& cam, const float* up_mu,
                                      const float* up_cov, const float* up_col, const float* up_op) {
  ensure_optimizer_state(ctx, s);
  if (s->n == 0) return;
  const CamParams cp = make_cam_params(cam);
  const unsigned grid = (unsigned)((s->n + kPbThreads - 1) / kPbThreads);
  auto go = [&](auto kern) {
    kern<<<grid, kPbThreads, 0, ctx->stream>>>(s->params.as<float>(), s->capacity, s->n, cp, up_mu, up_cov, up_col,
                                               up_op, s->grads.as<float>());
  };
  switch (s->sh_degree) {
    case 0: go(project_bwd_explicit_kernel<0>); break;
    case 1: go(project_bwd_explicit_kernel<1>); break;
    case 2: go(project_bwd_explicit_kernel<2>); break;
    default: go(project_bwd_explicit_kernel<3>); break;
  }
  note_launch();
  SK_CUDA(cudaGetLastError());
}

void remap_moments(sk_ctx* ctx, sk_scene* s, const int32_t* old_to_new_dev, int64_t new_n) {
  ensure_optimizer_state(ctx, s);
  const int64_t new_cap = std::max(s->capacity, round_capacity(new_n));
  const size_t cells = (size_t)s->comps * new_cap;
  DevBuf& nm = s->adam_m_alt;
  DevBuf& nv = s->adam_v_alt;
  ensure<float>(nm, cells);
  ensure<float>(nv, cells);
  SK_CUDA(cudaMemsetAsync(nm.ptr, 0, cells * sizeof(float), ctx->stream));
  SK_CUDA(cudaMemsetAsync(nv.ptr, 0, cells * sizeof(float), ctx->stream));
  if (s->n > 0) {
    remap_moments_kernel<<<dim3((unsigned)((s->n + 255) / 256), (unsigned)s->comps), 256, 0, ctx->stream>>>(
        s->adam_m.as<float>(), s->adam_v.as<float>(), s->capacity, s->n, old_to_new_dev, nm.as<float>(),
        nv.as<float>(), new_cap);
    note_launch();
    SK_CUDA(cudaGetLastError());
  }
  s->adam_m.swap(nm);
  s->adam_v.swap(nv);
  if (new_cap != s->capacity) {
    // the parameter buffer follows the new stride (its values are replaced by
    // the caller's next sk_scene_set_params)
    DevBuf np;
    ensure<float>(np, cells);
    s->params.swap(np);
    s->capacity = new_cap;
    s->grads.release();
    for (DevBuf* b : {&s->s_d, &s->s_p_raw, &s->s_p, &s->grad_norm_acc, &s->abs_grad_acc, &s->grad3d_acc,
                      &s->views_seen, &s->max_radius2d})
      b->release();
  }
  s->n = new_n;
  s->rest_n = -1;
  ensure_optimizer_state(ctx, s);
}

void adam_step_sh_rest(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs) {
  ensure_optimizer_state(ctx, s);
  if (s->sh_degree == 0) return;
  // SceneOptimizer::step_sh_rest (adam.hpp:146-153): the SH-rest group alone
  AdamParams ap = make_adam(s, lrs, 0.0f, true);
  for (int g = 0; g < 5; ++g) {
    if (ap.active[g]) s->adam_t[g] -= 1;
    ap.active[g] = 0;
  }
  adam_range(ctx, s, ap, s->grads.as<float>(), s->capacity, 0, s->n);
}

void reset_opacity_state(sk_ctx* ctx, sk_scene* s) {
  ensure_optimizer_state(ctx, s);
  const size_t o = (size_t)SK_COMP_OPACITY * s->capacity;
  SK_CUDA(cudaMemsetAsync(s->adam_m.as<float>() + o, 0, sizeof(float) * s->capacity, ctx->stream));
  SK_CUDA(cudaMemsetAsync(s->adam_v.as<float>() + o, 0, sizeof(float) * s->capacity, ctx->stream));
}

// Single-GPU step: K9 and K10 fused (project_bwd_adam_kernel). The gradient
// buffer is not written.
void launch_project_backward_adam(sk_ctx* ctx, sk_scene* s, sk_frame* f, const LearningRates& lrs, float position_lr,
                                  bool update_sh_rest, bool do_stats, const StepReadback& rb) {
  ensure_optimizer_state(ctx, s);
  require(s->capacity % 4 == 0, "adam: scene capacity must be a multiple of 4");
  const AdamParams ap = make_adam(s, lrs, position_lr, update_sh_rest);
  if (s->n == 0) return;
  const CamParams cp = make_cam_params(f->camera);
  const unsigned grid = (unsigned)((s->n + kPbThreads - 1) / kPbThreads);
  auto go = [&](auto kern) {
    kern<<<grid, kPbThreads, 0, ctx->stream>>>(s->params.as<float>(), s->capacity, s->n, cp, f->radius.as<float>(),
                                               f->conic4.as<float4>(), f->bgrads.as<float>(), f->n,
                                               s->adam_m.as<float>(), s->adam_v.as<float>(), ap, make_stats(s),
                                               do_stats, ctx->err_word.as<uint32_t>(), rb);
  };
  switch (s->sh_degree) {
    case 0: go(project_bwd_adam_kernel<0>); break;
    case 1: go(project_bwd_adam_kernel<1>); break;
    case 2: go(project_bwd_adam_kernel<2>); break;
    default: go(project_bwd_adam_kernel<3>); break;
  }
  note_launch();
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
