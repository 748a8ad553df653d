// Shared by the forward (rasterize.cu) and backward (rasterize_bwd.cu) blend
// kernels: the exact early-reject cut, the staged-entry ellipse box and the
// warp pixel block used for warp-uniform culling.
#pragma once

#include "state.h"

namespace sk {
namespace blend {

__device__ __forceinline__ float qcut_of(float opacity) {
  const float a = 255.0f * opacity;
  return a > 1.0f ? 2.0f * __logf(a) + 0.02f : -1.0f;
}

// Staged entry: position + q_cut, conic + opacity, box of {q <= q_cut}.
__device__ __forceinline__ void stage_entry(float2 mu, float4 co, float4& xyq, float4& bb) {
  const float qc = qcut_of(co.w);
  xyq = make_float4(mu.x, mu.y, qc, 0.0f);
  if (qc <= 0.0f) {
    bb = make_float4(1.0f, -1.0f, 1.0f, -1.0f);  // empty: never contributes
    return;
  }
  const float det = co.x * co.z - co.y * co.y;
  if (!(det > 0.0f && co.x > 0.0f && co.z > 0.0f)) {
    bb = make_float4(-3.0e38f, 3.0e38f, -3.0e38f, 3.0e38f);  // no culling
    return;
  }
  const float ex = sqrtf(qc * co.z / det) * 1.0001f + 0.01f;
  const float ey = sqrtf(qc * co.x / det) * 1.0001f + 0.01f;
  bb = make_float4(mu.x - ex, mu.x + ex, mu.y - ey, mu.y + ey);
}

template <int TS, int PIX>
struct WarpBlock {
  static constexpr int kWarpsX = TS / 8;
  int lx, ly0;    // pixel of k = 0 within the tile
  float x0, x1, y0, y1;  // the warp's pixel-centre rectangle (absolute)
  __device__ WarpBlock(int tx, int ty) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int bx = (w % kWarpsX) * 8, by = (w / kWarpsX) * (4 * PIX);
    lx = bx + (l & 7);
    ly0 = by + (l >> 3);
    x0 = (float)(tx * TS + bx);
    x1 = x0 + 7.0f;
    y0 = (float)(ty * TS + by);
    y1 = y0 + (float)(4 * PIX - 1);
  }
  __device__ bool misses(const float4& bb) const { return bb.y < x0 || bb.x > x1 || bb.w < y0 || bb.z > y1; }
};

}  // namespace blend
}  // namespace sk
