// Shared by the forward (rasterize.cu) and backward (rasterize_bwd.cu) blend
// kernels: the exact early-reject cut, the staged-entry ellipse box and the
// warp pixel block used for warp-uniform culling.
#pragma once

#include "state.h"

namespace sk {
namespace blend {

// cp.async (LDGSTS) helpers: global -> shared copies that hold no registers
// while in flight.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
// 2^x on MUFU.EX2 (the hardware exp __expf uses, without its pre-multiply)
__device__ __forceinline__ float exp2f_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Contribution-mask words (K6 -> K8): batch b of tile t (entries
// [range.x + 32 b, +32)) lives at word cmask_word(range.x, t) + b, times the
// number of K6 warps per tile. floor(begin / 32) + t never collides between
// tiles: tile t has at most floor(L / 32) + 1 batches.
__host__ __device__ __forceinline__ int64_t cmask_word(int begin, int tile) { return (int64_t)(begin >> 5) + tile; }
inline size_t cmask_words(int64_t pairs, int tiles) { return (size_t)(pairs >> 5) + (size_t)tiles + 2; }

__device__ __forceinline__ float cull_sqrt(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float cull_div(float a, float b) {
  return __fdividef(a, b);
}

// FAST (training-step) form of q for a pixel pair sharing the column
// (dx) and differing in row (dy = (dy0, dy1)): q = A + dy (B + c11 dy) with
// A = (c00 dx) dx, B = (2 c01) dx, in two packed FMAs. K6 and K8 form it with
// these same instructions, so their contribution decisions agree bit for bit.
__device__ __forceinline__ float2 fast_pair_q(float2 dy, float c11, float A, float B) {
  return __ffma2_rn(dy, __ffma2_rn(make_float2(c11, c11), dy, make_float2(B, B)), make_float2(A, A));
}

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
  const float ex = cull_sqrt(cull_div(qc * co.z, det)) * 1.0001f + 0.01f;
  const float ey = cull_sqrt(cull_div(qc * co.x, det)) * 1.0001f + 0.01f;
  bb = make_float4(mu.x - ex, mu.x + ex, mu.y - ey, mu.y + ey);
}

// Warp w of a TS x TS tile owns the 8 x 4·PIX pixel block starting at
// ((w % (TS/8)) * 8, (w / (TS/8)) * 4·PIX); lane l holds column l & 7 and rows
// (l >> 3) + 4k, k < PIX.
template <int TS, int PIX>
struct WarpBlock {
  static constexpr int kWarpsX = TS / 8;
  static constexpr int kWarps = TS * TS / PIX / 32;
  int lx, ly0;  // pixel of k = 0 within the tile
  __device__ WarpBlock() {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    lx = (w % kWarpsX) * 8 + (l & 7);
    ly0 = (w / kWarpsX) * (4 * PIX) + (l >> 3);
  }
  // true when warp w's pixel-centre rectangle misses the box bb
  __device__ static bool misses(const float4& bb, int w, int tx, int ty) {
    const float x0 = (float)(tx * TS + (w % kWarpsX) * 8);
    const float y0 = (float)(ty * TS + (w / kWarpsX) * (4 * PIX));
    return bb.y < x0 || bb.x > x0 + 7.0f || bb.w < y0 || bb.z > y0 + (float)(4 * PIX - 1);
  }
  // Exact test: does the ellipse {q <= q_cut} (conic co, centre mq.xy, cut
  // mq.z) reach a pixel centre of warp w's rectangle? The minimum of the
  // convex q over the rectangle is 0 inside it, else on an edge, where the
  // unconstrained minimiser along the edge is clamped to the edge. Slack of
  // 1e-3 relative + 1e-3 absolute keeps the test conservative under fp32
  // rounding. Only called for positive-definite conics with a box hit.
  __device__ static bool ellipse_hits(const float4& mq, const float4& co, int w, int tx, int ty) {
    const float x0 = (float)(tx * TS + (w % kWarpsX) * 8), x1 = x0 + 7.0f;
    const float y0 = (float)(ty * TS + (w / kWarpsX) * (4 * PIX)), y1 = y0 + (float)(4 * PIX - 1);
    if (mq.x >= x0 && mq.x <= x1 && mq.y >= y0 && mq.y <= y1) return true;
    const float a = co.x, b = co.y, c = co.z;
    const float ia = cull_div(1.0f, a), ic = cull_div(1.0f, c);
    float best = 3.0e38f;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float dx = (e ? x1 : x0) - mq.x;
      const float dy = fminf(fmaxf(mq.y - b * dx * ic, y0), y1) - mq.y;
      best = fminf(best, a * dx * dx + 2.0f * b * dx * dy + c * dy * dy);
      const float ey = (e ? y1 : y0) - mq.y;
      const float ex = fminf(fmaxf(mq.x - b * ey * ia, x0), x1) - mq.x;
      best = fminf(best, a * ex * ex + 2.0f * b * ex * ey + c * ey * ey);
    }
    return best <= mq.z * 1.001f + 1e-3f;
  }
  // Called by every lane of a staging warp for entry `chunk * 32 + lane` of the
  // batch: publishes, per compute warp, the 32-bit mask of the chunk's entries
  // whose ellipse reaches that warp's block (s_mask[w * chunks + chunk]). The
  // box test rejects most; the exact test runs on box hits of PD conics.
  __device__ static void publish(const float4& bb, const float4& mq, const float4& co, bool valid, int chunk,
                                 int chunks, int tx, int ty, uint32_t* s_mask) {
    const bool pd = co.x > 0.0f && co.z > 0.0f && co.x * co.z - co.y * co.y > 0.0f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      bool hit = valid && !misses(bb, w, tx, ty);
      if (hit && pd) hit = ellipse_hits(mq, co, w, tx, ty);
      const uint32_t bits = __ballot_sync(0xffffffffu, hit);
      if ((threadIdx.x & 31) == 0) s_mask[w * chunks + chunk] = bits;
    }
  }
};

}  // namespace blend
}  // namespace sk
