// K6 forward alpha blend (+ K12 footprint count) and K8 backward blend.
//
// K6 restates blend_forward (reference raster.hpp:194-248): integer pixel
// centres, q = ((c00 dx) dx + ((2 c01) dx) dy) + (c11 dy) dy, skip q < 0,
// alpha = min(0.99, o e^{-q/2}), skip alpha < 1/255, C += (T alpha) c,
// T *= 1 - alpha, and the entry that takes T below 1e-4 is blended before the
// pixel stops. One CTA per tile; the tile's list is staged through shared
// memory in CTA-sized batches and the CTA stops loading once every pixel has
// terminated. Compiled with -fmad=false and the shared deterministic exp, so
// images, transmittance and footprint counts match the CPU oracle bit for bit.
//
// Exact early rejects. alpha >= 1/255 requires q <= 2 ln(255 o); each staged
// entry carries q_cut = 2 ln(255 o) + 0.02 and the bounding box of the ellipse
// {q <= q_cut} (widened by 1e-4 relative + 0.01 px). Outside q_cut the
// reference's alpha is below 1/255 by a 1% margin (far above the 2-ulp exp
// error), so skipping changes no result. Warps own 8-pixel-wide blocks of the
// tile; a warp whose block misses an entry's box skips that entry with one
// warp-uniform test instead of evaluating 32 pixels.
//
// K8 restates blend_backward (raster.hpp:281-355) as a reverse walk from each
// pixel's last contributor (recorded by K6): T_before = T_after / (1 - alpha),
// suffix accumulated in the reference's reverse order, capped entries feed
// d_color only. Each thread owns PIX pixels (rows y, y+4, ...) of its warp's
// 8 x 4·PIX block, sums their partials per Gaussian in registers, and the warp
// then butterfly-reduces the 11 partials with shuffles (skipped when no lane
// contributes); lanes 0..10 issue one global atomic each.
#include "state.h"

namespace sk {
namespace {

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

template <int TS, int PIX, bool COUNT>
__global__ void __launch_bounds__(TS* TS / PIX, 8) blend_fwd_kernel(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ pair_val, const float2* __restrict__ mean2d,
    const float4* __restrict__ conic_op, const float4* __restrict__ rgbd, int W, int H, int tiles_x,
    float* __restrict__ image, float* __restrict__ final_t, int* __restrict__ n_contrib, int* __restrict__ last_entry,
    const uint8_t* __restrict__ mask, int* __restrict__ counts) {
  constexpr int NTH = TS * TS / PIX;        // threads; each owns PIX pixels
  constexpr int B = TS * TS > 256 ? 256 : TS * TS;  // staged entries per batch
  __shared__ float4 s_xyq[B];
  __shared__ float4 s_co[B];
  __shared__ float4 s_bb[B];
  __shared__ float4 s_rgb[COUNT ? 1 : B];
  __shared__ uint32_t s_id[COUNT ? B : 1];
  __shared__ float s_exp2[64];
  stage_exp2_table(s_exp2);  // published by the first __syncthreads_count below

  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const WarpBlock<TS, PIX> wb(tx, ty);
  const int px = tx * TS + wb.lx;
  const int2 range = ranges[tile];
  const float fpx = (float)px;

  float T[PIX], C0[PIX], C1[PIX], C2[PIX], fpy[PIX];
  int n[PIX], last[PIX];
  bool done[PIX];
  bool all_done = true;
#pragma unroll
  for (int k = 0; k < PIX; ++k) {
    const int py = ty * TS + wb.ly0 + 4 * k;
    fpy[k] = (float)py;
    T[k] = 1.0f;
    C0[k] = C1[k] = C2[k] = 0.0f;
    n[k] = last[k] = 0;
    const bool inside = px < W && py < H;
    // K12 (count-only pass): only masked pixels can increment a counter, so
    // unmasked pixels never traverse and fully unmasked tiles exit at once.
    done[k] = COUNT ? !(inside && mask[(size_t)py * W + px] != 0) : !inside;
    all_done = all_done && done[k];
  }

  for (int b0 = range.x; b0 < range.y; b0 += B) {
    if (__syncthreads_count(all_done) == NTH) break;
    for (int e = (int)threadIdx.x; e < B; e += NTH) {
      const int i = b0 + e;
      if (i < range.y) {
        const uint32_t g = pair_val[i];
        const float4 co = conic_op[g];
        float4 xyq, bb;
        stage_entry(mean2d[g], co, xyq, bb);
        s_xyq[e] = xyq;
        s_co[e] = co;
        s_bb[e] = bb;
        if (!COUNT) s_rgb[e] = rgbd[g];
        if (COUNT) s_id[e] = g;
      }
    }
    __syncthreads();
    const int cnt = min(B, range.y - b0);
    for (int j = 0; j < cnt && !all_done; ++j) {
      if (wb.misses(s_bb[j])) continue;  // warp-uniform
      const float4 mq = s_xyq[j];
      const float4 co = s_co[j];
#pragma unroll
      for (int k = 0; k < PIX; ++k) {
        const float dx = fpx - mq.x;
        const float dy = fpy[k] - mq.y;
        const float q = co.x * dx * dx + 2.0f * co.y * dx * dy + co.z * dy * dy;
        if (done[k] || !(q >= 0.0f && q <= mq.z)) continue;
        // -0.5 q lies in [-q_cut/2, 0], inside det_expf's core range
        float alpha = co.w * det_expf_core(-0.5f * q, s_exp2);
        alpha = (alpha < kAlphaCap) ? alpha : kAlphaCap;
        if (alpha < kAlphaMin) continue;
        if (COUNT) {
          // warp-aggregated increment: one atomic per distinct Gaussian
          const uint32_t id = s_id[j];
          const uint32_t act = __activemask();
          const uint32_t peers = __match_any_sync(act, id);
          if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&counts[id], __popc(peers));
        } else {
          const float4 c = s_rgb[j];
          const float w = T[k] * alpha;
          C0[k] = C0[k] + w * c.x;
          C1[k] = C1[k] + w * c.y;
          C2[k] = C2[k] + w * c.z;
          ++n[k];
          last[k] = b0 + j + 1;
        }
        T[k] = T[k] * (1.0f - alpha);
        if (T[k] < kTransmitMin) done[k] = true;
      }
      bool ad = true;
#pragma unroll
      for (int k = 0; k < PIX; ++k) ad = ad && done[k];
      all_done = ad;
    }
  }
  if (COUNT) return;
#pragma unroll
  for (int k = 0; k < PIX; ++k) {
    const int py = ty * TS + wb.ly0 + 4 * k;
    if (px < W && py < H) {
      const size_t p = (size_t)py * W + px;
      const size_t plane = (size_t)W * H;
      image[p] = C0[k];
      image[plane + p] = C1[k];
      image[2 * plane + p] = C2[k];
      final_t[p] = T[k];
      n_contrib[p] = n[k];
      last_entry[p] = last[k];
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float select_field(const float (&v)[kBGradFields], int f) {
  float r = v[0];
#pragma unroll
  for (int k = 1; k < kBGradFields; ++k) r = f == k ? v[k] : r;
  return r;
}

template <int TS, int PIX>
__global__ void __launch_bounds__(TS* TS / PIX) blend_bwd_kernel(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ pair_val, const float2* __restrict__ mean2d,
    const float4* __restrict__ conic_op, const float4* __restrict__ rgbd, int W, int H, int tiles_x,
    const float* __restrict__ final_t, const int* __restrict__ last_entry, const float* __restrict__ dimage,
    float* __restrict__ bgrads, int64_t gstride) {
  constexpr int NT = TS * TS / PIX;  // threads == batch size
  __shared__ float4 s_xyq[NT];
  __shared__ float4 s_co[NT];
  __shared__ float4 s_bb[NT];
  __shared__ float4 s_rgb[NT];
  __shared__ uint32_t s_id[NT];
  __shared__ int s_max_last;
  __shared__ float s_exp2[64];
  stage_exp2_table(s_exp2);

  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const WarpBlock<TS, PIX> wb(tx, ty);
  const int lane = threadIdx.x & 31;
  const int px = tx * TS + wb.lx;
  const int2 range = ranges[tile];
  const float fpx = (float)px;
  const size_t plane = (size_t)W * H;

  float T[PIX], suffix[PIX], d0[PIX], d1[PIX], d2[PIX], fpy[PIX];
  int last[PIX];
  int my_last = 0;
#pragma unroll
  for (int k = 0; k < PIX; ++k) {
    const int py = ty * TS + wb.ly0 + 4 * k;
    fpy[k] = (float)py;
    T[k] = 1.0f;
    suffix[k] = 0.0f;
    d0[k] = d1[k] = d2[k] = 0.0f;
    last[k] = 0;
    if (px < W && py < H) {
      const size_t p = (size_t)py * W + px;
      T[k] = final_t[p];
      last[k] = last_entry[p];
      d0[k] = dimage[p];
      d1[k] = dimage[plane + p];
      d2[k] = dimage[2 * plane + p];
    }
    my_last = max(my_last, last[k]);
  }
  if (threadIdx.x == 0) s_max_last = 0;
  __syncthreads();
  atomicMax(&s_max_last, my_last);
  __syncthreads();
  const int end = s_max_last;  // no pixel of the tile uses entries >= end
  const int warp_last = __reduce_max_sync(0xffffffffu, my_last);
  float pend[kBGradFields];
  uint32_t pend_id = 0;
  bool has_pend = false;

  for (int b_end = end; b_end > range.x; b_end -= NT) {
    const int b0 = max(range.x, b_end - NT);
    __syncthreads();
    const int i = b0 + (int)threadIdx.x;
    if (i < b_end) {
      const uint32_t g = pair_val[i];
      const float4 co = conic_op[g];
      float4 xyq, bb;
      stage_entry(mean2d[g], co, xyq, bb);
      s_xyq[threadIdx.x] = xyq;
      s_co[threadIdx.x] = co;
      s_bb[threadIdx.x] = bb;
      s_rgb[threadIdx.x] = rgbd[g];
      s_id[threadIdx.x] = g;
    }
    __syncthreads();
    const int jmax = min(b_end, warp_last) - b0;  // warp-uniform
    for (int j = jmax - 1; j >= 0; --j) {
      if (wb.misses(s_bb[j])) continue;  // warp-uniform
      const int idx = b0 + j;
      const float4 mq = s_xyq[j];
      const float4 co = s_co[j];
      float g_mu0 = 0.f, g_mu1 = 0.f, g_c00 = 0.f, g_c01 = 0.f, g_c11 = 0.f, g_r = 0.f, g_g = 0.f, g_b = 0.f,
            g_op = 0.f, g_a0 = 0.f, g_a1 = 0.f;
      bool contrib = false;
#pragma unroll
      for (int k = 0; k < PIX; ++k) {
        if (idx >= last[k]) continue;
        const float dx = fpx - mq.x;
        const float dy = fpy[k] - mq.y;
        const float q = co.x * dx * dx + 2.0f * co.y * dx * dy + co.z * dy * dy;
        if (!(q >= 0.0f && q <= mq.z)) continue;
        const float ge = det_expf_core(-0.5f * q, s_exp2);
        const float raw = co.w * ge;
        const bool capped = raw > kAlphaCap;
        const float alpha = capped ? kAlphaCap : raw;
        if (alpha < kAlphaMin) continue;
        contrib = true;
        const float4 c = s_rgb[j];
        const float one_m = 1.0f - alpha;
        const float inv_one_m = __frcp_rn(one_m);  // tolerance path: one reciprocal, two products
        const float t_before = T[k] * inv_one_m;
        T[k] = t_before;
        const float w = (c.x * d0[k] + c.y * d1[k]) + c.z * d2[k];
        const float d_alpha = t_before * w - suffix[k] * inv_one_m;
        const float ta = t_before * alpha;
        suffix[k] = suffix[k] + ta * w;
        g_r += ta * d0[k];
        g_g += ta * d1[k];
        g_b += ta * d2[k];
        if (!capped) {
          g_op += ge * d_alpha;
          const float d_q = -0.5f * alpha * d_alpha;
          g_c00 += d_q * (dx * dx);
          g_c01 += d_q * (dx * dy);
          g_c11 += d_q * (dy * dy);
          const float v0 = co.x * dx + co.y * dy;
          const float v1 = co.y * dx + co.z * dy;
          const float m0 = (-2.0f * d_q) * v0;
          const float m1 = (-2.0f * d_q) * v1;
          g_mu0 += m0;
          g_mu1 += m1;
          g_a0 += fabsf(m0);
          g_a1 += fabsf(m1);
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
        const float gv[kBGradFields] = {g_mu0, g_mu1, g_c00, g_c01, g_c11, g_r, g_g, g_b, g_op, g_a0, g_a1};
        if (has_pend) {
          // Two entries per reduction: the xor-16 stage hands the pending
          // entry to lanes 0-15 and the current one to lanes 16-31, then four
          // butterfly stages finish both (55 shuffles for 22 values).
          float keep[kBGradFields];
#pragma unroll
          for (int f = 0; f < kBGradFields; ++f) {
            const float give = lane < 16 ? gv[f] : pend[f];
            const float mine = lane < 16 ? pend[f] : gv[f];
            keep[f] = mine + __shfl_xor_sync(0xffffffffu, give, 16);
          }
#pragma unroll
          for (int o = 8; o > 0; o >>= 1)
#pragma unroll
            for (int f = 0; f < kBGradFields; ++f) keep[f] += __shfl_xor_sync(0xffffffffu, keep[f], o);
          const int fl = lane & 15;
          if (fl < kBGradFields)
            atomicAdd(&bgrads[(int64_t)fl * gstride + (lane < 16 ? pend_id : s_id[j])], select_field(keep, fl));
          has_pend = false;
        } else {
#pragma unroll
          for (int f = 0; f < kBGradFields; ++f) pend[f] = gv[f];
          pend_id = s_id[j];
          has_pend = true;
        }
      }
    }
  }
  if (has_pend) {  // warp-uniform: flush the last unpaired entry
#pragma unroll
    for (int f = 0; f < kBGradFields; ++f) pend[f] = warp_sum(pend[f]);
    if (lane < kBGradFields) atomicAdd(&bgrads[(int64_t)lane * gstride + pend_id], select_field(pend, lane));
  }
}

template <int TS, int PIX>
void fwd_dispatch(sk_ctx* ctx, sk_frame* f, const uint8_t* mask, int32_t* counts) {
  const int tiles = f->tiles_x * f->tiles_y;
  auto* ranges = f->ranges.as<int2>();
  const auto* mean2d = f->mean2d.as<float2>();
  const auto* co = f->conic_op.as<float4>();
  const auto* rgb = f->rgb_depth.as<float4>();
  if (mask)
    blend_fwd_kernel<TS, PIX, true><<<tiles, TS * TS / PIX, 0, ctx->stream>>>(
        ranges, f->pair_val, mean2d, co, rgb, f->width, f->height, f->tiles_x, f->image.as<float>(),
        f->final_t.as<float>(), f->n_contrib.as<int>(), f->last_entry.as<int>(), mask, counts);
  else
    blend_fwd_kernel<TS, PIX, false><<<tiles, TS * TS / PIX, 0, ctx->stream>>>(
        ranges, f->pair_val, mean2d, co, rgb, f->width, f->height, f->tiles_x, f->image.as<float>(),
        f->final_t.as<float>(), f->n_contrib.as<int>(), f->last_entry.as<int>(), nullptr, nullptr);
  note_launch();
}

template <int TS, int PIX>
void bwd_dispatch(sk_ctx* ctx, sk_frame* f) {
  const int tiles = f->tiles_x * f->tiles_y;
  blend_bwd_kernel<TS, PIX><<<tiles, TS * TS / PIX, 0, ctx->stream>>>(
      f->ranges.as<int2>(), f->pair_val, f->mean2d.as<float2>(), f->conic_op.as<float4>(), f->rgb_depth.as<float4>(),
      f->width, f->height, f->tiles_x, f->final_t.as<float>(), f->last_entry.as<int>(), f->dimage.as<float>(),
      f->bgrads.as<float>(), f->n);
  note_launch();
}

}  // namespace

void launch_blend_forward(sk_ctx* ctx, sk_frame* f, const uint8_t* mask, int32_t* counts) {
  if (f->tiles_x * f->tiles_y == 0) return;
  switch (f->tile_size) {
    case 8: fwd_dispatch<8, 1>(ctx, f, mask, counts); break;
    case 16: fwd_dispatch<16, 2>(ctx, f, mask, counts); break;
    case 32: fwd_dispatch<32, 4>(ctx, f, mask, counts); break;
    default: throw std::invalid_argument("tile_size must be 8, 16 or 32");
  }
  SK_CUDA(cudaGetLastError());
}

void launch_blend_backward(sk_ctx* ctx, sk_frame* f) {
  SK_CUDA(cudaMemsetAsync(f->bgrads.ptr, 0, sizeof(float) * kBGradFields * (size_t)f->n, ctx->stream));
  if (f->tiles_x * f->tiles_y == 0) return;
  switch (f->tile_size) {
    case 8: bwd_dispatch<8, 1>(ctx, f); break;
    case 16: bwd_dispatch<16, 2>(ctx, f); break;
    case 32: bwd_dispatch<32, 4>(ctx, f); break;
    default: throw std::invalid_argument("tile_size must be 8, 16 or 32");
  }
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
