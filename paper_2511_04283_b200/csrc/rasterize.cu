// K6 forward alpha blend (+ K12 footprint count).
//
// K6 restates blend_forward (reference raster.hpp:194-248): integer pixel
// centres, q = ((c00 dx) dx + ((2 c01) dx) dy) + (c11 dy) dy, skip q < 0,
// alpha = min(0.99, o e^{-q/2}), skip alpha < 1/255, C += (T alpha) c,
// T *= 1 - alpha, and the entry that takes T below 1e-4 is blended before the
// pixel stops. One CTA per tile; each warp walks the tile's list for its own
// pixel block (blend_fwd_warp_kernel) and stops once its pixels have
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
// K8 (the backward walk) lives in rasterize_bwd.cu.
#include "blend_common.cuh"

namespace sk {
namespace {

using namespace blend;

constexpr int kFwdMinBlocks = 8;  // resident 128-thread CTAs per SM (64 registers)

// K12: blend_forward(grid, pgs, &mask, &counter) (raster.hpp:194-248) as a
// count-only pass: the forward recurrence (same decisions, bit for bit, as
// K6) over masked pixels only, incrementing the counter of every Gaussian a
// masked pixel blends. One CTA per tile stages the list in CTA-sized batches;
// unmasked pixels never traverse and fully unmasked tiles exit at once.
template <int TS, int PIX>
__global__ void __launch_bounds__(TS* TS / PIX, 1024 / (TS * TS / PIX)) count_blend_kernel(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ pair_val, const float2* __restrict__ mean2d,
    const float4* __restrict__ conic_op, int W, int H, int tiles_x, const uint8_t* __restrict__ mask,
    int* __restrict__ counts, const uint32_t* __restrict__ err) {
  if (err && __ldg(err)) return;  // see blend_fwd_warp_kernel
  constexpr int NTH = TS * TS / PIX;                // threads; each owns PIX pixels
  constexpr int B = TS * TS > 256 ? 256 : TS * TS;  // staged entries per batch
  using WB = WarpBlock<TS, PIX>;
  constexpr int kChunks = B / 32;
  __shared__ float4 s_xyq[B];
  __shared__ float4 s_co[B];
  __shared__ uint32_t s_mask[WB::kWarps * kChunks];
  __shared__ uint32_t s_id[B];
  __shared__ float s_exp[kNegExpTable];
  stage_neg_exp_table(s_exp);  // published by the first __syncthreads_count below
  const SmemPinnedTable tab(s_exp);

  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const WB wb;
  const int warp = threadIdx.x >> 5;
  const int px = tx * TS + wb.lx;
  const int2 range = ranges[tile];
  const float fpx = (float)px;

  float T[PIX], fpy[PIX];
  bool done[PIX];
  bool all_done = true;
#pragma unroll
  for (int k = 0; k < PIX; ++k) {
    const int py = ty * TS + wb.ly0 + 4 * k;
    fpy[k] = (float)py;
    T[k] = 1.0f;
    done[k] = !(px < W && py < H && mask[(size_t)py * W + px] != 0);
    all_done = all_done && done[k];
  }

  for (int b0 = range.x; b0 < range.y; b0 += B) {
    if (__syncthreads_count(all_done) == NTH) break;
    for (int e = (int)threadIdx.x; e < B; e += NTH) {
      const int i = b0 + e;
      const bool valid = i < range.y;
      float4 bb = make_float4(1.0f, -1.0f, 1.0f, -1.0f), xyq = bb, co = bb;
      if (valid) {
        const uint32_t g = pair_val[i];
        co = conic_op[g];
        stage_entry(mean2d[g], co, xyq, bb);
        s_xyq[e] = xyq;
        s_co[e] = co;
        s_id[e] = g;
      }
      WB::publish(bb, xyq, co, valid, e >> 5, kChunks, tx, ty, s_mask);
    }
    __syncthreads();
    // Walk, in list order, only the entries whose box touches this warp's
    // block (bit masks published at staging).
    for (int c = 0; c < kChunks && !all_done; ++c) {
      uint32_t m = s_mask[warp * kChunks + c];
      while (m && !all_done) {
        const int j = c * 32 + __ffs(m) - 1;
        m &= m - 1;
        const float4 mq = s_xyq[j];
        const float4 co = s_co[j];
#pragma unroll
        for (int k = 0; k < PIX; ++k) {
          const float dx = fpx - mq.x;
          const float dy = fpy[k] - mq.y;
          const float q = co.x * dx * dx + 2.0f * co.y * dx * dy + co.z * dy * dy;
          if (done[k] || !(q >= 0.0f && q <= mq.z)) continue;
          // -0.5 q lies in [-q_cut/2, 0], inside det_expf's core range
          float alpha = co.w * det_expf_neg(-0.5f * q, tab);
          alpha = (alpha < kAlphaCap) ? alpha : kAlphaCap;
          if (alpha < kAlphaMin) continue;
          // warp-aggregated increment: one atomic per distinct Gaussian
          const uint32_t id = s_id[j];
          const uint32_t act = __activemask();
          const uint32_t peers = __match_any_sync(act, id);
          if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&counts[id], __popc(peers));
          T[k] = T[k] * (1.0f - alpha);
          if (T[k] < kTransmitMin) done[k] = true;
        }
        bool ad = true;
#pragma unroll
        for (int k = 0; k < PIX; ++k) ad = ad && done[k];
        all_done = ad;
      }
    }
  }
}

// K12 over K6's record (16x16 tiles): the masked pixels' contributors are
// exactly the entries up to each pixel's last_entry whose alpha reaches
// 1/255 — K6 of the same frame (exact form) recorded last_entry per pixel and,
// per (32-entry batch, 8x8 warp block), the mask of entries some pixel of the
// block blended. So a warp gathers only the marked entries of the batches up
// to its masked pixels' last entry, needs no transmittance, and decides
// alpha >= 1/255 with the hardware exp, recomputing the deterministic exp
// only within 1e-5 of the threshold (as K8 does): the same decisions as K6,
// bit for bit. Counts use one atomic per (entry, warp).
template <int PIX>
__global__ void __launch_bounds__(16 * 16 / PIX, 8) count_walk_kernel(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ pair_val, const float2* __restrict__ mean2d,
    const float4* __restrict__ conic_op, int W, int H, int tiles_x, const uint8_t* __restrict__ mask,
    const int* __restrict__ last_entry, const uint32_t* __restrict__ cmask, int* __restrict__ counts,
    const uint32_t* __restrict__ err) {
  if (err && __ldg(err)) return;  // see blend_fwd_warp_kernel
  constexpr int TS = 16;
  using WB = WarpBlock<TS, PIX>;
  constexpr int kWarps = WB::kWarps;
  __shared__ float4 s_xyq[kWarps][32];
  __shared__ float4 s_co[kWarps][32];
  __shared__ float s_exp[kNegExpTable];
  stage_neg_exp_table(s_exp);
  __syncthreads();
  const SmemPinnedTable tab(s_exp);
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const WB wb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int px = tx * TS + wb.lx;
  const int2 range = ranges[tile];
  const float fpx = (float)px;
  float fpy[PIX];
  int last[PIX];
  int my_last = range.x;
#pragma unroll
  for (int k = 0; k < PIX; ++k) {
    const int py = ty * TS + wb.ly0 + 4 * k;
    fpy[k] = (float)py;
    last[k] = range.x;  // unmasked / outside: no entry
    if (px < W && py < H && mask[(size_t)py * W + px] != 0) last[k] = last_entry[(size_t)py * W + px];
    my_last = max(my_last, last[k]);
  }
  const int warp_last = __reduce_max_sync(0xffffffffu, my_last);
  if (warp_last <= range.x) return;
  const int64_t wbase = cmask_word(range.x, tile);
  for (int kb = 0; range.x + 32 * kb < warp_last; ++kb) {
    const int b0 = range.x + 32 * kb;
    uint32_t m = __ldg(&cmask[(size_t)(wbase + kb) * kWarps + warp]);
    const int lim = warp_last - b0;
    if (lim < 32) m &= (1u << lim) - 1u;
    if (!m) continue;
    if ((m >> lane) & 1u) {
      const uint32_t g = pair_val[b0 + lane];
      const float4 co = conic_op[g];
      float4 xyq, bb;
      stage_entry(mean2d[g], co, xyq, bb);
      xyq.w = __uint_as_float(g);
      s_xyq[warp][lane] = xyq;
      s_co[warp][lane] = co;
    }
    __syncwarp();
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const float4 mq = s_xyq[warp][j];
      const float4 co = s_co[warp][j];
      const int idx = b0 + j;
      int hits = 0;
#pragma unroll
      for (int k = 0; k < PIX; ++k) {
        const float dx = fpx - mq.x;
        const float dy = fpy[k] - mq.y;
        const float q = co.x * dx * dx + 2.0f * co.y * dx * dy + co.z * dy * dy;  // K6's exact q
        if (idx >= last[k] || __float_as_uint(__fadd_rn(q, 0.0f)) > __float_as_uint(mq.z)) continue;
        float raw = co.w * exp2f_approx(q * -0.72134752044448170f);
        if (fabsf(raw - kAlphaMin) <= 1e-5f) raw = co.w * det_expf_neg(-0.5f * q, tab);
        hits += (raw < kAlphaCap ? raw : kAlphaCap) < kAlphaMin ? 0 : 1;
      }
      hits = __reduce_add_sync(0xffffffffu, hits);
      if (lane == 0 && hits) atomicAdd(&counts[__float_as_uint(mq.w)], hits);
    }
    __syncwarp();
  }
}

// K6, warp-staged variant: each warp walks the tile's list for its own
// 8 x 4·PIX pixel block independently — it stages 32 entries at a time (one
// per lane: gather, q-cut box, exact ellipse test against its own block),
// keeps only the hits (ballot) in its private shared slots and walks them. No
// CTA barrier inside the list walk, so warps neither wait for each other at
// batch boundaries nor keep staging after their own pixels have terminated;
// the price is that each warp gathers every entry (L1 serves the repeats).
// Per-pixel arithmetic is identical to blend_fwd_kernel (bit-exact).
//
// FAST (training steps, sk_train_step*/Trainer): alpha = o 2^{q (-log2 e / 2)}
// on MUFU.EX2 instead of the deterministic exp — the image is then within
// the north star's 1e-4 of the oracle's (not bit-equal), and K8 recomputes
// exactly the same alphas (same ops on the same bit-equal q), so the
// forward / backward pair stays self-consistent. Every parity-facing path
// (sk_render_forward, the density-event renders, K12) runs the exact form.
template <int TS, int PIX, bool FAST>
__global__ void __launch_bounds__(TS* TS / PIX, kFwdMinBlocks * 128 / (TS * TS / PIX)) blend_fwd_warp_kernel(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ pair_val, const float2* __restrict__ mean2d,
    const float4* __restrict__ conic_op, const float4* __restrict__ rgbd, int W, int H, int tiles_x,
    float* __restrict__ image, float* __restrict__ final_t, int* __restrict__ n_contrib, int* __restrict__ last_entry,
    uint32_t* __restrict__ cmask, const uint32_t* __restrict__ err) {
  // a training step whose pair count outgrew its buffer (or whose K1 raised an
  // error) skips the blend: it is replayed or fails (pipeline.cu, trainer.cu)
  if (err && __ldg(err)) return;
  using WB = WarpBlock<TS, PIX>;
  constexpr int kWarps = WB::kWarps;
  __shared__ float4 s_xyq[kWarps][32];
  __shared__ float4 s_gco[2][kWarps][32];
  __shared__ float2 s_gmu[2][kWarps][32];
  __shared__ float4 s_grgb[2][kWarps][32];
  __shared__ float s_exp[FAST ? 1 : kNegExpTable];
  if (!FAST) {
    stage_neg_exp_table(s_exp);
    __syncthreads();
  }
  const SmemPinnedTable tab(s_exp);

  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const WB wb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    done[k] = !(px < W && py < H);
    all_done = all_done && done[k];
    if (done[k]) fpy[k] = __int_as_float(0x7fc00000);
  }

  // Double-buffered gather: the records of batch k+1 are copied into this
  // warp's shared slots with cp.async (no registers held in flight) while
  // batch k is walked; the pair index of batch k+2 is loaded one batch ahead
  // so the copy never waits on it.
  int cur = 0;
  uint32_t g_next = 0;
  auto issue = [&](int buf, int bb, uint32_t g) {
    if (bb + lane < range.y) {
      cp_async16(&s_gco[buf][warp][lane], &conic_op[g]);
      cp_async8(&s_gmu[buf][warp][lane], &mean2d[g]);
      cp_async16(&s_grgb[buf][warp][lane], &rgbd[g]);
    }
    cp_async_commit();
  };
  if (range.x < range.y) {
    const uint32_t g0 = range.x + lane < range.y ? pair_val[range.x + lane] : 0u;
    issue(0, range.x, g0);
    g_next = range.x + 32 + lane < range.y ? pair_val[range.x + 32 + lane] : 0u;
  }
  for (int b0 = range.x; b0 < range.y; b0 += 32) {
    if (__all_sync(0xffffffffu, all_done)) break;
    if (b0 + 32 < range.y) {
      issue(cur ^ 1, b0 + 32, g_next);
      g_next = b0 + 64 + lane < range.y ? pair_val[b0 + 64 + lane] : 0u;
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int i = b0 + lane;
    bool hit = false;
    if (i < range.y) {
      const float4 co = s_gco[cur][warp][lane];
      float4 xyq, bb;
      stage_entry(s_gmu[cur][warp][lane], co, xyq, bb);
      hit = !WB::misses(bb, warp, tx, ty);
      const bool pd = co.x > 0.0f && co.z > 0.0f && co.x * co.z - co.y * co.y > 0.0f;
      if (hit && pd) hit = WB::ellipse_hits(xyq, co, warp, tx, ty);
      if (hit) s_xyq[warp][lane] = xyq;
    }
    const float4* s_co_w = s_gco[cur][warp];
    const float4* s_rgb_w = s_grgb[cur][warp];
    cur ^= 1;
    uint32_t m = __ballot_sync(0xffffffffu, hit);
    __syncwarp();
    uint32_t lane_bits = 0;  // entries of this batch one of my pixels blended
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const float4 mq = s_xyq[warp][j];
      const float4 co = s_co_w[j];
      if (FAST && PIX % 2 == 0) {
        // Training steps: q of the lane's pixel pairs (rows y, y + 4) in packed
        // f32x2 FMAs, q = A + dy (B + c11 dy) with A = (c00 dx) dx and
        // B = (2 c01) dx shared by the pair. K8's FAST walk forms q with the
        // same instructions, so both kernels make the same contribution
        // decisions (blend_common.cuh: fast_pair_q).
        const float dx = fpx - mq.x;
        const float A = __fmul_rn(__fmul_rn(co.x, dx), dx), B = __fmul_rn(__fmul_rn(2.0f, co.y), dx);
        const uint32_t qc = __float_as_uint(mq.z);
#pragma unroll
        for (int kp = 0; kp < PIX / 2; ++kp) {
          const int a = 2 * kp, b = 2 * kp + 1;
          const float2 dy = __fadd2_rn(make_float2(fpy[a], fpy[b]), make_float2(-mq.y, -mq.y));
          const float2 q = fast_pair_q(dy, co.z, A, B);
          bool ok0 = __float_as_uint(__fadd_rn(q.x, 0.0f)) <= qc;
          bool ok1 = __float_as_uint(__fadd_rn(q.y, 0.0f)) <= qc;
          if (!(ok0 || ok1)) continue;
          const float2 xe = __fmul2_rn(q, make_float2(-0.72134752044448170f, -0.72134752044448170f));
          float2 al = __fmul2_rn(make_float2(co.w, co.w), make_float2(exp2f_approx(xe.x), exp2f_approx(xe.y)));
          al.x = (al.x < kAlphaCap) ? al.x : kAlphaCap;
          al.y = (al.y < kAlphaCap) ? al.y : kAlphaCap;
          ok0 = ok0 && !(al.x < kAlphaMin);
          ok1 = ok1 && !(al.y < kAlphaMin);
          if (!(ok0 || ok1)) continue;
          lane_bits |= 1u << j;
          const float4 c = s_rgb_w[j];
          // both pixels in packed ops, a non-contributing one with alpha = 0
          // (T, C unchanged exactly); the colour sums may contract: K8 reads
          // only T and last_entry
          const float2 al2 = make_float2(ok0 ? al.x : 0.0f, ok1 ? al.y : 0.0f);
          float2 t2 = make_float2(T[a], T[b]);
          const float2 w2 = __fmul2_rn(t2, al2);
          float2 c0 = __ffma2_rn(w2, make_float2(c.x, c.x), make_float2(C0[a], C0[b]));
          float2 c1 = __ffma2_rn(w2, make_float2(c.y, c.y), make_float2(C1[a], C1[b]));
          float2 c2 = __ffma2_rn(w2, make_float2(c.z, c.z), make_float2(C2[a], C2[b]));
          t2 = __fmul2_rn(t2, __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-al2.x, -al2.y)));
          C0[a] = c0.x, C0[b] = c0.y;
          C1[a] = c1.x, C1[b] = c1.y;
          C2[a] = c2.x, C2[b] = c2.y;
          T[a] = t2.x, T[b] = t2.y;
          n[a] += ok0 ? 1 : 0;
          n[b] += ok1 ? 1 : 0;
          last[a] = ok0 ? b0 + j + 1 : last[a];
          last[b] = ok1 ? b0 + j + 1 : last[b];
          fpy[a] = t2.x < kTransmitMin ? __int_as_float(0x7fc00000) : fpy[a];
          fpy[b] = t2.y < kTransmitMin ? __int_as_float(0x7fc00000) : fpy[b];
        }
        continue;
      }
#pragma unroll
      for (int k = 0; k < PIX; ++k) {
        const float dx = fpx - mq.x;
        const float dy = fpy[k] - mq.y;
        const float q = co.x * dx * dx + 2.0f * co.y * dx * dy + co.z * dy * dy;
        if (__float_as_uint(__fadd_rn(q, 0.0f)) > __float_as_uint(mq.z)) continue;  // -0 -> +0
        float alpha = FAST ? co.w * exp2f_approx(q * -0.72134752044448170f) : co.w * det_expf_neg(-0.5f * q, tab);
        alpha = (alpha < kAlphaCap) ? alpha : kAlphaCap;
        if (alpha < kAlphaMin) continue;
        lane_bits |= 1u << j;
        const float4 c = s_rgb_w[j];
        const float w = T[k] * alpha;
        C0[k] = C0[k] + w * c.x;
        C1[k] = C1[k] + w * c.y;
        C2[k] = C2[k] + w * c.z;
        ++n[k];
        last[k] = b0 + j + 1;
        T[k] = T[k] * (1.0f - alpha);
        fpy[k] = T[k] < kTransmitMin ? __int_as_float(0x7fc00000) : fpy[k];
      }
    }
    {
      bool ad = true;
#pragma unroll
      for (int k = 0; k < PIX; ++k) ad = ad && isnan(fpy[k]);
      all_done = ad;
    }
    // contribution mask of this warp block for the batch (read by K8, which
    // then skips entries no pixel of its block blended); K8 never reads an
    // unwalked batch (every pixel's last contributor lies in a walked one)
    const uint32_t bits = __reduce_or_sync(0xffffffffu, lane_bits);
    if (cmask && lane == 0) cmask[(size_t)(cmask_word(range.x, tile) + ((b0 - range.x) >> 5)) * kWarps + warp] = bits;
    __syncwarp();
  }
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

// Workload counters of a rendered frame: pixel-Gaussian
// evaluations the reference's blend_forward loop visits (raster.hpp:219-235:
// every list entry up to and including the one that takes T below 1e-4, or
// the whole list) and the contributing ones (alpha >= 1/255). The terminating
// entry is always the pixel's last contributor, so visited = last_entry -
// range start for terminated pixels (final T < 1e-4), else the list length.
__global__ void pge_counts_kernel(const int2* __restrict__ ranges, const float* __restrict__ final_t,
                                  const int* __restrict__ n_contrib, const int* __restrict__ last_entry, int W,
                                  int H, int TS, int tiles_x, unsigned long long* __restrict__ out) {
  unsigned long long vis = 0, con = 0;
  const int64_t HW = (int64_t)W * H;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < HW; p += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(p / W), x = (int)(p % W);
    const int2 r = ranges[(y / TS) * tiles_x + x / TS];
    vis += (unsigned long long)(final_t[p] < kTransmitMin ? last_entry[p] - r.x : r.y - r.x);
    con += (unsigned long long)n_contrib[p];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vis += __shfl_xor_sync(0xffffffffu, vis, o);
    con += __shfl_xor_sync(0xffffffffu, con, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], vis);
    atomicAdd(&out[1], con);
  }
}

template <int TS, int PIX>
void fwd_dispatch(sk_ctx* ctx, sk_frame* f, const uint8_t* mask, int32_t* counts, bool fast) {
  const int tiles = f->tiles_x * f->tiles_y;
  auto* ranges = f->ranges.as<int2>();
  const auto* mean2d = f->mean2d.as<float2>();
  const auto* co = f->conic_op.as<float4>();
  const auto* rgb = f->rgb_depth.as<float4>();
  if (mask && TS == 16 && PIX == 2 && f->cmask_valid && !f->fast_blend)
    // the frame's last K6 (exact, on the current tile lists: binning clears
    // cmask_valid) recorded last_entry and the contribution masks
    count_walk_kernel<PIX><<<tiles, TS * TS / PIX, 0, ctx->stream>>>(
        ranges, f->pair_val, mean2d, co, f->width, f->height, f->tiles_x, mask, f->last_entry.as<int>(),
        f->cmask.as<uint32_t>(), counts, f->pairs < 0 ? ctx->err_word.as<uint32_t>() : nullptr);
  else if (mask)
    count_blend_kernel<TS, PIX><<<tiles, TS * TS / PIX, 0, ctx->stream>>>(
        ranges, f->pair_val, mean2d, co, f->width, f->height, f->tiles_x, mask, counts,
        f->pairs < 0 ? ctx->err_word.as<uint32_t>() : nullptr);
  else {
    uint32_t* cm = nullptr;
    if (TS == 16 && PIX == 2) {  // K8 consumes the masks at 16x16 tiles
      const size_t words = cmask_words(f->pairs < 0 ? f->pair_cap : f->pairs, tiles) * (size_t)(TS * TS / PIX / 32);
      // no clearing: K8 reads the words of batches up to its block's last
      // contributor only, all of which this K6 warp walked and wrote
      cm = ensure<uint32_t>(f->cmask, words);
    }
    f->cmask_valid = cm != nullptr;
    f->fast_blend = fast;
    auto go = [&](auto kern) {
      kern<<<tiles, TS * TS / PIX, 0, ctx->stream>>>(ranges, f->pair_val, mean2d, co, rgb, f->width, f->height,
                                                     f->tiles_x, f->image.as<float>(), f->final_t.as<float>(),
                                                     f->n_contrib.as<int>(), f->last_entry.as<int>(), cm,
                                                     f->pairs < 0 ? ctx->err_word.as<uint32_t>() : nullptr);
    };
    if (fast)
      go(blend_fwd_warp_kernel<TS, PIX, true>);
    else
      go(blend_fwd_warp_kernel<TS, PIX, false>);
  }
  note_launch();
}

}  // namespace

void frame_pge_counts(sk_ctx* ctx, sk_frame* f, int64_t* visited, int64_t* contributing) {
  auto* out = ensure<unsigned long long>(ctx->pge, 2);
  SK_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), ctx->stream));
  pge_counts_kernel<<<148 * 4, 256, 0, ctx->stream>>>(f->ranges.as<int2>(), f->final_t.as<float>(),
                                                      f->n_contrib.as<int>(), f->last_entry.as<int>(), f->width,
                                                      f->height, f->tile_size, f->tiles_x, out);
  note_launch();
  SK_CUDA(cudaGetLastError());
  unsigned long long h[2];
  SK_CUDA(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  SK_CUDA(cudaStreamSynchronize(ctx->stream));
  *visited = (int64_t)h[0];
  *contributing = (int64_t)h[1];
}

void launch_blend_forward(sk_ctx* ctx, sk_frame* f, const uint8_t* mask, int32_t* counts, bool fast) {
  if (f->tiles_x * f->tiles_y == 0) return;
  switch (f->tile_size) {
    case 8: fwd_dispatch<8, 1>(ctx, f, mask, counts, fast && !mask); break;
    case 16: fwd_dispatch<16, 2>(ctx, f, mask, counts, fast && !mask); break;
    case 32: fwd_dispatch<32, 4>(ctx, f, mask, counts, fast && !mask); break;
    default: throw std::invalid_argument("tile_size must be 8, 16 or 32");
  }
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
