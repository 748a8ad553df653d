// K8 backward blend: restates blend_backward (reference raster.hpp:281-355)
// as a reverse walk from each pixel's last contributor (recorded by K6):
// T_before = T_after / (1 - alpha), suffix accumulated in the reference's
// reverse order, capped entries feed d_color only. Each thread owns PIX
// pixels (rows y, y+4, ...) of its warp's 8 x 4·PIX block, sums their partials
// per Gaussian in registers, and the warp butterfly-reduces the 11 partials
// of two entries at a time with a shuffle reduce-scatter (23 shuffles per
// pair); lanes issue one global atomic each.
//
// Gradients are checked against the oracle within a tolerance, so this file
// is compiled with FMA contraction. The per-pixel contribution decision must
// still be K6's exactly (the walk must visit exactly the entries K6 blended):
// q is written with non-contracting round-to-nearest intrinsics (bit-equal
// to K6), alpha comes from the fast hardware exp, and only alphas within
// 1e-5 relative of the 1/255 and 0.99 thresholds (the fast exp is within
// ~1e-6) are recomputed with the shared deterministic exp.
#include "blend_common.cuh"

namespace sk {
namespace {

using namespace blend;

// Reduce-scatter of the 11 gradient partials of two entries (a: lanes 0-15
// after the first stage, b: lanes 16-31) over the warp: each butterfly stage
// hands half of the remaining values to the partner lane, so 11 + 6 + 3 + 2 + 1
// = 23 shuffles leave lane l holding the warp sum of one (entry, field):
// field = 6·bit3 + 3·bit2 + 2·bit1 + bit0 of entry (lane < 16 ? a : b), or
// nothing for the padding slots (bit1 & bit0, and field 11). Then every lane
// with a value issues one global atomic.
__device__ __forceinline__ void reduce_scatter_2x11(const float (&a)[kBGradFields], const float (&b)[kBGradFields],
                                                    uint32_t id_a, uint32_t id_b, bool write_b,
                                                    float* __restrict__ bgrads, int64_t gstride) {
  const int lane = threadIdx.x & 31;
  float k1[kBGradFields];
#pragma unroll
  for (int f = 0; f < kBGradFields; ++f) {
    const float give = lane < 16 ? b[f] : a[f];
    const float mine = lane < 16 ? a[f] : b[f];
    k1[f] = mine + __shfl_xor_sync(0xffffffffu, give, 16);
  }
  const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
  float k2[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const float lo = k1[i], hi = i + 6 < kBGradFields ? k1[i + 6] : 0.0f;
    k2[i] = (b3 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b3 ? lo : hi, 8);
  }
  float k3[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float lo = k2[i], hi = k2[i + 3];
    k3[i] = (b2 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b2 ? lo : hi, 4);
  }
  float k4[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float lo = k3[i], hi = i == 0 ? k3[2] : 0.0f;
    k4[i] = (b1 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b1 ? lo : hi, 2);
  }
  const float v = (b0 ? k4[1] : k4[0]) + __shfl_xor_sync(0xffffffffu, b0 ? k4[0] : k4[1], 1);
  const int field = (b3 ? 6 : 0) + (b2 ? 3 : 0) + (b1 ? 2 : 0) + (b0 ? 1 : 0);
  const bool valid = !(b1 && b0) && field < kBGradFields && (lane < 16 || write_b);
  if (valid) atomicAdd(&bgrads[(int64_t)field * gstride + (lane < 16 ? id_a : id_b)], v);
}

// 16x16 tiles: 128 threads (8x8 pixel block per warp, 2 pixels per thread,
// the same blocks as K6) and 7 resident CTAs (28 warps) per SM, which caps
// the kernel at 72 registers without spills. Measured against 64 threads x 4
// pixels (8x16 blocks): -12% K8 time; 7 CTAs/SM instead of 6: -4% more.
#ifndef SK_BWD_MINB
#define SK_BWD_MINB 7
#endif

// cp.async double-buffered gather on the mask path: measured 3% slower than
// the direct gather (it needs the extra buffer registers / smem and K8's
// gathers are already sparse), so off by default.
#ifndef SK_BWD_PAIRWALK
#define SK_BWD_PAIRWALK 0  // measured: 5% slower (register pressure)
#endif
#ifndef SK_BWD_BRANCHLESS
#define SK_BWD_BRANCHLESS 1  // measured: -6.8% K8 time
#endif
#ifndef SK_BWD_PIN
#define SK_BWD_PIN 1
#endif
#ifndef SK_BWD_UQ
// 1: q in [0, q_cut] as one unsigned compare of (q + 0) bits (K6's test), and
// the two near-threshold bands folded into one symmetric band around the
// midpoint of alpha_min and the cap (absolute half-width 1e-5 * cap, which
// contains both relative 1e-5 bands)
#define SK_BWD_UQ 1
#endif
#ifndef SK_BWD_SINGLE_LANE
#define SK_BWD_SINGLE_LANE 0  // measured: no gain (1.112 vs 1.101 ms)
#endif
#ifndef SK_BWD_DIRECT_MAX
#define SK_BWD_DIRECT_MAX 1
#endif
#ifndef SK_BWD_L1PF
#define SK_BWD_L1PF 0
#endif
#ifndef SK_BWD_ASYNC_GATHER
#define SK_BWD_ASYNC_GATHER 0
#endif
#ifndef SK_BWD_USE_CMASK
#define SK_BWD_USE_CMASK 1
#endif
#ifndef SK_BWD_PIX16
#define SK_BWD_PIX16 2
#endif
#ifndef SK_BWD_WARP_STAGED
#define SK_BWD_WARP_STAGED 1  // measured: 6.6% faster than the CTA-staged walk
#endif

template <int TS, int PIX, bool WS = SK_BWD_WARP_STAGED != 0, bool FASTEXP = true>
__global__ void __launch_bounds__(TS* TS / PIX, SK_BWD_MINB * 128 / (TS * TS / PIX)) blend_bwd_kernel(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ pair_val, const float2* __restrict__ mean2d,
    const float4* __restrict__ conic_op, const float4* __restrict__ rgbd, int W, int H, int tiles_x,
    const float* __restrict__ final_t, const int* __restrict__ last_entry, const float* __restrict__ dimage,
    float* __restrict__ bgrads, int64_t gstride, const uint32_t* __restrict__ cmask) {
  constexpr int NT = TS * TS / PIX;  // threads == batch size
  using WB = WarpBlock<TS, PIX>;
  constexpr int kChunks = NT / 32;
  // two buffers of NT slots for the asynchronous gather (slot buf * NT + j);
  // the other paths use the first NT
  constexpr int NB = SK_BWD_ASYNC_GATHER ? 2 * NT : NT;
#if SK_BWD_PIN
  // the walk's four staged arrays in one block whose shared-window base is
  // pinned in a register: the walk loads use it with immediate offsets
  // (plain indexing rematerialised each array's base with an S2R of the
  // cluster CTA id inside the loop)
  struct alignas(16) Staged {
    float4 xyq[NB];
    float4 co[NB];
    float4 rgb[NB];
    uint32_t id[NB];
  };
  __shared__ Staged s_st;
  float4(&s_xyq)[NB] = s_st.xyq;
  float4(&s_co)[NB] = s_st.co;
  float4(&s_rgb)[NB] = s_st.rgb;
  uint32_t(&s_id)[NB] = s_st.id;
  uint32_t st_base;
  asm volatile("mov.u32 %0, %1;" : "=r"(st_base) : "r"((uint32_t)__cvta_generic_to_shared(&s_st)));
  auto ld_f4 = [&](uint32_t off, int j) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(st_base + off + 16u * (uint32_t)j));
    return v;
  };
  auto ld_xyq = [&](int j) { return ld_f4(0u, j); };
  auto ld_co = [&](int j) { return ld_f4(16u * NB, j); };
  auto ld_rgb = [&](int j) { return ld_f4(32u * NB, j); };
  auto ld_id = [&](int j) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(st_base + 48u * NB + 4u * (uint32_t)j));
    return v;
  };
#else
  __shared__ float4 s_xyq[NB];
  __shared__ float4 s_co[NB];
  __shared__ float4 s_rgb[NB];
  __shared__ uint32_t s_id[NB];
  auto ld_xyq = [&](int j) { return s_xyq[j]; };
  auto ld_co = [&](int j) { return s_co[j]; };
  auto ld_rgb = [&](int j) { return s_rgb[j]; };
  auto ld_id = [&](int j) { return s_id[j]; };
#endif
  __shared__ uint32_t s_mask[WB::kWarps * kChunks];
  __shared__ float2 s_mu[SK_BWD_ASYNC_GATHER ? NB : 1];
  __shared__ int s_max_last;
  __shared__ float s_exp2[64];
  stage_exp2_table(s_exp2);
  const SmemTable tab(s_exp2);

  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const WB wb;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
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
  __syncthreads();  // also publishes the exp table
  if (!WS) atomicMax(&s_max_last, my_last);
  __syncthreads();
  const int end = s_max_last;  // no pixel of the tile uses entries >= end
  const int warp_last = __reduce_max_sync(0xffffffffu, my_last);
  float pend[kBGradFields];
  uint32_t pend_id = 0;
  bool has_pend = false;

  // Per-entry reverse-walk step for staged slot j (list position idx).
  // The 11 gradient partials of staged slot j (list position idx) over this
  // lane's pixels; returns whether one of them blended the entry.
  auto partials = [&](int j, int idx, float (&gv)[kBGradFields]) -> bool {
    const float4 mq = ld_xyq(j);
    const float4 co = ld_co(j);
    float g_mu0 = 0.f, g_mu1 = 0.f, g_c00 = 0.f, g_c01 = 0.f, g_c11 = 0.f, g_r = 0.f, g_g = 0.f, g_b = 0.f,
          g_op = 0.f, g_a0 = 0.f, g_a1 = 0.f;
    bool contrib = false;
#if SK_BWD_BRANCHLESS
    // Predicated form: every lane evaluates both of its pixels and masks the
    // non-contributing ones to exact zeros (alpha -> 0 leaves T and the
    // suffix unchanged), so the warp does not diverge / reconverge per
    // pixel; only the rare near-threshold exact-exp recompute branches.
#pragma unroll
    for (int k = 0; k < PIX; ++k) {
      const float dx = fpx - mq.x;
      const float dy = fpy[k] - mq.y;
      const float q = rn_add(rn_add(rn_mul(rn_mul(co.x, dx), dx), rn_mul(rn_mul(rn_mul(2.0f, co.y), dx), dy)),
                             rn_mul(rn_mul(co.z, dy), dy));
#if SK_BWD_UQ
      bool ok = idx < last[k] && __float_as_uint(__fadd_rn(q, 0.0f)) <= __float_as_uint(mq.z);
      float ge = __expf(-0.5f * q);
      float raw = co.w * ge;
      constexpr float kMid = (float)((1.0 / 255 + 0.99) / 2), kHalf = (float)((0.99 - 1.0 / 255) / 2);
      if (ok && fabsf(fabsf(raw - kMid) - kHalf) <= 1e-5f * kAlphaCap) {
#else
      bool ok = idx < last[k] && q >= 0.0f && q <= mq.z;
      float ge = __expf(-0.5f * q);
      float raw = co.w * ge;
      if (ok && (fabsf(raw - kAlphaMin) <= 1e-5f * kAlphaMin || fabsf(raw - kAlphaCap) <= 1e-5f * kAlphaCap)) {
#endif
        ge = det_expf_core(rn_mul(-0.5f, q), tab);
        raw = rn_mul(co.w, ge);
      }
      const bool capped = raw > kAlphaCap;
      const float alpha_c = capped ? kAlphaCap : raw;
      ok = ok && !(alpha_c < kAlphaMin);
      contrib = contrib || ok;
      const float alpha = ok ? alpha_c : 0.0f;
      const float4 c = ld_rgb(j);
      const float one_m = 1.0f - alpha;
      const float inv_one_m = __fdividef(1.0f, one_m);
      const float t_before = T[k] * inv_one_m;
      T[k] = t_before;
      const float w = (c.x * d0[k] + c.y * d1[k]) + c.z * d2[k];
      const float d_alpha = t_before * w - suffix[k] * inv_one_m;
      const float ta = t_before * alpha;
      suffix[k] = suffix[k] + ta * w;
      g_r += ta * d0[k];
      g_g += ta * d1[k];
      g_b += ta * d2[k];
      const bool geo = ok && !capped;
      g_op += geo ? ge * d_alpha : 0.0f;
      const float d_q = geo ? -0.5f * alpha * d_alpha : 0.0f;
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
#else
#pragma unroll
    for (int k = 0; k < PIX; ++k) {
      if (idx >= last[k]) continue;
      const float dx = fpx - mq.x;
      const float dy = fpy[k] - mq.y;
      // same association as K6: ((c00 dx) dx + ((2 c01) dx) dy) + (c11 dy) dy
      const float q = rn_add(rn_add(rn_mul(rn_mul(co.x, dx), dx), rn_mul(rn_mul(rn_mul(2.0f, co.y), dx), dy)),
                             rn_mul(rn_mul(co.z, dy), dy));
      if (!(q >= 0.0f && q <= mq.z)) continue;
      // Fast exp (MUFU ex2, ~1e-6 relative); the exact deterministic exp
      // only where alpha is within 1e-5 (relative) of a decision threshold,
      // so the skip / cap decisions are exactly K6's.
      float ge = FASTEXP ? __expf(-0.5f * q) : 0.0f;
      float raw = co.w * ge;
      if (!FASTEXP || fabsf(raw - kAlphaMin) <= 1e-5f * kAlphaMin || fabsf(raw - kAlphaCap) <= 1e-5f * kAlphaCap) {
        ge = det_expf_core(rn_mul(-0.5f, q), tab);
        raw = rn_mul(co.w, ge);
      }
      const bool capped = raw > kAlphaCap;
      const float alpha = capped ? kAlphaCap : raw;
      if (alpha < kAlphaMin) continue;
      contrib = true;
      const float4 c = ld_rgb(j);
      const float one_m = 1.0f - alpha;
      const float inv_one_m = __fdividef(1.0f, one_m);  // tolerance path: MUFU reciprocal, two products
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
#endif
    gv[0] = g_mu0; gv[1] = g_mu1; gv[2] = g_c00; gv[3] = g_c01; gv[4] = g_c11; gv[5] = g_r;
    gv[6] = g_g; gv[7] = g_b; gv[8] = g_op; gv[9] = g_a0; gv[10] = g_a1;
    return contrib;
  };

  auto walk_entry = [&](int j, int idx) {
    float gv0[kBGradFields];
    const bool contrib = partials(j, idx, gv0);
    const uint32_t cb = __ballot_sync(0xffffffffu, contrib);
#if SK_BWD_SINGLE_LANE
    if (__popc(cb) <= SK_BWD_DIRECT_MAX) {
      // few contributing lanes: each adds its own partials (one lane: they
      // are the warp sum), no shuffle reduction
      if (contrib) {
        const uint32_t id = ld_id(j);
#pragma unroll
        for (int f = 0; f < kBGradFields; ++f) atomicAdd(&bgrads[(int64_t)f * gstride + id], gv0[f]);
      }
    } else
#endif
    if (cb) {
      if (has_pend) {
        reduce_scatter_2x11(pend, gv0, pend_id, ld_id(j), true, bgrads, gstride);
        has_pend = false;
      } else {
#pragma unroll
        for (int f = 0; f < kBGradFields; ++f) pend[f] = gv0[f];
        pend_id = ld_id(j);
        has_pend = true;
      }
    }
  };

  if (WS && TS == 16 && cmask) {
    // Warp-staged over K6's batches with K6's contribution masks: only the
    // entries a pixel of this block blended in the forward pass are gathered
    // and walked (the others contribute nothing here), no ellipse tests.
    // K8 warp w covers K6 warps (8x8 blocks) x8 = w % 2, y8 in [y8a, y8b).
    const int base = warp * 32;
    const int x8 = warp % 2, y8a = (warp / 2) * (4 * PIX) / 8, y8b = ((warp / 2) * (4 * PIX) + 4 * PIX + 7) / 8;
    if (warp_last > range.x) {
      const int64_t wbase = cmask_word(range.x, tile);
      auto mask_of = [&](int kb) -> uint32_t {
        if (kb < 0) return 0u;
        uint32_t m = 0;
        for (int y8 = y8a; y8 < y8b; ++y8) m |= __ldg(&cmask[(size_t)(wbase + kb) * 4 + y8 * 2 + x8]);
        const int lim = warp_last - (range.x + 32 * kb);
        if (lim < 32) m &= (1u << lim) - 1u;
        return m;
      };
#if SK_BWD_ASYNC_GATHER
      // Batches in descending order; the records of batch kb-1 are copied
      // with cp.async while kb is walked, and the mask + pair index of kb-2
      // are loaded one batch ahead.
      auto issue = [&](int buf, int kb, uint32_t m, uint32_t g) {
        if ((m >> lane) & 1u) {
          const int slot = buf * NT + base + lane;
          cp_async16(&s_co[slot], &conic_op[g]);
          cp_async8(&s_mu[slot], &mean2d[g]);
          cp_async16(&s_rgb[slot], &rgbd[g]);
          s_id[slot] = g;
        }
        cp_async_commit();
      };
      auto gidx = [&](int kb, uint32_t m) -> uint32_t {
        return ((m >> lane) & 1u) ? pair_val[range.x + 32 * kb + lane] : 0u;
      };
      int kb = (warp_last - 1 - range.x) >> 5;
      uint32_t m_cur = mask_of(kb);
      issue(0, kb, m_cur, gidx(kb, m_cur));
      uint32_t m_next = mask_of(kb - 1);
      uint32_t g_next = gidx(kb - 1, m_next);
      int buf = 0;
      for (; kb >= 0; --kb) {
        const uint32_t m_prev = m_next;  // mask of batch kb - 1
        if (kb >= 1) {
          issue(buf ^ 1, kb - 1, m_next, g_next);
          m_next = mask_of(kb - 2);
          g_next = gidx(kb - 2, m_next);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        const int b0 = range.x + 32 * kb;
        uint32_t m = m_cur;
        if ((m >> lane) & 1u) {
          const int slot = buf * NT + base + lane;
          float4 xyq, bb;
          stage_entry(s_mu[slot], s_co[slot], xyq, bb);
          s_xyq[slot] = xyq;
        }
        __syncwarp();
        while (m) {
          const int bit = 31 - __clz(m);
          m ^= 1u << bit;
          walk_entry(buf * NT + base + bit, b0 + bit);
        }
        __syncwarp();
        m_cur = m_prev;
        buf ^= 1;
      }
#else
      for (int kb = (warp_last - 1 - range.x) >> 5; kb >= 0; --kb) {
        const int b0 = range.x + 32 * kb;
        uint32_t m = mask_of(kb);
        if (!m) continue;
#if SK_BWD_L1PF
        // L1 prefetch of the next batch's pair indices (no registers held)
        if (kb > 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(pair_val + b0 - 32 + lane));
#endif
        if ((m >> lane) & 1u) {
          const uint32_t g = pair_val[b0 + lane];
          float4 xyq, bb;
          const float4 co = conic_op[g];
          stage_entry(mean2d[g], co, xyq, bb);
          s_xyq[base + lane] = xyq;
          s_co[base + lane] = co;
          s_rgb[base + lane] = rgbd[g];
          s_id[base + lane] = g;
        }
        __syncwarp();
#if SK_BWD_PAIRWALK
        // entries taken two at a time straight into one reduce-scatter (every
        // masked entry has a contributing lane); one entry is carried over
        // only when a batch has an odd count
        while (m) {
          const int ba = 31 - __clz(m);
          m ^= 1u << ba;
          float ga[kBGradFields];
          partials(base + ba, b0 + ba, ga);
          const uint32_t ida = s_id[base + ba];
          if (has_pend) {
            reduce_scatter_2x11(pend, ga, pend_id, ida, true, bgrads, gstride);
            has_pend = false;
          } else if (m) {
            const int bb2 = 31 - __clz(m);
            m ^= 1u << bb2;
            float gb[kBGradFields];
            partials(base + bb2, b0 + bb2, gb);
            reduce_scatter_2x11(ga, gb, ida, s_id[base + bb2], true, bgrads, gstride);
          } else {
#pragma unroll
            for (int f = 0; f < kBGradFields; ++f) pend[f] = ga[f];
            pend_id = ida;
            has_pend = true;
          }
        }
#else
        while (m) {
          const int bit = 31 - __clz(m);
          m ^= 1u << bit;
          walk_entry(base + bit, b0 + bit);
        }
#endif
        __syncwarp();
      }
#endif
    }
  } else if (WS) {
    // Warp-staged: each warp gathers 32 entries at a time from its own last
    // contributor downward, keeps the hits on its block (ballot) in its
    // private slots and walks them; no CTA barrier inside the walk.
    const int base = warp * 32;
    for (int b_end = warp_last; b_end > range.x; b_end -= 32) {
      const int b0 = max(range.x, b_end - 32);
      const int i = b0 + lane;
      bool hit = false;
      if (i < b_end) {
        const uint32_t g = pair_val[i];
        const float4 co = conic_op[g];
        float4 xyq, bb;
        stage_entry(mean2d[g], co, xyq, bb);
        hit = !WB::misses(bb, warp, tx, ty);
        const bool pd = co.x > 0.0f && co.z > 0.0f && co.x * co.z - co.y * co.y > 0.0f;
        if (hit && pd) hit = WB::ellipse_hits(xyq, co, warp, tx, ty);
        if (hit) {
          s_xyq[base + lane] = xyq;
          s_co[base + lane] = co;
          s_rgb[base + lane] = rgbd[g];
          s_id[base + lane] = g;
        }
      }
      uint32_t m = __ballot_sync(0xffffffffu, hit);
      __syncwarp();
      while (m) {
        const int bit = 31 - __clz(m);
        m ^= 1u << bit;
        walk_entry(base + bit, b0 + bit);
      }
      __syncwarp();
    }
  } else {
  for (int b_end = end; b_end > range.x; b_end -= NT) {
    const int b0 = max(range.x, b_end - NT);
    __syncthreads();
    const int i = b0 + (int)threadIdx.x;
    const bool valid = i < b_end;
    float4 bb = make_float4(1.0f, -1.0f, 1.0f, -1.0f), xyq = bb, co = bb;
    if (valid) {
      const uint32_t g = pair_val[i];
      co = conic_op[g];
      stage_entry(mean2d[g], co, xyq, bb);
      s_xyq[threadIdx.x] = xyq;
      s_co[threadIdx.x] = co;
      s_rgb[threadIdx.x] = rgbd[g];
      s_id[threadIdx.x] = g;
    }
    WB::publish(bb, xyq, co, valid, warp, kChunks, tx, ty, s_mask);
    __syncthreads();
    // Reverse walk over the entries whose box touches this warp's block.
    const int jmax = min(b_end, warp_last) - b0;  // warp-uniform
    for (int c = (jmax - 1) >> 5; c >= 0; --c) {
      uint32_t m = s_mask[warp * kChunks + c];
      const int lim = jmax - c * 32;
      if (lim < 32) m &= (1u << lim) - 1u;
      while (m) {
        const int bit = 31 - __clz(m);
        m ^= 1u << bit;
        walk_entry(c * 32 + bit, b0 + c * 32 + bit);
      }
    }
  }
  }
  if (has_pend) {  // warp-uniform: flush the last unpaired entry
    float zero[kBGradFields];
#pragma unroll
    for (int f = 0; f < kBGradFields; ++f) zero[f] = 0.0f;
    reduce_scatter_2x11(pend, zero, pend_id, 0u, false, bgrads, gstride);
  }
}

template <int TS, int PIX>
void bwd_dispatch(sk_ctx* ctx, sk_frame* f) {
  const int tiles = f->tiles_x * f->tiles_y;
  blend_bwd_kernel<TS, PIX><<<tiles, TS * TS / PIX, 0, ctx->stream>>>(
      f->ranges.as<int2>(), f->pair_val, f->mean2d.as<float2>(), f->conic_op.as<float4>(), f->rgb_depth.as<float4>(),
      f->width, f->height, f->tiles_x, f->final_t.as<float>(), f->last_entry.as<int>(), f->dimage.as<float>(),
      f->bgrads.as<float>(), f->n,
      (SK_BWD_USE_CMASK && TS == 16 && f->cmask_valid) ? f->cmask.as<uint32_t>() : nullptr);
  note_launch();
}

}  // namespace

void launch_blend_backward(sk_ctx* ctx, sk_frame* f) {
  SK_CUDA(cudaMemsetAsync(f->bgrads.ptr, 0, sizeof(float) * kBGradFields * (size_t)f->n, ctx->stream));
  if (f->tiles_x * f->tiles_y == 0) return;
  switch (f->tile_size) {
    case 8: bwd_dispatch<8, 1>(ctx, f); break;
    case 16: bwd_dispatch<16, SK_BWD_PIX16>(ctx, f); break;
    case 32: bwd_dispatch<32, 4>(ctx, f); break;
    default: throw std::invalid_argument("tile_size must be 8, 16 or 32");
  }
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
