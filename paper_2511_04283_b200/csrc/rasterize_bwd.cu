// K8 backward blend: restates blend_backward (reference raster.hpp:281-355)
// as a reverse walk from each pixel's last contributor (recorded by K6):
// T_before = T_after / (1 - alpha), suffix accumulated in the reference's
// reverse order, capped entries feed d_color only. Each thread owns PIX
// pixels (rows y, y+4, ...) of its warp's 8 x 4·PIX block, sums their partials
// per Gaussian in registers, and the warp butterfly-reduces the 11 partials
// of two entries at a time with a shuffle reduce-scatter (23 shuffles per
// pair); lanes issue one global atomic each.
//
// Gradients are checked against the oracle within a tolerance; the file is
// compiled without FMA contraction (-fmad=false, builder.py) and every fused
// multiply-add of the gradient math is written explicitly (fmaf /
// __ffma2_rn). The per-pixel contribution decision must be K6's exactly
// (the walk must visit exactly the entries K6 blended): alpha comes from the
// fast hardware exp, and only alphas within 1e-5 relative of the 1/255 and
// 0.99 thresholds (the fast exp is within ~1e-6) are recomputed with the
// shared deterministic exp.
#include <type_traits>

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
// the same blocks as K6) and 8 resident CTAs (32 warps) per SM, which caps
// the kernel at 64 registers — without spills since the contribution-mask
// walk dropped its per-entry vote (measured: 8 CTAs -0.4% against 7, which
// was the best before; 64 threads x 4 pixels (8x16 blocks): +12% to +18%).
// (8x8 and 32x32 tiles keep the 7-CTA-equivalent budget: 32x32 would spill.)
constexpr int kBwdMinBlocks = 8;

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
// 1 / x on MUFU.RCP alone (x = 1 - alpha lies in [0.01, 1]: no range fix-ups)
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// The 11 gradient partials of one staged entry over a lane's pixel pair
// (rows y and y + 4 of its column), with the pair's arithmetic in packed
// f32x2 instructions (FFMA2 / FMUL2 / FADD2: one issue slot for both pixels).
// Per-pixel state (T, -suffix, dL/dimage, y) is held as float2 pairs.
//
// The contribution decision is K6's exactly: q is formed with non-contracting
// round-to-nearest ops in K6's association (the packed mul / add are
// correctly rounded per lane, so q is bit-equal to K6's), the fast MUFU exp
// decides except within 1e-5 of the 1/255 and 0.99 thresholds, where the
// shared deterministic exp recomputes alpha.
struct PairState {
  float2 T, ns, d0, d1, d2, fpy;  // T_after, -suffix, dL/dimage RGB, pixel y
  int last0, last1;
};

// FIRST: the partials are assigned rather than accumulated (the lane's
// first pixel pair of the entry; saves the adds of zero).
template <bool FAST, bool FIRST, typename Tab>
__device__ __forceinline__ bool pair_partials(const float4 mq, const float4 co, const float4 c, float fpx, int idx,
                                              PairState& st, const Tab& tab, float (&g)[kBGradFields]) {
  const float dx = fpx - mq.x;
  const float2 dy = __fadd2_rn(st.fpy, f2(-mq.y));
  // Exact frames: q = ((c00 dx) dx + ((2 c01) dx) dy) + (c11 dy) dy, bit-equal
  // to K6's exact walk, in scalar round-to-nearest ops (ptxas contracts
  // mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false, which would
  // change q's last bits). FAST frames: K6's packed form (fast_pair_q).
  const float A = __fmul_rn(__fmul_rn(co.x, dx), dx);
  const float B = __fmul_rn(__fmul_rn(2.0f, co.y), dx);
  // FAST frames: K6's packed form (fast_pair_q); exact frames: K6's scalar ops
  const float2 q = FAST ? fast_pair_q(dy, co.z, A, B)
                        : make_float2(rn_add(rn_add(A, rn_mul(B, dy.x)), rn_mul(rn_mul(co.z, dy.x), dy.x)),
                                      rn_add(rn_add(A, rn_mul(B, dy.y)), rn_mul(rn_mul(co.z, dy.y), dy.y)));
  // q in [0, q_cut] as one unsigned compare of (q + 0) bits (-0 -> +0; NaN / negative fail)
  const uint32_t qc = __float_as_uint(mq.z);
  bool ok0 = idx < st.last0 && __float_as_uint(__fadd_rn(q.x, 0.0f)) <= qc;
  bool ok1 = idx < st.last1 && __float_as_uint(__fadd_rn(q.y, 0.0f)) <= qc;
  // e^{-q/2} = 2^{q * (-log2(e) / 2)} on MUFU (the same bits as __expf(-q/2))
  const float2 xe = __fmul2_rn(q, f2(-0.72134752044448170f));
  float2 ge = make_float2(exp2f_approx(xe.x), exp2f_approx(xe.y));
  float2 raw = __fmul2_rn(f2(co.w), ge);
  // one symmetric band |(|raw - mid| - half)| <= 1e-5 * cap around both thresholds
  constexpr float kMid = (float)((1.0 / 255 + 0.99) / 2), kHalf = (float)((0.99 - 1.0 / 255) / 2);
  constexpr float kBand = 1e-5f * (float)kAlphaCap;
  // FAST (the frame's K6 ran the MUFU form): these are K6's alphas bit for bit
  if (!FAST && ok0 && fabsf(fabsf(raw.x - kMid) - kHalf) <= kBand) {
    ge.x = det_expf_core(rn_mul(-0.5f, q.x), tab);
    raw.x = rn_mul(co.w, ge.x);
  }
  if (!FAST && ok1 && fabsf(fabsf(raw.y - kMid) - kHalf) <= kBand) {
    ge.y = det_expf_core(rn_mul(-0.5f, q.y), tab);
    raw.y = rn_mul(co.w, ge.y);
  }
  const bool cap0 = raw.x > kAlphaCap, cap1 = raw.y > kAlphaCap;
  const float ac0 = cap0 ? kAlphaCap : raw.x, ac1 = cap1 ? kAlphaCap : raw.y;
  ok0 = ok0 && !(ac0 < kAlphaMin);
  ok1 = ok1 && !(ac1 < kAlphaMin);
  // non-contributing pixels: alpha = 0 leaves T, the suffix and every partial unchanged
  const float2 alpha = make_float2(ok0 ? ac0 : 0.0f, ok1 ? ac1 : 0.0f);
  // capped entries feed d_color only (raster.hpp:315, 333)
  const bool geo0 = ok0 && !cap0, geo1 = ok1 && !cap1;
  const float2 inv = make_float2(rcp_approx(1.0f - alpha.x), rcp_approx(1.0f - alpha.y));
  const float2 tb = __fmul2_rn(st.T, inv);  // T before the entry
  st.T = tb;
  const float2 w = __ffma2_rn(f2(c.z), st.d2, __ffma2_rn(f2(c.y), st.d1, __fmul2_rn(f2(c.x), st.d0)));
  const float2 d_alpha = __ffma2_rn(tb, w, __fmul2_rn(st.ns, inv));  // T w - suffix / (1 - alpha)
  const float2 ta = __fmul2_rn(tb, alpha);
  st.ns = __ffma2_rn(__fmul2_rn(ta, f2(-1.0f)), w, st.ns);
  // The pair's two terms of each partial are combined with the second
  // product fused (fma(p1, q1, p0 q0 + g)): one rounding fewer than summing
  // two rounded products, which matters on the cancelling sums of small
  // gradients.
  auto acc = [](float& gf, float2 a, float2 b) {
    gf = FIRST ? fmaf(a.y, b.y, a.x * b.x) : fmaf(a.y, b.y, fmaf(a.x, b.x, gf));
  };
  acc(g[5], ta, st.d0);
  acc(g[6], ta, st.d1);
  acc(g[7], ta, st.d2);
  acc(g[8], make_float2(geo0 ? ge.x : 0.0f, geo1 ? ge.y : 0.0f), d_alpha);  // e^{-q/2} d_alpha
  // ad = alpha d_alpha = -2 d_q on geometric entries (d_q = -alpha d_alpha / 2)
  const float2 ad = __fmul2_rn(make_float2(geo0 ? alpha.x : 0.0f, geo1 ? alpha.y : 0.0f), d_alpha);
  // d_conic (full-matrix convention) = d_q [dx^2, dx dy, dy^2] = -ad / 2 [..]
  // (the power-of-two scale commutes with the rounding)
  const float2 adh = __fmul2_rn(ad, f2(-0.5f));
  acc(g[2], adh, f2(dx * dx));
  acc(g[3], adh, __fmul2_rn(f2(dx), dy));
  acc(g[4], adh, __fmul2_rn(dy, dy));
  // d_mu = -2 d_q conic d
  const float2 m0 = __fmul2_rn(ad, __ffma2_rn(f2(co.y), dy, f2(co.x * dx)));
  const float2 m1 = __fmul2_rn(ad, __ffma2_rn(f2(co.z), dy, f2(co.y * dx)));
  if (FIRST) {
    g[0] = m0.x + m0.y;
    g[1] = m1.x + m1.y;
    g[9] = fabsf(m0.x) + fabsf(m0.y);
    g[10] = fabsf(m1.x) + fabsf(m1.y);
  } else {
    g[0] = (g[0] + m0.x) + m0.y;
    g[1] = (g[1] + m1.x) + m1.y;
    g[9] = (g[9] + fabsf(m0.x)) + fabsf(m0.y);
    g[10] = (g[10] + fabsf(m1.x)) + fabsf(m1.y);
  }
  return ok0 || ok1;
}

// Scalar form of the same step for one-pixel lanes (8x8 tiles); assigns g.
template <bool FAST, typename Tab>
__device__ __forceinline__ bool one_partials(const float4 mq, const float4 co, const float4 c, float fpx, float fpy,
                                             int idx, int last, float& T, float& ns, float d0, float d1, float d2,
                                             const Tab& tab, float (&g)[kBGradFields]) {
  const float dx = fpx - mq.x, dy = fpy - mq.y;
  const float q = rn_add(rn_add(rn_mul(rn_mul(co.x, dx), dx), rn_mul(rn_mul(rn_mul(2.0f, co.y), dx), dy)),
                         rn_mul(rn_mul(co.z, dy), dy));
  bool ok = idx < last && __float_as_uint(__fadd_rn(q, 0.0f)) <= __float_as_uint(mq.z);
  float ge = exp2f_approx(q * -0.72134752044448170f);
  float raw = co.w * ge;
  constexpr float kMid = (float)((1.0 / 255 + 0.99) / 2), kHalf = (float)((0.99 - 1.0 / 255) / 2);
  if (!FAST && ok && fabsf(fabsf(raw - kMid) - kHalf) <= 1e-5f * (float)kAlphaCap) {
    ge = det_expf_core(rn_mul(-0.5f, q), tab);
    raw = rn_mul(co.w, ge);
  }
  const bool capped = raw > kAlphaCap;
  const float ac = capped ? kAlphaCap : raw;
  ok = ok && !(ac < kAlphaMin);
  const float alpha = ok ? ac : 0.0f;
  const bool geo = ok && !capped;
  const float inv = rcp_approx(1.0f - alpha);
  const float tb = T * inv;
  T = tb;
  const float w = fmaf(c.z, d2, fmaf(c.y, d1, c.x * d0));
  const float d_alpha = fmaf(ns, inv, tb * w);
  const float ta = tb * alpha;
  ns = fmaf(-ta, w, ns);
  g[5] = ta * d0;
  g[6] = ta * d1;
  g[7] = ta * d2;
  g[8] = (geo ? ge : 0.0f) * d_alpha;
  const float ad = geo ? alpha * d_alpha : 0.0f;
  const float adh = -0.5f * ad;
  g[2] = adh * (dx * dx);
  g[3] = adh * (dx * dy);
  g[4] = adh * (dy * dy);
  const float m0 = ad * fmaf(co.y, dy, co.x * dx), m1 = ad * fmaf(co.z, dy, co.y * dx);
  g[0] = m0;
  g[1] = m1;
  g[9] = fabsf(m0);
  g[10] = fabsf(m1);
  return ok;
}

template <int TS, int PIX, bool FAST>
__global__ void __launch_bounds__(TS* TS / PIX, (TS == 16 ? kBwdMinBlocks : 7) * 128 / (TS * TS / PIX)) blend_bwd_kernel(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ pair_val, const float2* __restrict__ mean2d,
    const float4* __restrict__ conic_op, const float4* __restrict__ rgbd, int W, int H, int tiles_x,
    const float* __restrict__ final_t, const int* __restrict__ last_entry, const float* __restrict__ dimage,
    float* __restrict__ bgrads, int64_t gstride, const uint32_t* __restrict__ cmask,
    const uint32_t* __restrict__ err) {
  if (err && __ldg(err)) return;  // see blend_fwd_warp_kernel
  constexpr int NT = TS * TS / PIX;
  constexpr int NP = PIX / 2 > 0 ? PIX / 2 : 1;  // pixel pairs per lane (PIX = 1: one scalar pixel)
  using WB = WarpBlock<TS, PIX>;
  // The walk's four staged arrays in one block whose shared-window base is
  // pinned in a register: the walk loads use it with immediate offsets
  // (plain indexing rematerialised each array's base with an S2R of the
  // cluster CTA id inside the loop).
  struct alignas(16) Staged {
    float4 xyq[NT];
    float4 co[NT];
    float4 rgb[NT];
    uint32_t id[NT];
  };
  __shared__ Staged s_st;
  uint32_t st_base;
  asm volatile("mov.u32 %0, %1;" : "=r"(st_base) : "r"((uint32_t)__cvta_generic_to_shared(&s_st)));
  auto ld_f4 = [&](uint32_t off, int j) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(st_base + off + 16u * (uint32_t)j));
    return v;
  };
  auto ld_id = [&](int j) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(st_base + 48u * NT + 4u * (uint32_t)j));
    return v;
  };
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

  float T[PIX], d0[PIX], d1[PIX], d2[PIX], fpy[PIX];
  int last[PIX];
  int my_last = 0;
#pragma unroll
  for (int k = 0; k < PIX; ++k) {
    const int py = ty * TS + wb.ly0 + 4 * k;
    fpy[k] = (float)py;
    T[k] = 1.0f;
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
  PairState ps[NP];
  float T1 = T[0], ns1 = 0.0f;
  if (PIX >= 2) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int a = 2 * k, b = 2 * k + 1 < PIX ? 2 * k + 1 : 2 * k;
      ps[k].T = make_float2(T[a], T[b]);
      ps[k].ns = f2(0.0f);
      ps[k].d0 = make_float2(d0[a], d0[b]);
      ps[k].d1 = make_float2(d1[a], d1[b]);
      ps[k].d2 = make_float2(d2[a], d2[b]);
      ps[k].fpy = make_float2(fpy[a], fpy[b]);
      ps[k].last0 = last[a];
      ps[k].last1 = last[b];
    }
  }
  __syncthreads();  // publishes the exp table
  const int warp_last = __reduce_max_sync(0xffffffffu, my_last);

  // This lane's 11 partials of staged slot j (list position idx), the
  // -2 d_q scale folded in; returns whether some lane of the warp
  // contributed (warp-uniform). VOTE = false (the contribution-mask walk):
  // K6 marked the entry because a pixel of this very 8x8 block blended it,
  // with the same decision arithmetic, so the vote is known to be true; and
  // were it not, the entry's partials would all be zero and its atomics
  // would add zeros.
  auto partials = [&](int j, int idx, float (&gv)[kBGradFields], auto vote) {
    const float4 mq = ld_f4(0u, j);
    const float4 co = ld_f4(16u * NT, j);
    const float4 c = ld_f4(32u * NT, j);
    bool contrib;
    if (PIX >= 2) {
      contrib = pair_partials<FAST, true>(mq, co, c, fpx, idx, ps[0], tab, gv);
#pragma unroll
      for (int k = 1; k < NP; ++k) contrib = pair_partials<FAST, false>(mq, co, c, fpx, idx, ps[k], tab, gv) || contrib;
    } else {
      contrib = one_partials<FAST>(mq, co, c, fpx, fpy[0], idx, last[0], T1, ns1, d0[0], d1[0], d2[0], tab, gv);
    }
    if constexpr (decltype(vote)::value) return __any_sync(0xffffffffu, contrib) != 0;
    return true;
  };
  // Entries are reduced two at a time (reduce_scatter_2x11): the walk
  // alternates between computing into ga (the pending entry, kept across
  // batches) and gb, then reduces the pair, so no partials are copied.
  float ga[kBGradFields], gb[kBGradFields];
  uint32_t id_a = 0;
  bool has_a = false;
  // pops the highest set bit of m (reverse list order)
  auto pop = [](uint32_t& m) {
    uint32_t bit;
    asm("bfind.u32 %0, %1;" : "=r"(bit) : "r"(m));
    m ^= 1u << bit;
    return (int)bit;
  };
  const int base = warp * 32;
  auto walk = [&](uint32_t m, int b0, auto vote) {
    while (m) {
      if (!has_a) {
        const int bit = pop(m);
        if (partials(base + bit, b0 + bit, ga, vote)) {
          has_a = true;
          id_a = ld_id(base + bit);
        }
      } else {
        const int bit = pop(m);
        if (partials(base + bit, b0 + bit, gb, vote)) {
          reduce_scatter_2x11(ga, gb, id_a, ld_id(base + bit), true, bgrads, gstride);
          has_a = false;
        }
      }
    }
  };

  if (TS == 16 && cmask) {
    // Over K6's 32-entry batches with K6's contribution masks: only the
    // entries a pixel of this block blended in the forward pass are gathered
    // and walked (the others contribute nothing here), no ellipse tests.
    // K8 warp w covers K6 warps (8x8 blocks) x8 = w % 2, y8 in [y8a, y8b).
    const int x8 = warp % 2, y8a = (warp / 2) * (4 * PIX) / 8, y8b = ((warp / 2) * (4 * PIX) + 4 * PIX + 7) / 8;
    if (warp_last > range.x) {
      const int64_t wbase = cmask_word(range.x, tile);
      for (int kb = (warp_last - 1 - range.x) >> 5; kb >= 0; --kb) {
        const int b0 = range.x + 32 * kb;
        uint32_t m = 0;
        for (int y8 = y8a; y8 < y8b; ++y8) m |= __ldg(&cmask[(size_t)(wbase + kb) * 4 + y8 * 2 + x8]);
        const int lim = warp_last - b0;
        if (lim < 32) m &= (1u << lim) - 1u;
        if (!m) continue;
        if ((m >> lane) & 1u) {
          const uint32_t g = pair_val[b0 + lane];
          float4 xyq, bb;
          const float4 co = conic_op[g];
          stage_entry(mean2d[g], co, xyq, bb);
          s_st.xyq[base + lane] = xyq;
          s_st.co[base + lane] = co;
          s_st.rgb[base + lane] = rgbd[g];
          s_st.id[base + lane] = g;
        }
        __syncwarp();
        walk(m, b0, std::false_type{});
        __syncwarp();
      }
    }
  } else {
    // Each warp gathers 32 entries at a time from its own last contributor
    // downward, keeps the hits on its block (ballot) in its private slots
    // and walks them; no CTA barrier inside the walk.
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
          s_st.xyq[base + lane] = xyq;
          s_st.co[base + lane] = co;
          s_st.rgb[base + lane] = rgbd[g];
          s_st.id[base + lane] = g;
        }
      }
      const uint32_t m = __ballot_sync(0xffffffffu, hit);
      __syncwarp();
      walk(m, b0, std::true_type{});
      __syncwarp();
    }
  }
  if (has_a) {  // warp-uniform: flush the last unpaired entry
#pragma unroll
    for (int f = 0; f < kBGradFields; ++f) gb[f] = 0.0f;
    reduce_scatter_2x11(ga, gb, id_a, 0u, false, bgrads, gstride);
  }
}

template <int TS, int PIX>
void bwd_dispatch(sk_ctx* ctx, sk_frame* f) {
  const int tiles = f->tiles_x * f->tiles_y;
  auto kern = f->fast_blend ? blend_bwd_kernel<TS, PIX, true> : blend_bwd_kernel<TS, PIX, false>;
  kern<<<tiles, TS * TS / PIX, 0, ctx->stream>>>(
      f->ranges.as<int2>(), f->pair_val, f->mean2d.as<float2>(), f->conic_op.as<float4>(), f->rgb_depth.as<float4>(),
      f->width, f->height, f->tiles_x, f->final_t.as<float>(), f->last_entry.as<int>(), f->dimage.as<float>(),
      f->bgrads.as<float>(), f->n, (TS == 16 && f->cmask_valid) ? f->cmask.as<uint32_t>() : nullptr,
      f->pairs < 0 ? ctx->err_word.as<uint32_t>() : nullptr);
  note_launch();
}

}  // namespace

void launch_blend_backward(sk_ctx* ctx, sk_frame* f) {
  if (!f->bgrads_zeroed)
    SK_CUDA(cudaMemsetAsync(f->bgrads.ptr, 0, sizeof(float) * kBGradFields * (size_t)f->n, ctx->stream));
  f->bgrads_zeroed = false;
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
