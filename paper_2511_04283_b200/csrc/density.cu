// The paper's multi-view-consistent density control on the GPU:
//   K11 error maps      build_error_maps        (reference error_maps.hpp:22-43)
//   K12 count blend     blend_forward(mask,...) (raster.hpp:194-248 via adc.hpp:105-108)
//   K13 finalize        scores_from_counts      (adc.hpp:48-84)
//   K14 select          select_densify / select_prune (adc.hpp:135-153, 224-270)
//   K15 compact         apply_prune / apply_densify + AdamGroup::remap
//                       (adc.hpp:167-205, 273-289; adam.hpp:45-58)
// and Trainer::density_event (trainer.hpp:177-243) that sequences them.
//
// Everything here is compiled with -fmad=false: the error map, the mask,
// s_d and every selection flag are computed in the reference's fp32 order, so
// given identical inputs they are bit-identical to the CPU oracle. Footprint
// counts are exact integers (warp-aggregated atomics). Compaction is a
// three-class exclusive scan (survivors / clones / split children) followed by
// a scatter of parameters and Adam moments into fresh buffers.
#include <algorithm>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <thread>

#include "abi_util.h"
#include "trainer.h"


namespace sk {
namespace {

// Block-level min / max of non-negative floats (as ordered bits), then one
// atomic pair per CTA: a per-warp atomic on the same two words from every
// warp of a 2 MPix frame serialises ~130K atomics at one L2 slice (90 us).
__device__ __forceinline__ void block_minmax_atomic(uint32_t lo, uint32_t hi, uint32_t* __restrict__ lohi) {
  __shared__ uint32_t s_lo[32], s_hi[32];
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) s_lo[warp] = lo, s_hi[warp] = hi;
  __syncthreads();
  if (warp == 0) {
    lo = lane < nw ? s_lo[lane] : 0xffffffffu;
    hi = lane < nw ? s_hi[lane] : 0u;
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
      atomicMin(&lohi[0], lo);
      atomicMax(&lohi[1], hi);
    }
  }
}

// ---- K11: raw error map + min / max ---------------------------------------
// Grid-stride over the pixels (a few CTAs per SM); the 8-bit GT decoded
// byte / 255 through a table of the same IEEE quotients.
__global__ void __launch_bounds__(256) error_raw_kernel(const float* __restrict__ image, const void* __restrict__ gt,
                                                        bool gt_u8, int W, int H, float* __restrict__ raw,
                                                        uint32_t* __restrict__ lohi) {
  __shared__ float s_u8[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_u8[i] = __fdiv_rn((float)i, 255.0f);
  __syncthreads();
  const int64_t n = (int64_t)W * H;
  uint32_t lo = 0xffffffffu, hi = 0u;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    float d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float g = gt_u8 ? s_u8[static_cast<const uint8_t*>(gt)[p * 3 + c]] : static_cast<const float*>(gt)[p * 3 + c];
      d[c] = image[c * n + p] - g;
    }
    // (rendered - gt).cwiseAbs().sum() / T(3)
    const float v = ((fabsf(d[0]) + fabsf(d[1])) + fabsf(d[2])) / 3.0f;
    raw[p] = v;
    // raw >= 0: ordering of the float bits is the ordering of the values
    lo = min(lo, __float_as_uint(v));
    hi = max(hi, __float_as_uint(v));
  }
  block_minmax_atomic(lo, hi, lohi);
}

// normalized = (raw - lo) / (hi - lo) (all zero if degenerate); mask = normalized > tau
// (normalized may be null: the score pass only needs the mask)
__global__ void error_mask_kernel(const float* __restrict__ raw, const uint32_t* __restrict__ lohi, int64_t n,
                                  float tau, uint8_t* __restrict__ mask, float* __restrict__ normalized) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const float lo = __uint_as_float(lohi[0]), hi = __uint_as_float(lohi[1]);
  const float nv = hi > lo ? (raw[p] - lo) / (hi - lo) : 0.0f;
  mask[p] = nv > tau ? 1 : 0;
  if (normalized) normalized[p] = nv;
}

// ---- K13: s_d, s_p_raw in view order, then min-max of s_p_raw ---------------
// View j's count row / photometric value sit at slot (j % world) * kpr +
// j / world (rank-major blocks of the sharded score pass; the identity at
// world = 1); the sums run over j ascending as the reference's.
__global__ void scores_kernel(const int32_t* __restrict__ rows, int64_t row_stride, const float* __restrict__ photo,
                              int k, int world, int kpr, int64_t n, float* __restrict__ s_d,
                              float* __restrict__ s_p_raw, uint32_t* __restrict__ lohi) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float sd = 0.0f, sp = 0.0f;
  const bool ok = i < n;
  if (ok) {
    for (int j = 0; j < k; ++j) {
      const int slot = (j % world) * kpr + j / world;
      const float c = (float)rows[(int64_t)slot * row_stride + i];
      sd = sd + c;
      sp = sp + c * photo[slot];
    }
    s_d[i] = sd / (float)k;
    s_p_raw[i] = sp;
  }
  block_minmax_atomic(ok ? __float_as_uint(sp) : 0xffffffffu, ok ? __float_as_uint(sp) : 0u, lohi);
}

__global__ void minmax_normalize_kernel(const float* __restrict__ v, const uint32_t* __restrict__ lohi, int64_t n,
                                        float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float lo = __uint_as_float(lohi[0]), hi = __uint_as_float(lohi[1]);
  out[i] = hi > lo ? (v[i] - lo) / (hi - lo) : 0.0f;
}

__device__ __forceinline__ float max_scale(const float* p, int64_t stride, int64_t i) {
  const float s0 = det_expf(p[(SK_COMP_LOG_SCALE + 0) * stride + i]);
  const float s1 = det_expf(p[(SK_COMP_LOG_SCALE + 1) * stride + i]);
  const float s2 = det_expf(p[(SK_COMP_LOG_SCALE + 2) * stride + i]);
  float m = s0;
  if (s1 > m) m = s1;
  if (s2 > m) m = s2;
  return m;
}

// ---- K14: selection flags -------------------------------------------------------
__global__ void densify_flags_kernel(const float* __restrict__ p, int64_t stride, int64_t n,
                                     const float* __restrict__ s_d, const float* __restrict__ gn,
                                     const float* __restrict__ ag, const int* __restrict__ vs, float tau_d,
                                     float thr, float dense_cut, bool use_vcd, uint8_t* __restrict__ clone,
                                     uint8_t* __restrict__ split) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t c = 0, s = 0;
  const int seen = vs[i];
  if (seen != 0 && !(use_vcd && !(s_d[i] > tau_d))) {
    const float inv_seen = 1.0f / (float)seen;
    const float mean_grad = gn[i] * inv_seen;
    const float mean_abs = ag[i] * inv_seen;
    if (max_scale(p, stride, i) <= dense_cut) {
      c = mean_grad >= thr ? 1 : 0;
    } else {
      s = mean_abs >= thr ? 1 : 0;
    }
  }
  clone[i] = c;
  split[i] = s;
}

// early phase: vanilla candidates (key for the VCP ordering); late: the rule.
__global__ void prune_flags_kernel(const float* __restrict__ p, int64_t stride, int64_t n,
                                   const float* __restrict__ s_p, const float* __restrict__ max_r2d, bool early,
                                   bool size_rules, float min_op, float world_cut, float screen, float op_cut,
                                   bool use_vcp, float tau_p, uint8_t* __restrict__ flag, uint32_t* __restrict__ key,
                                   int* __restrict__ count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool f = false;
  if (i < n) {
    const float op = det_sigmoidf(p[SK_COMP_OPACITY * stride + i]);
    if (early) {
      f = op < min_op;
      if (size_rules) {
        f = f || max_scale(p, stride, i) > world_cut;
        f = f || max_r2d[i] > screen;
      }
      // ascending key == s_p descending (ties: index order, select_take_kernel); non-candidates last
      if (key) key[i] = f ? (0x7f800000u - __float_as_uint(s_p[i])) : 0xffffffffu;
    } else {
      f = (op < op_cut) || (use_vcp && s_p[i] > tau_p);
    }
    flag[i] = f ? 1 : 0;
  }
  const uint32_t b = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, __popc(b));
}

// VCP's "keep the ceil(|C|/2) highest s_p, ties by index" (adc.hpp:243-249)
// as a radix select on the candidate keys (ascending key == s_p descending,
// non-candidates 0xffffffff) instead of a full sort: four 8-bit MSB-first
// histogram passes find the take-th smallest key K*; every key < K* is
// taken, and of the keys == K* the first `rank` in index order.
struct SelectState {
  uint32_t prefix, mask;  // digits of K* fixed so far
  int rank;               // position still to find among keys matching the prefix (1-based)
  int pad;
};

__global__ void select_init_kernel(const int* __restrict__ count, SelectState* __restrict__ st,
                                   uint32_t* __restrict__ hist) {
  if (threadIdx.x == 0) *st = SelectState{0u, 0u, (*count + 1) / 2, 0};
  hist[threadIdx.x] = 0;
}

__global__ void select_hist_kernel(const uint32_t* __restrict__ key, int64_t n, const SelectState* __restrict__ st,
                                   int shift, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_h[256];
  s_h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t prefix = st->prefix, mask = st->mask;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = key[i];
    if ((k & mask) == prefix) atomicAdd(&s_h[(k >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  if (s_h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], s_h[threadIdx.x]);
}

// one CTA of 256: fixes the next digit of K* and clears the histogram
__global__ void select_step_kernel(SelectState* __restrict__ st, int shift, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_c[256];
  const int d = threadIdx.x;
  uint32_t x = hist[d];
  s_c[d] = x;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // inclusive scan
    const uint32_t y = d >= o ? s_c[d - o] : 0u;
    __syncthreads();
    s_c[d] += y;
    __syncthreads();
  }
  const int rank = st->rank;
  const uint32_t incl = s_c[d], excl = incl - x;
  __syncthreads();
  if (rank > 0 && (int)excl < rank && rank <= (int)incl) {
    st->prefix |= (uint32_t)d << shift;
    st->mask |= 0xffu << shift;
    st->rank = rank - (int)excl;
  }
  hist[d] = 0;
}

__global__ void __launch_bounds__(256) select_tie_count_kernel(const uint32_t* __restrict__ key, int64_t n,
                                                                const SelectState* __restrict__ st,
                                                                int3* __restrict__ block_counts) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const bool eq = i < n && st->rank > 0 && key[i] == st->prefix;
  const int c = __syncthreads_count(eq);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = make_int3(c, 0, 0);
}

__global__ void __launch_bounds__(256) select_take_kernel(const uint32_t* __restrict__ key, int64_t n,
                                                           const SelectState* __restrict__ st,
                                                           const int3* __restrict__ block_base,
                                                           uint8_t* __restrict__ flag) {
  __shared__ int s_w[8];
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const uint32_t kstar = st->prefix;
  const int rank = st->rank;  // 0: no candidate at all
  const uint32_t k = i < n ? key[i] : 0xffffffffu;
  const int eq = (i < n && rank > 0 && k == kstar) ? 1 : 0;
  // in-block exclusive count of equal keys before i
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t b = __ballot_sync(0xffffffffu, eq);
  if (lane == 0) s_w[warp] = __popc(b);
  __syncthreads();
  int before = block_base[blockIdx.x].x + __popc(b & ((1u << lane) - 1u));
  for (int w = 0; w < warp; ++w) before += s_w[w];
  if (i >= n) return;
  flag[i] = (rank > 0 && (k < kstar || (eq && before < rank))) ? 1 : 0;
}

// never empty the scene: keep the first index with the smallest s_p
__global__ void argmin_kernel(const float* __restrict__ s_p, int64_t n, unsigned long long* __restrict__ best) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = ~0ull;
  if (i < n) v = ((unsigned long long)__float_as_uint(s_p[i]) << 32) | (unsigned long long)i;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  if ((threadIdx.x & 31) == 0) atomicMin(best, v);
}

// ---- K15: compaction (apply_prune / apply_densify adc.hpp:166-205, 272-289 and
// the Adam moment remaps adam.hpp:45-58) in three kernels:
//   K15a  per 256-Gaussian block: counts of the three output classes
//         (non-split survivors, clones, split parents; pruned Gaussians are
//         neither cloned nor split, trainer.hpp:212-217);
//   K15b  one CTA: exclusive scans of the block counts and the totals;
//   K15c  per block: the same class flags, an in-block scan for each class,
//         then every Gaussian moves its 59 parameter / m / v rows (coalesced
//         along the Gaussian axis) to its destination slots and writes the
//         clone step and the split children's geometry.
// Output order (adc.hpp:179-201): survivors, then clones, then split pairs.
constexpr int kCompactBlock = 256;  // threads per block
constexpr int kCompactItems = 1;    // Gaussians per thread (measured: 4 per thread with float4 row
                                    // loads +22% K15 — strided stores)
constexpr int kCompactSpan = kCompactBlock * kCompactItems;

struct Classes {
  int keep, clone, split;  // 0 / 1 each
};
__device__ __forceinline__ Classes classify(const uint8_t* prune, const uint8_t* clone, const uint8_t* split,
                                            int64_t i, int64_t n) {
  Classes c{0, 0, 0};
  if (i < n && !prune[i]) {
    const bool sp = split[i] != 0;
    c.keep = sp ? 0 : 1;
    c.clone = clone[i] ? 1 : 0;
    c.split = sp ? 1 : 0;
  }
  return c;
}

// Block-wide exclusive scan of three per-thread counts; total = block sums.
__device__ __forceinline__ int3 block_excl_scan3(int3 v, int3* s_warp, int3& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int3 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, x.x, o), b = __shfl_up_sync(0xffffffffu, x.y, o),
              c = __shfl_up_sync(0xffffffffu, x.z, o);
    if (lane >= o) x.x += a, x.y += b, x.z += c;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  int3 wb = make_int3(0, 0, 0), tot = make_int3(0, 0, 0);
#pragma unroll
  for (int w = 0; w < kCompactBlock / 32; ++w) {
    const int3 t = s_warp[w];
    if (w < warp) wb.x += t.x, wb.y += t.y, wb.z += t.z;
    tot.x += t.x, tot.y += t.y, tot.z += t.z;
  }
  total = tot;
  return make_int3(wb.x + x.x - v.x, wb.y + x.y - v.y, wb.z + x.z - v.z);
}

__global__ void __launch_bounds__(kCompactBlock) compact_count_kernel(const uint8_t* __restrict__ prune,
                                                                      const uint8_t* __restrict__ clone,
                                                                      const uint8_t* __restrict__ split, int64_t n,
                                                                      int3* __restrict__ block_counts) {
  __shared__ int3 s_warp[kCompactBlock / 32];
  const int64_t i0 = (int64_t)blockIdx.x * kCompactSpan + (int64_t)threadIdx.x * kCompactItems;
  int3 v = make_int3(0, 0, 0);
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) {
    const Classes c = classify(prune, clone, split, i0 + k, n);
    v.x += c.keep, v.y += c.clone, v.z += c.split;
  }
  int3 tot;
  block_excl_scan3(v, s_warp, tot);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

// One CTA of 1024 threads: exclusive scan of the block counts in place (four
// consecutive blocks per thread, chunks of 4096), the class totals into
// totals[0..2].
__global__ void __launch_bounds__(1024) compact_scan_blocks_kernel(int3* __restrict__ block_counts, int nb,
                                                                   long long* __restrict__ totals) {
  __shared__ int3 s_w[32];
  __shared__ int3 s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int3 carry = make_int3(0, 0, 0);
  for (int b0 = 0; b0 < nb; b0 += 4096) {
    const int b = b0 + 4 * (int)threadIdx.x;
    int3 v[4], sum = make_int3(0, 0, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = b + k < nb ? block_counts[b + k] : make_int3(0, 0, 0);
      sum.x += v[k].x, sum.y += v[k].y, sum.z += v[k].z;
    }
    int3 x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int p = __shfl_up_sync(0xffffffffu, x.x, o), q = __shfl_up_sync(0xffffffffu, x.y, o),
                r = __shfl_up_sync(0xffffffffu, x.z, o);
      if (lane >= o) x.x += p, x.y += q, x.z += r;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int3 w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int p = __shfl_up_sync(0xffffffffu, w.x, o), q = __shfl_up_sync(0xffffffffu, w.y, o),
                  r = __shfl_up_sync(0xffffffffu, w.z, o);
        if (lane >= o) w.x += p, w.y += q, w.z += r;
      }
      s_w[lane] = w;  // inclusive warp prefix
      if (lane == 31) s_carry = w;
    }
    __syncthreads();
    const int3 wp = warp > 0 ? s_w[warp - 1] : make_int3(0, 0, 0);
    int3 run = make_int3(carry.x + wp.x + x.x - sum.x, carry.y + wp.y + x.y - sum.y, carry.z + wp.z + x.z - sum.z);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (b + k < nb) block_counts[b + k] = run;
      run.x += v[k].x, run.y += v[k].y, run.z += v[k].z;
    }
    const int3 c = s_carry;
    carry.x += c.x, carry.y += c.y, carry.z += c.z;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    totals[0] = carry.x;
    totals[1] = carry.y;
    totals[2] = carry.z;
  }
}

// The clone step and the split children's geometry (adc.hpp:184-201) of
// source Gaussian i, written over the verbatim copies of its rows.
__device__ __forceinline__ void compact_geometry(const float* __restrict__ src, int64_t stride, int64_t i,
                                                 int64_t clone_slot, int64_t split_slot, int64_t split_rank,
                                                 const float* __restrict__ grad3d, const int* __restrict__ views_seen,
                                                 float clone_lr, const float* __restrict__ eps, float log_shrink,
                                                 float* __restrict__ dst, int64_t dstride) {
  // clone mu -= lr * grad3d / views_seen (adc.hpp:184-189)
  if (clone_slot >= 0) {
    const int seen = views_seen[i];
    if (seen > 0) {
      const float vs = (float)seen;
      for (int k = 0; k < 3; ++k)
        dst[(SK_COMP_MU + k) * dstride + clone_slot] =
            src[(SK_COMP_MU + k) * stride + i] - clone_lr * (grad3d[k * stride + i] / vs);
    }
  }
  // split children: mu = parent mu + R (eps * s), log_scale - ln 1.6 (adc.hpp:190-201)
  if (split_slot >= 0) {
    float qw = src[3 * stride + i], qx = src[4 * stride + i], qy = src[5 * stride + i], qz = src[6 * stride + i];
    const float n2 = ((qw * qw + qx * qx) + qy * qy) + qz * qz;
    if (n2 > 0.0f) {
      const float nq = sqrtf(n2);
      qw = qw / nq;
      qx = qx / nq;
      qy = qy / nq;
      qz = qz / nq;
    }
    float R[3][3];
    R[0][0] = 1.0f - 2.0f * (qy * qy + qz * qz);
    R[0][1] = 2.0f * (qx * qy - qw * qz);
    R[0][2] = 2.0f * (qx * qz + qw * qy);
    R[1][0] = 2.0f * (qx * qy + qw * qz);
    R[1][1] = 1.0f - 2.0f * (qx * qx + qz * qz);
    R[1][2] = 2.0f * (qy * qz - qw * qx);
    R[2][0] = 2.0f * (qx * qz - qw * qy);
    R[2][1] = 2.0f * (qy * qz + qw * qx);
    R[2][2] = 1.0f - 2.0f * (qx * qx + qy * qy);
    float sc[3];
    for (int k = 0; k < 3; ++k) sc[k] = det_expf(src[(SK_COMP_LOG_SCALE + k) * stride + i]);
    for (int child = 0; child < 2; ++child) {
      const int64_t d = split_slot + child;
      float es[3];
      for (int k = 0; k < 3; ++k) es[k] = eps[split_rank * 6 + child * 3 + k] * sc[k];
      for (int k = 0; k < 3; ++k) {
        const float off = (R[k][0] * es[0] + R[k][1] * es[1]) + R[k][2] * es[2];
        dst[(SK_COMP_MU + k) * dstride + d] = src[(SK_COMP_MU + k) * stride + i] + off;
        dst[(SK_COMP_LOG_SCALE + k) * dstride + d] = src[(SK_COMP_LOG_SCALE + k) * stride + i] - log_shrink;
      }
    }
  }
}

__global__ void __launch_bounds__(kCompactBlock) compact_move_kernel(
    const uint8_t* __restrict__ prune, const uint8_t* __restrict__ clone, const uint8_t* __restrict__ split, int64_t n,
    const int3* __restrict__ block_base, const long long* __restrict__ totals, int comps,
    const float* __restrict__ src, const float* __restrict__ m_src, const float* __restrict__ v_src, int64_t stride,
    float* __restrict__ dst, float* __restrict__ m_dst, float* __restrict__ v_dst, int64_t dstride,
    const float* __restrict__ grad3d, const int* __restrict__ views_seen, float clone_lr,
    const float* __restrict__ eps, float log_shrink, int32_t* __restrict__ old_to_new) {
  __shared__ int3 s_warp[kCompactBlock / 32];
  const int64_t i0 = (int64_t)blockIdx.x * kCompactSpan + (int64_t)threadIdx.x * kCompactItems;
  Classes cl[kCompactItems];
  int3 v = make_int3(0, 0, 0);
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) {
    cl[k] = classify(prune, clone, split, i0 + k, n);
    v.x += cl[k].keep, v.y += cl[k].clone, v.z += cl[k].split;
  }
  int3 tot;
  const int3 local = block_excl_scan3(v, s_warp, tot);
  if (i0 >= n) return;
  const int3 base = block_base[blockIdx.x];
  const int64_t n_keep = totals[0], n_clone = totals[1];
  // destination slots of the thread's Gaussians (-1: absent)
  int64_t keep_slot[kCompactItems], clone_slot[kCompactItems], split_slot[kCompactItems], split_rank[kCompactItems];
  {
    int64_t kr = base.x + local.x, cr = base.y + local.y, sr = base.z + local.z;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
      keep_slot[k] = cl[k].keep ? kr : -1;
      clone_slot[k] = cl[k].clone ? n_keep + cr : -1;
      split_slot[k] = cl[k].split ? n_keep + n_clone + 2 * sr : -1;
      split_rank[k] = sr;
      kr += cl[k].keep, cr += cl[k].clone, sr += cl[k].split;
    }
  }
  // blockIdx.y = component group: group 0 moves the 11 geometry / opacity rows
  // and then writes the clone / split geometry over its own copies; the SH
  // rows are split evenly over the other groups (about four rows each)
  const int g = blockIdx.y, groups = gridDim.y;
  const int c0 = g == 0 ? 0 : SK_COMP_SH + (int)((int64_t)(comps - SK_COMP_SH) * (g - 1) / (groups - 1));
  const int c1 = g == 0 ? SK_COMP_SH : SK_COMP_SH + (int)((int64_t)(comps - SK_COMP_SH) * g / (groups - 1));
  if (g == 0 && old_to_new)
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k)
      if (i0 + k < n) old_to_new[i0 + k] = (int32_t)keep_slot[k];
  // rows: survivors keep m / v, clones and split children start at zero;
  // all rows are loaded unconditionally so the loads of several components
  // are in flight together
#pragma unroll 4
  for (int comp = c0; comp < c1; ++comp) {
    const size_t co = (size_t)comp * dstride;
    float xs[kCompactItems], ms[kCompactItems], vs[kCompactItems];
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
      const size_t so = (size_t)comp * stride + i0 + k;
      xs[k] = src[so];
      ms[k] = m_src[so];
      vs[k] = v_src[so];
    }
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
      if (keep_slot[k] >= 0) {
        dst[co + keep_slot[k]] = xs[k];
        m_dst[co + keep_slot[k]] = ms[k];
        v_dst[co + keep_slot[k]] = vs[k];
      }
      if (clone_slot[k] >= 0) {
        dst[co + clone_slot[k]] = xs[k];
        m_dst[co + clone_slot[k]] = 0.0f;
        v_dst[co + clone_slot[k]] = 0.0f;
      }
      if (split_slot[k] >= 0) {
        dst[co + split_slot[k]] = xs[k];
        dst[co + split_slot[k] + 1] = xs[k];
        m_dst[co + split_slot[k]] = m_dst[co + split_slot[k] + 1] = 0.0f;
        v_dst[co + split_slot[k]] = v_dst[co + split_slot[k] + 1] = 0.0f;
      }
    }
  }
  if (g != 0) return;
#pragma unroll 1
  for (int k = 0; k < kCompactItems; ++k) {
    const int64_t i = i0 + k;
    if (i >= n) break;
    compact_geometry(src, stride, i, clone_slot[k], split_slot[k], split_rank[k], grad3d, views_seen, clone_lr, eps,
                     log_shrink, dst, dstride);
  }
}


unsigned blocks(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

// SK_TRACE_EVENTS=1: synchronising host timestamps of the density-event
// sub-steps on stderr (diagnostics only; off by default).
void trace_point(sk_ctx* ctx, const char* what) {
  static const bool on = std::getenv("SK_TRACE_EVENTS") != nullptr;
  if (!on) return;
  static auto last = std::chrono::steady_clock::now();
  SK_CUDA(cudaStreamSynchronize(ctx->stream));
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[event] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

}  // namespace

// photometric = (1 - lambda) mean(raw) + lambda (1 - ssim) (error_maps.hpp:40-41)
// from the loss sums on the device, with the host's arithmetic (finish_loss:
// double means, then float): no host round trip per scored view.
__global__ void photometric_kernel(const double* __restrict__ sums, int width, int height, float lambda,
                                   float* __restrict__ out) {
  const double npx = (double)width * height;
  const double l1 = sums[0] / (3.0 * npx);
  const double ssim = sums[1] / (3.0 * npx);
  *out = (1.0f - lambda) * (float)l1 + lambda * (1.0f - (float)ssim);
}

// Renders the k views and leaves s_d / s_p_raw / s_p in the scene's table.
// gt: device images (u8 HWC) or host float HWC images (staged per view).
// One scored view (adc.hpp:101-108): render, error maps, photometric term,
// and the masked count pass into `row`, on context c (its stream, scratch and
// error word) with frame f.
void score_view(sk_ctx* c, sk_scene* s, sk_frame* f, const sk_camera& cam, const void* gt_in, bool gt_u8_device,
                float tau, float lambda, const sk_binning& bin, int32_t* row, float* dphoto) {
  // No host synchronisation: the pair count stays on the device (an overflow
  // of the frame's pair buffer raises kErrPairOverflow; score_pass then
  // regrows and scores again) and the photometric term is formed on the device.
  const int64_t n = s->n;
  frame_geometry(f, cam.width, cam.height, &bin);
  f->camera = cam;
  ensure_projected(f, n);
  launch_preprocess(c, s, cam, f, /*extras=*/false);
  bin_sort(c, f, /*deferred=*/true);
  ensure_image(f);
  launch_blend_forward(c, f, nullptr, nullptr);
  f->rendered = true;
  const int64_t npx = (int64_t)cam.width * cam.height;
  const void* gt = gt_in;
  if (!gt_u8_device) {
    void* g = f->gt.ensure(sizeof(float) * 3 * npx);
    h2d(c, g, static_cast<const float*>(gt_in), 3 * npx);
    gt = g;
  }
  float* raw = ensure<float>(c->ev.raw, npx);
  uint8_t* mask = ensure<uint8_t>(c->ev.mask, npx);
  uint32_t* lohi = ensure<uint32_t>(c->ev.lohi, 4);
  SK_CUDA(cudaMemsetAsync(lohi, 0xff, sizeof(uint32_t), c->stream));  // min: all ones
  SK_CUDA(cudaMemsetAsync(lohi + 1, 0, sizeof(uint32_t), c->stream));  // max: zero
  error_raw_kernel<<<std::min<unsigned>(blocks(npx), 148 * 8), 256, 0, c->stream>>>(
      f->image.as<float>(), gt, gt_u8_device, cam.width, cam.height, raw, lohi);
  note_launch();
  error_mask_kernel<<<blocks(npx), 256, 0, c->stream>>>(raw, lohi, npx, tau, mask, nullptr);
  note_launch();
  launch_loss(c, f, gt, gt_u8_device, lambda, false, nullptr);
  photometric_kernel<<<1, 1, 0, c->stream>>>(c->scalars.as<double>(), cam.width, cam.height, lambda, dphoto);
  note_launch();
  launch_blend_forward(c, f, mask, row);
}

// The second context of the two-stream score pass (own stream, sort / event
// scratch and error word, plus its frame), created on first use.
sk_ctx* score_helper(sk_ctx* ctx) {
  if (!ctx->helper) {
    sk_ctx* h = nullptr;
    if (sk_ctx_create(ctx->device, &h) != SK_OK) throw CudaError("score pass: cannot create the helper stream");
    ctx->helper = h;
    ctx->helper_frame = new sk_frame();
  }
  return ctx->helper;
}

// Renders the k views and leaves s_d / s_p_raw / s_p in the scene's table.
// gt: device images (u8 HWC) or host float HWC images (staged per view).
// With device GT (the Trainer's event) the views are split over two host
// threads / two streams (even views on ctx, odd views on a helper context):
// each view's host synchronisations (the pair count, the photometric sums)
// then only stall its own stream while the other stream's kernels keep the
// GPU busy. Views are independent (own count row, own photometric slot), so
// the result is identical to the sequential pass.
void score_pass(sk_ctx* ctx, sk_scene* s, sk_frame* f, const std::vector<sk_camera>& cams,
                const std::vector<const void*>& gts, bool gt_u8_device, float tau, float lambda,
                const sk_binning& bin, std::vector<float>* photo_out, const sk_comm* comm = nullptr) {
  EventScratch& ev = ctx->ev;
  const int k = (int)cams.size();
  require(k > 0, "accumulate_scores: no training views");
  ensure_score_table(ctx, s);
  const int64_t n = s->n;
  const int world = comm ? comm->world : 1;
  const int rank = comm ? comm->rank : 0;
  // views sharded round-robin over ranks; rank r's views fill block r of the
  // rank-major rows [world][kpr][n] (C3 all-gathers the blocks)
  const int kpr = (k + world - 1) / world;
  const int slots = world * kpr;
  auto slot_of = [&](int j) { return (j % world) * kpr + j / world; };
  int32_t* rows = ensure<int32_t>(ev.rows, (size_t)slots * std::max<int64_t>(n, 1));
  uint32_t* lohi = ensure<uint32_t>(ev.lohi, 4);
  float* dphoto = ensure<float>(ev.photo, slots);
  std::vector<float> photo(slots, 0.0f);
  ctx->event_mark(0);
  std::vector<int> mine;
  for (int j = 0; j < k; ++j)
    if (j % world == rank) mine.push_back(j);
  auto run_view = [&](sk_ctx* c, sk_frame* fr, int j) {
    const int sl = slot_of(j);
    score_view(c, s, fr, cams[j], gts[j], gt_u8_device, tau, lambda, bin, rows + (size_t)sl * n, dphoto + sl);
  };
  // Views round-robin over S streams, each driven by its own host thread and
  // context (scratch, error word) with its own frame: the streams' kernels
  // overlap on the GPU (a view is a chain of small binning kernels around
  // the heavy blends). SK_SCORE_STREAMS overrides S (SK_SCORE_ONE_STREAM=1:
  // one); the result does not depend on S (own count rows and photometric
  // slots per view).
  const char* one = std::getenv("SK_SCORE_ONE_STREAM");  // runtime override (tests / diagnostics)
  const char* ns = std::getenv("SK_SCORE_STREAMS");
  int nstreams = ns ? std::max(1, std::atoi(ns)) : 3;  // measured: 2 -> 49.1, 3 -> 48.5, 4 -> 49.1 ms per event
  if ((one && one[0] == '1') || !gt_u8_device) nstreams = 1;
  nstreams = std::max(1, std::min<int>(nstreams, (int)mine.size()));
  std::vector<sk_ctx*> cs{ctx};
  std::vector<sk_frame*> fs{f};
  for (int i = 1; i < nstreams; ++i) {
    cs.push_back(score_helper(cs.back()));
    fs.push_back(cs[i - 1]->helper_frame);
  }
  for (int attempt = 0;; ++attempt) {
    SK_CUDA(cudaMemsetAsync(rows, 0, sizeof(int32_t) * (size_t)slots * n, ctx->stream));
    if (nstreams == 1) {
      for (const int j : mine) run_view(ctx, f, j);
    } else {
      prepare_loss(ctx);  // one-time constant upload, before the threads use it
      cudaEvent_t e0 = nullptr;
      SK_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
      SK_CUDA(cudaEventRecord(e0, ctx->stream));  // rows zeroed before any stream counts
      for (int i = 1; i < nstreams; ++i) SK_CUDA(cudaStreamWaitEvent(cs[i]->stream, e0, 0));
      std::vector<std::exception_ptr> errs(nstreams);
      std::vector<std::thread> th;
      for (int i = 1; i < nstreams; ++i)
        th.emplace_back([&, i] {
          try {
            SK_CUDA(cudaSetDevice(cs[i]->device));
            for (size_t v = i; v < mine.size(); v += nstreams) run_view(cs[i], fs[i], mine[v]);
          } catch (...) {
            errs[i] = std::current_exception();
          }
        });
      try {
        for (size_t v = 0; v < mine.size(); v += nstreams) run_view(ctx, f, mine[v]);
      } catch (...) {
        errs[0] = std::current_exception();
      }
      for (auto& t : th) t.join();
      for (int i = 1; i < nstreams; ++i) {
        cudaEvent_t e1 = nullptr;
        SK_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        SK_CUDA(cudaEventRecord(e1, cs[i]->stream));
        SK_CUDA(cudaStreamWaitEvent(ctx->stream, e1, 0));
        SK_CUDA(cudaStreamSynchronize(cs[i]->stream));
        cudaEventDestroy(e1);
      }
      cudaEventDestroy(e0);
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    }
    uint32_t bits = 0;
    for (sk_ctx* c : cs) bits |= read_error_word(c);  // synchronises
    raise_device_errors(bits);
    if (!(bits & kErrPairOverflow)) break;
    require(attempt < 8, "accumulate_scores: pair buffer still overflowing");
    for (sk_frame* fr : fs) ensure<uint32_t>(fr->pval_a, 2 * std::max<size_t>(fr->pval_a.bytes / sizeof(uint32_t), 1024));
  }
  if (world > 1) allgather_scores(const_cast<sk_comm*>(comm), rows, kpr, n, dphoto, ctx->stream);  // C3
  ctx->event_mark(1);
  SK_CUDA(cudaMemsetAsync(lohi, 0xff, sizeof(uint32_t), ctx->stream));  // min: all ones
  SK_CUDA(cudaMemsetAsync(lohi + 1, 0, sizeof(uint32_t), ctx->stream));  // max: zero
  if (n > 0) {
    scores_kernel<<<blocks(n), 256, 0, ctx->stream>>>(rows, n, dphoto, k, world, kpr, n, s->s_d.as<float>(),
                                                       s->s_p_raw.as<float>(), lohi);
    note_launch();
    minmax_normalize_kernel<<<blocks(n), 256, 0, ctx->stream>>>(s->s_p_raw.as<float>(), lohi, n, s->s_p.as<float>());
    note_launch();
  }
  SK_CUDA(cudaGetLastError());
  ctx->event_mark(2);
  if (photo_out) {
    d2h(ctx, photo.data(), dphoto, slots);
    sync(ctx);
    photo_out->resize(k);
    for (int j = 0; j < k; ++j) (*photo_out)[j] = photo[slot_of(j)];
  }
}

void select_densify_flags(sk_ctx* ctx, sk_scene* s, float tau_d, float thr, float percent_dense, bool use_vcd,
                          float extent, uint8_t* clone, uint8_t* split) {
  ensure_score_table(ctx, s);
  if (s->n == 0) return;
  densify_flags_kernel<<<blocks(s->n), 256, 0, ctx->stream>>>(
      s->params.as<float>(), s->capacity, s->n, s->s_d.as<float>(), s->grad_norm_acc.as<float>(),
      s->abs_grad_acc.as<float>(), s->views_seen.as<int>(), tau_d, thr, percent_dense * extent, use_vcd, clone, split);
  note_launch();
}

void select_prune_flags(sk_ctx* ctx, sk_scene* s, int iteration, const sk_prune_params& pp, float extent,
                        uint8_t* prune) {
  ensure_score_table(ctx, s);
  const int64_t n = s->n;
  if (n == 0) return;
  EventScratch& ev = ctx->ev;
  const bool early = iteration < pp.densify_until;
  int* count = reinterpret_cast<int*>(ensure<uint32_t>(ev.lohi, 4) + 2);
  SK_CUDA(cudaMemsetAsync(count, 0, sizeof(int), ctx->stream));
  uint32_t* key = nullptr;
  if (early && pp.use_vcp) key = ensure<uint32_t>(ev.keys_a, n);
  const float op_cut = pp.use_vcp ? pp.opacity_late : pp.min_opacity;
  prune_flags_kernel<<<blocks(n), 256, 0, ctx->stream>>>(
      s->params.as<float>(), s->capacity, n, s->s_p.as<float>(), s->max_radius2d.as<float>(), early,
      iteration > pp.size_prune_from, pp.min_opacity, pp.world_size_frac * extent, pp.screen_size, op_cut,
      pp.use_vcp != 0, pp.tau_p, prune, key, count);
  note_launch();
  if (early && pp.use_vcp) {
    // keep the ceil(|C|/2) highest-scoring candidates (ties by index) as pruned
    auto* stv = reinterpret_cast<SelectState*>(ensure<uint32_t>(ev.keys_b, 4 + 256));
    uint32_t* hist = reinterpret_cast<uint32_t*>(stv + 1);
    select_init_kernel<<<1, 256, 0, ctx->stream>>>(count, stv, hist);
    note_launch();
    const unsigned hb = (unsigned)std::min<int64_t>(blocks(n), 148 * 4);
    for (int shift = 24; shift >= 0; shift -= 8) {
      select_hist_kernel<<<hb, 256, 0, ctx->stream>>>(key, n, stv, shift, hist);
      select_step_kernel<<<1, 256, 0, ctx->stream>>>(stv, shift, hist);
      note_launch();
      note_launch();
    }
    const int nb = (int)blocks(n);
    int3* block_base = reinterpret_cast<int3*>(ensure<int32_t>(ev.cls, 3 * (size_t)nb));
    long long* totals = ensure<long long>(ev.totals, 3);
    select_tie_count_kernel<<<nb, 256, 0, ctx->stream>>>(key, n, stv, block_base);
    compact_scan_blocks_kernel<<<1, 1024, 0, ctx->stream>>>(block_base, nb, totals);
    select_take_kernel<<<nb, 256, 0, ctx->stream>>>(key, n, stv, block_base, prune);
    note_launch();
    note_launch();
    note_launch();
  }
  int host_count = 0;
  d2h(ctx, &host_count, count, 1);
  sync(ctx);
  if (early && pp.use_vcp) host_count = (host_count + 1) / 2;
  if (host_count == n && n > 0) {
    unsigned long long* best = reinterpret_cast<unsigned long long*>(ensure<uint32_t>(ev.lohi, 4));
    const unsigned long long init = ~0ull;
    h2d(ctx, best, &init, 1);
    argmin_kernel<<<blocks(n), 256, 0, ctx->stream>>>(s->s_p.as<float>(), n, best);
    note_launch();
    unsigned long long b = 0;
    d2h(ctx, &b, best, 1);
    sync(ctx);
    const int64_t keep = (int64_t)(b & 0xffffffffull);
    const uint8_t zero = 0;
    h2d(ctx, prune + keep, &zero, 1);
  }
  SK_CUDA(cudaGetLastError());
}

// K15 on device flags; returns the new size. eps_dev: [n_split][6].
// eps_source(n_split) returns the 6·n_split split normals (host memory),
// called once the split count is known from the device scans.
int64_t compact_scene(sk_ctx* ctx, sk_scene* s, const uint8_t* prune, const uint8_t* clone, const uint8_t* split,
                      float clone_lr, const std::function<const float*(int64_t)>& eps_source,
                      int32_t* old_to_new_dev) {
  EventScratch& ev = ctx->ev;
  gather_moments(s, ctx->stream);  // the compaction moves whole moment rows (sharded C1, comm.cu)
  const int64_t n = s->n;
  if (n == 0) return 0;
  const int nb = (int)((n + kCompactSpan - 1) / kCompactSpan);
  int3* block_base = reinterpret_cast<int3*>(ensure<int32_t>(ev.cls, 3 * (size_t)nb));
  long long* totals = ensure<long long>(ev.totals, 3);
  compact_count_kernel<<<nb, kCompactBlock, 0, ctx->stream>>>(prune, clone, split, n, block_base);
  note_launch();
  compact_scan_blocks_kernel<<<1, 1024, 0, ctx->stream>>>(block_base, nb, totals);
  note_launch();
  long long tot[3];
  d2h(ctx, tot, totals, 3);
  sync(ctx);
  const int64_t n_keep = tot[0], n_clone = tot[1], n_split = tot[2];
  const int64_t new_n = n_keep + n_clone + 2 * n_split;
  float* eps = ensure<float>(ev.eps, 6 * (size_t)std::max<int64_t>(n_split, 1));
  trace_point(ctx, "compact: class counts + scan");
  const float* eps_host = eps_source(n_split);
  trace_point(ctx, "compact: split normals");
  if (n_split > 0) {
    require(eps_host != nullptr, "apply_densify: split requires eps normals");
    h2d(ctx, eps, eps_host, 6 * (size_t)n_split);
  }
  trace_point(ctx, "compact: eps upload");
  ensure_optimizer_state(ctx, s);
  const int64_t new_cap =
      new_n > s->capacity ? round_capacity(std::max<int64_t>(new_n, s->capacity + s->capacity / 2)) : s->capacity;
  // Output into the scene's persistent spare buffers (grow-only), swapped in
  // below: no cudaMalloc / cudaFree of the ~0.7 GB-per-1M state per event.
  DevBuf& np = s->params_alt;
  DevBuf& nm = s->adam_m_alt;
  DevBuf& nv = s->adam_v_alt;
  const size_t cells = (size_t)s->comps * new_cap;
  ensure<float>(np, cells);
  ensure<float>(nm, cells);
  ensure<float>(nv, cells);
  trace_point(ctx, "compact: buffers");
  const int groups = 1 + std::max(1, (s->comps - SK_COMP_SH + 3) / 4);
  const bool timed = ctx->timing && ctx->ev.move_ev[0];
  if (timed) SK_CUDA(cudaEventRecord(ctx->ev.move_ev[0], ctx->stream));
  compact_move_kernel<<<dim3(nb, groups), kCompactBlock, 0, ctx->stream>>>(
      prune, clone, split, n, block_base, totals, s->comps, s->params.as<float>(), s->adam_m.as<float>(),
      s->adam_v.as<float>(), s->capacity, np.as<float>(), nm.as<float>(), nv.as<float>(), new_cap,
      s->grad3d_acc.as<float>(), s->views_seen.as<int>(), clone_lr, eps, (float)std::log(1.6), old_to_new_dev);
  note_launch();
  SK_CUDA(cudaGetLastError());
  if (timed) SK_CUDA(cudaEventRecord(ctx->ev.move_ev[1], ctx->stream));
  sync(ctx);
  if (timed) {
    float ms = 0.0f;
    SK_CUDA(cudaEventElapsedTime(&ms, ctx->ev.move_ev[0], ctx->ev.move_ev[1]));
    ctx->ev.move_ms += ms;
  }
  trace_point(ctx, "compact: kernel");
  s->params.swap(np);
  s->adam_m.swap(nm);
  s->adam_v.swap(nv);
  if (new_cap != s->capacity) {
    s->capacity = new_cap;
    s->grads.release();
    for (DevBuf* b : {&s->s_d, &s->s_p_raw, &s->s_p, &s->grad_norm_acc, &s->abs_grad_acc, &s->grad3d_acc,
                      &s->views_seen, &s->max_radius2d})
      b->release();
  }
  s->n = new_n;
  ensure_optimizer_state(ctx, s);
  reset_score_table(ctx, s);
  // clear_rest() (trainer.hpp:242): every event clears the lazy SH-rest
  // accumulator, also when the compaction leaves the size unchanged (the
  // indices moved, or nothing was removed).
  s->rest_n = -1;
  trace_point(ctx, "compact: state reset");
  return new_n;
}

// Trainer::density_event (trainer.hpp:177-243).
void density_event(sk_trainer* t, int it, bool densify, bool prune) {
  sk_ctx* ctx = t->ctx;
  sk_scene* s = t->scene;
  const sk_train_config& cfg = t->cfg;
  const std::vector<int> sampled = t->rng.sample_without_replacement((int)t->data->train.size(), cfg.k);
  std::vector<sk_camera> cams;
  std::vector<const void*> gts;
  EventRecord rec;
  rec.iteration = it;
  rec.n_before = (int)s->n;
  for (const int si : sampled) {
    const int v = t->data->train[si];
    cams.push_back(t->data->cams[v]);
    gts.push_back(t->data->images[v]->ptr);
    rec.sampled.push_back(v);
  }
  const sk_binning bin = binning_from(cfg);
  trace_point(ctx, "event: enter");
  allreduce_stats(t->comm, s, ctx->stream);  // C2
  score_pass(ctx, s, &t->frame, cams, gts, true, (float)cfg.tau, (float)cfg.lambda, bin, &rec.photometric, t->comm);
  trace_point(ctx, "score pass (K views, K13)");

  const int64_t n = s->n;
  uint8_t* flags = ensure<uint8_t>(ctx->ev.flags, 3 * (size_t)std::max<int64_t>(n, 1));
  uint8_t* fclone = flags;
  uint8_t* fsplit = flags + n;
  uint8_t* fprune = flags + 2 * n;
  SK_CUDA(cudaMemsetAsync(flags, 0, 3 * (size_t)n, ctx->stream));
  const float extent = t->data->extent;
  if (densify)
    select_densify_flags(ctx, s, (float)cfg.tau_d, (float)cfg.grad_threshold, (float)cfg.percent_dense, cfg.vcd != 0,
                         extent, fclone, fsplit);
  if (prune) {
    sk_prune_params pp;
    pp.tau_p = (float)cfg.tau_p;
    pp.min_opacity = (float)cfg.prune_min_opacity;
    pp.opacity_late = (float)cfg.prune_opacity_late;
    pp.world_size_frac = (float)cfg.prune_world_size_frac;
    pp.screen_size = (float)cfg.prune_screen_size;
    pp.size_prune_from = cfg.size_prune_from;
    pp.densify_until = cfg.densify_until;
    pp.use_vcp = cfg.vcp;
    select_prune_flags(ctx, s, it, pp, extent, fprune);
  }
  ctx->event_mark(3);
  trace_point(ctx, "select (K14)");
  // The split count (for the Rng) comes from the device scans inside
  // compact_scene; the flags are only downloaded for the event record.
  const float pos_lr = expon_lr((float)cfg.lr_position * extent, (float)cfg.lr_position_final * extent, it,
                                cfg.iterations);
  std::vector<uint8_t> h;
  if (t->record_events) {
    h.resize(3 * (size_t)n);
    d2h(ctx, h.data(), flags, h.size());
  }
  std::vector<float> eps;
  int64_t n_split = 0;
  compact_scene(ctx, s, fprune, fclone, fsplit, pos_lr,
                [&](int64_t ns) -> const float* {
                  // 6 normals per split Gaussian, ascending index order (adc.hpp:190-197)
                  n_split = ns;
                  eps.resize(6 * (size_t)ns);
                  t->rng.normals(eps.data(), eps.size());
                  return eps.data();
                },
                nullptr);
  ctx->event_mark(4);
  if (ctx->timing && ctx->ev.tev[0]) {
    SK_CUDA(cudaEventSynchronize(ctx->ev.tev[4]));
    for (int i = 0; i < SK_NUM_EVENT_PHASES; ++i) {
      float ms = 0.0f;
      SK_CUDA(cudaEventElapsedTime(&ms, ctx->ev.tev[i], ctx->ev.tev[i + 1]));
      ctx->ev.phase_ms[i] += ms;
    }
    ++ctx->ev.timed_events;
  }
  if (t->record_events) {
    rec.prune.assign(h.begin() + 2 * n, h.begin() + 3 * n);
    rec.clone.assign(h.begin(), h.begin() + n);
    rec.split.assign(h.begin() + n, h.begin() + 2 * n);
    int64_t n_clone = 0, n_prune = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (rec.prune[i]) rec.clone[i] = rec.split[i] = 0;
      n_prune += rec.prune[i] != 0;
      n_clone += rec.clone[i] != 0;
    }
    rec.n_clone = (int)n_clone;
    rec.n_split = (int)n_split;
    rec.n_prune = (int)n_prune;
    rec.n_after = (int)s->n;
    t->events.push_back(std::move(rec));
  }
}

}  // namespace sk

using namespace sk;

extern "C" {

void sk_default_prune_params(sk_prune_params* p) {
  if (!p) return;
  *p = sk_prune_params{(float)0.9, (float)0.005, (float)0.1, (float)0.1, 20.0f, 3000, 15000, 1};
}

int sk_accumulate_scores(sk_ctx* ctx, sk_scene* s, int k, const sk_camera* cams, const float* images, float tau,
                         float lambda, const sk_binning* b, int32_t* counts_out, float* photo_out) {
  return guarded(ctx, [&] {
    require(k > 0, "accumulate_scores: no training views");
    arg(s && cams && images, "accumulate_scores: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    std::vector<sk_camera> cv(cams, cams + k);
    std::vector<const void*> gts;
    size_t off = 0;
    for (int j = 0; j < k; ++j) {
      gts.push_back(images + off);
      off += (size_t)cams[j].width * cams[j].height * 3;
    }
    sk_frame f;
    std::vector<float> photo;
    const sk_binning bin = b ? *b : sk_binning{0, 1.0f, (float)(1.0 / 255), 16};
    score_pass(ctx, s, &f, cv, gts, false, tau, lambda, bin, &photo);
    if (counts_out && s->n > 0) d2h(ctx, counts_out, ctx->ev.rows.ptr, (size_t)k * s->n);
    sync(ctx);
    if (photo_out) std::copy(photo.begin(), photo.end(), photo_out);
  });
}

// build_error_maps (error_maps.hpp:22-43) on explicit images: K11 raw map and
// min / max, the normalized map and strict mask, and the photometric term
// (K7 forward for the SSIM).
int sk_error_maps(sk_ctx* ctx, const float* rendered, const float* gt, int width, int height, float tau, float lambda,
                  float* raw_out, float* normalized_out, uint8_t* mask_out, float* photometric) {
  return guarded(ctx, [&] {
    arg(rendered && gt && width > 0 && height > 0, "build_error_maps: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    sk_frame f;
    frame_geometry(&f, width, height, nullptr);
    ensure_image(&f);
    const int64_t npx = (int64_t)width * height;
    hwc_to_planar(ctx, f.image.ptr, rendered, width, height);
    f.rendered = true;
    void* g = f.gt.ensure(sizeof(float) * 3 * npx);
    h2d(ctx, g, gt, 3 * npx);
    float* raw = ensure<float>(ctx->ev.raw, npx);
    uint8_t* mask = ensure<uint8_t>(ctx->ev.mask, npx);
    float* nrm = ensure<float>(f.loss_scratch, npx);
    uint32_t* lohi = ensure<uint32_t>(ctx->ev.lohi, 4);
    const uint32_t init[2] = {0xffffffffu, 0u};
    h2d(ctx, lohi, init, 2);
    error_raw_kernel<<<std::min<unsigned>(blocks(npx), 148 * 8), 256, 0, ctx->stream>>>(f.image.as<float>(), g, false,
                                                                                         width, height, raw, lohi);
    note_launch();
    error_mask_kernel<<<blocks(npx), 256, 0, ctx->stream>>>(raw, lohi, npx, tau, mask, nrm);
    note_launch();
    LossSums sums{};
    launch_loss(ctx, &f, g, false, lambda, false, &sums);
    sk_loss_values v{};
    finish_loss(width, height, lambda, sums, &v);
    if (photometric) *photometric = (1.0f - lambda) * (float)v.l1 + lambda * (1.0f - (float)v.ssim);
    if (raw_out) d2h(ctx, raw_out, raw, npx);
    if (normalized_out) d2h(ctx, normalized_out, nrm, npx);
    if (mask_out) d2h(ctx, mask_out, mask, npx);
    sync(ctx);
  });
}

// scores_from_counts (adc.hpp:69-84) on explicit count rows: K13.
int sk_scores_from_counts(sk_ctx* ctx, const int32_t* counts, const float* photometric, int k, int64_t n, float* s_d,
                          float* s_p_raw, float* s_p) {
  return guarded(ctx, [&] {
    require(k > 0, "scores_from_counts: need one count row and one photometric value per view");
    arg(n >= 0 && (n == 0 || counts) && photometric, "scores_from_counts: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    if (n == 0) return;
    int32_t* rows = ensure<int32_t>(ctx->ev.rows, (size_t)k * n);
    float* dphoto = ensure<float>(ctx->ev.photo, k);
    DevBuf out;
    float* o = ensure<float>(out, 3 * (size_t)n);
    uint32_t* lohi = ensure<uint32_t>(ctx->ev.lohi, 4);
    h2d(ctx, rows, counts, (size_t)k * n);
    h2d(ctx, dphoto, photometric, k);
    const uint32_t init[2] = {0xffffffffu, 0u};
    h2d(ctx, lohi, init, 2);
    scores_kernel<<<blocks(n), 256, 0, ctx->stream>>>(rows, n, dphoto, k, 1, k, n, o, o + n, lohi);
    note_launch();
    minmax_normalize_kernel<<<blocks(n), 256, 0, ctx->stream>>>(o + n, lohi, n, o + 2 * n);
    note_launch();
    SK_CUDA(cudaGetLastError());
    if (s_d) d2h(ctx, s_d, o, n);
    if (s_p_raw) d2h(ctx, s_p_raw, o + n, n);
    if (s_p) d2h(ctx, s_p, o + 2 * n, n);
    sync(ctx);
  });
}

int sk_select_densify(sk_ctx* ctx, sk_scene* s, float tau_d, float thr, float percent_dense, int use_vcd,
                      float extent, uint8_t* clone, uint8_t* split) {
  return guarded(ctx, [&] {
    arg(s && clone && split, "select_densify: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = s->n;
    uint8_t* f = ensure<uint8_t>(ctx->ev.flags, 3 * (size_t)std::max<int64_t>(n, 1));
    select_densify_flags(ctx, s, tau_d, thr, percent_dense, use_vcd != 0, extent, f, f + n);
    d2h(ctx, clone, f, n);
    d2h(ctx, split, f + n, n);
    sync(ctx);
  });
}

int sk_select_prune(sk_ctx* ctx, sk_scene* s, int iteration, const sk_prune_params* pp, float extent,
                    uint8_t* prune) {
  return guarded(ctx, [&] {
    arg(s && pp && prune, "select_prune: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = s->n;
    uint8_t* f = ensure<uint8_t>(ctx->ev.flags, 3 * (size_t)std::max<int64_t>(n, 1));
    select_prune_flags(ctx, s, iteration, *pp, extent, f + 2 * n);
    d2h(ctx, prune, f + 2 * n, n);
    sync(ctx);
  });
}

int sk_apply_prune_densify(sk_ctx* ctx, sk_scene* s, const uint8_t* prune, const uint8_t* clone, const uint8_t* split,
                           float clone_lr, const float* eps, int32_t* old_to_new, int64_t* new_size) {
  return guarded(ctx, [&] {
    arg(s != nullptr, "apply_densify: null scene");
    SK_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = s->n;
    uint8_t* f = ensure<uint8_t>(ctx->ev.flags, 3 * (size_t)std::max<int64_t>(n, 1));
    SK_CUDA(cudaMemsetAsync(f, 0, 3 * (size_t)n, ctx->stream));
    if (clone) h2d(ctx, f, clone, n);
    if (split) h2d(ctx, f + n, split, n);
    if (prune) h2d(ctx, f + 2 * n, prune, n);
    int32_t* o2n = old_to_new ? ensure<int32_t>(ctx->ev.old_to_new, (size_t)std::max<int64_t>(n, 1)) : nullptr;
    ensure_score_table(ctx, s);
    const int64_t nn = compact_scene(ctx, s, f + 2 * n, f, f + n, clone_lr, [&](int64_t) { return eps; }, o2n);
    if (old_to_new && n > 0) d2h(ctx, old_to_new, o2n, n);
    sync(ctx);
    if (new_size) *new_size = nn;
  });
}

int sk_trainer_record_events(sk_trainer* t, int on) {
  if (!t) return SK_ERR_INVALID_ARGUMENT;
  t->record_events = on != 0;
  return SK_OK;
}

int sk_trainer_num_events(const sk_trainer* t, int* n) {
  if (!t || !n) return SK_ERR_INVALID_ARGUMENT;
  *n = (int)t->events.size();
  return SK_OK;
}

int sk_trainer_event(const sk_trainer* t, int e, int32_t* header, uint8_t* clone, uint8_t* split, uint8_t* prune,
                     int32_t* sampled, float* photometric) {
  if (!t || e < 0 || e >= (int)t->events.size()) return SK_ERR_INVALID_ARGUMENT;
  const EventRecord& r = t->events[e];
  if (header) {
    header[0] = r.iteration;
    header[1] = r.n_before;
    header[2] = r.n_after;
    header[3] = r.n_clone;
    header[4] = r.n_split;
    header[5] = r.n_prune;
    header[6] = (int32_t)r.sampled.size();
  }
  if (clone) std::copy(r.clone.begin(), r.clone.end(), clone);
  if (split) std::copy(r.split.begin(), r.split.end(), split);
  if (prune) std::copy(r.prune.begin(), r.prune.end(), prune);
  if (sampled) std::copy(r.sampled.begin(), r.sampled.end(), sampled);
  if (photometric) std::copy(r.photometric.begin(), r.photometric.end(), photometric);
  return SK_OK;
}

}  // extern "C"
