// Deterministic fp32 transcendentals for the bit-exact part of the hot path.
//
// The reference evaluates std::exp / std::log (splatkit scene.hpp:25 scale(),
// types.hpp:28-30 sigmoid, raster.hpp:81 compact_threshold, raster.hpp:228 the
// blend alpha). glibc and CUDA libm do not agree to the last ulp, so a Gaussian
// sitting on a tile or alpha boundary could bin or blend differently on the CPU
// oracle and on the GPU. These helpers use only IEEE +,-,*,/, exact power-of-
// two scalings, a fixed 64-entry table and integer bit operations in a fixed
// order, so they produce identical bits on the host (compiled with
// -ffp-contract=off, no FMA) and on sm_100a (compiled with -fmad=false, IEEE
// div/sqrt, no flush-to-zero). Accuracy is within 2 ulp of the correctly
// rounded result; tests/test_oracle_kats.py checks that bound.
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SK_HD __host__ __device__ __forceinline__
#else
#define SK_HD inline
#endif

namespace sk {

SK_HD float bits_to_f32(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

SK_HD uint32_t f32_to_bits(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}

SK_HD float det_floorf(float x) {
#if defined(__CUDA_ARCH__)
  return floorf(x);
#else
  return __builtin_floorf(x);
#endif
}

// Round-to-nearest products and sums that the device compiler never fuses
// into FMAs, so functions written with them give the same bits in
// translation units compiled with or without -fmad=false.
SK_HD float rn_mul(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}
SK_HD float rn_add(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}
SK_HD float rn_sub(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fsub_rn(a, b);
#else
  return a - b;
#endif
}

// 2^(j/64), j = 0..63, rounded to float (bit patterns, identical everywhere).
#define SK_EXP2_TABLE                                                                                            \
  {0x3f800000u, 0x3f8164d2u, 0x3f82cd87u, 0x3f843a29u, 0x3f85aac3u, 0x3f871f62u, 0x3f88980fu, 0x3f8a14d5u,      \
   0x3f8b95c2u, 0x3f8d1adfu, 0x3f8ea43au, 0x3f9031dcu, 0x3f91c3d3u, 0x3f935a2bu, 0x3f94f4f0u, 0x3f96942du,      \
   0x3f9837f0u, 0x3f99e046u, 0x3f9b8d3au, 0x3f9d3edau, 0x3f9ef532u, 0x3fa0b051u, 0x3fa27043u, 0x3fa43516u,      \
   0x3fa5fed7u, 0x3fa7cd94u, 0x3fa9a15bu, 0x3fab7a3au, 0x3fad583fu, 0x3faf3b79u, 0x3fb123f6u, 0x3fb311c4u,      \
   0x3fb504f3u, 0x3fb6fd92u, 0x3fb8fbafu, 0x3fbaff5bu, 0x3fbd08a4u, 0x3fbf179au, 0x3fc12c4du, 0x3fc346cdu,      \
   0x3fc5672au, 0x3fc78d75u, 0x3fc9b9beu, 0x3fcbec15u, 0x3fce248cu, 0x3fd06334u, 0x3fd2a81eu, 0x3fd4f35bu,      \
   0x3fd744fdu, 0x3fd99d16u, 0x3fdbfbb8u, 0x3fde60f5u, 0x3fe0ccdfu, 0x3fe33f89u, 0x3fe5b907u, 0x3fe8396au,      \
   0x3feac0c7u, 0x3fed4f30u, 0x3fefe4bau, 0x3ff28177u, 0x3ff5257du, 0x3ff7d0dfu, 0x3ffa83b3u, 0x3ffd3e0cu}

#if defined(__CUDACC__)
__constant__ const uint32_t kExp2TableDev[64] = SK_EXP2_TABLE;
#endif
static const uint32_t kExp2TableHost[64] = SK_EXP2_TABLE;

// e^x for x in [-87, 88] (normal-range result). x = (64k + j) ln2/64 + r with
// |r| <= ln2/128 (Cody-Waite split of ln2/64 into a 9-bit head, so kf * head
// is exact for |k| < 2^14), e^r by a degree-3 polynomial, then the table and
// one exact power-of-two scaling. `table` holds the 64 SK_EXP2_TABLE floats.
template <class Tab>
SK_HD float det_expf_core_t(float x, const Tab& table) {
  const float kf = det_floorf(rn_add(rn_mul(x, 92.33248261689366f), 0.5f));  // 64 / ln2
  const int k = (int)kf;
  const float r = rn_sub(rn_sub(x, rn_mul(kf, 0.010833740234375f)), rn_mul(kf, -3.3155381258549027e-06f));
  float p = rn_add(rn_mul(r, 0.16666666666666666f), 0.5f);
  p = rn_add(rn_mul(p, r), 1.0f);
  p = rn_add(rn_mul(p, r), 1.0f);
  const int j = k & 63;
  const int e = (k - j) / 64;
  return rn_mul(rn_mul(table[j], p), bits_to_f32((uint32_t)(e + 127) << 23));
}

SK_HD float det_expf_core(float x, const float* table) { return det_expf_core_t(x, table); }

#if defined(__CUDACC__)
// The exp table staged in shared memory, read with ld.shared through a
// 32-bit shared-window address computed once per kernel (indexing a generic
// pointer to shared memory re-derives the CTA's window base on every access).
struct SmemTable {
  uint32_t base;
  __device__ explicit SmemTable(const float* s) : base((uint32_t)__cvta_generic_to_shared(s)) {}
  __device__ __forceinline__ float operator[](int j) const {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(base + 4u * (uint32_t)j));
    return v;
  }
};
// The same table with its shared-window base pinned in a register.
struct SmemPinnedTable {
  uint32_t base;
  // the asm keeps the converted address in one register (otherwise it is
  // rematerialised with an S2R of the cluster CTA id at every lookup)
  __device__ explicit SmemPinnedTable(const float* s) {
    asm volatile("mov.u32 %0, %1;" : "=r"(base) : "r"((uint32_t)__cvta_generic_to_shared(s)));
  }
  __device__ __forceinline__ float operator[](int j) const {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(base + 4u * (uint32_t)j));
    return v;
  }
};
SK_HD float det_expf_core(float x, const SmemTable& table) { return det_expf_core_t(x, table); }
SK_HD float det_expf_core(float x, const SmemPinnedTable& table) { return det_expf_core_t(x, table); }
#endif

SK_HD const float* exp2_table() {
#if defined(__CUDA_ARCH__)
  return reinterpret_cast<const float*>(kExp2TableDev);
#else
  return reinterpret_cast<const float*>(kExp2TableHost);
#endif
}

// e^x for any float: special cases, then the core (two scalings keep the
// subnormal / overflow ends exact). Kernels with many calls pass a copy of
// the table staged in shared memory (constant memory serialises divergent
// indices).
template <class Tab>
SK_HD float det_expf_t(float x, const Tab& table) {
  if (!(x == x)) return x;                             // NaN propagates
  if (x > 88.72283f) return bits_to_f32(0x7f800000u);  // +inf
  if (x < -103.97208f) return 0.0f;                    // below the smallest subnormal
  if (x >= -87.0f && x <= 88.0f) return det_expf_core_t(x, table);
  const float kf = det_floorf(x * 92.33248261689366f + 0.5f);
  const int k = (int)kf;
  const float r = (x - kf * 0.010833740234375f) - kf * -3.3155381258549027e-06f;
  float p = r * 0.16666666666666666f + 0.5f;
  p = p * r + 1.0f;
  p = p * r + 1.0f;
  const int j = k & 63;
  const int e = (k - j) / 64;
  const int e1 = e / 2;
  const int e2 = e - e1;
  const float t = table[j] * p;
  return (t * bits_to_f32((uint32_t)(e1 + 127) << 23)) * bits_to_f32((uint32_t)(e2 + 127) << 23);
}

SK_HD float det_expf(float x, const float* table = nullptr) { return det_expf_t(x, table ? table : exp2_table()); }
#if defined(__CUDACC__)
SK_HD float det_expf(float x, const SmemTable& table) { return det_expf_t(x, table); }
SK_HD float det_expf(float x, const SmemPinnedTable& table) { return det_expf_t(x, table); }
#endif

// Natural log of a positive finite float. x = m 2^e with m in [sqrt(.5),
// sqrt(2)); log m = 2 atanh(s), s = (m-1)/(m+1), odd series to s^9.
SK_HD float det_logf(float x) {
  if (!(x == x)) return x;
  if (x < 0.0f) return bits_to_f32(0x7fc00000u);   // NaN
  if (x == 0.0f) return bits_to_f32(0xff800000u);  // -inf
  if (x == bits_to_f32(0x7f800000u)) return x;
  int e_adj = 0;
  if (x < 1.17549435e-38f) {  // subnormal: renormalise exactly
    x = x * 8388608.0f;
    e_adj = -23;
  }
  const uint32_t u = f32_to_bits(x);
  int e = (int)((u >> 23) & 0xffu) - 127 + e_adj;
  float m = bits_to_f32((u & 0x007fffffu) | 0x3f800000u);
  if (m > 1.41421356f) {
    m = m * 0.5f;
    e = e + 1;
  }
  const float f = m - 1.0f;
  const float s = f / (2.0f + f);
  const float s2 = s * s;
  float poly = 1.11111111111111111e-01f;        // 1/9
  poly = poly * s2 + 1.42857142857142857e-01f;  // 1/7
  poly = poly * s2 + 2.0e-01f;                  // 1/5
  poly = poly * s2 + 3.33333333333333333e-01f;  // 1/3
  const float two_s = 2.0f * s;
  const float logm = two_s + (two_s * s2) * poly;
  const float ef = (float)e;
  return ef * 0.693145751953125f + (logm + ef * 1.428606820309417232e-06f);
}

// Activation used by the reference (types.hpp:28-30): 1 / (1 + e^{-x}).
SK_HD float det_sigmoidf(float x, const float* table = nullptr) { return 1.0f / (1.0f + det_expf(-x, table)); }
#if defined(__CUDACC__)
SK_HD float det_sigmoidf(float x, const SmemTable& table) { return 1.0f / (1.0f + det_expf(-x, table)); }
SK_HD float det_sigmoidf(float x, const SmemPinnedTable& table) { return 1.0f / (1.0f + det_expf(-x, table)); }
#endif

#if defined(__CUDACC__)
// e^x on [-5.71, 0] for the blend kernels (x = -q/2 with q <= q_cut < 11.11).
// Same Cody-Waite reduction and polynomial as det_expf_core, but the table
// is indexed by m = -k and already carries the power of two:
// T[m] = table[k & 63] * 2^((k - (k & 63)) / 64), built by adding the exponent
// to the table bits (exact). Since the scaling by 2^e is exact in the normal
// range, rn(T[m] * p) == rn(rn(table[j] * p) * 2^e): bit-identical to
// det_expf_core, with the index / exponent integer work removed.
constexpr int kNegExpTable = 528;
__device__ __forceinline__ void stage_neg_exp_table(float* s_table) {
  for (int m = threadIdx.x; m < kNegExpTable; m += blockDim.x) {
    const int k = -m, j = k & 63, e = (k - j) / 64;
    s_table[m] = bits_to_f32(kExp2TableDev[j] + ((uint32_t)e << 23));
  }
}
template <class Tab>
__device__ __forceinline__ float det_expf_neg(float x, const Tab& neg_table) {
  const float kf = det_floorf(rn_add(rn_mul(x, 92.33248261689366f), 0.5f));  // 64 / ln2
  const float r = rn_sub(rn_sub(x, rn_mul(kf, 0.010833740234375f)), rn_mul(kf, -3.3155381258549027e-06f));
  float p = rn_add(rn_mul(r, 0.16666666666666666f), 0.5f);
  p = rn_add(rn_mul(p, r), 1.0f);
  p = rn_add(rn_mul(p, r), 1.0f);
  return rn_mul(neg_table[-(int)kf], p);
}
#endif

#if defined(__CUDACC__)
// Stages the exp table into shared memory; call from all threads, then sync.
__device__ __forceinline__ void stage_exp2_table(float* s_table) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_table[i] = bits_to_f32(kExp2TableDev[i]);
}
#endif

}  // namespace sk
