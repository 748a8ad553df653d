// Deterministic fp32 transcendentals for the bit-exact part of the hot path.
//
// The reference evaluates std::exp / std::log (splatkit scene.hpp:25 scale(),
// types.hpp:28-30 sigmoid, raster.hpp:81 compact_threshold, raster.hpp:228 the
// blend alpha). glibc and CUDA libm do not agree to the last ulp, so a Gaussian
// sitting on a tile or alpha boundary could bin or blend differently on the CPU
// oracle and on the GPU. These helpers use only IEEE +,-,*,/ and integer bit
// operations in a fixed order, so they produce identical bits on the host
// (compiled with -ffp-contract=off, no FMA) and on sm_100a (compiled with
// -fmad=false, IEEE div/sqrt, no flush-to-zero). Accuracy is 1-2 ulp against
// the correctly rounded result; tests/test_detmath.py checks that bound.
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

// e^x. Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2, degree-7 Taylor
// polynomial in Horner form, then two exact power-of-two scalings.
SK_HD float det_expf(float x) {
  if (!(x == x)) return x;                       // NaN propagates
  if (x > 88.72283f) return bits_to_f32(0x7f800000u);  // +inf
  if (x < -103.97208f) return 0.0f;              // below the smallest subnormal
  const float kf = det_floorf(x * 1.44269504088896341f + 0.5f);
  const int k = (int)kf;
  const float r = (x - kf * 0.693145751953125f) - kf * 1.428606820309417232e-06f;
  float p = 1.98412698412698413e-04f;  // 1/5040
  p = p * r + 1.38888888888888889e-03f;  // 1/720
  p = p * r + 8.33333333333333333e-03f;  // 1/120
  p = p * r + 4.16666666666666667e-02f;  // 1/24
  p = p * r + 1.66666666666666667e-01f;  // 1/6
  p = p * r + 0.5f;
  p = p * r + 1.0f;
  p = p * r + 1.0f;
  const int k1 = k / 2;
  const int k2 = k - k1;
  const float s1 = bits_to_f32((uint32_t)(k1 + 127) << 23);
  const float s2 = bits_to_f32((uint32_t)(k2 + 127) << 23);
  return (p * s1) * s2;
}

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
SK_HD float det_sigmoidf(float x) { return 1.0f / (1.0f + det_expf(-x)); }

}  // namespace sk
