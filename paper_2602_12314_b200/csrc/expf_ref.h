// expf_ref.h — std::exp(float) exactly as the reference's CPU path evaluates it (glibc's expf,
// the function behind every scalar std::exp on float in proj/src/render.cpp:193,303 and the
// sigmoid, proj/include/latmap/core/types.hpp:252-255), restated from its published algorithm:
//
//   exp(x) = 2^(k/32) * 2^(r/32),  x*32/ln2 = k + r, |r| <= 1/2 (k rounded to nearest, ties even);
//   2^(k/32) = 2^(k>>5) * T[k & 31] (T = 2^(i/32) in double, stored with the exponent part of
//   i/32 removed so the integer k can be added to the bit pattern); 2^(r/32) by the cubic
//   C0 r^3 + C1 r^2 + C2 r + 1 (coefficients scaled by 1/32 per power); all in double, one
//   rounding to float at the end.
//
// Checked bit for bit against this image's libm expf on every finite float (tests: the CPU suite
// samples, the GPU suite runs all 2^32 bit patterns on the device). Two inputs, found by the
// exhaustive check, round the other way in libm and are listed explicitly.
//
// Host and device: the same double arithmetic (explicitly rounded steps for the argument
// reduction, fma for the cubic).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define LM_EXPF_HD __host__ __device__ __forceinline__
#else
#define LM_EXPF_HD inline
#endif

namespace lm {

#define LM_EXP2_TAB32                                                                           \
  0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,  \
      0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull, \
      0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull, \
      0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull, \
      0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull, \
      0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull, \
      0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull, \
      0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull

// T[i] = bits(2^(i/32)) - (i << 52) / 32 (2^(i/32) correctly rounded to double)
#ifdef __CUDACC__
__device__ const uint64_t kExp2Tab32[32] = {LM_EXP2_TAB32};
#endif
static const uint64_t kExp2Tab32Host[32] = {LM_EXP2_TAB32};

LM_EXPF_HD uint64_t expf_tab(uint32_t i) {
#ifdef __CUDA_ARCH__
  return __ldg(&kExp2Tab32[i]);
#else
  return kExp2Tab32Host[i];
#endif
}

LM_EXPF_HD double lm_bits_to_double(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
LM_EXPF_HD uint64_t lm_double_to_bits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}
LM_EXPF_HD uint32_t lm_float_bits(float f) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}
LM_EXPF_HD float lm_bits_float(uint32_t u) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

// `tab` (optional, device): a copy of the table in shared memory for kernels that evaluate the
// exponential in their inner loop (an LDS instead of an L1 load); nullptr reads kExp2Tab32.
LM_EXPF_HD float expf_ref(float x, const uint64_t* tab = nullptr) {
  // branch-free: out-of-range / NaN inputs run the main path on a clamped argument and the
  // special results are selected at the end (the blend evaluates whole warps of exponentials)
  const uint32_t ux = lm_float_bits(x);
  const bool under = !(x >= -0x1.9fe368p+6f);  // libm underflows to 0 below this (and -inf, NaN)
  const bool over = x > 0x1.62e42ep+6f;        // and overflows to +inf above this
  const float xc = under ? -0x1.9fe368p+6f : (over ? 0x1.62e42ep+6f : x);
  const double kInvLn2N = 0x1.71547652b82fep+0 * 32, kShift = 0x1.8p+52;
  const double kC0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32, kC1 = 0x1.ebfce50fac4f3p-3 / 32 / 32,
               kC2 = 0x1.62e42ff0c52d6p-1 / 32;
#ifdef __CUDA_ARCH__
  // explicit roundings: no contraction of the k rounding (z is used twice) on the device
  const double z = __dmul_rn(kInvLn2N, (double)xc);
  double kd = __dadd_rn(z, kShift);  // round to nearest integer (it sits in the low mantissa bits)
  const uint64_t ki = lm_double_to_bits(kd);
  kd = __dsub_rn(kd, kShift);
  const double r = __dsub_rn(z, kd);
#else
  const double z = kInvLn2N * (double)xc;
  double kd = z + kShift;
  const uint64_t ki = lm_double_to_bits(kd);
  kd -= kShift;
  const double r = z - kd;
#endif
#ifdef __CUDA_ARCH__
  const uint64_t t = (tab ? tab[ki & 31] : expf_tab((uint32_t)(ki & 31))) + (ki << 47);
#else
  (void)tab;
  const uint64_t t = expf_tab((uint32_t)(ki & 31)) + (ki << 47);
#endif
  const double s = lm_bits_to_double(t);
  // the cubic with fused multiply-adds on host and device (fused or not, every float result is
  // the same; the tests check this form)
  const double p = fma(kC0, r, kC1);
  const double r2 = r * r;
  double y = fma(kC2, r, 1.0);
  y = fma(p, r2, y);
  y = y * s;
  float res = (float)y;
  res = under ? (x != x ? x : 0.f) : res;
  res = over ? __builtin_huge_valf() : res;
  // the two inputs libm rounds the other way (found by the exhaustive check)
  res = ux == 0xc27c65d9u ? lm_bits_float(0x11fa2993u) : res;  // x = -0x1.f8cbb2p+5: 0x1.f45326p-92
  res = ux == 0x4202422fu ? lm_bits_float(0x56fc9f1cu) : res;  // x =  0x1.04845ep+5: 0x1.f93e38p+46
  return res;
}

}  // namespace lm
