// common.cuh — shared device helpers for the latent-map step kernels (sm_100a).
#pragma once
#include "expf_ref.h"
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace lm {

// Exact IEEE round-to-nearest float ops (no FMA contraction). Used wherever a
// discrete decision (bbox, clamp, termination, sort key) or bit-exact parity with
// the oracle depends on the rounding sequence of the reference's float code.
__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fd(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds_(double a, double b) { return __dsub_rn(a, b); }

// std::exp(float) bit for bit as the reference evaluates it on the CPU (glibc expf, restated in
// expf_ref.h; checked on all 2^32 inputs) — the oracle calls the same libm function.
__device__ __forceinline__ float exp_exact(float x) { return expf_ref(x); }
// the same with the 2^(i/32) table staged in shared memory (load_exp_table; inner loops)
__device__ __forceinline__ float exp_exact(float x, const uint64_t* s_tab) { return expf_ref(x, s_tab); }
// stage kExp2Tab32 into a 32-entry shared array (threads 0..31; caller synchronises)
__device__ __forceinline__ void load_exp_table(uint64_t* s_tab) {
  if (threadIdx.x < 32) s_tab[threadIdx.x] = kExp2Tab32[threadIdx.x];
}

// sigmoid, core/types.hpp:252-255
__device__ __forceinline__ float sigmoid_exact(float x) {
  if (x >= 0.f) return fd(1.f, fa(1.f, exp_exact(-x)));
  const float e = exp_exact(x);
  return fd(e, fa(1.f, e));
}

constexpr int kTile = 16;                 // tile edge in pixels
constexpr int kTilePixels = kTile * kTile;
constexpr float kZNear = 0.01f;           // RenderParams, splat/render.hpp:13-19
constexpr float kCovReg = 0.3f;
constexpr double kSigmaCut = 3.0;
constexpr float kAlphaMax = 0.999f;
constexpr float kTransmitStop = 1e-4f;

// Projected record, one per Gaussian (indexed by source). 48 bytes.
struct __align__(16) SplatRec {
  float mean_x, mean_y, depth, alpha;  // mean2d, camera z, decoded opacity
  float a00, a01, a10, a11;            // cov_inv (row-major)
  int32_t x0, x1, y0, y1;              // inclusive pixel bbox; x0 > x1 => not listed
};

// Ampere-style asynchronous global -> shared copies (LDGSTS), used to prefetch the next splat
// batch of the rasteriser while the current one is processed.
__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ int4 f4_as_i4(float4 v) {
  return make_int4(__float_as_int(v.x), __float_as_int(v.y), __float_as_int(v.z), __float_as_int(v.w));
}
__device__ __forceinline__ float4 i4_as_f4(int4 v) {
  return make_float4(__int_as_float(v.x), __int_as_float(v.y), __int_as_float(v.z), __int_as_float(v.w));
}

// 2^x and 1/x on the SFU (approximate; used only where gradient accuracy suffices)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Loads the compiler may not sink below a later branch (volatile asm executes exactly where it
// is written): used to put all of a thread's loads in one memory round trip ahead of an early exit.
__device__ __forceinline__ float4 ld_early4(const void* p) {
  float4 v;
  asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_early(const float* p) {
  float v;
  asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace lm

#define LM_CUDA_CHECK(expr)                                                            \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      return ::lm::set_cuda_error(_e, #expr, __FILE__, __LINE__);                       \
    }                                                                                  \
  } while (0)
