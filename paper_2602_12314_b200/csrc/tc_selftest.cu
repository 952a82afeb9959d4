// tc_selftest.cu — single-tile tcgen05 GEMM used to pin the UMMA descriptor / TMEM
// conventions of tc_common.cuh against torch on the GPU (tests/test_gpu_tcgen05.py):
// C[128 x N] = A[128 x K] * B[N x K]^T with either operand staged K-major or MN-major.
#include <cuda_runtime.h>

#include "expf_ref.h"
#include "kernels.h"
#include "tc_common.cuh"

namespace lm {

namespace {

__global__ void __launch_bounds__(128) umma_probe_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                         float* __restrict__ C, int N, int K, int a_mn, int b_mn) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  constexpr int M = 128;
  uint8_t* sa = smem;
  uint8_t* sb = smem + M * K * 2;
  // staging strides (bytes): K-major -> SBO = 16*K (row groups), LBO = 128 (k groups);
  // MN-major -> SBO = 128 (mn groups), LBO = 16*rows (k groups).
  const uint32_t a_sbo = a_mn ? 128u : 16u * K, a_lbo = a_mn ? 16u * M : 128u;
  const uint32_t b_sbo = b_mn ? 128u : 16u * K, b_lbo = b_mn ? 16u * N : 128u;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const uint32_t off = a_mn ? tc::core_off(k, r, a_lbo, a_sbo) : tc::core_off(r, k, a_sbo, a_lbo);
    *reinterpret_cast<__nv_bfloat16*>(sa + off) = __float2bfloat16_rn(A[e]);
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const uint32_t off = b_mn ? tc::core_off(k, r, b_lbo, b_sbo) : tc::core_off(r, k, b_sbo, b_lbo);
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = __float2bfloat16_rn(B[e]);
  }
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&taddr_s);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t taddr = taddr_s;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc_bf16(M, N, a_mn, b_mn);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t ad = tc::make_sdesc(tc::smem_u32(sa) + ks * 2 * a_lbo, a_lbo, a_sbo);
      const uint64_t bd = tc::make_sdesc(tc::smem_u32(sb) + ks * 2 * b_lbo, b_lbo, b_sbo);
      tc::mma_bf16(taddr, ad, bd, idesc, ks > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(taddr + ((uint32_t)(32 * w) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) C[(size_t)(32 * w + lane) * N + c0 + i] = v[i];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free<256>(taddr);
}

}  // namespace

int umma_selftest(cudaStream_t st, const float* A, const float* B, float* C, int N, int K, int a_mn, int b_mn) {
  if (N % 16 || N < 16 || N > 256 || K % 16 || K < 16 || K > 256) return 1;
  const size_t smem = (size_t)(128 + N) * K * 2;
  cudaFuncSetAttribute(umma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma_probe_kernel<<<1, 128, smem, st>>>(A, B, C, N, K, a_mn, b_mn);
  count_launch();
  return 0;
}

// exp_exact (expf_ref.h) on the float with bit pattern first + i, i < n
__global__ void expf_probe_kernel(uint64_t first, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = expf_ref(__uint_as_float((uint32_t)(first + (uint64_t)i)));
}
void expf_selftest(cudaStream_t st, uint64_t first, int64_t n, float* out) {
  expf_probe_kernel<<<148 * 16, 256, 0, st>>>(first, n, out);
  count_launch();
}

}  // namespace lm
