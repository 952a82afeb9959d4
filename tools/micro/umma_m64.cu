// Probe: where does a cta_group::1 M=64 tcgen05.mma put its 64 x N result in TMEM? Computes
// C = A B^T with A (64 x K) = row index in column 0 (so C[r][n] = r * B[n][0]) and dumps all
// 128 lanes x N columns.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../../paper_2602_12314_b200/csrc/tc_common.cuh"

__global__ void probe(float* out, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  constexpr int M = 64;
  uint8_t* sa = smem;
  uint8_t* sb = smem + M * K * 2;
  const uint32_t a_sbo = 16u * K, a_lbo = 128u, b_sbo = 16u * K, b_lbo = 128u;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(sa + lm::tc::core_off(r, k, a_sbo, a_lbo)) = __float2bfloat16_rn(k == 0 ? (float)(r + 1) : 0.f);
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + lm::tc::core_off(r, k, b_sbo, b_lbo)) = __float2bfloat16_rn(k == 0 ? (float)(r % 8 + 1) * 1000.f : 0.f);
  }
  lm::tc::fence_async_smem();
  if (threadIdx.x == 0) { lm::tc::mbar_init(&bar, 1); lm::tc::fence_mbar_init(); }
  if (threadIdx.x < 32) lm::tc::tmem_alloc<256>(&taddr_s);
  lm::tc::tc_fence_before();
  __syncthreads();
  lm::tc::tc_fence_after();
  const uint32_t taddr = taddr_s;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  // zero TMEM first (tcgen05.st via a store of zeros through an MMA with zero A would be simpler;
  // instead read whatever is there before and after)
  if (threadIdx.x == 0) {
    const uint32_t idesc = lm::tc::make_idesc_bf16(M, N, 0, 0);
    for (int ks = 0; ks < K / 16; ++ks)
      lm::tc::mma_bf16(taddr, lm::tc::make_sdesc(lm::tc::smem_u32(sa) + ks * 2 * a_lbo, a_lbo, a_sbo),
                   lm::tc::make_sdesc(lm::tc::smem_u32(sb) + ks * 2 * b_lbo, b_lbo, b_sbo), idesc, ks > 0);
    lm::tc::mma_commit(&bar);
  }
  lm::tc::mbar_wait(&bar, 0);
  lm::tc::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    lm::tc::tmem_ld16(taddr + ((uint32_t)(32 * w) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) out[(size_t)(32 * w + lane) * N + c0 + i] = v[i];
  }
  lm::tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) lm::tc::tmem_free<256>(taddr);
}

int main() {
  const int N = 32, K = 16;
  float* d;
  cudaMalloc(&d, 128 * N * 4);
  cudaMemset(d, 0, 128 * N * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, (64 + N) * K * 2>>>(d, N, K);
  float h[128 * 32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int l = 0; l < 128; ++l) {
    printf("lane %3d:", l);
    for (int c = 0; c < 12; ++c) printf(" %7.0f", h[l * N + c]);
    printf("\n");
  }
}
