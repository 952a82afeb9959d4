// Microbenchmark: stream a buffer into shared memory with cp.async.bulk (1-D TMA) from one
// elected thread per CTA, ring of S stages of C bytes each, nothing else. Reports GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra.uni D;\nbra.uni W;\nD:\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}

// each CTA streams `per_cta` bytes starting at its slice; units of `unit` bytes, each unit issued as
// unit/chunk copies of `chunk` bytes; S stages
__global__ void stream_kernel(const uint8_t* src, size_t per_cta, int unit, int chunk, int S, int* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const int nu = (int)(per_cta / unit);
  auto load = [&](int i) {
    const int s = i % S;
    expect_tx(&bar[s], unit);
    for (int c = 0; c < unit; c += chunk) g2s(sm + (size_t)s * unit + c, base + (size_t)i * unit + c, chunk, &bar[s]);
  };
  for (int i = 0; i < S && i < nu; ++i) load(i);
  int acc = 0;
  for (int i = 0; i < nu; ++i) {
    const int s = i % S;
    wait(&bar[s], (i / S) & 1);
    acc += sm[(size_t)s * unit];
    if (i + S < nu) load(i + S);
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  const size_t total = (size_t)148 * 2 * 1024 * 1024;  // 296 MB (> L2)
  uint8_t* buf;
  int* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, total);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int unit, chunk, S; } cfgs[] = {{65536, 65536, 2}, {65536, 65536, 3}, {32768, 32768, 4}, {32768, 1024, 4},
                                               {16384, 16384, 8}, {8192, 8192, 16}, {32768, 4096, 4}, {65536, 8192, 3}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto c : cfgs) {
    const size_t per = total / 148;
    const size_t per_cta = per / c.unit * c.unit;
    const size_t smem = (size_t)c.unit * c.S;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      stream_kernel<<<148, 32, smem>>>(buf, per_cta, c.unit, c.chunk, c.S, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("unit %6d chunk %6d stages %2d: %.1f GB/s (%s)\n", c.unit, c.chunk, c.S, per_cta * 148 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
