// adam.cu — fused Adam over every learnable block (K10).
// Reference: adam_step (proj/include/latmap/obj/adam.hpp:61-79) called block by block from
// MapOptimizer::step_map / step_dict (proj/src/pipeline.cpp:75-95), with the whole-block
// non-finite skip, per-block step counters, double-precision bias corrections and the
// quaternion renormalisation after the rotation step. The update arithmetic follows the
// reference's float op order without FMA, so given identical gradients it is bit-exact.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace lm {

namespace {

constexpr int kMaxBlocks = 8;
struct Blocks {
  AdamBlock b[kMaxBlocks];
  int n;
};

__device__ __forceinline__ int find_block(const Blocks& B, int64_t e) {
  for (int i = 0; i < B.n; ++i)
    if (e >= B.b[i].offset && e < B.b[i].offset + B.b[i].count) return i;
  return -1;
}

// Pass 1: per-block all-finite check (adam.hpp:65-68), 16-byte loads.
__global__ void adam_check_kernel(const float* __restrict__ grad, Blocks B, int64_t total, int32_t* flags) {
  const int64_t n4 = total / 4;
  const float4* g4 = reinterpret_cast<const float4*>(grad);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = g4[q];
    if (!(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w))) {
      const float vv[4] = {v.x, v.y, v.z, v.w};
      for (int i = 0; i < 4; ++i)
        if (!isfinite(vv[i])) {
          const int b = find_block(B, 4 * q + i);
          if (b >= 0) flags[b] = 1;
        }
    }
  }
  for (int64_t e = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(grad[e])) {
      const int b = find_block(B, e);
      if (b >= 0) flags[b] = 1;
    }
}

__device__ __forceinline__ float adam_elem(float& p, float g, float& m, float& v, float lr, float c1, float c2) {
  const float b1 = 0.9f, b2 = 0.999f;
  m = fa(fm(b1, m), fm(fs(1.f, b1), g));
  v = fa(fm(b2, v), fm(fs(1.f, b2), fm(g, g)));
  const float upd = fd(fm(lr, fd(m, c1)), fa(__fsqrt_rn(fd(v, c2)), 1e-8f));
  p = fs(p, upd);
  return p;
}

// Pass 2: update (adam.hpp:69-78); quaternion blocks renormalise rows (pipeline.cpp:78-84).
__global__ void adam_update_kernel(float* __restrict__ param, const float* __restrict__ grad, float* __restrict__ m,
                                   float* __restrict__ v, Blocks B, const int64_t* steps, const float* corr1,
                                   const float* corr2, int32_t table_len, const int32_t* flags,
                                   const int64_t* overflow) {
  if (overflow && *overflow) return;
  const int bi = blockIdx.y;
  const AdamBlock blk = B.b[bi];
  if (blk.kind < 0) return;
  const bool skip = flags[bi] != 0;  // skipped block: parameters untouched (rotations still renormalised)
  if (skip && blk.kind != 1) return;
  const int64_t t = steps[bi] + 1;
  const float c1 = t <= table_len ? corr1[t - 1] : 1.f;
  const float c2 = t <= table_len ? corr2[t - 1] : 1.f;
  if (blk.kind == 1) {
    const int64_t nq = blk.count / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t e = blk.offset + 4 * i;
      float q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float p = param[e + c];
        if (!skip) {
          float mm = m[e + c], vv = v[e + c];
          adam_elem(p, grad[e + c], mm, vv, blk.lr, c1, c2);
          m[e + c] = mm;
          v[e + c] = vv;
        }
        q[c] = p;
      }
      const float n = __fsqrt_rn(fa(fa(fa(fm(q[0], q[0]), fm(q[1], q[1])), fm(q[2], q[2])), fm(q[3], q[3])));
      if (n > 1e-12f) {
#pragma unroll
        for (int c = 0; c < 4; ++c) param[e + c] = fd(q[c], n);
      } else {
        param[e] = 1.f;
        param[e + 1] = param[e + 2] = param[e + 3] = 0.f;
      }
    }
    return;
  }
  // 16-byte vectors over the 4-aligned interior of the block, scalar head/tail
  const int64_t e0 = blk.offset, e1 = blk.offset + blk.count;
  const int64_t a0 = (e0 + 3) / 4 * 4, a1 = e1 / 4 * 4;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  if (a0 < a1) {
    for (int64_t q = a0 / 4 + tid; q < a1 / 4; q += nth) {
      float4 p = reinterpret_cast<float4*>(param)[q];
      const float4 g = reinterpret_cast<const float4*>(grad)[q];
      float4 mm = reinterpret_cast<float4*>(m)[q];
      float4 vv = reinterpret_cast<float4*>(v)[q];
      adam_elem(p.x, g.x, mm.x, vv.x, blk.lr, c1, c2);
      adam_elem(p.y, g.y, mm.y, vv.y, blk.lr, c1, c2);
      adam_elem(p.z, g.z, mm.z, vv.z, blk.lr, c1, c2);
      adam_elem(p.w, g.w, mm.w, vv.w, blk.lr, c1, c2);
      reinterpret_cast<float4*>(param)[q] = p;
      reinterpret_cast<float4*>(m)[q] = mm;
      reinterpret_cast<float4*>(v)[q] = vv;
    }
  }
  auto scalar = [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo + tid; e < hi; e += nth) {
      float p = param[e], mm = m[e], vv = v[e];
      adam_elem(p, grad[e], mm, vv, blk.lr, c1, c2);
      param[e] = p;
      m[e] = mm;
      v[e] = vv;
    }
  };
  if (a0 < a1) {
    scalar(e0, a0);
    scalar(a1, e1);
  } else {
    scalar(e0, e1);
  }
}

// Pass 3: counters (AdamState::step / skipped).
__global__ void adam_finish_kernel(Blocks B, int64_t* steps, int64_t* skipped, int32_t* flags, const int64_t* overflow) {
  const int i = threadIdx.x;
  if (i >= B.n) return;
  if (!(overflow && *overflow) && B.b[i].kind >= 0) {
    if (flags[i])
      skipped[i] += 1;
    else
      steps[i] += 1;
  }
  flags[i] = 0;
}

}  // namespace

void adam_flat(cudaStream_t st, float* param, const float* grad, float* m, float* v, const AdamBlock* blocks,
               int nblocks, int64_t* steps, int64_t* skipped, const float* corr1, const float* corr2,
               int32_t table_len, int32_t* flags, const int64_t* overflow) {
  Blocks B;
  B.n = nblocks;
  int64_t total = 0;
  for (int i = 0; i < nblocks; ++i) {
    B.b[i] = blocks[i];
    total = std::max(total, blocks[i].offset + blocks[i].count);
  }
  adam_check_kernel<<<148 * 4, 256, 0, st>>>(grad, B, total, flags);
  adam_update_kernel<<<dim3(148 * 2, nblocks), 256, 0, st>>>(param, grad, m, v, B, steps, corr1, corr2, table_len,
                                                              flags, overflow);
  adam_finish_kernel<<<1, 32, 0, st>>>(B, steps, skipped, flags, overflow);
  count_launch(3);
}

}  // namespace lm
