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

// Pass 1: per-block all-finite check (adam.hpp:65-68) over the active blocks only (kind >= 0),
// 16-byte loads over each block's 4-aligned interior.
__global__ void adam_check_kernel(const float* __restrict__ grad, Blocks B, int32_t* flags) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int bi = 0; bi < B.n; ++bi) {
    const AdamBlock blk = B.b[bi];
    if (blk.kind < 0 || blk.count <= 0) continue;
    const int64_t e0 = blk.offset, e1 = blk.offset + blk.count;
    const int64_t a0 = (e0 + 3) / 4 * 4, a1 = max(a0, e1 / 4 * 4);
    bool bad = false;
    for (int64_t q = a0 / 4 + tid; q < a1 / 4; q += nth) {
      const float4 v = reinterpret_cast<const float4*>(grad)[q];
      bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    }
    for (int64_t e = e0 + tid; e < min(a0, e1); e += nth) bad |= !isfinite(grad[e]);
    for (int64_t e = max(a1, e0) + tid; e < e1; e += nth) bad |= !isfinite(grad[e]);
    if (bad) flags[bi] = 1;
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
// Every CTA walks every block in turn (grid-stride inside each block), so each block is
// streamed by the whole GPU; rows / 4-aligned interiors use 16-byte vectors.
__device__ __forceinline__ void quat_row(float4& p, const float4& g, float4& mm, float4& vv, bool skip, float lr,
                                         float c1, float c2) {
  if (!skip) {
    adam_elem(p.x, g.x, mm.x, vv.x, lr, c1, c2);
    adam_elem(p.y, g.y, mm.y, vv.y, lr, c1, c2);
    adam_elem(p.z, g.z, mm.z, vv.z, lr, c1, c2);
    adam_elem(p.w, g.w, mm.w, vv.w, lr, c1, c2);
  }
  const float n = __fsqrt_rn(fa(fa(fa(fm(p.x, p.x), fm(p.y, p.y)), fm(p.z, p.z)), fm(p.w, p.w)));
  if (n > 1e-12f) {
    p = make_float4(fd(p.x, n), fd(p.y, n), fd(p.z, n), fd(p.w, n));
  } else {
    p = make_float4(1.f, 0.f, 0.f, 0.f);
  }
}

__global__ void __launch_bounds__(256, 5) adam_update_kernel(float* __restrict__ param, const float* __restrict__ grad,
                                                          float* __restrict__ m, float* __restrict__ v, Blocks B,
                                                          const int64_t* steps, const float* corr1,
                                                          const float* corr2, int32_t table_len, const int32_t* flags,
                                                          const double* overflow) {
  if (overflow && *overflow != 0.0) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int bi = 0; bi < B.n; ++bi) {
    const AdamBlock blk = B.b[bi];
    if (blk.kind < 0) continue;
    const bool skip = flags[bi] != 0;  // skipped block: parameters untouched (rotations still renormalised)
    if (skip && blk.kind != 1) continue;
    const int64_t t = steps[bi] + 1;
    const float c1 = t <= table_len ? corr1[t - 1] : 1.f;
    const float c2 = t <= table_len ? corr2[t - 1] : 1.f;
    const int64_t e0 = blk.offset, e1 = blk.offset + blk.count;
    if (blk.kind == 1) {
      const int64_t nq = blk.count / 4;
      if ((e0 & 3) == 0) {
        float4* p4 = reinterpret_cast<float4*>(param + e0);
        const float4* g4 = reinterpret_cast<const float4*>(grad + e0);
        float4* m4 = reinterpret_cast<float4*>(m + e0);
        float4* v4 = reinterpret_cast<float4*>(v + e0);
        for (int64_t i = tid; i < nq; i += nth) {
          float4 p = p4[i], mm = m4[i], vv = v4[i];
          quat_row(p, g4[i], mm, vv, skip, blk.lr, c1, c2);
          p4[i] = p;
          if (!skip) {
            m4[i] = mm;
            v4[i] = vv;
          }
        }
      } else {
        for (int64_t i = tid; i < nq; i += nth) {
          const int64_t e = e0 + 4 * i;
          float4 p = make_float4(param[e], param[e + 1], param[e + 2], param[e + 3]);
          float4 mm = make_float4(m[e], m[e + 1], m[e + 2], m[e + 3]);
          float4 vv = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
          const float4 g = make_float4(grad[e], grad[e + 1], grad[e + 2], grad[e + 3]);
          quat_row(p, g, mm, vv, skip, blk.lr, c1, c2);
          param[e] = p.x, param[e + 1] = p.y, param[e + 2] = p.z, param[e + 3] = p.w;
          if (!skip) {
            m[e] = mm.x, m[e + 1] = mm.y, m[e + 2] = mm.z, m[e + 3] = mm.w;
            v[e] = vv.x, v[e + 1] = vv.y, v[e + 2] = vv.z, v[e + 3] = vv.w;
          }
        }
      }
      continue;
    }
    // 16-byte vectors over the 4-aligned interior of the block, scalar head/tail
    const int64_t a0 = (e0 + 3) / 4 * 4, a1 = e1 / 4 * 4;
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
}

// Pass 3: counters (AdamState::step / skipped).
__global__ void adam_finish_kernel(Blocks B, int64_t* steps, int64_t* skipped, int32_t* flags, const double* overflow,
                                   int64_t* overflow_steps) {
  const int i = threadIdx.x;
  const bool ovf = overflow && *overflow != 0.0;
  if (i == 0 && ovf && overflow_steps) *overflow_steps += 1;  // sticky: read by latmap_session_overflow_steps
  if (i >= B.n) return;
  if (!ovf && B.b[i].kind >= 0) {
    if (flags[i])
      skipped[i] += 1;
    else
      steps[i] += 1;
  }
  flags[i] = 0;
}

}  // namespace

namespace {
// Sharded step: the per-block non-finite flags of this rank's gradient shard [begin, end), as
// doubles in the loss-partials tail (summed over ranks by the partials all-reduce).
__global__ void adam_check_range_kernel(const float* __restrict__ grad, Blocks B, int64_t begin, int64_t end,
                                        double* flags_out) {
  for (int64_t e = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < end; e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(grad[e])) {
      const int b = find_block(B, e);
      if (b >= 0) flags_out[b] = 1.0;
    }
}
__global__ void adam_flags_from_kernel(const double* ext, int32_t* flags, int n) {
  if (threadIdx.x < n) flags[threadIdx.x] = ext[threadIdx.x] != 0.0 ? 1 : 0;
}
}  // namespace

void adam_flat(cudaStream_t st, float* param, const float* grad, float* m, float* v, const AdamBlock* blocks,
               int nblocks, int64_t* steps, int64_t* skipped, const float* corr1, const float* corr2,
               int32_t table_len, int32_t* flags, const double* overflow, int64_t* overflow_steps, int64_t begin,
               int64_t end, const double* ext_flags) {
  Blocks B;
  B.n = nblocks;
  int64_t total = 0;
  for (int i = 0; i < nblocks; ++i) {
    B.b[i] = blocks[i];
    total = std::max(total, blocks[i].offset + blocks[i].count);
  }
  if (end < 0) end = total;
  // clip every block to [begin, end): counts may become 0, the block index (and with it the
  // step counter and skip flag of the reference's AdamState) is kept
  for (int i = 0; i < nblocks; ++i) {
    const int64_t b0 = std::max(B.b[i].offset, begin), b1 = std::min(B.b[i].offset + B.b[i].count, end);
    B.b[i].offset = b0;
    B.b[i].count = std::max<int64_t>(0, b1 - b0);
  }
  if (ext_flags) {
    adam_flags_from_kernel<<<1, 32, 0, st>>>(ext_flags, flags, nblocks);
  } else {
    adam_check_kernel<<<148 * 4, 256, 0, st>>>(grad, B, flags);
  }
  adam_update_kernel<<<148 * 5, 256, 0, st>>>(param, grad, m, v, B, steps, corr1, corr2, table_len, flags,
                                               overflow);
  adam_finish_kernel<<<1, 32, 0, st>>>(B, steps, skipped, flags, overflow, overflow_steps);
  count_launch(3);
}

void adam_check_range(cudaStream_t st, const float* grad, const AdamBlock* blocks, int nblocks, int64_t begin,
                      int64_t end, double* flags_out) {
  Blocks B;
  B.n = nblocks;
  for (int i = 0; i < nblocks; ++i) B.b[i] = blocks[i];
  if (end > begin) {
    adam_check_range_kernel<<<(unsigned)std::min<int64_t>((end - begin + 255) / 256, 148 * 4), 256, 0, st>>>(
        grad, B, begin, end, flags_out);
    count_launch();
  }
}

}  // namespace lm
