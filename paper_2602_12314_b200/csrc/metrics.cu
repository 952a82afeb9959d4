// metrics.cu — evaluation on the GPU: gather_supervision's pixel-mode
// row compaction (proj/src/objective.cpp:16-35), metric_cos / metric_miou / metric_psnr
// (proj/src/metrics.cpp:8-89) and query_map's scores (proj/src/evaluate.cpp:74-88). evaluate_map
// (evaluate.cpp:10-72) composes them with render and reconstruct in the host API.
//
// Per-row quantities follow the oracle's float conventions op for op (sequential sums in ascending
// index, no FMA, exp correctly rounded), so per-row values, predictions and the mIoU counts are
// bit-exact; the double means over rows / pixels are summed in a fixed two-level order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/latmap_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace lm {

namespace {

constexpr int kBlk = 256;

__device__ __forceinline__ float dot_seq(const float* a, const float* b, int d) {
  float s = 0.f;
  for (int i = 0; i < d; ++i) s = __fadd_rn(s, __fmul_rn(a[i], b[i]));
  return s;
}

__device__ void block_sum_d(double v, double* out_block) {
  __shared__ double s[kBlk / 32];
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kBlk / 32; ++w) t += s[w];
    *out_block = t;
  }
}

// metric_cos rows: 1 - dot / (max(|r|, 1e-8) max(|t|, 1e-8)), norms / dot in float (metrics.cpp:14-22)
__global__ void __launch_bounds__(kBlk) cos_rows_kernel(const float* __restrict__ rec, const float* __restrict__ tgt,
                                                        int64_t n, int d, double* __restrict__ part, int32_t* flagged) {
  const int64_t r = blockIdx.x * (int64_t)kBlk + threadIdx.x;
  double v = 0.0;
  if (r < n) {
    const float* x = rec + r * d;
    const float* y = tgt + r * d;
    double nu = (double)__fsqrt_rn(dot_seq(x, x, d));
    double nv = (double)__fsqrt_rn(dot_seq(y, y, d));
    if (nu < 1e-8 || nv < 1e-8) atomicOr(flagged, 1);
    nu = nu > 1e-8 ? nu : 1e-8;
    nv = nv > 1e-8 ? nv : 1e-8;
    v = 1.0 - (double)dot_seq(x, y, d) / (nu * nv);
  }
  block_sum_d(v, part + blockIdx.x);
}

// metric_miou rows: softmax over prototype scores, first maximum (metrics.cpp:37-56). The class
// scores are recomputed in each of the three passes (max, sum, argmax) instead of being stored:
// identical operations give identical values, and any number of classes fits.
__global__ void __launch_bounds__(kBlk) miou_rows_kernel(const float* __restrict__ emb, const int32_t* __restrict__ labels,
                                                         int64_t n, int d, const float* __restrict__ protos, int c,
                                                         unsigned long long* inter, unsigned long long* uni,
                                                         int32_t* bad) {
  const int64_t i = blockIdx.x * (int64_t)kBlk + threadIdx.x;
  if (i >= n) return;
  const int32_t gt = labels[i];
  if (gt < 0) return;
  if (gt >= c) {
    atomicOr(bad, 1);
    return;
  }
  const float* e = emb + i * d;
  float m = 0.f;
  for (int k = 0; k < c; ++k) {
    const float v = dot_seq(protos + (int64_t)k * d, e, d);
    if (k == 0 || v > m) m = v;
  }
  float s = 0.f;
  for (int k = 0; k < c; ++k) s = __fadd_rn(s, exp_exact(__fsub_rn(dot_seq(protos + (int64_t)k * d, e, d), m)));
  int pred = 0;
  float best = 0.f;
  for (int k = 0; k < c; ++k) {
    const float p = __fdiv_rn(exp_exact(__fsub_rn(dot_seq(protos + (int64_t)k * d, e, d), m)), s);
    if (k == 0 || p > best) best = p, pred = k;
  }
  if (pred == gt) {
    atomicAdd(inter + gt, 1ull);
    atomicAdd(uni + gt, 1ull);
  } else {
    atomicAdd(uni + gt, 1ull);
    atomicAdd(uni + pred, 1ull);
  }
}

__global__ void __launch_bounds__(kBlk) sqerr_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                                                     double* __restrict__ part) {
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kBlk + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlk) {
    const double dd = (double)a[i] - (double)b[i];
    v += dd * dd;
  }
  block_sum_d(v, part + blockIdx.x);
}

// query_map scores (evaluate.cpp:80-86)
__global__ void query_scores_kernel(const float* __restrict__ rec, int64_t n, int d, const float* __restrict__ emb,
                                    float* __restrict__ scores) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float qn = __fsqrt_rn(dot_seq(emb, emb, d));
  qn = qn > 1e-8f ? qn : 1e-8f;
  const float* x = rec + i * d;
  float rn = __fsqrt_rn(dot_seq(x, x, d));
  rn = rn > 1e-8f ? rn : 1e-8f;
  scores[i] = __fdiv_rn(dot_seq(x, emb, d), __fmul_rn(rn, qn));
}

// gather_supervision, pixel mode: rows of supervised pixels (assignment >= 0) in ascending pixel
// order. Pass 1 counts per block, a one-block scan makes the offsets, pass 2 emits query rows,
// target rows (optionally normalised as evaluate_map does, evaluate.cpp:38-42) and pixel ids.
__global__ void __launch_bounds__(kBlk) sup_count_kernel(const int32_t* __restrict__ asg, int64_t npx,
                                                         int32_t* __restrict__ cnt) {
  const int64_t p = blockIdx.x * (int64_t)kBlk + threadIdx.x;
  const int pred = p < npx && asg[p] >= 0;
  const int c = __syncthreads_count(pred);
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

__global__ void __launch_bounds__(1024) sup_scan_kernel(int32_t* cnt, int64_t nb, int64_t* total) {
  __shared__ int64_t s_run;
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int v = i < nb ? cnt[i] : 0;
    // inclusive scan of the chunk (Hillis-Steele over shared memory)
    __shared__ int64_t s[1024];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int64_t t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nb) cnt[i] = (int32_t)(s_run + s[threadIdx.x] - v);  // exclusive
    __syncthreads();
    if (threadIdx.x == 1023) s_run += s[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s_run;
}

__global__ void __launch_bounds__(kBlk) sup_emit_kernel(const int32_t* __restrict__ asg, int64_t npx,
                                                        const int32_t* __restrict__ off, const float* __restrict__ query,
                                                        int ds, const float* __restrict__ feats, int df, int normalize,
                                                        float* __restrict__ q_out, float* __restrict__ t_out,
                                                        int64_t* __restrict__ pix) {
  __shared__ int32_t s_w[kBlk / 32];
  const int64_t p = blockIdx.x * (int64_t)kBlk + threadIdx.x;
  const int32_t a = p < npx ? asg[p] : -1;
  const bool take = a >= 0;
  const unsigned ball = __ballot_sync(0xffffffffu, take);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_w[warp] = __popc(ball);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += s_w[w];
  if (!take) return;
  const int64_t r = off[blockIdx.x] + before + __popc(ball & ((1u << lane) - 1u));
  for (int c = 0; c < ds; ++c) q_out[r * ds + c] = query[p * ds + c];
  const float* f = feats + (int64_t)a * df;
  float inv = 1.f;
  if (normalize) {
    const float nrm = __fsqrt_rn(dot_seq(f, f, df));
    if (nrm > 1e-12f) inv = nrm;
  }
  for (int c = 0; c < df; ++c) t_out[r * df + c] = normalize ? (inv != 1.f ? __fdiv_rn(f[c], inv) : f[c]) : f[c];
  pix[r] = p;
}

double sum_parts(cudaStream_t st, const double* d_part, int64_t nb) {
  std::vector<double> h((size_t)nb);
  cudaMemcpyAsync(h.data(), d_part, sizeof(double) * nb, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}

}  // namespace

cudaError_t metric_cos_dev(cudaStream_t st, const float* rec, const float* tgt, int64_t n, int d, double* out,
                           int32_t* flagged) {
  *out = 0.0;
  if (flagged) *flagged = 0;
  if (n == 0) return cudaSuccess;
  const int64_t nb = (n + kBlk - 1) / kBlk;
  double* part = nullptr;
  int32_t* fl = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * nb, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&fl, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(fl, 0, sizeof(int32_t), st);
  cos_rows_kernel<<<(unsigned)nb, kBlk, 0, st>>>(rec, tgt, n, d, part, fl);
  count_launch();
  int32_t hf = 0;
  cudaMemcpyAsync(&hf, fl, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  *out = sum_parts(st, part, nb) / (double)n;
  if (flagged) *flagged = hf;
  cudaFreeAsync(part, st);
  cudaFreeAsync(fl, st);
  return cudaStreamSynchronize(st);
}

cudaError_t metric_miou_dev(cudaStream_t st, const float* emb, const int32_t* labels, int64_t n, int d,
                            const float* protos, int c, int64_t* inter, int64_t* uni, double* miou, bool* bad_label) {
  *miou = 0.0;
  *bad_label = false;
  for (int k = 0; k < c; ++k) inter[k] = uni[k] = 0;
  if (n == 0 || c == 0) return cudaSuccess;
  unsigned long long* d_cnt = nullptr;
  int32_t* d_bad = nullptr;
  cudaError_t e = cudaMallocAsync(&d_cnt, sizeof(unsigned long long) * 2 * c, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_bad, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 2 * c, st);
  cudaMemsetAsync(d_bad, 0, sizeof(int32_t), st);
  miou_rows_kernel<<<(unsigned)((n + kBlk - 1) / kBlk), kBlk, 0, st>>>(emb, labels, n, d, protos, c, d_cnt, d_cnt + c,
                                                                        d_bad);
  count_launch();
  std::vector<unsigned long long> h((size_t)2 * c);
  int32_t hb = 0;
  cudaMemcpyAsync(h.data(), d_cnt, sizeof(unsigned long long) * 2 * c, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hb, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  cudaFreeAsync(d_cnt, st);
  cudaFreeAsync(d_bad, st);
  if (e != cudaSuccess) return e;
  *bad_label = hb != 0;
  double sum = 0.0;
  int64_t inc = 0;
  for (int k = 0; k < c; ++k) {
    inter[k] = (int64_t)h[(size_t)k];
    uni[k] = (int64_t)h[(size_t)(c + k)];
    if (uni[k] == 0) continue;
    sum += (double)inter[k] / (double)uni[k];
    ++inc;
  }
  *miou = inc > 0 ? sum / (double)inc : 0.0;
  return cudaSuccess;
}

cudaError_t metric_psnr_dev(cudaStream_t st, const float* a, const float* b, int64_t n, double* db, int32_t* exact) {
  const int64_t nb = std::min<int64_t>((n + kBlk - 1) / kBlk, 148 * 8);
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * std::max<int64_t>(nb, 1), st);
  if (e != cudaSuccess) return e;
  double mse = 0.0;
  if (n > 0) {
    sqerr_kernel<<<(unsigned)nb, kBlk, 0, st>>>(a, b, n, part);
    count_launch();
    mse = sum_parts(st, part, nb) / (double)n;
  }
  cudaFreeAsync(part, st);
  if (mse == 0.0) {
    *db = 100.0;
    *exact = 1;
  } else {
    *db = 10.0 * std::log10(1.0 / mse);
    *exact = 0;
  }
  return cudaStreamSynchronize(st);
}

cudaError_t query_scores_dev(cudaStream_t st, const float* rec, int64_t n, int d, const float* emb, float* scores) {
  if (n == 0) return cudaSuccess;
  query_scores_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rec, n, d, emb, scores);
  count_launch();
  return cudaGetLastError();
}

cudaError_t gather_supervision_dev(cudaStream_t st, const float* query, int ds, const int32_t* asg, int64_t npx,
                                   const float* feats, int df, bool normalize, float* q_out, float* t_out,
                                   int64_t* pix, int64_t cap, int64_t* n_rows) {
  const int64_t nb = std::max<int64_t>(1, (npx + kBlk - 1) / kBlk);
  int32_t* cnt = nullptr;
  int64_t* tot = nullptr;
  cudaError_t e = cudaMallocAsync(&cnt, sizeof(int32_t) * nb, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&tot, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  sup_count_kernel<<<(unsigned)nb, kBlk, 0, st>>>(asg, npx, cnt);
  sup_scan_kernel<<<1, 1024, 0, st>>>(cnt, nb, tot);
  count_launch(2);
  int64_t n = 0;
  cudaMemcpyAsync(&n, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && n <= cap && q_out) {
    sup_emit_kernel<<<(unsigned)nb, kBlk, 0, st>>>(asg, npx, cnt, query, ds, feats, df, normalize ? 1 : 0, q_out, t_out,
                                                   pix);
    count_launch();
  }
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(tot, st);
  *n_rows = n;
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace lm
