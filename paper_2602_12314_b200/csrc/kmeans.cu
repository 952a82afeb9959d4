// kmeans.cu — streaming k-means dictionary maintenance on the GPU:
// weighted_kmeans and stream_kmeans_update (proj/src/stream_kmeans.cpp:94-196), called by
// process_keyframe_inner for dict_init = "kmeans" (proj/src/pipeline.cpp:201-205).
//
// The dense work runs on the device: the nearest-centre scores P C^T (a SIMT tile GEMM, the
// score matrix of the reference's assign_nearest), the per-row argmin with ties to the lower
// index, the k-means++ minimum squared distances, and the weighted centre sums of each Lloyd
// step. The steps that consume the caller's generator or define an order stay on the host, as
// in the reference: the k-means++ draw and prefix walk (uniform draws from the pipeline's
// std::mt19937_64 via a callback), empty-cluster re-seeding, the stable grouping of points by
// centre and the convergence test.
//
// Bit-exactness with the oracle's float conventions (oracle/latmap_oracle.h): no FMA (explicit
// __fmul_rn / __fadd_rn), every dot product / squared norm summed in ascending inner index,
// centre sums accumulated in ascending point order (points grouped by a stable sort), masses
// and cluster weights summed on the host in point order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace lm {

namespace {

// c2[j] = |C[j]|^2, ascending inner index.
__global__ void km_rownorm_kernel(const float* __restrict__ C, int64_t k, int dim, float* __restrict__ c2) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= k) return;
  const float* c = C + j * dim;
  float s = 0.f;
  for (int d = 0; d < dim; ++d) s = __fadd_rn(s, __fmul_rn(c[d], c[d]));
  c2[j] = s;
}

// S = P C^T (n x k), each entry accumulated without FMA in ascending inner index (64 x 64 tiles).
constexpr int kBM = 64, kBN = 64, kBK = 16;
__global__ void __launch_bounds__(256) km_score_kernel(const float* __restrict__ P, int64_t n,
                                                       const float* __restrict__ C, int64_t k, int dim,
                                                       float* __restrict__ S) {
  __shared__ float As[kBK][kBM + 4];
  __shared__ float Bs[kBK][kBN + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t i0 = (int64_t)blockIdx.y * kBM, j0 = (int64_t)blockIdx.x * kBN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < dim; k0 += kBK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int e = tid + l * 256, r = e / kBK, kk = e % kBK;
      const int64_t gi = i0 + r, gj = j0 + r;
      As[kk][r] = (gi < n && k0 + kk < dim) ? P[gi * dim + k0 + kk] : 0.f;
      Bs[kk][r] = (gj < k && k0 + kk < dim) ? C[gj * dim + k0 + kk] : 0.f;
    }
    __syncthreads();
    const int kend = min(kBK, dim - k0);
    for (int kk = 0; kk < kend; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) av[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = __fadd_rn(acc[r][c], __fmul_rn(av[r], bv[c]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t gi = i0 + ty * 4 + r;
    if (gi >= n) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t gj = j0 + tx * 4 + c;
      if (gj < k) S[gi * k + gj] = acc[r][c];
    }
  }
}

// assignment[r] = argmin_j (c2[j] - 2 S[r][j]), ties to the lower index (assign_nearest,
// stream_kmeans.cpp:24-33). One warp per row: each lane scans j = lane, lane + 32, ... in
// ascending order with a strict <, then the lanes' minima meet (value, then index).
__global__ void km_argmin_kernel(const float* __restrict__ S, const float* __restrict__ c2, int64_t n, int64_t k,
                                 int32_t* __restrict__ asg) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (r >= n) return;
  const int lane = threadIdx.x & 31;
  float best = FLT_MAX;
  int64_t bj = -1;
  for (int64_t j = lane; j < k; j += 32) {
    const float d = __fsub_rn(c2[j], __fmul_rn(2.f, S[r * k + j]));
    if (bj < 0 || d < best) best = d, bj = j;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (oj >= 0 && (bj < 0 || ob < best || (ob == best && oj < bj))) best = ob, bj = oj;
  }
  if (lane == 0) asg[r] = (int32_t)bj;
}

__global__ void km_fill_kernel(float* __restrict__ x, int64_t n, float v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// min_d2[i] = min(min_d2[i], min over j in [j0, j1) of |P[i] - C[j]|^2) (update_min_dist,
// stream_kmeans.cpp:38-45, applied for each centre row; the min is order-free). One thread per
// (point, centre) pair, squared norm in ascending inner index; distances are >= 0, so the
// float minimum is an integer minimum of the bit patterns.
__global__ void km_mind2_kernel(const float* __restrict__ P, int64_t n, const float* __restrict__ C, int64_t j0,
                                int64_t j1, int dim, float* __restrict__ min_d2) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = j1 - j0;
  if (q >= n * m) return;
  const int64_t i = q % n, j = j0 + q / n;
  const float* p = P + i * dim;
  const float* c = C + j * dim;
  float d = 0.f;
  for (int e = 0; e < dim; ++e) {
    const float t = __fsub_rn(p[e], c[e]);
    d = __fadd_rn(d, __fmul_rn(t, t));
  }
  atomicMin(reinterpret_cast<int*>(min_d2) + i, __float_as_int(d));
}

// C[j][e] = (sum over the points of cluster j in ascending order of w_i P[i][e]) / mass[j] for
// mass[j] > 0 (weighted_kmeans, stream_kmeans.cpp:120-131). One thread per (centre, column).
__global__ void km_center_kernel(const float* __restrict__ P, const float* __restrict__ W,
                                 const int32_t* __restrict__ order, const int32_t* __restrict__ seg,
                                 const float* __restrict__ mass, int64_t k, int dim, float* __restrict__ C) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= k * dim) return;
  const int64_t j = q / dim;
  const int e = (int)(q % dim);
  const float mj = mass[j];
  if (!(mj > 0.f)) return;
  float s = 0.f;
  for (int32_t t = seg[j]; t < seg[j + 1]; ++t) {
    const int32_t i = order[t];
    s = __fadd_rn(s, __fmul_rn(W[i], P[(int64_t)i * dim + e]));
  }
  C[q] = __fdiv_rn(s, mj);
}

// dst[r] = src[rows[r]] for r < nr (row gather, dim floats per row).
__global__ void km_gather_kernel(const float* __restrict__ src, const int32_t* __restrict__ rows, int64_t nr, int dim,
                                 float* __restrict__ dst) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nr * dim) return;
  const int64_t r = q / dim;
  dst[q] = src[(int64_t)rows[r] * dim + q % dim];
}

unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Per-thread pinned host buffer (grown on demand) for the k-means++ distance read-back.
float* pinned_floats(int64_t n) {
  static thread_local float* buf = nullptr;
  static thread_local int64_t cap = 0;
  if (n > cap) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    if (cudaMallocHost(&buf, sizeof(float) * std::max<int64_t>(n, 4096)) != cudaSuccess) return nullptr;
    cap = std::max<int64_t>(n, 4096);
  }
  return buf;
}

struct KmBufs {
  float *w = nullptr, *c2 = nullptr, *S = nullptr, *mind2 = nullptr, *mass = nullptr;
  int32_t *asg = nullptr, *order = nullptr, *seg = nullptr;
  cudaStream_t st;
  explicit KmBufs(cudaStream_t s) : st(s) {}
  ~KmBufs() {
    for (void* p : {(void*)w, (void*)c2, (void*)S, (void*)mind2, (void*)mass, (void*)asg, (void*)order, (void*)seg})
      if (p) cudaFreeAsync(p, st);
  }
};

// assign_nearest on the device; the assignment lands in `h_asg`.
cudaError_t km_assign(cudaStream_t st, KmBufs& b, const float* P, int64_t n, int dim, const float* C, int64_t k,
                      std::vector<int32_t>& h_asg) {
  km_rownorm_kernel<<<blocks_for(k, 128), 128, 0, st>>>(C, k, dim, b.c2);
  dim3 g((unsigned)((k + kBN - 1) / kBN), (unsigned)((n + kBM - 1) / kBM));
  km_score_kernel<<<g, 256, 0, st>>>(P, n, C, k, dim, b.S);
  km_argmin_kernel<<<blocks_for(n * 32, 256), 256, 0, st>>>(b.S, b.c2, n, k, b.asg);
  count_launch(3);
  h_asg.resize((size_t)n);
  cudaMemcpyAsync(h_asg.data(), b.asg, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st);
  return cudaStreamSynchronize(st);
}

}  // namespace

static double km_now() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static bool km_trace() {
  static int t = -1;
  if (t < 0) t = std::getenv("LATMAP_KM_TRACE") ? 1 : 0;
  return t == 1;
}

cudaError_t kmeans_weighted(cudaStream_t st, const float* P, const float* W, int64_t n, int dim, int64_t k,
                            double (*uni)(void*), void* user, const float* warm, int64_t n_warm, int max_iters,
                            float* C, float* cw, int* iterations) {
  const double t_start = km_now();
  double t_pp = 0;
  cudaMemsetAsync(C, 0, sizeof(float) * k * dim, st);
  for (int64_t j = 0; j < k; ++j) cw[j] = 0.f;
  *iterations = 0;
  if (n == 0) return cudaStreamSynchronize(st);
  KmBufs b(st);
  for (cudaError_t e : {cudaMallocAsync(&b.w, sizeof(float) * n, st), cudaMallocAsync(&b.c2, sizeof(float) * k, st),
                        cudaMallocAsync(&b.S, sizeof(float) * n * k, st),
                        cudaMallocAsync(&b.mind2, sizeof(float) * n, st),
                        cudaMallocAsync(&b.mass, sizeof(float) * k, st),
                        cudaMallocAsync(&b.asg, sizeof(int32_t) * n, st),
                        cudaMallocAsync(&b.order, sizeof(int32_t) * n, st),
                        cudaMallocAsync(&b.seg, sizeof(int32_t) * (k + 1), st)})
    if (e != cudaSuccess) return e;
  cudaMemcpyAsync(b.w, W, sizeof(float) * n, cudaMemcpyHostToDevice, st);
  // warm start fills the first rows (stream_kmeans.cpp:107-111)
  int64_t filled = 0;
  if (warm) {
    filled = std::min(k, n_warm);
    cudaMemcpyAsync(C, warm, sizeof(float) * filled * dim, cudaMemcpyDeviceToDevice, st);
  }
  // weighted k-means++ continuation (kmeanspp_fill, stream_kmeans.cpp:48-90); the minimum
  // distances to the warm rows are only needed when rows remain to be drawn
  if (filled < k) {
    km_fill_kernel<<<blocks_for(n, 256), 256, 0, st>>>(b.mind2, n, FLT_MAX);
    count_launch();
    if (filled > 0) {
      km_mind2_kernel<<<blocks_for(n * filled, 256), 256, 0, st>>>(P, n, C, 0, filled, dim, b.mind2);
      count_launch();
    }
    std::vector<uint8_t> used((size_t)n, 0);
    float* md = pinned_floats(n);  // min_d2 read back per draw (pinned: a short round trip)
    if (!md) return cudaErrorMemoryAllocation;
    int64_t j = filled;
    for (; j < k; ++j) {
      const bool use_d = j > 0 || filled > 0;
      if (use_d) {
        cudaMemcpyAsync(md, b.mind2, sizeof(float) * n, cudaMemcpyDeviceToHost, st);
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
      }
      double total = 0;
      for (int64_t i = 0; i < n; ++i) {
        double p = (double)W[i];
        if (use_d) p *= (double)md[i];
        total += p;
      }
      if (!(total > 0)) break;  // mass exhausted: it stays so (min_d2 only shrinks), no more draws
      int64_t pick = -1;
      const double target = uni(user) * total;
      double run = 0;
      for (int64_t i = 0; i < n; ++i) {
        double p = (double)W[i];
        if (use_d) p *= (double)md[i];
        run += p;
        if (run >= target) {
          pick = i;
          break;
        }
      }
      if (pick < 0) pick = n - 1;
      used[(size_t)pick] = 1;
      cudaMemcpyAsync(C + j * dim, P + pick * dim, sizeof(float) * dim, cudaMemcpyDeviceToDevice, st);
      km_mind2_kernel<<<blocks_for(n, 256), 256, 0, st>>>(P, n, C, j, j + 1, dim, b.mind2);
      count_launch();
    }
    if (j < k) {
      // the remaining rows take the first unused points, then wrap around (stream_kmeans.cpp:72-78);
      // no draw and no distance is consumed any more, so they are gathered in one launch
      std::vector<int32_t> rows;
      for (; j < k; ++j) {
        int64_t pick = -1;
        for (int64_t i = 0; i < n; ++i)
          if (!used[(size_t)i]) {
            pick = i;
            break;
          }
        if (pick < 0) pick = (j - filled) % n;
        used[(size_t)pick] = 1;
        rows.push_back((int32_t)pick);
      }
      const int64_t nr = (int64_t)rows.size();
      int32_t* d_rows = nullptr;
      if (cudaError_t e = cudaMallocAsync(&d_rows, sizeof(int32_t) * nr, st)) return e;
      cudaMemcpyAsync(d_rows, rows.data(), sizeof(int32_t) * nr, cudaMemcpyHostToDevice, st);
      km_gather_kernel<<<blocks_for(nr * dim, 256), 256, 0, st>>>(P, d_rows, nr, dim, C + (k - nr) * dim);
      count_launch();
      cudaFreeAsync(d_rows, st);
    }
  }
  if (km_trace()) {
    cudaStreamSynchronize(st);
    t_pp = km_now();
  }
  // Lloyd iterations (stream_kmeans.cpp:113-152)
  std::vector<int32_t> asg, prev;
  std::vector<uint8_t> claimed((size_t)n, 0);
  std::vector<float> mass((size_t)k);
  std::vector<int32_t> order((size_t)n), seg((size_t)k + 1);
  for (int it = 0; it < max_iters; ++it) {
    cudaError_t e = km_assign(st, b, P, n, dim, C, k, asg);
    if (e != cudaSuccess) return e;
    std::fill(mass.begin(), mass.end(), 0.f);
    std::fill(seg.begin(), seg.end(), 0);
    for (int64_t i = 0; i < n; ++i) {
      mass[(size_t)asg[(size_t)i]] += W[i];
      ++seg[(size_t)asg[(size_t)i] + 1];
    }
    for (int64_t j = 0; j < k; ++j) seg[(size_t)j + 1] += seg[(size_t)j];
    {
      std::vector<int32_t> cur(seg.begin(), seg.end() - 1);  // stable grouping by centre
      for (int64_t i = 0; i < n; ++i) order[(size_t)cur[(size_t)asg[(size_t)i]]++] = (int32_t)i;
    }
    cudaMemcpyAsync(b.order, order.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b.seg, seg.data(), sizeof(int32_t) * (k + 1), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b.mass, mass.data(), sizeof(float) * k, cudaMemcpyHostToDevice, st);
    km_center_kernel<<<blocks_for(k * dim, 256), 256, 0, st>>>(P, b.w, b.order, b.seg, b.mass, k, dim, C);
    count_launch();
    bool reseeded = false;
    for (int64_t j = 0; j < k; ++j) {
      if (mass[(size_t)j] > 0.f) continue;
      // re-seed at the heaviest still-unclaimed point (stream_kmeans.cpp:132-146)
      int64_t pick = -1;
      float best = -1.f;
      for (int64_t i = 0; i < n; ++i)
        if (!claimed[(size_t)i] && W[i] > best) best = W[i], pick = i;
      if (pick >= 0) {
        claimed[(size_t)pick] = 1;
        cudaMemcpyAsync(C + j * dim, P + pick * dim, sizeof(float) * dim, cudaMemcpyDeviceToDevice, st);
        reseeded = true;
      }
    }
    *iterations = it + 1;
    if (!reseeded && it > 0 && asg == prev) break;
    prev = asg;
  }
  cudaError_t e = km_assign(st, b, P, n, dim, C, k, asg);
  if (e != cudaSuccess) return e;
  for (int64_t j = 0; j < k; ++j) cw[j] = 0.f;
  for (int64_t i = 0; i < n; ++i) cw[(size_t)asg[(size_t)i]] += W[i];
  if (km_trace())
    std::fprintf(stderr, "[kmeans] n=%lld dim=%d k=%lld warm=%lld: k-means++ %.3f ms, %d Lloyd + final assign %.3f ms\n",
                 (long long)n, dim, (long long)k, (long long)n_warm, t_pp - t_start, *iterations, km_now() - t_pp);
  return cudaSuccess;
}

cudaError_t kmeans_stream_update(cudaStream_t st, const float* batch, int64_t n, int dim, float* atoms, float* anchor,
                                 float* weights, int64_t K, double (*uni)(void*), void* user, float decay) {
  if (n == 0) return cudaSuccess;
  // stage 1: compress the batch into min(n, K) weighted micro-centres (stream_kmeans.cpp:168-171)
  const int64_t m = std::min(n, K);
  std::vector<float> unit((size_t)n, 1.f), lw((size_t)m);
  float *lc = nullptr, *pooled = nullptr, *warm = nullptr;
  if (cudaError_t e0 = cudaMallocAsync(&lc, sizeof(float) * m * dim, st)) return e0;
  int iters = 0;
  cudaError_t e = kmeans_weighted(st, batch, unit.data(), n, dim, m, uni, user, nullptr, 0, 10, lc, lw.data(), &iters);
  if (e != cudaSuccess) return e;
  // stage 2: pool with the surviving atoms (old mass x decay), re-cluster to K warm-started
  int64_t old_count = 0;
  for (int64_t j = 0; j < K; ++j)
    if (weights[j] > 0.f) ++old_count;
  if (cudaError_t e1 = cudaMallocAsync(&pooled, sizeof(float) * (m + old_count) * dim, st)) return e1;
  if (cudaError_t e2 = cudaMallocAsync(&warm, sizeof(float) * std::max<int64_t>(old_count, 1) * dim, st)) return e2;
  std::vector<float> pw((size_t)(m + old_count));
  cudaMemcpyAsync(pooled, lc, sizeof(float) * m * dim, cudaMemcpyDeviceToDevice, st);
  for (int64_t j = 0; j < m; ++j) pw[(size_t)j] = lw[(size_t)j];
  std::vector<int32_t> live;
  for (int64_t j = 0; j < K; ++j) {
    if (!(weights[j] > 0.f)) continue;
    pw[(size_t)(m + (int64_t)live.size())] = weights[j] * decay;
    live.push_back((int32_t)j);
  }
  if (old_count > 0) {
    int32_t* d_live = nullptr;
    if (cudaError_t e3 = cudaMallocAsync(&d_live, sizeof(int32_t) * old_count, st)) return e3;
    cudaMemcpyAsync(d_live, live.data(), sizeof(int32_t) * old_count, cudaMemcpyHostToDevice, st);
    km_gather_kernel<<<blocks_for(old_count * dim, 256), 256, 0, st>>>(atoms, d_live, old_count, dim, warm);
    cudaMemcpyAsync(pooled + m * dim, warm, sizeof(float) * old_count * dim, cudaMemcpyDeviceToDevice, st);
    count_launch();
    cudaFreeAsync(d_live, st);
  }
  e = kmeans_weighted(st, pooled, pw.data(), m + old_count, dim, K, uni, user, old_count > 0 ? warm : nullptr,
                      old_count, 10, atoms, weights, &iters);
  if (e == cudaSuccess && anchor)
    e = cudaMemcpyAsync(anchor, atoms, sizeof(float) * K * dim, cudaMemcpyDeviceToDevice, st);
  cudaFreeAsync(lc, st);
  cudaFreeAsync(pooled, st);
  cudaFreeAsync(warm, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

}  // namespace lm
