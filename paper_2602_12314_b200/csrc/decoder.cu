// decoder.cu — dictionary-attention decoder + feature loss, fp32 SIMT path.
//
// Reference: reconstruct / reconstruct_backward / trust_region_penalty
// (proj/src/dictionary.cpp:25-101), feature_loss (proj/src/losses.cpp:257-294) and
// their assembly in total_objective (proj/src/objective.cpp:100-185).
//
// The step path uses the factored algebra of the feature loss: with keys
// Kd = D W^T, Gram M = D D^T and target scores G = E D^T (E = the frame's
// embedding table), every per-row quantity the loss and its backward need is a
// K-vector:  nu^2 = P.(P M),  dot = P.G[a],  dP = alpha (P M) + beta G[a],
// so F_hat = P D (n x d_f) is never materialised. The reductions become
//   d_atoms = (P^T diag(alpha) P) D + Bm E + R^T W,   d_proj = R D,  R = Q^T dS.
// The same algebra runs on tcgen05 in decoder_tc.cu for the bf16 configurations.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace lm {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) sgemm_kernel(int64_t M, int64_t N, int64_t K, float alpha,
                                                    const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ B, int64_t ldb, float beta,
                                                    float* __restrict__ C, int64_t ldc, int64_t kchunk, bool atomic) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t i0 = (int64_t)blockIdx.y * BM, j0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * kchunk;
  const int64_t ke = min(K, kb + kchunk);
  float acc[4][4] = {};
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int e = tid + l * 256;  // 0..1023
      // A tile: rows i0..i0+63, cols k0..k0+15 -> As[kk][ii]
      {
        const int ii = TA ? e % BM : e / BK;
        const int kk = TA ? e / BM : e % BK;
        const int64_t gi = i0 + ii, gk = k0 + kk;
        float v = 0.f;
        if (gi < M && gk < ke) v = TA ? A[gk * lda + gi] : A[gi * lda + gk];
        As[kk][ii] = v;
      }
      {
        const int jj = TB ? e / BK : e % BN;
        const int kk = TB ? e % BK : e / BN;
        const int64_t gj = j0 + jj, gk = k0 + kk;
        float v = 0.f;
        if (gj < N && gk < ke) v = TB ? B[gj * ldb + gk] : B[gk * ldb + gj];
        Bs[kk][jj] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) av[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] += av[r] * bv[c];
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t gi = i0 + ty * 4 + r;
    if (gi >= M) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t gj = j0 + tx * 4 + c;
      if (gj >= N) continue;
      float* dst = C + gi * ldc + gj;
      const float v = alpha * acc[r][c];
      if (atomic)
        atomicAdd(dst, v);
      else
        *dst = beta == 0.f ? v : v + beta * *dst;
    }
  }
}

// Row softmax with max subtraction (dictionary.cpp:39-44); one warp per row.
__global__ void softmax_rows_kernel(float* __restrict__ x, int64_t n, int k) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (r >= n) return;
  const int lane = threadIdx.x & 31;
  float* row = x + r * k;
  float m = -INFINITY;
  for (int j = lane; j < k; j += 32) m = fmaxf(m, row[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int j = lane; j < k; j += 32) {
    const float e = expf(row[j] - m);
    row[j] = e;
    s += e;
  }
  s = warp_sum(s);
  const float inv = 1.f / s;
  for (int j = lane; j < k; j += 32) row[j] *= inv;
}

// Per-row feature loss + softmax backward, one warp per pixel row.
//   buf1 = P (n x K), buf2 = P M (n x K) -> overwritten with dS.
__global__ void decoder_rows_kernel(const float* __restrict__ P, float* __restrict__ T, int64_t n, int k,
                                    const int32_t* __restrict__ assign, const float* __restrict__ gt,
                                    const float* __restrict__ nv, float inv_temp, float lambda_cos, float lambda_l2,
                                    const int64_t* __restrict__ nsup, float scale, float* __restrict__ alpha_r,
                                    float* __restrict__ beta_r, double* partials) {
  const float inv_nsup = *nsup > 0 ? 1.f / (float)*nsup : 0.f;
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  double cos_acc = 0.0, l2_acc = 0.0, zflag = 0.0;
  if (r < n) {
    const int32_t a = assign[r];
    const float* p = P + r * k;
    float* t = T + r * k;
    if (a < 0) {
      for (int j = lane; j < k; j += 32) t[j] = 0.f;
      if (lane == 0) {
        alpha_r[r] = 0.f;
        beta_r[r] = 0.f;
      }
    } else {
      const float* g = gt + (int64_t)a * k;
      float nu2 = 0.f, dot = 0.f;
      for (int j = lane; j < k; j += 32) {
        nu2 += p[j] * t[j];
        dot += p[j] * g[j];
      }
      nu2 = warp_sum(nu2);
      dot = warp_sum(dot);
      const float eps = 1e-8f;
      const float nu = sqrtf(fmaxf(nu2, 0.f)), vn = nv[a];
      const float nug = fmaxf(nu, eps), nvg = fmaxf(vn, eps);
      if (lane == 0) {
        if (nu < eps || vn < eps) zflag = 1.0;
        cos_acc = 1.0 - (double)(dot / (nug * nvg));
        l2_acc = (double)nu2 - 2.0 * (double)dot + (double)vn * (double)vn;
      }
      // dF = al * F_hat + be * F  (losses.cpp:279-282)
      const float al = scale * (lambda_cos * dot / (nug * nug * nug * nvg) * inv_nsup + 2.f * lambda_l2 * inv_nsup);
      const float be = scale * (-lambda_cos / (nug * nvg) * inv_nsup - 2.f * lambda_l2 * inv_nsup);
      const float c = al * nu2 + be * dot;
      for (int j = lane; j < k; j += 32) t[j] = p[j] * (al * t[j] + be * g[j] - c) * inv_temp;
      if (lane == 0) {
        alpha_r[r] = al;
        beta_r[r] = be;
      }
    }
  }
  __shared__ double s_red[3][32];
  const int wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_red[0][wid] = cos_acc;
    s_red[1][wid] = l2_acc;
    s_red[2][wid] = zflag;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double c0 = 0, c1 = 0, c2 = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      c0 += s_red[0][i];
      c1 += s_red[1][i];
      c2 = fmax(c2, s_red[2][i]);
    }
    if (c0 != 0.0) atomicAdd(&partials[4], c0);
    if (c1 != 0.0) atomicAdd(&partials[5], c1);
    if (c2 != 0.0) atomicMax((unsigned long long*)&partials[6], (unsigned long long)__double_as_longlong(1.0));
  }
}

// Bm^T[s][k] += beta_r P[r][k] over rows with assignment s; rows are pixels in raster
// order, so runs of equal s are long and are summed before one atomic per run.
__global__ void bm_accum_kernel(const float* __restrict__ P, const float* __restrict__ beta_r,
                                const int32_t* __restrict__ assign, int64_t n, int k, int64_t rows_per_block,
                                float* __restrict__ bmt) {
  const int64_t r0 = blockIdx.y * rows_per_block;
  const int64_t r1 = min(n, r0 + rows_per_block);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    int32_t cur = -1;
    float acc = 0.f;
    for (int64_t r = r0; r < r1; ++r) {
      const int32_t s = assign[r];
      if (s != cur) {
        if (cur >= 0 && acc != 0.f) atomicAdd(&bmt[(int64_t)cur * k + j], acc);
        cur = s;
        acc = 0.f;
      }
      if (s >= 0) acc += beta_r[r] * P[r * k + j];
    }
    if (cur >= 0 && acc != 0.f) atomicAdd(&bmt[(int64_t)cur * k + j], acc);
  }
}

__global__ void scale_rows_kernel(const float* __restrict__ P, const float* __restrict__ s, float* __restrict__ out,
                                  int64_t n, int k) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * k; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = P[e] * s[e / k];
}

__global__ void row_norms_kernel(const float* __restrict__ x, int64_t n, int d, float* __restrict__ out) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (r >= n) return;
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  for (int j = lane; j < d; j += 32) s += x[r * d + j] * x[r * d + j];
  s = warp_sum(s);
  if (lane == 0) out[r] = sqrtf(s);
}

// Per-frame target scores and norms: G[s][k] = E[s] . D[k] (G = E D^T), nv[s] = |E[s]|.
// CTA = 4 target rows x 32 keys (E rows staged in shared memory); each warp takes 4 keys at a
// time with 4 x (df / 128) independent float4 loads of D in flight per lane. Requires df % 4 == 0.
constexpr int kTsRows = 4, kTsKeys = 32;  // 4 rows: twice the CTAs of 8 (48 -> 96 at n_set = 48)
__global__ void __launch_bounds__(256) target_scores_kernel(const float* __restrict__ feats,
                                                            const float* __restrict__ atoms, int64_t n_set, int k,
                                                            int df, float* __restrict__ gt, float* __restrict__ nv) {
  extern __shared__ __align__(16) float s_e[];  // kTsRows x df
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t s0 = (int64_t)blockIdx.x * kTsRows;
  const int nr = (int)(n_set - s0 < kTsRows ? n_set - s0 : kTsRows);
  const int k0 = blockIdx.y * kTsKeys;
  for (int i = tid; i < kTsRows * df / 4; i += blockDim.x) {
    const int r = i / (df / 4);
    reinterpret_cast<float4*>(s_e)[i] =
        r < nr ? __ldg(reinterpret_cast<const float4*>(feats + (s0 + r) * df) + i % (df / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  if (blockIdx.y == 0 && warp < nr) {  // norms of the CTA's rows
    float sq = 0.f;
    for (int j = lane; j < df; j += 32) sq += s_e[warp * df + j] * s_e[warp * df + j];
    sq = warp_sum(sq);
    if (lane == 0) nv[s0 + warp] = sqrtf(sq);
  }
  const float4* e4 = reinterpret_cast<const float4*>(s_e);
  for (int kq = k0 + 4 * warp; kq < min(k, k0 + kTsKeys); kq += 32) {
    float acc[4][kTsRows];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < kTsRows; ++r) acc[u][r] = 0.f;
    for (int j = lane; j < df / 4; j += 32) {
      float4 d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        d[u] = kq + u < k ? __ldg(reinterpret_cast<const float4*>(atoms + (size_t)(kq + u) * df) + j)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < kTsRows; ++r) {
        const float4 e = e4[r * (df / 4) + j];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          acc[u][r] = fmaf(d[u].x, e.x, fmaf(d[u].y, e.y, fmaf(d[u].z, e.z, fmaf(d[u].w, e.w, acc[u][r]))));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < kTsRows; ++r) {
        const float v = warp_sum(acc[u][r]);
        if (lane == 0 && r < nr && kq + u < k) gt[(s0 + r) * k + kq + u] = v;
      }
  }
}

// d_atoms[k][:] += sum_s Bm^T[s][k] E[s][:]  (the frame's Bm E term). CTA = 4 keys x 128
// float4 columns; the E row load of each s is shared by the 4 keys. Requires df % 4 == 0.
__global__ void __launch_bounds__(128) bm_embed_kernel(const float* __restrict__ bmt, const float* __restrict__ feats,
                                                       int64_t n_set, int k, int df, float* __restrict__ d_atoms) {
  const int k0 = blockIdx.x * 4;
  const int c4 = blockIdx.y * blockDim.x + threadIdx.x;
  if (c4 >= df / 4) return;
  float4 acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int64_t sidx = 0; sidx < n_set; ++sidx) {
    const float4 e = __ldg(reinterpret_cast<const float4*>(feats + sidx * df) + c4);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float b = k0 + u < k ? __ldg(bmt + sidx * k + k0 + u) : 0.f;
      acc[u].x = fmaf(b, e.x, acc[u].x);
      acc[u].y = fmaf(b, e.y, acc[u].y);
      acc[u].z = fmaf(b, e.z, acc[u].z);
      acc[u].w = fmaf(b, e.w, acc[u].w);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (k0 + u >= k) break;
    float4* dst = reinterpret_cast<float4*>(d_atoms + (size_t)(k0 + u) * df) + c4;
    float4 d = *dst;
    d.x += acc[u].x;
    d.y += acc[u].y;
    d.z += acc[u].z;
    d.w += acc[u].w;
    *dst = d;
  }
}

// softmax backward rows (dictionary.cpp:69-74): d = P * (d - rowdot(P, d)) / temperature
__global__ void softmax_bwd_rows_kernel(const float* __restrict__ P, float* __restrict__ d, int64_t n, int k,
                                        float temperature) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (r >= n) return;
  const int lane = threadIdx.x & 31;
  const float* p = P + r * k;
  float* x = d + r * k;
  float dot = 0.f;
  for (int j = lane; j < k; j += 32) dot += p[j] * x[j];
  dot = warp_sum(dot);
  for (int j = lane; j < k; j += 32) x[j] = p[j] * (x[j] - dot) / temperature;
}

__global__ void scale_kernel(float* x, int64_t n, float s) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    x[e] *= s;
}

// trust_region_penalty (dictionary.cpp:85-101): one block per atom row.
__global__ void trust_kernel(const float* __restrict__ atoms, const float* __restrict__ anchor, int64_t k, int df,
                             float delta, float* d_atoms, float grad_scale, double* penalty) {
  __shared__ float red[32];
  const int64_t j = blockIdx.x;
  float ss = 0.f;
  for (int c = threadIdx.x; c < df; c += blockDim.x) {
    const float d = atoms[j * df + c] - anchor[j * df + c];
    ss += d * d;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float dist = sqrtf(red[0]);
  const float excess = dist - delta;
  if (excess > 0.f) {
    if (threadIdx.x == 0 && penalty) atomicAdd(penalty, (double)excess);
    if (d_atoms)
      for (int c = threadIdx.x; c < df; c += blockDim.x)
        d_atoms[j * df + c] += grad_scale * ((atoms[j * df + c] - anchor[j * df + c]) / dist);
  }
}

inline int grid_for(int64_t n, int per_block, int cap = 148 * 32) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + per_block - 1) / per_block, cap));
}

}  // namespace

// zero an M x N block of a row-major matrix with leading dimension ldc (one launch)
__global__ void zero_block_kernel(float* C, int64_t M, int64_t N, int64_t ldc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * N; e += (int64_t)gridDim.x * blockDim.x)
    C[(e / N) * ldc + e % N] = 0.f;
}
static void zero_block(cudaStream_t st, float* C, int64_t M, int64_t N, int64_t ldc) {
  if (ldc == N) {
    cudaMemsetAsync(C, 0, sizeof(float) * M * N, st);
  } else {
    zero_block_kernel<<<(unsigned)std::min<int64_t>((M * N + 255) / 256, 1184), 256, 0, st>>>(C, M, N, ldc);
    count_launch();
  }
}

void sgemm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, float alpha, const float* A,
           int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc, int split) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    if (split <= 1 && beta == 0.f) zero_block(st, C, M, N, ldc);
    return;
  }
  const int64_t gx = (N + BN - 1) / BN, gy = (M + BM - 1) / BM;
  if (split < 1) split = 1;
  // small output grids with long reductions: split K across CTAs (atomics into C); C is
  // pre-zeroed for beta == 0, accumulated into for beta == 1.
  if (split == 1 && !deterministic() && gx * gy < 148 && K >= 256 && (beta == 0.f || beta == 1.f)) {
    const int64_t want = (296 + gx * gy - 1) / (gx * gy);
    split = (int)std::max<int64_t>(1, std::min<int64_t>(want, K / 128));
    if (split > 1 && beta == 0.f) zero_block(st, C, M, N, ldc);
  }
  const int64_t kchunk = ((K + split - 1) / split + BK - 1) / BK * BK;
  const int gz = (int)((K + kchunk - 1) / kchunk);
  const bool atomic = gz > 1 || split > 1;
  dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)gz);
  if (!ta && !tb) sgemm_kernel<false, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, atomic);
  if (!ta && tb) sgemm_kernel<false, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, atomic);
  if (ta && !tb) sgemm_kernel<true, false><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, atomic);
  if (ta && tb) sgemm_kernel<true, true><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, atomic);
  count_launch();
}

// split-K factor of the long reductions (atomics); 1 in deterministic mode (fixed order)
static int split_for(int64_t M, int64_t N, int64_t K) {
  if (deterministic()) return 1;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int64_t s = (148 * 4 + tiles - 1) / tiles;
  s = std::min<int64_t>(s, std::max<int64_t>(1, K / 512));
  return (int)std::max<int64_t>(1, s);
}

void decoder_prepare(cudaStream_t st, DecoderWork& w, const float* atoms, const float* proj) {
  // Kd = D W^T (K x ds), M = D D^T (K x K)
  sgemm(st, false, true, w.k, w.ds, w.df, 1.f, atoms, w.df, proj, w.df, 0.f, w.kd, w.ds);
  sgemm(st, false, true, w.k, w.k, w.df, 1.f, atoms, w.df, atoms, w.df, 0.f, w.mm, w.k);
  decoder_tc_images(st, w);
  if (w.a_acc) cudaMemsetAsync(w.a_acc, 0, sizeof(float) * w.k * w.k, st);
  if (w.r_acc) cudaMemsetAsync(w.r_acc, 0, sizeof(float) * w.ds * w.k, st);
  w.tc_pending = false;
  w.tc_frames = 0;
}

void decoder_frame(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment, int64_t npx,
                   const float* feats, int64_t n_set, const int64_t* nsup, const float* atoms, const float* proj,
                   float temperature, float lambda_cos, float lambda_l2, float scale, bool want_grad, float* d_query,
                   float* d_proj, float* d_atoms, double* partials) {
  const int64_t k = w.k;
  const int ds = w.ds, df = w.df;
  const float inv_temp = 1.f / temperature;
  // per-frame target scores G^T = E D^T (n_set x K) and target norms
  decoder_targets(st, feats, n_set, atoms, k, df, w.gt, w.nv);
  // S = Q Kd^T / temperature ; P = softmax(S)
  sgemm(st, false, true, npx, k, ds, inv_temp, query, ds, w.kd, ds, 0.f, w.buf1, k);
  softmax_rows_kernel<<<grid_for(npx * 32, 256, 1 << 30), 256, 0, st>>>(w.buf1, npx, (int)k);
  count_launch();
  // buf2 = P M
  sgemm(st, false, false, npx, k, k, 1.f, w.buf1, k, w.mm, k, 0.f, w.buf2, k);
  decoder_rows_kernel<<<grid_for(npx * 32, 256, 1 << 30), 256, 0, st>>>(
      w.buf1, w.buf2, npx, (int)k, assignment, w.gt, w.nv, inv_temp, lambda_cos, lambda_l2,
      nsup, scale, w.alpha_r, w.beta_r, partials);
  count_launch();
  if (!want_grad) return;
  // d_query = dS Kd   (n x ds)
  sgemm(st, false, false, npx, ds, k, 1.f, w.buf2, k, w.kd, ds, 0.f, d_query, ds);
  // R = Q^T dS  (ds x K), reduction over pixels
  cudaMemsetAsync(w.r, 0, sizeof(float) * ds * k, st);
  sgemm(st, true, false, ds, k, npx, 1.f, query, ds, w.buf2, k, 0.f, w.r, k, split_for(ds, k, npx));
  // Bm^T (n_set x K)
  cudaMemsetAsync(w.bm, 0, sizeof(float) * n_set * k, st);
  {
    const int64_t rpb = deterministic() ? std::max<int64_t>(npx, 1) : 512;  // one row block: one writer
    dim3 g((unsigned)((k + 127) / 128), (unsigned)((npx + rpb - 1) / rpb));
    bm_accum_kernel<<<g, 128, 0, st>>>(w.buf1, w.beta_r, assignment, npx, (int)k, rpb, w.bm);
    count_launch();
  }
  // A = P^T diag(alpha) P  (K x K)
  scale_rows_kernel<<<grid_for(npx * k, 256), 256, 0, st>>>(w.buf1, w.alpha_r, w.buf2, npx, (int)k);
  count_launch();
  cudaMemsetAsync(w.a, 0, sizeof(float) * k * k, st);
  sgemm(st, true, false, k, k, npx, 1.f, w.buf1, k, w.buf2, k, 0.f, w.a, k, split_for(k, k, npx));
  // d_atoms += A D + Bm E + R^T W ;  d_proj += R D
  sgemm(st, false, false, k, df, k, 1.f, w.a, k, atoms, df, 1.f, d_atoms, df);
  decoder_bm_embed(st, w.bm, feats, n_set, k, df, d_atoms);
  sgemm(st, true, false, k, df, ds, 1.f, w.r, k, proj, df, 1.f, d_atoms, df);
  sgemm(st, false, false, ds, df, k, 1.f, w.r, k, atoms, df, 1.f, d_proj, df);
}

void decoder_target_norms(cudaStream_t st, const float* feats, int64_t n_set, int df, float* nv) {
  row_norms_kernel<<<grid_for(n_set * 32, 256), 256, 0, st>>>(feats, n_set, df, nv);
  count_launch();
}

void decoder_targets(cudaStream_t st, const float* feats, int64_t n_set, const float* atoms, int64_t k, int df,
                     float* gt, float* nv) {
  if (n_set <= 0) return;
  if (df % 4 == 0 && (reinterpret_cast<uintptr_t>(feats) & 15) == 0 && (reinterpret_cast<uintptr_t>(atoms) & 15) == 0) {
    const size_t sm = sizeof(float) * kTsRows * df;
    if (sm > 48 * 1024) cudaFuncSetAttribute(target_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid((unsigned)((n_set + kTsRows - 1) / kTsRows), (unsigned)((k + kTsKeys - 1) / kTsKeys));
    target_scores_kernel<<<grid, 256, sm, st>>>(feats, atoms, n_set, (int)k, df, gt, nv);
    count_launch();
  } else {
    sgemm(st, false, true, n_set, k, df, 1.f, feats, df, atoms, df, 0.f, gt, k);
    decoder_target_norms(st, feats, n_set, df, nv);
  }
}

void decoder_bm_embed(cudaStream_t st, const float* bmt, const float* feats, int64_t n_set, int64_t k, int df,
                      float* d_atoms) {
  if (n_set <= 0) return;
  if (df % 4 == 0 && (reinterpret_cast<uintptr_t>(feats) & 15) == 0 && (reinterpret_cast<uintptr_t>(d_atoms) & 15) == 0) {
    dim3 grid((unsigned)((k + 3) / 4), (unsigned)((df / 4 + 127) / 128));
    bm_embed_kernel<<<grid, 128, 0, st>>>(bmt, feats, n_set, (int)k, df, d_atoms);
    count_launch();
  } else {
    sgemm(st, true, false, k, df, n_set, 1.f, bmt, k, feats, df, 1.f, d_atoms, df);
  }
}

void reconstruct(cudaStream_t st, const float* q, int64_t n, int ds, const float* atoms, const float* proj, int64_t k,
                 int df, float temperature, float* out, float* attention, float* scratch_qw) {
  // logits = (Q W) D^T / temperature (dictionary.cpp:37)
  sgemm(st, false, false, n, df, ds, 1.f, q, ds, proj, df, 0.f, scratch_qw, df);
  sgemm(st, false, true, n, k, df, 1.f / temperature, scratch_qw, df, atoms, df, 0.f, attention, k);
  softmax_rows_kernel<<<grid_for(n * 32, 256, 1 << 30), 256, 0, st>>>(attention, n, (int)k);
  count_launch();
  sgemm(st, false, false, n, df, k, 1.f, attention, k, atoms, df, 0.f, out, df);
}

void reconstruct_backward(cudaStream_t st, const float* q, const float* att, int64_t n, int ds, const float* atoms,
                          const float* proj, int64_t k, int df, float temperature, const float* d_rec, float* d_q,
                          float* d_proj, float* d_atoms, float* s_nk, float* s_ndf, float* s_kdf) {
  // d_logits = dF D^T, softmax backward, / temperature (dictionary.cpp:68-74)
  sgemm(st, false, true, n, k, df, 1.f, d_rec, df, atoms, df, 0.f, s_nk, k);
  softmax_bwd_rows_kernel<<<grid_for(n * 32, 256, 1 << 30), 256, 0, st>>>(att, s_nk, n, (int)k, temperature);
  count_launch();
  // d_atoms = P^T dF + d_logits^T (Q W)   (dictionary.cpp:77-78)
  sgemm(st, false, false, n, df, ds, 1.f, q, ds, proj, df, 0.f, s_ndf, df);
  cudaMemsetAsync(d_atoms, 0, sizeof(float) * k * df, st);
  sgemm(st, true, false, k, df, n, 1.f, att, k, d_rec, df, 0.f, d_atoms, df, split_for(k, df, n));
  if (deterministic())  // accumulate with beta = 1 (no split: one writer per element)
    sgemm(st, true, false, k, df, n, 1.f, s_nk, k, s_ndf, df, 1.f, d_atoms, df, 1);
  else
    sgemm(st, true, false, k, df, n, 1.f, s_nk, k, s_ndf, df, 0.f, d_atoms, df, std::max(2, split_for(k, df, n)));
  // d_qw = d_logits D ; d_proj = Q^T d_qw ; d_q = d_qw W^T (dictionary.cpp:79-81)
  sgemm(st, false, false, n, df, k, 1.f, s_nk, k, atoms, df, 0.f, s_ndf, df);
  cudaMemsetAsync(d_proj, 0, sizeof(float) * ds * df, st);
  sgemm(st, true, false, ds, df, n, 1.f, q, ds, s_ndf, df, 0.f, d_proj, df,
        deterministic() ? 1 : std::max(2, split_for(ds, df, n)));
  sgemm(st, false, true, n, ds, df, 1.f, s_ndf, df, proj, df, 0.f, d_q, ds);
  (void)s_kdf;
}

void trust_region(cudaStream_t st, const float* atoms, const float* anchor, int64_t k, int df, float delta,
                  float* d_atoms, float grad_scale, double* penalty_out) {
  if (k <= 0) return;
  trust_kernel<<<(unsigned)k, 256, 0, st>>>(atoms, anchor, k, df, delta, d_atoms, grad_scale, penalty_out);
  count_launch();
}

}  // namespace lm
