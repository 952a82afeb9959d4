// decoder_tc.cu — dictionary-attention decoder + feature loss + backward on 5th-gen tensor
// cores (tcgen05.mma, bf16 operands, fp32 accumulators in TMEM), for K in {128, 256}.
//
// Reference semantics: reconstruct (proj/src/dictionary.cpp:25-53), feature_loss
// (proj/src/losses.cpp:257-294), reconstruct_backward (dictionary.cpp:55-83) as assembled by
// total_objective (proj/src/objective.cpp:100-185). Same factored algebra as decoder.cu:
//
//   S = Q Kd^T (Kd = D W^T),  P = softmax(S / tau),  t = P M (M = D D^T),
//   nu^2 = P.t,  dot = P.G[a] (G = E D^T),  dF = alpha F_hat + beta F (per-row scalars),
//   dS = P * (alpha t + beta G[a] - (alpha nu^2 + beta dot)) / tau,
//   dQ = dS Kd,  R^T = dS^T Q,  A = P^T diag(alpha) P,  Bm = P^T Ohb (Ohb[r][s] = beta_r [a_r == s])
//   d_atoms += A D + Bm E + R^T W,   d_proj += R D.
//
// DEC1 (persistent, 1 CTA / SM, 512 threads): per 128-pixel tile
//   MMA1 S -> TMEM[0,K); softmax epilogue writes bf16 e = exp(S - max) to smem (and streams it
//   to HBM for DEC2); MMA2 t = e M -> TMEM[0,K); loss / alpha / beta epilogue; dS (bf16)
//   overwrites e; MMA3 dQ = dS Kd -> TMEM[K,K+DS); MMA4 R^T += dS^T Q -> TMEM[K+DS, ...)
//   (accumulated across the CTA's tiles); dQ rows go to HBM.
// DEC2 (persistent, warp-specialised, two roles = two column halves of A): streams DEC1's e
//   tiles back with TMA, scales them by the row statistics and accumulates A[:, half] and Bm
//   in TMEM.
// Shared-memory operand tiles use the no-swizzle core-matrix layout of tc_common.cuh with
// row-group stride 128 B and column-group stride 16 * rows B, so one tile serves as a K-major
// operand (rows = M|N) and, transposed, as an MN-major operand (rows = K).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace lm {

namespace {

constexpr int kRows = 128;        // pixels per tile (UMMA M)
constexpr float kLog2e = 1.4426950408889634f;

struct Dec1Args {
  uint8_t* e_tiles;         // ntiles x (128 x K bf16) in the smem core-matrix layout (for DEC2)
  const float* query;       // npx x DS (fp32, raster order)
  const int32_t* assign;    // npx
  const float* kd;          // K x DS fp32 (D W^T)
  const float* mm;          // K x K  fp32 (D D^T)
  const float* gt;          // n_set x K fp32 (E D^T)
  const float* nv;          // n_set (target row norms)
  int64_t npx;
  float inv_temp, lambda_cos, lambda_l2, scale;
  const int64_t* nsup;      // supervised rows (device)
  float* d_query;           // npx x DS
  float4* row_stats;        // npx: (max S, 1/sum, alpha, beta)
  float* r_part;            // gridDim x K x DS
  double* loss_part;        // gridDim x 4
  int want_grad;
  int accum;                // add R^T into r_part (later frames of a step) instead of storing
  float2* row_nd;           // optional parity export: per-row (nu^2, dot)
  const uint8_t* img;       // bf16 core-matrix images of Kd then M (decoder_prepare), or null
};

template <int K, int DS>
__global__ void __launch_bounds__(512, 1) dec1_kernel(Dec1Args a) {
  constexpr int NT = 512;      // 16 warps: 4 TMEM lane groups x 4 column quarters
  constexpr int MH = K / 128;  // M halves of R^T
  constexpr int kColDQ = K, kColR = K + DS;
  constexpr int kTmemCols = (K + DS + MH * DS) <= 256 ? 256 : 512;
  constexpr int QC = K / 4;               // columns per quarter
  constexpr uint32_t kCS = 16u * kRows;   // column-group stride of 128-row tiles
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;                              // 128 x DS
  uint8_t* sKd = sQ + kRows * DS * 2;              // K x DS
  uint8_t* sP = sKd + K * DS * 2;                  // 128 x K  (e, then dS)
  uint8_t* sM = sP + kRows * K * 2;                // K x K
  float* s_red = reinterpret_cast<float*>(sM + K * K * 2);  // [4 quantities][4 quarters][128]
  __shared__ uint64_t bar[4];  // MMA1, MMA2, MMA3/4 completion; [3] the Kd / M image load
  __shared__ uint32_t s_taddr;
  __shared__ double s_loss[16][3];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp & 3, qt = warp >> 2;  // TMEM lane group, column quarter
  const int row = 32 * g + lane;
  const int c0 = qt * QC;
  auto red = [&](int q, int quarter) -> float& { return s_red[(q * 4 + quarter) * 128 + row]; };

  if (!a.img) {
    tc::load_tile_bf16(sKd, a.kd, K, DS, K, tid, NT);
    tc::load_tile_bf16(sM, a.mm, K, K, K, tid, NT);
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1);
    tc::fence_mbar_init();
    if (a.img) {  // the step's operand images (144 KB at K = 256): two bulk copies, waited before MMA1
      tc::mbar_expect_tx(&bar[3], (uint32_t)(K * DS * 2 + K * K * 2));
      tc::bulk_g2s(sKd, a.img, (uint32_t)(K * DS * 2), &bar[3]);
      tc::bulk_g2s(sM, a.img + K * DS * 2, (uint32_t)(K * K * 2), &bar[3]);
    }
  }
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&s_taddr);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s_taddr;
  const uint32_t tl = tmem + ((uint32_t)(32 * g) << 16);  // this warp's TMEM lane base
  uint32_t ph[3] = {0, 0, 0};

  const uint32_t idesc1 = tc::make_idesc_bf16(128, K, 0, 0);
  const uint32_t idesc3 = tc::make_idesc_bf16(128, DS, 0, 1);
  const uint32_t idesc4 = tc::make_idesc_bf16(128, DS, 1, 1);
  const uint32_t aQ = tc::smem_u32(sQ), aKd = tc::smem_u32(sKd), aP = tc::smem_u32(sP), aM = tc::smem_u32(sM);
  const float cl = kLog2e * a.inv_temp;
  const float inv_nsup = *a.nsup > 0 ? 1.f / (float)*a.nsup : 0.f;
  double cos_acc = 0.0, l2_acc = 0.0, zflag = 0.0;
  bool first = true;

  // Q tile prefetch: each thread owns 8 consecutive values (one 16-byte core row chunk)
  constexpr int QCH = kRows * DS / 8;  // 8-value chunks per tile
  static_assert(QCH <= NT, "one Q chunk per thread");
  const int qr = tid / (DS / 8), qc = (tid % (DS / 8)) * 8;
  float4 qpre[2];
  auto q_fetch = [&](int64_t r0, int valid) {
    if (tid < QCH && qr < valid) {
      const float4* src = reinterpret_cast<const float4*>(a.query + (r0 + qr) * DS + qc);
      qpre[0] = src[0];
      qpre[1] = src[1];
    } else {
      qpre[0] = qpre[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto q_store = [&]() {
    if (tid < QCH) {
      const float v[8] = {qpre[0].x, qpre[0].y, qpre[0].z, qpre[0].w, qpre[1].x, qpre[1].y, qpre[1].z, qpre[1].w};
      tc::st_row8(sQ, qr, qc, kCS, v);
    }
  };
  const int64_t ntiles = (a.npx + kRows - 1) / kRows;
  if ((int64_t)blockIdx.x < ntiles) {
    const int64_t r0 = (int64_t)blockIdx.x * kRows;
    q_fetch(r0, (int)(a.npx - r0 < kRows ? a.npx - r0 : kRows));
  }
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kRows;
    const int valid = (int)(a.npx - r0 < kRows ? a.npx - r0 : kRows);
    q_store();
    tc::fence_async_smem();
    __syncthreads();
    // ---- MMA1: S = Q Kd^T  -> TMEM[0, K)
    if (tid == 0) {
      if (a.img && first) tc::mbar_wait(&bar[3], 0);
      tc::tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < DS / 16; ++ks)
        tc::mma_bf16(tmem, tc::make_sdesc(aQ + ks * 2 * 2048, 2048, 128),
                     tc::make_sdesc(aKd + ks * 2 * (16 * K), 16 * K, 128), idesc1, ks > 0);
      tc::mma_commit(&bar[0]);
    }
    // row data for this tile (overlaps MMA1)
    const int64_t grow = r0 + row;
    const int32_t asg = row < valid ? a.assign[grow] : -1;
    const float* grow_ptr = a.gt + (int64_t)(asg < 0 ? 0 : asg) * K + c0;
    tc::mbar_wait(&bar[0], ph[0]);
    ph[0] ^= 1;
    tc::tc_fence_after();
    uint8_t* e_out = a.want_grad ? a.e_tiles + (size_t)tile * kRows * K * 2 + (size_t)(row >> 6) * 64 * K * 2 : nullptr;
    // ---- softmax: row max, then e = exp(S - max) (bf16) and the row sum
    float sv[QC];
#pragma unroll
    for (int c = 0; c < QC; c += 32) tc::tmem_ld32_nw(tl + c0 + c, sv + c);
    tc::tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < QC; c += 32) tc::tmem_reg_fence32(sv + c);
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < QC; ++i) mx = fmaxf(mx, sv[i]);
    red(0, qt) = mx;
    __syncthreads();
    mx = fmaxf(fmaxf(red(0, 0), red(0, 1)), fmaxf(red(0, 2), red(0, 3)));
    const float mxl = mx * cl;
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < QC; c += 8) {
      uint4 u;
      u.x = tc::pack_bf16(tc::ex2(fmaf(sv[c + 0], cl, -mxl)), tc::ex2(fmaf(sv[c + 1], cl, -mxl)));
      u.y = tc::pack_bf16(tc::ex2(fmaf(sv[c + 2], cl, -mxl)), tc::ex2(fmaf(sv[c + 3], cl, -mxl)));
      u.z = tc::pack_bf16(tc::ex2(fmaf(sv[c + 4], cl, -mxl)), tc::ex2(fmaf(sv[c + 5], cl, -mxl)));
      u.w = tc::pack_bf16(tc::ex2(fmaf(sv[c + 6], cl, -mxl)), tc::ex2(fmaf(sv[c + 7], cl, -mxl)));
      *reinterpret_cast<uint4*>(sP + tc::core_off(row, c0 + c, 128u, kCS)) = u;
      if (e_out)  // DEC2's copy, half-major: rows 0-63 then 64-127, each a contiguous 64-row tile
        *reinterpret_cast<uint4*>(e_out + tc::core_off(row & 63, c0 + c, 128u, 16u * 64)) = u;
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};  // sum the bf16-rounded e the MMA consumes
#pragma unroll
      for (int j = 0; j < 4; ++j) sum += __uint_as_float(w4[j] << 16) + __uint_as_float(w4[j] & 0xffff0000u);
    }
    red(1, qt) = sum;
    tc::fence_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    const float inv_sum = 1.f / ((red(1, 0) + red(1, 1)) + (red(1, 2) + red(1, 3)));
    // ---- MMA2: t = e M -> TMEM[0, K) (S is dead)
    if (tid == 0) {
      tc::tc_fence_after();
#pragma unroll 4
      for (int ks = 0; ks < K / 16; ++ks)
        tc::mma_bf16(tmem, tc::make_sdesc(aP + ks * 2 * 2048, 2048, 128),
                     tc::make_sdesc(aM + ks * 2 * (16 * K), 16 * K, 128), idesc1, ks > 0);
      tc::mma_commit(&bar[1]);
    }
    // dot = P.G[a] needs only e (read-only for MMA2 too) and the target-score row: computed
    // while MMA2 runs
    float dot = 0.f;
#pragma unroll
    for (int c = 0; c < QC; c += 8) {
      float e[8];
      tc::ld_row8(sP, row, c0 + c, kCS, e);
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(grow_ptr + c));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(grow_ptr + c + 4));
      const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) dot = fmaf(e[j], gv[j], dot);
    }
    tc::mbar_wait(&bar[1], ph[1]);
    ph[1] ^= 1;
    tc::tc_fence_after();
    // ---- per-row statistics: nu^2 = P.t, dot = P.G[a]   (P = e / sum, t = (e M) / sum)
    float tv[QC];
#pragma unroll
    for (int c = 0; c < QC; c += 32) tc::tmem_ld32_nw(tl + c0 + c, tv + c);
    tc::tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < QC; c += 32) tc::tmem_reg_fence32(tv + c);
    float nu2 = 0.f;
#pragma unroll
    for (int c = 0; c < QC; c += 8) {
      float e[8];
      tc::ld_row8(sP, row, c0 + c, kCS, e);
#pragma unroll
      for (int j = 0; j < 8; ++j) nu2 = fmaf(e[j], tv[c + j], nu2);
    }
    red(2, qt) = nu2;
    red(3, qt) = dot;
    __syncthreads();
    nu2 = ((red(2, 0) + red(2, 1)) + (red(2, 2) + red(2, 3))) * inv_sum * inv_sum;
    dot = ((red(3, 0) + red(3, 1)) + (red(3, 2) + red(3, 3))) * inv_sum;
    float al = 0.f, be = 0.f, cc = 0.f;
    if (asg >= 0) {
      const float eps = 1e-8f;
      const float nu = sqrtf(fmaxf(nu2, 0.f)), vn = a.nv[asg];
      const float nug = fmaxf(nu, eps), nvg = fmaxf(vn, eps);
      if (qt == 0) {
        if (nu < eps || vn < eps) zflag = 1.0;
        cos_acc += 1.0 - (double)(dot / (nug * nvg));
        l2_acc += (double)nu2 - 2.0 * (double)dot + (double)vn * (double)vn;
      }
      al = a.scale * (a.lambda_cos * dot / (nug * nug * nug * nvg) * inv_nsup + 2.f * a.lambda_l2 * inv_nsup);
      be = a.scale * (-a.lambda_cos / (nug * nvg) * inv_nsup - 2.f * a.lambda_l2 * inv_nsup);
      cc = al * nu2 + be * dot;
    }
    if (qt == 0 && row < valid) {
      a.row_stats[grow] = make_float4(mx, inv_sum, al, be);
      if (a.row_nd) a.row_nd[grow] = make_float2(nu2, dot);
    }
    // next tile's Q (consumed after this tile's MMA4 has read sQ)
    if (tile + gridDim.x < ntiles) {
      const int64_t nr0 = (tile + gridDim.x) * kRows;
      q_fetch(nr0, (int)(a.npx - nr0 < kRows ? a.npx - nr0 : kRows));
    }
    if (!a.want_grad) {
      tc::tc_fence_before();
      __syncthreads();
      continue;
    }
    // ---- dS = P (al t + be g - c) / tau  (bf16, overwrites e in sP: every thread rewrites only
    // the chunks it wrote and read itself, and MMA2 -- the last async reader -- has completed)
    const float ps = inv_sum * a.inv_temp;  // P = e * inv_sum
    const float al_t = al * inv_sum;        // al * t = al * inv_sum * (e M)
#pragma unroll
    for (int c = 0; c < QC; c += 8) {
      float e[8];
      tc::ld_row8(sP, row, c0 + c, kCS, e);
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(grow_ptr + c));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(grow_ptr + c + 4));
      const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) e[j] = e[j] * ps * fmaf(al_t, tv[c + j], fmaf(be, gv[j], -cc));
      tc::st_row8(sP, row, c0 + c, kCS, e);
    }
    tc::fence_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    // ---- MMA3: dQ = dS Kd -> TMEM[K, K+DS);  MMA4: R^T += dS^T Q -> TMEM[K+DS + DS*mh, ...)
    if (tid == 0) {
      tc::tc_fence_after();
#pragma unroll 4
      for (int ks = 0; ks < K / 16; ++ks)
        tc::mma_bf16(tmem + kColDQ, tc::make_sdesc(aP + ks * 2 * 2048, 2048, 128),
                     tc::make_sdesc(aKd + ks * 2 * 128, 128, 16 * K), idesc3, ks > 0);
#pragma unroll
      for (int mh = 0; mh < MH; ++mh)
#pragma unroll
        for (int ks = 0; ks < kRows / 16; ++ks)
          tc::mma_bf16(tmem + kColR + DS * mh, tc::make_sdesc(aP + mh * 16 * 2048 + ks * 2 * 128, 128, 2048),
                       tc::make_sdesc(aQ + ks * 2 * 128, 128, 2048), idesc4, (!first) || ks > 0);
      tc::mma_commit(&bar[2]);
    }
    first = false;
    tc::mbar_wait(&bar[2], ph[2]);
    ph[2] ^= 1;
    tc::tc_fence_after();
    if (qt == 0) {
      float v[DS];
#pragma unroll
      for (int c = 0; c < DS; c += 16) tc::tmem_ld16(tl + kColDQ + c, v + c);  // warp-aligned: all lanes load
      if (row < valid) {
        float4* dst = reinterpret_cast<float4*>(a.d_query + grow * DS);
#pragma unroll
        for (int c = 0; c < DS; c += 4) dst[c / 4] = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
      }
    }
    tc::tc_fence_before();
    __syncthreads();
  }
  // ---- flush per-CTA partials: R^T rows k = 32g + lane (+128 mh)
  if (qt == 1) {
#pragma unroll
    for (int mh = 0; mh < MH; ++mh) {
      float v[DS];
      if (first) {
#pragma unroll
        for (int c = 0; c < DS; ++c) v[c] = 0.f;
      } else {
#pragma unroll
        for (int c = 0; c < DS; c += 16) tc::tmem_ld16(tl + kColR + DS * mh + c, v + c);
      }
      float4* dst = reinterpret_cast<float4*>(a.r_part + ((size_t)blockIdx.x * K + mh * 128 + row) * DS);
#pragma unroll
      for (int c = 0; c < DS; c += 4) {
        float4 o = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        if (a.accum) {
          const float4 p = dst[c / 4];
          o.x += p.x, o.y += p.y, o.z += p.z, o.w += p.w;
        }
        dst[c / 4] = o;
      }
    }
  }
  cos_acc = warp_sum_d(cos_acc);
  l2_acc = warp_sum_d(l2_acc);
  zflag = warp_sum_d(zflag);
  if (lane == 0) {
    s_loss[warp][0] = cos_acc;
    s_loss[warp][1] = l2_acc;
    s_loss[warp][2] = zflag;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc::bulk_wait_all();
    double c0s = 0, c1s = 0, c2s = 0;
    for (int w = 0; w < 16; ++w) c0s += s_loss[w][0], c1s += s_loss[w][1], c2s += s_loss[w][2];
    a.loss_part[blockIdx.x * 4 + 0] = c0s;
    a.loss_part[blockIdx.x * 4 + 1] = c1s;
    a.loss_part[blockIdx.x * 4 + 2] = c2s;
  }
  if (warp == 0) tc::tmem_free<kTmemCols>(tmem);
}

struct Dec2Args {
  const uint8_t* e_tiles;    // from DEC1: per tile 128 x K bf16 e = exp(S - max), core-matrix layout
  const int32_t* assign;
  const float4* row_stats;   // (max, 1/sum, alpha, beta)
  int64_t npx;
  float* a_part;   // this frame's slot: gridDim x 2 halves x K x (K/2)
  float* bm_part;  // (gridDim/2) x K x 64  (role 0 only)
  int accum;       // add A into the slot (frames past the last slot) instead of storing
};

// DEC2: A = e^T diag(alpha / sum^2) e and Bm = e^T Ohb (Ohb[r][s] = beta_r / sum_r [a_r == s]),
// streaming the e tiles DEC1 exported -- no recomputation of S or exp. One CTA per group of
// tiles (kDec2Groups); A is symmetric, so at K = 256 only its blocks A00, A01, A11 are
// accumulated (3 x 128 TMEM columns, Bm's two 128-row halves take the other 128) and the drain
// writes A10 = A01^T. Warp-specialised: warp 8 (one elected lane) issues the TMA bulk loads and
// the MMAs; warps 0-7 build the scaled B operands (alpha / sum^2) e over all K columns and the
// one-hot Ohb. The pipeline unit is a half tile (64 pixel rows, one contiguous 32 KB copy: DEC1
// exports each tile half-major) in a ring of kStages stages.
//   bar_ld[s]    : half tile landed in sE[s]            (TMA complete_tx)
//   bar_built[s] : 8 builder warps filled sAP/sOh[s]     (8 arrivals)
//   bar_mma[s]   : MMAs reading sE/sAP/sOh[s] done       (tcgen05.commit)
// The load of half tile i into stage s is issued only after the MMAs of half tile i - kStages
// (the last user of s) completed, so a builder that sees bar_ld[s] may also overwrite sAP/sOh[s].
constexpr int kHalf = kRows / 2;  // pixel rows per pipeline unit
constexpr int kDec2Groups = 148;
constexpr int kDec2Slots = 8;  // per-frame A partial slots (see launch_tc)
template <int K>
constexpr int dec2_stages() {
  return K == 256 ? 3 : 4;
}
template <int K>
constexpr size_t dec2_smem() {
  return (size_t)dec2_stages<K>() * ((size_t)kHalf * K * 2 * 2 + (size_t)kHalf * 64 * 2);
}

template <int K>
__global__ void __launch_bounds__(288, 1) dec2_kernel(Dec2Args a) {
  constexpr int kStages = dec2_stages<K>();
  constexpr int MH = K / 128, NB = 64;
  // TMEM: the A blocks (128 columns each: A00 | A01 | A11 at K = 256, A at K = 128), then Bm
  constexpr int NBLK = MH == 2 ? 3 : 1;
  constexpr int kColB = NBLK * 128;
  constexpr int kTmemCols = kColB + MH * NB <= 256 ? 256 : 512;
  constexpr uint32_t kCH = 16u * kHalf;  // column-group stride of the 64-row half tiles
  constexpr uint32_t kTileBytes = kRows * K * 2;
  constexpr uint32_t kEB = kHalf * K * 2, kAPB = kHalf * K * 2, kOhB = kHalf * NB * 2;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sE0 = smem;                     // kStages x (64 x K)
  uint8_t* sAP0 = smem + kStages * kEB;    // kStages x (64 x K)
  uint8_t* sOh0 = sAP0 + kStages * kAPB;   // kStages x (64 x NB)
  __shared__ uint64_t bar_ld[kStages], bar_built[kStages], bar_mma[kStages];
  __shared__ uint32_t s_taddr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int group = blockIdx.x, ngroups = gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&bar_ld[i], 1);
      tc::mbar_init(&bar_built[i], 8);
      tc::mbar_init(&bar_mma[i], 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&s_taddr);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s_taddr;
  const int64_t ntiles = (a.npx + kRows - 1) / kRows;
  const int nmine = group < ntiles ? (int)((ntiles - 1 - group) / ngroups + 1) : 0;
  const int nh = 2 * nmine;  // half tiles of this CTA
  if (warp == 8) {
    // ---------------- producer: TMA loads + MMA issue (one lane)
    if (lane == 0 && nh > 0) {
      const uint32_t aAP0 = tc::smem_u32(sAP0), aOh0 = tc::smem_u32(sOh0), aE0 = tc::smem_u32(sE0);
      auto load = [&](int i) {  // DEC1 wrote each tile half-major: one contiguous copy per half tile
        const int s = i % kStages;
        const uint8_t* src = a.e_tiles + (size_t)(group + (int64_t)(i >> 1) * ngroups) * kTileBytes + (i & 1) * kEB;
        tc::mbar_expect_tx(&bar_ld[s], kEB);
        tc::bulk_g2s(sE0 + s * kEB, src, kEB, &bar_ld[s]);
      };
      for (int i = 0; i < kStages - 1 && i < nh; ++i) load(i);
      const uint32_t idA = tc::make_idesc_bf16(128, 128, 1, 1), idB = tc::make_idesc_bf16(128, NB, 1, 1);
      for (int it = 0; it < nh; ++it) {
        const int s = it % kStages;
        tc::mbar_wait(&bar_built[s], (it / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t aE = aE0 + s * kEB, aAP = aAP0 + s * kAPB, aOh = aOh0 + s * kOhB;
        // MN-major operands: 128 atoms = 16 column groups of the half tile
#pragma unroll
        for (int ks = 0; ks < kHalf / 16; ++ks) {
          const uint32_t acc = it > 0 || ks > 0;
          const uint64_t e0 = tc::make_sdesc(aE + ks * 2 * 128, 128, kCH);
          const uint64_t p0 = tc::make_sdesc(aAP + ks * 2 * 128, 128, kCH);
          const uint64_t oh = tc::make_sdesc(aOh + ks * 2 * 128, 128, kCH);
          tc::mma_bf16(tmem + 0, e0, p0, idA, acc);  // A00 (A at K = 128)
          tc::mma_bf16(tmem + kColB, e0, oh, idB, acc);  // Bm rows 0..127
          if constexpr (MH == 2) {
            const uint64_t e1 = tc::make_sdesc(aE + 16 * kCH + ks * 2 * 128, 128, kCH);
            const uint64_t p1 = tc::make_sdesc(aAP + 16 * kCH + ks * 2 * 128, 128, kCH);
            tc::mma_bf16(tmem + 128, e0, p1, idA, acc);       // A01
            tc::mma_bf16(tmem + 256, e1, p1, idA, acc);       // A11
            tc::mma_bf16(tmem + kColB + NB, e1, oh, idB, acc);  // Bm rows 128..255
          }
        }
        tc::mma_commit(&bar_mma[s]);
        // refill: half tile it + kStages - 1 into the stage half tile it - 1 used
        const int nx = it + kStages - 1;
        if (nx < nh) {
          if (it >= 1) tc::mbar_wait(&bar_mma[(it - 1) % kStages], ((it - 1) / kStages) & 1);
          load(nx);
        }
      }
    }
  } else {
    // ---------------- builders: (alpha / sum^2) e over all K columns and the beta / sum one-hot.
    // Thread = (row of the half tile, quarter of the columns); the row statistics of half tile
    // it + 1 are fetched while half tile it is built.
    const int row = tid & (kHalf - 1), q = tid / kHalf;
    auto fetch = [&](int i, float4& st, int32_t& asg) {  // asg = -2 marks a row past npx
      const int64_t r = (group + (int64_t)(i >> 1) * ngroups) * kRows + (i & 1) * kHalf + row;
      st = make_float4(0.f, 0.f, 0.f, 0.f);
      asg = -2;
      if (r < a.npx) {
        st = a.row_stats[r];
        asg = a.assign[r];
      }
    };
    float4 st_n;
    int32_t asg_n;
    if (nh > 0) fetch(0, st_n, asg_n);
    for (int it = 0; it < nh; ++it) {
      const int s = it % kStages;
      const float4 st = st_n;
      const int32_t asg = asg_n;
      if (it + 1 < nh) fetch(it + 1, st_n, asg_n);
      const float wa = st.z * st.y * st.y;  // alpha / sum^2
      const float wb = st.w * st.y;         // beta / sum
      tc::mbar_wait(&bar_ld[s], (it / kStages) & 1);
      const uint8_t* E = sE0 + s * kEB;
      uint8_t* AP = sAP0 + s * kAPB;
#pragma unroll
      for (int c = q * (K / 4); c < (q + 1) * (K / 4); c += 8) {
        float v[8];
        tc::ld_row8(E, row, c, kCH, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = asg != -2 ? v[j] * wa : 0.f;
        tc::st_row8(AP, row, c, kCH, v);
      }
      uint8_t* Oh = sOh0 + s * kOhB;
#pragma unroll
      for (int c = q * (NB / 4); c < (q + 1) * (NB / 4); c += 8) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = (asg == c + j) ? wb : 0.f;
        tc::st_row8(Oh, row, c, kCH, v);
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar_built[s]);
    }
    // all MMAs complete once the last half tile's commit arrives
    if (nh > 0) {
      tc::mbar_wait(&bar_mma[(nh - 1) % kStages], ((nh - 1) / kStages) & 1);
      tc::tc_fence_after();
    }
    // drain into the partial layout [group][column half][row][column within the half] (K x K/2
    // per half): TMEM lane group g holds rows 32g + lane of every block; the two warps of a lane
    // group take alternate 16-column chunks
    constexpr int NHALF = K / 2;
    const int g = warp & 3, h = warp >> 2;
    const int trow = 32 * g + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * g) << 16);
    auto put = [&](int i, int col, const float* v) {  // 16 values of A[i][col .. col+15]
      const int half = col / NHALF, jj = col % NHALF;
      float* dst = a.a_part + (((size_t)group * 2 + half) * K + i) * NHALF + jj;
      for (int u = 0; u < 16; u += 4) {
        float4 o = make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
        if (a.accum) {
          const float4 p = *reinterpret_cast<const float4*>(dst + u);
          o.x += p.x, o.y += p.y, o.z += p.z, o.w += p.w;
        }
        *reinterpret_cast<float4*>(dst + u) = o;
      }
    };
    for (int blk = 0; blk < NBLK; ++blk) {
      // blk 0: A00 (rows 0.., cols 0..); 1: A01 (rows 0.., cols 128..); 2: A11 (rows 128.., cols 128..)
      const int r0 = blk == 2 ? 128 : 0, cb = blk == 0 ? 0 : 128;
      for (int c = 16 * h; c < 128; c += 32) {
        float v[16];
        if (nh == 0) {
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        } else {
          tc::tmem_ld16(tl + blk * 128 + c, v);
        }
        put(r0 + trow, cb + c, v);
        if (blk == 1) {  // A10 = A01^T: rows 128 + c + u, column trow (lanes: consecutive columns)
          for (int u = 0; u < 16; ++u) {
            const int i = 128 + c + u;
            float* dst = a.a_part + (((size_t)group * 2 + 0) * K + i) * NHALF + trow;
            *dst = a.accum ? *dst + v[u] : v[u];
          }
        }
      }
    }
    for (int mh = 0; mh < MH; ++mh) {
      float* db = a.bm_part + ((size_t)group * K + mh * 128 + trow) * NB;
      for (int c = 16 * h; c < NB; c += 32) {
        float v[16];
        if (nh == 0) {
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        } else {
          tc::tmem_ld16(tl + kColB + mh * NB + c, v);
        }
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(db + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<kTmemCols>(tmem);
}

// Sum the per-CTA partials: this frame's Bm^T (n_set x K, zeroed beforehand) from (groups x K x
// 64) after every frame (do_bm); once per step (do_ar) the step-summed partials of A (K x K)
// from (groups x 2 roles x K x K/2) and R^T (K x DS) -> R (DS x K) into the accumulators. Each thread owns 4 consecutive partial entries (float4 loads) and a
// 1/kRedSplit share of the groups; the shares meet in global atomics (distinct addresses).
// Block (0, 0) also folds the loss partials into the frame's slots.
// One warp folds DEC1's per-CTA loss partials (groups x 4 doubles: cos, l2, non-finite flag) into
// the frame's slots: lane-strided sums, then a fixed xor tree (the same order every run).
__device__ __forceinline__ void fold_loss_partials(const double* __restrict__ loss_part, int groups,
                                                   double* partials) {
  const int lane = threadIdx.x & 31;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int gi = lane; gi < groups; gi += 32) {
    s0 += loss_part[gi * 4 + 0];
    s1 += loss_part[gi * 4 + 1];
    s2 += loss_part[gi * 4 + 2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    partials[4] += s0;
    partials[5] += s1;
    partials[6] = fmax(partials[6], s2 > 0.0 ? 1.0 : 0.0);
  }
}

constexpr int kRedSplit = 4;
__global__ void __launch_bounds__(256) dec_reduce_kernel(const float* __restrict__ a_part,
                                                         const float* __restrict__ bm_part,
                                                         const float* __restrict__ r_part,
                                                         const double* loss_part, int K, int DS, int n_set,
                                                         int groups1, int groups2, float* A, float* bmt, float* R,
                                                         double* partials, int do_ar, int do_bm) {
  const int NH = K / 2;
  const int64_t qa = do_ar ? (int64_t)K * K / 4 : 0, qb = do_bm ? (int64_t)K * 64 / 4 : 0,
                qr = do_ar ? (int64_t)K * DS / 4 : 0;
  const int split = blockIdx.y;
  if (loss_part && blockIdx.x == 0 && split == 0 && threadIdx.x < 32) fold_loss_partials(loss_part, groups1, partials);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < qa + qb + qr;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float4* src;
    size_t stride;  // in float4
    int ng;
    if (q < qa) {  // partial layout [g][role][i][jj], 4 consecutive jj
      const int64_t e = q * 4;
      const int role = (int)(e / ((int64_t)K * NH)), rem = (int)(e % ((int64_t)K * NH));
      src = reinterpret_cast<const float4*>(a_part) + (((size_t)role * K * NH) + rem) / 4;
      stride = (size_t)2 * K * NH / 4;
      ng = groups2;
    } else if (q < qa + qb) {  // [g][k][64]
      src = reinterpret_cast<const float4*>(bm_part) + (q - qa);
      stride = (size_t)K * 64 / 4;
      ng = groups2;
    } else {  // [g][k][DS]
      src = reinterpret_cast<const float4*>(r_part) + (q - qa - qb);
      stride = (size_t)K * DS / 4;
      ng = groups1;
    }
    const int per = (ng + (int)gridDim.y - 1) / (int)gridDim.y, g0 = split * per, g1 = min(ng, g0 + per);
    float4 acc[8];  // 8 independent 16-byte loads in flight per thread (the slots stream from HBM)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    int gi = g0;
    for (; gi + 8 <= g1; gi += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 v = __ldg(src + (size_t)(gi + u) * stride);
        acc[u].x += v.x; acc[u].y += v.y; acc[u].z += v.z; acc[u].w += v.w;
      }
    }
    for (; gi < g1; ++gi) {
      const float4 v = __ldg(src + (size_t)gi * stride);
      acc[0].x += v.x; acc[0].y += v.y; acc[0].z += v.z; acc[0].w += v.w;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc[u].x += acc[u + 4].x; acc[u].y += acc[u + 4].y; acc[u].z += acc[u + 4].z; acc[u].w += acc[u + 4].w;
    }
    const float4 t = make_float4((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x),
                                 (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y),
                                 (acc[0].z + acc[1].z) + (acc[2].z + acc[3].z),
                                 (acc[0].w + acc[1].w) + (acc[2].w + acc[3].w));
    const float tv[4] = {t.x, t.y, t.z, t.w};
    if (q < qa) {
      const int64_t e = q * 4;
      const int role = (int)(e / ((int64_t)K * NH)), rem = (int)(e % ((int64_t)K * NH));
      const int i = rem / NH, jj = rem % NH;
#pragma unroll
      for (int u = 0; u < 4; ++u) atomicAdd(&A[(size_t)i * K + role * NH + jj + u], tv[u]);
    } else if (q < qa + qb) {
      const int64_t e = (q - qa) * 4;
      const int k = (int)(e / 64), s0 = (int)(e % 64);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (s0 + u < n_set) atomicAdd(&bmt[(size_t)(s0 + u) * K + k], tv[u]);
    } else {
      const int64_t e = (q - qa - qb) * 4;
      const int k = (int)(e / DS), s0 = (int)(e % DS);
#pragma unroll
      for (int u = 0; u < 4; ++u) atomicAdd(&R[(size_t)(s0 + u) * K + k], tv[u]);
    }
  }
}

// This frame's d_atoms += Bm E from DEC2's per-group Bm partials (groups x K x 64), without
// materialising Bm^T. CTA = one key (K CTAs), 256 threads: phase 1 sums the partials of each
// (key, set) pair with four threads (a quarter of the groups each, 8 independent loads in
// flight); phase 2 forms the output row with two threads per float4 column (half the sets each).
__global__ void __launch_bounds__(256) bm_embed_fused_kernel(const float* __restrict__ bm_part, int groups, int K,
                                                             const float* __restrict__ feats, int n_set, int df,
                                                             float* __restrict__ d_atoms,
                                                             const double* __restrict__ loss_part, int loss_groups,
                                                             double* partials) {
  __shared__ float s_q[4][64];
  __shared__ float s_bm[64];
  __shared__ float4 s_out[128];
  const int tid = threadIdx.x, k0 = blockIdx.x;
  if (loss_part && blockIdx.x == 0 && tid < 32) fold_loss_partials(loss_part, loss_groups, partials);
  {
    const int sidx = tid & 63, qq = tid >> 6;  // set, quarter of the groups
    const float* src = bm_part + (size_t)k0 * 64 + sidx;
    const size_t gs = (size_t)K * 64;
    const int per = (groups + 3) / 4, g0 = min(groups, qq * per), g1 = min(groups, g0 + per);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int g = g0;
    for (; g + 8 <= g1; g += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += __ldg(src + (size_t)(g + u) * gs);
    }
    for (; g < g1; ++g) acc[0] += __ldg(src + (size_t)g * gs);
    s_q[qq][sidx] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
  __syncthreads();
  if (tid < 64) s_bm[tid] = (s_q[0][tid] + s_q[1][tid]) + (s_q[2][tid] + s_q[3][tid]);
  __syncthreads();
  const int hs = tid >> 7, s0 = hs ? n_set / 2 : 0, s1 = hs ? n_set : n_set / 2;
  for (int cb = 0; cb < df / 4; cb += 128) {
    const int c4 = cb + (tid & 127);
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c4 < df / 4) {
#pragma unroll 8
      for (int sidx = s0; sidx < s1; ++sidx) {
        const float4 e = __ldg(reinterpret_cast<const float4*>(feats + (size_t)sidx * df) + c4);
        const float b0 = s_bm[sidx];
        a0.x = fmaf(b0, e.x, a0.x), a0.y = fmaf(b0, e.y, a0.y), a0.z = fmaf(b0, e.z, a0.z), a0.w = fmaf(b0, e.w, a0.w);
      }
    }
    if (hs == 1) s_out[tid & 127] = a0;
    __syncthreads();
    if (hs == 0 && c4 < df / 4) {
      const float4 p0 = s_out[tid];
      float4* d0 = reinterpret_cast<float4*>(d_atoms + (size_t)k0 * df) + c4;
      float4 o = *d0;
      o.x += a0.x + p0.x, o.y += a0.y + p0.y, o.z += a0.z + p0.z, o.w += a0.w + p0.w;
      *d0 = o;
    }
    __syncthreads();
  }
}

template <int K, int DS>
void launch_tc(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment, int64_t npx,
               const float* feats, int64_t n_set, const int64_t* nsup, float temperature, float lambda_cos, float lambda_l2,
               float scale, bool want_grad, float* d_query, double* partials) {
  const int g1 = 148;
  const int g2 = kDec2Groups;  // one CTA per group
  const int accum = want_grad && w.tc_frames > 0 ? 1 : 0;
  Dec1Args d1{w.e_tiles, query, assignment, w.kd, w.mm, w.gt, w.nv, npx, 1.f / temperature, lambda_cos, lambda_l2,
              scale, nsup, d_query, reinterpret_cast<float4*>(w.row_stats),
              w.r_part, w.loss_part, want_grad ? 1 : 0, accum, reinterpret_cast<float2*>(w.row_nd), w.tc_img};
  const size_t sm1 = (size_t)kRows * DS * 2 + (size_t)K * DS * 2 + (size_t)kRows * K * 2 + (size_t)K * K * 2 +
                     16 * 128 * 4;
  static bool attr1 = false;
  if (!attr1) {
    cudaFuncSetAttribute(dec1_kernel<K, DS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    attr1 = true;
  }
  dec1_kernel<K, DS><<<g1, 512, sm1, st>>>(d1);
  count_launch();
  if (w.ev_dq) cudaEventRecord(w.ev_dq, st);  // the render backward needs only d_query
  if (!want_grad) {
    dec_reduce_kernel<<<dim3(1, 1), 32, 0, st>>>(nullptr, nullptr, nullptr, w.loss_part, 0, 0, 0, g1, 0, nullptr,
                                                 nullptr, nullptr, partials, 0, 0);
    count_launch();
    return;
  }
  // A partials: one slot per frame of the step (plain stores; decoder_finish_tc sums the slots),
  // the last slot accumulating when a step has more frames than slots
  const int slot = std::min(w.tc_frames, kDec2Slots - 1);
  const int accum2 = want_grad && w.tc_frames >= kDec2Slots ? 1 : 0;
  Dec2Args d2{w.e_tiles, assignment, reinterpret_cast<const float4*>(w.row_stats), npx,
              w.a_part + (size_t)slot * kDec2Groups * K * K, w.bm_part, accum2};
  const size_t sm2 = dec2_smem<K>();
  static bool attr2 = false;
  if (!attr2) {
    cudaFuncSetAttribute(dec2_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    attr2 = true;
  }
  dec2_kernel<K><<<g2, 288, sm2, st>>>(d2);
  count_launch();
  // this frame's loss partials are folded by the Bm embed that follows (decoder_frame_tc)
  w.tc_frames += 1;
}

}  // namespace

__global__ void tc_image_kernel(uint8_t* img, const float* __restrict__ kd, const float* __restrict__ mm, int K,
                                int DS) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
  tc::load_tile_bf16(img, kd, K, DS, K, tid, nthr);
  tc::load_tile_bf16(img + (size_t)K * DS * 2, mm, K, K, K, tid, nthr);
}

void decoder_tc_images(cudaStream_t st, DecoderWork& w) {
  if (!w.tc_img) return;
  tc_image_kernel<<<32, 256, 0, st>>>(w.tc_img, w.kd, w.mm, (int)w.k, w.ds);
  count_launch();
}

bool decoder_tc_supported(int64_t k, int ds, int64_t n_set) {
  return (k == 128 || k == 256) && ds == 32 && n_set <= 64;
}

size_t decoder_tc_scratch_floats(int64_t k, int ds, int64_t npx) {
  // row_stats (4/row) + r_part + a_part + bm_part + loss_part (as floats x2)
  return (size_t)npx * 4 + 148 * (size_t)k * ds + kDec2Slots * kDec2Groups * (size_t)k * k +
         kDec2Groups * (size_t)k * 64 + 148 * 4 * 2;
}

void decoder_frame_tc(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment, int64_t npx,
                      const float* feats, int64_t n_set, const int64_t* nsup, const float* atoms, const float* proj,
                      float temperature, float lambda_cos, float lambda_l2, float scale, bool want_grad, float* d_query,
                      float* d_proj, float* d_atoms, double* partials) {
  const int64_t k = w.k;
  const int ds = w.ds, df = w.df;
  // per-frame target scores G^T = E D^T and norms (tiny SIMT GEMMs)
  decoder_targets(st, feats, n_set, atoms, k, df, w.gt, w.nv);
  if (k == 256)
    launch_tc<256, 32>(st, w, query, assignment, npx, feats, n_set, nsup, temperature, lambda_cos, lambda_l2, scale,
                       want_grad, d_query, partials);
  else
    launch_tc<128, 32>(st, w, query, assignment, npx, feats, n_set, nsup, temperature, lambda_cos, lambda_l2, scale,
                       want_grad, d_query, partials);
  if (!want_grad) return;
  // d_atoms += Bm E for this frame's embedding table; A and R accumulate over the step's frames
  // and enter once in decoder_finish_tc (they multiply the same D, W in every frame)
  if (df % 4 == 0 && (reinterpret_cast<uintptr_t>(feats) & 15) == 0 && (reinterpret_cast<uintptr_t>(d_atoms) & 15) == 0) {
    bm_embed_fused_kernel<<<(unsigned)k, 256, 0, st>>>(w.bm_part, kDec2Groups, (int)k, feats, (int)n_set, df,
                                                           d_atoms, w.loss_part, 148, partials);
    count_launch();
  } else {
    cudaMemsetAsync(w.bm, 0, sizeof(float) * n_set * k, st);
    const int64_t quads = k * 64 / 4;
    dec_reduce_kernel<<<dim3((unsigned)((quads + 255) / 256), deterministic() ? 1 : kRedSplit), 256, 0, st>>>(
        nullptr, w.bm_part, nullptr, w.loss_part, (int)k, ds, (int)n_set, 148, kDec2Groups, nullptr, w.bm, nullptr,
        partials, 0, 1);
    count_launch();
    decoder_bm_embed(st, w.bm, feats, n_set, k, df, d_atoms);
  }
  w.tc_pending = true;
  (void)d_proj;
  (void)proj;
}

void decoder_finish_tc(cudaStream_t st, DecoderWork& w, const float* atoms, const float* proj, float* d_proj,
                       float* d_atoms) {
  if (!w.tc_pending) return;
  const int64_t k = w.k;
  const int ds = w.ds, df = w.df;
  if (w.tc_frames > 0) {  // the fused frames' A partials (one slot per frame) and step-summed R partials
    const int64_t quads = (k * k + k * ds) / 4;
    const int ngroups_a = kDec2Groups * std::min(w.tc_frames, kDec2Slots);
    dec_reduce_kernel<<<dim3((unsigned)((quads + 255) / 256), deterministic() ? 1 : 2 * kRedSplit), 256, 0, st>>>(
        w.a_part, nullptr, w.r_part, nullptr, (int)k, ds, 0, 148, ngroups_a, w.a_acc, nullptr, w.r_acc, nullptr, 1, 0);
    count_launch();
    w.tc_frames = 0;
  }
  // d_atoms += A D + R^T W ;  d_proj += R D   (R stored ds x K)
  sgemm(st, false, false, k, df, k, 1.f, w.a_acc, k, atoms, df, 1.f, d_atoms, df);
  sgemm(st, true, false, k, df, ds, 1.f, w.r_acc, k, proj, df, 1.f, d_atoms, df);
  sgemm(st, false, false, ds, df, k, 1.f, w.r_acc, k, atoms, df, 1.f, d_proj, df);
  w.tc_pending = false;
}

// Parity export: P[r][c] = e[r][c] * (1/sum_r), e read from the bf16 core-matrix tiles the
// kernels wrote for the last frame (DEC1 with gradients, DL1 always), 1/sum from row_stats.y.
__global__ void export_attention_kernel(const uint8_t* __restrict__ e_tiles, const float4* __restrict__ rs,
                                        int64_t npx, int K, int half_major, float* __restrict__ p) {
  const int64_t chunks = npx * (K / 8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (K / 8);
    const int c0 = (int)(i % (K / 8)) * 8;
    const int64_t tile = r / kRows;
    const int rr = (int)(r % kRows);
    float v[8];
    if (half_major)  // DEC1's export: two 64-row halves, each contiguous
      tc::ld_row8(e_tiles + (size_t)tile * kRows * K * 2 + (size_t)(rr / kHalf) * kHalf * K * 2, rr % kHalf, c0,
                  16u * kHalf, v);
    else
      tc::ld_row8(e_tiles + (size_t)tile * kRows * K * 2, rr, c0, 16u * kRows, v);
    const float inv = rs[r].y;
    float4* dst = reinterpret_cast<float4*>(p + r * K + c0);
    dst[0] = make_float4(v[0] * inv, v[1] * inv, v[2] * inv, v[3] * inv);
    dst[1] = make_float4(v[4] * inv, v[5] * inv, v[6] * inv, v[7] * inv);
  }
}

void decoder_export_attention(cudaStream_t st, const DecoderWork& w, int64_t npx, float* p_out) {
  const int64_t chunks = npx * (w.k / 8);
  export_attention_kernel<<<(unsigned)std::min<int64_t>((chunks + 255) / 256, 148 * 16), 256, 0, st>>>(
      w.e_tiles, reinterpret_cast<const float4*>(w.row_stats), npx, (int)w.k, w.last_path == 2 ? 1 : 0, p_out);
  count_launch();
}

}  // namespace lm
