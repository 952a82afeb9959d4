// decoder_dl.cu — large-dictionary decoder on tcgen05 (bf16 operands, fp32 TMEM accumulators)
// for K in {256, 512, 768, 1024}, d_s in {32, 64}, n_set <= 256 (BASELINE config 4: K = 1024,
// d_s = 64, d_f = 1024, 128 target cells).
//
// Reference semantics: reconstruct (proj/src/dictionary.cpp:25-53), feature_loss
// (proj/src/losses.cpp:257-294), reconstruct_backward (dictionary.cpp:55-83), assembled by
// total_objective (proj/src/objective.cpp:100-185). Same factored algebra as decoder.cu and
// decoder_tc.cu (S = Q Kd^T, P = softmax(S / tau), t = P M with M = D D^T, G = E D^T):
//
//   nu^2 = P.t,  dot = P.G[a],  dS = P * (alpha t + beta G[a] - (alpha nu^2 + beta dot)) / tau,
//   dQ = dS Kd,  R^T = dS^T Q,  A = P^T diag(alpha) P,  Bm = P^T Ohb.
//
// The fused DEC1/DEC2 pair of decoder_tc.cu keeps a whole 128 x K row tile (and M) on chip; at
// K = 1024 neither the S tile (1024 TMEM columns) nor M (2 MB) fits, so this path stages the
// K-wide row quantities through HBM in the same core-matrix tile layout, every GEMM on tcgen05:
//
//   DL1 dl_softmax_kernel  S = Q Kd^T in 256-column TMEM chunks (double-buffered), two passes:
//                          row max, then e = exp(S - max) -> bf16 e tiles + row sum + e.G[a].
//   DL2 dl_t_kernel        T = e M (128 x 256 units, 4-stage TMA-bulk pipeline of e / M blocks,
//                          double-buffered TMEM accumulator), epilogue stores T (fp16) and the
//                          per-unit partial of e.T (-> nu^2).
//   DL3 dl_back_kernel     two roles per row tile (key halves): per-row alpha/beta/loss, dS
//                          (bf16, smem) -> dQ += dS Kd and R^T += dS^T Q on tcgen05; writes the
//                          scaled B operand [alpha/sum^2 e | beta/sum onehot(a)] for DL4.
//   DL4 dl_gram_kernel     [A | Bm] = e^T [alpha e | Ohb] over all row tiles (split in row
//                          ranges), 256 x 256 upper-triangle units of the symmetric A only.
//   DL5 dl_reduce_kernel   deterministic sum of the per-CTA partials into the step accumulators.
//
// Tile layout in HBM and shared memory: the no-swizzle core-matrix layout of tc_common.cuh with
// 128 rows per tile, row-group stride 128 B and column-group stride 2048 B, so a 64-column
// block of a tile is 16 contiguous KB (one 1-D bulk copy) and the same bytes serve as a K-major
// operand (e as A of T = e M) and as an MN-major operand (e^T in the gram).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace lm {

namespace {

constexpr int kRows = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr uint32_t kCS = 2048;  // column-group stride of a 128-row tile

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void unpack_h8(uint4 u, float* v) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

// ------------------------------------------------------------------------------------------ DL1
struct Dl1Args {
  uint8_t* e_tiles;       // ntiles x (128 x K bf16)
  const float* query;     // npx x DS
  const int32_t* assign;  // npx
  const float* kd;        // K x DS fp32
  const float* gt;        // n_set x K fp32
  int64_t npx;
  int K;
  float inv_temp;
  float4* rs;             // npx: (max S, 1/sum, dot = P.G[a], 0)
  float* d_query;         // zeroed here (DL3 accumulates the two key halves)
  int zero_dq;
};

template <int DS>
__global__ void __launch_bounds__(512, 1) dl_softmax_kernel(Dl1Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int K = a.K;
  uint8_t* sKd = smem;               // K x DS (rows = K)
  uint8_t* sQ = smem + K * DS * 2;   // 128 x DS
  __shared__ uint64_t bar[2];
  __shared__ uint32_t s_taddr;
  __shared__ float s_red[3][4][kRows];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp & 3, h = warp >> 2;  // TMEM lane group, 64-column quarter of a chunk
  const int row = 32 * g + lane;
  tc::load_tile_bf16(sKd, a.kd, K, DS, K, tid, 512);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&s_taddr);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s_taddr;
  const uint32_t tl = tmem + ((uint32_t)(32 * g) << 16);
  uint32_t ph[2] = {0, 0};
  const uint32_t idesc = tc::make_idesc_bf16(128, 256, 0, 0);
  const uint32_t aQ = tc::smem_u32(sQ), aKd = tc::smem_u32(sKd);
  const uint32_t kdCS = 16u * K;
  const float cl = kLog2e * a.inv_temp;
  const int nch = K / 256;
  const int64_t ntiles = (a.npx + kRows - 1) / kRows;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kRows;
    const int valid = (int)(a.npx - r0 < kRows ? a.npx - r0 : kRows);
    tc::load_tile_bf16(sQ, a.query + r0 * DS, kRows, DS, valid, tid, 512);
    if (a.zero_dq) {
      float4* dq = reinterpret_cast<float4*>(a.d_query + r0 * DS);
      for (int i = tid; i < valid * DS / 4; i += 512) dq[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int32_t asg = row < valid && a.assign ? a.assign[r0 + row] : -1;  // no assignment: reconstruct only
    const float* gp = a.gt + (int64_t)(asg < 0 ? 0 : asg) * K;
    uint8_t* et = a.e_tiles + (size_t)tile * kRows * K * 2;
    tc::fence_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    auto issue = [&](int c, int buf) {
      tc::tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < DS / 16; ++ks)
        tc::mma_bf16(tmem + buf * 256, tc::make_sdesc(aQ + ks * 2 * kCS, kCS, 128),
                     tc::make_sdesc(aKd + c * 4096 + ks * 2 * kdCS, kdCS, 128), idesc, ks > 0);
      tc::mma_commit(&bar[buf]);
    };
    if (tid == 0) issue(0, 0);
    float mx = -INFINITY, ml = 0.f, sum = 0.f, dot = 0.f;
    for (int j = 0; j < 2 * nch; ++j) {
      const int buf = j & 1;
      if (tid == 0 && j + 1 < 2 * nch) issue((j + 1) % nch, buf ^ 1);
      tc::mbar_wait(&bar[buf], ph[buf]);
      ph[buf] ^= 1;
      tc::tc_fence_after();
      const int cb = (j % nch) * 256 + h * 64;  // key index of this thread's first column
      const uint32_t tcol = tl + buf * 256 + h * 64;
      if (j < nch) {
#pragma unroll 1
        for (int i = 0; i < 64; i += 32) {
          float v[32];
          tc::tmem_ld32(tcol + i, v);
#pragma unroll
          for (int k = 0; k < 32; ++k) mx = fmaxf(mx, v[k]);
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < 64; i += 32) {
          float v[32];
          tc::tmem_ld32(tcol + i, v);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = cb + i + 8 * q;
            uint4 u;
            u.x = tc::pack_bf16(tc::ex2(fmaf(v[8 * q + 0], cl, -ml)), tc::ex2(fmaf(v[8 * q + 1], cl, -ml)));
            u.y = tc::pack_bf16(tc::ex2(fmaf(v[8 * q + 2], cl, -ml)), tc::ex2(fmaf(v[8 * q + 3], cl, -ml)));
            u.z = tc::pack_bf16(tc::ex2(fmaf(v[8 * q + 4], cl, -ml)), tc::ex2(fmaf(v[8 * q + 5], cl, -ml)));
            u.w = tc::pack_bf16(tc::ex2(fmaf(v[8 * q + 6], cl, -ml)), tc::ex2(fmaf(v[8 * q + 7], cl, -ml)));
            *reinterpret_cast<uint4*>(et + tc::core_off(row, c, 128u, kCS)) = u;
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
            float e[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              e[2 * k] = __uint_as_float(w4[k] << 16);
              e[2 * k + 1] = __uint_as_float(w4[k] & 0xffff0000u);
              sum += e[2 * k] + e[2 * k + 1];
            }
            if (asg >= 0) {
              const float4 g0 = __ldg(reinterpret_cast<const float4*>(gp + c));
              const float4 g1 = __ldg(reinterpret_cast<const float4*>(gp + c + 4));
              dot = fmaf(e[0], g0.x, dot);
              dot = fmaf(e[1], g0.y, dot);
              dot = fmaf(e[2], g0.z, dot);
              dot = fmaf(e[3], g0.w, dot);
              dot = fmaf(e[4], g1.x, dot);
              dot = fmaf(e[5], g1.y, dot);
              dot = fmaf(e[6], g1.z, dot);
              dot = fmaf(e[7], g1.w, dot);
            }
          }
        }
      }
      tc::tc_fence_before();
      if (j == nch - 1) {
        s_red[0][h][row] = mx;
        __syncthreads();
        mx = fmaxf(fmaxf(s_red[0][0][row], s_red[0][1][row]), fmaxf(s_red[0][2][row], s_red[0][3][row]));
        ml = mx * cl;
      } else {
        __syncthreads();
      }
    }
    s_red[1][h][row] = sum;
    s_red[2][h][row] = dot;
    __syncthreads();
    if (h == 0 && row < valid) {
      const float inv = 1.f / ((s_red[1][0][row] + s_red[1][1][row]) + (s_red[1][2][row] + s_red[1][3][row]));
      const float dsum = (s_red[2][0][row] + s_red[2][1][row]) + (s_red[2][2][row] + s_red[2][3][row]);
      a.rs[r0 + row] = make_float4(mx, inv, dsum * inv, 0.f);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem);
}

// ------------------------------------------------------------------------------------------ DL2
struct Dl2Args {
  const uint8_t* e_tiles;  // ntiles x (128 x K bf16)
  const uint8_t* mt;       // (K/256) x (K/64) blocks of 256 x 64 bf16 (rows = 256): M[n][k]
  uint4* t_tiles;          // ntiles x [K/8][128] x 8 fp16: T = e M (|T| <= sum e <= K; fp16 keeps
                           // 11 bits, 4x finer than the bf16 e it multiplies)
  float* nu_part;          // (K/256) x ntiles*128: sum over the unit's columns of e * T
  int64_t npx;
  int K;
};

constexpr int kT_Stages = 4;
constexpr uint32_t kT_A = 16384, kT_B = 32768;

__global__ void __launch_bounds__(192, 1) dl_t_kernel(Dl2Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kT_Stages], empty[kT_Stages], accf[2], acce[2];
  __shared__ uint32_t s_taddr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.K, KB = K / 64, NC = K / 256;
  const int64_t ntiles = (a.npx + kRows - 1) / kRows, units = ntiles * NC;
  auto sA = [&](int s) { return smem + s * (kT_A + kT_B); };
  auto sB = [&](int s) { return smem + s * (kT_A + kT_B) + kT_A; };
  if (tid == 0) {
    for (int i = 0; i < kT_Stages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&accf[i], 1);
      tc::mbar_init(&acce[i], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&s_taddr);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s_taddr;
  if (warp == 4) {
    if (lane == 0) {  // producer: TMA bulk loads of the e block and the M block of each k-step
      int st = 0;
      uint32_t ph = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t t = u / NC;
        const int nc = (int)(u % NC);
        const uint8_t* ea = a.e_tiles + (size_t)t * kRows * K * 2;
        const uint8_t* mb = a.mt + (size_t)nc * KB * kT_B;
        for (int ks = 0; ks < KB; ++ks) {
          tc::mbar_wait(&empty[st], ph ^ 1);
          tc::mbar_expect_tx(&full[st], kT_A + kT_B);
          tc::bulk_g2s(sA(st), ea + (size_t)ks * kT_A, kT_A, &full[st]);
          tc::bulk_g2s(sB(st), mb + (size_t)ks * kT_B, kT_B, &full[st]);
          if (++st == kT_Stages) st = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = tc::make_idesc_bf16(128, 256, 0, 0);
      int st = 0;
      uint32_t ph = 0;
      int i = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int buf = i & 1;
        tc::mbar_wait(&acce[buf], ((i >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        for (int ks = 0; ks < KB; ++ks) {
          tc::mbar_wait(&full[st], ph);
          tc::tc_fence_after();
          const uint32_t aa = tc::smem_u32(sA(st)), ab = tc::smem_u32(sB(st));
#pragma unroll
          for (int k16 = 0; k16 < 4; ++k16)
            tc::mma_bf16(tmem + buf * 256, tc::make_sdesc(aa + k16 * 2 * kCS, kCS, 128),
                         tc::make_sdesc(ab + k16 * 2 * 4096, 4096, 128), idesc, (ks | k16) != 0);
          tc::mma_commit(&empty[st]);
          if (++st == kT_Stages) st = 0, ph ^= 1;
        }
        tc::mma_commit(&accf[buf]);
      }
    }
  } else {  // epilogue: warps 0-3, one pixel row per thread
    const int row = 32 * warp + lane;
    const int64_t ntr = ntiles * kRows;
    int i = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int buf = i & 1;
      const int64_t t = u / NC;
      const int nc = (int)(u % NC);
      const uint8_t* et = a.e_tiles + (size_t)t * kRows * K * 2;
      uint4* tt = a.t_tiles + (size_t)t * kRows * (K / 8);
      tc::mbar_wait(&accf[buf], (i >> 1) & 1);
      tc::tc_fence_after();
      float nu = 0.f;
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + buf * 256 + c, v);
        const int col = nc * 256 + c;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float e[8];
          tc::ld_row8(et, row, col + 8 * q, kCS, e);
#pragma unroll
          for (int k = 0; k < 8; ++k) nu = fmaf(e[k], v[8 * q + k], nu);
        }
#pragma unroll
        for (int f = 0; f < 4; ++f)
          tt[(size_t)(col / 8 + f) * kRows + row] =
              make_uint4(pack_h2(v[8 * f], v[8 * f + 1]), pack_h2(v[8 * f + 2], v[8 * f + 3]),
                         pack_h2(v[8 * f + 4], v[8 * f + 5]), pack_h2(v[8 * f + 6], v[8 * f + 7]));
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acce[buf]);
      a.nu_part[(size_t)nc * ntr + t * kRows + row] = nu;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem);
}

// M (K x K fp32, symmetric) -> the B-operand blocks of dl_t_kernel.
__global__ void dl_tile_m_kernel(const float* __restrict__ mm, int K, uint8_t* __restrict__ mt) {
  const int KB = K / 64;
  const int64_t chunks = (int64_t)K * K / 8;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < chunks; q += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(q / (K / 8)), k0 = (int)(q % (K / 8)) * 8;
    const int nc = n / 256, nl = n % 256, ks = k0 / 64, kl = k0 % 64;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = mm[(size_t)n * K + k0 + i];
    tc::st_row8(mt + ((size_t)nc * KB + ks) * kT_B, nl, kl, 4096u, v);
  }
}

// D (K x N fp32, row-major) -> B-operand blocks of dl_rec_kernel: block (nc, ks) holds
// B[n][k] = D[k][n] for n in [256 nc, 256 nc + 256), k in [64 ks, 64 ks + 64).
__global__ void dl_tile_dt_kernel(const float* __restrict__ d, int K, int N, uint8_t* __restrict__ bt) {
  const int KB = K / 64;
  const int64_t chunks = (int64_t)N * K / 8;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < chunks; q += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(q / (K / 8)), k0 = (int)(q % (K / 8)) * 8;
    const int nc = n / 256, nl = n % 256, ks = k0 / 64, kl = k0 % 64;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = d[(size_t)(k0 + i) * N + n];
    tc::st_row8(bt + ((size_t)nc * KB + ks) * kT_B, nl, kl, 4096u, v);
  }
}

// Standalone reconstruct (dictionary.cpp:25-53), F_hat = (e D) / sum: DL1's bf16 e tiles times
// D on tcgen05, 128 x 256 output units through the same 4-stage TMA pipeline and double-
// buffered TMEM accumulator as dl_t_kernel; the epilogue scales each row by 1/sum (DL1's row
// statistics) and writes fp32 rows.
struct DlRecArgs {
  const uint8_t* e_tiles;  // ntiles x (128 x K bf16)
  const uint8_t* bt;       // (N/256) x (K/64) blocks of 256 x 64 bf16: D^T
  const float4* rs;        // npx: (max S, 1/sum, -, -)
  float* out;              // npx x N
  int64_t npx;
  int K, N;
};

__global__ void __launch_bounds__(192, 1) dl_rec_kernel(DlRecArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kT_Stages], empty[kT_Stages], accf[2], acce[2];
  __shared__ uint32_t s_taddr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.K, KB = K / 64, NC = a.N / 256;
  const int64_t ntiles = (a.npx + kRows - 1) / kRows, units = ntiles * NC;
  auto sA = [&](int s) { return smem + s * (kT_A + kT_B); };
  auto sB = [&](int s) { return smem + s * (kT_A + kT_B) + kT_A; };
  if (tid == 0) {
    for (int i = 0; i < kT_Stages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&accf[i], 1);
      tc::mbar_init(&acce[i], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&s_taddr);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s_taddr;
  if (warp == 4) {
    if (lane == 0) {  // producer: the e block and the D^T block of each k-step
      int st = 0;
      uint32_t ph = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t t = u / NC;
        const int nc = (int)(u % NC);
        const uint8_t* ea = a.e_tiles + (size_t)t * kRows * K * 2;
        const uint8_t* bb = a.bt + (size_t)nc * KB * kT_B;
        for (int ks = 0; ks < KB; ++ks) {
          tc::mbar_wait(&empty[st], ph ^ 1);
          tc::mbar_expect_tx(&full[st], kT_A + kT_B);
          tc::bulk_g2s(sA(st), ea + (size_t)ks * kT_A, kT_A, &full[st]);
          tc::bulk_g2s(sB(st), bb + (size_t)ks * kT_B, kT_B, &full[st]);
          if (++st == kT_Stages) st = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = tc::make_idesc_bf16(128, 256, 0, 0);
      int st = 0;
      uint32_t ph = 0;
      int i = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int buf = i & 1;
        tc::mbar_wait(&acce[buf], ((i >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        for (int ks = 0; ks < KB; ++ks) {
          tc::mbar_wait(&full[st], ph);
          tc::tc_fence_after();
          const uint32_t aa = tc::smem_u32(sA(st)), ab = tc::smem_u32(sB(st));
#pragma unroll
          for (int k16 = 0; k16 < 4; ++k16)
            tc::mma_bf16(tmem + buf * 256, tc::make_sdesc(aa + k16 * 2 * kCS, kCS, 128),
                         tc::make_sdesc(ab + k16 * 2 * 4096, 4096, 128), idesc, (ks | k16) != 0);
          tc::mma_commit(&empty[st]);
          if (++st == kT_Stages) st = 0, ph ^= 1;
        }
        tc::mma_commit(&accf[buf]);
      }
    }
  } else {  // epilogue: warps 0-3, one row per thread
    const int row = 32 * warp + lane;
    int i = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int buf = i & 1;
      const int64_t t = u / NC;
      const int nc = (int)(u % NC);
      const int64_t r = t * kRows + row;
      const float inv = r < a.npx ? a.rs[r].y : 0.f;
      tc::mbar_wait(&accf[buf], (i >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + buf * 256 + c, v);
        if (r < a.npx) {
          float4* dst = reinterpret_cast<float4*>(a.out + r * a.N + nc * 256 + c);
#pragma unroll
          for (int f = 0; f < 8; ++f)
            dst[f] = make_float4(v[4 * f] * inv, v[4 * f + 1] * inv, v[4 * f + 2] * inv, v[4 * f + 3] * inv);
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acce[buf]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem);
}

// ------------------------------------------------------------------------------------------ DL3
struct Dl3Args {
  const uint8_t* e_tiles;
  const uint4* t_tiles;
  const float* nu_part;
  const float4* rs;
  const float* query;
  const int32_t* assign;
  const float* kd;
  const float* gt;
  const float* nv;
  uint8_t* ae_tiles;   // ntiles x (128 x (K + NB) bf16): [alpha/sum^2 e | beta/sum onehot(a)]
  float* d_query;      // npx x DS, zeroed by DL1; the two key halves add into it
  float* r_part;       // gridDim x (K/2) x DS: per-CTA R^T of the role's key half
  double* loss_part;   // gridDim x 4
  int64_t npx;
  int K, NB;
  float inv_temp, lambda_cos, lambda_l2, scale;
  const int64_t* nsup;  // supervised rows (device)
  int want_grad;
  float2* row_nd;       // optional parity export: per-row (nu^2, dot)
};

template <int N>
__device__ __forceinline__ void tmem_ldq(uint32_t taddr, float* v) {
  if constexpr (N == 8)
    tc::tmem_ld8(taddr, v);
  else
    tc::tmem_ld16(taddr, v);
}

template <int DS>
__global__ void __launch_bounds__(512, 1) dl_back_kernel(Dl3Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int K = a.K, KH = K / 2, PB = KH / 128, NTOT = K + a.NB;
  uint8_t* sKd = smem;                 // KH x DS (rows = KH): this role's key half of Kd
  uint8_t* sQ = sKd + KH * DS * 2;     // 128 x DS
  uint8_t* sD0 = sQ + kRows * DS * 2;  // 2 x (128 x 128): dS of one 128-key block
  __shared__ uint64_t bar[2];
  __shared__ uint32_t s_taddr;
  __shared__ double s_loss[16][3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp & 3, sub = warp >> 2;  // TMEM lane group, 32-key quarter of a block
  constexpr int DQ = DS / 4;                  // dQ / R^T columns per thread
  const int row = 32 * g + lane;
  const int role = blockIdx.x & 1, group = blockIdx.x >> 1, ngroups = gridDim.x >> 1;
  if (a.want_grad) tc::load_tile_bf16(sKd, a.kd + (size_t)role * KH * DS, KH, DS, KH, tid, 512);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&s_taddr);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s_taddr;
  const uint32_t tl = tmem + ((uint32_t)(32 * g) << 16);
  const uint32_t aKd = tc::smem_u32(sKd), aQ = tc::smem_u32(sQ);
  const uint32_t kdCS = 16u * KH;
  const uint32_t idq = tc::make_idesc_bf16(128, DS, 0, 1), ir = tc::make_idesc_bf16(128, DS, 1, 1);
  const int64_t ntiles = (a.npx + kRows - 1) / kRows, ntr = ntiles * kRows;
  const int NC = K / 256;
  const float inv_nsup = *a.nsup > 0 ? 1.f / (float)*a.nsup : 0.f;
  int pc = 0;
  bool first = true;
  double cos_acc = 0.0, l2_acc = 0.0, zflag = 0.0;
  for (int64_t tile = group; tile < ntiles; tile += ngroups) {
    const int64_t r0 = tile * kRows;
    const int valid = (int)(a.npx - r0 < kRows ? a.npx - r0 : kRows);
    if (a.want_grad) tc::load_tile_bf16(sQ, a.query + r0 * DS, kRows, DS, valid, tid, 512);
    // per-row loss quantities (objective.cpp:100-185 via the factored algebra)
    const int32_t asg = row < valid && a.assign ? a.assign[r0 + row] : -1;  // no assignment: reconstruct only
    const float4 st = row < valid ? a.rs[r0 + row] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float inv_sum = st.y, dot = st.z;
    float nu2 = 0.f;
    for (int nc = 0; nc < NC; ++nc) nu2 += a.nu_part[(size_t)nc * ntr + r0 + row];
    nu2 *= inv_sum * inv_sum;
    float al = 0.f, be = 0.f, cc = 0.f;
    if (asg >= 0) {
      const float eps = 1e-8f;
      const float nu = sqrtf(fmaxf(nu2, 0.f)), vn = a.nv[asg];
      const float nug = fmaxf(nu, eps), nvg = fmaxf(vn, eps);
      if (role == 0 && sub == 0) {
        if (nu < eps || vn < eps) zflag = 1.0;
        cos_acc += 1.0 - (double)(dot / (nug * nvg));
        l2_acc += (double)nu2 - 2.0 * (double)dot + (double)vn * (double)vn;
      }
      al = a.scale * (a.lambda_cos * dot / (nug * nug * nug * nvg) * inv_nsup + 2.f * a.lambda_l2 * inv_nsup);
      be = a.scale * (-a.lambda_cos / (nug * nvg) * inv_nsup - 2.f * a.lambda_l2 * inv_nsup);
      cc = al * nu2 + be * dot;
    }
    if (a.row_nd && role == 0 && sub == 0 && row < valid) a.row_nd[r0 + row] = make_float2(nu2, dot);
    if (!a.want_grad) continue;
    const float ps = inv_sum * a.inv_temp, al_t = al * inv_sum, wa = al * inv_sum * inv_sum, wb = be * inv_sum;
    const float* gp = a.gt + (int64_t)(asg < 0 ? 0 : asg) * K;
    const uint8_t* et = a.e_tiles + (size_t)tile * kRows * K * 2;
    const uint4* tt = a.t_tiles + (size_t)tile * kRows * (K / 8);
    uint8_t* aet = a.ae_tiles + (size_t)tile * kRows * NTOT * 2;
    if (role == 0) {  // one-hot block of the gram's B operand: beta / sum at column a
      for (int c8 = 8 * sub; c8 < a.NB; c8 += 32) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = (asg == c8 + j) ? wb : 0.f;
        tc::st_row8(aet, row, K + c8, kCS, v);
      }
    }
    for (int p = 0; p < PB; ++p, ++pc) {
      const int buf = pc & 1, use = pc >> 1;
      if (use >= 1) tc::mbar_wait(&bar[buf], (use - 1) & 1);  // MMAs that read sD[buf] are done
      uint8_t* sD = sD0 + buf * 32768;
      const int kb = role * KH + p * 128 + sub * 32;  // key of this thread's first column
      // all loads of the block first (the ae stores below could otherwise alias them)
      uint4 ev[4], th[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = kb + 8 * q;
        ev[q] = *reinterpret_cast<const uint4*>(et + tc::core_off(row, c, 128u, kCS));
        th[q] = tt[(size_t)(c / 8) * kRows + row];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = kb + 8 * q;
        const uint32_t w4[4] = {ev[q].x, ev[q].y, ev[q].z, ev[q].w};
        float e[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          e[2 * k] = __uint_as_float(w4[k] << 16);
          e[2 * k + 1] = __uint_as_float(w4[k] & 0xffff0000u);
        }
        const float4 g0 = __ldg(reinterpret_cast<const float4*>(gp + c));
        const float4 g1 = __ldg(reinterpret_cast<const float4*>(gp + c + 4));
        float tv[8];
        unpack_h8(th[q], tv);
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        float d[8], w8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          d[j] = e[j] * ps * fmaf(al_t, tv[j], fmaf(be, gv[j], -cc));
          w8[j] = e[j] * wa;
        }
        tc::st_row8(sD, row, sub * 32 + 8 * q, kCS, d);
        tc::st_row8(aet, row, c, kCS, w8);
      }
      tc::fence_async_smem();
      tc::tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::tc_fence_after();
        const uint32_t aD = tc::smem_u32(sD);
        // dQ (+)= dS[:, block] Kd[block, :]
#pragma unroll
        for (int k16 = 0; k16 < 8; ++k16)
          tc::mma_bf16(tmem, tc::make_sdesc(aD + k16 * 2 * kCS, kCS, 128),
                       tc::make_sdesc(aKd + (p * 16 + 2 * k16) * 128, 128, kdCS), idq, (p | k16) != 0);
        // R^T[block] += dS[:, block]^T Q
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc::mma_bf16(tmem + DS + p * DS, tc::make_sdesc(aD + ks * 2 * 128, 128, kCS),
                       tc::make_sdesc(aQ + ks * 2 * 128, 128, kCS), ir, (!first) || ks > 0);
        tc::mma_commit(&bar[buf]);
      }
    }
    first = false;
    {
      const int lp = pc - 1;
      tc::mbar_wait(&bar[lp & 1], (lp >> 1) & 1);  // every MMA of this tile has completed
      tc::tc_fence_after();
    }
    // dQ: this role's half of the key sum; exactly two adds onto the zeroed row (order-free)
    {
      float v[DQ];
      tmem_ldq<DQ>(tl + sub * DQ, v);
      if (row < valid) {
        float4* dst = reinterpret_cast<float4*>(a.d_query + (r0 + row) * DS + sub * DQ);
#pragma unroll
        for (int c = 0; c < DQ; c += 4) atomicAdd(dst + c / 4, make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]));
      }
    }
    tc::tc_fence_before();
    __syncthreads();
  }
  if (a.want_grad) {
    // R^T partial of this CTA: accumulator lane = key within the 128-key block
    for (int p = 0; p < PB; ++p) {
      float* dst = a.r_part + ((size_t)blockIdx.x * KH + p * 128 + row) * DS + sub * DQ;
      float v[DQ];
      if (first) {
#pragma unroll
        for (int i = 0; i < DQ; ++i) v[i] = 0.f;
      } else {
        tmem_ldq<DQ>(tl + DS + p * DS + sub * DQ, v);
      }
#pragma unroll
      for (int i = 0; i < DQ; i += 4)
        *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
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
    double c0s = 0, c1s = 0, c2s = 0;
    for (int w = 0; w < 16; ++w) c0s += s_loss[w][0], c1s += s_loss[w][1], c2s += s_loss[w][2];
    a.loss_part[blockIdx.x * 4 + 0] = c0s;
    a.loss_part[blockIdx.x * 4 + 1] = c1s;
    a.loss_part[blockIdx.x * 4 + 2] = c2s;
  }
  if (warp == 0) tc::tmem_free<512>(tmem);
}

// ------------------------------------------------------------------------------------------ DL4
struct Dl4Args {
  const uint8_t* e_tiles;   // ntiles x (128 x K)
  const uint8_t* ae_tiles;  // ntiles x (128 x NTOT)
  int nunits_a, splits_a, nunits_b, splits_b;
  int64_t ntiles;
  int K, NTOT;
  float* part;              // max(splits) x K x NTOT (only the units' blocks are written)
};

// One stage = 64 pixel rows (half a tile) of the A operand (256 keys) and of the B operand (w
// columns), copied as 1 KB column-group pieces into a 64-row core-matrix layout (column-group
// stride 1024 B). Output tile 256 keys x w in two TMEM accumulators: 128 KB of operands per
// 16.8 MFLOP, a third less L2 traffic per flop than 128-key units (the gram is L2-bound).
constexpr int kG_Stages = 3;
constexpr uint32_t kG_Half = 32768, kG_Stage = 2 * kG_Half, kG_CS = 1024;

// One 4-D TMA box: 64 rows (two 512-byte row pieces) x `box_cg` column groups of one tile.
__device__ __forceinline__ void tma_half(void* dst, const CUtensorMap* map, int piece, int cg, int64_t tile,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(piece), "r"(cg), "r"((int)tile), "r"(tc::smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(192, 1) dl_gram_kernel(const __grid_constant__ CUtensorMap tm_e,
                                                         const __grid_constant__ CUtensorMap tm_ae,
                                                         const __grid_constant__ CUtensorMap tm_oh, Dl4Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kG_Stages], empty[kG_Stages], accf;
  __shared__ uint32_t s_taddr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // CTA -> (unit, row split). A units: M pair mp (keys [256 mp, +256)) x N chunk nc in
  // [mp, K / 256) (upper triangle of the symmetric A); Bm units: every mp x the chunks >= K / 256.
  // A units take splits_a row ranges, the narrower Bm units splits_b.
  const int KC = a.K / 256, nchunks = (a.NTOT + 255) / 256, nbc = nchunks - KC;
  int cta = blockIdx.x, splits, split, mp = 0, nc;
  if (cta < a.nunits_a * a.splits_a) {
    splits = a.splits_a;
    split = cta / a.nunits_a;
    int rem = cta % a.nunits_a;
    while (rem >= KC - mp) rem -= KC - mp, ++mp;
    nc = mp + rem;
  } else {
    cta -= a.nunits_a * a.splits_a;
    splits = a.splits_b;
    split = cta / a.nunits_b;
    const int rem = cta % a.nunits_b;
    mp = rem / nbc;
    nc = KC + rem % nbc;
  }
  const int w = min(256, a.NTOT - nc * 256);
  const int64_t t0 = split * a.ntiles / splits, t1 = (split + 1) * a.ntiles / splits;
  if (tid == 0) {
    for (int i = 0; i < kG_Stages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(&accf, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&s_taddr);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s_taddr;
  if (warp == 4) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const CUtensorMap* mb = nc < KC ? &tm_ae : &tm_oh;
      for (int64_t t = t0; t < t1; ++t) {
        for (int hh = 0; hh < 2; ++hh) {
          uint8_t* dst = smem + st * kG_Stage;
          tc::mbar_wait(&empty[st], ph ^ 1);
          tc::mbar_expect_tx(&full[st], kG_Half + (uint32_t)w * 128u);
          tma_half(dst, &tm_e, 2 * hh, 32 * mp, t, &full[st]);
          tma_half(dst + kG_Half, mb, 2 * hh, 32 * nc, t, &full[st]);
          if (++st == kG_Stages) st = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && t1 > t0) {
      const uint32_t idesc = tc::make_idesc_bf16(128, w, 1, 1);
      int st = 0;
      uint32_t ph = 0;
      for (int64_t t = t0; t < t1; ++t) {
        for (int hh = 0; hh < 2; ++hh) {
          tc::mbar_wait(&full[st], ph);
          tc::tc_fence_after();
          const uint32_t as = tc::smem_u32(smem + st * kG_Stage), bs = as + kG_Half;
#pragma unroll
          for (int m2 = 0; m2 < 2; ++m2)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_bf16(tmem + m2 * 256, tc::make_sdesc(as + m2 * 16 * kG_CS + ks * 2 * 128, 128, kG_CS),
                           tc::make_sdesc(bs + ks * 2 * 128, 128, kG_CS), idesc, (t > t0) || hh > 0 || ks > 0);
          tc::mma_commit(&empty[st]);
          if (++st == kG_Stages) st = 0, ph ^= 1;
        }
      }
      tc::mma_commit(&accf);
    }
  } else {
    const int row = 32 * warp + lane;
    if (t1 > t0) {
      tc::mbar_wait(&accf, 0);
      tc::tc_fence_after();
    }
    for (int m2 = 0; m2 < 2; ++m2) {
      float* dst = a.part + ((size_t)split * a.K + mp * 256 + m2 * 128 + row) * a.NTOT + nc * 256;
      for (int c = 0; c < w; c += 16) {
        float v[16];
        if (t1 > t0) {
          tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + m2 * 256 + c, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(dst + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem);
}

// ------------------------------------------------------------------------------------------ DL5
// A (K x K) += sum over splits of the gram partial at (min(i,j), max(i,j)) (A is symmetric; only
// upper-triangle units were computed: (min, max) always lies in one); Bm^T (n_set x K) = the partial's columns K..K+n_set;
// R (DS x K) += sum over the DL3 CTAs of their R^T partials; loss partials folded once.
__global__ void __launch_bounds__(256) dl_reduce_kernel(const float* __restrict__ part, int splits_a, int splits_b,
                                                        int K, int NTOT,
                                                        int n_set, const float* __restrict__ r_part, int r_groups,
                                                        int DS, const double* __restrict__ loss_part, int loss_n,
                                                        float* A, float* bmt, float* R, double* partials) {
  if (blockIdx.x == 0 && threadIdx.x < 3) {
    const int which = threadIdx.x;
    double s = 0.0;
    for (int i = 0; i < loss_n; ++i) s += loss_part[i * 4 + which];
    if (which == 2)
      partials[6] = fmax(partials[6], s > 0.0 ? 1.0 : 0.0);
    else
      partials[4 + which] += s;
  }
  const int KH = K / 2;
  const int64_t na = (int64_t)K * K, nb = (int64_t)n_set * K, nr = (int64_t)DS * K;
  const size_t pstride = (size_t)K * NTOT;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < na + nb + nr;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (q < na) {
      const int i = (int)(q / K), j = (int)(q % K);
      const size_t o = (size_t)min(i, j) * NTOT + max(i, j);
      float s = 0.f;
      for (int sp = 0; sp < splits_a; ++sp) s += part[sp * pstride + o];
      A[q] += s;
    } else if (q < na + nb) {
      const int64_t e = q - na;
      const int s_ = (int)(e / K), k = (int)(e % K);
      const size_t o = (size_t)k * NTOT + K + s_;
      float s = 0.f;
      for (int sp = 0; sp < splits_b; ++sp) s += part[sp * pstride + o];
      bmt[e] = s;
    } else {
      const int64_t e = q - na - nb;
      const int d = (int)(e / K), k = (int)(e % K);
      const int role = k / KH, kl = k % KH;
      float s = 0.f;
      for (int gi = 0; gi < r_groups; ++gi) s += r_part[((size_t)(2 * gi + role) * KH + kl) * DS + d];
      R[e] += s;
    }
  }
}

constexpr int kBackGroups = 74;  // DL3 grid = 2 roles x 74 groups

int nb_for(int64_t n_set) { return (int)std::max<int64_t>(16, (n_set + 15) / 16 * 16); }

// Gram work split: na A units of 256 x 256 (upper triangle), nbu Bm units of 256 x (NB per
// chunk), sa / sb row splits of each, sa * na + sb * nbu <= 148 CTAs of about equal MMA work.
void dl_gram_plan(int K, int NB, int64_t ntiles, int& na, int& nbu, int& sa, int& sb) {
  const int KC = K / 256, nbc = (NB + 255) / 256;
  na = KC * (KC + 1) / 2;
  nbu = KC * nbc;
  const double wb = (double)std::min(NB, 256) / 256.0 * nbc;  // Bm work per unit, in A units
  const double per = (na + nbu * wb) / 148.0;                  // work per CTA
  sa = std::max(1, (int)(1.0 / per));
  sb = std::max(1, (int)(wb / per));
  while (na * sa + nbu * sb > 148 && (sa > 1 || sb > 1)) {
    if (sa >= sb && sa > 1) --sa; else --sb;
  }
  sa = (int)std::min<int64_t>(sa, ntiles);
  sb = (int)std::min<int64_t>(sb, ntiles);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return fn;
}

// A tile array [ntiles][ncg column groups][128 rows][8 bf16] viewed as the 4-D tensor
// (256 elements = 32 rows x 8, 4 row pieces, ncg, ntiles); a box of (256, 2, box_cg, 1) is 64
// rows x box_cg column groups, landing in shared memory as a 64-row core-matrix tile.
bool half_tile_map(CUtensorMap* m, const void* base, int ncg, int64_t ntiles, int box_cg) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {256, 4, (cuuint64_t)ncg, (cuuint64_t)ntiles};
  cuuint64_t strides[3] = {512, 2048, (cuuint64_t)ncg * 2048};
  cuuint32_t box[4] = {256, 2, (cuuint32_t)box_cg, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename F>
void set_smem(F* f, size_t bytes) {
  // per kernel (not per function type: the DS instantiations of a kernel share one type, and an
  // attribute set for one must not cap the other)
  static std::vector<std::pair<const void*, size_t>> done;
  for (auto& d : done)
    if (d.first == reinterpret_cast<const void*>(f)) {
      if (d.second < bytes) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        d.second = bytes;
      }
      return;
    }
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  done.emplace_back(reinterpret_cast<const void*>(f), bytes);
}

template <int DS>
void launch_dl(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment, int64_t npx,
               int64_t n_set, const int64_t* nsup, float temperature, float lambda_cos, float lambda_l2, float scale,
               bool want_grad, float* d_query, double* partials) {
  const int K = (int)w.k;
  const int NB = nb_for(n_set), NTOT = K + NB;
  const int64_t ntiles = (npx + kRows - 1) / kRows;
  const float inv_temp = 1.f / temperature;
  // DL1
  {
    Dl1Args d{w.e_tiles, query, assignment, w.kd, w.gt, npx, K, inv_temp, reinterpret_cast<float4*>(w.row_stats),
              d_query, want_grad ? 1 : 0};
    const size_t sm = (size_t)K * DS * 2 + (size_t)kRows * DS * 2;
    set_smem(dl_softmax_kernel<DS>, sm);
    dl_softmax_kernel<DS><<<148, 512, sm, st>>>(d);
    count_launch();
  }
  // DL2
  {
    Dl2Args d{w.e_tiles, w.dl_mt, reinterpret_cast<uint4*>(w.dl_t), w.dl_nu, npx, K};
    const size_t sm = (size_t)kT_Stages * (kT_A + kT_B);
    set_smem(dl_t_kernel, sm);
    const int64_t units = ntiles * (K / 256);
    dl_t_kernel<<<(unsigned)std::min<int64_t>(148, units), 192, sm, st>>>(d);
    count_launch();
  }
  // DL3
  {
    Dl3Args d{w.e_tiles, reinterpret_cast<const uint4*>(w.dl_t), w.dl_nu, reinterpret_cast<const float4*>(w.row_stats), query, assignment, w.kd,
              w.gt, w.nv, w.dl_ae, d_query, w.r_part + 148 * (size_t)K * DS, w.loss_part, npx, K, NB, inv_temp, lambda_cos, lambda_l2,
              scale, nsup, want_grad ? 1 : 0, reinterpret_cast<float2*>(w.row_nd)};
    const size_t sm = (size_t)(K / 2) * DS * 2 + (size_t)kRows * DS * 2 + 2 * 32768;
    set_smem(dl_back_kernel<DS>, sm);
    dl_back_kernel<DS><<<2 * kBackGroups, 512, sm, st>>>(d);
    count_launch();
  }
  if (w.ev_dq) cudaEventRecord(w.ev_dq, st);  // d_query complete: the render backward may start (DL4 overlaps it)
  if (!want_grad) {
    dl_reduce_kernel<<<1, 32, 0, st>>>(nullptr, 0, 0, 0, 0, 0, nullptr, 0, 0, w.loss_part, 2 * kBackGroups,
                                        nullptr, nullptr, nullptr, partials);
    count_launch();
    return;
  }
  // DL4: units = upper-triangle blocks of A (full 256-column chunks) + the Bm chunks (NB <= 256
  // columns); row splits chosen so each CTA gets about 1/148 of the MMA work
  int na, nbu, sa, sb;
  dl_gram_plan(K, NB, ntiles, na, nbu, sa, sb);
  {
    Dl4Args d{w.e_tiles, w.dl_ae, na, sa, nbu, sb, ntiles, K, NTOT, w.dl_part};
    const size_t sm = (size_t)kG_Stages * kG_Stage;
    set_smem(dl_gram_kernel, sm);
    CUtensorMap tm_e, tm_ae, tm_oh;
    const bool ok = half_tile_map(&tm_e, w.e_tiles, K / 8, ntiles, 32) &&
                    half_tile_map(&tm_ae, w.dl_ae, NTOT / 8, ntiles, 32) &&
                    half_tile_map(&tm_oh, w.dl_ae, NTOT / 8, ntiles, std::min(NB, 256) / 8);
    if (!ok) {
      cudaGetLastError();
      set_sticky_error("decoder_dl: cuTensorMapEncodeTiled unavailable or rejected the gram operand maps");
      return;
    }
    dl_gram_kernel<<<na * sa + nbu * sb, 192, sm, st>>>(tm_e, tm_ae, tm_oh, d);
    count_launch();
  }
  {
    const int64_t total = (int64_t)K * K + n_set * K + (int64_t)DS * K;
    dl_reduce_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, st>>>(
        w.dl_part, sa, sb, K, NTOT, (int)n_set, w.r_part + 148 * (size_t)K * DS, kBackGroups, DS, w.loss_part, 2 * kBackGroups, w.a_acc,
        w.bm, w.r_acc, partials);
    count_launch();
  }
}

}  // namespace

bool reconstruct_tc_supported(int64_t k, int ds, int df) {
  return k >= 256 && k <= 1024 && k % 256 == 0 && (ds == 32 || ds == 64) && df >= 256 && df % 256 == 0;
}

cudaError_t reconstruct_tc(cudaStream_t st, const float* q, int64_t n, int ds, const float* atoms, const float* proj,
                           int64_t k, int df, float temperature, float* out) {
  if (n == 0) return cudaSuccess;
  const int K = (int)k;
  const int64_t ntiles = (n + kRows - 1) / kRows;
  float *kd = nullptr, *rs = nullptr;
  uint8_t *et = nullptr, *bt = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync(&kd, sizeof(float) * k * ds, st)) || (e = cudaMallocAsync(&rs, sizeof(float) * 4 * n, st)) ||
      (e = cudaMallocAsync(&et, (size_t)ntiles * kRows * K * 2, st)) ||
      (e = cudaMallocAsync(&bt, (size_t)K * df * 2, st)))
    return e;
  sgemm(st, false, true, k, ds, df, 1.f, atoms, df, proj, df, 0.f, kd, ds);  // Kd = D W^T
  dl_tile_dt_kernel<<<(unsigned)std::min<int64_t>(((int64_t)K * df / 8 + 255) / 256, 148 * 8), 256, 0, st>>>(
      atoms, K, df, bt);
  count_launch();
  Dl1Args d1{et, q, nullptr, kd, nullptr, n, K, 1.f / temperature, reinterpret_cast<float4*>(rs), nullptr, 0};
  const size_t sm1 = (size_t)K * ds * 2 + (size_t)kRows * ds * 2;
  if (ds == 64) {
    set_smem(dl_softmax_kernel<64>, sm1);
    dl_softmax_kernel<64><<<148, 512, sm1, st>>>(d1);
  } else {
    set_smem(dl_softmax_kernel<32>, sm1);
    dl_softmax_kernel<32><<<148, 512, sm1, st>>>(d1);
  }
  count_launch();
  DlRecArgs dr{et, bt, reinterpret_cast<const float4*>(rs), out, n, K, df};
  const size_t sm = (size_t)kT_Stages * (kT_A + kT_B);
  set_smem(dl_rec_kernel, sm);
  const int64_t units = ntiles * (df / 256);
  dl_rec_kernel<<<(unsigned)std::min<int64_t>(148, units), 192, sm, st>>>(dr);
  count_launch();
  cudaFreeAsync(kd, st);
  cudaFreeAsync(rs, st);
  cudaFreeAsync(et, st);
  cudaFreeAsync(bt, st);
  return cudaGetLastError();
}

bool decoder_dl_supported(int64_t k, int ds, int64_t n_set) {
  return k >= 256 && k <= 1024 && k % 256 == 0 && (ds == 32 || ds == 64) && n_set >= 1 && n_set <= 256;
}

size_t decoder_dl_part_floats(int64_t k) {
  // gram partials: max(splits) x K x (K + NB), NB <= 256
  int smax = 1;
  for (int nb = 16; nb <= 256; nb += 16) {
    int na, nbu, sa, sb;
    dl_gram_plan((int)k, nb, 1 << 30, na, nbu, sa, sb);
    smax = std::max(smax, std::max(sa, sb));
  }
  return (size_t)smax * (size_t)k * (size_t)(k + 256);
}

void decoder_dl_prepare(cudaStream_t st, DecoderWork& w) {
  if (!w.dl_mt) return;
  const int K = (int)w.k;
  dl_tile_m_kernel<<<(unsigned)std::min<int64_t>(((int64_t)K * K / 8 + 255) / 256, 148 * 8), 256, 0, st>>>(
      w.mm, K, w.dl_mt);
  count_launch();
}

void decoder_frame_dl(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment, int64_t npx,
                      const float* feats, int64_t n_set, const int64_t* nsup, const float* atoms, float temperature,
                      float lambda_cos, float lambda_l2, float scale, bool want_grad, float* d_query,
                      float* d_atoms, double* partials) {
  const int64_t k = w.k;
  const int df = w.df;
  decoder_targets(st, feats, n_set, atoms, k, df, w.gt, w.nv);
  if (w.ds == 64)
    launch_dl<64>(st, w, query, assignment, npx, n_set, nsup, temperature, lambda_cos, lambda_l2, scale, want_grad,
                  d_query, partials);
  else
    launch_dl<32>(st, w, query, assignment, npx, n_set, nsup, temperature, lambda_cos, lambda_l2, scale, want_grad,
                  d_query, partials);
  if (!want_grad) return;
  decoder_bm_embed(st, w.bm, feats, n_set, k, df, d_atoms);
  w.tc_pending = true;
}

}  // namespace lm
