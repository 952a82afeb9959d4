// render.cu — 3DGS front end + tile rasteriser, forward and backward (sm_100a).
//
// Replaces the reference's tile-free scanline renderer (proj/src/render.cpp):
//   K1 project_kernel      <- project_one + splat_bounds      (render.cpp:42-91,153-167)
//   K2 scan_tiles_kernel   <- splats_by_row                    (render.cpp:93-101)
//   K3 scatter_kernel      <- per-pixel candidate lists        (render.cpp:174-178)
//   K3b tile_sort_kernel   <- sort_pixel std::sort per pixel   (render.cpp:104-112)
//   K4 raster_fwd_kernel   <- blend loop                       (render.cpp:183-210)
//   K8 raster_bwd_kernel   <- render_backward pixel pass       (render.cpp:275-358)
//   K9 project_bwd_kernel  <- render_backward projection pass  (render.cpp:368-429)
//
// Canonical tile list: for a 16x16 tile, every Gaussian whose inclusive 3-sigma
// bbox meets the tile, ordered by (camera z, source). A pixel's reference
// candidate list is exactly the subsequence whose bbox contains the pixel, in the
// same order, so the blend reproduces the reference per-pixel semantics. The
// projection, bbox, sort keys, alpha', clamp and termination decisions use the
// reference's float op sequence without FMA contraction, so they are bit-exact.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace lm {

namespace {

constexpr float kNegHalfLog2eF = -0.72134752044448170f;  // -0.5 * log2(e)

struct Cam {
  float r[9];  // rot_cw (world -> camera), row-major
  float o[3];  // camera origin (pose translation)
  Intr intr;
  int32_t tiles_x, tiles_y;
};

// project_one + splat_bounds with the reference's exact float/double op order.
__device__ __forceinline__ bool project_exact(const float* __restrict__ p, const float* __restrict__ q,
                                              const float* __restrict__ lsc, float logit, const Cam& c,
                                              SplatRec& out, float* cov2d_out = nullptr) {
  const float d0 = fs(p[0], c.o[0]), d1 = fs(p[1], c.o[1]), d2 = fs(p[2], c.o[2]);
  float pc[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) pc[i] = fa(fa(fm(c.r[3 * i], d0), fm(c.r[3 * i + 1], d1)), fm(c.r[3 * i + 2], d2));
  const float z = pc[2];
  if (!(z > kZNear)) return false;
  const float qn = __fsqrt_rn(fa(fa(fa(fm(q[0], q[0]), fm(q[1], q[1])), fm(q[2], q[2])), fm(q[3], q[3])));
  if (!(qn > 0.f) || !isfinite(qn)) return false;
  const float w = fd(q[0], qn), x = fd(q[1], qn), y = fd(q[2], qn), zq = fd(q[3], qn);
  float rg[9];
  rg[0] = fs(1.f, fm(2.f, fa(fm(y, y), fm(zq, zq))));
  rg[1] = fm(2.f, fs(fm(x, y), fm(w, zq)));
  rg[2] = fm(2.f, fa(fm(x, zq), fm(w, y)));
  rg[3] = fm(2.f, fa(fm(x, y), fm(w, zq)));
  rg[4] = fs(1.f, fm(2.f, fa(fm(x, x), fm(zq, zq))));
  rg[5] = fm(2.f, fs(fm(y, zq), fm(w, x)));
  rg[6] = fm(2.f, fs(fm(x, zq), fm(w, y)));
  rg[7] = fm(2.f, fa(fm(y, zq), fm(w, x)));
  rg[8] = fs(1.f, fm(2.f, fa(fm(x, x), fm(y, y))));
  float sc[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) sc[i] = exp_exact(lsc[i]);
  float m[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      m[3 * i + j] = fm(fa(fa(fm(c.r[3 * i], rg[j]), fm(c.r[3 * i + 1], rg[3 + j])), fm(c.r[3 * i + 2], rg[6 + j])),
                        sc[j]);
  float cc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      cc[3 * i + j] = fa(fa(fm(m[3 * i], m[3 * j]), fm(m[3 * i + 1], m[3 * j + 1])), fm(m[3 * i + 2], m[3 * j + 2]));
  const float fx = c.intr.fx, fy = c.intr.fy;
  const float mx = fa(fd(fm(fx, pc[0]), z), c.intr.cx);
  const float my = fa(fd(fm(fy, pc[1]), z), c.intr.cy);
  const float zz = fm(z, z);
  const float J[6] = {fd(fx, z), 0.f, fd(fm(-fx, pc[0]), zz), 0.f, fd(fy, z), fd(fm(-fy, pc[1]), zz)};
  float t[6];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      t[3 * i + j] = fa(fa(fm(J[3 * i], cc[j]), fm(J[3 * i + 1], cc[3 + j])), fm(J[3 * i + 2], cc[6 + j]));
  float cv[4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      cv[2 * i + j] = fa(fa(fm(t[3 * i], J[3 * j]), fm(t[3 * i + 1], J[3 * j + 1])), fm(t[3 * i + 2], J[3 * j + 2]));
  cv[0] = fa(cv[0], kCovReg);
  cv[3] = fa(cv[3], kCovReg);
  const float det = fs(fm(cv[0], cv[3]), fm(cv[1], cv[2]));
  if (!(det > 0.f) || !isfinite(det)) return false;
  // splat_bounds in double (render.cpp:75-91)
  const double rx = dm(kSigmaCut, __dsqrt_rn((double)cv[0]));
  const double ry = dm(kSigmaCut, __dsqrt_rn((double)cv[3]));
  const double u = (double)mx, v = (double)my;
  if (!isfinite(u) || !isfinite(v) || !isfinite(rx) || !isfinite(ry)) return false;
  const double lo_x = ceil(ds_(u, rx)), hi_x = floor(da(u, rx));
  const double lo_y = ceil(ds_(v, ry)), hi_y = floor(da(v, ry));
  const int W = c.intr.width, H = c.intr.height;
  if (hi_x < 0 || hi_y < 0 || lo_x > (double)(W - 1) || lo_y > (double)(H - 1)) return false;
  const int x0 = (int)(lo_x > 0.0 ? lo_x : 0.0);
  const int x1 = (int)((double)(W - 1) < hi_x ? (double)(W - 1) : hi_x);
  const int y0 = (int)(lo_y > 0.0 ? lo_y : 0.0);
  const int y1 = (int)((double)(H - 1) < hi_y ? (double)(H - 1) : hi_y);
  if (!(x0 <= x1 && y0 <= y1)) return false;
  out.mean_x = mx;
  out.mean_y = my;
  out.depth = z;
  out.alpha = sigmoid_exact(logit);
  out.a00 = fd(cv[3], det);
  out.a01 = fd(-cv[1], det);
  out.a10 = fd(-cv[2], det);
  out.a11 = fd(cv[0], det);
  out.x0 = x0;
  out.x1 = x1;
  out.y0 = y0;
  out.y1 = y1;
  if (cov2d_out)
    for (int i = 0; i < 4; ++i) cov2d_out[i] = cv[i];
  return true;
}

constexpr int kHistMax = 12288;  // tiles counted in shared memory (48 KB)
constexpr uint32_t kCulledKey = 0xffffffffu;  // depth key of a culled Gaussian (z bits < 0x7f800000)

// K1: project every Gaussian, write its record, count tile pairs.
__global__ void __launch_bounds__(256) project_kernel(MapPtrs map, Cam cam, SplatRec* __restrict__ rec,
                                                      uint32_t* __restrict__ dkey, int32_t* __restrict__ tile_count,
                                                      int64_t* counters) {
  extern __shared__ int32_t s_hist[];
  const int ntiles = cam.tiles_x * cam.tiles_y;
  const bool use_smem = ntiles <= kHistMax;
  if (use_smem)
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_hist[t] = 0;
  __syncthreads();
  int vis = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < map.n; i += (int64_t)gridDim.x * blockDim.x) {
    SplatRec r;
    const bool ok = project_exact(map.pos + 3 * i, map.rot + 4 * i, map.lsc + 3 * i, map.opa[i], cam, r);
    if (!ok) {
      r = SplatRec{0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 1, 0};
    } else {
      ++vis;
      const int tx0 = r.x0 / kTile, tx1 = r.x1 / kTile, ty0 = r.y0 / kTile, ty1 = r.y1 / kTile;
      for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
          const int t = ty * cam.tiles_x + tx;
          if (use_smem)
            atomicAdd(&s_hist[t], 1);
          else
            atomicAdd(&tile_count[t], 1);
        }
    }
    dkey[i] = ok ? __float_as_uint(r.depth) : kCulledKey;
    reinterpret_cast<float4*>(rec + i)[0] = make_float4(r.mean_x, r.mean_y, r.depth, r.alpha);
    reinterpret_cast<float4*>(rec + i)[1] = make_float4(r.a00, r.a01, r.a10, r.a11);
    reinterpret_cast<int4*>(rec + i)[2] = make_int4(r.x0, r.x1, r.y0, r.y1);
  }
  vis = __reduce_add_sync(0xffffffffu, vis);
  if ((threadIdx.x & 31) == 0 && vis) atomicAdd((unsigned long long*)&counters[1], (unsigned long long)vis);
  __syncthreads();
  if (use_smem)
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x)
      if (s_hist[t]) atomicAdd(&tile_count[t], s_hist[t]);
}

constexpr int kOrderBuckets = 512;
__device__ __forceinline__ int order_bucket(int c) { return kOrderBuckets - 1 - min(kOrderBuckets - 1, c >> 3); }

// K2: exclusive scan of per-tile counts (one block) + the longest-first tile dispatch order.
__global__ void __launch_bounds__(1024) scan_tiles_kernel(const int32_t* __restrict__ count, int32_t* offset,
                                                          int32_t* cursor, int ntiles, int64_t* counters,
                                                          int64_t pair_cap, int64_t* step_overflow,
                                                          int32_t* order) {
  __shared__ int64_t s_part[1024];
  const int per = (ntiles + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per;
  int64_t sum = 0;
  for (int i = 0; i < per; ++i)
    if (b + i < ntiles) sum += count[b + i];
  s_part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    int64_t v = threadIdx.x >= (unsigned)o ? s_part[threadIdx.x - o] : 0;
    __syncthreads();
    s_part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = s_part[threadIdx.x] - sum;
  for (int i = 0; i < per; ++i)
    if (b + i < ntiles) {
      offset[b + i] = (int32_t)run;
      cursor[b + i] = (int32_t)run;
      run += count[b + i];
    }
  // Dispatch order for the blend kernels: tiles by descending list length (coarse buckets of
  // 8 splats), so the longest tiles start first and the last wave is made of short tiles.
  if (order) {
    __shared__ int32_t s_bk[kOrderBuckets];
    for (int i = threadIdx.x; i < kOrderBuckets; i += blockDim.x) s_bk[i] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) atomicAdd(&s_bk[order_bucket(count[t])], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run2 = 0;
      for (int i = 0; i < kOrderBuckets; ++i) {
        const int c = s_bk[i];
        s_bk[i] = run2;
        run2 += c;
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) order[atomicAdd(&s_bk[order_bucket(count[t])], 1)] = t;
  }
  if (threadIdx.x == blockDim.x - 1) {
    offset[ntiles] = (int32_t)s_part[threadIdx.x];
    counters[0] = s_part[threadIdx.x];
    counters[2] = s_part[threadIdx.x] > pair_cap ? 1 : 0;
    if (step_overflow && s_part[threadIdx.x] > pair_cap) *step_overflow = 1;
  }
}

// K3: scatter (depth_bits << 32 | source) keys into their tile buckets. Each block first
// counts its pairs per tile in shared memory, reserves one contiguous range per (block, tile)
// with a single global atomic, then fills it (slot order inside a bucket is irrelevant: the
// per-tile sort below makes the list canonical). 2048 Gaussians per block keep the number of
// global reservations (blocks x touched tiles) low; culled Gaussians are skipped via the
// projection's depth keys without touching their records. Footprints above kBigFootprint tiles
// (Gaussians close to the camera: hundreds to thousands of tiles, config 3) are not walked
// here: they are appended to a global list that K3c spreads over every warp of the GPU.
constexpr int kScatterPerThread = 4;
constexpr int kScatterThreads = 512;
constexpr int kBigFootprint = 24;  // tiles
__global__ void __launch_bounds__(kScatterThreads, 2) scatter_kernel(const SplatRec* __restrict__ rec,
                                                      const uint32_t* __restrict__ dkey, int64_t n, int tiles_x,
                                                      int ntiles, int32_t* cursor, uint64_t* __restrict__ keys,
                                                      int64_t pair_cap, int32_t* __restrict__ big, int64_t* counters) {
  extern __shared__ int32_t s_cnt[];
  int32_t* s_base = s_cnt + ntiles;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_cnt[t] = 0;
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * blockDim.x * kScatterPerThread;
  uint32_t dk[kScatterPerThread];
  int4 bb[kScatterPerThread];
#pragma unroll
  for (int r = 0; r < kScatterPerThread; ++r) {
    const int64_t i = b0 + (int64_t)r * blockDim.x + threadIdx.x;
    dk[r] = i < n ? dkey[i] : kCulledKey;
    bb[r] = make_int4(1, 0, 1, 0);
  }
#pragma unroll
  for (int r = 0; r < kScatterPerThread; ++r)
    if (dk[r] != kCulledKey) bb[r] = reinterpret_cast<const int4*>(rec + b0 + (int64_t)r * blockDim.x + threadIdx.x)[2];
#pragma unroll
  for (int r = 0; r < kScatterPerThread; ++r) {
    if (dk[r] == kCulledKey) continue;
    const int tx0 = bb[r].x / kTile, tx1 = bb[r].y / kTile, ty0 = bb[r].z / kTile, ty1 = bb[r].w / kTile;
    if ((tx1 - tx0 + 1) * (ty1 - ty0 + 1) > kBigFootprint) {
      big[atomicAdd(reinterpret_cast<unsigned long long*>(counters + 4), 1ull)] =
          (int32_t)(b0 + (int64_t)r * blockDim.x + threadIdx.x);
      dk[r] = kCulledKey;  // emitted by K3c
      continue;
    }
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(&s_cnt[ty * tiles_x + tx], 1);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    const int c = s_cnt[t];
    if (c) s_base[t] = atomicAdd(&cursor[t], c);
    s_cnt[t] = 0;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kScatterPerThread; ++r) {
    if (dk[r] == kCulledKey) continue;
    const uint64_t key = ((uint64_t)dk[r] << 32) | (uint32_t)(b0 + (int64_t)r * blockDim.x + threadIdx.x);
    for (int ty = bb[r].z / kTile; ty <= bb[r].w / kTile; ++ty)
      for (int tx = bb[r].x / kTile; tx <= bb[r].y / kTile; ++tx) {
        const int t = ty * tiles_x + tx;
        const int64_t pos = (int64_t)s_base[t] + atomicAdd(&s_cnt[t], 1);
        if (pos < pair_cap) keys[pos] = key;
      }
  }
}

// K3c: the large footprints K3 deferred, one warp per Gaussian (grid-stride over the global
// list), a lane per tile; each pair takes its slot with one global atomic on the tile cursor
// (slot order is again irrelevant).
__global__ void __launch_bounds__(256) scatter_big_kernel(const SplatRec* __restrict__ rec,
                                                          const uint32_t* __restrict__ dkey,
                                                          const int32_t* __restrict__ big, const int64_t* counters,
                                                          int tiles_x, int32_t* cursor, uint64_t* __restrict__ keys,
                                                          int64_t pair_cap) {
  const int64_t nbig = counters[4];
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t e = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); e < nbig; e += nw) {
    const int32_t src = big[e];
    const int4 q = reinterpret_cast<const int4*>(rec + src)[2];
    const uint64_t key = ((uint64_t)dkey[src] << 32) | (uint32_t)src;
    const int tx0 = q.x / kTile, ty0 = q.z / kTile, w = q.y / kTile - tx0 + 1, nt = w * (q.w / kTile - ty0 + 1);
    for (int t = lane; t < nt; t += 32) {
      const int tile = (ty0 + t / w) * tiles_x + tx0 + t % w;
      const int64_t pos = atomicAdd(&cursor[tile], 1);
      if (pos < pair_cap) keys[pos] = key;
    }
  }
}

// K3b: per-tile bitonic sort of the (depth, source) keys -> canonical order. Keys are unique,
// so the result is deterministic whatever order K3's atomics produced. 512 threads hold KPT
// consecutive keys each (blocked layout): compare-exchange partners at distance j < KPT are in
// the same thread's registers, j < 32 KPT in the same warp (shuffles), larger j go through
// shared memory (10 of the 66 stages at P = 2048).
constexpr int kSortThreads = 512;
constexpr int kSortCap = 8192;  // keys sorted in one pass (16 per thread, 64 KB of shared memory)

template <int KPT, int J>
__device__ __forceinline__ void bitonic_reg_stage(uint64_t (&v)[KPT], int tid, int k) {
#pragma unroll
  for (int e = 0; e < KPT; ++e)
    if ((e & J) == 0) {
      const bool asc = (((tid * KPT + e) & k) == 0);
      const uint64_t a = v[e], b = v[e | J];
      if ((a > b) == asc) {
        v[e] = b;
        v[e | J] = a;
      }
    }
}

template <int KPT>
__device__ void bitonic_block(uint64_t (&v)[KPT], uint64_t* s, int P) {
  const int tid = threadIdx.x;
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < KPT) {
        if (j == 1) bitonic_reg_stage<KPT, 1>(v, tid, k);
        if constexpr (KPT > 2) if (j == 2) bitonic_reg_stage<KPT, 2>(v, tid, k);
        if constexpr (KPT > 4) if (j == 4) bitonic_reg_stage<KPT, 4>(v, tid, k);
        if constexpr (KPT > 8) if (j == 8) bitonic_reg_stage<KPT, 8>(v, tid, k);
      } else if (j < 32 * KPT) {
        const int lm = j / KPT;
        const bool lower = (tid & lm) == 0;
#pragma unroll
        for (int e = 0; e < KPT; ++e) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], lm);
          const bool asc = (((tid * KPT + e) & k) == 0);
          v[e] = (lower == asc) ? (v[e] < o ? v[e] : o) : (v[e] < o ? o : v[e]);
        }
      } else {
        __syncthreads();
#pragma unroll
        for (int e = 0; e < KPT; ++e) s[tid * KPT + e] = v[e];
        __syncthreads();
        const bool lower = ((tid * KPT) & j) == 0;
#pragma unroll
        for (int e = 0; e < KPT; ++e) {
          const int i = tid * KPT + e;
          const uint64_t o = s[i ^ j];
          const bool asc = ((i & k) == 0);
          v[e] = (lower == asc) ? (v[e] < o ? v[e] : o) : (v[e] < o ? o : v[e]);
        }
      }
    }
}

template <int KPT>
__device__ void sort_chunk(uint64_t* g, int n, uint64_t* s) {
  constexpr int P = KPT * kSortThreads;
  uint64_t v[KPT];
#pragma unroll
  for (int e = 0; e < KPT; ++e) {
    const int i = threadIdx.x * KPT + e;
    v[e] = i < n ? g[i] : ~0ull;
  }
  bitonic_block<KPT>(v, s, P);
#pragma unroll
  for (int e = 0; e < KPT; ++e) {
    const int i = threadIdx.x * KPT + e;
    if (i < n) g[i] = v[e];
  }
}

__device__ void sort_chunk_any(uint64_t* g, int n, uint64_t* s) {
  if (n <= 512) sort_chunk<1>(g, n, s);
  else if (n <= 1024) sort_chunk<2>(g, n, s);
  else if (n <= 2048) sort_chunk<4>(g, n, s);
  else if (n <= 4096) sort_chunk<8>(g, n, s);
  else sort_chunk<16>(g, n, s);
}

// Per-tile stable LSD radix sort on the depth half of the keys (4 passes of 8 bits) in shared
// memory, then the rare runs of equal depth are put in source order (the key's low half). The
// 512 threads form 16 warps; warp w owns elements [w*32*EPT, (w+1)*32*EPT) in EPT rounds of 32,
// and an element's rank among equal digits before it is (round peers below it, __match_any)
// + (warp's running count) + (exclusive scan over (digit, warp) in digit-major order).
constexpr int kRadixCap = 4096;  // tile lists up to this length take the radix path (EPT <= 8)
constexpr size_t kTileSortSmem = 2 * kRadixCap * 8 + 16 * 257 * 4;  // >= kSortCap * 8

__device__ void tile_radix_sort(uint64_t* __restrict__ g, int n, uint64_t* s_a, uint64_t* s_b, uint32_t* s_h) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ept = (n + kSortThreads - 1) / kSortThreads;
  for (int i = tid; i < n; i += kSortThreads) s_a[i] = g[i];
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t* s_w = s_h;  // [16 warps][257] (padded: conflict-free column walks)
#pragma unroll 1
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 32 + 8 * pass;
    {  // a digit shared by every key (the exponent byte, typically) leaves the order unchanged
      const uint32_t d0 = (uint32_t)(s_a[0] >> shift) & 255u;
      bool differs = false;
      for (int i = tid; i < n; i += kSortThreads) differs |= ((uint32_t)(s_a[i] >> shift) & 255u) != d0;
      if (!__syncthreads_or(differs)) continue;
    }
    for (int i = tid; i < 257 * 16; i += kSortThreads) s_w[i] = 0u;
    __syncthreads();
    uint64_t k[8];
    uint32_t loc[8];
    int d[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r >= ept) break;
      const int i = (warp * ept + r) * 32 + lane;
      k[r] = i < n ? s_a[i] : 0ull;
      d[r] = i < n ? (int)((k[r] >> shift) & 255u) : 256;
      uint32_t peers = 0xffffffffu;  // lanes with the same 9-bit digit (ballots: cheaper than match.any)
#pragma unroll
      for (int b = 0; b < 9; ++b) {
        const bool bit = (d[r] >> b) & 1;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
      const bool ok = d[r] < 256;
      loc[r] = __popc(peers & lt) + (ok ? s_w[warp * 257 + (ok ? d[r] : 0)] : 0u);
      __syncwarp();
      if (ok && (peers & lt) == 0u) s_w[warp * 257 + d[r]] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    {  // exclusive scan over (digit, warp) in digit-major order: entry e = tid * 8 + j
      uint32_t v[8], sum = 0;
      const int dd = tid >> 1, w0 = (tid & 1) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = s_w[(w0 + j) * 257 + dd];
        sum += v[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      __shared__ uint32_t s_ws[16];
      if (lane == 31) s_ws[warp] = incl;
      __syncthreads();
      uint32_t wb = lane < 16 && lane < warp ? s_ws[lane] : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wb += __shfl_xor_sync(0xffffffffu, wb, o);
      uint32_t run = wb + incl - sum;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s_w[(w0 + j) * 257 + dd] = run;
        run += v[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r >= ept) break;
      if (d[r] < 256) s_b[s_w[warp * 257 + d[r]] + loc[r]] = k[r];
    }
    __syncthreads();
    uint64_t* sw = s_a;
    s_a = s_b;
    s_b = sw;
  }
  // equal depths (rare): order each run by source
  for (int i = tid; i < n; i += kSortThreads) {
    const uint32_t di = (uint32_t)(s_a[i] >> 32);
    const bool start = i == 0 || (uint32_t)(s_a[i - 1] >> 32) != di;
    if (start && i + 1 < n && (uint32_t)(s_a[i + 1] >> 32) == di) {
      int e = i + 1;
      while (e < n && (uint32_t)(s_a[e] >> 32) == di) ++e;
      for (int a = i + 1; a < e; ++a) {  // insertion sort of [i, e) by the full key
        const uint64_t x = s_a[a];
        int b = a - 1;
        while (b >= i && s_a[b] > x) {
          s_a[b + 1] = s_a[b];
          --b;
        }
        s_a[b + 1] = x;
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += kSortThreads) g[i] = s_a[i];
}

__global__ void __launch_bounds__(kSortThreads, 2) tile_sort_kernel(const int32_t* __restrict__ offset, uint64_t* keys,
                                                                 uint64_t* tmp, int64_t pair_cap,
                                                                 const int64_t* counters) {
  extern __shared__ uint64_t s_keys[];
  if (counters[2]) return;  // overflowed: step is discarded and re-run by the host
  const int t = blockIdx.x;
  const int start = offset[t], n = offset[t + 1] - start;
  if (n <= 1) return;
  uint64_t* g = keys + start;
  if (n <= kRadixCap) {
    tile_radix_sort(g, n, s_keys, s_keys + kRadixCap, reinterpret_cast<uint32_t*>(s_keys + 2 * kRadixCap));
    return;
  }
  if (n <= kSortCap) {
    sort_chunk_any(g, n, s_keys);
    return;
  }
  // Oversized tile: sort kSortCap chunks, then merge runs pairwise in global memory.
  for (int c0 = 0; c0 < n; c0 += kSortCap) {
    sort_chunk<16>(g + c0, min(kSortCap, n - c0), s_keys);
    __syncthreads();
  }
  uint64_t* src = g;
  uint64_t* dst = tmp + start;
  for (int width = kSortCap; width < n; width <<= 1) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int run0 = (i / (2 * width)) * 2 * width;
      const int mid = min(run0 + width, n), end = min(run0 + 2 * width, n);
      const uint64_t v = src[i];
      int pos;
      if (i < mid) {  // element of run A: rank within A + number of B elements < v
        int lo = mid, hi = end;
        while (lo < hi) {
          const int m = (lo + hi) >> 1;
          if (src[m] < v) lo = m + 1; else hi = m;
        }
        pos = run0 + (i - run0) + (lo - mid);
      } else {  // element of run B: rank within B + number of A elements < v
        int lo = run0, hi = mid;
        while (lo < hi) {
          const int m = (lo + hi) >> 1;
          if (src[m] < v) lo = m + 1; else hi = m;
        }
        pos = run0 + (i - mid) + (lo - run0);
      }
      dst[pos] = v;
    }
    __syncthreads();
    uint64_t* sw = src;
    src = dst;
    dst = sw;
  }
  if (src != g)
    for (int i = threadIdx.x; i < n; i += blockDim.x) g[i] = src[i];
}

// Pixel `pl` (0..255) of a 16x16 tile in the blend kernels: warp w = pl / 32 covers an 8x4 pixel
// block (w & 1: left/right half, w / 2: 4-row band), lane i = pl % 32 pixel (i % 8, i / 8) of it.
// Square-ish warp footprints meet fewer splat bboxes than 16x2 strips and waste fewer lanes.
__device__ __forceinline__ int tile_dx(int pl) { return ((pl >> 5) & 1) * 8 + (pl & 7); }
__device__ __forceinline__ int tile_dy(int pl) { return (pl >> 6) * 4 + ((pl >> 3) & 3); }

struct RasterArgs {
  const SplatRec* rec;
  const float* colors;
  const float* feats;
  int32_t ds;
  const int32_t* offset;
  const uint64_t* keys;  // per-tile lists: (depth bits << 32 | source)
  int32_t tiles_x, width, height;
  float *color, *depth, *query, *alpha;
  int32_t* px_last;
  float* px_T;
  int32_t* tile_max_last;
  const int64_t* counters;
  const int32_t* order;  // dispatch order (longest tile lists first)
};

// K4: forward blend, one CTA per 16x16 tile, one thread per pixel. alpha', the clamp, the
// transmittance and the termination test always use the reference's float op sequence
// (bit-exact decisions); EXACT additionally accumulates colour/depth/alpha/query with
// separately rounded products and sums (bit-exact images), otherwise with FMA.
template <int DSP, bool EXACT>
__global__ void __launch_bounds__(kTilePixels) raster_fwd_kernel(RasterArgs a) {
  constexpr int kFwdBatch = DSP >= 64 ? 128 : 256;
  __shared__ SplatRec s_rec[kFwdBatch];
  __shared__ float s_col[kFwdBatch * 3];
  __shared__ float s_feat[kFwdBatch * DSP];
  __shared__ int32_t s_max;
  __shared__ uint64_t s_etab[32];
  if (a.counters[2]) return;
  load_exp_table(s_etab);  // published by the first __syncthreads_and of the batch loop
  const int tile = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int px = (tile % a.tiles_x) * kTile + (threadIdx.x % kTile);
  const int py = (tile / a.tiles_x) * kTile + (threadIdx.x / kTile);
  const bool inside = px < a.width && py < a.height;
  const int start = a.offset[tile], end = a.offset[tile + 1];
  if (threadIdx.x == 0) s_max = 0;
  float T = 1.f, acc_c0 = 0.f, acc_c1 = 0.f, acc_c2 = 0.f, acc_d = 0.f, acc_a = 0.f;
  float acc_q[DSP];
#pragma unroll
  for (int c = 0; c < DSP; ++c) acc_q[c] = 0.f;
  bool done = !inside;
  int last = end - start;
  const float fx = (float)px, fy = (float)py;
  for (int base = start; base < end; base += kFwdBatch) {
    if (__syncthreads_and(done)) break;
    const int i = base + threadIdx.x;
    if (threadIdx.x < kFwdBatch && i < end) {
      const uint32_t src = (uint32_t)a.keys[i];
      s_rec[threadIdx.x] = a.rec[src];
      s_col[threadIdx.x * 3 + 0] = a.colors[3 * (size_t)src + 0];
      s_col[threadIdx.x * 3 + 1] = a.colors[3 * (size_t)src + 1];
      s_col[threadIdx.x * 3 + 2] = a.colors[3 * (size_t)src + 2];
      const float* f = a.feats + (size_t)src * a.ds;
#pragma unroll
      for (int c = 0; c < DSP; ++c) s_feat[threadIdx.x * DSP + c] = c < a.ds ? f[c] : 0.f;
    }
    __syncthreads();
    const int cnt = min(kFwdBatch, end - base);
    if (!done) {
      for (int j = 0; j < cnt; ++j) {
        const SplatRec& s = s_rec[j];
        if (px < s.x0 || px > s.x1 || py < s.y0 || py > s.y1) continue;
        const float dx = fs(fx, s.mean_x);
        const float dy = fs(fy, s.mean_y);
        const float rho = fa(fa(fm(fm(s.a00, dx), dx), fm(fm(fm(2.f, s.a01), dx), dy)), fm(fm(s.a11, dy), dy));
        // exact mode: libm expf restated (bit-exact blend decisions); fast mode: the SFU exp2
        float al = EXACT ? fm(s.alpha, exp_exact(fm(-0.5f, rho), s_etab)) : fm(s.alpha, ex2_approx(fm(kNegHalfLog2eF, rho)));
        if (al > kAlphaMax) al = kAlphaMax;
        const float w = fm(al, T);
        if (EXACT) {
          acc_c0 = fa(acc_c0, fm(w, s_col[j * 3 + 0]));
          acc_c1 = fa(acc_c1, fm(w, s_col[j * 3 + 1]));
          acc_c2 = fa(acc_c2, fm(w, s_col[j * 3 + 2]));
          acc_d = fa(acc_d, fm(w, s.depth));
#pragma unroll
          for (int c = 0; c < DSP; ++c) acc_q[c] = fa(acc_q[c], fm(w, s_feat[j * DSP + c]));
        } else {
          acc_c0 = fmaf(w, s_col[j * 3 + 0], acc_c0);
          acc_c1 = fmaf(w, s_col[j * 3 + 1], acc_c1);
          acc_c2 = fmaf(w, s_col[j * 3 + 2], acc_c2);
          acc_d = fmaf(w, s.depth, acc_d);
#pragma unroll
          for (int c = 0; c < DSP; ++c) acc_q[c] = fmaf(w, s_feat[j * DSP + c], acc_q[c]);
        }
        acc_a = fa(acc_a, w);
        T = fm(T, fs(1.f, al));
        if (T < kTransmitStop) {
          done = true;
          last = base - start + j + 1;
          break;
        }
      }
    }
  }
  if (inside) {
    const size_t p = (size_t)py * a.width + px;
    a.color[3 * p + 0] = acc_c0;
    a.color[3 * p + 1] = acc_c1;
    a.color[3 * p + 2] = acc_c2;
    a.depth[p] = acc_d;
    a.alpha[p] = acc_a;
    float* q = a.query + p * a.ds;
#pragma unroll
    for (int c = 0; c < DSP; ++c)
      if (c < a.ds) q[c] = acc_q[c];
    a.px_last[p] = last;
    a.px_T[p] = T;
  }
  __syncthreads();
  if (inside) atomicMax(&s_max, last);
  __syncthreads();
  if (threadIdx.x == 0) a.tile_max_last[tile] = s_max;
}

struct RasterBwdArgs {
  const SplatRec* rec;
  const float* colors;
  const float* feats;
  int32_t ds;
  const int32_t* offset;
  const uint64_t* keys;  // per-tile lists: (depth bits << 32 | source)
  int32_t tiles_x, width, height;
  const int32_t* px_last;
  const float* px_T;
  const int32_t* tile_max_last;
  const float *d_color, *d_depth, *d_query;
  float* geo_acc;  // N x 8: dmean_u, dmean_v, dA00, dA01, dA11, dz, dg
  float* g_col;    // N x 3
  float* g_feat;   // N x ds
  const int32_t* order;
  const int64_t* counters;
  // deterministic mode (nullptr = float atomics): per (splat, tile) partial rows, splat-major,
  // tiles of a splat in row-major order: row = splat_off[src] + rank(tile in the splat's rect)
  float* pair_part;
  const int64_t* splat_off;
};

constexpr int kBwdBatch = 16;  // splats per batch (one MMA M tile)
// deterministic partial row: [geo 8 | colour 3, pad | features ds padded to 4]
__host__ __device__ constexpr int det_width(int ds) { return 12 + (ds + 3) / 4 * 4; }

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// 3xTF32 operand split by truncation: hi keeps the top 10 mantissa bits, lo = x - hi (exact
// in fp32) truncated likewise; |x - hi - lo| < 2^-20 |x|. Three integer/fp ops instead of the
// six of two cvt.rna.tf32 conversions (which lower to FSETP + IADD + LOP3 each on sm_100a).
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi)) & 0xffffe000u;
}
// D += A * B, m16n8k8, tf32 inputs, fp32 accumulate (legacy warp MMA, used for small in-kernel reductions)
__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// K4 (fast mode, ds >= 8): same per-pixel decisions and colour/depth/alpha accumulation as
// raster_fwd_kernel<DSP, false>; the query channels, which dominate the per-(pixel, splat) work,
// are accumulated on the tensor cores instead: per warp and 16-splat sub-batch the blend weights
// W (32 pixels x 16 splats, from the scalar pass) multiply the splats' features F (16 x DSP),
// Q += W F as 3xTF32 m16n8k8 MMAs (~fp32 accurate, different summation order than the scalar loop).
template <int DSP>
__global__ void __launch_bounds__(kTilePixels, DSP >= 64 ? 1 : 2) raster_fwd_mma_kernel(RasterArgs a) {
  constexpr int FB = 128;           // splats per shared-memory batch
  constexpr int FP = DSP + 8;       // feature pitch: B-fragment loads hit distinct banks
  constexpr int WP = 40;            // per-warp [splat][pixel] weight pitch
  constexpr int NQ = DSP / 8;       // n-tiles (8 channels each)
  constexpr int RP = 16 + (DSP + 3) / 4 * 4;  // raw staging row: [SplatRec 12 | colour 3 | - | features]
  extern __shared__ __align__(16) float s_dyn[];
  float* s_fh = s_dyn;                      // [FB][FP] tf32 hi
  float* s_fl = s_fh + FB * FP;             // [FB][FP] tf32 lo
  float* s_w = s_fl + FB * FP;              // [8 warps][16][WP]
  float* s_raw = s_w + 8 * 16 * WP;         // [FB][RP] cp.async staging of the next batch
  __shared__ float4 s_sp[FB][3];            // {mean_x, mean_y, a00, 2 a01} {a11, alpha, depth, -} {x0, x1-x0, y0, y1-y0}
  __shared__ float s_col[FB * 3];
  __shared__ int32_t s_max;
  if (a.counters[2]) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, cq = lane & 3;
  const int tile = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tx0 = (tile % a.tiles_x) * kTile, ty0 = (tile / a.tiles_x) * kTile;
  const int px = tx0 + tile_dx(tid), py = ty0 + tile_dy(tid);
  const bool inside = px < a.width && py < a.height;
  const int start = a.offset[tile], end = a.offset[tile + 1];
  if (tid == 0) s_max = 0;
  const bool vec_feat = (a.ds & 3) == 0 && (reinterpret_cast<uintptr_t>(a.feats) & 15) == 0;
  // thread t < FB stages splat t of a batch: record, colour and features into s_raw (cp.async)
  auto stage = [&](uint32_t src) {
    float* row = s_raw + tid * RP;
    const float4* rg = reinterpret_cast<const float4*>(a.rec + src);
    cp_async16(row, rg);
    cp_async16(row + 4, rg + 1);
    cp_async16(row + 8, rg + 2);
    cp_async4(row + 12, a.colors + 3 * (size_t)src);
    cp_async4(row + 13, a.colors + 3 * (size_t)src + 1);
    cp_async4(row + 14, a.colors + 3 * (size_t)src + 2);
    const float* f = a.feats + (size_t)src * a.ds;
    if (vec_feat) {
      for (int c = 0; c < a.ds; c += 4) cp_async16(row + 16 + c, f + c);
    } else {
      for (int c = 0; c < a.ds; ++c) cp_async4(row + 16 + c, f + c);
    }
  };
  uint32_t nsrc = 0;
  if (tid < FB) {
    if (start + tid < end) stage((uint32_t)a.keys[start + tid]);
    cp_async_commit();
    if (start + FB + tid < end) nsrc = (uint32_t)a.keys[start + FB + tid];
  }
  float T = 1.f, acc_c0 = 0.f, acc_c1 = 0.f, acc_c2 = 0.f, acc_d = 0.f, acc_a = 0.f;
  float q[2][NQ][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NQ; ++nt) q[mt][nt][0] = q[mt][nt][1] = q[mt][nt][2] = q[mt][nt][3] = 0.f;
  bool done = !inside;
  int last = end - start;
  const float fx = (float)px, fy = (float)py;
  float* sw = s_w + warp * 16 * WP;
  // this warp's pixel block: columns bx0 .. bx0 + 7, rows by0 .. by0 + 3
  const int bx0 = tx0 + (warp & 1) * 8, by0 = ty0 + (warp >> 1) * 4;
  for (int base = start; base < end; base += FB) {
    cp_async_wait_all();
    if (__syncthreads_and(done)) break;
    const int cnt = min(FB, end - base);
    // ---- unpack the staged batch: tf32 hi/lo feature rows, record terms, colours
    for (int e = tid; e < cnt * DSP; e += kTilePixels) {
      const int j = e / DSP, c = e % DSP;
      const float v = c < a.ds ? s_raw[j * RP + 16 + c] : 0.f;
      uint32_t hi, lo;
      split_tf32(v, hi, lo);
      s_fh[j * FP + c] = __uint_as_float(hi);
      s_fl[j * FP + c] = __uint_as_float(lo);
    }
    if (cnt < FB)  // zero the tail of the last sub-batch so padded splats contribute nothing
      for (int e = cnt * DSP + tid; e < ((cnt + 15) & ~15) * DSP; e += kTilePixels) {
        const int j = e / DSP, c = e % DSP;
        s_fh[j * FP + c] = 0.f;
        s_fl[j * FP + c] = 0.f;
      }
    if (tid < cnt) {
      const float* row = s_raw + tid * RP;
      const float4 r0 = *reinterpret_cast<const float4*>(row);      // mean_x, mean_y, depth, alpha
      const float4 r1 = *reinterpret_cast<const float4*>(row + 4);  // a00, a01, a10, a11
      // the conic prescaled by -log2(e)/2: the exp2 argument is one FMA chain per pixel
      s_sp[tid][0] = make_float4(r0.x, r0.y, kNegHalfLog2eF * r1.x, kNegHalfLog2eF * (2.f * r1.y));
      s_sp[tid][1] = make_float4(kNegHalfLog2eF * r1.w, r0.w, r0.z, 0.f);
      int4 bb = *reinterpret_cast<const int4*>(row + 8);
      bb.y -= bb.x;  // extents: one unsigned compare per axis in the per-pixel test
      bb.w -= bb.z;
      s_sp[tid][2] = i4_as_f4(bb);
      s_col[tid * 3 + 0] = row[12];
      s_col[tid * 3 + 1] = row[13];
      s_col[tid * 3 + 2] = row[14];
    }
    __syncthreads();
    // ---- prefetch the next batch into the (now free) staging rows
    if (tid < FB && base + FB < end) {
      if (base + FB + tid < end) stage(nsrc);
      cp_async_commit();
      nsrc = base + 2 * FB + tid < end ? (uint32_t)a.keys[base + 2 * FB + tid] : 0u;
    }
    for (int sb = 0; sb < cnt; sb += 16) {
      if (__all_sync(0xffffffffu, done)) break;
      // splats of the sub-batch whose bbox meets the warp's 8x4 block (any other has no pixel of
      // the warp in its bbox: every blend weight is 0 and the sub-batch is skipped or zero-filled)
      bool meets = false;
      if (lane < 16 && sb + lane < cnt) {
        const int4 bb = f4_as_i4(s_sp[sb + lane][2]);
        meets = bb.x <= bx0 + 7 && bb.x + bb.y >= bx0 && bb.z <= by0 + 3 && bb.z + bb.w >= by0;
      }
      const uint32_t wmask = __ballot_sync(0xffffffffu, meets);
      if (wmask == 0u) continue;
#pragma unroll
      for (int j4 = 0; j4 < 16; j4 += 4) {
        if (((wmask >> j4) & 15u) == 0u) {
#pragma unroll
          for (int u = 0; u < 4; ++u) sw[(j4 + u) * WP + lane] = 0.f;
          continue;
        }
        // alpha' of four splats evaluated independently (ILP over the exact exp), then the
        // transmittance chain in order
        float alv[4];
        bool ok[4];
        bool any = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = sb + j4 + u;
          const int4 bb = f4_as_i4(s_sp[j][2]);
          ok[u] = !done && j < cnt && (unsigned)(px - bb.x) <= (unsigned)bb.y && (unsigned)(py - bb.z) <= (unsigned)bb.w;
          any |= ok[u];
        }
        if (__any_sync(0xffffffffu, any)) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 s0 = s_sp[sb + j4 + u][0];
            const float4 s1 = s_sp[sb + j4 + u][1];
            const float dx = fx - s0.x;
            const float dy = fy - s0.y;
            // fast mode: exp(-rho/2) on the SFU (ex2.approx, ~2^-22 relative), the argument as one
            // FMA chain over the prescaled conic -- what the backward replays; the exact-mode kernel
            // (raster_fwd_kernel<DSP, true>) keeps the reference's op order and libm expf
            const float pw = fmaf(dx, fmaf(s0.z, dx, s0.w * dy), s1.x * dy * dy);
            float al = s1.y * ex2_approx(pw);
            alv[u] = al > kAlphaMax ? kAlphaMax : al;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = sb + j4 + u;
          float w = 0.f;
          if (ok[u] && !done) {
            const float al = alv[u];
            w = fm(al, T);
            acc_c0 = fmaf(w, s_col[j * 3 + 0], acc_c0);
            acc_c1 = fmaf(w, s_col[j * 3 + 1], acc_c1);
            acc_c2 = fmaf(w, s_col[j * 3 + 2], acc_c2);
            acc_d = fmaf(w, s_sp[j][1].z, acc_d);
            acc_a = fa(acc_a, w);
            T = fm(T, fs(1.f, al));
            if (T < kTransmitStop) {
              done = true;
              last = base - start + j + 1;
            }
          }
          sw[(j4 + u) * WP + lane] = w;
        }
      }
      __syncwarp();
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        uint32_t ah[2][4], alo[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int r = 16 * mt + g;
          split_tf32(sw[(8 * ks + cq) * WP + r], ah[mt][0], alo[mt][0]);
          split_tf32(sw[(8 * ks + cq) * WP + r + 8], ah[mt][1], alo[mt][1]);
          split_tf32(sw[(8 * ks + cq + 4) * WP + r], ah[mt][2], alo[mt][2]);
          split_tf32(sw[(8 * ks + cq + 4) * WP + r + 8], ah[mt][3], alo[mt][3]);
        }
        const int j0 = sb + 8 * ks + cq;
#pragma unroll
        for (int nt = 0; nt < NQ; ++nt) {
          uint32_t bh[2], bl[2];
          bh[0] = __float_as_uint(s_fh[j0 * FP + 8 * nt + g]);
          bh[1] = __float_as_uint(s_fh[(j0 + 4) * FP + 8 * nt + g]);
          bl[0] = __float_as_uint(s_fl[j0 * FP + 8 * nt + g]);
          bl[1] = __float_as_uint(s_fl[(j0 + 4) * FP + 8 * nt + g]);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            mma_tf32(q[mt][nt], alo[mt], bh);
            mma_tf32(q[mt][nt], ah[mt], bl);
            mma_tf32(q[mt][nt], ah[mt], bh);
          }
        }
      }
      __syncwarp();
    }
  }
  cp_async_wait_all();
  if (inside) {
    const size_t p = (size_t)py * a.width + px;
    a.color[3 * p + 0] = acc_c0;
    a.color[3 * p + 1] = acc_c1;
    a.color[3 * p + 2] = acc_c2;
    a.depth[p] = acc_d;
    a.alpha[p] = acc_a;
    a.px_last[p] = last;
    a.px_T[p] = T;
  }
  // query from the accumulator fragments: rows = the warp's pixels, columns = channels
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int pl = 32 * warp + 16 * mt + g + 8 * hh;
      const int qx = tx0 + tile_dx(pl), qy = ty0 + tile_dy(pl);
      if (qx < a.width && qy < a.height) {
        float* qo = a.query + ((size_t)qy * a.width + qx) * a.ds;
#pragma unroll
        for (int nt = 0; nt < NQ; ++nt) {
          const int c = 8 * nt + 2 * cq;
          if (c < a.ds) qo[c] = q[mt][nt][2 * hh];
          if (c + 1 < a.ds) qo[c + 1] = q[mt][nt][2 * hh + 1];
        }
      }
    }
  __syncthreads();
  if (inside) atomicMax(&s_max, last);
  __syncthreads();
  if (tid == 0) a.tile_max_last[tile] = s_max;
}

// K8: reverse sweep of render_backward (render.cpp:315-353), one CTA per 16x16 tile, one
// thread per pixel. Transmittance before each blended splat is recovered by division from
// the forward's final T. Per batch of 16 splats each thread records, per (pixel, splat),
//   w = alpha' T (blend weight), drho = -alpha' dalpha / 2, dg = dalpha alpha'/alpha.
// The per-splat sums over the tile's pixels are then tensor-core reductions (3xTF32 split,
// ~fp32 accurate):  [dcolor, dz, dfeat] = W^T U  (U = per-pixel upstream [uc, uz, uq]),
// and the drho moments  sum drho * [1, x, y, x^2, xy, y^2]  (+ sum dg), from which
// dmean and dA (render.cpp:345-352) follow per splat in closed form.
// Two barriers per batch. Phase 1: the warps' sweep and tensor-core reductions of batch i,
// the tf32 split of batch i+1 (staged one batch earlier) and the cp.async staging of batch
// i+2 (record, colour, features; 16 lanes of warp 0). Phase 2: each (splat, output slot) sums
// its entries over the active warps' partials and forms the closed-form gradients. A warp
// whose 8x4 pixel block meets none of the batch's bboxes, or whose pixels all stopped before
// the batch, skips the batch's sweep and contributes nothing.
template <int DSP>
__global__ void __launch_bounds__(kTilePixels, DSP >= 64 ? 1 : 2) raster_bwd_kernel(RasterBwdArgs a) {
  constexpr int NU = ((4 + DSP) + 7) / 8 * 8;  // U columns: uc0..2, uz, uq[DSP], pad
  constexpr int NT = NU / 8;                   // n-tiles of the W^T U product
  // U row pitch = 8 mod 16 plus a column XOR swizzle on row bit 2: both the row-fragment
  // (value MMA) and the column-fragment (W^T U MMA) loads are bank conflict free
  constexpr int UP = NU % 16 == 8 ? NU : NU + 8;
  constexpr int NACC = NU + 8 + 8;             // per-splat partial entries: W^T U | drho moments | dg
  constexpr int NUP = NU + 4;                  // splat-row pitch (B-fragment loads hit distinct banks)
  constexpr int PP = (NACC + 23) / 32 * 32 + 8;  // per-warp partial pitch (= 8 mod 32)
  // per-warp [splat][pixel] pitch: 32 with an XOR swizzle of the pixel index by the splat row
  // (conflict-free row writes and fragment reads), 36 padded when the partials need the room
  constexpr int WP = 16 * PP <= 3 * kBwdBatch * 32 ? 32 : 36;
  // raw staging row (floats): [SplatRec 12 | colour 3 | source bits | features DSP (padded to 4)]
  constexpr int RP = 16 + (DSP + 3) / 4 * 4 + ((DSP + 3) / 4 % 2 == 0 ? 4 : 0);
  static_assert(16 * PP <= 3 * kBwdBatch * WP, "warp partials must fit the warp's staging area");
  auto uidx = [](int p, int c) { return p * UP + (c ^ (((p >> 2) & 1) << 2)); };
  auto widx = [](int j, int p) { return j * WP + (WP == 32 ? (p ^ ((j & 7) << 2)) : p); };
  extern __shared__ __align__(16) float s_dyn[];
  float* s_u = s_dyn;                                          // [256][UP] per-pixel upstream rows
  float* s_wbase = s_dyn + kTilePixels * UP;                   // [8 warps][3][16 * WP]: W, drho, dg
  __shared__ __align__(16) float s_fh[2][kBwdBatch * NUP];   // splat rows [c0 c1 c2 z f...], tf32 hi
  __shared__ __align__(16) float s_fl[2][kBwdBatch * NUP];   //   ... and tf32 lo
  __shared__ __align__(16) float s_raw[2][kBwdBatch * RP];   // cp.async staging
  // per splat: {mx, my, q00', 2q01'} {q11', alpha, A00, A01} {x0, x1 - x0, y0, y1 - y0}
  // {A10, A11, source bits, -}; a padding row has x0 = INT_MAX / 2 (meets no pixel)
  __shared__ __align__(16) float4 s_sp[2][4][kBwdBatch];  // [slot][field][splat]
  __shared__ int32_t s_wact[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tx0 = (tile % a.tiles_x) * kTile, ty0 = (tile / a.tiles_x) * kTile;
  const int px = tx0 + tile_dx(tid), py = ty0 + tile_dy(tid);
  const bool inside = px < a.width && py < a.height;
  if (a.counters[2]) return;  // tile lists overflowed: the step is discarded and re-run
  const int start = a.offset[tile];
  const int tend = start + a.tile_max_last[tile];
  if (tend <= start) return;
  const int nbatch = (tend - start + kBwdBatch - 1) / kBwdBatch;
  auto batch_lo = [&](int b) { return max(start, tend - kBwdBatch * (b + 1)); };
  auto batch_hi = [&](int b) { return tend - kBwdBatch * b; };
  const bool vec_feat = (a.ds & 3) == 0 && (reinterpret_cast<uintptr_t>(a.feats) & 15) == 0;
  // warp 0, lanes 0..15: stage splat `lane` of batch b (source src) into raw buffer `buf`
  auto stage = [&](int buf, int b, uint32_t src) {
    float* row = s_raw[buf] + lane * RP;
    if (lane < batch_hi(b) - batch_lo(b)) {
      const float4* rg = reinterpret_cast<const float4*>(a.rec + src);
      cp_async16(row, rg);
      cp_async16(row + 4, rg + 1);
      cp_async16(row + 8, rg + 2);
      cp_async4(row + 12, a.colors + 3 * (size_t)src);
      cp_async4(row + 13, a.colors + 3 * (size_t)src + 1);
      cp_async4(row + 14, a.colors + 3 * (size_t)src + 2);
      row[15] = __uint_as_float(src);
      const float* f = a.feats + (size_t)src * a.ds;
      if (vec_feat) {
        for (int c = 0; c < a.ds; c += 4) cp_async16(row + 16 + c, f + c);
      } else {
        for (int c = 0; c < a.ds; ++c) cp_async4(row + 16 + c, f + c);
      }
      for (int c = a.ds; c < RP - 16; ++c) row[16 + c] = 0.f;
    } else {
      for (int c = 0; c < RP; ++c) row[c] = 0.f;
      reinterpret_cast<int32_t*>(row)[8] = 1;  // empty bbox (x0 > x1)
    }
  };
  auto src_of = [&](int b) -> uint32_t {  // lanes < 16: source of splat `lane` of batch b
    if (b >= nbatch) return 0u;
    const int lo = batch_lo(b);
    return lane < batch_hi(b) - lo ? (uint32_t)a.keys[lo + lane] : 0u;
  };
  constexpr float kNegHalfLog2e = -0.72134752044448170f;  // -0.5 * log2(e)
  // split staged raw buffer `buf` into the tf32 hi/lo splat rows and per-splat terms of slot `sb`
  auto split_batch = [&](int buf, int sb) {
    const float* raw = s_raw[buf];
    for (int e = tid; e < kBwdBatch * NU; e += kTilePixels) {
      const int j = e / NU, c = e % NU;
      const float* row = raw + j * RP;
      const float v = c < 3 ? row[12 + c] : (c == 3 ? row[2] : (c - 4 < DSP ? row[16 + c - 4] : 0.f));
      uint32_t h, l;
      split_tf32(v, h, l);
      s_fh[sb][j * NUP + c] = __uint_as_float(h);
      s_fl[sb][j * NUP + c] = __uint_as_float(l);
    }
    if (tid < kBwdBatch) {
      const float* row = raw + tid * RP;
      s_sp[sb][0][tid] = make_float4(row[0], row[1], kNegHalfLog2e * row[4], kNegHalfLog2e * (2.f * row[5]));
      s_sp[sb][1][tid] = make_float4(kNegHalfLog2e * row[7], row[3], row[4], row[5]);
      int4 bb = *reinterpret_cast<const int4*>(row + 8);
      bb.y -= bb.x;
      bb.w -= bb.z;
      if (bb.y < 0 || bb.w < 0) bb = make_int4(0x3fffffff, 0, 0x3fffffff, 0);
      s_sp[sb][2][tid] = i4_as_f4(bb);
      s_sp[sb][3][tid] = make_float4(row[6], row[7], row[15], 0.f);
    }
  };
  const size_t p = inside ? (size_t)py * a.width + px : 0;
  // prologue: stage batches 0 and 1, fetch the sources of batch 2
  uint32_t nsrc = 0;
  if (warp == 0 && lane < kBwdBatch) {
    stage(0, 0, src_of(0));
    if (nbatch > 1) stage(1, 1, src_of(1));
    cp_async_commit();
    nsrc = src_of(2);
  }
  // per-pixel upstream row U[p] = [uc0, uc1, uc2, uz, uq...] (zero outside the image)
  int last = 0;
  float T = 1.f;
  {
    float uc0 = 0.f, uc1 = 0.f, uc2 = 0.f, uz = 0.f;
    if (inside) {
      if (a.d_color) {
        uc0 = a.d_color[3 * p];
        uc1 = a.d_color[3 * p + 1];
        uc2 = a.d_color[3 * p + 2];
      }
      if (a.d_depth) uz = a.d_depth[p];
      last = a.px_last[p];
      T = a.px_T[p];
    }
    s_u[uidx(tid, 0)] = uc0;
    s_u[uidx(tid, 1)] = uc1;
    s_u[uidx(tid, 2)] = uc2;
    s_u[uidx(tid, 3)] = uz;
    if constexpr (NU - (4 + DSP) == 4)  // the 4 pad columns are one swizzled float4
      *reinterpret_cast<float4*>(s_u + uidx(tid, 4 + DSP)) = make_float4(0.f, 0.f, 0.f, 0.f);
    else
#pragma unroll
      for (int c = 4 + DSP; c < NU; ++c) s_u[uidx(tid, c)] = 0.f;
    // query gradients: the tile's 16 pixel rows are contiguous runs of 16 * ds floats, read
    // cooperatively (coalesced 16-byte loads when ds % 4 == 0)
    const bool vq = a.d_query && (a.ds & 3) == 0 && (reinterpret_cast<uintptr_t>(a.d_query) & 15) == 0;
    if (vq) {
      const int q4 = a.ds / 4;
      for (int i = tid; i < kTilePixels * (DSP / 4); i += kTilePixels) {
        const int pl = i / (DSP / 4), c4 = i % (DSP / 4);
        const int qx = tx0 + tile_dx(pl), qy = ty0 + tile_dy(pl);
        float* dst = s_u + uidx(pl, 4 + 4 * c4);  // the swizzle keeps 4-column groups contiguous
        if (c4 < q4 && qx < a.width && qy < a.height)
          cp_async16(dst, reinterpret_cast<const float4*>(a.d_query) + ((size_t)qy * a.width + qx) * q4 + c4);
        else
          *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
#pragma unroll
      for (int c = 0; c < DSP; ++c)
        s_u[uidx(tid, 4 + c)] = (inside && a.d_query && c < a.ds) ? a.d_query[p * a.ds + c] : 0.f;
    }
  }
  const int warp_last = __reduce_max_sync(0xffffffffu, last);
  // this warp's pixel block: columns bx0 .. bx0 + 7, rows by0 .. by0 + 3
  const int bx0 = tx0 + (warp & 1) * 8, by0 = ty0 + (warp >> 1) * 4;
  // MMA lane coordinates
  const int g = lane >> 2, cq = lane & 3;
  // B fragments of the pixel moment matrix X[p][q] = [1, x', y', x'^2, x'y', y'^2, 0, 0] for the
  // warp's 32 pixels (k-steps of 8 pixels); x', y' are tile-centred (exact in tf32).
  uint32_t xb[4][2];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int pl = 32 * warp + 8 * ks + cq + 4 * hh;  // tile-linear pixel of this B element (row k)
      const float xx = (float)tile_dx(pl) - 7.5f, yy = (float)tile_dy(pl) - 7.5f;
      float v = 0.f;
      switch (g) {  // column n = g
        case 0: v = 1.f; break;
        case 1: v = xx; break;
        case 2: v = yy; break;
        case 3: v = xx * xx; break;
        case 4: v = xx * yy; break;
        case 5: v = yy * yy; break;
        default: v = 0.f;
      }
      xb[ks][hh] = __float_as_uint(v);
    }
  const float fx = (float)px, fy = (float)py;
  float s_after = 0.f;
  float* sw_w = s_wbase + (warp * 3 + 0) * kBwdBatch * WP;
  float* sw_r = s_wbase + (warp * 3 + 1) * kBwdBatch * WP;
  float* sw_g = s_wbase + (warp * 3 + 2) * kBwdBatch * WP;
  cp_async_wait_all();
  __syncthreads();
  split_batch(0, 0);
  __syncthreads();
  for (int it = 0; it < nbatch; ++it) {
    const int lo = batch_lo(it);
    const int cnt = batch_hi(it) - lo;
    const int cur = it & 1;
    // ======== phase 1
    // stage batch it+2 into the raw buffer batch it used (split in the previous phase 1)
    if (warp == 0 && lane < kBwdBatch && it + 2 < nbatch) {
      stage(cur, it + 2, nsrc);
      cp_async_commit();
      nsrc = src_of(it + 3);
    }
    // split batch it+1 (landed before the previous barrier) for the next phase 1
    if (it + 1 < nbatch) split_batch(cur ^ 1, cur ^ 1);
    const float* fh = s_fh[cur];
    const float* fl = s_fl[cur];
    // warp activity: some pixel of the block still blends at this batch and some bbox meets it
    uint32_t wmask = 0u;  // splats of the batch whose bbox meets the warp's block
    if ((lo - start) < warp_last) {
      bool meets = false;
      if (lane < cnt) {
        const int4 bb = f4_as_i4(s_sp[cur][2][lane]);
        meets = bb.x <= bx0 + 7 && bb.x + bb.y >= bx0 && bb.z <= by0 + 3 && bb.z + bb.w >= by0;
      }
      wmask = __ballot_sync(0xffffffffu, meets);
    }
    const bool act = wmask != 0u;
    if (lane == 0) s_wact[warp] = act ? 1 : 0;
    if (act) {
      // ---- value[p][j] = U[p] . [c_j, z_j, f_j] for the warp's 32 pixels x 16 splats on the tensor
      // cores (3xTF32), staged through sw_g as [splat][pixel] (each thread then reads its own
      // pixel's column and overwrites that slot with dg)
      {
        float va[2][2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) va[mt][nt][0] = va[mt][nt][1] = va[mt][nt][2] = va[mt][nt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < NU / 8; ++ks) {
          uint32_t uh[2][4], ul[2][4];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const int pr = 32 * warp + 16 * mt + g;
            split_tf32(s_u[uidx(pr, 8 * ks + cq)], uh[mt][0], ul[mt][0]);
            split_tf32(s_u[uidx(pr + 8, 8 * ks + cq)], uh[mt][1], ul[mt][1]);
            split_tf32(s_u[uidx(pr, 8 * ks + cq + 4)], uh[mt][2], ul[mt][2]);
            split_tf32(s_u[uidx(pr + 8, 8 * ks + cq + 4)], uh[mt][3], ul[mt][3]);
          }
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int fo = (8 * nt + g) * NUP + 8 * ks + cq;
            const uint32_t bh[2] = {__float_as_uint(fh[fo]), __float_as_uint(fh[fo + 4])};
            const uint32_t bl[2] = {__float_as_uint(fl[fo]), __float_as_uint(fl[fo + 4])};
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              mma_tf32(va[mt][nt], ul[mt], bh);
              mma_tf32(va[mt][nt], uh[mt], bl);
              mma_tf32(va[mt][nt], uh[mt], bh);
            }
          }
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int r = 8 * nt + 2 * cq, c = 16 * mt + g;
            sw_g[widx(r, c)] = va[mt][nt][0];
            sw_g[widx(r + 1, c)] = va[mt][nt][1];
            sw_g[widx(r, c + 8)] = va[mt][nt][2];
            sw_g[widx(r + 1, c + 8)] = va[mt][nt][3];
          }
        __syncwarp();
      }
      // ---- per-pixel reverse sweep over the batch. alpha' of four splats is evaluated
      // independently (ILP), then the transmittance recovery / d_alpha chain runs serially.
      // The set of blended (pixel, splat) pairs comes from the forward (px_last), so alpha' only
      // needs gradient accuracy here (SFU exp2 / reciprocal).
      const int jl = last - (lo - start);  // splats j < jl of this batch are in the pixel's blend list
#pragma unroll
      for (int j4 = kBwdBatch - 4; j4 >= 0; j4 -= 4) {
        float alv[4], ex[4], rv[4];
        bool ok[4], unc[4];
        bool any = false;
#pragma unroll
        for (int u = 3; u >= 0; --u) {
          const int j = j4 + u;
          const int4 bb = f4_as_i4(s_sp[cur][2][j]);
          ok[u] = j < jl && (unsigned)(px - bb.x) <= (unsigned)bb.y && (unsigned)(py - bb.z) <= (unsigned)bb.w;
          any |= ok[u];
        }
        if (__any_sync(0xffffffffu, any)) {
#pragma unroll
          for (int u = 3; u >= 0; --u) {
            const float4 s0 = s_sp[cur][0][j4 + u];
            const float4 s1 = s_sp[cur][1][j4 + u];
            const float dx = fx - s0.x;
            const float dy = fy - s0.y;
            const float pw = fmaf(dx, fmaf(s0.z, dx, s0.w * dy), s1.x * dy * dy);
            ex[u] = ex2_approx(pw);
            float al = s1.y * ex[u];
            unc[u] = !(al > kAlphaMax);
            if (!unc[u]) al = kAlphaMax;
            alv[u] = al;
            rv[u] = rcp_approx(1.f - al);
          }
        }
#pragma unroll
        for (int u = 3; u >= 0; --u) {
          const int j = j4 + u;
          float w = 0.f, drho = 0.f, dg = 0.f;
          if (ok[u]) {
            const float Tb = T * rv[u];
            w = alv[u] * Tb;
            const float value = sw_g[widx(j, lane)];
            const float d_alpha = Tb * value - s_after * rv[u];
            s_after = fmaf(w, value, s_after);
            if (unc[u]) {
              dg = d_alpha * ex[u];
              drho = -0.5f * alv[u] * d_alpha;
            }
            T = Tb;
          }
          sw_w[widx(j, lane)] = w;
          sw_r[widx(j, lane)] = drho;
          sw_g[widx(j, lane)] = dg;
        }
      }
      __syncwarp();
      // ---- tensor-core reductions over the warp's 32 pixels
      float dwu[NT][4];
      float dmo[2][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dwu[nt][0] = dwu[nt][1] = dwu[nt][2] = dwu[nt][3] = 0.f;
      dmo[0][0] = dmo[0][1] = dmo[0][2] = dmo[0][3] = dmo[1][0] = dmo[1][1] = dmo[1][2] = dmo[1][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        // A = W^T (rows: splats j, cols: pixels) ; split into tf32 hi/lo
        uint32_t ah[4], al_[4];
        split_tf32(sw_w[widx(g, 8 * ks + cq)], ah[0], al_[0]);
        split_tf32(sw_w[widx(g + 8, 8 * ks + cq)], ah[1], al_[1]);
        split_tf32(sw_w[widx(g, 8 * ks + cq + 4)], ah[2], al_[2]);
        split_tf32(sw_w[widx(g + 8, 8 * ks + cq + 4)], ah[3], al_[3]);
        const int prow = 32 * warp + 8 * ks + cq;  // pixel (k index) of b0; b1 is +4
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          uint32_t bh[2], bl[2];
          split_tf32(s_u[uidx(prow, 8 * nt + g)], bh[0], bl[0]);
          split_tf32(s_u[uidx(prow + 4, 8 * nt + g)], bh[1], bl[1]);
          mma_tf32(dwu[nt], ah, bh);
          mma_tf32(dwu[nt], ah, bl);
          mma_tf32(dwu[nt], al_, bh);
        }
        // A = [drho ; dg]^T (2 m-tiles), B = X (exact)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const float* src = mt ? sw_g : sw_r;
          uint32_t rh[4], rl[4];
          split_tf32(src[widx(g, 8 * ks + cq)], rh[0], rl[0]);
          split_tf32(src[widx(g + 8, 8 * ks + cq)], rh[1], rl[1]);
          split_tf32(src[widx(g, 8 * ks + cq + 4)], rh[2], rl[2]);
          split_tf32(src[widx(g + 8, 8 * ks + cq + 4)], rh[3], rl[3]);
          mma_tf32(dmo[mt], rh, xb[ks]);
          mma_tf32(dmo[mt], rl, xb[ks]);
        }
      }
      // ---- warp partials (rows = splats) into the warp's own staging area
      __syncwarp();
      float* part = sw_w;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        *reinterpret_cast<float2*>(part + g * PP + 8 * nt + 2 * cq) = make_float2(dwu[nt][0], dwu[nt][1]);
        *reinterpret_cast<float2*>(part + (g + 8) * PP + 8 * nt + 2 * cq) = make_float2(dwu[nt][2], dwu[nt][3]);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int base = NU + 8 * mt;
        *reinterpret_cast<float2*>(part + g * PP + base + 2 * cq) = make_float2(dmo[mt][0], dmo[mt][1]);
        *reinterpret_cast<float2*>(part + (g + 8) * PP + base + 2 * cq) = make_float2(dmo[mt][2], dmo[mt][3]);
      }
    }
    __syncthreads();
    // ======== phase 2: per-splat sums of the active warps' partials (fixed warp order), closed
    // forms and global accumulation. Threads [0, 4 * DSP) own one float4 feature column of one
    // splat each; warp 7 owns the geometry + colour row of every splat (two lanes per splat, one
    // per half of the warps). All partial reads are 16-byte.
    {
      int wm = 0;
#pragma unroll
      for (int w8 = 0; w8 < 8; ++w8) wm |= s_wact[w8] << w8;
      constexpr int WS = 3 * kBwdBatch * WP;  // warp stride of the partial areas
      constexpr int FC = DSP / 4;             // float4 feature columns per splat
      const int DW = det_width(a.ds);
      auto det_row = [&](int j, size_t src) -> float* {  // (splat, tile) partial row, deterministic mode
        const int4 bb = f4_as_i4(s_sp[cur][2][j]);
        const int rtx0 = bb.x / kTile, rtx1 = (bb.x + bb.y) / kTile, rty0 = bb.z / kTile;
        const int rank = (ty0 / kTile - rty0) * (rtx1 - rtx0 + 1) + (tx0 / kTile - rtx0);
        return a.pair_part + (size_t)(a.splat_off[src] + rank) * DW;
      };
      auto add4 = [](float4& v, const float* q) {
        const float4 t = *reinterpret_cast<const float4*>(q);
        v.x += t.x, v.y += t.y, v.z += t.z, v.w += t.w;
      };
      const bool vf = (a.ds & 3) == 0 && (reinterpret_cast<uintptr_t>(a.g_feat) & 15) == 0;
      for (int e = tid; e < kBwdBatch * FC; e += kTilePixels) {
        const int j = e / FC, c0 = 4 * (e % FC);
        if (j < cnt && c0 < a.ds) {
          const float* pj = s_wbase + j * PP + 4 + c0;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int w8 = 0; w8 < 8; ++w8)
            if (wm & (1 << w8)) add4(v, pj + w8 * WS);
          const size_t src = __float_as_uint(s_sp[cur][3][j].z);
          if (a.pair_part) {
            reinterpret_cast<float4*>(det_row(j, src) + 12)[c0 / 4] = v;
          } else if (vf) {
            if (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f)
              atomicAdd(reinterpret_cast<float4*>(a.g_feat + src * a.ds + c0), v);
          } else {
            const float vv[4] = {v.x, v.y, v.z, v.w};
            for (int c = 0; c < 4 && c0 + c < a.ds; ++c)
              if (vv[c] != 0.f) atomicAdd(&a.g_feat[src * a.ds + c0 + c], vv[c]);
          }
        }
      }
      if (warp == 7) {
        const int j = lane & 15, h = lane >> 4;  // lane pair (j, j + 16): warps 0-3 and 4-7
        // [c0 c1 c2 z] | drho moments M0..M3 | M4 M5 - - | dg moment, - - -
        float4 cz = make_float4(0.f, 0.f, 0.f, 0.f), ma = cz, mb = cz, mg = cz;
        const float* pj = s_wbase + j * PP;
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) {
          const int w8 = 4 * h + w4;
          if (wm & (1 << w8)) {
            const float* q = pj + w8 * WS;
            add4(cz, q);
            add4(ma, q + NU);
            add4(mb, q + NU + 4);
            add4(mg, q + NU + 8);
          }
        }
        auto xadd = [](float4& v) {
          v.x += __shfl_xor_sync(0xffffffffu, v.x, 16);
          v.y += __shfl_xor_sync(0xffffffffu, v.y, 16);
          v.z += __shfl_xor_sync(0xffffffffu, v.z, 16);
          v.w += __shfl_xor_sync(0xffffffffu, v.w, 16);
        };
        xadd(cz);
        xadd(ma);
        xadd(mb);
        mg.x += __shfl_xor_sync(0xffffffffu, mg.x, 16);
        if (h == 0 && j < cnt) {
          const float4 sp0 = s_sp[cur][0][j], sp1 = s_sp[cur][1][j], sp3 = s_sp[cur][3][j];
          const size_t src = __float_as_uint(sp3.z);
          // moments M0..M5 of the drho rows -> dmean_u, dmean_v, dA00, dA01 | dA11, dz, dg
          const float up = sp0.x - ((float)tx0 + 7.5f), vp = sp0.y - ((float)ty0 + 7.5f);
          const float m0 = ma.x, m1 = ma.y, m2 = ma.z, m3 = ma.w, m4 = mb.x, m5 = mb.y;
          const float sdx = m1 - up * m0, sdy = m2 - vp * m0;
          const float4 g0 = make_float4(-2.f * (sp1.z * sdx + sp1.w * sdy), -2.f * (sp3.x * sdx + sp3.y * sdy),
                                        m3 - 2.f * up * m1 + up * up * m0, m4 - vp * m1 - up * m2 + up * vp * m0);
          const float4 g1 = make_float4(m5 - 2.f * vp * m2 + vp * vp * m0, cz.w, mg.x, 0.f);
          if (a.pair_part) {
            float* det = det_row(j, src);
            reinterpret_cast<float4*>(det)[0] = g0;
            reinterpret_cast<float4*>(det)[1] = g1;
            det[8] = cz.x;
            det[9] = cz.y;
            det[10] = cz.z;
          } else {
            if (g0.x != 0.f || g0.y != 0.f || g0.z != 0.f || g0.w != 0.f)
              atomicAdd(reinterpret_cast<float4*>(a.geo_acc + src * 8), g0);
            if (g1.x != 0.f || g1.y != 0.f || g1.z != 0.f)
              atomicAdd(reinterpret_cast<float4*>(a.geo_acc + src * 8) + 1, g1);
            if (cz.x != 0.f) atomicAdd(&a.g_col[src * 3 + 0], cz.x);
            if (cz.y != 0.f) atomicAdd(&a.g_col[src * 3 + 1], cz.y);
            if (cz.z != 0.f) atomicAdd(&a.g_col[src * 3 + 2], cz.z);
          }
        }
      }
    }
    cp_async_wait_all();  // batch it+2 (issuing lanes of warp 0), visible after the barrier
    __syncthreads();
  }
}

struct ProjBwdArgs {
  MapPtrs map;
  MapPtrs grads;
  const SplatRec* rec;
  float* geo_acc;
  float rcw[9], rwc[9], o[3];
  float fx, fy, cx, cy;
};

// One frame's projection-backward contribution of one Gaussian (render.cpp:368-429), from the
// Gaussian's frame-independent terms (position p, normalised quaternion qh = (w, x, y, z) with its
// norm qn, rotation rg, scales sc), the frame's record (r0 = mean, depth, alpha; r1 = cov_inv)
// and accumulators ac = (dmean_u, dmean_v, dA00, dA01, dA11, dz, dg).
struct PbContrib {
  float opa, lsc[3], rot[4], pos[3];
};
__device__ __forceinline__ PbContrib proj_bwd_frame(const float* p, const float* qh, float qn, const float* rg,
                                                    const float* sc, float4 r0, float4 r1, const float* ac,
                                                    const float* rcw, const float* rwc, const float* o, float fx,
                                                    float fy) {
  PbContrib out;
  const float qw = qh[0], qx = qh[1], qy = qh[2], qz = qh[3];
  const float d0 = p[0] - o[0], d1 = p[1] - o[1], d2 = p[2] - o[2];
  float pc[3];
  for (int r = 0; r < 3; ++r) pc[r] = rcw[3 * r] * d0 + rcw[3 * r + 1] * d1 + rcw[3 * r + 2] * d2;
  float rcg[9], m[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      rcg[3 * r + c] = rcw[3 * r] * rg[c] + rcw[3 * r + 1] * rg[3 + c] + rcw[3 * r + 2] * rg[6 + c];
      m[3 * r + c] = rcg[3 * r + c] * sc[c];
    }
  float cc[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) cc[3 * r + c] = m[3 * r] * m[3 * c] + m[3 * r + 1] * m[3 * c + 1] + m[3 * r + 2] * m[3 * c + 2];
  const float x = pc[0], y = pc[1], z = pc[2];
  const float J[6] = {fx / z, 0.f, -fx * x / (z * z), 0.f, fy / z, -fy * y / (z * z)};
  const float A[4] = {r1.x, r1.y, r1.z, r1.w};  // cov_inv from the forward record (identical values)
  const float alpha = r0.w;
  out.opa = ac[6] * alpha * (1.f - alpha);
  const float dA[4] = {ac[2], ac[3], ac[3], ac[4]};
  float t1[4], dc[4];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) t1[2 * r + c] = -A[2 * r] * dA[c] - A[2 * r + 1] * dA[2 + c];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) dc[2 * r + c] = t1[2 * r] * A[c] + t1[2 * r + 1] * A[2 + c];
  float jdc[6];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 2; ++c) jdc[2 * r + c] = J[r] * dc[c] + J[3 + r] * dc[2 + c];
  float dcc[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) dcc[3 * r + c] = jdc[2 * r] * J[c] + jdc[2 * r + 1] * J[3 + c];
  float dcj[6], djac[6];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) dcj[3 * r + c] = 2.f * (dc[2 * r] * J[c] + dc[2 * r + 1] * J[3 + c]);
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) djac[3 * r + c] = dcj[3 * r] * cc[c] + dcj[3 * r + 1] * cc[3 + c] + dcj[3 * r + 2] * cc[6 + c];
  float dm_[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      dm_[3 * r + c] = 2.f * (dcc[3 * r] * m[c] + dcc[3 * r + 1] * m[3 + c] + dcc[3 * r + 2] * m[6 + c]);
  float drg[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      drg[3 * r + c] = (rcw[r] * dm_[c] + rcw[3 + r] * dm_[3 + c] + rcw[6 + r] * dm_[6 + c]) * sc[c];
  for (int c = 0; c < 3; ++c) out.lsc[c] = (rcg[c] * dm_[c] + rcg[3 + c] * dm_[3 + c] + rcg[6 + c] * dm_[6 + c]) * sc[c];
  const float dw[9] = {0.f, -qz, qy, qz, 0.f, -qx, -qy, qx, 0.f};
  const float dxm[9] = {0.f, qy, qz, qy, -2.f * qx, -qw, qz, qw, -2.f * qx};
  const float dym[9] = {-2.f * qy, qx, qw, qx, 0.f, qz, -qw, qz, -2.f * qy};
  const float dzm[9] = {-2.f * qz, -qw, qx, qw, -2.f * qz, qy, qx, qy, 0.f};
  float dq[4] = {0.f, 0.f, 0.f, 0.f};
  for (int r = 0; r < 9; ++r) {
    dq[0] += dw[r] * drg[r];
    dq[1] += dxm[r] * drg[r];
    dq[2] += dym[r] * drg[r];
    dq[3] += dzm[r] * drg[r];
  }
  for (int r = 0; r < 4; ++r) dq[r] *= 2.f;
  const float qd = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
  for (int r = 0; r < 4; ++r) out.rot[r] = (dq[r] - qh[r] * qd) / qn;
  float dp[3] = {0.f, 0.f, 0.f};
  const float z2 = z * z, z3 = z2 * z;
  dp[0] += ac[0] * fx / z;
  dp[2] += ac[0] * (-fx * x / z2);
  dp[1] += ac[1] * fy / z;
  dp[2] += ac[1] * (-fy * y / z2);
  dp[0] += djac[2] * (-fx / z2);
  dp[1] += djac[5] * (-fy / z2);
  dp[2] += djac[0] * (-fx / z2) + djac[2] * (2.f * fx * x / z3) + djac[4] * (-fy / z2) + djac[5] * (2.f * fy * y / z3);
  dp[2] += ac[5];
  for (int r = 0; r < 3; ++r) out.pos[r] = rwc[3 * r] * dp[0] + rwc[3 * r + 1] * dp[1] + rwc[3 * r + 2] * dp[2];
  return out;
}

// The frame-independent terms of a Gaussian: normalised quaternion, its rotation, scales.
__device__ __forceinline__ void proj_bwd_common(const float* q, const float* ls, float* qh, float& qn, float* rg,
                                                float* sc) {
  qn = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const float qw = q[0] / qn, qx = q[1] / qn, qy = q[2] / qn, qz = q[3] / qn;
  qh[0] = qw, qh[1] = qx, qh[2] = qy, qh[3] = qz;
  rg[0] = 1.f - 2.f * (qy * qy + qz * qz), rg[1] = 2.f * (qx * qy - qw * qz), rg[2] = 2.f * (qx * qz + qw * qy);
  rg[3] = 2.f * (qx * qy + qw * qz), rg[4] = 1.f - 2.f * (qx * qx + qz * qz), rg[5] = 2.f * (qy * qz - qw * qx);
  rg[6] = 2.f * (qx * qz - qw * qy), rg[7] = 2.f * (qy * qz + qw * qx), rg[8] = 1.f - 2.f * (qx * qx + qy * qy);
  sc[0] = expf(ls[0]), sc[1] = expf(ls[1]), sc[2] = expf(ls[2]);
}

// K9: projection backward (render.cpp:368-429), one thread per Gaussian. The gradient adds
// are __fadd_rn (no contraction), so the multi-frame kernel below reproduces them bit for bit.
__global__ void __launch_bounds__(256, 4) project_bwd_kernel(ProjBwdArgs a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= a.map.n) return;
  const float4* rv = reinterpret_cast<const float4*>(a.rec + i);
  // every load is issued before the culled test (one memory round trip instead of two; a culled
  // Gaussian's extra bytes cost less than the serialised latency): 16-byte loads of the record,
  // the accumulators (re-zeroed below for the next frame), the quaternion
  const int4 bb = reinterpret_cast<const int4*>(a.rec + i)[2];
  const float4 r0 = ld_early4(rv), r1 = ld_early4(rv + 1);
  float4* acc4 = reinterpret_cast<float4*>(a.geo_acc + 8 * i);
  const float4 g0 = ld_early4(acc4), g1 = ld_early4(acc4 + 1);
  const float ac[7] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z};
  const float pv[3] = {ld_early(a.map.pos + 3 * i), ld_early(a.map.pos + 3 * i + 1), ld_early(a.map.pos + 3 * i + 2)};
  const float4 q4 = (reinterpret_cast<uintptr_t>(a.map.rot) & 15) == 0
                        ? ld_early4(reinterpret_cast<const float4*>(a.map.rot) + i)
                        : make_float4(a.map.rot[4 * i], a.map.rot[4 * i + 1], a.map.rot[4 * i + 2], a.map.rot[4 * i + 3]);
  const float lv[3] = {ld_early(a.map.lsc + 3 * i), ld_early(a.map.lsc + 3 * i + 1), ld_early(a.map.lsc + 3 * i + 2)};
  const float q[4] = {q4.x, q4.y, q4.z, q4.w};
  // the gradient read-modify-writes: loads issued here, independent of the math below
  const float go = ld_early(a.grads.opa + i);
  const float gl[3] = {ld_early(a.grads.lsc + 3 * i), ld_early(a.grads.lsc + 3 * i + 1), ld_early(a.grads.lsc + 3 * i + 2)};
  const float gr[4] = {ld_early(a.grads.rot + 4 * i), ld_early(a.grads.rot + 4 * i + 1), ld_early(a.grads.rot + 4 * i + 2),
                       ld_early(a.grads.rot + 4 * i + 3)};
  const float gp[3] = {ld_early(a.grads.pos + 3 * i), ld_early(a.grads.pos + 3 * i + 1), ld_early(a.grads.pos + 3 * i + 2)};
  // culled (empty bbox): no accumulation happened, nothing is written. The test only guards the
  // stores, so the loads above are all in flight together
  const bool vis = bb.x <= bb.y;
  if (!vis) return;
  acc4[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  acc4[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  float qh[4], qn, rg[9], sc[3];
  proj_bwd_common(q, lv, qh, qn, rg, sc);
  const PbContrib c = proj_bwd_frame(pv, qh, qn, rg, sc, r0, r1, ac, a.rcw, a.rwc, a.o, a.fx, a.fy);
  a.grads.opa[i] = __fadd_rn(go, c.opa);
  for (int k = 0; k < 3; ++k) a.grads.lsc[3 * i + k] = __fadd_rn(gl[k], c.lsc[k]);
  for (int k = 0; k < 4; ++k) a.grads.rot[4 * i + k] = __fadd_rn(gr[k], c.rot[k]);
  for (int k = 0; k < 3; ++k) a.grads.pos[3 * i + k] = __fadd_rn(gp[k], c.pos[k]);
}

// K9 over a step's frames at once: the gradients are read and written once, with the same float
// additions in the same order as frame-by-frame K9.
constexpr int kPbFrames = 8;
struct ProjBwdMultiArgs {
  MapPtrs map;
  MapPtrs grads;
  int nf;
  const SplatRec* rec[kPbFrames];
  float* geo_acc[kPbFrames];
  float rcw[kPbFrames][9], rwc[kPbFrames][9], o[kPbFrames][3];
  float fx[kPbFrames], fy[kPbFrames];
};
// One thread per Gaussian, frames in order; the next frame's record and accumulators are loaded
// while the current frame's contribution is computed.
__global__ void __launch_bounds__(256, 3) project_bwd_multi_kernel(ProjBwdMultiArgs a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= a.map.n) return;
  const float pv[3] = {ld_early(a.map.pos + 3 * i), ld_early(a.map.pos + 3 * i + 1), ld_early(a.map.pos + 3 * i + 2)};
  const float4 q4 = (reinterpret_cast<uintptr_t>(a.map.rot) & 15) == 0
                        ? ld_early4(reinterpret_cast<const float4*>(a.map.rot) + i)
                        : make_float4(a.map.rot[4 * i], a.map.rot[4 * i + 1], a.map.rot[4 * i + 2], a.map.rot[4 * i + 3]);
  const float lv[3] = {ld_early(a.map.lsc + 3 * i), ld_early(a.map.lsc + 3 * i + 1), ld_early(a.map.lsc + 3 * i + 2)};
  const float q[4] = {q4.x, q4.y, q4.z, q4.w};
  float go = ld_early(a.grads.opa + i);
  float gl[3] = {ld_early(a.grads.lsc + 3 * i), ld_early(a.grads.lsc + 3 * i + 1), ld_early(a.grads.lsc + 3 * i + 2)};
  float gr[4] = {ld_early(a.grads.rot + 4 * i), ld_early(a.grads.rot + 4 * i + 1), ld_early(a.grads.rot + 4 * i + 2),
                 ld_early(a.grads.rot + 4 * i + 3)};
  float gp[3] = {ld_early(a.grads.pos + 3 * i), ld_early(a.grads.pos + 3 * i + 1), ld_early(a.grads.pos + 3 * i + 2)};
  float qh[4], qn, rg[9], sc[3];
  proj_bwd_common(q, lv, qh, qn, rg, sc);
  bool any = false;
  auto load = [&](int b, int4& bb, float4& r0, float4& r1, float4& g0, float4& g1) {
    const float4* rv = reinterpret_cast<const float4*>(a.rec[b] + i);
    bb = reinterpret_cast<const int4*>(a.rec[b] + i)[2];
    r0 = ld_early4(rv);
    r1 = ld_early4(rv + 1);
    const float4* acc4 = reinterpret_cast<const float4*>(a.geo_acc[b] + 8 * i);
    g0 = ld_early4(acc4);
    g1 = ld_early4(acc4 + 1);
  };
  int4 bb;
  float4 r0, r1, g0, g1;
  load(0, bb, r0, r1, g0, g1);
  for (int b = 0; b < a.nf; ++b) {
    int4 nbb = bb;
    float4 nr0 = r0, nr1 = r1, ng0 = g0, ng1 = g1;
    if (b + 1 < a.nf) load(b + 1, nbb, nr0, nr1, ng0, ng1);
    if (bb.x <= bb.y) {  // visible in frame b
      any = true;
      float4* acc4 = reinterpret_cast<float4*>(a.geo_acc[b] + 8 * i);
      acc4[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      acc4[1] = make_float4(0.f, 0.f, 0.f, 0.f);
      const float ac[7] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z};
      const PbContrib c = proj_bwd_frame(pv, qh, qn, rg, sc, r0, r1, ac, a.rcw[b], a.rwc[b], a.o[b], a.fx[b], a.fy[b]);
      go = __fadd_rn(go, c.opa);
      for (int k = 0; k < 3; ++k) gl[k] = __fadd_rn(gl[k], c.lsc[k]);
      for (int k = 0; k < 4; ++k) gr[k] = __fadd_rn(gr[k], c.rot[k]);
      for (int k = 0; k < 3; ++k) gp[k] = __fadd_rn(gp[k], c.pos[k]);
    }
    bb = nbb, r0 = nr0, r1 = nr1, g0 = ng0, g1 = ng1;
  }
  if (!any) return;
  a.grads.opa[i] = go;
  for (int k = 0; k < 3; ++k) a.grads.lsc[3 * i + k] = gl[k];
  for (int k = 0; k < 4; ++k) a.grads.rot[4 * i + k] = gr[k];
  for (int k = 0; k < 3; ++k) a.grads.pos[3 * i + k] = gp[k];
}

// project_gaussian (render.cpp:118-132): one Gaussian, returns cov2d (not its inverse).
__global__ void project_single_kernel(const float* in, Cam cam, float* out) {
  const float* p = in;
  const float* q = in + 3;
  const float* ls = in + 7;
  const float logit = in[10];
  SplatRec r;
  float cv[4];
  const bool ok = project_exact(p, q, ls, logit, cam, r, cv);
  out[0] = ok ? 1.f : 0.f;
  if (!ok) return;
  out[1] = r.mean_x;
  out[2] = r.mean_y;
  for (int i = 0; i < 4; ++i) out[3 + i] = cv[i];
  out[7] = r.depth;
}

template <int DSP>
void launch_fwd(cudaStream_t st, int ntiles, const RasterArgs& a, bool exact) {
  if (exact) {
    raster_fwd_kernel<DSP, true><<<ntiles, kTilePixels, 0, st>>>(a);
  } else if constexpr (DSP >= 8) {
    const size_t smem = sizeof(float) * (2 * 128 * (DSP + 8) + 8 * 16 * 40 + 128 * (16 + (DSP + 3) / 4 * 4));
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(raster_fwd_mma_kernel<DSP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    raster_fwd_mma_kernel<DSP><<<ntiles, kTilePixels, smem, st>>>(a);
  } else {
    raster_fwd_kernel<DSP, false><<<ntiles, kTilePixels, 0, st>>>(a);
  }
}
template <int DSP>
void launch_bwd(cudaStream_t st, int ntiles, const RasterBwdArgs& a) {
  constexpr int NU = ((4 + DSP) + 7) / 8 * 8;
  constexpr int UP = NU % 16 == 8 ? NU : NU + 8;
  constexpr int NACC = NU + 16, PP = (NACC + 23) / 32 * 32 + 8;
  constexpr int WP = 16 * PP <= 3 * kBwdBatch * 32 ? 32 : 36;  // as in raster_bwd_kernel
  const size_t smem = sizeof(float) * ((size_t)kTilePixels * UP + 8 * 3 * kBwdBatch * WP);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(raster_bwd_kernel<DSP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  raster_bwd_kernel<DSP><<<ntiles, kTilePixels, smem, st>>>(a);
}

int pad_ds(int ds) {
  if (ds <= 4) return 4;
  if (ds <= 8) return 8;
  if (ds <= 16) return 16;
  if (ds <= 32) return 32;
  if (ds <= 64) return 64;
  return -1;
}

}  // namespace

void project_single(cudaStream_t st, const float* d_in11, const float rot_cw[9], const float origin[3],
                    const Intr& intr, float* d_out8) {
  Cam cam;
  for (int i = 0; i < 9; ++i) cam.r[i] = rot_cw[i];
  for (int i = 0; i < 3; ++i) cam.o[i] = origin[i];
  cam.intr = intr;
  cam.tiles_x = cam.tiles_y = 1;
  project_single_kernel<<<1, 1, 0, st>>>(d_in11, cam, d_out8);
  count_launch();
}

void render_forward(cudaStream_t st, const MapPtrs& map, const float rot_cw[9], const float origin[3],
                    const Intr& intr, RenderWork& w, float* color, float* depth, float* query, float* alpha,
                    bool zero_outputs, bool count_only, bool blend, bool exact) {
  Cam cam;
  for (int i = 0; i < 9; ++i) cam.r[i] = rot_cw[i];
  for (int i = 0; i < 3; ++i) cam.o[i] = origin[i];
  cam.intr = intr;
  cam.tiles_x = w.tiles_x;
  cam.tiles_y = w.tiles_y;
  const int ntiles = w.tiles_x * w.tiles_y;
  const size_t npx = (size_t)intr.width * intr.height;
  cudaMemsetAsync(w.tile_count, 0, sizeof(int32_t) * ntiles, st);
  cudaMemsetAsync(w.counters, 0, sizeof(int64_t) * 8, st);
  if (zero_outputs) {
    cudaMemsetAsync(color, 0, sizeof(float) * npx * 3, st);
    cudaMemsetAsync(depth, 0, sizeof(float) * npx, st);
    cudaMemsetAsync(query, 0, sizeof(float) * npx * map.ds, st);
    cudaMemsetAsync(alpha, 0, sizeof(float) * npx, st);
  }
  const int grid1 = 148 * 4;  // 64 registers: 4 CTAs of 256 per SM
  const size_t hist_smem = ntiles <= kHistMax ? sizeof(int32_t) * ntiles : 0;
  if (map.n > 0) {
    project_kernel<<<grid1, 256, hist_smem, st>>>(map, cam, w.rec, w.dkey, w.tile_count, w.counters);
    count_launch();
  }
  scan_tiles_kernel<<<1, 1024, 0, st>>>(w.tile_count, w.tile_offset, w.tile_cursor, ntiles, w.counters, w.pair_cap,
                                        w.step_overflow, w.tile_order);
  count_launch();
  if (count_only) return;
  if (map.n > 0) {
    const size_t sc_smem = sizeof(int32_t) * 2 * ntiles;
    static bool sc_attr = false;
    if (!sc_attr) {
      cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4 * kHistMax);
      sc_attr = true;
    }
    const unsigned sc_grid =
        (unsigned)((map.n + kScatterThreads * kScatterPerThread - 1) / (kScatterThreads * kScatterPerThread));
    scatter_kernel<<<sc_grid, kScatterThreads, sc_smem, st>>>(w.rec, w.dkey, map.n, w.tiles_x, ntiles, w.tile_cursor, w.keys,
                                                 w.pair_cap, w.big, w.counters);
    scatter_big_kernel<<<148 * 4, 256, 0, st>>>(w.rec, w.dkey, w.big, w.counters, w.tiles_x, w.tile_cursor, w.keys,
                                                w.pair_cap);
    count_launch(2);
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tile_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSortSmem);
    attr_set = true;
  }
  tile_sort_kernel<<<ntiles, kSortThreads, kTileSortSmem, st>>>(w.tile_offset, w.keys, w.keys_tmp, w.pair_cap,
                                                              w.counters);
  count_launch();
  if (!blend) return;
  render_blend(st, map, intr, w, color, depth, query, alpha, exact);
}

void render_blend(cudaStream_t st, const MapPtrs& map, const Intr& intr, RenderWork& w, float* color, float* depth,
                  float* query, float* alpha, bool exact) {
  const int ntiles = w.tiles_x * w.tiles_y;
  RasterArgs a{w.rec, map.col, map.feat, map.ds, w.tile_offset, w.keys, w.tiles_x, intr.width, intr.height,
               color, depth, query, alpha, w.px_last, w.px_T, w.tile_max_last, w.counters, w.tile_order};
  switch (pad_ds(map.ds)) {
    case 4: launch_fwd<4>(st, ntiles, a, exact); break;
    case 8: launch_fwd<8>(st, ntiles, a, exact); break;
    case 16: launch_fwd<16>(st, ntiles, a, exact); break;
    case 32: launch_fwd<32>(st, ntiles, a, exact); break;
    case 64: launch_fwd<64>(st, ntiles, a, exact); break;
    default: break;
  }
  count_launch();
}

// ---- deterministic backward (K8 writes per-(splat, tile) partial rows; these kernels place and
// reduce them in a fixed order: a splat's tiles in row-major order of its tile rectangle)
__global__ void det_count_kernel(const SplatRec* __restrict__ rec, int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 bb = reinterpret_cast<const int4*>(rec + i)[2];
    cnt[i] = (bb.x > bb.y || bb.z > bb.w) ? 0
                                           : (int64_t)(bb.y / kTile - bb.x / kTile + 1) * (bb.w / kTile - bb.z / kTile + 1);
  }
}
// exclusive scan in place, 1024 elements per block: local scan + block totals
__global__ void __launch_bounds__(1024) det_scan_local_kernel(int64_t* __restrict__ v, int64_t n,
                                                               int64_t* __restrict__ block_sum) {
  __shared__ int64_t s[1024];
  const int64_t i = blockIdx.x * 1024 + threadIdx.x;
  const int64_t x = i < n ? v[i] : 0;
  s[threadIdx.x] = x;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t t = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  if (i < n) v[i] = s[threadIdx.x] - x;
  if (threadIdx.x == 1023) block_sum[blockIdx.x] = s[1023];
}
__global__ void det_scan_blocks_kernel(int64_t* block_sum, int64_t nb) {  // one thread: nb is small
  int64_t run = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t x = block_sum[b];
    block_sum[b] = run;
    run += x;
  }
}
__global__ void det_scan_add_kernel(int64_t* __restrict__ v, int64_t n, const int64_t* __restrict__ block_sum) {
  const int64_t i = blockIdx.x * 1024 + threadIdx.x;
  if (i < n) v[i] += block_sum[blockIdx.x];
}
// per (splat, float4 slot): sum the splat's rows in order; geo -> geo_acc (store), colour and
// features added into the map gradients (one writer per element)
__global__ void det_reduce_kernel(const float* __restrict__ part, const int64_t* __restrict__ off,
                                  const int64_t* __restrict__ cnt, int64_t n, int ds, float* __restrict__ geo_acc,
                                  float* __restrict__ g_col, float* __restrict__ g_feat) {
  const int DW = det_width(ds), slots = DW / 4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * slots; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / slots;
    const int q = (int)(e % slots);
    const int64_t c = cnt[i];
    if (c == 0) continue;
    const float4* p = reinterpret_cast<const float4*>(part + (size_t)off[i] * DW) + q;
    float4 acc = p[0];
    for (int64_t r = 1; r < c; ++r) {
      const float4 v = p[(size_t)r * (DW / 4)];
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
    if (q < 2) {
      reinterpret_cast<float4*>(geo_acc + i * 8)[q] = acc;
    } else if (q == 2) {
      g_col[i * 3 + 0] += acc.x, g_col[i * 3 + 1] += acc.y, g_col[i * 3 + 2] += acc.z;
    } else {
      const int c0 = 4 * (q - 3);
      const float vv[4] = {acc.x, acc.y, acc.z, acc.w};
      for (int k = 0; k < 4 && c0 + k < ds; ++k) g_feat[i * ds + c0 + k] += vv[k];
    }
  }
}

namespace {
thread_local bool t_deterministic = false;
}
void set_deterministic(bool on) { t_deterministic = on; }
bool deterministic() { return t_deterministic; }

cudaError_t DetScratch::ensure(int64_t n, int64_t pairs, int ds) {
  cudaError_t e = cudaSuccess;
  if (n > n_cap) {
    if (cnt) cudaFree(cnt), cnt = nullptr;
    if (off) cudaFree(off), off = nullptr;
    if (blocks) cudaFree(blocks), blocks = nullptr;
    n_cap = 0;
    const int64_t nb = (n + 1023) / 1024;
    if ((e = cudaMalloc(&cnt, sizeof(int64_t) * n)) || (e = cudaMalloc(&off, sizeof(int64_t) * n)) ||
        (e = cudaMalloc(&blocks, sizeof(int64_t) * nb)))
      return e;
    n_cap = n;
  }
  const int64_t need = pairs * det_width(ds);
  if (need > part_cap) {
    if (part) cudaFree(part), part = nullptr;
    part_cap = 0;
    if ((e = cudaMalloc(&part, sizeof(float) * need))) return e;
    part_cap = need;
  }
  return e;
}

void DetScratch::release() {
  for (void* p : {(void*)cnt, (void*)off, (void*)blocks, (void*)part})
    if (p) cudaFree(p);
  cnt = off = blocks = nullptr;
  part = nullptr;
  n_cap = part_cap = 0;
}

void render_backward(cudaStream_t st, const MapPtrs& map, const float rot_cw[9], const float rot_wc[9],
                     const float origin[3], const Intr& intr, const RenderWork& w, const float* d_color,
                     const float* d_depth, const float* d_query, float* geo_acc, const MapPtrs& grads,
                     bool project, DetScratch* det) {
  const int ntiles = w.tiles_x * w.tiles_y;
  RasterBwdArgs a{w.rec, map.col, map.feat, map.ds, w.tile_offset, w.keys, w.tiles_x, intr.width, intr.height,
                  w.px_last, w.px_T, w.tile_max_last, d_color, d_depth, d_query, geo_acc, grads.col, grads.feat,
                  w.tile_order, w.counters, nullptr, nullptr};
  if (det && map.n > 0) {
    // rows of every (splat, tile) pair (capacity: the tile-pair arrays), zeroed: pairs no tile
    // processed (beyond a tile's last blended entry, empty tiles) contribute nothing
    if (det->ensure(map.n, w.pair_cap, map.ds) != cudaSuccess) {
      set_sticky_error("render_backward: deterministic scratch allocation failed");
      return;
    }
    const unsigned g = (unsigned)std::min<int64_t>((map.n + 255) / 256, 148 * 8);
    det_count_kernel<<<g, 256, 0, st>>>(w.rec, map.n, det->cnt);
    cudaMemcpyAsync(det->off, det->cnt, sizeof(int64_t) * map.n, cudaMemcpyDeviceToDevice, st);
    const int64_t nb = (map.n + 1023) / 1024;
    det_scan_local_kernel<<<(unsigned)nb, 1024, 0, st>>>(det->off, map.n, det->blocks);
    det_scan_blocks_kernel<<<1, 1, 0, st>>>(det->blocks, nb);
    det_scan_add_kernel<<<(unsigned)nb, 1024, 0, st>>>(det->off, map.n, det->blocks);
    cudaMemsetAsync(det->part, 0, sizeof(float) * w.pair_cap * det_width(map.ds), st);
    count_launch(4);
    a.pair_part = det->part;
    a.splat_off = det->off;
  }
  switch (pad_ds(map.ds)) {
    case 4: launch_bwd<4>(st, ntiles, a); break;
    case 8: launch_bwd<8>(st, ntiles, a); break;
    case 16: launch_bwd<16>(st, ntiles, a); break;
    case 32: launch_bwd<32>(st, ntiles, a); break;
    case 64: launch_bwd<64>(st, ntiles, a); break;
    default: break;
  }
  count_launch();
  if (a.pair_part) {
    const int64_t work = map.n * (det_width(map.ds) / 4);
    det_reduce_kernel<<<(unsigned)std::min<int64_t>((work + 255) / 256, 148 * 16), 256, 0, st>>>(
        det->part, det->off, det->cnt, map.n, map.ds, geo_acc, grads.col, grads.feat);
    count_launch();
  }
  if (!project) return;
  render_project_backward(st, map, rot_cw, rot_wc, origin, intr, w, geo_acc, grads);
}

void render_project_backward_multi(cudaStream_t st, const MapPtrs& map, int nf, const float* const* rot_cw,
                                   const float* const* rot_wc, const float* const* origin, const Intr& intr,
                                   const RenderWork* const* w, float* const* geo_acc, const MapPtrs& grads) {
  if (map.n <= 0) return;
  for (int f0 = 0; f0 < nf; f0 += kPbFrames) {
    ProjBwdMultiArgs pa;
    pa.map = map;
    pa.grads = grads;
    pa.nf = std::min(kPbFrames, nf - f0);
    for (int b = 0; b < pa.nf; ++b) {
      pa.rec[b] = w[f0 + b]->rec;
      pa.geo_acc[b] = geo_acc[f0 + b];
      for (int i = 0; i < 9; ++i) pa.rcw[b][i] = rot_cw[f0 + b][i], pa.rwc[b][i] = rot_wc[f0 + b][i];
      for (int i = 0; i < 3; ++i) pa.o[b][i] = origin[f0 + b][i];
      pa.fx[b] = intr.fx;
      pa.fy[b] = intr.fy;
    }
    project_bwd_multi_kernel<<<(unsigned)((map.n + 255) / 256), 256, 0, st>>>(pa);
    count_launch();
  }
}

void render_project_backward(cudaStream_t st, const MapPtrs& map, const float rot_cw[9], const float rot_wc[9],
                             const float origin[3], const Intr& intr, const RenderWork& w, float* geo_acc,
                             const MapPtrs& grads) {
  if (map.n > 0) {
    ProjBwdArgs pa;
    pa.map = map;
    pa.grads = grads;
    pa.rec = w.rec;
    pa.geo_acc = geo_acc;
    for (int i = 0; i < 9; ++i) {
      pa.rcw[i] = rot_cw[i];
      pa.rwc[i] = rot_wc[i];
    }
    for (int i = 0; i < 3; ++i) pa.o[i] = origin[i];
    pa.fx = intr.fx;
    pa.fy = intr.fy;
    pa.cx = intr.cx;
    pa.cy = intr.cy;
    project_bwd_kernel<<<(unsigned)((map.n + 255) / 256), 256, 0, st>>>(pa);
    count_launch();
  }
}

}  // namespace lm
