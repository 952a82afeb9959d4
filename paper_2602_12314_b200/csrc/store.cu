// store.cu — voxel-hash global map store and the active-set gather / scatter (K11).
//
// Reference: voxel_of / hash_voxel / VoxelHashStore / insert_global (proj/src/voxel_hash.cpp:9-115)
// and fetch_local / sync (proj/src/active_set.cpp:7-128).
//
// The global record pool lives in pinned, device-mapped host memory (the host-resident
// global map); a device mirror of the record positions serves the radius scans. The hash
// table stays on the host and is probed sequentially (insertion order defines record indices
// and duplicate / overflow rejections, voxel_hash.cpp:35-71), with voxel keys and hashes for a
// batch computed on the device (double-precision floor, wrapping u32 multiply / xor, u64 mod).
// fetch_local / the fetch step of sync are a device radius test (the reference's float op
// order, no FMA) over the whole pool mirror with an order-preserving compaction, and the
// gather reads the selected records from mapped host memory straight into device buffers;
// the writeback scatter writes device records back into the pinned pool.
#include <algorithm>
#include <chrono>
#include <functional>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/latmap_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace lm {

namespace {

constexpr int kProbeLimit = 8;

__host__ __device__ inline void voxel_of(const float* p, float vs, int32_t* k) {
  k[0] = (int32_t)floor((double)p[0] / (double)vs);
  k[1] = (int32_t)floor((double)p[1] / (double)vs);
  k[2] = (int32_t)floor((double)p[2] / (double)vs);
}
__host__ __device__ inline int64_t hash_voxel(const int32_t* k, int64_t cap) {
  const uint32_t h = ((uint32_t)k[0] * 73856093u) ^ ((uint32_t)k[1] * 19349663u) ^ ((uint32_t)k[2] * 83492791u);
  return (int64_t)((uint64_t)h % (uint64_t)cap);
}

// K11a: keys and home slots of a batch of records (AoS, rs floats each, position first).
__global__ void keys_kernel(const float* __restrict__ recs, int64_t n, int rs, float vs, int64_t cap,
                            int32_t* __restrict__ keys, int64_t* __restrict__ home) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k[3];
    voxel_of(recs + i * rs, vs, k);
    keys[3 * i] = k[0];
    keys[3 * i + 1] = k[1];
    keys[3 * i + 2] = k[2];
    home[i] = hash_voxel(k, cap);
  }
}

// Radius test in the reference's float order: dx*dx + dy*dy + dz*dz <= r2 (active_set.cpp:16-19).
__device__ __forceinline__ bool in_radius(const float* p, float cx, float cy, float cz, float r2) {
  const float dx = fs(p[0], cx), dy = fs(p[1], cy), dz = fs(p[2], cz);
  return fa(fa(fm(dx, dx), fm(dy, dy)), fm(dz, dz)) <= r2;
}

// K11b: per-block counts of in-radius, not-present pool records.
constexpr int kScanBlock = 1024;
__global__ void __launch_bounds__(kScanBlock) radius_count_kernel(const float* __restrict__ pos, int64_t n, float cx,
                                                                   float cy, float cz, float r2,
                                                                   const uint8_t* __restrict__ present,
                                                                   int32_t* __restrict__ block_counts) {
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  const bool hit = i < n && (!present || !present[i]) && in_radius(pos + 3 * i, cx, cy, cz, r2);
  const int c = __syncthreads_count(hit);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = c;
}

// K11c: exclusive scan of the block counts (one block of 1024 threads, chunks of 1024 counts:
// warp shuffles, then one scan of the 32 warp totals).
__global__ void __launch_bounds__(1024) block_scan_kernel(int32_t* counts, int64_t nblocks, int64_t* total) {
  __shared__ int64_t s_w[32];
  __shared__ int64_t s_carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nblocks; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nblocks ? counts[i] : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t y = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += t;
      }
      s_w[lane] = y;  // inclusive warp totals
    }
    __syncthreads();
    const int64_t carry = s_carry;
    const int64_t excl = carry + (w ? s_w[w - 1] : 0) + x - v;
    if (i < nblocks) counts[i] = (int32_t)excl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_w[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s_carry;
}

// K11d: order-preserving compaction of the hits (ascending record index).
__global__ void __launch_bounds__(kScanBlock) radius_emit_kernel(const float* __restrict__ pos, int64_t n, float cx,
                                                                  float cy, float cz, float r2,
                                                                  const uint8_t* __restrict__ present,
                                                                  const int32_t* __restrict__ block_offsets,
                                                                  int64_t* __restrict__ out) {
  __shared__ int32_t s_warp[kScanBlock / 32];
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  const bool hit = i < n && (!present || !present[i]) && in_radius(pos + 3 * i, cx, cy, cz, r2);
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_warp[w] = __popc(m);
  __syncthreads();
  if (w == 0) {
    int v = s_warp[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    s_warp[lane] = v - s_warp[lane];  // exclusive
  }
  __syncthreads();
  if (hit) out[block_offsets[blockIdx.x] + s_warp[w] + __popc(m & ((1u << lane) - 1u))] = i;
}

// K11b' single-pass radius compaction (decoupled look-back): each block takes the next ticket,
// tests kRcEach consecutive records per thread (kRcPer per block), publishes its hit count, adds the
// counts of the blocks before it (flag P: inclusive prefix, A: own count only) and emits its hits
// in ascending record order. status[] (one word per block: flag << 62 | value) and the ticket
// are zeroed before the launch; the last block writes the total.
constexpr int kRcThreads = 512, kRcEach = 8, kRcPer = kRcEach * kRcThreads;
__global__ void __launch_bounds__(kRcThreads) radius_compact_kernel(const float* __restrict__ pos, int64_t n, float cx,
                                                                    float cy, float cz, float r2,
                                                                    const uint8_t* __restrict__ present,
                                                                    unsigned long long* status, int* ticket,
                                                                    int64_t* __restrict__ out, int64_t* total) {
  __shared__ int s_bid;
  __shared__ int32_t s_warp[kRcThreads / 32];
  __shared__ long long s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t bid = s_bid;
  const int64_t i0 = bid * kRcPer + kRcEach * (int64_t)tid;
  bool hit[kRcEach];
  if (i0 + kRcEach - 1 < n) {
    const float4* p4 = reinterpret_cast<const float4*>(pos + 3 * i0);
    float v[3 * kRcEach];
#pragma unroll
    for (int q = 0; q < 3 * kRcEach / 4; ++q) {
      const float4 t = p4[q];
      v[4 * q] = t.x, v[4 * q + 1] = t.y, v[4 * q + 2] = t.z, v[4 * q + 3] = t.w;
    }
#pragma unroll
    for (int k = 0; k < kRcEach; ++k) hit[k] = (!present || !present[i0 + k]) && in_radius(v + 3 * k, cx, cy, cz, r2);
  } else {
#pragma unroll
    for (int k = 0; k < kRcEach; ++k)
      hit[k] = i0 + k < n && (!present || !present[i0 + k]) && in_radius(pos + 3 * (i0 + k), cx, cy, cz, r2);
  }
  int c = 0;
#pragma unroll
  for (int k = 0; k < kRcEach; ++k) c += (int)hit[k];
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int y = lane < kRcThreads / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    if (lane < kRcThreads / 32) s_warp[lane] = y;  // inclusive warp totals
  }
  __syncthreads();
  const int agg = s_warp[kRcThreads / 32 - 1];
  constexpr unsigned long long kA = 1ull << 62, kP = 2ull << 62, kMask = (1ull << 62) - 1;
  if (tid == 0) atomicExch(&status[bid], (bid == 0 ? kP : kA) | (unsigned long long)agg);
  if (w == 0 && bid > 0) {  // warp look-back over windows of 32 predecessors
    long long prefix = 0;
    for (int64_t j = bid - 1;;) {
      const int64_t jj = j - lane;
      const unsigned long long st = jj >= 0 ? atomicAdd(&status[jj], 0ull) : kP;  // before block 0: P, 0
      const unsigned f = (unsigned)(st >> 62);
      if (__any_sync(0xffffffffu, f == 0)) continue;  // a predecessor has not published yet
      const unsigned pm = __ballot_sync(0xffffffffu, f == 2);
      const int first = pm ? __ffs(pm) - 1 : 32;  // the nearest predecessor with an inclusive prefix
      long long v = lane <= first ? (long long)(st & kMask) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      prefix += v;
      if (pm) break;
      j -= 32;
    }
    if (lane == 0) {
      atomicExch(&status[bid], kP | (unsigned long long)(prefix + agg));
      s_prefix = prefix;
    }
  } else if (tid == 0) {
    s_prefix = 0;
  }
  if (tid == 0 && (bid + 1) * kRcPer >= n) {
    __threadfence();
  }
  __syncthreads();
  if (tid == 0 && (bid + 1) * kRcPer >= n) *total = s_prefix + agg;
  __syncthreads();
  int64_t o = s_prefix + (w ? s_warp[w - 1] : 0) + x - c;
#pragma unroll
  for (int k = 0; k < kRcEach; ++k)
    if (hit[k]) out[o++] = i0 + k;
}

// K11e: gather records (mapped host pool -> device AoS) and scatter (device AoS -> mapped pool).
__global__ void gather_kernel(const float* __restrict__ pool, const int64_t* __restrict__ idx, int64_t n, int rs,
                              float* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / rs, c = e % rs;
    out[e] = pool[idx[r] * rs + c];
  }
}
// rows -> their records in the mapped host pool, 8 bytes per store when rows are 8-byte aligned
// (even rs), else 4
__global__ void scatter_rec_kernel(float* __restrict__ pool, const int64_t* __restrict__ idx, int64_t n, int rs,
                                   const float* __restrict__ in) {
  if (rs & 1) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rs; e += (int64_t)gridDim.x * blockDim.x)
      pool[idx[e / rs] * rs + e % rs] = in[e];
    return;
  }
  const int h = rs / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * h; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / h, c = e % h;
    reinterpret_cast<float2*>(pool + idx[r] * rs)[c] = reinterpret_cast<const float2*>(in + r * rs)[c];
  }
}
__global__ void pos_scatter_kernel(float* __restrict__ pos_mirror, const int64_t* __restrict__ idx, int64_t n, int rs,
                                   const float* __restrict__ in) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * 3; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / 3, c = e % 3;
    pos_mirror[idx[r] * 3 + c] = in[r * rs + c];
  }
}
// prune test for the active entries + present flags of the kept records
__global__ void prune_kernel(const float* __restrict__ recs, const int64_t* __restrict__ resolved, int64_t n, int rs,
                             float cx, float cy, float cz, float r2, uint8_t* __restrict__ kept,
                             uint8_t* __restrict__ present) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = resolved[i];
    const bool k = rr >= 0 && in_radius(recs + i * rs, cx, cy, cz, r2);
    kept[i] = k;
    if (k) present[rr] = 1;
  }
}
__global__ void copy_rows_kernel(const float* __restrict__ in, const int64_t* __restrict__ rows, int64_t n, int rs,
                                 float* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / rs, c = e % rs;
    out[e] = in[rows[r] * rs + c];
  }
}

// ---- device-resident sync (latmap_store_sync_device): row selections as order-preserving
// compactions, counts kept on the device until the end.
// sel: 0 written-back rows (tracked and dirty), 1 newborn rows (untracked), 2 kept rows
__device__ __forceinline__ bool sel_row(int mode, int64_t i, const int64_t* __restrict__ origin,
                                        const uint8_t* __restrict__ dirty, const uint8_t* __restrict__ kept) {
  if (mode == 0) return origin[i] >= 0 && (!dirty || dirty[i]);
  if (mode == 1) return origin[i] < 0;
  return kept[i] != 0;
}
__global__ void __launch_bounds__(kScanBlock) sel_count_kernel(int mode, int64_t n, const int64_t* __restrict__ origin,
                                                               const uint8_t* __restrict__ dirty,
                                                               const uint8_t* __restrict__ kept,
                                                               int32_t* __restrict__ block_counts) {
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  const int c = __syncthreads_count(i < n && sel_row(mode, i, origin, dirty, kept));
  if (threadIdx.x == 0) block_counts[blockIdx.x] = c;
}
// rows in ascending order -> out_rows; out_val (optional) = origin[row]
__global__ void __launch_bounds__(kScanBlock) sel_emit_kernel(int mode, int64_t n, const int64_t* __restrict__ origin,
                                                              const uint8_t* __restrict__ dirty,
                                                              const uint8_t* __restrict__ kept,
                                                              const int32_t* __restrict__ block_offsets,
                                                              int64_t* __restrict__ out_rows, int64_t* __restrict__ out_val) {
  __shared__ int32_t s_warp[kScanBlock / 32];
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  const bool hit = i < n && sel_row(mode, i, origin, dirty, kept);
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_warp[w] = __popc(m);
  __syncthreads();
  if (w == 0) {
    int v = s_warp[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    s_warp[lane] = v - s_warp[lane];
  }
  __syncthreads();
  if (hit) {
    const int64_t j = block_offsets[blockIdx.x] + s_warp[w] + __popc(m & ((1u << lane) - 1u));
    out_rows[j] = i;
    if (out_val) out_val[j] = origin[i];
  }
}
__global__ void copy_i64_kernel(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}
__global__ void scatter_i64_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ vals, int64_t n,
                                   int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[rows[i]] = vals[i];
}
// copy_rows / gather / pos_scatter with the row count (and an output row offset) read on the device
__global__ void copy_rows_dev_kernel(const float* __restrict__ in, const int64_t* __restrict__ rows,
                                     const int64_t* __restrict__ count, int64_t cap_rows, int rs, float* __restrict__ out) {
  const int64_t n = min(*count, cap_rows);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / rs, c = e % rs;
    out[e] = in[rows[r] * rs + c];
  }
}
__global__ void pos_scatter_dev_kernel(float* __restrict__ pos_mirror, const int64_t* __restrict__ idx,
                                       const int64_t* __restrict__ count, int rs, const float* __restrict__ in) {
  const int64_t n = *count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * 3; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / 3, c = e % 3;
    pos_mirror[idx[r] * 3 + c] = in[r * rs + c];
  }
}
__global__ void scatter_rec_dev_kernel(float* __restrict__ pool, const int64_t* __restrict__ idx,
                                       const int64_t* __restrict__ count, int rs, const float* __restrict__ in) {
  const int64_t n = *count;
  if (rs & 1) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rs; e += (int64_t)gridDim.x * blockDim.x)
      pool[idx[e / rs] * rs + e % rs] = in[e];
    return;
  }
  const int h = rs / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * h; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / h, c = e % h;
    reinterpret_cast<float2*>(pool + idx[r] * rs)[c] = reinterpret_cast<const float2*>(in + r * rs)[c];
  }
}
// assemble: d_out = kept rows (in row order) ++ fetched records (ascending index); out_origin
// likewise. cnt = {nk, fetched}; nothing is written when nk + fetched > cap.
__global__ void assemble_kernel(const float* __restrict__ active, const int64_t* __restrict__ keep_rows,
                                const int64_t* __restrict__ resolved, const float* __restrict__ pool,
                                const int64_t* __restrict__ fetch, const int64_t* __restrict__ cnt, int64_t cap,
                                int rs, float* __restrict__ out, int64_t* __restrict__ out_origin) {
  const int64_t nk = cnt[0], nf = cnt[1];
  if (nk + nf > cap) return;
  const int64_t total = (nk + nf) * rs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / rs, c = e % rs;
    if (r < nk) {
      const int64_t row = keep_rows[r];
      out[e] = active[row * rs + c];
      if (c == 0 && out_origin) out_origin[r] = resolved[row];
    } else {
      const int64_t rec = fetch[r - nk];
      out[e] = pool[rec * rs + c];
      if (c == 0 && out_origin) out_origin[r] = rec;
    }
  }
}

inline unsigned grid_of(int64_t n, int per = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 16));
}

}  // namespace

int64_t compact_blocks(int64_t n) { return std::max<int64_t>(1, (n + kScanBlock - 1) / kScanBlock); }

cudaError_t compact_mask(cudaStream_t st, const uint8_t* mask, int64_t n, int64_t* out_idx, int32_t* blocks,
                         int64_t* count) {
  const int64_t nb = compact_blocks(n);
  sel_count_kernel<<<(unsigned)nb, kScanBlock, 0, st>>>(2, n, nullptr, nullptr, mask, blocks);
  block_scan_kernel<<<1, 1024, 0, st>>>(blocks, nb, count);
  sel_emit_kernel<<<(unsigned)nb, kScanBlock, 0, st>>>(2, n, nullptr, nullptr, mask, blocks, out_idx, nullptr);
  count_launch(3);
  return cudaGetLastError();
}

}  // namespace lm

using namespace lm;

struct latmap_store {
  latmap_ctx* ctx = nullptr;
  cudaStream_t st = nullptr;
  int64_t capacity = 0;
  int32_t ds = 0, rs = 0;
  struct Slot {
    int64_t record = -1;
    int32_t key[3] = {0, 0, 0};
  };
  std::vector<Slot> slots;
  float* pool = nullptr;  // pinned + mapped host memory, pool_cap x rs
  float* pool_dev = nullptr;  // device alias of `pool`
  int64_t pool_cap = 0, size = 0;
  std::vector<int32_t> keys;  // 3 per record
  int64_t stats[5] = {0, 0, 0, 0, 0};
  float* d_pos = nullptr;  // device mirror of record positions
  int64_t d_pos_cap = 0;
  // sync's writeback into the pinned pool runs on its own stream, overlapping the rest of the
  // frame; every later access to the pool waits for it (wb_wait)
  cudaStream_t wb_st = nullptr;
  cudaEvent_t wb_ev = nullptr;
  bool wb_pending = false;
  // pinned staging for sync's index lists (async uploads, no pageable staging copies)
  int64_t* h_stage = nullptr;
  int64_t h_stage_cap = 0;
  // device-resident sync scratch (grow-only): rows [n] x 4 lists, present [pool], fetch [pool],
  // block counts, counters {nwb, nnb, nk, fetched, ...}; a pinned readback of the counters
  int64_t *dv_res = nullptr, *dv_wb_rows = nullptr, *dv_wb_idx = nullptr, *dv_rows2 = nullptr;
  int64_t dv_n_cap = 0;
  uint8_t* dv_present = nullptr;
  int64_t* dv_fetch = nullptr;
  int64_t dv_pool_cap = 0;
  int32_t* dv_cnt = nullptr;
  int64_t dv_cnt_cap = 0;
  int64_t* dv_counts = nullptr;  // [0] nwb [1] nnb [2] nk [3] fetched [4] scan total (device)
  unsigned long long* dv_status = nullptr;  // radius_compact_kernel look-back words (+ ticket)
  int64_t dv_status_cap = 0;
  int64_t* h_counts = nullptr;   // pinned copy of dv_counts
  float* dv_wb_tmp = nullptr;    // written-back rows staged for the pool scatter (wb stream)
  int64_t dv_tmp_cap = 0;
  // scratch
  std::string err;
};

namespace {

latmap_status sfail(latmap_store* s, latmap_status code, const std::string& msg) {
  if (s) s->err = msg;
  return code;
}
#define S_CHECK(s, expr)                                                              \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) return sfail(s, LATMAP_ERR_CUDA, cudaGetErrorString(_e));  \
  } while (0)

void wb_wait(const latmap_store* s) {
  if (s->wb_pending) {
    cudaEventSynchronize(s->wb_ev);
    const_cast<latmap_store*>(s)->wb_pending = false;
  }
}

latmap_status ensure_pool(latmap_store* s, int64_t need) {
  if (need <= s->pool_cap) return LATMAP_OK;
  wb_wait(s);  // no writeback may target the pool being replaced
  int64_t cap = std::max<int64_t>(need, std::max<int64_t>(1024, s->pool_cap * 2));
  float* np = nullptr;
  S_CHECK(s, cudaHostAlloc(&np, sizeof(float) * cap * s->rs, cudaHostAllocMapped));
  if (s->pool) {
    std::memcpy(np, s->pool, sizeof(float) * s->size * s->rs);
    cudaFreeHost(s->pool);
  }
  s->pool = np;
  S_CHECK(s, cudaHostGetDevicePointer(&s->pool_dev, np, 0));
  s->pool_cap = cap;
  float* nd = nullptr;
  S_CHECK(s, cudaMalloc(&nd, sizeof(float) * cap * 3));
  if (s->d_pos) {
    S_CHECK(s, cudaMemcpyAsync(nd, s->d_pos, sizeof(float) * s->size * 3, cudaMemcpyDeviceToDevice, s->st));
    S_CHECK(s, cudaStreamSynchronize(s->st));
    cudaFree(s->d_pos);
  }
  s->d_pos = nd;
  s->d_pos_cap = cap;
  return LATMAP_OK;
}

// VoxelHashStore::probe (voxel_hash.cpp:35-50) with a precomputed home slot.
int64_t probe(latmap_store* s, const int32_t* key, int64_t home, bool for_insert, int64_t* free_slot) {
  if (free_slot) *free_slot = -1;
  const int limit = (int)std::min<int64_t>(kProbeLimit, s->capacity);
  for (int i = 0; i < limit; ++i) {
    const int64_t sl = (home + i) % s->capacity;
    const latmap_store::Slot& slot = s->slots[sl];
    ++s->stats[4];
    if (slot.record < 0) {
      if (for_insert && free_slot && *free_slot < 0) *free_slot = sl;
      return -1;
    }
    if (slot.key[0] == key[0] && slot.key[1] == key[1] && slot.key[2] == key[2]) return sl;
  }
  return -1;
}

// VoxelHashStore::insert (voxel_hash.cpp:52-71); record written into the pinned pool.
int64_t insert_one(latmap_store* s, const int32_t* key, int64_t home, const float* rec, bool rec_on_device,
                   float* d_stage) {
  int64_t free_slot = -1;
  if (probe(s, key, home, true, &free_slot) >= 0) {
    ++s->stats[2];
    return -1;
  }
  if (free_slot < 0) {
    ++s->stats[3];
    return -1;
  }
  if (ensure_pool(s, s->size + 1) != LATMAP_OK) return -2;
  const int64_t r = s->size++;
  if (!rec_on_device) std::memcpy(s->pool + r * s->rs, rec, sizeof(float) * s->rs);
  (void)d_stage;
  s->keys.insert(s->keys.end(), key, key + 3);
  s->slots[free_slot].record = r;
  std::memcpy(s->slots[free_slot].key, key, 12);
  ++s->stats[0];
  return r;
}

}  // namespace

extern "C" {

void latmap_voxel_of(const float p[3], float voxel_size, int32_t key[3]) { lm::voxel_of(p, voxel_size, key); }

int64_t latmap_hash_voxel(const int32_t key[3], int64_t capacity) {
  return capacity > 0 ? lm::hash_voxel(key, capacity) : -1;
}

latmap_status latmap_store_create(latmap_ctx* ctx, int64_t capacity, int32_t query_dim, latmap_store** out) {
  if (!ctx || !out || capacity <= 0 || query_dim < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  auto* s = new latmap_store();
  s->ctx = ctx;
  s->st = (cudaStream_t)latmap_ctx_stream(ctx);
  s->capacity = capacity;
  s->ds = query_dim;
  s->rs = 14 + query_dim;
  s->slots.resize((size_t)capacity);
  if (cudaStreamCreateWithFlags(&s->wb_st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->wb_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete s;
    return LATMAP_ERR_CUDA;
  }
  *out = s;
  return LATMAP_OK;
}

latmap_status latmap_store_destroy(latmap_store* s) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  cudaDeviceSynchronize();
  if (s->pool) cudaFreeHost(s->pool);
  if (s->d_pos) cudaFree(s->d_pos);
  if (s->wb_ev) cudaEventDestroy(s->wb_ev);
  if (s->h_stage) cudaFreeHost(s->h_stage);
  for (void* p : {(void*)s->dv_res, (void*)s->dv_wb_rows, (void*)s->dv_wb_idx, (void*)s->dv_rows2,
                  (void*)s->dv_present, (void*)s->dv_fetch, (void*)s->dv_cnt, (void*)s->dv_counts, (void*)s->dv_status,
                  (void*)s->dv_wb_tmp})
    if (p) cudaFree(p);
  if (s->h_counts) cudaFreeHost(s->h_counts);
  if (s->wb_st) cudaStreamDestroy(s->wb_st);
  delete s;
  return LATMAP_OK;
}

int64_t latmap_store_size(const latmap_store* s) { return s ? s->size : -1; }

void latmap_store_stats(const latmap_store* s, int64_t out[5]) {
  if (s && out) std::memcpy(out, s->stats, sizeof(s->stats));
}

const char* latmap_store_last_error(const latmap_store* s) { return s ? s->err.c_str() : ""; }

int64_t latmap_store_insert(latmap_store* s, const int32_t key[3], const float* rec) {
  if (!s || !rec) return -1;
  const int64_t r = insert_one(s, key, lm::hash_voxel(key, s->capacity), rec, false, nullptr);
  if (r >= 0) {
    cudaMemcpyAsync(s->d_pos + r * 3, rec, 12, cudaMemcpyHostToDevice, s->st);
    cudaStreamSynchronize(s->st);
  }
  return r;
}

int32_t latmap_store_update(latmap_store* s, const int32_t key[3], const float* rec) {
  if (!s || !rec) return 0;
  wb_wait(s);
  const int64_t hit = probe(s, key, lm::hash_voxel(key, s->capacity), false, nullptr);
  if (hit < 0) return 0;
  const int64_t r = s->slots[hit].record;
  std::memcpy(s->pool + r * s->rs, rec, sizeof(float) * s->rs);
  cudaMemcpyAsync(s->d_pos + r * 3, rec, 12, cudaMemcpyHostToDevice, s->st);
  cudaStreamSynchronize(s->st);
  ++s->stats[1];
  return 1;
}

int64_t latmap_store_find(latmap_store* s, const int32_t key[3]) {
  if (!s) return -1;
  const int64_t hit = probe(s, key, lm::hash_voxel(key, s->capacity), false, nullptr);
  return hit < 0 ? -1 : s->slots[hit].record;
}

latmap_status latmap_store_get_records(const latmap_store* s, int64_t first, int64_t count, float* out,
                                       int32_t* keys_out) {
  if (!s || first < 0 || first + count > s->size) return LATMAP_ERR_INVALID_ARGUMENT;
  wb_wait(s);
  cudaStreamSynchronize(s->st);
  if (out) std::memcpy(out, s->pool + first * s->rs, sizeof(float) * count * s->rs);
  if (keys_out) std::memcpy(keys_out, s->keys.data() + first * 3, sizeof(int32_t) * count * 3);
  return LATMAP_OK;
}

// insert_global (voxel_hash.cpp:101-115): keys / home slots on the device, sequential probe on
// the host in record order (identical record indices and rejections).
latmap_status latmap_store_insert_global(latmap_store* s, const float* recs, int64_t n, float voxel_size,
                                         int64_t* inserted) {
  if (!s || (n > 0 && !recs)) return LATMAP_ERR_INVALID_ARGUMENT;
  if (!(voxel_size > 0.f)) return sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "voxel_of: voxel_size must be > 0");
  if (inserted) *inserted = 0;
  if (n == 0) return LATMAP_OK;
  float* d_recs = nullptr;
  int32_t* d_keys = nullptr;
  int64_t* d_home = nullptr;
  S_CHECK(s, cudaMallocAsync(&d_recs, sizeof(float) * n * s->rs, s->st));
  S_CHECK(s, cudaMallocAsync(&d_keys, sizeof(int32_t) * n * 3, s->st));
  S_CHECK(s, cudaMallocAsync(&d_home, sizeof(int64_t) * n, s->st));
  S_CHECK(s, cudaMemcpyAsync(d_recs, recs, sizeof(float) * n * s->rs, cudaMemcpyHostToDevice, s->st));
  keys_kernel<<<grid_of(n), 256, 0, s->st>>>(d_recs, n, s->rs, voxel_size, s->capacity, d_keys, d_home);
  count_launch();
  std::vector<int32_t> keys((size_t)n * 3);
  std::vector<int64_t> home((size_t)n);
  S_CHECK(s, cudaMemcpyAsync(keys.data(), d_keys, sizeof(int32_t) * n * 3, cudaMemcpyDeviceToHost, s->st));
  S_CHECK(s, cudaMemcpyAsync(home.data(), d_home, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s->st));
  S_CHECK(s, cudaStreamSynchronize(s->st));
  if (ensure_pool(s, s->size + n) != LATMAP_OK) return LATMAP_ERR_OUT_OF_MEMORY;
  const int64_t first = s->size;
  int64_t ins = 0;
  for (int64_t i = 0; i < n; ++i) ins += insert_one(s, &keys[3 * i], home[i], recs + i * s->rs, false, nullptr) >= 0;
  // position mirror for the new records
  std::vector<float> pos((size_t)(s->size - first) * 3);
  for (int64_t r = first; r < s->size; ++r) std::memcpy(&pos[(r - first) * 3], s->pool + r * s->rs, 12);
  if (!pos.empty())
    S_CHECK(s, cudaMemcpyAsync(s->d_pos + first * 3, pos.data(), sizeof(float) * pos.size(), cudaMemcpyHostToDevice,
                               s->st));
  S_CHECK(s, cudaFreeAsync(d_recs, s->st));
  S_CHECK(s, cudaFreeAsync(d_keys, s->st));
  S_CHECK(s, cudaFreeAsync(d_home, s->st));
  S_CHECK(s, cudaStreamSynchronize(s->st));
  if (inserted) *inserted = ins;
  return LATMAP_OK;
}

// Rebuild from a dump (artifacts.cpp:54-63 LoadedMap -> VoxelHashStore::insert per record in dump
// order): explicit keys, so record indices follow the dump and rejections match insert().
latmap_status latmap_store_insert_keyed(latmap_store* s, const int32_t* keys, const float* recs, int64_t n,
                                        int64_t* inserted) {
  if (!s || n < 0 || (n > 0 && (!recs || !keys))) return LATMAP_ERR_INVALID_ARGUMENT;
  if (inserted) *inserted = 0;
  if (n == 0) return LATMAP_OK;
  if (ensure_pool(s, s->size + n) != LATMAP_OK) return LATMAP_ERR_OUT_OF_MEMORY;
  const int64_t first = s->size;
  int64_t ins = 0;
  for (int64_t i = 0; i < n; ++i)
    ins += insert_one(s, &keys[3 * i], lm::hash_voxel(&keys[3 * i], s->capacity), recs + i * s->rs, false,
                      nullptr) >= 0;
  std::vector<float> pos((size_t)(s->size - first) * 3);
  for (int64_t r = first; r < s->size; ++r) std::memcpy(&pos[(r - first) * 3], s->pool + r * s->rs, 12);
  if (!pos.empty())
    S_CHECK(s, cudaMemcpyAsync(s->d_pos + first * 3, pos.data(), sizeof(float) * pos.size(), cudaMemcpyHostToDevice,
                               s->st));
  S_CHECK(s, cudaStreamSynchronize(s->st));
  if (inserted) *inserted = ins;
  return LATMAP_OK;
}

// fetch_local (active_set.cpp:7-36): ascending record indices of the records within `radius`,
// optional gather of their records into a device AoS buffer (records x (14 + ds) floats).
latmap_status latmap_store_fetch_local(latmap_store* s, const float center[3], float radius, int64_t* origin,
                                       int64_t cap, int64_t* count, float* d_records) {
  if (!s || !count) return LATMAP_ERR_INVALID_ARGUMENT;
  if (!(radius > 0.f)) return sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "fetch_local: radius must be > 0");
  wb_wait(s);
  *count = 0;
  if (s->size == 0) return LATMAP_OK;
  const float r2 = radius * radius;
  const int64_t nb = (s->size + kScanBlock - 1) / kScanBlock;
  int32_t* d_cnt = nullptr;
  int64_t* d_total = nullptr;
  int64_t* d_idx = nullptr;
  S_CHECK(s, cudaMallocAsync(&d_cnt, sizeof(int32_t) * nb, s->st));
  S_CHECK(s, cudaMallocAsync(&d_total, sizeof(int64_t), s->st));
  S_CHECK(s, cudaMallocAsync(&d_idx, sizeof(int64_t) * s->size, s->st));
  radius_count_kernel<<<(unsigned)nb, kScanBlock, 0, s->st>>>(s->d_pos, s->size, center[0], center[1], center[2], r2,
                                                               nullptr, d_cnt);
  block_scan_kernel<<<1, 1024, 0, s->st>>>(d_cnt, nb, d_total);
  radius_emit_kernel<<<(unsigned)nb, kScanBlock, 0, s->st>>>(s->d_pos, s->size, center[0], center[1], center[2], r2,
                                                              nullptr, d_cnt, d_idx);
  count_launch(3);
  int64_t total = 0;
  S_CHECK(s, cudaMemcpyAsync(&total, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, s->st));
  S_CHECK(s, cudaStreamSynchronize(s->st));
  *count = total;
  latmap_status ret = LATMAP_OK;
  if (origin) {
    if (total > cap) {
      ret = sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "fetch_local: output capacity too small");
    } else if (total > 0) {
      S_CHECK(s, cudaMemcpyAsync(origin, d_idx, sizeof(int64_t) * total, cudaMemcpyDeviceToHost, s->st));
    }
  }
  if (d_records && total > 0 && ret == LATMAP_OK) {
    gather_kernel<<<grid_of(total * s->rs), 256, 0, s->st>>>(s->pool_dev, d_idx, total, s->rs, d_records);
    count_launch();
  }
  S_CHECK(s, cudaFreeAsync(d_cnt, s->st));
  S_CHECK(s, cudaFreeAsync(d_total, s->st));
  S_CHECK(s, cudaFreeAsync(d_idx, s->st));
  S_CHECK(s, cudaStreamSynchronize(s->st));
  return ret;
}

// sync (active_set.cpp:38-128). Active records live on the device (AoS, n x (14 + ds));
// origin / dirty / kept_mask / out_origin are host arrays; out_records is a device buffer.
// stats: written_back, newborn_inserted, newborn_rejected, pruned, fetched.
latmap_status latmap_store_sync(latmap_store* s, const float* d_active, const int64_t* origin, const uint8_t* dirty,
                                int64_t n, const float center[3], float radius, float voxel_size, float* d_out,
                                int64_t* out_origin, int64_t cap, uint8_t* kept_mask, int64_t stats_out[5],
                                int64_t* out_count) {
  if (!s || !center || !out_count || (n > 0 && (!d_active || !origin || !dirty))) return LATMAP_ERR_INVALID_ARGUMENT;
  if (!(voxel_size > 0.f)) return sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "voxel_of: voxel_size must be > 0");
  const int rs = s->rs;
  int64_t st5[5] = {0, 0, 0, 0, 0};
  wb_wait(s);  // the previous sync's writeback
  // LATMAP_SYNC_TRACE=1: per-step wall times (each step synchronised; development only)
  static const bool trace = std::getenv("LATMAP_SYNC_TRACE") != nullptr;
  auto tmark = [&, t0 = std::chrono::steady_clock::now()](const char* what) mutable {
    if (!trace) return;
    cudaStreamSynchronize(s->st);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "sync %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const int64_t nn = std::max<int64_t>(n, 1);
  if (s->h_stage_cap < 4 * nn) {  // the previous sync ended with a stream synchronize: free to replace
    if (s->h_stage) cudaFreeHost(s->h_stage);
    s->h_stage = nullptr;
    s->h_stage_cap = 0;
    S_CHECK(s, cudaHostAlloc(&s->h_stage, sizeof(int64_t) * 4 * nn + sizeof(int64_t) * 4 * (nn / 4), 0));
    s->h_stage_cap = 4 * nn + 4 * (nn / 4);
  }
  int64_t* resolved = s->h_stage;            // n entries
  int64_t* wb_rows = s->h_stage + nn;        // <= n
  int64_t* wb_idx = s->h_stage + 2 * nn;     // <= n
  int64_t* keep_rows = s->h_stage + 3 * nn;  // <= n
  std::fill(resolved, resolved + nn, int64_t(-1));
  int64_t nwb = 0;
  // ---- step 1: writeback. Dirty tracked entries overwrite their record in place (origin voxel
  // retained); newborns insert under the voxel of their optimised position, in row order.
  std::vector<int64_t> nb_rows;
  float* wb_tmp = nullptr;
  int64_t* wb_idx_dev = nullptr;
  int64_t wb_n = 0;
  // every device temporary of this call, and an exit guard: an error return launches the
  // deferred pool writeback (the position mirror already holds those rows) and frees what is
  // still allocated, then synchronizes, so the pool, the mirror and h_stage stay consistent
  std::vector<void*> live;
  auto amalloc = [&](auto** p, size_t bytes) {
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), bytes, s->st);
    if (e == cudaSuccess) live.push_back(*p);
    return e;
  };
  auto afree = [&](void* p) {
    live.erase(std::remove(live.begin(), live.end(), p), live.end());
    return cudaFreeAsync(p, s->st);
  };
  struct ExitGuard {
    std::function<void()> f;
    ~ExitGuard() {
      if (f) f();
    }
  } guard{[&]() {
    if (wb_n > 0 && wb_tmp && wb_idx_dev)
      scatter_rec_kernel<<<grid_of(wb_n * rs / 2), 256, 0, s->st>>>(s->pool_dev, wb_idx_dev, wb_n, rs, wb_tmp);
    for (void* p : live) cudaFreeAsync(p, s->st);
    cudaStreamSynchronize(s->st);
  }};
  for (int64_t i = 0; i < n; ++i) {
    if (origin[i] >= 0) {
      resolved[i] = origin[i];
      if (dirty[i]) {
        wb_rows[nwb] = i;
        wb_idx[nwb++] = origin[i];
      }
    } else {
      nb_rows.push_back(i);
    }
  }
  int64_t *d_rows = nullptr, *d_idx2 = nullptr;
  if (nwb > 0) {
    float* d_tmp = nullptr;
    S_CHECK(s, amalloc(&d_rows, sizeof(int64_t) * nwb));
    S_CHECK(s, amalloc(&d_idx2, sizeof(int64_t) * nwb));
    S_CHECK(s, amalloc(&d_tmp, sizeof(float) * nwb * rs));
    S_CHECK(s, cudaMemcpyAsync(d_rows, wb_rows, sizeof(int64_t) * nwb, cudaMemcpyHostToDevice, s->st));
    S_CHECK(s, cudaMemcpyAsync(d_idx2, wb_idx, sizeof(int64_t) * nwb, cudaMemcpyHostToDevice, s->st));
    copy_rows_kernel<<<grid_of(nwb * rs), 256, 0, s->st>>>(d_active, d_rows, nwb, rs, d_tmp);
    // the position mirror now (the radius scan below reads it); the pool rows over PCIe on the
    // writeback stream, overlapping everything after this sync (the rows fetched below are never
    // written back ones: those are present or pruned)
    pos_scatter_kernel<<<grid_of(nwb * 3), 256, 0, s->st>>>(s->d_pos, d_idx2, nwb, rs, d_tmp);
    count_launch(2);
    S_CHECK(s, afree(d_rows));
    wb_tmp = d_tmp, wb_idx_dev = d_idx2, wb_n = nwb;  // pool rows: launched when this sync is done
    st5[0] = nwb;
  }
  tmark("writeback");
  const int64_t nnb = (int64_t)nb_rows.size();
  if (nnb > 0) {
    float* d_nb = nullptr;
    int32_t* d_keys = nullptr;
    int64_t* d_home = nullptr;
    S_CHECK(s, amalloc(&d_rows, sizeof(int64_t) * nnb));
    S_CHECK(s, amalloc(&d_nb, sizeof(float) * nnb * rs));
    S_CHECK(s, amalloc(&d_keys, sizeof(int32_t) * nnb * 3));
    S_CHECK(s, amalloc(&d_home, sizeof(int64_t) * nnb));
    S_CHECK(s, cudaMemcpyAsync(d_rows, nb_rows.data(), sizeof(int64_t) * nnb, cudaMemcpyHostToDevice, s->st));
    copy_rows_kernel<<<grid_of(nnb * rs), 256, 0, s->st>>>(d_active, d_rows, nnb, rs, d_nb);
    keys_kernel<<<grid_of(nnb), 256, 0, s->st>>>(d_nb, nnb, rs, voxel_size, s->capacity, d_keys, d_home);
    count_launch(2);
    std::vector<float> nb((size_t)nnb * rs);
    std::vector<int32_t> keys((size_t)nnb * 3);
    std::vector<int64_t> home((size_t)nnb);
    S_CHECK(s, cudaMemcpyAsync(nb.data(), d_nb, sizeof(float) * nnb * rs, cudaMemcpyDeviceToHost, s->st));
    S_CHECK(s, cudaMemcpyAsync(keys.data(), d_keys, sizeof(int32_t) * nnb * 3, cudaMemcpyDeviceToHost, s->st));
    S_CHECK(s, cudaMemcpyAsync(home.data(), d_home, sizeof(int64_t) * nnb, cudaMemcpyDeviceToHost, s->st));
    S_CHECK(s, cudaStreamSynchronize(s->st));  // also orders the writeback scatter before host pool reads
    if (ensure_pool(s, s->size + nnb) != LATMAP_OK) return LATMAP_ERR_OUT_OF_MEMORY;
    const int64_t first = s->size;
    for (int64_t j = 0; j < nnb; ++j) {
      const int64_t r = insert_one(s, &keys[3 * j], home[j], &nb[j * rs], false, nullptr);
      if (r >= 0) {
        resolved[nb_rows[j]] = r;
        ++st5[1];
      } else {
        ++st5[2];
      }
    }
    std::vector<float> pos((size_t)(s->size - first) * 3);
    for (int64_t r = first; r < s->size; ++r) std::memcpy(&pos[(r - first) * 3], s->pool + r * rs, 12);
    if (!pos.empty())
      S_CHECK(s, cudaMemcpyAsync(s->d_pos + first * 3, pos.data(), sizeof(float) * pos.size(), cudaMemcpyHostToDevice,
                                 s->st));
    S_CHECK(s, afree(d_nb));
    S_CHECK(s, afree(d_keys));
    S_CHECK(s, afree(d_home));
    S_CHECK(s, afree(d_rows));
  }
  tmark("newborns");
  // ---- step 2: prune in-radius tracked entries, mark their records present
  const float r2 = radius * radius;
  uint8_t* d_present = nullptr;
  uint8_t* d_kept = nullptr;
  int64_t* d_res = nullptr;
  S_CHECK(s, amalloc(&d_present, std::max<int64_t>(s->size, 1)));
  S_CHECK(s, cudaMemsetAsync(d_present, 0, std::max<int64_t>(s->size, 1), s->st));
  std::vector<uint8_t> kept((size_t)std::max<int64_t>(n, 1), 0);
  if (n > 0) {
    S_CHECK(s, amalloc(&d_kept, n));
    S_CHECK(s, amalloc(&d_res, sizeof(int64_t) * n));
    S_CHECK(s, cudaMemcpyAsync(d_res, resolved, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s->st));
    prune_kernel<<<grid_of(n), 256, 0, s->st>>>(d_active, d_res, n, rs, center[0], center[1], center[2], r2, d_kept,
                                                d_present);
    count_launch();
    S_CHECK(s, cudaMemcpyAsync(kept.data(), d_kept, n, cudaMemcpyDeviceToHost, s->st));
  }
  tmark("prune");
  // ---- step 3: fetch not-present in-radius records in ascending index order
  const int64_t nb = std::max<int64_t>(1, (s->size + kScanBlock - 1) / kScanBlock);
  int32_t* d_cnt = nullptr;
  int64_t* d_total = nullptr;
  int64_t* d_fetch = nullptr;
  S_CHECK(s, amalloc(&d_cnt, sizeof(int32_t) * nb));
  S_CHECK(s, amalloc(&d_total, sizeof(int64_t)));
  S_CHECK(s, amalloc(&d_fetch, sizeof(int64_t) * std::max<int64_t>(s->size, 1)));
  int64_t fetched = 0;
  if (s->size > 0) {
    radius_count_kernel<<<(unsigned)nb, kScanBlock, 0, s->st>>>(s->d_pos, s->size, center[0], center[1], center[2],
                                                                 r2, d_present, d_cnt);
    block_scan_kernel<<<1, 1024, 0, s->st>>>(d_cnt, nb, d_total);
    radius_emit_kernel<<<(unsigned)nb, kScanBlock, 0, s->st>>>(s->d_pos, s->size, center[0], center[1], center[2],
                                                                r2, d_present, d_cnt, d_fetch);
    count_launch(3);
    S_CHECK(s, cudaMemcpyAsync(&fetched, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, s->st));
  }
  S_CHECK(s, cudaStreamSynchronize(s->st));
  tmark("scan");
  int64_t nk = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (resolved[i] < 0) continue;  // rejected newborn drops out
    if (kept[i])
      keep_rows[nk++] = i;
    else
      ++st5[3];
  }
  st5[4] = fetched;
  const int64_t total = nk + fetched;
  *out_count = total;
  if (kept_mask)
    for (int64_t i = 0; i < n; ++i) kept_mask[i] = kept[i];
  if (stats_out) std::memcpy(stats_out, st5, sizeof(st5));
  latmap_status ret = LATMAP_OK;
  if (total > cap) {
    ret = sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "sync: output capacity too small");
  } else {
    // ---- assemble: kept (original order) ++ fetched (ascending)
    if (nk > 0) {
      int64_t* d_k = nullptr;
      S_CHECK(s, amalloc(&d_k, sizeof(int64_t) * nk));
      S_CHECK(s, cudaMemcpyAsync(d_k, keep_rows, sizeof(int64_t) * nk, cudaMemcpyHostToDevice, s->st));
      copy_rows_kernel<<<grid_of(nk * rs), 256, 0, s->st>>>(d_active, d_k, nk, rs, d_out);
      count_launch();
      S_CHECK(s, afree(d_k));
      if (out_origin)
        for (int64_t j = 0; j < nk; ++j) out_origin[j] = resolved[keep_rows[j]];
    }
    if (fetched > 0) {
      gather_kernel<<<grid_of(fetched * rs), 256, 0, s->st>>>(s->pool_dev, d_fetch, fetched, rs, d_out + nk * rs);
      count_launch();
      if (out_origin)
        S_CHECK(s, cudaMemcpyAsync(out_origin + nk, d_fetch, sizeof(int64_t) * fetched, cudaMemcpyDeviceToHost,
                                   s->st));
    }
  }
  tmark("assemble");
  S_CHECK(s, afree(d_present));
  if (d_kept) S_CHECK(s, afree(d_kept));
  if (d_res) S_CHECK(s, afree(d_res));
  S_CHECK(s, afree(d_cnt));
  S_CHECK(s, afree(d_total));
  S_CHECK(s, afree(d_fetch));
  S_CHECK(s, cudaStreamSynchronize(s->st));
  guard.f = nullptr;  // success: nothing to undo
  if (wb_n > 0) {
    // the written-back rows reach the pinned pool over PCIe after this sync's own transfers (which
    // would otherwise queue behind ~184 B x rows of posted writes), overlapping the caller's next
    // work; the rows fetched above were never written back ones (those are present or pruned)
    S_CHECK(s, cudaEventRecord(s->wb_ev, s->st));
    S_CHECK(s, cudaStreamWaitEvent(s->wb_st, s->wb_ev, 0));
    scatter_rec_kernel<<<grid_of(wb_n * rs / 2), 256, 0, s->wb_st>>>(s->pool_dev, wb_idx_dev, wb_n, rs, wb_tmp);
    count_launch();
    S_CHECK(s, cudaFreeAsync(wb_tmp, s->wb_st));
    S_CHECK(s, cudaFreeAsync(wb_idx_dev, s->wb_st));
    S_CHECK(s, cudaEventRecord(s->wb_ev, s->wb_st));
    s->wb_pending = true;
  }
  return ret;
}


namespace {
// order-preserving radius compaction of the pool positions into out (ascending), count -> *total
latmap_status radius_compact(latmap_store* s, const float center[3], float r2, const uint8_t* present, int64_t* out,
                             int64_t* total) {
  const int64_t ps = s->size;
  const int64_t nb = (ps + kRcPer - 1) / kRcPer;
  if (s->dv_status_cap < nb + 1) {
    if (s->dv_status) cudaFree(s->dv_status);
    s->dv_status_cap = nb + 1 + nb / 4;
    S_CHECK(s, cudaMalloc(&s->dv_status, sizeof(unsigned long long) * s->dv_status_cap));
  }
  S_CHECK(s, cudaMemsetAsync(s->dv_status, 0, sizeof(unsigned long long) * (nb + 1), s->st));
  radius_compact_kernel<<<(unsigned)nb, kRcThreads, 0, s->st>>>(
      s->d_pos, ps, center[0], center[1], center[2], r2, present, s->dv_status,
      reinterpret_cast<int*>(s->dv_status + nb), out, total);
  count_launch();
  return LATMAP_OK;
}
}  // namespace

// sync (active_set.cpp:38-128) with every per-row array on the device: origin / dirty / kept /
// out_origin are device buffers, the row selections are order-preserving device compactions and
// the counts come back once (plus once more when newborns need the host's probe order).
latmap_status latmap_store_sync_device(latmap_store* s, const float* d_active, const int64_t* d_origin,
                                       const uint8_t* d_dirty, int64_t n, const float center[3], float radius,
                                       float voxel_size, float* d_out, int64_t* d_out_origin, int64_t cap,
                                       uint8_t* d_kept, int64_t stats_out[5], int64_t* out_count) {
  if (!s || !center || !out_count || n < 0 || (n > 0 && (!d_active || !d_origin || !d_kept)))
    return LATMAP_ERR_INVALID_ARGUMENT;
  if (!(voxel_size > 0.f)) return sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "voxel_of: voxel_size must be > 0");
  const int rs = s->rs;
  cudaStream_t st = s->st;
  wb_wait(s);  // the previous sync's writeback (it reads dv_wb_tmp / dv_wb_idx / dv_counts)
  int64_t st5[5] = {0, 0, 0, 0, 0};
  const int64_t nn = std::max<int64_t>(n, 1);
  auto grow64 = [&](int64_t*& p, int64_t need) -> cudaError_t {
    if (p) cudaFree(p);
    return cudaMalloc(&p, sizeof(int64_t) * need);
  };
  if (s->dv_n_cap < nn) {
    S_CHECK(s, grow64(s->dv_res, nn + nn / 4));
    S_CHECK(s, grow64(s->dv_wb_rows, nn + nn / 4));
    S_CHECK(s, grow64(s->dv_wb_idx, nn + nn / 4));
    S_CHECK(s, grow64(s->dv_rows2, nn + nn / 4));
    if (s->dv_wb_tmp) cudaFree(s->dv_wb_tmp);
    S_CHECK(s, cudaMalloc(&s->dv_wb_tmp, sizeof(float) * (nn + nn / 4) * rs));
    s->dv_n_cap = nn + nn / 4;
  }
  if (!s->dv_counts) {
    S_CHECK(s, cudaMalloc(&s->dv_counts, sizeof(int64_t) * 8));
    S_CHECK(s, cudaHostAlloc(&s->h_counts, sizeof(int64_t) * 8, 0));
  }
  auto ensure_blocks = [&](int64_t rows) -> cudaError_t {
    const int64_t nb = compact_blocks(rows) + 1;
    if (s->dv_cnt_cap >= nb) return cudaSuccess;
    if (s->dv_cnt) cudaFree(s->dv_cnt);
    s->dv_cnt_cap = nb + nb / 4;
    return cudaMalloc(&s->dv_cnt, sizeof(int32_t) * s->dv_cnt_cap);
  };
  S_CHECK(s, ensure_blocks(n));
  S_CHECK(s, cudaMemsetAsync(s->dv_counts, 0, sizeof(int64_t) * 8, st));
  const int64_t nbn = compact_blocks(n);
  if (n > 0) {
    copy_i64_kernel<<<grid_of(n), 256, 0, st>>>(d_origin, n, s->dv_res);  // resolved = origin (newborns: -1)
    // newborn rows (row order) and written-back rows with their records
    sel_count_kernel<<<(unsigned)nbn, kScanBlock, 0, st>>>(1, n, d_origin, d_dirty, nullptr, s->dv_cnt);
    block_scan_kernel<<<1, 1024, 0, st>>>(s->dv_cnt, nbn, s->dv_counts + 1);
    sel_emit_kernel<<<(unsigned)nbn, kScanBlock, 0, st>>>(1, n, d_origin, d_dirty, nullptr, s->dv_cnt, s->dv_rows2,
                                                          nullptr);
    sel_count_kernel<<<(unsigned)nbn, kScanBlock, 0, st>>>(0, n, d_origin, d_dirty, nullptr, s->dv_cnt);
    block_scan_kernel<<<1, 1024, 0, st>>>(s->dv_cnt, nbn, s->dv_counts + 0);
    sel_emit_kernel<<<(unsigned)nbn, kScanBlock, 0, st>>>(0, n, d_origin, d_dirty, nullptr, s->dv_cnt, s->dv_wb_rows,
                                                          s->dv_wb_idx);
    copy_rows_dev_kernel<<<grid_of(n * rs), 256, 0, st>>>(d_active, s->dv_wb_rows, s->dv_counts + 0, n, rs,
                                                          s->dv_wb_tmp);
    pos_scatter_dev_kernel<<<grid_of(n * 3), 256, 0, st>>>(s->d_pos, s->dv_wb_idx, s->dv_counts + 0, rs,
                                                           s->dv_wb_tmp);
    count_launch(9);
  }
  S_CHECK(s, cudaMemcpyAsync(s->h_counts, s->dv_counts, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, st));
  S_CHECK(s, cudaStreamSynchronize(st));
  const int64_t nwb = s->h_counts[0], nnb = s->h_counts[1];
  st5[0] = nwb;
  int64_t ins = 0;
  if (nnb > 0) {
    // newborns insert under the voxel of their optimised position in row order (the host probe
    // sequence defines record indices and rejections, active_set.cpp:56-70)
    std::vector<int64_t> rows((size_t)nnb);
    float* d_nb = nullptr;
    int32_t* d_keys = nullptr;
    int64_t *d_home = nullptr, *d_pairs = nullptr;
    S_CHECK(s, cudaMemcpyAsync(rows.data(), s->dv_rows2, sizeof(int64_t) * nnb, cudaMemcpyDeviceToHost, st));
    S_CHECK(s, cudaMallocAsync(&d_nb, sizeof(float) * nnb * rs, st));
    S_CHECK(s, cudaMallocAsync(&d_keys, sizeof(int32_t) * nnb * 3, st));
    S_CHECK(s, cudaMallocAsync(&d_home, sizeof(int64_t) * nnb, st));
    S_CHECK(s, cudaMallocAsync(&d_pairs, sizeof(int64_t) * nnb * 2, st));
    copy_rows_kernel<<<grid_of(nnb * rs), 256, 0, st>>>(d_active, s->dv_rows2, nnb, rs, d_nb);
    keys_kernel<<<grid_of(nnb), 256, 0, st>>>(d_nb, nnb, rs, voxel_size, s->capacity, d_keys, d_home);
    count_launch(2);
    std::vector<float> nb((size_t)nnb * rs);
    std::vector<int32_t> keys((size_t)nnb * 3);
    std::vector<int64_t> home((size_t)nnb);
    S_CHECK(s, cudaMemcpyAsync(nb.data(), d_nb, sizeof(float) * nnb * rs, cudaMemcpyDeviceToHost, st));
    S_CHECK(s, cudaMemcpyAsync(keys.data(), d_keys, sizeof(int32_t) * nnb * 3, cudaMemcpyDeviceToHost, st));
    S_CHECK(s, cudaMemcpyAsync(home.data(), d_home, sizeof(int64_t) * nnb, cudaMemcpyDeviceToHost, st));
    S_CHECK(s, cudaStreamSynchronize(st));
    if (ensure_pool(s, s->size + nnb) != LATMAP_OK) return LATMAP_ERR_OUT_OF_MEMORY;
    const int64_t first = s->size;
    std::vector<int64_t> pr;  // (row, record) of the inserted newborns
    for (int64_t j = 0; j < nnb; ++j) {
      const int64_t r = insert_one(s, &keys[3 * j], home[j], &nb[j * rs], false, nullptr);
      if (r >= 0) {
        pr.push_back(rows[j]);
        pr.push_back(r);
        ++ins;
      }
    }
    st5[1] = ins;
    st5[2] = nnb - ins;
    if (ins > 0) {
      std::vector<int64_t> rr((size_t)ins), rv((size_t)ins);
      for (int64_t j = 0; j < ins; ++j) rr[j] = pr[2 * j], rv[j] = pr[2 * j + 1];
      S_CHECK(s, cudaMemcpyAsync(d_pairs, rr.data(), sizeof(int64_t) * ins, cudaMemcpyHostToDevice, st));
      S_CHECK(s, cudaMemcpyAsync(d_pairs + nnb, rv.data(), sizeof(int64_t) * ins, cudaMemcpyHostToDevice, st));
      scatter_i64_kernel<<<grid_of(ins), 256, 0, st>>>(d_pairs, d_pairs + nnb, ins, s->dv_res);
      count_launch();
    }
    std::vector<float> pos((size_t)(s->size - first) * 3);
    for (int64_t r = first; r < s->size; ++r) std::memcpy(&pos[(r - first) * 3], s->pool + r * rs, 12);
    if (!pos.empty())
      S_CHECK(s, cudaMemcpyAsync(s->d_pos + first * 3, pos.data(), sizeof(float) * pos.size(), cudaMemcpyHostToDevice,
                                 st));
    S_CHECK(s, cudaStreamSynchronize(st));  // host staging vectors go out of scope
    S_CHECK(s, cudaFreeAsync(d_nb, st));
    S_CHECK(s, cudaFreeAsync(d_keys, st));
    S_CHECK(s, cudaFreeAsync(d_home, st));
    S_CHECK(s, cudaFreeAsync(d_pairs, st));
  }
  // pool-sized scratch (the pool may have grown by the newborns)
  const int64_t ps = std::max<int64_t>(s->size, 1);
  if (s->dv_pool_cap < ps) {
    if (s->dv_present) cudaFree(s->dv_present);
    S_CHECK(s, grow64(s->dv_fetch, ps + ps / 4));
    S_CHECK(s, cudaMalloc(&s->dv_present, ps + ps / 4));
    s->dv_pool_cap = ps + ps / 4;
  }
  S_CHECK(s, ensure_blocks(s->size));
  // prune in-radius tracked entries, mark their records present; kept rows (row order)
  const float r2 = radius * radius;
  S_CHECK(s, cudaMemsetAsync(s->dv_present, 0, ps, st));
  if (n > 0) {
    prune_kernel<<<grid_of(n), 256, 0, st>>>(d_active, s->dv_res, n, rs, center[0], center[1], center[2], r2, d_kept,
                                             s->dv_present);
    sel_count_kernel<<<(unsigned)nbn, kScanBlock, 0, st>>>(2, n, nullptr, nullptr, d_kept, s->dv_cnt);
    block_scan_kernel<<<1, 1024, 0, st>>>(s->dv_cnt, nbn, s->dv_counts + 2);
    sel_emit_kernel<<<(unsigned)nbn, kScanBlock, 0, st>>>(2, n, nullptr, nullptr, d_kept, s->dv_cnt, s->dv_rows2,
                                                          nullptr);
    count_launch(4);
  }
  // fetch: not-present in-radius records, ascending index
  if (s->size > 0) {
    const latmap_status rc = radius_compact(s, center, r2, s->dv_present, s->dv_fetch, s->dv_counts + 3);
    if (rc != LATMAP_OK) return rc;
  }
  // assemble (nothing written when the output capacity is too small)
  if (d_out && cap > 0) {
    assemble_kernel<<<grid_of((n + s->size) * rs), 256, 0, st>>>(d_active, s->dv_rows2, s->dv_res, s->pool_dev,
                                                                 s->dv_fetch, s->dv_counts + 2, cap, rs, d_out,
                                                                 d_out_origin);
    count_launch();
  }
  S_CHECK(s, cudaMemcpyAsync(s->h_counts, s->dv_counts, sizeof(int64_t) * 4, cudaMemcpyDeviceToHost, st));
  S_CHECK(s, cudaStreamSynchronize(st));
  const int64_t nk = s->h_counts[2], fetched = s->h_counts[3];
  st5[3] = (n - nnb + ins) - nk;
  st5[4] = fetched;
  *out_count = nk + fetched;
  if (stats_out) std::memcpy(stats_out, st5, sizeof(st5));
  latmap_status ret = LATMAP_OK;
  if (nk + fetched > cap) ret = sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "sync: output capacity too small");
  if (nwb > 0) {  // written-back rows to the pinned pool over PCIe, overlapping the caller's next work
    S_CHECK(s, cudaEventRecord(s->wb_ev, st));
    S_CHECK(s, cudaStreamWaitEvent(s->wb_st, s->wb_ev, 0));
    scatter_rec_dev_kernel<<<grid_of(nwb * rs / 2), 256, 0, s->wb_st>>>(s->pool_dev, s->dv_wb_idx, s->dv_counts + 0,
                                                                       rs, s->dv_wb_tmp);
    count_launch();
    S_CHECK(s, cudaEventRecord(s->wb_ev, s->wb_st));
    s->wb_pending = true;
  }
  return ret;
}


// fetch_local with device outputs (d_origin: ascending record indices, d_records optional AoS
// gather) and the store's persistent scratch: the radius scan (count, scan, emit) and one count
// readback. *count = hits (also when > cap: nothing is written then).
latmap_status latmap_store_fetch_local_device(latmap_store* s, const float center[3], float radius, int64_t* d_origin,
                                              int64_t cap, float* d_records, int64_t* count) {
  if (!s || !center || (!count && (d_origin || d_records))) return LATMAP_ERR_INVALID_ARGUMENT;
  if (!(radius > 0.f)) return sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "fetch_local: radius must be > 0");
  wb_wait(s);
  if (count) *count = 0;
  if (s->size == 0) return LATMAP_OK;
  cudaStream_t st = s->st;
  const int64_t ps = s->size;
  if (!s->dv_counts) {
    S_CHECK(s, cudaMalloc(&s->dv_counts, sizeof(int64_t) * 8));
    S_CHECK(s, cudaHostAlloc(&s->h_counts, sizeof(int64_t) * 8, 0));
  }
  const int64_t nb = compact_blocks(ps);
  if (s->dv_cnt_cap < nb + 1) {
    if (s->dv_cnt) cudaFree(s->dv_cnt);
    s->dv_cnt_cap = nb + 1 + nb / 4;
    S_CHECK(s, cudaMalloc(&s->dv_cnt, sizeof(int32_t) * s->dv_cnt_cap));
  }
  if (s->dv_pool_cap < ps) {
    if (s->dv_present) cudaFree(s->dv_present);
    if (s->dv_fetch) cudaFree(s->dv_fetch);
    S_CHECK(s, cudaMalloc(&s->dv_fetch, sizeof(int64_t) * (ps + ps / 4)));
    S_CHECK(s, cudaMalloc(&s->dv_present, ps + ps / 4));
    s->dv_pool_cap = ps + ps / 4;
  }
  const float r2 = radius * radius;
  // emit straight into the caller's buffer when it can hold every record, else into scratch
  int64_t* out = d_origin && cap >= ps ? d_origin : s->dv_fetch;
  {
    const latmap_status rc = radius_compact(s, center, r2, nullptr, out, s->dv_counts + 4);
    if (rc != LATMAP_OK) return rc;
  }
  if (!count) return LATMAP_OK;  // scan only: the count stays on the device (timing)
  S_CHECK(s, cudaMemcpyAsync(s->h_counts + 4, s->dv_counts + 4, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  S_CHECK(s, cudaStreamSynchronize(st));
  const int64_t total = s->h_counts[4];
  *count = total;
  if (d_origin && total > cap) return sfail(s, LATMAP_ERR_INVALID_ARGUMENT, "fetch_local: output capacity too small");
  if (d_origin && out != d_origin && total > 0)
    S_CHECK(s, cudaMemcpyAsync(d_origin, out, sizeof(int64_t) * total, cudaMemcpyDeviceToDevice, st));
  if (d_records && total > 0) {
    gather_kernel<<<grid_of(total * s->rs), 256, 0, st>>>(s->pool_dev, out, total, s->rs, d_records);
    count_launch();
  }
  return LATMAP_OK;
}

}  // extern "C"
