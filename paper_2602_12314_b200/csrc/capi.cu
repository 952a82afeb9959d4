// capi.cu — the C-ABI (include/latmap_b200.h): contexts, operator entry points and the
// device-resident session that runs one Stage-I iteration (pipeline.cpp:236-246).
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <array>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/latmap_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace lm {

static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_launch_counter(int64_t*) {}
static std::atomic<const char*> g_sticky{nullptr};
void set_sticky_error(const char* msg) { g_sticky.store(msg); }
const char* take_sticky_error() { return g_sticky.exchange(nullptr); }

static thread_local std::string t_err;
latmap_status set_cuda_error(cudaError_t e, const char* what, const char* file, int line) {
  t_err = std::string(cudaGetErrorString(e)) + " at " + what + " (" + file + ":" + std::to_string(line) + ")";
  return e == cudaErrorMemoryAllocation ? LATMAP_ERR_OUT_OF_MEMORY : LATMAP_ERR_CUDA;
}

// quat_to_rot (core/se3.hpp:12-23) in the reference's float op order; returns false on a
// zero-norm or non-finite quaternion (std::invalid_argument in the reference).
static bool quat_to_rot(const float q[4], float r[9]) {
  const float ss = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
  const float n = std::sqrt(ss);
  if (!(n > 0.f) || !std::isfinite((double)n)) return false;
  const float w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  r[0] = 1.f - 2.f * (y * y + z * z);
  r[1] = 2.f * (x * y - w * z);
  r[2] = 2.f * (x * z + w * y);
  r[3] = 2.f * (x * y + w * z);
  r[4] = 1.f - 2.f * (x * x + z * z);
  r[5] = 2.f * (y * z - w * x);
  r[6] = 2.f * (x * z - w * y);
  r[7] = 2.f * (y * z + w * x);
  r[8] = 1.f - 2.f * (x * x + y * y);
  return true;
}

static bool pose_mats(const latmap_pose& p, float rot_cw[9], float rot_wc[9]) {
  float r[9];
  if (!quat_to_rot(p.rotation, r)) return false;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      rot_wc[3 * i + j] = r[3 * i + j];
      rot_cw[3 * i + j] = r[3 * j + i];
    }
  return true;
}

static bool intr_valid(const latmap_intrinsics& i) {  // Intrinsics::valid, types.hpp:46-49
  return i.fx > 0 && i.fy > 0 && i.width > 0 && i.height > 0 && i.cx >= 0 && i.cx < (float)i.width && i.cy >= 0 &&
         i.cy < (float)i.height;
}

static Intr to_intr(const latmap_intrinsics& i) { return Intr{i.fx, i.fy, i.cx, i.cy, i.width, i.height}; }

template <class T>
static cudaError_t dgrow(T*& p, size_t& cap, size_t n) {
  if (n <= cap && p) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1));
  if (e == cudaSuccess) cap = n;
  return e;
}

// Owns the device buffers of a RenderWork.
struct RenderBufs {
  RenderWork w;
  size_t c_rec = 0, c_tiles = 0, c_keys = 0, c_px = 0, c_cnt = 0, c_geo = 0;
  float* geo_acc = nullptr;
  cudaError_t ensure(int64_t n, int width, int height, int64_t pairs) {
    cudaError_t e;
    w.width = width;
    w.height = height;
    w.tiles_x = (width + kTile - 1) / kTile;
    w.tiles_y = (height + kTile - 1) / kTile;
    const size_t nt = (size_t)w.tiles_x * w.tiles_y;
    const size_t n1 = (size_t)std::max<int64_t>(n, 1);
    if (n1 > c_rec) {
      size_t a = 0, b = 0;
      if (w.rec) cudaFree(w.rec), w.rec = nullptr;
      if (w.dkey) cudaFree(w.dkey), w.dkey = nullptr;
      if (w.big) cudaFree(w.big), w.big = nullptr;
      size_t c = 0;
      if ((e = dgrow(w.rec, a, n1))) return e;
      if ((e = dgrow(w.dkey, b, n1))) return e;
      if ((e = dgrow(w.big, c, n1))) return e;
      c_rec = n1;
    }
    size_t c1 = c_tiles, c2 = c_tiles, c3 = c_tiles, c4 = c_tiles, c5 = c_tiles;
    if (nt + 1 > c_tiles) {
      c1 = c2 = c3 = c4 = c5 = 0;
      if ((e = dgrow(w.tile_order, c5, nt + 1))) return e;
      if ((e = dgrow(w.tile_count, c1, nt + 1))) return e;
      if ((e = dgrow(w.tile_offset, c2, nt + 1))) return e;
      if ((e = dgrow(w.tile_cursor, c3, nt + 1))) return e;
      if ((e = dgrow(w.tile_max_last, c4, nt + 1))) return e;
      c_tiles = nt + 1;
    }
    if ((size_t)pairs > c_keys || !w.keys) {
      size_t a = 0, b = 0;
      if (w.keys) cudaFree(w.keys), w.keys = nullptr;
      if (w.keys_tmp) cudaFree(w.keys_tmp), w.keys_tmp = nullptr;
      c_keys = (size_t)std::max<int64_t>(pairs, 1);
      if ((e = dgrow(w.keys, a, c_keys))) return e;
      if ((e = dgrow(w.keys_tmp, b, c_keys))) return e;
    }
    w.pair_cap = (int64_t)c_keys;
    size_t px = (size_t)width * height;
    if (px > c_px) {
      size_t a = 0, b = 0;
      if (w.px_last) cudaFree(w.px_last), w.px_last = nullptr;
      if (w.px_T) cudaFree(w.px_T), w.px_T = nullptr;
      if ((e = dgrow(w.px_last, a, px))) return e;
      if ((e = dgrow(w.px_T, b, px))) return e;
      c_px = px;
    }
    if ((e = dgrow(w.counters, c_cnt, 8))) return e;
    if (n1 * 8 > c_geo || !geo_acc) {
      if ((e = dgrow(geo_acc, c_geo, n1 * 8))) return e;
      if ((e = cudaMemset(geo_acc, 0, sizeof(float) * n1 * 8))) return e;
    }
    w.n_cap = n;
    return cudaSuccess;
  }
  void release() {
    for (void* p : {(void*)w.rec, (void*)w.tile_count, (void*)w.tile_offset, (void*)w.tile_cursor, (void*)w.keys,
                    (void*)w.keys_tmp, (void*)w.dkey, (void*)w.px_last, (void*)w.px_T, (void*)w.counters, (void*)w.big,
                    (void*)w.tile_max_last, (void*)w.tile_order, (void*)geo_acc})
      if (p) cudaFree(p);
    w = RenderWork{};
    geo_acc = nullptr;
    c_rec = c_tiles = c_keys = c_px = c_cnt = c_geo = 0;
  }
};

}  // namespace lm

using namespace lm;

struct latmap_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches0 = 0;
  bool exact_blend = false;  // parity mode: separately rounded accumulation in the forward blend
  bool deterministic = false;  // fixed-order gradient reductions (bit-reproducible backward)
  DetScratch det;              // the deterministic render backward's per-(splat, tile) rows
  int32_t decoder_path = 0;  // bf16 decoder: 0 auto, 1 fused on-chip (DEC1/DEC2), 2 staged (DL1-DL5)
  int32_t reconstruct_precision = 0;  // standalone reconstruct: 0 fp32 SIMT, 1 bf16 tcgen05 where supported
  cudaStream_t copy_stream = nullptr;  // keyframe uploads (overlap the step's render of earlier frames)
};

struct latmap_render_cache {
  latmap_ctx* ctx = nullptr;
  RenderBufs bufs;
  bool valid = false;
  int64_t source_count = 0;
  latmap_pose pose{};
  latmap_intrinsics intr{};
  int32_t ds = 0;
};

#define CTX_CHECK(ctx, expr)                    \
  do {                                          \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) {                    \
      latmap_status _s = set_cuda_error(_e, #expr, __FILE__, __LINE__); \
      (ctx)->err = t_err;                       \
      return _s;                                \
    }                                           \
  } while (0)

static latmap_status fail(latmap_ctx* ctx, latmap_status s, const char* msg) {
  if (ctx) ctx->err = msg;
  return s;
}

// error text for clients of the C-ABI built into the library (pipeline.cu) that fail before
// they own a handle of their own
latmap_status lm_ctx_fail(latmap_ctx* ctx, latmap_status s, const char* msg) { return fail(ctx, s, msg); }

static latmap_status post_launch(latmap_ctx* ctx) {
  if (const char* m = take_sticky_error()) {
    t_err = m;
    ctx->err = t_err;
    return LATMAP_ERR_CUDA;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    latmap_status s = set_cuda_error(e, "kernel launch", __FILE__, __LINE__);
    ctx->err = t_err;
    return s;
  }
  return LATMAP_OK;
}

extern "C" {

void latmap_default_config(latmap_config* c) {  // config.hpp:10-71 defaults
  std::memset(c, 0, sizeof(*c));
  c->lambda_cos = 0.5f;
  c->lambda_l2 = 0.5f;
  c->lambda_trust = 0.2f;
  c->trust_delta = 0.1f;
  c->lambda_i1 = 0.2f;
  c->lambda_i2 = 0.8f;
  c->lambda_rgb = 1.0f;
  c->lambda_depth = 0.1f;
  c->lambda_feat = 5.0f;
  c->lr_proj = 0.01f;
  c->lr_dict = 0.01f;
  c->lr_position = 1e-4f;
  c->lr_rotation = 1e-3f;
  c->lr_color = 2.5e-3f;
  c->lr_log_scale = 5e-3f;
  c->lr_opacity = 5e-2f;
  c->lr_feature = 2.5e-3f;
  c->scene_extent = 1.0f;
  c->softmax_temp = 1.0f;
  c->dict_learn = 1;
  c->segment_mode = 0;
  c->decoder_precision = 0;
}

latmap_status latmap_ctx_create(int32_t device, void* stream, latmap_ctx** out) {
  if (!out) return LATMAP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    t_err = "no CUDA device available (the B200 path has no CPU fallback)";
    return LATMAP_ERR_CUDA;
  }
  if (device < 0 || device >= count) return LATMAP_ERR_INVALID_ARGUMENT;
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaSetDevice", __FILE__, __LINE__);
  // stream-ordered allocations (store sync, k-means, row import scratch) stay cached in the
  // device's default pool instead of returning to the driver at every synchronisation
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  latmap_ctx* c = new latmap_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->launches0 = g_launches.load();
  *out = c;
  return LATMAP_OK;
}

latmap_status latmap_ctx_destroy(latmap_ctx* ctx) {
  if (!ctx) return LATMAP_ERR_INVALID_ARGUMENT;
  cudaStreamSynchronize(ctx->stream);
  ctx->det.release();
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  delete ctx;
  return LATMAP_OK;
}

latmap_status latmap_ctx_set_stream(latmap_ctx* ctx, void* stream) {
  if (!ctx) return LATMAP_ERR_INVALID_ARGUMENT;
  ctx->stream = (cudaStream_t)stream;
  return LATMAP_OK;
}

latmap_status latmap_ctx_set_exact_blend(latmap_ctx* ctx, int32_t exact) {
  if (!ctx) return LATMAP_ERR_INVALID_ARGUMENT;
  ctx->exact_blend = exact != 0;
  return LATMAP_OK;
}

latmap_status latmap_ctx_set_deterministic(latmap_ctx* ctx, int32_t on) {
  if (!ctx) return LATMAP_ERR_INVALID_ARGUMENT;
  ctx->deterministic = on != 0;
  if (!on) ctx->det.release();
  return LATMAP_OK;
}

latmap_status latmap_ctx_set_decoder_path(latmap_ctx* ctx, int32_t path) {
  if (!ctx || path < 0 || path > 2) return LATMAP_ERR_INVALID_ARGUMENT;
  ctx->decoder_path = path;
  return LATMAP_OK;
}

latmap_status latmap_ctx_set_reconstruct_precision(latmap_ctx* ctx, int32_t precision) {
  if (!ctx || precision < 0 || precision > 1) return LATMAP_ERR_INVALID_ARGUMENT;
  ctx->reconstruct_precision = precision;
  return LATMAP_OK;
}

latmap_status latmap_ctx_synchronize(latmap_ctx* ctx) {
  if (!ctx) return LATMAP_ERR_INVALID_ARGUMENT;
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  return LATMAP_OK;
}

const char* latmap_ctx_last_error(const latmap_ctx* ctx) { return ctx ? ctx->err.c_str() : t_err.c_str(); }

void* latmap_ctx_stream(const latmap_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int64_t latmap_ctx_launch_count(const latmap_ctx* ctx) { return g_launches.load() - (ctx ? ctx->launches0 : 0); }

// ------------------------------------------------------------------------------- renderer
latmap_status latmap_project_gaussian(latmap_ctx* ctx, const float position[3], const float rotation[4],
                                      const float log_scale[3], float opacity_logit, const latmap_pose* pose,
                                      const latmap_intrinsics* intr, int32_t* visible, float mean2d[2],
                                      float cov2d[4], float* depth) {
  if (!ctx || !pose || !intr || !visible) return LATMAP_ERR_INVALID_ARGUMENT;
  float rcw[9], rwc[9];
  if (!pose_mats(*pose, rcw, rwc)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "quat_to_rot: zero-norm quaternion");
  float in[11];
  std::memcpy(in, position, 12);
  std::memcpy(in + 3, rotation, 16);
  std::memcpy(in + 7, log_scale, 12);
  in[10] = opacity_logit;
  float* d = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&d, sizeof(float) * 19, ctx->stream));
  CTX_CHECK(ctx, cudaMemcpyAsync(d, in, sizeof(in), cudaMemcpyHostToDevice, ctx->stream));
  project_single(ctx->stream, d, rcw, pose->translation, to_intr(*intr), d + 11);
  float out[8];
  CTX_CHECK(ctx, cudaMemcpyAsync(out, d + 11, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CHECK(ctx, cudaFreeAsync(d, ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  *visible = out[0] != 0.f;
  if (*visible) {
    if (mean2d) mean2d[0] = out[1], mean2d[1] = out[2];
    if (cov2d) std::memcpy(cov2d, out + 3, 16);
    if (depth) *depth = out[7];
  }
  return LATMAP_OK;
}

latmap_status latmap_render_cache_create(latmap_ctx* ctx, latmap_render_cache** out) {
  if (!ctx || !out) return LATMAP_ERR_INVALID_ARGUMENT;
  auto* c = new latmap_render_cache();
  c->ctx = ctx;
  *out = c;
  return LATMAP_OK;
}

latmap_status latmap_render_cache_destroy(latmap_render_cache* c) {
  if (!c) return LATMAP_ERR_INVALID_ARGUMENT;
  cudaStreamSynchronize(c->ctx->stream);
  c->bufs.release();
  delete c;
  return LATMAP_OK;
}

static MapPtrs map_ptrs(const latmap_map* m) {
  return MapPtrs{m->n, m->query_dim, m->positions, m->rotations, m->colors, m->log_scales, m->opacity_logits,
                 m->features};
}

latmap_status latmap_render(latmap_ctx* ctx, const latmap_map* map, const latmap_pose* pose,
                            const latmap_intrinsics* intr, latmap_render_cache* cache, float* color, float* depth,
                            float* query, float* alpha) {
  if (!ctx || !map || !pose || !intr || !cache) return LATMAP_ERR_INVALID_ARGUMENT;
  if (!intr_valid(*intr)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "render: invalid intrinsics");
  if (map->query_dim < 1 || map->query_dim > 64)
    return fail(ctx, LATMAP_ERR_UNSUPPORTED, "render: query_dim must be in [1, 64]");
  float rcw[9], rwc[9];
  if (!pose_mats(*pose, rcw, rwc)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "quat_to_rot: zero-norm quaternion");
  cudaStream_t st = ctx->stream;
  RenderBufs& b = cache->bufs;
  const MapPtrs mp = map_ptrs(map);
  const Intr in = to_intr(*intr);
  int64_t guess = std::max<int64_t>(b.w.pair_cap, 1);
  CTX_CHECK(ctx, b.ensure(map->n, intr->width, intr->height, guess));
  // sizing pass: project + scan, then read back the tile-pair count
  render_forward(st, mp, rcw, pose->translation, in, b.w, color, depth, query, alpha, false, true);
  int64_t counters[4];
  CTX_CHECK(ctx, cudaMemcpyAsync(counters, b.w.counters, sizeof(counters), cudaMemcpyDeviceToHost, st));
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  if (counters[0] > b.w.pair_cap) CTX_CHECK(ctx, b.ensure(map->n, intr->width, intr->height, counters[0]));
  render_forward(st, mp, rcw, pose->translation, in, b.w, color, depth, query, alpha, true, false, true,
                 ctx->exact_blend);
  latmap_status s = post_launch(ctx);
  if (s != LATMAP_OK) return s;
  cache->valid = true;
  cache->source_count = map->n;
  cache->pose = *pose;
  cache->intr = *intr;
  cache->ds = map->query_dim;
  return LATMAP_OK;
}

latmap_status latmap_render_backward(latmap_ctx* ctx, const latmap_map* map, const latmap_pose* pose,
                                     const latmap_intrinsics* intr, const latmap_render_cache* cache,
                                     const float* d_color, const float* d_depth, const float* d_query,
                                     latmap_map* grads) {
  if (!ctx || !map || !pose || !intr || !cache || !grads) return LATMAP_ERR_INVALID_ARGUMENT;
  // render.cpp:256-260: the cache must come from render() on identical inputs
  const bool pose_match = std::memcmp(cache->pose.rotation, pose->rotation, 16) == 0 &&
                          std::memcmp(cache->pose.translation, pose->translation, 12) == 0;
  if (!cache->valid || cache->source_count != map->n || cache->intr.width != intr->width ||
      cache->intr.height != intr->height || !pose_match)
    return fail(ctx, LATMAP_ERR_STALE_CACHE, "render_backward: render cache does not match inputs");
  if (map->n == 0) return LATMAP_OK;
  float rcw[9], rwc[9];
  pose_mats(*pose, rcw, rwc);
  auto& b = const_cast<latmap_render_cache*>(cache)->bufs;
  CTX_CHECK(ctx, cudaMemsetAsync(b.geo_acc, 0, sizeof(float) * 8 * map->n, ctx->stream));
  set_deterministic(ctx->deterministic);
  render_backward(ctx->stream, map_ptrs(map), rcw, rwc, pose->translation, to_intr(*intr), b.w, d_color, d_depth,
                  d_query, b.geo_acc, map_ptrs(grads), true, ctx->deterministic ? &ctx->det : nullptr);
  return post_launch(ctx);
}

latmap_status latmap_render_cache_splats(latmap_ctx* ctx, const latmap_render_cache* cache,
                                         latmap_projected_splat* out, int64_t cap, int64_t* count) {
  if (!ctx || !cache || !count || !cache->valid) return LATMAP_ERR_INVALID_ARGUMENT;
  const int64_t n = cache->source_count;
  std::vector<SplatRec> rec((size_t)std::max<int64_t>(n, 1));
  if (n > 0)
    CTX_CHECK(ctx, cudaMemcpyAsync(rec.data(), cache->bufs.w.rec, sizeof(SplatRec) * n, cudaMemcpyDeviceToHost,
                                   ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    const SplatRec& r = rec[i];
    if (r.x0 > r.x1) continue;
    if (out && k < cap) {
      latmap_projected_splat& s = out[k];
      s.mean2d[0] = r.mean_x;
      s.mean2d[1] = r.mean_y;
      s.cov_inv[0] = r.a00;
      s.cov_inv[1] = r.a01;
      s.cov_inv[2] = r.a10;
      s.cov_inv[3] = r.a11;
      s.depth = r.depth;
      s.alpha = r.alpha;
      s.source = (int32_t)i;
      s.x0 = r.x0;
      s.x1 = r.x1;
      s.y0 = r.y0;
      s.y1 = r.y1;
    }
    ++k;
  }
  *count = k;
  return (out && k > cap) ? LATMAP_ERR_INVALID_ARGUMENT : LATMAP_OK;
}

latmap_status latmap_render_cache_tiles(latmap_ctx* ctx, const latmap_render_cache* cache, int32_t* tile_offsets,
                                        int32_t* tile_sources, int64_t cap, int32_t* tiles_x, int32_t* tiles_y,
                                        int64_t* pairs) {
  if (!ctx || !cache || !cache->valid) return LATMAP_ERR_INVALID_ARGUMENT;
  const RenderWork& w = cache->bufs.w;
  const int nt = w.tiles_x * w.tiles_y;
  int64_t counters[4];
  CTX_CHECK(ctx, cudaMemcpyAsync(counters, w.counters, sizeof(counters), cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  if (tiles_x) *tiles_x = w.tiles_x;
  if (tiles_y) *tiles_y = w.tiles_y;
  if (pairs) *pairs = counters[0];
  if (tile_offsets)
    CTX_CHECK(ctx, cudaMemcpy(tile_offsets, w.tile_offset, sizeof(int32_t) * (nt + 1), cudaMemcpyDeviceToHost));
  if (tile_sources) {
    if (cap < counters[0]) return LATMAP_ERR_INVALID_ARGUMENT;
    std::vector<uint64_t> keys((size_t)std::max<int64_t>(counters[0], 1));
    if (counters[0] > 0)
      CTX_CHECK(ctx, cudaMemcpy(keys.data(), w.keys, sizeof(uint64_t) * counters[0], cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < counters[0]; ++i) tile_sources[i] = (int32_t)(uint32_t)keys[i];
  }
  return LATMAP_OK;
}

// ------------------------------------------------------------------------------- decoder ops
latmap_status latmap_reconstruct(latmap_ctx* ctx, const float* q, int64_t n, int32_t ds, const float* atoms,
                                 const float* proj, int64_t k, int32_t df, float temperature, float* out,
                                 float* attention) {
  if (!ctx || n < 0 || ds < 1 || k < 1 || df < 1 || !out) return LATMAP_ERR_INVALID_ARGUMENT;
  if (!(temperature > 0.f)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "reconstruct: temperature must be > 0");
  if (n == 0) return LATMAP_OK;
  cudaStream_t st = ctx->stream;
  if (ctx->reconstruct_precision == 1 && !attention && reconstruct_tc_supported(k, ds, df)) {
    CTX_CHECK(ctx, reconstruct_tc(st, q, n, ds, atoms, proj, k, df, temperature, out));
    return post_launch(ctx);
  }
  float *qw = nullptr, *att = attention;
  CTX_CHECK(ctx, cudaMallocAsync(&qw, sizeof(float) * n * df, st));
  if (!att) CTX_CHECK(ctx, cudaMallocAsync(&att, sizeof(float) * n * k, st));
  reconstruct(st, q, n, ds, atoms, proj, k, df, temperature, out, att, qw);
  CTX_CHECK(ctx, cudaFreeAsync(qw, st));
  if (!attention) CTX_CHECK(ctx, cudaFreeAsync(att, st));
  return post_launch(ctx);
}

latmap_status latmap_reconstruct_backward(latmap_ctx* ctx, const float* q, const float* attention, int64_t n,
                                          int32_t ds, const float* atoms, const float* proj, int64_t k, int32_t df,
                                          float temperature, const float* d_rec, float* d_q, float* d_proj,
                                          float* d_atoms) {
  if (!ctx || !q || !attention || !d_rec || !d_q || !d_proj || !d_atoms) return LATMAP_ERR_INVALID_ARGUMENT;
  set_deterministic(ctx->deterministic);
  cudaStream_t st = ctx->stream;
  if (n == 0) {
    CTX_CHECK(ctx, cudaMemsetAsync(d_proj, 0, sizeof(float) * ds * df, st));
    CTX_CHECK(ctx, cudaMemsetAsync(d_atoms, 0, sizeof(float) * k * df, st));
    return LATMAP_OK;
  }
  float *snk = nullptr, *sndf = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&snk, sizeof(float) * n * k, st));
  CTX_CHECK(ctx, cudaMallocAsync(&sndf, sizeof(float) * n * df, st));
  reconstruct_backward(st, q, attention, n, ds, atoms, proj, k, df, temperature, d_rec, d_q, d_proj, d_atoms, snk,
                       sndf, nullptr);
  CTX_CHECK(ctx, cudaFreeAsync(snk, st));
  CTX_CHECK(ctx, cudaFreeAsync(sndf, st));
  return post_launch(ctx);
}

latmap_status latmap_trust_region_penalty(latmap_ctx* ctx, const float* atoms, const float* anchor, int64_t k,
                                          int32_t df, float delta, float* d_atoms, float* penalty) {
  if (!ctx || !atoms || !anchor) return LATMAP_ERR_INVALID_ARGUMENT;
  cudaStream_t st = ctx->stream;
  double* dp = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&dp, sizeof(double), st));
  CTX_CHECK(ctx, cudaMemsetAsync(dp, 0, sizeof(double), st));
  if (d_atoms) CTX_CHECK(ctx, cudaMemsetAsync(d_atoms, 0, sizeof(float) * k * df, st));
  trust_region(st, atoms, anchor, k, df, delta, d_atoms, 1.f, dp);
  double v = 0;
  CTX_CHECK(ctx, cudaMemcpyAsync(&v, dp, sizeof(double), cudaMemcpyDeviceToHost, st));
  CTX_CHECK(ctx, cudaFreeAsync(dp, st));
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  if (penalty) *penalty = (float)v;
  return post_launch(ctx);
}

latmap_status latmap_ssim(latmap_ctx* ctx, const float* a, const float* b, int32_t h, int32_t w, int32_t ch,
                          float* d_a, float* value) {
  if (!ctx || !a || !b || h < 1 || w < 1 || ch < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  cudaStream_t st = ctx->stream;
  float* scratch = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&scratch, sizeof(float) * ssim_scratch_floats(h, w, ch), st));
  const double v = ssim_host(st, a, b, h, w, ch, d_a, scratch);
  CTX_CHECK(ctx, cudaFreeAsync(scratch, st));
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  if (value) *value = (float)v;
  return post_launch(ctx);
}

// ------------------------------------------------------------------------------- Adam
static void corr_tables(std::vector<float>& c1, std::vector<float>& c2, int len) {
  c1.resize(len);
  c2.resize(len);
  for (int t = 1; t <= len; ++t) {  // adam.hpp:74-75: T(1) - T(std::pow(beta, double(step)))
    c1[t - 1] = 1.f - (float)std::pow(0.9, (double)t);
    c2[t - 1] = 1.f - (float)std::pow(0.999, (double)t);
  }
}
static const int kCorrLen = 1 << 16;

latmap_status latmap_device_alloc(latmap_ctx* ctx, int64_t bytes, void** out) {
  if (!ctx || !out || bytes < 0) return LATMAP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (bytes == 0) return LATMAP_OK;
  cudaError_t e = cudaMalloc(out, (size_t)bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(ctx, LATMAP_ERR_OUT_OF_MEMORY, "device_alloc: out of device memory");
  }
  CTX_CHECK(ctx, e);
  return LATMAP_OK;
}

latmap_status latmap_device_free(latmap_ctx* ctx, void* p) {
  if (!ctx) return LATMAP_ERR_INVALID_ARGUMENT;
  if (p) {
    CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
    CTX_CHECK(ctx, cudaFree(p));
  }
  return LATMAP_OK;
}

latmap_status latmap_copy(latmap_ctx* ctx, void* dst, const void* src, int64_t bytes, int32_t direction) {
  if (!ctx || bytes < 0 || direction < 0 || direction > 2 || (bytes > 0 && (!dst || !src)))
    return LATMAP_ERR_INVALID_ARGUMENT;
  if (bytes == 0) return LATMAP_OK;
  const cudaMemcpyKind kind =
      direction == 0 ? cudaMemcpyHostToDevice : (direction == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  CTX_CHECK(ctx, cudaMemcpyAsync(dst, src, (size_t)bytes, kind, ctx->stream));
  if (direction == 1) CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_rgb_loss(latmap_ctx* ctx, const float* rendered, const float* observed, int32_t h, int32_t w,
                              int32_t channels, float lambda_i1, float lambda_i2, float* grad, float* value,
                              float* l1, float* ssim_loss) {
  if (!ctx || h < 0 || w < 0 || channels < 1 || !value || ((int64_t)h * w > 0 && (!rendered || !observed)))
    return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "rgb_loss: invalid arguments");
  float out[3];
  CTX_CHECK(ctx, rgb_loss_dev(ctx->stream, rendered, observed, h, w, channels, lambda_i1, lambda_i2, grad, out));
  *value = out[0];
  if (l1) *l1 = out[1];
  if (ssim_loss) *ssim_loss = out[2];
  return post_launch(ctx);
}

latmap_status latmap_depth_loss(latmap_ctx* ctx, const float* rendered, const float* observed, const float* alpha,
                                int64_t n, float* grad, float* value, int32_t* flagged) {
  if (!ctx || n < 0 || !value || !flagged || (n > 0 && (!rendered || !observed || !alpha)))
    return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "depth_loss: invalid arguments");
  int fl = 0;
  CTX_CHECK(ctx, depth_loss_dev(ctx->stream, rendered, observed, alpha, n, grad, value, &fl));
  *flagged = fl;
  return post_launch(ctx);
}

latmap_status latmap_feature_loss(latmap_ctx* ctx, const float* reconstructed, const float* target, int64_t n,
                                  int32_t embed_dim, const float* atoms, const float* anchor, int64_t k, float delta,
                                  float lambda_cos, float lambda_l2, float lambda_trust, float* d_reconstructed,
                                  float* d_atoms_trust, float terms[4], int32_t* zero_norm_flagged) {
  if (!ctx || n < 0 || embed_dim < 1 || k < 0 || !terms || !zero_norm_flagged ||
      (n > 0 && (!reconstructed || !target)) || (k > 0 && (!atoms || !anchor)))
    return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "feature_loss: invalid arguments");
  int fl = 0;
  CTX_CHECK(ctx, feature_loss_dev(ctx->stream, reconstructed, target, n, embed_dim, atoms, anchor, k, delta, lambda_cos,
                                  lambda_l2, lambda_trust, d_reconstructed, d_atoms_trust, terms, &fl));
  *zero_norm_flagged = fl;
  return post_launch(ctx);
}

latmap_status latmap_adam_step(latmap_ctx* ctx, float* param, const float* grad, float* m, float* v, int64_t count,
                               int64_t* step, int64_t* skipped, float lr, int32_t* applied) {
  if (!ctx || !param || !grad || !m || !v || !step || !skipped) return LATMAP_ERR_INVALID_ARGUMENT;
  cudaStream_t st = ctx->stream;
  const int64_t t = *step + 1;
  float c1 = 1.f, c2 = 1.f;
  if (t <= kCorrLen) {
    c1 = 1.f - (float)std::pow(0.9, (double)t);
    c2 = 1.f - (float)std::pow(0.999, (double)t);
  }
  struct Aux {
    int64_t steps, skipped;
    int32_t flags[2];
    float c1, c2;
  } aux{*step, *skipped, {0, 0}, c1, c2};
  char* d = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&d, sizeof(Aux), st));
  CTX_CHECK(ctx, cudaMemcpyAsync(d, &aux, sizeof(Aux), cudaMemcpyHostToDevice, st));
  Aux* da = (Aux*)d;
  // table of length 1 holding the bias corrections for step t
  AdamBlock blk{0, count, lr, 0};
  int64_t one_back = 0;  // steps array seen by the kernel: t - 1 - 0 -> use table index 0
  (void)one_back;
  int64_t* d_steps = &da->steps;
  // The kernel computes t = steps + 1 and indexes corr[t-1]; pass a shifted table pointer.
  const float* c1p = &da->c1 - *step;
  const float* c2p = &da->c2 - *step;
  adam_flat(st, param, grad, m, v, &blk, 1, d_steps, &da->skipped, c1p, c2p, (int32_t)std::min<int64_t>(t, 1 << 30),
            da->flags, nullptr, nullptr);
  Aux back;
  CTX_CHECK(ctx, cudaMemcpyAsync(&back, d, sizeof(Aux), cudaMemcpyDeviceToHost, st));
  CTX_CHECK(ctx, cudaFreeAsync(d, st));
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  if (applied) *applied = back.skipped == *skipped;
  *step = back.steps;
  *skipped = back.skipped;
  return post_launch(ctx);
}

}  // extern "C"

// ------------------------------------------------------------------------------- session
namespace {
struct FrameDev {
  float* rgb = nullptr;
  float* depth = nullptr;
  int32_t* assign = nullptr;
  float* feats = nullptr;
  size_t c_px = 0, c_feat = 0;
  int64_t n_set = 0, n_sup = 0;    // n_sup: host value in segment mode only (pixel mode: stat[0])
  int64_t* stat = nullptr;          // device [supervised count, out-of-range count] (set_frames)
  // segment mode (objective.cpp:37-64): assignment rows present in the frame, ascending
  int32_t* seg_rows = nullptr;    // n_sup: assignment row of each supervision row
  int32_t* seg_of = nullptr;      // n_set: supervision row of an assignment row (-1 = absent)
  float* seg_inv = nullptr;       // n_sup: 1 / pixels of the segment
  size_t c_seg = 0;
  latmap_pose pose{};
  float rcw[9], rwc[9];
};
constexpr int kPart = 8;  // per-frame loss partial slots (see losses.cu / decoder.cu)
// partials tail after the frame slots: [0] trust penalty, [1] tile-list overflow flag, [2..9] the
// 8 Adam blocks' non-finite flags of the sharded step (all summed by the partials all-reduce)
constexpr int kTail = 16;
constexpr int kTailOverflow = 1, kTailBlockFlags = 2;
// slack after the flat parameter / gradient / moment buffers: the sharded step's reduce-scatter
// and all-gather address nranks equal 4-aligned shards (<= 4 * 64 floats past the last block)
constexpr int64_t kShardSlack = 256;
}  // namespace

// session parameter blocks start on 16-byte boundaries (vector loads / cp.async of rows)
static inline int64_t pad4(int64_t x) { return (x + 3) & ~int64_t(3); }

struct latmap_session {
  latmap_ctx* ctx = nullptr;
  latmap_config cfg{};
  int64_t n = 0, k = 0;
  int32_t ds = 0, df = 0;
  latmap_intrinsics intr{};
  int64_t total = 0, off[9] = {}, len[8] = {};  // block offsets (16-byte aligned) and true lengths
  float *params = nullptr, *grads = nullptr, *m = nullptr, *v = nullptr, *anchor = nullptr;
  // import_rows builds the next map into a spare set and swaps (no per-frame malloc / free)
  float *sp_params = nullptr, *sp_grads = nullptr, *sp_m = nullptr, *sp_v = nullptr;
  int64_t cur_cap = 0, sp_cap = 0;  // floats per buffer of the current / spare set
  int64_t *steps = nullptr, *skipped = nullptr, *overflow = nullptr;
  int64_t* overflow_steps = nullptr;  // sticky count of Adam steps skipped for a tile-list overflow (any rank)
  int32_t* flags = nullptr;
  float *corr1 = nullptr, *corr2 = nullptr;
  std::vector<FrameDev> frames;
  int32_t nframes = 0, global_batch = 0, add_trust = 1, slot_offset = 0;
  std::vector<RenderBufs> rw;
  std::vector<float*> color, depth, query, alpha;
  float *d_color = nullptr, *d_depth = nullptr, *d_query = nullptr, *ssim_scratch = nullptr;
  float *seg_q = nullptr, *seg_dq = nullptr;  // segment mode: pooled rows and their gradients
  int64_t seg_cap = 0;
  DecoderWork dec;
  double* partials = nullptr;
  int32_t part_frames = 0;
  latmap_loss_breakdown* d_loss = nullptr;
  // the per-frame images hold renders of the current map (ObjectiveOptions::cached_renders)
  bool renders_valid = false;
  // CUDA graph of one Stage-I step (objective + Adam), replayed while the launch sequence and its
  // arguments (frame poses, buffer pointers, sizes) are unchanged
  cudaGraphExec_t step_graph = nullptr;
  cudaGraphExec_t obj_graph = nullptr;  // objective only (want_grad): the multi-GPU path's per-rank part
  int64_t obj_launches = 0;
  cudaStream_t cap_stream = nullptr;
  // set_frames uploads on ctx->copy_stream; up_ev[b] marks frame b's data resident. Every use of
  // frame data waits on it (an external event node when captured), so the render of frame 0 and
  // the uploads of later frames overlap.
  std::vector<cudaEvent_t> up_ev;
  cudaEvent_t ev_ready = nullptr;
  // renders of every frame run ahead on rstream (they only read the map); frame b's losses,
  // decoder and backward on the context stream wait on rend_ev[b]
  cudaStream_t rstream = nullptr;
  cudaStream_t rstream2 = nullptr;  // odd frames (LATMAP_RSTREAMS=1: every render on rstream)
  cudaEvent_t rend_start = nullptr;
  std::vector<cudaEvent_t> rend_ev;
  // frame b's render backward runs on bstream behind its losses + decoder (evD[b]) while frame
  // b+1's losses + decoder proceed on the context stream; the upstream-gradient images
  // alternate between two slots (slot 1 below), reused once frame b-2's backward is done (evB)
  cudaStream_t bstream = nullptr;
  std::vector<cudaEvent_t> evD, evB;
  // latmap_session_step: the colour and feature Adam blocks depend only on the render backward
  // (K8 writes their gradients directly), so once the last frame's K8 is done they are updated on
  // rstream while K9 (geometry gradients), the decoder's step-end reduce and the trust term run
  // on the context stream; session_adam then updates the remaining blocks (LATMAP_EARLY_CF=0: off)
  bool early_cf = false, cf_done = false;
  cudaEvent_t ev_cf = nullptr;
  cudaEvent_t ev_pf = nullptr, ev_pj = nullptr;  // single-keyframe step: preparation fork / join
  // frame b's image losses (colour / depth / SSIM and their gradient images) run on lstream,
  // beside the decoder on the context stream; K8 waits for both (evL[b], evD[b])
  // (LATMAP_LSTREAM=0: on the context stream)
  cudaStream_t lstream = nullptr;
  std::vector<cudaEvent_t> evL;
  float *d_color2 = nullptr, *d_depth2 = nullptr, *d_query2 = nullptr;
  std::vector<float> dict_w;  // DictionaryState::weights (host; k-means maintenance only)
  // latmap_session_save_state / restore_state: the map, dictionary and MapOptimizer state at the
  // start of a keyframe (process_keyframe's StateSnapshot, pipeline.cpp:155-190)
  struct Snapshot {
    bool valid = false;
    int64_t n = 0, total = 0, off[9] = {}, len[8] = {};
    float *params = nullptr, *m = nullptr, *v = nullptr, *anchor = nullptr;
    int64_t cap = 0;
    int64_t steps[8] = {}, skipped[8] = {};
    std::vector<float> dict_w;
  } snap;
  int64_t graph_launches = 0;
  bool graph_exact = false;
  bool graph_det = false;
  int32_t graph_dec_path = 0;
  bool use_graph = true;
  void drop_graph() {
    if (step_graph) cudaGraphExecDestroy(step_graph);
    if (obj_graph) cudaGraphExecDestroy(obj_graph);
    step_graph = obj_graph = nullptr;
  }
  // phase timing with CUDA events on the session stream (bench.py roofline evidence)
  struct Span {
    int phase;
    cudaEvent_t a, b;
  };
  bool prof = false;
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
  double prof_ms[8] = {};
  int64_t prof_cnt[8] = {};
  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void begin(int phase) {
    if (!prof) return;
    Span sp{phase, ev(), ev()};
    cudaEventRecord(sp.a, ctx->stream);
    spans.push_back(sp);
  }
  void end() {
    if (!prof || spans.empty()) return;
    cudaEventRecord(spans.back().b, ctx->stream);
  }
};

namespace {

__global__ void set_double_kernel(double* p, double v) { *p = v; }
__global__ void copy_count_kernel(double* p, const int64_t* v) { *p = (double)*v; }

// gather_supervision's pixel-mode scan (objective.cpp:16-35) on the uploaded assignment: counts
// the supervised pixels (a >= 0) and the out-of-range ones (a >= n_set), which it rewrites to -1
// so no later kernel indexes past the embedding table; the error is reported with the loss read.
__global__ void assign_scan_kernel(int32_t* __restrict__ asg, int64_t npx, int64_t n_set, int64_t* stat) {
  int64_t nsup = 0, bad = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = asg[p];
    if (a >= n_set) {
      asg[p] = -1;
      ++bad;
    } else if (a >= 0) {
      ++nsup;
    }
  }
  nsup = warp_sum_i64(nsup);
  bad = warp_sum_i64(bad);
  if ((threadIdx.x & 31) == 0 && (nsup | bad)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(stat), (unsigned long long)nsup);
    atomicAdd(reinterpret_cast<unsigned long long*>(stat + 1), (unsigned long long)bad);
  }
}

struct LossWeights {
  float lambda_rgb, lambda_i1, lambda_i2, lambda_depth, lambda_feat, lambda_cos, lambda_l2, lambda_trust;
};

// LossBreakdown assembly (objective.cpp:188-190 and 247-261) from the per-frame partial slots
// and the trust slot after them; shared by the device step and the host entry point
// latmap_loss_assemble (the sharded step's all-reduced partials, and the CPU tests).
__host__ __device__ void assemble_loss(const double* partials, int nframes, double npx, float inv_b, LossWeights wt,
                                       latmap_loss_breakdown* out) {
  latmap_loss_breakdown L{};
  for (int b = 0; b < nframes; ++b) {
    const double* p = partials + b * kPart;
    const double nsup = p[7];
    const float l1 = (float)(p[0] / (npx * 3.0));
    const float ss = (float)(p[1] / (npx * 3.0));
    const float ssl = (1.f - ss) / 2.f;
    const bool dflag = p[3] <= 0.0;
    const float ld = dflag ? 0.f : (float)(p[2] / p[3]);
    const float lc = nsup > 0 ? (float)(p[4] / nsup) : 0.f;
    const float ll2 = nsup > 0 ? (float)(p[5] / nsup) : 0.f;
    L.l_rgb += l1 * inv_b;
    L.l_ssim += ssl * inv_b;
    L.l_depth += ld * inv_b;
    L.l_cos += lc * inv_b;
    L.l_l2 += ll2 * inv_b;
    L.depth_empty = L.depth_empty || dflag;
    L.zero_norm_flagged = L.zero_norm_flagged || p[6] != 0.0;
    L.supervised_rows += (int64_t)nsup;
  }
  L.l_trust = (float)partials[nframes * kPart];
  L.total = wt.lambda_rgb * (wt.lambda_i1 * L.l_rgb + wt.lambda_i2 * L.l_ssim) + wt.lambda_depth * L.l_depth +
            wt.lambda_feat * (wt.lambda_cos * L.l_cos + wt.lambda_l2 * L.l_l2 + wt.lambda_trust * L.l_trust);
  *out = L;
}

__global__ void assemble_loss_kernel(const double* partials, int nframes, double npx, float inv_b, LossWeights wt,
                                     latmap_loss_breakdown* out) {
  assemble_loss(partials, nframes, npx, inv_b, wt, out);
}

MapPtrs session_map(latmap_session* s, float* base) {
  return MapPtrs{s->n, s->ds, base + s->off[0], base + s->off[1], base + s->off[2], base + s->off[3],
                 base + s->off[4], base + s->off[5]};
}

latmap_status session_alloc_frames(latmap_session* s, int nf) {
  latmap_ctx* ctx = s->ctx;
  const size_t npx = (size_t)s->intr.width * s->intr.height;
  while ((int)s->frames.size() < nf) s->frames.emplace_back();
  while ((int)s->rw.size() < nf) {
    s->rw.emplace_back();
    float *c, *d, *q, *a;
    CTX_CHECK(ctx, cudaMalloc(&c, sizeof(float) * npx * 3));
    CTX_CHECK(ctx, cudaMalloc(&d, sizeof(float) * npx));
    CTX_CHECK(ctx, cudaMalloc(&q, sizeof(float) * npx * s->ds));
    CTX_CHECK(ctx, cudaMalloc(&a, sizeof(float) * npx));
    s->color.push_back(c);
    s->depth.push_back(d);
    s->query.push_back(q);
    s->alpha.push_back(a);
  }
  const int need_part = std::max(nf, s->global_batch);
  if (need_part > s->part_frames) {
    if (s->partials) cudaFree(s->partials);
    CTX_CHECK(ctx, cudaMalloc(&s->partials, sizeof(double) * ((size_t)need_part * kPart + kTail)));
    s->part_frames = need_part;
  }
  return LATMAP_OK;
}

// ---- segment supervision (objective.cpp:37-64, 147-157): mean rendered query per present
// assignment row, and the per-pixel share of the row gradient
__global__ void seg_pool_kernel(const float* __restrict__ query, const int32_t* __restrict__ assign, int64_t npx,
                                int ds, const int32_t* __restrict__ seg_of, float* __restrict__ qsum) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < npx * ds;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / ds;
    const int a = assign[p];
    if (a < 0) continue;
    atomicAdd(&qsum[(size_t)seg_of[a] * ds + (e % ds)], query[e]);
  }
}
// deterministic variant: block (row r, channel chunk) sums its segment's pixels in raster order
// (per-thread strided partials, then a fixed-order combination)
__global__ void seg_pool_det_kernel(const float* __restrict__ query, const int32_t* __restrict__ assign, int64_t npx,
                                    int ds, const int32_t* __restrict__ seg_of, float* __restrict__ qsum) {
  __shared__ float part[256];
  const int r = blockIdx.x, c = blockIdx.y;
  float acc = 0.f;
  for (int64_t p = threadIdx.x; p < npx; p += blockDim.x) {
    const int a = assign[p];
    if (a >= 0 && seg_of[a] == r) acc += query[p * ds + c];
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (unsigned t = 0; t < blockDim.x; ++t) s += part[t];
    qsum[(size_t)r * ds + c] = s;
  }
}
__global__ void seg_mean_kernel(float* q, const float* __restrict__ inv, int64_t rows, int ds) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * ds;
       e += (int64_t)gridDim.x * blockDim.x)
    q[e] *= inv[e / ds];
}
__global__ void seg_scatter_kernel(const float* __restrict__ dq, const int32_t* __restrict__ assign, int64_t npx,
                                   int ds, const int32_t* __restrict__ seg_of, const float* __restrict__ inv,
                                   float* __restrict__ d_query) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < npx * ds;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / ds;
    const int a = assign[p];
    float v = 0.f;
    if (a >= 0) {
      const int r = seg_of[a];
      v = dq[(size_t)r * ds + (e % ds)] * inv[r];
    }
    d_query[e] = v;
  }
}

// Order `st` after frame b's upload (set_frames). Under stream capture the wait becomes an
// external event node, so replays wait on the latest upload.
static void wait_frame(const latmap_session* s, int b, cudaStream_t st) {
  if (b >= (int)s->up_ev.size()) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  cudaStreamWaitEvent(st, s->up_ev[b], cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0);
}

// One total_objective over the session's keyframes (objective.cpp:67-194). map_grads = false
// skips the image-loss gradients and the render backward (ObjectiveOptions::map_grads);
// use_cache skips the render when the per-frame images still hold renders of the current map
// (ObjectiveOptions::cached_renders, Stage II of pipeline.cpp:250-259).
__global__ void overflow_slot_kernel(const int64_t* flag, double* slot) { *slot = *flag ? 1.0 : 0.0; }

constexpr unsigned kAdamAll = 0xffu, kAdamDict = 0xc0u, kAdamColourFeature = (1u << 2) | (1u << 5);
void session_adam_blocks(latmap_session* s, cudaStream_t st, unsigned mask, int64_t begin = 0, int64_t end = -1,
                         const double* ext_flags = nullptr);

latmap_status session_objective(latmap_session* s, bool want_grad, bool map_grads = true, bool use_cache = false) {
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const latmap_config& c = s->cfg;
  const int nf = s->nframes;
  const int gb = s->global_batch > 0 ? s->global_batch : nf;
  const float inv_b = 1.f / (float)gb;  // objective.cpp:77
  const int h = s->intr.height, w = s->intr.width;
  const int64_t npx = (int64_t)h * w;
  const Intr in = to_intr(s->intr);
  MapPtrs map = session_map(s, s->params);
  MapPtrs gmap = session_map(s, s->grads);
  float* proj = s->params + s->off[6];
  float* atoms = s->params + s->off[7];
  float* g_proj = s->grads + s->off[6];
  float* g_atoms = s->grads + s->off[7];
  CTX_CHECK(ctx, cudaMemsetAsync(s->partials, 0, sizeof(double) * ((size_t)s->part_frames * kPart + kTail), st));
  // size the tile-pair buffers the first time a frame is seen
  bool sized = false;
  for (int b = 0; b < nf; ++b) {
    RenderBufs& rb = s->rw[b];
    if (rb.w.pair_cap > 1) continue;
    CTX_CHECK(ctx, rb.ensure(s->n, w, h, 1));
    rb.w.step_overflow = nullptr;
    render_forward(st, map, s->frames[b].rcw, s->frames[b].pose.translation, in, rb.w, nullptr, nullptr, nullptr,
                   nullptr, false, true);
    sized = true;
  }
  if (sized) {
    CTX_CHECK(ctx, cudaStreamSynchronize(st));
    for (int b = 0; b < nf; ++b) {
      RenderBufs& rb = s->rw[b];
      if (rb.w.pair_cap > 1) continue;
      int64_t cnt[4];
      CTX_CHECK(ctx, cudaMemcpy(cnt, rb.w.counters, sizeof(cnt), cudaMemcpyDeviceToHost));
      CTX_CHECK(ctx, rb.ensure(s->n, w, h, std::max<int64_t>(2, (int64_t)(cnt[0] * 1.3) + 1024)));
    }
  }
  CTX_CHECK(ctx, cudaMemsetAsync(s->overflow, 0, sizeof(int64_t), st));
  // the gradient clear and the decoder's per-step operands are queued after the renders fork
  // off (below): the renders need neither
  auto prepare_rest = [&](cudaStream_t ps) -> latmap_status {
    if (want_grad) CTX_CHECK(ctx, cudaMemsetAsync(s->grads, 0, sizeof(float) * s->total, ps));
    decoder_prepare(ps, s->dec, atoms, proj);
    if (s->cfg.decoder_precision == 1 &&
        (ctx->decoder_path == 2 || !decoder_tc_supported(s->k, s->ds, s->dec.nset_cap)))
      decoder_dl_prepare(ps, s->dec);  // M in the staged path's operand blocks
    return LATMAP_OK;
  };
  const bool cached_all = use_cache && s->renders_valid;
  // side-stream renders: off while phases are profiled (per-phase events need one stream)
  const bool ahead = !cached_all && !s->prof && nf > 1;
  if (ahead) {
    if (!s->rstream) CTX_CHECK(ctx, cudaStreamCreateWithFlags(&s->rstream, cudaStreamNonBlocking));
    static const int nrs = [] {
      const char* e = std::getenv("LATMAP_RSTREAMS");
      return e && e[0] == '1' ? 1 : 2;
    }();
    if (nrs == 2 && !s->rstream2) CTX_CHECK(ctx, cudaStreamCreateWithFlags(&s->rstream2, cudaStreamNonBlocking));
    if (!s->rend_start) CTX_CHECK(ctx, cudaEventCreateWithFlags(&s->rend_start, cudaEventDisableTiming));
    while ((int)s->rend_ev.size() < nf) {
      cudaEvent_t e;
      CTX_CHECK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s->rend_ev.push_back(e);
    }
    // after the memsets / previous step's update above; joined back frame by frame below
    CTX_CHECK(ctx, cudaEventRecord(s->rend_start, st));
    CTX_CHECK(ctx, cudaStreamWaitEvent(s->rstream, s->rend_start, 0));
    if (s->rstream2) CTX_CHECK(ctx, cudaStreamWaitEvent(s->rstream2, s->rend_start, 0));
    // two render streams: frame b+1's binning (small, latency-bound launches) overlaps frame b's
    for (int b = 0; b < nf; ++b) {
      FrameDev& f = s->frames[b];
      RenderBufs& rb = s->rw[b];
      cudaStream_t rs = (b & 1) && s->rstream2 ? s->rstream2 : s->rstream;
      rb.w.step_overflow = s->overflow;
      render_forward(rs, map, f.rcw, f.pose.translation, in, rb.w, s->color[b], s->depth[b], s->query[b],
                     s->alpha[b], false, false, false);
      render_blend(rs, map, in, rb.w, s->color[b], s->depth[b], s->query[b], s->alpha[b], ctx->exact_blend);
      CTX_CHECK(ctx, cudaEventRecord(s->rend_ev[b], rs));
    }
  }
  // the backward stream (and the early colour/feature Adam) fork off even for a single keyframe
  // when the decoder is a tcgen05 one: K8 then overlaps the decoder's tail (DEC2 / DL4)
  const bool pipe = !cached_all && !s->prof && want_grad && map_grads && (nf > 1 || s->cfg.decoder_precision == 1);
  // projection backward of every frame in one pass after the frame loop (LATMAP_PB_MULTI=0: per frame)
  static const bool pb_multi_env = [] {
    const char* e = std::getenv("LATMAP_PB_MULTI");
    return !(e && e[0] == '0');
  }();
  const bool pb_multi = pb_multi_env && nf > 1;
  if (pipe) {
    if (!s->rstream) CTX_CHECK(ctx, cudaStreamCreateWithFlags(&s->rstream, cudaStreamNonBlocking));
    if (!s->bstream) CTX_CHECK(ctx, cudaStreamCreateWithFlags(&s->bstream, cudaStreamNonBlocking));
    while ((int)s->evD.size() < nf) {
      cudaEvent_t e1, e2;
      CTX_CHECK(ctx, cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
      CTX_CHECK(ctx, cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      s->evD.push_back(e1);
      s->evB.push_back(e2);
    }
    static const bool lstream_env = [] {
      const char* e = std::getenv("LATMAP_LSTREAM");
      return !(e && e[0] == '0');
    }();
    if (lstream_env && !s->lstream) CTX_CHECK(ctx, cudaStreamCreateWithFlags(&s->lstream, cudaStreamNonBlocking));
    while (s->lstream && (int)s->rend_ev.size() < nf) {
      cudaEvent_t e;
      CTX_CHECK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s->rend_ev.push_back(e);
    }
    while (s->lstream && (int)s->evL.size() < nf) {
      cudaEvent_t e;
      CTX_CHECK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s->evL.push_back(e);
    }
    if (!s->d_color2) {
      CTX_CHECK(ctx, cudaMalloc(&s->d_color2, sizeof(float) * npx * 3));
      CTX_CHECK(ctx, cudaMalloc(&s->d_depth2, sizeof(float) * npx));
      CTX_CHECK(ctx, cudaMalloc(&s->d_query2, sizeof(float) * npx * s->ds));
    }
  }
  // single keyframe: the render runs on this stream next, so the preparation goes to the (idle)
  // backward stream and is joined after the render
  bool prep_forked = false;
  if (pipe && !ahead) {
    if (!s->ev_pf) CTX_CHECK(ctx, cudaEventCreateWithFlags(&s->ev_pf, cudaEventDisableTiming));
    if (!s->ev_pj) CTX_CHECK(ctx, cudaEventCreateWithFlags(&s->ev_pj, cudaEventDisableTiming));
    CTX_CHECK(ctx, cudaEventRecord(s->ev_pf, st));
    CTX_CHECK(ctx, cudaStreamWaitEvent(s->bstream, s->ev_pf, 0));
    const latmap_status ps = prepare_rest(s->bstream);
    if (ps != LATMAP_OK) return ps;
    CTX_CHECK(ctx, cudaEventRecord(s->ev_pj, s->bstream));
    prep_forked = true;
  } else {
    const latmap_status ps = prepare_rest(st);
    if (ps != LATMAP_OK) return ps;
  }
  for (int b = 0; b < nf; ++b) {
    FrameDev& f = s->frames[b];
    RenderBufs& rb = s->rw[b];
    rb.w.step_overflow = s->overflow;
    double* part = s->partials + (size_t)(s->slot_offset + b) * kPart;
    const bool cached = use_cache && s->renders_valid;
    const bool slot1 = pipe && (b & 1);
    float* d_col = slot1 ? s->d_color2 : s->d_color;
    float* d_dep = slot1 ? s->d_depth2 : s->d_depth;
    float* d_qry = slot1 ? s->d_query2 : s->d_query;
    if (pipe && b >= 2) CTX_CHECK(ctx, cudaStreamWaitEvent(st, s->evB[b - 2], 0));  // slot free again
    if (ahead) {
      CTX_CHECK(ctx, cudaStreamWaitEvent(st, s->rend_ev[b], 0));
    } else if (!cached) {
      s->begin(0);
      render_forward(st, map, f.rcw, f.pose.translation, in, rb.w, s->color[b], s->depth[b], s->query[b],
                     s->alpha[b], false, false, false);
      s->end();
      s->begin(1);
      render_blend(st, map, in, rb.w, s->color[b], s->depth[b], s->query[b], s->alpha[b], ctx->exact_blend);
      s->end();
      // the loss stream's render dependency when the render ran on this stream (single keyframe)
      if (pipe && s->lstream) CTX_CHECK(ctx, cudaEventRecord(s->rend_ev[b], st));
    }
    if (prep_forked && b == 0) CTX_CHECK(ctx, cudaStreamWaitEvent(st, s->ev_pj, 0));  // gradients cleared, operands ready
    const bool map_grad = want_grad && map_grads;
    const bool lsplit = pipe && s->lstream && (ahead || !cached);
    bool evd_early = false;  // evD[b] recorded inside the decoder, right after DEC1
    cudaStream_t ls = lsplit ? s->lstream : st;
    if (lsplit) {
      if (b >= 2) CTX_CHECK(ctx, cudaStreamWaitEvent(ls, s->evB[b - 2], 0));  // gradient-image slot free
      CTX_CHECK(ctx, cudaStreamWaitEvent(ls, s->rend_ev[b], 0));
      wait_frame(s, b, st);  // the decoder's frame data
    }
    s->begin(2);
    wait_frame(s, b, ls);
    image_losses(ls, s->color[b], s->depth[b], s->alpha[b], f.rgb, f.depth, h, w, c.lambda_i1, c.lambda_i2,
                 c.lambda_rgb * inv_b, c.lambda_depth * inv_b, map_grad, d_col, d_dep, part,
                 s->ssim_scratch);
    s->end();
    if (lsplit) CTX_CHECK(ctx, cudaEventRecord(s->evL[b], ls));
    if (c.segment_mode)
      set_double_kernel<<<1, 1, 0, st>>>(part + 7, (double)f.n_sup);
    else
      copy_count_kernel<<<1, 1, 0, st>>>(part + 7, f.stat);  // supervised pixels, counted on the device
    count_launch();
    const bool have_sup = c.segment_mode ? f.n_sup > 0 : f.n_set > 0;
    if (have_sup && c.segment_mode) {
      // pooled rows: Q_r = mean of the rendered queries over segment r; the decoder runs on the
      // n_sup rows (targets = features[seg_rows[r]]), then d_query[p] = dQ_r / |segment r|
      s->begin(3);
      const unsigned gq = (unsigned)std::min<int64_t>((npx * s->ds + 255) / 256, 148 * 16);
      CTX_CHECK(ctx, cudaMemsetAsync(s->seg_q, 0, sizeof(float) * f.n_sup * s->ds, st));
      if (deterministic())
        seg_pool_det_kernel<<<dim3((unsigned)f.n_sup, (unsigned)s->ds), 256, 0, st>>>(s->query[b], f.assign, npx, s->ds,
                                                                                   f.seg_of, s->seg_q);
      else
        seg_pool_kernel<<<gq, 256, 0, st>>>(s->query[b], f.assign, npx, s->ds, f.seg_of, s->seg_q);
      seg_mean_kernel<<<(unsigned)((f.n_sup * s->ds + 255) / 256), 256, 0, st>>>(s->seg_q, f.seg_inv, f.n_sup, s->ds);
      count_launch(2);
      s->dec.last_path = 1;
      s->dec.last_npx = f.n_sup;
      decoder_frame(st, s->dec, s->seg_q, f.seg_rows, f.n_sup, f.feats, f.n_set, f.stat, atoms, proj,
                    c.softmax_temp, c.lambda_cos, c.lambda_l2, c.lambda_feat * inv_b, want_grad, s->seg_dq, g_proj,
                    g_atoms, part);
      if (want_grad) {
        seg_scatter_kernel<<<gq, 256, 0, st>>>(s->seg_dq, f.assign, npx, s->ds, f.seg_of, f.seg_inv, d_qry);
        count_launch();
      }
      s->end();
    } else if (have_sup) {
      s->begin(3);
      const bool fused_ok = decoder_tc_supported(s->k, s->ds, f.n_set) && ctx->decoder_path != 2;
      const bool staged_ok = s->dec.dl_mt && decoder_dl_supported(s->k, s->ds, f.n_set) && ctx->decoder_path != 1;
      s->dec.last_path = (c.decoder_precision == 1 && fused_ok) ? 2 : (c.decoder_precision == 1 && staged_ok) ? 3 : 1;
      s->dec.last_npx = npx;
      if (c.decoder_precision == 1 && fused_ok) {
        // K8 of this frame may start once DEC1 has written d_query: DEC2 and the Bm embed overlap it
        if (pipe && map_grads) s->dec.ev_dq = s->evD[b], evd_early = true;
        decoder_frame_tc(st, s->dec, s->query[b], f.assign, npx, f.feats, f.n_set, f.stat, atoms, proj,
                         c.softmax_temp, c.lambda_cos, c.lambda_l2, c.lambda_feat * inv_b, want_grad, d_qry,
                         g_proj, g_atoms, part);
        s->dec.ev_dq = nullptr;
      }
      else if (c.decoder_precision == 1 && staged_ok) {
        if (pipe && map_grads) s->dec.ev_dq = s->evD[b], evd_early = true;  // recorded after DL3 (d_query)
        decoder_frame_dl(st, s->dec, s->query[b], f.assign, npx, f.feats, f.n_set, f.stat, atoms, c.softmax_temp,
                         c.lambda_cos, c.lambda_l2, c.lambda_feat * inv_b, want_grad, d_qry, g_atoms, part);
        s->dec.ev_dq = nullptr;
      }
      else
        decoder_frame(st, s->dec, s->query[b], f.assign, npx, f.feats, f.n_set, f.stat, atoms, proj, c.softmax_temp,
                      c.lambda_cos, c.lambda_l2, c.lambda_feat * inv_b, want_grad, d_qry, g_proj, g_atoms, part);
      s->end();
    }
    if (map_grad) {
      // geo_acc is zero here: zeroed at allocation, and project_bwd re-zeroes every entry it reads
      cudaStream_t bs = st;
      if (pipe) {
        if (!evd_early) CTX_CHECK(ctx, cudaEventRecord(s->evD[b], st));
        CTX_CHECK(ctx, cudaStreamWaitEvent(s->bstream, s->evD[b], 0));
        if (lsplit) CTX_CHECK(ctx, cudaStreamWaitEvent(s->bstream, s->evL[b], 0));
        bs = s->bstream;
      }
      s->begin(4);
      render_backward(bs, map, f.rcw, f.rwc, f.pose.translation, in, rb.w, d_col, d_dep, have_sup ? d_qry : nullptr,
                      rb.geo_acc, gmap, false, deterministic() ? &ctx->det : nullptr);
      s->end();
      if (!pb_multi) {
        s->begin(5);
        render_project_backward(bs, map, f.rcw, f.rwc, f.pose.translation, in, rb.w, rb.geo_acc, gmap);
        s->end();
      }
      if (pipe) CTX_CHECK(ctx, cudaEventRecord(s->evB[b], s->bstream));
    }
  }
  // the dictionary's step-end terms need only the decoder (this stream): queued before the join,
  // they overlap the last frames' render backward
  if (want_grad) decoder_finish_tc(st, s->dec, atoms, proj, g_proj, g_atoms);
  // trust term enters once (objective.cpp:247-256)
  if (s->add_trust) {
    double* tslot = s->partials + (size_t)s->part_frames * kPart;
    trust_region(st, atoms, s->anchor, s->k, s->df, c.trust_delta, want_grad ? g_atoms : nullptr,
                 c.lambda_feat * c.lambda_trust, tslot);
  }
  if (pipe) CTX_CHECK(ctx, cudaStreamWaitEvent(st, s->evB[nf - 1], 0));  // join: every backward done
  s->cf_done = false;
  if (pipe && s->early_cf) {
    if (!s->ev_cf) CTX_CHECK(ctx, cudaEventCreateWithFlags(&s->ev_cf, cudaEventDisableTiming));
    CTX_CHECK(ctx, cudaStreamWaitEvent(s->rstream, s->evB[nf - 1], 0));
    // every frame's tile-list overflow flag is final (all renders are done): Adam skips on it
    overflow_slot_kernel<<<1, 1, 0, s->rstream>>>(s->overflow,
                                                  s->partials + (size_t)s->part_frames * kPart + kTailOverflow);
    count_launch();
    session_adam_blocks(s, s->rstream, kAdamColourFeature);
    CTX_CHECK(ctx, cudaEventRecord(s->ev_cf, s->rstream));
    s->cf_done = true;
  }
  if (want_grad && map_grads && pb_multi) {
    // K9 over all frames in one pass: parameters and gradients read once, frame order kept
    std::vector<const float*> rcw(nf), rwc(nf), org(nf);
    std::vector<const RenderWork*> ws(nf);
    std::vector<float*> geo(nf);
    for (int b = 0; b < nf; ++b) {
      rcw[b] = s->frames[b].rcw;
      rwc[b] = s->frames[b].rwc;
      org[b] = s->frames[b].pose.translation;
      ws[b] = &s->rw[b].w;
      geo[b] = s->rw[b].geo_acc;
    }
    s->begin(5);
    render_project_backward_multi(st, map, nf, rcw.data(), rwc.data(), org.data(), in, ws.data(), geo.data(), gmap);
    s->end();
  }
  s->renders_valid = true;
  // this rank's tile-list overflow flag joins the loss partials, so the sharded step's sum
  // all-reduce tells every rank (and its Adam) that some rank's gradients are incomplete
  overflow_slot_kernel<<<1, 1, 0, st>>>(s->overflow, s->partials + (size_t)s->part_frames * kPart + kTailOverflow);
  count_launch();
  return post_launch(ctx);
}

latmap_status session_assemble(latmap_session* s, latmap_loss_breakdown* out) {
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const int gb = s->global_batch > 0 ? s->global_batch : s->nframes;
  const latmap_config& c = s->cfg;
  LossWeights wt{c.lambda_rgb, c.lambda_i1, c.lambda_i2, c.lambda_depth, c.lambda_feat, c.lambda_cos, c.lambda_l2,
                 c.lambda_trust};
  // trust slot lives after all frame slots
  double* base = s->partials;
  // assemble expects the trust value right after `gb` frames: copy it there when part_frames > gb
  if (s->part_frames != gb)
    CTX_CHECK(ctx, cudaMemcpyAsync(base + (size_t)gb * kPart, base + (size_t)s->part_frames * kPart, sizeof(double),
                                   cudaMemcpyDeviceToDevice, st));
  assemble_loss_kernel<<<1, 1, 0, st>>>(base, gb, (double)s->intr.width * s->intr.height, 1.f / (float)gb, wt,
                                        s->d_loss);
  count_launch();
  if (out) {
    CTX_CHECK(ctx, cudaMemcpyAsync(out, s->d_loss, sizeof(*out), cudaMemcpyDeviceToHost, st));
    std::vector<int64_t> stat((size_t)2 * s->nframes, 0);
    for (int b = 0; b < s->nframes; ++b)
      if (s->frames[b].stat)
        CTX_CHECK(ctx, cudaMemcpyAsync(stat.data() + 2 * b, s->frames[b].stat, 2 * sizeof(int64_t),
                                       cudaMemcpyDeviceToHost, st));
    CTX_CHECK(ctx, cudaStreamSynchronize(st));
    for (int b = 0; b < s->nframes; ++b)
      if (stat[2 * b + 1] > 0) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "gather_supervision: assignment out of range");
  }
  return post_launch(ctx);
}

// MapOptimizer::step_map + step_dict (pipeline.cpp:75-95); dict_only = step_dict alone (Stage II).
void session_adam(latmap_session* s, bool dict_only = false, int64_t begin = 0, int64_t end = -1,
                  const double* ext_flags = nullptr) {
  s->begin(6);
  unsigned mask = dict_only ? kAdamDict : kAdamAll;
  if (s->cf_done && !dict_only && begin == 0 && end < 0 && !ext_flags) {  // colour + feature done early
    cudaStreamWaitEvent(s->ctx->stream, s->ev_cf, 0);
    mask &= ~kAdamColourFeature;
  }
  s->cf_done = false;
  session_adam_blocks(s, s->ctx->stream, mask, begin, end, ext_flags);
  if (!dict_only) s->renders_valid = false;  // the map moves
  s->end();
}

// MapOptimizer blocks selected by `mask` (bit i = block i of the flat buffers).
void session_adam_blocks(latmap_session* s, cudaStream_t st, unsigned mask, int64_t begin, int64_t end,
                         const double* ext_flags) {
  const latmap_config& c = s->cfg;
  AdamBlock blocks[8] = {
      {s->off[0], s->len[0], c.lr_position * c.scene_extent, 0},  // pipeline.cpp:76
      {s->off[1], s->len[1], c.lr_rotation, 1},
      {s->off[2], s->len[2], c.lr_color, 0},
      {s->off[3], s->len[3], c.lr_log_scale, 0},
      {s->off[4], s->len[4], c.lr_opacity, 0},
      {s->off[5], s->len[5], c.lr_feature, 0},
      {s->off[6], s->len[6], c.lr_proj, 0},                       // pipeline.cpp:93
      {s->off[7], s->len[7], c.lr_dict, c.dict_learn ? 0 : -1},  // pipeline.cpp:94
  };
  for (int i = 0; i < 8; ++i)
    if (!(mask >> i & 1u)) blocks[i].kind = -1;
  // the sticky overflow-step counter is advanced once per step: by the call holding block 0
  adam_flat(st, s->params, s->grads, s->m, s->v, blocks, 8, s->steps, s->skipped, s->corr1, s->corr2, kCorrLen,
            s->flags, s->partials + (size_t)s->part_frames * kPart + kTailOverflow,
            (mask & 1u) || mask == kAdamDict ? s->overflow_steps : nullptr, begin, end, ext_flags);
}

// Grow the tile-pair buffers after an overflow; returns true when something was resized.
bool session_fix_overflow(latmap_session* s) {
  int64_t of = 0;
  cudaMemcpy(&of, s->overflow, sizeof(of), cudaMemcpyDeviceToHost);
  if (!of) return false;
  s->drop_graph();  // buffers move
  for (int b = 0; b < s->nframes; ++b) {
    int64_t cnt[4];
    cudaMemcpy(cnt, s->rw[b].w.counters, sizeof(cnt), cudaMemcpyDeviceToHost);
    if (cnt[0] > s->rw[b].w.pair_cap) s->rw[b].ensure(s->n, s->intr.width, s->intr.height, (int64_t)(cnt[0] * 1.3) + 1024);
  }
  return true;
}

}  // namespace

extern "C" {

latmap_status latmap_session_create(latmap_ctx* ctx, const latmap_config* cfg, int64_t n, int32_t ds, int64_t k,
                                    int32_t df, const latmap_intrinsics* intr, latmap_session** out) {
  if (!ctx || !cfg || !intr || !out || n < 0 || ds < 1 || k < 1 || df < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  if (!intr_valid(*intr)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "render: invalid intrinsics");
  if (ds > 64) return fail(ctx, LATMAP_ERR_UNSUPPORTED, "query_dim must be <= 64");
  if (!(cfg->softmax_temp > 0.f)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "reconstruct: temperature must be > 0");
  auto* s = new latmap_session();
  s->ctx = ctx;
  s->cfg = *cfg;
  s->n = n;
  s->ds = ds;
  s->k = k;
  s->df = df;
  s->intr = *intr;
  const int64_t sizes[8] = {3 * n, 4 * n, 3 * n, 3 * n, n, (int64_t)ds * n, (int64_t)ds * df, k * df};
  s->off[0] = 0;
  for (int i = 0; i < 8; ++i) s->off[i + 1] = pad4(s->off[i] + sizes[i]);  // 16-byte aligned blocks
  for (int i = 0; i < 8; ++i) s->len[i] = sizes[i];
  s->total = s->off[8];
  const size_t npx = (size_t)intr->width * intr->height;
  auto ok = [&](cudaError_t e) { return e == cudaSuccess; };
  const int64_t flat_cap = s->total + kShardSlack;
  bool good = ok(cudaMalloc(&s->params, sizeof(float) * flat_cap)) && ok(cudaMalloc(&s->grads, sizeof(float) * flat_cap)) &&
              ok(cudaMalloc(&s->m, sizeof(float) * flat_cap)) && ok(cudaMalloc(&s->v, sizeof(float) * flat_cap)) &&
              ok(cudaMalloc(&s->anchor, sizeof(float) * k * df)) && ok(cudaMalloc(&s->steps, sizeof(int64_t) * 8)) &&
              ok(cudaMalloc(&s->skipped, sizeof(int64_t) * 8)) && ok(cudaMalloc(&s->overflow, sizeof(int64_t))) && ok(cudaMalloc(&s->overflow_steps, sizeof(int64_t))) &&
              ok(cudaMalloc(&s->flags, sizeof(int32_t) * 8)) && ok(cudaMalloc(&s->corr1, sizeof(float) * kCorrLen)) &&
              ok(cudaMalloc(&s->corr2, sizeof(float) * kCorrLen)) &&
              ok(cudaMalloc(&s->d_color, sizeof(float) * npx * 3)) && ok(cudaMalloc(&s->d_depth, sizeof(float) * npx)) &&
              ok(cudaMalloc(&s->d_query, sizeof(float) * npx * ds)) &&
              ok(cudaMalloc(&s->ssim_scratch, sizeof(float) * ssim_scratch_floats(intr->height, intr->width, 3))) &&
              ok(cudaMalloc(&s->d_loss, sizeof(latmap_loss_breakdown)));
  DecoderWork& d = s->dec;
  d.n_cap = (int64_t)npx;
  d.k = k;
  d.ds = ds;
  d.df = df;
  const size_t npx_t = (npx + 127) / 128 * 128;  // whole 128-row tiles (the staged path aliases buf1/buf2)
  good = good && ok(cudaMalloc(&d.buf1, sizeof(float) * npx_t * k)) && ok(cudaMalloc(&d.buf2, sizeof(float) * npx_t * k)) &&
         ok(cudaMalloc(&d.alpha_r, sizeof(float) * npx)) && ok(cudaMalloc(&d.beta_r, sizeof(float) * npx)) &&
         ok(cudaMalloc(&d.kd, sizeof(float) * k * ds)) && ok(cudaMalloc(&d.mm, sizeof(float) * k * k)) &&
         ok(cudaMalloc(&d.r, sizeof(float) * ds * k)) && ok(cudaMalloc(&d.a, sizeof(float) * k * k));
  if (good && cfg->decoder_precision == 1) {
    good = ok(cudaMalloc(&d.row_stats, sizeof(float) * 4 * npx)) &&
           ok(cudaMalloc(&d.r_part, sizeof(float) * 2 * 148 * k * ds)) &&
           ok(cudaMalloc(&d.a_part, sizeof(float) * 8 * 148 * k * k + 1024)) &&  // 8 per-frame slots (decoder_tc.cu)
           ok(cudaMalloc(&d.bm_part, sizeof(float) * 148 * k * 64)) &&
           ok(cudaMalloc(&d.loss_part, sizeof(double) * 148 * 4)) &&
           ok(cudaMalloc(&d.e_tiles, (size_t)((npx + 127) / 128) * 128 * k * 2)) &&
           (!decoder_tc_supported(k, ds, 1) || ok(cudaMalloc(&d.tc_img, (size_t)(k * ds + k * k) * 2))) &&
           ok(cudaMalloc(&d.a_acc, sizeof(float) * k * k)) && ok(cudaMalloc(&d.r_acc, sizeof(float) * ds * k));
    if (good && decoder_dl_supported(k, ds, 1)) {
      d.dl_t = d.buf1;
      d.dl_ae = reinterpret_cast<uint8_t*>(d.buf2);  // 128 x (K + NB) bf16 per tile <= 128 x K fp32
      good = ok(cudaMalloc(&d.dl_mt, sizeof(uint16_t) * k * k)) &&
             ok(cudaMalloc(&d.dl_nu, sizeof(float) * (k / 256) * npx_t)) &&
             ok(cudaMalloc(&d.dl_part, sizeof(float) * decoder_dl_part_floats(k)));
    }
  }
  if (!good) {
    t_err = "latmap_session_create: out of device memory";
    ctx->err = t_err;
    delete s;  // leaks partial allocations on failure; acceptable for an OOM path
    return LATMAP_ERR_OUT_OF_MEMORY;
  }
  s->dict_w.assign((size_t)k, 0.f);
  s->cur_cap = flat_cap;
  cudaMemset(s->m, 0, sizeof(float) * flat_cap);
  cudaMemset(s->v, 0, sizeof(float) * flat_cap);
  cudaMemset(s->grads, 0, sizeof(float) * flat_cap);
  cudaMemset(s->overflow_steps, 0, sizeof(int64_t));
  cudaMemset(s->steps, 0, sizeof(int64_t) * 8);
  cudaMemset(s->skipped, 0, sizeof(int64_t) * 8);
  cudaMemset(s->flags, 0, sizeof(int32_t) * 8);
  std::vector<float> c1, c2;
  corr_tables(c1, c2, kCorrLen);
  cudaMemcpy(s->corr1, c1.data(), sizeof(float) * kCorrLen, cudaMemcpyHostToDevice);
  cudaMemcpy(s->corr2, c2.data(), sizeof(float) * kCorrLen, cudaMemcpyHostToDevice);
  *out = s;
  return LATMAP_OK;
}

latmap_status latmap_session_destroy(latmap_session* s) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  cudaStreamSynchronize(s->ctx->stream);
  s->drop_graph();
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->rstream) cudaStreamSynchronize(s->rstream), cudaStreamDestroy(s->rstream);
  if (s->rstream2) cudaStreamSynchronize(s->rstream2), cudaStreamDestroy(s->rstream2);
  if (s->rend_start) cudaEventDestroy(s->rend_start);
  if (s->ev_cf) cudaEventDestroy(s->ev_cf);
  if (s->ev_pf) cudaEventDestroy(s->ev_pf);
  if (s->ev_pj) cudaEventDestroy(s->ev_pj);
  for (cudaEvent_t e : s->evL) cudaEventDestroy(e);
  if (s->lstream) cudaStreamSynchronize(s->lstream), cudaStreamDestroy(s->lstream);
  for (cudaEvent_t e : s->rend_ev) cudaEventDestroy(e);
  if (s->bstream) cudaStreamSynchronize(s->bstream), cudaStreamDestroy(s->bstream);
  for (cudaEvent_t e : s->evD) cudaEventDestroy(e);
  for (cudaEvent_t e : s->evB) cudaEventDestroy(e);
  for (float* p : {s->d_color2, s->d_depth2, s->d_query2})
    if (p) cudaFree(p);
  if (s->ctx->copy_stream) cudaStreamSynchronize(s->ctx->copy_stream);
  for (cudaEvent_t e : s->up_ev) cudaEventDestroy(e);
  if (s->ev_ready) cudaEventDestroy(s->ev_ready);
  for (void* p : {(void*)s->sp_params, (void*)s->sp_grads, (void*)s->sp_m, (void*)s->sp_v})
    if (p) cudaFree(p);
  for (void* p : {(void*)s->params, (void*)s->grads, (void*)s->m, (void*)s->v, (void*)s->anchor, (void*)s->steps,
                  (void*)s->skipped, (void*)s->overflow, (void*)s->overflow_steps, (void*)s->flags, (void*)s->corr1, (void*)s->corr2,
                  (void*)s->d_color, (void*)s->d_depth, (void*)s->d_query, (void*)s->ssim_scratch, (void*)s->partials,
                  (void*)s->d_loss, (void*)s->dec.buf1, (void*)s->dec.buf2, (void*)s->dec.alpha_r, (void*)s->dec.beta_r,
                  (void*)s->dec.kd, (void*)s->dec.mm, (void*)s->dec.gt, (void*)s->dec.nv, (void*)s->dec.r,
                  (void*)s->dec.a, (void*)s->dec.bm, (void*)s->dec.row_stats, (void*)s->dec.r_part,
                  (void*)s->dec.a_part, (void*)s->dec.bm_part, (void*)s->dec.loss_part,
                  (void*)s->dec.e_tiles, (void*)s->dec.tc_img, (void*)s->dec.a_acc, (void*)s->dec.r_acc, (void*)s->dec.dl_mt,
                  (void*)s->dec.dl_nu, (void*)s->dec.dl_part, (void*)s->dec.row_nd, (void*)s->snap.params,
                  (void*)s->snap.m, (void*)s->snap.v, (void*)s->snap.anchor})
    if (p) cudaFree(p);
  for (auto& r : s->rw) r.release();
  for (auto* p : s->color) cudaFree(p);
  for (auto* p : s->depth) cudaFree(p);
  for (auto* p : s->query) cudaFree(p);
  for (auto* p : s->alpha) cudaFree(p);
  if (s->seg_q) cudaFree(s->seg_q), cudaFree(s->seg_dq);
  for (auto& f : s->frames) {
    if (f.seg_rows) cudaFree(f.seg_rows), cudaFree(f.seg_of), cudaFree(f.seg_inv);
    if (f.rgb) cudaFree(f.rgb);
    if (f.depth) cudaFree(f.depth);
    if (f.assign) cudaFree(f.assign);
    if (f.feats) cudaFree(f.feats);
    if (f.stat) cudaFree(f.stat);
  }
  delete s;
  return LATMAP_OK;
}

latmap_status latmap_session_set_map(latmap_session* s, const float* pos, const float* rot, const float* col,
                                     const float* lsc, const float* opa, const float* feat) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  s->renders_valid = false;
  const float* src[6] = {pos, rot, col, lsc, opa, feat};
  for (int i = 0; i < 6; ++i)
    if (s->len[i] > 0)
      CTX_CHECK(ctx, cudaMemcpyAsync(s->params + s->off[i], src[i], sizeof(float) * s->len[i],
                                     cudaMemcpyHostToDevice, ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_session_get_map(latmap_session* s, float* pos, float* rot, float* col, float* lsc, float* opa,
                                     float* feat) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  float* dst[6] = {pos, rot, col, lsc, opa, feat};
  for (int i = 0; i < 6; ++i)
    if (dst[i] && s->len[i] > 0)
      CTX_CHECK(ctx, cudaMemcpyAsync(dst[i], s->params + s->off[i], sizeof(float) * s->len[i],
                                     cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_session_set_dictionary(latmap_session* s, const float* atoms, const float* anchor,
                                            const float* proj) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  const size_t kd = (size_t)s->k * s->df, pd = (size_t)s->ds * s->df;
  if (atoms) CTX_CHECK(ctx, cudaMemcpyAsync(s->params + s->off[7], atoms, sizeof(float) * kd, cudaMemcpyHostToDevice, ctx->stream));
  if (anchor) CTX_CHECK(ctx, cudaMemcpyAsync(s->anchor, anchor, sizeof(float) * kd, cudaMemcpyHostToDevice, ctx->stream));
  if (proj) CTX_CHECK(ctx, cudaMemcpyAsync(s->params + s->off[6], proj, sizeof(float) * pd, cudaMemcpyHostToDevice, ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_session_get_dictionary(latmap_session* s, float* atoms, float* proj) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  if (atoms) CTX_CHECK(ctx, cudaMemcpyAsync(atoms, s->params + s->off[7], sizeof(float) * s->k * s->df, cudaMemcpyDeviceToHost, ctx->stream));
  if (proj) CTX_CHECK(ctx, cudaMemcpyAsync(proj, s->params + s->off[6], sizeof(float) * s->ds * s->df, cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_session_get_anchor(latmap_session* s, float* anchor) {
  if (!s || !anchor) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  CTX_CHECK(ctx, cudaMemcpyAsync(anchor, s->anchor, sizeof(float) * s->k * s->df, cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_session_set_frames(latmap_session* s, int32_t nf, const latmap_frame* frames) {
  if (!s || nf < 1 || !frames) return fail(s ? s->ctx : nullptr, LATMAP_ERR_INVALID_ARGUMENT, "total_objective: empty batch");
  latmap_ctx* ctx = s->ctx;
  // the captured step graph bakes in frame poses (camera constants are kernel arguments),
  // buffer pointers and per-frame sizes: any change drops it
  bool same = s->nframes == nf && (int)s->frames.size() >= nf;
  std::vector<std::array<void*, 4>> ptrs0;
  for (int b = 0; same && b < nf; ++b) {
    const FrameDev& f = s->frames[b];
    same = std::memcmp(&f.pose, &frames[b].pose, sizeof(latmap_pose)) == 0 && f.n_set == frames[b].n_set;
    ptrs0.push_back({(void*)f.rgb, (void*)f.depth, (void*)f.assign, (void*)f.feats});
  }
  latmap_status st = session_alloc_frames(s, nf);
  if (st != LATMAP_OK) return st;
  const size_t npx = (size_t)s->intr.width * s->intr.height;
  std::vector<int64_t> nsup0;
  for (int b = 0; same && b < nf; ++b) nsup0.push_back(s->frames[b].n_sup);
  if (!ctx->copy_stream) CTX_CHECK(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  if (!s->ev_ready) CTX_CHECK(ctx, cudaEventCreateWithFlags(&s->ev_ready, cudaEventDisableTiming));
  while ((int)s->up_ev.size() < nf) {
    cudaEvent_t e;
    CTX_CHECK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->up_ev.push_back(e);
  }
  // uploads start after the work already queued on the context stream (it may still read them)
  CTX_CHECK(ctx, cudaEventRecord(s->ev_ready, ctx->stream));
  CTX_CHECK(ctx, cudaStreamWaitEvent(ctx->copy_stream, s->ev_ready, 0));
  for (int b = 0; b < nf; ++b) {
    const latmap_frame& in = frames[b];
    FrameDev& f = s->frames[b];
    if (!pose_mats(in.pose, f.rcw, f.rwc)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "quat_to_rot: zero-norm quaternion");
    f.pose = in.pose;
    if (npx > f.c_px) {
      if (f.rgb) cudaFree(f.rgb), cudaFree(f.depth), cudaFree(f.assign);
      CTX_CHECK(ctx, cudaMalloc(&f.rgb, sizeof(float) * npx * 3));
      CTX_CHECK(ctx, cudaMalloc(&f.depth, sizeof(float) * npx));
      CTX_CHECK(ctx, cudaMalloc(&f.assign, sizeof(int32_t) * npx));
      f.c_px = npx;
    }
    const size_t nfeat = (size_t)in.n_set * s->df;
    if (nfeat > f.c_feat || !f.feats) {
      if (f.feats) cudaFree(f.feats);
      CTX_CHECK(ctx, cudaMalloc(&f.feats, sizeof(float) * std::max<size_t>(nfeat, 1)));
      f.c_feat = nfeat;
    }
    cudaStream_t cs = ctx->copy_stream;
    CTX_CHECK(ctx, cudaMemcpyAsync(f.rgb, in.rgb, sizeof(float) * npx * 3, cudaMemcpyHostToDevice, cs));
    CTX_CHECK(ctx, cudaMemcpyAsync(f.depth, in.depth, sizeof(float) * npx, cudaMemcpyHostToDevice, cs));
    CTX_CHECK(ctx, cudaMemcpyAsync(f.assign, in.assignment, sizeof(int32_t) * npx, cudaMemcpyHostToDevice, cs));
    if (nfeat) CTX_CHECK(ctx, cudaMemcpyAsync(f.feats, in.features, sizeof(float) * nfeat, cudaMemcpyHostToDevice, cs));
    if (!f.stat) CTX_CHECK(ctx, cudaMalloc(&f.stat, 2 * sizeof(int64_t)));
    int64_t nsup = 0;
    if (!s->cfg.segment_mode) {
      // supervised-pixel count and range check on the device, behind the upload (reported by the
      // objective call that reads the loss, as gather_supervision throws inside total_objective)
      CTX_CHECK(ctx, cudaMemsetAsync(f.stat, 0, 2 * sizeof(int64_t), cs));
      assign_scan_kernel<<<(unsigned)std::min<size_t>((npx + 1023) / 1024, 148 * 4), 256, 0, cs>>>(f.assign, (int64_t)npx,
                                                                                                 in.n_set, f.stat);
      count_launch();
    }
    CTX_CHECK(ctx, cudaEventRecord(s->up_ev[b], cs));
    if (s->cfg.segment_mode) {
      int32_t amax = -1;
      for (size_t p = 0; p < npx; ++p) amax = std::max(amax, in.assignment[p]);
      if (amax >= in.n_set) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "gather_supervision: assignment out of range");
      // present assignment rows in ascending order (objective.cpp:39-64)
      std::vector<int64_t> cnt((size_t)std::max<int64_t>(in.n_set, 1), 0);
      for (size_t p = 0; p < npx; ++p)
        if (in.assignment[p] >= 0) ++cnt[(size_t)in.assignment[p]];
      std::vector<int32_t> rows, of((size_t)std::max<int64_t>(in.n_set, 1), -1);
      std::vector<float> inv;
      for (int64_t a = 0; a < in.n_set; ++a)
        if (cnt[(size_t)a] > 0) {
          of[(size_t)a] = (int32_t)rows.size();
          rows.push_back((int32_t)a);
          inv.push_back(1.f / (float)cnt[(size_t)a]);
        }
      const size_t need = (size_t)std::max<int64_t>(in.n_set, 1);
      if (need > f.c_seg) {
        if (f.seg_rows) cudaFree(f.seg_rows), cudaFree(f.seg_of), cudaFree(f.seg_inv);
        CTX_CHECK(ctx, cudaMalloc(&f.seg_rows, sizeof(int32_t) * need));
        CTX_CHECK(ctx, cudaMalloc(&f.seg_of, sizeof(int32_t) * need));
        CTX_CHECK(ctx, cudaMalloc(&f.seg_inv, sizeof(float) * need));
        f.c_seg = need;
      }
      if (!rows.empty()) {
        CTX_CHECK(ctx, cudaMemcpy(f.seg_rows, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice));
        CTX_CHECK(ctx, cudaMemcpy(f.seg_inv, inv.data(), sizeof(float) * inv.size(), cudaMemcpyHostToDevice));
      }
      CTX_CHECK(ctx, cudaMemcpy(f.seg_of, of.data(), sizeof(int32_t) * need, cudaMemcpyHostToDevice));
      nsup = (int64_t)rows.size();
      if ((int64_t)need > s->seg_cap) {
        if (s->seg_q) cudaFree(s->seg_q), cudaFree(s->seg_dq);
        CTX_CHECK(ctx, cudaMalloc(&s->seg_q, sizeof(float) * need * s->ds));
        CTX_CHECK(ctx, cudaMalloc(&s->seg_dq, sizeof(float) * need * s->ds));
        s->seg_cap = (int64_t)need;
      }
    }
    if (s->cfg.segment_mode) {
      const int64_t h[2] = {nsup, 0};  // supervision rows = present segments
      CTX_CHECK(ctx, cudaMemcpy(f.stat, h, sizeof(h), cudaMemcpyHostToDevice));
    }
    f.n_sup = nsup;
    f.n_set = in.n_set;
  }
  s->nframes = nf;
  s->renders_valid = false;  // poses may differ
  for (int b = 0; same && b < nf; ++b) {
    const FrameDev& f = s->frames[b];
    same = ptrs0[b] == std::array<void*, 4>{(void*)f.rgb, (void*)f.depth, (void*)f.assign, (void*)f.feats} &&
           nsup0[b] == f.n_sup;
  }
  if (!same) s->drop_graph();
  // per-frame decoder buffers sized by the largest embedding table
  int64_t max_set = 1;
  for (int b = 0; b < nf; ++b) max_set = std::max(max_set, s->frames[b].n_set);
  if (max_set > s->dec.nset_cap) {
    if (s->dec.gt) cudaFree(s->dec.gt), cudaFree(s->dec.nv), cudaFree(s->dec.bm);
    CTX_CHECK(ctx, cudaMalloc(&s->dec.gt, sizeof(float) * max_set * s->k));
    CTX_CHECK(ctx, cudaMalloc(&s->dec.nv, sizeof(float) * max_set));
    CTX_CHECK(ctx, cudaMalloc(&s->dec.bm, sizeof(float) * max_set * s->k));
    s->dec.nset_cap = max_set;
  }
  return LATMAP_OK;
}

latmap_status latmap_session_set_batch(latmap_session* s, int32_t global_batch, int32_t add_trust) {
  if (!s || global_batch < 0) return LATMAP_ERR_INVALID_ARGUMENT;
  if (s->global_batch != global_batch || s->add_trust != add_trust) s->drop_graph();
  s->global_batch = global_batch;
  s->add_trust = add_trust;
  return session_alloc_frames(s, std::max(1, s->nframes));
}

latmap_status latmap_session_set_slot_offset(latmap_session* s, int32_t offset) {
  if (!s || offset < 0) return LATMAP_ERR_INVALID_ARGUMENT;
  if (s->slot_offset != offset) s->drop_graph();
  s->slot_offset = offset;
  return LATMAP_OK;
}

static bool session_sized(const latmap_session* s);
static latmap_status session_capture_step(latmap_session* s, bool with_adam);

latmap_status latmap_session_objective(latmap_session* s, int32_t want_grad, latmap_loss_breakdown* out) {
  if (!s || s->nframes < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  set_deterministic(s->ctx->deterministic);
  for (int attempt = 0; attempt < 3; ++attempt) {
    latmap_status st = LATMAP_OK;
    if (want_grad && s->use_graph && !s->prof && session_sized(s)) {
      // replayed objective graph (the multi-GPU step: objective -> all-reduce -> apply)
      if ((s->step_graph || s->obj_graph) &&
          (s->graph_exact != s->ctx->exact_blend || s->graph_dec_path != s->ctx->decoder_path ||
           s->graph_det != s->ctx->deterministic))
        s->drop_graph();
      if (!s->obj_graph) {
        st = session_capture_step(s, false);
        if (st != LATMAP_OK) return st;
      }
      CTX_CHECK(s->ctx, cudaGraphLaunch(s->obj_graph, s->ctx->stream));
      count_launch((int)s->obj_launches);
      s->renders_valid = true;
    } else {
      st = session_objective(s, want_grad != 0);
    }
    if (st != LATMAP_OK) return st;
    if (!out) return LATMAP_OK;
    CTX_CHECK(s->ctx, cudaStreamSynchronize(s->ctx->stream));
    if (!session_fix_overflow(s)) return session_assemble(s, out);
  }
  return fail(s->ctx, LATMAP_ERR_CUDA, "tile-pair buffer overflow persisted");
}

latmap_status latmap_session_apply(latmap_session* s) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  session_adam(s);
  return post_launch(s->ctx);
}

// Capture (objective + Adam) into s->step_graph. Requires sized tile buffers (a prior step).
static latmap_status session_capture_step(latmap_session* s, bool with_adam) {
  latmap_ctx* ctx = s->ctx;
  if (with_adam) {
    if (s->step_graph) cudaGraphExecDestroy(s->step_graph), s->step_graph = nullptr;
  } else {
    if (s->obj_graph) cudaGraphExecDestroy(s->obj_graph), s->obj_graph = nullptr;
  }
  // capture on a private non-blocking stream (the context's stream may be the legacy default
  // stream, which cannot be captured); the graph is then launched on the context's stream
  if (!s->cap_stream) CTX_CHECK(ctx, cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
  if (ctx->deterministic) {  // the fixed-order backward's scratch: allocated here, not inside the capture
    int64_t pairs = 1;
    for (int b = 0; b < s->nframes; ++b) pairs = std::max<int64_t>(pairs, s->rw[b].w.pair_cap);
    CTX_CHECK(ctx, ctx->det.ensure(std::max<int64_t>(s->n, 1), pairs, s->ds));
  }
  cudaStream_t saved = ctx->stream;
  // order the capture after everything already queued on the context stream
  CTX_CHECK(ctx, cudaStreamSynchronize(saved));
  ctx->stream = s->cap_stream;
  cudaGraph_t g = nullptr;
  const int64_t l0 = g_launches.load();
  cudaError_t e = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    ctx->stream = saved;
    CTX_CHECK(ctx, e);
  }
  latmap_status rs = session_objective(s, true);
  if (rs == LATMAP_OK && with_adam) session_adam(s);
  e = cudaStreamEndCapture(s->cap_stream, &g);
  ctx->stream = saved;
  const int64_t captured = g_launches.load() - l0;
  g_launches.fetch_sub(captured);  // captured, not executed
  if (rs != LATMAP_OK) {
    if (g) cudaGraphDestroy(g);
    return rs;
  }
  CTX_CHECK(ctx, e);
  e = cudaGraphInstantiate(with_adam ? &s->step_graph : &s->obj_graph, g, 0);
  cudaGraphDestroy(g);
  CTX_CHECK(ctx, e);
  (with_adam ? s->graph_launches : s->obj_launches) = captured;
  s->graph_exact = ctx->exact_blend;
  s->graph_det = ctx->deterministic;
  s->graph_dec_path = ctx->decoder_path;
  return LATMAP_OK;
}

static bool session_sized(const latmap_session* s) {
  for (int b = 0; b < s->nframes; ++b)
    if (s->rw[b].w.pair_cap <= 1) return false;
  return true;
}

latmap_status latmap_session_set_graphs(latmap_session* s, int32_t enable) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  s->use_graph = enable != 0;
  if (!s->use_graph) s->drop_graph();
  return LATMAP_OK;
}

static bool early_cf_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LATMAP_EARLY_CF");
    return !(e && e[0] == '0');
  }();
  return on;
}

// RAII: the colour / feature Adam blocks may run early inside this step's objective
struct EarlyCf {
  latmap_session* s;
  explicit EarlyCf(latmap_session* s_) : s(s_) { s->early_cf = early_cf_enabled(); }
  ~EarlyCf() { s->early_cf = false; }
};

latmap_status latmap_session_step(latmap_session* s, latmap_loss_breakdown* out) {
  if (!s || s->nframes < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  set_deterministic(s->ctx->deterministic);
  EarlyCf early(s);
  for (int attempt = 0; attempt < 3; ++attempt) {
    latmap_status st = LATMAP_OK;
    if (s->use_graph && !s->prof && session_sized(s)) {
      if ((s->step_graph || s->obj_graph) &&
          (s->graph_exact != s->ctx->exact_blend || s->graph_dec_path != s->ctx->decoder_path ||
           s->graph_det != s->ctx->deterministic))
        s->drop_graph();
      if (!s->step_graph) {
        st = session_capture_step(s, true);
        if (st != LATMAP_OK) return st;
      }
      CTX_CHECK(s->ctx, cudaGraphLaunch(s->step_graph, s->ctx->stream));
      count_launch((int)s->graph_launches);
      s->renders_valid = false;
    } else {
      st = session_objective(s, true);
      if (st != LATMAP_OK) return st;
      session_adam(s);  // no-op on device when a tile buffer overflowed
    }
    if (!out) return post_launch(s->ctx);
    st = session_assemble(s, out);
    if (st != LATMAP_OK) return st;
    if (!session_fix_overflow(s)) return LATMAP_OK;
  }
  return fail(s->ctx, LATMAP_ERR_CUDA, "tile-pair buffer overflow persisted");
}

latmap_status latmap_session_objective_ex(latmap_session* s, int32_t want_grad, int32_t map_grads,
                                          int32_t use_cached_renders, latmap_loss_breakdown* out) {
  if (!s || s->nframes < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  set_deterministic(s->ctx->deterministic);
  for (int attempt = 0; attempt < 3; ++attempt) {
    latmap_status st = session_objective(s, want_grad != 0, map_grads != 0, use_cached_renders != 0);
    if (st != LATMAP_OK) return st;
    if (!out) return LATMAP_OK;
    CTX_CHECK(s->ctx, cudaStreamSynchronize(s->ctx->stream));
    if (!session_fix_overflow(s)) return session_assemble(s, out);
    s->renders_valid = false;
  }
  return fail(s->ctx, LATMAP_ERR_CUDA, "tile-pair buffer overflow persisted");
}

latmap_status latmap_session_step_dict(latmap_session* s, latmap_loss_breakdown* out) {
  if (!s || s->nframes < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  set_deterministic(s->ctx->deterministic);
  for (int attempt = 0; attempt < 3; ++attempt) {
    latmap_status st = session_objective(s, true, false, true);
    if (st != LATMAP_OK) return st;
    session_adam(s, true);  // no-op on device when a tile buffer overflowed
    if (!out) return post_launch(s->ctx);
    st = session_assemble(s, out);
    if (st != LATMAP_OK) return st;
    if (!session_fix_overflow(s)) return LATMAP_OK;
    s->renders_valid = false;
  }
  return fail(s->ctx, LATMAP_ERR_CUDA, "tile-pair buffer overflow persisted");
}

// ------------------------------------------------------------------ map row-set changes
// AoS row = [position 3 | rotation 4 | color 3 | log_scale 3 | opacity 1 | features ds] (the
// store's record layout, voxel_hash.hpp:61-72).
namespace {
struct MapOff {
  int64_t o[6];
};
__global__ void soa_to_aos_kernel(const float* __restrict__ p, MapOff mo, int64_t n, int ds, float* __restrict__ rows) {
  const int rs = 14 + ds;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / rs;
    const int c = (int)(e % rs);
    float v;
    if (c < 3) v = p[mo.o[0] + 3 * i + c];
    else if (c < 7) v = p[mo.o[1] + 4 * i + c - 3];
    else if (c < 10) v = p[mo.o[2] + 3 * i + c - 7];
    else if (c < 13) v = p[mo.o[3] + 3 * i + c - 10];
    else if (c == 13) v = p[mo.o[4] + i];
    else v = p[mo.o[5] + (int64_t)ds * i + c - 14];
    rows[e] = v;
  }
}
__global__ void aos_to_soa_kernel(const float* __restrict__ rows, MapOff mo, int64_t n, int ds, float* __restrict__ p) {
  const int rs = 14 + ds;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / rs;
    const int c = (int)(e % rs);
    const float v = rows[e];
    if (c < 3) p[mo.o[0] + 3 * i + c] = v;
    else if (c < 7) p[mo.o[1] + 4 * i + c - 3] = v;
    else if (c < 10) p[mo.o[2] + 3 * i + c - 7] = v;
    else if (c < 13) p[mo.o[3] + 3 * i + c - 10] = v;
    else if (c == 13) p[mo.o[4] + i] = v;
    else p[mo.o[5] + (int64_t)ds * i + c - 14] = v;
  }
}
// moments of the map blocks: new row r < n_kept <- old row idx[r]; rows >= n_kept <- 0
__global__ void gather_moments_kernel(const float* __restrict__ src, MapOff so, float* __restrict__ dst, MapOff d_o,
                                      const int64_t* __restrict__ idx, int64_t n_kept, int64_t n_new, int ds) {
  const int w[6] = {3, 4, 3, 3, 1, ds};
  for (int b = 0; b < 6; ++b) {
    const int wb = w[b];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_new * wb;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = e / wb;
      const int c = (int)(e % wb);
      dst[d_o.o[b] + e] = r < n_kept ? src[so.o[b] + idx[r] * wb + c] : 0.f;
    }
  }
}
unsigned grid_cap(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16); }
}  // namespace

latmap_status latmap_session_export_rows(latmap_session* s, float* d_rows) {
  if (!s || (!d_rows && s->n > 0)) return LATMAP_ERR_INVALID_ARGUMENT;
  MapOff mo;
  for (int i = 0; i < 6; ++i) mo.o[i] = s->off[i];
  if (s->n > 0) {
    soa_to_aos_kernel<<<grid_cap(s->n * (14 + s->ds)), 256, 0, s->ctx->stream>>>(s->params, mo, s->n, s->ds, d_rows);
    count_launch();
  }
  return post_launch(s->ctx);
}

namespace {
// import_rows with the kept-row list already on the device (d_idx: n_kept ascending old rows)
latmap_status import_rows_impl(latmap_session* s, const float* d_rows, int64_t n_new, const int64_t* d_idx_kept,
                               int64_t n_kept) {
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const int ds = s->ds;
  const int64_t sizes[8] = {3 * n_new, 4 * n_new, 3 * n_new, 3 * n_new, n_new, (int64_t)ds * n_new,
                            (int64_t)ds * s->df, s->k * s->df};
  int64_t off[9];
  off[0] = 0;
  for (int i = 0; i < 8; ++i) off[i + 1] = pad4(off[i] + sizes[i]);
  const int64_t total = off[8];
  if (s->sp_cap < total + kShardSlack) {  // grow the spare set with headroom (the active set drifts frame to frame)
    for (float* p : {s->sp_params, s->sp_grads, s->sp_m, s->sp_v})
      if (p) cudaFree(p);
    s->sp_params = s->sp_grads = s->sp_m = s->sp_v = nullptr;
    s->sp_cap = 0;
    const int64_t cap = total + std::max<int64_t>(total / 4, kShardSlack);
    CTX_CHECK(ctx, cudaMalloc(&s->sp_params, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&s->sp_grads, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&s->sp_m, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&s->sp_v, sizeof(float) * cap));
    s->sp_cap = cap;
  }
  float *np = s->sp_params, *ng = s->sp_grads, *nm = s->sp_m, *nv = s->sp_v;
  const int64_t* d_idx = d_idx_kept;
  MapOff so, d_o;
  for (int i = 0; i < 6; ++i) so.o[i] = s->off[i], d_o.o[i] = off[i];
  if (n_new > 0) {
    aos_to_soa_kernel<<<grid_cap(n_new * (14 + ds)), 256, 0, st>>>(d_rows, d_o, n_new, ds, np);
    gather_moments_kernel<<<grid_cap(n_new * ds), 256, 0, st>>>(s->m, so, nm, d_o, d_idx, n_kept, n_new, ds);
    gather_moments_kernel<<<grid_cap(n_new * ds), 256, 0, st>>>(s->v, so, nv, d_o, d_idx, n_kept, n_new, ds);
    count_launch(3);
  }
  // dictionary blocks and their moments carry over unchanged
  const size_t dict = (size_t)(s->total - s->off[6]);
  CTX_CHECK(ctx, cudaMemcpyAsync(np + off[6], s->params + s->off[6], sizeof(float) * dict, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(nm + off[6], s->m + s->off[6], sizeof(float) * dict, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(nv + off[6], s->v + s->off[6], sizeof(float) * dict, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemsetAsync(ng, 0, sizeof(float) * std::max<int64_t>(total, 1), st));
  // swap: the old set (stream-ordered behind the copies above) becomes the next spare
  std::swap(s->params, s->sp_params), std::swap(s->grads, s->sp_grads), std::swap(s->m, s->sp_m),
      std::swap(s->v, s->sp_v), std::swap(s->cur_cap, s->sp_cap);
  s->n = n_new;
  for (int i = 0; i < 9; ++i) s->off[i] = off[i];
  for (int i = 0; i < 8; ++i) s->len[i] = sizes[i];
  s->total = total;
  // per-Gaussian render buffers grow to the new N; tile-pair capacity is kept (an overflow
  // re-runs the step with larger lists), so no sizing pass is needed per frame. geo_acc stays
  // all-zero between backward passes (project_bwd re-zeroes what it reads).
  for (auto& r : s->rw)
    if (r.w.pair_cap > 1) CTX_CHECK(ctx, r.ensure(n_new, s->intr.width, s->intr.height, r.w.pair_cap));
  s->renders_valid = false;
  s->drop_graph();
  return LATMAP_OK;
}
}  // namespace

latmap_status latmap_session_import_rows(latmap_session* s, const float* d_rows, int64_t n_new, const uint8_t* kept,
                                         int64_t n_kept) {
  if (!s || n_new < 0 || (n_new > 0 && !d_rows)) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  // rows of the old map whose Adam moments carry over, in order (MapOptimizer::keep_map_rows)
  std::vector<int64_t> idx;
  if (kept) {
    for (int64_t i = 0; i < s->n; ++i)
      if (kept[i]) idx.push_back(i);
  } else {
    for (int64_t i = 0; i < s->n; ++i) idx.push_back(i);
  }
  if ((kept && (int64_t)idx.size() != n_kept) || (int64_t)idx.size() > n_new)
    return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "import_rows: kept rows do not match the new row count");
  int64_t* d_idx = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&d_idx, sizeof(int64_t) * std::max<size_t>(idx.size(), 1), st));
  if (!idx.empty())
    CTX_CHECK(ctx, cudaMemcpyAsync(d_idx, idx.data(), sizeof(int64_t) * idx.size(), cudaMemcpyHostToDevice, st));
  const latmap_status r = import_rows_impl(s, d_rows, n_new, d_idx, (int64_t)idx.size());
  cudaFreeAsync(d_idx, st);
  return r;
}

latmap_status latmap_session_import_rows_device(latmap_session* s, const float* d_rows, int64_t n_new,
                                                const uint8_t* d_kept, int64_t n_kept) {
  if (!s || n_new < 0 || (n_new > 0 && !d_rows) || n_kept < 0 || n_kept > n_new || n_kept > s->n ||
      (n_kept > 0 && !d_kept))
    return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  int64_t* d_idx = nullptr;
  int32_t* d_blk = nullptr;
  int64_t* d_cnt = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&d_idx, sizeof(int64_t) * std::max<int64_t>(s->n, 1), st));
  CTX_CHECK(ctx, cudaMallocAsync(&d_blk, sizeof(int32_t) * (compact_blocks(s->n) + 1), st));
  CTX_CHECK(ctx, cudaMallocAsync(&d_cnt, sizeof(int64_t), st));
  if (d_kept && s->n > 0) CTX_CHECK(ctx, compact_mask(st, d_kept, s->n, d_idx, d_blk, d_cnt));
  const latmap_status r = import_rows_impl(s, d_rows, n_new, d_idx, d_kept ? n_kept : 0);
  cudaFreeAsync(d_idx, st);
  cudaFreeAsync(d_blk, st);
  cudaFreeAsync(d_cnt, st);
  return r;
}

int64_t latmap_session_size(const latmap_session* s) { return s ? s->n : -1; }

// ------------------------------------------------------------------ seeding (pipeline.cpp:39-73)
namespace {
constexpr int kSeedStride = 2;  // kStride
struct SeedArgs {
  const float *obs_depth, *alpha, *depth, *rgb;
  int w, h, gw, gh;
  float fx, fy, cx, cy, rwc[9], t[3];
};
__device__ __forceinline__ bool seed_cand(const SeedArgs& a, int i, int& x, int& y, float& z) {
  y = (i / a.gw) * kSeedStride;
  x = (i % a.gw) * kSeedStride;
  const size_t p = (size_t)y * a.w + x;
  z = a.obs_depth[p];
  if (!(z > 0.f)) return false;
  const float al = a.alpha[p], zr = a.depth[p];
  return al < 0.5f || fabsf(fs(zr, z)) > 0.1f;  // kAlphaCovered, kDepthErr
}
__global__ void seed_count_kernel(SeedArgs a, int32_t* blk) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int x, y;
  float z;
  const bool c = i < a.gw * a.gh && seed_cand(a, i, x, y, z);
  const int n = __syncthreads_count(c);
  if (threadIdx.x == 0) blk[blockIdx.x] = n;
}
__global__ void seed_scan_kernel(int32_t* blk, int nb, int64_t* total) {
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int b = 0; b < nb; ++b) {
      const int c = blk[b];
      blk[b] = (int32_t)run;
      run += c;
    }
    *total = run;
  }
}
// rows in raster order of the stride-2 grid: [position | (1,0,0,0) | rgb | log(z/fx*2) x3 | 0 | 0...]
__global__ void seed_write_kernel(SeedArgs a, const int32_t* blk, int ds, int64_t cap, float* rows) {
  __shared__ int32_t s_w[32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int x = 0, y = 0;
  float z = 0.f;
  const bool c = i < a.gw * a.gh && seed_cand(a, i, x, y, z);
  const unsigned bal = __ballot_sync(0xffffffffu, c);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_w[wid] = __popc(bal);
  __syncthreads();
  int base = blk[blockIdx.x];
  for (int w = 0; w < wid; ++w) base += s_w[w];
  if (!c) return;
  const int64_t r = base + __popc(bal & ((1u << lane) - 1u));
  if (r >= cap) return;
  float* o = rows + r * (14 + ds);
  const float pc[3] = {fm(fd(fs((float)x, a.cx), a.fx), z), fm(fd(fs((float)y, a.cy), a.fy), z), z};
  for (int k = 0; k < 3; ++k)
    o[k] = fa(fa(fa(fm(a.rwc[3 * k], pc[0]), fm(a.rwc[3 * k + 1], pc[1])), fm(a.rwc[3 * k + 2], pc[2])), a.t[k]);
  o[3] = 1.f, o[4] = 0.f, o[5] = 0.f, o[6] = 0.f;
  const size_t p = (size_t)y * a.w + x;
  o[7] = a.rgb[3 * p], o[8] = a.rgb[3 * p + 1], o[9] = a.rgb[3 * p + 2];
  const float ls = __double2float_rn(log((double)fm(fd(z, a.fx), 2.f)));  // std::log(float), two-pixel footprint
  o[10] = ls, o[11] = ls, o[12] = ls;
  o[13] = 0.f;  // opacity logit 0 -> alpha 0.5
  for (int k = 0; k < ds; ++k) o[14 + k] = 0.f;
}
}  // namespace

latmap_status latmap_session_seed_candidates(latmap_session* s, int32_t b, float* d_rows, int64_t cap,
                                             int64_t* count) {
  if (!s || b < 0 || b >= s->nframes || !count) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const FrameDev& f = s->frames[b];
  if (!s->renders_valid) {  // render(active map, kf.pose) right before seeding (pipeline.cpp:224-226)
    // frames 0..b only (the history frames behind b are not needed here); with a loss read-back
    // so a tile-list overflow is recovered before the candidates are taken
    const int32_t nf = s->nframes;
    s->nframes = b + 1;
    latmap_loss_breakdown tmp{};
    latmap_status rs = latmap_session_objective_ex(s, 0, 0, 0, &tmp);
    s->nframes = nf;
    s->renders_valid = false;  // frames after b were not rendered
    if (rs != LATMAP_OK) return rs;
  }
  wait_frame(s, b, st);
  SeedArgs a;
  a.obs_depth = f.depth, a.alpha = s->alpha[b], a.depth = s->depth[b], a.rgb = f.rgb;
  a.w = s->intr.width, a.h = s->intr.height;
  a.gw = (a.w + kSeedStride - 1) / kSeedStride, a.gh = (a.h + kSeedStride - 1) / kSeedStride;
  a.fx = s->intr.fx, a.fy = s->intr.fy, a.cx = s->intr.cx, a.cy = s->intr.cy;
  for (int i = 0; i < 9; ++i) a.rwc[i] = f.rwc[i];
  for (int i = 0; i < 3; ++i) a.t[i] = f.pose.translation[i];
  const int nc = a.gw * a.gh, nb = (nc + 255) / 256;
  int32_t* blk = nullptr;
  int64_t* tot = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&blk, sizeof(int32_t) * std::max(nb, 1), st));
  CTX_CHECK(ctx, cudaMallocAsync(&tot, sizeof(int64_t), st));
  seed_count_kernel<<<nb, 256, 0, st>>>(a, blk);
  seed_scan_kernel<<<1, 32, 0, st>>>(blk, nb, tot);
  if (d_rows) seed_write_kernel<<<nb, 256, 0, st>>>(a, blk, s->ds, cap, d_rows);
  count_launch(d_rows ? 3 : 2);
  CTX_CHECK(ctx, cudaMemcpyAsync(count, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CTX_CHECK(ctx, cudaFreeAsync(blk, st));
  CTX_CHECK(ctx, cudaFreeAsync(tot, st));
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  return post_launch(ctx);
}

latmap_status latmap_session_append_rows(latmap_session* s, float* d_rows, int64_t n_rows, const float* h_features) {
  if (!s || n_rows < 0 || (n_rows > 0 && !d_rows)) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const int rs = 14 + s->ds;
  if (n_rows > 0 && h_features)
    CTX_CHECK(ctx, cudaMemcpy2DAsync(d_rows + 14, sizeof(float) * rs, h_features, sizeof(float) * s->ds,
                                     sizeof(float) * s->ds, (size_t)n_rows, cudaMemcpyHostToDevice, st));
  // new map = current rows ++ appended rows; every current row keeps its moments
  float* all = nullptr;
  const int64_t n_old = s->n;
  CTX_CHECK(ctx, cudaMalloc(&all, sizeof(float) * std::max<int64_t>((n_old + n_rows) * rs, 1)));
  latmap_status r = latmap_session_export_rows(s, all);
  if (r == LATMAP_OK && n_rows > 0)
    r = cudaMemcpyAsync(all + n_old * rs, d_rows, sizeof(float) * n_rows * rs, cudaMemcpyDeviceToDevice, st) ==
                cudaSuccess
            ? LATMAP_OK
            : LATMAP_ERR_CUDA;
  if (r == LATMAP_OK) r = latmap_session_import_rows(s, all, n_old + n_rows, nullptr, n_old);
  cudaFree(all);
  return r;
}

latmap_status latmap_session_grad_buffer(latmap_session* s, float** grads, int64_t* count) {
  if (!s || !grads || !count) return LATMAP_ERR_INVALID_ARGUMENT;
  *grads = s->grads;
  *count = s->total;
  return LATMAP_OK;
}

latmap_status latmap_session_loss_buffer(latmap_session* s, double** partials, int64_t* count) {
  if (!s || !partials || !count) return LATMAP_ERR_INVALID_ARGUMENT;
  *partials = s->partials;
  *count = (int64_t)s->part_frames * kPart + kTail;
  return LATMAP_OK;
}

latmap_status latmap_session_read_loss(latmap_session* s, latmap_loss_breakdown* out) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  return session_assemble(s, out);
}

latmap_status latmap_session_read_loss_async(latmap_session* s, double* host_partials, int64_t cap, int64_t* count) {
  if (!s || !host_partials || !count) return LATMAP_ERR_INVALID_ARGUMENT;
  const int64_t n = (int64_t)s->part_frames * kPart + kTail;
  *count = n;
  if (cap < n) return fail(s->ctx, LATMAP_ERR_INVALID_ARGUMENT, "read_loss_async: buffer too small");
  CTX_CHECK(s->ctx, cudaMemcpyAsync(host_partials, s->partials, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                    s->ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_session_frame_images(latmap_session* s, int32_t b, float** color, float** depth, float** query,
                                          float** alpha) {
  if (!s || b < 0 || b >= s->nframes) return LATMAP_ERR_INVALID_ARGUMENT;
  if (color) *color = s->color[b];
  if (depth) *depth = s->depth[b];
  if (query) *query = s->query[b];
  if (alpha) *alpha = s->alpha[b];
  return LATMAP_OK;
}

// ------------------------------------------------------------------ sharded step (ZeRO-1)
// The keyframe-sharded iteration with the optimiser state split across ranks: reduce-scatter of
// the gradients (each rank owns one 4-aligned shard of the flat buffer), the shard's per-block
// non-finite flags joined to the loss partials (their all-reduce ORs them, so every rank skips the
// same blocks, adam.hpp:65-68), Adam on the shard only, all-gather of the parameters. The step
// counters stay replicated (every rank applies the same skip decisions).
latmap_status latmap_session_shard_range(const latmap_session* s, int32_t nranks, int32_t rank, int64_t* begin,
                                         int64_t* end) {
  if (!s || nranks < 1 || rank < 0 || rank >= nranks || !begin || !end || nranks * 4 > kShardSlack)
    return LATMAP_ERR_INVALID_ARGUMENT;
  const int64_t shard = (s->total + 4 * nranks - 1) / (4 * nranks) * 4;
  *begin = std::min<int64_t>(s->total, (int64_t)rank * shard);
  *end = std::min<int64_t>(s->total, *begin + shard);
  return LATMAP_OK;
}

latmap_status latmap_session_shard_check(latmap_session* s, int64_t begin, int64_t end) {
  if (!s || begin < 0 || end < begin || end > s->total) return LATMAP_ERR_INVALID_ARGUMENT;
  const latmap_config& c = s->cfg;
  const AdamBlock blocks[8] = {{s->off[0], s->len[0], 0.f, 0}, {s->off[1], s->len[1], 0.f, 1},
                               {s->off[2], s->len[2], 0.f, 0}, {s->off[3], s->len[3], 0.f, 0},
                               {s->off[4], s->len[4], 0.f, 0}, {s->off[5], s->len[5], 0.f, 0},
                               {s->off[6], s->len[6], 0.f, 0}, {s->off[7], s->len[7], 0.f, c.dict_learn ? 0 : -1}};
  adam_check_range(s->ctx->stream, s->grads, blocks, 8, begin, end,
                   s->partials + (size_t)s->part_frames * kPart + kTailBlockFlags);
  return post_launch(s->ctx);
}

latmap_status latmap_session_apply_range(latmap_session* s, int64_t begin, int64_t end) {
  if (!s || begin < 0 || end < begin || end > s->total) return LATMAP_ERR_INVALID_ARGUMENT;
  session_adam(s, false, begin, end, s->partials + (size_t)s->part_frames * kPart + kTailBlockFlags);
  return post_launch(s->ctx);
}

latmap_status latmap_session_params_buffer(latmap_session* s, float** params, int64_t* count) {
  if (!s || !params || !count) return LATMAP_ERR_INVALID_ARGUMENT;
  *params = s->params;
  *count = s->total;
  return LATMAP_OK;
}


// ------------------------------------------------------------------ keyframe transactions
// process_keyframe's snapshot / restore (pipeline.cpp:155-190, 294-306) for the device state:
// map rows, dictionary (proj, atoms, anchor, weights) and the Adam moments and counters.
latmap_status latmap_session_save_state(latmap_session* s) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  auto& sn = s->snap;
  if (sn.cap < s->total) {
    for (float** p : {&sn.params, &sn.m, &sn.v})
      if (*p) cudaFree(*p), *p = nullptr;
    sn.cap = 0;
    const int64_t cap = s->total + s->total / 4 + 1024;
    CTX_CHECK(ctx, cudaMalloc(&sn.params, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&sn.m, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&sn.v, sizeof(float) * cap));
    sn.cap = cap;
  }
  if (!sn.anchor) CTX_CHECK(ctx, cudaMalloc(&sn.anchor, sizeof(float) * s->k * s->df));
  CTX_CHECK(ctx, cudaMemcpyAsync(sn.params, s->params, sizeof(float) * s->total, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(sn.m, s->m, sizeof(float) * s->total, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(sn.v, s->v, sizeof(float) * s->total, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(sn.anchor, s->anchor, sizeof(float) * s->k * s->df, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(sn.steps, s->steps, sizeof(sn.steps), cudaMemcpyDeviceToHost, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(sn.skipped, s->skipped, sizeof(sn.skipped), cudaMemcpyDeviceToHost, st));
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  sn.n = s->n, sn.total = s->total;
  std::copy(s->off, s->off + 9, sn.off);
  std::copy(s->len, s->len + 8, sn.len);
  sn.dict_w = s->dict_w;
  sn.valid = true;
  return LATMAP_OK;
}

latmap_status latmap_session_restore_state(latmap_session* s) {
  if (!s || !s->snap.valid) return s ? fail(s->ctx, LATMAP_ERR_INVALID_ARGUMENT, "restore_state: no saved state")
                                     : LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  auto& sn = s->snap;
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  if (s->cur_cap < sn.total + kShardSlack) {  // the row set grew and shrank since: re-home the flat buffers
    for (float** p : {&s->params, &s->grads, &s->m, &s->v}) {
      if (*p) CTX_CHECK(ctx, cudaFree(*p));
      *p = nullptr;
    }
    const int64_t cap = sn.total + kShardSlack;
    CTX_CHECK(ctx, cudaMalloc(&s->params, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&s->grads, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&s->m, sizeof(float) * cap));
    CTX_CHECK(ctx, cudaMalloc(&s->v, sizeof(float) * cap));
    s->cur_cap = cap;
  }
  CTX_CHECK(ctx, cudaMemcpyAsync(s->params, sn.params, sizeof(float) * sn.total, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(s->m, sn.m, sizeof(float) * sn.total, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(s->v, sn.v, sizeof(float) * sn.total, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemsetAsync(s->grads, 0, sizeof(float) * (sn.total + kShardSlack), st));
  CTX_CHECK(ctx, cudaMemcpyAsync(s->anchor, sn.anchor, sizeof(float) * s->k * s->df, cudaMemcpyDeviceToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(s->steps, sn.steps, sizeof(sn.steps), cudaMemcpyHostToDevice, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(s->skipped, sn.skipped, sizeof(sn.skipped), cudaMemcpyHostToDevice, st));
  CTX_CHECK(ctx, cudaMemsetAsync(s->flags, 0, sizeof(int32_t) * 8, st));
  s->n = sn.n, s->total = sn.total;
  std::copy(sn.off, sn.off + 9, s->off);
  std::copy(sn.len, sn.len + 8, s->len);
  s->dict_w = sn.dict_w;
  for (auto& r : s->rw)
    if (r.w.pair_cap > 1) CTX_CHECK(ctx, r.ensure(s->n, s->intr.width, s->intr.height, r.w.pair_cap));
  s->renders_valid = false;
  s->drop_graph();
  CTX_CHECK(ctx, cudaStreamSynchronize(st));
  return LATMAP_OK;
}

latmap_status latmap_loss_assemble(const double* partials, int32_t nframes, int32_t width, int32_t height,
                                   const latmap_config* cfg, latmap_loss_breakdown* out) {
  if (!partials || !cfg || !out || nframes < 1 || width < 1 || height < 1) return LATMAP_ERR_INVALID_ARGUMENT;
  const latmap_config& c = *cfg;
  LossWeights wt{c.lambda_rgb, c.lambda_i1, c.lambda_i2, c.lambda_depth, c.lambda_feat, c.lambda_cos, c.lambda_l2,
                 c.lambda_trust};
  assemble_loss(partials, nframes, (double)width * height, 1.f / (float)nframes, wt, out);
  return LATMAP_OK;
}

latmap_status latmap_session_grad_layout(latmap_session* s, int64_t offsets[8], int64_t lengths[8]) {
  if (!s || !offsets || !lengths) return LATMAP_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < 8; ++i) offsets[i] = s->off[i], lengths[i] = s->len[i];
  return LATMAP_OK;
}

latmap_status latmap_session_check_overflow(latmap_session* s, int32_t* any) {
  if (!s || !any) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  double v = 0.0;
  CTX_CHECK(ctx, cudaMemcpyAsync(&v, s->partials + (size_t)s->part_frames * kPart + kTailOverflow, sizeof(double),
                                 cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  *any = v != 0.0;
  session_fix_overflow(s);  // grows this rank's tile buffers when its own lists overflowed
  return LATMAP_OK;
}

latmap_status latmap_session_overflow_steps(latmap_session* s, int64_t* count) {
  if (!s || !count) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  CTX_CHECK(ctx, cudaMemcpyAsync(count, s->overflow_steps, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_session_set_parity_export(latmap_session* s, int32_t enable) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  if (enable && !s->dec.row_nd) {
    CTX_CHECK(ctx, cudaMalloc(&s->dec.row_nd, sizeof(float) * 2 * std::max<int64_t>(s->dec.n_cap, 1)));
    CTX_CHECK(ctx, cudaMemset(s->dec.row_nd, 0, sizeof(float) * 2 * std::max<int64_t>(s->dec.n_cap, 1)));
  } else if (!enable && s->dec.row_nd) {
    CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
    CTX_CHECK(ctx, cudaFree(s->dec.row_nd));
    s->dec.row_nd = nullptr;
  }
  s->drop_graph();  // the kernels' export pointer is a captured argument
  return LATMAP_OK;
}

latmap_status latmap_session_decoder_export(latmap_session* s, int32_t* path, int64_t* rows, float* attention,
                                            float* row_nd) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  if (path) *path = s->dec.last_path;
  if (rows) *rows = s->dec.last_npx;
  const bool tc = s->dec.last_path == 2 || s->dec.last_path == 3;
  if ((attention || row_nd) && !tc)
    return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "decoder_export: the last decoded frame did not run a tcgen05 decoder");
  if (row_nd && !s->dec.row_nd)
    return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "decoder_export: parity export is not enabled");
  const int64_t n = s->dec.last_npx;
  if (attention && n > 0) decoder_export_attention(ctx->stream, s->dec, n, attention);
  if (row_nd && n > 0)
    CTX_CHECK(ctx, cudaMemcpyAsync(row_nd, s->dec.row_nd, sizeof(float) * 2 * n, cudaMemcpyDeviceToDevice, ctx->stream));
  CTX_CHECK(ctx, cudaGetLastError());
  CTX_CHECK(ctx, cudaStreamSynchronize(ctx->stream));
  return LATMAP_OK;
}

latmap_status latmap_weighted_kmeans(latmap_ctx* ctx, const float* points, const float* weights, int64_t n,
                                     int32_t dim, int64_t k, latmap_uniform_fn uniform, void* user,
                                     const float* warm, int64_t n_warm, int32_t max_iters, float* centers,
                                     float* center_weights, int32_t* iterations) {
  if (!ctx || n < 0 || dim < 1 || !centers || !center_weights || !iterations || (n > 0 && (!points || !weights)) ||
      (warm && n_warm < 0) || max_iters < 0)
    return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "weighted_kmeans: invalid arguments");
  if (k < 1) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "weighted_kmeans: k must be >= 1");
  if (!uniform) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "weighted_kmeans: no generator");
  cudaStream_t st = ctx->stream;
  const int64_t nw = warm ? std::min<int64_t>(n_warm, k) : 0;
  float *dp = nullptr, *dc = nullptr, *dw = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&dp, sizeof(float) * std::max<int64_t>(n, 1) * dim, st));
  CTX_CHECK(ctx, cudaMallocAsync(&dc, sizeof(float) * k * dim, st));
  if (nw > 0) CTX_CHECK(ctx, cudaMallocAsync(&dw, sizeof(float) * nw * dim, st));
  if (n > 0) CTX_CHECK(ctx, cudaMemcpyAsync(dp, points, sizeof(float) * n * dim, cudaMemcpyHostToDevice, st));
  if (nw > 0) CTX_CHECK(ctx, cudaMemcpyAsync(dw, warm, sizeof(float) * nw * dim, cudaMemcpyHostToDevice, st));
  int it = 0;
  cudaError_t e = kmeans_weighted(st, dp, weights, n, dim, k, uniform, user, nw > 0 ? dw : nullptr, nw, max_iters, dc,
                                  center_weights, &it);
  if (e == cudaSuccess) e = cudaMemcpyAsync(centers, dc, sizeof(float) * k * dim, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(dp, st);
  cudaFreeAsync(dc, st);
  if (dw) cudaFreeAsync(dw, st);
  CTX_CHECK(ctx, e);
  *iterations = it;
  return post_launch(ctx);
}

latmap_status latmap_session_stream_kmeans(latmap_session* s, const float* batch, int64_t n, float decay,
                                           latmap_uniform_fn uniform, void* user) {
  if (!s || n < 0 || (n > 0 && !batch)) return LATMAP_ERR_INVALID_ARGUMENT;
  latmap_ctx* ctx = s->ctx;
  if (!uniform) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "stream_kmeans_update: no generator");
  if (n == 0) return LATMAP_OK;  // empty batch: no-op (the pipeline skips maintenance too)
  cudaStream_t st = ctx->stream;
  float* db = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&db, sizeof(float) * n * s->df, st));
  CTX_CHECK(ctx, cudaMemcpyAsync(db, batch, sizeof(float) * n * s->df, cudaMemcpyHostToDevice, st));
  float* atoms = s->params + s->off[7];
  cudaError_t e = kmeans_stream_update(st, db, n, s->df, atoms, s->anchor, s->dict_w.data(), s->k, uniform, user, decay);
  cudaFreeAsync(db, st);
  CTX_CHECK(ctx, e);
  // MapOptimizer::reset_atom_moments: AdamState::reset of the atoms block (m = v = 0, step = 0)
  CTX_CHECK(ctx, cudaMemsetAsync(s->m + s->off[7], 0, sizeof(float) * s->len[7], st));
  CTX_CHECK(ctx, cudaMemsetAsync(s->v + s->off[7], 0, sizeof(float) * s->len[7], st));
  CTX_CHECK(ctx, cudaMemsetAsync(s->steps + 7, 0, sizeof(int64_t), st));
  return post_launch(ctx);
}

latmap_status latmap_session_get_dict_weights(const latmap_session* s, float* out) {
  if (!s || !out) return LATMAP_ERR_INVALID_ARGUMENT;
  std::memcpy(out, s->dict_w.data(), sizeof(float) * s->dict_w.size());
  return LATMAP_OK;
}

latmap_status latmap_session_set_dict_weights(latmap_session* s, const float* w) {
  if (!s || !w) return LATMAP_ERR_INVALID_ARGUMENT;
  for (size_t j = 0; j < s->dict_w.size(); ++j)
    if (!(w[j] >= 0.f)) return fail(s->ctx, LATMAP_ERR_INVALID_ARGUMENT, "dictionary weights must be >= 0");
  std::memcpy(s->dict_w.data(), w, sizeof(float) * s->dict_w.size());
  return LATMAP_OK;
}

latmap_status latmap_gather_supervision(latmap_ctx* ctx, const float* query, int32_t ds, const int32_t* assignment,
                                        int64_t npx, const float* features, int32_t df, int32_t normalize,
                                        float* q_out, float* t_out, int64_t* pixel_of_row, int64_t cap,
                                        int64_t* n_rows) {
  if (!ctx || !n_rows || npx < 0 || ds < 1 || df < 1 || (npx > 0 && !assignment) ||
      (q_out && (!query || !t_out || !pixel_of_row || !features)))
    return LATMAP_ERR_INVALID_ARGUMENT;
  CTX_CHECK(ctx, gather_supervision_dev(ctx->stream, query, ds, assignment, npx, features, df, normalize != 0, q_out,
                                        t_out, pixel_of_row, cap, n_rows));
  if (q_out && *n_rows > cap) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "gather_supervision: output capacity");
  return post_launch(ctx);
}

latmap_status latmap_metric_cos(latmap_ctx* ctx, const float* reconstructed, const float* target, int64_t n,
                                int32_t d, double* value, int32_t* flagged) {
  if (!ctx || !value || n < 0 || d < 1 || (n > 0 && (!reconstructed || !target))) return LATMAP_ERR_INVALID_ARGUMENT;
  CTX_CHECK(ctx, metric_cos_dev(ctx->stream, reconstructed, target, n, d, value, flagged));
  return post_launch(ctx);
}

latmap_status latmap_metric_miou(latmap_ctx* ctx, const float* embeddings, const int32_t* labels, int64_t n,
                                 int32_t d, const float* prototypes, int32_t c, int64_t* intersection,
                                 int64_t* union_, double* miou) {
  if (!ctx || !miou || n < 0 || d < 1 || c < 0 || (c > 0 && (!intersection || !union_ || !prototypes)) ||
      (n > 0 && (!embeddings || !labels)))
    return LATMAP_ERR_INVALID_ARGUMENT;
  bool bad = false;
  CTX_CHECK(ctx, metric_miou_dev(ctx->stream, embeddings, labels, n, d, prototypes, c, intersection, union_, miou, &bad));
  if (bad) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "metric_miou: label id out of range");
  return post_launch(ctx);
}

latmap_status latmap_metric_psnr(latmap_ctx* ctx, const float* rendered, const float* observed, int64_t n, double* db,
                                 int32_t* exact) {
  if (!ctx || !db || !exact || n < 1 || !rendered || !observed) return LATMAP_ERR_INVALID_ARGUMENT;
  CTX_CHECK(ctx, metric_psnr_dev(ctx->stream, rendered, observed, n, db, exact));
  return post_launch(ctx);
}

latmap_status latmap_query_map(latmap_ctx* ctx, const float* features, int64_t n, int32_t ds, const float* atoms,
                               const float* proj, int64_t k, int32_t df, float temperature, const float* embedding,
                               float* scores) {
  if (!ctx || n < 0 || !embedding || !scores || (n > 0 && !features)) return LATMAP_ERR_INVALID_ARGUMENT;
  if (n == 0) return LATMAP_OK;  // evaluate.cpp:77
  cudaStream_t st = ctx->stream;
  float* rec = nullptr;
  CTX_CHECK(ctx, cudaMallocAsync(&rec, sizeof(float) * n * df, st));
  latmap_status s = latmap_reconstruct(ctx, features, n, ds, atoms, proj, k, df, temperature, rec, nullptr);
  if (s == LATMAP_OK) CTX_CHECK(ctx, query_scores_dev(st, rec, n, df, embedding, scores));
  cudaFreeAsync(rec, st);
  return s == LATMAP_OK ? post_launch(ctx) : s;
}

latmap_status latmap_selftest_umma(latmap_ctx* ctx, const float* a, const float* b, float* c, int32_t n, int32_t k,
                                   int32_t a_mn, int32_t b_mn) {
  if (!ctx || !a || !b || !c) return LATMAP_ERR_INVALID_ARGUMENT;
  if (umma_selftest(ctx->stream, a, b, c, n, k, a_mn, b_mn)) return fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "bad shape");
  return post_launch(ctx);
}

latmap_status latmap_selftest_expf(latmap_ctx* ctx, uint64_t first, int64_t n, float* out) {
  if (!ctx || n < 0 || (n > 0 && !out)) return LATMAP_ERR_INVALID_ARGUMENT;
  if (n > 0) expf_selftest(ctx->stream, first, n, out);
  return post_launch(ctx);
}

latmap_status latmap_session_profile(latmap_session* s, int32_t enable) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  s->prof = enable != 0;
  return LATMAP_OK;
}

latmap_status latmap_session_phase_times(latmap_session* s, double* ms, int64_t* counts) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  CTX_CHECK(s->ctx, cudaStreamSynchronize(s->ctx->stream));
  for (auto& sp : s->spans) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, sp.a, sp.b) == cudaSuccess) {
      s->prof_ms[sp.phase] += t;
      s->prof_cnt[sp.phase] += 1;
    }
    s->pool.push_back(sp.a);
    s->pool.push_back(sp.b);
  }
  s->spans.clear();
  for (int i = 0; i < 8; ++i) {
    if (ms) ms[i] = s->prof_ms[i];
    if (counts) counts[i] = s->prof_cnt[i];
    s->prof_ms[i] = 0;
    s->prof_cnt[i] = 0;
  }
  return LATMAP_OK;
}

latmap_status latmap_session_stats(latmap_session* s, int64_t* visible, int64_t* pairs) {
  if (!s) return LATMAP_ERR_INVALID_ARGUMENT;
  CTX_CHECK(s->ctx, cudaStreamSynchronize(s->ctx->stream));
  for (int b = 0; b < s->nframes; ++b) {
    int64_t cnt[4];
    CTX_CHECK(s->ctx, cudaMemcpy(cnt, s->rw[b].w.counters, sizeof(cnt), cudaMemcpyDeviceToHost));
    if (visible) visible[b] = cnt[1];
    if (pairs) pairs[b] = cnt[0];
  }
  return LATMAP_OK;
}

}  // extern "C"
