// latmap_b200.hpp — C++ host layer over the C-ABI (latmap_b200.h), mirroring the reference
// operator API of proj/include/latmap/** (names, argument meaning, error behaviour):
//   latmap_b200::render / render_backward        <- latmap::render / render_backward (splat/render.hpp:103-119)
//   latmap_b200::reconstruct / reconstruct_backward / trust_region_penalty
//                                                <- dict/dictionary.hpp:63-77
//   latmap_b200::Session::total_objective / step  <- total_objective (obj/objective.hpp:49-54) +
//                                                   MapOptimizer::step_map/step_dict (pipe/pipeline.hpp:52-69)
//   latmap_b200::Pipeline / select_keyframe       <- PipelineState, process_keyframe (pipe/pipeline.hpp:82-107)
// Status codes map back to the reference's exceptions: LATMAP_ERR_INVALID_ARGUMENT ->
// std::invalid_argument, LATMAP_ERR_STALE_CACHE -> std::runtime_error, anything else ->
// latmap_b200::device_error. Device buffers are caller-owned raw pointers (any allocator).
#pragma once
#include <algorithm>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "latmap_b200.h"

namespace latmap_b200 {

struct device_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(latmap_status s, const latmap_ctx* ctx) {
  if (s == LATMAP_OK) return;
  const std::string msg = latmap_ctx_last_error(ctx);
  if (s == LATMAP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (s == LATMAP_ERR_STALE_CACHE) throw std::runtime_error(msg);
  throw device_error(msg.empty() ? "latmap_b200: device error" : msg);
}

// One context per host thread, bound to a device and a CUDA stream (cudaStream_t as void*).
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) { check(latmap_ctx_create(device, stream, &h_), nullptr); }
  ~Context() {
    if (h_) latmap_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  latmap_ctx* get() const { return h_; }
  void synchronize() { check(latmap_ctx_synchronize(h_), h_); }

 private:
  latmap_ctx* h_ = nullptr;
};

// std::uniform_real_distribution<double>(0, 1) over the caller's generator, as a C callback
// (k-means++ draws exactly what stream_kmeans.cpp:58-71 draws from the pipeline's rng).
template <class Rng>
double uniform01_trampoline(void* user) {
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  return uni(*static_cast<Rng*>(user));
}

// sample_history (pipeline.cpp:19-37): up to `count` of the n history keyframes, uniform without
// replacement by a partial Fisher-Yates over indices, drawing from the pipeline's generator
// exactly as the reference does (one uniform_int_distribution<size_t>(k, n - 1) per slot).
template <class Rng>
std::vector<size_t> sample_history(size_t n, int count, Rng& rng) {
  std::vector<size_t> out;
  if (n == 0 || count <= 0) return out;
  if (n <= size_t(count)) {
    for (size_t i = 0; i < n; ++i) out.push_back(i);
    return out;
  }
  std::vector<size_t> idx(n);
  for (size_t i = 0; i < n; ++i) idx[i] = i;
  for (int k = 0; k < count; ++k) {
    std::uniform_int_distribution<size_t> pick(size_t(k), n - 1);
    std::swap(idx[size_t(k)], idx[pick(rng)]);
    out.push_back(idx[size_t(k)]);
  }
  return out;
}

// weighted_kmeans (stream_kmeans.hpp:18-21) on the device; points row-major n x dim.
struct WeightedKmeansResult {
  std::vector<float> centers;  // k x dim
  std::vector<float> weights;  // k
  int iterations = 0;
};
template <class Rng>
WeightedKmeansResult weighted_kmeans(Context& ctx, const std::vector<float>& points, const std::vector<float>& weights,
                                     int64_t dim, int64_t k, Rng& rng, const std::vector<float>* warm = nullptr,
                                     int max_iters = 10) {
  const int64_t n = dim > 0 ? (int64_t)points.size() / dim : 0;
  if ((int64_t)weights.size() != n) throw std::invalid_argument("weighted_kmeans: weight count");
  WeightedKmeansResult r;
  r.centers.assign((size_t)(std::max<int64_t>(k, 0) * dim), 0.f);
  r.weights.assign((size_t)std::max<int64_t>(k, 0), 0.f);
  int32_t it = 0;
  check(latmap_weighted_kmeans(ctx.get(), points.data(), weights.data(), n, (int32_t)dim, k, &uniform01_trampoline<Rng>,
                               &rng, warm ? warm->data() : nullptr, warm ? (int64_t)warm->size() / dim : 0, max_iters,
                               r.centers.data(), r.weights.data(), &it),
        ctx.get());
  r.iterations = it;
  return r;
}

// RenderOutputT's cache half (splats + fingerprint); the images are caller-owned device buffers.
class RenderCache {
 public:
  explicit RenderCache(Context& ctx) : ctx_(&ctx) { check(latmap_render_cache_create(ctx.get(), &h_), ctx.get()); }
  ~RenderCache() {
    if (h_) latmap_render_cache_destroy(h_);
  }
  RenderCache(const RenderCache&) = delete;
  RenderCache& operator=(const RenderCache&) = delete;
  latmap_render_cache* get() const { return h_; }
  // RenderOutput::splats in source order (host copy).
  std::vector<latmap_projected_splat> splats() const {
    int64_t n = 0;
    check(latmap_render_cache_splats(ctx_->get(), h_, nullptr, 0, &n), ctx_->get());
    std::vector<latmap_projected_splat> out((size_t)n);
    check(latmap_render_cache_splats(ctx_->get(), h_, out.data(), n, &n), ctx_->get());
    return out;
  }

 private:
  Context* ctx_;
  latmap_render_cache* h_ = nullptr;
};

struct RenderImages {  // device pointers: color HxWx3, depth HxW, query HxWxds, alpha HxW
  float *color, *depth, *query, *alpha;
};

// render (splat/render.hpp:103-105)
inline void render(Context& ctx, const latmap_map& map, const latmap_pose& pose, const latmap_intrinsics& intr,
                   RenderCache& cache, const RenderImages& out) {
  check(latmap_render(ctx.get(), &map, &pose, &intr, cache.get(), out.color, out.depth, out.query, out.alpha),
        ctx.get());
}

// render_backward (splat/render.hpp:116-119); gradients are accumulated into `grads`.
inline void render_backward(Context& ctx, const latmap_map& map, const latmap_pose& pose,
                            const latmap_intrinsics& intr, const RenderCache& cache, const float* d_color,
                            const float* d_depth, const float* d_query, latmap_map& grads) {
  check(latmap_render_backward(ctx.get(), &map, &pose, &intr, cache.get(), d_color, d_depth, d_query, &grads),
        ctx.get());
}

// reconstruct (dict/dictionary.hpp:63-65)
inline void reconstruct(Context& ctx, const float* queries, int64_t n, int32_t query_dim, const float* atoms,
                        const float* proj, int64_t k, int32_t embed_dim, float temperature, float* out,
                        float* attention = nullptr) {
  check(latmap_reconstruct(ctx.get(), queries, n, query_dim, atoms, proj, k, embed_dim, temperature, out, attention),
        ctx.get());
}

// trust_region_penalty (dict/dictionary.hpp:75-77)
inline float trust_region_penalty(Context& ctx, const float* atoms, const float* anchor, int64_t k, int32_t df,
                                  float delta, float* d_atoms = nullptr) {
  float v = 0.f;
  check(latmap_trust_region_penalty(ctx.get(), atoms, anchor, k, df, delta, d_atoms, &v), ctx.get());
  return v;
}

// Device-resident GaussianMap + DictionaryState + MapOptimizer; one step() is one Stage-I
// iteration (pipeline.cpp:236-246).
class Session {
 public:
  Session(Context& ctx, const latmap_config& cfg, int64_t n, int32_t query_dim, int64_t k, int32_t embed_dim,
          const latmap_intrinsics& intr)
      : ctx_(&ctx), k_(k) {
    check(latmap_session_create(ctx.get(), &cfg, n, query_dim, k, embed_dim, &intr, &h_), ctx.get());
  }
  ~Session() {
    if (h_) latmap_session_destroy(h_);
  }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
  void set_map(const float* pos, const float* rot, const float* col, const float* lsc, const float* opa,
               const float* feat) {
    check(latmap_session_set_map(h_, pos, rot, col, lsc, opa, feat), ctx_->get());
  }
  void set_dictionary(const float* atoms, const float* anchor, const float* proj) {
    check(latmap_session_set_dictionary(h_, atoms, anchor, proj), ctx_->get());
  }
  void set_frames(const std::vector<latmap_frame>& frames) {
    check(latmap_session_set_frames(h_, (int32_t)frames.size(), frames.data()), ctx_->get());
  }
  // total_objective with gradients (objective.cpp:67-194)
  latmap_loss_breakdown total_objective() {
    latmap_loss_breakdown out{};
    check(latmap_session_objective(h_, 1, &out), ctx_->get());
    return out;
  }
  // MapOptimizer::step_map + step_dict (pipeline.cpp:75-95)
  void apply() { check(latmap_session_apply(h_), ctx_->get()); }
  latmap_loss_breakdown step() {
    latmap_loss_breakdown out{};
    check(latmap_session_step(h_, &out), ctx_->get());
    return out;
  }
  // total_objective with ObjectiveOptions::map_grads / cached_renders (objective.hpp:33-43)
  latmap_loss_breakdown total_objective(bool map_grads, bool use_cached_renders) {
    latmap_loss_breakdown out{};
    check(latmap_session_objective_ex(h_, 1, map_grads ? 1 : 0, use_cached_renders ? 1 : 0, &out), ctx_->get());
    return out;
  }
  // Stage II iteration: cached renders + MapOptimizer::step_dict (pipeline.cpp:250-259)
  latmap_loss_breakdown step_dict() {
    latmap_loss_breakdown out{};
    check(latmap_session_step_dict(h_, &out), ctx_->get());
    return out;
  }
  // Stage I x stage1 then Stage II x stage2 of process_keyframe_inner (pipeline.cpp:236-259);
  // returns the last LossBreakdown (KeyframeLog::loss).
  latmap_loss_breakdown optimize_keyframe(int stage1, int stage2) {
    latmap_loss_breakdown out{};
    bool have = false;
    for (int it = 0; it < stage1; ++it) out = step(), have = true;
    for (int it = 0; it < stage2; ++it) out = step_dict(), have = true;
    if (!have) check(latmap_session_objective_ex(h_, 0, 0, 0, &out), ctx_->get());
    return out;
  }
  // active-set row changes (keep_map_rows + append); rows are device AoS [n][14 + query_dim]
  void export_rows(float* d_rows) { check(latmap_session_export_rows(h_, d_rows), ctx_->get()); }
  void import_rows(const float* d_rows, int64_t n_new, const std::vector<uint8_t>* kept) {
    int64_t nk = 0;
    if (kept)
      for (uint8_t k : *kept) nk += k != 0;
    check(latmap_session_import_rows(h_, d_rows, n_new, kept ? kept->data() : nullptr, nk), ctx_->get());
  }
  int64_t size() const { return latmap_session_size(h_); }
  // seed_gaussians + append_newborns (pipeline.cpp:39-73, 224-230): candidates on the device,
  // features ~ N(0, 0.01) drawn here from the pipeline's generator in row order (as the reference
  // does); d_scratch must hold the frame's stride-2 grid rows ((W/2) x (H/2) x (14 + query_dim)).
  template <class Rng>
  int64_t seed_gaussians(int32_t frame, int32_t query_dim, Rng& rng, float* d_scratch, int64_t scratch_rows) {
    int64_t n = 0;
    check(latmap_session_seed_candidates(h_, frame, d_scratch, scratch_rows, &n), ctx_->get());
    n = std::min(n, scratch_rows);
    std::normal_distribution<float> gauss(0.0f, 0.01f);
    std::vector<float> feats((size_t)n * query_dim);
    for (auto& v : feats) v = gauss(rng);
    check(latmap_session_append_rows(h_, d_scratch, n, feats.data()), ctx_->get());
    return n;
  }
  // Dictionary maintenance for dict_init = "kmeans" (pipeline.cpp:201-205): stream_kmeans_update
  // with the keyframe's embedding rows (host, n x embed_dim) and the pipeline's generator, then
  // reset_atom_moments.
  template <class Rng>
  void stream_kmeans(const float* batch, int64_t n, Rng& rng, float decay = 1.0f) {
    check(latmap_session_stream_kmeans(h_, batch, n, decay, &uniform01_trampoline<Rng>, &rng), ctx_->get());
  }
  std::vector<float> dict_weights() const {
    std::vector<float> w((size_t)k_);
    check(latmap_session_get_dict_weights(h_, w.data()), ctx_->get());
    return w;
  }
  latmap_session* get() const { return h_; }

 private:
  Context* ctx_;
  int64_t k_ = 0;
  latmap_session* h_ = nullptr;
};

// PipelineState + process_keyframe + run_pipeline's flush (pipe/pipeline.hpp:82-107) over the
// C-ABI pipeline; argument errors -> std::invalid_argument, device errors -> device_error.
class Pipeline {
 public:
  Pipeline(Context& ctx, const latmap_config& cfg, const latmap_pipeline_config& pc, const latmap_intrinsics& intr)
      : ctx_(&ctx) {
    check(latmap_pipeline_create(ctx.get(), &cfg, &pc, &intr, &h_), ctx.get());
  }
  ~Pipeline() {
    if (h_) latmap_pipeline_destroy(h_);
  }
  Pipeline(const Pipeline&) = delete;
  Pipeline& operator=(const Pipeline&) = delete;
  latmap_keyframe_log process_keyframe(const latmap_frame& kf, int32_t frame_index) {
    latmap_keyframe_log row{};
    pcheck(latmap_pipeline_process_keyframe(h_, &kf, frame_index, &row));
    return row;
  }
  void flush(int64_t stats[5] = nullptr) { pcheck(latmap_pipeline_flush(h_, stats)); }
  latmap_session* session() const { return latmap_pipeline_session(h_); }
  latmap_store* store() const { return latmap_pipeline_store(h_); }

 private:
  void pcheck(latmap_status s) const {
    if (s == LATMAP_OK) return;
    const std::string msg = latmap_pipeline_last_error(h_);
    if (s == LATMAP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw device_error(msg.empty() ? "latmap_b200: device error" : msg);
  }
  Context* ctx_;
  latmap_pipeline* h_ = nullptr;
};

inline bool select_keyframe(int frame_index, int stride) {
  const int32_t r = latmap_select_keyframe(frame_index, stride);
  if (r < 0) throw std::invalid_argument("select_keyframe: stride must be >= 1");
  return r != 0;
}

}  // namespace latmap_b200
