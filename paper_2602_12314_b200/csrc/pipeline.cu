// The pipeline around the optimisation step: PipelineState,
// process_keyframe and run_pipeline's final flush (proj/src/pipeline.cpp:106-330,
// proj/include/latmap/pipe/pipeline.hpp:14-115), written as a client of the public C-ABI: the
// device session (map, dictionary, Adam moments), the device/pinned voxel-hash store, and the
// host-side bookkeeping the reference keeps next to them (history ring, std::mt19937_64, ActiveSet
// origins and dirty flags, travel distance). Every draw from the generator happens in the
// reference's order (stream k-means++ picks, history sampling, seeded features), so a run is
// reproducible against the reference's control flow for a given seed.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/latmap_b200.h"

latmap_status lm_ctx_fail(latmap_ctx* ctx, latmap_status s, const char* msg);  // capi.cu

namespace {

constexpr int kSeedStride = 2;  // pipeline.cpp:43

struct HostKeyframe {  // KeyframeT<float> (types.hpp:225-234), embeddings row-normalised
  int32_t frame_index = 0;
  latmap_pose pose{};
  std::vector<float> rgb, depth, features;
  std::vector<int32_t> assignment;
  int64_t n_set = 0;
};

double uniform01(void* user) {
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  return uni(*static_cast<std::mt19937_64*>(user));
}

}  // namespace

struct latmap_pipeline {
  latmap_ctx* ctx = nullptr;
  latmap_config cfg{};
  latmap_pipeline_config pc{};
  latmap_intrinsics intr{};
  latmap_session* s = nullptr;
  latmap_store* store = nullptr;
  // HistoryBuffer (pipeline.hpp:14-36)
  std::vector<std::shared_ptr<const HostKeyframe>> hist;
  size_t head = 0;
  std::mt19937_64 rng;
  float traveled = 0.f;
  bool have_last = false;
  float last[3] = {0, 0, 0};
  int32_t keyframes_processed = 0;
  int64_t peak_active = 0, reservoir_seen = 0;
  bool anchor_init = false;
  std::vector<float> persistent_anchor;
  // ActiveSet::origin / dirty (active_set.hpp:10-26); the rows live in the session
  std::vector<int64_t> origin;
  std::vector<uint8_t> dirty;
  // device scratch: seeding candidates, exported active rows, sync output
  float *d_seed = nullptr, *d_rows = nullptr, *d_out = nullptr;
  int64_t seed_cap = 0, rows_cap = 0, out_cap = 0;
  std::vector<int64_t> out_origin;
  std::vector<uint8_t> kept;
  bool failed = false;
  std::string err;
  int32_t fault_stage = 0;  // test hook (latmap_pipeline_inject_fault): fail the next keyframe at this point
};

namespace {

latmap_status pfail(latmap_pipeline* p, latmap_status st, const std::string& msg) {
  p->err = msg;
  return st;
}

// A device-side failure: inside process_keyframe the caller restores the keyframe's snapshot
// (and clears the flag); elsewhere (flush) the pipeline refuses further work.
latmap_status poison(latmap_pipeline* p, latmap_status st, const char* where, bool store_err = false) {
  p->failed = true;
  const char* m = store_err ? latmap_store_last_error(p->store) : latmap_ctx_last_error(p->ctx);
  p->err = std::string(where) + ": " + (m && *m ? m : "device error");
  return st;
}

#define PL_TRY(call, where)                        \
  do {                                             \
    latmap_status _st = (call);                    \
    if (_st != LATMAP_OK) return poison(p, _st, where); \
  } while (0)

latmap_status grow(latmap_pipeline* p, float** buf, int64_t* cap, int64_t need_floats) {
  if (*cap >= need_floats) return LATMAP_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  const int64_t n = std::max<int64_t>(need_floats + need_floats / 8, 1024);
  if (cudaMalloc(buf, sizeof(float) * n) != cudaSuccess) {
    *cap = 0;
    return pfail(p, LATMAP_ERR_OUT_OF_MEMORY, "pipeline: device scratch allocation failed");
  }
  *cap = n;
  return LATMAP_OK;
}

float row_norm(const float* r, int64_t d) {  // Eigen row().norm(): sqrt of the sum of squares
  float s = 0.f;
  for (int64_t j = 0; j < d; ++j) s += r[j] * r[j];
  return std::sqrt(s);
}

// sample_history (pipeline.cpp:19-37)
std::vector<size_t> sample_history(size_t n, int count, std::mt19937_64& rng) {
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

// sync (active_set.cpp:38-128) of the session's rows against the store, then
// MapOptimizer::keep_map_rows + the new ActiveSet (pipeline.cpp:276-281, 322-329).
latmap_status do_sync(latmap_pipeline* p, const float center[3], int64_t stats[5]) {
  const int64_t rs = 14 + p->pc.query_dim;
  const int64_t n = latmap_session_size(p->s);
  if (n > 0) {
    if (grow(p, &p->d_rows, &p->rows_cap, n * rs) != LATMAP_OK) return LATMAP_ERR_OUT_OF_MEMORY;
    PL_TRY(latmap_session_export_rows(p->s, p->d_rows), "sync: export_rows");
  }
  const int64_t cap = latmap_store_size(p->store) + n + 1;
  if (grow(p, &p->d_out, &p->out_cap, cap * rs) != LATMAP_OK) return LATMAP_ERR_OUT_OF_MEMORY;
  p->out_origin.resize((size_t)cap);
  p->kept.assign((size_t)std::max<int64_t>(n, 1), 0);
  int64_t cnt = 0;
  latmap_status st = latmap_store_sync(p->store, n ? p->d_rows : nullptr, p->origin.data(), p->dirty.data(), n, center,
                                       p->pc.local_radius, p->pc.voxel_size, p->d_out, p->out_origin.data(), cap,
                                       p->kept.data(), stats, &cnt);
  if (st != LATMAP_OK) return poison(p, st, "sync", true);
  int64_t nk = 0;
  for (int64_t i = 0; i < n; ++i) nk += p->kept[(size_t)i] != 0;
  PL_TRY(latmap_session_import_rows(p->s, p->d_out, cnt, n ? p->kept.data() : nullptr, n ? nk : 0),
         "sync: import_rows");
  p->origin.assign(p->out_origin.begin(), p->out_origin.begin() + cnt);
  p->dirty.assign((size_t)cnt, 0);
  return LATMAP_OK;
}

latmap_status validate(const latmap_config& c, const latmap_pipeline_config& pc, const latmap_intrinsics& in,
                       std::string* msg) {
  auto req = [&](bool ok, const char* m) {
    if (!ok && msg->empty()) *msg = std::string("config: ") + m;
    return ok;
  };
  bool ok = true;  // Config::validate (config.cpp:110-133), pipeline-level subset + the objective's
  ok &= req(pc.query_dim >= 1 && pc.embed_dim >= 1, "dimensions must be >= 1");
  ok &= req(pc.query_dim <= pc.embed_dim, "query_dim must be <= embed_dim");
  ok &= req(pc.dict_size >= 1, "dict_size must be >= 1");
  ok &= req(c.lambda_cos >= 0 && c.lambda_l2 >= 0 && c.lambda_trust >= 0 && c.lambda_i1 >= 0 && c.lambda_i2 >= 0 &&
                c.lambda_rgb >= 0 && c.lambda_depth >= 0 && c.lambda_feat >= 0,
            "loss weights must be >= 0");
  ok &= req(c.trust_delta >= 0, "trust_delta must be >= 0");
  ok &= req(pc.stage1_iters >= 0 && pc.stage2_iters >= 0, "iteration counts must be >= 0");
  ok &= req(pc.keyframe_stride >= 1, "keyframe_stride must be >= 1");
  ok &= req(pc.history_sample >= 0 && pc.history_capacity >= 1, "history sizes invalid");
  ok &= req(pc.voxel_size > 0, "voxel_size must be > 0");
  ok &= req(pc.local_radius > 0 && pc.sync_distance >= 0, "sync geometry invalid");
  ok &= req(pc.hash_capacity >= 1, "hash_capacity must be >= 1");
  ok &= req(c.softmax_temp > 0, "softmax_temp must be > 0");
  ok &= req(pc.dict_decay > 0 && pc.dict_decay <= 1, "dict_decay must be in (0,1]");
  ok &= req(pc.dict_init == 0 || pc.dict_init == 1, "dict_init must be kmeans|random");
  ok &= req(in.fx > 0 && in.fy > 0 && in.width > 0 && in.height > 0 && in.cx >= 0 && in.cx < float(in.width) &&
                in.cy >= 0 && in.cy < float(in.height),
            "invalid intrinsics");
  return ok ? LATMAP_OK : LATMAP_ERR_INVALID_ARGUMENT;
}

void destroy(latmap_pipeline* p) {
  if (p->s) latmap_session_destroy(p->s);
  if (p->store) latmap_store_destroy(p->store);
  for (float* b : {p->d_seed, p->d_rows, p->d_out})
    if (b) cudaFree(b);
  delete p;
}

}  // namespace

extern "C" {

void latmap_default_pipeline_config(latmap_pipeline_config* pc) {
  if (!pc) return;
  std::memset(pc, 0, sizeof(*pc));
  pc->query_dim = 32, pc->embed_dim = 64, pc->dict_size = 2000;  // config.hpp:12-14
  pc->stage1_iters = 1, pc->stage2_iters = 5;                     // :33-34
  pc->history_sample = 5, pc->history_capacity = 200;             // :36-37
  pc->voxel_size = 0.01f, pc->local_radius = 5.0f, pc->sync_distance = 1.0f;  // :39-41
  pc->hash_capacity = int64_t(1) << 20, pc->local_mapping = 1;    // :42-43
  pc->keyframe_stride = 4, pc->seed = 0;                          // :45-46
  pc->dict_init = 0, pc->dict_decay = 1.0f, pc->trust_anchor_persistent = 0;  // :49-53
}

int32_t latmap_select_keyframe(int32_t frame_index, int32_t stride) {
  if (stride < 1) return -1;  // pipeline.cpp:14-17 throws std::invalid_argument
  return frame_index % stride == 0;
}

const char* latmap_pipeline_last_error(const latmap_pipeline* p) { return p ? p->err.c_str() : ""; }

latmap_status latmap_pipeline_create(latmap_ctx* ctx, const latmap_config* cfg, const latmap_pipeline_config* pc,
                                     const latmap_intrinsics* intr, latmap_pipeline** out) {
  if (!ctx || !cfg || !pc || !intr || !out) return LATMAP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  auto* p = new latmap_pipeline();
  p->ctx = ctx, p->cfg = *cfg, p->pc = *pc, p->intr = *intr;
  std::string msg;
  if (validate(*cfg, *pc, *intr, &msg) != LATMAP_OK) {
    delete p;  // no pipeline handle to read the message from: it goes to the context
    return lm_ctx_fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, msg.c_str());
  }
  p->rng.seed(pc->seed);
  latmap_status st = latmap_session_create(ctx, cfg, 0, pc->query_dim, pc->dict_size, pc->embed_dim, intr, &p->s);
  if (st == LATMAP_OK) st = latmap_store_create(ctx, pc->hash_capacity, pc->query_dim, &p->store);
  // PipelineState::PipelineState (pipeline.cpp:106-121): zero atoms / anchor / weights, the
  // projection ~ N(0, 0.1) drawn row-major from the seeded generator
  if (st == LATMAP_OK) {
    const size_t kd = (size_t)pc->dict_size * pc->embed_dim, pd = (size_t)pc->query_dim * pc->embed_dim;
    std::vector<float> zeros(kd, 0.f), proj(pd), w((size_t)pc->dict_size, 0.f);
    std::normal_distribution<float> gauss(0.0f, 0.1f);
    for (auto& v : proj) v = gauss(p->rng);
    st = latmap_session_set_dictionary(p->s, zeros.data(), zeros.data(), proj.data());
    if (st == LATMAP_OK) st = latmap_session_set_dict_weights(p->s, w.data());
  }
  // one captured graph per keyframe batch only pays when Stage I repeats
  if (st == LATMAP_OK && pc->stage1_iters < 3) st = latmap_session_set_graphs(p->s, 0);
  if (st == LATMAP_OK) {
    const int64_t gw = (intr->width + kSeedStride - 1) / kSeedStride, gh = (intr->height + kSeedStride - 1) / kSeedStride;
    p->seed_cap = gw * gh;
    int64_t dummy = 0;
    st = grow(p, &p->d_seed, &dummy, p->seed_cap * (14 + pc->query_dim));
  }
  if (st != LATMAP_OK) {
    destroy(p);
    return st;
  }
  *out = p;
  return LATMAP_OK;
}

latmap_status latmap_pipeline_destroy(latmap_pipeline* p) {
  if (!p) return LATMAP_ERR_INVALID_ARGUMENT;
  destroy(p);
  return LATMAP_OK;
}

latmap_session* latmap_pipeline_session(latmap_pipeline* p) { return p ? p->s : nullptr; }
latmap_store* latmap_pipeline_store(latmap_pipeline* p) { return p ? p->store : nullptr; }

latmap_status latmap_pipeline_state(const latmap_pipeline* p, int64_t out[6]) {
  if (!p || !out) return LATMAP_ERR_INVALID_ARGUMENT;
  out[0] = p->keyframes_processed, out[1] = p->peak_active, out[2] = (int64_t)p->hist.size();
  out[3] = p->reservoir_seen, out[4] = p->failed ? 1 : 0;
  float tr = p->traveled;
  int32_t bits;
  std::memcpy(&bits, &tr, 4);
  out[5] = bits;  // traveled (float bits)
  return LATMAP_OK;
}

latmap_status latmap_pipeline_active_set(const latmap_pipeline* p, int64_t* origin, uint8_t* dirty) {
  if (!p) return LATMAP_ERR_INVALID_ARGUMENT;
  if (origin) std::copy(p->origin.begin(), p->origin.end(), origin);
  if (dirty) std::copy(p->dirty.begin(), p->dirty.end(), dirty);
  return LATMAP_OK;
}

}  // extern "C"

namespace {
latmap_status injected(latmap_pipeline* p, int32_t stage) {
  if (p->fault_stage != stage) return LATMAP_OK;
  p->fault_stage = 0;
  return pfail(p, LATMAP_ERR_CUDA, "injected fault (latmap_pipeline_inject_fault stage " + std::to_string(stage) + ")");
}

// process_keyframe_inner (pipeline.cpp:192-290)
latmap_status process_keyframe_inner(latmap_pipeline* p, const latmap_frame* kf, int32_t frame_index,
                                     latmap_keyframe_log* out) {
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t npx = (int64_t)p->intr.width * p->intr.height;
  const int32_t ed = p->pc.embed_dim, qd = p->pc.query_dim;
  // argument checks before any state changes (the reference's throw-and-restore leaves the
  // state untouched for these)
  if (!kf->rgb || !kf->depth || !kf->assignment || kf->n_set < 0 || (kf->n_set > 0 && !kf->features))
    return pfail(p, LATMAP_ERR_INVALID_ARGUMENT, "process_keyframe: missing frame arrays");
  for (int64_t i = 0; i < npx; ++i)
    if (kf->assignment[i] >= kf->n_set)
      return pfail(p, LATMAP_ERR_INVALID_ARGUMENT, "gather_supervision: assignment index out of range");

  latmap_keyframe_log row{};
  row.frame_index = frame_index;
  auto k = std::make_shared<HostKeyframe>();
  k->frame_index = frame_index, k->pose = kf->pose, k->n_set = kf->n_set;
  k->rgb.assign(kf->rgb, kf->rgb + npx * 3);
  k->depth.assign(kf->depth, kf->depth + npx);
  k->assignment.assign(kf->assignment, kf->assignment + npx);
  k->features.assign(kf->features ? kf->features : nullptr, kf->features ? kf->features + kf->n_set * ed : nullptr);
  for (int64_t r = 0; r < kf->n_set; ++r) {  // normalize_embedding_rows (pipeline.cpp:125-130)
    float* f = k->features.data() + r * ed;
    const float n = row_norm(f, ed);
    if (n > 1e-12f)
      for (int32_t j = 0; j < ed; ++j) f[j] /= n;
  }

  // 1. dictionary maintenance (pipeline.cpp:200-218)
  if (k->n_set > 0) {
    if (p->pc.dict_init == 0) {
      PL_TRY(latmap_session_stream_kmeans(p->s, k->features.data(), k->n_set, p->pc.dict_decay, &uniform01, &p->rng),
             "stream_kmeans_update");
    } else {  // random_dict_update (pipeline.cpp:136-153), then anchor = atoms
      const int64_t K = p->pc.dict_size;
      std::vector<float> atoms((size_t)K * ed), w((size_t)K);
      PL_TRY(latmap_session_get_dictionary(p->s, atoms.data(), nullptr), "random_dict_update");
      PL_TRY(latmap_session_get_dict_weights(p->s, w.data()), "random_dict_update");
      for (int64_t r = 0; r < k->n_set; ++r) {
        ++p->reservoir_seen;
        int64_t slot = -1;
        if (p->reservoir_seen <= K) {
          slot = p->reservoir_seen - 1;
        } else if (!p->cfg.dict_learn) {
          std::uniform_int_distribution<int64_t> pick(0, p->reservoir_seen - 1);
          const int64_t j = pick(p->rng);
          if (j < K) slot = j;
        }
        if (slot >= 0) {
          std::copy(k->features.begin() + r * ed, k->features.begin() + (r + 1) * ed, atoms.begin() + slot * ed);
          w[(size_t)slot] = 1.0f;
        }
      }
      PL_TRY(latmap_session_set_dictionary(p->s, atoms.data(), atoms.data(), nullptr), "random_dict_update");
      PL_TRY(latmap_session_set_dict_weights(p->s, w.data()), "random_dict_update");
    }
    if (p->pc.trust_anchor_persistent) {
      if (!p->anchor_init) {
        p->persistent_anchor.resize((size_t)p->pc.dict_size * ed);
        PL_TRY(latmap_session_get_anchor(p->s, p->persistent_anchor.data()), "persistent anchor");
        p->anchor_init = true;
      }
      PL_TRY(latmap_session_set_dictionary(p->s, nullptr, p->persistent_anchor.data(), nullptr), "persistent anchor");
    }
  }

  // 2. batch = the new keyframe + up to history_sample replayed ones (pipeline.cpp:220-222)
  std::vector<size_t> pick = sample_history(p->hist.size(), p->pc.history_sample, p->rng);
  std::vector<std::shared_ptr<const HostKeyframe>> batch{k};
  for (size_t i : pick) batch.push_back(p->hist[i]);
  std::vector<latmap_frame> frames(batch.size());
  for (size_t b = 0; b < batch.size(); ++b) {
    const HostKeyframe& h = *batch[b];
    frames[b] = latmap_frame{h.pose, h.rgb.data(), h.depth.data(), h.assignment.data(),
                             h.n_set ? h.features.data() : nullptr, h.n_set};
  }
  PL_TRY(latmap_session_set_frames(p->s, (int32_t)frames.size(), frames.data()), "set_frames");

  // 3. seeding against a render of the current map (pipeline.cpp:224-230)
  {
    int64_t n = 0;
    PL_TRY(latmap_session_seed_candidates(p->s, 0, p->d_seed, p->seed_cap, &n), "seed_gaussians");
    n = std::min(n, p->seed_cap);
    std::normal_distribution<float> gauss(0.0f, 0.01f);
    std::vector<float> feats((size_t)n * qd);
    for (auto& v : feats) v = gauss(p->rng);
    if (n > 0) PL_TRY(latmap_session_append_rows(p->s, p->d_seed, n, feats.data()), "append_newborns");
    row.seeded = n;
    p->origin.resize(p->origin.size() + (size_t)n, -1);
    p->dirty.resize(p->dirty.size() + (size_t)n, 1);
  }
  if (latmap_status fst = injected(p, 1)) return fst;

  // 4. Stage I, 5. Stage II (pipeline.cpp:232-266)
  bool have_loss = false;
  for (int it = 0; it < p->pc.stage1_iters; ++it) {
    PL_TRY(latmap_session_step(p->s, &row.loss), "stage I");
    have_loss = true;
    std::fill(p->dirty.begin(), p->dirty.end(), uint8_t(1));
  }
  for (int it = 0; it < p->pc.stage2_iters; ++it) {
    PL_TRY(latmap_session_step_dict(p->s, &row.loss), "stage II");
    have_loss = true;
  }
  if (!have_loss) PL_TRY(latmap_session_objective_ex(p->s, 0, 0, 0, &row.loss), "objective");
  if (latmap_status fst = injected(p, 2)) return fst;

  // 6. history push (HistoryBuffer::push)
  if ((int)p->hist.size() < p->pc.history_capacity) {
    p->hist.push_back(k);
  } else {
    p->hist[p->head] = k;
    p->head = (p->head + 1) % (size_t)p->pc.history_capacity;
  }

  // 7. travel and periodic synchronisation (pipeline.cpp:271-283)
  const float* t = k->pose.translation;
  if (p->have_last) {
    const float dx = t[0] - p->last[0], dy = t[1] - p->last[1], dz = t[2] - p->last[2];
    p->traveled += std::sqrt(dx * dx + dy * dy + dz * dz);
  }
  std::copy(t, t + 3, p->last);
  p->have_last = true;
  if (p->pc.local_mapping && p->traveled >= p->pc.sync_distance) {  // should_sync (active_set.hpp:51)
    latmap_status st = do_sync(p, t, row.sync);
    if (st != LATMAP_OK) return st;
    p->traveled = 0.f;
    row.synced = 1;
  }
  if (latmap_status fst = injected(p, 3)) return fst;

  ++p->keyframes_processed;
  const int64_t na = latmap_session_size(p->s);
  p->peak_active = std::max(p->peak_active, na);
  row.active_count = na;
  row.global_count = latmap_store_size(p->store);
  std::vector<float> w((size_t)p->pc.dict_size);
  PL_TRY(latmap_session_get_dict_weights(p->s, w.data()), "dict weights");
  float mass = 0.f;
  for (float v : w) mass += v;
  row.dict_weight_mass = double(mass);
  row.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (out) *out = row;
  return LATMAP_OK;
}

}  // namespace

extern "C" {

// process_keyframe (pipeline.cpp:292-312): the keyframe runs as a transaction. The state the
// reference snapshots (ActiveSet rows / origin / dirty, DictionaryState, MapOptimizer, travel,
// counters, persistent anchor, rng; pipeline.cpp:155-190) is saved first and restored when the
// keyframe fails, so the pipeline continues from the state before it. As in the reference the
// history buffer and the store are not part of the snapshot.
latmap_status latmap_pipeline_process_keyframe(latmap_pipeline* p, const latmap_frame* kf, int32_t frame_index,
                                               latmap_keyframe_log* out) {
  if (!p || !kf) return LATMAP_ERR_INVALID_ARGUMENT;
  if (p->failed) return pfail(p, LATMAP_ERR_INVALID_ARGUMENT, "pipeline: state lost after a failed keyframe (" + p->err + ")");
  struct Host {
    std::mt19937_64 rng;
    float traveled;
    bool have_last;
    float last[3];
    int32_t keyframes_processed;
    int64_t peak_active, reservoir_seen;
    bool anchor_init;
    std::vector<float> persistent_anchor;
    std::vector<int64_t> origin;
    std::vector<uint8_t> dirty;
  } snap{p->rng, p->traveled, p->have_last, {p->last[0], p->last[1], p->last[2]}, p->keyframes_processed,
         p->peak_active, p->reservoir_seen, p->anchor_init, p->persistent_anchor, p->origin, p->dirty};
  if (latmap_session_save_state(p->s) != LATMAP_OK) return poison(p, LATMAP_ERR_CUDA, "process_keyframe snapshot");
  const latmap_status st = process_keyframe_inner(p, kf, frame_index, out);
  if (st == LATMAP_OK) return LATMAP_OK;
  const std::string why = p->err;
  if (latmap_session_restore_state(p->s) != LATMAP_OK) return poison(p, st, "process_keyframe restore");
  p->rng = snap.rng, p->traveled = snap.traveled, p->have_last = snap.have_last;
  std::copy(snap.last, snap.last + 3, p->last);
  p->keyframes_processed = snap.keyframes_processed, p->peak_active = snap.peak_active;
  p->reservoir_seen = snap.reservoir_seen, p->anchor_init = snap.anchor_init;
  p->persistent_anchor = std::move(snap.persistent_anchor);
  p->origin = std::move(snap.origin), p->dirty = std::move(snap.dirty);
  p->failed = false;  // the inner failure poisoned the pipeline; the restore un-poisons it
  p->err = why;
  return st;
}

latmap_status latmap_pipeline_inject_fault(latmap_pipeline* p, int32_t stage) {
  if (!p || stage < 0 || stage > 3) return LATMAP_ERR_INVALID_ARGUMENT;
  p->fault_stage = stage;
  return LATMAP_OK;
}

// run_pipeline's final flush (pipeline.cpp:318-330): the whole active set written back.
latmap_status latmap_pipeline_flush(latmap_pipeline* p, int64_t stats[5]) {
  if (!p) return LATMAP_ERR_INVALID_ARGUMENT;
  if (p->failed) return pfail(p, LATMAP_ERR_INVALID_ARGUMENT, "pipeline: state lost after a failed keyframe (" + p->err + ")");
  int64_t local[5] = {0, 0, 0, 0, 0};
  if (latmap_session_size(p->s) > 0) {
    std::fill(p->dirty.begin(), p->dirty.end(), uint8_t(1));
    const float zero[3] = {0, 0, 0};
    latmap_status st = do_sync(p, p->have_last ? p->last : zero, local);
    if (st != LATMAP_OK) return st;
  }
  if (stats) std::copy(local, local + 5, stats);
  return LATMAP_OK;
}

}  // extern "C"
