// ref_capi.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// extern "C" shim over the REFERENCE library itself (oracle/_ref/liblatmap_ref.a, compiled from
// /root/reference/proj/src by oracle/ref/Makefile), so Python can run the unmodified reference on
// raw arrays: to pin the oracle restatement bit for bit, and as the CPU baseline of bench.py
// (`cpu_baseline.kind = "reference"`). Nothing in the product links or loads this.
//
// Layouts: the reference's fp32 row-major SoA (proj/include/latmap/core/types.hpp:95-100);
// images H x W x C interleaved; poses (w, x, y, z | tx, ty, tz), camera-to-world.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <vector>

#include "latmap/core/config.hpp"
#include "latmap/obj/objective.hpp"
#include "latmap/pipe/pipeline.hpp"
#include "latmap/splat/render.hpp"

using namespace latmap;

extern "C" {

struct latmap_ref_map {
  int64_t n;
  int32_t ds;
  const float *positions, *rotations, *colors, *log_scales, *opacity_logits, *features;
};
struct latmap_ref_frame {
  float pose[7];
  const float* rgb;          // H x W x 3
  const float* depth;        // H x W
  const int32_t* assignment;  // H x W
  const float* features;     // n_set x df
  int64_t n_set;
};
struct latmap_ref_intr {
  float fx, fy, cx, cy;
  int32_t width, height;
};
// The latmap::Config fields on the path (config.hpp:10-71); the rest keep their defaults.
struct latmap_ref_config {
  float trust_delta, lambda_cos, lambda_l2, lambda_trust, lambda_i1, lambda_i2, lambda_rgb, lambda_depth,
      lambda_feat, lr_proj, lr_dict, lr_position, lr_rotation, lr_color, lr_log_scale, lr_opacity, lr_feature,
      scene_extent, softmax_temp;
  int32_t dict_learn, segment_mode, num_threads;
};
struct latmap_ref_loss {
  float l_rgb, l_ssim, l_depth, l_cos, l_l2, l_trust, total;
  int64_t supervised_rows;
  int32_t depth_empty, zero_norm_flagged;
};
// The pipeline fields of latmap::Config (config.hpp:10-63), as api.PipelineConfig orders them.
struct latmap_ref_pipeline_config {
  int32_t query_dim, embed_dim, dict_size, stage1_iters, stage2_iters, history_sample, history_capacity;
  float voxel_size, local_radius, sync_distance;
  int64_t hash_capacity;
  int32_t local_mapping, keyframe_stride;
  uint64_t seed;
  int32_t dict_init;  // 0 kmeans, 1 random
  float dict_decay;
  int32_t trust_anchor_persistent;
};
// KeyframeLog (pipe/pipeline.hpp:70-80) without the wall time.
struct latmap_ref_keyframe_log {
  int32_t frame_index;
  latmap_ref_loss loss;
  int64_t seeded, active_count, global_count;
  double dict_weight_mass;
  int32_t synced;
  int64_t sync[5];  // written_back, newborn_inserted, newborn_rejected, pruned, fetched
};

}  // extern "C"

namespace {

thread_local std::string g_err;

GaussianMap make_map(const latmap_ref_map& m) {
  GaussianMap g;
  g.resize(m.n, m.ds);
  if (m.n > 0) {
    std::memcpy(g.positions.data(), m.positions, sizeof(float) * m.n * 3);
    std::memcpy(g.rotations.data(), m.rotations, sizeof(float) * m.n * 4);
    std::memcpy(g.colors.data(), m.colors, sizeof(float) * m.n * 3);
    std::memcpy(g.log_scales.data(), m.log_scales, sizeof(float) * m.n * 3);
    std::memcpy(g.opacity_logits.data(), m.opacity_logits, sizeof(float) * m.n);
    std::memcpy(g.features.data(), m.features, sizeof(float) * m.n * m.ds);
  }
  return g;
}

Pose make_pose(const float* p) {
  Pose q;
  q.rotation = Vec4f(p[0], p[1], p[2], p[3]);
  q.translation = Vec3f(p[4], p[5], p[6]);
  return q;
}

Intrinsics make_intr(const latmap_ref_intr& i) {
  Intrinsics o;
  o.fx = i.fx, o.fy = i.fy, o.cx = i.cx, o.cy = i.cy, o.width = i.width, o.height = i.height;
  return o;
}

Config make_config(const latmap_ref_config& c, int query_dim, int embed_dim, int dict_size) {
  Config o;
  o.query_dim = query_dim, o.embed_dim = embed_dim, o.dict_size = dict_size;
  o.trust_delta = c.trust_delta, o.lambda_cos = c.lambda_cos, o.lambda_l2 = c.lambda_l2;
  o.lambda_trust = c.lambda_trust, o.lambda_i1 = c.lambda_i1, o.lambda_i2 = c.lambda_i2;
  o.lambda_rgb = c.lambda_rgb, o.lambda_depth = c.lambda_depth, o.lambda_feat = c.lambda_feat;
  o.lr_proj = c.lr_proj, o.lr_dict = c.lr_dict, o.lr_position = c.lr_position, o.lr_rotation = c.lr_rotation;
  o.lr_color = c.lr_color, o.lr_log_scale = c.lr_log_scale, o.lr_opacity = c.lr_opacity;
  o.lr_feature = c.lr_feature, o.scene_extent = c.scene_extent, o.softmax_temp = c.softmax_temp;
  o.dict_learn = c.dict_learn != 0;
  o.feature_supervision = c.segment_mode ? "segment" : "pixel";
  o.num_threads = c.num_threads;
  return o;
}

Keyframe make_frame(const latmap_ref_frame& f, const latmap_ref_intr& in, int df) {
  Keyframe k;
  const int h = in.height, w = in.width;
  k.pose = make_pose(f.pose);
  k.rgb = Image(h, w, 3);
  std::memcpy(k.rgb.data.data(), f.rgb, sizeof(float) * h * w * 3);
  k.depth = Image(h, w, 1);
  std::memcpy(k.depth.data.data(), f.depth, sizeof(float) * h * w);
  k.embeddings.height = h, k.embeddings.width = w;
  k.embeddings.assignment.assign(f.assignment, f.assignment + size_t(h) * w);
  k.embeddings.features.setZero(f.n_set, df);
  if (f.n_set > 0) std::memcpy(k.embeddings.features.data(), f.features, sizeof(float) * f.n_set * df);
  return k;
}

DictionaryState make_dict(const float* atoms, const float* anchor, const float* proj, int64_t k, int32_t ds,
                          int32_t df, float temperature) {
  DictionaryState d;
  d.init(k, ds, df);
  std::memcpy(d.atoms.data(), atoms, sizeof(float) * k * df);
  std::memcpy(d.anchor.data(), anchor, sizeof(float) * k * df);
  std::memcpy(d.proj.data(), proj, sizeof(float) * ds * df);
  d.temperature = temperature;
  return d;
}

void copy_loss(const LossBreakdown<float>& l, latmap_ref_loss* o) {
  o->l_rgb = l.l_rgb, o->l_ssim = l.l_ssim, o->l_depth = l.l_depth, o->l_cos = l.l_cos, o->l_l2 = l.l_l2;
  o->l_trust = l.l_trust, o->total = l.total, o->supervised_rows = l.supervised_rows;
  o->depth_empty = l.depth_empty, o->zero_norm_flagged = l.zero_norm_flagged;
}

void copy_map_grads(const MapGradientsT<float>& g, float* out) {
  // flat [positions | rotations | colors | log_scales | opacity | features]
  const int64_t n = g.positions.rows(), ds = g.features.cols();
  float* p = out;
  std::memcpy(p, g.positions.data(), sizeof(float) * n * 3), p += n * 3;
  std::memcpy(p, g.rotations.data(), sizeof(float) * n * 4), p += n * 4;
  std::memcpy(p, g.colors.data(), sizeof(float) * n * 3), p += n * 3;
  std::memcpy(p, g.log_scales.data(), sizeof(float) * n * 3), p += n * 3;
  std::memcpy(p, g.opacity_logits.data(), sizeof(float) * n), p += n;
  std::memcpy(p, g.features.data(), sizeof(float) * n * ds);
}

struct Session {
  GaussianMap map;
  DictionaryState dict;
  std::vector<Keyframe> frames;
  Intrinsics intr;
  Config cfg;
  MapOptimizer opt;
  int threads = 1;
};

}  // namespace

extern "C" {

const char* latmap_ref_last_error() { return g_err.c_str(); }

// render<float> (render.hpp:103-105)
int latmap_ref_render(const latmap_ref_map* m, const float pose[7], const latmap_ref_intr* intr, int32_t threads,
                      float* color, float* depth, float* query, float* alpha) {
  try {
    const RenderOutput out = render(make_map(*m), make_pose(pose), make_intr(*intr), threads);
    std::memcpy(color, out.color.data.data(), sizeof(float) * out.color.size());
    std::memcpy(depth, out.depth.data.data(), sizeof(float) * out.depth.size());
    if (query) std::memcpy(query, out.query.data.data(), sizeof(float) * out.query.size());
    std::memcpy(alpha, out.alpha.data.data(), sizeof(float) * out.alpha.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// total_objective<float> (objective.hpp:49-54); grads (may be NULL): map grads flat + d_proj + d_atoms
int latmap_ref_total_objective(const latmap_ref_map* m, const float* atoms, const float* anchor, const float* proj,
                               int64_t k, int32_t df, float temperature, const latmap_ref_frame* frames,
                               int32_t nframes, const latmap_ref_intr* intr, const latmap_ref_config* cfg,
                               int32_t threads, latmap_ref_loss* loss, float* map_grads, float* d_proj,
                               float* d_atoms) {
  try {
    const GaussianMap map = make_map(*m);
    const DictionaryState dict = make_dict(atoms, anchor, proj, k, m->ds, df, temperature);
    std::vector<Keyframe> kfs;
    for (int b = 0; b < nframes; ++b) kfs.push_back(make_frame(frames[b], *intr, df));
    std::vector<const Keyframe*> batch;
    for (const auto& f : kfs) batch.push_back(&f);
    const Config c = make_config(*cfg, m->ds, df, int(k));
    ObjectiveOptions<float> opts;
    opts.threads = threads;
    ObjectiveGrads<float> g;
    const bool want = map_grads || d_proj || d_atoms;
    const LossBreakdown<float> l = total_objective(map, dict, batch, make_intr(*intr), c, want ? &g : nullptr, opts);
    copy_loss(l, loss);
    if (want) {
      if (map_grads) copy_map_grads(g.map, map_grads);
      if (d_proj) std::memcpy(d_proj, g.d_proj.data(), sizeof(float) * g.d_proj.size());
      if (d_atoms) std::memcpy(d_atoms, g.d_atoms.data(), sizeof(float) * g.d_atoms.size());
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// A persistent reference "session" for timing the Stage-I iteration (pipeline.cpp:236-246):
// total_objective with gradients, then MapOptimizer::step_map + step_dict (pipeline.cpp:75-95).
void* latmap_ref_session_create(const latmap_ref_map* m, const float* atoms, const float* anchor, const float* proj,
                                int64_t k, int32_t df, float temperature, const latmap_ref_frame* frames,
                                int32_t nframes, const latmap_ref_intr* intr, const latmap_ref_config* cfg,
                                int32_t threads) {
  try {
    auto* s = new Session();
    s->map = make_map(*m);
    s->dict = make_dict(atoms, anchor, proj, k, m->ds, df, temperature);
    for (int b = 0; b < nframes; ++b) s->frames.push_back(make_frame(frames[b], *intr, df));
    s->intr = make_intr(*intr);
    s->cfg = make_config(*cfg, m->ds, df, int(k));
    s->threads = threads;
    return s;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int latmap_ref_session_step(void* h, latmap_ref_loss* loss) {
  auto* s = static_cast<Session*>(h);
  try {
    std::vector<const Keyframe*> batch;
    for (const auto& f : s->frames) batch.push_back(&f);
    ObjectiveOptions<float> opts;
    opts.threads = s->threads;
    ObjectiveGrads<float> g;
    const LossBreakdown<float> l = total_objective(s->map, s->dict, batch, s->intr, s->cfg, &g, opts);
    s->opt.step_map(s->map, g.map, s->cfg);
    s->opt.step_dict(s->dict, g.d_proj, g.d_atoms, s->cfg, s->cfg.dict_learn);
    if (loss) copy_loss(l, loss);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// total_objective alone (with gradients) on the session's state, no optimiser step.
int latmap_ref_session_objective(void* h, latmap_ref_loss* loss) {
  auto* s = static_cast<Session*>(h);
  try {
    std::vector<const Keyframe*> batch;
    for (const auto& f : s->frames) batch.push_back(&f);
    ObjectiveOptions<float> opts;
    opts.threads = s->threads;
    ObjectiveGrads<float> g;
    const LossBreakdown<float> l = total_objective(s->map, s->dict, batch, s->intr, s->cfg, &g, opts);
    if (loss) copy_loss(l, loss);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The map after the session's steps, flat like the map gradients; the dictionary's atoms / proj.
int latmap_ref_session_get(void* h, float* map_flat, float* atoms, float* proj) {
  auto* s = static_cast<Session*>(h);
  MapGradientsT<float> tmp;
  tmp.positions = s->map.positions, tmp.rotations = s->map.rotations, tmp.colors = s->map.colors;
  tmp.log_scales = s->map.log_scales, tmp.opacity_logits = s->map.opacity_logits, tmp.features = s->map.features;
  if (map_flat) copy_map_grads(tmp, map_flat);
  if (atoms) std::memcpy(atoms, s->dict.atoms.data(), sizeof(float) * s->dict.atoms.size());
  if (proj) std::memcpy(proj, s->dict.proj.data(), sizeof(float) * s->dict.proj.size());
  return 0;
}

void latmap_ref_session_destroy(void* h) { delete static_cast<Session*>(h); }


// ---- the reference's keyframe pipeline (PipelineState / process_keyframe / run_pipeline's final
// flush, pipeline.cpp:106-330), for an independent check of csrc/pipeline.cu
void* latmap_ref_pipeline_create(const latmap_ref_config* c, const latmap_ref_pipeline_config* pc,
                                 const latmap_ref_intr* in) {
  try {
    Config cfg = make_config(*c, pc->query_dim, pc->embed_dim, pc->dict_size);
    cfg.stage1_iters = pc->stage1_iters, cfg.stage2_iters = pc->stage2_iters;
    cfg.history_sample = pc->history_sample, cfg.history_capacity = pc->history_capacity;
    cfg.voxel_size = pc->voxel_size, cfg.local_radius = pc->local_radius, cfg.sync_distance = pc->sync_distance;
    cfg.hash_capacity = pc->hash_capacity, cfg.local_mapping = pc->local_mapping != 0;
    cfg.keyframe_stride = pc->keyframe_stride, cfg.seed = pc->seed;
    cfg.dict_init = pc->dict_init == 1 ? "random" : "kmeans";
    cfg.dict_decay = pc->dict_decay, cfg.trust_anchor_persistent = pc->trust_anchor_persistent != 0;
    return new PipelineState(cfg, make_intr(*in));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int latmap_ref_pipeline_process(void* h, const latmap_ref_frame* f, int32_t frame_index,
                                latmap_ref_keyframe_log* out) {
  auto* st = static_cast<PipelineState*>(h);
  try {
    Keyframe kf = make_frame(*f, latmap_ref_intr{st->intr.fx, st->intr.fy, st->intr.cx, st->intr.cy, st->intr.width,
                                                 st->intr.height},
                             st->cfg.embed_dim);
    kf.frame_index = frame_index;
    const KeyframeLog row = process_keyframe(*st, std::move(kf));
    if (out) {
      out->frame_index = row.frame_index;
      copy_loss(row.loss, &out->loss);
      out->seeded = row.seeded, out->active_count = row.active_count, out->global_count = row.global_count;
      out->dict_weight_mass = row.dict_weight_mass;
      out->synced = row.synced;
      out->sync[0] = row.sync.written_back, out->sync[1] = row.sync.newborn_inserted;
      out->sync[2] = row.sync.newborn_rejected, out->sync[3] = row.sync.pruned, out->sync[4] = row.sync.fetched;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// run_pipeline's final flush (pipeline.cpp:320-330); stats[5] as SyncStats
int latmap_ref_pipeline_flush(void* h, int64_t* stats) {
  auto* st = static_cast<PipelineState*>(h);
  try {
    SyncStats ss;
    if (st->active.size() > 0) {
      std::vector<uint8_t> kept;
      st->active.mark_all_dirty();
      const Vec3f center = st->have_last_pos ? st->last_pos : Vec3f::Zero();
      ActiveSet next = sync(st->store, st->active, center, st->cfg.local_radius, st->cfg.voxel_size, &ss, &kept);
      st->opt.keep_map_rows(kept);
      st->active = std::move(next);
    }
    if (stats) {
      stats[0] = ss.written_back, stats[1] = ss.newborn_inserted, stats[2] = ss.newborn_rejected;
      stats[3] = ss.pruned, stats[4] = ss.fetched;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// active-set origins, the dictionary (atoms, proj, per-atom weights) and the store size
int64_t latmap_ref_pipeline_get(void* h, int64_t* origin, float* atoms, float* proj, float* weights,
                                int64_t* store_size) {
  auto* st = static_cast<PipelineState*>(h);
  const int64_t n = (int64_t)st->active.origin.size();
  if (origin) std::memcpy(origin, st->active.origin.data(), sizeof(int64_t) * n);
  if (atoms) std::memcpy(atoms, st->dict.atoms.data(), sizeof(float) * st->dict.atoms.size());
  if (proj) std::memcpy(proj, st->dict.proj.data(), sizeof(float) * st->dict.proj.size());
  if (weights)
    for (Eigen::Index i = 0; i < st->dict.weights.size(); ++i) weights[i] = (float)st->dict.weights[i];
  if (store_size) *store_size = st->store.size();
  return n;
}

void latmap_ref_pipeline_destroy(void* h) { delete static_cast<PipelineState*>(h); }

}  // extern "C"
