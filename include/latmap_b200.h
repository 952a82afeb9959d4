/*
 * latmap_b200.h — C-ABI of the B200-native latent-map optimisation step.
 *
 * Drop-in boundary for the reference operator API in
 * /root/reference/proj/include/latmap/ (LatentAM CPU reference). Every entry
 * point names the reference interface it replaces (file:line, relative to
 * /root/reference/proj/). Conventions:
 *   - extern "C", plain pointers and sizes, no C++ types, no exceptions;
 *   - tensors are fp32 row-major in the reference's SoA layouts
 *     (core/types.hpp:19-22,93-100); "device" pointers live on the context's GPU;
 *   - every call returns a latmap_status; the C++ layer (latmap_b200.hpp) maps
 *     LATMAP_ERR_INVALID_ARGUMENT -> std::invalid_argument and
 *     LATMAP_ERR_STALE_CACHE -> std::runtime_error, as the reference throws;
 *   - one context per host thread; calls on a context are stream-ordered on the
 *     stream it was created with (or set via latmap_ctx_set_stream).
 * There is no CPU fallback: without a CUDA device every call fails with
 * LATMAP_ERR_CUDA.
 */
#ifndef LATMAP_B200_H
#define LATMAP_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LATMAP_OK = 0,
  LATMAP_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  LATMAP_ERR_STALE_CACHE = 2,      /* std::runtime_error: render.cpp:256-260, dictionary.cpp:59-64 */
  LATMAP_ERR_CUDA = 3,
  LATMAP_ERR_OUT_OF_MEMORY = 4,
  LATMAP_ERR_UNSUPPORTED = 5
} latmap_status;

typedef struct latmap_ctx latmap_ctx;
typedef struct latmap_render_cache latmap_render_cache;
typedef struct latmap_session latmap_session;

/* Intrinsics, core/types.hpp:41-50 */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
} latmap_intrinsics;

/* PoseT<float>: (w,x,y,z) rotation + translation, camera-to-world, core/types.hpp:27-38 */
typedef struct {
  float rotation[4];
  float translation[3];
} latmap_pose;

/* GaussianMapT<float> / MapGradientsT<float> view (device pointers),
 * core/types.hpp:93-199, splat/render.hpp:57-92 */
typedef struct {
  int64_t n;
  int32_t query_dim;
  float* positions;      /* n x 3 */
  float* rotations;      /* n x 4 */
  float* colors;         /* n x 3 */
  float* log_scales;     /* n x 3 */
  float* opacity_logits; /* n     */
  float* features;       /* n x query_dim */
} latmap_map;

/* ProjectedSplat<float>, splat/render.hpp:31-39 */
typedef struct {
  float mean2d[2];
  float cov_inv[4]; /* row-major 2x2 */
  float depth;
  float alpha;
  int32_t source, x0, x1, y0, y1;
} latmap_projected_splat;

/* LossBreakdown<float>, obj/objective.hpp:12-24 */
typedef struct {
  float l_rgb, l_ssim, l_depth, l_cos, l_l2, l_trust, total;
  int64_t supervised_rows;
  int32_t depth_empty, zero_norm_flagged;
} latmap_loss_breakdown;

/* Hot-path subset of latmap::Config, core/config.hpp:10-71 (same defaults). */
typedef struct {
  float lambda_cos, lambda_l2, lambda_trust, trust_delta;
  float lambda_i1, lambda_i2, lambda_rgb, lambda_depth, lambda_feat;
  float lr_proj, lr_dict, lr_position, lr_rotation, lr_color, lr_log_scale, lr_opacity, lr_feature;
  float scene_extent;
  float softmax_temp;         /* DictionaryStateT::temperature (pipeline.cpp:116) */
  int32_t dict_learn;         /* step_dict learn_atoms (pipeline.cpp:91-95) */
  int32_t segment_mode;       /* feature_supervision == "segment" (objective.cpp:78) */
  int32_t decoder_precision;  /* 0: fp32 SIMT (bit-faithful algebra), 1: bf16 tcgen05 */
} latmap_config;

/* KeyframeT<float> as host arrays, core/types.hpp:224-248 */
typedef struct {
  latmap_pose pose;
  const float* rgb;          /* H x W x 3 */
  const float* depth;        /* H x W     */
  const int32_t* assignment; /* H x W, -1 = unsupervised (EmbeddingSetT, types.hpp:204-221) */
  const float* features;     /* n_set x embed_dim */
  int64_t n_set;
} latmap_frame;

/* ---------------------------------------------------------------- context */
latmap_status latmap_ctx_create(int32_t device, void* cuda_stream, latmap_ctx** out);
latmap_status latmap_ctx_destroy(latmap_ctx* ctx);
latmap_status latmap_ctx_set_stream(latmap_ctx* ctx, void* cuda_stream);
latmap_status latmap_ctx_synchronize(latmap_ctx* ctx);
/* Parity mode for the forward blend: 1 = colour/depth/query accumulated with separately rounded
 * products and sums in the reference's order (bit-exact images); 0 (default) = FMA accumulation
 * (images within 1e-6 relative). alpha', clamp and termination decisions are exact in both. */
latmap_status latmap_ctx_set_exact_blend(latmap_ctx* ctx, int32_t exact);
/* bf16 (tcgen05) decoder kernels: 0 = auto (fused on-chip DEC1/DEC2 when K in {128, 256},
 * d_s = 32, n_set <= 64; else the staged DL1-DL5 path for K in {256..1024}, d_s in {32, 64},
 * n_set <= 256; else fp32 SIMT), 1 = fused only, 2 = staged whenever it supports the shape.
 * Replaces no reference interface (the reference has one fp32 CPU decoder,
 * proj/src/dictionary.cpp:25-83); results agree within the bf16 tolerances either way. */
latmap_status latmap_ctx_set_decoder_path(latmap_ctx* ctx, int32_t path);
/* Standalone reconstruct precision (latmap_reconstruct, latmap_query_map): 0 fp32 (default),
 * 1 bf16 tcgen05 where the shape is supported. */
latmap_status latmap_ctx_set_reconstruct_precision(latmap_ctx* ctx, int32_t precision);
/* Deterministic mode: every gradient reduction in a fixed order instead of float atomics, so
 * gradients are bit-identical run to run (the reference's guarantee, render.cpp:272-273,358,
 * test_render.cpp:142-151). The render backward writes one partial row per (splat, tile) pair and
 * sums a splat's rows in the row-major order of its tile rectangle; the decoders' split-K /
 * per-CTA partial reductions run unsplit; segment pooling sums in raster order. Slower; off by
 * default. Loss values are sums in double (reported to double rounding). */
latmap_status latmap_ctx_set_deterministic(latmap_ctx* ctx, int32_t on);
const char* latmap_ctx_last_error(const latmap_ctx* ctx);
/* Device memory for callers that hold only this header (the Eigen-typed drop-in layer):
 * alloc / free (free synchronises the context stream) and copies on the context stream,
 * direction 0 host->device, 1 device->host (synchronous), 2 device->device. */
latmap_status latmap_device_alloc(latmap_ctx* ctx, int64_t bytes, void** out);
latmap_status latmap_device_free(latmap_ctx* ctx, void* p);
latmap_status latmap_copy(latmap_ctx* ctx, void* dst, const void* src, int64_t bytes, int32_t direction);
/* The cudaStream_t the context's calls are ordered on (as void*). */
void* latmap_ctx_stream(const latmap_ctx* ctx);
/* Kernels launched by this context since creation (evidence for the bench). */
int64_t latmap_ctx_launch_count(const latmap_ctx* ctx);
void latmap_default_config(latmap_config* cfg);

/* ---------------------------------------------------------------- renderer */
/* project_gaussian, splat/render.hpp:97-99 (host values in, host values out).
 * *visible = 0 when culled (std::nullopt). */
latmap_status latmap_project_gaussian(latmap_ctx* ctx, const float position[3], const float rotation[4],
                                      const float log_scale[3], float opacity_logit,
                                      const latmap_pose* pose, const latmap_intrinsics* intr,
                                      int32_t* visible, float mean2d[2], float cov2d[4], float* depth);

/* RenderOutputT::splats + fingerprint holder (splat/render.hpp:41-53). */
latmap_status latmap_render_cache_create(latmap_ctx* ctx, latmap_render_cache** out);
latmap_status latmap_render_cache_destroy(latmap_render_cache* cache);

/* render, splat/render.hpp:103-105. Device outputs: color HxWx3, depth HxW, query HxWxds, alpha HxW.
 * Fills `cache` (projected splats, (tile, depth)-sorted tile lists, per-pixel blend extents). */
latmap_status latmap_render(latmap_ctx* ctx, const latmap_map* map, const latmap_pose* pose,
                            const latmap_intrinsics* intr, latmap_render_cache* cache, float* color,
                            float* depth, float* query, float* alpha);

/* render_backward, splat/render.hpp:116-119. Upstream images may be NULL (= zero).
 * Gradients are ACCUMULATED (+=) into `grads` (device); LATMAP_ERR_STALE_CACHE when
 * the cache fingerprint does not match (render.cpp:256-260). */
latmap_status latmap_render_backward(latmap_ctx* ctx, const latmap_map* map, const latmap_pose* pose,
                                     const latmap_intrinsics* intr, const latmap_render_cache* cache,
                                     const float* d_color, const float* d_depth, const float* d_query,
                                     latmap_map* grads);

/* Parity exports (host buffers): splats in source order (RenderOutput::splats), and the
 * canonical tile lists (16x16 tiles; per tile the sources whose bbox meets it, ordered by
 * (depth, source)). Pass NULL buffers to query sizes. */
latmap_status latmap_render_cache_splats(latmap_ctx* ctx, const latmap_render_cache* cache,
                                         latmap_projected_splat* out, int64_t cap, int64_t* count);
latmap_status latmap_render_cache_tiles(latmap_ctx* ctx, const latmap_render_cache* cache,
                                        int32_t* tile_offsets, int32_t* tile_sources, int64_t cap,
                                        int32_t* tiles_x, int32_t* tiles_y, int64_t* pairs);

/* ---------------------------------------------------------------- decoder (device pointers) */
/* reconstruct, dict/dictionary.hpp:63-65: out = softmax(Q W D^T / temperature) D.
 * attention (n x K) optional (AttentionCache::attention). With the context's reconstruct
 * precision set to 1, no attention requested, K in {256, 512, 768, 1024}, query_dim in {32, 64}
 * and embed_dim a multiple of 256, the product runs on the tensor cores (bf16 operands, fp32
 * accumulation: the precision of the configs' bf16 decoder); otherwise in fp32. query_map and
 * evaluation go through this entry point. */
latmap_status latmap_reconstruct(latmap_ctx* ctx, const float* queries, int64_t n, int32_t query_dim,
                                 const float* atoms, const float* proj, int64_t k, int32_t embed_dim,
                                 float temperature, float* out, float* attention);
/* reconstruct_backward, dict/dictionary.hpp:67-70 (general upstream d_rec). */
latmap_status latmap_reconstruct_backward(latmap_ctx* ctx, const float* queries, const float* attention,
                                          int64_t n, int32_t query_dim, const float* atoms,
                                          const float* proj, int64_t k, int32_t embed_dim,
                                          float temperature, const float* d_rec, float* d_queries,
                                          float* d_proj, float* d_atoms);
/* trust_region_penalty, dict/dictionary.hpp:75-77. d_atoms may be NULL. penalty: host float. */
latmap_status latmap_trust_region_penalty(latmap_ctx* ctx, const float* atoms, const float* anchor,
                                          int64_t k, int32_t embed_dim, float delta, float* d_atoms,
                                          float* penalty);

/* ---------------------------------------------------------------- losses (device pointers) */
/* ssim, obj/losses.hpp:12-13; d_a optional (overwritten). Returns the mean SSIM in *value. */
latmap_status latmap_ssim(latmap_ctx* ctx, const float* a, const float* b, int32_t h, int32_t w,
                          int32_t channels, float* d_a, float* value);

/* rgb_loss, obj/losses.hpp:33-34 (losses.cpp:200-224): lambda_i1 mean|a - b| + lambda_i2 (1 - SSIM)/2
 * over H x W x channels images (device). grad (device, may be NULL) receives the gradient w.r.t.
 * `rendered`; value / l1 / ssim_loss are host floats (l1, ssim_loss may be NULL). */
latmap_status latmap_rgb_loss(latmap_ctx* ctx, const float* rendered, const float* observed, int32_t h, int32_t w,
                              int32_t channels, float lambda_i1, float lambda_i2, float* grad, float* value,
                              float* l1, float* ssim_loss);
/* depth_loss, obj/losses.hpp:38-40 (losses.cpp:226-255): mean |rendered - observed| over pixels
 * with observed > 0 and alpha > 0.5; *flagged = 1 (value 0, grad all zero) when none qualifies.
 * n = H x W; grad (device, may be NULL). */
latmap_status latmap_depth_loss(latmap_ctx* ctx, const float* rendered, const float* observed, const float* alpha,
                                int64_t n, float* grad, float* value, int32_t* flagged);
/* feature_loss, obj/losses.hpp:43-58 (losses.cpp:257-294): terms = {value, cos_term, l2_term,
 * trust_term} (host); d_reconstructed (n x embed_dim) and d_atoms_trust (k x embed_dim,
 * lambda_trust-scaled) are device outputs, either may be NULL. */
latmap_status latmap_feature_loss(latmap_ctx* ctx, const float* reconstructed, const float* target, int64_t n,
                                  int32_t embed_dim, const float* atoms, const float* anchor, int64_t k, float delta,
                                  float lambda_cos, float lambda_l2, float lambda_trust, float* d_reconstructed,
                                  float* d_atoms_trust, float terms[4], int32_t* zero_norm_flagged);

/* ---------------------------------------------------------------- optimiser */
/* adam_step, obj/adam.hpp:61-79 on one device block. *step / *skipped are the host-side
 * AdamState counters (updated); returns *applied = 0 when the block had a non-finite grad. */
latmap_status latmap_adam_step(latmap_ctx* ctx, float* param, const float* grad, float* m, float* v,
                               int64_t count, int64_t* step, int64_t* skipped, float lr,
                               int32_t* applied);

/* ---------------------------------------------------------------- device-resident session */
/* The throughput path: GaussianMap + DictionaryState + MapOptimizer moments stay in HBM;
 * one latmap_session_step == one Stage-I iteration (pipeline.cpp:236-246):
 * total_objective (objective.cpp:67-194) -> step_map -> step_dict (pipeline.cpp:75-95). */
latmap_status latmap_session_create(latmap_ctx* ctx, const latmap_config* cfg, int64_t n,
                                    int32_t query_dim, int64_t k, int32_t embed_dim,
                                    const latmap_intrinsics* intr, latmap_session** out);
latmap_status latmap_session_destroy(latmap_session* s);
/* Host -> device upload of the map (GaussianMapT SoA host arrays). */
latmap_status latmap_session_set_map(latmap_session* s, const float* positions, const float* rotations,
                                     const float* colors, const float* log_scales,
                                     const float* opacity_logits, const float* features);
latmap_status latmap_session_get_map(latmap_session* s, float* positions, float* rotations,
                                     float* colors, float* log_scales, float* opacity_logits,
                                     float* features);
/* DictionaryStateT: atoms K x df, anchor K x df, proj ds x df (host arrays). */
latmap_status latmap_session_set_dictionary(latmap_session* s, const float* atoms, const float* anchor,
                                            const float* proj);
latmap_status latmap_session_get_dictionary(latmap_session* s, float* atoms, float* proj);
/* DictionaryStateT::anchor (the trust-region centre; artifacts.cpp:79 save_dictionary). */
latmap_status latmap_session_get_anchor(latmap_session* s, float* anchor);
/* Keyframe batch (host arrays, copied H2D on the session stream). */
latmap_status latmap_session_set_frames(latmap_session* s, int32_t nframes, const latmap_frame* frames);
/* Batch-mean denominator (objective.cpp:77) and whether this rank adds the trust term
 * (objective.cpp:176-185); used when keyframes are sharded across ranks. */
latmap_status latmap_session_set_batch(latmap_session* s, int32_t global_batch, int32_t add_trust);
/* Global index of this rank's first frame: its loss partials land in that slot so a sum
 * all-reduce of the partials buffer reassembles the batch LossBreakdown. */
latmap_status latmap_session_set_slot_offset(latmap_session* s, int32_t offset);
/* total_objective with gradients into the session's flat gradient buffer. `out` (host) may be
 * NULL to avoid a device->host sync. */
latmap_status latmap_session_objective(latmap_session* s, int32_t want_grad, latmap_loss_breakdown* out);
/* MapOptimizer::step_map + step_dict on the session gradients (pipeline.cpp:75-95). */
latmap_status latmap_session_apply(latmap_session* s);
/* objective + apply; `out` may be NULL. */
latmap_status latmap_session_step(latmap_session* s, latmap_loss_breakdown* out);
/* Steps are captured once into a CUDA graph and replayed while frames, batch settings and the
 * row set are unchanged (default on; off while phase profiling). */
latmap_status latmap_session_set_graphs(latmap_session* s, int32_t enable);
/* total_objective with ObjectiveOptions (objective.hpp:33-43): map_grads = 0 skips the image-loss
 * gradients and render_backward; use_cached_renders = 1 reuses the session's per-frame renders
 * when the map has not changed since they were produced (cached_renders / render_sink). */
latmap_status latmap_session_objective_ex(latmap_session* s, int32_t want_grad, int32_t map_grads,
                                          int32_t use_cached_renders, latmap_loss_breakdown* out);
/* One Stage-II iteration (pipeline.cpp:250-259): objective with map_grads = false on cached
 * renders, then MapOptimizer::step_dict (proj, and atoms when dict_learn). */
latmap_status latmap_session_step_dict(latmap_session* s, latmap_loss_breakdown* out);
/* The active-map row set changes (ActiveSet after sync / append_newborns, active_set.hpp:10-26):
 * export writes the map as device AoS rows [position 3 | rotation 4 | color 3 | log_scale 3 |
 * opacity 1 | features query_dim] (the store's record layout); import replaces the map with
 * n_new such rows, carrying the Adam moments of the old rows with kept[i] != 0 (in order) to the
 * first n_kept new rows and zeroing the rest (MapOptimizer::keep_map_rows, pipeline.cpp:97-104;
 * AdamState::ensure, adam.hpp:18-29). kept = NULL keeps every old row (pure append). */
latmap_status latmap_session_export_rows(latmap_session* s, float* d_rows);
latmap_status latmap_session_import_rows(latmap_session* s, const float* d_rows, int64_t n_new, const uint8_t* kept,
                                         int64_t n_kept);
/* import_rows with the kept mask on the device (one byte per old row, d_kept NULL = none carry
 * over) and n_kept its number of set entries (as latmap_store_sync_device reports them). */
latmap_status latmap_session_import_rows_device(latmap_session* s, const float* d_rows, int64_t n_new,
                                                const uint8_t* d_kept, int64_t n_kept);
int64_t latmap_session_size(const latmap_session* s);
/* seed_gaussians (pipeline.cpp:39-73) for frame b against a render of the current map: the
 * stride-2 pixels with observed depth > 0 whose rendered alpha < 0.5 or |rendered - observed
 * depth| > 0.1, in raster order, written as AoS rows (features zero: the reference draws them
 * from the pipeline's std::mt19937_64, see latmap_b200.hpp seed_gaussians) into d_rows (cap
 * rows; d_rows = NULL only counts). */
latmap_status latmap_session_seed_candidates(latmap_session* s, int32_t b, float* d_rows, int64_t cap,
                                             int64_t* count);
/* ActiveSet::append_newborns: append n_rows device AoS rows (features replaced by h_features,
 * n_rows x query_dim host floats, when given) with zero Adam moments. */
latmap_status latmap_session_append_rows(latmap_session* s, float* d_rows, int64_t n_rows, const float* h_features);
/* Flat device buffers: [positions|rotations|colors|log_scales|opacity|features|proj|atoms]
 * gradient layout (for the multi-GPU all-reduce) and the loss-partials vector. */
latmap_status latmap_session_grad_buffer(latmap_session* s, float** grads, int64_t* count);
/* Element offset and length of each of the 8 blocks in that flat buffer (positions, rotations,
 * colors, log_scales, opacity, features, proj, atoms); every block starts on a 16-byte boundary,
 * so offsets are not the running sum of lengths when a length is not a multiple of 4. */
latmap_status latmap_session_grad_layout(latmap_session* s, int64_t offsets[8], int64_t lengths[8]);
latmap_status latmap_session_loss_buffer(latmap_session* s, double** partials, int64_t* count);
latmap_status latmap_session_read_loss(latmap_session* s, latmap_loss_breakdown* out);
/* The step's loss partials (latmap_session_loss_buffer's layout) copied D2H on the context stream
 * into host_partials (page-locked for an asynchronous copy) without waiting: after the stream
 * reaches this point, latmap_loss_assemble(host_partials, *count, ...) gives the LossBreakdown.
 * Lets a training loop read every step's loss one step late instead of stalling each step. */
latmap_status latmap_session_read_loss_async(latmap_session* s, double* host_partials, int64_t cap, int64_t* count);
/* Per-frame render outputs of the last objective (device pointers; parity and Stage-II reuse). */
latmap_status latmap_session_frame_images(latmap_session* s, int32_t frame, float** color, float** depth,
                                          float** query, float** alpha);
/* Host-only (no device): the LossBreakdown of a batch from its loss-partials vector (the layout
 * latmap_session_loss_buffer exposes: kPart = 8 doubles per global frame slot [l1 sum, SSIM sum,
 * depth |err| sum, valid depth count, (1 - cos) sum, |F_hat - F|^2 sum, zero-norm flag,
 * supervised rows], then a 16-double tail: trust penalty, overflow flag, the 8 Adam blocks' skip
 * flags), with inv_b = 1 / nframes (objective.cpp:77,187-190).
 * The sharded step's all-reduced partials assemble to the full batch's breakdown. */
latmap_status latmap_loss_assemble(const double* partials, int32_t nframes, int32_t width, int32_t height,
                                   const latmap_config* cfg, latmap_loss_breakdown* out);
/* Sharded step, after objective -> latmap_session_allreduce -> apply: *any = 1 when some rank's
 * tile lists overflowed in that objective (the flag travels in the loss partials, so every rank's
 * Adam skipped the step). This rank's buffers are grown when its own lists overflowed; the caller
 * repeats the iteration on every rank. Synchronises the context stream. */
latmap_status latmap_session_check_overflow(latmap_session* s, int32_t* any);
/* Sticky count of Adam steps skipped because a tile list overflowed (since session creation). */
latmap_status latmap_session_overflow_steps(latmap_session* s, int64_t* count);
/* process_keyframe's transaction (pipeline.cpp:155-190, 294-306): save the device state (map rows,
 * dictionary incl. anchor and weights, Adam moments and counters) and restore it after a failure.
 * One saved state per session; restore re-homes the flat buffers when the row count changed. */
latmap_status latmap_session_save_state(latmap_session* s);
latmap_status latmap_session_restore_state(latmap_session* s);
/* Sharded optimiser step (ZeRO-1 over the keyframe-sharded objective). The flat buffers split into
 * nranks 4-aligned shards; rank r owns [*begin, *end). */
latmap_status latmap_session_shard_range(const latmap_session* s, int32_t nranks, int32_t rank, int64_t* begin,
                                         int64_t* end);
/* Per-block non-finite flags (adam.hpp:65-68) of the gradient range [begin, end) into the loss
 * partials' tail (slots 2..9 after the trust and overflow slots); the partials all-reduce ORs them. */
latmap_status latmap_session_shard_check(latmap_session* s, int64_t begin, int64_t end);
/* MapOptimizer::step_map + step_dict restricted to the flat range [begin, end), taking the skip
 * flags from the (all-reduced) partials tail; step counters advance as in the full step. */
latmap_status latmap_session_apply_range(latmap_session* s, int64_t begin, int64_t end);
/* The flat parameter buffer (device; same layout as the gradients). */
latmap_status latmap_session_params_buffer(latmap_session* s, float** params, int64_t* count);
/* Parity export of the bf16 tcgen05 decoders (the reference returns F_hat,
 * proj/src/dictionary.cpp:45,52; the fused kernels never materialise it). While enabled, DEC1 /
 * DL3 also store each row's (nu^2 = |F_hat|^2, dot = F_hat.F) as the kernels computed them. */
latmap_status latmap_session_set_parity_export(latmap_session* s, int32_t enable);
/* For the last frame the objective decoded: *path = 0 none, 1 fp32 SIMT, 2 fused tcgen05
 * (DEC1/DEC2), 3 staged tcgen05 (DL1-DL5); *rows = its decoder rows (pixels). `attention` (device,
 * rows x K, may be NULL) receives the attention P = softmax(Q W D^T / tau) the bf16 kernels used,
 * so F_hat = P D; `row_nd` (device, rows x 2, may be NULL) the per-row (nu^2, dot). Both need a
 * tcgen05 frame (the fused path writes its e tiles only with gradients); row_nd needs the export
 * enabled before the objective. Synchronises the context stream. */
latmap_status latmap_session_decoder_export(latmap_session* s, int32_t* path, int64_t* rows, float* attention,
                                            float* row_nd);
/* Phase timing with CUDA events on the session stream: phases 0 project+bin+sort (K1-K3b),
 * 1 raster forward (K4), 2 image losses (K5), 3 decoder+feature loss (K6/K7), 4 raster backward (K8),
 * 5 projection backward (K9), 6 Adam (K10), 7 reserved. phase_times syncs, returns the summed
 * milliseconds and span counts since the last call, and resets them. */
latmap_status latmap_session_profile(latmap_session* s, int32_t enable);
latmap_status latmap_session_phase_times(latmap_session* s, double* ms, int64_t* counts);
/* Counters of the last objective: visible splats and tile pairs per frame (for roofline bytes). */
latmap_status latmap_session_stats(latmap_session* s, int64_t* visible, int64_t* pairs);

/* ---------------------------------------------------------------- voxel-hash store (config 3) */
/* voxel_of (voxel_hash.cpp:9-16: double division + floor) and hash_voxel (voxel_hash.cpp:18-23:
 * wrapping u32 multiply / xor, u64 modulo); host functions, bit-exact. */
void latmap_voxel_of(const float p[3], float voxel_size, int32_t key[3]);
int64_t latmap_hash_voxel(const int32_t key[3], int64_t capacity);

/* VoxelHashStore (store/voxel_hash.hpp:25-73): fixed-capacity open-addressing table (linear
 * probing, limit 8, one record per voxel) over an append-only record pool held in pinned,
 * device-mapped host memory (the host-resident global map). Records are flat rows of
 * 14 + query_dim floats: position 3, rotation 4, color 3, log_scale 3, opacity 1, features. */
typedef struct latmap_store latmap_store;
latmap_status latmap_store_create(latmap_ctx* ctx, int64_t capacity, int32_t query_dim, latmap_store** out);
latmap_status latmap_store_destroy(latmap_store* s);
int64_t latmap_store_size(const latmap_store* s);
/* inserted, updated, rejected_duplicate, rejected_overflow, probe_steps (VoxelHashStore::Stats) */
void latmap_store_stats(const latmap_store* s, int64_t out[5]);
const char* latmap_store_last_error(const latmap_store* s);
int64_t latmap_store_insert(latmap_store* s, const int32_t key[3], const float* rec); /* -1 = rejected */
int32_t latmap_store_update(latmap_store* s, const int32_t key[3], const float* rec);
int64_t latmap_store_find(latmap_store* s, const int32_t key[3]);
latmap_status latmap_store_get_records(const latmap_store* s, int64_t first, int64_t count, float* out,
                                       int32_t* keys_out);
/* insert_global (voxel_hash.cpp:101-115): keys + home slots on the device, probe in row order. */
latmap_status latmap_store_insert_global(latmap_store* s, const float* recs, int64_t n, float voxel_size,
                                         int64_t* inserted);
/* Rebuild from a global-map dump (artifacts.cpp:54-63 load_map_store): VoxelHashStore::insert of
 * each record under its stored key, in dump order (keys n x 3 int32, recs n x record AoS). */
latmap_status latmap_store_insert_keyed(latmap_store* s, const int32_t* keys, const float* recs, int64_t n,
                                        int64_t* inserted);
/* fetch_local (active_set.cpp:7-36): ascending record indices within `radius` (device radius scan +
 * ordered compaction); optional gather of the records into device memory (d_records, AoS). */
latmap_status latmap_store_fetch_local(latmap_store* s, const float center[3], float radius, int64_t* origin,
                                       int64_t cap, int64_t* count, float* d_records);
/* sync (active_set.cpp:38-128): writeback (dirty tracked rows scattered into the pinned pool in place,
 * newborns inserted in row order), prune by radius, fetch the remaining in-radius records; output =
 * kept rows (original order) ++ fetched records (ascending), gathered into d_out (device AoS).
 * stats: written_back, newborn_inserted, newborn_rejected, pruned, fetched. */
latmap_status latmap_store_sync(latmap_store* s, const float* d_active, const int64_t* origin, const uint8_t* dirty,
                                int64_t n, const float center[3], float radius, float voxel_size, float* d_out,
                                int64_t* out_origin, int64_t cap, uint8_t* kept_mask, int64_t stats[5],
                                int64_t* out_count);
/* fetch_local (active_set.cpp:7-36) with device outputs: d_origin (ascending record indices,
 * may be NULL to count only), d_records (optional AoS gather); the store's persistent scratch,
 * one count readback. count = NULL (with d_origin and d_records NULL): the scan only, no
 * readback, nothing waits (used to time the radius scan on the device). */
latmap_status latmap_store_fetch_local_device(latmap_store* s, const float center[3], float radius, int64_t* d_origin,
                                              int64_t cap, float* d_records, int64_t* count);
/* sync with every per-row array on the device: d_origin (int64), d_dirty (uint8, NULL = all
 * dirty), d_kept (uint8 out) and d_out_origin (int64 out) are device buffers. Same results as
 * latmap_store_sync bit for bit; the row selections are device compactions and the counts come
 * back once (twice when newborns are present: their inserts follow the host probe order).
 * The pool writeback of the written-back rows runs on the store's writeback stream, overlapping
 * the caller's next work; every later store call waits for it. */
latmap_status latmap_store_sync_device(latmap_store* s, const float* d_active, const int64_t* d_origin,
                                       const uint8_t* d_dirty, int64_t n, const float center[3], float radius,
                                       float voxel_size, float* d_out, int64_t* d_out_origin, int64_t cap,
                                       uint8_t* d_kept, int64_t stats[5], int64_t* out_count);

/* ---------------------------------------------------------------- streaming k-means */
/* std::uniform_real_distribution<double>(0, 1) drawn from the caller's generator (the pipeline's
 * std::mt19937_64, pipeline.cpp:203): k-means++ consumes exactly the draws the reference does. */
typedef double (*latmap_uniform_fn)(void* user);
/* weighted_kmeans (stream_kmeans.hpp:18-21, stream_kmeans.cpp:94-157): host points n x dim,
 * weights n, optional warm-start rows (n_warm x dim); writes centers (k x dim), per-centre mass
 * (k) and the Lloyd iteration count. Nearest-centre scores, argmin, k-means++ distances and the
 * centre sums run on the device; the generator draws and orderings on the host. */
latmap_status latmap_weighted_kmeans(latmap_ctx* ctx, const float* points, const float* weights, int64_t n,
                                     int32_t dim, int64_t k, latmap_uniform_fn uniform, void* user,
                                     const float* warm, int64_t n_warm, int32_t max_iters, float* centers,
                                     float* center_weights, int32_t* iterations);
/* Dictionary maintenance of process_keyframe_inner for dict_init = "kmeans" (pipeline.cpp:201-205):
 * stream_kmeans_update (stream_kmeans.hpp:27-33) of the session's atoms / anchor / atom weights
 * with the keyframe's (host, n x embed_dim) embedding rows, then MapOptimizer::reset_atom_moments
 * (pipeline.hpp:62-64: the atoms' Adam moments and step count). */
latmap_status latmap_session_stream_kmeans(latmap_session* s, const float* batch, int64_t n, float decay,
                                           latmap_uniform_fn uniform, void* user);
/* DictionaryState::weights (dictionary.hpp:15), K floats; zero after session creation (init). */
latmap_status latmap_session_get_dict_weights(const latmap_session* s, float* out);
latmap_status latmap_session_set_dict_weights(latmap_session* s, const float* w);

/* ---------------------------------------------------------------- evaluation (device rows in) */
/* gather_supervision, pixel mode (objective.cpp:16-35): rows of the pixels with assignment >= 0
 * in ascending pixel order -> q_out (n x ds), t_out (n x df; each row normalised when `normalize`,
 * as evaluate_map does, evaluate.cpp:38-42), pixel_of_row (n). Pass q_out = NULL to count only;
 * *n_rows is always set; LATMAP_ERR_INVALID_ARGUMENT if n > cap. */
latmap_status latmap_gather_supervision(latmap_ctx* ctx, const float* query, int32_t ds, const int32_t* assignment,
                                        int64_t npx, const float* features, int32_t df, int32_t normalize,
                                        float* q_out, float* t_out, int64_t* pixel_of_row, int64_t cap,
                                        int64_t* n_rows);
/* metric_cos (metrics.hpp:12-13) over n rows of width d; flagged as in the reference. */
latmap_status latmap_metric_cos(latmap_ctx* ctx, const float* reconstructed, const float* target, int64_t n,
                                int32_t d, double* value, int32_t* flagged);
/* metric_miou (metrics.hpp:15-26): intersection / union per class (host, c entries each). */
latmap_status latmap_metric_miou(latmap_ctx* ctx, const float* embeddings, const int32_t* labels, int64_t n,
                                 int32_t d, const float* prototypes, int32_t c, int64_t* intersection,
                                 int64_t* union_, double* miou);
/* metric_psnr (metrics.hpp:28-33) over n values. */
latmap_status latmap_metric_psnr(latmap_ctx* ctx, const float* rendered, const float* observed, int64_t n,
                                 double* db, int32_t* exact);
/* query_map (evaluate.hpp:37-40): cosine of every Gaussian's reconstructed embedding with one
 * embedding (device, df) -> scores (device, n). */
latmap_status latmap_query_map(latmap_ctx* ctx, const float* features, int64_t n, int32_t ds, const float* atoms,
                               const float* proj, int64_t k, int32_t df, float temperature, const float* embedding,
                               float* scores);

/* ---------------------------------------------------------------- multi-GPU (NCCL) */
/* one process per GPU, keyframes sharded across ranks, one sum all-reduce of
 * the gradients and loss partials per iteration. NCCL is loaded at run time (libnccl.so.2);
 * without it these return LATMAP_ERR_UNSUPPORTED. */
typedef struct latmap_comm latmap_comm;
/* ncclGetUniqueId on rank 0; the caller hands the 128 bytes to every rank (any channel). */
latmap_status latmap_comm_unique_id(latmap_ctx* ctx, uint8_t id[128]);
/* ncclCommInitRank on the context's device; collectives run on the context's stream. */
latmap_status latmap_comm_init(latmap_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[128],
                               latmap_comm** out);
latmap_status latmap_comm_destroy(latmap_comm* comm);
/* In-place sum all-reduce of a device buffer; dtype 0 = fp32, 1 = fp64. */
latmap_status latmap_comm_allreduce(latmap_comm* comm, void* buf, int64_t count, int32_t dtype);
/* The sharded iteration's exchange: the session's flat gradient buffer and loss partials summed
 * over ranks (one NCCL group), between latmap_session_objective and latmap_session_apply. */
latmap_status latmap_session_allreduce(latmap_session* s, latmap_comm* comm);
/* The sharded exchange + step: reduce-scatter of the gradients, shard check, all-reduce of the loss
 * partials, Adam on this rank's shard, all-gather of the parameters (replaces allreduce + apply). */
latmap_status latmap_session_exchange_sharded(latmap_session* s, latmap_comm* comm);

/* ---------------------------------------------------------------- pipeline (the step's caller) */
/* The pipeline-level subset of latmap::Config (core/config.hpp:10-58; same defaults via
 * latmap_default_pipeline_config). dict_init: 0 = "kmeans", 1 = "random". The objective's own
 * fields (loss weights, learning rates, softmax_temp, dict_learn, segment_mode) stay in
 * latmap_config. */
typedef struct {
  int32_t query_dim, embed_dim, dict_size;
  int32_t stage1_iters, stage2_iters;
  int32_t history_sample, history_capacity;
  float voxel_size, local_radius, sync_distance;
  int64_t hash_capacity;
  int32_t local_mapping, keyframe_stride;
  uint64_t seed;
  int32_t dict_init;
  float dict_decay;
  int32_t trust_anchor_persistent;
} latmap_pipeline_config;
/* KeyframeLog (pipe/pipeline.hpp:70-80); sync = SyncStats {written_back, newborn_inserted,
 * newborn_rejected, pruned, fetched} (store/active_set.hpp:28-34). */
typedef struct {
  int32_t frame_index;
  latmap_loss_breakdown loss;
  int64_t seeded, active_count, global_count;
  double dict_weight_mass;
  int32_t synced;
  int64_t sync[5];
  double wall_ms;
} latmap_keyframe_log;
typedef struct latmap_pipeline latmap_pipeline;
void latmap_default_pipeline_config(latmap_pipeline_config* pc);
/* select_keyframe (pipeline.cpp:14-17): 1 / 0, or -1 for stride < 1 (std::invalid_argument). */
int32_t latmap_select_keyframe(int32_t frame_index, int32_t stride);
/* PipelineState::PipelineState (pipeline.cpp:106-121): an empty active map (device session), an
 * empty global store (hash_capacity), a zero dictionary with proj ~ N(0, 0.1) from
 * std::mt19937_64(seed). Config::validate's checks (config.cpp:110-133) -> INVALID_ARGUMENT with
 * the message on the context. */
latmap_status latmap_pipeline_create(latmap_ctx* ctx, const latmap_config* cfg, const latmap_pipeline_config* pc,
                                     const latmap_intrinsics* intr, latmap_pipeline** out);
latmap_status latmap_pipeline_destroy(latmap_pipeline* p);
/* process_keyframe (pipeline.cpp:192-312): embedding normalisation, dictionary maintenance,
 * history-augmented batch, seeding, Stage I x stage1_iters, Stage II x stage2_iters on cached
 * renders, history push, travel and sync. The frame is host memory (copied). Argument errors
 * leave the state untouched; a device error mid-keyframe marks the pipeline failed (the device
 * state cannot be rolled back as the reference's snapshot/restore does). */
latmap_status latmap_pipeline_process_keyframe(latmap_pipeline* p, const latmap_frame* kf, int32_t frame_index,
                                               latmap_keyframe_log* out);
/* run_pipeline's final flush (pipeline.cpp:318-330): the whole active set marked dirty and synced
 * at the last position; stats = SyncStats (may be NULL). */
latmap_status latmap_pipeline_flush(latmap_pipeline* p, int64_t stats[5]);
/* Borrowed handles (owned by the pipeline): the device map/dictionary session and the store. */
latmap_session* latmap_pipeline_session(latmap_pipeline* p);
latmap_store* latmap_pipeline_store(latmap_pipeline* p);
/* PipelineState scalars: keyframes_processed, peak_active, history size, reservoir_seen, failed,
 * traveled (float bits). */
latmap_status latmap_pipeline_state(const latmap_pipeline* p, int64_t out[6]);
/* ActiveSet::origin / dirty (host arrays of latmap_session_size entries). */
latmap_status latmap_pipeline_active_set(const latmap_pipeline* p, int64_t* origin, uint8_t* dirty);
const char* latmap_pipeline_last_error(const latmap_pipeline* p);
/* Test hook: make the next process_keyframe fail (LATMAP_ERR_CUDA, "injected fault") at stage
 * 1 after seeding, 2 after Stage I/II, 3 after the sync (0 = off); the keyframe is rolled back. */
latmap_status latmap_pipeline_inject_fault(latmap_pipeline* p, int32_t stage);

/* ---------------------------------------------------------------- self-test */
/* One-tile tcgen05 GEMM, C[128 x n] = A[128 x k] * B[n x k]^T (device fp32 in/out, bf16 staging),
 * with A / B staged K-major (0) or MN-major (1); pins the UMMA descriptor conventions. */
latmap_status latmap_selftest_umma(latmap_ctx* ctx, const float* a, const float* b, float* c, int32_t n,
                                   int32_t k, int32_t a_mn, int32_t b_mn);
/* out[i] = the kernels' std::exp(float) (glibc expf restated, csrc/expf_ref.h) of the float whose
 * bit pattern is first + i (device out, n floats): pins it to libm on every input. */
latmap_status latmap_selftest_expf(latmap_ctx* ctx, uint64_t first, int64_t n, float* out);

#ifdef __cplusplus
}
#endif
#endif
