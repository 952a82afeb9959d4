/*
 * latmap_oracle.h — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement ("port") of the reference LatentAM hot path
 * (/root/reference/proj, C++/Eigen), used ONLY as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg. The product
 * path (paper_2602_12314_b200, liblatmap_b200.so) never links or calls it.
 *
 * Parity pin: the reference cannot be built here (Eigen3 + doctest absent, see
 * DESIGN.md §Oracle), so this restatement is pinned against every known-answer
 * test, brute-force oracle and finite-difference check the reference's own
 * suites hold for the path (tests/test_oracle_*.py cite each one).
 *
 * Arithmetic conventions (they DEFINE the oracle's float bits; the CUDA exact
 * paths mirror them op for op):
 *   - no FMA contraction (-ffp-contract=off; x86-64 baseline has no FMA);
 *   - float exp is (float)exp((double)x) (reference: std::exp on float);
 *   - fixed-size Eigen products are summed left to right over the inner index;
 *   - dynamic GEMMs accumulate over the inner index in ascending order;
 *   - reductions (norm, dot, sum) are sequential in index order.
 *
 * Every entry point exists twice: *_f32 (T=float) and *_f64 (T=double),
 * mirroring the reference's explicit instantiations (render.cpp:434-447 etc.).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
} lm_intr; /* Intrinsics, types.hpp:41-50 */

typedef struct {
  int32_t ix, iy, iz;
} lm_voxel_key; /* VoxelKey, voxel_hash.hpp:10-13 */

#define LM_DECLARE(T, S)                                                                        \
  typedef struct {                                                                              \
    int64_t n;                                                                                  \
    int32_t ds;                                                                                 \
    T *pos, *rot, *col, *lsc, *opa, *feat; /* GaussianMapT SoA, types.hpp:93-199 */             \
  } lm_map##S;                                                                                  \
  typedef struct {                                                                              \
    T rot[4];                                                                                   \
    T trans[3]; /* PoseT (w,x,y,z), camera-to-world, types.hpp:27-38 */                         \
  } lm_pose##S;                                                                                 \
  typedef struct {                                                                              \
    T mean[2];                                                                                  \
    T cov_inv[4];                                                                               \
    T depth, alpha;                                                                             \
    int32_t source, x0, x1, y0, y1; /* ProjectedSplat, render.hpp:31-39 */                      \
  } lm_splat##S;                                                                                \
  typedef struct {                                                                              \
    T l_rgb, l_ssim, l_depth, l_cos, l_l2, l_trust, total;                                      \
    int64_t supervised_rows;                                                                    \
    int32_t depth_empty, zero_norm_flagged; /* LossBreakdown, objective.hpp:12-24 */            \
  } lm_loss##S;                                                                                 \
  typedef struct {                                                                              \
    lm_pose##S pose;                                                                            \
    const T* rgb;               /* H x W x 3 */                                                 \
    const T* depth;             /* H x W     */                                                 \
    const int32_t* assignment;  /* H x W, -1 = unsupervised */                                  \
    const T* features;          /* n_set x d_f */                                               \
    int64_t n_set;              /* KeyframeT/EmbeddingSetT, types.hpp:204-248 */                \
  } lm_frame##S;                                                                                \
  typedef struct {                                                                              \
    int32_t segment_mode, dict_grads, map_grads;                                                \
    T lambda_cos, lambda_l2, lambda_trust, trust_delta;                                         \
    T lambda_i1, lambda_i2, lambda_rgb, lambda_depth, lambda_feat;                              \
    T lr_proj, lr_dict, lr_position, lr_rotation, lr_color, lr_log_scale, lr_opacity,           \
        lr_feature, scene_extent;                                                               \
    int32_t dict_learn; /* Config subset, config.hpp:10-71 */                                   \
  } lm_cfg##S;                                                                                  \
  int lm_quat_to_rot##S(const T q[4], T r[9]);                                                  \
  int lm_project_gaussian##S(const T pos[3], const T rot[4], const T lsc[3], T opa,             \
                             const lm_pose##S* pose, const lm_intr* intr, T mean2d[2],          \
                             T cov2d[4], T* depth);                                             \
  int lm_render##S(const lm_map##S* map, const lm_pose##S* pose, const lm_intr* intr,          \
                   int threads, T* color, T* depth, T* query, T* alpha, lm_splat##S* splats,    \
                   int64_t cap, int64_t* n_splats);                                             \
  int lm_render_backward##S(const lm_map##S* map, const lm_pose##S* pose, const lm_intr* intr,  \
                            const lm_splat##S* splats, int64_t n_splats, const T* d_color,      \
                            const T* d_depth, const T* d_query, int threads, lm_map##S* grads); \
  T lm_ssim##S(const T* a, const T* b, int h, int w, int c, T* d_a);                            \
  int lm_rgb_loss##S(const T* rendered, const T* observed, int h, int w, int c, T lambda_i1,    \
                     T lambda_i2, int want_grad, T* grad, T* l1, T* ssim_loss, T* value);       \
  int lm_depth_loss##S(const T* rendered, const T* observed, const T* alpha, int64_t n,         \
                       int want_grad, T* grad, T* value, int32_t* flagged);                     \
  T lm_trust_region_penalty##S(const T* atoms, const T* anchor, int64_t k, int64_t df, T delta, \
                               T* d_atoms);                                                     \
  int lm_feature_loss##S(const T* rec, const T* tgt, int64_t n, int64_t df, const T* atoms,     \
                         const T* anchor, int64_t k, T delta, T lambda_cos, T lambda_l2,        \
                         T lambda_trust, int want_grad, T* d_rec, T* d_atoms_trust,             \
                         T* cos_term, T* l2_term, T* trust_term, T* value, int32_t* zflag);     \
  double lm_dictionary_checksum##S(const T* atoms, int64_t k, int64_t df, const T* proj,        \
                                   int64_t ds);                                                 \
  int lm_reconstruct##S(const T* q, int64_t n, int64_t ds, const T* atoms, int64_t k,           \
                        int64_t df, const T* proj, T temperature, T* out, T* attention);        \
  int lm_reconstruct_backward##S(const T* q, const T* attention, int64_t n, int64_t ds,         \
                                 const T* atoms, int64_t k, int64_t df, const T* proj,          \
                                 T temperature, const T* d_rec, T* d_q, T* d_proj, T* d_atoms); \
  int64_t lm_gather_supervision##S(const T* query, int h, int w, int ds,                        \
                                   const int32_t* assignment, const T* features, int64_t n_set, \
                                   int64_t df, int segment_mode, T* q_out, T* t_out,            \
                                   int64_t* pixel_of_row);                                      \
  int lm_total_objective##S(const lm_map##S* map, const T* atoms, const T* anchor,              \
                            const T* proj, int64_t k, int64_t df, T temperature,                \
                            const lm_frame##S* frames, int nframes, const lm_intr* intr,        \
                            const lm_cfg##S* cfg, int threads, int want_grad,                   \
                            lm_map##S* map_grads, T* d_proj, T* d_atoms, lm_loss##S* out);      \
  int lm_adam_step##S(T* param, const T* grad, T* m, T* v, int64_t count, int64_t* step,        \
                      int64_t* skipped, T lr);                                                  \
  void lm_renorm_quats##S(T* rot, int64_t n);                                                   \
  /* weighted_kmeans / stream_kmeans_update (stream_kmeans.cpp:94-196); uni draws */            \
  /* std::uniform_real_distribution<double>(0, 1) from the caller's generator */                \
  int lm_weighted_kmeans##S(const T* points, const T* weights, int64_t n, int64_t dim,          \
                            int64_t k, double (*uni)(void*), void* rng, const T* warm,          \
                            int64_t n_warm, int max_iters, T* centers, T* cweights,             \
                            int* iterations);                                                   \
  int lm_stream_kmeans_update##S(const T* batch, int64_t n, int64_t dim, T* atoms, T* anchor,   \
                                 T* weights, int64_t k, double (*uni)(void*), void* rng,        \
                                 T decay);

LM_DECLARE(float, _f32)
LM_DECLARE(double, _f64)

/* ---- std::mt19937_64 and std::uniform_real_distribution<double>(0, 1) (libstdc++
 * generate_canonical), the generator the reference pipeline threads through k-means++
 * (stream_kmeans.cpp:58) and seeding (pipeline.cpp:46) ---- */
typedef struct {
  uint64_t mt[312];
  int32_t idx;
} lm_mt64;
void lm_mt64_seed(lm_mt64* r, uint64_t seed);
uint64_t lm_mt64_next(lm_mt64* r);
double lm_mt64_uniform01(void* r);

/* Threads for the dense products (row-split; bit-identical for every count). Default 1, like
 * the reference's single-threaded Eigen (proj/CMakeLists.txt:11 links no OpenMP). */
void lm_oracle_set_gemm_threads(int n);
/* libm expf of the floats with bit patterns first .. first + n - 1 (threads split the range). */
void lm_expf_bits(uint64_t first, int64_t n, float* out, int threads);

/* ---- evaluation metrics (float, metrics.cpp:8-89, evaluate.cpp:74-88) ---- */
double lm_metric_cos(const float* rec, const float* tgt, int64_t n, int64_t d, int32_t* flagged);
/* intersection / union_ per class (c entries each); returns mIoU; -1 on a label >= c */
double lm_metric_miou(const float* emb, const int32_t* labels, int64_t n, int64_t d, const float* protos,
                      int64_t c, int64_t* inter, int64_t* uni);
double lm_metric_psnr(const float* a, const float* b, int64_t n, int32_t* exact);
/* query_map scores from reconstructed rows (n x d) against one embedding */
void lm_query_scores(const float* rec, int64_t n, int64_t d, const float* embedding, float* scores);

/* ---- voxel hash store (float only, voxel_hash.hpp / active_set.hpp) ---- */
lm_voxel_key lm_voxel_of(const float p[3], float voxel_size);
int64_t lm_hash_voxel(lm_voxel_key k, int64_t capacity);

typedef struct lm_store lm_store; /* VoxelHashStore */
lm_store* lm_store_create(int64_t capacity, int32_t query_dim);
void lm_store_destroy(lm_store* s);
int64_t lm_store_insert(lm_store* s, lm_voxel_key key, const float* rec);
int32_t lm_store_update(lm_store* s, lm_voxel_key key, const float* rec);
int64_t lm_store_find(const lm_store* s, lm_voxel_key key);
int64_t lm_store_size(const lm_store* s);
int32_t lm_store_check_unique_keys(const lm_store* s);
/* record layout (flat, 14 + d_s floats): pos3 rot4 col3 lsc3 opa1 feat[d_s] */
void lm_store_get_record(const lm_store* s, int64_t index, float* rec);
void lm_store_set_record(lm_store* s, int64_t index, const float* rec);
lm_voxel_key lm_store_record_key(const lm_store* s, int64_t index);
void lm_store_stats(const lm_store* s, int64_t out[5]);
int64_t lm_insert_global(lm_store* s, const float* recs, int64_t n, float voxel_size);
/* fetch_local: returns count, writes record indices (ascending) into origin (cap entries). */
int64_t lm_fetch_local(const lm_store* s, const float center[3], float radius, int64_t* origin,
                       int64_t cap);
/* sync (active_set.cpp:38-128): active records (n x (14+ds)) + origin + dirty ->
 * out records/origin (cap), kept_mask (n); stats[5] = written_back, newborn_inserted,
 * newborn_rejected, pruned, fetched. Returns out count, -1 on capacity error. */
int64_t lm_sync(lm_store* s, const float* active, const int64_t* origin, const uint8_t* dirty,
                int64_t n, const float center[3], float radius, float voxel_size, float* out_recs,
                int64_t* out_origin, int64_t cap, uint8_t* kept_mask, int64_t stats[5]);

#ifdef __cplusplus
}
#endif
