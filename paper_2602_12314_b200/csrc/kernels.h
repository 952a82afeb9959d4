// kernels.h — host-side launchers of the latent-map step kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace lm {

struct Intr {
  float fx, fy, cx, cy;
  int32_t width, height;
};

struct MapPtrs {  // device SoA (GaussianMapT / MapGradientsT)
  int64_t n;
  int32_t ds;
  float *pos, *rot, *col, *lsc, *opa, *feat;
};

// Per-frame render workspace (RenderOutput::splats + the tile lists).
struct RenderWork {
  int64_t n_cap = 0;     // Gaussians the buffers are sized for
  int32_t tiles_x = 0, tiles_y = 0, width = 0, height = 0;
  int64_t pair_cap = 0;  // capacity of the (tile, depth) key arrays
  SplatRec* rec = nullptr;          // n_cap
  int32_t* tile_count = nullptr;    // ntiles
  int32_t* tile_offset = nullptr;   // ntiles + 1
  int32_t* tile_cursor = nullptr;   // ntiles
  uint64_t* keys = nullptr;         // pair_cap, (depth_bits << 32 | source), sorted per tile
  uint64_t* keys_tmp = nullptr;     // pair_cap, merge scratch for oversized tiles
  uint32_t* dkey = nullptr;         // n_cap: float bits of camera z (0xffffffff = culled)
  int32_t* px_last = nullptr;       // H*W: tile-list entries consumed by the pixel
  float* px_T = nullptr;            // H*W: transmittance after the last blended splat
  int64_t* counters = nullptr;      // [0] pairs, [1] visible, [2] overflow, [3] big tiles, [4] big footprints
  int32_t* big = nullptr;           // n_cap: Gaussians whose footprint K3 defers to K3c
  int32_t* tile_max_last = nullptr; // ntiles: max px_last over the tile
  int32_t* tile_order = nullptr;    // ntiles: blend dispatch order (longest lists first)
  int64_t* step_overflow = nullptr;  // optional session-level overflow flag
};

// Renderer: project (K1) -> scan (K2) -> scatter (K3) -> per-tile sort -> blend (K4).
void render_forward(cudaStream_t st, const MapPtrs& map, const float rot_cw[9], const float origin[3],
                    const Intr& intr, RenderWork& w, float* color, float* depth, float* query,
                    float* alpha, bool zero_outputs, bool count_only = false, bool blend = true,
                    bool exact = false);
// K4 only (after render_forward(..., blend=false)).
void render_blend(cudaStream_t st, const MapPtrs& map, const Intr& intr, RenderWork& w, float* color, float* depth,
                  float* query, float* alpha, bool exact = false);
void project_single(cudaStream_t st, const float* d_in11, const float rot_cw[9], const float origin[3],
                    const Intr& intr, float* d_out8);
// Deterministic backward scratch: per-splat pair counts / offsets and the per-(splat, tile)
// partial rows K8 writes instead of float atomics; reduced in a fixed order.
struct DetScratch {
  int64_t *cnt = nullptr, *off = nullptr, *blocks = nullptr;
  float* part = nullptr;
  int64_t n_cap = 0, part_cap = 0;
  cudaError_t ensure(int64_t n, int64_t pairs, int ds);
  void release();
};
// Backward: blend replay + reverse sweep (K8) -> projection backward (K9). Accumulates.
void render_backward(cudaStream_t st, const MapPtrs& map, const float rot_cw[9], const float rot_wc[9],
                     const float origin[3], const Intr& intr, const RenderWork& w, const float* d_color,
                     const float* d_depth, const float* d_query, float* geo_acc, const MapPtrs& grads,
                     bool project = true, DetScratch* det = nullptr);
// Deterministic reductions for the calling host thread (set by the C-ABI entry points from the
// context): gradient sums in a fixed order instead of float atomics (render backward, the
// decoders' partial reductions, segment pooling).
void set_deterministic(bool on);
bool deterministic();
// K9 only (after render_backward(..., project=false)).
void render_project_backward(cudaStream_t st, const MapPtrs& map, const float rot_cw[9], const float rot_wc[9],
                             const float origin[3], const Intr& intr, const RenderWork& w, float* geo_acc,
                             const MapPtrs& grads);
// K9 over nf frames in one pass (frame order kept: the same gradient bits as nf K9 launches).
void render_project_backward_multi(cudaStream_t st, const MapPtrs& map, int nf, const float* const* rot_cw,
                                   const float* const* rot_wc, const float* const* origin, const Intr& intr,
                                   const RenderWork* const* w, float* const* geo_acc, const MapPtrs& grads);

// Image-space losses (K5). partials[...] are double accumulators (see capi.cu).
void image_losses(cudaStream_t st, const float* color, const float* depth, const float* alpha,
                  const float* rgb_t, const float* depth_t, int h, int w, float lambda_i1, float lambda_i2,
                  float rgb_scale, float depth_scale, bool want_grad, float* d_color, float* d_depth,
                  double* partials, float* ssim_scratch);
double ssim_host(cudaStream_t st, const float* a, const float* b, int h, int w, int c, float* d_a,
                 float* scratch);
size_t ssim_scratch_floats(int h, int w, int c);
// Standalone loss operators (losses.hpp:12-58): device images / rows in, host scalars out; the
// gradient pointers may be NULL. out = {value, l1, ssim_loss} / {value, cos, l2, trust}.
cudaError_t rgb_loss_dev(cudaStream_t st, const float* rendered, const float* observed, int h, int w, int ch,
                         float lambda_i1, float lambda_i2, float* grad, float out[3]);
cudaError_t depth_loss_dev(cudaStream_t st, const float* rendered, const float* observed, const float* alpha,
                           int64_t n, float* grad, float* value, int* flagged);
cudaError_t feature_loss_dev(cudaStream_t st, const float* rec, const float* tgt, int64_t n, int df,
                             const float* atoms, const float* anchor, int64_t k, float delta, float lambda_cos,
                             float lambda_l2, float lambda_trust, float* d_rec, float* d_atoms_trust, float out[4],
                             int* zero_norm_flagged);

// Generic SIMT SGEMM: C = alpha * op(A) * op(B) + beta * C, row-major; split-K via atomics when
// `split` > 1 (then beta must be applied by the caller beforehand, beta ignored).
void sgemm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, float alpha,
           const float* A, int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
           int split = 1);

// Decoder (factored algebra, fp32 SIMT path) — see decoder.cu.
struct DecoderWork {
  int64_t n_cap = 0, k = 0;
  int32_t ds = 0, df = 0;
  float *buf1 = nullptr, *buf2 = nullptr;  // n x K
  float *alpha_r = nullptr, *beta_r = nullptr;
  float *kd = nullptr;   // K x ds   (D W^T)
  float *mm = nullptr;   // K x K    (D D^T)
  float *gt = nullptr;   // n_set x K (E D^T)
  float *nv = nullptr;   // n_set
  float *r = nullptr;    // ds x K   (Q^T dS)
  float *a = nullptr;    // K x K    (P^T diag(alpha) P)
  float *bm = nullptr;   // n_set x K (Bm^T)
  int64_t nset_cap = 0;
  // tcgen05 path scratch (decoder_tc.cu)
  float* row_stats = nullptr;  // npx x 4: max S, 1/sum, alpha, beta
  float* r_part = nullptr;     // 2 x 148 x K x ds (fused path step sums, staged path per frame)
  float* a_part = nullptr;     // 8 frame slots x 148 groups x 2 halves x K x K/2
  float* bm_part = nullptr;    // 74 x K x 64
  double* loss_part = nullptr; // 148 x 4
  uint8_t* e_tiles = nullptr;  // ceil(npx/128) x 128 x K bf16 (DEC1 -> DEC2)
  uint8_t* tc_img = nullptr;   // bf16 core-matrix images of Kd (K x ds) then M (K x K): DEC1's operands, per step
  float* a_acc = nullptr;      // K x K: sum over the step's frames of P^T diag(alpha) P
  float* r_acc = nullptr;      // ds x K: sum over the step's frames of Q^T dS
  bool tc_pending = false;     // a_acc / r_acc hold contributions not yet applied
  int tc_frames = 0;           // fused-path frames whose A / R partials are summed in a_part / r_part
  cudaEvent_t ev_dq = nullptr; // optional: recorded right after DEC1 (d_query complete; DEC2 still to run)
  // staged large-K tcgen05 path scratch (decoder_dl.cu)
  uint8_t* dl_mt = nullptr;    // K x K bf16: M in the B-operand blocks of the T GEMM
  float* dl_t = nullptr;       // ntiles x 128 x K fp16: T = e M (aliases buf1)
  uint8_t* dl_ae = nullptr;    // ntiles x 128 x (K + NB) bf16: gram B operand (aliases buf2)
  float* dl_nu = nullptr;      // (K/256) x ntiles*128: partial e.T per 256-column unit
  float* dl_part = nullptr;    // gram partials
  // parity export (latmap_session_set_parity_export): per-row (nu^2 = |F_hat|^2, dot = F_hat.F)
  // as the bf16 kernels computed them, for the last decoded frame; the attention P of that frame
  // is recoverable from e_tiles and row_stats (decoder_export_attention).
  float* row_nd = nullptr;     // npx x 2
  int32_t last_path = 0;       // decoder of the last decoded frame: 0 none, 1 fp32 SIMT, 2 fused tc, 3 staged tc
  int64_t last_npx = 0;
};
void decoder_prepare(cudaStream_t st, DecoderWork& w, const float* atoms, const float* proj);
void decoder_tc_images(cudaStream_t st, DecoderWork& w);  // Kd / M -> tc_img (fused tcgen05 path)
// Fused feature loss + decoder backward for one frame (pixel mode). Accumulates into d_proj,
// d_atoms (scaled by lambda_feat * inv_b) and writes d_query (HxWxds, scaled likewise).
// nsup: device int64, the supervised-row count (inv_nsup = 1 / nsup, 0 without supervision).
void decoder_frame(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment,
                   int64_t npx, const float* feats, int64_t n_set, const int64_t* nsup, const float* atoms,
                   const float* proj, float temperature, float lambda_cos, float lambda_l2, float scale,
                   bool want_grad, float* d_query, float* d_proj, float* d_atoms, double* partials);
void decoder_target_norms(cudaStream_t st, const float* feats, int64_t n_set, int df, float* nv);
// G = E D^T (n_set x K) and |E| rows in one launch (falls back to sgemm + norms for df % 4 != 0).
void decoder_targets(cudaStream_t st, const float* feats, int64_t n_set, const float* atoms, int64_t k, int df,
                     float* gt, float* nv);
// d_atoms += Bm E with Bm^T stored n_set x K.
void decoder_bm_embed(cudaStream_t st, const float* bmt, const float* feats, int64_t n_set, int64_t k, int df,
                      float* d_atoms);
// tcgen05 / TMEM path (bf16 operands, fp32 accumulation) for K in {128, 256}, d_s = 32, n_set <= 64.
bool decoder_tc_supported(int64_t k, int ds, int64_t n_set);
// Standalone reconstruct on tcgen05 (bf16 operands, fp32 accumulation; decoder_dl.cu):
// out (n x df) = softmax(Q W D^T / temperature) D, for K in {256, ..., 1024}, ds in {32, 64},
// df a multiple of 256.
bool reconstruct_tc_supported(int64_t k, int ds, int df);
// Order-preserving compaction of a device byte mask: out_idx = ascending i with mask[i] != 0,
// *count (device) = their number; blocks: compact_blocks(n) int32 scratch (store.cu).
int64_t compact_blocks(int64_t n);
cudaError_t compact_mask(cudaStream_t st, const uint8_t* mask, int64_t n, int64_t* out_idx, int32_t* blocks,
                         int64_t* count);
cudaError_t reconstruct_tc(cudaStream_t st, const float* q, int64_t n, int ds, const float* atoms, const float* proj,
                           int64_t k, int df, float temperature, float* out);
void decoder_frame_tc(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment,
                      int64_t npx, const float* feats, int64_t n_set, const int64_t* nsup, const float* atoms,
                      const float* proj, float temperature, float lambda_cos, float lambda_l2, float scale,
                      bool want_grad, float* d_query, float* d_proj, float* d_atoms, double* partials);
// Staged tcgen05 path for large dictionaries (decoder_dl.cu): K in {256..1024} (multiple of 256),
// d_s in {32, 64}, n_set <= 256. Same outputs and accumulators as decoder_frame_tc.
bool decoder_dl_supported(int64_t k, int ds, int64_t n_set);
size_t decoder_dl_part_floats(int64_t k);
void decoder_dl_prepare(cudaStream_t st, DecoderWork& w);
void decoder_frame_dl(cudaStream_t st, DecoderWork& w, const float* query, const int32_t* assignment,
                      int64_t npx, const float* feats, int64_t n_set, const int64_t* nsup, const float* atoms,
                      float temperature, float lambda_cos, float lambda_l2, float scale, bool want_grad,
                      float* d_query, float* d_atoms, double* partials);
// Attention P (npx x K fp32, row-major) of the last tcgen05-decoded frame: e (bf16, core-matrix
// tiles) times 1/sum from row_stats.
void decoder_export_attention(cudaStream_t st, const DecoderWork& w, int64_t npx, float* p_out);
// Applies the step-accumulated A and R of the tcgen05 frames: d_atoms += A D + R^T W, d_proj += R D.
void decoder_finish_tc(cudaStream_t st, DecoderWork& w, const float* atoms, const float* proj, float* d_proj,
                       float* d_atoms);
void reconstruct(cudaStream_t st, const float* q, int64_t n, int ds, const float* atoms, const float* proj,
                 int64_t k, int df, float temperature, float* out, float* attention, float* scratch_qw);
void reconstruct_backward(cudaStream_t st, const float* q, const float* att, int64_t n, int ds,
                          const float* atoms, const float* proj, int64_t k, int df, float temperature,
                          const float* d_rec, float* d_q, float* d_proj, float* d_atoms, float* s_nk,
                          float* s_ndf, float* s_kdf);
void trust_region(cudaStream_t st, const float* atoms, const float* anchor, int64_t k, int df, float delta,
                  float* d_atoms, float grad_scale, double* penalty_out);

// Adam (K10) over the session's flat parameter vector.
struct AdamBlock {
  int64_t offset, count;
  float lr;
  int32_t kind;  // 0 plain, 1 quaternion block (renormalise rows of 4), -1 disabled
};
void adam_flat(cudaStream_t st, float* param, const float* grad, float* m, float* v, const AdamBlock* blocks,
               int nblocks, int64_t* steps, int64_t* skipped, const float* corr1, const float* corr2,
               int32_t table_len, int32_t* flags, const double* overflow, int64_t* overflow_steps,
               int64_t begin = 0, int64_t end = -1, const double* ext_flags = nullptr);
// Sharded step: per-block non-finite flags of grad[begin, end) into flags_out[block] (doubles, 1 = bad).
void adam_check_range(cudaStream_t st, const float* grad, const AdamBlock* blocks, int nblocks, int64_t begin,
                      int64_t end, double* flags_out);

// Streaming k-means (kmeans.cu): device points / centres / atoms, host weights.
cudaError_t kmeans_weighted(cudaStream_t st, const float* P, const float* W, int64_t n, int dim, int64_t k,
                            double (*uni)(void*), void* user, const float* warm, int64_t n_warm, int max_iters,
                            float* C, float* cw, int* iterations);
cudaError_t kmeans_stream_update(cudaStream_t st, const float* batch, int64_t n, int dim, float* atoms, float* anchor,
                                 float* weights, int64_t K, double (*uni)(void*), void* user, float decay);

// Evaluation (metrics.cu): device rows in, host scalars out.
cudaError_t metric_cos_dev(cudaStream_t st, const float* rec, const float* tgt, int64_t n, int d, double* out,
                           int32_t* flagged);
cudaError_t metric_miou_dev(cudaStream_t st, const float* emb, const int32_t* labels, int64_t n, int d,
                            const float* protos, int c, int64_t* inter, int64_t* uni, double* miou, bool* bad_label);
cudaError_t metric_psnr_dev(cudaStream_t st, const float* a, const float* b, int64_t n, double* db, int32_t* exact);
cudaError_t query_scores_dev(cudaStream_t st, const float* rec, int64_t n, int d, const float* emb, float* scores);
cudaError_t gather_supervision_dev(cudaStream_t st, const float* query, int ds, const int32_t* asg, int64_t npx,
                                   const float* feats, int df, bool normalize, float* q_out, float* t_out,
                                   int64_t* pix, int64_t cap, int64_t* n_rows);

void expf_selftest(cudaStream_t st, uint64_t first, int64_t n, float* out);
int umma_selftest(cudaStream_t st, const float* A, const float* B, float* C, int N, int K, int a_mn, int b_mn);

void set_launch_counter(int64_t* c);
// Host-side failure inside a launcher (no CUDA error to carry it): recorded here, reported and
// cleared by the next post-launch check of the C-ABI.
void set_sticky_error(const char* msg);
const char* take_sticky_error();
void count_launch(int n = 1);

}  // namespace lm
