/*
 * latmap_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE (see latmap_oracle.h).
 *
 * CPU restatement of the reference hot path, compiled twice (T=float -> *_f32,
 * T=double -> *_f64) plus once for the integer voxel-hash store (LM_ONCE).
 * Each function cites the reference file:line it follows. Paths are relative to
 * /root/reference/proj/.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "latmap_oracle.h"

#ifndef LM_ONCE

#if LM_DOUBLE
typedef double T;
#define S(x) x##_f64
static inline T lm_exp(T x) { return exp(x); }
static inline T lm_sqrt(T x) { return sqrt(x); }
static inline T lm_fabs(T x) { return fabs(x); }
#else
typedef float T;
#define S(x) x##_f32
/* std::exp(float) is what the reference calls (render.cpp:193,303, types.hpp:252-255): the C
 * library's expf, the same function the compiled reference (oracle/_ref) uses on this image.
 * (Round 1 used the correctly rounded (float)exp((double)x); libm differs from it on ~7e-5 of
 * inputs.) */
static inline T lm_exp(T x) { return expf(x); }
/* float sqrt / abs stay in float (Eigen's array().sqrt(), std::abs on float). */
static inline T lm_sqrt(T x) { return sqrtf(x); }
static inline T lm_fabs(T x) { return fabsf(x); }
#endif

#define MAP S(lm_map)
#define POSE S(lm_pose)
#define SPLAT S(lm_splat)
#define LOSS S(lm_loss)
#define FRAME S(lm_frame)
#define CFG S(lm_cfg)

/* RenderParams, render.hpp:13-19 */
#define K_ZNEAR ((T)0.01)
#define K_COVREG ((T)0.3)
#define K_SIGMACUT 3.0
#define K_ALPHAMAX ((T)0.999)
#define K_TSTOP ((T)1e-4)

static inline T sq_norm3(const T* v) { return (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]; }

/* sigmoid, types.hpp:252-255 */
static inline T lm_sigmoid(T x) {
  return x >= (T)0 ? (T)1 / ((T)1 + lm_exp(-x)) : lm_exp(x) / ((T)1 + lm_exp(x));
}

/* 3x3 row-major product, inner index summed left to right. */
static void mat3_mul(const T* a, const T* b, T* c) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c[3 * i + j] = (a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j]) + a[3 * i + 2] * b[6 + j];
}

/* quat_to_rot, core/se3.hpp:12-23 (normalises internally; zero norm invalid). */
int S(lm_quat_to_rot)(const T q[4], T r[9]) {
  T n = lm_sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  if (!(n > (T)0) || !isfinite((double)n)) return -1;
  const T w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  r[0] = (T)1 - (T)2 * (y * y + z * z);
  r[1] = (T)2 * (x * y - w * z);
  r[2] = (T)2 * (x * z + w * y);
  r[3] = (T)2 * (x * y + w * z);
  r[4] = (T)1 - (T)2 * (x * x + z * z);
  r[5] = (T)2 * (y * z - w * x);
  r[6] = (T)2 * (x * z - w * y);
  r[7] = (T)2 * (y * z + w * x);
  r[8] = (T)1 - (T)2 * (x * x + y * y);
  return 0;
}

/* rot_from_unit_quat, render.cpp:13-21 */
static void rot_from_unit_quat(const T* q, T* r) {
  const T w = q[0], x = q[1], y = q[2], z = q[3];
  r[0] = (T)1 - (T)2 * (y * y + z * z);
  r[1] = (T)2 * (x * y - w * z);
  r[2] = (T)2 * (x * z + w * y);
  r[3] = (T)2 * (x * y + w * z);
  r[4] = (T)1 - (T)2 * (x * x + z * z);
  r[5] = (T)2 * (y * z - w * x);
  r[6] = (T)2 * (x * z - w * y);
  r[7] = (T)2 * (y * z + w * x);
  r[8] = (T)1 - (T)2 * (x * x + y * y);
}

typedef struct {
  int visible;
  T p_cam[3], q_hat[4], q_norm, rot_gauss[9], scale[3], m[9], cov_cam[9], jac[6], mean2d[2],
      cov2d[4], cov_inv[4], alpha;
} FullProj;

/* project_one, render.cpp:42-72 */
static void project_one(const T* p, const T* q, const T* lsc, T logit, const T* rot_cw,
                        const T* origin, const lm_intr* intr, FullProj* f) {
  memset(f, 0, sizeof(*f));
  T d[3] = {p[0] - origin[0], p[1] - origin[1], p[2] - origin[2]};
  for (int i = 0; i < 3; ++i)
    f->p_cam[i] = (rot_cw[3 * i] * d[0] + rot_cw[3 * i + 1] * d[1]) + rot_cw[3 * i + 2] * d[2];
  const T z = f->p_cam[2];
  if (!(z > K_ZNEAR)) return;
  f->q_norm = lm_sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  if (!(f->q_norm > (T)0) || !isfinite((double)f->q_norm)) return;
  for (int i = 0; i < 4; ++i) f->q_hat[i] = q[i] / f->q_norm;
  rot_from_unit_quat(f->q_hat, f->rot_gauss);
  for (int i = 0; i < 3; ++i) f->scale[i] = lm_exp(lsc[i]);
  T rg[9];
  mat3_mul(rot_cw, f->rot_gauss, rg);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) f->m[3 * i + j] = rg[3 * i + j] * f->scale[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      f->cov_cam[3 * i + j] = (f->m[3 * i] * f->m[3 * j] + f->m[3 * i + 1] * f->m[3 * j + 1]) +
                              f->m[3 * i + 2] * f->m[3 * j + 2];
  const T fx = (T)intr->fx, fy = (T)intr->fy;
  const T x = f->p_cam[0], y = f->p_cam[1];
  f->mean2d[0] = fx * x / z + (T)intr->cx;
  f->mean2d[1] = fy * y / z + (T)intr->cy;
  f->jac[0] = fx / z;
  f->jac[1] = (T)0;
  f->jac[2] = -fx * x / (z * z);
  f->jac[3] = (T)0;
  f->jac[4] = fy / z;
  f->jac[5] = -fy * y / (z * z);
  T tmp[6];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      tmp[3 * i + j] = (f->jac[3 * i] * f->cov_cam[j] + f->jac[3 * i + 1] * f->cov_cam[3 + j]) +
                       f->jac[3 * i + 2] * f->cov_cam[6 + j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      f->cov2d[2 * i + j] = (tmp[3 * i] * f->jac[3 * j] + tmp[3 * i + 1] * f->jac[3 * j + 1]) +
                            tmp[3 * i + 2] * f->jac[3 * j + 2];
  f->cov2d[0] += K_COVREG;
  f->cov2d[3] += K_COVREG;
  const T det = f->cov2d[0] * f->cov2d[3] - f->cov2d[1] * f->cov2d[2];
  if (!(det > (T)0) || !isfinite((double)det)) return;
  f->cov_inv[0] = f->cov2d[3] / det;
  f->cov_inv[1] = -f->cov2d[1] / det;
  f->cov_inv[2] = -f->cov2d[2] / det;
  f->cov_inv[3] = f->cov2d[0] / det;
  f->alpha = lm_sigmoid(logit);
  f->visible = 1;
}

/* splat_bounds, render.cpp:75-91 (double precision). */
static int splat_bounds(const T* mean, const T* cov2d, const lm_intr* intr, int32_t* x0,
                        int32_t* x1, int32_t* y0, int32_t* y1) {
  const double rx = K_SIGMACUT * sqrt((double)cov2d[0]);
  const double ry = K_SIGMACUT * sqrt((double)cov2d[3]);
  const double u = (double)mean[0], v = (double)mean[1];
  if (!isfinite(u) || !isfinite(v) || !isfinite(rx) || !isfinite(ry)) return 0;
  const double lo_x = ceil(u - rx), hi_x = floor(u + rx);
  const double lo_y = ceil(v - ry), hi_y = floor(v + ry);
  if (hi_x < 0 || hi_y < 0 || lo_x > intr->width - 1 || lo_y > intr->height - 1) return 0;
  *x0 = (int32_t)(lo_x > 0.0 ? lo_x : 0.0);
  *x1 = (int32_t)((double)(intr->width - 1) < hi_x ? (double)(intr->width - 1) : hi_x);
  *y0 = (int32_t)(lo_y > 0.0 ? lo_y : 0.0);
  *y1 = (int32_t)((double)(intr->height - 1) < hi_y ? (double)(intr->height - 1) : hi_y);
  return *x0 <= *x1 && *y0 <= *y1;
}

static void pose_rot_cw(const POSE* pose, T* rot_cw, T* rot_wc) {
  T r[9];
  S(lm_quat_to_rot)(pose->rot, r);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      rot_cw[3 * i + j] = r[3 * j + i];
      if (rot_wc) rot_wc[3 * i + j] = r[3 * i + j];
    }
}

/* project_gaussian, render.cpp:118-132. Returns 1 when visible. */
int S(lm_project_gaussian)(const T pos[3], const T rot[4], const T lsc[3], T opa,
                           const POSE* pose, const lm_intr* intr, T mean2d[2], T cov2d[4],
                           T* depth) {
  T rot_cw[9];
  if (S(lm_quat_to_rot)(pose->rot, rot_cw) != 0) return -1;
  pose_rot_cw(pose, rot_cw, NULL);
  FullProj f;
  project_one(pos, rot, lsc, opa, rot_cw, pose->trans, intr, &f);
  if (!f.visible) return 0;
  int32_t x0, x1, y0, y1;
  if (!splat_bounds(f.mean2d, f.cov2d, intr, &x0, &x1, &y0, &y1)) return 0;
  memcpy(mean2d, f.mean2d, sizeof(T) * 2);
  memcpy(cov2d, f.cov2d, sizeof(T) * 4);
  *depth = f.p_cam[2];
  return 1;
}

/* ---------------- parallel_chunks, core/parallel.hpp:19-35 ---------------- */
typedef void (*chunk_fn)(void* ctx, int64_t begin, int64_t end, int tid);
typedef struct {
  chunk_fn fn;
  void* ctx;
  int64_t b, e;
  int tid;
} chunk_job;
static void* chunk_tramp(void* p) {
  chunk_job* j = (chunk_job*)p;
  j->fn(j->ctx, j->b, j->e, j->tid);
  return NULL;
}
static void parallel_chunks(int64_t total, int threads, chunk_fn fn, void* ctx) {
  if (threads < 1) threads = 1;
  if (threads == 1 || total < 2 * threads) {
    fn(ctx, 0, total, 0);
    return;
  }
  pthread_t th[256];
  chunk_job jobs[256];
  if (threads > 256) threads = 256;
  int64_t chunk = (total + threads - 1) / threads;
  int nt = 0;
  for (int t = 0; t < threads; ++t) {
    int64_t b = t * chunk, e = b + chunk < total ? b + chunk : total;
    if (b >= e) break;
    jobs[nt] = (chunk_job){fn, ctx, b, e, t};
    pthread_create(&th[nt], NULL, chunk_tramp, &jobs[nt]);
    ++nt;
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

/* ---------------- per-row / per-pixel candidate lists (render.cpp:93-112) ---------------- */
typedef struct {
  int32_t* v;
  int64_t n, cap;
} ivec;
static void iv_push(ivec* a, int32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 16;
    a->v = (int32_t*)realloc(a->v, sizeof(int32_t) * (size_t)a->cap);
  }
  a->v[a->n++] = x;
}

typedef struct {
  T depth;
  int32_t source, k;
} sort_item;
static int sort_cmp(const void* pa, const void* pb) {
  const sort_item* a = (const sort_item*)pa;
  const sort_item* b = (const sort_item*)pb;
  if (a->depth != b->depth) return a->depth < b->depth ? -1 : 1;
  return (a->source > b->source) - (a->source < b->source);
}
/* sort_pixel, render.cpp:104-112: order by (depth, source). */
static void sort_pixel(const SPLAT* splats, ivec* idx, sort_item* scratch) {
  for (int64_t i = 0; i < idx->n; ++i) {
    const SPLAT* s = &splats[idx->v[i]];
    scratch[i] = (sort_item){s->depth, s->source, idx->v[i]};
  }
  qsort(scratch, (size_t)idx->n, sizeof(sort_item), sort_cmp);
  for (int64_t i = 0; i < idx->n; ++i) idx->v[i] = scratch[i].k;
}

/* splats_by_row, render.cpp:93-101 */
static ivec* splats_by_row(const SPLAT* splats, int64_t n, int h) {
  ivec* rows = (ivec*)calloc((size_t)h, sizeof(ivec));
  for (int32_t k = 0; k < (int32_t)n; ++k)
    for (int32_t y = splats[k].y0; y <= splats[k].y1; ++y) iv_push(&rows[y], k);
  return rows;
}
static void free_rows(ivec* rows, int h) {
  for (int y = 0; y < h; ++y) free(rows[y].v);
  free(rows);
}

/* ---------------- render, render.cpp:133-214 ---------------- */
typedef struct {
  const MAP* map;
  const SPLAT* splats;
  int64_t n_splats;
  const ivec* rows;
  int h, w;
  T *color, *depth, *query, *alpha;
} render_ctx;

static void render_rows(void* pc, int64_t yb, int64_t ye, int tid) {
  (void)tid;
  render_ctx* c = (render_ctx*)pc;
  const int w = c->w, ds = c->map->ds;
  ivec* cols = (ivec*)calloc((size_t)w, sizeof(ivec));
  sort_item* scratch = (sort_item*)malloc(sizeof(sort_item) * (size_t)(c->n_splats + 1));
  for (int64_t y = yb; y < ye; ++y) {
    for (int x = 0; x < w; ++x) cols[x].n = 0;
    const ivec* row = &c->rows[y];
    for (int64_t r = 0; r < row->n; ++r) {
      const SPLAT* s = &c->splats[row->v[r]];
      for (int32_t x = s->x0; x <= s->x1; ++x) iv_push(&cols[x], row->v[r]);
    }
    for (int x = 0; x < w; ++x) {
      ivec* idx = &cols[x];
      if (idx->n == 0) continue;
      sort_pixel(c->splats, idx, scratch);
      T trans = (T)1;
      T acc_c[3] = {0, 0, 0};
      T acc_d = 0, acc_a = 0;
      T* qrow = c->query + ((size_t)y * w + x) * ds;
      for (int64_t i = 0; i < idx->n; ++i) {
        const SPLAT* s = &c->splats[idx->v[i]];
        const T dx = (T)x - s->mean[0];
        const T dy = (T)y - s->mean[1];
        const T rho = s->cov_inv[0] * dx * dx + (T)2 * s->cov_inv[1] * dx * dy +
                      s->cov_inv[3] * dy * dy;
        T a = s->alpha * lm_exp((T)(-0.5) * rho);
        if (a > K_ALPHAMAX) a = K_ALPHAMAX;
        const T wgt = a * trans;
        const T* col = c->map->col + (size_t)s->source * 3;
        acc_c[0] += wgt * col[0];
        acc_c[1] += wgt * col[1];
        acc_c[2] += wgt * col[2];
        acc_d += wgt * s->depth;
        acc_a += wgt;
        const T* f = c->map->feat + (size_t)s->source * ds;
        for (int cc = 0; cc < ds; ++cc) qrow[cc] += wgt * f[cc];
        trans *= ((T)1 - a);
        if (trans < K_TSTOP) break;
      }
      size_t p = (size_t)y * w + x;
      c->color[p * 3 + 0] = acc_c[0];
      c->color[p * 3 + 1] = acc_c[1];
      c->color[p * 3 + 2] = acc_c[2];
      c->depth[p] = acc_d;
      c->alpha[p] = acc_a;
    }
  }
  for (int x = 0; x < w; ++x) free(cols[x].v);
  free(cols);
  free(scratch);
}

static int intr_valid(const lm_intr* i) {
  return i->fx > 0 && i->fy > 0 && i->width > 0 && i->height > 0 && i->cx >= 0 &&
         i->cx < (float)i->width && i->cy >= 0 && i->cy < (float)i->height;
}

int S(lm_render)(const MAP* map, const POSE* pose, const lm_intr* intr, int threads, T* color,
                 T* depth, T* query, T* alpha, SPLAT* splats, int64_t cap, int64_t* n_splats) {
  if (!intr_valid(intr)) return -1; /* render.cpp:136 invalid_argument */
  const int h = intr->height, w = intr->width, ds = map->ds;
  memset(color, 0, sizeof(T) * (size_t)h * w * 3);
  memset(depth, 0, sizeof(T) * (size_t)h * w);
  memset(query, 0, sizeof(T) * (size_t)h * w * ds);
  memset(alpha, 0, sizeof(T) * (size_t)h * w);
  T rot_cw[9];
  pose_rot_cw(pose, rot_cw, NULL);
  int64_t ns = 0;
  for (int64_t i = 0; i < map->n; ++i) {
    FullProj f;
    project_one(map->pos + 3 * i, map->rot + 4 * i, map->lsc + 3 * i, map->opa[i], rot_cw,
                pose->trans, intr, &f);
    if (!f.visible) continue;
    SPLAT s;
    if (!splat_bounds(f.mean2d, f.cov2d, intr, &s.x0, &s.x1, &s.y0, &s.y1)) continue;
    if (ns >= cap) return -2;
    s.mean[0] = f.mean2d[0];
    s.mean[1] = f.mean2d[1];
    memcpy(s.cov_inv, f.cov_inv, sizeof(T) * 4);
    s.depth = f.p_cam[2];
    s.alpha = f.alpha;
    s.source = (int32_t)i;
    splats[ns++] = s;
  }
  *n_splats = ns;
  ivec* rows = splats_by_row(splats, ns, h);
  render_ctx c = {map, splats, ns, rows, h, w, color, depth, query, alpha};
  parallel_chunks(h, threads, render_rows, &c);
  free_rows(rows, h);
  return 0;
}

/* ---------------- render_backward, render.cpp:253-432 ---------------- */
#define ACC_STRIDE(ds) (10 + (ds))
typedef struct {
  int32_t k;
  T alpha_eff, weight, trans;
  int clamped;
} blend_step;

typedef struct {
  const MAP* map;
  const SPLAT* splats;
  int64_t n_splats;
  const ivec* rows;
  int h, w;
  const T *d_color, *d_depth, *d_query;
  T** partials;
} bwd_ctx;

static void bwd_rows(void* pc, int64_t yb, int64_t ye, int tid) {
  bwd_ctx* c = (bwd_ctx*)pc;
  const int w = c->w, ds = c->map->ds;
  const int stride = ACC_STRIDE(ds);
  T* acc = c->partials[tid];
  ivec* cols = (ivec*)calloc((size_t)w, sizeof(ivec));
  sort_item* scratch = (sort_item*)malloc(sizeof(sort_item) * (size_t)(c->n_splats + 1));
  blend_step* steps = (blend_step*)malloc(sizeof(blend_step) * (size_t)(c->n_splats + 1));
  for (int64_t y = yb; y < ye; ++y) {
    for (int x = 0; x < w; ++x) cols[x].n = 0;
    const ivec* row = &c->rows[y];
    for (int64_t r = 0; r < row->n; ++r) {
      const SPLAT* s = &c->splats[row->v[r]];
      for (int32_t x = s->x0; x <= s->x1; ++x) iv_push(&cols[x], row->v[r]);
    }
    for (int x = 0; x < w; ++x) {
      ivec* idx = &cols[x];
      if (idx->n == 0) continue;
      sort_pixel(c->splats, idx, scratch);
      const size_t p = (size_t)y * w + x;
      const T* uc = c->d_color ? c->d_color + p * 3 : NULL;
      const T uz = c->d_depth ? c->d_depth[p] : (T)0;
      const T* uq = c->d_query ? c->d_query + p * ds : NULL;
      /* replay (render.cpp:294-309) */
      int64_t ns = 0;
      T trans = (T)1;
      for (int64_t i = 0; i < idx->n; ++i) {
        const SPLAT* s = &c->splats[idx->v[i]];
        const T dx = (T)x - s->mean[0];
        const T dy = (T)y - s->mean[1];
        const T rho = s->cov_inv[0] * dx * dx + (T)2 * s->cov_inv[1] * dx * dy +
                      s->cov_inv[3] * dy * dy;
        T a = s->alpha * lm_exp((T)(-0.5) * rho);
        const int clamped = a > K_ALPHAMAX;
        if (clamped) a = K_ALPHAMAX;
        steps[ns++] = (blend_step){idx->v[i], a, a * trans, trans, clamped};
        trans *= ((T)1 - a);
        if (trans < K_TSTOP) break;
      }
      /* reverse sweep (render.cpp:315-353) */
      T s_after = (T)0;
      for (int64_t it = ns - 1; it >= 0; --it) {
        const blend_step* st = &steps[it];
        const SPLAT* s = &c->splats[st->k];
        const int64_t src = s->source;
        const T* colr = c->map->col + src * 3;
        const T* fr = c->map->feat + src * ds;
        T value = (T)0;
        if (uc) value += uc[0] * colr[0] + uc[1] * colr[1] + uc[2] * colr[2];
        value += uz * s->depth;
        if (uq)
          for (int cc = 0; cc < ds; ++cc) value += uq[cc] * fr[cc];
        T* a = acc + (size_t)st->k * stride;
        if (uc) {
          a[7] += st->weight * uc[0];
          a[8] += st->weight * uc[1];
          a[9] += st->weight * uc[2];
        }
        a[5] += st->weight * uz;
        if (uq)
          for (int cc = 0; cc < ds; ++cc) a[10 + cc] += st->weight * uq[cc];
        const T d_alpha = st->trans * value - s_after / ((T)1 - st->alpha_eff);
        s_after += st->weight * value;
        if (st->clamped) continue;
        const T dx = (T)x - s->mean[0];
        const T dy = (T)y - s->mean[1];
        const T g = st->alpha_eff / s->alpha;
        a[6] += d_alpha * g;
        const T d_rho = (T)(-0.5) * st->alpha_eff * d_alpha;
        const T ad_x = s->cov_inv[0] * dx + s->cov_inv[1] * dy;
        const T ad_y = s->cov_inv[2] * dx + s->cov_inv[3] * dy;
        a[0] += d_rho * (T)(-2) * ad_x;
        a[1] += d_rho * (T)(-2) * ad_y;
        a[2] += d_rho * dx * dx;
        a[3] += d_rho * dx * dy;
        a[4] += d_rho * dy * dy;
      }
    }
  }
  for (int x = 0; x < w; ++x) free(cols[x].v);
  free(cols);
  free(scratch);
  free(steps);
}

typedef struct {
  const MAP* map;
  const SPLAT* splats;
  const T* acc;
  const T *rot_cw, *rot_wc, *origin;
  const lm_intr* intr;
  MAP* grads;
} proj_bwd_ctx;

/* projection backward, render.cpp:368-429 */
static void proj_bwd_chunk(void* pc, int64_t kb, int64_t ke, int tid) {
  (void)tid;
  proj_bwd_ctx* c = (proj_bwd_ctx*)pc;
  const int ds = c->map->ds;
  const int stride = ACC_STRIDE(ds);
  const T fx = (T)c->intr->fx, fy = (T)c->intr->fy;
  for (int64_t k = kb; k < ke; ++k) {
    const SPLAT* s = &c->splats[k];
    const int64_t i = s->source;
    const T* a = c->acc + (size_t)k * stride;
    c->grads->col[3 * i + 0] += a[7];
    c->grads->col[3 * i + 1] += a[8];
    c->grads->col[3 * i + 2] += a[9];
    for (int cc = 0; cc < ds; ++cc) c->grads->feat[(size_t)i * ds + cc] += a[10 + cc];
    FullProj f;
    project_one(c->map->pos + 3 * i, c->map->rot + 4 * i, c->map->lsc + 3 * i, c->map->opa[i],
                c->rot_cw, c->origin, c->intr, &f);
    if (!f.visible) continue;
    c->grads->opa[i] += a[6] * f.alpha * ((T)1 - f.alpha);
    /* d_cov2d = -A * dA * A (render.cpp:387-389) */
    const T da[4] = {a[2], a[3], a[3], a[4]};
    T t1[4], dc[4];
    for (int r = 0; r < 2; ++r)
      for (int q = 0; q < 2; ++q) t1[2 * r + q] = (-f.cov_inv[2 * r]) * da[q] + (-f.cov_inv[2 * r + 1]) * da[2 + q];
    for (int r = 0; r < 2; ++r)
      for (int q = 0; q < 2; ++q) dc[2 * r + q] = t1[2 * r] * f.cov_inv[q] + t1[2 * r + 1] * f.cov_inv[2 + q];
    /* d_cov_cam = J^T dC J (3x3) */
    T jt_dc[6]; /* 3x2 */
    for (int r = 0; r < 3; ++r)
      for (int q = 0; q < 2; ++q) jt_dc[2 * r + q] = f.jac[r] * dc[q] + f.jac[3 + r] * dc[2 + q];
    T dcc[9];
    for (int r = 0; r < 3; ++r)
      for (int q = 0; q < 3; ++q) dcc[3 * r + q] = jt_dc[2 * r] * f.jac[q] + jt_dc[2 * r + 1] * f.jac[3 + q];
    /* d_jac = 2 * dC * J * cov_cam (2x3) */
    T dcj[6], djac[6];
    for (int r = 0; r < 2; ++r)
      for (int q = 0; q < 3; ++q) dcj[3 * r + q] = ((T)2 * dc[2 * r]) * f.jac[q] + ((T)2 * dc[2 * r + 1]) * f.jac[3 + q];
    for (int r = 0; r < 2; ++r)
      for (int q = 0; q < 3; ++q)
        djac[3 * r + q] = (dcj[3 * r] * f.cov_cam[q] + dcj[3 * r + 1] * f.cov_cam[3 + q]) +
                          dcj[3 * r + 2] * f.cov_cam[6 + q];
    /* d_m = 2 * d_cov_cam * m */
    T dcc2[9], dm[9];
    for (int r = 0; r < 9; ++r) dcc2[r] = (T)2 * dcc[r];
    mat3_mul(dcc2, f.m, dm);
    /* d_rot_gauss = rot_cw^T * d_m * diag(scale) */
    T rwt[9], t3[9], drg[9];
    for (int r = 0; r < 3; ++r)
      for (int q = 0; q < 3; ++q) rwt[3 * r + q] = c->rot_cw[3 * q + r];
    mat3_mul(rwt, dm, t3);
    for (int r = 0; r < 3; ++r)
      for (int q = 0; q < 3; ++q) drg[3 * r + q] = t3[3 * r + q] * f.scale[q];
    T rcg[9];
    mat3_mul(c->rot_cw, f.rot_gauss, rcg);
    for (int cc = 0; cc < 3; ++cc) {
      T dot = (rcg[cc] * dm[cc] + rcg[3 + cc] * dm[3 + cc]) + rcg[6 + cc] * dm[6 + cc];
      c->grads->lsc[3 * i + cc] += dot * f.scale[cc];
    }
    const T qw = f.q_hat[0], qx = f.q_hat[1], qy = f.q_hat[2], qz = f.q_hat[3];
    const T dw[9] = {0, -qz, qy, qz, 0, -qx, -qy, qx, 0};
    const T dxm[9] = {0, qy, qz, qy, (T)(-2) * qx, -qw, qz, qw, (T)(-2) * qx};
    const T dym[9] = {(T)(-2) * qy, qx, qw, qx, 0, qz, -qw, qz, (T)(-2) * qy};
    const T dzm[9] = {(T)(-2) * qz, -qw, qx, qw, (T)(-2) * qz, qy, qx, qy, 0};
    T dqh[4] = {0, 0, 0, 0};
    for (int r = 0; r < 9; ++r) {
      dqh[0] += dw[r] * drg[r];
      dqh[1] += dxm[r] * drg[r];
      dqh[2] += dym[r] * drg[r];
      dqh[3] += dzm[r] * drg[r];
    }
    for (int r = 0; r < 4; ++r) dqh[r] = (T)2 * dqh[r];
    const T qdot = ((f.q_hat[0] * dqh[0] + f.q_hat[1] * dqh[1]) + f.q_hat[2] * dqh[2]) + f.q_hat[3] * dqh[3];
    for (int r = 0; r < 4; ++r) c->grads->rot[4 * i + r] += (dqh[r] - f.q_hat[r] * qdot) / f.q_norm;
    const T x = f.p_cam[0], y = f.p_cam[1], z = f.p_cam[2];
    T dp[3] = {0, 0, 0};
    dp[0] += a[0] * fx / z;
    dp[2] += a[0] * (-fx * x / (z * z));
    dp[1] += a[1] * fy / z;
    dp[2] += a[1] * (-fy * y / (z * z));
    dp[0] += djac[2] * (-fx / (z * z));
    dp[1] += djac[5] * (-fy / (z * z));
    dp[2] += djac[0] * (-fx / (z * z)) + djac[2] * ((T)2 * fx * x / (z * z * z)) +
             djac[4] * (-fy / (z * z)) + djac[5] * ((T)2 * fy * y / (z * z * z));
    dp[2] += a[5];
    for (int r = 0; r < 3; ++r)
      c->grads->pos[3 * i + r] +=
          (c->rot_wc[3 * r] * dp[0] + c->rot_wc[3 * r + 1] * dp[1]) + c->rot_wc[3 * r + 2] * dp[2];
  }
}

int S(lm_render_backward)(const MAP* map, const POSE* pose, const lm_intr* intr,
                          const SPLAT* splats, int64_t n_splats, const T* d_color,
                          const T* d_depth, const T* d_query, int threads, MAP* grads) {
  /* grads are accumulated (+=) into caller-zeroed buffers (MapGradientsT::resize_like). */
  if (n_splats == 0) return 0;
  const int h = intr->height, w = intr->width, ds = map->ds;
  if (threads < 1) threads = 1;
  ivec* rows = splats_by_row(splats, n_splats, h);
  const size_t stride = (size_t)ACC_STRIDE(ds);
  T** partials = (T**)malloc(sizeof(T*) * (size_t)threads);
  for (int t = 0; t < threads; ++t)
    partials[t] = (T*)calloc((size_t)n_splats * stride, sizeof(T));
  bwd_ctx c = {map, splats, n_splats, rows, h, w, d_color, d_depth, d_query, partials};
  parallel_chunks(h, threads, bwd_rows, &c);
  /* reduce partials in thread order (render.cpp:358) */
  for (int t = 1; t < threads; ++t)
    for (size_t i = 0; i < (size_t)n_splats * stride; ++i) partials[0][i] += partials[t][i];
  T rot_cw[9], rot_wc[9];
  pose_rot_cw(pose, rot_cw, rot_wc);
  proj_bwd_ctx pc = {map, splats, partials[0], rot_cw, rot_wc, pose->trans, intr, grads};
  parallel_chunks(n_splats, threads, proj_bwd_chunk, &pc);
  for (int t = 0; t < threads; ++t) free(partials[t]);
  free(partials);
  free_rows(rows, h);
  return 0;
}

/* ---------------- losses, losses.cpp ---------------- */
#define KWIN 11
#define KRAD 5
/* ssim_kernel, losses.cpp:13-25 */
static void ssim_kernel(T* k) {
  double w[KWIN], sum = 0;
  for (int i = 0; i < KWIN; ++i) {
    double d = i - KRAD;
    w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
    k[i] = (T)w[i];
    sum += w[i];
  }
  for (int i = 0; i < KWIN; ++i) k[i] = (T)((double)k[i] / sum);
}
static inline int reflect101(int i, int n) {
  if (i < 0) return -i;
  if (i >= n) return 2 * n - 2 - i;
  return i;
}
/* filter_plane, losses.cpp:34-54 */
static void filter_plane(const T* kern, const T* in, T* out, T* tmp, int h, int w) {
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      T acc = 0;
      for (int k = -KRAD; k <= KRAD; ++k) acc += kern[k + KRAD] * in[(size_t)y * w + reflect101(x + k, w)];
      tmp[(size_t)y * w + x] = acc;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      T acc = 0;
      for (int k = -KRAD; k <= KRAD; ++k) acc += kern[k + KRAD] * tmp[(size_t)reflect101(y + k, h) * w + x];
      out[(size_t)y * w + x] = acc;
    }
}
/* filter_plane_adjoint, losses.cpp:57-75 */
static void filter_plane_adjoint(const T* kern, const T* in, T* out, T* tmp, int h, int w) {
  size_t n = (size_t)h * w;
  memset(tmp, 0, sizeof(T) * n);
  memset(out, 0, sizeof(T) * n);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      T v = in[(size_t)y * w + x];
      for (int k = -KRAD; k <= KRAD; ++k) tmp[(size_t)reflect101(y + k, h) * w + x] += kern[k + KRAD] * v;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      T v = tmp[(size_t)y * w + x];
      for (int k = -KRAD; k <= KRAD; ++k) out[(size_t)y * w + reflect101(x + k, w)] += kern[k + KRAD] * v;
    }
}

/* ssim_global, losses.cpp:85-129 */
static T ssim_global(const T* a, const T* b, int h, int w, int ch, T* d_a) {
  const T c1 = (T)0.01 * (T)0.01, c2 = (T)0.03 * (T)0.03;
  const int64_t n = (int64_t)h * w;
  T total = 0;
  for (int c = 0; c < ch; ++c) {
    T mx = 0, my = 0;
    for (int64_t i = 0; i < n; ++i) {
      mx += a[i * ch + c];
      my += b[i * ch + c];
    }
    mx /= (T)n;
    my /= (T)n;
    T vx = 0, vy = 0, cov = 0;
    for (int64_t i = 0; i < n; ++i) {
      T dx = a[i * ch + c] - mx, dy = b[i * ch + c] - my;
      vx += dx * dx;
      vy += dy * dy;
      cov += dx * dy;
    }
    vx /= (T)n;
    vy /= (T)n;
    cov /= (T)n;
    const T a1 = (T)2 * mx * my + c1, a2 = (T)2 * cov + c2;
    const T b1 = mx * mx + my * my + c1, b2 = vx + vy + c2;
    const T s = (a1 * a2) / (b1 * b2);
    total += s;
    if (d_a) {
      const T ds_dmx = (T)2 * my * a2 / (b1 * b2) - s * (T)2 * mx / b1;
      const T ds_dvx = -s / b2;
      const T ds_dcov = (T)2 * a1 / (b1 * b2);
      for (int64_t i = 0; i < n; ++i) {
        T dx = a[i * ch + c] - mx, dy = b[i * ch + c] - my;
        d_a[i * ch + c] += (ds_dmx / (T)n + ds_dvx * (T)2 * dx / (T)n + ds_dcov * dy / (T)n) / (T)ch;
      }
    }
  }
  return total / (T)ch;
}

/* ssim, losses.cpp:133-198. d_a (optional) is overwritten. */
T S(lm_ssim)(const T* a, const T* b, int h, int w, int ch, T* d_a) {
  const size_t n = (size_t)h * w;
  if (d_a) memset(d_a, 0, sizeof(T) * n * ch);
  if (h < KWIN || w < KWIN) return ssim_global(a, b, h, w, ch, d_a);
  T kern[KWIN];
  ssim_kernel(kern);
  const T c1 = (T)0.01 * (T)0.01, c2 = (T)0.03 * (T)0.03;
  T* buf = (T*)malloc(sizeof(T) * n * 14);
  T *px = buf, *py = buf + n, *tmp = buf + 2 * n, *mx = buf + 3 * n, *my = buf + 4 * n,
    *ex2 = buf + 5 * n, *ey2 = buf + 6 * n, *exy = buf + 7 * n, *work = buf + 8 * n,
    *dmu = buf + 9 * n, *de2 = buf + 10 * n, *dexy = buf + 11 * n, *adj = buf + 12 * n;
  T total = 0;
  for (int c = 0; c < ch; ++c) {
    for (size_t i = 0; i < n; ++i) {
      px[i] = a[i * ch + c];
      py[i] = b[i * ch + c];
    }
    filter_plane(kern, px, mx, tmp, h, w);
    filter_plane(kern, py, my, tmp, h, w);
    for (size_t i = 0; i < n; ++i) work[i] = px[i] * px[i];
    filter_plane(kern, work, ex2, tmp, h, w);
    for (size_t i = 0; i < n; ++i) work[i] = py[i] * py[i];
    filter_plane(kern, work, ey2, tmp, h, w);
    for (size_t i = 0; i < n; ++i) work[i] = px[i] * py[i];
    filter_plane(kern, work, exy, tmp, h, w);
    for (size_t i = 0; i < n; ++i) {
      const T sx2 = ex2[i] - mx[i] * mx[i];
      const T sy2 = ey2[i] - my[i] * my[i];
      const T sxy = exy[i] - mx[i] * my[i];
      const T a1 = (T)2 * mx[i] * my[i] + c1;
      const T a2 = (T)2 * sxy + c2;
      const T b1 = mx[i] * mx[i] + my[i] * my[i] + c1;
      const T b2 = sx2 + sy2 + c2;
      const T s = (a1 * a2) / (b1 * b2);
      total += s;
      if (d_a) {
        dmu[i] = (T)2 * my[i] * (a2 - a1) / (b1 * b2) - s * (T)2 * mx[i] / b1 + s * (T)2 * mx[i] / b2;
        de2[i] = -s / b2;
        dexy[i] = (T)2 * a1 / (b1 * b2);
      }
    }
    if (d_a) {
      const T scale = (T)1 / ((T)n * (T)ch);
      filter_plane_adjoint(kern, dmu, adj, tmp, h, w);
      for (size_t i = 0; i < n; ++i) d_a[i * ch + c] += adj[i] * scale;
      filter_plane_adjoint(kern, de2, adj, tmp, h, w);
      for (size_t i = 0; i < n; ++i) d_a[i * ch + c] += (T)2 * px[i] * adj[i] * scale;
      filter_plane_adjoint(kern, dexy, adj, tmp, h, w);
      for (size_t i = 0; i < n; ++i) d_a[i * ch + c] += py[i] * adj[i] * scale;
    }
  }
  free(buf);
  return total / ((T)n * (T)ch);
}

/* rgb_loss, losses.cpp:200-224 */
int S(lm_rgb_loss)(const T* rendered, const T* observed, int h, int w, int ch, T lambda_i1,
                   T lambda_i2, int want_grad, T* grad, T* l1_out, T* ssim_loss, T* value) {
  const size_t sz = (size_t)h * w * ch;
  const T n = (T)sz;
  T l1 = 0;
  for (size_t i = 0; i < sz; ++i) {
    T d = rendered[i] - observed[i];
    l1 += lm_fabs(d);
    if (want_grad) grad[i] = lambda_i1 * (d > 0 ? (T)1 : (d < 0 ? (T)(-1) : (T)0)) / n;
  }
  *l1_out = l1 / n;
  T* d_ssim = want_grad ? (T*)malloc(sizeof(T) * sz) : NULL;
  T s = S(lm_ssim)(rendered, observed, h, w, ch, d_ssim);
  *ssim_loss = ((T)1 - s) / (T)2;
  if (want_grad) {
    for (size_t i = 0; i < sz; ++i) grad[i] += lambda_i2 * (T)(-0.5) * d_ssim[i];
    free(d_ssim);
  }
  *value = lambda_i1 * *l1_out + lambda_i2 * *ssim_loss;
  return 0;
}

/* depth_loss, losses.cpp:226-255 */
int S(lm_depth_loss)(const T* rendered, const T* observed, const T* alpha, int64_t n,
                     int want_grad, T* grad, T* value, int32_t* flagged) {
  int64_t valid = 0;
  T sum = 0;
  if (want_grad) memset(grad, 0, sizeof(T) * (size_t)n);
  for (int64_t i = 0; i < n; ++i)
    if (observed[i] > (T)0 && alpha[i] > (T)0.5) {
      sum += lm_fabs(rendered[i] - observed[i]);
      ++valid;
    }
  *flagged = 0;
  *value = 0;
  if (valid == 0) {
    *flagged = 1;
    return 0;
  }
  *value = sum / (T)valid;
  if (want_grad)
    for (int64_t i = 0; i < n; ++i)
      if (observed[i] > (T)0 && alpha[i] > (T)0.5) {
        T d = rendered[i] - observed[i];
        grad[i] = (d > 0 ? (T)1 : (d < 0 ? (T)(-1) : (T)0)) / (T)valid;
      }
  return 0;
}

/* trust_region_penalty, dictionary.cpp:85-101 */
T S(lm_trust_region_penalty)(const T* atoms, const T* anchor, int64_t k, int64_t df, T delta,
                             T* d_atoms) {
  if (d_atoms) memset(d_atoms, 0, sizeof(T) * (size_t)(k * df));
  T total = 0;
  T* diff = (T*)malloc(sizeof(T) * (size_t)df);
  for (int64_t j = 0; j < k; ++j) {
    T ss = 0;
    for (int64_t c = 0; c < df; ++c) {
      diff[c] = atoms[j * df + c] - anchor[j * df + c];
      ss += diff[c] * diff[c];
    }
    T dist = lm_sqrt(ss);
    T excess = dist - delta;
    if (excess > (T)0) {
      total += excess;
      if (d_atoms)
        for (int64_t c = 0; c < df; ++c) d_atoms[j * df + c] = diff[c] / dist;
    }
  }
  free(diff);
  return total;
}

/* feature_loss, losses.cpp:257-294 */
int S(lm_feature_loss)(const T* rec, const T* tgt, int64_t n, int64_t df, const T* atoms,
                       const T* anchor, int64_t k, T delta, T lambda_cos, T lambda_l2,
                       T lambda_trust, int want_grad, T* d_rec, T* d_atoms_trust, T* cos_term,
                       T* l2_term, T* trust_term, T* value, int32_t* zflag) {
  const T eps = (T)1e-8;
  T ct = 0, lt = 0;
  *zflag = 0;
  if (want_grad) memset(d_rec, 0, sizeof(T) * (size_t)(n * df));
  for (int64_t r = 0; r < n; ++r) {
    const T* u = rec + r * df;
    const T* v = tgt + r * df;
    T su = 0, sv = 0, dot = 0, sd = 0;
    for (int64_t c = 0; c < df; ++c) su += u[c] * u[c];
    for (int64_t c = 0; c < df; ++c) sv += v[c] * v[c];
    const T nu = lm_sqrt(su), nv = lm_sqrt(sv);
    if (nu < eps || nv < eps) *zflag = 1;
    const T nug = nu > eps ? nu : eps, nvg = nv > eps ? nv : eps;
    for (int64_t c = 0; c < df; ++c) dot += u[c] * v[c];
    const T cosv = dot / (nug * nvg);
    ct += ((T)1 - cosv);
    for (int64_t c = 0; c < df; ++c) {
      T d = u[c] - v[c];
      sd += d * d;
    }
    lt += sd;
    if (want_grad) {
      T* g = d_rec + r * df;
      for (int64_t c = 0; c < df; ++c)
        g[c] += lambda_cos * (-(v[c] / (nug * nvg) - dot * u[c] / (nug * nug * nug * nvg))) / (T)n;
      for (int64_t c = 0; c < df; ++c) g[c] += lambda_l2 * (T)2 * (u[c] - v[c]) / (T)n;
    }
  }
  if (n > 0) {
    ct /= (T)n;
    lt /= (T)n;
  }
  *cos_term = ct;
  *l2_term = lt;
  *trust_term = S(lm_trust_region_penalty)(atoms, anchor, k, df, delta, want_grad ? d_atoms_trust : NULL);
  if (want_grad)
    for (int64_t i = 0; i < k * df; ++i) d_atoms_trust[i] = lambda_trust * d_atoms_trust[i];
  *value = lambda_cos * ct + lambda_l2 * lt + lambda_trust * *trust_term;
  return 0;
}

/* ---------------- dense products (Eigen MatX stand-ins) ----------------
 * Every product element is summed over the inner index in ASCENDING order, one separately
 * rounded multiply and add per term (no FMA: -ffp-contract=off); this order is the oracle's
 * definition of Eigen's float GEMM bits. The loops are blocked (4 output rows share each B row
 * load; 256-column / 128-inner panels stay in L1/L2) and split by output rows over
 * lm_oracle_set_gemm_threads() threads (default 1, like the reference's Eigen without OpenMP).
 * Neither changes the per-element order, so results are bit-identical for every thread count. */
extern int lm_oracle_gemm_threads_value;
#define GJ 256
#define GK 128
typedef struct {
  int64_t M, N, K;
  const T* A;
  const T* B;
  T* C;
} gemm_job;
/* C(MxN) = A(MxK) B(KxN) for rows [i0, i1). */
static void gemm_nn_rows(void* pc, int64_t i0, int64_t i1, int tid) {
  const gemm_job* g = (const gemm_job*)pc;
  const int64_t N = g->N, K = g->K;
  for (int64_t i = i0; i < i1; ++i) memset(g->C + i * N, 0, sizeof(T) * (size_t)N);
  for (int64_t jb = 0; jb < N; jb += GJ) {
    const int64_t je = jb + GJ < N ? jb + GJ : N, nj = je - jb;
    for (int64_t kb = 0; kb < K; kb += GK) {
      const int64_t ke = kb + GK < K ? kb + GK : K;
      int64_t i = i0;
      for (; i + 4 <= i1; i += 4) {
        T* c0 = g->C + i * N + jb;
        T* c1 = c0 + N;
        T* c2 = c1 + N;
        T* c3 = c2 + N;
        const T* a = g->A + i * K;
        for (int64_t k = kb; k < ke; ++k) {
          const T a0 = a[k], a1 = a[K + k], a2 = a[2 * K + k], a3 = a[3 * K + k];
          const T* b = g->B + k * N + jb;
          for (int64_t j = 0; j < nj; ++j) {
            const T bj = b[j];
            c0[j] += a0 * bj;
            c1[j] += a1 * bj;
            c2[j] += a2 * bj;
            c3[j] += a3 * bj;
          }
        }
      }
      for (; i < i1; ++i) {
        T* c = g->C + i * N + jb;
        for (int64_t k = kb; k < ke; ++k) {
          const T av = g->A[i * K + k];
          const T* b = g->B + k * N + jb;
          for (int64_t j = 0; j < nj; ++j) c[j] += av * b[j];
        }
      }
    }
  }
}
static int gemm_threads(int64_t rows, int64_t work) {
  int t = lm_oracle_gemm_threads_value;
  if (work < (int64_t)1 << 22) t = 1;
  return (int64_t)t > rows ? (int)(rows > 0 ? rows : 1) : t;
}
static void gemm_nn(int64_t M, int64_t N, int64_t K, const T* A, const T* B, T* C) {
  gemm_job g = {M, N, K, A, B, C};
  parallel_chunks(M, gemm_threads(M, M * N * K), gemm_nn_rows, &g);
}
static T* transpose(int64_t R, int64_t Cc, const T* A) {
  T* t = (T*)malloc(sizeof(T) * (size_t)(R * Cc));
  for (int64_t ib = 0; ib < R; ib += 32)
    for (int64_t jb = 0; jb < Cc; jb += 32)
      for (int64_t i = ib; i < ib + 32 && i < R; ++i)
        for (int64_t j = jb; j < jb + 32 && j < Cc; ++j) t[j * R + i] = A[i * Cc + j];
  return t;
}
/* C(MxN) = A(MxK) B^T, B is NxK. */
static void gemm_nt(int64_t M, int64_t N, int64_t K, const T* A, const T* B, T* C) {
  T* bt = transpose(N, K, B);
  gemm_nn(M, N, K, A, bt, C);
  free(bt);
}
/* C(MxN) = A^T B, A is KxM, B is KxN: output rows [i0, i1), inner index k ascending. */
static void gemm_tn_rows(void* pc, int64_t i0, int64_t i1, int tid) {
  const gemm_job* g = (const gemm_job*)pc;
  const int64_t M = g->M, N = g->N, K = g->K;
  for (int64_t i = i0; i < i1; ++i) memset(g->C + i * N, 0, sizeof(T) * (size_t)N);
  for (int64_t jb = 0; jb < N; jb += GJ) {
    const int64_t je = jb + GJ < N ? jb + GJ : N, nj = je - jb;
    for (int64_t kb = 0; kb < K; kb += GK) {
      const int64_t ke = kb + GK < K ? kb + GK : K;
      int64_t i = i0;
      for (; i + 4 <= i1; i += 4) {
        T* c0 = g->C + i * N + jb;
        T* c1 = c0 + N;
        T* c2 = c1 + N;
        T* c3 = c2 + N;
        for (int64_t k = kb; k < ke; ++k) {
          const T* a = g->A + k * M + i;
          const T a0 = a[0], a1 = a[1], a2 = a[2], a3 = a[3];
          const T* b = g->B + k * N + jb;
          for (int64_t j = 0; j < nj; ++j) {
            const T bj = b[j];
            c0[j] += a0 * bj;
            c1[j] += a1 * bj;
            c2[j] += a2 * bj;
            c3[j] += a3 * bj;
          }
        }
      }
      for (; i < i1; ++i) {
        T* c = g->C + i * N + jb;
        for (int64_t k = kb; k < ke; ++k) {
          const T av = g->A[k * M + i];
          const T* b = g->B + k * N + jb;
          for (int64_t j = 0; j < nj; ++j) c[j] += av * b[j];
        }
      }
    }
  }
}
static void gemm_tn(int64_t M, int64_t N, int64_t K, const T* A, const T* B, T* C) {
  gemm_job g = {M, N, K, A, B, C};
  parallel_chunks(M, gemm_threads(M, M * N * K), gemm_tn_rows, &g);
}

/* dictionary_checksum, dictionary.cpp:10-23 */
double S(lm_dictionary_checksum)(const T* atoms, int64_t k, int64_t df, const T* proj, int64_t ds) {
  double s = 0;
  for (int64_t i = 0; i < k * df; ++i) s += (double)atoms[i];
  for (int64_t i = 0; i < ds * df; ++i) s += 3.0 * (double)proj[i];
  return s + (double)k + 17.0 * (double)ds;
}

/* reconstruct, dictionary.cpp:25-53. attention (n x K) optional. */
int S(lm_reconstruct)(const T* q, int64_t n, int64_t ds, const T* atoms, int64_t k, int64_t df,
                      const T* proj, T temperature, T* out, T* attention) {
  if (!(temperature > (T)0)) return -1;
  T* qw = (T*)malloc(sizeof(T) * (size_t)(n * df));
  T* logits = attention ? attention : (T*)malloc(sizeof(T) * (size_t)(n * k));
  gemm_nn(n, df, ds, q, proj, qw);
  gemm_nt(n, k, df, qw, atoms, logits);
  for (int64_t i = 0; i < n * k; ++i) logits[i] = logits[i] / temperature;
  for (int64_t r = 0; r < n; ++r) {
    T* l = logits + r * k;
    T m = l[0];
    for (int64_t j = 1; j < k; ++j)
      if (l[j] > m) m = l[j];
    for (int64_t j = 0; j < k; ++j) l[j] = lm_exp(l[j] - m);
    T sum = 0;
    for (int64_t j = 0; j < k; ++j) sum += l[j];
    for (int64_t j = 0; j < k; ++j) l[j] = l[j] / sum;
  }
  gemm_nn(n, df, k, logits, atoms, out);
  free(qw);
  if (!attention) free(logits);
  return 0;
}

/* reconstruct_backward, dictionary.cpp:55-83 */
int S(lm_reconstruct_backward)(const T* q, const T* attention, int64_t n, int64_t ds,
                               const T* atoms, int64_t k, int64_t df, const T* proj,
                               T temperature, const T* d_rec, T* d_q, T* d_proj, T* d_atoms) {
  T* dl = (T*)malloc(sizeof(T) * (size_t)(n * k));
  gemm_nt(n, k, df, d_rec, atoms, dl);
  for (int64_t r = 0; r < n; ++r) {
    const T* p = attention + r * k;
    T* d = dl + r * k;
    T dot = 0;
    for (int64_t j = 0; j < k; ++j) dot += p[j] * d[j];
    for (int64_t j = 0; j < k; ++j) d[j] = p[j] * (d[j] - dot);
  }
  for (int64_t i = 0; i < n * k; ++i) dl[i] = dl[i] / temperature;
  T* qw = (T*)malloc(sizeof(T) * (size_t)(n * df));
  gemm_nn(n, df, ds, q, proj, qw);
  T* t2 = (T*)malloc(sizeof(T) * (size_t)(k * df));
  gemm_tn(k, df, n, attention, d_rec, d_atoms);
  gemm_tn(k, df, n, dl, qw, t2);
  for (int64_t i = 0; i < k * df; ++i) d_atoms[i] = d_atoms[i] + t2[i];
  T* dqw = qw; /* reuse */
  gemm_nn(n, df, k, dl, atoms, dqw);
  gemm_tn(ds, df, n, q, dqw, d_proj);
  gemm_nt(n, ds, df, dqw, proj, d_q);
  free(dl);
  free(qw);
  free(t2);
  return 0;
}

/* gather_supervision, objective.cpp:7-65. Returns the row count; with NULL outputs it only
 * counts. segment mode averages queries per present assignment row. */
int64_t S(lm_gather_supervision)(const T* query, int h, int w, int ds, const int32_t* assignment,
                                 const T* features, int64_t n_set, int64_t df, int segment_mode,
                                 T* q_out, T* t_out, int64_t* pixel_of_row) {
  const int64_t npx = (int64_t)h * w;
  if (!segment_mode) {
    int64_t r = 0;
    for (int64_t p = 0; p < npx; ++p) {
      int32_t a = assignment[p];
      if (a < 0) continue;
      if (q_out) {
        for (int c = 0; c < ds; ++c) q_out[r * ds + c] = query[p * ds + c];
        memcpy(t_out + r * df, features + (int64_t)a * df, sizeof(T) * (size_t)df);
        if (pixel_of_row) pixel_of_row[r] = p;
      }
      ++r;
    }
    return r;
  }
  int64_t* cnt = (int64_t*)calloc((size_t)n_set, sizeof(int64_t));
  for (int64_t p = 0; p < npx; ++p)
    if (assignment[p] >= 0) cnt[assignment[p]]++;
  int64_t present = 0;
  for (int64_t a = 0; a < n_set; ++a) present += cnt[a] > 0;
  if (q_out) {
    int64_t r = 0;
    for (int64_t a = 0; a < n_set; ++a) {
      if (!cnt[a]) continue;
      T* qr = q_out + r * ds;
      for (int c = 0; c < ds; ++c) qr[c] = 0;
      for (int64_t p = 0; p < npx; ++p)
        if (assignment[p] == a)
          for (int c = 0; c < ds; ++c) qr[c] += query[p * ds + c];
      for (int c = 0; c < ds; ++c) qr[c] /= (T)cnt[a];
      memcpy(t_out + r * df, features + a * df, sizeof(T) * (size_t)df);
      if (pixel_of_row) pixel_of_row[r] = a; /* segment row -> assignment id */
      ++r;
    }
  }
  free(cnt);
  return present;
}

/* total_objective, objective.cpp:67-194 (map/dict gradients zeroed and accumulated here). */
int S(lm_total_objective)(const MAP* map, const T* atoms, const T* anchor, const T* proj,
                          int64_t k, int64_t df, T temperature, const FRAME* frames, int nframes,
                          const lm_intr* intr, const CFG* cfg, int threads, int want_grad,
                          MAP* mg, T* d_proj, T* d_atoms, LOSS* out) {
  if (nframes <= 0) return -1;
  const int h = intr->height, w = intr->width, ds = map->ds;
  const int64_t npx = (int64_t)h * w;
  const T inv_b = (T)1 / (T)nframes;
  memset(out, 0, sizeof(*out));
  if (want_grad) {
    memset(mg->pos, 0, sizeof(T) * (size_t)(map->n * 3));
    memset(mg->rot, 0, sizeof(T) * (size_t)(map->n * 4));
    memset(mg->col, 0, sizeof(T) * (size_t)(map->n * 3));
    memset(mg->lsc, 0, sizeof(T) * (size_t)(map->n * 3));
    memset(mg->opa, 0, sizeof(T) * (size_t)(map->n));
    memset(mg->feat, 0, sizeof(T) * (size_t)(map->n * ds));
    memset(d_proj, 0, sizeof(T) * (size_t)(ds * df));
    memset(d_atoms, 0, sizeof(T) * (size_t)(k * df));
  }
  T* color = (T*)malloc(sizeof(T) * (size_t)npx * 3);
  T* depth = (T*)malloc(sizeof(T) * (size_t)npx);
  T* query = (T*)malloc(sizeof(T) * (size_t)npx * ds);
  T* alpha = (T*)malloc(sizeof(T) * (size_t)npx);
  SPLAT* splats = (SPLAT*)malloc(sizeof(SPLAT) * (size_t)(map->n + 1));
  T* rgb_grad = (T*)malloc(sizeof(T) * (size_t)npx * 3);
  T* dep_grad = (T*)malloc(sizeof(T) * (size_t)npx);
  T* d_query = (T*)malloc(sizeof(T) * (size_t)npx * ds);
  const int want_map_grad = want_grad && cfg->map_grads;
  for (int b = 0; b < nframes; ++b) {
    const FRAME* kf = &frames[b];
    int64_t ns = 0;
    S(lm_render)(map, &kf->pose, intr, threads, color, depth, query, alpha, splats, map->n + 1, &ns);
    T l1, sl, rv, dv;
    int32_t dflag;
    S(lm_rgb_loss)(color, kf->rgb, h, w, 3, cfg->lambda_i1, cfg->lambda_i2, want_map_grad, rgb_grad,
                   &l1, &sl, &rv);
    S(lm_depth_loss)(depth, kf->depth, alpha, npx, want_map_grad, dep_grad, &dv, &dflag);
    const int64_t nsup = S(lm_gather_supervision)(query, h, w, ds, kf->assignment, kf->features,
                                                  kf->n_set, df, cfg->segment_mode, NULL, NULL, NULL);
    T ct = 0, lt = 0, tt = 0, fv = 0;
    int32_t zf = 0;
    T *sq = NULL, *st = NULL, *rec = NULL, *attn = NULL, *drec = NULL, *dat = NULL;
    int64_t* prow = NULL;
    if (nsup > 0) {
      sq = (T*)malloc(sizeof(T) * (size_t)(nsup * ds));
      st = (T*)malloc(sizeof(T) * (size_t)(nsup * df));
      prow = (int64_t*)malloc(sizeof(int64_t) * (size_t)nsup);
      S(lm_gather_supervision)(query, h, w, ds, kf->assignment, kf->features, kf->n_set, df,
                               cfg->segment_mode, sq, st, prow);
      rec = (T*)malloc(sizeof(T) * (size_t)(nsup * df));
      attn = (T*)malloc(sizeof(T) * (size_t)(nsup * k));
      S(lm_reconstruct)(sq, nsup, ds, atoms, k, df, proj, temperature, rec, attn);
      drec = (T*)malloc(sizeof(T) * (size_t)(nsup * df));
      dat = (T*)malloc(sizeof(T) * (size_t)(k * df));
      S(lm_feature_loss)(rec, st, nsup, df, atoms, anchor, k, cfg->trust_delta, cfg->lambda_cos,
                         cfg->lambda_l2, cfg->lambda_trust, want_grad, drec, dat, &ct, &lt, &tt, &fv,
                         &zf);
    }
    out->l_rgb += l1 * inv_b;
    out->l_ssim += sl * inv_b;
    out->l_depth += dv * inv_b;
    out->l_cos += ct * inv_b;
    out->l_l2 += lt * inv_b;
    out->depth_empty = out->depth_empty || dflag;
    out->zero_norm_flagged = out->zero_norm_flagged || zf;
    out->supervised_rows += nsup;
    if (want_grad) {
      int have_dq = 0;
      if (nsup > 0) {
        T* dq = (T*)malloc(sizeof(T) * (size_t)(nsup * ds));
        T* dp = (T*)malloc(sizeof(T) * (size_t)(ds * df));
        T* da = (T*)malloc(sizeof(T) * (size_t)(k * df));
        S(lm_reconstruct_backward)(sq, attn, nsup, ds, atoms, k, df, proj, temperature, drec, dq, dp, da);
        if (cfg->dict_grads) {
          const T sc = cfg->lambda_feat * inv_b;
          for (int64_t i = 0; i < ds * df; ++i) d_proj[i] += sc * dp[i];
          for (int64_t i = 0; i < k * df; ++i) d_atoms[i] += sc * da[i];
        }
        if (cfg->map_grads) {
          memset(d_query, 0, sizeof(T) * (size_t)npx * ds);
          const T scale = cfg->lambda_feat * inv_b;
          if (!cfg->segment_mode) {
            for (int64_t r = 0; r < nsup; ++r)
              for (int c = 0; c < ds; ++c) d_query[prow[r] * ds + c] += scale * dq[r * ds + c];
          } else {
            for (int64_t r = 0; r < nsup; ++r) {
              const int32_t a = (int32_t)prow[r];
              int64_t cnt = 0;
              for (int64_t p = 0; p < npx; ++p) cnt += kf->assignment[p] == a;
              const T per_pix = scale / (T)cnt;
              for (int64_t p = 0; p < npx; ++p)
                if (kf->assignment[p] == a)
                  for (int c = 0; c < ds; ++c) d_query[p * ds + c] += per_pix * dq[r * ds + c];
            }
          }
          have_dq = 1;
        }
        free(dq);
        free(dp);
        free(da);
      }
      if (cfg->map_grads) {
        for (int64_t i = 0; i < npx * 3; ++i) rgb_grad[i] *= cfg->lambda_rgb * inv_b;
        if (!dflag)
          for (int64_t i = 0; i < npx; ++i) dep_grad[i] *= cfg->lambda_depth * inv_b;
        S(lm_render_backward)(map, &kf->pose, intr, splats, ns, rgb_grad, dflag ? NULL : dep_grad,
                              have_dq ? d_query : NULL, threads, mg);
      }
    }
    free(sq);
    free(st);
    free(prow);
    free(rec);
    free(attn);
    free(drec);
    free(dat);
  }
  const T trust = S(lm_trust_region_penalty)(atoms, anchor, k, df, cfg->trust_delta, NULL);
  out->l_trust = trust;
  if (want_grad && cfg->dict_grads) {
    T* tg = (T*)malloc(sizeof(T) * (size_t)(k * df));
    S(lm_trust_region_penalty)(atoms, anchor, k, df, cfg->trust_delta, tg);
    const T sc = cfg->lambda_feat * cfg->lambda_trust;
    for (int64_t i = 0; i < k * df; ++i) d_atoms[i] += sc * tg[i];
    free(tg);
  }
  out->total = cfg->lambda_rgb * (cfg->lambda_i1 * out->l_rgb + cfg->lambda_i2 * out->l_ssim) +
               cfg->lambda_depth * out->l_depth +
               cfg->lambda_feat * (cfg->lambda_cos * out->l_cos + cfg->lambda_l2 * out->l_l2 +
                                   cfg->lambda_trust * out->l_trust);
  free(color);
  free(depth);
  free(query);
  free(alpha);
  free(splats);
  free(rgb_grad);
  free(dep_grad);
  free(d_query);
  return 0;
}

/* adam_step, obj/adam.hpp:61-79 (beta1 0.9, beta2 0.999, eps 1e-8; moments pre-sized). */
int S(lm_adam_step)(T* param, const T* grad, T* m, T* v, int64_t count, int64_t* step,
                    int64_t* skipped, T lr) {
  for (int64_t i = 0; i < count; ++i)
    if (!isfinite((double)grad[i])) {
      ++*skipped;
      return 0;
    }
  ++*step;
  const T b1 = (T)0.9, b2 = (T)0.999;
  for (int64_t i = 0; i < count; ++i) {
    m[i] = b1 * m[i] + ((T)1 - b1) * grad[i];
    v[i] = b2 * v[i] + ((T)1 - b2) * (grad[i] * grad[i]);
  }
  const T corr1 = (T)1 - (T)pow(0.9, (double)*step);
  const T corr2 = (T)1 - (T)pow(0.999, (double)*step);
  for (int64_t i = 0; i < count; ++i)
    param[i] -= lr * (m[i] / corr1) / (lm_sqrt(v[i] / corr2) + (T)1e-8);
  return 1;
}

/* quaternion renormalisation after the rotation step, pipeline.cpp:78-84 */
void S(lm_renorm_quats)(T* rot, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    T* q = rot + 4 * i;
    const T nn = lm_sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    if (nn > (T)1e-12f) {
      for (int c = 0; c < 4; ++c) q[c] = q[c] / nn;
    } else {
      q[0] = 1;
      q[1] = q[2] = q[3] = 0;
    }
  }
}


/* ------------------------------------------------------------------ streaming k-means */

/* assign_nearest, stream_kmeans.cpp:11-36: score = P C^T (ascending inner index),
 * d = |c|^2 - 2 score, ties to the lower center index. */
static void S(km_assign)(const T* P, int64_t n, int64_t dim, const T* C, int64_t k, int64_t* asg) {
  if (k == 0) {
    for (int64_t r = 0; r < n; ++r) asg[r] = 0;
    return;
  }
  T* c2 = (T*)malloc(sizeof(T) * (size_t)k);
  for (int64_t j = 0; j < k; ++j) {
    T s = 0;
    for (int64_t d = 0; d < dim; ++d) s += C[j * dim + d] * C[j * dim + d];
    c2[j] = s;
  }
  for (int64_t r = 0; r < n; ++r) {
    T best = 0;
    int64_t bj = 0;
    for (int64_t j = 0; j < k; ++j) {
      T sc = 0;
      for (int64_t d = 0; d < dim; ++d) sc += P[r * dim + d] * C[j * dim + d];
      const T dd = c2[j] - (T)2 * sc;
      if (j == 0 || dd < best) {
        best = dd;
        bj = j;
      }
    }
    asg[r] = bj;
  }
  free(c2);
}

/* update_min_dist, stream_kmeans.cpp:38-45 */
static void S(km_update_min)(const T* P, int64_t n, int64_t dim, const T* c, T* min_d2) {
  for (int64_t i = 0; i < n; ++i) {
    T d = 0;
    for (int64_t e = 0; e < dim; ++e) {
      const T t = P[i * dim + e] - c[e];
      d += t * t;
    }
    if (d < min_d2[i]) min_d2[i] = d;
  }
}

/* kmeanspp_fill, stream_kmeans.cpp:48-90: weighted k-means++ continuation of rows [filled, k). */
static void S(km_pp_fill)(const T* P, const T* W, int64_t n, int64_t dim, T* centers, int64_t k,
                          int64_t filled, double (*uni)(void*), void* rng) {
  T* min_d2 = (T*)malloc(sizeof(T) * (size_t)n);
  uint8_t* used = (uint8_t*)calloc((size_t)n, 1);
  for (int64_t i = 0; i < n; ++i) min_d2[i] = LM_DOUBLE ? (T)1.7976931348623157e308 : (T)3.40282346638528859812e+38F;
  for (int64_t j = 0; j < filled; ++j) S(km_update_min)(P, n, dim, centers + j * dim, min_d2);
  for (int64_t j = filled; j < k; ++j) {
    double total = 0;
    for (int64_t i = 0; i < n; ++i) {
      double p = (double)W[i];
      if (j > 0 || filled > 0) p *= (double)min_d2[i];
      total += p;
    }
    int64_t pick = -1;
    if (total > 0) {
      const double target = uni(rng) * total;
      double run = 0;
      for (int64_t i = 0; i < n; ++i) {
        double p = (double)W[i];
        if (j > 0 || filled > 0) p *= (double)min_d2[i];
        run += p;
        if (run >= target) {
          pick = i;
          break;
        }
      }
      if (pick < 0) pick = n - 1;
    } else {
      for (int64_t i = 0; i < n; ++i)
        if (!used[i]) {
          pick = i;
          break;
        }
      if (pick < 0) pick = (j - filled) % n;
    }
    used[pick] = 1;
    memcpy(centers + j * dim, P + pick * dim, sizeof(T) * (size_t)dim);
    S(km_update_min)(P, n, dim, centers + j * dim, min_d2);
  }
  free(min_d2);
  free(used);
}

/* weighted_kmeans, stream_kmeans.cpp:94-157 */
int S(lm_weighted_kmeans)(const T* P, const T* W, int64_t n, int64_t dim, int64_t k, double (*uni)(void*),
                          void* rng, const T* warm, int64_t n_warm, int max_iters, T* centers, T* cw,
                          int* iterations) {
  if (k < 1) return -1;
  memset(centers, 0, sizeof(T) * (size_t)(k * dim));
  for (int64_t j = 0; j < k; ++j) cw[j] = 0;
  *iterations = 0;
  if (n == 0) return 0;
  int64_t filled = 0;
  if (warm) {
    filled = k < n_warm ? k : n_warm;
    memcpy(centers, warm, sizeof(T) * (size_t)(filled * dim));
  }
  S(km_pp_fill)(P, W, n, dim, centers, k, filled, uni, rng);
  int64_t* asg = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* prev = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  uint8_t* claimed = (uint8_t*)calloc((size_t)n, 1);
  T* mass = (T*)malloc(sizeof(T) * (size_t)k);
  T* sums = (T*)malloc(sizeof(T) * (size_t)(k * dim));
  for (int it = 0; it < max_iters; ++it) {
    S(km_assign)(P, n, dim, centers, k, asg);
    for (int64_t j = 0; j < k; ++j) mass[j] = 0;
    memset(sums, 0, sizeof(T) * (size_t)(k * dim));
    for (int64_t i = 0; i < n; ++i) {
      mass[asg[i]] += W[i];
      for (int64_t e = 0; e < dim; ++e) sums[asg[i] * dim + e] += W[i] * P[i * dim + e];
    }
    int reseeded = 0;
    for (int64_t j = 0; j < k; ++j) {
      if (mass[j] > (T)0) {
        for (int64_t e = 0; e < dim; ++e) centers[j * dim + e] = sums[j * dim + e] / mass[j];
      } else {
        int64_t pick = -1;
        T best = (T)-1;
        for (int64_t i = 0; i < n; ++i)
          if (!claimed[i] && W[i] > best) {
            best = W[i];
            pick = i;
          }
        if (pick >= 0) {
          claimed[pick] = 1;
          memcpy(centers + j * dim, P + pick * dim, sizeof(T) * (size_t)dim);
          reseeded = 1;
        }
      }
    }
    *iterations = it + 1;
    if (!reseeded && it > 0 && memcmp(asg, prev, sizeof(int64_t) * (size_t)n) == 0) break;
    memcpy(prev, asg, sizeof(int64_t) * (size_t)n);
  }
  S(km_assign)(P, n, dim, centers, k, asg);
  for (int64_t j = 0; j < k; ++j) cw[j] = 0;
  for (int64_t i = 0; i < n; ++i) cw[asg[i]] += W[i];
  free(asg);
  free(prev);
  free(claimed);
  free(mass);
  free(sums);
  return 0;
}

/* stream_kmeans_update, stream_kmeans.cpp:159-196 (state = atoms / anchor / weights, K rows). */
int S(lm_stream_kmeans_update)(const T* batch, int64_t n, int64_t dim, T* atoms, T* anchor, T* weights, int64_t k,
                               double (*uni)(void*), void* rng, T decay) {
  if (n == 0) return 0;
  const int64_t m = n < k ? n : k;
  T* unit = (T*)malloc(sizeof(T) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) unit[i] = (T)1;
  T* lc = (T*)malloc(sizeof(T) * (size_t)(m * dim));
  T* lw = (T*)malloc(sizeof(T) * (size_t)m);
  int iters = 0;
  S(lm_weighted_kmeans)(batch, unit, n, dim, m, uni, rng, NULL, 0, 10, lc, lw, &iters);
  int64_t old_count = 0;
  for (int64_t j = 0; j < k; ++j)
    if (weights[j] > (T)0) ++old_count;
  T* pooled = (T*)malloc(sizeof(T) * (size_t)((m + old_count) * dim));
  T* pw = (T*)malloc(sizeof(T) * (size_t)(m + old_count));
  T* warm = (T*)malloc(sizeof(T) * (size_t)((old_count > 0 ? old_count : 1) * dim));
  memcpy(pooled, lc, sizeof(T) * (size_t)(m * dim));
  memcpy(pw, lw, sizeof(T) * (size_t)m);
  int64_t at = 0;
  for (int64_t j = 0; j < k; ++j) {
    if (weights[j] > (T)0) {
      memcpy(pooled + (m + at) * dim, atoms + j * dim, sizeof(T) * (size_t)dim);
      pw[m + at] = weights[j] * decay;
      memcpy(warm + at * dim, atoms + j * dim, sizeof(T) * (size_t)dim);
      ++at;
    }
  }
  S(lm_weighted_kmeans)(pooled, pw, m + old_count, dim, k, uni, rng, old_count > 0 ? warm : NULL, old_count, 10,
                        atoms, weights, &iters);
  memcpy(anchor, atoms, sizeof(T) * (size_t)(k * dim));
  free(unit);
  free(lc);
  free(lw);
  free(pooled);
  free(pw);
  free(warm);
  return 0;
}

#else /* LM_ONCE: voxel hash store, voxel_hash.cpp / active_set.cpp */
/* libm expf (what the reference's std::exp(float) calls) of the floats with bit patterns
 * first .. first + n - 1, split over threads: the checker of the device's restated expf. */
typedef struct {
  uint64_t first;
  float* out;
} expf_job;
typedef struct {
  void (*fn)(void*, int64_t, int64_t, int);
  void* ctx;
  int64_t b, e;
  int tid;
} once_job;
static void* once_tramp(void* p) {
  once_job* j = (once_job*)p;
  j->fn(j->ctx, j->b, j->e, j->tid);
  return NULL;
}
static void parallel_chunks_once(int64_t total, int threads, void (*fn)(void*, int64_t, int64_t, int), void* ctx) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  once_job jobs[256];
  const int64_t chunk = (total + threads - 1) / threads;
  int nt = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t b = t * chunk, e = b + chunk < total ? b + chunk : total;
    if (b >= e) break;
    jobs[nt] = (once_job){fn, ctx, b, e, t};
    pthread_create(&th[nt], NULL, once_tramp, &jobs[nt]);
    ++nt;
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}
static void expf_chunk(void* pc, int64_t b, int64_t e, int tid) {
  const expf_job* j = (const expf_job*)pc;
  for (int64_t i = b; i < e; ++i) {
    const uint32_t u = (uint32_t)(j->first + (uint64_t)i);
    float x;
    memcpy(&x, &u, 4);
    j->out[i] = expf(x);
  }
}
void lm_expf_bits(uint64_t first, int64_t n, float* out, int threads) {
  expf_job j = {first, out};
  parallel_chunks_once(n, threads, expf_chunk, &j);
}
int lm_oracle_gemm_threads_value = 1;
void lm_oracle_set_gemm_threads(int n) { lm_oracle_gemm_threads_value = n < 1 ? 1 : (n > 256 ? 256 : n); }

/* ------------------------------------------------------------------ evaluation metrics */
static float lmo_dot(const float* a, const float* b, int64_t d) {
  float s = 0.f;
  for (int64_t i = 0; i < d; ++i) s += a[i] * b[i];
  return s;
}

/* metric_cos, metrics.cpp:8-24: float row norms / dot (Eigen on float rows), double mean. */
double lm_metric_cos(const float* rec, const float* tgt, int64_t n, int64_t d, int32_t* flagged) {
  if (flagged) *flagged = 0;
  if (n == 0) return 0.0;
  double sum = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    double nu = (double)sqrtf(lmo_dot(rec + r * d, rec + r * d, d));
    double nv = (double)sqrtf(lmo_dot(tgt + r * d, tgt + r * d, d));
    if ((nu < 1e-8 || nv < 1e-8) && flagged) *flagged = 1;
    nu = nu > 1e-8 ? nu : 1e-8;
    nv = nv > 1e-8 ? nv : 1e-8;
    sum += 1.0 - (double)lmo_dot(rec + r * d, tgt + r * d, d) / (nu * nv);
  }
  return sum / (double)n;
}

/* metric_miou, metrics.cpp:26-73: softmax over prototype scores (float; exp correctly rounded),
 * prediction = first maximum of the probabilities; classes absent from both are excluded. */
double lm_metric_miou(const float* emb, const int32_t* labels, int64_t n, int64_t d, const float* protos, int64_t c,
                      int64_t* inter, int64_t* uni) {
  for (int64_t k = 0; k < c; ++k) inter[k] = uni[k] = 0;
  float* sc = (float*)malloc(sizeof(float) * (size_t)(c > 0 ? c : 1));
  for (int64_t i = 0; i < n; ++i) {
    const int32_t gt = labels[i];
    if (gt < 0) continue;
    if (gt >= c) {
      free(sc);
      return -1.0;
    }
    float m = 0.f;
    for (int64_t k = 0; k < c; ++k) {
      sc[k] = lmo_dot(protos + k * d, emb + i * d, d);
      if (k == 0 || sc[k] > m) m = sc[k];
    }
    float s = 0.f;
    for (int64_t k = 0; k < c; ++k) {
      sc[k] = expf(sc[k] - m);
      s += sc[k];
    }
    int64_t pred = 0;
    float best = 0.f;
    for (int64_t k = 0; k < c; ++k) {
      const float p = sc[k] / s;
      if (k == 0 || p > best) best = p, pred = k;
    }
    if (pred == gt) {
      ++inter[gt];
      ++uni[gt];
    } else {
      ++uni[gt];
      ++uni[pred];
    }
  }
  free(sc);
  double sum = 0.0;
  int64_t inc = 0;
  for (int64_t k = 0; k < c; ++k) {
    if (uni[k] == 0) continue;
    sum += (double)inter[k] / (double)uni[k];
    ++inc;
  }
  return inc > 0 ? sum / (double)inc : 0.0;
}

/* metric_psnr, metrics.cpp:75-89 */
double lm_metric_psnr(const float* a, const float* b, int64_t n, int32_t* exact) {
  double mse = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double dd = (double)a[i] - (double)b[i];
    mse += dd * dd;
  }
  mse /= (double)n;
  if (mse == 0.0) {
    if (exact) *exact = 1;
    return 100.0;
  }
  if (exact) *exact = 0;
  return 10.0 * log10(1.0 / mse);
}

/* query_map, evaluate.cpp:74-88 (scores of reconstructed rows vs one embedding) */
void lm_query_scores(const float* rec, int64_t n, int64_t d, const float* emb, float* scores) {
  float qn = sqrtf(lmo_dot(emb, emb, d));
  qn = qn > 1e-8f ? qn : 1e-8f;
  for (int64_t i = 0; i < n; ++i) {
    float rn = sqrtf(lmo_dot(rec + i * d, rec + i * d, d));
    rn = rn > 1e-8f ? rn : 1e-8f;
    scores[i] = lmo_dot(rec + i * d, emb, d) / (rn * qn);
  }
}


/* ------------------------------------------------------------------ std::mt19937_64 */
/* The 64-bit Mersenne Twister with the C++ standard's parameters ([rand.predef]:
 * w=64 n=312 m=156 r=31 a=0xb5026f5aa96619e9 u=29 d=0x5555555555555555 s=17
 * b=0x71d67fffeda60000 t=37 c=0xfff7eee000000000 l=43 f=6364136223846793005). */
void lm_mt64_seed(lm_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t lm_mt64_next(lm_mt64* r) {
  if (r->idx >= 312) {
    const uint64_t lower = (1ULL << 31) - 1, upper = ~lower;
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xb5026f5aa96619e9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71d67fffeda60000ULL;
  y ^= (y << 37) & 0xfff7eee000000000ULL;
  y ^= y >> 43;
  return y;
}

/* std::uniform_real_distribution<double>(0, 1) over mt19937_64 with libstdc++'s
 * generate_canonical<double, 53>: one draw (53 <= 64 bits), (double)x / 2^64, values that
 * round to 1 clamp to nextafter(1, 0); then a + (b - a) * u with a = 0, b = 1. */
double lm_mt64_uniform01(void* rp) {
  const double sum = (double)lm_mt64_next((lm_mt64*)rp);
  double ret = sum / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret * (1.0 - 0.0) + 0.0;
}



#define PROBE_LIMIT 8

/* voxel_of, voxel_hash.cpp:9-16 */
lm_voxel_key lm_voxel_of(const float p[3], float voxel_size) {
  lm_voxel_key k;
  k.ix = (int32_t)floor((double)p[0] / (double)voxel_size);
  k.iy = (int32_t)floor((double)p[1] / (double)voxel_size);
  k.iz = (int32_t)floor((double)p[2] / (double)voxel_size);
  return k;
}

/* hash_voxel, voxel_hash.cpp:18-23 */
int64_t lm_hash_voxel(lm_voxel_key v, int64_t capacity) {
  if (capacity <= 0) return -1;
  const uint32_t h = ((uint32_t)v.ix * 73856093u) ^ ((uint32_t)v.iy * 19349663u) ^
                     ((uint32_t)v.iz * 83492791u);
  return (int64_t)((uint64_t)h % (uint64_t)capacity);
}

typedef struct {
  int64_t record;
  lm_voxel_key key;
} slot_t;

struct lm_store {
  int64_t capacity;
  int32_t ds, rs;
  slot_t* slots;
  float* pool;
  lm_voxel_key* keys;
  int64_t size, pool_cap;
  int64_t stats[5]; /* inserted, updated, rejected_duplicate, rejected_overflow, probe_steps */
};

lm_store* lm_store_create(int64_t capacity, int32_t query_dim) {
  if (capacity <= 0) return NULL;
  lm_store* s = (lm_store*)calloc(1, sizeof(lm_store));
  s->capacity = capacity;
  s->ds = query_dim;
  s->rs = 14 + query_dim;
  s->slots = (slot_t*)malloc(sizeof(slot_t) * (size_t)capacity);
  for (int64_t i = 0; i < capacity; ++i) s->slots[i].record = -1;
  return s;
}
void lm_store_destroy(lm_store* s) {
  if (!s) return;
  free(s->slots);
  free(s->pool);
  free(s->keys);
  free(s);
}
static int key_eq(lm_voxel_key a, lm_voxel_key b) { return a.ix == b.ix && a.iy == b.iy && a.iz == b.iz; }

/* VoxelHashStore::probe, voxel_hash.cpp:35-50 */
static int64_t probe(const lm_store* cs, lm_voxel_key key, int for_insert, int64_t* free_slot) {
  lm_store* s = (lm_store*)cs;
  if (free_slot) *free_slot = -1;
  const int64_t start = lm_hash_voxel(key, s->capacity);
  const int limit = (int)(s->capacity < PROBE_LIMIT ? s->capacity : PROBE_LIMIT);
  for (int i = 0; i < limit; ++i) {
    const int64_t sl = (start + i) % s->capacity;
    const slot_t* slot = &s->slots[sl];
    ++s->stats[4];
    if (slot->record < 0) {
      if (for_insert && free_slot && *free_slot < 0) *free_slot = sl;
      return -1;
    }
    if (key_eq(slot->key, key)) return sl;
  }
  return -1;
}

/* VoxelHashStore::insert, voxel_hash.cpp:52-71 */
int64_t lm_store_insert(lm_store* s, lm_voxel_key key, const float* rec) {
  int64_t free_slot = -1;
  const int64_t hit = probe(s, key, 1, &free_slot);
  if (hit >= 0) {
    ++s->stats[2];
    return -1;
  }
  if (free_slot < 0) {
    ++s->stats[3];
    return -1;
  }
  if (s->size == s->pool_cap) {
    s->pool_cap = s->pool_cap ? s->pool_cap * 2 : 1024;
    s->pool = (float*)realloc(s->pool, sizeof(float) * (size_t)(s->pool_cap * s->rs));
    s->keys = (lm_voxel_key*)realloc(s->keys, sizeof(lm_voxel_key) * (size_t)s->pool_cap);
  }
  memcpy(s->pool + s->size * s->rs, rec, sizeof(float) * (size_t)s->rs);
  s->keys[s->size] = key;
  s->slots[free_slot].record = s->size;
  s->slots[free_slot].key = key;
  ++s->stats[0];
  return s->size++;
}
/* VoxelHashStore::update, voxel_hash.cpp:73-79 */
int32_t lm_store_update(lm_store* s, lm_voxel_key key, const float* rec) {
  const int64_t hit = probe(s, key, 0, NULL);
  if (hit < 0) return 0;
  memcpy(s->pool + s->slots[hit].record * s->rs, rec, sizeof(float) * (size_t)s->rs);
  ++s->stats[1];
  return 1;
}
/* VoxelHashStore::find, voxel_hash.cpp:81-84 */
int64_t lm_store_find(const lm_store* s, lm_voxel_key key) {
  const int64_t hit = probe(s, key, 0, NULL);
  return hit < 0 ? -1 : s->slots[hit].record;
}
int64_t lm_store_size(const lm_store* s) { return s->size; }
static int key_cmp(const void* pa, const void* pb) {
  const lm_voxel_key* a = (const lm_voxel_key*)pa;
  const lm_voxel_key* b = (const lm_voxel_key*)pb;
  if (a->ix != b->ix) return a->ix < b->ix ? -1 : 1;
  if (a->iy != b->iy) return a->iy < b->iy ? -1 : 1;
  return (a->iz > b->iz) - (a->iz < b->iz);
}
/* check_unique_keys, voxel_hash.cpp:86-99 */
int32_t lm_store_check_unique_keys(const lm_store* s) {
  lm_voxel_key* occ = (lm_voxel_key*)malloc(sizeof(lm_voxel_key) * (size_t)(s->size + 1));
  int64_t n = 0;
  for (int64_t i = 0; i < s->capacity; ++i)
    if (s->slots[i].record >= 0) occ[n++] = s->slots[i].key;
  qsort(occ, (size_t)n, sizeof(lm_voxel_key), key_cmp);
  int ok = 1;
  for (int64_t i = 1; i < n; ++i)
    if (key_eq(occ[i], occ[i - 1])) ok = 0;
  free(occ);
  return ok;
}
void lm_store_get_record(const lm_store* s, int64_t index, float* rec) {
  memcpy(rec, s->pool + index * s->rs, sizeof(float) * (size_t)s->rs);
}
void lm_store_set_record(lm_store* s, int64_t index, const float* rec) {
  memcpy(s->pool + index * s->rs, rec, sizeof(float) * (size_t)s->rs);
}
lm_voxel_key lm_store_record_key(const lm_store* s, int64_t index) { return s->keys[index]; }
void lm_store_stats(const lm_store* s, int64_t out[5]) { memcpy(out, s->stats, sizeof(s->stats)); }

/* insert_global, voxel_hash.cpp:101-115 */
int64_t lm_insert_global(lm_store* s, const float* recs, int64_t n, float voxel_size) {
  int64_t ins = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float* r = recs + i * s->rs;
    ins += lm_store_insert(s, lm_voxel_of(r, voxel_size), r) >= 0;
  }
  return ins;
}

static inline int in_radius(const float* p, const float c[3], float r2) {
  const float dx = p[0] - c[0];
  const float dy = p[1] - c[1];
  const float dz = p[2] - c[2];
  return dx * dx + dy * dy + dz * dz <= r2;
}

/* fetch_local, active_set.cpp:7-36 */
int64_t lm_fetch_local(const lm_store* s, const float center[3], float radius, int64_t* origin,
                       int64_t cap) {
  if (!(radius > 0)) return -1;
  const float r2 = radius * radius;
  int64_t n = 0;
  for (int64_t i = 0; i < s->size; ++i)
    if (in_radius(s->pool + i * s->rs, center, r2)) {
      if (n >= cap) return -2;
      origin[n++] = i;
    }
  return n;
}

/* sync, active_set.cpp:38-128 */
int64_t lm_sync(lm_store* s, const float* active, const int64_t* origin, const uint8_t* dirty,
                int64_t n, const float center[3], float radius, float voxel_size, float* out_recs,
                int64_t* out_origin, int64_t cap, uint8_t* kept_mask, int64_t stats[5]) {
  const int rs = s->rs;
  memset(stats, 0, sizeof(int64_t) * 5);
  if (kept_mask) memset(kept_mask, 0, (size_t)n);
  int64_t* resolved = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) {
    const float* g = active + i * rs;
    resolved[i] = -1;
    if (origin[i] >= 0) {
      resolved[i] = origin[i];
      if (dirty[i]) {
        lm_store_set_record(s, origin[i], g);
        ++stats[0];
      }
    } else {
      const int64_t rec = lm_store_insert(s, lm_voxel_of(g, voxel_size), g);
      if (rec >= 0) {
        resolved[i] = rec;
        ++stats[1];
      } else {
        ++stats[2];
      }
    }
  }
  uint8_t* present = (uint8_t*)calloc((size_t)(s->size + 1), 1);
  const float r2 = radius * radius;
  int64_t w = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (resolved[i] < 0) continue;
    if (in_radius(active + i * rs, center, r2)) {
      if (w >= cap) return -1;
      memcpy(out_recs + w * rs, active + i * rs, sizeof(float) * (size_t)rs);
      out_origin[w++] = resolved[i];
      present[resolved[i]] = 1;
      if (kept_mask) kept_mask[i] = 1;
    } else {
      ++stats[3];
    }
  }
  for (int64_t rec = 0; rec < s->size; ++rec) {
    if (present[rec]) continue;
    if (in_radius(s->pool + rec * rs, center, r2)) {
      if (w >= cap) return -1;
      memcpy(out_recs + w * rs, s->pool + rec * rs, sizeof(float) * (size_t)rs);
      out_origin[w++] = rec;
      ++stats[4];
    }
  }
  free(resolved);
  free(present);
  return w;
}

#endif
