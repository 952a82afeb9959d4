// losses.cu — image-space losses (K5): L1 RGB, masked depth L1, SSIM forward + adjoint.
// Replaces rgb_loss / depth_loss / ssim (proj/src/losses.cpp:133-255).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace lm {

namespace {

constexpr int kWin = 11, kRad = 5;

struct SsimKernel {
  float k[kWin];
};

// ssim_kernel, losses.cpp:13-25 (double weights rounded to float, then normalised).
SsimKernel make_kernel() {
  SsimKernel s;
  double w[kWin], sum = 0;
  for (int i = 0; i < kWin; ++i) {
    const double d = i - kRad;
    w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
    s.k[i] = (float)w[i];
    sum += w[i];
  }
  for (int i = 0; i < kWin; ++i) s.k[i] = (float)((double)s.k[i] / sum);
  return s;
}

__device__ __forceinline__ int refl(int i, int n) {
  if (i < 0) return -i;
  if (i >= n) return 2 * n - 2 - i;
  return i;
}

__device__ __forceinline__ void block_add_double(double v, double* out) {
  __shared__ double s_red[32];
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? s_red[lane] : 0.0;
    v = warp_sum_d(v);
    if (lane == 0 && v != 0.0) atomicAdd(out, v);
  }
  __syncthreads();
}

// Pass 1: L1 RGB (losses.cpp:200-214) and masked depth L1 (losses.cpp:226-255).
__global__ void __launch_bounds__(256) l1_depth_kernel(const float* __restrict__ color, const float* __restrict__ depth,
                                                       const float* __restrict__ alpha, const float* __restrict__ rgb_t,
                                                       const float* __restrict__ depth_t, int64_t npx, float lambda_i1,
                                                       float n_rgb, bool want_grad, float* d_color, float* d_depth,
                                                       double* partials) {
  double l1 = 0.0, dsum = 0.0, dcount = 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float d = fs(color[3 * p + c], rgb_t[3 * p + c]);
      l1 += (double)fabsf(d);
      if (want_grad) {
        const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        d_color[3 * p + c] = fd(fm(lambda_i1, sg), n_rgb);
      }
    }
    const float o = depth_t[p];
    const bool valid = o > 0.f && alpha[p] > 0.5f;
    float sg = 0.f;
    if (valid) {
      const float d = fs(depth[p], o);
      dsum += (double)fabsf(d);
      dcount += 1.0;
      sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    }
    if (want_grad) d_depth[p] = sg;
  }
  block_add_double(l1, &partials[0]);
  block_add_double(dsum, &partials[2]);
  block_add_double(dcount, &partials[3]);
}

// Pass 1, four pixels per thread (16-byte loads and stores; npx % 4 == 0, aligned buffers). With
// fold_color the objective weight is applied here with the same two roundings finalize applies
// (objective.cpp:164-165), so d_color is final and finalize only touches d_depth.
__global__ void __launch_bounds__(256) l1_depth4_kernel(const float4* __restrict__ color, const float4* __restrict__ depth,
                                                        const float4* __restrict__ alpha, const float4* __restrict__ rgb_t,
                                                        const float4* __restrict__ depth_t, int64_t n4, float lambda_i1,
                                                        float n_rgb, bool want_grad, bool fold_color, float rgb_scale,
                                                        float4* d_color, float4* d_depth, double* partials) {
  double l1 = 0.0, dsum = 0.0, dcount = 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n4; p += (int64_t)gridDim.x * blockDim.x) {
    const float4 c0 = color[3 * p], c1 = color[3 * p + 1], c2 = color[3 * p + 2];
    const float4 t0 = rgb_t[3 * p], t1 = rgb_t[3 * p + 1], t2 = rgb_t[3 * p + 2];
    const float4 dp = depth[p], al = alpha[p], dt = depth_t[p];
    const float cv[12] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, c2.x, c2.y, c2.z, c2.w};
    const float tv[12] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w, t2.x, t2.y, t2.z, t2.w};
    float g[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const float d = fs(cv[i], tv[i]);
      l1 += (double)fabsf(d);
      const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
      g[i] = fd(fm(lambda_i1, sg), n_rgb);
      if (fold_color) g[i] = fm(g[i], rgb_scale);
    }
    const float dv[4] = {dp.x, dp.y, dp.z, dp.w}, av[4] = {al.x, al.y, al.z, al.w}, ov[4] = {dt.x, dt.y, dt.z, dt.w};
    float gd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float o = ov[j];
      const bool valid = o > 0.f && av[j] > 0.5f;
      float sg = 0.f;
      if (valid) {
        const float d = fs(dv[j], o);
        dsum += (double)fabsf(d);
        dcount += 1.0;
        sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
      }
      gd[j] = sg;
    }
    if (want_grad) {
      d_color[3 * p] = make_float4(g[0], g[1], g[2], g[3]);
      d_color[3 * p + 1] = make_float4(g[4], g[5], g[6], g[7]);
      d_color[3 * p + 2] = make_float4(g[8], g[9], g[10], g[11]);
      d_depth[p] = make_float4(gd[0], gd[1], gd[2], gd[3]);
    }
  }
  block_add_double(l1, &partials[0]);
  block_add_double(dsum, &partials[2]);
  block_add_double(dcount, &partials[3]);
}

// d_depth only (d_color already final): four pixels per thread.
__global__ void finalize_depth4_kernel(float4* d_depth, int64_t n4, float depth_scale, const double* partials) {
  const double valid = partials[3];
  const float fv = (float)valid;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n4; p += (int64_t)gridDim.x * blockDim.x) {
    float4 v = d_depth[p];
    if (valid > 0.0) {
      v.x = fm(fd(v.x, fv), depth_scale), v.y = fm(fd(v.y, fv), depth_scale);
      v.z = fm(fd(v.z, fv), depth_scale), v.w = fm(fd(v.w, fv), depth_scale);
    } else {
      v = make_float4(0.f, 0.f, 0.f, 0.f);  // depth flagged: no gradient (objective.cpp:165-169)
    }
    d_depth[p] = v;
  }
}

// Fold the objective weights into the upstream images (objective.cpp:164-170).
__global__ void finalize_upstream_kernel(float* d_color, float* d_depth, int64_t npx, float rgb_scale,
                                         float depth_scale, const double* partials) {
  const double valid = partials[3];
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 3; ++c) d_color[3 * p + c] = fm(d_color[3 * p + c], rgb_scale);
    if (valid > 0.0)
      d_depth[p] = fm(fd(d_depth[p], (float)valid), depth_scale);
    else
      d_depth[p] = 0.f;  // depth flagged: no gradient (objective.cpp:165-169)
  }
}

// SSIM, horizontal pass: 5 filtered quantities per channel (filter_plane, losses.cpp:34-54).
__global__ void ssim_h_kernel(const float* __restrict__ a, const float* __restrict__ b, int h, int w, int ch,
                              SsimKernel K, float* __restrict__ hq) {
  const int64_t n = (int64_t)h * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * ch; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const int64_t p = e % n;
    const int y = (int)(p / w), x = (int)(p % w);
    float s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
    for (int k = -kRad; k <= kRad; ++k) {
      const int64_t q = ((int64_t)y * w + refl(x + k, w)) * ch + c;
      const float av = a[q], bv = b[q], kw = K.k[k + kRad];
      s0 += kw * av;
      s1 += kw * bv;
      s2 += kw * (av * av);
      s3 += kw * (bv * bv);
      s4 += kw * (av * bv);
    }
    float* o = hq + (int64_t)c * 5 * n;
    o[p] = s0;
    o[n + p] = s1;
    o[2 * n + p] = s2;
    o[3 * n + p] = s3;
    o[4 * n + p] = s4;
  }
}

// SSIM, vertical pass + per-pixel map and its adjoint seeds (losses.cpp:161-177).
__global__ void __launch_bounds__(256) ssim_v_kernel(const float* __restrict__ hq, int h, int w, int ch, SsimKernel K,
                                                     bool grad, float* __restrict__ seeds, double* sum_out) {
  const float c1 = 0.01f * 0.01f, c2 = 0.03f * 0.03f;
  const int64_t n = (int64_t)h * w;
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * ch; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const int64_t p = e % n;
    const int y = (int)(p / w), x = (int)(p % w);
    const float* in = hq + (int64_t)c * 5 * n;
    float q[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = -kRad; k <= kRad; ++k) {
      const int64_t r = (int64_t)refl(y + k, h) * w + x;
      const float kw = K.k[k + kRad];
#pragma unroll
      for (int t = 0; t < 5; ++t) q[t] += kw * in[t * n + r];
    }
    const float mx = q[0], my = q[1];
    const float sx2 = q[2] - mx * mx, sy2 = q[3] - my * my, sxy = q[4] - mx * my;
    const float a1 = 2.f * mx * my + c1, a2 = 2.f * sxy + c2;
    const float b1 = mx * mx + my * my + c1, b2 = sx2 + sy2 + c2;
    const float s = (a1 * a2) / (b1 * b2);
    acc += (double)s;
    if (grad) {
      float* sd = seeds + (int64_t)c * 3 * n;
      sd[p] = 2.f * my * (a2 - a1) / (b1 * b2) - s * 2.f * mx / b1 + s * 2.f * mx / b2;
      sd[n + p] = -s / b2;
      sd[2 * n + p] = 2.f * a1 / (b1 * b2);
    }
  }
  block_add_double(acc, sum_out);
}

// SSIM value only (no gradient requested): both separable passes fused per 32x16 output tile
// with a 5-pixel reflect-101 halo in shared memory, one channel at a time. Each thread slides the
// 11-tap window over 4 consecutive outputs (horizontal: a row segment, vertical: a column
// segment), loading each input once; every output keeps the float expressions and the tap order
// of ssim_h_kernel + ssim_v_kernel (so the same values).
constexpr int kSTX = 32, kSTY = 16, kSHX = kSTX + 2 * kRad, kSHY = kSTY + 2 * kRad;
constexpr int kSOut = 4;  // horizontal outputs per thread
constexpr int kVOut = kSTY / 8;  // vertical outputs per thread (256 threads = 32 columns x 8 segments)
__global__ void __launch_bounds__(256) ssim_fused_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                         int h, int w, int ch, SsimKernel K, double* sum_out) {
  __shared__ float s_a[3][kSHY][kSHX + 1], s_b[3][kSHY][kSHX + 1];
  __shared__ float s_h[5][kSHY][kSTX + 1];
  const float c1 = 0.01f * 0.01f, c2 = 0.03f * 0.03f;
  const int x0 = blockIdx.x * kSTX, y0 = blockIdx.y * kSTY;
  const int tid = threadIdx.x;
  double acc = 0.0;
  for (int cb = 0; cb < ch; cb += 3) {
  const int nc = min(3, ch - cb);
  for (int i = tid; i < kSHY * kSHX; i += blockDim.x) {  // halos of up to 3 channels, one reflected index
    const int yy = i / kSHX, xx = i % kSHX;
    const int gy = refl(min(y0 - kRad + yy, h - 1 + kRad), h), gx = refl(min(x0 - kRad + xx, w - 1 + kRad), w);
    const int64_t q = ((int64_t)gy * w + gx) * ch + cb;
    for (int c = 0; c < nc; ++c) {
      s_a[c][yy][xx] = a[q + c];
      s_b[c][yy][xx] = b[q + c];
    }
  }
  __syncthreads();
  for (int c = 0; c < nc; ++c) {
    // horizontal: kSHY rows x (kSTX / kSOut) segments
    for (int t = tid; t < kSHY * (kSTX / kSOut); t += blockDim.x) {
      const int yy = t / (kSTX / kSOut), xs = (t % (kSTX / kSOut)) * kSOut;
      float av[kSOut + 2 * kRad], bv[kSOut + 2 * kRad];
#pragma unroll
      for (int i = 0; i < kSOut + 2 * kRad; ++i) {
        av[i] = s_a[c][yy][xs + i];
        bv[i] = s_b[c][yy][xs + i];
      }
#pragma unroll
      for (int o = 0; o < kSOut; ++o) {
        float s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
          const float x = av[o + k], y = bv[o + k], kw = K.k[k];
          s0 += kw * x;
          s1 += kw * y;
          s2 += kw * (x * x);
          s3 += kw * (y * y);
          s4 += kw * (x * y);
        }
        s_h[0][yy][xs + o] = s0;
        s_h[1][yy][xs + o] = s1;
        s_h[2][yy][xs + o] = s2;
        s_h[3][yy][xs + o] = s3;
        s_h[4][yy][xs + o] = s4;
      }
    }
    __syncthreads();
    // vertical: kSTX columns x 8 segments of kVOut rows = 256 threads
    {
      const int xx = tid % kSTX, ys = (tid / kSTX) * kVOut;
      float q[kVOut][5];
#pragma unroll
      for (int o = 0; o < kVOut; ++o)
#pragma unroll
        for (int t = 0; t < 5; ++t) q[o][t] = 0.f;
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        float col[kVOut + 2 * kRad];
#pragma unroll
        for (int i = 0; i < kVOut + 2 * kRad; ++i) col[i] = s_h[t][ys + i][xx];
#pragma unroll
        for (int o = 0; o < kVOut; ++o)
#pragma unroll
          for (int k = 0; k < kWin; ++k) q[o][t] += K.k[k] * col[o + k];
      }
#pragma unroll
      for (int o = 0; o < kVOut; ++o) {
        const int y = y0 + ys + o, x = x0 + xx;
        if (y < h && x < w) {
          const float mx = q[o][0], my = q[o][1];
          const float sx2 = q[o][2] - mx * mx, sy2 = q[o][3] - my * my, sxy = q[o][4] - mx * my;
          const float a1 = 2.f * mx * my + c1, a2 = 2.f * sxy + c2;
          const float b1 = mx * mx + my * my + c1, b2 = sx2 + sy2 + c2;
          acc += (double)((a1 * a2) / (b1 * b2));
        }
      }
    }
    __syncthreads();
  }
  }
  block_add_double(acc, sum_out);
}

// Adjoint of one separable pass along an axis (filter_plane_adjoint, losses.cpp:57-75),
// in gather form: out[i'] = sum over preimages i of refl with refl(i) == i'.
__device__ __forceinline__ float adj_gather(const float* in, int64_t stride, int len, int ip, const SsimKernel& K) {
  float acc = 0.f;
  int pre[3];
  int np = 0;
  pre[np++] = ip;
  if (ip >= 1 && ip <= kRad) pre[np++] = -ip;
  const int r = 2 * len - 2 - ip;
  if (r >= len && r <= len - 1 + kRad && ip <= len - 2) pre[np++] = r;
  for (int t = 0; t < np; ++t)
#pragma unroll
    for (int k = -kRad; k <= kRad; ++k) {
      const int y = pre[t] - k;
      if (y >= 0 && y < len) acc += K.k[k + kRad] * in[(int64_t)y * stride];
    }
  return acc;
}

__global__ void ssim_adj_v_kernel(const float* __restrict__ seeds, int h, int w, int ch, SsimKernel K,
                                  float* __restrict__ tmp) {
  const int64_t n = (int64_t)h * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * ch * 3; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t plane = e / n;
    const int64_t p = e % n;
    const int y = (int)(p / w), x = (int)(p % w);
    tmp[plane * n + p] = adj_gather(seeds + plane * n + x, w, h, y, K);
  }
}

__global__ void ssim_adj_h_kernel(const float* __restrict__ tmp, const float* __restrict__ a,
                                  const float* __restrict__ b, int h, int w, int ch, SsimKernel K, float scale,
                                  float out_scale, bool accumulate, float* __restrict__ d_a) {
  const int64_t n = (int64_t)h * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * ch; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const int64_t p = e % n;
    const int y = (int)(p / w), x = (int)(p % w);
    const float* base = tmp + (int64_t)c * 3 * n + (int64_t)y * w;
    const float g0 = adj_gather(base, 1, w, x, K);
    const float g1 = adj_gather(base + n, 1, w, x, K);
    const float g2 = adj_gather(base + 2 * n, 1, w, x, K);
    const int64_t q = p * ch + c;
    float v = g0 * scale;
    v += 2.f * a[q] * g1 * scale;
    v += b[q] * g2 * scale;
    v *= out_scale;
    d_a[q] = accumulate ? d_a[q] + v : v;
  }
}

// ssim_global, losses.cpp:85-129 (images smaller than the window). One block.
__global__ void ssim_global_kernel(const float* a, const float* b, int h, int w, int ch, float* d_a, float out_scale,
                                   bool accumulate, double* sum_out) {
  // fixed-order block reductions (per-thread partials, summed by thread 0 in thread order), so the
  // result does not depend on warp scheduling
  __shared__ double part[256][3];
  __shared__ double red[5];
  const float c1 = 0.01f * 0.01f, c2 = 0.03f * 0.03f;
  const int n = h * w;
  double total = 0.0;
  auto block_sum = [&](double x, double y, double z, double* out) {
    part[threadIdx.x][0] = x, part[threadIdx.x][1] = y, part[threadIdx.x][2] = z;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sx = 0, sy = 0, sz = 0;
      for (unsigned t = 0; t < blockDim.x; ++t) sx += part[t][0], sy += part[t][1], sz += part[t][2];
      out[0] = sx, out[1] = sy, out[2] = sz;
    }
    __syncthreads();
  };
  for (int c = 0; c < ch; ++c) {
    double sx = 0, sy = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      sx += a[i * ch + c];
      sy += b[i * ch + c];
    }
    block_sum(sx, sy, 0.0, red);
    const float mx = (float)(red[0] / n), my = (float)(red[1] / n);
    double vx = 0, vy = 0, cv = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const float dx = a[i * ch + c] - mx, dy = b[i * ch + c] - my;
      vx += dx * dx;
      vy += dy * dy;
      cv += dx * dy;
    }
    block_sum(vx, vy, cv, red + 2);
    const float fvx = (float)(red[2] / n), fvy = (float)(red[3] / n), fcv = (float)(red[4] / n);
    const float a1 = 2.f * mx * my + c1, a2 = 2.f * fcv + c2;
    const float b1 = mx * mx + my * my + c1, b2 = fvx + fvy + c2;
    const float s = (a1 * a2) / (b1 * b2);
    total += s;
    if (d_a) {
      const float ds_dmx = 2.f * my * a2 / (b1 * b2) - s * 2.f * mx / b1;
      const float ds_dvx = -s / b2;
      const float ds_dcov = 2.f * a1 / (b1 * b2);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const float dx = a[i * ch + c] - mx, dy = b[i * ch + c] - my;
        const float g = (ds_dmx / n + ds_dvx * 2.f * dx / n + ds_dcov * dy / n) / ch * out_scale;
        d_a[i * ch + c] = accumulate ? d_a[i * ch + c] + g : g;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(sum_out, total / ch * (double)n * ch);  // returned as a per-pixel sum
}

// SSIM value (as a sum over pixels and channels into *sum_out) and, when d_a is given,
// out_scale * dSSIM/da written (or added) into d_a.
void ssim_run(cudaStream_t st, const float* a, const float* b, int h, int w, int ch, float* d_a, float out_scale,
              bool accumulate, float* scratch, double* sum_out) {
  const SsimKernel K = make_kernel();
  const int64_t n = (int64_t)h * w;
  if (h < kWin || w < kWin) {
    ssim_global_kernel<<<1, 256, 0, st>>>(a, b, h, w, ch, d_a, out_scale, accumulate, sum_out);
    count_launch();
    return;
  }
  if (!d_a) {
    ssim_fused_kernel<<<dim3((w + kSTX - 1) / kSTX, (h + kSTY - 1) / kSTY), 256, 0, st>>>(a, b, h, w, ch, K,
                                                                                              sum_out);
    count_launch();
    return;
  }
  float* hq = scratch;
  float* seeds = scratch + 5 * n * ch;
  float* tmp = seeds + 3 * n * ch;
  const int grid = (int)std::min<int64_t>((n * ch + 255) / 256, 148 * 16);
  ssim_h_kernel<<<grid, 256, 0, st>>>(a, b, h, w, ch, K, hq);
  ssim_v_kernel<<<grid, 256, 0, st>>>(hq, h, w, ch, K, d_a != nullptr, seeds, sum_out);
  count_launch(2);
  if (d_a) {
    const float scale = 1.f / ((float)n * (float)ch);
    const int g3 = (int)std::min<int64_t>((n * ch * 3 + 255) / 256, 148 * 16);
    ssim_adj_v_kernel<<<g3, 256, 0, st>>>(seeds, h, w, ch, K, tmp);
    ssim_adj_h_kernel<<<grid, 256, 0, st>>>(tmp, a, b, h, w, ch, K, scale, out_scale, accumulate, d_a);
    count_launch(2);
  }
}

}  // namespace

size_t ssim_scratch_floats(int h, int w, int c) { return (size_t)h * w * c * 11; }

double ssim_host(cudaStream_t st, const float* a, const float* b, int h, int w, int c, float* d_a, float* scratch) {
  double* d_sum;
  cudaMallocAsync(&d_sum, sizeof(double), st);
  cudaMemsetAsync(d_sum, 0, sizeof(double), st);
  ssim_run(st, a, b, h, w, c, d_a, 1.f, false, scratch, d_sum);
  double s = 0;
  cudaMemcpyAsync(&s, d_sum, sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_sum, st);
  cudaStreamSynchronize(st);
  return s / ((double)h * w * c);
}

void image_losses(cudaStream_t st, const float* color, const float* depth, const float* alpha, const float* rgb_t,
                  const float* depth_t, int h, int w, float lambda_i1, float lambda_i2, float rgb_scale,
                  float depth_scale, bool want_grad, float* d_color, float* d_depth, double* partials,
                  float* ssim_scratch) {
  const int64_t npx = (int64_t)h * w;
  const int grid = (int)std::min<int64_t>((npx + 255) / 256, 148 * 8);
  // SSIM forward always runs (losses.cpp:217); its gradient only matters when lambda_i2 != 0.
  const bool ssim_grad = want_grad && lambda_i2 != 0.f;
  auto al16 = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = npx % 4 == 0 && al16(color) && al16(depth) && al16(alpha) && al16(rgb_t) && al16(depth_t) &&
                   al16(d_color) && al16(d_depth) && (!want_grad || (d_color && d_depth));
  if (vec) {
    const int64_t n4 = npx / 4;
    const int g4 = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
    l1_depth4_kernel<<<g4, 256, 0, st>>>(reinterpret_cast<const float4*>(color), reinterpret_cast<const float4*>(depth),
                                         reinterpret_cast<const float4*>(alpha), reinterpret_cast<const float4*>(rgb_t),
                                         reinterpret_cast<const float4*>(depth_t), n4, lambda_i1, (float)(npx * 3),
                                         want_grad, !ssim_grad, rgb_scale, reinterpret_cast<float4*>(d_color),
                                         reinterpret_cast<float4*>(d_depth), partials);
  } else {
    l1_depth_kernel<<<grid, 256, 0, st>>>(color, depth, alpha, rgb_t, depth_t, npx, lambda_i1, (float)(npx * 3),
                                          want_grad, d_color, d_depth, partials);
  }
  count_launch();
  ssim_run(st, color, rgb_t, h, w, 3, ssim_grad ? d_color : nullptr, lambda_i2 * -0.5f, true, ssim_scratch,
           &partials[1]);
  if (want_grad) {
    if (vec && !ssim_grad) {
      const int64_t n4 = npx / 4;
      finalize_depth4_kernel<<<(int)std::min<int64_t>((n4 + 255) / 256, 148 * 8), 256, 0, st>>>(
          reinterpret_cast<float4*>(d_depth), n4, depth_scale, partials);
    } else {
      finalize_upstream_kernel<<<grid, 256, 0, st>>>(d_color, d_depth, npx, rgb_scale, depth_scale, partials);
    }
    count_launch();
  }
}


// ---------------------------------------------------------------- standalone losses (C-ABI)
// rgb_loss / depth_loss / feature_loss, obj/losses.hpp:12-58 (proj/src/losses.cpp:200-294), as
// separate device operators on caller-owned images / rows. The step fuses these into the frame
// loop (image_losses above, the decoders' epilogues); these are the reference's operator API.
namespace {

__global__ void __launch_bounds__(256) rgb_l1_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                     int64_t n, float lambda_i1, float* grad, double* sum) {
  double l1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = fs(a[i], b[i]);
    l1 += (double)fabsf(d);
    if (grad) grad[i] = fd(fm(lambda_i1, d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)), (float)n);
  }
  block_add_double(l1, sum);
}

__global__ void __launch_bounds__(256) depth_sum_kernel(const float* __restrict__ r, const float* __restrict__ o,
                                                        const float* __restrict__ al, int64_t n, double* acc) {
  double sum = 0.0, cnt = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (o[i] > 0.f && al[i] > 0.5f) {
      sum += (double)fabsf(fs(r[i], o[i]));
      cnt += 1.0;
    }
  block_add_double(sum, &acc[0]);
  block_add_double(cnt, &acc[1]);
}

__global__ void depth_grad_kernel(const float* __restrict__ r, const float* __restrict__ o,
                                  const float* __restrict__ al, int64_t n, const double* acc, float* grad) {
  const float valid = (float)acc[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float g = 0.f;
    if (valid > 0.f && o[i] > 0.f && al[i] > 0.5f) {
      const float d = fs(r[i], o[i]);
      g = fd(d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f), valid);
    }
    grad[i] = g;
  }
}

// one warp per row: |u|, |v|, u.v, |u - v|^2 (float, lane-strided), then the row gradient
// dF = lambda_cos (-(v / (|u||v|) - dot u / (|u|^3 |v|))) / n + lambda_l2 2 (u - v) / n
__global__ void __launch_bounds__(256) feature_rows_kernel(const float* __restrict__ u, const float* __restrict__ v,
                                                           int64_t n, int df, float lambda_cos, float lambda_l2,
                                                           float* d_rec, double* acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  double cos_acc = 0.0, l2_acc = 0.0, flag = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const float* ur = u + r * df;
    const float* vr = v + r * df;
    float uu = 0.f, vv = 0.f, uv = 0.f, dd = 0.f;
    for (int c = lane; c < df; c += 32) {
      const float a = ur[c], b = vr[c];
      uu = fmaf(a, a, uu);
      vv = fmaf(b, b, vv);
      uv = fmaf(a, b, uv);
      const float e = a - b;
      dd = fmaf(e, e, dd);
    }
    uu = warp_sum(uu);
    vv = warp_sum(vv);
    uv = warp_sum(uv);
    dd = warp_sum(dd);
    const float eps = 1e-8f, nu = sqrtf(uu), nv = sqrtf(vv);
    const float nug = fmaxf(nu, eps), nvg = fmaxf(nv, eps);
    if (lane == 0) {
      if (nu < eps || nv < eps) flag = 1.0;
      cos_acc += 1.0 - (double)(uv / (nug * nvg));
      l2_acc += (double)dd;
    }
    if (d_rec) {
      const float inv_n = 1.f / (float)n;
      const float a_u = lambda_cos * uv / (nug * nug * nug * nvg) * inv_n + 2.f * lambda_l2 * inv_n;
      const float a_v = -lambda_cos / (nug * nvg) * inv_n - 2.f * lambda_l2 * inv_n;
      float* gr = d_rec + r * df;
      for (int c = lane; c < df; c += 32) gr[c] = fmaf(a_u, ur[c], a_v * vr[c]);
    }
  }
  block_add_double(cos_acc, &acc[0]);
  block_add_double(l2_acc, &acc[1]);
  block_add_double(flag, &acc[2]);
}

}  // namespace

cudaError_t rgb_loss_dev(cudaStream_t st, const float* rendered, const float* observed, int h, int w, int ch,
                         float lambda_i1, float lambda_i2, float* grad, float out[3]) {
  const int64_t n = (int64_t)h * w * ch;
  double* acc = nullptr;
  float* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&acc, sizeof(double) * 2, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&scratch, sizeof(float) * std::max<size_t>(ssim_scratch_floats(h, w, ch), 1), st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(acc, 0, sizeof(double) * 2, st);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  if (n > 0) {
    rgb_l1_kernel<<<grid, 256, 0, st>>>(rendered, observed, n, lambda_i1, grad, &acc[0]);
    count_launch();
    // SSIM always (losses.cpp:217); its adjoint is added into grad scaled by -lambda_i2 / 2
    ssim_run(st, rendered, observed, h, w, ch, grad, lambda_i2 * -0.5f, true, scratch, &acc[1]);
  }
  double hv[2] = {0, 0};
  cudaMemcpyAsync(hv, acc, sizeof(hv), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(acc, st);
  cudaFreeAsync(scratch, st);
  e = cudaStreamSynchronize(st);
  const float l1 = n > 0 ? (float)(hv[0] / (double)n) : 0.f;
  const float ss = n > 0 ? (float)(hv[1] / (double)n) : 1.f;
  out[1] = l1;
  out[2] = (1.f - ss) / 2.f;
  out[0] = lambda_i1 * out[1] + lambda_i2 * out[2];
  return e;
}

cudaError_t depth_loss_dev(cudaStream_t st, const float* rendered, const float* observed, const float* alpha,
                           int64_t n, float* grad, float* value, int* flagged) {
  double* acc = nullptr;
  cudaError_t e = cudaMallocAsync(&acc, sizeof(double) * 2, st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(acc, 0, sizeof(double) * 2, st);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
  if (n > 0) {
    depth_sum_kernel<<<grid, 256, 0, st>>>(rendered, observed, alpha, n, acc);
    count_launch();
    if (grad) {
      depth_grad_kernel<<<grid, 256, 0, st>>>(rendered, observed, alpha, n, acc, grad);
      count_launch();
    }
  }
  double hv[2] = {0, 0};
  cudaMemcpyAsync(hv, acc, sizeof(hv), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(acc, st);
  e = cudaStreamSynchronize(st);
  *flagged = hv[1] == 0.0;
  *value = hv[1] > 0.0 ? (float)(hv[0] / hv[1]) : 0.f;
  return e;
}

cudaError_t feature_loss_dev(cudaStream_t st, const float* rec, const float* tgt, int64_t n, int df,
                             const float* atoms, const float* anchor, int64_t k, float delta, float lambda_cos,
                             float lambda_l2, float lambda_trust, float* d_rec, float* d_atoms_trust, float out[4],
                             int* zero_norm_flagged) {
  double* acc = nullptr;
  cudaError_t e = cudaMallocAsync(&acc, sizeof(double) * 4, st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(acc, 0, sizeof(double) * 4, st);
  if (n > 0) {
    const int grid = (int)std::min<int64_t>((n + 7) / 8, 148 * 16);
    feature_rows_kernel<<<grid, 256, 0, st>>>(rec, tgt, n, df, lambda_cos, lambda_l2, d_rec, acc);
    count_launch();
  }
  if (d_atoms_trust) cudaMemsetAsync(d_atoms_trust, 0, sizeof(float) * k * df, st);
  trust_region(st, atoms, anchor, k, df, delta, d_atoms_trust, lambda_trust, &acc[3]);
  double hv[4] = {0, 0, 0, 0};
  cudaMemcpyAsync(hv, acc, sizeof(hv), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(acc, st);
  e = cudaStreamSynchronize(st);
  out[1] = n > 0 ? (float)(hv[0] / (double)n) : 0.f;  // cos_term
  out[2] = n > 0 ? (float)(hv[1] / (double)n) : 0.f;  // l2_term
  out[3] = (float)hv[3];                              // trust_term
  out[0] = lambda_cos * out[1] + lambda_l2 * out[2] + lambda_trust * out[3];
  *zero_norm_flagged = hv[2] != 0.0;
  return e;
}

}  // namespace lm
