// Memory-bound kernels of the CNN training step (K3/K4/K5-support of DESIGN.md): batch-norm
// statistics / apply / backward with fused ReLU and residual, pooling, softmax
// cross-entropy, split-K reduction, weight flip, zero-upsampling, column sums and the
// fused Adam / SGD updates.  All activations are NHWC bf16 rows [rows][C] with a channel
// stride (so DenseNet concat buffers are read in place); statistics and gradients fp32.
// Every reduction is two-level and fixed-order -> results are deterministic run to run.
// 8 channels (one 16-byte vector) per thread in the elementwise kernels.
#include "cvb_common.cuh"
#include <cuda_bf16.h>
#include <math.h>

namespace {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ void load8(const bf16* p, float v[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}
__device__ __forceinline__ void store8(bf16* p, const float v[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

constexpr int ST_THREADS = 256;

__device__ __forceinline__ void ld8f(const float* p, float v[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// ---- per-channel sum / sum of squares (two-level) -------------------------------------
// grid.x = blocks over rows; thread (rl, g) handles channel group g (8 channels) of rows
// rl, rl + RL, ... inside the block's row range.  Partial layout: [blk][2][C].
__global__ void chan_stats_partial(const bf16* __restrict__ x, int64_t rows, int C, int cs, int64_t rows_per_blk,
                                   float* __restrict__ part) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int RL = ST_THREADS / G;  // row lanes (G <= 256 guaranteed by host)
  const int t = threadIdx.x, g = t % G, rl = t / G;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk, r1 = min(rows, r0 + rows_per_blk);
  float s[8] = {0}, q[8] = {0};
  if (rl < RL) {
    for (int64_t r = r0 + rl; r < r1; r += RL) {
      float v[8];
      load8(x + r * cs + g * 8, v);
#pragma unroll
      for (int i = 0; i < 8; i++) { s[i] += v[i]; q[i] += v[i] * v[i]; }
    }
  }
  extern __shared__ float sh[];  // [RL][G][16]
  if (rl < RL) {
#pragma unroll
    for (int i = 0; i < 8; i++) { sh[(rl * G + g) * 16 + i] = s[i]; sh[(rl * G + g) * 16 + 8 + i] = q[i]; }
  }
  __syncthreads();
  for (int idx = t; idx < G * 16; idx += ST_THREADS) {
    const int gg = idx / 16, k = idx % 16;
    float acc = 0.f;
    for (int l = 0; l < RL; l++) acc += sh[(l * G + gg) * 16 + k];
    const int c = gg * 8 + (k & 7);
    part[((int64_t)blockIdx.x * 2 + (k >> 3)) * C + c] = acc;
  }
}

// Sum the [nblk][2][C] partials: block = 32 channels x 32 warps; warp w sums blocks w, w+32,
// ... (coalesced across the 32 channels, independent loads), then a fixed-order smem
// combine -> deterministic.
constexpr int FIN_WARPS = 32;
__device__ __forceinline__ void sum_partials(const float* __restrict__ part, int nblk, int C, int c, double& s,
                                             double& q) {
  __shared__ double sh[2][FIN_WARPS][32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  double a = 0, b2 = 0;
  if (c < C) {
#pragma unroll 4
    for (int b = w; b < nblk; b += FIN_WARPS) {
      a += part[(int64_t)(2 * b) * C + c];
      b2 += part[(int64_t)(2 * b + 1) * C + c];
    }
  }
  sh[0][w][l] = a;
  sh[1][w][l] = b2;
  __syncthreads();
  s = 0; q = 0;
  for (int k = 0; k < FIN_WARPS; k++) { s += sh[0][k][l]; q += sh[1][k][l]; }
}

__global__ void __launch_bounds__(FIN_WARPS * 32) bn_finalize(const float* __restrict__ part, int nblk, int C, double count, float eps,
                            float* __restrict__ mean, float* __restrict__ rstd, float* __restrict__ run_mean,
                            float* __restrict__ run_var, float momentum) {
  CVB_PDL_PROLOGUE();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s, q;
  sum_partials(part, nblk, C, c, s, q);
  if (threadIdx.x >= 32 || c >= C) return;
  const double m = s / count;
  double var = q / count - m * m;
  if (var < 0) var = 0;
  mean[c] = (float)m;
  rstd[c] = (float)(1.0 / sqrt(var + (double)eps));
  if (run_mean) {
    const double unb = count > 1 ? var * count / (count - 1) : var;
    run_mean[c] = (float)((1.0 - momentum) * run_mean[c] + momentum * m);
    run_var[c] = (float)((1.0 - momentum) * run_var[c] + momentum * unb);
  }
}

// ---- y = act(gamma * (x - mean) * rstd + beta [+ res]) ---------------------------------
__global__ void bn_apply(const bf16* __restrict__ x, int64_t rows, int C, int xcs, const float* __restrict__ mean,
                         const float* __restrict__ rstd, const float* __restrict__ gamma, const float* __restrict__ beta,
                         const bf16* __restrict__ res, int rcs, int relu, bf16* __restrict__ y, int ycs, int ycoff) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * G) return;
  const int64_t r = i / G;
  const int g = (int)(i - r * G);
  float v[8], o[8];
  load8(x + r * xcs + g * 8, v);
  float rv[8];
  if (res) load8(res + r * rcs + g * 8, rv);
  // per-channel parameters as 16-byte vectors (8 loads instead of 32 scalar ones)
  float mu[8], rs[8], ga[8], be[8];
  ld8f(mean + g * 8, mu); ld8f(rstd + g * 8, rs); ld8f(gamma + g * 8, ga); ld8f(beta + g * 8, be);
#pragma unroll
  for (int k = 0; k < 8; k++) {
    float z = (v[k] - mu[k]) * (ga[k] * rs[k]) + be[k];
    if (res) z += rv[k];
    o[k] = relu ? fmaxf(z, 0.f) : z;
  }
  store8(y + r * ycs + ycoff + g * 8, o);
}

// ---- batch-norm backward, reduction pass ----------------------------------------------
// dz = dy * mask (mask = y > 0 when relu; y = the layer output, or recomputed from x when
// y == nullptr).  Partials [blk][2][C] of sum(dz) and sum(dz * xhat); optionally stores dz.
__global__ void bn_bwd_partial(const bf16* __restrict__ dy, int dycs, const bf16* __restrict__ x, int xcs,
                               const bf16* __restrict__ y, int ycs, int64_t rows, int C, const float* __restrict__ mean,
                               const float* __restrict__ rstd, const float* __restrict__ gamma, const float* __restrict__ beta,
                               int relu, int64_t rows_per_blk, float* __restrict__ part, bf16* __restrict__ dz_out) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int RL = ST_THREADS / G;
  const int t = threadIdx.x, g = t % G, rl = t / G;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk, r1 = min(rows, r0 + rows_per_blk);
  float s[8] = {0}, q[8] = {0};
  float mu[8], rs[8], ga[8], be[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const int c = g * 8 + k;
    mu[k] = mean[c]; rs[k] = rstd[c]; ga[k] = gamma[c]; be[k] = beta[c];
  }
  if (rl < RL) {
    for (int64_t r = r0 + rl; r < r1; r += RL) {
      float d[8], xv[8], yv[8];
      load8(dy + r * dycs + g * 8, d);
      load8(x + r * xcs + g * 8, xv);
      if (relu && y) load8(y + r * ycs + g * 8, yv);
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const float xh = (xv[k] - mu[k]) * rs[k];
        if (relu) {
          const float z = y ? yv[k] : xh * ga[k] + be[k];
          if (!(z > 0.f)) d[k] = 0.f;
        }
        s[k] += d[k];
        q[k] += d[k] * xh;
      }
      if (dz_out) store8(dz_out + r * C + g * 8, d);
    }
  }
  extern __shared__ float sh[];
  if (rl < RL) {
#pragma unroll
    for (int i = 0; i < 8; i++) { sh[(rl * G + g) * 16 + i] = s[i]; sh[(rl * G + g) * 16 + 8 + i] = q[i]; }
  }
  __syncthreads();
  for (int idx = t; idx < G * 16; idx += ST_THREADS) {
    const int gg = idx / 16, k = idx % 16;
    float acc = 0.f;
    for (int l = 0; l < RL; l++) acc += sh[(l * G + gg) * 16 + k];
    part[((int64_t)blockIdx.x * 2 + (k >> 3)) * C + gg * 8 + (k & 7)] = acc;
  }
}

__global__ void __launch_bounds__(FIN_WARPS * 32) bn_bwd_finalize(const float* __restrict__ part, int nblk, int C, float* __restrict__ dbeta,
                                float* __restrict__ dgamma) {
  CVB_PDL_PROLOGUE();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s, q;
  sum_partials(part, nblk, C, c, s, q);
  if (threadIdx.x >= 32 || c >= C) return;
  dbeta[c] = (float)s;
  dgamma[c] = (float)q;
}

// dx = gamma * rstd * (dz - dbeta/M - xhat * dgamma/M)   (dz recomputed like the partial pass)
__global__ void bn_bwd_apply(const bf16* __restrict__ dy, int dycs, const bf16* __restrict__ x, int xcs,
                             const bf16* __restrict__ y, int ycs, int64_t rows, int C, const float* __restrict__ mean,
                             const float* __restrict__ rstd, const float* __restrict__ gamma, const float* __restrict__ beta,
                             int relu, const float* __restrict__ dbeta, const float* __restrict__ dgamma,
                             bf16* __restrict__ dx, int dxcs, float* __restrict__ dx32, int accum32) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * G) return;
  const int64_t r = i / G;
  const int g = (int)(i - r * G);
  const float invM = 1.0f / (float)rows;
  float d[8], xv[8], yv[8], o[8];
  load8(dy + r * dycs + g * 8, d);
  load8(x + r * xcs + g * 8, xv);
  if (relu && y) load8(y + r * ycs + g * 8, yv);
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const int c = g * 8 + k;
    const float xh = (xv[k] - mean[c]) * rstd[c];
    if (relu) {
      const float z = y ? yv[k] : xh * gamma[c] + beta[c];
      if (!(z > 0.f)) d[k] = 0.f;
    }
    o[k] = gamma[c] * rstd[c] * (d[k] - dbeta[c] * invM - xh * dgamma[c] * invM);
  }
  if (dx32) {
    float* p = dx32 + r * dxcs + g * 8;
#pragma unroll
    for (int k = 0; k < 8; k++) p[k] = accum32 ? p[k] + o[k] : o[k];
  } else {
    store8(dx + r * dxcs + g * 8, o);
  }
}

// ---- pooling --------------------------------------------------------------------------
__global__ void maxpool_fwd(const bf16* __restrict__ x, int n, int h, int w, int C, int k, int s, int p, int oh, int ow,
                            bf16* __restrict__ y, int ycs) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * oh * ow * G) return;
  const int g = (int)(i % G);
  int64_t pix = i / G;
  const int ox = (int)(pix % ow), oy = (int)((pix / ow) % oh), b = (int)(pix / ((int64_t)ow * oh));
  float m[8];
#pragma unroll
  for (int c = 0; c < 8; c++) m[c] = -INFINITY;
  for (int dy = 0; dy < k; dy++) {
    const int iy = oy * s - p + dy;
    if (iy < 0 || iy >= h) continue;
    for (int dx = 0; dx < k; dx++) {
      const int ix = ox * s - p + dx;
      if (ix < 0 || ix >= w) continue;
      float v[8];
      load8(x + (((int64_t)b * h + iy) * w + ix) * C + g * 8, v);
#pragma unroll
      for (int c = 0; c < 8; c++) if (v[c] > m[c]) m[c] = v[c];
    }
  }
  store8(y + pix * ycs + g * 8, m);
}

// gather form: each input element collects dy of every window whose FIRST arg-max it is
__global__ void maxpool_bwd(const bf16* __restrict__ x, const bf16* __restrict__ dyp, int n, int h, int w, int C, int k,
                            int s, int p, int oh, int ow, bf16* __restrict__ dx) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * h * w * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ix = (int)(pix % w), iy = (int)((pix / w) % h), b = (int)(pix / ((int64_t)w * h));
  float acc[8] = {0};
  const int oy0 = max(0, (iy + p - k + s) / s), oy1 = min(oh - 1, (iy + p) / s);
  const int ox0 = max(0, (ix + p - k + s) / s), ox1 = min(ow - 1, (ix + p) / s);
  for (int oy = oy0; oy <= oy1; oy++) {
    for (int ox = ox0; ox <= ox1; ox++) {
      // recompute the window's first arg-max (row-major scan, strict >)
      float m[8];
      int am[8];
#pragma unroll
      for (int c = 0; c < 8; c++) { m[c] = -INFINITY; am[c] = -1; }
      for (int dy = 0; dy < k; dy++) {
        const int yy = oy * s - p + dy;
        if (yy < 0 || yy >= h) continue;
        for (int dx2 = 0; dx2 < k; dx2++) {
          const int xx = ox * s - p + dx2;
          if (xx < 0 || xx >= w) continue;
          float v[8];
          load8(x + (((int64_t)b * h + yy) * w + xx) * C + g * 8, v);
#pragma unroll
          for (int c = 0; c < 8; c++) if (v[c] > m[c]) { m[c] = v[c]; am[c] = yy * w + xx; }
        }
      }
      float d[8];
      load8(dyp + (((int64_t)b * oh + oy) * ow + ox) * C + g * 8, d);
      const int me = iy * w + ix;
#pragma unroll
      for (int c = 0; c < 8; c++) if (am[c] == me) acc[c] += d[c];
    }
  }
  store8(dx + pix * C + g * 8, acc);
}

// forward with the window's first arg-max (offset dy*k+dx, row-major scan, strict >) kept
// per output element: the backward then needs no window re-scan
__global__ void maxpool_fwd_idx(const bf16* __restrict__ x, int n, int h, int w, int C, int k, int s, int p, int oh,
                                int ow, bf16* __restrict__ y, int ycs, uint8_t* __restrict__ idx) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * oh * ow * G) return;
  const int g = (int)(i % G);
  int64_t pix = i / G;
  const int ox = (int)(pix % ow), oy = (int)((pix / ow) % oh), b = (int)(pix / ((int64_t)ow * oh));
  float m[8];
  uint32_t am[8];
#pragma unroll
  for (int c = 0; c < 8; c++) { m[c] = -INFINITY; am[c] = 0; }
  for (int dy = 0; dy < k; dy++) {
    const int iy = oy * s - p + dy;
    if (iy < 0 || iy >= h) continue;
    for (int dx = 0; dx < k; dx++) {
      const int ix = ox * s - p + dx;
      if (ix < 0 || ix >= w) continue;
      float v[8];
      load8(x + (((int64_t)b * h + iy) * w + ix) * C + g * 8, v);
#pragma unroll
      for (int c = 0; c < 8; c++) if (v[c] > m[c]) { m[c] = v[c]; am[c] = (uint32_t)(dy * k + dx); }
    }
  }
  store8(y + pix * ycs + g * 8, m);
  uint2 packed = make_uint2(am[0] | (am[1] << 8) | (am[2] << 16) | (am[3] << 24),
                            am[4] | (am[5] << 8) | (am[6] << 16) | (am[7] << 24));
  *reinterpret_cast<uint2*>(idx + pix * C + g * 8) = packed;
}

// gather: input (iy, ix) takes dy of every window (oy, ox) whose stored arg-max is it
// 3x3 / stride-2 / pad-1 (the DenseNet stem pool) with every window load in flight: the generic
// kernels walk runtime-k loops with runtime divisions, one dependent load at a time.  Same
// comparison / accumulation order as the generic forms -> identical outputs.
__global__ void maxpool3s2_fwd_idx(const bf16* __restrict__ x, int n, int h, int w, int C, int oh, int ow,
                                   bf16* __restrict__ y, int ycs, uint8_t* __restrict__ idx) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * oh * ow * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ox = (int)(pix % ow), oy = (int)((pix / ow) % oh), b = (int)(pix / ((int64_t)ow * oh));
  uint4 u[9];
#pragma unroll
  for (int q = 0; q < 9; q++) {
    const int iy = 2 * oy - 1 + q / 3, ix = 2 * ox - 1 + q % 3;
    u[q] = (iy >= 0 && iy < h && ix >= 0 && ix < w)
               ? *reinterpret_cast<const uint4*>(x + (((int64_t)b * h + iy) * w + ix) * C + g * 8)
               : make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);   // -inf: never > m
  }
  float m[8];
  uint32_t am[8];
#pragma unroll
  for (int c = 0; c < 8; c++) { m[c] = -INFINITY; am[c] = 0; }
#pragma unroll
  for (int q = 0; q < 9; q++) {
    const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u[q]);
#pragma unroll
    for (int c2 = 0; c2 < 4; c2++) {
      const float2 f = __bfloat1622float2(hv[c2]);
      if (f.x > m[2 * c2]) { m[2 * c2] = f.x; am[2 * c2] = (uint32_t)q; }
      if (f.y > m[2 * c2 + 1]) { m[2 * c2 + 1] = f.y; am[2 * c2 + 1] = (uint32_t)q; }
    }
  }
  store8(y + pix * ycs + g * 8, m);
  uint2 packed = make_uint2(am[0] | (am[1] << 8) | (am[2] << 16) | (am[3] << 24),
                            am[4] | (am[5] << 8) | (am[6] << 16) | (am[7] << 24));
  *reinterpret_cast<uint2*>(idx + pix * C + g * 8) = packed;
}

__global__ void maxpool3s2_bwd_idx(const uint8_t* __restrict__ idx, const bf16* __restrict__ dyp, int n, int h, int w,
                                   int C, int oh, int ow, bf16* __restrict__ dx) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * h * w * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ix = (int)(pix % w), iy = (int)((pix / w) % h), b = (int)(pix / ((int64_t)w * h));
  // windows covering (iy, ix): oy in [iy >> 1, (iy + 1) >> 1], ox likewise (clipped)
  const int oy0 = iy >> 1, oy1 = min(oh - 1, (iy + 1) >> 1), ox0 = ix >> 1, ox1 = min(ow - 1, (ix + 1) >> 1);
  uint2 a[4];
  uint4 d[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int oy = oy0 + (q >> 1), ox = ox0 + (q & 1);
    if (oy <= oy1 && ox <= ox1) {
      const int64_t o = (((int64_t)b * oh + oy) * ow + ox) * C + g * 8;
      a[q] = *reinterpret_cast<const uint2*>(idx + o);
      d[q] = *reinterpret_cast<const uint4*>(dyp + o);
    }
  }
  float acc[8] = {0};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int oy = oy0 + (q >> 1), ox = ox0 + (q & 1);
    if (oy <= oy1 && ox <= ox1) {
      const uint32_t me = (uint32_t)((iy - (oy * 2 - 1)) * 3 + (ix - (ox * 2 - 1)));
      float dv[8];
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&d[q]);
#pragma unroll
      for (int c2 = 0; c2 < 4; c2++) { const float2 f = __bfloat1622float2(hv[c2]); dv[2 * c2] = f.x; dv[2 * c2 + 1] = f.y; }
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const uint32_t am = ((c < 4 ? a[q].x : a[q].y) >> (8 * (c & 3))) & 0xffu;
        if (am == me) acc[c] += dv[c];
      }
    }
  }
  store8(dx + pix * C + g * 8, acc);
}

__global__ void maxpool_bwd_idx(const uint8_t* __restrict__ idx, const bf16* __restrict__ dyp, int n, int h, int w,
                                int C, int k, int s, int p, int oh, int ow, bf16* __restrict__ dx) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * h * w * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ix = (int)(pix % w), iy = (int)((pix / w) % h), b = (int)(pix / ((int64_t)w * h));
  float acc[8] = {0};
  const int oy0 = max(0, (iy + p - k + s) / s), oy1 = min(oh - 1, (iy + p) / s);
  const int ox0 = max(0, (ix + p - k + s) / s), ox1 = min(ow - 1, (ix + p) / s);
  for (int oy = oy0; oy <= oy1; oy++) {
    for (int ox = ox0; ox <= ox1; ox++) {
      const uint32_t me = (uint32_t)((iy - (oy * s - p)) * k + (ix - (ox * s - p)));
      const int64_t o = (((int64_t)b * oh + oy) * ow + ox) * C + g * 8;
      const uint2 a = *reinterpret_cast<const uint2*>(idx + o);
      float d[8];
      load8(dyp + o, d);
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const uint32_t am = ((c < 4 ? a.x : a.y) >> (8 * (c & 3))) & 0xffu;
        if (am == me) acc[c] += d[c];
      }
    }
  }
  store8(dx + pix * C + g * 8, acc);
}

// 2x2 stride-2 max-pool forward: the four window loads issued together (the generic kernel's
// runtime k loop issues them one after another); same comparison order -> identical output
__global__ void maxpool2_fwd(const bf16* __restrict__ x, int n, int h, int w, int C, int oh, int ow,
                             bf16* __restrict__ y, int ycs) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * oh * ow * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ox = (int)(pix % ow), oy = (int)((pix / ow) % oh), b = (int)(pix / ((int64_t)ow * oh));
  float v[4][8], m[8];
#pragma unroll
  for (int q = 0; q < 4; q++)
    load8(x + (((int64_t)b * h + 2 * oy + (q >> 1)) * w + 2 * ox + (q & 1)) * C + g * 8, v[q]);
#pragma unroll
  for (int c = 0; c < 8; c++) {
    m[c] = -INFINITY;
#pragma unroll
    for (int q = 0; q < 4; q++) if (v[q][c] > m[c]) m[c] = v[q][c];
  }
  store8(y + pix * ycs + g * 8, m);
}

// 2x2 / stride-2 windows do not overlap: one thread per output pixel and 8-channel group
// routes dy to the window's first arg-max and writes zeros to the other three inputs.
__global__ void maxpool2_bwd(const bf16* __restrict__ x, const bf16* __restrict__ dyp, int n, int h, int w, int C,
                             int oh, int ow, bf16* __restrict__ dx) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * oh * ow * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ox = (int)(pix % ow), oy = (int)((pix / ow) % oh), b = (int)(pix / ((int64_t)ow * oh));
  float v[4][8], d[8];
  int64_t base[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    base[q] = (((int64_t)b * h + 2 * oy + (q >> 1)) * w + 2 * ox + (q & 1)) * C + g * 8;
    load8(x + base[q], v[q]);
  }
  load8(dyp + pix * C + g * 8, d);
  float o[4][8];
#pragma unroll
  for (int c = 0; c < 8; c++) {
    int am = 0;
    float m = v[0][c];
#pragma unroll
    for (int q = 1; q < 4; q++) if (v[q][c] > m) { m = v[q][c]; am = q; }
#pragma unroll
    for (int q = 0; q < 4; q++) o[q][c] = (q == am) ? d[c] : 0.f;
  }
#pragma unroll
  for (int q = 0; q < 4; q++) store8(dx + base[q], o[q]);
}

__global__ void avgpool_fwd(const bf16* __restrict__ x, int n, int h, int w, int C, int xcs, int k, int oh, int ow,
                            bf16* __restrict__ y, int ycs) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * oh * ow * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ox = (int)(pix % ow), oy = (int)((pix / ow) % oh), b = (int)(pix / ((int64_t)ow * oh));
  float a[8] = {0};
  for (int dy = 0; dy < k; dy++)
    for (int dx = 0; dx < k; dx++) {
      float v[8];
      load8(x + (((int64_t)b * h + oy * k + dy) * w + ox * k + dx) * xcs + g * 8, v);
#pragma unroll
      for (int c = 0; c < 8; c++) a[c] += v[c];
    }
  const float inv = 1.0f / (k * k);
#pragma unroll
  for (int c = 0; c < 8; c++) a[c] *= inv;
  store8(y + pix * ycs + g * 8, a);
}

// 2x2 average pool (DenseNet transitions): the four window loads in flight, same summation order
__global__ void avgpool2_fwd(const bf16* __restrict__ x, int n, int h, int w, int C, int xcs, int oh, int ow,
                             bf16* __restrict__ y, int ycs) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * oh * ow * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ox = (int)(pix % ow), oy = (int)((pix / ow) % oh), b = (int)(pix / ((int64_t)ow * oh));
  float v[4][8], a[8] = {0};
#pragma unroll
  for (int q = 0; q < 4; q++)
    load8(x + (((int64_t)b * h + oy * 2 + (q >> 1)) * w + ox * 2 + (q & 1)) * xcs + g * 8, v[q]);
#pragma unroll
  for (int q = 0; q < 4; q++)
#pragma unroll
    for (int c = 0; c < 8; c++) a[c] += v[q][c];
#pragma unroll
  for (int c = 0; c < 8; c++) a[c] *= 0.25f;
  store8(y + pix * ycs + g * 8, a);
}

__global__ void avgpool_bwd(const bf16* __restrict__ dy, int n, int h, int w, int C, int k, int oh, int ow,
                            bf16* __restrict__ dx, int dxcs) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * h * w * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int ix = (int)(pix % w), iy = (int)((pix / w) % h), b = (int)(pix / ((int64_t)w * h));
  float v[8];
  const int ox = ix / k, oy = iy / k;
  if (ox < ow && oy < oh) {
    load8(dy + (((int64_t)b * oh + oy) * ow + ox) * C + g * 8, v);
    const float inv = 1.0f / (k * k);
#pragma unroll
    for (int c = 0; c < 8; c++) v[c] *= inv;
  } else {
#pragma unroll
    for (int c = 0; c < 8; c++) v[c] = 0.f;
  }
  store8(dx + pix * dxcs + g * 8, v);
}

// global average pool: x [n][hw][C] (stride xcs) -> y [n][C] bf16
__global__ void gap_fwd(const bf16* __restrict__ x, int n, int hw, int C, int xcs, bf16* __restrict__ y) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * G) return;
  const int b = i / G, g = i % G;
  float a[8] = {0};
  for (int j = 0; j < hw; j++) {
    float v[8];
    load8(x + ((int64_t)b * hw + j) * xcs + g * 8, v);
#pragma unroll
    for (int c = 0; c < 8; c++) a[c] += v[c];
  }
  const float inv = 1.0f / hw;
#pragma unroll
  for (int c = 0; c < 8; c++) a[c] *= inv;
  store8(y + (int64_t)b * C + g * 8, a);
}

__global__ void gap_bwd(const bf16* __restrict__ dy, int n, int hw, int C, bf16* __restrict__ dx) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * hw * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int b = (int)(pix / hw);
  float v[8];
  load8(dy + (int64_t)b * C + g * 8, v);
  const float inv = 1.0f / hw;
#pragma unroll
  for (int c = 0; c < 8; c++) v[c] *= inv;
  store8(dx + pix * C + g * 8, v);
}

// ---- softmax cross-entropy: one warp per row, classes <= 32*4 ----------------------------
__global__ void softmax_xent(const float* __restrict__ logits, int B, int C, const int32_t* __restrict__ labels,
                             float scale, float* __restrict__ row_loss, bf16* __restrict__ dlogits, int ldd) {
  CVB_PDL_PROLOGUE();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= B) return;
  const float* l = logits + (int64_t)row * ldd;   // logits and dlogits share the row stride
  float v[4];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 4; j++) { const int c = lane + 32 * j; v[j] = c < C ? l[c] : -INFINITY; mx = fmaxf(mx, v[j]); }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float se = 0.f;
#pragma unroll
  for (int j = 0; j < 4; j++) { const int c = lane + 32 * j; if (c < C) se += expf(v[j] - mx); }
  for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  const int lab = labels[row];
  const float lse = logf(se) + mx;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int c = lane + 32 * j;
    if (c < C) {
      const float pr = expf(v[j] - lse);
      dlogits[(int64_t)row * ldd + c] = __float2bfloat16_rn((pr - (c == lab ? 1.f : 0.f)) * scale);
      if (c == lab) row_loss[row] = lse - v[j];
    }
  }
}

// softmax-CE + mean loss in one launch: every block writes its rows' losses, the last block
// to finish (device-scope counter) sums all rows in index order -> deterministic.
__global__ void softmax_xent_mean(const float* __restrict__ logits, int B, int C, const int32_t* __restrict__ labels,
                                  float scale, float* __restrict__ row_loss, bf16* __restrict__ dlogits, int ldd,
                                  float* __restrict__ loss_out, unsigned* __restrict__ counter) {
  CVB_PDL_PROLOGUE();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row < B) {
    const float* l = logits + (int64_t)row * ldd;
    float v[4];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 4; j++) { const int c = lane + 32 * j; v[j] = c < C ? l[c] : -INFINITY; mx = fmaxf(mx, v[j]); }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f;
#pragma unroll
    for (int j = 0; j < 4; j++) { const int c = lane + 32 * j; if (c < C) se += expf(v[j] - mx); }
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int lab = labels[row];
    const float lse = logf(se) + mx;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int c = lane + 32 * j;
      if (c < C) {
        const float pr = expf(v[j] - lse);
        dlogits[(int64_t)row * ldd + c] = __float2bfloat16_rn((pr - (c == lab ? 1.f : 0.f)) * scale);
        if (c == lab) row_loss[row] = lse - v[j];
      }
    }
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double sh[256];
  double a = 0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) a += __ldcg(row_loss + i);
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) { loss_out[0] = (float)(sh[0] / B); *counter = 0u; }
}

// deterministic sum of n floats into out[0] (single block)
__global__ void sum_small(const float* __restrict__ x, int n, float scale, float* __restrict__ out) {
  CVB_PDL_PROLOGUE();
  __shared__ double sh[256];
  double a = 0;
  for (int i = threadIdx.x; i < n; i += 256) a += x[i];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = (float)(sh[0] * scale);
}

// ---- misc -------------------------------------------------------------------------------
// Split-K reduction out[i] (+)= scale * sum_s part[s][i].  The split count of a conv wgrad is
// large (up to 148) and its element count small, so one thread per element would be a chain
// of `splits` dependent L2 round trips: instead a 256-thread block covers 32 consecutive
// elements (lanes, coalesced) x 8 split groups (warps); each thread sums a contiguous range of
// splits with 8 loads in flight, and the 8 group sums are added in fixed order (deterministic).
__global__ void reduce_splits_flat(const float* __restrict__ part, int splits, int64_t count, float* __restrict__ out,
                                   int accumulate, float scale) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  float a = 0.f;
  for (int s = 0; s < splits; s++) a += part[s * count + i];
  a *= scale;
  out[i] = accumulate ? out[i] + a : a;
}

// The same over float4 groups (count % 4 == 0, 16-byte aligned): four splits' loads in flight
// per thread, summed in split order (identical result to the scalar form).
__global__ void reduce_splits_flat4(const float4* __restrict__ part, int splits, int64_t count4,
                                    float4* __restrict__ out, int accumulate, float scale) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count4) return;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  int s = 0;
  for (; s + 4 <= splits; s += 4) {
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = __ldcg(part + (int64_t)(s + j) * count4 + i);
#pragma unroll
    for (int j = 0; j < 4; j++) { a.x += v[j].x; a.y += v[j].y; a.z += v[j].z; a.w += v[j].w; }
  }
  for (; s < splits; s++) {
    const float4 v = __ldcg(part + (int64_t)s * count4 + i);
    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
  }
  a.x *= scale; a.y *= scale; a.z *= scale; a.w *= scale;
  if (accumulate) { const float4 o = out[i]; a.x = o.x + a.x; a.y = o.y + a.y; a.z = o.z + a.z; a.w = o.w + a.w; }
  out[i] = a;
}

constexpr int RS_GROUPS = 8;
__global__ void __launch_bounds__(256) reduce_splits(const float* __restrict__ part, int splits, int64_t count,
                                                     float* __restrict__ out, int accumulate, float scale) {
  CVB_PDL_PROLOGUE();
  __shared__ float sh[RS_GROUPS][32];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  const int per = (splits + RS_GROUPS - 1) / RS_GROUPS;
  const int s0 = grp * per, s1 = min(splits, s0 + per);
  float a = 0.f;
  if (i < count) {
    int s = s0;
    for (; s + 8 <= s1; s += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = __ldcg(part + (int64_t)(s + j) * count + i);
#pragma unroll
      for (int j = 0; j < 8; j++) a += v[j];
    }
    for (; s < s1; s++) a += __ldcg(part + (int64_t)s * count + i);
  }
  sh[grp][lane] = a;
  __syncthreads();
  if (grp == 0 && i < count) {
    float t = sh[0][lane];
#pragma unroll
    for (int g = 1; g < RS_GROUPS; g++) t += sh[g][lane];
    t *= scale;
    out[i] = accumulate ? out[i] + t : t;
  }
}

// split-K epilogue of a dense layer: out[r][c] = act(sum_s part[s][r][c] + bias[c])
__global__ void reduce_splits_act(const float* __restrict__ part, int splits, int rows, int cols,
                                  const float* __restrict__ bias, int relu, void* __restrict__ out, int out_f32,
                                  int64_t ldo) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t count = (int64_t)rows * cols;
  if (i >= count) return;
  const int r = (int)(i / cols), c = (int)(i - (int64_t)r * cols);
  float a = 0.f;
  for (int s = 0; s < splits; s++) a += part[s * count + i];
  if (bias) a += bias[c];
  if (relu) a = fmaxf(a, 0.f);
  if (out_f32) reinterpret_cast<float*>(out)[(int64_t)r * ldo + c] = a;
  else reinterpret_cast<bf16*>(out)[(int64_t)r * ldo + c] = __float2bfloat16_rn(a);
}

// wt[ci][kh'][kw'][co] = w[co][KH-1-kh'][KW-1-kw'][ci]
__global__ void weight_flip(const bf16* __restrict__ w, int cout, int kh, int kw, int cin, bf16* __restrict__ wt) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)cout * kh * kw * cin;
  if (i >= total) return;
  const int co = (int)(i % cout);
  int64_t r = i / cout;
  const int x = (int)(r % kw); r /= kw;
  const int y = (int)(r % kh);
  const int ci = (int)(r / kh);
  wt[i] = w[(((int64_t)co * kh + (kh - 1 - y)) * kw + (kw - 1 - x)) * cin + ci];
}

// All stride-1 dgrad weight flips of the model in one launch (run after the optimiser):
// desc[l] = {src offset, dst offset, cout, kh, kw, cin} into the flat bf16 weight / flipped
// buffers; blockIdx.y = layer.
__global__ void weight_flip_batched(const bf16* __restrict__ pb, bf16* __restrict__ fb, const int64_t* __restrict__ desc) {
  // 32 x 32 (cout x cin) tiles of one tap through shared memory: coalesced 64-byte rows in and
  // out (the element-wise form with 64-bit index divisions ran at 0.9 TB/s); the flipped tap
  // of source tap t is taps-1-t (both spatial axes reversed)
  __shared__ bf16 tile[32][34];
  CVB_PDL_PROLOGUE();
  const int64_t* d = desc + 6 * blockIdx.y;
  const int64_t src = d[0], dst = d[1];
  const int cout = (int)d[2], kh = (int)d[3], kw = (int)d[4], cin = (int)d[5];
  const int taps = kh * kw, tco = (cout + 31) / 32, tci = (cin + 31) / 32, per_tap = tco * tci;
  const int ntiles = taps * per_tap;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 256 threads: 32 x 8
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tap = t / per_tap, rem = t - tap * per_tap, co0 = (rem / tci) * 32, ci0 = (rem % tci) * 32;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int co = co0 + ty + 8 * k, ci = ci0 + tx;
      if (co < cout && ci < cin) tile[ty + 8 * k][tx] = pb[src + ((int64_t)co * taps + tap) * cin + ci];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int ci = ci0 + ty + 8 * k, co = co0 + tx;
      if (co < cout && ci < cin) fb[dst + ((int64_t)ci * taps + (taps - 1 - tap)) * cout + co] = tile[tx][ty + 8 * k];
    }
    __syncthreads();
  }
}

// Batched transposes of bf16 matrices: job j = {src offset, dst offset, rows, cols, src row
// stride, dst row stride}: dst[c * dst_ld + r] = src[r * src_ld + c] (elements).  One launch
// refreshes every derived weight layout of a step after the optimiser: the flipped stride-1
// dgrad weights (one job per tap) and the per-output-parity class weights of the stride-2
// dgrads (one job per (class, tap)).  32 x 32 tiles through shared memory, 64-byte rows in/out.
// 64x64 tiles of every job in one flat tile index (a per-block prefix over the jobs' tile counts,
// then a binary search per tile): the grid is sized by the total work, not by the largest job
// times the job count (the 32x32 form launched ~50k mostly idle blocks per ResNet-18 step).  Jobs
// whose offsets, strides and extents are multiples of 8 move 16-byte vectors through a swizzled
// tile (conflict-free scatter, 128-byte coalesced rows both ways); others take an element path.
constexpr int TP_T = 64;
constexpr int TP_MAX_JOBS = 8192;

__device__ __forceinline__ int tp_tiles(int64_t rows, int64_t cols) {
  return (int)(((rows + TP_T - 1) / TP_T) * ((cols + TP_T - 1) / TP_T));
}

__global__ void __launch_bounds__(256) transpose_batched(const bf16* __restrict__ src, bf16* __restrict__ dst,
                                                         const int64_t* __restrict__ desc, int njobs) {
  extern __shared__ int s_pref[];                 // njobs + 1 tile prefix
  __shared__ __align__(16) bf16 tile[TP_T][TP_T];   // [col][row], 16-byte chunks XOR-swizzled by col
  __shared__ int s_warp[8];
  CVB_PDL_PROLOGUE();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // ---- exclusive prefix of the jobs' tile counts (each thread a contiguous segment) ----
  const int seg = (njobs + 255) / 256, j0 = min(njobs, tid * seg), j1 = min(njobs, j0 + seg);
  int mine = 0;
  for (int j = j0; j < j1; j++) mine += tp_tiles(desc[6 * j + 2], desc[6 * j + 3]);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < wid; w++) base += s_warp[w];
  int run = base + incl - mine;
  for (int j = j0; j < j1; j++) { s_pref[j] = run; run += tp_tiles(desc[6 * j + 2], desc[6 * j + 3]); }
  if (tid == 255) s_pref[njobs] = base + incl;
  __syncthreads();
  const int total = s_pref[njobs];
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int lo = 0, hi = njobs - 1;   // last job with s_pref[j] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pref[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const int64_t* d = desc + 6 * lo;
    const int64_t so = d[0], dof = d[1], rows = d[2], cols = d[3], sld = d[4], dld = d[5];
    const int lt = t - s_pref[lo], tc = (int)((cols + TP_T - 1) / TP_T);
    const int64_t r0 = (int64_t)(lt / tc) * TP_T, c0 = (int64_t)(lt % tc) * TP_T;
    if (((so | dof | rows | cols | sld | dld) & 7) == 0) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int i = tid + 256 * h, r = i >> 3, ch = i & 7;
        if (r0 + r < rows && c0 + ch * 8 < cols) {
          const uint4 v = *reinterpret_cast<const uint4*>(src + so + (r0 + r) * sld + c0 + ch * 8);
          const bf16* e = reinterpret_cast<const bf16*>(&v);
          // element (r, c = 8ch + k) -> tile[c][8 * ((r >> 3) ^ ch) + (r & 7)]  (c >> 3 == ch)
          const int col = (((r >> 3) ^ ch) << 3) | (r & 7);
#pragma unroll
          for (int k = 0; k < 8; k++) tile[ch * 8 + k][col] = e[k];
        }
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int i = tid + 256 * h, c = i >> 3, rch = i & 7;
        if (c0 + c < cols && r0 + rch * 8 < rows)
          *reinterpret_cast<uint4*>(dst + dof + (c0 + c) * dld + r0 + rch * 8) =
              *reinterpret_cast<const uint4*>(&tile[c][(rch ^ (c >> 3)) << 3]);
      }
      __syncthreads();
    } else {
      for (int i = tid; i < TP_T * TP_T; i += 256) {
        const int64_t r = r0 + (i & (TP_T - 1)), c = c0 + (i >> 6);
        if (r < rows && c < cols) dst[dof + c * dld + r] = src[so + r * sld + c];
      }
    }
  }
}

// ---- space-to-depth stem (7x7 stride-2 pad-3 conv == 4x4 stride-1 conv on 2x2 s2d input) ----
// xs[n][i][j][(2a+b)*C + c] = x[n][2i+a][2j+b][c]
__global__ void space_to_depth2(const bf16* __restrict__ x, int n, int h, int w, int C, bf16* __restrict__ xs) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8, oh = h / 2, ow = w / 2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one 16-byte group of the output
  if (i >= (int64_t)n * oh * ow * 4 * G) return;
  const int g = (int)(i % (4 * G));
  const int64_t pix = i / (4 * G);
  const int ph = g / G, cg = g % G, a = ph >> 1, b = ph & 1;
  const int j = (int)(pix % ow), ii = (int)((pix / ow) % oh), nn = (int)(pix / ((int64_t)ow * oh));
  *reinterpret_cast<uint4*>(xs + pix * 4 * C + g * 8) =
      *reinterpret_cast<const uint4*>(x + (((int64_t)nn * h + 2 * ii + a) * w + 2 * j + b) * C + cg * 8);
}

// ws[co][u][v][(2a+b)*C + c] = w[co][2u+a-1][2v+b-1][c] (zero where the 7x7 tap does not exist)
__global__ void s2d_weights(const bf16* __restrict__ w, int cout, int C, bf16* __restrict__ ws) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)cout * 16 * 4 * C) return;
  const int c = (int)(i % C);
  int64_t r = i / C;
  const int ph = (int)(r % 4); r /= 4;
  const int v = (int)(r % 4); r /= 4;
  const int u = (int)(r % 4);
  const int co = (int)(r / 4);
  const int kh = 2 * u + (ph >> 1) - 1, kw = 2 * v + (ph & 1) - 1;
  ws[i] = (kh >= 0 && kw >= 0) ? w[(((int64_t)co * 7 + kh) * 7 + kw) * C + c] : __float2bfloat16_rn(0.f);
}

// dw[co][kh][kw][c] (+)= dws[co][u][v][(2a+b)*C + c] with kh = 2u+a-1, kw = 2v+b-1 (fp32)
__global__ void s2d_weights_grad(const float* __restrict__ dws, int cout, int C, float* __restrict__ dw) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)cout * 49 * C) return;
  const int c = (int)(i % C);
  int64_t r = i / C;
  const int kw = (int)(r % 7); r /= 7;
  const int kh = (int)(r % 7);
  const int co = (int)(r / 7);
  const int u = (kh + 1) >> 1, a = (kh + 1) & 1, v = (kw + 1) >> 1, b = (kw + 1) & 1;
  dw[i] = dws[((((int64_t)co * 4 + u) * 4 + v) * 4 + (2 * a + b)) * C + c];
}

__global__ void zero_upsample(const bf16* __restrict__ dy, int n, int oh, int ow, int C, int dycs, bf16* __restrict__ out,
                              int uh, int uw) {
  CVB_PDL_PROLOGUE();
  const int G = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * uh * uw * G) return;
  const int g = (int)(i % G);
  const int64_t pix = i / G;
  const int x = (int)(pix % uw), y = (int)((pix / uw) % uh), b = (int)(pix / ((int64_t)uw * uh));
  uint4 v = make_uint4(0, 0, 0, 0);
  if (!(x & 1) && !(y & 1)) v = *reinterpret_cast<const uint4*>(dy + (((int64_t)b * oh + (y >> 1)) * ow + (x >> 1)) * dycs + g * 8);
  *reinterpret_cast<uint4*>(out + pix * C + g * 8) = v;
}

// column sums of a row-major [rows][cols] bf16/fp32 matrix -> fp32 (bias gradients)
__global__ void col_sum(const void* __restrict__ x, int is_f32, int64_t rows, int cols, int64_t ld, float* __restrict__ out,
                        int accumulate) {
  CVB_PDL_PROLOGUE();
  // 32 columns x 32 row lanes per block; fixed-order two-level sum (deterministic)
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int rl = threadIdx.x >> 5;
  __shared__ float sh[32][33];
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (c < cols) {
    auto at = [&](int64_t r) -> float {
      return is_f32 ? __ldg(reinterpret_cast<const float*>(x) + r * ld + c)
                    : __bfloat162float(reinterpret_cast<const bf16*>(x)[r * ld + c]);
    };
    int64_t r = rl;
    for (; r + 96 < rows; r += 128) { a0 += at(r); a1 += at(r + 32); a2 += at(r + 64); a3 += at(r + 96); }
    for (; r < rows; r += 32) a0 += at(r);
  }
  sh[rl][threadIdx.x & 31] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (rl == 0 && c < cols) {
    float s = 0.f;
    for (int l = 0; l < 32; l++) s += sh[l][threadIdx.x];
    out[c] = accumulate ? out[c] + s : s;
  }
}

// relu backward on a bf16 matrix in place: dx = dy * (y > 0)
__global__ void relu_bwd(bf16* __restrict__ dy, const bf16* __restrict__ y, int64_t n8) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  float d[8], v[8];
  load8(dy + i * 8, d);
  load8(y + i * 8, v);
#pragma unroll
  for (int k = 0; k < 8; k++) if (!(v[k] > 0.f)) d[k] = 0.f;
  store8(dy + i * 8, d);
}

__global__ void relu_fwd(bf16* __restrict__ x, int64_t n8) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  float v[8];
  load8(x + i * 8, v);
#pragma unroll
  for (int k = 0; k < 8; k++) v[k] = fmaxf(v[k], 0.f);
  store8(x + i * 8, v);
}

// torch.optim.Adam (no weight decay, no amsgrad) over flat fp32 buffers; refreshes the
// bf16 compute copy.  step_size = lr / (1 - b1^t), inv_bc2_sqrt = 1 / sqrt(1 - b2^t).
// Device-side step counter so a captured CUDA graph can be replayed: step += 1 and the
// bias-correction factors are recomputed on the device every replay.
__global__ void adam_step(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                          bf16* __restrict__ pb, int64_t n, float b1, float b2, float eps, float step_size,
                          float inv_bc2_sqrt, float grad_scale, const float* __restrict__ sched,
                          const float* __restrict__ skip) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (skip && *skip != 0.f)) return;
  if (sched) { step_size = sched[0]; inv_bc2_sqrt = sched[1]; }
  const float gi = g[i] * grad_scale;
  const float mi = b1 * m[i] + (1.f - b1) * gi;
  const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  const float denom = sqrtf(vi) * inv_bc2_sqrt + eps;
  const float pi = p[i] - step_size * (mi / denom);
  p[i] = pi;
  if (pb) pb[i] = __float2bfloat16_rn(pi);
}

// Device-counter Adam in one launch.  sched holds the bias corrections of the UPCOMING step
// (1/(1-b1^t), 1/sqrt(1-b2^t)), written by the last CTA of the previous launch (all CTAs
// have read them by then), so CTAs only read two floats; the very first step (counter 0)
// derives them in place.  The last CTA also advances the step counter.
__device__ __forceinline__ void adam_bias_corr(int t, float b1, float b2, float* c1, float* c2) {
  *c1 = (float)(1.0 / (1.0 - pow((double)b1, (double)t)));
  *c2 = (float)(1.0 / sqrt(1.0 - pow((double)b2, (double)t)));
}

__global__ void adam_step_dev(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                              float* __restrict__ v, bf16* __restrict__ pb, int64_t n, float lr, float b1, float b2,
                              float eps, float grad_scale, int32_t* step, float* sched, unsigned* counter,
                              const float* __restrict__ skip) {
  CVB_PDL_PROLOGUE();
  // verdict gate: a non-zero skip word (a failed shard tag on any rank, summed into the
  // gradient exchange) leaves parameters, moments and the step counter untouched.  The word
  // is written only by stream-ordered predecessors, so every CTA reads the same value.
  if (skip && *skip != 0.f) return;
  __shared__ float ss[2];
  __shared__ bool last;
  __shared__ int t_s;
  if (threadIdx.x == 0) {
    const int t = *(volatile int32_t*)step + 1;
    t_s = t;
    if (t == 1) adam_bias_corr(1, b1, b2, &ss[0], &ss[1]);
    else { ss[0] = *(volatile float*)&sched[0]; ss[1] = *(volatile float*)&sched[1]; }
  }
  __syncthreads();
  // grid-stride (a few CTAs per SM): the completion counter below is one same-address atomic
  // per CTA, which serialises in L2 -- thousands of CTAs would cost ~10 us
  const float step_size = lr * ss[0], inv_bc2_sqrt = ss[1];
  const int64_t n4 = (n & 3) == 0 && !(((uintptr_t)p | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v) & 15) &&
                             !((uintptr_t)pb & 7) ? n / 4 : 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n4; k += (int64_t)gridDim.x * blockDim.x) {
    float4 pv = reinterpret_cast<float4*>(p)[k], mv = reinterpret_cast<float4*>(m)[k], vv = reinterpret_cast<float4*>(v)[k];
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + k);
    float* pp = &pv.x; float* mp = &mv.x; float* vp = &vv.x; const float* gp = &gv.x;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const float gi = gp[j] * grad_scale;
      mp[j] = b1 * mp[j] + (1.f - b1) * gi;
      vp[j] = b2 * vp[j] + (1.f - b2) * gi * gi;
      const float denom = sqrtf(vp[j]) * inv_bc2_sqrt + eps;
      pp[j] = pp[j] - step_size * (mp[j] / denom);
    }
    reinterpret_cast<float4*>(p)[k] = pv;
    reinterpret_cast<float4*>(m)[k] = mv;
    reinterpret_cast<float4*>(v)[k] = vv;
    if (pb) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pv.x, pv.y), hi = __floats2bfloat162_rn(pv.z, pv.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(pb)[k] = u;
    }
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i] * grad_scale;
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float denom = sqrtf(vi) * inv_bc2_sqrt + eps;
    const float pi = p[i] - step_size * (mi / denom);
    p[i] = pi;
    if (pb) pb[i] = __float2bfloat16_rn(pi);
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *step = t_s;
    adam_bias_corr(t_s + 1, b1, b2, &sched[0], &sched[1]);   // the next step's corrections
    *counter = 0u;
  }
}

// torch.optim.SGD with momentum (dampening 0, no nesterov) + optional weight decay
__global__ void sgd_step(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ buf, bf16* __restrict__ pb,
                         int64_t n, float lr, float momentum, float wd, float grad_scale, int first) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float d = g[i] * grad_scale + wd * p[i];
  if (momentum != 0.f) { d = first ? d : momentum * buf[i] + d; buf[i] = d; }
  const float pi = p[i] - lr * d;
  p[i] = pi;
  if (pb) pb[i] = __float2bfloat16_rn(pi);
}

// strided 2-D cast: y[r][c] = bf16(x[r][c]) with row strides (DenseNet concat-gradient slices)
__global__ void cast_rows(const float* __restrict__ x, int64_t ldx, bf16* __restrict__ y, int64_t ldy, int64_t rows,
                          int cols) {
  CVB_PDL_PROLOGUE();
  const int G = cols / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * G) return;
  const int64_t r = i / G;
  const int g = (int)(i - r * G);
  const float4* s = reinterpret_cast<const float4*>(x + r * ldx + g * 8);
  float4 a = s[0], b = s[1];
  float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  store8(y + r * ldy + g * 8, v);
}

__global__ void cast_f32_bf16(const float* __restrict__ x, bf16* __restrict__ y, int64_t n) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __float2bfloat16_rn(x[i]);
}

inline unsigned nblocks(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

int stats_blocks(int64_t rows, int C, int64_t* rpb) {
  int nsm = cvb_num_sms();
  int64_t target = (int64_t)nsm * 2;
  int64_t per = (rows + target - 1) / target;
  if (per < 64) per = 64;
  *rpb = per;
  return (int)((rows + per - 1) / per);
}

}  // namespace

// ======================================= C ABI ==========================================
#define STREAM (cudaStream_t)stream

// Batch-norm forward statistics over rows of x ([rows][C], channel stride xcs).  ws must hold
// cvb_bn_workspace_floats(rows, C) floats.  Writes mean/rstd; updates running stats if given.
CVB_API int64_t cvb_bn_fused_workspace_floats(int C);
CVB_API int64_t cvb_bn_workspace_floats(int64_t rows, int C) {
  int64_t rpb;
  const int64_t a = (int64_t)stats_blocks(rows, C, &rpb) * 2 * C, b = cvb_bn_fused_workspace_floats(C);
  return a > b ? a : b;
}

CVB_API int cvb_bn_stats(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd, float eps,
                         float* run_mean, float* run_var, float momentum, void* stream) {
  if (C % 8 || C / 8 > ST_THREADS) { cvb_set_error("bn_stats: C must be a multiple of 8, <= 2048"); return CVB_EINVAL; }
  int64_t rpb;
  int nb = stats_blocks(rows, C, &rpb);
  const int G = C / 8, RL = ST_THREADS / G;
  cvb_launch(chan_stats_partial, nb, ST_THREADS, RL * G * 16 * sizeof(float), STREAM, (const bf16*)x, rows, C, xcs, rpb, ws);
  cvb_launch(bn_finalize, (C + 31) / 32, FIN_WARPS * 32, 0, STREAM, ws, nb, C, (double)rows, eps, mean, rstd, run_mean,
                                                             run_var, momentum);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_bn_apply(const void* x, int64_t rows, int C, int xcs, const float* mean, const float* rstd,
                         const float* gamma, const float* beta, const void* res, int rcs, int relu, void* y, int ycs,
                         int ycoff, void* stream) {
  cvb_launch(bn_apply, nblocks(rows * (C / 8)), 256, 0, STREAM, (const bf16*)x, rows, C, xcs, mean, rstd, gamma, beta,
                                                       (const bf16*)res, rcs, relu, (bf16*)y, ycs, ycoff);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

// Batch-norm (+ReLU) backward.  dy: grad of the layer output; y (optional): layer output for
// the ReLU mask (else recomputed from x).  Writes dgamma/dbeta (fp32) and dx (bf16, stride
// dxcs) or, if dx32 != NULL, fp32 dx (accumulated when accum32).  dz_out (optional, [rows][C]
// bf16) receives the masked output gradient (the residual branch's gradient).
CVB_API int cvb_bn_backward(const void* dy, int dycs, const void* x, int xcs, const void* y, int ycs, int64_t rows, int C,
                            const float* mean, const float* rstd, const float* gamma, const float* beta, int relu,
                            float* ws, float* dgamma, float* dbeta, void* dx, int dxcs, float* dx32, int accum32,
                            void* dz_out, void* stream) {
  if (C % 8 || C / 8 > ST_THREADS) { cvb_set_error("bn_backward: bad C"); return CVB_EINVAL; }
  int64_t rpb;
  int nb = stats_blocks(rows, C, &rpb);
  const int G = C / 8, RL = ST_THREADS / G;
  cvb_launch(bn_bwd_partial, nb, ST_THREADS, RL * G * 16 * sizeof(float), STREAM, 
      (const bf16*)dy, dycs, (const bf16*)x, xcs, (const bf16*)y, ycs, rows, C, mean, rstd, gamma, beta, relu, rpb, ws,
      (bf16*)dz_out);
  cvb_launch(bn_bwd_finalize, (C + 31) / 32, FIN_WARPS * 32, 0, STREAM, ws, nb, C, dbeta, dgamma);
  if (dx || dx32)
    cvb_launch(bn_bwd_apply, nblocks(rows * G), 256, 0, STREAM, (const bf16*)dy, dycs, (const bf16*)x, xcs, (const bf16*)y, ycs,
                                                        rows, C, mean, rstd, gamma, beta, relu, dbeta, dgamma, (bf16*)dx,
                                                        dxcs, dx32, accum32);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_maxpool_fwd(const void* x, int n, int h, int w, int C, int k, int s, int p, void* y, int oh, int ow,
                            int ycs, void* stream) {
  if (k == 2 && s == 2 && p == 0 && h == 2 * oh && w == 2 * ow)
    cvb_launch(maxpool2_fwd, nblocks((int64_t)n * oh * ow * (C / 8)), 256, 0, STREAM, (const bf16*)x, n, h, w, C, oh, ow,
               (bf16*)y, ycs);
  else
    cvb_launch(maxpool_fwd, nblocks((int64_t)n * oh * ow * (C / 8)), 256, 0, STREAM, (const bf16*)x, n, h, w, C, k, s, p, oh,
               ow, (bf16*)y, ycs);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_maxpool_bwd(const void* x, const void* dy, int n, int h, int w, int C, int k, int s, int p, int oh,
                            int ow, void* dx, void* stream) {
  if (k == 2 && s == 2 && p == 0 && h == 2 * oh && w == 2 * ow)
    cvb_launch(maxpool2_bwd, nblocks((int64_t)n * oh * ow * (C / 8)), 256, 0, STREAM, (const bf16*)x, (const bf16*)dy, n, h, w,
                                                                              C, oh, ow, (bf16*)dx);
  else
    cvb_launch(maxpool_bwd, nblocks((int64_t)n * h * w * (C / 8)), 256, 0, STREAM, (const bf16*)x, (const bf16*)dy, n, h, w, C,
                                                                           k, s, p, oh, ow, (bf16*)dx);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_maxpool_fwd_idx(const void* x, int n, int h, int w, int C, int k, int s, int p, void* y, int oh, int ow,
                                int ycs, void* idx, void* stream) {
  if (C % 8 || k * k > 256) { cvb_set_error("maxpool_fwd_idx: bad shape"); return CVB_EINVAL; }
  if (k == 3 && s == 2 && p == 1 && oh == (h - 1) / 2 + 1 && ow == (w - 1) / 2 + 1)
    cvb_launch(maxpool3s2_fwd_idx, nblocks((int64_t)n * oh * ow * (C / 8)), 256, 0, STREAM, (const bf16*)x, n, h, w, C, oh,
               ow, (bf16*)y, ycs, (uint8_t*)idx);
  else
    cvb_launch(maxpool_fwd_idx, nblocks((int64_t)n * oh * ow * (C / 8)), 256, 0, STREAM, (const bf16*)x, n, h, w, C, k, s, p,
               oh, ow, (bf16*)y, ycs, (uint8_t*)idx);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_maxpool_bwd_idx(const void* idx, const void* dy, int n, int h, int w, int C, int k, int s, int p, int oh,
                                int ow, void* dx, void* stream) {
  if (k == 3 && s == 2 && p == 1 && oh == (h - 1) / 2 + 1 && ow == (w - 1) / 2 + 1)
    cvb_launch(maxpool3s2_bwd_idx, nblocks((int64_t)n * h * w * (C / 8)), 256, 0, STREAM, (const uint8_t*)idx,
               (const bf16*)dy, n, h, w, C, oh, ow, (bf16*)dx);
  else
    cvb_launch(maxpool_bwd_idx, nblocks((int64_t)n * h * w * (C / 8)), 256, 0, STREAM, (const uint8_t*)idx, (const bf16*)dy,
               n, h, w, C, k, s, p, oh, ow, (bf16*)dx);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_avgpool_fwd(const void* x, int n, int h, int w, int C, int xcs, int k, void* y, int ycs, void* stream) {
  const int oh = h / k, ow = w / k;
  if (k == 2)
    cvb_launch(avgpool2_fwd, nblocks((int64_t)n * oh * ow * (C / 8)), 256, 0, STREAM, (const bf16*)x, n, h, w, C, xcs, oh, ow,
               (bf16*)y, ycs);
  else
    cvb_launch(avgpool_fwd, nblocks((int64_t)n * oh * ow * (C / 8)), 256, 0, STREAM, (const bf16*)x, n, h, w, C, xcs, k, oh,
               ow, (bf16*)y, ycs);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_avgpool_bwd(const void* dy, int n, int h, int w, int C, int k, void* dx, int dxcs, void* stream) {
  const int oh = h / k, ow = w / k;
  cvb_launch(avgpool_bwd, nblocks((int64_t)n * h * w * (C / 8)), 256, 0, STREAM, (const bf16*)dy, n, h, w, C, k, oh, ow, (bf16*)dx, dxcs);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_gap_fwd(const void* x, int n, int hw, int C, int xcs, void* y, void* stream) {
  cvb_launch(gap_fwd, nblocks((int64_t)n * (C / 8)), 256, 0, STREAM, (const bf16*)x, n, hw, C, xcs, (bf16*)y);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_gap_bwd(const void* dy, int n, int hw, int C, void* dx, void* stream) {
  cvb_launch(gap_bwd, nblocks((int64_t)n * hw * (C / 8)), 256, 0, STREAM, (const bf16*)dy, n, hw, C, (bf16*)dx);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

// Softmax cross-entropy: loss_out[0] = mean over the B rows * loss_scale; dlogits (bf16,
// row stride ldd) = (softmax - onehot) * grad_scale.  row_ws: B floats.
CVB_API int cvb_softmax_xent(const float* logits, int B, int C, const int32_t* labels, float grad_scale, float* row_ws,
                             float* loss_out, void* dlogits, int ldd, void* stream) {
  if (C > 128) { cvb_set_error("softmax_xent: C > 128"); return CVB_EINVAL; }
  static unsigned* counters[64] = {nullptr};
  int dev = 0;
  CVB_CUDA(cudaGetDevice(&dev));
  if (!counters[dev]) {
    CVB_CUDA(cudaMalloc(&counters[dev], sizeof(unsigned)));
    CVB_CUDA(cudaMemset(counters[dev], 0, sizeof(unsigned)));
    CVB_CUDA(cudaDeviceSynchronize());
  }
  cvb_launch(softmax_xent_mean, nblocks((int64_t)B * 32), 256, 0, STREAM, logits, B, C, labels, grad_scale, row_ws,
             (bf16*)dlogits, ldd, loss_out, counters[dev]);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_reduce_splits(const float* part, int splits, int64_t count, float* out, int accumulate, float scale,
                              void* stream) {
  if (splits >= 16)   // deep split-K (conv wgrad): split groups per element
    cvb_launch(reduce_splits, (int)((count + 31) / 32), 256, 0, STREAM, part, splits, count, out, accumulate, scale);
  else if (count % 4 == 0 && !((uintptr_t)part & 15) && !((uintptr_t)out & 15) && !getenv("CVB_REDUCE_SCALAR"))
    cvb_launch(reduce_splits_flat4, nblocks(count / 4), 256, 0, STREAM, (const float4*)part, splits, count / 4,
               (float4*)out, accumulate, scale);
  else
    cvb_launch(reduce_splits_flat, nblocks(count), 256, 0, STREAM, part, splits, count, out, accumulate, scale);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_reduce_splits_act(const float* part, int splits, int rows, int cols, const float* bias, int relu,
                                  void* out, int out_f32, int64_t ldo, void* stream) {
  cvb_launch(reduce_splits_act, nblocks((int64_t)rows * cols), 256, 0, STREAM, part, splits, rows, cols, bias, relu, out, out_f32,
                                                                      ldo);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_weight_flip(const void* w, int cout, int kh, int kw, int cin, void* wt, void* stream) {
  cvb_launch(weight_flip, nblocks((int64_t)cout * kh * kw * cin), 256, 0, STREAM, (const bf16*)w, cout, kh, kw, cin, (bf16*)wt);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_weight_flip_batched(const void* pb, void* fb, const int64_t* desc_dev, int nlayers, int64_t max_elems,
                                    void* stream) {
  if (nlayers <= 0) return CVB_OK;
  unsigned gx = (unsigned)((max_elems + 1023) / 1024);   // one 32 x 32 tile per CTA iteration
  if (gx > 512) gx = 512;
  if (gx < 1) gx = 1;
  cvb_launch(weight_flip_batched, dim3(gx, nlayers), 256, 0, STREAM, (const bf16*)pb, (bf16*)fb, desc_dev);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_transpose_batched(const void* src, void* dst, const int64_t* desc_dev, int njobs, int64_t max_elems,
                                  void* stream) {
  if (njobs <= 0) return CVB_OK;
  static bool attr = false;
  if (!attr) {
    CVB_CUDA(cudaFuncSetAttribute(transpose_batched, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (TP_MAX_JOBS + 1) * (int)sizeof(int)));
    attr = true;
  }
  for (int j = 0; j < njobs; j += TP_MAX_JOBS) {   // the tile prefix lives in shared memory
    const int nj = njobs - j < TP_MAX_JOBS ? njobs - j : TP_MAX_JOBS;
    const int64_t tiles = (int64_t)nj * ((max_elems + TP_T * TP_T - 1) / (TP_T * TP_T) + 1);
    const int64_t cap = 4ll * cvb_num_sms();
    const unsigned g = (unsigned)(tiles < cap ? tiles : cap);
    cvb_launch(transpose_batched, dim3(g), 256, (size_t)(nj + 1) * sizeof(int), STREAM, (const bf16*)src,
               (bf16*)dst, desc_dev + 6 * (int64_t)j, nj);
    CVB_CHECK_LAUNCH();
  }
  return CVB_OK;
}

// Space-to-depth stem helpers (DenseNet's 7x7 stride-2 stem as a 4x4 stride-1 halo conv).
CVB_API int cvb_space_to_depth2(const void* x, int n, int h, int w, int C, void* xs, void* stream) {
  if (C % 8 || h % 2 || w % 2) { cvb_set_error("space_to_depth2: bad shape"); return CVB_EINVAL; }
  cvb_launch(space_to_depth2, nblocks((int64_t)n * (h / 2) * (w / 2) * (C / 2)), 256, 0, STREAM, (const bf16*)x, n, h,
             w, C, (bf16*)xs);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_s2d_weights(const void* w7, int cout, int C, void* ws, void* stream) {
  cvb_launch(s2d_weights, nblocks((int64_t)cout * 64 * C), 256, 0, STREAM, (const bf16*)w7, cout, C, (bf16*)ws);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_s2d_weights_grad(const float* dws, int cout, int C, float* dw7, void* stream) {
  cvb_launch(s2d_weights_grad, nblocks((int64_t)cout * 49 * C), 256, 0, STREAM, dws, cout, C, dw7);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_zero_upsample(const void* dy, int n, int oh, int ow, int C, int dycs, void* out, void* stream) {
  const int uh = 2 * oh - 1, uw = 2 * ow - 1;
  cvb_launch(zero_upsample, nblocks((int64_t)n * uh * uw * (C / 8)), 256, 0, STREAM, (const bf16*)dy, n, oh, ow, C, dycs, (bf16*)out, uh, uw);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_col_sum(const void* x, int is_f32, int64_t rows, int cols, int64_t ld, float* out, int accumulate,
                        void* stream) {
  cvb_launch(col_sum, (cols + 31) / 32, 1024, 0, STREAM, x, is_f32, rows, cols, ld, out, accumulate);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_relu_fwd(void* x, int64_t n, void* stream) {
  cvb_launch(relu_fwd, nblocks(n / 8), 256, 0, STREAM, (bf16*)x, n / 8);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_relu_bwd(void* dy, const void* y, int64_t n, void* stream) {
  cvb_launch(relu_bwd, nblocks(n / 8), 256, 0, STREAM, (bf16*)dy, (const bf16*)y, n / 8);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

// step > 0: host-side bias correction for that step.  step <= 0: device counter mode --
// step_dev is incremented on the device and the factors land in sched_dev (2 floats).
CVB_API int cvb_adam_step(float* p, const float* g, float* m, float* v, void* pb, int64_t n, float lr, float b1, float b2,
                          float eps, int64_t step, float grad_scale, int32_t* step_dev, float* sched_dev,
                          const float* skip_dev, void* stream) {
  if (step > 0) {
    const double bc1 = 1.0 - pow((double)b1, (double)step), bc2 = 1.0 - pow((double)b2, (double)step);
    cvb_launch(adam_step, nblocks(n), 256, 0, STREAM, p, g, m, v, (bf16*)pb, n, b1, b2, eps, (float)(lr / bc1),
                                              (float)(1.0 / sqrt(bc2)), grad_scale, nullptr, skip_dev);
  } else {
    if (!step_dev || !sched_dev) { cvb_set_error("adam_step: device counter mode needs step_dev/sched_dev"); return CVB_EINVAL; }
    // sched_dev[2] (as an unsigned, zero-initialised by the caller) is the CTA completion counter
    const int64_t nb = nblocks(n), cap = 4 * (int64_t)cvb_num_sms();
    cvb_launch(adam_step_dev, (int)(nb < cap ? nb : cap), 256, 0, STREAM, p, g, m, v, (bf16*)pb, n, lr, b1, b2, eps, grad_scale, step_dev,
               sched_dev, reinterpret_cast<unsigned*>(sched_dev + 2), skip_dev);
  }
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

// slot = (verdict word != 0) ? 1 : 0 -- the step's snapshot of the sticky decrypt verdict,
// taken while no decrypt is in flight; it travels in the gradient exchange and gates Adam.
__global__ void verdict_snapshot(const uint32_t* __restrict__ word, float* __restrict__ slot) {
  CVB_PDL_PROLOGUE();
  if (threadIdx.x == 0) *slot = *word ? 1.f : 0.f;
}

CVB_API int cvb_verdict_snapshot(const uint32_t* word, float* slot, void* stream) {
  if (!word || !slot) { cvb_set_error("verdict_snapshot: null argument"); return CVB_EINVAL; }
  cvb_launch(verdict_snapshot, 1, 32, 0, STREAM, word, slot);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_sgd_step(float* p, const float* g, float* buf, void* pb, int64_t n, float lr, float momentum, float wd,
                         float grad_scale, int first, void* stream) {
  cvb_launch(sgd_step, nblocks(n), 256, 0, STREAM, p, g, buf, (bf16*)pb, n, lr, momentum, wd, grad_scale, first);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_cast_rows(const float* x, int64_t ldx, void* y, int64_t ldy, int64_t rows, int cols, void* stream) {
  if (cols % 8) { cvb_set_error("cast_rows: cols must be a multiple of 8"); return CVB_EINVAL; }
  cvb_launch(cast_rows, nblocks(rows * (cols / 8)), 256, 0, STREAM, x, ldx, (bf16*)y, ldy, rows, cols);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

CVB_API int cvb_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream) {
  cvb_launch(cast_f32_bf16, nblocks(n), 256, 0, STREAM, x, (bf16*)y, n);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}
