// The reference trainer's numeric core on the GPU (K2/K3/K4 of DESIGN.md).
//
// Replaces covault.workload.run_training (/root/reference/pkg/src/covault/workload.py:48-71;
// sigmoid :44-45).  One epoch = one full-batch gradient step (:57-70), split into two
// stream-ordered device calls so the data-parallel trainer can all-reduce the F+1 gradient
// sums between them:
//   cvb_logistic_grad_dev   g_i = sum_r delta_r * x_ri, g_b = sum_r delta_r over the rows given
//   cvb_logistic_apply_dev  w_i -= (lr * g_i) / n,  b -= (lr * g_b) / n        (:68-70)
// Two modes:
//   mode 0 "exact": bit-identical to the reference's Python floats.  Every operation is an
//     explicitly rounded IEEE binary64 op (__dmul_rn/__dadd_rn/__ddiv_rn: no FMA
//     contraction) in the reference's order.  The only parallelism the reference order
//     admits is used: logits are independent per row (one thread per row, features in
//     order, :61-63, reading the feature-major copy Xt so a warp's loads coalesce) and each
//     gradient component is an in-order sum over rows (one thread per feature, rows in file
//     order, :65-67; the CTA stages row tiles through shared memory so the dependent add
//     chains never wait on HBM).  Reproduces DEMO_MODEL_SHA256.
//   mode 1 "fast": one pass over X per epoch (8 B per element: the HBM roofline): a CTA owns
//     a block of rows, reduces each row's logit across its threads, and accumulates
//     delta * x into per-thread registers from the same loaded row; per-CTA partials are
//     reduced in a fixed order.  Order differs from the reference -> tolerance gate.
#include "cvb_common.cuh"
#include <math.h>
#include <stdlib.h>

namespace {

constexpr int LT = 256;          // threads per CTA
constexpr int FPT = 16;          // fast mode: at most this many features per thread in registers (f <= 4096)
constexpr int GT_ROWS = 256;     // exact gradient: rows per shared-memory tile

__global__ void transpose_f64(const double* __restrict__ X, int64_t n, int64_t f, double* __restrict__ Xt) {
  __shared__ double t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < n && c < f) t[k][threadIdx.x] = X[r * f + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < n && c < f) Xt[c * n + r] = t[threadIdx.x][k];
  }
}

// sigma_r(z) - y with the reference's rounding sequence (workload.py:44-45, :64)
__device__ __forceinline__ double delta_exact(double z, double y) {
  const double t = __dadd_rn(1.0, fabs(z));
  const double q = __ddiv_rn(z, t);
  const double s = __dadd_rn(1.0, q);
  return __dsub_rn(__dmul_rn(0.5, s), y);
}

// one thread per row: z = b; z += w_i * x_i in feature order (workload.py:61-63)
__global__ void lr_logits_exact(const double* __restrict__ Xt, const double* __restrict__ y,
                                const double* __restrict__ w, const double* __restrict__ b,
                                int64_t n, int64_t f, double* __restrict__ delta) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double z = *b;
  int64_t i = 0;
  for (; i + 8 <= f; i += 8) {     // loads issued ahead of the dependent add chain
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = Xt[(i + k) * n + r];
#pragma unroll
    for (int k = 0; k < 8; k++) z = __dadd_rn(z, __dmul_rn(w[i + k], x[k]));
  }
  for (; i < f; i++) z = __dadd_rn(z, __dmul_rn(w[i], Xt[i * n + r]));
  delta[r] = delta_exact(z, y[r]);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}

// one thread per feature (the last thread of the grid takes the bias), rows summed in file
// order.  A CTA is one warp covering 32 consecutive features; tiles of GT_ROWS rows x 32
// features are copied into shared memory with cp.async (no registers held, one 256-byte
// row segment per warp instruction) GT_STAGES-1 tiles ahead, so the dependent add chains
// (~8 cycles per row) never wait on HBM.
constexpr int GT_STAGES = 3;
constexpr size_t GT_SMEM = (size_t)GT_STAGES * GT_ROWS * 33 * sizeof(double);   // 32 features + delta

__global__ void __launch_bounds__(32) lr_grad_exact(const double* __restrict__ X, const double* __restrict__ delta,
                                                    int64_t n, int64_t f, double* __restrict__ g) {
  extern __shared__ __align__(16) double gsm[];   // [stage][row][33]: 32 features, then delta
  const int lane = threadIdx.x;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  const int64_t ntiles = (n + GT_ROWS - 1) / GT_ROWS;
  auto load = [&](int64_t tix) {
    if (tix < ntiles) {
      double* st = gsm + (size_t)(tix % GT_STAGES) * GT_ROWS * 33;
      const int64_t r0 = tix * GT_ROWS;
      for (int k = 0; k < GT_ROWS; k++) {
        const int64_t r = r0 + k;
        const bool v = r < n && i < f;
        cp_async8(st + k * 33 + lane, v ? X + r * f + i : X, v);
      }
      for (int k = lane; k < GT_ROWS; k += 32) {
        const bool v = r0 + k < n;
        cp_async8(st + k * 33 + 32, v ? delta + r0 + k : delta, v);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");   // (an empty group keeps the count uniform)
  };
  double acc = 0.0;
  for (int k = 0; k < GT_STAGES - 1; k++) load(k);
  for (int64_t t = 0; t < ntiles; t++) {
    load(t + GT_STAGES - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(GT_STAGES - 1) : "memory");
    __syncwarp();
    const double* st = gsm + (size_t)(t % GT_STAGES) * GT_ROWS * 33;
    const int rows = (int)min((int64_t)GT_ROWS, n - t * GT_ROWS);
    if (i < f) {
      for (int k = 0; k < rows; k++) acc = __dadd_rn(acc, __dmul_rn(st[k * 33 + 32], st[k * 33 + lane]));
    } else if (i == f) {
      for (int k = 0; k < rows; k++) acc = __dadd_rn(acc, st[k * 33 + 32]);
    }
    __syncwarp();   // this stage is refilled by the load GT_STAGES-1 tiles on
  }
  if (i <= f) g[i] = acc;
}

// fast mode, f <= LT*FP: one pass over X.  CTA c owns rows [c*rpc, (c+1)*rpc).
template <int FP>
__global__ void __launch_bounds__(LT, FP <= 12 ? 2 : 1) lr_epoch_fast(const double* __restrict__ X, const double* __restrict__ y,
                                                       const double* __restrict__ w, const double* __restrict__ b,
                                                       int64_t n, int64_t f, int64_t rpc, double* __restrict__ gpart) {
  __shared__ double red[2][LT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double wr[FP], gr[FP], xa[FP], xb[FP];
#pragma unroll
  for (int k = 0; k < FP; k++) {
    const int64_t i = threadIdx.x + (int64_t)k * LT;
    wr[k] = i < f ? w[i] : 0.0;
    gr[k] = 0.0;
  }
  double gb = 0.0;
  const double bias = *b;
  const int64_t r0 = (int64_t)blockIdx.x * rpc, r1 = min(n, r0 + rpc);
  auto ld = [&](int64_t r, double* x) {
#pragma unroll
    for (int k = 0; k < FP; k++) {
      const int64_t i = threadIdx.x + (int64_t)k * LT;
      x[k] = (r < r1 && i < f) ? __ldcs(X + r * f + i) : 0.0;
    }
  };
  auto row = [&](int64_t r, const double* cur, int p) {
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < FP; k++) z = fma(wr[k], cur[k], z);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) z += __shfl_xor_sync(0xffffffffu, z, s);
    if (lane == 0) red[p][wid] = z;
    __syncthreads();
    double zt = bias;
#pragma unroll
    for (int k = 0; k < LT / 32; k++) zt += red[p][k];
    const double d = 0.5 * (1.0 + zt / (1.0 + fabs(zt))) - y[r];
#pragma unroll
    for (int k = 0; k < FP; k++) gr[k] = fma(d, cur[k], gr[k]);
    gb += d;
  };
  // rows in pairs with register double buffering: the next row's loads are in flight while
  // this row is reduced; red[p] is rewritten two rows later, after another barrier
  if (r0 < r1) ld(r0, xa);
  for (int64_t r = r0; r < r1; r += 2) {
    ld(r + 1, xb);
    row(r, xa, 0);
    if (r + 1 >= r1) break;
    ld(r + 2, xa);
    row(r + 1, xb, 1);
  }
  double* out = gpart + (int64_t)blockIdx.x * (f + 1);
#pragma unroll
  for (int k = 0; k < FP; k++) {
    const int64_t i = threadIdx.x + (int64_t)k * LT;
    if (i < f) out[i] = gr[k];
  }
  if (threadIdx.x == 0) out[f] = gb;
}

// fast mode, any f: warp per row for the logit, then a row-block gradient pass (two passes)
__global__ void lr_logits_fast(const double* __restrict__ X, const double* __restrict__ y,
                               const double* __restrict__ w, const double* __restrict__ b,
                               int64_t n, int64_t f, double* __restrict__ delta) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  double z = 0.0;
  for (int64_t i = lane; i < f; i += 32) z = fma(w[i], X[r * f + i], z);
  for (int s = 16; s > 0; s >>= 1) z += __shfl_xor_sync(0xffffffffu, z, s);
  z += *b;
  if (lane == 0) delta[r] = 0.5 * (1.0 + z / (1.0 + fabs(z))) - y[r];
}

__global__ void lr_grad_fast(const double* __restrict__ X, const double* __restrict__ delta, int64_t n,
                             int64_t f, int64_t rows_per_block, double* __restrict__ gpart) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(n, r0 + rows_per_block);
  if (i > f) return;
  double g = 0.0;
  if (i < f) for (int64_t r = r0; r < r1; r++) g = fma(delta[r], X[r * f + i], g);
  else for (int64_t r = r0; r < r1; r++) g += delta[r];
  gpart[(int64_t)blockIdx.y * (f + 1) + i] = g;
}

// fixed-order sum of the per-CTA partials
__global__ void lr_reduce_parts(const double* __restrict__ gpart, int64_t nparts, int64_t f, double* __restrict__ g) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > f) return;
  double s = 0.0;
  for (int64_t k = 0; k < nparts; k++) s += gpart[k * (f + 1) + i];
  g[i] = s;
}

// w_i -= (lr * g_i) / n ; b -= (lr * g_b) / n   (workload.py:68-70), rounded like the reference
__global__ void lr_apply(const double* __restrict__ g, int64_t f, double lr, double nrows, double* __restrict__ w,
                         double* __restrict__ b) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > f) return;
  const double u = __ddiv_rn(__dmul_rn(lr, g[i]), nrows);
  if (i < f) w[i] = __dsub_rn(w[i], u);
  else *b = __dsub_rn(*b, u);
}

int fast_parts(int64_t n, int64_t f, int64_t* rpc) {
  const int64_t ctas = 2 * (int64_t)cvb_num_sms();
  if (f <= (int64_t)LT * FPT) {
    *rpc = (n + ctas - 1) / ctas;
    return (int)((n + *rpc - 1) / *rpc);
  }
  *rpc = 512;
  return (int)((n + 511) / 512);
}

}  // namespace

// doubles of scratch cvb_logistic_grad_dev needs (delta per row + per-CTA partials)
CVB_API int64_t cvb_logistic_scratch_doubles(int64_t n, int64_t f, int mode) {
  if (n <= 0 || f <= 0) return 0;
  if (mode == 0) return n;
  int64_t rpc;
  const int64_t parts = fast_parts(n, f, &rpc);
  return n + parts * (f + 1);
}

// Xt[c][r] = X[r][c] (the exact mode's feature-major copy), on the device
CVB_API int cvb_logistic_transpose_dev(const double* X, int64_t n, int64_t f, double* Xt, void* stream) {
  if (!X || !Xt || n <= 0 || f <= 0) { cvb_set_error("logistic_transpose: bad arguments"); return CVB_EINVAL; }
  dim3 grid((unsigned)((f + 31) / 32), (unsigned)((n + 31) / 32));
  transpose_f64<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(X, n, f, Xt);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

// One epoch's gradient sums over the n rows given (a whole dataset, or one rank's contiguous
// row block): g[0..f) = sum_r delta_r x_r, g[f] = sum_r delta_r, delta_r = sigma_r(z_r) - y_r
// with z_r = b + w.x_r.  mode 0 needs Xt (cvb_logistic_transpose_dev); mode 1 ignores it.
CVB_API int cvb_logistic_grad_dev(const double* X, const double* Xt, const double* y, int64_t n, int64_t f,
                                  const double* w, const double* b, int mode, double* g, double* scratch,
                                  void* stream) {
  if (!X || !y || !w || !b || !g || !scratch || n <= 0 || f <= 0 || (mode == 0 && !Xt) || mode < 0 || mode > 1) {
    cvb_set_error("logistic_grad: bad arguments");
    return CVB_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double* delta = scratch;
  if (mode == 0) {
    lr_logits_exact<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(Xt, y, w, b, n, f, delta);
    static unsigned long long attr = 0;
    if (cvb_first_on_device(&attr))
      CVB_CUDA(cudaFuncSetAttribute(lr_grad_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GT_SMEM));
    lr_grad_exact<<<(unsigned)((f + 1 + 31) / 32), 32, GT_SMEM, s>>>(X, delta, n, f, g);
  } else {
    int64_t rpc;
    const int parts = fast_parts(n, f, &rpc);
    double* gpart = scratch + n;
    if (f <= (int64_t)LT * FPT) {
      const int64_t fp = (f + LT - 1) / LT;
      if (fp <= 4) lr_epoch_fast<4><<<parts, LT, 0, s>>>(X, y, w, b, n, f, rpc, gpart);
      else if (fp <= 8) lr_epoch_fast<8><<<parts, LT, 0, s>>>(X, y, w, b, n, f, rpc, gpart);
      else if (fp <= 12) lr_epoch_fast<12><<<parts, LT, 0, s>>>(X, y, w, b, n, f, rpc, gpart);
      else lr_epoch_fast<16><<<parts, LT, 0, s>>>(X, y, w, b, n, f, rpc, gpart);
    } else {
      lr_logits_fast<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(X, y, w, b, n, f, delta);
      dim3 gg((unsigned)((f + 1 + 255) / 256), (unsigned)parts);
      lr_grad_fast<<<gg, 256, 0, s>>>(X, delta, n, f, rpc, gpart);
    }
    lr_reduce_parts<<<(unsigned)((f + 1 + 255) / 256), 256, 0, s>>>(gpart, parts, f, g);
  }
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

// w_i -= (lr * g_i) / nrows ; b -= (lr * g_b) / nrows   (nrows = the GLOBAL row count)
CVB_API int cvb_logistic_apply_dev(const double* g, int64_t f, double lr, double nrows, double* w, double* b,
                                   void* stream) {
  if (!g || !w || !b || f <= 0) { cvb_set_error("logistic_apply: bad arguments"); return CVB_EINVAL; }
  lr_apply<<<(unsigned)((f + 1 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(g, f, lr, nrows, w, b);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

// Drop-in numeric core of covault.workload.run_training with host buffers: X n x f row-major
// binary64, y n labels; writes f weights and the bias.  Synchronous; frees everything on
// every path.
CVB_API int cvb_logistic_train(const double* X, const double* y, int64_t n, int64_t f, double lr,
                               int64_t epochs, int mode, double* w_out, double* b_out) {
  if (!X || !y || !w_out || !b_out || n <= 0 || f <= 0 || epochs < 0 || mode < 0 || mode > 1) {
    cvb_set_error("logistic_train: bad arguments");
    return CVB_EINVAL;
  }
  const size_t xb = (size_t)n * f * sizeof(double);
  const int64_t sc = cvb_logistic_scratch_doubles(n, f, mode);
  cudaStream_t s = nullptr;
  double *dX = nullptr, *dXt = nullptr, *dy = nullptr, *dw = nullptr, *dg = nullptr, *dsc = nullptr;
  int rc = CVB_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
#define LR_TRY(expr)                                                                      \
  do {                                                                                    \
    if (e == cudaSuccess && (e = (expr)) != cudaSuccess)                                  \
      cvb_set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e));  \
  } while (0)
  if (e != cudaSuccess) { cvb_set_error("logistic_train: stream -> %s", cudaGetErrorString(e)); return CVB_ECUDA; }
  LR_TRY(cudaMallocAsync((void**)&dX, xb, s));
  LR_TRY(cudaMallocAsync((void**)&dy, n * sizeof(double), s));
  LR_TRY(cudaMallocAsync((void**)&dw, (f + 1) * sizeof(double), s));   // weights, then the bias
  LR_TRY(cudaMallocAsync((void**)&dg, (f + 1) * sizeof(double), s));
  LR_TRY(cudaMallocAsync((void**)&dsc, sc * sizeof(double), s));
  if (mode == 0) LR_TRY(cudaMallocAsync((void**)&dXt, xb, s));
  LR_TRY(cudaMemcpyAsync(dX, X, xb, cudaMemcpyHostToDevice, s));
  LR_TRY(cudaMemcpyAsync(dy, y, n * sizeof(double), cudaMemcpyHostToDevice, s));
  LR_TRY(cudaMemsetAsync(dw, 0, (f + 1) * sizeof(double), s));
  if (e == cudaSuccess && mode == 0) rc = cvb_logistic_transpose_dev(dX, n, f, dXt, s);
  for (int64_t ep = 0; ep < epochs && e == cudaSuccess && rc == CVB_OK; ep++) {
    rc = cvb_logistic_grad_dev(dX, dXt, dy, n, f, dw, dw + f, mode, dg, dsc, s);
    if (rc == CVB_OK) rc = cvb_logistic_apply_dev(dg, f, lr, (double)n, dw, dw + f, s);
  }
  LR_TRY(cudaMemcpyAsync(w_out, dw, f * sizeof(double), cudaMemcpyDeviceToHost, s));
  LR_TRY(cudaMemcpyAsync(b_out, dw + f, sizeof(double), cudaMemcpyDeviceToHost, s));
#undef LR_TRY
  const cudaError_t es = cudaStreamSynchronize(s);
  if (e == cudaSuccess && es != cudaSuccess) {
    e = es;
    cvb_set_error("logistic_train: %s", cudaGetErrorString(es));
  }
  for (double* p : {dX, dXt, dy, dw, dg, dsc})
    if (p) cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (rc != CVB_OK) return rc;
  return e == cudaSuccess ? CVB_OK : CVB_ECUDA;
}
