// The reference trainer's numeric core on the GPU (K2/K3/K4 of DESIGN.md).
//
// Replaces covault.workload.run_training (/root/reference/pkg/src/covault/workload.py:48-71;
// sigmoid :44-45).  Two modes:
//   mode 0 "exact": bit-identical to the reference's Python floats.  Every operation is an
//     explicitly rounded IEEE binary64 op (__dmul_rn/__dadd_rn/__ddiv_rn: no FMA
//     contraction) in the reference's order.  The only parallelism the reference order
//     admits is used: logits are independent per row (one thread per row, features in
//     order, :61-63) and each gradient component is an in-order sum over rows (one thread
//     per feature, rows in file order, :65-67).  Reproduces DEMO_MODEL_SHA256.
//   mode 1 "fast": same math, but row reductions are parallel tree sums (order differs ->
//     checked by relative tolerance).
// X is kept twice in HBM: row-major for the per-feature gradient pass (coalesced across
// features) and feature-major for the per-row logit pass (coalesced across rows).
#include "cvb_common.cuh"
#include <math.h>
#include <stdlib.h>

__global__ void lr_logits_exact(const double* __restrict__ Xt, const double* __restrict__ y,
                                const double* __restrict__ w, const double* __restrict__ b,
                                int64_t n, int64_t f, double* __restrict__ delta) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double z = *b;
  for (int64_t i = 0; i < f; i++) z = __dadd_rn(z, __dmul_rn(w[i], Xt[i * n + r]));
  double t = __dadd_rn(1.0, fabs(z));
  double q = __ddiv_rn(z, t);
  double s = __dadd_rn(1.0, q);
  delta[r] = __dsub_rn(__dmul_rn(0.5, s), y[r]);
}

// one thread per feature (+1 for the bias), rows summed in file order
__global__ void lr_grad_update_exact(const double* __restrict__ X, const double* __restrict__ delta,
                                     int64_t n, int64_t f, double lr, double nrows,
                                     double* __restrict__ w, double* __restrict__ b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > f) return;
  double g = 0.0;
  if (i < f) {
    for (int64_t r = 0; r < n; r++) g = __dadd_rn(g, __dmul_rn(delta[r], X[r * f + i]));
    w[i] = __dsub_rn(w[i], __ddiv_rn(__dmul_rn(lr, g), nrows));
  } else {
    for (int64_t r = 0; r < n; r++) g = __dadd_rn(g, delta[r]);
    *b = __dsub_rn(*b, __ddiv_rn(__dmul_rn(lr, g), nrows));
  }
}

// ---- fast mode: parallel reductions ------------------------------------------------------
__global__ void lr_logits_fast(const double* __restrict__ X, const double* __restrict__ y,
                               const double* __restrict__ w, const double* __restrict__ b,
                               int64_t n, int64_t f, double* __restrict__ delta) {
  // one warp per row, coalesced over features
  int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (r >= n) return;
  double z = 0.0;
  for (int64_t i = lane; i < f; i += 32) z += w[i] * X[r * f + i];
  for (int s = 16; s > 0; s >>= 1) z += __shfl_xor_sync(0xffffffffu, z, s);
  z += *b;
  if (lane == 0) delta[r] = 0.5 * (1.0 + z / (1.0 + fabs(z))) - y[r];
}

__global__ void lr_grad_fast(const double* __restrict__ X, const double* __restrict__ delta, int64_t n,
                             int64_t f, int64_t rows_per_block, double* __restrict__ gpart) {
  // block (bx, by): features [bx*256, +256), rows [by*rows_per_block, ...)
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(n, r0 + rows_per_block);
  if (i > f) return;
  double g = 0.0;
  if (i < f) for (int64_t r = r0; r < r1; r++) g += delta[r] * X[r * f + i];
  else for (int64_t r = r0; r < r1; r++) g += delta[r];
  gpart[(int64_t)blockIdx.y * (f + 1) + i] = g;
}

__global__ void lr_update_fast(const double* __restrict__ gpart, int64_t nparts, int64_t f, double lr,
                               double nrows, double* __restrict__ w, double* __restrict__ b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > f) return;
  double g = 0.0;
  for (int64_t k = 0; k < nparts; k++) g += gpart[k * (f + 1) + i];
  if (i < f) w[i] -= lr * g / nrows;
  else *b -= lr * g / nrows;
}

// Drop-in numeric core of covault.workload.run_training: host buffers in/out (the CSV is
// parsed on the host with Python float(), which is correctly rounded like the reference).
// X: n x f row-major binary64, y: n labels; writes f weights and the bias.
CVB_API int cvb_logistic_train(const double* X, const double* y, int64_t n, int64_t f, double lr,
                                  int64_t epochs, int mode, double* w_out, double* b_out) {
  if (!X || !y || !w_out || !b_out || n <= 0 || f <= 0 || epochs < 0) {
    cvb_set_error("logistic_train: bad arguments");
    return CVB_EINVAL;
  }
  cudaStream_t s;
  CVB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  size_t xb = (size_t)n * f * sizeof(double);
  double *dX = nullptr, *dXt = nullptr, *dy = nullptr, *dw = nullptr, *db = nullptr, *dd = nullptr, *dg = nullptr;
  const int64_t rows_per_block = 512;
  int64_t nparts = (n + rows_per_block - 1) / rows_per_block;
  CVB_CUDA(cudaMallocAsync((void**)&dX, xb, s));
  CVB_CUDA(cudaMallocAsync((void**)&dy, n * sizeof(double), s));
  CVB_CUDA(cudaMallocAsync((void**)&dw, f * sizeof(double), s));
  CVB_CUDA(cudaMallocAsync((void**)&db, sizeof(double), s));
  CVB_CUDA(cudaMallocAsync((void**)&dd, n * sizeof(double), s));
  CVB_CUDA(cudaMemcpyAsync(dX, X, xb, cudaMemcpyHostToDevice, s));
  CVB_CUDA(cudaMemcpyAsync(dy, y, n * sizeof(double), cudaMemcpyHostToDevice, s));
  CVB_CUDA(cudaMemsetAsync(dw, 0, f * sizeof(double), s));
  CVB_CUDA(cudaMemsetAsync(db, 0, sizeof(double), s));
  if (mode == 0) {
    // feature-major copy for the per-row pass (host transpose keeps the device code trivial)
    double* Xt = (double*)malloc(xb);
    if (!Xt) return CVB_ENOMEM;
    for (int64_t r = 0; r < n; r++)
      for (int64_t i = 0; i < f; i++) Xt[i * n + r] = X[r * f + i];
    CVB_CUDA(cudaMallocAsync((void**)&dXt, xb, s));
    CVB_CUDA(cudaMemcpyAsync(dXt, Xt, xb, cudaMemcpyHostToDevice, s));
    CVB_CUDA(cudaStreamSynchronize(s));
    free(Xt);
  } else {
    CVB_CUDA(cudaMallocAsync((void**)&dg, nparts * (f + 1) * sizeof(double), s));
  }
  double nrows = (double)n;
  for (int64_t e = 0; e < epochs; e++) {
    if (mode == 0) {
      lr_logits_exact<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dXt, dy, dw, db, n, f, dd);
      lr_grad_update_exact<<<(unsigned)((f + 1 + 255) / 256), 256, 0, s>>>(dX, dd, n, f, lr, nrows, dw, db);
    } else {
      lr_logits_fast<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(dX, dy, dw, db, n, f, dd);
      dim3 g((unsigned)((f + 1 + 255) / 256), (unsigned)nparts);
      lr_grad_fast<<<g, 256, 0, s>>>(dX, dd, n, f, rows_per_block, dg);
      lr_update_fast<<<(unsigned)((f + 1 + 255) / 256), 256, 0, s>>>(dg, nparts, f, lr, nrows, dw, db);
    }
    CVB_CHECK_LAUNCH();
  }
  CVB_CUDA(cudaMemcpyAsync(w_out, dw, f * sizeof(double), cudaMemcpyDeviceToHost, s));
  CVB_CUDA(cudaMemcpyAsync(b_out, db, sizeof(double), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(dX, s); cudaFreeAsync(dy, s); cudaFreeAsync(dw, s); cudaFreeAsync(db, s); cudaFreeAsync(dd, s);
  if (dXt) cudaFreeAsync(dXt, s);
  if (dg) cudaFreeAsync(dg, s);
  CVB_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
  return CVB_OK;
}
