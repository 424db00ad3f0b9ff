/*
 * cvb_nn.h -- C ABI of the CNN training-step kernels (sm_100a).
 *
 * The reference has NO code for this part of the path: its trainer is an fp64 logistic
 * toy (pkg/src/covault/workload.py:48-71) and the CIFAR CNN / medical model exist only as
 * paper prose.  These entry points are what the B200
 * trainer (paper_2103_16898_b200/nets.py, trainer.py) calls behind the reference's
 * run_training(params, data) signature; DESIGN.md documents the model definitions.
 *
 * Activations: NHWC bf16 rows [N*H*W][C] with a channel stride (cs) so concat buffers are
 * read/written in place.  Weights: bf16 [Cout][KH][KW][Cin] (K-major).  Grads/optimiser
 * state: fp32.  All calls are asynchronous on `stream` (a cudaStream_t).
 */
#ifndef CVB_NN_H
#define CVB_NN_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- tcgen05 implicit-GEMM engine ------------------------------------------------------ */
/* y[n,oh,ow,yoff+co] = bias[co] + sum x[n, oh*s-pad+kh, ow*s-pad+kw, ci] * w[co][kh][kw][ci] */
int cvb_conv2d_fwd(const void* x, int n, int h, int w, int cin, int xcs, const void* wt, int cout, int kh, int kw,
                   int stride, int pad, void* y, int oh, int ow, int ycs, int yoff, const float* bias, int y_f32,
                   int accumulate, void* stream);
/* fp32 partial weight gradients part[split][cout][kh*kw*cin]; *splits_out receives the count */
/* dX of a stride-2 conv by output-parity classes (no zero-upsampled dY): 4 gather convs of dY
   through parity views of dx; wscratch = cout*kh*kw*cin bf16 (the per-class weight matrices,
   written here from w -- or, with w == NULL, already written, e.g. by cvb_transpose_batched).
   Returns CVB_EINVAL (nothing launched) for unsupported geometry; classes without taps need
   accumulate=1. */
int cvb_conv2d_dgrad_s2(const void* dy, int n, int oh, int ow, int cout, int dycs, const void* w, int cin, int kh,
                        int kw, int pad, void* dx, int h, int wd, int dxcs, int accumulate, void* wscratch,
                        void* stream);
/* dX of a 3x3 pad-1 stride-2 conv as two gather convs of dY, one per output ROW parity a, each
   producing both column parities (N = 2*cin: dx[2i+a][2j+b][ci] as channel b*cin+ci of output
   pixel (i, j)); dY taps (dh, dw): conv 0 (0,0) (0,1); conv 1 (0,0) (0,1) (1,0) (1,1).  wrows =
   conv 0's [2cin][2][cout] then conv 1's [2cin][4][cout] bf16, rows (b, ci) of tap (dh, dw) =
   w[co][a+1-2dh][b+1-2dw][ci], zero where that tap does not exist.  Needs dx [n][2oh][2ow][cin]
   contiguous (dxcs == cin), else CVB_EINVAL without launching. */
int cvb_conv2d_dgrad_s2_rows(const void* dy, int n, int oh, int ow, int cout, int dycs, int cin, void* dx, int h,
                             int wd, int dxcs, int accumulate, const void* wrows, void* stream);
int cvb_conv2d_wgrad(const void* dy, int n, int oh, int ow, int cout, int dycs, const void* x, int h, int w, int cin,
                     int xcs, int kh, int kw, int stride, int pad, float* part, int max_splits, int* splits_out,
                     void* stream);
/* C[M][N] (+bias) = sum_k A(m,k) B(n,k); A [M][K] (a_major 0) or [K][M] (1); B [N][K] or [K][N] */
int cvb_gemm(const void* a, int a_major, int64_t lda, const void* b, int b_major, int64_t ldb, int M, int N, int K,
             void* c, int64_t ldc, int c_f32, const float* bias, int splits, int accumulate, void* stream);
int cvb_gemm_ex(const void* a, int a_major, int64_t lda, const void* b, int b_major, int64_t ldb, int M, int N, int K,
                void* c, int64_t ldc, int c_f32, const float* bias, int splits, int accumulate, int max_bn,
                void* stream);   /* cvb_gemm with N tiles of at most max_bn columns */
int cvb_gemm_splits_used(int K, int splits);
/* profiling aids (not on the hot path): raw tcgen05.mma issue rate; CTA-0 pipeline timeline
 * of the last GEMM launched with CVB_GEMM_DBG=4 (5 x 4096 clock64 stamps) */
long long cvb_debug_mma_cycles(int n_mma, int bn, int issuers, int a_halo);
int cvb_debug_trace(long long* host_out);

/* ---- batch norm (+ReLU, +residual) --------------------------------------------------------- */
int64_t cvb_bn_workspace_floats(int64_t rows, int C);
int cvb_bn_stats(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd, float eps,
                 float* run_mean, float* run_var, float momentum, void* stream);
int cvb_bn_apply(const void* x, int64_t rows, int C, int xcs, const float* mean, const float* rstd, const float* gamma,
                 const float* beta, const void* res, int rcs, int relu, void* y, int ycs, int ycoff, void* stream);
int cvb_bn_backward(const void* dy, int dycs, const void* x, int xcs, const void* y, int ycs, int64_t rows, int C,
                    const float* mean, const float* rstd, const float* gamma, const float* beta, int relu, float* ws,
                    float* dgamma, float* dbeta, void* dx, int dxcs, float* dx32, int accum32, void* dz_out,
                    void* stream);
/* single-launch (cooperative, grid-barrier) forms of the above: statistics + finalisation +
   elementwise pass in one kernel; y == NULL in cvb_bn_forward computes statistics only */
int64_t cvb_bn_fused_workspace_floats(int C);
int cvb_bn_forward(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd, float eps,
                   float* run_mean, float* run_var, float momentum, const float* gamma, const float* beta,
                   const void* res, int rcs, int relu, void* y, int ycs, int ycoff, void* stream);
/* DenseNet: input gradient of the BNs over a concat range, formed once from every later layer's
   dY slice after those layers ran the statistics pass only (cvb_bn_backward_fused with dx = dx32 =
   NULL): out[r][c] = base[r][c] + sum_l gamma_l*rstd*(dz_l - dbeta_l/M - xhat*dgamma_l/M) for c in
   [0, nc), dz_l = dy_l * [gamma_l*xhat + beta_l > 0]; layers summed in array order.  The pointer
   arrays (host, nl <= 32) are offset to the range's first channel; out (bf16, or fp32 if out_f32)
   may alias base. */
int cvb_bn_gather_dx(const void* x, int xcs, int64_t rows, int nc, const float* mean, const float* rstd,
                     const float* base, int bcs, int nl, const void* const* dy, const int* dycs,
                     const float* const* gamma, const float* const* beta, const float* const* dgamma,
                     const float* const* dbeta, void* out, int ocs, int out_f32, void* stream);
/* cvb_bn_forward with the batch statistics computed only for channels [st_off, st_off + st_C)
   (the other channels' mean/rstd are inputs; no running statistics): DenseNet's newest concat
   slice and the normalisation of the whole prefix in one launch. */
int cvb_bn_forward_range(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd, float eps,
                         float* run_mean, float* run_var, float momentum, const float* gamma, const float* beta,
                         const void* res, int rcs, int relu, void* y, int ycs, int ycoff, int st_off, int st_C,
                         void* stream);
int cvb_bn_backward_fused(const void* dy, int dycs, const void* x, int xcs, const void* y, int ycs, int64_t rows,
                          int C, const float* mean, const float* rstd, const float* gamma, const float* beta, int relu,
                          float* ws, float* dgamma, float* dbeta, void* dx, int dxcs, float* dx32, int accum32,
                          void* dz_out, void* stream);
/* ReLU mask instead of y (residual layers): cvb_bn_forward_mask also writes mask[rows][C/8] bytes,
   bit k of byte g = (y[row][8g + k] > 0) exactly as stored in bf16; cvb_bn_backward_fused_mask
   reads it in place of y (1/16 of the bytes). */
int cvb_bn_forward_mask(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd, float eps,
                        float* run_mean, float* run_var, float momentum, const float* gamma, const float* beta,
                        const void* res, int rcs, int relu, void* y, int ycs, int ycoff, void* mask, void* stream);
int cvb_bn_backward_fused_mask(const void* dy, int dycs, const void* x, int xcs, const void* mask, int64_t rows,
                               int C, const float* mean, const float* rstd, const float* gamma, const float* beta,
                               int relu, float* ws, float* dgamma, float* dbeta, void* dx, int dxcs, float* dx32,
                               int accum32, void* dz_out, void* stream);

/* ---- pooling -------------------------------------------------------------------------------- */
int cvb_maxpool_fwd(const void* x, int n, int h, int w, int C, int k, int s, int p, void* y, int oh, int ow, int ycs,
                    void* stream);
int cvb_maxpool_bwd(const void* x, const void* dy, int n, int h, int w, int C, int k, int s, int p, int oh, int ow,
                    void* dx, void* stream);
/* arg-max variants: the forward stores each output element's window offset (uint8, same
   [n][oh][ow][C] layout), the backward gathers from it without re-scanning windows */
int cvb_maxpool_fwd_idx(const void* x, int n, int h, int w, int C, int k, int s, int p, void* y, int oh, int ow,
                        int ycs, void* idx, void* stream);
int cvb_maxpool_bwd_idx(const void* idx, const void* dy, int n, int h, int w, int C, int k, int s, int p, int oh,
                        int ow, void* dx, void* stream);
int cvb_avgpool_fwd(const void* x, int n, int h, int w, int C, int xcs, int k, void* y, int ycs, void* stream);
int cvb_avgpool_bwd(const void* dy, int n, int h, int w, int C, int k, void* dx, int dxcs, void* stream);
int cvb_gap_fwd(const void* x, int n, int hw, int C, int xcs, void* y, void* stream);
int cvb_gap_bwd(const void* dy, int n, int hw, int C, void* dx, void* stream);

/* ---- loss, reductions, layout helpers ---------------------------------------------------------- */
int cvb_softmax_xent(const float* logits, int B, int C, const int32_t* labels, float grad_scale, float* row_ws,
                     float* loss_out, void* dlogits, int ldd, void* stream);
/* Fused classifier head (csrc/head.cu): Linear(fin -> C <= 16, weights padded to 16 rows) forward,
 * softmax cross-entropy (row_loss, mean loss, dlogits scaled by `scale`) and the layer's backward
 * (dw [16][fin], db [16], dx = dlogits W optionally masked by x > 0, dprev_b = column sums of dx)
 * in one cooperative launch.  fin a multiple of 256, <= 1024; part holds
 * cvb_head_workspace_floats(B, fin) floats.  Replaces gemm + softmax_xent + gemm + col_sum + gemm
 * (+ relu_bwd + col_sum) of the unfused head. */
int cvb_head_train(const void* x, int64_t ldx, const void* w, const float* bias, const int32_t* labels, int B,
                   int fin, int C, float scale, int relu_mask, float* logits, void* dlogits, float* row_loss,
                   float* loss, void* dx, int64_t lddx, float* dw, float* db, float* dprev_b, float* part,
                   void* stream);
int64_t cvb_head_workspace_floats(int B, int fin);
int cvb_reduce_splits(const float* part, int splits, int64_t count, float* out, int accumulate, float scale,
                      void* stream);
/* split-K epilogue of a dense layer: out[r][c] = act(sum_s part[s][r][c] + bias[c]) */
int cvb_reduce_splits_act(const float* part, int splits, int rows, int cols, const float* bias, int relu, void* out,
                          int out_f32, int64_t ldo, void* stream);
/* all stride-1 dgrad weight flips in one launch: desc_dev = nlayers x {src, dst, cout, kh, kw, cin}
   (int64 element offsets into pb / fb) */
/* Batched bf16 matrix transposes (one launch per 8192 jobs): desc_dev = njobs x {src off, dst off, rows, cols,
   src row stride, dst row stride} (elements); dst[c*dst_ld + r] = src[r*src_ld + c].  Used for
   the flipped stride-1 dgrad weights (a job per tap) and the stride-2 dgrad parity-class
   weights (a job per class and tap) after every optimiser step. */
int cvb_transpose_batched(const void* src, void* dst, const int64_t* desc_dev, int njobs, int64_t max_elems,
                          void* stream);
int cvb_weight_flip_batched(const void* pb, void* fb, const int64_t* desc_dev, int nlayers, int64_t max_elems,
                            void* stream);
/* space-to-depth stem: the 7x7 stride-2 pad-3 conv on x [n][h][w][C] equals a 4x4 stride-1 pad-2
   conv on xs = s2d(x) [n][h/2][w/2][4C] with weights s2d_weights(w) [cout][4][4][4C]; the weight
   gradient maps back with s2d_weights_grad (fp32) */
int cvb_space_to_depth2(const void* x, int n, int h, int w, int C, void* xs, void* stream);
int cvb_s2d_weights(const void* w7, int cout, int C, void* ws, void* stream);
int cvb_s2d_weights_grad(const float* dws, int cout, int C, float* dw7, void* stream);
int cvb_weight_flip(const void* w, int cout, int kh, int kw, int cin, void* wt, void* stream);
int cvb_zero_upsample(const void* dy, int n, int oh, int ow, int C, int dycs, void* out, void* stream);
int cvb_col_sum(const void* x, int is_f32, int64_t rows, int cols, int64_t ld, float* out, int accumulate, void* stream);
int cvb_relu_fwd(void* x, int64_t n, void* stream);
int cvb_relu_bwd(void* dy, const void* y, int64_t n, void* stream);

/* ---- fused optimisers over flat fp32 buffers (refresh the bf16 compute copy pb) ---------------- */
/* step > 0: host bias correction; step <= 0: device counter in one launch (step_dev += 1;
 * sched_dev holds 4 floats, zero-initialised: [0..1] the next step's bias corrections
 * 1/(1-b1^t), 1/sqrt(1-b2^t) (cached for fixed b1, b2), [2] the CTA counter),
 * so a captured CUDA graph replays correctly. */
/* skip_dev (nullable): when *skip_dev != 0 the update is skipped entirely (parameters, moments,
 * step counter) -- the decrypt-verdict gate of an encrypted training step. */
int cvb_adam_step(float* p, const float* g, float* m, float* v, void* pb, int64_t n, float lr, float b1, float b2,
                  float eps, int64_t step, float grad_scale, int32_t* step_dev, float* sched_dev,
                  const float* skip_dev, void* stream);
/* *slot = (*word != 0) ? 1.0f : 0.0f  (one thread; the per-step verdict snapshot) */
int cvb_verdict_snapshot(const uint32_t* word, float* slot, void* stream);
int cvb_sgd_step(float* p, const float* g, float* buf, void* pb, int64_t n, float lr, float momentum, float wd,
                 float grad_scale, int first, void* stream);
int cvb_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream);
/* y[r][c] = bf16(x[r][c]) with row strides (concat-gradient slices) */
int cvb_cast_rows(const float* x, int64_t ldx, void* y, int64_t ldy, int64_t rows, int cols, void* stream);

#ifdef __cplusplus
}
#endif
#endif
