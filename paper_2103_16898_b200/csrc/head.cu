// Fused classifier head of one training step (K6h of DESIGN.md): the last Linear layer's
// forward, the softmax cross-entropy loss and the layer's whole backward in ONE launch.
//
// Replaces, for the head of every model (nets.py Net.head_train), the seven launches
//   gemm(fwd, +bias) -> softmax_xent_mean -> gemm(wgrad) -> col_sum(db) -> gemm(dgrad)
//   [-> relu_bwd -> col_sum(previous layer's bias grad)]
// of the CNN step's loss head (the north-star CNN has no reference code -- PAPER.md:441-443,
// :475-477 prose only).  The unfused launches stay available
// (CVB_UNFUSED_HEAD=1) and are the parity reference in tests/test_head_gpu.py.
//
// The head is tiny (B x fin x 16 with fin <= 1024) and launch-bound, so it runs on CUDA cores:
//   phase 1 (row chunks of 8, one warp per row): logits = x W^T + b (fp32 accumulate of bf16
//     operands, W staged in shared memory), row softmax / loss / dlogits (bf16, scaled by
//     1/global_batch), dx = dlogits W (bf16, optionally masked by x > 0 = the preceding
//     ReLU), and per-CTA partial sums of dW = dlogits^T x, db and colsum(dx) in fixed order;
//   grid barrier (cooperative launch: all CTAs co-resident, capturable into CUDA graphs);
//   phase 2: every output element sums the CTA partials in CTA order; CTA 0 reduces the
//     per-row losses (double, fixed order) to the mean.
// Everything is deterministic (no floating-point atomics).
#include "cvb_common.cuh"
#include <cuda_bf16.h>

namespace {

typedef __nv_bfloat16 bf16;
constexpr int HT = 256;    // threads per CTA
constexpr int HR = 8;      // rows per chunk (one per warp)
constexpr int HO = 16;     // padded classes (Linear pads fout to 16)

struct HeadArgs {
  const bf16* x; int64_t ldx;      // [B][ldx] head input
  const bf16* w;                   // [16][fin] bf16 weights (rows >= C are zero)
  const float* bias;               // [16]
  const int32_t* labels;           // [B]
  int B, fin, C, relu_mask;
  float scale;                     // dlogits scale (1 / global batch)
  float* logits;                   // [B][16] fp32
  bf16* dlogits;                   // [B][16]
  float* row_loss;                 // [B]
  float* loss;                     // [1] mean over the B rows
  bf16* dx; int64_t lddx;          // [B][lddx] or null
  float* dw;                       // [16][fin] fp32
  float* db;                       // [16] fp32
  float* dprev_b;                  // [fin] column sums of dx, or null
  float* part;                     // [grid][E] per-CTA partials
  int64_t E;                       // partial stride: 16*fin + fin + 16
  unsigned* bar;                   // grid barrier {arrivals, generation}
};

__device__ __forceinline__ void unpack8(const uint4& u, float v[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}

__device__ __forceinline__ uint4 pack8(const float v[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  return u;
}

__device__ __forceinline__ void head_grid_sync(unsigned* bar) { cvb_grid_barrier(bar); }   // two-level (cvb_common.cuh)

__global__ void __launch_bounds__(HT) head_train_kernel(const __grid_constant__ HeadArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int fin = a.fin;
  bf16* ws = reinterpret_cast<bf16*>(smem);            // [16][fin]
  bf16* xs = ws + HO * fin;                             // [HR][fin] this chunk's input rows
  bf16* dxs = xs + HR * fin;                            // [HR][fin] this chunk's dx rows
  float* dls = reinterpret_cast<float*>(dxs + HR * fin);   // [HR][16] bf16-rounded dlogits
  CVB_PDL_PROLOGUE();
  for (int i = threadIdx.x; i < HO * fin / 8; i += HT)
    reinterpret_cast<uint4*>(ws)[i] = __ldg(reinterpret_cast<const uint4*>(a.w) + i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* mypart = a.part + (int64_t)blockIdx.x * a.E;
  const int kg_n = fin / 8;

  for (int chunk = blockIdx.x, it = 0; chunk * HR < a.B; chunk += gridDim.x, ++it) {
    const int row = chunk * HR + warp;
    if (row < a.B) {
      float acc[HO];
#pragma unroll
      for (int o = 0; o < HO; o++) acc[o] = 0.f;
      for (int k0 = lane * 8; k0 < fin; k0 += 256) {
        const uint4 u = *reinterpret_cast<const uint4*>(a.x + (int64_t)row * a.ldx + k0);
        *reinterpret_cast<uint4*>(xs + warp * fin + k0) = u;
        float hv[8];
        unpack8(u, hv);
#pragma unroll
        for (int o = 0; o < HO; o++) {
          float wv[8];
          unpack8(*reinterpret_cast<const uint4*>(ws + o * fin + k0), wv);
#pragma unroll
          for (int j = 0; j < 8; j++) acc[o] = fmaf(hv[j], wv[j], acc[o]);
        }
      }
#pragma unroll
      for (int o = 0; o < HO; o++)
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], s);
      // every lane now holds the row's 16 logits
      float mx = -INFINITY;
#pragma unroll
      for (int o = 0; o < HO; o++) {
        acc[o] += __ldg(a.bias + o);
        if (o < a.C) mx = fmaxf(mx, acc[o]);
      }
      float se = 0.f;
#pragma unroll
      for (int o = 0; o < HO; o++)
        if (o < a.C) se += expf(acc[o] - mx);
      const float lse = logf(se) + mx;
      const int lab = a.labels[row];
      float dl[HO];
#pragma unroll
      for (int o = 0; o < HO; o++) {
        const float g = o < a.C ? (expf(acc[o] - lse) - (o == lab ? 1.f : 0.f)) * a.scale : 0.f;
        dl[o] = __bfloat162float(__float2bfloat16_rn(g));
        if (lane == o) {
          a.logits[(int64_t)row * HO + o] = acc[o];
          a.dlogits[(int64_t)row * HO + o] = __float2bfloat16_rn(dl[o]);
          dls[warp * HO + o] = dl[o];
        }
        if (lane == 0 && o == lab) a.row_loss[row] = lse - acc[o];
      }
      // dx = dlogits W (bf16 operands, fp32 accumulate), masked by the preceding ReLU
      for (int k0 = lane * 8; k0 < fin; k0 += 256) {
        float d[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int o = 0; o < HO; o++) {
          float wv[8];
          unpack8(*reinterpret_cast<const uint4*>(ws + o * fin + k0), wv);
#pragma unroll
          for (int j = 0; j < 8; j++) d[j] = fmaf(dl[o], wv[j], d[j]);
        }
        if (a.relu_mask) {
          float hv[8];
          unpack8(*reinterpret_cast<const uint4*>(xs + warp * fin + k0), hv);
#pragma unroll
          for (int j = 0; j < 8; j++) d[j] = hv[j] > 0.f ? d[j] : 0.f;
        }
        const uint4 u = pack8(d);
        *reinterpret_cast<uint4*>(dxs + warp * fin + k0) = u;
        if (a.dx) *reinterpret_cast<uint4*>(a.dx + (int64_t)row * a.lddx + k0) = u;
      }
    } else {
      if (lane < HO) dls[warp * HO + lane] = 0.f;
      for (int k0 = lane * 8; k0 < fin; k0 += 256) {
        *reinterpret_cast<uint4*>(xs + warp * fin + k0) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dxs + warp * fin + k0) = make_uint4(0, 0, 0, 0);
      }
    }
    __syncthreads();
    // this chunk's contribution to the CTA partials (fixed row order; CTA-private RMW)
    for (int idx = threadIdx.x; idx < HO * kg_n; idx += HT) {
      const int o = idx / kg_n, k0 = (idx - o * kg_n) * 8;
      float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int r = 0; r < HR; r++) {
        const float d = dls[r * HO + o];
        float xv[8];
        unpack8(*reinterpret_cast<const uint4*>(xs + r * fin + k0), xv);
#pragma unroll
        for (int j = 0; j < 8; j++) s[j] = fmaf(d, xv[j], s[j]);
      }
      float4* dst = reinterpret_cast<float4*>(mypart + o * fin + k0);
      if (it) {
        const float4 p0 = dst[0], p1 = dst[1];
        s[0] += p0.x; s[1] += p0.y; s[2] += p0.z; s[3] += p0.w;
        s[4] += p1.x; s[5] += p1.y; s[6] += p1.z; s[7] += p1.w;
      }
      dst[0] = make_float4(s[0], s[1], s[2], s[3]);
      dst[1] = make_float4(s[4], s[5], s[6], s[7]);
    }
    if (a.dprev_b) {
      for (int kg = threadIdx.x; kg < kg_n; kg += HT) {
        float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int r = 0; r < HR; r++) {
          float v[8];
          unpack8(*reinterpret_cast<const uint4*>(dxs + r * fin + kg * 8), v);
#pragma unroll
          for (int j = 0; j < 8; j++) s[j] += v[j];
        }
        float4* dst = reinterpret_cast<float4*>(mypart + HO * fin + kg * 8);
        if (it) {
          const float4 p0 = dst[0], p1 = dst[1];
          s[0] += p0.x; s[1] += p0.y; s[2] += p0.z; s[3] += p0.w;
          s[4] += p1.x; s[5] += p1.y; s[6] += p1.z; s[7] += p1.w;
        }
        dst[0] = make_float4(s[0], s[1], s[2], s[3]);
        dst[1] = make_float4(s[4], s[5], s[6], s[7]);
      }
    }
    if (threadIdx.x < HO) {
      float s = 0.f;
#pragma unroll
      for (int r = 0; r < HR; r++) s += dls[r * HO + threadIdx.x];
      float* dst = mypart + HO * fin + fin + threadIdx.x;
      *dst = it ? *dst + s : s;
    }
    __syncthreads();   // the next chunk overwrites xs / dxs / dls
  }

  head_grid_sync(a.bar);

  // phase 2: sum the CTA partials -- 32 consecutive outputs per pass of a CTA (lanes,
  // coalesced) x 8 groups of CTAs (warps, 8 loads in flight each), groups added in fixed order
  __shared__ float red[HT / 32][32];
  const int64_t n_out = (int64_t)HO * fin + fin + HO;
  const int G = (int)gridDim.x, per = (G + HT / 32 - 1) / (HT / 32);
  const int c0 = warp * per, c1 = min(G, c0 + per);
  for (int64_t e0 = (int64_t)blockIdx.x * 32; e0 < n_out; e0 += (int64_t)gridDim.x * 32) {
    const int64_t e = e0 + lane;
    float s = 0.f;
    if (e < n_out) {
      int c = c0;
      for (; c + 8 <= c1; c += 8) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] = __ldcg(a.part + (int64_t)(c + j) * a.E + e);
#pragma unroll
        for (int j = 0; j < 8; j++) s += v[j];
      }
      for (; c < c1; c++) s += __ldcg(a.part + (int64_t)c * a.E + e);
    }
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && e < n_out) {
      float t = red[0][lane];
#pragma unroll
      for (int w = 1; w < HT / 32; w++) t += red[w][lane];
      if (e < (int64_t)HO * fin) a.dw[e] = t;
      else if (e < (int64_t)HO * fin + fin) { if (a.dprev_b) a.dprev_b[e - (int64_t)HO * fin] = t; }
      else a.db[e - (int64_t)HO * fin - fin] = t;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    __shared__ double sh[HT];
    double s = 0;
    for (int i = threadIdx.x; i < a.B; i += HT) s += __ldcg(a.row_loss + i);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int st = HT / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
      __syncthreads();
    }
    if (threadIdx.x == 0) a.loss[0] = (float)(sh[0] / a.B);
  }
}

size_t head_smem(int fin) { return (size_t)(HO + 2 * HR) * fin * sizeof(bf16) + HR * HO * sizeof(float); }

int head_grid(int B, int fin, int* grid) {
  int dev = 0;
  CVB_CUDA(cudaGetDevice(&dev));
  static int attr_dev[64] = {0};
  if (dev < 0 || dev >= 64) { cvb_set_error("head: device index out of range"); return CVB_EINVAL; }
  if (!attr_dev[dev]) {
    CVB_CUDA(cudaFuncSetAttribute(head_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)head_smem(1024)));
    attr_dev[dev] = 1;
  }
  int per_sm = 0;
  CVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, head_train_kernel, HT, head_smem(fin)));
  if (per_sm < 1) { cvb_set_error("head: kernel does not fit on an SM"); return CVB_EINVAL; }
  const int chunks = (B + HR - 1) / HR, sms = cvb_num_sms();
  const int cap = per_sm * sms;
  *grid = chunks < sms ? chunks : sms;   // at most one CTA per SM: phase 2 spreads over them
  if (*grid > cap) *grid = cap;
  return CVB_OK;
}

int64_t head_E(int fin) { return ((int64_t)HO * fin + fin + HO + 3) / 4 * 4; }

}  // namespace

// Floats of partials workspace cvb_head_train needs for a batch of B rows of fin features.
CVB_API int64_t cvb_head_workspace_floats(int B, int fin) {
  if (B <= 0 || fin <= 0) return -1;
  const int chunks = (B + HR - 1) / HR, sms = cvb_num_sms();
  return (int64_t)(chunks < sms ? chunks : sms) * head_E(fin);
}

// Fused classifier head: forward (logits), softmax cross-entropy (row_loss, loss, dlogits) and
// backward (dw, db, dx, optional column sums of dx) of a Linear(fin -> C <= 16) layer whose
// weights are padded to 16 rows.  labels must lie in [0, C).
CVB_API int cvb_head_train(const void* x, int64_t ldx, const void* w, const float* bias, const int32_t* labels, int B,
                           int fin, int C, float scale, int relu_mask, float* logits, void* dlogits, float* row_loss,
                           float* loss, void* dx, int64_t lddx, float* dw, float* db, float* dprev_b, float* part,
                           void* stream) {
  if (!x || !w || !bias || !labels || !logits || !dlogits || !row_loss || !loss || !dw || !db || !part) {
    cvb_set_error("head_train: null argument");
    return CVB_EINVAL;
  }
  if (B <= 0 || C <= 0 || C > HO || fin <= 0 || fin % 256 || fin > 1024 || ldx % 8 || ldx < fin ||
      (dx && (lddx % 8 || lddx < fin))) {
    cvb_set_error("head_train: need 0 < C <= 16, fin a multiple of 256 and <= 1024, row strides multiples of 8");
    return CVB_EINVAL;
  }
  if (((uintptr_t)x | (uintptr_t)w | (uintptr_t)part | (uintptr_t)dw | (uintptr_t)dx | (uintptr_t)dprev_b) & 15) {
    cvb_set_error("head_train: x, w, dx, dw, dprev_b and part must be 16-byte aligned");
    return CVB_EINVAL;
  }
  int grid = 0;
  int rc = head_grid(B, fin, &grid);
  if (rc) return rc;
  int dev = 0;
  CVB_CUDA(cudaGetDevice(&dev));
  static unsigned* bars[64] = {nullptr};
  if (!bars[dev]) {
    CVB_CUDA(cudaMalloc(&bars[dev], CVB_GRID_BAR_WORDS * sizeof(unsigned)));
    CVB_CUDA(cudaMemset(bars[dev], 0, CVB_GRID_BAR_WORDS * sizeof(unsigned)));
  }
  HeadArgs a;
  a.x = (const bf16*)x; a.ldx = ldx; a.w = (const bf16*)w; a.bias = bias; a.labels = labels;
  a.B = B; a.fin = fin; a.C = C; a.relu_mask = relu_mask; a.scale = scale;
  a.logits = logits; a.dlogits = (bf16*)dlogits; a.row_loss = row_loss; a.loss = loss;
  a.dx = (bf16*)dx; a.lddx = lddx; a.dw = dw; a.db = db; a.dprev_b = dprev_b; a.part = part;
  a.E = head_E(fin); a.bar = bars[dev];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(HT);
  cfg.dynamicSmemBytes = head_smem(fin);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CVB_CUDA(cudaLaunchKernelEx(&cfg, head_train_kernel, a));
  return CVB_OK;
}
