// Record decoder of the decrypt-and-normalise loader (K1b of DESIGN.md).
//
// Consumes a verified plaintext shard of fixed-size binary records (CIFAR-10 binary layout:
// 1 label byte + C*H*W CHW pixel bytes; the medical set uses the same layout with C=1,
// H=W=224) that the GCM kernel wrote to HBM, and produces the training input tile:
// NHWC with channels zero-padded to `cpad` (so every pixel is one 16-byte row for the
// implicit-GEMM conv TMA boxes), value (x/255 - mean_c) / std_c in bf16 or fp32, plus int32
// labels.  One thread per pixel: byte reads of a channel plane are contiguous across the
// warp, output rows are 16/32-byte vector stores contiguous across the warp.
// The reference equivalent is Volume.get + bytes.decode + parse_dataset
// (/root/reference/pkg/src/covault/volume.py:185-197, workload.py:24-41), which parses CSV
// text; the binary record payload is the B200 dataset format.
#include "cvb_common.cuh"
#include <cuda_bf16.h>

struct RecParams {
  const uint8_t* pt;
  int64_t nrec, rec_bytes, hw, c, cpad;
  float scale[8], shift[8];  // v = x * scale_c + shift_c
  void* out;
  int32_t* labels;
};

template <typename T>
__global__ void records_to_nhwc(const __grid_constant__ RecParams p) {
  CVB_PDL_PROLOGUE();
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = p.nrec * p.hw;
  if (gid >= total) return;
  int64_t r = gid / p.hw, px = gid - r * p.hw;
  const uint8_t* rec = p.pt + r * p.rec_bytes;
  if (px == 0) p.labels[r] = rec[0];
  T v[8];
#pragma unroll
  for (int c = 0; c < 8; c++) {
    float x = 0.f;
    if (c < p.c) x = __fmaf_rn((float)rec[1 + c * p.hw + px], p.scale[c], p.shift[c]);   // one rounding
    v[c] = (T)x;
  }
  T* out = reinterpret_cast<T*>(p.out) + gid * p.cpad;
  if (sizeof(T) == 2) {
    *reinterpret_cast<uint4*>(out) = *reinterpret_cast<uint4*>(v);
  } else {
    reinterpret_cast<uint4*>(out)[0] = reinterpret_cast<uint4*>(v)[0];
    reinterpret_cast<uint4*>(out)[1] = reinterpret_cast<uint4*>(v)[1];
  }
}

// dtype: 0 = bf16, 1 = fp32.  cpad must be 8 (one 16-byte bf16 row / 32-byte fp32 row).
CVB_API int cvb_records_to_nhwc(const uint8_t* pt_dev, int64_t nrec, int64_t rec_bytes, int64_t c,
                                   int64_t h, int64_t w, const float* mean, const float* std,
                                   int dtype, void* out_dev, int32_t* labels_dev, void* stream) {
  if (!pt_dev || !out_dev || !labels_dev || c < 1 || c > 8 || rec_bytes != 1 + c * h * w || nrec < 0) {
    cvb_set_error("records_to_nhwc: bad arguments");
    return CVB_EINVAL;
  }
  if (nrec == 0) return CVB_OK;
  RecParams p;
  memset(&p, 0, sizeof(p));
  p.pt = pt_dev; p.nrec = nrec; p.rec_bytes = rec_bytes; p.hw = h * w; p.c = c; p.cpad = 8;
  for (int i = 0; i < 8; i++) {
    float m = (mean && i < c) ? mean[i] : 0.f, sd = (std && i < c) ? std[i] : 1.f;
    p.scale[i] = 1.0f / (255.0f * sd);
    p.shift[i] = -m / sd;
  }
  p.out = out_dev; p.labels = labels_dev;
  int64_t total = nrec * p.hw;
  unsigned grid = (unsigned)((total + 255) / 256);
  if (dtype == 0) cvb_launch(records_to_nhwc<__nv_bfloat16>, grid, 256, 0, (cudaStream_t)stream, p);
  else cvb_launch(records_to_nhwc<float>, grid, 256, 0, (cudaStream_t)stream, p);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}
