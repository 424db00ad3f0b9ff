// Shared helpers for the covault-b200 CUDA library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#define CVB_OK 0
#define CVB_AUTH_FAIL 1
#define CVB_EINVAL (-1)
#define CVB_ECUDA (-2)
#define CVB_ENOMEM (-3)

void cvb_set_error(const char* fmt, ...);

#define CVB_CUDA(expr)                                                                 \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      cvb_set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return CVB_ECUDA;                                                                \
    }                                                                                  \
  } while (0)

#define CVB_CHECK_LAUNCH()                                                             \
  do {                                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess) {                                                           \
      cvb_set_error("%s:%d launch -> %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return CVB_ECUDA;                                                                \
    }                                                                                  \
  } while (0)

// SM count of the current device, cached per device (safe to call during graph capture).
static inline int cvb_num_sms() {
  static int cache[64] = {0};
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
}

#define CVB_API extern "C" __attribute__((visibility("default")))
