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

// True the first time it is called for the current device with this flag word (one bit per
// device): per-device one-time setup such as cudaFuncSetAttribute, which is per device.
static inline bool cvb_first_on_device(unsigned long long* mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(mask, __ATOMIC_ACQUIRE) & bit) return false;
  __atomic_fetch_or(mask, bit, __ATOMIC_ACQ_REL);
  return true;
}

// ---- grid-wide barrier for co-resident (cooperative / persistent) grids -------------------
// One arrival counter + a generation word every CTA polls; returns the counter to zero.
// (A two-level variant -- 16-CTA group counters on separate lines -- measured 5-10% slower on
// the BN kernels, so the flat form stays.)  Workspace: CVB_GRID_BAR_WORDS zeroed uint32 words.
#define CVB_GRID_BAR_WORDS 32
#ifdef __CUDACC__
__device__ __forceinline__ void cvb_grid_barrier(unsigned* bar) {
  // release/acquire form: one acq_rel arrival (releases this CTA's writes, ordered before it
  // by the __syncthreads), acquire polling of the generation word -- no full (sc) fences
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g, old;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
        if (cur == g) __nanosleep(32);
      } while (cur == g);
    }
  }
  __syncthreads();
}
#endif

#define CVB_API extern "C" __attribute__((visibility("default")))

// ---- programmatic dependent launch (PDL) -----------------------------------------------
// Every kernel launched through cvb_launch starts with CVB_PDL_PROLOGUE(): it waits for the
// previous kernel in the stream to complete (griddepcontrol.wait -- required in EVERY such
// kernel so completion stays transitive) and lets the next kernel be scheduled while this
// one drains (griddepcontrol.launch_dependents).  Inside a CUDA graph this turns the
// ~2-5 us launch gap + ramp of each of the step's ~50-1000 small kernels into overlap.
// Without the launch attribute both instructions are no-ops.
#define CVB_PDL_PROLOGUE()                                              \
  do {                                                                  \
    asm volatile("griddepcontrol.wait;" ::: "memory");                  \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");     \
  } while (0)

#include <stdlib.h>
#include <utility>
static inline bool cvb_pdl_enabled() {
  static int on = -1;
  if (on < 0) on = getenv("CVB_NO_PDL") ? 0 : 1;
  return on != 0;
}
template <typename... KArgs, typename... Args>
static inline cudaError_t cvb_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cvb_pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
