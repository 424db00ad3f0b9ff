// C-ABI plumbing shared by every entry point: error strings, version, device selection.
#include "cvb_common.cuh"
#include <stdarg.h>

static thread_local char g_err[512] = "";

void cvb_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

CVB_API const char* cvb_last_error(void) { return g_err; }

CVB_API int cvb_version(void) { return 1; }

// Make this library's CUDA runtime use the same device as the caller (torch).
CVB_API int cvb_set_device(int dev) {
  CVB_CUDA(cudaSetDevice(dev));
  return CVB_OK;
}

CVB_API int cvb_device_sync(void) {
  CVB_CUDA(cudaDeviceSynchronize());
  return CVB_OK;
}
