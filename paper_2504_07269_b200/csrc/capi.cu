// C-ABI plumbing: thread-local error message, version, device query.
#include <stdio.h>

#include <string>

#include "common.cuh"

namespace stfem {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %d (%s) at %s", (int)e, cudaGetErrorString(e), where);
  g_last_error = buf;
  return e == cudaErrorMemoryAllocation ? STFEM_ERR_NOMEM : STFEM_ERR_CUDA;
}

}  // namespace stfem

extern "C" const char* stfem_last_error(void) { return stfem::g_last_error.c_str(); }

extern "C" int stfem_version(void) { return 1; }

extern "C" int stfem_cuda_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

// Column block of a row-strided complex array between host and device
// (cudaMemcpy2DAsync): rows x ncols complex128, leading dimensions in elements.
// kind 0: host -> device, 1: device -> host.  Used by the pipelined
// host-buffer solve (H2D of chunk c+1 overlaps the transform of chunk c).
extern "C" int stfem_copy_cols(void* dst, int64_t ld_dst, const void* src, int64_t ld_src, int64_t ncols,
                               int64_t rows, int32_t kind, void* stream) {
  if (!dst || !src) return stfem::fail(STFEM_ERR_ARG, "copy_cols: null pointer");
  if (ncols < 0 || rows < 0 || ld_dst < ncols || ld_src < ncols)
    return stfem::fail(STFEM_ERR_DIM, "copy_cols: bad dimensions");
  if (ncols == 0 || rows == 0) return STFEM_OK;
  STFEM_CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)ld_dst * 16, src, (size_t)ld_src * 16, (size_t)ncols * 16,
                                   (size_t)rows, kind == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                   (cudaStream_t)stream));
  return STFEM_OK;
}
