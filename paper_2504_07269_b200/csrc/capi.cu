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
