// C-ABI plumbing shared by every translation unit: thread-local last error,
// launch checking and device queries.
#include <string>

#include "common.cuh"

namespace {
thread_local std::string g_last_error;
int g_sm_count = 0;
}  // namespace

namespace cf {

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return CF_OK;
}

int sm_count() {
  if (g_sm_count == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      g_sm_count = v;
    else
      g_sm_count = 148;
  }
  return g_sm_count;
}

}  // namespace cf

extern "C" {
int cf_version(void) { return 1; }
const char* cf_last_error(void) { return g_last_error.c_str(); }
int cf_device_sm_count(void) { return cf::sm_count(); }
}
