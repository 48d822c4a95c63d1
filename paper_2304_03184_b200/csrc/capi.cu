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

namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// random double: sign, exponent in [-e_span, e_span], significand random or
// one of the adversarial patterns (all ones, all zeros, lowest bit only)
__device__ __forceinline__ double rand_double(uint64_t h, int e_span) {
  const uint64_t h2 = mix64(h);
  uint64_t mant = h2 & 0xfffffffffffffull;
  switch ((h >> 60) & 7) {
    case 0: mant = 0xfffffffffffffull; break;
    case 1: mant = 0; break;
    case 2: mant = 1; break;
    default: break;
  }
  const int e = (int)((h >> 8) % (uint64_t)(2 * e_span + 1)) - e_span;
  const uint64_t bits = ((h & 1ull) << 63) | ((uint64_t)(e + 1023) << 52) | mant;
  return __longlong_as_double((long long)bits);
}

__global__ void selftest_div_kernel(int64_t n, uint64_t seed, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed ^ mix64((uint64_t)i));
    const double b = rand_double(h, (i & 1) ? 8 : 600);
    const ExactDiv by_b(b);
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
      const double a = (j == 7) ? 0.0 * b : rand_double(mix64(h + 1 + j), (i & 1) ? 8 : 600);
      const double q0 = x_div(a, b), q1 = by_b(a);
      local += __double_as_longlong(q0) != __double_as_longlong(q1) && !(q0 != q0 && q1 != q1);
    }
  }
  if (local) atomicAdd(bad, local);
}
}  // namespace

extern "C" {
int cf_selftest_exact_div(int64_t n, uint64_t seed, int64_t* mismatches) {
  if (n < 0 || !mismatches) return cf::fail(CF_E_BAD_ARG, "cf_selftest_exact_div: bad args");
  unsigned long long* d = nullptr;
  CF_CHECK_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  cudaMemset(d, 0, sizeof(unsigned long long));
  selftest_div_kernel<<<cf::grid_for(n, 256, 8), 256>>>(n, seed, d);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cf::fail(CF_E_CUDA, std::string("cf_selftest_exact_div: ") + cudaGetErrorString(e));
  *mismatches = (int64_t)h;
  return CF_OK;
}

int cf_version(void) { return 1; }
const char* cf_last_error(void) { return g_last_error.c_str(); }
int cf_device_sm_count(void) { return cf::sm_count(); }
}

