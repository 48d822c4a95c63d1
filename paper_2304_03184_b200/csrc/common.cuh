// Shared helpers: status plumbing, launch sizing, IEEE-exact fp64 arithmetic.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <initializer_list>
#include <utility>

#include "../../include/capfields_b200.h"

namespace cf {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);
int sm_count();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// grid for a grid-stride kernel: enough CTAs for `per_sm` resident CTAs on every SM
inline unsigned grid_for(int64_t n, int block, int per_sm = 8) {
  int64_t need = (n + block - 1) / block;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (need < 1) need = 1;
  return (unsigned)(need < cap ? need : cap);
}

// Programmatic dependent launch (PDL): the kernel is launched while its stream
// predecessor drains, so its launch latency and prologue overlap the
// predecessor's tail. Kernels launched this way call pdl_wait() before touching
// any memory the predecessor reads or writes, and pdl_trigger() once their CTA's
// work is done (launch-completion of the next kernel); both are no-ops for a
// normal launch. In a captured graph these become programmatic edges.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Fill n 32-bit words with `value` by a kernel. The frame's buffer resets use this
// instead of cudaMemsetAsync: memset nodes in the frame's graph went through the
// copy engine and queued behind the previous frame's image read-back.
static __global__ void fill_u32_kernel(uint32_t* __restrict__ p, uint32_t value, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = value;
}
inline void fill_u32(void* p, uint32_t value, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int block = 256;
  int64_t grid = (n + block - 1) / block;
  if (grid > 1024) grid = 1024;
  fill_u32_kernel<<<(unsigned)grid, block, 0, st>>>(reinterpret_cast<uint32_t*>(p), value, n);
}

}  // namespace cf

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#define CF_CHECK_CUDA(call)                                                                 \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess) return cf::fail(CF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// IEEE round-to-nearest fp64 ops that ptxas may not contract into FMAs. The
// reference evaluates every expression as separate numpy ufunc calls, each a
// correctly rounded binary op; using these keeps the device result bit-equal.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double x_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double x_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double x_sub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double x_div(double a, double b) { return __ddiv_rn(a, b); }

// Correctly rounded a / b for many numerators over one denominator: with
// y = RN(1/b) and the faithful q = RN(a*y), the exact residual r = a - b*q
// (one FMA) gives RN(a/b) = RN(q + r*y) (Markstein's theorem; __ddiv_rn ends
// with the same correction step after refining y). Bit-equal to x_div; the
// residual is exact only away from the subnormal range, so tiny or huge
// operands take __ddiv_rn.
struct ExactDiv {
  double b, y;
  bool fast;
  __device__ __forceinline__ explicit ExactDiv(double b_) : b(b_) {
    y = __drcp_rn(b_);
    const double ab = fabs(b_);
    fast = ab > 0x1p-500 && ab < 0x1p500;
  }
  __device__ __forceinline__ double operator()(double a) const {
    const double aa = fabs(a);
    if (!fast || !(aa < 0x1p500) || (aa < 0x1p-500 && a != 0.0)) return __ddiv_rn(a, b);
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, b, a);
    return r == 0.0 ? q : __fma_rn(r, y, q);  // r == 0: q exact (keeps the sign of a zero quotient)
  }
};

__device__ __forceinline__ float f_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float f_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float f_sub(float a, float b) { return __fadd_rn(a, -b); }

struct d3 {
  double x, y, z;
};

__device__ __forceinline__ d3 load_d3(const double* p) { return d3{p[0], p[1], p[2]}; }
__device__ __forceinline__ void store_d3(double* p, d3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}

// sum((a - b)**2) with numpy's sequential reduction order: (dx*dx + dy*dy) + dz*dz
__device__ __forceinline__ double sqdist(d3 a, d3 b) {
  double dx = x_sub(a.x, b.x), dy = x_sub(a.y, b.y), dz = x_sub(a.z, b.z);
  return x_add(x_add(x_mul(dx, dx), x_mul(dy, dy)), x_mul(dz, dz));
}

// Order-preserving uint64 keys of doubles (x < y <=> key(x) < key(y); no NaNs): a
// float64 bounding box by integer atomicMin / atomicMax
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

namespace cf {
// Several fills in ONE launch, launched with PDL (waits for the stream predecessor
// before writing): the frame's counter / bit-grid resets between its kernels.
struct FillSpan {
  void* p;
  uint32_t v;
  int64_t n;  // 32-bit words
};
struct FillList {
  FillSpan s[4];
  int count;
};
static __global__ void fill_list_kernel(FillList L) {
  pdl_wait();
  for (int k = 0; k < L.count; ++k) {
    uint32_t* p = reinterpret_cast<uint32_t*>(L.s[k].p);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.s[k].n;
         i += (int64_t)gridDim.x * blockDim.x)
      p[i] = L.s[k].v;
  }
  pdl_trigger();
}
inline void fill_list(cudaStream_t st, std::initializer_list<FillSpan> spans) {
  FillList L{};
  int64_t most = 1;
  for (const FillSpan& f : spans) {
    if (f.n <= 0 || L.count == 4) continue;
    L.s[L.count++] = f;
    most = f.n > most ? f.n : most;
  }
  if (L.count == 0) return;
  int64_t grid = (most + 255) / 256;
  if (grid > 1024) grid = 1024;
  cf::launch_pdl(fill_list_kernel, dim3((unsigned)grid), dim3(256), 0, st, L);
}
}  // namespace cf
