// Optimiser and weight-layout kernels of the training step (SPEC train_step,
// SPEC.md:390-398, 421): fused Adam over flat fp32 parameter arrays (hash tables,
// MLP master weights) and the fp32 -> fp16 canonical-layout repack that feeds the
// tcgen05 kernels after every update.
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"

namespace {

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float c1,
                            float c2, float gs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i] * gs;
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi * c1) / (sqrtf(vi * c2) + eps);
  }
}

__global__ void pack_kernel(const float* __restrict__ w, int n, int k, int np, int kp, uint8_t* __restrict__ blob) {
  const int total = np * kp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int r = e / kp, c = e % kp;
    const float x = (r < n && c < k) ? w[r * k + c] : 0.0f;
    *reinterpret_cast<__half*>(blob + tc::core_offset(r, c, kp)) = __float2half_rn(x);
  }
}

// out[c] += sum_{r < n} x[r * ld + c], c < 128: fp16 rows, fp32 accumulation
// (DeformNet's theta gradient needs the column sums of dL/dpre1 over a frame)
__global__ void colsum128_kernel(const __half* __restrict__ x, int64_t n, int ld, float* __restrict__ out) {
  __shared__ float part[256];
  const int c = threadIdx.x & 127, rg = threadIdx.x >> 7;
  float acc = 0.0f;
  for (int64_t r = (int64_t)blockIdx.x * 2 + rg; r < n; r += (int64_t)gridDim.x * 2)
    acc += __half2float(x[r * ld + c]);
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < 128) atomicAdd(out + c, part[threadIdx.x] + part[threadIdx.x + 128]);
}

}  // namespace

extern "C" {

int cf_colsum128_f16(const void* x, int64_t n, int ld, float* out, void* stream) {
  if (!x || !out || n < 0 || ld < 128) return cf::fail(CF_E_BAD_ARG, "cf_colsum128_f16: bad args");
  if (n == 0) return CF_OK;
  colsum128_kernel<<<cf::grid_for((n + 1) / 2, 1, 4), 256, 0, cf::as_stream(stream)>>>(
      reinterpret_cast<const __half*>(x), n, ld, out);
  return cf::check_launch("cf_colsum128_f16");
}

int cf_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float beta1, float beta2, float eps,
            int step, float grad_scale, void* stream) {
  if (!p || !g || !m || !v || n < 0 || step < 1) return cf::fail(CF_E_BAD_ARG, "cf_adam: bad args");
  if (n == 0) return CF_OK;
  const float c1 = 1.0f / (1.0f - powf(beta1, (float)step)), c2 = 1.0f / (1.0f - powf(beta2, (float)step));
  adam_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(p, g, m, v, n, lr, beta1, beta2, eps, c1,
                                                                          c2, grad_scale);
  return cf::check_launch("cf_adam");
}

int cf_pack_weight(const float* w, int n, int k, uint8_t* blob, void* stream) {
  if (!w || !blob || n < 1 || k < 1) return cf::fail(CF_E_BAD_ARG, "cf_pack_weight: bad args");
  const int np = (n + 15) / 16 * 16, kp = (k + 15) / 16 * 16;
  pack_kernel<<<cf::grid_for((int64_t)np * kp, 256, 2), 256, 0, cf::as_stream(stream)>>>(w, n, k, np, kp, blob);
  return cf::check_launch("cf_pack_weight");
}

}  // extern "C"
