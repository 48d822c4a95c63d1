// Optimiser and weight-layout kernels of the training step (SPEC train_step,
// SPEC.md:390-398, 421): fused Adam over flat fp32 parameter arrays (hash tables,
// MLP master weights) and the fp32 -> fp16 canonical-layout repack that feeds the
// tcgen05 kernels after every update.
#include <cuda_fp16.h>

#include <algorithm>

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

// ---------------------------------------------------------------- dW = dY X^T
// Split-K weight-gradient GEMM on tcgen05: C[128 x N] += A[128 x K] B[N x K]^T with
// both operands K-major (row stride lda / ldb elements) — the feature-major saved
// activations and dL/dpre of DeformNet, where K = the frame's samples. Each CTA
// (one per SM) owns a contiguous range of 64-wide K tiles: cp.async (16 B, zero-
// filled past K) into a 4-stage ring of canonical K-major smem tiles, one elected
// thread issues 4 MMAs (K = 16) per tile into a 128 x N fp32 TMEM accumulator and
// commits to the stage's mbarrier, which gates the stage's refill. The partial
// product is added into C with fp32 atomics (one per element per CTA).
constexpr int kGKT = 64;     // K per stage
constexpr int kGStages = 4;

// 16-byte async copy of the 8 halves at k .. k+7 of a row; the part past K is zero-filled
__device__ __forceinline__ void cp_async_k8(uint32_t dst, const __half* row, int64_t k, int64_t K) {
  const int64_t left = K - k;
  const int bytes = left >= 8 ? 16 : (left > 0 ? (int)left * 2 : 0);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(row + (left > 0 ? k : 0)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int N>
__global__ void __launch_bounds__(128, 1) gemm_kmajor_kernel(const __half* __restrict__ A, int64_t lda,
                                                             const __half* __restrict__ B, int64_t ldb, int64_t K,
                                                             float* __restrict__ C, int ldc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kGStages];
  __shared__ uint32_t tmem_base;
  constexpr int kStageA = 128 * kGKT * 2, kStageB = N * kGKT * 2, kStage = kStageA + kStageB;
  const int tid = threadIdx.x, warp = tid / 32;
  const int64_t T = (K + kGKT - 1) / kGKT;
  const int64_t per = (T + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per, nt = max((int64_t)0, min(per, T - t0));
  if (nt == 0) return;
  if (tid == 0) {
    for (int q = 0; q < kGStages; ++q) tc::bar_init(&mbar[q], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<N < 32 ? 32 : N>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t sbase = tc::smem_u32(smem);
  auto load = [&](int stage, int64_t tile) {
    const int64_t k0 = (t0 + tile) * kGKT;
    const uint32_t sa = sbase + stage * kStage, sb = sa + kStageA;
    // 16-byte chunks: (row, c) with c = 8-half group along K; 8 consecutive lanes read a row's 128 B
#pragma unroll
    for (int i = 0; i < (128 * 8) / 128; ++i) {
      const int q = tid + 128 * i, r = q >> 3, c = q & 7;
      cp_async_k8(sa + tc::core_offset(r, 8 * c, kGKT), A + r * lda, k0 + 8 * c, K);
    }
#pragma unroll
    for (int i = 0; i < (N * 8 + 127) / 128; ++i) {
      const int q = tid + 128 * i, r = q >> 3, c = q & 7;
      if (r < N) cp_async_k8(sb + tc::core_offset(r, 8 * c, kGKT), B + r * ldb, k0 + 8 * c, K);
    }
  };
#pragma unroll
  for (int s = 0; s < kGStages - 1; ++s) {
    if (s < nt) load(s, s);
    cp_async_commit();
  }
  constexpr uint32_t idesc = tc::idesc_f16(128, N);
  for (int64_t i = 0; i < nt; ++i) {
    const int stage = (int)(i % kGStages);
    cp_async_wait<kGStages - 2>();
    tc::fence_async_smem();  // cp.async (generic proxy) -> tcgen05.mma (async proxy)
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      const uint32_t sa = sbase + stage * kStage, sb = sa + kStageA;
#pragma unroll
      for (int ks = 0; ks < kGKT / 16; ++ks) {
        const uint64_t ad = tc::sdesc(sa + ks * 256, 128, kGKT * 16);
        const uint64_t bd = tc::sdesc(sb + ks * 256, 128, kGKT * 16);
        tc::mma_f16(tmem_base, ad, bd, idesc, (i > 0 || ks > 0) ? 1u : 0u);
      }
      tc::mma_commit(&mbar[stage]);
    }
    const int64_t j = i + kGStages - 1;  // refill the stage the previous tile's MMAs read
    if (j < nt) {
      if (i >= 1) tc::bar_wait(&mbar[(i - 1) % kGStages], (uint32_t)(((i - 1) / kGStages) & 1));
      load((int)(j % kGStages), j);
    }
    cp_async_commit();
  }
  tc::bar_wait(&mbar[(nt - 1) % kGStages], (uint32_t)(((nt - 1) / kGStages) & 1));
  tc::fence_after();
  const int row = warp * 32 + (tid & 31);
#pragma unroll 1
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    float* dst = C + (int64_t)row * ldc + c0;
#pragma unroll
    for (int c = 0; c < 32; ++c) atomicAdd(dst + c, v[c]);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<N < 32 ? 32 : N>(tmem_base);
}

}  // namespace

extern "C" {

int cf_gemm_kmajor_f16(const void* A, int64_t lda, const void* B, int64_t ldb, int n_cols, int64_t K, float* C,
                       int ldc, void* stream) {
  if (!A || !B || !C || K < 0 || lda < K || ldb < K || (n_cols != 128 && n_cols != 64 && n_cols != 32) ||
      ldc < n_cols)
    return cf::fail(CF_E_BAD_ARG, "cf_gemm_kmajor_f16: bad args (128 x {32,64,128}, lda/ldb >= K)");
  if ((lda | ldb) % 8 != 0 || (reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) % 16 != 0)
    return cf::fail(CF_E_BAD_ARG, "cf_gemm_kmajor_f16: operands need 16-byte aligned rows (lda, ldb % 8 == 0)");
  if (K == 0) return CF_OK;
  const int64_t T = (K + kGKT - 1) / kGKT;
  const unsigned grid = (unsigned)std::min<int64_t>(T, cf::sm_count());
  cudaStream_t st = cf::as_stream(stream);
  auto run = [&](auto kern, int N) -> int {
    const int smem = kGStages * (128 + N) * kGKT * 2;
    CF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, 128, smem, st>>>(reinterpret_cast<const __half*>(A), lda, reinterpret_cast<const __half*>(B), ldb,
                                  K, C, ldc);
    return CF_OK;
  };
  int rc = n_cols == 128 ? run(gemm_kmajor_kernel<128>, 128)
                         : (n_cols == 64 ? run(gemm_kmajor_kernel<64>, 64) : run(gemm_kmajor_kernel<32>, 32));
  if (rc) return rc;
  return cf::check_launch("cf_gemm_kmajor_f16");
}

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
