// Optimiser and weight-layout kernels of the training step (SPEC train_step,
// SPEC.md:390-398, 421): fused Adam over flat fp32 parameter arrays (hash tables,
// MLP master weights) and the fp32 -> fp16 canonical-layout repack that feeds the
// tcgen05 kernels after every update.
#include <cuda_fp16.h>

#include <cuda.h>
#include <cudaTypedefs.h>

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

__global__ void pack_kernel(const float* __restrict__ w, int n, int k, int np, int kp, uint8_t* __restrict__ blob,
                            uint8_t* __restrict__ blob_lo) {
  const int total = np * kp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int r = e / kp, c = e % kp;
    const float x = (r < n && c < k) ? w[r * k + c] : 0.0f;
    const __half h = __float2half_rn(x);
    *reinterpret_cast<__half*>(blob + tc::core_offset(r, c, kp)) = h;
    if (blob_lo) *reinterpret_cast<__half*>(blob_lo + tc::core_offset(r, c, kp)) = __float2half_rn(x - __half2float(h));
  }
}

// ---------------------------------------------------------------- dW = dY X^T
// Split-K weight-gradient GEMM on tcgen05: C[128 x N] += A[128 x K] B[N x K]^T with
// both operands K-major (row stride lda / ldb elements) — the feature-major saved
// activations and dL/dpre of DeformNet, where K = the frame's samples. Each CTA
// (one per SM) owns a contiguous range of 64-wide K tiles. Warp-specialised: one
// thread streams the tiles with TMA (2-D boxes of 8 halves x rows, zero fill past
// K) into a 6-stage ring, one thread issues 4 MMAs (K = 16) per tile into a
// 128 x N fp32 TMEM accumulator and commits each stage back to the producer; the
// four warps then add the partial product into C with fp32 atomics.
//
// A TMA box of 64 halves x R rows with the 128-byte swizzle lands as the canonical
// K-major SWIZZLE_128B layout: 128-byte rows, 8-row atoms of 1024 B (SBO), the 16 B
// chunks of row r XOR-permuted by r % 8; a K = 16 step advances the start by 32 B.
constexpr int kGKT = 64;  // K per stage
constexpr int kGStages = 6;

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;           // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: next 8-row atom
  d |= (uint64_t)1 << 46;           // version
  d |= (uint64_t)2 << 61;           // layout: SWIZZLE_128B
  return d;
}

template <int N>
__global__ void __launch_bounds__(128, 1) gemm_kmajor_kernel(const __grid_constant__ CUtensorMap map_a,
                                                             const __grid_constant__ CUtensorMap map_b, int64_t K,
                                                             float* __restrict__ C, int ldc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kGStages], empty[kGStages], done;
  __shared__ uint32_t tmem_base;
  constexpr int kStageA = 128 * kGKT * 2, kStageB = N * kGKT * 2, kStage = kStageA + kStageB;
  const int tid = threadIdx.x, warp = tid / 32;
  const int64_t T = (K + kGKT - 1) / kGKT;
  const int64_t per = (T + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per, nt = max((int64_t)0, min(per, T - t0));
  if (nt == 0) return;
  if (tid == 0) {
    for (int q = 0; q < kGStages; ++q) {
      tc::bar_init(&full[q], 1);
      tc::bar_init(&empty[q], 1);
    }
    tc::bar_init(&done, 1);
    tc::bar_fence_init();
  }
  if (warp == 2) tc::tmem_alloc<N < 32 ? 32 : N>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t sbase = tc::smem_u32(smem);
  if (tid == 0) {
    // TMA producer
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % kGStages);
      if (i >= kGStages) tc::bar_wait(&empty[st], (uint32_t)(((i / kGStages) - 1) & 1));
      bar_expect_tx(&full[st], kStage);
      const int k0 = (int)((t0 + i) * kGKT);
      const uint32_t sa = sbase + st * kStage, sb = sa + kStageA;
      tma_load_2d(sa, &map_a, k0, 0, &full[st]);
      tma_load_2d(sb, &map_b, k0, 0, &full[st]);
    }
  } else if (tid == 32) {
    // MMA issuer
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % kGStages);
      tc::bar_wait(&full[st], (uint32_t)((i / kGStages) & 1));
      tc::fence_after();
      const uint32_t sa = sbase + st * kStage, sb = sa + kStageA;
#pragma unroll
      for (int ks = 0; ks < kGKT / 16; ++ks) {
        const uint64_t ad = sdesc_sw128(sa + ks * 32);
        const uint64_t bd = sdesc_sw128(sb + ks * 32);
        tc::mma_f16(tmem_base, ad, bd, idesc, (i > 0 || ks > 0) ? 1u : 0u);
      }
      tc::mma_commit(&empty[st]);
    }
    tc::mma_commit(&done);
  }
  tc::bar_wait(&done, 0);
  __syncwarp();  // producer / issuer lanes rejoin their warps before the aligned TMEM loads
  tc::fence_after();
  const int row = warp * 32 + (tid & 31);
  const bool vec4 = (ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(C) % 16) == 0;
#pragma unroll 1
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    float* dst = C + (int64_t)row * ldc + c0;
    if (vec4) {
#pragma unroll
      for (int c = 0; c < 32; c += 4)
        atomicAdd(reinterpret_cast<float4*>(dst + c), make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]));
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) atomicAdd(dst + c, v[c]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_free<N < 32 ? 32 : N>(tmem_base);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// rows x K fp16, row stride ld elements; boxes of 64 halves (128 B) x rows, 128B swizzle
bool make_map(CUtensorMap* map, const void* base, int rows, int64_t K, int64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
  if (K >= (int64_t)1 << 31) return cf::fail(CF_E_BAD_ARG, "cf_gemm_kmajor_f16: K must be < 2^31");
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, 128, K, lda) || !make_map(&mb, B, n_cols, K, ldb))
    return cf::fail(CF_E_CUDA, "cf_gemm_kmajor_f16: cuTensorMapEncodeTiled failed");
  const int64_t T = (K + kGKT - 1) / kGKT;
  const unsigned grid = (unsigned)std::min<int64_t>(T, cf::sm_count());
  cudaStream_t st = cf::as_stream(stream);
  auto run = [&](auto kern, int N) -> int {
    const int smem = kGStages * (128 + N) * kGKT * 2;
    CF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, 128, smem, st>>>(ma, mb, K, C, ldc);
    return CF_OK;
  };
  int rc = n_cols == 128 ? run(gemm_kmajor_kernel<128>, 128)
                         : (n_cols == 64 ? run(gemm_kmajor_kernel<64>, 64) : run(gemm_kmajor_kernel<32>, 32));
  if (rc) return rc;
  return cf::check_launch("cf_gemm_kmajor_f16");
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
  pack_kernel<<<cf::grid_for((int64_t)np * kp, 256, 2), 256, 0, cf::as_stream(stream)>>>(w, n, k, np, kp, blob,
                                                                                          nullptr);
  return cf::check_launch("cf_pack_weight");
}

int cf_pack_weight_split(const float* w, int n, int k, uint8_t* blob, uint8_t* blob_lo, void* stream) {
  if (!w || !blob || !blob_lo || n < 1 || k < 1) return cf::fail(CF_E_BAD_ARG, "cf_pack_weight_split: bad args");
  const int np = (n + 15) / 16 * 16, kp = (k + 15) / 16 * 16;
  pack_kernel<<<cf::grid_for((int64_t)np * kp, 256, 2), 256, 0, cf::as_stream(stream)>>>(w, n, k, np, kp, blob,
                                                                                          blob_lo);
  return cf::check_launch("cf_pack_weight_split");
}

}  // extern "C"
