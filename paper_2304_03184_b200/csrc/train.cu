// Optimiser and weight-layout kernels of the training step (SPEC train_step,
// SPEC.md:390-398, 421): fused Adam over flat fp32 parameter arrays (hash tables,
// MLP master weights) and the fp32 -> fp16 canonical-layout repack that feeds the
// tcgen05 kernels after every update.
#include <cuda_fp16.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>

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
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(tc::smem_u32(bar))
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

// ---------------------------------------------------------------- grouped dW, K on the device
// Up to kMaxDw weight-gradient problems of one field in ONE launch (a 1-D grid, problem
// p on CTAs [cta0[p], cta0[p + 1])): C_p[m_p x n_p] += A_p[m_p x K] B_p[n_p x K]^T, both
// operands K-major fp16 (K-blocked feature-major saves, K = samples), K = min(*count, capacity) read on the
// device — no host sync, and the launch is graph-capturable. Same pipeline as
// gemm_kmajor_kernel with runtime shapes: the A box is always 128 rows (TMA fills
// rows >= m_p with zeros, the MMA is M = 128), the B box n_mma rows (n_p rounded up
// to 16), the epilogue adds only rows < m_p and columns < n_p.
constexpr int kMaxDw = 10;
struct DwProb {
  CUtensorMap a, b;
  float* C;
  int ldc, m, n, n_mma;
};
struct DwGroup {
  DwProb p[kMaxDw];
  int cta0[kMaxDw + 1];  // problem p owns CTAs [cta0[p], cta0[p + 1]) of the 1-D grid
  const int* count;
  int64_t capacity;
};

// A stage holds kDwBoxes consecutive 64-wide K boxes of each operand, loaded back to
// back: every operand row (one feature, K contiguous) is then read kDwBoxes x 128 B at
// a time instead of 128 B per stage period (DRAM row-buffer locality).
constexpr int kDwBoxes = 2, kDwStages = kGStages / kDwBoxes, kDwKT = kGKT * kDwBoxes;
constexpr int kDwBox = 128 * kGKT * 2;  // one 64 x 128-row box, 16 KB

__global__ void __launch_bounds__(128, 1) dw_grouped_kernel(const __grid_constant__ DwGroup G) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kDwStages], empty[kDwStages], done;
  __shared__ uint32_t tmem_base;
  int pi = 0;
  while ((int)blockIdx.x >= G.cta0[pi + 1]) ++pi;
  const DwProb& P = G.p[pi];
  const int bx = (int)blockIdx.x - G.cta0[pi], gx = G.cta0[pi + 1] - G.cta0[pi];
  const int N = P.n_mma;
  constexpr int kStageA = kDwBoxes * kDwBox, kStage = 2 * kStageA;
  const uint32_t tx = (uint32_t)(kDwBox + N * kGKT * 2);  // one box pair
  const int tid = threadIdx.x, warp = tid / 32;
  const int64_t K = min((int64_t)*G.count, G.capacity);
  const int64_t T = (K + kDwKT - 1) / kDwKT;
  const int64_t per = (T + gx - 1) / gx;
  const int64_t t0 = (int64_t)bx * per, nt = max((int64_t)0, min(per, T - t0));
  if (nt == 0) return;
  if (tid == 0) {
    for (int q = 0; q < kDwStages; ++q) {
      tc::bar_init(&full[q], 1);
      tc::bar_init(&empty[q], 1);
    }
    tc::bar_init(&done, 1);
    tc::bar_fence_init();
  }
  if (warp == 2) tc::tmem_alloc<128>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t sbase = tc::smem_u32(smem);
  // boxes of the stage that hold columns < roundup(K, 64) (the caller's zero-padded range)
  auto nbox = [&](int64_t i) {
    const int64_t k0 = (t0 + i) * kDwKT;
    return (int)min((int64_t)kDwBoxes, (K - k0 + kGKT - 1) / kGKT);
  };
  if (tid == 0) {
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % kDwStages);
      if (i >= kDwStages) tc::bar_wait(&empty[st], (uint32_t)(((i / kDwStages) - 1) & 1));
      const int nb = nbox(i);
      bar_expect_tx(&full[st], tx * (uint32_t)nb);
      const int k0 = (int)((t0 + i) * kDwKT);
      const uint32_t sa = sbase + st * kStage, sb = sa + kStageA;
      for (int b = 0; b < nb; ++b) {  // K-blocked operands: block k0 / 64 + b, all rows
        tma_load_3d(sa + b * kDwBox, &P.a, 0, 0, k0 / kGKT + b, &full[st]);
        tma_load_3d(sb + b * kDwBox, &P.b, 0, 0, k0 / kGKT + b, &full[st]);
      }
    }
  } else if (tid == 32) {
    const uint32_t idesc = tc::idesc_f16(128, N);
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % kDwStages);
      tc::bar_wait(&full[st], (uint32_t)((i / kDwStages) & 1));
      tc::fence_after();
      const uint32_t sa = sbase + st * kStage, sb = sa + kStageA;
      const int nb = nbox(i);
      for (int b = 0; b < nb; ++b)
#pragma unroll
        for (int ks = 0; ks < kGKT / 16; ++ks)
          tc::mma_f16(tmem_base, sdesc_sw128(sa + b * kDwBox + ks * 32), sdesc_sw128(sb + b * kDwBox + ks * 32),
                      idesc, (i > 0 || b > 0 || ks > 0) ? 1u : 0u);
      tc::mma_commit(&empty[st]);
    }
    tc::mma_commit(&done);
  }
  tc::bar_wait(&done, 0);
  __syncwarp();
  tc::fence_after();
  const int row = warp * 32 + (tid & 31);
#pragma unroll 1
  for (int c0 = 0; c0 < N; c0 += 32) {  // warp-uniform: tcgen05.ld is warp-collective
    float v[32];
    tc::tmem_ld32(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    if (row < P.m) {
      float* dst = P.C + (int64_t)row * P.ldc + c0;
      const int nc = min(32, P.n - c0);
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < nc) atomicAdd(dst + c, v[c]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_free<128>(tmem_base);
}

// ---------------------------------------------------------------- step control on the device
// Masked / depth-valid ray counts of every key frame of the step: one CTA per frame
// (frame f's rays at f * stride); counts (F, 4) = [n_m human, n_d human, n_m object,
// n_d object]. Exact integer sums, written (no accumulation: no reset needed).
__global__ void __launch_bounds__(1024) train_counts_kernel(const uint8_t* __restrict__ mask_h,
                                                            const uint8_t* __restrict__ mask_o,
                                                            const float* __restrict__ depth, int64_t n_rays,
                                                            int64_t stride, int* __restrict__ counts) {
  const int64_t base = (int64_t)blockIdx.x * stride;
  int c[4] = {0, 0, 0, 0};
  for (int64_t i = threadIdx.x; i < n_rays; i += blockDim.x) {
    const bool h = mask_h[base + i] != 0, o = mask_o[base + i] != 0, d = depth[base + i] > 0.f;
    c[0] += h;
    c[1] += h && d;
    c[2] += o;
    c[3] += o && d;
  }
  __shared__ int red[32][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    for (int o = 16; o > 0; o >>= 1) c[q] += __shfl_xor_sync(0xffffffffu, c[q], o);
  if ((threadIdx.x & 31) == 0)
    for (int q = 0; q < 4; ++q) red[threadIdx.x / 32][q] = c[q];
  __syncthreads();
  if (threadIdx.x < 4) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += red[w][threadIdx.x];
    counts[blockIdx.x * 4 + threadIdx.x] = t;
  }
}

// Per-step normalisers from the (rank-summed) counts: norms (2 fields, F, 3) =
// [1/max(n_m,1), 1/max(n_d,1), loss scale]; the loss scale of a field is the power of
// two 2^floor(log2(min over its frames with n_m > 0 of n_m)) (the per-sample
// gradients of the 1/n-normalised loss are O(1/n): scaled they sit inside the fp16
// range of the backward operands); adam_scale[q] = 1 / (F * scale_q) divides it and
// the mean over frames out; stats (2 fields x 2) zeroed; ++step (Adam's bias
// correction). One thread per field.
__global__ void train_norms_kernel(const int* __restrict__ counts, int n_frames, float* __restrict__ norms,
                                   float* __restrict__ adam_scale, float* __restrict__ stats, int* __restrict__ step,
                                   uint64_t* __restrict__ seed) {
  const int q = threadIdx.x;
  if (q >= 2) return;
  int mn = 0;
  for (int f = 0; f < n_frames; ++f) {
    const int m = counts[f * 4 + 2 * q];
    if (m > 0 && (mn == 0 || m < mn)) mn = m;
  }
  const float scale = mn > 0 ? ldexpf(1.0f, 31 - __clz(mn)) : 1.0f;
  for (int f = 0; f < n_frames; ++f) {
    const int m = counts[f * 4 + 2 * q], d = counts[f * 4 + 2 * q + 1];
    float* o = norms + ((int64_t)q * n_frames + f) * 4;
    o[0] = 1.0f / (float)max(m, 1);
    o[1] = 1.0f / (float)max(d, 1);
    o[2] = scale;
    o[3] = 1.0f / (float)n_frames;  // the reported losses: mean over frames
  }
  adam_scale[q] = 1.0f / ((float)n_frames * scale);
  stats[2 * q] = 0.f;
  stats[2 * q + 1] = 0.f;
  __syncwarp(0x3u);
  if (q == 0) {
    const int st = *step + 1;
    *step = st;
    if (seed) *seed = (uint64_t)st * 0x9E3779B97F4A7C15ull;  // the step's sampling seed offset
  }
}

// dW of DeformNet layer 1 from the GEMM over [features | 1] (tmp (rows, ldt), columns
// 0..n_x-1 the feature part, column n_x = sum_s dpre1): G[:, :n_x] += tmp[:, :n_x],
// G[:, n_x + j] += tmp[:, n_x] * theta[j] (theta is the same for every sample of the
// frame); tmp is zeroed for the next frame.
__global__ void dw_pose_cols_kernel(float* __restrict__ tmp, int rows, int ldt, int n_x,
                                    const float* __restrict__ theta, int n_theta, float* __restrict__ G, int ldg) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const float cs = tmp[(int64_t)r * ldt + n_x];
  for (int c = threadIdx.x; c < n_x + n_theta; c += blockDim.x)
    G[(int64_t)r * ldg + c] += c < n_x ? tmp[(int64_t)r * ldt + c] : cs * theta[c - n_x];
  __syncthreads();
  for (int c = threadIdx.x; c <= n_x; c += blockDim.x) tmp[(int64_t)r * ldt + c] = 0.f;
}

// Multi-tensor Adam: every trained tensor of the step in one launch (blockIdx.y =
// tensor). Bias corrections from the device step counter, the gradient scale from
// the device (cf_train_norms), grads zeroed after use (the next step accumulates
// into them), optional fp16 copy of the updated parameters.
constexpr int kMaxAdam = 24;
struct AdamT {
  float* p;
  float* g;
  float* m;
  float* v;
  __half* p16;
  int64_t n;
  float lr;
  int scale_idx;
};
struct AdamGroup {
  AdamT t[kMaxAdam];
  const int* step;
  const float* scale;
  float b1, b2, eps;
};

__global__ void adam_multi_kernel(const __grid_constant__ AdamGroup A) {
  const AdamT& T = A.t[blockIdx.y];
  const int step = *A.step;
  const float c1 = 1.0f / (1.0f - powf(A.b1, (float)step)), c2 = 1.0f / (1.0f - powf(A.b2, (float)step));
  const float gs = A.scale ? A.scale[T.scale_idx] : 1.0f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T.n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = T.g[i] * gs;
    const float mi = A.b1 * T.m[i] + (1.f - A.b1) * gi;
    const float vi = A.b2 * T.v[i] + (1.f - A.b2) * gi * gi;
    T.m[i] = mi;
    T.v[i] = vi;
    T.g[i] = 0.f;
    const float p = T.p[i] - T.lr * (mi * c1) / (sqrtf(vi * c2) + A.eps);
    T.p[i] = p;
    if (T.p16) T.p16[i] = __float2half_rn(p);
  }
}

// Multi-matrix fp32 -> fp16 UMMA canonical repack (forward blobs with their split
// residual, transposed blobs of the backward) in one launch (blockIdx.y = item).
// Packed matrix P (rows x cols, padded to 16): P[r][c] = W[r][col0 + c] or, when
// transposed, W[c][col0 + r] (W row stride ldw).
constexpr int kMaxPack = 32;
struct PackItem {
  const float* w;
  uint8_t* blob;
  uint8_t* blob_lo;
  int rows, cols, ldw, col0, transpose;
};
struct PackGroup {
  PackItem it[kMaxPack];
};

__global__ void pack_multi_kernel(const __grid_constant__ PackGroup G) {
  const PackItem& I = G.it[blockIdx.y];
  const int rp = (I.rows + 15) / 16 * 16, cp = (I.cols + 15) / 16 * 16;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rp * cp; e += gridDim.x * blockDim.x) {
    const int r = e / cp, c = e % cp;
    float x = 0.0f;
    if (r < I.rows && c < I.cols)
      x = I.transpose ? I.w[(int64_t)c * I.ldw + I.col0 + r] : I.w[(int64_t)r * I.ldw + I.col0 + c];
    const __half h = __float2half_rn(x);
    *reinterpret_cast<__half*>(I.blob + tc::core_offset(r, c, cp)) = h;
    if (I.blob_lo) *reinterpret_cast<__half*>(I.blob_lo + tc::core_offset(r, c, cp)) = __float2half_rn(x - __half2float(h));
  }
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

// rows x K fp16, row stride ld elements; boxes of 64 halves (128 B) x box_rows (default
// rows; more than rows = zero-filled), 128B swizzle
bool make_map(CUtensorMap* map, const void* base, int rows, int64_t K, int64_t ld, int box_rows = 0) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)(box_rows > 0 ? box_rows : rows)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the K-blocked operand of cf_dw_grouped: a (rows_stored, K) fp16 matrix as K / 64
// blocks of (rows_stored, 64); the map exposes its first `rows` rows (rows beyond them,
// up to the box, read as zeros) and a box of 64 x box_rows x 1 block, 128-byte swizzle
bool make_map_kb(CUtensorMap* map, const void* base, int rows, int64_t rows_stored, int64_t K, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
  const cuuint64_t strides[2] = {128, (cuuint64_t)rows_stored * 128};
  const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
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

int cf_dw_grouped(const cf_dw_problem* probs, int n, const int* count, int64_t capacity, void* stream) {
  if (!probs || n < 1 || n > kMaxDw || !count || capacity < 0)
    return cf::fail(CF_E_BAD_ARG, "cf_dw_grouped: bad args (1..10 problems, count, capacity)");
  if (capacity == 0) return CF_OK;
  if (capacity >= (int64_t)1 << 31 || capacity % 64 != 0)
    return cf::fail(CF_E_BAD_ARG, "cf_dw_grouped: capacity must be a multiple of 64 below 2^31");
  DwGroup G{};
  G.count = count;
  G.capacity = capacity;
  for (int i = 0; i < n; ++i) {
    const cf_dw_problem& q = probs[i];
    if (!q.A || !q.B || !q.C || q.m < 1 || q.m > 128 || q.n < 1 || q.n > 128 || q.a_rows < q.m ||
        q.b_rows < q.n || q.ldc < q.n)
      return cf::fail(CF_E_BAD_ARG, "cf_dw_grouped: problem shape (m, n in 1..128, a_rows >= m, b_rows >= n)");
    if ((reinterpret_cast<uintptr_t>(q.A) | reinterpret_cast<uintptr_t>(q.B)) % 16 != 0)
      return cf::fail(CF_E_BAD_ARG, "cf_dw_grouped: operands need 16-byte alignment");
    DwProb& P = G.p[i];
    P.n_mma = (q.n + 15) / 16 * 16;
    if (!make_map_kb(&P.a, q.A, q.m, q.a_rows, capacity, 128) || !make_map_kb(&P.b, q.B, q.n, q.b_rows, capacity, P.n_mma))
      return cf::fail(CF_E_CUDA, "cf_dw_grouped: cuTensorMapEncodeTiled failed");
    P.C = q.C;
    P.ldc = q.ldc;
    P.m = q.m;
    P.n = q.n;
  }
  // two waves of one CTA per SM split between the problems in proportion to the rows
  // each streams (+ a share for the setup and epilogue), instead of a wave per problem:
  // fewer ramps and atomic epilogues (1 wave: 32.6, 2: 31.5, 3: 31.8, 4: 31.6, a wave
  // per problem: 32.6 ms per training step)
  const int64_t T = (capacity + kDwKT - 1) / kDwKT;
  const int total = (int)std::max<int64_t>(n, std::min<int64_t>(T * n, 2 * (int64_t)cf::sm_count()));
  double wsum = 0.0, w[kMaxDw];
  for (int i = 0; i < n; ++i) wsum += (w[i] = probs[i].m + probs[i].n + 32.0);
  G.cta0[0] = 0;
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += w[i];
    const int end = std::max(G.cta0[i] + 1, (int)std::lround(total * acc / wsum));
    G.cta0[i + 1] = std::min(end, total - (n - 1 - i));
  }
  for (int i = n + 1; i <= kMaxDw; ++i) G.cta0[i] = G.cta0[n];
  const int smem = kDwStages * 2 * kDwBoxes * kDwBox;
  CF_CHECK_CUDA(cudaFuncSetAttribute(dw_grouped_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dw_grouped_kernel<<<(unsigned)G.cta0[n], 128, smem, cf::as_stream(stream)>>>(G);
  return cf::check_launch("cf_dw_grouped");
}

int cf_train_counts(const uint8_t* mask_h, const uint8_t* mask_o, const float* gt_depth, int64_t n_rays,
                    int n_frames, int64_t frame_stride, int* counts, void* stream) {
  if (!mask_h || !mask_o || !gt_depth || !counts || n_rays < 0 || n_frames < 1 || frame_stride < n_rays)
    return cf::fail(CF_E_BAD_ARG, "cf_train_counts: bad args");
  train_counts_kernel<<<n_frames, 1024, 0, cf::as_stream(stream)>>>(mask_h, mask_o, gt_depth, n_rays, frame_stride,
                                                                   counts);
  return cf::check_launch("cf_train_counts");
}

int cf_train_norms(const int* counts, int n_frames, float* norms, float* adam_scale, float* stats, int* step,
                   uint64_t* seed, void* stream) {
  if (!counts || n_frames < 1 || !norms || !adam_scale || !stats || !step)
    return cf::fail(CF_E_BAD_ARG, "cf_train_norms: bad args");
  train_norms_kernel<<<1, 32, 0, cf::as_stream(stream)>>>(counts, n_frames, norms, adam_scale, stats, step, seed);
  return cf::check_launch("cf_train_norms");
}

int cf_dw_pose_cols(float* tmp, int rows, int ldt, int n_x, const float* theta, int n_theta, float* G, int ldg,
                    void* stream) {
  if (!tmp || !theta || !G || rows < 1 || n_x < 1 || ldt <= n_x || n_theta < 0 || ldg < n_x + n_theta)
    return cf::fail(CF_E_BAD_ARG, "cf_dw_pose_cols: bad args");
  dw_pose_cols_kernel<<<rows, 128, 0, cf::as_stream(stream)>>>(tmp, rows, ldt, n_x, theta, n_theta, G, ldg);
  return cf::check_launch("cf_dw_pose_cols");
}

int cf_adam_multi(const cf_adam_tensor* ts, int n, float beta1, float beta2, float eps, const int* step,
                  const float* scale, void* stream) {
  if (!ts || n < 1 || n > kMaxAdam || !step) return cf::fail(CF_E_BAD_ARG, "cf_adam_multi: bad args (1..24 tensors)");
  AdamGroup A{};
  int64_t nmax = 0;
  for (int i = 0; i < n; ++i) {
    const cf_adam_tensor& t = ts[i];
    if (!t.p || !t.g || !t.m || !t.v || t.n < 0 || (scale && t.scale_idx < 0))
      return cf::fail(CF_E_BAD_ARG, "cf_adam_multi: bad tensor");
    A.t[i] = AdamT{t.p, t.g, t.m, t.v, reinterpret_cast<__half*>(t.p16), t.n, t.lr, t.scale_idx};
    nmax = std::max(nmax, t.n);
  }
  A.step = step;
  A.scale = scale;
  A.b1 = beta1;
  A.b2 = beta2;
  A.eps = eps;
  if (nmax == 0) return CF_OK;
  const unsigned gx = (unsigned)std::min<int64_t>((nmax + 255) / 256, (int64_t)cf::sm_count() * 8);
  adam_multi_kernel<<<dim3(gx, (unsigned)n), 256, 0, cf::as_stream(stream)>>>(A);
  return cf::check_launch("cf_adam_multi");
}

int cf_pack_multi(const cf_pack_item* items, int n, void* stream) {
  if (!items || n < 1 || n > kMaxPack) return cf::fail(CF_E_BAD_ARG, "cf_pack_multi: bad args (1..32 items)");
  PackGroup G{};
  int emax = 0;
  for (int i = 0; i < n; ++i) {
    const cf_pack_item& q = items[i];
    if (!q.w || !q.blob || q.rows < 1 || q.cols < 1 || q.col0 < 0 ||
        (q.transpose ? q.ldw < q.col0 + q.rows : q.ldw < q.col0 + q.cols))
      return cf::fail(CF_E_BAD_ARG, "cf_pack_multi: bad item");
    G.it[i] = PackItem{q.w, q.blob, q.blob_lo, q.rows, q.cols, q.ldw, q.col0, q.transpose};
    emax = std::max(emax, (q.rows + 15) / 16 * 16 * ((q.cols + 15) / 16 * 16));
  }
  pack_multi_kernel<<<dim3((unsigned)((emax + 255) / 256), (unsigned)n), 256, 0, cf::as_stream(stream)>>>(G);
  return cf::check_launch("cf_pack_multi");
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
