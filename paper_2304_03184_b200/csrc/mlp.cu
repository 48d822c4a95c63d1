// Fused tiny-MLP chain on the 5th-gen tensor cores (tcgen05, kind::f16,
// fp16 operands, fp32 accumulation in TMEM). One persistent CTA per SM with two
// independent 128-sample "slots" (4 warps each): while one slot runs its
// epilogue (TMEM -> registers -> ReLU -> fp16 -> smem), the other slot's MMAs
// run, so the tensor pipe and the CUDA cores overlap. All layer weights stay
// resident in shared memory for the kernel's lifetime; activations never leave
// the SM between layers.
//
// cf_mlp_forward is the generic entry (SPEC FieldNetworks / DeformNet,
// SPEC.md:349-356): y = L_n(relu(... relu(L_1(x)))), biases optional, no output
// activation; the field kernels in field.cu reuse the same layer step.
#include <vector>

#include "common.cuh"
#include "tc.cuh"

namespace {

constexpr int kMaxLayers = 8;
constexpr int kSlotThreads = 128;
constexpr int kSlots = 2;
constexpr int kMaxWidth = 128;

struct ChainDesc {
  int n_layers;
  int k[kMaxLayers];    // input width of layer l (multiple of 16)
  int n[kMaxLayers];    // output width (multiple of 16, <= 128)
  int w_off[kMaxLayers];  // byte offset of layer l in the packed weight blob
  int b_off[kMaxLayers];  // float offset of the bias (or -1)
  int w_bytes;
  int k0_real;          // real input width (<= k[0]), rest zero-padded
  int out_cols;         // columns written per sample (<= n[last])
};

__global__ void __launch_bounds__(kSlots* kSlotThreads, 1)
    mlp_chain_kernel(ChainDesc D, const uint8_t* __restrict__ wblob, const float* __restrict__ bias,
                     const float* __restrict__ x, int64_t n_rows, float* __restrict__ y) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* w_s = smem;                                          // weights
  uint8_t* a_s = smem + ((D.w_bytes + 1023) / 1024) * 1024;      // kSlots x (128 x 128 fp16)
  __shared__ uint64_t mbar[kSlots];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x;
  const int slot = tid / kSlotThreads;
  const int r = tid % kSlotThreads;  // row of this thread within the tile == TMEM lane
  const int warp = tid / 32;

  // stage weights (once per CTA)
  for (int i = tid * 16; i < D.w_bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(w_s + i) = *reinterpret_cast<const uint4*>(wblob + i);
  if (tid == 0) {
    for (int s = 0; s < kSlots; ++s) tc::bar_init(&mbar[s], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<kSlots * kMaxWidth>(&tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  uint8_t* abuf = a_s + slot * (128 * kMaxWidth * 2);
  // lane quarter of this warp: (warp % 4) * 32, column block of this slot
  const uint32_t tmem_slot = tmem_base + (uint32_t)(slot * kMaxWidth);
  const uint32_t tmem_row = tmem_slot + ((uint32_t)((warp % 4) * 32) << 16);
  uint32_t phase = 0;
  const int64_t n_tiles = (n_rows + 127) / 128;

  for (int64_t tile = (int64_t)blockIdx.x * kSlots + slot; tile < n_tiles; tile += (int64_t)gridDim.x * kSlots) {
    const int64_t row = tile * 128 + r;
    const bool live = row < n_rows;
    // layer-0 input -> fp16 canonical buffer
    for (int k0 = 0; k0 < D.k[0]; k0 += 8) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = k0 + i;
        v[i] = (live && k < D.k0_real) ? x[row * D.k0_real + k] : 0.0f;
      }
      tc::st_row8(abuf, r, k0, D.k[0], v);
    }
    for (int l = 0; l < D.n_layers; ++l) {
      tc::fence_async_smem();
      tc::fence_before();
      tc::named_sync(1 + slot, kSlotThreads);
      if (r < 32) {  // the slot's first warp issues
        tc::fence_after();
        tc::layer_ss_warp(tmem_slot, abuf, w_s + D.w_off[l], D.k[l], D.n[l], &mbar[slot]);
      }
      tc::bar_wait(&mbar[slot], phase);
      phase ^= 1u;
      tc::fence_after();
      const bool last = (l == D.n_layers - 1);
      const float* b = D.b_off[l] >= 0 ? bias + D.b_off[l] : nullptr;
      for (int c0 = 0; c0 < D.n[l]; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem_row + (uint32_t)c0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (b) v[i] += b[c0 + i];
          if (!last) v[i] = fmaxf(v[i], 0.0f);
        }
        if (last) {
          if (live)
            for (int i = 0; i < 16; ++i)
              if (c0 + i < D.out_cols) y[row * D.out_cols + c0 + i] = v[i];
        } else {
          tc::st_row8(abuf, r, c0, D.n[l], v);
          tc::st_row8(abuf, r, c0 + 8, D.n[l], v + 8);
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<kSlots * kMaxWidth>(tmem_base);
}

}  // namespace

extern "C" {

// layers: widths[0..n_layers] (widths[0] = input width, real), weights fp16
// packed per layer in the canonical layout (see tc.cuh) with K padded to 16 and
// N padded to 16; biases fp32 (n_layers x 128, row l used if has_bias[l]).
int cf_mlp_forward(int n_layers, const int* widths, const uint8_t* wblob_dev, int w_bytes, const float* bias_dev,
                   const int* has_bias, const float* x, int64_t n_rows, float* y, void* stream) {
  if (n_layers < 1 || n_layers > kMaxLayers || !widths) return cf::fail(CF_E_BAD_ARG, "cf_mlp_forward: bad layers");
  ChainDesc D{};
  D.n_layers = n_layers;
  int off = 0;
  for (int l = 0; l < n_layers; ++l) {
    const int kin = (widths[l] + 15) / 16 * 16;
    const int nout = (widths[l + 1] + 15) / 16 * 16;
    if (kin > kMaxWidth || nout > kMaxWidth) return cf::fail(CF_E_BAD_ARG, "cf_mlp_forward: width > 128");
    D.k[l] = kin;
    D.n[l] = nout;
    D.w_off[l] = off;
    D.b_off[l] = (has_bias && has_bias[l]) ? l * kMaxWidth : -1;
    off += kin * nout * 2;
  }
  if (off != w_bytes) return cf::fail(CF_E_BAD_ARG, "cf_mlp_forward: weight blob size mismatch");
  D.w_bytes = w_bytes;
  D.k0_real = widths[0];
  D.out_cols = widths[n_layers];
  const int smem = ((w_bytes + 1023) / 1024) * 1024 + kSlots * 128 * kMaxWidth * 2;
  if (smem > 227 * 1024) return cf::fail(CF_E_BAD_ARG, "cf_mlp_forward: weights exceed shared memory");
  if (n_rows == 0) return CF_OK;
  CF_CHECK_CUDA(cudaFuncSetAttribute(mlp_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int64_t tiles = (n_rows + 127) / 128;
  int64_t grid = (tiles + kSlots - 1) / kSlots;
  if (grid > cf::sm_count()) grid = cf::sm_count();
  mlp_chain_kernel<<<(unsigned)grid, kSlots * kSlotThreads, smem, cf::as_stream(stream)>>>(D, wblob_dev, bias_dev, x,
                                                                                           n_rows, y);
  return cf::check_launch("cf_mlp_forward");
}

}  // extern "C"
