// Radiance-field evaluation of compacted samples, as a chain of
// stage kernels sized for what bounds each stage on B200:
//
//   hash_f16_kernel   CUDA cores, L2 gathers. Thread per sample at full
//                     occupancy (latency hiding needs many warps; ncu showed
//                     the fused variant stalled 55% on long-scoreboard gathers
//                     with 8 warps/SM); 8*CH corner loads in flight per thread.
//                     Writes 32 fp16 features (64 B) per sample.
//   deform_mlp_kernel tcgen05: DeformNet 32->128x4->3 (theta folded into the
//                     layer-1 bias), 3 slots x 128 samples per persistent CTA,
//                     weights (108 KB fp16) resident in smem, accumulators and
//                     (2 slots) activations in TMEM (TS-form MMAs).
//                     Epilogue: dv = 0.05 tanh(.), xc = x + dv / side.
//   color_mlp_kernel  tcgen05 TS form: E_g 32->64->16 (sigma = exp, 15 geo) and
//                     E_c [geo, SH4(dir)] 32->64->64->3 (sigmoid), 5 slots.
//
// Human:  hash_d(xu) -> deform_mlp -> hash_c(xc) -> color_mlp
// Object: hash_c(xu) -> color_mlp
// Between stages only 64 B/sample (features) or 16 B/sample (xc) touch HBM.
#include "common.cuh"
#include "tc.cuh"
#include <algorithm>

namespace {

constexpr int kSlotThreads = 128;

// ------------------------------------------------------------------ hash stage

// Hash features of L levels, CH levels at a time: all 8*CH corner gathers of a
// chunk are issued before any is consumed. Same arithmetic as hashgrid.cu.
// load one table entry (F values, fp32 or fp16) as fp32
template <int F>
__device__ __forceinline__ void ld_entry(const float* __restrict__ base, uint32_t idx, float* v) {
  if constexpr (F == 2) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(base) + idx);
    v[0] = f.x;
    v[1] = f.y;
  } else {
    const float4 f = __ldg(reinterpret_cast<const float4*>(base) + idx);
    v[0] = f.x;
    v[1] = f.y;
    v[2] = f.z;
    v[3] = f.w;
  }
}
template <int F>
__device__ __forceinline__ void ld_entry(const __half* __restrict__ base, uint32_t idx, float* v) {
  if constexpr (F == 2) {
    const float2 f = __half22float2(__ldg(reinterpret_cast<const __half2*>(base) + idx));
    v[0] = f.x;
    v[1] = f.y;
  } else {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(base) + idx);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  }
}

// table: (entries, F) row-major, fp32 or fp16 (TT); interpolation in fp32.
// Measured: the deformation grid (F = 4) reads its fp16 copy (16 -> 8 B gathers:
// 39 -> 28 us); the canonical grid (F = 2) stays fp32, where the two extra
// conversions per corner outweighed the halved bytes (45 -> 59 us).
template <int F, int L, int CH, class TT>
__device__ __forceinline__ void hash_features(const cf_hashgrid_desc& D, const TT* __restrict__ table, float x,
                                              float y, float z, float* feat, int l_base = 0) {
  static_assert(L % CH == 0, "chunk must divide the level count");
  x = fminf(fmaxf(x, 0.0f), 1.0f);
  y = fminf(fmaxf(y, 0.0f), 1.0f);
  z = fminf(fmaxf(z, 0.0f), 1.0f);
  const uint32_t mask = (1u << D.log2_table) - 1u;
#pragma unroll
  for (int l0 = 0; l0 < L; l0 += CH) {
    float t[CH][8][F];
    float w[CH][8];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int l = l_base + l0 + c;
      const int N = D.resolution[l];
      const float s = (float)N;
      const float pos[3] = {f_mul(x, s), f_mul(y, s), f_mul(z, s)};
      uint32_t g[3];
      float fr[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int gi = (int)floorf(pos[a]);
        gi = gi > N - 1 ? N - 1 : gi;
        g[a] = (uint32_t)gi;
        fr[a] = f_sub(pos[a], (float)gi);
      }
      const uint32_t stride = (uint32_t)N + 1u;
      const bool dense = D.dense[l] != 0;
      const TT* base = table + D.offset[l] * F;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t cx = g[0] + (k & 1), cy = g[1] + ((k >> 1) & 1), cz = g[2] + ((k >> 2) & 1);
        const uint32_t idx = dense ? (cx + cy * stride + cz * stride * stride)
                                   : ((cx ^ (cy * 2654435761u) ^ (cz * 805459861u)) & mask);
        ld_entry<F>(base, idx, t[c][k]);
        const float wx = (k & 1) ? fr[0] : f_sub(1.0f, fr[0]);
        const float wy = (k & 2) ? fr[1] : f_sub(1.0f, fr[1]);
        const float wz = (k & 4) ? fr[2] : f_sub(1.0f, fr[2]);
        w[c][k] = f_mul(f_mul(wx, wy), wz);
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int f = 0; f < F; ++f) {
        float acc = f_mul(w[c][0], t[c][0][f]);
#pragma unroll
        for (int k = 1; k < 8; ++k) acc = f_add(acc, f_mul(w[c][k], t[c][k][f]));
        feat[(l0 + c) * F + f] = acc;
      }
  }
}

// 32 features of a valid sample (flag > 0) -> fp16 row; invalid -> zeros
// SPLIT threads per sample, each doing L / SPLIT consecutive levels and writing
// its 32 / SPLIT features of the row: SPLIT > 1 multiplies the warps in flight
// for small sample counts (the object field), where one thread per sample left
// the SMs mostly idle.
// F32 ("fp32" precision mode): the 32 features are written as fp32 (128 B / sample)
// instead of fp16.
template <int F, int L, int CH, int SPLIT, class TT, bool F32 = false>
__global__ void __launch_bounds__(128) hash_f16_kernel(cf_hashgrid_desc D, const TT* __restrict__ table,
                                                       const float4* __restrict__ x, const int* __restrict__ count,
                                                       int64_t capacity, uint4* __restrict__ out) {
  constexpr int LS = L / SPLIT, NF = LS * F;  // levels and features per thread
  static_assert(L % SPLIT == 0 && NF % 8 == 0, "whole 16-byte chunks per thread");
  pdl_wait();
  const int64_t n = min((int64_t)*count, capacity) * SPLIT;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = SPLIT == 1 ? t : t / SPLIT;
    const int part = SPLIT == 1 ? 0 : (int)(t % SPLIT);
    const float4 p = x[s];
    float feat[NF];
    if (p.w > 0.0f) {
      if constexpr (SPLIT == 1)
        hash_features<F, LS, CH, TT>(D, table, p.x, p.y, p.z, feat);
      else
        hash_features<F, LS, (CH < LS ? CH : LS), TT>(D, table, p.x, p.y, p.z, feat, part * LS);
    } else {
#pragma unroll
      for (int i = 0; i < NF; ++i) feat[i] = 0.0f;
    }
    if constexpr (F32) {
      float4* o = reinterpret_cast<float4*>(out) + s * 8 + part * (NF / 4);
#pragma unroll
      for (int q = 0; q < NF / 4; ++q)
        o[q] = make_float4(feat[4 * q], feat[4 * q + 1], feat[4 * q + 2], feat[4 * q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < NF / 8; ++q) {
        __half2 h[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(feat[8 * q + 2 * i], feat[8 * q + 2 * i + 1]);
        out[s * 4 + part * (NF / 8) + q] = *reinterpret_cast<uint4*>(h);
      }
    }
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ MLP slots

struct Slot {
  uint8_t* abuf;
  const uint8_t* w_s;
  uint64_t* bar;
  uint32_t tmem;      // slot column base (lane 0)
  uint32_t tmem_row;  // + this warp's lane quarter
  uint32_t phase;
  int slot, r;
};

// issue one layer from the slot's A buffer and wait until its accumulator is in TMEM
__device__ __forceinline__ void run_layer(Slot& S, int w_off, int K, int N) {
  tc::fence_async_smem();
  tc::fence_before();
  tc::named_sync(1 + S.slot, kSlotThreads);
  if (S.r < 32) {  // the slot's first warp issues (tc::layer_ss_warp)
    tc::fence_after();
    tc::layer_ss_warp(S.tmem, S.abuf, S.w_s + w_off, K, N, S.bar);
  }
  tc::bar_wait(S.bar, S.phase);
  S.phase ^= 1u;
  tc::fence_after();
}

// hidden-layer epilogue: (+bias) ReLU -> fp16 -> A buffer with K = N
template <int N>
__device__ __forceinline__ void relu_to_abuf(Slot& S, const float* bias) {
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(S.tmem_row + (uint32_t)c0, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = fmaxf(bias ? v[i] + bias[c0 + i] : v[i], 0.0f);
#pragma unroll
    for (int q = 0; q < 4; ++q) tc::st_row8(S.abuf, S.r, c0 + 8 * q, N, v + 8 * q);
  }
}

// copy one 64-byte fp16 feature row into the A buffer (K = 32)

template <int SLOTS, int TMEM_COLS>
__device__ __forceinline__ void slots_setup(const uint8_t* __restrict__ wblob, int w_bytes, uint8_t* smem,
                                            uint64_t* mbar, uint32_t* tmem_base) {
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid * 16; i < w_bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = *reinterpret_cast<const uint4*>(wblob + i);
  if (tid == 0) {
    for (int s = 0; s < SLOTS; ++s) tc::bar_init(&mbar[s], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<TMEM_COLS>(tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}

template <int SLOTS, int COLS, int ABYTES>
__device__ __forceinline__ Slot make_slot(uint8_t* smem, int w_bytes, uint64_t* mbar, uint32_t tmem_base) {
  Slot S;
  const int tid = threadIdx.x;
  S.slot = tid / kSlotThreads;
  S.r = tid % kSlotThreads;
  S.w_s = smem;
  S.abuf = smem + ((w_bytes + 1023) / 1024) * 1024 + S.slot * ABYTES;
  S.bar = &mbar[S.slot];
  S.tmem = tmem_base + (uint32_t)(S.slot * COLS);
  S.tmem_row = S.tmem + ((uint32_t)(((tid / 32) % 4) * 32) << 16);
  S.phase = 0;
  return S;
}

// ---------------------------------------------------------------- DeformNet

// Each layer is MMA -> epilogue -> MMA per 128-sample slot, so the tensor pipe
// is busy only while some slot is in its MMA phase: the kernel runs as many
// slots as TMEM allows. Two slots keep their activations in TMEM and use the
// "TS" MMA form (A from TMEM, weights B from smem): D (128 fp32 columns) +
// A (64 packed fp16x2 columns) each. The third slot's D takes the remaining 128
// columns and its A lives in shared memory (SS form) — 512 columns in all.
// 8 warps per slot: warps w and w+4 share a TMEM lane quarter and split the
// columns; the epilogue is tcgen05.ld -> (+bias) -> cvt.relu.f16x2 ->
// tcgen05.st (TS) or st.shared in the canonical layout (SS).
constexpr int kDeformSlots = 3;
constexpr int kDeformSlotThreads = 256;
constexpr int kDeformW = (128 * 32 + 3 * 128 * 128 + 16 * 128) * 2;  // 110,592 B
constexpr int kDeformA = 128 * 128 * 2;                              // SS slot's A buffer

struct TsSlot {
  uint64_t* bar;
  uint8_t* abuf;   // SS slot: A in smem (nullptr for TS slots)
  uint32_t d;      // D columns (+ lane quarter)
  uint32_t a;      // TS: A columns (+ lane quarter)
  uint32_t d0, a0; // slot base columns (MMA operands)
  uint32_t phase;
  int slot, r, half;
};

// one layer: the slot's A writes are complete and visible -> one thread issues
// the MMAs -> all wait for the commit
__device__ __forceinline__ void ts_layer(TsSlot& S, const uint8_t* w, int K, int N) {
  if (S.abuf) tc::fence_async_smem();
  else tc::tmem_wait_st();
  tc::fence_before();
  tc::named_sync(1 + S.slot, kDeformSlotThreads);
  if (threadIdx.x % kDeformSlotThreads < 32) {  // the slot's first warp issues
    tc::fence_after();
    if (S.abuf) tc::layer_ss_warp(S.d0, S.abuf, w, K, N, S.bar);
    else tc::layer_ts_warp(S.d0, S.a0, w, K, N, S.bar);
  }
  tc::bar_wait(S.bar, S.phase);
  S.phase ^= 1u;
  tc::fence_after();
}

// The training saves (the dW GEMMs' operands) are K-blocked feature-major: a (rows, S)
// fp16 matrix stored as S / 64 blocks of (rows, 64), element (c, s) at
// kb_col(s, rows) + 64 c — one dW TMA box (64 samples x the operand's rows) is then one
// contiguous run of HBM instead of a 128-byte piece of every feature row.
__device__ __forceinline__ int64_t kb_col(int64_t s, int rows) { return (s >> 6) * rows * 64 + (s & 63); }
constexpr int64_t kKbLd = 64;  // column stride inside a block

// Store this thread's 32 fp16 values (16 packed pairs, columns col .. col+31) into a
// column-major (feature-major) matrix: column c of the sample at dst[c * ld]. Lanes
// are consecutive samples, so every store is a coalesced 64-byte warp segment.
__device__ __forceinline__ void store_cols_f16(uint16_t* dst, int64_t ld, int col, const uint32_t* h) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    dst[(int64_t)(col + 2 * i) * ld] = (uint16_t)(h[i] & 0xffffu);
    dst[(int64_t)(col + 2 * i + 1) * ld] = (uint16_t)(h[i] >> 16);
  }
}

// 16 fp16 values (8 packed pairs) of sample s as columns col .. col+15 of a
// feature-major block (column c at dst[c * ld + s])
__device__ __forceinline__ void store_cols16_f16(uint16_t* dst, int64_t ld, int64_t s, int col, const uint32_t* h) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    dst[(int64_t)(col + 2 * i) * ld + s] = (uint16_t)(h[i] & 0xffffu);
    dst[(int64_t)(col + 2 * i + 1) * ld + s] = (uint16_t)(h[i] >> 16);
  }
}

// hidden epilogue of a 128-wide layer: this warp's 64 columns -> (+bias) ReLU -> fp16 -> A
__device__ __forceinline__ void ts_relu128(const TsSlot& S, const float* bias) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int col = 64 * S.half + 32 * c;
    uint32_t r[32];
    tc::tmem_ld32_nowait(S.d + (uint32_t)col, r);
    tc::tmem_wait_ld();
    uint32_t h[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float x0 = __uint_as_float(r[2 * i]), x1 = __uint_as_float(r[2 * i + 1]);
      if (bias) {
        x0 += bias[col + 2 * i];
        x1 += bias[col + 2 * i + 1];
      }
      h[i] = tc::relu_f16x2(x0, x1);
    }
    if (S.abuf) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(S.abuf + tc::core_offset(S.r, col + 8 * q, 128)) =
            make_uint4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
    } else {
      tc::tmem_st16(S.a + (uint32_t)(col / 2), h);
    }
  }
}

// the fp16-mode render forward (the training forward is deform_mlp_prec_kernel<true>)
__global__ void __launch_bounds__(kDeformSlots* kDeformSlotThreads, 1)
    deform_mlp_kernel(const uint8_t* __restrict__ wblob, const float* __restrict__ bias1, float delta_scale,
                      float inv_side, const float4* __restrict__ xu, const uint4* __restrict__ dfeat,
                      const int* __restrict__ count, int64_t capacity, float4* __restrict__ xc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kDeformSlots];
  __shared__ uint32_t tmem_base;
  __shared__ float s_bias[128];
  const int tid = threadIdx.x, warp = tid / 32;
  if (tid < 128) s_bias[tid] = bias1[tid];
  for (int i = tid * 16; i < kDeformW; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = *reinterpret_cast<const uint4*>(wblob + i);
  if (tid == 0) {
    for (int q = 0; q < kDeformSlots; ++q) tc::bar_init(&mbar[q], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_wait();  // weights staged and TMEM allocated while the previous kernel drained
  TsSlot S;
  S.slot = tid / kDeformSlotThreads;
  const int ws = warp % (kDeformSlotThreads / 32);  // warp within the slot
  S.half = ws / 4;                                 // column half
  S.r = (ws % 4) * 32 + (tid & 31);                // sample row = TMEM lane
  S.bar = &mbar[S.slot];
  S.phase = 0;
  const uint32_t lane_q = (uint32_t)((ws % 4) * 32) << 16;
  // TMEM columns: slot 0 D [0,128) A [128,192); slot 1 D [192,320) A [320,384); slot 2 (SS) D [384,512)
  S.d0 = tmem_base + (uint32_t)(S.slot * 192);
  S.a0 = S.d0 + 128u;
  S.abuf = S.slot == 2 ? smem + kDeformW : nullptr;
  S.d = S.d0 + lane_q;
  S.a = S.a0 + lane_q;
  constexpr int o1 = 0, o2 = 128 * 32 * 2, o3 = o2 + 128 * 128 * 2, o4 = o3 + 128 * 128 * 2, o5 = o4 + 128 * 128 * 2;
  const int64_t n = min((int64_t)*count, capacity);
  const int64_t n_tiles = (n + 127) / 128;
  const int64_t tstride = (int64_t)gridDim.x * kDeformSlots;
  // this thread's half of its row's 32 input features (2 x 16 B), prefetched one tile ahead
  int64_t tile = (int64_t)blockIdx.x * kDeformSlots + S.slot;
  uint4 nxt[2];
  {
    const int64_t s0 = tile * 128 + S.r;
#pragma unroll
    for (int q = 0; q < 2; ++q) nxt[q] = (s0 < n) ? dfeat[s0 * 4 + 2 * S.half + q] : make_uint4(0, 0, 0, 0);
  }
  for (; tile < n_tiles; tile += tstride) {
    const int64_t s = tile * 128 + S.r;
    const bool live = s < n;
    if (S.abuf) {
#pragma unroll
      for (int q = 0; q < 2; ++q)
        *reinterpret_cast<uint4*>(S.abuf + tc::core_offset(S.r, 16 * S.half + 8 * q, 32)) = nxt[q];
    } else {
      const uint32_t w8[8] = {nxt[0].x, nxt[0].y, nxt[0].z, nxt[0].w, nxt[1].x, nxt[1].y, nxt[1].z, nxt[1].w};
      tc::tmem_st8(S.a + (uint32_t)(8 * S.half), w8);
    }
    const float4 xs = (live && S.half == 0) ? xu[s] : make_float4(0.f, 0.f, 0.f, 0.f);
    ts_layer(S, smem + o1, 32, 128);
    {
      const int64_t sn = (tile + tstride) * 128 + S.r;
#pragma unroll
      for (int q = 0; q < 2; ++q) nxt[q] = (sn < n) ? dfeat[sn * 4 + 2 * S.half + q] : make_uint4(0, 0, 0, 0);
    }
    ts_relu128(S, s_bias);
    ts_layer(S, smem + o2, 128, 128);
    ts_relu128(S, nullptr);
    ts_layer(S, smem + o3, 128, 128);
    ts_relu128(S, nullptr);
    ts_layer(S, smem + o4, 128, 128);
    ts_relu128(S, nullptr);
    ts_layer(S, smem + o5, 128, 16);
    if (S.half == 0) {
      float v[16];
      tc::tmem_ld16(S.d, v);
      if (live) {
        float4 p = xs;
        if (p.w > 0.0f) {
          p.x = f_add(p.x, f_mul(delta_scale * tanhf(v[0]), inv_side));
          p.y = f_add(p.y, f_mul(delta_scale * tanhf(v[1]), inv_side));
          p.z = f_add(p.z, f_mul(delta_scale * tanhf(v[2]), inv_side));
        }
        xc[s] = p;
      }
    }
    // the next tile's first A write happens after this tile's last MMA completed
    // (ts_layer waited on its commit); its first MMA is issued only after every
    // thread of the slot passed the next barrier, i.e. finished reading this D
  }
  pdl_trigger();
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem_base);
}

// ---------------------------------------------------------------- E_g / E_c

// real spherical harmonics up to degree 3 (16 coefficients), unit direction
__device__ __forceinline__ void sh16(float x, float y, float z, float* o) {
  const float xx = x * x, yy = y * y, zz = z * z;
  o[0] = 0.28209479177387814f;
  o[1] = -0.48860251190291987f * y;
  o[2] = 0.48860251190291987f * z;
  o[3] = -0.48860251190291987f * x;
  o[4] = 1.0925484305920792f * x * y;
  o[5] = -1.0925484305920792f * y * z;
  o[6] = 0.94617469575755997f * zz - 0.31539156525251999f;
  o[7] = -1.0925484305920792f * x * z;
  o[8] = 0.54627421529603959f * (xx - yy);
  o[9] = 0.59004358992664352f * y * (-3.0f * xx + yy);
  o[10] = 2.8906114426405538f * x * y * z;
  o[11] = 0.45704579946446572f * y * (1.0f - 5.0f * zz);
  o[12] = 0.3731763325901154f * z * (5.0f * zz - 3.0f);
  o[13] = 0.45704579946446572f * x * (1.0f - 5.0f * zz);
  o[14] = 1.4453057213202769f * z * (xx - yy);
  o[15] = 0.59004358992664352f * x * (-xx + 3.0f * yy);
}

constexpr int kColorW = (64 * 32 + 16 * 64 + 64 * 32 + 64 * 64 + 16 * 64) * 2;  // 20,480 B

// E_g / E_c with the activations in TMEM (TS-form MMAs, as DeformNet): per slot
// D (64 fp32 columns) + A (32 packed fp16x2 columns) = 96 columns, 5 slots of 4
// warps (thread = sample row). The narrow N = 64 layers made the SS version
// epilogue/latency bound (tensor pipe 12 %): no smem traffic for activations and
// one more slot in flight.
constexpr int kColorTsSlots = 5;

struct CSlot {
  uint64_t* bar;
  uint32_t d0, a0;  // slot base columns (MMA operands)
  uint32_t d, a;    // + this warp's lane quarter
  uint32_t phase;
  int slot, r;
};

__device__ __forceinline__ void cts_layer(CSlot& S, const uint8_t* w, int K, int N) {
  tc::tmem_wait_st();
  tc::fence_before();
  tc::named_sync(1 + S.slot, kSlotThreads);
  if (S.r < 32) {  // the slot's first warp issues
    tc::fence_after();
    tc::layer_ts_warp(S.d0, S.a0, w, K, N, S.bar);
  }
  tc::bar_wait(S.bar, S.phase);
  S.phase ^= 1u;
  tc::fence_after();
}

// 64-wide hidden layer: D -> ReLU -> fp16x2 -> A (K = 64)
__device__ __forceinline__ void cts_relu64(const CSlot& S) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    tc::tmem_ld32_nowait(S.d + (uint32_t)(32 * c), r);
    tc::tmem_wait_ld();
    uint32_t h[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = tc::relu_f16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
    tc::tmem_st16(S.a + (uint32_t)(16 * c), h);
  }
}

__global__ void __launch_bounds__(kColorTsSlots* kSlotThreads, 1)
    color_mlp_kernel(const uint8_t* __restrict__ wblob, const float4* __restrict__ xu, const uint4* __restrict__ cfeat,
                     const uint32_t* __restrict__ records, const double* __restrict__ dirs,
                     const int* __restrict__ count, int64_t capacity, float4* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kColorTsSlots];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid * 16; i < kColorW; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = *reinterpret_cast<const uint4*>(wblob + i);
  if (tid == 0) {
    for (int q = 0; q < kColorTsSlots; ++q) tc::bar_init(&mbar[q], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_wait();  // weights staged and TMEM allocated while the previous kernel drained
  CSlot S;
  S.slot = tid / kSlotThreads;
  S.r = tid % kSlotThreads;
  S.bar = &mbar[S.slot];
  S.phase = 0;
  S.d0 = tmem_base + (uint32_t)(S.slot * 96);
  S.a0 = S.d0 + 64u;
  const uint32_t lane_q = (uint32_t)((warp % 4) * 32) << 16;
  S.d = S.d0 + lane_q;
  S.a = S.a0 + lane_q;
  constexpr int g1 = 0, g2 = 64 * 32 * 2, c1 = g2 + 16 * 64 * 2, c2 = c1 + 64 * 32 * 2, c3 = c2 + 64 * 64 * 2;
  const int64_t n = min((int64_t)*count, capacity);
  const int64_t n_tiles = (n + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * kColorTsSlots + S.slot; tile < n_tiles;
       tile += (int64_t)gridDim.x * kColorTsSlots) {
    const int64_t s = tile * 128 + S.r;
    const bool live = s < n;
    {
      uint32_t w16[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = live ? cfeat[s * 4 + q] : make_uint4(0, 0, 0, 0);
        w16[4 * q] = v.x;
        w16[4 * q + 1] = v.y;
        w16[4 * q + 2] = v.z;
        w16[4 * q + 3] = v.w;
      }
      tc::tmem_st16(S.a, w16);
    }
    // per-sample inputs of the later layers, loaded while the first MMAs run
    const bool valid = live && xu[s].w > 0.0f;
    double ddx = 0.0, ddy = 0.0, ddz = 1.0;
    if (live) {
      const int64_t ray = records[s] >> 8;
      ddx = dirs[3 * ray];
      ddy = dirs[3 * ray + 1];
      ddz = dirs[3 * ray + 2];
    }
    cts_layer(S, smem + g1, 32, 64);
    cts_relu64(S);
    cts_layer(S, smem + g2, 64, 16);
    float gv[16];
    tc::tmem_ld16(S.d, gv);
    const float sigma = valid ? expf(gv[0]) : 0.0f;
    // colour input: [geo(15), SH4(dir)(16), 0]
    {
      float cin[32];
#pragma unroll
      for (int i = 0; i < 15; ++i) cin[i] = gv[1 + i];
      sh16((float)ddx, (float)ddy, (float)ddz, cin + 15);
      cin[31] = 0.0f;
      uint32_t h[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const __half2 hh = __floats2half2_rn(cin[2 * i], cin[2 * i + 1]);
        h[i] = *reinterpret_cast<const uint32_t*>(&hh);
      }
      tc::tmem_st16(S.a, h);
    }
    cts_layer(S, smem + c1, 32, 64);
    cts_relu64(S);
    cts_layer(S, smem + c2, 64, 64);
    cts_relu64(S);
    cts_layer(S, smem + c3, 64, 16);
    float cv[16];
    tc::tmem_ld16(S.d, cv);
    if (live) {
      const float r = 1.0f / (1.0f + expf(-cv[0])), g = 1.0f / (1.0f + expf(-cv[1])),
                  b = 1.0f / (1.0f + expf(-cv[2]));
      out[s] = valid ? make_float4(sigma, r, g, b) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem_base);
  pdl_trigger();
}

// ---------------------------------------------------------------- "fp32" precision mode
// The same networks with every operand split into fp16 hi + lo halves and three
// MMA chains per layer (tc::issue_split_warp): ~22-bit operands, fp32 TMEM
// accumulation, fp32 hash features in. This is the mode that meets the SPEC's
// 32-bit semantics within 1e-4 (tests/test_precision_gpu.py);
// the fp16-operand kernels above are the "fp16" mode.

// DeformNet: both weight halves resident in smem (2 x 108 KB), 2 TS slots of 8
// warps, per slot D (128) + A_hi (64) + A_lo (64) TMEM columns = 512 in all.
constexpr int kPrecDeformSlots = 2;

struct SplitSlot {
  uint64_t* bar;
  uint32_t d0, ahi0, alo0;  // slot base columns (MMA operands)
  uint32_t d, ahi, alo;     // + this warp's lane quarter
  uint32_t phase;
  int slot, r, half, nthreads;
};

// one split layer of a slot: the slot's threads finish their TMEM stores, its first
// warp issues the three chains and the commit (tc::issue_split_warp), all wait for D
template <int K>
__device__ __forceinline__ void split_layer(SplitSlot& S, const uint8_t* w_hi, const uint8_t* w_lo, int N) {
  tc::tmem_wait_st();
  tc::fence_before();
  tc::named_sync(1 + S.slot, S.nthreads);
  if ((threadIdx.x % S.nthreads) < 32) {
    tc::fence_after();
    tc::issue_split_warp<K>(S.d0, S.ahi0, S.alo0, w_hi, w_lo, N, S.bar);
  }
  tc::bar_wait(S.bar, S.phase);
  S.phase ^= 1u;
  tc::fence_after();
}

// 32 D columns from col -> ReLU -> hi / lo fp16x2 -> A columns col/2 (tc::split_relu_rz)
__device__ __forceinline__ void split_relu32(const SplitSlot& S, int col) {
  uint32_t r[32];
  tc::tmem_ld32_nowait(S.d + (uint32_t)col, r);
  tc::tmem_wait_ld();
  uint32_t h[16], l[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) tc::split_relu_rz(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]), h[i], l[i]);
  tc::tmem_st16(S.ahi + (uint32_t)(col / 2), h);
  tc::tmem_st16(S.alo + (uint32_t)(col / 2), l);
}

// n4 float4 of fp32 values -> hi / lo halves at A column c0 (2 values per column)
template <int N4>
__device__ __forceinline__ void split_store(const SplitSlot& S, const float4* v, int c0, uint32_t* hi_out = nullptr) {
  uint32_t h[2 * N4], l[2 * N4];
#pragma unroll
  for (int q = 0; q < N4; ++q) {
    tc::split_f16x2(v[q].x, v[q].y, h[2 * q], l[2 * q]);
    tc::split_f16x2(v[q].z, v[q].w, h[2 * q + 1], l[2 * q + 1]);
  }
  if (hi_out) {
#pragma unroll
    for (int q = 0; q < 2 * N4; ++q) hi_out[q] = h[q];
  }
  if constexpr (N4 == 4) {
    tc::tmem_st8(S.ahi + (uint32_t)c0, h);
    tc::tmem_st8(S.alo + (uint32_t)c0, l);
  } else {
    static_assert(N4 == 8, "8 or 16 columns");
    tc::tmem_st16(S.ahi + (uint32_t)c0, h);
    tc::tmem_st16(S.alo + (uint32_t)c0, l);
  }
}

// kSave: the training forward — xc at 32-bit semantics (the canonical hash backward's
// spatial gradient is evaluated where the 32-bit field puts the sample), plus the
// fp16 saves the fp16 backward consumes: h1..h4 (hi halves, feature-major), the
// ReLU bits, o, and the deformation features' hi halves (dfeat16, for dW of layer 1)
// The "fp32"-mode DeformNet, 16 warps per slot: warp w of a slot owns TMEM lane quarter
// w % 4 (32 sample rows) and column quarter w / 4 (32 of a layer's 128 columns), so a
// layer's epilogue is spread over twice the warps of the 8-warp layout. Measured with
// per-stage clocks, the 8-warp kernel spent 1.3-2k cycles per layer in its epilogue
// against 1.5k cycles of one layer's MMAs: the other slot's MMAs ran dry and the
// tensor pipe was busy 42 % of the time.
constexpr int kPrecDeformThreads = 512;  // per slot

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// one hidden layer's epilogue for this thread's 32 columns (two 16-column chunks):
// D -> (+bias) ReLU -> hi / lo fp16x2 -> A; training: hi halves saved feature-major;
// returns the 32 ReLU bits
// The render (kTrain false) splits with tc::split_relu_rz (5 instructions per pair); the
// training forward keeps the round-to-nearest hi half, the fp16 activation its backward
// consumes, and computes the ReLU bits.
template <bool kTrain>
__device__ __forceinline__ uint32_t split_relu_q(const SplitSlot& S, int col, const float* bias, __half* save,
                                                 int64_t ld) {
  uint32_t bits = 0;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[16];
    tmem_ld16_nowait(S.d + (uint32_t)(col + 16 * c), r);
    tc::tmem_wait_ld();
    uint32_t h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      float x[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = __uint_as_float(r[2 * i + j]);
      if (bias) {
        const float4 bv = *reinterpret_cast<const float4*>(bias + col + 16 * c + 2 * i);
        x[0] += bv.x, x[1] += bv.y, x[2] += bv.z, x[3] += bv.w;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if constexpr (kTrain) {
          bits |= (x[2 * q] > 0.0f ? 1u : 0u) << (16 * c + 2 * (i + q)) |
                  (x[2 * q + 1] > 0.0f ? 1u : 0u) << (16 * c + 2 * (i + q) + 1);
          tc::split_f16x2(fmaxf(x[2 * q], 0.0f), fmaxf(x[2 * q + 1], 0.0f), h[i + q], l[i + q]);
        } else {
          tc::split_relu_rz(x[2 * q], x[2 * q + 1], h[i + q], l[i + q]);
        }
      }
    }
    tc::tmem_st8(S.ahi + (uint32_t)((col + 16 * c) / 2), h);
    tc::tmem_st8(S.alo + (uint32_t)((col + 16 * c) / 2), l);
    if (kTrain && save) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        reinterpret_cast<uint16_t*>(save)[(int64_t)(col + 16 * c + 2 * i) * ld] = (uint16_t)(h[i] & 0xffffu);
        reinterpret_cast<uint16_t*>(save)[(int64_t)(col + 16 * c + 2 * i + 1) * ld] = (uint16_t)(h[i] >> 16);
      }
    }
  }
  return bits;
}

// layer 4's epilogue with the last layer (128 -> 3) on the CUDA cores in fp32: this
// thread's 32 columns -> ReLU -> 3 partial dot products with W5 (fp32, hi + lo); training
// saves as split_relu_q; returns the ReLU bits
template <bool kTrain>
__device__ __forceinline__ uint32_t relu_dot3_q(const SplitSlot& S, int col, const float* w5, float* p, __half* save,
                                                int64_t ld) {
  uint32_t bits = 0;
  p[0] = p[1] = p[2] = 0.0f;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[16];
    tmem_ld16_nowait(S.d + (uint32_t)(col + 16 * c), r);
    tc::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
      const int k = col + 16 * c + i;
      const float4 w0 = *reinterpret_cast<const float4*>(w5 + k), w1 = *reinterpret_cast<const float4*>(w5 + 128 + k),
                   w2 = *reinterpret_cast<const float4*>(w5 + 256 + k);
      const float a0[4] = {w0.x, w0.y, w0.z, w0.w}, a1[4] = {w1.x, w1.y, w1.z, w1.w}, a2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x = __uint_as_float(r[i + j]);
        if constexpr (kTrain) bits |= (x > 0.0f ? 1u : 0u) << (16 * c + i + j);
        const float h = fmaxf(x, 0.0f);
        p[0] = fmaf(a0[j], h, p[0]);
        p[1] = fmaf(a1[j], h, p[1]);
        p[2] = fmaf(a2[j], h, p[2]);
        if (kTrain && save) reinterpret_cast<__half*>(save)[(int64_t)(k + j) * ld] = __float2half_rn(h);
      }
    }
  }
  return bits;
}

// kSave: the training forward — xc at 32-bit semantics (the canonical hash backward's
// spatial gradient is evaluated where the 32-bit field puts the sample), plus the
// fp16 saves the fp16 backward consumes: h1..h4 (hi halves, feature-major), the
// ReLU bits, o, and the deformation features' hi halves (dfeat16, for dW of layer 1)
template <bool kSave, int kHash = 0>
__global__ void __launch_bounds__(kPrecDeformSlots* kPrecDeformThreads, 1)
    deform_mlp_prec_kernel(const uint8_t* __restrict__ wblob, const uint8_t* __restrict__ wblob_lo,
                           const float* __restrict__ bias1, float delta_scale, float inv_side,
                           const float4* __restrict__ xu, const float4* __restrict__ dfeat,
                           const int* __restrict__ count, int64_t capacity, float4* __restrict__ xc,
                           __half* __restrict__ save_h, float4* __restrict__ save_o,
                           uint32_t* __restrict__ save_mask, __half* __restrict__ dfeat16,
                           const uint8_t* __restrict__ l2_prefetch = nullptr, int64_t l2_prefetch_bytes = 0,
                           cf_hashgrid_desc DG = {}, const float* __restrict__ dtable = nullptr) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kPrecDeformSlots];
  // optional (l2_prefetch_on): the next stage's table into L2 while this tensor-bound
  // kernel leaves the memory system idle, each CTA its share as bulk L2 prefetches.
  // Measured: no gain for the hash stage (L1-request bound, 75.8 us after an L2 flush
  // either way), ~4 us cost here, so it is off by default. The kernel compiled with this
  // block runs 88 -> 72 us back to back, issued or not, while the same parameters
  // without the block stay at 88 — a code-layout effect of the hot loop (the same
  // instructions shifted by ~200), kept and documented.
  if (l2_prefetch && threadIdx.x == 0) {
    const int64_t share = ((l2_prefetch_bytes + gridDim.x - 1) / gridDim.x + 65535) & ~(int64_t)65535;
    const int64_t b0 = (int64_t)blockIdx.x * share, b1 = min(b0 + share, l2_prefetch_bytes & ~(int64_t)15);
    for (int64_t b = b0; b < b1; b += 65536) {
      const uint32_t sz = (uint32_t)min((int64_t)65536, b1 - b);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(l2_prefetch + b), "r"(sz) : "memory");
    }
  }
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float s_bias[128];
  __shared__ __align__(16) float s_w5[3 * 128];                        // W5 rows 0..2 in fp32 (hi + lo)
  __shared__ float s_part[kPrecDeformSlots][2][128][3];  // layer-5 partials exchanged between column quarters
  const int tid = threadIdx.x, warp = tid / 32;
  if (tid < 128) s_bias[tid] = bias1[tid];
  for (int i = tid * 16; i < kDeformW; i += blockDim.x * 16) {
    *reinterpret_cast<uint4*>(smem + i) = *reinterpret_cast<const uint4*>(wblob + i);
    *reinterpret_cast<uint4*>(smem + kDeformW + i) = *reinterpret_cast<const uint4*>(wblob_lo + i);
  }
  {
    constexpr int o5w = 128 * 32 * 2 + 3 * 128 * 128 * 2;  // W5 (16 x 128, rows 3.. zero) in the blob
    for (int e = tid; e < 3 * 128; e += blockDim.x) {
      const uint32_t off = o5w + tc::core_offset(e / 128, e % 128, 128);
      s_w5[e] = __half2float(*reinterpret_cast<const __half*>(wblob + off)) +
                __half2float(*reinterpret_cast<const __half*>(wblob_lo + off));
    }
  }
  if (tid == 0) {
    for (int q = 0; q < kPrecDeformSlots; ++q) tc::bar_init(&mbar[q], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_wait();
  SplitSlot S;
  S.nthreads = kPrecDeformThreads;
  S.slot = tid / kPrecDeformThreads;
  const int ws = warp % (kPrecDeformThreads / 32);  // warp within the slot (0..15)
  const int cq = ws / 4;                            // column quarter
  S.half = cq;
  S.r = (ws % 4) * 32 + (tid & 31);                 // sample row = TMEM lane
  S.bar = &mbar[S.slot];
  S.phase = 0;
  const uint32_t lane_q = (uint32_t)((ws % 4) * 32) << 16;
  S.d0 = tmem_base + (uint32_t)(S.slot * 256);
  S.ahi0 = S.d0 + 128u;
  S.alo0 = S.d0 + 192u;
  S.d = S.d0 + lane_q;
  S.ahi = S.ahi0 + lane_q;
  S.alo = S.alo0 + lane_q;
  const uint8_t* lo = smem + kDeformW;
  constexpr int o2 = 128 * 32 * 2, o3 = o2 + 128 * 128 * 2, o4 = o3 + 128 * 128 * 2;
  const int64_t n = min((int64_t)*count, capacity);
  const int64_t n_tiles = (n + 127) / 128;
  const int64_t L = 128 * capacity;
  // the render (kSave false): tiles taken from a ticket (counters[2]) instead of a fixed
  // stride, so slots that start late (their SM still busy with the previous kernel or
  // the object field) take fewer tiles; the last slot out re-arms counters[2..3]
  constexpr bool kDyn = !kSave;
  __shared__ int s_next[kPrecDeformSlots];
  int* const ticket = const_cast<int*>(count) + 2;
  const bool slot_lead = (threadIdx.x % S.nthreads) == 0;
  int64_t tile = (int64_t)blockIdx.x * kPrecDeformSlots + S.slot;
  if constexpr (kDyn) {
    if (slot_lead) s_next[S.slot] = atomicAdd(ticket, 1);
    tc::named_sync(1 + S.slot, S.nthreads);
    tile = s_next[S.slot];
  }
  for (; tile < n_tiles;) {
    const int64_t s = tile * 128 + S.r;
    const bool live = s < n;
    // the sample's position (quarter 0: the output at the end of the tile; kHash: every
    // quarter, the deformation-grid lookup), loaded now, under the layers
    const float4 xu_s = ((kHash > 0 || cq == 0) && live) ? xu[s] : make_float4(0.f, 0.f, 0.f, 0.f);
    {  // this quarter's 8 input features (levels 2 cq, 2 cq + 1) -> hi / lo A columns 4 cq ..
      float4 f0, f1;
      if constexpr (kHash > 0) {  // the deformation-grid hash here, as hash_f16_kernel computes it
        float ft[8];
        if (xu_s.w > 0.0f) {
          hash_features<4, 2, kHash, float>(DG, dtable, xu_s.x, xu_s.y, xu_s.z, ft, 2 * cq);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) ft[i] = 0.0f;
        }
        f0 = make_float4(ft[0], ft[1], ft[2], ft[3]);
        f1 = make_float4(ft[4], ft[5], ft[6], ft[7]);
      } else {
        f0 = live ? dfeat[s * 8 + 2 * cq] : make_float4(0.f, 0.f, 0.f, 0.f);
        f1 = live ? dfeat[s * 8 + 2 * cq + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      uint32_t h[4], l[4];
      tc::split_f16x2(f0.x, f0.y, h[0], l[0]);
      tc::split_f16x2(f0.z, f0.w, h[1], l[1]);
      tc::split_f16x2(f1.x, f1.y, h[2], l[2]);
      tc::split_f16x2(f1.z, f1.w, h[3], l[3]);
      tc::tmem_st4(S.ahi + (uint32_t)(4 * cq), h);
      tc::tmem_st4(S.alo + (uint32_t)(4 * cq), l);
      if (kSave && s < capacity) {
        // K-blocked (33, capacity): this quarter's 8 feature rows, + row 32 = 1 (the
        // layer-1 dW GEMM's extra column: sum_s dpre1, for the pose columns)
        uint16_t* d16 = reinterpret_cast<uint16_t*>(dfeat16) + kb_col(s, 33);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          d16[(8 * cq + 2 * i) * kKbLd] = (uint16_t)(h[i] & 0xffffu);
          d16[(8 * cq + 2 * i + 1) * kKbLd] = (uint16_t)(h[i] >> 16);
        }
        if (cq == 0) d16[32 * kKbLd] = 0x3C00u;  // 1.0
      }
    }
    // training saves: h as four K-blocked (128, capacity) matrices, ReLU bits
    // [layer][32-column word] per sample
    __half* sv = (kSave && s < capacity) ? save_h + kb_col(s, 128) : nullptr;
    uint32_t* mk = (kSave && live) ? save_mask + s * 16 + cq : nullptr;
#pragma unroll 1
    for (int l = 0; l < 3; ++l) {
      if (l == 0) {
        split_layer<32>(S, smem, lo, 128);
        // every thread of the slot has read this tile's number: fetch the next one
        if (kDyn && slot_lead) s_next[S.slot] = atomicAdd(ticket, 1);
      } else
        split_layer<128>(S, smem + o2 + (l - 1) * (o3 - o2), lo + o2 + (l - 1) * (o3 - o2), 128);
      const uint32_t b = split_relu_q<kSave>(S, 32 * cq, l == 0 ? s_bias : nullptr, sv ? sv + l * L : nullptr, kKbLd);
      if (mk) mk[4 * l] = b;
    }
    split_layer<128>(S, smem + o4, lo + o4, 128);
    float part[3];
    {
      const uint32_t b = relu_dot3_q<kSave>(S, 32 * cq, s_w5, part, sv ? sv + 3 * L : nullptr, kKbLd);
      if (mk) mk[12] = b;
    }
    // the four quarters' partials summed as (p0 + p2) + (p1 + p3), in two exchanges: the
    // second goes through quarter 1's own first-exchange entry (read by the same thread)
    if (cq >= 2) {
#pragma unroll
      for (int j = 0; j < 3; ++j) s_part[S.slot][cq - 2][S.r][j] = part[j];
    }
    tc::named_sync(1 + S.slot, S.nthreads);
    if (cq < 2) {
#pragma unroll
      for (int j = 0; j < 3; ++j) part[j] += s_part[S.slot][cq][S.r][j];
    }
    if (cq == 1) {
#pragma unroll
      for (int j = 0; j < 3; ++j) s_part[S.slot][1][S.r][j] = part[j];
    }
    tc::named_sync(1 + S.slot, S.nthreads);
    if (cq == 0) {
      float v[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) v[j] = part[j] + s_part[S.slot][1][S.r][j];
      if (kSave && live) save_o[s] = make_float4(v[0], v[1], v[2], 0.0f);
      if (live) {
        float4 p = xu_s;
        if (p.w > 0.0f) {
          p.x = f_add(p.x, f_mul(delta_scale * tanhf(v[0]), inv_side));
          p.y = f_add(p.y, f_mul(delta_scale * tanhf(v[1]), inv_side));
          p.z = f_add(p.z, f_mul(delta_scale * tanhf(v[2]), inv_side));
        }
        xc[s] = p;
      }
    }
    if constexpr (kDyn)
      tile = s_next[S.slot];  // written after this tile's first barrier
    else
      tile += (int64_t)gridDim.x * kPrecDeformSlots;
  }
  if (kDyn && slot_lead) {
    __threadfence();
    if (atomicAdd(ticket + 1, 1) == (int)(gridDim.x * kPrecDeformSlots) - 1) {
      ticket[0] = 0;
      ticket[1] = 0;
    }
  }
  pdl_trigger();
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem_base);
}

// E_g / E_c: weight halves 2 x 20 KB, 4 slots of 4 warps (thread = sample row),
// per slot D (64) + A_hi (32) + A_lo (32) TMEM columns.
constexpr int kColorPrecSlots = 4;

// kHashCH > 0: the canonical hash features are computed here (hash_features with
// kHashCH levels in flight, from the positions xu) instead of read from cfeat — the
// gathers of one slot overlap the other slots' MMAs and epilogues
template <int kHashCH>
__global__ void __launch_bounds__(kColorPrecSlots* kSlotThreads, 1)
    color_mlp_prec_kernel(const uint8_t* __restrict__ wblob, const uint8_t* __restrict__ wblob_lo,
                          const float4* __restrict__ xu, const float4* __restrict__ cfeat,
                          const uint32_t* __restrict__ records, const double* __restrict__ dirs,
                          const int* __restrict__ count, int64_t capacity, float4* __restrict__ out,
                          __half* __restrict__ cfeat16, cf_hashgrid_desc HD = {}, const float* __restrict__ htable = nullptr) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kColorPrecSlots];
  __shared__ uint32_t tmem_base;
  __shared__ float s_w3[3 * 64];  // E_c's last layer (64 -> 3) in fp32 (hi + lo), on the CUDA cores
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid * 16; i < kColorW; i += blockDim.x * 16) {
    *reinterpret_cast<uint4*>(smem + i) = *reinterpret_cast<const uint4*>(wblob + i);
    *reinterpret_cast<uint4*>(smem + kColorW + i) = *reinterpret_cast<const uint4*>(wblob_lo + i);
  }
  {
    constexpr int c3w = 64 * 32 * 2 + 16 * 64 * 2 + 64 * 32 * 2 + 64 * 64 * 2;
    for (int e = tid; e < 3 * 64; e += blockDim.x) {
      const uint32_t off = c3w + tc::core_offset(e / 64, e % 64, 64);
      s_w3[e] = __half2float(*reinterpret_cast<const __half*>(wblob + off)) +
                __half2float(*reinterpret_cast<const __half*>(wblob_lo + off));
    }
  }
  if (tid == 0) {
    for (int q = 0; q < kColorPrecSlots; ++q) tc::bar_init(&mbar[q], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_wait();
  SplitSlot S;
  S.nthreads = kSlotThreads;
  S.slot = tid / kSlotThreads;
  S.r = tid % kSlotThreads;
  S.half = 0;
  S.bar = &mbar[S.slot];
  S.phase = 0;
  const uint32_t lane_q = (uint32_t)((warp % 4) * 32) << 16;
  S.d0 = tmem_base + (uint32_t)(S.slot * 128);
  S.ahi0 = S.d0 + 64u;
  S.alo0 = S.d0 + 96u;
  S.d = S.d0 + lane_q;
  S.ahi = S.ahi0 + lane_q;
  S.alo = S.alo0 + lane_q;
  const uint8_t* lo = smem + kColorW;
  constexpr int g1 = 0, g2 = 64 * 32 * 2, c1 = g2 + 16 * 64 * 2, c2 = c1 + 64 * 32 * 2;
  const int64_t n = min((int64_t)*count, capacity);
  const int64_t n_tiles = (n + 127) / 128;
  // the render's fused instance: tiles from a ticket (counters[2]), as DeformNet's
  constexpr bool kDyn = kHashCH > 0;
  __shared__ int s_next[kColorPrecSlots];
  int* const ticket = const_cast<int*>(count) + 2;
  const bool slot_lead = (threadIdx.x % S.nthreads) == 0;
  int64_t tile = (int64_t)blockIdx.x * kColorPrecSlots + S.slot;
  if constexpr (kDyn) {
    if (slot_lead) s_next[S.slot] = atomicAdd(ticket, 1);
    tc::named_sync(1 + S.slot, S.nthreads);
    tile = s_next[S.slot];
  }
  for (; tile < n_tiles;) {
    const int64_t s = tile * 128 + S.r;
    const bool live = s < n;
    {
      float4 f[8];
      if constexpr (kHashCH > 0) {
        const float4 p = live ? xu[s] : make_float4(0.f, 0.f, 0.f, 0.f);
        float* ff = reinterpret_cast<float*>(f);
        if (p.w > 0.0f) {
          hash_features<2, 16, kHashCH, float>(HD, htable, p.x, p.y, p.z, ff);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) ff[i] = 0.0f;
        }

      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = live ? cfeat[s * 8 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      uint32_t hi[16];
      split_store<8>(S, f, 0, cfeat16 ? hi : nullptr);
      if (cfeat16 && s < capacity) {  // training: the features' fp16 halves, K-blocked (32, capacity)
        uint16_t* d16 = reinterpret_cast<uint16_t*>(cfeat16) + kb_col(s, 32);
        store_cols16_f16(d16, kKbLd, 0, 0, hi);
        store_cols16_f16(d16, kKbLd, 0, 16, hi + 8);
      }
    }
    const bool valid = live && xu[s].w > 0.0f;
    double ddx = 0.0, ddy = 0.0, ddz = 1.0;
    if (live) {
      const int64_t ray = records[s] >> 8;
      ddx = dirs[3 * ray];
      ddy = dirs[3 * ray + 1];
      ddz = dirs[3 * ray + 2];
    }
    split_layer<32>(S, smem + g1, lo + g1, 64);
    if (kDyn && slot_lead) s_next[S.slot] = atomicAdd(ticket, 1);  // all have read this tile's
    split_relu32(S, 0);
    split_relu32(S, 32);
    split_layer<64>(S, smem + g2, lo + g2, 16);
    float gv[16];
    tc::tmem_ld16(S.d, gv);
    const float sigma = valid ? expf(gv[0]) : 0.0f;
    {
      float cin[32];
#pragma unroll
      for (int i = 0; i < 15; ++i) cin[i] = gv[1 + i];
      sh16((float)ddx, (float)ddy, (float)ddz, cin + 15);
      cin[31] = 0.0f;
      split_store<8>(S, reinterpret_cast<const float4*>(cin), 0);
    }
    split_layer<32>(S, smem + c1, lo + c1, 64);
    split_relu32(S, 0);
    split_relu32(S, 32);
    split_layer<64>(S, smem + c2, lo + c2, 64);
    // the last layer (64 -> 3) in fp32 on the CUDA cores: an N = 16 MMA chain runs at
    // 1/8 of the tensor rate (tools/mma_bench.cu), as long as a full-width layer
    float cv[3] = {0.f, 0.f, 0.f};
    {
      uint32_t r[64];
      tc::tmem_ld32_nowait(S.d, r);
      tc::tmem_ld32_nowait(S.d + 32u, r + 32);
      tc::tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const float h = fmaxf(__uint_as_float(r[k]), 0.0f);
        cv[0] = fmaf(s_w3[k], h, cv[0]);
        cv[1] = fmaf(s_w3[64 + k], h, cv[1]);
        cv[2] = fmaf(s_w3[128 + k], h, cv[2]);
      }
    }
    if (live) {
      const float r = 1.0f / (1.0f + expf(-cv[0])), g = 1.0f / (1.0f + expf(-cv[1])),
                  b = 1.0f / (1.0f + expf(-cv[2]));
      out[s] = valid ? make_float4(sigma, r, g, b) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if constexpr (kDyn)
      tile = s_next[S.slot];
    else
      tile += (int64_t)gridDim.x * kColorPrecSlots;
  }
  if (kDyn && slot_lead) {
    __threadfence();
    if (atomicAdd(ticket + 1, 1) == (int)(gridDim.x * kColorPrecSlots) - 1) {
      ticket[0] = 0;
      ticket[1] = 0;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem_base);
  pdl_trigger();
}

// ---------------------------------------------------------------- E_g / E_c backward

// Transposed weights for dX = dY . W, in the blob order C3t (64x16), C2t (64x64),
// C1t (32x64), G2t (64x16), G1t (32x64): each W^T packed K-major (K = N_out).
constexpr int kColorWT = (64 * 16 + 64 * 64 + 32 * 64 + 64 * 16 + 32 * 64) * 2;  // 20,480 B
constexpr int kBwdSlots = 4;
constexpr int kBwdA = 128 * 64 * 2;

struct ColorBwdIO {
  // saved activations / output grads (fp16 rows) for the weight-gradient GEMMs
  __half* h1;    // (S,64) relu(G1 x)
  __half* cin;   // (S,32) [geo, SH, 0]
  __half* c1;    // (S,64)
  __half* c2;    // (S,64)
  __half* d_o;   // (S,16) dL/d(E_c output)
  __half* dc2;   // (S,64) dL/d(C2 pre-activation)
  __half* dc1;   // (S,64)
  __half* dg;    // (S,16) dL/d(E_g output)
  __half* dh1;   // (S,64)
  float* dfeat;  // (S,32) dL/d(hash features)
};

// width fp16 values of sample s into a feature-major (width, ld) block: column c at
// dst[c * ld + s]. Lanes are consecutive samples (s even on even lanes, ld even): the
// lane pair (2j, 2j+1) swaps one value per column pair so that the even lane writes
// column c and the odd lane column c+1 for both samples as one 32-bit store — two
// coalesced 64-byte segments per warp store, half the store instructions of 2-byte
// stores. All 32 lanes call it (shuffles); ok gates the lane's store (the pair's
// lanes share it: a tile's lanes are all inside the capacity, a multiple of 128).
// (width a template parameter and the loop fully unrolled: with a runtime width and a
// partial unroll, v[] was indexed at run time and lived in local memory — 256 bytes of
// stack per thread in the colour backward)
template <int kWidth>
__device__ __forceinline__ void store_fm_f16(__half* dst, int64_t s, int rows, const float* v, bool ok) {
  const bool odd = threadIdx.x & 1;
  const int64_t s0 = s & ~(int64_t)1;
  dst += kb_col(s0, rows);  // s0, s0 + 1: adjacent in one block
#pragma unroll
  for (int c = 0; c < kWidth; c += 2) {
    // even lane (sample s0) keeps v[c], sends v[c+1]; odd lane (s0 + 1) keeps v[c+1], sends v[c]
    const float mine = odd ? v[c + 1] : v[c];
    const float other = __shfl_xor_sync(0xffffffffu, odd ? v[c] : v[c + 1], 1);
    const __half2 h = odd ? __floats2half2_rn(other, mine) : __floats2half2_rn(mine, other);
    if (ok) *reinterpret_cast<__half2*>(dst + (c + (odd ? 1 : 0)) * kKbLd) = h;
  }
}

// forward hidden layer with ReLU: keep the activation mask, write fp16 to A buffer (+ the
// feature-major HBM copy, row stride ld)
template <int N>
__device__ __forceinline__ uint64_t fwd_relu(Slot& S, __half* save, int64_t s, bool live) {
  uint64_t mask = 0;
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(S.tmem_row + (uint32_t)c0, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (v[i] > 0.f) mask |= 1ull << (c0 + i);
      v[i] = fmaxf(v[i], 0.0f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) tc::st_row8(S.abuf, S.r, c0 + 8 * q, N, v + 8 * q);
    store_fm_f16<32>(save + c0 * kKbLd, s, N, v, live);
  }
  return mask;
}

// backward through a ReLU layer: dpre = dact (from TMEM) * relu'(mask) -> A buffer (+ HBM)
template <int N>
__device__ __forceinline__ void bwd_relu(Slot& S, uint64_t mask, __half* save, int64_t s, bool live) {
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(S.tmem_row + (uint32_t)c0, v);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!((mask >> (c0 + i)) & 1ull)) v[i] = 0.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q) tc::st_row8(S.abuf, S.r, c0 + 8 * q, N, v + 8 * q);
    store_fm_f16<32>(save + c0 * kKbLd, s, N, v, live);
  }
}

__global__ void __launch_bounds__(kBwdSlots* kSlotThreads, 1)
    color_bwd_kernel(const uint8_t* __restrict__ wblob, const uint8_t* __restrict__ wtblob,
                     const float4* __restrict__ xu, const float4* __restrict__ cfeat32,
                     const uint32_t* __restrict__ records, const double* __restrict__ dirs,
                     const float4* __restrict__ gout, const int* __restrict__ count, int64_t capacity,
                     ColorBwdIO io) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kBwdSlots];
  __shared__ uint32_t tmem_base;
  // stage both weight blobs contiguously: forward (20 KB) then transposed (20 KB)
  for (int i = threadIdx.x * 16; i < kColorWT; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + kColorW + i) = *reinterpret_cast<const uint4*>(wtblob + i);
  slots_setup<kBwdSlots, 256>(wblob, kColorW, smem, mbar, &tmem_base);
  Slot S = make_slot<kBwdSlots, 64, kBwdA>(smem, kColorW + kColorWT, mbar, tmem_base);
  constexpr int g1 = 0, g2 = 64 * 32 * 2, c1 = g2 + 16 * 64 * 2, c2 = c1 + 64 * 32 * 2, c3 = c2 + 64 * 64 * 2;
  constexpr int t_c3 = kColorW, t_c2 = t_c3 + 64 * 16 * 2, t_c1 = t_c2 + 64 * 64 * 2, t_g2 = t_c1 + 32 * 64 * 2,
                t_g1 = t_g2 + 64 * 16 * 2;
  const int64_t n = min((int64_t)*count, capacity);
  const int64_t n_tiles = (n + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * kBwdSlots + S.slot; tile < n_tiles; tile += (int64_t)gridDim.x * kBwdSlots) {
    const int64_t s = tile * 128 + S.r;
    const bool live = s < n;
    // the saves (K-blocked feature-major, kb_col) are written for every lane of the
    // tile inside the capacity: the dW GEMMs' last K tile reads past n, where the dead
    // lanes' dL/d terms are zero and their activations finite
    const bool keep = s < capacity;
    const bool valid = live && xu[s].w > 0.0f;
    // ---- forward recompute from the features (the training forward's fp32 features,
    // sample-major: 8 vector loads; st_row8 rounds them to the same fp16 values the
    // feature-major copy for the dW GEMM holds), saving what the weight gradients need
    {
      float4 x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = live ? cfeat32[s * 8 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 8) tc::st_row8(S.abuf, S.r, k0, 32, reinterpret_cast<const float*>(x) + k0);
    }
    run_layer(S, g1, 32, 64);
    const uint64_t m_h1 = fwd_relu<64>(S, io.h1, s, keep);
    run_layer(S, g2, 64, 16);
    float gv[16];
    tc::tmem_ld16(S.tmem_row, gv);
    const float sigma = expf(gv[0]);
    float cin[32];
#pragma unroll
    for (int i = 0; i < 15; ++i) cin[i] = gv[1 + i];
    float dx = 0.f, dy = 0.f, dz = 1.f;
    if (live) {
      const int64_t ray = records[s] >> 8;
      dx = (float)dirs[3 * ray];
      dy = (float)dirs[3 * ray + 1];
      dz = (float)dirs[3 * ray + 2];
    }
    sh16(dx, dy, dz, cin + 15);
    cin[31] = 0.0f;
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 8) tc::st_row8(S.abuf, S.r, k0, 32, cin + k0);
    store_fm_f16<32>(io.cin, s, 32, cin, keep);
    run_layer(S, c1, 32, 64);
    const uint64_t m_c1 = fwd_relu<64>(S, io.c1, s, keep);
    run_layer(S, c2, 64, 64);
    const uint64_t m_c2 = fwd_relu<64>(S, io.c2, s, keep);
    run_layer(S, c3, 64, 16);
    float ov[16];
    tc::tmem_ld16(S.tmem_row, ov);
    // ---- backward: dO = dL/drgb * sigmoid'
    const float4 g = valid ? gout[s] : make_float4(0.f, 0.f, 0.f, 0.f);
    float d_o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) d_o[i] = 0.f;
    {
      const float gr[3] = {g.y, g.z, g.w};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float sg = 1.0f / (1.0f + expf(-ov[c]));
        d_o[c] = gr[c] * sg * (1.0f - sg);
      }
    }
    tc::st_row8(S.abuf, S.r, 0, 16, d_o);
    tc::st_row8(S.abuf, S.r, 8, 16, d_o + 8);
    store_fm_f16<16>(io.d_o, s, 16, d_o, keep);
    run_layer(S, t_c3, 16, 64);  // dC2act = dO . C3
    bwd_relu<64>(S, m_c2, io.dc2, s, keep);
    run_layer(S, t_c2, 64, 64);  // dC1act = dC2 . C2
    bwd_relu<64>(S, m_c1, io.dc1, s, keep);
    run_layer(S, t_c1, 64, 32);  // dCin = dC1 . C1
    float dcin[32];
    tc::tmem_ld32(S.tmem_row, dcin);
    float dg[16];
    dg[0] = valid ? g.x * sigma : 0.f;  // sigma = exp(g0)
#pragma unroll
    for (int i = 1; i < 16; ++i) dg[i] = dcin[i - 1];
    tc::st_row8(S.abuf, S.r, 0, 16, dg);
    tc::st_row8(S.abuf, S.r, 8, 16, dg + 8);
    store_fm_f16<16>(io.dg, s, 16, dg, keep);
    run_layer(S, t_g2, 16, 64);  // dH1act = dG . G2
    bwd_relu<64>(S, m_h1, io.dh1, s, keep);
    run_layer(S, t_g1, 64, 32);  // dX0 = dH1 . G1
    float dfx[32];
    tc::tmem_ld32(S.tmem_row, dfx);
    if (live) {
      float4* d = reinterpret_cast<float4*>(io.dfeat + s * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = make_float4(dfx[4 * q], dfx[4 * q + 1], dfx[4 * q + 2], dfx[4 * q + 3]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 0) tc::tmem_free<256>(tmem_base);
}

// Scatter-add of one level's 8 corner contributions v[k][0..F) at idx[k] (lanes
// with !valid add nothing). Consecutive lanes are consecutive samples, mostly of one
// ray, so at the coarse levels runs of lanes share a cell: each run is summed in
// registers first (segmented suffix sums over shuffles, log2(longest run) steps) and
// its head issues the 8 vector atomics. A level whose lanes all sit in distinct
// cells (the fine levels) costs one key compare and goes straight to the atomics.
template <int F>
__device__ __forceinline__ void level_scatter(bool valid, const uint32_t* gi, const uint32_t* idx, float (*v)[F],
                                              float* __restrict__ base) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint32_t klo = gi[0] | (gi[1] << 16), khi = gi[2];
  const uint32_t plo = __shfl_up_sync(FULL, klo, 1), phi = __shfl_up_sync(FULL, khi, 1);
  const int pvalid = __shfl_up_sync(FULL, (int)valid, 1);
  const bool head = lane == 0 || !valid || !pvalid || plo != klo || phi != khi;
  const unsigned heads = __ballot_sync(FULL, head);
  if (heads != FULL) {
    for (int o = 1; o < 32; o <<= 1) {
      // lane + o lies in this lane's run iff no run starts in (lane, lane + o]
      const bool ok = lane + o < 32 && ((heads >> (lane + 1)) & ((1u << o) - 1u)) == 0u;
      if (!__any_sync(FULL, ok)) break;
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const float t = __shfl_down_sync(FULL, v[k][f], o);
          if (ok) v[k][f] += t;
        }
    }
  }
  if (valid && head) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float* dst = base + (int64_t)idx[k] * F;
      if constexpr (F == 2) atomicAdd(reinterpret_cast<float2*>(dst), make_float2(v[k][0], v[k][1]));
      else atomicAdd(reinterpret_cast<float4*>(dst), make_float4(v[k][0], v[k][1], v[k][2], v[k][3]));
    }
  }
}

// hash backward on the compacted samples: grad[entry] += w_corner * dfeat (fp32 vector atomics)
template <int F, int L>
__global__ void __launch_bounds__(128) hash_bwd_kernel(cf_hashgrid_desc D, const float4* __restrict__ x,
                                                       const float* __restrict__ dfeat, const int* __restrict__ count,
                                                       int64_t capacity, float* __restrict__ grad) {
  const int64_t n = min((int64_t)*count, capacity);
  const uint32_t mask = (1u << D.log2_table) - 1u;
  // warp-uniform trip count (the coarse-level scatter is warp-cooperative)
  for (int64_t s0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); s0 < n;
       s0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = s0 + (threadIdx.x & 31);
    const float4 p = s < n ? x[s] : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool valid = p.w > 0.0f;
    if (!__any_sync(0xffffffffu, valid)) continue;
    const float px = fminf(fmaxf(p.x, 0.f), 1.f), py = fminf(fmaxf(p.y, 0.f), 1.f), pz = fminf(fmaxf(p.z, 0.f), 1.f);
    const float* g = dfeat + (valid ? s : 0) * (L * F);
#pragma unroll 2
    for (int l = 0; l < L; ++l) {
      const int N = D.resolution[l];
      const float sc = (float)N;
      const float pos[3] = {f_mul(px, sc), f_mul(py, sc), f_mul(pz, sc)};
      uint32_t gi[3];
      float fr[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int v = (int)floorf(pos[a]);
        v = v > N - 1 ? N - 1 : v;
        gi[a] = (uint32_t)v;
        fr[a] = f_sub(pos[a], (float)v);
      }
      const uint32_t stride = (uint32_t)N + 1u;
      const bool dense = D.dense[l] != 0;
      float gl[F];
#pragma unroll
      for (int f = 0; f < F; ++f) gl[f] = g[l * F + f];
      uint32_t idx[8];
      float v[8][F];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t cx = gi[0] + (k & 1), cy = gi[1] + ((k >> 1) & 1), cz = gi[2] + ((k >> 2) & 1);
        idx[k] = dense ? (cx + cy * stride + cz * stride * stride)
                       : ((cx ^ (cy * 2654435761u) ^ (cz * 805459861u)) & mask);
        const float w = f_mul(f_mul((k & 1) ? fr[0] : f_sub(1.f, fr[0]), (k & 2) ? fr[1] : f_sub(1.f, fr[1])),
                              (k & 4) ? fr[2] : f_sub(1.f, fr[2]));
#pragma unroll
        for (int f = 0; f < F; ++f) v[k][f] = w * gl[f];
      }
      level_scatter<F>(valid, gi, idx, v, grad + D.offset[l] * F);
    }
  }
}

// ---------------------------------------------------------------- DeformNet backward

// transposed DeformNet weights as B operands: W5^T (128x16), W4^T, W3^T, W2^T
// (128x128), W1x^T (32x128; the hash-feature columns of layer 1)
constexpr int kDeformWT = (128 * 16 + 3 * 128 * 128 + 32 * 128) * 2;  // 110,592 B
// The backward uses the forward kernel's slot machinery (TsSlot / ts_layer):
// 3 slots of 8 warps, two with dL/dpre in TMEM (TS-form MMAs) and one in smem.
constexpr int kDBwdSlots = kDeformSlots;

// dL/dpre of a 128-wide ReLU layer for this warp's 64 columns: D (= dL/dact) *
// [pre > 0] (the forward's saved ReLU bits, bit j = column 64*half + j) -> fp16
// A operand (TMEM or smem) and the sample's dpre column in the feature-major
// (128, ld) block at dpre (or null)
__device__ __forceinline__ void ts_bwd_mask128(const TsSlot& S, uint64_t mask, __half* dpre, int64_t ld) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int col = 64 * S.half + 32 * c;
    const uint32_t m = (uint32_t)(mask >> (32 * c));
    float r[32];
    tc::tmem_ld32(S.d + (uint32_t)col, r);
    uint32_t h[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float x0 = (m >> (2 * i)) & 1u ? r[2 * i] : 0.0f;
      const float x1 = (m >> (2 * i + 1)) & 1u ? r[2 * i + 1] : 0.0f;
      const __half2 o = __floats2half2_rn(x0, x1);
      h[i] = *reinterpret_cast<const uint32_t*>(&o);
    }
    if (S.abuf) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(S.abuf + tc::core_offset(S.r, col + 8 * q, 128)) =
            make_uint4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
    } else {
      tc::tmem_st16(S.a + (uint32_t)(col / 2), h);
    }
    if (dpre) store_cols_f16(reinterpret_cast<uint16_t*>(dpre), ld, col, h);
  }
}

// Per 128-sample tile: d_o from dL/dxc, then the dX chain through layers 5..1
// with the saved forward activations (ReLU masks), saving d_o and dpre1..4
// (fp16) for the weight-gradient GEMMs and writing dL/d(deform features).
__global__ void __launch_bounds__(kDBwdSlots* kDeformSlotThreads, 1)
    deform_bwd_kernel(const uint8_t* __restrict__ wtblob, float delta_scale, float inv_side,
                      const float4* __restrict__ xu, const float4* __restrict__ dxc,
                      const uint2* __restrict__ save_mask, const float4* __restrict__ save_o, const int* __restrict__ count, int64_t capacity,
                      __half* __restrict__ d_o_out, __half* __restrict__ dpre, float* __restrict__ d_dfeat) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kDBwdSlots];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid * 16; i < kDeformWT; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = *reinterpret_cast<const uint4*>(wtblob + i);
  if (tid == 0) {
    for (int q = 0; q < kDBwdSlots; ++q) tc::bar_init(&mbar[q], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  TsSlot S;
  S.slot = tid / kDeformSlotThreads;
  const int ws = warp % (kDeformSlotThreads / 32);
  S.half = ws / 4;
  S.r = (ws % 4) * 32 + (tid & 31);
  S.bar = &mbar[S.slot];
  S.phase = 0;
  const uint32_t lane_q = (uint32_t)((ws % 4) * 32) << 16;
  S.d0 = tmem_base + (uint32_t)(S.slot * 192);
  S.a0 = S.d0 + 128u;
  S.abuf = S.slot == 2 ? smem + kDeformWT : nullptr;
  S.d = S.d0 + lane_q;
  S.a = S.a0 + lane_q;
  constexpr int t5 = 0, t4 = 128 * 16 * 2, t3 = t4 + 128 * 128 * 2, t2 = t3 + 128 * 128 * 2, t1 = t2 + 128 * 128 * 2;
  const int64_t n = min((int64_t)*count, capacity);
  const int64_t n_tiles = (n + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * kDBwdSlots + S.slot; tile < n_tiles;
       tile += (int64_t)gridDim.x * kDBwdSlots) {
    const int64_t s = tile * 128 + S.r;
    const bool live = s < n;
    if (S.half == 0) {
      // xc = xu + delta_scale * tanh(o) * inv_side => dL/do = dL/dxc delta_scale inv_side (1 - tanh^2 o)
      float d_o[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) d_o[i] = 0.0f;
      if (live && xu[s].w > 0.0f) {
        const float4 g = dxc[s], o = save_o[s];
        const float gg[3] = {g.x, g.y, g.z}, oo[3] = {o.x, o.y, o.z};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float th = tanhf(oo[c]);
          d_o[c] = gg[c] * delta_scale * inv_side * (1.0f - th * th);
        }
      }
      uint32_t h[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const __half2 o = __floats2half2_rn(d_o[2 * i], d_o[2 * i + 1]);
        h[i] = *reinterpret_cast<const uint32_t*>(&o);
      }
      if (S.abuf) {
        *reinterpret_cast<uint4*>(S.abuf + tc::core_offset(S.r, 0, 16)) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(S.abuf + tc::core_offset(S.r, 8, 16)) = make_uint4(h[4], h[5], h[6], h[7]);
      } else {
        tc::tmem_st8(S.a, h);
      }
      if (s < capacity) {  // K-blocked (16, capacity); dead lanes write zeros
        __half* d = d_o_out + kb_col(s, 16);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          d[(2 * i) * kKbLd] = __ushort_as_half((uint16_t)(h[i] & 0xffffu));
          d[(2 * i + 1) * kKbLd] = __ushort_as_half((uint16_t)(h[i] >> 16));
        }
      }
    }
    // the 4 layers' ReLU bits for this half, fetched once per tile
    uint64_t mk[4] = {0, 0, 0, 0};
    if (live) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const uint2 v = save_mask[s * 8 + 2 * l + S.half];
        mk[l] = (uint64_t)v.x | (uint64_t)v.y << 32;
      }
    }
    // dpre1..4: four K-blocked (128, capacity) matrices (layer l at dpre + l * L); dead lanes
    // of the tile (mask 0) write zeros, read by the dW GEMMs' last K tile
    __half* dp = s < capacity ? dpre + kb_col(s, 128) : nullptr;
    const int64_t L = 128 * capacity;
    ts_layer(S, smem + t5, 16, 128);  // dh4 = d_o . W5
    ts_bwd_mask128(S, mk[3], dp ? dp + 3 * L : nullptr, kKbLd);
    ts_layer(S, smem + t4, 128, 128);  // dh3 = dpre4 . W4
    ts_bwd_mask128(S, mk[2], dp ? dp + 2 * L : nullptr, kKbLd);
    ts_layer(S, smem + t3, 128, 128);  // dh2 = dpre3 . W3
    ts_bwd_mask128(S, mk[1], dp ? dp + L : nullptr, kKbLd);
    ts_layer(S, smem + t2, 128, 128);  // dh1 = dpre2 . W2
    ts_bwd_mask128(S, mk[0], dp, kKbLd);
    ts_layer(S, smem + t1, 128, 32);  // dL/dfeat = dpre1 . W1x
    if (S.half == 0) {
      float dfx[32];
      tc::tmem_ld32(S.d, dfx);
      if (live) {
        float4* d = reinterpret_cast<float4*>(d_dfeat + s * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = make_float4(dfx[4 * q], dfx[4 * q + 1], dfx[4 * q + 2], dfx[4 * q + 3]);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem_base);
}

// Canonical hash backward that also returns the spatial gradient of the
// positions (carried into DeformNet): per level, the 8 corner entries are
// gathered and dL/dx_a = sum_l N_l sum_k (dfeat_l . t_k) dw_k/dfr_a, with
// w_k = wx wy wz (wx = fr_x or 1 - fr_x); zero on clamped axes.
template <int F, int L>
__global__ void __launch_bounds__(128) hash_bwd_dx_kernel(cf_hashgrid_desc D, const float* __restrict__ table,
                                                          const float4* __restrict__ x,
                                                          const float* __restrict__ dfeat,
                                                          const int* __restrict__ count, int64_t capacity,
                                                          float* __restrict__ grad, float4* __restrict__ dx_out) {
  const int64_t n = min((int64_t)*count, capacity);
  const uint32_t mask = (1u << D.log2_table) - 1u;
  // warp-uniform trip count (the coarse-level scatter is warp-cooperative)
  for (int64_t s0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); s0 < n;
       s0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = s0 + (threadIdx.x & 31);
    const float4 p = s < n ? x[s] : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool valid = p.w > 0.0f;
    if (s < n && !valid) dx_out[s] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!__any_sync(0xffffffffu, valid)) continue;
    const float q[3] = {p.x, p.y, p.z};
    float pc[3], inside[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      pc[a] = fminf(fmaxf(q[a], 0.f), 1.f);
      inside[a] = (q[a] >= 0.f && q[a] <= 1.f) ? 1.f : 0.f;
    }
    const float* g = dfeat + (valid ? s : 0) * (L * F);
    float dx[3] = {0.f, 0.f, 0.f};
#pragma unroll 2
    for (int l = 0; l < L; ++l) {
      const int N = D.resolution[l];
      const float sc = (float)N;
      const float pos[3] = {f_mul(pc[0], sc), f_mul(pc[1], sc), f_mul(pc[2], sc)};
      uint32_t gi[3];
      float fr[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int v = (int)floorf(pos[a]);
        v = v > N - 1 ? N - 1 : v;
        gi[a] = (uint32_t)v;
        fr[a] = f_sub(pos[a], (float)v);
      }
      const uint32_t stride = (uint32_t)N + 1u;
      const bool dense = D.dense[l] != 0;
      float gl[F];
#pragma unroll
      for (int f = 0; f < F; ++f) gl[f] = g[l * F + f];
      const float* tb = table + D.offset[l] * F;  // the values the forward interpolated
      float dl[3] = {0.f, 0.f, 0.f};
      uint32_t idx[8];
      float v[8][F];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t cx = gi[0] + (k & 1), cy = gi[1] + ((k >> 1) & 1), cz = gi[2] + ((k >> 2) & 1);
        idx[k] = dense ? (cx + cy * stride + cz * stride * stride)
                       : ((cx ^ (cy * 2654435761u) ^ (cz * 805459861u)) & mask);
        const float wx = (k & 1) ? fr[0] : f_sub(1.f, fr[0]);
        const float wy = (k & 2) ? fr[1] : f_sub(1.f, fr[1]);
        const float wz = (k & 4) ? fr[2] : f_sub(1.f, fr[2]);
        const float w = f_mul(f_mul(wx, wy), wz);
#pragma unroll
        for (int f = 0; f < F; ++f) v[k][f] = w * gl[f];
        float tv[F];
        ld_entry<F>(tb, idx[k], tv);
        float a = 0.f;  // dfeat_l . t_k
#pragma unroll
        for (int f = 0; f < F; ++f) a += gl[f] * tv[f];
        dl[0] += a * ((k & 1) ? 1.f : -1.f) * wy * wz;
        dl[1] += a * ((k & 2) ? 1.f : -1.f) * wx * wz;
        dl[2] += a * ((k & 4) ? 1.f : -1.f) * wx * wy;
      }
      level_scatter<F>(valid, gi, idx, v, grad + D.offset[l] * F);
#pragma unroll
      for (int a = 0; a < 3; ++a) dx[a] += sc * dl[a];
    }
    if (valid) dx_out[s] = make_float4(dx[0] * inside[0], dx[1] * inside[1], dx[2] * inside[2], 0.f);
  }
}

// ---------------------------------------------------------------- density grid (occupancy refresh)
// Occupancy from the trained density (K12; the SPEC leaves ray-marching acceleration
// open): per cell of a res^3 grid over the field's unit cube, the E_g
// density logit g0 (sigma = exp(g0)) at the cell centre u = (i + 0.5) / res (fp32 of
// the float64 quotient), hash features exactly as hash_features, the MLP in fp32 with
// un-contracted sequential sums (a_j = sum_i W1[j][i] f_i in i order, then
// g0 = sum_j W2[0][j] relu(a_j) in j order). Kept as a log-density with a max-decay
// update g = max(g + log_decay, g0) (an EMA of the max density in log space), the
// cell is occupied when g > log_threshold. Every operation is an exact fp32 op, so
// the oracle restates it bit for bit. One warp = 32 consecutive z cells = one word.
__global__ void __launch_bounds__(256) density_grid_kernel(cf_hashgrid_desc D, const float* __restrict__ table,
                                                           const float* __restrict__ W1, const float* __restrict__ W2,
                                                           int res, float log_decay, float log_thr,
                                                           float* __restrict__ logits, uint32_t* __restrict__ raw) {
  __shared__ float sW1[64 * 32], sW2[64];
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) sW1[i] = W1[i];
  if (threadIdx.x < 64) sW2[threadIdx.x] = W2[threadIdx.x];
  __syncthreads();
  const int64_t total = (int64_t)res * res * res;
  const double inv = 1.0 / (double)res;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c - (threadIdx.x & 31) < total;
       c += (int64_t)gridDim.x * blockDim.x) {
    bool on = false;
    if (c < total) {
      const int64_t x = c / ((int64_t)res * res), y = (c / res) % res, z = c % res;
      const float ux = __double2float_rn(((double)x + 0.5) * inv), uy = __double2float_rn(((double)y + 0.5) * inv),
                  uz = __double2float_rn(((double)z + 0.5) * inv);
      float f[32];
      hash_features<2, 16, 4, float>(D, table, ux, uy, uz, f);
      float g0 = 0.0f;
      for (int j = 0; j < 64; ++j) {
        float a = f_mul(sW1[j * 32], f[0]);
#pragma unroll
        for (int i = 1; i < 32; ++i) a = f_add(a, f_mul(sW1[j * 32 + i], f[i]));
        const float h = fmaxf(a, 0.0f);
        g0 = j == 0 ? f_mul(sW2[0], h) : f_add(g0, f_mul(sW2[j], h));
      }
      const float g = fmaxf(f_add(logits[c], log_decay), g0);
      logits[c] = g;
      on = g > log_thr;
    }
    const unsigned word = __ballot_sync(0xffffffffu, on);
    if ((threadIdx.x & 31) == 0 && c < total) raw[c >> 5] = word;
  }
}

// Chebyshev (box) dilation of a bit grid by r cells along one axis (0 = z, within and
// across the 32-cell words; 1 = y; 2 = x), no wrap. res % 32 == 0.
__global__ void bits_dilate_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int res, int axis,
                                   int r) {
  const int wpr = res / 32;  // words per z row
  const int64_t words = (int64_t)res * res * wpr;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int zw = (int)(w % wpr);
    const int64_t row = w / wpr;  // x * res + y
    const int y = (int)(row % res), x = (int)(row / res);
    uint32_t v = src[w];
    if (axis == 0) {
      const uint64_t lo = zw > 0 ? src[w - 1] : 0u, hi = zw + 1 < wpr ? src[w + 1] : 0u;
      const uint64_t cur = src[w];
      for (int k = 1; k <= r; ++k) {
        // bit b of the result sees bits b - k (from lower z) and b + k (from higher z)
        v |= (uint32_t)((cur << k) | (lo >> (32 - k)));
        v |= (uint32_t)((cur >> k) | (hi << (32 - k)));
      }
    } else {
      for (int k = -r; k <= r; ++k) {
        const int yy = axis == 1 ? y + k : y, xx = axis == 2 ? x + k : x;
        if (k == 0 || yy < 0 || yy >= res || xx < 0 || xx >= res) continue;
        v |= src[((int64_t)xx * res + yy) * wpr + zw];
      }
    }
    dst[w] = v;
  }
}

// the DeformNet kernel's L2 prefetch of the canonical table (CF_L2_PREFETCH=1): off by
// default — measured, the hash stage after it gains nothing (it is L1-request bound)
// and the kernel loses ~4 us issuing it
bool l2_prefetch_on() {
  static const bool on = [] { const char* e = getenv("CF_L2_PREFETCH"); return e && atoi(e) != 0; }();
  return on;
}

unsigned persistent_grid(int64_t capacity, int slots) {
  const int64_t tiles = (capacity + 127) / 128;
  int64_t g = (tiles + slots - 1) / slots;
  if (g > cf::sm_count()) g = cf::sm_count();
  return (unsigned)(g < 1 ? 1 : g);
}

// Scratch of the training forward (cf_field_desc.train), S = capacity: the fp16
// features feature-major for the backward and the dW GEMMs, then the fp32 working
// set of the 32-bit forward. Offsets in bytes; S % 8 == 0 keeps every block 16-byte
// aligned (TMA rows, float4).
struct TrainLayout {
  int64_t cfeat16, dfeat16, xc, dfeat32, cfeat32, total;
};
inline TrainLayout train_layout(int64_t S) {
  TrainLayout L;
  L.cfeat16 = 0;               // (32, S) fp16 canonical features
  L.dfeat16 = S * 64;          // (33, S) fp16 deformation features + a row of ones
  L.xc = L.dfeat16 + S * 66;   // (S) float4 canonical positions
  L.dfeat32 = L.xc + S * 16;   // (S, 32) fp32 deformation features
  L.cfeat32 = L.dfeat32 + S * 128;  // (S, 32) fp32 canonical features
  L.total = L.cfeat32 + S * 128;
  return L;
}

// "fp32" precision mode of cf_field_stage: fp32 tables (the deformation grid's fp32
// parameters, not its fp16 copy), fp32 features, split-fp16 MLPs
int field_stage_precise(const cf_field_desc* FD, const cf_march_out* S, const double* dirs, const float* xu_f,
                        float* out_f, void* scratch, int stage, cudaStream_t st) {
  auto run = [&](int s) { return stage < 0 || stage == s; };
  const int64_t cap = S->capacity;
  if (FD->train) {
    // training forward at 32-bit semantics (fp32 tables and features, split-fp16 MMAs):
    // xc, sigma and rgb are the 32-bit field's (the L1 depth term's sign and the
    // spatial gradient dL/dxc are evaluated where the SPEC's field is), plus the fp16
    // feature-major saves the fp16 backward and the dW GEMMs consume (train_layout)
    if (cap % 8 != 0) return cf::fail(CF_E_BAD_ARG, "cf_field_forward: training needs capacity % 8 == 0");
    if (FD->has_deform && (!FD->save_h || !FD->save_o || !FD->save_mask))
      return cf::fail(CF_E_BAD_ARG, "cf_field_forward: training the human field needs save_h, save_o, save_mask");
    const TrainLayout TL = train_layout(cap);
    uint8_t* sb = static_cast<uint8_t*>(scratch);
    __half* cfeat16 = reinterpret_cast<__half*>(sb + TL.cfeat16);
    float4* cfeat32 = reinterpret_cast<float4*>(sb + TL.cfeat32);
    const float4* xu = reinterpret_cast<const float4*>(xu_f);
    const float4* xcan = xu;
    const unsigned hgrid = cf::grid_for(cap, 128, 16);
    if (FD->has_deform) {
      float4* xc = reinterpret_cast<float4*>(sb + TL.xc);
      float4* dfeat32 = reinterpret_cast<float4*>(sb + TL.dfeat32);
      if (run(0))
        cf::launch_pdl(hash_f16_kernel<4, 8, 2, 1, float, true>, hgrid, 128, 0, st, FD->dgrid,
                       reinterpret_cast<const float*>(FD->dtable), xu, S->counters, cap,
                       reinterpret_cast<uint4*>(dfeat32));
      if (run(1)) {
        const int smem = 2 * kDeformW;
        CF_CHECK_CUDA(cudaFuncSetAttribute(deform_mlp_prec_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cf::launch_pdl(deform_mlp_prec_kernel<true>, persistent_grid(cap, kPrecDeformSlots),
                       kPrecDeformSlots * kPrecDeformThreads, smem, st, FD->wblob, FD->wblob_lo, FD->dbias,
                       FD->delta_scale, FD->inv_side, xu, static_cast<const float4*>(dfeat32), S->counters, cap, xc,
                       reinterpret_cast<__half*>(FD->save_h), reinterpret_cast<float4*>(FD->save_o), FD->save_mask,
                       reinterpret_cast<__half*>(sb + TL.dfeat16),
                       static_cast<const uint8_t*>(nullptr), (int64_t)0, cf_hashgrid_desc{},
                       static_cast<const float*>(nullptr));
      }
      xcan = xc;
    }
    if (run(2)) {
      if (FD->has_deform)
        cf::launch_pdl(hash_f16_kernel<2, 16, 4, 1, float, true>, hgrid, 128, 0, st, FD->cgrid,
                       reinterpret_cast<const float*>(FD->ctable), xcan, S->counters, cap,
                       reinterpret_cast<uint4*>(cfeat32));
      else
        cf::launch_pdl(hash_f16_kernel<2, 16, 4, 4, float, true>, cf::grid_for(cap * 4, 128, 16), 128, 0, st,
                       FD->cgrid, reinterpret_cast<const float*>(FD->ctable), xcan, S->counters, cap,
                       reinterpret_cast<uint4*>(cfeat32));
    }
    if (run(3)) {
      const int off = FD->has_deform ? kDeformW : 0;
      const int csmem = 2 * kColorW;
      CF_CHECK_CUDA(cudaFuncSetAttribute(color_mlp_prec_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem));
      cf::launch_pdl(color_mlp_prec_kernel<0>, persistent_grid(cap, kColorPrecSlots), kColorPrecSlots * kSlotThreads,
                     csmem, st, FD->wblob + off, FD->wblob_lo + off, xu, static_cast<const float4*>(cfeat32),
                     S->records, dirs, S->counters, cap, reinterpret_cast<float4*>(out_f), cfeat16, cf_hashgrid_desc{},
                     static_cast<const float*>(nullptr));
    }
    return cf::check_launch("cf_field_forward (training)");
  }
  if (FD->save_h) return cf::fail(CF_E_BAD_ARG, "cf_field_forward: saves are a training-mode (train = 1) output");
  const float4* xu = reinterpret_cast<const float4*>(xu_f);
  float4* out = reinterpret_cast<float4*>(out_f);
  float4* cfeat = reinterpret_cast<float4*>(scratch);  // (cap, 32) fp32
  const float4* xcan = xu;
  const unsigned hgrid = cf::grid_for(cap, 128, 16);
  if (FD->has_deform) {
    float4* dfeat = cfeat + cap * 8;
    float4* xc = dfeat + cap * 8;
    // the deformation-grid hash inside DeformNet (render, split_stages = 0): each thread
    // looks up its quarter's 2 levels at the tile head (2 levels of gathers in flight)
    // instead of reading the 128 B/sample the hash kernel wrote — hash 46 + DeformNet 82
    // -> 121 us serialised, 0.403 -> 0.391 ms per frame; bit-identical to the split path
    const int dfused = FD->split_stages ? 0 : 2;
    if (run(0) && !dfused)
      cf::launch_pdl(hash_f16_kernel<4, 8, 2, 2, float, true>, cf::grid_for(cap * 2, 128, 16), 128, 0, st, FD->dgrid,
                     reinterpret_cast<const float*>(FD->dtable), xu, S->counters, cap, reinterpret_cast<uint4*>(dfeat));
    if (run(1)) {
      const int smem = 2 * kDeformW;
      auto kern = dfused ? deform_mlp_prec_kernel<false, 2> : deform_mlp_prec_kernel<false, 0>;
      CF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      cf::launch_pdl(kern, persistent_grid(cap, kPrecDeformSlots),
                     kPrecDeformSlots * kPrecDeformThreads, smem, st, FD->wblob, FD->wblob_lo, FD->dbias,
                     FD->delta_scale, FD->inv_side, xu, static_cast<const float4*>(dfeat), S->counters, cap, xc,
                     static_cast<__half*>(nullptr), static_cast<float4*>(nullptr), static_cast<uint32_t*>(nullptr),
                     static_cast<__half*>(nullptr),
                     l2_prefetch_on() ? static_cast<const uint8_t*>(FD->ctable) : nullptr,
                     (int64_t)(FD->cgrid.offset[FD->cgrid.n_levels] * FD->cgrid.n_features * 4), FD->dgrid,
                     reinterpret_cast<const float*>(FD->dtable));
    }
    xcan = xc;
  }
  // the canonical hash fused into the E_g / E_c kernel (kHashCH = 4 levels in flight):
  // each slot's gathers overlap the other slots' MMAs and epilogues, and the 128 B/sample
  // feature round trip through HBM goes away (hash 76 + colour 37 -> 84 us after an L2
  // flush); output bit-identical to the split stages (test_fused_color_kernel_equals_stages)
  const int fused = FD->split_stages ? 0 : 4;
  if (run(2) && !fused) {
    if (FD->has_deform)
      cf::launch_pdl(hash_f16_kernel<2, 16, 4, 1, float, true>, hgrid, 128, 0, st, FD->cgrid,
                     reinterpret_cast<const float*>(FD->ctable), xcan, S->counters, cap, reinterpret_cast<uint4*>(cfeat));
    else
      cf::launch_pdl(hash_f16_kernel<2, 16, 4, 4, float, true>, cf::grid_for(cap * 4, 128, 16), 128, 0, st, FD->cgrid,
                     reinterpret_cast<const float*>(FD->ctable), xcan, S->counters, cap,
                     reinterpret_cast<uint4*>(cfeat));
  }
  if (run(3)) {
    const int off = FD->has_deform ? kDeformW : 0;
    const int csmem = 2 * kColorW;
    if (fused) {
      auto kern = color_mlp_prec_kernel<4>;
      CF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem));
      unsigned grid = persistent_grid(cap, kColorPrecSlots);
      // a field on a side stream (the render's object field) leaves the other SMs to the
      // kernels beside it (its slots take tiles from the ticket: fewer CTAs only lengthen it)
      if (FD->max_ctas > 0) grid = std::min(grid, (unsigned)FD->max_ctas);
      cf::launch_pdl(kern, grid, kColorPrecSlots * kSlotThreads, csmem, st,
                     FD->wblob + off, FD->wblob_lo + off, xcan, static_cast<const float4*>(cfeat), S->records, dirs,
                     S->counters, cap, out, static_cast<__half*>(nullptr), FD->cgrid,
                     reinterpret_cast<const float*>(FD->ctable));
    } else {
      CF_CHECK_CUDA(cudaFuncSetAttribute(color_mlp_prec_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem));
      cf::launch_pdl(color_mlp_prec_kernel<0>, persistent_grid(cap, kColorPrecSlots), kColorPrecSlots * kSlotThreads,
                     csmem, st, FD->wblob + off, FD->wblob_lo + off, xu, static_cast<const float4*>(cfeat),
                     S->records, dirs, S->counters, cap, out, static_cast<__half*>(nullptr), cf_hashgrid_desc{},
                     static_cast<const float*>(nullptr));
    }
  }
  return cf::check_launch("cf_field_forward (precise)");
}

}  // namespace

extern "C" {

int cf_density_grid_update(const cf_hashgrid_desc* G, const float* table, const float* W1, const float* W2, int res,
                           float log_decay, float log_threshold, int dilate, float* logits, uint32_t* bits,
                           uint32_t* scratch, void* stream) {
  if (!G || !table || !W1 || !W2 || res < 32 || res % 32 != 0 || dilate < 0 || dilate > 32 || !logits || !bits ||
      !scratch || G->n_features != 2 || G->n_levels != 16)
    return cf::fail(CF_E_BAD_ARG, "cf_density_grid_update: bad args (16 x F2 grid, res % 32 == 0)");
  cudaStream_t st = cf::as_stream(stream);
  const int64_t total = (int64_t)res * res * res, words = total / 32;
  uint32_t* raw = dilate > 0 ? scratch : bits;
  density_grid_kernel<<<cf::grid_for(total, 256, 8), 256, 0, st>>>(*G, table, W1, W2, res, log_decay, log_threshold,
                                                                   logits, raw);
  if (dilate > 0) {
    const unsigned g = cf::grid_for(words, 256, 8);
    bits_dilate_kernel<<<g, 256, 0, st>>>(scratch, bits, res, 0, dilate);
    bits_dilate_kernel<<<g, 256, 0, st>>>(bits, scratch, res, 1, dilate);
    bits_dilate_kernel<<<g, 256, 0, st>>>(scratch, bits, res, 2, dilate);
  }
  return cf::check_launch("cf_density_grid_update");
}

int cf_field_train_layout(int64_t capacity, int64_t* offsets) {
  if (capacity < 0 || !offsets) return cf::fail(CF_E_BAD_ARG, "cf_field_train_layout: bad args");
  const TrainLayout L = train_layout(capacity);
  offsets[0] = L.cfeat16;
  offsets[1] = L.dfeat16;
  offsets[2] = L.xc;
  offsets[3] = L.dfeat32;
  offsets[4] = L.cfeat32;
  offsets[5] = L.total;
  return CF_OK;
}

int cf_field_scratch_bytes(const cf_field_desc* FD, int64_t capacity, int64_t* bytes) {
  if (!FD || !bytes || capacity < 0) return cf::fail(CF_E_BAD_ARG, "cf_field_scratch_bytes: bad args");
  // cfeat (64 B fp16 / 128 B fp32) [+ dfeat (same) + xc (16 B)] per sample
  const int64_t feat = FD->precise ? 128 : 64;
  *bytes = capacity * (feat + (FD->has_deform ? feat + 16 : 0));
  if (FD->train) *bytes = train_layout(capacity).total;
  return CF_OK;
}

int cf_field_forward(const cf_field_desc* FD, const cf_march_out* S, const double* dirs, const float* xu_f,
                     float* out_f, void* scratch, void* stream) {
  return cf_field_stage(FD, S, dirs, xu_f, out_f, scratch, -1, stream);
}

int cf_color_backward(const cf_field_desc* FD, const uint8_t* wt_blob, const cf_march_out* S, const double* dirs,
                      const float* xu, const float* grad_out, const void* scratch, const cf_color_bwd_io* io,
                      void* stream) {
  if (!FD || !wt_blob || !S || !dirs || !xu || !grad_out || !scratch || !io || !io->dfeat)
    return cf::fail(CF_E_BAD_ARG, "cf_color_backward: bad args");
  if (!FD->train) return cf::fail(CF_E_BAD_ARG, "cf_color_backward: needs the training forward's scratch (train = 1)");
  const int64_t cap = S->capacity;
  if (cap == 0) return CF_OK;
  ColorBwdIO o{reinterpret_cast<__half*>(io->h1),  reinterpret_cast<__half*>(io->cin),
               reinterpret_cast<__half*>(io->c1),  reinterpret_cast<__half*>(io->c2),
               reinterpret_cast<__half*>(io->d_o), reinterpret_cast<__half*>(io->dc2),
               reinterpret_cast<__half*>(io->dc1), reinterpret_cast<__half*>(io->dg),
               reinterpret_cast<__half*>(io->dh1), io->dfeat};
  const int smem = kColorW + kColorWT + kBwdSlots * kBwdA;
  CF_CHECK_CUDA(cudaFuncSetAttribute(color_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const uint8_t* cw = FD->wblob + (FD->has_deform ? kDeformW : 0);
  color_bwd_kernel<<<persistent_grid(cap, kBwdSlots), kBwdSlots * kSlotThreads, smem, cf::as_stream(stream)>>>(
      cw, wt_blob, reinterpret_cast<const float4*>(xu),
      reinterpret_cast<const float4*>(static_cast<const uint8_t*>(scratch) + train_layout(cap).cfeat32), S->records, dirs,
      reinterpret_cast<const float4*>(grad_out), S->counters, cap, o);
  return cf::check_launch("cf_color_backward");
}

int cf_field_hash_backward(const cf_field_desc* FD, const cf_march_out* S, const float* xu, const void* scratch,
                           const float* dfeat, float* table_grad, float* dx_out, void* stream) {
  if (!FD || !S || !xu || !scratch || !dfeat || !table_grad || (dx_out && !FD->ctable))
    return cf::fail(CF_E_BAD_ARG, "cf_field_hash_backward: bad args");
  const int64_t cap = S->capacity;
  if (cap == 0) return CF_OK;
  // the canonical grid saw xc (human: after DeformNet, stored in scratch) or xu (object)
  const float4* x = reinterpret_cast<const float4*>(xu);
  if (!FD->train) return cf::fail(CF_E_BAD_ARG, "cf_field_hash_backward: needs the training forward's scratch");
  if (FD->has_deform)
    x = reinterpret_cast<const float4*>(static_cast<const uint8_t*>(scratch) + train_layout(cap).xc);
  if (dx_out)
    hash_bwd_dx_kernel<2, 16><<<cf::grid_for(cap, 128, 16), 128, 0, cf::as_stream(stream)>>>(
        FD->cgrid, reinterpret_cast<const float*>(FD->ctable), x, dfeat, S->counters, cap, table_grad,
        reinterpret_cast<float4*>(dx_out));
  else
    hash_bwd_kernel<2, 16><<<cf::grid_for(cap, 128, 16), 128, 0, cf::as_stream(stream)>>>(
        FD->cgrid, x, dfeat, S->counters, cap, table_grad);
  return cf::check_launch("cf_field_hash_backward");
}

int cf_deform_backward(const cf_field_desc* FD, const uint8_t* wt_blob, const cf_march_out* S, const float* xu,
                       const float* dxc, const cf_deform_bwd_io* io, void* stream) {
  if (!FD || !FD->has_deform || !wt_blob || !S || !xu || !dxc || !io || !io->save_mask || !io->save_o || !io->d_o ||
      !io->dpre || !io->d_dfeat)
    return cf::fail(CF_E_BAD_ARG, "cf_deform_backward: bad args");
  const int64_t cap = S->capacity;
  if (cap == 0) return CF_OK;
  const int smem = kDeformWT + kDeformA;  // weights + the SS slot's A buffer
  CF_CHECK_CUDA(cudaFuncSetAttribute(deform_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  deform_bwd_kernel<<<persistent_grid(cap, kDBwdSlots), kDBwdSlots * kDeformSlotThreads, smem,
                      cf::as_stream(stream)>>>(
      wt_blob, FD->delta_scale, FD->inv_side, reinterpret_cast<const float4*>(xu),
      reinterpret_cast<const float4*>(dxc), reinterpret_cast<const uint2*>(io->save_mask),
      reinterpret_cast<const float4*>(io->save_o), S->counters, cap, reinterpret_cast<__half*>(io->d_o),
      reinterpret_cast<__half*>(io->dpre), io->d_dfeat);
  return cf::check_launch("cf_deform_backward");
}

int cf_deform_hash_backward(const cf_field_desc* FD, const cf_march_out* S, const float* xu, const float* d_dfeat,
                            float* table_grad, void* stream) {
  if (!FD || !FD->has_deform || !S || !xu || !d_dfeat || !table_grad)
    return cf::fail(CF_E_BAD_ARG, "cf_deform_hash_backward: bad args");
  const int64_t cap = S->capacity;
  if (cap == 0) return CF_OK;
  hash_bwd_kernel<4, 8><<<cf::grid_for(cap, 128, 16), 128, 0, cf::as_stream(stream)>>>(
      FD->dgrid, reinterpret_cast<const float4*>(xu), d_dfeat, S->counters, cap, table_grad);
  return cf::check_launch("cf_deform_hash_backward");
}

int cf_field_stage(const cf_field_desc* FD, const cf_march_out* S, const double* dirs, const float* xu_f,
                   float* out_f, void* scratch, int stage, void* stream) {
  auto run = [&](int s) { return stage < 0 || stage == s; };
  if (!FD || !S || !FD->wblob || !FD->ctable || !scratch || (FD->has_deform && (!FD->dtable || !FD->dbias)))
    return cf::fail(CF_E_BAD_ARG, "cf_field_forward: bad args");
  if (FD->cgrid.n_levels != 16 || FD->cgrid.n_features != 2 ||
      (FD->has_deform && (FD->dgrid.n_levels != 8 || FD->dgrid.n_features != 4)))
    return cf::fail(CF_E_BAD_ARG, "cf_field_forward: grids must be 16x F2 (canonical) and 8x F4 (deform)");
  if (FD->w_bytes != (FD->has_deform ? kDeformW : 0) + kColorW)
    return cf::fail(CF_E_BAD_ARG, "cf_field_forward: weight blob size mismatch");
  if ((FD->precise || FD->train) && !FD->wblob_lo)
    return cf::fail(CF_E_BAD_ARG, "cf_field_forward: precise / training mode needs wblob_lo");
  cudaStream_t st = cf::as_stream(stream);
  const int64_t cap = S->capacity;
  if (cap == 0) return CF_OK;
  if (FD->precise || FD->train) return field_stage_precise(FD, S, dirs, xu_f, out_f, scratch, stage, st);
  const float4* xu = reinterpret_cast<const float4*>(xu_f);
  float4* out = reinterpret_cast<float4*>(out_f);
  uint4* cfeat = reinterpret_cast<uint4*>(scratch);
  const float4* xcan = xu;
  const unsigned hgrid = cf::grid_for(cap, 128, 16);
  if (FD->has_deform) {
    uint4* dfeat = cfeat + cap * 4;
    float4* xc = reinterpret_cast<float4*>(dfeat + cap * 4);
    if (run(0))
      cf::launch_pdl(hash_f16_kernel<4, 8, 2, 1, __half>, hgrid, 128, 0, st, FD->dgrid, reinterpret_cast<const __half*>(FD->dtable), xu, S->counters, cap, dfeat);
    if (run(1)) {
      const int smem = kDeformW + kDeformA;
      CF_CHECK_CUDA(cudaFuncSetAttribute(deform_mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      cf::launch_pdl(deform_mlp_kernel, persistent_grid(cap, kDeformSlots), kDeformSlots * kDeformSlotThreads, smem,
                     st, FD->wblob, FD->dbias, FD->delta_scale, FD->inv_side, xu, dfeat, S->counters, cap, xc);
    }
    xcan = xc;
  }
  if (run(2)) {
    if (FD->has_deform)
      cf::launch_pdl(hash_f16_kernel<2, 16, 4, 1, float>, hgrid, 128, 0, st, FD->cgrid, reinterpret_cast<const float*>(FD->ctable), xcan, S->counters, cap,
                     cfeat);
    else  // object field: few samples
      cf::launch_pdl(hash_f16_kernel<2, 16, 4, 4, float>, cf::grid_for(cap * 4, 128, 16), 128, 0, st, FD->cgrid, reinterpret_cast<const float*>(FD->ctable),
                     xcan, S->counters, cap, cfeat);
  }
  if (run(3)) {
    const int csmem = kColorW;
    const uint8_t* cw = FD->wblob + (FD->has_deform ? kDeformW : 0);
    cf::launch_pdl(color_mlp_kernel, persistent_grid(cap, kColorTsSlots), kColorTsSlots * kSlotThreads, csmem, st, cw, xu, cfeat, S->records, dirs, S->counters, cap, out);
  }
  return cf::check_launch("cf_field_forward");
}

}  // extern "C"
