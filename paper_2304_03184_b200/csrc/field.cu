// Fused radiance-field evaluation of compacted samples, one persistent CTA per
// SM, two 128-sample slots (4 warps each). Per slot and tile, everything stays
// on chip: hash-grid gathers (CUDA cores, L2-resident tables) write fp16
// features straight into the UMMA A-operand buffer in shared memory, each MLP
// layer is a chain of tcgen05.mma (M=128, N<=128, K=16 steps) accumulating in
// TMEM, and the epilogue (TMEM -> registers -> bias/ReLU -> fp16 -> smem) feeds
// the next layer. Weights of all networks (128 KB fp16) are loaded into smem
// once per CTA.
//
// Human field:
//   x   = canonicalised sample (unit cube), from cf_human_canon
//   dv  = 0.05 * tanh(DeformNet(hash_d(x)))          32 -> 128 x4 -> 3 (theta folded in layer-1 bias)
//   xc  = x + dv / side
//   g   = E_g(hash_c(xc))                             32 -> 64 -> 16 ; sigma = exp(g0), geo = g1..15
//   rgb = sigmoid(E_c([geo, SH4(dir)]))               32 -> 64 -> 64 -> 3
// Object field: the same without the deformation stage.
#include "common.cuh"
#include "tc.cuh"

namespace {

constexpr int kSlotThreads = 128;
constexpr int kSlots = 2;
constexpr int kABytes = 128 * 128 * 2;  // A buffer per slot (K <= 128)

struct Slot {
  uint8_t* abuf;
  uint8_t* w_s;
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
  if (S.r == 0) {
    tc::fence_after();
    tc::issue_layer(S.tmem, S.abuf, S.w_s + w_off, K, N);
    tc::mma_commit(S.bar);
  }
  tc::bar_wait(S.bar, S.phase);
  S.phase ^= 1u;
  tc::fence_after();
}

// hidden-layer epilogue: (+bias) ReLU -> fp16 -> A buffer with K = N
__device__ __forceinline__ void relu_to_abuf(Slot& S, int N, const float* bias) {
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(S.tmem_row + (uint32_t)c0, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaxf(bias ? v[i] + bias[c0 + i] : v[i], 0.0f);
    tc::st_row8(S.abuf, S.r, c0, N, v);
    tc::st_row8(S.abuf, S.r, c0 + 8, N, v + 8);
  }
}

template <int F>
__device__ __forceinline__ void hash_features(const cf_hashgrid_desc& D, const float* __restrict__ table, float x,
                                              float y, float z, float* feat) {
  x = fminf(fmaxf(x, 0.0f), 1.0f);
  y = fminf(fmaxf(y, 0.0f), 1.0f);
  z = fminf(fmaxf(z, 0.0f), 1.0f);
  const uint32_t mask = (1u << D.log2_table) - 1u;
#pragma unroll 1
  for (int l = 0; l < D.n_levels; ++l) {
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
    const float* base = table + D.offset[l] * F;
    float t[8][F];
    float w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t cx = g[0] + (k & 1), cy = g[1] + ((k >> 1) & 1), cz = g[2] + ((k >> 2) & 1);
      const uint32_t idx =
          dense ? (cx + cy * stride + cz * stride * stride) : ((cx ^ (cy * 2654435761u) ^ (cz * 805459861u)) & mask);
      if constexpr (F == 2) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(base) + idx);
        t[k][0] = v.x;
        t[k][1] = v.y;
      } else {
        const float4 v = __ldg(reinterpret_cast<const float4*>(base) + idx);
        t[k][0] = v.x;
        t[k][1] = v.y;
        t[k][2] = v.z;
        t[k][3] = v.w;
      }
      const float wx = (k & 1) ? fr[0] : f_sub(1.0f, fr[0]);
      const float wy = (k & 2) ? fr[1] : f_sub(1.0f, fr[1]);
      const float wz = (k & 4) ? fr[2] : f_sub(1.0f, fr[2]);
      w[k] = f_mul(f_mul(wx, wy), wz);
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
      float acc = f_mul(w[0], t[0][f]);
#pragma unroll
      for (int k = 1; k < 8; ++k) acc = f_add(acc, f_mul(w[k], t[k][f]));
      feat[l * F + f] = acc;
    }
  }
}

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

struct Offsets {
  int d[5], g[2], c[3];
};

__global__ void __launch_bounds__(kSlots* kSlotThreads, 1)
    field_kernel(cf_field_desc FD, Offsets W, const double* __restrict__ dirs, const uint32_t* __restrict__ records,
                 const int* __restrict__ count, int64_t capacity, const float4* __restrict__ xu,
                 float4* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[kSlots];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid * 16; i < FD.w_bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = *reinterpret_cast<const uint4*>(FD.wblob + i);
  if (tid == 0) {
    for (int s = 0; s < kSlots; ++s) tc::bar_init(&mbar[s], 1);
    tc::bar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<kSlots * 128>(&tmem_base);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  Slot S;
  S.slot = tid / kSlotThreads;
  S.r = tid % kSlotThreads;
  S.w_s = smem;
  S.abuf = smem + ((FD.w_bytes + 1023) / 1024) * 1024 + S.slot * kABytes;
  S.bar = &mbar[S.slot];
  S.tmem = tmem_base + (uint32_t)(S.slot * 128);
  S.tmem_row = S.tmem + ((uint32_t)((warp % 4) * 32) << 16);
  S.phase = 0;

  const int64_t n = min((int64_t)*count, capacity);
  const int64_t n_tiles = (n + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * kSlots + S.slot; tile < n_tiles; tile += (int64_t)gridDim.x * kSlots) {
    const int64_t s = tile * 128 + S.r;
    const bool live = s < n;
    float4 x = live ? xu[s] : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool valid = live && x.w > 0.0f;
    float feat[32];
    if (FD.has_deform) {
      if (valid) hash_features<4>(FD.dgrid, FD.dtable, x.x, x.y, x.z, feat);
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (!valid) feat[i] = 0.0f;
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 8) tc::st_row8(S.abuf, S.r, k0, 32, feat + k0);
      run_layer(S, W.d[0], 32, 128);
      relu_to_abuf(S, 128, FD.dbias);
      for (int l = 1; l < 4; ++l) {
        run_layer(S, W.d[l], 128, 128);
        relu_to_abuf(S, 128, nullptr);
      }
      run_layer(S, W.d[4], 128, 16);
      float v[16];
      tc::tmem_ld16(S.tmem_row, v);
      x.x = f_add(x.x, f_mul(FD.delta_scale * tanhf(v[0]), FD.inv_side));
      x.y = f_add(x.y, f_mul(FD.delta_scale * tanhf(v[1]), FD.inv_side));
      x.z = f_add(x.z, f_mul(FD.delta_scale * tanhf(v[2]), FD.inv_side));
    }
    if (valid) hash_features<2>(FD.cgrid, FD.ctable, x.x, x.y, x.z, feat);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!valid) feat[i] = 0.0f;
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 8) tc::st_row8(S.abuf, S.r, k0, 32, feat + k0);
    run_layer(S, W.g[0], 32, 64);
    relu_to_abuf(S, 64, nullptr);
    run_layer(S, W.g[1], 64, 16);
    float gv[16];
    tc::tmem_ld16(S.tmem_row, gv);
    const float sigma = valid ? expf(gv[0]) : 0.0f;
    // colour input: [geo(15), SH4(dir)(16), 0]
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
    run_layer(S, W.c[0], 32, 64);
    relu_to_abuf(S, 64, nullptr);
    run_layer(S, W.c[1], 64, 64);
    relu_to_abuf(S, 64, nullptr);
    run_layer(S, W.c[2], 64, 16);
    float cv[16];
    tc::tmem_ld16(S.tmem_row, cv);
    if (live) {
      const float r = 1.0f / (1.0f + expf(-cv[0])), g = 1.0f / (1.0f + expf(-cv[1])),
                  b = 1.0f / (1.0f + expf(-cv[2]));
      out[s] = valid ? make_float4(sigma, r, g, b) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<kSlots * 128>(tmem_base);
}

}  // namespace

extern "C" {

int cf_field_forward(const cf_field_desc* FD, const cf_march_out* S, const double* dirs, const float* xu,
                     float* out, void* stream) {
  if (!FD || !S || !FD->wblob || !FD->ctable || (FD->has_deform && (!FD->dtable || !FD->dbias)))
    return cf::fail(CF_E_BAD_ARG, "cf_field_forward: bad args");
  if (FD->cgrid.n_levels * FD->cgrid.n_features != 32 || FD->cgrid.n_features != 2 ||
      (FD->has_deform && (FD->dgrid.n_levels * FD->dgrid.n_features != 32 || FD->dgrid.n_features != 4)))
    return cf::fail(CF_E_BAD_ARG, "cf_field_forward: grids must encode to 32 features (F=2 canonical, F=4 deform)");
  Offsets W{};
  int off = 0;
  auto take = [&](int n, int k) {
    const int o = off;
    off += n * k * 2;
    return o;
  };
  if (FD->has_deform) {
    W.d[0] = take(128, 32);
    for (int l = 1; l < 4; ++l) W.d[l] = take(128, 128);
    W.d[4] = take(16, 128);
  }
  W.g[0] = take(64, 32);
  W.g[1] = take(16, 64);
  W.c[0] = take(64, 32);
  W.c[1] = take(64, 64);
  W.c[2] = take(16, 64);
  if (off != FD->w_bytes) return cf::fail(CF_E_BAD_ARG, "cf_field_forward: weight blob size mismatch");
  const int smem = ((off + 1023) / 1024) * 1024 + kSlots * kABytes;
  CF_CHECK_CUDA(cudaFuncSetAttribute(field_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int64_t max_tiles = (S->capacity + 127) / 128;
  int64_t grid = (max_tiles + kSlots - 1) / kSlots;
  if (grid > cf::sm_count()) grid = cf::sm_count();
  if (grid < 1) return CF_OK;
  field_kernel<<<(unsigned)grid, kSlots * kSlotThreads, smem, cf::as_stream(stream)>>>(
      *FD, W, dirs, S->records, S->counters, S->capacity, reinterpret_cast<const float4*>(xu),
      reinterpret_cast<float4*>(out));
  return cf::check_launch("cf_field_forward");
}

}  // extern "C"
