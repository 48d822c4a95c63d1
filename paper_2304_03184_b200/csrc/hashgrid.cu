// Multi-resolution hash-grid encoding (SPEC nrf.hash_encode, SPEC.md:345-348,
// 363-371; hyper-parameters config.py:56-60). Level rule:
//   N_l = floor(N_min * b^l), b = exp((ln N_max - ln N_min) / (L - 1))
//   dense level  if (N_l + 1)^3 <= T : idx = x + y (N_l+1) + z (N_l+1)^2
//   hashed level otherwise          : idx = (x * 1 ^ y * 2654435761 ^ z * 805459861) mod T
//   pos = clamp(p, 0, 1) * N_l (fp32), cell = min(floor(pos), N_l - 1), frac = pos - cell
//   feature = sum over corners c = 0..7 (bit0 -> x) of (wx*wy)*wz * table[c]
// All fp32 arithmetic is un-contracted and in that fixed order, so indices are
// bit-exact and features bit-equal to the float32 numpy restatement in oracle/.
// Table layout in HBM: (entries, F) float32, level l at rows [offset_l, offset_l+size_l).
#include <cmath>

#include "common.cuh"

namespace {

struct Corner {
  uint32_t idx[8];
  float w[8];
};

__device__ __forceinline__ void level_corners(const cf_hashgrid_desc& D, int l, float px, float py, float pz,
                                              Corner& c) {
  const int N = D.resolution[l];
  const float s = (float)N;
  const float pos[3] = {f_mul(px, s), f_mul(py, s), f_mul(pz, s)};
  uint32_t g[3];
  float fr[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int gi = (int)floorf(pos[a]);
    gi = gi > N - 1 ? N - 1 : gi;
    g[a] = (uint32_t)gi;
    fr[a] = f_sub(pos[a], (float)gi);
  }
  const uint32_t mask = (1u << D.log2_table) - 1u;
  const uint32_t stride = (uint32_t)N + 1u;
  const bool dense = D.dense[l] != 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = g[0] + (k & 1), y = g[1] + ((k >> 1) & 1), z = g[2] + ((k >> 2) & 1);
    c.idx[k] = dense ? (x + y * stride + z * stride * stride) : ((x ^ (y * 2654435761u) ^ (z * 805459861u)) & mask);
    const float wx = (k & 1) ? fr[0] : f_sub(1.0f, fr[0]);
    const float wy = (k & 2) ? fr[1] : f_sub(1.0f, fr[1]);
    const float wz = (k & 4) ? fr[2] : f_sub(1.0f, fr[2]);
    c.w[k] = f_mul(f_mul(wx, wy), wz);
  }
}

__device__ __forceinline__ void load_unit(const float* p, float& x, float& y, float& z) {
  x = fminf(fmaxf(p[0], 0.0f), 1.0f);
  y = fminf(fmaxf(p[1], 0.0f), 1.0f);
  z = fminf(fmaxf(p[2], 0.0f), 1.0f);
}

template <int F>
struct Vec;
template <>
struct Vec<2> {
  using T = float2;
};
template <>
struct Vec<4> {
  using T = float4;
};

template <int F>
__device__ __forceinline__ void vacc(float* acc, float w, const typename Vec<F>::T& t, bool first) {
  const float* tv = reinterpret_cast<const float*>(&t);
#pragma unroll
  for (int f = 0; f < F; ++f) acc[f] = first ? f_mul(w, tv[f]) : f_add(acc[f], f_mul(w, tv[f]));
}

template <int F>
__global__ void __launch_bounds__(128) encode_kernel(cf_hashgrid_desc D, const float* __restrict__ table,
                                                     const float* __restrict__ pts, int64_t n,
                                                     float* __restrict__ out) {
  using VT = typename Vec<F>::T;
  const VT* tab = reinterpret_cast<const VT*>(table);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float x, y, z;
    load_unit(pts + 3 * i, x, y, z);
    float* o = out + i * (int64_t)(D.n_levels * F);
#pragma unroll 2
    for (int l = 0; l < D.n_levels; ++l) {
      Corner c;
      level_corners(D, l, x, y, z, c);
      VT t[8];
      const VT* base = tab + D.offset[l];
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] = __ldg(base + c.idx[k]);
      float acc[F];
#pragma unroll
      for (int k = 0; k < 8; ++k) vacc<F>(acc, c.w[k], t[k], k == 0);
#pragma unroll
      for (int f = 0; f < F; ++f) o[l * F + f] = acc[f];
    }
  }
}

template <int F>
__global__ void __launch_bounds__(128) encode_bwd_kernel(cf_hashgrid_desc D, const float* __restrict__ pts,
                                                         const float* __restrict__ dfeat, int64_t n,
                                                         float* __restrict__ grad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float x, y, z;
    load_unit(pts + 3 * i, x, y, z);
    const float* g = dfeat + i * (int64_t)(D.n_levels * F);
    for (int l = 0; l < D.n_levels; ++l) {
      float gl[F];
#pragma unroll
      for (int f = 0; f < F; ++f) gl[f] = g[l * F + f];
      Corner c;
      level_corners(D, l, x, y, z, c);
      float* base = grad + D.offset[l] * F;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float* dst = base + (int64_t)c.idx[k] * F;
        if constexpr (F == 2) {
          atomicAdd(reinterpret_cast<float2*>(dst), make_float2(c.w[k] * gl[0], c.w[k] * gl[1]));
        } else {
          atomicAdd(reinterpret_cast<float4*>(dst),
                    make_float4(c.w[k] * gl[0], c.w[k] * gl[1], c.w[k] * gl[2], c.w[k] * gl[3]));
        }
      }
    }
  }
}

__global__ void indices_kernel(cf_hashgrid_desc D, const float* __restrict__ pts, int64_t n, uint32_t* idx_out,
                               float* w_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float x, y, z;
    load_unit(pts + 3 * i, x, y, z);
    for (int l = 0; l < D.n_levels; ++l) {
      Corner c;
      level_corners(D, l, x, y, z, c);
      for (int k = 0; k < 8; ++k) {
        const int64_t o = (i * D.n_levels + l) * 8 + k;
        if (idx_out) idx_out[o] = c.idx[k];
        if (w_out) w_out[o] = c.w[k];
      }
    }
  }
}

int check_desc(const cf_hashgrid_desc* d) {
  if (!d || d->n_levels < 1 || d->n_levels > CF_MAX_LEVELS || (d->n_features != 2 && d->n_features != 4) ||
      d->log2_table < 4 || d->log2_table > 24)
    return cf::fail(CF_E_BAD_ARG, "hash grid: bad descriptor");
  return CF_OK;
}

}  // namespace

extern "C" {

int cf_hashgrid_init(cf_hashgrid_desc* d, int n_levels, int n_features, int log2_table, int base_res, int max_res) {
  if (!d || n_levels < 1 || n_levels > CF_MAX_LEVELS || base_res < 1 || max_res < base_res)
    return cf::fail(CF_E_BAD_ARG, "cf_hashgrid_init: bad args");
  d->n_levels = n_levels;
  d->n_features = n_features;
  d->log2_table = log2_table;
  d->base_resolution = base_res;
  d->max_resolution = max_res;
  const double b = n_levels > 1 ? std::exp((std::log((double)max_res) - std::log((double)base_res)) / (n_levels - 1)) : 1.0;
  const int64_t T = 1LL << log2_table;
  int64_t off = 0;
  for (int l = 0; l < CF_MAX_LEVELS; ++l) {
    if (l >= n_levels) {
      d->resolution[l] = 0;
      d->dense[l] = 0;
      d->offset[l] = off;
      continue;
    }
    const int N = (int)std::floor(base_res * std::pow(b, (double)l) + 1e-9);
    const int64_t dense_size = (int64_t)(N + 1) * (N + 1) * (N + 1);
    d->resolution[l] = N;
    d->dense[l] = dense_size <= T ? 1 : 0;
    d->offset[l] = off;
    const int64_t size = d->dense[l] ? ((dense_size + 7) / 8) * 8 : T;
    off += size;
  }
  d->offset[CF_MAX_LEVELS] = off;
  return check_desc(d);
}

int cf_hashgrid_encode(const cf_hashgrid_desc* d, const float* table, const float* pts, int64_t n, float* out,
                       void* stream) {
  if (int rc = check_desc(d)) return rc;
  if (n == 0) return CF_OK;
  const unsigned grid = cf::grid_for(n, 128, 16);
  if (d->n_features == 2)
    encode_kernel<2><<<grid, 128, 0, cf::as_stream(stream)>>>(*d, table, pts, n, out);
  else
    encode_kernel<4><<<grid, 128, 0, cf::as_stream(stream)>>>(*d, table, pts, n, out);
  return cf::check_launch("cf_hashgrid_encode");
}

int cf_hashgrid_encode_bwd(const cf_hashgrid_desc* d, const float* pts, const float* dfeat, int64_t n,
                           float* table_grad, void* stream) {
  if (int rc = check_desc(d)) return rc;
  if (n == 0) return CF_OK;
  const unsigned grid = cf::grid_for(n, 128, 16);
  if (d->n_features == 2)
    encode_bwd_kernel<2><<<grid, 128, 0, cf::as_stream(stream)>>>(*d, pts, dfeat, n, table_grad);
  else
    encode_bwd_kernel<4><<<grid, 128, 0, cf::as_stream(stream)>>>(*d, pts, dfeat, n, table_grad);
  return cf::check_launch("cf_hashgrid_encode_bwd");
}

int cf_hashgrid_indices(const cf_hashgrid_desc* d, const float* pts, int64_t n, uint32_t* idx_out, float* w_out,
                        void* stream) {
  if (int rc = check_desc(d)) return rc;
  if (n == 0) return CF_OK;
  indices_kernel<<<cf::grid_for(n, 128, 8), 128, 0, cf::as_stream(stream)>>>(*d, pts, n, idx_out, w_out);
  return cf::check_launch("cf_hashgrid_indices");
}

}  // extern "C"
