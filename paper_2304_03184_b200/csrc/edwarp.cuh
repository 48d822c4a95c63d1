// One-point ED warp on the coarse buckets: exact k-NN (ties by index) ->
// Gaussian weights -> DQB -> (inverse) apply, the body of
// edgraph._blend_for + warp_backward_batch / warp_forward_batch
// (edgraph.py:139-183) for a single float64 point.
#pragma once
#include "buckets.cuh"
#include "dq.cuh"

template <int K>
__device__ __forceinline__ bool blend_apply(const TopK<K>& top, const double* __restrict__ dqs, int k, double r2,
                                            bool inverse, d3 p, d3& out);

template <int K>
__device__ __forceinline__ bool ed_warp_point(const BucketParams& P, const int* __restrict__ cell_start,
                                              const double4* __restrict__ sorted, const double* __restrict__ dqs,
                                              int k, double r2, bool inverse, d3 p, d3& out) {
  TopK<K> top;
  top.init(k);
  bucket_knn<K>(P, cell_start, sorted, p, top);
  return blend_apply<K>(top, dqs, k, r2, inverse, p, out);
}

// Small graphs: exhaustive scan of the anchors staged in shared memory (every
// thread reads the same anchor at once — a broadcast, no bank conflicts).
// Same (d2, index) order, hence bit-identical to the bucket search.
template <int K>
__device__ __forceinline__ bool ed_warp_point_smem(const double4* __restrict__ s_anchors,
                                                   const float4* __restrict__ s_af, int n,
                                                   const double* __restrict__ dqs, int k, double r2, bool inverse,
                                                   d3 p, d3& out) {
  TopK<K> top;
  top.init(k);
  // fp32 prefilter: a candidate whose fp32 squared distance exceeds the current
  // k-th best by more than the fp32 error bound cannot enter the top-k, so only
  // survivors pay the exact float64 evaluation. The error of the fp32 d^2 (from
  // rounding p and the anchor to fp32) is <= ~2|d| sqrt(3) 2^-23 max|coord|;
  // `slack` bounds it for coordinates up to `mag` (s_af[0].w = max |anchor coord|).
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  const float mag = fmaxf(fmaxf(fabsf(px), fmaxf(fabsf(py), fabsf(pz))), s_af[0].w) + 1.0f;
  const float slack = 64.0f * 1.1920929e-7f * mag * mag;
  float bound = __int_as_float(0x7f800000);  // +inf until k candidates are in
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    const float4 af = s_af[i];
    const float dx = px - af.x, dy = py - af.y, dz = pz - af.z;
    const float fd = dx * dx + dy * dy + dz * dz;
    if (fd > bound) continue;
    const double4 a = s_anchors[i];
    top.insert(sqdist(p, d3{a.x, a.y, a.z}), i);
    bound = (float)top.worst_d() * (1.0f + 4.0f * 1.1920929e-7f) + slack;
  }
  return blend_apply<K>(top, dqs, k, r2, inverse, p, out);
}

// Warp-cooperative culling for the exhaustive scan (all 32 lanes must call it,
// `live` marks lanes holding a sample). The warp's samples are spatially
// coherent (consecutive compacted samples of neighbouring rays), so:
//  1. bbox B of the warp's samples (fp32);
//  2. U = k-th smallest, over all nodes, of the farthest distance^2 from B —
//     every sample in B has its k-th neighbour within U;
//  3. only nodes whose nearest distance^2 to B is <= U (+ fp32 slack) can be
//     in any lane's top-k; the warp walks that candidate set uniformly
//     (ballot masks, smem broadcast reads), each lane ranking its own sample
//     exactly in float64. Identical result to scanning every node.
template <int K>
__device__ __forceinline__ bool ed_warp_point_cull(const double4* __restrict__ s_anchors,
                                                   const float4* __restrict__ s_af, int n,
                                                   const double* __restrict__ dqs, int k, double r2, bool inverse,
                                                   d3 p, bool live, d3& out) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  const float INF = __int_as_float(0x7f800000);
  float lo[3] = {live ? px : INF, live ? py : INF, live ? pz : INF};
  float hi[3] = {live ? px : -INF, live ? py : -INF, live ? pz : -INF};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(FULL, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(FULL, hi[a], o));
    }
  const float mag = fmaxf(fmaxf(fmaxf(fabsf(lo[0]), fabsf(hi[0])), fmaxf(fmaxf(fabsf(lo[1]), fabsf(hi[1])),
                                                                       fmaxf(fabsf(lo[2]), fabsf(hi[2])))),
                          s_af[0].w) + 1.0f;
  const float slack = 64.0f * 1.1920929e-7f * mag * mag;
  // per-lane k smallest farthest-distances of its nodes (i = lane, lane+32, ...)
  float best[K];
#pragma unroll
  for (int j = 0; j < K; ++j) best[j] = INF;
  for (int i = lane; i < n; i += 32) {
    const float4 a = s_af[i];
    const float ex = fmaxf(fabsf(a.x - lo[0]), fabsf(a.x - hi[0]));
    const float ey = fmaxf(fabsf(a.y - lo[1]), fabsf(a.y - hi[1]));
    const float ez = fmaxf(fabsf(a.z - lo[2]), fabsf(a.z - hi[2]));
    float v = ex * ex + ey * ey + ez * ez;
#pragma unroll
    for (int j = 0; j < K; ++j) {  // insertion into the sorted per-lane list
      const float lo_v = fminf(v, best[j]);
      v = fmaxf(v, best[j]);
      best[j] = lo_v;
    }
  }
  // k rounds of a warp-wide min with removal -> the k-th smallest overall
  float U = INF;
  for (int r = 0; r < k; ++r) {
    float m = best[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(FULL, m, o));
    U = m;
    const unsigned owner = __ballot_sync(FULL, best[0] == m);
    if (lane == __ffs(owner) - 1) {  // pop the head of the owning lane's list
#pragma unroll
      for (int j = 0; j < K - 1; ++j) best[j] = best[j + 1];
      best[K - 1] = INF;
    }
  }
  const float cut = U + 2.0f * slack;
  TopK<K> top;
  top.init(k);
  float bound = INF;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int i = c0 + lane;
    bool cand = false;
    if (i < n) {
      const float4 a = s_af[i];
      const float dx = fmaxf(fmaxf(lo[0] - a.x, a.x - hi[0]), 0.f);
      const float dy = fmaxf(fmaxf(lo[1] - a.y, a.y - hi[1]), 0.f);
      const float dz = fmaxf(fmaxf(lo[2] - a.z, a.z - hi[2]), 0.f);
      cand = dx * dx + dy * dy + dz * dz <= cut;
    }
    unsigned mask = __ballot_sync(FULL, cand);
    while (mask) {
      const int b = __ffs(mask) - 1;
      mask &= mask - 1;
      const int node = c0 + b;
      const float4 af = s_af[node];
      const float ddx = px - af.x, ddy = py - af.y, ddz = pz - af.z;
      if (ddx * ddx + ddy * ddy + ddz * ddz > bound) continue;
      const double4 a = s_anchors[node];
      top.insert(sqdist(p, d3{a.x, a.y, a.z}), node);
      bound = (float)top.worst_d() * (1.0f + 4.0f * 1.1920929e-7f) + slack;
    }
  }
  if (!live) return false;
  return blend_apply<K>(top, dqs, k, r2, inverse, p, out);
}

template <int K>
__device__ __forceinline__ bool blend_apply(const TopK<K>& top, const double* __restrict__ dqs, int k, double r2,
                                            bool inverse, d3 p, d3& out) {
  double w[K];
  bool valid = false;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j < k) {
      w[j] = exp(x_div(-top.d[j], r2));
      valid |= w[j] > 1e-6;
    }
  DqbAcc acc;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j < k) acc.add(valid ? w[j] : 1.0, load_dq(dqs + 8 * (int64_t)top.i[j]));
  dq8 b = acc.result();
  if (inverse) b = dq_conj(b);
  out = dq_apply(b, p);
  return valid;
}
