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
__device__ __forceinline__ bool ed_warp_point_smem(const double4* __restrict__ s_anchors, int n,
                                                   const double* __restrict__ dqs, int k, double r2, bool inverse,
                                                   d3 p, d3& out) {
  TopK<K> top;
  top.init(k);
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    const double4 a = s_anchors[i];
    top.insert(sqdist(p, d3{a.x, a.y, a.z}), i);
  }
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
