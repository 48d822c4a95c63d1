// Register-resident k-smallest selection keyed by (squared distance, index):
// ties broken by the smaller index, i.e. the order of the reference's stable
// argsort (knnfield.py:29,39; edgraph.py:127-130).
#pragma once
#include <float.h>
#include "common.cuh"

__device__ __forceinline__ bool key_less(double d1, int i1, double d2, int i2) {
  return d1 < d2 || (d1 == d2 && i1 < i2);
}

template <int K>
struct TopK {
  double d[K];
  int i[K];
  int k;          // runtime k <= K
  double worst_d;  // == d[k-1]
  int worst_i;

  __device__ __forceinline__ void init(int kk) {
    k = kk;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      d[j] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      i[j] = 0x7fffffff;
    }
    worst_d = d[0];
    worst_i = i[0];
  }

  __device__ __forceinline__ void insert(double nd, int ni) {
    if (!key_less(nd, ni, worst_d, worst_i)) return;
#pragma unroll
    for (int j = K - 1; j >= 0; --j) {
      if (j < k) {
        if (j > 0 && key_less(nd, ni, d[j - 1], i[j - 1])) {
          d[j] = d[j - 1];
          i[j] = i[j - 1];
        } else if (key_less(nd, ni, d[j], i[j])) {
          d[j] = nd;
          i[j] = ni;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j == k - 1) {
        worst_d = d[j];
        worst_i = i[j];
      }
  }
};
