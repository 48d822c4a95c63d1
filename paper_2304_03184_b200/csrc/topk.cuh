// Register-resident k-smallest selection keyed by (squared distance, index):
// ties broken by the smaller index, i.e. the order of the reference's stable
// argsort (knnfield.py:29,39; edgraph.py:127-130). K is the exact k (every
// kernel is dispatched on it), so all slot indices are compile-time constants
// and the arrays stay in registers.
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

  __device__ __forceinline__ void init(int /*k == K*/ = K) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      d[j] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      i[j] = 0x7fffffff;
    }
  }

  __device__ __forceinline__ double worst_d() const { return d[K - 1]; }

  __device__ __forceinline__ void insert(double nd, int ni) {
    if (!key_less(nd, ni, d[K - 1], i[K - 1])) return;
#pragma unroll
    for (int j = K - 1; j >= 0; --j) {
      if (j > 0 && key_less(nd, ni, d[j - 1], i[j - 1])) {
        d[j] = d[j - 1];
        i[j] = i[j - 1];
      } else if (key_less(nd, ni, d[j], i[j])) {
        d[j] = nd;
        i[j] = ni;
      }
    }
  }
};

// Run f.template operator()<K>() for the exact runtime k (1..8, 16).
template <class F>
__device__ __host__ __forceinline__ int dispatch_k(int k, F&& f) {
  switch (k) {
    case 1: return f.template operator()<1>();
    case 2: return f.template operator()<2>();
    case 3: return f.template operator()<3>();
    case 4: return f.template operator()<4>();
    case 5: return f.template operator()<5>();
    case 6: return f.template operator()<6>();
    case 7: return f.template operator()<7>();
    case 8: return f.template operator()<8>();
    case 16: return f.template operator()<16>();
    default: return -1;
  }
}
