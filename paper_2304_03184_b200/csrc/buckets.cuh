// Coarse uniform voxel buckets over a point set (deformed ED nodes, posed skin
// vertices) and the exact ring-search k-NN that runs on them. The search visits
// Chebyshev rings of cells around the query's cell and stops once the k-th best
// squared distance is strictly below the squared distance to every unvisited
// cell (with a relative safety margin), so its result equals the exhaustive
// (d2, index)-ordered top-k bit for bit.
#pragma once
#include "common.cuh"
#include "topk.cuh"

struct BucketParams {
  double origin[3];
  double h;        // cubic cell edge
  double margin;   // conservative slack for the termination bound
  int g[3];        // cells per axis
  int n;           // points
};

struct cf_buckets {
  int64_t max_points = 0;
  int max_grid_res = 0;
  BucketParams* params = nullptr;  // device
  int* cell_start = nullptr;       // device, max_cells + 1
  int* point_cell = nullptr;       // device, max_points
  int* point_slot = nullptr;       // device, max_points
  double4* sorted = nullptr;       // device, max_points: (x, y, z, id as double)
  int grid_res = 0;                // last build
  // cell candidate lists (cf_buckets_build_candidates): for every cell, the
  // points that can be among the k nearest of ANY query inside that cell
  int* ccl_count = nullptr;        // device, max_cells + 1 (count, then exclusive start)
  int* ccl_len = nullptr;          // device, max_cells
  int* ccl_ids = nullptr;          // device, ccl_cap
  int64_t ccl_cap = 0;
  int ccl_k = 0;                   // k the lists are valid for (0 = not built)
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ void bucket_cell(const BucketParams& P, d3 p, int c[3]) {
  double q[3] = {p.x, p.y, p.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double f = floor((q[a] - P.origin[a]) / P.h);
    f = fmin(fmax(f, -1.0), (double)P.g[a]);  // keep the int conversion in range
    c[a] = clampi((int)f, 0, P.g[a] - 1);
  }
}

template <int K>
__device__ __forceinline__ void scan_range(int b, int e, const double4* __restrict__ sorted, d3 p, TopK<K>& top) {
  for (int t = b; t < e; ++t) {
    const double4 s = sorted[t];
    top.insert(sqdist(p, d3{s.x, s.y, s.z}), (int)s.w);
  }
}

// Exact k-NN of p over the bucketed point set. `pts` are the un-sorted source
// points (distances are evaluated on them only through the sorted copy, which
// holds identical values).
template <int K>
// `cutoff2`: callers that only use neighbours within sqrt(cutoff2) (occupancy,
// LBS validity) stop once every unvisited cell is farther than that; the result
// is then exact for every neighbour within the cutoff (others may be missing).
__device__ __forceinline__ void bucket_knn(const BucketParams& P, const int* __restrict__ cell_start,
                                           const double4* __restrict__ sorted, d3 p, TopK<K>& top,
                                           double cutoff2 = 1.0e300) {
  int c0[3];
  bucket_cell(P, p, c0);
  const double q[3] = {p.x, p.y, p.z};
  const int gmax = max(P.g[0], max(P.g[1], P.g[2]));
  for (int r = 0; r <= gmax; ++r) {
    const int z0 = max(c0[2] - r, 0), z1 = min(c0[2] + r, P.g[2] - 1);
    const int y0 = max(c0[1] - r, 0), y1 = min(c0[1] + r, P.g[1] - 1);
    const int x0 = max(c0[0] - r, 0), x1 = min(c0[0] + r, P.g[0] - 1);
    for (int z = z0; z <= z1; ++z) {
      const bool zedge = (z == c0[2] - r) || (z == c0[2] + r);
      for (int y = y0; y <= y1; ++y) {
        const int row = (z * P.g[1] + y) * P.g[0];
        // cells of one x-run are contiguous, so their points are one contiguous range
        if (zedge || (y == c0[1] - r) || (y == c0[1] + r)) {
          scan_range(cell_start[row + x0], cell_start[row + x1 + 1], sorted, p, top);
        } else {
          if (c0[0] - r >= 0) scan_range(cell_start[row + c0[0] - r], cell_start[row + c0[0] - r + 1], sorted, p, top);
          if (c0[0] + r < P.g[0])
            scan_range(cell_start[row + c0[0] + r], cell_start[row + c0[0] + r + 1], sorted, p, top);
        }
      }
    }
    // lower bound on the distance to any cell outside the visited box
    const int lo[3] = {x0, y0, z0}, hi[3] = {x1, y1, z1};
    double bound = __longlong_as_double(0x7ff0000000000000LL);
    bool covered = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (lo[a] > 0) {
        covered = false;
        bound = fmin(bound, q[a] - (P.origin[a] + lo[a] * P.h));
      }
      if (hi[a] < P.g[a] - 1) {
        covered = false;
        bound = fmin(bound, (P.origin[a] + (hi[a] + 1) * P.h) - q[a]);
      }
    }
    if (covered) break;
    bound -= P.margin;
    if (bound > 0.0 && (top.worst_d() < bound * bound || bound * bound > cutoff2)) break;
  }
}

namespace cf {
int buckets_build(cf_buckets* b, const double* pts, int64_t n, int grid_res, cudaStream_t st);
}
