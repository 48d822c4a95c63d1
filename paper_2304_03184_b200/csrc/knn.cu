// Per-frame node deformation, coarse node buckets, and the fused exact
// k-NN + dual-quaternion blend kernels behind
//   edgraph.warp_backward_batch / warp_forward_batch  (edgraph.py:139-183)
//   knnfield.brute_force_query / brute_force_neighbors_batch (knnfield.py:20-42)
// All geometry is float64 in the reference's evaluation order (dq.cuh), so the
// k-NN indices are bit-identical and the positions match to the last bits of exp().
#include <algorithm>
#include <cmath>

#include <cooperative_groups.h>

#include "buckets.cuh"
#include "dq.cuh"
#include "edwarp.cuh"

namespace {

constexpr double kWeightFloor = 1e-6;  // edgraph.py:24

__global__ void deform_nodes_kernel(const double* __restrict__ nodes, const double* __restrict__ dqs, int64_t n,
                                    double* __restrict__ anchors) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    dq8 q = load_dq(dqs + 8 * i);
    store_d3(anchors + 3 * i, dq_apply(q, load_d3(nodes + 3 * i)));
  }
  pdl_trigger();
}

// Small graphs (n <= 1024, one CTA): the deformed nodes plus the per-frame anchor
// block the canonicalisation reads straight from L1 — float64 copies (double4), fp32
// copies (float4, [0].w = max |coordinate|) and the float64 bbox — built once per
// frame instead of once per CTA of every canonicalisation launch.
__global__ void __launch_bounds__(1024) deform_nodes_block_kernel(const double* __restrict__ nodes,
                                                                  const double* __restrict__ dqs, int n,
                                                                  double* __restrict__ anchors,
                                                                  uint8_t* __restrict__ block) {
  pdl_wait();
  double4* a64 = reinterpret_cast<double4*>(block);
  float4* a32 = reinterpret_cast<float4*>(block + 32 * (size_t)n);
  double* box = reinterpret_cast<double*>(block + 48 * (size_t)n);
  __shared__ double s_lo[32][3], s_hi[32][3];
  __shared__ float s_mag[32];
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  float mag = 0.f;
  float4 af = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < n) {
    const d3 a = dq_apply(load_dq(dqs + 8 * (int64_t)i), load_d3(nodes + 3 * (int64_t)i));
    store_d3(anchors + 3 * (int64_t)i, a);
    a64[i] = make_double4(a.x, a.y, a.z, 0.0);
    af = make_float4((float)a.x, (float)a.y, (float)a.z, 0.f);
    mag = fmaxf(fabsf(af.x), fmaxf(fabsf(af.y), fabsf(af.z)));
    lo[0] = hi[0] = a.x;
    lo[1] = hi[1] = a.y;
    lo[2] = hi[2] = a.z;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mag = fmaxf(mag, __shfl_xor_sync(0xffffffffu, mag, o));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  }
  if (lane == 0) {
    s_mag[warp] = mag;
    for (int a = 0; a < 3; ++a) {
      s_lo[warp][a] = lo[a];
      s_hi[warp][a] = hi[a];
    }
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = (int)(blockDim.x >> 5);
    mag = lane < nw ? s_mag[lane] : 0.f;
    for (int a = 0; a < 3; ++a) {
      lo[a] = lane < nw ? s_lo[lane][a] : INFINITY;
      hi[a] = lane < nw ? s_hi[lane][a] : -INFINITY;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mag = fmaxf(mag, __shfl_xor_sync(0xffffffffu, mag, o));
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
        hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
      }
    }
    if (lane == 0) {
      for (int a = 0; a < 3; ++a) {
        box[a] = lo[a];
        box[3 + a] = hi[a];
      }
      s_mag[0] = mag;
    }
  }
  __syncthreads();
  if (i == 0) af.w = s_mag[0];
  if (i < n) a32[i] = af;
  pdl_trigger();
}

// Candidate grid of a small graph (the render path's k-NN, n <= 1024): a per-frame
// grid of cells over the anchors' bbox grown by the ED support radius R (a sample
// farther than R from every node has all Gaussian weights below the validity
// floor); per cell the nodes that can be among the k nearest of ANY point of the
// cell: U = the k-th smallest (with multiplicity) over all nodes of the farthest
// distance^2 from the cell box to the node bounds the k-th neighbour distance^2 of
// every point in the cell, and a node whose nearest distance^2 to the box exceeds U
// cannot be closer than that (ties included: <=). The bounds are taken in fp32 with
// margins that only grow the lists (see the kernel); lists hold node ids ascending,
// up to cmax; a fuller cell is marked 0xFFFF (its samples scan every node).

__device__ __forceinline__ void cand_grid_geometry(const double* box, double r2, int G, CandGridHdr& H) {
  const double R = sqrt(13.815510557964274 * r2 * (1.0 + 1e-5)) * (1.0 + 1e-9) + 1e-9;
  double ext[3], mx = 0.0;
  for (int a = 0; a < 3; ++a) {
    H.origin[a] = box[a] - R;
    ext[a] = (box[3 + a] + R) - H.origin[a];
    mx = fmax(mx, ext[a]);
  }
  H.h = mx / G;
  H.inv_h = 1.0 / H.h;
  for (int a = 0; a < 3; ++a) H.dims[a] = max(1, min(G, (int)ceil(ext[a] * H.inv_h)));
}

template <int K>
__global__ void __launch_bounds__(64) cand_grid_kernel(const uint8_t* __restrict__ block, int n, int k, double r2,
                                                       int G, int cmax, uint8_t* __restrict__ cand) {
  extern __shared__ float4 s_a[];  // the frame's nodes (fp32 copies)
  pdl_wait();
  const float4* a32 = reinterpret_cast<const float4*>(block + 32 * (size_t)n);
  const double* box = reinterpret_cast<const double*>(block + 48 * (size_t)n);
  CandGridHdr H;
  cand_grid_geometry(box, r2, G, H);
  H.cmax = cmax;
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<CandGridHdr*>(cand) = H;
  if ((int64_t)blockIdx.x * blockDim.x >= (int64_t)H.dims[0] * H.dims[1] * H.dims[2]) return;  // (CTA-uniform)
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_a[i] = a32[i];
  __syncthreads();
  uint16_t* lists = reinterpret_cast<uint16_t*>(cand + 64);
  const int64_t cells = (int64_t)H.dims[0] * H.dims[1] * H.dims[2];
  const float INF = __int_as_float(0x7f800000);
  // one thread per cell, the nodes broadcast from shared memory. fp32 with margins that
  // keep the list a superset: U is rounded up (an upper bound of the k-th neighbour
  // distance^2 of every point of the cell), each node's nearest distance^2 to the cell
  // rounded down (fp32 coordinates of ~1 m carry < 1e-7 relative error, the margins
  // are 1e-4 relative + 1e-9 m^2); the samples then rank the list exactly in float64.
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x) {
    const int cx = (int)(c / ((int64_t)H.dims[1] * H.dims[2])), cy = (int)((c / H.dims[2]) % H.dims[1]),
              cz = (int)(c % H.dims[2]);
    const float lo[3] = {(float)(H.origin[0] + cx * H.h), (float)(H.origin[1] + cy * H.h),
                         (float)(H.origin[2] + cz * H.h)};
    const float hf = (float)H.h;
    const float hi[3] = {lo[0] + hf, lo[1] + hf, lo[2] + hf};
    float best[K];  // the K smallest farthest-distances^2 (with multiplicity), ascending
#pragma unroll
    for (int j = 0; j < K; ++j) best[j] = INF;
    for (int i = 0; i < n; ++i) {
      const float4 a = s_a[i];
      const float ex = fmaxf(fabsf(a.x - lo[0]), fabsf(a.x - hi[0]));
      const float ey = fmaxf(fabsf(a.y - lo[1]), fabsf(a.y - hi[1]));
      const float ez = fmaxf(fabsf(a.z - lo[2]), fabsf(a.z - hi[2]));
      float v = ex * ex + ey * ey + ez * ez;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const float lo_v = fminf(v, best[j]);
        v = fmaxf(v, best[j]);
        best[j] = lo_v;
      }
    }
    const float cut = best[K - 1] * (1.0f + 1e-4f) + 1e-9f;
    uint16_t* L = lists + c * cand_stride(cmax);
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      const float4 a = s_a[i];
      const float dx = fmaxf(fmaxf(lo[0] - a.x, a.x - hi[0]), 0.f);
      const float dy = fmaxf(fmaxf(lo[1] - a.y, a.y - hi[1]), 0.f);
      const float dz = fmaxf(fmaxf(lo[2] - a.z, a.z - hi[2]), 0.f);
      if ((dx * dx + dy * dy + dz * dz) * (1.0f - 1e-4f) - 1e-9f <= cut) {
        if (cnt < cmax) L[1 + cnt] = (uint16_t)i;
        ++cnt;
      }
    }
    L[0] = cnt <= cmax ? (uint16_t)cnt : (uint16_t)0xFFFF;
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ transforms drop-ins
// dq_blend (transforms.py:180-196) over n rows of k neighbours, in the reference's
// evaluation order (DqbAcc: sign-aligned to the row's first real part, sequential
// weighted sum, dq_normalize). Argument errors are flagged per row into *err (the
// largest code wins, as the reference checks the negative weights first):
// 2 = a negative weight (ValueError), 1 = a row whose weights sum to <= 0
// (DegenerateWeightsError); cf_dq_status turns the flag into the status.
__global__ void dq_blend_kernel(const double* __restrict__ w, const double* __restrict__ dqs, int64_t n, int k,
                                double* __restrict__ out, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool neg = false;
    double wsum = 0.0;
    DqbAcc acc;
    for (int j = 0; j < k; ++j) {
      const double wj = w[i * k + j];
      neg |= wj < 0.0;
      wsum = j == 0 ? wj : x_add(wsum, wj);
      acc.add(wj, load_dq(dqs + 8 * (i * k + j)));
    }
    if (err && (neg || wsum <= 0.0 || k == 0)) atomicMax(err, neg ? 2 : 1);
    const dq8 b = acc.result();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      out[8 * i + c] = b.r[c];
      out[8 * i + 4 + c] = b.d[c];
    }
  }
}

// dq_apply (transforms.py:174-177): rotate by the real part, add the translation
__global__ void dq_apply_kernel(const double* __restrict__ dq, int64_t dq_stride, const double* __restrict__ p,
                                int64_t p_stride, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    store_d3(out + 3 * i, dq_apply(load_dq(dq + dq_stride * i), load_d3(p + p_stride * i)));
}

// ------------------------------------------------------------------ buckets

// grid of G cells along the longest extent of the bbox [mn, mx]
__device__ __forceinline__ void bucket_params_finish(const double* mn, const double* mx, int n, int G,
                                                     BucketParams* P) {
  double ext = 0.0, scale = 0.0;
  for (int a = 0; a < 3; ++a) {
    ext = fmax(ext, mx[a] - mn[a]);
    scale = fmax(scale, fmax(fabs(mn[a]), fabs(mx[a])));
  }
  if (!(ext > 0.0)) ext = fmax(scale, 1.0) * 1e-3;
  const double h = ext * (1.0 + 1e-9) / G;
  for (int a = 0; a < 3; ++a) {
    P->origin[a] = mn[a] - 1e-12 * (fabs(mn[a]) + ext);
    int g = (int)ceil((mx[a] - P->origin[a]) / h);
    P->g[a] = g < 1 ? 1 : (g > G ? G : g);
  }
  P->h = h;
  P->margin = 1e-10 * (scale + ext) + 1e-300;
  P->n = n;
}

__device__ __forceinline__ void bucket_params_body(const double* __restrict__ pts, int n, int G, BucketParams* P) {
  __shared__ double smin[3][32], smax[3][32];
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int a = 0; a < 3; ++a) {
      double v = pts[3 * i + a];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    for (int a = 0; a < 3; ++a) {
      smin[a][w] = lo[a];
      smax[a][w] = hi[a];
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    double mn[3], mx[3];
    for (int a = 0; a < 3; ++a) {
      mn[a] = smin[a][0];
      mx[a] = smax[a][0];
      for (int j = 1; j < nw; ++j) {
        mn[a] = fmin(mn[a], smin[a][j]);
        mx[a] = fmax(mx[a], smax[a][j]);
      }
    }
    bucket_params_finish(mn, mx, n, G, P);
  }
}

__device__ __forceinline__ void bucket_count_body(const double* __restrict__ pts, int n, const BucketParams* __restrict__ Pp,
                                    int* __restrict__ counts, int* __restrict__ point_cell,
                                    int* __restrict__ point_slot) {
  const BucketParams P = *Pp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int c[3];
    bucket_cell(P, load_d3(pts + 3 * i), c);
    const int cell = (c[2] * P.g[1] + c[1]) * P.g[0] + c[0];
    point_cell[i] = cell;
    point_slot[i] = atomicAdd(counts + cell, 1);
  }
}

// single-CTA exclusive scan, in place: counts[0..ncells] -> starts
__device__ __forceinline__ void bucket_scan_body(int* __restrict__ cells, const BucketParams* __restrict__ Pp) {
  // each thread owns a contiguous chunk: serial sum, block scan of the chunk
  // totals, serial write-back (2 barriers regardless of the cell count)
  __shared__ int warp_tot[32];
  const int ncells = Pp->g[0] * Pp->g[1] * Pp->g[2];
  const int n = ncells + 1;
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int b = min(n, (int)threadIdx.x * chunk), e = min(n, b + chunk);
  int v = 0;
  for (int i = b; i < e; ++i) v += (i < ncells) ? cells[i] : 0;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = (threadIdx.x < (blockDim.x >> 5)) ? warp_tot[threadIdx.x] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (threadIdx.x >= o) t += y;
    }
    if (threadIdx.x < (blockDim.x >> 5)) warp_tot[threadIdx.x] = t;
  }
  __syncthreads();
  int run = (w > 0 ? warp_tot[w - 1] : 0) + x - v;
  for (int i = b; i < e; ++i) {
    const int c = (i < ncells) ? cells[i] : 0;
    cells[i] = run;
    run += c;
  }
}

__device__ __forceinline__ void bucket_scatter_body(const double* __restrict__ pts, int n, const int* __restrict__ cell_start,
                                      const int* __restrict__ point_cell, const int* __restrict__ point_slot,
                                      double4* __restrict__ sorted) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int dst = cell_start[point_cell[i]] + point_slot[i];
    sorted[dst] = make_double4(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], (double)i);
  }
}

__global__ void bucket_params_kernel(const double* __restrict__ pts, int n, int G, BucketParams* P) {
  bucket_params_body(pts, n, G, P);
}
__global__ void bucket_count_kernel(const double* __restrict__ pts, int n, const BucketParams* __restrict__ Pp,
                                    int* __restrict__ counts, int* __restrict__ point_cell,
                                    int* __restrict__ point_slot) {
  bucket_count_body(pts, n, Pp, counts, point_cell, point_slot);
}
__global__ void bucket_scan_kernel(int* __restrict__ cells, const BucketParams* __restrict__ Pp) {
  bucket_scan_body(cells, Pp);
}
__global__ void bucket_scatter_kernel(const double* __restrict__ pts, int n, const int* __restrict__ cell_start,
                                      const int* __restrict__ point_cell, const int* __restrict__ point_slot,
                                      double4* __restrict__ sorted) {
  bucket_scatter_body(pts, n, cell_start, point_cell, point_slot, sorted);
}

// single-CTA exclusive scan of an int array in shared memory (n = ncells + 1 entries)
__device__ __forceinline__ void smem_scan(int* __restrict__ a, int n) {
  __shared__ int warp_tot[32];
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int b = min(n, (int)threadIdx.x * chunk), e = min(n, b + chunk);
  int v = 0;
  for (int i = b; i < e; ++i) v += a[i];
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = (threadIdx.x < (blockDim.x >> 5)) ? warp_tot[threadIdx.x] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (threadIdx.x >= o) t += y;
    }
    if (threadIdx.x < (blockDim.x >> 5)) warp_tot[threadIdx.x] = t;
  }
  __syncthreads();
  int run = (w > 0 ? warp_tot[w - 1] : 0) + x - v;
  for (int i = b; i < e; ++i) {
    const int c = a[i];
    a[i] = run;
    run += c;
  }
}

// The whole build in one CTA with the cell counts in shared memory (per-frame
// skin vertices: 6 890 points, 31^3 cells): shared-memory atomics and scan,
// one coalesced write of cell_start — no global atomics or round trips.
constexpr int kSmemBucketCells = 48 * 1024;
__global__ void __launch_bounds__(1024) bucket_build_smem_kernel(const double* __restrict__ pts, int n, int G,
                                                                 BucketParams* P, int* __restrict__ cell_start,
                                                                 int* __restrict__ point_cell,
                                                                 int* __restrict__ point_slot,
                                                                 double4* __restrict__ sorted) {
  extern __shared__ int s_cnt[];
  pdl_wait();
  const int cells_max = G * G * G;
  for (int i = threadIdx.x; i <= cells_max; i += blockDim.x) s_cnt[i] = 0;
  bucket_params_body(pts, n, G, P);
  __syncthreads();
  const BucketParams Pl = *P;
  const int ncells = Pl.g[0] * Pl.g[1] * Pl.g[2];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int c[3];
    bucket_cell(Pl, load_d3(pts + 3 * i), c);
    const int cell = (c[2] * Pl.g[1] + c[1]) * Pl.g[0] + c[0];
    point_cell[i] = cell;
    point_slot[i] = atomicAdd(s_cnt + cell, 1);
  }
  __syncthreads();
  smem_scan(s_cnt, ncells + 1);
  __syncthreads();
  for (int i = threadIdx.x; i <= ncells; i += blockDim.x) cell_start[i] = s_cnt[i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int dst = s_cnt[point_cell[i]] + point_slot[i];
    sorted[dst] = make_double4(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], (double)i);
  }
  pdl_trigger();
}

// The build spread over a thread-block cluster of kBucketCluster CTAs (one per
// SM), with the cell counts in CTA 0's shared memory and every CTA counting /
// scattering its slice of the points through distributed shared memory: the
// per-point phases run on 8 SMs instead of one, and the phase boundaries are
// cluster barriers instead of kernel launches (per-frame skin vertices: 6 890
// points, 31^3 cells).
constexpr int kBucketCluster = 8;
__global__ void __cluster_dims__(kBucketCluster, 1, 1) __launch_bounds__(1024)
    bucket_build_cluster_kernel(const double* __restrict__ pts, int n, int G, BucketParams* P,
                                int* __restrict__ cell_start, int* __restrict__ point_cell,
                                int* __restrict__ point_slot, double4* __restrict__ sorted) {
  extern __shared__ int s_cnt[];  // cell counts, used in CTA 0
  __shared__ double s_box[6];     // this CTA's partial bbox (lo xyz, hi xyz)
  __shared__ double s_w[6][32];
  __shared__ BucketParams s_P;    // CTA 0: the grid parameters
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, stride = kBucketCluster * blockDim.x;
  const int first = rank * blockDim.x + tid;
  pdl_wait();
  if (rank == 0)
    for (int i = tid; i <= G * G * G; i += blockDim.x) s_cnt[i] = 0;
  // 1. partial bounding boxes
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = first; i < n; i += stride)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double v = pts[3 * i + a];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  if ((tid & 31) == 0)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      s_w[a][tid >> 5] = lo[a];
      s_w[3 + a][tid >> 5] = hi[a];
    }
  __syncthreads();
  if (tid < 6) {
    double v = s_w[tid][0];
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j) v = tid < 3 ? fmin(v, s_w[tid][j]) : fmax(v, s_w[tid][j]);
    s_box[tid] = v;
  }
  cl.sync();
  // 2. CTA 0: grid parameters from the cluster's bbox
  if (rank == 0 && tid == 0) {
    double mn[3], mx[3];
    for (int a = 0; a < 3; ++a) {
      mn[a] = INFINITY;
      mx[a] = -INFINITY;
    }
    for (int r = 0; r < kBucketCluster; ++r) {
      const double* b = cl.map_shared_rank(s_box, r);
      for (int a = 0; a < 3; ++a) {
        mn[a] = fmin(mn[a], b[a]);
        mx[a] = fmax(mx[a], b[3 + a]);
      }
    }
    bucket_params_finish(mn, mx, n, G, &s_P);
    *P = s_P;
  }
  cl.sync();
  const BucketParams Pl = *cl.map_shared_rank(&s_P, 0);
  int* cnt0 = cl.map_shared_rank(s_cnt, 0);
  const int ncells = Pl.g[0] * Pl.g[1] * Pl.g[2];
  // 3. counts (DSMEM atomics into CTA 0)
  for (int i = first; i < n; i += stride) {
    int c[3];
    bucket_cell(Pl, load_d3(pts + 3 * i), c);
    const int cell = (c[2] * Pl.g[1] + c[1]) * Pl.g[0] + c[0];
    point_cell[i] = cell;
    point_slot[i] = atomicAdd(cnt0 + cell, 1);
  }
  cl.sync();
  // 4. CTA 0: exclusive scan -> cell starts
  if (rank == 0) {
    smem_scan(s_cnt, ncells + 1);
    __syncthreads();
    for (int i = tid; i <= ncells; i += blockDim.x) cell_start[i] = s_cnt[i];
  }
  cl.sync();
  // 5. scatter (starts read from CTA 0 through DSMEM)
  for (int i = first; i < n; i += stride) {
    const int dst = cnt0[point_cell[i]] + point_slot[i];
    sorted[dst] = make_double4(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], (double)i);
  }
  cl.sync();  // CTA 0's shared memory stays alive until every CTA is done with it
  pdl_trigger();
}

// the whole build in one CTA for small point sets (per-frame ED nodes / skin
// vertices): one launch instead of four plus a memset
__global__ void __launch_bounds__(1024) bucket_build_small_kernel(const double* __restrict__ pts, int n, int G,
                                                                  BucketParams* P, int* __restrict__ cell_start,
                                                                  int* __restrict__ point_cell,
                                                                  int* __restrict__ point_slot,
                                                                  double4* __restrict__ sorted) {
  pdl_wait();
  const int cells = G * G * G;
  for (int i = threadIdx.x; i <= cells; i += blockDim.x) cell_start[i] = 0;
  bucket_params_body(pts, n, G, P);
  __syncthreads();
  bucket_count_body(pts, n, P, cell_start, point_cell, point_slot);
  __syncthreads();
  bucket_scan_body(cell_start, P);
  __syncthreads();
  bucket_scatter_body(pts, n, cell_start, point_cell, point_slot, sorted);
  pdl_trigger();
}

// ------------------------------------------------------------------ cell candidate lists
// For cell C with centre c and half-diagonal hd, any query p in C has
// d_k(p) <= d_k(c) + hd, so every member x of p's k-NN satisfies
// |c - x| <= |c - p| + |p - x| <= d_k(c) + 2 hd. The list of C is exactly the
// points within that radius (float64, relative slack 1e-9): scanning it yields
// the exact (d2, index)-ordered k-NN of any query inside C.

__device__ __forceinline__ d3 bucket_center(const BucketParams& P, int cell) {
  const int x = cell % P.g[0], y = (cell / P.g[0]) % P.g[1], z = cell / (P.g[0] * P.g[1]);
  return d3{P.origin[0] + (x + 0.5) * P.h, P.origin[1] + (y + 0.5) * P.h, P.origin[2] + (z + 0.5) * P.h};
}

template <int K>
__global__ void __launch_bounds__(128, 4) ccl_kernel(const BucketParams* __restrict__ Pp,
                                                     const int* __restrict__ cell_start,
                                                     const double4* __restrict__ sorted, int phase,
                                                     int* __restrict__ count, int* __restrict__ len,
                                                     int* __restrict__ ids, int64_t cap) {
  __shared__ BucketParams sP;
  if (threadIdx.x == 0) sP = *Pp;
  __syncthreads();
  const BucketParams P = sP;
  const int ncells = P.g[0] * P.g[1] * P.g[2];
  if (phase == 0 && blockIdx.x == 0 && threadIdx.x == 0) count[ncells] = 0;
  const double hd = 0.5 * P.h * 1.7320508075688772 * 1.001;
  for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < ncells; cell += gridDim.x * blockDim.x) {
    const d3 c = bucket_center(P, cell);
    TopK<K> top;
    top.init(K);
    bucket_knn<K>(P, cell_start, sorted, c, top);
    const double R = sqrt(top.worst_d()) + 2.0 * hd;
    const double R2 = R * R * (1.0 + 1e-9) + 1e-300;
    const double cq[3] = {c.x, c.y, c.z};
    int lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = clampi((int)floor((cq[a] - R - P.origin[a]) / P.h), 0, P.g[a] - 1);
      hi[a] = clampi((int)floor((cq[a] + R - P.origin[a]) / P.h), 0, P.g[a] - 1);
    }
    int m = 0;
    int64_t base = 0;
    bool ok = true;
    if (phase == 1) {
      base = count[cell];
      ok = len[cell] >= 0 && base + len[cell] <= cap;
      if (!ok) {
        len[cell] = -1;  // list does not fit: queries of this cell use the ring search
        continue;
      }
    }
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y) {
        const int row = (z * P.g[1] + y) * P.g[0];
        const int b = cell_start[row + lo[0]], e = cell_start[row + hi[0] + 1];
        for (int t = b; t < e; ++t) {
          const double4 s = sorted[t];
          if (sqdist(c, d3{s.x, s.y, s.z}) <= R2) {
            if (phase == 1) ids[base + m] = (int)s.w;
            ++m;
          }
        }
      }
    if (phase == 0) {
      count[cell] = m;
      len[cell] = m;
    }
  }
}

// exact k-NN of p from its cell's candidate list; false if p is outside the
// grid box or the list was not materialised (caller falls back to the ring search)
template <int K>
__device__ __forceinline__ bool ccl_knn(const BucketParams& P, const int* __restrict__ start,
                                        const int* __restrict__ len, const int* __restrict__ ids,
                                        const double* __restrict__ pts, d3 p, TopK<K>& top) {
  const double q[3] = {p.x, p.y, p.z};
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double f = (q[a] - P.origin[a]) / P.h;
    if (!(f >= 0.0) || f > (double)P.g[a]) return false;
    c[a] = clampi((int)f, 0, P.g[a] - 1);
  }
  const int cell = (c[2] * P.g[1] + c[1]) * P.g[0] + c[0];
  const int L = len[cell];
  if (L < 0) return false;
  const int b = start[cell];
  for (int j = 0; j < L; ++j) {
    const int id = ids[b + j];
    top.insert(sqdist(p, load_d3(pts + 3 * (int64_t)id)), id);
  }
  return true;
}

// ------------------------------------------------------------------ k-NN + blend

struct WarpArgs {
  const double* anchors;
  const double* dqs;
  int n_nodes;
  int k;
  double r2;  // radius * radius
  int mode;
  const double* pts;
  int64_t n_pts;
  int64_t* idx_out;
  double* w_out;
  double* pc_out;
  uint8_t* valid_out;
};

template <int K>
__device__ __forceinline__ void finish_query(const WarpArgs& A, int64_t q, d3 p, const TopK<K>& top) {
  double w[K];
  bool valid = false;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j < A.k) {
      // np.exp(-d2 / (r * r))
      w[j] = exp(ExactDiv(A.r2)(-top.d[j]));
      valid |= w[j] > kWeightFloor;
    }
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j < A.k) {
      if (A.idx_out) A.idx_out[q * A.k + j] = top.i[j];
      if (A.w_out) A.w_out[q * A.k + j] = w[j];
    }
  if (A.valid_out) A.valid_out[q] = valid ? 1 : 0;
  if (A.mode == CF_NEIGHBORS_ONLY || !A.pc_out) return;
  DqbAcc acc;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j < A.k) {
      double wj;
      if (A.mode == CF_BRUTE_QUERY)
        wj = fmax(w[j], 1e-300);  // knnfield.py:41
      else
        wj = valid ? w[j] : 1.0;  // edgraph.py:149
      acc.add(wj, load_dq(A.dqs + 8 * (int64_t)top.i[j]));
    }
  dq8 b = acc.result();
  if (A.mode != CF_WARP_FORWARD) b = dq_conj(b);
  store_d3(A.pc_out + 3 * q, dq_apply(b, p));
}

template <int K>
__global__ void __launch_bounds__(128, 4) knn_brute_kernel(WarpArgs A) {
  constexpr int TILE = 512;
  __shared__ double4 tile[TILE];
  const int64_t nblk = (A.n_pts + blockDim.x - 1) / blockDim.x;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t q = blk * blockDim.x + threadIdx.x;
    const bool live = q < A.n_pts;
    d3 p = live ? load_d3(A.pts + 3 * q) : d3{0.0, 0.0, 0.0};
    TopK<K> top;
    top.init(A.k);
    for (int base = 0; base < A.n_nodes; base += TILE) {
      const int cnt = min(TILE, A.n_nodes - base);
      __syncthreads();
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const double* a = A.anchors + 3 * (int64_t)(base + t);
        tile[t] = make_double4(a[0], a[1], a[2], 0.0);
      }
      __syncthreads();
      if (live)
        for (int t = 0; t < cnt; ++t) {
          const double4 s = tile[t];
          top.insert(sqdist(p, d3{s.x, s.y, s.z}), base + t);
        }
    }
    if (live) finish_query<K>(A, q, p, top);
  }
}

template <int K>
__global__ void __launch_bounds__(128, 4) knn_bucket_kernel(WarpArgs A, const BucketParams* __restrict__ Pp,
                                                         const int* __restrict__ cell_start,
                                                         const double4* __restrict__ sorted,
                                                         const int* __restrict__ ccl_start,
                                                         const int* __restrict__ ccl_len,
                                                         const int* __restrict__ ccl_ids) {
  __shared__ BucketParams sP;
  if (threadIdx.x == 0) sP = *Pp;
  __syncthreads();
  const BucketParams P = sP;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < A.n_pts; q += (int64_t)gridDim.x * blockDim.x) {
    const d3 p = load_d3(A.pts + 3 * q);
    TopK<K> top;
    top.init(A.k);
    if (!ccl_ids || !ccl_knn<K>(P, ccl_start, ccl_len, ccl_ids, A.anchors, p, top))
      bucket_knn<K>(P, cell_start, sorted, p, top);
    finish_query<K>(A, q, p, top);
  }
}

// Hierarchical exact k-NN for graphs of up to 8192 nodes: the queries are
// visited in a spatial order (`order`, e.g. Morton codes of the query cells) so
// a warp's 32 queries are neighbours; the warp culls the nodes against its
// queries' bounding box and ranks the survivors per lane, fp32 first and
// float64 for the final top-k (edwarp.cuh cull_topk). The fp32 copies of the
// nodes live in shared memory (16 B / node); the float64 coordinates are read
// from global memory for the few survivors. Results are written at the
// original query index: identical to the exhaustive kernel.
constexpr int kCullMaxNodes = 8192;
template <int K>
__global__ void __launch_bounds__(256) knn_cull_kernel(WarpArgs A, const int* __restrict__ order) {
  extern __shared__ float4 s_af[];
  __shared__ unsigned s_mag;
  if (threadIdx.x == 0) s_mag = 0u;
  __syncthreads();
  float mag = 0.f;
  for (int i = threadIdx.x; i < A.n_nodes; i += blockDim.x) {
    const double* a = A.anchors + 3 * (int64_t)i;
    const float x = (float)a[0], y = (float)a[1], z = (float)a[2];
    s_af[i] = make_float4(x, y, z, 0.f);
    mag = fmaxf(mag, fmaxf(fabsf(x), fmaxf(fabsf(y), fabsf(z))));
  }
  atomicMax(&s_mag, __float_as_uint(mag));
  __syncthreads();
  if (threadIdx.x == 0) s_af[0].w = __uint_as_float(s_mag);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (A.n_pts + 31) / 32;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w < n_warps; w += wstride) {
    const int64_t slot = w * 32 + lane;
    const bool live = slot < A.n_pts;
    const int64_t q = live ? (order ? (int64_t)order[slot] : slot) : 0;
    const d3 p = live ? load_d3(A.pts + 3 * q) : d3{0.0, 0.0, 0.0};
    TopK<K> top;
    cull_topk<K, 13>([&](int i) { return load_d3(A.anchors + 3 * (int64_t)i); }, s_af, A.n_nodes, A.k, p, live,
                     top);
    if (live) finish_query<K>(A, q, p, top);
  }
}

template <int K>
int launch_knn(const cf_buckets* b, const WarpArgs& A, cudaStream_t st) {
  const int block = 128;
  if (b) {
    const bool ccl = b->ccl_k >= K;
    knn_bucket_kernel<K><<<cf::grid_for(A.n_pts, block, 8), block, 0, st>>>(
        A, b->params, b->cell_start, b->sorted, ccl ? b->ccl_count : nullptr, ccl ? b->ccl_len : nullptr,
        ccl ? b->ccl_ids : nullptr);
  } else {
    knn_brute_kernel<K><<<cf::grid_for(A.n_pts, block, 8), block, 0, st>>>(A);
  }
  return cf::check_launch("knn_warp");
}

}  // namespace

namespace cf {

int buckets_build(cf_buckets* b, const double* pts, int64_t n, int grid_res, cudaStream_t st) {
  if (!b || n < 1 || n > b->max_points) return fail(CF_E_BAD_ARG, "buckets_build: bad handle or point count");
  int G = grid_res;
  if (G <= 0) G = (int)std::ceil(std::cbrt((double)n / 2.0) * 2.0);
  G = std::max(1, std::min(G, b->max_grid_res));
  b->grid_res = G;
  b->ccl_k = 0;  // candidate lists describe the previous point set
  const int64_t cells = (int64_t)G * G * G;
  if (n >= 2048 && n <= 65536 && cells + 1 <= kSmemBucketCells) {
    const size_t smem = sizeof(int) * (size_t)(cells + 1);
    CF_CHECK_CUDA(cudaFuncSetAttribute(bucket_build_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(int) * kSmemBucketCells)));
    cf::launch_pdl(bucket_build_cluster_kernel, kBucketCluster, 1024, smem, st, pts, (int)n, G, b->params,
                   b->cell_start, b->point_cell, b->point_slot, b->sorted);
    return check_launch("buckets_build");
  }
  if (n <= 65536 && cells + 1 <= kSmemBucketCells) {
    const size_t smem = sizeof(int) * (size_t)(cells + 1);
    CF_CHECK_CUDA(cudaFuncSetAttribute(bucket_build_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(int) * kSmemBucketCells)));
    cf::launch_pdl(bucket_build_smem_kernel, 1, 1024, smem, st, pts, (int)n, G, b->params, b->cell_start,
                   b->point_cell, b->point_slot, b->sorted);
    return check_launch("buckets_build");
  }
  if (n <= 65536 && cells <= (1 << 18)) {
    cf::launch_pdl(bucket_build_small_kernel, 1, 1024, 0, st, pts, (int)n, G, b->params, b->cell_start, b->point_cell,
                                                  b->point_slot, b->sorted);
    return check_launch("buckets_build");
  }
  cf::fill_list(st, {{b->cell_start, 0u, cells + 1}});
  bucket_params_kernel<<<1, 1024, 0, st>>>(pts, (int)n, G, b->params);
  bucket_count_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(pts, (int)n, b->params, b->cell_start, b->point_cell,
                                                             b->point_slot);
  bucket_scan_kernel<<<1, 1024, 0, st>>>(b->cell_start, b->params);
  bucket_scatter_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(pts, (int)n, b->cell_start, b->point_cell,
                                                               b->point_slot, b->sorted);
  return check_launch("buckets_build");
}

}  // namespace cf

extern "C" {

int cf_deform_nodes(const double* nodes, const double* dqs, int64_t n, double* anchors, void* stream) {
  if (n < 0 || (n > 0 && (!nodes || !dqs || !anchors))) return cf::fail(CF_E_BAD_ARG, "cf_deform_nodes: bad args");
  if (n == 0) return CF_OK;
  cf::launch_pdl(deform_nodes_kernel, cf::grid_for(n, 128, 4), 128, 0, cf::as_stream(stream), nodes, dqs, n, anchors);
  return cf::check_launch("cf_deform_nodes");
}

int cf_dq_blend(const double* weights, const double* dqs, int64_t n, int k, double* out, int* err, void* stream) {
  if (n < 0 || k < 0 || (n > 0 && (!out || (k > 0 && (!weights || !dqs)))))
    return cf::fail(CF_E_BAD_ARG, "cf_dq_blend: bad args");
  if (n == 0) return CF_OK;
  dq_blend_kernel<<<cf::grid_for(n, 128, 8), 128, 0, cf::as_stream(stream)>>>(weights, dqs, n, k, out, err);
  return cf::check_launch("cf_dq_blend");
}

int cf_dq_status(const int* err, void* stream) {
  if (!err) return cf::fail(CF_E_BAD_ARG, "cf_dq_status: bad args");
  int h = 0;
  CF_CHECK_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, cf::as_stream(stream)));
  CF_CHECK_CUDA(cudaStreamSynchronize(cf::as_stream(stream)));
  if (h == 2) return cf::fail(CF_E_BAD_ARG, "blend weights must be nonnegative");
  if (h == 1) return cf::fail(CF_E_DEGENERATE, "all blend weights are zero");
  return CF_OK;
}

int cf_dq_apply(const double* dq, int64_t dq_stride, const double* p, int64_t p_stride, int64_t n, double* out,
                void* stream) {
  if (n < 0 || (n > 0 && (!dq || !p || !out)) || dq_stride < 0 || p_stride < 0)
    return cf::fail(CF_E_BAD_ARG, "cf_dq_apply: bad args");
  if (n == 0) return CF_OK;
  dq_apply_kernel<<<cf::grid_for(n, 128, 8), 128, 0, cf::as_stream(stream)>>>(dq, dq_stride, p, p_stride, n, out);
  return cf::check_launch("cf_dq_apply");
}

int cf_cand_grid_bytes(int grid_res, int cmax, int64_t* bytes) {
  if (grid_res < 1 || grid_res > 128 || cmax < 1 || cmax > 4096 || !bytes)
    return cf::fail(CF_E_BAD_ARG, "cf_cand_grid_bytes: bad args");
  *bytes = 64 + (int64_t)grid_res * grid_res * grid_res * cand_stride(cmax) * 2;
  return CF_OK;
}

int cf_cand_grid_build(const void* block, int64_t n, int k, double radius, int grid_res, int cmax, void* cand,
                       void* stream) {
  if (!block || !cand || n < 1 || n > 1024 || k < 1 || k > 8 || !(radius > 0) || grid_res < 1 || grid_res > 128 ||
      cmax < 1 || cmax > 4096)
    return cf::fail(CF_E_BAD_ARG, "cf_cand_grid_build: bad args");
  const int64_t cells = (int64_t)grid_res * grid_res * grid_res;  // (upper bound of the grid's cells)
  // one thread per cell, 64-thread CTAs over the grid's upper bound of cells (the
  // frame's actual grid is known on the device only; surplus CTAs exit at once)
  const unsigned grid = (unsigned)std::max<int64_t>(1, (cells + 63) / 64);
  cudaStream_t st = cf::as_stream(stream);
  dispatch_k(k, [&]<int K>() {
    cf::launch_pdl(cand_grid_kernel<K>, grid, 64, (size_t)n * sizeof(float4), st, static_cast<const uint8_t*>(block),
                   (int)n, k, radius * radius, grid_res, cmax, static_cast<uint8_t*>(cand));
    return 0;
  });
  return cf::check_launch("cf_cand_grid_build");
}

int cf_anchor_block_bytes(int64_t n, int64_t* bytes) {
  if (n < 0 || !bytes) return cf::fail(CF_E_BAD_ARG, "cf_anchor_block_bytes: bad args");
  *bytes = 48 * n + 48;
  return CF_OK;
}

int cf_deform_nodes_block(const double* nodes, const double* dqs, int64_t n, double* anchors, void* block,
                          void* stream) {
  if (n < 1 || n > 1024 || !nodes || !dqs || !anchors || !block || reinterpret_cast<uintptr_t>(block) % 16 != 0)
    return cf::fail(CF_E_BAD_ARG, "cf_deform_nodes_block: bad args (1 <= n <= 1024, 16-byte aligned block)");
  cf::launch_pdl(deform_nodes_block_kernel, 1, 1024, 0, cf::as_stream(stream), nodes, dqs, (int)n, anchors,
                 static_cast<uint8_t*>(block));
  return cf::check_launch("cf_deform_nodes_block");
}

// The handle's buffers come from the stream-ordered allocator, so a handle can be
// destroyed on a stream without a host synchronisation (cf_buckets_destroy_async):
// the frees are ordered after the work already queued on that stream.
int cf_buckets_create(int64_t max_points, int max_grid_res, cf_buckets_t** out) {
  if (!out || max_points < 1 || max_grid_res < 1 || max_grid_res > 256)
    return cf::fail(CF_E_BAD_ARG, "cf_buckets_create: bad args");
  cf_buckets* b = new cf_buckets();
  b->max_points = max_points;
  b->max_grid_res = max_grid_res;
  const int64_t cells = (int64_t)max_grid_res * max_grid_res * max_grid_res;
  cudaStream_t st = 0;
  auto alloc = [&](void** p, size_t bytes) { return cudaMallocAsync(p, bytes, st); };
  cudaError_t e = alloc(reinterpret_cast<void**>(&b->params), sizeof(BucketParams));
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&b->cell_start), sizeof(int) * (cells + 1));
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&b->point_cell), sizeof(int) * max_points);
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&b->point_slot), sizeof(int) * max_points);
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&b->sorted), sizeof(double4) * max_points);
  b->ccl_cap = std::max<int64_t>(max_points * 64, 1 << 20);
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&b->ccl_count), sizeof(int) * (cells + 1));
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&b->ccl_len), sizeof(int) * cells);
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&b->ccl_ids), sizeof(int) * b->ccl_cap);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // usable from every stream
  if (e != cudaSuccess) {
    cf_buckets_destroy(b);
    return cf::fail(CF_E_CUDA, std::string("cf_buckets_create: ") + cudaGetErrorString(e));
  }
  *out = b;
  return CF_OK;
}

int cf_buckets_destroy_async(cf_buckets_t* b, void* stream) {
  if (!b) return CF_OK;
  cudaStream_t st = cf::as_stream(stream);
  void* ptrs[] = {b->params, b->cell_start, b->point_cell, b->point_slot, b->sorted, b->ccl_count, b->ccl_len,
                  b->ccl_ids};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, st);
  delete b;
  return cf::check_launch("cf_buckets_destroy_async");
}

int cf_buckets_destroy(cf_buckets_t* b) {
  if (!b) return CF_OK;
  const int rc = cf_buckets_destroy_async(b, nullptr);
  cudaStreamSynchronize(0);
  return rc;
}

int cf_buckets_build_candidates(cf_buckets_t* b, int k, void* stream) {
  if (!b || b->grid_res == 0 || k < 1) return cf::fail(CF_E_BAD_ARG, "cf_buckets_build_candidates: bad args");
  cudaStream_t st = cf::as_stream(stream);
  const int64_t cells = (int64_t)b->grid_res * b->grid_res * b->grid_res;
  const unsigned grid = cf::grid_for(cells, 128, 8);
  b->ccl_k = 0;
  const int rc = dispatch_k(k, [&]<int K>() {
    ccl_kernel<K><<<grid, 128, 0, st>>>(b->params, b->cell_start, b->sorted, 0, b->ccl_count, b->ccl_len, nullptr,
                                        b->ccl_cap);
    bucket_scan_kernel<<<1, 1024, 0, st>>>(b->ccl_count, b->params);
    ccl_kernel<K><<<grid, 128, 0, st>>>(b->params, b->cell_start, b->sorted, 1, b->ccl_count, b->ccl_len,
                                        b->ccl_ids, b->ccl_cap);
    return 0;
  });
  if (rc < 0) return cf::fail(CF_E_BAD_ARG, "cf_buckets_build_candidates: k must be 1..8 or 16");
  b->ccl_k = k;
  return cf::check_launch("cf_buckets_build_candidates");
}

int cf_buckets_build(cf_buckets_t* b, const double* pts, int64_t n, int grid_res, void* stream) {
  return cf::buckets_build(b, pts, n, grid_res, cf::as_stream(stream));
}

int cf_knn_warp_cull(const double* anchors, const double* dqs, int64_t n_nodes, int k, double radius, int mode,
                     const double* pts, const int* order, int64_t n_pts, int64_t* idx_out, double* w_out,
                     double* pc_out, uint8_t* valid_out, void* stream) {
  if (n_nodes < 1 || n_nodes > kCullMaxNodes)
    return cf::fail(CF_E_BAD_ARG, "cf_knn_warp_cull: 1 <= n_nodes <= 8192 (use the bucketed cf_knn_warp above)");
  if (mode < CF_WARP_BACKWARD || mode > CF_NEIGHBORS_ONLY) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp_cull: bad mode");
  if (!(radius > 0.0)) return cf::fail(CF_E_BAD_ARG, "influence radius must be positive");
  if (k < 1) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp_cull: k must be >= 1");
  if (k > n_nodes) k = (int)n_nodes;
  if (mode != CF_NEIGHBORS_ONLY && !dqs) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp_cull: dqs required");
  if (n_pts == 0) return CF_OK;
  WarpArgs A{anchors, dqs, (int)n_nodes, k, radius * radius, mode, pts, n_pts, idx_out, w_out, pc_out, valid_out};
  cudaStream_t st = cf::as_stream(stream);
  const size_t smem = sizeof(float4) * (size_t)n_nodes;
  const int rc = dispatch_k(k, [&]<int K>() {
    if (K > 8) return -1;  // the K+2 key list lives in registers
    CF_CHECK_CUDA(cudaFuncSetAttribute(knn_cull_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(float4) * kCullMaxNodes)));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, knn_cull_kernel<K>, 256, smem);
    const int64_t warps = (n_pts + 31) / 32;
    int64_t grid = std::min<int64_t>((warps + 7) / 8, (int64_t)cf::sm_count() * std::max(per_sm, 1));
    knn_cull_kernel<K><<<(unsigned)std::max<int64_t>(grid, 1), 256, smem, st>>>(A, order);
    return cf::check_launch("cf_knn_warp_cull");
  });
  if (rc < 0) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp_cull: k must be 1..8");
  return rc;
}

int cf_knn_warp(const cf_buckets_t* buckets, const double* anchors, const double* dqs, int64_t n_nodes, int k,
                double radius, int mode, const double* pts, int64_t n_pts, int64_t* idx_out, double* w_out,
                double* pc_out, uint8_t* valid_out, void* stream) {
  if (n_nodes < 1 || n_nodes > (1LL << 30)) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp: graph needs at least one node");
  if (mode < CF_WARP_BACKWARD || mode > CF_NEIGHBORS_ONLY) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp: bad mode");
  if (!(radius > 0.0)) return cf::fail(CF_E_BAD_ARG, "influence radius must be positive");
  if (k < 1) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp: k must be >= 1");
  if (k > n_nodes) k = (int)n_nodes;  // edgraph.py:43, knnfield.py:27
  if (k > 16) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp: k > 16 unsupported");
  if (mode != CF_NEIGHBORS_ONLY && !dqs) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp: dqs required");
  if (buckets && buckets->grid_res == 0) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp: buckets not built");
  if (n_pts == 0) return CF_OK;
  WarpArgs A{anchors, dqs, (int)n_nodes, k, radius * radius, mode, pts, n_pts, idx_out, w_out, pc_out, valid_out};
  cudaStream_t st = cf::as_stream(stream);
  const int rc = dispatch_k(k, [&]<int K>() { return launch_knn<K>(buckets, A, st); });
  if (rc < 0) return cf::fail(CF_E_BAD_ARG, "cf_knn_warp: k must be 1..8 or 16");
  return rc;
}

}  // extern "C"
