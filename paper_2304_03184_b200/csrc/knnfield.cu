// Constant-time motion-prior lookup (the paper's "LUT-based fast search"):
//   canonical s-NN voxel field      KnnField._build_canonical_field  knnfield.py:93-120
//   per-frame live map + collision  KnnField.update_live_map         knnfield.py:124-167
//   one-ring dilation               KnnField._dilate_once            knnfield.py:169-188
//   O(1) per-sample query           KnnField.query_motion_batch      knnfield.py:197-222
// Layout in HBM: neighbor_idx (r^3, s) int32 x-major (flat = i*r*r + j*r + k),
// live map (r^3) int32, -1 = empty — built dense in a scratch buffer shared by all
// frames and kept per frame as 8^3 bricks (brick table + the occupied bricks). The collision rule "nearest warped centre
// wins, ties -> smaller canonical voxel" is a two-phase atomicMin: first on the
// float64 distance bits (order-preserving for non-negative doubles), then on the
// canonical index among the exact-distance winners.
#include "dq.cuh"
#include "topk.cuh"

namespace {

struct Grid {
  double bmin[3];
  double voxel;
  int res;
};

__device__ __forceinline__ d3 voxel_center(const Grid& g, int64_t flat) {
  const int64_t r = g.res;
  const int64_t x = flat / (r * r), y = (flat / r) % r, z = flat % r;
  // bbox_min + (ijk + 0.5) * voxel_size   (knnfield.py:78-84)
  return d3{x_add(g.bmin[0], x_mul((double)x + 0.5, g.voxel)), x_add(g.bmin[1], x_mul((double)y + 0.5, g.voxel)),
            x_add(g.bmin[2], x_mul((double)z + 0.5, g.voxel))};
}

// floor((p - bbox_min) / voxel_size) with inside flag and clip (knnfield.py:86-91)
__device__ __forceinline__ int64_t flat_index(const Grid& g, d3 p, bool& inside, int64_t ijk[3]) {
  const double q[3] = {p.x, p.y, p.z};
  inside = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double f = floor(x_div(x_sub(q[a], g.bmin[a]), g.voxel));
    f = fmin(fmax(f, -1.0), (double)g.res);
    int64_t v = (int64_t)f;
    inside &= (v >= 0) && (v < g.res);
    ijk[a] = v < 0 ? 0 : (v > g.res - 1 ? g.res - 1 : v);
  }
  return (ijk[0] * g.res + ijk[1]) * g.res + ijk[2];
}

// Expanded-form squared distance of the canonical field build:
// sum(c*c) + |n|^2 - 2 * (c @ n), where the BLAS dot is an FMA chain
// fma(c2, n2, fma(c1, n1, c0*n0)) (matches OpenBLAS dgemm on K=3).
template <int K>
__global__ void __launch_bounds__(128, 4) field_build_kernel(const double* __restrict__ nodes, int n, int s, Grid g,
                                                          double sup2, int32_t* __restrict__ out) {
  constexpr int TILE = 512;
  __shared__ double4 tile[TILE];  // (x, y, z, |n|^2)
  const int64_t total = (int64_t)g.res * g.res * g.res;
  const int64_t nblk = (total + blockDim.x - 1) / blockDim.x;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t v = blk * blockDim.x + threadIdx.x;
    const bool live = v < total;
    const d3 c = voxel_center(g, live ? v : 0);
    const double cc = x_add(x_add(x_mul(c.x, c.x), x_mul(c.y, c.y)), x_mul(c.z, c.z));
    TopK<K> top;
    top.init(s);
    for (int base = 0; base < n; base += TILE) {
      const int cnt = min(TILE, n - base);
      __syncthreads();
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const double* a = nodes + 3 * (int64_t)(base + t);
        tile[t] = make_double4(a[0], a[1], a[2], x_add(x_add(x_mul(a[0], a[0]), x_mul(a[1], a[1])), x_mul(a[2], a[2])));
      }
      __syncthreads();
      if (live)
        for (int t = 0; t < cnt; ++t) {
          const double4 a = tile[t];
          const double dot = __fma_rn(c.z, a.z, __fma_rn(c.y, a.y, x_mul(c.x, a.x)));
          const double d2 = x_sub(x_add(cc, a.w), x_mul(2.0, dot));
          top.insert(d2, base + t);
        }
    }
    if (live) {
      const bool ok = top.d[0] <= sup2;
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (j < s) out[v * s + j] = ok ? top.i[j] : -1;
    }
  }
}

__global__ void live_init_kernel(uint64_t* __restrict__ best, uint32_t* __restrict__ winner, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    best[i] = ~0ull;
    winner[i] = 0xffffffffu;
  }
}

// Warp one in-support canonical voxel centre with canonical-distance weights.
__device__ __forceinline__ bool warp_voxel(const Grid& g, const double* __restrict__ nodes,
                                           const double* __restrict__ dqs, const int32_t* __restrict__ nbr_row, int s,
                                           double r2, int64_t k, int64_t& f, double& dist) {
  const d3 c = voxel_center(g, k);
  DqbAcc acc;
  for (int j = 0; j < s; ++j) {
    const int64_t nb = nbr_row[j];
    const double d2 = sqdist(c, load_d3(nodes + 3 * nb));
    const double w = fmax(exp(x_div(-d2, r2)), 1e-300);
    acc.add(w, load_dq(dqs + 8 * nb));
  }
  const d3 wp = dq_apply(acc.result(), c);
  bool inside;
  int64_t ijk[3];
  f = flat_index(g, wp, inside, ijk);
  const d3 lc{x_add(g.bmin[0], x_mul((double)ijk[0] + 0.5, g.voxel)),
              x_add(g.bmin[1], x_mul((double)ijk[1] + 0.5, g.voxel)),
              x_add(g.bmin[2], x_mul((double)ijk[2] + 0.5, g.voxel))};
  dist = sqdist(wp, lc);
  return inside;
}

__global__ void live_phase_kernel(const double* __restrict__ nodes, const double* __restrict__ dqs,
                                  const int32_t* __restrict__ nidx, int s, Grid g, double r2, int phase,
                                  uint64_t* __restrict__ best, uint32_t* __restrict__ winner) {
  const int64_t total = (int64_t)g.res * g.res * g.res;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* row = nidx + k * s;
    if (row[0] < 0) continue;
    int64_t f;
    double dist;
    if (!warp_voxel(g, nodes, dqs, row, s, r2, k, f, dist)) continue;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(dist);
    if (phase == 0)
      atomicMin((unsigned long long*)(best + f), bits);
    else if (best[f] == bits)
      atomicMin(winner + f, (uint32_t)k);
  }
}

// gather-only dilation from the pre-dilation map, neighbour order -x,+x,-y,+y,-z,+z
__global__ void live_dilate_kernel(const uint32_t* __restrict__ winner, int res, int32_t* __restrict__ live) {
  const int64_t r = res, total = r * r * r;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; f += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = (int32_t)winner[f];
    if (v < 0) {
      const int64_t i = f / (r * r), j = (f / r) % r, k = f % r;
      const int64_t stride[3] = {r * r, r, 1};
      const int64_t c[3] = {i, j, k};
#pragma unroll
      for (int a = 0; a < 3 && v < 0; ++a) {
        if (c[a] >= 1) {
          const int32_t u = (int32_t)winner[f - stride[a]];
          if (u >= 0) {
            v = u;
            break;
          }
        }
        if (c[a] <= r - 2) {
          const int32_t u = (int32_t)winner[f + stride[a]];
          if (u >= 0) {
            v = u;
            break;
          }
        }
      }
    }
    live[f] = v;
  }
}

// ---- sparse live maps: bricks of 8^3 voxels. brick_index (B^3 int32, B = ceil(res / 8),
// brick (bi, bj, bk) at (bi * B + bj) * B + bk) holds the brick's block number in
// `bricks` (512 int32 each, voxel (x, y, z) of the brick at (x * 8 + y) * 8 + z) or -1
// when every voxel of the brick is empty. A live map is mostly empty space (the body
// fills a few % of its bbox): 512 MiB dense per frame at 512^3 -> the occupied bricks.
constexpr int kBrick = 8;

__device__ __forceinline__ int32_t sparse_lookup(const int32_t* __restrict__ bidx, const int32_t* __restrict__ bricks,
                                                 int res, int64_t f) {
  const int64_t r = res, B = (r + kBrick - 1) / kBrick;
  const int64_t i = f / (r * r), j = (f / r) % r, k = f % r;
  const int32_t b = bidx[((i / kBrick) * B + j / kBrick) * B + k / kBrick];
  return b < 0 ? -1 : bricks[(int64_t)b * (kBrick * kBrick * kBrick) + ((i % kBrick) * kBrick + j % kBrick) * kBrick + k % kBrick];
}

// warp per brick: flag[b] = any voxel of the brick set
__global__ void brick_flag_kernel(const int32_t* __restrict__ live, int res, int32_t* __restrict__ flag) {
  const int64_t r = res, B = (r + kBrick - 1) / kBrick, nb = B * B * B;
  const int lane = threadIdx.x & 31;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < nb;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t bi = b / (B * B), bj = (b / B) % B, bk = b % B;
    bool any = false;
    for (int v = lane; v < kBrick * kBrick * kBrick; v += 32) {
      const int64_t i = bi * kBrick + v / (kBrick * kBrick), j = bj * kBrick + (v / kBrick) % kBrick,
                    k = bk * kBrick + v % kBrick;
      if (i < r && j < r && k < r) any |= live[(i * r + j) * r + k] >= 0;
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) flag[b] = any ? 1 : 0;
  }
}

// one CTA: exclusive scan of the flags -> block numbers (or -1), count -> n_out
__global__ void __launch_bounds__(1024) brick_scan_kernel(int32_t* __restrict__ idx, int64_t nb, int32_t* n_out) {
  __shared__ int32_t s_sum[1024];
  const int64_t per = (nb + blockDim.x - 1) / blockDim.x, lo = threadIdx.x * per, hi = min(lo + per, nb);
  int32_t c = 0;
  for (int64_t b = lo; b < hi; ++b) c += idx[b];
  s_sum[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // inclusive Hillis-Steele
    const int32_t v = threadIdx.x >= (unsigned)o ? s_sum[threadIdx.x - o] : 0;
    __syncthreads();
    s_sum[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = s_sum[threadIdx.x] - c;
  for (int64_t b = lo; b < hi; ++b) {
    const int32_t f = idx[b];
    idx[b] = f ? run : -1;
    run += f;
  }
  if (threadIdx.x == blockDim.x - 1) *n_out = s_sum[threadIdx.x];
}

// warp per brick: copy the set bricks' 512 voxels (voxels past the grid edge: -1)
__global__ void brick_pack_kernel(const int32_t* __restrict__ live, int res, const int32_t* __restrict__ bidx,
                                  int32_t* __restrict__ bricks) {
  const int64_t r = res, B = (r + kBrick - 1) / kBrick, nb = B * B * B;
  const int lane = threadIdx.x & 31;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < nb;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t o = bidx[b];
    if (o < 0) continue;
    const int64_t bi = b / (B * B), bj = (b / B) % B, bk = b % B;
    for (int v = lane; v < kBrick * kBrick * kBrick; v += 32) {
      const int64_t i = bi * kBrick + v / (kBrick * kBrick), j = bj * kBrick + (v / kBrick) % kBrick,
                    k = bk * kBrick + v % kBrick;
      bricks[(int64_t)o * (kBrick * kBrick * kBrick) + v] = (i < r && j < r && k < r) ? live[(i * r + j) * r + k] : -1;
    }
  }
}

__global__ void brick_unpack_kernel(const int32_t* __restrict__ bidx, const int32_t* __restrict__ bricks, int res,
                                    int32_t* __restrict__ live) {
  const int64_t r = res, total = r * r * r;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; f += (int64_t)gridDim.x * blockDim.x)
    live[f] = sparse_lookup(bidx, bricks, res, f);
}

// kSparse: the live map as brick_index (live) + bricks
template <int K, bool kSparse = false>
__global__ void __launch_bounds__(128, 4) query_kernel(const int32_t* __restrict__ live, const int32_t* __restrict__ nidx,
                                                    const double* __restrict__ dqs,
                                                    const double* __restrict__ anchors, int s, Grid g, double r2,
                                                    const double* __restrict__ pts, int64_t n, int64_t* nbr_out,
                                                    double* w_out, double* pc_out, uint8_t* valid_out,
                                                    const int32_t* __restrict__ bricks = nullptr) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const d3 p = load_d3(pts + 3 * q);
    bool inside;
    int64_t ijk[3];
    const int64_t f = flat_index(g, p, inside, ijk);
    int64_t kv = inside ? (int64_t)(kSparse ? sparse_lookup(live, bricks, g.res, f) : live[f]) : -1;
    bool valid = kv >= 0;
    const int64_t ks = valid ? kv : 0;
    int nb[K];
    double w[K];
    double wmax = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < s) {
        nb[j] = nidx[ks * s + j];
        const int64_t nsafe = nb[j] > 0 ? nb[j] : 0;
        const double d2 = sqdist(p, load_d3(anchors + 3 * nsafe));
        w[j] = nb[j] >= 0 ? exp(x_div(-d2, r2)) : 0.0;
        wmax = fmax(wmax, w[j]);
      }
    valid = valid && (wmax > 1e-6);
    DqbAcc acc;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < s) {
        const int64_t nsafe = nb[j] > 0 ? nb[j] : 0;
        acc.add(fmax(valid ? w[j] : 1.0, 1e-300), load_dq(dqs + 8 * nsafe));
      }
    const d3 pc = dq_apply(dq_conj(acc.result()), p);
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < s) {
        if (nbr_out) nbr_out[q * s + j] = nb[j];
        if (w_out) w_out[q * s + j] = w[j];
      }
    if (pc_out) store_d3(pc_out + 3 * q, pc);
    if (valid_out) valid_out[q] = valid ? 1 : 0;
  }
}

Grid make_grid(const double* bmin, double voxel, int res) {
  Grid g;
  for (int a = 0; a < 3; ++a) g.bmin[a] = bmin[a];
  g.voxel = voxel;
  g.res = res;
  return g;
}

}  // namespace

extern "C" {

int cf_knnfield_build(const double* nodes, int64_t n, int s, int res, const double* bbox_min, double voxel_size,
                      double support_radius, int32_t* neighbor_idx, void* stream) {
  if (res < 8) return cf::fail(CF_E_BAD_ARG, "resolution must be at least 8");
  if (n < 1 || s < 1 || !bbox_min || !(voxel_size > 0.0)) return cf::fail(CF_E_BAD_ARG, "cf_knnfield_build: bad args");
  if (s > n) s = (int)n;
  if (s > 16) return cf::fail(CF_E_BAD_ARG, "cf_knnfield_build: s > 16 unsupported");
  const Grid g = make_grid(bbox_min, voxel_size, res);
  const double sup2 = support_radius * support_radius;
  const int64_t total = (int64_t)res * res * res;
  cudaStream_t st = cf::as_stream(stream);
  const unsigned grid = cf::grid_for(total, 128, 8);
  if (dispatch_k(s, [&]<int K>() {
        field_build_kernel<K><<<grid, 128, 0, st>>>(nodes, (int)n, s, g, sup2, neighbor_idx);
        return 0;
      }) < 0)
    return cf::fail(CF_E_BAD_ARG, "cf_knnfield_build: s must be 1..8 or 16");
  return cf::check_launch("cf_knnfield_build");
}

int cf_knnfield_update(const double* nodes, const double* dqs, int64_t n, const int32_t* neighbor_idx, int s, int res,
                       const double* bbox_min, double voxel_size, double radius, int32_t* live_out,
                       uint64_t* scratch_u64, int32_t* scratch_i32, void* stream) {
  if (res < 8 || n < 1 || s < 1 || !scratch_u64 || !scratch_i32 || !live_out)
    return cf::fail(CF_E_BAD_ARG, "cf_knnfield_update: bad args");
  if (s > n) s = (int)n;
  const Grid g = make_grid(bbox_min, voxel_size, res);
  const int64_t total = (int64_t)res * res * res;
  cudaStream_t st = cf::as_stream(stream);
  const unsigned grid = cf::grid_for(total, 256, 8);
  uint32_t* winner = reinterpret_cast<uint32_t*>(scratch_i32);
  live_init_kernel<<<grid, 256, 0, st>>>(scratch_u64, winner, total);
  live_phase_kernel<<<grid, 256, 0, st>>>(nodes, dqs, neighbor_idx, s, g, radius * radius, 0, scratch_u64, winner);
  live_phase_kernel<<<grid, 256, 0, st>>>(nodes, dqs, neighbor_idx, s, g, radius * radius, 1, scratch_u64, winner);
  live_dilate_kernel<<<grid, 256, 0, st>>>(winner, res, live_out);
  return cf::check_launch("cf_knnfield_update");
}

static int knnfield_query(const int32_t* live, const int32_t* bricks, const int32_t* neighbor_idx,
                          const double* dqs_frame, const double* anchors_frame, int s, int res, const double* bbox_min,
                          double voxel_size, double radius, const double* pts, int64_t n_pts, int64_t* nbr_out,
                          double* w_out, double* pc_out, uint8_t* valid_out, void* stream) {
  if (res < 8 || s < 1 || s > 16 || !live || !neighbor_idx || !dqs_frame || !anchors_frame)
    return cf::fail(CF_E_BAD_ARG, "cf_knnfield_query: bad args");
  if (n_pts == 0) return CF_OK;
  const Grid g = make_grid(bbox_min, voxel_size, res);
  cudaStream_t st = cf::as_stream(stream);
  const unsigned grid = cf::grid_for(n_pts, 128, 8);
  const double r2 = radius * radius;
#define CF_Q(KK)                                                                                                    \
  do {                                                                                                              \
    if (bricks)                                                                                                     \
      query_kernel<KK, true><<<grid, 128, 0, st>>>(live, neighbor_idx, dqs_frame, anchors_frame, s, g, r2, pts,     \
                                                   n_pts, nbr_out, w_out, pc_out, valid_out, bricks);               \
    else                                                                                                            \
      query_kernel<KK, false><<<grid, 128, 0, st>>>(live, neighbor_idx, dqs_frame, anchors_frame, s, g, r2, pts,    \
                                                    n_pts, nbr_out, w_out, pc_out, valid_out);                      \
  } while (0)
  if (s <= 1) CF_Q(1);
  else if (s <= 2) CF_Q(2);
  else if (s <= 4) CF_Q(4);
  else if (s <= 8) CF_Q(8);
  else CF_Q(16);
#undef CF_Q
  return cf::check_launch("cf_knnfield_query");
}

int cf_knnfield_query(const int32_t* live, const int32_t* neighbor_idx, const double* dqs_frame,
                      const double* anchors_frame, int s, int res, const double* bbox_min, double voxel_size,
                      double radius, const double* pts, int64_t n_pts, int64_t* nbr_out, double* w_out,
                      double* pc_out, uint8_t* valid_out, void* stream) {
  return knnfield_query(live, nullptr, neighbor_idx, dqs_frame, anchors_frame, s, res, bbox_min, voxel_size, radius,
                        pts, n_pts, nbr_out, w_out, pc_out, valid_out, stream);
}

int cf_knnfield_query_sparse(const int32_t* brick_index, const int32_t* bricks, const int32_t* neighbor_idx,
                             const double* dqs_frame, const double* anchors_frame, int s, int res,
                             const double* bbox_min, double voxel_size, double radius, const double* pts,
                             int64_t n_pts, int64_t* nbr_out, double* w_out, double* pc_out, uint8_t* valid_out,
                             void* stream) {
  if (!bricks) return cf::fail(CF_E_BAD_ARG, "cf_knnfield_query_sparse: bad args");
  return knnfield_query(brick_index, bricks, neighbor_idx, dqs_frame, anchors_frame, s, res, bbox_min, voxel_size,
                        radius, pts, n_pts, nbr_out, w_out, pc_out, valid_out, stream);
}

int cf_knnfield_brick_count(int res, int64_t* n_bricks_total) {
  if (res < 8 || !n_bricks_total) return cf::fail(CF_E_BAD_ARG, "cf_knnfield_brick_count: bad args");
  const int64_t B = (res + kBrick - 1) / kBrick;
  *n_bricks_total = B * B * B;
  return CF_OK;
}

int cf_knnfield_brick_index(const int32_t* live_dense, int res, int32_t* brick_index, int32_t* n_set, void* stream) {
  if (res < 8 || !live_dense || !brick_index || !n_set) return cf::fail(CF_E_BAD_ARG, "cf_knnfield_brick_index: bad args");
  const int64_t B = (res + kBrick - 1) / kBrick, nb = B * B * B;
  cudaStream_t st = cf::as_stream(stream);
  brick_flag_kernel<<<cf::grid_for(nb * 32, 256, 8), 256, 0, st>>>(live_dense, res, brick_index);
  brick_scan_kernel<<<1, 1024, 0, st>>>(brick_index, nb, n_set);
  return cf::check_launch("cf_knnfield_brick_index");
}

int cf_knnfield_brick_pack(const int32_t* live_dense, int res, const int32_t* brick_index, int32_t* bricks,
                           void* stream) {
  if (res < 8 || !live_dense || !brick_index || !bricks) return cf::fail(CF_E_BAD_ARG, "cf_knnfield_brick_pack: bad args");
  const int64_t B = (res + kBrick - 1) / kBrick, nb = B * B * B;
  brick_pack_kernel<<<cf::grid_for(nb * 32, 256, 8), 256, 0, cf::as_stream(stream)>>>(live_dense, res, brick_index,
                                                                                        bricks);
  return cf::check_launch("cf_knnfield_brick_pack");
}

int cf_knnfield_brick_unpack(const int32_t* brick_index, const int32_t* bricks, int res, int32_t* live_dense,
                             void* stream) {
  if (res < 8 || !brick_index || !live_dense) return cf::fail(CF_E_BAD_ARG, "cf_knnfield_brick_unpack: bad args");
  const int64_t total = (int64_t)res * res * res;
  brick_unpack_kernel<<<cf::grid_for(total, 256, 8), 256, 0, cf::as_stream(stream)>>>(brick_index, bricks, res,
                                                                                       live_dense);
  return cf::check_launch("cf_knnfield_brick_unpack");
}

}  // extern "C"
