// Ray generation, occupancy grids, occupancy-skipped ray marching, sample
// canonicalisation and front-to-back compositing — the SPEC render path
// (volume_render SPEC.md:381-389, render_view SPEC.md:399-407,
// composite SPEC.md:555-563) with the occupancy skipping of DESIGN.md §6.
//
// Layouts in HBM: rays = one float64 origin + (R,3) float64 unit directions;
// occupancy = bit grid (res^3 bits, x-major flat index, 32 cells per word);
// compacted samples = uint32 record (ray << 8 | sample) grouped per ray in
// ascending sample order, with per-ray (offset, count); canonicalised samples
// = float4 (x, y, z in the field's unit cube, flag).
#include "edwarp.cuh"

namespace {

#ifndef CF_CANON_MINB
#define CF_CANON_MINB 5  // resident CTAs/SM the canonicalisation kernel is compiled for
#endif
// graphs up to this many nodes are scanned exhaustively from shared memory
// (cheaper than the bucket ring search's divergent loops at render sizes)
constexpr int kSmemAnchors = 1024;

__device__ __forceinline__ bool occ_test(const cf_occ_grid& g, const uint32_t* __restrict__ bits, d3 p) {
  // floor((p - min) * (1 / cell)): a multiply by the correctly rounded
  // reciprocal instead of a float64 division (the oracle uses the same formula)
  const double q[3] = {p.x, p.y, p.z};
  const double inv = 1.0 / g.cell;
  int64_t c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double f = floor(x_mul(x_sub(q[a], g.min[a]), inv));
    if (!(f >= 0.0) || f >= (double)g.res) return false;
    c[a] = (int64_t)f;
  }
  const int64_t flat = (c[0] * g.res + c[1]) * g.res + c[2];
  return (__ldg(bits + (flat >> 5)) >> (flat & 31)) & 1u;
}

// occ_test split in two for batched lookups: the flat cell index (-1 outside the
// grid), branch-free, with the reciprocal hoisted by the caller (same arithmetic)
__device__ __forceinline__ int64_t occ_flat(const cf_occ_grid& g, double inv, d3 p) {
  const double q[3] = {p.x, p.y, p.z};
  bool ok = true;
  int64_t c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double f = floor(x_mul(x_sub(q[a], g.min[a]), inv));
    ok = ok && (f >= 0.0) && f < (double)g.res;
    c[a] = ok ? (int64_t)f : 0;
  }
  return ok ? (c[0] * g.res + c[1]) * g.res + c[2] : -1;
}

__device__ __forceinline__ d3 cell_center(const cf_occ_grid& g, int64_t flat) {
  const int64_t r = g.res;
  const int64_t x = flat / (r * r), y = (flat / r) % r, z = flat % r;
  return d3{x_add(g.min[0], x_mul((double)x + 0.5, g.cell)), x_add(g.min[1], x_mul((double)y + 0.5, g.cell)),
            x_add(g.min[2], x_mul((double)z + 0.5, g.cell))};
}

// t_i = t_near + (i + 0.5) * dt ;  p = o + t * d   (float64, un-contracted)
__device__ __forceinline__ double sample_t(const cf_march_desc& M, int i) {
  return x_add(M.t_near, x_mul((double)i + 0.5, M.dt));
}
// depth of compacted sample s: explicit (training sampler) or the uniform t_i
__device__ __forceinline__ double rec_t(const cf_march_desc& M, int64_t s, uint32_t rec) {
  return M.sample_t ? M.sample_t[s] : sample_t(M, (int)(rec & 255u));
}
// per-frame values into shared memory: origin s[0..2], object pose R s[3..11],
// t s[12..14] — from the device frame block when set (a captured graph replays
// frames by rewriting it), else from the by-value descriptor. Block-wide.
__device__ __forceinline__ void load_frame(const cf_march_desc& M, double* s) {
  if (threadIdx.x == 0) {  // constant indices only: no local copy of the by-value descriptor
#pragma unroll
    for (int i = 0; i < 3; ++i) s[i] = M.frame ? M.frame[i] : M.origin[i];
#pragma unroll
    for (int i = 0; i < 9; ++i) s[3 + i] = M.frame ? M.frame[3 + i] : M.obj_R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) s[12 + i] = M.frame ? M.frame[12 + i] : M.obj_t[i];
  }
  __syncthreads();
}

__device__ __forceinline__ d3 sample_p(d3 o, d3 d, double t) {
  return d3{x_add(o.x, x_mul(t, d.x)), x_add(o.y, x_mul(t, d.y)), x_add(o.z, x_mul(t, d.z))};
}
// object-local point R^T (p - t), summed ((R0i q0 + R1i q1) + R2i q2)
__device__ __forceinline__ d3 to_object(const double* R, const double* t, d3 p) {
  const double q0 = x_sub(p.x, t[0]), q1 = x_sub(p.y, t[1]), q2 = x_sub(p.z, t[2]);
  double o[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = x_add(x_add(x_mul(q0, R[i]), x_mul(q1, R[3 + i])), x_mul(q2, R[6 + i]));
  return d3{o[0], o[1], o[2]};
}

// camera parameters into shared memory: R[9], fx, fy, cx, cy — from the device
// block cam.params when set (graph replay), else the by-value fields. Block-wide.
__device__ __forceinline__ void load_camera(const cf_camera& cam, double* s_cam) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < 9; ++i) s_cam[i] = cam.params ? cam.params[i] : cam.R[i];
    s_cam[9] = cam.params ? cam.params[9] : cam.fx;
    s_cam[10] = cam.params ? cam.params[10] : cam.fy;
    s_cam[11] = cam.params ? cam.params[11] : cam.cx;
    s_cam[12] = cam.params ? cam.params[12] : cam.cy;
  }
  __syncthreads();
}

// unit direction of pixel i (camera.py:94-108: R (u-cx)/fx, (v-cy)/fy, 1), normalised
// local pixel i of a row shard: image row row0 + (i / width) * row_stride
__device__ __forceinline__ d3 pixel_dir(const double* s_cam, const ExactDiv& by_fx, const ExactDiv& by_fy, int width,
                                        int i, int row0 = 0, int row_stride = 1) {
  const int v_i = i / width;
  const double u = (double)(i - v_i * width), v = (double)(row0 + v_i * row_stride);
  const double dc[3] = {by_fx(x_sub(u, s_cam[11])), by_fy(x_sub(v, s_cam[12])), 1.0};
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    d[a] = __fma_rn(dc[2], s_cam[3 * a + 2], __fma_rn(dc[1], s_cam[3 * a + 1], x_mul(dc[0], s_cam[3 * a])));
  const ExactDiv by_nrm(sqrt(x_add(x_add(x_mul(d[0], d[0]), x_mul(d[1], d[1])), x_mul(d[2], d[2]))));
  return d3{by_nrm(d[0]), by_nrm(d[1]), by_nrm(d[2])};
}

__global__ void rays_kernel(cf_camera cam, double* __restrict__ dirs) {
  pdl_wait();
  __shared__ double s_cam[13];
  load_camera(cam, s_cam);
  const int n = cam.width * cam.height;
  const ExactDiv by_fx(s_cam[9]), by_fy(s_cam[10]);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    store_d3(dirs + 3 * (int64_t)i,
             pixel_dir(s_cam, by_fx, by_fy, cam.width, i, cam.row0, cam.row_stride > 0 ? cam.row_stride : 1));
  pdl_trigger();
}

// cells whose centre lies within `radius` of any bucketed point
__global__ void __launch_bounds__(128, 4) occ_points_kernel(cf_occ_grid g, const BucketParams* __restrict__ Pp,
                                                         const int* __restrict__ cell_start,
                                                         const double4* __restrict__ sorted, double r2,
                                                         uint32_t* __restrict__ bits) {
  __shared__ BucketParams sP;
  if (threadIdx.x == 0) sP = *Pp;
  __syncthreads();
  const int64_t total = (int64_t)g.res * g.res * g.res;
  const int64_t words = (total + 31) / 32;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x) & ~31LL; base < words * 32;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = base + (threadIdx.x & 31) + (threadIdx.x & ~31);
    bool on = false;
    if (cell < total) {
      TopK<1> top;
      top.init(1);
      bucket_knn<1>(sP, cell_start, sorted, cell_center(g, cell), top, r2);
      on = top.d[0] <= r2;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, on);
    if ((threadIdx.x & 31) == 0 && (cell >> 5) < words) bits[cell >> 5] = word;
  }
}

// solid origin-centred box dilated by shell: sdf(centre) <= shell
__global__ void occ_box_kernel(cf_occ_grid g, double hx, double hy, double hz, double shell, uint32_t* bits) {
  const int64_t total = (int64_t)g.res * g.res * g.res;
  const int64_t words = (total + 31) / 32;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x) & ~31LL; base < words * 32;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = base + (threadIdx.x & 31) + (threadIdx.x & ~31);
    bool on = false;
    if (cell < total) {
      const d3 c = cell_center(g, cell);
      const double q[3] = {x_sub(fabs(c.x), hx), x_sub(fabs(c.y), hy), x_sub(fabs(c.z), hz)};
      const double m0 = fmax(q[0], 0.0), m1 = fmax(q[1], 0.0), m2 = fmax(q[2], 0.0);
      const double o = sqrt(x_add(x_add(x_mul(m0, m0), x_mul(m1, m1)), x_mul(m2, m2)));
      const double in = fmin(fmax(q[0], fmax(q[1], q[2])), 0.0);
      on = x_add(o, in) <= shell;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, on);
    if ((threadIdx.x & 31) == 0 && (cell >> 5) < words) bits[cell >> 5] = word;
  }
}

// forward-warp every occupied canonical cell centre into live space and set
// the 3x3x3 block of live cells around it
template <int K>
__global__ void __launch_bounds__(128, 4) occ_splat_kernel(const uint32_t* __restrict__ cbits, cf_occ_grid cg,
                                                        const BucketParams* __restrict__ Pp,
                                                        const int* __restrict__ cell_start,
                                                        const double4* __restrict__ sorted,
                                                        const double* __restrict__ dqs, int k, double r2,
                                                        cf_occ_grid lg, uint32_t* __restrict__ lbits) {
  __shared__ BucketParams sP;
  if (threadIdx.x == 0) sP = *Pp;
  __syncthreads();
  const int64_t total = (int64_t)cg.res * cg.res * cg.res;
  for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell < total;
       cell += (int64_t)gridDim.x * blockDim.x) {
    if (!((cbits[cell >> 5] >> (cell & 31)) & 1u)) continue;
    d3 x;
    if (!ed_warp_point<K>(sP, cell_start, sorted, dqs, k, r2, false, cell_center(cg, cell), x)) continue;
    const double q[3] = {x.x, x.y, x.z};
    int64_t c[3];
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double f = floor(x_div(x_sub(q[a], lg.min[a]), lg.cell));
      ok &= (f >= -1.0) && (f <= (double)lg.res);
      c[a] = ok ? (int64_t)f : 0;
    }
    if (!ok) continue;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const int64_t a = c[0] + dx, b = c[1] + dy, z = c[2] + dz;
          if (a < 0 || b < 0 || z < 0 || a >= lg.res || b >= lg.res || z >= lg.res) continue;
          const int64_t f = (a * lg.res + b) * lg.res + z;
          atomicOr(lbits + (f >> 5), 1u << (f & 31));
        }
  }
}

// Sample indices whose t lies in the ray's [t_enter, t_exit] through box
// [lo, hi], widened by one sample on each side (a conservative superset: any
// sample outside it is outside the box, hence in no set cell). i0 > i1 = none.
__device__ __forceinline__ void sample_range(const cf_march_desc& M, d3 o, d3 d, const double* lo, const double* hi,
                                             int& i0, int& i1) {
  const double oq[3] = {o.x, o.y, o.z}, dq[3] = {d.x, d.y, d.z};
  double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (fabs(dq[a]) < 1e-300) {
      if (oq[a] < lo[a] || oq[a] > hi[a]) t0 = INFINITY;
      continue;
    }
    // any reciprocal within ~1e-7 relative will do: the index range below keeps a
    // one-sample margin (dt ~ cm) on both ends, far beyond the rounding of t0/t1
    const double inv = (double)__frcp_rn((float)dq[a]);
    double ta = (lo[a] - oq[a]) * inv, tb = (hi[a] - oq[a]) * inv;
    if (ta > tb) {
      const double s = ta;
      ta = tb;
      tb = s;
    }
    t0 = fmax(t0, ta);
    t1 = fmin(t1, tb);
  }
  if (!(t0 <= t1)) {
    i0 = 1;
    i1 = 0;
    return;
  }
  const double inv_dt = (double)__frcp_rn((float)M.dt);
  const double f0 = floor((t0 - M.t_near) * inv_dt - 0.5) - 1.0, f1 = ceil((t1 - M.t_near) * inv_dt - 0.5) + 1.0;
  i0 = (int)fmax(f0, 0.0);
  i1 = (int)fmin(f1, (double)(M.n_samples - 1));
}

// Static part of the forward warp of the occupied canonical cells (once per
// sequence): exact canonical k-NN and Gaussian weights, i.e. the reference's
// canonical_blend_info (edgraph.py:186-195). Compacted (order irrelevant).
template <int K>
__global__ void __launch_bounds__(128, 4) occ_cache_kernel(const uint32_t* __restrict__ cbits, cf_occ_grid cg,
                                                        const BucketParams* __restrict__ Pp,
                                                        const int* __restrict__ cell_start,
                                                        const double4* __restrict__ sorted, int k, double r2,
                                                        int64_t capacity, int* __restrict__ cell_out,
                                                        int* __restrict__ nbr_out, double* __restrict__ w_out,
                                                        int* __restrict__ count) {
  __shared__ BucketParams sP;
  if (threadIdx.x == 0) sP = *Pp;
  __syncthreads();
  const int64_t total = (int64_t)cg.res * cg.res * cg.res;
  for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell < total;
       cell += (int64_t)gridDim.x * blockDim.x) {
    if (!((cbits[cell >> 5] >> (cell & 31)) & 1u)) continue;
    TopK<K> top;
    top.init(k);
    bucket_knn<K>(sP, cell_start, sorted, cell_center(cg, cell), top);
    double w[K];
    bool valid = false;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < k) {
        w[j] = exp(x_div(-top.d[j], r2));
        valid |= w[j] > 1e-6;
      }
    if (!valid) continue;  // forward warp invalid: the cell is never splatted
    const int slot = atomicAdd(count, 1);
    if (slot >= capacity) continue;
    cell_out[slot] = (int)cell;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < k) {
        nbr_out[(int64_t)slot * k + j] = top.i[j];
        w_out[(int64_t)slot * k + j] = w[j];
      }
  }
}

// per frame: blend the cached neighbours' dqs, apply, set the centre live cell
template <int K>
__global__ void occ_splat_cached_kernel(const int* __restrict__ cells, const int* __restrict__ nbr,
                                        const double* __restrict__ w, const int* __restrict__ count,
                                        int64_t capacity, int k, const double* __restrict__ dqs, cf_occ_grid cg,
                                        cf_occ_grid lg, uint32_t* __restrict__ centre_bits, int* __restrict__ bbox) {
  pdl_wait();
  const int64_t n = min((int64_t)*count, capacity);
  int lo[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff}, hi[3] = {-0x7fffffff, -0x7fffffff, -0x7fffffff};
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    DqbAcc acc;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < k) acc.add(w[s * k + j], load_dq(dqs + 8 * (int64_t)nbr[s * k + j]));
    const d3 x = dq_apply(acc.result(), cell_center(cg, cells[s]));
    const double q[3] = {x.x, x.y, x.z};
    int64_t c[3];
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double f = floor(x_div(x_sub(q[a], lg.min[a]), lg.cell));
      ok &= (f >= -1.0) && (f <= (double)lg.res);
      c[a] = ok ? (int64_t)f : 0;
    }
    if (!ok) continue;
    // centre cell may lie one cell outside the grid: record it clamped into a
    // 1-cell-padded index space so the dilation still reaches the border cells
    const int64_t P = lg.res + 2;
    const int64_t f = ((c[0] + 1) * P + (c[1] + 1)) * P + (c[2] + 1);
    atomicOr(centre_bits + (f >> 5), 1u << (f & 31));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = min(lo[a], (int)c[a]);
      hi[a] = max(hi[a], (int)c[a]);
    }
  }
  if (!bbox) return;
  // centre bbox (warp-reduced); the dilate kernel widens it to the live-cell bbox
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if ((threadIdx.x & 31) == 0 && lo[a] <= hi[a]) {
      atomicMin(bbox + a, lo[a]);
      atomicMax(bbox + 3 + a, hi[a]);
    }
  }
  pdl_trigger();
}

__device__ __forceinline__ uint64_t window64(const uint32_t* __restrict__ bits, int64_t start) {
  const int64_t w = start >> 5;
  const int sh = (int)(start & 31);
  const uint64_t lo = (uint64_t)bits[w] | ((uint64_t)bits[w + 1] << 32);
  const uint64_t hi = bits[w + 2];
  return (lo >> sh) | (sh ? (hi << (64 - sh)) : 0ull);
}

// live = 3x3x3 dilation of the padded centre set, cropped to the grid
__global__ void occ_dilate_kernel(const uint32_t* __restrict__ centre_bits, int res, uint32_t* __restrict__ live,
                                  int* __restrict__ bbox) {
  pdl_wait();
  const int64_t r = res, P = r + 2, total = r * r * r;
  const int64_t words = (total + 31) / 32;
  if (bbox && blockIdx.x == 0 && threadIdx.x == 0) {
    // centre bbox -> live-cell bbox of the 3x3x3 dilation cropped to the grid
    for (int a = 0; a < 3; ++a) {
      const int lo = bbox[a], hi = bbox[3 + a];
      if (lo > hi) continue;
      bbox[a] = max(lo - 1, 0);
      bbox[3 + a] = min(hi + 1, res - 1);
    }
  }
  if ((res & 31) == 0) {  // rows are whole words: 9 row windows of 34 bits per output word
    const int64_t wpr = r / 32;
    for (int64_t wi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wi < words;
         wi += (int64_t)gridDim.x * blockDim.x) {
      const int64_t row = wi / wpr, kb = wi % wpr, i = row / r, j = row % r;
      uint64_t acc = 0;
#pragma unroll
      for (int di = 0; di < 3; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          const uint64_t win = window64(centre_bits, ((i + di) * P + (j + dj)) * P + kb * 32);
          acc |= win | (win >> 1) | (win >> 2);
        }
      live[wi] = (uint32_t)acc;
    }
    return;
  }
  for (int64_t wi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wi < words; wi += (int64_t)gridDim.x * blockDim.x) {
    uint32_t out = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t f = wi * 32 + b;
      if (f >= total) break;
      const int64_t i = f / (r * r) + 1, j = (f / r) % r + 1, kk = f % r + 1;
      bool on = false;
      for (int di = -1; di <= 1 && !on; ++di)
        for (int dj = -1; dj <= 1 && !on; ++dj) {
          const int64_t g = ((i + di) * P + (j + dj)) * P + kk;
          // three consecutive k bits g-1, g, g+1
          for (int dk = -1; dk <= 1; ++dk) {
            const int64_t h = g + dk;
            if ((centre_bits[h >> 5] >> (h & 31)) & 1u) {
              on = true;
              break;
            }
          }
        }
      if (on) out |= 1u << b;
    }
    live[wi] = out;
  }
  pdl_trigger();
}

// bbox of the set cells, one CTA (block-reduced, no host init needed)
__global__ void __launch_bounds__(1024) occ_bbox_kernel(const uint32_t* __restrict__ bits, cf_occ_grid g,
                                                        int* __restrict__ bbox) {
  __shared__ int s[6];
  if (threadIdx.x < 3) {
    s[threadIdx.x] = 0x7fffffff;
    s[3 + threadIdx.x] = -1;
  }
  __syncthreads();
  const int64_t r = g.res, total = r * r * r, words = (total + 31) / 32;
  int lo[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff}, hi[3] = {-1, -1, -1};
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) {
    uint32_t b = bits[w];
    while (b) {
      const int j = __ffs(b) - 1;
      b &= b - 1;
      const int64_t f = w * 32 + j;
      if (f >= total) break;
      const int c[3] = {(int)(f / (r * r)), (int)((f / r) % r), (int)(f % r)};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = min(lo[a], c[a]);
        hi[a] = max(hi[a], c[a]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&s[a], lo[a]);
      atomicMax(&s[3 + a], hi[a]);
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) bbox[threadIdx.x] = s[threadIdx.x];
}

__device__ __forceinline__ int warp_excl_scan(int v, int& total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// occupancy-skipped sample compaction, one thread per ray, up to two fields:
// occupancy masks of samples i0..i1 (< 128). Samples go in batches of 4 — cell
// indices first, then the 4 bit-word loads in flight together (one dependent load
// per sample was the march's latency chain) — and each hit is merged into the mask
// word by selects, so the masks stay in registers without unrolling a loop per word
// (a runtime word index would put them in local memory; four unrolled word loops
// blew the instruction cache).
template <class Flat>
__device__ __forceinline__ void scan_samples(int i0, int i1, Flat flat_of, const uint32_t* __restrict__ bits,
                                             uint32_t (&m)[4]) {
  m[0] = m[1] = m[2] = m[3] = 0u;
  for (int i = i0; i <= i1; i += 4) {
    int64_t f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) f[j] = i + j <= i1 ? flat_of(i + j) : -1;
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = f[j] >= 0 ? __ldg(bits + (f[j] >> 5)) : 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t b = (f[j] >= 0 ? (v[j] >> (f[j] & 31)) & 1u : 0u) << ((i + j) & 31);
      const int w = (i + j) >> 5;
      m[0] |= w == 0 ? b : 0u;
      m[1] |= w == 1 ? b : 0u;
      m[2] |= w == 2 ? b : 0u;
      m[3] |= w == 3 ? b : 0u;
    }
  }
}

// kRays: the march also generates the ray directions (one thread per pixel) and
// writes them to dirs for the later stages, instead of reading them
template <bool kRays>
__global__ void __launch_bounds__(128) march_kernel(cf_march_desc M, cf_camera cam, double* __restrict__ dirs,
                                                    const uint32_t* __restrict__ hbits,
                                                    const uint32_t* __restrict__ obits, cf_march_out H,
                                                    cf_march_out O) {
  pdl_wait();
  __shared__ double s_fr[15];
  __shared__ double s_cam[13];
  if (kRays) load_camera(cam, s_cam);
  load_frame(M, s_fr);
  const ExactDiv by_fx(kRays ? s_cam[9] : 1.0), by_fy(kRays ? s_cam[10] : 1.0);
  const double* obj_R = s_fr + 3;
  const double* obj_t = s_fr + 12;
  const d3 o{s_fr[0], s_fr[1], s_fr[2]};
  // boxes that contain every set cell: the live cell bbox, the object grid
  double hlo[3], hhi[3], olo[3], ohi[3];
  bool hempty = false;
  for (int a = 0; a < 3; ++a) {
    int lo = 0, hi = M.human_grid.res - 1;
    if (M.human_cell_bbox) {
      lo = M.human_cell_bbox[a];
      hi = M.human_cell_bbox[3 + a];
    }
    hempty |= lo > hi;
    hlo[a] = M.human_grid.min[a] + lo * M.human_grid.cell;
    hhi[a] = M.human_grid.min[a] + (hi + 1) * M.human_grid.cell;
    olo[a] = M.object_grid.min[a];
    ohi[a] = M.object_grid.min[a] + M.object_grid.res * M.object_grid.cell;
  }
  const d3 oo = to_object(obj_R, obj_t, o);
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < M.n_rays; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ray = base + threadIdx.x;
    const bool live = ray < M.n_rays;
    d3 d{0.0, 0.0, 1.0};
    if (live) {
      if (kRays) {
        d = pixel_dir(s_cam, by_fx, by_fy, cam.width, (int)ray, cam.row0, cam.row_stride > 0 ? cam.row_stride : 1);
        store_d3(dirs + 3 * ray, d);
      } else {
        d = load_d3(dirs + 3 * ray);
      }
    }
    uint32_t hm[4] = {0, 0, 0, 0}, om[4] = {0, 0, 0, 0};  // occupancy masks of up to 128 samples
    int hc = 0, oc = 0;
    if (live && hbits && !hempty) {
      int i0, i1;
      sample_range(M, o, d, hlo, hhi, i0, i1);
      const double inv = 1.0 / M.human_grid.cell;
      scan_samples(
          i0, i1, [&](int i) { return occ_flat(M.human_grid, inv, sample_p(o, d, sample_t(M, i))); }, hbits, hm);
      hc = __popc(hm[0]) + __popc(hm[1]) + __popc(hm[2]) + __popc(hm[3]);
    }
    if (live && obits) {
      // the object box is clipped in object space: ray (R^T (o - t), R^T d)
      const d3 od{d.x * obj_R[0] + d.y * obj_R[3] + d.z * obj_R[6],
                  d.x * obj_R[1] + d.y * obj_R[4] + d.z * obj_R[7],
                  d.x * obj_R[2] + d.y * obj_R[5] + d.z * obj_R[8]};
      int i0, i1;
      sample_range(M, oo, od, olo, ohi, i0, i1);
      const double inv = 1.0 / M.object_grid.cell;
      scan_samples(
          i0, i1,
          [&](int i) { return occ_flat(M.object_grid, inv, to_object(obj_R, obj_t, sample_p(o, d, sample_t(M, i)))); },
          obits, om);
      oc = __popc(om[0]) + __popc(om[1]) + __popc(om[2]) + __popc(om[3]);
    }
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const cf_march_out& out = f == 0 ? H : O;
      if (!out.records) continue;
      const int c = f == 0 ? hc : oc;
      const uint32_t m[4] = {f == 0 ? hm[0] : om[0], f == 0 ? hm[1] : om[1], f == 0 ? hm[2] : om[2],
                             f == 0 ? hm[3] : om[3]};
      int wtot;
      const int excl = warp_excl_scan(c, wtot);
      int wbase = 0;
      if ((threadIdx.x & 31) == 0 && wtot > 0) wbase = atomicAdd(out.counters, wtot);
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (!live) continue;
      int64_t pos = (int64_t)wbase + excl;
      const bool fits = pos + c <= out.capacity;
      out.ray_offset[ray] = (int)pos;
      out.ray_count[ray] = fits ? c : 0;
      if (!fits) {
        if (c > 0) atomicExch(out.counters + 1, 1);
        continue;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t bitsw = m[w];
        while (bitsw) {
          const int b = __ffs(bitsw) - 1;
          bitsw &= bitsw - 1;
          out.records[pos++] = ((uint32_t)ray << 8) | (uint32_t)(w * 32 + b);
        }
      }
    }
  }
  pdl_trigger();
}

// p_c = Tinv [p, 1] (Tinv: (3,4) row-major)
__device__ __forceinline__ d3 lbs_apply(const double* __restrict__ T, d3 p) {
  return d3{T[0] * p.x + T[1] * p.y + T[2] * p.z + T[3], T[4] * p.x + T[5] * p.y + T[6] * p.z + T[7],
            T[8] * p.x + T[9] * p.y + T[10] * p.z + T[11]};
}

// backward-LBS fallback of a sample outside the ED support: its nearest posed
// skin vertex (exact 1-NN on the vertex buckets) within lbs_max_dist -> that
// vertex's inverse blended transform. No vertex can be that close when the
// sample is that far from the vertex grid's box (which holds every vertex).
__device__ __forceinline__ bool lbs_fallback(const BucketParams& sL, const int* __restrict__ lcs,
                                             const double4* __restrict__ ls, const cf_human_warp& W, d3 p, d3& pt) {
  const double q[3] = {p.x, p.y, p.z};
  double d2b = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double e = fmax(fmax(sL.origin[a] - q[a], q[a] - (sL.origin[a] + sL.g[a] * sL.h)), 0.0);
    d2b += e * e;
  }
  TopK<1> top;
  top.init(1);
  if (d2b <= W.lbs_max_d2 * (1.0 + 1e-9)) bucket_knn<1>(sL, lcs, ls, p, top, W.lbs_max_d2);
  if (!(top.d[0] <= W.lbs_max_d2)) return false;
  pt = lbs_apply(W.vert_Tinv + 12 * (int64_t)top.i[0], p);
  return true;
}

// canonical unit-cube coordinates + flag (1 = ED, 2 = LBS, 0 = empty)
__device__ __forceinline__ float4 canon_out(const cf_human_warp& W, d3 pt, float flag) {
  if (!(flag > 0.0f)) return make_float4(0.f, 0.f, 0.f, 0.f);
  return make_float4(__double2float_rn(x_mul(x_sub(pt.x, W.canon_min[0]), W.inv_side)),
                     __double2float_rn(x_mul(x_sub(pt.y, W.canon_min[1]), W.inv_side)),
                     __double2float_rn(x_mul(x_sub(pt.z, W.canon_min[2]), W.inv_side)), flag);
}

// human samples: live point -> ED backward warp (exact k-NN + DQB^-1), falling back
// to backward LBS outside the ED support; -> canonical unit cube.
// kBlock (graphs of <= 1024 nodes): the k-NN scans the frame's anchor block
// (cf_deform_nodes_block: float64 + fp32 copies, bbox; 48 B per node), copied into
// shared memory once per CTA (one barrier; reading it through L1 instead measured
// 72 -> 82 us), with the warp-cooperative culling; else the coarse buckets. Warps
// pull 32-sample chunks from a ticket
// (count[2]; per-chunk cost varies with the LBS fallback and the candidate-set
// size), fetching the next ticket while the current chunk runs.
template <int K, bool kBlock, bool kGrid = false>  // kGrid: the candidate-grid path only (the render)
__global__ void __launch_bounds__(128, CF_CANON_MINB) human_canon_kernel(cf_march_desc M, const double* __restrict__ dirs,
                                                          const uint32_t* __restrict__ records,
                                                          int* count, int64_t capacity,
                                                          cf_human_warp W, const BucketParams* __restrict__ EPp,
                                                          const int* __restrict__ ecs, const double4* __restrict__ es,
                                                          const BucketParams* __restrict__ LPp,
                                                          const int* __restrict__ lcs, const double4* __restrict__ ls,
                                                          float4* __restrict__ xu) {
  extern __shared__ __align__(16) uint8_t s_blk[];  // kBlock: the anchor block (48 n + 48 B), node dqs (64 n B)
  pdl_wait();
  if (kBlock) {  // one coalesced copy of the prebuilt block and of the node dqs, one barrier
    const int words = (48 * W.n_nodes + 48) / 16;
    const uint4* src = static_cast<const uint4*>(W.anchor_block);
    for (int i = threadIdx.x; i < words; i += blockDim.x) reinterpret_cast<uint4*>(s_blk)[i] = src[i];
    const uint4* dsrc = reinterpret_cast<const uint4*>(W.dqs);
    uint4* ddst = reinterpret_cast<uint4*>(s_blk + 48 * (size_t)W.n_nodes + 48);
    for (int i = threadIdx.x; i < 4 * W.n_nodes; i += blockDim.x) ddst[i] = dsrc[i];
    __syncthreads();
  }
  // kBlock: the blend reads the node dqs from shared memory (its k loads of 64 bytes
  // each, right after the ranking, were a second dependent global round trip)
  const double* s_dqs = kBlock ? reinterpret_cast<const double*>(s_blk + 48 * (size_t)W.n_nodes + 48) : W.dqs;
  const double4* a64 = reinterpret_cast<const double4*>(s_blk);
  const float4* a32 = reinterpret_cast<const float4*>(s_blk + 32 * (size_t)W.n_nodes);
  const double* box = reinterpret_cast<const double*>(s_blk + 48 * (size_t)W.n_nodes);
  const CandGridHdr* cgrid = static_cast<const CandGridHdr*>(W.cand_grid);
  const uint16_t* clists = cgrid ? reinterpret_cast<const uint16_t*>(static_cast<const uint8_t*>(W.cand_grid) + 64)
                                 : nullptr;
  // A sample farther than R from the anchors' bbox has every Gaussian weight
  // below the validity floor: d^2 / r^2 > -ln(1e-6) (1 + 1e-5) => w < 1e-6. Such
  // samples skip the k-NN (ED invalid, as the exact evaluation would find) and
  // stay out of the warp's culling box — training's uniform samples along the
  // whole ray [0.3 m, 5 m] are mostly of this kind.
  const double rsup2 = 13.815510557964274 * W.r2 * (1.0 + 1e-5);
  const d3 o = M.frame ? d3{M.frame[0], M.frame[1], M.frame[2]} : d3{M.origin[0], M.origin[1], M.origin[2]};
  const int64_t n = min((int64_t)count[0], capacity);
  const int lane = threadIdx.x & 31;
  int* ticket = count + 2;
  int64_t base = 0;
  if (lane == 0) base = atomicAdd(ticket, 32);
  base = __shfl_sync(0xffffffffu, base, 0);
  while (base < n) {  // warp-uniform: the culled scan is warp-cooperative
    int64_t next = 0;
    if (lane == 0) next = atomicAdd(ticket, 32);  // in flight while this chunk runs
    const int64_t s = base + lane;
    const bool live = s < n;
    const uint32_t rec = live ? records[s] : 0u;
    const int64_t ray = rec >> 8;
    const d3 p = live ? sample_p(o, load_d3(dirs + 3 * ray), rec_t(M, s, rec)) : d3{0.0, 0.0, 0.0};
    d3 pt;
    float flag = 0.0f;
    bool near = live;
    if (kBlock && live) {
      const double q[3] = {p.x, p.y, p.z};
      double d2 = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double e = fmax(fmax(box[a] - q[a], q[a] - box[3 + a]), 0.0);
        d2 += e * e;
      }
      near = d2 <= rsup2;
    }
    bool ed_ok;
    if (kGrid || (kBlock && cgrid)) {
      // the cell's candidate list (cf_cand_grid_build): exact float64 ranking of the few
      // nodes that can be among the k nearest of any point of the cell
      ed_ok = false;
      if (live && near) {
        const double q[3] = {p.x, p.y, p.z};
        int64_t cell = 0;
        bool in = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double f = floor(x_mul(x_sub(q[a], cgrid->origin[a]), cgrid->inv_h));
          const int ca = f < 0.0 ? 0 : (f >= (double)cgrid->dims[a] ? cgrid->dims[a] - 1 : (int)f);
          in &= f >= 0.0 && f < (double)cgrid->dims[a];  // (outside: rounding at the grid's edge -> every node)
          cell = cell * cgrid->dims[a] + ca;
        }
        TopK<K> top;
        top.init(W.k);
        // the list 8 entries (16 bytes) per load, the next 8 in flight while these are
        // ranked (one dependent 2-byte load per candidate was the k-NN's latency chain)
        const uint4* L4 = reinterpret_cast<const uint4*>(clists + cell * cand_stride(cgrid->cmax));
        uint4 v = in ? __ldg(L4) : make_uint4(0xFFFFu, 0u, 0u, 0u);
        const int cnt = (int)(v.x & 0xFFFFu);
        if (cnt == 0xFFFF) {  // a crowded cell: every node
          for (int i = 0; i < W.n_nodes; ++i) {
            const double4 a = a64[i];
            top.insert(sqdist(p, d3{a.x, a.y, a.z}), i);
          }
        } else {
          for (int e0 = 0; e0 <= cnt; e0 += 8) {  // list position e: entry e - 1 (0 = count)
            const uint4 nxt = e0 + 8 <= cnt ? __ldg(L4 + (e0 >> 3) + 1) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 1
            for (int u = (e0 == 0 ? 1 : 0); u < 8 && e0 + u <= cnt; ++u) {
              const uint32_t w = u < 2 ? v.x : u < 4 ? v.y : u < 6 ? v.z : v.w;
              const int i = (int)((u & 1) ? w >> 16 : w & 0xFFFFu);
              const double4 a = a64[i];
              top.insert(sqdist(p, d3{a.x, a.y, a.z}), i);
            }
            v = nxt;
          }
        }
        ed_ok = blend_apply<K>(top, s_dqs, W.k, W.r2, true, p, pt);
      }
    } else if constexpr (!kGrid) {
      ed_ok = kBlock ? ed_warp_point_cull<K>(a64, a32, W.n_nodes, s_dqs, W.k, W.r2, true, p, near, pt)
                     : (live && ed_warp_point<K>(*EPp, ecs, es, W.dqs, W.k, W.r2, true, p, pt));
    }
    if (live) {
      if (ed_ok) flag = 1.0f;
      else if (LPp && lbs_fallback(*LPp, lcs, ls, W, p, pt)) flag = 2.0f;
      xu[s] = canon_out(W, pt, flag);
    }
    base = __shfl_sync(0xffffffffu, next, 0);
  }
  // the last warp out re-arms the ticket for the next launch on these counters
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ticket + 1, 1) == (int)(gridDim.x * (blockDim.x >> 5)) - 1) {
      ticket[0] = 0;
      ticket[1] = 0;
    }
  }
  pdl_trigger();
}

// The backward-LBS fallback as its own pass, for the render: the canonicalisation runs
// without it (samples the ED warp does not reach get flag 0) as soon as the march and
// the ED chain are done, and this pass completes those samples after the per-frame LBS
// setup (posed vertices, inverse transforms and their box, on the side stream) — that
// chain no longer sits between the march and the canonicalisation, and the render
// needs no vertex buckets. Per warp: the samples of flag 0 within lbs_max_dist of the
// posed vertices' box (lbs_fallback's rejection) are taken one at a time, the 32 lanes
// scan the vertices and reduce (d^2, index) — the exact 1-NN with ties by index that
// bucket_knn<1> finds — and the owner lane applies that vertex's inverse transform
// (lbs_apply, as lbs_fallback): bit-identical to the fused call.
__global__ void __launch_bounds__(128) human_lbs_fallback_kernel(cf_march_desc M, const double* __restrict__ dirs,
                                                                 const uint32_t* __restrict__ records,
                                                                 const int* __restrict__ count, int64_t capacity,
                                                                 cf_human_warp W, const double* __restrict__ posed,
                                                                 int64_t V, const unsigned long long* __restrict__ box,
                                                                 float4* __restrict__ xu) {
  pdl_wait();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const d3 o = M.frame ? d3{M.frame[0], M.frame[1], M.frame[2]} : d3{M.origin[0], M.origin[1], M.origin[2]};
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = dkey_inv(box[a]);
    hi[a] = dkey_inv(box[3 + a]);
  }
  const int64_t n = min((int64_t)count[0], capacity);
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < n;
       base += warps * 32) {
    const int64_t s = base + lane;
    bool need = s < n && xu[s].w == 0.0f;
    d3 p{0.0, 0.0, 0.0};
    if (need) {
      const uint32_t rec = records[s];
      p = sample_p(o, load_d3(dirs + 3 * (int64_t)(rec >> 8)), rec_t(M, s, rec));
      const double q[3] = {p.x, p.y, p.z};
      double d2b = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double e = fmax(fmax(lo[a] - q[a], q[a] - hi[a]), 0.0);
        d2b += e * e;
      }
      need = d2b <= W.lbs_max_d2 * (1.0 + 1e-9);
    }
    unsigned todo = __ballot_sync(FULL, need);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const d3 pj{__shfl_sync(FULL, p.x, j), __shfl_sync(FULL, p.y, j), __shfl_sync(FULL, p.z, j)};
      double bd = __longlong_as_double(0x7ff0000000000000LL);
      int bi = 0x7fffffff;
      for (int64_t v = lane; v < V; v += 32) {
        const double d = sqdist(pj, load_d3(posed + 3 * v));
        if (key_less(d, (int)v, bd, bi)) {
          bd = d;
          bi = (int)v;
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const double d2 = __shfl_xor_sync(FULL, bd, off);
        const int i2 = __shfl_xor_sync(FULL, bi, off);
        if (key_less(d2, i2, bd, bi)) {
          bd = d2;
          bi = i2;
        }
      }
      if (lane == j && bd <= W.lbs_max_d2) xu[s] = canon_out(W, lbs_apply(W.vert_Tinv + 12 * (int64_t)bi, p), 2.0f);
    }
  }
  pdl_trigger();
}

// ------------------------------------------------------------ valid-sample compaction
// The training step's empty samples (flag 0: human samples no warp reaches, ~26 % at
// configs[2], object samples outside the object's box — mostly the uniform samples
// along the rays) have sigma = 0 and no gradient: the field forward / backward run on
// the compacted valid ones (records, xu) and only the composite sees every sample. Per warp: ballot + one atomic; vidx[j] = the full index of
// compacted sample j, inv[s] = its compacted index or -1.
__global__ void compact_valid_kernel(const int* __restrict__ count, int64_t capacity,
                                     const uint32_t* __restrict__ records, const float4* __restrict__ xu,
                                     uint32_t* __restrict__ rec_c, float4* __restrict__ xu_c, int* __restrict__ vidx,
                                     int* __restrict__ inv, int* __restrict__ count_c) {
  const int64_t n = min((int64_t)*count, capacity);
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = base + threadIdx.x;
    const bool live = s < n;
    const float4 x = live ? xu[s] : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool ok = live && x.w > 0.0f;
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    int wbase = 0;
    if (lane == 0 && m) wbase = atomicAdd(count_c, __popc(m));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (!live) continue;
    const int pos = wbase + __popc(m & ((1u << lane) - 1u));
    if (ok) {
      rec_c[pos] = records[s];
      xu_c[pos] = x;
      vidx[pos] = (int)s;
    }
    inv[s] = ok ? pos : -1;
  }
}

// out[s] = out_c[inv[s]] for the valid samples, zero for the others
__global__ void scatter_rows_kernel(const int* __restrict__ count, int64_t capacity, const int* __restrict__ inv,
                                    const float4* __restrict__ src, float4* __restrict__ dst) {
  const int64_t n = min((int64_t)*count, capacity);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const int j = inv[s];
    dst[s] = j >= 0 ? src[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// dst[j] = src[vidx[j]] over the compacted samples
__global__ void gather_rows_kernel(const int* __restrict__ count_c, int64_t capacity, const int* __restrict__ vidx,
                                   const float4* __restrict__ src, float4* __restrict__ dst) {
  const int64_t n = min((int64_t)*count_c, capacity);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    dst[j] = src[vidx[j]];
}

// rigid object samples: live point -> object-local frame -> unit cube
__global__ void object_canon_kernel(cf_march_desc M, const double* __restrict__ dirs,
                                    const uint32_t* __restrict__ records, const int* __restrict__ count,
                                    int64_t capacity, const double* obj_min, double inv_side,
                                    float4* __restrict__ xu) {
  pdl_wait();
  __shared__ double s_fr[15];
  load_frame(M, s_fr);
  const int64_t n = min((int64_t)*count, capacity);
  const d3 o{s_fr[0], s_fr[1], s_fr[2]};
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t rec = records[s];
    const int64_t ray = rec >> 8;
    const d3 p = to_object(s_fr + 3, s_fr + 12, sample_p(o, load_d3(dirs + 3 * ray), rec_t(M, s, rec)));
    const float4 u = make_float4(__double2float_rn(x_mul(x_sub(p.x, M.obj_min[0]), M.obj_inv_side)),
                                 __double2float_rn(x_mul(x_sub(p.y, M.obj_min[1]), M.obj_inv_side)),
                                 __double2float_rn(x_mul(x_sub(p.z, M.obj_min[2]), M.obj_inv_side)), 1.0f);
    // the object field is defined on its box (the render's object grid): a sample
    // outside [0, 1]^3 (training's uniform samples) is empty
    const bool in = u.x >= 0.f && u.x <= 1.f && u.y >= 0.f && u.y <= 1.f && u.z >= 0.f && u.z <= 1.f;
    xu[s] = in ? u : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  pdl_trigger();
}

// depth t and step delta of the j-th sample of a ray segment: uniform march
// (t_i, dt), or explicit training depths (delta = t_{j+1} - t_j, dt for the last)
__device__ __forceinline__ void seg_t_delta(const cf_march_desc& M, const cf_march_out& F, int off, int cnt, int j,
                                            float& t, float& delta) {
  if (M.sample_t) {
    const double tj = M.sample_t[off + j];
    t = (float)tj;
    delta = (j + 1 < cnt) ? (float)(M.sample_t[off + j + 1] - tj) : (float)M.dt;
  } else {
    t = (float)sample_t(M, (int)(F.records[off + j] & 255u));
    delta = (float)M.dt;
  }
}

// One ray's front-to-back accumulation, 4 samples per step: their field values and
// depths are loaded together before the sequential accumulation (the loop's loads were
// one dependent round trip per sample); same operations in the same order as sample by
// sample, stopping after the sample that takes T below t_term.
__device__ __forceinline__ void ray_accumulate(const cf_march_desc& M, const cf_march_out& F,
                                               const float4* __restrict__ field, float t_term, int off, int cnt,
                                               float& T, float& r, float& g, float& b, float& dep) {
  for (int j0 = 0; j0 < cnt; j0 += 4) {
    float4 f[4];
    float t[4], delta[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j0 + u < cnt) {
        f[u] = field[off + j0 + u];
        seg_t_delta(M, F, off, cnt, j0 + u, t[u], delta[u]);
      }
    }
    bool stop = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (stop || j0 + u >= cnt) break;
      const float alpha = 1.0f - expf(-f[u].x * delta[u]);
      const float w = T * alpha;
      r += w * f[u].y;
      g += w * f[u].z;
      b += w * f[u].w;
      dep += w * t[u];
      T *= 1.0f - alpha;
      stop = T < t_term;
    }
    if (stop) break;
  }
}

// front-to-back alpha compositing: alpha_i = 1 - exp(-sigma_i * dt),
// T_i = prod_{j<i} (1 - alpha_j); stops once T < t_term
__global__ void composite_kernel(cf_march_desc M, cf_march_out F, const float4* __restrict__ field, float t_term,
                                 float* __restrict__ rgb, float* __restrict__ depth, float* __restrict__ opacity) {
  pdl_wait();
  for (int64_t ray = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ray < M.n_rays;
       ray += (int64_t)gridDim.x * blockDim.x) {
    const int off = F.ray_offset[ray], cnt = F.ray_count[ray];
    float T = 1.0f, r = 0.f, g = 0.f, b = 0.f, dep = 0.f, op = 0.f;
    ray_accumulate(M, F, field, t_term, off, cnt, T, r, g, b, dep);
    op = 1.0f - T;  // = sum T_i alpha_i (telescoping), without its rounding drift
    rgb[3 * ray] = r;
    rgb[3 * ray + 1] = g;
    rgb[3 * ray + 2] = b;
    depth[ray] = dep / fmaxf(op, 1e-6f);
    opacity[ray] = op;
  }
  pdl_trigger();
}

// human-field composite of a ray fused with the layer choice:
// the object layer was composited before (side stream); writes the human layer's
// rgb/depth/opacity too (same values as composite_kernel)
__global__ void composite_final_kernel(cf_march_desc M, cf_march_out F, const float4* __restrict__ field,
                                       float t_term, float* __restrict__ rgb, float* __restrict__ depth,
                                       float* __restrict__ opacity, const float* __restrict__ orgb,
                                       const float* __restrict__ od, const float* __restrict__ oo, float bg0,
                                       float bg1, float bg2, float* __restrict__ out, uint8_t* __restrict__ layer) {
  pdl_wait();
  for (int64_t ray = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ray < M.n_rays;
       ray += (int64_t)gridDim.x * blockDim.x) {
    const int off = F.ray_offset[ray], cnt = F.ray_count[ray];
    float T = 1.0f, r = 0.f, g = 0.f, b = 0.f, dep = 0.f, op = 0.f;
    ray_accumulate(M, F, field, t_term, off, cnt, T, r, g, b, dep);
    op = 1.0f - T;  // = sum T_i alpha_i (telescoping), without its rounding drift
    const float hd = dep / fmaxf(op, 1e-6f);
    rgb[3 * ray] = r;
    rgb[3 * ray + 1] = g;
    rgb[3 * ray + 2] = b;
    depth[ray] = hd;
    opacity[ray] = op;
    const bool h = op > 0.5f, o = orgb && oo[ray] > 0.5f;
    int L = 0;
    if (h && o) L = hd <= od[ray] ? 1 : 2;
    else if (h) L = 1;
    else if (o) L = 2;
    out[3 * ray] = L == 1 ? r : (L == 2 ? orgb[3 * ray] : bg0);
    out[3 * ray + 1] = L == 1 ? g : (L == 2 ? orgb[3 * ray + 1] : bg1);
    out[3 * ray + 2] = L == 1 ? b : (L == 2 ? orgb[3 * ray + 2] : bg2);
    if (layer) layer[ray] = (uint8_t)L;
  }
  pdl_trigger();
}

// Loss (lambda_depth config.py:55) and compositing backward.
//   L = 1/Nm sum_masked |rgb - gt|^2 + lambda / Nd sum_masked,valid-depth |depth - gt_depth|
// d rgb = sum w c, D = sum w t, O = sum w, depth = D / max(O, 1e-6):
//   dL/dc_j     = w_j dL/drgb
//   dL/dsigma_j = delta_j [ sum_v g_v (T_{j+1} v_j - (S_v - P_v,j)) ]   v in {r,g,b, t, 1}
// (S_v: ray total, P_v,j: prefix through sample j). Samples after early
// termination get zero gradient, exactly mirroring the forward.
__global__ void composite_bwd_kernel(cf_march_desc M, cf_march_out F, const float4* __restrict__ field,
                                     float t_term, const float* __restrict__ gt_rgb,
                                     const float* __restrict__ gt_depth, const uint8_t* __restrict__ mask,
                                     float lambda, const float* __restrict__ norm,
                                     float4* __restrict__ grad, float* __restrict__ loss) {
  // normalisers from the device (cf_train_norms: the frame's masked / depth-valid ray
  // counts, summed over ranks) and the field's power-of-two loss scale
  const float inv_nm = norm[0], inv_nd = norm[1], gscale = norm[2], wl = norm[3];
  float lc = 0.f, ld = 0.f;
  for (int64_t ray = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ray < M.n_rays;
       ray += (int64_t)gridDim.x * blockDim.x) {
    const int off = F.ray_offset[ray], cnt = F.ray_count[ray];
    // forward again: totals and the number of samples used
    float T = 1.f, S[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    int used = 0;
    for (int j = 0; j < cnt; ++j) {
      const float4 f = field[off + j];
      float t, delta;
      seg_t_delta(M, F, off, cnt, j, t, delta);
      const float a = 1.0f - expf(-f.x * delta), w = T * a;
      S[0] += w * f.y;
      S[1] += w * f.z;
      S[2] += w * f.w;
      S[3] += w * t;
      T *= 1.0f - a;
      used = j + 1;
      if (T < t_term) break;
    }
    S[4] = 1.0f - T;  // opacity as the forward computes it
    float gv[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    if (mask[ray]) {
      for (int c = 0; c < 3; ++c) {
        const float e = S[c] - gt_rgb[3 * ray + c];
        lc += e * e * inv_nm * wl;
        gv[c] = 2.0f * e * inv_nm * gscale;
      }
      const float gd = gt_depth[ray];
      if (gd > 0.f) {
        const float O = fmaxf(S[4], 1e-6f), depth = S[3] / O, e = depth - gd;
        ld += fabsf(e) * inv_nd * wl;
        const float gdep = lambda * inv_nd * gscale * (e > 0.f ? 1.f : (e < 0.f ? -1.f : 0.f));
        gv[3] = gdep / O;
        gv[4] = S[4] > 1e-6f ? -gdep * S[3] / (S[4] * S[4]) : 0.f;
      }
    }
    T = 1.f;
    float P[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < cnt; ++j) {
      if (j >= used) {
        grad[off + j] = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      const float4 f = field[off + j];
      float t, delta;
      seg_t_delta(M, F, off, cnt, j, t, delta);
      const float a = 1.0f - expf(-f.x * delta), w = T * a;
      const float v[5] = {f.y, f.z, f.w, t, 1.0f};
      const float Tn = T * (1.0f - a);
      float ds = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        P[q] += w * v[q];
        ds += gv[q] * (Tn * v[q] - (S[q] - P[q]));
      }
      P[4] = 1.0f - Tn;  // opacity prefix, matching S[4] = 1 - T_end
      ds += gv[4] * (Tn - (S[4] - P[4]));
      grad[off + j] = make_float4(delta * ds, w * gv[0], w * gv[1], w * gv[2]);
      T = Tn;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lc += __shfl_xor_sync(0xffffffffu, lc, o);
    ld += __shfl_xor_sync(0xffffffffu, ld, o);
  }
  if ((threadIdx.x & 31) == 0 && loss) {
    atomicAdd(loss, lc);
    atomicAdd(loss + 1, ld);
  }
}

// counter-based uniform in [0,1): splitmix64 of (seed, ray, j) -> 53-bit mantissa
__device__ __forceinline__ double u01(uint64_t seed, uint64_t ray, uint64_t j) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (ray * 64ull + j + 1ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}

// Training rays of one key frame (the ray-batch sampler on the
// device): n pixels drawn uniformly with replacement from the frame's foreground
// pixel list (u01 of (seed, i)); their targets are gathered from the frame's
// HBM-resident images and their exact camera rays generated (pixel_dir).
__global__ void keyframe_rays_kernel(cf_camera cam, const int* __restrict__ fg, int64_t n_fg, int64_t n,
                                     uint64_t seed, const uint64_t* __restrict__ seed_off, const float* __restrict__ rgb, const float* __restrict__ depth,
                                     const uint8_t* __restrict__ mask_h, const uint8_t* __restrict__ mask_o,
                                     int* __restrict__ pix_out, double* __restrict__ dirs, float* __restrict__ rgb_o,
                                     float* __restrict__ depth_o, uint8_t* __restrict__ mh_o,
                                     uint8_t* __restrict__ mo_o) {
  __shared__ double s_cam[13];
  load_camera(cam, s_cam);
  const ExactDiv by_fx(s_cam[9]), by_fy(s_cam[10]);
  if (seed_off) seed += *seed_off;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = min((int64_t)(u01(seed, (uint64_t)i, 0) * (double)n_fg), n_fg - 1);
    const int px = fg[k];
    if (pix_out) pix_out[i] = px;
    store_d3(dirs + 3 * i, pixel_dir(s_cam, by_fx, by_fy, cam.width, px));
    rgb_o[3 * i] = rgb[3 * (int64_t)px];
    rgb_o[3 * i + 1] = rgb[3 * (int64_t)px + 1];
    rgb_o[3 * i + 2] = rgb[3 * (int64_t)px + 2];
    depth_o[i] = depth[px];
    mh_o[i] = mask_h[px];
    mo_o[i] = mask_o[px];
  }
}

// Depth-guided training samples: a masked ray with valid depth d
// gets n_guided stratified samples in [d - 6 s, d + 6 s] (clamped to
// [t_near, t_far]) merged with n_uniform stratified samples over [t_near, t_far];
// without depth, n_empty stratified samples. Sorted per ray; t in float64:
//   t = lo + ((j + u) / n) * (hi - lo)      (un-contracted, u = u01(seed, ray, slot))
// Stratum j of the guided set uses slot j, of the uniform set slot 32 + j.
__global__ void __launch_bounds__(128) train_sample_kernel(cf_march_desc M, const float* __restrict__ gt_depth,
                                                           const uint8_t* __restrict__ mask, int n_guided,
                                                           int n_uniform, int n_empty, double sigma_d,
                                                           uint64_t seed, const uint64_t* __restrict__ seed_off,
                                                           int64_t ray0, cf_march_out F, double* __restrict__ t_out) {
  if (seed_off) seed += *seed_off;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < M.n_rays; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ray = base + threadIdx.x;
    const bool live = ray < M.n_rays && mask[ray] != 0;
    const float d = live ? gt_depth[ray] : 0.f;
    const bool guided = live && d > 0.f;
    const int c = !live ? 0 : (guided ? n_guided + n_uniform : n_empty);
    int wtot;
    const int excl = warp_excl_scan(c, wtot);
    int wbase = 0;
    if ((threadIdx.x & 31) == 0 && wtot > 0) wbase = atomicAdd(F.counters, wtot);
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (ray >= M.n_rays) continue;
    const int64_t pos = (int64_t)wbase + excl;
    const bool fits = pos + c <= F.capacity;
    F.ray_offset[ray] = (int)pos;
    F.ray_count[ray] = fits ? c : 0;
    if (!fits) {
      if (c > 0) atomicExch(F.counters + 1, 1);
      continue;
    }
    if (c == 0) continue;
    auto strat = [&](double lo, double hi, int n, int j, int slot) {
      return x_add(lo, x_mul(x_div((double)j + u01(seed, (uint64_t)(ray0 + ray), slot), (double)n), x_sub(hi, lo)));
    };
    if (!guided) {
      for (int j = 0; j < n_empty; ++j) {
        t_out[pos + j] = strat(M.t_near, M.t_far, n_empty, j, j);
        F.records[pos + j] = ((uint32_t)ray << 8) | (uint32_t)j;
      }
      continue;
    }
    const double lo = fmax(M.t_near, x_sub((double)d, x_mul(6.0, sigma_d)));
    const double hi = fmin(M.t_far, x_add((double)d, x_mul(6.0, sigma_d)));
    // merge two sorted stratified sets
    int a = 0, b = 0;
    double ta = strat(lo, hi, n_guided, 0, 0), tb = strat(M.t_near, M.t_far, n_uniform, 0, 32);
    for (int j = 0; j < c; ++j) {
      const bool takeA = b >= n_uniform || (a < n_guided && ta <= tb);
      const double t = takeA ? ta : tb;
      if (takeA) {
        ++a;
        if (a < n_guided) ta = strat(lo, hi, n_guided, a, a);
      } else {
        ++b;
        if (b < n_uniform) tb = strat(M.t_near, M.t_far, n_uniform, b, 32 + b);
      }
      t_out[pos + j] = t;
      F.records[pos + j] = ((uint32_t)ray << 8) | (uint32_t)j;
    }
  }
}

// depth-occlusion composite: nearer layer with opacity > 0.5
__global__ void layers_kernel(int64_t n, const float* __restrict__ hr, const float* __restrict__ hd,
                              const float* __restrict__ ho, const float* __restrict__ orgb,
                              const float* __restrict__ od, const float* __restrict__ oo, float bg0, float bg1,
                              float bg2, float* __restrict__ out, uint8_t* __restrict__ layer) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool h = hr && ho[i] > 0.5f, o = orgb && oo[i] > 0.5f;
    int L = 0;
    if (h && o) L = hd[i] <= od[i] ? 1 : 2;
    else if (h) L = 1;
    else if (o) L = 2;
    const float* src = L == 1 ? hr + 3 * i : (L == 2 ? orgb + 3 * i : nullptr);
    out[3 * i] = src ? src[0] : bg0;
    out[3 * i + 1] = src ? src[1] : bg1;
    out[3 * i + 2] = src ? src[2] : bg2;
    if (layer) layer[i] = (uint8_t)L;
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(256) store_to_host_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                            int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// several small copies (device or UVA-mapped pinned host sources) in ONE launch:
// one CTA per entry, 16-byte moves where both ends allow it
__global__ void __launch_bounds__(256) copy_batch_kernel(cf_copy_list L) {
  const int e = blockIdx.x;
  if (e >= L.n) return;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(L.src[e]);
  uint8_t* dst = reinterpret_cast<uint8_t*>(L.dst[e]);
  const int64_t bytes = L.bytes[e];
  if ((((uintptr_t)src | (uintptr_t)dst | (uintptr_t)bytes) & 15) == 0) {
    for (int64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  } else {
    for (int64_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  }
}

}  // namespace

extern "C" {

int cf_camera_rays(const cf_camera* cam, double* dirs, void* stream) {
  if (!cam || cam->width < 1 || cam->height < 1 || !dirs || (int64_t)cam->width * cam->height > INT32_MAX)
    return cf::fail(CF_E_BAD_ARG, "cf_camera_rays: bad args");
  const int64_t n = (int64_t)cam->width * cam->height;
  cf::launch_pdl(rays_kernel, cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream), *cam, dirs);
  return cf::check_launch("cf_camera_rays");
}

int cf_occ_from_points(const cf_buckets_t* pts, const cf_occ_grid* g, double radius, uint32_t* bits, void* stream) {
  if (!pts || !g || g->res < 1 || pts->grid_res == 0) return cf::fail(CF_E_BAD_ARG, "cf_occ_from_points: bad args");
  const int64_t total = (int64_t)g->res * g->res * g->res;
  occ_points_kernel<<<cf::grid_for(total, 128, 8), 128, 0, cf::as_stream(stream)>>>(*g, pts->params, pts->cell_start,
                                                                                   pts->sorted, radius * radius, bits);
  return cf::check_launch("cf_occ_from_points");
}

int cf_occ_box_shell(const cf_occ_grid* g, const double* half_extents, double shell, uint32_t* bits, void* stream) {
  if (!g || g->res < 1 || !half_extents) return cf::fail(CF_E_BAD_ARG, "cf_occ_box_shell: bad args");
  const int64_t total = (int64_t)g->res * g->res * g->res;
  occ_box_kernel<<<cf::grid_for(total, 256, 4), 256, 0, cf::as_stream(stream)>>>(
      *g, half_extents[0], half_extents[1], half_extents[2], shell, bits);
  return cf::check_launch("cf_occ_box_shell");
}

int cf_occ_splat(const uint32_t* canon_bits, const cf_occ_grid* cg, const cf_buckets_t* node_buckets,
                 const double* dqs, int k, double radius, const cf_occ_grid* lg, uint32_t* live_bits, void* stream) {
  if (!canon_bits || !cg || !lg || !node_buckets || node_buckets->grid_res == 0 || k < 1 || k > 8)
    return cf::fail(CF_E_BAD_ARG, "cf_occ_splat: bad args");
  cudaStream_t st = cf::as_stream(stream);
  const int64_t lwords = ((int64_t)lg->res * lg->res * lg->res + 31) / 32;
  cf::fill_list(st, {{live_bits, 0u, lwords}});
  const int64_t total = (int64_t)cg->res * cg->res * cg->res;
  const unsigned grid = cf::grid_for(total, 128, 8);
  const double r2 = radius * radius;
  dispatch_k(k, [&]<int K>() {
    occ_splat_kernel<K><<<grid, 128, 0, st>>>(canon_bits, *cg, node_buckets->params, node_buckets->cell_start,
                                              node_buckets->sorted, dqs, k, r2, *lg, live_bits);
    return 0;
  });
  return cf::check_launch("cf_occ_splat");
}

int cf_occ_cache(const uint32_t* canon_bits, const cf_occ_grid* cg, const cf_buckets_t* node_buckets, int k,
                 double radius, int64_t capacity, int* cells, int* nbr, double* w, int* count, void* stream) {
  if (!canon_bits || !cg || !node_buckets || node_buckets->grid_res == 0 || k < 1 || k > 8 || !count)
    return cf::fail(CF_E_BAD_ARG, "cf_occ_cache: bad args");
  cudaStream_t st = cf::as_stream(stream);
  cf::fill_list(st, {{count, 0u, 1}});
  const int64_t total = (int64_t)cg->res * cg->res * cg->res;
  const unsigned grid = cf::grid_for(total, 128, 8);
  dispatch_k(k, [&]<int K>() {
    occ_cache_kernel<K><<<grid, 128, 0, st>>>(canon_bits, *cg, node_buckets->params, node_buckets->cell_start,
                                              node_buckets->sorted, k, radius * radius, capacity, cells, nbr, w,
                                              count);
    return 0;
  });
  return cf::check_launch("cf_occ_cache");
}

int cf_occ_splat_cached(const int* cells, const int* nbr, const double* w, const int* count, int64_t capacity, int k,
                        const double* dqs, const cf_occ_grid* cg, const cf_occ_grid* lg, uint32_t* scratch_bits,
                        uint32_t* live_bits, int* live_bbox, void* stream) {
  if (!cells || !nbr || !w || !count || !dqs || !cg || !lg || !scratch_bits || !live_bits || k < 1 || k > 8)
    return cf::fail(CF_E_BAD_ARG, "cf_occ_splat_cached: bad args");
  cudaStream_t st = cf::as_stream(stream);
  const int64_t P = lg->res + 2;
  // lo = 0x7f7f7f7f, hi = 0x80808080 (negative)
  cf::fill_list(st, {{scratch_bits, 0u, (P * P * P + 31) / 32 + 3}, {live_bbox, 0x7f7f7f7fu, live_bbox ? 3 : 0},
                     {live_bbox ? live_bbox + 3 : nullptr, 0x80808080u, live_bbox ? 3 : 0}});
  const unsigned grid = cf::grid_for(capacity, 256, 4);
  if (k <= 4)
    cf::launch_pdl(occ_splat_cached_kernel<4>, grid, 256, 0, st, cells, nbr, w, count, capacity, k, dqs, *cg, *lg, scratch_bits,
                                                     live_bbox);
  else
    cf::launch_pdl(occ_splat_cached_kernel<8>, grid, 256, 0, st, cells, nbr, w, count, capacity, k, dqs, *cg, *lg, scratch_bits,
                                                     live_bbox);
  const int64_t words = ((int64_t)lg->res * lg->res * lg->res + 31) / 32;
  cf::launch_pdl(occ_dilate_kernel, cf::grid_for(words, 256, 8), 256, 0, st, scratch_bits, lg->res, live_bits, live_bbox);
  return cf::check_launch("cf_occ_splat_cached");
}

int cf_occ_bbox(const uint32_t* bits, const cf_occ_grid* g, int* bbox, void* stream) {
  if (!bits || !g || !bbox || g->res < 1) return cf::fail(CF_E_BAD_ARG, "cf_occ_bbox: bad args");
  occ_bbox_kernel<<<1, 1024, 0, cf::as_stream(stream)>>>(bits, *g, bbox);
  return cf::check_launch("cf_occ_bbox");
}

int cf_march(const cf_march_desc* M, const double* dirs, const uint32_t* human_bits, const uint32_t* object_bits,
             const cf_march_out* human, const cf_march_out* object, void* stream) {
  if (!M || !dirs || M->n_samples < 1 || M->n_samples > 128 || M->n_rays < 0 || M->n_rays >= (1LL << 24))
    return cf::fail(CF_E_BAD_ARG, "cf_march: bad args (<= 128 samples, < 2^24 rays)");
  cf_march_out H{}, O{};
  if (human && human_bits) H = *human;
  if (object && object_bits) O = *object;
  cudaStream_t st = cf::as_stream(stream);
  cf::fill_list(st, {{H.counters, 0u, H.records ? 4 : 0}, {O.counters, 0u, O.records ? 4 : 0}});
  if (M->n_rays == 0) return CF_OK;
  cf::launch_pdl(march_kernel<false>, cf::grid_for(M->n_rays, 128, 8), 128, 0, st, *M, cf_camera{},
                 const_cast<double*>(dirs), H.records ? human_bits : nullptr, O.records ? object_bits : nullptr, H, O);
  return cf::check_launch("cf_march");
}

int cf_rays_march(const cf_camera* cam, const cf_march_desc* M, double* dirs, const uint32_t* human_bits,
                  const uint32_t* object_bits, const cf_march_out* human, const cf_march_out* object, void* stream) {
  if (!cam || !M || !dirs || M->n_samples < 1 || M->n_samples > 128 || cam->width < 1 || cam->height < 1 ||
      (int64_t)cam->width * cam->height != M->n_rays || M->n_rays >= (1LL << 24))
    return cf::fail(CF_E_BAD_ARG, "cf_rays_march: bad args (n_rays = width*height < 2^24, <= 128 samples)");
  cf_march_out H{}, O{};
  if (human && human_bits) H = *human;
  if (object && object_bits) O = *object;
  cudaStream_t st = cf::as_stream(stream);
  cf::fill_list(st, {{H.counters, 0u, H.records ? 4 : 0}, {O.counters, 0u, O.records ? 4 : 0}});
  cf::launch_pdl(march_kernel<true>, cf::grid_for(M->n_rays, 128, 8), 128, 0, st, *M, *cam, dirs,
                 H.records ? human_bits : nullptr, O.records ? object_bits : nullptr, H, O);
  return cf::check_launch("cf_rays_march");
}

int cf_human_canon(const cf_march_desc* M, const double* dirs, const cf_march_out* F, const cf_human_warp* W,
                   const cf_buckets_t* anchor_buckets, const cf_buckets_t* vert_buckets, float* xu_f, void* stream) {
  float4* xu = reinterpret_cast<float4*>(xu_f);
  const bool smem = W && W->anchor_block && W->n_nodes > 0 && W->n_nodes <= kSmemAnchors;
  if (!M || !F || !W || W->k < 1 || W->k > 8 || (!smem && (!anchor_buckets || anchor_buckets->grid_res == 0)))
    return cf::fail(CF_E_BAD_ARG, "cf_human_canon: bad args");
  if (W->n_nodes > 0 && W->n_nodes <= kSmemAnchors && !W->anchor_block)
    return cf::fail(CF_E_BAD_ARG, "cf_human_canon: graphs of <= 1024 nodes need the anchor block (cf_deform_nodes_block)");
  const bool lbs = vert_buckets && W->vert_Tinv;
  cudaStream_t st = cf::as_stream(stream);
  const size_t dsm = smem ? (size_t)(48 * W->n_nodes + 48 + 64 * W->n_nodes) : 0;  // anchor block + node dqs
  // persistent: exactly the resident CTAs (the ticket balances the work)
#define CF_HC(KK, SM, GR)                                                                                         \
  int per_sm = 0;                                                                                                \
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, human_canon_kernel<KK, SM, GR>, 128, dsm);              \
  const unsigned grid = cf::grid_for(F->capacity, 128, per_sm > 0 ? per_sm : 1);                                 \
  cf::launch_pdl(human_canon_kernel<KK, SM, GR>, grid, 128, dsm, st, \
      *M, dirs, F->records, F->counters, F->capacity, *W, anchor_buckets ? anchor_buckets->params : nullptr,    \
      anchor_buckets ? anchor_buckets->cell_start : nullptr, anchor_buckets ? anchor_buckets->sorted : nullptr, \
      lbs ? vert_buckets->params : nullptr, lbs ? vert_buckets->cell_start : nullptr,                            \
      lbs ? vert_buckets->sorted : nullptr, xu)
  dispatch_k(W->k, [&]<int K>() {
    if (smem && W->cand_grid) {
      CF_HC(K, true, true);
    } else if (smem) {
      CF_HC(K, true, false);
    } else {
      CF_HC(K, false, false);
    }
    return 0;
  });
#undef CF_HC
  return cf::check_launch("cf_human_canon");
}

int cf_human_lbs_fallback(const cf_march_desc* M, const double* dirs, const cf_march_out* F, const cf_human_warp* W,
                          const double* verts_posed, int64_t n_verts, const uint64_t* posed_box, float* xu_f,
                          void* stream) {
  if (!M || !F || !W || !verts_posed || n_verts < 1 || n_verts >= 0x7fffffff || !posed_box || !W->vert_Tinv || !xu_f)
    return cf::fail(CF_E_BAD_ARG, "cf_human_lbs_fallback: bad args");
  cf::launch_pdl(human_lbs_fallback_kernel, cf::grid_for(F->capacity, 128 * 32, 8), 128, 0, cf::as_stream(stream), *M,
                 dirs, F->records, F->counters, F->capacity, *W, verts_posed, n_verts,
                 reinterpret_cast<const unsigned long long*>(posed_box), reinterpret_cast<float4*>(xu_f));
  return cf::check_launch("cf_human_lbs_fallback");
}

int cf_compact_valid(const cf_march_out* F, const float* xu, const cf_march_out* C, float* xu_c, int* vidx, int* inv,
                     void* stream) {
  if (!F || !C || !xu || !xu_c || !vidx || !inv || !C->records || !C->counters || C->capacity < F->capacity)
    return cf::fail(CF_E_BAD_ARG, "cf_compact_valid: bad args");
  cudaStream_t st = cf::as_stream(stream);
  cf::fill_list(st, {{C->counters, 0u, 4}});
  if (F->capacity == 0) return CF_OK;
  compact_valid_kernel<<<cf::grid_for(F->capacity, 256, 8), 256, 0, st>>>(
      F->counters, F->capacity, F->records, reinterpret_cast<const float4*>(xu), C->records,
      reinterpret_cast<float4*>(xu_c), vidx, inv, C->counters);
  return cf::check_launch("cf_compact_valid");
}

int cf_scatter_rows(const cf_march_out* F, const int* inv, const float* src, float* dst, void* stream) {
  if (!F || !inv || !src || !dst) return cf::fail(CF_E_BAD_ARG, "cf_scatter_rows: bad args");
  if (F->capacity == 0) return CF_OK;
  scatter_rows_kernel<<<cf::grid_for(F->capacity, 256, 8), 256, 0, cf::as_stream(stream)>>>(
      F->counters, F->capacity, inv, reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst));
  return cf::check_launch("cf_scatter_rows");
}

int cf_gather_rows(const cf_march_out* C, const int* vidx, const float* src, float* dst, void* stream) {
  if (!C || !vidx || !src || !dst) return cf::fail(CF_E_BAD_ARG, "cf_gather_rows: bad args");
  if (C->capacity == 0) return CF_OK;
  gather_rows_kernel<<<cf::grid_for(C->capacity, 256, 8), 256, 0, cf::as_stream(stream)>>>(
      C->counters, C->capacity, vidx, reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst));
  return cf::check_launch("cf_gather_rows");
}

int cf_object_canon(const cf_march_desc* M, const double* dirs, const cf_march_out* F, float* xu_f, void* stream) {
  float4* xu = reinterpret_cast<float4*>(xu_f);
  if (!M || !F) return cf::fail(CF_E_BAD_ARG, "cf_object_canon: bad args");
  cf::launch_pdl(object_canon_kernel, cf::grid_for(F->capacity, 256, 4), 256, 0, cf::as_stream(stream), *M, dirs, F->records, F->counters, F->capacity, M->obj_min, M->obj_inv_side, xu);
  return cf::check_launch("cf_object_canon");
}

int cf_composite(const cf_march_desc* M, const cf_march_out* F, const float* field_f, float t_term, float* rgb,
                 float* depth, float* opacity, void* stream) {
  if (!M || !F || !rgb || !depth || !opacity) return cf::fail(CF_E_BAD_ARG, "cf_composite: bad args");
  const float4* field = reinterpret_cast<const float4*>(field_f);
  if (M->n_rays == 0) return CF_OK;
  cf::launch_pdl(composite_kernel, cf::grid_for(M->n_rays, 128, 8), 128, 0, cf::as_stream(stream), *M, *F, field, t_term, rgb,
                                                                                        depth, opacity);
  return cf::check_launch("cf_composite");
}

int cf_keyframe_rays(const cf_camera* cam, const int* fg_pixels, int64_t n_fg, int64_t n_rays, uint64_t seed,
                     const uint64_t* seed_offset, const float* rgb, const float* depth, const uint8_t* mask_h, const uint8_t* mask_o, int* pix_out,
                     double* dirs, float* rgb_out, float* depth_out, uint8_t* mask_h_out, uint8_t* mask_o_out,
                     void* stream) {
  if (!cam || !fg_pixels || n_fg < 1 || n_rays < 0 || !rgb || !depth || !mask_h || !mask_o || !dirs || !rgb_out ||
      !depth_out || !mask_h_out || !mask_o_out)
    return cf::fail(CF_E_BAD_ARG, "cf_keyframe_rays: bad args");
  if (n_rays == 0) return CF_OK;
  keyframe_rays_kernel<<<cf::grid_for(n_rays, 256, 4), 256, 0, cf::as_stream(stream)>>>(
      *cam, fg_pixels, n_fg, n_rays, seed, seed_offset, rgb, depth, mask_h, mask_o, pix_out, dirs, rgb_out, depth_out, mask_h_out,
      mask_o_out);
  return cf::check_launch("cf_keyframe_rays");
}

int cf_train_sample(const cf_march_desc* M, const float* gt_depth, const uint8_t* mask, int n_guided, int n_uniform,
                    int n_empty, double sigma_d, uint64_t seed, const uint64_t* seed_offset, int64_t ray_id0,
                    const cf_march_out* F, double* t_out, void* stream) {
  if (!M || !F || !gt_depth || !mask || !t_out || n_guided < 1 || n_uniform < 1 || n_empty < 1 ||
      n_guided + n_uniform > 128 || n_empty > 128 || n_guided > 32)
    return cf::fail(CF_E_BAD_ARG, "cf_train_sample: bad args");
  cudaStream_t st = cf::as_stream(stream);
  cf::fill_list(st, {{F->counters, 0u, 4}});
  if (M->n_rays == 0) return CF_OK;
  train_sample_kernel<<<cf::grid_for(M->n_rays, 128, 8), 128, 0, st>>>(*M, gt_depth, mask, n_guided, n_uniform,
                                                                        n_empty, sigma_d, seed, seed_offset, ray_id0, *F,
                                                                        t_out);
  return cf::check_launch("cf_train_sample");
}

int cf_loss_composite_bwd(const cf_march_desc* M, const cf_march_out* F, const float* field, float t_term,
                          const float* gt_rgb, const float* gt_depth, const uint8_t* mask, float lambda_depth,
                          const float* norm, float* grad, float* loss, void* stream) {
  if (!M || !F || !field || !gt_rgb || !gt_depth || !mask || !grad || !norm)
    return cf::fail(CF_E_BAD_ARG, "cf_loss_composite_bwd: bad args");
  if (M->n_rays == 0) return CF_OK;
  composite_bwd_kernel<<<cf::grid_for(M->n_rays, 128, 8), 128, 0, cf::as_stream(stream)>>>(
      *M, *F, reinterpret_cast<const float4*>(field), t_term, gt_rgb, gt_depth, mask, lambda_depth, norm,
      reinterpret_cast<float4*>(grad), loss);
  return cf::check_launch("cf_loss_composite_bwd");
}

int cf_composite_layers(int64_t n, const float* h_rgb, const float* h_depth, const float* h_opac, const float* o_rgb,
                        const float* o_depth, const float* o_opac, const float* bg, float* out, uint8_t* layer,
                        void* stream) {
  if (n < 0 || !bg || !out) return cf::fail(CF_E_BAD_ARG, "cf_composite_layers: bad args");
  if (n == 0) return CF_OK;
  cf::launch_pdl(layers_kernel, cf::grid_for(n, 256, 4), 256, 0, cf::as_stream(stream), n, h_rgb, h_depth, h_opac, o_rgb, o_depth,
                                                                             o_opac, bg[0], bg[1], bg[2], out, layer);
  return cf::check_launch("cf_composite_layers");
}

int cf_composite_final(const cf_march_desc* M, const cf_march_out* F, const float* field, float t_term, float* rgb,
                       float* depth, float* opacity, const float* o_rgb, const float* o_depth, const float* o_opac,
                       const float* bg, float* out, uint8_t* layer, void* stream) {
  if (!M || !F || !field || !rgb || !depth || !opacity || !bg || !out || (o_rgb && (!o_depth || !o_opac)))
    return cf::fail(CF_E_BAD_ARG, "cf_composite_final: bad args");
  if (M->n_rays == 0) return CF_OK;
  cf::launch_pdl(composite_final_kernel, cf::grid_for(M->n_rays, 128, 8), 128, 0, cf::as_stream(stream), *M, *F,
                 reinterpret_cast<const float4*>(field), t_term, rgb, depth, opacity, o_rgb, o_depth, o_opac, bg[0],
                 bg[1], bg[2], out, layer);
  return cf::check_launch("cf_composite_final");
}

// Device -> pinned-host copy by a few SMs storing straight into the (UVA-mapped)
// pinned buffer: unlike a copy-engine memcpy it never queues in front of the next
// frame's small host -> device uploads, so the read-back overlaps the next view.
// Small host -> device upload by one CTA reading the pinned (UVA-mapped) source: it
// never waits behind a copy-engine read-back of the previous view.
int cf_load_from_host(void* dst, const void* src_host, int64_t bytes, void* stream) {
  if (!dst || !src_host || bytes < 0 || (bytes % 16) != 0 || ((uintptr_t)dst | (uintptr_t)src_host) % 16 != 0)
    return cf::fail(CF_E_BAD_ARG, "cf_load_from_host: 16-byte aligned buffers and sizes required");
  if (bytes == 0) return CF_OK;
  void* src = nullptr;
  CF_CHECK_CUDA(cudaHostGetDevicePointer(&src, const_cast<void*>(src_host), 0));
  store_to_host_kernel<<<1, 256, 0, cf::as_stream(stream)>>>(reinterpret_cast<const uint4*>(src),
                                                             reinterpret_cast<uint4*>(dst), bytes / 16);
  return cf::check_launch("cf_load_from_host");
}

int cf_store_to_host(const void* src, void* dst_host, int64_t bytes, int ctas, void* stream) {
  if (!src || !dst_host || bytes < 0 || (bytes % 16) != 0 || ((uintptr_t)src | (uintptr_t)dst_host) % 16 != 0)
    return cf::fail(CF_E_BAD_ARG, "cf_store_to_host: 16-byte aligned buffers and sizes required");
  if (bytes == 0) return CF_OK;
  void* dst = nullptr;
  CF_CHECK_CUDA(cudaHostGetDevicePointer(&dst, dst_host, 0));
  store_to_host_kernel<<<ctas < 1 ? 8 : ctas, 256, 0, cf::as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), bytes / 16);
  return cf::check_launch("cf_store_to_host");
}

int cf_copy_batch(const cf_copy_list* list, void* stream) {
  if (!list || list->n < 0 || list->n > CF_COPY_BATCH_MAX) return cf::fail(CF_E_BAD_ARG, "cf_copy_batch: bad list");
  if (list->n == 0) return CF_OK;
  cf_copy_list L = *list;
  for (int e = 0; e < L.n; ++e) {
    if (!L.src[e] || !L.dst[e] || L.bytes[e] < 0) return cf::fail(CF_E_BAD_ARG, "cf_copy_batch: bad entry");
    cudaPointerAttributes a;
    CF_CHECK_CUDA(cudaPointerGetAttributes(&a, L.src[e]));
    if (a.type == cudaMemoryTypeHost) {
      if (!a.devicePointer) return cf::fail(CF_E_BAD_ARG, "cf_copy_batch: host source is not mapped (pin it)");
      L.src[e] = a.devicePointer;
    } else if (a.type == cudaMemoryTypeUnregistered) {
      return cf::fail(CF_E_BAD_ARG, "cf_copy_batch: pageable host source (pin it)");
    }
  }
  copy_batch_kernel<<<L.n, 256, 0, cf::as_stream(stream)>>>(L);
  return cf::check_launch("cf_copy_batch");
}

}  // extern "C"
