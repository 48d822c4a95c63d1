// Key-frame selection (Eq. 5-7):
// blur gate, per-node visibility maps and the pool's dissimilarity scan, batched on
// the device. The exact evaluation order every kernel follows is frozen in
// oracle/keyframes.py (and DESIGN.md §3.6); integer sums are exact, so the blur
// score and every pool decision are bit-identical to the oracle.
#include "common.cuh"

namespace {

__device__ __forceinline__ int64_t luma_at(const uint8_t* __restrict__ rgb, int W, int i, int j) {
  const uint8_t* p = rgb + 3 * ((int64_t)i * W + j);
  return 299 * (int64_t)p[0] + 587 * (int64_t)p[1] + 114 * (int64_t)p[2];
}

// 9-tap box sum along one axis with clamped borders (unnormalised)
__device__ __forceinline__ int64_t box9(const uint8_t* __restrict__ rgb, int H, int W, int i, int j, bool vertical) {
  int64_t s = 0;
#pragma unroll
  for (int d = -4; d <= 4; ++d) {
    if (vertical) {
      const int ii = min(max(i + d, 0), H - 1);
      s += luma_at(rgb, W, ii, j);
    } else {
      const int jj = min(max(j + d, 0), W - 1);
      s += luma_at(rgb, W, i, jj);
    }
  }
  return s;
}

// Crété-Roffet sums: sums[0..3] += (s_F_v, s_V_v, s_F_h, s_V_h) over the image
__global__ void __launch_bounds__(256) blur_sums_kernel(const uint8_t* __restrict__ rgb, int H, int W,
                                                        unsigned long long* __restrict__ sums) {
  int64_t acc[4] = {0, 0, 0, 0};
  const int64_t n = (int64_t)H * W;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / W), j = (int)(q % W);
    const int64_t y = luma_at(rgb, W, i, j);
    if (i > 0) {
      const int64_t dF = llabs(y - luma_at(rgb, W, i - 1, j));
      const int64_t dB = llabs(box9(rgb, H, W, i, j, true) - box9(rgb, H, W, i - 1, j, true));
      acc[0] += 9 * dF;
      acc[1] += max((int64_t)0, 9 * dF - dB);
    }
    if (j > 0) {
      const int64_t dF = llabs(y - luma_at(rgb, W, i, j - 1));
      const int64_t dB = llabs(box9(rgb, H, W, i, j, false) - box9(rgb, H, W, i, j - 1, false));
      acc[2] += 9 * dF;
      acc[3] += max((int64_t)0, 9 * dF - dB);
    }
  }
  __shared__ int64_t red[4][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    int64_t v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[c][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    int64_t v = 0;
    for (int k = 0; k < (int)(blockDim.x / 32); ++k) v += red[threadIdx.x][k];
    atomicAdd(&sums[threadIdx.x], (unsigned long long)v);
  }
}

__global__ void blur_finish_kernel(const unsigned long long* __restrict__ sums, double* __restrict__ score) {
  const double sfv = (double)(int64_t)sums[0], svv = (double)(int64_t)sums[1];
  const double sfh = (double)(int64_t)sums[2], svh = (double)(int64_t)sums[3];
  // (s_F - s_V) is formed in int64 first, as the oracle does
  const double bv = sums[0] == 0 ? 1.0 : __ddiv_rn((double)((int64_t)sums[0] - (int64_t)sums[1]), sfv);
  const double bh = sums[2] == 0 ? 1.0 : __ddiv_rn((double)((int64_t)sums[2] - (int64_t)sums[3]), sfh);
  (void)svv;
  (void)svh;
  *score = bv > bh ? bv : bh;
}

// Eq. 5: one thread per node, one warp writes 32 bits
__global__ void __launch_bounds__(256) visibility_kernel(const double* __restrict__ nodes, int n,
                                                         const double* __restrict__ depth, int H, int W,
                                                         cf_vis_camera cam, double eps, uint32_t* __restrict__ bits) {
  const int i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  if (i0 >= n) return;
  const int i = i0 + (threadIdx.x & 31);
  bool vis = false;
  if (i < n) {
    const double p0 = nodes[3 * i], p1 = nodes[3 * i + 1], p2 = nodes[3 * i + 2];
    double pc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      pc[k] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(p0, cam.R[3 * k]), __dmul_rn(p1, cam.R[3 * k + 1])),
                                  __dmul_rn(p2, cam.R[3 * k + 2])),
                        cam.t[k]);
    const double z = pc[2];
    if (z > 0.0) {
      const double u = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, pc[0]), z), cam.cx);
      const double v = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, pc[1]), z), cam.cy);
      if (u >= 0.0 && u <= (double)(W - 1) && v >= 0.0 && v <= (double)(H - 1)) {
        const int ui = (int)rint(u), vi = (int)rint(v);  // round half to even, as np.round
        const double D = depth[(int64_t)vi * W + ui];
        vis = D > 0.0 && fabs(__dsub_rn(z, D)) < eps;
      }
    }
  }
  const unsigned word = __ballot_sync(0xffffffffu, vis);
  if ((threadIdx.x & 31) == 0) bits[i0 / 32] = word;
}

// dissimilarity of the candidate to every pool entry (one warp per entry: lanes
// popcount the visibility xor, lane 0 accumulates the pose / time terms in the
// oracle's order), then the pool decision by one CTA.
__global__ void __launch_bounds__(256) pool_scan_kernel(cf_pool_desc P, cf_pool_entry C, double* __restrict__ dissim,
                                                        cf_pool_decision* __restrict__ dec) {
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32, nw = blockDim.x / 32;
  for (int e = w; e < P.count; e += nw) {
    double E;
    if (P.kind == CF_POOL_HUMAN) {
      int pc = 0;
      const uint32_t* va = P.vis + (int64_t)e * P.vis_words;
      for (int k = lane; k < P.vis_words; k += 32) pc += __popc(va[k] ^ C.vis[k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
      double acc = 0.0;
      if (lane == 0) {
        const double* ta = P.theta + (int64_t)e * P.n_theta;
        for (int k = 0; k < P.n_theta; ++k) {
          const double d = __dsub_rn(ta[k], C.theta[k]);
          acc = __dadd_rn(acc, __dmul_rn(P.beta_pose[k], __dmul_rn(d, d)));
        }
      }
      const double dt = __dsub_rn((double)P.t[e], (double)C.t);
      E = __dadd_rn(__dadd_rn(acc, __dmul_rn(P.beta_vis, (double)pc)), __dmul_rn(P.beta_t, __dmul_rn(dt, dt)));
    } else {
      const double* da = P.d + 3 * (int64_t)e;
      const double dx = __dsub_rn(da[0], C.d[0]), dy = __dsub_rn(da[1], C.d[1]), dz = __dsub_rn(da[2], C.d[2]);
      const double dt = __dsub_rn((double)P.t[e], (double)C.t);
      E = __dadd_rn(__dmul_rn(P.beta_d, __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz))),
                    __dmul_rn(P.beta_t, __dmul_rn(dt, dt)));
    }
    if (lane == 0) dissim[e] = E;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // min and the eviction candidate (smallest dissimilarity, ties -> oldest)
    int best = -1;
    double mn = 0.0;
    for (int e = 0; e < P.count; ++e) {
      const double v = dissim[e];
      if (best < 0 || v < mn || (v == mn && P.t[e] < P.t[best])) {
        best = e;
        mn = v;
      }
    }
    cf_pool_decision d;
    d.min_dissim = mn;
    d.nearest = best;
    if (P.count == 0) {
      d.insert = 1;
      d.evict = -1;
    } else if (!(mn > P.gamma)) {
      d.insert = 0;
      d.evict = -1;
    } else {
      d.insert = 1;
      d.evict = P.count >= P.capacity ? best : -1;
    }
    *dec = d;
  }
}

}  // namespace

extern "C" {

int cf_blur_score(const uint8_t* rgb, int height, int width, unsigned long long* sums, double* score, void* stream) {
  if (!rgb || !sums || !score || height < 16 || width < 16)
    return cf::fail(CF_E_BAD_ARG, "cf_blur_score: bad args (image must be at least 16x16)");
  cudaStream_t st = cf::as_stream(stream);
  CF_CHECK_CUDA(cudaMemsetAsync(sums, 0, 4 * sizeof(unsigned long long), st));
  blur_sums_kernel<<<cf::grid_for((int64_t)height * width, 256, 4), 256, 0, st>>>(rgb, height, width, sums);
  blur_finish_kernel<<<1, 1, 0, st>>>(sums, score);
  return cf::check_launch("cf_blur_score");
}

int cf_visibility_map(const double* nodes, int n, const double* depth, int height, int width,
                      const cf_vis_camera* cam, double eps, uint32_t* bits, void* stream) {
  if (n < 0 || !cam || height < 1 || width < 1 || (n > 0 && (!nodes || !depth || !bits)))
    return cf::fail(CF_E_BAD_ARG, "cf_visibility_map: bad args");
  if (n == 0) return CF_OK;
  visibility_kernel<<<(n + 255) / 256, 256, 0, cf::as_stream(stream)>>>(nodes, n, depth, height, width, *cam, eps,
                                                                        bits);
  return cf::check_launch("cf_visibility_map");
}

int cf_pool_scan(const cf_pool_desc* pool, const cf_pool_entry* cand, double* dissim, cf_pool_decision* decision,
                 void* stream) {
  if (!pool || !cand || !dissim || !decision || pool->count < 0 || pool->capacity < 1 ||
      pool->count > pool->capacity)
    return cf::fail(CF_E_BAD_ARG, "cf_pool_scan: bad args");
  if (pool->kind == CF_POOL_HUMAN && (pool->n_theta < 0 || pool->n_theta > 4096 || (pool->count > 0 &&
                                      (!pool->theta || !pool->vis || !pool->beta_pose || !cand->theta || !cand->vis))))
    return cf::fail(CF_E_BAD_ARG, "cf_pool_scan: human pool needs theta / visibility / beta_pose");
  if (pool->kind == CF_POOL_OBJECT && pool->count > 0 && (!pool->d || !cand->d))
    return cf::fail(CF_E_BAD_ARG, "cf_pool_scan: object pool needs translations");
  if (pool->kind != CF_POOL_HUMAN && pool->kind != CF_POOL_OBJECT)
    return cf::fail(CF_E_BAD_ARG, "cf_pool_scan: unknown pool kind");
  if (pool->count > 0 && !pool->t) return cf::fail(CF_E_BAD_ARG, "cf_pool_scan: pool needs times");
  pool_scan_kernel<<<1, 256, 0, cf::as_stream(stream)>>>(*pool, *cand, dissim, decision);
  return cf::check_launch("cf_pool_scan");
}

}  // extern "C"
