// Linear blend skinning, forward (skeleton.lbs_batch, skeleton.py:142-149) and
// the builder-defined backward warp of the hybrid deformation:
// a live sample takes the blended bone transform of its nearest posed skin
// vertex (exact 1-NN on the vertex buckets, ties by index) and applies its
// inverse. Per frame, every vertex's blended 3x4 transform and its inverse
// are precomputed, so the per-sample cost is one NN search + one affine map.
#include "buckets.cuh"

namespace {

__global__ void lbs_forward_kernel(const double* __restrict__ A, int J, const double* __restrict__ pts,
                                   const double* __restrict__ W, int64_t n, double* __restrict__ out) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double p[4] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], 1.0};
    double o[3] = {0.0, 0.0, 0.0};
    for (int j = 0; j < J; ++j) {
      const double w = W[i * J + j];
      if (w == 0.0) continue;
      const double* M = A + 16 * j;
#pragma unroll
      for (int a = 0; a < 3; ++a)
        o[a] += w * (M[4 * a] * p[0] + M[4 * a + 1] * p[1] + M[4 * a + 2] * p[2] + M[4 * a + 3] * p[3]);
    }
    out[3 * i] = o[0];
    out[3 * i + 1] = o[1];
    out[3 * i + 2] = o[2];
  }
  pdl_trigger();
}

// T_v = sum_j W[v,j] A_j[:3,:]; Tinv_v = [R^-1 | -R^-1 t]
__global__ void lbs_vertex_kernel(const double* __restrict__ A, int J, const double* __restrict__ W, int64_t V,
                                  double* __restrict__ T, double* __restrict__ Tinv) {
  pdl_wait();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    double m[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < J; ++j) {
      const double w = W[v * J + j];
      if (w == 0.0) continue;
#pragma unroll
      for (int e = 0; e < 12; ++e) m[e] += w * A[16 * j + e];
    }
    // inverse of the 3x3 block via the adjugate
    const double a = m[0], b = m[1], c = m[2], d = m[4], e = m[5], f = m[6], g = m[8], h = m[9], k = m[10];
    const double A00 = e * k - f * h, A01 = c * h - b * k, A02 = b * f - c * e;
    const double A10 = f * g - d * k, A11 = a * k - c * g, A12 = c * d - a * f;
    const double A20 = d * h - e * g, A21 = b * g - a * h, A22 = a * e - b * d;
    const double det = a * A00 + b * A10 + c * A20;
    const double id = 1.0 / det;
    const double R[9] = {A00 * id, A01 * id, A02 * id, A10 * id, A11 * id, A12 * id, A20 * id, A21 * id, A22 * id};
    const double t[3] = {m[3], m[7], m[11]};
    double* o = Tinv + 12 * v;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      o[4 * r] = R[3 * r];
      o[4 * r + 1] = R[3 * r + 1];
      o[4 * r + 2] = R[3 * r + 2];
      o[4 * r + 3] = -(R[3 * r] * t[0] + R[3 * r + 1] * t[1] + R[3 * r + 2] * t[2]);
    }
    if (T)
#pragma unroll
      for (int e2 = 0; e2 < 12; ++e2) T[12 * v + e2] = m[e2];
  }
  pdl_trigger();
}

// Per-frame setup of every skin vertex in one pass: blended transform T_v, its
// inverse, and the posed position (the lbs_forward arithmetic). The bone
// transforms are staged in shared memory and the vertex's weight row is read
// with independent vector loads up front (the separate kernels were latency
// bound: 24 dependent weight loads per thread).
constexpr int kMaxBones = 64;
__global__ void __launch_bounds__(128) lbs_setup_kernel(const double* __restrict__ A, int J,
                                                        const double* __restrict__ verts,
                                                        const double* __restrict__ W, int64_t V,
                                                        double* __restrict__ T, double* __restrict__ Tinv,
                                                        double* __restrict__ posed,
                                                        unsigned long long* __restrict__ box) {
  __shared__ double sA[kMaxBones * 16];
  pdl_wait();
  for (int i = threadIdx.x; i < J * 16; i += blockDim.x) sA[i] = A[i];
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const double p[4] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2], 1.0};
    double m[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    double o[3] = {0.0, 0.0, 0.0};
    const double* wr = W + v * J;
    for (int j0 = 0; j0 < J; j0 += 8) {
      double w8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w8[q] = j0 + q < J ? wr[j0 + q] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double w = w8[q];
        if (w == 0.0) continue;
        const double* M = sA + 16 * (j0 + q);
#pragma unroll
        for (int e = 0; e < 12; ++e) m[e] += w * M[e];
#pragma unroll
        for (int a = 0; a < 3; ++a)
          o[a] += w * (M[4 * a] * p[0] + M[4 * a + 1] * p[1] + M[4 * a + 2] * p[2] + M[4 * a + 3] * p[3]);
      }
    }
    posed[3 * v] = o[0];
    posed[3 * v + 1] = o[1];
    posed[3 * v + 2] = o[2];
    if (box) {  // the posed vertices' bounding box (keys, cf_lbs_setup); lanes with no vertex are inert
      const unsigned act = __activemask();
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        unsigned long long lo = dkey(o[a]), hi = lo;
        for (int off = 16; off > 0; off >>= 1) {
          const unsigned long long l2 = __shfl_xor_sync(act, lo, off), h2 = __shfl_xor_sync(act, hi, off);
          if ((act >> ((threadIdx.x ^ off) & 31)) & 1u) {
            lo = l2 < lo ? l2 : lo;
            hi = h2 > hi ? h2 : hi;
          }
        }
        if ((threadIdx.x & 31) == __ffs(act) - 1) {
          atomicMin(box + a, lo);
          atomicMax(box + 3 + a, hi);
        }
      }
    }
    const double a = m[0], b = m[1], c = m[2], d = m[4], e = m[5], f = m[6], g = m[8], h = m[9], k = m[10];
    const double A00 = e * k - f * h, A01 = c * h - b * k, A02 = b * f - c * e;
    const double A10 = f * g - d * k, A11 = a * k - c * g, A12 = c * d - a * f;
    const double A20 = d * h - e * g, A21 = b * g - a * h, A22 = a * e - b * d;
    const double det = a * A00 + b * A10 + c * A20;
    const double id = 1.0 / det;
    const double R[9] = {A00 * id, A01 * id, A02 * id, A10 * id, A11 * id, A12 * id, A20 * id, A21 * id, A22 * id};
    const double t[3] = {m[3], m[7], m[11]};
    double* oi = Tinv + 12 * v;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      oi[4 * r] = R[3 * r];
      oi[4 * r + 1] = R[3 * r + 1];
      oi[4 * r + 2] = R[3 * r + 2];
      oi[4 * r + 3] = -(R[3 * r] * t[0] + R[3 * r + 1] * t[1] + R[3 * r + 2] * t[2]);
    }
    if (T)
#pragma unroll
      for (int e2 = 0; e2 < 12; ++e2) T[12 * v + e2] = m[e2];
  }
  pdl_trigger();
}

template <bool kBuckets>
__global__ void __launch_bounds__(128, 4) lbs_backward_kernel(const BucketParams* __restrict__ Pp,
                                                           const int* __restrict__ cell_start,
                                                           const double4* __restrict__ sorted,
                                                           const double* __restrict__ verts, int64_t V,
                                                           const double* __restrict__ Tinv, double max_d2,
                                                           const double* __restrict__ pts, int64_t n,
                                                           int64_t* vert_out, double* pc_out, uint8_t* valid_out) {
  __shared__ BucketParams sP;
  if (kBuckets) {
    if (threadIdx.x == 0) sP = *Pp;
    __syncthreads();
  }
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const d3 p = load_d3(pts + 3 * q);
    TopK<1> top;
    top.init(1);
    if (kBuckets) {
      bucket_knn<1>(sP, cell_start, sorted, p, top);
    } else {
      for (int64_t v = 0; v < V; ++v) top.insert(sqdist(p, load_d3(verts + 3 * v)), (int)v);
    }
    const int64_t v = top.i[0];
    const double* M = Tinv + 12 * v;
    const double pc[3] = {M[0] * p.x + M[1] * p.y + M[2] * p.z + M[3], M[4] * p.x + M[5] * p.y + M[6] * p.z + M[7],
                          M[8] * p.x + M[9] * p.y + M[10] * p.z + M[11]};
    if (vert_out) vert_out[q] = v;
    if (pc_out) {
      pc_out[3 * q] = pc[0];
      pc_out[3 * q + 1] = pc[1];
      pc_out[3 * q + 2] = pc[2];
    }
    if (valid_out) valid_out[q] = top.d[0] <= max_d2 ? 1 : 0;
  }
}

// Central finite differences of forward LBS w.r.t. the pose (tracking.py:244-256,
// _lbs_theta_jacobian): A_pm = (2T, J, 4, 4) with A_pm[2k] = A(theta + h e_k),
// A_pm[2k+1] = A(theta - h e_k); one thread per (point, k).
__device__ __forceinline__ void lbs_point(const double* __restrict__ A, int J, const double* __restrict__ w,
                                          const double* p, double* o) {
  o[0] = o[1] = o[2] = 0.0;
  for (int j = 0; j < J; ++j) {
    const double wj = w[j];
    if (wj == 0.0) continue;
    const double* M = A + 16 * j;
#pragma unroll
    for (int a = 0; a < 3; ++a) o[a] += wj * (M[4 * a] * p[0] + M[4 * a + 1] * p[1] + M[4 * a + 2] * p[2] + M[4 * a + 3]);
  }
}

__global__ void __launch_bounds__(128) lbs_theta_jac_kernel(const double* __restrict__ Apm, int T, int J,
                                                            const double* __restrict__ pts,
                                                            const double* __restrict__ W, int64_t n, double inv2h,
                                                            double* __restrict__ out) {
  const int64_t total = n * T;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / T;
    const int k = (int)(q % T);
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double hi[3], lo[3];
    lbs_point(Apm + (int64_t)(2 * k) * 16 * J, J, W + i * J, p, hi);
    lbs_point(Apm + (int64_t)(2 * k + 1) * 16 * J, J, W + i * J, p, lo);
#pragma unroll
    for (int a = 0; a < 3; ++a) out[(i * 3 + a) * T + k] = (hi[a] - lo[a]) * inv2h;
  }
}

}  // namespace

extern "C" {

int cf_lbs_forward(const double* A, int J, const double* pts, const double* weights, int64_t n_pts, double* out,
                   void* stream) {
  if (J < 1 || n_pts < 0) return cf::fail(CF_E_BAD_ARG, "cf_lbs_forward: bad args");
  if (n_pts == 0) return CF_OK;
  cf::launch_pdl(lbs_forward_kernel, cf::grid_for(n_pts, 128, 8), 128, 0, cf::as_stream(stream), A, J, pts, weights, n_pts, out);
  return cf::check_launch("cf_lbs_forward");
}

int cf_lbs_vertex_transforms(const double* A, int J, const double* vert_weights, int64_t n_verts, double* T_out,
                             double* Tinv_out, void* stream) {
  if (J < 1 || n_verts < 1 || !Tinv_out) return cf::fail(CF_E_BAD_ARG, "cf_lbs_vertex_transforms: bad args");
  cf::launch_pdl(lbs_vertex_kernel, cf::grid_for(n_verts, 128, 4), 128, 0, cf::as_stream(stream), A, J, vert_weights, n_verts,
                                                                                       T_out, Tinv_out);
  return cf::check_launch("cf_lbs_vertex_transforms");
}

int cf_lbs_setup(const double* A, int J, const double* verts, const double* vert_weights, int64_t n_verts,
                 double* T_out, double* Tinv_out, double* posed_out, uint64_t* posed_box, void* stream) {
  if (J < 1 || J > kMaxBones || n_verts < 1 || !A || !verts || !vert_weights || !Tinv_out || !posed_out)
    return cf::fail(CF_E_BAD_ARG, "cf_lbs_setup: bad args");
  cudaStream_t st = cf::as_stream(stream);
  unsigned long long* box = reinterpret_cast<unsigned long long*>(posed_box);
  if (box) {  // lo keys to all-ones, hi keys to zero
    uint32_t* w = reinterpret_cast<uint32_t*>(box);
    cf::fill_list(st, {{w, 0xffffffffu, 6}, {w + 6, 0u, 6}});
  }
  // 64 threads per CTA: a few thousand vertices still spread over ~all SMs
  cf::launch_pdl(lbs_setup_kernel, cf::grid_for(n_verts, 64, 4), 64, 0, st, A, J, verts, vert_weights, n_verts, T_out,
                 Tinv_out, posed_out, box);
  return cf::check_launch("cf_lbs_setup");
}

int cf_lbs_backward(const cf_buckets_t* vert_buckets, const double* verts_posed, const double* vert_Tinv,
                    int64_t n_verts, double max_dist, const double* pts, int64_t n_pts, int64_t* vert_out,
                    double* pc_out, uint8_t* valid_out, void* stream) {
  if (n_verts < 1 || !vert_Tinv || (!vert_buckets && !verts_posed))
    return cf::fail(CF_E_BAD_ARG, "cf_lbs_backward: bad args");
  if (vert_buckets && vert_buckets->grid_res == 0) return cf::fail(CF_E_BAD_ARG, "cf_lbs_backward: buckets not built");
  if (n_pts == 0) return CF_OK;
  const unsigned grid = cf::grid_for(n_pts, 128, 8);
  cudaStream_t st = cf::as_stream(stream);
  const double md2 = max_dist * max_dist;
  if (vert_buckets)
    lbs_backward_kernel<true><<<grid, 128, 0, st>>>(vert_buckets->params, vert_buckets->cell_start,
                                                     vert_buckets->sorted, verts_posed, n_verts, vert_Tinv, md2, pts,
                                                     n_pts, vert_out, pc_out, valid_out);
  else
    lbs_backward_kernel<false><<<grid, 128, 0, st>>>(nullptr, nullptr, nullptr, verts_posed, n_verts, vert_Tinv, md2,
                                                      pts, n_pts, vert_out, pc_out, valid_out);
  return cf::check_launch("cf_lbs_backward");
}

int cf_lbs_theta_jacobian(const double* A_pm, int n_theta, int J, const double* pts, const double* weights,
                          int64_t n_pts, double fd_step, double* out, void* stream) {
  if (!A_pm || n_theta < 1 || J < 1 || n_pts < 0 || !(fd_step > 0.0) || (n_pts > 0 && (!pts || !weights || !out)))
    return cf::fail(CF_E_BAD_ARG, "cf_lbs_theta_jacobian: bad args");
  if (n_pts == 0) return CF_OK;
  lbs_theta_jac_kernel<<<cf::grid_for(n_pts * n_theta, 128, 8), 128, 0, cf::as_stream(stream)>>>(
      A_pm, n_theta, J, pts, weights, n_pts, 1.0 / (2.0 * fd_step), out);
  return cf::check_launch("cf_lbs_theta_jacobian");
}

}  // extern "C"
