// Projective data association of the non-rigid tracker (
// tracking.py:60-150): the depth map's camera-facing normals by central differences
// of the backprojected points (depth_normals) and, per live model point, the
// projected depth pixel -> subpixel target, its normal and the distance / normal
// gates (find_correspondences). One thread per pixel / point, float64 in the
// reference's elementwise operation order; the 3x3 pose products are evaluated as
// ((x0 R_k0 + x1 R_k1) + x2 R_k2) + t_k without FMA (the reference uses BLAS there).
#include "common.cuh"

namespace {

__device__ __forceinline__ void pose_apply(const cf_rigid& T, const double* x, double* o) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
    o[k] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(x[0], T.R[3 * k]), __dmul_rn(x[1], T.R[3 * k + 1])),
                               __dmul_rn(x[2], T.R[3 * k + 2])),
                     T.t[k]);
}

// camera.py:47-55 backproject (pixel, depth) -> world, depth already clamped by the caller
__device__ __forceinline__ void backproject(const cf_pinhole& c, const cf_rigid& pose, double u, double v, double d,
                                            double* w) {
  const double pc[3] = {__dmul_rn(__ddiv_rn(__dsub_rn(u, c.cx), c.fx), d),
                        __dmul_rn(__ddiv_rn(__dsub_rn(v, c.cy), c.fy), d), d};
  pose_apply(pose, pc, w);
}

// camera.py:81-86 backproject_map at (row, col): zeros where the depth is invalid
__device__ __forceinline__ void map_point(const double* depth, int W, const cf_pinhole& c, const cf_rigid& pose,
                                          int row, int col, double* w) {
  const double d = depth[(int64_t)row * W + col];
  backproject(c, pose, (double)col, (double)row, fmax(d, 1e-12), w);
  if (!(d > 0.0)) w[0] = w[1] = w[2] = 0.0;
}

__device__ __forceinline__ double norm3(const double* a) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a[0], a[0]), __dmul_rn(a[1], a[1])), __dmul_rn(a[2], a[2])));
}

// tracking.py:60-80
__global__ void __launch_bounds__(256) normals_kernel(const double* __restrict__ depth, int H, int W, cf_pinhole cam,
                                                      cf_rigid pose, double* __restrict__ nrm) {
  const int64_t n = (int64_t)H * W;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(q / W), col = (int)(q % W);
    double out[3] = {0.0, 0.0, 0.0};
    if (row >= 1 && row < H - 1 && col >= 1 && col < W - 1) {
      auto dep = [&](int r, int c) { return depth[(int64_t)r * W + c]; };
      const bool valid = dep(row, col + 1) > 0.0 && dep(row, col - 1) > 0.0 && dep(row + 1, col) > 0.0 &&
                         dep(row - 1, col) > 0.0 && dep(row, col) > 0.0;
      double pr[3], pl[3], pd[3], pu[3];
      map_point(depth, W, cam, pose, row, col + 1, pr);
      map_point(depth, W, cam, pose, row, col - 1, pl);
      map_point(depth, W, cam, pose, row + 1, col, pd);
      map_point(depth, W, cam, pose, row - 1, col, pu);
      const double dx[3] = {__dsub_rn(pr[0], pl[0]), __dsub_rn(pr[1], pl[1]), __dsub_rn(pr[2], pl[2])};
      const double dy[3] = {__dsub_rn(pd[0], pu[0]), __dsub_rn(pd[1], pu[1]), __dsub_rn(pd[2], pu[2])};
      // np.cross(dy, dx)
      const double cr[3] = {__dsub_rn(__dmul_rn(dy[1], dx[2]), __dmul_rn(dy[2], dx[1])),
                            __dsub_rn(__dmul_rn(dy[2], dx[0]), __dmul_rn(dy[0], dx[2])),
                            __dsub_rn(__dmul_rn(dy[0], dx[1]), __dmul_rn(dy[1], dx[0]))};
      const double nn = norm3(cr);
      if (valid && nn > 1e-12) {
        const double den = fmax(nn, 1e-12);
#pragma unroll
        for (int a = 0; a < 3; ++a) out[a] = __ddiv_rn(cr[a], den);
      }
    }
    // face the camera: flip where n . (camera centre - point) < 0
    double p[3];
    map_point(depth, W, cam, pose, row, col, p);
    const double tc[3] = {__dsub_rn(pose.t[0], p[0]), __dsub_rn(pose.t[1], p[1]), __dsub_rn(pose.t[2], p[2])};
    const double dot = __dadd_rn(__dadd_rn(__dmul_rn(out[0], tc[0]), __dmul_rn(out[1], tc[1])), __dmul_rn(out[2], tc[2]));
    const double sgn = dot < 0.0 ? -1.0 : 1.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) nrm[3 * q + a] = __dmul_rn(out[a], sgn);
  }
}

// tracking.py:83-150, one thread per model point
__global__ void __launch_bounds__(256) corr_kernel(const double* __restrict__ pts, const double* __restrict__ pnrm,
                                                   int64_t n, const double* __restrict__ depth, int H, int W,
                                                   const uint8_t* __restrict__ mask, const double* __restrict__ nmap,
                                                   cf_pinhole cam, cf_rigid pose, cf_rigid w2c, double tau,
                                                   double cos_max, double* __restrict__ target,
                                                   double* __restrict__ n_u, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keep[i] = 0;
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double pc[3];
    pose_apply(w2c, p, pc);
    const double z = pc[2];
    if (!(z > 0.0)) continue;
    const double u = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, pc[0]), z), cam.cx);
    const double v = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, pc[1]), z), cam.cy);
    const double ur = rint(u), vr = rint(v);  // np.round: half to even
    if (!(ur >= 0.0 && ur < (double)W && vr >= 0.0 && vr < (double)H)) continue;
    const int ui = (int)ur, vi = (int)vr;
    const double d = depth[(int64_t)vi * W + ui];
    if (!(d > 0.0)) continue;
    if (mask && mask[(int64_t)vi * W + ui] == 0) continue;
    // subpixel target where the bilinear footprint is fully valid
    double tu = ur, tv = vr, td = d;
    const double x0 = floor(u), y0 = floor(v);
    bool sub = x0 >= 0.0 && x0 < (double)(W - 1) && y0 >= 0.0 && y0 < (double)(H - 1);
    const int x0c = (int)fmin(fmax(x0, 0.0), (double)(W - 2)), y0c = (int)fmin(fmax(y0, 0.0), (double)(H - 2));
    const int64_t b00 = (int64_t)y0c * W + x0c;
    const double c0 = depth[b00], c1 = depth[b00 + 1], c2 = depth[b00 + W], c3 = depth[b00 + W + 1];
    sub = sub && c0 > 0.0 && c1 > 0.0 && c2 > 0.0 && c3 > 0.0;
    if (mask) sub = sub && mask[b00] > 0 && mask[b00 + W] > 0 && mask[b00 + 1] > 0 && mask[b00 + W + 1] > 0;
    if (sub) {
      const double fx = __dsub_rn(u, (double)x0c), fy = __dsub_rn(v, (double)y0c);
      const double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy);
      td = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(c0, gx), gy), __dmul_rn(__dmul_rn(c1, fx), gy)),
                               __dmul_rn(__dmul_rn(c2, gx), fy)),
                     __dmul_rn(__dmul_rn(c3, fx), fy));
      tu = u;
      tv = v;
    }
    double t[3];
    backproject(cam, pose, tu, tv, td, t);
    const double* nu = nmap + 3 * ((int64_t)vi * W + ui);
    const double dd[3] = {__dsub_rn(p[0], t[0]), __dsub_rn(p[1], t[1]), __dsub_rn(p[2], t[2])};
    const double nup[3] = {nu[0], nu[1], nu[2]};
    const double ang = __dadd_rn(__dadd_rn(__dmul_rn(pnrm[3 * i], nup[0]), __dmul_rn(pnrm[3 * i + 1], nup[1])),
                                 __dmul_rn(pnrm[3 * i + 2], nup[2]));
    const bool ok = norm3(dd) < tau && norm3(nup) > 0.5 && ang > cos_max;
    if (ok) {
      keep[i] = 1;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        target[3 * i + a] = t[a];
        n_u[3 * i + a] = nup[a];
      }
    }
  }
}

// rigid_icp (tracking.py:560-620): live = pose(model), rotated normals
__global__ void __launch_bounds__(256) rigid_xform_kernel(const double* __restrict__ pts, const double* __restrict__ nrm,
                                                          int64_t n, cf_rigid T, double* __restrict__ out_p,
                                                          double* __restrict__ out_n) {
  cf_rigid Rt = T;
  Rt.t[0] = Rt.t[1] = Rt.t[2] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double o[3];
    pose_apply(T, pts + 3 * i, o);
    out_p[3 * i] = o[0], out_p[3 * i + 1] = o[1], out_p[3 * i + 2] = o[2];
    pose_apply(Rt, nrm + 3 * i, o);  // normals @ R^T (+ 0)
    out_n[3 * i] = o[0], out_n[3 * i + 1] = o[1], out_n[3 * i + 2] = o[2];
  }
}

// point-to-plane residual r = n_u . (p - u) of the kept pairs (0 elsewhere)
__global__ void __launch_bounds__(256) icp_residual_kernel(const double* __restrict__ live,
                                                           const uint8_t* __restrict__ keep,
                                                           const double* __restrict__ tgt,
                                                           const double* __restrict__ nu, int64_t n,
                                                           double* __restrict__ r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (keep[i]) {
      const double* p = live + 3 * i;
      v = __dadd_rn(__dadd_rn(__dmul_rn(nu[3 * i], __dsub_rn(p[0], tgt[3 * i])),
                              __dmul_rn(nu[3 * i + 1], __dsub_rn(p[1], tgt[3 * i + 1]))),
                    __dmul_rn(nu[3 * i + 2], __dsub_rn(p[2], tgt[3 * i + 2])));
    }
    r[i] = v;
  }
}

// Huber-weighted normal equations: sums[0..21) = upper triangle of Jr^T Jr (row-major),
// sums[21..27) = Jr^T (w r); Jr = w [p x n_u, n_u], w = sqrt(min(1, knee / |r|))
__global__ void __launch_bounds__(256) icp_normal_eq_kernel(const double* __restrict__ live,
                                                            const uint8_t* __restrict__ keep,
                                                            const double* __restrict__ nu,
                                                            const double* __restrict__ r, int64_t n, double knee,
                                                            double* __restrict__ sums) {
  double acc[27];
#pragma unroll
  for (int k = 0; k < 27; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    const double* p = live + 3 * i;
    const double* m = nu + 3 * i;
    const double ri = r[i];
    const double w = sqrt(fmin(1.0, knee / fmax(fabs(ri), 1e-300)));
    const double j[6] = {w * (p[1] * m[2] - p[2] * m[1]), w * (p[2] * m[0] - p[0] * m[2]),
                         w * (p[0] * m[1] - p[1] * m[0]), w * m[0], w * m[1], w * m[2]};
    const double rw = w * ri;
    int q = 0;
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int b = a; b < 6; ++b) acc[q++] += j[a] * j[b];
#pragma unroll
    for (int a = 0; a < 6; ++a) acc[21 + a] += j[a] * rw;
  }
  __shared__ double red[27][8];
  const int lane = threadIdx.x & 31, wp = threadIdx.x / 32;
#pragma unroll
  for (int k = 0; k < 27; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[k][wp] = v;
  }
  __syncthreads();
  if (threadIdx.x < 27) {
    double v = 0.0;
    for (int k = 0; k < (int)(blockDim.x / 32); ++k) v += red[threadIdx.x][k];
    atomicAdd(&sums[threadIdx.x], v);
  }
}

}  // namespace

extern "C" {

int cf_depth_normals(const double* depth, int height, int width, const cf_pinhole* cam, const cf_rigid* cam_pose,
                     double* normals, void* stream) {
  if (!depth || !cam || !cam_pose || !normals || height < 1 || width < 1)
    return cf::fail(CF_E_BAD_ARG, "cf_depth_normals: bad args");
  const int64_t n = (int64_t)height * width;
  normals_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(depth, height, width, *cam, *cam_pose,
                                                                             normals);
  return cf::check_launch("cf_depth_normals");
}

int cf_find_correspondences(const double* pts, const double* pt_normals, int64_t n, const double* depth, int height,
                            int width, const uint8_t* mask, const double* normals_map, const cf_pinhole* cam,
                            const cf_rigid* cam_pose, const cf_rigid* world_to_cam, double tau, double cos_max,
                            double* target, double* n_u, uint8_t* keep, void* stream) {
  if (n < 0 || !depth || !normals_map || !cam || !cam_pose || !world_to_cam || height < 1 || width < 1 ||
      (n > 0 && (!pts || !pt_normals || !target || !n_u || !keep)))
    return cf::fail(CF_E_BAD_ARG, "cf_find_correspondences: bad args");
  if (n == 0) return CF_OK;
  corr_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(
      pts, pt_normals, n, depth, height, width, mask, normals_map, *cam, *cam_pose, *world_to_cam, tau, cos_max,
      target, n_u, keep);
  return cf::check_launch("cf_find_correspondences");
}

int cf_rigid_transform(const double* pts, const double* normals, int64_t n, const cf_rigid* T, double* out_pts,
                       double* out_normals, void* stream) {
  if (n < 0 || !T || (n > 0 && (!pts || !normals || !out_pts || !out_normals)))
    return cf::fail(CF_E_BAD_ARG, "cf_rigid_transform: bad args");
  if (n == 0) return CF_OK;
  rigid_xform_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(pts, normals, n, *T, out_pts,
                                                                                 out_normals);
  return cf::check_launch("cf_rigid_transform");
}

int cf_icp_residuals(const double* live, const uint8_t* keep, const double* target, const double* n_u, int64_t n,
                     double* r, void* stream) {
  if (n < 0 || (n > 0 && (!live || !keep || !target || !n_u || !r)))
    return cf::fail(CF_E_BAD_ARG, "cf_icp_residuals: bad args");
  if (n == 0) return CF_OK;
  icp_residual_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(live, keep, target, n_u, n, r);
  return cf::check_launch("cf_icp_residuals");
}

int cf_icp_normal_equations(const double* live, const uint8_t* keep, const double* n_u, const double* r, int64_t n,
                            double knee, double* sums, void* stream) {
  if (n < 0 || !sums || (n > 0 && (!live || !keep || !n_u || !r)))
    return cf::fail(CF_E_BAD_ARG, "cf_icp_normal_equations: bad args");
  cudaStream_t st = cf::as_stream(stream);
  cf::fill_u32(sums, 0u, 27 * 2, st);
  if (n == 0) return CF_OK;
  icp_normal_eq_kernel<<<cf::grid_for(n, 256, 2), 256, 0, st>>>(live, keep, n_u, r, n, knee, sums);
  return cf::check_launch("cf_icp_normal_equations");
}

}  // extern "C"
