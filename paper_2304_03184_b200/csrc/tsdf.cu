// Rigid-object TSDF volume (tracking front-end; tsdf.py:17-171):
// weighted-average integration of a depth map, trilinear sampling and
// central-difference gradients, the axis-scan zero-crossing surface and the
// per-pixel ray cast. One thread per voxel / query / pixel, float64 throughout in
// the reference's elementwise operation order (numpy evaluates these expressions
// elementwise, so the order is the source's); the 3x3 rigid transforms are
// evaluated as ((x0 R_k0 + x1 R_k1) + x2 R_k2) + t_k without FMA contraction.
#include "common.cuh"

namespace {

__device__ __forceinline__ void rigid_apply(const cf_rigid& T, double x0, double x1, double x2, double* o) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
    o[k] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(x0, T.R[3 * k]), __dmul_rn(x1, T.R[3 * k + 1])),
                               __dmul_rn(x2, T.R[3 * k + 2])),
                     T.t[k]);
}

__device__ __forceinline__ double center_coord(const cf_tsdf_desc& V, int a, int idx) {
  // origin + (idx + 0.5) * voxel (tsdf.py:27-28)
  return __dadd_rn(V.origin[a], __dmul_rn(__dadd_rn((double)idx, 0.5), V.voxel));
}

// tsdf.py:33-61
__global__ void __launch_bounds__(256) integrate_kernel(cf_tsdf_desc V, const double* __restrict__ depth, int H, int W,
                                                        const uint8_t* __restrict__ mask, cf_rigid vol_to_world,
                                                        cf_rigid world_to_cam, cf_pinhole cam) {
  const int r = V.resolution;
  const int64_t n = (int64_t)r * r * r;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / ((int64_t)r * r)), j = (int)((q / r) % r), k = (int)(q % r);
    double pw[3], pc[3];
    rigid_apply(vol_to_world, center_coord(V, 0, i), center_coord(V, 1, j), center_coord(V, 2, k), pw);
    rigid_apply(world_to_cam, pw[0], pw[1], pw[2], pc);
    const double z = pc[2];
    if (!(z > 0.0)) continue;
    // camera.py:65-79 project_batch, then round half to even (tsdf.py:42-43)
    const double u = rint(__dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, pc[0]), z), cam.cx));
    const double v = rint(__dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, pc[1]), z), cam.cy));
    if (!(u >= 0.0 && u < (double)W && v >= 0.0 && v < (double)H)) continue;
    const int64_t pix = (int64_t)v * W + (int64_t)u;
    if (mask && mask[pix] == 0) continue;
    const double d = depth[pix];
    if (!(d > 0.0)) continue;
    const double sdf = __dsub_rn(d, z);
    if (!(sdf >= -V.trunc)) continue;
    const double val = fmin(1.0, __ddiv_rn(sdf, V.trunc));
    const double w_old = V.weight[q];
    V.tsdf[q] = __ddiv_rn(__dadd_rn(__dmul_rn(V.tsdf[q], w_old), val), __dadd_rn(w_old, 1.0));
    V.weight[q] = fmin(__dadd_rn(w_old, 1.0), 64.0);
  }
}

// tsdf.py:63-88: trilinear value and validity (inside and some corner observed).
// by_voxel divides exactly (== div.rn). A point outside the volume is invalid
// whatever the corners hold, so its gathers are skipped (only `valid` is used then;
// the value returned is the reference's clipped-corner interpolation otherwise).
__device__ double sample_point(const cf_tsdf_desc& V, const ExactDiv& by_voxel, const double* p, bool* valid,
                               bool need_value_outside = true, bool* inside_out = nullptr) {
  const int r = V.resolution;
  int i0[3];
  double f[3];
  bool inside = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double g = __dsub_rn(by_voxel(__dsub_rn(p[a], V.origin[a])), 0.5);
    const double fl = floor(g);
    f[a] = __dsub_rn(g, fl);
    inside = inside && fl >= 0.0 && fl < (double)(r - 1);
    i0[a] = (int)fmin(fmax(fl, 0.0), (double)(r - 2));
  }
  if (inside_out) *inside_out = inside;
  if (!inside && !need_value_outside) {
    *valid = false;
    return 0.0;
  }
  double out = 0.0;
  bool observed = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dx = c >> 2, dy = (c >> 1) & 1, dz = c & 1;  // loop order dx, dy, dz
    const double wgt = __dmul_rn(__dmul_rn(dx ? f[0] : __dsub_rn(1.0, f[0]), dy ? f[1] : __dsub_rn(1.0, f[1])),
                                 dz ? f[2] : __dsub_rn(1.0, f[2]));
    const int64_t q = ((int64_t)(i0[0] + dx) * r + (i0[1] + dy)) * r + (i0[2] + dz);
    out = __dadd_rn(out, __dmul_rn(wgt, V.tsdf[q]));
    observed = observed || V.weight[q] > 0.0;
  }
  *valid = inside && observed;
  return out;
}

// tsdf.py:90-100: central differences per metre
__device__ void gradient_point(const cf_tsdf_desc& V, const ExactDiv& by_voxel, const double* p, double* g) {
  const double h = V.voxel;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double ph[3] = {p[0], p[1], p[2]}, pl[3] = {p[0], p[1], p[2]};
    ph[a] = __dadd_rn(p[a], h);
    pl[a] = __dsub_rn(p[a], h);
    bool ok;
    const double hi = sample_point(V, by_voxel, ph, &ok), lo = sample_point(V, by_voxel, pl, &ok);
    g[a] = __ddiv_rn(__dsub_rn(hi, lo), __dmul_rn(2.0, h));
  }
}

__global__ void __launch_bounds__(256) sample_kernel(cf_tsdf_desc V, const double* __restrict__ pts, int64_t n,
                                                     double* __restrict__ val, uint8_t* __restrict__ valid,
                                                     double* __restrict__ grad) {
  const ExactDiv by_voxel(V.voxel);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const double p[3] = {pts[3 * s], pts[3 * s + 1], pts[3 * s + 2]};
    if (val) {
      bool ok;
      val[s] = sample_point(V, by_voxel, p, &ok);
      if (valid) valid[s] = ok ? 1 : 0;
    }
    if (grad) {
      double g[3];
      gradient_point(V, by_voxel, p, g);
      grad[3 * s] = g[0];
      grad[3 * s + 1] = g[1];
      grad[3 * s + 2] = g[2];
    }
  }
}

// tsdf.py:134-171: one thread per ray (all rays share the step sequence t_k)
__global__ void __launch_bounds__(128) raycast_kernel(cf_tsdf_desc V, cf_pinhole cam, cf_rigid cam_rot,
                                                      cf_rigid vol_rot, const double* __restrict__ o, int stride,
                                                      int cols, int64_t n_rays, double t0, double step, double max_t,
                                                      double* __restrict__ pts, double* __restrict__ nrm,
                                                      uint8_t* __restrict__ hit) {
  const int64_t ray = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ray >= n_rays) return;
  const double u = (double)((ray % cols) * stride), v = (double)((ray / cols) * stride);
  // camera.py:94-108: camera-frame direction, rotated to world, normalised
  double dw[3];
  rigid_apply(cam_rot, __ddiv_rn(__dsub_rn(u, cam.cx), cam.fx), __ddiv_rn(__dsub_rn(v, cam.cy), cam.fy), 1.0, dw);
  const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dw[0], dw[0]), __dmul_rn(dw[1], dw[1])),
                                         __dmul_rn(dw[2], dw[2])));
  double d[3];
  rigid_apply(vol_rot, __ddiv_rn(dw[0], nn), __ddiv_rn(dw[1], nn), __ddiv_rn(dw[2], nn), d);
  const ExactDiv by_voxel(V.voxel);
  double t = t0, prev_t = t0, prev_val = 1.0, surf_t = 0.0;
  bool found = false, entered = false;
  // Steps before the ray reaches the valid box (p in [o + v/2, o + (r - 1/2) v) per
  // axis) only advance t (invalid samples change nothing else): take them as bare
  // additions, up to a slab-test entry bound backed off by two voxels.
  {
    double t_in = -1e300, t_out = 1e300;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double lo = V.origin[a] + 0.5 * V.voxel, hi = V.origin[a] + ((double)V.resolution - 0.5) * V.voxel;
      if (d[a] != 0.0) {
        const double ta = (lo - o[a]) / d[a], tb = (hi - o[a]) / d[a];
        t_in = fmax(t_in, fmin(ta, tb));
        t_out = fmin(t_out, fmax(ta, tb));
      } else if (o[a] < lo - V.voxel || o[a] > hi + V.voxel) {
        t_in = 1e300;  // parallel to this slab and outside it: never inside
      }
    }
    const double skip_to = (t_out < t_in) ? max_t : t_in - 2.0 * V.voxel;
    while (t < max_t && t < skip_to) {
      prev_t = t;
      t = __dadd_rn(t, step);
    }
  }
  while (t < max_t) {
    const double p[3] = {__dadd_rn(o[0], __dmul_rn(t, d[0])), __dadd_rn(o[1], __dmul_rn(t, d[1])),
                         __dadd_rn(o[2], __dmul_rn(t, d[2]))};
    bool ok, inside;
    const double val = sample_point(V, by_voxel, p, &ok, false, &inside);  // outside: invalid, value unused
    // the valid box is convex and each coordinate of p is monotone in t: a ray that
    // has left it never re-enters, and nothing after that can hit
    if (inside) entered = true;
    else if (entered) break;
    if (ok && prev_val > 0.0 && val <= 0.0) {
      const double frac = __ddiv_rn(prev_val, __dsub_rn(prev_val, val));
      surf_t = __dadd_rn(prev_t, __dmul_rn(frac, __dsub_rn(t, prev_t)));
      found = true;
      break;
    }
    if (ok) prev_val = val;
    prev_t = t;
    t = __dadd_rn(t, step);
  }
  uint8_t good = 0;
  if (found) {
    const double p[3] = {__dadd_rn(o[0], __dmul_rn(surf_t, d[0])), __dadd_rn(o[1], __dmul_rn(surf_t, d[1])),
                         __dadd_rn(o[2], __dmul_rn(surf_t, d[2]))};
    double g[3];
    gradient_point(V, by_voxel, p, g);
    const double gn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])),
                                           __dmul_rn(g[2], g[2])));
    if (gn > 1e-9) {
      good = 1;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        pts[3 * ray + a] = p[a];
        nrm[3 * ray + a] = __ddiv_rn(g[a], gn);
      }
    }
  }
  hit[ray] = good;
}

// tsdf.py:102-132: zero crossings of observed voxel pairs along `axis`, written in
// the row-major order of the (r-1 along axis) slice
__global__ void __launch_bounds__(256) crossings_kernel(cf_tsdf_desc V, int axis, double* __restrict__ pts,
                                                        uint8_t* __restrict__ flag) {
  const int r = V.resolution;
  const int ni = axis == 0 ? r - 1 : r, nj = axis == 1 ? r - 1 : r, nk = axis == 2 ? r - 1 : r;
  const int64_t n = (int64_t)ni * nj * nk;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / ((int64_t)nj * nk)), j = (int)((q / nk) % nj), k = (int)(q % nk);
    const int64_t qa = ((int64_t)i * r + j) * r + k;
    const int64_t qb = qa + (axis == 0 ? (int64_t)r * r : (axis == 1 ? r : 1));
    const double a = V.tsdf[qa], b = V.tsdf[qb];
    const bool cross = __dmul_rn(a, b) <= 0.0 && a != b && V.weight[qa] > 0.0 && V.weight[qb] > 0.0 &&
                       fabs(a) < 1.0 && fabs(b) < 1.0;
    flag[q] = cross ? 1 : 0;
    if (cross) {
      const double frac = __ddiv_rn(a, __dsub_rn(a, b));
      const int idx[3] = {i, j, k};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double base = center_coord(V, c, idx[c]);
        pts[3 * q + c] = __dadd_rn(base, c == axis ? __dmul_rn(frac, V.voxel) : 0.0);
      }
    }
  }
}

}  // namespace

extern "C" {

int cf_tsdf_integrate(const cf_tsdf_desc* V, const double* depth, int height, int width, const uint8_t* mask,
                      const cf_rigid* vol_to_world, const cf_rigid* world_to_cam, const cf_pinhole* cam, void* stream) {
  if (!V || !V->tsdf || !V->weight || V->resolution < 2 || !depth || height < 1 || width < 1 || !vol_to_world ||
      !world_to_cam || !cam)
    return cf::fail(CF_E_BAD_ARG, "cf_tsdf_integrate: bad args");
  const int64_t n = (int64_t)V->resolution * V->resolution * V->resolution;
  integrate_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(*V, depth, height, width, mask,
                                                                                *vol_to_world, *world_to_cam, *cam);
  return cf::check_launch("cf_tsdf_integrate");
}

int cf_tsdf_sample(const cf_tsdf_desc* V, const double* pts, int64_t n, double* val, uint8_t* valid, double* grad,
                   void* stream) {
  if (!V || V->resolution < 2 || n < 0 || (n > 0 && !pts) || (!val && !grad))
    return cf::fail(CF_E_BAD_ARG, "cf_tsdf_sample: bad args");
  if (n == 0) return CF_OK;
  sample_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(*V, pts, n, val, valid, grad);
  return cf::check_launch("cf_tsdf_sample");
}

int cf_tsdf_raycast(const cf_tsdf_desc* V, const cf_pinhole* cam, const cf_rigid* cam_rot, const cf_rigid* vol_rot,
                    const double* origin, int stride, double t0, double step, double max_t, double* pts, double* nrm,
                    uint8_t* hit, void* stream) {
  if (!V || !cam || !cam_rot || !vol_rot || !origin || stride < 1 || !pts || !nrm || !hit || !(step > 0.0))
    return cf::fail(CF_E_BAD_ARG, "cf_tsdf_raycast: bad args");
  const int cols = (cam->width + stride - 1) / stride, rows = (cam->height + stride - 1) / stride;
  const int64_t n = (int64_t)cols * rows;
  raycast_kernel<<<(unsigned)((n + 127) / 128), 128, 0, cf::as_stream(stream)>>>(
      *V, *cam, *cam_rot, *vol_rot, origin, stride, cols, n, t0, step, max_t, pts, nrm, hit);
  return cf::check_launch("cf_tsdf_raycast");
}

int cf_tsdf_crossings(const cf_tsdf_desc* V, int axis, double* pts, uint8_t* flag, void* stream) {
  if (!V || V->resolution < 2 || axis < 0 || axis > 2 || !pts || !flag)
    return cf::fail(CF_E_BAD_ARG, "cf_tsdf_crossings: bad args");
  const int64_t n = (int64_t)(V->resolution - 1) * V->resolution * V->resolution;
  crossings_kernel<<<cf::grid_for(n, 256, 8), 256, 0, cf::as_stream(stream)>>>(*V, axis, pts, flag);
  return cf::check_launch("cf_tsdf_crossings");
}

}  // extern "C"
