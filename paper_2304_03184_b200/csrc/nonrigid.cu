// Non-rigid tracking energy and Gauss-Newton system on the device (
// tracking.py:270-508): the blended ED warp of the tracked surface samples
// (apply_blended, edgraph.py:198-205), the data / bind / reg / pose terms of
// energy_terms (tracking.py:288-336) and their Jacobian rows of _assemble
// (tracking.py:358-508), written straight into CSR at row / entry offsets the host
// computes from the term sizes, and the LM step update of the node transforms
// (_apply_step, tracking.py:502-508). One thread per sample / node / edge /
// correspondence; energies are summed with fp64 atomics.
#include "common.cuh"
#include "dq.cuh"

namespace {

constexpr double kHuberKnee = 0.01;  // tracking.py:23

__device__ __forceinline__ double huber_rho(double e) {
  const double a = fabs(e);
  return a <= kHuberKnee ? e * e : kHuberKnee * (2.0 * a - kHuberKnee);
}
__device__ __forceinline__ double huber_weight(double e) {
  const double a = fabs(e);
  return a <= kHuberKnee ? 1.0 : kHuberKnee / fmax(a, 1e-300);
}

__device__ __forceinline__ d3 ld3(const double* p) { return d3{p[0], p[1], p[2]}; }

// apply_blended: DQB of the k fixed neighbours with weights max(w, 1e-300)
__global__ void __launch_bounds__(128) nr_warp_kernel(const double* __restrict__ dqs, const int* __restrict__ idx,
                                                      const double* __restrict__ w, int k,
                                                      const double* __restrict__ pts,
                                                      const double* __restrict__ nrm, int64_t n,
                                                      double* __restrict__ out_p, double* __restrict__ out_n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    DqbAcc acc;
    for (int j = 0; j < k; ++j) acc.add(fmax(w[i * k + j], 1e-300), load_dq(dqs + 8 * (int64_t)idx[i * k + j]));
    const dq8 b = acc.result();
    const d3 p = dq_apply(b, ld3(pts + 3 * i));
    const d3 q = quat_rotate(b.r, ld3(nrm + 3 * i));
    out_p[3 * i] = p.x, out_p[3 * i + 1] = p.y, out_p[3 * i + 2] = p.z;
    out_n[3 * i] = q.x, out_n[3 * i + 1] = q.y, out_n[3 * i + 2] = q.z;
  }
}

// Energy of a term: one CTA per term (grid-stride over its rows), each thread's partial
// in a fixed order, then a fixed-order tree over the block and a plain store — the same
// sum every run (the LM accept test compares energies; atomics made near-ties flip).
__device__ __forceinline__ void block_energy_store(double e, double* __restrict__ energy) {
  __shared__ double red[1024];
  red[threadIdx.x] = e;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *energy = red[0];
}

// data term: r = n . (v - u) on the blended warp; row c: 6 entries per neighbour
// [s g wn_j, s n wn_j] at columns 6 nbr_j + 0..5 (g = v x n, s = sqrt(w huber_weight(r)))
__global__ void __launch_bounds__(1024) nr_data_kernel(const double* __restrict__ warped, const int64_t* __restrict__ ci,
                                                      const double* __restrict__ cu, const double* __restrict__ cn,
                                                      int64_t C, const int* __restrict__ bidx,
                                                      const double* __restrict__ bwn, int k, double wdata,
                                                      double* __restrict__ val, int* __restrict__ col,
                                                      double* __restrict__ res, double* __restrict__ energy) {
  double e = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = ci[c];
    const d3 v = ld3(warped + 3 * i), u = ld3(cu + 3 * c), m = ld3(cn + 3 * c);
    const double r = x_add(x_add(x_mul(m.x, x_sub(v.x, u.x)), x_mul(m.y, x_sub(v.y, u.y))), x_mul(m.z, x_sub(v.z, u.z)));
    e += huber_rho(r);
    if (!val) continue;
    const double s = sqrt(wdata * huber_weight(r));
    const d3 g = cross3(v, m);
    const double sg[3] = {s * g.x, s * g.y, s * g.z}, sm[3] = {s * m.x, s * m.y, s * m.z};
    for (int j = 0; j < k; ++j) {
      const double wn = bwn[i * k + j];
      const int nb = bidx[i * k + j];
      const int64_t o = (c * k + j) * 6;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        val[o + a] = sg[a] * wn;
        col[o + a] = 6 * nb + a;
        val[o + 3 + a] = sm[a] * wn;
        col[o + 3 + a] = 6 * nb + 3 + a;
      }
    }
    res[c] = s * r;
  }
  block_energy_store(e, energy);
}

// bind term per node i (rows 3i .. 3i+2 of the block): r = dq_apply(dq_i, x_i) - LBS(x_i);
// row a: -s [v]_x[a] (cols 6i..6i+2), s I[a] (cols 6i+3..6i+5), -s Jth[i,a,:] (cols 6n..)
__global__ void __launch_bounds__(1024) nr_bind_kernel(const double* __restrict__ dqs, const double* __restrict__ nodes,
                                                      const double* __restrict__ node_lbs,
                                                      const double* __restrict__ jth, int n, int T, double s,
                                                      double* __restrict__ val, int* __restrict__ col,
                                                      double* __restrict__ res, double* __restrict__ energy) {
  double e = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const d3 v = dq_apply(load_dq(dqs + 8 * (int64_t)i), ld3(nodes + 3 * i));
    const double r[3] = {v.x - node_lbs[3 * i], v.y - node_lbs[3 * i + 1], v.z - node_lbs[3 * i + 2]};
    e += (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
    if (!val) continue;
    const double sk[3][3] = {{0.0, -v.z, v.y}, {v.z, 0.0, -v.x}, {-v.y, v.x, 0.0}};
    for (int a = 0; a < 3; ++a) {
      const int64_t o = ((int64_t)3 * i + a) * (6 + T);
      for (int b = 0; b < 3; ++b) {
        val[o + b] = -s * sk[a][b];
        col[o + b] = 6 * i + b;
        val[o + 3 + b] = a == b ? s : 0.0;
        col[o + 3 + b] = 6 * i + 3 + b;
      }
      for (int t = 0; t < T; ++t) {
        val[o + 6 + t] = -s * jth[((int64_t)i * 3 + a) * T + t];
        col[o + 6 + t] = 6 * n + t;
      }
      res[3 * i + a] = s * r[a];
    }
  }
  block_energy_store(e, energy);
}

// reg term per edge (i, j): a = dq_i(x_j), b = dq_j(x_j), r = a - b; 12 entries per row
__global__ void __launch_bounds__(1024) nr_reg_kernel(const double* __restrict__ dqs, const double* __restrict__ nodes,
                                                     const int64_t* __restrict__ edges, int64_t E, double s,
                                                     double* __restrict__ val, int* __restrict__ col,
                                                     double* __restrict__ res, double* __restrict__ energy) {
  double e = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < E; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)edges[2 * q], j = (int)edges[2 * q + 1];
    const d3 xj = ld3(nodes + 3 * j);
    const d3 a = dq_apply(load_dq(dqs + 8 * (int64_t)i), xj), b = dq_apply(load_dq(dqs + 8 * (int64_t)j), xj);
    const double r[3] = {a.x - b.x, a.y - b.y, a.z - b.z};
    e += (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
    if (!val) continue;
    const double ska[3][3] = {{0.0, -a.z, a.y}, {a.z, 0.0, -a.x}, {-a.y, a.x, 0.0}};
    const double skb[3][3] = {{0.0, -b.z, b.y}, {b.z, 0.0, -b.x}, {-b.y, b.x, 0.0}};
    for (int row = 0; row < 3; ++row) {
      const int64_t o = (3 * q + row) * 12;
      for (int c = 0; c < 3; ++c) {
        val[o + c] = -s * ska[row][c];
        col[o + c] = 6 * i + c;
        val[o + 3 + c] = s * skb[row][c];
        col[o + 3 + c] = 6 * j + c;
        val[o + 6 + c] = row == c ? s : 0.0;
        col[o + 6 + c] = 6 * i + 3 + c;
        val[o + 9 + c] = row == c ? -s : 0.0;
        col[o + 9 + c] = 6 * j + 3 + c;
      }
      res[3 * q + row] = s * r[row];
    }
  }
  block_energy_store(e, energy);
}

// pose term per correspondence p: r = n . (LBS(x_p) - u); row: s (n . Jth[p]) over theta
__global__ void __launch_bounds__(1024) nr_pose_kernel(const double* __restrict__ lbs_pts, const double* __restrict__ pu,
                                                      const double* __restrict__ pn, const double* __restrict__ jth,
                                                      int64_t P, int T, int n_nodes, double wpose,
                                                      double* __restrict__ val, int* __restrict__ col,
                                                      double* __restrict__ res, double* __restrict__ energy) {
  double e = 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const d3 l = ld3(lbs_pts + 3 * p), u = ld3(pu + 3 * p), m = ld3(pn + 3 * p);
    const double r = (m.x * (l.x - u.x) + m.y * (l.y - u.y)) + m.z * (l.z - u.z);
    e += huber_rho(r);
    if (!val) continue;
    const double s = sqrt(wpose * huber_weight(r));
    for (int t = 0; t < T; ++t) {
      const double* J = jth + p * 3 * T;
      val[p * T + t] = ((m.x * J[t] + m.y * J[T + t]) + m.z * J[2 * T + t]) * s;
      col[p * T + t] = 6 * n_nodes + t;
    }
    res[p] = s * r;
  }
  block_energy_store(e, energy);
}

// _apply_step: dq_i <- normalize(dq(quat(xi_i[:3]), xi_i[3:]) * dq_i)
__global__ void __launch_bounds__(128) nr_step_kernel(const double* __restrict__ dqs, const double* __restrict__ delta,
                                                      int n, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* xi = delta + 6 * (int64_t)i;
    const double ang = sqrt((xi[0] * xi[0] + xi[1] * xi[1]) + xi[2] * xi[2]);
    const double half = 0.5 * ang;
    const double kk = ang < 1e-12 ? 0.5 - ang * ang / 48.0 : sin(half) / ang;
    dq8 u;
    u.r[0] = cos(half), u.r[1] = kk * xi[0], u.r[2] = kk * xi[1], u.r[3] = kk * xi[2];
    const double tq[4] = {0.0, xi[3], xi[4], xi[5]};
    double du[4];
    qmul(tq, u.r, du);
#pragma unroll
    for (int c = 0; c < 4; ++c) u.d[c] = 0.5 * du[c];
    const dq8 q = load_dq(dqs + 8 * (int64_t)i);
    dq8 m;
    qmul(u.r, q.r, m.r);
    double d1[4], d2[4];
    qmul(u.r, q.d, d1);
    qmul(u.d, q.r, d2);
#pragma unroll
    for (int c = 0; c < 4; ++c) m.d[c] = d1[c] + d2[c];
    const dq8 o = dq_normalize(m);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      out[8 * (int64_t)i + c] = o.r[c];
      out[8 * (int64_t)i + 4 + c] = o.d[c];
    }
  }
}

}  // namespace

extern "C" {

int cf_nr_warp(const double* dqs, const int* idx, const double* w, int k, const double* pts, const double* normals,
               int64_t n, double* out_pts, double* out_normals, void* stream) {
  if (k < 1 || n < 0 || (n > 0 && (!dqs || !idx || !w || !pts || !normals || !out_pts || !out_normals)))
    return cf::fail(CF_E_BAD_ARG, "cf_nr_warp: bad args");
  if (n == 0) return CF_OK;
  nr_warp_kernel<<<cf::grid_for(n, 128, 8), 128, 0, cf::as_stream(stream)>>>(dqs, idx, w, k, pts, normals, n, out_pts,
                                                                            out_normals);
  return cf::check_launch("cf_nr_warp");
}

int cf_nr_terms(const cf_nr_system* S, void* stream) {
  if (!S || !S->energy) return cf::fail(CF_E_BAD_ARG, "cf_nr_terms: bad args");
  cudaStream_t st = cf::as_stream(stream);
  cf::fill_u32(S->energy, 0u, 2 * 4, st);  // data, bind, reg, pose
  const bool J = S->val != nullptr;
  // a term's Jacobian rows are written only when val is set and its jac_terms bit is on;
  // its energy is always evaluated (the reference's energy_terms computes every term)
  auto on = [&](int bit) { return J && (S->jac_terms & (1 << bit)); };
  auto V = [&](int64_t e, int bit) { return on(bit) ? S->val + e : nullptr; };
  auto Cc = [&](int64_t e, int bit) { return on(bit) ? S->col + e : nullptr; };
  auto R = [&](int64_t r, int bit) { return on(bit) ? S->res + r : nullptr; };
  if (S->n_data > 0)
    nr_data_kernel<<<1, 1024, 0, st>>>(S->warped, S->data_idx, S->data_u, S->data_n, S->n_data, S->blend_idx,
                                       S->blend_wn, S->k, S->w_data, V(S->data_entry0, 0), Cc(S->data_entry0, 0),
                                       R(S->data_row0, 0), S->energy + 0);
  if (S->do_bind)
    nr_bind_kernel<<<1, 1024, 0, st>>>(S->dqs, S->nodes, S->node_lbs, S->node_jth, S->n_nodes, S->n_theta,
                                       S->s_bind, V(S->bind_entry0, 1), Cc(S->bind_entry0, 1), R(S->bind_row0, 1),
                                       S->energy + 1);
  if (S->n_edges > 0)
    nr_reg_kernel<<<1, 1024, 0, st>>>(S->dqs, S->nodes, S->edges, S->n_edges, S->s_reg, V(S->reg_entry0, 2),
                                      Cc(S->reg_entry0, 2), R(S->reg_row0, 2), S->energy + 2);
  if (S->n_pose > 0)
    nr_pose_kernel<<<1, 1024, 0, st>>>(S->pose_lbs, S->pose_u, S->pose_n, S->pose_jth, S->n_pose, S->n_theta,
                                       S->n_nodes, S->w_pose, V(S->pose_entry0, 3), Cc(S->pose_entry0, 3),
                                       R(S->pose_row0, 3), S->energy + 3);
  return cf::check_launch("cf_nr_terms");
}

int cf_nr_step(const double* dqs, const double* delta, int n, double* out, void* stream) {
  if (n < 0 || (n > 0 && (!dqs || !delta || !out))) return cf::fail(CF_E_BAD_ARG, "cf_nr_step: bad args");
  if (n == 0) return CF_OK;
  nr_step_kernel<<<cf::grid_for(n, 128, 4), 128, 0, cf::as_stream(stream)>>>(dqs, delta, n, out);
  return cf::check_launch("cf_nr_step");
}

}  // extern "C"
