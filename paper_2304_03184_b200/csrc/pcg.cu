// Jacobi-preconditioned CG on the damped Gauss-Newton normal equations of the
// non-rigid tracker (tracking.py:158-193):
//   (J^T J + lambda diag(J^T J)) x = -J^T r
// as ONE cooperative persistent kernel: the whole iteration (two CSR SpMVs, three
// dot products, the vector updates and the stopping tests) runs between grid-wide
// barriers, so a solve is a single launch instead of ~10 launches and 3 host syncs
// per iteration. J and J^T are CSR (J^T built once per system). Dot products are
// block partials reduced in a fixed order after each barrier (deterministic).
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kPcgThreads = 256;

struct PcgWork {
  double *b, *res, *z, *p, *Ap, *minv, *lamd, *t, *part;
};

// sum of this block's `v` (all threads get it); writes the block partial
__device__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) smem[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kPcgThreads / 32; ++k) s += smem[k];
    smem[32] = s;
  }
  __syncthreads();
  s = smem[32];
  __syncthreads();
  return s;
}

// row `row` of a CSR matrix times v, by one warp (lanes stride the row's entries)
__device__ __forceinline__ double warp_row_dot(const cf_csr& M, int64_t row, const double* __restrict__ v) {
  const int lane = threadIdx.x & 31;
  const int a = M.rowptr[row], b = M.rowptr[row + 1];
  double s = 0.0;
  for (int k = a + lane; k < b; k += 32) s += __ldg(M.val + k) * v[__ldg(M.col + k)];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// grid total of the per-block partials part[0 .. gridDim.x) (fixed order), to every thread
__device__ double grid_total(const double* part, double* smem) {
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kPcgThreads) v += part[b];
  return block_sum(v, smem);
}

__global__ void __launch_bounds__(kPcgThreads) pcg_kernel(cf_csr J, cf_csr JT, const double* __restrict__ r,
                                                          double lambda, int max_iters, double tol,
                                                          double* __restrict__ x, PcgWork W, int* __restrict__ iters) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double smem[40];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t gwarp = tid / 32, nwarps = nthr / 32;
  const int lane = threadIdx.x & 31;
  const int n = JT.rows;  // unknowns
  // b = -J^T r, diag(J^T J), preconditioner, x = 0, res = b, z = M^-1 res, p = z
  // (SpMVs: one warp per row; elementwise work: one thread per unknown)
  for (int64_t i = gwarp; i < n; i += nwarps) {
    const double s = warp_row_dot(JT, i, r);
    double d = 0.0;
    for (int k = JT.rowptr[i] + lane; k < JT.rowptr[i + 1]; k += 32) d += JT.val[k] * JT.val[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) {
      W.b[i] = -s;
      W.lamd[i] = d;  // diag(J^T J) for now
    }
  }
  grid.sync();
  double any = 0.0, bb = 0.0, rz = 0.0;
  for (int64_t i = tid; i < n; i += nthr) {
    const double d = W.lamd[i];
    const double b = W.b[i];
    const double damped = (1.0 + lambda) * d;
    const double mi = damped > 1e-300 ? 1.0 / fmax(damped, 1e-300) : 0.0;
    W.res[i] = b;
    W.minv[i] = mi;
    W.lamd[i] = lambda * d;
    const double z = mi * b;
    W.z[i] = z;
    W.p[i] = z;
    x[i] = 0.0;
    any += b != 0.0 ? 1.0 : 0.0;
    bb += b * b;
    rz += b * z;
  }
  const double s_any = block_sum(any, smem), s_bb = block_sum(bb, smem), s_rz = block_sum(rz, smem);
  if (threadIdx.x == 0) {
    W.part[blockIdx.x] = s_any;
    W.part[gridDim.x + blockIdx.x] = s_bb;
    W.part[2 * gridDim.x + blockIdx.x] = s_rz;
  }
  grid.sync();
  const double n_any = grid_total(W.part, smem);
  const double b_norm = sqrt(grid_total(W.part + gridDim.x, smem));
  rz = grid_total(W.part + 2 * gridDim.x, smem);
  int it = 0;
  if (n_any > 0.0) {
    for (; it < max_iters; ++it) {
      grid.sync();  // p complete; partial slots free
      // t = J p
      for (int64_t row = gwarp; row < J.rows; row += nwarps) {
        const double s = warp_row_dot(J, row, W.p);
        if (lane == 0) W.t[row] = s;
      }
      grid.sync();
      // Ap = J^T t + lam_d p ; pAp
      double pap = 0.0;
      for (int64_t i = gwarp; i < n; i += nwarps) {
        const double s = warp_row_dot(JT, i, W.t);
        if (lane == 0) {
          const double ap = s + W.lamd[i] * W.p[i];
          W.Ap[i] = ap;
          pap += W.p[i] * ap;
        }
      }
      pap = block_sum(pap, smem);
      if (threadIdx.x == 0) W.part[blockIdx.x] = pap;
      grid.sync();
      pap = grid_total(W.part, smem);
      if (pap <= 0.0) break;
      const double alpha = rz / pap;
      double rr = 0.0;
      for (int64_t i = tid; i < n; i += nthr) {
        x[i] += alpha * W.p[i];
        const double rs = W.res[i] - alpha * W.Ap[i];
        W.res[i] = rs;
        rr += rs * rs;
      }
      rr = block_sum(rr, smem);
      if (threadIdx.x == 0) W.part[gridDim.x + blockIdx.x] = rr;
      grid.sync();
      if (sqrt(grid_total(W.part + gridDim.x, smem)) <= tol * b_norm) {
        ++it;
        break;
      }
      double rzn = 0.0;
      for (int64_t i = tid; i < n; i += nthr) {
        const double z = W.minv[i] * W.res[i];
        W.z[i] = z;
        rzn += W.res[i] * z;
      }
      rzn = block_sum(rzn, smem);
      if (threadIdx.x == 0) W.part[2 * gridDim.x + blockIdx.x] = rzn;
      grid.sync();
      rzn = grid_total(W.part + 2 * gridDim.x, smem);
      const double beta = rzn / rz;
      for (int64_t i = tid; i < n; i += nthr) W.p[i] = W.z[i] + beta * W.p[i];
      rz = rzn;
    }
  }
  if (tid == 0 && iters) *iters = it;
}

}  // namespace

extern "C" {

int cf_pcg_workspace_doubles(int rows, int cols, int64_t* n_doubles) {
  if (rows < 0 || cols < 0 || !n_doubles) return cf::fail(CF_E_BAD_ARG, "cf_pcg_workspace_doubles: bad args");
  *n_doubles = 7 * (int64_t)cols + rows + 3 * 1024;
  return CF_OK;
}

int cf_pcg_solve(const cf_csr* J, const cf_csr* JT, const double* r, double lm_lambda, int max_iters, double tol,
                 double* x, double* work, int* iters, void* stream) {
  if (!J || !JT || !r || !x || !work || max_iters < 0 || J->rows < 0 || J->cols < 0 || JT->rows != J->cols ||
      JT->cols != J->rows || !J->rowptr || !JT->rowptr)
    return cf::fail(CF_E_BAD_ARG, "cf_pcg_solve: bad args (JT must be J transposed)");
  if (J->cols == 0) return CF_OK;
  static int occ = 0;
  if (occ == 0) CF_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pcg_kernel, kPcgThreads, 0));
  const int64_t need = (std::max<int64_t>(J->rows, J->cols) * 32 + kPcgThreads - 1) / kPcgThreads;  // warp per row
  // as many CTAs as rows need (up to co-residency): the warp-per-row SpMVs are
  // latency-bound, so parallelism beats the cheaper barrier of a smaller grid
  int grid = (int)std::min<int64_t>(need, (int64_t)occ * cf::sm_count());
  grid = std::max(1, std::min(grid, 1024));
  const int64_t n = J->cols;
  PcgWork W;
  W.b = work;
  W.res = W.b + n;
  W.z = W.res + n;
  W.p = W.z + n;
  W.Ap = W.p + n;
  W.minv = W.Ap + n;
  W.lamd = W.minv + n;
  W.t = W.lamd + n;
  W.part = W.t + J->rows;
  cf_csr Jv = *J, JTv = *JT;
  void* args[] = {&Jv, &JTv, (void*)&r, &lm_lambda, &max_iters, &tol, &x, &W, &iters};
  CF_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)pcg_kernel, dim3(grid), dim3(kPcgThreads), args, 0,
                                            cf::as_stream(stream)));
  return cf::check_launch("cf_pcg_solve");
}

}  // extern "C"
