// One-point ED warp on the coarse buckets: exact k-NN (ties by index) ->
// Gaussian weights -> DQB -> (inverse) apply, the body of
// edgraph._blend_for + warp_backward_batch / warp_forward_batch
// (edgraph.py:139-183) for a single float64 point.
#pragma once
#include "buckets.cuh"
#include "dq.cuh"

// header of a candidate grid (cf_cand_grid_build, knn.cu), followed at byte 64 by the
// per-cell lists: uint16 count (0xFFFF = more than cmax) then cmax node ids, each list
// padded to a 16-byte multiple (cand_stride entries) so a reader takes 8 at a time
struct CandGridHdr {
  double origin[3];
  double h, inv_h;
  int dims[3];
  int cmax;
};
static_assert(sizeof(CandGridHdr) <= 64, "candidate-grid header");
__host__ __device__ constexpr int64_t cand_stride(int cmax) { return ((int64_t)cmax + 1 + 7) & ~(int64_t)7; }

template <int K>
__device__ __forceinline__ bool blend_apply(const TopK<K>& top, const double* __restrict__ dqs, int k, double r2,
                                            bool inverse, d3 p, d3& out);

template <int K>
__device__ __forceinline__ bool ed_warp_point(const BucketParams& P, const int* __restrict__ cell_start,
                                              const double4* __restrict__ sorted, const double* __restrict__ dqs,
                                              int k, double r2, bool inverse, d3 p, d3& out) {
  TopK<K> top;
  top.init(k);
  bucket_knn<K>(P, cell_start, sorted, p, top);
  return blend_apply<K>(top, dqs, k, r2, inverse, p, out);
}

// Small graphs: exhaustive scan of the anchors staged in shared memory (every
// thread reads the same anchor at once — a broadcast, no bank conflicts).
// Same (d2, index) order, hence bit-identical to the bucket search.
template <int K>
__device__ __forceinline__ bool ed_warp_point_smem(const double4* __restrict__ s_anchors,
                                                   const float4* __restrict__ s_af, int n,
                                                   const double* __restrict__ dqs, int k, double r2, bool inverse,
                                                   d3 p, d3& out) {
  TopK<K> top;
  top.init(k);
  // fp32 prefilter: a candidate whose fp32 squared distance exceeds the current
  // k-th best by more than the fp32 error bound cannot enter the top-k, so only
  // survivors pay the exact float64 evaluation. The error of the fp32 d^2 (from
  // rounding p and the anchor to fp32) is <= ~2|d| sqrt(3) 2^-23 max|coord|;
  // `slack` bounds it for coordinates up to `mag` (s_af[0].w = max |anchor coord|).
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  const float mag = fmaxf(fmaxf(fabsf(px), fmaxf(fabsf(py), fabsf(pz))), s_af[0].w) + 1.0f;
  const float slack = 64.0f * 1.1920929e-7f * mag * mag;
  float bound = __int_as_float(0x7f800000);  // +inf until k candidates are in
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    const float4 af = s_af[i];
    const float dx = px - af.x, dy = py - af.y, dz = pz - af.z;
    const float fd = dx * dx + dy * dy + dz * dz;
    if (fd > bound) continue;
    const double4 a = s_anchors[i];
    top.insert(sqdist(p, d3{a.x, a.y, a.z}), i);
    bound = (float)top.worst_d() * (1.0f + 4.0f * 1.1920929e-7f) + slack;
  }
  return blend_apply<K>(top, dqs, k, r2, inverse, p, out);
}

// ballot of the nodes (w*32 + lane) whose nearest distance^2 to the box [lo, hi] is <= cut
__device__ __forceinline__ unsigned cull_ballot(const float4* __restrict__ s_af, int n, int i, const float* lo,
                                                const float* hi, float cut) {
  bool cand = false;
  if (i < n) {
    const float4 a = s_af[i];
    const float dx = fmaxf(fmaxf(lo[0] - a.x, a.x - hi[0]), 0.f);
    const float dy = fmaxf(fmaxf(lo[1] - a.y, a.y - hi[1]), 0.f);
    const float dz = fmaxf(fmaxf(lo[2] - a.z, a.z - hi[2]), 0.f);
    cand = dx * dx + dy * dy + dz * dz <= cut;
  }
  return __ballot_sync(0xffffffffu, cand);
}

// Warp-cooperative culling for the exhaustive scan (all 32 lanes must call it,
// `live` marks lanes holding a sample). The warp's samples are spatially
// coherent (consecutive compacted samples of neighbouring rays), so:
//  1. bbox B of the warp's samples (fp32);
//  2. U = k-th smallest, over all nodes, of the farthest distance^2 from B —
//     every sample in B has its k-th neighbour within U;
//  3. only nodes whose nearest distance^2 to B is <= U (+ fp32 slack) can be
//     in any lane's top-k; the warp walks that candidate set uniformly
//     (ballot masks, smem broadcast reads): pass 1 ranks the candidates per
//     lane in fp32, pass 2 re-ranks the few that can still be in the top-k
//     exactly in float64. Identical result to scanning every node.
// n <= 2^IDXB (pass 1 packs the node index into IDXB key bits). `a64(i)` returns
// node i in float64 (shared or global memory); s_af holds the fp32 copies with
// s_af[0].w = max |coordinate|. Lanes with live = false only cooperate.
template <int K, int IDXB, class A64>
__device__ __forceinline__ void cull_topk(const A64& a64, const float4* __restrict__ s_af, int n, int k, d3 p,
                                          bool live, TopK<K>& top) {
  static_assert(IDXB >= 1 && IDXB <= 16, "node index bits");
  constexpr unsigned IMASK = (1u << IDXB) - 1u;
  // 2x the relative truncation of the fp32 d^2 by IDXB low bits: 2^(IDXB - 22)
  constexpr float TRUNC = 1.0f / (float)(1u << (22 - IDXB));
  const unsigned FULL = 0xffffffffu;
  top.init(k);
  const int lane = threadIdx.x & 31;
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  const float INF = __int_as_float(0x7f800000);
  float lo[3] = {live ? px : INF, live ? py : INF, live ? pz : INF};
  float hi[3] = {live ? px : -INF, live ? py : -INF, live ? pz : -INF};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(FULL, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(FULL, hi[a], o));
    }
  const float mag = fmaxf(fmaxf(fmaxf(fabsf(lo[0]), fabsf(hi[0])), fmaxf(fmaxf(fabsf(lo[1]), fabsf(hi[1])),
                                                                       fmaxf(fabsf(lo[2]), fabsf(hi[2])))),
                          s_af[0].w) + 1.0f;
  const float slack = 64.0f * 1.1920929e-7f * mag * mag;
  // per-lane k smallest farthest-distances of its nodes (i = lane, lane+32, ...)
  float best[K];
#pragma unroll
  for (int j = 0; j < K; ++j) best[j] = INF;
  for (int i = lane; i < n; i += 32) {
    const float4 a = s_af[i];
    const float ex = fmaxf(fabsf(a.x - lo[0]), fabsf(a.x - hi[0]));
    const float ey = fmaxf(fabsf(a.y - lo[1]), fabsf(a.y - hi[1]));
    const float ez = fmaxf(fabsf(a.z - lo[2]), fabsf(a.z - hi[2]));
    float v = ex * ex + ey * ey + ez * ez;
#pragma unroll
    for (int j = 0; j < K; ++j) {  // insertion into the sorted per-lane list
      const float lo_v = fminf(v, best[j]);
      v = fmaxf(v, best[j]);
      best[j] = lo_v;
    }
  }
  // k rounds of a warp-wide min with removal -> the k-th smallest overall
  float U = INF;
  for (int r = 0; r < k; ++r) {
    float m = best[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(FULL, m, o));
    U = m;
    const unsigned owner = __ballot_sync(FULL, best[0] == m);
    if (lane == __ffs(owner) - 1) {  // pop the head of the owning lane's list
#pragma unroll
      for (int j = 0; j < K - 1; ++j) best[j] = best[j + 1];
      best[K - 1] = INF;
    }
  }
  const float cut = U + 2.0f * slack;
  // Pass 1 (fp32 only): each lane keeps the L = K+2 smallest keys over the
  // warp's candidate set, key = (fp32 d^2 bits with the low IDXB mantissa bits
  // replaced by the node index) — non-negative floats order as their bits, so
  // one unsigned min/max pair per slot keeps the list sorted.
  constexpr int L = K + 2;
  unsigned key[L];
#pragma unroll
  for (int j = 0; j < L; ++j) key[j] = 0xffffffffu;
  const int nw = (n + 31) >> 5;
  for (int w = 0; w < nw; ++w) {
    unsigned mask = cull_ballot(s_af, n, (w << 5) + lane, lo, hi, cut);
    while (mask) {
      const int node = (w << 5) + __ffs(mask) - 1;
      mask &= mask - 1;
      const float4 af = s_af[node];
      const float ddx = px - af.x, ddy = py - af.y, ddz = pz - af.z;
      unsigned v = (__float_as_uint(ddx * ddx + ddy * ddy + ddz * ddz) & ~IMASK) | (unsigned)node;
#pragma unroll
      for (int j = 0; j < L; ++j) {
        const unsigned lo_v = min(v, key[j]);
        v = max(v, key[j]);
        key[j] = lo_v;
      }
    }
  }
  // Every node of the exact top-k has fp32 d^2 <= fcut: the k-th exact d^2 is
  // <= (k-th smallest fp32 d^2) + slack <= trunc(key[K-1]) (1 + TRUNC) + slack,
  // and each fp32 d^2 is within slack of its exact value. Truncation only lowers
  // keys, so key <= fcut_key <=> trunc(fp32 d^2) <= fcut. The list is complete
  // when its last slot is beyond fcut (or empty): every node outside it has a
  // key >= key[L-1].
  const float fcut = __uint_as_float(key[K - 1] & ~IMASK) * (1.0f + TRUNC) + 2.0f * slack;
  const unsigned fcut_key = __float_as_uint(fcut) | IMASK;
  const bool complete = key[L - 1] > fcut_key;
  if (__all_sync(FULL, complete || !live)) {
    // Pass 2: exact float64 ranking of the (typically k) survivors per lane
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (key[j] <= fcut_key) {
        const int node = (int)(key[j] & IMASK);
        top.insert(sqdist(p, a64(node)), node);
      }
  } else {
    // rare near-tie band wider than the list: exact scan of the candidate set
    float bound = INF;
    for (int w = 0; w < nw; ++w) {
      unsigned mask = cull_ballot(s_af, n, (w << 5) + lane, lo, hi, cut);
      while (mask) {
        const int node = (w << 5) + __ffs(mask) - 1;
        mask &= mask - 1;
        const float4 af = s_af[node];
        const float ddx = px - af.x, ddy = py - af.y, ddz = pz - af.z;
        if (ddx * ddx + ddy * ddy + ddz * ddz > bound) continue;
        top.insert(sqdist(p, a64(node)), node);
        bound = (float)top.worst_d() * (1.0f + 4.0f * 1.1920929e-7f) + slack;
      }
    }
  }
}

// render path: anchors staged in shared memory, n <= 1024
template <int K>
__device__ __forceinline__ bool ed_warp_point_cull(const double4* __restrict__ s_anchors,
                                                   const float4* __restrict__ s_af, int n,
                                                   const double* __restrict__ dqs, int k, double r2, bool inverse,
                                                   d3 p, bool live, d3& out) {
  if (!__any_sync(0xffffffffu, live)) return false;  // warp-uniform
  TopK<K> top;
  cull_topk<K, 10>([&](int i) { const double4 a = s_anchors[i]; return d3{a.x, a.y, a.z}; }, s_af, n, k, p, live,
                   top);
  if (!live) return false;
  return blend_apply<K>(top, dqs, k, r2, inverse, p, out);
}

template <int K>
__device__ __forceinline__ bool blend_apply(const TopK<K>& top, const double* __restrict__ dqs, int k, double r2,
                                            bool inverse, d3 p, d3& out) {
  double w[K];
  bool valid = false;
  const ExactDiv by_r2(r2);
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j < k) {
      w[j] = exp(by_r2(-top.d[j]));
      valid |= w[j] > 1e-6;
    }
  DqbAcc acc;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j < k) acc.add(valid ? w[j] : 1.0, load_dq(dqs + 8 * (int64_t)top.i[j]));
  dq8 b = acc.result();
  if (inverse) b = dq_conj(b);
  out = dq_apply(b, p);
  return valid;
}
