// Dual-quaternion algebra in float64, evaluated in exactly the operation order
// of the reference's numpy code (capfields/transforms.py), so a device result
// is bit-equal to the reference for the same float64 inputs.
//   quat_mul        transforms.py:27-40
//   quat_rotate     transforms.py:56-63   (np.cross order: a1*b2 - a2*b1, ...)
//   dq_normalize    transforms.py:137-144
//   dq_inverse      transforms.py:147-149 (conjugate of both parts)
//   dq_translation  transforms.py:164-166
//   dq_apply        transforms.py:174-177
//   dq_blend        transforms.py:180-196 (sign-aligned to the first entry)
#pragma once
#include "common.cuh"

struct dq8 {
  double r[4];  // real  [w, x, y, z]
  double d[4];  // dual  [w, x, y, z]
};

__device__ __forceinline__ dq8 load_dq(const double* p) {
  dq8 q;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    q.r[i] = p[i];
    q.d[i] = p[4 + i];
  }
  return q;
}

__device__ __forceinline__ void qmul(const double* a, const double* b, double* o) {
  const double w1 = a[0], x1 = a[1], y1 = a[2], z1 = a[3];
  const double w2 = b[0], x2 = b[1], y2 = b[2], z2 = b[3];
  o[0] = x_sub(x_sub(x_sub(x_mul(w1, w2), x_mul(x1, x2)), x_mul(y1, y2)), x_mul(z1, z2));
  o[1] = x_sub(x_add(x_add(x_mul(w1, x2), x_mul(x1, w2)), x_mul(y1, z2)), x_mul(z1, y2));
  o[2] = x_add(x_add(x_sub(x_mul(w1, y2), x_mul(x1, z2)), x_mul(y1, w2)), x_mul(z1, x2));
  o[3] = x_add(x_sub(x_add(x_mul(w1, z2), x_mul(x1, y2)), x_mul(y1, x2)), x_mul(z1, w2));
}

__device__ __forceinline__ d3 cross3(d3 a, d3 b) {
  return d3{x_sub(x_mul(a.y, b.z), x_mul(a.z, b.y)), x_sub(x_mul(a.z, b.x), x_mul(a.x, b.z)),
            x_sub(x_mul(a.x, b.y), x_mul(a.y, b.x))};
}

// v + w*t + cross(qv, t), t = 2*cross(qv, v)
__device__ __forceinline__ d3 quat_rotate(const double* q, d3 v) {
  d3 qv{q[1], q[2], q[3]};
  const double w = q[0];
  d3 c = cross3(qv, v);
  d3 t{x_mul(2.0, c.x), x_mul(2.0, c.y), x_mul(2.0, c.z)};
  d3 c2 = cross3(qv, t);
  return d3{x_add(x_add(v.x, x_mul(w, t.x)), c2.x), x_add(x_add(v.y, x_mul(w, t.y)), c2.y),
            x_add(x_add(v.z, x_mul(w, t.z)), c2.z)};
}

// 2 * quat_mul(dual, conj(real))[1:]
__device__ __forceinline__ d3 dq_translation(const dq8& q) {
  double cr[4] = {q.r[0], -q.r[1], -q.r[2], -q.r[3]};
  double o[4];
  qmul(q.d, cr, o);
  return d3{x_mul(2.0, o[1]), x_mul(2.0, o[2]), x_mul(2.0, o[3])};
}

__device__ __forceinline__ d3 dq_apply(const dq8& q, d3 p) {
  d3 a = quat_rotate(q.r, p);
  d3 t = dq_translation(q);
  return d3{x_add(a.x, t.x), x_add(a.y, t.y), x_add(a.z, t.z)};
}

__device__ __forceinline__ dq8 dq_conj(const dq8& q) {
  dq8 o;
  o.r[0] = q.r[0];
  o.d[0] = q.d[0];
#pragma unroll
  for (int i = 1; i < 4; ++i) {
    o.r[i] = -q.r[i];
    o.d[i] = -q.d[i];
  }
  return o;
}

__device__ __forceinline__ dq8 dq_normalize(const dq8& q) {
  double n = sqrt(x_add(x_add(x_add(x_mul(q.r[0], q.r[0]), x_mul(q.r[1], q.r[1])), x_mul(q.r[2], q.r[2])),
                       x_mul(q.r[3], q.r[3])));
  dq8 o;
  const ExactDiv by_n(n);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o.r[i] = by_n(q.r[i]);
    o.d[i] = by_n(q.d[i]);
  }
  double s = x_add(x_add(x_add(x_mul(o.r[0], o.d[0]), x_mul(o.r[1], o.d[1])), x_mul(o.r[2], o.d[2])),
                  x_mul(o.r[3], o.d[3]));
#pragma unroll
  for (int i = 0; i < 4; ++i) o.d[i] = x_sub(o.d[i], x_mul(s, o.r[i]));
  return o;
}

// Streaming blend accumulator: add neighbours in order j = 0..k-1; the first
// neighbour fixes the sign reference (transforms.py:194-195).
struct DqbAcc {
  double ref[4];
  dq8 acc;
  bool first;
  __device__ __forceinline__ DqbAcc() : first(true) {}
  __device__ __forceinline__ void add(double w, const dq8& q) {
    if (first) {
#pragma unroll
      for (int i = 0; i < 4; ++i) ref[i] = q.r[i];
    }
    double dot = x_add(x_add(x_add(x_mul(ref[0], q.r[0]), x_mul(ref[1], q.r[1])), x_mul(ref[2], q.r[2])),
                      x_mul(ref[3], q.r[3]));
    double ws = dot < 0.0 ? -w : w;  // (w * sign) exact
    if (first) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc.r[i] = x_mul(ws, q.r[i]);
        acc.d[i] = x_mul(ws, q.d[i]);
      }
      first = false;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc.r[i] = x_add(acc.r[i], x_mul(ws, q.r[i]));
        acc.d[i] = x_add(acc.d[i], x_mul(ws, q.d[i]));
      }
    }
  }
  __device__ __forceinline__ dq8 result() const { return dq_normalize(acc); }
};
