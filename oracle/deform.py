"""ORACLE (test infrastructure only) — stage 1 of the hot path on the CPU.

A float64 numpy restatement of the reference's deformation algorithms. Every
arithmetic expression is evaluated in the same order as the reference (numpy
elementwise ufuncs, sequential small reductions), so outputs are bit-equal to
the reference for the same inputs apart from the last bits of exp() when the
platform's libm differs. Pinned by tests/test_oracle_golden.py.
"""
from __future__ import annotations

import numpy as np

WEIGHT_FLOOR = 1e-6  # capfields/edgraph.py:24
CHUNK = 4096


# --------------------------------------------------------------- quaternions
# capfields/transforms.py:27-40 (product), :56-63 (rotation), :137-196 (dual quats)

def qmul(a, b):
    aw, ax, ay, az = (a[..., i] for i in range(4))
    bw, bx, by, bz = (b[..., i] for i in range(4))
    return np.stack([
        aw * bw - ax * bx - ay * by - az * bz,
        aw * bx + ax * bw + ay * bz - az * by,
        aw * by - ax * bz + ay * bw + az * bx,
        aw * bz + ax * by - ay * bx + az * bw,
    ], axis=-1)


def _cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def qrot(q, v):
    u = q[..., 1:]
    t = 2.0 * _cross(u, v)
    return v + q[..., :1] * t + _cross(u, t)


def dq_translation(dq):
    real_conj = dq[..., :4] * np.array([1.0, -1.0, -1.0, -1.0])
    return 2.0 * qmul(dq[..., 4:], real_conj)[..., 1:]


def dq_apply(dq, p):
    return qrot(dq[..., :4], p) + dq_translation(dq)


def dq_conj(dq):
    return dq * np.array([1.0, -1.0, -1.0, -1.0, 1.0, -1.0, -1.0, -1.0])


def dq_normalize(dq):
    re, du = dq[..., :4], dq[..., 4:]
    norm = np.sqrt(np.sum(re * re, axis=-1, keepdims=True))
    re = re / norm
    du = du / norm
    du = du - np.sum(re * du, axis=-1, keepdims=True) * re
    return np.concatenate([re, du], axis=-1)


def dq_blend(w, dqs):
    """Sign-aligned (to neighbour 0) weighted blend, normalised (transforms.py:180-196)."""
    dots = np.sum(dqs[..., :1, :4] * dqs[..., :, :4], axis=-1, keepdims=True)
    sgn = np.where(dots < 0, -1.0, 1.0)
    return dq_normalize(np.sum(w[..., None] * sgn * dqs, axis=-2))


def dq_from_rt(R, t):
    """Rotation matrix + translation -> packed unit dual quaternion (transforms.py:89-106,154-161)."""
    R = np.asarray(R, dtype=np.float64)
    m = R
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    if tr > 0:
        s = np.sqrt(tr + 1.0) * 2.0
        q = np.array([0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s])
    elif m[0, 0] >= m[1, 1] and m[0, 0] >= m[2, 2]:
        s = np.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2.0
        q = np.array([(m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s])
    elif m[1, 1] >= m[2, 2]:
        s = np.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2.0
        q = np.array([(m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s])
    else:
        s = np.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2.0
        q = np.array([(m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s])
    q = q / np.linalg.norm(q)
    tq = np.concatenate([[0.0], np.asarray(t, dtype=np.float64)])
    return np.concatenate([q, 0.5 * qmul(tq, q)])


# --------------------------------------------------------------- exact k-NN

def knn_exact(anchors, pts, k):
    """(idx, d2) of the k nearest anchors, key (d2, index) — the stable-argsort
    order of brute_force_query (knnfield.py:36-39). Chunked (N, n) matrices."""
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    k = min(k, len(anchors))
    idx = np.empty((len(pts), k), dtype=np.int64)
    d2o = np.empty((len(pts), k))
    for s in range(0, len(pts), CHUNK):
        p = pts[s:s + CHUNK]
        d2 = np.sum((p[:, None, :] - anchors[None]) ** 2, axis=-1)
        if k < d2.shape[1]:
            # preselect, then order the candidates by (d2, index)
            cand = np.sort(np.argpartition(d2, k - 1, axis=1)[:, :k], axis=1)
            kth = np.take_along_axis(d2, cand, axis=1).max(axis=1, keepdims=True)
            # include every node tied with the k-th distance so ties resolve by index
            tie = d2 <= kth
            if (tie.sum(axis=1) > k).any():
                order = np.argsort(d2, axis=1, kind="stable")[:, :k]
            else:
                sub = np.take_along_axis(d2, cand, axis=1)
                order = np.take_along_axis(cand, np.argsort(sub, axis=1, kind="stable"), axis=1)
        else:
            order = np.argsort(d2, axis=1, kind="stable")[:, :k]
        idx[s:s + CHUNK] = order
        d2o[s:s + CHUNK] = np.take_along_axis(d2, order, axis=1)
    return idx, d2o


def deformed_nodes(nodes, dqs):
    """edgraph.py:134-136"""
    return dq_apply(np.asarray(dqs, dtype=np.float64), np.asarray(nodes, dtype=np.float64))


def warp(nodes, radius, k, dqs, pts, direction="backward"):
    """warp_backward_batch / warp_forward_batch (edgraph.py:139-183) with exact
    (d2, index)-ordered neighbours. Returns (idx, w, p_out, valid)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    dqs = np.asarray(dqs, dtype=np.float64)
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    anchors = deformed_nodes(nodes, dqs) if direction == "backward" else nodes
    idx, d2 = knn_exact(anchors, pts, k)
    w = np.exp(-d2 / (radius * radius))
    valid = w.max(axis=1) > WEIGHT_FLOOR
    blended = dq_blend(np.where(valid[:, None], w, 1.0), dqs[idx])
    if direction == "backward":
        blended = dq_conj(blended)
    return idx, w, dq_apply(blended, pts), valid


def brute_force_query(nodes, radius, dqs, pts, s):
    """knnfield.py:32-42 -> (idx, w, p_c)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    dqs = np.asarray(dqs, dtype=np.float64)
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    idx, d2 = knn_exact(deformed_nodes(nodes, dqs), pts, s)
    w = np.exp(-d2 / (radius ** 2))
    blended = dq_blend(np.maximum(w, 1e-300), dqs[idx])
    return idx, w, dq_apply(dq_conj(blended), pts)


# --------------------------------------------------------------- KnnField

class Field:
    """KnnField restatement (knnfield.py:45-222)."""

    def __init__(self, nodes, radius, resolution, s, bbox=None, support_radius=None):
        self.nodes = np.asarray(nodes, dtype=np.float64)
        self.radius = float(radius)
        self.res = int(resolution)
        self.s = int(min(s, len(self.nodes)))
        self.sup = float(support_radius if support_radius is not None else 2.0 * radius)
        if bbox is None:
            pad = self.sup + 2.0 * radius
            lo, hi = self.nodes.min(axis=0) - pad, self.nodes.max(axis=0) + pad
        else:
            lo, hi = (np.asarray(b, dtype=np.float64) for b in bbox)
        self.bmin = lo
        self.voxel = float((hi - lo).max() / self.res)
        self.nidx = self._build()
        self.live = {}
        self.lut = {}

    def centers(self, flat):
        r = self.res
        ijk = np.stack([flat // (r * r), (flat // r) % r, flat % r], axis=-1).astype(np.float64)
        return self.bmin + (ijk + 0.5) * self.voxel

    def flat_index(self, p):
        r = self.res
        ijk = np.floor((p - self.bmin) / self.voxel).astype(np.int64)
        inside = np.all((ijk >= 0) & (ijk < r), axis=-1)
        ijk = np.clip(ijk, 0, r - 1)
        return (ijk[..., 0] * r + ijk[..., 1]) * r + ijk[..., 2], inside

    def _build(self):
        """knnfield.py:93-120: expanded-form d2 through BLAS, (d2, index) order."""
        total = self.res ** 3
        out = np.full((total, self.s), -1, dtype=np.int32)
        nn2 = np.sum(self.nodes * self.nodes, axis=1)
        for a in range(0, total, 65536):
            flat = np.arange(a, min(a + 65536, total))
            c = self.centers(flat)
            d2 = np.sum(c * c, axis=1)[:, None] + nn2[None] - 2.0 * (c @ self.nodes.T)
            order = np.argsort(d2, axis=1, kind="stable")[:, :self.s]
            ok = np.take_along_axis(d2, order[:, :1], axis=1)[:, 0] <= self.sup ** 2
            out[flat[ok]] = order[ok].astype(np.int32)
        return out

    def update(self, fid, dqs):
        """knnfield.py:124-188: warp in-support centres, argmin (dist, k) per live voxel, dilate."""
        if fid in self.live:
            raise ValueError(f"frame {fid} already registered")
        dqs = np.asarray(dqs, dtype=np.float64)
        r = self.res
        total = r ** 3
        sup = np.nonzero(self.nidx[:, 0] >= 0)[0]
        fs, ks, ds = [], [], []
        for a in range(0, len(sup), 65536):
            k = sup[a:a + 65536]
            c = self.centers(k)
            nb = self.nidx[k].astype(np.int64)
            d2 = np.sum((c[:, None, :] - self.nodes[nb]) ** 2, axis=-1)
            w = np.exp(-d2 / (self.radius ** 2))
            warped = dq_apply(dq_blend(np.maximum(w, 1e-300), dqs[nb]), c)
            f, inside = self.flat_index(warped)
            lc = self.centers(f)
            dist = np.sum((warped - lc) ** 2, axis=-1)
            fs.append(f[inside]); ks.append(k[inside]); ds.append(dist[inside])
        f = np.concatenate(fs); k = np.concatenate(ks); dist = np.concatenate(ds)
        order = np.lexsort((k, dist, f))
        f, k = f[order], k[order]
        first = np.ones(len(f), dtype=bool)
        first[1:] = f[1:] != f[:-1]
        vol = np.full(total, -1, dtype=np.int32)
        vol[f[first]] = k[first]
        self.live[fid] = self._dilate(vol)
        self.lut[fid] = dqs.copy()

    def _dilate(self, vol):
        r = self.res
        v = vol.reshape(r, r, r)
        out = v.copy()
        empty = v < 0
        for axis in range(3):
            for side in (-1, +1):  # source neighbour at index - 1, then + 1
                src = np.full_like(v, -1)
                sl_dst = [slice(None)] * 3
                sl_src = [slice(None)] * 3
                if side == -1:
                    sl_dst[axis], sl_src[axis] = slice(1, r), slice(0, r - 1)
                else:
                    sl_dst[axis], sl_src[axis] = slice(0, r - 1), slice(1, r)
                src[tuple(sl_dst)] = v[tuple(sl_src)]
                take = empty & (src >= 0) & (out < 0)
                out[take] = src[take]
        return out.reshape(-1)

    def query(self, pts, fid):
        """knnfield.py:197-222 -> (nbr, w, p_c, valid)."""
        pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
        dqs = self.lut[fid]
        f, inside = self.flat_index(pts)
        kv = np.where(inside, self.live[fid][np.where(inside, f, 0)], -1)
        valid = kv >= 0
        nbr = self.nidx[np.where(valid, kv, 0)].astype(np.int64)
        nb = np.maximum(nbr, 0)
        q = dqs[nb]
        anchors = dq_apply(q, self.nodes[nb])
        d2 = np.sum((pts[:, None, :] - anchors) ** 2, axis=-1)
        w = np.where(nbr >= 0, np.exp(-d2 / (self.radius ** 2)), 0.0)
        valid &= w.max(axis=1) > WEIGHT_FLOOR
        blended = dq_blend(np.maximum(np.where(valid[:, None], w, 1.0), 1e-300), q)
        return nbr, w, dq_apply(dq_conj(blended), pts), valid


# --------------------------------------------------------------- skeleton / LBS

def rotvec_to_matrix(rv):
    """transforms.py:66-86 (quat_from_rotvec -> quat_to_matrix)."""
    rv = np.asarray(rv, dtype=np.float64)
    ang = np.linalg.norm(rv, axis=-1, keepdims=True)
    small = ang < 1e-12
    with np.errstate(invalid="ignore", divide="ignore"):
        s = np.where(small, 0.5 - ang * ang / 48.0, np.sin(0.5 * ang) / np.where(small, 1.0, ang))
    q = np.concatenate([np.cos(0.5 * ang), s * rv], axis=-1)
    w, x, y, z = (q[..., i] for i in range(4))
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], axis=-1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], axis=-1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], axis=-1),
    ], axis=-2)


def global_transforms(parents, offsets, theta):
    """forward_kinematics (skeleton.py:121-132)."""
    J = len(parents)
    R = rotvec_to_matrix(np.asarray(theta, dtype=np.float64).reshape(J, 3))
    G = np.zeros((J, 4, 4))
    for j in range(J):
        L = np.eye(4)
        L[:3, :3] = R[j]
        L[:3, 3] = offsets[j]
        G[j] = L if parents[j] < 0 else G[parents[j]] @ L
    return G


def bone_transforms(parents, offsets, theta):
    """skinning_transforms (skeleton.py:135-139): A_j = G_j(theta) G_j(0)^-1."""
    G = global_transforms(parents, offsets, theta)
    G0 = global_transforms(parents, offsets, np.zeros(3 * len(parents)))
    return G @ np.linalg.inv(G0)


def lbs(A, pts, weights):
    """lbs_batch (skeleton.py:142-149): sum_j w_j A_j [p, 1]."""
    pts = np.asarray(pts, dtype=np.float64)
    ph = np.concatenate([pts, np.ones((len(pts), 1))], axis=-1)
    per_bone = np.einsum("jab,nb->nja", A[:, :3, :], ph)
    return np.einsum("nj,nja->na", np.asarray(weights, dtype=np.float64), per_bone)


def lbs_backward(A, verts_rest, vert_weights, pts, max_dist):
    """Builder-defined backward LBS: nearest posed vertex (ties by
    index), inverse of its blended bone transform. -> (vert, p_c, valid)."""
    W = np.asarray(vert_weights, dtype=np.float64)
    T = np.einsum("vj,jab->vab", W, A[:, :3, :])          # (V, 3, 4)
    posed = np.einsum("vab,vb->va", T, np.concatenate([verts_rest, np.ones((len(verts_rest), 1))], axis=-1))
    idx, d2 = knn_exact(posed, pts, 1)
    v = idx[:, 0]
    Rinv = np.linalg.inv(T[v, :, :3])
    pc = np.einsum("nab,nb->na", Rinv, np.asarray(pts, dtype=np.float64) - T[v, :, 3])
    return v, pc, d2[:, 0] <= max_dist * max_dist, posed
