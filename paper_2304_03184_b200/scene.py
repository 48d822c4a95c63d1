"""Synthetic human + rigid object scene: the input generator of tests and bench.

Host-side data setup (not on the per-sample path), restating the reference's
scripted scene so the GPU box — which has no /root/reference — builds the same
inputs: the 24-joint capsule humanoid (skeleton.py:71-118), its rest-pose
surface samples (synthetic.py:160-192), greedy ED-node thinning
(edgraph.py:90-118), the scripted pose theta(t) (synthetic.py:93-110), the GT
node motions (synthetic.py:122-131), skin weights (skeleton.py:170-188), the
orbiting box (synthetic.py:29-45) and the look-at camera (camera.py:94-128).
tests/test_scene.py pins it against the reference.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------- the rig

PARENTS = np.array([-1, 0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 9, 9, 12, 13, 14, 16, 17, 18, 19, 20, 21])
OFFSETS = np.array([
    [0.00, 1.00, 0.00], [+0.09, -0.06, 0.00], [-0.09, -0.06, 0.00], [0.00, +0.12, 0.00],
    [0.00, -0.40, 0.00], [0.00, -0.40, 0.00], [0.00, +0.13, 0.00], [0.00, -0.40, 0.00],
    [0.00, -0.40, 0.00], [0.00, +0.13, 0.00], [0.00, -0.05, 0.10], [0.00, -0.05, 0.10],
    [0.00, +0.12, 0.00], [+0.08, +0.06, 0.00], [-0.08, +0.06, 0.00], [0.00, +0.13, 0.00],
    [+0.11, 0.00, 0.00], [-0.11, 0.00, 0.00], [+0.26, 0.00, 0.00], [-0.26, 0.00, 0.00],
    [+0.24, 0.00, 0.00], [-0.24, 0.00, 0.00], [+0.09, 0.00, 0.00], [-0.09, 0.00, 0.00],
])
_RADII = {(1, 2): 0.085, (3, 6, 9): 0.105, (4, 5): 0.065, (7, 8): 0.050, (10, 11): 0.038, (12,): 0.045,
          (13, 14): 0.055, (15,): 0.085, (16, 17): 0.048, (18, 19): 0.042, (20, 21): 0.036, (22, 23): 0.032}
BONE_RADII = np.zeros(24)
for _js, _r in _RADII.items():
    BONE_RADII[list(_js)] = _r
N_JOINTS = 24


def rest_joints() -> np.ndarray:
    pos = np.zeros((N_JOINTS, 3))
    for j in range(N_JOINTS):
        pos[j] = OFFSETS[j] + (pos[PARENTS[j]] if PARENTS[j] >= 0 else 0.0)
    return pos


def _rotmats(rv: np.ndarray) -> np.ndarray:
    ang = np.linalg.norm(rv, axis=-1, keepdims=True)
    small = ang < 1e-12
    with np.errstate(invalid="ignore", divide="ignore"):
        s = np.where(small, 0.5 - ang * ang / 48.0, np.sin(0.5 * ang) / np.where(small, 1.0, ang))
    w = np.cos(0.5 * ang)[..., 0]
    x, y, z = (s * rv)[..., 0], (s * rv)[..., 1], (s * rv)[..., 2]
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def forward_kinematics(theta: np.ndarray) -> np.ndarray:
    R = _rotmats(np.asarray(theta, dtype=np.float64).reshape(N_JOINTS, 3))
    G = np.zeros((N_JOINTS, 4, 4))
    for j in range(N_JOINTS):
        L = np.eye(4)
        L[:3, :3] = R[j]
        L[:3, 3] = OFFSETS[j]
        G[j] = L if PARENTS[j] < 0 else G[PARENTS[j]] @ L
    return G


def skinning_transforms(theta: np.ndarray) -> np.ndarray:
    """A_j = G_j(theta) G_j(0)^-1, (24, 4, 4) float64 (per-frame host setup)."""
    return forward_kinematics(theta) @ np.linalg.inv(forward_kinematics(np.zeros(3 * N_JOINTS)))


def _segments():
    pos = rest_joints()
    j = np.arange(1, N_JOINTS)
    return pos[PARENTS[j]], pos[j], BONE_RADII[j], PARENTS[j]


def _seg_dist(p, a, b):
    ab = b - a
    ap = p[:, None, :] - a[None]
    t = np.clip(np.sum(ap * ab[None], -1) / np.maximum(np.sum(ab * ab, -1), 1e-12), 0.0, 1.0)
    return np.linalg.norm(p[:, None, :] - (a[None] + t[..., None] * ab[None]), axis=-1)


def bone_weights(points: np.ndarray, k: int = 4, power: float = 4.0) -> np.ndarray:
    """Top-k normalised (d + 1e-3)^-power weights to the rest bone segments, (N, 24)."""
    a, b, _, drv = _segments()
    d = _seg_dist(np.atleast_2d(points), a, b)
    col = np.full((len(d), N_JOINTS), np.inf)
    for s, j in enumerate(drv):
        col[:, j] = np.minimum(col[:, j], d[:, s])
    inv = np.where(np.isfinite(col), 1.0 / (col + 1e-3) ** power, 0.0)
    cut = np.partition(inv, -k, axis=1)[:, -k][:, None]
    inv = np.where(inv >= cut, inv, 0.0)
    return inv / inv.sum(axis=1, keepdims=True)


def sample_nodes(points: np.ndarray, radius: float) -> np.ndarray:
    """Greedy radius thinning in input order (edgraph.py:90-118)."""
    kept = np.zeros((0, 3))
    r2 = radius * radius
    for p in points:
        if len(kept) == 0 or np.min(np.sum((kept - p) ** 2, axis=1)) >= r2:
            kept = np.vstack([kept, p])
    return kept


def dq_from_rt(R: np.ndarray, t: np.ndarray) -> np.ndarray:
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
    tw, tx, ty, tz = 0.0, *np.asarray(t, dtype=np.float64)
    w, x, y, z = q
    dual = 0.5 * np.array([tw * w - tx * x - ty * y - tz * z, tw * x + tx * w + ty * z - tz * y,
                           tw * y - tx * z + ty * w + tz * x, tw * z + tx * y - ty * x + tz * w])
    return np.concatenate([q, dual])


# ----------------------------------------------------------------- camera

@dataclass
class PinholeCamera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray = field(default_factory=lambda: np.eye(3))  # camera-to-world rotation
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def pixel_rays(self, uv: np.ndarray):
        """camera.py:94-108: world origins (N,3) and unit directions."""
        uv = np.asarray(uv, dtype=np.float64)
        d = np.stack([(uv[:, 0] - self.cx) / self.fx, (uv[:, 1] - self.cy) / self.fy, np.ones(len(uv))], -1)
        d = d @ self.R.T
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        return np.broadcast_to(self.t, d.shape).copy(), d

    def all_rays(self):
        us, vs = np.meshgrid(np.arange(self.width, dtype=np.float64), np.arange(self.height, dtype=np.float64))
        return self.pixel_rays(np.stack([us.reshape(-1), vs.reshape(-1)], -1))


def look_at(eye, target, up=(0.0, 1.0, 0.0)):
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    return np.stack([right, down, fwd], axis=1), eye


# ----------------------------------------------------------------- scene

@dataclass
class SceneConfig:
    frames: int = 10
    width: int = 64
    height: int = 64
    spin_turns: float = 0.25
    arm_swing: float = 0.4
    arm_swing_cycles: float = 2.0
    object_orbit_degrees: float = 360.0
    object_spin_degrees: float = 180.0
    node_sample_radius: float = 0.0805   # -> exactly 128 ED nodes
    influence_radius: float = 0.1
    n_skin_verts: int = 6890


class Scene:
    """Scripted capsule humanoid + textured box (seeded)."""

    def __init__(self, cfg: SceneConfig | None = None, seed: int = 0):
        self.cfg = cfg = cfg or SceneConfig()
        rng = np.random.default_rng(seed)
        # the reference draws palette / phases first; keep the stream aligned
        self.palette = rng.uniform(0.25, 0.9, size=(N_JOINTS, 3))
        rng.uniform(0, 2 * np.pi, size=N_JOINTS)
        rng.uniform(0, 2 * np.pi, size=N_JOINTS)
        rng.uniform(0, 2 * np.pi, size=3)
        fx = 280.0 * cfg.width / 256.0
        R, t = look_at([0.0, 1.15, 2.4], [0.0, 0.95, 0.0])
        self.camera = PinholeCamera(fx, fx, cfg.width / 2.0, cfg.height / 2.0, cfg.width, cfg.height, R, t)
        self.template_points, self.template_bones = self._surface(rng, 16000)
        self.nodes = sample_nodes(self.template_points, cfg.node_sample_radius)
        d2 = np.sum((self.nodes[:, None] - self.template_points[None]) ** 2, axis=-1)
        self.node_bones = self.template_bones[np.argmin(d2, axis=1)]
        pick = np.random.default_rng(seed).choice(len(self.template_points), cfg.n_skin_verts, replace=False)
        self.skin_verts = self.template_points[pick]
        self.skin_weights = bone_weights(self.skin_verts)
        self.box_half = np.array([0.11, 0.16, 0.13])

    def _surface(self, rng, n):
        a, b, r, drv = _segments()
        axis = b - a
        seg_len = np.linalg.norm(axis, axis=-1)
        axis_n = axis / np.sqrt(np.maximum(np.sum(axis * axis, -1), 1e-12))[:, None]
        ref = np.where(np.abs(axis_n[:, 1:2]) < 0.9, np.array([[0.0, 1.0, 0.0]]), np.array([[1.0, 0.0, 0.0]]))
        u = np.cross(axis_n, ref)
        u /= np.linalg.norm(u, axis=-1, keepdims=True)
        v = np.cross(axis_n, u)
        areas = 2 * np.pi * r * seg_len + 4 * np.pi * r * r
        counts = np.maximum((n * areas / areas.sum()).astype(int), 8)
        pts, bones = [], []
        for i in range(len(a)):
            m = counts[i]
            tt = rng.uniform(0, 1, m)
            phi = rng.uniform(0, 2 * np.pi, m)
            on_cap = rng.uniform(0, 1, m) < (4 * np.pi * r[i] ** 2) / areas[i]
            radial = np.cos(phi)[:, None] * u[i] + np.sin(phi)[:, None] * v[i]
            cyl = a[i] + tt[:, None] * (b[i] - a[i]) + r[i] * radial
            sd = rng.normal(size=(m, 3))
            sd /= np.linalg.norm(sd, axis=-1, keepdims=True)
            at_a = rng.uniform(0, 1, m) < 0.5
            comp = sd @ axis_n[i]
            flip = (at_a & (comp > 0)) | (~at_a & (comp < 0))
            sd[flip] -= 2 * comp[flip, None] * axis_n[i]
            cap = np.where(at_a[:, None], a[i], b[i]) + r[i] * sd
            pts.append(np.where(on_cap[:, None], cap, cyl))
            bones.append(np.full(m, drv[i]))
        return np.concatenate(pts), np.concatenate(bones)

    # -- motion script ------------------------------------------------------

    def _u(self, fid):
        return fid / max(1, self.cfg.frames - 1)

    def theta(self, fid: int) -> np.ndarray:
        u = self._u(fid)
        th = np.zeros(3 * N_JOINTS)
        th[1] = 2 * np.pi * self.cfg.spin_turns * u
        ang = self.cfg.arm_swing * np.sin(2 * np.pi * self.cfg.arm_swing_cycles * u)
        th[3 * 16 + 2] = ang
        th[3 * 17 + 2] = -0.6 * ang
        return th

    def bone_transforms(self, fid: int) -> np.ndarray:
        return skinning_transforms(self.theta(fid))

    def node_dqs(self, fid: int) -> np.ndarray:
        """GT ED-node motion of frame fid (synthetic.py:122-131)."""
        A = self.bone_transforms(fid)
        return np.stack([dq_from_rt(A[b, :3, :3], A[b, :3, 3]) for b in self.node_bones])

    def posed_segments(self, fid: int):
        """World capsule segments (A, B), radii and driver joints of frame fid."""
        G = forward_kinematics(self.theta(fid))
        pos = G[:, :3, 3]
        j = np.arange(1, N_JOINTS)
        return pos[PARENTS[j]], pos[j], BONE_RADII[j], PARENTS[j]

    def raycast(self, o: np.ndarray, d: np.ndarray, fid: int):
        """Analytic ray cast of the posed capsules and the box (training targets):
        -> t_human, t_object (inf = miss; distance along the unit ray), rgb, masks."""
        A, B, R, drv = self.posed_segments(fid)
        o = np.asarray(o, dtype=np.float64)
        d = np.asarray(d, dtype=np.float64)
        n = len(d)
        t_h = np.full(n, np.inf)
        hit_cap = np.zeros(n, dtype=np.int64)
        for i in range(len(A)):
            ba = B[i] - A[i]
            oa = o - A[i]
            baba = ba @ ba
            bard = d @ ba
            baoa = oa @ ba
            rdoa = np.sum(oa * d, -1)
            oaoa = np.sum(oa * oa, -1)
            a = baba - bard * bard
            b = baba * rdoa - baoa * bard
            c = baba * oaoa - baoa * baoa - R[i] * R[i] * baba
            h = b * b - a * c
            with np.errstate(invalid="ignore", divide="ignore"):
                t = (-b - np.sqrt(np.maximum(h, 0.0))) / a
            y = baoa + t * bard
            ok = (h >= 0) & (np.abs(a) > 1e-12) & (t > 1e-6) & (y > 0) & (y < baba)
            tc = np.where(ok, t, np.inf)
            for cen in (A[i], B[i]):  # end caps
                oc = o - cen
                bq = np.sum(oc * d, -1)
                cq = np.sum(oc * oc, -1) - R[i] * R[i]
                h2 = bq * bq - cq
                ts = -bq - np.sqrt(np.maximum(h2, 0.0))
                tc = np.where((h2 >= 0) & (ts > 1e-6) & (ts < tc), ts, tc)
            better = tc < t_h
            t_h = np.where(better, tc, t_h)
            hit_cap = np.where(better, i, hit_cap)
        Rb, tb = self.object_pose(fid)
        ol = (o - tb) @ Rb
        dl = d @ Rb
        with np.errstate(divide="ignore", invalid="ignore"):
            t1 = (-self.box_half - ol) / dl
            t2 = (self.box_half - ol) / dl
        te = np.minimum(t1, t2).max(-1)
        tx = np.maximum(t1, t2).min(-1)
        t_o = np.where((tx >= te) & (te > 1e-6), te, np.inf)
        rgb = np.zeros((n, 3))
        hum = np.isfinite(t_h) & (t_h <= t_o)
        obj = np.isfinite(t_o) & (t_o < t_h)
        rgb[hum] = self.palette[drv[hit_cap[hum]]]
        if obj.any():
            p = ol[obj] + te[obj, None] * dl[obj]
            rgb[obj] = np.clip(0.52 + 0.42 * np.sin(18.0 * p), 0.0, 1.0)
        return t_h, t_o, rgb, hum, obj

    def object_pose(self, fid: int):
        """World pose (R, t) of the box at frame fid (synthetic.py:37-45)."""
        u = self._u(fid)
        orbit = _rotmats(np.array([0.0, np.deg2rad(self.cfg.object_orbit_degrees) * u, 0.0]))
        spin = _rotmats(np.array([0.0, np.deg2rad(self.cfg.object_spin_degrees) * u, 0.0]))
        base = _rotmats(np.array([0.42, 0.55, 0.12]))
        c0, oc = np.array([0.62, 0.95, 0.15]), np.array([0.0, 0.95, 0.0])
        return spin @ base, oc + orbit @ (c0 - oc)
