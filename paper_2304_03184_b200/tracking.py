"""Non-rigid tracking on the GPU — drop-ins for capfields.tracking's data association
(depth_normals, find_correspondences; tracking.py:60-150) and the inner solver of its
Levenberg-Marquardt loop (pcg_solve, tracking.py:158-193).

SURVEY §8(f) 4. The Jacobi-preconditioned CG on (J^T J + lambda diag(J^T J)) x =
-J^T r runs as one cooperative kernel (csrc/pcg.cu, `cf_pcg_solve`): both sparse
products, the dot products and the stopping tests happen on the device between
grid-wide barriers. `GaussNewtonSystem` uploads J once and builds J^T on the device,
so the LM loop's retries at growing damping (tracking.py:523-536) reuse it.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import InsufficientOverlapError

PCG_ITERS = 32    # tracking.py:24-29
PCG_TOL = 1e-6
FD_STEP = 1e-6
CORR_DIST = 0.03
CORR_NORMAL_DEG = 60.0


def _cam_parts(cam):
    from .tsdf import _cam_pose, _inverse, _pinhole, _rigid
    Rc, tc = _cam_pose(cam)
    Rwc, twc = _inverse(Rc, tc)
    return _pinhole(cam), _rigid(Rc, tc), _rigid(Rwc, twc)


def _dev(a, dtype=torch.float64):
    d = _lib.require_cuda()
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(np.asarray(a)))
    return t.to(d, dtype).contiguous()


def depth_normals(depth, cam, as_tensor: bool = False):
    """World-space, camera-facing normals of a depth map (tracking.py:60-80); zero
    vectors mark invalid pixels."""
    D = _dev(depth)
    H, W = int(D.shape[0]), int(D.shape[1])
    pin, pose, _ = _cam_parts(cam)
    out = torch.empty((H, W, 3), dtype=torch.float64, device=D.device)
    _lib.call("cf_depth_normals", D.data_ptr(), H, W, _lib.byref(pin), _lib.byref(pose), out.data_ptr(),
              _lib.stream_ptr())
    return out if as_tensor else out.cpu().numpy()


def find_correspondences(model_points, model_normals, depth, cam, mask=None, tau: float = CORR_DIST,
                         normal_deg: float = CORR_NORMAL_DEG, normals_map=None):
    """Projective association -> (model indices, targets, depth normals) (tracking.py:83-150)."""
    on_dev = isinstance(model_points, torch.Tensor) and model_points.is_cuda
    P = _dev(np.atleast_2d(model_points) if not on_dev else model_points)
    N = _dev(model_normals)
    D = _dev(depth)
    H, W = int(D.shape[0]), int(D.shape[1])
    M = None if mask is None else _dev(np.asarray(mask.cpu() if isinstance(mask, torch.Tensor) else mask) > 0,
                                       torch.uint8)
    nm = depth_normals(D, cam, as_tensor=True) if normals_map is None else _dev(normals_map)
    pin, pose, w2c = _cam_parts(cam)
    n = int(P.shape[0])
    tgt = torch.empty((n, 3), dtype=torch.float64, device=D.device)
    nu = torch.empty((n, 3), dtype=torch.float64, device=D.device)
    keep = torch.empty(n, dtype=torch.uint8, device=D.device)
    _lib.call("cf_find_correspondences", P.data_ptr(), N.data_ptr(), n, D.data_ptr(), H, W,
              None if M is None else M.data_ptr(), nm.data_ptr(), _lib.byref(pin), _lib.byref(pose),
              _lib.byref(w2c), float(tau), float(np.cos(np.deg2rad(normal_deg))), tgt.data_ptr(), nu.data_ptr(),
              keep.data_ptr(), _lib.stream_ptr())
    k = keep.bool()
    idx = torch.nonzero(k).reshape(-1)
    out = (idx, tgt[k], nu[k])
    return out if on_dev else tuple(t.cpu().numpy() for t in out)


def _rotmat(rv) -> np.ndarray:
    """rotmat_from_rotvec (transforms.py:66-111), numpy's operation order."""
    rv = np.asarray(rv, dtype=np.float64)
    ang = np.linalg.norm(rv, axis=-1, keepdims=True)
    half = 0.5 * ang
    small = ang < 1e-12
    with np.errstate(invalid="ignore", divide="ignore"):
        k = np.where(small, 0.5 - ang * ang / 48.0, np.sin(half) / np.where(small, 1.0, ang))
    w, (x, y, z) = np.cos(half)[0], k * rv
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


class _Pose:
    """Rigid transform with the reference Se3's rotation / translation attributes."""

    def __init__(self, R, t):
        self.rotation = np.asarray(R, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(t, dtype=np.float64).reshape(3)


def rigid_icp(volume_or_model, depth, cam, mask, init, max_iters: int = 15, tau: float = 0.05,
              min_pixels: int = 30, normal_deg: float = 30.0):
    """Projective point-to-plane ICP refining init (canonical -> world), tracking.py:560-620.

    Per iteration on the device: model transform, association, residuals and the
    Huber-weighted 6x6 normal equations; the host solves the 6x6 system (with the
    reference's Tikhonov damping and trust region) and composes the pose."""
    from .tsdf import TsdfVolume, _rigid
    D = _dev(depth)
    M = None if mask is None else _dev(np.asarray(mask.cpu() if isinstance(mask, torch.Tensor) else mask) > 0,
                                       torch.uint8)
    valid = (D > 0) if M is None else ((D > 0) & (M > 0))
    n_valid = int(valid.sum())
    if n_valid < min_pixels:
        raise InsufficientOverlapError(f"only {n_valid} valid depth pixels")
    if isinstance(volume_or_model, TsdfVolume):
        mp, mn = volume_or_model.extract_surface()
        if len(mp) < min_pixels:
            raise InsufficientOverlapError("TSDF surface is empty")
    else:
        mp, mn = volume_or_model
    P, N = _dev(mp), _dev(mn)
    n = int(P.shape[0])
    H, W = int(D.shape[0]), int(D.shape[1])
    nmap = depth_normals(D, cam, as_tensor=True)
    pin, cpose, w2c = _cam_parts(cam)
    live = torch.empty_like(P)
    ln = torch.empty_like(N)
    tgt = torch.empty_like(P)
    nu = torch.empty_like(P)
    keep = torch.empty(n, dtype=torch.uint8, device=D.device)
    r = torch.empty(n, dtype=torch.float64, device=D.device)
    sums = torch.empty(27, dtype=torch.float64, device=D.device)
    cos_max = float(np.cos(np.deg2rad(normal_deg)))
    R = np.asarray(init.rotation, dtype=np.float64).copy()
    t = np.asarray(init.translation, dtype=np.float64).copy()
    s = _lib.stream_ptr()
    iu = np.triu_indices(6)
    for _ in range(max_iters):
        _lib.call("cf_rigid_transform", P.data_ptr(), N.data_ptr(), n, _lib.byref(_rigid(R, t)), live.data_ptr(),
                  ln.data_ptr(), s)
        _lib.call("cf_find_correspondences", live.data_ptr(), ln.data_ptr(), n, D.data_ptr(), H, W,
                  None if M is None else M.data_ptr(), nmap.data_ptr(), _lib.byref(pin), _lib.byref(cpose),
                  _lib.byref(w2c), float(tau), cos_max, tgt.data_ptr(), nu.data_ptr(), keep.data_ptr(), s)
        _lib.call("cf_icp_residuals", live.data_ptr(), keep.data_ptr(), tgt.data_ptr(), nu.data_ptr(), n,
                  r.data_ptr(), s)
        k = keep.bool()
        ar = r[k].abs()
        C = int(ar.numel())
        if C < min_pixels:
            raise InsufficientOverlapError(f"only {C} ICP correspondences")
        sa = torch.sort(ar).values  # np.median: the middle value, or the mean of the two middle ones
        med = float(sa[C // 2]) if C % 2 else float((sa[C // 2 - 1] + sa[C // 2]) / 2.0)
        knee = max(3.0 * med, 1e-5)
        _lib.call("cf_icp_normal_equations", live.data_ptr(), keep.data_ptr(), nu.data_ptr(), r.data_ptr(), n,
                  knee, sums.data_ptr(), s)
        h = sums.cpu().numpy()
        A = np.zeros((6, 6))
        A[iu] = h[:21]
        A = A + np.triu(A, 1).T
        A += (1e-6 * np.trace(A) / 6.0 + 1e-12) * np.eye(6)
        delta = np.linalg.solve(A, -h[21:])
        rot_n = np.linalg.norm(delta[:3])
        tr_n = np.linalg.norm(delta[3:])
        delta *= min(1.0, 0.2 / max(rot_n, 1e-12), 0.05 / max(tr_n, 1e-12))
        Ru = _rotmat(delta[:3])
        R, t = Ru @ R, Ru @ t + delta[3:]  # Se3.compose (transforms.py:289-290)
        if np.max(np.abs(delta)) < 1e-12:
            break
    return _Pose(R, t)


def lbs_theta_jacobian(skel, theta, pts, weights, as_tensor: bool = False):
    """Central finite differences of lbs_batch w.r.t. theta -> (P, 3, T)
    (_lbs_theta_jacobian, tracking.py:244-256): the 2T perturbed poses' forward
    kinematics in one device launch (records.skinning_transforms), then one thread
    per (point, pose component)."""
    from .records import skinning_transforms
    theta = np.asarray(theta, dtype=np.float64).reshape(-1)
    T = len(theta)
    th = np.repeat(theta[None], 2 * T, axis=0)
    for k in range(T):  # the reference's theta + e and theta - e (tracking.py:250-254)
        e = np.zeros(T)
        e[k] = FD_STEP
        th[2 * k] = theta + e
        th[2 * k + 1] = theta - e
    d = _lib.require_cuda()
    A = skinning_transforms(torch.from_numpy(th).to(d), skel)
    P = pts.to(d, torch.float64).contiguous() if isinstance(pts, torch.Tensor) else _dev(np.atleast_2d(pts))
    Wt = _dev(weights)
    n = int(P.shape[0])
    J = int(A.shape[1])
    out = torch.empty((n, 3, T), dtype=torch.float64, device=d)
    _lib.call("cf_lbs_theta_jacobian", A.data_ptr(), T, J, P.data_ptr(), Wt.data_ptr(), n, FD_STEP, out.data_ptr(),
              _lib.stream_ptr())
    return out if as_tensor else out.cpu().numpy()


def _csr_parts(J):
    """(val, col, rowptr, rows, cols) from a scipy.sparse matrix or a tuple."""
    if hasattr(J, "tocsr"):
        J = J.tocsr()
        return J.data, J.indices, J.indptr, J.shape[0], J.shape[1]
    val, col, rowptr, shape = J
    return val, col, rowptr, int(shape[0]), int(shape[1])


class GaussNewtonSystem:
    """A Jacobian J (rows x cols, CSR) and residual r resident in HBM, with J^T."""

    def __init__(self, J, r):
        d = _lib.require_cuda()
        val, col, rowptr, rows, cols = _csr_parts(J)
        self.rows, self.cols = int(rows), int(cols)
        as_t = lambda a, dt: (a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))).to(d, dt)  # noqa: E731
        self.val = as_t(val, torch.float64).contiguous()
        self.col = as_t(col, torch.int32).contiguous()
        self.rowptr = as_t(rowptr, torch.int32).contiguous()
        r = torch.as_tensor(np.asarray(r, dtype=np.float64) if not isinstance(r, torch.Tensor) else r)
        self.r = r.to(d, torch.float64).contiguous()
        if self.r.numel() != self.rows or self.rowptr.numel() != self.rows + 1:
            raise ValueError("residual / row pointer length does not match the Jacobian")
        # J^T on the device: stable sort of the entries by (column, row)
        nnz = self.val.numel()
        row = torch.repeat_interleave(torch.arange(self.rows, device=d, dtype=torch.int64),
                                      (self.rowptr[1:] - self.rowptr[:-1]).to(torch.int64))
        # (column, row) keys are unique, so any sort is the stable one; 32-bit keys when
        # they fit (a 64-bit radix sort costs ~5 ms per system here)
        key = self.col.to(torch.int64) * max(self.rows, 1) + row
        if self.cols * max(self.rows, 1) < 2 ** 31:
            key = key.to(torch.int32)
        order = torch.sort(key).indices
        self.tval = self.val[order].contiguous()
        self.tcol = row[order].to(torch.int32).contiguous()
        counts = torch.bincount(self.col.to(torch.int64), minlength=self.cols)
        self.trowptr = torch.cat([torch.zeros(1, dtype=torch.int64, device=d), torch.cumsum(counts, 0)]).to(
            torch.int32).contiguous()
        self.J = self._desc(self.val, self.col, self.rowptr, self.rows, self.cols, nnz)
        self.JT = self._desc(self.tval, self.tcol, self.trowptr, self.cols, self.rows, nnz)
        nd = ctypes.c_int64()
        _lib.call("cf_pcg_workspace_doubles", self.rows, self.cols, ctypes.byref(nd))
        self.work = torch.empty(int(nd.value), dtype=torch.float64, device=d)
        self.iters = torch.zeros(1, dtype=torch.int32, device=d)

    @staticmethod
    def _desc(val, col, rowptr, rows, cols, nnz) -> _lib.Csr:
        c = _lib.Csr()
        c.val, c.col, c.rowptr = val.data_ptr(), col.data_ptr(), rowptr.data_ptr()
        c.rows, c.cols, c.nnz = rows, cols, nnz
        return c

    def solve(self, lm_lambda: float, max_iters: int = PCG_ITERS, tol: float = PCG_TOL) -> torch.Tensor:
        """x (cols,) on the device; `last_iters` holds the iteration count (device)."""
        x = torch.empty(self.cols, dtype=torch.float64, device=self.val.device)
        _lib.call("cf_pcg_solve", _lib.byref(self.J), _lib.byref(self.JT), self.r.data_ptr(), float(lm_lambda),
                  int(max_iters), float(tol), x.data_ptr(), self.work.data_ptr(), self.iters.data_ptr(),
                  _lib.stream_ptr())
        return x


def pcg_solve(J, r, lm_lambda: float, max_iters: int = PCG_ITERS, tol: float = PCG_TOL) -> np.ndarray:
    """Solve (J^T J + lm_lambda diag(J^T J)) x = -J^T r by Jacobi-PCG (tracking.py:158-193)."""
    return GaussNewtonSystem(J, r).solve(lm_lambda, max_iters, tol).cpu().numpy()


__all__ = ["PCG_ITERS", "PCG_TOL", "CORR_DIST", "CORR_NORMAL_DEG", "GaussNewtonSystem", "pcg_solve",
           "depth_normals", "find_correspondences", "rigid_icp", "InsufficientOverlapError", "lbs_theta_jacobian",
           "NonrigidTracker", "SolveState", "EnergyWeights"]


# ---------------------------------------------------------------------------
# non-rigid tracker (tracking.py:196-556) with every per-iteration stage on the device
# ---------------------------------------------------------------------------

LM_LAMBDA_INIT = 1e-3   # tracking.py:26-27
LM_LAMBDA_CAP = 1e6
EDGE_K = 8


class EnergyWeights:
    """tracking.py:37-49."""

    def __init__(self, data=1.0, bind=1.0, reg=4.0, prior=0.01, pose=0.02, inter=1.0):
        self.data, self.bind, self.reg, self.prior, self.pose, self.inter = data, bind, reg, prior, pose, inter
        for name in ("data", "bind", "reg", "prior", "pose", "inter"):
            if getattr(self, name) < 0:
                raise ValueError(f"energy weight {name} must be nonnegative")


class SolveState:
    """Node dual quaternions (n, 8) on the device and the pose theta (T,) on the host."""

    def __init__(self, dqs, theta):
        self.dqs_dev = _dev(dqs)
        self.theta = np.asarray(theta, dtype=np.float64).copy()

    @property
    def dqs(self) -> np.ndarray:
        return self.dqs_dev.cpu().numpy()

    def copy(self) -> "SolveState":
        return SolveState(self.dqs_dev.clone(), self.theta.copy())


class NonrigidTracker:
    """GPU drop-in for capfields.tracking.NonrigidTracker (tracking.py:259-556): the same
    constructor and solve(); `model` is duck-typed (graph.nodes / radius / knn_k,
    skeleton.parents / offsets / joint_limits, points, normals, lbs_weights,
    node_lbs_weights, edges); object_volume is this package's TsdfVolume."""

    def __init__(self, model, cam, weights=None, surface_samples: int = 4096, max_iters: int = 8,
                 object_volume=None, seed: int = 0):
        self.object_volume = object_volume  # a tsdf.TsdfVolume (device) or None
        self.object_pose = _Pose(np.eye(3), np.zeros(3))  # canonical -> world, set by the object tracker
        from .knnfield import brute_force_neighbors_batch
        self.model, self.cam = model, cam
        self.weights = weights or EnergyWeights()
        self.max_iters = max_iters
        rng = np.random.default_rng(seed)
        pts, nrm = np.asarray(model.points, dtype=np.float64), np.asarray(model.normals, dtype=np.float64)
        take = min(surface_samples, len(pts))
        sel = rng.choice(len(pts), size=take, replace=False)  # tracking.py:286-291
        self.sub_pts, self.sub_normals = pts[sel], nrm[sel]
        self.sub_lbs = np.asarray(model.lbs_weights, dtype=np.float64)[sel]
        g = model.graph
        self.nodes = np.asarray(g.nodes, dtype=np.float64)
        k = int(min(g.knn_k, len(self.nodes)))
        idx = brute_force_neighbors_batch(g, self.sub_pts, k)  # exact, ties by index (edgraph.py:121-131)
        d2 = np.sum((self.sub_pts[:, None, :] - self.nodes[idx]) ** 2, axis=-1)
        w = np.exp(-d2 / (g.radius * g.radius))  # canonical_blend_info (edgraph.py:186-195)
        wn = w / np.maximum(w.sum(axis=1, keepdims=True), 1e-300)
        self.k = k
        self.d_idx, self.d_w, self.d_wn = _dev(idx, torch.int32), _dev(w), _dev(wn)
        self.d_pts, self.d_nrm = _dev(self.sub_pts), _dev(self.sub_normals)
        self.d_lbs = _dev(self.sub_lbs)
        self.d_nodes = _dev(self.nodes)
        self.node_w = np.asarray(model.node_lbs_weights, dtype=np.float64)
        self.d_node_w = _dev(self.node_w)
        e = model.edges if getattr(model, "edges", None) is not None else g.edges(EDGE_K)
        self.edges = np.asarray(e, dtype=np.int64).reshape(-1, 2)
        self.d_edges = _dev(self.edges, torch.int64)
        self.skel = model.skeleton
        self.lim = np.repeat(np.asarray(model.skeleton.joint_limits, dtype=np.float64), 3)
        self.dom = _dev(np.argmax(self.sub_lbs, axis=1), torch.int64)
        n = len(self.nodes)
        dq = np.zeros((n, 8))
        dq[:, 0] = 1.0
        self.state = SolveState(dq, np.zeros(3 * len(np.asarray(model.skeleton.parents))))
        self._e = torch.zeros(4, dtype=torch.float64, device=self.d_nodes.device)

    # -- per-state quantities ----------------------------------------------------

    def _bones(self, theta):
        from .records import skinning_transforms
        return skinning_transforms(torch.from_numpy(np.asarray(theta, dtype=np.float64)[None]).to(
            self.d_nodes.device), self.skel)[0].contiguous()

    def _lbs(self, A, pts, w):
        out = torch.empty_like(pts)
        _lib.call("cf_lbs_forward", A.data_ptr(), int(A.shape[0]), pts.data_ptr(), w.data_ptr(), int(pts.shape[0]),
                  out.data_ptr(), _lib.stream_ptr())
        return out

    def warp_subset(self, state):
        out_p, out_n = torch.empty_like(self.d_pts), torch.empty_like(self.d_nrm)
        _lib.call("cf_nr_warp", state.dqs_dev.data_ptr(), self.d_idx.data_ptr(), self.d_w.data_ptr(), self.k,
                  self.d_pts.data_ptr(), self.d_nrm.data_ptr(), int(self.d_pts.shape[0]), out_p.data_ptr(),
                  out_n.data_ptr(), _lib.stream_ptr())
        return out_p, out_n

    def _associate(self, state, D, mask, nmap):
        warped, wn = self.warp_subset(state)
        data_corr = find_correspondences(warped, wn, D, self.cam, mask=mask, normals_map=nmap)
        A = self._bones(state.theta)
        lp = self._lbs(A, self.d_pts, self.d_lbs)
        ln = torch.einsum("nab,nb->na", A[self.dom][:, :3, :3], self.d_nrm).contiguous()
        pose_corr = find_correspondences(lp, ln, D, self.cam, mask=mask, normals_map=nmap)
        return data_corr, pose_corr

    def _inter(self, state):
        """Interpenetration term (tracking.py:326-331, 481-496): penetration depth of the
        live nodes inside the object volume -> (pen (n,), active ids, live nodes, m)."""
        from .tsdf import _inverse
        n = len(self.nodes)
        live = torch.empty_like(self.d_nodes)
        _lib.call("cf_deform_nodes", self.d_nodes.data_ptr(), state.dqs_dev.data_ptr(), n, live.data_ptr(),
                  _lib.stream_ptr())
        R, t = _inverse(np.asarray(self.object_pose.rotation), np.asarray(self.object_pose.translation))
        Rt = torch.from_numpy(np.ascontiguousarray(R)).to(live.device)
        q = (live @ Rt.t() + torch.from_numpy(t).to(live.device)).contiguous()  # inv.apply (Se3.apply)
        phi, ok = self.object_volume.sample(q)
        pen = torch.where(ok, torch.clamp(-phi, min=0.0), torch.zeros_like(phi))
        return pen, q, live, Rt

    def _system(self, state, data_corr, pose_corr, with_jacobian: bool):
        """energy_terms (tracking.py:288-336) and, with_jacobian, _assemble (358-508)."""
        w = self.weights
        n, T = len(self.nodes), len(state.theta)
        A = self._bones(state.theta)
        warped, _ = self.warp_subset(state)
        conv = lambda c: (_dev(np.asarray(c[0]).reshape(-1), torch.int64) if not isinstance(c[0], torch.Tensor)  # noqa: E731
                          else c[0], _dev(np.asarray(c[1]).reshape(-1, 3)) if not isinstance(c[1], torch.Tensor)
                          else c[1], _dev(np.asarray(c[2]).reshape(-1, 3)) if not isinstance(c[2], torch.Tensor)
                          else c[2])
        ci, cu, cn = conv(data_corr)
        pi, pu, pn = conv(pose_corr)
        node_lbs = self._lbs(A, self.d_nodes, self.d_node_w)
        P = int(pi.numel())
        pose_lbs = self._lbs(A, self.d_pts[pi].contiguous(), self.d_lbs[pi].contiguous()) if P else None
        lim_r = np.maximum(0.0, np.abs(state.theta) - self.lim)
        act = np.nonzero(lim_r > 0)[0]
        C, E = int(ci.numel()), len(self.edges)
        use = dict(data=C > 0 and w.data > 0, bind=w.bind > 0, reg=E > 0 and w.reg > 0, prior=w.prior > 0 and len(act),
                   pose=P > 0 and w.pose > 0)
        inter = None
        if self.object_volume is not None:
            pen, q, live, Rt = self._inter(state)
            self._inter_e = float((pen * pen).sum())
            iact = torch.nonzero(pen > 0).reshape(-1)
            use["inter"] = w.inter > 0 and int(iact.numel()) > 0
            inter = (pen, q, live, Rt, iact)
        else:
            self._inter_e = 0.0
            use["inter"] = False
        S = _lib.NrSystem()
        S.dqs, S.nodes, S.n_nodes, S.n_theta = state.dqs_dev.data_ptr(), self.d_nodes.data_ptr(), n, T
        S.warped, S.n_data = warped.data_ptr(), C
        if C:
            S.data_idx, S.data_u, S.data_n = ci.data_ptr(), cu.data_ptr(), cn.data_ptr()
        S.blend_idx, S.blend_wn, S.k, S.w_data = self.d_idx.data_ptr(), self.d_wn.data_ptr(), self.k, w.data
        S.do_bind, S.node_lbs, S.s_bind = 1, node_lbs.data_ptr(), float(np.sqrt(w.bind))
        S.edges, S.n_edges, S.s_reg = self.d_edges.data_ptr(), E, float(np.sqrt(w.reg))
        S.n_pose, S.w_pose = P, w.pose
        if P:
            S.pose_lbs, S.pose_u, S.pose_n = pose_lbs.data_ptr(), pu.data_ptr(), pn.data_ptr()
        S.energy = self._e.data_ptr()
        J = r = None
        if with_jacobian:
            sizes = [("data", C if use["data"] else 0, 6 * self.k), ("bind", 3 * n if use["bind"] else 0, 6 + T),
                     ("reg", 3 * E if use["reg"] else 0, 12), ("prior", len(act) if use["prior"] else 0, 1),
                     ("pose", P if use["pose"] else 0, T),
                     ("inter", int(inter[4].numel()) if use["inter"] else 0, 6)]
            rows = sum(s[1] for s in sizes)
            if rows == 0:
                _lib.call("cf_nr_terms", _lib.byref(S), _lib.stream_ptr())
                return self._energy(state, lim_r), None, None
            nnz = sum(s[1] * s[2] for s in sizes)
            d = self.d_nodes.device
            val = torch.zeros(nnz, dtype=torch.float64, device=d)
            col = torch.zeros(nnz, dtype=torch.int32, device=d)
            res = torch.zeros(rows, dtype=torch.float64, device=d)
            row0, ent0, off = 0, 0, {}
            for name, nr, per in sizes:
                off[name] = (row0, ent0)
                row0 += nr
                ent0 += nr * per
            S.val, S.col, S.res = val.data_ptr(), col.data_ptr(), res.data_ptr()
            S.data_row0, S.data_entry0 = off["data"]
            S.bind_row0, S.bind_entry0 = off["bind"]
            S.reg_row0, S.reg_entry0 = off["reg"]
            S.pose_row0, S.pose_entry0 = off["pose"]
            # every energy is evaluated; only the used terms write Jacobian rows
            S.jac_terms = (int(bool(use["data"])) | int(bool(use["bind"])) << 1 | int(bool(use["reg"])) << 2
                           | int(bool(use["pose"])) << 3)
            if use["bind"]:
                jn = lbs_theta_jacobian(self.skel, state.theta, self.d_nodes, self.d_node_w, as_tensor=True)
                S.node_jth = jn.data_ptr()
            if use["pose"]:
                jp = lbs_theta_jacobian(self.skel, state.theta, self.d_pts[pi].contiguous(),
                                        self.d_lbs[pi].contiguous(), as_tensor=True)
                S.pose_jth = jp.data_ptr()
            _lib.call("cf_nr_terms", _lib.byref(S), _lib.stream_ptr())
            if use["prior"]:  # quadratic joint-limit rows (tracking.py:445-456)
                s = np.sqrt(w.prior)
                r0, e0 = off["prior"]
                val[e0:e0 + len(act)] = torch.from_numpy(s * np.sign(state.theta[act])).to(d)
                col[e0:e0 + len(act)] = torch.from_numpy((6 * n + act).astype(np.int32)).to(d)
                res[r0:r0 + len(act)] = torch.from_numpy(s * lim_r[act]).to(d)
            if use["inter"]:  # rows s [v x m, m], m = -(grad_q R_inv) (tracking.py:481-496)
                pen, q, live, Rt, iact = inter
                si = float(np.sqrt(w.inter))
                g = self.object_volume.gradient(q[iact].contiguous())
                m = -(g @ Rt)
                gom = torch.linalg.cross(live[iact], m)
                r0, e0 = off["inter"]
                ni = int(iact.numel())
                val[e0:e0 + 6 * ni] = (si * torch.cat([gom, m], 1)).reshape(-1)
                col[e0:e0 + 6 * ni] = (6 * iact[:, None] + torch.arange(6, device=d)[None]).reshape(-1).to(torch.int32)
                res[r0:r0 + ni] = si * pen[iact]
            counts = torch.cat([torch.full((nr,), per, dtype=torch.int64, device=d) for _, nr, per in sizes if nr])
            rowptr = torch.cat([torch.zeros(1, dtype=torch.int64, device=d), torch.cumsum(counts, 0)]).to(torch.int32)
            J = (val, col, rowptr, (rows, 6 * n + T))
            r = res
        else:
            _lib.call("cf_nr_terms", _lib.byref(S), _lib.stream_ptr())
        return self._energy(state, lim_r), J, r

    def _energy(self, state, lim_r=None):
        w = self.weights
        e = self._e.cpu().numpy()
        if lim_r is None:
            lim_r = np.maximum(0.0, np.abs(state.theta) - self.lim)
        out = {"data": float(e[0]), "bind": float(e[1]), "reg": float(e[2]), "prior": float(np.sum(lim_r ** 2)),
               "pose": float(e[3]), "inter": float(getattr(self, "_inter_e", 0.0))}
        out["total"] = (w.data * out["data"] + w.bind * out["bind"] + w.reg * out["reg"] + w.prior * out["prior"]
                        + w.pose * out["pose"] + w.inter * out["inter"])
        return out

    def energy_terms(self, state, data_corr, pose_corr) -> dict:
        return self._system(state, data_corr, pose_corr, False)[0]

    def _apply_step(self, state, delta):
        n = len(self.nodes)
        out = torch.empty_like(state.dqs_dev)
        _lib.call("cf_nr_step", state.dqs_dev.data_ptr(), delta.data_ptr(), n, out.data_ptr(), _lib.stream_ptr())
        return SolveState(out, state.theta + delta[6 * n:].cpu().numpy())

    def solve(self, depth, mask, frame_id: int, init=None):
        """LM outer loop with correspondences refreshed every iteration (tracking.py:510-544)."""
        state = (init or self.state).copy()
        if not isinstance(state, SolveState):
            state = SolveState(state.dqs, state.theta)
        lm = LM_LAMBDA_INIT
        D = _dev(depth)
        M = None if mask is None else _dev(np.asarray(mask.cpu() if isinstance(mask, torch.Tensor) else mask) > 0,
                                           torch.uint8)
        nmap = depth_normals(D, self.cam, as_tensor=True)
        info = {"accepted": [], "warning": False, "iterations": 0, "energies": []}
        best = state
        delta = None
        for it in range(self.max_iters):
            data_corr, pose_corr = self._associate(state, D, M, nmap)
            e0, J, r = self._system(state, data_corr, pose_corr, True)
            info["energies"].append(e0)
            if J is None:
                break
            sysm = GaussNewtonSystem(J, r)
            stepped = False
            while lm <= LM_LAMBDA_CAP:
                delta = sysm.solve(lm)
                cand = self._apply_step(state, delta)
                e1 = self.energy_terms(cand, data_corr, pose_corr)
                if e1["total"] <= e0["total"] + 1e-15:
                    info["accepted"].append((e0["total"], e1["total"]))
                    state = cand
                    best = cand
                    lm = max(lm * 0.5, 1e-9)
                    stepped = True
                    break
                lm *= 10.0
            info["iterations"] = it + 1
            if not stepped:
                info["warning"] = True
                break
            if float(delta.abs().max()) < 1e-10:
                break
        self.state = best
        return best, info
