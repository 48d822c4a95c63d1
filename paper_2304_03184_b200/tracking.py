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
    P = _dev(np.atleast_2d(pts))
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
        as_t = lambda a, dt: torch.as_tensor(np.asarray(a), dtype=dt).to(d)  # noqa: E731
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
        order = torch.argsort(self.col.to(torch.int64) * max(self.rows, 1) + row, stable=True)
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
           "depth_normals", "find_correspondences", "rigid_icp", "InsufficientOverlapError", "lbs_theta_jacobian"]
