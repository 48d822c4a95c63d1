"""Rigid-object TSDF volume on the GPU — drop-in for capfields.tsdf (tsdf.py:17-176).

SURVEY §8(f) 4, the tracking front-end's volumetric model: integration, trilinear
sampling, gradients, zero-crossing surface extraction and ray casting run in
csrc/tsdf.cu (`cf_tsdf_*`), one thread per voxel / point / pixel, float64 in the
reference's operation order. The volume lives in HBM; `tsdf` / `weight` read back
host copies, as the reference's numpy attributes.

Cameras and poses are duck-typed: a reference `Camera` (fx, fy, cx, cy, width,
height, pose: Se3 camera-to-world) or this package's `PinholeCamera` (R, t); poses
with `rotation` / `translation` (Se3) or `R` / `t`.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import dev, host, is_device

MAX_WEIGHT = 64.0


def _rt(pose):
    if pose is None:
        return np.eye(3), np.zeros(3)
    if hasattr(pose, "rotation"):
        return np.asarray(pose.rotation, dtype=np.float64), np.asarray(pose.translation, dtype=np.float64)
    return np.asarray(pose.R, dtype=np.float64), np.asarray(pose.t, dtype=np.float64)


def _cam_pose(cam):
    return _rt(cam.pose if hasattr(cam, "pose") else cam)


def _inverse(R, t):
    """Se3.inverse (transforms.py:293-295), the same numpy expression."""
    rt = R.T
    return rt, -rt @ t


def _rigid(R, t) -> _lib.Rigid:
    T = _lib.Rigid()
    Rf = np.asarray(R, dtype=np.float64).reshape(-1)
    for i in range(9):
        T.R[i] = float(Rf[i])
    for i in range(3):
        T.t[i] = float(t[i])
    return T


def _pinhole(cam) -> _lib.Pinhole:
    c = _lib.Pinhole()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


class TsdfVolume:
    """Truncated signed distance volume anchored in the object's canonical frame."""

    def __init__(self, resolution: int, voxel_size: float, origin, truncation: float | None = None):
        self.resolution = int(resolution)
        if self.resolution < 2:
            raise ValueError("resolution must be at least 2")
        self.voxel_size = float(voxel_size)
        self.origin = np.asarray(origin, dtype=np.float64).reshape(3)
        self.truncation = float(truncation if truncation is not None else 4.0 * voxel_size)
        d = _lib.require_cuda()
        r = self.resolution
        self.tsdf_dev = torch.ones((r, r, r), dtype=torch.float64, device=d)
        self.weight_dev = torch.zeros((r, r, r), dtype=torch.float64, device=d)

    # -- reference attributes ---------------------------------------------------

    @property
    def tsdf(self) -> np.ndarray:
        return host(self.tsdf_dev)

    @property
    def weight(self) -> np.ndarray:
        return host(self.weight_dev)

    def _desc(self) -> _lib.TsdfDesc:
        V = _lib.TsdfDesc()
        V.tsdf, V.weight = self.tsdf_dev.data_ptr(), self.weight_dev.data_ptr()
        V.resolution, V.voxel, V.trunc = self.resolution, self.voxel_size, self.truncation
        for a in range(3):
            V.origin[a] = float(self.origin[a])
        return V

    def voxel_centers(self) -> np.ndarray:
        """(r, r, r, 3) centres origin + (ijk + 0.5) voxel (tsdf.py:24-30)."""
        r = self.resolution
        ax = torch.arange(r, dtype=torch.float64, device=self.tsdf_dev.device)
        g = torch.stack(torch.meshgrid(ax, ax, ax, indexing="ij"), dim=-1)
        o = torch.as_tensor(self.origin, device=g.device)
        return host(o + (g + 0.5) * self.voxel_size)

    # -- operations -------------------------------------------------------------

    def integrate(self, depth, cam, pose, mask=None) -> None:
        """Weighted-average TSDF update from one depth map (tsdf.py:33-61); pose maps
        volume coordinates to world."""
        D = dev(depth)
        if D.dim() != 2:
            raise ValueError("depth must be (H, W)")
        H, W = int(D.shape[0]), int(D.shape[1])
        M = None
        if mask is not None:
            M = dev(np.asarray(host(mask) if is_device(mask) else mask) > 0, dtype=torch.uint8)
            if tuple(M.shape) != (H, W):
                raise ValueError("mask must match the depth map")
        Rv, tv = _rt(pose)
        Rc, tc = _cam_pose(cam)
        Rwc, twc = _inverse(Rc, tc)
        V = self._desc()
        _lib.call("cf_tsdf_integrate", _lib.byref(V), D.data_ptr(), H, W, None if M is None else M.data_ptr(),
                  _lib.byref(_rigid(Rv, tv)), _lib.byref(_rigid(Rwc, twc)), _lib.byref(_pinhole(cam)),
                  _lib.stream_ptr())

    def _query(self, pts, want_val=True, want_grad=False):
        on_dev = is_device(pts)
        P = dev(pts if on_dev else np.atleast_2d(np.asarray(pts, dtype=np.float64)), shape_last=3)
        n = int(P.shape[0])
        val = torch.empty(n, dtype=torch.float64, device=P.device) if want_val else None
        ok = torch.empty(n, dtype=torch.uint8, device=P.device) if want_val else None
        g = torch.empty((n, 3), dtype=torch.float64, device=P.device) if want_grad else None
        V = self._desc()
        _lib.call("cf_tsdf_sample", _lib.byref(V), P.data_ptr(), n, _lib.ptr(val), _lib.ptr(ok), _lib.ptr(g),
                  _lib.stream_ptr())
        return on_dev, val, ok, g

    def sample(self, pts):
        """Trilinear TSDF values and validity at canonical points (tsdf.py:63-88)."""
        on_dev, val, ok, _ = self._query(pts)
        ok = ok.bool()
        return (val, ok) if on_dev else (host(val), host(ok))

    def gradient(self, pts):
        """Central-difference gradient per metre (tsdf.py:90-100)."""
        on_dev, _, _, g = self._query(pts, want_val=False, want_grad=True)
        return g if on_dev else host(g)

    def _normals(self, pts: torch.Tensor):
        g = self.gradient(pts)
        nrm = torch.sqrt((g[:, 0] * g[:, 0] + g[:, 1] * g[:, 1]) + g[:, 2] * g[:, 2])
        ok = nrm > 1e-9
        return pts[ok], g[ok] / nrm[ok][:, None]

    def extract_surface(self, step: float | None = None):
        """Zero-crossing surface points + normals via axis scans (tsdf.py:102-132)."""
        r = self.resolution
        V = self._desc()
        out = []
        for axis in range(3):
            n = (r - 1) * r * r
            P = torch.empty((n, 3), dtype=torch.float64, device=self.tsdf_dev.device)
            F = torch.empty(n, dtype=torch.uint8, device=P.device)
            _lib.call("cf_tsdf_crossings", _lib.byref(V), axis, P.data_ptr(), F.data_ptr(), _lib.stream_ptr())
            out.append(P[F.bool()])
        pts = torch.cat(out, 0)
        if pts.shape[0] == 0:
            return np.zeros((0, 3)), np.zeros((0, 3))
        p, nrm = self._normals(pts)
        return host(p), host(nrm)

    def raycast(self, cam, pose, stride: int = 1):
        """March every `stride`-th pixel's ray through the volume -> surface points and
        normals in the volume frame (tsdf.py:134-171)."""
        Rc, tc = _cam_pose(cam)
        Rv, tv = _rt(pose)
        Ri, ti = _inverse(Rv, tv)
        o = np.broadcast_to(tc, (1, 3)) @ Ri.T + ti  # inv.apply of the (shared) ray origin
        extent = self.resolution * self.voxel_size
        max_t = np.linalg.norm(self.origin + extent - o, axis=-1).max() + extent
        d = self.tsdf_dev.device
        cols = (int(cam.width) + stride - 1) // stride
        rows = (int(cam.height) + stride - 1) // stride
        n = cols * rows
        O = torch.from_numpy(np.ascontiguousarray(o[0])).to(d)
        P = torch.empty((n, 3), dtype=torch.float64, device=d)
        N = torch.empty((n, 3), dtype=torch.float64, device=d)
        H = torch.empty(n, dtype=torch.uint8, device=d)
        V = self._desc()
        _lib.call("cf_tsdf_raycast", _lib.byref(V), _lib.byref(_pinhole(cam)), _lib.byref(_rigid(Rc, np.zeros(3))),
                  _lib.byref(_rigid(Ri, np.zeros(3))), O.data_ptr(), int(stride), 1e-3, 0.5 * self.voxel_size,
                  float(max_t), P.data_ptr(), N.data_ptr(), H.data_ptr(), _lib.stream_ptr())
        hit = H.bool()
        return host(P[hit]), host(N[hit])


def tsdf_integrate(vol: TsdfVolume, depth, cam, pose, mask=None) -> TsdfVolume:
    vol.integrate(depth, cam, pose, mask=mask)
    return vol


__all__ = ["MAX_WEIGHT", "TsdfVolume", "tsdf_integrate"]
