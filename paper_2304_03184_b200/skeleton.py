"""Linear blend skinning on the GPU — drop-in for capfields.skeleton.lbs_batch,
plus the backward (live -> rest) LBS of the hybrid deformation.

Per-frame forward kinematics of the 24-joint rig is host-side setup (24 4x4
products, as in the reference skeleton.py:121-139); every per-point blend runs
in csrc/lbs.cu.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import dev, host, is_device
from .edgraph import Buckets
from . import scene as _rig


def _bone_transforms(skel, theta) -> np.ndarray:
    if skel is None or (np.array_equal(np.asarray(skel.parents), _rig.PARENTS)
                        and np.allclose(np.asarray(skel.offsets), _rig.OFFSETS, rtol=0, atol=0)):
        return _rig.skinning_transforms(np.asarray(theta, dtype=np.float64))
    raise ValueError("only the 24-joint default humanoid rig is supported")


def lbs_batch(skel, theta, points, weights):
    """Forward LBS of rest-pose points (N,3) with weights (N,J) (skeleton.py:142-149)."""
    A = dev(_bone_transforms(skel, theta))
    on_dev = is_device(points)
    p = dev(points if on_dev else np.atleast_2d(np.asarray(points, dtype=np.float64)), shape_last=3)
    W = dev(weights)
    out = torch.empty_like(p)
    _lib.call("cf_lbs_forward", A.data_ptr(), int(A.shape[0]), p.data_ptr(), W.data_ptr(), int(p.shape[0]),
              out.data_ptr(), _lib.stream_ptr())
    return out if on_dev else host(out)


class BackwardLBS:
    """Backward LBS warp: skin vertices (V,3) with weights (V,J)
    are posed per frame; a live sample takes the inverse blended transform of
    its nearest posed vertex (exact 1-NN on coarse buckets, ties by index)."""

    def __init__(self, verts_rest, vert_weights, max_dist: float = 0.2):
        self.verts = dev(verts_rest, shape_last=3)
        self.W = dev(vert_weights)
        self.V = int(self.verts.shape[0])
        self.J = int(self.W.shape[1])
        self.max_dist = float(max_dist)
        self.posed = torch.empty_like(self.verts)
        self.T = torch.empty((self.V, 12), dtype=torch.float64, device=self.verts.device)
        self.Tinv = torch.empty_like(self.T)
        self.buckets = Buckets(self.V)
        self.box = torch.empty(6, dtype=torch.int64, device=self.verts.device)  # posed bbox keys (cf_lbs_setup)

    def set_pose(self, A, buckets: bool = True) -> None:
        """Per-frame setup from bone transforms A (J,4,4): numpy, or a CUDA tensor used in
        place. buckets=False skips the vertex buckets (the render's fallback pass scans
        the posed vertices instead); build_buckets() adds them later."""
        self.A = A.contiguous() if is_device(A) else dev(np.asarray(A, dtype=np.float64))
        s = _lib.stream_ptr()
        # blended vertex transforms + inverses + posed vertices (+ their box) in one kernel
        _lib.call("cf_lbs_setup", self.A.data_ptr(), self.J, self.verts.data_ptr(), self.W.data_ptr(), self.V,
                  self.T.data_ptr(), self.Tinv.data_ptr(), self.posed.data_ptr(), self.box.data_ptr(), s)
        if buckets:
            self.build_buckets()

    def build_buckets(self) -> None:
        self.buckets.build(self.posed)

    def warp(self, pts: torch.Tensor):
        n = pts.shape[0]
        d = pts.device
        vert = torch.empty(n, dtype=torch.int64, device=d)
        pc = torch.empty((n, 3), dtype=torch.float64, device=d)
        valid = torch.empty(n, dtype=torch.uint8, device=d)
        _lib.call("cf_lbs_backward", self.buckets.handle, self.posed.data_ptr(), self.Tinv.data_ptr(), self.V,
                  self.max_dist, pts.data_ptr(), int(n), vert.data_ptr(), pc.data_ptr(), valid.data_ptr(),
                  _lib.stream_ptr())
        return vert, pc, valid.bool()

    def __call__(self, pts):
        on_dev = is_device(pts)
        p = dev(pts if on_dev else np.atleast_2d(np.asarray(pts, dtype=np.float64)), shape_last=3)
        v, pc, valid = self.warp(p)
        if on_dev:
            return v, pc, valid
        return host(v), host(pc), host(valid)
