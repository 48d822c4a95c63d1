"""Embedded-deformation warps on the GPU — drop-in for capfields.edgraph.

Same names, argument meaning and error behaviour as the reference
(capfields/edgraph.py:31-215); the per-sample work runs in the sm_100a
`cf_knn_warp` kernel (exact bucketed k-NN over deformed nodes + DQB in float64,
bit-identical neighbour indices). numpy inputs give numpy outputs; CUDA tensor
inputs give CUDA tensor outputs with no host round trip.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import dev, host, is_device
from .errors import OutOfSupportError

WEIGHT_FLOOR = 1e-6  # edgraph.py:24


@dataclass
class EDGraph:
    """Canonical node set (edgraph.py:31-59): nodes (n,3), Gaussian radius, knn_k."""

    nodes: np.ndarray
    radius: float = 0.1
    knn_k: int = 4

    def __post_init__(self):
        self.nodes = np.atleast_2d(np.asarray(self.nodes, dtype=np.float64))
        if len(self.nodes) == 0:
            raise ValueError("graph needs at least one node")
        if self.radius <= 0:
            raise ValueError("influence radius must be positive")
        self.knn_k = int(min(self.knn_k, len(self.nodes)))

    @property
    def n_nodes(self) -> int:
        return len(self.nodes)


@dataclass
class GraphMotion:
    """Per-frame node transforms, packed (n, 8) dual quaternions (edgraph.py:62-87)."""

    frame_id: int
    dqs: np.ndarray

    def __post_init__(self):
        self.dqs = np.asarray(self.dqs, dtype=np.float64)
        if self.dqs.ndim != 2 or self.dqs.shape[1] != 8:
            raise ValueError("dqs must be (n, 8) packed dual quaternions")

    @staticmethod
    def identity(frame_id: int, n_nodes: int) -> "GraphMotion":
        dqs = np.zeros((n_nodes, 8))
        dqs[:, 0] = 1.0
        return GraphMotion(frame_id, dqs)


class FrameMotion:
    """Device-resident state of one (graph, motion) pair: nodes, dqs, deformed
    anchors and their coarse buckets. Built once per frame and reused by every
    warp call of that frame (the render path's per-frame setup)."""

    def __init__(self, graph, motion, buckets=True):
        nodes = graph.nodes
        self.n = int(len(nodes))
        self.k = int(min(getattr(graph, "knn_k", 4), self.n))
        self.radius = float(graph.radius)
        self.nodes = dev(nodes, shape_last=3)
        self.dqs = dev(motion.dqs, shape_last=8)
        if self.dqs.shape[0] != self.n:
            raise ValueError("motion node count does not match the graph")
        self.anchors = torch.empty_like(self.nodes)
        _lib.call("cf_deform_nodes", self.nodes.data_ptr(), self.dqs.data_ptr(), self.n, self.anchors.data_ptr(),
                  _lib.stream_ptr())
        self.canon_buckets = None
        self.live_buckets = None
        if buckets is not False and buckets is not None:
            self.live_buckets = buckets if isinstance(buckets, Buckets) else Buckets(self.n)
            self.live_buckets.build(self.anchors, candidates_k=self.k)

    def canonical_buckets(self) -> "Buckets":
        if self.canon_buckets is None:
            self.canon_buckets = Buckets(self.n)
            self.canon_buckets.build(self.nodes, candidates_k=self.k)
        return self.canon_buckets


class Buckets:
    """Owning wrapper of a cf_buckets_t handle (coarse voxel bucketing)."""

    def __init__(self, max_points: int, max_grid_res: int = 64):
        h = _lib._p()
        _lib.call("cf_buckets_create", int(max_points), int(max_grid_res), _lib.ctypes.byref(h))
        self.handle = h.value
        self.max_points = int(max_points)

    def build(self, pts: torch.Tensor, grid_res: int = 0, candidates_k: int = 0) -> None:
        """Counting-sort `pts` into the grid; with candidates_k > 0 also build the
        per-cell candidate lists for k-NN queries with k <= candidates_k."""
        self._pts = pts  # keep alive for stream-ordered use
        _lib.call("cf_buckets_build", self.handle, pts.data_ptr(), int(pts.shape[0]), int(grid_res), _lib.stream_ptr())
        if candidates_k > 0:
            _lib.call("cf_buckets_build_candidates", self.handle, int(min(candidates_k, pts.shape[0])),
                      _lib.stream_ptr())

    def __del__(self):
        # stream-ordered: the frees follow the work queued on the current stream (no host sync)
        h = getattr(self, "handle", None)
        if h and _lib._lib is not None:
            _lib._lib.cf_buckets_destroy_async(h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            self.handle = None


def knn_warp(anchors: torch.Tensor, dqs: torch.Tensor | None, k: int, radius: float, mode: int, pts: torch.Tensor,
             buckets: Buckets | None, want_idx=False, want_w=False, want_pc=True, want_valid=True):
    """Raw device call of cf_knn_warp; returns (idx, w, pc, valid) tensors (None where not requested)."""
    n = pts.shape[0]
    k = int(min(k, anchors.shape[0]))
    d = pts.device
    idx = torch.empty((n, k), dtype=torch.int64, device=d) if want_idx else None
    w = torch.empty((n, k), dtype=torch.float64, device=d) if want_w else None
    pc = torch.empty((n, 3), dtype=torch.float64, device=d) if want_pc else None
    valid = torch.empty((n,), dtype=torch.uint8, device=d) if want_valid else None
    _lib.call("cf_knn_warp", buckets.handle if buckets is not None else None, anchors.data_ptr(),
              dqs.data_ptr() if dqs is not None else None, int(anchors.shape[0]), k, float(radius), int(mode),
              pts.data_ptr(), int(n), _lib.ptr(idx), _lib.ptr(w), _lib.ptr(pc), _lib.ptr(valid), _lib.stream_ptr())
    return idx, w, pc, valid


def morton_order(pts: torch.Tensor) -> torch.Tensor:
    """int32 permutation visiting `pts` (N,3) in Morton (Z-curve) order of a 1024^3
    grid over their bounding box: consecutive queries are spatial neighbours, which
    is what the warp-level culling of cf_knn_warp_cull needs."""
    lo = pts.min(0).values
    ext = (pts.max(0).values - lo).clamp_min(1e-12)
    c = ((pts - lo) / ext * 1023.0).clamp(0, 1023).to(torch.int64)

    def spread(x):  # 10 bits -> every third bit
        x = (x | (x << 16)) & 0x030000FF
        x = (x | (x << 8)) & 0x0300F00F
        x = (x | (x << 4)) & 0x030C30C3
        return (x | (x << 2)) & 0x09249249

    code = spread(c[:, 0]) | (spread(c[:, 1]) << 1) | (spread(c[:, 2]) << 2)
    return torch.argsort(code).to(torch.int32)


def knn_warp_cull(anchors: torch.Tensor, dqs: torch.Tensor | None, k: int, radius: float, mode: int,
                  pts: torch.Tensor, order: torch.Tensor | None = None, want_idx=False, want_w=False, want_pc=True,
                  want_valid=True):
    """Hierarchical exact k-NN warp (n <= 8192 nodes, k <= 8) of cf_knn_warp_cull:
    queries in Morton order, warp-level culling, fp32 ranking, float64 top-k.
    Same outputs as knn_warp, bit-identical indices."""
    n = pts.shape[0]
    k = int(min(k, anchors.shape[0]))
    d = pts.device
    if order is None and n > 0:
        order = morton_order(pts)
    idx = torch.empty((n, k), dtype=torch.int64, device=d) if want_idx else None
    w = torch.empty((n, k), dtype=torch.float64, device=d) if want_w else None
    pc = torch.empty((n, 3), dtype=torch.float64, device=d) if want_pc else None
    valid = torch.empty((n,), dtype=torch.uint8, device=d) if want_valid else None
    _lib.call("cf_knn_warp_cull", anchors.data_ptr(), dqs.data_ptr() if dqs is not None else None,
              int(anchors.shape[0]), k, float(radius), int(mode), pts.data_ptr(), _lib.ptr(order), int(n),
              _lib.ptr(idx), _lib.ptr(w), _lib.ptr(pc), _lib.ptr(valid), _lib.stream_ptr())
    return idx, w, pc, valid


def _as_pts(pts):
    if is_device(pts):
        return dev(pts, shape_last=3), True
    return dev(np.atleast_2d(np.asarray(pts, dtype=np.float64)), shape_last=3), False


def _out(t, on_dev):
    return t if on_dev else host(t)


def deformed_nodes(graph, motion) -> np.ndarray:
    """Live-space node positions (edgraph.py:134-136)."""
    return host(FrameMotion(graph, motion, buckets=False).anchors)


def warp_backward_batch(graph, motion, pts_live, strict: bool = False, search: str = "bucket",
                        frame: FrameMotion | None = None):
    """Live -> canonical warp (edgraph.py:174-183); returns (pts_c, valid).
    search: "bucket" (voxel buckets + ring search), "cull" (Morton-ordered warp
    culling, n <= 8192, k <= 8) or "brute" — identical results."""
    pts, on_dev = _as_pts(pts_live)
    fm = frame or FrameMotion(graph, motion, buckets=(search == "bucket"))
    if search == "cull":
        _, _, pc, valid = knn_warp_cull(fm.anchors, fm.dqs, fm.k, fm.radius, _lib.CF_WARP_BACKWARD, pts)
    else:
        _, _, pc, valid = knn_warp(fm.anchors, fm.dqs, fm.k, fm.radius, _lib.CF_WARP_BACKWARD, pts,
                                   fm.live_buckets if search == "bucket" else None)
    valid = valid.bool()
    if strict and not bool(valid.all()):
        raise OutOfSupportError("point outside deformed node influence")
    return _out(pc, on_dev), _out(valid, on_dev)


def warp_forward_batch(graph, motion, pts, strict: bool = False, search: str = "bucket"):
    """Canonical -> live warp (edgraph.py:154-162); returns (warped, valid)."""
    p, on_dev = _as_pts(pts)
    fm = FrameMotion(graph, motion, buckets=False)
    b = fm.canonical_buckets() if search == "bucket" else None
    _, _, out, valid = knn_warp(fm.nodes, fm.dqs, fm.k, fm.radius, _lib.CF_WARP_FORWARD, p, b)
    valid = valid.bool()
    if strict and not bool(valid.all()):
        raise OutOfSupportError("point outside node influence")
    return _out(out, on_dev), _out(valid, on_dev)


def warp_forward(graph, motion, p_canonical):
    out, _ = warp_forward_batch(graph, motion, np.asarray(p_canonical, dtype=np.float64)[None], strict=True)
    return out[0]


def warp_backward(graph, motion, p_live):
    out, _ = warp_backward_batch(graph, motion, np.asarray(p_live, dtype=np.float64)[None], strict=True)
    return out[0]
