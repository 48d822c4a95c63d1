"""Constant-time motion-prior lookup on the GPU — drop-in for capfields.knnfield.

KnnField keeps the reference's public attributes (knnfield.py:45-236):
`neighbor_idx`, `live_maps`, `lookup_table`, `bbox_min`, `voxel_size`,
`resolution`, `s`, `support_radius`; the tables live in HBM and are copied to
host lazily when a numpy attribute is read. All construction / update / query
work runs in the sm_100a kernels of csrc/knnfield.cu.
"""
from __future__ import annotations

from collections.abc import Mapping

import numpy as np
import torch

from . import _lib
from ._tensors import dev, host, is_device
from .edgraph import EDGraph, GraphMotion, FrameMotion, knn_warp, knn_warp_cull, Buckets
from .errors import OutOfSupportError


def brute_force_neighbors_batch(graph, pts, s: int) -> np.ndarray:
    """Exact s nearest node indices, ties by index (knnfield.py:25-29)."""
    p = dev(np.atleast_2d(np.asarray(pts, dtype=np.float64)), shape_last=3)
    nodes = dev(graph.nodes, shape_last=3)
    idx, _, _, _ = knn_warp(nodes, None, s, float(graph.radius), _lib.CF_NEIGHBORS_ONLY, p, None, want_idx=True,
                            want_pc=False, want_valid=False)
    return host(idx)


def brute_force_neighbors(graph, p, s: int) -> np.ndarray:
    return brute_force_neighbors_batch(graph, np.asarray(p, dtype=np.float64)[None], s)[0]


def brute_force_query(graph, motion, pts_live, s: int, search: str = "brute"):
    """Exact (indices, weights, canonical pts) over deformed nodes (knnfield.py:32-42).

    search="brute" is the exhaustive kernel; "bucket" the voxel-bucket ring search;
    "cull" the Morton-ordered warp-culled search (n <= 8192, s <= 8); all
    bit-identical."""
    on_dev = is_device(pts_live)
    p = dev(pts_live if on_dev else np.atleast_2d(np.asarray(pts_live, dtype=np.float64)), shape_last=3)
    fm = FrameMotion(graph, motion, buckets=(search == "bucket"))
    if search == "cull":
        idx, w, pc, _ = knn_warp_cull(fm.anchors, fm.dqs, s, fm.radius, _lib.CF_BRUTE_QUERY, p,
                                      want_idx=True, want_w=True, want_valid=False)
    else:
        idx, w, pc, _ = knn_warp(fm.anchors, fm.dqs, s, fm.radius, _lib.CF_BRUTE_QUERY, p, fm.live_buckets,
                                 want_idx=True, want_w=True, want_valid=False)
    if on_dev:
        return idx, w, pc
    return host(idx), host(w), host(pc)


class _LiveMaps(Mapping):
    """dict-like view of per-frame live maps; values expanded from the frame's bricks
    and copied to host on access."""

    def __init__(self, field: "KnnField"):
        self._f = field

    def __getitem__(self, fid):
        return host(self._f.live_map_dense(fid))

    def __iter__(self):
        return iter(self._f._live_dev)

    def __len__(self):
        return len(self._f._live_dev)

    def __contains__(self, fid):
        return fid in self._f._live_dev


class KnnField:
    """Canonical KNN voxel field + per-frame live index maps + motion table."""

    def __init__(self, graph, resolution: int = 512, s: int = 4, bbox=None, support_radius: float | None = None):
        if resolution < 8:
            raise ValueError("resolution must be at least 8")
        self.graph = graph
        self.resolution = int(resolution)
        n = len(graph.nodes)
        self.s = int(min(s, n))
        self.support_radius = float(support_radius if support_radius is not None else 2.0 * graph.radius)
        nodes = np.asarray(graph.nodes, dtype=np.float64)
        if bbox is None:
            margin = self.support_radius + 2.0 * graph.radius  # knnfield.py:61-69
            lo = nodes.min(axis=0) - margin
            hi = nodes.max(axis=0) + margin
        else:
            lo, hi = np.asarray(bbox[0], dtype=np.float64), np.asarray(bbox[1], dtype=np.float64)
        self.bbox_min = lo
        self.voxel_size = float((hi - lo).max() / self.resolution)
        self._bmin_c = (_lib.ctypes.c_double * 3)(*[float(v) for v in lo])
        self._nodes_dev = dev(nodes, shape_last=3)
        r3 = self.resolution ** 3
        self._nidx_dev = torch.empty((r3, self.s), dtype=torch.int32, device=self._nodes_dev.device)
        _lib.call("cf_knnfield_build", self._nodes_dev.data_ptr(), n, self.s, self.resolution, self._bmin_c,
                  self.voxel_size, self.support_radius, self._nidx_dev.data_ptr(), _lib.stream_ptr())
        self._nidx_host = None
        self._live_dev: dict[int, torch.Tensor] = {}
        self._frame_slots: dict[int, int] = {}
        self._lut_blocks: list[np.ndarray] = []
        self._lut_dev: dict[int, torch.Tensor] = {}
        self._anchors_dev: dict[int, torch.Tensor] = {}
        self._scratch_u64 = None
        self._scratch_i32 = None
        self._scratch_live = None
        nb = _lib.ctypes.c_int64()
        _lib.call("cf_knnfield_brick_count", self.resolution, _lib.ctypes.byref(nb))
        self._n_bricks = int(nb.value)
        self.live_maps = _LiveMaps(self)

    # -- reference attributes -------------------------------------------------

    @property
    def neighbor_idx(self) -> np.ndarray:
        if self._nidx_host is None:
            self._nidx_host = host(self._nidx_dev)
        return self._nidx_host

    @property
    def lookup_table(self) -> np.ndarray:
        if not self._lut_blocks:
            return np.zeros((0, 8))
        return np.concatenate(self._lut_blocks, axis=0)

    def _voxel_centers(self, flat_idx: np.ndarray) -> np.ndarray:
        r = self.resolution
        flat_idx = np.asarray(flat_idx)
        ijk = np.stack([flat_idx // (r * r), (flat_idx // r) % r, flat_idx % r], axis=-1).astype(np.float64)
        return self.bbox_min + (ijk + 0.5) * self.voxel_size

    def _flat_index(self, pts: np.ndarray):
        r = self.resolution
        ijk = np.floor((np.asarray(pts, dtype=np.float64) - self.bbox_min) / self.voxel_size).astype(np.int64)
        inside = np.all((ijk >= 0) & (ijk < r), axis=-1)
        ijk = np.clip(ijk, 0, r - 1)
        return ijk[..., 0] * r * r + ijk[..., 1] * r + ijk[..., 2], inside

    def in_support_voxels(self) -> np.ndarray:
        return np.nonzero(self.neighbor_idx[:, 0] >= 0)[0]

    def voxel_diagonal(self) -> float:
        return float(self.voxel_size * np.sqrt(3.0))

    def frame_offset(self, frame_id: int) -> int:
        if frame_id not in self._frame_slots:
            raise OutOfSupportError(f"frame {frame_id} not registered")
        return self._frame_slots[frame_id] * len(self.graph.nodes)

    # -- per-frame update -----------------------------------------------------

    def update_live_map(self, motion) -> None:
        """Warp in-support canonical voxels to live space (knnfield.py:124-167)."""
        fid = motion.frame_id
        if fid in self._frame_slots:
            raise ValueError(f"frame {fid} already registered")
        dqs_np = np.asarray(motion.dqs, dtype=np.float64)
        n = len(self.graph.nodes)
        if dqs_np.shape[0] != n:
            raise ValueError("motion node count does not match the graph")
        r3 = self.resolution ** 3
        d = self._nodes_dev.device
        if self._scratch_u64 is None:
            # dense scratch shared by every frame's update (2 GiB at 512^3, freed by
            # release_scratch); a frame keeps only its bricks (SURVEY §7 hard part 6)
            self._scratch_u64 = torch.empty(r3, dtype=torch.int64, device=d)
            self._scratch_i32 = torch.empty(r3, dtype=torch.int32, device=d)
            self._scratch_live = torch.empty(r3, dtype=torch.int32, device=d)
        dqs = dev(dqs_np, shape_last=8)
        dense = self._scratch_live
        s = _lib.stream_ptr()
        _lib.call("cf_knnfield_update", self._nodes_dev.data_ptr(), dqs.data_ptr(), n, self._nidx_dev.data_ptr(),
                  self.s, self.resolution, self._bmin_c, self.voxel_size, float(self.graph.radius), dense.data_ptr(),
                  self._scratch_u64.data_ptr(), self._scratch_i32.data_ptr(), s)
        bidx = torch.empty(self._n_bricks, dtype=torch.int32, device=d)
        n_set = torch.empty(1, dtype=torch.int32, device=d)
        _lib.call("cf_knnfield_brick_index", dense.data_ptr(), self.resolution, bidx.data_ptr(), n_set.data_ptr(), s)
        bricks = torch.empty(max(int(n_set.item()), 1) * 512, dtype=torch.int32, device=d)  # one sync per registration
        _lib.call("cf_knnfield_brick_pack", dense.data_ptr(), self.resolution, bidx.data_ptr(), bricks.data_ptr(), s)
        live = (bidx, bricks)
        anchors = torch.empty_like(self._nodes_dev)
        _lib.call("cf_deform_nodes", self._nodes_dev.data_ptr(), dqs.data_ptr(), n, anchors.data_ptr(),
                  _lib.stream_ptr())
        self._live_dev[fid] = live
        self._lut_dev[fid] = dqs
        self._anchors_dev[fid] = anchors
        self._frame_slots[fid] = len(self._frame_slots)
        self._lut_blocks.append(dqs_np.copy())

    def live_map_dense(self, frame_id: int) -> torch.Tensor:
        """The frame's live map as the reference's dense (r^3,) int32 array (device)."""
        bidx, bricks = self._live_dev[frame_id]
        out = torch.empty(self.resolution ** 3, dtype=torch.int32, device=bidx.device)
        _lib.call("cf_knnfield_brick_unpack", bidx.data_ptr(), bricks.data_ptr(), self.resolution, out.data_ptr(),
                  _lib.stream_ptr())
        return out

    def live_map_bytes(self, frame_id: int) -> int:
        """Device bytes the frame's live map occupies (brick table + set bricks)."""
        bidx, bricks = self._live_dev[frame_id]
        return bidx.numel() * 4 + bricks.numel() * 4

    def release_scratch(self) -> None:
        """Free the dense update scratch (re-allocated by the next update_live_map)."""
        self._scratch_u64 = self._scratch_i32 = self._scratch_live = None

    # -- queries --------------------------------------------------------------

    def query_motion_batch(self, pts_live, frame_id: int, strict: bool = False):
        """O(1) lookup -> (indices, weights, p_canonical, valid) (knnfield.py:197-222)."""
        self.frame_offset(frame_id)  # raises for an unregistered frame
        on_dev = is_device(pts_live)
        p = dev(pts_live if on_dev else np.atleast_2d(np.asarray(pts_live, dtype=np.float64)), shape_last=3)
        n_pts = p.shape[0]
        d = p.device
        nbr = torch.empty((n_pts, self.s), dtype=torch.int64, device=d)
        w = torch.empty((n_pts, self.s), dtype=torch.float64, device=d)
        pc = torch.empty((n_pts, 3), dtype=torch.float64, device=d)
        valid = torch.empty(n_pts, dtype=torch.uint8, device=d)
        bidx, bricks = self._live_dev[frame_id]
        _lib.call("cf_knnfield_query_sparse", bidx.data_ptr(), bricks.data_ptr(), self._nidx_dev.data_ptr(),
                  self._lut_dev[frame_id].data_ptr(), self._anchors_dev[frame_id].data_ptr(), self.s, self.resolution,
                  self._bmin_c, self.voxel_size, float(self.graph.radius), p.data_ptr(), n_pts, nbr.data_ptr(),
                  w.data_ptr(), pc.data_ptr(), valid.data_ptr(), _lib.stream_ptr())
        valid = valid.bool()
        if strict and not bool(valid.all()):
            raise OutOfSupportError("query outside the mapped live volume")
        if on_dev:
            return nbr, w, pc, valid
        return host(nbr), host(w), host(pc), host(valid)

    def query_motion(self, p_live, frame_id: int):
        nbr, w, p_c, _ = self.query_motion_batch(np.asarray(p_live, dtype=np.float64)[None], frame_id, strict=True)
        return nbr[0], w[0], p_c[0]


def build_knn_field(graph, resolution: int, s: int, **kw) -> KnnField:
    return KnnField(graph, resolution=resolution, s=s, **kw)


def query_motion(field: KnnField, p_live, frame_id: int):
    return field.query_motion(p_live, frame_id)


def update_live_map(field: KnnField, motion) -> None:
    field.update_live_map(motion)


__all__ = [
    "EDGraph", "GraphMotion", "KnnField", "Buckets", "brute_force_neighbors", "brute_force_neighbors_batch",
    "brute_force_query", "build_knn_field", "query_motion", "update_live_map",
]
