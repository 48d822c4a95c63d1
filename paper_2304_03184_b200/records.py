"""Motion-prior stream ingestion — drop-in for capfields.records'
motion-prior half (records.py:89-147), plus the device LUT the render path reads.

* `MotionPriorWriter` / `load_motion_priors` keep the reference's names, file
  format (CFMP v1) and errors (`RecordFormatError`, records.py:24); the codec is the
  native one in csrc/records.cu (`cf_mp_write` / `cf_mp_scan` / `cf_mp_read`).
* `MotionPriorStream` decodes a whole stream into pinned host memory, uploads it
  once into HBM (node dqs, pose, object pose of every frame) and runs the
  skeleton's forward kinematics for every frame in one device kernel
  (`cf_skinning_transforms`, skeleton.py:121-139). `Renderer.load_prior` then takes
  a frame's rows straight from the LUT: no per-frame host work or upload.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .edgraph import GraphMotion
from .errors import RecordFormatError
from . import scene as _rig

MOTION_MAGIC = b"CFMP"
VERSION = 1


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


@dataclass
class SkeletonPose:
    """Pose vector of a skeleton (skeleton.py:56-68); `skeleton` may be None (default rig)."""

    skeleton: object
    theta: np.ndarray = field(default_factory=lambda: np.zeros(3 * _rig.N_JOINTS))

    def __post_init__(self):
        self.theta = np.asarray(self.theta, dtype=np.float64).reshape(-1)
        nj = getattr(self.skeleton, "n_joints", _rig.N_JOINTS)
        if len(self.theta) != 3 * nj:
            raise ValueError("theta length must be 3 * number of joints")


@dataclass
class Se3:
    """Rigid transform (transforms.py:258-270)."""

    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)


@dataclass
class MotionPrior:
    """Per-frame motion estimate handed from tracking to rendering (records.py:89-100)."""

    frame_id: int
    graph_motion: GraphMotion
    pose: SkeletonPose
    object_pose: Se3

    def __post_init__(self):
        if self.graph_motion.frame_id != self.frame_id:
            raise ValueError("graph motion frame id mismatch")


class MotionPriorWriter:
    """Append-only CFMP v1 stream (records.py:103-126). Accepts the reference's
    MotionPrior objects as well as this module's (duck-typed)."""

    def __init__(self, path: str, n_nodes: int, n_theta: int):
        self.path = _path(path)
        self.n_nodes = int(n_nodes)
        self.n_theta = int(n_theta)
        _lib.call("cf_mp_write", self.path, 1, self.n_nodes, self.n_theta, 0, None, None, None, None, None)

    def append(self, prior) -> None:
        self.append_batch([prior])

    def append_batch(self, priors) -> None:
        """Append several frames with one native call."""
        c = len(priors)
        if c == 0:
            return
        fids = np.array([p.frame_id for p in priors], dtype=np.int64)
        dqs = np.ascontiguousarray(np.stack([np.asarray(p.graph_motion.dqs, dtype=np.float64) for p in priors]))
        theta = np.ascontiguousarray(np.stack([np.asarray(p.pose.theta, dtype=np.float64).reshape(-1)
                                               for p in priors]))
        rot = np.ascontiguousarray(np.stack([np.asarray(p.object_pose.rotation, dtype=np.float64).reshape(9)
                                             for p in priors]))
        trans = np.ascontiguousarray(np.stack([np.asarray(p.object_pose.translation, dtype=np.float64).reshape(3)
                                               for p in priors]))
        if dqs.shape[1:] != (self.n_nodes, 8) or theta.shape[1] != self.n_theta:
            raise ValueError("prior shape differs from the stream's n_nodes / n_theta")
        _lib.call("cf_mp_write", self.path, 0, self.n_nodes, self.n_theta, c, _ptr(fids), _ptr(dqs), _ptr(theta),
                  _ptr(rot), _ptr(trans))

    def close(self) -> None:
        pass  # every append is flushed and closed natively

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def scan_motion_priors(path) -> _lib.MpInfo:
    info = _lib.MpInfo()
    _lib.call("cf_mp_scan", _path(path), _lib.byref(info))
    return info


def read_motion_arrays(path, first: int = 0, count: int | None = None, pin: bool = False):
    """Decode frames [first, first + count) -> (frame_ids, dqs, theta, rot, trans) host arrays."""
    info = scan_motion_priors(path)
    if count is None:
        count = info.n_frames - first
    nn, nt = info.n_nodes, info.n_theta

    def buf(shape, dtype):
        if pin and torch.cuda.is_available():
            return torch.empty(shape, dtype=dtype).pin_memory().numpy()
        return np.empty(shape, dtype=np.int64 if dtype == torch.int64 else np.float64)

    fids = buf((count,), torch.int64)
    dqs = buf((count, nn, 8), torch.float64)
    theta = buf((count, nt), torch.float64)
    rot = buf((count, 3, 3), torch.float64)
    trans = buf((count, 3), torch.float64)
    _lib.call("cf_mp_read", _path(path), first, count, _ptr(fids), _ptr(dqs), _ptr(theta), _ptr(rot), _ptr(trans))
    return fids, dqs, theta, rot, trans


def load_motion_priors(path: str, skeleton=None) -> list[MotionPrior]:
    """All frames of a stream as MotionPrior objects (records.py:128-147)."""
    fids, dqs, theta, rot, trans = read_motion_arrays(path)
    return [MotionPrior(int(f), GraphMotion(int(f), dqs[i]), SkeletonPose(skeleton, theta[i]), Se3(rot[i], trans[i]))
            for i, f in enumerate(fids)]


def _rig_arrays(skeleton):
    if skeleton is None:
        return np.asarray(_rig.PARENTS, dtype=np.int32), np.asarray(_rig.OFFSETS, dtype=np.float64)
    return (np.ascontiguousarray(np.asarray(skeleton.parents), dtype=np.int32),
            np.ascontiguousarray(np.asarray(skeleton.offsets), dtype=np.float64))


def skinning_transforms(theta: torch.Tensor, skeleton=None) -> torch.Tensor:
    """Device FK for a batch of poses: theta (F, 3J) -> A (F, J, 4, 4) float64
    (skinning_transforms, skeleton.py:135-139, for every frame in one launch)."""
    parents, offsets = _rig_arrays(skeleton)
    J = len(parents)
    th = theta.to(torch.float64).reshape(-1, 3 * J).contiguous()
    A = torch.empty((th.shape[0], J, 4, 4), dtype=torch.float64, device=th.device)
    _lib.call("cf_skinning_transforms", th.data_ptr(), th.shape[0], _ptr(parents), _ptr(offsets), J, A.data_ptr(),
              _lib.stream_ptr())
    return A


class MotionPriorStream:
    """A CFMP stream resident in HBM: the render path's per-frame motion LUT.

    Attributes (device tensors, frame-major): `dqs` (F, n, 8) f64, `theta` (F, 3J) f64,
    `obj_R` (F, 3, 3), `obj_t` (F, 3), `bone_A` (F, J, 4, 4) f64 (device FK);
    `frame_ids` (F,) host int64. `lookup_table` mirrors KnnField's (F*n, 8) LUT."""

    def __init__(self, path: str, skeleton=None, device=None):
        device = device or _lib.require_cuda()
        fids, dqs, theta, rot, trans = read_motion_arrays(path, pin=True)
        self.frame_ids = np.array(fids)
        self.n_frames, self.n_nodes = dqs.shape[0], dqs.shape[1]
        self._slot = {int(f): i for i, f in enumerate(self.frame_ids)}
        up = lambda a: torch.from_numpy(a).to(device, non_blocking=True)  # noqa: E731
        self.dqs, self.theta, self.obj_R, self.obj_t = up(dqs), up(theta), up(rot), up(trans)
        self.bone_A = skinning_transforms(self.theta, skeleton)
        self._host = (dqs, theta, rot, trans)  # pinned sources stay alive until the copies ran
        torch.cuda.current_stream().synchronize()

    def __len__(self) -> int:
        return self.n_frames

    def slot(self, frame_id: int) -> int:
        if int(frame_id) not in self._slot:
            raise KeyError(f"frame {frame_id} not in the stream")
        return self._slot[int(frame_id)]

    @property
    def lookup_table(self) -> torch.Tensor:
        return self.dqs.reshape(-1, 8)

    def graph_motion(self, frame_id: int) -> GraphMotion:
        return GraphMotion(int(frame_id), self.dqs[self.slot(frame_id)].cpu().numpy())

    def theta_bias(self, nets) -> torch.Tensor:
        """DeformNet pose bias of every frame: (F, 128) fp32 = theta W1[:, 32:]^T."""
        W = torch.as_tensor(np.asarray(nets.layers["D1"][:, 32:], dtype=np.float32), device=self.theta.device)
        return (self.theta.to(torch.float32) @ W.t()).contiguous()

    def load_into(self, renderer, frame_id: int, dbias: torch.Tensor | None = None) -> None:
        """Stage one frame of the LUT into a Renderer (device-to-device, no host sync)."""
        i = self.slot(frame_id)
        if renderer.human is not None:
            if dbias is None:
                dbias = self.theta_bias(renderer.human.nets)[i]
            renderer.load_prior(self.dqs[i], self.bone_A[i], dbias)
        if renderer.obj is not None:
            renderer.set_object_pose(self._host[2][i], self._host[3][i])  # host frame block


__all__ = ["MOTION_MAGIC", "VERSION", "RecordFormatError", "MotionPrior", "MotionPriorWriter", "MotionPriorStream",
           "SkeletonPose", "Se3", "load_motion_priors", "read_motion_arrays", "scan_motion_priors",
           "skinning_transforms"]
