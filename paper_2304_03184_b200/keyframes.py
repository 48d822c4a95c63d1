"""Key-frame selection on the GPU: blur gate, Eq. 5 visibility maps,
Eq. 6/7 dissimilarities, the capacity-100 spatial pool and the spatial-temporal
refinement set.

The reference package has no key-frame code, so the names and semantics follow
SPEC's `keyframes` module; the evaluation order SPEC leaves open is frozen in
oracle/keyframes.py (the test checker) and DESIGN.md §3.6. Kernels:
csrc/keyframes.cu (`cf_blur_score`, `cf_visibility_map`, `cf_pool_scan`). The pool
lives in HBM; each update is one scan launch plus a 24-byte decision readback.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import dev, is_device

TORSO_JOINTS = (0, 3, 6, 9, 12, 13, 14, 15)
BETA_TORSO, BETA_LIMB, BETA_VIS, BETA_H = 0.1, 0.02, 0.01, 0.02
BETA_D, BETA_O = 1.0, 0.02
GAMMA, CAPACITY, EPS_VIS, TAU_BLUR = 2.5, 100, 0.01, 0.6


def pose_weights(n_joints: int = 24, torso=TORSO_JOINTS) -> np.ndarray:
    w = np.full(3 * n_joints, BETA_LIMB)
    for j in torso:
        w[3 * j: 3 * j + 3] = BETA_TORSO
    return w


def blur_score(rgb) -> float:
    """Crété-Roffet blurriness of an 8-bit RGB image (H, W, 3): 0 sharp .. 1 blurred
    (SPEC.md:448-457); a constant image scores 1.0."""
    img = rgb if is_device(rgb) else torch.from_numpy(np.ascontiguousarray(np.asarray(rgb, dtype=np.uint8)))
    img = img.to(_lib.require_cuda(), torch.uint8).contiguous()
    if img.dim() != 3 or img.shape[2] != 3:
        raise ValueError("blur_score expects an (H, W, 3) uint8 image")
    H, W = int(img.shape[0]), int(img.shape[1])
    if H < 16 or W < 16:
        raise ValueError("blur_score needs an image of at least 16x16")
    sums = torch.empty(4, dtype=torch.int64, device=img.device)
    score = torch.empty(1, dtype=torch.float64, device=img.device)
    _lib.call("cf_blur_score", img.data_ptr(), H, W, sums.data_ptr(), score.data_ptr(), _lib.stream_ptr())
    return float(score.item())


def _vis_camera(cam) -> _lib.VisCamera:
    """World->camera of a pinhole camera given camera-to-world (R, t) attributes or a
    reference-style `pose` (Se3 camera-to-world, camera.py:27-35)."""
    if hasattr(cam, "pose"):
        Rcw, tcw = np.asarray(cam.pose.rotation, dtype=np.float64), np.asarray(cam.pose.translation, dtype=np.float64)
    else:
        Rcw, tcw = np.asarray(cam.R, dtype=np.float64), np.asarray(cam.t, dtype=np.float64)
    Rwc = Rcw.T  # Se3.inverse (transforms.py:293-295)
    twc = -Rwc @ tcw
    c = _lib.VisCamera()
    for i in range(9):
        c.R[i] = float(Rwc.reshape(-1)[i])
    for i in range(3):
        c.t[i] = float(twc[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    return c


def world_to_cam(cam):
    """(R_wc, t_wc) exactly as the visibility kernel receives them."""
    c = _vis_camera(cam)
    return np.array(list(c.R)).reshape(3, 3), np.array(list(c.t))


def visibility_bits(nodes, depth, cam, eps: float = EPS_VIS) -> torch.Tensor:
    """Eq. 5 for n deformed nodes against a depth map (metres, 0 invalid) -> packed
    visibility words (ceil(n/32),) int32 on the device."""
    p = dev(nodes, shape_last=3)
    D = dev(depth)
    if D.dim() != 2:
        raise ValueError("depth must be (H, W)")
    n = int(p.shape[0])
    bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device=p.device)
    c = _vis_camera(cam)
    _lib.call("cf_visibility_map", p.data_ptr(), n, D.data_ptr(), int(D.shape[0]), int(D.shape[1]),
              _lib.byref(c), float(eps), bits.data_ptr(), _lib.stream_ptr())
    return bits


def unpack_bits(words, n: int) -> np.ndarray:
    w = (words.cpu().numpy() if isinstance(words, torch.Tensor) else np.asarray(words)).astype(np.uint32)
    return ((w[np.arange(n) // 32] >> (np.arange(n) % 32).astype(np.uint32)) & 1).astype(bool)


def pack_bits(vis, n: int) -> torch.Tensor:
    """Visibility as device words: packed int32 words pass through; a bool (n,) map
    is packed on the device (bit i of word i // 32 = node i)."""
    d = _lib.require_cuda()
    if isinstance(vis, torch.Tensor) and vis.dtype == torch.int32:
        return vis.to(d)
    b = torch.as_tensor(np.asarray(vis.cpu() if isinstance(vis, torch.Tensor) else vis, dtype=bool)).to(d)
    if b.numel() != n:
        raise ValueError("visibility length must equal the node count")
    words = max(1, (n + 31) // 32)
    full = torch.zeros(words * 32, dtype=torch.int32, device=d)
    full[:n] = b.to(torch.int32)
    sh = torch.arange(32, dtype=torch.int32, device=d)
    return (full.view(words, 32) << sh).sum(1, dtype=torch.int32)


def visibility_map(nodes, depth, cam, eps: float = EPS_VIS) -> np.ndarray:
    """SPEC visibility_map -> bool (n,) (Eq. 5)."""
    n = len(nodes)
    return unpack_bits(visibility_bits(nodes, depth, cam, eps), n)


@dataclass
class FrameSummary:
    """frame id (= time), pose theta, node visibility bits, object
    translation d, blur score. `visibility` may be packed words on the device."""

    frame_id: int
    theta: np.ndarray | None = None
    visibility: object = None
    d: np.ndarray | None = None
    blur: float = 0.0


class KeyFramePool:
    """Capacity-`capacity` spatial pool of one field (kind "human": Eq. 6 over pose,
    visibility and time; "object": Eq. 7 over translation and time), resident in HBM
    (SPEC.md:440-443,483-491)."""

    def __init__(self, kind: str = "human", n_nodes: int = 0, capacity: int = CAPACITY, gamma: float = GAMMA,
                 n_theta: int = 72, beta_pose=None):
        if kind not in ("human", "object"):
            raise ValueError("kind must be 'human' or 'object'")
        d = _lib.require_cuda()
        self.kind, self.capacity, self.gamma = kind, int(capacity), float(gamma)
        self.n_theta, self.n_nodes = int(n_theta), int(n_nodes)
        self.words = max(1, (self.n_nodes + 31) // 32)
        self.theta = torch.zeros((self.capacity, self.n_theta), dtype=torch.float64, device=d)
        self.vis = torch.zeros((self.capacity, self.words), dtype=torch.int32, device=d)
        self.t = torch.zeros(self.capacity, dtype=torch.int64, device=d)
        self.d = torch.zeros((self.capacity, 3), dtype=torch.float64, device=d)
        bp = pose_weights(self.n_theta // 3) if beta_pose is None else np.asarray(beta_pose, dtype=np.float64)
        self.beta_pose = dev(bp)
        self.dissim = torch.zeros(max(self.capacity, 1), dtype=torch.float64, device=d)
        self._dec = torch.zeros(3, dtype=torch.float64, device=d)  # 24-byte cf_pool_decision
        self._cand = {"theta": torch.zeros(self.n_theta, dtype=torch.float64, device=d),
                      "vis": torch.zeros(self.words, dtype=torch.int32, device=d),
                      "d": torch.zeros(3, dtype=torch.float64, device=d)}
        self.frame_ids: list[int] = []  # entry slot -> frame id
        self.count = 0

    def __len__(self) -> int:
        return self.count

    def _desc(self) -> _lib.PoolDesc:
        P = _lib.PoolDesc()
        P.kind = _lib.CF_POOL_HUMAN if self.kind == "human" else _lib.CF_POOL_OBJECT
        P.count, P.capacity, P.n_theta, P.vis_words = self.count, self.capacity, self.n_theta, self.words
        P.theta, P.vis, P.t, P.d = (self.theta.data_ptr(), self.vis.data_ptr(), self.t.data_ptr(),
                                    self.d.data_ptr())
        P.beta_pose = self.beta_pose.data_ptr()
        P.beta_vis = BETA_VIS
        P.beta_t = BETA_H if self.kind == "human" else BETA_O
        P.beta_d, P.gamma = BETA_D, self.gamma
        return P

    def _stage(self, s: FrameSummary) -> _lib.PoolEntry:
        c = self._cand
        if self.kind == "human":
            c["theta"].copy_(torch.as_tensor(np.asarray(s.theta, dtype=np.float64)).reshape(-1), non_blocking=False)
            c["vis"].copy_(pack_bits(s.visibility, self.n_nodes))
        else:
            c["d"].copy_(torch.as_tensor(np.asarray(s.d, dtype=np.float64)).reshape(3))
        e = _lib.PoolEntry()
        e.theta, e.vis, e.t, e.d = c["theta"].data_ptr(), c["vis"].data_ptr(), int(s.frame_id), c["d"].data_ptr()
        return e

    def scan(self, s: FrameSummary):
        """Dissimilarity of `s` to every entry (device (count,) f64) and the decision
        (insert, evict_slot, nearest_slot, min_dissim)."""
        P, e = self._desc(), self._stage(s)
        _lib.call("cf_pool_scan", _lib.byref(P), _lib.byref(e), self.dissim.data_ptr(), self._dec.data_ptr(),
                  _lib.stream_ptr())
        raw = self._dec.cpu().numpy().tobytes()
        dec = _lib.PoolDecision.from_buffer_copy(raw)
        return self.dissim[: self.count], (bool(dec.insert), dec.evict, dec.nearest, dec.min_dissim)

    def update(self, s: FrameSummary):
        """pool_update -> (inserted, evicted frame id or None)."""
        _, (ins, evict, _, _) = self.scan(s)
        if not ins:
            return False, None
        evicted = None
        if evict >= 0:
            evicted = self.frame_ids[evict]
            slot = evict
        else:
            slot = self.count
            self.count += 1
            self.frame_ids.append(None)
        c = self._cand
        self.theta[slot].copy_(c["theta"])
        self.vis[slot].copy_(c["vis"])
        self.d[slot].copy_(c["d"])
        self.t[slot] = int(s.frame_id)
        self.frame_ids[slot] = int(s.frame_id)
        return True, evicted

    def refinement_set(self, view: FrameSummary, recent_ids, m: int = 10) -> list[int]:
        """refinement_set: the m entries least dissimilar to the render
        view (ties -> oldest) followed by the m most recent frames, duplicates removed."""
        out: list[int] = []
        if self.count:
            dis, _ = self.scan(view)
            key = torch.stack([dis, self.t[: self.count].to(torch.float64)], 1).cpu().numpy()
            order = sorted(range(self.count), key=lambda e: (key[e, 0], key[e, 1]))
            out = [self.frame_ids[e] for e in order[:m]]
        for f in list(recent_ids)[-m:][::-1]:
            if int(f) not in out:
                out.append(int(f))
        return out


def summarize(frame_id: int, theta=None, nodes=None, depth=None, cam=None, d=None, eps: float = EPS_VIS,
              rgb=None) -> FrameSummary:
    """FrameSummary of a tracked frame: visibility of the deformed nodes (device bits),
    pose, object translation and (optionally) the blur score."""
    vis = visibility_bits(nodes, depth, cam, eps) if nodes is not None else None
    return FrameSummary(int(frame_id), None if theta is None else np.asarray(theta, dtype=np.float64), vis,
                        None if d is None else np.asarray(d, dtype=np.float64),
                        blur_score(rgb) if rgb is not None else 0.0)


def fixed_interval_selector(n_frames: int, n_keep: int = CAPACITY) -> list[int]:
    """Ablation baseline: stride = sequence / n_keep, ceil(N / stride) frames."""
    stride = max(1, int(n_frames) // int(n_keep))
    return list(range(0, int(n_frames), stride))


__all__ = ["FrameSummary", "KeyFramePool", "blur_score", "visibility_map", "visibility_bits", "summarize",
           "fixed_interval_selector", "pose_weights", "unpack_bits", "world_to_cam"]
