"""Key-frame training step on the GPU — SPEC train_step (
PAPER Eq. 8): depth-guided samples -> hybrid canonicalisation -> hash + tcgen05
MLP forward -> masked L2 colour + 0.1 L1 depth -> compositing backward ->
tcgen05 E_g/E_c backward -> hash-grid backward (atomics) -> Adam.

Human and object fields are updated independently on their own masked rays.
Trained: the canonical hash grids and E_g/E_c of both fields, and the human's
DeformNet with its deformation grid (TrainConfig.train_deform): the canonical
hash backward also returns dL/dxc (spatial gradient of the trilinear
interpolation), which flows through xc = xu + 0.05 tanh(o) / side into the
tcgen05 DeformNet backward and on into the deformation-grid hash backward.

Every launch of a step is a kernel of this package and nothing in it waits on the
host: the frames' masked / depth-valid ray counts, the loss normalisers and the
power-of-two loss scale are computed on the device (cf_train_counts /
cf_train_norms), the weight gradients dW = dY^T X are one grouped tcgen05 launch
per field and frame with the sample count read on the device (cf_dw_grouped over
the K-blocked feature-major fp16 saves), Adam is one multi-tensor launch that also zeroes the
gradients, and the fp16 weight blobs are repacked by one launch. So the whole step
(key-frame ray draw included, `Trainer.capture`) replays as one CUDA graph.

Multi-GPU: rays are sharded across ranks (`shard_batch`; the sampler's jitter is a
hash of the GLOBAL ray id, so a ray draws the same samples in any shard); the
per-frame ray counts are summed over ranks before the loss is normalised, so the
sum of the ranks' gradients is the gradient of the global batch's loss; each
field's gradients live in one flat bucket that is all-reduced (sum, NCCL over
NVLink) as soon as that field's last backward is enqueued — the human bucket while
the last frame's object backward still runs.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .render import Renderer, _FieldBuffers

COLOR_LAYERS = ("G1", "G2", "C1", "C2", "C3")
DEFORM_LAYERS = ("D1", "D2", "D3", "D4", "D5")
_FIELD_INDEX = {"human": 0, "object": 1}


@dataclass
class TrainConfig:
    lr_hash: float = 1e-2       # config.py:61
    lr_net: float = 1e-3        # config.py:62
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-15
    lambda_depth: float = 0.1   # config.py:55
    n_guided: int = 32          # config.py:49-51
    n_uniform: int = 16
    n_empty: int = 64
    depth_sigma: float = 0.02   # config.py:52
    train_deform: bool = True   # also train DeformNet + its grid (needs FrameBatch.theta)


@dataclass
class FrameBatch:
    """Rays of one key frame: its motion prior and the per-ray targets (device tensors)."""
    dqs: torch.Tensor          # (n_nodes, 8) f64
    bone_A: torch.Tensor       # (24, 4, 4) f64
    dbias: torch.Tensor        # (128,) f32 DeformNet pose bias
    obj_R: np.ndarray
    obj_t: np.ndarray
    dirs: torch.Tensor         # (R, 3) f64 unit directions from the camera centre
    gt_rgb: torch.Tensor       # (R, 3) f32
    gt_depth: torch.Tensor     # (R,) f32 distance along the ray, <= 0 = no depth
    mask_h: torch.Tensor       # (R,) u8 human mask
    mask_o: torch.Tensor       # (R,) u8 object mask
    theta: torch.Tensor | None = None  # (72,) f32 pose; DeformNet training recomputes dbias from it
    origin: np.ndarray | None = None   # (3,) f64 camera centre of the key frame (the rays' origin)
    ray0: int = 0                      # global id of the first ray (data-parallel shards)
    theta64: torch.Tensor | None = None  # (72,) f64 copy of theta (made once, reused by every step)

    def pose64(self) -> torch.Tensor:
        if self.theta64 is None:
            self.theta64 = self.theta.to(torch.float64).contiguous()
        return self.theta64


def shard_batch(b: FrameBatch, rank: int, world: int) -> FrameBatch:
    """A rank's contiguous share of a key frame's rays (ray0 = their global id)."""
    sl = shard_rays(b.dirs.shape[0], rank, world)
    return replace(b, dirs=b.dirs[sl], gt_rgb=b.gt_rgb[sl], gt_depth=b.gt_depth[sl], mask_h=b.mask_h[sl],
                   mask_o=b.mask_o[sl], ray0=b.ray0 + sl.start)


class KeyFrame:
    """A key frame resident in HBM: its images at full resolution
    (rgb (H*W,3) f32, depth (H*W,) f32 with <= 0 = none, human/object masks u8),
    its camera and its motion prior / object pose. sample() draws a FrameBatch of
    training rays on the device (cf_keyframe_rays)."""

    def __init__(self, camera, rgb, depth, mask_h, mask_o, dqs, bone_A, dbias, theta, obj_R, obj_t):
        self.cam = _lib.Camera()
        Rf = np.asarray(camera.R, dtype=np.float64).reshape(9)
        for i in range(9):
            self.cam.R[i] = Rf[i]
        self.cam.fx, self.cam.fy = float(camera.fx), float(camera.fy)
        self.cam.cx, self.cam.cy = float(camera.cx), float(camera.cy)
        self.cam.width, self.cam.height = int(camera.width), int(camera.height)
        self.origin = np.asarray(camera.t, dtype=np.float64).reshape(3).copy()
        self.rgb = rgb.contiguous()
        self.depth = depth.contiguous()
        self.mask_h = mask_h.contiguous()
        self.mask_o = mask_o.contiguous()
        self.fg = torch.nonzero((self.mask_h | self.mask_o).view(-1)).view(-1).to(torch.int32)
        self.dqs, self.bone_A, self.theta, self.dbias = dqs, bone_A, theta, dbias
        self.theta64 = theta.to(torch.float64).contiguous() if theta is not None else None
        self.obj_R, self.obj_t = obj_R, obj_t

    def batch_buffers(self, n_rays: int) -> FrameBatch:
        d = self.rgb.device
        return FrameBatch(dqs=self.dqs, bone_A=self.bone_A, dbias=self.dbias, obj_R=self.obj_R, obj_t=self.obj_t,
                          dirs=torch.empty((n_rays, 3), dtype=torch.float64, device=d),
                          gt_rgb=torch.empty((n_rays, 3), dtype=torch.float32, device=d),
                          gt_depth=torch.empty(n_rays, dtype=torch.float32, device=d),
                          mask_h=torch.empty(n_rays, dtype=torch.uint8, device=d),
                          mask_o=torch.empty(n_rays, dtype=torch.uint8, device=d), theta=self.theta,
                          origin=self.origin, theta64=self.theta64)

    def draw(self, b: FrameBatch, seed: int, seed_offset: torch.Tensor | None = None) -> FrameBatch:
        """Fill b's rays (fresh pixels every call: seed, + *seed_offset on the device)."""
        n = b.dirs.shape[0]
        _lib.call("cf_keyframe_rays", _lib.byref(self.cam), self.fg.data_ptr(), int(self.fg.numel()), int(n),
                  ctypes.c_uint64(seed), seed_offset.data_ptr() if seed_offset is not None else None,
                  self.rgb.data_ptr(), self.depth.data_ptr(), self.mask_h.data_ptr(), self.mask_o.data_ptr(), None,
                  b.dirs.data_ptr(), b.gt_rgb.data_ptr(), b.gt_depth.data_ptr(), b.mask_h.data_ptr(),
                  b.mask_o.data_ptr(), _lib.stream_ptr())
        return b

    def sample(self, n_rays: int, seed: int) -> FrameBatch:
        return self.draw(self.batch_buffers(n_rays), seed)


def _pad16(x: int) -> int:
    return (x + 15) // 16 * 16


def _item(w, rows, cols, ldw, col0, transpose, blob, blob_lo):
    return _lib.PackItem(w.data_ptr(), blob, blob_lo, rows, cols, ldw, col0, transpose)


class ColorParams:
    """fp32 master weights of E_g/E_c on the device, their grads (views into the
    field's flat gradient bucket) and Adam moments; the fp16 forward / transposed
    blobs are repacked from them after every update (pack_items)."""

    def __init__(self, nets, device, grads: dict):
        self.nets = nets
        self.W = {k: torch.from_numpy(nets.layers[k].astype(np.float32)).to(device).contiguous() for k in COLOR_LAYERS}
        self.G = {k: grads[k] for k in COLOR_LAYERS}
        self.m = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.v = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.off = nets.w_bytes - 20480  # colour part of the forward blob (after DeformNet)
        self.wt_blob = torch.empty(20480, dtype=torch.uint8, device=device)

    def pack_items(self):
        it = []
        o = self.off
        for k in COLOR_LAYERS:  # forward blob: W (n_out x n_in) with its split residual
            w = self.W[k]
            n, kk = w.shape
            it.append(_item(w, n, kk, kk, 0, 0, self.nets.blob.data_ptr() + o, self.nets.blob_lo.data_ptr() + o))
            o += _pad16(n) * _pad16(kk) * 2
        o = 0
        for k in ("C3", "C2", "C1", "G2", "G1"):  # backward blob: W^T
            w = self.W[k]
            n, kk = w.shape
            it.append(_item(w, kk, n, kk, 0, 1, self.wt_blob.data_ptr() + o, None))
            o += _pad16(kk) * _pad16(n) * 2
        return it


class DeformParams:
    """fp32 master weights of DeformNet (D1 = [hash(32) | theta(72)] columns), their
    grads (views into the human field's bucket) and Adam moments."""

    def __init__(self, nets, device, grads: dict):
        self.nets = nets
        self.W = {k: torch.from_numpy(nets.layers[k].astype(np.float32)).to(device).contiguous() for k in DEFORM_LAYERS}
        self.W["D1"] = nets.d1  # shared with the renderer: its per-frame pose bias reads the trained W1
        self.G = {k: grads[k] for k in DEFORM_LAYERS}
        self.m = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.v = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.wt_blob = torch.empty(110592, dtype=torch.uint8, device=device)
        self.d1_tmp = torch.zeros((128, 48), dtype=torch.float32, device=device)  # [dW1 features | sum dpre1]

    def pack_items(self):
        W = self.W
        ld1 = int(W["D1"].shape[1])
        it = []
        o = 0
        for w, rows, cols, ldw in ((W["D1"], 128, 32, ld1), (W["D2"], 128, 128, 128), (W["D3"], 128, 128, 128),
                                   (W["D4"], 128, 128, 128), (W["D5"], 3, 128, 128)):
            it.append(_item(w, rows, cols, ldw, 0, 0, self.nets.blob.data_ptr() + o, self.nets.blob_lo.data_ptr() + o))
            o += _pad16(rows) * _pad16(cols) * 2
        o = 0
        for w, rows, cols, ldw in ((W["D5"], 128, 3, 128), (W["D4"], 128, 128, 128), (W["D3"], 128, 128, 128),
                                   (W["D2"], 128, 128, 128), (W["D1"], 32, 128, ld1)):
            it.append(_item(w, rows, cols, ldw, 0, 1, self.wt_blob.data_ptr() + o, None))
            o += _pad16(rows) * _pad16(cols) * 2
        return it


class _DeformBuffers:
    def __init__(self, cap, device):
        # feature-major (rows, capacity): the kernels' stores coalesce across samples and
        # the dW GEMMs read them K-major
        self.save_h = torch.empty((512, cap), dtype=torch.float16, device=device)
        self.save_o = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.save_mask = torch.empty((cap, 16), dtype=torch.int32, device=device)
        self.d_o = torch.empty((16, cap), dtype=torch.float16, device=device)
        self.dpre = torch.empty((512, cap), dtype=torch.float16, device=device)
        self.d_dfeat = torch.empty((cap, 32), dtype=torch.float32, device=device)
        self.dxc = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.io = _lib.DeformBwdIO(self.save_h.data_ptr(), self.save_o.data_ptr(), self.save_mask.data_ptr(),
                                   self.d_o.data_ptr(), self.dpre.data_ptr(), self.d_dfeat.data_ptr())


class _BwdBuffers:
    """E_g/E_c backward saves, feature-major (width, capacity) fp16."""

    def __init__(self, cap, device):
        h = lambda w: torch.empty((w, cap), dtype=torch.float16, device=device)  # noqa: E731
        self.h1, self.cin, self.c1, self.c2 = h(64), h(32), h(64), h(64)
        self.d_o, self.dc2, self.dc1, self.dg, self.dh1 = h(16), h(64), h(64), h(16), h(64)
        self.dfeat = torch.empty((cap, 32), dtype=torch.float32, device=device)
        self.grad = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.t = torch.empty(cap, dtype=torch.float64, device=device)
        self.io = _lib.ColorBwdIO(*[getattr(self, n).data_ptr() for n in
                                    ("h1", "cin", "c1", "c2", "d_o", "dc2", "dc1", "dg", "dh1", "dfeat")])


class _CompactBuffers:
    """A field's valid samples (flag > 0), compacted (cf_compact_valid): the field
    forward / backward run on these; vidx / inv map them to the full sample set the
    composite sees. (Human: samples no warp reaches; object: samples outside its box.)"""

    def __init__(self, cap, device):
        self.records = torch.empty(cap, dtype=torch.int32, device=device)
        self.counters = torch.zeros(4, dtype=torch.int32, device=device)
        self.xu = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.out = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.grad = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.vidx = torch.empty(cap, dtype=torch.int32, device=device)
        self.inv = torch.empty(cap, dtype=torch.int32, device=device)
        self.mo = _lib.MarchOut(self.records.data_ptr(), None, None, self.counters.data_ptr(), int(cap))


def _flat_bucket(shapes: dict, device) -> tuple[torch.Tensor, dict]:
    """One zeroed fp32 buffer holding every gradient of a field (the all-reduce bucket)."""
    total = sum(int(np.prod(s)) for s in shapes.values())
    flat = torch.zeros(total, dtype=torch.float32, device=device)
    views, o = {}, 0
    for k, s in shapes.items():
        n = int(np.prod(s))
        views[k] = flat[o:o + n].view(s)
        o += n
    return flat, views


class Trainer:
    """SPEC train_step for the human + object fields of a Renderer."""

    def __init__(self, renderer: Renderer, max_rays: int, cfg: TrainConfig | None = None):
        self.r = renderer
        self.cfg = cfg = cfg or TrainConfig()
        d = renderer.dirs.device
        self.device = d
        self.max_rays = int(max_rays)
        per_ray = max(cfg.n_guided + cfg.n_uniform, cfg.n_empty)
        cap = -(-self.max_rays * per_ray // 128) * 128  # whole 128-sample tiles (the saves' last K tile)
        self.cap = cap
        offs = (ctypes.c_int64 * 6)()
        _lib.call("cf_field_train_layout", cap, offs)
        self.layout = list(offs)
        self.fields = []
        for name, field in (("human", renderer.human), ("object", renderer.obj)):
            if field is None:
                continue
            deform = name == "human" and cfg.train_deform
            shapes = {"ctable": tuple(field.cgrid.table.shape)}
            shapes.update({k: tuple(field.nets.layers[k].shape) for k in COLOR_LAYERS})
            if deform:
                shapes["dtable"] = tuple(field.dgrid.table.shape)
                shapes.update({k: tuple(field.nets.layers[k].shape) for k in DEFORM_LAYERS})
            flat, g = _flat_bucket(shapes, d)
            buf = _FieldBuffers(self.max_rays, cap, d)
            buf.scratch = torch.empty(self.layout[5], dtype=torch.uint8, device=d)
            st = {"name": name, "q": _FIELD_INDEX[name], "field": field, "buf": buf, "bwd": _BwdBuffers(cap, d),
                  "flat": flat, "tgrad": g["ctable"], "params": ColorParams(field.nets, d, g),
                  "tm": torch.zeros_like(field.cgrid.table), "tv": torch.zeros_like(field.cgrid.table)}
            if deform:
                st["deform"] = DeformParams(field.nets, d, g)
                st["dbufs"] = _DeformBuffers(cap, d)
                st["dtgrad"] = g["dtable"]
                st["dtm"] = torch.zeros_like(field.dgrid.table)
                st["dtv"] = torch.zeros_like(field.dgrid.table)
                st["dbias"] = torch.empty(128, dtype=torch.float32, device=d)
            st["cbuf"] = _CompactBuffers(cap, d)
            self.fields.append(st)
        self.M = _lib.MarchDesc()
        ctypes.memmove(ctypes.byref(self.M), ctypes.byref(renderer.M), ctypes.sizeof(self.M))
        self.M.frame = None  # the trainer passes its frame (origin, object pose) by value
        # device-side step control
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=d)
        self.seed_dev = torch.zeros(1, dtype=torch.int64, device=d)
        self.adam_scale = torch.ones(2, dtype=torch.float32, device=d)
        self.stats = torch.zeros((2, 2), dtype=torch.float32, device=d)
        self.counts = None
        self.norms = None
        self.step_count = 0
        self.seed = 1234
        self._adam = None
        self._pack = None
        self._pack_weights()

    # -- per-step control ------------------------------------------------------

    def _ensure_frames(self, n_frames: int):
        if self.counts is None or self.counts.shape[0] != n_frames:
            self.counts = torch.zeros((n_frames, 4), dtype=torch.int32, device=self.device)
            self.norms = torch.zeros((2, n_frames, 4), dtype=torch.float32, device=self.device)

    def prepare(self, batches, group=None):
        """Count the masked / depth-valid rays of every frame, sum them over ranks
        (data parallel) and derive the step's normalisers and loss scales on the device."""
        self._ensure_frames(len(batches))
        s = _lib.stream_ptr()
        for f, b in enumerate(batches):
            n = int(b.dirs.shape[0])
            _lib.call("cf_train_counts", b.mask_h.data_ptr(), b.mask_o.data_ptr(), b.gt_depth.data_ptr(), n, 1,
                      max(n, 1), self.counts[f].data_ptr(), s)
        if _world(group) > 1:
            import torch.distributed as dist
            dist.all_reduce(self.counts, group=group)
        _lib.call("cf_train_norms", self.counts.data_ptr(), len(batches), self.norms.data_ptr(),
                  self.adam_scale.data_ptr(), self.stats.data_ptr(), self.step_dev.data_ptr(),
                  self.seed_dev.data_ptr(), s)

    def grad_scale(self, name: str) -> float:
        """The field's loss scale of the last prepared step (host read: tests / tools)."""
        return float(self.norms[_FIELD_INDEX[name], 0, 2])

    # -- one key frame -----------------------------------------------------------

    def _frame(self, f: int, b: FrameBatch, st):
        r, cfg, s = self.r, self.cfg, _lib.stream_ptr()
        buf, bwd, P = st["buf"], st["bwd"], st["params"]
        field, q = st["field"], st["q"]
        n_rays = int(b.dirs.shape[0])
        if n_rays > self.max_rays:
            raise ValueError("frame batch larger than max_rays")
        mask = b.mask_h if st["name"] == "human" else b.mask_o
        M = self.M
        M.n_rays = n_rays
        M.sample_t = None
        norm = self.norms[q, f].data_ptr()
        _lib.call("cf_train_sample", _lib.byref(M), b.gt_depth.data_ptr(), mask.data_ptr(), cfg.n_guided,
                  cfg.n_uniform, cfg.n_empty, cfg.depth_sigma, ctypes.c_uint64(self.seed + 7919 * f + 104729 * q),
                  self.seed_dev.data_ptr(), int(b.ray0), _lib.byref(buf.mo), bwd.t.data_ptr(), s)
        M.sample_t = bwd.t.data_ptr()
        dp = st.get("deform")
        dirs = b.dirs.data_ptr()
        if st["name"] == "human":
            _lib.call("cf_human_canon", _lib.byref(M), dirs, _lib.byref(buf.mo), _lib.byref(r.hw),
                      r._anchor_buckets.handle, field.lbs.buckets.handle, buf.xu.data_ptr(), s)
            desc = field.desc(r.dbias, "fp32")
            if dp is not None:
                if b.theta is None:
                    raise ValueError("DeformNet training needs FrameBatch.theta")
                # this frame's pose bias W1[:, 32:] theta from the current (trained) W1
                th = b.pose64()
                _lib.call("cf_pose_bias", dp.W["D1"].data_ptr(), int(dp.W["D1"].shape[1]), 32, 128, th.data_ptr(),
                          int(th.numel()), st["dbias"].data_ptr(), s)
                desc.dbias = st["dbias"].data_ptr()
                desc.save_h = st["dbufs"].save_h.data_ptr()
                desc.save_o = st["dbufs"].save_o.data_ptr()
                desc.save_mask = st["dbufs"].save_mask.data_ptr()
        else:
            _lib.call("cf_object_canon", _lib.byref(M), dirs, _lib.byref(buf.mo), buf.xu.data_ptr(), s)
            desc = field.desc("fp32")
        desc.train = 1  # 32-bit forward + the fp16 feature-major saves of the backward
        st["desc"] = desc
        scratch = buf.scratch.data_ptr()
        # the field runs on the compacted valid samples (human: reached by a warp; object:
        # inside its box), the composite on all of them
        cb = st.get("cbuf")
        if cb is not None:
            _lib.call("cf_compact_valid", _lib.byref(buf.mo), buf.xu.data_ptr(), _lib.byref(cb.mo), cb.xu.data_ptr(),
                      cb.vidx.data_ptr(), cb.inv.data_ptr(), s)
            fmo, fxu, fout, fgrad, fcount = cb.mo, cb.xu, cb.out, cb.grad, cb.counters
        else:
            fmo, fxu, fout, fgrad, fcount = buf.mo, buf.xu, buf.out, bwd.grad, buf.counters
        _lib.call("cf_field_forward", _lib.byref(desc), _lib.byref(fmo), dirs, fxu.data_ptr(), fout.data_ptr(), scratch,
                  s)
        if cb is not None:
            _lib.call("cf_scatter_rows", _lib.byref(buf.mo), cb.inv.data_ptr(), cb.out.data_ptr(), buf.out.data_ptr(), s)
        _lib.call("cf_loss_composite_bwd", _lib.byref(M), _lib.byref(buf.mo), buf.out.data_ptr(), r.cfg.t_term,
                  b.gt_rgb.data_ptr(), b.gt_depth.data_ptr(), mask.data_ptr(), cfg.lambda_depth, norm,
                  bwd.grad.data_ptr(), self.stats[q].data_ptr(), s)
        if cb is not None:
            _lib.call("cf_gather_rows", _lib.byref(cb.mo), cb.vidx.data_ptr(), bwd.grad.data_ptr(), cb.grad.data_ptr(),
                      s)
        _lib.call("cf_color_backward", _lib.byref(desc), P.wt_blob.data_ptr(), _lib.byref(fmo), dirs,
                  fxu.data_ptr(), fgrad.data_ptr(), scratch, _lib.byref(bwd.io), s)
        db = st.get("dbufs")
        _lib.call("cf_field_hash_backward", _lib.byref(desc), _lib.byref(fmo), fxu.data_ptr(), scratch,
                  bwd.dfeat.data_ptr(), st["tgrad"].data_ptr(), db.dxc.data_ptr() if dp is not None else None, s)
        if dp is not None:
            _lib.call("cf_deform_backward", _lib.byref(desc), dp.wt_blob.data_ptr(), _lib.byref(fmo),
                      fxu.data_ptr(), db.dxc.data_ptr(), _lib.byref(db.io), s)
            _lib.call("cf_deform_hash_backward", _lib.byref(desc), _lib.byref(fmo), fxu.data_ptr(),
                      db.d_dfeat.data_ptr(), st["dtgrad"].data_ptr(), s)
        # weight gradients dW = dY^T X over the field's samples: one grouped tcgen05
        # launch, both operands feature-major (K = samples), K read on the device
        probs = self._dw_problems(st)
        arr = (_lib.DwProblem * len(probs))(*probs)
        _lib.call("cf_dw_grouped", arr, len(probs), fcount.data_ptr(), self.cap, s)
        if dp is not None:
            # theta is the same for every sample of the frame: dW1[:, 32:] = (sum_s dpre1) theta^T
            th = b.theta
            _lib.call("cf_dw_pose_cols", dp.d1_tmp.data_ptr(), 128, 48, 32, th.data_ptr(), int(th.numel()),
                      dp.G["D1"].data_ptr(), int(dp.G["D1"].shape[1]), s)

    def _dw_problems(self, st):
        cap, bwd, G = self.cap, st["bwd"], st["params"].G
        x0 = st["buf"].scratch.data_ptr() + self.layout[0]  # canonical features (32, cap)

        def prob(A, ra, m, B, rb, n, C, ldc):  # K-blocked operands of ra / rb stored rows
            return _lib.DwProblem(A, ra, m, B, rb, n, C.data_ptr(), ldc)

        ps = [prob(bwd.dh1.data_ptr(), 64, 64, x0, 32, 32, G["G1"], 32),
              prob(bwd.dg.data_ptr(), 16, 16, bwd.h1.data_ptr(), 64, 64, G["G2"], 64),
              prob(bwd.dc1.data_ptr(), 64, 64, bwd.cin.data_ptr(), 32, 31, G["C1"], 31),
              prob(bwd.dc2.data_ptr(), 64, 64, bwd.c1.data_ptr(), 64, 64, G["C2"], 64),
              prob(bwd.d_o.data_ptr(), 16, 3, bwd.c2.data_ptr(), 64, 64, G["C3"], 64)]
        dp = st.get("deform")
        if dp is not None:
            db, GD = st["dbufs"], dp.G
            h = lambda l: db.save_h[128 * l].data_ptr()  # noqa: E731  h_{l+1}: K-blocked (128, cap)
            dpre = lambda l: db.dpre[128 * l].data_ptr()  # noqa: E731
            xd = st["buf"].scratch.data_ptr() + self.layout[1]  # [deform features | 1] (33, cap)
            ps += [prob(db.d_o.data_ptr(), 16, 3, h(3), 128, 128, GD["D5"], 128),
                   prob(dpre(3), 128, 128, h(2), 128, 128, GD["D4"], 128),
                   prob(dpre(2), 128, 128, h(1), 128, 128, GD["D3"], 128),
                   prob(dpre(1), 128, 128, h(0), 128, 128, GD["D2"], 128),
                   prob(dpre(0), 128, 128, xd, 33, 33, dp.d1_tmp, 48)]
        return ps

    def set_frame(self, b: FrameBatch):
        """The key frame's warp state (prior -> deformed nodes, LBS, live occupancy in the
        renderer's per-frame buffers) and its camera centre / object pose (by value in
        the trainer's own march descriptor: the renderer's frame block, i.e. its novel
        view, is never read)."""
        if b.origin is None:
            raise ValueError("FrameBatch.origin (the key frame's camera centre) is required")
        r = self.r
        r.load_prior(b.dqs, b.bone_A, b.dbias)
        r.prepare_frame()
        o = np.asarray(b.origin, dtype=np.float64).reshape(3)
        oR = np.asarray(b.obj_R, dtype=np.float64).reshape(9)
        ot = np.asarray(b.obj_t, dtype=np.float64).reshape(3)
        for a in range(3):
            self.M.origin[a] = o[a]
            self.M.obj_t[a] = ot[a]
        for a in range(9):
            self.M.obj_R[a] = oR[a]

    # -- the step ------------------------------------------------------------------

    def step(self, batches, group=None, update: bool = True):
        """One optimisation step over the key-frame batches -> {field: (L_color, L_depth)}
        (device tensors, means over the frames). Data parallel (torch.distributed
        initialised with world > 1, or `group`): the batches are this rank's shards; ray
        counts and gradient buckets are summed over ranks. update=False stops before
        Adam (the summed, loss-scaled gradients stay in the buckets)."""
        self.prepare(batches, group)
        world = _world(group)
        works = []
        saved = self.r._save_frame_state()
        try:
            for f, b in enumerate(batches):
                self.set_frame(b)
                for st in self.fields:
                    self._frame(f, b, st)
                    if world > 1 and f == len(batches) - 1:
                        works.append(_allreduce_async(st["flat"], group))
        finally:
            # the renderer's own frame (prior, pending setup) is back for its next view
            self.r._restore_frame_state(saved)
        for w in works:
            w.wait()
        self.step_count += 1
        if update:
            self._update()
        return {st["name"]: self.stats[st["q"]] for st in self.fields}

    def _update(self):
        """Adam over every trained tensor (one launch, grads zeroed) and the fp16 repack
        of the networks' weight blobs (one launch)."""
        cfg = self.cfg
        if self._adam is None:
            ts = []
            for st in self.fields:
                q = st["q"]
                t = st["field"].cgrid.table
                ts.append(_lib.AdamTensor(t.data_ptr(), st["tgrad"].data_ptr(), st["tm"].data_ptr(),
                                          st["tv"].data_ptr(), None, t.numel(), cfg.lr_hash, q))
                P = st["params"]
                for k in COLOR_LAYERS:
                    ts.append(_lib.AdamTensor(P.W[k].data_ptr(), P.G[k].data_ptr(), P.m[k].data_ptr(),
                                              P.v[k].data_ptr(), None, P.W[k].numel(), cfg.lr_net, q))
                if "deform" in st:
                    g = st["field"].dgrid
                    ts.append(_lib.AdamTensor(g.table.data_ptr(), st["dtgrad"].data_ptr(), st["dtm"].data_ptr(),
                                              st["dtv"].data_ptr(), g.table_f16.data_ptr() if g.read_half else None,
                                              g.table.numel(), cfg.lr_hash, q))
                    D = st["deform"]
                    for k in DEFORM_LAYERS:
                        ts.append(_lib.AdamTensor(D.W[k].data_ptr(), D.G[k].data_ptr(), D.m[k].data_ptr(),
                                                  D.v[k].data_ptr(), None, D.W[k].numel(), cfg.lr_net, q))
            self._adam = (_lib.AdamTensor * len(ts))(*ts)
        _lib.call("cf_adam_multi", self._adam, len(self._adam), cfg.beta1, cfg.beta2, cfg.eps,
                  self.step_dev.data_ptr(), self.adam_scale.data_ptr(), _lib.stream_ptr())
        self._pack_weights()

    def _pack_weights(self):
        if self._pack is None:
            items = []
            for st in self.fields:
                items += st["params"].pack_items()
                if "deform" in st:
                    items += st["deform"].pack_items()
            self._pack = (_lib.PackItem * len(items))(*items)
        _lib.call("cf_pack_multi", self._pack, len(self._pack), _lib.stream_ptr())

    def update_occupancy(self):
        """Refresh both fields' occupancy bits from their trained density (the renderer's
        march then skips what the field learned to be empty and keeps what it learned
        to fill, instead of the geometry-initialised grids); run every few steps,
        outside a captured step. The renderer's live occupancy is rebuilt with its next
        view."""
        dt = float(self.r.M.dt)
        for st in self.fields:
            W = st["params"].W
            st["field"].refresh_occupancy(W["G1"], W["G2"], dt)
        self.r._setup_pending = self.r.human is not None and getattr(self.r, "_dqs", None) is not None

    def set_learning_rates(self, lr_hash: float, lr_net: float):
        """New learning rates (the Adam launch table is rebuilt; a captured step must be
        captured again)."""
        self.cfg.lr_hash, self.cfg.lr_net = float(lr_hash), float(lr_net)
        self._adam = None

    # -- the captured step -----------------------------------------------------------

    def capture(self, keyframes, rays_per_frame: int, group=None):
        """CUDA-graph the whole step over `keyframes` — ray draw (fresh pixels and
        samples every replay: the seeds advance on the device), counts, forward,
        backward, dW, Adam, repack — and return a callable that replays it and returns
        the step's {field: (L_color, L_depth)} device tensors. The draw gives rank r the
        rays [r R, (r + 1) R) of each frame's global batch (R = rays_per_frame).
        Data-parallel capture needs an NCCL group (the collectives are captured with the
        kernels). The warm-up run before the capture is a real optimisation step."""
        world = _world(group)
        rank = 0
        if world > 1:
            import torch.distributed as dist
            if dist.get_backend(group) != "nccl":
                raise ValueError("Trainer.capture with world > 1 needs an NCCL process group")
            rank = dist.get_rank(group)
        bufs = [kf.batch_buffers(rays_per_frame) for kf in keyframes]
        for b in bufs:
            b.ray0 = rank * rays_per_frame

        def body():
            for f, (kf, b) in enumerate(zip(keyframes, bufs)):
                kf.draw(b, seed=(f * 64 + rank) * 1000003, seed_offset=self.seed_dev)
            return self.step(bufs, group)

        side = torch.cuda.Stream(device=self.device)  # warm-up: lazy state exists before the capture
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            body()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = body()

        def replay():
            g.replay()
            self.step_count += 1
            return out
        replay.graph = g
        return replay


def _world(group=None) -> int:
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 1
    return dist.get_world_size(group)


def _allreduce_async(flat: torch.Tensor, group=None):
    import torch.distributed as dist
    return dist.all_reduce(flat, group=group, async_op=True)


def sync_host_weights(trainer: "Trainer") -> None:
    """Copy the trained fp32 weights back into the FieldNets host arrays (the
    renderer's per-frame DeformNet pose bias is computed from them)."""
    for st in trainer.fields:
        nets = st["field"].nets
        for k, w in st["params"].W.items():
            nets.layers[k] = w.cpu().numpy().astype(np.float32)
        if "deform" in st:
            for k, w in st["deform"].W.items():
                nets.layers[k] = w.cpu().numpy().astype(np.float32)


def allreduce_grads(tensors, group=None):
    """Sum gradient buckets over ranks (NCCL on GPUs, gloo on CPU). The training loss
    is normalised by the GLOBAL ray counts (Trainer.prepare), so the sum is the
    global batch's gradient."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    for t in tensors:
        dist.all_reduce(t, group=group)


def shard_rays(n_rays: int, rank: int, world: int) -> slice:
    """Contiguous, balanced share of a global ray batch for one rank."""
    base, extra = divmod(n_rays, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))
