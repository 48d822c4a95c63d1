"""Key-frame training step on the GPU — SPEC train_step (
PAPER Eq. 8): depth-guided samples -> hybrid canonicalisation -> hash + tcgen05
MLP forward -> masked L2 colour + 0.1 L1 depth -> compositing backward ->
tcgen05 E_g/E_c backward -> hash-grid backward (atomics) -> Adam.

Human and object fields are updated independently on their own masked rays.
Round 1 trains the canonical hash grids and E_g/E_c of both fields; the human's
DeformNet (and its grid) are applied forward-only (frozen). The weight-gradient
reductions dW = dY^T X over the saved fp16 activations are plain GEMMs (cuBLAS via
torch.mm); every other step is a kernel of this package.

Multi-GPU: rays are sharded across ranks; `allreduce_grads` sums the flat
gradient buckets over NCCL (NVLink) and each rank applies the same Adam update.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .render import Renderer, _FieldBuffers

COLOR_LAYERS = ("G1", "G2", "C1", "C2", "C3")


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


class ColorParams:
    """fp32 master weights of E_g/E_c on the device, their grads and Adam moments;
    repacks the fp16 forward and transposed blobs after every update."""

    def __init__(self, nets, device):
        self.nets = nets
        self.W = {k: torch.from_numpy(nets.layers[k].astype(np.float32)).to(device).contiguous() for k in COLOR_LAYERS}
        self.G = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.m = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.v = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.off = nets.w_bytes - 20480  # colour part of the forward blob (after DeformNet)
        self.wt_blob = torch.empty(20480, dtype=torch.uint8, device=device)
        self.pack()

    def pack(self):
        s = _lib.stream_ptr()
        o = self.off
        for k in COLOR_LAYERS:
            w = self.W[k]
            n, kk = w.shape
            _lib.call("cf_pack_weight", w.data_ptr(), n, kk, self.nets.blob.data_ptr() + o, s)
            o += ((n + 15) // 16 * 16) * ((kk + 15) // 16 * 16) * 2
        o = 0
        for k in ("C3", "C2", "C1", "G2", "G1"):
            wt = self.W[k].t().contiguous()
            self._keep = getattr(self, "_keep", []) + [wt]
            n, kk = wt.shape
            _lib.call("cf_pack_weight", wt.data_ptr(), n, kk, self.wt_blob.data_ptr() + o, s)
            o += ((n + 15) // 16 * 16) * ((kk + 15) // 16 * 16) * 2
        self._keep = []

    def zero_grad(self):
        for g in self.G.values():
            g.zero_()


class _BwdBuffers:
    def __init__(self, cap, device):
        h = lambda w: torch.empty((cap, w), dtype=torch.float16, device=device)  # noqa: E731
        self.h1, self.cin, self.c1, self.c2 = h(64), h(32), h(64), h(64)
        self.d_o, self.dc2, self.dc1, self.dg, self.dh1 = h(16), h(64), h(64), h(16), h(64)
        self.dfeat = torch.empty((cap, 32), dtype=torch.float32, device=device)
        self.grad = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.t = torch.empty(cap, dtype=torch.float64, device=device)
        self.io = _lib.ColorBwdIO(*[getattr(self, n).data_ptr() for n in
                                    ("h1", "cin", "c1", "c2", "d_o", "dc2", "dc1", "dg", "dh1", "dfeat")])


class Trainer:
    """SPEC train_step for the human + object fields of a Renderer."""

    def __init__(self, renderer: Renderer, max_rays: int, cfg: TrainConfig | None = None):
        self.r = renderer
        self.cfg = cfg or TrainConfig()
        d = renderer.dirs.device
        self.max_rays = int(max_rays)
        cap = self.max_rays * max(self.cfg.n_guided + self.cfg.n_uniform, self.cfg.n_empty)
        self.fields = []
        for name, field in (("human", renderer.human), ("object", renderer.obj)):
            if field is None:
                continue
            st = {"name": name, "field": field, "buf": _FieldBuffers(self.max_rays, cap, d),
                  "bwd": _BwdBuffers(cap, d), "params": ColorParams(field.nets, d)}
            st["tgrad"] = torch.zeros_like(field.cgrid.table)
            st["tm"] = torch.zeros_like(field.cgrid.table)
            st["tv"] = torch.zeros_like(field.cgrid.table)
            self.fields.append(st)
        self.dirs = torch.empty((self.max_rays, 3), dtype=torch.float64, device=d)
        self.M = _lib.MarchDesc()
        ctypes.memmove(ctypes.byref(self.M), ctypes.byref(renderer.M), ctypes.sizeof(self.M))
        self.M.frame = None  # the trainer passes its frame (origin, object pose) by value
        self.loss = torch.zeros(2, dtype=torch.float32, device=d)
        self.step_count = 0
        self.seed = 1234

    # -- one key frame -----------------------------------------------------------

    def _frame(self, b: FrameBatch, st, stats):
        r, cfg, s = self.r, self.cfg, _lib.stream_ptr()
        buf, bwd, P = st["buf"], st["bwd"], st["params"]
        field = st["field"]
        n_rays = b.dirs.shape[0]
        mask = b.mask_h if st["name"] == "human" else b.mask_o
        n_m = int(mask.sum())
        if n_m == 0:
            return
        n_d = int(((b.gt_depth > 0) & (mask > 0)).sum())
        M = self.M
        M.n_rays = n_rays
        M.sample_t = None
        self.seed += 1
        _lib.call("cf_train_sample", _lib.byref(M), b.gt_depth.data_ptr(), mask.data_ptr(), cfg.n_guided,
                  cfg.n_uniform, cfg.n_empty, cfg.depth_sigma, ctypes.c_uint64(self.seed), _lib.byref(buf.mo),
                  bwd.t.data_ptr(), s)
        M.sample_t = bwd.t.data_ptr()
        if st["name"] == "human":
            _lib.call("cf_human_canon", _lib.byref(M), self.dirs.data_ptr(), _lib.byref(buf.mo), _lib.byref(r.hw),
                      r._anchor_buckets.handle, field.lbs.buckets.handle, buf.xu.data_ptr(), s)
            desc = r.hdesc
        else:
            _lib.call("cf_object_canon", _lib.byref(M), self.dirs.data_ptr(), _lib.byref(buf.mo), buf.xu.data_ptr(), s)
            desc = r.odesc
        scratch = r._scratch(buf, desc)
        _lib.call("cf_field_forward", _lib.byref(desc), _lib.byref(buf.mo), self.dirs.data_ptr(), buf.xu.data_ptr(),
                  buf.out.data_ptr(), scratch.data_ptr(), s)
        _lib.call("cf_loss_composite_bwd", _lib.byref(M), _lib.byref(buf.mo), buf.out.data_ptr(), r.cfg.t_term,
                  b.gt_rgb.data_ptr(), b.gt_depth.data_ptr(), mask.data_ptr(), cfg.lambda_depth, 1.0 / n_m,
                  1.0 / max(n_d, 1), bwd.grad.data_ptr(), stats.data_ptr(), s)
        _lib.call("cf_color_backward", _lib.byref(desc), P.wt_blob.data_ptr(), _lib.byref(buf.mo),
                  self.dirs.data_ptr(), buf.xu.data_ptr(), bwd.grad.data_ptr(), scratch.data_ptr(),
                  _lib.byref(bwd.io), s)
        _lib.call("cf_field_hash_backward", _lib.byref(desc), _lib.byref(buf.mo), buf.xu.data_ptr(),
                  scratch.data_ptr(), bwd.dfeat.data_ptr(), st["tgrad"].data_ptr(), s)
        # weight gradients dW = dY^T X over this frame's samples (plain GEMMs)
        n = int(buf.counters[0])
        if n == 0:
            return
        x0 = scratch[: n * 64].view(torch.float16).view(n, 32)
        # fp16 operands on the tensor cores, fp32 accumulation (reduced-precision
        # split-K reduction disabled), fp32 gradient accumulation across frames
        torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
        f = lambda t: t[:n]  # noqa: E731
        G = P.G
        G["C3"] += (f(bwd.d_o).t() @ f(bwd.c2)).float()[:3]
        G["C2"] += (f(bwd.dc2).t() @ f(bwd.c1)).float()
        G["C1"] += (f(bwd.dc1).t() @ f(bwd.cin)).float()[:, :31]
        G["G2"] += (f(bwd.dg).t() @ f(bwd.h1)).float()
        G["G1"] += (f(bwd.dh1).t() @ x0).float()

    def set_frame(self, b: FrameBatch):
        r = self.r
        r.load_prior(b.dqs, b.bone_A, b.dbias)
        r.set_object_pose(b.obj_R, b.obj_t)
        r.prepare_frame()
        n = b.dirs.shape[0]
        if n > self.max_rays:
            raise ValueError("frame batch larger than max_rays")
        self.dirs[:n].copy_(b.dirs)
        fr = r._frame_host  # origin[3], obj_R[9], obj_t[3] of the renderer's frame block
        for a in range(3):
            self.M.origin[a] = fr[a]
            self.M.obj_t[a] = fr[12 + a]
        for a in range(9):
            self.M.obj_R[a] = fr[3 + a]
        torch.cuda.current_stream().wait_event(r._lbs_done)

    def step(self, batches, allreduce=None):
        """One optimisation step over the key-frame batches -> {field: (L_color, L_depth)}."""
        out = {}
        for st in self.fields:
            st["tgrad"].zero_()
            st["params"].zero_grad()
            st["stats"] = torch.zeros(2, dtype=torch.float32, device=self.dirs.device)
        for b in batches:
            self.set_frame(b)
            for st in self.fields:
                self._frame(b, st, st["stats"])
        if allreduce is not None:
            allreduce([st["tgrad"] for st in self.fields] + [g for st in self.fields for g in st["params"].G.values()])
        self.step_count += 1
        cfg, s = self.cfg, _lib.stream_ptr()
        nb = float(len(batches))
        for st in self.fields:
            t = st["field"].cgrid.table
            _lib.call("cf_adam", t.data_ptr(), st["tgrad"].data_ptr(), st["tm"].data_ptr(), st["tv"].data_ptr(),
                      t.numel(), cfg.lr_hash, cfg.beta1, cfg.beta2, cfg.eps, self.step_count, 1.0 / nb, s)
            P = st["params"]
            for k in COLOR_LAYERS:
                _lib.call("cf_adam", P.W[k].data_ptr(), P.G[k].data_ptr(), P.m[k].data_ptr(), P.v[k].data_ptr(),
                          P.W[k].numel(), cfg.lr_net, cfg.beta1, cfg.beta2, cfg.eps, self.step_count, 1.0 / nb, s)
            P.pack()
            out[st["name"]] = st["stats"] / nb
        return out


def allreduce_grads(tensors, group=None):
    """Sum gradient buckets over ranks (NCCL on GPUs, gloo on CPU), then average."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, group=group)
    flat /= dist.get_world_size()
    o = 0
    for t in tensors:
        n = t.numel()
        t.copy_(flat[o:o + n].view_as(t))
        o += n


def shard_rays(n_rays: int, rank: int, world: int) -> slice:
    """Contiguous, balanced share of a global ray batch for one rank."""
    base, extra = divmod(n_rays, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))
