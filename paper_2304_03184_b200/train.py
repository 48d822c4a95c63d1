"""Key-frame training step on the GPU — SPEC train_step (
PAPER Eq. 8): depth-guided samples -> hybrid canonicalisation -> hash + tcgen05
MLP forward -> masked L2 colour + 0.1 L1 depth -> compositing backward ->
tcgen05 E_g/E_c backward -> hash-grid backward (atomics) -> Adam.

Human and object fields are updated independently on their own masked rays.
Trained: the canonical hash grids and E_g/E_c of both fields, and the human's
DeformNet with its deformation grid (TrainConfig.train_deform): the canonical
hash backward also returns dL/dxc (spatial gradient of the trilinear
interpolation), which flows through xc = xu + 0.05 tanh(o) / side into the
tcgen05 DeformNet backward and on into the deformation-grid hash backward. The
weight-gradient reductions dW = dY^T X over the saved fp16 activations are plain
GEMMs (cuBLAS via torch.mm); every other step is a kernel of this package.

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
        self.obj_R, self.obj_t = obj_R, obj_t

    def sample(self, n_rays: int, seed: int) -> FrameBatch:
        d = self.rgb.device
        dirs = torch.empty((n_rays, 3), dtype=torch.float64, device=d)
        rgb = torch.empty((n_rays, 3), dtype=torch.float32, device=d)
        depth = torch.empty(n_rays, dtype=torch.float32, device=d)
        mh = torch.empty(n_rays, dtype=torch.uint8, device=d)
        mo = torch.empty(n_rays, dtype=torch.uint8, device=d)
        _lib.call("cf_keyframe_rays", _lib.byref(self.cam), self.fg.data_ptr(), int(self.fg.numel()), int(n_rays),
                  ctypes.c_uint64(seed), self.rgb.data_ptr(), self.depth.data_ptr(), self.mask_h.data_ptr(),
                  self.mask_o.data_ptr(), None, dirs.data_ptr(), rgb.data_ptr(), depth.data_ptr(), mh.data_ptr(),
                  mo.data_ptr(), _lib.stream_ptr())
        return FrameBatch(dqs=self.dqs, bone_A=self.bone_A, dbias=self.dbias, obj_R=self.obj_R, obj_t=self.obj_t,
                          dirs=dirs, gt_rgb=rgb, gt_depth=depth, mask_h=mh, mask_o=mo, theta=self.theta,
                          origin=self.origin)


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
            _lib.call("cf_pack_weight_split", w.data_ptr(), n, kk, self.nets.blob.data_ptr() + o,
                      self.nets.blob_lo.data_ptr() + o, s)
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


DEFORM_LAYERS = ("D1", "D2", "D3", "D4", "D5")


class DeformParams:
    """fp32 master weights of DeformNet (D1 = [hash(32) | theta(72)] columns), their
    grads and Adam moments; repacks the forward blob's DeformNet part and the
    transposed blob of the backward kernel after every update."""

    def __init__(self, nets, device):
        self.nets = nets
        self.W = {k: torch.from_numpy(nets.layers[k].astype(np.float32)).to(device).contiguous() for k in DEFORM_LAYERS}
        self.W["D1"] = nets.d1  # shared with the renderer: its per-frame pose bias reads the trained W1
        self.G = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.m = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.v = {k: torch.zeros_like(v) for k, v in self.W.items()}
        self.wt_blob = torch.empty(110592, dtype=torch.uint8, device=device)
        self.pack()

    def bias(self, theta: torch.Tensor) -> torch.Tensor:
        """Per-frame layer-1 pose term W1[:, 32:] @ theta (fp32, device)."""
        return (self.W["D1"][:, 32:] @ theta.to(self.W["D1"].device, torch.float32)).contiguous()

    def pack(self):
        s = _lib.stream_ptr()
        mats = [self.W["D1"][:, :32].contiguous(), self.W["D2"], self.W["D3"], self.W["D4"], self.W["D5"]]
        o = 0
        for w in mats:
            n, kk = w.shape
            _lib.call("cf_pack_weight_split", w.data_ptr(), n, kk, self.nets.blob.data_ptr() + o,
                      self.nets.blob_lo.data_ptr() + o, s)
            o += ((n + 15) // 16 * 16) * ((kk + 15) // 16 * 16) * 2
        keep = [self.W["D5"].t().contiguous(), self.W["D4"].t().contiguous(), self.W["D3"].t().contiguous(),
                self.W["D2"].t().contiguous(), self.W["D1"][:, :32].t().contiguous()]
        o = 0
        for wt in keep:
            n, kk = wt.shape
            _lib.call("cf_pack_weight", wt.data_ptr(), n, kk, self.wt_blob.data_ptr() + o, s)
            o += ((n + 15) // 16 * 16) * ((kk + 15) // 16 * 16) * 2

    def zero_grad(self):
        for g in self.G.values():
            g.zero_()


class _DeformBuffers:
    def __init__(self, cap, device):
        # feature-major (512, capacity): the kernels' stores coalesce across samples
        self.save_h = torch.empty((512, cap), dtype=torch.float16, device=device)
        self.save_o = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.save_mask = torch.empty((cap, 16), dtype=torch.int32, device=device)
        self.d_o = torch.empty((cap, 16), dtype=torch.float16, device=device)
        self.dpre = torch.empty((512, cap), dtype=torch.float16, device=device)
        self.d_dfeat = torch.empty((cap, 32), dtype=torch.float32, device=device)
        self.dxc = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.io = _lib.DeformBwdIO(self.save_h.data_ptr(), self.save_o.data_ptr(), self.save_mask.data_ptr(),
                                   self.d_o.data_ptr(),
                                   self.dpre.data_ptr(), self.d_dfeat.data_ptr())


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
            if name == "human" and self.cfg.train_deform:
                st["deform"] = DeformParams(field.nets, d)
                st["dbufs"] = _DeformBuffers(cap, d)
                st["dtgrad"] = torch.zeros_like(field.dgrid.table)
                st["dtm"] = torch.zeros_like(field.dgrid.table)
                st["dtv"] = torch.zeros_like(field.dgrid.table)
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
        dp = st.get("deform")
        if st["name"] == "human":
            _lib.call("cf_human_canon", _lib.byref(M), self.dirs.data_ptr(), _lib.byref(buf.mo), _lib.byref(r.hw),
                      r._anchor_buckets.handle, field.lbs.buckets.handle, buf.xu.data_ptr(), s)
            # the training forward: DeformNet at 32-bit semantics with the fp16 saves the
            # fp16 backward consumes (cf_field_forward with save_h in the "fp32" mode)
            desc = field.desc(r.dbias, "fp32" if dp is not None else "fp16")
            if dp is not None:
                # this frame's pose bias from the current W1, forward saves on
                if b.theta is None:
                    raise ValueError("DeformNet training needs FrameBatch.theta")
                st["dbias"] = dp.bias(b.theta)
                desc.dbias = st["dbias"].data_ptr()
                desc.save_h = st["dbufs"].save_h.data_ptr()
                desc.save_o = st["dbufs"].save_o.data_ptr()
                desc.save_mask = st["dbufs"].save_mask.data_ptr()
        else:
            _lib.call("cf_object_canon", _lib.byref(M), self.dirs.data_ptr(), _lib.byref(buf.mo), buf.xu.data_ptr(), s)
            desc = field.desc("fp16")
        scratch = r._scratch(buf, desc)
        _lib.call("cf_field_forward", _lib.byref(desc), _lib.byref(buf.mo), self.dirs.data_ptr(), buf.xu.data_ptr(),
                  buf.out.data_ptr(), scratch.data_ptr(), s)
        if st.get("gscale") is None:
            st["gscale"] = loss_scale(n_m)
        _lib.call("cf_loss_composite_bwd", _lib.byref(M), _lib.byref(buf.mo), buf.out.data_ptr(), r.cfg.t_term,
                  b.gt_rgb.data_ptr(), b.gt_depth.data_ptr(), mask.data_ptr(), cfg.lambda_depth, 1.0 / n_m,
                  1.0 / max(n_d, 1), st["gscale"], bwd.grad.data_ptr(), stats.data_ptr(), s)
        _lib.call("cf_color_backward", _lib.byref(desc), P.wt_blob.data_ptr(), _lib.byref(buf.mo),
                  self.dirs.data_ptr(), buf.xu.data_ptr(), bwd.grad.data_ptr(), scratch.data_ptr(),
                  _lib.byref(bwd.io), s)
        db = st.get("dbufs")
        _lib.call("cf_field_hash_backward", _lib.byref(desc), _lib.byref(buf.mo), buf.xu.data_ptr(),
                  scratch.data_ptr(), bwd.dfeat.data_ptr(), st["tgrad"].data_ptr(),
                  db.dxc.data_ptr() if dp is not None else None, s)
        if dp is not None:
            _lib.call("cf_deform_backward", _lib.byref(desc), dp.wt_blob.data_ptr(), _lib.byref(buf.mo),
                      buf.xu.data_ptr(), db.dxc.data_ptr(), _lib.byref(db.io), s)
            _lib.call("cf_deform_hash_backward", _lib.byref(desc), _lib.byref(buf.mo), buf.xu.data_ptr(),
                      db.d_dfeat.data_ptr(), st["dtgrad"].data_ptr(), s)
        # weight gradients dW = dY^T X over this frame's samples (plain GEMMs)
        n = int(buf.counters[0])
        if n == 0:
            return
        # The GEMM row count is rounded up to one of 8 sizes per power of two (within
        # the buffers) so that frames with different sample counts reuse cuBLASLt's
        # cached plans (a new shape costs ~4 ms of host-side heuristics); the padding
        # rows of both operands are zeroed, so they add nothing (zero dY alone is not
        # enough: stale X rows may hold inf/NaN bit patterns, and 0 * NaN = NaN).
        q = 1 << max(n.bit_length() - 4, 10)
        cap = buf.mo.capacity
        n_pad = min(-(-n // q) * q, cap)
        pads = [bwd.d_o, bwd.dc2, bwd.dc1, bwd.dg, bwd.dh1, bwd.c2, bwd.c1, bwd.cin, bwd.h1]
        pads += [scratch[n * 64: n_pad * 64]]  # colour-MLP input rows (x0 below)
        if dp is not None:
            pads += [db.d_o, scratch[cap * 64 + n * 64: cap * 64 + n_pad * 64]]
            db.dpre[:, n:n_pad].zero_()
            db.save_h[:, n:n_pad].zero_()
        for t in pads:
            (t[n:n_pad] if t.dim() == 2 else t).zero_()
        n, n_true = n_pad, n
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
        if dp is not None:
            xd = scratch[cap * 64: cap * 64 + n * 64].view(torch.float16).view(n, 32)  # deform-grid features
            H, DP, DO = db.save_h[:, :n], db.dpre[:, :n], db.d_o[:n]  # H, DP feature-major
            GD = dp.G
            GD["D5"] += (DO.t() @ H[384:512].t()).float()[:3]
            # dW_l = dpre_l h_{l-1}^T over the frame's samples: both operands feature-major
            # (K = samples contiguous), split-K on tcgen05 accumulating into the fp32 grads
            ld = db.save_h.stride(0)
            for l, key in ((3, "D4"), (2, "D3"), (1, "D2")):
                _lib.call("cf_gemm_kmajor_f16", db.dpre[128 * l].data_ptr(), ld, db.save_h[128 * (l - 1)].data_ptr(),
                          ld, 128, n, GD[key].data_ptr(), 128, s)
            GD["D1"][:, :32] += (DP[0:128] @ xd).float()
            # theta is the same for every sample of the frame: dW1_theta = (sum_s dpre1) theta^T
            csum = DP[0:128, :n_true].sum(1, dtype=torch.float32)
            GD["D1"][:, 32:] += torch.outer(csum, b.theta.to(DP.device, torch.float32))

    def set_frame(self, b: FrameBatch):
        """The key frame's warp state (prior -> deformed nodes, LBS, live occupancy in the
        renderer's per-frame buffers) and its camera centre / object pose (by value in
        the trainer's own march descriptor: the renderer's frame block, i.e. its novel
        view, is never read)."""
        if b.origin is None:
            raise ValueError("FrameBatch.origin (the key frame's camera centre) is required")
        r = self.r
        n = b.dirs.shape[0]
        if n > self.max_rays:
            raise ValueError("frame batch larger than max_rays")
        r.load_prior(b.dqs, b.bone_A, b.dbias)
        r.prepare_frame()
        self.dirs[:n].copy_(b.dirs)
        o = np.asarray(b.origin, dtype=np.float64).reshape(3)
        oR = np.asarray(b.obj_R, dtype=np.float64).reshape(9)
        ot = np.asarray(b.obj_t, dtype=np.float64).reshape(3)
        for a in range(3):
            self.M.origin[a] = o[a]
            self.M.obj_t[a] = ot[a]
        for a in range(9):
            self.M.obj_R[a] = oR[a]
        torch.cuda.current_stream().wait_event(r._lbs_done)

    def step(self, batches, allreduce=None):
        """One optimisation step over the key-frame batches -> {field: (L_color, L_depth)}."""
        out = {}
        for st in self.fields:
            st["tgrad"].zero_()
            st["params"].zero_grad()
            if "deform" in st:
                st["dtgrad"].zero_()
                st["deform"].zero_grad()
            st["stats"] = torch.zeros(2, dtype=torch.float32, device=self.dirs.device)
        for st in self.fields:  # one loss scale per field and step (every frame's grads add up)
            mk = [b.mask_h if st["name"] == "human" else b.mask_o for b in batches]
            st["gscale"] = loss_scale(min(int(m.sum()) for m in mk))
        saved = self.r._save_frame_state()
        try:
            for b in batches:
                self.set_frame(b)
                for st in self.fields:
                    self._frame(b, st, st["stats"])
        finally:
            # the renderer's own frame (prior, pending setup) is back for its next view
            self.r._restore_frame_state(saved)
        if allreduce is not None:
            bufs = [st["tgrad"] for st in self.fields] + [g for st in self.fields for g in st["params"].G.values()]
            for st in self.fields:
                if "deform" in st:
                    bufs += [st["dtgrad"]] + list(st["deform"].G.values())
            allreduce(bufs)
        self.step_count += 1
        cfg, s = self.cfg, _lib.stream_ptr()
        nb = float(len(batches))
        for st in self.fields:
            unscale = 1.0 / (nb * st["gscale"])  # mean over frames, loss scale divided out
            t = st["field"].cgrid.table
            _lib.call("cf_adam", t.data_ptr(), st["tgrad"].data_ptr(), st["tm"].data_ptr(), st["tv"].data_ptr(),
                      t.numel(), cfg.lr_hash, cfg.beta1, cfg.beta2, cfg.eps, self.step_count, unscale, s)
            st["field"].cgrid.refresh_f16()
            P = st["params"]
            for k in COLOR_LAYERS:
                _lib.call("cf_adam", P.W[k].data_ptr(), P.G[k].data_ptr(), P.m[k].data_ptr(), P.v[k].data_ptr(),
                          P.W[k].numel(), cfg.lr_net, cfg.beta1, cfg.beta2, cfg.eps, self.step_count, unscale, s)
            P.pack()
            if "deform" in st:
                t = st["field"].dgrid.table
                _lib.call("cf_adam", t.data_ptr(), st["dtgrad"].data_ptr(), st["dtm"].data_ptr(), st["dtv"].data_ptr(),
                          t.numel(), cfg.lr_hash, cfg.beta1, cfg.beta2, cfg.eps, self.step_count, unscale, s)
                st["field"].dgrid.refresh_f16()
                D = st["deform"]
                for k in DEFORM_LAYERS:
                    _lib.call("cf_adam", D.W[k].data_ptr(), D.G[k].data_ptr(), D.m[k].data_ptr(), D.v[k].data_ptr(),
                              D.W[k].numel(), cfg.lr_net, cfg.beta1, cfg.beta2, cfg.eps, self.step_count, unscale,
                              s)
                D.pack()
            out[st["name"]] = st["stats"] / nb
        return out


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


def loss_scale(n_masked: int) -> float:
    """Power-of-two loss scale of a field's backward: the per-sample gradients of the
    1/n-normalised loss are O(1/n); scaled by 2^floor(log2 n) they are O(1), inside
    the fp16 range of the backward's tensor-core operands (no subnormal underflow)."""
    return float(2.0 ** max(0, int(np.floor(np.log2(max(1, n_masked))))))


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
