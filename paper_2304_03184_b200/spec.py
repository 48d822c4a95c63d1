"""The SPEC's call surface of stages 2-4 over the GPU
classes: hash_encode, canonicalize_human, volume_render, render_view, train_step and
composite with the SPEC's arguments and results. The work is the same CUDA path
the Renderer / Trainer run (csrc/render.cu, field.cu, train.cu); these functions
only stage the caller's rays / points as a sample batch. The reference package has
no code for these stages; the SPEC is the contract.

    hash_encode(grid, p)                          SPEC.md:363   (nrf.hash_encode)
    canonicalize_human(p_live, prior, knn, dnet)
    volume_render(field, rays)
    train_step(fields, batch, optimizer_state)
    render_view(fields, cam, prior, image_size)
    composite(human, object, background)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import dev, host, is_device
from .errors import OutOfSupportError
from .nrf import hash_encode  # noqa: F401  (SPEC hash_encode, re-exported)
from .render import Renderer, _FieldBuffers

__all__ = ["hash_encode", "canonicalize_human", "RaySample", "volume_render", "train_step", "render_view",
           "composite"]


@dataclass
class RaySample:
    """SPEC RaySample for a batch of rays from one centre: origin (3,),
    unit directions (R, 3), strictly increasing sample depths t (R, S), S <= 256."""
    origin: np.ndarray
    dirs: object
    t: object


def _batch(renderer: Renderer, dirs: torch.Tensor, t: torch.Tensor):
    """A compacted sample batch over R rays x S samples (record = ray << 8 | i), as
    the march writes it, with explicit depths (cf_march_desc.sample_t)."""
    R, S = t.shape
    if S > 256 or R >= (1 << 24):
        raise ValueError("at most 256 samples per ray and 2^24 rays")
    d = dirs.device
    buf = _FieldBuffers(R, R * S, d)
    ray = torch.arange(R, dtype=torch.int32, device=d)
    rec = (ray[:, None] << 8) | torch.arange(S, dtype=torch.int32, device=d)[None, :]
    buf.records.copy_(rec.reshape(-1))
    buf.ray_offset.copy_(ray * S)
    buf.ray_count.fill_(S)
    buf.counters.zero_()
    buf.counters[0] = R * S
    M = _lib.MarchDesc()
    ctypes.memmove(ctypes.byref(M), ctypes.byref(renderer.M), ctypes.sizeof(M))
    M.frame = None
    M.n_rays = R
    tt = t.reshape(-1).contiguous()
    M.sample_t = tt.data_ptr()
    return buf, M, tt


def canonicalize_human(p_live, prior, knn: Renderer, dnet=None, strict: bool = False):
    """SPEC canonicalize_human: p_t = the backward warp of the live
    points under the frame's motion prior, then p_canonical = p_t + dnet(hash_d(p_t) ⊕ θ).
    prior = (node_dqs (n,8), theta (72,), bone_A (24,4,4)); knn = the Renderer whose
    human field holds the warp structures (exact ED k-NN + DQB⁻¹ with the backward-LBS
    fallback); dnet = that HumanField (its DeformNet and deformation grid),
    or None for p_t. Returns (p_canonical (N,3) metres, valid (N,) bool); strict raises
    OutOfSupportError for a point no warp reaches (SPEC: out-of-support propagates)."""
    r = knn
    h = r.human
    on_dev = is_device(p_live)
    p = dev(p_live, shape_last=3)
    node_dqs, theta, bone_A = prior
    r.load_prior(dev(node_dqs, shape_last=8), dev(np.asarray(bone_A, dtype=np.float64)),
                 dev(h.nets.theta_bias(theta), dtype=torch.float32))
    r.prepare_frame()
    N = int(p.shape[0])
    if N == 0:
        out = torch.empty((0, 3), dtype=torch.float64, device=p.device)
        return (out, torch.empty(0, dtype=torch.bool, device=p.device)) if on_dev else (host(out), np.zeros(0, bool))
    # each point is a one-sample "ray" from the origin: p = 0 + 1 * p exactly
    buf, M, tt = _batch(r, p, torch.ones((N, 1), dtype=torch.float64, device=p.device))
    for a in range(3):
        M.origin[a] = 0.0
    s = _lib.stream_ptr()
    _lib.call("cf_human_canon", _lib.byref(M), p.data_ptr(), _lib.byref(buf.mo), _lib.byref(r.hw),
              r._anchor_buckets.handle, h.lbs.buckets.handle, buf.xu.data_ptr(), s)
    x = buf.xu
    if dnet is not None:
        desc = dnet.desc(r.dbias, "fp32")
        nb = ctypes.c_int64()
        _lib.call("cf_field_scratch_bytes", _lib.byref(desc), N, ctypes.byref(nb))
        scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=p.device)
        for stage in (0, 1):  # deformation-grid hash, DeformNet -> xc
            _lib.call("cf_field_stage", _lib.byref(desc), _lib.byref(buf.mo), p.data_ptr(), buf.xu.data_ptr(),
                      buf.out.data_ptr(), scratch.data_ptr(), stage, s)
        x = scratch[N * 256: N * 256 + N * 16].view(torch.float32).view(N, 4)  # precise layout: cfeat | dfeat | xc
    valid = x[:, 3] > 0
    pc = x[:, :3].double() / h.inv_side + torch.as_tensor(h.canon_min, dtype=torch.float64, device=p.device)
    pc = torch.where(valid[:, None], pc, torch.full_like(pc, float("nan")))
    if strict and not bool(valid.all()):
        raise OutOfSupportError("point outside the support of every warp")
    return (pc, valid) if on_dev else (host(pc), host(valid))


def volume_render(renderer: Renderer, rays: RaySample, field: str = "human"):
    """SPEC volume_render of one field of the renderer's current frame
    along caller-given rays: the field is evaluated at every sample (no occupancy
    skipping) and composited front to back: alpha_i = 1 - exp(-sigma_i delta_i),
    delta_i = t_{i+1} - t_i (the last: the renderer's spacing), rgb = sum T_i alpha_i c_i,
    depth = sum T_i alpha_i t_i / max(opacity, 1e-6), opacity = sum T_i alpha_i.
    Returns (rgb (R,3), depth (R,), opacity (R,)) f32."""
    r = renderer
    on_dev = is_device(rays.dirs)
    dirs = dev(rays.dirs, shape_last=3)
    t = dev(rays.t)
    if t.dim() != 2 or t.shape[0] != dirs.shape[0] or t.shape[1] < 2:
        raise ValueError("rays.t must be (R, S >= 2) for R rays")  # SPEC pre: >= 2 samples
    r.prepare_frame()
    buf, M, tt = _batch(r, dirs, t)
    o = np.asarray(rays.origin, dtype=np.float64).reshape(3)
    fr = r._frame_host  # the frame's object pose: obj_R [3:12], obj_t [12:15]
    for a in range(3):
        M.origin[a] = o[a]
        M.obj_t[a] = fr[12 + a]
    for a in range(9):
        M.obj_R[a] = fr[3 + a]
    s = _lib.stream_ptr()
    n = buf.mo.capacity
    if field == "human":
        h = r.human
        _lib.call("cf_human_canon", _lib.byref(M), dirs.data_ptr(), _lib.byref(buf.mo), _lib.byref(r.hw),
                  r._anchor_buckets.handle, h.lbs.buckets.handle, buf.xu.data_ptr(), s)
        desc = h.desc(r.dbias, "fp32")
    elif field == "object":
        _lib.call("cf_object_canon", _lib.byref(M), dirs.data_ptr(), _lib.byref(buf.mo), buf.xu.data_ptr(), s)
        desc = r.obj.desc("fp32")
    else:
        raise ValueError("field must be 'human' or 'object'")
    nb = ctypes.c_int64()
    _lib.call("cf_field_scratch_bytes", _lib.byref(desc), n, ctypes.byref(nb))
    scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=dirs.device)
    _lib.call("cf_field_forward", _lib.byref(desc), _lib.byref(buf.mo), dirs.data_ptr(), buf.xu.data_ptr(),
              buf.out.data_ptr(), scratch.data_ptr(), s)
    _lib.call("cf_composite", _lib.byref(M), _lib.byref(buf.mo), buf.out.data_ptr(), r.cfg.t_term,
              buf.rgb.data_ptr(), buf.depth.data_ptr(), buf.opacity.data_ptr(), s)
    out = (buf.rgb, buf.depth, buf.opacity)
    return out if on_dev else tuple(host(x) for x in out)


def render_view(renderer: Renderer, cam, prior=None, obj_pose=None):
    """SPEC render_view: full-frame march of both fields for camera
    `cam` (R, t, fx, fy, cx, cy; the renderer's image size), human rays canonicalised
    with the prior (node_dqs, theta, bone_A), object rays by the inverse object pose
    (R_o, t_o). Returns {"human": (rgb (H,W,3), depth (H,W), opacity (H,W)),
    "object": (...), "image": the composite (H,W,3)} as numpy arrays."""
    r = renderer
    if prior is not None:
        node_dqs, theta, bone_A = prior
        R_o, t_o = obj_pose if obj_pose is not None else (np.eye(3), np.zeros(3))
        r.set_frame(node_dqs, theta, bone_A, R_o, t_o)
    img = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    torch.cuda.current_stream().synchronize()
    H, W = r.rows, r.W
    out = {"image": host(img).reshape(H, W, 3)}
    for name, b in (("human", r.hb), ("object", r.ob)):
        if b is not None:
            out[name] = (host(b.rgb).reshape(H, W, 3), host(b.depth).reshape(H, W), host(b.opacity).reshape(H, W))
    return out


def train_step(trainer, batch):
    """SPEC train_step: one Adam step of both fields on the key-frame
    ray batches -> {field: (L_color, L_depth)} (means over the frames)."""
    out = trainer.step(batch)
    return {k: tuple(float(x) for x in v.cpu()) for k, v in out.items()}


def composite(human, obj, background):
    """SPEC composite: per pixel the layer with the smaller depth
    among those with opacity > 0.5 wins, else the background. human / obj = (rgb (N,3),
    depth (N,), opacity (N,)) (any leading shape), background = rgb 3-vector."""
    shp = np.shape(human[1])
    n = int(np.prod(shp)) if len(shp) else 1
    hr, hd, ho = (dev(x, dtype=torch.float32).reshape(n, -1) for x in human)
    orr_, od, oo = (dev(x, dtype=torch.float32).reshape(n, -1) for x in obj)
    bg = (ctypes.c_float * 3)(*[float(v) for v in background])
    out = torch.empty((n, 3), dtype=torch.float32, device=hr.device)
    layer = torch.empty(n, dtype=torch.uint8, device=hr.device)
    _lib.call("cf_composite_layers", n, hr.data_ptr(), hd.data_ptr(), ho.data_ptr(), orr_.data_ptr(), od.data_ptr(),
              oo.data_ptr(), bg, out.data_ptr(), layer.data_ptr(), _lib.stream_ptr())
    return host(out).reshape(*shp, 3)
