"""ORACLE (test infrastructure only) — 64-bit analytic gradients of the key-frame
training loss (SPEC train_step: masked L2 colour + lambda L1 depth)
with respect to every trained parameter: both hash tables, E_g / E_c and DeformNet
(incl. its pose columns). float64 torch autograd on the CPU over the oracle's field
(oracle/render.py: deform_forward, deformed_coords, color_forward, composite), with
the hash corner selection recomputed in float64.

Pinned by SPEC's gradient invariant (acceptance 4 SPEC.md:607): the
analytic gradient matches central finite differences (perturbation 1e-5, 64-bit)
within 1e-3 relative on a 16-ray probe batch — tests/test_oracle_grad.py. The device
training kernels are then compared against these gradients (tests/test_train_gpu.py).
"""
from __future__ import annotations

import numpy as np
import torch

from . import nrf as on
from .render import sh16

CANON = (16, 2, 19, 16, 2048)
DEFORM = (8, 4, 17, 16, 256)
PRIMES = (1, 2654435761, 805459861)


def hash_encode_t(table, x, grid, cell32=False):
    """Trilinear multi-resolution hash features of x (N,3) in
    float64 torch, differentiable in table and x; corner choice as hash_corners."""
    L, F, log2T, nmin, nmax = grid
    levels, _ = on.hash_levels(L, log2T, nmin, nmax)
    mask = (1 << log2T) - 1
    xc = torch.clamp(x, 0.0, 1.0)
    feats = []
    for N, dense, off in levels:
        pos = xc * float(N)
        if cell32:
            # the cell chosen from the fp32 product, as the kernels and oracle/nrf.py do
            # (DESIGN 4's fp32 position): an f64 product can land on the other side of a
            # cell face, where the interpolant's normal derivative jumps (device checks)
            p32 = (xc.detach().to(torch.float32) * torch.tensor(float(N), dtype=torch.float32)).to(x.dtype)
        else:  # exact cell: the interpolant is continuous (finite-difference checks)
            p32 = pos.detach()
        g = torch.minimum(torch.floor(p32), torch.tensor(float(N - 1), dtype=x.dtype))
        fr = pos - g
        gi = g.to(torch.int64)
        f = 0
        for k in range(8):
            b = (k & 1, (k >> 1) & 1, (k >> 2) & 1)
            c = [gi[:, a] + b[a] for a in range(3)]
            if dense:
                idx = c[0] + c[1] * (N + 1) + c[2] * (N + 1) ** 2
            else:
                idx = ((c[0] * PRIMES[0]) ^ (c[1] * PRIMES[1]) ^ (c[2] * PRIMES[2])) & 0xFFFFFFFF & mask
            w = 1
            for a in range(3):
                w = w * (fr[:, a] if b[a] else 1.0 - fr[:, a])
            f = f + w[:, None] * table[off + idx]
        feats.append(f)
    return torch.cat(feats, 1)


def _mlp(x, Ws, bias=None):
    h = x
    for l, W in enumerate(Ws):
        h = h @ W.t()
        if l == 0 and bias is not None:
            h = h + bias
        if l < len(Ws) - 1:
            h = torch.relu(h)
    return h


def field_t(params, xu, dirs, inv_side, theta=None, keep=None, xc_value=None, cell32=False):
    """(sigma, rgb) of samples xu (N,4: unit coords + flag) as float64 torch. keep: an
    optional dict that receives the intermediates fd, o, xc, fc (gradients retained);
    xc_value: optional (N,3) canonical positions to evaluate the canonical grid at;
    cell32: choose hash cells from the fp32 product as the device does."""
    x = torch.as_tensor(xu[:, :3], dtype=torch.float64)
    if "dtable" in params:
        fd = hash_encode_t(params["dtable"], x, DEFORM, cell32)
        th = torch.as_tensor(theta, dtype=torch.float64)
        D1 = params["D1"]
        o = _mlp(fd, [D1[:, :32], params["D2"], params["D3"], params["D4"], params["D5"]], D1[:, 32:] @ th)
        x = x + 0.05 * torch.tanh(o[:, :3]) * inv_side
        if xc_value is not None:
            # evaluate the canonical grid at given positions (the device forward's xc),
            # gradients still flowing through the deformation: the trilinear interpolant's
            # normal derivative jumps across cell faces, so the backward is compared where
            # the forward put the sample (xc itself is checked by the forward parity tests)
            x = torch.as_tensor(np.asarray(xc_value), dtype=torch.float64) + (x - x.detach())
        if keep is not None:
            keep.update(fd=fd, o=o)
    fc = hash_encode_t(params["ctable"], x, CANON, cell32)
    if keep is not None:
        keep.update(xc=x, fc=fc)
        for v in keep.values():
            if v.requires_grad:
                v.retain_grad()
    g = _mlp(fc, [params["G1"], params["G2"]])
    sigma = torch.exp(g[:, 0])
    sh = torch.as_tensor(sh16(np.asarray(dirs)), dtype=torch.float64)
    c = _mlp(torch.cat([g[:, 1:16], sh], 1), [params["C1"], params["C2"], params["C3"]])
    rgb = torch.sigmoid(c[:, :3])
    valid = torch.as_tensor(xu[:, 3] > 0)
    return sigma * valid, rgb * valid[:, None]


def loss_t(params, batch, lam=0.1, color_only=False):
    """Masked L2 colour + lam L1 depth over the probe rays (normalised by the masked /
    depth-valid ray counts, as cf_loss_composite_bwd). batch: dict with xu (N,4), dirs
    (N,3), ray (N,), t (N,) sorted per ray, delta (N,), gt_rgb (R,3), gt_depth (R,),
    mask (R,), inv_side, theta."""
    sigma, rgb = field_t(params, batch["xu"], batch["dirs"], batch["inv_side"], batch.get("theta"),
                         batch.get("keep"), batch.get("xc_value"), batch.get("cell32", False))
    ray = torch.as_tensor(batch["ray"])
    t = torch.as_tensor(batch["t"], dtype=torch.float64)
    delta = torch.as_tensor(batch["delta"], dtype=torch.float64)
    R = len(batch["gt_rgb"])
    tau = sigma * delta
    alpha = 1.0 - torch.exp(-tau)
    # T_i = exp(-sum_{j<i} sigma_j delta_j) per ray (samples grouped per ray)
    logT = -tau
    starts = np.searchsorted(batch["ray"], np.arange(R))
    ends = np.searchsorted(batch["ray"], np.arange(R), side="right")
    parts = []
    for a, b in zip(starts, ends):
        seg = logT[a:b]
        parts.append(torch.cat([seg.new_zeros(1), torch.cumsum(seg, 0)[:-1]]) if b > a else seg)
    cum = torch.cat(parts)
    w = torch.exp(cum) * alpha
    out = torch.zeros((R, 5), dtype=torch.float64).index_add(0, ray, torch.stack(
        [w * rgb[:, 0], w * rgb[:, 1], w * rgb[:, 2], w * t, w], 1))
    mask = torch.as_tensor(batch["mask"] > 0)
    gt = torch.as_tensor(batch["gt_rgb"], dtype=torch.float64)
    n_m = max(int(mask.sum()), 1)
    lc = (((out[:, :3] - gt) ** 2).sum(1) * mask).sum() / n_m
    if color_only:
        return lc
    gd = torch.as_tensor(batch["gt_depth"], dtype=torch.float64)
    dm = mask & (gd > 0)
    n_d = max(int(dm.sum()), 1)
    depth = out[:, 3] / torch.clamp(out[:, 4], min=1e-6)
    ld = (torch.abs(depth - gd) * dm).sum() / n_d
    return lc + lam * ld


def as_params(tables_and_layers, requires_grad=True):
    return {k: torch.tensor(np.asarray(v, dtype=np.float64), requires_grad=requires_grad)
            for k, v in tables_and_layers.items()}


def gradients(values, batch, **kw):
    """{name: dL/dname} (float64 numpy) at the parameter values `values`."""
    P = as_params(values)
    L = loss_t(P, batch, **kw)
    L.backward()
    return float(L.detach()), {k: p.grad.numpy() for k, p in P.items()}


def loss_value(values, batch, **kw):
    with torch.no_grad():
        return float(loss_t(as_params(values, requires_grad=False), batch, **kw))
