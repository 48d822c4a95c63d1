"""SPEC gradient invariant (acceptance 4) on the oracle:
the 64-bit analytic gradients of the training loss (oracle/grad.py) match central
finite differences (perturbation 1e-5) within 1e-3 relative on a 16-ray probe
batch, for the canonical and deformation hash tables, E_g / E_c and DeformNet.
CPU only; the device training kernels are compared against these gradients in
tests/test_train_gpu.py::test_device_gradients_vs_f64_oracle."""
import numpy as np
import pytest
import torch

from oracle import deform as od
from oracle import grad as og
from oracle import render as orr
from paper_2304_03184_b200.scene import Scene, SceneConfig

H = 1e-5
RTOL = 1e-3


def kaiming(rng, n_out, n_in):
    b = np.sqrt(6.0 / n_in)
    return rng.uniform(-b, b, size=(n_out, n_in))


def probe_params(rng, total_c, total_d):
    P = {"ctable": rng.uniform(-0.3, 0.3, size=(total_c, 2)), "dtable": rng.uniform(-0.3, 0.3, size=(total_d, 4)),
         "G1": kaiming(rng, 64, 32), "G2": kaiming(rng, 16, 64), "C1": kaiming(rng, 64, 31),
         "C2": kaiming(rng, 64, 64), "C3": kaiming(rng, 3, 64), "D1": kaiming(rng, 128, 104),
         "D2": kaiming(rng, 128, 128), "D3": kaiming(rng, 128, 128), "D4": kaiming(rng, 128, 128),
         "D5": kaiming(rng, 3, 128) * 0.3}
    P["G2"][0] *= 4.0  # a denser field: visible opacity on the probe rays
    return {k: v.astype(np.float32).astype(np.float64) for k, v in P.items()}


def probe_batch(n_rays=16, n_samples=48, fid=7, seed=0):
    """16 rays through the human of frame fid, samples in +-12 cm of the surface,
    canonicalised with the oracle's hybrid warp; targets from the analytic ray cast."""
    sc = Scene(SceneConfig(width=64, height=64), seed=0)
    o, d = sc.camera.all_rays()
    th, to, rgb, hum, obj = sc.raycast(o, d, fid)
    rng = np.random.default_rng(seed)
    rays = rng.choice(np.nonzero(hum)[0], n_rays, replace=False)
    side = 1.0
    nodes = np.asarray(sc.nodes)
    lo, hi = nodes.min(0), nodes.max(0)
    side = float((hi - lo).max() + 2 * 0.15)
    cmin = (lo + hi) / 2 - side / 2
    t = np.sort(th[rays][:, None] + rng.uniform(-0.12, 0.12, size=(n_rays, n_samples)), axis=1)
    ray = np.repeat(np.arange(n_rays), n_samples)
    tt = t.reshape(-1)
    delta = np.concatenate([np.append(np.diff(t[r]), 0.24 / n_samples) for r in range(n_rays)])
    p = np.asarray(sc.camera.t)[None] + tt[:, None] * d[rays][ray]
    xu = orr.human_canon(p, nodes, sc.node_dqs(fid), 4, 0.1, sc.bone_transforms(fid), sc.skin_verts,
                         sc.skin_weights, 0.2, cmin, 1.0 / side)
    return sc, {"xu": xu, "dirs": d[rays][ray], "ray": ray, "t": tt, "delta": delta, "gt_rgb": rgb[rays],
                "gt_depth": th[rays].astype(np.float32), "mask": np.ones(n_rays, np.uint8), "inv_side": 1.0 / side,
                "theta": sc.theta(fid).astype(np.float32)}


@pytest.fixture(scope="module")
def probe():
    from oracle import nrf as on
    sc, batch = probe_batch()
    _, tc = on.hash_levels(16, 19, 16, 2048)
    _, td = on.hash_levels(8, 17, 16, 256)
    params = probe_params(np.random.default_rng(1), tc, td)
    assert (batch["xu"][:, 3] > 0).mean() > 0.3
    L, g = og.gradients(params, batch)
    return params, batch, L, g


def _central(params, batch, name, idx):
    p = {k: (v.copy() if k == name else v) for k, v in params.items()}
    x0 = p[name][idx]
    p[name][idx] = x0 + H
    lp = og.loss_value(p, batch)
    p[name][idx] = x0 - H
    lm = og.loss_value(p, batch)
    return (lp - lm) / (2 * H)


@pytest.mark.parametrize("name,count", [("ctable", 6), ("dtable", 6), ("G1", 3), ("G2", 3), ("C1", 3), ("C2", 3),
                                        ("C3", 3), ("D1", 4), ("D2", 3), ("D3", 3), ("D4", 3), ("D5", 3)])
def test_analytic_matches_central_differences(probe, name, count):
    params, batch, L, g = probe
    assert L > 0
    flat = np.abs(g[name]).reshape(-1)
    assert flat.max() > 0, name
    for f in np.argsort(flat)[::-1][:count]:
        idx = np.unravel_index(f, g[name].shape)
        fd = _central(params, batch, name, idx)
        an = g[name][idx]
        assert abs(fd - an) <= RTOL * abs(an), (name, idx, fd, an)


def test_pose_columns_of_deformnet_have_gradient(probe):
    params, batch, L, g = probe
    assert np.abs(g["D1"][:, 32:]).max() > 0  # theta enters layer 1


def test_oracle_loss_matches_numpy_composite(probe):
    """The autograd loss's compositing = oracle/render.composite (float64)."""
    params, batch, L, g = probe
    with torch.no_grad():
        P = og.as_params(params, requires_grad=False)
        sigma, rgb = og.field_t(P, batch["xu"], batch["dirs"], batch["inv_side"], batch["theta"])
    R = len(batch["gt_rgb"])
    out = np.zeros(R)
    op = np.zeros(R)
    rgbc = np.zeros((R, 3))
    for r in range(R):
        sel = batch["ray"] == r
        T = 1.0
        for s, c, dl in zip(sigma.numpy()[sel], rgb.numpy()[sel], batch["delta"][sel]):
            a = 1.0 - np.exp(-s * dl)
            rgbc[r] += T * a * c
            op[r] += T * a
            T *= 1.0 - a
    lc = ((rgbc - batch["gt_rgb"]) ** 2).sum(1).mean()
    assert abs(og.loss_value(params, batch, color_only=True) - lc) <= 1e-12 * max(1.0, lc)
    assert 0.05 < op.mean() < 1.0
