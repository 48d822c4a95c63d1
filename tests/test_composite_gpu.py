"""The device compositing kernel (cf_composite, render.cu composite_kernel) on
SPEC volume_render's worked examples and invariants (
acceptance 5), fed synthetic density sequences directly:

  sigma == 0                      -> rgb 0, opacity 0
  constant sigma over length l    -> opacity = 1 - exp(-sigma l) within 1e-5
  near-opaque thin slab at t*     -> depth within one sample spacing of t*
  telescoping sum T_i a_i + T_end = 1 within 1e-6 (random densities)
and against the float64 oracle composite on random rays (1e-5).
"""
import numpy as np
import pytest
import torch

from oracle import render as orr
from paper_2304_03184_b200 import _lib

pytestmark = pytest.mark.gpu

T_NEAR, T_FAR, S = 0.3, 5.0, 128


def device_composite(sigma, rgb=None, t_term=0.0):
    """sigma (R, S) -> device (rgb, depth, opacity) with every sample of every ray."""
    sigma = np.asarray(sigma, dtype=np.float32)
    R = sigma.shape[0]
    field = np.zeros((R * S, 4), dtype=np.float32)
    field[:, 0] = sigma.reshape(-1)
    field[:, 1:] = (0.2, 0.5, 0.9) if rgb is None else np.asarray(rgb, np.float32).reshape(-1, 3)
    d = torch.device("cuda")
    ray = np.repeat(np.arange(R), S)
    i = np.tile(np.arange(S), R)
    rec = torch.from_numpy(((ray << 8) | i).astype(np.int32)).to(d)
    off = torch.from_numpy((np.arange(R) * S).astype(np.int32)).to(d)
    cnt = torch.full((R,), S, dtype=torch.int32, device=d)
    counters = torch.tensor([R * S, 0, 0, 0], dtype=torch.int32, device=d)
    mo = _lib.MarchOut(rec.data_ptr(), off.data_ptr(), cnt.data_ptr(), counters.data_ptr(), R * S)
    M = _lib.MarchDesc()
    M.n_rays, M.n_samples, M.t_near, M.t_far = R, S, T_NEAR, T_FAR
    M.dt = (T_FAR - T_NEAR) / S
    f = torch.from_numpy(field).to(d)
    out_rgb = torch.empty((R, 3), dtype=torch.float32, device=d)
    depth = torch.empty(R, dtype=torch.float32, device=d)
    op = torch.empty(R, dtype=torch.float32, device=d)
    _lib.call("cf_composite", _lib.byref(M), _lib.byref(mo), f.data_ptr(), t_term, out_rgb.data_ptr(),
              depth.data_ptr(), op.data_ptr(), _lib.stream_ptr())
    torch.cuda.synchronize()
    return out_rgb.cpu().numpy(), depth.cpu().numpy(), op.cpu().numpy(), (ray, i, field, M.dt)


def test_zero_density():
    rgb, depth, op, _ = device_composite(np.zeros((4, S)))
    assert (rgb == 0).all() and (op == 0).all()


def test_constant_density_analytic():
    sig = np.array([0.05, 0.5, 1.0, 1.9], dtype=np.float32)
    rgb, depth, op, (_, _, _, dt) = device_composite(np.repeat(sig[:, None], S, 1))
    ell = S * dt
    assert np.abs(op - (1.0 - np.exp(-sig.astype(np.float64) * ell))).max() <= 1e-5


def test_thin_slab_depth():
    dt = (T_FAR - T_NEAR) / S
    stars = np.array([0.9, 2.35, 4.1])
    sig = np.zeros((3, S), np.float32)
    for r, t_star in enumerate(stars):
        sig[r, int((t_star - T_NEAR) / dt)] = 5e3
    rgb, depth, op, _ = device_composite(sig)
    assert (op > 0.999).all() and np.abs(depth - stars).max() <= dt


def test_telescoping_and_oracle():
    rng = np.random.default_rng(5)
    sig = (rng.exponential(0.3, (256, S)) * (rng.random((256, S)) < 0.5)).astype(np.float32)
    cols = rng.random((256 * S, 3)).astype(np.float32)
    rgb, depth, op, (ray, i, field, dt) = device_composite(sig, cols)
    a = 1.0 - np.exp(-sig.astype(np.float64) * float(np.float32(dt)))
    T_end = np.prod(1.0 - a, axis=1)
    assert np.abs(op + T_end - 1.0).max() <= 1e-6
    ref_rgb, ref_depth, ref_op = orr.composite(256, ray, i, field, T_NEAR, dt, t_term=0.0)
    assert np.abs(rgb - ref_rgb).max() <= 1e-5 and np.abs(op - ref_op).max() <= 1e-5
    ok = ref_op > 1e-3
    assert np.allclose(depth[ok], ref_depth[ok], rtol=1e-5)
