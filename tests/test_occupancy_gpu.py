"""Occupancy refresh from the trained density (cf_density_grid_update):
the per-cell density logits and the occupancy decisions (max-decay update,
threshold, box dilation) bit-exact against oracle/render.py, and the render march
driven by the refreshed bits instead of the geometry-initialised shell."""
import numpy as np
import pytest
import torch

from oracle import render as orr
from paper_2304_03184_b200 import _lib
from paper_2304_03184_b200.nrf import HashGrid, HashGridConfig
from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
from paper_2304_03184_b200.scene import Scene, SceneConfig

pytestmark = pytest.mark.gpu


def _update(grid, W1, W2, res, logits, log_decay, log_thr, dilate):
    bits = torch.empty(res ** 3 // 32, dtype=torch.int32, device="cuda")
    scratch = torch.empty_like(bits)
    _lib.call("cf_density_grid_update", _lib.byref(grid.desc), grid.table.data_ptr(), W1.data_ptr(), W2.data_ptr(),
              res, log_decay, log_thr, dilate, logits.data_ptr(), bits.data_ptr(), scratch.data_ptr(),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    return orr.unpack_bits(bits.cpu().numpy(), res ** 3)


@pytest.mark.parametrize("dilate", [0, 1, 3])
def test_density_grid_bitexact(dilate):
    res = 32
    rng = np.random.default_rng(5)
    grid = HashGrid(HashGridConfig(), init_scale=0.5, seed=3)
    W1 = torch.from_numpy(rng.normal(scale=0.4, size=(64, 32)).astype(np.float32)).cuda()
    W2 = torch.from_numpy(rng.normal(scale=0.3, size=(16, 64)).astype(np.float32)).cuda()
    logits = torch.full((res ** 3,), float("-inf"), dtype=torch.float32, device="cuda")
    log_decay, log_thr = float(np.log(0.95)), 0.35
    # first update from -inf: g = g0
    got = _update(grid, W1, W2, res, logits, log_decay, log_thr, dilate)
    g0 = orr.density_logits(grid.table.cpu().numpy(), W1.cpu().numpy(), W2.cpu().numpy(), res)
    ref_g, ref_on = orr.density_grid_update(np.full(res ** 3, -np.inf, np.float32), g0, log_decay, log_thr, res,
                                            dilate)
    assert np.array_equal(logits.cpu().numpy(), ref_g)
    assert np.array_equal(got, ref_on)
    assert 0.05 < (ref_g > np.float32(log_thr)).mean() < 0.95  # a real mix of (undilated) decisions
    # second update after the field changed: the max-decay keeps the old density where it was higher
    prev = logits.cpu().numpy()
    grid.table.mul_(0.5)
    W2[0].mul_(-1.0)
    got = _update(grid, W1, W2, res, logits, log_decay, log_thr, dilate)
    g0 = orr.density_logits(grid.table.cpu().numpy(), W1.cpu().numpy(), W2.cpu().numpy(), res)
    ref_g, ref_on = orr.density_grid_update(prev, g0, log_decay, log_thr, res, dilate)
    assert np.array_equal(logits.cpu().numpy(), ref_g)
    assert np.array_equal(got, ref_on)
    assert (ref_g >= prev + np.float32(log_decay)).all()


def test_refresh_drives_the_march():
    """A field the training made empty renders no human sample at all; one made dense
    everywhere marches far more samples than the geometry shell allowed."""
    sc = Scene(SceneConfig(width=96, height=96), seed=0)
    cfg = RenderConfig(n_samples=64)
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, table_scale=0.1)
    of = ObjectField(sc.box_half, cfg, table_scale=0.1)
    r = Renderer(hf, of, 96, 96, cfg)
    fid = 4
    cam = sc.camera

    def frame():
        r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), *sc.object_pose(fid))
        r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
        torch.cuda.synchronize()
        return r.sample_counts()

    h0, o0 = frame()
    assert h0 > 0 and o0 > 0
    rng = np.random.default_rng(1)
    W1 = torch.from_numpy(rng.normal(scale=1.0, size=(64, 32)).astype(np.float32)).cuda()
    W2 = torch.zeros((16, 64), dtype=torch.float32, device="cuda")
    W2[0] = -100.0  # sigma <= 1 / m everywhere: below the occupancy threshold
    hf.refresh_occupancy(W1, W2, r.M.dt)
    of.refresh_occupancy(W1, W2, r.M.dt)
    assert not orr.unpack_bits(hf.canon_bits.cpu().numpy(), cfg.canon_occ_res ** 3).any()
    assert frame() == (0, 0)
    W2[0] = 100.0  # dense wherever any hidden unit fires: nearly everywhere
    hf.refresh_occupancy(W1, W2, r.M.dt)
    of.refresh_occupancy(W1, W2, r.M.dt)
    h2, o2 = frame()
    assert h2 > 2 * h0 and o2 > o0
