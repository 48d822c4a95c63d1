"""The SPEC call surface of stages 2-4 (paper_2304_03184_b200/spec.py) on the B200,
checked with the SPEC's own examples."""
import numpy as np
import pytest
import torch

from oracle import deform as od
from paper_2304_03184_b200 import spec
from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
from paper_2304_03184_b200.scene import Scene, SceneConfig
from paper_2304_03184_b200.train import FrameBatch, Trainer, TrainConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world():
    sc = Scene(SceneConfig(width=64, height=64), seed=0)
    cfg = RenderConfig(n_samples=64)
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, zero_deform_out=True,
                    table_scale=0.5)
    of = ObjectField(sc.box_half, cfg, table_scale=0.5)
    r = Renderer(hf, of, 64, 64, cfg)
    return sc, cfg, hf, of, r


def _prior(sc, fid):
    return sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid)


def test_canonicalize_identity_motion_zero_dnet(world):
    """identity motion + zero-initialised DeformNet output -> p_canonical = p_live
    (to the fp32 unit-cube coordinates the field works in)."""
    sc, cfg, hf, of, r = world
    n = len(sc.nodes)
    ident = np.zeros((n, 8))
    ident[:, 0] = 1.0
    rng = np.random.default_rng(0)
    p = sc.nodes[rng.integers(0, n, 3000)] + rng.normal(scale=0.02, size=(3000, 3))
    A0 = np.broadcast_to(np.eye(4), (24, 4, 4)).copy()
    pc, valid = spec.canonicalize_human(p, (ident, np.zeros(72), A0), r, hf)
    assert valid.mean() > 0.99
    assert np.abs(pc[valid] - p[valid]).max() <= 2e-6 * hf.side


def test_canonicalize_zero_dnet_is_the_warp(world):
    """zero-initialised DeformNet output -> p_canonical = p_t, the backward warp
    (SPEC.md:377), here checked against the oracle's exact ED warp."""
    sc, cfg, hf, of, r = world
    fid = 6
    rng = np.random.default_rng(1)
    anchors = od.deformed_nodes(sc.nodes, sc.node_dqs(fid))
    p = anchors[rng.integers(0, len(anchors), 2000)] + rng.normal(scale=0.02, size=(2000, 3))
    pt, valid_t = spec.canonicalize_human(p, _prior(sc, fid), r, None)
    pc, valid = spec.canonicalize_human(p, _prior(sc, fid), r, hf)
    assert np.array_equal(valid, valid_t) and np.array_equal(pt[valid], pc[valid])
    _, _, ref, ov = od.warp(sc.nodes, 0.1, 4, sc.node_dqs(fid), p, "backward")
    ed = valid & ov
    assert ed.mean() > 0.9
    assert np.abs(pc[ed] - ref[ed]).max() <= 2e-6 * hf.side  # fp32 unit-cube coordinates


def test_canonicalize_strict_out_of_support(world):
    sc, cfg, hf, of, r = world
    far = np.array([[50.0, 50.0, 50.0], sc.nodes[0]])
    pc, valid = spec.canonicalize_human(far, _prior(sc, 0), r, hf)
    assert not valid[0] and valid[1] and np.isnan(pc[0]).all()
    with pytest.raises(spec.OutOfSupportError):
        spec.canonicalize_human(far, _prior(sc, 0), r, hf, strict=True)


def test_volume_render_empty_and_render_view(world):
    """sigma = 0 (rays that miss the human: no sample in any warp's support) -> rgb 0,
    opacity 0; render_view's per-field layers composite to its image."""
    sc, cfg, hf, of, r = world
    fid = 3
    cam = sc.camera
    out = spec.render_view(r, cam, _prior(sc, fid), sc.object_pose(fid))
    img = spec.composite(out["human"], out["object"], cfg.background)
    assert np.array_equal(img, out["image"])
    # rays pointing away from the scene
    o = np.asarray(cam.t, dtype=np.float64)
    dirs = np.tile(-np.asarray(cam.R, dtype=np.float64)[2], (16, 1))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    t = np.tile(np.linspace(0.3, 5.0, 32), (16, 1))
    rgb, depth, op = spec.volume_render(r, spec.RaySample(o, dirs, t), "human")
    assert np.array_equal(rgb, np.zeros_like(rgb)) and np.array_equal(op, np.zeros_like(op))


def test_volume_render_matches_the_view(world):
    """volume_render along the camera's own rays, with the depths of the samples the
    march kept for them, reproduces the view's human layer (same kernels; rays whose
    kept samples are consecutive, so delta_i = t_{i+1} - t_i is the march's spacing)."""
    sc, cfg, hf, of, r = world
    fid = 5
    cam = sc.camera
    out = spec.render_view(r, cam, _prior(sc, fid), sc.object_pose(fid))
    _, dirs = cam.all_rays()
    hb = r.hb
    off, cnt = hb.ray_offset.cpu().numpy(), hb.ray_count.cpu().numpy()
    rec = hb.records[:int(hb.counters[0])].cpu().numpy().view(np.uint32)
    cand = {}
    for ray in np.nonzero(cnt >= 4)[0]:
        i = (rec[off[ray]:off[ray] + cnt[ray]] & 255).astype(np.int64)
        if i[-1] - i[0] == len(i) - 1:
            cand.setdefault(len(i), []).append((ray, i))
    S, rays = max(cand.items(), key=lambda kv: len(kv[1]))
    assert len(rays) >= 10
    ids = np.array([q for q, _ in rays])
    dt = (cfg.t_far - cfg.t_near) / cfg.n_samples
    t = np.stack([cfg.t_near + (i + 0.5) * dt for _, i in rays])  # the march's t_i (same float64 ops)
    rgb, depth, op = spec.volume_render(r, spec.RaySample(cam.t, dirs[ids], t), "human")
    h_rgb, h_depth, h_op = (x.reshape(len(dirs), -1)[ids] for x in out["human"])
    assert np.allclose(op, h_op[:, 0], atol=1e-5) and np.allclose(rgb, h_rgb, atol=1e-5)
    assert np.allclose(depth, h_depth[:, 0], rtol=1e-5)


def test_composite_examples():
    """nearer opaque layer wins, both transparent -> background."""
    bg = (0.1, 0.2, 0.3)
    h = (np.array([[1, 0, 0], [1, 0, 0], [1, 0, 0]], float), np.array([1.0, 3.0, 1.0]), np.array([0.9, 0.9, 0.2]))
    o = (np.array([[0, 1, 0], [0, 1, 0], [0, 1, 0]], float), np.array([2.0, 2.0, 0.5]), np.array([0.9, 0.9, 0.3]))
    img = spec.composite(h, o, bg)
    assert np.allclose(img[0], [1, 0, 0]) and np.allclose(img[1], [0, 1, 0]) and np.allclose(img[2], bg)


def test_train_step_masked_out_and_separation(world):
    """all mask bits 0 -> losses 0 and parameters unchanged; human-only rays leave the
    object field bit-identical."""
    sc, cfg, hf, of, r = world
    fid = 2
    o, d = sc.camera.all_rays()
    th, to, rgb, hum, obj = sc.raycast(o, d, fid)
    R, t = sc.object_pose(fid)
    T = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")  # noqa: E731

    def batch(mh, mo):
        depth = np.where(hum, th, np.where(obj, to, 0.0))
        return FrameBatch(dqs=T(sc.node_dqs(fid), torch.float64), bone_A=T(sc.bone_transforms(fid), torch.float64),
                          dbias=T(hf.nets.theta_bias(sc.theta(fid)), torch.float32), obj_R=R, obj_t=t,
                          theta=T(sc.theta(fid), torch.float32), dirs=T(d, torch.float64),
                          gt_rgb=T(rgb, torch.float32), gt_depth=T(depth, torch.float32),
                          mask_h=T(mh, torch.uint8), mask_o=T(mo, torch.uint8), origin=np.asarray(sc.camera.t))
    tr = Trainer(r, max_rays=len(d), cfg=TrainConfig())
    snap = lambda f: [f.cgrid.table.clone(), f.nets.blob.clone()]  # noqa: E731
    h0, o0 = snap(hf), snap(of)
    losses = spec.train_step(tr, [batch(np.zeros_like(hum), np.zeros_like(obj))])
    assert losses == {"human": (0.0, 0.0), "object": (0.0, 0.0)}
    assert all(torch.equal(a, b) for a, b in zip(h0 + o0, snap(hf) + snap(of)))
    losses = spec.train_step(tr, [batch(hum, np.zeros_like(obj))])
    assert losses["human"][0] > 0 and losses["object"] == (0.0, 0.0)
    assert not torch.equal(h0[0], hf.cgrid.table)
    assert all(torch.equal(a, b) for a, b in zip(o0, snap(of)))
