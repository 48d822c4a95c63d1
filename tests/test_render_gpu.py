"""Render path parity on the B200 (C1 frame: 64x64 rays, 64 samples/ray, 128 ED
nodes + 6890 skin verts, 16-level 2^19 grid), stage by stage against the
oracle fed with the previous stage's device output:
  occupancy bits, march sample sets, ED/LBS flags      bit-exact
  canonical coordinates (float32)                      ED: bit-exact; LBS: 1e-6
  field sigma / rgb ("fp16" mode: fp16 tensor-core     see FIELD_* below
  operands) vs the kernel-precision oracle             (the "fp32" mode: test_precision_gpu.py)
  composite rgb / opacity / depth                      1e-5 abs
  layer choice                                         bit-exact
"""
import numpy as np
import pytest
import torch

from oracle import deform as od
from oracle import render as orr
from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
from paper_2304_03184_b200.scene import Scene, SceneConfig

pytestmark = pytest.mark.gpu

FIELD_RGB_ATOL = 2e-3     # fp16 activations: one-ulp flips of intermediate rounding
FIELD_SIGMA_RTOL = 2e-2


def words(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.fixture(scope="module")
def setup():
    sc = Scene(SceneConfig(width=64, height=64), seed=0)
    cfg = RenderConfig(n_samples=64, precision="fp16")
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, seed=0, zero_deform_out=False,
                    table_scale=0.5)
    of = ObjectField(sc.box_half, cfg, seed=1, table_scale=0.5)
    for f, s in ((hf, 6.0), (of, 14.0)):  # denser random fields so both layers win somewhere
        f.nets.layers["G2"][0] *= s
        f.nets.repack()
    r = Renderer(hf, of, 64, 64, cfg)
    fid = 7
    R, t = sc.object_pose(fid)
    r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), R, t)
    cam = sc.camera
    img = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    torch.cuda.synchronize()
    r.check_overflow()
    return sc, cfg, hf, of, r, fid, img


def field_samples(buf):
    n = int(buf.counters[0])
    rec = buf.records[:n].cpu().numpy().view(np.uint32)
    return n, (rec >> 8).astype(np.int64), (rec & 255).astype(np.int64)


def test_rays(setup):
    sc, cfg, hf, of, r, fid, img = setup
    _, d = sc.camera.all_rays()
    assert np.allclose(r.dirs.cpu().numpy(), d, rtol=0, atol=1e-15)


def test_occupancy_bits_bitexact(setup):
    sc, cfg, hf, of, r, fid, img = setup
    g = hf.canon_occ
    on = orr.occ_from_points(sc.template_points, list(g.min), g.cell, g.res, cfg.canon_occ_radius)
    got = orr.unpack_bits(words(hf.canon_bits), g.res ** 3)
    assert np.array_equal(got, on) and on.sum() > 1000
    og = of.occ
    ob = orr.occ_box_shell(list(og.min), og.cell, og.res, sc.box_half, cfg.obj_shell)
    assert np.array_equal(orr.unpack_bits(words(of.bits), og.res ** 3), ob)
    lg = r.live_occ
    live = orr.occ_splat(got, (list(g.min), g.cell, g.res), sc.nodes, sc.node_dqs(fid), cfg.ed_k, cfg.ed_radius,
                         (list(lg.min), lg.cell, lg.res))
    assert np.array_equal(orr.unpack_bits(words(r.live_bits), lg.res ** 3), live)
    f = np.nonzero(live)[0]
    ijk = np.stack([f // lg.res ** 2, (f // lg.res) % lg.res, f % lg.res], -1)
    assert list(r.live_bbox.cpu().numpy()) == list(ijk.min(0)) + list(ijk.max(0))


def test_march_sets_bitexact(setup):
    sc, cfg, hf, of, r, fid, img = setup
    dirs = r.dirs.cpu().numpy()
    lg, og = r.live_occ, of.occ
    R, t = sc.object_pose(fid)
    ref = orr.march(sc.camera.t, dirs, cfg.n_samples, cfg.t_near, r.M.dt,
                    orr.unpack_bits(words(r.live_bits), lg.res ** 3), (list(lg.min), lg.cell, lg.res),
                    orr.unpack_bits(words(of.bits), og.res ** 3), (list(og.min), og.cell, og.res), R, t)
    for name, buf in (("human", r.hb), ("object", r.ob)):
        n, ray, i = field_samples(buf)
        rr, ri = ref[name]
        assert n == len(rr) and n > 0
        got = np.sort(ray * 256 + i)
        assert np.array_equal(got, np.sort(rr * 256 + ri))
        # per-ray grouping, ascending i
        off = buf.ray_offset.cpu().numpy()
        cnt = buf.ray_count.cpu().numpy()
        assert cnt.sum() == n
        rec_ray = ray
        for q in np.nonzero(cnt)[0][:200]:
            seg = slice(off[q], off[q] + cnt[q])
            assert (rec_ray[seg] == q).all() and (np.diff(i[seg]) > 0).all()


def test_human_canon(setup):
    sc, cfg, hf, of, r, fid, img = setup
    n, ray, i = field_samples(r.hb)
    p = orr.sample_points(sc.camera.t, r.dirs.cpu().numpy(), ray, i, cfg.t_near, r.M.dt)
    ref = orr.human_canon(p, sc.nodes, sc.node_dqs(fid), cfg.ed_k, cfg.ed_radius, sc.bone_transforms(fid),
                          sc.skin_verts, sc.skin_weights, cfg.lbs_max_dist, hf.canon_min, hf.inv_side)
    got = r.hb.xu[:n].cpu().numpy()
    assert np.array_equal(got[:, 3], ref[:, 3])
    ed = ref[:, 3] == 1
    lbs = ref[:, 3] == 2
    assert ed.mean() > 0.5
    ulp = np.abs(got[ed, :3].view(np.int32) - ref[ed, :3].view(np.int32))
    assert ulp.max() <= 1 and (ulp == 0).mean() > 0.999
    assert np.allclose(got[lbs, :3], ref[lbs, :3], rtol=0, atol=1e-6)


def _field_ref(layers, has_deform, xu, dirs, grid, dgrid=None, dbias=None, inv_side=1.0):
    # the field kernels read the fp16 copy of the tables: the oracle gets the same values
    return orr.field_forward(layers, has_deform, xu, dirs, grid.table_as_read().cpu().numpy(),
                             dgrid.table_as_read().cpu().numpy() if dgrid is not None else None, dbias, inv_side)


def _check_field(got, ref):
    assert np.array_equal(got[:, 0] == 0, ref[:, 0] == 0)
    rel = np.abs(got[:, 0] - ref[:, 0]) / np.maximum(np.abs(ref[:, 0]), 1e-6)
    assert np.quantile(rel, 0.999) <= FIELD_SIGMA_RTOL, np.quantile(rel, [0.5, 0.99, 0.999, 1.0])
    err = np.abs(got[:, 1:] - ref[:, 1:])
    assert np.quantile(err, 0.999) <= FIELD_RGB_ATOL, np.quantile(err, [0.5, 0.99, 0.999, 1.0])
    assert np.median(err) <= 1e-4


def test_field_forward_human(setup):
    sc, cfg, hf, of, r, fid, img = setup
    n, ray, i = field_samples(r.hb)
    xu = r.hb.xu[:n].cpu().numpy()
    dirs = r.dirs.cpu().numpy()[ray]
    ref = _field_ref(hf.nets.layers, True, xu, dirs, hf.cgrid, hf.dgrid, hf.nets.theta_bias(sc.theta(fid)),
                     hf.inv_side)
    _check_field(r.hb.out[:n].cpu().numpy(), ref)


def test_field_forward_object(setup):
    sc, cfg, hf, of, r, fid, img = setup
    n, ray, i = field_samples(r.ob)
    xu = r.ob.xu[:n].cpu().numpy()
    R, t = sc.object_pose(fid)
    p = orr.sample_points(sc.camera.t, r.dirs.cpu().numpy(), ray, i, cfg.t_near, r.M.dt)
    ref_xu = orr.object_canon(p, R, t, of.obj_min, of.inv_side)
    assert np.array_equal(xu, ref_xu)
    ref = _field_ref(of.nets.layers, False, xu, r.dirs.cpu().numpy()[ray], of.cgrid)
    _check_field(r.ob.out[:n].cpu().numpy(), ref)


def test_composite_and_layers(setup):
    sc, cfg, hf, of, r, fid, img = setup
    res = {}
    for name, buf in (("human", r.hb), ("object", r.ob)):
        n, ray, i = field_samples(buf)
        rgb, dep, op = orr.composite(r.n_rays, ray, i, buf.out[:n].cpu().numpy(), cfg.t_near, r.M.dt, cfg.t_term)
        assert np.allclose(buf.rgb.cpu().numpy(), rgb, atol=1e-5)
        assert np.allclose(buf.opacity.cpu().numpy(), op, atol=1e-5)
        ok = op > 1e-3
        assert np.allclose(buf.depth.cpu().numpy()[ok], dep[ok], rtol=1e-4)
        res[name] = (buf.rgb.cpu().numpy(), buf.depth.cpu().numpy(), buf.opacity.cpu().numpy())
    out, L = orr.layers(res["human"], res["object"], cfg.background)
    assert np.array_equal(r.layer.cpu().numpy(), L)
    assert np.array_equal(img.cpu().numpy(), out)
    assert (L == 1).sum() > 0 and (L == 2).sum() > 0


def test_render_deterministic(setup):
    sc, cfg, hf, of, r, fid, img = setup
    a = img.clone()
    cam = sc.camera
    b = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    assert torch.equal(a, b)


def test_march_full_frame_bitexact():
    """configs[1] (512x512, 128 samples/ray, frame 7): the march (float64 tests
    inside each ray's clipped interval of the occupied box) must give exactly the
    oracle's decisions for all 33.5 M nominal samples (oracle in ray chunks)."""
    sc = Scene(SceneConfig(width=512, height=512), seed=0)
    cfg = RenderConfig(n_samples=128)
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, seed=0)
    of = ObjectField(sc.box_half, cfg, seed=1)
    r = Renderer(hf, of, 512, 512, cfg)
    fid = 7
    R, t = sc.object_pose(fid)
    r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), R, t)
    cam = sc.camera
    r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    torch.cuda.synchronize()
    r.check_overflow()
    dirs = r.dirs.cpu().numpy()
    lg, og = r.live_occ, of.occ
    live = orr.unpack_bits(words(r.live_bits), lg.res ** 3)
    obj = orr.unpack_bits(words(of.bits), og.res ** 3)
    want = {"human": [], "object": []}
    chunk = 16384
    for a in range(0, len(dirs), chunk):
        ref = orr.march(sc.camera.t, dirs[a:a + chunk], cfg.n_samples, cfg.t_near, r.M.dt, live,
                        (list(lg.min), lg.cell, lg.res), obj, (list(og.min), og.cell, og.res), R, t)
        for name in want:
            rr, ri = ref[name]
            want[name].append((rr + a) * 256 + ri)
    for name, buf in (("human", r.hb), ("object", r.ob)):
        n, ray, i = field_samples(buf)
        exp = np.concatenate(want[name])
        assert n == len(exp) and n > 10000
        assert np.array_equal(np.sort(ray * 256 + i), np.sort(exp))


def test_row_sharded_render_equals_full_frame(setup):
    """Multi-GPU frames deal image rows round-robin; each shard's rays
    are generated from the full frame's pixel rows, so the reassembled image is
    bit-identical to the single-GPU render (two shards emulated on one GPU)."""
    from paper_2304_03184_b200.render import assemble_row_shards
    sc, cfg, hf, of, r, fid, img = setup
    R, t = sc.object_pose(fid)
    cam = sc.camera
    full = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy).clone()
    parts = []
    for rank in range(2):
        rs = Renderer(hf, of, 64, 64, cfg, row_shard=(rank, 2))
        rs.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), R, t)
        parts.append(rs.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy).clone())
        assert torch.equal(rs.dirs, r.dirs.view(64, 64, 3)[rank::2].reshape(-1, 3))
    torch.cuda.synchronize()
    assert torch.equal(assemble_row_shards(parts, 64, 64), full)


def test_human_canon_dense_graph_and_eager_equals_graph():
    """A 2048-node ED graph takes the bucketed ring-search path of the
    canonicalisation (graphs > 1024 nodes), against the oracle; and the eager
    launch sequence (cuda_graphs=False) renders the same image as the replayed
    frame graph."""
    sc = Scene(SceneConfig(width=64, height=64), seed=0)
    rng = np.random.default_rng(5)
    nodes = sc.template_points[rng.choice(len(sc.template_points), 2048, replace=False)]
    fid = 7
    A = sc.bone_transforms(fid)
    near = np.argmin(((nodes[:, None] - sc.template_points[None, ::4]) ** 2).sum(-1), 1)
    bones = sc.template_bones[::4][near]
    dqs = np.stack([od.dq_from_rt(A[b, :3, :3], A[b, :3, 3]) for b in bones])
    R, t = sc.object_pose(fid)
    cam = sc.camera
    imgs = []
    for graphs in (False, True):
        cfg = RenderConfig(n_samples=64, cuda_graphs=graphs)
        hf = HumanField(nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, seed=0,
                        zero_deform_out=False, table_scale=0.5)
        of = ObjectField(sc.box_half, cfg, seed=1, table_scale=0.5)
        r = Renderer(hf, of, 64, 64, cfg)
        for _ in range(3):  # eager, capture, replay
            r.set_frame(dqs, sc.theta(fid), A, R, t)
            img = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
        torch.cuda.synchronize()
        r.check_overflow()
        imgs.append(img.clone())
    assert torch.equal(imgs[0], imgs[1])
    n, ray, i = field_samples(r.hb)
    p = orr.sample_points(sc.camera.t, r.dirs.cpu().numpy(), ray, i, cfg.t_near, r.M.dt)
    ref = orr.human_canon(p, nodes, dqs, cfg.ed_k, cfg.ed_radius, A, sc.skin_verts, sc.skin_weights,
                          cfg.lbs_max_dist, hf.canon_min, hf.inv_side)
    got = r.hb.xu[:n].cpu().numpy()
    assert n > 1000 and np.array_equal(got[:, 3], ref[:, 3])
    ed = ref[:, 3] == 1
    ulp = np.abs(got[ed, :3].view(np.int32) - ref[ed, :3].view(np.int32))
    assert ulp.max() <= 1 and (ulp == 0).mean() > 0.999


def test_render_to_host_readback(setup):
    """render_to_host: the read-back of view k is issued by view k+1 (after its
    uploads) or by waiting on the handle; both deliver the view's exact image."""
    sc, cfg, hf, of, r, fid, img = setup
    cam = sc.camera
    ref = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy).clone()
    h1, host1 = r.render_to_host(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    h2, host2 = r.render_to_host(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)  # issues h1's copy
    h1.synchronize()
    assert torch.equal(host1, ref.cpu())
    h2.synchronize()  # nothing issued it: the handle does
    assert torch.equal(host2, ref.cpu())


def test_small_copy_entry_points():
    """cf_copy_batch (device and pinned-host sources), cf_load_from_host and
    cf_store_to_host move the bytes exactly."""
    from paper_2304_03184_b200 import _lib
    g = torch.Generator().manual_seed(0)
    srcs = [torch.randn(1024, generator=g, dtype=torch.float64).pin_memory(), torch.randn(13, dtype=torch.float64).cuda(),
            torch.randint(0, 255, (37,), dtype=torch.uint8).pin_memory()]
    dsts = [torch.empty(1024, dtype=torch.float64, device="cuda"), torch.empty(13, dtype=torch.float64, device="cuda"),
            torch.empty(37, dtype=torch.uint8, device="cuda")]
    L = _lib.CopyList()
    for i, (s_, d_) in enumerate(zip(srcs, dsts)):
        L.src[i], L.dst[i], L.bytes[i] = s_.data_ptr(), d_.data_ptr(), s_.numel() * s_.element_size()
    L.n = 3
    _lib.call("cf_copy_batch", _lib.byref(L), _lib.stream_ptr())
    torch.cuda.synchronize()
    for s_, d_ in zip(srcs, dsts):
        assert torch.equal(d_.cpu(), s_.cpu())
    with pytest.raises(ValueError):  # pageable host memory is refused
        L2 = _lib.CopyList()
        pageable = torch.zeros(16, dtype=torch.float64)
        L2.n, L2.src[0], L2.dst[0], L2.bytes[0] = 1, pageable.data_ptr(), dsts[0].data_ptr(), 128
        _lib.call("cf_copy_batch", _lib.byref(L2), _lib.stream_ptr())
    h = torch.randn(4096, dtype=torch.float32).pin_memory()
    dv = torch.empty(4096, dtype=torch.float32, device="cuda")
    _lib.call("cf_load_from_host", dv.data_ptr(), h.data_ptr(), 4096 * 4, _lib.stream_ptr())
    back = torch.empty(4096, dtype=torch.float32).pin_memory()
    _lib.call("cf_store_to_host", dv.data_ptr(), back.data_ptr(), 4096 * 4, 8, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(back, h)


def test_load_pose_device_fk_matches_host_prior(setup):
    """Renderer.load_pose (node dqs + theta; FK and the DeformNet pose bias on the
    device) renders the frame the host-side prior (set_frame: host FK, host bias) does."""
    import torch as _t
    sc, cfg, hf, of, r, fid, img = setup
    cam = sc.camera
    a = img.clone()
    r.load_pose(_t.from_numpy(sc.node_dqs(fid)).cuda(), _t.from_numpy(sc.theta(fid)).cuda())
    R, t = sc.object_pose(fid)
    r.set_object_pose(R, t)
    b = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy).clone()
    _t.cuda.synchronize()
    assert np.allclose(r._A.cpu().numpy(), sc.bone_transforms(fid), rtol=0, atol=1e-12)
    assert np.allclose(r.dbias.cpu().numpy(), hf.nets.theta_bias(sc.theta(fid)), rtol=1e-5, atol=1e-6)
    assert float((a - b).abs().max()) <= 1e-4
    # back to the host prior: identical to the first render
    r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), R, t)
    c = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    assert _t.equal(a, c)


@pytest.mark.parametrize("fid,cmax", [(0, 64), (7, 64), (7, 6)])
def test_candidate_grid_equals_culled_scan(fid, cmax):
    """The hierarchical k-NN of the canonicalisation (per-frame candidate grid,
    cf_cand_grid_build) gives bit-identical canonical coordinates and flags to the
    warp-cooperative culled scan over every node, on a full 256^2 view (cmax = 6: most
    cells overflow their list and take the every-node path)."""
    sc = Scene(SceneConfig(width=256, height=256), seed=0)
    out = []
    for res in (48, 0):
        cfg = RenderConfig(n_samples=128, cand_grid_res=res, cand_grid_cmax=cmax)
        hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, table_scale=0.1)
        r = Renderer(hf, None, 256, 256, cfg)
        r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid))
        cam = sc.camera
        r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
        torch.cuda.synchronize()
        n, ray, i = field_samples(r.hb)
        xu = r.hb.xu[:n].cpu().numpy()
        order = np.lexsort((i, ray))
        out.append((ray[order], i[order], xu[order]))
    (r0, i0, x0), (r1, i1, x1) = out
    assert len(r0) > 10000
    assert np.array_equal(r0, r1) and np.array_equal(i0, i1)
    assert np.array_equal(x0.view(np.uint32), x1.view(np.uint32))


def test_lbs_fallback_pass_equals_fused(setup):
    """The render's separate backward-LBS pass (cf_human_lbs_fallback: a warp scan of
    the posed vertices, no buckets) gives the fused cf_human_canon output (bucket
    1-NN) bit for bit. The ED radius is shrunk so every sample falls back; points
    near the posed skin and far away (rejected by the posed box)."""
    import ctypes

    from paper_2304_03184_b200 import _lib, spec
    sc, cfg, hf, of, r = setup[:5]
    r.set_frame(sc.node_dqs(4), sc.theta(4), sc.bone_transforms(4), *sc.object_pose(4))
    r.prepare_frame()
    h = r.human
    rng = np.random.default_rng(7)
    posed = h.lbs.posed.cpu().numpy()
    near = posed[rng.integers(0, len(posed), 6000)] + rng.normal(scale=0.08, size=(6000, 3))
    far = rng.uniform(-4, 4, size=(1000, 3))
    p = torch.as_tensor(np.concatenate([near, far]), dtype=torch.float64, device="cuda")
    n = p.shape[0]
    buf, M, tt = spec._batch(r, p, torch.ones((n, 1), dtype=torch.float64, device="cuda"))
    for a in range(3):
        M.origin[a] = 0.0
    hw = _lib.HumanWarp()
    ctypes.memmove(ctypes.byref(hw), ctypes.byref(r.hw), ctypes.sizeof(hw))
    hw.r2 = 1e-12  # no sample within any ED node's support
    s = _lib.stream_ptr()
    _lib.call("cf_human_canon", _lib.byref(M), p.data_ptr(), _lib.byref(buf.mo), _lib.byref(hw),
              r._anchor_buckets.handle, h.lbs.buckets.handle, buf.xu.data_ptr(), s)
    fused = buf.xu[:n].clone()
    buf.xu.fill_(123.0)
    _lib.call("cf_human_canon", _lib.byref(M), p.data_ptr(), _lib.byref(buf.mo), _lib.byref(hw),
              r._anchor_buckets.handle, None, buf.xu.data_ptr(), s)
    assert int((buf.xu[:n, 3] != 0).sum()) == 0
    _lib.call("cf_human_lbs_fallback", _lib.byref(M), p.data_ptr(), _lib.byref(buf.mo), _lib.byref(hw),
              h.lbs.posed.data_ptr(), h.lbs.V, h.lbs.box.data_ptr(), buf.xu.data_ptr(), s)
    split = buf.xu[:n]
    assert int((fused[:, 3] == 2).sum()) > 4000 and int((fused[:, 3] == 0).sum()) >= 1000
    assert torch.equal(fused, split)
