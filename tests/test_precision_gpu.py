"""Field parity at the SPEC's numeric type ("float64 core", SPEC.md:422
"32-bit in nrf training"; north_star: "within a stated tolerance (e.g. 1e-4
relative in fp32)").

The "fp32" precision mode (RenderConfig.precision, the default) is checked stage by
stage against the oracle's 32-bit semantics (`oracle.nrf.mlp_forward_f32`: fp32
tables / features / weights, float64 arithmetic), each stage fed the previous
stage's device output:

  deformation-grid features (hot-path hash kernel)   bit-exact (float32)
  DeformNet -> xc                                    |dxc| <= XC_ATOL
  canonical-grid features (hot-path hash kernel)     bit-exact (float32)
  E_g / E_c -> sigma, rgb                            sigma rel <= 1e-4, rgb abs <= 1e-5

and end to end (tables -> sigma / rgb) with the tolerance stated in FIELD_E2E_*:
a one-ulp change of xc moves a 2048-resolution level's features by ~N * ulp *
|table| ~ 1e-4 |table|, so the end-to-end bound carries that conditioning of the
finest hash level. The "fp16" mode's hot-path hash kernels are also checked
bit-exactly (fp16-rounded features), and its drift from the 32-bit semantics is
measured and bounded (what the fast mode costs in accuracy).
"""
import numpy as np
import pytest
import torch

from oracle import nrf as on
from oracle import render as orr
from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
from paper_2304_03184_b200.scene import Scene, SceneConfig

pytestmark = pytest.mark.gpu

XC_ATOL = 4e-7            # ~6 float32 ulps of a unit coordinate: 0.05/side * |dv|, |dv| <= 1.6e-5
SIGMA_RTOL = 1e-4         # E_g / E_c stage, fp32 mode
RGB_ATOL = 1e-5
# end to end (tables -> sigma, rgb), fp32 mode: bounded by the conditioning of the
# finest hash levels, not by the kernels — test_e2e_tolerance_is_the_problems_conditioning
# shows the oracle itself moves as much when xc is perturbed by one float32 ulp
FIELD_E2E_SIGMA_RTOL = 2e-3   # max; 99.9th percentile <= 1e-3 (measured 4.1e-4 / 5.1e-4)
FIELD_E2E_RGB_ATOL = 1e-4     # max; measured 2.3e-5
CGRID = (16, 2, 19, 16, 2048)
DGRID = (8, 4, 17, 16, 256)


def _scene_fields(precision, fuse=False):
    sc = Scene(SceneConfig(width=64, height=64), seed=0)
    cfg = RenderConfig(n_samples=64, precision=precision, fuse_hash=fuse)
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, seed=0, zero_deform_out=False,
                    table_scale=0.5)
    of = ObjectField(sc.box_half, cfg, seed=1, table_scale=0.5)
    hf.nets.layers["D5"] *= 10.0  # |dv| up to ~1: tanh far from linear
    for f, s in ((hf, 6.0), (of, 14.0)):
        f.nets.layers["G2"][0] *= s
        f.nets.repack()
    return sc, cfg, hf, of


@pytest.fixture(scope="module", params=["fp32", "fp16"])
def rendered(request):
    """One view with the stage-by-stage kernels (fuse_hash=False: both grids' hash
    features land in the field scratch, so each stage can be checked on its own); the
    render's fused hash + MLP kernels are checked against this path in
    test_fused_hash_kernels_equal_stages."""
    precision = request.param
    sc, cfg, hf, of = _scene_fields(precision)
    r = Renderer(hf, of, 64, 64, cfg)
    r.cfg.cuda_graphs = False
    fid = 7
    R, t = sc.object_pose(fid)
    r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), R, t)
    cam = sc.camera
    r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    torch.cuda.synchronize()
    r.check_overflow()
    return precision, sc, cfg, hf, of, r, fid


def _by_record(buf):
    """The view's field outputs ordered by record (the march's compaction order is
    that of its warps' atomics, not fixed)."""
    n = int(buf.counters[0])
    rec = buf.records[:n].cpu().numpy().view(np.uint32)
    order = np.argsort(rec, kind="stable")
    return rec[order], buf.out[:n].cpu().numpy()[order]


def test_fused_hash_kernels_equal_stages():
    """The render's fp32 mode looks the hash grids up inside the MLP kernels (the
    deformation grid in DeformNet, deform_mlp_prec_kernel<false, 2>; the canonical grid
    in E_g / E_c, color_mlp_prec_kernel<4>) instead of reading the separate hash
    kernels' output: same functions, so the field outputs are bit-equal to the
    stage-by-stage path, human and object."""
    fid = 3
    out = {}
    for fuse in (False, True):
        sc, cfg, hf, of = _scene_fields("fp32", fuse=fuse)  # same seeds: the same fields
        r = Renderer(hf, of, 64, 64, cfg)
        r.cfg.cuda_graphs = False
        R, t = sc.object_pose(fid)
        r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), R, t)
        cam = sc.camera
        r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
        torch.cuda.synchronize()
        assert bool(r.hdesc.split_stages) != fuse
        out[fuse] = (_by_record(r.hb), _by_record(r.ob))
    for f in range(2):
        (ra, oa), (rb, ob) = out[False][f], out[True][f]
        assert len(ra) > 100 and np.array_equal(ra, rb)
        assert np.array_equal(oa.view(np.int32), ob.view(np.int32))


def _scratch_views(r, buf, desc, has_deform, precision):
    """(cfeat, dfeat, xc) of the last view from the field scratch (layout: capi header)."""
    n = int(buf.counters[0])
    cap = buf.mo.capacity
    raw = r._scratch(buf, desc)
    fb = 128 if precision == "fp32" else 64
    dt = torch.float32 if precision == "fp32" else torch.float16
    cfeat = raw[: n * fb].view(dt).view(n, 32).float().cpu().numpy()
    if not has_deform:
        return n, cfeat, None, None
    dfeat = raw[cap * fb: cap * fb + n * fb].view(dt).view(n, 32).float().cpu().numpy()
    xc = raw[2 * cap * fb: 2 * cap * fb + n * 16].view(torch.float32).view(n, 4).cpu().numpy()
    return n, cfeat, dfeat, xc


def _samples(buf, n):
    rec = buf.records[:n].cpu().numpy().view(np.uint32)
    return (rec >> 8).astype(np.int64)


def _f16(x):
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def test_hot_path_hash_kernels_bitexact(rendered):
    """The render path's own hash kernels (field.cu hash_f16_kernel, both grids)
    against oracle.nrf.hash_encode: float32 features bit-equal ("fp32" mode) or
    their fp16 rounding bit-equal ("fp16" mode)."""
    precision, sc, cfg, hf, of, r, fid = rendered
    n, cfeat, dfeat, xc = _scratch_views(r, r.hb, r.hdesc, True, precision)
    xu = r.hb.xu[:n].cpu().numpy()
    ok = xu[:, 3] > 0
    assert ok.sum() > 1000
    dtab = (hf.dgrid.table if precision == "fp32" else hf.dgrid.table_as_read()).cpu().numpy()
    ref_d = on.hash_encode(dtab, xu[ok, :3], *DGRID)
    ref_c = on.hash_encode(hf.cgrid.table.cpu().numpy(), xc[ok, :3], *CGRID)
    if precision == "fp16":
        ref_d, ref_c = _f16(ref_d), _f16(ref_c)
    assert np.array_equal(dfeat[ok].view(np.int32), ref_d.view(np.int32))
    assert np.array_equal(cfeat[ok].view(np.int32), ref_c.view(np.int32))
    assert (dfeat[~ok] == 0).all() and (cfeat[~ok] == 0).all()
    # object field (4 threads per sample)
    n, cfeat, _, _ = _scratch_views(r, r.ob, r.odesc, False, precision)
    xo = r.ob.xu[:n].cpu().numpy()
    ref = on.hash_encode(of.cgrid.table.cpu().numpy(), xo[:, :3], *CGRID)
    if precision == "fp16":
        ref = _f16(ref)
    assert np.array_equal(cfeat.view(np.int32), ref.view(np.int32))


def test_deformnet_stage(rendered):
    """DeformNet on the device's deformation features -> xc vs the oracle."""
    precision, sc, cfg, hf, of, r, fid = rendered
    n, cfeat, dfeat, xc = _scratch_views(r, r.hb, r.hdesc, True, precision)
    xu = r.hb.xu[:n].cpu().numpy()
    ok = xu[:, 3] > 0
    v = orr.deform_forward(hf.nets.layers, dfeat[ok], hf.nets.theta_bias(sc.theta(fid)), precision)
    ref = orr.deformed_coords(xu[ok], v, hf.inv_side)
    err = np.abs(xc[ok, :3] - ref)
    assert np.abs(v).max() > 0.3  # a non-trivial deformation
    tol = XC_ATOL if precision == "fp32" else 2e-5
    assert err.max() <= tol, np.quantile(err, [0.5, 0.999, 1.0])


def test_color_stage(rendered):
    """E_g / E_c on the device's canonical features -> sigma / rgb vs the oracle."""
    precision, sc, cfg, hf, of, r, fid = rendered
    for field, buf, desc, deform in ((hf, r.hb, r.hdesc, True), (of, r.ob, r.odesc, False)):
        n, cfeat, _, _ = _scratch_views(r, buf, desc, deform, precision)
        ray = _samples(buf, n)
        xu = buf.xu[:n].cpu().numpy()
        ok = xu[:, 3] > 0
        ref = orr.color_forward(field.nets.layers, cfeat[ok], r.dirs.cpu().numpy()[ray[ok]], precision)
        got = buf.out[:n].cpu().numpy()[ok]
        rel = np.abs(got[:, 0] - ref[:, 0]) / np.abs(ref[:, 0])
        err = np.abs(got[:, 1:] - ref[:, 1:])
        if precision == "fp32":
            assert rel.max() <= SIGMA_RTOL, np.quantile(rel, [0.5, 0.999, 1.0])
            assert err.max() <= RGB_ATOL, np.quantile(err, [0.5, 0.999, 1.0])
        else:  # fp16 operands vs the kernel-precision oracle: accumulation order only
            assert np.quantile(rel, 0.999) <= 2e-2 and np.quantile(err, 0.999) <= 2e-3
        assert (buf.out[:n].cpu().numpy()[~ok] == 0).all()


def _field_e2e_error(precision, sc, hf, of, r, fid):
    """Device field output vs the oracle's 32-bit semantics from the tables."""
    out = {}
    for name, field, buf in (("human", hf, r.hb), ("object", of, r.ob)):
        n = int(buf.counters[0])
        ray = _samples(buf, n)
        xu = buf.xu[:n].cpu().numpy()
        dirs = r.dirs.cpu().numpy()[ray]
        if name == "human":
            ref = orr.field_forward(field.nets.layers, True, xu, dirs, field.cgrid.table.cpu().numpy(),
                                    field.dgrid.table.cpu().numpy(), field.nets.theta_bias(sc.theta(fid)),
                                    field.inv_side, precision="fp32")
        else:
            ref = orr.field_forward(field.nets.layers, False, xu, dirs, field.cgrid.table.cpu().numpy(),
                                    precision="fp32")
        got = buf.out[:n].cpu().numpy()
        ok = xu[:, 3] > 0
        rel = np.abs(got[ok, 0] - ref[ok, 0]) / np.abs(ref[ok, 0])
        err = np.abs(got[ok, 1:] - ref[ok, 1:])
        out[name] = (rel, err)
    return out


def test_field_end_to_end_vs_fp32_semantics(rendered):
    """Tables -> sigma / rgb against the SPEC's 32-bit semantics. fp32 mode: within
    FIELD_E2E_*; fp16 mode: its drift, measured (percentiles in the message)."""
    precision, sc, cfg, hf, of, r, fid = rendered
    for name, (rel, err) in _field_e2e_error(precision, sc, hf, of, r, fid).items():
        q = (np.quantile(rel, [0.5, 0.999, 1.0]), np.quantile(err, [0.5, 0.999, 1.0]))
        if precision == "fp32":
            assert np.quantile(rel, 0.999) <= 1e-3 and rel.max() <= FIELD_E2E_SIGMA_RTOL, (name, q)
            assert np.quantile(err, 0.999) <= 1e-5 * 5 and err.max() <= FIELD_E2E_RGB_ATOL, (name, q)
        else:
            # the fp16 mode is ~2 orders of magnitude less accurate (measured 99.9th pct:
            # sigma 5.5e-2 relative, rgb 2.2e-3): bounded, not 1e-4
            assert np.quantile(rel, 0.999) <= 1e-1 and np.quantile(err, 0.999) <= 5e-3, (name, q)


def test_e2e_tolerance_is_the_problems_conditioning(rendered):
    """The oracle against itself with xc moved by one float32 ulp: the sigma / rgb
    change is of the same size as the fp32 device mode's end-to-end error, i.e. no
    32-bit evaluation order can do much better on this field (the 2048-resolution
    level turns one ulp of xc ~ 6e-8 into ~1e-4 of the features)."""
    precision, sc, cfg, hf, of, r, fid = rendered
    if precision != "fp32":
        pytest.skip("conditioning is mode independent")
    n, cfeat, dfeat, xc = _scratch_views(r, r.hb, r.hdesc, True, precision)
    ok = r.hb.xu[:n].cpu().numpy()[:, 3] > 0
    dirs = r.dirs.cpu().numpy()[_samples(r.hb, n)[ok]]
    x = xc[ok, :3]
    ctab = hf.cgrid.table.cpu().numpy()
    a = orr.color_forward(hf.nets.layers, on.hash_encode(ctab, x, *CGRID), dirs)
    b = orr.color_forward(hf.nets.layers, on.hash_encode(ctab, np.nextafter(x, np.float32(2)), *CGRID), dirs)
    rel = np.abs(a[:, 0] - b[:, 0]) / np.abs(a[:, 0])
    dev_rel, _ = _field_e2e_error(precision, sc, hf, of, r, fid)["human"]
    assert np.quantile(rel, 0.999) >= 0.25 * np.quantile(dev_rel, 0.999), (np.quantile(rel, 0.999),
                                                                           np.quantile(dev_rel, 0.999))


def test_composite_fp32_mode(rendered):
    precision, sc, cfg, hf, of, r, fid = rendered
    for buf in (r.hb, r.ob):
        n = int(buf.counters[0])
        rec = buf.records[:n].cpu().numpy().view(np.uint32)
        ray, i = (rec >> 8).astype(np.int64), (rec & 255).astype(np.int64)
        rgb, dep, op = orr.composite(r.n_rays, ray, i, buf.out[:n].cpu().numpy(), cfg.t_near, r.M.dt, cfg.t_term)
        assert np.allclose(buf.rgb.cpu().numpy(), rgb, atol=1e-5)
        assert np.allclose(buf.opacity.cpu().numpy(), op, atol=1e-5)
