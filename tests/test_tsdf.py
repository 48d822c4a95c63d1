"""Rigid-object TSDF on the GPU (tsdf.py:17-176) against vectors the
reference itself produced (tests/golden/make_tsdf.py), plus the reference's own
test cases (tests/test_tsdf.py:1-107) re-run through the device volume.

Tolerances: the reference evaluates the 3x3 rigid transforms with BLAS (summation
order / FMA unknown), the kernels in a fixed order without FMA, so voxel depths can
differ by an ulp; every value is compared at 1e-9 and every decision (weights,
validity, hit / surface counts) exactly.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


class _Pose:
    def __init__(self, R, t):
        self.rotation, self.translation = np.asarray(R), np.asarray(t)


class _Cam:
    def __init__(self, fx, fy, cx, cy, w, h, R=np.eye(3), t=np.zeros(3)):
        self.fx, self.fy, self.cx, self.cy, self.width, self.height = fx, fy, cx, cy, int(w), int(h)
        self.pose = _Pose(R, t)


@pytest.fixture(scope="module")
def ref():
    with np.load(os.path.join(GOLDEN, "tsdf_ref.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def vol(ref):
    from paper_2304_03184_b200.tsdf import TsdfVolume, tsdf_integrate
    c = ref["cam"]
    cam = _Cam(*c, R=ref["cam_R"], t=ref["cam_t"])
    r, vs, ox, oy, oz, _ = ref["vol"]
    v = TsdfVolume(int(r), vs, np.array([ox, oy, oz]))
    poses = [_Pose(R, t) for R, t in zip(ref["pose_R"], ref["pose_t"])]
    tsdf_integrate(v, ref["depths"][0], cam, poses[0])
    tsdf_integrate(v, ref["depths"][1], cam, poses[1], mask=ref["mask"])
    tsdf_integrate(v, ref["depths"][2], cam, poses[2])
    return v, cam, poses


def test_integrate_matches_reference(ref, vol):
    v = vol[0]
    assert np.array_equal(v.weight, ref["weight"])
    assert np.abs(v.tsdf - ref["tsdf"]).max() <= 1e-9


def test_sample_and_gradient_match_reference(ref, vol):
    v = vol[0]
    val, ok = v.sample(ref["pts"])
    assert np.array_equal(ok, ref["ok"])
    assert np.abs(val - ref["val"]).max() <= 1e-9
    g = v.gradient(ref["pts"][:500])
    assert np.abs(g - ref["grad"]).max() <= 1e-7


def test_surface_and_raycast_match_reference(ref, vol):
    v, cam, poses = vol
    sp, sn = v.extract_surface()
    assert sp.shape == ref["surf_p"].shape
    assert np.abs(sp - ref["surf_p"]).max() <= 1e-9 and np.abs(sn - ref["surf_n"]).max() <= 1e-6
    rp, rn = v.raycast(cam, poses[2], stride=2)
    assert rp.shape == ref["ray_p"].shape and len(rp) > 50
    assert np.abs(rp - ref["ray_p"]).max() <= 1e-9 and np.abs(rn - ref["ray_n"]).max() <= 1e-6


# ---- the reference's own cases (tests/test_tsdf.py), through the device volume

MAX_WEIGHT = 64.0


def plane_depth_cam(z=1.0, size=64):
    return _Cam(float(size), float(size), size / 2, size / 2, size, size), np.full((size, size), z)


def small_volume():
    from paper_2304_03184_b200.tsdf import TsdfVolume
    return TsdfVolume(resolution=32, voxel_size=0.02, origin=np.array([-0.32, -0.32, 0.67]))


ID = _Pose(np.eye(3), np.zeros(3))


def test_double_integration_idempotent_values():
    from paper_2304_03184_b200.tsdf import tsdf_integrate
    cam, depth = plane_depth_cam()
    v = small_volume()
    tsdf_integrate(v, depth, cam, ID)
    t1, w1 = v.tsdf.copy(), v.weight.copy()
    tsdf_integrate(v, depth, cam, ID)
    assert np.allclose(v.tsdf, t1, atol=1e-12)
    touched = w1 > 0
    assert np.allclose(v.weight[touched], np.minimum(2 * w1[touched], MAX_WEIGHT))


def test_weight_cap():
    cam, depth = plane_depth_cam()
    v = small_volume()
    for _ in range(70):
        v.integrate(depth, cam, ID)
    assert v.weight.max() == MAX_WEIGHT


def test_surface_voxels_near_zero_and_behind_untouched():
    cam, depth = plane_depth_cam(z=1.0)
    v = small_volume()
    v.integrate(depth, cam, ID)
    centers = v.voxel_centers()
    on_plane = np.abs(centers[..., 2] - 1.0) < 0.25 * v.voxel_size
    sel = on_plane & (v.weight > 0)
    assert sel.sum() > 10
    assert np.abs(v.tsdf[sel]).max() < 1e-12
    behind = centers[..., 2] > 1.0 + v.truncation + v.voxel_size
    assert (v.weight[behind] == 0).all() and (v.tsdf[behind] == 1.0).all()


def test_mask_limits_update():
    cam, depth = plane_depth_cam(z=1.0)
    mask = np.zeros(depth.shape, dtype=np.uint8)
    mask[:, : depth.shape[1] // 2] = 1
    v = small_volume()
    v.integrate(depth, cam, ID, mask=mask)
    c = v.voxel_centers().reshape(-1, 3)
    u = cam.fx * c[:, 0] / c[:, 2] + cam.cx
    right = u > depth.shape[1] // 2 + 1
    assert (v.weight.reshape(-1)[right] == 0).all()
    assert (v.weight > 0).sum() > 0


def test_sample_gradient_surface_raycast_on_plane():
    cam, depth = plane_depth_cam(z=1.0)
    v = small_volume()
    for _ in range(8):
        v.integrate(depth, cam, ID)
    vals, ok = v.sample(np.array([[0.0, 0.0, 1.0], [0.05, -0.03, 1.0]]))
    assert ok.all() and np.abs(vals).max() < 0.1
    v = small_volume()
    v.integrate(depth, cam, ID)
    g = v.gradient(np.array([[0.0, 0.0, 1.0]]))[0]
    assert (g / np.linalg.norm(g))[2] < -0.95
    pts, normals = v.extract_surface()
    assert len(pts) > 50 and np.abs(pts[:, 2] - 1.0).max() < v.voxel_size
    assert (np.abs(normals[:, 2]) > 0.9).mean() > 0.95
    pts, normals = v.raycast(cam, ID, stride=4)
    assert len(pts) > 20 and np.abs(pts[:, 2] - 1.0).max() < v.voxel_size
