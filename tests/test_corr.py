"""Data association of the non-rigid tracker on the GPU (
tracking.py:60-150) against vectors the reference produced on its own tracking-test
scene (tests/golden/make_corr.py): the depth normal map and the tracker's two
find_correspondences calls (warped ED model, skeleton-only model) plus an unmasked
call that computes the normals itself. The reference evaluates the camera pose
products with BLAS, the kernels in a fixed order, so values are compared at 1e-12
and the kept index sets exactly.
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
    def __init__(self, c, R, t):
        self.fx, self.fy, self.cx, self.cy = (float(v) for v in c[:4])
        self.width, self.height = int(c[4]), int(c[5])
        self.pose = _Pose(R, t)


@pytest.fixture(scope="module")
def ref():
    with np.load(os.path.join(GOLDEN, "corr_ref.npz")) as z:
        return {k: z[k] for k in z.files}


def test_depth_normals(ref):
    from paper_2304_03184_b200.tracking import depth_normals
    cam = _Cam(ref["cam"], ref["cam_R"], ref["cam_t"])
    n = depth_normals(ref["depth"], cam)
    assert np.array_equal(np.abs(n).sum(-1) > 0, np.abs(ref["nmap"]).sum(-1) > 0)
    assert np.abs(n - ref["nmap"]).max() <= 1e-12


def test_find_correspondences(ref):
    from paper_2304_03184_b200.tracking import find_correspondences
    cam = _Cam(ref["cam"], ref["cam_R"], ref["cam_t"])
    for pts, nrm, mask, nmap, key in ((ref["warped"], ref["wn"], ref["mask"], ref["nmap"], "d"),
                                      (ref["lp"], ref["ln"], ref["mask"], ref["nmap"], "p"),
                                      (ref["warped"], ref["wn"], None, None, "n")):
        idx, tgt, nu = find_correspondences(pts, nrm, ref["depth"], cam, mask=mask, normals_map=nmap)
        ri, rt, rn = ref[f"{key}i"], ref[f"{key}u"], ref[f"{key}n"]
        assert np.array_equal(idx, ri), key
        assert len(idx) > 100
        assert np.abs(tgt - rt).max() <= 1e-12 and np.abs(nu - rn).max() <= 1e-12, key


def test_lbs_theta_jacobian():
    """Central-difference pose Jacobian of forward LBS (tracking.py:244-256) vs the
    reference's on its tracked bend pose (tests/golden/make_lbsjac.py). The FD step is
    1e-6, so ulp-level differences in the bone transforms (device FK vs numpy/BLAS)
    become ~1e-10 in the quotient: compared at 1e-8."""
    from paper_2304_03184_b200.tracking import lbs_theta_jacobian
    with np.load(os.path.join(GOLDEN, "lbsjac_ref.npz")) as z:
        g = {k: z[k] for k in z.files}
    for pts, w, key in ((g["nodes"], g["nw"], "jn"), (g["pts"], g["pw"], "jp")):
        j = lbs_theta_jacobian(None, g["theta"], pts, w)
        assert j.shape == g[key].shape
        assert np.abs(j - g[key]).max() <= 1e-8, (key, np.abs(j - g[key]).max())
