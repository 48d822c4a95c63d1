"""Rigid object ICP on the GPU (tracking.py:560-620) against the
reference's own poses on its TestRigidIcp scenes (tests/golden/make_icp.py): the
fixed point at the truth, the recovered perturbation, and a spinning object tracked
without a mask. The 6x6 normal equations are summed in a different order than the
reference's BLAS products, so poses are compared at 1e-9 (rotation entries, metres).
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
    with np.load(os.path.join(GOLDEN, "icp_ref.npz")) as z:
        return {k: z[k] for k in z.files}


def test_rigid_icp_matches_reference(ref):
    from paper_2304_03184_b200.tracking import rigid_icp
    cam = _Cam(ref["cam"], ref["cam_R"], ref["cam_t"])
    for i, it in ((0, 4), (1, 15)):
        p = rigid_icp((ref["pts0"], ref["nrm0"]), ref["depth0"], cam, ref["mask0"],
                      _Pose(ref[f"init{i}_R"], ref[f"init{i}_t"]), max_iters=it)
        assert np.abs(p.rotation - ref[f"out{i}_R"]).max() <= 1e-9, i
        assert np.abs(p.translation - ref[f"out{i}_t"]).max() <= 1e-9, i
    p = rigid_icp((ref["pts1"], ref["nrm1"]), ref["depth1"], cam, None, _Pose(np.eye(3), np.zeros(3)))
    assert np.abs(p.rotation - ref["out2_R"]).max() <= 1e-9
    assert np.abs(p.translation - ref["out2_t"]).max() <= 1e-9


def test_rigid_icp_insufficient_overlap(ref):
    from paper_2304_03184_b200.errors import InsufficientOverlapError
    from paper_2304_03184_b200.tracking import rigid_icp
    cam = _Cam(ref["cam"], ref["cam_R"], ref["cam_t"])
    with pytest.raises(InsufficientOverlapError):
        rigid_icp((np.zeros((0, 3)), np.zeros((0, 3))), ref["depth0"], cam, np.zeros_like(ref["mask0"]),
                  _Pose(np.eye(3), np.zeros(3)))
