"""The synthetic-scene generator (product-side input setup) reproduces the
reference's SyntheticScene (synthetic.py:48-131) — pinned by golden vectors."""
import numpy as np

from oracle import deform as od
from paper_2304_03184_b200.scene import Scene, SceneConfig, bone_weights


def test_scene_matches_reference(stage1):
    g = stage1
    sc = Scene(SceneConfig(), seed=0)
    assert len(sc.template_points) == int(g["E_n_template"])
    assert np.array_equal(sc.template_points[:200], g["E_template_head"])
    assert np.allclose(sc.template_points.sum(axis=0), g["E_template_sum"], rtol=0, atol=1e-9)
    assert sc.nodes.shape == (128, 3)
    assert np.array_equal(sc.nodes, g["E_nodes"])
    assert np.array_equal(sc.node_bones, g["E_node_bones"])
    assert np.array_equal(sc.theta(7), g["E_theta7"])
    assert np.allclose(sc.node_dqs(7), g["E_dqs7"], rtol=0, atol=1e-14)
    assert np.allclose(sc.camera.R, g["E_cam_R"], atol=1e-15)
    assert np.allclose(sc.camera.t, g["E_cam_t"], atol=1e-15)
    o, d = sc.camera.all_rays()
    assert np.allclose(o, g["E_ray_o"], atol=1e-15) and np.allclose(d, g["E_ray_d"], atol=1e-15)
    assert np.allclose(sc.skin_verts, sc.template_points[g["E_skin_idx"]])
    assert np.allclose(sc.skin_weights[:300], g["E_skin_w_head"], atol=1e-14)
    R, t = sc.object_pose(7)
    assert np.allclose(R, g["E_obj_pose7"][:3, :3], atol=1e-14) and np.allclose(t, g["E_obj_pose7"][:3, 3], atol=1e-14)


def test_dq_from_rt_roundtrip():
    sc = Scene(SceneConfig(), seed=0)
    A = sc.bone_transforms(3)
    for b in range(24):
        dq = od.dq_from_rt(A[b, :3, :3], A[b, :3, 3])
        p = np.array([[0.1, 0.2, 0.3]])
        assert np.allclose(od.dq_apply(dq[None], p), p @ A[b, :3, :3].T + A[b, :3, 3], atol=1e-12)
