"""Pin the stage-1 oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py). CPU only."""
import numpy as np

from oracle import deform as od


def test_dq_blend_apply_bitexact(stage1):
    g = stage1
    b = od.dq_blend(g["A_w"], g["A_dqs"])
    assert np.array_equal(b, g["A_blend"])
    assert np.array_equal(od.dq_apply(b, g["A_pts"]), g["A_apply"])


def test_warps_match_reference(stage1):
    g = stage1
    _, _, pc, valid = od.warp(g["B_nodes"], 0.1, 4, g["B_dqs"], g["B_q"], "backward")
    assert np.array_equal(valid, g["B_back_valid"])
    # bit-equal up to the last bits of exp(); positions within 1e-12
    assert np.allclose(pc, g["B_back"], rtol=0, atol=1e-12)
    _, _, fw, fvalid = od.warp(g["B_nodes"], 0.1, 4, g["B_dqs"], g["B_q"], "forward")
    assert np.array_equal(fvalid, g["B_fwd_valid"])
    assert np.allclose(fw, g["B_fwd"], rtol=0, atol=1e-12)


def test_brute_force_query_indices_bitexact(stage1):
    g = stage1
    for s in (4, 8):
        idx, w, pc = od.brute_force_query(g["B_nodes"], 0.1, g["B_dqs"], g["B_q"], s)
        assert np.array_equal(idx, g[f"B_bf{s}_idx"])
        assert np.allclose(w, g[f"B_bf{s}_w"], rtol=1e-15, atol=0)
        ok = np.isfinite(g[f"B_bf{s}_pc"]).all(axis=1)
        assert np.array_equal(np.isfinite(pc).all(axis=1), ok)
        assert np.allclose(pc[ok], g[f"B_bf{s}_pc"][ok], rtol=0, atol=1e-12)


def test_knnfield_matches_reference(stage1):
    g = stage1
    f = od.Field(g["C_nodes"], 0.1, 32, 4)
    assert np.array_equal(f.bmin, g["C_bbox_min"]) and f.voxel == float(g["C_voxel"])
    assert np.array_equal(f.nidx, g["C_nidx"])
    f.update(0, g["C_dqs"])
    assert np.array_equal(f.live[0], g["C_live"])
    nbr, w, pc, valid = f.query(g["C_q"], 0)
    assert np.array_equal(nbr, g["C_nbr"])
    assert np.array_equal(valid, g["C_valid"])
    assert np.allclose(w, g["C_w"], rtol=1e-15, atol=0)
    assert np.allclose(pc[valid], g["C_pc"][valid], rtol=0, atol=1e-12)


def test_lbs_matches_reference(stage1):
    g = stage1
    from paper_2304_03184_b200 import scene
    A = od.bone_transforms(scene.PARENTS, scene.OFFSETS, g["D_theta"])
    assert np.allclose(A, g["D_A"], rtol=0, atol=1e-14)
    assert np.allclose(od.lbs(A, g["D_pts"], g["D_w"]), g["D_lbs"], rtol=0, atol=1e-13)


def test_scene_samples_warp(stage1):
    g = stage1
    _, _, pc, valid = od.warp(g["E_nodes"], 0.1, 4, g["E_dqs7"], g["E_samples"], "backward")
    assert np.array_equal(valid, g["E_back_valid"])
    assert np.allclose(pc, g["E_back"], rtol=0, atol=1e-12)
    idx, _ = od.knn_exact(od.deformed_nodes(g["E_nodes"], g["E_dqs7"]), g["E_samples"], 4)
    assert np.array_equal(idx, g["E_idx"])
