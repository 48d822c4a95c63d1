"""Golden rigid-ICP poses from the REAL reference (tracking.py:560-620).

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_icp.py
Scenes and models follow the reference's TestRigidIcp (tests/test_tracking.py:190-230);
a third case tracks a spinning object into frame 3 without a mask. Writes
tests/golden/icp_ref.npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.config import RunConfig  # noqa: E402
from capfields.synthetic import SyntheticScene  # noqa: E402
from capfields.tracking import depth_normals, rigid_icp  # noqa: E402
from capfields.transforms import Se3  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def object_scene(**kw):
    base = dict(frames=60, width=128, height=128, fx=150.0, fy=150.0, human=False,
                object_orbit_degrees=0.0, object_spin_degrees=0.0)
    base.update(kw)
    return SyntheticScene(RunConfig(**base), seed=7)


def model_from_frame(scene, fid=0):
    fr = scene.render(fid)
    ys, xs = np.nonzero(fr.mask_object & (fr.depth > 0))
    uv = np.stack([xs, ys], axis=-1).astype(np.float64)
    pts = scene.camera.backproject_batch(uv, fr.depth[ys, xs])
    nm = depth_normals(fr.depth, scene.camera)
    normals = nm[ys, xs]
    ok = np.linalg.norm(normals, axis=1) > 0.5
    return fr, pts[ok][::2], normals[ok][::2]


def main():
    out = {}
    scene = object_scene()
    fr, pts, normals = model_from_frame(scene)
    cam = scene.camera
    out["cam"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height])
    out["cam_R"], out["cam_t"] = cam.pose.rotation, cam.pose.translation
    init = Se3.from_rotvec_trans(np.deg2rad(2.0) * np.array([0.3, 0.8, 0.52]), [0.006, -0.005, 0.006])
    cases = [(Se3.identity(), 4, True), (init, 15, True)]
    scene2 = object_scene(object_spin_degrees=40.0)
    fr2 = scene2.render(3)
    _, pts2, normals2 = model_from_frame(scene2, 0)
    out["depth0"], out["mask0"], out["pts0"], out["nrm0"] = fr.depth, fr.mask_object.astype(np.uint8), pts, normals
    out["depth1"], out["pts1"], out["nrm1"] = fr2.depth, pts2, normals2
    for i, (ini, it, masked) in enumerate(cases):
        p = rigid_icp((pts, normals), fr.depth, cam, fr.mask_object, ini, max_iters=it)
        out[f"init{i}_R"], out[f"init{i}_t"] = ini.rotation, ini.translation
        out[f"out{i}_R"], out[f"out{i}_t"] = p.rotation, p.translation
    p = rigid_icp((pts2, normals2), fr2.depth, cam, None, Se3.identity())
    out["out2_R"], out["out2_t"] = p.rotation, p.translation
    np.savez_compressed(os.path.join(HERE, "icp_ref.npz"), **out)
    print("model", len(pts), len(pts2), "pose2 t", p.translation)


if __name__ == "__main__":
    main()
