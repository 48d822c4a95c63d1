"""Golden data-association vectors from the REAL reference tracker.

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_corr.py
On the bend scene of the reference's tracking test (tests/test_tracking.py:153-172),
after two tracked frames: depth_normals of frame 3 (tracking.py:60-80) and the
tracker's two find_correspondences calls (tracking.py:83-150, 340-354). Writes
tests/golden/corr_ref.npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.config import RunConfig  # noqa: E402
from capfields.skeleton import lbs_batch, skinning_transforms  # noqa: E402
from capfields.synthetic import SyntheticScene  # noqa: E402
from capfields.tracking import NonrigidTracker, TrackingModel, depth_normals, find_correspondences  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    cfg = RunConfig(frames=6, width=128, height=128, fx=150.0, fy=150.0, spin_turns=0.0, arm_swing=0.0,
                    bend_joint=16, bend_degrees=15.0, node_radius=0.08)
    scene = SyntheticScene(cfg, seed=6)
    model = TrackingModel(scene.graph, scene.skeleton, scene.template_points, scene.template_normals)
    tracker = NonrigidTracker(model, scene.camera, surface_samples=1500)
    for fid in range(2):
        f = scene.render(fid)
        tracker.solve(f.depth, f.mask_human, fid)
    f = scene.render(3)
    cam = scene.camera
    state = tracker.state
    nmap = depth_normals(f.depth, cam)
    warped, wn = tracker.warp_subset(state)
    di, du, dn = find_correspondences(warped, wn, f.depth, cam, mask=f.mask_human, normals_map=nmap)
    lp = lbs_batch(model.skeleton, state.theta, tracker.sub_pts, tracker.sub_lbs)
    A = skinning_transforms(model.skeleton, state.theta)
    ln = np.einsum("nab,nb->na", A[np.argmax(tracker.sub_lbs, axis=1)][:, :3, :3], tracker.sub_normals)
    pi, pu, pn = find_correspondences(lp, ln, f.depth, cam, mask=f.mask_human, normals_map=nmap)
    ni, nu_, nn = find_correspondences(warped, wn, f.depth, cam)  # no mask, normals computed inside
    np.savez_compressed(os.path.join(HERE, "corr_ref.npz"), depth=f.depth, mask=f.mask_human.astype(np.uint8),
                        cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height]),
                        cam_R=cam.pose.rotation, cam_t=cam.pose.translation, nmap=nmap,
                        warped=warped, wn=wn, di=di, du=du, dn=dn, lp=lp, ln=ln, pi=pi, pu=pu, pn=pn,
                        ni=ni, nu=nu_, nn=nn)
    print("data", len(di), "pose", len(pi), "nomask", len(ni), "of", len(warped))


if __name__ == "__main__":
    main()
