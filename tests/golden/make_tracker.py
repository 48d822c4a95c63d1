"""Golden non-rigid tracking run of the REAL reference (tracking.py:259-556).

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tracker.py
The reference's test_tracks_synthetic_bend setting (tests/test_tracking.py:153-172),
4 frames: the model arrays, each frame's depth and mask, and the reference's solved
node transforms, pose, LM info and the ground-truth node positions. Writes
tests/golden/tracker_ref.npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.config import RunConfig  # noqa: E402
from capfields.synthetic import SyntheticScene  # noqa: E402
from capfields.tracking import NonrigidTracker, TrackingModel  # noqa: E402
from capfields.transforms import dq_apply  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    cfg = RunConfig(frames=6, width=128, height=128, fx=150.0, fy=150.0, spin_turns=0.0, arm_swing=0.0,
                    bend_joint=16, bend_degrees=15.0, node_radius=0.08)
    scene = SyntheticScene(cfg, seed=6)
    model = TrackingModel(scene.graph, scene.skeleton, scene.template_points, scene.template_normals)
    tracker = NonrigidTracker(model, scene.camera, surface_samples=1500)
    g, sk, cam = model.graph, model.skeleton, scene.camera
    out = dict(nodes=g.nodes, radius=np.array(g.radius), knn_k=np.array(g.knn_k), points=model.points,
               normals=model.normals, lbs_weights=model.lbs_weights, node_lbs_weights=model.node_lbs_weights,
               edges=model.edges, parents=sk.parents, offsets=sk.offsets, joint_limits=sk.joint_limits,
               cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height]), cam_R=cam.pose.rotation,
               cam_t=cam.pose.translation)
    for fid in range(4):
        f = scene.render(fid)
        state, info = tracker.solve(f.depth, f.mask_human, fid)
        out[f"depth{fid}"], out[f"mask{fid}"] = f.depth, f.mask_human.astype(np.uint8)
        out[f"dqs{fid}"], out[f"theta{fid}"] = state.dqs, state.theta
        out[f"iters{fid}"] = np.array(info["iterations"])
        out[f"e0_{fid}"] = np.array([e["total"] for e in info["energies"]])
        out[f"gt{fid}"] = dq_apply(scene.gt_prior(fid).graph_motion.dqs, g.nodes)
        est = dq_apply(state.dqs, g.nodes)
        print(fid, "iters", info["iterations"], "err vs gt", np.linalg.norm(est - out[f"gt{fid}"], axis=1).mean())
    np.savez_compressed(os.path.join(HERE, "tracker_ref.npz"), **out)


if __name__ == "__main__":
    main()
