"""Golden pose Jacobians of forward LBS from the REAL reference tracker.

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_lbsjac.py
_lbs_theta_jacobian (tracking.py:244-256) at the tracked pose of the bend scene
(tests/test_tracking.py:153-172, after two frames) for the ED nodes with their
skinning weights (the bind term) and for 300 surface samples (the pose term).
Writes tests/golden/lbsjac_ref.npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.config import RunConfig  # noqa: E402
from capfields.synthetic import SyntheticScene  # noqa: E402
from capfields.tracking import NonrigidTracker, TrackingModel, _lbs_theta_jacobian  # noqa: E402

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
    theta = tracker.state.theta.copy()
    nodes, nw = model.graph.nodes, model.node_lbs_weights
    pts, pw = tracker.sub_pts[:300], tracker.sub_lbs[:300]
    jn = _lbs_theta_jacobian(model.skeleton, theta, nodes, nw)
    jp = _lbs_theta_jacobian(model.skeleton, theta, pts, pw)
    np.savez_compressed(os.path.join(HERE, "lbsjac_ref.npz"), theta=theta, nodes=nodes, nw=nw, pts=pts, pw=pw,
                        jn=jn, jp=jp)
    print("theta |.|", np.abs(theta).max(), "jn", jn.shape, "jp", jp.shape)


if __name__ == "__main__":
    main()
