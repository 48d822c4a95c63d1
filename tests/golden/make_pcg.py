"""Golden Gauss-Newton systems of the REAL reference tracker and its pcg_solve.

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_pcg.py
The system is the reference's own _assemble (tracking.py:358-508) on the synthetic
bend scene of its test_tracks_synthetic_bend (tests/test_tracking.py:153-172) after
two tracked frames; pcg_solve (tracking.py:158-193) is run at three damping values
and with a tight tolerance. Writes tests/golden/pcg_ref.npz (CSR arrays, r, x).
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.config import RunConfig  # noqa: E402
from capfields.synthetic import SyntheticScene  # noqa: E402
from capfields.tracking import NonrigidTracker, TrackingModel, depth_normals, pcg_solve  # noqa: E402

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
    state = tracker.state.copy()
    normals = depth_normals(f.depth, scene.camera)
    data_corr, pose_corr = tracker._associate(state, f.depth, f.mask_human, normals)
    J, r = tracker._assemble(state, data_corr, pose_corr)
    J = J.tocsr()
    J.sort_indices()
    out = dict(val=J.data, col=J.indices.astype(np.int32), rowptr=J.indptr.astype(np.int32),
               shape=np.array(J.shape), r=r)
    cases = [(1e-4, 32, 1e-6), (1e-2, 32, 1e-6), (1.0, 32, 1e-6), (1e-3, 400, 1e-12)]
    for i, (lam, it, tol) in enumerate(cases):
        out[f"x{i}"] = pcg_solve(J, r, lam, max_iters=it, tol=tol)
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "pcg_ref.npz"), **out)
    print("J", J.shape, "nnz", J.nnz)


if __name__ == "__main__":
    main()
