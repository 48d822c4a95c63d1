"""Golden CFMP motion-prior stream written by the REAL reference writer.

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_records.py
Writes tests/golden/motions_ref.bin (records.py:103-120, as the reference's own
round-trip test builds it, tests/test_io.py:124-151) and motions_ref.npz with the
arrays that went in plus the reference's skinning_transforms of every pose
(skeleton.py:135-139), so the CPU codec tests and the device-FK test need no
reference at run time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.edgraph import GraphMotion  # noqa: E402
from capfields.records import MotionPrior, MotionPriorWriter, load_motion_priors  # noqa: E402
from capfields.skeleton import SkeletonPose, default_humanoid, skinning_transforms  # noqa: E402
from capfields.transforms import DualQuaternion, Se3  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    skel = default_humanoid()
    rng = np.random.default_rng(1)
    path = os.path.join(HERE, "motions_ref.bin")
    fids, dqs_all, thetas, rots, trans = [], [], [], [], []
    with MotionPriorWriter(path, n_nodes=5, n_theta=72) as wr:
        for t in range(6):
            dqs = np.stack([DualQuaternion.from_rotvec_trans(rng.normal(size=3), rng.normal(size=3)).packed()
                            for _ in range(5)])
            theta = rng.normal(size=72) * (0.1 if t < 4 else 1.5)
            if t == 5:
                theta[::3] = 0.0
                theta[:9] = 0.0  # zero-angle joints take the small-angle branch
            fid = [0, 1, 2, 3, 7, 42][t]
            pose = Se3.from_rotvec_trans(rng.normal(size=3) * 0.1, rng.normal(size=3))
            wr.append(MotionPrior(fid, GraphMotion(fid, dqs), SkeletonPose(skel, theta), pose))
            fids.append(fid)
            dqs_all.append(dqs)
            thetas.append(theta)
            rots.append(pose.rotation)
            trans.append(pose.translation)
    back = load_motion_priors(path, skel)
    assert len(back) == 6
    A = np.stack([skinning_transforms(skel, th) for th in thetas])
    np.savez(os.path.join(HERE, "motions_ref.npz"), frame_ids=np.array(fids, dtype=np.int64),
             dqs=np.stack(dqs_all), theta=np.stack(thetas), rot=np.stack(rots), trans=np.stack(trans), bone_A=A,
             parents=np.asarray(skel.parents, dtype=np.int32), offsets=np.asarray(skel.offsets, dtype=np.float64))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
