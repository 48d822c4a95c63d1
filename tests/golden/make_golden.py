"""Generate the golden fixtures of stage 1 from the REAL reference package.

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
Writes tests/golden/stage1.npz. The GPU box never imports the reference; the
tests compare the CUDA path and the oracle against these committed vectors.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.config import RunConfig  # noqa: E402
from capfields.edgraph import EDGraph, GraphMotion, sample_ed_nodes, warp_backward_batch, warp_forward_batch  # noqa: E402
from capfields.knnfield import KnnField, brute_force_query  # noqa: E402
from capfields.skeleton import bone_weights, default_humanoid, lbs_batch, skinning_transforms  # noqa: E402
from capfields.synthetic import SyntheticScene  # noqa: E402
from capfields.transforms import DualQuaternion, dq_apply, dq_blend  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "stage1.npz")


def random_motion(n, rng, rot=0.3, trans=0.05):
    return np.stack([DualQuaternion.from_rotvec_trans(rot * rng.normal(size=3), trans * rng.normal(size=3)).packed()
                     for _ in range(n)])


def main():
    g = {}
    rng = np.random.default_rng(1234)

    # A. dual-quaternion blend + apply (transforms.py:174-196)
    dqs = random_motion(4 * 300, rng, rot=1.2, trans=0.3).reshape(300, 4, 8)
    dqs[::7, 2] *= -1.0  # antipodal entries exercise the sign alignment
    w = rng.uniform(0.0, 1.0, size=(300, 4))
    pts = rng.normal(size=(300, 3))
    b = dq_blend(w, dqs)
    g.update(A_dqs=dqs, A_w=w, A_pts=pts, A_blend=b, A_apply=dq_apply(b, pts))

    # B. ED warps over a random graph (edgraph.py:154-183, knnfield.py:32-42)
    nodes = rng.uniform(0.0, 1.0, size=(128, 3))
    graph = EDGraph(nodes, radius=0.1, knn_k=4)
    motion = GraphMotion(0, random_motion(128, rng, rot=0.2, trans=0.03))
    q = np.concatenate([nodes[rng.integers(0, 128, 2500)] + rng.normal(scale=0.04, size=(2500, 3)),
                        rng.uniform(-0.2, 1.2, size=(500, 3))])
    pc, valid = warp_backward_batch(graph, motion, q)
    fw, fvalid = warp_forward_batch(graph, motion, q)
    g.update(B_nodes=nodes, B_radius=0.1, B_dqs=motion.dqs, B_q=q, B_back=pc, B_back_valid=valid,
             B_fwd=fw, B_fwd_valid=fvalid)
    for s in (4, 8):
        idx, ww, pcs = brute_force_query(graph, motion, q, s)
        g[f"B_bf{s}_idx"], g[f"B_bf{s}_w"], g[f"B_bf{s}_pc"] = idx, ww, pcs

    # C. KnnField (knnfield.py:45-222)
    fnodes = np.random.default_rng(7).uniform(0.0, 1.0, size=(60, 3))
    fgraph = EDGraph(fnodes, radius=0.1)
    field = KnnField(fgraph, resolution=32, s=4)
    fm = GraphMotion(0, random_motion(60, rng, rot=0.15, trans=0.02))
    field.update_live_map(fm)
    fq = np.concatenate([fnodes[rng.integers(0, 60, 1500)] + rng.normal(scale=0.03, size=(1500, 3)),
                         rng.uniform(-0.3, 1.3, size=(300, 3))])
    nbr, fw_, fpc, fvalid_ = field.query_motion_batch(fq, 0)
    g.update(C_nodes=fnodes, C_dqs=fm.dqs, C_nidx=field.neighbor_idx, C_live=field.live_maps[0],
             C_bbox_min=field.bbox_min, C_voxel=field.voxel_size, C_q=fq, C_nbr=nbr, C_w=fw_, C_pc=fpc,
             C_valid=fvalid_)

    # D. skeleton / LBS (skeleton.py:121-188)
    skel = default_humanoid()
    theta = np.zeros(72)
    theta[1] = 0.7
    theta[3 * 16 + 2] = 0.35
    theta[3 * 18 + 2] = -0.5
    A = skinning_transforms(skel, theta)
    lp = rng.uniform(-0.6, 0.6, size=(400, 3)) + np.array([0.0, 1.0, 0.0])
    lw = bone_weights(skel, lp)
    g.update(D_theta=theta, D_A=A, D_pts=lp, D_w=lw, D_lbs=lbs_batch(skel, theta, lp, lw))

    # E. the C1 synthetic scene (synthetic.py:48-131)
    cfg = RunConfig(frames=10, spin_turns=0.25, arm_swing=0.4, node_radius=0.08, width=64, height=64,
                    fx=70.0, fy=70.0)
    scene = SyntheticScene(cfg, seed=0)
    sgraph = sample_ed_nodes(scene.template_points, 0.0805)
    d2 = np.sum((sgraph.nodes[:, None] - scene.template_points[None]) ** 2, axis=-1)
    node_bones = scene.template_bones[np.argmin(d2, axis=1)]
    prior = scene.gt_prior(7)
    from capfields.transforms import dq_from_rt
    A7 = skinning_transforms(scene.skeleton, scene.theta_at(7))
    dqs7 = np.stack([dq_from_rt(A7[b, :3, :3], A7[b, :3, 3]) for b in node_bones])
    sel = np.random.default_rng(0).choice(len(scene.template_points), 6890, replace=False)
    g.update(E_template_head=scene.template_points[:200], E_template_sum=scene.template_points.sum(axis=0),
             E_n_template=len(scene.template_points), E_nodes=sgraph.nodes, E_node_bones=node_bones,
             E_theta7=scene.theta_at(7), E_dqs7=dqs7, E_cam_R=scene.camera.pose.rotation,
             E_cam_t=scene.camera.pose.translation, E_skin_idx=sel, E_obj_pose7=scene.object_pose_abs(7).matrix(),
             E_skin_w_head=bone_weights(scene.skeleton, scene.template_points[sel[:300]]),
             E_prior_dqs_head=prior.graph_motion.dqs[:20])
    uv = np.stack(np.meshgrid(np.arange(64.0), np.arange(64.0)), -1).reshape(-1, 2)
    o, d = scene.camera.pixel_rays(uv)
    g.update(E_ray_o=o, E_ray_d=d)
    # samples of C1: 64 per ray at t_i = 0.3 + (i + 0.5) * 4.7 / 64, a 1/16 subset of the rays
    t = 0.3 + (np.arange(64) + 0.5) * (5.0 - 0.3) / 64
    sub = np.arange(0, 4096, 16)
    samp = (o[sub, None, :] + t[None, :, None] * d[sub, None, :]).reshape(-1, 3)
    sg = EDGraph(sgraph.nodes, radius=0.1, knn_k=4)
    sm = GraphMotion(7, dqs7)
    spc, svalid = warp_backward_batch(sg, sm, samp)
    sidx, sw, _ = brute_force_query(sg, sm, samp, 4)
    g.update(E_samples=samp, E_back=spc, E_back_valid=svalid, E_idx=sidx, E_w=sw)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
