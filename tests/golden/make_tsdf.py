"""Golden TSDF vectors from the REAL reference (tsdf.py:17-176).

Run in the builder container (the only place /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tsdf.py
Writes tests/golden/tsdf_ref.npz: the inputs (depth maps, mask, camera, poses) and
the reference's volume after three integrations, sample / gradient values at random
points, the extracted surface and a stride-2 ray cast.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from capfields.camera import Camera  # noqa: E402
from capfields.transforms import Se3  # noqa: E402
from capfields.tsdf import TsdfVolume, tsdf_integrate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sphere_depth(cam: Camera, center, radius, back=1.9):
    """Ray-cast depth (camera z) of a sphere in front of a back plane z_world = back."""
    h, w = cam.height, cam.width
    us, vs = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    uv = np.stack([us.reshape(-1), vs.reshape(-1)], -1)
    o, d = cam.pixel_rays(uv)
    oc = o - center
    b = (d * oc).sum(-1)
    c = (oc * oc).sum(-1) - radius * radius
    disc = b * b - c
    t_s = np.where(disc > 0, -b - np.sqrt(np.maximum(disc, 0)), np.inf)
    t_p = np.where(np.abs(d[:, 2]) > 1e-9, (back - o[:, 2]) / d[:, 2], np.inf)
    t = np.minimum(t_s, np.where(t_p > 0, t_p, np.inf))
    pts = o + t[:, None] * d
    z = cam.world_to_cam().apply(pts)[:, 2]
    z = np.where(np.isfinite(t), z, 0.0)
    return z.reshape(h, w)


def main():
    rng = np.random.default_rng(11)
    cam = Camera(fx=71.3, fy=70.9, cx=31.7, cy=24.2, width=64, height=48,
                 pose=Se3.from_rotvec_trans(np.array([0.03, -0.05, 0.01]), np.array([0.02, -0.01, 0.0])))
    poses = [Se3.from_rotvec_trans(np.array([0.0, 0.1, 0.02]), np.array([0.01, 0.0, 0.05])),
             Se3.from_rotvec_trans(np.array([0.02, 0.12, 0.0]), np.array([0.015, -0.01, 0.05])),
             Se3.from_rotvec_trans(np.array([-0.01, 0.08, 0.03]), np.array([0.0, 0.01, 0.045]))]
    depths = [sphere_depth(cam, np.array([0.03, 0.01, 1.3]) + 0.004 * k, 0.237) for k in range(3)]
    depths[1][rng.random(depths[1].shape) < 0.03] = 0.0  # dropouts
    mask = np.ones((48, 64), np.uint8)
    mask[:, 40:] = 0
    vol = TsdfVolume(resolution=40, voxel_size=0.0173, origin=np.array([-0.3311, -0.3207, 0.9871]))
    tsdf_integrate(vol, depths[0], cam, poses[0])
    tsdf_integrate(vol, depths[1], cam, poses[1], mask=mask)
    tsdf_integrate(vol, depths[2], cam, poses[2])
    pts = vol.origin + rng.uniform(-0.05, 40 * 0.0173 + 0.05, size=(2000, 3))
    val, ok = vol.sample(pts)
    grad = vol.gradient(pts[:500])
    sp, sn = vol.extract_surface()
    rp, rn = vol.raycast(cam, poses[2], stride=2)
    np.savez_compressed(os.path.join(HERE, "tsdf_ref.npz"), depths=np.stack(depths), mask=mask,
             cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height]),
             cam_R=cam.pose.rotation, cam_t=cam.pose.translation,
             pose_R=np.stack([p.rotation for p in poses]), pose_t=np.stack([p.translation for p in poses]),
             vol=np.array([40, 0.0173, -0.3311, -0.3207, 0.9871, vol.truncation]),
             tsdf=vol.tsdf, weight=vol.weight, pts=pts, val=val, ok=ok, grad=grad,
             surf_p=sp, surf_n=sn, ray_p=rp, ray_n=rn)
    print("surface", len(sp), "raycast", len(rp), "observed", int((vol.weight > 0).sum()))


if __name__ == "__main__":
    main()
