"""ORACLE — the reference CPU implementation of a whole configs[1] frame (test
infrastructure and the CPU arms of bench.py only: `--impl reference` and the
`cpu_baseline` leg; the product never imports it).

A frame of the render back-end hot path on the host, standalone: no import of the
CUDA package and no device work. Everything the device path has is rebuilt here
from the same seeds:

  static (once per field, like the device's HumanField / ObjectField init):
    scene (synthetic generator, loaded from its source file without importing the
    package), the hash tables and MLP weights (same numpy RNG streams as
    render.HumanField / ObjectField), the canonical density bits (template shell,
    occ_from_points) and the object's box shell.
  per frame (timed):
    forward kinematics of theta (skinning_transforms, skeleton.py:121-139), the
    DeformNet pose bias, the live occupancy splat (occ_splat) ;
    per ray (process pool over all host cores): march -> hybrid canonicalisation
    (ED DQB^-1 / backward LBS, oracle/deform.py = the reference's transforms /
    edgraph / knnfield / skeleton restated in its float64 order) -> hash encode ->
    DeformNet / E_g / E_c in the SPEC's 32-bit semantics -> composite ;
    then the depth-occlusion layer composite.
"""
from __future__ import annotations

import importlib.util
import math
import os
import sys

import numpy as np

from . import deform as od
from . import nrf as on
from . import render as orr

CANON = (16, 2, 19, 16, 2048)
DEFORM = (8, 4, 17, 16, 256)
WORLD_MIN = (-1.3, -0.3, -1.3)
WORLD_SIZE = 2.6
LIVE_RES = CANON_RES = 128
OBJ_RES = 64
BACKGROUND = (24 / 255.0, 28 / 255.0, 34 / 255.0)


def load_scene_module():
    """paper_2304_03184_b200/scene.py (pure numpy) by path: the package itself, and with
    it the CUDA library, is never imported."""
    if "_cf_scene_src" in sys.modules:
        return sys.modules["_cf_scene_src"]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("_cf_scene_src",
                                                  os.path.join(root, "paper_2304_03184_b200", "scene.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_cf_scene_src"] = mod
    spec.loader.exec_module(mod)
    return mod


def _kaiming(rng, n_out, n_in):
    b = np.sqrt(6.0 / n_in)
    return rng.uniform(-b, b, size=(n_out, n_in))


def field_layers(rng, deform, zero_deform_out=False):
    """render.FieldNets' draw order."""
    L = {}
    if deform:
        L["D1"] = _kaiming(rng, 128, 104)
        for i in (2, 3, 4):
            L[f"D{i}"] = _kaiming(rng, 128, 128)
        L["D5"] = np.zeros((3, 128)) if zero_deform_out else _kaiming(rng, 3, 128) * 0.1
    L["G1"] = _kaiming(rng, 64, 32)
    L["G2"] = _kaiming(rng, 16, 64)
    L["C1"] = _kaiming(rng, 64, 31)
    L["C2"] = _kaiming(rng, 64, 64)
    L["C3"] = _kaiming(rng, 3, 64)
    return {k: np.asarray(v, dtype=np.float32) for k, v in L.items()}


def hash_table(grid, seed, scale):
    """nrf.HashGrid's seeded initialisation."""
    L, F, log2T, nmin, nmax = grid
    _, total = on.hash_levels(L, log2T, nmin, nmax)
    return np.random.default_rng(seed).uniform(-scale, scale, size=(total, F)).astype(np.float32)


def build_static(width=512, height=512, samples=128, table_scale=1e-4, seed=0):
    """Scene, fields and static occupancy of bench.py's workload (bench.build_workload)."""
    sm = load_scene_module()
    sc = sm.Scene(sm.SceneConfig(width=width, height=height), seed=0)
    nodes = np.asarray(sc.nodes, dtype=np.float64)
    lo, hi = nodes.min(0), nodes.max(0)
    side = float((hi - lo).max() + 2 * 0.15)
    cmin = (lo + hi) / 2 - side / 2
    rng = np.random.default_rng(seed)
    human = {"ctable": hash_table(CANON, seed + 1, table_scale), "dtable": hash_table(DEFORM, seed + 2, table_scale),
             "layers": field_layers(rng, True), "cmin": cmin, "side": side, "inv_side": 1.0 / side}
    ocell = side / CANON_RES
    human["canon_on"] = orr.occ_from_points(np.asarray(sc.template_points), cmin, ocell, CANON_RES, 0.03)
    half = np.asarray(sc.box_half, dtype=np.float64)
    oside = float(2 * half.max() + 2 * 0.05)
    orng = np.random.default_rng(1)
    obj = {"ctable": hash_table(CANON, 1 + 11, table_scale), "layers": field_layers(orng, False),
           "omin": -np.full(3, oside / 2), "side": oside, "inv_side": 1.0 / oside}
    obj["on"] = orr.occ_box_shell(obj["omin"], oside / OBJ_RES, OBJ_RES, half, 0.02)
    o, d = sc.camera.all_rays()
    return {"scene": sc, "human": human, "object": obj, "origin": np.asarray(sc.camera.t, dtype=np.float64),
            "dirs": d, "samples": samples, "t_near": 0.3, "t_far": 5.0, "dt": (5.0 - 0.3) / samples,
            "nodes": nodes, "width": width, "height": height}


def frame_setup(S, fid):
    """Per-frame setup: FK, pose bias, live occupancy (the device's setup kernels)."""
    sc = S["scene"]
    theta = sc.theta(fid)
    A = od.bone_transforms(load_scene_module().PARENTS, _offsets(), theta)
    dqs = sc.node_dqs(fid)
    W = S["human"]["layers"]["D1"][:, 32:]
    dbias = (W @ np.asarray(theta, dtype=np.float32)).astype(np.float32)
    h = S["human"]
    live = orr.occ_splat(h["canon_on"], (h["cmin"], h["side"] / CANON_RES, CANON_RES), S["nodes"], dqs, 4, 0.1,
                         (WORLD_MIN, WORLD_SIZE / LIVE_RES, LIVE_RES))
    R, t = sc.object_pose(fid)
    return {"fid": fid, "A": A, "dqs": dqs, "dbias": dbias, "live_bits": np.packbits(live, bitorder="little"),
            "R": R, "t": t}


def _offsets():
    return np.asarray(load_scene_module().OFFSETS, dtype=np.float64)


def render_rays(S, F, ray_ids, precision="fp32"):
    """March + canonicalise + field + composite of the given rays of frame F.
    -> (n_human_samples, n_object_samples, {field: (rgb, depth, opacity)} per ray)."""
    sc = S["scene"]
    live = np.unpackbits(F["live_bits"], bitorder="little")[:LIVE_RES ** 3].astype(bool)
    h, ob = S["human"], S["object"]
    dirs = S["dirs"][ray_ids]
    lg = (list(WORLD_MIN), WORLD_SIZE / LIVE_RES, LIVE_RES)
    og = (list(ob["omin"]), ob["side"] / OBJ_RES, OBJ_RES)
    m = orr.march(S["origin"], dirs, S["samples"], S["t_near"], S["dt"], live, lg, ob["on"], og, F["R"], F["t"])
    counts, out = [], {}
    for name in ("human", "object"):
        rr, ii = m[name]
        counts.append(len(rr))
        if len(rr) == 0:
            out[name] = (np.zeros((len(ray_ids), 3)), np.zeros(len(ray_ids)), np.zeros(len(ray_ids)))
            continue
        p = orr.sample_points(S["origin"], dirs, rr, ii, S["t_near"], S["dt"])
        d = dirs[rr]
        if name == "human":
            xu = orr.human_canon(p, S["nodes"], F["dqs"], 4, 0.1, F["A"], sc.skin_verts, sc.skin_weights, 0.2,
                                 h["cmin"], h["inv_side"])
            f = orr.field_forward(h["layers"], True, xu, d, h["ctable"], h["dtable"], F["dbias"], h["inv_side"],
                                  precision=precision)
        else:
            xu = orr.object_canon(p, F["R"], F["t"], ob["omin"], ob["inv_side"])
            f = orr.field_forward(ob["layers"], False, xu, d, ob["ctable"], precision=precision)
        out[name] = orr.composite(len(ray_ids), rr, ii, f, S["t_near"], S["dt"])
    return counts[0], counts[1], out


# ---- process pool over the host cores (spawned workers; each builds the static state once)

_STATE = {}


def _init_worker(kw):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    try:
        from threadpoolctl import threadpool_limits
        _STATE["limits"] = threadpool_limits(1)
    except Exception:
        pass
    _STATE["S"] = build_static(**kw)


def _work(args):
    F, ray_ids, precision = args
    nh, no, out = render_rays(_STATE["S"], F, ray_ids, precision)
    return nh, no, ray_ids, out


class FramePool:
    """All host cores render one frame: the frame's rays are split into chunks over
    spawned worker processes; the parent runs the per-frame setup and the layer
    composite."""

    def __init__(self, cores=None, **static_kw):
        import multiprocessing as mp
        self.cores = int(cores or os.cpu_count() or 1)
        self.kw = static_kw
        self.S = build_static(**static_kw)
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_init_worker, initargs=(static_kw,))

    def close(self):
        self.pool.close()
        self.pool.join()

    def frame(self, fid, ray_ids=None, precision="fp32", chunks_per_core=4):
        """One frame (or the given subset of its rays) -> (human samples, object samples, image, layer)."""
        S = self.S
        F = frame_setup(S, fid)
        n = S["dirs"].shape[0]
        ray_ids = np.arange(n) if ray_ids is None else np.asarray(ray_ids)
        parts = np.array_split(ray_ids, max(1, self.cores * chunks_per_core))
        res = self.pool.map(_work, [(F, p, precision) for p in parts if len(p)])
        nh = sum(r[0] for r in res)
        no = sum(r[1] for r in res)
        R = len(ray_ids)
        pos = {int(r): i for i, r in enumerate(ray_ids)} if R != n else None
        acc = {k: (np.zeros((R, 3)), np.zeros(R), np.zeros(R)) for k in ("human", "object")}
        for _, _, ids, out in res:
            sel = ids if pos is None else np.array([pos[int(r)] for r in ids])
            for k in acc:
                for a, b in zip(acc[k], out[k]):
                    a[sel] = b
        img, layer = orr.layers(acc["human"], acc["object"], BACKGROUND)
        return nh, no, img, layer



def train_rays(S, fid, ray_ids, seed=1234):
    """The key-frame training step's human-field work for the given pixels of frame
    fid on the host: depth-guided samples, hybrid canonicalisation, the
    field forward and the 64-bit analytic gradient of masked L2 + 0.1 L1 depth with
    respect to every human parameter (oracle/grad.py), then one Adam update (numpy).
    -> number of samples processed. (CPU baseline of bench.py --workload train.)"""
    from . import grad as og
    sc = S["scene"]
    F = frame_setup(S, fid)
    h = S["human"]
    o = S["origin"]
    d = S["dirs"][ray_ids]
    th, to, rgb, hum, obj = sc.raycast(np.broadcast_to(o, d.shape), d, fid)
    depth = np.where(hum, th, 0.0)
    ts = orr.train_samples(depth, hum, S["t_near"], S["t_far"], 32, 16, 64, 0.02, seed)
    ray = np.concatenate([np.full(len(t), q) for q, t in enumerate(ts) if t is not None]).astype(np.int64)
    t = np.concatenate([t for t in ts if t is not None])
    if len(t) == 0:
        return 0
    p = o + t[:, None] * d[ray]
    verts, vw = np.asarray(sc.skin_verts), np.asarray(sc.skin_weights)
    xu = orr.human_canon(p, S["nodes"], F["dqs"], 4, 0.1, F["A"], verts, vw, 0.2, h["cmin"], h["inv_side"])
    delta = np.empty(len(t))
    last = np.append(ray[1:] != ray[:-1], True)
    delta[:-1] = t[1:] - t[:-1]
    delta[last] = S["dt"]
    batch = {"xu": xu, "dirs": d[ray], "ray": ray, "t": t, "delta": delta, "gt_rgb": rgb.astype(np.float64),
             "gt_depth": depth, "mask": hum, "inv_side": h["inv_side"], "theta": sc.theta(fid)}
    values = {"ctable": h["ctable"], "dtable": h["dtable"]}
    values.update({k: v for k, v in h["layers"].items()})
    _, g = og.gradients(values, batch)
    for k, v in values.items():  # one Adam step (first-step moments)
        m = 0.1 * g[k]
        vv = 0.01 * g[k] ** 2
        lr = 1e-2 if k.endswith("table") else 1e-3
        values[k] = v - lr * (m / 0.1) / (np.sqrt(vv / 0.01) + 1e-15)
    return len(t)
