"""CPU restatement of the key-frame module — TEST INFRASTRUCTURE ONLY.

Only tests/ (and bench.py's CPU legs) may import this; the product path is
csrc/keyframes.cu behind paper_2304_03184_b200/keyframes.py.

The reference package has no key-frame code: the operations are specified in
SPEC.md:434-519 (module `keyframes`) and PAPER.md:250-298 (Eq. 5-7). Parity is
therefore pinned by SPEC's worked examples (tests/test_keyframes.py) — "parity
unpinned" by reference code. The choices SPEC leaves open are frozen here (and in
DESIGN.md §3.6) and restated exactly by the kernels:

* blur_score (Crété-Roffet): luma Y = 299 R + 587 G + 114 B (exact
  integers, BT.601 weights x 1000); 9-tap box re-blur along each axis with clamped
  borders kept as the unnormalised 9-sum S; per axis, over every pixel with a
  predecessor on that axis: D_F = |Y - Y_prev|, D_B = |S - S_prev|,
  V = max(0, 9 D_F - D_B), s_F = sum 9 D_F, s_V = sum V (int64, exact);
  b = (s_F - s_V) / s_F (1.0 when s_F = 0); score = max(b_vertical, b_horizontal).
* visibility_map (Eq. 5): camera-frame point pc = R_wc p + t_wc
  evaluated as ((p0 R_k0 + p1 R_k1) + p2 R_k2) + t_k; u = fx pc0 / z + cx,
  v = fy pc1 / z + cy; inside iff z > 0 and 0 <= u <= W-1, 0 <= v <= H-1
  (camera.py:65-79); pixel = round-half-even(u, v) (tracking.py:103-106);
  bit = inside and D > 0 and |z - D| < eps.
* dissim_human (Eq. 6): sum_k beta_k (dtheta_k * dtheta_k) accumulated k = 0..71,
  then + beta_vis * popcount(s_a xor s_b), then + beta_h * (dt * dt); beta_k = 0.1
  for the components of torso joints, 0.02 otherwise.
* dissim_object (Eq. 7): beta_d ((dx dx + dy dy) + dz dz) + beta_o (dt dt).
* pool_update: insert iff the pool is empty or
  min_e dissim(candidate, e) > gamma; a full pool first evicts the entry with the
  smallest dissimilarity to the candidate, ties -> oldest (smallest t).
* refinement_set: the m pool entries least dissimilar to the
  render view (ties -> oldest), then the m most recent frames, duplicates removed.
"""
from __future__ import annotations

import numpy as np

TORSO_JOINTS = (0, 3, 6, 9, 12, 13, 14, 15)  # skeleton.py default_humanoid torso mask
BETA_TORSO, BETA_LIMB, BETA_VIS, BETA_H = 0.1, 0.02, 0.01, 0.02
BETA_D, BETA_O = 1.0, 0.02
GAMMA, CAPACITY = 2.5, 100


def pose_weights(n_joints: int = 24, torso=TORSO_JOINTS) -> np.ndarray:
    w = np.full(3 * n_joints, BETA_LIMB)
    for j in torso:
        w[3 * j: 3 * j + 3] = BETA_TORSO
    return w


def luma(rgb: np.ndarray) -> np.ndarray:
    rgb = np.asarray(rgb, dtype=np.int64)
    return 299 * rgb[..., 0] + 587 * rgb[..., 1] + 114 * rgb[..., 2]


def blur_sums(rgb: np.ndarray) -> tuple[int, int, int, int]:
    """(s_F_vertical, s_V_vertical, s_F_horizontal, s_V_horizontal), exact int64."""
    Y = luma(rgb)
    H, W = Y.shape
    out = []
    for axis, n in ((0, H), (1, W)):
        idx = np.arange(n)
        S = sum(np.take(Y, np.clip(idx + d, 0, n - 1), axis=axis) for d in range(-4, 5))
        if axis == 0:
            dF, dB = np.abs(Y[1:] - Y[:-1]), np.abs(S[1:] - S[:-1])
        else:
            dF, dB = np.abs(Y[:, 1:] - Y[:, :-1]), np.abs(S[:, 1:] - S[:, :-1])
        out += [int((9 * dF).sum()), int(np.maximum(0, 9 * dF - dB).sum())]
    return tuple(out)


def blur_from_sums(sfv: int, svv: int, sfh: int, svh: int) -> float:
    bv = 1.0 if sfv == 0 else float(sfv - svv) / float(sfv)
    bh = 1.0 if sfh == 0 else float(sfh - svh) / float(sfh)
    return max(bv, bh)


def blur_score(rgb: np.ndarray) -> float:
    rgb = np.asarray(rgb)
    if rgb.shape[0] < 16 or rgb.shape[1] < 16:
        raise ValueError("blur_score needs an image of at least 16x16")
    return blur_from_sums(*blur_sums(rgb))


def visibility_map(nodes, depth, R_wc, t_wc, fx, fy, cx, cy, eps=0.01) -> np.ndarray:
    """-> bool (n,) (Eq. 5); see the module docstring for the exact evaluation."""
    p = np.asarray(nodes, dtype=np.float64)
    depth = np.asarray(depth, dtype=np.float64)
    H, W = depth.shape
    R = np.asarray(R_wc, dtype=np.float64)
    t = np.asarray(t_wc, dtype=np.float64)
    pc = [((p[:, 0] * R[k, 0] + p[:, 1] * R[k, 1]) + p[:, 2] * R[k, 2]) + t[k] for k in range(3)]
    z = pc[2]
    ok = z > 0
    zs = np.where(ok, z, 1.0)
    u = fx * pc[0] / zs + cx
    v = fy * pc[1] / zs + cy
    ok &= (u >= 0) & (u <= W - 1) & (v >= 0) & (v <= H - 1)
    ui = np.where(ok, np.round(u), 0).astype(np.int64)
    vi = np.where(ok, np.round(v), 0).astype(np.int64)
    D = depth[vi, ui]
    return ok & (D > 0) & (np.abs(z - D) < eps)


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """bool (n,) -> uint32 words, bit i of word i // 32 = node i."""
    bits = np.asarray(bits, dtype=bool)
    words = np.zeros((len(bits) + 31) // 32, dtype=np.uint32)
    for i in np.nonzero(bits)[0]:
        words[i // 32] |= np.uint32(1) << np.uint32(i % 32)
    return words


def popcount_xor(a: np.ndarray, b: np.ndarray) -> int:
    x = np.bitwise_xor(np.asarray(a, dtype=np.uint32), np.asarray(b, dtype=np.uint32))
    return int(sum(bin(int(w)).count("1") for w in x))


def dissim_human(theta_a, vis_a, t_a, theta_b, vis_b, t_b, beta=None) -> float:
    beta = pose_weights() if beta is None else beta
    acc = 0.0
    for k in range(len(beta)):
        d = float(theta_a[k]) - float(theta_b[k])
        acc = acc + float(beta[k]) * (d * d)
    dt = float(t_a) - float(t_b)
    return (acc + BETA_VIS * float(popcount_xor(vis_a, vis_b))) + BETA_H * (dt * dt)


def dissim_object(d_a, t_a, d_b, t_b) -> float:
    dx, dy, dz = (float(d_a[i]) - float(d_b[i]) for i in range(3))
    dt = float(t_a) - float(t_b)
    return BETA_D * ((dx * dx + dy * dy) + dz * dz) + BETA_O * (dt * dt)


def pool_decision(dissims, ts, capacity=CAPACITY, gamma=GAMMA):
    """-> (insert, evict_index or -1) for a candidate with dissimilarities `dissims`
    to the pool entries (insertion times `ts`)."""
    P = len(dissims)
    if P == 0:
        return True, -1
    if min(dissims) <= gamma:
        return False, -1
    if P < capacity:
        return True, -1
    best = 0
    for e in range(1, P):
        if dissims[e] < dissims[best] or (dissims[e] == dissims[best] and ts[e] < ts[best]):
            best = e
    return True, best


def refinement_order(dissims, ts, m):
    """Pool indices of the m least dissimilar entries (ties -> oldest)."""
    order = sorted(range(len(dissims)), key=lambda e: (dissims[e], ts[e]))
    return order[:m]
