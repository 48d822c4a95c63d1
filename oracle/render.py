"""ORACLE (test infrastructure only) — the render path on the CPU, stage by stage.

Each function restates one device stage of DESIGN.md §3-§6 (SPEC.md:372-407,
555-563 plus the builder-defined occupancy) with the same float64 / float32
operation order where the stage produces indices or decisions, so those are
compared bit-exactly; the field and composite stages are compared within the
tolerances stated in tests/test_render_gpu.py.
"""
from __future__ import annotations

import numpy as np

from . import deform as od
from . import nrf as on


def unpack_bits(words, n):
    b = np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")
    return b[:n].astype(bool)


def cell_centers(gmin, cell, res, flat):
    r = res
    ijk = np.stack([flat // (r * r), (flat // r) % r, flat % r], -1).astype(np.float64)
    return np.asarray(gmin, dtype=np.float64) + (ijk + 0.5) * cell


def cell_of(p, gmin, cell, res):
    """flat index and inside flag: floor((p - min) * (1 / cell)) in [0, res) (render.cu:occ_test)."""
    f = np.floor((p - np.asarray(gmin, dtype=np.float64)) * (1.0 / cell))
    inside = np.all((f >= 0) & (f < res), axis=-1)
    fi = np.where(inside[:, None], f, 0).astype(np.int64)
    return (fi[:, 0] * res + fi[:, 1]) * res + fi[:, 2], inside


def _sqd(a, b):
    d = a - b
    return (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]


def occ_from_points(points, gmin, cell, res, radius):
    from scipy.spatial import cKDTree
    flat = np.arange(res ** 3)
    c = cell_centers(gmin, cell, res, flat)
    tree = cKDTree(points)
    d, j = tree.query(c, k=4, distance_upper_bound=radius * 1.001 + 1e-9)
    on = np.zeros(len(c), dtype=bool)
    for col in range(4):
        ok = np.isfinite(d[:, col])
        jj = np.where(ok, j[:, col], 0)
        on |= ok & (_sqd(c, points[jj]) <= radius * radius)
    return on


def occ_box_shell(gmin, cell, res, half, shell):
    c = cell_centers(gmin, cell, res, np.arange(res ** 3))
    q = np.abs(c) - np.asarray(half)
    m = np.maximum(q, 0.0)
    o = np.sqrt((m[:, 0] * m[:, 0] + m[:, 1] * m[:, 1]) + m[:, 2] * m[:, 2])
    inn = np.minimum(np.maximum(q[:, 0], np.maximum(q[:, 1], q[:, 2])), 0.0)
    return (o + inn) <= shell


def occ_splat(canon_on, cg, nodes, dqs, k, radius, lg):
    """Forward-warp occupied canonical cell centres, set 3x3x3 live cells."""
    cmin, ccell, cres = cg
    lmin, lcell, lres = lg
    flat = np.nonzero(canon_on)[0]
    x = cell_centers(cmin, ccell, cres, flat)
    _, _, xl, valid = od.warp(nodes, radius, k, dqs, x, "forward")
    xl = xl[valid]
    f = np.floor((xl - np.asarray(lmin)) / lcell)
    ok = np.all((f >= -1) & (f <= lres), axis=1)
    f = f[ok].astype(np.int64)
    live = np.zeros(lres ** 3, dtype=bool)
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                g = f + np.array([dx, dy, dz])
                inb = np.all((g >= 0) & (g < lres), axis=1)
                g = g[inb]
                live[(g[:, 0] * lres + g[:, 1]) * lres + g[:, 2]] = True
    return live


def sample_t(t_near, dt, i):
    return t_near + (np.asarray(i, dtype=np.float64) + 0.5) * dt


def sample_points(origin, dirs, ray, i, t_near, dt):
    t = sample_t(t_near, dt, i)
    return np.asarray(origin)[None] + t[:, None] * dirs[ray]


def to_object(p, R, t):
    q = p - np.asarray(t)
    R = np.asarray(R).reshape(3, 3)
    return np.stack([(q[:, 0] * R[0, i] + q[:, 1] * R[1, i]) + q[:, 2] * R[2, i] for i in range(3)], -1)


def march(origin, dirs, S, t_near, dt, live_on, lg, obj_on=None, og=None, objR=None, objt=None):
    """Per field: (ray, i) of every occupied sample, rays ascending, i ascending."""
    n = len(dirs)
    ray = np.repeat(np.arange(n), S)
    i = np.tile(np.arange(S), n)
    p = sample_points(origin, dirs, ray, i, t_near, dt)
    out = {}
    f, ins = cell_of(p, *lg)
    keep = ins & live_on[f]
    out["human"] = (ray[keep], i[keep])
    if obj_on is not None:
        f, ins = cell_of(to_object(p, objR, objt), *og)
        keep = ins & obj_on[f]
        out["object"] = (ray[keep], i[keep])
    return out


def human_canon(p, nodes, dqs, k, radius, A, verts, vweights, max_dist, cmin, inv_side):
    """ED DQB^-1 warp, backward-LBS fallback; -> xu float32 (N,4) (x,y,z,flag)."""
    _, _, pt, ved = od.warp(nodes, radius, k, dqs, p, "backward")
    flag = np.where(ved, 1.0, 0.0)
    if A is not None and (~ved).any():
        _, pl, vl, _ = od.lbs_backward(A, verts, vweights, p[~ved], max_dist)
        sub = pt[~ved]
        sub[vl] = pl[vl]
        pt[~ved] = sub
        fl = flag[~ved]
        fl[vl] = 2.0
        flag[~ved] = fl
    xu = ((pt - np.asarray(cmin)) * inv_side).astype(np.float32)
    xu[flag == 0] = 0.0
    return np.concatenate([xu, flag[:, None].astype(np.float32)], axis=1)


def object_canon(p, R, t, omin, inv_side):
    """Object-local unit-cube coordinates + flag: the object field is defined on its box
    (the render's object grid); a sample outside [0, 1]^3 is empty (flag 0, xu 0)."""
    q = to_object(p, R, t)
    xu = ((q - np.asarray(omin)) * inv_side).astype(np.float32)
    inside = np.all((xu >= 0) & (xu <= 1), axis=1)
    xu[~inside] = 0.0
    return np.concatenate([xu, inside[:, None].astype(np.float32)], axis=1)


def sh16(d):
    x, y, z = (d[:, i].astype(np.float32) for i in range(3))
    xx, yy, zz = x * x, y * y, z * z
    return np.stack([
        np.full_like(x, 0.28209479177387814), -0.48860251190291987 * y, 0.48860251190291987 * z,
        -0.48860251190291987 * x, 1.0925484305920792 * x * y, -1.0925484305920792 * y * z,
        0.94617469575755997 * zz - 0.31539156525251999, -1.0925484305920792 * x * z,
        0.54627421529603959 * (xx - yy), 0.59004358992664352 * y * (-3.0 * xx + yy), 2.8906114426405538 * x * y * z,
        0.45704579946446572 * y * (1.0 - 5.0 * zz), 0.3731763325901154 * z * (5.0 * zz - 3.0),
        0.45704579946446572 * x * (1.0 - 5.0 * zz), 1.4453057213202769 * z * (xx - yy),
        0.59004358992664352 * x * (-xx + 3.0 * yy)], -1).astype(np.float32)


def deform_forward(layers, fd, dbias, precision="fp32"):
    """DeformNet raw outputs (N,3) float64 from the deformation-grid features fd."""
    mlp = on.mlp_forward_f32 if precision == "fp32" else on.mlp_forward
    Ws = [layers["D1"][:, :32], layers["D2"], layers["D3"], layers["D4"], layers["D5"]]
    return mlp(Ws, fd, [dbias, None, None, None, None])[:, :3]


def deformed_coords(xu, v, inv_side):
    """xc = xu + 0.05 tanh(v) / side in float32 (field.cu deform_mlp epilogue)."""
    x = xu[:, :3].astype(np.float32).copy()
    delta = np.float32(0.05) * np.tanh(v.astype(np.float32))
    return x + delta * np.float32(inv_side)


def color_forward(layers, fc, dirs, precision="fp32"):
    """E_g / E_c from the canonical features fc -> (N,4) float32 (sigma, r, g, b)."""
    mlp = on.mlp_forward_f32 if precision == "fp32" else on.mlp_forward
    g = mlp([layers["G1"], layers["G2"]], fc).astype(np.float32)
    sigma = np.exp(g[:, 0])
    cin = np.concatenate([g[:, 1:16], sh16(dirs)], axis=1)
    c = mlp([layers["C1"], layers["C2"], layers["C3"]], cin).astype(np.float32)
    rgb = 1.0 / (1.0 + np.exp(-c[:, :3]))
    return np.concatenate([sigma[:, None], rgb], axis=1).astype(np.float32)


def field_forward(layers, has_deform, xu, dirs, ctable, dtable=None, dbias=None, inv_side=1.0,
                  cgrid=(16, 2, 19, 16, 2048), dgrid=(8, 4, 17, 16, 256), precision="fp16"):
    """Field -> (N,4) float32 (sigma, r, g, b); zeros where flag == 0.
    precision "fp32": SPEC 32-bit semantics (fp32 tables, features and weights);
    "fp16": kernel precision of the fp16 device mode (fp16 MLP operands; pass the
    fp16-rounded deformation table the kernels read)."""
    x = xu[:, :3].astype(np.float32).copy()
    valid = xu[:, 3] > 0
    if has_deform:
        fd = on.hash_encode(dtable, x, *dgrid)
        x = deformed_coords(xu, deform_forward(layers, fd, dbias, precision), inv_side)
    fc = on.hash_encode(ctable, x, *cgrid)
    if precision == "fp16":
        fc = fc.astype(np.float16).astype(np.float32)  # the kernels hand fp16 features to the MLP
    out = color_forward(layers, fc, dirs, precision)
    out[~valid] = 0.0
    return out


def composite(n_rays, ray, i, field, t_near, dt, t_term=1e-4):
    """Front-to-back compositing with early termination."""
    rgb = np.zeros((n_rays, 3))
    depth = np.zeros(n_rays)
    opac = np.zeros(n_rays)
    order = np.lexsort((i, ray))
    ray, i, field = ray[order], i[order], field[order]
    bounds = np.searchsorted(ray, np.arange(n_rays + 1))
    dtf = np.float32(dt)
    for r in range(n_rays):
        a, b = bounds[r], bounds[r + 1]
        T = 1.0
        for j in range(a, b):
            s, cr, cg, cb = field[j]
            alpha = 1.0 - np.exp(-float(s) * float(dtf))
            w = T * alpha
            rgb[r] += w * np.array([cr, cg, cb])
            depth[r] += w * sample_t(t_near, dt, i[j])
            opac[r] += w
            T *= 1.0 - alpha
            if T < t_term:
                break
    return rgb, depth / np.maximum(opac, 1e-6), opac


def layers(h, o, bg):
    """Depth-occlusion composite -> (rgb, layer)."""
    n = len(bg) if h is None and o is None else len((h or o)[0])
    hr, hd, ho = h if h is not None else (None, None, np.zeros(n))
    orr, odd, oo = o if o is not None else (None, None, np.zeros(n))
    hon, oon = ho > 0.5, oo > 0.5
    L = np.zeros(n, dtype=np.uint8)
    both = hon & oon
    L[both] = np.where(hd[both] <= odd[both], 1, 2)
    L[hon & ~oon] = 1
    L[oon & ~hon] = 2
    out = np.tile(np.asarray(bg, dtype=np.float32), (n, 1))
    if hr is not None:
        out[L == 1] = hr[L == 1]
    if orr is not None:
        out[L == 2] = orr[L == 2]
    return out, L


# ----------------------------------------------------------------- training sampler

def u01(seed, ray, j):
    """splitmix64(seed + golden * (ray*64 + j + 1)) -> [0,1) with 53 bits (render.cu:u01)."""
    M64 = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (ray * 64 + j + 1)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return float(z >> 11) * 2.0 ** -53


def train_samples(gt_depth, mask, t_near, t_far, n_guided, n_uniform, n_empty, sigma_d, seed):
    """Depth-guided samples per ray -> list of sorted t arrays (None for unmasked)."""
    out = []
    for ray, (d, m) in enumerate(zip(gt_depth, mask)):
        if not m:
            out.append(None)
            continue
        strat = lambda lo, hi, n, j, slot: lo + ((j + u01(seed, ray, slot)) / n) * (hi - lo)  # noqa: E731
        if not d > 0:
            out.append(np.array([strat(t_near, t_far, n_empty, j, j) for j in range(n_empty)]))
            continue
        lo = max(t_near, float(d) - 6.0 * sigma_d)
        hi = min(t_far, float(d) + 6.0 * sigma_d)
        a = [strat(lo, hi, n_guided, j, j) for j in range(n_guided)]
        b = [strat(t_near, t_far, n_uniform, j, 32 + j) for j in range(n_uniform)]
        merged, i, k = [], 0, 0
        while i < len(a) or k < len(b):
            if k >= len(b) or (i < len(a) and a[i] <= b[k]):
                merged.append(a[i]); i += 1
            else:
                merged.append(b[k]); k += 1
        out.append(np.array(merged))
    return out


def density_logits(table, W1, W2, res):
    """E_g density logit g0 at every cell centre u = (i + 0.5) / res of a res^3 grid,
    x-major, restating density_grid_kernel (field.cu) bit for bit: hash features as
    hash_encode (fp32, bit-exact with the kernels), then un-contracted fp32 sums in the
    kernel's order: a_j = sum_i W1[j, i] f_i (i ascending), g0 = sum_j W2[0, j] relu(a_j)."""
    u = ((np.arange(res, dtype=np.float64) + 0.5) / res).astype(np.float32)
    x, y, z = np.meshgrid(u, u, u, indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)
    f = on.hash_encode(table, pts).astype(np.float32)
    W1 = np.asarray(W1, dtype=np.float32)
    W2 = np.asarray(W2, dtype=np.float32)
    g0 = None
    for j in range(64):
        a = W1[j, 0] * f[:, 0]
        for i in range(1, 32):
            a = a + W1[j, i] * f[:, i]
        h = np.maximum(a, np.float32(0))
        g0 = W2[0, 0] * h if j == 0 else g0 + W2[0, j] * h
    return g0


def dilate_box(on_grid, r):
    """Chebyshev (box) dilation of a (res, res, res) bool grid by r cells per axis, no wrap."""
    out = on_grid.copy()
    for axis in range(3):
        src = out.copy()
        n = src.shape[axis]
        for k in range(1, r + 1):
            if k >= n:
                break
            sl_dst = [slice(None)] * 3
            sl_src = [slice(None)] * 3
            sl_dst[axis], sl_src[axis] = slice(k, None), slice(0, n - k)
            out[tuple(sl_dst)] |= src[tuple(sl_src)]
            sl_dst[axis], sl_src[axis] = slice(0, n - k), slice(k, None)
            out[tuple(sl_dst)] |= src[tuple(sl_src)]
    return out


def density_grid_update(logits, g0, log_decay, log_thr, res, dilate):
    """cf_density_grid_update's decisions: g = max(logits + log_decay, g0) in fp32,
    occupied = g > log_threshold, box-dilated by `dilate` cells -> (g, flat bool bits)."""
    g = np.maximum(np.asarray(logits, dtype=np.float32) + np.float32(log_decay), np.asarray(g0, dtype=np.float32))
    occ = (g > np.float32(log_thr)).reshape(res, res, res)
    if dilate > 0:
        occ = dilate_box(occ, dilate)
    return g, occ.ravel()
