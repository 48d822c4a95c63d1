"""Pin the stage 2-4 oracle on SPEC.md's worked examples (the reference has no
code or tests for these stages — parity unpinned beyond these). CPU only."""
import numpy as np

from oracle import nrf as on


def test_hash_levels_rule():
    levels, total = on.hash_levels(16, 19, 16, 2048)
    res = [N for N, _, _ in levels]
    assert res[0] == 16 and res[-1] == 2048
    assert all(b > a for a, b in zip(res, res[1:]))  # strictly increasing
    assert [d for _, d, _ in levels][:5] == [True] * 5 and not any(d for _, d, _ in levels[5:])
    assert total == sum(((N + 1) ** 3 + 7) // 8 * 8 if d else 1 << 19 for N, d, _ in levels)


def test_corner_equals_table_entry_and_center_is_mean():
    rng = np.random.default_rng(0)
    levels, total = on.hash_levels(16, 19, 16, 2048)
    table = rng.uniform(-1, 1, size=(total, 2)).astype(np.float32)
    for l in (0, 3, 7, 15):
        N, dense, off = levels[l]
        g = rng.integers(0, N, size=(50, 3))
        x = (g.astype(np.float32) / np.float32(N)).astype(np.float32)
        exact = (g.astype(np.float64) / N)
        ok = np.all((x.astype(np.float64) * N) == g, axis=1)  # representable grid corners
        feat = on.hash_encode(table, x)[:, 2 * l:2 * l + 2]
        idx, w = on.hash_corners(x, levels[l], 19)
        assert np.array_equal(feat[ok], table[off + idx[ok, 0]])
        xc = ((g + 0.5) / N).astype(np.float32)
        featc = on.hash_encode(table, xc)[:, 2 * l:2 * l + 2]
        idc, wc = on.hash_corners(xc, levels[l], 19)
        okc = np.all(np.isclose(wc, 0.125, atol=1e-3), axis=1)
        mean = table[off + idc].mean(axis=1)
        assert np.allclose(featc[okc], mean[okc], atol=2e-3)


def test_hash_deterministic_and_clamped():
    rng = np.random.default_rng(1)
    _, total = on.hash_levels(16, 19, 16, 2048)
    table = rng.uniform(-1, 1, size=(total, 2)).astype(np.float32)
    x = rng.uniform(-0.2, 1.2, size=(100, 3)).astype(np.float32)
    a = on.hash_encode(table, x)
    assert np.array_equal(a, on.hash_encode(table, x))
    assert np.array_equal(a, on.hash_encode(table, np.clip(x, 0, 1)))


def test_mlp_kernel_precision_matches_fp64_loosely():
    rng = np.random.default_rng(2)
    Ws = [rng.normal(size=(64, 32)) * 0.2, rng.normal(size=(16, 64)) * 0.2]
    x = rng.normal(size=(100, 32))
    ref = np.maximum(x @ Ws[0].T, 0) @ Ws[1].T
    assert np.allclose(on.mlp_forward(Ws, x), ref, rtol=2e-2, atol=2e-2)


# ---- volume_render examples and invariants (acceptance 5)

def _uniform_ray(sig, t_near=0.3, t_far=5.0, rgb=(0.2, 0.5, 0.9)):
    from oracle import render as orr
    S = len(sig)
    dt = (t_far - t_near) / S
    f = np.zeros((S, 4), dtype=np.float32)
    f[:, 0] = sig
    f[:, 1:] = rgb
    return orr.composite(1, np.zeros(S, np.int64), np.arange(S), f, t_near, dt, t_term=0.0), dt


def test_volume_render_zero_density():
    (rgb, depth, op), _ = _uniform_ray(np.zeros(128))
    assert (rgb == 0).all() and op[0] == 0.0  # black background, opacity 0


def test_volume_render_constant_density_analytic():
    for sigma in (0.05, 0.5, 1.0, 1.9):
        (rgb, depth, op), dt = _uniform_ray(np.full(128, sigma, np.float32))
        ell = 128 * dt
        assert abs(op[0] - (1.0 - np.exp(-float(np.float32(sigma)) * ell))) <= 1e-5


def test_volume_render_thin_slab_depth():
    S, t_near, t_far = 128, 0.3, 5.0
    dt = (t_far - t_near) / S
    for t_star in (0.9, 2.35, 4.1):
        i0 = int((t_star - t_near) / dt)
        sig = np.zeros(S, np.float32)
        sig[i0] = 5e3  # near-opaque slab one sample thick
        (rgb, depth, op), _ = _uniform_ray(sig, t_near, t_far)
        assert op[0] > 0.999 and abs(depth[0] - t_star) <= dt


def test_volume_render_telescoping():
    rng = np.random.default_rng(5)
    for _ in range(20):
        sig = (rng.exponential(0.3, 128) * (rng.random(128) < 0.5)).astype(np.float32)
        (rgb, depth, op), dt = _uniform_ray(sig)
        T_end = np.prod(1.0 - (1.0 - np.exp(-sig.astype(np.float64) * float(np.float32(dt)))))
        assert abs(op[0] + T_end - 1.0) <= 1e-6
