"""Key-frame selection (Eq. 5-7).

No reference code exists for this module: the oracle (oracle/keyframes.py) is pinned
by SPEC's worked examples (CPU tests below), and the kernels are compared with the
oracle bit for bit: exact integer blur sums, identical visibility bits, identical
float64 dissimilarities and the same pool decisions over long candidate streams.
"""
import numpy as np
import pytest

from oracle import keyframes as ok

# ---------------------------------------------------------------- oracle vs SPEC


def _checker(n=64, cell=4):
    y, x = np.mgrid[0:n, 0:n]
    v = (((y // cell) + (x // cell)) % 2 * 255).astype(np.uint8)
    return np.repeat(v[..., None], 3, axis=2)


def _box_blur(img, k=5):
    f = img.astype(np.float64)
    pad = np.pad(f, ((k, k), (k, k), (0, 0)), mode="edge")
    out = np.zeros_like(f)
    for dy in range(-k, k + 1):
        for dx in range(-k, k + 1):
            out += pad[k + dy: k + dy + f.shape[0], k + dx: k + dx + f.shape[1]]
    return np.round(out / (2 * k + 1) ** 2).astype(np.uint8)


def test_oracle_blur_spec_examples():
    assert ok.blur_score(np.full((32, 32, 3), 77, np.uint8)) == 1.0          # constant -> 1.0
    sharp = _checker()
    assert ok.blur_score(sharp) < ok.blur_score(_box_blur(sharp))          # monotone
    rng = np.random.default_rng(0)
    for _ in range(100):
        h, w = rng.integers(16, 40, size=2)
        s = ok.blur_score(rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8))
        assert 0.0 <= s <= 1.0
    with pytest.raises(ValueError):
        ok.blur_score(np.zeros((8, 32, 3), np.uint8))


class _Cam:
    fx = fy = 100.0
    cx, cy = 31.5, 31.5
    R = np.eye(3)
    t = np.zeros(3)


def test_oracle_visibility_spec_examples():
    depth = np.zeros((64, 64))
    depth[32, 32] = 1.005
    depth[40, 40] = 1.020
    nodes = np.array([[0.005, 0.005, 1.0], [0.085, 0.085, 1.0], [5.0, 0.0, 1.0], [0.0, 0.0, -1.0]])
    R, t = np.eye(3), np.zeros(3)
    bits = ok.visibility_map(nodes, depth, R, t, 100.0, 100.0, 31.5, 31.5, eps=0.01)
    assert bits.tolist() == [True, False, False, False]  # 0.005 < eps; 0.02 > eps; off-image; behind


def test_oracle_dissim_spec_examples():
    th = np.zeros(72)
    vis = ok.pack_bits(np.zeros(100, bool))
    assert ok.dissim_human(th, vis, 3, th, vis, 3) == 0.0
    assert ok.dissim_human(th, vis, 5, th, vis, 0) == pytest.approx(0.5, abs=1e-15)
    th2 = th.copy()
    th2[0] = 1.0  # joint 0 (pelvis) is a torso joint
    assert ok.dissim_human(th2, vis, 0, th, vis, 0) == pytest.approx(0.1, abs=1e-15)
    v2 = ok.pack_bits(np.arange(100) < 7)
    assert ok.dissim_human(th, v2, 0, th, vis, 0) == pytest.approx(0.07, abs=1e-15)
    d = np.zeros(3)
    assert ok.dissim_object(d, 1, d, 1) == 0.0
    assert ok.dissim_object(np.array([0.3, 0.4, 0.0]), 0, d, 0) == pytest.approx(0.25, abs=1e-15)
    assert ok.dissim_object(d, 10, d, 0) == pytest.approx(2.0, abs=1e-15)


def test_oracle_pool_rules():
    assert ok.pool_decision([], []) == (True, -1)                          # empty pool -> insert
    assert ok.pool_decision([2.4, 9.0], [0, 1]) == (False, -1)             # 2.4 < gamma -> reject
    ds = [3.0 + i for i in range(100)]
    ds[37] = 2.6
    ts = list(range(100))
    assert ok.pool_decision(ds, ts) == (True, 37)                          # full pool: evict nearest
    ds[12] = 2.6
    assert ok.pool_decision(ds, ts) == (True, 12)                          # tie -> oldest
    assert ok.refinement_order([5.0, 1.0, 3.0], [0, 1, 2], 10) == [1, 2, 0]


# ---------------------------------------------------------------- GPU vs oracle

@pytest.mark.gpu
def test_blur_kernel_bitexact():
    from paper_2304_03184_b200 import keyframes as kf
    rng = np.random.default_rng(1)
    imgs = [np.full((16, 16, 3), 9, np.uint8), _checker(), _box_blur(_checker()),
            rng.integers(0, 256, size=(37, 53, 3), dtype=np.uint8),
            _box_blur(rng.integers(0, 256, size=(512, 512, 3), dtype=np.uint8), 2),
            rng.integers(0, 256, size=(1080, 1920, 3), dtype=np.uint8)]
    for img in imgs:
        assert kf.blur_score(img) == ok.blur_score(img)


@pytest.mark.gpu
def test_visibility_kernel_bitexact_and_spec():
    from paper_2304_03184_b200 import keyframes as kf
    from paper_2304_03184_b200.scene import look_at
    depth = np.zeros((64, 64))
    depth[32, 32] = 1.005
    depth[40, 40] = 1.020
    nodes = np.array([[0.005, 0.005, 1.0], [0.085, 0.085, 1.0], [5.0, 0.0, 1.0], [0.0, 0.0, -1.0]])
    assert kf.visibility_map(nodes, depth, _Cam()).tolist() == [True, False, False, False]
    rng = np.random.default_rng(2)
    for trial in range(6):
        R, t = look_at(rng.normal(size=3) * 0.3 + np.array([0.0, 1.0, 2.5]), np.array([0.0, 1.0, 0.0]))
        cam = type("C", (), dict(fx=280.0, fy=280.0, cx=127.5, cy=127.5, R=R, t=t))()
        n = [100, 1024, 8192, 7303, 33, 4096][trial]
        nodes = rng.normal(size=(n, 3)) * 0.4 + np.array([0.0, 1.0, 0.0])
        Rwc, twc = kf.world_to_cam(cam)
        # a depth map whose pixels at the projected nodes sit within / outside eps
        depth = rng.uniform(0.5, 4.0, size=(256, 256))
        pc = nodes @ Rwc.T + twc
        u = np.round(280.0 * pc[:, 0] / pc[:, 2] + 127.5).astype(int)
        v = np.round(280.0 * pc[:, 1] / pc[:, 2] + 127.5).astype(int)
        ins = (u >= 0) & (u < 256) & (v >= 0) & (v < 256) & (pc[:, 2] > 0)
        depth[v[ins], u[ins]] = pc[ins, 2] + rng.uniform(-0.02, 0.02, size=ins.sum())
        depth[rng.random(depth.shape) < 0.05] = 0.0
        got = kf.visibility_map(nodes, depth, cam)
        ref = ok.visibility_map(nodes, depth, Rwc, twc, 280.0, 280.0, 127.5, 127.5)
        assert np.array_equal(got, ref), trial
        assert got.sum() > 0


def _random_summary(rng, fid, n_nodes, spread):
    th = rng.normal(size=72) * spread
    vis = rng.random(n_nodes) < 0.5
    return th, vis, rng.normal(size=3) * spread


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["human", "object"])
def test_pool_stream_matches_oracle(kind):
    """A 400-frame candidate stream through the device pool and through the oracle's
    rules: identical dissimilarities (bit-exact f64), insert / evict sequence, and
    refinement sets."""
    from paper_2304_03184_b200 import keyframes as kf
    rng = np.random.default_rng(7 if kind == "human" else 8)
    n_nodes = 300
    cap = 20
    pool = kf.KeyFramePool(kind, n_nodes=n_nodes, capacity=cap)
    ent = []  # oracle pool: (fid, theta, packed vis, d)
    inserted = 0
    for fid in range(400):
        th, vis, d = _random_summary(rng, fid, n_nodes, 0.6 if kind == "human" else 1.2)
        s = kf.FrameSummary(fid, th, vis, d)
        pv = ok.pack_bits(vis)
        if kind == "human":
            ds = [ok.dissim_human(th, pv, fid, e[1], e[2], e[0]) for e in ent]
        else:
            ds = [ok.dissim_object(d, fid, e[3], e[0]) for e in ent]
        got_d, _ = pool.scan(s)
        assert np.array_equal(got_d.cpu().numpy(), np.array(ds, dtype=np.float64)), fid
        ins, ev = ok.pool_decision(ds, [e[0] for e in ent], capacity=cap)
        g_ins, g_ev = pool.update(s)
        assert g_ins == ins, fid
        if ins:
            inserted += 1
            if ev >= 0:
                assert g_ev == ent[ev][0]
                ent[ev] = (fid, th, pv, d)
            else:
                assert g_ev is None
                ent.append((fid, th, pv, d))
        assert len(pool) == len(ent) <= cap
        assert sorted(f for f in pool.frame_ids) == sorted(e[0] for e in ent)
    assert inserted > cap  # the stream exercised eviction
    th, vis, d = _random_summary(rng, 400, n_nodes, 0.6)
    view = kf.FrameSummary(400, th, vis, d)
    pv = ok.pack_bits(vis)
    if kind == "human":
        ds = [ok.dissim_human(th, pv, 400, e[1], e[2], e[0]) for e in ent]
    else:
        ds = [ok.dissim_object(d, 400, e[3], e[0]) for e in ent]
    order = ok.refinement_order(ds, [e[0] for e in ent], 10)
    expect = [ent[i][0] for i in order]
    recent = list(range(390, 400))
    for f in recent[::-1]:
        if f not in expect:
            expect.append(f)
    assert pool.refinement_set(view, recent, m=10) == expect


@pytest.mark.gpu
def test_pool_spec_examples():
    from paper_2304_03184_b200 import keyframes as kf
    pool = kf.KeyFramePool("object", capacity=100)
    z = np.zeros(3)
    assert pool.update(kf.FrameSummary(0, d=z)) == (True, None)           # empty pool -> imported
    d0, (ins, _, _, mn) = pool.scan(kf.FrameSummary(10, d=z))
    assert mn == pytest.approx(2.0, abs=1e-15) and not ins                # 2.0 < gamma
    d0, (ins, _, _, mn) = pool.scan(kf.FrameSummary(0, d=np.array([0.3, 0.4, 0.0])))
    assert mn == pytest.approx(0.25, abs=1e-15)
    hp = kf.KeyFramePool("human", n_nodes=64, capacity=100)
    th = np.zeros(72)
    hp.update(kf.FrameSummary(3, th, np.zeros(64, bool)))
    th2 = th.copy()
    th2[0] = 1.0
    _, (_, _, _, mn) = hp.scan(kf.FrameSummary(3, th2, np.zeros(64, bool)))
    assert mn == pytest.approx(0.1, abs=1e-15)
    # a full pool keeps its size
    full = kf.KeyFramePool("object", capacity=100)
    for i in range(100):
        assert full.update(kf.FrameSummary(i, d=np.array([10.0 * i, 0, 0])))[0]
    ins, ev = full.update(kf.FrameSummary(200, d=np.array([10.0 * 37 + 2.0, 0, 0])))
    assert ins and ev == 37 and len(full) == 100 and 200 in full.frame_ids
    assert kf.fixed_interval_selector(1000) == list(range(0, 1000, 10))
    assert len(kf.fixed_interval_selector(1234)) == -(-1234 // 12)
