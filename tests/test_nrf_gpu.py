"""Stages 2-3 parity on the B200: hash encoding (bit-exact indices, bit-equal
features) and the tcgen05 MLP chain (vs the kernel-precision oracle)."""
import numpy as np
import pytest
import torch

from oracle import nrf as on
from paper_2304_03184_b200 import nrf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [nrf.HashGridConfig(), nrf.HashGridConfig(8, 4, 17, 16, 256)])
def test_hash_encode_bitexact(cfg):
    rng = np.random.default_rng(0)
    levels, total = on.hash_levels(cfg.n_levels, cfg.log2_table, cfg.base_resolution, cfg.max_resolution)
    table = rng.uniform(-1, 1, size=(total, cfg.n_features)).astype(np.float32)
    g = nrf.HashGrid(cfg, table=table)
    assert g.n_entries == total
    assert [(N, d, o) for N, d, o in g.levels()] == levels
    x = np.concatenate([rng.uniform(0, 1, size=(50000, 3)), rng.uniform(-0.1, 1.1, size=(2000, 3)),
                        np.array([[0, 0, 0], [1, 1, 1], [1, 0, 1]])]).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    idx, w = g.indices(xt)
    idx, w = idx.cpu().numpy().view(np.uint32), w.cpu().numpy()
    for l, lv in enumerate(levels):
        oi, ow = on.hash_corners(x, lv, cfg.log2_table)
        assert np.array_equal(idx[:, l], oi), f"level {l} indices"
        assert np.array_equal(w[:, l], ow), f"level {l} weights"
    feat = nrf.hash_encode(g, xt).cpu().numpy()
    ref = on.hash_encode(table, x, cfg.n_levels, cfg.n_features, cfg.log2_table, cfg.base_resolution,
                         cfg.max_resolution)
    assert np.array_equal(feat, ref)


def test_hash_encode_bwd():
    cfg = nrf.HashGridConfig()
    rng = np.random.default_rng(1)
    g = nrf.HashGrid(cfg)
    x = rng.uniform(0, 1, size=(20000, 3)).astype(np.float32)
    df = rng.normal(size=(20000, 32)).astype(np.float32)
    grad = torch.zeros_like(g.table)
    g.encode_backward(torch.from_numpy(x).cuda(), torch.from_numpy(df).cuda(), grad)
    ref = on.hash_encode_bwd(x, df)
    got = grad.cpu().numpy()
    assert np.allclose(got, ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("widths,bias", [((32, 64, 16), False), ((31, 64, 64, 3), False),
                                          ((32, 128, 128, 128, 128, 3), True), ((104, 128, 16), True)])
def test_mlp_chain_tcgen05(widths, bias):
    rng = np.random.default_rng(len(widths))
    biases = [rng.normal(size=w) * 0.1 if bias else None for w in widths[1:]]
    net = nrf.MLP(widths, seed=3, biases=biases)
    n = 128 * 37 + 5  # partial last tile
    x = rng.normal(size=(n, widths[0])).astype(np.float32)
    y = net(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = on.mlp_forward(net.weights, x, biases)
    scale = np.abs(ref).max()
    err = np.abs(y - ref)
    # fp16 operands, fp32 accumulation: intermediate fp16 rounding can flip by one ulp
    assert err.max() <= 2e-3 * scale, (err.max(), scale)
    assert np.median(err) <= 1e-5 * scale + 1e-6


def test_mlp_empty_and_large():
    net = nrf.MLP((32, 64, 16), seed=0)
    assert net(torch.zeros((0, 32), device="cuda")).shape == (0, 16)
    x = torch.randn((1 << 20, 32), device="cuda")
    y = net(x)
    ref = on.mlp_forward(net.weights, x[:4096].cpu().numpy())
    assert np.allclose(y[:4096].cpu().numpy(), ref, rtol=1e-2, atol=1e-2)
