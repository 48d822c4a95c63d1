"""Multi-rank host logic of the training step on CPU (gloo, world size 2): ray
sharding covers the global batch exactly once, and the gradient-bucket
all-reduce averages every bucket across ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_03184_b200.train import allreduce_grads, shard_rays


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank-dependent local gradients: table grads + small MLP grads
        g_table = torch.full((1000, 2), float(rank + 1))
        g_w = torch.arange(12, dtype=torch.float32).view(3, 4) * (rank + 1)
        allreduce_grads([g_table, g_w])
        sl = shard_rays(10001, rank, world)
        q.put((rank, float(g_table[0, 0]), g_w.tolist(), sl.start, sl.stop))
    finally:
        dist.destroy_process_group()


def test_allreduce_and_sharding_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g0, gw, a, b in res:
        assert g0 == pytest.approx(1.5)  # mean of 1 and 2
        assert gw == (torch.arange(12, dtype=torch.float32).view(3, 4) * 1.5).tolist()
    spans = [(a, b) for _, _, _, a, b in res]
    assert spans[0][0] == 0 and spans[-1][1] == 10001 and spans[0][1] == spans[1][0]


def test_shard_rays_balanced():
    for n in (0, 1, 7, 1 << 18):
        for w in (1, 2, 4, 8):
            sl = [shard_rays(n, r, w) for r in range(w)]
            assert sl[0].start == 0 and sl[-1].stop == n
            assert all(a.stop == b.start for a, b in zip(sl, sl[1:]))
            sizes = [s.stop - s.start for s in sl]
            assert max(sizes) - min(sizes) <= 1
