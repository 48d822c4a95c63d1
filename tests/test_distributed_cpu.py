"""Multi-rank host logic on CPU (gloo, world size 2): training-ray sharding
covers the global batch exactly once, the gradient-bucket all-reduce sums
every bucket across ranks, and the row-sharded multi-GPU render reassembles the
frame from the ranks' round-robin rows."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_03184_b200.render import assemble_row_shards, gather_row_shards, row_shard_rows
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
        # row-sharded frame (H = 7 rows of W = 3 pixels): pixel value = its image row
        W, H = 3, 7
        rows = row_shard_rows(H, rank, world)
        part = torch.tensor([[float(v)] * 3 for v in rows for _ in range(W)])
        frame = gather_row_shards(part, W, H)
        ok = torch.equal(frame, torch.arange(H, dtype=torch.float32).repeat_interleave(W)[:, None].repeat(1, 3))
        q.put((rank, float(g_table[0, 0]), g_w.tolist(), sl.start, sl.stop, ok))
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
    for rank, g0, gw, a, b, ok in res:
        assert g0 == pytest.approx(3.0)  # sum of 1 and 2 (the loss is normalised by global counts)
        assert gw == (torch.arange(12, dtype=torch.float32).view(3, 4) * 3.0).tolist()
        assert ok, f"rank {rank}: row-sharded frame not reassembled"
    spans = [(a, b) for _, _, _, a, b, _ in res]
    assert spans[0][0] == 0 and spans[-1][1] == 10001 and spans[0][1] == spans[1][0]


def test_shard_rays_balanced():
    for n in (0, 1, 7, 1 << 18):
        for w in (1, 2, 4, 8):
            sl = [shard_rays(n, r, w) for r in range(w)]
            assert sl[0].start == 0 and sl[-1].stop == n
            assert all(a.stop == b.start for a, b in zip(sl, sl[1:]))
            sizes = [s.stop - s.start for s in sl]
            assert max(sizes) - min(sizes) <= 1


def test_row_shards_cover_and_assemble():
    for H in (1, 7, 1080):
        for w in (1, 2, 3, 8):
            rows = [list(row_shard_rows(H, r, w)) for r in range(w)]
            assert sorted(sum(rows, [])) == list(range(H))
    W, H, w = 4, 9, 4
    full = torch.arange(H * W * 3, dtype=torch.float32).view(H * W, 3)
    parts = [full.view(H, W, 3)[r::w].reshape(-1, 3) for r in range(w)]
    assert torch.equal(assemble_row_shards(parts, W, H), full)


def test_shard_batch_keeps_global_ray_ids():
    """shard_batch: the ranks' shards cover a key frame's rays once, in order, and each
    carries the global id of its first ray (the sampler hashes global ids)."""
    import numpy as np

    from paper_2304_03184_b200.train import FrameBatch, shard_batch
    R = 1001
    t = lambda *shape: torch.arange(int(np.prod(shape)), dtype=torch.float32).reshape(*shape)  # noqa: E731
    b = FrameBatch(dqs=None, bone_A=None, dbias=None, obj_R=None, obj_t=None, dirs=t(R, 3), gt_rgb=t(R, 3),
                   gt_depth=t(R), mask_h=t(R), mask_o=t(R), ray0=5)
    for world in (1, 2, 3, 8):
        parts = [shard_batch(b, r, world) for r in range(world)]
        assert torch.equal(torch.cat([p.dirs for p in parts]), b.dirs)
        assert torch.equal(torch.cat([p.gt_depth for p in parts]), b.gt_depth)
        starts = [p.ray0 for p in parts]
        assert starts[0] == 5 and all(p.ray0 + p.dirs.shape[0] == q.ray0 for p, q in zip(parts, parts[1:]))
