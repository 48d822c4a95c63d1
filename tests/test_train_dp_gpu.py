"""Data-parallel training step (ADVICE r1 train.py:281): two ranks
(processes, gloo) each run the real Trainer.step on their shard of every key frame's
rays; the ray counts and gradient buckets are summed over the ranks. The summed
gradients must equal one process's step on the union batch (float-atomic
summation order aside), and so must the parameters after the Adam update.

Both ranks share cuda:0 of the test box: their kernels never wait on each other
(the collectives are gloo's host-side all-reduces), so this checks the sharded
step's arithmetic, not NVLink performance."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build():
    from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
    from paper_2304_03184_b200.scene import Scene, SceneConfig
    from paper_2304_03184_b200.train import Trainer, TrainConfig
    from test_train_gpu import make_batch
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    sc = Scene(SceneConfig(width=96, height=96), seed=0)
    cfg = RenderConfig(n_samples=64)
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, zero_deform_out=False,
                    table_scale=0.1)
    of = ObjectField(sc.box_half, cfg, table_scale=0.1)
    r = Renderer(hf, of, 96, 96, cfg)
    R, t = sc.object_pose(0)
    r.set_frame(sc.node_dqs(0), sc.theta(0), sc.bone_transforms(0), R, t)
    rng = np.random.default_rng(0)
    batches = [make_batch(sc, hf, fid, 2048, rng, dev) for fid in (0, 3, 7)]
    tr = Trainer(r, max_rays=2048, cfg=TrainConfig())
    return tr, batches


def _snapshot(tr):
    out = {}
    for st in tr.fields:
        out[st["name"] + "/grad"] = st["flat"].cpu().numpy().copy()
    return out


def _params(tr):
    out = {}
    for st in tr.fields:
        out[st["name"] + "/ctable"] = st["field"].cgrid.table.cpu().numpy().copy()
        for k, w in st["params"].W.items():
            out[st["name"] + "/" + k] = w.cpu().numpy().copy()
        if "deform" in st:
            for k, w in st["deform"].W.items():
                out[st["name"] + "/" + k] = w.cpu().numpy().copy()
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2304_03184_b200.train import shard_batch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr, batches = _build()
        shards = [shard_batch(b, rank, world) for b in batches]
        tr.step(shards, update=False)
        torch.cuda.synchronize()
        grads = _snapshot(tr)
        counts = tr.counts.cpu().numpy().copy()
        tr._update()
        torch.cuda.synchronize()
        q.put((rank, grads, counts, _params(tr)))
    finally:
        dist.destroy_process_group()


def test_sharded_step_equals_union_step():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the single-process step on the union batch
    tr, batches = _build()
    tr.step(batches, update=False)
    torch.cuda.synchronize()
    ref = _snapshot(tr)
    ref_counts = tr.counts.cpu().numpy()
    tr._update()
    torch.cuda.synchronize()
    ref_params = _params(tr)
    for rank, grads, counts, params in res:
        assert np.array_equal(counts, ref_counts), rank  # ray counts summed over the ranks
        for k, g in ref.items():
            err = np.abs(grads[k] - g).max()
            assert err <= 1e-5 * np.abs(g).max(), (rank, k, err, np.abs(g).max())
    # both ranks applied the same update, equal to the union step's (Adam's first step
    # is ~lr * sign(g): entries whose gradient is ~0 may differ by summation order)
    for k, p in ref_params.items():
        a, b = res[0][3][k], res[1][3][k]
        assert np.array_equal(a, b), k
        frac = np.mean(np.abs(a - p) > 1e-6)
        assert frac < 1e-3, (k, frac)
