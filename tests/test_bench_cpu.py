"""bench.py's harness on the CPU: `--gpus N` spawns N ranks itself (torchrun re-exec),
the reference arm runs standalone on the host cores (no product library mapped), and
the max / sum over ranks used for the timing are correct under gloo at world size 2."""
import json
import os
import subprocess
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_spawns_two_ranks_and_runs_standalone():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--width", "96", "--height", "96", "--samples", "32"]
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 prints, rank 1 exits without work
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["same_config"] is True
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["native_libs_loaded"] == []  # no product .so in the reference arm


def _worker(rank, world, port, q):
    import bench
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx = bench.max_over_ranks(dist, float(rank + 1))
    sm = bench.sum_over_ranks(dist, float(10 * (rank + 1)))
    bench.barrier(dist)
    q.put((rank, mx, sm))
    dist.destroy_process_group()


def test_max_and_sum_over_ranks_gloo():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
    assert got == [(0, 2.0, 30.0), (1, 2.0, 30.0)]


def test_gpu_arm_refuses_without_devices():
    import torch
    if torch.cuda.is_available():
        return
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0 and "CUDA device" in (out.stderr + out.stdout)


def test_roofline_of_fused_stages_is_the_slower_resource():
    """A fused stage (MLP FLOPs + the hash gathers it does itself) reports the resource
    with the longer ideal time, the other one listed; unfused stages keep one bound."""
    sys.path.insert(0, ROOT)
    import bench
    peaks = {"bf16_tflops": (1600.0, "t"), "hash_c_gbs": (4000.0, "t"), "hash_d_gbs": (10000.0, "t"),
             "hbm_gbs": (6500.0, "t")}
    hs = 300_000
    fused = bench.stage_costs(hs, 40_000, 512 * 512, "fp32", fused=True)
    split = bench.stage_costs(hs, 40_000, 512 * 512, "fp32", fused=False)
    e = bench.roofline_entry("human_color_mlp", fused["human_color_mlp"], 0.08, peaks)
    gather = hs * 16 * 8 * 8 / 0.08e-3 / 1e9 / 4000.0
    tensor = hs * 20480.0 / 0.08e-3 / 1e12 / 1600.0
    assert e["bound"] == "gather" and abs(e["frac"] - gather) < 1e-9
    assert sorted(c["bound"] for c in e["components"]) == ["gather", "tensor"]
    assert abs(min(c["frac"] for c in e["components"]) - tensor) < 1e-9
    d = bench.roofline_entry("human_deform_mlp", fused["human_deform_mlp"], 0.12, peaks)
    assert d["frac"] == max(c["frac"] for c in d["components"])
    s = bench.roofline_entry("human_deform_mlp", split["human_deform_mlp"], 0.08, peaks)
    assert s["bound"] == "tensor" and "components" not in s
