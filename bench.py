#!/usr/bin/env python
"""Headline benchmark: deformed samples/s and ms per 512x512 frame (BASELINE.json
`metric`, workload configs[1]: 512^2 novel-view render of the synthetic human +
rigid object, 128 samples/ray, 1 B200; N GPUs = N independent ranks, each
rendering its own frame stream — weak scaling, no data-path collective).

A step = one frame: load the frame's motion prior (ED node dqs, bone transforms,
DeformNet pose bias, object pose), per-frame setup (deformed nodes, buckets,
backward-LBS vertex transforms, live occupancy splat) and the full render
(rays, occupancy-skipped march, hybrid canonicalisation, fused hash+tcgen05
field, compositing, layer composite).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "deformed samples/s (warp+hash+MLP+composite); ms per 512² frame; 1/2/4/8 B200"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--width", type=int, default=512)
    ap.add_argument("--height", type=int, default=512)
    ap.add_argument("--samples", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp16-mode", action="store_true", help="skip the secondary fp16-mode measurement")
    ap.add_argument("--workload", default="render", choices=["render", "train", "knn", "frontend"],
                    help="render = configs[1] (the headline); train = configs[2] key-frame training step; "
                         "knn = configs[3] dense-graph k-NN scaling")
    ap.add_argument("--train-rays", type=int, default=1 << 18)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp16"],
                    help="field arithmetic: fp32 = SPEC 32-bit semantics (split-fp16 tensor-core operands, fp32 "
                         "tables / features); fp16 = fp16 operands and features")
    ap.add_argument("--shard", default="frames", choices=["frames", "rows"],
                    help="render at N GPUs: frames = each rank renders whole frames (weak scaling, the "
                         "headline); rows = the ranks split every frame's rows round-robin and all-gather the "
                         "image (strong scaling, configs[4], e.g. --width 1920 --height 1080)")
    return ap.parse_args()


# ----------------------------------------------------------------- distributed

def relaunch(args) -> int:
    """`--gpus N` without a launcher: re-exec this command under torch.distributed.run
    with N ranks (one per GPU, rendezvous on 127.0.0.1). The GPU arm refuses to run
    with fewer than N visible devices."""
    import socket
    import subprocess
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(args):
    """Rank / world from the launcher's environment; one NCCL rank per GPU (gloo
    without CUDA). The world must be the --gpus the command asked for."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        cuda = torch.cuda.is_available()
        if cuda:
            if torch.cuda.device_count() < world:
                raise SystemExit(f"{world} ranks need {world} GPUs, {torch.cuda.device_count()} visible")
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if cuda else "gloo")
        pg = dist
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def _reduce(pg, v: float, op) -> float:
    if pg is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    pg.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(pg, v: float) -> float:
    return v if pg is None else _reduce(pg, v, pg.ReduceOp.MAX)


def sum_over_ranks(pg, v: float) -> float:
    return v if pg is None else _reduce(pg, v, pg.ReduceOp.SUM)


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons = [], set()
        self.period, self.index = period, index
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, b in names.items():
                    if mask & b:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------- workload

def build_workload(args, rank):
    from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
    from paper_2304_03184_b200.scene import Scene, SceneConfig
    sc = Scene(SceneConfig(width=args.width, height=args.height), seed=0)
    cfg = RenderConfig(n_samples=args.samples, precision=getattr(args, "precision", "fp32"))
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, seed=0, zero_deform_out=False)
    of = ObjectField(sc.box_half, cfg, seed=1)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    shard = (rank, world) if getattr(args, "shard", "frames") == "rows" else None
    r = Renderer(hf, of, args.width, args.height, cfg, row_shard=shard)
    frames = []
    for fid in range(sc.cfg.frames):
        R, t = sc.object_pose(fid)
        # the frame's motion prior as the tracker emits it (a CFMP record): node dqs,
        # pose theta, object pose; FK and the DeformNet pose bias run on the device
        frames.append(dict(dqs=sc.node_dqs(fid), theta=sc.theta(fid), R=R, t=t))
    return sc, cfg, hf, of, r, frames


def load_peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver: HBM copy, cuBLAS bf16) and
    profiles/r02_peaks.json (tools/peaks.cu: L2 random gathers, FP64 / FP32 FMA)."""
    peaks, src = {}, {}
    for name, path in (("driver", os.path.join(ROOT, "MEASURED_PEAKS.json")),
                       ("micro", os.path.join(ROOT, "profiles", "r02_peaks.json"))):
        try:
            d = json.load(open(path))
            peaks.update(d)
            src[name] = os.path.relpath(path, ROOT)
        except Exception:
            pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    return {"hbm_gbs": (hbm, "measured HBM copy, " + src.get("driver", "fallback B200_PROFILING.md")),
            "bf16_tflops": (float(peaks.get("bf16_tflops", 1590.0)),
                            "measured cuBLAS bf16 burst (fp16 kind::f16 dense rate equal), "
                            + src.get("driver", "fallback")),
            "l2_gather8_gbs": (float(peaks.get("l2_gather_8B_64MiB_gbs", 2300.0)),
                               "measured L2-resident random 8 B gathers, " + src.get("micro", "-")),
            "l2_gather16_gbs": (float(peaks.get("l2_gather_16B_64MiB_gbs", 4600.0)),
                                "measured L2-resident random 16 B gathers, " + src.get("micro", "-")),
            "fp64_tflops": (float(peaks.get("fp64_fma_tflops", 34.0)), "measured FP64 FMA, " + src.get("micro", "-")),
            "hash_c_gbs": (float(peaks.get("hash_gather_canonical_16x2p19xF2_f32_gbs", 4180.0)),
                           "measured gather-only ceiling of the canonical grid's own access pattern, "
                           + src.get("micro", "-")),
            "hash_d_gbs": (float(peaks.get("hash_gather_deform_8x2p17xF4_f32_gbs", 9750.0)),
                           "measured gather-only ceiling of the deformation grid's access pattern (fp32 entries), "
                           + src.get("micro", "-"))}


def stage_costs(hs, os_, n_rays, precision, fused=False):
    """Algorithmic work per launch of each render stage:
    (bound, work, unit, how). Hash stages: every level's 8 corner gathers (SURVEY 8(d)
    K8) against the measured gather-only ceiling of the same grid's access pattern
    (tools/peaks.cu hash_gather: L1 reuse between neighbouring samples included);
    MLPs: the math FLOPs (the fp32 mode issues 3x as split-fp16 MMAs)."""
    f32 = precision == "fp32"
    ent_d = 16 if f32 else 8   # deformation grid entry (F = 4): fp32 / fp16 copy
    return {
        "human_canon": ("hbm", hs * 57.0, "B", "57 B/sample (SURVEY 8d K5/K6: pos 12 + p_c 12 + idx 16 + w 16 + valid 1)"),
        "human_hash_d": ("hash_d", hs * 8 * 8 * ent_d, "B", f"8 levels x 8 corners x {ent_d} B"),
        "human_deform_mlp": [("tensor", hs * 110592.0, "FLOP",
                              "2(32x128 + 3x128x128 + 128x16) FLOP/sample" + (" (x3 issued: split fp16)" if f32 else ""))]
                            + ([("hash_d", hs * 8 * 8 * ent_d, "B",
                                 f"deformation-grid hash fused in: 8 levels x 8 corners x {ent_d} B")] if fused else []),
        "human_hash_c": ("hash_c", hs * 16 * 8 * 8, "B", "16 levels x 8 corners x 8 B"),
        "human_color_mlp": [("tensor", hs * 20480.0, "FLOP",
                             "2(32x64 + 64x16 + 32x64 + 64x64 + 64x16) FLOP/sample" + (" (x3 issued)" if f32 else ""))]
                           + ([("hash_c", hs * 16 * 8 * 8, "B", "canonical hash fused in: 16 levels x 8 corners x 8 B")]
                              if fused else []),
        "object_field": ("hash_c", os_ * 16 * 8 * 8, "B", "hash (16 levels x 8 x 8 B) + E_g/E_c; gather-bound"),
        "march": ("hbm", n_rays * 32.0 + 4.0 * (hs + os_), "B", "B/ray: dir 24 + offset/count 8, + 4 B/record"),
        "human_composite": ("hbm", (hs) * 16.0 + n_rays * 40.0, "B", "field 16 B/sample + 40 B/ray out"),
    }


def roofline_entry(name, cost, ms, peaks):
    """One stage against its bound. A fused stage (a list of costs: e.g. the MLP's
    FLOPs and the hash gathers it does itself) is bound by the resource whose ideal
    time is the longest; that resource's entry is reported, the others listed."""
    if isinstance(cost, list):
        parts = [roofline_entry(name, c, ms, peaks) for c in cost]
        if len(parts) == 1:
            return parts[0]
        best = dict(max(parts, key=lambda e: e["frac"]))
        best["components"] = [{x: e[x] for x in ("bound", "achieved", "peak", "unit", "frac", "per_unit")}
                              for e in parts]
        best["per_unit"] = " + ".join(e["per_unit"] for e in parts) + " (one kernel; bound = the slower resource)"
        return best
    bound, work, unit, how = cost
    if bound == "tensor":
        ach = work / (ms / 1e3) / 1e12
        peak, src = peaks["bf16_tflops"]
        return {"kernel": name, "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "per_unit": how, "peak_source": src, "ms": ms}
    key = {"hbm": "hbm_gbs", "l2_8": "l2_gather8_gbs", "l2_16": "l2_gather16_gbs", "hash_c": "hash_c_gbs",
           "hash_d": "hash_d_gbs"}[bound]
    ach = work / (ms / 1e3) / 1e9
    peak, src = peaks[key]
    return {"kernel": name, "bound": "hbm" if bound == "hbm" else ("gather" if bound.startswith("hash") else "l2"),
            "achieved": ach, "peak": peak,
            "unit": "GB/s", "frac": ach / peak, "per_unit": how, "peak_source": src, "ms": ms}


def count_launches(fn):
    """Kernels one call of fn launches (CUPTI via torch.profiler, graph replays
    included): (ours, others, names). Ours = kernels of this package's library."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    ours, other, names = 0, 0, set()
    for e in prof.events():
        if str(getattr(e, "device_type", "")).endswith("CUDA") is False:
            continue
        n = e.name
        if n.startswith("Memcpy") or n.startswith("Memset") or "cudaGraph" in n or n.startswith("cuda"):
            continue
        foreign = ("at::" in n or "cublas" in n.lower() or "nvjet" in n or "cutlass" in n or "nccl" in n.lower())
        if foreign:
            other += 1
        else:
            ours += 1
        n = n.replace("(anonymous namespace)::", "").replace("void ", "")
        names.add(n.split("(")[0].split("<")[0][:60])
    return ours, other, sorted(names)


def run_ours(args, rank, world, pg):
    import torch
    sc, cfg, hf, of, r, frames = build_workload(args, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    cam = sc.camera
    # device-resident inputs (value) and pinned host inputs (e2e): the frame's motion prior
    dframes = [(torch.from_numpy(f["dqs"]).to(dev), torch.from_numpy(f["theta"]).to(dev), f["R"], f["t"])
               for f in frames]
    hframes = [(torch.from_numpy(f["dqs"]).pin_memory(), torch.from_numpy(f["theta"]).pin_memory(), f["R"], f["t"])
               for f in frames]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    rows_mode = args.shard == "rows" and world > 1
    if rows_mode:
        from paper_2304_03184_b200.render import gather_row_shards

    def step(fi, src):
        dqs, theta, R, t = src[fi]
        r.load_pose(dqs, theta)
        r.set_object_pose(R, t)
        img = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
        if rows_mode:  # every rank renders its rows of the frame; the frame is all-gathered (NCCL)
            img = gather_row_shards(img, args.width, args.height)
        return img

    nF = len(frames)
    counts = []  # processed samples per frame (deterministic), untimed
    for fi in range(nF):
        step(fi, dframes)
        torch.cuda.synchronize()
        r.check_overflow()
        counts.append(r.sample_counts())
    fofs = 0 if rows_mode else rank  # frames mode: ranks start at different frames
    for w in range(max(args.warmup, 3)):
        step((w + fofs) % nF, dframes)
    torch.cuda.synchronize()

    def timed_loop(n_steps, precision_label):
        barrier(pg)
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(n_steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(n_steps)]
        done = 0
        with ClockSampler(torch.cuda.current_device()) as clk:
            t_issue = time.perf_counter()
            for k in range(n_steps):
                fi = (k + fofs) % nF
                flush.zero_()
                starts[k].record()
                step(fi, dframes)
                ends[k].record()
                done += counts[fi][0] + counts[fi][1]
            t_issue = time.perf_counter() - t_issue
            torch.cuda.synchronize()
        barrier(pg)
        ms_local = float(np.sum([s.elapsed_time(e) for s, e in zip(starts, ends)]))
        return ms_local, done, t_issue, clk.summary()

    # ---- timed region: K steps, device-resident inputs, L2 flushed between steps
    ms_local, processed, t_issue, clocks = timed_loop(args.steps, args.precision)
    ms_total = max_over_ranks(pg, ms_local)
    processed_all = sum_over_ranks(pg, float(processed))
    value = processed_all / (ms_total / 1e3)
    ms_per_step = ms_total / args.steps

    # ---- kernels per step (CUPTI, the graph replay of one step)
    ours, other, names = count_launches(lambda: step(fofs % nF, dframes))

    # ---- per-kernel times: the same frame serialised on one stream (graph variant with
    # an event after every stage); stage = gap to the previous event
    r.cfg.serial = True
    stage_runs = []
    for k in range(min(args.steps, 30)):
        flush.zero_()
        r.marks = []
        step((k + fofs) % nF, dframes)
        torch.cuda.synchronize()
        ev = [(name, e) for _, name, e in r.marks]
        stage_runs.append({ev[j][0]: ev[j - 1][1].elapsed_time(ev[j][1]) for j in range(1, len(ev))})
        r.marks = None
    r.cfg.serial = False
    stage_ms = {k: float(np.mean([m[k] for m in stage_runs])) for k in stage_runs[0]}
    serial_ms = float(sum(stage_ms.values()))

    # ---- the "fp16" precision mode on the same frames (the fast mode)
    fp16 = None
    if args.precision == "fp32" and not args.no_fp16_mode:
        r.set_precision("fp16")
        for w in range(3):
            step((w + fofs) % nF, dframes)
        ms16, done16, _, _ = timed_loop(args.steps, "fp16")
        r.set_precision(args.precision)
        ms16 = max_over_ranks(pg, ms16)
        fp16 = {"value": sum_over_ranks(pg, float(done16)) / (ms16 / 1e3), "unit": UNIT,
                "ms_per_step": ms16 / args.steps,
                "dtype": "f64 deform / fp16 hash features / fp16-in fp32-acc MLP",
                "accuracy": "sigma 5.5e-2 / rgb 2.2e-3 vs the fp32 semantics (99.9th pct, tests/test_precision_gpu.py)"}

    # ---- e2e: pinned host prior -> device, render through the public API, image -> pinned host
    e2e = None
    if not args.no_e2e:
        h2d = sum(int(x.numel() * x.element_size()) for x in hframes[0][:2]) + 28 * 8  # + frame block

        def step_host(fi):
            dqs, theta, R, t = hframes[fi]
            r.load_pose(dqs, theta)
            r.set_object_pose(R, t)
            if rows_mode:
                img = gather_row_shards(r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy), args.width,
                                        args.height)
                return None, img.cpu()
            return r.render_to_host(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)

        for w in range(3):
            ev, img_host = step_host(w % nF)
            if ev is not None:
                ev.synchronize()
        d2h = int(img_host.numel() * img_host.element_size())
        torch.cuda.synchronize()
        barrier(pg)
        t0 = time.perf_counter()
        pending = None
        for k in range(args.steps):
            handle = step_host((k + fofs) % nF)
            if pending is not None and pending[0] is not None:
                pending[0].synchronize()  # step k-1's image is in host memory
            pending = handle
        if pending[0] is not None:
            pending[0].synchronize()
        wall = time.perf_counter() - t0
        barrier(pg)
        wall = max_over_ranks(pg, wall)
        e2e = {"value": processed_all / wall, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": wall * 1e3 / args.steps,
               "path": "Renderer.load_pose(pinned dqs, theta) + set_object_pose + render_to_host (fp32 image)"}

    # ---- roofline: dominant kernel of the serialised frame, every stage against its bound
    hs = float(np.mean([counts[(k + fofs) % nF][0] for k in range(args.steps)]))
    os_ = float(np.mean([counts[(k + fofs) % nF][1] for k in range(args.steps)]))
    peaks = load_peaks()
    costs = stage_costs(hs, os_, r.n_rays, args.precision,
                        fused=bool(r.hdesc.precise) and not bool(r.hdesc.split_stages))
    stages = {k: roofline_entry(k, costs[k], stage_ms[k], peaks) for k in costs if k in stage_ms}
    dom = max(stages, key=lambda k: stages[k]["ms"])
    roof = dict(stages[dom])
    try:  # DRAM bytes per launch from the committed ncu --set full capture (profiles/)
        tr_map = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        tr_map = {}

    def traffic_of(k):
        t = tr_map.get(f"{args.precision}:{k}")
        return float(t["dram_bytes_per_launch"]) if isinstance(t, dict) else None
    roof["traffic"] = traffic_of(dom)
    roof["traffic_source"] = "profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum of one launch)"
    roof["all_stages"] = {k: dict({x: v[x] for x in ("ms", "bound", "achieved", "peak", "unit", "frac")},
                                  traffic=traffic_of(k)) for k, v in stages.items()}
    roof["timing"] = (f"per-kernel CUDA events of the frame replayed serialised on one stream (sum {serial_ms:.3f} "
                      f"ms vs {ms_per_step:.3f} ms overlapped)")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if rows_mode else "weak",
        "vs_baseline": None,
        "dtype": ("fp32 semantics: f64 deform, f32 hash tables + features, split-fp16 (hi+lo, 3 MMA chains) "
                  "tcgen05 MLPs with fp32 accumulation" if args.precision == "fp32" else
                  "f64 deform / fp16 hash features / fp16-in fp32-acc MLP"),
        "data": "synthetic (seeded scene, random-init fields)",
        "config": {"workload": f"{args.width}x{args.height} novel-view render, human+rigid object, "
                               f"{args.samples} samples/ray, occupancy-skipped (configs[1])",
                   "precision": args.precision,
                   "rays_per_frame": r.n_rays, "nominal_samples_per_frame": r.n_rays * args.samples,
                   "processed_samples_per_frame": hs + os_, "human_samples_per_frame": hs,
                   "object_samples_per_frame": os_, "ed_nodes": int(len(sc.nodes)),
                   "skin_verts": int(len(sc.skin_verts)),
                   "hash": "16 levels x 2^19 x F2 (canonical) + 8 x 2^17 x F4 (deform)",
                   "step": "motion prior (node dqs + theta + object pose) -> device FK + pose bias + warp setup + "
                           "live occupancy -> full render",
                   "l2": "flushed (256 MiB write) between timed steps, outside the per-step events",
                   "parallelism": (f"{world} ranks, rows of every frame dealt round-robin, frame all-gathered "
                                   "(NCCL) inside the step" if rows_mode else
                                   f"{world} rank(s), each rendering its own frame stream (rays sharded by frame, "
                                   "no data-path collective)")},
        "ms_per_frame": ms_per_step,
        "nominal_samples_per_s": (r.n_rays * args.samples * args.steps * world) / (ms_total / 1e3),
        "stage_ms_serialised": stage_ms,
        "host_issue_ms_per_step": t_issue * 1e3 / args.steps,
        "roofline": roof,
        "gpu_launches": ours * args.steps,
        "gpu_launches_detail": {"per_step": ours, "foreign_kernels_per_step": other, "kernels": names,
                                "how": "CUPTI (torch.profiler) over one graph-replayed step"},
        "e2e": e2e,
        "fp16_mode": fp16,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, budget_s=20.0)
    if rank == 0:
        print(json.dumps(line))


# ----------------------------------------------------------------- CPU path (oracle)

def _cpu_rows(args, frac):
    """A row-strided subset of the frame's rays (every m-th image row, all columns)."""
    m = max(1, int(round(1.0 / frac)))
    rows = np.arange(0, args.height, m)
    return (rows[:, None] * args.width + np.arange(args.width)[None, :]).reshape(-1), m


def cpu_baseline(args, budget_s=20.0):
    """The reference algorithm on the host cores (oracle/pipeline.py, a standalone CPU
    restatement: no device work, no product code), on a bounded sample of the same
    workload: every m-th row of frame 7 incl. the frame's setup."""
    from oracle.pipeline import FramePool
    pool = FramePool(width=args.width, height=args.height, samples=args.samples)
    try:
        ids, m = _cpu_rows(args, 1.0 / 16)
        pool.frame(7, ids[: len(ids) // 4], precision=args.precision)  # warm the workers
        t0 = time.perf_counter()
        done, reps = 0, 0
        while reps < 1 or (time.perf_counter() - t0 < budget_s and reps < 4):
            nh, no, _, _ = pool.frame(7, ids, precision=args.precision)
            done += nh + no
            reps += 1
        el = time.perf_counter() - t0
    finally:
        pool.close()
    return {"value": done / el, "unit": UNIT, "cores": pool.cores, "kind": "port",
            "sample": f"oracle/pipeline.py (numpy restatement of the reference + SPEC, {args.precision} semantics): "
                      f"every {m}th row of frame 7 ({len(ids)} rays x {args.samples} samples, occupancy-skipped) incl. "
                      f"the frame's FK / pose bias / live-occupancy setup, {reps} rep(s), {pool.cores} spawned "
                      f"processes x 1 BLAS thread"}


def _repo_libs_loaded():
    """Shared objects of this repository mapped into this process (the reference arm
    must show none: it runs no product code)."""
    try:
        maps = open("/proc/self/maps").read().split("\n")
    except OSError:
        return None
    return sorted({ln.split()[-1] for ln in maps if ln.endswith(".so") and ln.split()[-1].startswith(ROOT)})


def run_reference(args, rank, world):
    """--impl reference: the reference's algorithm on the host cores — oracle/pipeline.py,
    a standalone CPU restatement (the reference package is pure Python and has no render
    path to install). Same config (the full configs[1] frame: per-frame
    setup + every ray), same metric. Rank 0 only; no device, no product code."""
    if rank != 0:
        return
    from oracle.pipeline import FramePool
    pool = FramePool(width=args.width, height=args.height, samples=args.samples)
    try:
        nF = 10
        t0 = time.perf_counter()
        nh, no, _, _ = pool.frame(7, precision=args.precision)  # warm-up, full frame
        t_frame = time.perf_counter() - t0
        # each step is the full frame unless K of them would not fit in a few minutes:
        # then every m-th row of the frame (same config, bounded sample)
        budget = 150.0
        frac = min(1.0, budget / max(t_frame * (args.steps + max(0, args.warmup - 1)), 1e-9))
        ids, m = (None, 1) if frac >= 1.0 else _cpu_rows(args, frac)
        for w in range(max(0, args.warmup - 1)):
            pool.frame(w % nF, ids, precision=args.precision)
        t0 = time.perf_counter()
        done = 0
        for k in range(args.steps):
            nh, no, _, _ = pool.frame(k % nF, ids, precision=args.precision)
            done += nh + no
        el = time.perf_counter() - t0
    finally:
        pool.close()
    v = done / el
    sample = ("full frame per step" if m == 1 else f"every {m}th row of the frame per step") + \
        f" (frames 0-9 in turn), per-frame setup included; {pool.cores} spawned processes x 1 BLAS thread"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": f"f64 deform / {args.precision} semantics field (numpy)", "data": "synthetic",
            "impl": "reference", "same_config": True, "native_libs_loaded": _repo_libs_loaded(),
            "config": {"workload": f"{args.width}x{args.height} novel-view render, human+rigid object, "
                                   f"{args.samples} samples/ray, occupancy-skipped (configs[1])",
                       "precision": args.precision, "parallelism": f"{pool.cores} host processes"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": pool.cores, "kind": "port",
                             "sample": "oracle/pipeline.py: " + sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_train(args, rank, world, pg):
    """configs[2]: key-frame training step, 2^18 rays (global; sharded over ranks)
    drawn from the 10 key frames, forward + backward + Adam, gradients all-reduced.
    The key frames' images live in HBM; every step draws fresh rays from their
    foreground pixels on the device. The whole step (draw, counts, 10 frames x 2
    fields of forward / backward / dW, bucket all-reduce, Adam, repack) is one CUDA
    graph (Trainer.capture). e2e: the public eager API, Trainer.step, on batches
    uploaded every step from pinned host memory, the losses read back."""
    import torch
    from paper_2304_03184_b200.train import KeyFrame, Trainer, TrainConfig, shard_rays
    sc, cfg, hf, of, r, frames = build_workload(args, rank)
    cam = sc.camera
    r.rays(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    dev = torch.device("cuda", torch.cuda.current_device())
    per_frame = int(np.ceil(args.train_rays / world / len(frames)))
    o, d = cam.all_rays()
    T = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x), dtype=dt, device=dev)  # noqa: E731
    keyframes = []
    for fid, f in enumerate(frames):
        # the key frame's images (targets of the human / object pixels), once, untimed
        th, to, rgb, hum, obj = sc.raycast(o, d, fid)
        depth = np.where(hum, th, np.where(obj, to, 0.0))
        keyframes.append(KeyFrame(cam, T(rgb, torch.float32), T(depth, torch.float32), T(hum, torch.uint8),
                                  T(obj, torch.uint8), T(f["dqs"], torch.float64),
                                  T(sc.bone_transforms(fid), torch.float64),
                                  T(hf.nets.theta_bias(f["theta"]), torch.float32), T(f["theta"], torch.float32),
                                  f["R"], f["t"]))
    tr = Trainer(r, max_rays=per_frame, cfg=TrainConfig())
    group = None if world == 1 else torch.distributed.group.WORLD
    step = tr.capture(keyframes, per_frame, group)  # (its warm-up is a real step)
    for _ in range(max(0, args.warmup - 1)):
        step()
    torch.cuda.synchronize()
    barrier(pg)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        a.record()
        for _ in range(args.steps):
            step()
        b.record()
        torch.cuda.synchronize()
    clk = clocks.summary()
    barrier(pg)
    ms = max_over_ranks(pg, a.elapsed_time(b))
    # samples of a step from its (rank-summed) ray counts: 32 guided + 16 uniform per
    # masked ray with depth, 64 uniform without, per field and frame
    c = tr.counts.cpu().numpy().astype(np.int64)
    per_step = float(sum(48 * c[:, 2 * q + 1] + 64 * (c[:, 2 * q] - c[:, 2 * q + 1]) for q in range(2)).sum())
    ours, other, names = count_launches(step)
    launches = {"per_step": ours, "foreign_kernels_per_step": other, "kernels": names,
                "how": "CUPTI (torch.profiler) over one graph replay"}
    stage_ms, roof = train_stage_roofline(tr, keyframes, per_frame, rank)
    # e2e: eager public API, this step's ray batches uploaded from pinned host memory
    e2e = None
    if not args.no_e2e:
        host = []
        for kf in keyframes:
            bt = kf.sample(per_frame, seed=rank + 17)
            host.append({k: getattr(bt, k).cpu().pin_memory() for k in ("dirs", "gt_rgb", "gt_depth", "mask_h",
                                                                        "mask_o")})
        bufs = [kf.batch_buffers(per_frame) for kf in keyframes]
        for bt in bufs:
            bt.ray0 = rank * per_frame
        h2d = sum(v.numel() * v.element_size() for hb in host for v in hb.values())
        loss_h = torch.empty((2, 2), dtype=torch.float32).pin_memory()

        def e2e_step():
            for bt, hb in zip(bufs, host):
                for k, v in hb.items():
                    getattr(bt, k).copy_(v, non_blocking=True)
            out = tr.step(bufs, group)
            loss_h.copy_(tr.stats, non_blocking=True)
            return out
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier(pg)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        el = max_over_ranks(pg, time.perf_counter() - t0)
        e2e = {"value": per_step * args.steps / el, "unit": "samples/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 16, "ms_per_step": el * 1e3 / args.steps,
               "path": "Trainer.step (eager) on ray batches copied from pinned host memory every step, "
                       "losses read back"}
    line = {"metric": "training samples/s (fwd+bwd+Adam, warp+hash+MLP+composite)", "value":
            per_step * args.steps / (ms / 1e3), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64 deform / fp32-semantics forward (split-fp16 tcgen05) / fp16-operand fp32-acc backward / "
                     "f32 tables, grads, Adam",
            "data": "synthetic (analytic ray-cast targets of the scripted scene)",
            "config": {"workload": f"key-frame training step (configs[2]): {args.train_rays} rays over 10 frames "
                                   f"drawn on the device every step from the HBM-resident key-frame images, "
                                   f"32 guided + 16 uniform / 64 empty samples per ray",
                       "samples_per_step": per_step, "rays_per_frame_per_rank": per_frame,
                       "step": "one CUDA graph: draw + counts + 10 frames x (human, object) fwd/bwd/dW + "
                               "bucket all-reduce + multi-tensor Adam + repack",
                       "l2": "inputs (hash tables 64 MB + 47 MB, per-frame activations) larger than L2",
                       "parallelism": f"dp{world} (rays sharded, ray counts and gradient buckets summed)"},
            "gpu_launches": launches["per_step"] * args.steps, "gpu_launches_detail": launches,
            "clocks": clk, "e2e": e2e, "stage_ms_per_step": stage_ms, "roofline": roof}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = train_cpu_baseline()
    if rank == 0:
        print(json.dumps(line))


# per-sample bytes of the dW GEMM operands (cf_dw_grouped: A and B rows, fp16, read once)
_DW_BYTES = {"human": 2 * ((64 + 32) + (16 + 64) + (64 + 31) + (64 + 64) + (3 + 64)
                           + (3 + 128) + 3 * (128 + 128) + (128 + 33)),
             "object": 2 * ((64 + 32) + (16 + 64) + (64 + 31) + (64 + 64) + (3 + 64))}


def train_stage_roofline(tr, keyframes, per_frame, rank):
    """Per-kernel device time of one eager step (CUDA events around each launch of the
    kernels named below, on the launching stream) and the roofline of the dominant one
    (algorithmic bytes or FLOPs per sample x the step's samples, per field)."""
    import torch
    from paper_2304_03184_b200 import _lib
    names = {"cf_dw_grouped": "dw_grouped", "cf_color_backward": "color_bwd", "cf_field_forward": "field_fwd",
             "cf_field_hash_backward": "hash_bwd_c", "cf_human_canon": "human_canon",
             "cf_deform_backward": "deform_bwd", "cf_deform_hash_backward": "hash_bwd_d",
             "cf_loss_composite_bwd": "loss_composite_bwd"}
    marks = []
    dw_samples = []  # (field, the dW launch's K: the field's compacted sample count) per launch
    real = _lib.call
    count_of = {st["cbuf"].counters.data_ptr(): st for st in tr.fields}

    def timed(name, *a):
        if name not in names:
            return real(name, *a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        real(name, *a)
        e1.record()
        marks.append((names[name], e0, e1))
        if name == "cf_dw_grouped":
            st = count_of[a[2]]
            dw_samples.append((st["name"], st["cbuf"].counters[0].clone()))
    bufs = [kf.batch_buffers(per_frame) for kf in keyframes]
    for f, (kf, b) in enumerate(zip(keyframes, bufs)):
        kf.draw(b, seed=f * 64 + rank + 99)
        b.ray0 = rank * per_frame
    torch.cuda.synchronize()
    _lib.call = timed
    try:
        tr.step(bufs, None, update=False)
        torch.cuda.synchronize()
    finally:
        _lib.call = real
    ms = {}
    for n, e0, e1 in marks:
        ms[n] = ms.get(n, 0.0) + e0.elapsed_time(e1)
    peaks = load_peaks()
    work = float(sum(int(k) * _DW_BYTES[q] for q, k in dw_samples))
    t = ms["dw_grouped"]
    ach = work / (t / 1e3) / 1e9
    peak, src = peaks["hbm_gbs"]
    roof = {"kernel": "dw_grouped (tcgen05 split-K weight gradients, 2 launches per frame)", "bound": "hbm",
            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "per_unit": "fp16 operand rows read once per field sample (the compacted valid ones, the GEMMs' K): "
                        "human 3,052 B (E_g/E_c 932 + DeformNet 2,120), object 932 B",
            "peak_source": src, "ms": t, "traffic": None,
            "timing": "CUDA events around each launch of one eager step (update=False), summed per kernel"}
    top = max(ms, key=ms.get)
    roof["dominant_by_time"] = top
    return {k: round(v, 3) for k, v in sorted(ms.items(), key=lambda kv: -kv[1])}, roof


def train_cpu_baseline(budget_s=15.0):
    """The training step's human-field work on the host (oracle/pipeline.train_rays: the
    SPEC's algorithm in numpy / float64 torch autograd, one process, no device work) on
    a bounded sample of the key frame's foreground rays."""
    import torch
    from oracle import pipeline as op
    torch.set_num_threads(os.cpu_count() or 1)
    S = op.build_static(width=512, height=512, samples=128, table_scale=1e-4)
    sc = S["scene"]
    o, d = sc.camera.all_rays()
    _, _, _, hum, _ = sc.raycast(o, d, 3)
    fg = np.nonzero(hum)[0]
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    done, reps = 0, 0
    while reps < 1 or time.perf_counter() - t0 < budget_s:
        done += op.train_rays(S, 3, rng.choice(fg, 64), seed=reps)
        reps += 1
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": "samples/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"oracle/pipeline.train_rays: {reps} x 64 human rays of key frame 3 (depth-guided samples, "
                      f"hybrid canonicalisation, fp32-semantics field, float64 autograd gradients of every human "
                      f"parameter, Adam) in one process (torch intra-op threads = cores)"}


def run_knn(args, rank, world, pg):
    """configs[3]: dense ED graph scaling — exact k-NN + DQB^-1 backward warp of
    2^20 queries over n = 1024..8192 deformed nodes, k = 4/8: hierarchical bucket
    search vs the exhaustive GPU kernel (bit-identical results checked here)."""
    import torch
    from oracle import deform as od
    from paper_2304_03184_b200 import _lib
    from paper_2304_03184_b200.edgraph import Buckets, knn_warp, knn_warp_cull, morton_order
    from paper_2304_03184_b200.scene import Scene, SceneConfig
    sc = Scene(SceneConfig(), seed=0)
    rng = np.random.default_rng(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    rows = []
    for n in (1024, 2048, 4096, 8192):
        nodes = sc.template_points[rng.choice(len(sc.template_points), n, replace=False)]
        A = sc.bone_transforms(7)
        bones = sc.template_bones[np.argmin(((nodes[:, None] - sc.template_points[None, :4000]) ** 2).sum(-1), 1)]
        dqs = np.stack([od.dq_from_rt(A[b, :3, :3], A[b, :3, 3]) for b in bones])
        anchors = od.deformed_nodes(nodes, dqs)
        half = 1 << 19
        q = np.concatenate([anchors[rng.integers(0, n, half)] + rng.normal(scale=0.02, size=(half, 3)),
                            rng.uniform(anchors.min(0), anchors.max(0), size=(half, 3))])
        a_t = torch.from_numpy(anchors).to(dev)
        d_t = torch.from_numpy(dqs).to(dev)
        q_t = torch.from_numpy(q).to(dev)
        b = Buckets(n)
        for k in (4, 8):
            res = {}

            def culled():  # Morton sort of the queries (per call) + warp-culled exact search
                return knn_warp_cull(a_t, d_t, k, 0.1, _lib.CF_WARP_BACKWARD, q_t, morton_order(q_t),
                                     want_idx=True)

            def bucketed():  # per-frame build (buckets + candidate lists) + ring search
                b.build(a_t, candidates_k=k)
                return knn_warp(a_t, d_t, k, 0.1, _lib.CF_WARP_BACKWARD, q_t, b, want_idx=True)

            def brute():
                return knn_warp(a_t, d_t, k, 0.1, _lib.CF_WARP_BACKWARD, q_t, None, want_idx=True)

            for name, fn in (("culled", culled), ("bucketed", bucketed), ("brute", brute)):
                for _ in range(2):
                    out = fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 5
                e0.record()
                for _ in range(reps):
                    out = fn()
                e1.record()
                torch.cuda.synchronize()
                res[name] = (len(q) * reps / (e0.elapsed_time(e1) / 1e3), out[0])
            same = bool(torch.equal(res["culled"][1], res["brute"][1]) and
                        torch.equal(res["bucketed"][1], res["brute"][1]))
            rows.append({"n_nodes": n, "k": k, "hierarchical_qps": res["culled"][0],
                         "bucketed_qps": res["bucketed"][0], "brute_force_qps": res["brute"][0],
                         "speedup": res["culled"][0] / res["brute"][0], "indices_identical": same})
    # KnnField (the paper's O(1) LUT search, knnfield.py:45-222) on the scene's 128-node
    # graph: canonical field build, per-frame live map, and the query of 2^20 live points
    from paper_2304_03184_b200.edgraph import EDGraph, GraphMotion
    from paper_2304_03184_b200.knnfield import KnnField
    graph = EDGraph(sc.nodes, radius=0.1, knn_k=4)
    field_rows = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for res in (64, 128, 256):
        torch.cuda.synchronize()
        e0.record()
        kf = KnnField(graph, resolution=res, s=4)
        e1.record()
        torch.cuda.synchronize()
        build_ms = e0.elapsed_time(e1)
        upd = []
        for fid in range(3):
            e0.record()
            kf.update_live_map(GraphMotion(fid, sc.node_dqs(fid)))
            e1.record()
            torch.cuda.synchronize()
            upd.append(e0.elapsed_time(e1))
        anchors = od.deformed_nodes(np.asarray(sc.nodes), sc.node_dqs(2))
        q = torch.from_numpy(anchors[rng.integers(0, len(anchors), 1 << 20)]
                             + rng.normal(scale=0.03, size=(1 << 20, 3))).to(dev)
        kf.query_motion_batch(q, 2)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            out = kf.query_motion_batch(q, 2)
        e1.record()
        torch.cuda.synchronize()
        qps = 5 * (1 << 20) / (e0.elapsed_time(e1) / 1e3)
        field_rows.append({"resolution": res, "build_ms": build_ms, "update_live_map_ms": float(np.median(upd[1:])),
                           "query_qps": qps, "valid_fraction": float(out[3].float().mean())})
    line = {"metric": "exact k-NN + DQB^-1 backward warps/s (dense ED graph, configs[3])",
            "value": min(r["hierarchical_qps"] for r in rows), "unit": "queries/s", "n_gpus": 1,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic (template subsets, GT motion, 2^20 queries)",
            "config": {"workload": "configs[3]: n = 1024..8192 nodes, k = 4/8, half near-surface / half uniform "
                                   "queries; hierarchical = Morton sort of the queries + warp-culled search "
                                   "(sort included per call); bucketed = voxel buckets + candidate lists + ring "
                                   "search (build included per call); brute = exhaustive kernel"}, "rows": rows,
            "knnfield": {"graph": "scene, 128 nodes, s = 4", "rows": field_rows,
                         "reference_cpu": "SURVEY 8(a): build 2 s @64^3 .. 58 s @256^3; live map 0.04 .. 1.65 s; "
                                          "query 0.25-0.36 M samples/s"}}
    if rank == 0:
        print(json.dumps(line))


def run_frontend(args, rank, world, pg):
    """SURVEY §8(f) 2-3, the stages either side of the path: motion-prior ingestion
    (CFMP decode + one upload + device FK of every frame) and key-frame selection
    per tracked frame (blur gate on the 512^2 RGB, Eq. 5 visibility of the deformed
    nodes, Eq. 6 scan + update of a 100-entry pool incl. the decision readback)."""
    import tempfile
    import time
    import torch
    from oracle import keyframes as okf
    from paper_2304_03184_b200 import keyframes as kf, records
    from paper_2304_03184_b200.scene import Scene, SceneConfig
    sc = Scene(SceneConfig(), seed=0)
    rng = np.random.default_rng(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    n_nodes, n_frames = 8192, 1000
    # -- ingestion: a 1000-frame stream of an 8192-node graph (~540 MB)
    path = os.path.join(tempfile.mkdtemp(), "motions.bin")
    wr = records.MotionPriorWriter(path, n_nodes, 72)
    dq = np.zeros((n_nodes, 8))
    dq[:, 0] = 1.0
    batch = [records.MotionPrior(f, records.GraphMotion(f, dq), records.SkeletonPose(None, sc.theta(f % 10)),
                                 records.Se3()) for f in range(100)]
    for rep in range(n_frames // 100):
        for i, b in enumerate(batch):
            b.frame_id = b.graph_motion.frame_id = rep * 100 + i
        wr.append_batch(batch)
    records.MotionPriorStream(path)  # warm (page cache, pinned pool)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = records.MotionPriorStream(path)
    torch.cuda.synchronize()
    ingest_s = time.perf_counter() - t0
    th = st.theta
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    records.skinning_transforms(th)
    e0.record()
    for _ in range(10):
        records.skinning_transforms(th)
    e1.record()
    torch.cuda.synchronize()
    fk_us = e0.elapsed_time(e1) * 100.0  # per call of 1000 frames, us
    os.remove(path)
    # -- key-frame selection per tracked frame
    W = H = 512
    rgbs = [torch.from_numpy(rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)).to(dev) for _ in range(4)]
    depth = torch.from_numpy(rng.uniform(0.5, 4.0, size=(H, W))).to(dev)
    nodes = torch.from_numpy(sc.template_points[rng.choice(len(sc.template_points), n_nodes, replace=False)]).to(dev)
    cam = sc.camera
    pool = kf.KeyFramePool("human", n_nodes=n_nodes, capacity=100, gamma=0.0)  # every frame inserted / evicts
    thetas = torch.from_numpy(rng.normal(size=(64, 72)) * 0.3)

    def frame(f):
        b = kf.blur_score(rgbs[f % 4])
        vis = kf.visibility_bits(nodes, depth, cam)
        pool.update(kf.FrameSummary(f, thetas[f % 64].numpy(), vis))
        return b

    for f in range(args.warmup + 100):
        frame(f)
    torch.cuda.synchronize()
    K = max(args.steps, 200)
    t0 = time.perf_counter()
    for f in range(K):
        frame(1000 + f)
    torch.cuda.synchronize()
    sel_ms = (time.perf_counter() - t0) * 1e3 / K
    # CPU oracle of the same per-frame selection work (blur + visibility + 100-entry scan), 1 core
    rgb_h, depth_h, nodes_h = rgbs[0].cpu().numpy(), depth.cpu().numpy(), nodes.cpu().numpy()
    Rwc, twc = kf.world_to_cam(cam)
    ent = [(i, rng.normal(size=72), okf.pack_bits(rng.random(n_nodes) < 0.5)) for i in range(100)]
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        okf.blur_score(rgb_h)
        vb = okf.pack_bits(okf.visibility_map(nodes_h, depth_h, Rwc, twc, cam.fx, cam.fy, cam.cx, cam.cy))
        ds = [okf.dissim_human(thetas[0].numpy(), vb, 5000, e[1], e[2], e[0]) for e in ent]
        okf.pool_decision(ds, [e[0] for e in ent])
    cpu_ms = (time.perf_counter() - t0) * 1e3 / reps
    # -- rigid-object TSDF (tracking front-end): 256^3 volume, 512^2 depth of a sphere
    from paper_2304_03184_b200.tsdf import TsdfVolume

    class _P:
        rotation, translation = np.eye(3), np.zeros(3)
    tcam = type("C", (), dict(fx=560.0, fy=560.0, cx=255.5, cy=255.5, width=512, height=512, pose=_P()))()
    us, vs = np.meshgrid(np.arange(512.0), np.arange(512.0))
    dx, dy = (us - 255.5) / 560.0, (vs - 255.5) / 560.0
    dn = np.sqrt(dx * dx + dy * dy + 1.0)
    b = 1.3 / dn
    disc = b * b - (1.3 * 1.3 - 0.3 * 0.3)
    tdepth = np.where(disc > 0, (b - np.sqrt(np.maximum(disc, 0))) / dn, 0.0)  # camera z of the sphere hit
    tv = TsdfVolume(256, 0.7 / 256, np.array([-0.35, -0.35, 0.95]))
    tdev = torch.from_numpy(tdepth).to(dev)
    for _ in range(3):
        tv.integrate(tdev, tcam, _P())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tv.integrate(tdev, tcam, _P())
    e1.record()
    torch.cuda.synchronize()
    integ_ms = e0.elapsed_time(e1) / 10
    tv.raycast(tcam, _P(), stride=1)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        rp, _ = tv.raycast(tcam, _P(), stride=1)
    e1.record()
    torch.cuda.synchronize()
    ray_ms = e0.elapsed_time(e1) / 5
    # -- non-rigid tracking solve: the reference tracker's own Gauss-Newton system
    import scipy.sparse as sps
    from oracle import tracking as otr
    from paper_2304_03184_b200.tracking import GaussNewtonSystem
    with np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden", "pcg_ref.npz")) as z:
        pj = {k: z[k] for k in z.files}
    gn = GaussNewtonSystem((pj["val"], pj["col"], pj["rowptr"], pj["shape"]), pj["r"])
    for _ in range(3):
        gn.solve(1e-4)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        gn.solve(1e-4)
    e1.record()
    torch.cuda.synchronize()
    pcg_us = e0.elapsed_time(e1) * 1e3 / 20
    Js = sps.csr_matrix((pj["val"], pj["col"], pj["rowptr"]), shape=tuple(pj["shape"]))
    t0 = time.perf_counter()
    for _ in range(5):
        otr.pcg_solve_sparse(Js, pj["r"], 1e-4)
    pcg_cpu_us = (time.perf_counter() - t0) * 1e6 / 5
    # -- non-rigid tracking: the reference's bend-tracking scene (tests/golden/tracker_ref.npz)
    from paper_2304_03184_b200.tracking import NonrigidTracker
    with np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden", "tracker_ref.npz")) as z:
        tz = {k: z[k] for k in z.files}

    class _NS:
        def __init__(self, **kw):
            self.__dict__.update(kw)
    tmodel = _NS(graph=_NS(nodes=tz["nodes"], radius=float(tz["radius"]), knn_k=int(tz["knn_k"])),
                 skeleton=_NS(parents=tz["parents"], offsets=tz["offsets"], joint_limits=tz["joint_limits"]),
                 points=tz["points"], normals=tz["normals"], lbs_weights=tz["lbs_weights"],
                 node_lbs_weights=tz["node_lbs_weights"], edges=tz["edges"])
    c = tz["cam"]
    tcam2 = _NS(fx=float(c[0]), fy=float(c[1]), cx=float(c[2]), cy=float(c[3]), width=int(c[4]), height=int(c[5]),
                pose=_NS(rotation=tz["cam_R"], translation=tz["cam_t"]))
    NonrigidTracker(tmodel, tcam2, surface_samples=1500).solve(tz["depth0"], tz["mask0"], 0)  # warm
    torch.cuda.synchronize()
    ntr = NonrigidTracker(tmodel, tcam2, surface_samples=1500)
    t0 = time.perf_counter()
    n_iters = 0
    for fid in range(4):
        _, tinfo = ntr.solve(tz[f"depth{fid}"], tz[f"mask{fid}"], fid)
        n_iters += tinfo["iterations"]
    torch.cuda.synchronize()
    track_ms = (time.perf_counter() - t0) * 1e3 / 4
    line = {"metric": "front-end stages: key-frame selection per tracked frame; motion-prior ingestion",
            "value": 1e3 / sel_ms, "unit": "tracked frames/s (selection)", "n_gpus": 1, "higher_is_better": True,
            "ms_per_frame_selection": sel_ms, "dtype": "u8 / f64 / int",
            "data": "synthetic (random 512^2 RGB and depth, 8192 template nodes, 1000-frame CFMP stream)",
            "ingest": {"frames": n_frames, "n_nodes": n_nodes, "stream_bytes": int(st.dqs.numel() * 8 + n_frames * 700),
                       "decode_upload_fk_s": ingest_s, "fk_us_per_1000_frames": fk_us},
            "tsdf": {"resolution": 256, "integrate_ms": integ_ms, "voxels_per_s": 256 ** 3 / (integ_ms * 1e-3),
                     "raycast_512x512_ms": ray_ms, "raycast_hits": int(len(rp))},
            "nonrigid_tracking": {"scene": "reference bend test, 142 nodes, 1500 surface samples, 128^2 depth",
                                  "ms_per_frame": track_ms, "lm_iterations_per_frame": n_iters / 4,
                                  "reference_cpu_s_per_frame": "2.9 (measured in the build container, 8 cores)"},
            "pcg": {"system": f"{int(pj['shape'][0])}x{int(pj['shape'][1])}, nnz {len(pj['val'])} (reference tracker)",
                    "iterations": 32, "gpu_us_per_solve": pcg_us, "cpu_scipy_us_per_solve": pcg_cpu_us},
            "cpu_baseline": {"value": 1e3 / cpu_ms, "unit": "tracked frames/s", "cores": 1, "kind": "port",
                             "sample": "oracle blur + visibility + 100-entry Eq. 6 scan, 3 frames"},
            "config": {"workload": "SURVEY 8(f) 2-3 front-end stages; selection = blur(512^2) + visibility(8192 "
                                   "nodes) + pool scan/update (100 entries, decision readback each frame)"}}
    if rank == 0:
        print(json.dumps(line))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":  # host cores only: no process group, no device
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, int(os.environ.get("RANK", "0")), world)
        return
    rank, world, local, pg = dist_setup(args)
    if args.workload == "render" and not __import__("torch").cuda.is_available():
        raise SystemExit("bench.py: the render workload needs a CUDA device (there is no CPU fallback)")
    if args.workload == "train":
        run_train(args, rank, world, pg)
    elif args.workload == "knn":
        run_knn(args, rank, world, pg)
    elif args.workload == "frontend":
        run_frontend(args, rank, world, pg)
    else:
        run_ours(args, rank, world, pg)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
