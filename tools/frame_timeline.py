"""Per-kernel timeline of one graph-replayed bench frame (CUPTI via torch.profiler)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile


class A:
    width = height = 512
    samples = 128
    precision = os.environ.get("PREC", "fp32")


def main():
    import bench
    torch.cuda.set_device(0)
    sc, cfg, hf, of, r, frames = bench.build_workload(A, 0)
    cam = sc.camera
    dev = torch.device("cuda", 0)
    df = [(torch.from_numpy(f["dqs"]).to(dev), torch.from_numpy(f["theta"]).to(dev), f["R"], f["t"]) for f in frames]

    def step(fi):
        dqs, theta, R, t = df[fi]
        r.load_pose(dqs, theta)
        r.set_object_pose(R, t)
        return r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    for i in range(8):
        step(i % len(df))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(3):
            step(5)
        torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if not str(getattr(e, "device_type", "")).endswith("CUDA"):
            continue
        n = e.name.replace("(anonymous namespace)::", "").replace("void ", "")
        if n.startswith("cuda") or "Graph" in n:
            continue
        ev.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", -1), n.split("(")[0][:48]))
    ev.sort()
    # the last frame: from the last march_kernel backwards to the previous composite_final
    idx = [i for i, e in enumerate(ev) if e[3].startswith("march_kernel")]
    start_i = idx[-1]
    while start_i > 0 and not ev[start_i - 1][3].startswith("composite_final"):
        start_i -= 1
    t0 = ev[start_i][0]
    for s, e, sid, n in ev[start_i:]:
        print(f"{(s - t0):8.1f} {(e - t0):8.1f} {e - s:7.1f}  stream {sid:3d}  {n}")


if __name__ == "__main__":
    main()
