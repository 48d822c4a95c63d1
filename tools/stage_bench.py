"""Time single human field stages (back to back, CUDA events) of the human chain at the bench config (512^2, 128 samples).
usage: python tools/stage_bench.py [stage ...]   (0 hash_d, 1 deform MLP, 2 hash_c, 3 color MLP)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2304_03184_b200 import _lib


class A:
    width = height = 512
    samples = 128
    precision = os.environ.get("PREC", "fp32")


def main():
    import bench
    torch.cuda.set_device(0)

    sc, cfg, hf, of, r, frames = bench.build_workload(A, 0)
    cam = sc.camera
    r.cfg.serial = True
    f = frames[5]
    r.load_pose(torch.from_numpy(f["dqs"]).cuda(), torch.from_numpy(f["theta"]).cuda())
    r.set_object_pose(f["R"], f["t"])
    r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
    torch.cuda.synchronize()
    hb = r.hb
    n = int(hb.counters[0])
    print("human samples", n, "capacity", hb.mo.capacity)
    s = _lib.stream_ptr()
    scratch = r._scratch(hb, r.hdesc).data_ptr()
    stages = [int(x) for x in sys.argv[1:]] or [1]
    out0 = hb.out.clone()
    for st in stages:
        def run():
            _lib.call("cf_field_stage", _lib.byref(r.hdesc), _lib.byref(hb.mo), r.dirs.data_ptr(), hb.xu.data_ptr(),
                      hb.out.data_ptr(), scratch, st, s)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 20)
        print(f"stage {st}: back-to-back median {np.median(ts):.1f} us  min {np.min(ts):.1f} us")
    # re-run the full chain and compare against the first render's output (same kernels)
    for st in range(4):
        _lib.call("cf_field_stage", _lib.byref(r.hdesc), _lib.byref(hb.mo), r.dirs.data_ptr(), hb.xu.data_ptr(),
                  hb.out.data_ptr(), scratch, st, s)
    torch.cuda.synchronize()
    print("chain output identical:", bool(torch.equal(out0[:n], hb.out[:n])))


if __name__ == "__main__":
    main()
