"""Probe: time the human canonicalisation kernel variants on the 512^2 C2 frame."""
import ctypes, numpy as np, torch
from paper_2304_03184_b200 import _lib
from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
from paper_2304_03184_b200.scene import Scene, SceneConfig
sc = Scene(SceneConfig(width=512, height=512), seed=0)
cfg = RenderConfig()
hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg)
of = ObjectField(sc.box_half, cfg)
r = Renderer(hf, of, 512, 512, cfg)
R, t = sc.object_pose(7)
r.set_frame(sc.node_dqs(7), sc.theta(7), sc.bone_transforms(7), R, t)
cam = sc.camera
r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy)
torch.cuda.synchronize()
hb = r.hb
n = int(hb.counters[0])
flags = hb.xu[:n, 3].cpu().numpy()
print("samples", n, "ED", (flags == 1).mean(), "LBS", (flags == 2).mean(), "none", (flags == 0).mean())
def timeit(w, nb, lb, reps=20):
    s = _lib.stream_ptr()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(3):
        _lib.call("cf_human_canon", _lib.byref(r.M), r.dirs.data_ptr(), _lib.byref(hb.mo), _lib.byref(w), nb, lb, hb.xu.data_ptr(), s)
    e0.record()
    for i in range(reps):
        _lib.call("cf_human_canon", _lib.byref(r.M), r.dirs.data_ptr(), _lib.byref(hb.mo), _lib.byref(w), nb, lb, hb.xu.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
w = r.hw
print("smem+lbs   us", timeit(w, r._anchor_buckets.handle, hf.lbs.buckets.handle))
w2 = _lib.HumanWarp(); ctypes.memmove(ctypes.byref(w2), ctypes.byref(w), ctypes.sizeof(w2)); w2.vert_Tinv = None
print("smem nolbs us", timeit(w2, r._anchor_buckets.handle, None))
w3 = _lib.HumanWarp(); ctypes.memmove(ctypes.byref(w3), ctypes.byref(w), ctypes.sizeof(w3)); w3.n_nodes = 100000
print("bucket+lbs us", timeit(w3, r._anchor_buckets.handle, hf.lbs.buckets.handle))
# pure knn+blend through cf_knn_warp on the same points
o = np.asarray(cam.t); rec = hb.records[:n].cpu().numpy().view(np.uint32)
ray = (rec >> 8).astype(np.int64); i = (rec & 255).astype(np.int64)
tt = 0.3 + (i + 0.5) * r.M.dt
p = torch.from_numpy(o[None] + tt[:, None] * r.dirs.cpu().numpy()[ray]).cuda()
from paper_2304_03184_b200.edgraph import knn_warp
anchors = r._anchors; dqs = r._dqs
for mode, b in (("bucket", r._anchor_buckets), ("brute", None)):
    for _ in range(3): knn_warp(anchors, dqs, 4, 0.1, _lib.CF_WARP_BACKWARD, p, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): knn_warp(anchors, dqs, 4, 0.1, _lib.CF_WARP_BACKWARD, p, b)
    e1.record(); torch.cuda.synchronize()
    print("cf_knn_warp", mode, "us", e0.elapsed_time(e1) / 20 * 1e3)
