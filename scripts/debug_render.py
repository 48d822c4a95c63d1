import numpy as np, torch
from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
from paper_2304_03184_b200.scene import Scene, SceneConfig
sc = Scene(SceneConfig(width=64, height=64), seed=0)
cfg = RenderConfig(n_samples=64)
hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, seed=0, zero_deform_out=False, table_scale=0.5)
of = ObjectField(sc.box_half, cfg, seed=1, table_scale=0.5)
for f in (hf, of):
    f.nets.layers["G2"][0] *= 6.0
    f.nets.repack()
r = Renderer(hf, of, 64, 64, cfg)
R, t = sc.object_pose(7)
r.set_frame(sc.node_dqs(7), sc.theta(7), sc.bone_transforms(7), R, t)
img = r.render(sc.camera.R, sc.camera.t, sc.camera.fx, sc.camera.fy, sc.camera.cx, sc.camera.cy)
torch.cuda.synchronize()
print("counts", r.sample_counts())
for name, b in (("h", r.hb), ("o", r.ob)):
    n = int(b.counters[0]); out = b.out[:n].cpu().numpy()
    print(name, "sigma q", np.quantile(out[:,0],[0,.5,.9,1]), "opac max", b.opacity.max().item(), "rays", (b.ray_count>0).sum().item(), "per-ray max", b.ray_count.max().item())
