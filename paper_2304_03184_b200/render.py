"""Novel-view rendering of the human + rigid-object scene on the GPU — the SPEC
render path (canonicalize_human SPEC.md:372-380, volume_render :381-389,
render_view :399-407, composite :555-563) with occupancy skipping.

Per frame (every step a CUDA kernel, stream-ordered, no host sync): deformed
nodes + live buckets -> backward-LBS vertex transforms -> live occupancy splat ;
per view: rays -> march (occupancy-skipped compaction) -> canonicalise (ED
DQB^-1 / LBS fallback | rigid) -> fused field (hash + tcgen05 MLPs) ->
front-to-back composite -> depth-occlusion layer composite.

The launch sequence is static: per-frame inputs live in fixed device buffers
(prior tensors, a 28-double frame block holding the camera and object pose), so
it is captured once into a CUDA graph and replayed per view — the host cost of a
frame is a few small copies and one graph launch instead of ~25 launches.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._tensors import dev
from .edgraph import Buckets, FrameMotion, EDGraph, GraphMotion
from .nrf import HashGrid, HashGridConfig, pack_weight
from .skeleton import BackwardLBS

CANON_GRID = HashGridConfig(16, 2, 19, 16, 2048)   # config.py:56-60
DEFORM_GRID = HashGridConfig(8, 4, 17, 16, 256)    # SPEC.md:419 (L=8, F=4); T, N_max frozen in DESIGN.md §4


class _ReadBack:
    """Handle of one view's image read-back (Renderer.render_to_host)."""

    def __init__(self, renderer, slot, img, ready):
        self.r, self.slot, self.img, self.ready, self.event = renderer, slot, img, ready, None

    def _ensure(self):
        if self.event is None:  # no later view issued it: issue it now
            self.r._issue_readback(self)

    def synchronize(self) -> None:
        self._ensure()
        self.event.synchronize()

    def query(self) -> bool:
        self._ensure()
        return self.event.query()


@dataclass
class RenderConfig:
    n_samples: int = 128          # C2: 128 samples / ray
    t_near: float = 0.3           # config.py:53-54
    t_far: float = 5.0
    t_term: float = 1e-4          # early ray termination
    ed_k: int = 4
    ed_radius: float = 0.1
    lbs_max_dist: float = 0.2
    world_min: tuple = (-1.3, -0.3, -1.3)   # live-space occupancy volume (cube)
    world_size: float = 2.6
    live_occ_res: int = 128
    canon_occ_res: int = 128
    canon_occ_radius: float = 0.03   # geometry-initialised density bits
    obj_occ_res: int = 64
    obj_shell: float = 0.02
    # occupancy refresh from the trained density (refresh_occupancy): a cell is occupied
    # when its max-decayed density keeps one sample's opacity 1 - exp(-sigma dt) above
    # occ_alpha; the log-density decays by occ_decay per refresh
    # hierarchical k-NN of the canonicalisation (graphs <= 1024 nodes): a per-frame grid of
    # cand_grid_res cells along the longest side with per-cell candidate lists (0 = the
    # warp-cooperative culled scan instead)
    cand_grid_res: int = 48
    cand_grid_cmax: int = 64
    fuse_hash: bool = True  # fp32 mode: hash lookups inside the MLP kernels (cf_field_desc.split_stages = 0)
    occ_alpha: float = 0.01
    occ_decay: float = 0.95
    background: tuple = (24 / 255.0, 28 / 255.0, 34 / 255.0)   # config.py bg_r/g/b
    # "fp32": fp32 hash tables and features, split-fp16 (hi + lo) tensor-core MLP operands —
    # the SPEC's 32-bit semantics within 1e-4; "fp16": fp16 operands and
    # features, fp16 copy of the deformation table
    precision: str = "fp32"
    cuda_graphs: bool = True      # replay the captured frame (False: launch every kernel each view)
    serial: bool = False          # every launch on the caller's stream (per-kernel timing; no side stream)


def _precise(precision: str) -> bool:
    if precision not in ("fp32", "fp16"):
        raise ValueError(f"precision must be 'fp32' or 'fp16', not {precision!r}")
    return precision == "fp32"


def _kaiming(rng, n_out, n_in):
    b = np.sqrt(6.0 / n_in)
    return rng.uniform(-b, b, size=(n_out, n_in))


def _refresh_density(field, W1, W2, dt, dilate, bits) -> None:
    cfg = field.cgrid.table.device
    res = field.occ.res if isinstance(field, ObjectField) else field.cfg.canon_occ_res
    if getattr(field, "density_logits", None) is None:
        field.density_logits = torch.full((res ** 3,), float("-inf"), dtype=torch.float32, device=cfg)
        field._density_scratch = torch.empty(res ** 3 // 32, dtype=torch.int32, device=cfg)
    c = field.cfg
    log_thr = float(np.log(-np.log1p(-c.occ_alpha) / dt))  # sigma_thr = -ln(1 - alpha) / dt
    W1 = W1.to(torch.float32).contiguous()
    W2 = W2.to(torch.float32).contiguous()
    _lib.call("cf_density_grid_update", _lib.byref(field.cgrid.desc), field.cgrid.table.data_ptr(), W1.data_ptr(),
              W2.data_ptr(), res, float(np.log(c.occ_decay)), log_thr, dilate, field.density_logits.data_ptr(),
              bits.data_ptr(), field._density_scratch.data_ptr(), _lib.stream_ptr())
    field._density_keep = (W1, W2)  # alive until the stream-ordered kernel ran


def occ_grid(gmin, size, res) -> _lib.OccGrid:
    g = _lib.OccGrid()
    for a in range(3):
        g.min[a] = float(gmin[a])
    g.cell = float(size) / res
    g.res = int(res)
    return g


class FieldNets:
    """Weights of one field: [DeformNet], E_g, E_c (fp32 on the host). The device blobs
    hold them in the tcgen05 operand layout: `blob` = fp16(W), `blob_lo` =
    fp16(W - fp16(W)) (used by the "fp32" precision mode)."""

    def __init__(self, rng, deform: bool, zero_deform_out: bool = True, theta_dim: int = 72):
        self.deform = deform
        L = {}
        if deform:
            L["D1"] = _kaiming(rng, 128, 32 + theta_dim)   # hash_d(32) (+) theta(72)
            for i in (2, 3, 4):
                L[f"D{i}"] = _kaiming(rng, 128, 128)
            L["D5"] = np.zeros((3, 128)) if zero_deform_out else _kaiming(rng, 3, 128) * 0.1
        L["G1"] = _kaiming(rng, 64, 32)
        L["G2"] = _kaiming(rng, 16, 64)
        L["C1"] = _kaiming(rng, 64, 31)
        L["C2"] = _kaiming(rng, 64, 64)
        L["C3"] = _kaiming(rng, 3, 64)
        self.layers = {k: np.asarray(v, dtype=np.float32) for k, v in L.items()}
        self.repack()

    def repack(self) -> None:
        """Upload the host weights in the tcgen05 operand layout (hi and lo halves)."""
        self.layers = {k: np.asarray(v, dtype=np.float32) for k, v in self.layers.items()}
        order = (["D1h", "D2", "D3", "D4", "D5"] if self.deform else []) + ["G1", "G2", "C1", "C2", "C3"]
        mats = [self.layers["D1"][:, :32] if k == "D1h" else self.layers[k] for k in order]
        blob = np.concatenate([pack_weight(m) for m in mats])
        self.w_bytes = int(blob.size)
        self.blob = dev(blob.copy(), dtype=torch.uint8)
        self.blob_lo = dev(np.concatenate([pack_weight(m, lo=True) for m in mats]).copy(), dtype=torch.uint8)
        # DeformNet layer 1 in fp32 on the device: its pose columns give the per-frame
        # bias on the device (cf_pose_bias); the trainer updates this tensor in place
        if self.deform:
            if getattr(self, "d1", None) is None:
                self.d1 = dev(self.layers["D1"], dtype=torch.float32)
            else:
                self.d1.copy_(torch.from_numpy(self.layers["D1"]))

    def theta_bias(self, theta) -> np.ndarray:
        """DeformNet layer-1 pose term W1[:, 32:] @ theta, folded into a per-frame bias (fp32)."""
        W = self.layers["D1"][:, 32:].astype(np.float32)
        return (W @ np.asarray(theta, dtype=np.float32)).astype(np.float32)


class HumanField:
    """Canonical human radiance field + its static canonical occupancy."""

    def __init__(self, nodes, template_points, skin_verts, skin_weights, cfg: RenderConfig | None = None,
                 seed: int = 0, zero_deform_out: bool = True, table_scale: float = 1e-4):
        self.cfg = cfg = cfg or RenderConfig()
        nodes = np.asarray(nodes, dtype=np.float64)
        lo, hi = nodes.min(0), nodes.max(0)
        self.side = float((hi - lo).max() + 2 * 0.15)
        self.canon_min = (lo + hi) / 2 - self.side / 2
        self.inv_side = 1.0 / self.side
        rng = np.random.default_rng(seed)
        self.cgrid = HashGrid(CANON_GRID, init_scale=table_scale, seed=seed + 1)
        self.dgrid = HashGrid(DEFORM_GRID, init_scale=table_scale, seed=seed + 2, read_half=True)
        self.nets = FieldNets(rng, deform=True, zero_deform_out=zero_deform_out)
        self.graph = EDGraph(nodes, radius=cfg.ed_radius, knn_k=cfg.ed_k)
        self.nodes = dev(nodes, shape_last=3)
        self.node_buckets = Buckets(len(nodes))
        self.node_buckets.build(self.nodes)
        self.lbs = BackwardLBS(skin_verts, skin_weights, max_dist=cfg.lbs_max_dist)
        # geometry-initialised canonical density bits (stand-in for a trained density grid)
        self.canon_occ = occ_grid(self.canon_min, self.side, cfg.canon_occ_res)
        self._tpl = dev(template_points, shape_last=3)
        tb = Buckets(len(template_points))
        tb.build(self._tpl)
        nwords = (cfg.canon_occ_res ** 3 + 31) // 32
        self.canon_bits = torch.empty(nwords, dtype=torch.int32, device=self.nodes.device)
        _lib.call("cf_occ_from_points", tb.handle, _lib.byref(self.canon_occ), cfg.canon_occ_radius,
                  self.canon_bits.data_ptr(), _lib.stream_ptr())
        self._tb = tb
        self.build_occ_cache()

    def build_occ_cache(self) -> None:
        """Static canonical k-NN of the occupied cells (re-run when canon_bits change; the
        buffers hold every cell of the grid, so a refresh never reallocates them and views
        captured in CUDA graphs stay valid; the count lives on the device)."""
        cfg = self.cfg
        d = self.nodes.device
        if getattr(self, "occ_cells", None) is None:
            cap = cfg.canon_occ_res ** 3
            self.occ_cells = torch.empty(cap, dtype=torch.int32, device=d)
            self.occ_nbr = torch.empty((cap, cfg.ed_k), dtype=torch.int32, device=d)
            self.occ_w = torch.empty((cap, cfg.ed_k), dtype=torch.float64, device=d)
            self.occ_count = torch.zeros(1, dtype=torch.int32, device=d)
            self.occ_cap = cap
        cap = self.occ_cap
        _lib.call("cf_occ_cache", self.canon_bits.data_ptr(), _lib.byref(self.canon_occ), self.node_buckets.handle,
                  cfg.ed_k, cfg.ed_radius, cap, self.occ_cells.data_ptr(), self.occ_nbr.data_ptr(),
                  self.occ_w.data_ptr(), self.occ_count.data_ptr(), _lib.stream_ptr())

    def refresh_occupancy(self, W1: torch.Tensor, W2: torch.Tensor, dt: float) -> None:
        """Canonical density bits from the trained field (cf_density_grid_update): the
        E_g density at the canonical cell centres, max-decayed, thresholded at the
        density whose one-sample opacity is cfg.occ_alpha (sample spacing dt), dilated
        by the DeformNet offset bound (|dv| <= 0.05 m per axis: a sample's canonical
        point xu + dv is within that many cells of xu's cell), then the cached canonical
        k-NN of the occupied cells is rebuilt. Replaces the geometry shell."""
        _refresh_density(self, W1, W2, dt, int(np.ceil(0.05 / (self.side / self.cfg.canon_occ_res))),
                         self.canon_bits)
        self.build_occ_cache()

    def desc(self, dbias: torch.Tensor, precision: str | None = None) -> _lib.FieldDesc:
        precise = _precise(precision or self.cfg.precision)
        d = _lib.FieldDesc()
        d.has_deform = 1
        d.split_stages = int(not self.cfg.fuse_hash)
        d.dgrid = self.dgrid.desc
        d.dtable = (self.dgrid.table if precise else self.dgrid.table_for_kernels()).data_ptr()
        d.cgrid = self.cgrid.desc
        d.ctable = self.cgrid.table_for_kernels().data_ptr()
        d.wblob = self.nets.blob.data_ptr()
        d.wblob_lo = self.nets.blob_lo.data_ptr()
        d.precise = int(precise)
        d.w_bytes = self.nets.w_bytes
        d.dbias = dbias.data_ptr()
        d.delta_scale = 0.05
        d.inv_side = self.inv_side
        return d


class ObjectField:
    """Object-local rigid radiance field (static box geometry for its occupancy)."""

    def __init__(self, half_extents, cfg: RenderConfig | None = None, seed: int = 1, table_scale: float = 1e-4):
        self.cfg = cfg = cfg or RenderConfig()
        self.half = np.asarray(half_extents, dtype=np.float64)
        self.side = float(2 * self.half.max() + 2 * 0.05)
        self.obj_min = -np.full(3, self.side / 2)
        self.inv_side = 1.0 / self.side
        rng = np.random.default_rng(seed)
        self.cgrid = HashGrid(CANON_GRID, init_scale=table_scale, seed=seed + 11)
        self.nets = FieldNets(rng, deform=False)
        self.occ = occ_grid(self.obj_min, self.side, cfg.obj_occ_res)
        nwords = (cfg.obj_occ_res ** 3 + 31) // 32
        self.bits = torch.empty(nwords, dtype=torch.int32, device=self.cgrid.table.device)
        h = (ctypes.c_double * 3)(*self.half)
        _lib.call("cf_occ_box_shell", _lib.byref(self.occ), h, cfg.obj_shell, self.bits.data_ptr(), _lib.stream_ptr())

    def refresh_occupancy(self, W1: torch.Tensor, W2: torch.Tensor, dt: float) -> None:
        """Object density bits from the trained field (cf_density_grid_update, no dilation:
        the object field has no deformation). Replaces the box shell."""
        _refresh_density(self, W1, W2, dt, 0, self.bits)

    def desc(self, precision: str | None = None) -> _lib.FieldDesc:
        d = _lib.FieldDesc()
        d.has_deform = 0
        d.split_stages = int(not self.cfg.fuse_hash)
        d.cgrid = self.cgrid.desc
        d.ctable = self.cgrid.table_for_kernels().data_ptr()
        d.wblob = self.nets.blob.data_ptr()
        d.wblob_lo = self.nets.blob_lo.data_ptr()
        d.precise = int(_precise(precision or self.cfg.precision))
        d.w_bytes = self.nets.w_bytes
        d.delta_scale = 0.05
        d.inv_side = self.inv_side
        return d


_FRAME_DOUBLES = 28


def _sm_count(device) -> int:
    return torch.cuda.get_device_properties(device).multi_processor_count


class _FieldBuffers:
    def __init__(self, n_rays, capacity, device):
        self.records = torch.empty(capacity, dtype=torch.int32, device=device)
        self.ray_offset = torch.empty(n_rays, dtype=torch.int32, device=device)
        self.ray_count = torch.empty(n_rays, dtype=torch.int32, device=device)
        self.counters = torch.zeros(4, dtype=torch.int32, device=device)  # emitted, overflow, work ticket
        self.xu = torch.empty((capacity, 4), dtype=torch.float32, device=device)
        self.out = torch.empty((capacity, 4), dtype=torch.float32, device=device)
        self.rgb = torch.empty((n_rays, 3), dtype=torch.float32, device=device)
        self.depth = torch.empty(n_rays, dtype=torch.float32, device=device)
        self.opacity = torch.empty(n_rays, dtype=torch.float32, device=device)
        self.mo = _lib.MarchOut(self.records.data_ptr(), self.ray_offset.data_ptr(), self.ray_count.data_ptr(),
                                self.counters.data_ptr(), int(capacity))


def row_shard_rows(height: int, rank: int, world: int) -> range:
    """Image rows of rank `rank` when the rows of a frame are dealt round-robin."""
    return range(rank, height, world)


def assemble_row_shards(parts, width: int, height: int):
    """Interleave the ranks' row-shard images (rank r: rows r, r + world, ...) into
    the (height * width, C) frame."""
    world = len(parts)
    c = parts[0].shape[-1]
    full = parts[0].new_empty((height, width, c))
    for r, part in enumerate(parts):
        full[r::world] = part.reshape(-1, width, c)
    return full.reshape(height * width, c)


def gather_row_shards(part, width: int, height: int, group=None):
    """All-gather the ranks' row-shard images (NCCL on GPUs, gloo on CPU) and
    interleave them into the full (height * width, C) frame on every rank."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    c = part.shape[-1]
    rows_max = -(-height // world)
    buf = part.new_zeros((rows_max * width, c))
    buf[: part.shape[0]] = part
    got = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(got, buf, group=group)
    parts = [g[: len(row_shard_rows(height, r, world)) * width] for r, g in enumerate(got)]
    return assemble_row_shards(parts, width, height)


def _copy_list(pairs) -> None:
    """Device-to-device copies (src, dst) of contiguous tensors as one cf_copy_batch launch."""
    L = _lib.CopyList()
    for src, dst in pairs:
        L.src[L.n], L.dst[L.n] = src.data_ptr(), dst.data_ptr()
        L.bytes[L.n] = src.numel() * src.element_size()
        L.n += 1
    _lib.call("cf_copy_batch", _lib.byref(L), _lib.stream_ptr())


class Renderer:
    """render_view for one human + one rigid object."""

    def __init__(self, human: HumanField | None, obj: ObjectField | None, width: int, height: int,
                 cfg: RenderConfig | None = None, capacity_per_ray: int | None = None,
                 row_shard: tuple[int, int] | None = None):
        """row_shard = (rank, world): render only image rows rank, rank + world, ...
        (multi-GPU frames); `image` then holds those rows in order and
        assemble_row_shards() interleaves the ranks' parts back into the frame."""
        self.cfg = cfg = cfg or RenderConfig()
        self.human, self.obj = human, obj
        self.W, self.H = int(width), int(height)
        self.row0, self.row_stride = (0, 1) if row_shard is None else (int(row_shard[0]), int(row_shard[1]))
        if not (0 <= self.row0 < self.row_stride):
            raise ValueError("row_shard must be (rank, world) with 0 <= rank < world")
        self.rows = len(range(self.row0, self.H, self.row_stride))
        self.n_rays = self.W * self.rows
        d = _lib.require_cuda()
        cap = self.n_rays * int(capacity_per_ray or cfg.n_samples)
        self.dirs = torch.empty((self.n_rays, 3), dtype=torch.float64, device=d)
        self.hb = _FieldBuffers(self.n_rays, cap, d) if human else None
        self.ob = _FieldBuffers(self.n_rays, cap, d) if obj else None
        # two image buffers, alternated per view: a view's image can be read back
        # (render_to_host) while the next view renders into the other one
        self._images = [torch.empty((self.n_rays, 3), dtype=torch.float32, device=d) for _ in range(2)]
        self._img_slot = 0
        self.image = self._images[0]
        self._copy_stream = None
        self._host_images = [None, None]
        self._copy_done = [None, None]
        self._pending_rb = None
        self.layer = torch.empty(self.n_rays, dtype=torch.uint8, device=d)
        self.live_occ = occ_grid(cfg.world_min, cfg.world_size, cfg.live_occ_res)
        self.live_bits = torch.zeros((cfg.live_occ_res ** 3 + 31) // 32, dtype=torch.int32, device=d)
        self.bg = (ctypes.c_float * 3)(*cfg.background)
        self.M = _lib.MarchDesc()
        self.M.n_samples = cfg.n_samples
        self.M.t_near, self.M.t_far = cfg.t_near, cfg.t_far
        self.M.dt = (cfg.t_far - cfg.t_near) / cfg.n_samples
        self.M.human_grid = self.live_occ
        self.live_bbox = torch.zeros(6, dtype=torch.int32, device=d)
        P = cfg.live_occ_res + 2
        self.live_scratch = torch.zeros((P ** 3 + 31) // 32 + 3, dtype=torch.int32, device=d)
        self.M.human_cell_bbox = self.live_bbox.data_ptr()
        if obj:
            self.M.object_grid = obj.occ
            for a in range(3):
                self.M.obj_min[a] = obj.obj_min[a]
            self.M.obj_inv_side = obj.inv_side
        self.frame = None
        self.marks = None
        # side stream: the per-frame LBS chain and the object field run next to the
        # human chain (stream priorities and a later object fork were measured: no gain)
        self.side = torch.cuda.Stream(device=d)
        self._lbs_done = torch.cuda.Event()
        self._ed_done = torch.cuda.Event()
        self.side_ed = torch.cuda.Stream(device=d)
        self._obj_done = torch.cuda.Event()
        self._lbs_done.record(torch.cuda.current_stream())
        self._ed_done.record(torch.cuda.current_stream())
        # frame block: origin[3], obj_R[9], obj_t[3] | camera R[9], fx, fy, cx, cy
        self.frame_dev = torch.zeros(_FRAME_DOUBLES, dtype=torch.float64, device=d)
        self._frame_host = np.zeros(_FRAME_DOUBLES)
        self._staging = [torch.zeros(_FRAME_DOUBLES, dtype=torch.float64).pin_memory() for _ in range(4)]
        self._staging_ev = [None] * len(self._staging)
        self._slot = 0
        self.M.frame = self.frame_dev.data_ptr()
        self.cam = _lib.Camera()
        self.cam.width, self.cam.height = self.W, self.rows
        self.cam.row0, self.cam.row_stride = self.row0, self.row_stride
        self.cam.params = self.frame_dev.data_ptr() + 15 * 8
        self._setup_pending = False   # per-frame human setup still to run (load_prior since the last view)
        self._graphs = {}             # (with_setup,) -> torch.cuda.CUDAGraph

    # -- per-frame setup ------------------------------------------------------

    def set_frame(self, node_dqs=None, theta=None, bone_A=None, obj_R=None, obj_t=None):
        """Register the frame's motion prior: ED node dqs, SMPL-style pose (theta, bone
        transforms) and the object pose (object-to-world)."""
        if self.human is not None:
            h = self.human
            self.load_prior(dev(node_dqs, shape_last=8), dev(np.asarray(bone_A, dtype=np.float64)),
                            dev(h.nets.theta_bias(theta), dtype=torch.float32))
        if self.obj is not None:
            self.set_object_pose(obj_R, obj_t)

    def load_pose(self, dqs: torch.Tensor, theta: torch.Tensor) -> None:
        """Per-frame human prior as the tracker emits it (a CFMP record, records.py:98-126):
        node dqs (n,8) f64 and pose theta (72,) f64, device or pinned host tensors. The
        frame's setup runs the forward kinematics (cf_skinning_transforms, skeleton.py:
        121-139) and the DeformNet pose bias (cf_pose_bias) on the device, then the warp
        setup — no host FK, no host matvec."""
        self._prior_buffers()
        if getattr(self, "_theta", None) is None:
            self._theta = torch.empty(self.human.lbs.J * 3, dtype=torch.float64, device=self.dirs.device)
            from .records import _rig_arrays
            self._rig = _rig_arrays(None)
        self._defer_copy(self._dqs, dqs)
        self._defer_copy(self._theta, theta)
        self._pose_on_device = True
        self._setup_pending = True

    def _prior_buffers(self) -> None:
        h = self.human
        if getattr(self, "_dqs", None) is None:
            n = len(h.graph.nodes)
            self._dqs = torch.empty((n, 8), dtype=torch.float64, device=self.dirs.device)
            self._anchors = torch.empty((n, 3), dtype=torch.float64, device=self.dirs.device)
            self._A = torch.empty((h.lbs.J, 4, 4), dtype=torch.float64, device=self.dirs.device)
            self.dbias = torch.empty(128, dtype=torch.float32, device=self.dirs.device)
            self._anchor_buckets = Buckets(n)
        if getattr(self, "hw", None) is None:
            w = _lib.HumanWarp()
            w.dqs = self._dqs.data_ptr()
            w.k = self.cfg.ed_k
            w.r2 = self.cfg.ed_radius ** 2
            w.vert_Tinv = h.lbs.Tinv.data_ptr()
            w.lbs_max_d2 = self.cfg.lbs_max_dist ** 2
            for a in range(3):
                w.canon_min[a] = h.canon_min[a]
            w.inv_side = h.inv_side
            w.anchors = self._anchors.data_ptr()
            w.n_nodes = int(self._anchors.shape[0])
            if w.n_nodes <= 1024:  # the frame's anchor block for the culled k-NN (cf_deform_nodes_block)
                nb = ctypes.c_int64()
                _lib.call("cf_anchor_block_bytes", w.n_nodes, ctypes.byref(nb))
                self._anchor_block = torch.empty(int(nb.value), dtype=torch.uint8, device=self.dirs.device)
                w.anchor_block = self._anchor_block.data_ptr()
                if self.cfg.cand_grid_res > 0:  # the per-frame candidate grid of the k-NN
                    _lib.call("cf_cand_grid_bytes", self.cfg.cand_grid_res, self.cfg.cand_grid_cmax,
                              ctypes.byref(nb))
                    self._cand_grid = torch.empty(int(nb.value), dtype=torch.uint8, device=self.dirs.device)
                    w.cand_grid = self._cand_grid.data_ptr()
            self.hw = w
            self.hdesc = h.desc(self.dbias, self.cfg.precision)

    def load_prior(self, dqs: torch.Tensor, bone_A: torch.Tensor, dbias: torch.Tensor) -> None:
        """Per-frame human prior from device-resident tensors (no host sync): node
        dqs (n,8) f64, bone transforms (J,4,4) f64, DeformNet pose bias (128,) f32.
        Staged into the renderer's fixed buffers; the setup kernels run with the
        next view (inside its graph)."""
        self._prior_buffers()
        self._pose_on_device = False
        # enqueued with the next view's frame block as one batched copy (sources must
        # stay valid until that view, or prepare_frame, is issued)
        for dst, src in ((self._dqs, dqs), (self._A, bone_A), (self.dbias, dbias)):
            self._defer_copy(dst, src)
        self._setup_pending = True

    def _human_setup(self, lbs_buckets: bool = True) -> None:
        """The frame's human setup kernels: backward-LBS chain on the side stream,
        deformed nodes + live occupancy splat on the current stream. lbs_buckets=False
        (the view): no posed-vertex buckets — the view's fallback pass scans the
        posed vertices; prepare_frame adds the buckets for the fused callers."""
        self._flush_copies()
        s = _lib.stream_ptr()
        h = self.human
        n = self._dqs.shape[0]
        # the backward-LBS chain (FK of theta, vertex transforms, posed vertices, their
        # buckets) is independent of the ED chain: run it on the side stream (and the
        # pose bias and the deformed nodes, which only the canonicalisation and the
        # field read, after the same event)
        main = torch.cuda.current_stream()
        side = self._side_stream()
        self._fork(main, side)
        with torch.cuda.stream(side):
            ss = _lib.stream_ptr()
            if getattr(self, "_pose_on_device", False):  # FK + pose bias of the frame's theta
                parents, offsets = self._rig
                _lib.call("cf_skinning_transforms", self._theta.data_ptr(), 1, parents.ctypes.data,
                          offsets.ctypes.data, len(parents), self._A.data_ptr(), ss)
                _lib.call("cf_pose_bias", h.nets.d1.data_ptr(), 32 + 3 * len(parents), 32, 128,
                          self._theta.data_ptr(), 3 * len(parents), self.dbias.data_ptr(), ss)
            h.lbs.set_pose(self._A, buckets=lbs_buckets)
            self._lbs_buckets_current = lbs_buckets
            self._mark("lbs_setup")
            self._lbs_done.record(side)
        # the ED chain (deformed nodes, their anchor block and candidate grid, or buckets)
        # on a third stream, next to the LBS chain and the main stream's occupancy + march
        ed = self._ed_stream()
        self._fork(main, ed)
        with torch.cuda.stream(ed):
            es = _lib.stream_ptr()
            if n <= 1024:
                _lib.call("cf_deform_nodes_block", h.nodes.data_ptr(), self._dqs.data_ptr(), n,
                          self._anchors.data_ptr(), self._anchor_block.data_ptr(), es)
                if getattr(self, "_cand_grid", None) is not None:
                    _lib.call("cf_cand_grid_build", self._anchor_block.data_ptr(), n, self.cfg.ed_k,
                              self.cfg.ed_radius, self.cfg.cand_grid_res, self.cfg.cand_grid_cmax,
                              self._cand_grid.data_ptr(), es)
            else:
                _lib.call("cf_deform_nodes", h.nodes.data_ptr(), self._dqs.data_ptr(), n, self._anchors.data_ptr(), es)
                self._anchor_buckets.build(self._anchors)
            self._mark("ed_warp_setup")
            self._ed_done.record(ed)
        _lib.call("cf_occ_splat_cached", h.occ_cells.data_ptr(), h.occ_nbr.data_ptr(), h.occ_w.data_ptr(),
                  h.occ_count.data_ptr(), h.occ_cap, self.cfg.ed_k, self._dqs.data_ptr(), _lib.byref(h.canon_occ),
                  _lib.byref(self.live_occ), self.live_scratch.data_ptr(), self.live_bits.data_ptr(),
                  self.live_bbox.data_ptr(), s)
        self._mark("ed_setup")

    def _save_frame_state(self):
        """Snapshot of the per-frame state another user of the warp buffers (the
        trainer's key frames) overwrites: the prior buffers (one batched device copy
        into buffers kept for this) and the pose flag."""
        if self.human is None or getattr(self, "_dqs", None) is None:
            return None
        self._flush_copies()  # a prior staged but not yet issued belongs to the snapshot
        bufs = [self._dqs, self._A, self.dbias] + ([self._theta] if getattr(self, "_theta", None) is not None else [])
        snap = getattr(self, "_snap", None)
        if snap is None or len(snap) != len(bufs):
            snap = self._snap = [torch.empty_like(b) for b in bufs]
        _copy_list(list(zip(bufs, snap)))
        return (list(zip(snap, bufs)), getattr(self, "_pose_on_device", False))

    def _restore_frame_state(self, saved) -> None:
        """Restore a _save_frame_state snapshot (one batched device copy); the frame's
        setup (deformed nodes, LBS, live occupancy) re-runs with the next view."""
        if saved is None:
            return
        pairs, pose_on_device = saved
        _copy_list(pairs)
        self._pose_on_device = pose_on_device
        self._setup_pending = True

    def set_object_pose(self, obj_R, obj_t) -> None:
        """Object-to-world pose of the frame (frame block, uploaded with the next view)."""
        self._frame_host[3:12] = np.asarray(obj_R, dtype=np.float64).reshape(9)
        self._frame_host[12:15] = np.asarray(obj_t, dtype=np.float64).reshape(3)
        if getattr(self, "odesc", None) is None:
            self.odesc = self.obj.desc(self.cfg.precision)

    # -- per-view --------------------------------------------------------------

    def rays(self, R, t, fx, fy, cx, cy):
        """Camera of the view (frame block) and its ray directions."""
        self._set_camera(R, t, fx, fy, cx, cy)
        self._upload_frame()
        self._flush_copies()
        self._rays()

    def _set_camera(self, R, t, fx, fy, cx, cy):
        self._frame_host[0:3] = np.asarray(t, dtype=np.float64).reshape(3)
        self._frame_host[15:24] = np.asarray(R, dtype=np.float64).reshape(9)
        self._frame_host[24:28] = (float(fx), float(fy), float(cx), float(cy))

    def _upload_frame(self):
        """Frame block -> device through a ring of pinned staging slots (a slot is
        reused only after its previous copy completed)."""
        i = self._slot
        self._slot = (i + 1) % len(self._staging)
        if self._staging_ev[i] is not None:
            self._staging_ev[i].synchronize()
        buf = self._staging[i]
        buf.numpy()[:] = self._frame_host
        self._defer_copy(self.frame_dev, buf, staging_slot=i)

    def _defer_copy(self, dst: torch.Tensor, src: torch.Tensor, staging_slot: int | None = None) -> None:
        if not hasattr(self, "_pending_copies"):
            self._pending_copies = {}
        self._pending_copies[dst.data_ptr()] = (dst, src, staging_slot)

    def _flush_copies(self) -> None:
        """Issue the deferred small copies (prior + frame block) as ONE kernel launch
        on the current stream; sources that cannot be read by the device (pageable
        host memory, dtype / size mismatch) fall back to a stream-ordered copy_."""
        pend = getattr(self, "_pending_copies", None)
        if not pend:
            return
        L = _lib.CopyList()
        rest = []
        slots = []
        for dst, src, slot in pend.values():
            ok = (src.dtype == dst.dtype and src.numel() == dst.numel() and src.is_contiguous()
                  and dst.is_contiguous() and (src.is_cuda or src.is_pinned()) and L.n < 8)
            if ok:
                L.src[L.n], L.dst[L.n] = src.data_ptr(), dst.data_ptr()
                L.bytes[L.n] = src.numel() * src.element_size()
                L.n += 1
            else:
                rest.append((dst, src))
            if slot is not None:
                slots.append(slot)
        _lib.call("cf_copy_batch", _lib.byref(L), _lib.stream_ptr())
        for dst, src in rest:
            dst.copy_(src, non_blocking=True)
        if slots:
            ev = torch.cuda.Event()
            ev.record()
            for i in slots:
                self._staging_ev[i] = ev
        pend.clear()

    def _rays(self):
        _lib.call("cf_camera_rays", _lib.byref(self.cam), self.dirs.data_ptr(), _lib.stream_ptr())
        self.M.n_rays = self.n_rays

    def _scratch(self, buf, desc) -> torch.Tensor:
        """Per-field scratch of cf_field_forward (allocated once)."""
        if getattr(buf, "scratch", None) is None:
            # sized for the larger ("fp32") layout: a view may switch precision
            # (set_precision) while graphs captured earlier keep pointing here
            d = _lib.FieldDesc()
            ctypes.memmove(ctypes.byref(d), ctypes.byref(desc), ctypes.sizeof(d))
            d.precise = 1
            nb = ctypes.c_int64()
            _lib.call("cf_field_scratch_bytes", _lib.byref(d), int(buf.mo.capacity), ctypes.byref(nb))
            buf.scratch = torch.empty(max(int(nb.value), 16), dtype=torch.uint8, device=self.dirs.device)
        return buf.scratch

    def _mark(self, name):
        """Timing event after a stage, on the stream it ran on: marks hold
        (stream id, name, event); a stage's time is the gap to the previous mark
        of the same stream."""
        if self.marks is not None:
            # inside a graph capture: an external event, recorded by every replay
            e = torch.cuda.Event(enable_timing=True, external=getattr(self, "_capturing", False))
            st = torch.cuda.current_stream()
            e.record(st)
            self.marks.append((st.cuda_stream, name, e))

    def _ed_stream(self) -> torch.cuda.Stream:
        """The stream of the per-frame ED chain (or the caller's, in serial mode)."""
        return torch.cuda.current_stream() if self.cfg.serial else self.side_ed

    def _side_stream(self) -> torch.cuda.Stream:
        """The stream of the LBS chain and the object field: a second stream, or the
        caller's stream in serial mode (cfg.serial)."""
        return torch.cuda.current_stream() if self.cfg.serial else self.side

    def set_precision(self, precision: str) -> None:
        """Switch the field arithmetic ("fp32" / "fp16") of the following views."""
        _precise(precision)
        self.cfg.precision = precision
        if getattr(self, "hdesc", None) is not None:
            self.hdesc = self.human.desc(self.dbias, precision)
        if getattr(self, "odesc", None) is not None:
            self.odesc = self.obj.desc(precision)

    @staticmethod
    def _fork(src: torch.cuda.Stream, dst: torch.cuda.Stream) -> None:
        ev = torch.cuda.Event()
        ev.record(src)
        dst.wait_event(ev)

    def render_to_host(self, R, t, fx, fy, cx, cy):
        """render() and read the image back into pinned host memory without
        blocking: returns (handle, host image); the image is valid once
        handle.synchronize() returned (or handle.query() is True).

        The device-to-host copy runs on a copy stream. It is issued when the NEXT
        view has enqueued its uploads (or when the handle is waited on), so the
        read-back overlaps that view's kernels but never the host link traffic of
        its inputs (uploads queued behind a 3 MB read-back delayed every frame)."""
        img = self.render(R, t, fx, fy, cx, cy)
        slot = self._img_slot ^ 1  # the buffer render() just used
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(device=self.dirs.device)
        if self._host_images[slot] is None:
            self._host_images[slot] = torch.empty(img.shape, dtype=img.dtype).pin_memory()
        ready = torch.cuda.Event()
        ready.record()
        rb = _ReadBack(self, slot, img, ready)
        self._pending_rb = rb
        return rb, self._host_images[slot]  # reused two views later

    def _issue_readback(self, rb, after=None) -> None:
        """Enqueue rb's copy on the copy stream after `after` (an event on the
        current stream), or after the view's own completion event."""
        self._copy_stream.wait_event(after if after is not None else rb.ready)
        with torch.cuda.stream(self._copy_stream):
            self._host_images[rb.slot].copy_(rb.img, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._copy_stream)
        rb.event = ev
        self._copy_done[rb.slot] = ev
        if self._pending_rb is rb:
            self._pending_rb = None

    def prepare_frame(self) -> None:
        """Run the pending per-frame human setup now (eager launches) — for callers
        that use the frame's warp state without rendering a view (training)."""
        if self._setup_pending and self.human is not None:
            self._human_setup()
            # the side-stream LBS and ED chains are done before the caller's next launch
            torch.cuda.current_stream().wait_event(self._lbs_done)
            torch.cuda.current_stream().wait_event(self._ed_done)
        elif self.human is not None and not getattr(self, "_lbs_buckets_current", True):
            # the frame's setup ran with a view (no vertex buckets): add them now
            self.human.lbs.build_buckets()
            self._lbs_buckets_current = True
        self._setup_pending = False

    def render(self, R, t, fx, fy, cx, cy):
        """All stages of one novel view; returns the composited image tensor (H*W, 3).
        Replays the captured graph of the view (cfg.cuda_graphs). If `self.marks` is
        a list, it is replaced by [(stream, name, event)] for "start" and each stage
        (read them after synchronizing, before the next view)."""
        self._set_camera(R, t, fx, fy, cx, cy)
        self._upload_frame()
        self._flush_copies()
        if getattr(self, "_pending_rb", None) is not None:
            # the previous view's read-back starts once this view's uploads are done
            after = torch.cuda.Event()
            after.record()
            self._issue_readback(self._pending_rb, after)
        setup = self._setup_pending and self.human is not None
        self._setup_pending = False
        timed = self.marks is not None
        slot = self._img_slot
        self._img_slot ^= 1
        self.image = self._images[slot]
        if self._copy_done[slot] is not None:  # this buffer's previous read-back must be done
            torch.cuda.current_stream().wait_event(self._copy_done[slot])
        key = (setup, timed, slot, self.cfg.serial, self.cfg.precision)
        if not self.cfg.cuda_graphs or (key not in self._graphs and not getattr(self, "_eager_done", False)):
            # eager launches (also the first view: lazily allocated state must exist before capture)
            if timed:
                self.marks = []
                self._mark("start")
            self._launch_view(setup)
            self._eager_done = True
            return self.image
        if key not in self._graphs:
            g = torch.cuda.CUDAGraph()
            main = torch.cuda.current_stream()
            cap = torch.cuda.Stream(device=self.dirs.device)
            self._fork(main, cap)
            self._capturing = True
            try:
                with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                    if timed:
                        self.marks = []
                        self._mark("start")
                    self._launch_view(setup)
            finally:
                self._capturing = False
            main.wait_stream(cap)
            self._graphs[key] = (g, self.marks if timed else None)
        g, marks = self._graphs[key]
        g.replay()
        if timed:
            self.marks = marks
        return self.image

    def _launch_view(self, setup: bool):
        s = _lib.stream_ptr()
        if setup:
            self._human_setup(lbs_buckets=False)
        hb, ob = self.hb, self.ob
        # ray generation fused into the march (directions written for the later stages)
        self.M.n_rays = self.n_rays
        _lib.call("cf_rays_march", _lib.byref(self.cam), _lib.byref(self.M), self.dirs.data_ptr(),
                  self.live_bits.data_ptr() if hb else None, self.obj.bits.data_ptr() if ob else None,
                  _lib.byref(hb.mo) if hb else None, _lib.byref(ob.mo) if ob else None, s)
        self._mark("march")
        main = torch.cuda.current_stream()

        def object_field():
            # the object field is independent of the human one: side stream (running it
            # serially on the main stream measured 330 -> 355 us per frame)
            side = self._side_stream()
            self._fork(main, side)
            with torch.cuda.stream(side):
                so = _lib.stream_ptr()
                _lib.call("cf_object_canon", _lib.byref(self.M), self.dirs.data_ptr(), _lib.byref(ob.mo),
                          ob.xu.data_ptr(), so)
                self._mark("object_canon")
                # beside the human chain the object field keeps to an eighth of the SMs, leaving
                # the rest to the DeformNet kernel that starts while it runs (0.353 -> 0.348 ms
                # per frame; 8 CTAs made it the critical path); serialised: the whole GPU
                self.odesc.max_ctas = 0 if self.cfg.serial else max(16, _sm_count(self.dirs.device) // 8)
                _lib.call("cf_field_forward", _lib.byref(self.odesc), _lib.byref(ob.mo), self.dirs.data_ptr(),
                          ob.xu.data_ptr(), ob.out.data_ptr(), self._scratch(ob, self.odesc).data_ptr(), so)
                self._mark("object_field")
                _lib.call("cf_composite", _lib.byref(self.M), _lib.byref(ob.mo), ob.out.data_ptr(),
                          self.cfg.t_term, ob.rgb.data_ptr(), ob.depth.data_ptr(), ob.opacity.data_ptr(), so)
                self._mark("object_composite")
                self._obj_done.record(side)

        if ob:
            object_field()
        if hb:
            h = self.human
            # the canonicalisation needs the ED chain; the backward-LBS fallback (posed
            # vertices + buckets from the side stream's LBS chain) runs as its own pass
            # after it, so the LBS chain overlaps the march and the ED canonicalisation
            if setup:
                main.wait_event(self._ed_done)
            _lib.call("cf_human_canon", _lib.byref(self.M), self.dirs.data_ptr(), _lib.byref(hb.mo),
                      _lib.byref(self.hw), self._anchor_buckets.handle, None, hb.xu.data_ptr(), s)
            if setup:
                main.wait_event(self._lbs_done)
            _lib.call("cf_human_lbs_fallback", _lib.byref(self.M), self.dirs.data_ptr(), _lib.byref(hb.mo),
                      _lib.byref(self.hw), h.lbs.posed.data_ptr(), h.lbs.V, h.lbs.box.data_ptr(),
                      hb.xu.data_ptr(), s)
            self._mark("human_canon")
            scratch = self._scratch(hb, self.hdesc).data_ptr()
            fused = self.hdesc.precise and not self.hdesc.split_stages  # stages 0 / 2 run inside 1 / 3
            for stage, name in enumerate(("human_hash_d", "human_deform_mlp", "human_hash_c", "human_color_mlp")):
                if stage in (0, 2) and fused:
                    continue
                _lib.call("cf_field_stage", _lib.byref(self.hdesc), _lib.byref(hb.mo), self.dirs.data_ptr(),
                          hb.xu.data_ptr(), hb.out.data_ptr(), scratch, stage, s)
                self._mark(name)
            if ob:
                main.wait_event(self._obj_done)
            # human composite fused with the layer choice against the object layer
            _lib.call("cf_composite_final", _lib.byref(self.M), _lib.byref(hb.mo), hb.out.data_ptr(),
                      self.cfg.t_term, hb.rgb.data_ptr(), hb.depth.data_ptr(), hb.opacity.data_ptr(),
                      ob.rgb.data_ptr() if ob else None, ob.depth.data_ptr() if ob else None,
                      ob.opacity.data_ptr() if ob else None, self.bg, self.image.data_ptr(), self.layer.data_ptr(), s)
            self._mark("human_composite")
        else:
            if ob:
                main.wait_event(self._obj_done)
            _lib.call("cf_composite_layers", self.n_rays, None, None, None, ob.rgb.data_ptr() if ob else None,
                      ob.depth.data_ptr() if ob else None, ob.opacity.data_ptr() if ob else None, self.bg,
                      self.image.data_ptr(), self.layer.data_ptr(), s)
            self._mark("layers")

    def sample_counts(self):
        """(human, object) processed-sample counts of the last view (syncs)."""
        h = int(self.hb.counters[0]) if self.hb else 0
        o = int(self.ob.counters[0]) if self.ob else 0
        return h, o

    def check_overflow(self):
        for b in (self.hb, self.ob):
            if b is not None and int(b.counters[1]) != 0:
                raise RuntimeError("sample buffer overflow: raise capacity_per_ray")
