"""Motion-prior ingestion: the native CFMP codec against a stream
written by the reference's own MotionPriorWriter (tests/golden/make_records.py,
records.py:103-147; the reference round-trip test is tests/test_io.py:124-151),
its error behaviour, and the device forward kinematics against the reference's
skinning_transforms (skeleton.py:135-139).

The codec is host code in the C-ABI library: the CPU tests call it without a GPU.
"""
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal

from paper_2304_03184_b200 import records, scene
from paper_2304_03184_b200.errors import RecordFormatError

BIN = os.path.join(GOLDEN, "motions_ref.bin")


@pytest.fixture(scope="module")
def ref():
    with np.load(os.path.join(GOLDEN, "motions_ref.npz")) as z:
        return {k: z[k] for k in z.files}


def test_rig_matches_reference(ref):
    assert np.array_equal(ref["parents"], scene.PARENTS)
    assert bits_equal(ref["offsets"], scene.OFFSETS)


def test_scan_and_read_bit_exact(ref):
    info = records.scan_motion_priors(BIN)
    assert (info.n_frames, info.n_nodes, info.n_theta, info.bytes) == (6, 5, 72, os.path.getsize(BIN))
    fids, dqs, theta, rot, trans = records.read_motion_arrays(BIN)
    assert np.array_equal(fids, ref["frame_ids"])
    for a, k in ((dqs, "dqs"), (theta, "theta"), (rot, "rot"), (trans, "trans")):
        assert bits_equal(a, ref[k]), k
    # a sub-range decodes the same rows
    f2, d2, t2, r2, tr2 = records.read_motion_arrays(BIN, first=2, count=3)
    assert np.array_equal(f2, ref["frame_ids"][2:5]) and bits_equal(d2, ref["dqs"][2:5])
    assert bits_equal(t2, ref["theta"][2:5]) and bits_equal(r2, ref["rot"][2:5]) and bits_equal(tr2, ref["trans"][2:5])


def test_load_motion_priors(ref):
    back = records.load_motion_priors(BIN)
    assert len(back) == 6
    for i, p in enumerate(back):
        assert p.frame_id == ref["frame_ids"][i] == p.graph_motion.frame_id
        assert bits_equal(p.graph_motion.dqs, ref["dqs"][i])
        assert bits_equal(p.pose.theta, ref["theta"][i])
        assert bits_equal(p.object_pose.rotation, ref["rot"][i])
        assert bits_equal(p.object_pose.translation, ref["trans"][i])


def test_writer_byte_identical(tmp_path, ref):
    """Our writer re-encodes the reference's stream byte for byte (one frame at a
    time, as MotionPriorWriter.append, and batched)."""
    priors = records.load_motion_priors(BIN)
    p1 = str(tmp_path / "a.bin")
    with records.MotionPriorWriter(p1, n_nodes=5, n_theta=72) as wr:
        for p in priors:
            wr.append(p)
    p2 = str(tmp_path / "b.bin")
    records.MotionPriorWriter(p2, 5, 72).append_batch(priors)
    gold = open(BIN, "rb").read()
    assert open(p1, "rb").read() == gold
    assert open(p2, "rb").read() == gold


def test_empty_stream(tmp_path):
    p = str(tmp_path / "e.bin")
    records.MotionPriorWriter(p, 3, 72)
    assert records.scan_motion_priors(p).n_frames == 0
    assert records.load_motion_priors(p) == []


def test_frame_id_mismatch_rejected():
    from paper_2304_03184_b200.edgraph import GraphMotion
    with pytest.raises(ValueError):
        records.MotionPrior(1, GraphMotion.identity(0, 3), records.SkeletonPose(None), records.Se3())


def _corrupt(tmp_path, data: bytes) -> str:
    p = str(tmp_path / "bad.bin")
    with open(p, "wb") as f:
        f.write(data)
    return p


def test_format_errors(tmp_path):
    gold = open(BIN, "rb").read()
    cases = {
        "magic": b"CFGR" + gold[4:],
        "version": gold[:4] + struct.pack("<I", 2) + gold[8:],
        "truncated header": gold[:10],
        "truncated payload": gold[:-5],
        "partial frame id": gold + b"\x01\x02\x03",
        "array length": gold[:16 + 8] + struct.pack("<I", 39) + gold[16 + 12:],
    }
    for what, data in cases.items():
        with pytest.raises(RecordFormatError):
            records.load_motion_priors(_corrupt(tmp_path, data))
        assert issubclass(RecordFormatError, ValueError), what


def test_append_shape_checked(tmp_path):
    priors = records.load_motion_priors(BIN)
    w = records.MotionPriorWriter(str(tmp_path / "t.bin"), 4, 72)
    with pytest.raises(ValueError):
        w.append(priors[0])  # 5-node prior into a 4-node stream
    p = str(tmp_path / "s.bin")
    records.MotionPriorWriter(p, 5, 72).append(priors[0])
    with pytest.raises(ValueError):
        records.read_motion_arrays(p, first=0, count=5)  # range beyond the stream


@pytest.mark.gpu
def test_device_fk_vs_reference(ref):
    """One launch for all frames; 1e-12 against the reference's skinning_transforms
    (numpy/BLAS summation order and libm sin/cos differ from the device's by ulps)."""
    import torch
    th = torch.from_numpy(ref["theta"]).cuda()
    A = records.skinning_transforms(th).cpu().numpy()
    assert A.shape == ref["bone_A"].shape
    assert np.abs(A - ref["bone_A"]).max() <= 1e-12
    assert np.array_equal(A[:, :, 3], ref["bone_A"][:, :, 3])


@pytest.mark.gpu
def test_device_fk_many_frames_vs_oracle():
    """Batched over 1,000 random poses (the oracle restatement of the same FK)."""
    import torch
    from oracle import deform as od
    rng = np.random.default_rng(3)
    theta = rng.normal(size=(1000, 72)) * rng.uniform(0.0, 2.0, size=(1000, 1))
    theta[::17] = 0.0
    A = records.skinning_transforms(torch.from_numpy(theta).cuda()).cpu().numpy()
    for f in range(0, 1000, 37):
        ref = od.bone_transforms(scene.PARENTS, scene.OFFSETS, theta[f])
        assert np.abs(A[f] - ref).max() <= 1e-12, f


@pytest.mark.gpu
def test_stream_resident_lut(ref):
    import torch
    st = records.MotionPriorStream(BIN)
    assert len(st) == 6 and np.array_equal(st.frame_ids, ref["frame_ids"])
    assert bits_equal(st.dqs.cpu().numpy(), ref["dqs"])
    assert bits_equal(st.lookup_table.cpu().numpy(), ref["dqs"].reshape(-1, 8))
    assert np.abs(st.bone_A.cpu().numpy() - ref["bone_A"]).max() <= 1e-12
    assert bits_equal(st.graph_motion(42).dqs, ref["dqs"][5])
    with pytest.raises(KeyError):
        st.slot(5)
    assert st.dqs.device.type == "cuda" and st.bone_A.dtype == torch.float64


@pytest.mark.gpu
def test_stream_drives_the_renderer(tmp_path):
    """A scene's priors written as a CFMP stream, resident in HBM, render the same
    frame as the host-side prior path (device FK vs host FK differ by ulps)."""
    import torch
    from paper_2304_03184_b200.render import HumanField, ObjectField, RenderConfig, Renderer
    from paper_2304_03184_b200.scene import Scene, SceneConfig
    sc = Scene(SceneConfig(width=64, height=64), seed=0)
    cfg = RenderConfig(n_samples=64)
    hf = HumanField(sc.nodes, sc.template_points, sc.skin_verts, sc.skin_weights, cfg, seed=0, zero_deform_out=False,
                    table_scale=0.5)
    of = ObjectField(sc.box_half, cfg, seed=1, table_scale=0.5)
    path = str(tmp_path / "scene.bin")
    with records.MotionPriorWriter(path, len(sc.nodes), 72) as wr:
        for fid in range(sc.cfg.frames):
            R, t = sc.object_pose(fid)
            wr.append(records.MotionPrior(fid, records.GraphMotion(fid, sc.node_dqs(fid)),
                                          records.SkeletonPose(None, sc.theta(fid)), records.Se3(R, t)))
    st = records.MotionPriorStream(path)
    fid = 7
    assert np.abs(st.bone_A[fid].cpu().numpy() - sc.bone_transforms(fid)).max() <= 1e-12
    cam = sc.camera
    r = Renderer(hf, of, 64, 64, cfg)
    R, t = sc.object_pose(fid)
    r.set_frame(sc.node_dqs(fid), sc.theta(fid), sc.bone_transforms(fid), R, t)
    a = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy).clone()
    st.load_into(r, fid)
    b = r.render(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy).clone()
    torch.cuda.synchronize()
    d = (a - b).abs()
    assert a.abs().sum() > 0
    assert float(d.max()) <= 1e-2 and float(d.mean()) <= 1e-5, (float(d.max()), float(d.mean()))
