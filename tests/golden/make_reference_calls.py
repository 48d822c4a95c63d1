"""Record every hot-path call the REFERENCE'S OWN TESTS make, with the reference's
answer (test infrastructure; run here, where /root/reference exists):

    python tests/golden/make_reference_calls.py

It runs the reference test modules tests/test_transforms.py, test_edgraph.py,
test_knnfield.py and test_skeleton.py (/root/reference/pkg/tests) in-process with
the reference's drop-in surface wrapped by a recorder: dq_blend, dq_apply
(transforms.py:174-196), deformed_nodes, warp_backward_batch, warp_forward_batch
(edgraph.py:134-183), brute_force_query (knnfield.py:32-42), KnnField and its
update_live_map / query_motion_batch / query_motion (knnfield.py:45-229) and
lbs_batch (skeleton.py:142-149). Each top-level call (calls the reference makes
internally are not recorded) is stored with its inputs and either its outputs or
the exception class it raised. tests/test_reference_calls_gpu.py replays them through
this package's GPU implementation on the B200 (where /root/reference does not exist).
The reference's tests themselves must pass while recording (the script checks).
"""
from __future__ import annotations

import gzip
import os
import pickle
import sys

import numpy as np

REF = "/root/reference/pkg"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_calls.pkl.gz")


def main():
    sys.path.insert(0, os.path.join(REF, "src"))
    import pytest

    import capfields.edgraph as E
    import capfields.knnfield as K
    import capfields.skeleton as S
    import capfields.transforms as T

    calls = []
    depth = [0]
    fields = {}

    def conv(x):
        if isinstance(x, E.EDGraph):
            return {"__graph__": True, "nodes": np.array(x.nodes), "radius": float(x.radius), "knn_k": int(x.knn_k)}
        if isinstance(x, E.GraphMotion):
            return {"__motion__": True, "frame_id": int(x.frame_id), "dqs": np.array(x.dqs)}
        if isinstance(x, S.Skeleton):
            return {"__skel__": True, "parents": np.array(x.parents), "offsets": np.array(x.offsets)}
        if isinstance(x, K.KnnField):
            return {"__field__": fields[id(x)]}
        if isinstance(x, np.ndarray):
            return np.array(x)
        if isinstance(x, (list, tuple)):
            return type(x)(conv(v) for v in x)
        return x

    def wrap(name, fn, method=False):
        def w(*a, **kw):
            top = depth[0] == 0
            depth[0] += 1
            entry = {"fn": name, "args": conv(a), "kw": conv(kw)} if top else None
            try:
                out = fn(*a, **kw)
                if top:
                    if name == "KnnField":
                        pass  # outputs recorded below from the instance
                    else:
                        entry["out"] = conv(out)
                return out
            except Exception as e:  # noqa: BLE001
                if top:
                    entry["exc"] = type(e).__name__
                raise
            finally:
                depth[0] -= 1
                if top:
                    calls.append(entry)
        return w

    # free functions (the test modules import them by name after this patching)
    for mod, names in ((T, ["dq_blend", "dq_apply"]),
                       (E, ["deformed_nodes", "warp_backward_batch", "warp_forward_batch"]),
                       (K, ["brute_force_query"]), (S, ["lbs_batch"])):
        for n in names:
            setattr(mod, n, wrap(f"{mod.__name__.split('.')[-1]}.{n}", getattr(mod, n)))
    # KnnField: construction, live-map updates and queries, tied to an instance id
    init0, upd0, qb0, q0 = K.KnnField.__init__, K.KnnField.update_live_map, K.KnnField.query_motion_batch, \
        K.KnnField.query_motion

    def init(self, *a, **kw):
        top = depth[0] == 0
        fid = len(fields)
        entry = {"fn": "KnnField", "field": fid, "args": conv(a), "kw": conv(kw)} if top else None
        depth[0] += 1
        try:
            init0(self, *a, **kw)
            fields[id(self)] = fid
            if top:
                entry["out"] = {"s": int(self.s), "neighbor_idx": np.array(self.neighbor_idx),
                                "bbox_min": np.array(self.bbox_min), "voxel_size": float(self.voxel_size),
                                "resolution": int(self.resolution), "support_radius": float(self.support_radius)}
        except Exception as e:  # noqa: BLE001
            if top:
                entry["exc"] = type(e).__name__
            raise
        finally:
            depth[0] -= 1
            if top:
                calls.append(entry)

    def method(name, fn, out_fn):
        def m(self, *a, **kw):
            top = depth[0] == 0
            entry = {"fn": f"KnnField.{name}", "field": fields.get(id(self)), "args": conv(a), "kw": conv(kw)} \
                if top else None
            depth[0] += 1
            try:
                out = fn(self, *a, **kw)
                if top:
                    entry["out"] = out_fn(self, a, out)
                return out
            except Exception as e:  # noqa: BLE001
                if top:
                    entry["exc"] = type(e).__name__
                raise
            finally:
                depth[0] -= 1
                if top:
                    calls.append(entry)
        return m

    def live_out(self, a, out):
        m = a[0]
        return {"live_map": np.array(self.live_maps[m.frame_id]), "lookup_table": np.array(self.lookup_table)}

    K.KnnField.__init__ = init
    K.KnnField.update_live_map = method("update_live_map", upd0, live_out)
    K.KnnField.query_motion_batch = method("query_motion_batch", qb0, lambda self, a, out: conv(out))
    K.KnnField.query_motion = method("query_motion", q0, lambda self, a, out: conv(out))

    tests = [os.path.join(REF, "tests", f) for f in ("test_transforms.py", "test_edgraph.py", "test_knnfield.py",
                                                      "test_skeleton.py")]
    rc = pytest.main(["-q", "-p", "no:cacheprovider", *tests])
    if rc != 0:
        raise SystemExit(f"the reference's tests failed while recording (rc {rc})")
    # drop exact duplicate calls (the timing test repeats one query batch)
    seen, uniq = set(), []
    for c in calls:
        key = pickle.dumps((c["fn"], c.get("field"), c["args"], c["kw"]))
        if key in seen:
            continue
        seen.add(key)
        uniq.append(c)
    with gzip.open(OUT, "wb") as f:
        pickle.dump({"source": "reference tests: test_transforms/test_edgraph/test_knnfield/test_skeleton",
                     "calls": uniq}, f, protocol=4)
    print(f"{len(calls)} calls ({len(uniq)} distinct) -> {OUT} ({os.path.getsize(OUT) / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
