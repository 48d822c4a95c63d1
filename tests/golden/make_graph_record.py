"""Golden CFGR graph dump written by the REAL reference (records.py:39-86).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_graph_record.py
Writes tests/golden/graph_ref.bin (17 nodes, 3 motions, as tests/test_io.py:88-108) and
graph_ref.txt (graph_debug_dump of it).
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from capfields.edgraph import EDGraph, GraphMotion  # noqa: E402
from capfields.records import graph_debug_dump, save_graph  # noqa: E402
from capfields.transforms import DualQuaternion  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(3)
g = EDGraph(rng.normal(size=(17, 3)), radius=0.123, knn_k=5)
motions = [GraphMotion(t * 7, np.stack([DualQuaternion.from_rotvec_trans(rng.normal(size=3), rng.normal(size=3)).packed()
                                       for _ in range(17)])) for t in range(3)]
save_graph(os.path.join(HERE, "graph_ref.bin"), g, motions)
open(os.path.join(HERE, "graph_ref.txt"), "w").write(graph_debug_dump(g, motions))
