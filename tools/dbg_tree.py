"""debug: GPU tree vs oracle on a small random set; prints the first differing node"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1607_08220_b200.core import PointSet
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
rng = np.random.default_rng(3)
rows = rng.random((n, 3), dtype=np.float32).astype(np.float64)
ps = PointSet.from_rows(rows)
tree = build_local_tree(ps, BuildConfig(bucket_size=32, seed=7))
ref = O.build_tree(ps.coords, ps.ids, bucket_size=32, seed=7)
print("nodes", tree.n_nodes, len(ref.node_dim), "depth", tree.depth, ref.depth)
for f in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
    a, b = getattr(tree, f), getattr(ref, f)
    if a.shape != b.shape:
        print(f, "shape", a.shape, b.shape); continue
    bad = np.nonzero(a != b)[0]
    print(f, "mismatches", len(bad), bad[:10], a[bad[:5]], b[bad[:5]])
print("ids equal", np.array_equal(tree.points.ids, ref.ids))
