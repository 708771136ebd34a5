"""GPU traversal counters vs the reference traversal's (oracle) on a C2-like sample."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1607_08220_b200 import core, local_tree as lt, local_query as lq
from paper_1607_08220_b200.workloads import make_points_numpy
rows = make_points_numpy("C2", 4_000_000, seed=77).astype(np.float64)
ps = core.PointSet.from_rows(rows)
tree = lt.build_local_tree(ps, lt.BuildConfig(bucket_size=32))
sel = np.random.default_rng(5).choice(rows.shape[0], 100_000, replace=False)
q = rows[sel]
d, i, c, ctr = lq.find_knn_batch(tree, q, 5, exclude_ids=ps.ids[sel])
print("gpu (k+1 list): nodes %.1f leaves %.2f points %.1f" % tuple(ctr.mean(0)))
ot = O.OracleTree(tree.node_dim, tree.node_value, tree.node_left, tree.node_right, tree.node_count, None,
                  tree.points.coords, tree.points.ids, tree.depth)
_, _, _, rc = O.knn(ot, q[:20000], 6)
print("reference (k=6): nodes %.1f leaves %.2f points %.1f" % tuple(rc.mean(0)))
