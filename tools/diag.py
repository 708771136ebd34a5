"""Debug helper: first differing node between the GPU tree and the oracle, and KNN kernel A/B."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from datagen import golden_cases, make_rows
from oracle import oracle as O
from paper_1607_08220_b200 import core, local_tree as lt, local_query as lq, _native as N

case = golden_cases()["aniso3_5000"]
ps = core.PointSet.create(case["coords"], case["ids"])
t = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
r = O.build_tree(ps.coords, ps.ids, **case["cfg"])
print("nodes", t.n_nodes, r.n_nodes, "depth", t.depth, r.depth, t.build_info)
for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
    a, b = getattr(t, key), getattr(r, key)
    if a.shape != b.shape or not np.array_equal(a, b):
        m = min(a.shape[0], b.shape[0])
        i = int(np.nonzero(a[:m] != b[:m])[0][0]) if (a[:m] != b[:m]).any() else m
        print(key, "first diff at", i)
        lo = max(0, i - 3)
        for j in range(lo, min(m, i + 4)):
            print("  ", j, t.node_dim[j], r.node_dim[j], t.node_value[j], r.node_value[j], t.node_left[j], r.node_left[j],
                  t.node_right[j], r.node_right[j], t.node_count[j], r.node_count[j])
        break
rows = make_rows(200000, 3, 5, "halo-f32")
ps = core.PointSet.from_rows(rows)
t = lt.build_local_tree(ps, lt.BuildConfig())
q = rows[:3000]
bd, bi, bc = O.brute_knn(ps.coords, ps.ids, q, 6)
for name, fl in (("persistent", 0), ("thread", N.KD_THREAD_PER_QUERY), ("nosort", N.KD_NO_SORT)):
    d, i, c, ctr = lq.find_knn_batch(t, q, 6, flags=fl)
    bad = np.nonzero((d != bd).any(1) | (i != bi).any(1))[0]
    print(name, "mismatching queries:", len(bad), "of", len(q), "ctr mean", ctr.mean(0))
    for b in bad[:3]:
        print("   q", b, "got", d[b], i[b], "want", bd[b], bi[b])
