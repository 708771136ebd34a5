"""A/B of the 3-D KNN kernels on one BASELINE config: packet vs per-lane (default)
(KD_KNN_PACKET).  python tools/knn_ab.py C2 [reps]  -> ms per batch, GPU counters, equality."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1607_08220_b200 import _native as N
from paper_1607_08220_b200.local_query import find_knn_device
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
from paper_1607_08220_b200.workloads import CONFIGS, make_points, make_queries

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = CONFIGS[cfg]
dev = torch.device("cuda", 0)
rows = make_points(cfg, dev, seed=1000)
q, ex = make_queries(cfg, rows, dev, seed=2000)
tree = build_local_tree_device(rows.t().contiguous(), None, BuildConfig(bucket_size=w.leaf, seed=0))
torch.cuda.synchronize()
res = {}
for name, fl in (("packet", N.KD_KNN_PACKET), ("lane", 0)):
    ts = []
    for r in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = find_knn_device(tree, q, w.k, exclude_ids=ex, flags=fl)
        b.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(b))
    d, i, c, _ = find_knn_device(tree, q, w.k, exclude_ids=ex, flags=fl, counters=True)
    ctr = find_knn_device(tree, q, w.k, exclude_ids=ex, flags=fl, counters=True)[3].double().mean(0).tolist()
    res[name] = (d, i, c)
    print(f"{cfg} {name:7s} {min(ts):8.3f} ms  ({w.q / min(ts) / 1e3:.1f} M q/s)  counters nodes/buckets/points "
          f"{ctr[0]:.1f} {ctr[1]:.2f} {ctr[2]:.1f}", flush=True)
a, b = res["packet"], res["lane"]
print("equal:", all(torch.equal(x, y) for x, y in zip(a, b)))
