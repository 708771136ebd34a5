"""High-D KNN diagnostics: packet vs one-thread-per-query kernels on a C4-like tree (counters, time)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1607_08220_b200 import core, local_tree as lt, local_query as lq, _native as N
from paper_1607_08220_b200.workloads import make_points, make_queries

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
rows = make_points("C4", "cuda", seed=1000, n=n)
qs, _ = make_queries("C4", rows, "cuda", seed=2000, q=nq)
ps = core.PointSet.from_rows(rows.cpu().numpy().astype(np.float64))
tree = lt.build_local_tree(ps, lt.BuildConfig(bucket_size=64))
q = qs.cpu().numpy()
for name, fl in (("packet", 0), ("thread", N.KD_THREAD_PER_QUERY)):
    lq.find_knn_batch(tree, q[:512], 10, flags=fl)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d, i, c, ctr = lq.find_knn_batch(tree, q, 10, flags=fl)
    dt = time.perf_counter() - t0
    print(f"{name}: {nq / dt:.0f} q/s  nodes {ctr[:, 0].mean():.0f} leaves {ctr[:, 1].mean():.0f} points {ctr[:, 2].mean():.0f}")
    if name == "packet":
        ref = (d.copy(), i.copy())
    else:
        print("identical:", np.array_equal(ref[0], d), np.array_equal(ref[1], i))
