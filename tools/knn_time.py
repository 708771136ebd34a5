"""Time the default KNN path on BASELINE configs and print a checksum of the result rows
(for A/B of environment-selected kernel variants across processes).
python tools/knn_time.py C2,C3 [reps]"""
import os, sys, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1607_08220_b200.local_query import find_knn_device
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
from paper_1607_08220_b200.workloads import CONFIGS, make_points, make_queries

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "C2").split(","):
    w = CONFIGS[cfg]
    rows = make_points(cfg, dev, seed=1000)
    q, ex = make_queries(cfg, rows, dev, seed=2000)
    tree = build_local_tree_device(rows.t().contiguous(), None, BuildConfig(bucket_size=w.leaf, seed=0))
    del rows
    torch.cuda.synchronize()
    out = None
    ts = []
    for r in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = find_knn_device(tree, q, w.k, exclude_ids=ex, out=out)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    d, i, c, _ = out
    valid = (torch.arange(w.k, device=dev)[None, :] < c[:, None])
    h = hashlib.sha256()
    h.update(torch.where(valid, d, torch.zeros_like(d)).sum(0).cpu().numpy().tobytes())
    h.update(torch.where(valid, i, torch.zeros_like(i)).sum(0).cpu().numpy().tobytes())
    h.update(c.sum().cpu().numpy().tobytes())
    ts.sort()
    print(f"{cfg} knn min {ts[0]:8.3f} ms  median {ts[len(ts)//2]:8.3f} ms  ({w.q / ts[0] / 1e3:.1f} M q/s)  "
          f"checksum {h.hexdigest()[:16]}  env " +
          " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("KDB_")), flush=True)
    del tree, q, ex, out
    torch.cuda.empty_cache()
