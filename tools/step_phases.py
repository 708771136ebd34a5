"""bench.py-like steps (build + KNN) with the build's internal phase split next to the
outer CUDA-event times: python tools/step_phases.py [C3] [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1607_08220_b200.local_query import find_knn_device
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
from paper_1607_08220_b200.workloads import CONFIGS, make_points, make_queries
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 6
w = CONFIGS[cfg]
rows = make_points(cfg, "cuda", seed=1000)
coords = rows.t().contiguous()
q, ex = make_queries(cfg, rows, "cuda", seed=2000)
tree = out = None
for i in range(ns):
    del tree, out
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    tree = build_local_tree_device(coords, None, BuildConfig(bucket_size=w.leaf))
    e[1].record()
    out = find_knn_device(tree, q, w.k, exclude_ids=ex)
    e[2].record()
    torch.cuda.synchronize()
    b = tree.build_info
    print(f"{cfg} step {i}: outer build {e[0].elapsed_time(e[1]):8.3f} ms (inner {b['build_ms']:8.3f} = "
          f"{b['ms_levels']:.3f} + {b['ms_subtree']:.3f} + {b['ms_finish']:.3f}), knn {e[1].elapsed_time(e[2]):8.3f} ms",
          flush=True)
