"""Small C4-like run for profiling the warp-per-query kernel under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1607_08220_b200 import core, local_tree as lt, local_query as lq
from paper_1607_08220_b200.workloads import make_points, make_queries
rows = make_points("C4", "cuda", seed=1000, n=4_000_000)
qs, _ = make_queries("C4", rows, "cuda", seed=2000, q=100_000)
tree = lt.build_local_tree_device(rows.t().contiguous(), None, lt.BuildConfig(bucket_size=64))
lq.find_knn_device(tree, qs, 10)
torch.cuda.synchronize()
