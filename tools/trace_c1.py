"""Host-side level timeline of a C1 build (1M uniform points), KDB_TRACE=1."""
import os, sys
os.environ["KDB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
from paper_1607_08220_b200.workloads import make_points
rows = make_points("C1", "cuda", seed=1000, n=1_000_000)
coords = rows.t().contiguous()
for i in range(4):
    torch.cuda.synchronize()
    print("---- build", i, file=sys.stderr)
    t = build_local_tree_device(coords, None, BuildConfig(bucket_size=32))
    torch.cuda.synchronize()
    print("build_ms", t.build_info["build_ms"], file=sys.stderr)
    del t
