"""Host-side level timeline of one C2 build with and without caller ids (KDB_TRACE=1)."""
import os, sys
os.environ["KDB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
from paper_1607_08220_b200.workloads import make_points
rows = make_points("C2", "cuda", seed=1000, n=64_000_000)
coords = rows.t().contiguous()
ids = torch.arange(64_000_000, dtype=torch.int64, device="cuda")
for i, idv in enumerate([None, ids, None, ids]):
    torch.cuda.synchronize()
    print("---- build", i, "ids" if idv is not None else "no ids", file=sys.stderr)
    t = build_local_tree_device(coords, idv, BuildConfig(bucket_size=32))
    torch.cuda.synchronize()
    print("build_ms", t.build_info["build_ms"], file=sys.stderr)
    del t
