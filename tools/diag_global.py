"""Where the single-rank global-tier step spends its time (torchrun --nproc-per-node 1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1607_08220_b200.cluster import ClusterConfig, DevicePoints, rank_build_global
from paper_1607_08220_b200.comm import TorchComm
from paper_1607_08220_b200.dist_device import DeviceRegions, rank_query_device
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
from paper_1607_08220_b200.local_query import find_knn_device
from paper_1607_08220_b200.workloads import make_points, make_queries
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
comm = TorchComm()
n, q = 64_000_000, 16_000_000
rows = make_points("C2", dev, seed=1000, n=n); coords = rows.t().contiguous()
ids = torch.arange(n, dtype=torch.int64, device=dev)
queries, sel = make_queries("C2", rows, dev, seed=2000, q=q)
qids = torch.arange(q, dtype=torch.int64, device=dev)
bcfg = BuildConfig(bucket_size=32)
def timed(name, f, reps=3):
    for _ in range(2): r = f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): r = f()
    torch.cuda.synchronize(); print(f"{name}: {(time.perf_counter() - t0) / reps * 1e3:.1f} ms", flush=True)
    return r
timed("build no ids", lambda: build_local_tree_device(coords, None, bcfg))
tree = timed("build ids", lambda: build_local_tree_device(coords, ids, bcfg))
timed("global P=1", lambda: rank_build_global(comm, DevicePoints(coords, ids), ClusterConfig(seed=0)))
gt, pts, _ = rank_build_global(comm, DevicePoints(coords, ids), ClusterConfig(seed=0))
timed("knn local", lambda: find_knn_device(tree, queries, 5, exclude_ids=sel))
timed("query device P=1", lambda: rank_query_device(comm, tree, DeviceRegions(gt, dev), qids, queries, 5, excl=sel))
dist.destroy_process_group()
