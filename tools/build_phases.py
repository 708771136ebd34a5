"""Build phase split (CUDA events inside kd_tree_build) over repeated builds:
python tools/build_phases.py [C2|C3] [builds]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
from paper_1607_08220_b200.workloads import CONFIGS, make_points
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 6
rows = make_points(cfg, "cuda", seed=1000)
coords = rows.t().contiguous()
t = None
for i in range(nb):
    del t
    t = build_local_tree_device(coords, None, BuildConfig(bucket_size=CONFIGS[cfg].leaf))
    torch.cuda.synchronize()
    b = t.build_info
    print(f"{cfg} build {i}: {b['build_ms']:8.3f} ms = levels {b['ms_levels']:7.3f} + subtree {b['ms_subtree']:7.3f}"
          f" + finish {b['ms_finish']:6.3f}  ({b['levels']} levels, {b['tasks']} tasks)", flush=True)
