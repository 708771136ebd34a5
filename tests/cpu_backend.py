"""TEST INFRASTRUCTURE: a CPU stand-in for the rank-local device work of the
global tier, so the SPMD protocol (cluster.py / dist_query.py) can run in the
CPU-only suite -- on in-process thread ranks and on gloo world_size-2 process
groups.  Histograms, partitions, local builds and local KNN are delegated to
the C oracle (the checker); the product path always uses CudaBackend.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O


class OracleTreeView:
    """Adapter giving the oracle tree the LocalTree attribute surface."""

    def __init__(self, t: O.OracleTree):
        self.t = t
        self.node_dim, self.node_value = t.node_dim, t.node_value
        self.node_left, self.node_right, self.node_count = t.node_left, t.node_right, t.node_count
        self.depth = t.depth
        from paper_1607_08220_b200.core import PointSet
        self.points = PointSet(t.coords, t.ids)

    @property
    def n_nodes(self):
        return self.t.n_nodes

    @property
    def count(self):
        return self.t.coords.shape[1]


class CpuOracleBackend:
    name = "cpu-oracle"

    def histogram(self, pts, dim, boundaries):
        vals = pts.coords[dim].double().cpu().numpy()
        return O.histogram(vals, boundaries)

    def partition(self, pts, plane):
        from paper_1607_08220_b200.cluster import DevicePoints
        row = pts.coords[plane.dim].double()
        low = row < plane.value
        order = torch.cat([torch.nonzero(low).flatten(), torch.nonzero(~low).flatten()])
        return DevicePoints(pts.coords[:, order].contiguous(), pts.ids[order].contiguous()), int(low.sum())

    def build(self, pts, cfg):
        coords = pts.coords.double().cpu().numpy()
        ids = pts.ids.cpu().numpy().view(np.uint64)
        return OracleTreeView(O.build_tree(coords, ids, bucket_size=cfg.bucket_size,
                                           local_sample_m=cfg.local_sample_m, variance_sample=cfg.variance_sample,
                                           seed=cfg.seed, threads=1))

    def knn(self, tree, queries, k, radii=None):
        q = queries.double().cpu().numpy()
        r = np.inf if radii is None else radii.double().cpu().numpy()
        if q.shape[0] == 0 or tree.count == 0:
            m = q.shape[0]
            return np.zeros((m, k)), np.zeros((m, k), np.uint64), np.zeros(m, np.int64), np.zeros((m, 3), np.int64)
        return O.knn(tree.t, q, k, radii=r, threads=1)
