"""TEST INFRASTRUCTURE: a CPU stand-in for the rank-local device work of the
global tier, so the SPMD protocol (cluster.py / dist_query.py) runs in the
CPU-only suite -- on in-process thread ranks and on gloo process groups.
Histograms, builds and local KNN are delegated to the C oracle (the checker);
splits, routing and merging are numpy/torch restatements of the reference
(cluster.py:96-154, :292-294; dist_query.py:156-161).  The product path always
uses cluster.CudaBackend (the CUDA kernels); nothing here is imported by it.
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


def _row_bytes(dims, es):
    return ((dims * es + 7) // 8) * 8 + 8


class CpuOracleBackend:
    name = "cpu-oracle"

    def histogram(self, pts, dim, boundaries):
        vals = pts.coords[dim].double().cpu().numpy()
        c, e = O.histogram(vals, boundaries)
        return torch.as_tensor(c), torch.as_tensor(e)

    def split_rows(self, pts, dim, value):
        n, dims = pts.count, pts.dims
        low = pts.coords[dim].double() < value
        order = torch.cat([torch.nonzero(low).flatten(), torch.nonzero(~low).flatten()])
        es = pts.coords.element_size()
        w = _row_bytes(dims, es)
        rows = torch.zeros((n, w), dtype=torch.uint8)
        c = pts.coords[:, order].t().contiguous().view(torch.uint8).reshape(n, dims * es)
        rows[:, :dims * es] = c
        rows[:, w - 8:] = pts.ids[order].contiguous().view(torch.uint8).reshape(n, 8)
        return rows, low.sum().reshape(1).to(torch.int64)

    def unpack_rows(self, rows, dims, dtype):
        from paper_1607_08220_b200.cluster import DevicePoints
        n = rows.shape[0]
        es = torch.empty((), dtype=dtype).element_size()
        w = _row_bytes(dims, es)
        c = rows[:, :dims * es].contiguous().view(dtype).reshape(n, dims).t().contiguous()
        i = rows[:, w - 8:].contiguous().view(torch.int64).reshape(n)
        return DevicePoints(c, i)

    def build(self, pts, cfg):
        coords = pts.coords.double().cpu().numpy()
        ids = pts.ids.cpu().numpy().view(np.uint64)
        return OracleTreeView(O.build_tree(coords, ids, bucket_size=cfg.bucket_size,
                                           local_sample_m=cfg.local_sample_m, variance_sample=cfg.variance_sample,
                                           seed=cfg.seed, threads=1))

    def knn(self, tree, q, k, radii=None, excl=None, counters=False):
        qn = q.double().cpu().numpy()
        m = qn.shape[0]
        if m == 0 or tree.count == 0:
            z = (np.zeros((m, k)), np.zeros((m, k), np.uint64), np.zeros(m, np.int64), np.zeros((m, 3), np.int64))
        else:
            r = np.inf if radii is None else radii.double().cpu().numpy()
            kk = k + (1 if excl is not None else 0)
            d, i, c, ctr = O.knn(tree.t, qn, kk, radii=r, threads=1)
            if excl is not None:  # top-(k+1) minus the excluded id, truncated to k
                ex = excl.cpu().numpy().view(np.uint64)
                d2, i2, c2 = np.zeros((m, k)), np.zeros((m, k), np.uint64), np.zeros(m, np.int64)
                for j in range(m):
                    keep = i[j, :c[j]] != ex[j]
                    dd, ii = d[j, :c[j]][keep][:k], i[j, :c[j]][keep][:k]
                    c2[j] = len(dd)
                    d2[j, :len(dd)], i2[j, :len(ii)] = dd, ii
                d, i, c = d2, i2, c2
            z = (d, i, c, ctr)
        d, i, c, ctr = z
        return (torch.as_tensor(d), torch.as_tensor(np.ascontiguousarray(i).view(np.int64)), torch.as_tensor(c),
                torch.as_tensor(ctr) if counters else None)

    def route(self, regions, q, radii=None, within=False):
        """GlobalTree.owner_of (ties right) + ranks strictly within the radius."""
        qn = q.double().cpu().numpy()
        m, p = qn.shape[0], regions.p
        pdim, pval = regions.pdim.cpu().numpy(), regions.pval.cpu().numpy()
        lo, hi = regions.lo.cpu().numpy(), regions.hi.cpu().numpy()
        heap = np.zeros(m, dtype=np.int64)
        for _ in range(p.bit_length() - 1):
            heap = 2 * heap + 1 + (qn[np.arange(m), pdim[heap]] >= pval[heap])
        owner = heap - (p - 1)
        wm = None
        if within:
            r = np.full(m, np.inf) if radii is None else radii.double().cpu().numpy()
            wm = np.zeros(m, dtype=np.int64)
            for rk in range(p):
                s = np.zeros(m)
                for d in range(qn.shape[1]):
                    qd = qn[:, d]
                    o = np.where(qd < lo[rk, d], lo[rk, d] - qd, np.where(qd > hi[rk, d], qd - hi[rk, d], 0.0))
                    s = s + o * o
                wm |= ((s < r) & (owner != rk)).astype(np.int64) << rk
        return torch.as_tensor(owner.astype(np.int32)), (torch.as_tensor(wm) if within else None)

    def merge(self, k, ld, li, lc, my_rank, slot, rd, ri, rc, rrank):
        """dist_query.py:156-161 per owned query: pool, duplicates flagged, lexsort (d, id)."""
        m = ld.shape[0]
        ld, li, lc = ld.numpy(), li.numpy().view(np.uint64), lc.numpy()
        slot, rd, ri, rc, rrank = slot.numpy(), rd.numpy(), ri.numpy().view(np.uint64), rc.numpy(), rrank.numpy()
        od, oi = np.zeros((m, k)), np.zeros((m, k), np.uint64)
        orank, oc = np.zeros((m, k), np.int32), np.zeros(m, np.int64)
        dup = 0
        by = {}
        for t in range(slot.shape[0]):
            by.setdefault(int(slot[t]), []).append(t)
        for j in range(m):
            d = [ld[j, :lc[j]]] + [rd[t, :rc[t]] for t in by.get(j, [])]
            p = [li[j, :lc[j]]] + [ri[t, :rc[t]] for t in by.get(j, [])]
            r = [np.full(lc[j], my_rank)] + [np.full(rc[t], rrank[t]) for t in by.get(j, [])]
            d, p, r = np.concatenate(d), np.concatenate(p), np.concatenate(r)
            if np.unique(p).shape[0] != p.shape[0]:
                dup = 1
            o = np.lexsort((p, d))[:k]
            oc[j] = o.shape[0]
            od[j, :o.shape[0]], oi[j, :o.shape[0]], orank[j, :o.shape[0]] = d[o], p[o], r[o]
        return (torch.as_tensor(od), torch.as_tensor(oi.view(np.int64)), torch.as_tensor(orank), torch.as_tensor(oc),
                torch.tensor([dup], dtype=torch.int32))
