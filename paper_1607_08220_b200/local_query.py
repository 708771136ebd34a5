"""Exact KNN over one local tree on the GPU (drop-in for ``kdknn.local_query``).

``find_knn_batch`` (reference local_query.py:175-216) validates exactly like the
reference, then runs ``kd_knn`` of the C-ABI: one thread per query, queries
ordered by their home leaf so warps traverse coherently, binary64 leaf scans in
the reference's operation order (bit-identical distances), exact
(sq_dist, point_id) tie-breaking.  ``workers`` is accepted and ignored.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .core import KnnResult
from .local_tree import LocalTree

__all__ = ["find_knn", "find_knn_batch", "count_visited", "find_knn_device"]


def find_knn_batch(tree: LocalTree, queries, k: int, radii=np.inf, workers: int = 1, *,
                   exclude_ids=None, counters: bool = True, device: int = 0, flags: int = 0,
                   reference_walk: bool = False):
    """Exact KNN for a block of queries against one tree.

    Returns (dists (nq,k) f64, ids (nq,k) u64, counts (nq,) i64, counters (nq,3) i64);
    row i holds counts[i] valid entries sorted by (sq_dist, point_id).  ``radii``
    is a scalar or per-query array of squared radii (strict).  ``exclude_ids``
    (extension): one point id per query that is never returned (self-exclusion).
    ``reference_walk`` (extension): traverse exactly as the reference does
    (local_query.py:72-172: binary64 incremental bounds, pruning at bound >= r') --
    results and counters are then bit-identical to the reference's, its tie quirk
    included; the default walk has the brute-force oracle's tie semantics and counts
    its own (shorter) traversal.
    """
    if k < 1:
        raise ValueError("k must be >= 1")
    q = np.ascontiguousarray(queries, dtype=np.float64)
    if q.ndim != 2:
        raise ValueError("queries must be (nq, dims)")
    nq = q.shape[0]
    if tree.count and q.shape[1] != tree.dims:
        raise ValueError(f"query dims {q.shape[1]} != tree dims {tree.dims}")
    if np.isscalar(radii):
        r = None if np.isinf(radii) and radii > 0 else np.full(nq, float(radii))
    else:
        r = np.ascontiguousarray(radii, dtype=np.float64)
        if r.shape != (nq,):
            raise ValueError("radii must be a scalar or one value per query")
    out_d = np.empty((nq, k), dtype=np.float64)
    out_i = np.empty((nq, k), dtype=np.uint64)
    out_c = np.zeros(nq, dtype=np.int64)
    out_ctr = np.zeros((nq, 3), dtype=np.int64)
    if nq == 0:
        return out_d, out_i, out_c, out_ctr
    if tree.count == 0 or tree.n_nodes == 0:
        return out_d, out_i, out_c, out_ctr
    ex = None
    if exclude_ids is not None:
        ex = np.ascontiguousarray(exclude_ids, dtype=np.uint64)
        if ex.shape != (nq,):
            raise ValueError("exclude_ids must hold one id per query")
    nt = tree.native(device)
    if reference_walk:
        flags |= N.KD_KNN_REFERENCE
    N.check(N.lib.kd_knn(nt.handle, q.ctypes.data, nq, k, None if r is None else r.ctypes.data,
                         None if ex is None else ex.ctypes.data, out_d.ctypes.data, out_i.ctypes.data,
                         out_c.ctypes.data, out_ctr.ctypes.data if counters else None, flags, None))
    return out_d, out_i, out_c, out_ctr


def find_knn(tree: LocalTree, q, k: int, sq_radius: float = np.inf, query_id: int = 0,
             rank: int = 0) -> KnnResult:
    """Single-query entry point (local_query.py:219-226)."""
    q = np.asarray(q, dtype=np.float64).reshape(1, -1)
    d, i, c, _ = find_knn_batch(tree, q, k, sq_radius)
    n = int(c[0])
    return KnnResult.from_sorted(query_id, d[0, :n], i[0, :n], np.full(n, rank, dtype=np.int64), k)


def count_visited(tree: LocalTree, q, k: int, sq_radius: float = np.inf) -> dict:
    """Traversal counters for one query (local_query.py:229-237): the reference's own walk
    is replayed on the device, so the counters equal the reference's."""
    q = np.asarray(q, dtype=np.float64).reshape(1, -1)
    _, _, _, ctr = find_knn_batch(tree, q, k, sq_radius, reference_walk=True)
    return {"nodes_visited": int(ctr[0, 0]), "buckets_scanned": int(ctr[0, 1]),
            "points_compared": int(ctr[0, 2])}


def find_knn_device(tree: LocalTree, queries, k: int, radii=None, exclude_ids=None, counters: bool = False,
                    sort_queries: bool = True, stream=None, out=None, flags: int = 0):
    """Device-tensor variant: queries (nq, dims) float64 CUDA tensor.  Returns
    torch tensors (dists, ids(int64 view of uint64), counts, counters|None)."""
    import torch
    if k < 1:
        raise ValueError("k must be >= 1")
    if queries.dim() != 2 or queries.dtype != torch.float64 or not queries.is_cuda:
        raise ValueError("queries must be an (nq, dims) float64 CUDA tensor")
    queries = queries.contiguous()
    nq = queries.shape[0]
    dev = queries.device
    if tree.count and queries.shape[1] != tree.dims:
        raise ValueError(f"query dims {queries.shape[1]} != tree dims {tree.dims}")
    tdev = tree.native(dev.index or 0).info().device
    if (dev.index or 0) != tdev:
        raise ValueError(f"queries are on cuda:{dev.index or 0} but the tree lives on cuda:{tdev}")

    def _per_query(t, name, dtypes):
        if t is None:
            return None
        if t.shape != (nq,) or t.dtype not in dtypes or t.device != dev:
            raise ValueError(f"{name} must be an ({nq},) {'/'.join(str(d) for d in dtypes)} tensor on {dev}")
        return t.contiguous()

    radii = _per_query(radii, "radii", (torch.float64,))
    exclude_ids = _per_query(exclude_ids, "exclude_ids", (torch.int64, torch.uint64))
    if out is None:
        od = torch.empty((nq, k), dtype=torch.float64, device=dev)
        oi = torch.empty((nq, k), dtype=torch.int64, device=dev)
        oc = torch.empty((nq,), dtype=torch.int64, device=dev)
        octr = torch.empty((nq, 3), dtype=torch.int64, device=dev) if counters else None
    else:
        od, oi, oc, octr = out
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    flags = flags | N.KD_DEVICE_PTRS | (0 if sort_queries else N.KD_NO_SORT)
    nt = tree.native(dev.index or 0)
    N.check(N.lib.kd_knn(nt.handle, queries.data_ptr(), nq, k,
                         radii.data_ptr() if radii is not None else None,
                         exclude_ids.data_ptr() if exclude_ids is not None else None,
                         od.data_ptr(), oi.data_ptr(), oc.data_ptr(),
                         octr.data_ptr() if octr is not None else None, flags, C.c_void_p(st)))
    return od, oi, oc, octr
