"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the C oracle (kdknn_oracle.c).

The oracle is the checker for the CUDA path, never the product: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference`` arm) may import this module.  The product package
``paper_1607_08220_b200`` never imports it.

Functions mirror the reference entry points they restate:

* :func:`build_tree`  -- ``kdknn.local_tree.build_local_tree`` (local_tree.py:436-574)
* :func:`knn`         -- ``kdknn.local_query.find_knn_batch`` (local_query.py:175-216)
* :func:`brute_knn`   -- ``oracle_topk`` (pkg/tests/conftest.py:8-18)
* :func:`sample_indices`, :func:`node_seed`, :func:`histogram`,
  :func:`select_median` -- ``kdknn.median`` primitives (median.py:51-166)
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "kdknn_oracle.c")

_lib = None


def compile_oracle(force: bool = False) -> str:
    """Compile kdknn_oracle.c -> oracle/liboracle.so (gcc, OpenMP, no FMA)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return LIB_PATH


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def lib():
    global _lib
    if _lib is None:
        compile_oracle()
        L = C.CDLL(LIB_PATH)
        L.kdo_node_seed.restype = C.c_uint64
        L.kdo_node_seed.argtypes = [C.c_uint64] * 3
        L.kdo_sample_indices.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p]
        L.kdo_histogram.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.kdo_select_median.restype = C.c_int64
        L.kdo_select_median.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
        L.kdo_build.restype = C.c_void_p
        L.kdo_build.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                C.c_uint64, C.c_int]
        L.kdo_tree_n_nodes.restype = C.c_int64
        L.kdo_tree_n_nodes.argtypes = [C.c_void_p]
        L.kdo_tree_depth.restype = C.c_int64
        L.kdo_tree_depth.argtypes = [C.c_void_p]
        L.kdo_tree_export.argtypes = [C.c_void_p] * 7
        L.kdo_tree_free.argtypes = [C.c_void_p]
        L.kdo_knn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                              C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int64,
                              C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.kdo_brute_knn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_void_p,
                                    C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int]
        _lib = L
    return _lib


def node_seed(seed: int, path: int, salt: int) -> int:
    m = 0xFFFFFFFFFFFFFFFF
    return int(lib().kdo_node_seed(seed & m, path & m, salt & m))


def sample_indices(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(m, dtype=np.int64)
    lib().kdo_sample_indices(n, m, seed & 0xFFFFFFFFFFFFFFFF, _p(out))
    return out


def histogram(values, boundaries):
    values = np.ascontiguousarray(values, dtype=np.float64)
    b = np.ascontiguousarray(boundaries, dtype=np.float64)
    counts = np.empty(b.shape[0] + 1, dtype=np.int64)
    equals = np.empty(max(b.shape[0], 1), dtype=np.int64)
    lib().kdo_histogram(_p(values), values.shape[0], _p(b), b.shape[0], _p(counts), _p(equals))
    return counts, equals[: b.shape[0]]


def select_median(counts) -> tuple[int, int]:
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    below = np.zeros(1, dtype=np.int64)
    bi = lib().kdo_select_median(counts.shape[0] - 1, _p(counts), _p(below))
    return int(bi), int(below[0])


@dataclass
class OracleTree:
    """Reference-layout tree (local_tree.py:71-108) built by the C oracle."""
    node_dim: np.ndarray
    node_value: np.ndarray
    node_left: np.ndarray
    node_right: np.ndarray
    node_count: np.ndarray
    perm: np.ndarray          # packed row i holds input point perm[i]
    coords: np.ndarray        # packed (D, n) f64
    ids: np.ndarray           # packed u64 ids
    depth: int

    @property
    def n_nodes(self):
        return self.node_dim.shape[0]


def build_tree(coords, ids=None, bucket_size=32, local_sample_m=1024, variance_sample=1024,
               seed=0, threads=0) -> OracleTree:
    """coords: (D, n) array (any float dtype; upcast to f64 exactly)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    D, n = coords.shape
    ids = np.arange(n, dtype=np.uint64) if ids is None else np.ascontiguousarray(ids, dtype=np.uint64)
    L = lib()
    h = L.kdo_build(_p(coords), n, D, bucket_size, local_sample_m, variance_sample,
                    seed & 0xFFFFFFFFFFFFFFFF, threads)
    if not h:
        raise ValueError("oracle build failed")
    try:
        nn = int(L.kdo_tree_n_nodes(h))
        depth = int(L.kdo_tree_depth(h))
        nd = np.empty(nn, np.int32); nv = np.empty(nn, np.float64)
        nl = np.empty(nn, np.int32); nr = np.empty(nn, np.int32); nc = np.empty(nn, np.int64)
        perm = np.empty(n, np.int64)
        L.kdo_tree_export(h, _p(nd), _p(nv), _p(nl), _p(nr), _p(nc), _p(perm))
    finally:
        L.kdo_tree_free(h)
    return OracleTree(nd, nv, nl, nr, nc, perm, np.ascontiguousarray(coords[:, perm]), ids[perm], depth)


def knn(tree: OracleTree, queries, k, radii=np.inf, threads=0):
    """Reference traversal (local_query.py:72-172) over an oracle/reference tree.
    Returns (dists (nq,k), ids (nq,k), counts (nq,), counters (nq,3))."""
    q = np.ascontiguousarray(queries, dtype=np.float64)
    if q.ndim != 2:
        raise ValueError("queries must be (nq, dims)")
    nq = q.shape[0]
    r = np.full(nq, float(radii)) if np.isscalar(radii) else np.ascontiguousarray(radii, dtype=np.float64)
    od = np.zeros((nq, k), np.float64); oi = np.zeros((nq, k), np.uint64)
    oc = np.zeros(nq, np.int64); octr = np.zeros((nq, 3), np.int64)
    coords = np.ascontiguousarray(tree.coords, dtype=np.float64)
    ids = np.ascontiguousarray(tree.ids, dtype=np.uint64)
    D, n = coords.shape
    lib().kdo_knn(_p(np.ascontiguousarray(tree.node_dim, np.int32)),
                  _p(np.ascontiguousarray(tree.node_value, np.float64)),
                  _p(np.ascontiguousarray(tree.node_left, np.int32)),
                  _p(np.ascontiguousarray(tree.node_right, np.int32)), tree.node_dim.shape[0],
                  _p(coords), n, _p(ids), D, int(tree.depth), _p(q), nq, k, _p(r),
                  _p(od), _p(oi), _p(oc), _p(octr), threads)
    return od, oi, oc, octr


def brute_knn(coords, ids, queries, k, radii=None, threads=0):
    """oracle_topk (conftest.py:8-18) for a batch: (dists, ids, counts)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    D, n = coords.shape
    ids = np.arange(n, dtype=np.uint64) if ids is None else np.ascontiguousarray(ids, dtype=np.uint64)
    q = np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, D)
    nq = q.shape[0]
    od = np.zeros((nq, k), np.float64); oi = np.zeros((nq, k), np.uint64); oc = np.zeros(nq, np.int64)
    if radii is None:
        rp = None
    else:
        rp = np.full(nq, float(radii)) if np.isscalar(radii) else np.ascontiguousarray(radii, np.float64)
    lib().kdo_brute_knn(_p(coords), n, _p(ids), D, _p(q), nq, k, None if rp is None else _p(rp),
                        _p(od), _p(oi), _p(oc), threads)
    return od, oi, oc
