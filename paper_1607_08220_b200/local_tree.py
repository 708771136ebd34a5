"""Per-rank kd-tree construction on the GPU (drop-in for ``kdknn.local_tree``).

``build_local_tree`` (reference local_tree.py:436-574) runs entirely on the
device through ``kd_tree_build`` of the C-ABI: breadth-first levels with exact
sampled-histogram split selection and a stable segmented partition, then
shared-memory subtrees, then the canonical preorder stitch.  The resulting
tree is byte-identical to the reference's (node arrays, packed ids, depth) for
the same points and ``BuildConfig`` -- tests/test_gpu_parity.py checks this
against the oracle and the golden fixtures.

``LocalTree`` keeps the reference's field names (local_tree.py:71-108); for
device-built trees the arrays are exported lazily on first access, so the
query path never copies the tree back to the host.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import PointSet, SplitPlane

__all__ = ["BuildConfig", "LocalTree", "build_local_tree", "build_local_tree_device", "pack_buckets"]


@dataclass(frozen=True)
class BuildConfig:
    """Reference BuildConfig (local_tree.py:48-68).  ``workers`` and
    ``branch_factor_per_worker`` steer the reference's CPU thread pool; the
    device build is worker-invariant by construction and ignores them."""

    bucket_size: int = 32
    local_sample_m: int = 1024
    variance_sample: int = 1024
    branch_factor_per_worker: int = 10
    seed: int = 0
    workers: int = 1

    def __post_init__(self):
        if self.bucket_size < 1:
            raise ValueError("bucket_size must be >= 1")
        if self.local_sample_m < 1 or self.variance_sample < 1:
            raise ValueError("sample sizes must be >= 1")
        if self.branch_factor_per_worker < 1:
            raise ValueError("branch_factor_per_worker must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")

    def native(self) -> N.kd_build_cfg:
        return N.kd_build_cfg(self.bucket_size, self.local_sample_m, self.variance_sample,
                              self.seed & 0xFFFFFFFFFFFFFFFF)


_FIELDS = ("node_dim", "node_value", "node_left", "node_right", "node_count", "points", "depth",
           "leaf_starts", "leaf_lengths")


class LocalTree:
    """Flat preorder kd-tree with packed leaf buckets (local_tree.py:71-108).

    node_dim[i] >= 0: interior with plane (node_dim, node_value) and children
    node_left / node_right; node_dim[i] == -1: leaf whose bucket is packed rows
    [node_left, node_left + node_right).  Device-built trees hold a native
    handle and materialise these arrays on demand.
    """

    def __init__(self, node_dim=None, node_value=None, node_left=None, node_right=None, node_count=None,
                 points=None, depth=None, leaf_starts=None, leaf_lengths=None, *, _native=None, _info=None):
        self._native = _native
        self._info = _info
        self._vals = {}
        if node_dim is not None:
            self._vals = dict(node_dim=node_dim, node_value=node_value, node_left=node_left,
                              node_right=node_right, node_count=node_count, points=points, depth=int(depth),
                              leaf_starts=leaf_starts, leaf_lengths=leaf_lengths)
        self._import_dev = None

    # -- lazy export -----------------------------------------------------
    def _materialize(self):
        if self._vals:
            return
        inf = self._info
        nn, n, d = int(inf.n_nodes), int(inf.n), int(inf.dims)
        nd = np.empty(nn, np.int32); nv = np.empty(nn, np.float64)
        nl = np.empty(nn, np.int32); nr = np.empty(nn, np.int32); nc = np.empty(nn, np.int64)
        coords = np.empty((d, n), np.float64); ids = np.empty(n, np.uint64)
        arr = N.kd_tree_arrays(nd.ctypes.data, nv.ctypes.data, nl.ctypes.data, nr.ctypes.data, nc.ctypes.data,
                               coords.ctypes.data, ids.ctypes.data, None)
        N.check(N.lib.kd_tree_export(self._native.handle, C.byref(arr)))
        leaf = nd < 0
        self._vals = dict(node_dim=nd, node_value=nv, node_left=nl, node_right=nr, node_count=nc,
                          points=PointSet(coords, ids), depth=int(inf.depth),
                          leaf_starts=nl[leaf].astype(np.int64), leaf_lengths=nr[leaf].astype(np.int64))

    def __getattr__(self, name):
        if name in _FIELDS:
            self._materialize()
            return self._vals[name]
        raise AttributeError(name)

    @property
    def n_nodes(self) -> int:
        return int(self._info.n_nodes) if self._native is not None else int(self.node_dim.shape[0])

    @property
    def n_leaves(self) -> int:
        return int(self._info.n_leaves) if self._native is not None else int(self.leaf_starts.shape[0])

    @property
    def count(self) -> int:
        return int(self._info.n) if self._native is not None else self.points.count

    @property
    def dims(self) -> int:
        return int(self._info.dims) if self._native is not None else self.points.dims

    def plane(self, node: int) -> SplitPlane:
        return SplitPlane(int(self.node_dim[node]), float(self.node_value[node]))

    @property
    def build_info(self):
        """Device build statistics (ms, levels, subtree tasks, slow-path nodes)."""
        if self._native is None:
            return None
        inf = self._info
        return {"build_ms": inf.build_ms, "ms_levels": inf.build_ms_levels, "ms_subtree": inf.build_ms_subtree,
                "ms_finish": inf.build_ms_finish, "levels": int(inf.build_levels), "tasks": int(inf.build_tasks),
                "slow_nodes": int(inf.build_slow_nodes), "dtype": "f32" if inf.dtype == N.KD_F32 else "f64"}

    # -- device handle ---------------------------------------------------
    def native(self, device: int = 0) -> N.NativeTree:
        """Device-resident handle; host-constructed trees are uploaded once."""
        if self._native is not None:
            return self._native
        if self._import_dev is not None:
            return self._import_dev
        pts = self.points
        coords = np.ascontiguousarray(pts.coords, dtype=np.float64)
        dtype = N.KD_F32 if _f32_exact(coords) else N.KD_F64
        nd = np.ascontiguousarray(self.node_dim, np.int32)
        nv = np.ascontiguousarray(self.node_value, np.float64)
        nl = np.ascontiguousarray(self.node_left, np.int32)
        nr = np.ascontiguousarray(self.node_right, np.int32)
        nc = np.ascontiguousarray(self.node_count, np.int64)
        ids = np.ascontiguousarray(pts.ids, np.uint64)
        arr = N.kd_tree_arrays(nd.ctypes.data, nv.ctypes.data, nl.ctypes.data, nr.ctypes.data, nc.ctypes.data,
                               coords.ctypes.data, ids.ctypes.data, None)
        h = C.c_void_p()
        N.check(N.lib.kd_tree_import(C.byref(arr), nd.shape[0], pts.count, pts.dims, int(self.depth), dtype,
                                     device, C.byref(h)))
        self._import_dev = N.NativeTree(h.value)
        return self._import_dev


def _f32_exact(coords: np.ndarray) -> bool:
    """True when every binary64 coordinate is exactly a binary32 value (then the
    device stores float32: half the bytes, identical arithmetic after upcast)."""
    if coords.size == 0:
        return True
    with np.errstate(over="ignore"):
        c32 = coords.astype(np.float32)
    return bool(np.array_equal(c32.astype(np.float64), coords))


def _wrap(h: int) -> LocalTree:
    nt = N.NativeTree(h)
    return LocalTree(_native=nt, _info=nt.info())


def build_local_tree(points: PointSet, cfg: BuildConfig, timings: dict | None = None,
                     device: int = 0) -> LocalTree:
    """GPU build_local_tree (local_tree.py:436-574); identical output for any
    ``cfg.workers``.  ``timings`` receives 'pack' (fused into the build, 0.0),
    'device_ms' (CUDA-event time of the build) and 'wall' seconds."""
    coords = np.ascontiguousarray(points.coords, dtype=np.float64)
    ids = np.ascontiguousarray(points.ids, dtype=np.uint64)
    d, n = coords.shape
    t0 = time.perf_counter()
    if _f32_exact(coords):
        buf, dtype = np.ascontiguousarray(coords.astype(np.float32)), N.KD_F32
    else:
        buf, dtype = coords, N.KD_F64
    h = C.c_void_p()
    cfgn = cfg.native()
    N.check(N.lib.kd_tree_build(buf.ctypes.data if n else None, dtype, n, d, ids.ctypes.data if n else None,
                                C.byref(cfgn), device, 0, None, C.byref(h)))
    tree = _wrap(h.value)
    if timings is not None:
        timings["pack"] = 0.0
        timings["device_ms"] = float(tree._info.build_ms)
        timings["wall"] = time.perf_counter() - t0
    return tree


def build_local_tree_device(coords, ids=None, cfg: BuildConfig = BuildConfig(), stream=None) -> LocalTree:
    """Build from device-resident torch tensors: coords (dims, n) float32/float64
    CUDA tensor (SoA), ids (n,) int64/uint64 CUDA tensor or None (ids = row)."""
    import torch
    if coords.dim() != 2 or not coords.is_cuda:
        raise ValueError("coords must be a (dims, n) CUDA tensor")
    coords = coords.contiguous()
    dtype = {torch.float32: N.KD_F32, torch.float64: N.KD_F64}.get(coords.dtype)
    if dtype is None:
        raise ValueError("coords must be float32 or float64")
    d, n = coords.shape
    if ids is not None:
        ids = ids.contiguous()
        if ids.shape != (n,) or ids.element_size() != 8 or not ids.is_cuda:
            raise ValueError("ids must be an (n,) 64-bit CUDA tensor")
    st = stream if stream is not None else torch.cuda.current_stream(coords.device).cuda_stream
    h = C.c_void_p()
    cfgn = cfg.native()
    N.check(N.lib.kd_tree_build(coords.data_ptr() if n else None, dtype, n, d,
                                ids.data_ptr() if ids is not None else None, C.byref(cfgn),
                                coords.device.index or 0, N.KD_DEVICE_PTRS, C.c_void_p(st), C.byref(h)))
    return _wrap(h.value)


def pack_buckets(points: PointSet, order) -> PointSet:
    """Columnar reorder by a bucket-contiguous permutation (local_tree.py:402-405)."""
    order = np.asarray(order, dtype=np.int64)
    return PointSet(np.ascontiguousarray(points.coords[:, order]), points.ids[order])
