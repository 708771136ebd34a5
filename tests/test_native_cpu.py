"""CPU-side checks of the boundary: the CUDA library loads without a GPU, exports
every symbol include/kdtree_b200.h declares, and the host layer validates like
the reference (same exception types) before any device work."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "kdtree_b200.h")).read()
    return re.findall(r"KD_API\s+[\w\s\*]+?\b(kd_\w+)\s*\(", src)


def test_header_declares_entry_points():
    syms = header_symbols()
    assert set(syms) >= {"kd_tree_build", "kd_knn", "kd_tree_import", "kd_tree_export", "kd_tree_free"}


def test_library_exports_every_declared_symbol():
    from paper_1607_08220_b200 import _native as N
    lib = C.CDLL(N.LIB_PATH)
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert set(N.EXPORTED) == set(header_symbols())
    assert N.lib.kd_version() >= 10000


def test_flag_constants_match_header():
    from paper_1607_08220_b200 import _native as N
    src = open(os.path.join(ROOT, "include", "kdtree_b200.h")).read()
    flags = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(KD_[A-Z_]+)\s+(\d+)u", src)}
    assert flags == {"KD_DEVICE_PTRS": N.KD_DEVICE_PTRS, "KD_NO_SORT": N.KD_NO_SORT,
                     "KD_THREAD_PER_QUERY": N.KD_THREAD_PER_QUERY, "KD_KNN_PACKET": N.KD_KNN_PACKET,
                     "KD_KNN_REFERENCE": N.KD_KNN_REFERENCE}
    assert len(set(flags.values())) == len(flags) and all(v & (v - 1) == 0 for v in flags.values())


def test_library_is_sm100a():
    from paper_1607_08220_b200 import _native as N
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    from paper_1607_08220_b200 import _native as N
    assert C.sizeof(N.kd_build_cfg) == 32
    assert C.sizeof(N.kd_tree_info) == 4 * 8 + 4 * 4 + 8 + 3 * 8 + 3 * 8
    assert C.sizeof(N.kd_tree_arrays) == 8 * 8


def test_c_abi_rejects_bad_arguments_without_gpu():
    from paper_1607_08220_b200 import _native as N
    h = C.c_void_p()
    cfg = N.kd_build_cfg(0, 1024, 1024, 0)  # bucket 0
    rc = N.lib.kd_tree_build(None, N.KD_F32, 10, 3, None, C.byref(cfg), 0, 0, None, C.byref(h))
    assert rc == N.KD_EINVAL
    with pytest.raises(ValueError):
        N.check(rc)
    cfg = N.kd_build_cfg(32, 4096, 1024, 0)
    rc = N.lib.kd_tree_build(None, N.KD_F32, 0, 3, None, C.byref(cfg), 0, 0, None, C.byref(h))
    assert rc == N.KD_EUNSUPPORTED
    rc = N.lib.kd_knn(None, None, 0, 5, None, None, None, None, None, None, 0, None)
    assert rc == N.KD_EINVAL


def test_build_config_validation_matches_reference():
    from paper_1607_08220_b200.local_tree import BuildConfig
    cfg = BuildConfig()
    assert (cfg.bucket_size, cfg.local_sample_m, cfg.branch_factor_per_worker) == (32, 1024, 10)
    for bad in (dict(bucket_size=0), dict(workers=0), dict(local_sample_m=0), dict(branch_factor_per_worker=0)):
        with pytest.raises(ValueError):
            BuildConfig(**bad)


def test_find_knn_batch_validates_before_device():
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.local_query import find_knn_batch
    from paper_1607_08220_b200.local_tree import LocalTree
    ps = PointSet.from_rows(np.random.default_rng(0).uniform(size=(10, 2)))
    tree = LocalTree(np.array([-1], np.int32), np.zeros(1), np.array([0], np.int32), np.array([10], np.int32),
                     np.array([10]), ps, 0, np.array([0]), np.array([10]))
    with pytest.raises(ValueError):
        find_knn_batch(tree, np.zeros((1, 2)), 0)
    with pytest.raises(ValueError):
        find_knn_batch(tree, np.zeros(2), 1)
    with pytest.raises(ValueError):
        find_knn_batch(tree, np.zeros((1, 3)), 1)


def test_f32_exactness_detection():
    from paper_1607_08220_b200.local_tree import _f32_exact
    assert _f32_exact(np.random.default_rng(0).random((3, 100), dtype=np.float32).astype(np.float64))
    assert not _f32_exact(np.random.default_rng(0).uniform(size=(3, 100)))


def test_pointset_contract():
    from paper_1607_08220_b200.core import PointSet, squared_distance, min_sq_dist_to_region, Region
    with pytest.raises(ValueError):
        PointSet.from_rows([[0.0, np.nan]])
    with pytest.raises(ValueError):
        PointSet.from_rows([[0.0], [1.0]], ids=np.array([7, 7], dtype=np.uint64))
    assert squared_distance(np.array([0.0, 0.0]), np.array([3.0, 4.0])) == 25.0
    assert min_sq_dist_to_region(np.array([12.0, 13.0]), Region(np.zeros(2), np.full(2, 10.0))) == 13.0
