"""ctypes binding of libkdtree_b200.so (include/kdtree_b200.h).

The product path has no CPU fallback: if the CUDA library is missing this
module raises at import, and every call surfaces the library's error code as
the reference's exception type (ValueError / MemoryError / RuntimeError,
SURVEY.md §8(b) "Errors").
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KDB_LIB_PATH") or os.path.join(_HERE, "libkdtree_b200.so")  # override: A/B builds

KD_OK, KD_EINVAL, KD_ECUDA, KD_EUNSUPPORTED, KD_ENOMEM = 0, -1, -2, -3, -4
KD_F32, KD_F64 = 1, 2
KD_DEVICE_PTRS, KD_NO_SORT, KD_THREAD_PER_QUERY, KD_KNN_PACKET, KD_KNN_REFERENCE = 1, 2, 4, 8, 16

EXPORTED = ("kd_version", "kd_last_error", "kd_device_count", "kd_tree_build", "kd_tree_import",
            "kd_tree_get_info", "kd_tree_export", "kd_knn", "kd_tree_free", "kd_histogram", "kd_split_rows",
            "kd_route", "kd_unpack_rows", "kd_merge_topk")


class kd_build_cfg(C.Structure):
    _fields_ = [("bucket_size", C.c_int64), ("local_sample_m", C.c_int64),
                ("variance_sample", C.c_int64), ("seed", C.c_uint64)]


class kd_tree_info(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n", C.c_int64), ("n_leaves", C.c_int64), ("depth", C.c_int64),
                ("dims", C.c_int32), ("dtype", C.c_int32), ("device", C.c_int32), ("reserved", C.c_int32),
                ("build_ms", C.c_double), ("build_levels", C.c_int64), ("build_tasks", C.c_int64),
                ("build_slow_nodes", C.c_int64), ("build_ms_levels", C.c_double),
                ("build_ms_subtree", C.c_double), ("build_ms_finish", C.c_double)]


class kd_tree_arrays(C.Structure):
    _fields_ = [("node_dim", C.c_void_p), ("node_value", C.c_void_p), ("node_left", C.c_void_p),
                ("node_right", C.c_void_p), ("node_count", C.c_void_p), ("coords", C.c_void_p),
                ("ids", C.c_void_p), ("perm", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA library {LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.kd_version.restype = C.c_int
    L.kd_last_error.restype = C.c_char_p
    L.kd_device_count.argtypes = [C.POINTER(C.c_int)]
    L.kd_tree_build.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.POINTER(kd_build_cfg),
                                C.c_int, C.c_uint, C.c_void_p, C.POINTER(C.c_void_p)]
    L.kd_tree_import.argtypes = [C.POINTER(kd_tree_arrays), C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int,
                                 C.c_int, C.POINTER(C.c_void_p)]
    L.kd_tree_get_info.argtypes = [C.c_void_p, C.POINTER(kd_tree_info)]
    L.kd_tree_export.argtypes = [C.c_void_p, C.POINTER(kd_tree_arrays)]
    L.kd_knn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p]
    L.kd_tree_free.argtypes = [C.c_void_p]
    ab = os.environ.get("KDB_LIB_PATH") is not None  # an A/B build may predate some entry points
    for name, types in (("kd_histogram", [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_uint, C.c_void_p]),
                        ("kd_split_rows", [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_double,
                                           C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p]),
                        ("kd_unpack_rows", [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_uint, C.c_void_p]),
                        ("kd_merge_topk", [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                           C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint,
                                           C.c_void_p]),
                        ("kd_route", [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint,
                                      C.c_void_p])):
        if ab and not hasattr(L, name):
            continue
        getattr(L, name).argtypes = types
    if ab:
        return L
    for name in EXPORTED:
        getattr(L, name)
    return L


lib = _load()


def check(code: int) -> None:
    if code == KD_OK:
        return
    msg = (lib.kd_last_error() or b"").decode(errors="replace")
    if code in (KD_EINVAL, KD_EUNSUPPORTED):
        raise ValueError(msg)
    if code == KD_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def device_count() -> int:
    n = C.c_int(0)
    rc = lib.kd_device_count(C.byref(n))
    return n.value if rc == KD_OK else 0


class NativeTree:
    """Owning handle of a device-resident tree."""

    def __init__(self, handle: int):
        self.handle = C.c_void_p(handle)

    def info(self) -> kd_tree_info:
        inf = kd_tree_info()
        check(lib.kd_tree_get_info(self.handle, C.byref(inf)))
        return inf

    def close(self):
        if self.handle and self.handle.value:
            lib.kd_tree_free(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
