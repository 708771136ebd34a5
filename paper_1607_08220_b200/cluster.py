"""Global spatial partition across GPUs (drop-in for ``kdknn.cluster``).

The top log2(P) levels of the kd-tree split the points across ranks (PAPER.md
"global kd-tree"; reference cluster.py:354-417).  Same result as the
reference -- planes, per-rank point sets and their order, hence local trees and
engine bundles byte-identical -- but organised around device collectives
instead of the reference's per-group message exchange:

per level (groups of G = P >> level consecutive ranks, all groups at once):

1. every rank draws its 256-point sample (SplitMix64 Fisher-Yates, median.py:74-85)
   and ONE ``all_gather`` of fixed-size sample tensors gives every rank every
   group's sample;
2. every rank derives, for every group, the max-variance dimension order and the
   distinct sampled values (numpy on a few KB, the reference's exact arithmetic);
3. rounds over candidate dimensions: each rank histograms ALL its points of the
   round's dimension against its group's boundaries on the GPU
   (``kd_histogram``: counts + exact-equal counts), writes them into its group's
   segment of one buffer, and ONE ``all_reduce`` (NCCL) sums every group at once
   (cluster.py:246-248 group_sum_reduce).  Every rank then decides every group's
   plane with the reference's rule (median.py:143-166 closest-to-half boundary,
   the inclusive ``nextafter`` fallback of cluster.py:262-273, next dimension) --
   so no plane all-gather is needed and an unsplittable group raises on every
   rank together;
4. redistribution (cluster.py:281-351 semantics): ``kd_split_rows`` writes the
   rank's points as packed rows, low side first, stable; an ``all_gather`` of the
   (low, high) counts lets every rank compute the balanced contiguous-slice plan;
   ONE ``alltoallv`` moves the rows (NCCL over NVLink) and ``kd_unpack_rows``
   restores SoA.  Received blocks arrive in sender-rank order, the reference's
   concatenation order.

Per level the host reads back the samples, the summed histograms and the counts
(small tensors); all point data stays on the device.
"""

from __future__ import annotations

import ctypes as C
import struct
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .comm import run_ranks
from .core import PointSet, Region, SplitPlane, min_sq_dist_to_region

__all__ = ["ClusterConfig", "GlobalTree", "RankState", "UnsplittableDataError", "build_global_tree",
           "choose_global_split_dimension", "redistribute", "owner_of", "ranks_within", "sample_points",
           "derive_seed", "sample_indices", "DevicePoints", "CudaBackend", "rank_build_global", "DeviceRegions"]

_M64 = 0xFFFFFFFFFFFFFFFF
_GAMMA = 0x9E3779B97F4A7C15
_GLOBAL_PATH_TAG = 1 << 40   # cluster.py:54
_SALT_GLOBAL_SAMPLE = 101    # cluster.py:55


class UnsplittableDataError(RuntimeError):
    """A rank group holds >= 2 points identical in every dimension (cluster.py:58-59)."""


def _mix64(z: int) -> int:
    z = (z + _GAMMA) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_seed(seed: int, path: int, salt: int) -> int:
    """median.py:189-194 / :69-71 -- per-node sub-seed, u64 wraparound."""
    return _mix64((seed & _M64) ^ _mix64(path & _M64) ^ _mix64(((salt & _M64) * _GAMMA) & _M64))


def sample_indices(n: int, m: int, seed: int) -> np.ndarray:
    """median.py:74-85: m draws of a partial Fisher-Yates over 0..n-1 (sparse swap map)."""
    state = seed & _M64
    swapped: dict[int, int] = {}
    out = np.empty(m, dtype=np.int64)
    for j in range(m):
        state = (state + _GAMMA) & _M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        z ^= z >> 31
        r = j + z % (n - j)
        vj, vr = swapped.get(j, j), swapped.get(r, r)
        swapped[j], swapped[r] = vr, vj
        out[j] = vr
    return out


@dataclass(frozen=True)
class ClusterConfig:
    """cluster.py:62-72."""

    global_sample_m: int = 256
    seed: int = 0
    workers: int = 1

    def __post_init__(self):
        if self.global_sample_m < 1:
            raise ValueError("global_sample_m must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


@dataclass(frozen=True, eq=False)
class GlobalTree:
    """Complete binary partition tree with P leaves (cluster.py:75-169); planes
    in heap order, leaf i = rank i, ties go right."""

    dims: int
    plane_dims: np.ndarray
    plane_values: np.ndarray

    @property
    def rank_count(self) -> int:
        return int(self.plane_dims.shape[0]) + 1

    @property
    def levels(self) -> int:
        return self.rank_count.bit_length() - 1

    def owner_of(self, q) -> int:
        idx, npl = 0, self.plane_dims.shape[0]
        while idx < npl:
            idx = 2 * idx + 1 + (0 if q[self.plane_dims[idx]] < self.plane_values[idx] else 1)
        return idx - npl

    def owner_of_batch(self, queries) -> np.ndarray:
        queries = np.asarray(queries, dtype=np.float64)
        heap = np.zeros(queries.shape[0], dtype=np.int64)
        rows = np.arange(queries.shape[0])
        for _ in range(self.levels):
            go_right = queries[rows, self.plane_dims[heap]] >= self.plane_values[heap]
            heap = 2 * heap + 1 + go_right
        return heap - self.plane_dims.shape[0]

    def region_of(self, rank: int) -> Region:
        region = Region.unbounded(self.dims)
        idx = 0
        for lv in range(self.levels):
            high = (rank >> (self.levels - 1 - lv)) & 1
            lo_half, hi_half = region.split(SplitPlane(int(self.plane_dims[idx]), float(self.plane_values[idx])))
            region = hi_half if high else lo_half
            idx = 2 * idx + 1 + high
        return region

    def regions(self) -> list:
        return [self.region_of(r) for r in range(self.rank_count)]

    def region_bounds(self) -> tuple[np.ndarray, np.ndarray]:
        regs = self.regions()
        return (np.ascontiguousarray(np.stack([r.lower for r in regs]), dtype=np.float64),
                np.ascontiguousarray(np.stack([r.upper for r in regs]), dtype=np.float64))

    def ranks_within(self, q, sq_radius: float) -> np.ndarray:
        """Ranks (owner excluded) whose region is strictly closer than the radius."""
        owner = self.owner_of(q)
        return np.asarray([r for r in range(self.rank_count)
                           if r != owner and min_sq_dist_to_region(q, self.region_of(r)) < sq_radius],
                          dtype=np.int64)

    def to_bytes(self) -> bytes:
        return (struct.pack("<II", self.dims, self.rank_count)
                + np.ascontiguousarray(self.plane_dims, dtype="<i4").tobytes()
                + np.ascontiguousarray(self.plane_values, dtype="<f8").tobytes())

    @staticmethod
    def from_bytes(blob: bytes) -> "GlobalTree":
        dims, p = struct.unpack_from("<II", blob, 0)
        pdim = np.frombuffer(blob, dtype="<i4", count=p - 1, offset=8).astype(np.int32)
        pval = np.frombuffer(blob, dtype="<f8", count=p - 1, offset=8 + 4 * (p - 1)).astype(np.float64)
        return GlobalTree(int(dims), pdim, pval)


def owner_of(gt: GlobalTree, q) -> int:
    return gt.owner_of(np.asarray(q, dtype=np.float64))


def ranks_within(gt: GlobalTree, q, sq_radius) -> np.ndarray:
    return gt.ranks_within(np.asarray(q, dtype=np.float64), float(sq_radius))


# ---------------------------------------------------------------------------------------------
class DevicePoints:
    """A rank's points on its device: coords (dims, n) float32|float64 SoA + int64 ids (uint64 bits)."""

    def __init__(self, coords, ids):
        self.coords = coords
        self.ids = ids

    @property
    def count(self) -> int:
        return int(self.coords.shape[1])

    @property
    def dims(self) -> int:
        return int(self.coords.shape[0])

    @staticmethod
    def from_pointset(ps: PointSet, device, f32: bool) -> "DevicePoints":
        import torch
        c = torch.as_tensor(np.ascontiguousarray(ps.coords, dtype=np.float32 if f32 else np.float64))
        i = torch.as_tensor(np.ascontiguousarray(ps.ids, dtype=np.uint64).view(np.int64))
        return DevicePoints(c.to(device), i.to(device))

    def to_pointset(self) -> PointSet:
        c = self.coords.double().cpu().numpy()
        i = self.ids.cpu().numpy().view(np.uint64)
        return PointSet(np.ascontiguousarray(c), np.ascontiguousarray(i))

    def take(self, sel):
        return DevicePoints(self.coords[:, sel].contiguous(), self.ids[sel].contiguous())


class DeviceRegions:
    """The replicated global tree on a rank's device: planes + region boxes."""

    def __init__(self, gt: GlobalTree, device):
        import torch
        self.p = gt.rank_count
        self.dims = gt.dims
        lo, hi = gt.region_bounds()
        self.pdim = torch.as_tensor(np.ascontiguousarray(gt.plane_dims, dtype=np.int32)).to(device)
        self.pval = torch.as_tensor(np.ascontiguousarray(gt.plane_values, dtype=np.float64)).to(device)
        self.lo = torch.as_tensor(lo).to(device)
        self.hi = torch.as_tensor(hi).to(device)


def _dtype_code(coords) -> int:
    import torch
    return N.KD_F32 if coords.dtype == torch.float32 else N.KD_F64


def _stream(t):
    import torch
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


class CudaBackend:
    """Rank-local device work of the global tier: the sm_100a kernels behind the C-ABI.
    Every method only enqueues work on the current stream and returns device tensors."""

    name = "cuda"

    def histogram(self, pts: DevicePoints, dim: int, boundaries: np.ndarray):
        """(counts (nb+1,), equals (nb,)) int64 device tensors (median.py:243-265)."""
        import torch
        dev = pts.coords.device
        nb = int(boundaries.shape[0])
        out = torch.zeros(2 * nb + 1, dtype=torch.int64, device=dev)
        if pts.count:
            b = torch.as_tensor(np.ascontiguousarray(boundaries, dtype=np.float64)).to(dev)
            N.check(N.lib.kd_histogram(pts.coords[dim].data_ptr(), _dtype_code(pts.coords), pts.count,
                                       b.data_ptr(), nb, out.data_ptr(), out[nb + 1:].data_ptr(),
                                       N.KD_DEVICE_PTRS, _stream(pts.coords)))
        return out[:nb + 1], out[nb + 1:]

    def split_rows(self, pts: DevicePoints, dim: int, value: float):
        """Packed rows (low side first, stable) + the low-side count (1,) on the device."""
        import torch
        dev = pts.coords.device
        es = pts.coords.element_size()
        w = ((pts.dims * es + 7) // 8) * 8 + 8
        rows = torch.empty((pts.count, w), dtype=torch.uint8, device=dev)
        n_low = torch.zeros(1, dtype=torch.int64, device=dev)
        N.check(N.lib.kd_split_rows(pts.coords.data_ptr(), _dtype_code(pts.coords), pts.count, pts.dims,
                                    pts.ids.data_ptr(), dim, float(value), rows.data_ptr(), n_low.data_ptr(),
                                    N.KD_DEVICE_PTRS, _stream(pts.coords)))
        return rows, n_low

    def unpack_rows(self, rows, dims: int, dtype) -> DevicePoints:
        import torch
        n = rows.shape[0]
        coords = torch.empty((dims, n), dtype=dtype, device=rows.device)
        ids = torch.empty(n, dtype=torch.int64, device=rows.device)
        if n:
            N.check(N.lib.kd_unpack_rows(rows.data_ptr(), n, dims, _dtype_code(coords), coords.data_ptr(),
                                         ids.data_ptr(), N.KD_DEVICE_PTRS, _stream(rows)))
        return DevicePoints(coords, ids)

    def build(self, pts: DevicePoints, build_cfg):
        from .local_tree import build_local_tree_device
        return build_local_tree_device(pts.coords, pts.ids, build_cfg)

    def knn(self, tree, q, k: int, radii=None, excl=None, counters: bool = False):
        """(dists (m,k) f64, ids (m,k) int64 bits of u64, counts (m,), counters (m,3)|None) on the device."""
        import torch
        from .local_query import find_knn_device
        m = q.shape[0]
        if m == 0 or tree.count == 0:
            z = torch.zeros
            return (z((m, k), dtype=torch.float64, device=q.device), z((m, k), dtype=torch.int64, device=q.device),
                    z(m, dtype=torch.int64, device=q.device),
                    z((m, 3), dtype=torch.int64, device=q.device) if counters else None)
        return find_knn_device(tree, q.contiguous(), k, radii=radii, exclude_ids=excl, counters=counters)

    def route(self, regions: DeviceRegions, q, radii=None, within: bool = False):
        """(owner rank int32 (m,), bitmask of other ranks within r (m,) int64 | None)."""
        import torch
        m = q.shape[0]
        owner = torch.zeros(m, dtype=torch.int32, device=q.device)
        wm = torch.zeros(m, dtype=torch.int64, device=q.device) if within else None
        if m:
            N.check(N.lib.kd_route(regions.pdim.data_ptr() if regions.p > 1 else None,
                                   regions.pval.data_ptr() if regions.p > 1 else None, regions.p,
                                   regions.lo.data_ptr(), regions.hi.data_ptr(), q.contiguous().data_ptr(), m,
                                   regions.dims, radii.data_ptr() if radii is not None else None, owner.data_ptr(),
                                   wm.data_ptr() if within else None, N.KD_DEVICE_PTRS, _stream(q)))
        return owner, wm

    def merge(self, k: int, ld, li, lc, my_rank: int, slot, rd, ri, rc, rrank):
        """kd_merge_topk: (dists, ids, ranks int32, counts, duplicate flag (1,) int32) on the device."""
        import torch
        m = ld.shape[0]
        dev = ld.device
        od = torch.zeros((m, k), dtype=torch.float64, device=dev)
        oi = torch.zeros((m, k), dtype=torch.int64, device=dev)
        orank = torch.zeros((m, k), dtype=torch.int32, device=dev)
        oc = torch.zeros(m, dtype=torch.int64, device=dev)
        dup = torch.zeros(1, dtype=torch.int32, device=dev)
        nr = slot.shape[0]
        if m:
            N.check(N.lib.kd_merge_topk(m, k, ld.data_ptr(), li.data_ptr(), lc.data_ptr(), my_rank, nr,
                                        slot.data_ptr() if nr else None, rd.data_ptr() if nr else None,
                                        ri.data_ptr() if nr else None, rc.data_ptr() if nr else None,
                                        rrank.data_ptr() if nr else None, od.data_ptr(), oi.data_ptr(),
                                        orank.data_ptr(), oc.data_ptr(), dup.data_ptr(), N.KD_DEVICE_PTRS,
                                        _stream(ld)))
        return od, oi, orank, oc, dup


_CUDA = CudaBackend()


def sample_points(pts, m: int, seed: int):
    """min(m, n) points without replacement, deterministically (cluster.py:190-198)."""
    n = pts.count
    if n == 0:
        return pts.take(np.empty(0, dtype=np.int64)) if isinstance(pts, PointSet) else None
    picked = sample_indices(n, min(m, n), seed)
    if isinstance(pts, PointSet):
        return pts.take(picked)
    import torch
    return pts.take(torch.as_tensor(picked, device=pts.coords.device))


# ---------------------------------------------------------------------------------------------
def _median_split(boundaries: np.ndarray, g_counts: np.ndarray, g_equals: np.ndarray, group_n: int):
    """The reference's plane rule for one candidate dimension (cluster.py:253-273 with
    median.py:143-166): the boundary whose cumulative fraction is closest to 1/2
    (first minimum), accepted when both sides are non-empty; else the best
    non-degenerate cut at a boundary (exclusive) or just above it (inclusive,
    nextafter); None when the dimension is constant over the group."""
    nb = boundaries.shape[0]
    cum = np.cumsum(g_counts[:nb])
    total = int(g_counts.sum())
    if total > 0 and nb > 0:
        i = int(np.argmin(np.abs(cum / total - 0.5)))
        below = int(cum[i])
        if group_n < 2 or 0 < below < group_n:
            return float(boundaries[i])
    le = cum + g_equals[:nb]
    best_diff, best_value = None, None
    for i in range(nb):
        for value, below in ((boundaries[i], cum[i]), (np.nextafter(boundaries[i], np.inf), le[i])):
            if 0 < below < group_n:
                diff = abs(int(below) / group_n - 0.5)
                if best_diff is None or diff < best_diff:
                    best_diff, best_value = diff, float(value)
    return best_value


def _level_planes(comm, pts: DevicePoints, cfg: ClusterConfig, level: int, backend) -> dict:
    """Every group's plane at this level, decided identically on every rank."""
    import torch
    p, me, dims = comm.size, comm.rank, pts.dims
    gsize = p >> level
    ngroups = p // gsize
    mine = me // gsize
    dev = pts.coords.device
    m = cfg.global_sample_m
    # 1. samples: one fixed-size all-gather for all groups
    seed = derive_seed(cfg.seed, _GLOBAL_PATH_TAG + level, _SALT_GLOBAL_SAMPLE + me)
    take = min(m, pts.count)
    sbuf = torch.zeros((m + 1, dims), dtype=torch.float64, device=dev)
    if take:
        idx = torch.as_tensor(sample_indices(pts.count, take, seed), device=dev)
        sbuf[:take] = pts.coords[:, idx].t().double()
    sbuf[m, 0] = take
    allS = comm.all_gather_t(sbuf).cpu().numpy()
    rows, order = {}, {}
    for g in range(ngroups):
        parts = [allS[r, :int(allS[r, m, 0])] for r in range(g * gsize, (g + 1) * gsize)]
        rows[g] = np.concatenate(parts, axis=0)
        if rows[g].shape[0]:
            order[g] = np.argsort(-np.var(rows[g], axis=0), kind="mergesort")
    # an empty group keeps well-formed regions with any plane (cluster.py:231-235)
    planes = {g: SplitPlane(0, 0.0) for g in range(ngroups) if rows[g].shape[0] == 0}
    # 2. rounds over candidate dimensions; one all-reduce sums every group's histogram
    for rnd in range(dims):
        todo = [g for g in range(ngroups) if g not in planes]
        if not todo:
            break
        bnd = {g: np.unique(rows[g][:, int(order[g][rnd])]) for g in todo}
        nbm = max(b.shape[0] for b in bnd.values())
        hist = torch.zeros((ngroups, 2 * nbm + 2), dtype=torch.int64, device=dev)
        if mine in bnd:
            nb = bnd[mine].shape[0]
            counts, equals = backend.histogram(pts, int(order[mine][rnd]), bnd[mine])
            hist[mine, :nb + 1] = counts
            hist[mine, nbm + 1:nbm + 1 + nb] = equals
            hist[mine, -1] = pts.count
        red = comm.all_reduce_t(hist).cpu().numpy()
        for g in todo:
            nb = bnd[g].shape[0]
            group_n = int(red[g, -1])
            if group_n == 0:
                planes[g] = SplitPlane(0, 0.0)
                continue
            v = _median_split(bnd[g], red[g, :nb + 1], red[g, nbm + 1:nbm + 1 + nb], group_n)
            if v is not None:
                planes[g] = SplitPlane(int(order[g][rnd]), v)
    bad = [g for g in range(ngroups) if g not in planes]
    if bad:
        g = bad[0]
        raise UnsplittableDataError(
            f"rank group {tuple(range(g * gsize, (g + 1) * gsize))} at level {level} holds points identical "
            f"in every of {dims} dimensions; cannot split into nonempty halves")
    return planes


def _slice_plan(counts: np.ndarray, group: range, me: int) -> np.ndarray:
    """Rows this rank sends to each rank (cluster.py:302-346 contiguous-slice plan):
    each side's points form a virtual sequence ordered by (sender rank, stable
    local order); its receivers (lower / upper half of the group) take slices of
    total//H (+1 for the first total%H).  Returns send counts per rank, in the
    order the rows sit in this rank's split buffer (low side, then high side)."""
    send = np.zeros(counts.shape[0], dtype=np.int64)
    half = len(group) // 2
    for side, recv in ((0, list(group)[:half]), (1, list(group)[half:])):
        sizes = [int(counts[r, side]) for r in group]
        total = sum(sizes)
        share, rem = divmod(total, len(recv))
        my0 = sum(sizes[:group.index(me)])
        my1 = my0 + sizes[group.index(me)]
        r0 = 0
        for i, r in enumerate(recv):
            r1 = r0 + share + (1 if i < rem else 0)
            send[r] += max(0, min(my1, r1) - max(my0, r0))
            r0 = r1
    return send


def redistribute(comm, group, pts: DevicePoints, plane: SplitPlane, backend=_CUDA) -> tuple[DevicePoints, int]:
    """Exchange points inside `group` (consecutive ranks) so its lower half holds
    coord < value (cluster.py:281-351 semantics).  Returns (new points, rows sent)."""
    import torch
    group = range(group[0], group[-1] + 1)
    rows, n_low = backend.split_rows(pts, plane.dim, plane.value)
    counts = comm.all_gather_t(torch.cat([n_low, n_low.new_full((1,), pts.count) - n_low])).cpu().numpy()
    send = _slice_plan(counts, group, comm.rank)
    recv, _ = comm.alltoallv(rows, send.tolist())
    return backend.unpack_rows(recv, pts.dims, pts.coords.dtype), int(send.sum() - send[comm.rank])


def rank_build_global(comm, pts: DevicePoints, cfg: ClusterConfig, backend=_CUDA):
    """One rank's side of the global construction (SPMD, cluster.py:354-389
    semantics).  Returns (GlobalTree, this rank's points, stats)."""
    import torch
    p, me = comm.size, comm.rank
    levels = p.bit_length() - 1
    dims = pts.dims
    plane_dims = np.full(max(p - 1, 0), -1, dtype=np.int32)
    plane_values = np.zeros(max(p - 1, 0), dtype=np.float64)
    stats = {"points_moved": 0, "t_global_split": 0.0, "t_redistribute": 0.0}
    for level in range(levels):
        t0 = time.perf_counter()
        planes = _level_planes(comm, pts, cfg, level, backend)
        for g, pl in planes.items():
            plane_dims[(1 << level) - 1 + g] = pl.dim
            plane_values[(1 << level) - 1 + g] = pl.value
        stats["t_global_split"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        gsize = p >> level
        group = range((me // gsize) * gsize, (me // gsize + 1) * gsize)
        pts, sent = redistribute(comm, group, pts, planes[me // gsize], backend)
        stats["points_moved"] += sent
        stats["t_redistribute"] += time.perf_counter() - t0
    gt = GlobalTree(dims, plane_dims, plane_values)
    if pts.count and levels:
        reg = gt.region_of(me)
        lo = torch.as_tensor(reg.lower, device=pts.coords.device)[:, None]
        hi = torch.as_tensor(reg.upper, device=pts.coords.device)[:, None]
        c = pts.coords
        if c.dtype != torch.float64:
            # region bounds are split values, i.e. coordinates: when they are exact in the storage type
            # the check runs on the stored values (no binary64 copy of the rank's points per build)
            lo_c, hi_c = lo.to(c.dtype), hi.to(c.dtype)
            if bool((lo_c.double() == lo).all()) and bool((hi_c.double() == hi).all()):
                lo, hi = lo_c, hi_c
            else:
                c = c.double()
        if bool(((c < lo) | (c > hi)).any()):
            raise AssertionError(f"rank {me}: point outside its region after redistribution")
    return gt, pts, stats


def choose_global_split_dimension(comm, pts: DevicePoints, cfg: ClusterConfig, level: int = 0) -> int:
    """Max-variance dimension of this rank's group sample (cluster.py:214-225)."""
    import torch
    p, me, dims = comm.size, comm.rank, pts.dims
    gsize = p >> level
    m = cfg.global_sample_m
    seed = derive_seed(cfg.seed, _GLOBAL_PATH_TAG + level, _SALT_GLOBAL_SAMPLE + me)
    take = min(m, pts.count)
    sbuf = torch.zeros((m + 1, dims), dtype=torch.float64, device=pts.coords.device)
    if take:
        sbuf[:take] = pts.coords[:, torch.as_tensor(sample_indices(pts.count, take, seed),
                                                    device=pts.coords.device)].t().double()
    sbuf[m, 0] = take
    allS = comm.all_gather_t(sbuf).cpu().numpy()
    g0 = (me // gsize) * gsize
    rows = np.concatenate([allS[r, :int(allS[r, m, 0])] for r in range(g0, g0 + gsize)], axis=0)
    if rows.shape[0] == 0:
        return 0
    return int(np.argsort(-np.var(rows, axis=0), kind="mergesort")[0])


@dataclass
class RankState:
    """Everything one rank holds after construction (cluster.py:172-179)."""

    rank: int
    points: PointSet
    global_tree: GlobalTree
    tree: object = None


def _f32_all(parts) -> bool:
    from .local_tree import _f32_exact
    return all(_f32_exact(p.coords) for p in parts)


def _check_inputs(points_per_rank: list):
    p = len(points_per_rank)
    if p < 1 or (p & (p - 1)) != 0:
        raise ValueError(f"rank count {p} is not a power of two")
    if len({ps.dims for ps in points_per_rank}) != 1:
        raise ValueError("inconsistent dimensionality across ranks")
    if sum(ps.count for ps in points_per_rank) == 0:
        raise ValueError("empty dataset")


def build_global_device(points_per_rank: list, cfg: ClusterConfig, backend=_CUDA):
    """The global tier over in-process ranks, every rank's points kept on its device.
    Returns (per-rank DevicePoints, GlobalTree, per-rank stats)."""
    _check_inputs(points_per_rank)
    f32 = _f32_all(points_per_rank)

    def prog(comm, ps):
        return rank_build_global(comm, DevicePoints.from_pointset(ps, comm.device, f32), cfg, backend)

    res = run_ranks(len(points_per_rank), prog, [(ps,) for ps in points_per_rank])
    blobs = {r[0].to_bytes() for r in res}
    if len(blobs) != 1:
        raise AssertionError("global tree replicas differ across ranks")
    return [r[1] for r in res], res[0][0], [r[2] for r in res]


def build_global_tree(points_per_rank: list, cfg: ClusterConfig, backend=_CUDA):
    """cluster.py:392-417 driver: (GlobalTree, redistributed per-rank PointSets, stats)."""
    _check_inputs(points_per_rank)
    if len(points_per_rank) == 1:
        gt = GlobalTree(points_per_rank[0].dims, np.empty(0, dtype=np.int32), np.empty(0, dtype=np.float64))
        return gt, list(points_per_rank), [{"points_moved": 0, "t_global_split": 0.0, "t_redistribute": 0.0}]
    dev_pts, gt, stats = build_global_device(points_per_rank, cfg, backend)
    return gt, [d.to_pointset() for d in dev_pts], stats
