"""Global spatial partition across GPUs (drop-in for ``kdknn.cluster``).

The top log2(P) levels of the kd-tree split the points across ranks
(cluster.py:354-417 of the reference): per level, every rank group all-gathers
a 256-point sample per rank, picks the max-variance dimension of the sample,
histograms ALL its local points against the distinct sampled values on the GPU
(``kd_histogram``), sum-reduces the histograms over the group and selects the
boundary closest to the median (same binary64 arithmetic as
median.py:143-166); degenerate splits fall back to inclusive candidates just
above a boundary, then to the next dimension.  Points are then exchanged so the
lower half of the group holds coord < value, balanced by the reference's
contiguous-slice plan (cluster.py:281-351): the stable device partition
(``kd_partition``) feeds an all-to-all of SoA point blocks (NCCL over NVLink in
the multi-process backend).  Every rank ends with exactly the points, in exactly
the order, the reference would give it -- so its local tree, and the engine
bundle, are byte-identical to the reference's.

Small control data (samples, histograms, planes, counts) is handled on the
host with numpy, exactly as the reference does.
"""

from __future__ import annotations

import ctypes as C
import struct
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .comm import ClusterAborted, run_ranks
from .core import PointSet, Region, SplitPlane, min_sq_dist_to_region

__all__ = ["ClusterConfig", "GlobalTree", "RankState", "UnsplittableDataError", "build_global_tree",
           "choose_global_split_dimension", "redistribute", "owner_of", "ranks_within", "sample_points",
           "derive_seed", "sample_indices", "DevicePoints", "CudaBackend", "rank_build_global"]

_M64 = 0xFFFFFFFFFFFFFFFF
_GAMMA = 0x9E3779B97F4A7C15
_GLOBAL_PATH_TAG = 1 << 40   # cluster.py:54
_SALT_GLOBAL_SAMPLE = 101    # cluster.py:55
STRIDE = 32


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
    """median.py:74-85 partial Fisher-Yates over arange(n) (sparse swap map)."""
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
        nq = queries.shape[0]
        idx = np.zeros(nq, dtype=np.int64)
        for _ in range(self.levels):
            d = self.plane_dims[idx]
            v = self.plane_values[idx]
            idx = 2 * idx + 1 + (queries[np.arange(nq), d] >= v).astype(np.int64)
        return idx - self.plane_dims.shape[0]

    def region_of(self, rank: int) -> Region:
        region = Region.unbounded(self.dims)
        idx, levels = 0, self.levels
        for lv in range(levels):
            bit = (rank >> (levels - 1 - lv)) & 1
            low, high = region.split(SplitPlane(int(self.plane_dims[idx]), float(self.plane_values[idx])))
            region = high if bit else low
            idx = 2 * idx + 1 + bit
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
        out = [r for r in range(self.rank_count)
               if r != owner and min_sq_dist_to_region(q, self.region_of(r)) < sq_radius]
        return np.asarray(sorted(out), dtype=np.int64)

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
    """A rank's points on its GPU: coords (dims, n) float32|float64 SoA + int64 ids (uint64 bits)."""

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

    def slice(self, a, b):
        return DevicePoints(self.coords[:, a:b].contiguous(), self.ids[a:b].contiguous())


def _dtype_code(coords) -> int:
    import torch
    return N.KD_F32 if coords.dtype == torch.float32 else N.KD_F64


class CudaBackend:
    """Rank-local device work of the global tier: the sm_100a kernels behind the C-ABI."""

    name = "cuda"

    def histogram(self, pts, dim, boundaries):
        return device_histogram(pts, dim, boundaries)

    def partition(self, pts, plane):
        return device_partition(pts, plane)

    def build(self, pts, build_cfg):
        from .local_tree import build_local_tree_device
        return build_local_tree_device(pts.coords, pts.ids, build_cfg)

    def knn(self, tree, queries, k, radii=None):
        """queries (m, D) float64 tensor on the tree's device -> host numpy
        (dists, ids u64, counts, counters)."""
        from .local_query import find_knn_device
        if queries.shape[0] == 0 or tree.count == 0:
            m = queries.shape[0]
            return (np.zeros((m, k)), np.zeros((m, k), np.uint64), np.zeros(m, np.int64), np.zeros((m, 3), np.int64))
        d, i, c, ctr = find_knn_device(tree, queries.contiguous(), k, radii=radii, counters=True)
        return d.cpu().numpy(), i.cpu().numpy().view(np.uint64), c.cpu().numpy(), ctr.cpu().numpy()


_CUDA = CudaBackend()


def device_histogram(pts: DevicePoints, dim: int, boundaries: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """histogram_with_equals of the rank's coordinate row `dim` on the GPU."""
    import torch
    nb = boundaries.shape[0]
    counts = np.zeros(nb + 1, dtype=np.int64)
    equals = np.zeros(nb, dtype=np.int64)
    if pts.count == 0:
        return counts, equals
    b = np.ascontiguousarray(boundaries, dtype=np.float64)
    row = pts.coords[dim]
    with torch.cuda.device(pts.coords.device):
        db = torch.as_tensor(b).to(pts.coords.device)
        dc = torch.empty(nb + 1, dtype=torch.int64, device=pts.coords.device)
        de = torch.empty(nb, dtype=torch.int64, device=pts.coords.device)
        st = torch.cuda.current_stream(pts.coords.device).cuda_stream
        N.check(N.lib.kd_histogram(row.data_ptr(), _dtype_code(pts.coords), pts.count, db.data_ptr(), nb,
                                   dc.data_ptr(), de.data_ptr(), N.KD_DEVICE_PTRS, C.c_void_p(st)))
        return dc.cpu().numpy(), de.cpu().numpy()


def device_partition(pts: DevicePoints, plane: SplitPlane) -> tuple[DevicePoints, int]:
    """Stable split: coord[dim] < value first (cluster.py:292-294)."""
    import torch
    if pts.count == 0:
        return pts, 0
    with torch.cuda.device(pts.coords.device):
        oc = torch.empty_like(pts.coords)
        oi = torch.empty_like(pts.ids)
        nl = C.c_int64(0)
        st = torch.cuda.current_stream(pts.coords.device).cuda_stream
        N.check(N.lib.kd_partition(pts.coords.data_ptr(), _dtype_code(pts.coords), pts.count, pts.dims,
                                   pts.ids.data_ptr(), plane.dim, float(plane.value), oc.data_ptr(), oi.data_ptr(),
                                   C.byref(nl), N.KD_DEVICE_PTRS, C.c_void_p(st)))
        return DevicePoints(oc, oi), int(nl.value)


def sample_points(pts, m: int, seed: int):
    """min(m, n) points without replacement, deterministically (cluster.py:190-198)."""
    n = pts.count
    if n == 0:
        return pts.take([]) if isinstance(pts, PointSet) else None
    picked = sample_indices(n, min(m, n), seed)
    if isinstance(pts, PointSet):
        return pts.take(picked)
    import torch
    return pts.take(torch.as_tensor(picked, device=pts.coords.device))


def _group_of(rank: int, p: int, level: int) -> tuple:
    g = p >> level
    base = (rank // g) * g
    return tuple(range(base, base + g))


def _gather_group_sample(comm, group, pts: DevicePoints, cfg: ClusterConfig, level: int) -> np.ndarray:
    seed = derive_seed(cfg.seed, _GLOBAL_PATH_TAG + level, _SALT_GLOBAL_SAMPLE + comm.rank)
    s = sample_points(pts, cfg.global_sample_m, seed)
    rows = s.coords.double().t().cpu().numpy() if s is not None and s.count else np.empty((0, pts.dims))
    parts = comm.all_gather(rows)
    rows = [parts[r] for r in group if parts[r].shape[0]]
    return np.concatenate(rows, axis=0) if rows else np.empty((0, pts.dims), dtype=np.float64)


def _select_median(boundaries: np.ndarray, counts: np.ndarray) -> tuple[int, int]:
    """median.py:143-166 in binary64 (first minimum == strict `<` ties-low)."""
    nb = boundaries.shape[0]
    total = int(counts.sum())
    if total <= 0 or nb == 0:
        return -1, 0
    cum = np.cumsum(counts[:nb])
    diff = np.abs(cum / total - 0.5)
    i = int(np.argmin(diff))
    return i, int(cum[i])


def choose_global_split_dimension(comm, group, pts: DevicePoints, cfg: ClusterConfig, level: int = 0) -> int:
    rows = _gather_group_sample(comm, group, pts, cfg, level)
    if rows.shape[0] == 0:
        return 0
    return int(np.argsort(-np.var(rows, axis=0), kind="mergesort")[0])


def _choose_planes(comm, group, pts: DevicePoints, cfg: ClusterConfig, level: int, backend=_CUDA) -> SplitPlane:
    """cluster.py:228-278, restructured into rounds every rank takes part in (one
    candidate dimension per round) so that collectives stay matched across groups."""
    dims = pts.dims
    rows = _gather_group_sample(comm, group, pts, cfg, level)
    order = np.argsort(-np.var(rows, axis=0), kind="mergesort") if rows.shape[0] else np.zeros(dims, np.int64)
    decided = rows.shape[0] == 0  # empty group: any plane keeps regions well-formed
    plane = SplitPlane(0, 0.0)
    group_n = 0
    for t in range(dims):
        payload = None
        if not decided:
            d = int(order[t])
            boundaries = np.unique(rows[:, d])
            counts, equals = backend.histogram(pts, d, boundaries)
            payload = np.concatenate([counts, equals, [pts.count]]).astype(np.int64)
        gathered = comm.all_gather(payload)
        if not decided:
            red = np.sum([gathered[r] for r in group], axis=0)
            nb = boundaries.shape[0]
            g_counts, g_equals, group_n = red[:nb + 1], red[nb + 1:2 * nb + 1], int(red[-1])
            if group_n == 0:
                plane, decided = SplitPlane(0, 0.0), True
            else:
                lt = np.cumsum(g_counts)[:nb]
                bi, _ = _select_median(boundaries, g_counts)
                value = float(boundaries[bi])
                below = int(lt[np.searchsorted(boundaries, value)])
                if group_n < 2 or 0 < below < group_n:
                    plane, decided = SplitPlane(d, value), True
                else:
                    le = lt + g_equals
                    best_diff, best_value = None, None
                    for i in range(nb):
                        for cv, cb in ((boundaries[i], lt[i]), (np.nextafter(boundaries[i], np.inf), le[i])):
                            if 0 < cb < group_n:
                                diff = abs(cb / group_n - 0.5)
                                if best_diff is None or diff < best_diff:
                                    best_diff, best_value = diff, float(cv)
                    if best_value is not None:
                        plane, decided = SplitPlane(d, best_value), True
        flags = comm.all_gather(decided)
        if all(flags):
            break
    flags = comm.all_gather(decided)
    if not all(flags):
        bad = [r for r in range(comm.size) if not flags[r]]
        raise UnsplittableDataError(
            f"rank group(s) containing {bad} at level {level} hold {group_n if not decided else 'some'} points "
            f"identical in every of {dims} dimensions; cannot split into nonempty halves")
    return plane


def redistribute(comm, group, pts: DevicePoints, plane: SplitPlane, backend=_CUDA) -> tuple[DevicePoints, int]:
    """cluster.py:281-351: lower half of the group gets coord < value; receivers
    take contiguous slices total//H (+1 for the first total%H) of the virtual
    sequence ordered by (sender rank, stable local order)."""
    import torch
    group = tuple(group)
    half = len(group) // 2
    receivers = {0: group[:half], 1: group[half:]}
    parted, nl = backend.partition(pts, plane)
    side_rng = {0: (0, nl), 1: (nl, pts.count)}
    counts = comm.all_gather((nl, pts.count - nl))
    per_rank = {r: counts[r] for r in group}
    sends, mine, sent = {}, [], 0
    me = comm.rank
    if me in group:
        for side in (0, 1):
            recv = receivers[side]
            total = sum(per_rank[r][side] for r in group)
            share, rem = divmod(total, len(recv))
            targets = {r: share + (1 if i < rem else 0) for i, r in enumerate(recv)}
            rstart, pos = {}, 0
            for r in recv:
                rstart[r] = pos
                pos += targets[r]
            soff, pos = {}, 0
            for r in group:
                soff[r] = pos
                pos += per_rank[r][side]
            my0, my1 = soff[me], soff[me] + per_rank[me][side]
            for r in recv:
                lo, hi = max(my0, rstart[r]), min(my1, rstart[r] + targets[r])
                if lo >= hi:
                    continue
                a = side_rng[side][0] + (lo - my0)
                blk = parted.slice(a, a + (hi - lo))
                if r == me:
                    mine.append(blk)
                else:
                    sends[r] = (blk.coords, blk.ids)
                    sent += hi - lo
    got = comm.alltoall(sends)
    blocks = []
    for src in sorted(set(got) | ({me} if mine else set())):
        if src == me:
            blocks.extend(mine)
        else:
            c, i = got[src]
            blocks.append(DevicePoints(c, i))
    blocks = [b for b in blocks if b.count]
    if blocks:
        new = DevicePoints(torch.cat([b.coords for b in blocks], dim=1).contiguous(),
                           torch.cat([b.ids for b in blocks]).contiguous())
    else:
        new = DevicePoints(pts.coords[:, :0].contiguous(), pts.ids[:0].contiguous())
    return new, sent


def rank_build_global(comm, pts: DevicePoints, cfg: ClusterConfig, backend=_CUDA):
    """cluster.py:354-389 for one rank (SPMD)."""
    import torch
    p = comm.size
    levels = p.bit_length() - 1
    dims = pts.dims
    plane_dims = np.full(max(p - 1, 0), -1, dtype=np.int32)
    plane_values = np.zeros(max(p - 1, 0), dtype=np.float64)
    stats = {"points_moved": 0, "t_global_split": 0.0, "t_redistribute": 0.0}
    for level in range(levels):
        group = _group_of(comm.rank, p, level)
        heap_idx = (1 << level) - 1 + (comm.rank >> (levels - level))
        t0 = time.perf_counter()
        plane = _choose_planes(comm, group, pts, cfg, level, backend)
        for idx, d, v in comm.all_gather((heap_idx, plane.dim, plane.value)):
            if plane_dims[idx] != -1 and (plane_dims[idx] != d or plane_values[idx] != v):
                raise AssertionError("rank group disagreed on a split plane")
            plane_dims[idx], plane_values[idx] = d, v
        stats["t_global_split"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        pts, sent = redistribute(comm, group, pts, plane, backend)
        stats["points_moved"] += sent
        stats["t_redistribute"] += time.perf_counter() - t0
    gt = GlobalTree(dims, plane_dims, plane_values)
    if pts.count and levels:
        reg = gt.region_of(comm.rank)
        lo = torch.as_tensor(reg.lower, device=pts.coords.device).to(pts.coords.dtype)[:, None]
        hi = torch.as_tensor(reg.upper, device=pts.coords.device).to(pts.coords.dtype)[:, None]
        if not bool(((pts.coords >= lo) & (pts.coords <= hi)).all()):
            raise AssertionError(f"rank {comm.rank}: point outside its region after redistribution")
    return gt, pts, stats


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


def build_global_tree(points_per_rank: list, cfg: ClusterConfig):
    """cluster.py:392-417 driver over in-process ranks.  Returns the replicated
    GlobalTree, the redistributed per-rank PointSets and per-rank stats."""
    p = len(points_per_rank)
    if p < 1 or (p & (p - 1)) != 0:
        raise ValueError(f"rank count {p} is not a power of two")
    if len({ps.dims for ps in points_per_rank}) != 1:
        raise ValueError("inconsistent dimensionality across ranks")
    if sum(ps.count for ps in points_per_rank) == 0:
        raise ValueError("empty dataset")
    if p == 1:
        gt = GlobalTree(points_per_rank[0].dims, np.empty(0, dtype=np.int32), np.empty(0, dtype=np.float64))
        return gt, list(points_per_rank), [{"points_moved": 0, "t_global_split": 0.0, "t_redistribute": 0.0}]
    dev_pts, gts, stats = build_global_device(points_per_rank, cfg)
    return gts, [d.to_pointset() for d in dev_pts], stats


def build_global_device(points_per_rank: list, cfg: ClusterConfig):
    """Same as build_global_tree, but keeps every rank's points on its GPU."""
    f32 = _f32_all(points_per_rank)

    def prog(comm, ps):
        dp = DevicePoints.from_pointset(ps, comm.device, f32)
        return rank_build_global(comm, dp, cfg)

    res = run_ranks(len(points_per_rank), prog, [(ps,) for ps in points_per_rank])
    trees = [r[0] for r in res]
    for t in trees[1:]:
        if t.to_bytes() != trees[0].to_bytes():
            raise AssertionError("global tree replicas differ across ranks")
    return [r[1] for r in res], trees[0], [r[2] for r in res]
