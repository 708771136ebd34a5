"""Rank-to-rank communication for the global tier (replaces kdknn.transport / wire).

The reference simulates MPI ranks as threads exchanging byte frames
(transport.py:33-187, wire.py).  Here every exchange carries device tensors and
the protocol code is written once, SPMD, against two collectives:

* ``all_gather(obj)``   -- every rank contributes a small host object (numpy
  arrays, tuples); returns the rank-ordered list.  Group collectives of the
  reference (group_all_gather / group_sum_reduce) are all-gathers whose group
  slice each member reads.
* ``alltoall(sends)``   -- point-to-point blocks: ``sends[dst]`` is a tuple of
  device tensors; returns ``{src: tuple}``.

Two backends:

* :class:`ThreadComm` -- P ranks as threads of one process (the reference's
  execution model, so ``build_engine(points, RunConfig(ranks=P))`` keeps its
  single-call API).  Rank r runs on CUDA device r % device_count; blocks move by
  reference (same device) or device-to-device copy.
* :class:`TorchComm` -- one process per GPU under torchrun:
  ``torch.distributed`` all_gather_object for the small control data and
  ``all_to_all_single`` over NCCL (NVLink/NVSwitch) for point/query blocks; gloo
  on CPU for the multi-process host tests.

A failure on any thread aborts the whole in-process cluster (transport.py:89-104):
surviving ranks raise :class:`ClusterAborted` instead of deadlocking.
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Sequence

__all__ = ["ClusterAborted", "ThreadCluster", "ThreadComm", "TorchComm", "run_ranks"]


class ClusterAborted(RuntimeError):
    """Raised in surviving ranks when another rank failed (transport.py:29-30)."""


class ThreadCluster:
    def __init__(self, size: int):
        if size < 1:
            raise ValueError("rank_count must be >= 1")
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots: list = [None] * size
        self.mail: list = [[None] * size for _ in range(size)]
        self.failed = threading.Event()

    def abort(self):
        self.failed.set()
        self.barrier.abort()


class ThreadComm:
    """In-process rank endpoint (threads share one address space)."""

    def __init__(self, cluster: ThreadCluster, rank: int):
        self.cluster = cluster
        self.rank = rank
        self.size = cluster.size
        self.bytes_moved = 0

    @property
    def device(self):
        import torch
        n = torch.cuda.device_count()
        return torch.device("cuda", self.rank % n) if n else torch.device("cpu")

    def _wait(self):
        try:
            self.cluster.barrier.wait()
        except threading.BrokenBarrierError:
            raise ClusterAborted("another rank failed") from None

    def all_gather(self, obj):
        c = self.cluster
        self._wait()
        c.slots[self.rank] = obj
        self._wait()
        out = list(c.slots)
        self._wait()
        return out

    def alltoall(self, sends: dict):
        c = self.cluster
        self._wait()
        for dst, payload in sends.items():
            c.mail[self.rank][dst] = payload
        self._wait()
        got = {}
        dev = self.device
        for src in range(self.size):
            p = c.mail[src][self.rank]
            if p is not None:
                got[src] = tuple(t.to(dev, non_blocking=True) if hasattr(t, "to") else t for t in p)
                if src != self.rank:
                    self.bytes_moved += sum(t.numel() * t.element_size() for t in p if hasattr(t, "numel"))
        self._wait()
        for src in range(self.size):
            c.mail[src][self.rank] = None
        self._wait()
        return got

    def barrier(self):
        self._wait()


class TorchComm:
    """torch.distributed endpoint (one process per GPU; NCCL, or gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.bytes_moved = 0

    @property
    def device(self):
        import torch
        if self.dist.get_backend(self.group) == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def all_gather(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def alltoall(self, sends: dict):
        """Blocks are tuples of tensors with identical structure on every rank
        (same count, dtypes and trailing shapes); leading dims may differ."""
        import torch
        dev = self.device
        # describe every block so receivers know split sizes and shapes
        meta = {d: [(tuple(t.shape), str(t.dtype)) for t in p] for d, p in sends.items()}
        all_meta = self.all_gather(meta)
        template = next((p for p in sends.values()), None)
        if template is None:
            for m in all_meta:
                for v in m.values():
                    template = v
                    break
                if template is not None:
                    break
        if template is None:
            return {}
        nfields = len(template)
        got = {}
        recv_shapes = {src: all_meta[src].get(self.rank) for src in range(self.size)}
        for f in range(nfields):
            send_parts, send_splits, recv_splits = [], [], []
            dtype = None
            for d in range(self.size):
                if d in sends:
                    t = sends[d][f].to(dev).contiguous()
                    dtype = t.dtype
                    send_parts.append(t.reshape(-1))
                    send_splits.append(t.numel())
                else:
                    send_splits.append(0)
            for src in range(self.size):
                shp = recv_shapes[src]
                if shp is None:
                    recv_splits.append(0)
                else:
                    n = 1
                    for s in shp[f][0]:
                        n *= s
                    recv_splits.append(n)
                    dtype = dtype or getattr(torch, shp[f][1].replace("torch.", ""))
            if dtype is None:
                continue
            send = torch.cat(send_parts) if send_parts else torch.empty(0, dtype=dtype, device=dev)
            recv = torch.empty(sum(recv_splits), dtype=dtype, device=dev)
            self.dist.all_to_all_single(recv, send, recv_splits, send_splits, group=self.group)
            self.bytes_moved += int(sum(send_splits) - (send_splits[self.rank] if self.rank < len(send_splits) else 0)) \
                * send.element_size()
            off = 0
            for src in range(self.size):
                shp = recv_shapes[src]
                if shp is None:
                    continue
                n = recv_splits[src]
                got.setdefault(src, [None] * nfields)[f] = recv[off:off + n].reshape(shp[f][0])
                off += n
        return {s: tuple(v) for s, v in got.items()}

    def barrier(self):
        self.dist.barrier(group=self.group)


def run_ranks(rank_count: int, program: Callable, args_per_rank: Sequence[tuple]) -> list:
    """SPMD launch of `program(comm, *args)` on in-process ranks (transport.py:151-187).
    The first failure aborts the cluster and is re-raised."""
    cluster = ThreadCluster(rank_count)

    def body(r):
        try:
            return program(ThreadComm(cluster, r), *args_per_rank[r])
        except BaseException:
            cluster.abort()
            raise

    if rank_count == 1:
        return [body(0)]
    with ThreadPoolExecutor(max_workers=rank_count) as pool:
        futs = [pool.submit(body, r) for r in range(rank_count)]
        results, first = [], None
        for f in futs:
            try:
                results.append(f.result())
            except ClusterAborted as e:
                first = first or e
                results.append(None)
            except BaseException as e:  # noqa: BLE001
                if first is None or isinstance(first, ClusterAborted):
                    first = e
                results.append(None)
        if first is not None:
            raise first
        return results
