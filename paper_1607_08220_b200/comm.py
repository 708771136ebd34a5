"""Rank-to-rank communication for the global tier (replaces kdknn.transport / wire).

The reference simulates MPI ranks as threads exchanging byte frames
(transport.py:33-187, wire.py:63-147).  Here every exchange is a collective on
tensors that stay on the rank's device, written once, SPMD:

* ``all_gather_t(x)``      same-shape tensor from every rank -> (P, *x.shape)
* ``all_reduce_t(x)``      element-wise sum over ranks (the reference's
  group_sum_reduce: each group writes its own segment of a shared buffer)
* ``alltoallv(rows, send_counts)``  variable all-to-all of 2-D row blocks:
  ``rows`` holds the rows for rank 0, then rank 1, ... (``send_counts[r]`` of
  them); returns the received rows in source-rank order and the per-source
  counts.  One count exchange (a P-element tensor) and one data exchange; every
  rank always enters both collectives, whatever it sends or receives.

Records of several fields travel as packed byte rows (``pack_rows`` /
``unpack_rows``): one collective per exchange, whatever the number of fields.

Backends:

* :class:`ThreadComm` -- P ranks as threads of one process (the reference's
  execution model, so ``build_engine(points, RunConfig(ranks=P))`` keeps its
  single-call API).  Rank r runs on CUDA device r % device_count; blocks move
  by reference (same device) or device-to-device copy.
* :class:`TorchComm` -- one process per GPU under torchrun: ``torch.distributed``
  collectives on the rank's tensors -- NCCL over NVLink / NVSwitch for CUDA
  tensors, gloo for the CPU multi-process tests.

A failure on any thread aborts the whole in-process cluster (transport.py:89-104):
surviving ranks raise :class:`ClusterAborted` instead of deadlocking.
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Sequence

__all__ = ["ClusterAborted", "ThreadCluster", "ThreadComm", "TorchComm", "run_ranks", "pack_rows", "unpack_rows"]


class ClusterAborted(RuntimeError):
    """Raised in surviving ranks when another rank failed (transport.py:29-30)."""


def pack_rows(*fields):
    """Fields of n rows each ((n,) or (n, c) tensors of any dtype, one device) ->
    (n, W) uint8 rows and the layout needed by :func:`unpack_rows`."""
    import torch
    n = fields[0].shape[0]
    parts, spec = [], []
    for f in fields:
        cols = 1
        for e in f.shape[1:]:
            cols *= e
        spec.append((f.dtype, cols, tuple(f.shape[1:])))
        if n == 0:
            parts.append(torch.empty((0, cols * f.element_size()), dtype=torch.uint8, device=f.device))
        else:
            parts.append(f.reshape(n, cols).contiguous().view(torch.uint8).reshape(n, cols * f.element_size()))
    return torch.cat(parts, dim=1) if len(parts) > 1 else parts[0], spec


def unpack_rows(rows, spec):
    """Inverse of :func:`pack_rows` (fields come back contiguous)."""
    import torch
    out, off = [], 0
    n = rows.shape[0]
    for dtype, cols, tail in spec:
        es = torch.empty((), dtype=dtype).element_size()
        w = cols * es
        if n == 0:
            out.append(torch.empty((0,) + tail, dtype=dtype, device=rows.device))
        else:
            col = torch.empty((n, w), dtype=torch.uint8, device=rows.device)
            col.copy_(rows[:, off:off + w])
            out.append(col.view(dtype).reshape((n,) + tail))
        off += w
    return out


class ThreadCluster:
    def __init__(self, size: int):
        if size < 1:
            raise ValueError("rank_count must be >= 1")
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots: list = [None] * size
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

    def _exchange(self, mine):
        """Publish `mine`, return every rank's value (rank order)."""
        c = self.cluster
        self._wait()
        c.slots[self.rank] = mine
        self._wait()
        out = list(c.slots)
        self._wait()
        return out

    def all_gather(self, obj):
        """Small host objects (test / driver utility; the protocol uses tensors)."""
        return self._exchange(obj)

    def all_gather_t(self, x):
        import torch
        dev = self.device
        return torch.stack([t.to(dev) for t in self._exchange(x)])

    def all_reduce_t(self, x):
        parts = self._exchange(x)
        dev = self.device
        acc = parts[0].to(dev).clone()
        for t in parts[1:]:
            acc += t.to(dev)
        return acc

    def alltoallv(self, rows, send_counts):
        import torch
        sc = [int(v) for v in (send_counts.tolist() if hasattr(send_counts, "tolist") else send_counts)]
        allp = self._exchange((rows, sc))
        dev = self.device
        blocks, rc = [], []
        cross = False
        for src, (r, c) in enumerate(allp):
            off = sum(c[:self.rank])
            blk = r[off:off + c[self.rank]]
            rc.append(int(c[self.rank]))
            if src != self.rank:
                self.bytes_moved += blk.numel() * blk.element_size()
            cross |= blk.device != dev
            blocks.append(blk.to(dev, non_blocking=True))
        out = torch.cat(blocks) if blocks else rows[:0].to(dev)
        if cross and dev.type == "cuda":
            torch.cuda.synchronize(dev)  # peer blocks copied before their owners move on
        self._wait()  # every rank has taken its blocks before senders reuse their buffers
        return out, rc

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
        """Small host objects (driver utility; the protocol uses tensors)."""
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def all_gather_t(self, x):
        import torch
        x = x.to(self.device).contiguous()
        out = torch.empty((self.size,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_gather_into_tensor(out, x, group=self.group)
        else:
            self.dist.all_gather(list(out.unbind(0)), x, group=self.group)
        return out

    def all_reduce_t(self, x):
        x = x.to(self.device).contiguous().clone()
        self.dist.all_reduce(x, group=self.group)
        return x

    def alltoallv(self, rows, send_counts):
        import torch
        dev = self.device
        p = self.size
        rows = rows.to(dev).contiguous()
        sc_t = (send_counts.to(dev, torch.int64) if hasattr(send_counts, "to")
                else torch.tensor(list(send_counts), dtype=torch.int64, device=dev)).contiguous()
        rc_t = torch.empty(p, dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(rc_t, sc_t, group=self.group)
        both = torch.cat([sc_t, rc_t]).tolist()  # the one host read of the exchange
        sc, rc = both[:p], both[p:]
        w = rows.shape[1] if rows.dim() == 2 else 1
        out = torch.empty((sum(rc), w), dtype=rows.dtype, device=dev)
        self.dist.all_to_all_single(out.view(-1), rows.view(-1), [c * w for c in rc], [c * w for c in sc],
                                    group=self.group)
        self.bytes_moved += (sum(sc) - sc[self.rank]) * w * rows.element_size()
        return (out if rows.dim() == 2 else out.view(-1)), rc

    def barrier(self):
        self.dist.barrier(group=self.group)


def run_ranks(rank_count: int, program: Callable, args_per_rank: Sequence[tuple]) -> list:
    """SPMD launch of `program(comm, *args)` on in-process ranks (transport.py:151-187).
    The first failure aborts the cluster and is re-raised."""
    cluster = ThreadCluster(rank_count)

    def body(r):
        import torch
        try:
            if torch.cuda.is_available():
                torch.cuda.set_device(r % torch.cuda.device_count())
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
