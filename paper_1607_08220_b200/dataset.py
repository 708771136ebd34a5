"""Dataset files and interchange codecs (SPEC.md "External Interfaces"; kdknn.wire).

* ``pkd1`` dataset files: magic ``PKD1``, little-endian u32 dims,
  u64 count, u64 seed, ids (u64 x count), then the coordinates column-major
  (f64, dimension 0 for every point, then dimension 1, ...).  Column-major on
  disk is the device's SoA layout, so :func:`load_pkd1_device` maps the file and
  copies each coordinate column straight into the device buffer (f32 when every
  value is exactly binary32, as the build prefers) -- no host transposition.
* CSV ingestion: one point per line, optional leading id column.
* The reference's inter-rank byte codecs (wire.py:33-147: length-prefixed
  frames; point / query / request / response blocks, ids u64 then columns f64),
  kept for interoperability with tools that speak them.  The engine itself
  exchanges packed device rows (comm.py), not these frames.
"""

from __future__ import annotations

import struct

import numpy as np

from .core import PointSet

__all__ = ["write_pkd1", "read_pkd1", "load_pkd1_device", "read_csv", "write_csv",
           "KIND_POINTS", "KIND_GATHER", "KIND_QUERIES", "KIND_REQUESTS", "KIND_RESPONSES",
           "pack_frame", "unpack_frame", "split_stream", "encode_points", "decode_points", "encode_queries",
           "decode_queries", "encode_requests", "decode_requests", "encode_responses", "decode_responses"]

_PKD1 = b"PKD1"
_PKD1_HEAD = struct.Struct("<4sIQQ")  # magic, dims, count, seed


def write_pkd1(path, points: PointSet, seed: int = 0) -> None:
    with open(path, "wb") as f:
        f.write(_PKD1_HEAD.pack(_PKD1, points.dims, points.count, seed & 0xFFFFFFFFFFFFFFFF))
        f.write(np.ascontiguousarray(points.ids, dtype="<u8").tobytes())
        f.write(np.ascontiguousarray(points.coords, dtype="<f8").tobytes())


def _pkd1_view(path):
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    if raw.shape[0] < _PKD1_HEAD.size:
        raise ValueError("invalid header: file shorter than the pkd1 header")
    magic, dims, count, seed = _PKD1_HEAD.unpack(bytes(raw[:_PKD1_HEAD.size]))
    if magic != _PKD1:
        raise ValueError("invalid header: not a pkd1 dataset (bad magic)")
    need = _PKD1_HEAD.size + 8 * count + 8 * dims * count
    if raw.shape[0] != need:
        raise ValueError(f"invalid header: pkd1 body is {raw.shape[0] - _PKD1_HEAD.size} bytes, expected "
                         f"{need - _PKD1_HEAD.size} for {count} points x {dims} dims")
    off = _PKD1_HEAD.size
    ids = raw[off:off + 8 * count].view("<u8")
    cols = raw[off + 8 * count:need].view("<f8").reshape(dims, count)
    return int(dims), int(count), int(seed), ids, cols


def read_pkd1(path) -> tuple[PointSet, int]:
    """(PointSet, seed); validation as PointSet.create (finite coords, unique ids)."""
    dims, count, seed, ids, cols = _pkd1_view(path)
    return PointSet.create(np.array(cols, dtype=np.float64), np.array(ids, dtype=np.uint64)), seed


def load_pkd1_device(path, device="cuda", chunk: int = 1 << 24):
    """Stream a pkd1 file into device SoA buffers: (coords (dims, n) float32|float64,
    ids (n,) int64 bits of u64, seed).  Columns are copied in chunks through one
    pinned staging buffer; float32 is kept when every coordinate is exact in it."""
    import torch
    dims, count, seed, ids, cols = _pkd1_view(path)
    f32 = True
    for d in range(dims):
        for s in range(0, count, chunk):
            c = np.asarray(cols[d, s:s + chunk])
            if not np.isfinite(c).all():
                raise ValueError("non-finite coordinate")
            with np.errstate(over="ignore"):
                f32 &= bool(np.array_equal(c.astype(np.float32).astype(np.float64), c))
    dt = torch.float32 if f32 else torch.float64
    out = torch.empty((dims, count), dtype=dt, device=device)
    stage = torch.empty(min(chunk, max(count, 1)), dtype=dt).pin_memory()
    for d in range(dims):
        for s in range(0, count, chunk):
            e = min(count, s + chunk)
            torch.cuda.current_stream(out.device).synchronize()  # the staging buffer is free again
            stage[:e - s].copy_(torch.from_numpy(np.array(cols[d, s:e])))
            out[d, s:e].copy_(stage[:e - s], non_blocking=True)
    dev_ids = torch.from_numpy(np.array(ids, dtype=np.uint64).view(np.int64)).to(device)
    if torch.unique(dev_ids).shape[0] != count:
        raise ValueError("duplicate point ids")
    torch.cuda.current_stream(out.device).synchronize()
    return out, dev_ids, seed


def read_csv(path, dims: int | None = None, has_ids: bool | None = None) -> PointSet:
    """One point per line; an optional leading id column (detected when a line
    has dims + 1 fields, or forced with has_ids)."""
    rows = np.loadtxt(path, delimiter=",", ndmin=2, dtype=np.float64)
    if rows.shape[0] == 0:
        return PointSet.empty(dims or 0)
    if has_ids is None:
        has_ids = dims is not None and rows.shape[1] == dims + 1
    if has_ids:
        ids = rows[:, 0]
        if not np.array_equal(ids, np.round(ids)) or (ids < 0).any():
            raise ValueError("id column must hold non-negative integers")
        return PointSet.create(np.ascontiguousarray(rows[:, 1:].T), ids.astype(np.uint64))
    if dims is not None and rows.shape[1] != dims:
        raise ValueError(f"expected {dims} columns, got {rows.shape[1]}")
    return PointSet.from_rows(rows)


def write_csv(path, points: PointSet, with_ids: bool = True) -> None:
    cols = [points.ids.astype(np.float64)[:, None]] if with_ids else []
    np.savetxt(path, np.hstack(cols + [points.coords.T]), delimiter=",", fmt="%.17g")


# ---- inter-rank codecs (wire.py byte layouts) ----------------------------------------------
KIND_POINTS, KIND_GATHER, KIND_QUERIES, KIND_REQUESTS, KIND_RESPONSES = 1, 2, 3, 4, 5
_FRAME = struct.Struct("<IBI")  # length of the rest, kind, sender


def pack_frame(kind: int, sender: int, payload: bytes) -> bytes:
    return _FRAME.pack(len(payload) + 5, kind, sender) + payload


def unpack_frame(frame: bytes) -> tuple[int, int, bytes]:
    length, kind, sender = _FRAME.unpack_from(frame, 0)
    if length != len(frame) - 4:
        raise ValueError(f"frame length {length} does not match buffer {len(frame) - 4}")
    return kind, sender, frame[_FRAME.size:]


def split_stream(buf: bytes) -> list:
    frames, off = [], 0
    while off < len(buf):
        if len(buf) - off < 4:
            raise ValueError("truncated frame header")
        end = off + 4 + struct.unpack_from("<I", buf, off)[0]
        if end > len(buf):
            raise ValueError("truncated frame body")
        frames.append(buf[off:end])
        off = end
    return frames


class _Reader:
    def __init__(self, blob: bytes, off: int = 0):
        self.blob, self.off = blob, off

    def arr(self, dtype: str, n: int):
        a = np.frombuffer(self.blob, dtype=dtype, count=n, offset=self.off)
        self.off += a.nbytes
        return a

    def head(self, fmt: str):
        v = struct.unpack_from(fmt, self.blob, self.off)
        self.off += struct.calcsize(fmt)
        return v


def _cols(rows_or_soa, soa: bool) -> bytes:
    a = np.asarray(rows_or_soa, dtype="<f8")
    return np.ascontiguousarray(a if soa else a.T).tobytes()


def encode_points(ps: PointSet) -> bytes:
    return struct.pack("<II", ps.count, ps.dims) + np.ascontiguousarray(ps.ids, "<u8").tobytes() + _cols(ps.coords, True)


def decode_points(payload: bytes) -> PointSet:
    rd = _Reader(payload)
    count, dims = rd.head("<II")
    ids = rd.arr("<u8", count).astype(np.uint64)
    return PointSet(np.ascontiguousarray(rd.arr("<f8", dims * count).reshape(dims, count), dtype=np.float64), ids)


def encode_queries(qids, coords) -> bytes:
    coords = np.asarray(coords)
    return struct.pack("<II", *coords.shape) + np.ascontiguousarray(qids, "<u8").tobytes() + _cols(coords, False)


def decode_queries(payload: bytes):
    rd = _Reader(payload)
    count, dims = rd.head("<II")
    qids = rd.arr("<u8", count).astype(np.uint64)
    return qids, np.ascontiguousarray(rd.arr("<f8", dims * count).reshape(dims, count).T, dtype=np.float64)


def encode_requests(qids, sq_r_primes, coords, k: int) -> bytes:
    coords = np.asarray(coords)
    return (struct.pack("<III", coords.shape[0], coords.shape[1], k) + np.ascontiguousarray(qids, "<u8").tobytes()
            + np.ascontiguousarray(sq_r_primes, "<f8").tobytes() + _cols(coords, False))


def decode_requests(payload: bytes):
    rd = _Reader(payload)
    count, dims, k = rd.head("<III")
    qids = rd.arr("<u8", count).astype(np.uint64)
    rps = rd.arr("<f8", count).astype(np.float64)
    return qids, rps, np.ascontiguousarray(rd.arr("<f8", dims * count).reshape(dims, count).T, np.float64), int(k)


def encode_responses(qids, counts, dists, pids, ranks) -> bytes:
    parts = [struct.pack("<I", len(qids))]
    for a, dt in ((qids, "<u8"), (counts, "<u4"), (dists, "<f8"), (pids, "<u8"), (ranks, "<u4")):
        parts.append(np.ascontiguousarray(a, dt).tobytes())
    return b"".join(parts)


def decode_responses(payload: bytes):
    rd = _Reader(payload)
    (nq,) = rd.head("<I")
    qids = rd.arr("<u8", nq).astype(np.uint64)
    counts = rd.arr("<u4", nq).astype(np.int64)
    tot = int(counts.sum())
    return (qids, counts, rd.arr("<f8", tot).astype(np.float64), rd.arr("<u8", tot).astype(np.uint64),
            rd.arr("<u4", tot).astype(np.int64))
