"""Dataset files (pkd1, CSV) and the reference's inter-rank codecs.

The codec byte strings are golden output of the real kdknn.wire
(tests/golden/make_wire_golden.py); pkd1 follows SPEC.md:501 byte for byte."""

import os
import struct

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def W():
    return np.load(os.path.join(GOLD, "wire.npz"))


def test_codecs_match_reference_bytes(W):
    from paper_1607_08220_b200 import dataset as ds
    from paper_1607_08220_b200.core import PointSet
    ps = PointSet(W["coords"], W["ids"])
    got = {
        "points": ds.encode_points(ps), "queries": ds.encode_queries(W["qid"], W["q"]),
        "requests": ds.encode_requests(W["qid"], W["rp"], W["q"], 7),
        "responses": ds.encode_responses(W["qid"], W["cnt"], W["dd"], W["pp"], W["rk"]),
    }
    got["frame"] = ds.pack_frame(ds.KIND_REQUESTS, 6, got["requests"])
    for k, v in got.items():
        assert v == W[f"bytes_{k}"].tobytes(), k
    back = ds.decode_points(got["points"])
    assert np.array_equal(back.coords, ps.coords) and np.array_equal(back.ids, ps.ids)
    qid, q = ds.decode_queries(got["queries"])
    assert np.array_equal(qid, W["qid"]) and np.array_equal(q, W["q"])
    qid, rp, q, k = ds.decode_requests(got["requests"])
    assert k == 7 and np.array_equal(rp, W["rp"]) and np.array_equal(q, W["q"])
    qid, cnt, dd, pp, rk = ds.decode_responses(got["responses"])
    assert np.array_equal(cnt, W["cnt"]) and np.array_equal(dd, W["dd"]) and np.array_equal(pp, W["pp"])
    assert np.array_equal(rk, W["rk"])
    kind, sender, payload = ds.unpack_frame(got["frame"])
    assert (kind, sender, payload) == (ds.KIND_REQUESTS, 6, got["requests"])
    assert ds.split_stream(got["frame"] + got["frame"]) == [got["frame"]] * 2
    with pytest.raises(ValueError, match="truncated"):
        ds.split_stream(got["frame"][:-1])


def test_pkd1_layout_and_roundtrip(tmp_path):
    from paper_1607_08220_b200 import dataset as ds
    from paper_1607_08220_b200.core import PointSet
    rng = np.random.default_rng(3)
    ps = PointSet.create(rng.random((3, 50)), rng.permutation(1000)[:50].astype(np.uint64))
    path = tmp_path / "a.pkd1"
    ds.write_pkd1(path, ps, seed=42)
    blob = path.read_bytes()
    # magic, u32 dims, u64 count, u64 seed, ids, column-major f64 coords
    assert blob[:4] == b"PKD1" and struct.unpack_from("<IQQ", blob, 4) == (3, 50, 42)
    assert blob[24:24 + 400] == ps.ids.astype("<u8").tobytes()
    assert blob[424:] == ps.coords.astype("<f8").tobytes()
    back, seed = ds.read_pkd1(path)
    assert seed == 42 and np.array_equal(back.coords, ps.coords) and np.array_equal(back.ids, ps.ids)
    path.write_bytes(b"XKD1" + blob[4:])
    with pytest.raises(ValueError, match="invalid header"):
        ds.read_pkd1(path)
    path.write_bytes(blob[:-8])
    with pytest.raises(ValueError, match="invalid header"):
        ds.read_pkd1(path)
    empty = tmp_path / "e.pkd1"
    ds.write_pkd1(empty, PointSet.empty(2))
    assert ds.read_pkd1(empty)[0].count == 0


def test_csv_ingestion(tmp_path):
    from paper_1607_08220_b200 import dataset as ds
    from paper_1607_08220_b200.core import PointSet
    ps = PointSet.create(np.random.default_rng(1).random((2, 20)), np.arange(100, 120, dtype=np.uint64))
    p = tmp_path / "p.csv"
    ds.write_csv(p, ps)
    back = ds.read_csv(p, dims=2)
    assert np.array_equal(back.ids, ps.ids) and np.array_equal(back.coords, ps.coords)
    ds.write_csv(p, ps, with_ids=False)
    back = ds.read_csv(p)
    assert np.array_equal(back.ids, np.arange(20, dtype=np.uint64)) and np.array_equal(back.coords, ps.coords)
    p.write_text("1,0.5,0.5\n1,0.25,0.75\n")
    with pytest.raises(ValueError, match="duplicate"):
        ds.read_csv(p, dims=2)


@pytest.mark.gpu
def test_pkd1_device_load_builds_the_same_tree(tmp_path, oracle):
    import torch
    from paper_1607_08220_b200 import dataset as ds
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree, build_local_tree_device
    rows = np.random.default_rng(5).random((100_000, 3), dtype=np.float32).astype(np.float64)
    ps = PointSet.from_rows(rows, ids=np.arange(7, 100_007, dtype=np.uint64))
    path = tmp_path / "u.pkd1"
    ds.write_pkd1(path, ps)
    coords, ids, _ = ds.load_pkd1_device(path, "cuda", chunk=30_000)
    assert coords.dtype == torch.float32
    a = build_local_tree_device(coords, ids, BuildConfig(seed=2))
    b = build_local_tree(ps, BuildConfig(seed=2))
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(a, key), getattr(b, key)), key
    assert np.array_equal(a.points.ids, b.points.ids)
