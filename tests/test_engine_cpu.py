"""Global tier (cluster.py / dist_query.py / engine.py) on CPU: the SPMD protocol
with in-process thread ranks and with a gloo world_size-2 process group, local
work delegated to the oracle stand-in backend (tests/cpu_backend.py).  Checked
against golden fixtures from the real reference's build_engine / Engine.query:
bundle bytes, global planes, per-rank counts, forwarding counters, neighbours."""

import hashlib
import json
import os

import numpy as np
import pytest

from cpu_backend import CpuOracleBackend
from datagen import engine_cases

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = engine_cases()


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "engine.json")) as f:
        return json.load(f), np.load(os.path.join(GOLD, "engine_knn.npz"))


@pytest.mark.parametrize("name", sorted(CASES))
def test_engine_bundle_and_queries_match_reference(gold, name):
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.engine import RunConfig, build_engine, bundle_to_bytes, bundle_from_bytes
    meta, arrays = gold
    rows, cfg, queries, k = CASES[name]
    eng, rep = build_engine(PointSet.from_rows(rows), RunConfig(**cfg), backend=CpuOracleBackend())
    want = meta[name]
    assert eng.ranks[0].global_tree.to_bytes().hex() == want["global_tree"]
    assert [r.tree.count for r in eng.ranks] == want["rank_counts"]
    assert rep.points_moved == want["points_moved"]
    blob = bundle_to_bytes(eng)
    assert len(blob) == want["bundle_len"]
    assert hashlib.sha256(blob).hexdigest() == want["bundle_sha256"]
    assert bundle_to_bytes(bundle_from_bytes(blob)) == blob
    res, qrep = eng.query(queries, k=k)
    d = np.array([[x.sq_dist for x in r.neighbors] for r in res])
    i = np.array([[x.point_id for x in r.neighbors] for r in res], dtype=np.uint64)
    assert np.array_equal(d, arrays[f"{name}/dists"]) and np.array_equal(i, arrays[f"{name}/ids"])
    for key in ("queries_forwarded", "requests_sent", "requests_received", "soundness_violations",
                "nodes_visited", "points_compared"):
        assert getattr(qrep, key) == want[key], key


def test_pipelining_and_slice_invariance():
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.dist_query import QueryBatch, distributed_knn, run_pipelined
    from paper_1607_08220_b200.engine import RunConfig, build_engine
    rows, cfg, queries, k = CASES["eng_u3_20000_p4"]
    eng, _ = build_engine(PointSet.from_rows(rows), RunConfig(**cfg), backend=CpuOracleBackend())
    b = CpuOracleBackend()
    base, _ = distributed_knn(eng.ranks, QueryBatch.create(queries, k=k), backend=b)
    view = lambda rs: [(r.query_id, n.point_id, n.sq_dist) for r in rs for n in r.neighbors]  # noqa: E731
    for bs in (1, 7, 64):
        for piped in (True, False):
            got, st = run_pipelined(eng.ranks, QueryBatch.create(queries, k=k, batch_size=bs), pipelined=piped,
                                    backend=b)
            assert view(got) == view(base)
            assert sum(s.soundness_violations for s in st) == 0


def test_reference_errors():
    from paper_1607_08220_b200.cluster import ClusterConfig, UnsplittableDataError, build_global_tree
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.engine import RunConfig
    with pytest.raises(ValueError, match="power of two"):
        RunConfig(ranks=3)
    with pytest.raises(ValueError, match="empty dataset"):
        build_global_tree([PointSet.empty(2), PointSet.empty(2)], ClusterConfig())
    with pytest.raises(ValueError, match="power of two"):
        build_global_tree([PointSet.empty(2)] * 3, ClusterConfig())


def _gloo_worker(rank, world, port, rows, cfg, queries, k, outq):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1607_08220_b200.cluster import DevicePoints, rank_build_global
        from paper_1607_08220_b200.comm import TorchComm
        from paper_1607_08220_b200.core import PointSet
        from paper_1607_08220_b200.dist_query import QueryBatch, rank_query_program
        from paper_1607_08220_b200.engine import RankState, RunConfig, _split_contiguous
        rc = RunConfig(**cfg)
        comm = TorchComm()
        be = CpuOracleBackend()
        part = _split_contiguous(PointSet.from_rows(rows), world)[rank]
        gt, pts, st = rank_build_global(comm, DevicePoints.from_pointset(part, "cpu", False), rc.cluster_config(), be)
        tree = be.build(pts, rc.build_config(1))
        batch = QueryBatch.create(queries, k)
        pos = np.arange(batch.count)
        m = pos % world == rank
        res, stats = rank_query_program(comm, RankState(rank, None, gt, tree), batch, pos[m].astype(np.uint64),
                                        batch.coords[m], 64, True, be)
        outq.put((rank, gt.to_bytes().hex(), pts.ids.numpy().tolist(), {int(q): (v[0].tolist(), v[1].tolist())
                                                                         for q, v in res.items()},
                  stats.queries_forwarded, st["points_moved"]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_reference():
    import torch.multiprocessing as mp
    rows, cfg, queries, k = CASES["eng_f32_50000_p2"]
    meta = json.load(open(os.path.join(GOLD, "engine.json")))["eng_f32_50000_p2"]
    arrays = np.load(os.path.join(GOLD, "engine_knn.npz"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, rows, cfg, queries, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[0][1] == outs[1][1] == meta["global_tree"]
    assert [len(o[2]) for o in outs] == meta["rank_counts"]
    assert sum(o[5] for o in outs) == meta["points_moved"]
    assert sum(o[4] for o in outs) == meta["queries_forwarded"]
    merged = {}
    for o in outs:
        merged.update(o[3])
    for qi in range(queries.shape[0]):
        d, i = merged[qi]
        assert d == arrays["eng_f32_50000_p2/dists"][qi].tolist()
        assert i == arrays["eng_f32_50000_p2/ids"][qi].tolist()
