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
from oracle import oracle as O
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


def _gloo_worker(rank, world, port, rows, cfg, queries, k, slice_size, outq):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_1607_08220_b200.cluster import DevicePoints, DeviceRegions, rank_build_global
        from paper_1607_08220_b200.comm import TorchComm
        from paper_1607_08220_b200.core import PointSet
        from paper_1607_08220_b200.dist_query import QueryStats, rank_query
        from paper_1607_08220_b200.engine import RunConfig, _split_contiguous
        rc = RunConfig(**cfg)
        comm = TorchComm()
        be = CpuOracleBackend()
        part = _split_contiguous(PointSet.from_rows(rows), world)[rank]
        gt, pts, st = rank_build_global(comm, DevicePoints.from_pointset(part, "cpu", False), rc.cluster_config(), be)
        tree = be.build(pts, rc.build_config(1))
        pos = np.arange(queries.shape[0])
        mine = pos[pos % world == rank]
        qs = QueryStats(rank=rank)
        d, i, r, c = rank_query(comm, tree, DeviceRegions(gt, torch.device("cpu")), torch.as_tensor(queries[mine]), k,
                                slice_size=slice_size, pipelined=True, backend=be, stats=qs)
        res = {int(q): (d[j, :c[j]].tolist(), i[j, :c[j]].numpy().view(np.uint64).tolist(), r[j, :c[j]].tolist())
               for j, q in enumerate(mine)}
        outq.put((rank, gt.to_bytes().hex(), pts.ids.numpy().tolist(), res, qs.queries_forwarded, st["points_moved"],
                  comm.bytes_moved))
    finally:
        dist.destroy_process_group()


def _run_gloo(world, rows, cfg, queries, k, slice_size):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() * 7 + world) % 2000
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, rows, cfg, queries, k, slice_size, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return outs


def test_gloo_world2_matches_reference():
    rows, cfg, queries, k = CASES["eng_f32_50000_p2"]
    meta = json.load(open(os.path.join(GOLD, "engine.json")))["eng_f32_50000_p2"]
    arrays = np.load(os.path.join(GOLD, "engine_knn.npz"))
    outs = _run_gloo(2, rows, cfg, queries, k, 64)
    assert outs[0][1] == outs[1][1] == meta["global_tree"]
    assert [len(o[2]) for o in outs] == meta["rank_counts"]
    assert sum(o[5] for o in outs) == meta["points_moved"]
    assert sum(o[4] for o in outs) == meta["queries_forwarded"]
    merged = {}
    for o in outs:
        merged.update(o[3])
    for qi in range(queries.shape[0]):
        d, i, _ = merged[qi]
        assert d == arrays["eng_f32_50000_p2/dists"][qi].tolist()
        assert i == arrays["eng_f32_50000_p2/ids"][qi].tolist()


def test_gloo_world4_presorted_idle_ranks():
    """Pre-sorted input: at the first global level rank 0 already holds exactly its
    share of the low side (it neither sends nor receives), and the queries all come
    from one corner (most ranks receive no queries and no requests) -- every rank
    must still enter every collective.  Results equal the in-process (thread-rank)
    engine and the brute-force oracle."""
    from paper_1607_08220_b200.cluster import ClusterConfig, build_global_tree
    from paper_1607_08220_b200.core import PointSet
    rng = np.random.default_rng(41)
    rows = rng.random((8000, 3))
    rows = rows[np.argsort(rows[:, 0], kind="stable")]
    rows[:, 0] *= 4.0  # x dominates the variance: level 0 splits x at the median
    queries = rows[:60] + 1e-4
    k = 5
    outs = _run_gloo(4, rows, dict(ranks=4, seed=3), queries, k, 16)
    gt_in, parts_in, stats_in = build_global_tree(
        [PointSet.from_rows(rows[a:b], ids=np.arange(a, b, dtype=np.uint64)) for a, b in
         ((0, 2000), (2000, 4000), (4000, 6000), (6000, 8000))], ClusterConfig(seed=3), CpuOracleBackend())
    assert all(o[1] == gt_in.to_bytes().hex() for o in outs)
    assert [o[2] for o in outs] == [p.ids.view(np.int64).tolist() for p in parts_in]
    assert sum(o[5] for o in outs) == sum(s["points_moved"] for s in stats_in)
    ps = PointSet.from_rows(rows)
    bd, bi, bc = O.brute_knn(ps.coords, ps.ids, queries, k)
    merged = {}
    for o in outs:
        merged.update(o[3])
    for qi in range(queries.shape[0]):
        d, i, _ = merged[qi]
        assert d == bd[qi, :bc[qi]].tolist() and i == bi[qi, :bc[qi]].tolist()


def test_c5_shards_int64_ids_three_levels_thread_ranks():
    """BASELINE configs[4] in miniature: 8 in-process ranks (3 global levels), each
    holding one C5-law shard whose ids are (shard << 32) | row (>= 2^32), queries
    ingested round-robin -- neighbours (uint64 ids) equal the brute-force oracle."""
    import torch
    from paper_1607_08220_b200.cluster import ClusterConfig, DevicePoints, DeviceRegions, rank_build_global
    from paper_1607_08220_b200.comm import run_ranks
    from paper_1607_08220_b200.dist_query import QueryStats, rank_query
    from paper_1607_08220_b200.local_tree import BuildConfig
    from paper_1607_08220_b200.workloads import make_shard
    p, n, nq, k = 8, 3000, 40, 5
    shards = [make_shard("C5", s, "cpu", n=n, q=nq) for s in range(p)]
    be = CpuOracleBackend()

    def prog(comm):
        pts, ids, q = shards[comm.rank]
        gt, mine, _ = rank_build_global(comm, DevicePoints(pts.t().contiguous(), ids), ClusterConfig(seed=4), be)
        assert gt.levels == 3
        tree = be.build(mine, BuildConfig(seed=4))
        d, i, r, c = rank_query(comm, tree, DeviceRegions(gt, torch.device("cpu")), q, k, slice_size=64,
                                backend=be, stats=QueryStats(rank=comm.rank))
        return q.numpy(), d.numpy(), i.numpy().view(np.uint64), c.numpy()

    outs = run_ranks(p, prog, [() for _ in range(p)])
    coords = np.ascontiguousarray(torch.cat([s[0] for s in shards]).t().double().numpy())
    ids = torch.cat([s[1] for s in shards]).numpy().view(np.uint64)
    assert ids.max() >= np.uint64(7 << 32)
    for q, d, i, c in outs:
        bd, bi, bc = O.brute_knn(coords, ids, q, k)
        assert np.array_equal(c, bc) and np.array_equal(d, bd) and np.array_equal(i, bi)
