"""Global tier on the GPU (CudaBackend): kd_histogram / kd_split_rows / device local
builds / device KNN behind the SPMD protocol.  Bundles must equal the real
reference's byte for byte; neighbours must equal the brute-force oracle;
forwarding counters must equal the reference's (they depend only on r')."""

import hashlib
import json
import os

import numpy as np
import pytest

from datagen import engine_cases, make_rows

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = engine_cases()


@pytest.mark.parametrize("name", sorted(CASES))
def test_engine_gpu_matches_reference(name, oracle):
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.engine import RunConfig, build_engine, bundle_from_bytes, bundle_to_bytes
    meta = json.load(open(os.path.join(GOLD, "engine.json")))[name]
    rows, cfg, queries, k = CASES[name]
    ps = PointSet.from_rows(rows)
    eng, rep = build_engine(ps, RunConfig(**cfg))
    assert eng.ranks[0].global_tree.to_bytes().hex() == meta["global_tree"]
    assert rep.points_moved == meta["points_moved"]
    blob = bundle_to_bytes(eng)
    assert hashlib.sha256(blob).hexdigest() == meta["bundle_sha256"]
    res, qrep = eng.query(queries, k=k)
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, queries, k)
    for qi, r in enumerate(res):
        assert [x.sq_dist for x in r.neighbors] == bd[qi, :bc[qi]].tolist()
        assert [x.point_id for x in r.neighbors] == bi[qi, :bc[qi]].tolist()
        r.check(k=k, total_in_scope=ps.count)
    for key in ("queries_forwarded", "requests_sent", "requests_received", "soundness_violations"):
        assert getattr(qrep, key) == meta[key], key
    # a bundle-loaded engine answers identically (trees re-uploaded from host arrays)
    back = bundle_from_bytes(blob)
    res2, _ = back.query(queries, k=k)
    assert [(r.query_id, n.point_id, n.sq_dist) for r in res for n in r.neighbors] == \
           [(r.query_id, n.point_id, n.sq_dist) for r in res2 for n in r.neighbors]


@pytest.mark.parametrize("p", [1, 2, 4, 8, 16])
def test_exactness_and_p_invariance(p, oracle):
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.engine import RunConfig, build_engine
    rows = make_rows(20000, 3, 5)
    ps = PointSet.from_rows(rows)
    eng, _ = build_engine(ps, RunConfig(ranks=p, seed=5))
    q = np.random.default_rng(4).uniform(size=(200, 3))
    res, rep = eng.query(q, k=5)
    bd, bi, _ = oracle.brute_knn(ps.coords, ps.ids, q, 5)
    got = np.array([[x.point_id for x in r.neighbors] for r in res], dtype=np.uint64)
    assert np.array_equal(got, bi)
    assert rep.soundness_violations == 0 and rep.requests_sent == rep.requests_received


def test_unsplittable_raises():
    from paper_1607_08220_b200.cluster import ClusterConfig, UnsplittableDataError, build_global_tree
    from paper_1607_08220_b200.core import PointSet
    rows = np.tile([1.0, 2.0], (50, 1))
    parts = [PointSet.from_rows(rows[:25]), PointSet.from_rows(rows[25:], ids=np.arange(25, 50, dtype=np.uint64))]
    with pytest.raises(UnsplittableDataError):
        build_global_tree(parts, ClusterConfig(seed=0))


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_device_resident_protocol(p, oracle):
    """dist_query.rank_query over in-process ranks (device tensors through the
    communicator, kd_merge_topk on the owner), global tier built with the device
    kernels, self-exclusion ids travelling with queries and requests."""
    import torch
    from paper_1607_08220_b200.cluster import ClusterConfig, DevicePoints, DeviceRegions, rank_build_global
    from paper_1607_08220_b200.comm import run_ranks
    from paper_1607_08220_b200.dist_query import QueryStats, rank_query
    from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
    rows = make_rows(60000, 3, 23, "halo-f32")
    n = rows.shape[0]
    qsel = np.random.default_rng(3).choice(n, 3000, replace=False)
    k = 5

    def prog(comm):
        dev = comm.device
        lo, hi = round(comm.rank * n / p), round((comm.rank + 1) * n / p)
        c = torch.as_tensor(rows[lo:hi].T.astype(np.float32)).to(dev).contiguous()
        ids = torch.arange(lo, hi, dtype=torch.int64, device=dev)
        gt, pts, _ = rank_build_global(comm, DevicePoints(c, ids), ClusterConfig(seed=1))
        tree = build_local_tree_device(pts.coords, pts.ids, BuildConfig(seed=1))
        mine = qsel[qsel % p == comm.rank]
        q = torch.as_tensor(rows[mine]).to(dev)
        ex = torch.as_tensor(mine.astype(np.int64)).to(dev)
        st = QueryStats(rank=comm.rank)
        d, i, r, cnt = rank_query(comm, tree, DeviceRegions(gt, dev), q, k, excl=ex, slice_size=700, stats=st)
        return mine, d.cpu().numpy(), i.cpu().numpy(), cnt.cpu().numpy(), st

    outs = run_ranks(p, prog, [() for _ in range(p)])
    coords = np.ascontiguousarray(rows.T)
    ids = np.arange(n, dtype=np.uint64)
    for mine, d, i, cnt, st in outs:
        bd, bi, bc = oracle.brute_knn(coords, ids, rows[mine], k + 1)
        for r in range(mine.shape[0]):
            keep = bi[r, :bc[r]] != mine[r]
            assert np.array_equal(d[r], bd[r, :bc[r]][keep][:k])
            assert np.array_equal(i[r].view(np.uint64), bi[r, :bc[r]][keep][:k])
        assert (cnt == k).all()
        assert st.soundness_violations == 0


def test_query_arrays_equals_objects(oracle):
    from paper_1607_08220_b200.core import PointSet
    from paper_1607_08220_b200.engine import RunConfig, build_engine
    rows = make_rows(30000, 3, 8, "halo-f32")
    ps = PointSet.from_rows(rows)
    eng, _ = build_engine(ps, RunConfig(ranks=4, seed=2))
    q = rows[::97] + 1e-5
    (d, i, r, c), rep = eng.query_arrays(q, k=6)
    res, _ = eng.query(q, k=6)
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, 6)
    assert np.array_equal(c, bc) and np.array_equal(d, bd) and np.array_equal(i, bi)
    for j, rr in enumerate(res):
        assert [x.point_id for x in rr.neighbors] == i[j, :c[j]].tolist()
        assert [x.rank for x in rr.neighbors] == r[j, :c[j]].tolist()
    # neighbour ranks: the rank whose region holds the point
    owners = eng.ranks[0].global_tree.owner_of_batch(ps.coords.T[i[c > 0][:, 0].astype(np.int64)])
    assert np.array_equal(owners, r[c > 0][:, 0])


def test_c5_shards_int64_ids_three_levels_gpu(oracle):
    """BASELINE configs[4] in miniature on the GPU: 8 thread ranks (3 global levels),
    one C5-law shard each (ids (shard << 32) | row), the device protocol end to end."""
    import torch
    from paper_1607_08220_b200.cluster import ClusterConfig, DevicePoints, DeviceRegions, rank_build_global
    from paper_1607_08220_b200.comm import run_ranks
    from paper_1607_08220_b200.dist_query import QueryStats, rank_query
    from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
    from paper_1607_08220_b200.workloads import make_shard
    p, n, nq, k = 8, 200_000, 2000, 5

    def prog(comm):
        pts, ids, q = make_shard("C5", comm.rank, comm.device, n=n, q=nq)
        gt, mine, _ = rank_build_global(comm, DevicePoints(pts.t().contiguous(), ids), ClusterConfig(seed=4))
        tree = build_local_tree_device(mine.coords, mine.ids, BuildConfig(seed=4))
        st = QueryStats(rank=comm.rank)
        d, i, r, c = rank_query(comm, tree, DeviceRegions(gt, comm.device), q, k, slice_size=4096, stats=st)
        return (pts.cpu(), ids.cpu(), q.cpu().numpy(), d.cpu().numpy(), i.cpu().numpy().view(np.uint64),
                c.cpu().numpy(), st)

    outs = run_ranks(p, prog, [() for _ in range(p)])
    coords = np.ascontiguousarray(torch.cat([o[0] for o in outs]).t().double().numpy())
    ids = torch.cat([o[1] for o in outs]).numpy().view(np.uint64)
    for _, _, q, d, i, c, st in outs:
        sel = np.arange(0, q.shape[0], 7)
        bd, bi, bc = oracle.brute_knn(coords, ids, q[sel], k)
        assert np.array_equal(c[sel], bc) and np.array_equal(d[sel], bd) and np.array_equal(i[sel], bi)
        assert st.soundness_violations == 0
    assert sum(o[6].queries_forwarded for o in outs) > 0


@pytest.mark.parametrize("name", ["u3_2000", "f32_u3_20000", "aniso3_5000"])
def test_packet_kernel_matches_brute_force(name, oracle):
    """The opt-in warp-per-packet kernel (KD_KNN_PACKET) gives the oracle's answers."""
    from datagen import golden_cases
    from paper_1607_08220_b200 import _native as N
    from paper_1607_08220_b200 import core, local_query as lq, local_tree as lt
    case = golden_cases()[name]
    ps = core.PointSet.create(case["coords"], case["ids"])
    tree = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
    for k in (1, 5, 8):
        d, i, c, _ = lq.find_knn_batch(tree, case["queries"], k, flags=N.KD_KNN_PACKET)
        bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, case["queries"], k)
        m = np.arange(k)[None, :] < c[:, None]
        assert np.array_equal(c, bc)
        assert np.array_equal(np.where(m, d, 0), np.where(m, bd, 0)) and np.array_equal(np.where(m, i, 0),
                                                                                          np.where(m, bi, 0))


def _nccl_world1_worker(port, outq):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    try:
        from paper_1607_08220_b200.comm import TorchComm, pack_rows, unpack_rows
        c = TorchComm()
        x = torch.arange(6, dtype=torch.int64, device=dev).reshape(2, 3)
        g = c.all_gather_t(x)
        r = c.all_reduce_t(x)
        q = torch.rand((5, 3), dtype=torch.float64, device=dev)
        rows, spec = pack_rows(torch.arange(5, device=dev), q, torch.arange(5, dtype=torch.int32, device=dev))
        got, rc = c.alltoallv(rows, torch.tensor([5], device=dev))
        a, b, cc = unpack_rows(got, spec)
        empty, rc0 = c.alltoallv(rows[:0], [0])
        outq.put((g.shape == (1, 2, 3) and torch.equal(g[0], x), torch.equal(r, x), rc == [5] and rc0 == [0],
                  torch.equal(b, q) and torch.equal(a, torch.arange(5, device=dev)), empty.shape[0] == 0))
    finally:
        dist.destroy_process_group()


def test_torchcomm_nccl_collectives_world1():
    """The NCCL code paths of TorchComm (all_gather_into_tensor, all_reduce,
    all_to_all_single with split lists, packed rows) on CUDA tensors."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(29700 + os.getpid() % 200, q))
    p.start()
    res = q.get(timeout=180)
    p.join(timeout=60)
    assert p.exitcode == 0 and all(res), res
