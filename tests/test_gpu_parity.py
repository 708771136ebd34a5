"""GPU parity: the CUDA build and query through the C-ABI against the oracle.

* trees: byte-identical to the reference (golden fixtures from the real
  reference, and the C oracle on further seeded inputs);
* neighbours: ids identical, distances bit-identical to the brute-force oracle
  (pkg/tests/conftest.py:8-18 semantics: (sq_dist, id) order, strict radius).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from datagen import big_cases, golden_cases, make_rows

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = golden_cases()


@pytest.fixture(scope="module")
def api():
    from paper_1607_08220_b200 import core, local_query, local_tree
    return core, local_tree, local_query


def tree_equal(tree, want, prefix=""):
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        got = getattr(tree, key)
        exp = want[f"{prefix}{key}"] if isinstance(want, dict) or hasattr(want, "files") else getattr(want, key)
        assert np.array_equal(got, exp), f"{key} differs"
        if key == "node_value":
            assert np.array_equal(got.view(np.uint64), np.asarray(exp).view(np.uint64)), "node_value bits differ"


def masked(d, i, c):
    m = np.arange(d.shape[1])[None, :] < c[:, None]
    return np.where(m, d, 0.0), np.where(m, i, 0)


@pytest.mark.parametrize("name", sorted(CASES))
def test_tree_bytes_match_reference_golden(api, name):
    core, lt, _ = api
    case = CASES[name]
    trees = np.load(os.path.join(GOLD, "trees.npz"))
    ps = core.PointSet.create(case["coords"], case["ids"])
    tree = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(tree, key), trees[f"{name}/{key}"]), key
    assert np.array_equal(tree.points.ids, trees[f"{name}/ids"])
    assert tree.depth == int(trees[f"{name}/depth"])
    # packed coordinates are the input rows in packed order
    order = {int(v): j for j, v in enumerate(ps.ids)}
    perm = np.array([order[int(v)] for v in tree.points.ids], dtype=np.int64)
    assert np.array_equal(tree.points.coords, ps.coords[:, perm])


@pytest.mark.parametrize("name", sorted(CASES))
def test_knn_matches_brute_force_golden(api, name):
    core, lt, lq = api
    case = CASES[name]
    knn = np.load(os.path.join(GOLD, "knn.npz"))
    ps = core.PointSet.create(case["coords"], case["ids"])
    tree = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
    for k in case["ks"]:
        d, i, c, _ = lq.find_knn_batch(tree, case["queries"], k)
        assert np.array_equal(c, knn[f"{name}/k{k}/brute_counts"])
        md, mi = masked(d, i, c)
        assert np.array_equal(md, knn[f"{name}/k{k}/brute_dists"])
        assert np.array_equal(mi, knn[f"{name}/k{k}/brute_ids"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_knn_on_imported_reference_tree(api, name):
    """Upload the reference's own tree (golden arrays) and query it on the GPU."""
    core, lt, lq = api
    case = CASES[name]
    trees = np.load(os.path.join(GOLD, "trees.npz"))
    knn = np.load(os.path.join(GOLD, "knn.npz"))
    ps = core.PointSet.create(case["coords"], case["ids"])
    ids = trees[f"{name}/ids"]
    pos = {int(v): j for j, v in enumerate(ps.ids)}
    perm = np.array([pos[int(v)] for v in ids], dtype=np.int64)
    nd = trees[f"{name}/node_dim"]
    leaf = nd < 0
    tree = lt.LocalTree(nd, trees[f"{name}/node_value"], trees[f"{name}/node_left"], trees[f"{name}/node_right"],
                        trees[f"{name}/node_count"], core.PointSet(np.ascontiguousarray(ps.coords[:, perm]), ids),
                        int(trees[f"{name}/depth"]), trees[f"{name}/node_left"][leaf].astype(np.int64),
                        trees[f"{name}/node_right"][leaf].astype(np.int64))
    for k in case["ks"]:
        d, i, c, _ = lq.find_knn_batch(tree, case["queries"], k)
        md, mi = masked(d, i, c)
        assert np.array_equal(c, knn[f"{name}/k{k}/brute_counts"])
        assert np.array_equal(md, knn[f"{name}/k{k}/brute_dists"])
        assert np.array_equal(mi, knn[f"{name}/k{k}/brute_ids"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_reference_walk_equals_reference_outputs_and_counters(api, name):
    """KD_KNN_REFERENCE replays local_query.py:72-172 on the device: dists, ids, counts and
    the (nodes visited, buckets scanned, points compared) counters equal what the real
    reference returned for the same tree and queries (golden), tie quirk included."""
    core, lt, lq = api
    case = CASES[name]
    knn = np.load(os.path.join(GOLD, "knn.npz"))
    ps = core.PointSet.create(case["coords"], case["ids"])
    tree = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
    for k in case["ks"]:
        d, i, c, ctr = lq.find_knn_batch(tree, case["queries"], k, reference_walk=True)
        assert np.array_equal(c, knn[f"{name}/k{k}/counts"])
        md, mi = masked(d, i, c)
        assert np.array_equal(md, knn[f"{name}/k{k}/dists"])
        assert np.array_equal(mi, knn[f"{name}/k{k}/ids"])
        assert np.array_equal(ctr, knn[f"{name}/k{k}/counters"])
    if case.get("radius") is not None:
        k = case["ks"][0]
        d, i, c, _ = lq.find_knn_batch(tree, case["queries"], k, radii=case["radius"], reference_walk=True)
        assert np.array_equal(c, knn[f"{name}/r/counts"])
        md, mi = masked(d, i, c)
        assert np.array_equal(md, knn[f"{name}/r/dists"]) and np.array_equal(mi, knn[f"{name}/r/ids"])


def test_reference_walk_keeps_the_tie_quirk(api):
    """the reference returns id 9 where the brute-force oracle returns id 3."""
    core, lt, lq = api
    case = CASES["q5_quirk"]
    ps = core.PointSet.create(case["coords"], case["ids"])
    tree = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
    _, i_ref, _, _ = lq.find_knn_batch(tree, case["queries"], 1, reference_walk=True)
    _, i_def, _, _ = lq.find_knn_batch(tree, case["queries"], 1)
    assert int(i_ref[0, 0]) == 9 and int(i_def[0, 0]) == 3


def test_count_visited_equals_reference_counters(api):
    core, lt, lq = api
    case = CASES["u3_2000"]
    knn = np.load(os.path.join(GOLD, "knn.npz"))
    ps = core.PointSet.create(case["coords"], case["ids"])
    tree = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
    k = case["ks"][0]
    want = knn[f"u3_2000/k{k}/counters"]
    for j in (0, 7, 19):
        c = lq.count_visited(tree, case["queries"][j], k)
        assert [c["nodes_visited"], c["buckets_scanned"], c["points_compared"]] == list(want[j])


def _caterpillar(core, lt, n):
    """A hand-made tree of depth n-1 (deeper than the fast kernels' fixed stack): node 2i splits
    the sorted 2-D points at x_{i+1}, its left child is the one-point leaf {x_i}."""
    xs = np.arange(n, dtype=np.float64) * 0.5 + np.linspace(0, 0.1, n)
    coords = np.stack([xs, np.sin(np.arange(n))]).astype(np.float64)
    ids = np.arange(100, 100 + n, dtype=np.uint64)
    nn = 2 * n - 1
    nd = np.full(nn, -1, np.int32); nv = np.zeros(nn); nl = np.zeros(nn, np.int32); nr = np.zeros(nn, np.int32)
    nc = np.zeros(nn, np.int64)
    for i in range(n - 1):
        p = 2 * i
        nd[p], nv[p], nl[p], nr[p], nc[p] = 0, xs[i + 1], p + 1, p + 2, n - i
        nl[p + 1], nr[p + 1], nc[p + 1] = i, 1, 1  # leaf: (start, length)
    nl[nn - 1], nr[nn - 1], nc[nn - 1] = n - 1, 1, 1
    leaf = nd < 0
    return lt.LocalTree(nd, nv, nl, nr, nc, core.PointSet(coords, ids), n - 1, nl[leaf].astype(np.int64),
                        nr[leaf].astype(np.int64)), coords, ids


def test_tree_deeper_than_the_fixed_stack(api, oracle):
    """depth 59 > KNN_MAX_DEPTH: kd_knn falls back to the depth-sized walk (kd_walk.cu)."""
    core, lt, lq = api
    tree, coords, ids = _caterpillar(core, lt, 60)
    q = np.random.default_rng(11).uniform([-1, -1], [31, 1], size=(500, 2))
    for k, kw in ((1, {}), (5, {}), (40, {}), (5, dict(radii=4.0)), (3, dict(exclude_ids=np.full(500, 130, np.uint64)))):
        d, i, c, _ = lq.find_knn_batch(tree, q, k, **kw)
        sel = ids != 130 if "exclude_ids" in kw else np.ones(len(ids), bool)
        bd, bi, bc = oracle.brute_knn(coords[:, sel], ids[sel], q, k, radii=kw.get("radii"))
        assert np.array_equal(c, bc)
        assert np.array_equal(masked(d, i, c)[0], masked(bd, bi, bc)[0])
        assert np.array_equal(masked(d, i, c)[1], masked(bd, bi, bc)[1])


def test_misaligned_device_input(oracle):
    """A device buffer that is only 4-byte aligned (a view one element into a tensor): the TMA tile
    loads need 16-byte-aligned sources, so the build copies such an input first."""
    import torch
    from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
    n = 70001
    rows = make_rows(n, 3, 9, "f32")
    flat = torch.empty(3 * n + 1, dtype=torch.float32, device="cuda")
    view = flat[1:].view(3, n)
    view.copy_(torch.from_numpy(np.ascontiguousarray(rows.T.astype(np.float32))))
    assert view.data_ptr() % 16 == 4 and view.is_contiguous()
    tree = build_local_tree_device(view, None, BuildConfig(bucket_size=32, seed=3))
    ref = oracle.build_tree(np.ascontiguousarray(rows.T), bucket_size=32, seed=3)
    for f in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(tree, f), getattr(ref, f)), f
    assert np.array_equal(tree.points.ids, ref.ids)


def test_radius_queries(api, oracle):
    core, lt, lq = api
    for name in ("u3_2000", "f32_u3_20000"):
        case = CASES[name]
        ps = core.PointSet.create(case["coords"], case["ids"])
        tree = lt.build_local_tree(ps, lt.BuildConfig(**case["cfg"]))
        for r in (case["radius"], 0.0, 1e-9):
            d, i, c, _ = lq.find_knn_batch(tree, case["queries"], 5, radii=r)
            bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, case["queries"], 5, radii=r)
            assert np.array_equal(c, bc)
            md, mi = masked(d, i, c)
            bmd, bmi = masked(bd, bi, bc)
            assert np.array_equal(md, bmd) and np.array_equal(mi, bmi)
        # per-query radii
        rr = np.random.default_rng(3).uniform(0, 0.02, size=case["queries"].shape[0])
        d, i, c, _ = lq.find_knn_batch(tree, case["queries"], 5, radii=rr)
        bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, case["queries"], 5, radii=rr)
        assert np.array_equal(c, bc)
        assert np.array_equal(masked(d, i, c)[1], masked(bd, bi, bc)[1])


def _digest(tree):
    h = hashlib.sha256()
    for a in (tree.node_dim.astype("<i4"), tree.node_value.astype("<f8"), tree.node_left.astype("<i4"),
              tree.node_right.astype("<i4"), tree.node_count.astype("<i8"), tree.points.ids.astype("<u8")):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.int64(tree.depth).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", sorted(big_cases()))
def test_big_tree_checksums(api, oracle, name):
    core, lt, lq = api
    with open(os.path.join(GOLD, "big_checksums.json")) as f:
        want = json.load(f)[name]
    coords, cfg, q, k = big_cases()[name]
    ps = core.PointSet.create(coords)
    tree = lt.build_local_tree(ps, lt.BuildConfig(**cfg))
    assert tree.n_nodes == want["n_nodes"] and tree.depth == want["depth"]
    assert _digest(tree) == want["tree_sha256"]
    d, i, c, _ = lq.find_knn_batch(tree, q, k)
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, k)
    assert np.array_equal(c, bc) and np.array_equal(d, bd) and np.array_equal(i, bi)


STRESS = [
    ("uniform", 3, 50_000, 32), ("duplicate-heavy", 3, 30_000, 16), ("halo-f32", 3, 80_000, 32),
    ("uniform", 2, 40_000, 8), ("uniform", 10, 20_000, 64), ("f32", 3, 150_000, 32), ("uniform", 1, 5000, 4),
    ("duplicate-heavy", 2, 6000, 1),
]


@pytest.mark.parametrize("kind,dims,n,bucket", STRESS)
@pytest.mark.parametrize("seed", [0, 1])
def test_stress_tree_and_knn_vs_oracle(api, oracle, kind, dims, n, bucket, seed):
    core, lt, lq = api
    rows = make_rows(n, dims, 500 + seed, kind)
    ps = core.PointSet.from_rows(rows)
    cfg = lt.BuildConfig(bucket_size=bucket, seed=seed)
    tree = lt.build_local_tree(ps, cfg)
    ref = oracle.build_tree(ps.coords, ps.ids, bucket_size=bucket, seed=seed)
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(tree, key), getattr(ref, key)), key
    assert np.array_equal(tree.points.ids, ref.ids) and tree.depth == ref.depth
    rng = np.random.default_rng(seed)
    q = np.concatenate([rng.uniform(rows.min(0), rows.max(0), size=(300, dims)), rows[:100]])
    for k in (1, 6, 17, 40):
        d, i, c, _ = lq.find_knn_batch(tree, q, k)
        bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, k)
        assert np.array_equal(c, bc)
        md, mi = masked(d, i, c)
        bmd, bmi = masked(bd, bi, bc)
        assert np.array_equal(md, bmd) and np.array_equal(mi, bmi)


def test_self_exclusion_matches_k_plus_one(api, oracle):
    core, lt, lq = api
    rows = make_rows(50_000, 3, 9, "halo-f32")
    ps = core.PointSet.from_rows(rows)
    tree = lt.build_local_tree(ps, lt.BuildConfig())
    sel = np.random.default_rng(1).choice(50_000, 2000, replace=False)
    q = rows[sel]
    d, i, c, _ = lq.find_knn_batch(tree, q, 5, exclude_ids=ps.ids[sel])
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, 6)
    for r in range(len(sel)):
        keep = bi[r, :bc[r]] != ps.ids[sel[r]]
        assert np.array_equal(d[r], bd[r, :bc[r]][keep][:5])
        assert np.array_equal(i[r], bi[r, :bc[r]][keep][:5])


@pytest.mark.parametrize("k,dims,kind", [(1, 3, "halo-f32"), (5, 3, "duplicate-heavy"), (10, 10, "f32"), (31, 3, "f32"),
                                          (32, 3, "halo-f32"), (40, 2, "f32")])
def test_exclusion_any_id_matches_oracle(api, oracle, k, dims, kind):
    """exclude_ids with self ids, ids of other points and ids absent from the tree:
    every row equals the brute-force top-k of the point set minus that id."""
    core, lt, lq = api
    rows = make_rows(20_000, dims, 31 + k, kind)
    ps = core.PointSet.from_rows(rows)
    tree = lt.build_local_tree(ps, lt.BuildConfig(bucket_size=16))
    rng = np.random.default_rng(k)
    sel = rng.choice(20_000, 1500, replace=False)
    q = rows[sel]
    ex = ps.ids[sel].copy()
    ex[::3] = ps.ids[rng.choice(20_000, len(ex[::3]))]   # some other point's id
    ex[1::7] = np.uint64(10**12)                          # an id not in the tree
    d, i, c, _ = lq.find_knn_batch(tree, q, k, exclude_ids=ex)
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, k + 1)
    for r in range(len(sel)):
        keep = bi[r, :bc[r]] != ex[r]
        wd, wi = bd[r, :bc[r]][keep][:k], bi[r, :bc[r]][keep][:k]
        assert c[r] == len(wd)
        assert np.array_equal(d[r, :c[r]], wd) and np.array_equal(i[r, :c[r]], wi)


def test_large_uniform_tree_and_sampled_knn(api, oracle):
    core, lt, lq = api
    rows = make_rows(2_000_000, 3, 21, "f32")
    ps = core.PointSet.from_rows(rows)
    tree = lt.build_local_tree(ps, lt.BuildConfig(seed=3))
    ref = oracle.build_tree(ps.coords, ps.ids, seed=3)
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(tree, key), getattr(ref, key)), key
    assert np.array_equal(tree.points.ids, ref.ids)
    q = np.random.default_rng(2).random((3000, 3), dtype=np.float32).astype(np.float64)
    d, i, c, _ = lq.find_knn_batch(tree, q, 5)
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, 5)
    assert np.array_equal(d, bd) and np.array_equal(i, bi)


def test_big_root_node_tree_parity(api, oracle):
    """A 5M-point clustered set: the root level exceeds 2^22 points (64-bit Fisher-Yates
    keys in k_sample) -- whole tree byte-equal to the oracle."""
    core, lt, lq = api
    rows = make_rows(5_000_000, 3, 91, "halo-f32")
    ps = core.PointSet.from_rows(rows)
    tree = lt.build_local_tree(ps, lt.BuildConfig(seed=13))
    ref = oracle.build_tree(ps.coords, ps.ids, seed=13)
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(tree, key), getattr(ref, key)), key
    assert np.array_equal(tree.points.ids, ref.ids) and tree.depth == ref.depth


@pytest.mark.parametrize("dims,kind,n,seed", [(3, "uniform", 6_000_000, 31), (2, "f32", 6_000_000, 32)])
def test_large_trees_binary64_and_2d(api, oracle, dims, kind, n, seed):
    """6M points that are NOT binary32-exact (binary64 storage: k_sample / fy_hash / k_scatter_tma
    instantiated for double) and 6M 2-D float points (the 2-D TMA partition): breadth-first levels
    with more than 1024 nodes of more than 4096 points, whole tree byte-equal to the oracle."""
    core, lt, lq = api
    rows = make_rows(n, dims, seed, kind)
    ps = core.PointSet.from_rows(rows)
    tree = lt.build_local_tree(ps, lt.BuildConfig(seed=seed))
    ref = oracle.build_tree(ps.coords, ps.ids, seed=seed)
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(tree, key), getattr(ref, key)), key
    assert np.array_equal(tree.points.ids, ref.ids) and tree.depth == ref.depth
    q = make_rows(2000, dims, seed + 1, kind)
    d, i, c, _ = lq.find_knn_batch(tree, q, 5)
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, 5)
    assert np.array_equal(c, bc) and np.array_equal(d, bd) and np.array_equal(i, bi)


def test_large_duplicate_heavy_tree_parity(api, oracle):
    """1.5M points, 40 % of them stacked on 50 sites: degenerate breadth-first nodes,
    constant dimensions, exact-fallback splits -- tree byte-equal, KNN equal to brute force."""
    core, lt, lq = api
    rng = np.random.default_rng(92)
    base = rng.random((900_000, 3), dtype=np.float32)
    sites = rng.random((50, 3), dtype=np.float32)
    rows = np.concatenate([base, sites[rng.integers(0, 50, 600_000)]]).astype(np.float64)
    ps = core.PointSet.from_rows(rows)
    tree = lt.build_local_tree(ps, lt.BuildConfig(seed=14))
    ref = oracle.build_tree(ps.coords, ps.ids, seed=14)
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        assert np.array_equal(getattr(tree, key), getattr(ref, key)), key
    assert np.array_equal(tree.points.ids, ref.ids)
    q = np.concatenate([sites[:20], rng.random((980, 3), dtype=np.float32)]).astype(np.float64)
    d, i, c, _ = lq.find_knn_batch(tree, q, 8)
    bd, bi, bc = oracle.brute_knn(ps.coords, ps.ids, q, 8)
    assert np.array_equal(c, bc) and np.array_equal(d, bd) and np.array_equal(i, bi)


class TestReferenceSemantics:
    """Reference test cases re-pointed at the drop-in (pkg/tests/test_local_query.py, test_local_tree.py)."""

    def test_single_point_tree(self, api):
        core, lt, lq = api
        ps = core.PointSet.from_rows([[0.5, 0.5]])
        res = lq.find_knn(lt.build_local_tree(ps, lt.BuildConfig(seed=0)), np.array([0.1, 0.9]), k=1)
        assert res.neighbors[0].point_id == 0
        assert res.neighbors[0].sq_dist == core.squared_distance(np.array([0.1, 0.9]), np.array([0.5, 0.5]))

    def test_tie_by_id(self, api):
        core, lt, lq = api
        ps = core.PointSet.from_rows([[0.3, 0.3], [0.3, 0.3], [0.9, 0.9]], ids=np.array([7, 2, 1], np.uint64))
        res = lq.find_knn(lt.build_local_tree(ps, lt.BuildConfig(seed=1)), np.array([0.3, 0.3]), k=1)
        assert res.neighbors[0].sq_dist == 0.0 and res.neighbors[0].point_id == 2

    def test_k_larger_than_n_and_empty(self, api):
        core, lt, lq = api
        ps = core.PointSet.from_rows(np.random.default_rng(5).uniform(size=(17, 3)))
        res = lq.find_knn(lt.build_local_tree(ps, lt.BuildConfig(seed=2)), np.zeros(3), k=50)
        assert len(res.neighbors) == 17 and res.r_prime == np.inf
        empty = lt.build_local_tree(core.PointSet.empty(2), lt.BuildConfig())
        assert empty.n_nodes == 0 and lq.find_knn(empty, np.zeros(2), k=3).neighbors == ()

    def test_counters(self, api):
        core, lt, lq = api
        ps = core.PointSet.from_rows(np.random.default_rng(0).uniform(size=(20, 2)))
        c = lq.count_visited(lt.build_local_tree(ps, lt.BuildConfig(bucket_size=32)), np.zeros(2), k=1)
        assert c == {"nodes_visited": 1, "buckets_scanned": 1, "points_compared": 20}
        ps = core.PointSet.from_rows(np.random.default_rng(1).uniform(size=(500, 2)))
        tree = lt.build_local_tree(ps, lt.BuildConfig(bucket_size=16, seed=1))
        c = lq.count_visited(tree, np.full(2, 0.5), k=500)
        assert c["buckets_scanned"] == tree.n_leaves and c["points_compared"] == 500

    def test_pruning_on_large_uniform(self, api):
        core, lt, lq = api
        ps = core.PointSet.from_rows(np.random.default_rng(7).uniform(size=(1_000_000, 3)))
        tree = lt.build_local_tree(ps, lt.BuildConfig(seed=7))
        _, _, _, ctr = lq.find_knn_batch(tree, np.random.default_rng(4).uniform(size=(100, 3)), k=5)
        assert ctr[:, 1].mean() / tree.n_leaves < 0.01

    def test_all_identical_degenerate_leaf(self, api):
        core, lt, _ = api
        tree = lt.build_local_tree(core.PointSet.from_rows(np.tile([1.5, 2.5], (1000, 1))), lt.BuildConfig(seed=3))
        assert tree.n_leaves == 1 and tree.node_count[0] == 1000

    def test_large_degenerate_leaf_above_shared_limit(self, api, oracle):
        core, lt, _ = api
        rows = np.concatenate([np.tile([0.25, 0.75, 0.5], (5000, 1)), make_rows(3000, 3, 4)])
        ps = core.PointSet.from_rows(rows)
        tree = lt.build_local_tree(ps, lt.BuildConfig(seed=1))
        ref = oracle.build_tree(ps.coords, ps.ids, seed=1)
        assert np.array_equal(tree.node_dim, ref.node_dim) and np.array_equal(tree.points.ids, ref.ids)
        assert (tree.leaf_lengths == 5000).sum() == 1
