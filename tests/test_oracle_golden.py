"""Pin the C oracle against the real reference (golden fixtures from tests/golden/make_golden.py).

CPU-only.  If these pass, the oracle reproduces the reference byte for byte:
SplitMix64 seeds, Fisher-Yates draws, histograms, median selection, whole
local trees (node arrays, packed ids, depth) and KNN outputs incl. counters.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from datagen import big_cases, golden_cases

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def prim():
    return np.load(os.path.join(GOLD, "primitives.npz"))


@pytest.fixture(scope="module")
def trees():
    return np.load(os.path.join(GOLD, "trees.npz"))


@pytest.fixture(scope="module")
def knn():
    return np.load(os.path.join(GOLD, "knn.npz"))


CASES = golden_cases()


def test_node_seed_table(oracle, prim):
    for s, p, salt, want in prim["seed_table"]:
        assert oracle.node_seed(int(s), int(p), int(salt)) == int(want)


def test_fisher_yates_draws(oracle, prim):
    for i, (n, m, seed) in enumerate(prim["fy_params"]):
        got = oracle.sample_indices(int(n), int(m), int(seed))
        assert np.array_equal(got, prim[f"fy_{i}"])


def test_histogram_and_select(oracle, prim):
    for i in range(4):
        counts, equals = oracle.histogram(prim[f"hist_vals_{i}"], prim[f"hist_bnd_{i}"])
        assert np.array_equal(counts, prim[f"hist_counts_{i}"])
        assert np.array_equal(equals, prim[f"hist_equals_{i}"])
        assert list(oracle.select_median(counts)) == prim[f"hist_sel_{i}"].tolist()


def test_known_answers(oracle):
    # reference tests/test_median.py:117-156 bin conventions and medians
    c, _ = oracle.histogram([0.5, 1.5, 2.5], [1.0, 2.0, 3.0])
    assert c.tolist() == [1, 1, 1, 0]
    c, _ = oracle.histogram([1.0, 2.0, 3.0], [1.0, 2.0, 3.0])
    assert c.tolist() == [0, 1, 1, 1]
    c, e = oracle.histogram([1.0, 1.0, 1.5, 2.0, 0.0], [1.0, 2.0])
    assert c.tolist() == [1, 3, 1] and e.tolist() == [2, 1]
    assert oracle.select_median([0, 5, 5, 0])[0] == 1
    assert oracle.select_median([0, 0])[0] == -1


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("threads", [1, 4])
def test_tree_bytes_match_reference(oracle, trees, name, threads):
    case = CASES[name]
    t = oracle.build_tree(case["coords"], case["ids"], threads=threads, **case["cfg"])
    for key in ("node_dim", "node_value", "node_left", "node_right", "node_count"):
        want = trees[f"{name}/{key}"]
        got = getattr(t, key)
        assert got.dtype == want.dtype and np.array_equal(got, want), key
    assert np.array_equal(t.ids, trees[f"{name}/ids"])
    assert t.depth == int(trees[f"{name}/depth"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_knn_matches_reference(oracle, knn, name):
    case = CASES[name]
    t = oracle.build_tree(case["coords"], case["ids"], **case["cfg"])
    q = case["queries"]
    for k in case["ks"]:
        d, i, c, ctr = oracle.knn(t, q, k)
        cm = np.arange(k)[None, :] < c[:, None]
        assert np.array_equal(c, knn[f"{name}/k{k}/counts"])
        assert np.array_equal(np.where(cm, d, 0.0), knn[f"{name}/k{k}/dists"])
        assert np.array_equal(np.where(cm, i, 0), knn[f"{name}/k{k}/ids"])
        assert np.array_equal(ctr, knn[f"{name}/k{k}/counters"])
        bd, bi, bc = oracle.brute_knn(case["coords"], case["ids"], q, k)
        assert np.array_equal(bc, knn[f"{name}/k{k}/brute_counts"])
        bm = np.arange(k)[None, :] < bc[:, None]
        assert np.array_equal(np.where(bm, bd, 0.0), knn[f"{name}/k{k}/brute_dists"])
        assert np.array_equal(np.where(bm, bi, 0), knn[f"{name}/k{k}/brute_ids"])
    if case["radius"] is not None:
        k = case["ks"][0]
        d, i, c, _ = oracle.knn(t, q, k, radii=case["radius"])
        cm = np.arange(k)[None, :] < c[:, None]
        assert np.array_equal(c, knn[f"{name}/r/counts"])
        assert np.array_equal(np.where(cm, d, 0.0), knn[f"{name}/r/dists"])
        assert np.array_equal(np.where(cm, i, 0), knn[f"{name}/r/ids"])


def test_q5_quirk_recorded(knn):
    # the reference prunes `bound >= r'` and loses an exact
    # tie with a smaller id; the brute-force oracle (the parity target) keeps it.
    assert int(knn["q5_quirk/k1/ids"][0, 0]) == 9
    assert int(knn["q5_quirk/k1/brute_ids"][0, 0]) == 3


def _digest(t):
    h = hashlib.sha256()
    for a in (t.node_dim.astype("<i4"), t.node_value.astype("<f8"), t.node_left.astype("<i4"),
              t.node_right.astype("<i4"), t.node_count.astype("<i8"), t.ids.astype("<u8")):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.int64(t.depth).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", sorted(big_cases()))
def test_big_tree_checksums(oracle, name):
    with open(os.path.join(GOLD, "big_checksums.json")) as f:
        want = json.load(f)[name]
    coords, cfg, q, k = big_cases()[name]
    t = oracle.build_tree(coords, **cfg, threads=0)
    assert t.n_nodes == want["n_nodes"] and t.depth == want["depth"]
    assert _digest(t) == want["tree_sha256"]
    d, i, c, ctr = oracle.knn(t, q, k)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(d.astype("<f8")).tobytes())
    h.update(np.ascontiguousarray(i.astype("<u8")).tobytes())
    assert h.hexdigest() == want["knn_sha256"]
