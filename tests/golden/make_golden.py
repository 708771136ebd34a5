"""Generate the golden fixtures that pin the oracle (and, through it, the GPU path).

Run ONCE in the development container, where the reference package is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the unmodified reference ``kdknn`` from /root/reference/pkg/src and
records, for seeded synthetic inputs, the reference's own outputs:

* ``primitives.npz`` -- SplitMix64 node seeds (median.py:69-71), Fisher-Yates
  draws (median.py:74-85), histograms (median.py:128-140) and median selections
  (median.py:143-166);
* ``trees.npz`` -- ``build_local_tree`` outputs (local_tree.py:436-574): node
  arrays, packed ids and depth for every case in CASES;
* ``knn.npz`` -- ``find_knn_batch`` outputs (local_query.py:175-216) over those
  trees and the ``oracle_topk`` brute force (pkg/tests/conftest.py:8-18);
* ``big_checksums.json`` -- sha256 of the tree arrays for larger inputs whose
  coordinates are regenerated from a seeded generator (too big to commit).

Nothing here (nor /root/reference) is read at GPU-test time; only the .npz/.json
fixtures travel.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from kdknn import median as M  # noqa: E402
from kdknn.core import PointSet  # noqa: E402
from kdknn.local_query import find_knn_batch  # noqa: E402
from kdknn.local_tree import BuildConfig, build_local_tree  # noqa: E402
from conftest import oracle_topk  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from datagen import golden_cases, big_cases, engine_cases  # noqa: E402


def tree_arrays(tree):
    return dict(node_dim=tree.node_dim.astype(np.int32), node_value=tree.node_value.astype(np.float64),
                node_left=tree.node_left.astype(np.int32), node_right=tree.node_right.astype(np.int32),
                node_count=tree.node_count.astype(np.int64), ids=tree.points.ids.astype(np.uint64),
                depth=np.int64(tree.depth))


def tree_digest(tree) -> str:
    h = hashlib.sha256()
    for a in (tree.node_dim.astype("<i4"), tree.node_value.astype("<f8"), tree.node_left.astype("<i4"),
              tree.node_right.astype("<i4"), tree.node_count.astype("<i8"), tree.points.ids.astype("<u8")):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.int64(tree.depth).tobytes())
    return h.hexdigest()


def primitives():
    out = {}
    seeds = []
    for s in (0, 1, 7, 2**63 + 5):
        for p in (1, 2, 3, 1000, 2**40 + 3):
            for salt in (0, 1, 4, 101):
                seeds.append((s, p, salt, int(M.derive_seed(s, p, salt))))
    out["seed_table"] = np.array(seeds, dtype=np.uint64)
    fy = []
    for (n, m, seed) in [(1, 1, 3), (5, 5, 9), (10, 3, 1), (1000, 1024 if 1000 >= 1024 else 1000, 42),
                         (5000, 1024, 7), (1 << 20, 1024, 11), (3000, 256, 2**63 + 1)]:
        idx = M._sample_indices(np.int64(n), np.int64(m), np.uint64(seed))
        fy.append((n, m, seed, np.asarray(idx, dtype=np.int64)))
    out["fy_params"] = np.array([(a, b, c) for a, b, c, _ in fy], dtype=np.uint64)
    for i, (_, _, _, idx) in enumerate(fy):
        out[f"fy_{i}"] = idx
    rng = np.random.default_rng(123)
    for i, (nv, nsamp) in enumerate([(1000, 64), (5000, 1024), (300, 300), (50, 7)]):
        vals = np.round(rng.normal(size=nv), 2)  # coarse values -> many exact ties
        iv = M.build_intervals(M.sample_values(vals, nsamp, seed=i))
        counts, equals = M.histogram_with_equals(vals, iv)
        bi, below = M._select_median(iv.boundaries, counts)
        out[f"hist_vals_{i}"] = vals
        out[f"hist_bnd_{i}"] = iv.boundaries
        out[f"hist_counts_{i}"] = counts
        out[f"hist_equals_{i}"] = equals
        out[f"hist_sel_{i}"] = np.array([bi, below], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **out)


def trees_and_knn():
    trees, knn = {}, {}
    for name, case in golden_cases().items():
        coords, ids, cfg, queries, ks, radius = (case["coords"], case["ids"], case["cfg"], case["queries"],
                                                 case["ks"], case.get("radius"))
        ps = PointSet.create(coords, ids)
        tree = build_local_tree(ps, BuildConfig(**cfg))
        for key, val in tree_arrays(tree).items():
            trees[f"{name}/{key}"] = val
        for k in ks:
            d, i, c, ctr = find_knn_batch(tree, queries, k)
            bd = np.zeros((queries.shape[0], k)); bi = np.zeros((queries.shape[0], k), np.uint64)
            bc = np.zeros(queries.shape[0], np.int64)
            for qi in range(queries.shape[0]):
                od, oi = oracle_topk(ps, queries[qi], k)
                bc[qi] = len(od); bd[qi, :len(od)] = od; bi[qi, :len(od)] = oi
            cm = np.arange(k)[None, :] < c[:, None]
            knn[f"{name}/k{k}/dists"] = np.where(cm, d, 0.0)
            knn[f"{name}/k{k}/ids"] = np.where(cm, i, 0).astype(np.uint64)
            knn[f"{name}/k{k}/counts"] = c
            knn[f"{name}/k{k}/counters"] = ctr
            knn[f"{name}/k{k}/brute_dists"] = bd
            knn[f"{name}/k{k}/brute_ids"] = bi
            knn[f"{name}/k{k}/brute_counts"] = bc
        if radius is not None:
            k = ks[0]
            d, i, c, ctr = find_knn_batch(tree, queries, k, radii=radius)
            cm = np.arange(k)[None, :] < c[:, None]
            knn[f"{name}/r/dists"] = np.where(cm, d, 0.0)
            knn[f"{name}/r/ids"] = np.where(cm, i, 0).astype(np.uint64)
            knn[f"{name}/r/counts"] = c
        print(f"  {name}: n={ps.count} D={ps.dims} nodes={tree.n_nodes} depth={tree.depth}")
    np.savez_compressed(os.path.join(HERE, "trees.npz"), **trees)
    np.savez_compressed(os.path.join(HERE, "knn.npz"), **knn)


def big():
    out = {}
    for name, (coords, cfg, queries, k) in big_cases().items():
        ps = PointSet.create(coords)
        tree = build_local_tree(ps, BuildConfig(**cfg, workers=8))
        d, i, c, ctr = find_knn_batch(tree, queries, k, workers=8)
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(d.astype("<f8")).tobytes())
        h.update(np.ascontiguousarray(i.astype("<u8")).tobytes())
        out[name] = {"tree_sha256": tree_digest(tree), "knn_sha256": h.hexdigest(),
                     "n_nodes": int(tree.n_nodes), "depth": int(tree.depth),
                     "mean_nodes_visited": float(ctr[:, 0].mean()),
                     "mean_points_compared": float(ctr[:, 2].mean())}
        print(f"  big {name}: {out[name]}")
    with open(os.path.join(HERE, "big_checksums.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def engine():
    """build_engine + Engine.query (engine.py:159-217) -> bundle digest, counters, results."""
    from kdknn.engine import RunConfig, build_engine, bundle_to_bytes
    out, arrays = {}, {}
    for name, (rows, cfg, queries, k) in engine_cases().items():
        ps = PointSet.from_rows(rows)
        eng, rep = build_engine(ps, RunConfig(**cfg))
        blob = bundle_to_bytes(eng)
        res, qrep = eng.query(queries, k=k)
        d = np.array([[n.sq_dist for n in r.neighbors] for r in res])
        i = np.array([[n.point_id for n in r.neighbors] for r in res], dtype=np.uint64)
        arrays[f"{name}/dists"] = d
        arrays[f"{name}/ids"] = i
        out[name] = {"bundle_sha256": hashlib.sha256(blob).hexdigest(), "bundle_len": len(blob),
                     "global_tree": eng.ranks[0].global_tree.to_bytes().hex(), "points_moved": rep.points_moved,
                     "rank_counts": [int(r.points.count) for r in eng.ranks],
                     "queries_forwarded": qrep.queries_forwarded, "requests_sent": qrep.requests_sent,
                     "requests_received": qrep.requests_received, "soundness_violations": qrep.soundness_violations,
                     "nodes_visited": qrep.nodes_visited, "points_compared": qrep.points_compared}
        print(f"  engine {name}: forwarded={qrep.queries_forwarded} moved={rep.points_moved}")
    with open(os.path.join(HERE, "engine.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "engine_knn.npz"), **arrays)


if __name__ == "__main__":
    primitives()
    trees_and_knn()
    big()
    engine()
