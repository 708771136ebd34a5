"""Seeded synthetic inputs shared by the golden-fixture generator and the tests.

Every array is a pure function of its seed (numpy PCG64), so the fixture
generator (run once against the real reference) and the tests (run here and on
the GPU box) see identical inputs.  Generators follow the reference tests'
data shapes: ``make_points`` mirrors pkg/tests/test_local_query.py:10-21
(uniform / duplicate-heavy), the anisotropic/constant-dimension/identical
cases mirror pkg/tests/test_local_tree.py:82-95 and :148-153.
"""

from __future__ import annotations

import numpy as np


def make_rows(n, dims, seed, kind="uniform"):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.uniform(size=(n, dims))
    if kind == "duplicate-heavy":
        rows = rng.uniform(size=(n, dims))
        n_dup = max(1, int(0.4 * n))
        sites = rows[rng.integers(0, max(1, n - n_dup), size=n_dup)]
        rows[n - n_dup:] = sites
        return rows
    if kind == "f32":
        return rng.random((n, dims), dtype=np.float32).astype(np.float64)
    if kind == "halo-f32":
        # clustered 3D stand-in for BASELINE config 2 (small): Gaussian halos + 20% uniform, wrapped mod 1
        nh = 64
        centres = rng.random((nh, dims))
        sig = np.exp(rng.uniform(np.log(1e-3), np.log(1e-2), size=nh))
        w = rng.pareto(1.5, size=nh) + 1.0
        w /= w.sum()
        n_bg = n // 5
        h = rng.choice(nh, size=n - n_bg, p=w)
        pts = centres[h] + rng.normal(size=(n - n_bg, dims)) * sig[h, None]
        rows = np.concatenate([pts, rng.random((n_bg, dims))])
        rows = np.mod(rows, 1.0).astype(np.float32)
        rows[rows >= 1.0] = 0.0
        return rows.astype(np.float64)
    raise ValueError(kind)


def golden_cases():
    """name -> dict(coords (D,n) f64, ids u64, cfg BuildConfig kwargs, queries, ks, radius)."""
    cases = {}

    def add(name, rows, cfg, nq=40, ks=(5,), radius=None, ids=None, qseed=None, extra_q=8):
        rows = np.asarray(rows, dtype=np.float64)
        n, dims = rows.shape
        rng = np.random.default_rng(1000 + len(cases) if qseed is None else qseed)
        lo = rows.min(axis=0) if n else np.zeros(dims)
        hi = rows.max(axis=0) if n else np.ones(dims)
        q = rng.uniform(lo - 0.05 * (hi - lo + 1e-9), hi + 0.05 * (hi - lo + 1e-9), size=(nq, dims))
        if n:
            q = np.concatenate([q, rows[: min(extra_q, n)]])
        cases[name] = dict(coords=np.ascontiguousarray(rows.T),
                           ids=np.arange(n, dtype=np.uint64) if ids is None else np.asarray(ids, np.uint64),
                           cfg=cfg, queries=np.ascontiguousarray(q), ks=tuple(ks), radius=radius)

    add("u3_2000", make_rows(2000, 3, 1), dict(bucket_size=32, seed=0), ks=(1, 5, 40), radius=0.01)
    add("u2_300_b8", make_rows(300, 2, 2), dict(bucket_size=8, seed=3), ks=(1, 3, 300))
    add("dup2_2000_b8", make_rows(2000, 2, 9, "duplicate-heavy"), dict(bucket_size=8, seed=9), ks=(3, 7))
    add("d10_3000_b64", make_rows(3000, 10, 21), dict(bucket_size=64, seed=21), ks=(7, 10))
    add("f32_u3_20000", make_rows(20000, 3, 42, "f32"), dict(bucket_size=32, seed=42), ks=(5, 6), radius=0.0004)
    add("halo3_20000", make_rows(20000, 3, 77, "halo-f32"), dict(bucket_size=32, seed=5), ks=(5,))
    for n in (1, 2, 3, 33):
        add(f"tiny{n}", make_rows(n, 2, n), dict(bucket_size=8, seed=n), ks=(1, 3, n), nq=8)
    add("identical_1000", np.tile([1.5, 2.5], (1000, 1)), dict(seed=3), ks=(4,), nq=6)
    rng = np.random.default_rng(17)
    add("mixed_dups_b8", np.concatenate([rng.uniform(size=(100, 2)), np.tile([0.5, 0.5], (40, 1))]),
        dict(bucket_size=8, seed=7), ks=(1, 5, 50))
    rng = np.random.default_rng(9)
    base = rng.uniform(size=(400, 2))
    add("dup_sites_1000", np.concatenate([base, np.tile(base[0], (300, 1)), np.tile(base[1], (300, 1))]),
        dict(seed=4), ks=(3, 11))
    rng = np.random.default_rng(31)
    add("constdim3_3000", np.stack([rng.uniform(size=3000), rng.uniform(size=3000), np.full(3000, 0.25)], 1),
        dict(seed=2), ks=(5,))
    rng = np.random.default_rng(32)
    add("aniso3_5000", np.stack([rng.uniform(0, 100, 5000), rng.uniform(0, 1, 5000), rng.uniform(0, 0.01, 5000)], 1),
        dict(seed=6, local_sample_m=256, variance_sample=128), ks=(5,))
    rng = np.random.default_rng(33)
    add("grid2_4096_b4", np.stack(np.meshgrid(np.arange(64.0), np.arange(64.0)), -1).reshape(-1, 2),
        dict(bucket_size=4, seed=1), ks=(1, 4, 9))
    add("ids_perm_1500", make_rows(1500, 3, 34), dict(seed=8), ks=(5,),
        ids=np.random.default_rng(35).permutation(10**6)[:1500].astype(np.uint64) * 7 + 3)
    # exact tie at a pruned boundary (reference returns id 9, oracle id 3)
    add("q5_quirk", [[-3, 0], [-2, 0], [-1, 0], [1, 0], [5, 0], [6, 0]], dict(bucket_size=1, seed=0),
        ks=(1, 2), nq=0, ids=np.array([10, 11, 9, 3, 12, 13], np.uint64))
    cases["q5_quirk"]["queries"] = np.array([[0.0, 0.0], [2.0, 0.0], [-2.0, 0.0]])
    return cases


def big_cases():
    """Larger inputs pinned by checksum only: name -> (coords (D,n), cfg, queries, k)."""
    out = {}
    rows = make_rows(300_000, 3, 7, "f32")
    q = np.random.default_rng(8).random((5000, 3), dtype=np.float32).astype(np.float64)
    out["f32_u3_300k"] = (np.ascontiguousarray(rows.T), dict(bucket_size=32, seed=7), q, 5)
    rows = make_rows(200_000, 3, 78, "halo-f32")
    out["halo3_200k"] = (np.ascontiguousarray(rows.T), dict(bucket_size=32, seed=11), rows[:3000].copy(), 6)
    rows = make_rows(100_000, 10, 79, "f32")
    q = np.random.default_rng(80).random((300, 10), dtype=np.float32).astype(np.float64)
    out["f32_u10_100k_b64"] = (np.ascontiguousarray(rows.T), dict(bucket_size=64, seed=12), q, 10)
    return out


def engine_cases():
    """Multi-rank cases for build_engine / Engine.query: name -> (rows, RunConfig kwargs, queries, k)."""
    out = {}

    def q_for(rows, seed, nq=300):
        rng = np.random.default_rng(seed)
        lo, hi = rows.min(0), rows.max(0)
        return np.concatenate([rng.uniform(lo, hi, size=(nq - 50, rows.shape[1])), rows[:50]])

    rows = make_rows(20000, 3, 5)
    out["eng_u3_20000_p4"] = (rows, dict(ranks=4, seed=5), q_for(rows, 1), 5)
    out["eng_u3_20000_p8"] = (rows, dict(ranks=8, seed=6), q_for(rows, 2), 5)
    rows = make_rows(50000, 3, 11, "f32")
    out["eng_f32_50000_p2"] = (rows, dict(ranks=2, seed=11), q_for(rows, 3), 6)
    rows = make_rows(2000, 2, 9, "duplicate-heavy")
    out["eng_dup2_2000_p4"] = (rows, dict(ranks=4, seed=9), q_for(rows, 4), 3)
    rows = make_rows(5000, 3, 13)
    out["eng_u3_5000_p16"] = (rows, dict(ranks=16, seed=13, batch_size=64), q_for(rows, 5), 5)
    rows = make_rows(40000, 3, 17, "halo-f32")
    out["eng_halo_40000_p8"] = (rows, dict(ranks=8, seed=2, bucket_size=16), q_for(rows, 6), 5)
    rows = make_rows(6000, 10, 19)
    out["eng_d10_6000_p4"] = (rows, dict(ranks=4, seed=3, bucket_size=64), q_for(rows, 7, 100), 7)
    return out
