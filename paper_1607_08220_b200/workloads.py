"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The paper's cosmology / plasma / Daya Bay datasets are not available (no
network); these generators reproduce the shapes, sizes and value distributions
BASELINE.json names.  All coordinates are float32; ids are the row index.
Generation runs on the GPU with a seeded torch generator (a 64M-point host
array would take longer to make than to index).

  C1  uniform 3D          N=1,000,000   Q=100,000 same law        k=5  leaf 32
  C2  clustered 3D        N=64,000,000  Q=16,000,000 dataset rows k=5  leaf 32 (self excluded)
  C3  anisotropic sheet   N=256,000,000 Q=64,000,000 same law     k=5  leaf 32
  C4  10-D Gaussian mix   N=16,000,000  Q=4,000,000 same law      k=10 leaf 64
  C5  clustered 3D, 65,536 halos, N=2,000,000,000 over 8 GPUs (250M per GPU shard),
      Q=500,000,000 fresh draws (62.5M per shard), k=5, leaf 32, int64 ids >= 2^32

Multi-GPU runs generate per-shard data on each GPU (``make_shard``): the halo
catalogue (centres, widths, weights) is drawn once from a fixed seed, the points
of shard s from seed(s) -- torch's CUDA generator is counter-based (Philox), so
every GPU draws its own shard without a host array.  C3 keeps its stated total
N at any GPU count (8 fixed shards assigned to ranks: strong scaling); C5 is one
250M-point shard per GPU (weak scaling, 2B points at 8 GPUs) whose ids are
(shard << 32) | row -- all above 2^32 but shard 0's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    q: int
    dims: int
    k: int
    leaf: int
    queries_from_data: bool


CONFIGS = {
    "C1": Workload("C1-uniform3d", 1_000_000, 100_000, 3, 5, 32, False),
    "C2": Workload("C2-clustered3d", 64_000_000, 16_000_000, 3, 5, 32, True),
    "C3": Workload("C3-plasma3d", 256_000_000, 64_000_000, 3, 5, 32, False),
    "C4": Workload("C4-gauss10d", 16_000_000, 4_000_000, 10, 10, 64, False),
    "C5": Workload("C5-clustered3d-2B", 2_000_000_000, 500_000_000, 3, 5, 32, False),
}
C5_SHARDS = 8          # BASELINE configs[4]: 8 GPUs
C3_SHARDS = 8          # fixed partition of C3's 256M points / 64M queries for strong scaling


def _halo_catalogue(torch, nh, g, dev):
    centres = torch.rand((nh, 3), generator=g, device=dev, dtype=torch.float64)
    lo, hi = math.log(1e-3), math.log(1e-2)
    sig = torch.exp(torch.rand(nh, generator=g, device=dev, dtype=torch.float64) * (hi - lo) + lo)
    u = 1.0 - torch.rand(nh, generator=g, device=dev, dtype=torch.float64)  # (0, 1]
    w = u.pow(-1.0 / 1.5)  # Pareto(alpha=1.5, x_m=1) == numpy pareto(1.5) + 1
    return centres, sig, w


def _halo_rows(torch, n, nh, g, dev, catalogue=None):
    centres, sig, w = catalogue if catalogue is not None else _halo_catalogue(torch, nh, g, dev)
    n_bg = n // 5
    n_h = n - n_bg
    out = torch.empty((n, 3), device=dev, dtype=torch.float32)
    step = 1 << 26  # bounded f64 temporaries for the 250M-point shards
    for s in range(0, n_h, step):
        e = min(n_h, s + step)
        h = torch.multinomial(w, e - s, replacement=True, generator=g)
        pts = centres[h] + torch.randn((e - s, 3), generator=g, device=dev, dtype=torch.float64) * sig[h, None]
        out[s:e] = pts.remainder_(1.0).to(torch.float32)
        del h, pts
    for s in range(n_h, n, step):
        e = min(n, s + step)
        out[s:e] = torch.rand((e - s, 3), generator=g, device=dev, dtype=torch.float64).to(torch.float32)
    out[out >= 1.0] = 0.0  # periodic box: an f32 value rounded up to 1.0 wraps to 0
    return out


def _sheet_rows(torch, n, g, dev):
    x = torch.rand(n, generator=g, device=dev, dtype=torch.float64)
    z = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 0.25
    u = torch.rand(n, generator=g, device=dev, dtype=torch.float64).clamp_(1e-300, 1 - 1e-16)
    y_sheet = 0.25 + 0.005 * torch.log(u / (1 - u))  # logistic(0.25, s=0.005) ~ sech^2((y-.25)/.01)
    y_floor = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 0.5
    floor = torch.rand(n, generator=g, device=dev) < 0.10
    y = torch.where(floor, y_floor, y_sheet).clamp_(0.0, 0.5)
    return torch.stack([x, y, z], 1).to(torch.float32)


def _gauss10_rows(torch, n, g, dev, nc=64):
    means = torch.rand((nc, 10), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    a = torch.randn((nc, 10, 10), generator=g, device=dev, dtype=torch.float64)
    qm, r = torch.linalg.qr(a)
    qm = qm * torch.sign(torch.diagonal(r, dim1=1, dim2=2))[:, None, :]  # Haar
    lam = torch.exp(torch.rand((nc, 10), generator=g, device=dev, dtype=torch.float64) * math.log(1e3) - math.log(1e3))
    scale = qm * lam.sqrt()[:, None, :]  # Q diag(sqrt(lam))
    c = torch.randint(0, nc, (n,), generator=g, device=dev)
    z = torch.randn((n, 10), generator=g, device=dev, dtype=torch.float64)
    out = torch.empty((n, 10), device=dev, dtype=torch.float32)
    step = 1 << 22
    for s in range(0, n, step):
        e = min(n, s + step)
        out[s:e] = (means[c[s:e]] + torch.einsum("nij,nj->ni", scale[c[s:e]], z[s:e])).to(torch.float32)
    return out


def make_points(cfg: str, device="cuda", seed: int = 1000, n: int | None = None):
    """(n, dims) float32 CUDA tensor of points for config `cfg` (C1..C4)."""
    import torch
    w = CONFIGS[cfg]
    n = w.n if n is None else n
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if cfg == "C1":
        return torch.rand((n, 3), generator=g, device=device, dtype=torch.float32)
    if cfg == "C2":
        return _halo_rows(torch, n, 4096, g, device)
    if cfg == "C3":
        return _sheet_rows(torch, n, g, device)
    if cfg == "C4":
        return _gauss10_rows(torch, n, g, device)
    if cfg == "C5":  # one shard of the 65,536-halo law (the CPU baseline's bounded sample)
        return make_shard("C5", 0, device, n=n, q=1)[0]
    raise ValueError(cfg)


def make_shard(cfg: str, shard: int, device="cuda", n: int | None = None, q: int | None = None):
    """(points (n, 3) float32, ids (n,) int64, queries (q, 3) float64) of one shard.
    C5: 250M points / 62.5M queries per shard, 65,536-halo catalogue shared by all
    shards, ids (shard << 32) | row.  C3: 1/8 of its 256M points / 64M queries."""
    import torch
    w = CONFIGS[cfg]
    if cfg == "C5":
        n = w.n // C5_SHARDS if n is None else n
        q = w.q // C5_SHARDS if q is None else q
        gc = torch.Generator(device=device)
        gc.manual_seed(5005)
        cat = _halo_catalogue(torch, 65536, gc, device)
        g = torch.Generator(device=device)
        g.manual_seed(6000 + shard)
        pts = _halo_rows(torch, n, 65536, g, device, cat)
        g.manual_seed(7000 + shard)
        qs = _halo_rows(torch, q, 65536, g, device, cat).to(torch.float64)
        ids = torch.arange(n, dtype=torch.int64, device=device) + (shard << 32)
        return pts, ids, qs
    if cfg == "C3":
        n = w.n // C3_SHARDS if n is None else n
        q = w.q // C3_SHARDS if q is None else q
        g = torch.Generator(device=device)
        g.manual_seed(1100 + shard)
        pts = _sheet_rows(torch, n, g, device)
        g.manual_seed(2100 + shard)
        qs = _sheet_rows(torch, q, g, device).to(torch.float64)
        ids = torch.arange(n, dtype=torch.int64, device=device) + shard * n
        return pts, ids, qs
    raise ValueError(f"{cfg}: sharded generation is defined for C3 and C5")


def make_queries(cfg: str, rows, device="cuda", seed: int = 2000, q: int | None = None):
    """(queries (q, dims) float64, exclude_ids int64 or None).  C2 draws dataset
    rows without replacement and excludes each query's own id (self-match)."""
    import torch
    w = CONFIGS[cfg]
    q = w.q if q is None else q
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if w.queries_from_data:
        sel = torch.randperm(rows.shape[0], generator=g, device=device)[:q]
        return rows[sel].to(torch.float64), sel.to(torch.int64)
    if cfg == "C1":
        return torch.rand((q, 3), generator=g, device=device, dtype=torch.float32).to(torch.float64), None
    if cfg == "C3":
        return _sheet_rows(torch, q, g, device).to(torch.float64), None
    if cfg == "C4":
        return make_points("C4", device, seed=seed, n=q).to(torch.float64), None
    raise ValueError(cfg)


def make_points_numpy(cfg: str, n: int, seed: int = 1000):
    """Host (numpy) sample of the same law -- for the CPU baseline's bounded sample."""
    import numpy as np
    rng = np.random.default_rng(seed)
    if cfg == "C1":
        return rng.random((n, 3), dtype=np.float32)
    if cfg == "C2":
        nh = 4096
        centres = rng.random((nh, 3))
        sig = np.exp(rng.uniform(math.log(1e-3), math.log(1e-2), size=nh))
        w = rng.pareto(1.5, size=nh) + 1.0
        w /= w.sum()
        n_bg = n // 5
        h = rng.choice(nh, size=n - n_bg, p=w)
        rows = np.concatenate([centres[h] + rng.normal(size=(n - n_bg, 3)) * sig[h, None], rng.random((n_bg, 3))])
        rows = np.mod(rows, 1.0).astype(np.float32)
        rows[rows >= 1.0] = 0.0
        return rows
    raise ValueError(cfg)
