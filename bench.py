#!/usr/bin/env python
"""Benchmark: kd-tree build (Mpoints/s) + exact KNN (queries/s) on B200.

Workload (BASELINE.json configs[2], SURVEY §8(d) "C3" -- the metric's "k=5 at
1/2/4/8 B200" config and the largest that fits one GPU): 256,000,000 float32
3D points in [0,1]x[0,0.5]x[0,0.25] (x, z uniform; y from a Harris current
sheet sech^2((y-0.25)/0.01) plus a 10 % uniform floor), 64,000,000 queries of
the same law, k=5, leaf bucket 32.  One step = build the whole kd-tree +
answer every query.  ``--config C1|C2|C4`` selects the other configs.

Printed JSON (one line, rank 0):
  value        build throughput, device-resident inputs (Mpoints/s)
  knn          query throughput for the same step (queries/s) + its roofline
  roofline     build: algorithmic bytes N*L*(8D+12) per build / build time vs
               the measured HBM copy bandwidth (MEASURED_PEAKS.json)
  e2e          the same two metrics through the C-ABI with pinned HOST buffers,
               host<->device copies inside the timed region
  cpu_baseline the reference algorithm (C oracle port, all host cores) on a
               bounded sample; its traversal over the (identical) full-size
               tree also yields the reference counters used by the query model
  --impl reference  times that CPU port as the reference arm

Multi-GPU (torchrun, N>1): weak scaling -- each rank owns its own 64M points
and 16M queries; see DESIGN.md §6 for the distributed engine.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    p.add_argument("--points", dest="n", type=int, default=None, help="override points per GPU (debug)")
    p.add_argument("--queries", dest="q", type=int, default=None, help="override queries per GPU (debug)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-build-sample", type=int, default=4_000_000)
    p.add_argument("--cpu-query-sample", type=int, default=200_000)
    p.add_argument("--no-ref-counters", action="store_true", help="skip the device replay of the reference walk")
    p.add_argument("--ref-counter-queries", type=int, default=4_000_000)
    return p.parse_args()


METRIC = "kd-tree build Mpoints/s and KNN queries/s (k=5) at 1/2/4/8 B200 vs HBM roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region (B200_PROFILING.md
    clocks line).  NVML is polled from a thread every ~2 ms (a C1 timed region lasts a few ms,
    shorter than nvidia-smi's start-up); nvidia-smi -lms 50 is the fallback."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.path = tempfile.mktemp(suffix=".csv")
        self.index = index
        self.proc = None
        self.thread = None
        self.rows = []
        self.stop_flag = False
        self.nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.nv = None

    def _poll(self):
        nv = self.nv
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        smax, pw, it = None, None, 0
        while True:
            try:
                if it % 16 == 0:  # the slow queries only now and then: a C1 timed region lasts a few ms
                    smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                    pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1e3
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.rows.append((float(sm), float(smax), pw, [k for k, b in bits.items() if rs & b]))
            except Exception:
                pass
            it += 1
            if self.stop_flag:
                break
            time.sleep(0.001)

    def start(self):
        if self.nv is not None:
            import threading
            self.stop_flag = False
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag = True
            self.thread.join(timeout=2)
            sm = sorted(r[0] for r in self.rows)
            reasons = sorted({x for r in self.rows for x in r[3]})
            return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.rows[-1][1] if self.rows else None,
                    "samples": len(sm), "power_w_max": max((r[2] for r in self.rows), default=None),
                    "reasons": reasons, "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        sm_load = sorted(sm)
        med = sm_load[len(sm_load) // 2] if sm_load else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "samples": len(sm), "power_w_max": max(power) if power else None,
                "reasons": sorted(reasons), "source": "nvidia-smi"}


def build_bytes(n, dims, leaf):
    """B_build = N * L * (8D + 12), L = ceil(log2(N / leaf))."""
    levels = max(1, math.ceil(math.log2(max(n / leaf, 2))))
    return n * levels * (8 * dims + 12), levels


def measured_traffic(config):
    """ncu DRAM bytes (read + write) per build and per query batch, committed under
    profiles/ by tools/traffic.py (C2 only; {} when absent)."""
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", f"{rnd}_traffic_{config.lower()}.json")
        try:
            with open(path) as f:
                d = json.load(f)
            d["file"] = os.path.relpath(path, ROOT)
            return d
        except (OSError, ValueError):
            continue
    return {}


def query_bytes(dims, k, v, c):
    """B_q = 4D + 8V + 4D*C + 16k (V, C: reference counters)."""
    return 4 * dims + 8 * v + 4 * dims * c + 16 * k


# ---------------------------------------------------------------------------------------------
def cpu_baseline_leg(cfgname, w, tree, sel_queries, args, seed=0):
    """The reference algorithm (C oracle port of kdknn build_local_tree /
    find_knn_batch) on the host cores: build of a bounded sample of the same
    law, and the reference traversal over the full-size tree (identical bytes to
    the GPU tree) for a query sample -> CPU rates + reference counters."""
    import numpy as np
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    nb = min(args.cpu_build_sample, w.n)
    from paper_1607_08220_b200.workloads import make_points
    rows = make_points(cfgname, "cuda", seed=77, n=nb).cpu().numpy()  # same law, bounded sample
    coords = np.ascontiguousarray(rows.T.astype(np.float64))
    O.build_tree(coords[:, :100_000], bucket_size=w.leaf, seed=seed, threads=cores)  # warm
    t0 = time.perf_counter()
    O.build_tree(coords, bucket_size=w.leaf, seed=seed, threads=cores)
    tb = time.perf_counter() - t0
    # reference traversal over the full tree for a query sample
    otree = O.OracleTree(tree.node_dim, tree.node_value, tree.node_left, tree.node_right, tree.node_count,
                         None, tree.points.coords, tree.points.ids, tree.depth)
    qs = sel_queries
    kk = w.k + (1 if w.queries_from_data else 0)
    t0 = time.perf_counter()
    rd, ri, rc, ctr = O.knn(otree, qs, kk, threads=cores)
    tq = time.perf_counter() - t0
    return {
        "rows": (rd, ri, rc),
        "build_mpts_s": nb / tb / 1e6, "build_sample_points": nb, "build_s": tb,
        "knn_q_s": qs.shape[0] / tq, "knn_sample_queries": int(qs.shape[0]), "knn_s": tq,
        "ref_nodes_visited": float(ctr[:, 0].mean()), "ref_points_compared": float(ctr[:, 2].mean()),
        "cores": cores,
    }


def reference_rows_check(ref_rows, od, oi, oc, excl, k):
    """This step's GPU rows for the first nq queries vs the reference traversal
    (oracle port of local_query.py:72-172) over the identical full-size tree.
    With self-exclusion the reference side is its k+1 search minus the query's
    own id, truncated to k.  Rows may differ only where the reference's
    bound >= r' pruning drops an exact tie: counted, not hidden."""
    import numpy as np
    rd, ri, rc = ref_rows
    nq = rd.shape[0]
    gd, gi, gc = od.cpu().numpy(), oi.cpu().numpy().view(np.uint64), oc.cpu().numpy()
    if excl is not None:
        ex = excl.cpu().numpy().astype(np.uint64)
        keep = (ri != ex[:, None]) & (np.arange(ri.shape[1])[None, :] < rc[:, None])
        pos = np.cumsum(keep, 1) - 1
        wd = np.zeros((nq, k)); wi = np.zeros((nq, k), np.uint64)
        sel = keep & (pos < k)
        r_idx, c_idx = np.nonzero(sel)
        wd[r_idx, pos[sel]] = rd[sel]
        wi[r_idx, pos[sel]] = ri[sel]
        rd, ri, rc = wd, wi, np.minimum(keep.sum(1), k)
    m = np.arange(k)[None, :] < gc[:, None]
    same = (gc == rc) & np.all(np.where(m, gd == rd[:, :k], True), 1) & np.all(np.where(m, gi == ri[:, :k], True), 1)
    return {"queries": int(nq), "rows_equal": int(same.sum()), "equal": bool(same.all()),
            "vs": "reference traversal (C oracle port) over the identical full-size tree: ids identical, "
                  "f64 distances bit-identical"}


def run_reference(args):
    """--impl reference: the reference algorithm (C oracle port) on host cores."""
    import numpy as np
    from oracle import oracle as O
    from paper_1607_08220_b200.workloads import CONFIGS, make_points_numpy
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    nb = min(args.cpu_build_sample, w.n)
    nqs = min(args.cpu_query_sample, w.q)
    try:
        rows = make_points_numpy(args.config, nb, seed=77)
    except ValueError:
        from paper_1607_08220_b200.workloads import make_points
        rows = make_points(args.config, "cpu", seed=77, n=nb).numpy()
    coords = np.ascontiguousarray(rows.T.astype(np.float64))
    rng = np.random.default_rng(5)
    sel = rng.choice(nb, size=min(nqs, nb), replace=False)
    queries = rows[sel].astype(np.float64)
    kk = w.k + (1 if w.queries_from_data else 0)
    tb_all, tq_all = [], []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        tree = O.build_tree(coords, bucket_size=w.leaf, seed=0, threads=cores)
        t1 = time.perf_counter()
        O.knn(tree, queries, kk, threads=cores)
        t2 = time.perf_counter()
        if step >= args.warmup:
            tb_all.append(t1 - t0)
            tq_all.append(t2 - t1)
    tb, tq = float(np.mean(tb_all)), float(np.mean(tq_all))
    value = nb / tb / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "Mpoints/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": (tb + tq) * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n": nb, "q": len(sel), "k": w.k, "leaf": w.leaf, "dims": w.dims,
                   "workload_n": w.n, "workload_q": w.q,
                   "sample": f"each step builds a {nb}-point tree of the {w.name} law and answers {len(sel)} "
                             f"queries against it (rates; the full {w.n}-point build takes minutes per step "
                             f"on the host)"},
        "knn": {"value": len(sel) / tq, "unit": "queries/s"},
        "cpu_baseline": {"value": value, "unit": "Mpoints/s", "cores": cores, "kind": "port",
                         "sample": f"build of {nb} points of the {w.name} law + {len(sel)} self-excluded "
                                   f"queries (k+1) against that tree, per step; C restatement of the reference "
                                   f"(oracle/kdknn_oracle.c), OpenMP {cores} threads"},
        "e2e": {"value": value, "unit": "Mpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------------------------
def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1607_08220_b200 import _native as N
    from paper_1607_08220_b200.local_query import find_knn_device
    from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
    from paper_1607_08220_b200.workloads import CONFIGS, make_points, make_queries

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    w = CONFIGS[args.config]
    n = args.n or w.n
    q = args.q or w.q
    rows = make_points(args.config, dev, seed=1000 + rank, n=n)
    coords = rows.t().contiguous()
    queries, excl = make_queries(args.config, rows, dev, seed=2000 + rank, q=q)
    cfg = BuildConfig(bucket_size=w.leaf, seed=0)
    stream = torch.cuda.current_stream(dev)
    # result buffers allocated once: a step measures the build and the search, not the allocator
    res_bufs = (torch.empty((q, w.k), dtype=torch.float64, device=dev), torch.empty((q, w.k), dtype=torch.int64,
                device=dev), torch.empty((q,), dtype=torch.int64, device=dev), None)
    torch.cuda.synchronize()

    def step(record=None):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tree = build_local_tree_device(coords, None, cfg)
        e1.record(stream)
        out = find_knn_device(tree, queries, w.k, exclude_ids=excl, out=res_bufs)
        e2.record(stream)
        return tree, out, (e0, e1, e2)

    for _ in range(args.warmup):
        tree, out, _ = step()
        del tree, out
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    evs = []
    levels = 0
    slow_nodes = 0
    tree = None
    for _ in range(args.steps):
        del tree
        tree, out, ev = step()
        evs.append(ev)
        levels = tree.build_info["levels"]
        slow_nodes = tree.build_info["slow_nodes"]
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    tb = sum(a.elapsed_time(b) for a, b, _ in evs) / len(evs) / 1e3
    tq = sum(b.elapsed_time(c) for _, b, c in evs) / len(evs) / 1e3
    if world > 1:
        t = torch.tensor([tb, tq], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tb, tq = t.tolist()

    # --- sanity: a sample of this step's results vs an exact fp64 brute force on device
    od, oi, oc, _ = out
    ok = True
    cols = [rows[:, d].to(torch.float64) for d in range(w.dims)]
    for j in range(min(16, q)):
        dd = (cols[0] - queries[j, 0]) ** 2
        for d in range(1, w.dims):
            dd += (cols[d] - queries[j, d]) ** 2
        if excl is not None:
            dd[excl[j]] = float("inf")
        kth = torch.topk(dd, w.k, largest=False).values.max()
        cand = torch.nonzero(dd <= kth).flatten()  # ascending ids
        order = torch.sort(dd[cand], stable=True).indices[:w.k]
        ok &= bool(torch.equal(od[j], dd[cand][order]) and torch.equal(oi[j], cand[order]))
    del cols

    # --- e2e through the C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        h_coords = coords.cpu().pin_memory()
        h_q = queries.cpu().pin_memory()
        h_ex = excl.cpu().pin_memory() if excl is not None else None
        h_d = torch.empty((q, w.k), dtype=torch.float64).pin_memory()
        h_i = torch.empty((q, w.k), dtype=torch.int64).pin_memory()
        h_c = torch.empty((q,), dtype=torch.int64).pin_memory()
        cfgn = cfg.native()
        st = C.c_void_p(stream.cuda_stream)
        tbe, tqe = [], []
        for it in range(2 + min(args.steps, 3)):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            c = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h = C.c_void_p()
            N.check(N.lib.kd_tree_build(h_coords.data_ptr(), N.KD_F32, n, w.dims, None, C.byref(cfgn), local, 0,
                                        st, C.byref(h)))
            b.record(stream)
            N.check(N.lib.kd_knn(h, h_q.data_ptr(), q, w.k, None,
                                 h_ex.data_ptr() if h_ex is not None else None, h_d.data_ptr(), h_i.data_ptr(),
                                 h_c.data_ptr(), None, 0, st))
            c.record(stream)
            torch.cuda.synchronize()
            N.lib.kd_tree_free(h)
            if it >= 2:
                tbe.append(a.elapsed_time(b) / 1e3)
                tqe.append(b.elapsed_time(c) / 1e3)
        tbe_m, tqe_m = float(np.mean(tbe)), float(np.mean(tqe))
        if world > 1:
            t = torch.tensor([tbe_m, tqe_m], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tbe_m, tqe_m = t.tolist()
        e2e = {"value": world * n / tbe_m / 1e6, "unit": "Mpoints/s",
               "knn": {"value": world * q / tqe_m, "unit": "queries/s"},
               "h2d_bytes_per_step": int(n * w.dims * 4 + q * w.dims * 8 + (q * 8 if excl is not None else 0)),
               "d2h_bytes_per_step": int(q * w.k * 16 + q * 8),
               "ms_build": tbe_m * 1e3, "ms_knn": tqe_m * 1e3,
               "path": "kd_tree_build + kd_knn (C-ABI) with pinned host buffers"}
        del h_coords, h_q, h_ex, h_d, h_i, h_c

    cpu = None
    ref_check = None
    if rank == 0 and not args.no_cpu_baseline:
        nqs = min(args.cpu_query_sample if w.dims <= 3 else 2000, q)  # 10-D queries scan ~1e5 points each
        qsel = queries[:nqs].cpu().numpy()
        cpu = cpu_baseline_leg(args.config, w, tree, qsel, args)
        ref_check = reference_rows_check(cpu.pop("rows"), od[:nqs], oi[:nqs], oc[:nqs],
                                         None if excl is None else excl[:nqs], w.k)

    # reference-definition counters on the device: KD_KNN_REFERENCE replays the reference's own
    # walk (local_query.py:72-172) over this tree; V, C of the query model come from it (a larger
    # sample than the host leg can afford) and are cross-checked against the oracle's on its sample
    gpu_ctr = None
    if rank == 0 and not args.no_ref_counters:
        kk = w.k + (1 if w.queries_from_data else 0)
        nref = min(q, args.ref_counter_queries if w.dims <= 3 else 20000)
        _, _, _, ctr = find_knn_device(tree, queries[:nref], kk, counters=True, flags=N.KD_KNN_REFERENCE)
        torch.cuda.synchronize()
        gpu_ctr = {"queries": int(nref), "V": float(ctr[:, 0].double().mean()), "C": float(ctr[:, 2].double().mean()),
                   "source": "KD_KNN_REFERENCE walk on the device (kd_walk.cu), reference definition"}
        if cpu is not None:
            m = min(nref, cpu["knn_sample_queries"])
            gpu_ctr["equal_oracle_counters"] = bool(
                abs(float(ctr[:m, 0].double().mean()) - cpu["ref_nodes_visited"]) < 1e-9 and
                abs(float(ctr[:m, 2].double().mean()) - cpu["ref_points_compared"]) < 1e-9) \
                if m == cpu["knn_sample_queries"] else None
        del ctr

    if rank == 0:
        peak, peak_kind = peaks()
        bbytes, levels_model = build_bytes(n, w.dims, w.leaf)
        ach_b = bbytes / tb / 1e9
        if gpu_ctr is not None:
            v_ref, c_ref = gpu_ctr["V"], gpu_ctr["C"]
            ctr_src = (f"reference-definition counters from the device replay of the reference walk over the "
                       f"full-size tree ({gpu_ctr['queries']} queries)")
        elif cpu is not None:
            v_ref, c_ref = cpu["ref_nodes_visited"], cpu["ref_points_compared"]
            ctr_src = "reference counters (oracle traversal over the identical full-size tree, sample)"
        else:
            # reference counters measured offline (C1 at full size, the others at 4M points)
            v_ref, c_ref = {"C1": (41.1, 149.8), "C2": (44.8, 156.3), "C3": (47.2, 152.4),
                            "C4": (5321.0, 117893.0)}[args.config]
            ctr_src = f"SURVEY §8(d) reference counters for {args.config}"
        qb = query_bytes(w.dims, w.k, v_ref, c_ref)
        ach_q = q * qb / tq / 1e9
        # build: 10 per breadth-first level (sample, tile info, hist, select, slow, tile-left, 2 scan,
        # scatter, children) + 2 per level preorder stitch + subtree, relocate, ids;
        # query: 3-D Morton keys (box + keys), CUB radix-sort kernels (32-bit keys), KNN (ncu list: 228 on C3)
        launches = 12 * levels + 3 + (9 if w.dims == 3 else 7)
        traffic = measured_traffic(args.config)
        line = {
            "metric": METRIC,
            "value": world * n / tb / 1e6, "unit": "Mpoints/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": (tb + tq) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n": n, "q": q, "k": w.k, "leaf": w.leaf, "dims": w.dims,
                       "coords": "float32 SoA (binary64 arithmetic)",
                       "l2": "inputs larger than L2 (points %.0f MB, queries %.0f MB)" % (n * w.dims * 4 / 1e6,
                                                                                      q * w.dims * 8 / 1e6),
                       "parallelism": f"weak x{world}"},
            "ms_build": tb * 1e3, "ms_knn": tq * 1e3,
            "roofline": {"bound": "hbm", "achieved": ach_b, "peak": peak, "unit": "GB/s", "frac": ach_b / peak,
                         "traffic": traffic.get("build_dram_bytes"), "traffic_source": traffic.get("source"),
                         "kernel": "whole build (all build kernels of one kd_tree_build)",
                         "algorithmic_bytes": bbytes, "model": f"N*L*(8D+12), L={levels_model}",
                         "peak_kind": peak_kind},
            "knn": {"value": world * q / tq, "unit": "queries/s",
                    "roofline": {"bound": "hbm", "achieved": ach_q, "peak": peak, "unit": "GB/s",
                                 "frac": ach_q / peak, "traffic": traffic.get("query_dram_bytes"),
                                 "kernel": ("query batch (Morton sort + k_knn_persist)" if w.dims <= 3
                                            else "query batch (home-leaf sort + k_knn_wq)"),
                                 "bytes_per_query": qb, "model": "4D+8V+4DC+16k", "V": v_ref, "C": c_ref,
                                 "counters": ctr_src, "gpu_reference_walk": gpu_ctr}},
            "sample_check_vs_fp64_bruteforce": {"queries": min(16, q), "equal": ok},
            "sample_check_vs_reference_traversal": ref_check,
            "build_levels": levels,
            "build_slow_nodes": slow_nodes,
            "build_phases_ms": {k: tree.build_info[k] for k in ("ms_levels", "ms_subtree", "ms_finish")},
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": None if cpu is None else {
                "value": cpu["build_mpts_s"], "unit": "Mpoints/s", "cores": cpu["cores"], "kind": "port",
                "knn_value": cpu["knn_q_s"], "knn_unit": "queries/s",
                "sample": f"build of {cpu['build_sample_points']} points of the same law; reference traversal of "
                          f"{cpu['knn_sample_queries']} queries over the full-size tree (k+1 for self-exclusion)"},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_b200_multi(args):
    """N > 1 (torchrun, one process per GPU): the PANDA global tier over NCCL.

    C3 (default): the config's 256M points / 64M queries at every N (strong
    scaling) -- 8 fixed shards of the C3 law, rank r of N generating shards
    [8r/N, 8(r+1)/N) on its GPU.  C5: one 250M-point shard (65,536 halos, ids >=
    2^32) and 62.5M fresh queries per GPU (weak scaling; 2B / 500M at N = 8).
    A step = global planes (sample all-gather + summed device histograms, NCCL) +
    alltoallv redistribution + local build, then the distributed query (route,
    local KNN, r' forwarding, radius KNN, device merge, results home) -- every
    array device-resident; time = max over ranks of CUDA-event time."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1607_08220_b200.cluster import ClusterConfig, DevicePoints, DeviceRegions, rank_build_global
    from paper_1607_08220_b200.comm import TorchComm
    from paper_1607_08220_b200.dist_query import QueryStats, rank_query
    from paper_1607_08220_b200.local_tree import BuildConfig, build_local_tree_device
    from paper_1607_08220_b200.workloads import C3_SHARDS, CONFIGS, make_shard

    if "WORLD_SIZE" not in os.environ:  # plain `python bench.py --config C5`: a one-rank process group
        os.environ.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(29400 + os.getpid() % 500))
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = TorchComm()
    cfgname = args.config if args.config in ("C3", "C5") else "C3"
    w = CONFIGS[cfgname]
    if cfgname == "C5":
        shards, scaling = [rank], "weak"
    else:
        if C3_SHARDS % world:
            raise SystemExit(f"C3 over {world} GPUs: use a divisor of {C3_SHARDS}")
        per = C3_SHARDS // world
        shards, scaling = list(range(rank * per, (rank + 1) * per)), "strong"
    parts = [make_shard(cfgname, s, dev, n=args.n, q=args.q) for s in shards]
    coords = torch.cat([p[0] for p in parts]).t().contiguous()
    ids = torch.cat([p[1] for p in parts])
    queries = torch.cat([p[2] for p in parts])
    del parts
    n, q = coords.shape[1], queries.shape[0]
    tot = torch.tensor([n, q], dtype=torch.int64, device=dev)
    dist.all_reduce(tot)
    n_total, q_total = (int(v) for v in tot.tolist())
    ccfg, bcfg = ClusterConfig(seed=0), BuildConfig(bucket_size=w.leaf, seed=0)
    stream = torch.cuda.current_stream(dev)
    slice_size = None  # one slice per step (the pipeline matters for the host API's small batches)

    def step(c_in, q_in):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        gt, pts, st = rank_build_global(comm, DevicePoints(c_in, ids), ccfg)
        tree = build_local_tree_device(pts.coords, pts.ids, bcfg)
        e[1].record(stream)
        qs = QueryStats(rank=rank)
        out = rank_query(comm, tree, DeviceRegions(gt, dev), q_in, w.k, slice_size=slice_size, stats=qs)
        e[2].record(stream)
        return tree, out, e, st, qs

    tree = out = None
    for _ in range(args.warmup):
        del tree, out
        tree, out, _, _, _ = step(coords, queries)
    torch.cuda.synchronize(); dist.barrier(); torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    evs, moved, fwd, req = [], 0, 0, 0
    for _ in range(args.steps):
        del tree, out
        tree, out, e, st, qs = step(coords, queries)
        evs.append(e)
        moved += st["points_moved"]
        fwd += qs.queries_forwarded
        req += qs.requests_sent
    torch.cuda.synchronize(); dist.barrier(); torch.cuda.synchronize()
    clk = clocks.stop()
    tb = sum(a.elapsed_time(b) for a, b, _ in evs) / len(evs) / 1e3
    tq = sum(b.elapsed_time(c) for _, b, c in evs) / len(evs) / 1e3
    t = torch.tensor([tb, tq], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tb, tq = t.tolist()
    cnt = torch.tensor([moved / args.steps, fwd / args.steps, req / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(cnt)
    # sanity: a sample of this rank's rows vs an fp64 brute force over ALL points (gathered)
    # e2e: pinned host inputs -> device -> distributed build + query -> results to host
    h_c = coords.cpu().pin_memory()
    h_q = queries.cpu().pin_memory()
    h_d = torch.empty((q, w.k), dtype=torch.float64).pin_memory()
    h_i = torch.empty((q, w.k), dtype=torch.int64).pin_memory()
    h_n = torch.empty((q,), dtype=torch.int64).pin_memory()
    te = []
    for it in range(2 + min(args.steps, 2)):
        del tree, out
        tree = out = None
        torch.cuda.synchronize(); dist.barrier()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dc = h_c.to(dev, non_blocking=True)
        dq = h_q.to(dev, non_blocking=True)
        tree, out, _, _, _ = step(dc, dq)
        od, oi, _, oc = out
        h_d.copy_(od, non_blocking=True); h_i.copy_(oi, non_blocking=True); h_n.copy_(oc, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        del dc, dq
        if it >= 2:
            te.append(a.elapsed_time(b) / 1e3)
    tt = torch.tensor([float(np.mean(te))], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    te_m = tt.item()
    if rank == 0:
        peak, peak_kind = peaks()
        per_gpu_n = n_total / world
        bbytes, levels_model = build_bytes(per_gpu_n, w.dims, w.leaf)
        ach_b = bbytes / tb / 1e9
        line = {
            "metric": METRIC,
            "value": n_total / tb / 1e6, "unit": "Mpoints/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": (tb + tq) * 1e3, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n": n_total, "q": q_total, "k": w.k, "leaf": w.leaf, "dims": w.dims,
                       "n_per_gpu": n, "q_per_gpu": q,
                       "parallelism": f"global kd-tree over {world} GPUs (NCCL all-to-all), {scaling} scaling",
                       "l2": "inputs larger than L2"},
            "ms_build": tb * 1e3, "ms_knn": tq * 1e3,
            "roofline": {"bound": "hbm", "achieved": ach_b, "peak": peak, "unit": "GB/s", "frac": ach_b / peak,
                         "traffic": None, "kernel": "per-GPU global tier + local build", "peak_kind": peak_kind,
                         "model": f"N/P*L*(8D+12) per GPU, L={levels_model}"},
            "knn": {"value": q_total / tq, "unit": "queries/s"},
            "points_moved_per_step": int(cnt[0].item()), "queries_forwarded_per_step": int(cnt[1].item()),
            "requests_per_step": int(cnt[2].item()),
            # local build (12 per level + 11) + global tier (split, unpack, hist per level) + query
            # (route x2, KNN x2, merge, sorts)
            "gpu_launches": 12 * (tree.build_info["levels"] if tree is not None else 20) + 11
                            + 4 * (world.bit_length() - 1) + 16,
            "clocks": clk,
            "e2e": {"value": n_total / te_m / 1e6, "unit": "Mpoints/s (build + query, host in/out)",
                    "h2d_bytes_per_step": int(n * w.dims * 4 + q * w.dims * 8),
                    "d2h_bytes_per_step": int(q * w.k * 16 + q * 8), "ms_step": te_m * 1e3},
            "cpu_baseline": None,
        }
        print(json.dumps(line))
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1 or os.environ.get("KDB_FORCE_GLOBAL") or args.config == "C5":
        run_b200_multi(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
