"""Device-resident distributed KNN for large batches (the 5-step protocol of
dist_query.py:186-341 with every per-query step on the GPU).

Per rank (SPMD over a communicator):
  1. ``kd_route`` gives each query's owner rank; queries travel to their owner
     with one all-to-all of device tensors (NCCL all_to_all_single over NVLink
     under ``TorchComm``).
  2. The owner runs ``kd_knn`` (r = inf); r' = k-th distance when full.
  3. ``kd_route`` with radii = r' gives, per query, the bitmask of other ranks
     whose region is strictly closer than r'; each (query, rank) pair becomes a
     request (id, coords, r') in a second all-to-all.
  4. Receivers run ``kd_knn`` with per-query radii r' and reply (k slots per
     request, count) in a third all-to-all.
  5. The owner merges its own k and the replies by (sq_dist, point_id) -- a
     stable device sort -- keeps k, and a fourth all-to-all returns the rows to
     the ingesting rank in its original order.

Results are identical to ``distributed_knn`` (and to the brute-force oracle).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

__all__ = ["rank_query_device", "DeviceRegions"]


class DeviceRegions:
    """The replicated global tree on a rank's device (planes + region boxes)."""

    def __init__(self, gt, device):
        import torch
        self.p = gt.rank_count
        self.dims = gt.dims
        lo, hi = gt.region_bounds()
        self.pdim = torch.as_tensor(np.ascontiguousarray(gt.plane_dims, dtype=np.int32)).to(device)
        self.pval = torch.as_tensor(np.ascontiguousarray(gt.plane_values, dtype=np.float64)).to(device)
        self.lo = torch.as_tensor(lo).to(device)
        self.hi = torch.as_tensor(hi).to(device)

    def route(self, q, radii=None, want_within=False):
        import torch
        nq = q.shape[0]
        owner = torch.empty(nq, dtype=torch.int32, device=q.device)
        within = torch.empty(nq, dtype=torch.int64, device=q.device) if want_within else None
        if nq:
            st = torch.cuda.current_stream(q.device).cuda_stream
            N.check(N.lib.kd_route(self.pdim.data_ptr() if self.p > 1 else None,
                                   self.pval.data_ptr() if self.p > 1 else None, self.p, self.lo.data_ptr(),
                                   self.hi.data_ptr(), q.data_ptr(), nq, self.dims,
                                   radii.data_ptr() if radii is not None else None, owner.data_ptr(),
                                   within.data_ptr() if want_within else None, N.KD_DEVICE_PTRS, C.c_void_p(st)))
        return owner, within


def _split_by(dest, p, *tensors):
    """Stable grouping of rows by destination rank -> {dest: tuple of row blocks}."""
    import torch
    order = torch.argsort(dest, stable=True)
    counts = torch.bincount(dest, minlength=p).cpu().tolist()
    out, off = {}, 0
    for r in range(p):
        if counts[r]:
            sel = order[off:off + counts[r]]
            out[r] = tuple(t[sel] for t in tensors)
        off += counts[r]
    return out


def _merge_topk(qidx, d, ids, nq, k):
    """Per query index keep the k smallest (d, id) pairs (lexicographic), sorted."""
    import torch
    # stable sorts: by id, then by d, then by query index  ->  (qidx, d, id) order
    o = torch.argsort(ids, stable=True)
    o = o[torch.argsort(d[o], stable=True)]
    o = o[torch.argsort(qidx[o], stable=True)]
    qs, ds, is_ = qidx[o], d[o], ids[o]
    counts = torch.bincount(qs, minlength=nq)
    starts = torch.cumsum(counts, 0) - counts
    rank = torch.arange(qs.shape[0], device=qs.device) - starts[qs]
    keep = rank < k
    out_d = torch.zeros((nq, k), dtype=torch.float64, device=qs.device)
    out_i = torch.zeros((nq, k), dtype=torch.int64, device=qs.device)
    out_d[qs[keep], rank[keep]] = ds[keep]
    out_i[qs[keep], rank[keep]] = is_[keep]
    return out_d, out_i, torch.clamp(counts, max=k)


def rank_query_device(comm, tree, regions: DeviceRegions, qids, q, k: int, excl=None, stats: dict | None = None):
    """One rank's side of the protocol for device tensors qids (int64), q (nq, D)
    float64 and optional excl (int64 point id per query, never returned).
    Returns (dists (nq,k), ids (nq,k) int64 bits of uint64, counts) in the input order."""
    import torch
    from .local_query import find_knn_device
    dev = q.device
    p = comm.size
    me = comm.rank
    nq = q.shape[0]
    if p == 1:  # one rank owns every query: the local search is the answer
        if nq and tree.count:
            d, i, c, _ = find_knn_device(tree, q.contiguous(), k, exclude_ids=excl)
            return d, i, c
        return (torch.zeros((nq, k), dtype=torch.float64, device=dev), torch.zeros((nq, k), dtype=torch.int64, device=dev),
                torch.zeros(nq, dtype=torch.int64, device=dev))
    local_pos = torch.arange(nq, device=dev, dtype=torch.int64)
    ex = excl if excl is not None else torch.full((nq,), -1, dtype=torch.int64, device=dev)
    # 1. route to owners
    owner, _ = regions.route(q)
    sends = _split_by(owner.long(), p, local_pos, q, ex)
    got = comm.alltoall(sends) if p > 1 else {0: sends.get(0, (local_pos[:0], q[:0], ex[:0]))}
    srcs = sorted(got)
    src_of = torch.cat([torch.full((got[s][0].shape[0],), s, dtype=torch.int64, device=dev) for s in srcs]) \
        if srcs else torch.empty(0, dtype=torch.int64, device=dev)
    o_pos = torch.cat([got[s][0] for s in srcs]) if srcs else local_pos[:0]
    o_q = torch.cat([got[s][1] for s in srcs]).contiguous() if srcs else q[:0]
    o_ex = torch.cat([got[s][2] for s in srcs]).contiguous() if srcs else ex[:0]
    m = o_q.shape[0]
    # 2. local KNN, r'
    if m and tree.count:
        ld, li, lc, _ = find_knn_device(tree, o_q, k, exclude_ids=o_ex if excl is not None else None)
    else:
        ld = torch.zeros((m, k), dtype=torch.float64, device=dev)
        li = torch.zeros((m, k), dtype=torch.int64, device=dev)
        lc = torch.zeros(m, dtype=torch.int64, device=dev)
    md, mi, mc = ld, li, lc  # queries nobody else can improve keep their local rows
    forwarded = 0
    n_req = 0
    if p > 1:
        rp = torch.where(lc == k, ld[:, k - 1], torch.full_like(ld[:, 0], float("inf"))) if m else ld[:, 0]
        # 3. forward to ranks within r'
        _, within = regions.route(o_q, radii=rp.contiguous(), want_within=True)
        fq = torch.nonzero(within != 0).flatten()  # owned queries with requests (ascending)
        forwarded = int(fq.shape[0])
        bits = ((within[fq][:, None] >> torch.arange(p, device=dev)[None, :]) & 1).bool()  # (f, p)
        rf, rr = torch.nonzero(bits, as_tuple=True)
        rq = fq[rf]
        n_req = int(rq.shape[0])
        req = _split_by(rr, p, rq, o_q[rq], rp[rq], o_ex[rq])
        inbox = comm.alltoall(req)
        # 4. serve requests with radius r'
        replies = {}
        for s in sorted(inbox):
            tq, tc, tr, te = inbox[s]
            if tq.shape[0] and tree.count:
                dd, ii, cc, _ = find_knn_device(tree, tc.contiguous(), k, radii=tr.contiguous(),
                                                exclude_ids=te.contiguous() if excl is not None else None)
            else:
                dd = torch.zeros((tq.shape[0], k), dtype=torch.float64, device=dev)
                ii = torch.zeros((tq.shape[0], k), dtype=torch.int64, device=dev)
                cc = torch.zeros(tq.shape[0], dtype=torch.int64, device=dev)
            replies[s] = (tq, dd, ii, cc)
        back = comm.alltoall(replies)
        # 5. merge (sq_dist, id) for the forwarded queries only (local slot f = position in fq)
        if forwarded:
            slot_of = torch.full((m,), -1, dtype=torch.int64, device=dev)
            slot_of[fq] = torch.arange(forwarded, device=dev)
            karange = torch.arange(k, device=dev)
            cand_q = [torch.arange(forwarded, device=dev).repeat_interleave(k)]
            cand_d, cand_i = [ld[fq].reshape(-1)], [li[fq].reshape(-1)]
            ok = [(karange[None, :] < lc[fq][:, None]).reshape(-1)]
            for s in sorted(back):
                tq, dd, ii, cc = back[s]
                cand_q.append(slot_of[tq].repeat_interleave(k))
                cand_d.append(dd.reshape(-1))
                cand_i.append(ii.reshape(-1))
                ok.append((karange[None, :] < cc[:, None]).reshape(-1))
            okm = torch.cat(ok)
            cq, cd, ci = torch.cat(cand_q)[okm], torch.cat(cand_d)[okm], torch.cat(cand_i)[okm]
            # uint64 order == int64 order of the bits for ids < 2^63
            fd, fi, fc = _merge_topk(cq, cd, ci, forwarded, k)
            md, mi, mc = ld.clone(), li.clone(), lc.clone()
            md[fq], mi[fq], mc[fq] = fd, fi, fc
    if p == 1:
        out_d, out_i, out_c = torch.zeros((nq, k), dtype=torch.float64, device=dev), \
            torch.zeros((nq, k), dtype=torch.int64, device=dev), torch.zeros(nq, dtype=torch.int64, device=dev)
        out_d[o_pos], out_i[o_pos], out_c[o_pos] = md, mi, mc
    else:
        # return rows to the ingesting rank
        home = _split_by(src_of, p, o_pos, md, mi, mc)
        ret = comm.alltoall(home)
        out_d = torch.zeros((nq, k), dtype=torch.float64, device=dev)
        out_i = torch.zeros((nq, k), dtype=torch.int64, device=dev)
        out_c = torch.zeros(nq, dtype=torch.int64, device=dev)
        for s in ret:
            pos, dd, ii, cc = ret[s]
            out_d[pos] = dd
            out_i[pos] = ii
            out_c[pos] = cc
    if stats is not None:
        stats["queries_forwarded"] = stats.get("queries_forwarded", 0) + forwarded
        stats["requests_sent"] = stats.get("requests_sent", 0) + n_req
        stats["queries_owned"] = stats.get("queries_owned", 0) + m
    return out_d, out_i, out_c
