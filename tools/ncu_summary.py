"""Summarise one ncu --set full capture exported as CSV (details, raw, source pages):
    python tools/ncu_summary.py PREFIX   ->  PREFIX_details.csv, PREFIX_raw.csv, PREFIX_source.csv
Prints key metrics, DRAM bytes, the stall mix and the hottest CUDA source lines."""
import collections, csv, os, sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L2 Hit Rate', 'L1/TEX Hit Rate', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Compute (SM) Throughput', 'Executed Ipc Active',
        'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp', 'Grid Size', 'Block Size',
        'Dynamic Shared Memory Per Block', 'Static Shared Memory Per Block', 'Executed Instructions']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum']


def details(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    mi, vi, ui = h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    ki = h.index('Kernel Name')
    seen = {}
    for r in rows[1:]:
        if len(r) > vi and r[mi] in WANT and r[mi] not in seen:
            seen[r[mi]] = f"{r[vi]} {r[ui]}"
    return rows[1][ki] if len(rows) > 1 else '?', seen


def raw(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    out = {}
    for m in RAW:
        if m in h:
            i = h.index(m)
            out[m] = f"{v[i]} {u[i]}"
    stalls = {}
    for i, m in enumerate(h):
        if m.startswith('smsp__average_warp_latency_issue_stalled_') or m.startswith('smsp__average_warps_issue_stalled_'):
            if m.endswith('_per_issue_active.ratio'):
                try:
                    stalls[m.split('stalled_')[1].replace('_per_issue_active.ratio', '')] = float(v[i])
                except ValueError:
                    pass
    return out, stalls


def source(path, top=12):
    rows = list(csv.reader(open(path)))
    agg = collections.defaultdict(lambda: [0.0, 0.0, ''])
    fname, hdr = None, None
    for r in rows:
        if not r:
            continue
        if r[0] == 'File Path':
            fname = os.path.basename(r[1])
            continue
        if r[0] == 'Line No':
            hdr = r
            ws, ie = hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
            continue
        if hdr is None or len(r) <= ie or not r[0].strip():
            continue
        try:
            s, ins = float(r[ws] or 0), float(r[ie] or 0)
        except ValueError:
            continue
        a = agg[(fname, r[0])]
        a[0] += s
        a[1] += ins
        if r[1].strip():
            a[2] = r[1].strip()[:90]
    tot = sum(a[0] for a in agg.values()) or 1.0
    toti = sum(a[1] for a in agg.values()) or 1.0
    lines = [f"  {100 * a[0] / tot:5.1f}% stall-samples {100 * a[1] / toti:5.1f}% instr  {k[0]}:{k[1]}  {a[2]}"
             for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]]
    return lines


if __name__ == '__main__':
    for pre in sys.argv[1:]:
        name, d = details(pre + '_details.csv')
        print(f"===== {name[:150]}")
        for k in WANT:
            if k in d:
                print(f"  {k:40s} {d[k]}")
        if os.path.exists(pre + '_raw.csv'):
            r, st = raw(pre + '_raw.csv')
            for k, v in r.items():
                print(f"  {k:40s} {v}")
            if st:
                tot = sum(st.values()) or 1.0
                print('  stalls (cycles per issued instr): ' + ', '.join(
                    f"{k}={v:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
        if os.path.exists(pre + '_source.csv'):
            print('  hottest source lines:')
            print('\n'.join(source(pre + '_source.csv')))
