"""Aggregate an ncu --page source --print-source sass,cuda CSV by CUDA source line."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.defaultdict(lambda: [0.0, 0.0, '', 0.0])
fname, hdr = None, None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        ws, ie = hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
        te = hdr.index('Thread Instructions Executed') if 'Thread Instructions Executed' in hdr else None
        continue
    if hdr is None or len(r) <= ie:
        continue
    try:
        s, ins = float(r[ws] or 0), float(r[ie] or 0)
    except ValueError:
        continue
    a = agg[(fname, r[0])]
    a[0] += s
    a[1] += ins
    try:
        a[3] += float(r[te] or 0) if te is not None else 0.0
    except ValueError:
        pass
    if r[1].strip():
        a[2] = r[1].strip()[:100]
tot = sum(a[0] for a in agg.values())
toti = sum(a[1] for a in agg.values())
print('samples', tot, 'warp-instructions', toti, 'avg active threads', sum(a[3] for a in agg.values()) / max(toti, 1))
for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * a[0] / tot:5.1f}% {100 * a[1] / toti:5.1f}%i {a[3] / max(a[1], 1):4.1f}thr {k[0]}:{k[1]} {a[2]}")
