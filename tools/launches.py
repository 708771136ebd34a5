"""Summarise an ncu launch list (gpu__time_duration) for the last build+query step."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, idi = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID')
seq = []
for r in rows[hi + 1:]:
    try:
        seq.append((int(r[idi]), r[ki], float(r[vi].replace(',', ''))))
    except (ValueError, IndexError):
        pass
inits = [i for i, (_, n, _) in enumerate(seq) if 'k_init' in n]
start = inits[-1]
end = [i for i in range(start, len(seq)) if 'k_knn' in seq[i][1]][0]
agg = collections.defaultdict(lambda: [0, 0.0])
for _, n, v in seq[start:end + 1]:
    short = n.split('(')[0].replace('void ', '')[:70]
    agg[short][0] += 1
    agg[short][1] += v
tot = sum(v for _, v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v / 1e6:9.3f} ms {100 * v / tot:5.1f}% x{c:4d} {k}")
print('total', tot / 1e6, 'ms over', end - start + 1, 'launches')
