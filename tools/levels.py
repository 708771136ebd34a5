"""Per-level kernel times of the last build in an ncu launch list (gpu__time_duration)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
seq = [(r[ki], float(r[vi].replace(',', ''))) for r in rows[hi + 1:] if len(r) > vi]
st = [i for i, (n, _) in enumerate(seq) if 'k_init' in n][-1]
out = []
for n, v in seq[st:]:
    s = n.split('(')[0].replace('void ', '').replace('kdb::', '').split('<')[0]
    if s == 'k_hist':
        out.append({})
    if s == 'k_subtree':
        print('k_subtree', round(v / 1e3), 'us')
        break
    if out:
        out[-1][s] = out[-1].get(s, 0) + v / 1e3
    elif s == 'k_sample':
        pend = pend + v / 1e3 if 'pend' in dir() else v / 1e3
for i, d in enumerate(out):
    print(i, ' '.join(f"{k}={v:.0f}" for k, v in d.items() if v > 5))
