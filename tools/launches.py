"""Summarise an ncu launch list (gpu__time_duration, optionally dram__bytes_{read,write}) for the
last build+query step of a bench run:  python tools/launches.py launches.csv [--json out.json]

Prints per-kernel time / share / DRAM bytes; --json also writes the per-build and per-query DRAM
traffic (sum over the build kernels / the query kernels of that step) that bench.py reports as
roofline.traffic."""
import collections, csv, json, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    try:
        lid = int(r[idi])
        val = float(r[vi].replace(',', ''))
    except (ValueError, IndexError):
        continue
    ent = launch.setdefault(lid, {'name': r[ki]})
    ent[r[mi]] = val
seq = list(launch.values())
# the last step = the launches after the previous step's KNN kernel up to the last KNN kernel
# (a query batch may launch several KNN kernels in a row: k_knn_home + k_knn_persist)
kdbi = [i for i, e in enumerate(seq) if 'kdb::' in e['name']]
isknn = lambda e: 'kdb::k_knn' in e['name'] and 'k_knn_walk' not in e['name']  # (the walk: counters, untimed)
knn = [i for n, i in enumerate(kdbi) if isknn(seq[i]) and (n + 1 == len(kdbi) or not isknn(seq[kdbi[n + 1]]))]
end = knn[-1]
start = knn[-2] + 1 if len(knn) > 1 else 0
seq = seq[:start] + [e for e in seq[start:end + 1] if 'kdb::' in e['name'] or 'CUB' in e['name']]
end = len(seq) - 1
T = 'gpu__time_duration.sum'
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
build_b = query_b = 0.0
build_t = query_t = 0.0
first_query = [i for i in range(start, end + 1) if any(q in seq[i]['name'] for q in ('k_leaf_of', 'k_qbox', 'k_morton'))]
qstart = first_query[0] if first_query else end
for i, e in enumerate(seq[start:end + 1], start):
    short = e['name'].split('(')[0].replace('void ', '')[:70]
    b = e.get('dram__bytes_read.sum', 0.0) + e.get('dram__bytes_write.sum', 0.0)
    agg[short][0] += 1
    agg[short][1] += e.get(T, 0.0)
    agg[short][2] += b
    if i < qstart:
        build_b += b; build_t += e.get(T, 0.0)
    else:
        query_b += b; query_t += e.get(T, 0.0)
tot = sum(v[1] for v in agg.values())
for k, (c, v, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    extra = f" {b / 1e9:8.3f} GB {b / max(v, 1):7.1f} GB/s" if b else ""
    print(f"{v / 1e6:9.3f} ms {100 * v / tot:5.1f}% x{c:4d}{extra} {k}")
print(f'total {tot / 1e6:.3f} ms over {end - start + 1} launches; build {build_t / 1e6:.3f} ms '
      f'{build_b / 1e9:.3f} GB, query {query_t / 1e6:.3f} ms {query_b / 1e9:.3f} GB')
if len(sys.argv) > 3 and sys.argv[2] == '--json':
    with open(sys.argv[3], 'w') as f:
        json.dump({'build_dram_bytes': build_b, 'query_dram_bytes': query_b, 'build_ncu_ms': build_t / 1e6,
                   'query_ncu_ms': query_t / 1e6,
                   'source': 'ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum '
                             '--clock-control none, last build+query step of bench.py (cold-cache, serialised)'},
                  f, indent=1)
