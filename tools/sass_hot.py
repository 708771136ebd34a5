"""Hottest SASS instructions / opcode mix of an ncu --page source --csv (SASS view) export:
    python tools/sass_hot.py file_source.csv [top]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = [r for r in rows if r and r[0] == 'Address'][0]
ai, si = h.index('Address'), h.index('Source')
ws, ie = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
ti = h.index('Thread Instructions Executed')
body = [r for r in rows[rows.index(h) + 1:] if len(r) > ie]
tot_s = sum(float(r[ws] or 0) for r in body) or 1
tot_i = sum(float(r[ie] or 0) for r in body) or 1
ops = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in body:
    op = r[si].split()[0] if r[si].split() else '?'
    if op.startswith('@'):
        op = r[si].split()[1]
    op = op.split('.')[0]
    ops[op][0] += float(r[ws] or 0); ops[op][1] += float(r[ie] or 0); ops[op][2] += float(r[ti] or 0)
print(f"total warp instr {tot_i:.3e}, thread instr {sum(v[2] for v in ops.values()):.3e}")
print("opcode mix (stall%, instr%):")
for k, v in sorted(ops.items(), key=lambda x: -x[1][1])[:20]:
    print(f"  {k:10s} {100*v[0]/tot_s:5.1f}% {100*v[1]/tot_i:5.1f}%  avg thr {v[2]/max(v[1],1):5.1f}")
print("hottest instructions by stall samples:")
for r in sorted(body, key=lambda r: -float(r[ws] or 0))[:top]:
    print(f"  {r[ai]} {100*float(r[ws] or 0)/tot_s:5.1f}% {100*float(r[ie] or 0)/tot_i:5.2f}%i  {r[si][:80]}")
