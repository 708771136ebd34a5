"""Per-CUDA-line stall samples / instructions: ncu SASS source page + nvdisasm line info.
    python tools/sass_lines.py SOURCE_CSV CUBIN FUNC_SUBSTR [top]
(the ncu page's absolute addresses are rebased to the function start and matched with
`nvdisasm -g -fun` offsets of the same cubin)"""
import collections, csv, re, subprocess, sys
src, cubin, fsub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(src)))
h = [r for r in rows if r and r[0] == 'Address'][0]
ai, si = h.index('Address'), h.index('Source')
ws, ie = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
te = h.index('Thread Instructions Executed')
body = [r for r in rows[rows.index(h) + 1:] if len(r) > ie and r[ai].startswith('0x')]
base = min(int(r[ai], 16) for r in body)
dis = subprocess.check_output(['nvdisasm', '-g', '-c', cubin], text=True, stderr=subprocess.DEVNULL)
# locate the function
funcs = re.split(r'\n\s*\.text\.', dis)
blk = [f for f in funcs if fsub in f.split('\n')[0]]
if not blk:
    sys.exit('function not found')
blk = max(blk, key=len)
line_of = {}
cur = None
for ln in blk.split('\n'):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in body:
    off = int(r[ai], 16) - base
    k = line_of.get(off, '?')
    agg[k][0] += float(r[ws] or 0)
    agg[k][1] += float(r[ie] or 0)
    agg[k][2] += float(r[te] or 0)
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
srcfiles = {}
print(f'warp instructions {ti:.0f}  avg active threads {sum(v[2] for v in agg.values()) / ti:.2f}')
for k, (s, i, t) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    txt = ''
    if ':' in k:
        fn, no = k.rsplit(':', 1)
        try:
            if fn not in srcfiles:
                import glob
                p = glob.glob(f'/root/repo/**/{fn}', recursive=True)
                srcfiles[fn] = open(p[0]).read().split('\n') if p else []
            txt = srcfiles[fn][int(no) - 1].strip()[:70]
        except Exception:
            pass
    print(f"{100 * s / ts:5.1f}% stall {100 * i / ti:5.1f}% instr {t / max(i, 1):5.1f} thr  {k:22s} {txt}")
