"""Summarise ncu --page details / --page source CSV exports (key metrics, stall mix, top SASS ops)."""
import collections, csv, sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L2 Hit Rate', 'L1/TEX Hit Rate', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Compute (SM) Throughput', 'Executed Ipc Active',
        'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp', 'Dynamic Shared Memory Per Block',
        'Block Limit Registers', 'Block Limit Shared Mem']


def details(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    mi, vi, ui = h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    seen = {}
    for r in rows[1:]:
        if len(r) > vi and r[mi] in WANT and r[mi] not in seen:
            seen[r[mi]] = f"{r[vi]} {r[ui]}"
    return seen


def source(path, top=12):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ws = hdr.index('Warp Stall Sampling (All Samples)')
    stalls = [i for i, x in enumerate(hdr) if x.startswith('stall_') and 'Not Issued' not in x]
    agg, ops, lines = collections.Counter(), collections.Counter(), []
    tot = 0.0
    for r in rows[2:]:
        try:
            v = float(r[ws])
        except (ValueError, IndexError):
            continue
        tot += v
        toks = r[1].strip().split()
        op = toks[1] if toks and toks[0].startswith('@') and len(toks) > 1 else (toks[0] if toks else '?')
        ops[op.split('.')[0]] += v
        lines.append((v, r[0], r[1].strip()[:90]))
        for i in stalls:
            try:
                agg[hdr[i]] += float(r[i])
            except ValueError:
                pass
    return tot, agg, ops, sorted(lines, reverse=True)[:top]


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("=====", p)
        for k, v in details(f"ncu_{p}_details.csv").items():
            print(f"  {k:40s} {v}")
        tot, agg, ops, lines = source(f"ncu_{p}_source.csv")
        print("  stalls:", ", ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in agg.most_common(7)))
        print("  ops   :", ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in ops.most_common(10)))
