"""per-level times of the build kernels in the last step of an ncu launch list"""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); idi=h.index('ID'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
L=collections.OrderedDict()
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    e=L.setdefault(int(r[idi]),{'n':r[ki].split('(')[0].replace('void ','').replace('kdb::',''),'g':r[gi]})
    e[r[mi]]=float(r[vi].replace(',',''))
seq=list(L.values())
knn=[i for i,e in enumerate(seq) if 'k_knn' in e['n']]
s=[e for e in seq[knn[-2]+1:knn[-1]+1]]
lvl=-1; rows=collections.defaultdict(dict)
for e in s:
    n=e['n'].split('<')[0]
    if n in('k_sample','k_sample_cta'):
        if not (n=='k_sample' and 'k_sample' in rows[lvl]): lvl+=1
    t=e.get('gpu__time_duration.sum',0)/1e3
    rows[lvl][n]=rows[lvl].get(n,0)+t
cols=['k_sample','k_sample_cta','k_hist','k_select','k_slow','k_count','k_scatter','k_children']
print('lvl '+' '.join(f'{c[2:9]:>8s}' for c in cols))
for l in sorted(rows):
    if l<0: continue
    print(f'{l:3d} '+' '.join(f'{rows[l].get(c,0):8.1f}' for c in cols))
