# KNN time vs Morton key bits (KDB_MORTON_BITS)
for b in ${BITS:-32 24 21 16}; do
  KDB_MORTON_BITS=$b timeout 600 python bench.py --config ${CFG:-C3} --steps 5 --warmup 3 --no-cpu-baseline --no-ref-counters --no-e2e 2>&1 | tail -1 > /tmp/line.json
  python -c "import json; d=json.load(open('/tmp/line.json')); print('bits', $b, 'knn ms', round(d['ms_knn'],2), 'equal', d['sample_check_vs_fp64_bruteforce'])"
done
