# e2e KNN time vs the number of chunks of the host-buffer pipeline (KDB_KNN_CHUNKS)
for c in ${CHUNKS:-4 8 16 32}; do
  KDB_KNN_CHUNKS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ref-counters 2>&1 | tail -1 > /tmp/line.json
  python -c "import json; d=json.load(open('/tmp/line.json')); print('chunks', $c, 'e2e build ms', round(d['e2e']['ms_build'],1), 'e2e knn ms', round(d['e2e']['ms_knn'],1))"
done
