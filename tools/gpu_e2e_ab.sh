# e2e A/B over the host-buffer KNN chunk count
for c in ${CHUNKS:-8 16 32}; do
  KDB_KNN_CHUNKS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_e2e_$c.log 2>&1
  tail -1 gpurun_out/b_e2e_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $c', 'knn', round(d['ms_knn'],2), 'e2e knn', round(d['e2e']['ms_knn'],2), 'e2e build', round(d['e2e']['ms_build'],2))"
done
