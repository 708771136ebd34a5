# all single-GPU configs: one short bench line each (device-resident + e2e), no CPU leg
mkdir -p gpurun_out
for c in C1 C3 C4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c build ms',round(d['ms_build'],3),'knn ms',round(d['ms_knn'],3),'Mpts/s',round(d['value'],1),'q/s',round(d['knn']['value']/1e6,1),'M ok',d['sample_check_vs_fp64_bruteforce'],'slow',d.get('build_slow_nodes'),'e2e',round(d['e2e']['ms_build'],2),round(d['e2e']['ms_knn'],2))" 2>/dev/null || tail -3 gpurun_out/bench_$c.log
done
