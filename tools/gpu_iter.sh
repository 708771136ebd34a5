# one GPU iteration: parity tests, bench (A/B over env settings in $AB), launch list summary
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for ab in ${AB:-DEFAULT=1}; do
  env $ab timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.log 2>&1
  tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ab','build',round(d.get('ms_build'),3),'knn',round(d.get('ms_knn'),3),round(d['value'],1), d['sample_check_vs_fp64_bruteforce'], 'slow', d.get('build_slow_nodes'))" || tail -5 gpurun_out/b.log
done
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cur.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cur.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/launches_cur.csv | head -14
fi
