# one ncu --set full capture per "name:regex:skip" spec in $SPECS, exported as CSV (details, raw, sass, cuda source)
mkdir -p gpurun_out
ARGS=${BENCH_ARGS:-"--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"}
for spec in $SPECS; do
  name=${spec%%:*}; rest=${spec#*:}; rx=${rest%%:*}; skip=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" --launch-skip $skip -c 1 -o /tmp/full_$name -f python bench.py $ARGS > gpurun_out/ncu_full_$name.log 2>&1; echo "ncu full $name rc=$?"
  ncu -i /tmp/full_$name.ncu-rep --page details --csv > gpurun_out/full_${name}_details.csv 2>/dev/null
  ncu -i /tmp/full_$name.ncu-rep --page raw --csv > gpurun_out/full_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/full_$name.ncu-rep --page source --csv > gpurun_out/full_${name}_source.csv 2>/dev/null
  ncu -i /tmp/full_$name.ncu-rep --page source --print-source cuda --csv > gpurun_out/full_${name}_cuda.csv 2>/dev/null
done
ls -la gpurun_out
