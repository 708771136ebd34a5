# ncu launch list (time + DRAM bytes) of one build+query step of bench.py -> gpurun_out/launches_$CFG.csv + summary
CFG=${CFG:-C3}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ref-counters > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launches.py gpurun_out/launches_$CFG.csv --json gpurun_out/traffic_$CFG.json > gpurun_out/launches_${CFG}_summary.txt 2>&1
cat gpurun_out/launches_${CFG}_summary.txt | cut -c1-150
