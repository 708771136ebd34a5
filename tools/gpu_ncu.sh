# ncu evidence: launch list with time + DRAM bytes for every kernel, then --set full of the top kernels,
# exported to CSV on the box (the .ncu-rep files are too large to bring back)
mkdir -p gpurun_out
ARGS=${BENCH_ARGS:-"--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"}
if [ -z "$NO_LAUNCH" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
fi
for k in ${NCU_KERNELS:-k_knn_persist k_subtree k_sample k_scatter k_hist}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip ${NCU_SKIP:-0} -c 1 -o /tmp/full_$k -f python bench.py $ARGS > gpurun_out/ncu_full_$k.log 2>&1; echo "ncu full $k rc=$?"
  for pg in details raw source; do ncu -i /tmp/full_$k.ncu-rep --page $pg --csv > gpurun_out/full_${k}_$pg.csv 2>/dev/null; done
  ls -la gpurun_out/full_${k}_*.csv
done
