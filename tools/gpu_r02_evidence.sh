# round-2 evidence: benches (C3 default + C1/C2/C4 + reference arm), launch list with DRAM bytes (C3),
# ncu --set full of the top kernels on C3
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench C3 rc=$?"
for c in C1 C2 C4; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launches.py gpurun_out/launches_c3.csv --json gpurun_out/r02_traffic_c3.json > gpurun_out/launches_c3_summary.txt 2>&1
SPECS="knn:k_knn_persist:1 sub:k_subtree:1 hist:k_hist:35 samp:k_sample:13 scat:k_scatter:34" BENCH_ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline" bash tools/gpu_ncu_one.sh > gpurun_out/ncu_one.log 2>&1; echo "ncu full rc=$?"
