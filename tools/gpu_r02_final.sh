# full GPU evidence pass: all -m gpu tests, smoke, benches (C3 default both arms, C2), C3 launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --config C2 > gpurun_out/bench_C2.log 2>&1; echo "bench C2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launches.py gpurun_out/launches_c3.csv --json gpurun_out/r02_traffic_c3.json > gpurun_out/launches_c3_summary.txt 2>&1
SPECS="knn:k_knn_persist:1" BENCH_ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline" bash tools/gpu_ncu_one.sh > gpurun_out/ncu_one.log 2>&1; echo "ncu full rc=$?"
