# round-2 final evidence: all -m gpu tests, smoke, benches (C3 both arms, C1/C2/C4), C3 launch list + DRAM traffic,
# ncu --set full of the top kernels (one launch each)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
CFG=C3 bash tools/gpu_launches.sh > gpurun_out/launch_run.log 2>&1; echo "launch list rc=$?"
cp gpurun_out/traffic_C3.json profiles/r02_traffic_c3.json 2>/dev/null   # bench.py reads roofline.traffic from here
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2>&1; echo "bench C3 rc=$?"; tail -1 gpurun_out/bench_c3.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
for c in C1 C2 C4; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
SPECS="knn:k_knn_persist:1 sub:k_subtree:1 scat:k_scatter_tma:34 samp:^k_sample\$:13 hist:k_hist:35" BENCH_ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ref-counters" bash tools/gpu_ncu_one.sh > gpurun_out/ncu_one.log 2>&1; echo "ncu full rc=$?"
for n in knn sub scat samp hist; do python tools/ncu_summary.py gpurun_out/full_$n > gpurun_out/ncu_full_${n}_c3.txt 2>&1; done
