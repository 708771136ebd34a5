# round-2 first pass: host facts, BASELINE-scale parity, bench C3 (both arms), C3 launch list with DRAM bytes
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi) > gpurun_out/host.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_scale.py -m gpu -x -q -s > gpurun_out/scale_tests.log 2>&1; echo "scale rc=$?"; tail -8 gpurun_out/scale_tests.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_c3.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_c3.csv --json gpurun_out/r02_traffic_c3.json > gpurun_out/launches_c3_summary.txt 2>&1; tail -3 gpurun_out/launches_c3_summary.txt
