# iteration: GPU parity suite, then bench configs given in $CFGS (default C3), then a KDB_TRACE'd C3 build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
for c in ${CFGS:-C3}; do
timeout 900 python bench.py --config $c ${BENCH_ARGS} > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-1500
done
