mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_scale.py > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
for c in ${CFGS:-C1 C2 C3}; do timeout 600 python tools/knn_ab.py $c 3 2>&1 | tail -4; done
