mkdir -p gpurun_out
for m in 0 2; do KDB_KNN_SCAN=$m timeout 900 python tools/knn_time.py ${CFGS:-C2,C3} 5 2>&1 | grep -v Warning | tail -3; done | tee gpurun_out/scan_ab.log
KDB_KNN_SCAN=2 timeout 1200 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_scale.py > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
