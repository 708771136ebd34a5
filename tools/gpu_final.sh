# end-of-round evidence: everything tools/gpu_evidence.sh does, plus the other single-GPU configs
bash tools/gpu_evidence.sh
for c in C1 C3 C4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
done
KDB_FORCE_GLOBAL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_global1.log 2>&1; echo "global1 rc=$?"
