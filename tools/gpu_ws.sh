set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_pcg_semantics.py tests/test_gpu_batch_edges.py -x -q > gpurun_out/gputest_quick.log 2>&1; echo quick=$?
for v in "" "NPCG_LINE_CLUSTER=4" "NPCG_LINE_CFG=35" "NPCG_STREAMS=1" "NPCG_STREAMS=4"; do
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > "gpurun_out/bench_ws_$v.log" 2>&1; echo "bench $v=$?"
done
NPCG_STREAMS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 60 --csv --log-file gpurun_out/launches_ws.csv python bench.py --profile-only > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
