set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_pcg_semantics.py tests/test_gpu_batch_edges.py -x -q > gpurun_out/gputest_quick.log 2>&1; echo quick=$?
for v in "" "NPCG_LINE_CFG=66" "NPCG_LINE_CFG=66 NPCG_STREAMS=1" "NPCG_LINE_CFG=66 NPCG_STREAMS=4"; do
  env $v timeout 150 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > "gpurun_out/bench_ws4_$v.log" 2>&1; echo "bench $v=$?"
done
