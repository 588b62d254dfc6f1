mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batch_edges.py tests/test_gpu_pcg_semantics.py -x -q 2>&1 | tail -5 > gpurun_out/lag.log
for v in "" 66; do
  echo "== NPCG_LINE_CFG=$v" >> gpurun_out/lag.log
  NPCG_LINE_CFG=$v timeout 200 python tools/quick_step.py 2>&1 | tail -2 >> gpurun_out/lag.log
done
