mkdir -p gpurun_out
: > gpurun_out/g3.log
for v in "" 66; do
  echo "== NPCG_LINE_CFG=$v" >> gpurun_out/g3.log
  NPCG_LINE_CFG=$v timeout 200 python tools/quick_step.py 2>&1 | tail -2 >> gpurun_out/g3.log
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batch_edges.py tests/test_gpu_pcg_semantics.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2 >> gpurun_out/g3.log
