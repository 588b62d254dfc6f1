set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batch_edges.py tests/test_gpu_pcg_semantics.py tests/test_gpu_parity.py -x -q > gpurun_out/kr_tests.log 2>&1; echo tests=$?
: > gpurun_out/kr_sweep.log
for kr in 1 2 4; do for cl in 2 4; do for st in 1 2 4; do
  echo "== KR=$kr CL=$cl STREAMS=$st" >> gpurun_out/kr_sweep.log
  NPCG_LINE_KR=$kr NPCG_LINE_CLUSTER=$cl NPCG_STREAMS=$st timeout 200 python tools/quick_step.py 2>&1 | tail -2 >> gpurun_out/kr_sweep.log
done; done; done
