mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batch_edges.py tests/test_gpu_fullsize.py -x -q > gpurun_out/kr_tests.log 2>&1; echo tests=$?
: > gpurun_out/kr_sweep.log
for v in "1 2 2" "2 4 1"; do set -- $v
  echo "== KR=$1 CL=$2 STREAMS=$3" >> gpurun_out/kr_sweep.log
  NPCG_LINE_KR=$1 NPCG_LINE_CLUSTER=$2 NPCG_STREAMS=$3 timeout 200 python tools/quick_step.py 2>&1 | tail -2 >> gpurun_out/kr_sweep.log
done
for cfg in "" 36 35; do
  echo "== cfg3 NPCG_LINE_CFG=$cfg" >> gpurun_out/kr_sweep.log
  NPCG_LINE_CFG=$cfg timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('gnn'), d['roofline'].get('kernel_ms'))" >> gpurun_out/kr_sweep.log 2>&1
done
