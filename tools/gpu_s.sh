mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batch_edges.py tests/test_gpu_pcg_semantics.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3 > gpurun_out/s.log
for i in 1 2; do
NPCG_STREAMS=1 timeout 200 python tools/quick_step.py 2>&1 | tail -1 >> gpurun_out/s.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d['roofline']['pcg_iteration']['frac_of_measured'])" >> gpurun_out/s.log 2>&1; done
