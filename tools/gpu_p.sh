mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batch_edges.py tests/test_gpu_pcg_semantics.py -x -q 2>&1 | tail -3 > gpurun_out/p.log
for v in 1 0 1; do
echo "== NPCG_LINE_PUPD=$v" >> gpurun_out/p.log
NPCG_LINE_PUPD=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d['roofline']['pcg_iteration']['frac_of_measured'], d['roofline']['kernel_ms'])" >> gpurun_out/p.log 2>&1; done
