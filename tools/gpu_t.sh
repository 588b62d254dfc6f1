mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pcg_semantics.py tests/test_gpu_batch_edges.py tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_3d.py -x -q 2>&1 | tail -3 > gpurun_out/t.log
for w in trained seeded; do
timeout 600 python bench.py --weights $w --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$w.json
python -c "
import sys,json
d=json.loads(open('gpurun_out/bench_$w.json').read()); print('$w', d['value'], d['ms_per_step'], d['e2e']['value'], d['iterations'], d['gnn']['ms'], d['gnn']['pcg_ms'], d['roofline']['pcg_iteration']['frac_of_measured'], d['roofline']['kernel_ms'], d['context'])" >> gpurun_out/t.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-700 >> gpurun_out/t.log
