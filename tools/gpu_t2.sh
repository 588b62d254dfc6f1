mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_northstar.py -x -q 2>&1 | tail -3 > gpurun_out/t.log
for i in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_trained.json
python -c "
import sys,json
d=json.loads(open('gpurun_out/bench_trained.json').read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['iterations'], d['gnn'], d['roofline']['pcg_iteration'], d['roofline']['frac'], d['roofline']['launch_ms'])" >> gpurun_out/t.log 2>&1
done
