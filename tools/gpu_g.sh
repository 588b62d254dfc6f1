mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_northstar.py tests/test_gpu_3d.py -x -q 2>&1 | tail -3 > gpurun_out/g.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-context --no-e2e 2>&1 | tail -1 > gpurun_out/bench_x.json
python -c "
import sys,json
d=json.loads(open('gpurun_out/bench_x.json').read()); print(d['value'], d['ms_per_step'], d['gnn'])" >> gpurun_out/g.log 2>&1
done
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['ms_per_step'], d['gnn'])" >> gpurun_out/g.log 2>&1
