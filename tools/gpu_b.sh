mkdir -p gpurun_out
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d['roofline']['pcg_iteration']['frac_of_measured'])"; done > gpurun_out/b.log 2>&1
