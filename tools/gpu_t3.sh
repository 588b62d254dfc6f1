mkdir -p gpurun_out
: > gpurun_out/t.log
for v in "1 seeded" "2 seeded" "1 seeded" "2 seeded"; do set -- $v
NPCG_STREAMS=$1 timeout 600 python bench.py --weights $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1 > gpurun_out/bench_x.json
python -c "
import sys,json
d=json.loads(open('gpurun_out/bench_x.json').read()); print('streams $1 $2', d['value'], d['ms_per_step'], d['gnn']['ms'], d['gnn']['pcg_ms'], d['roofline']['pcg_iteration']['frac_of_measured'], d['roofline']['kernel_ms'])" >> gpurun_out/t.log 2>&1
done
