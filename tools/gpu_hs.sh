mkdir -p gpurun_out
: > gpurun_out/hs.log
for v in 0 40 100 300 0 100; do
NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_s$v.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-context --no-e2e 2>&1 | tail -1 > gpurun_out/bench_x.json
python -c "
import sys,json
d=json.loads(open('gpurun_out/bench_x.json').read()); print('sleep $v', d['value'], d['ms_per_step'], d['gnn']['pcg_ms'], d['roofline']['pcg_iteration']['frac_of_measured'], {k:round(v/120*1000,1) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/hs.log 2>&1
done
