mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pcg_semantics.py tests/test_gpu_batch_edges.py tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3 > gpurun_out/x.log
for v in 1 0 1 0; do
NPCG_XUPD_STREAM=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-context 2>&1 | tail -1 > gpurun_out/bench_x.json
python -c "
import sys,json
d=json.loads(open('gpurun_out/bench_x.json').read()); print('xupd $v', d['value'], d['ms_per_step'], d['e2e']['value'], d['gnn']['ms'], d['gnn']['pcg_ms'], d['roofline']['pcg_iteration']['frac_of_measured'], {k:round(v/120*1000,1) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/x.log 2>&1
done
