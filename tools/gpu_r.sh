mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pcg_semantics.py tests/test_gpu_batch_edges.py tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3 > gpurun_out/r.log
for i in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-context --no-e2e 2>&1 | tail -1 > gpurun_out/bench_x.json
python -c "
import sys,json
d=json.loads(open('gpurun_out/bench_x.json').read()); print(d['value'], d['ms_per_step'], d['gnn']['pcg_ms'], d['roofline']['pcg_iteration']['frac_of_measured'], {k:round(v/120*1000,1) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/r.log 2>&1
done
