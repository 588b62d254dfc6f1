# fused-kernel check: correctness first, then cluster variants of the bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_pcg_semantics.py tests/test_gpu_batch_edges.py -x -q > gpurun_out/gputest_quick.log 2>&1; echo quick=$?
timeout 900 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputest.log 2>&1; echo tests=$?
for c in 2 4; do NPCG_LINE_CLUSTER=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1; echo bench_c$c=$?; done
