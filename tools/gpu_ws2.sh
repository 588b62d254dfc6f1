set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_pcg_semantics.py tests/test_gpu_batch_edges.py tests/test_gpu_fullsize.py -x -q > gpurun_out/gputest_quick.log 2>&1; echo quick=$?
NPCG_STREAMS=1 NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_trace.so timeout 120 python tools/trace_ws.py > gpurun_out/trace_ws.log 2>&1; echo trace=$?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ydiv.log 2>&1; echo bench=$?
