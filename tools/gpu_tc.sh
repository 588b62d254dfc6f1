set -x
mkdir -p gpurun_out
K=64 timeout 300 python tools/gnn_tc_check.py > gpurun_out/gnn_tc_check.log 2>&1; echo check=$?
K=256 timeout 300 python tools/gnn_tc_check.py > gpurun_out/gnn_tc_check256.log 2>&1; echo check256=$?
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/gputest_parity.log 2>&1; echo parity=$?
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_tc.log 2>&1; echo cfg3=$?
