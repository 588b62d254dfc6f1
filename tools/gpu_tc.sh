set -x
mkdir -p gpurun_out
K=64 timeout 300 python tools/gnn_tc_check.py > gpurun_out/gnn_tc_check.log 2>&1; echo check=$?
K=256 timeout 300 python tools/gnn_tc_check.py > gpurun_out/gnn_tc_check256.log 2>&1; echo check256=$?
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/gputest_parity.log 2>&1; echo parity=$?
