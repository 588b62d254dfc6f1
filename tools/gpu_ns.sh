set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_parity.py -x -q > gpurun_out/gputest_ns.log 2>&1; echo ns=$?
