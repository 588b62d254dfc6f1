mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/kr_tests.log 2>&1; echo tests=$?
