set -x
mkdir -p gpurun_out
timeout 600 python tools/cfg3_iters.py > gpurun_out/cfg3_iters.log 2>&1; echo iters=$?
timeout 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_kernels.py -x -q > gpurun_out/gputest_fs.log 2>&1; echo fs=$?
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.log 2>&1; echo cfg3=$?
