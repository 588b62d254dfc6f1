set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_3d.py -x -q > gpurun_out/flags_t3d.log 2>&1; echo t3d=$?
CFG=4 timeout 300 python tools/bench_3d.py > gpurun_out/flags_cfg4.log 2>&1; echo c4=$?
CFG=4 NPCG_LEVELFLAGS=0 timeout 300 python tools/bench_3d.py > gpurun_out/flags_cfg4_bar.log 2>&1; echo c4b=$?
CFG=5 timeout 300 python tools/bench_3d.py > gpurun_out/flags_cfg5.log 2>&1; echo c5=$?
CFG=5 BATCH=1 timeout 300 python tools/bench_3d.py > gpurun_out/flags_cfg5_b1.log 2>&1; echo c5b1=$?
CFG=5 BATCH=16 timeout 300 python tools/bench_3d.py > gpurun_out/flags_cfg5_b16.log 2>&1; echo c5b16=$?
