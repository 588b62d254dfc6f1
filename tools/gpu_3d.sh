set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_3d.py -x -q > gpurun_out/gputest_3d.log 2>&1; echo t3d=$?
CFG=4 timeout 900 python tools/bench_3d.py > gpurun_out/bench_cfg4.log 2>&1; echo cfg4=$?
CFG=4 NPCG_LEVELSYNC_OCC=1 timeout 900 python tools/bench_3d.py > gpurun_out/bench_cfg4_occ1.log 2>&1; echo cfg4o1=$?
CFG=4 NPCG_LEVELSYNC_OCC=4 timeout 900 python tools/bench_3d.py > gpurun_out/bench_cfg4_occ4.log 2>&1; echo cfg4o4=$?
