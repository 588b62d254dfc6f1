set -x
mkdir -p gpurun_out
CFG=5 BATCH=1 STEPS=1 NPCG_LEVELSYNC=0 timeout 900 python tools/bench_3d.py > gpurun_out/bench_cfg5_b1_chunked.log 2>&1; echo a=$?
CFG=5 BATCH=1 STEPS=1 NPCG_LEVELSYNC_OCC=1 timeout 900 python tools/bench_3d.py > gpurun_out/bench_cfg5_b1_occ1.log 2>&1; echo b=$?
CFG=5 BATCH=4 STEPS=1 NPCG_LEVELSYNC=0 timeout 900 python tools/bench_3d.py > gpurun_out/bench_cfg5_b4_chunked.log 2>&1; echo c=$?
