set -x
mkdir -p gpurun_out
SW="w0s20:NPCG_LEVELFLAG_WIDTH=0,NPCG_LEVELFLAG_SLEEP=20;w1s20:NPCG_LEVELFLAG_WIDTH=1;w2s20:NPCG_LEVELFLAG_WIDTH=2;w4s20:NPCG_LEVELFLAG_WIDTH=4;w2s100:NPCG_LEVELFLAG_WIDTH=2,NPCG_LEVELFLAG_SLEEP=100;w2s0:NPCG_LEVELFLAG_SLEEP=0;w1s100:NPCG_LEVELFLAG_WIDTH=1,NPCG_LEVELFLAG_SLEEP=100"
CFG=4 SWEEP="$SW" timeout 400 python tools/bench_3d.py > gpurun_out/sweep_cfg4.log 2>&1; echo c4=$?
CFG=5 BATCH=1 SWEEP="$SW" timeout 400 python tools/bench_3d.py > gpurun_out/sweep_cfg5_b1.log 2>&1; echo c5b1=$?
CFG=5 BATCH=8 SWEEP="$SW" timeout 500 python tools/bench_3d.py > gpurun_out/sweep_cfg5_b8.log 2>&1; echo c5b8=$?
