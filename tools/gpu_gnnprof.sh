mkdir -p gpurun_out
NPCG_STREAMS=1 timeout 300 python bench.py --profile-only > gpurun_out/plain.log 2>&1 && \
NPCG_STREAMS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r2_launches_gnn.csv python bench.py --profile-only > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
