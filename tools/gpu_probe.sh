set -x
mkdir -p gpurun_out
for st in 1 2; do for c in 2 4; do NPCG_STREAMS=$st NPCG_LINE_CLUSTER=$c timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_s${st}_c$c.log 2>&1; done; done
NPCG_STREAMS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 60 --csv --log-file gpurun_out/launches_fused.csv python bench.py --profile-only > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
