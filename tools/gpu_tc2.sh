set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_tc.log 2>&1; echo cfg3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mp_edge_tc|mp_kernel" -s 3 -c 3 -o gpurun_out/prof_gnn_tc python bench.py --config 3 --profile-only --batch 4 > gpurun_out/ncu_gnn_tc.log 2>&1; echo ncu=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/gputest.log 2>&1; echo tests=$?
