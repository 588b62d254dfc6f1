set -x
mkdir -p gpurun_out
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo cfg2=$?
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo cfg3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mp_kernel" -s 4 -c 2 -o gpurun_out/prof_gnn python bench.py --config 3 --profile-only --batch 4 > gpurun_out/ncu_gnn.log 2>&1; echo ncu=$?
