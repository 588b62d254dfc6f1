set -x
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
NPCG_STREAMS=4 timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "^{" > gpurun_out/bench_s4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 300 --csv --log-file gpurun_out/launches_r1v6.csv python bench.py --profile-only > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trsv_line|spmv_ell|pupd_ell|diag_scale" -s 400 -c 5 -o gpurun_out/prof_r1v6 python bench.py --profile-only > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
