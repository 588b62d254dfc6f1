set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench_final.log 2>&1; echo bench=$?
NPCG_STREAMS=1 timeout 300 python bench.py --profile-only > gpurun_out/plain.log 2>&1 && \
NPCG_STREAMS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 150 --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --profile-only > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
NPCG_STREAMS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ldlt_line|spmv_ell|pupd_ell" -s 300 -c 3 -o gpurun_out/r2_prof_pcg_final python bench.py --profile-only > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ncu -i gpurun_out/r2_prof_pcg_final.ncu-rep --page details > gpurun_out/r2_prof_pcg_final_details.txt 2>&1
ncu -i gpurun_out/r2_prof_pcg_final.ncu-rep --page raw --csv > gpurun_out/r2_prof_pcg_final_raw.csv 2>&1
