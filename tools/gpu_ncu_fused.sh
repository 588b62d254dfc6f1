set -x
mkdir -p gpurun_out
NPCG_STREAMS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ldlt_line|spmv_ell" -s 200 -c 2 -o gpurun_out/prof_fused python bench.py --profile-only > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
