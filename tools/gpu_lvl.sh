set -x
mkdir -p gpurun_out
CFG=4 PROFILE_ONLY=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"level_flag" -s 2 -c 2 -o gpurun_out/r2_prof_cfg4_flag python tools/bench_3d.py > gpurun_out/ncu_cfg4.log 2>&1; echo ncu=$?
