set -x
mkdir -p gpurun_out
# launch list of the default bench (cold, serialised) and full captures of the top kernels
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 200 --csv --log-file gpurun_out/r2_launches.csv python bench.py --profile-only > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ldlt_line|spmv_ell|pupd_ell" -s 300 -c 3 -o gpurun_out/r2_prof_pcg python bench.py --profile-only > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mp_tc_kernel" -s 2 -c 2 -o gpurun_out/r2_prof_gnn python bench.py --config 3 --profile-only --batch 4 > gpurun_out/ncu_gnn.log 2>&1; echo ncu3=$?
# race / sync checks of the spin-waiting solve kernels (small problems)
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_kernels.py -q -k "apply_inverse_bitwise or line_solve or wide_grid" > gpurun_out/r2_racecheck.log 2>&1; echo race=$?
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_kernels.py -q -k "apply_inverse_bitwise or wide_grid" > gpurun_out/r2_synccheck.log 2>&1; echo sync=$?
