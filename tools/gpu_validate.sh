# End-of-round validation on one B200 (under gpurun): smoke, every GPU test, the bench arms,
# the ncu launch list of the default step and one full capture of the PCG kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/gputest.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 python bench.py --weights seeded --no-cpu-baseline > gpurun_out/bench_seeded.log 2>&1; echo seeded=$?
timeout 900 python bench.py --config 3 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo cfg3=$?
timeout 300 python bench.py --profile-only > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --profile-only > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ldlt_line|spmv_ell_kernel<7, 0, 1>|pupd_ell|mp_tc_kernel" -s 10 -c 5 -o gpurun_out/r2_prof_final python bench.py --profile-only > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ncu -i gpurun_out/r2_prof_final.ncu-rep --page details > gpurun_out/r2_prof_final_details.txt 2>&1
ncu -i gpurun_out/r2_prof_final.ncu-rep --page raw --csv > gpurun_out/r2_prof_final_raw.csv 2>&1
CFG=4 timeout 700 python tools/bench_3d.py > gpurun_out/bench_cfg4.log 2>&1; echo c4=$?
CFG=5 timeout 1500 python tools/bench_3d.py > gpurun_out/bench_cfg5.log 2>&1; echo c5=$?
timeout 300 python tools/bench_train.py > gpurun_out/bench_train.log 2>&1; echo train=$?
