set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_kernels.py -q > gpurun_out/flags_t3d.log 2>&1; echo t3d=$?
CFG=4 SWEEP="vw4:NPCG_SPMV_VW4=1" timeout 400 python tools/bench_3d.py > gpurun_out/sweep_cfg4.log 2>&1; echo c4=$?
CFG=4 NPCG_SPMV_VW4=0 SWEEP="vw2:NPCG_SPMV_VW4=0" timeout 400 python tools/bench_3d.py >> gpurun_out/sweep_cfg4.log 2>&1; echo c4=$?
CFG=4 timeout 400 python tools/bench_3d.py > gpurun_out/flags_cfg4.log 2>&1; echo c4=$?
