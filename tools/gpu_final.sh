set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/gputest.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.log 2>&1; echo cfg3=$?
timeout 300 python tools/bench_train.py > gpurun_out/bench_train.log 2>&1; echo train=$?
CFG=4 timeout 600 python tools/bench_3d.py > gpurun_out/bench_cfg4.log 2>&1; echo c4=$?
