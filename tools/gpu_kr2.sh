mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batch_edges.py -x -q > gpurun_out/kr_tests.log 2>&1; echo tests=$?
: > gpurun_out/kr_sweep.log
for v in "1 2 1" "1 2 2" "2 2 1" "2 2 2" "2 2 4" "2 4 1" "2 4 2" "2 4 4" "4 4 1" "4 4 2"; do set -- $v
  echo "== KR=$1 CL=$2 STREAMS=$3" >> gpurun_out/kr_sweep.log
  NPCG_LINE_KR=$1 NPCG_LINE_CLUSTER=$2 NPCG_STREAMS=$3 timeout 200 python tools/quick_step.py 2>&1 | tail -2 >> gpurun_out/kr_sweep.log
done
export NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_trace.so
for v in "NPCG_LINE_KR=1" "NPCG_LINE_KR=2 NPCG_LINE_CLUSTER=2" "NPCG_LINE_KR=2 NPCG_LINE_CLUSTER=4"; do
  echo "== $v"; env $v NPCG_STREAMS=1 timeout 200 python tools/trace_ws.py 2>&1 | grep -v "nan\|Warn\|ret" | tail -20
done > gpurun_out/trace2.log 2>&1
