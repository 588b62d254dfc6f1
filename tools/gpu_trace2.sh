mkdir -p gpurun_out
export NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_trace.so
for v in "NPCG_LINE_KR=1" "NPCG_LINE_KR=1 NPCG_LINE_CLUSTER=4" "NPCG_LINE_KR=2 NPCG_LINE_CLUSTER=4"; do
  echo "== $v"; env $v NPCG_STREAMS=1 timeout 200 python tools/trace_ws.py 2>&1 | tail -30
done > gpurun_out/trace2.log 2>&1
