set -x
mkdir -p gpurun_out
for v in "" "NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_ell16.so" "NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_ell8.so" "NPCG_STREAMS=3" "NPCG_STREAMS=4"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > "gpurun_out/bench_v_$(echo $v | tr '/=' '__' | tail -c 40).log" 2>&1; echo "bench $v=$?"
done
