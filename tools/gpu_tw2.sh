mkdir -p gpurun_out
KS=32,48,64,96 EPOCHS=80 LR=3e-4 MESHES=32 OUT=gpurun_out/w_big.json timeout 1200 python tools/train_bench_weights.py > gpurun_out/train_big.log 2>&1
KS=24,32,40,48 EPOCHS=120 LR=1e-4 MESHES=64 OUT=gpurun_out/w_more.json timeout 1200 python tools/train_bench_weights.py > gpurun_out/train_more.log 2>&1
