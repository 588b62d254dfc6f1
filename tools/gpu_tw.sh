mkdir -p gpurun_out
EPOCHS=40 LR=1e-3 MESHES=32 timeout 900 python tools/train_bench_weights.py > gpurun_out/train_w1.log 2>&1; cp gpurun_out/poisson_f64_trained.json gpurun_out/w_lr1e-3.json
EPOCHS=60 LR=3e-4 MESHES=32 timeout 900 python tools/train_bench_weights.py > gpurun_out/train_w2.log 2>&1; cp gpurun_out/poisson_f64_trained.json gpurun_out/w_lr3e-4.json
