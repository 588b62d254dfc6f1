#!/bin/bash
# repeat the config-1 step and report any system that fails to converge
for i in $(seq 1 ${REPS:-4}); do
  MAXIT=1500 timeout 300 python tools/quick_step.py 2>&1 | grep iters
done
