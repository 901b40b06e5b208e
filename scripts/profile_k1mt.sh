#!/bin/bash
# ncu --set full of the transposed-momentum K1 kernel (one launch, full 1B set)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
$CMD > gpurun_out/k1mt_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_momentum_score" -c 2 -o gpurun_out/prof_k1 $CMD > gpurun_out/ncu_k1.log 2>&1
echo "exit $?" >> gpurun_out/ncu_k1.log
