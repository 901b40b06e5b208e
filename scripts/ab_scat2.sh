#!/bin/bash
set -u
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for v in 0 1 2 3; do
  DION2_SCATTER_VAR=$v timeout 300 $B > gpurun_out/abs2_1b_$v.log 2>&1
  DION2_SCATTER_VAR=$v timeout 300 $B --config stress --alpha 0.0625 > gpurun_out/abs2_st_$v.log 2>&1
done
