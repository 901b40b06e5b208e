#!/bin/bash
# Bench the NS variants of one build back to back (one GPU).  Output: gpurun_out/v_*.log
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for v in "${@}"; do
  name=$(echo "$v" | tr ' =' '_-')
  env $v timeout 300 $B > gpurun_out/v_${name}.log 2>&1
done
