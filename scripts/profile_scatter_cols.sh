#!/bin/bash
# ncu --set full of one column-scatter launch (1B set and 8B set, one step each)
mkdir -p gpurun_out
for cfg in 1b 8b; do
  CMD="python bench.py --config $cfg --layers 8 --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep --no-details"
  $CMD > gpurun_out/sc_plain_$cfg.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:k_scatter_cols" -c 1 -o gpurun_out/prof_sc_$cfg $CMD > gpurun_out/ncu_sc_$cfg.log 2>&1
  echo "exit $?" >> gpurun_out/ncu_sc_$cfg.log
done
