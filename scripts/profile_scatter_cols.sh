#!/bin/bash
# ncu --set full of one column-scatter launch (8B set, one step)
mkdir -p gpurun_out
CMD="python bench.py --config 8b --layers 8 --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
$CMD > gpurun_out/sc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_scatter_cols_t" -c 1 -o gpurun_out/prof_sc $CMD > gpurun_out/ncu_sc.log 2>&1
echo "exit $?" >> gpurun_out/ncu_sc.log
