#!/bin/bash
# Round-end evidence on one GPU: default bench line, 8B and stress lines, launch list, DRAM
# traffic of the streaming kernels, --set full of one 6-layer step.  Output under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/ev_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1
timeout 600 python bench.py --config 8b --no-cpu --no-e2e --no-sweep --no-alpha1 > gpurun_out/ev_bench_8b.log 2>&1
timeout 600 python bench.py --config stress --alpha 0.0625 --no-e2e --no-sweep > gpurun_out/ev_bench_stress.log 2>&1
PROF_COUNT=24 bash scripts/profile.sh
