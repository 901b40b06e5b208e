#!/bin/bash
# Round-end evidence on one GPU: default bench line (+ details sidecar), 8B, stress and
# 16-layer lines, then scripts/profile.sh (launch list, DRAM traffic, --set full of one step).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/ev_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1
cp gpurun_out/bench_details_1b_n1.json gpurun_out/ev_details_1b.json 2>/dev/null
timeout 600 python bench.py --config 8b --no-cpu --no-e2e --no-sweep --no-alpha1 > gpurun_out/ev_bench_8b.log 2>&1
timeout 600 python bench.py --config stress --alpha 0.0625 --no-e2e --no-sweep > gpurun_out/ev_bench_stress.log 2>&1
timeout 600 python bench.py --config 1b16 --no-cpu --no-e2e --no-sweep > gpurun_out/ev_bench_1b16.log 2>&1
PROF_COUNT=${PROF_COUNT:-40} PROF_LAYERS=${PROF_LAYERS:-24} bash scripts/profile.sh
