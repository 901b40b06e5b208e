#!/bin/bash
# Direct peer exchange (DION2_FLAG_DIST_DIRECT) against the copy / NCCL exchange:
#   loopback per-rank estimate at P = 2, 8 and the one-rank NCCL step (symmetric windows).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/loopback_phases.py --world 2 8 > gpurun_out/direct_lb_copy.json 2> gpurun_out/direct_lb_copy.err
timeout 900 python scripts/loopback_phases.py --world 2 8 --direct > gpurun_out/direct_lb_direct.json 2> gpurun_out/direct_lb_direct.err
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep --no-details"
DION2_BENCH_DIST=1 timeout 600 $B > gpurun_out/direct_n1_nccl.log 2>&1
DION2_BENCH_DIST=1 DION2_BENCH_DIRECT=1 timeout 600 $B > gpurun_out/direct_n1_direct.log 2>&1
