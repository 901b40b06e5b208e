#!/bin/bash
# ncu --set full of the fused pre-stage (one launch, 1B set) after the same command exits 0.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep --layers ${PROF_LAYERS:-24}"
$CMD > gpurun_out/pf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pre_fused -s 1 -c 1 -o gpurun_out/pf $CMD > gpurun_out/pf_ncu.log 2>&1
echo "exit $?" >> gpurun_out/pf_ncu.log
