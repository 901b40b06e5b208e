#!/bin/bash
# ncu --set full of the NS launches of one full-size step (1B set); PROF_K selects the kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep --no-graph --no-details"
$CMD > gpurun_out/pn_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${PROF_K:-k_ns_apply_pair}" -s ${PROF_S:-0} -c ${PROF_C:-2} -o gpurun_out/prof_${PROF_TAG:-ns} $CMD > gpurun_out/ncu_${PROF_TAG:-ns}.log 2>&1
echo "exit $?" >> gpurun_out/ncu_${PROF_TAG:-ns}.log
