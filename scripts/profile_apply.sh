#!/bin/bash
# Apply-phase evidence at full size (1B set): per-phase times with the 1-SM apply and with the
# pair kernel for the apply (DION2_NS_PAIR=all), then ncu --set full of the two apply launches
# and one gram launch of a step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep --no-graph --no-details"
$CMD > gpurun_out/pa_default.log 2>&1
DION2_NS_PAIR=all $CMD > gpurun_out/pa_pairall.log 2>&1
CMD1="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep --no-graph --no-details"
$CMD1 > gpurun_out/pa_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_ns_gemm" -s 0 -c 12 -o gpurun_out/prof_ns $CMD1 > gpurun_out/ncu_ns.log 2>&1
echo "exit $?" >> gpurun_out/ncu_ns.log
