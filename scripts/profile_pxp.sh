#!/bin/bash
# ncu --set full of the Gram-space p x p launches (poly, C.A, C.B of iteration 0) at full size
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
$CMD > gpurun_out/pxp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_ns_gemm_tc_pair" -s 1 -c 3 -o gpurun_out/prof_pxp $CMD > gpurun_out/ncu_pxp.log 2>&1
echo "exit $?" >> gpurun_out/ncu_pxp.log
