#!/bin/bash
# ncu --set full of one gram / poly / apply launch, default kernels and all-pair kernels
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep --layers 6"
$CMD > gpurun_out/pa_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_ns_gemm" -s 15 -c 3 -o gpurun_out/prof_ns $CMD > gpurun_out/ncu_ns.log 2>&1
echo "exit $?" >> gpurun_out/ncu_ns.log
DION2_NS_PAIR=all $CMD > gpurun_out/pa_plain2.log 2>&1 && \
DION2_NS_PAIR=all ncu --set full --clock-control none --import-source on -k "regex:k_ns_gemm" -s 15 -c 3 -o gpurun_out/prof_ns_pair $CMD > gpurun_out/ncu_ns_pair.log 2>&1
echo "exit $?" >> gpurun_out/ncu_ns_pair.log
