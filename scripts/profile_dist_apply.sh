#!/bin/bash
# ncu of the owner apply (1-SM k_ns_gemm_tc) in the distributed step at N = 1, in-place pieces on / off
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for v in 1 0; do
  DION2_BENCH_DIST=1 DION2_DIST_INPLACE=$v $CMD > gpurun_out/pda_plain_$v.log 2>&1 && \
  DION2_BENCH_DIST=1 DION2_DIST_INPLACE=$v ncu --set full --clock-control none -k regex:k_ns_gemm_tc -s 2 -c 1 -o gpurun_out/pda_$v $CMD > gpurun_out/pda_ncu_$v.log 2>&1
  echo "exit $?" >> gpurun_out/pda_ncu_$v.log
done
