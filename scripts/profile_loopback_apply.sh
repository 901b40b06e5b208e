#!/bin/bash
# ncu of the owner apply (1-SM k_ns_gemm_tc<256>) in the loopback distributed step at P = 1,
# in-place pieces (1) vs copies (0)
set -u
mkdir -p gpurun_out
CMD="python scripts/loopback_phases.py --world 1 --steps 1"
for v in 1 0; do
  DION2_DIST_INPLACE=$v $CMD > gpurun_out/pla_plain_$v.log 2>&1 && \
  DION2_DIST_INPLACE=$v ncu --set full --clock-control none --kernel-name-base demangled -k "regex:gemm_tc<" -c 1 -s 1 -o gpurun_out/plb_$v $CMD > gpurun_out/pla_ncu_$v.log 2>&1
  echo "exit $?" >> gpurun_out/pla_ncu_$v.log
done
