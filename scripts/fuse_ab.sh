#!/bin/bash
# A/B of the fused pre-stage (k_pre_fused.cu) on the 1B set: parity tests, then the bench
# with the fusion off / on at several gather lags.  Output under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider \
  -k "${TESTK:-pre_fused or phase_timing or one_layer or nonfinite or determinism or random}" > gpurun_out/fuse_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/fuse_tests.log
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
DION2_PRE_FUSE=0 timeout 300 $B > gpurun_out/fuse_off.log 2>&1
for lag in ${LAGS:-32 96 192}; do
  DION2_FUSE_LAG_MB=$lag timeout 300 $B > gpurun_out/fuse_lag$lag.log 2>&1
done
DION2_FUSE_NOHINT=1 timeout 300 $B > gpurun_out/fuse_nohint.log 2>&1
