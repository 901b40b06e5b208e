#!/bin/bash
set -u
mkdir -p gpurun_out
for v in 1 2 0; do
  DION2_DIST_INPLACE=$v timeout 900 python scripts/loopback_phases.py --world 1 2 > gpurun_out/dip3_loop_$v.log 2>&1
done
DION2_DIST_INPLACE=2 timeout 900 python -m pytest tests/test_gpu_dist.py -q --timeout 300 -p no:cacheprovider > gpurun_out/dip3_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/dip3_tests.log
