#!/bin/bash
set -u
mkdir -p gpurun_out
for v in 1 0; do
  DION2_DIST_INPLACE=$v timeout 900 python scripts/loopback_phases.py --world 1 2 8 > gpurun_out/dip2_loop_$v.log 2>&1
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep > gpurun_out/dip2_bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_dpsync.py -q --timeout 300 -p no:cacheprovider > gpurun_out/dip2_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/dip2_tests.log
