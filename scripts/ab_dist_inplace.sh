#!/bin/bash
# in-place rank pieces for the owner NS (DION2_DIST_INPLACE): distributed parity + loopback phases
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_dpsync.py -q --timeout 300 -p no:cacheprovider > gpurun_out/dip_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/dip_tests.log
DION2_DIST_INPLACE=0 timeout 900 python -m pytest tests/test_gpu_dist.py -q --timeout 300 -p no:cacheprovider >> gpurun_out/dip_tests.log 2>&1
echo "pytest(off) exit $?" >> gpurun_out/dip_tests.log
timeout 900 python scripts/loopback_phases.py --world 1 2 4 8 > gpurun_out/dip_loop_on.log 2>&1
DION2_DIST_INPLACE=0 timeout 900 python scripts/loopback_phases.py --world 1 2 4 8 > gpurun_out/dip_loop_off.log 2>&1
DION2_BENCH_DIST=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep > gpurun_out/dip_bench.log 2>&1
