#!/bin/bash
set -u
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for v in 2 3; do
  DION2_K1MT_PIPE=$v timeout 300 $B > gpurun_out/abk_1b_$v.log 2>&1
done
timeout 300 $B --config 8b > gpurun_out/abk_8b_3.log 2>&1
timeout 300 $B --config stress --alpha 0.0625 > gpurun_out/abk_stress_3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -k "transposed or storage or column" > gpurun_out/abk_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/abk_tests.log
