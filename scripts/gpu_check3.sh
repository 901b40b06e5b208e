#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q --timeout 300 -p no:cacheprovider -k "select or stress or column or transposed or tie or nonfinite or random or one_layer or full or storage or ragged" > gpurun_out/chk3_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/chk3_tests.log
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
timeout 300 $B --config stress --alpha 0.0625 > gpurun_out/chk3_stress.log 2>&1
timeout 300 $B --config 8b > gpurun_out/chk3_8b.log 2>&1
