#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q --timeout 300 -p no:cacheprovider -k "column or transposed or storage or ragged or auto or one_layer or full or config1 or stress or random or alpha or lr_zero or dist or loopback" > gpurun_out/abs_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/abs_tests.log
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for cfg in 1b stress 8b; do
  A=""; [ $cfg = stress ] && A="--alpha 0.0625"
  timeout 300 $B --config $cfg $A > gpurun_out/abs_${cfg}_idx.log 2>&1
  DION2_SCATTER_MASK=1 timeout 300 $B --config $cfg $A > gpurun_out/abs_${cfg}_mask.log 2>&1
done
