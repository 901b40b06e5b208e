#!/bin/bash
set -u
mkdir -p gpurun_out
DION2_NS_PAIRCFG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -k "gram or ns_forms or schedules or one_layer or alpha or stress or split_k or small_p or ragged or config1" > gpurun_out/abp_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/abp_tests.log
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for v in 0 1 0 1; do
  DION2_NS_PAIRCFG=$v timeout 300 $B > gpurun_out/abp_1b_$v.log 2>&1
  python scripts/show_bench.py gpurun_out/abp_1b_$v.log | grep -E "ms/step|ns_" >> gpurun_out/abp_summary.txt
done
