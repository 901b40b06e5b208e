#!/bin/bash
# TMA-staged rows gather (k_gather_tma.cu) vs the register-streaming kernel: parity, then A/B
set -u
mkdir -p gpurun_out
rm -f gpurun_out/abg_summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q --timeout 300 -p no:cacheprovider -x > gpurun_out/abg_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/abg_tests.log
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for v in 0 4 6 0 4; do
  DION2_GATHER_TMA=$v timeout 300 $B > gpurun_out/abg_1b_$v.log 2>&1
  python scripts/show_bench.py gpurun_out/abg_1b_$v.log | grep -E "ms/step|gather_rows" >> gpurun_out/abg_summary.txt
done
