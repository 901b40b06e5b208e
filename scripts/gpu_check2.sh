#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -k "gram or ns_forms or schedules or one_layer or alpha or stress or split_k or small_p or ragged or config1 or determinism or timing" > gpurun_out/chk2_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/chk2_tests.log
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
timeout 300 $B > gpurun_out/chk2_1b.log 2>&1
timeout 300 $B --config stress --alpha 0.0625 > gpurun_out/chk2_stress.log 2>&1

