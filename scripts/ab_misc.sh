#!/bin/bash
# A/B runs on one box: 2-SM apply (DION2_NS_PAIR=all); stress (configs[4]) and 8B bench lines.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
timeout 300 $B > gpurun_out/ab_base.log 2>&1
DION2_NS_PAIR=all timeout 300 $B > gpurun_out/ab_pairall.log 2>&1
DION2_NS_PAIR=all timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gram or ns_forms or schedules or one_layer or alpha_sweep" -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1
timeout 300 python bench.py --config stress --alpha 0.0625 --steps 10 --warmup 3 --no-alpha1 --no-e2e --no-sweep > gpurun_out/ab_stress.log 2>&1
DION2_NS_PAIR=all timeout 300 python bench.py --config stress --alpha 0.0625 --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep > gpurun_out/ab_stress_pairall.log 2>&1
