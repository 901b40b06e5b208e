#!/bin/bash
# GPU test suite, then the 1B headline and the stress config (configs[4]) bench lines.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep > gpurun_out/chk_1b.log 2>&1
timeout 300 python bench.py --config stress --alpha 0.0625 --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep > gpurun_out/chk_stress.log 2>&1
DION2_GRAM_SPLITK=1 timeout 300 python bench.py --config stress --alpha 0.0625 --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep > gpurun_out/chk_stress_nosplit.log 2>&1
