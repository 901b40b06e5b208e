#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/chk4_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/chk4_tests.log
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e"
timeout 600 $B > gpurun_out/chk4_1b.log 2>&1
