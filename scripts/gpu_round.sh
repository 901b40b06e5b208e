#!/bin/bash
# One gpurun call: GPU parity tests, then a short bench.  Output under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ "${RUN_DEBUG:-0}" = "1" ]; then
  DION2_DEBUG_SYNC=1 timeout 600 python scripts/debug_step.py > gpurun_out/debug.log 2>&1
  echo "debug exit $?" >> gpurun_out/debug.log
fi
if [ "${RUN_TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
  echo "pytest exit $?" >> gpurun_out/gputest.log
fi
if [ "${RUN_BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench.log
fi
