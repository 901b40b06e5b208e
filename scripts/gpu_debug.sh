#!/bin/bash
mkdir -p gpurun_out
DION2_DEBUG_SYNC=1 timeout 600 python scripts/debug_step.py > gpurun_out/debug.log 2>&1
echo "debug exit $?" >> gpurun_out/debug.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -k "nonfinite or alpha_sweep or small_p" > gpurun_out/gputest2.log 2>&1
echo "pytest exit $?" >> gpurun_out/gputest2.log
