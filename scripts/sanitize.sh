#!/bin/bash
# compute-sanitizer (memcheck only: one tool per gpurun call) over scripts/sanitize_step.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/sanitize_step.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool ${SAN_TOOL:-memcheck} --error-exitcode 9 python scripts/sanitize_step.py \
  > gpurun_out/sanitize_${SAN_TOOL:-memcheck}.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_${SAN_TOOL:-memcheck}.log
