#!/bin/bash
# On a lease with >= 2 GPUs: the world-2 NCCL tests (owner-compute step with the NCCL and the
# direct exchange, DP-sync with both, FSDP2) and the bench at N = 2, 4, 8 (as many as visible).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NG=$(python -c "import torch; print(torch.cuda.device_count())")
echo "visible GPUs: $NG" > gpurun_out/mg_summary.txt
timeout 1200 python -m pytest tests/test_gpu_multirank.py -m gpu -q > gpurun_out/mg_tests.log 2>&1
echo "multirank tests rc=$?" >> gpurun_out/mg_summary.txt
for N in 2 4 8; do
  [ "$N" -gt "$NG" ] && break
  for direct in 1 0; do
    DION2_BENCH_DIRECT=$direct timeout 900 python bench.py --gpus $N --steps 10 --warmup 3 --no-cpu --no-sweep \
      > gpurun_out/mg_bench_n${N}_d${direct}.log 2>&1
    echo "bench N=$N direct=$direct rc=$? $(tail -1 gpurun_out/mg_bench_n${N}_d${direct}.log | cut -c1-200)" >> gpurun_out/mg_summary.txt
  done
done
