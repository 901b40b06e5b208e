#!/bin/bash
# bench the chunked pipeline at several chunk counts (same box, back to back)
mkdir -p gpurun_out
for c in ${CHUNKS:-1 2 3 4}; do
  DION2_CHUNKS=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep > gpurun_out/bench_c$c.log 2>&1
done
