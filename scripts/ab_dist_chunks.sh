#!/bin/bash
# Owner-chunk overlap of the distributed step in loopback: step time per chunk count
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CHUNKS:-1 2 3}; do
  DION2_DIST_CHUNKS=$c timeout 900 python scripts/loopback_phases.py --world ${WORLDS:-2 8} > gpurun_out/dchunks_$c.json 2> gpurun_out/dchunks_$c.err
done
