#!/bin/bash
# A/B of the NS kernel variants at full size (1B set): per-phase times from the details sidecar
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep"
for v in ${VARIANTS:-default 1sm_apply}; do
  if [ "$v" = default ]; then timeout 600 $B > gpurun_out/abns_$v.log 2>&1
  else DION2_NS_PAIR=$v timeout 600 $B > gpurun_out/abns_$v.log 2>&1; fi
  cp gpurun_out/bench_details_1b_n1.json gpurun_out/abns_details_$v.json 2>/dev/null
done
