#!/bin/bash
# A/B of kernel variants at full size (1B set): per-phase times from the details sidecar.
# VARIANTS="name:VAR=val,VAR2=val name2 ..." ("default" = no overrides)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-e2e --no-sweep ${AB_ARGS}"
for spec in ${VARIANTS:-default}; do
  name=${spec%%:*}
  envs=""
  [ "$spec" != "$name" ] && envs=$(echo "${spec#*:}" | tr ',' ' ')
  env $envs timeout 600 $B > gpurun_out/abns_$name.log 2>&1
  cp gpurun_out/bench_details_${AB_CFG:-1b}_n1.json gpurun_out/abns_details_$name.json 2>/dev/null
done
