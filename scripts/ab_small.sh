#!/bin/bash
# small A/B: TMA gather stages (6 / 8), host-upload chunks (2 / 4 / 8)
set -u
mkdir -p gpurun_out
rm -f gpurun_out/abs_small.txt
B="python bench.py --steps 10 --warmup 3 --no-alpha1 --no-cpu --no-sweep"
for v in 6 8; do
  DION2_GATHER_TMA=$v timeout 300 $B --no-e2e > gpurun_out/abs_g$v.log 2>&1
  python scripts/show_bench.py gpurun_out/abs_g$v.log | grep -E "ms/step|gather_rows" >> gpurun_out/abs_small.txt
done
for c in 2 8; do
  DION2_HOST_CHUNKS=$c timeout 600 $B > gpurun_out/abs_c$c.log 2>&1
  tail -n 1 gpurun_out/abs_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $c e2e', d['e2e']['value'])" >> gpurun_out/abs_small.txt
done
