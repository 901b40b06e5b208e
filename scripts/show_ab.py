"""Summarise scripts/ab_ns.sh output: step time and per-phase ms per variant."""
import glob
import json
import os
import sys

root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
for log in sorted(glob.glob(os.path.join(root, "abns_*.log"))):
    name = os.path.basename(log)[5:-4]
    try:
        line = json.loads(open(log).read().strip().splitlines()[-1])
        det = json.load(open(os.path.join(root, f"abns_details_{name}.json")))
    except Exception as e:  # noqa: BLE001
        print(name, "no result", e)
        continue
    ph = {k: round(v["ms_per_step"], 3) for k, v in det["phases"].items()}
    keys = sys.argv[1:] or list(ph)
    print(f"{name:14s} {line['value']:.3f}", {k: ph.get(k) for k in keys})
