"""Print the headline and per-phase table of bench.py JSON lines (files given on argv)."""
import json
import sys

for f in sys.argv[1:]:
    line = [l for l in open(f) if l.startswith("{")]
    if not line:
        print(f, "no JSON line;", open(f).read()[-600:])
        continue
    j = json.loads(line[-1])
    r = j.get("roofline", {})
    print(f"{f}: {j['value']:.3f} {j['unit']}  roofline {r.get('kernel')} frac {r.get('frac')}  "
          f"e2e {j.get('e2e', {}).get('value')}  clocks {j.get('clocks', {}).get('sm_mhz')}")
    for k, v in j.get("phases", {}).items():
        print(f"    {k:16s} {v['ms_per_step']:.3f} ms  x{v['launches_per_step']:.0f}  "
              f"{v.get('tflops', 0):7.1f} TF/s  hbm {v.get('frac_hbm', 0):.3f}")
