"""Per-phase device time of the single-GPU step on L layers of the 1B set (a P = 24/L rank's
owned-matrix mix at 1 layer per ... e.g. --layers 3 = 18 matrices, the P = 8 owner's share).

    python scripts/probe_phases.py --layers 3 [--steps 5]
"""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import layer_set_1b  # noqa: E402
from paper_2512_16928_b200 import Dion2, get_phase_times, set_phase_timing  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--alpha", type=float, default=0.25)
    args = ap.parse_args()
    shapes = layer_set_1b(args.layers)
    mts = [m > n for (m, n) in shapes]
    Ws = [torch.randn(m, n, device="cuda") / math.sqrt(n) for (m, n) in shapes]
    Ms = [torch.zeros(n, m, device="cuda") if mt else torch.zeros(m, n, device="cuda") for (m, n), mt in zip(shapes, mts)]
    Gs = [torch.randn(m, n, device="cuda") for (m, n) in shapes]
    opt = Dion2(alpha=args.alpha, m_transposed=mts)
    for _ in range(2):
        opt.step(Ws, Ms, Gs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        opt.step(Ws, Ms, Gs)
    e1.record()
    torch.cuda.synchronize()
    set_phase_timing(True)
    for _ in range(args.steps):
        opt.step(Ws, Ms, Gs)
    ph = get_phase_times()
    set_phase_timing(False)
    print(json.dumps({"layers": args.layers, "matrices": len(shapes), "ms_per_step": e0.elapsed_time(e1) / args.steps,
                      "phases_ms": {k: v[0] / args.steps for k, v in ph.items() if v[1]},
                      "launches": {k: v[1] / args.steps for k, v in ph.items() if v[1]}}, indent=1))


if __name__ == "__main__":
    main()
