"""Per-phase device time of the owner-compute step in loopback mode (all P ranks on one GPU).

Loopback runs every rank's kernels back to back on one device, so phase time / P estimates
one rank's compute at P GPUs (the exchanges are device copies here, NVLink there).

    python scripts/loopback_phases.py --world 2 4 8
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
from paper_2512_16928_b200 import dion2 as D  # noqa: E402
from paper_2512_16928_b200 import get_phase_times, set_phase_timing  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--direct", action="store_true", help="direct peer exchange (DION2_FLAG_DIST_DIRECT)")
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays (Dion2Loopback(cuda_graph=True))")
    args = ap.parse_args()
    shapes = layer_set_1b(24)
    out = {}
    for P in args.world:
        info = D.dist_info(shapes, P, 0, alpha=args.alpha)
        mts = [ax == 1 for ax in info["axis"]]
        Ws, Ms, Gs = [], [], []
        for r in range(P):
            ir = D.dist_info(shapes, P, r, alpha=args.alpha, m_transposed=mts)
            w, m, g = [], [], []
            for (sr, sc), mt, (_, n) in zip(ir["shard"], mts, shapes):
                w.append(torch.randn(sr, sc, device="cuda") / math.sqrt(n))
                m.append(torch.zeros((sc, sr) if mt else (sr, sc), device="cuda"))
                g.append(torch.randn(sr, sc, device="cuda"))
            Ws.append(w), Ms.append(m), Gs.append(g)
        opt = D.Dion2Loopback(shapes, P, alpha=args.alpha, m_transposed=mts, dist_direct=args.direct,
                              cuda_graph=args.graph)
        for _ in range(3 if args.graph else 1):  # graph mode captures on the second call
            opt.step(Ws, Ms, Gs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            opt.step(Ws, Ms, Gs)
        e1.record()
        torch.cuda.synchronize()
        total = e0.elapsed_time(e1) / args.steps
        set_phase_timing(True)
        opt_e = D.Dion2Loopback(shapes, P, alpha=args.alpha, m_transposed=mts, dist_direct=args.direct)
        opt_e.step(Ws, Ms, Gs)
        get_phase_times()  # drop the plan-building step's events
        for _ in range(args.steps):
            opt_e.step(Ws, Ms, Gs)
        ph = get_phase_times()
        set_phase_timing(False)
        out[P] = {"ms_all_ranks": total, "ms_per_rank_est": total / P,
                  "phases_ms_per_rank": {k: v[0] / args.steps / P for k, v in ph.items() if v[1]},
                  # rank 0's bytes sent (the loopback transport counts rank 0's side)
                  "exchange_bytes_rank0": opt.last_comm_bytes}
        del Ws, Ms, Gs, opt
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
