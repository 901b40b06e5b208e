"""Soak / determinism check: many steps of the same seeded trajectory in CUDA-graph mode and in
eager mode (single GPU), and the loopback distributed step with the direct exchange in graph vs
eager mode; the final W and M must be bit-identical (a race between launches, e.g. across the
programmatic-dependent-launch overlap, would show as a mismatch).

    python scripts/soak.py --steps 300 --layers 4
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
from paper_2512_16928_b200 import Dion2  # noqa: E402
from paper_2512_16928_b200 import dion2 as D  # noqa: E402


def state(shapes, mts, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    W = [torch.randn(m, n, device="cuda", generator=g) / math.sqrt(n) for (m, n) in shapes]
    M = [torch.zeros((n, m) if mt else (m, n), device="cuda") for (m, n), mt in zip(shapes, mts)]
    G = [torch.empty(m, n, device="cuda") for (m, n) in shapes]
    return W, M, G


def run_single(shapes, steps, graph):
    mts = [m > n for (m, n) in shapes]
    W, M, G = state(shapes, mts, 1)
    opt = Dion2(alpha=0.25, m_transposed=mts, cuda_graph=graph)
    gen = torch.Generator(device="cuda").manual_seed(2)
    for t in range(steps):
        for x in G:
            x.normal_(generator=gen)
        opt.step(W, M, G, lr=0.02 * (1 - t / (2 * steps)))
    torch.cuda.synchronize()
    assert opt.status()[0] == 0
    return W, M


def run_loopback(shapes, world, steps, graph):
    info = D.dist_info(shapes, world, 0)
    axes = info["axis"]
    W, M, G = [], [], []
    for r in range(world):
        ir = D.dist_info(shapes, world, r)
        g = torch.Generator(device="cuda").manual_seed(10 + r)
        W.append([torch.randn(sr, sc, device="cuda", generator=g) / 32 for (sr, sc) in ir["shard"]])
        M.append([torch.zeros(sr, sc, device="cuda") for (sr, sc) in ir["shard"]])
        G.append([torch.empty(sr, sc, device="cuda") for (sr, sc) in ir["shard"]])
    opt = D.Dion2Loopback(shapes, world, alpha=0.25, dist_direct=True, cuda_graph=graph)
    gen = torch.Generator(device="cuda").manual_seed(3)
    for t in range(steps):
        for gr in G:
            for x in gr:
                x.normal_(generator=gen)
        opt.step(W, M, G)
    torch.cuda.synchronize()
    del axes
    return [w for ws in W for w in ws], [m for ms in M for m in ms]


def same(a, b):
    return all(torch.equal(x, y) for x, y in zip(a, b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--layers", type=int, default=4)
    args = ap.parse_args()
    shapes = layer_set_1b(args.layers)
    out = {}
    Wg, Mg = run_single(shapes, args.steps, True)
    We, Me = run_single(shapes, args.steps, False)
    out["single_graph_vs_eager_bitwise"] = same(Wg, We) and same(Mg, Me)
    Wg2, Mg2 = run_single(shapes, args.steps, True)
    out["single_graph_rerun_bitwise"] = same(Wg, Wg2) and same(Mg, Mg2)
    lw, lm = run_loopback(shapes, 4, args.steps // 3, True)
    ew, em = run_loopback(shapes, 4, args.steps // 3, False)
    out["loopback_direct_graph_vs_eager_bitwise"] = same(lw, ew) and same(lm, em)
    out["steps"] = args.steps
    out["layers"] = args.layers
    print(json.dumps(out))


if __name__ == "__main__":
    main()
