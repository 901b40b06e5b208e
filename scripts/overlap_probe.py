"""Feasibility probe: the 1B set split into its 48 large (512 x 8192 NS) and 96 square matrices,
stepped (a) as one batched call, (b) as two calls back to back on one stream, (c) as two
calls on two streams at once (the GPU overlaps whatever kernels fit side by side).

    python scripts/overlap_probe.py
"""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import layer_set_1b  # noqa: E402
from paper_2512_16928_b200 import Dion2  # noqa: E402


def state(shapes, mts):
    Ws = [torch.randn(m, n, device="cuda") / math.sqrt(n) for (m, n) in shapes]
    Ms = [torch.zeros((n, m) if t else (m, n), device="cuda") for (m, n), t in zip(shapes, mts)]
    Gs = [torch.randn(m, n, device="cuda") for (m, n) in shapes]
    return Ws, Ms, Gs


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


shapes = layer_set_1b(24)
big = [s for s in shapes if max(s) == 8192]
small = [s for s in shapes if max(s) == 2048]
mt = lambda ss: [m > n for (m, n) in ss]  # noqa: E731
Wa, Ma, Ga = state(shapes, mt(shapes))
Wb, Mb, Gb = state(big, mt(big))
Ws, Ms, Gs = state(small, mt(small))
one = Dion2(alpha=0.25, m_transposed=mt(shapes))
ob = Dion2(alpha=0.25, m_transposed=mt(big))
osm = Dion2(alpha=0.25, m_transposed=mt(small))
s1, s2 = torch.cuda.Stream(priority=-1), torch.cuda.Stream()
out = {"one_call": timeit(lambda: one.step(Wa, Ma, Ga))}
out["two_calls_one_stream"] = timeit(lambda: (ob.step(Wb, Mb, Gb), osm.step(Ws, Ms, Gs)))
out["big_only"] = timeit(lambda: ob.step(Wb, Mb, Gb))
out["small_only"] = timeit(lambda: osm.step(Ws, Ms, Gs))


def two_streams():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    ob.step(Wb, Mb, Gb, stream=s1)
    osm.step(Ws, Ms, Gs, stream=s2)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


out["two_calls_two_streams"] = timeit(two_streams)
print(json.dumps(out, indent=1))
