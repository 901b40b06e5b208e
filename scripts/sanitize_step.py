"""A few small Dion2 steps exercising every kernel family (row / transposed-M / generic
paths, split-K gram, both NS forms, column scatter by index walk, random selection); with
DION2_DEBUG_SYNC=1 every launch is synchronised and checked.  Under compute-sanitizer:
    compute-sanitizer --tool memcheck python scripts/sanitize_step.py

    DION2_DEBUG_SYNC=1 python scripts/sanitize_step.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import gen_grad, gen_w0  # noqa: E402
from paper_2512_16928_b200 import Dion2  # noqa: E402

shapes = [(512, 1024), (1024, 512), (2048, 512), (300, 520), (520, 300), (512, 4096), (7, 33), (256, 128)]
mt = [m > n and m % 256 == 0 for (m, n) in shapes]
for form in ("auto", "direct"):
    for sel in ("l1", "random"):
        Ws = [torch.from_numpy(gen_w0(m, n, 1, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Ms = [torch.zeros(n, m, device="cuda") if t else torch.zeros(m, n, device="cuda") for (m, n), t in zip(shapes, mt)]
        opt = Dion2(alpha=0.25, m_transposed=mt, ns_form=form, select=sel)
        for t in range(2):
            Gs = [torch.from_numpy(gen_grad(m, n, 1, i, t)).cuda() for i, (m, n) in enumerate(shapes)]
            opt.step(Ws, Ms, Gs)
        torch.cuda.synchronize()
        assert opt.status() == (0, -1), opt.status()
print("sanitize_step ok")
