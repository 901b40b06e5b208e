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
# bf16 weights, split-K gram (two long matrices), the distributed step and DP-sync in loopback
Wb = [torch.from_numpy(gen_w0(m, n, 3, i)).cuda().to(torch.bfloat16) for i, (m, n) in enumerate(shapes)]
Mb = [torch.zeros(m, n, device="cuda") for (m, n) in shapes]
Dion2(alpha=0.25).step(Wb, Mb, [torch.from_numpy(gen_grad(m, n, 3, i)).cuda() for i, (m, n) in enumerate(shapes)])
big = [(1024, 16384), (8192, 1024)]
Ws = [torch.from_numpy(gen_w0(m, n, 4, i)).cuda() for i, (m, n) in enumerate(big)]
Dion2(alpha=0.0625).step(Ws, [torch.zeros_like(w) for w in Ws],
                         [torch.from_numpy(gen_grad(m, n, 4, i)).cuda() for i, (m, n) in enumerate(big)])
torch.cuda.synchronize()
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_harness import run_parity_dist  # noqa: E402
r = run_parity_dist([(256, 512), (512, 256), (1024, 1024)], 0.25, 2, steps=2)
assert r.index_mismatch == 0, r
import test_gpu_dpsync as T  # noqa: E402
T._run(2, "bf16", 2e-2, steps=2)
print("sanitize_step ok")
