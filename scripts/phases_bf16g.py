"""Per-phase device time of the 1B-set step with fp32 and with bf16 gradients."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import layer_set_1b  # noqa: E402
from paper_2512_16928_b200 import Dion2, get_phase_times, set_phase_timing  # noqa: E402

shapes = layer_set_1b(24)
mts = [m > n for (m, n) in shapes]
Ws = [torch.randn(m, n, device="cuda") / math.sqrt(n) for (m, n) in shapes]
Ms = [torch.zeros((n, m) if mt else (m, n), device="cuda") for (m, n), mt in zip(shapes, mts)]
for dt in (torch.float32, torch.bfloat16):
    Gs = [torch.randn(m, n, device="cuda").to(dt) for (m, n) in shapes]
    opt = Dion2(alpha=0.25, m_transposed=mts)
    opt.step(Ws, Ms, Gs)
    torch.cuda.synchronize()
    set_phase_timing(True)
    for _ in range(3):
        opt.step(Ws, Ms, Gs)
    ph = get_phase_times()
    set_phase_timing(False)
    print(dt, {k: round(v[0] / 3, 3) for k, v in ph.items() if v[1]})
    del Gs, opt
    torch.cuda.empty_cache()
