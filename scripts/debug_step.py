import os, sys, math, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16928_b200 import Dion2
from bench import build_state, model_shapes
shapes = model_shapes("1b")
bufs, Ws, Ms, Gs = build_state(shapes, torch.device("cuda"))
for alpha in [0.25, 1.0, 0.25, 0.5, 0.125]:
    opt = Dion2(alpha=alpha)
    print("alpha", alpha, flush=True)
    opt.step(Ws, Ms, Gs)
    torch.cuda.synchronize()
    print("  ok", opt.status(), flush=True)
    del opt
    torch.cuda.empty_cache()
