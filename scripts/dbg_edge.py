"""Edge-case probe (debugging aid): a 1 x 1 weight batched with a larger matrix, two steps."""
import sys
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
import torch
from paper_2512_16928_b200 import Dion2

for shapes in ([(300, 1200), (1, 1)], [(1, 1)]):
    torch.manual_seed(0)
    W = [torch.randn(m, n, device="cuda") for m, n in shapes]
    M = [torch.zeros(m, n, device="cuda") for m, n in shapes]
    opt = Dion2(alpha=0.0625)
    j = len(shapes) - 1
    for t in range(3):
        G = [torch.randn(m, n, device="cuda") for m, n in shapes]
        O = [torch.full((max(1, round(0.0625 * min(m, n))) if m <= n else m, n if m <= n else max(1, round(0.0625 * n))),
                        -7.0, device="cuda") for m, n in shapes]
        Wb, Mb = W[j].item(), M[j].item()
        opt.step(W, M, G, O_out=O)
        torch.cuda.synchronize()
        g = G[j].item()
        m_acc = Mb + g
        exp_o = 0.697265625 * (1 if m_acc > 0 else -1)
        print(shapes, "t", t, "O", O[j].item(), "expected", exp_o, "dW", W[j].item() - Wb, "M", M[j].item(), "exp M", 0.95 * m_acc,
              "status", opt.status(), flush=True)
