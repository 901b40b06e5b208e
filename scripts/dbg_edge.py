"""Edge-case probe (debugging aid): short X with extreme spikes through the distributed step."""
import sys
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
from gpu_harness import run_parity_dist
for shapes, alpha, world in (([(32, 1600), (48, 3200)], 0.25, 2), ([(256, 2048), (1024, 512)], 0.0625, 4),
                             ([(128, 4096)], 0.25, 8)):
    for r, ratio in ((1, 250), (16, 250), (4, 100)):
        res = run_parity_dist(shapes, alpha, world, steps=2, structure=dict(kind="spike", rank=r, ratio=ratio))
        print(shapes, alpha, world, r, ratio, [round(x, 4) for x in res.dW_rel], res.index_mismatch, flush=True)
