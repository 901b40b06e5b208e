"""Edge-case probe (debugging aid): re-run one fuzz case by its seed."""
import sys
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
from gpu_harness import run_parity
r = run_parity([(2112, 1992), (1006, 2428), (1, 1)], 0.0625, "auto", "bf16", steps=2, row_scaled=True)
print([round(x, 6) for x in r.dW_rel], r.index_mismatch)
