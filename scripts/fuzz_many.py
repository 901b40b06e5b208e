"""Bulk seeded fuzzing against the oracle (bug hunting; the committed subset is tests/test_gpu_fuzz.py).

    python scripts/fuzz_many.py --cases 300 --start 10000 > gpurun_out/fuzz_many.json
"""
import argparse
import json
import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from gpu_harness import run_parity, run_parity_dist  # noqa: E402

ALPHAS = [0.0625, 0.125, 0.25, 0.5, 1.0]


def dim(rng, hi=3000):
    r = rng.random()
    if r < 0.4:
        return int(rng.integers(1, hi // 64)) * 64
    if r < 0.5:
        return int(rng.integers(1, 8))          # tiny
    return int(rng.integers(8, hi))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=100)
    ap.add_argument("--start", type=int, default=10000)
    args = ap.parse_args()
    fails, done = [], 0
    for i in range(args.start, args.start + args.cases):
        rng = np.random.default_rng(i)
        kind = rng.choice(["single", "single", "single", "dist"])
        try:
            if kind == "single":
                shapes = [(dim(rng), dim(rng)) for _ in range(int(rng.integers(1, 6)))]
                alpha = float(rng.choice(ALPHAS))
                kw = dict(m_transposed=bool(rng.random() < 0.5))
                o = int(rng.integers(0, 8))
                if o == 0:
                    kw["storage_transposed"] = True
                elif o == 1:
                    kw.update(select="random", sel_seed=int(rng.integers(0, 1 << 30)))
                elif o == 2:
                    kw["grad_bf16"] = True
                elif o == 3:
                    kw["structure"] = dict(kind="spike", rank=int(rng.choice([1, 4, 16])),
                                           ratio=float(rng.choice([20, 100, 250])))
                elif o == 4:
                    kw["structure"] = dict(kind="power", gamma=float(rng.choice([0.75, 1.0])))
                elif o == 5:
                    kw["ns_form"] = "direct"
                res = run_parity(shapes, alpha, "auto", "bf16", steps=2, row_scaled=True, **kw)
                ok = (res.index_mismatch == 0 and max(res.dW_rel) <= 2e-2 and res.unselected_w_bitwise
                      and res.unselected_m_bitwise and max(res.M_rel) <= 1e-5)
                rec = dict(i=i, kind="single", shapes=shapes, alpha=alpha, kw={k: str(v) for k, v in kw.items()},
                           dW=max(res.dW_rel), idx=res.index_mismatch, ok=ok)
            else:
                world = int(rng.choice([2, 3, 4, 8]))
                unit = 8 * world
                shapes = [(int(rng.integers(1, 40)) * unit, int(rng.integers(1, 40)) * unit)
                          for _ in range(int(rng.integers(1, 5)))]
                alpha = float(rng.choice([0.125, 0.25, 0.5]))
                direct = bool(rng.random() < 0.5)
                mt = bool(rng.random() < 0.5)
                structure = None
                if rng.random() < 0.3:
                    structure = dict(kind="spike", rank=int(rng.choice([1, 4, 16])),
                                     ratio=float(rng.choice([20, 100, 250])))
                res = run_parity_dist(shapes, alpha, world, steps=2, direct=direct, m_transposed=mt,
                                      structure=structure)
                ok = res.index_mismatch == 0 and max(res.dW_rel) <= 2e-2 and max(res.M_rel) <= 1e-5
                rec = dict(i=i, kind="dist", world=world, shapes=shapes, alpha=alpha, direct=direct, mt=mt,
                           structure=str(structure), dW=max(res.dW_rel), idx=res.index_mismatch, ok=ok)
        except Exception as e:  # noqa: BLE001
            msg = repr(e)
            # unsupported configurations are reported by the library, not failures of the step
            ok = "EUNSUPPORTED" in msg or "EINVAL_SHAPE" in msg
            rec = dict(i=i, kind=str(kind), error=msg[:300], ok=ok, tb=traceback.format_exc()[-600:] if not ok else "")
        done += 1
        if not rec["ok"]:
            fails.append(rec)
        print(json.dumps(rec), flush=True)
    print(json.dumps({"done": done, "failures": len(fails)}))


if __name__ == "__main__":
    main()
