"""bench.py's work accounting (-m "not gpu"): the algorithmic FLOPs and bytes behind the
reported roofline fractions, pinned to SURVEY.md section 8(d)'s table and to closed forms.

The per-unit figures: NS FLOPs T(4p^2 q + 2p^3) per matrix in the
direct form; in the Gram-space form with restarts (readings R23, R24) 4p^2 q + (4 Ts - 3) 2p^3 per
segment of Ts iterations (segments 3 + 2 at T = 5: 8p^2 q + 28 p^3); HBM bytes
m n (b_G + 8) for momentum + score and 10 k o each for the gather and the scatter.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth import layer_set_1b, layer_set_8b  # noqa: E402


def test_1b_set_shape_census():
    shapes = layer_set_1b(24)
    assert len(shapes) == 144
    assert sum(m * n for m, n in shapes) == 1_207_959_552  # 1.208 B parameters
    assert len(layer_set_8b(32)) == 224 and abs(sum(m * n for m, n in layer_set_8b(32)) - 6.98e9) < 0.01e9


@pytest.mark.parametrize("alpha,tflop", [(1.0, 61.85), (0.5, 13.92), (0.25, 3.29), (0.125, 0.80)])
def test_direct_ns_flops_match_survey_table(alpha, tflop):
    """SURVEY 8(d) cfg 2: NS FLOP 61.85 / 13.92 / 3.29 / 0.80 TFLOP for alpha 1 / 0.5 / 0.25 / 0.125."""
    f, _ = bench.work_model(layer_set_1b(24), alpha, ns_form="direct")
    assert abs(sum(f.values()) / 1e12 - tflop) < 0.01


def test_restart_segments():
    assert bench.ns_segments(5) == [3, 2]
    assert bench.ns_segments(1) == [1]
    assert bench.ns_segments(7) == [3, 3, 1]


def test_gram_form_flops_closed_form():
    """Gram space at alpha = 0.25: every matrix has p = 512 and q = 2048 or 8192 (q >= 2p);
    two restart segments (3 + 2 iterations)."""
    f, _ = bench.work_model(layer_set_1b(24), 0.25, ns_form="auto")
    p = 512
    want = sum(8 * p * p * q + ((4 * 3 - 3) + (4 * 2 - 3)) * 2 * p ** 3 for q in [2048] * 96 + [8192] * 48)
    assert abs(sum(f.values()) - want) < 1e3
    assert abs(sum(f.values()) / 1e12 - 1.78) < 0.005  # DESIGN 6: 1.78 TFLOP with the restart (1.85x fewer)
    # alpha = 1: the square matrices have q = p (direct form), the 2048 x 8192 ones q = 4p (Gram)
    sq = [(2048, 2048)] * 96
    f1, _ = bench.work_model(sq, 1.0, ns_form="auto")
    fd, _ = bench.work_model(sq, 1.0, ns_form="direct")
    assert sum(f1.values()) == sum(fd.values())
    rect = [(8192, 2048), (2048, 8192)]
    fa, _ = bench.work_model(rect, 1.0, ns_form="auto")
    assert sum(fa.values()) == 2 * (8 * 2048 ** 2 * 8192 + 14 * 2 * 2048 ** 3)


@pytest.mark.parametrize("alpha,gb", [(1.0, 33.8), (0.5, 24.2), (0.25, 19.3), (0.125, 16.9)])
def test_hbm_bytes_match_survey_table(alpha, gb):
    """SURVEY 8(d) cfg 2 algorithmic HBM bytes 33.8 / 24.2 / 19.3 / 16.9 GB: (12 + 16 alpha) B per
    parameter with fp32 G, plus the bf16 workspace traffic of X and O (4 B per selected
    element) that the per-phase accounting also charges."""
    _, b = bench.work_model(layer_set_1b(24), alpha)
    n = 1_207_959_552
    k1 = b["momentum_score"] + b["momentum_score_mt"]
    assert abs(k1 - 12 * n) / (12 * n) < 1e-3                     # + 4 d per matrix of scores
    sel = sum(v for k, v in b.items() if k.startswith(("gather", "scatter")))
    assert abs(sel - 20 * alpha * n) / (20 * alpha * n) < 1e-9     # 10 B in + 10 B out per selected element
    assert abs((k1 + sel - 4 * alpha * n) / 1e9 - gb) < 0.1


def test_stress_config_shapes():
    """configs[4]: 4096 x 32768 (rows mode, k = 256) and 28672 x 8192 (cols mode, k = 512) at
    alpha = 1/16; 43.1 and 151.7 GFLOP of NS (direct count)."""
    shapes = bench.model_shapes("stress")
    assert shapes == [(4096, 32768), (28672, 8192)]
    f0, _ = bench.work_model(shapes[:1], 0.0625, ns_form="direct")
    f1, _ = bench.work_model(shapes[1:], 0.0625, ns_form="direct")
    assert abs(sum(f0.values()) / 1e9 - 43.1) < 0.1 and abs(sum(f1.values()) / 1e9 - 151.7) < 0.1


def test_reference_arm_json_contract():
    """`bench.py --impl reference` (the fp64 oracle on the host cores, one layer per step,
    scaled to the model) prints one JSON line with the contract's keys, no GPU needed."""
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["higher_is_better"] is False and line["unit"] == "ms/step"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_mma_flops_credit_only_the_computed_tiles():
    """Tensor-core work: p = 512 -> 2 x 2 tiles of 256, 3 upper tiles computed for the symmetric
    products (gram, poly, p x p products); the apply is a full product."""
    f = bench.mma_flops([(2048, 2048)], 0.25)           # X 512 x 2048, Gram form
    p, q = 512, 2048
    want = sum(0.75 * 2 * p * p * q + 2 * p * p * q + 0.75 * (ts + 3 * ts - 3) * 2 * p ** 3 for ts in (3, 2))
    assert f == want
    assert abs(bench.mma_flops(layer_set_1b(24), 0.25) / 1e12 - 1.488) < 0.001


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """`bench.py --gpus N` without WORLD_SIZE re-runs itself under torch.distributed.run with N
    ranks on 127.0.0.1 (the driver's multi-GPU launch, done by the script itself)."""
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "3"]
