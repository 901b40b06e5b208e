"""Seeded shape fuzzing against the fp64 oracle (-m gpu).

Random matrix sets (ragged and tile-aligned sizes from 8 to 3000, both orientations, α from
1/16 to 1, M in W's layout or transposed) through the single-GPU step, and random rank counts
and shard-compatible shapes through the distributed step in loopback (plain and direct
exchange).  Same gates as the parity suite: exact index sets, 2e-2 on the cumulative update,
bitwise-untouched unselected rows / columns, momentum within 1e-5.  The cases are drawn from a
fixed seed, so a failure names a reproducible shape set.
"""
import numpy as np
import pytest

from gpu_harness import run_parity, run_parity_dist

pytestmark = pytest.mark.gpu

GATE = 2e-2
ALPHAS = [0.0625, 0.125, 0.25, 0.5, 1.0]


def _dim(rng):
    if rng.random() < 0.5:
        return int(rng.integers(1, 48)) * 64           # tile-aligned
    return int(rng.integers(8, 3000))                  # ragged


def _case(i):
    rng = np.random.default_rng(1000 + i)
    shapes = [(_dim(rng), _dim(rng)) for _ in range(int(rng.integers(1, 5)))]
    return shapes, float(rng.choice(ALPHAS)), bool(rng.random() < 0.5)


@pytest.mark.parametrize("i", range(40))
def test_fuzz_single_gpu(i):
    shapes, alpha, mt = _case(i)
    rng = np.random.default_rng(3000 + i)
    kw = {}
    if i % 4 == 1:  # an ill-conditioned (spiked) gradient spectrum
        kw["structure"] = dict(kind="spike", rank=int(rng.choice([1, 4, 16])), ratio=float(rng.choice([20, 100, 250])))
    elif i % 4 == 2:
        kw["grad_bf16"] = True
    res = run_parity(shapes, alpha, "auto", "bf16", steps=2, row_scaled=True, m_transposed=mt, **kw)
    assert res.index_mismatch == 0, (shapes, alpha, res)
    assert max(res.dW_rel) <= GATE, (shapes, alpha, mt, res)
    assert res.unselected_w_bitwise and res.unselected_m_bitwise, (shapes, alpha, res)
    assert max(res.M_rel) <= 1e-5, (shapes, alpha, res)


@pytest.mark.parametrize("i", range(16))
def test_fuzz_loopback_dist(i):
    rng = np.random.default_rng(2000 + i)
    world = int(rng.choice([2, 3, 4, 8]))
    unit = 8 * world  # every shard width o / P a multiple of 8
    shapes = [(int(rng.integers(4, 40)) * unit, int(rng.integers(4, 40)) * unit) for _ in range(int(rng.integers(2, 5)))]
    alpha = float(rng.choice([0.125, 0.25, 0.5]))
    direct = bool(rng.random() < 0.5)
    res = run_parity_dist(shapes, alpha, world, steps=2, direct=direct)
    assert res.index_mismatch == 0 and max(res.dW_rel) <= GATE and max(res.M_rel) <= 1e-5, \
        (world, shapes, alpha, direct, res)
