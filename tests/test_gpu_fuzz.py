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


@pytest.mark.parametrize("i", range(24))
def test_fuzz_options(i):
    """Random shapes crossed with the step's options: storage layout, random selection, full
    decay, the submatrix scale, bf16 gradients, forced evaluation form (Gram only where R25
    allows it: p >= 64), per-iteration coefficient tables."""
    shapes, alpha, mt = _case(100 + i)
    rng = np.random.default_rng(4000 + i)
    kw = dict(m_transposed=mt)
    opt = i % 6
    if opt == 0:
        kw["storage_transposed"] = True
    elif opt == 1:
        kw.update(select="random", sel_seed=int(rng.integers(0, 1 << 30)))
    elif opt == 2:
        kw["decay_mode"] = 1
    elif opt == 3:
        kw["scale_mode"] = 1
    elif opt == 4:
        kw["ns_form"] = "direct"
        kw["grad_bf16"] = True
    else:
        kw["ns_coeffs"] = [(3.4445, -4.7750, 2.0315)] * 3 + [(1.5, -0.5, 0.0)] * int(rng.integers(1, 6))
    res = run_parity(shapes, alpha, "auto", "bf16", steps=2, row_scaled=True, **kw)
    assert res.index_mismatch == 0, (shapes, alpha, kw, res)
    assert max(res.dW_rel) <= GATE, (shapes, alpha, kw, res)
    assert res.unselected_w_bitwise, (shapes, alpha, kw, res)
    if kw.get("decay_mode") != 1:
        assert res.unselected_m_bitwise, (shapes, alpha, kw, res)
    assert max(res.M_rel) <= 1e-5, (shapes, alpha, kw, res)


@pytest.mark.parametrize("i", range(8))
def test_fuzz_dpsync_loopback(i):
    """Compressed DP-sync on random shapes: replicas stay bit-identical (NCCL-emulating and direct
    reduce give the same bits) and match the oracle's replica model."""
    import torch
    import oracle as O
    from paper_2512_16928_b200 import dion2 as D
    from synth import gen_grad, gen_w0
    rng = np.random.default_rng(5000 + i)
    world = int(rng.choice([2, 3, 4]))
    shapes = [(_dim(rng), _dim(rng)) for _ in range(int(rng.integers(1, 4)))]
    alpha = float(rng.choice([0.125, 0.25, 0.5]))
    outs = []
    for direct in (False, True):
        W = [[torch.from_numpy(gen_w0(m, n, 7, j)).cuda() for j, (m, n) in enumerate(shapes)] for _ in range(world)]
        M = [[torch.zeros(m, n, device="cuda") for (m, n) in shapes] for _ in range(world)]
        opt = D.Dion2DpSync(loopback_world=world, alpha=alpha, seed=11, dist_direct=direct)
        Wr = [[gen_w0(m, n, 7, j).astype(np.float64) for j, (m, n) in enumerate(shapes)] for _ in range(world)]
        Mr = [[np.zeros((m, n)) for (m, n) in shapes] for _ in range(world)]
        for t in range(2):
            G = [[gen_grad(m, n, 50 + r, j, t) for j, (m, n) in enumerate(shapes)] for r in range(world)]
            opt.step(W, M, [[torch.from_numpy(g).cuda() for g in G[r]] for r in range(world)], step=t)
            cfg = O.OracleConfig(alpha=float(np.float32(alpha)), select="random", seed=11, step=t)
            for j in range(len(shapes)):
                O.dion2_step_dpsync([Wr[r][j] for r in range(world)], [Mr[r][j] for r in range(world)],
                                    [G[r][j].astype(np.float64) for r in range(world)], cfg, matrix_id=j)
        torch.cuda.synchronize()
        for j, (m, n) in enumerate(shapes):
            w0 = gen_w0(m, n, 7, j).astype(np.float64)
            for r in range(world):
                assert torch.equal(W[r][j], W[0][j])
            wg = W[0][j].cpu().double().numpy()
            err = np.linalg.norm((wg - w0) - (Wr[0][j] - w0)) / max(np.linalg.norm(Wr[0][j] - w0), 1e-30)
            assert err <= GATE, (world, shapes, alpha, direct, j, err)
        outs.append([w.clone() for w in W[0]])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
