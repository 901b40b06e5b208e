"""Full-size parity in the benchmark's launch configuration (-m gpu).

BASELINE configs[1] (the 1B set, 144 matrices, alpha = 0.25) stepped exactly as bench.py
times it: one batched call over all matrices, column-mode momentum stored transposed, the
default (Gram-space, restarted, fp16) Newton-Schulz plan.  SURVEY 8(c.3)'s 10-step trajectory:
the oracle follows a sample of matrices one at a time for all 10 steps (each matrix's step
depends only on its own W, M, G), on Gaussian gradients and on gradients with a fixed rank-4
spike (sigma_1 / median of the selected rows ~ 50-100, the momenta real training produces);
properties that hold at any size are checked on every matrix at every step:
  * the selected set is strictly ascending, in range, of size k;
  * unselected rows/columns of W are bit-identical, unselected M == fp32(M + G) bitwise.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from synth import layer_set_1b
from paper_2512_16928_b200 import Dion2

from gpu_harness import _tie_equivalent

pytestmark = pytest.mark.gpu

ALPHA = 0.25
SAMPLE = [0, 3, 4, 5, 64, 70, 143]  # q, o, up (cols, M^T), down of layer 0; k of layer 10; up/down later


def _state(shapes, mts, seed):
    total = sum(m * n for m, n in shapes)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    W = torch.empty(total, device="cuda").normal_(0.0, 1.0, generator=gen)
    M = torch.zeros(total, device="cuda")
    G = torch.empty(total, device="cuda")
    Ws, Ms, Gs, off = [], [], [], 0
    for (m, n), mt in zip(shapes, mts):
        Ws.append(W[off:off + m * n].view(m, n).mul_(1.0 / math.sqrt(n)))
        Ms.append(M[off:off + m * n].view((n, m) if mt else (m, n)))
        Gs.append(G[off:off + m * n].view(m, n))
        off += m * n
    return (W, M, G), Ws, Ms, Gs, gen


@pytest.mark.parametrize("spike", [0.0, 100.0])
def test_full_1b_set_trajectory(spike):
    shapes = layer_set_1b(24)
    assert len(shapes) == 144
    cfg = O.OracleConfig(alpha=float(np.float32(ALPHA)), mu=float(np.float32(0.95)), lr=float(np.float32(0.02)))
    axes = [O.resolve_axis(m, n, O.AXIS_AUTO) for (m, n) in shapes]
    mts = [ax == O.AXIS_COLS for ax in axes]
    ks = [O.select_count(cfg.alpha, m if ax == O.AXIS_ROWS else n) for (m, n), ax in zip(shapes, axes)]
    (Wf, Mf, Gf), Ws, Ms, Gs, gen = _state(shapes, mts, seed=7)
    Mv = lambda i: Ms[i].T if mts[i] else Ms[i]  # noqa: E731
    opt = Dion2(alpha=ALPHA, axis="auto", precision="bf16", m_transposed=mts)
    W0 = {i: Ws[i].cpu().numpy().astype(np.float64) for i in SAMPLE}
    Wr = {i: W0[i].copy() for i in SAMPLE}
    Mr = {i: np.zeros(shapes[i]) for i in SAMPLE}
    ties = 0
    spikes = []
    if spike:  # a fixed rank-4 spike per matrix: G = Z + spike * sqrt(max(m, n)) U V^T (synth recipe)
        for (m, n) in shapes:
            u = torch.linalg.qr(torch.randn(m, 4, device="cuda", generator=gen))[0]
            v = torch.linalg.qr(torch.randn(n, 4, device="cuda", generator=gen))[0]
            spikes.append((spike * math.sqrt(max(m, n))) * (u @ v.T))
    for t in range(10):
        Gf.normal_(0.0, 1.0, generator=gen)
        for i, sp in enumerate(spikes):
            Gs[i].add_(sp)
        Gc = {i: Gs[i].cpu().numpy().astype(np.float64) for i in SAMPLE}
        sel = [torch.empty(k, dtype=torch.int32, device="cuda") for k in ks]
        W_before, M_before = Wf.clone(), Mf.clone()
        opt.step(Ws, Ms, Gs, sel_out=sel, step=t)
        torch.cuda.synchronize()
        assert opt.status()[0] == 0
        # ---- every matrix: a valid index set, untouched complement (bitwise)
        off = 0
        for i, (m, n) in enumerate(shapes):
            s = sel[i].long()
            d = m if axes[i] == O.AXIS_ROWS else n
            assert s.numel() == ks[i] and int(s.min()) >= 0 and int(s.max()) < d
            assert bool((s[1:] > s[:-1]).all()), i
            unsel = torch.ones(d, dtype=torch.bool, device="cuda")
            unsel[s] = False
            wb = W_before[off:off + m * n].view(m, n)
            mb = M_before[off:off + m * n].view((n, m) if mts[i] else (m, n))
            mb = mb.T if mts[i] else mb
            expect_m = mb + Gs[i]
            if axes[i] == O.AXIS_ROWS:
                assert torch.equal(wb[unsel], Ws[i][unsel]), i
                assert torch.equal(expect_m[unsel], Mv(i)[unsel]), i
            else:
                assert torch.equal(wb[:, unsel], Ws[i][:, unsel]), i
                assert torch.equal(expect_m[:, unsel], Mv(i)[:, unsel]), i
            off += m * n
        del W_before, M_before
        # ---- sampled matrices: the oracle, one by one
        cfg.step = t
        for i in SAMPLE:
            Kg = sel[i].cpu().numpy().astype(np.int64)
            Wsave, Msave = Wr[i].copy(), Mr[i].copy()
            K, _, ax = O.dion2_step(Wr[i], Mr[i], Gc[i], cfg, matrix_id=i)
            if not np.array_equal(K, Kg):
                assert _tie_equivalent(Kg, K, O.l1_scores(Msave + Gc[i], ax)), (i, t)
                ties += 1
                Wr[i], Mr[i] = Wsave, Msave
                O.dion2_step(Wr[i], Mr[i], Gc[i], cfg, force_K=Kg)
    for i in SAMPLE:
        wg = Ws[i].cpu().numpy().astype(np.float64)
        d_ref, d_gpu = Wr[i] - W0[i], wg - W0[i]
        assert np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref) <= 2e-2, i
        mg = Mv(i).cpu().numpy().astype(np.float64)
        assert np.abs(mg - Mr[i]).max() / np.abs(Mr[i]).max() <= 1e-5, i
