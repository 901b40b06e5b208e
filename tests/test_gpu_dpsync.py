"""Compressed DP-sync on the GPU (-m gpu): replicas with local gradients, only M[K] averaged
(paper 3.2).  Checked against the oracle's replica model, which is itself pinned
(test_oracle_pins.py) to equal full gradient synchronisation."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
from synth import gen_grad, gen_w0
from paper_2512_16928_b200 import Dion2Error
from paper_2512_16928_b200 import dion2 as D

pytestmark = pytest.mark.gpu

SHAPES = [(256, 512), (512, 256), (384, 640), (1024, 512)]


def _run(world, precision, tol, steps=3, mode="loopback", m_transposed=False, direct=False, keep=None):
    """m_transposed: column-mode matrices keep M transposed (cols, rows) on every replica.
    direct: the peer-memory reduce (DION2_FLAG_DIST_DIRECT).  keep: a dict receiving W and M."""
    seed, alpha = 21, 0.25
    W0 = [gen_w0(m, n, 0, i) for i, (m, n) in enumerate(SHAPES)]
    reps = world if mode == "loopback" else 1
    mts = [m_transposed and m > n for (m, n) in SHAPES]
    Wg = [[torch.from_numpy(w).cuda() for w in W0] for _ in range(reps)]
    Mg = [[torch.zeros((n, m) if mt else (m, n), device="cuda") for (m, n), mt in zip(SHAPES, mts)]
          for _ in range(reps)]
    Wr = [[w.astype(np.float64) for w in W0] for _ in range(world)]
    Mr = [[np.zeros((m, n)) for (m, n) in SHAPES] for _ in range(world)]
    opt = D.Dion2DpSync(loopback_world=world if mode == "loopback" else 0, alpha=alpha, precision=precision,
                        seed=seed, m_transposed=mts, dist_direct=direct)
    for t in range(steps):
        G = [[gen_grad(m, n, 100 + r, i, t) for i, (m, n) in enumerate(SHAPES)] for r in range(world)]
        if mode == "loopback":
            opt.step(Wg, Mg, [[torch.from_numpy(g).cuda() for g in G[r]] for r in range(world)], step=t)
        else:
            import torch.distributed as dist
            me = dist.get_rank()  # this process is replica `me`: its own local gradient
            opt.step(Wg[0], Mg[0], [torch.from_numpy(g).cuda() for g in G[me]], step=t)
        cfg = O.OracleConfig(alpha=float(np.float32(alpha)), select="random", seed=seed, step=t)
        for i in range(len(SHAPES)):
            O.dion2_step_dpsync([Wr[r][i] for r in range(world)], [Mr[r][i] for r in range(world)],
                                [G[r][i].astype(np.float64) for r in range(world)], cfg, matrix_id=i)
    torch.cuda.synchronize()
    for i in range(len(SHAPES)):
        w0 = W0[i].astype(np.float64)
        for r in range(reps):
            assert torch.equal(Wg[r][i], Wg[0][i])          # replicas stay bit-identical
            wg = Wg[r][i].cpu().double().numpy()
            err = np.linalg.norm((wg - w0) - (Wr[r][i] - w0)) / np.linalg.norm(Wr[r][i] - w0)
            assert err <= tol, (i, r, err)
            rr = r if mode == "loopback" else __import__("torch.distributed").distributed.get_rank()
            mg = (Mg[r][i].T if mts[i] else Mg[r][i]).cpu().double().numpy()
            assert np.abs(mg - Mr[rr][i]).max() <= 1e-5 * np.abs(Mr[rr][i]).max()
    if keep is not None:
        keep["W"], keep["M"] = Wg, Mg
    return opt


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("precision,tol", [("bf16", 2e-2), ("fp32", 1e-5)])
def test_dpsync_loopback(world, precision, tol):
    opt = _run(world, precision, tol)
    k_o = sum(O.selected_bytes(m, n, 0.25, O.AXIS_AUTO, 4) for (m, n) in SHAPES)
    # ~alpha of full gradient sync: the selected fp32 rows plus two floats per matrix (the
    # largest score and the non-finite flag, combined so every replica takes the same decision)
    assert opt.last_comm_bytes == int(2.0 * (world - 1) / world * (k_o + 8 * len(SHAPES)))


@pytest.mark.parametrize("world", [2, 3])
def test_dpsync_loopback_transposed_momentum(world):
    _run(world, "bf16", 2e-2, m_transposed=True)


def test_dpsync_nccl_single_rank():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(s.getsockname()[1])
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        _run(1, "bf16", 2e-2, mode="nccl")
    finally:
        dist.destroy_process_group()


def test_dpsync_requires_random_selection():
    mk = lambda: [[torch.zeros(64, 64, device="cuda")] for _ in range(2)]  # noqa: E731
    opt = D.Dion2DpSync(loopback_world=2, select="l1")
    with pytest.raises(Dion2Error):
        opt.step(mk(), mk(), mk())


def test_dpsync_nonfinite_on_one_replica_skips_the_matrix_everywhere():
    """a non-finite gradient on ONE replica must not poison the others.  The replicas
    combine their non-finite flags with the all-reduce, so every replica skips that matrix (W
    unchanged, its selected momentum not overwritten with NaN rows) and reports it, and the
    replicas' W stay bit-identical."""
    world = 2
    W0 = [gen_w0(m, n, 0, i) for i, (m, n) in enumerate(SHAPES)]
    Wg = [[torch.from_numpy(w).cuda() for w in W0] for _ in range(world)]
    Mg = [[torch.zeros(m, n, device="cuda") for (m, n) in SHAPES] for _ in range(world)]
    G = [[torch.from_numpy(gen_grad(m, n, 100 + r, i, 0)).cuda() for i, (m, n) in enumerate(SHAPES)]
         for r in range(world)]
    G[1][2][3, 5] = float("nan")  # replica 1, matrix 2
    opt = D.Dion2DpSync(loopback_world=world, alpha=0.25, seed=3)
    opt.step(Wg, Mg, G, step=0)
    torch.cuda.synchronize()
    for r in range(world):
        assert opt.status(r) == (7, 2), (r, opt.status(r))
        assert torch.equal(Wg[r][2], Wg[0][2]) and torch.equal(Wg[r][2].cpu(), torch.from_numpy(W0[2]))
        assert torch.isfinite(Mg[0][2]).all()
        for i in (0, 1, 3):
            assert torch.equal(Wg[r][i], Wg[0][i]) and not torch.equal(Wg[r][i].cpu(), torch.from_numpy(W0[i]))


# ------------------------------------------------------------- direct peer-memory reduce
@pytest.mark.parametrize("world", [2, 3, 8])
def test_dpsync_loopback_direct_is_bitwise_the_allreduce(world):
    """DION2_FLAG_DIST_DIRECT: every replica reduces its slice of the packed buffer over all
    replicas' buffers (rank order) and writes it into every buffer -- the same sums, so W and M
    are bit-identical to the all-reduce emulation's, with the same byte count."""
    a, b = {}, {}
    o1 = _run(world, "bf16", 2e-2, keep=a)
    o2 = _run(world, "bf16", 2e-2, direct=True, keep=b)
    assert o1.last_comm_bytes == o2.last_comm_bytes
    for r in range(world):
        for i in range(len(SHAPES)):
            assert torch.equal(a["W"][r][i], b["W"][r][i]) and torch.equal(a["M"][r][i], b["M"][r][i]), (r, i)


def test_dpsync_nccl_single_rank_direct():
    """The symmetric-window path with a one-rank group: pack into the window, LSA barrier, the
    reduce kernel through the peer pointers, barrier, unpack from the output window."""
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(s.getsockname()[1])
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        opt = _run(1, "bf16", 2e-2, mode="nccl", direct=True)
        assert opt.exchange_mode() == "direct"
        del opt
        _run(1, "fp32", 1e-5, mode="nccl", direct=True)
        _run(1, "bf16", 2e-2, mode="nccl", direct=True, m_transposed=True)
    finally:
        dist.destroy_process_group()
