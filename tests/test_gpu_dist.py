"""GPU tests of the owner-compute distributed step (-m gpu).

One GPU is available: the multi-rank layout is exercised in loopback mode (all P
ranks in one process on one device, exchanges as device copies: the same kernels,
the same tables, the same piece offsets as the NCCL path), and the NCCL transport
itself with a single-rank NCCL process group (self send/recv and all-gather).
"""
import os
import socket

import numpy as np
import pytest
import torch

from synth import layer_set_1b

from gpu_harness import run_parity_dist

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _assert(res, tol=BF16_TOL):
    assert res.index_mismatch == 0, res
    assert max(res.dW_rel) <= tol, res
    assert max(res.M_rel) <= 1e-5, res


SHAPES = [(256, 512), (512, 256), (1024, 1024), (2048, 512), (512, 2048)]


@pytest.mark.parametrize("world", [1, 2, 4])
def test_loopback_parity(world):
    _assert(run_parity_dist(SHAPES, 0.25, world, steps=3))


@pytest.mark.parametrize("world", [1, 2, 4])
def test_loopback_transposed_momentum(world):
    """Column-mode matrices with their local M shards stored transposed (K1 transpose-add,
    row gather of M^T into the pieces; the exchanged pieces are unchanged)."""
    _assert(run_parity_dist(SHAPES + [(1024, 256), (4096, 1024)], 0.25, world, steps=3, m_transposed=True))


@pytest.mark.parametrize("world", [2, 8])
def test_loopback_1b_layer_transposed_momentum(world):
    _assert(run_parity_dist(layer_set_1b(1), 0.25, world, steps=2, m_transposed=True))


@pytest.mark.parametrize("world", [2, 8])
def test_loopback_one_layer_of_the_1b_set(world):
    _assert(run_parity_dist(layer_set_1b(1), 0.25, world, steps=2))


def test_loopback_8_ranks_one_layer_of_the_8b_set():
    """BASELINE configs[3] shapes on 8 (loopback) ranks."""
    from synth import layer_set_8b
    _assert(run_parity_dist(layer_set_8b(1), 0.25, 8, steps=1))


def test_loopback_8_ranks_stress_shapes():
    """BASELINE configs[4]: 4096 x 32768 and 28672 x 8192 at alpha = 0.0625 on 8 (loopback) ranks."""
    _assert(run_parity_dist([(4096, 32768), (28672, 8192)], 0.0625, 8, steps=1))


def test_loopback_random_selection():
    _assert(run_parity_dist(SHAPES, 0.25, 4, steps=3, select="random", sel_seed=99))


def test_loopback_alpha1_is_full_muon():
    _assert(run_parity_dist([(256, 512), (512, 256)], 1.0, 2, steps=2))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_transport_single_rank():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        res = run_parity_dist(SHAPES, 0.25, 1, steps=3, mode="nccl")
        _assert(res)
        _assert(run_parity_dist(SHAPES + [(1024, 256)], 0.25, 1, steps=2, mode="nccl", m_transposed=True))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks,world", [("2", 2), ("3", 4)])
def test_loopback_owner_chunks(chunks, world, monkeypatch):
    """DION2_DIST_CHUNKS: owner chunks whose exchanges (C2 / C3) run on a side stream and overlap
    the NS of the neighbouring chunk; sections ordered by chunk, in-place pieces per chunk."""
    monkeypatch.setenv("DION2_DIST_CHUNKS", chunks)
    _assert(run_parity_dist(SHAPES + [(1024, 256), (4096, 1024)], 0.25, world, steps=3, m_transposed=True))
    _assert(run_parity_dist(layer_set_1b(1), 0.25, world, steps=2))


# ------------------------------------------------------------- direct peer exchange
@pytest.mark.parametrize("world", [2, 4, 8])
def test_loopback_direct_exchange(world):
    """DION2_FLAG_DIST_DIRECT in loopback: K3 pushes the pieces into the owners' receive
    buffers and K7 pulls O from the owners' outgoing buffers (no exchange copies)."""
    _assert(run_parity_dist(SHAPES + [(1024, 256), (4096, 1024)], 0.25, world, steps=3, direct=True,
                            m_transposed=True))
    _assert(run_parity_dist(layer_set_1b(1), 0.25, world, steps=2, direct=True))


def test_loopback_direct_three_ranks():
    """A rank count that is not a power of two (o / P a multiple of 8 but not of 64: the owner's
    pieces are assembled by copies, pushed and pulled directly)."""
    _assert(run_parity_dist([(384, 768), (768, 384), (1536, 1536), (480, 1920)], 0.25, 3, steps=3, direct=True))


@pytest.mark.parametrize("world", [2, 8])
def test_loopback_direct_is_bitwise_the_copy_exchange(world):
    """Same kernels, same bytes, other addresses: W, M and the index sets after 3 steps are
    bit-identical with and without the direct exchange."""
    from paper_2512_16928_b200 import dion2 as D
    from synth import gen_grad, gen_w0
    shapes = SHAPES + layer_set_1b(1)
    infos = D.dist_info(shapes, world, 0)
    axes = infos["axis"]
    out = {}
    for direct in (False, True):
        opt = D.Dion2Loopback(shapes, world, alpha=0.25, dist_direct=direct)
        W = [[D.shard_of(torch.from_numpy(gen_w0(m, n, 0, i)), axes[i], world, r).cuda()
              for i, (m, n) in enumerate(shapes)] for r in range(world)]
        M = [[torch.zeros_like(w) for w in W[r]] for r in range(world)]
        for t in range(3):
            G = [[D.shard_of(torch.from_numpy(gen_grad(m, n, 0, i, t, row_scaled=True)), axes[i], world, r).cuda()
                  for i, (m, n) in enumerate(shapes)] for r in range(world)]
            opt.step(W, M, G, step=t)
        torch.cuda.synchronize()
        out[direct] = (W, M, opt.last_comm_bytes)
    for r in range(world):
        for i in range(len(shapes)):
            assert torch.equal(out[False][0][r][i], out[True][0][r][i]), (r, i)
            assert torch.equal(out[False][1][r][i], out[True][1][r][i]), (r, i)
    assert out[False][2] == out[True][2]


def test_nccl_direct_single_rank():
    """The NCCL symmetric-memory path with one rank: ncclMemAlloc'd windows registered
    symmetrically, a device communicator with an LSA barrier, peer pointers read on the device,
    K3 storing into / K7 loading from the (own) window through them, barriers between phases."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        res = run_parity_dist(SHAPES, 0.25, 1, steps=3, mode="nccl", direct=True)
        _assert(res)
        assert res.exchange == "direct", res.exchange  # the symmetric windows were set up, no fallback
        _assert(run_parity_dist(SHAPES + [(1024, 256)], 0.25, 1, steps=2, mode="nccl", m_transposed=True,
                                direct=True))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_loopback_bf16_state_direct_and_copy(world):
    """bf16 W and bf16 G through the distributed step (the sparse update rounds W once, the
    K1 reads bf16 gradients): the direct and the copy exchange give bit-identical W and M,
    and the cumulative update matches the single-GPU step on the same bf16 inputs within the
    NS tolerance."""
    from paper_2512_16928_b200 import Dion2
    from paper_2512_16928_b200 import dion2 as D
    from synth import gen_grad, gen_w0
    shapes = [(512, 1024), (1024, 512), (1024, 1024), (2048, 512)]
    axes = D.dist_info(shapes, world, 0)["axis"]
    W0 = [torch.from_numpy(gen_w0(m, n, 3, i)).to(torch.bfloat16) for i, (m, n) in enumerate(shapes)]
    Gs = [[torch.from_numpy(gen_grad(m, n, 3, i, t, row_scaled=True)).to(torch.bfloat16)
           for i, (m, n) in enumerate(shapes)] for t in range(3)]
    out = {}
    for direct in (False, True):
        opt = D.Dion2Loopback(shapes, world, alpha=0.25, dist_direct=direct)
        W = [[D.shard_of(W0[i], axes[i], world, r).cuda() for i in range(len(shapes))] for r in range(world)]
        M = [[torch.zeros(w.shape, device="cuda") for w in W[r]] for r in range(world)]
        for t in range(3):
            G = [[D.shard_of(Gs[t][i], axes[i], world, r).cuda() for i in range(len(shapes))] for r in range(world)]
            opt.step(W, M, G, step=t)
        torch.cuda.synchronize()
        out[direct] = (W, M)
    for r in range(world):
        for i in range(len(shapes)):
            assert torch.equal(out[False][0][r][i], out[True][0][r][i]), (r, i)
            assert torch.equal(out[False][1][r][i], out[True][1][r][i]), (r, i)
    # single-GPU reference on the same bf16 inputs
    single = Dion2(alpha=0.25)
    Ws = [w.clone().cuda() for w in W0]
    Ms = [torch.zeros(w.shape, device="cuda") for w in W0]
    for t in range(3):
        single.step(Ws, Ms, [g.cuda() for g in Gs[t]])
    torch.cuda.synchronize()
    for i in range(len(shapes)):
        Wd = torch.cat([out[True][0][r][i] for r in range(world)], dim=1 if axes[i] == 0 else 0).float()
        d_dist = (Wd - W0[i].cuda().float())
        d_single = (Ws[i].float() - W0[i].cuda().float())
        rel = (torch.linalg.norm(d_dist - d_single) / torch.linalg.norm(d_single)).item()
        assert rel <= 2e-2, (i, rel)


@pytest.mark.parametrize("direct", [False, True])
def test_nccl_graph_replay_is_bitwise_eager(direct):
    """Dion2Dist(cuda_graph=True): the step captured on its second identical call (NCCL calls or
    the direct-exchange barriers inside the graph) and replayed gives bit-identical W and M to
    the eager step, also when eta changes between replays (read on the device)."""
    import torch.distributed as dist
    from paper_2512_16928_b200 import dion2 as D
    from synth import gen_grad, gen_w0
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        shapes = SHAPES + [(1024, 256)]
        out = []
        for graph in (False, True):
            opt = D.Dion2Dist(shapes, alpha=0.25, dist_direct=direct, cuda_graph=graph)
            W = [torch.from_numpy(gen_w0(m, n, 4, i)).cuda() for i, (m, n) in enumerate(shapes)]
            M = [torch.zeros(m, n, device="cuda") for (m, n) in shapes]
            G = [torch.empty(m, n, device="cuda") for (m, n) in shapes]
            for t in range(5):
                for i, (m, n) in enumerate(shapes):
                    G[i].copy_(torch.from_numpy(gen_grad(m, n, 4, i, t, row_scaled=True)))
                opt.step(W, M, G, lr=0.02 * (1.0 - 0.1 * t))
            torch.cuda.synchronize()
            if graph:
                assert opt._graph is not None  # steps 3..5 replayed
            out.append((W, M))
            opt.release()
        for i in range(len(shapes)):
            assert torch.equal(out[0][0][i], out[1][0][i]), i
            assert torch.equal(out[0][1][i], out[1][1][i]), i
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,direct", [(2, False), (3, False), (4, True), (8, False)])
def test_short_x_exact_in_the_distributed_step(world, direct):
    """Short X (k <= 128, reading R25) in the distributed step: no pieces; every rank sums the
    partial Gram matrices of its column block (all-reduce) and applies the exact NS locally --
    within the final fp16 store of the oracle on extreme spikes, next to ordinary matrices."""
    u = 8 * world
    shapes = [(3 * u, 75 * u), (117 * u, 3 * u), (72 * u, 96 * u), (24 * u, 120 * u)]
    res = run_parity_dist(shapes, 0.5, world, steps=2, direct=direct,
                          structure=dict(kind="spike", rank=4, ratio=250))
    assert res.index_mismatch == 0 and max(res.M_rel) <= 1e-5, res
    short = [i for i, (m, n) in enumerate(shapes) if round(0.5 * min(m, n)) <= 128]
    assert short and max(res.dW_rel[i] for i in short) <= 2e-3, res
    assert max(res.dW_rel) <= BF16_TOL, res


@pytest.mark.parametrize("shapes,world", [([(576, 912), (24, 600), (696, 456), (672, 792)], 3),
                                          ([(120, 792), (936, 816), (936, 720), (936, 24)], 3)])
def test_fuzz_cases_short_x_distributed(shapes, world):
    """The two fuzz cases (profiles/r02_fuzz_100000.jsonl) that reached 2.2% before the
    distributed short-X path."""
    res = run_parity_dist(shapes, 0.5, world, steps=2, structure=dict(kind="spike", rank=4, ratio=250))
    assert res.index_mismatch == 0 and max(res.dW_rel) <= BF16_TOL and max(res.M_rel) <= 1e-5, res
