"""FSDP2 placement of the owner-compute layout (CPU, world_size 2, gloo).

`fully_shard(..., shard_placement_fn=dion2_placement())` must hand every rank exactly the
shards `dion2_step_batched_dist` reads (the non-selection axis, rows mode ->
column block, column mode -> row block; paper P:113 / P:272 run Dion2 inside FSDP2, P:274
selects along the shorter dimension), for the weights AND for the reduce-scattered
gradients, and `Dion2FSDP` must accept that layout and reject FSDP2's default Shard(0) on
a rows-mode matrix.  The step itself needs a GPU (tests/test_gpu_fsdp.py).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_16928_b200 import _build


@pytest.fixture(scope="module", autouse=True)
def _lib():
    _build.build()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Block(torch.nn.Module):
    """Weights (out, in): 256 x 64 (column mode), 64 x 256 and 128 x 128 (rows mode), plus a
    bias and a norm gain (1-D: FSDP2's default placement, another optimizer's parameters)."""

    def __init__(self):
        super().__init__()
        self.up = torch.nn.Linear(64, 256, bias=False)
        self.down = torch.nn.Linear(256, 64, bias=True)
        self.mix = torch.nn.Linear(64, 128, bias=False)
        self.out = torch.nn.Linear(128, 128, bias=False)
        self.norm = torch.nn.LayerNorm(128)

    def forward(self, x):
        h = self.down(torch.relu(self.up(x)))
        return self.norm(self.out(self.mix(h)))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from torch.distributed.device_mesh import init_device_mesh
        from torch.distributed.fsdp import fully_shard

        from paper_2512_16928_b200 import dion2 as D
        from paper_2512_16928_b200.fsdp import Dion2FSDP, dion2_placement, selection_axis

        torch.manual_seed(0)
        ref = Block()
        model = Block()
        model.load_state_dict(ref.state_dict())
        names = [n for n, p in ref.named_parameters() if p.dim() == 2]
        full_w = {n: p.detach().clone() for n, p in ref.named_parameters()}
        x = torch.randn(8, 64, generator=torch.Generator().manual_seed(1))
        ref(x).square().sum().backward()
        full_g = {n: p.grad.detach().clone() for n, p in ref.named_parameters()}

        mesh = init_device_mesh("cpu", (world,))
        fully_shard(model, mesh=mesh, shard_placement_fn=dion2_placement())
        model(x).square().sum().backward()
        params = dict(model.named_parameters())
        for n in names:
            p = params[n]
            ax = selection_axis(tuple(p.shape))
            assert p.placements[0].dim == (1 if ax == 0 else 0), (n, p.placements)
            inf = D.dist_info([tuple(p.shape)], world, rank)
            loc, gloc = p.to_local(), p.grad.to_local()
            assert tuple(loc.shape) == tuple(inf["shard"][0]) and loc.is_contiguous(), n
            assert torch.equal(loc, D.shard_of(full_w[n], ax, world, rank)), n
            assert tuple(gloc.shape) == tuple(loc.shape) and gloc.is_contiguous(), n
            assert torch.equal(gloc, D.shard_of(full_g[n], ax, world, rank)), n
        # 1-D parameters keep FSDP2's default placement
        assert params["norm.weight"].placements[0].dim == 0
        # the optimizer accepts exactly this layout (host-side checks; the step needs a GPU)
        opt = Dion2FSDP([params[n] for n in names], lr=0.02)
        assert [tuple(s) for s in opt._engines[0].info["shard"]] == [tuple(params[n].to_local().shape)
                                                                      for n in names]
        # FSDP2's default Shard(0) on a rows-mode matrix is not the step's layout
        bad = torch.nn.Linear(128, 64, bias=False)  # W 64 x 128: rows mode
        fully_shard(bad, mesh=mesh)
        try:
            Dion2FSDP(list(bad.parameters()))
            raise AssertionError("Shard(0) of a rows-mode matrix was accepted")
        except ValueError:
            pass
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_fsdp2_placement_is_the_owner_compute_layout():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out == {0: "ok", 1: "ok"}, out


def test_placement_follows_the_shorter_dimension():
    from paper_2512_16928_b200.fsdp import shard_dim
    assert shard_dim((2048, 8192)) == 1   # rows mode (m <= n, R8): column blocks
    assert shard_dim((8192, 2048)) == 0   # column mode: row blocks
    assert shard_dim((2048, 2048)) == 1   # square -> rows mode
    assert shard_dim((8192, 2048), axis="rows") == 1
