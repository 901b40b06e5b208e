"""GPU parity of the FSDP2 integration (-m gpu): `fully_shard(..., shard_placement_fn=
dion2_placement())` + `Dion2FSDP` against the fp64 oracle (paper P:113 / P:272: Dion2 inside
FSDP2).  One GPU: a one-rank NCCL group (FSDP2 and the distributed C-ABI step with P = 1);
the world-2 run is in test_gpu_multirank.py (skipped below 2 GPUs)."""
import os
import socket

import pytest
import torch

from gpu_harness import run_parity_fsdp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture
def nccl_world1():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("mt,direct", [(True, False), (False, False), (True, True)])
def test_fsdp_one_rank(nccl_world1, mt, direct):
    res = run_parity_fsdp([(256, 512), (512, 256), (1024, 1024), (2048, 512), (512, 2048)], 0.25, steps=3,
                          m_transposed=mt, direct=direct)
    assert max(res.dW_rel) <= 2e-2, res
    assert res.exchange == ["direct" if direct else "nccl"], res.exchange


def test_fsdp_training_loop(nccl_world1):
    """forward / backward through the FSDP2 module, then Dion2FSDP.step: only the selected
    rows (rows mode) / columns (column mode) of each weight change, k of them."""
    import torch.distributed as dist
    from torch.distributed.device_mesh import init_device_mesh
    from torch.distributed.fsdp import fully_shard
    from paper_2512_16928_b200.fsdp import Dion2FSDP, dion2_placement, selection_axis
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(512, 2048, bias=False), torch.nn.GELU(),
                                torch.nn.Linear(2048, 512, bias=False)).cuda()
    mesh = init_device_mesh("cuda", (dist.get_world_size(),))
    fully_shard(model, mesh=mesh, shard_placement_fn=dion2_placement())
    ws = [m.weight for m in (model[0], model[2])]
    opt = Dion2FSDP(ws, lr=0.02)
    before = [w.full_tensor().detach().clone() for w in ws]
    x = torch.randn(64, 512, device="cuda")
    model(x).square().mean().backward()
    opt.step()
    for w, b in zip(ws, before):
        d = (w.full_tensor().detach() != b)
        ax = selection_axis(tuple(w.shape))
        changed = d.any(dim=1) if ax == 0 else d.any(dim=0)
        k = round(0.25 * min(w.shape))
        assert int(changed.sum()) == k, (tuple(w.shape), int(changed.sum()), k)
