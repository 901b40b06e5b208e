"""FSDP2 integration of the owner-compute step (argument marshalling only).

The paper runs Dion2 inside PyTorch FSDP2 (PAPER.md P:15 footnote, §2 "implemented in
PyTorch FSDP2", §4 "the Dion codebase") and selects "the submatrix along the shorter
dimension of the momentum matrix".  The distributed C-ABI step
(`dion2_step_batched_dist`, include/dion2.h "Multi-GPU") takes every matrix sharded along its
NON-selection axis: a rows-mode matrix as column blocks, a column-mode matrix
as row blocks.  FSDP2 holds exactly that layout when it is asked to:

    fully_shard(module, mesh=mesh, shard_placement_fn=dion2_placement())

places rows-mode weights as `Shard(1)` and column-mode weights as `Shard(0)`, so on every
rank `param.to_local()` and `param.grad.to_local()` (reduce-scattered in the same placement)
ARE the shards the step reads and writes in place: no re-layout and no copy.

`Dion2FSDP` is a `torch.optim.Optimizer` over such 2-D parameters.  It keeps this rank's fp32
momentum shards and hands the local tensors of each parameter group to one batched
`Dion2Dist` step (one NCCL exchange for the whole group).  Parameters that are not matrices
(biases, norm gains) belong to another optimizer; the paper's setup (the Dion codebase) uses
AdamW for them.  Every computation runs in libdion2.so; nothing here touches tensor values.
"""
from typing import Callable, Dict, List, Optional

import torch

from .dion2 import Dion2Dist, dist_info

# dist_info()["axis"]: 0 = rows mode (k of the rows selected), 1 = column mode
_PLACEMENT_DIM = {0: 1, 1: 0}


def selection_axis(shape, **cfg_kw) -> int:
    """The axis the step selects along for a matrix of this GLOBAL shape under cfg_kw
    (axis="auto": the shorter dimension, reading R8): 0 = rows mode, 1 = column mode."""
    return int(dist_info([tuple(shape)], 1, 0, **cfg_kw)["axis"][0])


def shard_dim(shape, **cfg_kw) -> int:
    """The tensor dim FSDP2 must shard a (out, in) weight of this shape along: the
    non-selection axis (1 for rows mode, 0 for column mode)."""
    return _PLACEMENT_DIM[selection_axis(shape, **cfg_kw)]


def dion2_placement(**cfg_kw) -> Callable:
    """A `shard_placement_fn` for `torch.distributed.fsdp.fully_shard`: Shard(non-selection
    axis) for 2-D parameters, FSDP2's default (None) for everything else."""
    from torch.distributed.tensor import Shard

    def fn(param):
        if param.dim() != 2:
            return None
        return Shard(shard_dim(tuple(param.shape), **cfg_kw))

    return fn


def _local(t):
    return t.to_local() if hasattr(t, "to_local") else t


class Dion2FSDP(torch.optim.Optimizer):
    """Dion2 over FSDP2-sharded 2-D parameters (DTensors placed by `dion2_placement`), or
    over plain full tensors when the process group has one rank.

    One batched distributed step per parameter group.  lr and mu are read from the group at
    every step (schedulers may change them); alpha is fixed per group at construction (it
    sets k and with it the layout).  All other settings (select, ns_steps, ns_form,
    decay_mode, scale_mode, seed, ...) are passed through to `make_config`; the step counter
    keys random selection (R22).  m_transposed: keep column-mode momentum shards transposed
    (the single-GPU default layout)."""

    def __init__(self, params, lr: float = 0.02, mu: float = 0.95, alpha: float = 0.25, group=None,
                 m_transposed: bool = True, **cfg_kw):
        defaults = dict(lr=lr, mu=mu, alpha=alpha)
        super().__init__(params, defaults)
        self._cfg_kw = dict(cfg_kw)
        self._mt = bool(m_transposed)
        self._engines: List[Dion2Dist] = []
        self._steps = 0
        for g in self.param_groups:
            shapes, mts, pg = [], [], group
            for p in g["params"]:
                if p.dim() != 2:
                    raise ValueError("Dion2FSDP takes 2-D weight matrices only (give biases / norms to another "
                                     "optimizer)")
                shape = tuple(p.shape)  # a DTensor reports its GLOBAL shape
                ax = selection_axis(shape, alpha=g["alpha"], **cfg_kw)
                if hasattr(p, "placements"):
                    mesh = p.device_mesh
                    if mesh.ndim != 1:
                        raise ValueError("Dion2FSDP supports a 1-D FSDP mesh")
                    want = _PLACEMENT_DIM[ax]
                    pl = p.placements[0]
                    if not (pl.is_shard() and pl.dim == want):
                        raise ValueError(f"parameter of shape {shape} is placed {pl}; the step needs Shard({want}) "
                                         "(fully_shard(..., shard_placement_fn=dion2_placement()))")
                    mg = mesh.get_group()
                    if pg is None:
                        pg = mg
                    elif pg is not mg:
                        raise ValueError("all parameters of a group must share one FSDP mesh")
                shapes.append(shape)
                mts.append(self._mt and ax == 1)
            eng = Dion2Dist(shapes, group=pg, m_transposed=mts, alpha=g["alpha"], mu=g["mu"], lr=g["lr"],
                            **cfg_kw)
            for p, want in zip(g["params"], eng.info["shard"]):
                loc = _local(p.detach())
                if tuple(loc.shape) != tuple(want):
                    raise ValueError(f"local shard {tuple(loc.shape)} of a {tuple(p.shape)} parameter differs from "
                                     f"the step's layout {tuple(want)} (the sharded dim must divide by the world size)")
                if not loc.is_contiguous():
                    raise ValueError("local shards must be contiguous")
            self._engines.append(eng)

    def _momentum(self, p, transposed: bool) -> torch.Tensor:
        st: Dict = self.state[p]
        if "M" not in st:
            loc = _local(p.detach())
            shp = (loc.shape[1], loc.shape[0]) if transposed else tuple(loc.shape)
            st["M"] = torch.zeros(shp, dtype=torch.float32, device=loc.device)
        return st["M"]

    @torch.no_grad()
    def step(self, closure: Optional[Callable] = None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        for g, eng in zip(self.param_groups, self._engines):
            ps = g["params"]
            if any(p.grad is None for p in ps):
                raise ValueError("every parameter of a Dion2FSDP group needs a gradient (one batched step per group)")
            Ws = [_local(p) for p in ps]
            Gs = [_local(p.grad) for p in ps]
            Ms = [self._momentum(p, mt) for p, mt in zip(ps, eng.m_transposed)]
            eng.step(Ws, Ms, Gs, lr=g["lr"], mu=g["mu"], step=self._steps)
        self._steps += 1
        return loss

    def comm_bytes(self) -> int:
        """Bytes this rank sent in the last step (all groups)."""
        return sum(e.last_comm_bytes for e in self._engines)
