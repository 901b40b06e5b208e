"""Shared GPU-vs-oracle parity harness (used by the -m gpu tests, smoke() and bench).

Protocol: identical fp32 inputs on both sides (host
NumPy generation, copied to the device; the oracle converts the same fp32
values to fp64 exactly).  Both sides run T steps; index sets must agree
exactly except at legitimate near-ties (|s_i - s_(k)| <= 1e-6 s_(k) with the
oracle's fp64 scores), where the oracle adopts the GPU's set (force_K) so the
trajectories stay aligned.  Weights are compared on the cumulative update
dW = W_T - W_0 (relative Frobenius).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

import oracle as O
from synth import gen_grad, gen_grad_structured, gen_w0
from paper_2512_16928_b200 import Dion2

TIE_REL = 1e-6


@dataclass
class ParityResult:
    dW_rel: List[float] = field(default_factory=list)      # per matrix
    W_rel: List[float] = field(default_factory=list)
    M_rel: List[float] = field(default_factory=list)        # max|dM| / max|M|
    O_rel: List[float] = field(default_factory=list)        # last-step O, relative Frobenius
    ties: int = 0
    index_mismatch: int = 0
    unselected_w_bitwise: bool = True
    unselected_m_bitwise: bool = True


def oracle_cfg(alpha, axis, mu=0.95, lr=0.02, decay_mode=0, scale_mode=0):
    ax = {"rows": O.AXIS_ROWS, "cols": O.AXIS_COLS, "auto": O.AXIS_AUTO}[axis]
    # the library takes alpha/mu/lr as fp32: give the oracle the same values
    return O.OracleConfig(alpha=float(np.float32(alpha)), mu=float(np.float32(mu)), lr=float(np.float32(lr)),
                          axis=ax, decay_mode=decay_mode, scale_mode=scale_mode)


def _tie_equivalent(K_gpu, K_ref, scores):
    if np.array_equal(K_gpu, K_ref):
        return True
    k = len(K_ref)
    skth = np.sort(scores)[::-1][k - 1]
    diff = np.setxor1d(K_gpu, K_ref)
    return bool(np.all(np.abs(scores[diff] - skth) <= TIE_REL * max(skth, 1e-300)))


def run_parity(shapes: Sequence[Tuple[int, int]], alpha: float, axis: str = "auto", precision: str = "bf16",
               steps: int = 10, seed: int = 0, mu: float = 0.95, lr: float = 0.02, row_scaled: bool = False,
               decay_mode: int = 0, check_bitwise: bool = True, device: str = "cuda", select: str = "l1",
               sel_seed: int = 0, m_transposed: bool = False, grad_bf16: bool = False, ns_form: str = "auto",
               ns_coeffs=None, storage_transposed: bool = False, structure: Optional[dict] = None,
               scale_mode: int = 0) -> ParityResult:
    """m_transposed: store M transposed (cols x rows) for every column-mode matrix.
    storage_transposed: W, M, G of every matrix live as (n, m) tensors (JAX / Flax (in, out)
    layout, ABI v5); the comparisons use their logical (m, n) views.
    ns_form: "auto" | "direct" | "gram" (reading R23); ns_coeffs: per-iteration (a, b, c), T = len.
    structure: kwargs of synth.gen_grad_structured (ill-conditioned gradients) instead of N(0, 1).
    scale_mode: 1 = the submatrix scale sqrt(k/n) variant (f3)."""
    res = ParityResult()
    cfg_o = oracle_cfg(alpha, axis, mu, lr, decay_mode, scale_mode)
    cfg_o.select, cfg_o.seed = select, sel_seed
    ns_kw = dict(ns_form=ns_form)
    if ns_coeffs is not None:
        # the library holds the coefficients as fp32: give the oracle the same values
        ns_coeffs = [tuple(float(np.float32(v)) for v in abc) for abc in ns_coeffs]
        cfg_o.ns_coeffs = list(ns_coeffs)
        ns_kw.update(ns_steps=len(ns_coeffs), ns_coeffs=ns_coeffs)
    W0 = [gen_w0(m, n, seed, i) for i, (m, n) in enumerate(shapes)]
    stt = bool(storage_transposed)
    lay = lambda a: a.T.contiguous() if stt else a  # noqa: E731  (logical m x n -> device storage)
    Wg = [lay(torch.from_numpy(w).to(device)) for w in W0]
    Wv = lambda i: Wg[i].T if stt else Wg[i]  # noqa: E731  (the m x n view of W)
    # m_transposed applies to matrices whose STORAGE selection axis is columns (logical rows mode
    # under storage_transposed); "transposed" is relative to W's storage, i.e. the logical layout then
    mts = [m_transposed and ((O.resolve_axis(m, n, cfg_o.axis) == O.AXIS_COLS) != stt) for (m, n) in shapes]
    Mg = [torch.zeros(((n, m) if mt else (m, n)) if not stt else ((m, n) if mt else (n, m)), device=device)
          for (m, n), mt in zip(shapes, mts)]
    Mv = lambda i: Mg[i] if (stt and mts[i]) else (Mg[i].T if (mts[i] or stt) else Mg[i])  # noqa: E731
    Wr = [w.astype(np.float64) for w in W0]
    Mr = [np.zeros((m, n)) for (m, n) in shapes]
    opt = Dion2(alpha=alpha, mu=mu, lr=lr, axis=axis, precision=precision, decay_mode=decay_mode, select=select,
                seed=sel_seed, scale_mode=scale_mode, **ns_kw)
    ks = []
    for (m, n) in shapes:
        ax = O.resolve_axis(m, n, cfg_o.axis)
        ks.append(O.select_count(cfg_o.alpha, m if ax == O.AXIS_ROWS else n))
    for t in range(steps):
        if structure:
            G = [gen_grad_structured(m, n, seed, i, t, **structure) for i, (m, n) in enumerate(shapes)]
        else:
            G = [gen_grad(m, n, seed, i, t, row_scaled=row_scaled) for i, (m, n) in enumerate(shapes)]
        if grad_bf16:  # the oracle sees exactly the bf16 values the kernels read
            Gg = [torch.from_numpy(g).to(device).to(torch.bfloat16) for g in G]
            G = [g.float().cpu().numpy() for g in Gg]
            Gg = [lay(g) for g in Gg]
        else:
            Gg = [lay(torch.from_numpy(g).to(device)) for g in G]
        sel = [torch.empty(k, dtype=torch.int32, device=device) for k in ks]
        Oo = []
        for i, (m, n) in enumerate(shapes):
            ax = O.resolve_axis(m, n, cfg_o.axis)
            oshape = (ks[i], n) if ax == O.AXIS_ROWS else (m, ks[i])
            Oo.append(torch.empty(oshape[::-1] if stt else oshape, device=device))  # storage orientation
        if check_bitwise:
            Wb = [Wv(i).clone() for i in range(len(shapes))]
            Mb = [Mv(i).clone() for i in range(len(shapes))]
        opt.step(Wg, Mg, Gg, sel_out=sel, O_out=Oo, step=t, m_transposed=mts,
                 storage_transposed=[stt] * len(shapes))
        cfg_o.step = t
        torch.cuda.synchronize()
        for i, (m, n) in enumerate(shapes):
            Kg = sel[i].cpu().numpy().astype(np.int64)
            g64 = G[i].astype(np.float64)
            Wsave, Msave = Wr[i].copy(), Mr[i].copy()
            K, Oref, ax = O.dion2_step(Wr[i], Mr[i], g64, cfg_o, matrix_id=i)
            if not np.array_equal(K, Kg) and select == "l1":
                scores = O.l1_scores(Msave + g64, ax)
                if _tie_equivalent(Kg, K, scores):
                    res.ties += 1
                    Wr[i], Mr[i] = Wsave, Msave
                    K, Oref, ax = O.dion2_step(Wr[i], Mr[i], g64, cfg_o, force_K=Kg)
                else:
                    res.index_mismatch += 1
            elif not np.array_equal(K, Kg):
                res.index_mismatch += 1  # random rule: integer-exact, no tie allowance
            if t == steps - 1:
                og = (Oo[i].T if stt else Oo[i]).cpu().numpy().astype(np.float64)
                res.O_rel.append(float(np.linalg.norm(og - Oref) / max(np.linalg.norm(Oref), 1e-300)))
            if check_bitwise:
                # unselected rows/cols: W bit-identical, M == fp32(M_prev + G) bit-identical
                unsel = np.ones(m if ax == O.AXIS_ROWS else n, bool)
                unsel[Kg] = False
                wb, wa = Wb[i].cpu().numpy(), Wv(i).cpu().numpy()
                mb, ma = Mb[i].cpu().numpy(), Mv(i).cpu().numpy()
                expect_m = (mb + G[i]).astype(np.float32)
                if decay_mode == 0:
                    if ax == O.AXIS_ROWS:
                        res.unselected_w_bitwise &= bool(np.array_equal(wb[unsel], wa[unsel]))
                        res.unselected_m_bitwise &= bool(np.array_equal(expect_m[unsel], ma[unsel]))
                    else:
                        res.unselected_w_bitwise &= bool(np.array_equal(wb[:, unsel], wa[:, unsel]))
                        res.unselected_m_bitwise &= bool(np.array_equal(expect_m[:, unsel], ma[:, unsel]))
    _finish(res, shapes, [Wv(i) for i in range(len(shapes))], [Mv(i) for i in range(len(shapes))], Wr, Mr, W0,
            lr, ks)
    return res


def _dw_floor(dref, w0, lr=0.02, k=1):
    """Denominator of the cumulative-update error: ||dW_ref||, floored at 1e-6 ||W_0|| (~16 fp32
    ulps of W) and at 1e-3 lr sqrt(k) (a thousandth of one step's nominal update: O has ~unit
    singular values): the updates of steps with opposite signs can cancel (e.g. a 1 x 1 matrix
    whose Newton-Schulz output is +-0.697 each step), and below those floors the fp32 storage of W
    and the fp16 store of O, not the step, decide the difference."""
    return max(float(np.linalg.norm(dref)), 1e-6 * float(np.linalg.norm(np.asarray(w0, np.float64))),
               1e-3 * abs(lr) * float(np.sqrt(max(k, 1))), 1e-300)


def _finish(res, shapes, Wg, Mg, Wr, Mr, W0, lr=0.02, ks=None):
    for i in range(len(shapes)):
        wg = Wg[i].cpu().numpy().astype(np.float64)
        dref = Wr[i] - W0[i].astype(np.float64)
        dgpu = wg - W0[i].astype(np.float64)
        res.dW_rel.append(float(np.linalg.norm(dgpu - dref) / _dw_floor(dref, W0[i], lr, ks[i] if ks else 1)))
        res.W_rel.append(float(np.linalg.norm(wg - Wr[i]) / np.linalg.norm(Wr[i])))
        mg = Mg[i].cpu().numpy().astype(np.float64)
        res.M_rel.append(float(np.abs(mg - Mr[i]).max() / max(np.abs(Mr[i]).max(), 1e-300)))
    return res


def run_parity_dist(shapes, alpha, world, steps=3, seed=0, mode="loopback", axis="auto", mu=0.95, lr=0.02,
                    row_scaled=True, device="cuda", select="l1", sel_seed=0, m_transposed=False,
                    structure: Optional[dict] = None, direct: bool = False):
    """Distributed step (owner-compute, shards along the non-selection axis) against the
    fp64 oracle on the FULL matrices.  mode = "loopback" (all ranks in this process) or
    "nccl" (world must equal the initialised torch.distributed world; this process is
    one rank and holds only its shards; the full matrices are re-assembled with
    all_gather for the comparison).  direct: pieces pushed / pulled through peer memory
    (DION2_FLAG_DIST_DIRECT) instead of copied / sent."""
    from paper_2512_16928_b200 import dion2 as D
    res = ParityResult()
    cfg_o = oracle_cfg(alpha, axis, mu, lr)
    cfg_o.select, cfg_o.seed = select, sel_seed
    info = D.dist_info(shapes, world, 0, alpha=alpha, axis=axis, mu=mu, lr=lr)
    axes = info["axis"]
    W0 = [gen_w0(m, n, seed, i) for i, (m, n) in enumerate(shapes)]
    Wr = [w.astype(np.float64) for w in W0]
    Mr = [np.zeros((m, n)) for (m, n) in shapes]
    ks = []
    for (m, n) in shapes:
        ax = O.resolve_axis(m, n, cfg_o.axis)
        ks.append(O.select_count(cfg_o.alpha, m if ax == O.AXIS_ROWS else n))
    # transposed local M shards for the column-mode matrices (m_transposed)
    mts = [bool(m_transposed) and axes[i] == 1 for i in range(len(shapes))]
    if mode == "loopback":
        ranks = list(range(world))
        opt = D.Dion2Loopback(shapes, world, alpha=alpha, axis=axis, mu=mu, lr=lr, select=select, seed=sel_seed,
                              m_transposed=mts, dist_direct=direct)
    else:
        import torch.distributed as dist
        ranks = [dist.get_rank()]
        opt = D.Dion2Dist(shapes, alpha=alpha, axis=axis, mu=mu, lr=lr, select=select, seed=sel_seed,
                          m_transposed=mts, dist_direct=direct)
    full = lambda a, i: torch.from_numpy(a)  # noqa: E731
    Wg = {r: [D.shard_of(full(W0[i], i), axes[i], world, r).to(device) for i in range(len(shapes))] for r in ranks}
    Mg = {r: [torch.zeros((w.shape[1], w.shape[0]), device=device) if mts[i] else torch.zeros_like(w)
              for i, w in enumerate(Wg[r])] for r in ranks}
    Mv = {r: [Mg[r][i].T if mts[i] else Mg[r][i] for i in range(len(shapes))] for r in ranks}  # W-layout views

    def assemble(parts_by_rank, i):
        if mode == "loopback":
            blocks = [parts_by_rank[r][i] for r in range(world)]
        else:
            import torch.distributed as dist
            blocks = [torch.empty_like(parts_by_rank[ranks[0]][i]) for _ in range(world)]
            dist.all_gather(blocks, parts_by_rank[ranks[0]][i].contiguous())
        return torch.cat(blocks, dim=1 if axes[i] == 0 else 0)

    for t in range(steps):
        if structure:
            G = [gen_grad_structured(m, n, seed, i, t, **structure) for i, (m, n) in enumerate(shapes)]
        else:
            G = [gen_grad(m, n, seed, i, t, row_scaled=row_scaled) for i, (m, n) in enumerate(shapes)]
        Gg = {r: [D.shard_of(full(G[i], i), axes[i], world, r).to(device) for i in range(len(shapes))] for r in ranks}
        sel = {r: [torch.empty(k, dtype=torch.int32, device=device) for k in ks] for r in ranks}
        if mode == "loopback":
            opt.step([Wg[r] for r in ranks], [Mg[r] for r in ranks], [Gg[r] for r in ranks],
                     sel_out=[sel[r] for r in ranks], step=t)
        else:
            opt.step(Wg[ranks[0]], Mg[ranks[0]], Gg[ranks[0]], sel_out=sel[ranks[0]], step=t)
        cfg_o.step = t
        torch.cuda.synchronize()
        for i in range(len(shapes)):
            Kg = sel[ranks[0]][i].cpu().numpy().astype(np.int64)
            for r in ranks[1:]:  # every rank selects the same set
                if not np.array_equal(sel[r][i].cpu().numpy(), Kg):
                    res.index_mismatch += 1
            g64 = G[i].astype(np.float64)
            Wsave, Msave = Wr[i].copy(), Mr[i].copy()
            K, _, ax = O.dion2_step(Wr[i], Mr[i], g64, cfg_o, matrix_id=i)
            if not np.array_equal(K, Kg) and select != "l1":
                res.index_mismatch += 1
            elif not np.array_equal(K, Kg):
                if _tie_equivalent(Kg, K, O.l1_scores(Msave + g64, ax)):
                    res.ties += 1
                    Wr[i], Mr[i] = Wsave, Msave
                    O.dion2_step(Wr[i], Mr[i], g64, cfg_o, force_K=Kg)
                else:
                    res.index_mismatch += 1
    Wfull = [assemble(Wg, i) for i in range(len(shapes))]
    Mfull = [assemble(Mv, i) for i in range(len(shapes))]
    _finish(res, shapes, Wfull, Mfull, Wr, Mr, W0, lr, ks)
    res.comm_bytes = opt.last_comm_bytes
    res.exchange = opt.exchange_mode() if mode != "loopback" else ("direct" if direct else "copies")
    return res


def run_parity_fsdp(shapes, alpha, steps=3, seed=0, mu=0.95, lr=0.02, m_transposed=True, select="l1",
                    direct=False):
    """The FSDP2 integration (paper_2512_16928_b200.fsdp): one bias-free Linear per (out, in)
    shape, `fully_shard` with `dion2_placement()` on the initialised torch.distributed world,
    gradients set as DTensors in the parameters' placements, `Dion2FSDP.step`, against the
    fp64 oracle on the full matrices (p.full_tensor()).  Index sets are not exposed by the
    optimizer: a near-tie would show as a dW mismatch (gen_grad is row-scaled: none occur)."""
    import torch.distributed as dist
    from torch.distributed.device_mesh import init_device_mesh
    from torch.distributed.fsdp import fully_shard
    from torch.distributed.tensor import distribute_tensor
    from paper_2512_16928_b200.fsdp import Dion2FSDP, dion2_placement
    res = ParityResult()
    cfg_o = oracle_cfg(alpha, "auto", mu, lr)
    cfg_o.select = select
    mesh = init_device_mesh("cuda", (dist.get_world_size(),))
    model = torch.nn.Sequential(*[torch.nn.Linear(n, m, bias=False) for (m, n) in shapes]).cuda()  # never called
    W0 = [gen_w0(m, n, seed, i) for i, (m, n) in enumerate(shapes)]
    with torch.no_grad():
        for lin, w in zip(model, W0):
            lin.weight.copy_(torch.from_numpy(w))
    fully_shard(model, mesh=mesh, shard_placement_fn=dion2_placement(alpha=alpha))
    params = [lin.weight for lin in model]
    opt = Dion2FSDP(params, lr=lr, mu=mu, alpha=alpha, m_transposed=m_transposed, select=select, dist_direct=direct)
    Wr = [w.astype(np.float64) for w in W0]
    Mr = [np.zeros((m, n)) for (m, n) in shapes]
    for t in range(steps):
        G = [gen_grad(m, n, seed, i, t, row_scaled=True) for i, (m, n) in enumerate(shapes)]
        for p, g in zip(params, G):
            p.grad = distribute_tensor(torch.from_numpy(g).cuda(), mesh, p.placements)
        opt.step()
        cfg_o.step = t
        for i in range(len(shapes)):
            O.dion2_step(Wr[i], Mr[i], G[i].astype(np.float64), cfg_o, matrix_id=i)
    torch.cuda.synchronize()
    Wfull = [p.full_tensor().detach() for p in params]
    for i in range(len(shapes)):
        wg = Wfull[i].cpu().numpy().astype(np.float64)
        dref = Wr[i] - W0[i].astype(np.float64)
        res.dW_rel.append(float(np.linalg.norm(wg - W0[i] - dref) / _dw_floor(dref, W0[i], lr)))
        res.W_rel.append(float(np.linalg.norm(wg - Wr[i]) / np.linalg.norm(Wr[i])))
    res.comm_bytes = opt.comm_bytes()
    res.exchange = [e.exchange_mode() for e in opt._engines]
    return res
