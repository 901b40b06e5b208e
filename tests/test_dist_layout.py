"""Host-side logic of the owner-compute distributed step (-m "not gpu").

dion2_dist_info (C ABI, host only) decides the selection axis, the shard of every
matrix, its owner (LPT on NS FLOPs) and the per-peer byte counts of the exchange.
These tests check that every rank derives the same plan, that the two sides of
every exchange agree, that the exchanged volume scales with alpha, and -- in a
world_size-2 gloo process group -- that pieces laid out by those counts and
displacements reassemble into exactly the selected submatrix the oracle gathers.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2512_16928_b200 import _build
from paper_2512_16928_b200 import dion2 as D
from synth import gen_grad, layer_set_1b

SHAPES = [(256, 512), (512, 256), (1024, 1024), (2048, 512), (512, 2048)] + layer_set_1b(2)


@pytest.fixture(scope="module", autouse=True)
def _lib():
    _build.build()


TINY_K = 128  # short X (k <= 128, reading R25): summed partial Gram matrices, no pieces


def _piece_bytes(m, n, alpha, world):
    ax = O.resolve_axis(m, n, O.AXIS_AUTO)
    d, o = (m, n) if ax == O.AXIS_ROWS else (n, m)
    k = O.select_count(np.float32(alpha), d)
    raw = 0 if k <= TINY_K else k * (o // world) * 2
    return -(-raw // 256) * 256, k, o


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_every_rank_derives_the_same_plan(world):
    infos = [D.dist_info(SHAPES, world, r, alpha=0.25) for r in range(world)]
    for inf in infos[1:]:
        assert inf["axis"] == infos[0]["axis"] and inf["owner"] == infos[0]["owner"]
    for r in range(world):
        for o in range(world):
            # rank r sends to owner o exactly what o expects from r
            assert infos[r]["send_bytes"][o] == infos[o]["recv_bytes"][r]
    for i, (m, n) in enumerate(SHAPES):
        ax = infos[0]["axis"][i]
        assert infos[0]["shard"][i] == ((m, n // world) if ax == 0 else (m // world, n))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_owner_balance_is_lpt(world):
    inf = D.dist_info(SHAPES, world, 0, alpha=0.25)
    flops = []
    for (m, n) in SHAPES:
        _, k, o = _piece_bytes(m, n, 0.25, world)
        flops.append(5 * (4.0 * k * k * o + 2.0 * k ** 3))
    load = [0.0] * world
    for f, ow in zip(flops, inf["owner"]):
        load[ow] += f
    assert max(load) - min(load) <= max(flops) + 1e-6


@pytest.mark.parametrize("world", [2, 8])
def test_volume_scales_with_alpha(world):
    def total(alpha):
        inf = D.dist_info(SHAPES, world, 0, alpha=alpha)
        return sum(inf["send_bytes"])
    t25, t1 = total(0.25), total(1.0)
    assert 0.2 < t25 / t1 < 0.3
    # the analytic per-matrix piece size (k x o/P bf16) is what the plan moves
    expect = sum(_piece_bytes(m, n, 0.25, world)[0] for (m, n) in SHAPES)
    assert t25 == expect


@pytest.mark.parametrize("world", [1, 2, 8])
def test_transposed_momentum_shards_leave_the_exchange_unchanged(world):
    """ABI v4 dion2_shard.m_transposed is local to a rank: axis, owners and every byte count
    of the exchange are identical with and without it."""
    base = D.dist_info(SHAPES, world, 0, alpha=0.25)
    mts = [ax == 1 for ax in base["axis"]]
    assert any(mts)
    for r in range(world):
        a = D.dist_info(SHAPES, world, r, alpha=0.25)
        b = D.dist_info(SHAPES, world, r, alpha=0.25, m_transposed=mts)
        for key in ("axis", "owner", "shard", "send_bytes", "recv_bytes"):
            assert a[key] == b[key], key
        assert b["workspace_bytes"] > 0


def test_transposed_momentum_shard_validation():
    # rows-mode matrices cannot take a transposed momentum shard
    with pytest.raises(D.Dion2Error) as e:
        D.dist_info([(256, 512)], 2, 0, alpha=0.25, m_transposed=[True])
    assert e.value.code == 4  # DION2_EUNSUPPORTED
    arr = D._shards([(512, 256)], m_transposed=[True])
    arr[0].reserved = 1
    cfg = D.make_config(alpha=0.25)
    import ctypes
    n = 1
    ax, own = (ctypes.c_int32 * n)(), (ctypes.c_int32 * n)()
    sr, sc = (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
    sb, rb = (ctypes.c_int64 * 2)(), (ctypes.c_int64 * 2)()
    ws = ctypes.c_size_t(0)
    rc = D._lib().dion2_dist_info(arr, n, ctypes.byref(cfg), 2, 0, ax, own, sr, sc, sb, rb, ctypes.byref(ws))
    assert rc == 2  # DION2_EINVAL_SHAPE: reserved must be 0


def test_unsupported_layouts_are_rejected():
    with pytest.raises(D.Dion2Error):
        D.dist_info([(100, 300)], 3, 0, alpha=0.25)     # 300 / 3 = 100 columns: not a multiple of 8
    with pytest.raises(D.Dion2Error):
        D.dist_info([(1000, 10)], 2, 0, alpha=0.5)       # cols mode, 500-row shards: not a multiple of 8
    with pytest.raises(D.Dion2Error):
        D.dist_info([(1024, 1000)], 3, 0, alpha=0.5)     # 1000 columns do not split over 3 ranks
    D.dist_info([(8192, 4096)], 2, 0, alpha=0.5)         # cols mode, k = 2048 > 1024: generic tiles, supported


# ------------------------------------------------------------------ world_size 2, gloo
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        alpha = 0.25
        inf = D.dist_info(SHAPES, world, rank, alpha=alpha)
        # every process derives the same plan
        allinf = [None] * world
        dist.all_gather_object(allinf, {"owner": inf["owner"], "axis": inf["axis"]})
        assert all(a == allinf[0] for a in allinf)
        # each rank builds its send buffer: for owner o, its column block of X_j for every
        # j owned by o (matrix order), each piece padded to 256 B -- the layout the CUDA
        # pack kernels write into and the NCCL exchange moves
        fullX, send = {}, []
        for o in range(world):
            for j, (m, n) in enumerate(SHAPES):
                if inf["owner"][j] != o or _piece_bytes(m, n, alpha, world)[0] == 0:
                    continue
                M = gen_grad(m, n, 7, j, 0).astype(np.float64)
                ax = O.resolve_axis(m, n, O.AXIS_AUTO)
                s = O.l1_scores(M, ax)
                K = O.select_l1(s, O.select_count(np.float32(alpha), len(s)))
                X = M[K, :] if ax == O.AXIS_ROWS else M[:, K].T          # wide orientation, k x o
                fullX[j] = X
                qo = X.shape[1] // world
                piece = torch.from_numpy(X[:, rank * qo:(rank + 1) * qo].astype(np.float32)).to(torch.bfloat16)
                raw = piece.contiguous().view(torch.uint8).reshape(-1)
                pad = (-raw.numel()) % 256
                send.append(torch.cat([raw, torch.zeros(pad, dtype=torch.uint8)]))
        send = torch.cat(send) if send else torch.zeros(0, dtype=torch.uint8)
        assert send.numel() == sum(inf["send_bytes"])
        recv = torch.empty(sum(inf["recv_bytes"]), dtype=torch.uint8)
        dist.all_to_all_single(recv, send, inf["recv_bytes"], inf["send_bytes"])
        # the owner reassembles X_j = [piece_0 | piece_1 | ...] from the rank sections
        R = inf["recv_bytes"][0]
        off = 0
        for j, (m, n) in enumerate(SHAPES):
            if inf["owner"][j] != rank or j not in fullX:
                continue
            X = fullX[j]
            k, o = X.shape
            qo = o // world
            nb = k * qo * 2
            blocks = []
            for r in range(world):
                b = recv[r * R + off: r * R + off + nb].view(torch.bfloat16).reshape(k, qo)
                blocks.append(b.float().numpy())
            got = np.concatenate(blocks, axis=1)
            want = torch.from_numpy(X.astype(np.float32)).to(torch.bfloat16).float().numpy()
            assert np.array_equal(got, want), j
            off += nb + ((-nb) % 256)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_reassembles_the_selected_submatrix():
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
