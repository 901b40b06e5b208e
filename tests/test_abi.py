"""C-ABI library checks that need no GPU (-m "not gpu").

The library loads, exports every function include/dion2.h declares, and its
host-side logic (config defaults, validation, workspace sizing) behaves as
the header documents.  No compute call is made here.
"""
import ctypes
import os
import re

import pytest

from paper_2512_16928_b200 import _build
from paper_2512_16928_b200 import dion2 as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return D._lib()


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "dion2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dion2_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(D.EXPORTED)


def test_abi_version(lib):
    assert lib.dion2_abi_version() == 7


def test_config_defaults(lib):
    cfg = D.Dion2Config()
    assert lib.dion2_config_init(ctypes.byref(cfg)) == 0
    assert abs(cfg.alpha - 0.25) < 1e-7 and abs(cfg.mu - 0.95) < 1e-7 and abs(cfg.lr - 0.02) < 1e-7
    assert cfg.ns_steps == 5 and abs(cfg.ns_eps - 1e-7) < 1e-12
    assert [round(x, 4) for x in cfg.ns_coeffs[0]] == [3.4445, -4.775, 2.0315]
    assert cfg.axis == 2 and cfg.precision == 0 and cfg.decay_mode == 0
    assert cfg.ns_form == 0 and cfg.reserved0 == 0


@pytest.mark.parametrize("form,reserved", [(3, 0), (-1, 0), (0, 4), (0, 5), (0, 8)])
def test_ns_form_validation(lib, form, reserved):
    cfg = D.make_config()
    cfg.ns_form, cfg.reserved0 = form, reserved
    out = ctypes.c_size_t(0)
    assert lib.dion2_workspace_size(_mats([(64, 64)]), 1, ctypes.byref(cfg), ctypes.byref(out)) == 1  # DION2_EINVAL_CONFIG


def test_lr_device_flag_is_valid(lib):
    """reserved0 bit 0 = DION2_FLAG_LR_DEVICE (eta read from the workspace word); other bits reserved."""
    cfg = D.make_config(lr_device=True)
    assert cfg.reserved0 == 1
    out = ctypes.c_size_t(0)
    assert lib.dion2_workspace_size(_mats([(64, 64)]), 1, ctypes.byref(cfg), ctypes.byref(out)) == 0


def test_gram_form_workspace(lib):
    # Gram-space NS (reading R23) needs three extra p x p buffers per shape group; AUTO picks
    # it for q >= 2p only, FP32 precision never uses it
    wide, square = [(2048, 8192)], [(2048, 2048)]
    _, auto_w = _size(lib, wide)
    _, direct_w = _size(lib, wide, ns_form="direct")
    _, gram_w = _size(lib, wide, ns_form="gram")
    assert auto_w == gram_w and gram_w - direct_w >= 3 * 512 * 512 * 2
    _, auto_s = _size(lib, square, alpha=1.0)
    _, direct_s = _size(lib, square, alpha=1.0, ns_form="direct")
    assert auto_s == direct_s
    _, f32_d = _size(lib, wide, precision="fp32", ns_form="direct")
    _, f32_g = _size(lib, wide, precision="fp32", ns_form="gram")
    assert f32_d == f32_g


def _mats(shapes):
    arr = (D.Dion2Matrix * len(shapes))()
    for i, (m, n) in enumerate(shapes):
        arr[i].rows, arr[i].cols, arr[i].ld = m, n, n
    return arr


def _size(lib, shapes, **kw):
    cfg = D.make_config(**kw)
    out = ctypes.c_size_t(0)
    rc = lib.dion2_workspace_size(_mats(shapes), len(shapes), ctypes.byref(cfg), ctypes.byref(out))
    return rc, out.value


def test_gram_split_k_workspace(lib, monkeypatch):
    """Split-K gram (few long-K matrices: configs[4]): the plan reserves fp32 partials of
    tiles x slices x 256 x 256 only when the gram's upper-triangle pair tiles cover at most
    half of the 74 CTA pairs; slices = min(ceil(74 / tiles), k_blocks / 4)."""
    stress = [(4096, 32768), (28672, 8192)]      # alpha 1/16: (256, 32768) 1 tile + (512, 28672) 3 tiles
    monkeypatch.setenv("DION2_GRAM_SPLITK", "1")
    _, off = _size(lib, stress, alpha=0.0625)
    monkeypatch.delenv("DION2_GRAM_SPLITK")
    _, on = _size(lib, stress, alpha=0.0625)
    assert on - off >= 4 * 19 * 256 * 256 * 4 and on - off < 4 * 19 * 256 * 256 * 4 + 8192
    # the 1B set fills the GPU (432 tiles): no partials
    one_b = [(2048, 2048)] * 4 + [(8192, 2048), (2048, 8192)]
    monkeypatch.setenv("DION2_GRAM_SPLITK", "1")
    _, off1 = _size(lib, one_b * 24)
    monkeypatch.delenv("DION2_GRAM_SPLITK")
    _, on1 = _size(lib, one_b * 24)
    assert on1 == off1
    # fp32 validation path (SIMT NS): never split
    _, f32a = _size(lib, stress, alpha=0.0625, precision="fp32")
    monkeypatch.setenv("DION2_GRAM_SPLITK", "1")
    _, f32b = _size(lib, stress, alpha=0.0625, precision="fp32")
    assert f32a == f32b


def test_workspace_size_scales_with_alpha(lib):
    shapes = [(2048, 2048), (8192, 2048), (2048, 8192)]
    rc1, b1 = _size(lib, shapes, alpha=1.0)
    rc2, b2 = _size(lib, shapes, alpha=0.25)
    assert rc1 == 0 and rc2 == 0 and b1 > b2 > 0
    # the bf16 NS buffers dominate: X ping/pong (2 x p x q) + A, B (2 x p x p), 2 bytes each
    assert b2 >= 2 * 2 * (512 * 2048 * 3) + 2 * 2 * (512 * 512 * 3)


@pytest.mark.parametrize("kw,code", [
    (dict(alpha=0.0), 1), (dict(alpha=1.5), 1), (dict(mu=1.0), 1), (dict(mu=-0.1), 1), (dict(lr=-1.0), 1),
    (dict(ns_steps=0), 1), (dict(ns_steps=17), 1), (dict(ns_eps=0.0), 1),
])
def test_config_validation(lib, kw, code):
    rc, _ = _size(lib, [(64, 64)], **kw)
    assert rc == code


def test_select_rule_validation(lib):
    cfg = D.make_config(select="random", seed=5, step=7)
    out = ctypes.c_size_t(0)
    assert lib.dion2_workspace_size(_mats([(8, 8)]), 1, ctypes.byref(cfg), ctypes.byref(out)) == 0
    cfg.select = 2
    assert lib.dion2_workspace_size(_mats([(8, 8)]), 1, ctypes.byref(cfg), ctypes.byref(out)) == 1


def test_storage_transposed_flag(lib):
    """ABI v5 dion2_matrix.storage_transposed: rows / cols stay logical; a logical 8192 x 2048
    (cols mode) stored transposed is processed as the 2048 x 8192 storage's row selection, so
    it needs the rows-mode plan's workspace; invalid flag values are shape errors."""
    cfg = D.make_config(alpha=0.25)
    out = ctypes.c_size_t(0)
    logical = _mats([(8192, 2048)])
    logical[0].ld = 8192                     # storage is 2048 x 8192
    logical[0].storage_transposed = 1
    assert lib.dion2_workspace_size(logical, 1, ctypes.byref(cfg), ctypes.byref(out)) == 0
    st_bytes = out.value
    rows_mode = _mats([(2048, 8192)])
    assert lib.dion2_workspace_size(rows_mode, 1, ctypes.byref(cfg), ctypes.byref(out)) == 0
    assert st_bytes == out.value
    logical[0].ld = 2048                     # < the storage's 8192 columns
    assert lib.dion2_workspace_size(logical, 1, ctypes.byref(cfg), ctypes.byref(out)) == 2
    logical[0].ld, logical[0].storage_transposed = 8192, 2
    assert lib.dion2_workspace_size(logical, 1, ctypes.byref(cfg), ctypes.byref(out)) == 2


def test_shape_validation(lib):
    arr = _mats([(64, 64)])
    arr[0].ld = 32  # ld < cols
    cfg = D.make_config()
    out = ctypes.c_size_t(0)
    assert lib.dion2_workspace_size(arr, 1, ctypes.byref(cfg), ctypes.byref(out)) == 2
    assert _size(lib, [(0, 5)])[0] == 2
    assert _size(lib, [(10, 60000)], axis="cols")[0] == 2  # selection axis longer than DION2_MAX_SELECT_DIM


def test_step_rejects_before_touching_the_device(lib):
    cfg = D.make_config()
    arr = _mats([(64, 64)])  # NULL W/M/G
    assert lib.dion2_step_batched(arr, 1, ctypes.byref(cfg), None, 0, None) == 2
    arr[0].W = arr[0].M = arr[0].G = 16
    assert lib.dion2_step_batched(arr, 1, ctypes.byref(cfg), None, 0, None) == 3  # no workspace
    cfg.alpha = 2.0
    assert lib.dion2_step_batched(arr, 1, ctypes.byref(cfg), None, 0, None) == 1


def test_strerror(lib):
    for c in range(8):
        assert lib.dion2_strerror(c)
    assert lib.dion2_phase_name(0) == b"momentum_score"


def test_binding_refuses_cpu_tensors():
    import torch
    W = torch.zeros(4, 4)
    with pytest.raises(ValueError, match="CUDA"):
        D.describe([W], [W.clone()], [W.clone()])


def _randomise(cfg, rng):
    """Random, mostly invalid, config fields."""
    cfg.alpha = float(rng.choice([0.0, -0.5, 1e-9, 0.0625, 0.25, 1.0, 1.5, float("nan")]))
    cfg.mu = float(rng.choice([0.0, 0.95, 1.0, -1.0, 2.0]))
    cfg.ns_steps = int(rng.choice([0, 1, 5, 16, 17, -3]))
    cfg.axis = int(rng.integers(-1, 4))
    cfg.precision = int(rng.integers(-1, 3))
    cfg.select = int(rng.integers(-1, 3))
    cfg.decay_mode = int(rng.integers(-1, 3))
    cfg.scale_mode = int(rng.integers(-1, 3))
    cfg.grad_dtype = int(rng.integers(-1, 3))
    cfg.w_dtype = int(rng.integers(-1, 3))
    cfg.ns_form = int(rng.integers(-1, 4))


def test_host_validation_fuzz(lib):
    """Random configs and shapes through the host-only size query (dion2_workspace_size): every
    call returns a documented status code (0-4) and never crashes; a successful query is
    positive.  Even iterations randomise the config on valid shapes, odd ones randomise the
    shapes (zero, negative, over-long, short or huge row strides) under a valid config."""
    import numpy as np
    rng = np.random.default_rng(7)
    codes = set()
    for it in range(2000):
        cfg = D.make_config()
        if it % 2:
            cfg.alpha = float(rng.choice([0.0625, 0.25, 1.0]))
            shapes = [(int(rng.choice([0, 1, 7, 64, 300, 40000, -5])), int(rng.choice([0, 1, 9, 128, 2048, -1])))
                      for _ in range(int(rng.integers(1, 4)))]
        else:
            _randomise(cfg, rng)
            shapes = [(int(rng.choice([64, 300, 2048])), int(rng.choice([128, 512]))) for _ in range(2)]
        arr = (D.Dion2Matrix * len(shapes))()
        for i, (m, n) in enumerate(shapes):
            arr[i].rows, arr[i].cols = m, n
            arr[i].ld = int(rng.choice([n, n + 3, max(n - 1, 0), 1 << 40])) if it % 4 == 1 else n
        out = ctypes.c_size_t(0)
        rc = lib.dion2_workspace_size(arr, len(shapes), ctypes.byref(cfg), ctypes.byref(out))
        assert rc in (0, 1, 2, 3, 4), rc
        if rc == 0:
            assert out.value > 0
        codes.add(rc)
    assert {0, 1, 2} <= codes
