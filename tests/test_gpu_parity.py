"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle (-m gpu).

Gates (BASELINE.json north star):
  * index sets exact (ties within 1e-6 relative resolved by the harness);
  * cumulative dW within 1e-5 relative Frobenius on the fp32 validation path,
    within 2e-2 on the bf16 tensor-core path;
  * unselected rows/cols of W bit-identical, unselected M == fp32(M + G) bitwise.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen_grad, gen_w0, layer_set_1b
from paper_2512_16928_b200 import Dion2, get_phase_times, last_launch_count, set_phase_timing

from gpu_harness import run_parity

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
FP32_TOL = 1e-5


def _assert(res, tol):
    assert res.index_mismatch == 0, res
    assert max(res.dW_rel) <= tol, res
    assert res.unselected_w_bitwise and res.unselected_m_bitwise, res
    assert max(res.M_rel) <= 1e-5, res


# ---------------------------------------------------------------- configs[0]: 256x128, alpha=0.25, 10 steps
@pytest.mark.parametrize("axis", ["auto", "rows"])
def test_config1_fp32_validation_path(axis):
    _assert(run_parity([(256, 128)], 0.25, axis, "fp32", steps=10), FP32_TOL)


@pytest.mark.parametrize("axis", ["auto", "rows", "cols"])
def test_config1_bf16_tensor_core_path(axis):
    _assert(run_parity([(256, 128)], 0.25, axis, "bf16", steps=10), BF16_TOL)


# ---------------------------------------------------------------- ragged, multi-tile batches, every orientation
BATCH_AUTO = [(300, 520), (520, 300), (384, 384), (130, 1030), (7, 33)]


@pytest.mark.parametrize("precision,tol", [("fp32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("axis,shapes", [
    ("auto", BATCH_AUTO),
    ("rows", [(1000, 200), (300, 520)]),      # (1000,200): k=300 > n -> X = S^T
    ("cols", [(200, 1000), (520, 300)]),      # (200,1000): k=300 > m -> X = S
])
def test_ragged_batches(precision, tol, axis, shapes):
    _assert(run_parity(shapes, 0.3, axis, precision, steps=4, row_scaled=True), tol)


@pytest.mark.parametrize("alpha", [1.0, 0.5, 0.125])
def test_alpha_sweep_bf16(alpha):
    _assert(run_parity([(1024, 2048), (2048, 1024)], alpha, "auto", "bf16", steps=2), BF16_TOL)


@pytest.mark.parametrize("form,tol", [("direct", BF16_TOL), ("auto", 1e-2)])
def test_small_p_bf16_error(form, tol):
    """p = 32 (alpha = 0.125 on 256 rows): the round-1 bf16 DIRECT recipe's own error floor
    was ~2.1% there (R21); with fp16 X (R24) both forms meet the 2e-2 gate (emulated
    DIRECT 0.1-0.5%), and AUTO takes the Gram form (q >= 2p)."""
    _assert(run_parity([(256, 512), (512, 256)], 0.125, "auto", "bf16", steps=3, ns_form=form), tol)


# ---------------------------------------------------------------- NS evaluation form (reading R23)
def test_gram_form_is_tighter_on_wide_x():
    """AUTO picks the Gram-space form for q >= 2p; X is rounded to bf16 once instead of T
    times, so its error is well inside the bf16 gate (emulated: 0.3-0.5%)."""
    res = run_parity([(512, 2048), (2048, 512), (1024, 4096)], 0.25, "auto", "bf16", steps=2, row_scaled=True)
    _assert(res, 1e-2)


@pytest.mark.parametrize("form", ["direct", "gram"])
def test_both_ns_forms_on_the_1b_layer(form):
    _assert(run_parity(layer_set_1b(layers=1), 0.25, "auto", "bf16", steps=1, ns_form=form), BF16_TOL)


@pytest.mark.parametrize("coeffs", [
    [(3.4445, -4.7750, 2.0315)],                               # T = 1: C_0 is Q_T
    [(3.4445, -4.7750, 2.0315)] * 2,                           # T = 2: no A update after t = 0
    [(1.5, -0.5, 0.0)] * 3,                                    # cubic Newton-Schulz (c = 0)
    [(3.4445, -4.7750, 2.0315)] * 4 + [(2.0, -1.5, 0.5)],      # per-iteration coefficients
    [(1.5, -0.5, 0.0)] * 16,                                   # T = DION2_MAX_NS_STEPS (61 Gram products)
])
@pytest.mark.parametrize("form", ["direct", "gram"])
def test_ns_schedules(coeffs, form):
    shapes = [(256, 1024), (1024, 256), (130, 1030), (300, 520)]
    _assert(run_parity(shapes, 0.3, "auto", "bf16", steps=2, ns_form=form, ns_coeffs=coeffs), BF16_TOL)


def test_gram_form_large_tile_grid():
    """p_pad = 1280 (5 x 5 tile grid, 15 stored upper tiles; lower k-blocks read transposed
    from four different tile rows) and p_pad = 768, ragged p and q."""
    _assert(run_parity([(1100, 4400), (3000, 700)], 1.0, "auto", "bf16", steps=2, row_scaled=True), BF16_TOL)


def test_auto_mixes_both_ns_forms_in_one_call():
    """alpha = 0.8: (1024, 1024) keeps the direct form (p = 819, q = 1024: q < 2p padded or
    not), the other three take the Gram form: one batched call runs both launch lists."""
    _assert(run_parity([(600, 800), (512, 2048), (1024, 1024), (3000, 1000)], 0.8, "auto", "bf16", steps=2,
                       row_scaled=True), BF16_TOL)


def test_gram_form_forced_on_square_x():
    # q = p: AUTO would pick DIRECT; forcing GRAM must still be within the bf16 gate
    _assert(run_parity([(384, 384), (512, 768)], 1.0, "auto", "bf16", steps=2, ns_form="gram"), BF16_TOL)


@pytest.mark.parametrize("form", ["auto", "direct"])
@pytest.mark.parametrize("splitk", [None, "1", "3"])
def test_gram_split_k(form, splitk, monkeypatch):
    """Few long-K matrices (configs[4]-like): the gram launch splits K across CTA pairs (fp32
    partials, slices summed in order by k_splitk_reduce).  None: the library's choice (5 sym
    tiles -> 15 slices); "1": off; "3": forced.  Ragged q (9000), p_pad 256 and 512."""
    if splitk:
        monkeypatch.setenv("DION2_GRAM_SPLITK", splitk)
    _assert(run_parity([(512, 8192), (300, 9000), (2048, 4096)], 0.25, "auto", "bf16", steps=2, ns_form=form,
                       row_scaled=True), BF16_TOL)


def test_alpha1_is_full_muon_fp32():
    _assert(run_parity([(128, 384)], 1.0, "auto", "fp32", steps=5), FP32_TOL)


def test_one_layer_of_the_1b_set_bf16():
    """One transformer layer of BASELINE configs[1] at full size, alpha=0.25."""
    _assert(run_parity(layer_set_1b(layers=1), 0.25, "auto", "bf16", steps=2, check_bitwise=True), BF16_TOL)


def test_one_layer_of_the_8b_set_bf16():
    """One layer of BASELINE configs[3] (Llama-3-8B-like shapes), alpha = 0.25, full size."""
    from synth import layer_set_8b
    _assert(run_parity(layer_set_8b(1), 0.25, "auto", "bf16", steps=1, check_bitwise=True), BF16_TOL)


def test_stress_shapes_alpha_1_16():
    """BASELINE configs[4]: 4096 x 32768 (rows, k = 256) and 28672 x 8192 (cols, k = 512) at alpha = 0.0625."""
    _assert(run_parity([(4096, 32768), (28672, 8192)], 0.0625, "auto", "bf16", steps=1, check_bitwise=True),
            BF16_TOL)


@pytest.mark.parametrize("precision,tol", [("fp32", FP32_TOL), ("bf16", BF16_TOL)])
def test_random_selection(precision, tol):
    """Random rule: GPU Philox keys must select exactly the oracle's subset."""
    _assert(run_parity([(256, 128), (300, 520), (1024, 2048)], 0.25, "auto", precision, steps=4,
                       select="random", sel_seed=1234), tol)


@pytest.mark.parametrize("mt", [False, True])
def test_column_scatter_large_k(mt):
    """Column-mode scatter with 1024 < k <= 4096 (8-row staged O tiles; k = 1500, 2250, 2048
    ragged): the streaming scatter, with a generic or a transposed-M row gather."""
    _assert(run_parity([(4096, 2000), (6000, 3000), (8192, 2048)], 0.75, "auto", "bf16", steps=2,
                       m_transposed=mt, row_scaled=True), BF16_TOL)


@pytest.mark.parametrize("precision,tol,mt", [("bf16", BF16_TOL, False), ("fp32", FP32_TOL, False),
                                              ("bf16", BF16_TOL, True)])
def test_storage_transposed_layout(precision, tol, mt):
    """ABI v5: W, M, G stored (fan-in, fan-out) as JAX / Flax kernels are; axis (incl. the square
    tie-break), k and scale follow the logical shape.  Wide, tall, square and ragged matrices;
    with mt, the logical-layout momentum of the storage's column-mode matrices."""
    shapes = [(2048, 512), (512, 2048), (384, 384), (300, 520), (1000, 256)]
    _assert(run_parity(shapes, 0.25, "auto", precision, steps=3, row_scaled=True, storage_transposed=True,
                       m_transposed=mt), tol)


def test_transposed_momentum_for_column_mode():
    """f4: M stored transposed for column-mode matrices (row gather of M^T, transpose-add K1)."""
    shapes = [(520, 300), (1000, 256), (8192, 2048), (300, 520)]
    _assert(run_parity(shapes, 0.25, "auto", "bf16", steps=3, m_transposed=True, row_scaled=True), BF16_TOL)
    _assert(run_parity(shapes[:3], 0.25, "auto", "bf16", steps=2, m_transposed=True, grad_bf16=True), BF16_TOL)
    # alpha = 1: k = 1536 > 1024 -> generic-tile scatter, row gather of M^T
    _assert(run_parity([(2048, 1536), (520, 300)], 1.0, "auto", "bf16", steps=2, m_transposed=True), BF16_TOL)


@pytest.mark.parametrize("grad_bf16", [False, True])
@pytest.mark.parametrize("stages", [None, "2", "4"])
def test_pipelined_transposed_k1(grad_bf16, stages, monkeypatch):
    """The cp.async-pipelined transposed-M K1 (every column-mode matrix aligned, whole
    256 x 64 units): fp32 and bf16 G, the default 3 stages and the 2 / 4 stage variants."""
    if stages:
        monkeypatch.setenv("DION2_K1MT_PIPE", stages)
    shapes = [(8192, 2048), (1024, 512), (2048, 1024), (512, 2048)]
    _assert(run_parity(shapes, 0.25, "auto", "bf16", steps=3, m_transposed=True, grad_bf16=grad_bf16), BF16_TOL)


@pytest.mark.parametrize("stages", ["0", "4", "6"])
def test_tma_staged_rows_gather(stages, monkeypatch):
    """K3 rows path: the TMA-staged bulk-copy ring (4 / 6 stages) and the register-streaming
    fallback ("0"); rows of M and of M^T, multi-chunk rows (8192 > 2048), ragged k with zero
    X rows (k = 75 of p_pad = 256), bf16 gradients."""
    monkeypatch.setenv("DION2_GATHER_TMA", stages)
    shapes = [(512, 8192), (8192, 1024), (300, 520), (1024, 2048)]
    _assert(run_parity(shapes, 0.25, "auto", "bf16", steps=3, m_transposed=True, row_scaled=True), BF16_TOL)
    _assert(run_parity(shapes[:2], 0.25, "auto", "bf16", steps=2, grad_bf16=True), BF16_TOL)


def test_full_decay_ablation_fp32():
    _assert(run_parity([(96, 160)], 0.25, "auto", "fp32", steps=3, decay_mode=1), FP32_TOL)


# ---------------------------------------------------------------- exact selection (ties, tie-break)
def test_select_exact_ties_lowest_index():
    """Integer-valued G: every l1 score is exact in fp32, with many exact ties;
    K must equal the brute-force (score desc, index asc) set bit for bit."""
    rng = np.random.default_rng(0)
    m, n = 700, 40
    G = rng.integers(0, 3, size=(m, n)).astype(np.float32)
    G[100:200] = G[0]          # exact duplicates of row 0's l1 score
    W = torch.zeros(m, n, device="cuda")
    M = torch.zeros(m, n, device="cuda")
    sel = torch.empty(O.select_count(np.float32(0.25), m), dtype=torch.int32, device="cuda")
    Dion2(alpha=0.25, axis="rows").step([W], [M], [torch.from_numpy(G).cuda()], sel_out=[sel])
    s = np.abs(G.astype(np.float64)).sum(1)
    want = sorted(sorted(range(m), key=lambda i: (-s[i], i))[:len(sel)])
    assert sel.cpu().numpy().tolist() == want


@pytest.mark.parametrize("d", [1, 2, 5, 1024, 1025, 4097, 32768])
def test_select_sizes(d):
    m, n = (d, 8)
    G = gen_grad(m, n, 3, 0, 0, row_scaled=True)
    W = torch.zeros(m, n, device="cuda")
    M = torch.zeros(m, n, device="cuda")
    k = O.select_count(np.float32(0.25), m)
    sel = torch.empty(k, dtype=torch.int32, device="cuda")
    Dion2(alpha=0.25, axis="rows").step([W], [M], [torch.from_numpy(G).cuda()], sel_out=[sel])
    s = O.l1_scores(G.astype(np.float64), O.AXIS_ROWS)
    ref = O.select_l1(s, k)
    got = sel.cpu().numpy()
    if not np.array_equal(got, ref):  # allow fp32-vs-fp64 near-ties only
        kth = np.sort(s)[::-1][k - 1]
        assert np.all(np.abs(s[np.setxor1d(got, ref)] - kth) <= 1e-6 * kth)


# ---------------------------------------------------------------- edge cases
def test_lr_zero_leaves_w_bitwise():
    W = torch.from_numpy(gen_w0(128, 256)).cuda()
    W0 = W.clone()
    M = torch.zeros_like(W)
    Dion2(alpha=0.25, lr=0.0).step([W], [M], [torch.from_numpy(gen_grad(128, 256)).cuda()])
    assert torch.equal(W, W0)


def test_zero_input_leaves_w_unchanged_and_selects_lowest():
    W = torch.from_numpy(gen_w0(64, 96)).cuda()
    W0 = W.clone()
    M = torch.zeros_like(W)
    sel = torch.empty(16, dtype=torch.int32, device="cuda")
    Dion2(alpha=0.25).step([W], [M], [torch.zeros_like(W)], sel_out=[sel])
    assert torch.equal(W, W0)
    assert sel.cpu().tolist() == list(range(16))


def test_nonfinite_matrix_is_skipped_and_reported():
    Ws = [torch.from_numpy(gen_w0(64, 128, 0, i)).cuda() for i in range(3)]
    W0 = [w.clone() for w in Ws]
    Ms = [torch.zeros_like(w) for w in Ws]
    Gs = [torch.from_numpy(gen_grad(64, 128, 0, i)).cuda() for i in range(3)]
    Gs[1][5, 7] = float("nan")
    opt = Dion2(alpha=0.25)
    opt.step(Ws, Ms, Gs)
    rc, bad = opt.status()
    assert rc == 7 and bad == 1
    assert torch.equal(Ws[1], W0[1])
    assert not torch.equal(Ws[0], W0[0]) and not torch.equal(Ws[2], W0[2])
    # the NaN stays in M[1] (M <- M + G ran before the scores were checked): the next
    # step reports it again; once the caller resets that state, a step is clean
    opt.step(Ws, Ms, [torch.zeros_like(g) for g in Gs])
    assert opt.status() == (7, 1)
    Ms[1].zero_()
    opt.step(Ws, Ms, [torch.zeros_like(g) for g in Gs])
    assert opt.status() == (0, -1)


def test_cuda_graph_capture_replays_the_step():
    """The step enqueues only stream-ordered work once its plan exists (no host sync, no
    allocation): a CUDA graph captured after one eager step replays it bit for bit, PDL
    edges and the split-K / pipelined kernels included."""
    shapes = [(512, 1024), (1024, 512), (2048, 512), (300, 520), (512, 8192)]
    def init():
        Ws = [torch.from_numpy(gen_w0(m, n, 3, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Ms = [torch.zeros(n, m, device="cuda") if m > n else torch.zeros(m, n, device="cuda") for (m, n) in shapes]
        Gs = [torch.from_numpy(gen_grad(m, n, 3, i, 0, row_scaled=True)).cuda() for i, (m, n) in enumerate(shapes)]
        return Ws, Ms, Gs
    mt = [m > n for (m, n) in shapes]
    Wa, Ma, Ga = init()
    eager = Dion2(alpha=0.25, m_transposed=mt)
    for _ in range(4):
        eager.step(Wa, Ma, Ga)
    Wb, Mb, Gb = init()
    opt = Dion2(alpha=0.25, m_transposed=mt)
    opt.step(Wb, Mb, Gb)                     # builds the plan, uploads the tables
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        opt.step(Wb, Mb, Gb)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(Wa + Ma, Wb + Mb):
        assert torch.equal(a, b)


def test_cuda_graph_mode_equals_eager():
    """Dion2(cuda_graph=True): a key (tensors + config minus eta) repeated on consecutive calls
    is captured on its second call and replayed afterwards; keys that change every call (the
    alternating gradient buffers) run eagerly; a learning-rate schedule replays one graph (eta
    is read on the device, DION2_FLAG_LR_DEVICE); a second tensor set captures again.  Bitwise
    equal to the eager optimizer."""
    shapes = [(512, 1024), (2048, 512), (300, 520)]
    mt = [m > n for (m, n) in shapes]
    def init(seed):
        Ws = [torch.from_numpy(gen_w0(m, n, seed, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Ms = [torch.zeros(n, m, device="cuda") if t else torch.zeros(m, n, device="cuda")
              for (m, n), t in zip(shapes, mt)]
        return Ws, Ms
    data = [[torch.from_numpy(gen_grad(m, n, 4, i, t, row_scaled=True)).cuda() for i, (m, n) in enumerate(shapes)]
            for t in range(6)]
    outs = []
    for graph in (False, True):
        opt = Dion2(alpha=0.25, m_transposed=mt, cuda_graph=graph)
        Wa, Ma = init(7)
        Wb, Mb = init(8)
        G = [torch.empty(m, n, device="cuda") for (m, n) in shapes]
        for t in range(6):                     # same buffers: eager, eager + capture, replays
            for g, d in zip(G, data[t]):
                g.copy_(d)
            opt.step(Wa, Ma, G)
            if t == 3:
                opt.cfg_kw["lr"] = 0.01        # new key: eager, then capture, then replay
        for t in range(4):                     # alternating buffers: every key new, all eager
            opt.step(Wa, Ma, data[t % 2])
        G2 = [torch.empty(m, n, device="cuda") for (m, n) in shapes]
        for t in range(5):                     # a learning-rate schedule on fixed buffers: eta is read
            opt.cfg_kw["lr"] = 0.02 / (t + 1)  # from the workspace, so the graph replays (no re-capture)
            for g, d in zip(G2, data[t]):
                g.copy_(d)
            opt.step(Wa, Ma, G2)
        for t in range(3):
            opt.step(Wb, Mb, data[t])
        torch.cuda.synchronize()
        outs.append([x.clone() for x in Wa + Ma + Wb + Mb])
        if graph:
            assert len(opt._graphs) >= 2
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("graph", [False, True])
def test_step_host_pipelined_upload(graph):
    """Dion2.step_host: gradients from pinned host buffers, uploaded chunk by chunk on a side
    stream while earlier chunks step; same selections and M as the one-call step, dW within
    the bf16 rounding of a different split-K/batching (each chunk is its own batched call)."""
    shapes = [(512, 1024), (2048, 512), (300, 520), (1024, 1024), (512, 2048), (256, 128)]
    mt = [m > n for (m, n) in shapes]
    ks = [max(1, int(0.25 * (m if m <= n else n) + 0.5)) for (m, n) in shapes]
    def init():
        Ws = [torch.from_numpy(gen_w0(m, n, 9, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Ms = [torch.zeros(n, m, device="cuda") if t else torch.zeros(m, n, device="cuda")
              for (m, n), t in zip(shapes, mt)]
        return Ws, Ms
    Gh = [[torch.from_numpy(gen_grad(m, n, 9, i, t, row_scaled=True)).pin_memory() for i, (m, n) in enumerate(shapes)]
          for t in range(3)]
    W0, _ = init()
    Wa, Ma = init()
    Ga = [torch.empty(m, n, device="cuda") for (m, n) in shapes]
    sa = [torch.empty(k, dtype=torch.int32, device="cuda") for k in ks]
    ref = Dion2(alpha=0.25, m_transposed=mt)
    Wb, Mb = init()
    Gb = [torch.empty(m, n, device="cuda") for (m, n) in shapes]
    sb = [torch.empty(k, dtype=torch.int32, device="cuda") for k in ks]
    opt = Dion2(alpha=0.25, m_transposed=mt, cuda_graph=graph)
    for t in range(3):
        for g, h in zip(Ga, Gh[t]):
            g.copy_(h)
        ref.step(Wa, Ma, Ga, sel_out=sa)
        opt.step_host(Wb, Mb, Gb, Gh[t], sel_out=sb, chunks=3)
        torch.cuda.synchronize()
        for x, y in zip(sa, sb):
            assert torch.equal(x, y)
    assert opt.status() == (0, -1)
    for a, b, w0 in zip(Wa, Wb, W0):
        da, db = (a - w0).double(), (b - w0).double()
        assert (da - db).norm() <= 1e-2 * da.norm()
    for a, b in zip(Ma, Mb):
        assert (a - b).abs().max() <= 1e-6 * a.abs().max()


def test_lr_device_flag_through_the_c_abi():
    """DION2_FLAG_LR_DEVICE: eta comes from the fp32 word at byte 8 of the 4096-aligned workspace
    base (cfg.lr, deliberately different, is ignored by the kernels); bitwise equal to a step with
    cfg.lr = that eta.  Rows and column (index-walk) scatters."""
    import ctypes
    from paper_2512_16928_b200 import dion2 as D
    shapes = [(512, 1024), (2048, 512), (300, 520), (1000, 200)]
    def run(lr_device):
        Ws = [torch.from_numpy(gen_w0(m, n, 12, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Ms = [torch.zeros_like(w) for w in Ws]
        Gs = [torch.from_numpy(gen_grad(m, n, 12, i, 0, row_scaled=True)).cuda() for i, (m, n) in enumerate(shapes)]
        arr, _ = D.describe(Ws, Ms, Gs)
        cfg = D.make_config(alpha=0.3, lr=0.5 if lr_device else 0.0123, lr_device=lr_device)
        need = ctypes.c_size_t(0)
        assert D._lib().dion2_workspace_size(arr, len(Ws), ctypes.byref(cfg), ctypes.byref(need)) == 0
        ws = torch.zeros(need.value, dtype=torch.uint8, device="cuda")
        base = ws.data_ptr()
        off = ((base + 4095) & ~4095) - base + 8
        ws[off:off + 4].view(torch.float32).fill_(0.0123)
        rc = D._lib().dion2_step_batched(arr, len(Ws), ctypes.byref(cfg), base, ws.numel(),
                                         torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        return Ws + Ms
    for a, b in zip(run(False), run(True)):
        assert torch.equal(a, b)


def test_bitwise_determinism():
    shapes = [(512, 1024), (1024, 512)]
    outs = []
    for _ in range(2):
        Ws = [torch.from_numpy(gen_w0(m, n, 1, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Ms = [torch.zeros_like(w) for w in Ws]
        opt = Dion2(alpha=0.25)
        for t in range(3):
            opt.step(Ws, Ms, [torch.from_numpy(gen_grad(m, n, 1, i, t)).cuda() for i, (m, n) in enumerate(shapes)])
        outs.append([w.clone() for w in Ws] + [mm.clone() for mm in Ms])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_plan_cache_distinguishes_the_momentum_layout():
    """Same shapes, same config, same workspace: a step with transposed momentum after one with
    M in W's layout must not reuse the first plan (bitwise equal to a fresh optimizer)."""
    shapes = [(2048, 512), (1024, 256)]
    def fresh():
        W = [torch.from_numpy(gen_w0(m, n, 5, i)).cuda() for i, (m, n) in enumerate(shapes)]
        G = [torch.from_numpy(gen_grad(m, n, 5, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Mt = [torch.zeros(n, m, device="cuda") for (m, n) in shapes]
        return W, Mt, G
    opt = Dion2(alpha=0.25)
    W0, G0 = [torch.from_numpy(gen_w0(m, n, 6, i)).cuda() for i, (m, n) in enumerate(shapes)], None
    opt.step(W0, [torch.zeros_like(w) for w in W0], [torch.ones_like(w) for w in W0])
    Wa, Ma, Ga = fresh()
    opt.step(Wa, Ma, Ga, m_transposed=[True, True])
    Wb, Mb, Gb = fresh()
    Dion2(alpha=0.25).step(Wb, Mb, Gb, m_transposed=[True, True])
    torch.cuda.synchronize()
    for a, b in zip(Wa + Ma, Wb + Mb):
        assert torch.equal(a, b)


def test_bf16_gradient_input():
    _m, _n = 256, 512
    W = torch.from_numpy(gen_w0(_m, _n)).cuda()
    W0 = W.clone()
    M = torch.zeros_like(W)
    G = torch.from_numpy(gen_grad(_m, _n)).cuda()
    Gb = G.to(torch.bfloat16)
    Dion2(alpha=0.25).step([W], [M], [Gb])
    # momentum accumulated exactly the bf16 values
    Wr, Mr = W0.cpu().double().numpy(), np.zeros((_m, _n))
    O.dion2_step(Wr, Mr, Gb.float().cpu().double().numpy(), O.OracleConfig(alpha=0.25))
    dref = Wr - W0.cpu().double().numpy()
    dgpu = W.cpu().double().numpy() - W0.cpu().double().numpy()
    assert np.linalg.norm(dgpu - dref) / np.linalg.norm(dref) <= BF16_TOL


def test_phase_timing_and_launch_count():
    # X of 256 rows: the tensor-core Gram-space form; a 32-row X: the short-X NS (ns_mul phase)
    for (m, n), ns_phases in (((1024, 2048), ("ns_gram", "ns_poly", "ns_apply")), ((128, 512), ("ns_mul",))):
        Ws = [torch.from_numpy(gen_w0(m, n)).cuda()]
        Ms = [torch.zeros_like(Ws[0])]
        set_phase_timing(True)
        try:
            Dion2(alpha=0.25).step(Ws, Ms, [torch.ones_like(Ws[0])])
            times = get_phase_times()
        finally:
            set_phase_timing(False)
        pre = ("momentum_score", "select", "gather_rows")
        assert last_launch_count() >= len(ns_phases) + 2 + len(pre)
        for ph in pre + ns_phases + ("scatter_rows",):
            assert times[ph][1] >= 1 and times[ph][0] > 0, (m, n, ph, times)


def test_stream_calls_do_not_disturb_captured_graphs():
    """in graph mode a call with an explicit stream runs eagerly in the uncaptured
    workspace slot, so it cannot overwrite the descriptor table of a captured graph's plan
    (same shapes, other tensors).  Replays after such calls must still update their own W/M:
    bitwise equal to the eager optimizer on the same call sequence."""
    shapes = [(512, 1024), (1024, 512)]
    data = [[torch.from_numpy(gen_grad(m, n, 9, i, t, row_scaled=True)).cuda() for i, (m, n) in enumerate(shapes)]
            for t in range(4)]
    outs = []
    for graph in (False, True):
        opt = Dion2(alpha=0.25, cuda_graph=graph)
        Wa = [torch.from_numpy(gen_w0(m, n, 1, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Ma = [torch.zeros_like(w) for w in Wa]
        Wb = [torch.from_numpy(gen_w0(m, n, 2, i)).cuda() for i, (m, n) in enumerate(shapes)]
        Mb = [torch.zeros_like(w) for w in Wb]
        side = torch.cuda.Stream()
        for t in range(4):
            opt.step(Wa, Ma, data[0])                      # t >= 1: captured in slot 0, then replayed
            side.wait_stream(torch.cuda.current_stream())
            opt.step(Wb, Mb, data[t], stream=side)         # same shapes, other tensors, explicit stream
            torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        outs.append([x.clone() for x in Wa + Ma + Wb + Mb])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_dion2_step_entry_point():
    """dion2_step (one matrix) through the C ABI: bitwise equal to dion2_step_batched with n = 1."""
    import ctypes
    from paper_2512_16928_b200 import dion2 as D
    m, n = 384, 1024
    outs = []
    for single in (True, False):
        W = torch.from_numpy(gen_w0(m, n, 3)).cuda()
        M = torch.zeros_like(W)
        G = torch.from_numpy(gen_grad(m, n, 3)).cuda()
        arr, _ = D.describe([W], [M], [G])
        cfg = D.make_config(alpha=0.25)
        need = ctypes.c_size_t(0)
        assert D._lib().dion2_workspace_size(arr, 1, ctypes.byref(cfg), ctypes.byref(need)) == 0
        ws = torch.zeros(need.value, dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(2):
            if single:
                rc = D._lib().dion2_step(arr, ctypes.byref(cfg), ws.data_ptr(), ws.numel(), st)
            else:
                rc = D._lib().dion2_step_batched(arr, 1, ctypes.byref(cfg), ws.data_ptr(), ws.numel(), st)
            assert rc == 0
        bad = ctypes.c_int32(5)
        assert D._lib().dion2_get_status(ws.data_ptr(), st, ctypes.byref(bad)) == 0 and bad.value == -1
        assert D._lib().dion2_release_workspace(ws.data_ptr(), ws.numel()) >= 1
        outs.append((W.clone(), M.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("precision,tol", [("bf16", BF16_TOL), ("fp32", FP32_TOL)])
def test_submatrix_scale_mode(precision, tol):
    """f3: scale_mode = 1 scales the update by sqrt of the SUBMATRIX dimensions
    instead of the full W's sqrt(fan-out / fan-in); rows and column mode, both NS forms."""
    _assert(run_parity([(512, 1024), (1024, 512), (300, 520)], 0.25, "auto", precision, steps=3, scale_mode=1), tol)


def test_status_is_stream_scoped():
    """dion2_get_status synchronises the step's stream only: a long kernel on another stream
    is still running when it returns."""
    Ws = [torch.from_numpy(gen_w0(256, 512)).cuda()]
    Ms = [torch.zeros_like(Ws[0])]
    Gs = [torch.from_numpy(gen_grad(256, 512)).cuda()]
    opt = Dion2(alpha=0.25)
    other = torch.cuda.Stream()
    with torch.cuda.stream(other):
        torch.cuda._sleep(2_000_000_000)  # ~1 s of spinning on the other stream
    opt.step(Ws, Ms, Gs)
    assert opt.status() == (0, -1)
    assert not other.query()  # the other stream's kernel has not finished
    other.synchronize()


@pytest.mark.parametrize("form", ["auto", "direct"])
def test_bf16_weights(form):
    """f4 bf16-W variant (dion2_config.w_dtype = BF16): W held in bf16, the update computed in
    fp32 and rounded to nearest once.  Per-step parity: the oracle starts every
    step from the GPU's bf16 W (exact in fp64) and M; the GPU's new W must sit within the bf16
    rounding of the oracle's new W (half an ulp per element) plus the 2e-2 NS tolerance on the
    update, and unselected rows / columns of W must be bit-identical."""
    shapes = [(512, 1024), (1024, 512), (300, 520)]
    cfg = O.OracleConfig(alpha=0.25, mu=float(np.float32(0.95)), lr=float(np.float32(0.02)))
    Wb = [torch.from_numpy(gen_w0(m, n, 5, i)).cuda().to(torch.bfloat16) for i, (m, n) in enumerate(shapes)]
    Ms = [torch.zeros(m, n, device="cuda") for (m, n) in shapes]
    ks = [O.select_count(0.25, min(m, n)) for (m, n) in shapes]
    opt = Dion2(alpha=0.25, ns_form=form)
    for t in range(3):
        G = [gen_grad(m, n, 5, i, t, row_scaled=True) for i, (m, n) in enumerate(shapes)]
        W_before = [w.double().cpu().numpy() for w in Wb]
        M_before = [mm.double().cpu().numpy() for mm in Ms]
        sel = [torch.empty(k, dtype=torch.int32, device="cuda") for k in ks]
        opt.step(Wb, Ms, [torch.from_numpy(g).cuda() for g in G], sel_out=sel)
        torch.cuda.synchronize()
        for i in range(len(shapes)):
            Wr, Mr = W_before[i].copy(), M_before[i].copy()
            K, _, ax = O.dion2_step(Wr, Mr, G[i].astype(np.float64), cfg, force_K=sel[i].cpu().numpy())
            Kref = O.select_l1(O.l1_scores(M_before[i] + G[i], ax), ks[i])
            assert np.array_equal(K, Kref)
            wg = Wb[i].double().cpu().numpy()
            d_ref = Wr - W_before[i]
            ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(Wr), 1e-30))) - 7)
            bound = np.linalg.norm(0.5 * ulp[d_ref != 0]) + 2e-2 * np.linalg.norm(d_ref)
            assert np.linalg.norm(wg - Wr) <= bound, (i, t, np.linalg.norm(wg - Wr), bound)
            unsel = np.ones(shapes[i][0] if ax == O.AXIS_ROWS else shapes[i][1], bool)
            unsel[K] = False
            if ax == O.AXIS_ROWS:
                assert np.array_equal(wg[unsel], W_before[i][unsel])
            else:
                assert np.array_equal(wg[:, unsel], W_before[i][:, unsel])
            assert np.abs(Ms[i].double().cpu().numpy() - Mr).max() <= 1e-6 * np.abs(Mr).max()


@pytest.mark.parametrize("variant", ["1sm_apply", "all"])
def test_apply_kernel_variants(variant, monkeypatch):
    """The apply kernels selectable for A/B (DION2_NS_PAIR): the 1-SM kernel and the streaming
    pair kernel instead of the resident-A pair apply; both NS forms, p_pad 256 and 512, ragged q."""
    monkeypatch.setenv("DION2_NS_PAIR", variant)
    shapes = [(512, 2048), (2048, 512), (1024, 4096), (300, 1200), (1024, 1024)]
    _assert(run_parity(shapes, 0.25, "auto", "bf16", steps=2, row_scaled=True), BF16_TOL)
    _assert(run_parity(shapes[:3], 0.25, "auto", "bf16", steps=2, ns_form="direct"), BF16_TOL)
