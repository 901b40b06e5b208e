"""Pins for the fp64 oracle (-m "not gpu").

Each test ties an oracle function to something other than itself: a closed
form (SVD of the quintic iteration), brute force, an algebraic identity the
paper states (alpha=1 == Muon, Eq. error-feedback, Eq. orth-update), or a
worked example (tests/golden/, each with its citation).  A plausible slip in
the oracle (dropped term, wrong sign/index, transposed operand, pre- vs
post-decay NS input, wrong scale factor) fails at least one of these.
"""
import math
import os

import numpy as np
import pytest

import oracle as O
from synth import gen_grad, gen_scores_with_ties, gen_w0

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_rows(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ----------------------------------------------------------------------------- selection

def test_select_count_golden():
    for a, d, k in _read_rows("select_count.txt"):
        assert O.select_count(float(a), int(d)) == int(k)


def test_select_count_edges():
    assert O.select_count(1e-9, 100) == 1          # max(1, .)
    assert O.select_count(1.0, 1) == 1
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(ValueError):
            O.select_count(bad, 10)


def test_select_l1_golden_example():
    rows = {r[0]: r[1:] for r in _read_rows("select_l1_example.txt")}
    s = np.array([float(x) for x in rows["scores"]])
    k = O.select_count(float(rows["alpha"][0]), len(s))
    assert list(O.select_l1(s, k)) == [int(x) for x in rows["expect"]]


def _brute_topk(s, k):
    # pure Python: sort (index) by key (-score, index); independent of lexsort
    idx = sorted(range(len(s)), key=lambda i: (-float(s[i]), i))[:k]
    return sorted(idx)


def test_select_l1_brute_force_with_ties():
    for case in range(1000):
        d = 1 + (case * 37) % 97
        s = gen_scores_with_ties(d, seed=case, n_distinct=1 + case % 7)
        k = O.select_count([0.125, 0.25, 0.5, 1.0, 0.3][case % 5], d)
        assert list(O.select_l1(s, k)) == _brute_topk(s, k)


def test_select_alpha1_and_zero():
    s = np.zeros(9)
    assert list(O.select_l1(s, 4)) == [0, 1, 2, 3]      # all-zero -> lowest indices
    s = np.random.default_rng(0).random(11)
    assert list(O.select_l1(s, 11)) == list(range(11))  # alpha=1 -> all


def test_l1_scores_brute():
    M = np.random.default_rng(1).standard_normal((5, 7))
    rows = [sum(abs(M[i, j]) for j in range(7)) for i in range(5)]
    cols = [sum(abs(M[i, j]) for i in range(5)) for j in range(7)]
    np.testing.assert_allclose(O.l1_scores(M, O.AXIS_ROWS), rows, rtol=1e-14)
    np.testing.assert_allclose(O.l1_scores(M, O.AXIS_COLS), cols, rtol=1e-14)


def test_auto_axis_rule():
    assert O.resolve_axis(4, 8, O.AXIS_AUTO) == O.AXIS_ROWS
    assert O.resolve_axis(8, 4, O.AXIS_AUTO) == O.AXIS_COLS
    assert O.resolve_axis(5, 5, O.AXIS_AUTO) == O.AXIS_ROWS   # square -> rows (R8)


# ----------------------------------------------------------------------------- Newton-Schulz

def _quintic_closed_form(X, coeffs, eps):
    """O = U diag(p_T o ... o p_1(sigma_i / (||X||_F + eps))) V^T: an odd matrix
    polynomial acts on the singular values only."""
    U, sig, Vt = np.linalg.svd(X, full_matrices=False)
    x = sig / (np.linalg.norm(X) + eps)
    for a, b, c in coeffs:
        x = a * x + b * x ** 3 + c * x ** 5
    return (U * x) @ Vt, x


@pytest.mark.parametrize("shape", [(8, 3), (3, 8), (32, 64), (64, 256), (128, 512), (256, 32), (1, 17)])
def test_ns_matches_svd_closed_form(shape):
    X = np.random.default_rng(hash(shape) % 1000).standard_normal(shape)
    got = O.newton_schulz_auto(X)
    want, _ = _quintic_closed_form(X, O.DEFAULT_NS_COEFFS, O.DEFAULT_NS_EPS)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


def test_ns_custom_coefficient_table_closed_form():
    coeffs = [(4.0848, -6.8946, 2.9270), (3.9505, -6.3029, 2.6377), (3.7418, -5.5913, 2.3037),
              (2.8769, -3.1427, 1.2046), (2.8366, -3.0525, 1.2012)]
    X = np.random.default_rng(5).standard_normal((24, 40))
    got = O.newton_schulz(X, coeffs)
    want, _ = _quintic_closed_form(X, coeffs, O.DEFAULT_NS_EPS)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


def test_ns_triple_loop_brute_force():
    """Pure-Python lists and loops (no BLAS) on a 3x5 matrix."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((3, 5))
    Y = [[float(v) for v in row] for row in X]
    nrm = math.sqrt(sum(v * v for row in Y for v in row)) + O.DEFAULT_NS_EPS
    Y = [[v / nrm for v in row] for row in Y]
    for a, b, c in O.DEFAULT_NS_COEFFS:
        A = [[sum(Y[i][t] * Y[j][t] for t in range(5)) for j in range(3)] for i in range(3)]
        AA = [[sum(A[i][t] * A[t][j] for t in range(3)) for j in range(3)] for i in range(3)]
        B = [[b * A[i][j] + c * AA[i][j] for j in range(3)] for i in range(3)]
        Y = [[a * Y[i][j] + sum(B[i][t] * Y[t][j] for t in range(3)) for j in range(5)] for i in range(3)]
    np.testing.assert_allclose(O.newton_schulz(X), np.array(Y), rtol=0, atol=1e-14)


@pytest.mark.parametrize("shape,coeffs", [((16, 96), None), ((40, 90), [(1.5, -0.5, 0.0)] * 3),
                                          ((24, 200), [(3.4445, -4.7750, 2.0315)])])
def test_gram_space_form_is_the_same_map(shape, coeffs):
    """Reading R23 (the GPU's Gram-space evaluation) computes the oracle's map: with
    A_t = X_t X_t^T and C_t = a I + b A_t + c A_t^2, X_{t+1} = C_t X_t gives
    A_{t+1} = C_t A_t C_t and X_T = (C_{T-1} ... C_0) X_0.  Checked in fp64 against
    O.newton_schulz (independent: the test carries its own p x p recursion)."""
    coeffs = coeffs or O.DEFAULT_NS_COEFFS
    X = np.random.default_rng(11).standard_normal(shape)
    X0 = X / (np.linalg.norm(X) + O.DEFAULT_NS_EPS)
    A, Q = X0 @ X0.T, np.eye(shape[0])
    for a, b, c in coeffs:
        C = a * np.eye(shape[0]) + b * A + c * (A @ A)
        Q, A = C @ Q, C @ (C @ A)
    got = Q @ X0
    want = O.newton_schulz(X, coeffs)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


def test_ns_symmetries():
    rng = np.random.default_rng(7)
    X = rng.standard_normal((16, 48))
    P = np.eye(16)[rng.permutation(16)]
    assert np.abs(O.newton_schulz(P @ X) - P @ O.newton_schulz(X)).max() < 1e-13
    # scale invariance up to the eps term: eps/||cX|| -> 0
    assert np.abs(O.newton_schulz(1e3 * X) - O.newton_schulz(1e6 * X)).max() < 1e-10


def test_ns_zero_input_is_zero():
    assert not O.newton_schulz(np.zeros((4, 6))).any()


def test_ns_singular_value_band():
    """The north star's "within the known quintic band": sigma(O) = p^(5)(sigma_hat).
    For min sigma_hat >= 3e-3 that is [0.6818, 1.2024] (SURVEY finding 2; the SPEC's
    [0.6, 1.1] is false for these coefficients)."""
    for seed in range(20):
        X = np.random.default_rng(seed).standard_normal((64, 256))
        _, xh = _quintic_closed_form(X, [], O.DEFAULT_NS_EPS)
        s = np.linalg.svd(O.newton_schulz(X), compute_uv=False)
        if xh.min() >= 3e-3:
            assert s.min() >= 0.6818 - 1e-4 and s.max() <= 1.2024 + 1e-4


# ----------------------------------------------------------------------------- the step

def _state(m, n, seed=0):
    return gen_w0(m, n, seed).astype(np.float64), np.zeros((m, n)), seed


@pytest.mark.parametrize("shape", [(64, 96), (96, 64), (48, 48)])
def test_alpha1_equals_heavy_ball_muon(shape):
    """alpha=1: M <- M+G; O=NS(M); M <- mu*M is heavy-ball Muon M <- mu*M+G."""
    m, n = shape
    cfg = O.OracleConfig(alpha=1.0)
    W1, M1, _ = _state(m, n)
    W2, M2 = W1.copy(), M1.copy()
    for t in range(100):
        G = gen_grad(m, n, 0, 0, t).astype(np.float64)
        O.dion2_step(W1, M1, G, cfg)
        O.muon_step(W2, M2, G, cfg)
    assert np.abs(W1 - W2).max() < 1e-12
    # stored states differ by the decay placement: Dion2 keeps mu*(M+G), Muon keeps mu*M+G
    assert np.abs(M1 - 0.95 * M2).max() < 1e-12 * np.abs(M2).max()


def test_muon_two_step_unroll():
    m, n = 12, 20
    cfg = O.OracleConfig()
    W, M = np.zeros((m, n)), np.zeros((m, n))
    g1, g2 = gen_grad(m, n, 0, 0, 1).astype(np.float64), gen_grad(m, n, 0, 0, 2).astype(np.float64)
    O.muon_step(W, M, g1, cfg)
    o2 = O.muon_step(W, M, g2, cfg)
    np.testing.assert_allclose(o2, O.newton_schulz_auto(0.95 * g1 + g2), atol=1e-13)


@pytest.mark.parametrize("axis", [O.AXIS_ROWS, O.AXIS_COLS, O.AXIS_AUTO])
def test_sparsity_bitwise(axis):
    m, n = 40, 24
    cfg = O.OracleConfig(alpha=0.25, axis=axis)
    W, M, _ = _state(m, n)
    M[:] = gen_grad(m, n, 0, 9, 9)
    for t in range(3):
        G = gen_grad(m, n, 0, 0, t).astype(np.float64)
        W0, M0 = W.copy(), M.copy()
        K, Omat, ax = O.dion2_step(W, M, G, cfg)
        sel = np.zeros(m if ax == O.AXIS_ROWS else n, bool)
        sel[K] = True
        unsel = ~sel
        if ax == O.AXIS_ROWS:
            assert np.array_equal(W[unsel], W0[unsel])
            assert np.array_equal(M[unsel], (M0 + G)[unsel])          # accumulation only
            assert np.array_equal(M[sel], 0.95 * (M0 + G)[sel])       # Eq. (error-feedback)
        else:
            assert np.array_equal(W[:, unsel], W0[:, unsel])
            assert np.array_equal(M[:, unsel], (M0 + G)[:, unsel])
            assert np.array_equal(M[:, sel], 0.95 * (M0 + G)[:, sel])


def test_ns_input_is_pre_decay_and_post_accumulation():
    """Alg. 1: l.2 accumulate, l.4 NS on M[K] before l.5 decays it."""
    m, n = 16, 32
    cfg = O.OracleConfig(alpha=0.5, axis=O.AXIS_ROWS)
    W, M, _ = _state(m, n)
    M[:] = gen_grad(m, n, 0, 3, 3)
    G = gen_grad(m, n, 0, 0, 0).astype(np.float64)
    Mp = M + G
    K, Omat, _ = O.dion2_step(W, M, G, cfg)
    np.testing.assert_allclose(Omat, O.newton_schulz_auto(Mp[K]), atol=1e-14)
    assert list(K) == list(O.select_l1(np.abs(Mp).sum(1), 8))


def test_mu_zero_zeroes_selected():
    m, n = 20, 30
    W, M, _ = _state(m, n)
    G = gen_grad(m, n).astype(np.float64)
    K, _, _ = O.dion2_step(W, M, G, O.OracleConfig(alpha=0.5, mu=0.0, axis=O.AXIS_ROWS))
    assert not M[K].any()


def test_zero_input_leaves_w_unchanged():
    m, n = 16, 8
    W, M, _ = _state(m, n)
    W0 = W.copy()
    K, Omat, ax = O.dion2_step(W, M, np.zeros((m, n)), O.OracleConfig(alpha=0.5))
    assert ax == O.AXIS_COLS and list(K) == [0, 1, 2, 3]
    assert np.array_equal(W, W0) and not Omat.any()


@pytest.mark.parametrize("shape,axis", [((48, 96), O.AXIS_ROWS), ((96, 48), O.AXIS_COLS), ((64, 64), O.AXIS_ROWS)])
def test_update_rms_to_rms_closed_form(shape, axis):
    """Eq. (orth-update): ||dW||_RMS->RMS = eta * ||O||_2, and for quintic NS
    ||O||_2 = max_i p^(T)(sigma_hat_i) -- measured on the FULL-size dW."""
    m, n = shape
    cfg = O.OracleConfig(alpha=0.25, axis=axis)
    W, M, _ = _state(m, n)
    W0 = W.copy()
    G = gen_grad(m, n, 0, 1, 0).astype(np.float64)
    K, Omat, ax = O.dion2_step(W, M, G, cfg)
    X = G[K] if ax == O.AXIS_ROWS else G[:, K]
    _, x = _quintic_closed_form(X, O.DEFAULT_NS_COEFFS, O.DEFAULT_NS_EPS)
    got = O.rms_to_rms_norm(W - W0)
    assert abs(got / (cfg.lr * x.max()) - 1) < 1e-10


def test_rms_to_rms_of_exact_orthonormal_is_eta():
    m, n, eta = 24, 40, 0.02
    Q, _ = np.linalg.qr(np.random.default_rng(2).standard_normal((n, m)))
    dW = eta * math.sqrt(m / n) * Q.T                    # unit spectral norm O
    assert abs(O.rms_to_rms_norm(dW) - eta) < 1e-14


def test_cols_mode_is_rows_mode_on_transpose():
    m, n = 30, 18
    cfgc = O.OracleConfig(alpha=0.25, axis=O.AXIS_COLS)
    cfgr = O.OracleConfig(alpha=0.25, axis=O.AXIS_ROWS)
    W, M, _ = _state(m, n)
    M[:] = gen_grad(m, n, 0, 5, 5)
    G = gen_grad(m, n, 0, 0, 0).astype(np.float64)
    Wt, Mt = W.T.copy(), M.T.copy()
    W0 = W.copy()
    Kc, Oc, _ = O.dion2_step(W, M, G, cfgc)
    Kr, Or, _ = O.dion2_step(Wt, Mt, G.T.copy(), cfgr)
    assert list(Kc) == list(Kr)
    np.testing.assert_allclose(Oc, Or.T, atol=1e-14)
    np.testing.assert_allclose(M, Mt.T, atol=0)
    # scale: cols uses sqrt(m/n) of W (m x n); rows-on-transpose uses sqrt(n/m)
    np.testing.assert_allclose((W - W0), (Wt.T - W0) * (m / n), atol=1e-15)


def test_force_K_and_scale_mode():
    m, n = 32, 64
    W, M, _ = _state(m, n)
    W0 = W.copy()
    G = gen_grad(m, n).astype(np.float64)
    K = np.array([1, 5, 9, 30])
    Kout, Omat, _ = O.dion2_step(W, M, G, O.OracleConfig(alpha=0.125, axis=O.AXIS_ROWS, scale_mode=1), force_K=K)
    assert list(Kout) == list(K)
    np.testing.assert_allclose(W[K] - W0[K], -0.02 * math.sqrt(4 / 64) * Omat, atol=1e-15)


def test_full_decay_ablation():
    m, n = 16, 16
    W, M, _ = _state(m, n)
    G = gen_grad(m, n).astype(np.float64)
    O.dion2_step(W, M, G, O.OracleConfig(alpha=0.5, mu=0.0, decay_mode=1))
    assert not M.any()


def test_comm_volume_golden():
    for r, c, a, b, sel, full in _read_rows("comm_volume.txt"):
        r, c, b = int(r), int(c), int(b)
        assert O.selected_bytes(r, c, float(a), O.AXIS_AUTO, b) == int(sel)
        assert O.selected_bytes(r, c, 1.0, O.AXIS_AUTO, b) == int(full)
    # owner exchange (gather + scatter back) at alpha=1 is Muon's 2*m*n*b*(P-1)/P
    assert O.comm_volume(2048, 8192, 1.0, O.AXIS_AUTO, 8, 2) == 2 * 2048 * 8192 * 2 * 7 // 8


# ----------------------------------------------------------------------------- random selection

def test_philox_known_answer_vectors():
    for row in _read_rows("philox4x32_10_kat.txt"):
        v = [int(x, 16) for x in row]
        out = O.philox4x32_10(v[0:4], v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_select_random_is_a_valid_subset_and_deterministic():
    for d in (1, 7, 64, 1000):
        for alpha in (0.125, 0.25, 1.0):
            k = O.select_count(alpha, d)
            K = O.select_random(d, k, seed=3, matrix_id=5, step=11)
            assert len(K) == k and len(set(K.tolist())) == k and list(K) == sorted(K)
            assert K.min() >= 0 and K.max() < d
            assert np.array_equal(K, O.select_random(d, k, 3, 5, 11))
    assert list(O.select_random(9, 9, 1, 2, 3)) == list(range(9))          # alpha = 1 -> all
    assert not np.array_equal(O.select_random(512, 64, 0, 0, 1), O.select_random(512, 64, 0, 0, 2))
    assert not np.array_equal(O.select_random(512, 64, 0, 0, 1), O.select_random(512, 64, 0, 1, 1))
    assert not np.array_equal(O.select_random(512, 64, 0, 0, 1), O.select_random(512, 64, 1, 0, 1))


def test_select_random_is_uniform_chi_square():
    """Every index is selected with probability k/d: chi-square over 4000 keyed draws
    (d = 64, k = 16) at significance 0.001."""
    from scipy.stats import chisquare
    d, k, n = 64, 16, 4000
    counts = np.zeros(d)
    for step in range(n):
        counts[O.select_random(d, k, seed=7, matrix_id=0, step=step)] += 1
    assert chisquare(counts).pvalue > 1e-3
    # joint uniformity of pairs: a fixed pair is co-selected with p = k(k-1)/(d(d-1))
    both = sum(1 for step in range(n) if {0, 1} <= set(O.select_random(d, k, 7, 0, step).tolist()))
    p = k * (k - 1) / (d * (d - 1))
    assert abs(both - n * p) < 4 * math.sqrt(n * p * (1 - p))


def test_dion2_step_random_uses_the_keyed_subset():
    m, n = 48, 96
    W, M, _ = _state(m, n)
    G = gen_grad(m, n).astype(np.float64)
    cfg = O.OracleConfig(alpha=0.25, select="random", seed=9, step=4)
    K, Omat, ax = O.dion2_step(W, M, G, cfg, matrix_id=3)
    assert ax == O.AXIS_ROWS and np.array_equal(K, O.select_random(m, 12, 9, 3, 4))
    np.testing.assert_allclose(Omat, O.newton_schulz_auto(G[K]), atol=1e-14)


# ----------------------------------------------------------------------------- compressed DP-sync

@pytest.mark.parametrize("shape", [(48, 96), (96, 48)])
def test_compressed_dpsync_equals_full_gradient_sync(shape):
    """syncing only M[K,:] (random K) "suffices to compute the correct parameter
    update, just as full DP-sync would": over 20 steps the replicas' W stay identical and equal
    the trajectory of a single optimizer fed the AVERAGED gradient."""
    m, n = shape
    P, steps = 3, 20
    W0 = gen_w0(m, n).astype(np.float64)
    Ws = [W0.copy() for _ in range(P)]
    Ms = [np.zeros((m, n)) for _ in range(P)]
    Wf, Mf = W0.copy(), np.zeros((m, n))
    for t in range(steps):
        cfg = O.OracleConfig(alpha=0.25, select="random", seed=17, step=t)
        Gs = [gen_grad(m, n, r, 0, t).astype(np.float64) for r in range(P)]
        K = O.dion2_step_dpsync(Ws, Ms, Gs, cfg, matrix_id=2)
        Kf, _, _ = O.dion2_step(Wf, Mf, sum(Gs) / P, cfg, matrix_id=2)
        assert np.array_equal(K, Kf)
    for r in range(P):
        assert np.array_equal(Ws[r], Ws[0])
    assert np.abs(Ws[0] - Wf).max() < 1e-12
    # the momenta diverge across replicas, but their mean is the full-sync momentum
    assert not np.array_equal(Ms[0], Ms[1])
    assert np.abs(sum(Ms) / P - Mf).max() < 1e-12 * np.abs(Mf).max()
