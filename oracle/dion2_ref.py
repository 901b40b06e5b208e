"""fp64 CPU oracle for the Dion2 per-matrix optimizer step (arXiv 2512.16928).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2512_16928_b200``) never imports it, and
this module imports nothing from the product path: the two share no code.

Every function restates the paper step by step, in the paper's order and
notation, in NumPy float64.  Citations: ``P:n`` is line n of the paper text
(PAPER.md), ``S:n`` is line n of SPEC.md; the DESIGN.md section "Readings"
lists every place where the paper is silent and the reading taken here.

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``) tie each function to
something other than itself: the SVD closed form of the quintic iteration,
brute-force sorting, the alpha=1 == heavy-ball Muon identity, bitwise
sparsity, the spectral-norm closed form of the update, the paper/SPEC worked
examples in tests/golden/.  No function here is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

# Reading R1/R2: the paper names Newton-Schulz (Alg. 1
# l.4 P:186) but gives no coefficients or iteration count; we take the
# standard Muon quintic, 5 iterations, Frobenius pre-normalisation with
# eps = 1e-7.
DEFAULT_NS_COEFFS: Tuple[Tuple[float, float, float], ...] = ((3.4445, -4.7750, 2.0315),) * 5
DEFAULT_NS_EPS = 1e-7

AXIS_ROWS, AXIS_COLS, AXIS_AUTO = 0, 1, 2


@dataclass
class OracleConfig:
    """Hyper-parameters of Alg. 1.

    alpha: selection fraction (Alg. 1 "alpha-fraction")
    mu:    momentum decay factor, default 0.95 (Alg. 1 header)
    lr:    eta, default 0.02
    axis:  rows / cols / auto (auto = the shorter dimension)
    ns_coeffs, ns_eps: reading R1-R3
    decay_mode: 0 = selective decay Eq. (error-feedback);
                1 = full decay ablation M <- mu*M
    scale_mode: 0 = eta*sqrt(fan-out/fan-in) of the full W (Alg. 1 l.6);
                1 = submatrix dimensions (SPEC S:360 flag; not the paper's)
    """
    alpha: float = 0.25
    mu: float = 0.95
    lr: float = 0.02
    axis: int = AXIS_AUTO
    ns_coeffs: Sequence[Tuple[float, float, float]] = field(default_factory=lambda: list(DEFAULT_NS_COEFFS))
    ns_eps: float = DEFAULT_NS_EPS
    decay_mode: int = 0
    scale_mode: int = 0
    select: str = "l1"      # "l1" (Default) or "random"
    seed: int = 0           # random selection keying (reading R22)
    step: int = 0


def select_count(alpha: float, d: int) -> int:
    """k = max(1, round-half-up(alpha*d)), capped at d.

    Alg. 1 l.3 says only "alpha-fraction"; rounding is reading R7
    (S:209-217)."""
    if not (0.0 < alpha <= 1.0):
        raise ValueError("alpha must be in (0, 1]")
    if d < 1:
        raise ValueError("d must be >= 1")
    k = int(math.floor(alpha * d + 0.5))
    return min(d, max(1, k))


def resolve_axis(m: int, n: int, axis: int) -> int:
    """Auto selects along the shorter dimension ("we select the
    submatrix along the shorter dimension"); square -> rows (reading R8)."""
    if axis == AXIS_AUTO:
        return AXIS_ROWS if m <= n else AXIS_COLS
    if axis not in (AXIS_ROWS, AXIS_COLS):
        raise ValueError("bad axis")
    return axis


def l1_scores(M: np.ndarray, axis: int) -> np.ndarray:
    """Default Select_alpha scores: the l1 norm of every row (or column) of
    the momentum (Alg. 1 selection box)."""
    return np.abs(M).sum(axis=1) if axis == AXIS_ROWS else np.abs(M).sum(axis=0)


def select_l1(scores: np.ndarray, k: int) -> np.ndarray:
    """Top-k by (score descending, index ascending); returned ascending.

    Largest l1 norm; lower index wins ties (reading R9)."""
    d = scores.shape[0]
    order = np.lexsort((np.arange(d), -scores))  # primary: -score, secondary: index
    return np.sort(order[:k]).astype(np.int64)


_PHILOX_M0, _PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
_PHILOX_W0, _PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
_U32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Philox-4x32 with 10 rounds (Salmon et al., SC'11, "Parallel random numbers: as easy as
    1, 2, 3"), element-wise over uint64 arrays holding 32-bit lanes.  ctr: 4 arrays, key: 2."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & _U32 for x in ctr)
    k0, k1 = (np.asarray(x, dtype=np.uint64) & _U32 for x in key)
    for r in range(10):
        if r:
            k0 = (k0 + _PHILOX_W0) & _U32
            k1 = (k1 + _PHILOX_W1) & _U32
        p0 = c0 * np.uint64(_PHILOX_M0)   # exact: both factors < 2^32
        p1 = c2 * np.uint64(_PHILOX_M1)
        hi0, lo0 = p0 >> np.uint64(32), p0 & _U32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _U32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def random_keys(d: int, seed: int, matrix_id: int, step: int) -> np.ndarray:
    """One 32-bit key per index i of the selection axis: word 0 of
    Philox4x32-10(counter = (i, step_lo, step_hi, matrix_id), key = (seed_lo, seed_hi))
    (reading R22; keyed by (seed, matrix, step) like SPEC S:232)."""
    i = np.arange(d, dtype=np.uint64)
    z = np.zeros(d, dtype=np.uint64)
    out = philox4x32_10((i, z + (step & _U32), z + ((step >> 32) & _U32), z + (matrix_id & _U32)),
                        (z + (seed & _U32), z + ((seed >> 32) & _U32)))
    return out[0]


def select_random(d: int, k: int, seed: int, matrix_id: int, step: int) -> np.ndarray:
    """Random Select_alpha ("selecting uniformly at random"): the k indices
    with the smallest keys, lowest index on (probability ~2^-32) ties; ascending."""
    keys = random_keys(d, seed, matrix_id, step)
    order = np.lexsort((np.arange(d), keys))
    return np.sort(order[:k]).astype(np.int64)


def newton_schulz(X: np.ndarray, coeffs=DEFAULT_NS_COEFFS, eps: float = DEFAULT_NS_EPS) -> np.ndarray:
    """Quintic Newton-Schulz on a wide (rows <= cols) matrix.

    "Newton-Schulz iterations, which require only matrix multiplications and
    additions".  Pre-normalisation X0 = X/(||X||_F + eps) (reading R3,
    S:173); per iteration (a,b,c): A = X X^T, B = b A + c A A, X <- a X + B X
    (reading R5: algebraically the SPEC form X <- aX + b(XX^T)X + c(XX^T)^2 X,
    S:174)."""
    assert X.shape[0] <= X.shape[1], "newton_schulz expects the wide orientation"
    Y = X / (np.linalg.norm(X) + eps)
    for (a, b, c) in coeffs:
        A = Y @ Y.T
        B = b * A + c * (A @ A)
        Y = a * Y + B @ Y
    return Y


def newton_schulz_auto(X: np.ndarray, coeffs=DEFAULT_NS_COEFFS, eps: float = DEFAULT_NS_EPS) -> np.ndarray:
    """Iterate on the wide orientation, transpose back (reading R4)."""
    if X.shape[0] > X.shape[1]:
        return newton_schulz(X.T, coeffs, eps).T
    return newton_schulz(X, coeffs, eps)


def dion2_step(W: np.ndarray, M: np.ndarray, G: np.ndarray, cfg: OracleConfig,
               force_K: Optional[np.ndarray] = None, matrix_id: int = 0):
    """One step of Alg. 1 ("alpha-Dion2(G, M)") on one matrix.

    W, M: float64 [m x n], updated in place.  G: float64 [m x n].
    Returns (K, O, axis): the ascending selected indices, the orthonormalised
    submatrix in natural orientation (k x n for rows, m x k for cols), the
    resolved axis.  ``force_K`` replaces the selection (parity harness only,
    for legitimate near-ties).
    """
    m, n = W.shape
    # l.2  M <- M + G
    M += G
    # l.3  K <- Select_alpha(M)  (top l1 rows/cols)
    axis = resolve_axis(m, n, cfg.axis)
    s = l1_scores(M, axis)
    d = s.shape[0]
    k = select_count(cfg.alpha, d)
    if force_K is not None:
        K = np.asarray(force_K, dtype=np.int64)
    elif cfg.select == "random":
        K = select_random(d, k, cfg.seed, matrix_id, cfg.step)
    else:
        K = select_l1(s, k)
    # l.4  O <- NewtonSchulz(M[K, :])   (pre-decay: l.4 precedes l.5)
    X = M[K, :] if axis == AXIS_ROWS else M[:, K]
    O = newton_schulz_auto(X, cfg.ns_coeffs, cfg.ns_eps)
    # l.5  M[K, :] <- mu * M[K, :]   Eq. (error-feedback)
    if cfg.decay_mode == 0:
        if axis == AXIS_ROWS:
            M[K, :] *= cfg.mu
        else:
            M[:, K] *= cfg.mu
    else:  # full-decay ablation
        M *= cfg.mu
    # l.6  W[K, :] <- W[K, :] - eta*sqrt(fan-out/fan-in)*O  Eq. (orth-update)
    if cfg.scale_mode == 0:
        scale = cfg.lr * math.sqrt(m / n)
    else:
        sm, sn = X.shape
        scale = cfg.lr * math.sqrt(sm / sn)
    if axis == AXIS_ROWS:
        W[K, :] -= scale * O
    else:
        W[:, K] -= scale * O
    return K, O, axis


def dion2_step_dpsync(Ws, Ms, Gs, cfg: OracleConfig, matrix_id: int = 0):
    """Compressed DP-sync: P data-parallel replicas, each with its own local
    gradient G_r and its own (diverging) momentum M_r.  With a selection rule that needs no
    global state (random, "with uniform random selection, only the selected submatrix
    M[K,:] needs to be synchronized"), each replica accumulates M_r <- M_r + G_r, the shared
    K is drawn, only M_r[K,:] is averaged across replicas, and every replica then runs the
    rest of Alg. 1 on the synchronised rows (identical W updates everywhere).
    Ws, Ms: lists of per-replica float64 arrays (updated in place).  Returns K."""
    assert cfg.select == "random", "compressed DP-sync needs a selection rule without global state"
    P = len(Ws)
    m, n = Ws[0].shape
    for r in range(P):
        Ms[r] += Gs[r]
    axis = resolve_axis(m, n, cfg.axis)
    d = m if axis == AXIS_ROWS else n
    K = select_random(d, select_count(cfg.alpha, d), cfg.seed, matrix_id, cfg.step)
    if axis == AXIS_ROWS:
        avg = sum(Mr[K, :] for Mr in Ms) / P
        for Mr in Ms:
            Mr[K, :] = avg
    else:
        avg = sum(Mr[:, K] for Mr in Ms) / P
        for Mr in Ms:
            Mr[:, K] = avg
    # the rest of Alg. 1 on the synchronised rows: M += 0 (already accumulated), same K
    for r in range(P):
        dion2_step(Ws[r], Ms[r], np.zeros_like(Gs[r]), cfg, force_K=K, matrix_id=matrix_id)
    return K


def muon_step(W: np.ndarray, M: np.ndarray, G: np.ndarray, cfg: OracleConfig) -> np.ndarray:
    """Heavy-ball Muon ("O_Muon = Newton-Schulz(M)"):
    M <- mu*M + G; O = NS(M); W <- W - eta*sqrt(m/n)*O.  No Nesterov (reading R12)."""
    m, n = W.shape
    M *= cfg.mu
    M += G
    O = newton_schulz_auto(M, cfg.ns_coeffs, cfg.ns_eps)
    W -= cfg.lr * math.sqrt(m / n) * O
    return O


def rms_to_rms_norm(A: np.ndarray) -> float:
    """||A||_{RMS->RMS} = sqrt(fan-in/fan-out) * ||A||_2 for A in R^{fan-out x fan-in}
    (S:155-163)."""
    rows, cols = A.shape
    if not A.any():
        return 0.0
    return math.sqrt(cols / rows) * float(np.linalg.norm(A, 2))


def selected_bytes(m: int, n: int, alpha: float, axis: int, bytes_per_elem: int) -> int:
    """Bytes of the selected submatrix M[K,:] (or M[:,K]): the part that must be
    synchronised / moved (3.2; SPEC S:483-491 without index overhead)."""
    ax = resolve_axis(m, n, axis)
    d, o = (m, n) if ax == AXIS_ROWS else (n, m)
    return select_count(alpha, d) * o * bytes_per_elem


def comm_volume(m: int, n: int, alpha: float, axis: int, world: int, bytes_per_elem: int = 2) -> int:
    """Bytes one matrix's selected submatrix moves over the interconnect in the
    owner-compute scheme (gather to the owner, scatter O back): 2*k*o*b*(P-1)/P
    ("only the selected subset ... communicated")."""
    ax = resolve_axis(m, n, axis)
    d, o = (m, n) if ax == AXIS_ROWS else (n, m)
    k = select_count(alpha, d)
    return (2 * k * o * bytes_per_elem * (world - 1)) // world
