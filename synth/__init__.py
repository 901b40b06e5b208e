"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only shapes (the paper's layer sets)
and seeded random draws.  Recipe:
  W0 ~ N(0, 1/n) fp32, G_t ~ N(0, 1) fp32, M0 = 0, stream key
  (seed, matrix id, step) through NumPy's PCG64 SeedSequence.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def layer_set_1b(layers: int = 24, d: int = 2048, ffn: int = 8192) -> List[Tuple[int, int]]:
    """BASELINE configs[1]: per layer Wq, Wk, Wv, Wo (d x d), W_up (ffn x d),
    W_down (d x ffn); rows = fan-out, cols = fan-in."""
    per = [(d, d)] * 4 + [(ffn, d), (d, ffn)]
    return per * layers


def layer_set_8b(layers: int = 32) -> List[Tuple[int, int]]:
    """BASELINE configs[3]: Llama-3-8B-like shapes (GQA kv 1024, SwiGLU 14336)."""
    per = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096),
           (14336, 4096), (14336, 4096), (4096, 14336)]
    return per * layers


def rng(seed: int, mid: int, step: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, mid, step])))


def gen_w0(m: int, n: int, seed: int = 0, mid: int = 0) -> np.ndarray:
    return (rng(seed, mid, 1 << 30).standard_normal((m, n), dtype=np.float32) / np.float32(np.sqrt(n))).astype(np.float32)


def gen_grad(m: int, n: int, seed: int = 0, mid: int = 0, step: int = 0, row_scaled: bool = False) -> np.ndarray:
    """G ~ N(0,1) fp32; ``row_scaled`` multiplies row i by r_i ~ LogNormal(0, 0.5)
    (wider score gaps, selection tests only)."""
    r = rng(seed, mid, step)
    g = r.standard_normal((m, n), dtype=np.float32)
    if row_scaled:
        g *= r.lognormal(0.0, 0.5, size=(m, 1)).astype(np.float32)
    return g


def _orthonormal(r: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    q, _ = np.linalg.qr(r.standard_normal((rows, cols)))
    return q


def gen_grad_structured(m: int, n: int, seed: int = 0, mid: int = 0, step: int = 0, kind: str = "spike",
                        rank: int = 1, ratio: float = 50.0, gamma: float = 1.0) -> np.ndarray:
    """Ill-conditioned gradients (the low-rank-dominated momenta real training produces; DESIGN.md
    "Input recipe").  The singular directions U (m x r), V (n x r) are fixed per (seed, matrix),
    so they accumulate coherently in the momentum over steps; only the noise is per step.

    kind="spike": G = Z + ratio * sqrt(max(m, n)) * U V^T with r = rank equal spikes and
        Z ~ N(0, 1): sqrt(max(m, n)) is the scale of Z's singular values, so sigma_1 / median of
        G (and of a selected submatrix) is of order ``ratio``.
    kind="power": G = sqrt(max(m, n)) * U diag(i^-gamma) V^T + 1e-3 Z, r = min(m, n)."""
    fixed = rng(seed, mid, (1 << 29) + 1)
    r = rng(seed, mid, step)
    z = r.standard_normal((m, n), dtype=np.float32)
    big = float(np.sqrt(max(m, n)))
    if kind == "spike":
        rank = min(rank, m, n)
        u, v = _orthonormal(fixed, m, rank), _orthonormal(fixed, n, rank)
        g = z.astype(np.float64) + ratio * big * (u @ v.T)
    elif kind == "power":
        k = min(m, n)
        u, v = _orthonormal(fixed, m, k), _orthonormal(fixed, n, k)
        sig = np.arange(1, k + 1, dtype=np.float64) ** (-gamma)
        g = big * ((u * sig) @ v.T) + 1e-3 * z
    else:
        raise ValueError(kind)
    return g.astype(np.float32)


def gen_scores_with_ties(d: int, seed: int, n_distinct: int) -> np.ndarray:
    """Non-negative scores with many exact duplicates (tie-break tests)."""
    r = rng(seed, 0, 0)
    vals = r.random(n_distinct) * 10.0
    return vals[r.integers(0, n_distinct, size=d)]
