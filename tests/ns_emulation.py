"""NumPy rounding emulation of the GPU's Newton-Schulz evaluation (test infrastructure).

Each function reproduces the rounding points of a kernel recipe (fp32 accumulation, 16-bit
stores) on top of fp64 matmuls, so the recipes can be compared with the fp64 oracle
(``oracle.newton_schulz``) on inputs the GPU suite cannot afford at scale.  Used by
``tests/test_ns_forms_emulation.py`` (readings R21, R23, R24).

Recipes:
  * ``direct_bf16``  -- round-1 DIRECT form: bf16 X, A, C (reading R6).
  * ``gram_bf16x``   -- round-1 Gram-space form: bf16 X0, fp16 p x p recursion, bf16 Q_T.
  * ``direct_f16``   -- current DIRECT form: X stored as fp16 with the power-of-two prescale
                        2^(15 - exponent(max row l1)), fp16 A, C, X_t (reading R24).
  * ``gram_f16``     -- current Gram-space form: the same prescaled fp16 X0, fp16 recursion,
                        restarted from an explicit X_t whenever prod |a_t| of a segment would
                        exceed 64 (reading R24): [0, 3) + [3, 5) for the default quintic.
  * ``auto_f16``     -- the AUTO choice between the two (readings R23, R25).
"""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle as O

RESTART_GROWTH = 64.0


def bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def f16(x):
    return np.asarray(x, dtype=np.float16).astype(np.float64)


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def segments(coeffs, growth=RESTART_GROWTH):
    """Restart segments [t0, t1) of the Gram-space form (reading R24)."""
    out, t0, prod = [], 0, 1.0
    for t, (a, _, _) in enumerate(coeffs):
        a = max(1.0, abs(a))
        if t > t0 and prod * a > growth:
            out.append((t0, t))
            t0, prod = t, 1.0
        prod *= a
    out.append((t0, len(coeffs)))
    return out


def prescale(X):
    """xs = 2^e with e = 15 - exponent(max row l1) (frexp convention), clamped to [-100, 64]."""
    smax = float(np.abs(X).sum(axis=1).max())
    if smax <= 0.0:
        return 1.0
    _, E = math.frexp(smax)
    return 2.0 ** max(-100, min(64, 15 - E))


def direct_bf16(X, coeffs=O.DEFAULT_NS_COEFFS, eps=O.DEFAULT_NS_EPS):
    s = 1.0 / (np.linalg.norm(X) + eps)
    Xb = bf16(X)
    for t, (a, b, c) in enumerate(coeffs):
        sc = s if t == 0 else 1.0
        A = bf16(f32((sc * sc) * (Xb @ Xb.T)))
        C = bf16(f32(c * (A @ A.T) + b * A + a * np.eye(len(A))))
        Xb = bf16(f32(sc * (C @ Xb)))
    return Xb


def gram_bf16x(X, coeffs=O.DEFAULT_NS_COEFFS, eps=O.DEFAULT_NS_EPS):
    s = 1.0 / (np.linalg.norm(X) + eps)
    Xb = bf16(X)
    p, T = Xb.shape[0], len(coeffs)
    A = f16(f32((s * s) * (Xb @ Xb.T)))
    Q = None
    for t, (a, b, c) in enumerate(coeffs):
        last = t == T - 1
        C = f32(a * np.eye(p) + b * A + c * f32(A @ A))
        C = bf16(C) if (last and Q is None) else f16(C)
        Q = C if Q is None else (bf16 if last else f16)(f32(C @ Q))
        if not last:
            A = f16(f32(C @ f16(f32(C @ A))))
    return bf16(f32(s * (Q @ Xb)))


def _x0_f16(X, eps):
    xs = prescale(X)
    s = 1.0 / (np.linalg.norm(X) + eps)
    return f16(X * xs), s / xs   # stored X0, s' (s' * X0 = s * X)


def direct_f16(X, coeffs=O.DEFAULT_NS_COEFFS, eps=O.DEFAULT_NS_EPS):
    Xh, sc = _x0_f16(X, eps)
    for t, (a, b, c) in enumerate(coeffs):
        A = f16(f32((sc * sc) * (Xh @ Xh.T)))
        C = f16(f32(c * (A @ A.T) + b * A + a * np.eye(len(A))))
        Xh = f16(f32(sc * (C @ Xh)))
        sc = 1.0
    return Xh


def gram_f16(X, coeffs=O.DEFAULT_NS_COEFFS, eps=O.DEFAULT_NS_EPS, growth=RESTART_GROWTH):
    Xh, sc = _x0_f16(X, eps)
    p = Xh.shape[0]
    for (t0, t1) in segments(coeffs, growth):
        A = f16(f32((sc * sc) * (Xh @ Xh.T)))
        Q = None
        for tl, t in enumerate(range(t0, t1)):
            a, b, c = coeffs[t]
            last = t == t1 - 1
            C = f16(f32(c * f32(A @ A) + b * A + a * np.eye(p)))
            Q = C if Q is None else f16(f32(C @ Q))
            if not last:
                A = f16(f32(C @ f16(f32(C @ A))))
        Xh = f16(f32(sc * (Q @ Xh)))
        sc = 1.0
    return Xh


GRAM_MIN_P = 64  # reading R25 (csrc/runtime.h kGramMinP)
TINY_P = 128     # reading R25 (csrc/kernels.cuh kTinyP): high-precision Gram-space NS, fp16 store of X_T


def auto_f16(X, coeffs=O.DEFAULT_NS_COEFFS, eps=O.DEFAULT_NS_EPS):
    """ns_form AUTO for one matrix (readings R23, R25): an X of at most 128 rows is evaluated in
    fp64 and stored once as fp16 (k_ns_small); else the Gram form for wide X (q >= 2p) with
    p >= 64 rows, else the direct form."""
    p, q = X.shape
    if p <= TINY_P:
        return f16(O.newton_schulz(np.asarray(X, np.float64), coeffs, eps))
    if q >= 2 * p and p >= GRAM_MIN_P:
        return gram_f16(X, coeffs, eps)
    return direct_f16(X, coeffs, eps)


def rel(got, want):
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))
