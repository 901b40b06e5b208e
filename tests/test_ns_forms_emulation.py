"""Reading R23: rounding emulation of the two Newton-Schulz evaluation forms (-m "not gpu").

The GPU evaluates Alg. 1 l.4 either DIRECT (T iterations on the p x q matrix X, bf16
operands, reading R5) or in GRAM space (p x p fp16 recursion, X rounded to bf16 once,
include/dion2.h dion2_ns_form).  Both forms are emulated here in NumPy with the rounding
points of the kernels (fp32 accumulation, bf16 / fp16 stores) and compared with the fp64
oracle: the Gram form must be the more accurate one whenever AUTO picks it (q >= 2p), and
both must sit inside the 2e-2 bf16 gate the GPU parity tests use.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen_grad


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def _f16(x):
    return np.asarray(x, dtype=np.float16).astype(np.float64)


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def direct_form(X, coeffs=O.DEFAULT_NS_COEFFS, eps=O.DEFAULT_NS_EPS):
    """Kernel rounding of the DIRECT form: A = bf16(s^2 X X^T), C = bf16(aI + bA + cA A^T),
    X <- bf16(s C X) (s only at t = 0: X itself is stored unscaled, reading R5)."""
    s = 1.0 / (np.linalg.norm(X) + eps)
    Xb = _bf16(X)
    for t, (a, b, c) in enumerate(coeffs):
        sc = s if t == 0 else 1.0
        A = _bf16(_f32((sc * sc) * (Xb @ Xb.T)))
        C = _bf16(_f32(c * (A @ A.T) + b * A + a * np.eye(len(A))))
        Xb = _bf16(_f32(sc * (C @ Xb)))
    return Xb


def gram_form(X, coeffs=O.DEFAULT_NS_COEFFS, eps=O.DEFAULT_NS_EPS):
    """Kernel rounding of the GRAM form (dion2_api.cu append_gram_space_launches)."""
    s = 1.0 / (np.linalg.norm(X) + eps)
    Xb = _bf16(X)
    p = Xb.shape[0]
    T = len(coeffs)
    A = _f16(_f32((s * s) * (Xb @ Xb.T)))
    Q = None
    for t, (a, b, c) in enumerate(coeffs):
        last = t == T - 1
        C = _f32(a * np.eye(p) + b * A + c * _f32(A @ A))
        C = _bf16(C) if (last and Q is None) else _f16(C)
        if Q is None:
            Q = C
        else:
            Q = (_bf16 if last else _f16)(_f32(C @ Q))
        if not last:
            B = _f16(_f32(C @ A))
            A = _f16(_f32(C @ B))
    return _bf16(_f32(s * (Q @ Xb)))


def _rel(got, want):
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))


@pytest.mark.parametrize("shape", [(32, 256), (64, 512), (128, 1024), (96, 4096)])
def test_gram_form_is_more_accurate_when_auto_picks_it(shape):
    errs_d, errs_g = [], []
    for seed in range(2):
        X = gen_grad(*shape, seed=seed)
        want = O.newton_schulz(X.astype(np.float64))
        errs_d.append(_rel(direct_form(X), want))
        errs_g.append(_rel(gram_form(X), want))
    assert max(errs_g) < 0.6 * min(errs_d), (errs_g, errs_d)
    assert max(errs_g) < 1e-2 and max(errs_d) < 3e-2


def test_both_forms_inside_the_gate_on_square_x():
    X = gen_grad(192, 192, seed=3)
    want = O.newton_schulz(X.astype(np.float64))
    assert _rel(direct_form(X), want) < 2e-2
    assert _rel(gram_form(X), want) < 2e-2


@pytest.mark.parametrize("coeffs", [[(3.4445, -4.7750, 2.0315)], [(1.5, -0.5, 0.0)] * 3])
def test_gram_form_short_schedules(coeffs):
    X = gen_grad(48, 300, seed=1)
    want = O.newton_schulz(X.astype(np.float64), coeffs)
    assert _rel(gram_form(X, coeffs), want) < 1e-2


def test_gram_form_at_large_p():
    """AUTO also takes the Gram form for the 8B set's wide matrices (p = 1024 .. 4096): fp16
    Gram entries of order 1/(p sqrt(q)) reach the subnormal range there; the error must stay
    well inside the gate (emulated: p = 2048 0.35%, p = 4096 0.46%)."""
    X = gen_grad(2048, 8192, seed=0)
    want = O.newton_schulz(X.astype(np.float64))
    assert _rel(gram_form(X), want) < 1e-2
