"""Helpers shared by the test modules."""

import numpy as np


def seeded_A(S, L, seed, dtype=np.complex128):
    rng = np.random.default_rng(seed)
    s = np.sqrt(0.5)
    return (rng.normal(0, s, (S, L)) + 1j * rng.normal(0, s, (S, L))).astype(dtype)


def phi_gate(got, ref, scale, tol=1e-11):
    """SURVEY 8d fp64 gate: |a-b| <= tol * sum_k |c_k Re A_k| per site."""
    err = np.abs(np.asarray(got) - np.asarray(ref))
    bound = tol * np.maximum(np.asarray(scale), 1e-300)
    return bool(np.all(err <= bound)), float(np.max(err / bound))


R_IN, R_CUT = 0.8, 5.0


def seeded_shells(S, J, seed):
    """Neighbour positions [S, J, 3] uniform in volume in the 0.8-5.0 shell
    (SURVEY.md 8d); the same draw as tests/golden/make_golden_prod.py."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(S, J, 3))
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    r = (R_IN ** 3 + rng.uniform(size=(S, J)) * (R_CUT ** 3 - R_IN ** 3)) ** (1.0 / 3.0)
    return d * r[..., None]
