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
