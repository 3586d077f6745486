"""Shared parity helpers for the GPU suites (test infrastructure)."""
from __future__ import annotations

import numpy as np

import oracle_bindings as OB

# BASELINE.json north star: fp64 within 1e-10 relative error, normalised by
# the sum of absolute contributions per output entry.
REL_TOL = 1e-10


def assert_parity(got: np.ndarray, want: np.ndarray, norm: np.ndarray, what: str = ""):
    assert got.shape == want.shape, (got.shape, want.shape)
    err = np.abs(got - want)
    bound = REL_TOL * norm
    bad = err > bound
    if bad.any():
        i = int(np.argmax(err - bound))
        raise AssertionError(
            f"{what}: {int(bad.sum())} entries outside 1e-10*sum|contrib|; worst at {i}: "
            f"got {got[i]!r} want {want[i]!r} norm {norm[i]!r}")
    # exact zeros stay exact (empty rows, zero factors): sparsity is bit-exact
    zero = norm == 0
    assert np.all(got[zero] == 0.0), f"{what}: non-zero where every contribution is zero"


def oracle_with_norm(kind, csf, factors, ranks, residual=False):
    want = OB.oracle_nest(kind, csf, factors, ranks, residual=residual)
    norm = OB.oracle_abs_nest(kind, csf, factors, ranks, residual=residual)
    return want, norm
