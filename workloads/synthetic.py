"""Seeded synthetic arrays for the stand-alone boundary tests (no method arithmetic).

* ``porter_thomas_probs``: a block of probabilities with the Porter-Thomas
  shape of the paper's outputs (|a|^2 ~ Exp(mean 2^-n)), with a
  few exact zeros (rows and columns) to exercise the sampler's zero-mass rule.
* ``branch_slices``: random complex branch slices U[B, n_u], L[B, n_l] with
  the scale of real half states (|U_b[x]| ~ 2^-h/2).
"""
from __future__ import annotations

import numpy as np


def porter_thomas_probs(n_u: int, n_l: int, n_qubits: int, seed: int,
                        zero_rows: int = 1, zero_cols: int = 1) -> np.ndarray:
    rng = np.random.Generator(np.random.Philox(seed))
    p = rng.exponential(scale=2.0 ** -n_qubits, size=(n_u, n_l))
    if n_u > 2 and zero_rows:
        p[rng.choice(n_u, size=min(zero_rows, n_u - 1), replace=False), :] = 0.0
    if n_l > 2 and zero_cols:
        p[:, rng.choice(n_l, size=min(zero_cols, n_l - 1), replace=False)] = 0.0
    return np.ascontiguousarray(p, dtype=np.float64)


def branch_slices(n_branches: int, n_u: int, n_l: int, h: int, seed: int,
                  dtype=np.complex128) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.Generator(np.random.Philox(seed))
    s = 2.0 ** (-h / 2)
    U = (rng.standard_normal((n_branches, n_u)) + 1j * rng.standard_normal((n_branches, n_u))) * s
    L = (rng.standard_normal((n_branches, n_l)) + 1j * rng.standard_normal((n_branches, n_l))) * s
    return np.ascontiguousarray(U.astype(dtype)), np.ascontiguousarray(L.astype(dtype))
