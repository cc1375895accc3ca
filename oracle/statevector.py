"""Full state-vector simulator, gate by gate, no fusion (ORACLE — test infrastructure only).

Implements the plain definition (SURVEY §8(c) "Plain definition"):

    a(x) = <x| L_d ... L_1 H^{(x)n} |0...0>

where L_t is the product of layer t's gates (Supp. A Eq. 4) and
layer 0 is H on every qubit.  Qubit k is bit n-1-k of the basis index
(qubit 0 = most significant bit, Q8).  Every gate is applied as its
2x2 / 4x4 matrix on the reshaped state tensor; nothing is fused.
"""
from __future__ import annotations

import numpy as np

from . import gates as G


def apply_1q(psi: np.ndarray, n: int, k: int, M: np.ndarray) -> np.ndarray:
    """psi'[.., a, ..] = sum_b M[a, b] psi[.., b, ..] on qubit k (axis of bit n-1-k)."""
    psi3 = psi.reshape(1 << k, 2, 1 << (n - k - 1))
    return np.einsum("ab,ibj->iaj", M, psi3).reshape(-1)


def apply_2q(psi: np.ndarray, n: int, k1: int, k2: int, M4: np.ndarray) -> np.ndarray:
    """Apply a 4x4 matrix on qubits (k1, k2), basis |q_k1 q_k2>."""
    if k1 == k2:
        raise ValueError("two-qubit gate on one qubit")
    if k1 > k2:  # reorder the basis so that the first axis is the lower qubit index
        perm = [0, 2, 1, 3]
        M4 = M4[np.ix_(perm, perm)]
        k1, k2 = k2, k1
    psi5 = psi.reshape(1 << k1, 2, 1 << (k2 - k1 - 1), 2, 1 << (n - k2 - 1))
    M = M4.reshape(2, 2, 2, 2)
    return np.einsum("xyuv,iujvk->ixjyk", M, psi5).reshape(-1)


def initial_state(n: int) -> np.ndarray:
    """H^{(x)n}|0...0>, computed by applying H to each qubit of |0...0>."""
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1.0
    for k in range(n):
        psi = apply_1q(psi, n, k, G.H)
    return psi


def run_gates(psi: np.ndarray, n: int, gate_list) -> np.ndarray:
    """Apply ``gate_list`` = iterable of (layer, name_or_kind, q0, q1) in order.

    Kinds: 1/'SX', 2/'SY', 3/'T', 4/'CZ', and the branch gates 'P0', 'P1', 'Z'.
    """
    for (_, kind, q0, q1) in gate_list:
        if kind in (4, "CZ"):
            psi = apply_2q(psi, n, int(q0), int(q1), G.CZ)
        else:
            psi = apply_1q(psi, n, int(q0), G.SINGLE[kind])
    return psi


def simulate(circuit) -> np.ndarray:
    """Final full state of a ``workloads.Circuit`` (all 2^n amplitudes)."""
    n = circuit.n
    gl = sorted(circuit.gates, key=lambda g: g[0])
    return run_gates(initial_state(n), n, gl)
