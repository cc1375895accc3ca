"""Partitioned simulator, step by step in the paper's order (ORACLE — test infrastructure only).

Method (§2.1, Supp. A Eqs. 5-8, §2.3.1):

1. Bipartition the qubits: upper V_1 = rows [0, cut_row) (qubits 0..h_u-1),
   lower V_2 = the rest.  Every CZ with one endpoint in each half is
   a cut CZ (E_int,t).
2. Cut list: cut CZs ordered by (layer, upper qubit).  Branch b in [0, 2^c)
   takes bit g = (b >> (c-1-g)) & 1 for cut g (first cut = MSB; Q8).
3. Eq. 1: CZ = P0 (x) I + P1 (x) Z.  In branch b, cut g becomes
   P_{bit_g} on its upper endpoint and I (bit 0) or Z (bit 1) on its lower
   endpoint (Supp. Eq. 7; Q7).  No scalar coefficients.
4. Each half of each branch is simulated independently from H^{(x)h}|0> gate
   by gate (per-half normalisation 2^{-h/2}; Q12).
5. "after sampling the data and performing the tensor product, the results
   are finally added to the resultant vector": for sampled blocks
   S_u, S_l, A[i, j] += U_b[S_u[i]] * L_b[S_l[j]], in ascending b, fp64.

Local half indices: upper qubit k -> local k (bit h_u-1-k); lower qubit k ->
local k-h_u (bit h_l-1-(k-h_u)).  Full index x = (x_u << h_l) | x_l.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from . import statevector as SV

UPPER, LOWER = 0, 1


def cut_list(circuit) -> List[Tuple[int, int, int]]:
    """Cut CZs as (layer, q_upper, q_lower), ordered by (layer, q_upper)."""
    hu = circuit.h_upper
    cuts = []
    for (layer, kind, q0, q1) in circuit.gates:
        if kind != 4:
            continue
        a, b = int(q0), int(q1)
        if (a < hu) != (b < hu):
            up, lo = (a, b) if a < hu else (b, a)
            cuts.append((int(layer), up, lo))
    return sorted(cuts)


def branch_bit(b: int, g: int, c: int) -> int:
    """Bit of cut g in branch b; the first cut is the MSB (Q8)."""
    return (b >> (c - 1 - g)) & 1


def half_gates(circuit, half: int, cuts, b: int):
    """Gate list of one half of branch b, in local qubit indices (Supp. Eq. 7).

    Internal gates keep their layer order; the cut's branch gate (P0/P1 on the
    upper endpoint, I/Z on the lower endpoint) is placed in the cut's layer.
    """
    hu = circuit.h_upper
    c = len(cuts)
    lo_q, hi_q = (0, hu) if half == UPPER else (hu, circuit.n)
    out = []
    for (layer, kind, q0, q1) in circuit.gates:
        qs = [int(q0)] if kind != 4 else [int(q0), int(q1)]
        if all(lo_q <= q < hi_q for q in qs):
            if kind == 4:
                out.append((layer, 4, qs[0] - lo_q, qs[1] - lo_q))
            else:
                out.append((layer, kind, qs[0] - lo_q, 0))
    for g, (layer, qu, ql) in enumerate(cuts):
        bit = branch_bit(b, g, c)
        if half == UPPER:
            out.append((layer, "P1" if bit else "P0", qu - lo_q, 0))
        elif bit:
            out.append((layer, "Z", ql - lo_q, 0))
    out.sort(key=lambda g_: g_[0])  # stable: internal gates first, then branch gates, per layer
    return out


def branch_state(circuit, half: int, b: int, cuts=None) -> np.ndarray:
    """Final state of one half of branch b (all 2^h amplitudes)."""
    if cuts is None:
        cuts = cut_list(circuit)
    h = circuit.h_upper if half == UPPER else circuit.h_lower
    return SV.run_gates(SV.initial_state(h), h, half_gates(circuit, half, cuts, b))


def amplitudes(circuit, S_u: np.ndarray, S_l: np.ndarray, branches=None) -> np.ndarray:
    """A[i, j] = sum_b U_b[S_u[i]] L_b[S_l[j]] (flat mode: every branch from scratch, §2.3.1).

    ``branches`` restricts the sum to a subset of b (used for sharding tests);
    default all 2^c branches in ascending order.
    """
    cuts = cut_list(circuit)
    c = len(cuts)
    S_u = np.asarray(S_u, dtype=np.int64)
    S_l = np.asarray(S_l, dtype=np.int64)
    A = np.zeros((S_u.size, S_l.size), dtype=np.complex128)
    for b in (range(1 << c) if branches is None else branches):
        U_b = branch_state(circuit, UPPER, b, cuts)
        L_b = branch_state(circuit, LOWER, b, cuts)
        A += np.outer(U_b[S_u], L_b[S_l])
    return A


def slices(circuit, S_u, S_l):
    """Gathered branch slices U[b, i] = U_b[S_u[i]], L[b, j] = L_b[S_l[j]]."""
    cuts = cut_list(circuit)
    c = len(cuts)
    S_u = np.asarray(S_u, dtype=np.int64)
    S_l = np.asarray(S_l, dtype=np.int64)
    U = np.zeros((1 << c, S_u.size), dtype=np.complex128)
    L = np.zeros((1 << c, S_l.size), dtype=np.complex128)
    for b in range(1 << c):
        U[b] = branch_state(circuit, UPPER, b, cuts)[S_u]
        L[b] = branch_state(circuit, LOWER, b, cuts)[S_l]
    return U, L
