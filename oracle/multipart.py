"""Multi-part (t-way) partitioned simulator, step by step (ORACLE — test infrastructure only).

SURVEY §8(f) f4; §3 P:114 ("dividing the circuit into three or four parts is
more effective if the circuit depth is small"), Fig. 3 (2-, 3- and 4-part
schemes of the 64-qubit grid).  The paper describes the schemes but not the algebra for
t > 2; this oracle applies Eq. 1 to every CZ that crosses a part boundary, exactly
as the bipartition does (Supp. A Eqs. 5-8), with the reading of DESIGN.md R-f4:

1. Parts are horizontal bands of rows: part k = rows [r_k, r_{k+1}), with
   0 = r_0 < r_1 < ... < r_t = rows.  Qubit q = row*cols + col lies in the part whose band
   contains its row; part k holds qubits [r_k*cols, r_{k+1}*cols) (consecutive indices).
2. A cut CZ is a CZ whose endpoints lie in different parts (grid CZs are nearest
   neighbour, so always in adjacent parts k, k+1).  The cut list is ordered by
   (layer, upper qubit) over all boundaries; branch b in [0, 2^c) takes bit
   g = (b >> (c-1-g)) & 1 for cut g (first cut = MSB, the bipartition's Q8).
3. Eq. 1: CZ = P0 (x) I + P1 (x) Z.  In branch b, cut g becomes P_{bit_g} on its upper
   endpoint (the part above the boundary) and I / Z on its lower endpoint — the
   bipartition's Q7, applied at every boundary.  A middle part therefore carries Z's
   from its upper boundary and projectors from its lower boundary.
4. Every part of every branch is simulated independently from H^{(x)n_k}|0> gate by
   gate, normalisation 2^{-n_k/2} per part (any split with product 2^{-n/2} is exact).
5. For sampled index blocks S_0..S_{t-1} (part-local indices, qubit r_k*cols = MSB):
   A[i_0, ..., i_{t-1}] = sum_b  prod_k  psi^k_b[S_k[i_k]]   (flat, ascending b, fp64),
   the t-way generalisation of "performing the tensor product, the results are finally
   added to the resultant vector".

The full index of (x_0, ..., x_{t-1}) is the concatenation x_0 x_1 ... x_{t-1} (part 0 in the
most significant bits), consistent with the bipartition's (x_u << h_l) | x_l.

Pins (tests/test_oracle_multipart.py): brute force against the full state vector on tiny
grids for t = 2, 3, 4 (every amplitude); t = 2 equals ``partition.amplitudes``; the
depth <= 3 closed form; per-part branch norms.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from . import statevector as SV


def part_of_row(bounds: Sequence[int], row: int) -> int:
    """Index k of the band [bounds[k], bounds[k+1]) holding ``row``."""
    for k in range(len(bounds) - 1):
        if bounds[k] <= row < bounds[k + 1]:
            return k
    raise ValueError(f"row {row} outside the parts")


def full_bounds(circuit, row_cuts: Sequence[int]) -> List[int]:
    """[0, r_1, ..., r_{t-1}, rows] from the t-1 interior row boundaries (strictly increasing)."""
    b = [0] + [int(r) for r in row_cuts] + [circuit.rows]
    if any(b[i] >= b[i + 1] for i in range(len(b) - 1)):
        raise ValueError("row boundaries must be strictly increasing inside (0, rows)")
    return b


def cut_list(circuit, bounds) -> List[Tuple[int, int, int, int]]:
    """Cut CZs as (layer, q_upper, q_lower, boundary j), ordered by (layer, q_upper) (step 2)."""
    cols = circuit.cols
    cuts = []
    for (layer, kind, q0, q1) in circuit.gates:
        if kind != 4:
            continue
        a, b = int(q0), int(q1)
        pa, pb = part_of_row(bounds, a // cols), part_of_row(bounds, b // cols)
        if pa != pb:
            up, lo = (a, b) if a < b else (b, a)
            cuts.append((int(layer), up, lo, min(pa, pb)))
    return sorted(cuts)


def part_gates(circuit, bounds, k: int, cuts, b: int):
    """Gate list of part k in branch b, in part-local qubit indices (step 3).

    Internal gates keep their layer order; a cut's branch gate (P0 / P1 on the upper endpoint,
    I / Z on the lower endpoint) is placed in the cut's layer after the internal gates.
    """
    cols = circuit.cols
    lo_q, hi_q = bounds[k] * cols, bounds[k + 1] * cols
    c = len(cuts)
    out = []
    for (layer, kind, q0, q1) in circuit.gates:
        qs = [int(q0)] if kind != 4 else [int(q0), int(q1)]
        if all(lo_q <= q < hi_q for q in qs):
            if kind == 4:
                out.append((layer, 4, qs[0] - lo_q, qs[1] - lo_q))
            else:
                out.append((layer, kind, qs[0] - lo_q, 0))
    for g, (layer, qu, ql, _) in enumerate(cuts):
        bit = (b >> (c - 1 - g)) & 1
        if lo_q <= qu < hi_q:
            out.append((layer, "P1" if bit else "P0", qu - lo_q, 0))
        if lo_q <= ql < hi_q and bit:
            out.append((layer, "Z", ql - lo_q, 0))
    out.sort(key=lambda g_: g_[0])  # stable: internal gates first, then branch gates, per layer
    return out


def part_state(circuit, bounds, k: int, b: int, cuts=None) -> np.ndarray:
    """Final state of part k of branch b (all 2^{n_k} amplitudes, step 4)."""
    if cuts is None:
        cuts = cut_list(circuit, bounds)
    nk = (bounds[k + 1] - bounds[k]) * circuit.cols
    return SV.run_gates(SV.initial_state(nk), nk, part_gates(circuit, bounds, k, cuts, b))


def amplitudes(circuit, row_cuts: Sequence[int], blocks: Sequence[np.ndarray]) -> np.ndarray:
    """A[i_0, ..., i_{t-1}] = sum_b prod_k psi^k_b[S_k[i_k]] (step 5; flat, every branch from scratch)."""
    bounds = full_bounds(circuit, row_cuts)
    t = len(bounds) - 1
    if len(blocks) != t:
        raise ValueError("one index block per part")
    cuts = cut_list(circuit, bounds)
    blocks = [np.asarray(S, dtype=np.int64) for S in blocks]
    A = np.zeros(tuple(S.size for S in blocks), dtype=np.complex128)
    for b in range(1 << len(cuts)):
        term = np.ones((), dtype=np.complex128)
        for k in range(t):
            term = np.multiply.outer(term, part_state(circuit, bounds, k, b, cuts)[blocks[k]])
        A += term
    return A


def split_index(circuit, row_cuts: Sequence[int], x: int) -> List[int]:
    """Part-local indices (x_0, ..., x_{t-1}) of a full basis index x (part 0 = top bits)."""
    bounds = full_bounds(circuit, row_cuts)
    out = []
    shift = circuit.n
    for k in range(len(bounds) - 1):
        nk = (bounds[k + 1] - bounds[k]) * circuit.cols
        shift -= nk
        out.append((x >> shift) & ((1 << nk) - 1))
    return out
