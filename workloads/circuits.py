"""Universal random grid circuits (the paper's workload), as plain gate lists.

Reading used:

* Grid ``rows x cols``, qubit ``k = row*cols + col``.
* Layer 0 is H on every qubit and is implicit (not part of the gate list, not
  counted in ``depth``; Q2).
* CZ layouts ``H_s = {((i,j),(i,j+1)) : (2i+j) mod 4 = s}`` and
  ``V_s = {((i,j),(i+1,j)) : (i+2j) mod 4 = s}``, s = 0..3.
* With the cut between rows p-1 and p (p = cut_row, default rows/2), the two
  crossing layouts are V_{(p-1) mod 4} and V_{(p+1) mod 4}; X1 is the one
  with fewer crossing edges (tie: smaller s), X2 the other; V_a < V_b are the
  two non-crossing verticals.  CZ cycle t = 1..depth uses the layout at
  position ((t-1) mod 8) of ``[H0, H2, H1, H3, V_a, V_b, X1, X2]`` so that
  cut CZs occur only at layers 8a+7, 8a+8 (P:38, P:313 read as 8a+7).
* A single-qubit slot exists at (t, q) iff t >= 2, q in CZ(t-1), q not in
  CZ(t).  The first slot on a qubit gets T; a later slot is uniform over
  {SX, SY, T} minus the qubit's previous single-qubit gate unless that gate
  was T.  Draws are consumed in order t ascending, then q ascending.

These rules reproduce the Fig. 4 totals (CZ 192/270/312, single-qubit
302/412/472) and the Fig. 1 structure (27 gates, 2 cuts) exactly; the tests
in ``tests/test_workloads.py`` pin that.

This module is an input generator only: it contains no gate arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np

SX, SY, T, CZ = 1, 2, 3, 4
KIND_NAMES = {SX: "SX", SY: "SY", T: "T", CZ: "CZ"}
NO_QUBIT = 0xFFFFFFFF

Edge = Tuple[int, int]


@dataclass
class Circuit:
    rows: int
    cols: int
    depth: int
    cut_row: int
    # gates: (layer, kind, q0, q1); q1 = NO_QUBIT unless kind == CZ.
    gates: List[Tuple[int, int, int, int]] = field(default_factory=list)
    seed: int = 0

    @property
    def n(self) -> int:
        return self.rows * self.cols

    @property
    def h_upper(self) -> int:
        return self.cut_row * self.cols

    @property
    def h_lower(self) -> int:
        return self.n - self.h_upper

    def gate_array(self) -> np.ndarray:
        """[G, 4] uint32 array (layer, kind, q0, q1) in C-ABI ``qsim_gate`` order."""
        if not self.gates:
            return np.zeros((0, 4), dtype=np.uint32)
        return np.asarray(self.gates, dtype=np.uint32).reshape(-1, 4)

    def truncated(self, depth: int) -> "Circuit":
        """The same circuit restricted to layers 1..depth."""
        return Circuit(self.rows, self.cols, depth, self.cut_row,
                       [g for g in self.gates if g[0] <= depth], self.seed)

    def counts(self) -> Dict[str, int]:
        out = {name: 0 for name in KIND_NAMES.values()}
        for g in self.gates:
            out[KIND_NAMES[g[1]]] += 1
        return out


def layouts(rows: int, cols: int) -> Dict[str, List[Edge]]:
    """The 8 CZ layouts H0..H3, V0..V3 as lists of (qubit, qubit) edges."""
    out: Dict[str, List[Edge]] = {f"H{s}": [] for s in range(4)}
    out.update({f"V{s}": [] for s in range(4)})
    for i in range(rows):
        for j in range(cols - 1):
            out[f"H{(2 * i + j) % 4}"].append((i * cols + j, i * cols + j + 1))
    for i in range(rows - 1):
        for j in range(cols):
            out[f"V{(i + 2 * j) % 4}"].append((i * cols + j, (i + 1) * cols + j))
    return out


def cz_period(rows: int, cols: int, cut_row: int) -> List[List[Edge]]:
    """The 8-layer CZ period [H0, H2, H1, H3, V_a, V_b, X1, X2] for a cut above row ``cut_row``."""
    lay = layouts(rows, cols)
    p = cut_row
    cross_s = sorted({(p - 1) % 4, (p + 1) % 4})

    def n_cross(s: int) -> int:
        return sum(1 for (a, b) in lay[f"V{s}"] if a < p * cols <= b)

    x1, x2 = sorted(cross_s, key=lambda s: (n_cross(s), s))
    va, vb = sorted(s for s in range(4) if s not in cross_s)
    order = ["H0", "H2", "H1", "H3", f"V{va}", f"V{vb}", f"V{x1}", f"V{x2}"]
    return [lay[name] for name in order]


def generate(rows: int, cols: int, depth: int, seed: int, cut_row: int | None = None) -> Circuit:
    """Generate the seeded universal random circuit of the given grid and depth."""
    if cut_row is None:
        cut_row = rows // 2
    if rows < 1 or cols < 1 or depth < 0 or not (0 < cut_row < rows or rows == 1):
        raise ValueError("bad grid / depth / cut_row")
    period = cz_period(rows, cols, cut_row)
    rng = np.random.default_rng(seed)
    n = rows * cols
    prev = [0] * n          # previous single-qubit gate per qubit (0 = none yet)
    gates: List[Tuple[int, int, int, int]] = []
    cz_prev: set = set()
    for t in range(1, depth + 1):
        edges = period[(t - 1) % 8]
        cz_now = {q for e in edges for q in e}
        for (a, b) in sorted(edges):
            gates.append((t, CZ, a, b))
        if t >= 2:
            for q in sorted(cz_prev - cz_now):
                if prev[q] == 0:
                    kind = T
                else:
                    options = [k for k in (SX, SY, T) if prev[q] == T or k != prev[q]]
                    kind = options[int(rng.integers(len(options)))]
                prev[q] = kind
                gates.append((t, kind, q, NO_QUBIT))
        cz_prev = cz_now
    return Circuit(rows, cols, depth, cut_row, gates, seed)


# Workload configurations (BASELINE.json ``configs``).
# name: (rows, cols, depth, log2 n_u, log2 n_l); None = the full half range.
CONFIGS = {
    "C1": (4, 2, 8, None, None),     # Fig. 1: 8 qubits, all 256 amplitudes
    "C2": (4, 6, 16, None, None),    # 24 qubits, all 2^24 amplitudes
    "C3": (6, 7, 22, 10, 10),        # 42 qubits, 2^20 sampled amplitudes
    "C4": (8, 7, 22, 12, 12),        # 56 qubits, 2^24 sampled amplitudes
    "C5": (8, 8, 22, 14, 14),        # 64 qubits, 2^28 sampled amplitudes
}


def config_circuit(name: str, seed: int = 0) -> Circuit:
    rows, cols, depth, _, _ = CONFIGS[name]
    return generate(rows, cols, depth, seed)
