"""Pins of the multi-part oracle (Fig. 3) — CPU, no GPU.

Each pin ties ``oracle.multipart`` to something other than itself: brute force against the
full state vector (every amplitude of tiny grids, t = 2, 3, 4), the bipartition oracle at
t = 2, the depth <= 3 closed form, and the branch norms of every part.
"""
import numpy as np
import pytest

from workloads import generate
from oracle import statevector as SV, partition as P, multipart as MP

OMEGA = np.exp(1j * np.pi / 4)


def _full_blocks(circ, row_cuts):
    b = MP.full_bounds(circ, row_cuts)
    return [np.arange(1 << ((b[k + 1] - b[k]) * circ.cols)) for k in range(len(b) - 1)]


@pytest.mark.parametrize("grid,depth,row_cuts", [
    ((6, 2), 10, [2, 4]),        # 3 parts of 4 qubits, cuts at layers 7, 8 on both boundaries
    ((6, 2), 16, [1, 3]),        # 3 parts of 2 / 4 / 6 qubits, cuts at layers 5, 6, 13, 14
    ((8, 2), 8, [2, 4, 6]),      # 4 parts of 4 qubits
    ((5, 3), 12, [1, 2, 4]),     # 4 parts of 3 / 3 / 6 / 3 qubits
    ((4, 3), 16, [2]),           # t = 2
])
def test_multipart_equals_full_state(grid, depth, row_cuts):
    """Eq. 1 at every boundary: the t-way branch sum is the direct state (brute force, all amplitudes)."""
    circ = generate(*grid, depth, 3)
    cuts = MP.cut_list(circ, MP.full_bounds(circ, row_cuts))
    assert len(cuts) > 0 or depth < 5
    A = MP.amplitudes(circ, row_cuts, _full_blocks(circ, row_cuts))
    ref = SV.simulate(circ)
    assert np.abs(A.reshape(-1) - ref).max() < 1e-14


def test_two_parts_equal_bipartition():
    circ = generate(4, 4, 18, 5)
    rng = np.random.default_rng(0)
    Su = np.sort(rng.choice(256, 37, replace=False))
    Sl = np.sort(rng.choice(256, 21, replace=False))
    A = MP.amplitudes(circ, [2], [Su, Sl])
    assert np.abs(A - P.amplitudes(circ, Su, Sl)).max() < 1e-15
    # the cut lists agree (same order, boundary 0)
    assert [c[:3] for c in MP.cut_list(circ, [0, 2, 4])] == [tuple(c) for c in P.cut_list(circ)]


def test_depth3_closed_form_multipart():
    """Depth <= 3 is diagonal-only: a(x) = 2^{-n/2} w^{m1(x)} (-1)^{m2(x)} (Eqs. 4, 6)."""
    circ = generate(6, 2, 3, 1)
    n = circ.n
    x = np.arange(1 << n)
    bit = lambda k: (x >> (n - 1 - k)) & 1
    m1 = np.zeros_like(x)
    m2 = np.zeros_like(x)
    for (_, kind, q0, q1) in circ.gates:
        if kind == 3:
            m1 += bit(q0)
        else:
            m2 += bit(q0) & bit(q1)
    ref = 2.0 ** (-n / 2) * OMEGA ** m1 * (-1.0) ** m2
    A = MP.amplitudes(circ, [2, 4], _full_blocks(circ, [2, 4]))
    assert np.abs(A.reshape(-1) - ref).max() < 1e-15


def test_part_norms():
    """Each part is a projected / phased unitary evolution: ||psi^k_b||^2 = 1 for parts that only
    carry Z's (part 0 carries only projectors: sum over its own cut bits of the norms is 1)."""
    circ = generate(6, 2, 16, 2)
    bounds = MP.full_bounds(circ, [2, 4])
    cuts = MP.cut_list(circ, bounds)
    c = len(cuts)
    last = len(bounds) - 2
    for b in range(1 << c):
        psi = MP.part_state(circ, bounds, last, b, cuts)  # bottom part: only I / Z
        assert abs(np.vdot(psi, psi).real - 1) < 1e-13
    # top part: the projectors of boundary 0 split the state; summing over those bits gives 1
    b0_cuts = [g for g, cu in enumerate(cuts) if cu[3] == 0]
    tot = 0.0
    for m in range(1 << len(b0_cuts)):
        b = 0
        for j, g in enumerate(b0_cuts):
            if (m >> (len(b0_cuts) - 1 - j)) & 1:
                b |= 1 << (c - 1 - g)
        psi = MP.part_state(circ, bounds, 0, b, cuts)
        tot += np.vdot(psi, psi).real
    assert abs(tot - 1) < 1e-13


def test_split_index_roundtrip():
    circ = generate(5, 3, 4, 0)
    x = 0b101_110_011001_111
    assert MP.split_index(circ, [1, 2, 4], x) == [0b101, 0b110, 0b011001, 0b111]
