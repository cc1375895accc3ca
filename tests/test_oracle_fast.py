"""Pins of the multi-threaded oracle gate loop (oracle/fast.py, oracle/csrc/csim.c).

It must agree with the numpy oracle (``statevector.run_gates``, itself pinned to explicit
Kronecker operators in test_oracle.py) on every gate kind, qubit and CZ orientation, and with
closed forms that do not go through either implementation.
"""
import numpy as np
import pytest

from oracle import fast as F
from oracle import gates as G
from oracle import partition as OP
from oracle import statevector as SV
from workloads import generate

KINDS = [1, 2, 3, 4, "P0", "P1", "Z", "H"]
OMEGA = np.exp(1j * np.pi / 4)


def _random_list(rng, n, count):
    out = []
    for t in range(count):
        kind = KINDS[int(rng.integers(len(KINDS)))]
        q = int(rng.integers(n))
        q2 = int((q + 1 + rng.integers(n - 1)) % n)
        out.append((t, kind, q, q2))
    return out


@pytest.mark.parametrize("n", [2, 5, 9, 12])
@pytest.mark.parametrize("threads", [1, 3])
def test_matches_numpy_oracle(n, threads):
    rng = np.random.default_rng(n)
    for _ in range(4):
        gl = _random_list(rng, n, 60)
        psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        ref = SV.run_gates(psi.copy(), n, gl)
        got = F.run_gates(psi.copy(), n, gl, threads=threads)
        assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())


def test_single_gate_is_the_matrix_on_its_bit():
    """A one-qubit gate on qubit k mixes exactly the pairs (i, i | 2^(n-1-k)) by M[out, in]."""
    n, k = 4, 1
    for kind in (1, 2, 3, "H", "P1", "Z"):
        M = G.SINGLE[kind]
        for i0 in range(1 << n):
            if i0 & (1 << (n - 1 - k)):
                continue
            e = np.zeros(1 << n, dtype=np.complex128)
            e[i0] = 1.0
            got = F.run_gates(e, n, [(0, kind, k, 0)])
            i1 = i0 | (1 << (n - 1 - k))
            assert got[i0] == M[0, 0] and got[i1] == M[1, 0]
            assert np.count_nonzero(got) <= 2


def test_cz_negates_both_set():
    n = 5
    psi = np.ones(1 << n, dtype=np.complex128)
    F.run_gates(psi, n, [(0, 4, 3, 1)])
    x = np.arange(1 << n)
    both = ((x >> (n - 1 - 3)) & 1) & ((x >> (n - 1 - 1)) & 1)
    assert np.array_equal(psi, np.where(both == 1, -1.0, 1.0))


def test_initial_state_is_uniform():
    psi = F.initial_state(12)
    assert np.all(psi == 2.0 ** -6)
    assert np.abs(F.run_gates(F.initial_state(6), 6, [(0, "H", k, 0) for k in range(6)])[0] - 1.0) < 1e-14


def test_depth3_closed_form_h20():
    """Layers 1..3 are diagonal (T, CZ): a(x) = 2^{-h/2} w^{m1(x)} (-1)^{m2(x)} on a 20-qubit half."""
    circ = generate(4, 10, 3, 7)          # 40 qubits; upper half = 20 qubits
    assert circ.h_upper == 20
    cuts = OP.cut_list(circ)
    assert not cuts                        # no crossing CZ before layer 7
    h = circ.h_upper
    psi = F.branch_state(circ, OP.UPPER, 0, cuts)
    x = np.arange(1 << h)
    bit = lambda k: (x >> (h - 1 - k)) & 1
    m1 = np.zeros_like(x)
    m2 = np.zeros_like(x)
    for (layer, kind, q0, q1) in circ.gates:
        if q0 >= h or (kind == 4 and q1 >= h):
            continue
        if kind == 3:
            m1 += bit(q0)
        else:
            m2 += bit(q0) & bit(q1)
    ref = 2.0 ** (-h / 2) * OMEGA ** m1 * (-1.0) ** m2
    assert np.abs(psi - ref).max() < 1e-15


@pytest.mark.parametrize("half", [OP.UPPER, OP.LOWER])
def test_branch_state_matches_numpy(half):
    circ = generate(4, 5, 16, 3)
    cuts = OP.cut_list(circ)
    for b in (0, 5, (1 << len(cuts)) - 1):
        ref = OP.branch_state(circ, half, b, cuts)
        got = F.branch_state(circ, half, b, cuts, threads=2)
        assert np.abs(got - ref).max() < 1e-15
