"""Pins of the seeded workload generator against the paper's printed circuit inventories."""
import numpy as np
import pytest

from workloads import generate, layouts, cz_period, sample_block, CZ, synthetic


@pytest.mark.parametrize("grid", ["6x7", "8x7", "8x8"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_fig4_totals(gold, grid, seed):
    """Fig. 4: total / CZ / single-qubit gate counts at depth 22."""
    r, c = map(int, grid.split("x"))
    circ = generate(r, c, 22, seed)
    cnt = circ.counts()
    g = gold("fig4.json")[grid]
    assert cnt["CZ"] == g["CZ"]
    assert cnt["SX"] + cnt["SY"] + cnt["T"] == g["single"]
    assert len(circ.gates) == g["total"]


def test_fig1_gate_count(gold):
    """Fig. 1: 27 gates in the 4x2 depth-8 circuit."""
    g = gold("fig1.json")
    circ = generate(g["rows"], g["cols"], g["depth"], 0)
    assert len(circ.gates) == g["gates_original"]


def test_layouts_partition_edges():
    """The 8 layouts partition every grid edge exactly once and each is a matching."""
    for (r, c) in [(4, 2), (6, 7), (8, 7), (8, 8), (5, 5)]:
        lay = layouts(r, c)
        all_edges = [e for v in lay.values() for e in v]
        assert len(all_edges) == len(set(all_edges)) == r * (c - 1) + (r - 1) * c
        for edges in lay.values():
            qs = [q for e in edges for q in e]
            assert len(qs) == len(set(qs))


def test_layer_rules():
    """No qubit in two gates of one layer; singles only on qubits leaving a CZ."""
    circ = generate(8, 7, 22, 3)
    period = cz_period(8, 7, 4)
    for t in range(1, 23):
        qs = []
        for (layer, kind, q0, q1) in circ.gates:
            if layer == t:
                qs += [q0] if kind != CZ else [q0, q1]
        assert len(qs) == len(set(qs))
        if t >= 2:
            prev = {q for e in period[(t - 2) % 8] for q in e}
            now = {q for e in period[(t - 1) % 8] for q in e}
            singles = {g[2] for g in circ.gates if g[0] == t and g[1] != CZ}
            assert singles == prev - now


def test_cut_schedule_only_at_8a_plus_7_8():
    """Crossing CZs only at layers 8a+7 and 8a+8 (read as 8a+7)."""
    for (r, c) in [(4, 2), (6, 7), (8, 7), (8, 8)]:
        circ = generate(r, c, 30, 0)
        hu = circ.h_upper
        layers = {g[0] for g in circ.gates if g[1] == CZ and (g[2] < hu) != (g[3] < hu)}
        assert layers and all(t % 8 in (7, 0) for t in layers)


def test_determinism_and_blocks():
    a = generate(6, 7, 22, 5).gate_array()
    b = generate(6, 7, 22, 5).gate_array()
    assert np.array_equal(a, b)
    s = sample_block(21, 1024, 7)
    assert s.dtype == np.uint64 and s.size == 1024 and np.all(np.diff(s.astype(np.int64)) > 0)
    assert int(s.max()) < (1 << 21)
    assert np.array_equal(sample_block(4, 16, 0), np.arange(16, dtype=np.uint64))
    s28 = sample_block(28, 4096, 3)
    assert s28.size == 4096 and np.all(np.diff(s28.astype(np.int64)) > 0)
    p = synthetic.porter_thomas_probs(8, 9, 10, 1)
    assert p.shape == (8, 9) and (p >= 0).all()
