"""Planner / cost model through the C-ABI, no GPU needed.

Pins: Table 1 reproduced by qsim_eq2_time from Eq. 2's stated inputs
 and the cut counts of this repo's circuit generator (oracle.partition); Table 2
 and the 8x8 figure for the equivalent-qubit count N_e."""
import math

import pytest

from workloads import generate, CONFIGS
from oracle import partition as OP

Q = pytest.importorskip("paper_1802_06952_b200.qsim")

UNIT_S = {"s": 1.0, "min": 60.0, "h": 3600.0, "d": 86400.0}


def _sig3(x):
    return float(f"{x:.3g}")


def _n_i(qubits, depth, table):
    """n_1 = 1, n_2 = n_3 = 2, n_i = 8 / 10 / 12 for i > 3 (56 / 64 / 72 qubits)."""
    return [1.0, 2.0, 2.0] + [float(table["n_i"][str(qubits)])] * (depth - 3)


def test_table1_every_row(gold):
    t1 = gold("table1.json")
    for row in t1["rows"]:
        rows, cols = row["grid"]
        c = len(OP.cut_list(generate(rows, cols, row["depth"], 0)))
        m = 2.0 ** (c + 1)  # equivalent half circuits (Table 2 column 4)
        sec = Q.qsim_eq2_time(_n_i(row["qubits"], row["depth"], t1), m,
                              t1["t"][str(row["qubits"])], t1["s"])
        value, unit = row["printed"].split()
        assert _sig3(sec / UNIT_S[unit]) == float(value), (row, sec)


def test_table1_is_not_fitted_per_row(gold):
    """A wrong n_i rule (e.g. n_i = 8 from layer 1) or m = 2^c misses the printed rows."""
    t1 = gold("table1.json")
    row = t1["rows"][2]  # 56 qubits, depth 30, 2.62 h
    c = len(OP.cut_list(generate(8, 7, row["depth"], 0)))
    good = Q.qsim_eq2_time(_n_i(56, 30, t1), 2.0 ** (c + 1), 0.25, t1["s"])
    flat = Q.qsim_eq2_time([8.0] * 30, 2.0 ** (c + 1), 0.25, t1["s"])
    half_m = Q.qsim_eq2_time(_n_i(56, 30, t1), 2.0 ** c, 0.25, t1["s"])
    assert _sig3(good / 3600) == 2.62
    assert _sig3(flat / 3600) != 2.62 and _sig3(half_m / 3600) != 2.62


def test_eq2_edge_cases():
    assert Q.qsim_eq2_time([], 4.0, 1.0, 1.0) == 0.0
    assert Q.qsim_eq2_time([3.0], 1.0, 2.0, 4.0) == pytest.approx(1.5)
    with pytest.raises(Q.QsimError):
        Q.qsim_eq2_time([1.0], 1.0, 1.0, 0.0)


def _model(rows, cols, depth, nu=1 << 12, nl=1 << 12, gbps=5590.0):
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        circ = generate(rows, cols, depth, 0)
        Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
        return Q.qsim_cost_model(ctx, nu, nl, gbps)
    finally:
        Q.qsim_destroy(ctx)


def test_table2_equivalent_qubits(gold):
    """Table 2: N_e = 28 + c + 1 for the 8x7 grid at every printed depth breakpoint."""
    t2 = gold("table2.json")
    for d, c, ne in zip(t2["depths"], t2["cumulative_cuts"], t2["N_e"]):
        cm = _model(8, 7, d)
        assert (cm["n_cuts"], cm["N_e"]) == (c, ne), d
        assert cm["half_circuits"] == 2.0 ** (c + 1)
        assert cm["n_qubits"] == 56


def test_8x8_equivalent_qubits(gold):
    assert _model(8, 8, 22)["N_e"] == gold("table2.json")["8x8_d22_N_e"]


def test_regimes_and_tree_savings():
    """N_e <= N_m full vectors; N_m < N_e < N_r sampled blocks.  The branch tree does
    fewer layer sweeps than evolving every copy from scratch (§2.3.1)."""
    for name in ("C3", "C4", "C5"):
        r, c, d, _, _ = CONFIGS[name]
        cm = _model(r, c, d)
        assert cm["N_m"] == 34  # 183359 MiB / 8-byte amplitudes
        assert cm["regime"] == (0 if cm["N_e"] <= 34 else 1)
        assert 0 < cm["tree_sweeps"] < cm["flat_layer_evolutions"]
        assert cm["flat_layer_evolutions"] == cm["n_branches"] * 2 * d
        assert cm["lazy_gathers"] > 0
        state = 2.0 ** max(cm["h_upper"], cm["h_lower"]) * 8
        assert cm["sweep_bytes"] <= cm["tree_sweeps"] * 2 * state
        assert cm["predicted_s"] == pytest.approx(cm["sweep_bytes"] / 5590e9)
    small = _model(4, 2, 8)
    assert small["regime"] == 0 and small["tree_sweeps"] == 0  # shared-memory kernel path


def test_cost_model_errors():
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        with pytest.raises(Q.QsimError):
            Q.qsim_cost_model(ctx, 1, 1, 5590.0)  # no circuit
        circ = generate(4, 2, 8, 0)
        Q.qsim_load_circuit(ctx, 4, 2, 8, circ.gate_array())
        with pytest.raises(Q.QsimError):
            Q.qsim_cost_model(ctx, 1, 1, 0.0)
    finally:
        Q.qsim_destroy(ctx)


# ---------------------------------------------------------------- multi-part partitions (f4)
@pytest.mark.parametrize("grid,depth,row_cuts", [
    ((8, 8), 8, [3, 5]), ((8, 8), 8, [2, 4, 6]), ((8, 8), 22, [2, 4, 6]), ((8, 8), 22, [4]),
    ((8, 7), 12, [1, 4]), ((6, 2), 16, [1, 3]), ((5, 3), 12, [1, 2, 4]),
])
def test_multipart_plan_matches_oracle(grid, depth, row_cuts):
    """qsim_multipart_plan's parts and per-boundary cut counts are the oracle's (oracle.multipart)."""
    from oracle import multipart as MP
    circ = generate(*grid, depth, 0)
    bounds = MP.full_bounds(circ, row_cuts)
    cuts = MP.cut_list(circ, bounds)
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        Q.qsim_load_circuit(ctx, *grid, depth, circ.gate_array())
        p = Q.qsim_multipart_plan(ctx, row_cuts)
    finally:
        Q.qsim_destroy(ctx)
    t = len(bounds) - 1
    assert p["part_qubits"] == [(bounds[k + 1] - bounds[k]) * grid[1] for k in range(t)]
    c = [sum(1 for cu in cuts if cu[3] == j) for j in range(t - 1)]
    assert p["boundary_cuts"] == c
    cc = [0] + c + [0]
    states = sum(2.0 ** (p["part_qubits"][k] + cc[k] + cc[k + 1]) for k in range(t))
    assert p["log2_states"] == pytest.approx(math.log2(states), abs=1e-12)


def test_multipart_plan_fig3_anchor():
    """Fig. 3 caption: the 64-qubit bipartition at depth 22 'is equivalent to a 49-qubit
    circuit' — 2 halves x 2^16 copies x 2^32 amplitudes = 2^49 through the multi-part planner."""
    circ = generate(8, 8, 22, 0)
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        Q.qsim_load_circuit(ctx, 8, 8, 22, circ.gate_array())
        assert Q.qsim_multipart_plan(ctx, [4])["log2_states"] == pytest.approx(49.0, abs=1e-12)
        for bad in ([0], [8], [5, 3], [1, 2, 3, 4, 5, 6, 7, 7]):
            with pytest.raises(Q.QsimError):
                Q.qsim_multipart_plan(ctx, bad)
    finally:
        Q.qsim_destroy(ctx)
