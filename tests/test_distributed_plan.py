"""Distributed-half planner (§2.3.3) through the C-ABI, no GPU needed:
the layout schedule (global bits, fused local/global swaps) is host logic that runs at
qsim_load_circuit; the engine itself rejects any schedule that leaves a gate target on a global
bit, so a successful load is the check that every sweep's targets are local."""
import pytest

from workloads import generate
from oracle import partition as OP

Q = pytest.importorskip("paper_1802_06952_b200.qsim")


def _load(rows, cols, depth, world, distribute=1, seed=0, prec=None):
    circ = generate(rows, cols, depth, seed)
    ctx = Q.qsim_create(Q.QSIM_C64 if prec is None else prec, 0)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_DISTRIBUTE, distribute)
    Q.qsim_comm_init(ctx, 0, world, bytes(128))
    Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
    return ctx, circ


@pytest.mark.parametrize("grid", [(6, 7, 22), (8, 7, 22), (8, 8, 22), (6, 6, 14)])
@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("prec", [Q.QSIM_C64, Q.QSIM_C128])
def test_schedule_for_paper_grids(grid, world, prec):
    ctx, circ = _load(*grid, world, prec=prec)
    try:
        assert Q.qsim_rank_range(ctx) == (0, 1 << len(OP.cut_list(circ)))  # every rank runs every branch
    finally:
        Q.qsim_destroy(ctx)


def test_stress_schedule_has_swaps(monkeypatch):
    monkeypatch.setenv("QSIM_DIST_STRESS", "1")
    for world in (2, 4):
        ctx, _ = _load(6, 7, 14, world)
        Q.qsim_destroy(ctx)


def test_rejections():
    with pytest.raises(Q.QsimError, match="1, 2 or 4"):
        _load(8, 7, 22, 3)
    with pytest.raises(Q.QsimError, match="local qubits"):
        _load(5, 8, 14, 4)  # a 16-qubit half over 4 ranks: shards too small for a tile + swap bits
    ctx, circ = _load(8, 7, 22, 2, distribute=0)  # branch sharding: half the branches each
    try:
        assert Q.qsim_rank_range(ctx) == (0, 1 << (len(OP.cut_list(circ)) - 1))
    finally:
        Q.qsim_destroy(ctx)
