"""GPU parity of the multi-part partitions (Fig. 3).

``qsim_multipart_amplitudes`` (through the C-ABI) against the CPU oracle ``oracle.multipart``
(flat t-way branch sum) and the full state vector; tolerances as tests/test_gpu_parity.py
(c128 <= 1e-12 absolute, c64 <= 1e-5 of max|a|).  At sizes the oracle cannot reach, the
t-part result is compared with the bipartition path on the equivalent block (an identity that
holds at any size: both are the same amplitudes).
"""
import numpy as np
import pytest

from workloads import generate, sample_block
from oracle import statevector as SV, multipart as MP

Q = pytest.importorskip("paper_1802_06952_b200.qsim")
pytestmark = pytest.mark.gpu

PRECS = [Q.QSIM_C64, Q.QSIM_C128]
PNAME = {Q.QSIM_C64: "c64", Q.QSIM_C128: "c128"}


def assert_close(a, ref, prec, what=""):
    a = np.asarray(a, dtype=np.complex128)
    ref = np.asarray(ref, dtype=np.complex128)
    assert a.shape == ref.shape
    err = np.abs(a - ref).max()
    if prec == Q.QSIM_C128:
        assert err <= 1e-12, f"{what} c128 max abs err {err:.3e}"
    else:
        rel = err / np.abs(ref).max()
        assert rel <= 1e-5, f"{what} c64 max abs err / max|a| {rel:.3e}"


def run_multipart(circ, row_cuts, blocks, prec, opts=None):
    ctx = Q.qsim_create(prec, 0)
    try:
        for k, v in (opts or {}).items():
            Q.qsim_set_option(ctx, k, v)
        Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
        return Q.qsim_multipart_amplitudes(ctx, row_cuts, blocks, prec)
    finally:
        Q.qsim_destroy(ctx)


def _full_blocks(circ, row_cuts):
    b = MP.full_bounds(circ, row_cuts)
    return [np.arange(1 << ((b[k + 1] - b[k]) * circ.cols)) for k in range(len(b) - 1)]


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("grid,depth,row_cuts", [
    ((6, 2), 16, [1, 3]),       # 3 parts of 2 / 4 / 6 qubits, cuts at layers 5, 6, 13, 14
    ((8, 2), 8, [2, 4, 6]),     # 4 parts of 4 qubits
    ((5, 3), 12, [1, 2, 4]),    # 4 parts of 3 / 3 / 6 / 3 qubits
    ((4, 3), 16, [2]),          # t = 2 through the multi-part executor
    ((6, 2), 3, [2, 4]),        # depth 3: no cut at all (one branch per part)
    ((6, 2), 22, [2, 4]),       # a circuit ending on cut layers (7, 8, 15, 16 ... 22)
])
def test_multipart_all_amplitudes(grid, depth, row_cuts, prec):
    """Every amplitude of tiny grids against the direct state vector (small-state kernel parts)."""
    circ = generate(*grid, depth, 7)
    ref = SV.simulate(circ)
    A = run_multipart(circ, row_cuts, _full_blocks(circ, row_cuts), prec)
    assert_close(A.reshape(-1), ref, prec, f"{grid} d{depth} {row_cuts}")


@pytest.mark.parametrize("bfs", [1, 0], ids=["bfs", "dfs"])
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_multipart_tree_parts_vs_oracle(prec, bfs):
    """6x7 d5 in 3 parts of 14 qubits (tile-sweep branch trees, level-synchronous node-batched
    launches or depth-first), ragged permuted blocks vs the oracle."""
    circ = generate(6, 7, 5, 1)
    rng = np.random.default_rng(3)
    blocks = [rng.permutation(sample_block(14, n, s)) for n, s in ((37, 1), (64, 2), (29, 3))]
    ref = MP.amplitudes(circ, [2, 4], blocks)
    A = run_multipart(circ, [2, 4], blocks, prec, {Q.QSIM_OPT_BFS: bfs})
    assert_close(A, ref, prec, "6x7 d5 [2,4]")


@pytest.mark.parametrize("bfs", [1, 0], ids=["bfs", "dfs"])
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_multipart_mixed_parts_vs_oracle(prec, bfs):
    """7x4 d6 split 8 / 16 / 4 qubits: a small-state part, a tree part, a 4-qubit part; 2^8 branches."""
    circ = generate(7, 4, 6, 2)
    blocks = [np.arange(256)[::-5], sample_block(16, 41, 4), np.arange(16)]
    ref = MP.amplitudes(circ, [2, 6], blocks)
    A = run_multipart(circ, [2, 6], blocks, prec, {Q.QSIM_OPT_BFS: bfs})
    assert_close(A, ref, prec, "7x4 d6 [2,6]")


@pytest.mark.parametrize("bfs", [1, 0], ids=["bfs", "dfs"])
@pytest.mark.parametrize("row_cuts", [[2, 4, 6], [3, 5], [1, 4]])
def test_multipart_equals_bipartition_56q(row_cuts, bfs):
    """8x7 (56 qubits) d8: the t-part result equals the (oracle-checked) bipartition on the same block."""
    circ = generate(8, 7, 8, 0)
    prec = Q.QSIM_C128
    bounds = MP.full_bounds(circ, row_cuts)
    nq = [(bounds[k + 1] - bounds[k]) * 7 for k in range(len(bounds) - 1)]
    sizes = {4: [11, 9, 7, 5], 3: [13, 12, 10]}[len(nq)]
    blocks = [sample_block(nq[k], sizes[k], 10 + k) for k in range(len(nq))]
    A = run_multipart(circ, row_cuts, blocks, prec, {Q.QSIM_OPT_BFS: bfs})
    # the same amplitudes through the bipartition at row 4: split the concatenated index
    full = np.array([0], dtype=object)
    for k in range(len(nq)):
        full = np.add.outer(full * (1 << nq[k]), np.asarray(blocks[k], dtype=object))
    full = full.reshape(-1)
    xu = np.array([int(x) >> 28 for x in full], dtype=np.uint64)
    xl = np.array([int(x) & ((1 << 28) - 1) for x in full], dtype=np.uint64)
    Su, iu = np.unique(xu, return_inverse=True)
    Sl, il = np.unique(xl, return_inverse=True)
    ctx = Q.qsim_create(prec, 0)
    try:
        Q.qsim_load_circuit(ctx, 8, 7, 8, circ.gate_array(), 4)
        Q.qsim_evolve_halves(ctx, Su, Sl)
        B = Q.qsim_amplitudes(ctx, Su, Sl, prec)
    finally:
        Q.qsim_destroy(ctx)
    ref = B[iu, il].reshape(A.shape)
    assert np.abs(A - ref).max() <= 1e-12, np.abs(A - ref).max()


def test_multipart_errors():
    circ = generate(6, 2, 8, 0)
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        with pytest.raises(Q.QsimError):  # no circuit
            Q.qsim_multipart_amplitudes(ctx, [2, 4], [np.arange(4)] * 3, Q.QSIM_C64)
        Q.qsim_load_circuit(ctx, 6, 2, 8, circ.gate_array())
        for rc, bl in (([4, 2], [np.arange(4)] * 3),            # not increasing
                       ([2, 4], [np.arange(4)] * 2),            # one block missing
                       ([2, 4], [np.arange(4), np.arange(17), np.arange(4)]),   # index >= 2^4
                       ([2, 4], [np.arange(4), np.array([1, 1]), np.arange(4)])):  # duplicate
            with pytest.raises((Q.QsimError, ValueError)):
                Q.qsim_multipart_amplitudes(ctx, rc, bl, Q.QSIM_C64)
    finally:
        Q.qsim_destroy(ctx)
