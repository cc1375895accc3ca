"""GPU parity of the Porter-Thomas / Eq. 7 analyzer against oracle.stats.

Bar: counts (entries, zeros) bit-exact; moments within 1e-12 relative (fp64 sums in another
order); the z histogram bin-exact except for entries whose z lies within 1e-9 bins of an edge
(GPU log vs numpy log may round them to the other side); Eq. 7 expected counts within 1e-12
relative; the oracle's exact KS distance inside the GPU bracket [ks_lo, ks_hi] (1e-12 slack)."""
import numpy as np
import pytest

from workloads import generate, sample_block, synthetic
from oracle import statevector as SV, partition as OP, stats as OST

Q = pytest.importorskip("paper_1802_06952_b200.qsim")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = Q.qsim_create(Q.QSIM_C128, 0)
    yield c
    Q.qsim_destroy(c)


def check(res, ref, n_qubits, z_lo, z_hi, n_bins, mom_rtol=1e-12, ks_slack=1e-12):
    st, hist, expected = res
    assert st["count"] == ref["count"] and st["zeros"] == ref["zeros"]
    assert st["n_qubits"] == n_qubits and st["n_bins"] == n_bins
    assert st["mean_Np"] == pytest.approx(ref["mean_Np"], rel=mom_rtol, abs=1e-300)
    assert st["var_Np"] == pytest.approx(ref["var_Np"], rel=max(mom_rtol, 1e-10), abs=1e-12)
    t = (ref["z"] - z_lo) * (n_bins / (z_hi - z_lo))
    near = int(np.sum(np.abs(t - np.round(t)) < 1e-9))
    diff = np.abs(hist.astype(np.int64) - ref["hist"].astype(np.int64)).sum()
    diff += abs(int(st["below"]) - ref["below"]) + abs(int(st["above"]) - ref["above"])
    assert diff <= 2 * near, (diff, near)
    assert np.allclose(expected, ref["expected"], rtol=1e-12, atol=1e-9)
    assert st["ks_lo"] - ks_slack <= ref["ks"] <= st["ks_hi"] + ks_slack, (st["ks_lo"], ref["ks"], st["ks_hi"])
    npos = ref["count"] - ref["zeros"]
    if npos:
        # bracket width: one u bin plus the heaviest u bin's share
        assert st["ks_hi"] - st["ks_lo"] <= 2.0 ** -20 + 64.0 / npos + 1e-12


@pytest.mark.parametrize("n_u,n_l,seed", [(1024, 1000, 0), (37, 5, 1), (1, 1, 2), (4096, 4096, 3)])
def test_probs_parity(ctx, n_u, n_l, seed):
    """Synthetic Porter-Thomas blocks with zero rows / columns, ragged to C4's 2^24 entries."""
    n = 30
    p = synthetic.porter_thomas_probs(n_u, n_l, n, seed)
    z_lo, z_hi, nb = -12.0, 3.0, 150
    res = Q.qsim_porter_thomas(ctx, p, n, z_lo, z_hi, nb)
    check(res, OST.porter_thomas(p, n, z_lo, z_hi, nb), n, z_lo, z_hi, nb)
    again = Q.qsim_porter_thomas(ctx, p, n, z_lo, z_hi, nb)
    assert again[0] == res[0] and np.array_equal(again[1], res[1])  # deterministic


def test_degenerate_blocks(ctx):
    z = np.zeros(1000)
    st, hist, expected = Q.qsim_porter_thomas(ctx, z, 10, -1.0, 1.0, 8)
    assert st["zeros"] == 1000 and st["mean_Np"] == 0.0 and st["ks_lo"] == st["ks_hi"] == 0.0
    assert hist.sum() == 0 and np.all(expected == 0)
    u = np.full(64, 2.0 ** -6)  # uniform: z = 0 exactly, KS = 1 - 1/e
    for nb in (1, 4, 8192):
        res = Q.qsim_porter_thomas(ctx, u, 6, -1.0, 1.0, nb)
        check(res, OST.porter_thomas(u, 6, -1.0, 1.0, nb), 6, -1.0, 1.0, nb)
    st, hist, _ = Q.qsim_porter_thomas(ctx, u, 6, 5.0, 6.0, 3)  # every entry below the range
    assert st["below"] == 64 and hist.sum() == 0
    with pytest.raises(Q.QsimError):
        Q.qsim_porter_thomas(ctx, np.array([0.5, -0.1]), 1)
    with pytest.raises(Q.QsimError):
        Q.qsim_porter_thomas(ctx, u, 6, 1.0, 1.0, 4)


@pytest.mark.parametrize("prec", [Q.QSIM_C64, Q.QSIM_C128])
def test_block_c1(prec):
    """The evolved block (p = |a|^2 on the device) of C1 against the oracle's full state."""
    circ = generate(4, 2, 8, 0)
    p_ref = np.abs(SV.simulate(circ)) ** 2
    c = Q.qsim_create(prec, 0)
    try:
        Q.qsim_load_circuit(c, 4, 2, 8, circ.gate_array())
        Q.qsim_evolve_halves(c, np.arange(16), np.arange(16))
        res = Q.qsim_porter_thomas(c, None, 0, -8.0, 3.0, 44)
    finally:
        Q.qsim_destroy(c)
    tol = 1e-11 if prec == Q.QSIM_C128 else 1e-5
    st = res[0]
    ref = OST.porter_thomas(p_ref, 8, -8.0, 3.0, 44)
    assert st["count"] == 256 and st["n_qubits"] == 8
    assert st["mean_Np"] == pytest.approx(1.0, abs=tol * 10)  # full block: sum p = 1
    assert st["var_Np"] == pytest.approx(ref["var_Np"], rel=tol * 10)
    if prec == Q.QSIM_C128:
        check(res, ref, 8, -8.0, 3.0, 44, mom_rtol=1e-11, ks_slack=1e-9)


def test_block_tree_h14():
    """Tree-mode block (h = 14 halves, 2^7 branches) against the partitioned oracle."""
    circ = generate(4, 7, 14, 7)
    Su, Sl = sample_block(14, 300, 3), sample_block(14, 257, 4)
    p_ref = np.abs(OP.amplitudes(circ, Su, Sl)) ** 2
    c = Q.qsim_create(Q.QSIM_C128, 0)
    try:
        Q.qsim_load_circuit(c, 4, 7, 14, circ.gate_array())
        Q.qsim_evolve_halves(c, Su, Sl)
        res = Q.qsim_porter_thomas(c, None, 0, -10.0, 3.0, 52)
    finally:
        Q.qsim_destroy(c)
    check(res, OST.porter_thomas(p_ref, 28, -10.0, 3.0, 52), 28, -10.0, 3.0, 52, mom_rtol=1e-9, ks_slack=1e-9)
