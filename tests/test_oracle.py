"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test ties an oracle function to something other than itself: the paper's
printed worked example / tables, the CZ identity (Eq. 1), textbook identities
of the gate set, brute force via explicit Kronecker products, closed forms,
invariants and the Random123 known-answer vectors.
"""
import itertools
import math

import numpy as np
import pytest

from workloads import generate, CZ as KCZ
from oracle import gates as G, statevector as SV, partition as P, reconstruct as R
from oracle import sampler as S, stats as ST

X = np.array([[0, 1], [1, 0]], dtype=complex)
Y = np.array([[0, -1j], [1j, 0]], dtype=complex)
OMEGA = np.exp(1j * np.pi / 4)


# ---------------------------------------------------------------- gates
def test_cz_identity_eq1():
    """Eq. 1 (Supp. Eq. 2): CZ = P0 (x) I + P1 (x) Z."""
    assert np.array_equal(G.CZ, np.kron(G.P0, G.I2) + np.kron(G.P1, G.Z))
    assert np.array_equal(G.P0 + G.P1, G.I2)


def test_single_qubit_gate_identities():
    """SX, SY are principal square roots of X, Y (Q6); T_11 = (1+i)/sqrt2; H^2 = I."""
    assert np.allclose(G.SX @ G.SX, X, atol=1e-15)
    assert np.allclose(G.SY @ G.SY, Y, atol=1e-15)
    for M in (G.SX, G.SY, G.T, G.H):
        assert np.allclose(M.conj().T @ M, np.eye(2), atol=1e-15)
    # principal root: eigenvalues of SX, SY are 1 and i (principal roots of 1 and -1)
    for M in (G.SX, G.SY):
        ev = sorted(np.linalg.eigvals(M), key=lambda z: z.imag)
        assert np.allclose(ev, [1, 1j], atol=1e-14)
    assert G.T[1, 1] == pytest.approx((1 + 1j) / math.sqrt(2), abs=1e-16)
    assert np.allclose(np.linalg.matrix_power(G.T, 8), np.eye(2), atol=1e-14)
    assert np.allclose(G.H @ G.H, np.eye(2), atol=1e-15)
    assert np.allclose(G.H, (X + G.Z) / math.sqrt(2), atol=1e-16)


# ---------------------------------------------------------------- state vector
def _kron_op(n, k, M):
    return np.kron(np.kron(np.eye(1 << k), M), np.eye(1 << (n - k - 1)))


def _explicit_2q(n, k1, k2, M4):
    """Full 2^n operator of a 4x4 gate on qubits (k1, k2), built entry by entry."""
    N = 1 << n
    Op = np.zeros((N, N), dtype=complex)
    for x in range(N):
        b1 = (x >> (n - 1 - k1)) & 1
        b2 = (x >> (n - 1 - k2)) & 1
        for o1 in range(2):
            for o2 in range(2):
                y = x & ~(1 << (n - 1 - k1)) & ~(1 << (n - 1 - k2))
                y |= (o1 << (n - 1 - k1)) | (o2 << (n - 1 - k2))
                Op[y, x] += M4[2 * o1 + o2, 2 * b1 + b2]
    return Op


def test_apply_1q_matches_kron():
    rng = np.random.default_rng(0)
    n = 4
    for k in range(n):
        psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        M = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
        assert np.allclose(SV.apply_1q(psi, n, k, M), _kron_op(n, k, M) @ psi, atol=1e-13)


def test_apply_2q_matches_explicit():
    rng = np.random.default_rng(1)
    n = 4
    for k1, k2 in itertools.permutations(range(n), 2):
        psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        M4 = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
        assert np.allclose(SV.apply_2q(psi, n, k1, k2, M4), _explicit_2q(n, k1, k2, M4) @ psi,
                           atol=1e-12)


def test_initial_state_uniform():
    """H^{(x)n}|0> = 2^{-n/2} everywhere (n_1 = 1)."""
    psi = SV.initial_state(5)
    assert np.allclose(psi, 2 ** -2.5, atol=1e-16)


def test_norm_preserved():
    psi = SV.simulate(generate(4, 3, 16, 2))
    assert abs(np.vdot(psi, psi).real - 1) < 1e-13


def _closed_form_depth3(circ):
    """a(x) = 2^{-n/2} w^{m1(x)} (-1)^{m2(x)}: layers 1..3 hold only T and CZ (App. A.1; Eqs. 4, 6)."""
    n = circ.n
    x = np.arange(1 << n)
    bit = lambda k: (x >> (n - 1 - k)) & 1
    m1 = np.zeros_like(x)
    m2 = np.zeros_like(x)
    for (layer, kind, q0, q1) in circ.gates:
        assert kind in (3, 4), "depth<=3 circuits are diagonal-only"
        if kind == 3:
            m1 += bit(q0)
        else:
            m2 += bit(q0) & bit(q1)
    return 2.0 ** (-n / 2) * OMEGA ** m1 * (-1.0) ** m2


@pytest.mark.parametrize("grid", [(4, 4), (3, 5), (4, 3)])
def test_depth3_closed_form(grid):
    circ = generate(*grid, 3, 4)
    ref = _closed_form_depth3(circ)
    assert np.abs(SV.simulate(circ) - ref).max() < 1e-14
    hu, hl = circ.h_upper, circ.h_lower
    A = P.amplitudes(circ, np.arange(1 << hu), np.arange(1 << hl))
    assert np.abs(A.reshape(-1) - ref).max() < 1e-14


# ---------------------------------------------------------------- partition
def test_fig1_worked_example(gold):
    """Fig. 1 / §2.1: 2 cuts at layers 7, 8 -> 4 copies; 27 -> 112 gates;
    8 half-circuits of 4 qubits; N_e = 7; the sum of the copies is the direct 256-amplitude state."""
    g = gold("fig1.json")
    circ = generate(g["rows"], g["cols"], g["depth"], 0)
    cuts = P.cut_list(circ)
    assert [list(c) for c in cuts] == g["cuts"]
    c = len(cuts)
    assert 1 << c == g["copies"]
    assert sorted({t for t, _, _ in cuts}) == g["cut_layers"]
    total = 0
    for b in range(1 << c):
        total += len(P.half_gates(circ, P.UPPER, cuts, b)) + len(P.half_gates(circ, P.LOWER, cuts, b))
    assert total == g["gates_after_conversion"]
    assert 2 * (1 << c) == g["half_circuits"] and circ.h_upper == g["qubits_per_half"]
    assert circ.h_upper + math.log2(2 * (1 << c)) == g["N_e"]
    psi = SV.simulate(circ)
    A = P.amplitudes(circ, np.arange(16), np.arange(16))
    assert np.abs(A.reshape(-1) - psi).max() < 1e-14


@pytest.mark.parametrize("grid,depth,seed", [((4, 2), 8, 1), ((4, 3), 16, 0), ((4, 4), 22, 2),
                                             ((2, 3), 12, 3), ((4, 3), 9, 5), ((5, 3), 10, 6)])
def test_branch_sum_identity(grid, depth, seed):
    """Sum over the 2^c branches of upper (x) lower = direct state, all amplitudes (brute force)."""
    circ = generate(*grid, depth, seed)
    psi = SV.simulate(circ)
    A = P.amplitudes(circ, np.arange(1 << circ.h_upper), np.arange(1 << circ.h_lower))
    assert np.abs(A.reshape(-1) - psi).max() < 1e-13


def test_branch_norms():
    """sum_b ||U_b||^2 = 1 (projectors split the norm) and ||L_b|| = 1 (I/Z are unitary)."""
    circ = generate(4, 3, 16, 0)
    cuts = P.cut_list(circ)
    tot = 0.0
    for b in range(1 << len(cuts)):
        u = P.branch_state(circ, P.UPPER, b, cuts)
        l = P.branch_state(circ, P.LOWER, b, cuts)
        tot += np.vdot(u, u).real
        assert abs(np.vdot(l, l).real - 1) < 1e-13
    assert abs(tot - 1) < 1e-13


def test_table2_cut_counts(gold):
    """Table 2: cumulative cut CZs of the 8x7 grid and N_e = 28 + c + 1."""
    g = gold("table2.json")
    full = generate(8, 7, max(g["depths"]), 0)
    for d, cum, ne in zip(g["depths"], g["cumulative_cuts"], g["N_e"]):
        c = len(P.cut_list(full.truncated(d)))
        assert c == cum
        assert 28 + c + 1 == ne


def test_8x8_prefix_and_ne(gold):
    """§2.3.2: 8 cuts in the first 14 layers -> 256 prefixes; Fig. 3: 8x8 d22 ~ 49 qubits."""
    g = gold("table2.json")
    circ = generate(8, 8, 22, 0)
    assert len(P.cut_list(circ.truncated(14))) == g["8x8_cuts_by_layer_14"]
    assert 32 + len(P.cut_list(circ)) + 1 == g["8x8_d22_N_e"]


def test_reconstruct_branch_sum_matches_direct():
    """branch_sum over oracle slices reproduces the direct state on sampled blocks."""
    circ = generate(4, 3, 16, 7)
    psi = SV.simulate(circ).reshape(1 << circ.h_upper, 1 << circ.h_lower)
    Su = np.array([0, 3, 5, 63, 17])
    Sl = np.array([1, 2, 40, 9])
    U, L = P.slices(circ, Su, Sl)
    A = R.branch_sum(U, L)
    assert np.abs(A - psi[np.ix_(Su, Sl)]).max() < 1e-14
    p = R.probabilities(A)
    assert np.allclose(p, np.abs(psi[np.ix_(Su, Sl)]) ** 2, atol=1e-15)


# ---------------------------------------------------------------- sampler
def test_philox_kat(gold):
    for v in gold("philox_kat.json")["vectors"]:
        out = S.philox4x32_10([int(x, 16) for x in v["ctr"]], [int(x, 16) for x in v["key"]])
        assert [int(o) for o in out] == [int(x, 16) for x in v["out"]]


def test_uniforms_range_and_formula():
    u = S.uniforms(12345, 1000)
    assert (u >= 0).all() and (u < 1).all()
    o0, o1, _, _ = S.philox4x32_10((7, 0, 0, 0), (12345, 0))
    assert u[7] == ((int(o1) << 32 | int(o0)) >> 11) * 2.0 ** -53
    assert abs(u.mean() - 0.5) < 0.05


def test_cumsum_is_sequential():
    """np.cumsum is the left-to-right sequential sum the sampler contract defines."""
    rng = np.random.default_rng(3)
    for _ in range(5):
        a = rng.exponential(size=1001) * 10.0 ** rng.integers(-20, 0, size=1001)
        seq = list(itertools.accumulate(a.tolist()))
        assert np.array_equal(np.cumsum(a), np.array(seq))


def test_sampler_hand_computed():
    """p = [[0, 1], [3, 0]], W = 4: t = 4u < 1 -> (0, 1); t >= 1 -> (1, 0)."""
    p = np.array([[0.0, 1.0], [3.0, 0.0]])
    rows, cols, W = S.draw(p, 99, 400)
    u = S.uniforms(99, 400)
    assert W == 4.0
    exp_rows = (4 * u >= 1).astype(int)
    assert np.array_equal(rows, exp_rows)
    assert np.array_equal(cols, 1 - exp_rows)
    x, _ = S.sample(p, np.array([5, 9]), np.array([2, 6]), 3, 99, 400)
    assert set(x.tolist()) <= {(5 << 3) | 6, (9 << 3) | 2}


def test_sampler_distribution_and_zero_mass():
    from workloads import synthetic
    p = synthetic.porter_thomas_probs(6, 7, 6, 11, zero_rows=1, zero_cols=2)
    rows, cols, W = S.draw(p, 5, 200000)
    assert (p[rows, cols] > 0).all()
    counts = np.zeros_like(p)
    np.add.at(counts, (rows, cols), 1)
    expected = p / W * rows.size
    m = expected > 0
    chi2 = (((counts - expected) ** 2)[m] / expected[m]).sum()
    dof = m.sum() - 1
    assert chi2 < dof + 6 * math.sqrt(2 * dof)


# ---------------------------------------------------------------- stats
def test_gumbel_eq7():
    """Eq. 7 at alpha = 1: f(0) = e^{-1}, mode at 0, integrates to 1; Porter-Thomas KS."""
    assert ST.gumbel_pdf(0.0) == pytest.approx(math.exp(-1), rel=1e-15)
    z = np.linspace(-40, 6, 400001)
    assert abs(np.trapezoid(ST.gumbel_pdf(z), z) - 1) < 1e-6
    assert abs(z[np.argmax(ST.gumbel_pdf(z))]) < 1e-3
    rng = np.random.default_rng(0)
    Np = rng.exponential(size=200000)
    assert ST.ks_distance(np.log(Np)) < 0.005


def test_ks_distance_vs_scipy():
    """ks_distance against scipy's one-sample KS with gumbel_l, whose CDF is 1 - exp(-e^z):
    an independent implementation of both the statistic and Eq. 7's CDF."""
    from scipy import stats as sps
    rng = np.random.default_rng(3)
    for z in (np.log(rng.exponential(size=5000)), rng.normal(size=777), np.array([0.0]), np.array([-1.0, 2.0])):
        assert ST.ks_distance(z) == pytest.approx(sps.kstest(z, "gumbel_l").statistic, abs=1e-14)
    assert np.allclose(ST.gumbel_cdf(np.linspace(-30, 3, 99)), sps.gumbel_l.cdf(np.linspace(-30, 3, 99)),
                       rtol=1e-13, atol=1e-300)


def test_porter_thomas_analyzer_oracle():
    """f1 quantities: Exp(1)-distributed N p gives mean ~ var ~ 1; histogram plus
    out-of-range counts cover every p > 0 entry; expected counts equal n_pos * P(bin) from
    scipy's gumbel_l; the degenerate uniform block p = 1/N has z = 0, var 0 and KS distance
    max(F(0), 1 - F(0)) = 1 - 1/e."""
    from scipy import stats as sps
    n = 20
    rng = np.random.default_rng(11)
    p = rng.exponential(scale=2.0 ** -n, size=1 << 16)
    p[:5] = 0.0
    r = ST.porter_thomas(p, n, -6.0, 2.0, 64)
    assert r["count"] == 1 << 16 and r["zeros"] == 5
    assert abs(r["mean_Np"] - 1) < 0.02 and abs(r["var_Np"] - 1) < 0.05
    assert int(r["hist"].sum()) + r["below"] + r["above"] == (1 << 16) - 5
    P = np.diff(sps.gumbel_l.cdf(np.linspace(-6.0, 2.0, 65)))
    assert np.allclose(r["expected"], ((1 << 16) - 5) * P, rtol=1e-10)
    assert r["ks"] < 0.01
    # chi-square of the histogram against Eq. 7's counts
    e = r["expected"]
    m = e > 20
    chi2 = float(np.sum((r["hist"][m] - e[m]) ** 2 / e[m]))
    assert chi2 < m.sum() + 6 * math.sqrt(2 * m.sum())
    u = ST.porter_thomas(np.full(64, 2.0 ** -6), 6, -1.0, 1.0, 4)
    assert u["var_Np"] == 0.0 and u["mean_Np"] == 1.0
    assert list(u["hist"]) == [0, 0, 64, 0]
    assert u["ks"] == pytest.approx(1 - math.exp(-1), abs=1e-15)


@pytest.mark.parametrize("grid", [(4, 3, 12, 5), (4, 4, 16, 2)])
def test_rzz_both_endpoints_z(grid):
    """DESIGN.md R-zz: per cut CZ = sum_{a,b} H_ab Z^a (x) Z^b with H = [[1,1],[1,-1]]/2, so with Z on BOTH
    endpoints of a block's free cuts (the block's fixed cuts keep P_b (x) Z^b) and the lower rows of each
    block Walsh-Hadamard transformed over the free bits (1/2 per bit), the sum over all blocks of
    sum_a V_a (x) (H L)_a is the direct state — and any split of the sum over a (half pairs over two
    ranks) is a partition of the same terms."""
    rows, cols, d, seed = grid
    circ = generate(rows, cols, d, seed)
    cuts = P.cut_list(circ)
    c, hu = len(cuts), circ.h_upper
    m = min(c, 3)  # free cuts per block: the last m

    def half(half_i, b):
        lo, hi = (0, hu) if half_i == 0 else (hu, circ.n)
        out = [(l, k, q0 - lo, (q1 - lo) if k == 4 else 0) for (l, k, q0, q1) in circ.gates
               if all(lo <= q < hi for q in ([q0] if k != 4 else [q0, q1]))]
        for g, (layer, qu, ql) in enumerate(cuts):
            bit = (b >> (c - 1 - g)) & 1
            q = (qu if half_i == 0 else ql) - lo
            if half_i == 0 and g < c - m:
                out.append((layer, "P1" if bit else "P0", q, 0))
            elif bit:
                out.append((layer, "Z", q, 0))
        return sorted(out, key=lambda g_: g_[0])

    hl = circ.n - hu
    A = np.zeros((1 << hu, 1 << hl), dtype=np.complex128)
    split = np.zeros_like(A)
    for blk in range(1 << (c - m)):
        bs = [(blk << m) | a for a in range(1 << m)]
        V = np.array([SV.run_gates(SV.initial_state(hu), hu, half(0, b)) for b in bs])
        L = np.array([SV.run_gates(SV.initial_state(hl), hl, half(1, b)) for b in bs])
        for t_ in range(m):  # Walsh-Hadamard over the free bits, 1/2 per bit
            L = L.reshape(-1, 2, 1 << t_, 1 << hl)
            L = np.stack([(L[:, 0] + L[:, 1]) / 2, (L[:, 0] - L[:, 1]) / 2], axis=1).reshape(1 << m, 1 << hl)
        A += V.T @ L
        split += V[: len(bs) // 2].T @ L[: len(bs) // 2]
        split += V[len(bs) // 2:].T @ L[len(bs) // 2:]
    ref = SV.simulate(circ)
    assert np.abs(A.reshape(-1) - ref).max() < 1e-14
    assert np.abs(split.reshape(-1) - ref).max() < 1e-14


@pytest.mark.parametrize("grid", [(4, 3, 12, 5), (4, 4, 16, 2)])
def test_eq1_read_both_ways(grid):
    """DESIGN.md R6': CZ = P0 (x) I + P1 (x) Z = I (x) P0 + Z (x) P1, so with the projector put on the
    lower endpoint of any subset of the cuts the branch sum is still the direct state (Eq. 1)."""
    rows, cols, d, seed = grid
    circ = generate(rows, cols, d, seed)
    cuts = P.cut_list(circ)
    c, hu = len(cuts), circ.h_upper
    rng = np.random.default_rng(seed)
    p_upper = rng.integers(0, 2, c)
    assert 0 < p_upper.sum() < c or c < 2

    def half(half_i, b):
        lo, hi = (0, hu) if half_i == 0 else (hu, circ.n)
        out = [(l, k, q0 - lo, (q1 - lo) if k == 4 else 0) for (l, k, q0, q1) in circ.gates
               if all(lo <= q < hi for q in ([q0] if k != 4 else [q0, q1]))]
        for g, (layer, qu, ql) in enumerate(cuts):
            bit = (b >> (c - 1 - g)) & 1
            proj = bool(p_upper[g]) == (half_i == 0)
            q = (qu if half_i == 0 else ql) - lo
            if proj:
                out.append((layer, "P1" if bit else "P0", q, 0))
            elif bit:
                out.append((layer, "Z", q, 0))
        return sorted(out, key=lambda g_: g_[0])

    hl = circ.n - hu
    A = np.zeros((1 << hu, 1 << hl), dtype=np.complex128)
    for b in range(1 << c):
        U = SV.run_gates(SV.initial_state(hu), hu, half(0, b))
        L = SV.run_gates(SV.initial_state(hl), hl, half(1, b))
        A += np.outer(U, L)
    assert np.abs(A.reshape(-1) - SV.simulate(circ)).max() < 1e-14
