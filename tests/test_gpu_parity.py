"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star; DESIGN.md "Readings" Q13/Q14):
  c128: max |a - a_ref| <= 1e-12 (absolute)
  c64 : max |a - a_ref| / max |a_ref| <= 1e-5
Bitstring indexing and branch enumeration are bit-exact; the sampler is bit-exact
given identical probabilities.
"""
import numpy as np
import pytest

from workloads import generate, sample_block, synthetic
from oracle import statevector as SV, partition as OP, reconstruct as OR, sampler as OS, stats as OST

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


def run_block(circ, S_u, S_l, prec, mode=0, budget=0, ranges=None, opts=None):
    ctx = Q.qsim_create(prec, 0)
    try:
        if mode:
            Q.qsim_set_option(ctx, Q.QSIM_OPT_MODE, mode)
        if budget:
            Q.qsim_set_option(ctx, Q.QSIM_OPT_MEM_BUDGET, budget)
        for k, v in (opts or {}).items():
            Q.qsim_set_option(ctx, k, v)
        Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
        if ranges is None:
            Q.qsim_evolve_halves(ctx, S_u, S_l)
        else:
            Q.qsim_set_blocks(ctx, S_u, S_l)
            for (b0, b1) in ranges:
                Q.qsim_evolve_range(ctx, b0, b1)
        return Q.qsim_amplitudes(ctx, S_u, S_l, prec)
    finally:
        Q.qsim_destroy(ctx)


# ------------------------------------------------------------------ C1: Fig. 1
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_c1_fig1_all_amplitudes(prec):
    """Config 1: 4x2 d8, 2 cut CZs -> 4 copies, all 256 amplitudes vs the direct state vector."""
    circ = generate(4, 2, 8, 0)
    ref = SV.simulate(circ).reshape(16, 16)
    A = run_block(circ, np.arange(16), np.arange(16), prec)
    assert_close(A, ref, prec, "C1")


# ------------------------------------------------------------------ brute force on tiny grids
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("grid,depth,seed", [((4, 3), 16, 0), ((4, 4), 22, 2), ((2, 3), 12, 3),
                                             ((5, 3), 10, 6), ((3, 4), 20, 1), ((4, 5), 9, 4)])
def test_small_grids_full(prec, grid, depth, seed):
    circ = generate(*grid, depth, seed)
    ref = SV.simulate(circ).reshape(1 << circ.h_upper, 1 << circ.h_lower)
    A = run_block(circ, np.arange(1 << circ.h_upper), np.arange(1 << circ.h_lower), prec)
    assert_close(A, ref, prec, f"{grid} d{depth}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_permuted_ragged_blocks(prec):
    """Output follows the caller's block order; ragged sizes."""
    circ = generate(4, 4, 16, 5)
    ref = SV.simulate(circ).reshape(256, 256)
    rng = np.random.default_rng(0)
    Su = rng.permutation(256)[:37]
    Sl = rng.permutation(256)[:91]
    A = run_block(circ, Su, Sl, prec)
    assert_close(A, ref[np.ix_(Su, Sl)], prec, "permuted")


# ------------------------------------------------------------------ C2: all 2^24 amplitudes
@pytest.fixture(scope="module")
def c2_reference():
    circ = generate(4, 6, 16, 0)
    return circ, SV.simulate(circ).reshape(4096, 4096)


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_c2_all_amplitudes(prec, c2_reference):
    """Config 2: 24-qubit 4x6 d16, 2^12 branches, all 2^24 amplitudes vs the full state vector."""
    circ, ref = c2_reference
    A = run_block(circ, np.arange(4096), np.arange(4096), prec)
    assert_close(A, ref, prec, "C2")
    assert abs(np.sum(np.abs(A.astype(np.complex128)) ** 2) - 1.0) < (1e-10 if prec == Q.QSIM_C128 else 1e-4)


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_c2_tree_mode_matches(prec, c2_reference):
    """The tile-sweep branch tree (forced for h = 12, c128) agrees with the direct state."""
    circ, ref = c2_reference
    if prec == Q.QSIM_C64:
        pytest.skip("c64 tiles need h >= 13")
    Su = sample_block(12, 700, 1)
    Sl = sample_block(12, 333, 2)
    A = run_block(circ, Su, Sl, prec, mode=2)
    assert_close(A, ref[np.ix_(Su.astype(np.int64), Sl.astype(np.int64))], prec, "C2 tree")


# ------------------------------------------------------------------ tree mode vs partitioned oracle
@pytest.fixture(scope="module")
def h14_reference():
    circ = generate(4, 7, 14, 7)   # h = 14, cuts at layers 7 and 8 (c = 7)
    Su = sample_block(14, 300, 3)
    Sl = sample_block(14, 257, 4)
    return circ, Su, Sl, OP.amplitudes(circ, Su, Sl)


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_tree_mode_h14(prec, h14_reference):
    circ, Su, Sl, ref = h14_reference
    assert_close(run_block(circ, Su, Sl, prec), ref, prec, "h14 tree")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("lazy,kernel", [(0, 0), (1, 1), (0, 1), (1, 0), (3, 0), (3, 1), (2, 0), (2, 2), (2, 3)])
def test_tree_mode_h14_variants(prec, lazy, kernel, h14_reference):
    """Lazy tail depth, register-only vs TMA sweep kernel (auto / 2 / 3 stages)."""
    circ, Su, Sl, ref = h14_reference
    A = run_block(circ, Su, Sl, prec, opts={Q.QSIM_OPT_LAZY_LAST: lazy, Q.QSIM_OPT_SWEEP_KERNEL: kernel})
    assert_close(A, ref, prec, f"h14 lazy={lazy} kernel={kernel}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("bfs,lazy", [(0, 2), (1, 0), (1, 1), (1, 3)])
def test_tree_mode_h14_bfs(prec, bfs, lazy, h14_reference):
    """Level-synchronous subtrees (node-batched sweeps, per-node forks) on / off, with every lazy tail."""
    circ, Su, Sl, ref = h14_reference
    A = run_block(circ, Su, Sl, prec, opts={Q.QSIM_OPT_BFS: bfs, Q.QSIM_OPT_LAZY_LAST: lazy})
    assert_close(A, ref, prec, f"h14 bfs={bfs} lazy={lazy}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("zero_skip", ["0", "1"])
def test_tree_mode_h14_zero_skip(prec, zero_skip, h14_reference, monkeypatch):
    """Known-zero tiles of projected fork children skipped (default) or read (QSIM_ZERO_SKIP=0), depth-first."""
    monkeypatch.setenv("QSIM_ZERO_SKIP", zero_skip)
    circ, Su, Sl, ref = h14_reference
    A = run_block(circ, Su, Sl, prec, opts={Q.QSIM_OPT_BFS: 0})
    assert_close(A, ref, prec, f"h14 zero_skip={zero_skip}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("branch", [0, 77])
def test_c3_branch_sweep_kernels(prec, branch, c3_circuit):
    """C3-size leaf with the TMA sweep and the register-only sweep vs the oracle."""
    circ = c3_circuit
    ref = OP.branch_state(circ, 0, branch)
    for kernel in (0, 1):
        ctx = Q.qsim_create(prec, 0)
        try:
            Q.qsim_set_option(ctx, Q.QSIM_OPT_SWEEP_KERNEL, kernel)
            Q.qsim_load_circuit(ctx, 6, 7, 22, circ.gate_array())
            got = Q.qsim_branch_state(ctx, 0, branch, 21, prec)
        finally:
            Q.qsim_destroy(ctx)
        assert_close(got, ref, prec, f"C3 kernel={kernel}")


@pytest.fixture
def perm_mode(request, monkeypatch):
    """Forces the qubit-to-bit relabelling of tree halves (engine.cu choose_perm) for one test."""
    monkeypatch.setenv("QSIM_PERM", request.param)
    return request.param


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("perm_mode", ["id", "rev", "rand", "auto"], indirect=True)
def test_tree_mode_h14_relabelled(prec, perm_mode, h14_reference):
    """Every relabelling of the half qubits to physical bits gives the same amplitudes
    (gates, fused diagonals with CZ pairs at any distance, forks, lazy tail, gathers)."""
    circ, Su, Sl, ref = h14_reference
    for lazy in (0, 2):
        assert_close(run_block(circ, Su, Sl, prec, opts={Q.QSIM_OPT_LAZY_LAST: lazy}), ref, prec,
                     f"h14 perm={perm_mode} lazy={lazy}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("perm_mode", ["rev", "rand"], indirect=True)
def test_c3_branch_state_relabelled(prec, perm_mode, c3_circuit):
    """qsim_branch_state returns the leaf in canonical bit order under any relabelling."""
    circ = c3_circuit
    for half, branch in ((0, 9000), (1, 5)):
        ctx = Q.qsim_create(prec, 0)
        try:
            Q.qsim_load_circuit(ctx, 6, 7, 22, circ.gate_array())
            got = Q.qsim_branch_state(ctx, half, branch, 21, prec)
        finally:
            Q.qsim_destroy(ctx)
        assert_close(got, OP.branch_state(circ, half, branch), prec, f"C3 perm={perm_mode} half {half}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_tree_recompute_path_and_ranges(prec, h14_reference):
    """Memory budget of 2 states forces path recomputation; split ranges accumulate."""
    circ, Su, Sl, ref = h14_reference
    amp = 16 if prec == Q.QSIM_C128 else 8
    A = run_block(circ, Su, Sl, prec, budget=2 * (1 << 14) * amp + 1,
                  ranges=[(0, 5), (5, 64), (64, 128)])
    assert_close(A, ref, prec, "h14 budget")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_lazy_tail_full_size_consistency(prec):
    """C3 size (h = 21), 256 branches: lazy tail depth 2 and 1 agree with full leaf sweeps."""
    circ = generate(6, 7, 22, 4)
    Su = sample_block(21, 512, 8)
    Sl = sample_block(21, 384, 9)
    ref = run_block(circ, Su, Sl, prec, ranges=[(0, 256)], opts={Q.QSIM_OPT_LAZY_LAST: 0})
    for lazy in (1, 3):
        A = run_block(circ, Su, Sl, prec, ranges=[(0, 256)], opts={Q.QSIM_OPT_LAZY_LAST: lazy})
        assert_close(A, ref, prec, f"lazy {lazy}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_tree_last_layer_fork(prec):
    """Circuit ending exactly at a cut layer: the pending fork diagonal is applied at the gather."""
    circ = generate(4, 7, 8, 9)
    Su = sample_block(14, 128, 5)
    Sl = sample_block(14, 128, 6)
    ref = OP.amplitudes(circ, Su, Sl)
    assert_close(run_block(circ, Su, Sl, prec), ref, prec, "fork at last layer")


# ------------------------------------------------------------------ C3-size branch spot checks
@pytest.fixture(scope="module")
def c3_circuit():
    return generate(6, 7, 22, 0)


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("half,branch", [(0, 0), (1, 16383), (0, 9000), (1, 5)])
def test_c3_branch_state(prec, half, branch, c3_circuit):
    """One leaf half-state at full C3 size (h = 21, 22 layers) vs the oracle's branch circuit."""
    circ = c3_circuit
    ctx = Q.qsim_create(prec, 0)
    try:
        Q.qsim_load_circuit(ctx, 6, 7, 22, circ.gate_array())
        got = Q.qsim_branch_state(ctx, half, branch, 21, prec)
    finally:
        Q.qsim_destroy(ctx)
    ref = OP.branch_state(circ, half, branch)
    assert_close(got, ref, prec, f"C3 branch {branch} half {half}")


# ------------------------------------------------------------------ reconstruction GEMM
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("K,M,N", [(1000, 130, 77), (16, 64, 64), (3, 1, 200), (4096, 257, 129)])
def test_branch_sum(prec, K, M, N):
    dt = np.complex128 if prec == Q.QSIM_C128 else np.complex64
    U, L = synthetic.branch_slices(K, M, N, 21, seed=K + M, dtype=dt)
    ctx = Q.qsim_create(prec, 0)
    try:
        A = Q.qsim_branch_sum(ctx, U, L, prec)
    finally:
        Q.qsim_destroy(ctx)
    ref = OR.branch_sum(U, L)   # fp64 on the same (possibly fp32) inputs
    scale = np.abs(ref).max()
    assert np.abs(A - ref).max() <= 1e-12 * max(scale, 1e-300) * 10


# ------------------------------------------------------------------ sampler
@pytest.mark.parametrize("shape", [(37, 53), (1, 9), (128, 128), (300, 7)])
def test_sampler_bit_exact(shape):
    """Given identical probabilities the GPU sampler returns the oracle's bitstrings exactly."""
    nu, nl = shape
    p = synthetic.porter_thomas_probs(nu, nl, 20, seed=nu * 1000 + nl, zero_rows=1, zero_cols=2)
    Su = sample_block(10, nu, 1)
    Sl = sample_block(10, nl, 2)
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        got, W = Q.qsim_sample_probs(ctx, p, Su, Sl, 10, 777, 50000)
    finally:
        Q.qsim_destroy(ctx)
    ref, W_ref = OS.sample(p, Su, Sl, 10, 777, 50000)
    assert W == W_ref
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_end_to_end_sampling(prec):
    """qsim_sample on the reconstructed C2 sub-block: valid outcomes, oracle-consistent."""
    circ = generate(4, 4, 22, 1)
    psi = SV.simulate(circ).reshape(256, 256)
    Su, Sl = np.arange(256), np.arange(256)
    ctx = Q.qsim_create(prec, 0)
    try:
        Q.qsim_load_circuit(ctx, 4, 4, 22, circ.gate_array())
        Q.qsim_evolve_halves(ctx, Su, Sl)
        x, W = Q.qsim_sample(ctx, 42, 20000)
    finally:
        Q.qsim_destroy(ctx)
    p = np.abs(psi) ** 2
    assert abs(W - 1.0) < 1e-5
    xr, _ = OS.sample(p, Su, Sl, 8, 42, 20000)
    assert np.mean(x == xr) > 0.995   # identical except near CDF boundaries


# ------------------------------------------------------------------ full-size properties
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("grid", [(8, 7), (6, 7), (8, 8)])
def test_depth3_closed_form_full_size(prec, grid):
    """Depth <= 3 circuits are diagonal: a(x) = 2^{-n/2} w^{m1(x)} (-1)^{m2(x)} at 42/56 qubits."""
    rows, cols = grid
    circ = generate(rows, cols, 3, 11)
    h = circ.h_upper
    Su = sample_block(h, 64, 7)
    Sl = sample_block(h, 48, 8)
    A = run_block(circ, Su, Sl, prec)
    n = circ.n
    x = (Su.astype(object)[:, None] << h) | Sl.astype(object)[None, :]
    m1 = np.zeros(x.shape, dtype=np.int64)
    m2 = np.zeros(x.shape, dtype=np.int64)
    bit = np.vectorize(lambda v, k: (v >> (n - 1 - k)) & 1, otypes=[np.int64])
    for (_, kind, q0, q1) in circ.gates:
        if kind == 3:
            m1 += bit(x, q0)
        else:
            m2 += bit(x, q0) & bit(x, q1)
    ref = 2.0 ** (-n / 2) * np.exp(1j * np.pi / 4 * m1) * (-1.0) ** m2
    assert_close(A, ref, prec, "depth-3 closed form")


@pytest.mark.slow
def test_c3_full_run_porter_thomas_and_precisions():
    """Config 3 (42q d22, 2^14 branches, 1024 x 1024 block): c64 vs c128 agree and the block is
    Porter-Thomas distributed: mean(N p) = 1, var(N p) ~ 1, KS vs Eq. 7 small."""
    circ = generate(6, 7, 22, 0)
    Su = sample_block(21, 1024, 10)
    Sl = sample_block(21, 1024, 11)
    A64 = run_block(circ, Su, Sl, Q.QSIM_C64)
    A128 = run_block(circ, Su, Sl, Q.QSIM_C128)
    assert_close(A64, A128, Q.QSIM_C64, "C3 c64 vs c128")
    Np = np.abs(A128) ** 2 * 2.0 ** 42
    assert abs(Np.mean() - 1) < 0.01
    assert abs(Np.var() - 1) < 0.1
    assert OST.ks_distance(np.log(Np.ravel())) < 0.01
