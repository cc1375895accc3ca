"""Full-size parity: the production path at h = 14 (many tiles per CTA), 24, 28 and 32 against the
CPU oracle evolved branch by branch (VERDICT r01 "Next round" 1, last pins: "CPU
evolution of individual branches of a 28- or 32-qubit half, compared with the GPU leaf";
PAPER.md P:34-36 / P:175: the method is exact, every copy is a plain half-circuit).

The oracle side is ``oracle.fast`` (the numpy oracle's gate lists, applied by a plain C + OpenMP
loop; pinned in test_oracle_fast.py).  The GPU side goes through ``qsim_branch_values``: one
branch, the sampled indices as the block, i.e. the same deferred-fork tree, lazy tail and gathers
as ``qsim_evolve_range``.  Tolerances as test_gpu_parity.py (BASELINE north_star; R12/R13).
"""
import os

import numpy as np
import pytest

from oracle import fast as F
from oracle import partition as OP
from workloads import generate, sample_block

Q = pytest.importorskip("paper_1802_06952_b200.qsim")
pytestmark = pytest.mark.gpu

PRECS = [Q.QSIM_C64, Q.QSIM_C128]
PNAME = {Q.QSIM_C64: "c64", Q.QSIM_C128: "c128"}


def errs(a, ref):
    a = np.asarray(a, dtype=np.complex128)
    ref = np.asarray(ref, dtype=np.complex128)
    d = np.abs(a - ref).max()
    return d, d / np.abs(ref).max(), d / np.sqrt(np.mean(np.abs(ref) ** 2))


def assert_close(a, ref, prec, what=""):
    d, rel, rms = errs(a, ref)
    if prec == Q.QSIM_C128:
        assert d <= 1e-12, f"{what} c128 max abs err {d:.3e} (/rms {rms:.2e})"
    else:
        assert rel <= 1e-5, f"{what} c64 max abs err / max|a| {rel:.3e} (/rms {rms:.2e})"


def make_ctx(prec, circ, opts=None):
    ctx = Q.qsim_create(prec, 0)
    for k, v in (opts or {}).items():
        Q.qsim_set_option(ctx, k, v)
    Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
    return ctx


def oracle_values(circ, half, b, idx_list):
    """The oracle's leaf of (half, b) at each index array of idx_list (the state is dropped)."""
    psi = F.branch_state(circ, half, b)
    out = [psi[np.asarray(ix, dtype=np.int64)].copy() for ix in idx_list]
    del psi
    return out


def index_sample(h, n, seed):
    ix = sample_block(h, n, seed).astype(np.uint64)
    return np.concatenate([ix, np.array([0, (1 << h) - 1, (1 << h) - 2], dtype=np.uint64)])


# ------------------------------------------------------------------ h = 14, 22 layers, many tiles per CTA
@pytest.fixture(scope="module")
def d22_h14():
    """4x7 grid, depth 22 (two cut periods, c = 14): ragged branch ranges vs the oracle's sum."""
    circ = generate(4, 7, 22, 11)
    cuts = OP.cut_list(circ)
    Su = sample_block(14, 300, 21)
    Sl = sample_block(14, 257, 22)
    ranges = [(0, 64), (1000, 1100), ((1 << len(cuts)) - 37, 1 << len(cuts))]
    A = np.zeros((Su.size, Sl.size), dtype=np.complex128)
    for (b0, b1) in ranges:
        for b in range(b0, b1):
            u = F.branch_state(circ, OP.UPPER, b, cuts)[Su.astype(np.int64)]
            l = F.branch_state(circ, OP.LOWER, b, cuts)[Sl.astype(np.int64)]
            A += np.outer(u, l)
    return circ, Su, Sl, ranges, A


def run_ranges(circ, Su, Sl, ranges, prec, opts):
    ctx = make_ctx(prec, circ, opts)
    try:
        Q.qsim_set_blocks(ctx, Su, Sl)
        for (b0, b1) in ranges:
            Q.qsim_evolve_range(ctx, b0, b1)
        return Q.qsim_amplitudes(ctx, Su, Sl)
    finally:
        Q.qsim_destroy(ctx)


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("defer", [0, 1])
@pytest.mark.parametrize("bfs", [0, 1])
@pytest.mark.parametrize("lazy", [0, 2, 3, 4])
@pytest.mark.parametrize("frames", [0, 1])
def test_d22_h14_forks(prec, defer, bfs, lazy, frames, d22_h14, monkeypatch):
    """Deferred (default) and eager forks, depth-first and level-synchronous, lazy tail off / by the
    cost model / forced to two / three stages (cones of cones); with the frame executor on (the default,
    every state size) and off (the tree executors)."""
    monkeypatch.setenv("QSIM_FRAMES", str(frames))
    circ, Su, Sl, ranges, ref = d22_h14
    A = run_ranges(circ, Su, Sl, ranges, prec,
                   {Q.QSIM_OPT_DEFER: defer, Q.QSIM_OPT_BFS: bfs, Q.QSIM_OPT_LAZY_LAST: lazy})
    assert_close(A, ref, prec, f"d22 h14 defer={defer} bfs={bfs} lazy={lazy}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("nb", [0, 1, 2, -1])
@pytest.mark.parametrize("lazy", [0, 2, 4])
@pytest.mark.parametrize("frames", [0, 1])
def test_d22_h14_sibling_flips(prec, nb, lazy, frames, d22_h14, monkeypatch):
    """Sibling flips and Pauli frames: children of a Z^b fork read as child 0 through
    a bit flip and a diagonal (frames=0: for one sweep; frames=1: for as long as the frame moves
    through the sweeps), Z^b on both endpoints of the free cuts with the lower rows Walsh-Hadamard
    transformed (R-zz), and with 0 / 1 / 2 extra buffers the states overwritten in place restored by
    inverse sweeps (QSIM_OPT_FLIP_NB).  Every ragged range against the oracle's sum of outer products."""
    monkeypatch.setenv("QSIM_FRAMES", str(frames))
    circ, Su, Sl, ranges, ref = d22_h14
    ctx = make_ctx(prec, circ, {Q.QSIM_OPT_BFS: 0, Q.QSIM_OPT_FLIP: 1, Q.QSIM_OPT_FLIP_NB: nb,
                                Q.QSIM_OPT_LAZY_LAST: lazy})
    try:
        Q.qsim_set_blocks(ctx, Su, Sl)
        Q.qsim_stats_reset(ctx)
        for (b0, b1) in ranges:
            Q.qsim_evolve_range(ctx, b0, b1)
        A = Q.qsim_amplitudes(ctx, Su, Sl)
        st = Q.qsim_stats(ctx)
    finally:
        Q.qsim_destroy(ctx)
    assert_close(A, ref, prec, f"d22 h14 flips nb={nb} lazy={lazy}")
    assert st["flip_siblings"] > 0
    if nb == 0 and not frames:
        assert st["undo_sweeps"] > 0


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("bfs", [0, 1])
def test_d22_h14_projector_side(prec, bfs, d22_h14, monkeypatch):
    """R6' (QSIM_ROLES=1): the projector moved to the lower endpoint of the cuts whose two values a
    block sums; the block's fixed bits keep R6, so every partial range still equals the oracle's sum."""
    monkeypatch.setenv("QSIM_ROLES", "1")
    circ, Su, Sl, ranges, ref = d22_h14
    A = run_ranges(circ, Su, Sl, ranges, prec, {Q.QSIM_OPT_BFS: bfs})
    assert_close(A, ref, prec, f"d22 h14 roles bfs={bfs}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("ctas", [1, 3])
@pytest.mark.parametrize("kernel", [0, 2, 3])
@pytest.mark.parametrize("bfs", [0, 1])
def test_d22_h14_many_tiles_per_cta(prec, ctas, kernel, bfs, d22_h14):
    """Persistent grid capped at 1 / 3 CTAs: every CTA streams hundreds of tiles through the TMA
    pipeline (mbarrier phase wrap, 2 and 3 stage rotation, known-zero tiles) at h = 14."""
    circ, Su, Sl, ranges, ref = d22_h14
    A = run_ranges(circ, Su, Sl, ranges, prec,
                   {Q.QSIM_OPT_MAX_CTAS: ctas, Q.QSIM_OPT_SWEEP_KERNEL: kernel, Q.QSIM_OPT_BFS: bfs})
    assert_close(A, ref, prec, f"h14 ctas={ctas} kernel={kernel} bfs={bfs}")


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
@pytest.mark.parametrize("budget_states", [1, 2, 3])
def test_d22_h14_buffer_budget(prec, budget_states, d22_h14):
    """1-3 state buffers: the fork placement pins cuts and recomputes paths to fit (choose_tree)."""
    circ, Su, Sl, ranges, ref = d22_h14
    amp = 16 if prec == Q.QSIM_C128 else 8
    A = run_ranges(circ, Su, Sl, ranges, prec,
                   {Q.QSIM_OPT_MEM_BUDGET: budget_states * (1 << 14) * amp + 1, Q.QSIM_OPT_BFS: 0})
    assert_close(A, ref, prec, f"h14 budget {budget_states}")


# ------------------------------------------------------------------ h = 24: 6x8 grid, depth 22
@pytest.fixture(scope="module")
def h24():
    circ = generate(6, 8, 22, 0)
    cuts = OP.cut_list(circ)
    B = 1 << len(cuts)
    rng = np.random.default_rng(24)
    branches = [0, B - 1, int(rng.integers(B)), int(rng.integers(B))]
    idx = {half: index_sample(24, 4096, 30 + half) for half in (0, 1)}
    ref = {(half, b): oracle_values(circ, half, b, [idx[half]])[0] for half in (0, 1) for b in branches}
    full = F.branch_state(circ, OP.LOWER, branches[2], cuts)
    return circ, branches, idx, ref, full


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_h24_leaf_values(prec, h24):
    """6x8 d22 (h = 24, 2^11 tiles c64): branches 0, B-1 and two random ones, both halves."""
    circ, branches, idx, ref, _ = h24
    ctx = make_ctx(prec, circ)
    try:
        for half in (0, 1):
            for b in branches:
                got = Q.qsim_branch_values(ctx, half, b, idx[half])
                assert_close(got, ref[(half, b)], prec, f"h24 half {half} branch {b}")
    finally:
        Q.qsim_destroy(ctx)


@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_h24_full_leaf(prec, h24):
    """Every amplitude of one 24-qubit leaf (qsim_branch_state, canonical order)."""
    circ, branches, _, _, full = h24
    ctx = make_ctx(prec, circ)
    try:
        got = Q.qsim_branch_state(ctx, 1, branches[2])
    finally:
        Q.qsim_destroy(ctx)
    assert_close(got, full, prec, "h24 full leaf")


# ------------------------------------------------------------------ h = 28: C4 (8x7, depth 22)
@pytest.fixture(scope="module")
def c4_oracle():
    """Oracle leaves of C4 (56 qubits, c = 14) at sampled indices: branches 0 and the last four."""
    circ = generate(8, 7, 22, 0)
    cuts = OP.cut_list(circ)
    B = 1 << len(cuts)
    branches = [0, B - 4, B - 3, B - 2, B - 1]
    idx = {half: index_sample(28, 8192, 40 + half) for half in (0, 1)}
    Su, Sl = sample_block(28, 256, 50), sample_block(28, 256, 51)
    blk = {0: Su, 1: Sl}
    ref, slices = {}, {}
    for half in (0, 1):
        for b in branches:
            v, s = oracle_values(circ, half, b, [idx[half], blk[half]])
            ref[(half, b)] = v
            slices[(half, b)] = s
    A = sum(np.outer(slices[(0, b)], slices[(1, b)]) for b in range(B - 4, B))
    return circ, branches, idx, ref, Su, Sl, A


@pytest.mark.slow
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_c4_leaf_values(prec, c4_oracle):
    """C4 leaves (h = 28, 2^15 c64 tiles: ~220 per CTA) at 8195 indices, both halves."""
    circ, branches, idx, ref, *_ = c4_oracle
    ctx = make_ctx(prec, circ)
    try:
        for half in (0, 1):
            for b in branches:
                got = Q.qsim_branch_values(ctx, half, b, idx[half])
                assert_close(got, ref[(half, b)], prec, f"C4 half {half} branch {b}")
    finally:
        Q.qsim_destroy(ctx)


@pytest.mark.slow
@pytest.mark.parametrize("prec", PRECS, ids=PNAME.get)
def test_c4_block_of_four_branches(prec, c4_oracle):
    """qsim_evolve_range over the last 4 branches of C4 with 256 x 256 blocks: the tree, the
    gathered slices and the GEMM at full size vs the oracle's sum of outer products."""
    circ, _, _, _, Su, Sl, ref = c4_oracle
    B = 1 << 14
    ctx = make_ctx(prec, circ)
    try:
        Q.qsim_set_blocks(ctx, Su, Sl)
        Q.qsim_evolve_range(ctx, B - 4, B)
        A = Q.qsim_amplitudes(ctx, Su, Sl)
    finally:
        Q.qsim_destroy(ctx)
    assert_close(A, ref, prec, "C4 4-branch block")


# ------------------------------------------------------------------ C5: 64 qubits
@pytest.mark.slow
def test_c5_prefix_group_c64_vs_c128():
    """One first-period prefix group of C5 (256 branches, 64q d22) on a 4096 x 4096 block in both
    precisions: c64 within 1e-5 of max|a| of c128 (R12)."""
    circ = generate(8, 8, 22, 0)
    Su, Sl = sample_block(32, 4096, 60), sample_block(32, 4096, 61)
    out = {}
    for prec in PRECS:
        ctx = make_ctx(prec, circ)
        try:
            Q.qsim_set_blocks(ctx, Su, Sl)
            Q.qsim_evolve_range(ctx, 37 * 256, 38 * 256)
            out[prec] = Q.qsim_amplitudes(ctx, Su, Sl)
        finally:
            Q.qsim_destroy(ctx)
    d, rel, rms = errs(out[Q.QSIM_C64], out[Q.QSIM_C128])
    print(f"C5 group 37: c64 vs c128 max|d| {d:.3e}, /max|a| {rel:.3e}, /rms {rms:.3e}")
    assert rel <= 1e-5


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("QSIM_TEST_H32") != "1",
                    reason="h = 32 oracle leaves need 64 GiB of host RAM and minutes (QSIM_TEST_H32=1)")
@pytest.mark.parametrize("half", [0, 1])
def test_c5_leaf_values_h32(half):
    """C5 leaves (h = 32) of branches 0 and B-1 at 4099 indices, both precisions, vs the oracle."""
    circ = generate(8, 8, 22, 0)
    B = 1 << len(OP.cut_list(circ))
    idx = index_sample(32, 4096, 70 + half)
    for b in (0, B - 1):
        ref = oracle_values(circ, half, b, [idx])[0]
        for prec in PRECS:
            ctx = make_ctx(prec, circ)
            try:
                got = Q.qsim_branch_values(ctx, half, b, idx)
            finally:
                Q.qsim_destroy(ctx)
            d, rel, rms = errs(got, ref)
            print(f"C5 h32 half {half} branch {b} {PNAME[prec]}: max|d| {d:.3e} /max {rel:.3e} /rms {rms:.3e}")
            assert_close(got, ref, prec, f"C5 half {half} branch {b}")


def _c5_block(prec, Su, Sl, b0, b1, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    ctx = make_ctx(prec, generate(8, 8, 22, 0))
    try:
        Q.qsim_set_blocks(ctx, Su, Sl)
        Q.qsim_evolve_range(ctx, b0, b1)
        return Q.qsim_amplitudes(ctx, Su, Sl)
    finally:
        Q.qsim_destroy(ctx)


@pytest.mark.slow
def test_c5_frames_vs_tree(monkeypatch):
    """C5 (64q d22), branches [0, 4096) (one block of 12 free cuts) on a 512 x 512 block in c128: the
    Pauli-frame executor with expansion (one real state per half, leaves as sums of frame terms), with
    real splits only (QSIM_FRAME_EXPAND=0), and the plain branch-tree executor (QSIM_FRAMES=0: every
    leaf from its own sweeps) agree to 1e-12 of max|a|."""
    Su, Sl = sample_block(32, 512, 80), sample_block(32, 512, 81)
    ref = _c5_block(Q.QSIM_C128, Su, Sl, 0, 4096, {"QSIM_FRAMES": "0"}, monkeypatch)
    for env in ({"QSIM_FRAMES": "1", "QSIM_FRAME_EXPAND": "0"}, {"QSIM_FRAMES": "1", "QSIM_FRAME_EXPAND": "6"}):
        A = _c5_block(Q.QSIM_C128, Su, Sl, 0, 4096, env, monkeypatch)
        d, rel, rms = errs(A, ref)
        print(f"C5 [0, 4096) frames {env}: max|d| {d:.3e} /max {rel:.3e} /rms {rms:.3e}")
        assert rel <= 1e-12


@pytest.mark.slow
def test_c5_whole_job_c64_vs_c128(monkeypatch):
    """The whole C5 job (all 65536 branches, one block per half) on a 1024 x 1024 block: c64 within
    1e-5 of max|a| of c128 (R12), both through the frame executor."""
    Su, Sl = sample_block(32, 1024, 82), sample_block(32, 1024, 83)
    out = {p: _c5_block(p, Su, Sl, 0, 1 << 16, {}, monkeypatch) for p in PRECS}
    d, rel, rms = errs(out[Q.QSIM_C64], out[Q.QSIM_C128])
    print(f"C5 whole job c64 vs c128: max|d| {d:.3e} /max {rel:.3e} /rms {rms:.3e}")
    assert rel <= 1e-5
