"""C-ABI library checks that need no GPU: it loads, exports every symbol of
include/qsim.h, and the host front end (validation, cut list, branch enumeration)
is bit-exact against the oracle's independent derivation."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from workloads import generate, CONFIGS
from workloads.circuits import NO_QUBIT
from oracle import partition as OP

Q = pytest.importorskip("paper_1802_06952_b200.qsim")

HEADER = os.path.join(ROOT, "include", "qsim.h")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_header_symbols_exported():
    src = open(HEADER).read()
    declared = set(re.findall(r"\b(qsim_[a-z_0-9]+)\s*\(", src))
    assert declared, "no declarations parsed"
    out = subprocess.run(["nm", "-D", "--defined-only", Q.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = declared - exported
    assert not missing, f"declared but not exported: {missing}"
    assert declared == set(Q.EXPORTED)
    lib = ctypes.CDLL(Q.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", Q.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version():
    assert "sm_100a" in Q.qsim_version()


@pytest.mark.parametrize("name", list(CONFIGS))
@pytest.mark.parametrize("seed", [0, 1])
def test_partition_matches_oracle(name, seed):
    """Cut list and branch count: bit-exact vs the oracle's own derivation."""
    rows, cols, depth, _, _ = CONFIGS[name]
    circ = generate(rows, cols, depth, seed)
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
        c, nb, cuts = Q.qsim_partition(ctx)
        ref = OP.cut_list(circ)
        assert c == len(ref) and nb == 1 << len(ref)
        assert [tuple(map(int, r)) for r in cuts] == ref
        Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array(),
                            cut_layers=sorted({t for t, _, _ in ref}))
    finally:
        Q.qsim_destroy(ctx)


def test_expected_cut_counts():
    """c = 2 / 12 / 14 / 14 / 16 for C1..C5 (Table 2; §2.3.2)."""
    ctx = Q.qsim_create(Q.QSIM_C128, 0)
    try:
        for name, c_exp in zip(CONFIGS, [2, 12, 14, 14, 16]):
            rows, cols, depth, _, _ = CONFIGS[name]
            Q.qsim_load_circuit(ctx, rows, cols, depth, generate(rows, cols, depth, 3).gate_array())
            assert Q.qsim_partition(ctx)[0] == c_exp
    finally:
        Q.qsim_destroy(ctx)


def _expect(status, fn, *a, **k):
    with pytest.raises(Q.QsimError) as ei:
        fn(*a, **k)
    assert ei.value.status == status, str(ei.value)


def test_error_paths():
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        _expect(Q.QSIM_ESTATE, Q.qsim_partition, ctx)
        ok = np.array([[1, 4, 0, 1]], dtype=np.uint32)
        Q.qsim_load_circuit(ctx, 2, 2, 1, ok)
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 2, 2, 1, np.array([[1, 1, 4, NO_QUBIT]]))   # qubit >= n
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 2, 2, 1,
                np.array([[1, 4, 0, 1], [1, 1, 1, NO_QUBIT]]))                                       # overlap
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 2, 2, 1, np.array([[1, 4, 0, 3]]))          # not an edge
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 2, 2, 1, np.array([[2, 1, 0, NO_QUBIT]]))   # layer > depth
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 2, 2, 1, np.array([[1, 7, 0, NO_QUBIT]]))   # kind
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 2, 2, 1, np.array([[1, 1, 0, 2]]))          # q1 on single
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 9, 8, 1, np.zeros((0, 4)))                  # > 64 qubits
        _expect(Q.QSIM_EINVAL, Q.qsim_load_circuit, ctx, 2, 2, 1, np.array([[1, 4, 0, 2]]),
                cut_layers=[3])                                                                      # cut layers
        _expect(Q.QSIM_EINVAL, Q.qsim_set_option, ctx, 99, 1)
        _expect(Q.QSIM_EINVAL, Q.qsim_set_option, ctx, Q.QSIM_OPT_MODE, 7)
        Q.qsim_load_circuit(ctx, 2, 2, 1, ok)
        _expect(Q.QSIM_EINVAL, Q.qsim_set_blocks, ctx, [0, 4], [0])                                  # index >= 2^h
        _expect(Q.QSIM_EINVAL, Q.qsim_set_blocks, ctx, [1, 1], [0])                                  # duplicate
        _expect(Q.QSIM_ESTATE, Q.qsim_evolve_range, ctx, 0, 1)
        _expect(Q.QSIM_ESTATE, Q.qsim_amplitudes, ctx, [0], [0], Q.QSIM_C64)
    finally:
        Q.qsim_destroy(ctx)
    with pytest.raises(Q.QsimError):
        Q.qsim_create(7, 0)


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly():
    """Without a CUDA device every compute call fails with QSIM_ECUDA (no CPU fallback)."""
    ctx = Q.qsim_create(Q.QSIM_C64, 0)
    try:
        circ = generate(4, 2, 8, 0)
        Q.qsim_load_circuit(ctx, 4, 2, 8, circ.gate_array())
        _expect(Q.QSIM_ECUDA, Q.qsim_set_blocks, ctx, np.arange(16), np.arange(16))
        _expect(Q.QSIM_ECUDA, Q.qsim_sample_probs, ctx, np.ones((2, 2)), [0, 1], [0, 1], 1, 0, 4)
    finally:
        Q.qsim_destroy(ctx)
