"""Multi-threaded gate application for large half states (ORACLE — test infrastructure only).

``run_gates`` is ``statevector.run_gates`` with the per-gate pair loop in plain C + OpenMP
(``oracle/csrc/csim.c``): the same gate list, applied one gate at a time in list order with the
same 2x2 matrices (taken from ``oracle.gates``; the C file defines none), on an interleaved
complex128 state.  It exists because numpy's one-thread einsum takes minutes per gate list at
h = 28-32 (CPU evolution of individual 28- / 32-qubit branch halves).

Pinned in ``tests/test_oracle_fast.py`` against ``statevector.run_gates`` on random gate lists
(every kind, every qubit, n <= 12) and against the depth <= 3 closed form at h = 20; the initial
state H^{(x)h}|0> = 2^{-h/2} everywhere is pinned in ``tests/test_oracle.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import gates as G
from . import partition as OP

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "csim.c")
LIB = os.path.join(HERE, "_csim.so")
_lib = None


def build(force: bool = False) -> str:
    """gcc -O2 -fopenmp -shared (no -ffast-math: IEEE order of operations is kept)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", LIB, SRC], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        L.oracle_run_gates.restype = ctypes.c_int
        L.oracle_run_gates.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_fill.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int]
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def initial_state(n: int, threads: int = 0) -> np.ndarray:
    """H^{(x)n}|0...0> = 2^{-n/2} on every basis state (the closed form the numpy oracle's
    gate-by-gate initial_state is pinned to)."""
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().oracle_fill(psi.ctypes.data, n, 2.0 ** (-n / 2), 0.0, threads)
    return psi


def run_gates(psi: np.ndarray, n: int, gate_list, threads: int = 0) -> np.ndarray:
    """In place: apply ``gate_list`` = (layer, kind, q0, q1) items in order (kinds as in
    ``statevector.run_gates``: 1/'SX', 2/'SY', 3/'T', 4/'CZ', 'P0', 'P1', 'Z', 'H')."""
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous and psi.size == 1 << n
    gl = list(gate_list)
    codes = np.zeros(len(gl), dtype=np.int32)
    q0 = np.zeros(len(gl), dtype=np.int32)
    q1 = np.zeros(len(gl), dtype=np.int32)
    mats = np.zeros((len(gl), 8), dtype=np.float64)
    for i, (_, kind, a, b) in enumerate(gl):
        q0[i] = int(a)
        if kind in (4, "CZ"):
            codes[i] = 4
            q1[i] = int(b)
        else:
            codes[i] = 1
            M = G.SINGLE[kind]
            mats[i] = [M[0, 0].real, M[0, 0].imag, M[0, 1].real, M[0, 1].imag,
                       M[1, 0].real, M[1, 0].imag, M[1, 1].real, M[1, 1].imag]
    rc = lib().oracle_run_gates(psi.ctypes.data, n, len(gl), codes.ctypes.data, q0.ctypes.data,
                                q1.ctypes.data, mats.ctypes.data, threads)
    if rc != 0:
        raise ValueError("bad gate code")
    return psi


def branch_state(circuit, half: int, b: int, cuts=None, threads: int = 0) -> np.ndarray:
    """``partition.branch_state`` with the C gate loop: the same branch half-circuit
    (``partition.half_gates``: internal gates + P_b / Z^b of the cuts, Supp. Eq. 7)."""
    if cuts is None:
        cuts = OP.cut_list(circuit)
    h = circuit.h_upper if half == OP.UPPER else circuit.h_lower
    psi = initial_state(h, threads)
    return run_gates(psi, h, OP.half_gates(circuit, half, cuts, b), threads)
