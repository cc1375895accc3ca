"""Thin ctypes binding of the C-ABI in ``include/qsim.h`` (argument marshalling only).

Every function has the C name and forwards to ``libqsim.so``; every step of the hot
path runs in the library's CUDA kernels.  There is no CPU fallback: importing this
module fails loudly when the library has not been built, and every compute call
raises ``QsimError`` when no B200 is present.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QSIM_LIB") or os.path.join(_HERE, "libqsim.so")  # QSIM_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1802_06952_b200.build` "
                      "(there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

QSIM_OK, QSIM_EINVAL, QSIM_ENOMEM, QSIM_ENUMERIC, QSIM_ECUDA, QSIM_ENCCL, QSIM_ESTATE = 0, 2, 3, 4, 5, 6, 7
STATUS_NAMES = {0: "QSIM_OK", 2: "QSIM_EINVAL", 3: "QSIM_ENOMEM", 4: "QSIM_ENUMERIC", 5: "QSIM_ECUDA",
                6: "QSIM_ENCCL", 7: "QSIM_ESTATE"}
QSIM_C64, QSIM_C128 = 0, 1
QSIM_SX, QSIM_SY, QSIM_T, QSIM_CZ = 1, 2, 3, 4
QSIM_NO_QUBIT = 0xFFFFFFFF
QSIM_OPT_TIME_SWEEPS, QSIM_OPT_MODE, QSIM_OPT_MEM_BUDGET, QSIM_OPT_SWEEP_KERNEL, QSIM_OPT_LAZY_LAST = 1, 2, 3, 4, 5
QSIM_OPT_FUSE_LAYERS = 6
QSIM_OPT_DISTRIBUTE = 7
QSIM_OPT_BFS = 8
QSIM_OPT_MAX_CTAS = 9
QSIM_OPT_DEFER = 10
QSIM_OPT_FLIP = 11
QSIM_OPT_FLIP_NB = 12

EXPORTED = ["qsim_create", "qsim_destroy", "qsim_last_error", "qsim_version", "qsim_set_option",
            "qsim_set_stream", "qsim_load_circuit", "qsim_partition", "qsim_set_blocks",
            "qsim_evolve_range", "qsim_evolve_halves", "qsim_reset_block", "qsim_amplitudes",
            "qsim_sample", "qsim_sample_probs", "qsim_branch_sum", "qsim_branch_state",
            "qsim_nccl_unique_id", "qsim_comm_init", "qsim_rank_range", "qsim_stats",
            "qsim_stats_reset", "qsim_synchronize", "qsim_eq2_time", "qsim_cost_model",
            "qsim_porter_thomas", "qsim_multipart_plan", "qsim_multipart_amplitudes", "qsim_branch_values",
            "qsim_info"]


class qsim_cut(C.Structure):
    _fields_ = [("layer", C.c_uint32), ("q_upper", C.c_uint32), ("q_lower", C.c_uint32)]


class qsim_info_t(C.Structure):
    _fields_ = [("precision", C.c_uint32), ("have_circuit", C.c_uint32), ("h_upper", C.c_uint32),
                ("h_lower", C.c_uint32), ("n_cuts", C.c_uint32), ("n_upper", C.c_uint64),
                ("n_lower", C.c_uint64), ("device", C.c_int32)]


class qsim_stats_t(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("sweeps", C.c_uint64), ("sweep_states", C.c_uint64),
                ("sweep_bytes", C.c_double), ("sweep_ms", C.c_double), ("timed_sweeps", C.c_uint64),
                ("gemm_flops", C.c_double), ("gemm_ms", C.c_double), ("branches_evolved", C.c_uint64),
                ("lazy_gathers", C.c_uint64), ("layers_applied", C.c_uint64), ("sweep_bytes_moved", C.c_double),
                ("flip_siblings", C.c_uint64), ("undo_sweeps", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class qsim_cost_t(C.Structure):
    _fields_ = [("n_qubits", C.c_uint32), ("h_upper", C.c_uint32), ("h_lower", C.c_uint32),
                ("n_cuts", C.c_uint32), ("n_branches", C.c_double), ("half_circuits", C.c_double),
                ("N_e", C.c_uint32), ("N_m", C.c_uint32), ("regime", C.c_int32),
                ("flat_layer_evolutions", C.c_double), ("tree_sweeps", C.c_double),
                ("lazy_gathers", C.c_double), ("sweep_bytes", C.c_double), ("predicted_s", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class qsim_pt_t(C.Structure):
    _fields_ = [("count", C.c_double), ("zeros", C.c_double), ("mean_Np", C.c_double), ("var_Np", C.c_double),
                ("ks_lo", C.c_double), ("ks_hi", C.c_double), ("below", C.c_double), ("above", C.c_double),
                ("n_qubits", C.c_uint32), ("n_bins", C.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = C.c_void_p
_sig = {
    "qsim_porter_thomas": (C.c_int, [_P, _P, C.c_size_t, C.c_uint32, C.c_double, C.c_double, C.c_uint32, _P, _P,
                                     C.POINTER(qsim_pt_t)]),
    "qsim_eq2_time": (C.c_int, [_P, C.c_size_t, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "qsim_cost_model": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_double, _P]),
    "qsim_multipart_plan": (C.c_int, [_P, C.c_uint32, _P, _P, _P, C.POINTER(C.c_double)]),
    "qsim_multipart_amplitudes": (C.c_int, [_P, C.c_uint32, _P, _P, _P, _P]),
    "qsim_create": (C.c_int, [C.POINTER(_P), C.c_int, C.c_int]),
    "qsim_destroy": (None, [_P]),
    "qsim_last_error": (C.c_char_p, [_P]),
    "qsim_version": (C.c_char_p, []),
    "qsim_set_option": (C.c_int, [_P, C.c_int, C.c_int64]),
    "qsim_set_stream": (C.c_int, [_P, _P]),
    "qsim_load_circuit": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, _P, C.c_size_t, C.c_uint32,
                                    _P, C.c_size_t]),
    "qsim_partition": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), _P]),
    "qsim_set_blocks": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t]),
    "qsim_evolve_range": (C.c_int, [_P, C.c_uint64, C.c_uint64]),
    "qsim_evolve_halves": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t]),
    "qsim_reset_block": (C.c_int, [_P]),
    "qsim_amplitudes": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t, _P]),
    "qsim_sample": (C.c_int, [_P, C.c_uint64, C.c_size_t, _P, _P]),
    "qsim_sample_probs": (C.c_int, [_P, _P, _P, C.c_size_t, _P, C.c_size_t, C.c_uint32, C.c_uint64,
                                    C.c_size_t, _P, _P]),
    "qsim_branch_sum": (C.c_int, [_P, _P, _P, C.c_size_t, C.c_size_t, C.c_size_t, _P]),
    "qsim_branch_state": (C.c_int, [_P, C.c_int, C.c_uint64, _P]),
    "qsim_branch_values": (C.c_int, [_P, C.c_int, C.c_uint64, _P, C.c_size_t, _P]),
    "qsim_info": (C.c_int, [_P, C.POINTER(qsim_info_t)]),
    "qsim_nccl_unique_id": (C.c_int, [_P]),
    "qsim_comm_init": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "qsim_rank_range": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "qsim_stats": (C.c_int, [_P, C.POINTER(qsim_stats_t)]),
    "qsim_stats_reset": (C.c_int, [_P]),
    "qsim_synchronize": (C.c_int, [_P]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class QsimError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _check(ctx, status):
    if status != QSIM_OK:
        msg = _lib.qsim_last_error(ctx).decode() if ctx else ""
        raise QsimError(status, msg)


def qsim_version() -> str:
    return _lib.qsim_version().decode()


def qsim_create(prec: int = QSIM_C64, device: int = 0):
    ctx = _P()
    _check(None, _lib.qsim_create(C.byref(ctx), prec, device))
    return ctx


def qsim_destroy(ctx):
    _lib.qsim_destroy(ctx)


def qsim_last_error(ctx) -> str:
    return _lib.qsim_last_error(ctx).decode()


def qsim_set_option(ctx, key: int, value: int):
    _check(ctx, _lib.qsim_set_option(ctx, key, value))


def qsim_set_stream(ctx, cuda_stream: int | None):
    _check(ctx, _lib.qsim_set_stream(ctx, cuda_stream or None))


def qsim_load_circuit(ctx, rows, cols, depth, gates, cut_row=0, cut_layers=None):
    g = np.ascontiguousarray(np.asarray(gates, dtype=np.uint32).reshape(-1, 4))
    cl = None if cut_layers is None else np.ascontiguousarray(np.asarray(cut_layers, dtype=np.uint32))
    _check(ctx, _lib.qsim_load_circuit(ctx, rows, cols, depth, _ptr(g), g.shape[0], cut_row,
                                       _ptr(cl), 0 if cl is None else cl.size))


def qsim_partition(ctx):
    """Returns (c, n_branches, cuts[c, 3] as (layer, q_upper, q_lower))."""
    nc, nb = C.c_uint32(), C.c_uint64()
    _check(ctx, _lib.qsim_partition(ctx, C.byref(nc), C.byref(nb), None))
    cuts = np.zeros((nc.value, 3), dtype=np.uint32)
    if nc.value:
        _check(ctx, _lib.qsim_partition(ctx, C.byref(nc), C.byref(nb), _ptr(cuts)))
    return nc.value, nb.value, cuts


def qsim_set_blocks(ctx, upper_block, lower_block):
    u, l = _u64(upper_block), _u64(lower_block)
    _check(ctx, _lib.qsim_set_blocks(ctx, _ptr(u), u.size, _ptr(l), l.size))


def qsim_evolve_range(ctx, branch_begin: int, branch_end: int):
    _check(ctx, _lib.qsim_evolve_range(ctx, branch_begin, branch_end))


def qsim_evolve_halves(ctx, upper_block, lower_block):
    u, l = _u64(upper_block), _u64(lower_block)
    _check(ctx, _lib.qsim_evolve_halves(ctx, _ptr(u), u.size, _ptr(l), l.size))


def qsim_reset_block(ctx):
    _check(ctx, _lib.qsim_reset_block(ctx))


def qsim_amplitudes(ctx, upper_block, lower_block, prec: int = None, out=None, write=True):
    """Reconstructed block [n_u, n_l] of the ctx precision (``prec``, if given, must match it;
    a caller-supplied ``out`` must be a C-contiguous array of that dtype and shape)."""
    u, l = _u64(upper_block), _u64(lower_block)
    dt = _amp_dtype(ctx)
    if prec is not None and np.dtype(dt) != np.dtype(np.complex128 if prec == QSIM_C128 else np.complex64):
        raise ValueError("prec differs from the context's precision")
    if write and out is None:
        out = np.empty((u.size, l.size), dtype=dt)
    if write and (out.dtype != dt or out.size != u.size * l.size or not out.flags.c_contiguous):
        raise ValueError(f"out must be a C-contiguous {np.dtype(dt)} array of {u.size} x {l.size}")
    _check(ctx, _lib.qsim_amplitudes(ctx, _ptr(u), u.size, _ptr(l), l.size, _ptr(out) if write else None))
    return out


def qsim_sample(ctx, seed: int, n_draws: int, to_host: bool = True, out=None):
    if to_host and out is None:
        out = np.empty(n_draws, dtype=np.uint64)
    if not to_host:
        out = None
    assert out is None or (out.dtype == np.uint64 and out.size >= n_draws)
    mass = C.c_double(0.0)
    _check(ctx, _lib.qsim_sample(ctx, seed, n_draws, _ptr(out), C.byref(mass) if to_host else None))
    return out, mass.value


def qsim_sample_probs(ctx, p, upper_block, lower_block, h_lower: int, seed: int, n_draws: int):
    p = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
    u, l = _u64(upper_block), _u64(lower_block)
    assert p.size == u.size * l.size
    out = np.empty(n_draws, dtype=np.uint64)
    mass = C.c_double(0.0)
    _check(ctx, _lib.qsim_sample_probs(ctx, _ptr(p), _ptr(u), u.size, _ptr(l), l.size, h_lower, seed, n_draws,
                                       _ptr(out), C.byref(mass)))
    return out, mass.value


def qsim_porter_thomas(ctx, p=None, n_qubits: int = 0, z_lo: float = -12.0, z_hi: float = 4.0,
                       n_bins: int = 160):
    """Porter-Thomas / Eq. 7 analyzer (f1).  p=None: the evolved block.  Returns
    (stats dict, z histogram uint64[n_bins], Eq. 7 expected counts float64[n_bins])."""
    hist = np.zeros(n_bins, dtype=np.uint64)
    expected = np.zeros(n_bins, dtype=np.float64)
    r = qsim_pt_t()
    if p is not None:
        p = np.ascontiguousarray(np.asarray(p, dtype=np.float64)).ravel()
    _check(ctx, _lib.qsim_porter_thomas(ctx, _ptr(p), 0 if p is None else p.size, n_qubits, z_lo, z_hi, n_bins,
                                        _ptr(hist), _ptr(expected), C.byref(r)))
    return r.as_dict(), hist, expected


def qsim_branch_sum(ctx, U, L, prec: int):
    dt = np.complex128 if prec == QSIM_C128 else np.complex64
    U = np.ascontiguousarray(np.asarray(U, dtype=dt))
    L = np.ascontiguousarray(np.asarray(L, dtype=dt))
    A = np.empty((U.shape[1], L.shape[1]), dtype=np.complex128)
    _check(ctx, _lib.qsim_branch_sum(ctx, _ptr(U), _ptr(L), U.shape[0], U.shape[1], L.shape[1], _ptr(A)))
    return A


def qsim_info(ctx) -> dict:
    r = qsim_info_t()
    _check(ctx, _lib.qsim_info(ctx, C.byref(r)))
    return {f: getattr(r, f) for f, _ in qsim_info_t._fields_}


def _amp_dtype(ctx):
    return np.complex128 if qsim_info(ctx)["precision"] == QSIM_C128 else np.complex64


def qsim_branch_state(ctx, half: int, branch: int, h: int = None, prec: int = None):
    """The complete leaf half-state (2^h values of the ctx precision; h / prec are checked)."""
    inf = qsim_info(ctx)
    hh = inf["h_upper"] if half == 0 else inf["h_lower"]
    if h is not None and h != hh:
        raise ValueError(f"h = {h} but the loaded circuit's half has {hh} qubits")
    if prec is not None and prec != inf["precision"]:
        raise ValueError("prec differs from the context's precision")
    out = np.empty(1 << hh, dtype=_amp_dtype(ctx))
    _check(ctx, _lib.qsim_branch_state(ctx, half, branch, _ptr(out)))
    return out


def qsim_branch_values(ctx, half: int, branch: int, idx):
    """U_b[idx] / L_b[idx] of one branch through the production path (qsim.h)."""
    ix = _u64(idx)
    out = np.empty(ix.size, dtype=_amp_dtype(ctx))
    _check(ctx, _lib.qsim_branch_values(ctx, half, branch, _ptr(ix), ix.size, _ptr(out)))
    return out


def qsim_nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(None, _lib.qsim_nccl_unique_id(C.cast(buf, _P)))
    return bytes(buf)


def qsim_comm_init(ctx, rank: int, world: int, unique_id: bytes):
    buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
    _check(ctx, _lib.qsim_comm_init(ctx, rank, world, C.cast(buf, _P)))


def qsim_rank_range(ctx):
    b0, b1 = C.c_uint64(), C.c_uint64()
    _check(ctx, _lib.qsim_rank_range(ctx, C.byref(b0), C.byref(b1)))
    return b0.value, b1.value


def qsim_eq2_time(n_i, m: float, t: float, s: float) -> float:
    """Eq. 2: sum(n_i) * m * t / s seconds."""
    n = np.ascontiguousarray(np.asarray(n_i, dtype=np.float64))
    out = C.c_double()
    _check(None, _lib.qsim_eq2_time(_ptr(n), n.size, m, t, s, C.byref(out)))
    return out.value


def qsim_cost_model(ctx, n_upper: int, n_lower: int, hbm_gbps: float) -> dict:
    c = qsim_cost_t()
    _check(ctx, _lib.qsim_cost_model(ctx, n_upper, n_lower, hbm_gbps, C.byref(c)))
    return c.as_dict()


def qsim_multipart_plan(ctx, row_cuts) -> dict:
    """Parts (bands of rows split at ``row_cuts``) of the loaded circuit: qubits per part, cuts per
    boundary, log2 of the leaf amplitudes evolved (include/qsim.h)."""
    rc = np.ascontiguousarray(np.asarray(row_cuts, dtype=np.uint32))
    t = rc.size + 1
    pq = np.zeros(t, dtype=np.uint32)
    bc = np.zeros(max(t - 1, 1), dtype=np.uint32)
    l2 = C.c_double()
    _check(ctx, _lib.qsim_multipart_plan(ctx, t, _ptr(rc), _ptr(pq), _ptr(bc), C.byref(l2)))
    return {"part_qubits": pq.tolist(), "boundary_cuts": bc[:t - 1].tolist(), "log2_states": l2.value}


def qsim_multipart_amplitudes(ctx, row_cuts, blocks, prec: int) -> np.ndarray:
    """amps[i_0, ..., i_{t-1}] = sum_b prod_k psi^k_b[S_k[i_k]] for the blocks S_k (one per part)."""
    rc = np.ascontiguousarray(np.asarray(row_cuts, dtype=np.uint32))
    bl = [_u64(b) for b in blocks]
    if len(bl) != rc.size + 1:
        raise ValueError(f"{rc.size} row cuts make {rc.size + 1} parts; got {len(bl)} blocks")
    cat = np.ascontiguousarray(np.concatenate(bl)) if bl else np.zeros(0, dtype=np.uint64)
    nb = np.asarray([b.size for b in bl], dtype=np.uint64)
    out = np.zeros(tuple(b.size for b in bl), dtype=np.complex128 if prec == QSIM_C128 else np.complex64)
    _check(ctx, _lib.qsim_multipart_amplitudes(ctx, len(bl), _ptr(rc), _ptr(cat), _ptr(nb), _ptr(out)))
    return out


def qsim_stats(ctx) -> dict:
    s = qsim_stats_t()
    _check(ctx, _lib.qsim_stats(ctx, C.byref(s)))
    return s.as_dict()


def qsim_stats_reset(ctx):
    _check(ctx, _lib.qsim_stats_reset(ctx))


def qsim_synchronize(ctx):
    _check(ctx, _lib.qsim_synchronize(ctx))


class Simulator:
    """Convenience owner of a context (the same calls, bound to one ctx)."""

    def __init__(self, prec: int = QSIM_C64, device: int = 0):
        self.prec = prec
        self.ctx = qsim_create(prec, device)
        self.h_u = self.h_l = None

    def close(self):
        if self.ctx:
            qsim_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, circuit, cut_layers=None):
        qsim_load_circuit(self.ctx, circuit.rows, circuit.cols, circuit.depth, circuit.gate_array(),
                          circuit.cut_row, cut_layers)
        self.h_u, self.h_l = circuit.h_upper, circuit.h_lower
        return self

    def partition(self):
        return qsim_partition(self.ctx)

    def amplitudes(self, S_u, S_l):
        qsim_evolve_halves(self.ctx, S_u, S_l)
        return qsim_amplitudes(self.ctx, S_u, S_l, self.prec)

    def sample(self, seed, n):
        return qsim_sample(self.ctx, seed, n)

    def set_option(self, key, value):
        qsim_set_option(self.ctx, key, value)
        return self

    def stats(self):
        return qsim_stats(self.ctx)
