"""Micro-benchmark of single-layer tile sweeps by target placement (one branch, no cut).

Run with QSIM_PERM=id so the layout is the one described.  Builds an 8x7 grid circuit whose upper half (h = 28) repeats one layer of SX gates on chosen
qubits, evolves it with sweep timing on, and prints GB/s per case.  Local bit of qubit k is
27 - k: qubits 27 (vector bit, c64), 26..24 (lane bits 0-2), 23, 22 (vector bits 3, 4) and
21..0 (hi bits).

    python tools/sweep_micro.py [--precision c64] [--reps 24]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1802_06952_b200 import qsim as Q  # noqa: E402

CASES = {
    "hi4": [0, 5, 10, 15],
    "hi5": [0, 5, 10, 15, 20],
    "hi6": [0, 3, 6, 10, 15, 20],
    "hi7": [0, 3, 6, 9, 12, 15, 20],
    "hi4+v3": [0, 5, 10, 15, 23],
    "hi4+lane": [0, 5, 10, 15, 25],
    "hi2+low4": [3, 12, 22, 23, 25, 27],
    "vec": [27],
    # run length vs spread of the tile's rows (bit b = qubit 27 - b)
    "hi7lo": [20, 19, 18, 17, 16, 15, 14],   # bits 7..13, m = 0
    "hi7hi": [6, 5, 4, 3, 2, 1, 0],          # bits 21..27, m = 0
    "hi7mix": [20, 18, 16, 14, 4, 2, 0],     # m = 0
    "hi4lo": [17, 16, 15, 14],               # bits 10..13, m = 3
    "hi4hi": [3, 2, 1, 0],                   # bits 24..27, m = 3
    "hi6lo": [20, 19, 18, 17, 16, 15],       # m = 1
    "hi6hi": [5, 4, 3, 2, 1, 0],             # m = 1
    # lane-bit (shuffle) targets on top of 4 hi targets: qubits 25, 24, 23 = bits 2, 3, 4
    "hi4+l1": [0, 5, 10, 15, 25],
    "hi4+l2": [0, 5, 10, 15, 25, 24],
    "hi4+l3": [0, 5, 10, 15, 25, 24, 23],
}


def circuit(qubits, depth):
    g = []
    for layer in range(1, depth + 1):
        kind = Q.QSIM_SX if layer % 2 else Q.QSIM_SY
        for q in qubits:  # the same bits in both halves (lower qubit 28 + q has local bit 27 - q)
            g.append((layer, kind, q, Q.QSIM_NO_QUBIT))
            g.append((layer, kind, 28 + q, Q.QSIM_NO_QUBIT))
    return np.array(g, dtype=np.uint32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="c64")
    ap.add_argument("--reps", type=int, default=24)
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--kernel", type=int, default=0, help="QSIM_OPT_SWEEP_KERNEL")
    a = ap.parse_args()
    prec = Q.QSIM_C128 if a.precision == "c128" else Q.QSIM_C64
    for name in a.cases.split(","):
        ctx = Q.qsim_create(prec, 0)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_LAZY_LAST, 0)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_SWEEP_KERNEL, a.kernel)
        Q.qsim_load_circuit(ctx, 8, 7, a.reps, circuit(CASES[name], a.reps))
        Su = np.arange(64, dtype=np.uint64)
        Q.qsim_set_blocks(ctx, Su, Su)
        Q.qsim_evolve_range(ctx, 0, 1)  # warm-up
        Q.qsim_synchronize(ctx)
        Q.qsim_stats_reset(ctx)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
        Q.qsim_reset_block(ctx)
        Q.qsim_evolve_range(ctx, 0, 1)
        Q.qsim_synchronize(ctx)
        st = Q.qsim_stats(ctx)
        Q.qsim_destroy(ctx)
        print(json.dumps({"case": name, "sweeps": st["timed_sweeps"], "sweep_ms": st["sweep_ms"],
                          "GBps": st["sweep_bytes"] / (st["sweep_ms"] * 1e-3) / 1e9,
                          "avg_us": 1e3 * st["sweep_ms"] / max(1, st["timed_sweeps"])}), flush=True)


if __name__ == "__main__":
    main()
