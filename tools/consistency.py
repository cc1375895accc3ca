"""Cross-check of execution strategies at full size (no oracle reaches 56-64 qubits): one prefix group of
a config is evolved under several engine variants (qubit relabelling, lazy tail, sweep kernel) and the
partial blocks are compared entry by entry.  The variants share no plan: a layout or tail bug in one
of them shows up as a disagreement.

    python tools/consistency.py --config C5 --group 3 --variants auto/2,id/0,auto/0
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import generate, sample_block, CONFIGS  # noqa: E402


def block(cfg, group, perm, lazy, kernel, prec, nu, nl):
    rows, cols, depth, lu, ll = CONFIGS[cfg]
    circ = generate(rows, cols, depth, 0)
    os.environ["QSIM_PERM"] = perm
    ctx = Q.qsim_create(prec, 0)
    try:
        Q.qsim_set_option(ctx, Q.QSIM_OPT_LAZY_LAST, lazy)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_SWEEP_KERNEL, kernel)
        Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
        Su = sample_block(circ.h_upper, 1 << (lu or circ.h_upper), 1)[:nu]
        Sl = sample_block(circ.h_lower, 1 << (ll or circ.h_lower), 2)[:nl]
        Q.qsim_set_blocks(ctx, Su, Sl)
        _, nb, cuts = Q.qsim_partition(ctx)
        g = nb >> int(sum(1 for c in cuts if c[0] <= 8))
        Q.qsim_evolve_range(ctx, group * g, (group + 1) * g)
        return Q.qsim_amplitudes(ctx, Su, Sl, prec).astype(np.complex128)
    finally:
        Q.qsim_destroy(ctx)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--group", type=int, default=3)
    ap.add_argument("--variants", default="auto/2/0,id/0/0,auto/0/1")
    ap.add_argument("--precision", default="c64")
    ap.add_argument("--nu", type=int, default=2048)
    ap.add_argument("--nl", type=int, default=2048)
    a = ap.parse_args()
    prec = Q.QSIM_C128 if a.precision == "c128" else Q.QSIM_C64
    ref = None
    for v in a.variants.split(","):
        perm, lazy, kernel = v.split("/")
        A = block(a.config, a.group, perm, int(lazy), int(kernel), prec, a.nu, a.nl)
        if ref is None:
            ref, name = A, v
            print(json.dumps({"variant": v, "rms": float(np.sqrt(np.mean(np.abs(A) ** 2)))}), flush=True)
            continue
        d = np.abs(A - ref)
        print(json.dumps({"variant": v, "vs": name, "max_abs_diff": float(d.max()),
                          "max_rel_to_max": float(d.max() / np.abs(ref).max())}), flush=True)


if __name__ == "__main__":
    main()
