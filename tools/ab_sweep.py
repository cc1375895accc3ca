"""A/B timing of the sweep kernels on one prefix group of a config (CUDA events per launch).

    python tools/ab_sweep.py [--config C4] [--precision c64] [--kernels 0,1,2] [--branches 128]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import CONFIGS, generate, sample_block  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--precision", default="c64")
    ap.add_argument("--kernels", default="0,1,2")
    ap.add_argument("--branches", type=int, default=128)
    ap.add_argument("--lazy", default="2", help="QSIM_OPT_LAZY_LAST values, comma separated")
    ap.add_argument("--defer", default="1", help="QSIM_OPT_DEFER values (deferred forks), comma separated")
    a = ap.parse_args()
    rows, cols, depth, lu, ll = CONFIGS[a.config]
    circ = generate(rows, cols, depth, 0)
    prec = Q.QSIM_C128 if a.precision == "c128" else Q.QSIM_C64
    Su, Sl = sample_block(circ.h_upper, 1 << lu, 1), sample_block(circ.h_lower, 1 << ll, 2)
    out = {}
    for kern, lazy, defer in [(int(k), int(z), int(f)) for k in a.kernels.split(",") for z in a.lazy.split(",")
                              for f in a.defer.split(",")]:
        ctx = Q.qsim_create(prec, 0)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_SWEEP_KERNEL, kern)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_LAZY_LAST, lazy)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_DEFER, defer)
        Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
        Q.qsim_set_blocks(ctx, Su, Sl)
        Q.qsim_evolve_range(ctx, 0, a.branches)          # warm-up
        Q.qsim_synchronize(ctx)
        Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
        Q.qsim_stats_reset(ctx)
        t0 = time.perf_counter()
        Q.qsim_evolve_range(ctx, a.branches, 2 * a.branches)
        Q.qsim_synchronize(ctx)
        wall = time.perf_counter() - t0
        st = Q.qsim_stats(ctx)
        Q.qsim_destroy(ctx)
        out[(kern, lazy, defer)] = {"kernel": kern, "lazy": lazy, "defer": defer, "wall_s": wall, "sweeps": st["sweeps"], "sweep_ms": st["sweep_ms"],
                     "GBps": st["sweep_bytes"] / (st["sweep_ms"] / 1e3) / 1e9,
                     "avg_us": st["sweep_ms"] / max(1, st["timed_sweeps"]) * 1e3}
        print(json.dumps(out[(kern, lazy, defer)]), flush=True)


if __name__ == "__main__":
    main()
