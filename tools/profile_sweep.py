"""Small driver for ncu captures of the gate sweep: loads a config, evolves a few branches.

    python tools/profile_sweep.py [--config C4] [--precision c64] [--branches 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import CONFIGS, generate, sample_block  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--precision", default="c64")
    ap.add_argument("--branches", type=int, default=2)
    ap.add_argument("--kernel", type=int, default=0, help="QSIM_OPT_SWEEP_KERNEL")
    a = ap.parse_args()
    rows, cols, depth, lu, ll = CONFIGS[a.config]
    circ = generate(rows, cols, depth, 0)
    prec = Q.QSIM_C128 if a.precision == "c128" else Q.QSIM_C64
    ctx = Q.qsim_create(prec, 0)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_SWEEP_KERNEL, a.kernel)
    Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
    Q.qsim_set_blocks(ctx, sample_block(circ.h_upper, 1 << lu, 1), sample_block(circ.h_lower, 1 << ll, 2))
    Q.qsim_evolve_range(ctx, 0, a.branches)
    Q.qsim_synchronize(ctx)
    st = Q.qsim_stats(ctx)
    print({k: st[k] for k in ("sweeps", "kernel_launches", "sweep_bytes")})
    Q.qsim_destroy(ctx)


if __name__ == "__main__":
    main()
