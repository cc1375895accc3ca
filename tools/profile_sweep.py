"""Small driver for ncu captures: one bench step of a config (one first-period prefix group of
branches through the C-ABI: both half trees, gathers, GEMM, |a|^2 + draws), nothing else.

    python tools/profile_sweep.py [--config C5] [--precision c64] [--group 0] [--branches N]
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
    ap.add_argument("--config", default="C5")
    ap.add_argument("--precision", default="c64")
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--branches", type=int, default=0, help="branches per step (0: one prefix group)")
    ap.add_argument("--kernel", type=int, default=0, help="QSIM_OPT_SWEEP_KERNEL")
    a = ap.parse_args()
    rows, cols, depth, lu, ll = CONFIGS[a.config]
    circ = generate(rows, cols, depth, 0)
    prec = Q.QSIM_C128 if a.precision == "c128" else Q.QSIM_C64
    ctx = Q.qsim_create(prec, 0)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_SWEEP_KERNEL, a.kernel)
    Q.qsim_load_circuit(ctx, rows, cols, depth, circ.gate_array())
    c, B, cuts = Q.qsim_partition(ctx)
    first = sorted({int(x[0]) for x in cuts})[:2]
    per = a.branches or B >> sum(1 for x in cuts if int(x[0]) in first)
    Q.qsim_set_blocks(ctx, sample_block(circ.h_upper, 1 << lu, 1), sample_block(circ.h_lower, 1 << ll, 2))
    Q.qsim_evolve_range(ctx, a.group * per, (a.group + 1) * per)
    Q.qsim_sample(ctx, 7, 1 << 20, to_host=False)
    Q.qsim_synchronize(ctx)
    st = Q.qsim_stats(ctx)
    print({k: st[k] for k in ("sweeps", "kernel_launches", "sweep_bytes", "sweep_bytes_moved")})
    Q.qsim_destroy(ctx)


if __name__ == "__main__":
    main()
