"""Small end-to-end cases for compute-sanitizer (tests/test_gpu_sanitizer.py): C1 (Fig. 1, the
in-shared-memory kernel), C2-sized tree mode (h = 12, c128), and an h = 14 depth-22 deferred-fork
tree over a few branches (TMA sweep with 2 CTAs, node-batched levels on / off, lazy tail), plus the
sampler and the Porter-Thomas analyzer — every kernel family of the hot path, at sizes the
sanitizer's slowdown allows.  Exits non-zero on a numerical mismatch with the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import partition as OP, statevector as SV  # noqa: E402
from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import generate, sample_block  # noqa: E402


def block(circ, Su, Sl, prec, ranges, opts):
    ctx = Q.qsim_create(prec, 0)
    try:
        for k, v in opts.items():
            Q.qsim_set_option(ctx, k, v)
        Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
        Q.qsim_set_blocks(ctx, Su, Sl)
        for (b0, b1) in ranges:
            Q.qsim_evolve_range(ctx, b0, b1)
        A = Q.qsim_amplitudes(ctx, Su, Sl)
        x, W = Q.qsim_sample(ctx, 5, 4096)
        pt, _, _ = Q.qsim_porter_thomas(ctx, n_bins=64)
        return A, x, W
    finally:
        Q.qsim_destroy(ctx)


def main():
    bad = 0
    circ = generate(4, 2, 8, 0)
    ref = SV.simulate(circ).reshape(16, 16)
    for prec in (Q.QSIM_C64, Q.QSIM_C128):
        A, _, _ = block(circ, np.arange(16), np.arange(16), prec, [(0, 4)], {})
        bad += np.abs(A - ref).max() > 1e-5
    circ = generate(4, 7, 22, 11)
    Su, Sl = sample_block(14, 40, 3), sample_block(14, 24, 4)
    ref = OP.amplitudes(circ, Su, Sl, branches=range(1000, 1008))
    for bfs in (0, 1):
        A, _, _ = block(circ, Su, Sl, Q.QSIM_C128, [(1000, 1008)],
                        {Q.QSIM_OPT_BFS: bfs, Q.QSIM_OPT_MAX_CTAS: 2, Q.QSIM_OPT_LAZY_LAST: 3})
        bad += np.abs(A - ref).max() > 1e-12
    A, _, _ = block(circ, Su, Sl, Q.QSIM_C64, [(1000, 1008)], {Q.QSIM_OPT_MAX_CTAS: 2, Q.QSIM_OPT_SWEEP_KERNEL: 3})
    bad += np.abs(A - ref).max() / np.abs(ref).max() > 1e-5
    print("sanitize cases:", "FAIL" if bad else "ok")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
