"""2-, 3- and 4-part partitions of one circuit, timed through the C-ABI.

    python tools/multipart_bench.py --grid 8x8 --depth 8 --schemes 4 3,5 2,4,6 --amps 24

For each scheme (row cuts) the same number of sampled amplitudes (2^amps, split evenly over
the parts) is computed by ``qsim_multipart_amplitudes``; with --halves the bipartition is also
run through the default two-half path (``qsim_evolve_halves`` + ``qsim_amplitudes``) and the
two results are compared.  Prints one JSON line per run: wall time (host buffers in,
amplitudes out), sweep time and bytes (CUDA events per launch), GEMM flops, launches, the
planner's log2 leaf amplitudes, and mean(N |a|^2) over the block (~1 once scrambled).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import generate, sample_block  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="8x8")
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--schemes", nargs="+", default=["4", "3,5", "2,4,6"])
    ap.add_argument("--amps", type=int, default=24, help="log2 of the sampled amplitudes")
    ap.add_argument("--prec", default="c64")
    ap.add_argument("--halves", action="store_true", help="also run the two-half path")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    rows, cols = map(int, a.grid.split("x"))
    prec = Q.QSIM_C64 if a.prec == "c64" else Q.QSIM_C128
    circ = generate(rows, cols, a.depth, 0)
    for sch in a.schemes:
        rc = [int(x) for x in sch.split(",")]
        bounds = [0] + rc + [rows]
        t = len(bounds) - 1
        nq = [(bounds[k + 1] - bounds[k]) * cols for k in range(t)]
        per = [a.amps // t + (1 if k < a.amps % t else 0) for k in range(t)]
        blocks = [sample_block(nq[k], 1 << min(per[k], nq[k]), 100 + k) for k in range(t)]
        ctx = Q.qsim_create(prec, 0)
        try:
            Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
            Q.qsim_load_circuit(ctx, rows, cols, a.depth, circ.gate_array())
            plan = Q.qsim_multipart_plan(ctx, rc)
            best = None
            for _ in range(a.reps):
                Q.qsim_stats_reset(ctx)
                t0 = time.perf_counter()
                A = Q.qsim_multipart_amplitudes(ctx, rc, blocks, prec)
                wall = time.perf_counter() - t0
                st = Q.qsim_stats(ctx)
                if best is None or wall < best[0]:
                    best = (wall, st)
            wall, st = best
            line = {"grid": a.grid, "depth": a.depth, "prec": a.prec, "row_cuts": rc, "parts": nq,
                    "boundary_cuts": plan["boundary_cuts"], "log2_states": round(plan["log2_states"], 3),
                    "amplitudes": int(A.size), "wall_s": wall, "amps_per_s": A.size / wall,
                    "sweep_ms": st["sweep_ms"],
                    "sweep_GBps": (st["sweep_bytes"] / 1e6 / st["sweep_ms"]) if st["sweep_ms"] else None,
                    "sweeps": st["sweeps"], "launches": st["kernel_launches"], "gemm_tflop": st["gemm_flops"] / 1e12,
                    "mean_Np": float(np.mean(np.abs(A.astype(np.complex128)) ** 2) * 2.0 ** circ.n)}
            print(json.dumps(line), flush=True)
        finally:
            Q.qsim_destroy(ctx)
        if a.halves and len(rc) == 1:
            Su = np.asarray(blocks[0], dtype=np.uint64)
            Sl = np.asarray(blocks[1], dtype=np.uint64)
            ctx = Q.qsim_create(prec, 0)
            try:
                Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
                Q.qsim_load_circuit(ctx, rows, cols, a.depth, circ.gate_array(), rc[0])
                t0 = time.perf_counter()
                Q.qsim_evolve_halves(ctx, Su, Sl)
                B = Q.qsim_amplitudes(ctx, Su, Sl, prec)
                wall = time.perf_counter() - t0
                st = Q.qsim_stats(ctx)
                err = float(np.abs(B.astype(np.complex128) - A.astype(np.complex128)).max() / np.abs(B).max())
                print(json.dumps({"grid": a.grid, "depth": a.depth, "row_cuts": rc,
                                  "path": "two-half (qsim_evolve_halves)", "wall_s": wall,
                                  "amps_per_s": B.size / wall, "sweep_ms": st["sweep_ms"],
                                  "launches": st["kernel_launches"], "rel_diff_vs_multipart": err}), flush=True)
            finally:
                Q.qsim_destroy(ctx)


if __name__ == "__main__":
    main()
