"""Times the reconstruction GEMM alone through qsim_branch_sum (host slices, device-timed with the
library's CUDA events): python tools/gemm_bench.py [--K 8192] [--M 8192] [--N 8192] [--precision c128]
[--reps 3].  QSIM_GEMM=4m selects the four-product kernel (A/B)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1802_06952_b200 import qsim as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=8192)
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--N", type=int, default=8192)
ap.add_argument("--precision", default="c128")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
prec = Q.QSIM_C128 if a.precision == "c128" else Q.QSIM_C64
dt = np.complex128 if prec == Q.QSIM_C128 else np.complex64
rng = np.random.default_rng(1)
U = (rng.standard_normal((a.K, a.M)) + 1j * rng.standard_normal((a.K, a.M))).astype(dt)
L = (rng.standard_normal((a.K, a.N)) + 1j * rng.standard_normal((a.K, a.N))).astype(dt)
ctx = Q.qsim_create(prec, 0)
Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
for r in range(a.reps):
    Q.qsim_stats_reset(ctx)
    A = Q.qsim_branch_sum(ctx, U, L, prec)
    st = Q.qsim_stats(ctx)
    t = st["gemm_ms"] / 1e3
    print(json.dumps({"rep": r, "K": a.K, "M": a.M, "N": a.N, "precision": a.precision, "gemm_s": t,
                      "tflops_8mnk": st["gemm_flops"] / t / 1e12, "tflops_executed_3m": 0.75 * st["gemm_flops"] / t / 1e12}),
          flush=True)
if a.K * a.M * a.N <= (1 << 33):  # spot check against numpy on a corner
    ref = U[:, :64].T @ L[:, :64]
    print("max rel err (64x64 corner):", float(np.abs(A[:64, :64] - ref).max() / np.abs(ref).max()))
Q.qsim_destroy(ctx)
