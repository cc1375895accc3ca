"""Times the whole C5 job (every branch, one qsim_evolve_range) in one process: python tools/job_time.py
[--precision c64|c128] [--config C5] [--reps 2].  Prints the device time per job, the stats and the
host time spent issuing the job (the frame executor's bookkeeping)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import CONFIGS, generate, sample_block  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="c128")
ap.add_argument("--config", default="C5")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--time", action="store_true", help="events around every sweep / GEMM launch")
a = ap.parse_args()
rows, cols, depth, lu, ll = CONFIGS[a.config]
circ = generate(rows, cols, depth, a.seed)
Su = sample_block(circ.h_upper, 1 << lu, a.seed + 1)
Sl = sample_block(circ.h_lower, 1 << ll, a.seed + 2)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
prec = Q.QSIM_C128 if a.precision == "c128" else Q.QSIM_C64
ctx = Q.qsim_create(prec, 0)
Q.qsim_set_stream(ctx, stream.cuda_stream)
Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
c, B, cuts = Q.qsim_partition(ctx)
Q.qsim_set_blocks(ctx, Su, Sl)
if a.time:
    Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
for r in range(a.reps):
    Q.qsim_reset_block(ctx)
    Q.qsim_stats_reset(ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    Q.qsim_evolve_range(ctx, 0, B)
    t_issue = time.perf_counter() - t0
    Q.qsim_sample(ctx, 7, 1 << 20, to_host=False)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    st = Q.qsim_stats(ctx)
    print(json.dumps({"rep": r, "precision": a.precision, "job_s": t, "issue_s": t_issue,
                      "amps_per_s": Su.size * Sl.size / t, "sweeps": st["sweeps"], "undo": st["undo_sweeps"],
                      "launches": st["kernel_launches"], "gemm_flops": st["gemm_flops"],
                      "frame_leaves": st["flip_siblings"], "sweep_ms": st["sweep_ms"], "gemm_ms": st["gemm_ms"],
                      "gemm_tflops": st["gemm_flops"] / max(1e-9, st["gemm_ms"] / 1e3) / 1e12 if st["gemm_ms"] else None}), flush=True)
Q.qsim_destroy(ctx)
