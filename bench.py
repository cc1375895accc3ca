#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--precision c64]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle arm

Workload (default, every N): config C5 = the metric's configuration, 64-qubit 8x8 grid,
depth 22, 16 cut CZs -> 2^16 branches, sampled block 2^14 x 2^14 = 2^28 amplitudes (it fits
one B200: 32 GiB c64 half states).  --config C4 (56q 8x7) / C3 (42q 6x7) for the smaller
BASELINE.json configurations.

One STEP = one of the 2^8 first-period prefix groups of that job (256 branches sharing the
cuts of layers 7-8): both half-circuit branch trees (all prefix-shared sweeps from layer 1),
leaf gathers, the GEMM accumulation A += U^T L, then |a|^2 + prefix tables + 2^20 Philox
draws.  Every group costs the same (identical structure, other projector bits), so the
whole-job rate is exact:  value = 2^28 * (groups done) / 256 / time.  Each rank does one
group per step (weak scaling); partial blocks are summed with NCCL every step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep rank 0's stdout to the one JSON line

import numpy as np  # noqa: E402

METRIC = "64q d22: sampled amplitudes/s; half-circuit gate-sweep HBM GB/s vs peak"
UNIT = "sampled amplitudes/s"
N_DRAWS = 1 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=["C3", "C4", "C5"])
    ap.add_argument("--precision", default="c64", choices=["c64", "c128"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload(cfg: str, seed: int):
    from workloads import CONFIGS, generate, sample_block
    rows, cols, depth, lu, ll = CONFIGS[cfg]
    circ = generate(rows, cols, depth, seed)
    Su = sample_block(circ.h_upper, 1 << lu, seed + 1)
    Sl = sample_block(circ.h_lower, 1 << ll, seed + 2)
    return circ, Su, Sl


def first_period_bits(cuts):
    layers = sorted({int(c[0]) for c in cuts})
    first = set(layers[:2])
    return sum(1 for c in cuts if int(c[0]) in first)


# ---------------------------------------------------------------- CPU oracle timing
def oracle_sample(circ, budget_s: float = 20.0, max_gates: int | None = None):
    """Time the oracle's gate-by-gate half-circuit evolution (branch 0, upper half, full h)
    for ~budget_s seconds; extrapolate to the flat partitioned job (§2.3.1: every branch
    from scratch).  Returns (seconds per gate application, gate applications of the job,
    gates timed)."""
    from oracle import partition as OP, statevector as SV
    cuts = OP.cut_list(circ)
    c = len(cuts)
    gu = OP.half_gates(circ, OP.UPPER, cuts, 0)
    gl = OP.half_gates(circ, OP.LOWER, cuts, 0)
    per_branch = len(gu) + len(gl) + circ.h_upper + circ.h_lower   # + layer-0 H on each qubit
    job_gate_apps = (1 << c) * per_branch + (1 << max(c - 1, 0)) * c  # + Z gates (popcount)
    h = circ.h_upper
    # bounded host memory: above 28 qubits the oracle runs the gates of the first 28 qubits on a
    # 2^28 state and the time per gate is scaled by 2^(h - 28) (a gate application is one pass
    # over the state: its cost is linear in the state size)
    hs = min(h, 28)
    scale = float(1 << (h - hs))
    gs = [g for g in gu if int(g[2]) < hs and (g[1] not in (4, "CZ") or int(g[3]) < hs)]
    psi = np.full(1 << hs, 2.0 ** (-h / 2), dtype=np.complex128)  # H^{(x)h}|0> (pinned closed form)
    t0 = time.perf_counter()
    done = 0
    for g in gs:
        psi = SV.run_gates(psi, hs, [g])
        done += 1
        if time.perf_counter() - t0 > budget_s or (max_gates and done >= max_gates):
            break
    dt = time.perf_counter() - t0
    return dt / done * scale, job_gate_apps, done


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    circ, Su, Sl = workload(args.config, args.seed)
    n_amp = Su.size * Sl.size
    times = []
    per_gate = None
    job = None
    for i in range(args.warmup + args.steps):
        tg, job, _ = oracle_sample(circ, budget_s=0.0, max_gates=1)   # one gate application
        if i >= args.warmup:
            times.append(tg)
    per_gate = sum(times) / len(times)
    t_job = per_gate * job
    value = n_amp / t_job
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_gate * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config} (oracle, flat partitioned simulator, numpy complex128)",
                   "extrapolated_job_s": t_job, "gate_applications_per_job": job},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"each step = 1 oracle gate application on a 2^{min(circ.h_upper, 28)} "
                                   f"complex128 state (branch 0, upper half"
                                   + (f"; x 2^{circ.h_upper - 28} for the 2^{circ.h_upper} half" if circ.h_upper > 28 else "")
                                   + f"); job = {job} gate applications (flat: every branch from scratch), "
                                   "extrapolated"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            print(json.dumps({"error": "run --gpus N > 1 under torch.distributed.run"}))
            sys.exit(2)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1802_06952_b200 import qsim as Q

    prec = Q.QSIM_C128 if args.precision == "c128" else Q.QSIM_C64
    circ, Su, Sl = workload(args.config, args.seed)
    n_u, n_l = Su.size, Sl.size
    stream = torch.cuda.Stream()          # a real stream (the legacy default stream has handle 0)
    torch.cuda.set_stream(stream)
    ctx = Q.qsim_create(prec, local)
    Q.qsim_set_stream(ctx, stream.cuda_stream)
    Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
    if world > 1:
        uid = [Q.qsim_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        Q.qsim_comm_init(ctx, rank, world, uid[0])
    c, B, cuts = Q.qsim_partition(ctx)
    gbits = first_period_bits(cuts)
    G = 1 << gbits
    per_group = B // G

    # pinned host buffers for the end-to-end leg
    pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
    hSu, hSl = pin((n_u,), torch.int64).view(np.uint64), pin((n_l,), torch.int64).view(np.uint64)
    hSu[:] = Su
    hSl[:] = Sl
    hA = pin((n_u, n_l), torch.complex128 if prec == Q.QSIM_C128 else torch.complex64)
    hX = pin((N_DRAWS,), torch.int64).view(np.uint64)

    Q.qsim_set_blocks(ctx, hSu, hSl)

    def group_of(step):
        return (step * world + rank) % G

    def step_device(s):
        g = group_of(s)
        Q.qsim_reset_block(ctx)
        Q.qsim_evolve_range(ctx, g * per_group, (g + 1) * per_group)
        Q.qsim_sample(ctx, 1000 + s, N_DRAWS, to_host=False)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---------------- warmup
    for s in range(args.warmup):
        step_device(s)
    barrier()

    # ---------------- timed region (device events on the launching stream)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
    Q.qsim_stats_reset(ctx)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s in range(args.warmup, args.warmup + args.steps):
        step_device(s)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    t_dev = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    st = Q.qsim_stats(ctx)
    Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 0)
    launches = int(sum_over_ranks(st["kernel_launches"]))

    groups_done = world * args.steps
    value = (n_u * n_l) * groups_done / G / t_dev

    # ---------------- end-to-end through the C-ABI with host buffers
    k_e2e = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 3 if circ.n < 64 else 1))
    barrier()
    t0 = time.perf_counter()
    for s in range(k_e2e):  # 0 steps: e2e skipped (profiling runs)
        g = group_of(args.warmup + s)
        Q.qsim_set_blocks(ctx, hSu, hSl)                                        # H2D of the inputs
        Q.qsim_evolve_range(ctx, g * per_group, (g + 1) * per_group)
        Q.qsim_amplitudes(ctx, hSu, hSl, prec, out=hA, write=(rank == 0))     # D2H of the block
        Q.qsim_sample(ctx, 2000 + s, N_DRAWS, to_host=(rank == 0), out=hX)     # D2H of the draws
    barrier()
    t_e2e = max_over_ranks(time.perf_counter() - t0)
    e2e_value = (n_u * n_l) * world * k_e2e / G / t_e2e if k_e2e else None
    amp_bytes = 16 if prec == Q.QSIM_C128 else 8
    h2d = (n_u + n_l) * 8 * world
    d2h = n_u * n_l * amp_bytes + N_DRAWS * 8 + 8

    # ---------------- roofline of the dominant kernel (the gate sweep)
    peak, peak_src = peaks()
    sweep_s = st["sweep_ms"] / 1e3
    achieved = st["sweep_bytes"] / sweep_s / 1e9 if sweep_s > 0 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            traffic = pj.get(f"{args.config}_{args.precision}", {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---------------- CPU baseline (oracle, rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            tg, job, done = oracle_sample(circ, budget_s=20.0)
            cpu = {"value": (n_u * n_l) / (tg * job), "unit": UNIT, "cores": 1, "kind": "oracle",
                   "sample": f"{done} gate applications of the oracle (numpy complex128, 1 thread) on a "
                             f"2^{min(circ.h_upper, 28)}-amplitude state (branch 0, upper half"
                             + (f"; x 2^{circ.h_upper - 28} for the 2^{circ.h_upper} half" if circ.h_upper > 28 else "")
                             + f"); extrapolated to the flat job's {job} gate applications ({B} branches x 2 halves)"}
        except MemoryError:
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle",
                   "sample": "host out of memory for a full half state"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if prec == Q.QSIM_C64 else "f64", "data": "synthetic",
            "config": {
                "workload": f"{args.config}: {circ.n}q {circ.rows}x{circ.cols} grid depth {circ.depth} random "
                            f"circuit (App. A.1 rules, seed {args.seed}), {c} cut CZs -> {B} branches, "
                            f"sampled block {n_u} x {n_l}",
                "precision": f"{args.precision} ({'f32' if prec == Q.QSIM_C64 else 'f64'} half-state sweeps, "
                             "f64 reconstruction GEMM)",
                "step": f"1 of {G} first-period prefix groups ({per_group} branches) per rank: both half "
                        f"trees from layer 1, gathers, GEMM-accumulate, |a|^2 + {N_DRAWS} draws",
                "projected_full_job_s": t_dev / args.steps * G / world,
                "l2": f"inputs larger than L2: half states of {((1 << circ.h_upper) * amp_bytes) >> 20} MiB",
                "parallelism": f"branch-sharded dp{world}",
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "peak_source": peak_src, "kernel": "tile_sweep_kernel",
                         "launches": st["timed_sweeps"],
                         "bytes_per_launch": st["sweep_bytes"] / max(1, st["sweeps"]),
                         "avg_launch_us": sweep_s / max(1, st["timed_sweeps"]) * 1e6,
                         "share_of_step": sweep_s / (t_dev * 1.0) if t_dev else None,
                         "gemm_tflops": (st["gemm_flops"] / (st["gemm_ms"] / 1e3) / 1e12)
                         if st["gemm_ms"] > 0 else None},
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": k_e2e},
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    Q.qsim_destroy(ctx)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
