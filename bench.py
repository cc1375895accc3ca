#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--precision c64]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle arm

Workload (default, every N): config C5 = the metric's configuration, 64-qubit 8x8 grid,
depth 22, 16 cut CZs -> 2^16 branches, sampled block 2^14 x 2^14 = 2^28 amplitudes, in c128
(the paper's double precision: 64 GiB half states on one B200); the c64 figure follows as
"secondary".  --config C4 (56q 8x7) / C3 (42q 6x7) for the smaller BASELINE.json configurations.
The timed region carries no per-launch events; the roofline numbers come from one extra
profiling step with CUDA events around every sweep launch.

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
    ap.add_argument("--precision", default="c128", choices=["c64", "c128"])
    ap.add_argument("--secondary-steps", type=int, default=2,
                    help="timed steps of the other precision (reported as 'secondary'; 0: skip)")
    ap.add_argument("--ref-gates", type=int, default=4, help="oracle gate applications per reference step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--step", default="job", choices=["job", "group"],
                    help="job: one step = the whole job (every branch; ranks split the branch range); "
                         "group: one step = one first-period prefix group per rank (round-1 definition)")
    return ap.parse_args()


# FP64 tensor ceiling measured on B200 with tools/native/dmma_peak.cu (register-only m8n8k4 DMMAs,
# 8-32 warps per SM; profiles/r02/r02w_dmma_peak.txt)
DMMA_CEILING = 37.1


def fp64_peak():
    """FP64 tensor peak by the profiling recipe's rule: another dtype's measured peak x the nominal ratio
    (MEASURED_PEAKS.json bf16 burst x 45 / 2250, the B200 FP64-tensor / BF16 dense nominals)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]) * 45.0 / 2250.0, "MEASURED_PEAKS.json bf16_tflops x 45/2250 (FP64 tensor / BF16 nominal)"
    except Exception:
        return 45.0, "nominal B200 FP64 tensor (guide)"


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
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_gate_counts(circ):
    """Gate applications of the oracle's partitioned simulator (oracle/partition.py) on this circuit.
    flat: every branch from scratch (the oracle as it stands, §2.3.1): per branch and half the
    initial state (one pass) + the internal gates + the branch gates (P_b on every upper cut endpoint,
    Z on the lower ones whose bit is 1: c / 2 on average).  shared: the same gate lists with the
    prefix shared at every cut layer (the paper's §2.3.2 scheme): the gates of layer t run once per
    distinct branch prefix 2^{#cuts before t}, the branch gates of layer t once per 2^{#cuts <= t}."""
    from oracle import partition as OP
    cuts = OP.cut_list(circ)
    c = len(cuts)
    B = 1 << c
    hu = circ.h_upper
    per_layer = {}
    n_int = 0
    for (layer, kind, q0, q1) in circ.gates:
        qs = [int(q0)] if kind != 4 else [int(q0), int(q1)]
        if all(q < hu for q in qs) or all(q >= hu for q in qs):
            per_layer[int(layer)] = per_layer.get(int(layer), 0) + 1
            n_int += 1
    flat = B * (n_int + 2) + B * c + B * c // 2
    cut_layers = [cl for (cl, _, _) in cuts]
    shared = 2.0  # initial states
    for t in range(1, circ.depth + 1):
        before = sum(1 for cl in cut_layers if cl < t)
        at = sum(1 for cl in cut_layers if cl == t)
        shared += per_layer.get(t, 0) * 2.0 ** before
        shared += at * 2.0 ** (before + at) * 1.5  # P on the upper endpoint, Z (half of them) on the lower
    return flat, shared


class OracleClock:
    """The oracle (oracle/fast.py: the numpy oracle's gate lists applied one at a time by the plain C
    + OpenMP loop) timed on the box's host cores on a FULL half state of the workload (2^h complex128:
    64 GiB at C5) - branch 0, upper half, gates in list order."""

    def __init__(self, circ):
        from oracle import fast as OF, partition as OP
        self.OF = OF
        self.circ = circ
        self.h = circ.h_upper
        self.gates = OP.half_gates(circ, OP.UPPER, OP.cut_list(circ), 0)
        self.cores = OF.max_threads()
        t0 = time.perf_counter()
        self.psi = OF.initial_state(self.h, self.cores)
        self.t_init = time.perf_counter() - t0
        self.next = 0

    def run(self, n_gates: int, threads: int) -> float:
        """Applies the next n_gates gates of the list (cyclically); returns the seconds taken."""
        gl = [self.gates[(self.next + i) % len(self.gates)] for i in range(n_gates)]
        self.next += n_gates
        t0 = time.perf_counter()
        self.OF.run_gates(self.psi, self.h, gl, threads)
        return time.perf_counter() - t0

    def per_gate(self, budget_s: float, threads: int):
        done, spent = 0, 0.0
        while spent < budget_s or done == 0:
            spent += self.run(1, threads)
            done += 1
        return spent / done, done


def cpu_baseline(circ, n_amp, budget_s: float = 12.0):
    """cpu_baseline of the JSON line: the oracle on all host cores and on one core, extrapolated from
    the measured time per gate application on the full half state to the flat job (and, for
    reference, to the prefix-shared job)."""
    flat, shared = oracle_gate_counts(circ)
    oc = OracleClock(circ)
    tg_all, n_all = oc.per_gate(budget_s, oc.cores)
    tg_one, n_one = oc.per_gate(budget_s, 1)
    del oc.psi
    return {
        "value": n_amp / (tg_all * flat), "unit": UNIT, "cores": oc.cores, "kind": "oracle",
        "one_core_value": n_amp / (tg_one * flat),
        "prefix_shared_value": n_amp / (tg_all * shared),
        "cpu_model": cpu_model(),
        "sample": f"oracle (oracle/fast.py: numpy oracle gate lists, plain C + OpenMP pair loop, complex128) "
                  f"on a full 2^{circ.h_upper}-amplitude half state (branch 0, upper half): {n_all} gate "
                  f"applications on {oc.cores} threads ({tg_all:.3f} s each) and {n_one} on 1 thread "
                  f"({tg_one:.3f} s each); extrapolated to the flat job's {flat} gate applications "
                  f"(every branch from scratch, as oracle/partition.py runs it); prefix_shared_value: "
                  f"the same per-gate time x {shared:.4g} applications with prefixes shared at cut layers",
    }


def run_reference(args):
    """The reference arm: the oracle as it stands, timed on the host cores, each step a bounded
    sample of the workload (gate applications on the full half state, all cores)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    circ, Su, Sl = workload(args.config, args.seed)
    n_amp = Su.size * Sl.size
    flat, shared = oracle_gate_counts(circ)
    oc = OracleClock(circ)
    per_step = max(1, int(args.ref_gates))
    for _ in range(args.warmup):
        oc.run(per_step, oc.cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oc.run(per_step, oc.cores)
    t_steps = time.perf_counter() - t0
    per_gate = t_steps / (args.steps * per_step)
    value = n_amp / (per_gate * flat)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_steps / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config} (oracle: flat partitioned simulator, complex128, "
                               f"{oc.cores} host threads)",
                   "step": f"{per_step} oracle gate applications on the full 2^{circ.h_upper} half state",
                   "extrapolated_job_s": per_gate * flat, "gate_applications_per_job": flat,
                   "prefix_shared_job_s": per_gate * shared, "state_init_s": oc.t_init},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oc.cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"each step = {per_step} gate applications of the oracle (plain C + OpenMP "
                                   f"pair loop) on the full 2^{circ.h_upper} complex128 half state (branch 0, "
                                   f"upper half); job = {flat} gate applications (flat: every branch from "
                                   "scratch), extrapolated from the measured steps"},
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

    circ, Su, Sl = workload(args.config, args.seed)
    n_u, n_l = Su.size, Sl.size
    stream = torch.cuda.Stream()          # a real stream (the legacy default stream has handle 0)
    torch.cuda.set_stream(stream)
    uid = None
    if world > 1:
        box = [Q.qsim_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce(x, op):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    max_over_ranks = lambda x: reduce(x, dist.ReduceOp.MAX if dist else None)
    sum_over_ranks = lambda x: reduce(x, dist.ReduceOp.SUM if dist else None)
    pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
    hSu, hSl = pin((n_u,), torch.int64).view(np.uint64), pin((n_l,), torch.int64).view(np.uint64)
    hSu[:] = Su
    hSl[:] = Sl
    hX = pin((N_DRAWS,), torch.int64).view(np.uint64)

    def run_precision(prec, steps, warmup, full):
        """warmup + `steps` timed steps (no per-launch events inside the timed region); with `full`:
        the clocks sampler, one extra profiling step with events around every sweep / GEMM launch (the
        roofline numbers) and the end-to-end leg through the C-ABI with host buffers."""
        ctx = Q.qsim_create(prec, local)
        Q.qsim_set_stream(ctx, stream.cuda_stream)
        Q.qsim_load_circuit(ctx, circ.rows, circ.cols, circ.depth, circ.gate_array(), circ.cut_row)
        if world > 1:
            Q.qsim_comm_init(ctx, rank, world, uid)
        c, B, cuts = Q.qsim_partition(ctx)
        if args.step == "job":  # the whole job per step: this rank's prefix-aligned branch range
            G = 1
            per_group = B
            rb0, rb1 = Q.qsim_rank_range(ctx) if world > 1 else (0, B)
            range_of = lambda step: (rb0, rb1)
        else:
            G = 1 << first_period_bits(cuts)
            per_group = B // G
            group_of = lambda step: (step * world + rank) % G
            range_of = lambda step: (group_of(step) * per_group, (group_of(step) + 1) * per_group)
        Q.qsim_set_blocks(ctx, hSu, hSl)

        def step_device(s):
            Q.qsim_reset_block(ctx)
            Q.qsim_evolve_range(ctx, *range_of(s))
            Q.qsim_sample(ctx, 1000 + s, N_DRAWS, to_host=False)

        for s in range(warmup):
            step_device(s)
        barrier()
        Q.qsim_stats_reset(ctx)
        clocks = ClockSampler(local) if full else None
        if clocks:
            clocks.start()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for s in range(warmup, warmup + steps):
            step_device(s)
        ev1.record(stream)
        barrier()
        clk = clocks.stop() if clocks else None
        t_dev = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
        st = Q.qsim_stats(ctx)
        jobs = steps if args.step == "job" else world * steps / G  # jobs completed in the timed region
        out = {"c": c, "B": B, "G": G, "per_group": per_group, "t_dev": t_dev, "clocks": clk,
               "launches": int(sum_over_ranks(st["kernel_launches"])),
               "value": (n_u * n_l) * jobs / t_dev}
        if full:
            # profiling step: CUDA events around every sweep / GEMM launch on the launching stream
            Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 1)
            Q.qsim_stats_reset(ctx)
            barrier()
            ev0.record(stream)
            step_device(warmup + steps)
            ev1.record(stream)
            barrier()
            out["prof"] = Q.qsim_stats(ctx)
            out["prof_step_s"] = ev0.elapsed_time(ev1) / 1e3
            Q.qsim_set_option(ctx, Q.QSIM_OPT_TIME_SWEEPS, 0)
            # end-to-end through the C-ABI with host buffers
            hA = pin((n_u, n_l), torch.complex128 if prec == Q.QSIM_C128 else torch.complex64)
            k_e2e = args.e2e_steps if args.e2e_steps is not None else max(1, min(steps, 3 if circ.n < 64 else 1))
            barrier()
            t0 = time.perf_counter()
            for s in range(k_e2e):  # 0 steps: e2e skipped (profiling runs)
                Q.qsim_set_blocks(ctx, hSu, hSl)                                        # H2D of the inputs
                Q.qsim_evolve_range(ctx, *range_of(warmup + s))
                Q.qsim_amplitudes(ctx, hSu, hSl, out=hA, write=(rank == 0))            # D2H of the block
                Q.qsim_sample(ctx, 2000 + s, N_DRAWS, to_host=(rank == 0), out=hX)     # D2H of the draws
            barrier()
            t_e2e = max_over_ranks(time.perf_counter() - t0)
            jobs_e2e = k_e2e if args.step == "job" else world * k_e2e / G
            out["e2e"] = (n_u * n_l) * jobs_e2e / t_e2e if k_e2e else None
            out["e2e_steps"] = k_e2e
            del hA
        Q.qsim_destroy(ctx)
        return out

    def sustained_copy(seconds=3.0, nbytes=4 << 30):
        """torch device-to-device copy of a 4 GiB buffer back to back for ~3 s right after the timed
        region (same power / thermal state): read + write bytes / event time.  Context for the roofline
        (MEASURED_PEAKS.json holds a burst copy only); the roofline's peak stays the measured burst."""
        a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        b = torch.empty_like(a)
        b.copy_(a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n, t0 = 0, time.perf_counter()
        e0.record()
        while time.perf_counter() - t0 < seconds:
            for _ in range(8):
                b.copy_(a)
            n += 8
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        gbs = 2.0 * nbytes * n / (e0.elapsed_time(e1) / 1e3) / 1e9
        del a, b
        torch.cuda.empty_cache()
        return gbs

    prec = Q.QSIM_C128 if args.precision == "c128" else Q.QSIM_C64
    main_run = run_precision(prec, args.steps, args.warmup, True)
    copy_gbs = sustained_copy() if rank == 0 else None
    sec = None
    if args.secondary_steps > 0:
        other = Q.QSIM_C64 if prec == Q.QSIM_C128 else Q.QSIM_C128
        r = run_precision(other, args.secondary_steps, 1, False)
        sec = {"precision": "c64" if other == Q.QSIM_C64 else "c128",
               "dtype": "f32" if other == Q.QSIM_C64 else "f64", "value": r["value"],
               "ms_per_step": r["t_dev"] / args.secondary_steps * 1e3, "steps": args.secondary_steps, "warmup": 1}

    c, B, G, per_group = main_run["c"], main_run["B"], main_run["G"], main_run["per_group"]
    t_dev = main_run["t_dev"]
    amp_bytes = 16 if prec == Q.QSIM_C128 else 8
    h2d = (n_u + n_l) * 8 * world
    d2h = n_u * n_l * amp_bytes + N_DRAWS * 8 + 8

    # ---------------- rooflines from the profiling step: the reconstruction GEMM (the dominant kernel
    # since the frame executor cut the sweeps to one real state per half) and the gate sweep
    st = main_run["prof"]
    peak, peak_src = peaks()
    gemm_s = st["gemm_ms"] / 1e3
    f64_peak, f64_src = fp64_peak()
    gemm_exec = 0.75 * st["gemm_flops"] / gemm_s / 1e12 if gemm_s > 0 else None  # 3M: 6MNK executed
    gemm_alg = st["gemm_flops"] / gemm_s / 1e12 if gemm_s > 0 else None         # 8MNK convention
    sweep_s = st["sweep_ms"] / 1e3
    alg = st["sweep_bytes"] / sweep_s / 1e9 if sweep_s > 0 else None
    moved = st["sweep_bytes_moved"] / sweep_s / 1e9 if sweep_s > 0 else None
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
            cpu = cpu_baseline(circ, n_u * n_l)
        except MemoryError:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                   "sample": "host out of memory for a full half state"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": main_run["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong" if args.step == "job" else "weak", "vs_baseline": None,
            "dtype": "f32" if prec == Q.QSIM_C64 else "f64", "data": "synthetic",
            "config": {
                "workload": f"{args.config}: {circ.n}q {circ.rows}x{circ.cols} grid depth {circ.depth} random "
                            f"circuit (App. A.1 rules, seed {args.seed}), {c} cut CZs -> {B} branches, "
                            f"sampled block {n_u} x {n_l}",
                "precision": f"{args.precision} ({'f32' if prec == Q.QSIM_C64 else 'f64'} half-state sweeps, "
                             "f64 reconstruction GEMM)",
                "step": (f"the whole job: all {B} branches (split over {world} rank(s) by prefix-aligned "
                         f"ranges), both half trees from layer 1 (deferred forks, Pauli frames), leaf "
                         f"gathers, GEMM-accumulate, block reduction, |a|^2 + {N_DRAWS} draws")
                        if args.step == "job" else
                        (f"1 of {G} first-period prefix groups ({per_group} branches) per rank: both half "
                         f"trees from layer 1 (deferred forks), gathers, GEMM-accumulate, |a|^2 + {N_DRAWS} draws"),
                "projected_full_job_s": t_dev / args.steps * (1 if args.step == "job" else G / world),
                "l2": f"inputs larger than L2: half states of {((1 << circ.h_upper) * amp_bytes) >> 20} MiB",
                "parallelism": f"branch-sharded dp{world}",
            },
            "roofline": {"bound": "tensor", "kernel": "branch_gemm3m_kernel (FP64 DMMA m8n8k4, 3M complex form)",
                         "achieved": gemm_exec, "peak": f64_peak, "unit": "TFLOP/s",
                         "frac": (gemm_exec / f64_peak) if gemm_exec else None, "traffic": None,
                         "peak_source": f64_src,
                         "achieved_8mnk_convention": gemm_alg,
                         "dmma_ceiling_tflops": DMMA_CEILING,
                         "frac_of_dmma_ceiling": (gemm_exec / DMMA_CEILING) if gemm_exec else None,
                         "executed_flops_per_step": 0.75 * st["gemm_flops"],
                         "share_of_step": gemm_s / main_run["prof_step_s"] if main_run["prof_step_s"] else None,
                         "note": "achieved = executed real flops (6MNK: T1 = Ur Lr, T2 = Ui Li, T3 = (Ur+Ui)(Lr+Li)) / "
                                 "CUDA-event time of the GEMM launches in the profiling step; the 8MNK complex "
                                 "convention of SURVEY 8(d) is achieved_8mnk_convention; K is the number of frame-basis "
                                 "rows of the lower half when the frame basis applies (41,472 for C5), else the branches"},
            "roofline_sweep": {"bound": "hbm", "achieved": moved, "peak": peak, "unit": "GB/s",
                         "frac": (moved / peak) if moved else None, "traffic": traffic,
                         "achieved_algorithmic": alg,
                         "frac_algorithmic": (alg / peak) if alg else None,
                         "peak_source": peak_src, "kernel": "tile_sweep_tma_kernel",
                         "sustained_copy_gbs": copy_gbs,
                         "frac_of_sustained_copy": (moved / copy_gbs) if (moved and copy_gbs) else None,
                         "measured_in": "a separate profiling step after the timed region (CUDA events "
                                        "around every sweep launch on the launching stream)",
                         "launches": st["timed_sweeps"],
                         "bytes_per_launch": st["sweep_bytes"] / max(1, st["sweeps"]),
                         "moved_bytes_per_launch": st["sweep_bytes_moved"] / max(1, st["sweeps"]),
                         "avg_launch_us": sweep_s / max(1, st["timed_sweeps"]) * 1e6,
                         "share_of_step": sweep_s / main_run["prof_step_s"] if main_run["prof_step_s"] else None,
                         "gemm_tflops": (st["gemm_flops"] / (st["gemm_ms"] / 1e3) / 1e12)
                         if st["gemm_ms"] > 0 else None},
            "clocks": main_run["clocks"],
            "e2e": {"value": main_run["e2e"], "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": main_run["e2e_steps"]},
            "gpu_launches": main_run["launches"],
            "cpu_baseline": cpu,
            "secondary": sec,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
